"""Host stream source == reference generators, bit for bit (golden digests)."""

import hashlib

import numpy as np
import pytest

from paper_1309_0634_b200 import datagen as D
from paper_1309_0634_b200.errors import DataError, InvalidSpecError


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


def test_streams_match_reference(golden):
    for s in golden("streams.json")["streams"]:
        spec = D.DatasetSpec(D.DatasetKind(s["kind"]), s["n"], s["groups"],
                             s["exponent"], s["seed"])
        g, a = D.stream_for(spec).arrays()
        assert _digest(g, a) == s["digest"], s
        if "g" in s:
            assert g.tolist() == s["g"] and a.tolist() == s["a"]


def test_batches_match_reference(golden):
    for b in golden("streams.json")["batches"]:
        spec = D.DatasetSpec(D.DatasetKind.ZIPF, 150_000, 300, 1.0, 2)
        sizes, h = [], hashlib.sha256()
        for i, bt in enumerate(D.batches(D.stream_for(spec), b["batch_size"])):
            assert bt.index == i
            sizes.append(len(bt))
            h.update(np.ascontiguousarray(bt.groups, np.int64).tobytes())
        assert sizes[:5] == b["sizes_head"] and len(sizes) == b["n_batches"]
        assert sizes[-1] == b["last"] and h.hexdigest() == b["digest"]


def test_relabel_matches_reference(golden):
    r = golden("streams.json")["relabel"]
    g, a = D.relabel_groups(D.gen_zipf(3000, 40, 1.3, 8), np.asarray(r["perm"])).arrays()
    assert _digest(g, a) == r["digest"]


def test_replay_round_trip(tmp_path):
    st = D.gen_zipf(70_000, 77, 1.1, 5)
    path = tmp_path / "r.bin"
    assert D.write_replay(st, path) == 70_000
    g0, a0 = st.arrays()
    g1, a1 = D.read_replay(path).arrays()
    assert np.array_equal(g0, g1) and np.array_equal(a0, a1)
    gn, an = D.read_replay_arrays(path, 100, 50)
    assert gn.dtype == np.uint32 and an.dtype == np.int32
    assert np.array_equal(gn, g0[100:150]) and np.array_equal(an, a0[100:150])
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\x00" * 7)
    with pytest.raises(DataError):
        D.read_replay(bad)


def test_spec_validation():
    with pytest.raises(InvalidSpecError):
        D.DatasetSpec(D.DatasetKind.ZIPF, 10, 0)
    with pytest.raises(InvalidSpecError):
        D.DatasetSpec(D.DatasetKind.ZIPF, 10, 5, zipf_exponent=0)
    with pytest.raises(InvalidSpecError):
        list(D.batches(D.gen_uniform(5, 2), 0))


def test_mix64_is_bijective():
    ids = np.arange(0, 1_000_000, 997, dtype=np.int64)
    keys = D.mix64(ids)
    assert len(np.unique(keys)) == len(ids)
    assert np.array_equal(D.unmix64(keys), ids)


def test_drifting_zipf_moves_the_hot_set():
    st = D.drifting_zipf(40_000, 100, 1.5, epoch=10_000, seed=3)
    g, _ = st.arrays()
    hot = [int(np.bincount(g[i:i + 10_000], minlength=100).argmax())
           for i in range(0, 40_000, 10_000)]
    assert len(set(hot)) > 1
    g2, _ = D.drifting_zipf(40_000, 100, 1.5, epoch=10_000, seed=3).arrays()
    assert np.array_equal(g, g2)
