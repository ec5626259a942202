"""Host-side input validation of the public API (no GPU needed): values the
device representation cannot carry raise DataError before anything is
staged, so the store is never mutated (engine.py:281-282)."""

import numpy as np
import pytest
import torch

from paper_1309_0634_b200.errors import DataError
from paper_1309_0634_b200.stream_engine import _attrs_i32, _keys_u32


def test_int64_attrs_outside_int32_raise():
    a = np.array([1, -5, 2 ** 31, 7], dtype=np.int64)
    with pytest.raises(DataError, match="tuple 2 has attr 2147483648"):
        _attrs_i32(a)
    with pytest.raises(DataError, match="tuple 0 has attr -2147483649"):
        _attrs_i32(np.array([-(2 ** 31) - 1], dtype=np.int64))
    with pytest.raises(DataError, match="tuple 1 has attr"):
        _attrs_i32(torch.tensor([0, 2 ** 40], dtype=torch.int64))


def test_int32_range_attrs_pass_unchanged():
    a = np.array([-(2 ** 31), 0, 2 ** 31 - 1], dtype=np.int64)
    out = _attrs_i32(a)
    assert out.dtype == np.int32 and out.tolist() == a.tolist()
    t = _attrs_i32(torch.tensor([-(2 ** 31), 2 ** 31 - 1], dtype=torch.int64))
    assert t.dtype == torch.int32 and t.tolist() == [-(2 ** 31), 2 ** 31 - 1]


def test_float_attrs_rejected():
    with pytest.raises(DataError):
        _attrs_i32(np.array([1.5]))
    with pytest.raises(DataError):
        _attrs_i32(torch.tensor([1.5]))


def test_wide_group_ids_raise_instead_of_wrapping():
    # 2^32 + 3 would wrap to 3 (a valid id) as u32
    with pytest.raises(DataError, match="tuple 1 has group 4294967299"):
        _keys_u32(torch.tensor([1, 2 ** 32 + 3], dtype=torch.int64), 100)
    with pytest.raises(DataError, match="tuple 0 has group -1"):
        _keys_u32(torch.tensor([-1, 5], dtype=torch.int64), 100)
    with pytest.raises(DataError, match="tuple 2 has group -7"):
        _keys_u32(np.array([0, 1, -7], dtype=np.int64), 100)
    ok = _keys_u32(torch.tensor([0, 99], dtype=torch.int64), 100)
    assert ok.dtype == torch.int32 and ok.tolist() == [0, 99]


def test_hash_lists_blocks_and_balance():
    """Static hash partitioning (stream_engine.hash_lists): a partition of
    every id, ids ascending inside each list; large domains hash blocks of 8
    consecutive ids (one 32-byte sector of each per-group array), small ones
    single ids."""
    import numpy as np
    from paper_1309_0634_b200.stream_engine import hash_lists
    for G, P, block in ((1_000_000, 148, 8), (1000, 148, 1), (100_000, 148, 8), (5000, 64, 1)):
        lists = hash_lists(G, P)
        flat = np.concatenate([np.asarray(l, dtype=np.int64) for l in lists])
        assert np.array_equal(np.sort(flat), np.arange(G))
        assert all(np.all(np.diff(l) > 0) for l in lists if len(l) > 1)
        owner = np.empty(G, dtype=np.int64)
        for p, l in enumerate(lists):
            owner[l] = p
        blocks = owner[: G // block * block].reshape(-1, block)
        assert (blocks == blocks[:, :1]).all()              # a block never straddles partitions
        if G >= 1_000_000:
            sizes = np.array([len(l) for l in lists])
            assert sizes.max() <= 1.15 * G / P
