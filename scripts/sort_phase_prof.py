"""Experiment: per-phase clock64 cycles of the placement kernel (SS_SORT_PROF build).

    nvcc ... -DSS_SORT_PROF -o paper_1309_0634_b200/_lib/libss_b200_prof.so
    SS_B200_LIB=paper_1309_0634_b200/_lib/libss_b200_prof.so python scripts/sort_phase_prof.py c2
"""
import ctypes as C, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import torch
from paper_1309_0634_b200 import _lib as L
from paper_1309_0634_b200.stream_engine import StreamEngine

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
desc, kind, s, G, W, B, aggs, policy, split = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
eng = StreamEngine(G, W, n_partitions=148, aggregates=aggs, device=0, max_batch=B,
                   key_bits=64 if kind.endswith("64") else 32)
bal = eng.balancer_struct(policy, thread_threshold=max(1, B // 1480), pot=0.5, split=split)
bs = bench.make_batches(kind, s, G, B, 2, dev, 1)
lib = L.load()
fn = os.environ.get("SS_PROF_FN", "ss_debug_sort_prof")
prof = getattr(lib, fn)
prof.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
for i in range(4):
    eng.step(*bs[i % 2], bal)
out = (C.c_ulonglong * 8)()
prof(out, 1)
for i in range(6):
    eng.step(*bs[i % 2], bal)
prof(out, 1)
if fn != "ss_debug_sort_prof":
    names = ["prologue", "stage A", "scan B", "long units", "short units", "fold"]
elif os.environ.get("SS_PROF_OS"):
    names = ["tile copy wait", "zero+rank", "warp offsets", "digit scan+bases", "local scatter", "write-out"]
else:
    names = ["claim+zero", "stage+loads", "rank", "bins+publish+scan", "lookback", "scatter+write"]
tot = sum(out[i] for i in range(6))
for i, n in enumerate(names):
    print(f"{n:20s} {out[i] / 6 / 1e6:9.2f} Mcycles/step (summed over CTAs) {100 * out[i] / max(1, tot):5.1f}%")
