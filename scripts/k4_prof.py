"""Phase breakdown of the window update (k_ingest) at one config.

Needs a build with -DSS_K4_PROF loaded through SS_B200_LIB (thread 0 of every
CTA adds clock64 deltas per phase into g_k4_prof):
  nvcc <flags> -DSS_K4_PROF engine.cu -o _lib/libss_k4prof.so
  SS_B200_LIB=.../libss_k4prof.so python scripts/k4_prof.py --config c4
Phases: 0 loop head, 1 stage members (A), 2 scans (B), 3 long units,
4 short members, 5 fold into the per-group accumulators.
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1309_0634_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=10)
args = ap.parse_args()
ns = argparse.Namespace(batch=0, sub_batch=0, initial="hash", config=args.config)
dev = torch.device("cuda:0")
st = torch.cuda.Stream()
wl = bench.Workload(args.config, ns, dev, 1, 0, bench.P_DEFAULT, st)
lib = _lib.load()
f = lib.ss_debug_k4_prof
f.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
for i in range(8):
    wl.step(i)
torch.cuda.synchronize()
f(buf, 1)
for i in range(args.steps):
    wl.step(8 + i)
torch.cuda.synchronize()
f(buf, 0)
tot = sum(buf[i] for i in range(6)) or 1
names = ["head", "stage(A)", "scans(B)", "long units", "short members", "fold"]
for i in range(6):
    print(f"{names[i]:16s} {buf[i] / args.steps / 1e3:12.1f} kcyc/step  {100.0 * buf[i] / tot:5.1f} %")
wl.close()
