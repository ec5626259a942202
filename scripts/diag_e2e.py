"""Per-step wall times of the streaming e2e loop (diagnostic)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1309_0634_b200.stream_engine import StreamEngine
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
desc, kind, s, G, W, B, aggs, policy, split = bench.CONFIGS[name]
dev = torch.device('cuda', 0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
eng = StreamEngine(G, W, n_partitions=148, aggregates=aggs, max_batch=B, initial='hash',
                   key_bits=64 if kind.endswith('64') else 32)
eng.set_stream(st)
bal = eng.balancer_struct(policy, B // 1480, 0.5, split=split)
bs = bench.make_batches(kind, s, G, B, 2, dev, 7)
hosts = []
for g, a in bs:
    hg = torch.empty(B, dtype=g.dtype, pin_memory=True); hg.copy_(g)
    ha = torch.empty(B, dtype=torch.int32, pin_memory=True); ha.copy_(a)
    hosts.append((hg, ha))
for i in range(4):
    eng.step(*bs[i % 2], bal, sync=False)
torch.cuda.synchronize()
eng.set_host_emit(True)
t = [time.perf_counter()]
for i in range(10):
    eng.step(*hosts[i % 2], bal, sync=False)
    t.append(time.perf_counter())
    if i:
        eng.results_pull()
    t.append(time.perf_counter())
eng.results_pull()
torch.cuda.synchronize()
t.append(time.perf_counter())
d = np.diff(t) * 1e3
print(name, "step/pull ms:", np.round(d, 2).tolist())
