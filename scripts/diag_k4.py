"""Per-partition K4 time and work for a config (diagnostic, GPU box)."""
import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1309_0634_b200.stream_engine import StreamEngine
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
desc, kind, s, G, W, B, aggs, policy, split = bench.CONFIGS[name]
dev = torch.device('cuda', 0)
eng = StreamEngine(G, W, n_partitions=148, aggregates=aggs, max_batch=B, initial='hash')
bal = eng.balancer_struct(policy, B // 1480, 0.5, split=split)
bs = bench.make_batches(kind, s, G, B, 2, dev, 7)
for i in range(8):
    g, a = bs[i % 2]
    rep = eng.step(g, a, bal)
ns = eng.last_part_ns()
work = eng.last_part_work()
g2t, lists = eng.get_lists()
sizes = np.array([len(l) for l in lists])
loads = eng.last_loads()
o = np.argsort(-ns)[:8]
print(json.dumps({"cfg": name, "ratio": rep.load_ratio, "ns_max": int(ns.max()), "ns_med": int(np.median(ns)),
                  "work_max": int(work.max()), "work_med": int(np.median(work)), "work_sum": int(work.sum()),
                  "top": [[int(p), int(ns[p]), int(sizes[p]), int(loads[p]), int(work[p])] for p in o],
                  "members_max": int(sizes.max()), "members_med": int(np.median(sizes))}))
