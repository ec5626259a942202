"""Summarise a measurement pass (scripts/gpu_round.sh -> gpurun_out/round,
scripts/gpu_r2p.sh -> gpurun_out/round2) into profiles/: launch lists per
config, ncu --set full summaries, per-launch DRAM traffic.

    python scripts/make_profiles.py r2 round2"""
import csv, io, json, os, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
R = os.path.join(ROOT, "gpurun_out", sys.argv[2] if len(sys.argv) > 2 else "round")
P = os.path.join(ROOT, "profiles")
CONFIGS = ["c1", "c2", "c3", "c4", "c5"]


def run(*a):
    return subprocess.run(list(a), capture_output=True, text=True, cwd=ROOT).stdout


md = [f"# {tag} profiles (B200, sm_100a)\n",
      "Source: `scripts/gpu_round.sh` on one B200 (`gpurun`), summarised by",
      "`scripts/make_profiles.py`.  Launch lists: `ncu --metrics gpu__time_duration.sum",
      "--clock-control none` over `bench.py --steps 2 --warmup 3` (cold-cache, serialised",
      "launches: per-kernel SHARES carry over to the timed run, absolute times do not).",
      "Full captures: `ncu --set full --clock-control none --import-source on`,",
      "steady state (after warm-up).\n"]
for c in CONFIGS:
    f = os.path.join(R, f"launches_{c}.csv")
    if os.path.exists(f):
        shutil.copy(f, os.path.join(P, f"{tag}_launches_{c}.csv"))
        md.append(f"## Launch list per step, {c}\n\n```\n{run('python', 'scripts/launch_summary.py', f)}```\n")
traffic = {}
for c in CONFIGS:
    rep = os.path.join(R, f"full_{c}.ncu-rep")
    if not os.path.exists(rep):
        continue
    md.append(f"## ncu --set full, {c}\n\n```\n{run('python', 'scripts/ncu_summary.py', rep)}```\n")
    o = run("ncu", "-i", rep, "--page", "raw", "--csv")
    rows = list(csv.reader(io.StringIO(o)))
    h, u = rows[0], rows[1]
    d = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]

        def val(m):
            i = h.index(m)
            return float(r[i].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[i], 1)
        b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        for k, v in {"k_sort_pass": "place", "k_rank_place": "place", "k_os_pass": "place", "k_ingest": "ingest",
                     "k_count": "count", "k_key_count": "count"}.items():
            if k in name:
                d.setdefault(v, []).append(b)
    traffic[c] = {k: {"bytes_per_launch": sum(v) / len(v), "launches_captured": len(v)} for k, v in d.items()}
traffic["_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full "
                      "--clock-control none of bench.py (scripts/gpu_round.sh / gpu_r2p.sh), " + tag)
bench = ["## Bench lines (this round)\n", "```"]
for f in sorted(os.listdir(R)):
    if f.startswith("bench_") and f.endswith(".log"):
        lines = [l for l in open(os.path.join(R, f)) if l.startswith("{")]
        if lines:
            d = json.loads(lines[-1])
            bench.append(f"{f:22s} value={d.get('value', 0) / 1e9:8.3f} G/s  e2e={d.get('e2e', {}).get('value', 0) / 1e9:6.3f} G/s  "
                         f"ms/step={d.get('ms_per_step', 0) or 0:.3f}  path={d.get('path_roofline', {}).get('frac', 0):.3f}  "
                         f"load(plan)={d.get('load_ratio', {}).get('plan_mean', '-')}  "
                         f"load(part_ns)={d.get('load_ratio', {}).get('measured_part_ns_max_over_mean', '-')}")
bench.append("```\n")
md[7:7] = bench
open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(md))
json.dump(traffic, open(os.path.join(P, f"{tag}_traffic.json"), "w"), indent=1)
print("\n".join(bench))
