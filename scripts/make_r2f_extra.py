"""Summarise the extra measurement pass (scripts/gpu_r2f.sh extra ->
gpurun_out/r2f) into profiles/r2f_compare_policies.md,
r2f_partition_times.md and r2f_sanitizer.md."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = os.path.join(ROOT, "gpurun_out", "r2f")
P = os.path.join(ROOT, "profiles")


def jlines(f):
    f = os.path.join(R, f)
    if not os.path.exists(f):
        return []
    return [json.loads(l) for l in open(f) if l.startswith("{")]


md = ["# All balancer instantiations compared (round 2, final code, one B200)\n",
      "`scripts/compare_policies.py --config cN --steps 6 --warmup 12` (`scripts/gpu_r2f.sh extra`): every policy of "
      "balance.py:388-405, without and with hot-key splitting; tuples/s over 6 batches after 12 warm-up batches "
      "(CUDA events; 2 staged batches, so absolute rates sit below bench.py's), the plan's per-block max/mean load "
      "(tuples without splitting; values to store, min(count, W) per group, with it), the measured per-partition "
      "window-update time max/mean, moves per batch.\n"]
for c in ("c4", "c3"):
    rows = jlines(f"compare_{c}.log")
    if not rows:
        continue
    md += [f"## {c}\n", "| policy | split | G tuples/s | max/mean load (plan) | max/mean partition time (measured) | moves/batch |",
           "|---|---|---|---|---|---|"]
    for r in rows:
        pn = r["part_ns_max_over_mean"]
        md.append(f"| {r['policy']} | {'yes' if r['split'] else 'no'} | {r['tuples_per_s'] / 1e9:.2f} | "
                  f"{r['load_ratio_mean']:.3f} | {pn:.3f} | {r['moves_per_batch']:.1f} |" if pn is not None else
                  f"| {r['policy']} | {'yes' if r['split'] else 'no'} | {r['tuples_per_s'] / 1e9:.2f} | "
                  f"{r['load_ratio_mean']:.3f} | - | {r['moves_per_batch']:.1f} |")
    md.append("")
open(os.path.join(P, "r2f_compare_policies.md"), "w").write("\n".join(md) + "\n")

md = ["# Per-partition window-update time across the blocks (round 2, final code, one B200)\n",
      "`scripts/partition_times.py cN 12`: 12 batches of the bench config (2 staged batches), P = 148 partitions "
      "(processing units); the measured per-partition K4 time (ns, %globaltimer inside k_ingest summed over the "
      "partition's CTAs) of the last batch as a distribution over the 148 partitions, its max/mean over the last 6 "
      "batches, the per-partition work (values stored) and member counts; the plan's max/mean load for comparison.\n",
      "| config | policy | plan max/mean | part time max/mean (last 6 batches, mean / max) | part time min / p10 / median / p90 / max (us) | work max/mean | members min / median / max |",
      "|---|---|---|---|---|---|---|"]
for c in ("c1", "c2", "c3", "c4", "c5"):
    rows = jlines(f"parttimes_{c}.log")
    if not rows:
        continue
    r = rows[-1]
    t = r["part_ns"]
    m = r["members"]
    md.append(f"| {c.upper()} | {r['policy']} | {r['plan_load_ratio']:.2f} | "
              f"{r['part_ns_max_over_mean_last_half']['mean']:.2f} / {r['part_ns_max_over_mean_last_half']['max']:.2f} | "
              f"{t['min'] / 1e3:.1f} / {t['p10'] / 1e3:.1f} / {t['median'] / 1e3:.1f} / {t['p90'] / 1e3:.1f} / {t['max'] / 1e3:.1f} | "
              f"{r['part_work']['max_over_mean']:.2f} | {m['min']:.0f} / {m['median']:.0f} / {m['max']:.0f} |")
md.append("\nC2 runs the reference's group-reassignment policy alone (one group is ~10 % of the batch, so its "
          "partition carries it whole: the reference assignment is a bijection); C3-C5 add hot-key splitting, "
          "planned in values to store; C1 is the static hash with no rebalancing.\n")
open(os.path.join(P, "r2f_partition_times.md"), "w").write("\n".join(md))

md = ["# compute-sanitizer, round 2 final code (B200, scripts/gpu_r2f.sh extra)\n",
      "`scripts/sanitize_cases.py` runs the kernel families at small shapes -- the single-pass placement (sub-chunk "
      "mode), the radix passes, the look-back-free 7- and 10-bit passes, the bucketed passes, hot-key split shares, "
      "int64 keys (pipelined probe), MIN/MAX chunk summaries, the device trace and the policy kernels -- each checked "
      "against the numpy window identities.\n"]
for tool, f in (("memcheck", "memcheck.log"), ("racecheck (--racecheck-report hazard)", "racecheck.log")):
    fp = os.path.join(R, f)
    if os.path.exists(fp):
        lines = [l.rstrip() for l in open(fp) if l.startswith("ok ") or "SUMMARY" in l or "all cases" in l
                 or "Error" in l or "Hazard" in l]
        md += [f"## {tool}\n", "```", *lines[-40:], "```\n"]
open(os.path.join(P, "r2f_sanitizer.md"), "w").write("\n".join(md))
print("written")
