"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel:
launches, total us, share.  Usage: launch_summary.py launches.csv [skip_first_n]"""
import csv, sys, collections


def main(path, skip=0):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r["Metric Unit"]))
    rows = rows[skip:]
    agg = collections.OrderedDict()
    for name, v, u in rows:
        us = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(u, v)
        short = name.split("(")[0][:60]
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    # our kernels only (torch's data generation is not part of a step);
    # steps = launches of the count kernel
    agg = {k: v for k, v in agg.items() if "at::" not in k and "at_cuda_detail" not in k}
    steps = max(1, max((v[0] for k, v in agg.items() if "k_count" in k), default=1))
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':60s} {'n':>5s} {'us/step':>9s} {'avg_us':>9s} {'share':>6s}   ({steps} steps)")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:60s} {n:5d} {us / steps:9.2f} {us / n:9.2f} {us / tot:6.1%}")
    print(f"{'TOTAL per step':60s} {len(rows):5d} {tot / steps:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
