"""Top CUDA source lines of an .ncu-rep by sampled warp stalls (needs -lineinfo).
Usage: ncu_hotlines.py report.ncu-rep [top] [kernel-regex]"""
import csv, io, subprocess, sys


def main(path, top=25, kernel=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["-k", "regex:" + kernel]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    items, tot, hdr, fname = [], 0.0, None, "?"
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        si = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            v = float(r[si] or 0)
        except ValueError:
            continue
        if v <= 0:
            continue
        tot += v
        cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        reasons = sorted(((float(r[i] or 0), h) for i, h in cols), reverse=True)[:3]
        items.append((v, f"{fname}:{r[0]}", r[1].strip()[:80], reasons))
    items.sort(reverse=True)
    print(f"== {path}: total stall samples {tot:.0f}")
    for v, loc, s, rs in items[:top]:
        rr = ", ".join(f"{n[6:]}={100*x/tot:.1f}%" for x, n in rs if x > 0)
        print(f"{100*v/tot:5.1f}% {loc:18s} {s:80s} [{rr}]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, sys.argv[3] if len(sys.argv) > 3 else None)
