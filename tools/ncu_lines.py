"""Per-source-line instructions and stall samples from an ncu report's
source page (ncu -i REP --page source --csv --print-source cuda,sass).
Usage: ncu_lines.py <cs.csv> [top N] [phase spec name:file:first-last,...]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    cur = None
    agg = defaultdict(lambda: [0, 0, ""])
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or r[0] == "Function Name":
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        # source text may carry unescaped quotes: index the metrics from the end
        off = len(r) - len(hdr)
        ie = r[hdr.index("Instructions Executed") + off]
        ws = r[hdr.index("Warp Stall Sampling (All Samples)") + off]
        a = agg[(cur, ln)]
        a[0] += int(ie) if ie not in ("-", "") else 0
        a[1] += int(ws) if ws not in ("-", "") else 0
        a[2] = r[1][:90]
    tot_i = sum(v[0] for v in agg.values())
    tot_w = sum(v[1] for v in agg.values())
    print(f"total warp-instructions {tot_i}  stall samples {tot_w}")
    if len(sys.argv) > 3:
        for item in sys.argv[3].split(","):
            nm, f, rng = item.split(":")
            lo, hi = (int(v) for v in rng.split("-"))
            i = sum(v[0] for k, v in agg.items() if k[0] == f and lo <= k[1] <= hi)
            w = sum(v[1] for k, v in agg.items() if k[0] == f and lo <= k[1] <= hi)
            print(f"{nm:12s} inst {i:>11d} ({100 * i / tot_i:5.1f}%)  stalls {w:>7d} ({100 * w / max(tot_w, 1):5.1f}%)")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0]}:{k[1]:<5d} inst {v[0]:>10d} ({100 * v[0] / tot_i:4.1f}%) stalls {v[1]:>6d}  {v[2]}")


if __name__ == "__main__":
    main()
