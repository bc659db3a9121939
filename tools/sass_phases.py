"""Per-phase instruction / stall attribution of an ncu SASS source page:
instructions of inlined helpers are charged to the last kernel-body line
seen before them in address order.  Usage:
  sass_phases.py <ncu_sass.csv> <nvdisasm -g output> <kernel mangled name> <src basename> <body_first_line>
                 <phase spec: name:first-last,...>"""
import csv
import re
import sys
from collections import defaultdict


def main():
    ncsv, sass, kname, base, body0, spec = sys.argv[1:7]
    body0 = int(body0)
    phases = []
    for item in spec.split(","):
        nm, rng = item.split(":")
        a, b = rng.split("-")
        phases.append((nm, int(a), int(b)))
    rows = list(csv.reader(open(ncsv)))
    h = rows[1]
    iA, iI, iW = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    prof = []
    for r in rows[2:]:
        try:
            prof.append((int(r[iA], 16), int(r[iI]), int(r[iW])))
        except (ValueError, IndexError):
            pass
    pbase = prof[0][0]
    inside = False
    cur = None
    off2line = {}
    for ln in open(sass):
        if ln.startswith("//-----") or ".text." in ln:
            inside = (".text." + kname) in ln
            continue
        if not inside:
            continue
        if "//##" in ln:
            m = re.search(r'File "([^"]+)", line (\d+)', ln)
            if m and m.group(1).endswith(base) and int(m.group(2)) >= body0:
                cur = int(m.group(2))
            continue
        m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
        if m and cur is not None:
            off2line[int(m.group(1), 16)] = cur
    agg = defaultdict(lambda: [0, 0])
    tot = totw = 0
    for a, ni, nw in prof:
        l = off2line.get(a - pbase, -1)
        nm = "other"
        for (p, lo, hi) in phases:
            if lo <= l <= hi:
                nm = p
                break
        agg[nm][0] += ni
        agg[nm][1] += nw
        tot += ni
        totw += nw
    print("total inst", tot, "stall samples", totw)
    for nm, (ni, nw) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{nm:12s} inst {ni / tot * 100:5.1f}% ({ni / 1e6:7.1f}M)  stall {nw / totw * 100:5.1f}%")


if __name__ == "__main__":
    main()
