"""Join an ncu SASS source page (csv) with nvdisasm -g line info: per source
line instruction counts and stall samples.  Usage:
  sass_lines.py <ncu_sass.csv> <nvdisasm -g output> <kernel mangled name> [top]"""
import csv
import re
import sys
from collections import defaultdict


def main():
    ncsv, sass, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(ncsv)))
    h = rows[1]
    iA, iI, iW = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    iS = h.index("Source")
    prof = []
    for r in rows[2:]:
        try:
            prof.append((int(r[iA], 16), int(r[iI]), int(r[iW]), r[iS].strip()))
        except (ValueError, IndexError):
            pass
    base = prof[0][0]
    # offsets -> line
    inside = False
    line = None
    off2line = {}
    for ln in open(sass):
        if ln.startswith("//-----") or ".text." in ln:
            inside = (".text." + kname) in ln
            continue
        if not inside:
            continue
        m = re.search(r'File "([^"]*)", line (\d+)', ln) if "//##" in ln else None
        if m:
            line = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r'/\*([0-9a-f]{4,})\*/', ln)
        if m and line is not None:
            off2line[int(m.group(1), 16)] = line
    agg = defaultdict(lambda: [0, 0])
    tot = totw = 0
    for a, ni, nw, src in prof:
        l = off2line.get(a - base, ('?', -1))
        agg[l][0] += ni
        agg[l][1] += nw
        tot += ni
        totw += nw
    print("total inst", tot, "stall samples", totw)
    for l, (ni, nw) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{str(l):40s} inst {ni / tot * 100:5.1f}%  stall {nw / totw * 100:5.1f}%")


if __name__ == "__main__":
    main()
