"""Instructions and stall samples per source section of one file from an ncu
source page (ncu -i REP --page source --csv --print-source cuda,sass): the
file's functions and its `// ----` section comments split it; inlined helper
lines count where they are written.  Usage: ncu_functions.py <page.csv> <source file> [samples]"""
import csv
import re
import sys
from collections import defaultdict


def main():
    page, srcpath = sys.argv[1], sys.argv[2]
    nsamp = float(sys.argv[3]) if len(sys.argv) > 3 else float(1 << 26)
    base = srcpath.split("/")[-1]
    rows = list(csv.reader(open(page)))
    cur = None
    hdr = None
    agg = defaultdict(lambda: [0, 0])
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
        off = len(r) - len(hdr)
        ie = r[hdr.index("Instructions Executed") + off]
        ws = r[hdr.index("Warp Stall Sampling (All Samples)") + off]
        a = agg[(cur, ln)]
        a[0] += int(ie) if ie not in ("-", "") else 0
        a[1] += int(ws) if ws not in ("-", "") else 0
    tot = sum(v[0] for v in agg.values())
    totw = sum(v[1] for v in agg.values()) or 1
    src = open(srcpath).read().splitlines()
    marks = []
    for i, l in enumerate(src, 1):
        if (re.match(r"^(__device__|template|__global__|static|size_t|bool|int )", l) and "(" in l) or \
                l.strip().startswith("// ----"):
            marks.append((i, l.strip()[:78]))
    marks.append((len(src) + 1, "END"))
    out = []
    for (a, nm), (b, _) in zip(marks, marks[1:]):
        ins = sum(v[0] for k, v in agg.items() if k[0] == base and a <= k[1] < b)
        st = sum(v[1] for k, v in agg.items() if k[0] == base and a <= k[1] < b)
        if ins > 0.001 * tot:
            out.append((ins, st, a, nm))
    other = sum(v[0] for k, v in agg.items() if k[0] != base)
    print(f"warp-instructions (source page) {tot / 1e6:.1f} M = {32 * tot / nsamp:.1f} thread-instructions per sample; "
          f"other files (intrinsics headers) {other / 1e6:.1f} M; stall samples {totw}")
    print("   M instr      %  /sample  stall%  section")
    for ins, st, a, nm in sorted(out, key=lambda x: -x[0]):
        print(f"{ins / 1e6:10.2f} {100 * ins / tot:6.1f} {32 * ins / nsamp:8.1f} {100 * st / totw:7.1f}  L{a}: {nm}")


if __name__ == "__main__":
    main()
