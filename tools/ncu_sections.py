"""Per-barrier-section instruction and stall shares of one kernel from an ncu
report (SASS source page).  Usage: ncu_sections.py <report.ncu-rep> [blocks*warps]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    nb = float(sys.argv[2]) if len(sys.argv) > 2 else 131072.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    iA, iS = h.index("Address"), h.index("Source")
    iI, iW = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[iA], 16), int(r[iI]), int(r[iW]), r[iS].strip()))
        except (ValueError, IndexError):
            pass
    base = data[0][0]
    tot = sum(d[1] for d in data)
    totw = sum(d[2] for d in data) or 1
    print(f"instructions per unit {tot / nb:.1f}  (unit = {nb:.0f}), stall samples {totw}")
    acc = accw = 0
    start = 0
    for a, n, w, s in data:
        acc += n
        accw += w
        if "BAR.SYNC" in s or "BAR.ARV" in s:
            if acc / nb > 1:
                print(f"{start:6x}-{a - base:6x} {acc / nb:8.1f} ({acc / tot * 100:5.1f}%) "
                      f"stall {accw / totw * 100:5.1f}%  {s[:36]} x{n / nb:.2f}")
            acc = accw = 0
            start = a - base + 16
    print(f"{start:6x}-end   {acc / nb:8.1f} ({acc / tot * 100:5.1f}%) stall {accw / totw * 100:5.1f}%")


if __name__ == "__main__":
    main()
