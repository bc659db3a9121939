"""Print the last N kernel launches (name, us) of an ncu --metrics
gpu__time_duration.sum --csv launch list.  Usage: launches.py CSV [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
out = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"].replace(",", ""))
            out.append((d["Kernel Name"][:70], v / 1000.0 if d["Metric Unit"] == "ns" else v))
tot = 0.0
for name, us in out[-n:]:
    tot += us
    print("%9.1f us  %s" % (us, name))
print("%9.1f us  total of the last %d" % (tot, min(n, len(out))))
