"""Summaries of gpurun_out job files: bench JSON lines and ncu launch lists."""
import csv
import json
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    if f.endswith(".json"):
        for ln in open(f):
            if ln.startswith("{"):
                d = json.loads(ln)
                if "config" not in d:
                    print(f, d)
                    continue
                r = d.get("roofline") or {}
                print(f, d["config"].get("name"), "value", round(d["value"], 1), "enc", round(d.get("encode_ms", 0), 4),
                      "dec", round(d.get("decode_ms", 0), 4), "frac enc/dec",
                      round((r.get("encode") or {}).get("frac", 0), 3), round((r.get("decode") or {}).get("frac", 0), 3),
                      "ratio", round(d.get("ratio", 0), 4), "launches", d.get("gpu_launches"))
    elif f.endswith(".csv"):
        rows = list(csv.reader([l for l in open(f) if not l.startswith("==")]))
        if not rows:
            continue
        h = rows[0]
        ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
        d = defaultdict(dict)
        for r in rows[1:]:
            d[(int(r[iid]), r[ik][:48])][r[im]] = r[iv]
        for k, v in sorted(d.items())[-int(sys.argv[0] == "" or 6):]:
            print(k, {kk.split("__")[1] if "__" in kk else kk: vv for kk, vv in v.items()})
