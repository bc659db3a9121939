"""Summarise an ncu report (raw page) into profiles/<name>.json: per kernel
duration, DRAM bytes, instruction count, occupancy, stall breakdown."""
import csv, json, subprocess, sys

def summarize(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    hdr, units = r[0], r[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__shared_mem_per_block_dynamic",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]
    res = {}
    for vals in r[2:]:
        k = vals[hdr.index("Kernel Name")]
        d = {}
        for w in want:
            if w in hdr:
                i = hdr.index(w)
                d[w] = {"value": float(vals[i].replace(",", "")) if vals[i] else None, "unit": units[i]}
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(vals[i].replace(",", "")))
                except ValueError:
                    pass
        d["stall_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
        rb = d.get("dram__bytes_read.sum", {}).get("value") or 0
        wb = d.get("dram__bytes_write.sum", {}).get("value") or 0
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        ru = scale.get(d.get("dram__bytes_read.sum", {}).get("unit", "byte"), 1)
        wu = scale.get(d.get("dram__bytes_write.sum", {}).get("unit", "byte"), 1)
        d["dram_bytes_total"] = rb * ru + wb * wu
        res[k] = d
    json.dump(res, open(out, "w"), indent=1)
    return res

if __name__ == "__main__":
    print(json.dumps(summarize(sys.argv[1], sys.argv[2]), indent=1)[:3000])
