"""Summarise ncu --set full reports into JSON (per-launch time, DRAM traffic,
occupancy, throughput and the top stall reasons).

  python tools/ncu_summary.py out.json rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "time_us",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
             "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            if m in d and d[m] not in ("", "n/a"):
                d[m] = str(float(d[m].replace(",", "")) * scale.get(units.get(m, "").strip().lower(), 1.0))
        k = {"kernel": d.get("Kernel Name", "")}
        for m, name in WANT.items():
            v = d.get(m)
            if v is None or v == "":
                continue
            try:
                k[name] = float(v.replace(",", ""))
            except ValueError:
                k[name] = v
        unit = None
        stalls = {c: d[c] for c in hdr if c.startswith("smsp__average_warp_latency_issue_stalled_")
                  and c.endswith(".ratio")}
        top = sorted(((float(v.replace(",", "")), c.split("stalled_")[1].split(".")[0])
                      for c, v in stalls.items() if v not in ("", "n/a")), reverse=True)[:5]
        k["top_stalls_cycles_per_issue"] = {n: round(v, 2) for v, n in top}
        if "time_us" in k:
            # gpu__time_duration is reported in ns by default
            unit = d.get("gpu__time_duration.sum")
        res.append(k)
    return res


def main():
    out = sys.argv[1]
    allk = []
    for rep in sys.argv[2:]:
        allk += summarize(rep)
    json.dump(allk, open(out, "w"), indent=1)
    for k in allk:
        print(k["kernel"][:40], {x: k.get(x) for x in ("time_us", "dram_read_bytes", "dram_write_bytes", "regs")})


if __name__ == "__main__":
    main()
