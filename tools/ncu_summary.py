"""Summarise an .ncu-rep: per kernel time, DRAM bytes/throughput, occupancy, top stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
def g(r, k):
    i = col.get(k)
    return r[i] if i is not None else ""
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    name = g(r, "Kernel Name").split("(")[0].replace("unnamed>::", "")
    t = float(g(r, "gpu__time_duration.sum") or 0)
    rd = float(g(r, "dram__bytes_read.sum") or 0)
    wr = float(g(r, "dram__bytes_write.sum") or 0)
    ur = units[col["dram__bytes_read.sum"]]
    uw = units[col["dram__bytes_write.sum"]]
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    rdb, wrb = rd * scale.get(ur, 1), wr * scale.get(uw, 1)
    tu = units[col["gpu__time_duration.sum"]]
    ts = t * {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}.get(tu, 1e-3)
    st = sorted(((float(g(r, h) or 0), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for h in stalls), reverse=True)[:4]
    print(f"{name:22s} t={ts*1e6:8.1f}us dram={(rdb+wrb)/1e9:6.3f}GB ({(rdb+wrb)/ts/1e9 if ts else 0:6.0f} GB/s) "
          f"dram%={g(r,'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')[:5]} warps%={g(r,'sm__warps_active.avg.pct_of_peak_sustained_active')[:5]} "
          f"regs={g(r,'launch__registers_per_thread')} issue%={g(r,'smsp__issue_active.avg.pct_of_peak_sustained_active')[:5]} "
          f"stalls={[(n, round(v,1)) for v, n in st]}")
