"""Summarise an ncu --set full report (raw page) into profiles/: per kernel
time, DRAM bytes (and B/param for a known N), DRAM %, regs, occupancy.

  ncu -i REPORT --page raw --csv > raw.csv
  python tools/ncu_summary.py raw.csv N out.txt [traffic.json]
"""
import csv
import json
import sys

raw, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
traffic_path = sys.argv[4] if len(sys.argv) > 4 else None
rows = list(csv.reader(open(raw)))
hdr = rows[0]
col = {k: hdr.index(k) for k in hdr}
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]
lines = [f"# ncu --set full --clock-control none; N = {n} params; one launch per row",
         "kernel | time_us | dram_read_GB | dram_write_GB | B/param | dram%peak | regs | warps_active% | grid x block"]
traffic = json.load(open(traffic_path)) if traffic_path else {}
units = rows[1]
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
    def g(k):
        return r[col[k]] if k in col else "?"
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd = float(g("dram__bytes_read.sum")) * scale.get(units[col["dram__bytes_read.sum"]], 1.0)
    wr = float(g("dram__bytes_write.sum")) * scale.get(units[col["dram__bytes_write.sum"]], 1.0)
    bpp = (rd + wr) / n
    lines.append(f"{name} | {g('gpu__time_duration.sum')} | {rd/1e9:.4f} | {wr/1e9:.4f} | {bpp:.2f} | "
                 f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | {g('launch__registers_per_thread')} | "
                 f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')} | {g('launch__grid_size')} x {g('launch__block_size')}")
    traffic[name.split("<")[0].strip()] = {"dram_bytes_per_param": bpp, "source": out}
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
if traffic_path:
    json.dump(traffic, open(traffic_path, "w"), indent=1)
