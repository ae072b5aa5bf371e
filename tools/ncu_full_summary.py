#!/usr/bin/env python
"""Summarise an `ncu --set full` report: per launch the duration, DRAM bytes, achieved
GB/s, issue rate, occupancy and the warp-stall reasons above 0.5 (per issue-active cycle).
usage: ncu_full_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

BASE = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[col["Kernel Name"]].replace("void ", "").split("(")[0]
        vals = {h: r[col[h]] for h in BASE if h in col}

        def f(h):
            try:
                return float(vals.get(h, "nan").replace(",", ""))
            except ValueError:
                return float("nan")
        t_us = f("gpu__time_duration.sum")
        u = units[col["gpu__time_duration.sum"]]
        if u == "ns":
            t_us /= 1e3
        elif u == "ms":
            t_us *= 1e3
        mb = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
        ub = units[col["dram__bytes_read.sum"]]
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(ub, 1.0)
        mb *= scale
        print(f"{name}")
        print(f"  {t_us:8.2f} us  dram {mb:8.2f} MB  {mb / t_us * 1e3 if t_us else 0:7.0f} GB/s  "
              f"IPC/SM {f('sm__inst_executed.avg.per_cycle_active'):.2f}  "
              f"warp-inst {f('smsp__inst_executed.sum') / 1e6:.2f} M  "
              f"warps active {f('sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} %  "
              f"regs {vals.get('launch__registers_per_thread', '')}  "
              f"grid {vals.get('launch__grid_size', '')} x {vals.get('launch__block_size', '')}")
        st = []
        for h in stall:
            try:
                v = float(r[col[h]].replace(",", ""))
            except ValueError:
                continue
            if v > 0.5:
                st.append((h.replace("smsp__average_warps_issue_stalled_", "")
                           .replace("_per_issue_active.ratio", ""), v))
        print("  stalls: " + " ".join(f"{k}={v:.2f}" for k, v in sorted(st, key=lambda x: -x[1])))


if __name__ == "__main__":
    main()
