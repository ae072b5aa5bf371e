#!/usr/bin/env python
"""Per-launch table of an ncu CSV launch list (--csv --log-file) of one layer step: kernel,
duration, DRAM bytes and bandwidth (fraction of the measured HBM peak), tensor-pipe activity
(sm__pipe_tensor_cycles_active, % of elapsed; sm__inst_executed_pipe_tc, % of peak) and the
tensor-memory activity (sm__mem_tensor_cycles_active), plus each kernel's share of the step.
usage: ncu_launches.py launches.csv [out.txt]"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = {"gpu__time_duration.sum": "t", "dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr",
     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tc",
     "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active": "tci",
     "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tmem"}
SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}


def main():
    txt = open(sys.argv[1]).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    launches = {}
    order = []
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        if key not in launches:
            launches[key] = {}
            order.append(key)
        name = r["Metric Name"]
        if name in M:
            v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
            launches[key][M[name]] = v
    tot = sum(launches[k].get("t", 0.0) for k in order)
    lines = [f"{'kernel':60s} {'us':>7s} {'share':>6s} {'MB':>7s} {'GB/s':>7s} {'HBM%':>5s} "
             f"{'tc%':>5s} {'tcI%':>5s} {'tmem%':>6s}"]
    for k in order:
        d = launches[k]
        t = d.get("t", 0.0)
        mb = (d.get("rd", 0.0) + d.get("wr", 0.0)) / 1e6
        gbs = mb * 1e6 / (t * 1e-6) / 1e9 if t else 0.0
        nm = k[1].replace("void ", "").split("(")[0]
        nm = (nm[:57] + "...") if len(nm) > 60 else nm
        lines.append(f"{nm:60s} {t:7.2f} {100 * t / tot:5.1f}% {mb:7.1f} {gbs:7.0f} "
                     f"{100 * gbs / peak:4.0f}% {d.get('tc', 0):5.1f} {d.get('tci', 0):5.1f} "
                     f"{d.get('tmem', 0):6.1f}")
    lines.append(f"total {tot:.1f} us over {len(order)} launches (serialised, cold caches); "
                 f"HBM% of the measured {peak} GB/s")
    out = "\n".join(lines)
    print(out)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(out + "\n")


if __name__ == "__main__":
    main()
