"""Summarise an ncu --csv launch list: per kernel name (shortened), median duration,
DRAM bytes, achieved GB/s.  usage: ncu_summary.py launches.csv [skip_first_n_launches]"""
import csv, re, statistics, sys
from collections import OrderedDict, defaultdict
path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = defaultdict(dict)
names = {}
lines = [l for l in open(path) if l.startswith('"')]
for r in csv.DictReader(lines):
    i = int(r["ID"])
    names[i] = r["Kernel Name"]
    v = r["Metric Value"].replace(",", "")
    try:
        rows[i][r["Metric Name"]] = float(v)
    except ValueError:
        rows[i][r["Metric Name"]] = v
def short(n):
    n = re.sub(r"\(.*", "", n)
    n = n.replace("void ", "").replace("enc::", "").replace("__nv_bfloat16", "bf16")
    return n[:60]
agg = OrderedDict()
for i in sorted(rows):
    if i < skip: continue
    k = short(names[i])
    agg.setdefault(k, []).append(rows[i])
tot = 0.0
print(f"{'kernel':60s} {'n':>3s} {'us':>8s} {'MB':>8s} {'GB/s':>7s} {'regs':>5s}")
for k, lst in agg.items():
    t = statistics.median(x.get("gpu__time_duration.sum", 0) for x in lst) / 1e3
    b = statistics.median(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in lst)
    regs = lst[0].get("launch__registers_per_thread", "")
    tot += t * len(lst)
    print(f"{k:60s} {len(lst):3d} {t:8.1f} {b/1e6:8.1f} {b/t/1e3 if t else 0:7.0f} {regs!s:>5s}")
print("total us", round(tot, 1))
