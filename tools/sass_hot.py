"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv --print-source sass`,
with the dominant stall reasons of each.  usage: sass_hot.py page.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ia, isrc, iall, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
data = []
tot = 0
for r in rows[2:]:
    if len(r) < len(hdr) or r[ia] == "Address":
        continue
    s = float(r[iall] or 0)
    tot += s
    st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    data.append((s, r[ia][-5:], r[isrc].strip(), r[iex], st))
print(f"total samples {tot:.0f}")
# opcode histogram (executed instructions)
from collections import Counter
ops = Counter(); samp = Counter()
for s, a, src, ex, st in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += float(ex or 0); samp[op] += s
print("opcode       executed      stall-samples")
for op, n in ops.most_common(25):
    print(f"{op:12s} {n:12.0f}  {samp[op]:8.0f}")
print()
for s, a, src, ex, st in sorted(data, reverse=True)[:top]:
    print(f"{s:7.0f} {a} {src[:60]:60s} ex={ex:>8s} " + " ".join(f"{n}:{v:.0f}" for v, n in st if v))
