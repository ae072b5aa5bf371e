"""Opcode histogram per kernel from cuobjdump -sass of libencoder.so.
usage: sass_stats.py <substring of mangled name> [lib]"""
import collections, re, subprocess, sys
pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2007_00072_b200/libencoder.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, funcs = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1); funcs[cur] = []
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        funcs[cur].append(m.group(2))
for f, ops in funcs.items():
    if pat in f:
        c = collections.Counter(o.split(".")[0] for o in ops)
        print(f, "total", len(ops))
        print("  " + " ".join(f"{k}:{v}" for k, v in c.most_common(40)))
