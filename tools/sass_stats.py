#!/usr/bin/env python
"""Blackwell-native evidence from the built library's SASS (cuobjdump -sass): per kernel,
the count of tcgen05 MMA (UTC*MMA, incl. the .2CTA pair form), tcgen05 commits (UTCBAR),
TMEM loads / stores (LDTM / STTM), TMA loads / stores (UTMALDG / UTMASTG), bulk copies
(UBLKCP) and legacy tensor-core MMA (HMMA, which must be absent).
usage: sass_stats.py [libencoder.so] [out.txt]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTCHMMA", "UTCHMMA.2CTA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMALDG.2CTA",
       "UTMASTG", "UBLKCP", "HMMA"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return out.stdout.splitlines() if out.returncode == 0 else names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2007_00072_b200",
                                                             "libencoder.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                          check=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(1)
        base = op.split(".")[0]
        if base in ("UTCHMMA", "UTMALDG"):
            per[cur][base + (".2CTA" if ".2CTA" in op else "")] += 1
        elif base in ("UTCBAR", "LDTM", "STTM", "UTMASTG", "UBLKCP", "HMMA"):
            per[cur][base] += 1
    names = demangle(list(per))
    lines = [f"{'kernel':70s} " + " ".join(f"{o:>12s}" for o in OPS)]
    for (fn, cnt), nm in zip(per.items(), names):
        if not any(cnt.values()):
            continue
        nm = nm.replace("(anonymous namespace)::", "").split("(")[0]
        nm = nm if len(nm) <= 70 else nm[:67] + "..."
        lines.append(f"{nm:70s} " + " ".join(f"{cnt.get(o, 0):12d}" for o in OPS))
    tot = collections.Counter()
    for c in per.values():
        tot.update(c)
    lines.append(f"{'TOTAL':70s} " + " ".join(f"{tot.get(o, 0):12d}" for o in OPS))
    out = "\n".join(lines)
    print(out)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(out + "\n")


if __name__ == "__main__":
    main()
