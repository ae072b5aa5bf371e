"""Print registers / spills / smem per kernel from `nvcc -Xptxas -v` for every csrc/*.cu."""
import glob, os, re, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for f in sorted(glob.glob(os.path.join(ROOT, "paper_2007_00072_b200", "csrc", "*.cu"))):
    out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                          "-Xptxas", "-v", "-c", f, "-o", "/dev/null"], capture_output=True, text=True).stderr
    name = None
    for line in out.splitlines():
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            name = re.sub(r"\(.*", "", name).replace("enc::", "").replace("__nv_bfloat16", "bf16")
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            spill = (m.group(2), m.group(3))
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            if pat in name:
                print(f"{name:55s} regs {m.group(1):>4s} spill st/ld {spill[0]}/{spill[1]}")
            name = None
