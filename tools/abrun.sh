# usage: bash /tmp/abrun.sh tag "args..." ; prints summary
tag=$1; shift
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/ab_$tag.log 2>&1
python - <<PY
import json
l=[x for x in open("gpurun_out/ab_$tag.log") if x.startswith("{")][-1]
d=json.loads(l); print("$tag", round(d["ms_per_step"],4), round(d["e2e"]["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), {k:v for k,v in d["per_op_us"].items() if v and k in ("gemm_qkv","bsb_fwd","gemm_l1","gemm_l2_dx","bsb_bwd")})
PY
