#!/usr/bin/env python
"""Benchmark: BERT-large encoder layer fwd+bwd (BASELINE.json config "L": B=8, J=K=512,
H=16, P=64, I=1024, U=4096, bf16) per GPU, data-parallel over N GPUs (weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, NCCL)

A step = one forward + backward of the layer over one batch of synthetic input already
resident in HBM (+ the NCCL SUM all-reduce of the parameter gradients when N > 1).
Rank 0 prints one JSON line.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BERT-large encoder layer fwd+bwd tokens/s"
METRIC_STACK = "BERT-large encoder stack fwd+bwd tokens/s"   # --layers N > 1
METRIC_TRAIN = "BERT-large encoder stack training step (fwd+bwd+AdamW) tokens/s"  # + --optimizer
UNIT = "tokens/s"
WORKLOADS = {
    "L": "L: BERT-large encoder layer B=8/GPU J=K=512 H=16 P=64 I=1024 U=4096 p=0.1 GELU",
    "Bb": "Bb: BERT-base encoder layer B=96/GPU J=K=128 H=12 P=64 I=768 U=3072 p=0.1 GELU",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["L", "Bb"], default="L",
                    help="L: the paper's BERT-large layer (headline); Bb: BERT-base layer "
                         "(BASELINE.json configs[2])")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-flush", action="store_true", help="skip the L2 flush between steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=6)  # ~13 s of oracle work
    ap.add_argument("--breakdown", action="store_true", help="print the per-op table to stderr")
    ap.add_argument("--causal", action="store_true",
                    help="causal masking of the attention scores (PAPER.md:494; decoder-style "
                         "workload on the same kernels)")
    ap.add_argument("--optimizer", action="store_true",
                    help="with --layers: AdamW update of every layer inside the step (the "
                         "full training step of BASELINE config 4)")
    ap.add_argument("--no-prefetch", action="store_true",
                    help="e2e through encoder_layer_step_host (no cross-step input prefetch)")
    ap.add_argument("--attn-overlap", type=int, default=1, choices=[0, 1],
                    help="dV contraction beside the fused dA + BSB-bwd kernel "
                         "(ENC_OPT_ATTN_OVERLAP; default on: measured -6 us/step at L)")
    ap.add_argument("--bwd-side", type=int, default=None, choices=[0, 1, 2, 3],
                    help="ENC_OPT_BWD_SIDE: 1 = weight-gradient contractions on a side stream, "
                         "2 = and the column-sum finalize on a second one, 3 = only the "
                         "finalize (default: measured fastest with PDL at L and Bb)")
    ap.add_argument("--no-qkv-direct", action="store_true",
                    help="separate AIB / AIB-bwd passes instead of the in-place QKV layout")
    ap.add_argument("--no-attn-bh", action="store_true",
                    help="AV / dV / dQ / dK on the tiled tcgen05 kernel instead of the "
                         "per-(b, h) streaming kernel")
    ap.add_argument("--attn-backend", choices=["fused", "tc", "cublas"], default="fused",
                    help="attention: fused tcgen05 score kernels (QK^T+BSB, dA+BSB-bwd), "
                         "separate tcgen05 contractions, or cuBLAS contractions")
    ap.add_argument("--layers", type=int, default=1,
                    help="encoder layers per step (24 = the BERT-large encoder stack, config 4 "
                         "of BASELINE.json; per-layer gradient all-reduce for N > 1)")
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=VALUE",
                    help="extra enc_set_option(KEY, VALUE) on the layer context (repeatable; "
                         "include/encoder.h ENC_OPT_*)")
    ap.add_argument("--eager", action="store_true",
                    help="launch every step eagerly instead of replaying a CUDA graph")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ oracle timing
def time_oracle(dims, samples: int, dtype: str):
    """The fp64 CPU oracle as it stands, on one sequence (B=1 slice) per sample."""
    import numpy as np  # noqa: F401
    from oracle import encoder as E
    from synth import make_inputs, make_params
    d1 = dims.with_batch(1)
    prm = make_params(d1, dtype, "bench")
    inp = make_inputs(d1, dtype)
    cfg = E.Cfg(act=E.ACT_GELU_ERF)
    ts = []
    for _ in range(samples):
        t0 = time.perf_counter()
        Y, sv = E.encoder_layer_forward(inp["X"], prm, d1.H, cfg)
        E.encoder_layer_backward(inp["dY"], inp["X"], prm, d1.H, cfg, sv)
        ts.append(time.perf_counter() - t0)
    return ts


def cpu_cores():
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(v):
            return int(os.environ[v])
    return os.cpu_count()


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle timed on the host cores (rank 0 only)."""
    from synth import CONFIGS
    if rank != 0:
        return
    dims = CONFIGS[args.config]
    J = dims.J
    if args.warmup:
        time_oracle(dims, min(args.warmup, 1), args.dtype)
    ts = time_oracle(dims, args.steps, args.dtype)
    total = sum(ts)
    value = args.steps * J / total
    sample = f"1 sequence (B=1 slice of config {args.config}) fwd+bwd per step, fp64 numpy oracle"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOADS[args.config], "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def gemm_desc(args) -> str:
    opts = dict(tuple(int(x) for x in kv.split("=")) for kv in args.opt)
    if args.dtype != "bf16" or opts.get(8) == 0:
        return "cuBLASLt (tuned in the first warm-up step); BAD / BAD-bwd separate kernels"
    if opts.get(8) == 1:
        return "all on the hand-written tcgen05 kernel (CTA pairs), Linear1+BAD and " \
               "Linear2-dX+BAD-bwd fused"
    return "Linear1+BAD and Linear2-dX+BAD-bwd: hand-written fused tcgen05 kernels; plain " \
           "contractions: cuBLASLt (tuned in the first warm-up step) -- the measured selection"


def attention_desc(args, dims) -> str:
    backend = args.attn_backend
    if backend == "fused" and not (dims.J in (128, 512) and dims.P == 64 and args.dtype == "bf16"):
        backend = "tc" if args.dtype == "bf16" else "cublas"   # what the library selects
    opts = dict(tuple(int(x) for x in kv.split("=")) for kv in args.opt)
    if backend == "fused" and dims.J == 512 and opts.get(21, 1) and opts.get(15, 1):
        return ("fused tcgen05 QK^T+BSB+A.V (S in TMEM, A = keep*P written over it as the A.V "
                "operand) / dC.V^T+BSB-bwd (dA in TMEM, row term from C), dropout on load in "
                "A^T.dC, dS.K + dS^T.Q per (b,h)")
    return {"fused": "fused tcgen05 QK^T+BSB / dA+BSB-bwd (S, dA in TMEM), dropout on load in "
                     "the per-(b,h) A.V / A^T.dC contractions",
            "tc": "tcgen05 QK^T / dA contractions + separate BSB kernels, per-(b,h) A.V, "
                  "A^T.dC, dS.K + dS^T.Q",
            "cublas": "cuBLAS contractions + separate BSB kernels"}[backend]


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.bwd_side is None:
        args.bwd_side = 3   # with PDL: weight-gradient GEMMs on the main stream (a side stream
        # measured 1-2 % slower at L and Bb), only the last column-sum finalize beside them
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    from paper_2007_00072_b200 import _abi, dp, tally
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    from paper_2007_00072_b200.stack import EncoderStack
    from synth import CONFIGS, SEED_WEIGHTS, make_inputs, make_params

    # one process per GPU; ENC_DIST_BACKEND=gloo (test hook) lets several ranks share one GPU
    backend = os.environ.get("ENC_DIST_BACKEND", "nccl")
    local_dev = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    dims_global = CONFIGS[args.config].with_batch(CONFIGS[args.config].B * world)
    boff, B = dp.shard(dims_global.B, world, rank)
    dims = CONFIGS[args.config].with_batch(B)
    es = 2 if args.dtype == "bf16" else 4
    tdt = torch.bfloat16 if args.dtype == "bf16" else torch.float32

    cfg = LayerCfg(p_attn=0.1, p_hidden=0.1, p_ffn=0.1, act="gelu", batch_offset=boff,
                   causal=args.causal)
    stack = None
    if args.layers > 1:
        stack = EncoderStack(args.layers, dims, args.dtype, cfg)
        stack.set_params([make_params(dims, args.dtype, "bench", seed=SEED_WEIGHTS + i)
                          for i in range(args.layers)])
        layer = stack.layers[0]     # the layers share one context (options, timing, counts)
    else:
        layer = EncoderLayer(dims, args.dtype, cfg)
        layer.set_params(make_params(dims, args.dtype, "bench"))
    _abi.check("enc_set_option", _abi.load().enc_set_option(
        layer.ctx.ptr, 0, int(args.attn_backend in ("tc", "fused"))))
    _abi.check("enc_set_option", _abi.load().enc_set_option(
        layer.ctx.ptr, 1, int(args.attn_backend == "fused")))
    _abi.check("enc_set_option", _abi.load().enc_set_option(layer.ctx.ptr, 4, int(not args.no_attn_bh)))
    _abi.check("enc_set_option", _abi.load().enc_set_option(layer.ctx.ptr, 5,
                                                            int(not args.no_qkv_direct)))
    _abi.check("enc_set_option", _abi.load().enc_set_option(layer.ctx.ptr, 6,
                                                            int(args.bwd_side)))
    _abi.check("enc_set_option", _abi.load().enc_set_option(layer.ctx.ptr, 7,
                                                            int(args.attn_overlap)))
    for kv in args.opt:
        k, v = (int(x) for x in kv.split("="))
        _abi.check("enc_set_option", _abi.load().enc_set_option(layer.ctx.ptr, k, v))
    inp = make_inputs(dims_global, args.dtype)
    X = torch.tensor(inp["X"][boff:boff + B], device=dev).to(tdt)
    dY = torch.tensor(inp["dY"][boff:boff + B], device=dev).to(tdt)
    Y = torch.empty_like(X)
    dX = torch.empty_like(X)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    lib = _abi.load()
    nops = lib.enc_num_ops()
    names = [lib.enc_op_name(i).decode() for i in range(nops)]
    ms_buf = (_abi.c_float * nops)()

    # The step as a list of (device work, gradient buckets all-reduced right after it).
    # Data parallel: every all-reduce is issued as soon as its gradients are final and
    # overlaps the rest of the backward: one layer -> the FFN bucket after
    # the FFN half of the backward, the attention bucket after the rest; a stack -> each
    # layer's gradients after that layer's backward.
    if stack is None:
        if world > 1:
            parts = [(lambda: (layer.forward(X, None, Y),
                               layer.backward(X, dY, dX, part=layer.BWD_FFN)),
                      [layer.ffn_bucket]),
                     (lambda: layer.backward(X, dY, dX, part=layer.BWD_ATTN),
                      [layer.attn_bucket])]
        else:
            parts = [(lambda: (layer.forward(X, None, Y), layer.backward(X, dY, dX)), [])]
    elif world > 1:
        def bwd_layer(i):
            src = dY if i == args.layers - 1 else stack.grads_io[(i + 1) % 2]
            return lambda: stack.layers[i].backward(stack.acts[i], src, stack.grads_io[i % 2])
        parts = [(lambda: stack.forward(X), [])]
        parts += [(bwd_layer(i), [stack.layers[i].grad_flat])
                  for i in reversed(range(args.layers))]
    else:
        parts = [(lambda: (stack.forward(X), stack.backward(dY)), [])]

    # a training step of the stack: AdamW on every layer once its gradients are reduced
    post = []
    if stack is not None and args.optimizer:
        stack.init_optimizer()
        post = [stack.optimizer_step]

    def run_parts(fns, post_fns):
        works = []
        for fn, (_f, buckets) in zip(fns, parts):
            fn()
            if world > 1 and buckets:
                works += dp.allreduce_buckets(buckets, async_op=True)
        for w in works:
            w.wait()
        for fn in post_fns:
            fn()

    def step():
        run_parts([f for f, _b in parts], post)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # the first warm-up step is the explicit tuning pass of the cuBLASLt contractions (the
    # paper's "benchmark every algorithm"): ENC_OPT_GEMM_AUTOTUNE on for it,
    # off afterwards, so no timed or captured call measures, allocates or synchronises
    _abi.check("enc_set_option", lib.enc_set_option(layer.ctx.ptr, 3, 1))
    for i in range(args.warmup):
        step()
        if i == 0:
            torch.cuda.synchronize()
            _abi.check("enc_set_option", lib.enc_set_option(layer.ctx.ptr, 3, 0))
    barrier()

    # per-operator breakdown pass (all ops timed; not the timed region).  Run with the
    # side-stream overlaps off so every op's events bracket only its own kernels (an op on
    # the side stream would otherwise include its wait for the fused kernel beside it).
    set_opt = lambda k, v: _abi.check("enc_set_option", lib.enc_set_option(  # noqa: E731
        layer.ctx.ptr, k, v))
    set_opt(6, 0)
    set_opt(7, 0)
    lib.enc_set_timing(layer.ctx.ptr, (1 << nops) - 1)
    per_op = {n: [] for n in names}
    for _ in range(3):
        if not args.no_flush:
            flush.zero_()
        step()
        torch.cuda.synchronize()
        _abi.check("enc_op_times", lib.enc_op_times(layer.ctx.ptr, ms_buf))
        for i, n in enumerate(names):
            per_op[n].append(ms_buf[i])
    per_op = {n: statistics.median(v) for n, v in per_op.items()}
    set_opt(6, int(args.bwd_side))
    set_opt(7, int(args.attn_overlap))
    tc_path = args.attn_backend in ("fused", "tc") and args.dtype == "bf16"
    # which kernels run (layer defaults; --opt overrides): A not stored with dropout on load,
    # A.V inside the score kernel (R30) and the BSB-bwd row term from C (R26) at J = 512
    opts = dict(tuple(int(x) for x in kv.split("=")) for kv in args.opt)
    fa = args.attn_backend == "fused" and args.dtype == "bf16"
    on_load = fa and not args.no_attn_bh
    j512 = dims.J == 512 and dims.P == 64
    dc = on_load and j512 and opts.get(15, 1) != 0
    fused = tally.fused_bytes(dims, es, fused_attn=fa, direct=tc_path and not args.no_qkv_direct,
                              a_stored=not on_load, dc_term=dc,
                              fused_av=dc and opts.get(21, 1) != 0)
    flops = tally.gemm_flops(dims)
    dominant = max(per_op, key=per_op.get)
    dom_id = names.index(dominant)
    lib.enc_set_timing(layer.ctx.ptr, 1 << dom_id)
    l0 = lib.enc_launch_count(layer.ctx.ptr)
    for fn, _b in parts:
        fn()
    per_step_launches = lib.enc_launch_count(layer.ctx.ptr) - l0

    # ---------------- CUDA graphs of the step, one per part (one graph for N = 1); events of
    # the timed op (enabled above) are captured as event-record nodes of the graph; the
    # eager NCCL all-reduce issued after a part overlaps the replay of the next ones
    if not args.eager:
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for fn in [f for f, _b in parts] + post:
                fn()
        torch.cuda.current_stream(dev).wait_stream(side)
        graphs, post_graphs = [], []
        for fn, dst in [(f, graphs) for f, _b in parts] + [(f, post_graphs) for f in post]:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            dst.append(g)
        torch.cuda.synchronize()

        def step():  # noqa: F811
            run_parts([g.replay for g in graphs], [g.replay for g in post_graphs])
        for _ in range(2):
            step()
        torch.cuda.synchronize()

    # ---------------- timed region
    sampler = ClockSampler(local_dev)
    sampler.start()
    barrier()
    launches0 = lib.enc_launch_count(layer.ctx.ptr)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    dom_ms = []
    t_wall = time.perf_counter()
    for k in range(args.steps):
        if not args.no_flush:
            flush.zero_()
        ev[k][0].record()
        step()
        ev[k][1].record()
        torch.cuda.synchronize()
        _abi.check("enc_op_times", lib.enc_op_times(layer.ctx.ptr, ms_buf))
        dom_ms.append(ms_buf[dom_id])
    barrier()
    t_wall = time.perf_counter() - t_wall
    launches = lib.enc_launch_count(layer.ctx.ptr) - launches0
    if not args.eager:   # graph replays launch the captured kernels; count them per step
        launches = per_step_launches * args.steps
    clocks = sampler.stop()
    step_ms = sum(a.elapsed_time(b) for a, b in ev)
    step_ms = dp.max_over_ranks(step_ms, dev)
    ms_per_step = step_ms / args.steps
    tokens = dims_global.B * dims_global.J
    value = tokens / (ms_per_step * 1e-3)

    # ---------------- roofline of the dominant kernel
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_src = "measured"
    except OSError:
        peak_src = "fallback"
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    tc_peak = peaks.get("bf16_tflops_sustained", 1400.0)
    dom_avg_ms = statistics.mean(dom_ms)
    if dominant in fused:
        ach = fused[dominant] / (dom_avg_ms * 1e-3) / 1e9
        roof = {"kernel": dominant, "bound": "hbm", "achieved": ach, "peak": hbm_peak,
                "unit": "GB/s", "frac": ach / hbm_peak, "traffic": None,
                "algorithmic_bytes": fused[dominant], "peak_source": peak_src}
    else:
        ach = flops[dominant] / (dom_avg_ms * 1e-3) / 1e12
        if args.dtype == "fp32":
            tc_peak = tc_peak / 2.0 * 0.5   # no TF32: fp32 runs on CUDA cores (context only)
        roof = {"kernel": dominant, "bound": "tensor", "achieved": ach, "peak": tc_peak,
                "unit": "TFLOP/s", "frac": ach / tc_peak, "traffic": None,
                "algorithmic_flops": flops[dominant], "peak_source": peak_src + " (sustained)"}
    if stack is not None:   # the layers share the context's events: the last instance
        roof["instance"] = "last launch of the step (layer 0's backward / layer {}'s forward)" \
            .format(args.layers - 1)
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    # the committed ncu traffic figures are per launch at config L, bf16, default path
    if os.path.exists(traffic_path) and args.config == "L" and args.dtype == "bf16" \
            and args.attn_backend == "fused":
        try:
            roof["traffic"] = json.load(open(traffic_path)).get(dominant)
        except (OSError, ValueError):
            pass

    # ---------------- every operator's in-graph duration and roofline fraction: the step is
    # captured once more with event-record nodes around every operator (all timing bits
    # on) and replayed; fused ops against the HBM peak (algorithmic bytes, tally.py),
    # contractions against the tensor peak (flops).  Not the timed region.
    op_graph_us, op_frac = {}, {}
    if not args.eager and world == 1 and stack is None:
        lib.enc_set_timing(layer.ctx.ptr, (1 << nops) - 1)
        set_opt(6, 0)   # side-stream overlap off: each op's events bracket only its kernels
        g_all = torch.cuda.CUDAGraph()
        s_all = torch.cuda.Stream(dev)
        s_all.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s_all):
            run_parts([f for f, _b in parts], post)
        torch.cuda.current_stream(dev).wait_stream(s_all)
        with torch.cuda.graph(g_all):
            run_parts([f for f, _b in parts], post)
        reps = {n: [] for n in names}
        for _ in range(5):
            if not args.no_flush:
                flush.zero_()
            g_all.replay()
            torch.cuda.synchronize()
            _abi.check("enc_op_times", lib.enc_op_times(layer.ctx.ptr, ms_buf))
            for i, n in enumerate(names):
                reps[n].append(ms_buf[i])
        for n in names:
            t = statistics.median(reps[n])
            if t <= 0 or per_op[n] < 0:
                continue
            op_graph_us[n] = round(t * 1e3, 2)
            if n in fused and fused[n]:
                op_frac[n] = {"bound": "hbm", "frac": round(fused[n] / (t * 1e-3) / 1e9 / hbm_peak, 3)}
            elif n in flops:
                op_frac[n] = {"bound": "tensor",
                              "frac": round(flops[n] / (t * 1e-3) / 1e12 / tc_peak, 3)}
        set_opt(6, int(args.bwd_side))
        lib.enc_set_timing(layer.ctx.ptr, 1 << dom_id)
        del g_all

    # ---------------- end to end through the C ABI with host buffers
    Xh = X.cpu().pin_memory()
    dYh = dY.cpu().pin_memory()
    Yh = torch.empty_like(Xh).pin_memory()
    dXh = torch.empty_like(Xh).pin_memory()
    lib.enc_set_timing(layer.ctx.ptr, 0)
    if stack is not None:
        def host_step():
            stack.step_host(Xh, dYh, Yh, dXh)
            if post and world == 1:   # the training step's AdamW (N > 1: after the reduce)
                for fn in post:
                    fn()
        e2e_buckets = [lay.grad_flat for lay in stack.layers]
        e2e_api = (f"EncoderStack.step_host ({args.layers} layers"
                   + (" + AdamW" if post else "") + "; ")
    else:
        def host_step():
            layer.step_host(Xh, dYh, Yh, dXh, X, dY, Y, dX)
        e2e_buckets = [layer.ffn_bucket, layer.attn_bucket]
        e2e_api = "encoder_layer_step_host ("
    pipelined = stack is None and not args.no_prefetch
    g_e2e = None
    if pipelined:
        # a training loop over host batches: encoder_layer_step_host_pipelined prefetches
        # step s+1's X, dY during step s and copies Y, dX back during step s+1; device
        # buffers double-buffered; every step's copies are inside the timed region
        Xd, dYd = [X, torch.empty_like(X)], [dY, torch.empty_like(dY)]
        Yd, dXd = [Y, torch.empty_like(Y)], [dX, torch.empty_like(dX)]

        def pstep(a, nxt, first=False):
            # step of buffer parity a: next inputs into parity a^1, previous dX (a^1) out
            b = a ^ 1
            layer.step_host_pipelined(Xd[a], dYd[a], Yd[a], dXd[a], Yh,
                                      Xh if nxt else None, dYh if nxt else None, Xd[b], dYd[b],
                                      None if first else dXd[b], None if first else dXh)
            if world > 1:
                dp.allreduce_buckets(e2e_buckets)

        def last_dx(n):   # the loop's last dX copy
            dXh.copy_(dXd[(n - 1) & 1], non_blocking=True)

        def host_loop_eager(n):
            layer.prefetch_inputs(Xh, dYh, Xd[0], dYd[0])
            for i in range(n):
                pstep(i & 1, i + 1 < n, first=(i == 0))
            last_dx(n)
        host_loop_eager(4)
        torch.cuda.synchronize()
        g_pair = None
        if not args.eager and world == 1:
            # a pair of steps (parities 0, 1; each copying the next inputs in and the
            # previous dX out) captured as one graph; every call joins its copies, so the
            # replays chain in stream order
            g_pair = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_pair):
                pstep(0, True)
                pstep(1, True)
            g_pair.replay()
            torch.cuda.synchronize()

        def host_loop(n):
            if g_pair is None:
                host_loop_eager(n)
                return
            # first steps eager (no previous dX; the pair graph starts at parity 0), pairs
            # of steps that both copy next inputs from the graph, the last steps eager
            layer.prefetch_inputs(Xh, dYh, Xd[0], dYd[0])
            pstep(0, n > 1, first=True)
            i = 1
            if i < n - 1:
                pstep(1, True)
                i = 2
            while i + 2 < n:
                g_pair.replay()
                i += 2
            while i < n:
                pstep(i & 1, i + 1 < n)
                i += 1
            last_dx(n)
    else:
        for _ in range(2):
            host_step()
        torch.cuda.synchronize()
        # the call captured once in a CUDA graph (its copies from / to pinned host memory and
        # the copy-stream fork / join included) and replayed per step, like the device timing
        if not args.eager:
            g_e2e = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_e2e):
                host_step()
            g_e2e.replay()
            torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if pipelined:
        host_loop(args.steps)
    else:
        for _ in range(args.steps):
            if g_e2e is not None:
                g_e2e.replay()
            else:
                host_step()
            if world > 1:
                dp.allreduce_buckets(e2e_buckets)
                for fn in post:
                    fn()
    e1.record()
    barrier()
    e2e_ms = dp.max_over_ranks(e0.elapsed_time(e1), dev) / args.steps
    if pipelined:
        how = ("encoder_layer_step_host_pipelined (H2D X, dY of step s+1 from pinned host "
               "memory during step s; D2H Y of step s and dX of step s-1 on the copy-out "
               "stream; the loop's first input copy and last dX copy included), "
               + ("pairs of steps replayed as a CUDA graph" if g_pair is not None else "eager"))
    else:
        how = (e2e_api + "H2D X, dY from pinned host memory; D2H Y, dX) "
               + ("replayed as a CUDA graph" if g_e2e is not None else "eager"))
    e2e = {"value": tokens / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": 2 * X.numel() * es, "d2h_bytes_per_step": 2 * X.numel() * es,
           "ms_per_step": e2e_ms, "how": how}

    if args.breakdown and rank == 0:
        for n in names:
            extra = ""
            if n in fused:
                extra = f"{fused[n] / (per_op[n] * 1e-3) / 1e9:8.0f} GB/s"
            elif n in flops:
                extra = f"{flops[n] / (per_op[n] * 1e-3) / 1e12:8.1f} TF/s"
            print(f"  {n:14s} {per_op[n] * 1e3:9.1f} us  {extra}", file=sys.stderr)

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cd = CONFIGS[args.config]
            ts = time_oracle(cd, args.cpu_samples if args.config == "L" else 4 * args.cpu_samples,
                             args.dtype)
            cpu = {"value": cd.J * len(ts) / sum(ts), "unit": UNIT,
                   "cores": cpu_cores(), "kind": "oracle",
                   "sample": f"{len(ts)} x one sequence (B=1 slice of config {args.config}) "
                             f"fwd+bwd, fp64 numpy oracle, {sum(ts):.1f} s"}
        line = {
            "metric": METRIC if stack is None else (METRIC_TRAIN if post else METRIC_STACK),
            "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config] if stack is None
                       else f"Lx{args.layers}: {args.layers}-layer encoder stack of "
                            + WORKLOADS[args.config],
                       "layers": args.layers, "global_batch": dims_global.B,
                       "causal": bool(args.causal),
                       "optimizer": "AdamW (fp32 master, moments; one launch per layer)"
                       if post else None,
                       "seq_len": dims.J,
                       "parallelism": f"dp{world}",
                       "l2": "flushed (512 MB write) between steps" if not args.no_flush
                       else "not flushed", "graph": "eager launches" if args.eager
                       else f"CUDA graph replay (fwd+bwd, {len(parts)} graph(s) per step)",
                       "attention": attention_desc(args, dims),
                       "weight_contractions": gemm_desc(args),
                       "bwd_side_stream": {0: "none", 1: "dW", 2: "dW + finalize",
                                           3: "finalize"}.get(args.bwd_side, args.bwd_side),
                       "options": args.opt or None},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks, "wall_s_timed_region": t_wall,
            # ops fused away on this path (no launch of their own) are null
            "per_op_graph_us": op_graph_us or None, "rooflines": op_frac or None,
            "per_op_us": {n: (round(per_op[n] * 1e3, 2) if per_op[n] >= 0 else None)
                          for n in names},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


if __name__ == "__main__":
    main()
