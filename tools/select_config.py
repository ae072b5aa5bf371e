#!/usr/bin/env python
"""Configuration selection on the B200 (section 6.1; SPEC.md:384-413;
paper_2007_00072_b200/config_select.py for the graph and the SSSP).

Operators are the step's operators in Table A.1 order.  Each has per-operator
configurations -- the library's alternatives for it -- and every configuration consumes and
produces data layouts:

  qkv_fwd     Q/K/V algebraic fusion (Table A.2: separate, QK stacked, QKV stacked, KV
              stacked) x contraction (cuBLASLt / hand-written tcgen05) x output layout of the
              projections (QKV in place [B,J,3,H,P], or permuted Q,K,V [3,B,H,J,P] by AIB)
  attn_fwd    QK^T + BSB + A.V: cuBLAS, tiled tcgen05, tiled + per-(b,h) A.V, fused score
              kernel (A stored), fused score kernel + per-(b,h) dropout-on-load A.V (A never
              stored); consumes the QKV layout (cuBLAS only the permuted one) and produces the
              score layout (P and A, or P and 1-bit keep words) that the backward consumes
  out_fwd, l2_fwd, l2_dw, l1_dx, l1_dw, out_dx, out_dw   cuBLASLt / tcgen05
  ffn_fwd     Linear1 + BAD: cuBLASLt + BAD kernel / fused tcgen05 kernel
  ffn_bwd     Linear2-dX + BAD-bwd: cuBLASLt + BAD-bwd kernel / fused tcgen05 kernel
  bdrln_*     BDRLN / BDRLN-bwd kernel: warps per row (row groups of 2 / 3 / 4) or one warp
              per row
  attn_bwd    the backward of the attention path the forward chose (its layout)
  qkv_bwd     Q/K/V grouping of the backward x dX contraction x dW contraction

A layout node names the tensors in HBM between operators (the QKV layout and the attention
score layout carried through the step, since the backward consumes the forward's saved
tensors -- DESIGN.md R21).  Costs: every operator's in-graph time (CUDA-graph replay with an
event-record node pair around each operator, the event overhead subtracted), measured in a
set of sweep runs that together cover every (operator, configuration).  The selection graph
keeps the cheapest configuration per (in, out) layout pair and prunes configurations without
an input and an output edge; SSSP over it gives the configuration.

Check (the paper reports "within 6 % of an ideal configuration"): the whole step of
the SSSP choice, the library default, all-cuBLASLt, all-tcgen05 and --random random valid
configurations are timed as CUDA-graph replays; the file records the SSSP choice's ratio to
the fastest measured step.
  python tools/select_config.py --config L --out profiles/r2_config_selection_L.json
"""
import argparse
import json
import os
import random
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# option keys (include/encoder.h)
O_TC, O_FUSED, O_BH, O_DIRECT, O_SIDE = 0, 1, 4, 5, 6
O_MASK, O_FUS, O_FUS_BWD, O_BDRLN = 10, 12, 13, 14
# weight-contraction operator ids (ENC_OP_*)
OPID = {"gemm_qkv": 0, "gemm_out": 5, "gemm_l1": 7, "gemm_l2": 9, "gemm_l2_dx": 12,
        "gemm_l2_dw": 13, "gemm_l1_dx": 15, "gemm_l1_dw": 16, "gemm_out_dx": 18,
        "gemm_out_dw": 19, "gemm_qkv_dx": 26, "gemm_qkv_dw": 27}
ATTN = {   # path -> (attn_tc, attn_fused, attn_bh)
    "cublas": (0, 0, 0), "tiled": (1, 0, 0), "tiled_bh": (1, 0, 1), "fused": (1, 1, 0),
    "fused_bh": (1, 1, 1)}
BDRLN_SITES = ["bdrln_fwd1", "bdrln_fwd2", "bdrln_bwd2", "bdrln_bwd1"]   # variant nibbles 0..3


def knobs_to_options(k):
    """Library options of a full knob assignment."""
    mask = 0
    for op, bit in OPID.items():
        if k.get("tc:" + op, 0):
            mask |= 1 << bit
    tc, fused, bh = ATTN[k["attn"]]
    bd = 0
    for i, s in enumerate(BDRLN_SITES):
        bd |= k.get("bd:" + s, 0) << (4 * i)
    return {O_TC: tc, O_FUSED: fused, O_BH: bh, O_DIRECT: k["direct"], O_MASK: mask,
            O_FUS: k["fus"], O_FUS_BWD: k["fus_bwd"], O_BDRLN: bd, O_SIDE: 0}


def operators(I):
    """[(operator, [(config_id, in_layout, out_layout, timed ops, knobs)])] in step order."""
    gw = [0, 1] + [g for g in (2, 3, 4) if (I // 8) % g == 0 and (I // 8) // g <= 64]
    ops = []
    cfgs = []
    for fus in range(4):
        for impl in (0, 1):
            for direct in (0, 1):
                out = "qkv=inplace" if direct else "qkv=perm"
                cfgs.append((f"fus{fus}-{'tc' if impl else 'lt'}-{'inplace' if direct else 'perm'}",
                             "X", out, ["gemm_qkv", "aib_fwd"],
                             (("fus", fus), ("tc:gemm_qkv", impl), ("direct", direct))))
    ops.append(("qkv_fwd", cfgs))
    cfgs = []
    for q in ("inplace", "perm"):
        for path in ATTN:
            if path == "cublas" and q == "inplace":
                continue   # the in-place QKV layout is read by the tcgen05 kernels only
            cfgs.append((path, f"qkv={q}", f"qkv={q}|attn={path}",
                         ["gemm_qk", "bsb_fwd", "gemm_av"], (("attn", path),)))
    ops.append(("attn_fwd", cfgs))
    lay = "*"   # pass-through: these operators keep the carried layout

    def two(op, timed, bit):
        return [(("tc" if t else "lt"), lay, lay, timed, ((bit, t),)) for t in (0, 1)]

    ops.append(("out_fwd", two("out_fwd", ["gemm_out"], "tc:gemm_out")))
    ops.append(("bdrln_fwd1", [(f"v{v}", lay, lay, ["bdrln_fwd1"], (("bd:bdrln_fwd1", v),))
                               for v in gw]))
    ops.append(("ffn_fwd", [("lt+bad", lay, lay, ["gemm_l1", "bad_fwd"], (("tc:gemm_l1", 0),)),
                            ("tc-fused", lay, lay, ["gemm_l1", "bad_fwd"],
                             (("tc:gemm_l1", 1),))]))
    ops.append(("l2_fwd", two("l2_fwd", ["gemm_l2"], "tc:gemm_l2")))
    ops.append(("bdrln_fwd2", [(f"v{v}", lay, lay, ["bdrln_fwd2"], (("bd:bdrln_fwd2", v),))
                               for v in gw]))
    ops.append(("bdrln_bwd2", [(f"v{v}", lay, lay, ["bdrln_bwd2"], (("bd:bdrln_bwd2", v),))
                               for v in gw]))
    ops.append(("ffn_bwd", [("lt+bad", lay, lay, ["gemm_l2_dx", "bad_bwd"],
                             (("tc:gemm_l2_dx", 0),)),
                            ("tc-fused", lay, lay, ["gemm_l2_dx", "bad_bwd"],
                             (("tc:gemm_l2_dx", 1),))]))
    for op, t in (("l2_dw", "gemm_l2_dw"), ("l1_dx", "gemm_l1_dx"), ("l1_dw", "gemm_l1_dw")):
        ops.append((op, two(op, [t], "tc:" + t)))
    ops.append(("bdrln_bwd1", [(f"v{v}", lay, lay, ["bdrln_bwd1"], (("bd:bdrln_bwd1", v),))
                               for v in gw]))
    for op, t in (("out_dx", "gemm_out_dx"), ("out_dw", "gemm_out_dw")):
        ops.append((op, two(op, [t], "tc:" + t)))
    cfgs = []
    for q in ("inplace", "perm"):
        for path in ATTN:
            if path == "cublas" and q == "inplace":
                continue
            cfgs.append((path, f"qkv={q}|attn={path}", f"qkv={q}|attn={path}",
                         ["gemm_av_da", "gemm_av_dv", "bsb_bwd", "gemm_qk_dq", "gemm_qk_dk",
                          "aib_bwd"], (("attn", path),)))
    ops.append(("attn_bwd", cfgs))
    cfgs = []
    for fus in range(4):
        for dx in (0, 1):
            for dw in (0, 1):
                cfgs.append((f"fus{fus}-dx{'tc' if dx else 'lt'}-dw{'tc' if dw else 'lt'}", lay,
                             "Y", ["gemm_qkv_dx", "gemm_qkv_dw"],
                             (("fus_bwd", fus), ("tc:gemm_qkv_dx", dx), ("tc:gemm_qkv_dw", dw))))
    ops.append(("qkv_bwd", cfgs))
    return ops


def default_knobs():
    k = {"attn": "fused_bh", "direct": 1, "fus": 2, "fus_bwd": 2}
    for op in OPID:
        k["tc:" + op] = 0
    k["tc:gemm_l1"] = k["tc:gemm_l2_dx"] = 1
    for s in BDRLN_SITES:
        k["bd:" + s] = 0
    return k


def sweeps(I):
    """Full knob assignments whose runs together cover every (operator, configuration)."""
    out = []
    gw = [0, 1] + [g for g in (2, 3, 4) if (I // 8) % g == 0 and (I // 8) // g <= 64]
    for fus in range(4):
        for impl in (0, 1):
            for direct in (1, 0):
                k = default_knobs()
                k["fus"] = k["fus_bwd"] = fus
                k["direct"] = direct
                for op in OPID:
                    k["tc:" + op] = impl
                k["bd:bdrln_fwd1"] = k["bd:bdrln_fwd2"] = gw[(2 * fus + impl) % len(gw)]
                k["bd:bdrln_bwd1"] = k["bd:bdrln_bwd2"] = gw[(2 * fus + impl + 1) % len(gw)]
                out.append(k)
        for dx, dw in ((0, 1), (1, 0)):   # mixed backward Q/K/V contractions
            k = default_knobs()
            k["fus_bwd"] = fus
            k["tc:gemm_qkv_dx"], k["tc:gemm_qkv_dw"] = dx, dw
            out.append(k)
    for path in ATTN:
        for direct in ((0,) if path == "cublas" else (0, 1)):
            k = default_knobs()
            k["attn"], k["direct"] = path, direct
            out.append(k)
    for v in gw:   # every BDRLN variant at every site
        k = default_knobs()
        for s in BDRLN_SITES:
            k["bd:" + s] = v
        out.append(k)
    return out


def realize(path_cfgs):
    """Knob assignment of a selected path (every configuration's knobs)."""
    k = default_knobs()
    for c in path_cfgs:
        for kk, v in c.knobs:
            k[kk] = v
    return k


def random_knobs(rng, I):
    gw = [0, 1] + [g for g in (2, 3, 4) if (I // 8) % g == 0 and (I // 8) // g <= 64]
    k = default_knobs()
    k["attn"] = rng.choice(list(ATTN))
    k["direct"] = 0 if k["attn"] == "cublas" else rng.choice([0, 1])
    k["fus"], k["fus_bwd"] = rng.randrange(4), rng.randrange(4)
    for op in OPID:
        k["tc:" + op] = rng.choice([0, 1])
    for s in BDRLN_SITES:
        k["bd:" + s] = rng.choice(gw)
    return k


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="L", choices=["L", "Bb"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--random", type=int, default=16)
    ap.add_argument("--out", default="gpurun_out/config_selection.json")
    a = ap.parse_args()
    import torch
    from paper_2007_00072_b200 import _abi, ops as eops
    from paper_2007_00072_b200.config_select import (OpConfig, build_selection_graph,
                                                     emit_configuration, select_configuration)
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    from synth import CONFIGS, make_inputs, make_params
    dims = CONFIGS[a.config]
    I = dims.H * dims.P
    lib = _abi.load()
    nops = lib.enc_num_ops()
    names = [lib.enc_op_name(i).decode() for i in range(nops)]
    inp = make_inputs(dims, "bf16")
    prm = make_params(dims, "bf16", "bench")
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ms_buf = (_abi.c_float * nops)()
    layer = EncoderLayer(dims, "bf16", LayerCfg())
    layer.set_params(prm)

    def apply(k):
        for key, v in knobs_to_options(k).items():
            eops.enc_set_option(layer.ctx, key, v)

    def step():
        layer.forward(X)
        layer.backward(X, dY)

    # tune cuBLASLt once for every shape (explicit tuning pass, then off)
    eops.enc_set_option(layer.ctx, 3, 1)
    for k in (default_knobs(),) + tuple(s for s in sweeps(I)[:24]):
        apply(k)
        step()
    torch.cuda.synchronize()
    eops.enc_set_option(layer.ctx, 3, 0)

    def graph_of():
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        return g

    def time_step(k, n):
        apply(k)
        lib.enc_set_timing(layer.ctx.ptr, 0)
        g = graph_of()
        ts = []
        for _ in range(n):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    def per_op(k):
        """In-graph per-operator times (us) under knob assignment k, event overhead removed."""
        apply(k)
        lib.enc_set_timing(layer.ctx.ptr, (1 << nops) - 1)
        g = graph_of()
        reps = {n: [] for n in names}
        for _ in range(a.reps):
            flush.zero_()
            g.replay()
            torch.cuda.synchronize()
            _abi.check("enc_op_times", lib.enc_op_times(layer.ctx.ptr, ms_buf))
            for i, n in enumerate(names):
                reps[n].append(ms_buf[i] * 1e3)
        lib.enc_set_timing(layer.ctx.ptr, 0)
        return {n: statistics.median(v) for n, v in reps.items()}

    # event-record overhead per timed operator: the whole step with every timer on vs off
    k0 = default_knobs()
    base = time_step(k0, a.steps)
    t0 = per_op(k0)
    n_timed = sum(1 for v in t0.values() if v > 0)
    apply(k0)
    lib.enc_set_timing(layer.ctx.ptr, (1 << nops) - 1)
    gt = graph_of()
    tt = []
    for _ in range(a.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gt.replay()
        e1.record()
        torch.cuda.synchronize()
        tt.append(e0.elapsed_time(e1) * 1e3)
    lib.enc_set_timing(layer.ctx.ptr, 0)
    ovh = max(0.0, (statistics.median(tt) - base) / max(n_timed, 1))
    print(f"step {base:.1f} us; {n_timed} timed ops, event overhead {ovh:.2f} us each", flush=True)

    # sweep runs -> cost of every (operator, configuration)
    op_list = operators(I)
    cost = {}
    for k in sweeps(I):
        t = per_op(k)
        for op, cfgs in op_list:
            for cid, ain, aout, timed, kn in cfgs:
                if all(k.get(kk) == v for kk, v in kn):
                    # the QKV layout a configuration consumes / produces must be the run's
                    lay = aout if op == "qkv_fwd" else ain
                    if lay.startswith("qkv=") and \
                            k["direct"] != (1 if lay.startswith("qkv=inplace") else 0):
                        continue
                    c = sum(max(t[n] - ovh, 0.0) for n in timed if t[n] > 0)
                    key = (op, cid, ain, aout)
                    cost[key] = min(cost.get(key, 1e30), c)
    rows = []
    missing = []
    for op, cfgs in op_list:
        for cid, ain, aout, timed, kn in cfgs:
            key = (op, cid, ain, aout)
            if key not in cost:
                missing.append(key)
                continue
            rows.append((op, cid, ain, aout, max(cost[key], 1e-3), kn))
    if missing:
        print("not covered by the sweeps:", missing, flush=True)
    # layouts: the carried QKV / attention layout; pass-through operators are expanded over
    # every carried layout the graph can reach
    carried = sorted({r[3] for r in rows if r[0] == "attn_fwd"})
    configs = []
    for op, cid, ain, aout, c, kn in rows:
        if ain == "*":
            for L in carried:
                configs.append(OpConfig(op, cid, L, L if aout == "*" else aout, c, kn))
        else:
            configs.append(OpConfig(op, cid, ain, aout, c, kn))
    sg = build_selection_graph([o for o, _ in op_list], configs, "X", "Y")
    path, total = select_configuration(sg)
    chosen = realize(path)
    # check: whole steps
    rng = random.Random(2007)
    cands = {"sssp": chosen, "default": default_knobs()}
    for impl, tag in ((0, "all_lt"), (1, "all_tc")):
        k = default_knobs()
        for op in OPID:
            k["tc:" + op] = impl
        cands[tag] = k
    for i in range(a.random):
        cands[f"random{i}"] = random_knobs(rng, I)
    measured = {}
    for tag, k in cands.items():
        measured[tag] = time_step(k, a.steps)
        print(f"{tag:10s} {measured[tag]:8.1f} us", flush=True)
    best = min(measured, key=measured.get)
    extra = {"workload": a.config, "chosen_knobs": chosen,
             "chosen_options": {str(k): v for k, v in knobs_to_options(chosen).items()},
             "predicted_us": total, "event_overhead_us": ovh,
             "measured_step_us": measured, "best_measured": best,
             "sssp_vs_best": measured["sssp"] / measured[best],
             "sssp_vs_default": measured["sssp"] / measured["default"],
             "operators": [o for o, _ in op_list],
             "cost_table_us": [[op, cid, ain, aout, round(c, 2)]
                               for op, cid, ain, aout, c, _kn in rows],
             "configurations": len(configs), "nodes": len(sg.nodes()),
             "edges": sum(len(e) for e in sg.edges)}
    emit_configuration(path, total, a.out, extra)
    print(f"SSSP: predicted {total:.1f} us, measured {measured['sssp']:.1f} us; best measured "
          f"{best} {measured[best]:.1f} us; ratio {measured['sssp'] / measured[best]:.3f}; "
          f"vs default {measured['sssp'] / measured['default']:.3f}", flush=True)


if __name__ == "__main__":
    main()
