"""Whole-layer parity: encoder_layer_forward / encoder_layer_backward through the C ABI vs
the fp64 oracle on the same seeded inputs.

* fp32 path (TF32 off): end to end against the oracle, configs T and the paper's BERT-large
  layer L at full size, 1e-5 normwise relative (R14).
* bf16 path: stage by stage (R14) -- every stage's GPU output against the oracle
  stage applied to the GPU's own stored bf16 inputs of that stage (forward from the saved
  set, backward from the saved set and the backward temporaries), so the check isolates the
  implementation from the conditioning of bf16 storage; end-to-end bf16 errors are printed.
"""
import numpy as np
import pytest
import torch

from keepbits import decode
from oracle import encoder as E
from oracle import philox
from synth import CONFIGS, Dims, bf16_round, make_inputs, make_params
from tol import assert_parity, assert_parity_e2e, e2e_report, errors

pytestmark = pytest.mark.gpu

ACT = {"gelu": E.ACT_GELU_ERF, "gelu_tanh": E.ACT_GELU_TANH, "relu": E.ACT_RELU}
TDT = {"bf16": torch.bfloat16, "fp32": torch.float32}


def f64(t):
    return t.float().cpu().numpy().astype(np.float64)


# option ids of include/encoder.h (enc_set_option)
OPT_ATTN_TC, OPT_ATTN_FUSED, OPT_ATTN_BH, OPT_QKV_DIRECT, OPT_GEMM_TC = 0, 1, 4, 5, 8
OPT_GEMM_PAIR, OPT_GEMM_TC_MASK = 9, 10


def _ffn_fused(dtype, opts=None):
    """bf16 with ENC_OPT_GEMM_TC on (default): Linear1 + BAD and Linear2-dX + BAD-bwd run as
    one tcgen05 kernel each (dA1 is never written)."""
    o = opts or {}
    if OPT_GEMM_TC_MASK in o:
        return dtype == "bf16" and bool(o[OPT_GEMM_TC_MASK] >> 12 & 1)   # ENC_OP_GEMM_L2_DX
    return dtype == "bf16" and bool(o.get(OPT_GEMM_TC, 1))


def _paths(dims, dtype, opts=None):
    """Which attention path the library takes for these dims / options (mirrors api.cu)."""
    o = {OPT_ATTN_TC: 1, OPT_ATTN_FUSED: 1, OPT_ATTN_BH: 1, OPT_QKV_DIRECT: 1}
    o.update(opts or {})
    tc = bool(o[OPT_ATTN_TC]) and dtype == "bf16" and dims.P == 64 and dims.J % 128 == 0
    fused = tc and bool(o[OPT_ATTN_FUSED]) and dims.J in (128, 512)
    bh = bool(o[OPT_ATTN_BH]) and dims.P == 64 and dims.J % 128 == 0 and dims.J <= 512
    return {"tc": tc, "fused": fused, "drop_on_load": fused and bh}


def _setup(dims, dtype, act, key_padding, p=0.1, batch_offset=0, layer_id=0, weight_std=0.02,
           opts=None, causal=False):
    from paper_2007_00072_b200 import ops
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    prm = make_params(dims, dtype, "parity", weight_std=weight_std)
    inp = make_inputs(dims, dtype, key_padding=key_padding)
    cfg = LayerCfg(p_attn=p, p_hidden=p, p_ffn=p, act=act, layer_id=layer_id,
                   batch_offset=batch_offset, causal=causal)
    layer = EncoderLayer(dims, dtype, cfg)
    for key, val in (opts or {}).items():
        ops.enc_set_option(layer.ctx, key, val)
    layer.set_params(prm)
    X = torch.tensor(inp["X"], device="cuda").to(TDT[dtype])
    dY = torch.tensor(inp["dY"], device="cuda").to(TDT[dtype])
    M = None if inp["mask_bias"] is None else torch.tensor(inp["mask_bias"], device="cuda")
    Y = layer.forward(X, M)
    dX = layer.backward(X, dY)
    torch.cuda.synchronize()
    ocfg = E.Cfg(p_attn=p, p_hidden=p, p_ffn=p, act=ACT[act], layer_id=layer_id,
                 batch_offset=batch_offset, causal=causal)
    return layer, prm, inp, ocfg, f64(Y), f64(dX)


def _end_to_end(dims, dtype, act, key_padding, **kw):
    layer, prm, inp, ocfg, Y, dX = _setup(dims, dtype, act, key_padding, **kw)
    Yo, sv = E.encoder_layer_forward(inp["X"], prm, dims.H, ocfg, inp["mask_bias"])
    dXo, go, _ = E.encoder_layer_backward(inp["dY"], inp["X"], prm, dims.H, ocfg, sv)
    gpu = {"Y": Y, "dX": dX}
    ref = {"Y": Yo, "dX": dXo}
    for n in go:
        gpu["d" + n] = f64(layer.grads[n])
        ref["d" + n] = go[n]
    s = layer.saved_views()
    for n in ("Q", "K", "V", "P", "A", "C", "X1", "xhat1", "A1", "xhat2", "rstd1", "rstd2"):
        if n == "A" and _drop_on_load(dims, dtype):
            continue   # A = dropout(P) is never stored on this path
        gpu["saved." + n] = f64(s[n])
        ref["saved." + n] = sv[n]
    gpu["saved.h"] = f64(s["h"])
    ref["saved.h"] = sv["h"]
    return gpu, ref


def _drop_on_load(dims, dtype, opts=None):
    """The fused score kernels + per-(b,h) contractions (bf16, J = K = 512, P = 64) never
    store A: A.V and A^T.dC apply the stored keep bits to P on load."""
    return _paths(dims, dtype, opts)["drop_on_load"]


def _stagewise(dims, dtype, act, key_padding, opts=None, **kw):
    """(gpu, ref) pairs of every stage, the oracle fed with the GPU's stored inputs."""
    layer, prm, inp, ocfg, Y, dX = _setup(dims, dtype, act, key_padding, opts=opts, **kw)
    B, J, H, P, I = dims.B, dims.J, dims.H, dims.P, dims.I
    sub = lambda site: 4 * ocfg.layer_id + site  # noqa: E731
    sc, boff, seed = 1.0 / np.sqrt(P), ocfg.batch_offset, ocfg.seed
    W = {k: np.asarray(v, np.float64) for k, v in prm.items()}
    X = np.asarray(inp["X"], np.float64)
    dY = np.asarray(inp["dY"], np.float64)
    s = {k: f64(v) for k, v in layer.saved_views().items()
         if k != "keep_attn" and not (k == "A" and _drop_on_load(dims, dtype, opts))}
    # temporaries a fused kernel keeps on chip are never written: not read back
    unwritten = ({"dA"} if _paths(dims, dtype, opts)["fused"] else set()) | \
        ({"dA1"} if _ffn_fused(dtype, opts) else set())
    b = {k: f64(v) for k, v in layer.bwd_views().items() if k not in unwritten}
    g = {k: f64(v) for k, v in layer.grads.items()}
    pairs = []
    # ---- forward
    QKV = X @ W["Wqkv"].T
    Qo, Ko, Vo = E.aib_fwd(QKV, W["bqkv"], H, P)
    pairs += [("Q", s["Q"], Qo), ("K", s["K"], Ko), ("V", s["V"], Vo)]
    S = s["Q"] @ s["K"].transpose(0, 1, 3, 2)
    if dtype == "bf16" and not _paths(dims, dtype, opts)["fused"]:
        # the unfused paths store S in bf16 between the contraction and BSB: the BSB
        # stage's input is that stored S (the fused kernel keeps S in fp32 TMEM)
        S = bf16_round(S.astype(np.float32)).astype(np.float64)
    Po, Ao = E.bsb_fwd(S, inp["mask_bias"], sc, ocfg.p_attn, seed, sub(0), boff,
                       causal=ocfg.causal)
    pairs += [("P", s["P"], Po)]
    if _drop_on_load(dims, dtype, opts):
        # A is not stored: the contraction uses keep(P) * s from the stored P
        keep = philox.keep_mask_tensor((B, H, J, J), boff, ocfg.p_attn, seed, sub(0))
        s["A"] = np.where(keep, s["P"] * philox.dropout_scale(ocfg.p_attn), 0.0)
    else:
        pairs += [("A", s["A"], Ao)]
    Co = (s["A"] @ s["V"]).transpose(0, 2, 1, 3).reshape(B, J, I)
    pairs += [("C", s["C"], Co)]
    X1o, xh1o, r1o = E.bdrln_fwd(s["C"] @ W["Wo"].T, W["bo"], X, W["g1"], W["be1"],
                                 ocfg.ln_eps, ocfg.p_hidden, seed, sub(1), boff)
    pairs += [("X1", s["X1"], X1o), ("xhat1", s["xhat1"], xh1o)]
    pairs += [("h", s["h"], s["X1"] @ W["W1"].T + W["b1"])]
    # A1 from the stored activation input h (the fused epilogue computes it from h rounded)
    _, A1o = E.bad_fwd(s["h"], np.zeros_like(W["b1"]), ocfg.act, ocfg.p_ffn, seed, sub(2), boff)
    pairs += [("A1", s["A1"], A1o)]
    Yo, xh2o, r2o = E.bdrln_fwd(s["A1"] @ W["W2"].T, W["b2"], s["X1"], W["g2"], W["be2"],
                                ocfg.ln_eps, ocfg.p_hidden, seed, sub(3), boff)
    pairs += [("Y", Y, Yo), ("xhat2", s["xhat2"], xh2o)]
    fp32_pairs = [("rstd1", s["rstd1"], r1o), ("rstd2", s["rstd2"], r2o)]
    # ---- backward
    dz2o, dY2o, dg2o, dbe2o, db2o = E.bdrln_bwd(dY, s["xhat2"], s["rstd2"], W["g2"],
                                                ocfg.p_hidden, seed, sub(3), boff)
    pairs += [("dY2", b["dY2"], dY2o), ("dg2", g["g2"], dg2o), ("dbe2", g["be2"], dbe2o),
              ("db2", g["b2"], db2o)]
    pairs += [("dW2", g["W2"], np.einsum("bji,bju->iu", b["dY2"], s["A1"]))]
    if _ffn_fused(dtype, opts):
        # Linear2-dX + BAD-bwd in one kernel: dA1 stays in TMEM
        dA1 = b["dY2"] @ W["W2"]
    else:
        pairs += [("dA1", b["dA1"], b["dY2"] @ W["W2"])]
        dA1 = b["dA1"]
    dho, db1o = E.bad_bwd(dA1, s["h"], ocfg.act, ocfg.p_ffn, seed, sub(2), boff)
    pairs += [("dh", b["dh"], dho), ("db1", g["b1"], db1o)]
    pairs += [("dX1", b["dX1"], b["dh"] @ W["W1"] + dz2o),
              ("dW1", g["W1"], np.einsum("bju,bji->ui", b["dh"], s["X1"]))]
    dz1o, dYoo, dg1o, dbe1o, dboo = E.bdrln_bwd(b["dX1"], s["xhat1"], s["rstd1"], W["g1"],
                                                ocfg.p_hidden, seed, sub(1), boff)
    pairs += [("dYo", b["dYo"], dYoo), ("dg1", g["g1"], dg1o), ("dbe1", g["be1"], dbe1o),
              ("dbo", g["bo"], dboo)]
    pairs += [("dC", b["dC"], b["dYo"] @ W["Wo"]),
              ("dWo", g["Wo"], np.einsum("bji,bjk->ik", b["dYo"], s["C"]))]
    dCbh = b["dC"].reshape(B, J, H, P).transpose(0, 2, 1, 3)
    dAo = dCbh @ s["V"].transpose(0, 1, 3, 2)
    pairs += [("dV", b["dV"], s["A"].transpose(0, 1, 3, 2) @ dCbh)]
    if _paths(dims, dtype, opts)["fused"]:
        # fused kernels: the forward's stored keep-flag words are the oracle's mask exactly
        kb = layer.saved_views()["keep_attn"].cpu().numpy()
        assert np.array_equal(decode(kb, J), philox.keep_mask_tensor(
            (B, H, J, J), boff, ocfg.p_attn, seed, sub(0))), "attention keep bits"
        # fused dC V^T + BSB-bwd kernel: dA never leaves TMEM; dS from the fp64 product
        pairs += [("dS", b["dS"], E.bsb_bwd(dAo, s["P"], sc, ocfg.p_attn, seed, sub(0), boff))]
    else:
        pairs += [("dA", b["dA"], dAo)]
        pairs += [("dS", b["dS"], E.bsb_bwd(b["dA"], s["P"], sc, ocfg.p_attn, seed, sub(0),
                                            boff))]
    pairs += [("dQ", b["dQ"], b["dS"] @ s["K"]),
              ("dK", b["dK"], b["dS"].transpose(0, 1, 3, 2) @ s["Q"])]
    dQKVo, dbqkvo = E.aib_bwd(b["dQ"], b["dK"], b["dV"])
    pairs += [("dQKV", b["dQKV"], dQKVo), ("dbqkv", g["bqkv"], dbqkvo)]
    # Table A.2 variants with several Q/K/V groups accumulate dX group by group onto the
    # bf16 dX buffer (one rounding per group): the reference follows the same sequence
    groups = {0: [(0, 1), (1, 1), (2, 1)], 1: [(0, 2), (2, 1)], 3: [(0, 1), (1, 2)]}.get(
        (opts or {}).get(12, 2), [(0, 3)])
    dXref = dz1o
    if dtype == "bf16" and len(groups) > 1:   # dz1 is stored in the bf16 dX buffer first
        dXref = bf16_round(dXref.astype(np.float32)).astype(np.float64)
    for gi, (s0, c) in enumerate(groups):
        blk = slice(s0 * I, (s0 + c) * I)
        dXref = dXref + b["dQKV"][..., blk] @ W["Wqkv"][blk]
        if dtype == "bf16" and len(groups) > 1 and gi + 1 < len(groups):
            dXref = bf16_round(dXref.astype(np.float32)).astype(np.float64)
    pairs += [("dX", dX, dXref),
              ("dWqkv", g["Wqkv"], np.einsum("bjo,bji->oi", b["dQKV"], X))]
    return pairs, fp32_pairs


@pytest.mark.parametrize("act", ["gelu", "relu", "gelu_tanh"])
def test_layer_T_fp32(act):
    gpu, ref = _end_to_end(CONFIGS["T"], "fp32", act, key_padding=True, weight_std=0.2)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


def test_layer_T_fp32_batch_offset_and_layer_id():
    gpu, ref = _end_to_end(CONFIGS["T"], "fp32", "gelu", key_padding=False, batch_offset=6,
                           layer_id=7, weight_std=0.2)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


@pytest.mark.parametrize("key_padding", [False, True])
def test_layer_T_fp32_causal(key_padding):
    """The masking step (R22) end to end on the fp32 path."""
    gpu, ref = _end_to_end(CONFIGS["T"], "fp32", "gelu", key_padding=key_padding,
                           weight_std=0.2, causal=True)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


@pytest.mark.parametrize("fusion", [0, 1, 3])
def test_layer_T_fp32_qkv_fusion_variants(fusion):
    """Table A.2's algebraic-fusion variants of the Q/K/V projections
    compute the same layer: end to end at 1e-5 on the fp32 path."""
    gpu, ref = _end_to_end(CONFIGS["T"], "fp32", "gelu", key_padding=True, weight_std=0.2,
                           opts={12: fusion})
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


def test_layer_T_fp32_no_dropout():
    gpu, ref = _end_to_end(CONFIGS["T"], "fp32", "gelu", key_padding=True, p=0.0,
                           weight_std=0.2)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


def test_layer_L_fp32_full():
    """The paper's BERT-large layer (B=8, J=K=512, H=16, P=64, I=1024, U=4096) end to end
    on the fp32 path at full size: every output and saved tensor within 1e-5 normwise."""
    gpu, ref = _end_to_end(CONFIGS["L"], "fp32", "gelu", key_padding=True)
    for n in gpu:
        e = errors(gpu[n], ref[n])
        print(f"{n:14s} max_rel {e['max_rel']:.3e}")
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


@pytest.mark.parametrize("dims,act,kp", [
    (Dims(B=2, J=64, H=4, P=16, U=256), "gelu", True),      # cuBLAS attention path
    (Dims(B=3, J=40, H=2, P=24, U=96), "relu", True),       # cuBLAS attention path
    (Dims(B=2, J=256, H=4, P=64, U=1024), "gelu", True),    # tcgen05 attention path
    (Dims(B=2, J=512, H=2, P=64, U=512), "gelu", True),     # fused score kernels
    (Dims(B=3, J=128, H=12, P=64, U=3072), "gelu", True),   # BERT-base shape (config Bb)
])
def test_layer_small_bf16_stagewise(dims, act, kp):
    pairs, f32 = _stagewise(dims, "bf16", act, kp, weight_std=0.06)
    for n, g, o in pairs:
        assert_parity(n, g, o, "bf16")
    for n, g, o in f32:   # rstd of the bf16-rounded GEMM output: bf16-level agreement
        assert_parity(n, g, o, "bf16")


@pytest.mark.parametrize("opts", [
    {OPT_ATTN_BH: 0},                      # fused score kernels + tiled A.V (A stored)
    {OPT_QKV_DIRECT: 0},                   # fused + per-(b,h) with separate AIB passes
    {OPT_ATTN_FUSED: 0},                   # tiled QK^T + BSB kernels + per-(b,h)
    {OPT_ATTN_FUSED: 0, OPT_ATTN_BH: 0},   # all tiled tcgen05
    {OPT_ATTN_TC: 0},                      # cuBLAS attention
    {OPT_GEMM_TC: 0},                      # weight contractions on cuBLASLt, BAD separate
    {OPT_GEMM_TC_MASK: (1 << 7) | (1 << 12)},   # only the fused FFN kernels on tcgen05
    {OPT_GEMM_PAIR: 0},                    # single-CTA weight-contraction tiles
    {11: 1},                               # keep words generated ahead on the side stream
    {12: 0},                               # Table A.2: Q, K, V as separate contractions
    {12: 1},                               # Table A.2: Q and K stacked, V separate
    {12: 3},                               # Q, then K and V stacked (P:646 variant)
    {12: 0, 8: 1},                         # separate, all on the tcgen05 kernel
    {14: 0x1111},                          # BDRLN / BDRLN-bwd one warp per row
    {14: 0x4242},                          # BDRLN row groups of 2 / 4 warps per site
    {14: 0x5555},                          # wide row-group BDRLN kernels (8 groups per CTA)
])
def test_layer_bf16_stagewise_paths(opts):
    """Every attention-path option combination at a fused-capable shape (J = 512)."""
    pairs, f32 = _stagewise(Dims(B=2, J=512, H=2, P=64, U=512), "bf16", "gelu", True,
                            opts=opts, weight_std=0.06)
    for n, g, o in pairs + f32:
        assert_parity(n, g, o, "bf16")


@pytest.mark.parametrize("opts", [
    None,                                  # short-row fused score kernels, dropout on load
    {OPT_ATTN_BH: 0},                      # short-row fused kernels + tiled A.V (A stored)
    {OPT_ATTN_FUSED: 0},                   # tiled QK^T + BSB kernels + per-(b,h)
    {11: 1},                               # keep words generated ahead on the side stream
])
def test_layer_bf16_stagewise_paths_short(opts):
    """The attention-path options at the short-row shape J = 128 (config Bb's J, P)."""
    pairs, f32 = _stagewise(Dims(B=3, J=128, H=4, P=64, U=512), "bf16", "gelu", True,
                            opts=opts, weight_std=0.06)
    for n, g, o in pairs + f32:
        assert_parity(n, g, o, "bf16")


@pytest.mark.parametrize("dims,opts", [
    (Dims(B=2, J=512, H=2, P=64, U=512), None),               # fused score kernels
    (Dims(B=2, J=512, H=2, P=64, U=512), {OPT_ATTN_FUSED: 0}),  # tiled QK^T + BSB kernel
    (Dims(B=3, J=128, H=4, P=64, U=512), None),               # short-row fused kernels
    (Dims(B=3, J=128, H=4, P=64, U=512), {OPT_ATTN_FUSED: 0}),  # short-row tiled BSB
    (Dims(B=2, J=64, H=4, P=16, U=256), None),                # cuBLAS attention path
])
def test_layer_bf16_stagewise_causal(dims, opts):
    """Causal masking (R22) stage by stage on every attention path."""
    pairs, f32 = _stagewise(dims, "bf16", "gelu", True, opts=opts, weight_std=0.06, causal=True)
    for n, g, o in pairs + f32:
        assert_parity(n, g, o, "bf16")


def test_layer_L_bf16_stagewise():
    """Config L, bf16, every stage vs the oracle on the GPU's stored inputs."""
    pairs, f32 = _stagewise(CONFIGS["L"], "bf16", "gelu", key_padding=False)
    for n, g, o in pairs:
        e = errors(g, o)
        print(f"{n:8s} mixed {e['mixed']:.3e} mean_rel {e['mean_rel']:.3e}")
    for n, g, o in pairs:
        assert_parity(n, g, o, "bf16")
    for n, g, o in f32:   # rstd of the bf16-rounded GEMM output: bf16-level agreement
        assert_parity(n, g, o, "bf16")


def test_layer_L_bf16_end_to_end():
    """The north-star target: the paper's BERT-large layer (config L) in bf16, forward and
    backward end to end against the fp64 oracle on the same seeded inputs -- the output,
    dX, all twelve parameter gradients and every saved activation (tests/tol.py
    assert_parity_e2e: mean relative <= 5e-3 and max error within the bf16 element bound,
    or no larger than bf16 storage alone causes)."""
    import bf16_model
    dims = CONFIGS["L"]
    gpu, ref = _end_to_end(dims, "bf16", "gelu", key_padding=False)
    prm = make_params(dims, "bf16", "parity", weight_std=0.02)
    inp = make_inputs(dims, "bf16", key_padding=False)
    mod = bf16_model.layer(inp["X"], prm, dims.H, E.Cfg(p_attn=0.1, p_hidden=0.1, p_ffn=0.1),
                           inp["mask_bias"], dY=inp["dY"])
    failed = []
    for n in sorted(gpu):
        if n not in mod:
            continue
        rep = e2e_report(gpu[n], ref[n], mod[n])
        print(f"{n:14s} gpu: mixed {rep['gpu']['mixed']:.3f} mean_rel {rep['gpu']['mean_rel']:.2e}"
              f" | model: mixed {rep['model']['mixed']:.3f} mean_rel "
              f"{rep['model']['mean_rel']:.2e} | rms ratio {rep['rms_ratio']:.3f} max ratio "
              f"{rep['max_ratio']:.3f}")
        try:
            assert_parity_e2e(n, gpu[n], ref[n], mod[n])
        except AssertionError as ex:
            failed.append(str(ex))
    assert not failed, "\n".join(failed)


def test_backward_halves_equal_full_backward():
    """encoder_layer_backward_part(FFN) then (ATTN) == encoder_layer_backward, bitwise."""
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    dims = Dims(B=2, J=256, H=4, P=64, U=1024)
    prm = make_params(dims, "bf16", "parity", weight_std=0.06)
    inp = make_inputs(dims, "bf16", key_padding=True)
    layer = EncoderLayer(dims, "bf16", LayerCfg())
    layer.set_params(prm)
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    M = torch.tensor(inp["mask_bias"], device="cuda")
    layer.forward(X, M)
    dX_full = layer.backward(X, dY).clone()
    g_full = layer.grad_flat.clone()
    layer.grad_flat.zero_()
    dX = layer.backward(X, dY, part=layer.BWD_FFN)
    dX = layer.backward(X, dY, dX=dX, part=layer.BWD_ATTN)
    torch.cuda.synchronize()
    assert torch.equal(dX, dX_full)
    assert torch.equal(layer.grad_flat, g_full)


@pytest.mark.parametrize("graph", [False, True])
def test_attn_overlap_option_bitwise(graph):
    """ENC_OPT_ATTN_OVERLAP (dV on the side stream beside the fused dA + BSB-bwd kernel)
    changes only the schedule: dX and every gradient are bitwise those of the sequential
    backward, eager and graph-captured."""
    from paper_2007_00072_b200 import ops
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    dims = Dims(B=2, J=512, H=4, P=64, U=1024)
    prm = make_params(dims, "bf16", "parity", weight_std=0.05)
    inp = make_inputs(dims, "bf16")
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    out = []
    for ov in (0, 1):
        layer = EncoderLayer(dims, "bf16", LayerCfg())
        ops.enc_set_option(layer.ctx, ops.OPT_ATTN_OVERLAP, ov)
        layer.set_params(prm)
        layer.forward(X)
        dX = layer.backward(X, dY).clone()
        if graph:
            dXg = torch.empty_like(X)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                layer.forward(X)
                layer.backward(X, dY, dXg)
            layer.grad_flat.zero_()
            g.replay()
            torch.cuda.synchronize()
            dX = dXg.clone()
        torch.cuda.synchronize()
        out.append((dX.cpu(), layer.grad_flat.cpu()))
    assert torch.equal(out[0][0], out[1][0])
    assert torch.equal(out[0][1], out[1][1])


@pytest.mark.parametrize("dtype,dims,variant", [
    ("bf16", Dims(B=2, J=512, H=4, P=64, U=1024), 0),        # row-group BDRLN kernels
    ("bf16", Dims(B=2, J=512, H=4, P=64, U=1024), 0x1111),   # one warp per row at every site
    ("bf16", Dims(B=2, J=512, H=4, P=64, U=1024), 0x5555),   # wide row-group kernels
    ("bf16", Dims(B=3, J=128, H=2, P=64, U=264), 0),         # U % 32 != 0: ragged keep words
    ("fp32", Dims(B=2, J=16, H=2, P=8, U=64), 0),            # fp32: BDRLN bytes, BAD separate
])
def test_mask_bytes_option_bitwise(dtype, dims, variant):
    """ENC_OPT_MASK_BYTES (R27): the forward stores the BDRLN / BAD keep flags as
    bytes and the backward reads them instead of re-running Philox -- Y, dX and every
    gradient are bitwise those of the regenerating backward (the masks are the same)."""
    from paper_2007_00072_b200 import ops
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    prm = make_params(dims, dtype, "parity", weight_std=0.05)
    inp = make_inputs(dims, dtype, key_padding=True)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    X = torch.tensor(inp["X"], device="cuda").to(tdt)
    dY = torch.tensor(inp["dY"], device="cuda").to(tdt)
    M = torch.tensor(inp["mask_bias"], device="cuda")
    out = []
    for mb, ahead in ((0, 0), (1, 0), (1, 1)):   # (1, 1): bytes drawn ahead (R29 / R31)
        layer = EncoderLayer(dims, dtype, LayerCfg())
        ops.enc_set_option(layer.ctx, ops.OPT_MASK_BYTES, mb)
        ops.enc_set_option(layer.ctx, ops.OPT_MASK_AHEAD, ahead)
        ops.enc_set_option(layer.ctx, ops.OPT_BDRLN_VARIANT, variant)
        layer.set_params(prm)
        Y = layer.forward(X, M).clone()
        dX = layer.backward(X, dY).clone()
        torch.cuda.synchronize()
        out.append((Y.cpu(), dX.cpu(), layer.grad_flat.cpu()))
    for other in out[1:]:
        for a, b in zip(out[0], other):
            assert torch.equal(a, b)


@pytest.mark.parametrize("dims,causal", [
    (Dims(B=2, J=512, H=4, P=64, U=1024), False),
    (Dims(B=2, J=512, H=4, P=64, U=1024), True),
    (Dims(B=3, J=128, H=4, P=64, U=512), False),   # short-row score kernels
    (Dims(B=2, J=256, H=4, P=64, U=512), False),   # tiled score path (option inactive)
])
def test_av_keep_gen_option_bitwise(dims, causal):
    """ENC_OPT_AV_KEEP_GEN (R28): the attention keep words generated by the A.V
    kernel's dropout-on-load warps instead of the score kernel -- the stored words, Y, dX and
    every gradient are bitwise those of the other placement."""
    from paper_2007_00072_b200 import ops
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    prm = make_params(dims, "bf16", "parity", weight_std=0.05)
    inp = make_inputs(dims, "bf16", key_padding=True)
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    M = torch.tensor(inp["mask_bias"], device="cuda")
    out = []
    for gen in (0, 1):
        layer = EncoderLayer(dims, "bf16", LayerCfg(causal=causal))
        ops.enc_set_option(layer.ctx, ops.OPT_AV_KEEP_GEN, gen)
        layer.set_params(prm)
        layer.saved.zero_()   # regions a path does not write compare equal
        Y = layer.forward(X, M).clone()
        dX = layer.backward(X, dY).clone()
        torch.cuda.synchronize()
        out.append((Y.cpu(), dX.cpu(), layer.grad_flat.cpu(), layer.saved.cpu()))
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("opts", [{21: 1}, {21: 0}])
def test_layer_fused_av_stagewise(opts):
    """ENC_OPT_ATTN_FUSED_AV (R30): QK^T + BSB + A.V in one kernel -- every stage
    (P, keep words, C, ...) against the oracle fed the GPU's stored inputs, both settings."""
    pairs, f32 = _stagewise(Dims(B=2, J=512, H=4, P=64, U=512), "bf16", "gelu", True,
                            opts=opts, weight_std=0.06)
    for n, g, o in pairs + f32:
        assert_parity(n, g, o, "bf16")


@pytest.mark.parametrize("causal", [False, True])
def test_layer_fused_av_matches_two_kernels(causal):
    """The fused score + A.V kernel gives the two-kernel path's P and keep words bitwise, and
    C / the gradients within bf16 accumulation-order noise."""
    from paper_2007_00072_b200 import ops
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    dims = Dims(B=2, J=512, H=4, P=64, U=1024)
    prm = make_params(dims, "bf16", "parity", weight_std=0.05)
    inp = make_inputs(dims, "bf16", key_padding=True)
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    M = torch.tensor(inp["mask_bias"], device="cuda")
    out = []
    for fav in (0, 1):
        layer = EncoderLayer(dims, "bf16", LayerCfg(causal=causal))
        ops.enc_set_option(layer.ctx, ops.OPT_ATTN_FUSED_AV, fav)
        layer.set_params(prm)
        Y = layer.forward(X, M).clone()
        dX = layer.backward(X, dY).clone()
        torch.cuda.synchronize()
        views = layer.saved_views()
        out.append((Y.float().cpu(), dX.float().cpu(), layer.grad_flat.cpu(),
                    views["P"].cpu(), views["keep_attn"].cpu(), views["C"].float().cpu()))
    assert torch.equal(out[0][3], out[1][3])   # P
    assert torch.equal(out[0][4], out[1][4])   # keep words
    for i, name in ((0, "Y"), (1, "dX"), (2, "grads"), (5, "C")):
        a, b = out[0][i], out[1][i]
        err = (a - b).abs().max().item()
        scale = a.abs().max().item()
        assert err <= 2e-2 * scale + 1e-6, (name, err, scale)


@pytest.mark.parametrize("graph", [False, True])
def test_pdl_mask_bitwise(graph):
    """ENC_OPT_PDL (programmatic dependent launch) changes only when kernels start: with it
    off, at the default mask and with every class on, Y, dX, every gradient and the saved
    tensors are bitwise equal -- a kernel that read its predecessor's output before
    griddepcontrol.wait would show up here as a difference."""
    from paper_2007_00072_b200 import ops
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    dims = Dims(B=2, J=512, H=4, P=64, U=1024)
    prm = make_params(dims, "bf16", "parity", weight_std=0.05)
    inp = make_inputs(dims, "bf16", key_padding=True)
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    M = torch.tensor(inp["mask_bias"], device="cuda")
    out = []
    layer = EncoderLayer(dims, "bf16", LayerCfg())
    layer.set_params(prm)
    try:
        for mask in (0, 13, 31):
            ops.enc_set_option(layer.ctx, ops.OPT_PDL, mask)
            layer.saved.zero_()
            layer.grad_flat.zero_()
            if graph:
                Y, dX = torch.empty_like(X), torch.empty_like(X)
                layer.forward(X, M, Y)
                layer.backward(X, dY, dX)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    layer.forward(X, M, Y)
                    layer.backward(X, dY, dX)
                layer.saved.zero_()
                layer.grad_flat.zero_()
                g.replay()
            else:
                Y = layer.forward(X, M).clone()
                dX = layer.backward(X, dY).clone()
            torch.cuda.synchronize()
            out.append((Y.cpu(), dX.cpu(), layer.grad_flat.cpu(), layer.saved.cpu()))
    finally:
        ops.enc_set_option(layer.ctx, ops.OPT_PDL, 13)
    for other in out[1:]:
        for a, b in zip(out[0], other):
            assert torch.equal(a, b)
