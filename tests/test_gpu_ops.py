"""Per-operator parity: CUDA path (through the C ABI) vs the fp64 oracle on the same seeded
inputs.  Bit-exact for the dropout masks; north-star tolerances (tests/tol.py) for
floating point.  Shapes span several tiles plus ragged tails; config-L shapes are checked
on sampled batch slices the oracle computes one by one."""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from oracle import philox
from synth import make_positive_rows, make_tensor
from tol import assert_parity

pytestmark = pytest.mark.gpu

TDT = {"bf16": torch.bfloat16, "fp32": torch.float32}
SEED = 2007000072


@pytest.fixture(scope="module")
def ops():
    from paper_2007_00072_b200 import ops as _ops
    return _ops


@pytest.fixture(scope="module")
def ctx(ops):
    return ops.Context(0)


def dev(a, dtype):
    return torch.tensor(np.ascontiguousarray(a, np.float32), device="cuda").to(TDT[dtype])


def dev32(a):
    return torch.tensor(np.ascontiguousarray(a, np.float32), device="cuda")


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


# ------------------------------------------------------------------ dropout mask
@pytest.mark.parametrize("n,index0,p,sub", [
    (1 << 20, 0, 0.1, 0), (12345, 7, 0.1, 5), (4099, (1 << 35) + 3, 0.5, (3 << 32) + 1),
    (1000, 0, 0.0, 2), (777, 123456789, 0.9, 9)])
def test_dropout_mask_bit_exact(ops, n, index0, p, sub):
    keep = torch.empty(n, dtype=torch.uint8, device="cuda")
    ops.enc_dropout_mask(n, index0, p, SEED, sub, keep)
    ref = philox.keep_mask(index0, n, p, SEED, sub)
    assert np.array_equal(keep.cpu().numpy().astype(bool), ref)


# ------------------------------------------------------------------ BSB
BSB_SHAPES = [(2, 2, 16, 16), (3, 5, 7, 200), (2, 3, 9, 512), (1, 2, 5, 1024), (1, 1, 3, 4096),
              (1, 1, 2, 8),
              (1, 2, 7, 2056),   # K > 2048: two warps per row, the second range ragged
              (2, 1, 5, 3000),
              # K <= 128: several rows per warp (segmented reductions), ragged row counts
              (3, 2, 5, 128), (2, 3, 7, 64), (1, 3, 11, 32), (4, 12, 128, 128)]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", BSB_SHAPES)
@pytest.mark.parametrize("masked", [False, True])
def test_bsb_fwd(ops, ctx, dtype, shape, masked):
    B, H, J, K = shape
    S = make_tensor((B, H, J, K), 11, dtype, std=3.0)
    M = None
    if masked:
        M = np.zeros((B, K), np.float32)
        M[:, K // 2 + 1:] = -10000.0
    scale, p, sub, boff = 0.125, 0.1, 4, 3
    tS = dev(S, dtype)
    P = torch.empty_like(tS)
    A = torch.empty_like(tS)
    ops.enc_bsb_fwd(ctx, B, H, J, K, scale, tS, None if M is None else dev32(M), p, SEED, sub,
                    boff, P, A)
    Po, Ao = E.bsb_fwd(S, M, scale, p, SEED, sub, boff)
    assert_parity("P", host(P), Po, dtype)
    assert_parity("A", host(A), Ao, dtype)
    # dropped positions are exactly zero, kept ones are not
    keep = philox.keep_mask_tensor(S.shape, boff, p, SEED, sub)
    assert (host(A)[~keep] == 0).all()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(2, 2, 16, 16), (2, 3, 64, 64), (3, 2, 128, 128),
                                   (1, 2, 512, 512), (1, 1, 2056, 2056)])
@pytest.mark.parametrize("masked", [False, True])
def test_bsb_fwd_causal(ops, ctx, dtype, shape, masked):
    """Causal masking step (R22) on the unfused BSB kernels: short
    rows (several per warp), one warp per row and two warps per row."""
    B, H, J, K = shape
    S = make_tensor((B, H, J, K), 12, dtype, std=3.0)
    M = None
    if masked:
        M = np.zeros((B, K), np.float32)
        M[:, K - K // 4:] = -10000.0
    scale, p, sub, boff = 0.125, 0.1, 4, 3
    tS = dev(S, dtype)
    P = torch.empty_like(tS)
    A = torch.empty_like(tS)
    ops.enc_bsb_fwd(ctx, B, H, J, K, scale, tS, None if M is None else dev32(M), p, SEED, sub,
                    boff, P, A, causal=True)
    Po, Ao = E.bsb_fwd(S, M, scale, p, SEED, sub, boff, causal=True)
    hp = host(P)
    assert (hp[..., np.triu(np.ones((J, K), bool), 1)] == 0).all()
    assert_parity("P", hp, Po, dtype)
    assert_parity("A", host(A), Ao, dtype)


def test_bsb_fwd_causal_rejects_rectangular(ops, ctx):
    from paper_2007_00072_b200._abi import EncError
    t = torch.zeros((1, 1, 8, 16), device="cuda")
    with pytest.raises(EncError):
        ops.enc_bsb_fwd(ctx, 1, 1, 8, 16, 0.125, t, None, 0.1, SEED, 0, 0, t.clone(), t.clone(),
                        causal=True)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", BSB_SHAPES)
def test_bsb_bwd(ops, ctx, dtype, shape):
    B, H, J, K = shape
    dA = make_tensor((B, H, J, K), 12, dtype)
    Pm = make_positive_rows((B, H, J, K), 13, dtype)
    scale, p, sub, boff = 0.125, 0.1, 4, 2
    tdA = dev(dA, dtype)
    dS = torch.empty_like(tdA)
    ops.enc_bsb_bwd(ctx, B, H, J, K, scale, tdA, dev(Pm, dtype), p, SEED, sub, boff, dS)
    dSo = E.bsb_bwd(dA, Pm, scale, p, SEED, sub, boff)
    assert_parity("dS", host(dS), dSo, dtype)


# ------------------------------------------------------------------ BDRLN
LN_SHAPES = [(2, 16, 16), (3, 7, 1000), (2, 33, 1024), (1, 5, 768), (1, 3, 2048), (4, 5, 8),
             (8, 130, 768), (2, 37, 1536)]   # three warps per row (one or two chunks per lane)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", LN_SHAPES)
def test_bdrln_fwd(ops, ctx, dtype, shape):
    B, J, I = shape
    Y = make_tensor((B, J, I), 21, dtype)
    R = make_tensor((B, J, I), 22, dtype, std=2.0, mean=0.5)
    bias = make_tensor((I,), 23, "fp32", std=0.1)
    g = make_tensor((I,), 24, "fp32", std=0.1, mean=1.0)
    be = make_tensor((I,), 25, "fp32", std=0.1)
    p, sub, boff, eps = 0.1, 1, 5, 1e-5
    tY = dev(Y, dtype)
    out, xhat = torch.empty_like(tY), torch.empty_like(tY)
    rstd = torch.empty((B, J), dtype=torch.float32, device="cuda")
    ops.enc_bdrln_fwd(ctx, B, J, I, tY, dev32(bias), dev(R, dtype), dev32(g), dev32(be), eps, p,
                      SEED, sub, boff, out, xhat, rstd)
    oo, xo, ro = E.bdrln_fwd(Y, bias, R, g, be, eps, p, SEED, sub, boff)
    assert_parity("out", host(out), oo, dtype)
    assert_parity("xhat", host(xhat), xo, dtype)
    assert_parity("rstd", host(rstd), ro, "fp32")   # fp32 statistics in both paths


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", LN_SHAPES + [(8, 512, 1024)])
def test_bdrln_bwd(ops, ctx, dtype, shape):
    B, J, I = shape
    dOut = make_tensor((B, J, I), 31, dtype)
    xhat = make_tensor((B, J, I), 32, dtype)
    rstd = (np.random.default_rng(33).random((B, J)) + 0.5).astype(np.float32)
    g = make_tensor((I,), 34, "fp32", std=0.1, mean=1.0)
    p, sub, boff = 0.1, 3, 1
    tO = dev(dOut, dtype)
    dz, dy = torch.empty_like(tO), torch.empty_like(tO)
    dg, db, dbias = (torch.empty(I, dtype=torch.float32, device="cuda") for _ in range(3))
    ops.enc_bdrln_bwd(ctx, B, J, I, tO, dev(xhat, dtype), dev32(rstd), dev32(g), p, SEED, sub,
                      boff, dz, dy, dg, db, dbias)
    dzo, dyo, dgo, dbo, dbiaso = E.bdrln_bwd(dOut, xhat, rstd, g, p, SEED, sub, boff)
    assert_parity("dz", host(dz), dzo, dtype)
    assert_parity("dYpre", host(dy), dyo, dtype)
    # parameter gradients are fp32 column sums of exactly-representable inputs
    assert_parity("dgamma", host(dg), dgo, "fp32")
    assert_parity("dbeta", host(db), dbo, "fp32")
    if dtype == "fp32":
        assert_parity("dbias", host(dbias), dbiaso, "fp32")
    else:  # dbias sums the fp32 dYpre before its bf16 rounding; compare at bf16 bounds
        assert_parity("dbias", host(dbias), dbiaso, "bf16")
    # determinism: bitwise identical on a second run
    dg2 = torch.empty_like(dg)
    ops.enc_bdrln_bwd(ctx, B, J, I, tO, dev(xhat, dtype), dev32(rstd), dev32(g), p, SEED, sub,
                      boff, dz, dy, dg2, db, dbias)
    assert torch.equal(dg, dg2)


# ------------------------------------------------------------------ BAD
BAD_SHAPES = [(2, 16, 64), (3, 7, 1000), (2, 33, 4096), (1, 5, 3072), (2, 3, 8)]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", BAD_SHAPES)
@pytest.mark.parametrize("act", [E.ACT_GELU_ERF, E.ACT_GELU_TANH, E.ACT_RELU])
@pytest.mark.parametrize("p", [0.1, 0.0])
def test_bad_fwd_bwd(ops, ctx, dtype, shape, act, p):
    B, J, U = shape
    Y1 = make_tensor((B, J, U), 41, dtype, std=2.0)
    b1 = make_tensor((U,), 42, "fp32", std=0.1)
    dA1 = make_tensor((B, J, U), 43, dtype)
    sub, boff = 2, 4
    tY = dev(Y1, dtype)
    h, A1 = torch.empty_like(tY), torch.empty_like(tY)
    ops.enc_bad_fwd(ctx, B, J, U, tY, dev32(b1), act, p, SEED, sub, boff, h, A1)
    ho, A1o = E.bad_fwd(Y1, b1, act, p, SEED, sub, boff)
    assert_parity("h", host(h), ho, dtype)
    assert_parity("A1", host(A1), A1o, dtype)
    # backward on the GPU's own saved h (same activation-derivative decisions)
    hh = host(h)
    dh = torch.empty_like(tY)
    db1 = torch.empty(U, dtype=torch.float32, device="cuda")
    ops.enc_bad_bwd(ctx, B, J, U, dev(dA1, dtype), h, act, p, SEED, sub, boff, dh, db1)
    dho, db1o = E.bad_bwd(dA1, hh, act, p, SEED, sub, boff)
    assert_parity("dh", host(dh), dho, dtype)
    assert_parity("db1", host(db1), db1o, "fp32" if dtype == "fp32" else "bf16")


# ------------------------------------------------------------------ AIB / BEI
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("shape", [(2, 16, 2, 8), (3, 7, 5, 16), (2, 130, 16, 64), (1, 9, 1, 24)])
def test_aib_fwd_bwd(ops, ctx, dtype, shape):
    B, J, H, P = shape
    I = H * P
    QKV = make_tensor((B, J, 3 * I), 51, dtype)
    b = make_tensor((3 * I,), 52, "fp32", std=0.1)
    tq = dev(QKV, dtype)
    q, k, v = (torch.empty((B, H, J, P), dtype=TDT[dtype], device="cuda") for _ in range(3))
    ops.enc_aib_fwd(ctx, B, J, H, P, tq, dev32(b), q, k, v)
    Qo, Ko, Vo = E.aib_fwd(QKV, b, H, P)
    for n, g, o in (("Q", q, Qo), ("K", k, Ko), ("V", v, Vo)):
        assert_parity(n, host(g), o, dtype)
    dq, dk, dv = (make_tensor((B, H, J, P), 53 + i, dtype) for i in range(3))
    dqkv = torch.empty((B, J, 3 * I), dtype=TDT[dtype], device="cuda")
    db = torch.empty(3 * I, dtype=torch.float32, device="cuda")
    ops.enc_aib_bwd(ctx, B, J, H, P, dev(dq, dtype), dev(dk, dtype), dev(dv, dtype), dqkv, db)
    dqkvo, dbo = E.aib_bwd(dq, dk, dv)
    assert np.array_equal(host(dqkv), dqkvo)          # pure permutation: exact
    assert_parity("dbqkv", host(db), dbo, "fp32")


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_bei(ops, ctx, dtype):
    a = make_tensor((3, 17, 64), 61, dtype)
    b = make_tensor((3, 17, 64), 62, dtype)
    out = torch.empty((3, 17, 64), dtype=TDT[dtype], device="cuda")
    ops.enc_bei(ctx, dev(a, dtype), dev(b, dtype), out)
    assert_parity("bei", host(out), E.bei(a, b), dtype)


# ------------------------------------------------------------------ config-L shapes, sampled
def test_config_L_fused_ops_sampled(ops, ctx):
    """BSB / BSB-bwd / BDRLN / BAD at the paper's BERT-large shapes (B=8, H=16, J=K=512,
    I=1024, U=4096) in the launch configuration the layer uses; the oracle checks one
    sampled batch element (b=5) computed on its own with batch_offset=5."""
    B, H, J, I, U, dtype = 8, 16, 512, 1024, 4096, "bf16"
    b = 5
    S = make_tensor((B, H, J, J), 71, dtype, std=2.0)
    tS = dev(S, dtype)
    P, A = torch.empty_like(tS), torch.empty_like(tS)
    ops.enc_bsb_fwd(ctx, B, H, J, J, 0.125, tS, None, 0.1, SEED, 0, 0, P, A)
    Po, Ao = E.bsb_fwd(S[b:b + 1], None, 0.125, 0.1, SEED, 0, b)
    assert_parity("P[L]", host(P[b:b + 1]), Po, dtype)
    assert_parity("A[L]", host(A[b:b + 1]), Ao, dtype)
    dS = torch.empty_like(tS)
    ops.enc_bsb_bwd(ctx, B, H, J, J, 0.125, tS, P, 0.1, SEED, 0, 0, dS)
    dSo = E.bsb_bwd(S[b:b + 1], host(P[b:b + 1]), 0.125, 0.1, SEED, 0, b)
    assert_parity("dS[L]", host(dS[b:b + 1]), dSo, dtype)
    Y1 = make_tensor((B, J, U), 72, dtype)
    b1 = np.zeros(U, np.float32)
    tY = dev(Y1, dtype)
    h, A1 = torch.empty_like(tY), torch.empty_like(tY)
    ops.enc_bad_fwd(ctx, B, J, U, tY, dev32(b1), E.ACT_GELU_ERF, 0.1, SEED, 2, 0, h, A1)
    _, A1o = E.bad_fwd(Y1[b:b + 1], b1, E.ACT_GELU_ERF, 0.1, SEED, 2, b)
    assert_parity("A1[L]", host(A1[b:b + 1]), A1o, dtype)
