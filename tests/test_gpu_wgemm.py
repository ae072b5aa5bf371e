"""Parity of the hand-written tcgen05 weight contractions (csrc/wgemm.cu) through the C ABI:
enc_wgemm in the three operand forms of the layer (forward X W^T, dX = dY W, dW = dY^T X)
with bias / residual / split-K, and the two fused FFN kernels (Linear1 + BAD, Linear2-dX +
BAD-bwd) against the fp64 oracle (the contraction is its plain definition, a library
matmul of the same bf16 inputs; BAD / BAD-bwd are oracle/encoder.py).  Shapes span several
128 x 256 tiles plus ragged M / N / K tails; the config-L shapes are checked on sampled
rows computed one by one."""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from oracle import philox
from synth import make_tensor
from tol import assert_parity, errors

pytestmark = pytest.mark.gpu
SEED = 2007000072


@pytest.fixture(scope="module")
def ops():
    from paper_2007_00072_b200 import ops as _ops
    return _ops


@pytest.fixture(scope="module", params=[1, 0], ids=["pair", "single"])
def ctx(ops, request):
    """Both tile schedules: 256 x 256 tiles on CTA pairs (tcgen05.mma.cta_group::2, the
    default) and 128 x 256 tiles on single CTAs (ENC_OPT_GEMM_PAIR = 0)."""
    c = ops.Context(0)
    ops.enc_set_option(c, ops.OPT_GEMM_PAIR, request.param)
    return c


def bf(a):
    return torch.tensor(np.ascontiguousarray(a, np.float32), device="cuda").to(torch.bfloat16)


def f32(a):
    return torch.tensor(np.ascontiguousarray(a, np.float32), device="cuda")


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def _fp32_close(name, g, o):
    e = errors(g, o)
    # fp32 accumulation of bf16 products: normwise relative error ~ sqrt(K) 2^-24
    assert e["max_rel"] <= 2e-5, f"{name}: {e}"


SHAPES = [(128, 256, 64), (256, 512, 128), (300, 264, 200), (120, 72, 40), (512, 768, 1024),
          (1000, 1032, 520), (384, 256, 64)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("bias", [False, True])
def test_forward_form(ops, ctx, M, N, K, bias):
    """C = X W^T (+ b): A [M,K] K-major, B = W [N,K] K-major, bf16 output."""
    X = make_tensor((M, K), 1, "bf16")
    W = make_tensor((N, K), 2, "bf16", std=0.05)
    b = make_tensor((N,), 3, "fp32", std=0.1)
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    ops.enc_wgemm(ctx, bf(X), bf(W), C, tA=False, tB=True, bias=f32(b) if bias else None)
    ref = X.astype(np.float64) @ W.astype(np.float64).T + (b if bias else 0.0)
    assert_parity("C", host(C), ref, "bf16")


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("beta", [0, 1])
def test_dx_form(ops, ctx, M, N, K, beta):
    """dX = dY W (+ R): A [M,K] K-major, B = W [K,N] MN-major, bf16 output, beta = 1 adds
    the residual gradient already in C (paper `ebsb` / `bei`)."""
    dY = make_tensor((M, K), 4, "bf16")
    W = make_tensor((K, N), 5, "bf16", std=0.05)
    R = make_tensor((M, N), 6, "bf16")
    C = bf(R)
    ops.enc_wgemm(ctx, bf(dY), bf(W), C, tA=False, tB=False, beta=beta)
    ref = dY.astype(np.float64) @ W.astype(np.float64) + (R if beta else 0.0)
    assert_parity("dX", host(C), ref, "bf16")


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 304), (264, 136, 520),
                                   (1024, 1024, 4096), (768, 768, 2048), (384, 1024, 4096),
                                   (512, 256, 8192)])
def test_dw_form(ops, ctx, M, N, K):
    """dW = dY^T X: A = dY [K,M] MN-major, B = X [K,N] MN-major, fp32 output (split over K
    into the context workspace and summed in a fixed order when that fills more SMs)."""
    dY = make_tensor((K, M), 7, "bf16")
    X = make_tensor((K, N), 8, "bf16")
    C = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    ops.enc_wgemm(ctx, bf(dY), bf(X), C, tA=True, tB=False)
    ref = dY.astype(np.float64).T @ X.astype(np.float64)
    _fp32_close("dW", host(C), ref)
    # deterministic: a second run is bitwise identical
    C2 = torch.empty_like(C)
    ops.enc_wgemm(ctx, bf(dY), bf(X), C2, tA=True, tB=False)
    assert torch.equal(C, C2)


def test_strided_operands(ops, ctx):
    """Leading dimensions larger than the row (the Q/K/V column blocks of dQKV)."""
    M, N, K = 256, 256, 192
    big = make_tensor((M, 3 * K), 9, "bf16")
    W = make_tensor((N, K), 10, "bf16", std=0.05)
    tb = bf(big)
    A = tb[:, K:2 * K]
    C = torch.zeros(M, 2 * N, dtype=torch.bfloat16, device="cuda")
    from paper_2007_00072_b200 import _abi
    lib = _abi.load()
    rc = lib.enc_wgemm(ctx.ptr, M, N, K, A.data_ptr(), 3 * K, 0, bf(W).data_ptr(), K, 1,
                       C.data_ptr(), 2 * N, 0, 0, None, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    ref = big[:, K:2 * K].astype(np.float64) @ W.astype(np.float64).T
    assert_parity("C", host(C[:, :N]), ref, "bf16")
    assert float(C[:, N:].abs().max()) == 0.0   # nothing written past N


def test_config_L_shapes_sampled(ops, ctx):
    """The layer's twelve contraction shapes at config L (B*J = 4096, I = 1024, U = 4096),
    checked on 64 sampled output rows computed one by one in fp64."""
    BJ, I, U = 4096, 1024, 4096
    rng = np.random.default_rng(11)
    rows = np.sort(rng.choice(BJ, 64, replace=False))
    for (M, N, K, tA, tB, out) in [(BJ, 3 * I, I, 0, 1, "bf16"), (BJ, I, I, 0, 1, "bf16"),
                                   (BJ, U, I, 0, 1, "bf16"), (BJ, I, U, 0, 1, "bf16"),
                                   (BJ, U, I, 0, 0, "bf16"), (BJ, I, U, 0, 0, "bf16"),
                                   (BJ, I, 3 * I, 0, 0, "bf16")]:
        A = make_tensor((M, K), 12, "bf16")
        B = make_tensor((N, K) if tB else (K, N), 13, "bf16", std=0.03)
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        ops.enc_wgemm(ctx, bf(A), bf(B), C, tA=False, tB=bool(tB))
        Bd = B.astype(np.float64)
        ref = A[rows].astype(np.float64) @ (Bd.T if tB else Bd)
        assert_parity(f"C{(M, N, K, tB)}", host(C)[rows], ref, "bf16")
    for (M, N) in [(I, U), (U, I), (I, I), (3 * I, I)]:
        A = make_tensor((BJ, M), 14, "bf16")
        B = make_tensor((BJ, N), 15, "bf16")
        C = torch.empty(M, N, dtype=torch.float32, device="cuda")
        ops.enc_wgemm(ctx, bf(A), bf(B), C, tA=True, tB=False)
        sel = rows[rows < M]
        ref = A[:, sel].astype(np.float64).T @ B.astype(np.float64)
        _fp32_close(f"dW{(M, N)}", host(C)[sel], ref)


# ------------------------------------------------------------------ fused FFN kernels
FFN_SHAPES = [(2, 64, 64, 256), (3, 40, 48, 264), (1, 128, 1024, 4096), (2, 100, 96, 520),
              (2, 384, 256, 512)]


@pytest.mark.parametrize("B,J,I,U", FFN_SHAPES)
@pytest.mark.parametrize("act", [E.ACT_GELU_ERF, E.ACT_GELU_TANH, E.ACT_RELU])
@pytest.mark.parametrize("p", [0.1, 0.0])
def test_linear1_bad_fwd(ops, ctx, B, J, I, U, act, p):
    X1 = make_tensor((B, J, I), 21, "bf16")
    W1 = make_tensor((U, I), 22, "bf16", std=0.06)
    b1 = make_tensor((U,), 23, "fp32", std=0.1)
    sub, boff = 6, 3
    h = torch.empty(B, J, U, dtype=torch.bfloat16, device="cuda")
    A1 = torch.empty_like(h)
    ops.enc_linear1_bad_fwd(ctx, B, J, I, U, bf(X1), bf(W1), f32(b1), act, p, SEED, sub, boff,
                            h, A1)
    ho = X1.astype(np.float64) @ W1.astype(np.float64).T + b1
    assert_parity("h", host(h), ho, "bf16")
    # A1 from the stored (rounded) h, as the epilogue computes it
    _, A1o = E.bad_fwd(host(h), np.zeros(U), act, p, SEED, sub, boff)
    assert_parity("A1", host(A1), A1o, "bf16")
    keep = philox.keep_mask_tensor((B, J, U), boff, p, SEED, sub)
    assert not np.any(host(A1)[~keep]), "dropped elements must be exactly 0"


@pytest.mark.parametrize("B,J,I,U", FFN_SHAPES)
@pytest.mark.parametrize("act", [E.ACT_GELU_ERF, E.ACT_GELU_TANH, E.ACT_RELU])
@pytest.mark.parametrize("p", [0.1, 0.0])
def test_linear2_dx_bad_bwd(ops, ctx, B, J, I, U, act, p):
    dY2 = make_tensor((B, J, I), 31, "bf16")
    W2 = make_tensor((I, U), 32, "bf16", std=0.06)
    h = make_tensor((B, J, U), 33, "bf16", std=1.5)
    sub, boff = 6, 5
    dh = torch.empty(B, J, U, dtype=torch.bfloat16, device="cuda")
    db1 = torch.full((U,), float("nan"), dtype=torch.float32, device="cuda")
    ops.enc_linear2_dx_bad_bwd(ctx, B, J, I, U, bf(dY2), bf(W2), bf(h), act, p, SEED, sub, boff,
                               dh, db1)
    dA1 = dY2.astype(np.float64) @ W2.astype(np.float64)
    dho, db1o = E.bad_bwd(dA1, h.astype(np.float64), act, p, SEED, sub, boff)
    assert_parity("dh", host(dh), dho, "bf16")
    assert_parity("db1", host(db1), db1o, "bf16")
    keep = philox.keep_mask_tensor((B, J, U), boff, p, SEED, sub)
    assert not np.any(host(dh)[~keep])


def test_fused_ffn_errors(ops, ctx):
    from paper_2007_00072_b200._abi import EncError
    t = torch.empty(64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(EncError):   # U not a multiple of 8
        ops.enc_linear1_bad_fwd(ctx, 1, 8, 8, 12, t, t, t.float(), 0, 0.1, SEED, 2, 0, t, t)
    with pytest.raises(EncError):   # p whose threshold rounds to 65536
        ops.enc_linear1_bad_fwd(ctx, 1, 8, 8, 8, t, t, t.float(), 0, 0.999995, SEED, 2, 0, t, t)
