"""Parity of the fused tcgen05 score kernels against the fp64 oracle:
  enc_attn_fwd_fused  == BSB(Q K^T)          (oracle bsb_fwd on the fp64 product)
  enc_attn_bwd_fused  == BSB-bwd(dC V^T, P)  (oracle bsb_bwd on the fp64 product)
Dropout keep decisions must match exactly: dropped elements are exactly zero."""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from oracle import philox
from keepbits import decode
from synth import make_positive_rows, make_tensor
from tol import assert_parity

pytestmark = pytest.mark.gpu
SEED = 2007000072


@pytest.fixture(scope="module")
def ops():
    from paper_2007_00072_b200 import ops as _ops
    return _ops


@pytest.fixture(scope="module")
def ctx(ops):
    return ops.Context(0)


def dev(a):
    return torch.tensor(np.ascontiguousarray(a, np.float32), device="cuda").to(torch.bfloat16)


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


# J = 128: the short-row kernels (attn_short.cu), (b, h) pairs pipelined through 3 TMEM
# slots; (64, 12) gives > 3 pairs per CTA (slot reuse, barrier phase wrap), (5, 2) fewer
# pairs than SMs
SHORT = [(1, 1, 128), (5, 2, 128), (64, 12, 128)]


@pytest.mark.parametrize("B,H,J", [(1, 1, 512), (2, 3, 512), (8, 16, 512), (3, 2, 512)] + SHORT)
@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("p", [0.1, 0.0, 0.6])
@pytest.mark.parametrize("store_a", [True, False])
def test_fused_forward(ops, ctx, B, H, J, masked, p, store_a):
    """store_a=False: A is not written (the layer's dropout-on-load path); P and the keep
    words must be unchanged."""
    P = 64
    Q = make_tensor((B, H, J, P), 21, "bf16", std=0.8)
    K = make_tensor((B, H, J, P), 22, "bf16", std=0.8)
    M = None
    if masked:
        M = np.zeros((B, J), np.float32)
        for b in range(B):
            M[b, J // 2 + 17 * b:] = -10000.0
    boff, sub, scale = 5, 8, 0.125
    Pm = torch.full((B, H, J, J), float("nan"), dtype=torch.bfloat16, device="cuda")
    A = torch.full_like(Pm, float("nan"))
    bits = torch.full((B, H, J, J // 32), -1, dtype=torch.int32, device="cuda")
    Mt = None if M is None else torch.tensor(M, device="cuda")
    ops.enc_attn_fwd_fused(ctx, B, H, J, P, scale, dev(Q), dev(K), Mt, p, SEED, sub, boff, Pm,
                           A if store_a else None, keep_bits=bits)
    torch.cuda.synchronize()
    S = Q.astype(np.float64) @ K.astype(np.float64).transpose(0, 1, 3, 2)
    Po, Ao = E.bsb_fwd(S, M, scale, p, SEED, sub, boff)
    gP = host(Pm)
    assert np.isfinite(gP).all()
    assert_parity("P", gP, Po, "bf16")
    keep = philox.keep_mask_tensor(S.shape, boff, p, SEED, sub)
    if store_a:
        gA = host(A)
        assert np.isfinite(gA).all()
        assert_parity("A", gA, Ao, "bf16")
        assert (gA[~keep] == 0).all()
    else:
        assert np.isnan(host(A)).all(), "A written although not requested"
    # the stored keep-flag words are exactly the oracle's keep mask
    assert np.array_equal(decode(bits.cpu().numpy(), J), keep)
    assert np.allclose(gP.sum(-1), 1.0, atol=2e-2)


@pytest.mark.parametrize("B,H,J", [(1, 1, 512), (2, 3, 512), (8, 16, 512)] + SHORT)
@pytest.mark.parametrize("p", [0.1, 0.0, 0.6])
@pytest.mark.parametrize("stored", [False, True])
def test_fused_backward(ops, ctx, B, H, J, p, stored):
    """stored=True: the keep flags come from words the fused forward wrote (for the same
    seed / subsequence / batch offset) instead of being regenerated."""
    P = 64
    dC = make_tensor((B, J, H, P), 31, "bf16")          # [B,J,H,P]
    V = make_tensor((B, H, J, P), 32, "bf16")
    Pm = make_positive_rows((B, H, J, J), 33, "bf16")
    boff, sub, scale = 2, 4, 0.125
    dS = torch.full((B, H, J, J), float("nan"), dtype=torch.bfloat16, device="cuda")
    bits = None
    if stored:
        bits = torch.zeros((B, H, J, J // 32), dtype=torch.int32, device="cuda")
        q = dev(make_tensor((B, H, J, P), 34, "bf16"))
        junk = torch.empty((B, H, J, J), dtype=torch.bfloat16, device="cuda")
        ops.enc_attn_fwd_fused(ctx, B, H, J, P, scale, q, q, None, p, SEED, sub, boff, junk,
                               torch.empty_like(junk), keep_bits=bits)
    ops.enc_attn_bwd_fused(ctx, B, H, J, P, scale, dev(dC), dev(V), dev(Pm), p, SEED, sub, boff, dS,
                           keep_bits=bits)
    torch.cuda.synchronize()
    dA = dC.astype(np.float64).transpose(0, 2, 1, 3) @ V.astype(np.float64).transpose(0, 1, 3, 2)
    dSo = E.bsb_bwd(dA, Pm, scale, p, SEED, sub, boff)
    g = host(dS)
    assert np.isfinite(g).all()
    assert_parity("dS", g, dSo, "bf16")


@pytest.mark.parametrize("B,H,J", [(1, 1, 512), (2, 3, 512), (8, 16, 512)] + SHORT)
@pytest.mark.parametrize("p", [0.1, 0.0, 0.6])
@pytest.mark.parametrize("stored", [False, True])
def test_fused_backward_dc(ops, ctx, B, H, J, p, stored):
    """enc_attn_bwd_fused_dc: the BSB-bwd row term from the attention output C = A V
    (R26) -- C built here from the oracle's keep mask in fp64 and split into the
    two bf16 words the layer stores (C_hi, C_lo); dS must match the oracle's BSB-bwd (which
    forms sum_k dP P) within the bf16 tolerance, dropped elements included."""
    P = 64
    dC = make_tensor((B, J, H, P), 41, "bf16")          # [B,J,H,P]
    V = make_tensor((B, H, J, P), 42, "bf16")
    Pm = make_positive_rows((B, H, J, J), 43, "bf16")
    boff, sub, scale = 5, 4, 0.125
    keep = philox.keep_mask_tensor((B, H, J, J), boff, p, SEED, sub).astype(np.float64)
    A = Pm.astype(np.float64) * keep * philox.dropout_scale(p)
    C = np.ascontiguousarray(np.einsum("bhjk,bhkp->bjhp", A, V.astype(np.float64)))
    bits = None
    if stored:
        bits = torch.zeros((B, H, J, J // 32), dtype=torch.int32, device="cuda")
        q = dev(make_tensor((B, H, J, P), 44, "bf16"))
        junk = torch.empty((B, H, J, J), dtype=torch.bfloat16, device="cuda")
        ops.enc_attn_fwd_fused(ctx, B, H, J, P, scale, q, q, None, p, SEED, sub, boff, junk,
                               None, keep_bits=bits)
    dS = torch.full((B, H, J, J), float("nan"), dtype=torch.bfloat16, device="cuda")
    C_hi = torch.tensor(C, dtype=torch.float64).to(torch.bfloat16)
    C_lo = (torch.tensor(C, dtype=torch.float64) - C_hi.double()).to(torch.bfloat16)
    ops.enc_attn_bwd_fused_dc(ctx, B, H, J, P, scale, dev(dC), dev(V), dev(Pm), C_hi.cuda(),
                              C_lo.cuda(), p, SEED, sub, boff, dS, keep_bits=bits)
    torch.cuda.synchronize()
    dA = dC.astype(np.float64).transpose(0, 2, 1, 3) @ V.astype(np.float64).transpose(0, 1, 3, 2)
    dSo = E.bsb_bwd(dA, Pm, scale, p, SEED, sub, boff)
    g = host(dS)
    assert np.isfinite(g).all()
    assert_parity("dS", g, dSo, "bf16")


@pytest.mark.parametrize("B,H", [(1, 1), (2, 3), (8, 16)])
@pytest.mark.parametrize("p", [0.1, 0.0, 0.6])
@pytest.mark.parametrize("masked,causal", [(False, False), (True, False), (False, True)])
def test_fused_forward_av(ops, ctx, B, H, p, masked, causal):
    """enc_attn_fwd_fused_av (R30): one kernel for S = Q K^T, BSB and C = A V --
    P and C match the oracle (BSB then dropout(P) V in fp64), the keep words are exactly the
    oracle's mask, and C_lo is C's rounding residual (C_hi + C_lo is the fp32 result)."""
    _check_forward_av(ops, ctx, B, H, p, masked, causal)


@pytest.mark.parametrize("masked", [False, True])
def test_fused_forward_av_ragged_schedule(ops, ctx, masked):
    """B 5 x H 16 = 320 tiles on the balanced persistent grid (107 CTAs of 3 tiles but one of
    2): the K / V slot hand-over, the next tile's Q, K loads and the score MMA issued across
    tiles stop at each CTA's own last tile."""
    _check_forward_av(ops, ctx, 5, 16, 0.1, masked, False)


def _check_forward_av(ops, ctx, B, H, p, masked, causal):
    J, P = 512, 64
    Q = make_tensor((B, H, J, P), 51, "bf16", std=0.8)
    K = make_tensor((B, H, J, P), 52, "bf16", std=0.8)
    V = make_tensor((B, H, J, P), 53, "bf16")
    M = None
    if masked:
        M = np.zeros((B, J), np.float32)
        M[:, J - 48:] = -10000.0
    boff, sub, scale = 3, 4, 0.125
    Pm = torch.full((B, H, J, J), float("nan"), dtype=torch.bfloat16, device="cuda")
    bits = torch.full((B, H, J, J // 32), -1, dtype=torch.int32, device="cuda")
    C = torch.full((B, J, H, P), float("nan"), dtype=torch.bfloat16, device="cuda")
    Clo = torch.full_like(C, float("nan"))
    Mt = None if M is None else torch.tensor(M, device="cuda")
    ops.enc_attn_fwd_fused_av(ctx, B, H, J, P, scale, dev(Q), dev(K), dev(V), Mt, p, SEED, sub,
                              boff, Pm, bits, C, Clo, causal=causal)
    torch.cuda.synchronize()
    S = Q.astype(np.float64) @ K.astype(np.float64).transpose(0, 1, 3, 2)
    Po, _ = E.bsb_fwd(S, M, scale, p, SEED, sub, boff, causal=causal)
    gP = host(Pm)
    assert np.isfinite(gP).all()
    assert_parity("P", gP, Po, "bf16")
    keep = philox.keep_mask_tensor((B, H, J, J), boff, p, SEED, sub)
    assert np.array_equal(decode(bits.cpu().numpy(), J), keep)
    # C stage by stage: from the GPU's own P (the contraction's inputs as stored; the
    # end-to-end path from S is covered by the layer tests)
    Cg = host(C).transpose(0, 2, 1, 3)
    A_gpu = gP * keep.astype(np.float64) * philox.dropout_scale(p)
    assert_parity("C(gpu P)", Cg, A_gpu @ V.astype(np.float64), "bf16")
    hi_lo = host(C) + host(Clo)
    exact = (A_gpu @ V.astype(np.float64)).transpose(0, 2, 1, 3)
    assert np.abs(hi_lo - exact).max() <= 1e-3 * (np.abs(exact).max() + 1e-30)


@pytest.mark.parametrize("J,P", [(256, 64), (384, 64), (512, 32), (128, 32), (640, 64)])
def test_fused_unsupported_shapes(ops, ctx, J, P):
    """The fused kernels hold a whole 512-key score row (or whole 128 x 128 score matrices)
    in TMEM; other shapes are refused (the layer then takes the unfused tcgen05 path)."""
    from paper_2007_00072_b200._abi import EncError
    x = torch.zeros((1, 1, J, P), dtype=torch.bfloat16, device="cuda")
    o = torch.zeros((1, 1, J, J), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(EncError):
        ops.enc_attn_fwd_fused(ctx, 1, 1, J, P, 0.125, x, x, None, 0.1, SEED, 0, 0, o, o)


@pytest.mark.parametrize("B,H", [(1, 2), (2, 3)])
@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("p", [0.1, 0.0])
@pytest.mark.parametrize("J", [512, 128])
def test_fused_forward_causal(ops, ctx, B, H, masked, p, J):
    """Causal masking step (R22) inside the fused kernel: P is
    exactly zero above the diagonal (whole 32-column chunks and 64-column warp slices are
    fully masked for the early rows) and matches the oracle's causal BSB elsewhere; the
    fused backward run on that P matches the oracle's BSB-bwd."""
    P = 64
    Q = make_tensor((B, H, J, P), 31, "bf16", std=0.8)
    K = make_tensor((B, H, J, P), 32, "bf16", std=0.8)
    M = None
    if masked:
        M = np.zeros((B, J), np.float32)
        M[:, J - 40:] = -10000.0
    boff, sub, scale = 3, 4, 0.125
    Pm = torch.full((B, H, J, J), float("nan"), dtype=torch.bfloat16, device="cuda")
    bits = torch.full((B, H, J, J // 32), -1, dtype=torch.int32, device="cuda")
    Mt = None if M is None else torch.tensor(M, device="cuda")
    ops.enc_attn_fwd_fused(ctx, B, H, J, P, scale, dev(Q), dev(K), Mt, p, SEED, sub, boff, Pm,
                           None, keep_bits=bits, causal=True)
    torch.cuda.synchronize()
    S = Q.astype(np.float64) @ K.astype(np.float64).transpose(0, 1, 3, 2)
    Po, _ = E.bsb_fwd(S, M, scale, p, SEED, sub, boff, causal=True)
    gP = host(Pm)
    assert np.isfinite(gP).all()
    assert (gP[..., np.triu(np.ones((J, J), bool), 1)] == 0).all()
    assert_parity("P", gP, Po, "bf16")
    assert np.allclose(gP.sum(-1), 1.0, atol=2e-2)
    # backward from the causal P: dS vanishes above the diagonal
    dC = make_tensor((B, J, H, P), 33, "bf16", std=1.0)
    V = make_tensor((B, H, J, P), 34, "bf16", std=1.0)
    dS = torch.full_like(Pm, float("nan"))
    ops.enc_attn_bwd_fused(ctx, B, H, J, P, scale, dev(dC), dev(V), Pm, p, SEED, sub, boff, dS,
                           keep_bits=bits)
    torch.cuda.synchronize()
    dA = np.einsum("bjhp,bhkp->bhjk", dC.astype(np.float64), V.astype(np.float64))
    dSo = E.bsb_bwd(dA, gP, scale, p, SEED, sub, boff)
    gdS = host(dS)
    assert (gdS[..., np.triu(np.ones((J, J), bool), 1)] == 0).all()
    assert_parity("dS", gdS, dSo, "bf16")


@pytest.mark.parametrize("B,H,J,K", [(1, 1, 512, 512), (2, 3, 512, 512), (3, 2, 128, 128),
                                     (1, 2, 7, 192)])
@pytest.mark.parametrize("p", [0.1, 0.0, 0.6])
def test_keep_bits_kernel(ops, ctx, B, H, J, K, p):
    """enc_attn_keep_bits (the layer's side-stream launch) writes exactly the oracle's mask."""
    boff, sub = 3, 12
    bits = torch.full((B, H, J, K // 32), -1, dtype=torch.int32, device="cuda")
    ops.enc_attn_keep_bits(ctx, B, H, J, K, p, SEED, sub, boff, bits)
    torch.cuda.synchronize()
    keep = philox.keep_mask_tensor((B, H, J, K), boff, p, SEED, sub)
    assert np.array_equal(decode(bits.cpu().numpy(), K), keep)


@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("p", [0.1, 0.6])
@pytest.mark.parametrize("J", [512, 128])
def test_fused_forward_given_bits_equals_regenerated(ops, ctx, masked, p, J):
    """The fused forward reading precomputed keep words gives bitwise the P / A of the one
    that runs Philox itself."""
    B, H, P = 2, 3, 64
    Q = dev(make_tensor((B, H, J, P), 31, "bf16", std=0.8))
    K = dev(make_tensor((B, H, J, P), 32, "bf16", std=0.8))
    Mt = None
    if masked:
        M = np.zeros((B, J), np.float32)
        M[:, J * 3 // 5:] = -10000.0
        Mt = torch.tensor(M, device="cuda")
    boff, sub = 1, 4
    out = []
    for given in (False, True):
        Pm = torch.empty((B, H, J, J), dtype=torch.bfloat16, device="cuda")
        A = torch.empty_like(Pm)
        bits = torch.empty((B, H, J, J // 32), dtype=torch.int32, device="cuda")
        if given:
            ops.enc_attn_keep_bits(ctx, B, H, J, J, p, SEED, sub, boff, bits)
            ops.enc_attn_fwd_fused_bits(ctx, B, H, J, P, 0.125, Q, K, Mt, p, SEED, sub, boff, Pm, A,
                                        bits)
        else:
            ops.enc_attn_fwd_fused(ctx, B, H, J, P, 0.125, Q, K, Mt, p, SEED, sub, boff, Pm, A,
                                   keep_bits=bits)
        torch.cuda.synchronize()
        out.append((Pm, A, bits))
    assert torch.equal(out[0][0], out[1][0])
    assert torch.equal(out[0][1], out[1][1])
    assert torch.equal(out[0][2], out[1][2])
