"""Per-operator pins for oracle/encoder.py (CPU only): invariants, closed forms,
library special cases.  None of these re-types the oracle's formula."""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from oracle import philox

RNG = np.random.default_rng(7)


def test_softmax_rows_sum_to_one_and_are_positive():
    S = RNG.standard_normal((2, 3, 5, 24)) * 4
    M = np.where(RNG.random((2, 24)) < 0.3, -10000.0, 0.0)
    for mb in (None, M):
        P, A = E.bsb_fwd(S, mb, 0.125, 0.0, 1, 0)
        assert np.allclose(P.sum(-1), 1.0, atol=1e-12, rtol=0)
        assert (P >= 0).all()
        assert np.array_equal(P, A)           # p = 0: A is P


def test_softmax_constant_row_is_uniform_and_shift_invariant():
    S = np.full((1, 1, 2, 16), 3.0)
    P, _ = E.bsb_fwd(S, None, 0.5, 0.0, 1, 0)
    assert np.allclose(P, 1 / 16, atol=1e-15)
    S2 = RNG.standard_normal((1, 2, 3, 16))
    P1, _ = E.bsb_fwd(S2, None, 1.0, 0.0, 1, 0)
    P2, _ = E.bsb_fwd(S2 + 1000.0, None, 1.0, 0.0, 1, 0)   # max-subtraction path
    assert np.allclose(P1, P2, atol=1e-12)


def test_softmax_matches_torch_and_mask_bias_excludes_keys():
    S = RNG.standard_normal((2, 2, 4, 16))
    M = np.zeros((2, 16))
    M[:, 10:] = -10000.0
    P, _ = E.bsb_fwd(S, M, 0.3, 0.0, 1, 0)
    ref = torch.softmax(torch.tensor(S) * 0.3 + torch.tensor(M)[:, None, None, :], dim=-1).numpy()
    assert np.allclose(P, ref, atol=1e-14)
    assert P[..., 10:].max() < 1e-300 or P[..., 10:].max() < 1e-100


def test_dropout_applied_with_site_mask_and_scale():
    S = RNG.standard_normal((2, 2, 4, 16))
    p, seed, sub = 0.25, 99, 6
    P, A = E.bsb_fwd(S, None, 1.0, p, seed, sub, batch_offset=3)
    keep = philox.keep_mask_tensor(S.shape, 3, p, seed, sub)
    s = philox.dropout_scale(p)
    assert np.array_equal(A[~keep], np.zeros((~keep).sum()))
    assert np.allclose(A[keep], P[keep] * s, rtol=1e-15)


def test_softmax_backward_rows_sum_to_zero_and_match_autograd():
    S = RNG.standard_normal((2, 2, 3, 16))
    dA = RNG.standard_normal(S.shape)
    P, _ = E.bsb_fwd(S, None, 0.7, 0.0, 1, 0)
    dS = E.bsb_bwd(dA, P, 0.7, 0.0, 1, 0)
    assert np.allclose(dS.sum(-1), 0.0, atol=1e-13)
    St = torch.tensor(S, requires_grad=True)
    torch.softmax(0.7 * St, dim=-1).backward(torch.tensor(dA))
    assert np.allclose(dS, St.grad.numpy(), atol=1e-13)


@pytest.mark.parametrize("eps", [0.0, 1e-5, 0.5])
def test_layernorm_invariants(eps):
    Y = RNG.standard_normal((2, 5, 32)) * 3 + 1
    R = RNG.standard_normal((2, 5, 32))
    b = RNG.standard_normal(32) * 0.1
    g = np.ones(32)
    be = np.zeros(32)
    out, xhat, rstd = E.bdrln_fwd(Y, b, R, g, be, eps, 0.0, 1, 1)
    z = R + Y + b
    var = z.var(-1)
    assert np.allclose(xhat.mean(-1), 0.0, atol=1e-12)
    assert np.allclose(xhat.var(-1), var / (var + eps), atol=1e-12)
    assert np.allclose(out, xhat)
    assert np.allclose(rstd, 1.0 / np.sqrt(var + eps), rtol=1e-13)


def test_layernorm_forward_backward_match_torch():
    I = 24
    Y = RNG.standard_normal((3, 4, I))
    R = RNG.standard_normal((3, 4, I))
    b = RNG.standard_normal(I)
    g = 1 + RNG.standard_normal(I) * 0.1
    be = RNG.standard_normal(I) * 0.1
    dOut = RNG.standard_normal((3, 4, I))
    out, xhat, rstd = E.bdrln_fwd(Y, b, R, g, be, 1e-5, 0.0, 1, 1)
    tY = torch.tensor(Y, requires_grad=True)
    tb = torch.tensor(b, requires_grad=True)
    tR = torch.tensor(R, requires_grad=True)
    tg = torch.tensor(g, requires_grad=True)
    tbe = torch.tensor(be, requires_grad=True)
    ref = torch.nn.functional.layer_norm(tR + (tY + tb), (I,), tg, tbe, eps=1e-5)
    assert np.allclose(out, ref.detach().numpy(), atol=1e-12)
    ref.backward(torch.tensor(dOut))
    dz, dYpre, dg, dbe, db = E.bdrln_bwd(dOut, xhat, rstd, g, 0.0, 1, 1)
    assert np.allclose(dz, tR.grad.numpy(), atol=1e-12)
    assert np.allclose(dYpre, tY.grad.numpy(), atol=1e-12)
    assert np.allclose(db, tb.grad.numpy(), atol=1e-12)
    assert np.allclose(dg, tg.grad.numpy(), atol=1e-12)
    assert np.allclose(dbe, tbe.grad.numpy(), atol=1e-12)
    assert np.allclose(dz.sum(-1), 0.0, atol=1e-12)          # LN-bwd rows sum to 0


def test_bdrln_bwd_dropout_and_column_sums():
    I = 16
    dOut = RNG.standard_normal((2, 3, I))
    xhat = RNG.standard_normal((2, 3, I))
    rstd = RNG.random((2, 3)) + 0.5
    g = RNG.standard_normal(I)
    dz, dYpre, dg, dbe, db = E.bdrln_bwd(dOut, xhat, rstd, g, 0.3, 11, 5, batch_offset=1)
    keep = philox.keep_mask_tensor(dOut.shape, 1, 0.3, 11, 5)
    assert np.array_equal(dYpre[~keep], np.zeros((~keep).sum()))
    assert np.allclose(dYpre[keep], dz[keep] * philox.dropout_scale(0.3))
    assert np.array_equal(dbe, dOut.reshape(-1, I).sum(0))   # exact column sum
    assert np.allclose(db, dYpre.reshape(-1, I).sum(0))


@pytest.mark.parametrize("act,tfn", [
    (E.ACT_GELU_ERF, lambda x: torch.nn.functional.gelu(x)),
    (E.ACT_GELU_TANH, lambda x: torch.nn.functional.gelu(x, approximate="tanh")),
    (E.ACT_RELU, torch.relu),
])
def test_activation_and_derivative_match_torch(act, tfn):
    h = RNG.standard_normal(4000) * 3
    h = h[np.abs(h) > 1e-3]
    th = torch.tensor(h, requires_grad=True)
    y = tfn(th)
    y.sum().backward()
    assert np.allclose(E.act_fwd(h, act), y.detach().numpy(), atol=1e-14)
    assert np.allclose(E.act_bwd(h, act), th.grad.numpy(), atol=1e-13)


def test_bad_forward_backward():
    Y1 = RNG.standard_normal((2, 3, 32))
    b1 = RNG.standard_normal(32) * 0.1
    dA1 = RNG.standard_normal((2, 3, 32))
    h, A1 = E.bad_fwd(Y1, b1, E.ACT_GELU_ERF, 0.2, 3, 2, batch_offset=5)
    keep = philox.keep_mask_tensor(h.shape, 5, 0.2, 3, 2)
    s = philox.dropout_scale(0.2)
    th = torch.tensor(Y1 + b1, requires_grad=True)
    ref = torch.nn.functional.gelu(th) * torch.tensor(keep * s)
    assert np.allclose(A1, ref.detach().numpy(), atol=1e-14)
    ref.backward(torch.tensor(dA1))
    dh, db1 = E.bad_bwd(dA1, h, E.ACT_GELU_ERF, 0.2, 3, 2, batch_offset=5)
    assert np.allclose(dh, th.grad.numpy(), atol=1e-13)
    assert np.allclose(db1, dh.reshape(-1, 32).sum(0), atol=1e-13)


def test_aib_permutation_roundtrip():
    B, J, H, P = 2, 5, 3, 4
    QKV = RNG.standard_normal((B, J, 3 * H * P))
    b = RNG.standard_normal(3 * H * P)
    Q, K, V = E.aib_fwd(QKV, b, H, P)
    assert Q.shape == (B, H, J, P)
    # element (b, j, part t, head h, p) of QKV+b lands at [t][b, h, j, p]
    assert Q[1, 2, 3, 1] == QKV[1, 3, 0 * H * P + 2 * P + 1] + b[2 * P + 1]
    assert V[0, 1, 4, 3] == QKV[0, 4, 2 * H * P + 1 * P + 3] + b[2 * H * P + P + 3]
    dQKV, db = E.aib_bwd(Q, K, V)
    assert np.allclose(dQKV, QKV + b)
    assert np.allclose(db, (QKV + b).sum(axis=(0, 1)))


def test_bei_is_sum():
    a = RNG.standard_normal((2, 3, 4))
    c = RNG.standard_normal((2, 3, 4))
    assert np.array_equal(E.bei(a, c), a + c)
