"""Parity of the hand-written tcgen05/TMEM/TMA attention contractions (enc_attn_gemm) against
fp64 numpy matmuls of the same bf16 operands (Table A.1 rows :551, :553, :588-592)."""
import numpy as np
import pytest
import torch

from synth import make_tensor
from tol import assert_parity

pytestmark = pytest.mark.gpu


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


SHAPES = [(1, 1, 128, 64), (2, 3, 256, 64), (8, 16, 512, 64), (3, 2, 384, 64)]
# more (b, h) pairs than SMs (the per-(b, h) kernel loops), and J > 512 (tiled fallback)
SHAPES_BH = [(10, 16, 256, 64), (1, 2, 640, 64)]


@pytest.mark.parametrize("shape", SHAPES + SHAPES_BH)
@pytest.mark.parametrize("which", range(6))
@pytest.mark.parametrize("bh", [1, 0])
def test_attn_gemm(ops, ctx, shape, which, bh):
    """bh=1: AV / DV / DQ / DK on the per-(b, h) streaming kernel where it applies;
    bh=0: every form on the tiled kernel."""
    B, H, J, P = shape
    if shape in SHAPES_BH and not bh:
        pytest.skip("tiled kernel covered by SHAPES")
    ops.enc_set_option(ctx, ops.OPT_ATTN_BH, bh)
    K = J
    bhjp = (B, H, J, P)
    bhjk = (B, H, J, K)
    bjhp = (B, J, H, P)
    if which == ops.AG_QK:
        X, Y = make_tensor(bhjp, 1, "bf16"), make_tensor(bhjp, 2, "bf16")
        ref = X @ Y.transpose(0, 1, 3, 2)
        zshape = bhjk
    elif which == ops.AG_AV:
        X, Y = make_tensor(bhjk, 3, "bf16", std=0.05), make_tensor(bhjp, 4, "bf16")
        ref = (X @ Y).transpose(0, 2, 1, 3)          # C in [B,J,H,P]
        zshape = bjhp
    elif which == ops.AG_DA:
        X, Y = make_tensor(bjhp, 5, "bf16"), make_tensor(bhjp, 6, "bf16")
        ref = X.transpose(0, 2, 1, 3) @ Y.transpose(0, 1, 3, 2)
        zshape = bhjk
    elif which == ops.AG_DV:
        X, Y = make_tensor(bhjk, 7, "bf16", std=0.05), make_tensor(bjhp, 8, "bf16")
        ref = X.transpose(0, 1, 3, 2) @ Y.transpose(0, 2, 1, 3)
        zshape = bhjp
    elif which == ops.AG_DQ:
        X, Y = make_tensor(bhjk, 9, "bf16", std=0.05), make_tensor(bhjp, 10, "bf16")
        ref = X @ Y
        zshape = bhjp
    else:
        X, Y = make_tensor(bhjk, 11, "bf16", std=0.05), make_tensor(bhjp, 12, "bf16")
        ref = X.transpose(0, 1, 3, 2) @ Y
        zshape = bhjp
    Z = torch.full(zshape, float("nan"), dtype=torch.bfloat16, device="cuda")
    ops.enc_attn_gemm(ctx, which, B, H, J, P, dev(X), dev(Y), Z)
    torch.cuda.synchronize()
    ops.enc_set_option(ctx, ops.OPT_ATTN_BH, 1)
    got = host(Z)
    assert np.isfinite(got).all(), "unwritten output elements"
    # fp32 accumulation of exact bf16 products, one bf16 rounding of the result
    assert_parity(f"attn_gemm[{which}]", got, ref.astype(np.float64), "bf16")
    rel = np.abs(got - ref).max() / np.abs(ref).max()
    assert rel < 8e-3, rel
