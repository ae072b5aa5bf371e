"""Pins of oracle/optim.py (AdamW): torch.optim.AdamW in fp64 over several steps, and the
closed form of the first step (m_hat = g, v_hat = g^2, so the update is
-lr * g / (|g| + eps) - lr * wd * p)."""
import numpy as np
import pytest
import torch

from oracle.optim import adamw_step


@pytest.mark.parametrize("wd,scale", [(0.0, 1.0), (0.01, 1.0), (0.1, 0.5)])
def test_adamw_matches_torch(wd, scale):
    rng = np.random.default_rng(7)
    p0 = rng.standard_normal(257)
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    tp = torch.tensor(p0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.AdamW([tp], lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd)
    p, m, v = p0.copy(), np.zeros_like(p0), np.zeros_like(p0)
    for t in range(1, 6):
        g = rng.standard_normal(257) * (1 + t)
        tp.grad = torch.tensor(g * scale, dtype=torch.float64)
        opt.step()
        p, m, v = adamw_step(p, m, v, g, lr, b1, b2, eps, wd, t, grad_scale=scale)
        np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-13, atol=1e-15)
    st = opt.state[tp]
    np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-13)
    np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-13)


def test_adamw_first_step_closed_form():
    rng = np.random.default_rng(3)
    p0, g = rng.standard_normal(64), rng.standard_normal(64)
    lr, wd, eps = 0.01, 0.1, 1e-8
    p, m, v = adamw_step(p0, np.zeros(64), np.zeros(64), g, lr, 0.9, 0.999, eps, wd, 1)
    np.testing.assert_allclose(p, p0 - lr * wd * p0 - lr * g / (np.abs(g) + eps), rtol=1e-12)
    np.testing.assert_allclose(m, 0.1 * g, rtol=1e-15)
    np.testing.assert_allclose(v, 0.001 * g * g, rtol=1e-12)
