"""Oracle: AdamW parameter update in fp64 (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

The optimizer is outside the paper's method (the paper times encoder layers,
PAPER.md:147, :528); it completes the stack's training step.  The
definition followed, step by step, is AdamW with decoupled weight decay (Loshchilov &
Hutter; torch.optim.AdamW with amsgrad=False, maximize=False), at step t >= 1:

    g  = grad * grad_scale
    m  = b1 m + (1 - b1) g
    v  = b2 v + (1 - b2) g^2
    p  = p (1 - lr wd) - lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)

Pinned in tests/test_oracle_optim.py against torch.optim.AdamW (fp64, CPU) and the
closed form of the first step.
"""
from __future__ import annotations

import numpy as np


def adamw_step(p, m, v, grad, lr, b1, b2, eps, wd, t, grad_scale=1.0):
    """Returns (p, m, v) after one step; inputs are promoted to float64, not modified."""
    p = np.asarray(p, np.float64)
    m = np.asarray(m, np.float64)
    v = np.asarray(v, np.float64)
    g = np.asarray(grad, np.float64) * grad_scale
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    m_hat = m / (1.0 - b1 ** t)
    v_hat = v / (1.0 - b2 ** t)
    p = p * (1.0 - lr * wd) - lr * m_hat / (np.sqrt(v_hat) + eps)
    return p, m, v
