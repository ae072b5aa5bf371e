"""Parity tolerances (north_star; R14), applied per output tensor:
  fp32: ||g - o||_inf / ||o||_inf <= 1e-5
  bf16: max|g - o| / rms(o) <= 2e-2  and  sum|g - o| / sum|o| <= 5e-3
Dropout masks and integer outputs are compared bit for bit elsewhere."""
import numpy as np

FP32_REL = 1e-5
BF16_MAX_OVER_RMS = 2e-2
BF16_MEAN_REL = 5e-3


def errors(g, o):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    d = np.abs(g - o)
    return {
        "max_rel": float(d.max() / max(np.abs(o).max(), 1e-300)) if d.size else 0.0,
        "max_over_rms": float(d.max() / max(np.sqrt((o * o).mean()), 1e-300)) if d.size else 0.0,
        "mean_rel": float(d.sum() / max(np.abs(o).sum(), 1e-300)) if d.size else 0.0,
        "max_abs": float(d.max()) if d.size else 0.0,
    }


def assert_parity(name, g, o, dtype, scale=1.0):
    """scale > 1 loosens the bf16 bounds for quantities whose error budget is derived in
    DESIGN.md R14 (never used for fp32)."""
    e = errors(g, o)
    if dtype == "fp32":
        ok = e["max_rel"] <= FP32_REL
    else:
        ok = e["max_over_rms"] <= BF16_MAX_OVER_RMS * scale and e["mean_rel"] <= BF16_MEAN_REL * scale
    assert ok, f"{name} [{dtype}] parity failed: {e}"
    return e
