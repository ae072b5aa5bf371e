"""Parity tolerances (north_star; reading DESIGN.md R14), applied per output tensor o
(oracle, fp64) vs g (GPU):

  fp32: ||g - o||_inf / ||o||_inf <= 1e-5
  bf16: |g - o| <= 2e-2 * rms(o) + 2^-8 * |o| for every element   ("max-abs 2e-2", scaled)
        and sum|g - o| / sum|o| <= 5e-3                           ("mean relative 5e-3")

The north star's bf16 "max-abs 2e-2" cannot be read as an unscaled absolute bound: storing
a value |o| in [8, 16) in bf16 alone moves it by up to 2^-5 = 0.031 (half an ulp), and the
raw dW entries at config L are ~20.  The bound is therefore the absolute 2e-2 taken
relative to the tensor's scale, atol = 2e-2 * rms(o), plus the storage rounding of the
element itself: a bf16 store moves |o| by at most half an ulp = 2^-9 |o|, and an output
computed from bf16-stored inputs of the same magnitude carries at most one more such
rounding, so rtol = 2 * 2^-9 = 2^-8.  Dropout masks and integer outputs are compared bit
for bit elsewhere."""
import numpy as np

FP32_REL = 1e-5
BF16_TOL = 2e-2
BF16_RTOL = 2.0 ** -8
BF16_MEAN_REL = 5e-3


def errors(g, o):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    d = np.abs(g - o)
    if not d.size:
        return {"max_rel": 0.0, "mixed": 0.0, "mean_rel": 0.0, "max_abs": 0.0,
                "max_over_rms": 0.0}
    rms = max(np.sqrt((o * o).mean()), 1e-300)
    return {
        "max_rel": float(d.max() / max(np.abs(o).max(), 1e-300)),
        # <= 1 for bf16: |g - o| / (2e-2 rms + 2^-8 |o|)
        "mixed": float((d / (BF16_TOL * rms + BF16_RTOL * np.abs(o))).max()),
        "mean_rel": float(d.sum() / max(np.abs(o).sum(), 1e-300)),
        "max_abs": float(d.max()),
        "max_over_rms": float(d.max() / rms),
    }


def assert_parity(name, g, o, dtype):
    e = errors(g, o)
    if dtype == "fp32":
        ok = e["max_rel"] <= FP32_REL
    else:
        ok = e["mixed"] <= 1.0 and e["mean_rel"] <= BF16_MEAN_REL
    assert ok, f"{name} [{dtype}] parity failed: {e}"
    return e
