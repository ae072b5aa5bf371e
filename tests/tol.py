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


def e2e_report(g, o, m):
    """Errors of the GPU (g) and of the bf16-storage model (m, tests/bf16_model.py) against
    the fp64 oracle (o), and their ratios."""
    e, em = errors(g, o), errors(m, o)
    g64, o64, m64 = (np.asarray(x, np.float64) for x in (g, o, m))
    rms_g = float(np.sqrt(((g64 - o64) ** 2).mean())) if o64.size else 0.0
    rms_m = float(np.sqrt(((m64 - o64) ** 2).mean())) if o64.size else 0.0
    return {"gpu": e, "model": em, "rms_err_gpu": rms_g, "rms_err_model": rms_m,
            "rms_ratio": rms_g / max(rms_m, 1e-300),
            "max_ratio": e["max_abs"] / max(em["max_abs"], 1e-300)}


E2E_RMS_RATIO = 1.25
E2E_MAX_RATIO = 2.0


def assert_parity_e2e(name, g, o, m):
    """bf16 end to end (R14): the north star's mean relative error <= 5e-3, and the
    element bound of assert_parity -- or, where bf16 storage alone already exceeds it (the
    bf16-storage model m misses it too), errors of the same size as that model's: RMS error
    within 1.25x and max error within 2x of the model's distance to the oracle."""
    rep = e2e_report(g, o, m)
    e = rep["gpu"]
    ok = e["mean_rel"] <= BF16_MEAN_REL and (
        e["mixed"] <= 1.0 or (rep["model"]["mixed"] > 1.0 / E2E_MAX_RATIO
                              and rep["rms_ratio"] <= E2E_RMS_RATIO
                              and rep["max_ratio"] <= E2E_MAX_RATIO))
    assert ok, f"{name} [bf16 end to end] parity failed: {rep}"
    return rep
