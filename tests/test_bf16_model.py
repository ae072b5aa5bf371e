"""The bf16-storage model (tests/bf16_model.py) is the oracle's chain with rounding at the
storage points: with the rounding disabled it must reproduce the oracle exactly, and with
it enabled its distance to the oracle must be of bf16 size (it is the yardstick of the
end-to-end bf16 parity test)."""
import numpy as np

import bf16_model
from oracle import encoder as E
from synth import CONFIGS, make_inputs, make_params


def _run(monkey_identity):
    dims = CONFIGS["T"]
    prm = make_params(dims, "fp32", "parity", weight_std=0.2)
    inp = make_inputs(dims, "fp32", key_padding=True)
    cfg = E.Cfg(p_attn=0.1, p_hidden=0.1, p_ffn=0.1)
    Yo, sv = E.encoder_layer_forward(inp["X"], prm, dims.H, cfg, inp["mask_bias"])
    dXo, go, _ = E.encoder_layer_backward(inp["dY"], inp["X"], prm, dims.H, cfg, sv)
    saved_r = bf16_model.r
    if monkey_identity:
        bf16_model.r = lambda a: np.asarray(a, np.float64)
    try:
        m = bf16_model.layer(inp["X"], prm, dims.H, cfg, inp["mask_bias"], dY=inp["dY"])
    finally:
        bf16_model.r = saved_r
    ref = {"Y": Yo, "dX": dXo}
    for n in go:
        ref["d" + n] = go[n]
    for n in ("Q", "K", "V", "P", "C", "X1", "xhat1", "h", "A1", "xhat2", "rstd1", "rstd2"):
        ref["saved." + n] = sv[n]
    return m, ref


def test_model_without_rounding_is_the_oracle():
    m, ref = _run(True)
    assert set(m) == set(ref)
    for n in ref:
        np.testing.assert_allclose(m[n], ref[n], rtol=1e-12, atol=1e-12, err_msg=n)


def test_model_error_is_bf16_sized():
    m, ref = _run(False)
    for n in ref:
        d = np.abs(m[n] - ref[n]).sum() / max(np.abs(ref[n]).sum(), 1e-300)
        assert d < 2e-2, (n, d)
        if n != "dbe2":   # dbe2 = column sums of the exact input dY
            assert d > 0, n
