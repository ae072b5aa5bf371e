"""Encoder-decoder (cross) attention sublayer on the GPU (enc_xattn_*, SURVEY.md 8(f)4,
PAPER.md:646) against the fp64 oracle (oracle/encoder.py cross_attention_*, pinned to torch
in tests/test_oracle_xattn.py): fp32 end to end at 1e-5 on the cuBLAS attention path, bf16
on the tiled tcgen05 attention kernels with J != K (bf16-storage model bound, as the
encoder layer's end-to-end test), key padding and dropout."""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from synth import make_tensor
from tol import assert_parity, assert_parity_e2e

pytestmark = pytest.mark.gpu
SEED = 2007000072


def _params(I, dtype, std):
    out = {}
    for i, (n, s) in enumerate({"Wq": (I, I), "Wkv": (2 * I, I), "Wo": (I, I)}.items()):
        out[n] = make_tensor(s, 300 + i, dtype, std=std)
    for i, (n, s) in enumerate({"bq": (I,), "bkv": (2 * I,), "bo": (I,), "be": (I,)}.items()):
        out[n] = make_tensor(s, 310 + i, "fp32", std=0.1)
    out["g"] = 1.0 + make_tensor((I,), 320, "fp32", std=0.1)
    return out


def _run(B, J, K, H, P, dtype, p, masked, std):
    from paper_2007_00072_b200.layer import LayerCfg
    from paper_2007_00072_b200.xattn import CrossAttention
    I = H * P
    tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    X = make_tensor((B, J, I), 331, dtype)
    Mem = make_tensor((B, K, I), 332, dtype)
    dY = make_tensor((B, J, I), 333, dtype)
    prm = _params(I, dtype, std)
    mb = None
    if masked:
        mb = np.zeros((B, K), np.float32)
        mb[0, K // 2:] = -10000.0
    cfg = LayerCfg(p_attn=p, p_hidden=p, p_ffn=p, layer_id=5, batch_offset=2)
    xa = CrossAttention(B, J, K, H, P, dtype, cfg)
    xa.set_params(prm)
    dev = lambda a: torch.tensor(a, device="cuda").to(tdt)  # noqa: E731
    Mt = None if mb is None else torch.tensor(mb, device="cuda")
    Y = xa.forward(dev(X), dev(Mem), Mt)
    dX, dMem = xa.backward(dev(X), dev(Mem), dev(dY))
    torch.cuda.synchronize()
    ocfg = E.Cfg(p_attn=p, p_hidden=p, p_ffn=p, layer_id=5, batch_offset=2)
    Yo, sv = E.cross_attention_forward(X, Mem, prm, H, ocfg, mb)
    dXo, dMo, go = E.cross_attention_backward(dY, X, Mem, prm, H, ocfg, sv)
    h = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    gpu = {"Y": h(Y), "dX": h(dX), "dMem": h(dMem)}
    ref = {"Y": Yo, "dX": dXo, "dMem": dMo}
    for n in go:
        gpu["d" + n] = h(xa.grads[n])
        ref["d" + n] = go[n]
    return gpu, ref, (X, Mem, prm, H, ocfg, mb, dY)


@pytest.mark.parametrize("J,K", [(16, 24), (24, 8), (32, 32)])
@pytest.mark.parametrize("masked", [False, True])
def test_xattn_fp32(J, K, masked):
    gpu, ref, _ = _run(2, J, K, 2, 8, "fp32", 0.1, masked, 0.2)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


@pytest.mark.parametrize("J,K", [(128, 256), (256, 128), (128, 384)])
def test_xattn_bf16_tcgen05(J, K):
    """bf16, P = 64, J != K multiples of 128: the tiled tcgen05 attention contractions."""
    import bf16_model
    gpu, ref, (X, Mem, prm, H, ocfg, mb, dY) = _run(2, J, K, 2, 64, "bf16", 0.1, True, 0.05)
    mod = bf16_model.cross_attention(X, Mem, prm, H, ocfg, mb, dY=dY)
    # end to end through bf16 storage: the element bound, or errors of the size bf16
    # storage alone causes (tests/tol.py assert_parity_e2e)
    for n in gpu:
        assert_parity_e2e(n, gpu[n], ref[n], mod[n])
