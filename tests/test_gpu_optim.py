"""enc_adamw_step (csrc/optim.cu) against the fp64 oracle (oracle/optim.py): master
parameters and moments over three steps (fp32 arithmetic, normwise 1e-5), the model copies
written through the segment table (bf16: the master rounded to nearest even; fp32: equal),
and the stack's training step updating every layer's parameters."""
import numpy as np
import pytest
import torch

from oracle.optim import adamw_step

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def test_adamw_kernel_vs_oracle():
    from paper_2007_00072_b200 import _abi
    from paper_2007_00072_b200.ops import Context
    lib = _abi.load()
    ctx = Context(0)
    rng = np.random.default_rng(11)
    sizes, dts = [1024, 8, 4096 + 12, 36], [0, 1, 0, 1]
    n = sum(sizes)
    p0 = rng.standard_normal(n).astype(np.float32)
    master = torch.tensor(p0, device="cuda")
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    outs = [torch.zeros(sz, device="cuda", dtype=torch.bfloat16 if dt == 0 else torch.float32)
            for sz, dt in zip(sizes, dts)]
    segs, off = [], 0
    nodec = [0, 1, 0, 1]   # segments exempt from weight decay
    wdv = np.zeros(n)
    for sz, dt, o, nd in zip(sizes, dts, outs, nodec):
        segs.append(_abi.enc_opt_segment(off, sz, o.data_ptr(), dt, nd))
        wdv[off:off + sz] = 0.0 if nd else 1.0
        off += sz
    c_segs = (_abi.enc_opt_segment * len(segs))(*segs)
    lr, b1, b2, eps, wd, gs = 1e-2, 0.9, 0.999, 1e-6, 0.01, 0.5
    P, M, V = p0.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(1, 4):
        g = (rng.standard_normal(n) * t).astype(np.float32)
        gd = torch.tensor(g, device="cuda")
        _abi.check("enc_adamw_step", lib.enc_adamw_step(
            ctx.ptr, n, master.data_ptr(), m.data_ptr(), v.data_ptr(), gd.data_ptr(), c_segs,
            len(segs), lr, b1, b2, eps, wd, t, gs, torch.cuda.current_stream().cuda_stream))
        P, M, V = adamw_step(P, M, V, g, lr, b1, b2, eps, wd * wdv, t, grad_scale=gs)
    torch.cuda.synchronize()
    mp = master.cpu().numpy().astype(np.float64)
    assert _rel(mp, P) <= 1e-5
    assert _rel(m.cpu().numpy().astype(np.float64), M) <= 1e-5
    assert _rel(v.cpu().numpy().astype(np.float64), V) <= 1e-5
    off = 0
    for sz, dt, o in zip(sizes, dts, outs):
        want = master[off:off + sz]
        if dt == 0:
            assert torch.equal(o, want.to(torch.bfloat16))
        else:
            assert torch.equal(o, want)
        off += sz


def test_adamw_rejects_bad_segments():
    from paper_2007_00072_b200 import _abi
    from paper_2007_00072_b200.ops import Context
    lib = _abi.load()
    ctx = Context(0)
    x = torch.zeros(64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    gap = (_abi.enc_opt_segment * 2)(_abi.enc_opt_segment(0, 32, x.data_ptr(), 1),
                                     _abi.enc_opt_segment(36, 28, x.data_ptr(), 1))
    assert lib.enc_adamw_step(ctx.ptr, 64, x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(),
                              gap, 2, 1e-3, 0.9, 0.999, 1e-8, 0.0, 1, 1.0, st) != 0
    one = (_abi.enc_opt_segment * 1)(_abi.enc_opt_segment(0, 64, x.data_ptr(), 1))
    assert lib.enc_adamw_step(ctx.ptr, 64, x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(),
                              one, 1, 1e-3, 0.9, 0.999, 1e-8, 0.0, 0, 1.0, st) != 0   # step 0
    assert lib.enc_adamw_step(ctx.ptr, 64, x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(),
                              one, 1, 1e-3, 1.0, 0.999, 1e-8, 0.0, 1, 1.0, st) != 0   # b1 = 1


def test_stack_train_step_updates_parameters():
    """Two training steps of a 2-layer bf16 stack: every layer's parameters equal the
    oracle's AdamW applied to that layer's gradients of each step (master in fp32, model
    copy rounded to bf16 / kept fp32)."""
    from paper_2007_00072_b200.layer import FFN_BUCKET, ATTN_BUCKET, WEIGHTS, LayerCfg
    from paper_2007_00072_b200.stack import EncoderStack
    from synth import Dims, SEED_WEIGHTS, make_inputs, make_params
    dims = Dims(B=2, J=128, H=2, P=64, U=512)
    st = EncoderStack(2, dims, "bf16", LayerCfg())
    st.set_params([make_params(dims, "bf16", "parity", seed=SEED_WEIGHTS + i) for i in range(2)])
    st.init_optimizer()
    inp = make_inputs(dims, "bf16")
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    order = FFN_BUCKET + ATTN_BUCKET
    ref = [lay.master.double().cpu().numpy() for lay in st.layers]
    mom = [(np.zeros_like(r), np.zeros_like(r)) for r in ref]
    # weight decay on the weight matrices only (biases, LayerNorm gamma/beta exempt)
    wdv = np.concatenate([np.full(st.layers[0].params[n].numel(), 1.0 if n in WEIGHTS else 0.0)
                          for n in order])
    for t in (1, 2):
        st.forward(X)
        st.backward(dY)
        grads = [lay.grad_flat.double().cpu().numpy() for lay in st.layers]
        st.optimizer_step(lr=1e-3)
        torch.cuda.synchronize()
        for i, lay in enumerate(st.layers):
            ref[i], m, v = adamw_step(ref[i], mom[i][0], mom[i][1], grads[i], 1e-3, 0.9, 0.999,
                                      1e-6, 0.01 * wdv, t)
            mom[i] = (m, v)
            got = lay.master.double().cpu().numpy()
            assert _rel(got, ref[i]) <= 1e-5
            off = 0
            for name in order:
                p = lay.params[name]
                want = lay.master[off:off + p.numel()].view(p.shape).to(p.dtype)
                assert torch.equal(p, want), name
                off += p.numel()
