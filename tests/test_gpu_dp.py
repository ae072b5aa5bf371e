"""Data parallelism on the CUDA path (SURVEY.md 8(e) "DP equivalence test"):
two ranks share the GPU over gloo, each runs the layer through libencoder.so on its batch
shard with batch_offset = r * B_local, then dp.allreduce_buckets sums the flat gradient
buckets.  Against one process running the global batch on the same GPU:
  * the dropout keep bits of every rank are bit-identical to the global run's slice;
  * every rank's output rows equal the global run's rows (bf16: bit for bit, the kernels are
    row-local and the tcgen05 tiles the same);
  * the all-reduced gradients equal the global-batch gradients (fp32: 1e-5 normwise; bf16:
    the two summation orders differ only by fp32 rounding, 1e-4 normwise)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = {
    "T_fp32": (dict(B=4, J=16, H=2, P=8, U=64), "fp32"),
    "fused_bf16": (dict(B=2, J=512, H=2, P=64, U=512), "bf16"),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_layer(dims, dtype, boff, B, world_inputs):
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    from synth import Dims, make_params
    d = Dims(B=B, J=dims.J, H=dims.H, P=dims.P, U=dims.U)
    prm = make_params(dims, dtype, "parity", weight_std=0.1)
    tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    sl = slice(boff, boff + B)
    X = torch.tensor(world_inputs["X"][sl], device="cuda").to(tdt)
    dY = torch.tensor(world_inputs["dY"][sl], device="cuda").to(tdt)
    M = torch.tensor(world_inputs["mask_bias"][sl], device="cuda")
    layer = EncoderLayer(d, dtype, LayerCfg(p_attn=0.1, p_hidden=0.1, p_ffn=0.1, layer_id=3,
                                            batch_offset=boff))
    layer.set_params(prm)
    Y = layer.forward(X, M)
    layer.backward(X, dY)
    torch.cuda.synchronize()
    keep = layer.saved_views()["keep_attn"].clone()
    return layer, Y.clone(), keep


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2007_00072_b200 import dp
    from synth import Dims, make_inputs
    dkw, dtype = CASES[case]
    dims = Dims(**dkw)
    inp = make_inputs(dims, dtype, key_padding=True)
    boff, B = dp.shard(dims.B, world, rank)
    layer, Y, keep = _run_layer(dims, dtype, boff, B, inp)
    buckets = [layer.ffn_bucket.cpu(), layer.attn_bucket.cpu()]
    dp.allreduce_buckets(buckets)
    q.put((rank, Y.float().cpu().numpy(), keep.cpu().numpy(),
           [b.numpy() for b in buckets]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", list(CASES))
def test_two_ranks_equal_global_batch(case):
    from synth import Dims, make_inputs
    dkw, dtype = CASES[case]
    dims = Dims(**dkw)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, Y, keep, buckets = q.get(timeout=300)
        res[r] = (Y, keep, buckets)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the global batch in this process
    torch.cuda.set_device(0)
    inp = make_inputs(dims, dtype, key_padding=True)
    layer, Yg, keepg = _run_layer(dims, dtype, 0, dims.B, inp)
    Yg = Yg.float().cpu().numpy()
    keepg = keepg.cpu().numpy()
    gref = [b.cpu().numpy().astype(np.float64) for b in (layer.ffn_bucket, layer.attn_bucket)]
    Bl = dims.B // 2
    for r in range(2):
        Y, keep, buckets = res[r]
        sl = slice(r * Bl, (r + 1) * Bl)
        if dtype == "bf16":   # same tcgen05 tiles per row: bitwise
            assert np.array_equal(Y, Yg[sl]), f"rank {r} output rows differ"
        else:                 # cuBLAS may pick another fp32 algorithm for another M
            assert np.abs(Y - Yg[sl]).max() <= 1e-6 * np.abs(Yg).max(), f"rank {r} rows"
        if dtype == "bf16":
            assert np.array_equal(keep, keepg[sl]), f"rank {r} attention keep bits differ"
        tol = 1e-5 if dtype == "fp32" else 1e-4
        for a, b in zip(buckets, gref):
            err = np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)
            assert err <= tol, (r, err)
