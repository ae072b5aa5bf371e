"""Data-parallel host logic on CPU (gloo, world size 2): batch sharding with batch_offset,
the two-bucket flat gradient layout, and the SUM all-reduce reproduce the single-process
global-batch gradients (the per-rank compute here is the oracle; on the GPU box the same
dp.py / layer.py code drives libencoder.so under NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import encoder as E
from paper_2007_00072_b200 import dp
from paper_2007_00072_b200.layer import ATTN_BUCKET, FFN_BUCKET, param_shapes
from synth import Dims, make_inputs, make_params

DIMS = Dims(B=4, J=8, H=2, P=4, U=16)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _flat(grads, shapes):
    return [torch.tensor(np.concatenate([np.asarray(grads[n], np.float64).reshape(-1)
                                         for n in bucket]), dtype=torch.float64)
            for bucket in (FFN_BUCKET, ATTN_BUCKET)]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prm = make_params(DIMS, "fp32", "parity", weight_std=0.2)
    inp = make_inputs(DIMS, "fp32", key_padding=True)
    boff, B = dp.shard(DIMS.B, world, rank)
    cfg = E.Cfg(p_attn=0.2, p_hidden=0.2, p_ffn=0.2, layer_id=1, batch_offset=boff)
    sl = slice(boff, boff + B)
    Y, sv = E.encoder_layer_forward(inp["X"][sl], prm, DIMS.H, cfg, inp["mask_bias"][sl])
    _, g, _ = E.encoder_layer_backward(inp["dY"][sl], inp["X"][sl], prm, DIMS.H, cfg, sv)
    buckets = _flat(g, param_shapes(DIMS.I, DIMS.U))
    dp.allreduce_buckets(buckets)
    t = dp.max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put(([b.numpy() for b in buckets], t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard():
    assert dp.shard(16, 4, 3) == (12, 4)
    with pytest.raises(ValueError):
        dp.shard(10, 4, 0)


def test_world2_allreduce_equals_global_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    buckets, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    prm = make_params(DIMS, "fp32", "parity", weight_std=0.2)
    inp = make_inputs(DIMS, "fp32", key_padding=True)
    cfg = E.Cfg(p_attn=0.2, p_hidden=0.2, p_ffn=0.2, layer_id=1)
    Y, sv = E.encoder_layer_forward(inp["X"], prm, DIMS.H, cfg, inp["mask_bias"])
    _, g, _ = E.encoder_layer_backward(inp["dY"], inp["X"], prm, DIMS.H, cfg, sv)
    ref = _flat(g, param_shapes(DIMS.I, DIMS.U))
    for a, b in zip(buckets, ref):
        assert np.allclose(a, b.numpy(), rtol=1e-12, atol=1e-12)
