"""EncoderLayer: buffer management around encoder_layer_forward / encoder_layer_backward.

PyTorch supplies device memory (the caller-owned `saved`, `scratch`, parameter and
gradient buffers of include/encoder.h) and the CUDA stream; all compute runs in
libencoder.so.  Parameter gradients live in ONE flat fp32 buffer laid out as two
contiguous buckets so data parallelism can all-reduce them with one collective each
(DESIGN.md "Multi-GPU"): the FFN bucket (ready first in backward) then the attention bucket.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from ._abi import check
from .ops import Context

ACTS = {"gelu": _abi.ACT_GELU_ERF, "gelu_tanh": _abi.ACT_GELU_TANH, "relu": _abi.ACT_RELU}
TORCH_DT = {"bf16": torch.bfloat16, "fp32": torch.float32}
ABI_DT = {"bf16": _abi.ENC_BF16, "fp32": _abi.ENC_FP32}

FFN_BUCKET = ("W1", "W2", "b1", "b2", "g2", "be2")
WEIGHTS = ("Wqkv", "Wo", "W1", "W2")
ATTN_BUCKET = ("Wqkv", "Wo", "bqkv", "bo", "g1", "be1")


@dataclass
class LayerCfg:
    """enc_cfg (include/encoder.h); defaults follow DESIGN.md R3-R7."""
    p_attn: float = 0.1
    p_hidden: float = 0.1
    p_ffn: float = 0.1
    seed: int = 2007000072
    layer_id: int = 0
    batch_offset: int = 0
    ln_eps: float = 1e-5
    act: str = "gelu"
    causal: bool = False   # masking step: query j attends to keys k <= j

    def to_c(self) -> _abi.enc_cfg:
        return _abi.enc_cfg(self.p_attn, self.p_hidden, self.p_ffn, self.seed, self.layer_id,
                            self.batch_offset, self.ln_eps, ACTS[self.act], int(self.causal))


def param_shapes(I: int, U: int) -> dict:
    return {"Wqkv": (3 * I, I), "Wo": (I, I), "W1": (U, I), "W2": (I, U), "bqkv": (3 * I,),
            "bo": (I,), "b1": (U,), "b2": (I,), "g1": (I,), "be1": (I,), "g2": (I,), "be2": (I,)}


def c_dims(B, J, H, P, U) -> _abi.enc_dims:
    return _abi.enc_dims(B, J, J, H, P, P, H * P, U)


class EncoderLayer:
    """One BERT encoder layer (post-LN) on one GPU.

    dims: object with B (local batch), J, H, P, U.  dtype: 'bf16' or 'fp32'.
    """

    def __init__(self, dims, dtype: str = "bf16", cfg: LayerCfg | None = None,
                 ctx: Context | None = None, device=None, scratch: torch.Tensor | None = None):
        """scratch: optional shared temporaries buffer (layers of a stack run one at a time and
        may share it); allocated here when None or too small."""
        self.lib = _abi.load()
        self.B, self.J, self.H, self.P, self.U = dims.B, dims.J, dims.H, dims.P, dims.U
        self.I = self.H * self.P
        self.dtype = dtype
        self.tdt = TORCH_DT[dtype]
        self.adt = ABI_DT[dtype]
        self.cfg = cfg or LayerCfg()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.ctx = ctx or Context(self.device.index)
        self.dims = c_dims(self.B, self.J, self.H, self.P, self.U)
        sb, cb = ctypes.c_size_t(), ctypes.c_size_t()
        check("enc_layer_sizes", self.lib.enc_layer_sizes(ctypes.byref(self.dims), self.adt,
                                                          ctypes.byref(sb), ctypes.byref(cb)))
        self.saved = torch.empty(max(sb.value, 16), dtype=torch.uint8, device=self.device)
        if scratch is not None and scratch.numel() >= cb.value:
            self.scratch = scratch
        else:
            self.scratch = torch.empty(max(cb.value, 16), dtype=torch.uint8, device=self.device)
        shapes = param_shapes(self.I, self.U)
        self.params = {}
        for n, s in shapes.items():
            dt = self.tdt if n.startswith("W") else torch.float32
            self.params[n] = torch.zeros(s, dtype=dt, device=self.device)
        # flat fp32 gradient buffer: FFN bucket, then attention bucket
        order = FFN_BUCKET + ATTN_BUCKET
        sizes = [int(np.prod(shapes[n])) for n in order]
        self.grad_flat = torch.zeros(sum(sizes), dtype=torch.float32, device=self.device)
        self.grads = {}
        off = 0
        for n, sz in zip(order, sizes):
            self.grads[n] = self.grad_flat[off:off + sz].view(shapes[n])
            off += sz
        self.ffn_bucket = self.grad_flat[:sum(sizes[:len(FFN_BUCKET)])]
        self.attn_bucket = self.grad_flat[sum(sizes[:len(FFN_BUCKET)]):]
        self._refresh_structs()

    # ------------------------------------------------------------------ parameters
    def set_params(self, params: dict):
        for n, v in params.items():
            if n not in self.params:
                continue
            t = torch.as_tensor(np.asarray(v)) if not isinstance(v, torch.Tensor) else v
            self.params[n].copy_(t.to(self.params[n].dtype))
        self._refresh_structs()

    def _refresh_structs(self):
        self.c_params = _abi.enc_params(*[self.params[n].data_ptr() for n in _abi.PARAM_FIELDS])
        self.c_grads = _abi.enc_grads(*[self.grads[n].data_ptr() for n in _abi.PARAM_FIELDS])

    # ------------------------------------------------------------------ passes
    def _stream(self, stream):
        return (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream

    def forward(self, X: torch.Tensor, mask_bias: torch.Tensor | None = None,
                Y: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        assert X.dtype == self.tdt and X.is_contiguous() and X.is_cuda
        if Y is None:
            Y = torch.empty_like(X)
        cfg = self.cfg.to_c()
        check("encoder_layer_forward", self.lib.encoder_layer_forward(
            self.ctx.ptr, ctypes.byref(self.dims), self.adt, ctypes.byref(cfg),
            ctypes.byref(self.c_params), X.data_ptr(),
            None if mask_bias is None else mask_bias.data_ptr(), Y.data_ptr(),
            self.saved.data_ptr(), self.scratch.data_ptr(), self._stream(stream)))
        return Y

    BWD_FFN, BWD_ATTN = 1, 2

    def backward(self, X: torch.Tensor, dY: torch.Tensor, dX: torch.Tensor | None = None,
                 stream=None, part: int | None = None) -> torch.Tensor:
        """Whole backward, or one half (part=BWD_FFN: up to the final FFN-parameter
        gradients, then part=BWD_ATTN: the rest) so a gradient all-reduce can overlap."""
        assert dY.dtype == self.tdt and dY.is_contiguous() and dY.is_cuda
        if dX is None:
            dX = torch.empty_like(dY)
        cfg = self.cfg.to_c()
        args = (self.ctx.ptr, ctypes.byref(self.dims), self.adt, ctypes.byref(cfg),
                ctypes.byref(self.c_params), X.data_ptr(), self.saved.data_ptr(), dY.data_ptr(),
                dX.data_ptr(), ctypes.byref(self.c_grads), self.scratch.data_ptr())
        if part is None:
            check("encoder_layer_backward",
                  self.lib.encoder_layer_backward(*args, self._stream(stream)))
        else:
            check("encoder_layer_backward_part",
                  self.lib.encoder_layer_backward_part(*args, part, self._stream(stream)))
        return dX

    def step_host(self, X_host, dY_host, Y_host, dX_host, X_dev, dY_dev, Y_dev, dX_dev,
                  mask_bias=None, stream=None):
        """encoder_layer_step_host: H2D inputs, fwd + bwd, D2H Y and dX (host tensors
        should be pinned)."""
        cfg = self.cfg.to_c()
        check("encoder_layer_step_host", self.lib.encoder_layer_step_host(
            self.ctx.ptr, ctypes.byref(self.dims), self.adt, ctypes.byref(cfg),
            ctypes.byref(self.c_params), X_host.data_ptr(), dY_host.data_ptr(),
            Y_host.data_ptr(), dX_host.data_ptr(), X_dev.data_ptr(), dY_dev.data_ptr(),
            Y_dev.data_ptr(), dX_dev.data_ptr(),
            None if mask_bias is None else mask_bias.data_ptr(), ctypes.byref(self.c_grads),
            self.saved.data_ptr(), self.scratch.data_ptr(), self._stream(stream)))

    def prefetch_inputs(self, X_host, dY_host, X_dev, dY_dev, stream=None):
        """enc_prefetch_inputs: H2D copies of a step's inputs on the copy-in stream."""
        check("enc_prefetch_inputs", self.lib.enc_prefetch_inputs(
            self.ctx.ptr, ctypes.byref(self.dims), self.adt, X_host.data_ptr(),
            dY_host.data_ptr(), X_dev.data_ptr(), dY_dev.data_ptr(), self._stream(stream)))

    def step_host_pipelined(self, X_dev, dY_dev, Y_dev, dX_dev, Y_host, X_next_host=None,
                            dY_next_host=None, X_next_dev=None, dY_next_dev=None,
                            dX_prev_dev=None, dX_prev_host=None, mask_bias=None, stream=None):
        """encoder_layer_step_host_pipelined: one step on device-resident inputs; copies the
        next step's inputs in and the previous step's dX out while it runs (None to skip);
        Y copied back to Y_host.  Self-contained: all copies joined at the end."""
        cfg = self.cfg.to_c()

        def ptr(t):
            return None if t is None else t.data_ptr()
        check("encoder_layer_step_host_pipelined", self.lib.encoder_layer_step_host_pipelined(
            self.ctx.ptr, ctypes.byref(self.dims), self.adt, ctypes.byref(cfg),
            ctypes.byref(self.c_params), X_dev.data_ptr(), dY_dev.data_ptr(), Y_dev.data_ptr(),
            dX_dev.data_ptr(), Y_host.data_ptr(), ptr(X_next_host), ptr(dY_next_host),
            ptr(X_next_dev), ptr(dY_next_dev), ptr(dX_prev_dev), ptr(dX_prev_host),
            ptr(mask_bias), ctypes.byref(self.c_grads), self.saved.data_ptr(),
            self.scratch.data_ptr(), self._stream(stream)))

    # ------------------------------------------------------------------ configuration
    OPTION_KEYS = {"tc": 0, "fused": 1, "bh": 4, "direct": 5}

    def apply_config(self, fname):
        """Set the context's options from a configuration file written by the SSSP
        configuration selection (config_select.emit_configuration; "used to
        automatically define tensor layouts at the start of training")."""
        import json
        from .config_select import load_configuration
        with open(fname) as f:
            doc = json.load(f)
        if "chosen_options" in doc:   # per-operator selection (tools/select_config.py)
            for k, v in doc["chosen_options"].items():
                check("enc_set_option", self.lib.enc_set_option(self.ctx.ptr, int(k), int(v)))
            return doc["chosen_knobs"]
        _path, _total, knobs = load_configuration(fname)
        for k, v in knobs.items():
            check("enc_set_option",
                  self.lib.enc_set_option(self.ctx.ptr, self.OPTION_KEYS[k], int(v)))
        return knobs

    # ------------------------------------------------------------------ optimizer
    def init_optimizer(self):
        """AdamW state: fp32 master parameters in the gradient buffer's flat order (copied
        from the current parameters), first and second moments zeroed."""
        order = FFN_BUCKET + ATTN_BUCKET
        self.master = torch.cat([self.params[n].float().reshape(-1) for n in order])
        self.adam_m = torch.zeros_like(self.master)
        self.adam_v = torch.zeros_like(self.master)
        self.adam_t = 0
        segs, off = [], 0
        for n in order:
            t = self.params[n]
            dt = _abi.ENC_BF16 if t.dtype == torch.bfloat16 else _abi.ENC_FP32
            # biases and LayerNorm gamma/beta take no weight decay (the BERT recipe)
            segs.append(_abi.enc_opt_segment(off, t.numel(), t.data_ptr(), dt,
                                             0 if n in WEIGHTS else 1))
            off += t.numel()
        self.c_segs = (_abi.enc_opt_segment * len(segs))(*segs)

    def optimizer_step(self, lr=1e-4, betas=(0.9, 0.999), eps=1e-6, weight_decay=0.01,
                       grad_scale=1.0, stream=None):
        """enc_adamw_step on this layer's gradients (one launch): updates the master
        parameters and moments and rewrites the parameters the layer reads."""
        self.adam_t += 1
        check("enc_adamw_step", self.lib.enc_adamw_step(
            self.ctx.ptr, self.master.numel(), self.master.data_ptr(), self.adam_m.data_ptr(),
            self.adam_v.data_ptr(), self.grad_flat.data_ptr(), self.c_segs, len(self.c_segs),
            lr, betas[0], betas[1], eps, weight_decay, self.adam_t, grad_scale,
            self._stream(stream)))

    # ------------------------------------------------------------------ inspection
    def _pop_view(self, buf: torch.Tensor, ptr: int, ld: int) -> torch.Tensor:
        """[B,H,J,P] view of a P-wide attention operand with row stride `ld` (elements):
        ld == P head-major contiguous, else token-major (include/encoder.h qkv_ld)."""
        B, J, H, P = self.B, self.J, self.H, self.P
        es = torch.empty((), dtype=self.tdt).element_size()
        flat = buf.view(self.tdt)
        off = (ptr - buf.data_ptr()) // es
        if ld == P:
            return flat[off:off + B * H * J * P].view(B, H, J, P)
        return flat.as_strided((B, H, J, P), (J * ld, P, ld, 1), off)

    def saved_views(self) -> dict:
        """Tensors in `saved` (valid after forward()); Q, K, V may be strided views."""
        v = _abi.enc_saved_view()
        check("enc_saved_views", self.lib.enc_saved_views(self.ctx.ptr, ctypes.byref(self.dims),
                                                          self.adt, self.saved.data_ptr(),
                                                          ctypes.byref(v)))
        B, J, H, P, I, U = self.B, self.J, self.H, self.P, self.I, self.U
        shapes = {"P": (B, H, J, J), "A": (B, H, J, J), "C": (B, J, I), "X1": (B, J, I),
                  "xhat1": (B, J, I), "h": (B, J, U), "A1": (B, J, U), "xhat2": (B, J, I),
                  "rstd1": (B, J), "rstd2": (B, J), "keep_attn": (B, H, J, (J + 31) // 32)}
        base = self.saved.data_ptr()
        out = {}
        for n in _abi.SAVED_FIELDS:
            if n in ("Q", "K", "V"):
                out[n] = self._pop_view(self.saved, getattr(v, n), v.qkv_ld)
                continue
            off = getattr(v, n) - base
            dt = (torch.float32 if n.startswith("rstd") else
                  torch.int32 if n == "keep_attn" else self.tdt)
            numel = int(np.prod(shapes[n]))
            nbytes = numel * torch.empty((), dtype=dt).element_size()
            out[n] = self.saved[off:off + nbytes].view(dt).view(shapes[n])
        return out

    def bwd_views(self) -> dict:
        """Backward temporaries in `scratch` (valid after backward()); dQ, dK, dV may be
        strided views into dQKV."""
        v = _abi.enc_bwd_view()
        check("enc_bwd_views", self.lib.enc_bwd_views(self.ctx.ptr, ctypes.byref(self.dims),
                                                      self.adt, self.scratch.data_ptr(),
                                                      ctypes.byref(v)))
        B, J, H, P, I, U = self.B, self.J, self.H, self.P, self.I, self.U
        shapes = {"dY2": (B, J, I), "dA1": (B, J, U), "dh": (B, J, U), "dX1": (B, J, I),
                  "dYo": (B, J, I), "dC": (B, J, I), "dA": (B, H, J, J), "dS": (B, H, J, J),
                  "dQKV": (B, J, 3 * I)}
        base = self.scratch.data_ptr()
        es = torch.empty((), dtype=self.tdt).element_size()
        out = {}
        for n in _abi.BWD_FIELDS:
            if n in ("dQ", "dK", "dV"):
                out[n] = self._pop_view(self.scratch, getattr(v, n), v.dqkv_ld)
                continue
            off = getattr(v, n) - base
            numel = int(np.prod(shapes[n]))
            out[n] = self.scratch[off:off + numel * es].view(self.tdt).view(shapes[n])
        return out
