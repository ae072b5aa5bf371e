"""CrossAttention: buffer management around enc_xattn_forward / enc_xattn_backward -- the
encoder-decoder attention sublayer with the stacked key/value projection (
SURVEY.md 8(f)4).  Queries from X [B,J,I], keys and values from the memory Mem [B,K,I].
PyTorch supplies memory and the stream; every step runs in libencoder.so."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _abi
from ._abi import check
from .layer import ABI_DT, TORCH_DT, LayerCfg
from .ops import Context


def xattn_param_shapes(I: int) -> dict:
    return {"Wq": (I, I), "Wkv": (2 * I, I), "Wo": (I, I), "bq": (I,), "bkv": (2 * I,),
            "bo": (I,), "g": (I,), "be": (I,)}


class CrossAttention:
    def __init__(self, B, J, K, H, P, dtype="bf16", cfg: LayerCfg | None = None,
                 ctx: Context | None = None):
        self.lib = _abi.load()
        self.B, self.J, self.K, self.H, self.P = B, J, K, H, P
        self.I = H * P
        self.dtype, self.tdt, self.adt = dtype, TORCH_DT[dtype], ABI_DT[dtype]
        self.cfg = cfg or LayerCfg()
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.ctx = ctx or Context(self.device.index)
        self.dims = _abi.enc_dims(B, J, K, H, P, P, self.I, 0)
        sb, cb = ctypes.c_size_t(), ctypes.c_size_t()
        check("enc_xattn_sizes", self.lib.enc_xattn_sizes(ctypes.byref(self.dims), self.adt,
                                                          ctypes.byref(sb), ctypes.byref(cb)))
        self.saved = torch.empty(max(sb.value, 16), dtype=torch.uint8, device=self.device)
        self.scratch = torch.empty(max(cb.value, 16), dtype=torch.uint8, device=self.device)
        shapes = xattn_param_shapes(self.I)
        self.params = {n: torch.zeros(s, dtype=self.tdt if n.startswith("W") else torch.float32,
                                      device=self.device) for n, s in shapes.items()}
        self.grads = {n: torch.zeros(s, dtype=torch.float32, device=self.device)
                      for n, s in shapes.items()}
        self._refresh()

    def set_params(self, params: dict):
        for n, v in params.items():
            if n in self.params:
                t = v if isinstance(v, torch.Tensor) else torch.as_tensor(np.asarray(v))
                self.params[n].copy_(t.to(self.params[n].dtype))
        self._refresh()

    def _refresh(self):
        f = _abi.XATTN_PARAM_FIELDS
        self.c_params = _abi.enc_xattn_params(*[self.params[n].data_ptr() for n in f])
        self.c_grads = _abi.enc_xattn_grads(*[self.grads[n].data_ptr() for n in f])

    def forward(self, X, Mem, mask_bias=None, Y=None, stream=None):
        Y = torch.empty_like(X) if Y is None else Y
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check("enc_xattn_forward", self.lib.enc_xattn_forward(
            self.ctx.ptr, ctypes.byref(self.dims), self.adt, ctypes.byref(self.cfg.to_c()),
            ctypes.byref(self.c_params), X.data_ptr(), Mem.data_ptr(),
            None if mask_bias is None else mask_bias.data_ptr(), Y.data_ptr(),
            self.saved.data_ptr(), self.scratch.data_ptr(), s))
        return Y

    def backward(self, X, Mem, dY, stream=None):
        dX, dMem = torch.empty_like(X), torch.empty_like(Mem)
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        check("enc_xattn_backward", self.lib.enc_xattn_backward(
            self.ctx.ptr, ctypes.byref(self.dims), self.adt, ctypes.byref(self.cfg.to_c()),
            ctypes.byref(self.c_params), X.data_ptr(), Mem.data_ptr(), self.saved.data_ptr(),
            dY.data_ptr(), dX.data_ptr(), dMem.data_ptr(), ctypes.byref(self.c_grads),
            self.scratch.data_ptr(), s))
        return dX, dMem
