"""ctypes declaration of the C ABI in include/encoder.h (libencoder.so).

Argument marshalling only: every computation happens inside libencoder.so.  The library
is required -- importing the binding without it raises, and there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, c_char_p, c_double, c_float, c_int, c_int64, c_size_t, c_uint32, c_uint64,
                    c_void_p)

LIB_PATH = os.environ.get("ENC_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libencoder.so")

ENC_BF16 = 0
ENC_FP32 = 1
ACT_GELU_ERF, ACT_GELU_TANH, ACT_RELU = 0, 1, 2


class enc_dims(ctypes.Structure):
    _fields_ = [(n, c_int) for n in ("B", "J", "K", "H", "P", "W", "I", "U")]


class enc_cfg(ctypes.Structure):
    _fields_ = [("p_attn", c_float), ("p_hidden", c_float), ("p_ffn", c_float),
                ("seed", c_uint64), ("layer_id", c_uint32), ("batch_offset", c_int64),
                ("ln_eps", c_float), ("act", c_int), ("causal", c_int)]


PARAM_FIELDS = ("Wqkv", "Wo", "W1", "W2", "bqkv", "bo", "b1", "b2", "g1", "be1", "g2", "be2")
GRAD_FIELDS = tuple("d" + n for n in PARAM_FIELDS)
SAVED_FIELDS = ("Q", "K", "V", "P", "A", "C", "X1", "xhat1", "h", "A1", "xhat2", "rstd1", "rstd2",
                "keep_attn")


class enc_params(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in PARAM_FIELDS]


class enc_grads(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in GRAD_FIELDS]


class enc_saved_view(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in SAVED_FIELDS] + [("qkv_ld", c_int64)]


XATTN_PARAM_FIELDS = ("Wq", "Wkv", "Wo", "bq", "bkv", "bo", "g", "be")


class enc_xattn_params(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in XATTN_PARAM_FIELDS]


class enc_xattn_grads(ctypes.Structure):
    _fields_ = [("d" + n, c_void_p) for n in XATTN_PARAM_FIELDS]


class enc_opt_segment(ctypes.Structure):
    _fields_ = [("begin", c_int64), ("n", c_int64), ("out", c_void_p), ("dtype", c_int),
                ("no_decay", c_int)]


BWD_FIELDS = ("dY2", "dA1", "dh", "dX1", "dYo", "dC", "dA", "dS", "dQ", "dK", "dV", "dQKV")


class enc_bwd_view(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in BWD_FIELDS] + [("dqkv_ld", c_int64)]


# name -> (restype, argtypes); mirrors include/encoder.h exactly
_SIGS = {
    "enc_create": (c_int, [POINTER(c_void_p), c_int]),
    "enc_destroy": (None, [c_void_p]),
    "enc_strerror": (c_char_p, [c_int]),
    "enc_last_cuda_error": (c_int, []),
    "enc_version": (c_char_p, []),
    "enc_layer_sizes": (c_int, [POINTER(enc_dims), c_int, POINTER(c_size_t), POINTER(c_size_t)]),
    "enc_saved_views": (c_int, [c_void_p, POINTER(enc_dims), c_int, c_void_p,
                                POINTER(enc_saved_view)]),
    "enc_bwd_views": (c_int, [c_void_p, POINTER(enc_dims), c_int, c_void_p,
                              POINTER(enc_bwd_view)]),
    "encoder_layer_forward": (c_int, [c_void_p, POINTER(enc_dims), c_int, POINTER(enc_cfg),
                                      POINTER(enc_params), c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p]),
    "encoder_layer_backward": (c_int, [c_void_p, POINTER(enc_dims), c_int, POINTER(enc_cfg),
                                       POINTER(enc_params), c_void_p, c_void_p, c_void_p,
                                       c_void_p, POINTER(enc_grads), c_void_p, c_void_p]),
    "encoder_layer_backward_part": (c_int, [c_void_p, POINTER(enc_dims), c_int, POINTER(enc_cfg),
                                            POINTER(enc_params), c_void_p, c_void_p, c_void_p,
                                            c_void_p, POINTER(enc_grads), c_void_p, c_int,
                                            c_void_p]),
    "encoder_layer_step_host": (c_int, [c_void_p, POINTER(enc_dims), c_int, POINTER(enc_cfg),
                                        POINTER(enc_params), c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p, POINTER(enc_grads), c_void_p, c_void_p,
                                        c_void_p]),
    "enc_adamw_step": (c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                               POINTER(enc_opt_segment), c_int, c_double, c_double, c_double,
                               c_double, c_double, c_int, c_double, c_void_p]),
    "enc_prefetch_inputs": (c_int, [c_void_p, POINTER(enc_dims), c_int, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p]),
    "encoder_layer_step_host_pipelined": (c_int, [c_void_p, POINTER(enc_dims), c_int,
                                                  POINTER(enc_cfg), POINTER(enc_params),
                                                  c_void_p, c_void_p, c_void_p, c_void_p,
                                                  c_void_p, c_void_p, c_void_p, c_void_p,
                                                  c_void_p, c_void_p, c_void_p, c_void_p,
                                                  POINTER(enc_grads), c_void_p, c_void_p,
                                                  c_void_p]),
    "enc_dropout_mask": (c_int, [c_int64, c_int64, c_float, c_uint64, c_uint64, c_void_p,
                                 c_void_p]),
    "enc_aib_fwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                            c_void_p, c_void_p, c_void_p, c_void_p]),
    "enc_aib_bwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                            c_void_p, c_void_p, c_void_p, c_void_p]),
    "enc_bsb_fwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_float, c_void_p,
                            c_void_p, c_float, c_uint64, c_uint64, c_int64, c_void_p, c_void_p,
                            c_int, c_void_p]),
    "enc_bsb_bwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_float, c_void_p,
                            c_void_p, c_float, c_uint64, c_uint64, c_int64, c_void_p, c_void_p]),
    "enc_bdrln_fwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                              c_void_p, c_void_p, c_void_p, c_float, c_float, c_uint64,
                              c_uint64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "enc_bdrln_bwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                              c_void_p, c_void_p, c_float, c_uint64, c_uint64, c_int64,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "enc_bad_fwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                            c_float, c_uint64, c_uint64, c_int64, c_void_p, c_void_p, c_void_p]),
    "enc_bad_bwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                            c_float, c_uint64, c_uint64, c_int64, c_void_p, c_void_p, c_void_p]),
    "enc_num_ops": (c_int, []),
    "enc_op_name": (c_char_p, [c_int]),
    "enc_set_timing": (c_int, [c_void_p, c_uint64]),
    "enc_op_times": (c_int, [c_void_p, POINTER(c_float)]),
    "enc_launch_count": (c_uint64, [c_void_p]),
    "enc_attn_gemm": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                              c_void_p, c_void_p]),
    "enc_set_option": (c_int, [c_void_p, c_int, c_int]),
    "enc_attn_fwd_fused": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_float, c_void_p,
                                   c_void_p, c_void_p, c_float, c_uint64, c_uint64, c_int64,
                                   c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "enc_attn_bwd_fused": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_float, c_void_p,
                                   c_void_p, c_void_p, c_float, c_uint64, c_uint64, c_int64,
                                   c_void_p, c_void_p, c_void_p]),
    "enc_attn_fwd_fused_av": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_float, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_float, c_uint64, c_uint64,
                                      c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int,
                                      c_void_p]),
    "enc_attn_bwd_fused_dc": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_float, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p, c_float, c_uint64,
                                      c_uint64, c_int64, c_void_p, c_void_p, c_void_p]),
    "enc_bei": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "enc_xattn_sizes": (c_int, [POINTER(enc_dims), c_int, POINTER(c_size_t), POINTER(c_size_t)]),
    "enc_xattn_forward": (c_int, [c_void_p, POINTER(enc_dims), c_int, POINTER(enc_cfg),
                                  POINTER(enc_xattn_params), c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p]),
    "enc_xattn_backward": (c_int, [c_void_p, POINTER(enc_dims), c_int, POINTER(enc_cfg),
                                   POINTER(enc_xattn_params), c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, POINTER(enc_xattn_grads),
                                   c_void_p, c_void_p]),
    "enc_attn_keep_bits": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_float, c_uint64,
                                   c_uint64, c_int64, c_void_p, c_void_p]),
    "enc_attn_fwd_fused_bits": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_float, c_void_p,
                                        c_void_p, c_void_p, c_float, c_uint64, c_uint64, c_int64,
                                        c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "enc_wgemm": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_int64, c_int, c_void_p,
                          c_int64, c_int, c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p]),
    "enc_linear1_bad_fwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                                    c_void_p, c_int, c_float, c_uint64, c_uint64, c_int64,
                                    c_void_p, c_void_p, c_void_p]),
    "enc_linear2_dx_bad_bwd": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_void_p,
                                       c_void_p, c_void_p, c_int, c_float, c_uint64, c_uint64,
                                       c_int64, c_void_p, c_void_p, c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class EncError(RuntimeError):
    def __init__(self, fn, code, lib):
        msg = lib.enc_strerror(code).decode()
        if code == -4:
            msg += f" (cudaError {lib.enc_last_cuda_error()})"
        super().__init__(f"{fn} failed: {code} {msg}")
        self.code = code


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libencoder.so and declare every entry point.  Raises if it is missing."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib


def check(fn_name: str, code: int):
    if code != 0:
        raise EncError(fn_name, code, load())
