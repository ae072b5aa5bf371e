"""Decoder of the ENC_KEEP_BITS word layout (include/encoder.h): word w of a row holds the
keep flags of columns 32w..32w+31; column 32w + 8c + u is bit (u odd ? 31 : 15) - u//2 - 4c.
Test-side only: the expected flags always come from oracle.philox."""
import numpy as np


def bit_of(c: int, u: int) -> int:
    return (31 if u & 1 else 15) - u // 2 - 4 * c


def decode(words, K: int) -> np.ndarray:
    """words: integer array [..., ceil(K/32)] (any signed/unsigned 32-bit view) ->
    bool keep mask [..., K]."""
    w = np.asarray(words).astype(np.int64) & 0xFFFFFFFF
    out = np.zeros(w.shape[:-1] + (w.shape[-1] * 32,), dtype=bool)
    for c in range(4):
        for u in range(8):
            out[..., 8 * c + u::32] = (w >> bit_of(c, u)) & 1
    return out[..., :K]
