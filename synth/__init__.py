"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no softmax, LayerNorm, dropout,
activation, contraction).  It only draws random numbers with numpy's PCG64 and rounds
them to the storage precision of the path under test, so that the oracle (fp64 CPU,
`oracle/`) and the CUDA path (`paper_2007_00072_b200/`) see bit-identical inputs.
Neither of those imports the other; both import this.

Recipe:
  * X, dY ~ N(0, 1); weights ~ N(0, 0.02^2) truncated at 2 sigma (BERT init).
  * parity init: biases ~ N(0, 0.02^2), gamma ~ 1 + N(0, 0.1^2), beta ~ N(0, 0.1^2).
  * bench init: biases 0, gamma 1, beta 0 (values do not change speed).
  * "sharp" variant: weight std 0.06 so softmax rows are peaked.
  * key-padding case: per-sample valid lengths ~ U[J/2, J], additive bias -10000.
  * Seeds: weights 1234, inputs 5678 (generated for the GLOBAL batch, then sliced per
    rank), dropout seed 2007000072.
"""
from __future__ import annotations

from dataclasses import dataclass, asdict

import numpy as np

SEED_WEIGHTS = 1234
SEED_INPUTS = 5678
SEED_DROPOUT = 2007000072


@dataclass(frozen=True)
class Dims:
    """Paper notation (Fig. 1 caption): B batch, J/K sequence lengths,
    H heads, P/W key/value projection size, I = H*P embedding, U FFN width."""
    B: int
    J: int
    H: int
    P: int
    U: int

    @property
    def K(self) -> int:  # self-attention: K == J
        return self.J

    @property
    def W(self) -> int:  # W == P
        return self.P

    @property
    def I(self) -> int:  # noqa: E743
        return self.H * self.P

    def with_batch(self, B: int) -> "Dims":
        return Dims(B=B, J=self.J, H=self.H, P=self.P, U=self.U)

    def as_dict(self) -> dict:
        d = asdict(self)
        d.update(K=self.K, W=self.W, I=self.I)
        return d


# BASELINE.json "configs".
CONFIGS = {
    "T": Dims(B=2, J=16, H=2, P=8, U=64),          # tiny, fp32, oracle in seconds
    "L": Dims(B=8, J=512, H=16, P=64, U=4096),     # paper's BERT-large layer
    "Bb": Dims(B=96, J=128, H=12, P=64, U=3072),   # BERT-base, per GPU
}


def sweep_dims(J: int) -> Dims:
    """Config SW: BSB/BDRLN sweep at B=8, H=16, I=1024, J = 128..4096."""
    return Dims(B=8, J=J, H=16, P=64, U=4096)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32 that
    are exactly representable in bf16.  Pure storage rounding, no method arithmetic."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    u = ((u + rounding) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32).reshape(a.shape)


def to_storage(a: np.ndarray, dtype: str) -> np.ndarray:
    """float32 array representable in the storage dtype ('bf16' or 'fp32')."""
    a = np.asarray(a, dtype=np.float32)
    if dtype == "bf16":
        return bf16_round(a)
    if dtype == "fp32":
        return np.ascontiguousarray(a)
    raise ValueError(dtype)


def _trunc_normal(rng: np.random.Generator, shape, std: float) -> np.ndarray:
    x = rng.standard_normal(size=shape, dtype=np.float32)
    bad = np.abs(x) > 2.0
    while bad.any():
        x[bad] = rng.standard_normal(size=int(bad.sum()), dtype=np.float32)
        bad = np.abs(x) > 2.0
    return x * np.float32(std)


PARAM_NAMES = ("Wqkv", "bqkv", "Wo", "bo", "W1", "b1", "W2", "b2", "g1", "be1", "g2", "be2")
WEIGHT_NAMES = ("Wqkv", "Wo", "W1", "W2")


def make_params(dims: Dims, dtype: str = "bf16", init: str = "parity",
                seed: int = SEED_WEIGHTS, weight_std: float = 0.02) -> dict:
    """Layer parameters in nn.Linear convention (W[out, in]); weights in the activation
    storage dtype, biases / gamma / beta always fp32."""
    rng = np.random.default_rng(seed)
    I, U = dims.I, dims.U
    p = {
        "Wqkv": to_storage(_trunc_normal(rng, (3 * I, I), weight_std), dtype),
        "Wo": to_storage(_trunc_normal(rng, (I, I), weight_std), dtype),
        "W1": to_storage(_trunc_normal(rng, (U, I), weight_std), dtype),
        "W2": to_storage(_trunc_normal(rng, (I, U), weight_std), dtype),
    }
    if init == "parity":
        p["bqkv"] = (rng.standard_normal(3 * I, dtype=np.float32) * np.float32(0.02))
        p["bo"] = (rng.standard_normal(I, dtype=np.float32) * np.float32(0.02))
        p["b1"] = (rng.standard_normal(U, dtype=np.float32) * np.float32(0.02))
        p["b2"] = (rng.standard_normal(I, dtype=np.float32) * np.float32(0.02))
        p["g1"] = 1.0 + rng.standard_normal(I, dtype=np.float32) * np.float32(0.1)
        p["be1"] = rng.standard_normal(I, dtype=np.float32) * np.float32(0.1)
        p["g2"] = 1.0 + rng.standard_normal(I, dtype=np.float32) * np.float32(0.1)
        p["be2"] = rng.standard_normal(I, dtype=np.float32) * np.float32(0.1)
    elif init == "bench":
        for n, size in (("bqkv", 3 * I), ("bo", I), ("b1", U), ("b2", I), ("be1", I), ("be2", I)):
            p[n] = np.zeros(size, np.float32)
        p["g1"] = np.ones(I, np.float32)
        p["g2"] = np.ones(I, np.float32)
    else:
        raise ValueError(init)
    for n in PARAM_NAMES:
        p[n] = np.ascontiguousarray(p[n], dtype=np.float32)
    return p


def make_inputs(dims: Dims, dtype: str = "bf16", seed: int = SEED_INPUTS,
                key_padding: bool = False) -> dict:
    """Global-batch inputs: X [B,J,I], dY [B,J,I] (storage dtype), and optionally an
    additive key-padding bias M [B,K] (fp32; 0 for valid keys, -10000 for padded)."""
    rng = np.random.default_rng(seed)
    B, J, I = dims.B, dims.J, dims.I
    out = {
        "X": to_storage(rng.standard_normal((B, J, I), dtype=np.float32), dtype),
        "dY": to_storage(rng.standard_normal((B, J, I), dtype=np.float32), dtype),
        "mask_bias": None,
    }
    if key_padding:
        lens = rng.integers(J // 2, J + 1, size=B)
        m = np.zeros((B, dims.K), np.float32)
        for b in range(B):
            m[b, lens[b]:] = -10000.0
        out["mask_bias"] = m
    return out


def make_tensor(shape, seed: int, dtype: str = "bf16", std: float = 1.0,
                mean: float = 0.0) -> np.ndarray:
    """A seeded N(mean, std^2) tensor rounded to the storage dtype (per-op parity)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(shape, dtype=np.float32) * np.float32(std) + np.float32(mean)
    return to_storage(x, dtype)


def make_positive_rows(shape, seed: int, dtype: str = "bf16") -> np.ndarray:
    """Seeded rows that look like softmax outputs (positive, each row sums to ~1).
    Used as the saved-P input of the BSB-bwd parity test; drawn as normalised
    uniforms, which is input generation, not the method's softmax."""
    rng = np.random.default_rng(seed)
    x = rng.random(shape, dtype=np.float32) + np.float32(1e-3)
    x = x / x.sum(axis=-1, keepdims=True)
    return to_storage(x, dtype)
