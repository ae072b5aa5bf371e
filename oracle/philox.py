"""Oracle: Philox4x32-10 counter-based RNG and the regenerable dropout keep mask.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  fp64 / exact-integer numpy.

Philox4x32-10 follows Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as
1, 2, 3" (SC'11), Random123 reference: ten rounds of
    (hi0, lo0) = mulhilo(M0, c0); (hi1, lo1) = mulhilo(M1, c2)
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
with the key bumped by the Weyl constants between rounds.  Pinned by the Random123
known-answer vectors in tests/golden/philox_kat.txt.

The paper draws dropout masks with cuRAND and stores them (App. A.2
"For dropout operators ... we use cuRAND"; Table A.1 dropout rows at PAPER.md:556,
:562, :565 output 2x their input because the mask is written).  The north star asks for
masks regenerated in backward; the mask definition is DESIGN.md reading R5
(SURVEY.md 8(c) "Dropout mask -- the exact definition"):

    subseq = 4*layer_id + site                 site 0 attn probs, 1 attn-out hidden,
                                               2 FFN activation, 3 FFN-out hidden
    n      = row-major logical index (global batch index)
    g      = n >> 3, lane = n & 7
    (w0..w3) = Philox4x32-10(ctr=(g lo, g hi, subseq lo, subseq hi), key=(seed lo, seed hi))
    r      = (w[lane >> 1] >> (16 * (lane & 1))) & 0xFFFF
    keep   = r >= T,  T = floor(p * 65536 + 1/2)
    scale  = 65536 / (65536 - T)
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF


def _mulhilo(m: int, x: np.ndarray):
    prod = np.uint64(m) * x.astype(np.uint64)
    return (prod >> np.uint64(32)).astype(np.uint64), (prod & np.uint64(MASK32)).astype(np.uint64)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10.  All arguments broadcastable integer arrays holding
    uint32 values; returns four uint64 arrays holding the uint32 output words."""
    c = [np.asarray(v, dtype=np.uint64) & np.uint64(MASK32) for v in (c0, c1, c2, c3)]
    k0 = np.asarray(k0, dtype=np.uint64) & np.uint64(MASK32)
    k1 = np.asarray(k1, dtype=np.uint64) & np.uint64(MASK32)
    for rnd in range(10):
        if rnd > 0:  # key schedule: bump before rounds 2..10
            k0 = (k0 + np.uint64(W0)) & np.uint64(MASK32)
            k1 = (k1 + np.uint64(W1)) & np.uint64(MASK32)
        hi0, lo0 = _mulhilo(M0, c[0])
        hi1, lo1 = _mulhilo(M1, c[2])
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return tuple(c)


def dropout_threshold(p: float) -> int:
    """T = floor(p * 65536 + 1/2), computed in fp64 (R5)."""
    if not (0.0 <= p < 1.0):
        raise ValueError("dropout p must be in [0, 1)")
    return int(np.floor(np.float64(p) * 65536.0 + 0.5))


def dropout_scale(p: float) -> float:
    """Inverted-dropout scale s = 65536 / (65536 - T) in fp64."""
    T = dropout_threshold(p)
    return 65536.0 / (65536.0 - T)


def subsequence(layer_id: int, site: int) -> int:
    """Philox subsequence of a dropout site (R5)."""
    if site not in (0, 1, 2, 3):
        raise ValueError(site)
    return 4 * int(layer_id) + site


def lane_values(index0: int, count: int, seed: int, subseq: int) -> np.ndarray:
    """The 16-bit random value r(n) for logical indices n = index0 .. index0+count-1."""
    if count == 0:
        return np.zeros(0, np.uint64)
    index0 = int(index0)
    g0 = index0 >> 3
    g1 = (index0 + count - 1) >> 3
    g = np.uint64(g0) + np.arange(g1 - g0 + 1, dtype=np.uint64)   # one Philox call per group
    seed = int(seed)
    subseq = int(subseq)
    w = philox4x32_10(g & np.uint64(MASK32), g >> np.uint64(32), subseq & MASK32, subseq >> 32,
                      seed & MASK32, seed >> 32)
    # r for lane = 0..7 of every group: lane -> word lane>>1, half lane&1
    r = np.empty((g.size, 8), dtype=np.uint64)
    for lane in range(8):
        r[:, lane] = (w[lane >> 1] >> np.uint64(16 * (lane & 1))) & np.uint64(0xFFFF)
    start = index0 - (g0 << 3)
    return r.reshape(-1)[start:start + count]


def keep_mask(index0: int, count: int, p: float, seed: int, subseq: int) -> np.ndarray:
    """Boolean keep decisions for logical indices index0 .. index0+count-1."""
    T = dropout_threshold(p)
    if T == 0:
        return np.ones(count, dtype=bool)
    return lane_values(index0, count, seed, subseq) >= np.uint64(T)


def keep_mask_tensor(shape, batch_offset: int, p: float, seed: int, subseq: int) -> np.ndarray:
    """Keep mask for a tensor whose leading dim is the LOCAL batch, indexed row-major
    with the GLOBAL batch index b + batch_offset (masks independent of
    the data-parallel partition)."""
    shape = tuple(int(s) for s in shape)
    per_batch = int(np.prod(shape[1:])) if len(shape) > 1 else 1
    total = int(np.prod(shape))
    m = keep_mask(int(batch_offset) * per_batch, total, p, seed, subseq)
    return m.reshape(shape)
