"""Pins for oracle/philox.py (CPU only)."""
import os

import numpy as np
import pytest

from oracle import philox

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _kat_rows():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat_rows())
def test_philox_known_answers(ctr, key, out):
    w = philox.philox4x32_10(*ctr, *key)
    assert [int(x) for x in w] == out


def test_threshold_and_scale_closed_form():
    assert philox.dropout_threshold(0.0) == 0
    assert philox.dropout_scale(0.0) == 1.0
    assert philox.dropout_threshold(0.1) == 6554          # floor(6553.6 + 0.5)
    assert philox.dropout_scale(0.1) == 65536.0 / (65536.0 - 6554)
    assert philox.dropout_threshold(0.5) == 32768
    assert philox.dropout_scale(0.5) == 2.0
    with pytest.raises(ValueError):
        philox.dropout_threshold(1.0)
    with pytest.raises(ValueError):
        philox.dropout_threshold(-0.1)


def test_lane_mapping_matches_definition():
    """r(n) = 16-bit half (n&1) of word (n&7)>>1 of Philox(ctr=(g lo, g hi, sub lo, sub hi)),
    including a counter above 2^32 and a subsequence above 2^32."""
    seed = 0x123456789ABCDEF0
    sub = (5 << 32) + 3
    idx0 = (7 << 35) + 13          # g = idx0 >> 3 has a non-zero high word
    r = philox.lane_values(idx0, 40, seed, sub)
    for j in range(40):
        n = idx0 + j
        g, lane = n >> 3, n & 7
        w = philox.philox4x32_10(g & 0xFFFFFFFF, g >> 32, sub & 0xFFFFFFFF, sub >> 32,
                                 seed & 0xFFFFFFFF, seed >> 32)
        assert ((int(w[lane >> 1]) >> (16 * (lane & 1))) & 0xFFFF) == int(r[j])


def test_drop_rate_within_5_sigma():
    p = 0.1
    n = 1 << 22
    keep = philox.keep_mask(0, n, p, 2007000072, 0)
    p_eff = philox.dropout_threshold(p) / 65536.0
    sigma = np.sqrt(p_eff * (1 - p_eff) / n)
    assert abs((1.0 - keep.mean()) - p_eff) < 5 * sigma


def test_sites_and_seeds_are_independent_streams():
    a = philox.keep_mask(0, 1 << 16, 0.5, 1, philox.subsequence(0, 0))
    b = philox.keep_mask(0, 1 << 16, 0.5, 1, philox.subsequence(0, 1))
    c = philox.keep_mask(0, 1 << 16, 0.5, 2, philox.subsequence(0, 0))
    for x, y in ((a, b), (a, c)):
        agree = (x == y).mean()
        assert 0.48 < agree < 0.52


def test_batch_offset_slices_the_global_mask():
    shape = (6, 3, 5, 8)
    full = philox.keep_mask_tensor(shape, 0, 0.3, 42, 9)
    part = philox.keep_mask_tensor((2,) + shape[1:], 3, 0.3, 42, 9)
    assert np.array_equal(full[3:5], part)


def test_p_zero_keeps_everything():
    assert philox.keep_mask(17, 1000, 0.0, 5, 1).all()
