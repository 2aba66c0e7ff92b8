"""Space-to-depth stem lowering (host side): the 7x7 / stride-2 / pad-3 conv
on a <= 4-channel image equals a 4x4 / stride-1 / pad-1 conv on its 2x2
blocks behind a zero first row and column; the weight transform is exactly
invertible."""

import numpy as np

from oracle import levnet_oracle as O
from paper_2509_22857_b200.lowering import s2d_weight, s2d_weight_back


def _s2d(x):
    c, h, w = x.shape
    out = np.zeros((4 * c, h // 2, w // 2))
    for dy in range(2):
        for dx in range(2):
            out[(dy * 2 + dx) * c:(dy * 2 + dx + 1) * c] = x[:, dy::2, dx::2]
    return out


def test_s2d_weight_roundtrip():
    rng = np.random.default_rng(0)
    w = rng.normal(size=(5, 3, 7, 7))
    np.testing.assert_array_equal(s2d_weight_back(s2d_weight(w), {"cin": 3, "k": 7}), w)


def test_s2d_conv_equivalence():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(3, 16, 20))
    w = rng.normal(size=(4, 3, 7, 7))
    b = rng.normal(size=4)
    want = O.conv2d(x, w, b, 2, 3)
    xs = np.pad(_s2d(x), ((0, 0), (1, 0), (1, 0)))  # the ingest's zero first row / column
    got = O.conv2d(xs, s2d_weight(w), b, 1, 1)
    assert got.shape == want.shape
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)
