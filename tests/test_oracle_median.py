"""Pins of the oracle's median column reduction (NEXT row f4, L#24):
hand-worked examples, s = 1 (a pure transpose, equal to the mean), invalid
handling, and numpy's median (an independent library routine) rounded half up
in exact rational arithmetic."""
from fractions import Fraction

import numpy as np

from oracle import oracle as orc

INV = 0xFFFF


def _one(vals, q=4, D=128, R=8):
    img = np.array([vals], dtype=np.uint16)
    return int(orc.reduce(img, len(vals), q, INV, D, R, mode=1)[0, 0])


def test_median_hand_examples():
    # Q = 4 (1/16 px), R = 8 (1/256 px)
    assert _one([16, 48, 32]) == 512          # {1, 3, 2} px -> 2 px
    assert _one([16, 48]) == 512              # (1 + 3) / 2 = 2 px
    assert _one([16, 24]) == 320              # (1 + 1.5) / 2 = 1.25 px
    assert _one([16, 17]) == 264              # 1.03125 px = 264/256 exactly
    assert _one([16, 160, 17, 18, 900]) == 288  # sorted 16 17 18 160 900 -> 18/16 px
    # Q = R = 8: (1 + 2) / 2 = 1.5 units of 1/256 -> half up -> 2
    assert _one([1, 2], q=8) == 2
    assert _one([2, 1, 7, 4], q=8) == 3       # (2 + 4) / 2 = 3


def test_median_invalid_and_range():
    assert _one([INV, 48, INV]) == 768         # only 3 px valid
    assert _one([INV, INV]) == -1
    assert _one([128 * 16, 32], D=128) == 512  # 128 px >= D is invalid -> median of {2}
    # 127.9375 px stays (L#27: only the object model clamps below D - 1/2)
    assert _one([127 * 16 + 15], D=128) == (127 * 16 + 15) * 16
    assert _one([127 * 16 + 7], D=128) == (127 * 16 + 7) * 16      # 127.4375 px: unchanged


def test_median_s1_is_transpose_and_equals_mean():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 128 * 16, size=(37, 23)).astype(np.uint16)
    img[rng.random(img.shape) < 0.1] = INV
    a = orc.reduce(img, 1, 4, INV, 128, mode=1)
    b = orc.reduce(img, 1, 4, INV, 128, mode=0)
    assert (a == b).all()
    want = img.T[:, ::-1].astype(np.int64) * 16                     # not clamped (L#27)
    assert (a == np.where(img.T[:, ::-1] == INV, -1, want)).all()


def test_median_matches_numpy_median():
    rng = np.random.default_rng(11)
    for s, q in [(2, 4), (3, 4), (5, 4), (6, 2), (7, 8), (10, 4)]:
        H, W = 19, 6 * s + s // 2
        D = 64
        img = rng.integers(0, (D + 2) << q, size=(H, W)).astype(np.uint16)   # some >= D
        img[rng.random(img.shape) < 0.2] = INV
        got = orc.reduce(img, s, q, INV, D, mode=1)
        for c in range(W // s):
            for r in range(H):
                seg = img[r, c * s:(c + 1) * s].astype(np.int64)
                seg = seg[(seg != INV) & (seg < (D << q))]
                want = -1
                if len(seg):
                    med = Fraction(int(round(2 * np.median(seg))), 2)     # exact: half-integers
                    x = med * 256 / (1 << q)
                    want = int((x + Fraction(1, 2)).__floor__())          # not clamped (L#27)
                assert got[c, H - 1 - r] == want, (s, q, c, r, seg)
