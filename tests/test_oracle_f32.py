"""Pins of the oracle's f32 input decode (a1, L#28): a float disparity
in pixels, invalid if not finite, negative or >= D, converted once to the 1/256
grid half up, then reduced like fixed point.  Hand examples, the invalid cases,
and the identity with the u16 path on values on the 1/16 grid."""
import numpy as np

from oracle import oracle as orc


def _one(vals, D=128, s=None):
    img = np.array([vals], dtype=np.float32)
    return int(orc.reduce(img, s or len(vals), 0, 0, D)[0, 0])


def test_f32_hand_examples():
    assert _one([1.5, 2.0, 3.0]) == 555                 # (384 + 512 + 768) / 3 = 554.67 -> 555
    assert _one([1.001953125]) == 257                    # 256.5 -> half up
    assert _one([1.0019]) == 256                         # 256.49: below the half
    assert _one([0.0, -0.0]) == 0


def test_f32_invalid_cases():
    D = 64
    for bad in (np.nan, np.inf, -np.inf, -0.25, 64.0, 100.0):
        assert _one([bad, 10.0], D=D) == 2560           # only 10 px counts
        assert _one([bad], D=D) == -1
    assert _one([63.99], D=D) == 16381                   # floor(63.99 * 256 + 1/2), not clamped (L#27)


def test_f32_equals_u16_on_the_sixteenth_grid():
    rng = np.random.default_rng(9)
    k = rng.integers(0, 128 * 16, size=(23, 40)).astype(np.uint16)
    k[rng.random(k.shape) < 0.1] = 0xFFFF
    f = np.where(k == 0xFFFF, np.nan, k.astype(np.float64) / 16).astype(np.float32)
    for mode in (0, 1):
        for s in (1, 3, 5, 8):
            a = orc.reduce(k, s, 4, 0xFFFF, 128, mode=mode)
            b = orc.reduce(f, s, 0, 0, 128, mode=mode)
            assert (a == b).all(), (mode, s)
