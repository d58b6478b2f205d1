"""Pins of the oracle's data term, ground model, reduction and span mean against
values fixed outside the oracle (SPEC worked examples, closed forms, exact
rational arithmetic).  CPU only."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _model(**kw):
    base = dict(h=8, D=128, q=0, sigma=(1.0, 1.0, 1.0), p_out=0.15, a_norm=1.0)
    base.update(kw)
    return orc.Model(**base)


def test_eq4_spec_worked_examples():
    g = json.load(open(os.path.join(GOLD, "eq4_spec.json")))
    m = _model()
    assert abs(orc.eq4(m, 0.0, 1.0) - g["cost_at_d_eq_f"]) < g["abs_tol"]
    assert abs(orc.eq4(m, 1000.0, 1.0) - g["cost_far"]) < g["abs_tol"]


def test_eq4_branches_and_properties():
    """cap bound, monotone in |d-f|, symmetric, and the
    Gaussian branch's quadratic coefficient 1/(2 sigma^2)."""
    m = _model(D=64, p_out=0.1)
    cap = math.log(64) - math.log(0.1)
    for sigma in (0.5, 1.0, 2.0, 3.7):
        prev = -1.0
        for k in range(200):
            delta = k * 0.05
            c = orc.eq4(m, delta, sigma)
            assert c <= cap + 1e-12
            assert c >= prev - 1e-12
            assert c == orc.eq4(m, -delta, sigma)
            prev = c
        # second difference of the unclipped branch = 1/sigma^2 * h^2
        h = 0.01
        c0, c1, c2 = (orc.eq4(m, x, sigma) for x in (0.0, h, 2 * h))
        assert abs((c2 - 2 * c1 + c0) / h ** 2 - 1.0 / sigma ** 2) < 1e-5
        # constant term at delta = 0: ln A + ln(sigma sqrt(2 pi)) - ln(1 - p_out)
        assert abs(c0 - (math.log(sigma * math.sqrt(2 * math.pi)) - math.log(0.9))) < 1e-12


def test_pixel_costs_invalid_and_quantized():
    m = _model(q=11, D=128)
    cap = math.log(128) - math.log(0.15)
    capq = round(cap * 2048)
    assert orc.cost_sky(m, -1) == capq
    assert orc.cost_ground(m, -1, 3) == capq
    assert orc.cost_object(m, -1, 17) == capq
    # object pixel: disparity rounded half up to an integer (L#9): 2.5 -> 3
    assert orc.cost_object(m, 640, 3) == round(orc.eq4(m, 0.0, 1.0) * 2048)
    assert orc.cost_object(m, 639, 2) == round(orc.eq4(m, 0.0, 1.0) * 2048)
    # quantization is an integer number of 2^-q quanta
    for d in range(0, 128 * 256, 997):
        v = orc.cost_sky(m, d)
        assert v == int(v)
        assert abs(v / 2048 - orc.eq4(m, d / 256, 1.0)) <= 0.5 / 2048 + 1e-12


def test_ground_model_spec_example():
    """(Ground, alpha=0.5, v_horizon=100, v=80) -> 10.0.  Our rows count
    from the bottom (L#12) and the horizon is given as an image row, so
    v_horizon = (h-1) - horizon_row."""
    h = 200
    m = _model(h=h, alpha=0.5, horizon_row=(h - 1) - 100)
    assert orc.ground_R(m, 80) == 10 * 256
    assert orc.ground_R(m, 100) == 0
    assert orc.ground_R(m, 150) == 0          # clamped above the horizon (L#14)
    vals = [orc.ground_R(m, v) for v in range(h)]
    assert all(a >= b for a, b in zip(vals, vals[1:]))   # non-increasing


def test_alpha_from_camera():
    """L#21: alpha = B cos(theta)/H_cam with theta from the horizon offset; a
    level camera (horizon at the principal row) gives B/H_cam."""
    assert abs(orc.alpha(1000.0, 0.3, 1.2, 200.0, 200.0, 0.0) - 0.25) < 1e-12
    a = orc.alpha(1000.0, 0.3, 1.2, 150.0, 200.0, 0.0)
    assert abs(a - 0.25 * math.cos(math.atan(50 / 1000))) < 1e-12
    assert orc.alpha(1000.0, 0.3, 1.2, 150.0, 200.0, 0.7) == 0.7


def test_reduce_spec_examples():
    g = json.load(open(os.path.join(GOLD, "reduce_spec.json")))
    inv = 0xFFFF
    for case in g["cases"]:
        if "row" in case:
            row = np.array([inv if x is None else x * 16 for x in case["row"]], np.uint16)[None]
            out = orc.reduce(row, case["s"], 4, inv, 128)
            assert list(out[:, 0] / 256.0) == case["out"]
        else:
            img = np.array(case["rows"], np.uint16) * 16
            out = orc.reduce(img, case["s"], 4, inv, 128)
            assert out.shape == (case["n_cols"], case["h"])


def test_l27_only_the_object_model_clamps():
    """L#27: the reduction does not clamp (the pixel keeps d' in [D - 1/2, D) for
    the ground and sky terms of Eq. 4); the object model sees the pixel
    clamped below D - 1/2, so its pair-LUT index (L#9) is D - 1, the top of the
    D x D table of, and its span mean is taken over those values."""
    D = 64
    # reduction: the top of the range survives, 63.9375 px -> 63.9375 * 256
    assert orc.reduce(np.array([[63 * 16 + 15] * 5], np.uint16), 5, 4, 0xFFFF, D)[0, 0] == 63 * 256 + 240
    assert orc.reduce(np.array([[63 * 16 + 4] * 5], np.uint16), 5, 4, 0xFFFF, D)[0, 0] == 63 * 256 + 64
    # the 16-bit limit: only at D = 256 with 8 fractional bits (0xFFFF = invalid)
    assert orc.reduce(np.array([[65535] * 5], np.uint16), 5, 8, 0, 256)[0, 0] == 0xFFFE
    m = orc.Model(h=4, D=D, q=11, sigma=(1.0, 1.0, 100.0), alpha=0.0, horizon_row=0.0)
    top, edge = 63 * 256 + 240, 63 * 256 + 127             # 63.9375 px and D - 1/2 - 1/256
    # ground / sky: Eq. 4 of d' itself (sigma_S = 100 keeps it in the Gaussian branch)
    assert orc.cost_sky(m, top) > orc.cost_sky(m, edge)
    # object: pixel index D - 1 (the clamped value rounds to 63), not 64
    assert orc.cost_object(m, top, 63) == orc.cost_object(m, edge, 63) == orc.cost_object(m, 63 * 256, 63)
    # span mean over the clamped values: {63.9375, 61.1} -> {63.496, 61.1}: mean 62.30 -> 62,
    # where the unclamped mean 62.52 would round to 63
    col = np.array([top, 61 * 256 + 26, -1, -1], np.int32)
    assert orc.span_mean(m, col, 0, 1) == 62
    assert orc.span_mean(m, np.array([top, top, -1, -1], np.int32), 0, 1) == 63


def test_reduce_properties():
    rng = np.random.default_rng(3)
    inv = 0xFFFF
    img = rng.integers(0, 128 * 16, size=(9, 23)).astype(np.uint16)
    img[rng.random(img.shape) < 0.3] = inv
    # s = 1 is a pure transpose with row flip, values rescaled 1/16 -> 1/256
    out = orc.reduce(img, 1, 4, inv, 128)
    for c in range(23):
        for r in range(9):
            u = img[r, c]
            assert out[c, 8 - r] == (-1 if u == inv else int(u) * 16)
    # mean lies within [min, max] of the valid inputs and is exact half-up
    out = orc.reduce(img, 4, 4, inv, 128)
    for c in range(23 // 4):
        for r in range(9):
            vals = [int(x) for x in img[r, 4 * c:4 * c + 4] if x != inv]
            if not vals:
                assert out[c, 8 - r] == -1
                continue
            exact = Fraction(sum(vals) * 256, 16 * len(vals))
            assert out[c, 8 - r] == math.floor(exact + Fraction(1, 2))
            assert min(vals) * 16 <= out[c, 8 - r] <= max(vals) * 16
    # values decoding to >= D are invalid (L#23)
    img2 = np.array([[32 * 16, 40 * 16, 7 * 16]], np.uint16)
    out2 = orc.reduce(img2, 3, 4, inv, 32)
    assert out2[0, 0] == 7 * 256


def test_span_mean_exact_half_up():
    """f_n rounded half up in exact arithmetic (L#10) over the object
    disparities (each pixel clamped below D - 1/2, L#27, so f <= D - 1), no valid
    pixel -> 0 (L#11); checked against Python Fractions."""
    rng = np.random.default_rng(5)
    m = _model(h=40, D=16)
    for _ in range(300):
        col = rng.integers(0, 16 * 256, 40).astype(np.int32)
        col[rng.random(40) < 0.2] = -1
        # force exact .5 ties often
        col[rng.random(40) < 0.3] = rng.integers(0, 16) * 256 + 128
        vb = int(rng.integers(0, 40)); vt = int(rng.integers(vb, 40))
        vals = [min(int(x), 15 * 256 + 127) for x in col[vb:vt + 1] if x >= 0]
        if not vals:
            want = 0
        else:
            want = math.floor(Fraction(sum(vals), 256 * len(vals)) + Fraction(1, 2))
            assert want <= 15
        assert orc.span_mean(m, col, vb, vt) == want
    col = np.full(5, 15 * 256 + 200, np.int32)
    assert orc.span_mean(m, col, 0, 4) == 15                 # 15.78 -> object 15.496 -> 15


def test_stixel_data_is_sum_of_pixel_costs():
    rng = np.random.default_rng(7)
    m = _model(h=30, D=32, q=11, sigma=(2.0, 1.0, 0.5), alpha=0.5, horizon_row=10.0)
    col = rng.integers(0, 32 * 256, 30).astype(np.int32)
    col[rng.random(30) < 0.1] = -1
    for _ in range(50):
        vb = int(rng.integers(0, 30)); vt = int(rng.integers(vb, 30))
        f = int(rng.integers(0, 32))
        assert orc.stixel_data(m, col, orc.G, vb, vt, 0) == sum(
            orc.cost_ground(m, col[v], v) for v in range(vb, vt + 1))
        assert orc.stixel_data(m, col, orc.S, vb, vt, 0) == sum(
            orc.cost_sky(m, col[v]) for v in range(vb, vt + 1))
        assert orc.stixel_data(m, col, orc.O, vb, vt, f) == sum(
            orc.cost_object(m, col[v], f) for v in range(vb, vt + 1))
