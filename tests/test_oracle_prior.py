"""Pins of the oracle's prior model (orc_prior_first / orc_prior_trans and the
hoisted copies inside orc_solve_column) against hand-computed quanta of the
reading (tests/golden/prior_reading.json: P:66; DESIGN.md
L#1, L#15, L#16, L#22).  CPU only.

A misreading mirrored on both sides of the parity test (swapping gravity and
diving, flipping the ordering direction, dropping the BIC term, transposing
p_trans) would pass GPU parity; these values catch it on the oracle side, and
GPU parity then carries it to the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as orc

G, O, S = orc.G, orc.O, orc.S
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "prior_reading.json")))


def golden_model(q=None):
    g = GOLD["model"]
    return orc.Model(
        h=g["h"], D=g["D"], R_bits=g["R_bits"], q=g["q"] if q is None else q,
        p_first=tuple(g["p_first"]), p_trans=np.array(g["p_trans"], dtype=np.float64),
        p_ord=g["p_ord"], p_grav=g["p_grav"], p_blg=g["p_blg"], p_exist=g["p_exist"],
        ord_margin=g["ord_margin"], grav_margin=g["grav_margin"],
        alpha=g["alpha"], horizon_row=g["horizon_row"])


def _val(x):
    return math.inf if x == "inf" else x


def test_ground_model_of_the_golden_column():
    """The golden branches assume dg(v) = 0.5 (19 - v) px (L#12, L#14)."""
    m = golden_model()
    assert orc.ground_R(m, 5) == 7 * 256
    assert orc.ground_R(m, 4) == int(7.5 * 256)
    assert orc.ground_R(m, 19) == 0
    assert orc.ground_R(m, 20) == 0          # above the horizon: clamped at 0


@pytest.mark.parametrize("case", GOLD["first"], ids=lambda c: c["branch"])
def test_prior_first(case):
    m = golden_model()
    assert orc.prior_first(m, case["cls"]) == _val(case["expect"])


@pytest.mark.parametrize("case", GOLD["trans"], ids=lambda c: c["branch"])
def test_prior_trans(case):
    m = golden_model()
    got = orc.prior_trans(m, case["prev_cls"], case["prev_f"], case["cls"], case["vb"], case["f"])
    assert got == _val(case["expect"]), case["branch"]


def test_prior_continuous_mode():
    c = GOLD["continuous"]
    m = golden_model(q=0)
    for e in c["first"]:
        assert abs(orc.prior_first(m, e["cls"]) - e["expect"]) <= c["abs_tol"]
    for e in c["trans"]:
        got = orc.prior_trans(m, e["prev_cls"], e["prev_f"], e["cls"], e["vb"], e["f"])
        assert abs(got - e["expect"]) <= c["abs_tol"], e["branch"]


def test_dp_tables_use_the_golden_priors():
    """The hoisted prior constants inside orc_solve_column (prefix mode) and the
    per-candidate orc_prior_trans calls (direct mode) are the same reading: a
    two-stixel segmentation re-scored minus its data terms equals the golden
    first + transition quanta, and direct (orc_prior_trans per candidate) ==
    prefix (hoisted constants) on the same column."""
    m = golden_model()
    h = m.h
    quanta = {k: v["value"] for k, v in GOLD["quanta"].items() if "value" in v}
    # rows 0..5 at disparity 7 px (= dg(5) .. on the ground), rows 6..19 at 9 px
    col = np.array([7 * 256] * 6 + [9 * 256] * (h - 6), np.int32)
    for (c0, c1, j, want_prior) in [
        # dg(6) = 6.5 px: f = 9 > 6.5 + 1 -> floating (L#15)
        (G, O, 6, quanta["first_G"] + quanta["trans_GO"] + quanta["floating"]),
        (O, O, 6, quanta["first_O"] + quanta["trans_OO"] + quanta["ord_violated"]),  # 9 > 7 + 1
        (O, G, 6, quanta["first_O"] + quanta["trans_OG"]),
        (G, S, 6, quanta["first_G"] + quanta["trans_GS"]),
    ]:
        seg = [(0, j - 1, c0, 0.0), (j, h - 1, c1, 0.0)]
        data = (orc.stixel_data(m, col, c0, 0, j - 1, orc.span_mean(m, col, 0, j - 1))
                + orc.stixel_data(m, col, c1, j, h - 1, orc.span_mean(m, col, j, h - 1)))
        prior = orc.rescore(m, col, seg) - data
        assert prior == want_prior, (c0, c1)
    # DP == direct == prefix on this column, and the DP value re-scores
    s0, c0_ = orc.solve_column(m, col, mode=0)
    s1, c1_ = orc.solve_column(m, col, mode=1)
    assert s0 == s1 and c0_ == c1_ and orc.rescore(m, col, s1) == c1_


def test_sky_first_and_forbidden_pairs_never_appear():
    """Forbidden entries are +inf (P:66 staggering; L#16): on random columns no
    optimal list starts with sky or contains a forbidden pair, even with every
    allowed probability small."""
    rng = np.random.default_rng(5)
    m = golden_model()
    allowed = {(G, O), (G, S), (O, G), (O, O), (O, S)}
    for _ in range(40):
        col = rng.integers(0, m.D * 256, m.h).astype(np.int32)
        col[rng.random(m.h) < 0.2] = -1
        st, cost = orc.solve_column(m, col)
        assert math.isfinite(cost) and st[0][2] != S
        assert all((a[2], b[2]) in allowed for a, b in zip(st, st[1:]))
