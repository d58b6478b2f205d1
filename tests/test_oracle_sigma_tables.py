"""Pins of the oracle's NEXT f2 noise model sigma^c(f, v) (Eq. 4 with a
disparity-dependent object sigma and a row-dependent ground sigma; DESIGN.md
L#26): Eq. 4 closed forms per table entry, reduction to the constant model,
brute force on tiny columns, direct == prefix."""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from tests.test_oracle_dp import random_col, random_model


def _with_tables(m, rng):
    m.sigma_o_f = rng.uniform(0.6, 2.4, m.D)
    m.sigma_g_v = rng.uniform(0.8, 3.0, m.h)
    return m


def test_eq4_closed_form_per_entry():
    """cost at delta = 0 is ln(sigma sqrt(2 pi)) - ln(1 - p_out) (A_norm = 1),
    quantized: for every f and v the table's own sigma is used."""
    rng = np.random.default_rng(1)
    m = orc.Model(h=12, D=20, q=11)
    m.sigma_o_f = rng.uniform(0.5, 3.0, m.D)
    m.sigma_g_v = rng.uniform(0.5, 3.0, m.h)
    for f in range(m.D):
        want = round(2 ** 11 * (math.log(m.sigma_o_f[f] * math.sqrt(2 * math.pi)) - math.log(0.85)))
        assert orc.cost_object(m, 256 * f, f) == want
        # one disparity off: + 1 / (2 sigma_f^2), unless capped (pixels stay below D, L#23)
        x = math.log(m.sigma_o_f[f] * math.sqrt(2 * math.pi)) - math.log(0.85) + 1 / (2 * m.sigma_o_f[f] ** 2)
        cap = math.log(m.D) - math.log(0.15)
        g = f + 1 if f + 1 < m.D else f - 1
        assert orc.cost_object(m, 256 * g, f) == round(2 ** 11 * min(x, cap))
    for v in range(m.h):
        dg = orc.ground_R(m, v)
        want = round(2 ** 11 * (math.log(m.sigma_g_v[v] * math.sqrt(2 * math.pi)) - math.log(0.85)))
        assert orc.cost_ground(m, int(dg), v) == want


def test_constant_tables_reduce_to_the_constant_model():
    rng = np.random.default_rng(2)
    for _ in range(20):
        h, D = int(rng.integers(1, 30)), int(rng.integers(4, 33))
        m = random_model(rng, h, D)
        col = random_col(rng, h, D)
        a = orc.solve_column(m, col, mode=1)
        m.sigma_o_f = np.full(D, m.sigma[1])
        m.sigma_g_v = np.full(h, m.sigma[0])
        assert orc.solve_column(m, col, mode=1) == a


@pytest.mark.parametrize("h", [2, 4, 6])
def test_bruteforce_with_sigma_tables(h):
    rng = np.random.default_rng(30 + h)
    for _ in range(25):
        D = int(rng.integers(4, 17))
        m = _with_tables(random_model(rng, h, D, ordering=False), rng)
        col = random_col(rng, h, D)
        st, cost = orc.solve_column(m, col, mode=1)
        _, bcost, _ = orc.bruteforce(m, col)
        assert cost == bcost
        assert orc.rescore(m, col, st) == cost


def test_direct_equals_prefix_with_sigma_tables():
    rng = np.random.default_rng(40)
    for _ in range(15):
        h, D = int(rng.integers(1, 40)), int(rng.integers(4, 40))
        m = _with_tables(random_model(rng, h, D), rng)
        col = random_col(rng, h, D, invalid=0.2)
        assert orc.solve_column(m, col, mode=0) == orc.solve_column(m, col, mode=1)
