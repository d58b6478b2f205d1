"""A second, plain-Python statement of the Eq. 5-6 recurrence for
the parity pins -- TEST INFRASTRUCTURE ONLY.

It shares nothing with oracle/stixels_oracle.c: Eq. 4, the ground
model, the integer span mean (L#10), the priors (P:66, P:120,
L#1/L#15/L#16) and the recurrence are written out again here, directly from
the paper and the readings, with exact rational arithmetic where the paper's
quantity is a ratio.  It keeps, per (row k, class c), only the minimum cost and
the object value f of the last stixel of its argmin segmentation -- "the stixel
at the end of the segmentation associated with each minimum cost" --
and evaluates the prior of Eq. 6 against that stixel.  Candidate
order and ties follow L#17.  Exact mode (q > 0) only: every term is an integer
number of 2^-q quanta, so the comparison with the oracle is exact.
"""
from __future__ import annotations

import math
from fractions import Fraction

G, O, S, START = 0, 1, 2, 3
INF = math.inf


def solve(m, col):
    """m: oracle.Model-like (attributes h, D, q, p_out, a_norm, sigma, p_first,
    p_trans, p_ord, p_grav, p_blg, p_exist, ord_margin, grav_margin, alpha,
    horizon_row); col: h reduced disparities in 1/256 px (-1 invalid).
    Returns (cost in quanta, [(vb, vt, cls, f)] bottom to top)."""
    h, D, sc = m.h, m.D, 2 ** m.q

    def quant(x):
        return x if x == INF else float(round(x * sc))

    def nlp(p):
        return INF if p <= 0 else -math.log(p)

    cap = math.log(D / m.p_out)

    def pixel(d_px, f, sigma):         # Eq. 4 of one pixel, quantised
        if d_px is None:
            return quant(cap)
        gauss = math.log(m.a_norm * sigma * math.sqrt(2 * math.pi) / (1 - m.p_out))
        return quant(min(cap, gauss + (d_px - f) ** 2 / (2 * sigma * sigma)))

    def ground(v):                       # dg(v) in 1/256 px, clamped at 0, half up
        x = m.alpha * ((h - 1 - m.horizon_row) - v)
        return 0 if x <= 0 else math.floor(x * 256 + 0.5)

    val = [None if d < 0 else d for d in col]
    # the object model sees pixels clamped below D - 1/2 (L#27)
    obj = [None if d is None else min(d, (D - 1) * 256 + 127) for d in val]

    def mean(j, k):
        vs = [d for d in obj[j:k + 1] if d is not None]
        if not vs:
            return 0
        return min(D - 1, math.floor(Fraction(sum(vs), 256 * len(vs)) + Fraction(1, 2)))

    def data(c, j, k, f):
        tot = 0.0
        for v in range(j, k + 1):
            d = val[v]
            if c == G:
                tot += pixel(None if d is None else Fraction(d - ground(v), 256), 0, m.sigma[G])
            elif c == S:
                tot += pixel(None if d is None else Fraction(d, 256), 0, m.sigma[S])
            else:
                tot += pixel(None if d is None else (obj[v] + 128) // 256, f, m.sigma[O])
        return tot

    bic = nlp(m.p_exist)

    def first(c):
        return quant(nlp(m.p_first[c]) + bic)

    def trans(cp, fp, c, vb, f):
        t = quant(nlp(m.p_trans[cp][c]) + bic)
        if t == INF:
            return t
        if c == O and cp == O:             # ordering: upper object nearer -> violated
            t += quant(nlp(m.p_ord)) if f > fp + m.ord_margin else quant(nlp(1 - m.p_ord))
        if c == O and cp == G:             # gravity (nearer than ground) / diving (farther)
            g = ground(vb)
            if 256 * f > g + 256 * m.grav_margin:
                t += quant(nlp(m.p_grav))
            elif 256 * f < g - 256 * m.grav_margin:
                t += quant(nlp(m.p_blg))
            else:
                t += quant(nlp(1 - m.p_grav - m.p_blg))
        return t

    best = [[None] * 3 for _ in range(h)]    # (cost, j, c', f)
    for k in range(h):
        for c in range(3):
            f0 = mean(0, k) if c == O else 0
            cand = (data(c, 0, k, f0) + first(c), 0, START, f0)
            for j in range(1, k + 1):
                f = mean(j, k) if c == O else 0
                dt = data(c, j, k, f)
                for cp in range(3):
                    pc, _, _, pf = best[j - 1][cp]
                    x = dt + trans(cp, pf, c, j, f) + pc
                    if x < cand[0]:
                        cand = (x, j, cp, f)
            best[k][c] = cand
    c = min(range(3), key=lambda i: (best[h - 1][i][0], i))
    cost, out, k = best[h - 1][c][0], [], h - 1
    while True:
        _, j, cp, f = best[k][c]
        out.append((j, k, c, f))
        if j == 0:
            break
        k, c = j - 1, cp
    return cost, out[::-1]
