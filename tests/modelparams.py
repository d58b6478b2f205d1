"""One parameter description feeding both sides of a parity test.

The product's C ABI takes float32 parameters; the oracle takes doubles.  Both
are built from the same dict, the oracle receiving double(float32(x)) so the two
sides evaluate Eq. 4 and the priors on identical inputs.
"""
from __future__ import annotations

import copy

import numpy as np

G, O, S = 0, 1, 2


def f32(x):
    return float(np.float32(x))


def default_trans():
    t = np.ones((3, 3))
    t[G][G] = t[S][S] = t[S][G] = t[S][O] = 0.0
    return t


DEFAULTS = dict(
    focal_px=1000.0, baseline_m=0.3, camera_height_m=1.2, principal_row=0.0,
    ground_slope=0.4, horizon_frac=0.3,
    p_out=0.15, sigma=(2.0, 1.0, 0.5), a_norm=1.0,
    p_first=(1.0, float(np.exp(-2.0)), 0.0), p_trans=default_trans(),
    p_ord=0.2, p_grav=0.1, p_blg=0.04, p_exist=float(np.exp(-4.0)),
    ord_margin=1, grav_margin=1,
    stixel_width=5, max_disparity=128, disp_frac_bits=4, invalid_value=0xFFFF,
    cost_frac_bits=11, R_bits=8,
)


def make(**over):
    p = copy.deepcopy(DEFAULTS)
    p.update(over)
    return p


def horizon_row(p, H):
    return p.get("horizon_row", p["horizon_frac"] * H)


def oracle_model(p, H):
    """oracle.Model from a parameter dict for a frame of height H."""
    from oracle import oracle as orc
    hz = f32(horizon_row(p, H))
    alpha = orc.alpha(f32(p["focal_px"]), f32(p["baseline_m"]), f32(p["camera_height_m"]),
                      hz, f32(p["principal_row"]), f32(p["ground_slope"]))
    return orc.Model(
        h=H, D=p["max_disparity"], R_bits=p["R_bits"], q=p["cost_frac_bits"],
        p_out=f32(p["p_out"]), a_norm=f32(p["a_norm"]),
        sigma=tuple(f32(s) for s in p["sigma"]),
        p_first=tuple(f32(x) for x in p["p_first"]),
        p_trans=np.array([[f32(x) for x in row] for row in np.asarray(p["p_trans"])]),
        p_ord=f32(p["p_ord"]), p_grav=f32(p["p_grav"]), p_blg=f32(p["p_blg"]),
        p_exist=f32(p["p_exist"]), ord_margin=p["ord_margin"], grav_margin=p["grav_margin"],
        alpha=alpha, horizon_row=hz,
        sigma_o_f=None if p.get("sigma_object_f") is None
        else np.asarray(p["sigma_object_f"], np.float32).astype(np.float64),
        sigma_g_v=None if p.get("sigma_ground_v") is None
        else np.asarray(p["sigma_ground_v"], np.float32).astype(np.float64))
