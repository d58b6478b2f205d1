"""Python (ctypes) front end of the CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Wraps ``oracle/stixels_oracle.c`` (plain double-precision C, see its header for
the paper citations).  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  It imports nothing from the product package and the product package
imports nothing from here.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stixels_oracle.c")
_LIB = os.path.join(_HERE, "libstixels_oracle.so")

G, O, S, START = 0, 1, 2, 3
CLASS_NAMES = {G: "ground", O: "object", S: "sky"}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no GPU code).  FP contraction is off so the
    expressions evaluate exactly as written."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
           "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB


class _Model(ctypes.Structure):
    _fields_ = [
        ("h", ctypes.c_int), ("D", ctypes.c_int), ("R_bits", ctypes.c_int), ("q", ctypes.c_int),
        ("p_out", ctypes.c_double), ("a_norm", ctypes.c_double),
        ("sigma", ctypes.c_double * 3), ("p_first", ctypes.c_double * 3),
        ("p_trans", (ctypes.c_double * 3) * 3),
        ("p_ord", ctypes.c_double), ("p_grav", ctypes.c_double), ("p_blg", ctypes.c_double),
        ("p_exist", ctypes.c_double),
        ("ord_margin", ctypes.c_int), ("grav_margin", ctypes.c_int),
        ("alpha", ctypes.c_double), ("horizon_row", ctypes.c_double),
        ("sigma_o_f", ctypes.c_void_p), ("sigma_g_v", ctypes.c_void_p),
    ]


class _Stixel(ctypes.Structure):
    _fields_ = [("vb", ctypes.c_int), ("vt", ctypes.c_int), ("cls", ctypes.c_int),
                ("disp", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        P = ctypes.POINTER
        L.orc_eq4.restype = ctypes.c_double
        L.orc_eq4.argtypes = [P(_Model), ctypes.c_double, ctypes.c_double]
        L.orc_alpha.restype = ctypes.c_double
        L.orc_alpha.argtypes = [ctypes.c_double] * 6
        L.orc_ground_R.restype = ctypes.c_longlong
        L.orc_ground_R.argtypes = [P(_Model), ctypes.c_int]
        L.orc_reduce.restype = None
        L.orc_reduce.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_uint,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_reduce_median.restype = None
        L.orc_reduce_median.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_uint,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        for name in ("orc_cost_sky",):
            getattr(L, name).restype = ctypes.c_double
            getattr(L, name).argtypes = [P(_Model), ctypes.c_int]
        L.orc_cost_ground.restype = ctypes.c_double
        L.orc_cost_ground.argtypes = [P(_Model), ctypes.c_int, ctypes.c_int]
        L.orc_cost_object.restype = ctypes.c_double
        L.orc_cost_object.argtypes = [P(_Model), ctypes.c_int, ctypes.c_int]
        L.orc_round_disp.restype = ctypes.c_int
        L.orc_round_disp.argtypes = [P(_Model), ctypes.c_int]
        L.orc_span_mean.restype = ctypes.c_int
        L.orc_span_mean.argtypes = [P(_Model), ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.orc_stixel_data.restype = ctypes.c_double
        L.orc_stixel_data.argtypes = [P(_Model), ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int]
        L.orc_prior_first.restype = ctypes.c_double
        L.orc_prior_first.argtypes = [P(_Model), ctypes.c_int]
        L.orc_prior_trans.restype = ctypes.c_double
        L.orc_prior_trans.argtypes = [P(_Model)] + [ctypes.c_int] * 5
        L.orc_rescore.restype = ctypes.c_double
        L.orc_rescore.argtypes = [P(_Model), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.orc_solve_column.restype = ctypes.c_int
        L.orc_solve_column.argtypes = [P(_Model), ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                       P(ctypes.c_double), ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]
        L.orc_bruteforce_column.restype = ctypes.c_longlong
        L.orc_bruteforce_column.argtypes = [P(_Model), ctypes.c_void_p, ctypes.c_void_p,
                                            P(ctypes.c_int), P(ctypes.c_double)]
        L.orc_solve_frame.restype = None
        L.orc_solve_frame.argtypes = [P(_Model), ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p]
        L.orc_max_threads.restype = ctypes.c_int
    return _lib


def _default_trans():
    # [lower][upper]; forbidden: G above G, S above S, G above S, O above S (L#16)
    t = np.ones((3, 3))
    t[G][G] = 0.0
    t[S][S] = 0.0
    t[S][G] = 0.0
    t[S][O] = 0.0
    return t


@dataclass
class Model:
    """The stixel model in the paper's terms (defaults: DESIGN.md reading L#1)."""
    h: int
    D: int
    R_bits: int = 8
    q: int = 11
    p_out: float = 0.15
    a_norm: float = 1.0
    sigma: tuple = (2.0, 1.0, 0.5)
    p_first: tuple = (1.0, float(np.exp(-2.0)), 0.0)
    p_trans: np.ndarray = field(default_factory=_default_trans)
    p_ord: float = 0.2
    p_grav: float = 0.1
    p_blg: float = 0.04
    p_exist: float = float(np.exp(-4.0))
    ord_margin: int = 1
    grav_margin: int = 1
    alpha: float = 0.4
    horizon_row: float = 0.0
    sigma_o_f: np.ndarray | None = None   # NEXT f2: sigma_O(f), D entries (None: constant)
    sigma_g_v: np.ndarray | None = None   # NEXT f2: sigma_G(v), h entries (None: constant)

    def c(self) -> _Model:
        m = _Model()
        m.h, m.D, m.R_bits, m.q = self.h, self.D, self.R_bits, self.q
        m.p_out, m.a_norm = self.p_out, self.a_norm
        for i in range(3):
            m.sigma[i] = self.sigma[i]
            m.p_first[i] = self.p_first[i]
            for j in range(3):
                m.p_trans[i][j] = float(np.asarray(self.p_trans)[i][j])
        m.p_ord, m.p_grav, m.p_blg, m.p_exist = self.p_ord, self.p_grav, self.p_blg, self.p_exist
        m.ord_margin, m.grav_margin = self.ord_margin, self.grav_margin
        m.alpha, m.horizon_row = self.alpha, self.horizon_row
        # the double arrays must outlive the struct: keep them on the model
        self._so = None if self.sigma_o_f is None else np.ascontiguousarray(self.sigma_o_f, np.float64)
        self._sg = None if self.sigma_g_v is None else np.ascontiguousarray(self.sigma_g_v, np.float64)
        assert self._so is None or len(self._so) == self.D
        assert self._sg is None or len(self._sg) == self.h
        m.sigma_o_f = None if self._so is None else self._so.ctypes.data
        m.sigma_g_v = None if self._sg is None else self._sg.ctypes.data
        return m


def eq4(model: Model, delta: float, sigma: float) -> float:
    return lib().orc_eq4(ctypes.byref(model.c()), delta, sigma)


def alpha(focal_px, baseline_m, camera_height_m, horizon_row, principal_row, ground_slope):
    return lib().orc_alpha(focal_px, baseline_m, camera_height_m, horizon_row, principal_row,
                           ground_slope)


def ground_R(model: Model, v: int) -> int:
    return lib().orc_ground_R(ctypes.byref(model.c()), v)


def reduce(img: np.ndarray, s: int, q_bits: int, invalid: int, D: int, R_bits: int = 8,
           mode: int = 0):
    """img: [H][W] uint8/uint16 -> [n_cols][H] int32 reduced columns (model order).
    mode 0: mean of the valid pixels; 1: their median (NEXT f4, L#24)."""
    img = np.ascontiguousarray(img)
    H, W = img.shape
    n_cols = W // s
    out = np.zeros((n_cols, H), dtype=np.int32)
    fn = lib().orc_reduce if mode == 0 else lib().orc_reduce_median
    fn(img.ctypes.data, img.itemsize, W, H, W, s, q_bits, invalid, D, R_bits, out.ctypes.data)
    return out


def cost_ground(model, dR, v):
    return lib().orc_cost_ground(ctypes.byref(model.c()), int(dR), int(v))


def cost_sky(model, dR):
    return lib().orc_cost_sky(ctypes.byref(model.c()), int(dR))


def cost_object(model, dR, f):
    return lib().orc_cost_object(ctypes.byref(model.c()), int(dR), int(f))


def span_mean(model, col, vb, vt):
    col = np.ascontiguousarray(col, dtype=np.int32)
    return lib().orc_span_mean(ctypes.byref(model.c()), col.ctypes.data, vb, vt)


def stixel_data(model, col, cls, vb, vt, f):
    col = np.ascontiguousarray(col, dtype=np.int32)
    return lib().orc_stixel_data(ctypes.byref(model.c()), col.ctypes.data, cls, vb, vt, f)


def prior_first(model, cls):
    return lib().orc_prior_first(ctypes.byref(model.c()), cls)


def prior_trans(model, prev_cls, prev_f, cls, vb, f):
    return lib().orc_prior_trans(ctypes.byref(model.c()), prev_cls, prev_f, cls, vb, f)


def _to_list(arr, n):
    return [(arr[i].vb, arr[i].vt, arr[i].cls, arr[i].disp) for i in range(n)]


def rescore(model: Model, col, stixels) -> float:
    col = np.ascontiguousarray(col, dtype=np.int32)
    n = len(stixels)
    arr = (_Stixel * max(n, 1))()
    for i, (vb, vt, c, d) in enumerate(stixels):
        arr[i].vb, arr[i].vt, arr[i].cls, arr[i].disp = vb, vt, c, d
    return lib().orc_rescore(ctypes.byref(model.c()), col.ctypes.data, ctypes.byref(arr), n)


def solve_column(model: Model, col, mode: int = 1, tables: bool = False):
    """Eq. 5-6 DP + backtracking.  Returns (stixels, cost[, tables])."""
    col = np.ascontiguousarray(col, dtype=np.int32)
    h = model.h
    assert col.shape == (h,)
    arr = (_Stixel * h)()
    cost = ctypes.c_double()
    C = np.zeros((3, h)); aj = np.zeros((3, h), np.int32)
    ac = np.zeros((3, h), np.int32); F = np.zeros((3, h), np.int32)
    n = lib().orc_solve_column(ctypes.byref(model.c()), col.ctypes.data, mode, ctypes.byref(arr),
                               ctypes.byref(cost), C.ctypes.data, aj.ctypes.data, ac.ctypes.data,
                               F.ctypes.data)
    st = _to_list(arr, n)
    if tables:
        return st, cost.value, dict(C=C, argj=aj, argc=ac, F=F)
    return st, cost.value


def bruteforce(model: Model, col):
    col = np.ascontiguousarray(col, dtype=np.int32)
    arr = (_Stixel * 12)()
    n = ctypes.c_int()
    cost = ctypes.c_double()
    count = lib().orc_bruteforce_column(ctypes.byref(model.c()), col.ctypes.data,
                                        ctypes.byref(arr), ctypes.byref(n), ctypes.byref(cost))
    if count < 0:
        raise ValueError("brute force limited to 1 <= h <= 12")
    return _to_list(arr, n.value), cost.value, count


def solve_frame(model: Model, cols: np.ndarray, mode: int = 1, threads: int = 0):
    """cols: [n_cols][h] int32.  Returns (stixels[n_cols] lists, costs[n_cols])."""
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    n_cols, h = cols.shape
    assert h == model.h
    arr = (_Stixel * (n_cols * h))()
    count = np.zeros(n_cols, np.int32)
    cost = np.zeros(n_cols)
    lib().orc_solve_frame(ctypes.byref(model.c()), cols.ctypes.data, n_cols, mode, threads,
                          ctypes.byref(arr), count.ctypes.data, cost.ctypes.data)
    out = []
    for c in range(n_cols):
        base = c * h
        out.append([(arr[base + i].vb, arr[base + i].vt, arr[base + i].cls, arr[base + i].disp)
                    for i in range(count[c])])
    return out, cost


def max_threads() -> int:
    return lib().orc_max_threads()
