"""Thin ctypes binding of include/stixels.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of `libstixels.so`; this
module only converts Python/torch arguments into the C ABI's plain pointers and
sizes.  PyTorch is used for device memory and streams.  There is no CPU
fallback: if the library is missing or cannot be loaded this raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIB

GROUND, OBJECT, SKY = 0, 1, 2
U8, U16, F32 = 0, 1, 2
REDUCE_MEAN, REDUCE_MEDIAN = 0, 1

OK, ERR_ARG, ERR_PARAM, ERR_UNSUPPORTED, ERR_CUDA, ERR_CAPACITY = 0, -1, -2, -3, -4, -5


class StixelsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"stixels error {status}: {msg}")
        self.status = status


class Params(ctypes.Structure):
    """Mirror of `stixels_params` (include/stixels.h)."""
    _fields_ = [
        ("focal_px", ctypes.c_float), ("baseline_m", ctypes.c_float),
        ("camera_height_m", ctypes.c_float), ("horizon_row", ctypes.c_float),
        ("principal_row", ctypes.c_float), ("ground_slope", ctypes.c_float),
        ("p_out", ctypes.c_float), ("sigma", ctypes.c_float * 3), ("a_norm", ctypes.c_float),
        ("p_first", ctypes.c_float * 3), ("p_trans", (ctypes.c_float * 3) * 3),
        ("p_ord", ctypes.c_float), ("p_grav", ctypes.c_float), ("p_blg", ctypes.c_float),
        ("p_exist", ctypes.c_float),
        ("ord_margin", ctypes.c_int32), ("grav_margin", ctypes.c_int32),
        ("stixel_width", ctypes.c_int32), ("max_disparity", ctypes.c_int32),
        ("disp_format", ctypes.c_int32), ("disp_frac_bits", ctypes.c_int32),
        ("invalid_value", ctypes.c_uint32), ("reduce_mode", ctypes.c_int32),
        ("cost_frac_bits", ctypes.c_int32), ("max_stixels", ctypes.c_int32),
        ("sigma_object_f", ctypes.POINTER(ctypes.c_float)),    # NEXT f2 (NULL = constant)
        ("sigma_ground_v", ctypes.POINTER(ctypes.c_float)),
    ]


STIXEL_DTYPE = np.dtype([("bottom", "<u2"), ("top", "<u2"), ("cls", "u1"), ("pad", "u1", 3),
                         ("disparity", "<f4")])
assert STIXEL_DTYPE.itemsize == 12

_lib = None


_lib_path = LIB


def use_library(path: str) -> None:
    """Explicitly bind another build of the same ABI (A/B timing: bench.py --lib,
    scripts/ab_variant.py).  Must precede the first call into the library; the
    product path never calls it."""
    global _lib_path
    if _lib is not None and os.path.abspath(path) != os.path.abspath(_lib_path):
        raise RuntimeError("library already loaded from " + _lib_path)
    _lib_path = path


def lib() -> ctypes.CDLL:
    """Load libstixels.so (built in-tree by paper_1610_04124_b200.build).  Raises if absent."""
    global _lib
    if _lib is None:
        path = _lib_path
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built; run paper_1610_04124_b200.build.build() "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(path)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        P = ctypes.POINTER
        L.stixels_default_params.argtypes = [P(Params)]
        L.stixels_create.argtypes = [P(Params), i32, i32, i32, i32, vp, P(vp)]
        L.stixels_query.argtypes = [vp, P(i32), P(i32)]
        L.stixels_query_kernel.argtypes = [vp, P(i32), P(i32), P(i32)]
        L.stixels_compute.argtypes = [vp, vp, i64, i32, vp, vp, vp]
        L.stixels_compute_host.argtypes = [vp, vp, i64, i32, vp, vp, vp]
        L.stixels_reduce.argtypes = [vp, vp, i64, i32, vp]
        L.stixels_solve.argtypes = [vp, vp, i32, vp, vp, vp]
        L.stixels_sync.argtypes = [vp]
        L.stixels_last_launch_count.argtypes = [vp]
        L.stixels_query_launch.argtypes = [vp, P(i32), P(i32)]
        L.stixels_set_launch_plan.argtypes = [vp, i32]
        if hasattr(L, "stixels_skipped_cells"):   # (absent from A/B builds that predate it)
            L.stixels_skipped_cells.argtypes = [vp, P(ctypes.c_ulonglong)]
            L.stixels_set_chunk_bound.argtypes = [vp, i32]
        L.stixels_destroy.argtypes = [vp]
        L.stixels_error_string.argtypes = [i32]
        L.stixels_error_string.restype = ctypes.c_char_p
        L.stixels_last_error.argtypes = [vp]
        L.stixels_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


# stixels_query_kernel variants
DP_DENSE, DP_SPARSE, DP_PAIR2D, DP_INT32, DP_PAIR2D_DENSE = 0, 1, 2, 3, 4


EXPORTS = ("stixels_default_params", "stixels_create", "stixels_query", "stixels_query_kernel",
           "stixels_compute",
           "stixels_compute_host", "stixels_reduce", "stixels_solve", "stixels_sync",
           "stixels_last_launch_count", "stixels_query_launch", "stixels_set_launch_plan",
           "stixels_skipped_cells", "stixels_set_chunk_bound", "stixels_destroy", "stixels_error_string",
           "stixels_last_error")


def default_params() -> Params:
    p = Params()
    lib().stixels_default_params(ctypes.byref(p))
    return p


def params_from_dict(d: dict, H: int) -> Params:
    """Build Params from the shared test/bench parameter dict (tests/modelparams.py)."""
    p = default_params()
    for key in ("focal_px", "baseline_m", "camera_height_m", "principal_row", "ground_slope",
                "p_out", "a_norm", "p_ord", "p_grav", "p_blg", "p_exist"):
        setattr(p, key, float(d[key]))
    p.horizon_row = float(d.get("horizon_row", d["horizon_frac"] * H))
    for i in range(3):
        p.sigma[i] = float(d["sigma"][i])
        p.p_first[i] = float(d["p_first"][i])
        for j in range(3):
            p.p_trans[i][j] = float(np.asarray(d["p_trans"])[i][j])
    p.ord_margin, p.grav_margin = int(d["ord_margin"]), int(d["grav_margin"])
    p.stixel_width, p.max_disparity = int(d["stixel_width"]), int(d["max_disparity"])
    p.disp_format = int(d.get("disp_format", U16))
    p.disp_frac_bits = int(d["disp_frac_bits"])
    p.invalid_value = int(d["invalid_value"])
    p.cost_frac_bits = int(d["cost_frac_bits"])
    p.max_stixels = int(d.get("max_stixels", 0))
    p.reduce_mode = int(d.get("reduce_mode", REDUCE_MEAN))
    # NEXT f2 noise-model tables: the float32 arrays are kept alive on the struct
    # (stixels_create copies them)
    for key, n in (("sigma_object_f", p.max_disparity), ("sigma_ground_v", H)):
        if d.get(key) is not None:
            arr = np.ascontiguousarray(np.asarray(d[key], dtype=np.float32))
            assert arr.shape == (n,), (key, arr.shape, n)
            setattr(p, "_keep_" + key, arr)
            setattr(p, key, arr.ctypes.data_as(ctypes.POINTER(ctypes.c_float)))
    return p


def _check(st, handle=None):
    if st != OK:
        msg = lib().stixels_last_error(handle)
        raise StixelsError(st, (msg or b"").decode() or lib().stixels_error_string(st).decode())


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


class Handle:
    """Owns a `stixels_handle*` bound to one device and one CUDA stream."""

    def __init__(self, params: Params, width: int, height: int, max_batch: int,
                 device: int = 0, stream=None):
        import torch
        self.width, self.height, self.max_batch, self.device = width, height, max_batch, device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        h = ctypes.c_void_p()
        st = lib().stixels_create(ctypes.byref(params), width, height, max_batch, device,
                                  ctypes.c_void_p(stream.cuda_stream), ctypes.byref(h))
        _check(st, None)
        self._h = h
        n, c = ctypes.c_int(), ctypes.c_int()
        _check(lib().stixels_query(h, ctypes.byref(n), ctypes.byref(c)), h)
        self.n_cols, self.cap = n.value, c.value
        v, ds, cpc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().stixels_query_kernel(h, ctypes.byref(v), ctypes.byref(ds), ctypes.byref(cpc)), h)
        # DP kernel variant (DP_DENSE / DP_SPARSE / DP_PAIR2D / DP_INT32), W-row slots,
        # column groups per CTA
        self.dp_variant, self.dp_slots, self.cols_per_cta = v.value, ds.value, cpc.value
        self.bpp = {U8: 1, U16: 2, F32: 4}[params.disp_format]

    # -- allocation helpers (torch device memory) --------------------------
    def alloc_outputs(self, batch: int):
        import torch
        dev = torch.device("cuda", self.device)
        out = torch.empty((batch, self.n_cols, self.cap, 12), dtype=torch.uint8, device=dev)
        count = torch.empty((batch, self.n_cols), dtype=torch.int32, device=dev)
        cost = torch.empty((batch, self.n_cols), dtype=torch.float32, device=dev)
        return out, count, cost

    # -- C ABI calls ---------------------------------------------------------
    def compute(self, disp, out, count, cost=None, row_pitch_bytes=None):
        """disp: device tensor [batch][H][W] (u8/u16 as int16/uint8 storage)."""
        batch = disp.shape[0]
        pitch = row_pitch_bytes or disp.stride(1) * disp.element_size()
        _check(lib().stixels_compute(self._h, _ptr(disp), pitch, batch, _ptr(out), _ptr(count),
                                     _ptr(cost)), self._h)

    def compute_host(self, disp: np.ndarray, out: np.ndarray, count: np.ndarray,
                     cost: np.ndarray | None = None):
        """Host buffers (numpy; pinned memory recommended). Synchronous."""
        batch = disp.shape[0]
        pitch = disp.strides[1]
        cp = ctypes.c_void_p(cost.ctypes.data) if cost is not None else ctypes.c_void_p(0)
        _check(lib().stixels_compute_host(self._h, ctypes.c_void_p(disp.ctypes.data), pitch,
                                          batch, ctypes.c_void_p(out.ctypes.data),
                                          ctypes.c_void_p(count.ctypes.data), cp), self._h)

    def compute_host_ptr(self, disp_ptr, pitch, batch, out_ptr, count_ptr, cost_ptr=0):
        _check(lib().stixels_compute_host(self._h, ctypes.c_void_p(disp_ptr), pitch, batch,
                                          ctypes.c_void_p(out_ptr), ctypes.c_void_p(count_ptr),
                                          ctypes.c_void_p(cost_ptr)), self._h)

    def reduce(self, disp, cols, row_pitch_bytes=None):
        batch = disp.shape[0]
        pitch = row_pitch_bytes or disp.stride(1) * disp.element_size()
        _check(lib().stixels_reduce(self._h, _ptr(disp), pitch, batch, _ptr(cols)), self._h)

    def solve(self, cols, out, count, cost=None):
        batch = cols.shape[0]
        _check(lib().stixels_solve(self._h, _ptr(cols), batch, _ptr(out), _ptr(count),
                                   _ptr(cost)), self._h)

    def sync(self):
        _check(lib().stixels_sync(self._h), self._h)

    def last_launch_count(self) -> int:
        return lib().stixels_last_launch_count(self._h)

    def set_launch_plan(self, warps_per_column: int) -> None:
        """0 = automatic, 4 or 8 warps per column (stixels_set_launch_plan)."""
        _check(lib().stixels_set_launch_plan(self._h, warps_per_column), self._h)

    def skipped_cells(self) -> int:
        """Cumulative DP cells skipped by the exact chunk bound (stixels_skipped_cells)."""
        n = ctypes.c_ulonglong()
        _check(lib().stixels_skipped_cells(self._h, ctypes.byref(n)), self._h)
        return n.value

    def set_chunk_bound(self, mode: int) -> None:
        """0 = automatic, 1 = off, 2 = on (stixels_set_chunk_bound)."""
        _check(lib().stixels_set_chunk_bound(self._h, mode), self._h)

    def last_launch_shape(self) -> tuple[int, int]:
        """(warps per column, column groups per CTA) of the last DP launch."""
        cw, cpc = ctypes.c_int(), ctypes.c_int()
        _check(lib().stixels_query_launch(self._h, ctypes.byref(cw), ctypes.byref(cpc)), self._h)
        return cw.value, cpc.value

    def destroy(self):
        if getattr(self, "_h", None):
            lib().stixels_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def decode(out_bytes: np.ndarray, count: np.ndarray):
    """[batch][n_cols][cap][12] uint8 + counts -> list (per frame) of lists (per
    column) of (bottom, top, cls, disparity)."""
    arr = np.ascontiguousarray(out_bytes).view(STIXEL_DTYPE).reshape(out_bytes.shape[:3])
    res = []
    for b in range(arr.shape[0]):
        frame = []
        for c in range(arr.shape[1]):
            n = int(count[b, c])
            s = arr[b, c, :min(n, arr.shape[2])]
            frame.append([(int(x["bottom"]), int(x["top"]), int(x["cls"]), float(x["disparity"]))
                          for x in s])
        res.append(frame)
    return res
