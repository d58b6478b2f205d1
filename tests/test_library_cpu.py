"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports
every symbol include/stixels.h declares, and validates parameters (the host
checks run before any device call, so they are testable without a GPU)."""
import ctypes

import numpy as np
import os
import re
import subprocess

import pytest

from paper_1610_04124_b200 import build as B
from paper_1610_04124_b200 import stixels as S
from tests import modelparams as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "stixels.h")).read()
    return sorted(set(re.findall(r"\b(stixels_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_abi():
    names = declared_symbols()
    for n in ("stixels_create", "stixels_compute", "stixels_destroy", "stixels_query"):
        assert n in names
    assert set(names) == set(S.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (stixels_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    lib = S.lib()
    for n in declared_symbols():
        assert hasattr(lib, n)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header():
    assert ctypes.sizeof(S.Params) == 4 * (6 + 1 + 3 + 1 + 3 + 9 + 4 + 2 + 2 + 4 + 2) + 4 + 2 * 8
    assert S.STIXEL_DTYPE.itemsize == 12


def _create(p, W=1024, H=440, B_=1):
    h = ctypes.c_void_p()
    return S.lib().stixels_create(ctypes.byref(p), W, H, B_, 0, None, ctypes.byref(h))


@pytest.mark.parametrize("field,value,code", [
    ("p_out", 0.0, S.ERR_PARAM), ("p_out", 1.0, S.ERR_PARAM), ("max_disparity", 1, S.ERR_PARAM),
    ("max_disparity", 300, S.ERR_UNSUPPORTED), ("stixel_width", 0, S.ERR_PARAM),
    ("a_norm", 0.0, S.ERR_PARAM), ("p_ord", 1.5, S.ERR_PARAM), ("ord_margin", -1, S.ERR_PARAM),
    ("disp_frac_bits", 9, S.ERR_PARAM), ("disp_format", 3, S.ERR_PARAM), ("reduce_mode", 2, S.ERR_UNSUPPORTED),
    ("cost_frac_bits", 30, S.ERR_PARAM), ("horizon_row", float("inf"), S.ERR_PARAM),
])
def test_param_validation(field, value, code):
    p = S.default_params()
    setattr(p, field, value)
    assert _create(p) == code
    assert S.lib().stixels_last_error(None)


def test_structural_zeros_enforced():
    p = S.default_params()
    p.p_first[2] = 0.5                      # sky cannot be the bottom stixel
    assert _create(p) == S.ERR_PARAM
    p = S.default_params()
    p.p_trans[2][0] = 0.5                   # ground above sky (P:66 staggering)
    assert _create(p) == S.ERR_PARAM
    p = S.default_params()
    assert _create(p, W=4) == S.ERR_ARG     # width < s
    assert _create(p, H=2000) == S.ERR_UNSUPPORTED
    assert _create(p, B_=0) == S.ERR_ARG


def test_median_width_limit():
    p = S.default_params()
    p.reduce_mode = S.REDUCE_MEDIAN
    p.stixel_width = 65
    assert _create(p, W=1040) == S.ERR_UNSUPPORTED


def test_sigma_tables_validated():
    """NEXT f2 tables: entries must be finite and > 0 (checked before any device
    work); a wide object band is accepted (dense ring), so with no device the
    create gets as far as the CUDA error."""
    from tests import modelparams as mp
    D, H = 64, 120
    bad = np.full(D, 1.0, np.float32)
    bad[5] = 0.0
    assert _create(S.params_from_dict(mp.make(max_disparity=D, sigma_object_f=bad), H), H=H) == S.ERR_PARAM
    wide = np.full(D, 4.0, np.float32)
    assert _create(S.params_from_dict(mp.make(max_disparity=D, sigma_object_f=wide), H), H=H) == S.ERR_CUDA
    g = np.full(H, 1.0, np.float32)
    g[-1] = np.nan
    assert _create(S.params_from_dict(mp.make(max_disparity=D, sigma_ground_v=g), H), H=H) == S.ERR_PARAM


def test_max_batch_limit():
    """The reduction grid carries frames in gridDim.z: max_batch <= 65535."""
    p = S.default_params()
    assert _create(p, B_=65536) == S.ERR_UNSUPPORTED


def test_exact_mode_range_guard():
    p = S.default_params()
    p.max_disparity = 256
    p.cost_frac_bits = 12                   # 1024 * 7.44 nats * 4096 > 2^24
    assert _create(p, W=2048, H=1024) == S.ERR_UNSUPPORTED


def test_no_device_means_cuda_error_not_fallback():
    """With valid parameters and no usable GPU, create fails with a CUDA error:
    there is no CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = S.params_from_dict(mp.make(), 440)
    assert _create(p) == S.ERR_CUDA


def test_default_params_match_design_reading():
    p = S.default_params()
    d = mp.make()
    for k in ("p_out", "p_ord", "p_grav", "p_blg", "p_exist", "a_norm"):
        assert abs(getattr(p, k) - d[k]) < 1e-6
    assert list(p.sigma) == list(d["sigma"])
    assert p.max_disparity == 128 and p.stixel_width == 5 and p.cost_frac_bits == 11
