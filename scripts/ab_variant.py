#!/usr/bin/env python3
"""Build an A/B variant library libstixels_<name>.so from a modified kernels.cuh
(the product sources are untouched).  usage: ab_variant.py name path/to/kernels.cuh
Time it with STIXELS_LIB_VARIANT=name python bench.py ..."""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1610_04124_b200 import build as B   # noqa: E402

name, kern = sys.argv[1], sys.argv[2]
d = os.path.join("/tmp", f"stx_var_{name}")
os.makedirs(d, exist_ok=True)
shutil.copy(kern, os.path.join(d, "kernels.cuh"))
api = open(os.path.join(B.CSRC, "api.cu")).read().replace(
    '#include "../../include/stixels.h"', f'#include "{os.path.dirname(B.HEADER)}/stixels.h"')
open(os.path.join(d, "api.cu"), "w").write(api)
# kernels.cuh includes ../../include/stixels.h as well
k = open(os.path.join(d, "kernels.cuh")).read().replace(
    '#include "../../include/stixels.h"', f'#include "{os.path.dirname(B.HEADER)}/stixels.h"')
open(os.path.join(d, "kernels.cuh"), "w").write(k)
print(B.build(variant=name, src=os.path.join(d, "api.cu")))
