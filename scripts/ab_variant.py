#!/usr/bin/env python3
"""Build an A/B variant library scripts/ab/libstixels_<name>.so from a modified
kernels.cuh (the product sources are untouched).
usage: ab_variant.py name path/to/kernels.cuh [path/to/api.cu]
Time it with python bench.py --lib scripts/ab/libstixels_<name>.so ..."""
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
api_src = sys.argv[3] if len(sys.argv) > 3 else os.path.join(B.CSRC, "api.cu")
api = open(api_src).read().replace(
    '#include "../../include/stixels.h"', f'#include "{os.path.dirname(B.HEADER)}/stixels.h"')
open(os.path.join(d, "api.cu"), "w").write(api)
# kernels.cuh includes ../../include/stixels.h as well
k = open(os.path.join(d, "kernels.cuh")).read().replace(
    '#include "../../include/stixels.h"', f'#include "{os.path.dirname(B.HEADER)}/stixels.h"')
open(os.path.join(d, "kernels.cuh"), "w").write(k)
print(B.build(variant=name, src=os.path.join(d, "api.cu")))
