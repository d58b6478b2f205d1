#!/bin/bash
# A/B of the product library and named variants (scripts/ab/libstixels_<name>.so) on
# a few f1 shapes: prints "<lib> W H s D fps parity" per config.
# usage: bash scripts/ab_sweep.sh name1 [name2 ...]
cd ${GRAFT_REPO_ROOT:-.}
python -c "import oracle.oracle as o; o.build()" > /dev/null 2>&1
for v in base "$@"; do
  if [ "$v" = base ]; then LIBARG=""; else LIBARG="--lib scripts/ab/libstixels_$v.so"; fi
  timeout 600 python bench.py --sweep --steps 3 $LIBARG 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    if d.get('sweep') and (d['s'] == 5): print('$v', d['W'], d['H'], d['s'], d['D'], round(d['fps']), d.get('parity'))
"
done
