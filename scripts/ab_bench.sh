#!/bin/bash
# A/B timing on the GPU box: the product library and each named variant
# (scripts/ab/libstixels_<name>.so built by scripts/ab_variant.py), alternated twice.
# usage: bash scripts/ab_bench.sh name1 [name2 ...]
cd ${GRAFT_REPO_ROOT:-.}
python -c "import oracle.oracle as o; o.build()" > /dev/null 2>&1
for rep in 1 2; do
  for v in base "$@"; do
    if [ "$v" = base ]; then LIBARG=""; else LIBARG="--lib scripts/ab/libstixels_$v.so"; fi
    timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-cont --no-single $LIBARG > /tmp/ab_$v.json 2>/tmp/ab_$v.err || tail -3 /tmp/ab_$v.err
    python -c "import json; d=json.load(open('/tmp/ab_$v.json')); print('$v', round(d['value']), round(d['stage_ms']['dp'], 2), d['parity'])"
  done
done
