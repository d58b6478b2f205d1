#!/bin/bash
# GPU-box profile set of a round (after the same commands ran clean without ncu):
# launch list of the bench step (cold-cache, serialised -- compare shares), one
# --set full capture of dp_kernel and one of the K1 reduction.
# usage: bash scripts/gpu_profiles.sh tag [k1]   (k1: only the K1 capture; the reports of one call
# must stay under gpurun's 64 MiB)
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import oracle.oracle as o; o.build()" > /dev/null 2>&1
[ -z "$2" ] && timeout -k 10 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --batch 512 --steps 2 --warmup 1 --no-e2e --no-cpu --no-single --no-cont > gpurun_out/ncu_launch_$TAG.log 2>&1
[ -z "$2" ] && timeout -k 10 400 ncu --set full --clock-control none --import-source on -k regex:dp_kernel -s 1 -c 1 -o gpurun_out/dp_full_$TAG \
  python bench.py --batch 256 --steps 1 --warmup 1 --no-e2e --no-cpu --no-single --no-cont > gpurun_out/ncu_dp_$TAG.log 2>&1
[ -n "$2" ] && timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:reduce -s 1 -c 1 -o gpurun_out/k1_full_$TAG \
  python bench.py --batch 512 --steps 1 --warmup 1 --no-e2e --no-cpu --no-single --no-cont > gpurun_out/ncu_k1_$TAG.log 2>&1
ls gpurun_out/*_$TAG*
