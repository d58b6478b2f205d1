#!/bin/bash
# GPU-box run: build, gpu tests, bench, ncu launch list + one --set full capture of the DP kernel.
# usage: bash scripts/gpu_round.sh [tag] [skip_tests]
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
if [ -z "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
fi
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --batch 512 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_kernel -s 1 -c 1 -o gpurun_out/dp_full_$TAG python bench.py --batch 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
