#!/bin/bash
# GPU-box run: build, gpu tests, bench, ncu launch list + one --set full capture of the DP kernel.
# usage: bash scripts/gpu_round.sh [tag] [skip_tests]
# Every step is bounded (a kernel hang must not eat the budget); stops at the first failure.
cd ${GRAFT_REPO_ROOT:-.}
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
if [ -z "$2" ]; then
  timeout -k 10 240 python -m pytest tests -m gpu -x -q --timeout=90 2>&1 | tail -25
  [ ${PIPESTATUS[0]} -eq 0 ] || { echo "GPU TESTS FAILED/HUNG"; exit 1; }
fi
timeout -k 10 240 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err || { tail -5 gpurun_out/bench_$TAG.err; exit 1; }
cat gpurun_out/bench_$TAG.json
timeout -k 10 240 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --batch 512 --steps 2 --warmup 1 --no-e2e --no-cpu --no-single --no-cont > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:dp_kernel -s 1 -c 1 -o gpurun_out/dp_full_$TAG python bench.py --batch 256 --steps 1 --warmup 1 --no-e2e --no-cpu --no-single --no-cont > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
