#!/bin/bash
# parity tests + bench (no CPU leg) + optional ncu of given calls: bash tools/quick_gpu.sh <tag> [calls...]
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 600 python bench.py --no-cpu ${BENCH_ARGS} > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
for c in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(k_rows_fast|k_patch)$' -s 0 -c 1 -o gpurun_out/prof_${c}_${tag} python bench.py --profile --profile-call $c ${BENCH_ARGS} > gpurun_out/ncu_${c}_${tag}.log 2>&1
done
tail -3 gpurun_out/pytest_gpu_${tag}.log; cat gpurun_out/bench_${tag}.json; tail -3 gpurun_out/bench_${tag}.err
