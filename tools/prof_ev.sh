#!/bin/bash
# ncu --set full of the patch assembly kernel for each bench call: bash tools/prof_ev.sh <tag> psd plain hvp ...
tag=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(k_rows_fast|k_patch|k_tile_ev)$' -s 0 -c 1 -o gpurun_out/prof_${c}_${tag} python bench.py --profile --profile-call $c ${BENCH_ARGS} > gpurun_out/ncu_${c}_${tag}.log 2>&1
done
