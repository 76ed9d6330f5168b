#!/bin/bash
# Round-2 profile pass: ncu --set full of every timed kernel (one launch each,
# summarised on the box by tools/ncu_summary.py) + the launch list of the
# headline bench step. usage (under gpurun): bash tools/prof_r02.sh <tag>
tag=${1:-r02b}
mkdir -p gpurun_out
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
cap() {  # name regex skip command...
  local name=$1 re=$2 skip=$3; shift 3
  timeout 600 ncu -f --set full --clock-control none --import-source on --metrics $M -k "regex:$re" -s $skip -c 1 \
      -o /tmp/prof_$name "$@" > /tmp/ncu_$name.log 2>&1
  { echo "== $name ($*)"; python tools/ncu_summary.py /tmp/prof_$name.ncu-rep 14; } > gpurun_out/ncu_${tag}_$name.txt 2>&1
}
B="python bench.py --profile --no-cpu"
cap cloth_psd '^k_rows_fast$' 0 $B --profile-call psd
cap cloth_plain '^k_rows_fast$' 0 $B --profile-call plain
cap cloth_hvp '^k_rows_fast$' 0 $B --profile-call hvp --grid 2240
cap cloth_hvp_psd '^k_rows_fast$' 0 $B --profile-call hvp_psd --grid 2240
P="python tools/prof_configs.py --sub 10 --configs"
cap dir_hess '^k_rows_dirichlet$' 1 $P dirichlet
cap dir_hess_psd '^k_cta_dirichlet$' 0 $P dirichlet
cap dir_hvp '^k_cta_dirichlet$' 1 $P dirichlet
cap dir_hvp_psd '^k_cta_dirichlet$' 2 $P dirichlet
cap sph_grad '^k_rows_sphere$' 1 $P sphere
cap sph_hvp '^k_rows_sphere$' 2 $P sphere
cap sph_hvp_psd '^k_sphere_face_hvp_psd$' 0 $P sphere
cap smooth_grad '^k_rows_fast$' 1 $P smooth
cap smooth_hvp '^k_rows_fast$' 2 $P smooth
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --profile --no-cpu > /dev/null 2>&1
ls gpurun_out/ncu_${tag}_*.txt | wc -l
grep -h "^== \|Duration\|DRAM Throughput\|fp64 executed" gpurun_out/ncu_${tag}_*.txt
