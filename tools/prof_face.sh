#!/bin/bash
# ncu --set full captures of the face kernels at icosphere(sub), one report per
# launch, each summarised on the box (tools/ncu_summary.py) into gpurun_out/.
# usage (under gpurun): bash tools/prof_face.sh <sub> <tag>
sub=${1:-10}; tag=${2:-r02}
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
cap() {  # name regex skip configs
  ncu --set full --clock-control none --import-source on --metrics $M -k "regex:$2" -s $3 -c 1 \
      -o /tmp/prof_$1 python tools/prof_configs.py --sub $sub --configs $4 > /tmp/ncu_$1.log 2>&1
  { echo "== $1 (icosphere($sub))"; python tools/ncu_summary.py /tmp/prof_$1.ncu-rep 14; } > gpurun_out/ncu_${tag}_$1.txt 2>&1
}
cap dir_hess k_rows_dirichlet 1 dirichlet
cap dir_hess_psd k_rows_dirichlet 2 dirichlet
cap dir_hvp k_rows_dirichlet 3 dirichlet
cap face_psd k_face_psd 0 dirichlet
cap sph_grad k_rows_sphere 1 sphere
cap sph_hvp k_rows_sphere 2 sphere
cap sph_hvp_psd k_sphere_face_hvp_psd 0 sphere
cap smooth_hvp k_rows_fast 2 smooth
cat gpurun_out/ncu_${tag}_*.txt
