#!/bin/bash
# ncu --set full of the CTA face kernel (HESS and HVP) at icosphere(sub)
sub=${1:-9}; tag=${2:-cta}
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum
cap() {  # name regex skip configs
  ncu --set full --clock-control none --import-source on --metrics $M -k "regex:$2" -s $3 -c 1 \
      -o /tmp/prof_$1 python tools/prof_configs.py --sub $sub --configs $4 > /tmp/ncu_$1.log 2>&1
  { echo "== $1 (icosphere($sub))"; python tools/ncu_summary.py /tmp/prof_$1.ncu-rep 18; } > gpurun_out/ncu_${tag}_$1.txt 2>&1
}
cap cta_hess k_cta_dirichlet 1 dirichlet
cap cta_hvp k_cta_dirichlet 3 dirichlet
cat gpurun_out/ncu_${tag}_*.txt
