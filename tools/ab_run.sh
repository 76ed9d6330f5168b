#!/bin/bash
# Time bench.py --only calls against every ab_libs/lib_*.so (and the default
# library). usage (under gpurun): bash tools/ab_run.sh <grid> <call> [<call> ...]
g=$1; shift
for i in 1 2; do
  for lib in "" ab_libs/lib_*.so; do
    for call in "$@"; do
      echo "${lib:-base} $call $(MG_LIB=$lib timeout 300 python bench.py --only --grid $g --profile-call $call --steps 30 2>/dev/null | tail -1)"
    done
  done
done
