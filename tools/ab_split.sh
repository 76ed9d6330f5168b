#!/bin/bash
# A/B of the split (two threads per row) Hessian kernel vs one thread per row.
# usage (under gpurun): bash tools/ab_split.sh <tag> [extra make flags]
tag=${1:-abs}
mkdir -p gpurun_out
make -C paper_2509_00406_b200/csrc -j8 >/dev/null 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_reference_problem_gpu.py -x -q > gpurun_out/pytest_${tag}.log 2>&1; tail -2 gpurun_out/pytest_${tag}.log
for t in 1 0; do
  for c in psd plain; do
    echo "split=$t $c $(MG_ROW_SPLIT=$t timeout 300 python bench.py --only --profile-call $c --steps 20 2>/dev/null | tail -1)"
  done
done
