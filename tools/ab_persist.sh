#!/bin/bash
# A/B of the persistent Hessian row kernel (MG_PERSISTENT=1) vs one block per CTA.
make -C paper_2509_00406_b200/csrc -j8 >/dev/null 2>&1
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_reference_problem_gpu.py -x -q > gpurun_out/pytest_persist.log 2>&1; tail -1 gpurun_out/pytest_persist.log
for t in 1 0 1 0; do
  for c in psd plain; do
    echo "persist=$t $c $(MG_PERSISTENT=$t timeout 300 python bench.py --only --profile-call $c --steps 30 2>/dev/null | tail -1)"
  done
done
