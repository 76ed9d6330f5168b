# quick: traced paths (golden parity) + the traced bench leg
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_jit_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2b.log
timeout 600 python - > gpurun_out/traced_r2b.json 2> gpurun_out/traced_r2b.err <<'PY'
import json, bench
print(json.dumps(bench.run_traced(2048, 10, 6555.5, "measured")))
PY
timeout 300 python bench.py --only --profile-call psd --steps 30 --no-cpu > gpurun_out/only_r2b.txt 2>&1
tail -3 gpurun_out/pytest_r2b.log; cat gpurun_out/traced_r2b.json; tail -3 gpurun_out/traced_r2b.err; tail -2 gpurun_out/only_r2b.txt
