# full GPU suite + the grad / HVP row-kernel calls (compressed records)
mkdir -p gpurun_out
tag=${1:-r2c}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
for g in 2048 2240; do for c in hvp hvp_psd plain; do
  echo "grid $g $(timeout 300 python bench.py --only --grid $g --profile-call $c --steps 30 --no-cpu 2>/dev/null | tail -1)"
done; done > gpurun_out/only_${tag}.txt
timeout 900 python tools/bench_configs.py --sub 10 --configs smooth > gpurun_out/smooth_${tag}.jsonl 2>&1
timeout 900 python - > gpurun_out/c5_${tag}.json 2>&1 <<'PY'
import json, bench
r = bench.run_config5(6555.5, "measured")
print(json.dumps({k: {kk: v.get(kk) for kk in ("ms", "kernel_ms", "hbm_frac")} for k, v in r.items()}))
PY
tail -3 gpurun_out/pytest_${tag}.log; cat gpurun_out/only_${tag}.txt; grep '^{' gpurun_out/smooth_${tag}.jsonl | cut -c1-200; tail -2 gpurun_out/c5_${tag}.json
