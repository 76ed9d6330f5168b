# A/B of an environment switch on the grad / HVP calls: bash tools/ab_env.sh VAR "val1 val2"
var=$1; vals=$2
mkdir -p gpurun_out
for rep in 1 2; do
for v in $vals; do
  for g in 2048 2240; do for c in hvp hvp_psd; do
    echo "$var=$v grid $g $(env $var=$v timeout 300 python bench.py --only --grid $g --profile-call $c --steps 30 --no-cpu 2>/dev/null | tail -1)"
  done; done
  echo "$var=$v smooth $(env $var=$v timeout 600 python tools/bench_configs.py --sub 10 --configs smooth 2>/dev/null | grep '^{' | python -c "
import json,sys
print(' '.join(f\"{d['call']} {d['kernel_ms']:.4f} {d['hbm_frac']:.3f}\" for d in map(json.loads, sys.stdin)))")"
done
done
