# A/B of the flat row kernels (config-5 gradient / HVPs and the 2240^2 HVPs) against
# every ab_libs/lib_*.so and the default library. usage (under gpurun): bash tools/ab_flat.sh
for lib in "" ab_libs/lib_*.so; do
  for n in 7072; do MG_LIB=$lib timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import bench, json, os
out = bench.run_config5(6555.5, 'measured', $n)
print(os.environ.get('MG_LIB') or 'base', {k: round(v['kernel_ms'],4) for k,v in out.items()})
" 2>&1 | tail -1; done
done
bash tools/ab_run.sh 2240 hvp hvp_psd 2>&1 | tail -10
