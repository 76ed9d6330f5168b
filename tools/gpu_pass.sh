# One GPU-box pass: GPU test suite, smoke(), default bench line. usage (under gpurun): bash tools/gpu_pass.sh <tag>
tag=${1:-pass}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi_${tag}.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${tag}.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
tail -3 gpurun_out/pytest_gpu_${tag}.log; tail -2 gpurun_out/smoke_${tag}.log; cut -c1-3000 gpurun_out/bench_${tag}.json; tail -5 gpurun_out/bench_${tag}.err
