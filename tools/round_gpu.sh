#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench line, configs, launch list, ncu --set full captures.
# usage (from repo root, under gpurun): bash tools/round_gpu.sh <tag>
tag=${1:-r}
mkdir -p gpurun_out
make -C paper_2509_00406_b200/csrc -j8 > /dev/null 2>&1
nvidia-smi > gpurun_out/smi_${tag}.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_${tag}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 900 python tools/bench_configs.py --sub 10 > gpurun_out/configs_${tag}.jsonl 2> gpurun_out/configs_${tag}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv python bench.py --profile > gpurun_out/launches_${tag}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(k_rows_fast|k_patch)$' -s 0 -c 1 -o gpurun_out/prof_${tag} python bench.py --profile > gpurun_out/ncu_${tag}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_tile_ev$' -s 0 -c 1 -o gpurun_out/prof_hvp_${tag} python bench.py --profile --profile-call hvp > gpurun_out/ncu_hvp_${tag}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^(k_rows_dirichlet|k_face_psd)$' -c 3 -o gpurun_out/prof_dir_${tag} python tools/bench_configs.py --configs dirichlet --sub 8 --steps 1 > gpurun_out/ncu_dir_${tag}.log 2>&1
tail -3 gpurun_out/pytest_gpu_${tag}.log; tail -2 gpurun_out/smoke_${tag}.log; cat gpurun_out/bench_${tag}.json | cut -c1-600
