set -x
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
python bench.py --no-cpu 2>&1 | tail -1
for c in psd plain; do
  ncu --set full --clock-control none --import-source on -k regex:'^k_patch' -s 1 -c 1 -o gpurun_out/prof_${c}_r1c python bench.py --profile --profile-call $c > /dev/null 2>&1
done
