# usage: bash tools/gpu_profile.sh <tag> <calls...>   (ncu --set full of the patch kernel per call)
tag=$1; shift
for c in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:'^k_patch(_ev)?$' -s 1 -c 1 -o gpurun_out/prof_${c}_${tag} python bench.py --profile --profile-call $c --patch ${PATCH:-128} > gpurun_out/ncu_${c}_${tag}.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv python bench.py --profile > /dev/null 2>&1
