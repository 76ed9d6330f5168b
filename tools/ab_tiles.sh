#!/bin/bash
# A/B of the staged edge tile kernel (gradient / HVP) against the per-row kernel.
# usage (under gpurun): bash tools/ab_tiles.sh <tag>
tag=${1:-ab}
mkdir -p gpurun_out
make -C paper_2509_00406_b200/csrc -j8 >/dev/null
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${tag}.log 2>&1; tail -3 gpurun_out/pytest_${tag}.log
for t in 1 0; do
  MG_EDGE_TILES=$t timeout 600 python bench.py > gpurun_out/bench_${tag}_t$t.json 2> gpurun_out/bench_${tag}_t$t.err
  MG_EDGE_TILES=$t timeout 600 python tools/bench_configs.py --configs smooth > gpurun_out/smooth_${tag}_t$t.jsonl 2>&1
done
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
for t in ("1", "0"):
    try:
        d = json.loads(open(f"gpurun_out/bench_{tag}_t{t}.json").read().strip().splitlines()[-1])
        print("tiles", t, "value", d["value"], {k: (round(v["ms"], 4), round(v["hbm_frac"], 3)) for k, v in d["extras"].items()})
    except Exception as e:
        print("tiles", t, "bench failed", e)
    for line in open(f"gpurun_out/smooth_{tag}_t{t}.jsonl"):
        if line.startswith("{"):
            d = json.loads(line)
            print("  smooth", d["call"], round(d["ms"], 4), round(d["hbm_frac"], 3))
PY
