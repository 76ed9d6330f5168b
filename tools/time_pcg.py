"""Device PCG (mg_pcg) against the host-synchronised CG on the bench's cloth
Hessian (bench.run_pcg: 40 fixed iterations). usage: python tools/time_pcg.py [grid]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
p, x, v = bench.build_engine_cloth(n, "deterministic")
V = p.mesh.num_vertices
print(json.dumps(bench.run_pcg(p, p.hess.nnz_blocks, V)))
