"""Device time of the assembled-Hessian BSR matvec (Newton-CG inner product) on
the bench cloth (2048^2): ms and HBM fraction of its algorithmic bytes
(72 nnzb values + 4 nnzb columns + 8 (V+1) row starts + 24 V in + 24 V out)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402


def main():
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import ClothConfig, cloth_problem, default_pins, lumped_masses

    n = 2048
    pos, faces = mg.grid_arrays(n, 1.0 / (n - 1))
    mesh = mg.Mesh(pos, faces)
    rng = np.random.default_rng(0)
    target = pos + 0.01 / (n - 1) * rng.normal(size=pos.shape)
    cfg = ClothConfig(grid_n=n, spacing=1.0 / (n - 1))
    p = cloth_problem(cfg, mesh, target, masses=lumped_masses(mesh, 1.0), pinned=default_pins(n))
    p.x = (pos + 0.01 / (n - 1) * rng.normal(size=pos.shape)).ravel()
    p.eval_terms(psd_floor=1e-9)
    v = torch.from_numpy(rng.normal(size=3 * n * n)).cuda()
    for _ in range(3):
        p.hess.matvec(v)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        p.hess.matvec(v)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    V, nnzb = n * n, p.hess.nnz_blocks
    nbytes = 72 * nnzb + 4 * nnzb + 8 * (V + 1) + 48 * V
    peak, _ = bench.peaks()
    print(json.dumps({"matvec_ms": ms, "bytes": nbytes, "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / peak}))


if __name__ == "__main__":
    main()
