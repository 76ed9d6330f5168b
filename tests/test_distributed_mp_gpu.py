"""The multi-GPU code path end to end, as separate processes: two ranks (both
on cuda:0, gloo staging device buffers through host memory — NCCL refuses
two ranks on one device) each own a Morton shard, set ONLY their owned rows
of x and v, and let the halo exchange deliver the ribbon rows before every
call, exactly as `bench.py --gpus N` drives them. Energies (all_reduce),
owned gradient / Hessian rows / HVP rows reassemble to the reference's golden
vectors (<= 1e-10, pattern bit-exact)."""

import multiprocessing as mp
import socket

import numpy as np
import pytest

from golden_util import FLOOR, build_terms, load, rel, rel_scalar

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q, overlap=False, backend="gloo", partition="morton"):
    import os
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_00406_b200.distributed import DistributedProblem

        d = load(name)
        n = int(d["n"])
        faces = d["faces"]
        edges = d["edges"] if not len(faces) else None
        dp = DistributedProblem(d["positions"], faces, n, build_terms(d), fixed_vertices=d["fixed"].tolist(),
                                edges=edges, with_hessian=bool(d["with_hessian"]) and not overlap, overlap=overlap,
                                partition=partition)
        own = dp.plan.owned_global
        x, v = d["s0_x"].reshape(-1, n), d["s0_v0"].reshape(-1, n)
        dp.set_x_owned(x[own])  # ribbon rows of x arrive through the halo exchange
        out = {"rank": rank, "owned": own, "energy": dp.eval_terms()}
        out["grad"] = dp.grad_owned().cpu().numpy()
        out["hvp"] = dp.hvp_owned(v[own]).cpu().numpy()
        if partition == "range":  # contiguous owned rows: the direction written in place, results as views
            assert dp.owned_view(dp.problem.x_device).data_ptr() != 0
            vb = dp.v_owned_buffer()
            vb.copy_(torch.as_tensor(v[own], device=vb.device))
            assert np.array_equal(dp.hvp_owned(vb).cpu().numpy(), out["hvp"])
        out["hvp_psd"] = dp.hvp_owned(v[own], psd_floor=FLOOR).cpu().numpy()
        if dp.problem.with_hessian:
            out["hrows"] = dp.hess_rows_owned()
            out["psd_energy"] = dp.eval_terms(psd_floor=FLOOR)
        q.put(out)
    finally:
        dist.destroy_process_group()


CASES = [(n, False) for n in ("cloth64", "dirichlet_ico2", "sphere_ico2", "smooth_ico2", "mixed_fv_ev_v")]
# overlap: interior rows assembled while the ribbon exchange is in flight (gradient-mode shards)
CASES += [(n, True) for n in ("cloth64", "sphere_ico2", "smooth_ico2", "mixed_fv_ev_v")]


# NCCL: one rank (NCCL refuses two ranks on one device), so the NCCL branches
# of the exchange (device buffers, async work handles on the communicator's
# stream) and the energy all_reduce run on this one-GPU box
NCCL_CASES = [("cloth64", False), ("cloth64", True), ("dirichlet_ico2", False), ("mixed_fv_ev_v", True)]


@pytest.mark.parametrize("name,overlap", CASES)
def test_two_process_shards_match_reference(name, overlap):
    _run(name, overlap, 2, "gloo")


# id-range partition (owned rows one contiguous slice of the shard numbering)
@pytest.mark.parametrize("name,overlap", [("cloth64", False), ("cloth64", True), ("smooth_ico2", True),
                                          ("dirichlet_ico2", False)])
def test_two_process_range_partition(name, overlap):
    _run(name, overlap, 2, "gloo", "range")


@pytest.mark.parametrize("name,overlap", NCCL_CASES)
def test_nccl_shard_matches_reference(name, overlap):
    _run(name, overlap, 1, "nccl")


def _run(name, overlap, world, backend, partition="morton"):
    d = load(name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, overlap, backend, partition)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = int(d["n"])
    nv = len(d["positions"])
    g = np.full((nv, n), np.nan)
    y = np.full((nv, n), np.nan)
    yp = np.full((nv, n), np.nan)
    for r in res:
        g[r["owned"]] = r["grad"]
        y[r["owned"]] = r["hvp"]
        yp[r["owned"]] = r["hvp_psd"]
        assert rel_scalar(r["energy"], d["s0_energy"]) <= 1e-10  # every rank holds the reduced energy
    assert rel(g.ravel(), d["s0_grad"]) <= 1e-10
    assert rel(y.ravel(), d["s0_hvp0"]) <= 1e-10
    assert rel(yp.ravel(), d["s0_hvp_psd0"]) <= 1e-10
    if "hrows" in res[0]:
        ro, ci, hv = d["row_offsets"], d["col_indices"], d["s0_hess"]
        for r in res:
            assert rel_scalar(r["psd_energy"], d["s0_psd_energy"]) <= 1e-10
            offs, cols, vals = r["hrows"]
            for i, vtx in enumerate(r["owned"]):
                lo, hi = ro[vtx], ro[vtx + 1]
                assert np.array_equal(cols[offs[i]:offs[i + 1]], ci[lo:hi])
                assert np.max(np.abs(vals[offs[i]:offs[i + 1]] - hv[lo:hi]), initial=0.0) <= 1e-10 * np.abs(hv).max()
