#!/usr/bin/env python
"""Benchmark: mass-spring cloth Newton-step assembly on a 2048x2048 grid.

Headline workload (BASELINE.json configs[1]): `Problem.eval_terms(psd_floor=1e-9)`
— energy, gradient and block-CSR Hessian with per-element PSD clamp, exactly
what `newton_solve` calls each Newton iteration — on the ClothSim energy
(inertia + spring + gravity, default pins) over generate_grid(2048, 1/2047),
fp64. A step = one such evaluation. Unit = term-element evaluations / s
(2V + E per call).

  value   : device time per step (CUDA events on the launching stream, inputs
            resident in HBM; the 2.6 GB of inputs+outputs exceed the 126 MB L2,
            so no flush is needed)
  e2e     : the public API with host buffers: pinned x H2D, eval, energy +
            gradient D2H, every step
  roofline: HBM; algorithmic bytes of one call (inputs read once + outputs
            written once) / the assembly kernel's own device time
            (library-side CUDA events around that launch, same timed region);
            traffic = DRAM bytes of the same kernel from the committed ncu capture
  cpu_baseline: the CPU oracle port (oracle/, restating meshgrad) on a bounded
            256^2 sample of the same call, all host threads

Multi-GPU (torchrun, N ranks): weak scaling. The global cloth is a
2048 x (2048 N) grid partitioned by vertex ownership (distributed.py); each
rank assembles its owned rows after a halo exchange of ribbon x, and the energy
is all-reduced. Time = max over ranks.

`--impl reference` runs the reference arm: the CPU oracle port on the same
metric (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOOR = 1e-9
GRID = 2048
METRIC = "term-element evaluations/s, cloth Newton-step grad+Hessian assembly (psd_floor=1e-9)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--grid", type=int, default=GRID)
    ap.add_argument("--accumulation", default="deterministic", choices=["deterministic", "atomic"])
    ap.add_argument("--patch", type=int, default=64, help="owned rows per vertex patch (generic patch path)")
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary workloads")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE configs 2'/3/4 extras")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--profile", action="store_true", help="few steps, headline only (for ncu)")
    ap.add_argument("--profile-call", default="psd", choices=["psd", "plain", "hvp", "hvp_psd", "energy"],
                    help="which call --profile / --only runs")
    ap.add_argument("--only", action="store_true", help="time --profile-call alone (K steps) and print its ms")
    return ap.parse_args()


# ----------------------------------------------------------------- workloads

def grid_rect_arrays(nx, ny, spacing):
    """generate_grid's numbering and split on an nx x ny vertex rectangle."""
    ii, jj = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    pos = np.stack([ii.ravel() * spacing, jj.ravel() * spacing, np.zeros(nx * ny)], axis=1)
    j, i = np.meshgrid(np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    v00 = (j * nx + i).ravel()
    f = np.empty((2 * (nx - 1) * (ny - 1), 3), np.int64)
    f[0::2] = np.stack([v00, v00 + 1, v00 + nx + 1], 1)
    f[1::2] = np.stack([v00, v00 + nx + 1, v00 + nx], 1)
    return pos, f


def cloth_state(pos, n, seed=0):
    rng = np.random.default_rng(seed)
    sig = 0.01 / (n - 1)
    target = pos + sig * rng.normal(size=pos.shape)
    x = (pos + sig * rng.normal(size=pos.shape)).ravel()
    v = np.random.default_rng(1).normal(size=x.size)
    return target, x, v


def cloth_inputs(n, seed=0):
    from paper_2509_00406_b200.mesh import grid_arrays

    pos, faces = grid_arrays(n, 1.0 / (n - 1))
    target, x, v = cloth_state(pos, n, seed)
    return pos, faces, target, x, v


def cloth_sizes(n, ny=None):
    ny = n if ny is None else ny
    V = n * ny
    E = (n - 1) * ny + n * (ny - 1) + (n - 1) * (ny - 1)
    return V, E


# algorithmic bytes per call: inputs read once, outputs written once, int32 indices
def cloth_bytes(V, E, nnzb):
    # x, target, masses, rest lengths, edge endpoints; grad, Hessian blocks
    return 24 * V + 24 * V + 8 * V + 8 * E + 8 * E + 24 * V + 72 * nnzb


def cloth_hvp_bytes(V, E):
    # x, v, masses, rest lengths, edge endpoints; y
    return 24 * V + 24 * V + 8 * V + 8 * E + 8 * E + 24 * V


def cloth_energy_bytes(V, E):
    return 24 * V + 24 * V + 8 * V + 8 * E + 8 * E


def build_engine_cloth(n, accumulation, patch=64):
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import ClothConfig, cloth_problem, default_pins, lumped_masses

    pos, faces, target, x, v = cloth_inputs(n)
    mesh = mg.Mesh(pos, faces, patch_vertices=patch)
    cfg = ClothConfig(grid_n=n, spacing=1.0 / (n - 1))
    target_d = torch.from_numpy(target).cuda()
    masses_d = torch.from_numpy(lumped_masses(mesh, cfg.mass_density)).cuda()
    p = cloth_problem(cfg, mesh, target_d, masses=masses_d, pinned=default_pins(n), accumulation=accumulation)
    p.precompute_sparsity()
    p.x = x
    return p, x, v


def build_engine_cloth_shard(n, world, rank, accumulation):
    """Rank `rank`'s shard of the weak-scaling cloth: a 2048 x (2048 world) grid."""
    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.distributed import DistributedProblem
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    ny = n * world
    sp = 1.0 / (n - 1)
    pos, faces = grid_rect_arrays(n, ny, sp)
    target, x, v = cloth_state(pos, n)
    areas = 0.5 * np.linalg.norm(np.cross(pos[faces[:, 1]] - pos[faces[:, 0]], pos[faces[:, 2]] - pos[faces[:, 0]]), axis=1)
    masses = np.bincount(faces.ravel(), weights=np.repeat(areas / 3.0, 3), minlength=len(pos))
    edges = mg.mesh._host_edges(faces, None, len(pos))
    d = pos[edges[:, 1]] - pos[edges[:, 0]]
    h = 0.01
    terms = [("V", Inertia(masses, target)), ("EV", Spring(np.einsum("ij,ij->i", d, d), 0.5 * 1e4 * h * h)),
             ("V", Gravity(masses, np.array([0.0, -9.8, 0.0]), h * h))]
    pins = (n * (ny - 1), n * ny - 1)
    dp = DistributedProblem(pos, faces, 3, terms, fixed_vertices=pins, accumulation=accumulation)
    dp.set_x_global(x)
    dp.problem.precompute_sparsity()
    return dp, len(pos), len(edges)


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        return d.get(kernel)
    except Exception:
        return None


def time_device(fn, steps, warmup, dist=None):
    """Mean ms per step with CUDA events on the current stream; max over ranks."""
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(st)
    for i in range(steps):
        fn()
        ev[i + 1].record(st)
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    total = ev[0].elapsed_time(ev[-1])
    if dist is not None:
        t = torch.tensor([total], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
        dist.barrier()
    return total / steps, per


def time_with_kernel(p, fn, steps, warmup, dist=None):
    """(ms per step, ms per main-kernel launch) over the same timed region."""
    import gc

    gc.collect()  # no deferred destruction (cudaFree) of earlier problems inside the timed region
    p.set_kernel_timing(False)
    for _ in range(warmup):
        fn()
    p.set_kernel_timing(True)
    p.kernel_time()  # reset
    ms, _ = time_device(fn, steps, 0, dist)
    kt, cnt = p.kernel_time()
    p.set_kernel_timing(False)
    return ms, (kt / cnt if cnt else None)


def kernel_label(p, call):
    mode = {"psd": "HESS,psd", "plain": "HESS", "hvp": "HVP", "hvp_psd": "HVP,psd", "energy": "ENERGY"}[call]
    return f"k_rows_fast<{p.n},{mode},SPRING>"


# -------------------------------------------------------------- CPU baseline

def cpu_oracle_rate(n_sample, reps=1, psd=True):
    """Oracle port (oracle/) on a cloth n_sample^2 grid, all host threads."""
    from oracle import OracleProblem
    from oracle.engine import default_workers
    from paper_2509_00406_b200.apps import default_pins, lumped_masses
    from paper_2509_00406_b200.mesh import Mesh, _host_edges
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    pos, faces, target, x, _ = cloth_inputs(n_sample)
    nv = len(pos)
    edges = _host_edges(faces, None, nv)
    mesh = Mesh(pos, faces)
    mesh._edges = edges
    masses = lumped_masses(mesh, 1.0)
    d = pos[edges[:, 1]] - pos[edges[:, 0]]
    l2 = np.einsum("ij,ij->i", d, d)
    h = 0.01
    terms = [("V", Inertia(masses, target)), ("EV", Spring(l2, 0.5 * 1e4 * h * h)),
             ("V", Gravity(masses, np.array([0.0, -9.8, 0.0]), h * h))]
    workers = default_workers()
    op = OracleProblem(nv, faces, edges, 3, terms, with_hessian=True, fixed_vertices=default_pins(n_sample),
                       workers=workers, accumulation="atomic")
    op.eval_terms(x, psd_floor=FLOOR if psd else None)  # warm-up (layout outside the timed region)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        op.eval_terms(x, psd_floor=FLOOR if psd else None)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    units = 2 * nv + len(edges)
    return units / t, workers, f"cloth {n_sample}x{n_sample} ({units} term-elements), eval_terms(psd_floor=1e-9), median of {reps}"


# ------------------------------------------------------------------- arms

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sample = 256
    rates = []
    for _ in range(args.warmup):
        cpu_oracle_rate(sample, reps=1)
    for _ in range(args.steps):
        r, cores, desc = cpu_oracle_rate(sample, reps=1)
        rates.append(r)
    V, E = cloth_sizes(args.grid)
    val = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC,
        "value": val, "unit": "term-elements/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": (2 * V + E) / val * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cloth grid {args.grid}x{args.grid} Newton-step eval_terms(psd_floor=1e-9)",
                   "sample": f"each step: {desc}"},
        "cpu_baseline": {"value": val, "unit": "term-elements/s", "cores": cores, "kind": "port", "sample": desc},
        "e2e": {"value": val, "unit": "term-elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_engine(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as tdist

        # MG_BENCH_SHARED_GPU=1: every rank on cuda:0 over gloo (a functional run
        # of the N > 1 path on a one-GPU box; its timings are not scaling numbers)
        if os.environ.get("MG_BENCH_SHARED_GPU") == "1":
            local = 0
            torch.cuda.set_device(0)
            tdist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
    else:
        torch.cuda.set_device(0)

    n = args.grid
    t_setup = time.perf_counter()
    if world == 1:
        V, E = cloth_sizes(n)
        p, x, v = build_engine_cloth(n, args.accumulation, args.patch)
        dp = None
        step = lambda: p.eval_terms(psd_floor=FLOOR, sync=False)
    else:
        dp, V, E = build_engine_cloth_shard(n, world, rank, args.accumulation)
        p = dp.problem
        x = None
        step = lambda: dp.eval_terms(psd_floor=FLOOR, sync=False)
    t_setup = time.perf_counter() - t_setup
    units = 2 * V + E  # whole job
    nnzb_local = p.hess.nnz_blocks
    steps, warmup = (2, 1) if args.profile else (args.steps, max(args.warmup, 3))

    if (args.profile or args.only) and args.profile_call != "psd":
        vd = torch.from_numpy(np.random.default_rng(1).normal(size=p.num_dofs)).cuda()
        yd = torch.empty_like(vd)
        step = {"plain": lambda: p.eval_terms(sync=False),
                "hvp": lambda: p.hvp(p.x_device, vd, out=yd),
                "hvp_psd": lambda: p.hvp(p.x_device, vd, psd_floor=FLOOR, out=yd),
                "energy": lambda: p.eval_energy_only(p.x_device)}[args.profile_call]
    if args.profile:
        ms, _ = time_device(step, steps, warmup, dist)
        print(json.dumps({"profile": True, "ms_per_step": ms}), flush=True)
        return
    if args.only:
        ms, kms = time_with_kernel(p, step, steps, warmup, dist)
        print(json.dumps({"call": args.profile_call, "ms": ms, "kernel_ms": kms,
                          "lib": os.environ.get("MG_LIB", "default")}), flush=True)
        return

    clk = Clocks(local)  # sampled through warm-up + timed region (same kernel, same load)
    time.sleep(0.3)
    ms, kms = time_with_kernel(p, step, steps, warmup, dist)
    clocks = clk.stop()
    launches = p.launch_count() * steps
    value = units / (ms * 1e-3)
    peak, peak_kind = peaks()
    label = kernel_label(p, "psd")
    if world == 1:
        bytes_call = cloth_bytes(V, E, nnzb_local)
        achieved = bytes_call / (kms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": ncu_traffic(label), "peak_source": peak_kind, "kernel": label,
                    "algorithmic_bytes_per_launch": bytes_call, "kernel_ms": kms,
                    "kernel_share_of_step": kms / ms,
                    "bytes_note": "24V x + 24V target + 8V masses + 8E rest lengths + 8E edge ids + 24V grad + 72 nnzb H"}
    else:
        roofline = {"bound": "hbm", "kernel": label, "kernel_ms": kms, "note": "per-rank shard; see the N=1 line"}

    # e2e through the public API with host buffers
    if world == 1:
        x_host = torch.from_numpy(x).pin_memory()
        g_host = torch.empty(p.num_dofs, dtype=torch.float64).pin_memory()
        e_host = torch.empty(1, dtype=torch.float64).pin_memory()

        def e2e_step():
            p.x_device.copy_(x_host, non_blocking=True)
            p.eval_terms(psd_floor=FLOOR, sync=False)
            g_host.copy_(p.grad_device, non_blocking=True)
            e_host.copy_(p.energy_device, non_blocking=True)
    else:
        own = len(dp.plan.owned_global)
        x_host = torch.from_numpy(dp.problem.x.reshape(-1, 3)[np.flatnonzero(dp.plan.owned)].ravel()).pin_memory()
        x_dev = torch.empty(own * 3, dtype=torch.float64, device="cuda")
        g_host = torch.empty(own * 3, dtype=torch.float64).pin_memory()
        e_host = torch.empty(1, dtype=torch.float64).pin_memory()

        def e2e_step():
            x_dev.copy_(x_host, non_blocking=True)
            dp.set_x_owned(x_dev)
            dp.eval_terms(psd_floor=FLOOR, sync=False)
            g_host.copy_(dp.grad_owned().reshape(-1), non_blocking=True)
            e_host.copy_(dp.energy_device, non_blocking=True)

    ms_e2e, _ = time_device(e2e_step, max(3, steps // 2), 2, dist)
    e2e = {"value": units / (ms_e2e * 1e-3), "unit": "term-elements/s",
           "h2d_bytes_per_step": int(x_host.numel() * 8), "d2h_bytes_per_step": int(g_host.numel() * 8 + 8),
           "ms_per_step": ms_e2e, "path": "Problem.x (pinned H2D) -> eval_terms(psd_floor) -> grad + energy D2H"}

    extras = {}
    if not args.no_extras and world == 1:
        extras = run_extras(p, v, V, E, nnzb_local, steps, peak)
        if not args.no_configs:
            del p
            torch.cuda.empty_cache()
            extras.update(run_configs(peak))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r, cores, desc = cpu_oracle_rate(256, reps=3)
        cpu = {"value": r, "unit": "term-elements/s", "cores": cores, "kind": "port", "sample": desc}
    if rank == 0:
        F = 2 * (n - 1) * (n * world - 1)
        line = {
            "metric": METRIC,
            "value": value, "unit": "term-elements/s", "n_gpus": world, "steps": steps, "warmup": warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": (f"cloth grid {n}x{n * world} (V={V}, E={E}, F={F}) Newton-step "
                                    "eval_terms(psd_floor=1e-9), inertia+spring+gravity, 2 pins"),
                       "accumulation": args.accumulation, "nnzb_per_rank": nnzb_local,
                       "l2": "inputs+outputs 2.6 GB per GPU > 126 MB L2; no flush",
                       "parallelism": (f"vertex-partitioned shards x{world} (halo all_to_all + energy all_reduce)"
                                       if world > 1 else "1 GPU"),
                       "faces_per_s": F / (ms * 1e-3), "setup_s": t_setup},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_extras(p, v, V, E, nnzb, steps, peak):
    """Secondary calls of the same path, each with its kernel time and HBM fraction."""
    import torch

    out = {}
    xd = p.x_device
    vd = torch.from_numpy(v).cuda()
    y = torch.empty_like(vd)
    k = max(5, steps // 2)
    calls = [
        ("cloth_grad_hess", lambda: p.eval_terms(sync=False), cloth_bytes(V, E, nnzb)),
        ("cloth_hvp", lambda: p.hvp(xd, vd, out=y), cloth_hvp_bytes(V, E)),
        ("cloth_hvp_psd", lambda: p.hvp(xd, vd, psd_floor=FLOOR, out=y), cloth_hvp_bytes(V, E)),
        ("cloth_energy_only", lambda: p.eval_energy_only(xd), cloth_energy_bytes(V, E)),
    ]
    for name, fn, b in calls:
        ms, kms = time_with_kernel(p, fn, k, 3)
        t = kms if kms else ms
        out[name] = {"ms": ms, "kernel_ms": kms, "term_elements_per_s": (2 * V + E) / (ms * 1e-3),
                     "algorithmic_bytes": b, "hbm_frac": b / (t * 1e-3) / 1e9 / peak}
    return out


def run_configs(peak, sub=9):
    """The other BASELINE workloads, one call each (device ms, main-kernel ms,
    HBM fraction of the algorithmic bytes): the >= 10M-face cloth (config 2'),
    symmetric Dirichlet grad+Hessian (config 3) and sphere / smoothing HVPs
    (config 4) on icosphere(sub)."""
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import (distortion_problem, edge_length_problem, initial_sphere, rest_geometry,
                                            sphere_problem, tangent_bases)

    out = {}

    def rec(name, p, fn, units, unit, nbytes, k=10):
        ms, kms = time_with_kernel(p, fn, k, 3)
        t = kms if kms else ms
        out[name] = {"ms": ms, "kernel_ms": kms, unit + "_per_s": units / (ms * 1e-3), "algorithmic_bytes": nbytes,
                     "hbm_frac": nbytes / (t * 1e-3) / 1e9 / peak}

    # config 2': cloth 2240^2 (10.03M faces), Newton step
    n = 2240
    p, x, v = build_engine_cloth(n, "deterministic")
    V, E = cloth_sizes(n)
    vd = torch.from_numpy(v).cuda()
    y = torch.empty_like(vd)
    rec("cloth2240_grad_hess_psd", p, lambda: p.eval_terms(psd_floor=FLOOR, sync=False), 2 * V + E, "term_elements",
        cloth_bytes(V, E, p.hess.nnz_blocks))
    rec("cloth2240_hvp", p, lambda: p.hvp(p.x_device, vd, out=y), 2 * V + E, "term_elements", cloth_hvp_bytes(V, E))
    del p, vd, y
    torch.cuda.empty_cache()
    # config 3: symmetric Dirichlet on the punctured icosphere
    pos, faces, uv = mg.punctured_icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    rest_inv, areas = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in rest_geometry(mesh))
    p = distortion_problem(mesh, rest_inv, areas, with_hessian=True)
    p.precompute_sparsity()
    p.x = uv.ravel()
    V, F, nnzb = len(pos), len(faces), p.hess.nnz_blocks
    vd = torch.from_numpy(np.random.default_rng(1).normal(size=2 * V)).cuda()
    y = torch.empty_like(vd)
    rec(f"dirichlet_ico{sub}_grad_hess", p, lambda: p.eval_terms(sync=False), F, "faces",
        16 * V + 12 * F + 32 * F + 8 * F + 16 * V + 32 * nnzb)
    rec(f"dirichlet_ico{sub}_hvp", p, lambda: p.hvp(p.x_device, vd, out=y), F, "faces",
        16 * V + 16 * V + 12 * F + 32 * F + 8 * F + 16 * V)
    del p, vd, y
    torch.cuda.empty_cache()
    # config 4: sphere manifold HVP, smoothing HVP
    pos, faces = mg.icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    base = initial_sphere(mesh)
    b1, b2 = tangent_bases(base)
    base, b1, b2 = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (base, b1, b2))
    p = sphere_problem(mesh, base, b1, b2)
    V, F = len(pos), len(faces)
    p.x = 1e-5 * np.random.default_rng(0).normal(size=2 * V)  # tangent noise well below the edge length (no flips)
    vd = torch.from_numpy(np.random.default_rng(1).normal(size=2 * V)).cuda()
    y = torch.empty_like(vd)
    rec(f"sphere_ico{sub}_hvp", p, lambda: p.hvp(p.x_device, vd, out=y), F, "faces",
        16 * V + 16 * V + 72 * V + 12 * F + 16 * V)
    del p, vd, y
    p = edge_length_problem(mesh)
    p.x = pos.ravel()
    E = 3 * F // 2
    vd = torch.from_numpy(np.random.default_rng(1).normal(size=3 * V)).cuda()
    y = torch.empty_like(vd)
    rec(f"smooth_ico{sub}_hvp", p, lambda: p.hvp(p.x_device, vd, out=y), E, "edges", 24 * V + 8 * E + 24 * V)
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_engine(args)


if __name__ == "__main__":
    main()
