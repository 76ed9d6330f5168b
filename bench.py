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
  e2e     : the public API with host buffers, every step: pinned x H2D, eval,
            energy + gradient + the 2.1 GB of Hessian values D2H into pinned
            host memory (the reference's eval_terms leaves all three in host
            memory); extras.cloth_e2e_h_on_device is the same without the
            Hessian copy (a consumer that keeps H on the device)
  roofline: HBM; algorithmic bytes of one call (inputs read once + outputs
            written once) / the assembly kernel's own device time
            (library-side CUDA events around that launch, same timed region);
            traffic = DRAM bytes of the same kernel from the committed ncu
            capture (profiles/ncu_kernels.json)
  cpu_baseline: the CPU oracle port (oracle/, restating meshgrad's numpy
            path) on the SAME 2048^2 problem, all host threads, atomic
            accumulation (the reference CLI default): a bounded sample = a
            fixed stride of the call's 4096-element chunks, so the per-element
            rate is the full call's (the sample's elements / its time)
  extras  : the other calls of the path (grad+H, HVP, HVP(psd), energy probe),
            BASELINE configs 2' (cloth 2240^2, 10.0M faces), 3 (symmetric
            Dirichlet, punctured icosphere(10), 21M faces), 4 (sphere and
            smoothing HVPs, icosphere(10)) and 5 (cloth 7072^2, 100M faces,
            gradient + HVP) with a roofline object each: HBM fraction of the
            algorithmic bytes and, for the face kernels, the FP64 fraction of
            the ncu-executed flops (dadd + dmul + 2 dfma) against the measured
            FP64 peak (profiles/fp64_peak.json); `bound` is the unit ncu shows
            busier

Multi-GPU (torchrun, N ranks): weak scaling. The global cloth is a
2048 x (2048 N) grid partitioned by vertex ownership (distributed.py); each
rank assembles its owned rows after a halo exchange of ribbon x, and the energy
is all-reduced. Time = max over ranks.

`--impl reference` runs the reference arm: the CPU oracle port on the same
2048^2 problem and call (rank 0 only), each step a fixed-stride 1/16 sample of
the call's chunks; its extras time each of the five calls once at full size
(all threads, atomic) and a workers=1 deterministic sample of each.
"""

from __future__ import annotations

import argparse
import json
import os
import resource
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
    ap.add_argument("--sub", type=int, default=10, help="icosphere subdivisions of configs 3-4 (BASELINE: 10)")
    ap.add_argument("--grid5", type=int, default=7072, help="cloth grid of config 5 (BASELINE: 7072, 100M faces)")
    ap.add_argument("--accumulation", default="deterministic", choices=["deterministic", "atomic"])
    ap.add_argument("--patch", type=int, default=64, help="owned rows per vertex patch (generic patch path)")
    ap.add_argument("--no-extras", action="store_true", help="skip the secondary workloads")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE configs 2'/3/4/5 extras")
    ap.add_argument("--no-config5", action="store_true", help="skip the 100M-face config 5 extra")
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
    import torch

    from paper_2509_00406_b200.distributed import DistributedProblem
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    ny = n * world
    sp = 1.0 / (n - 1)
    pos, faces = grid_rect_arrays(n, ny, sp)
    target, x, v = cloth_state(pos, n)
    # lumped masses and rest lengths built on the rank's device (every rank
    # holds the whole grid's inputs; a host build is O(mesh) numpy per rank),
    # and passed as device attributes as on the N = 1 path (numpy attributes
    # are re-read on every call, the reference's live-closure semantics)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    pos_d, f_d = dev(pos), dev(faces)
    cr = torch.linalg.cross(pos_d[f_d[:, 1]] - pos_d[f_d[:, 0]], pos_d[f_d[:, 2]] - pos_d[f_d[:, 0]])
    area3 = (0.5 * torch.linalg.vector_norm(cr, dim=1) / 3.0).repeat_interleave(3)
    masses_d = torch.zeros(len(pos), dtype=torch.float64, device="cuda").index_add_(0, f_d.reshape(-1), area3)
    sides = torch.cat([f_d[:, [0, 1]], f_d[:, [1, 2]], f_d[:, [2, 0]]])
    keys = torch.unique(sides.min(dim=1).values * len(pos) + sides.max(dim=1).values)  # the engine's edge order
    dd = pos_d[keys % len(pos)] - pos_d[keys // len(pos)]
    l2 = (dd * dd).sum(dim=1)
    n_edges = keys.numel()
    del cr, area3, sides, keys, dd, pos_d, f_d
    h = 0.01
    terms = [("V", Inertia(masses_d, dev(target))), ("EV", Spring(l2, 0.5 * 1e4 * h * h)),
             ("V", Gravity(masses_d, np.array([0.0, -9.8, 0.0]), h * h))]
    pins = (n * (ny - 1), n * ny - 1)
    # id-range partition: horizontal 2048-row stripes of the row-major grid
    dp = DistributedProblem(pos, faces, 3, terms, fixed_vertices=pins, accumulation=accumulation, partition="range")
    dp.set_x_global(x)
    dp.problem.precompute_sparsity()
    return dp, len(pos), n_edges


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


def fp64_peak():
    """FP64 FMA throughput measured on this pool's B200 by tools/fp64_peak
    (MEASURED_PEAKS.json carries no FP64 figure); nominal 37 TF/s otherwise."""
    try:
        d = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())
        return float(d["fp64_tflops"]), "measured (tools/fp64_peak, profiles/fp64_peak.json)"
    except Exception:
        return 37.0, "nominal"


def ncu_kernel(label):
    """Per-launch ncu facts of a kernel from the committed captures
    (profiles/ncu_kernels.json): DRAM bytes, executed FP64 flops, DRAM% and
    FP64-pipe% (which unit binds)."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_kernels.json").read_text())
        return d.get(label) or {}
    except Exception:
        return {}


def roofline_obj(label, kernel_ms, nbytes, hbm_peak, hbm_src, note=None, workload="grid2048"):
    """Roofline object of one launch: the HBM fraction of the algorithmic
    bytes always; the FP64 fraction of the ncu-executed flops when the
    capture has them; `bound` = the unit ncu shows busier. ncu facts (DRAM
    traffic, executed flops) are per launch of the captured workload, so they
    are used only for that workload."""
    nk = ncu_kernel(label)
    if nk.get("workload", "grid2048") != workload:
        nk = {}
    achieved = nbytes / (kernel_ms * 1e-3) / 1e9
    r = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
         "traffic": nk.get("traffic"), "peak_source": hbm_src, "kernel": label,
         "algorithmic_bytes_per_launch": nbytes, "kernel_ms": kernel_ms, "hbm_frac": achieved / hbm_peak}
    if nk.get("fp64_flops"):
        fpk, fsrc = fp64_peak()
        tf = nk["fp64_flops"] / (kernel_ms * 1e-3) / 1e12
        r.update({"fp64_flops_per_launch": nk["fp64_flops"], "fp64_tflops": tf, "fp64_peak": fpk,
                  "fp64_peak_source": fsrc, "fp64_frac": tf / fpk,
                  "ncu_dram_pct": nk.get("dram_pct"), "ncu_fp64_pipe_pct": nk.get("fp64_pipe_pct")})
        if (nk.get("fp64_pipe_pct") or 0) > (nk.get("dram_pct") or 0):
            r.update({"bound": "fp64", "achieved": tf, "peak": fpk, "unit": "TFLOP/s", "frac": tf / fpk})
    if note:
        r["bytes_note"] = note
    return r


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

def cpu_info():
    info = {"cpu_count": os.cpu_count(), "numpy": np.__version__}
    try:
        info["affinity"] = len(os.sched_getaffinity(0))
    except AttributeError:
        pass
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name"):
                info["model"] = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return info


class CpuCloth:
    """The CPU oracle port (oracle/: the reference's numpy pipeline restated)
    on the same cloth problem as the engine's headline: same mesh, terms,
    pins and state. Setup (layout + pattern) is outside every timed region,
    as in the reference (apps/smooth.py:104)."""

    def __init__(self, n, workers, accumulation):
        from oracle import OracleProblem
        from paper_2509_00406_b200.apps import default_pins
        from paper_2509_00406_b200.mesh import _host_edges
        from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

        pos, faces, target, x, v = cloth_inputs(n)
        nv = len(pos)
        edges = _host_edges(faces, None, nv)
        areas = 0.5 * np.linalg.norm(np.cross(pos[faces[:, 1]] - pos[faces[:, 0]], pos[faces[:, 2]] - pos[faces[:, 0]]),
                                     axis=1)
        masses = np.bincount(faces.ravel(), weights=np.repeat(areas / 3.0, 3), minlength=nv)
        d = pos[edges[:, 1]] - pos[edges[:, 0]]
        h = 0.01
        terms = [("V", Inertia(masses, target)), ("EV", Spring(np.einsum("ij,ij->i", d, d), 0.5 * 1e4 * h * h)),
                 ("V", Gravity(masses, np.array([0.0, -9.8, 0.0]), h * h))]
        self.workers = workers
        self.op = OracleProblem(nv, faces, edges, 3, terms, with_hessian=True, fixed_vertices=default_pins(n),
                                workers=workers, accumulation=accumulation)
        self.x, self.v = x, v
        self.units = 2 * nv + len(edges)
        self.sizes = [sl.stop - sl.start for _, _, _, sl in self.op._tasks()]

    def call(self, name):
        o, x, v = self.op, self.x, self.v
        return {"eval_terms": lambda: o.eval_terms(x),
                "eval_terms_psd": lambda: o.eval_terms(x, psd_floor=FLOOR),
                "hvp": lambda: o.hvp(x, v),
                "hvp_psd": lambda: o.hvp(x, v, psd_floor=FLOOR),
                "energy_only": lambda: o.eval_energy_only(x)}[name]

    def sample(self, name, stride, k):
        """(term-elements, seconds) of one call restricted to chunks k, k+stride, ..."""
        self.op.task_slice = slice(k % stride, None, stride) if stride > 1 else None
        units = sum(self.sizes[k % stride::stride]) if stride > 1 else self.units
        t0 = time.perf_counter()
        self.call(name)()
        dt = time.perf_counter() - t0
        self.op.task_slice = None
        return units, dt

    def rate(self, name, stride, steps, warmup):
        for k in range(warmup):
            self.sample(name, stride, k)
        rates = []
        for k in range(steps):
            u, dt = self.sample(name, stride, warmup + k)
            rates.append(u / dt)
        return statistics.median(rates), rates


def cpu_config_rates(sub=8, stride=16, steps=3):
    """CPU oracle port rates of BASELINE configs 3 and 4 (all host threads,
    atomic accumulation, the reference CLI default): per call, the elements
    per second of a fixed-stride 1/stride chunk sample, median of `steps`
    after one warm-up. The oracle runs the reference's numpy path chunk by
    chunk (4096 elements), so its per-element rate does not depend on the
    mesh size; its setup (pattern, layout) on icosphere(10) would take
    minutes, so the sample mesh is icosphere(`sub`)."""
    from oracle import OracleProblem
    from oracle.engine import default_workers

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import initial_sphere, rest_geometry, tangent_bases
    from paper_2509_00406_b200.mesh import _host_edges
    from paper_2509_00406_b200.terms import EdgeLength, SphereBarrierStretch, SymDirichlet

    workers = default_workers()
    rng = np.random.default_rng(1)
    out = {}

    def rate(op, name, fn):
        sizes = [sl.stop - sl.start for _, _, _, sl in op._tasks()]
        rates = []
        for k in range(steps + 1):
            op.task_slice = slice(k % stride, None, stride)
            units = sum(sizes[k % stride::stride])
            t0 = time.perf_counter()
            fn()
            dt = time.perf_counter() - t0
            if k:
                rates.append(units / dt)
        op.task_slice = None
        return statistics.median(rates)

    pos, faces, uv = mg.punctured_icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    ri, ar = rest_geometry(mesh)
    op = OracleProblem(len(pos), faces, _host_edges(faces, None, len(pos)), 2,
                       [("FV", SymDirichlet(np.ascontiguousarray(ri).reshape(-1, 4), ar))], with_hessian=True,
                       workers=workers, accumulation="atomic")
    x, v = uv.ravel(), rng.normal(size=2 * len(pos))
    out["dirichlet"] = {"grad_hess": rate(op, "eval_terms", lambda: op.eval_terms(x)),
                        "hvp": rate(op, "hvp", lambda: op.hvp(x, v)), "unit": "faces/s"}
    del op
    pos, faces = mg.icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    edges = _host_edges(faces, None, len(pos))
    base = initial_sphere(mesh)
    b1, b2 = tangent_bases(base)
    op = OracleProblem(len(pos), faces, edges, 2, [("FV", SphereBarrierStretch(base, b1, b2, True, True))],
                       with_hessian=False, workers=workers, accumulation="atomic")
    x, v = 1e-5 * rng.normal(size=2 * len(pos)), rng.normal(size=2 * len(pos))
    out["sphere"] = {"grad": rate(op, "eval_terms", lambda: op.eval_terms(x)),
                     "hvp": rate(op, "hvp", lambda: op.hvp(x, v)), "unit": "faces/s"}
    del op
    op = OracleProblem(len(pos), faces, edges, 3, [("EV", EdgeLength())], with_hessian=False, workers=workers,
                       accumulation="atomic")
    x, v = pos.ravel(), rng.normal(size=3 * len(pos))
    out["smoothing"] = {"grad": rate(op, "eval_terms", lambda: op.eval_terms(x)),
                        "hvp": rate(op, "hvp", lambda: op.hvp(x, v)), "unit": "edges/s"}
    out.update({"cores": workers, "kind": "port", "sample": (
        f"icosphere({sub}) meshes (the per-element rate of the chunked numpy path is size-independent; setup on "
        f"icosphere(10) takes minutes), every {stride}th 4096-element chunk, median of {steps} after 1 warm-up, "
        f"atomic, {workers} threads"), "host": cpu_info()})
    return out


def cpu_baseline_line(n, stride=64, steps=3):
    """cpu_baseline of the engine arm: the oracle port on the same problem, all
    host threads, a 1/stride chunk sample of eval_terms(psd_floor) per step."""
    from oracle.engine import default_workers

    workers = default_workers()
    ref = CpuCloth(n, workers, "atomic")
    val, _ = ref.rate("eval_terms_psd", stride, steps, 1)
    return {"value": val, "unit": "term-elements/s", "cores": workers, "kind": "port",
            "sample": (f"cloth {n}x{n} (the headline problem, {ref.units} term-elements per full call), "
                       f"eval_terms(psd_floor=1e-9), atomic, {workers} threads; each sample = every {stride}th of the "
                       f"call's {len(ref.sizes)} 4096-element chunks (~{ref.units // stride} term-elements), "
                       f"median of {steps} after 1 warm-up"),
            "host": cpu_info()}


# ------------------------------------------------------------------- arms

def run_reference(args):
    """The reference arm: the oracle port (oracle/, the reference's numpy path
    restated and pinned to the reference's own outputs) on the SAME 2048^2
    problem and call as the engine arm, all host threads (atomic, the
    reference CLI default, cli.py:25,34-35). Each step = the call restricted
    to a fixed-stride 1/16 of its chunks (a bounded sample; the per-element
    rate is the full call's). Extras: each of the five calls once at full
    size, and a workers=1 deterministic 1/64 sample of each."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.engine import default_workers

    workers = default_workers()
    t_setup = time.perf_counter()
    ref = CpuCloth(args.grid, workers, "atomic")
    t_setup = time.perf_counter() - t_setup
    stride = 16
    val, rates = ref.rate("eval_terms_psd", stride, args.steps, args.warmup)
    ms = ref.units / val * 1e3
    desc = (f"each step: eval_terms(psd_floor=1e-9) on every {stride}th of the full 2048^2 call's "
            f"{len(ref.sizes)} 4096-element chunks (~{ref.units // stride} term-elements), {workers} threads, atomic; "
            f"ms_per_step = the full call's time at the measured rate")
    extras = {"setup_s": t_setup}
    full = {}
    for name in ("eval_terms", "eval_terms_psd", "hvp", "hvp_psd", "energy_only"):
        u, dt = ref.sample(name, 1, 0)
        full[name] = {"s": dt, "term_elements_per_s": u / dt}
    extras["full_calls_all_threads"] = full
    ref1 = CpuCloth.__new__(CpuCloth)
    ref1.__dict__.update(ref.__dict__)
    ref.op.workers, ref.op.accumulation = 1, "deterministic"
    one = {}
    for name in ("eval_terms", "eval_terms_psd", "hvp", "hvp_psd", "energy_only"):
        u, dt = ref.sample(name, 64, 0)
        one[name] = {"sample_s": dt, "term_elements_per_s": u / dt, "full_call_s_at_rate": ref.units / (u / dt)}
    extras["workers1_deterministic_1_64_sample"] = one
    line = {
        "impl": "reference", "metric": METRIC,
        "value": val, "unit": "term-elements/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": headline_config(args.grid, 1, args.accumulation),
        "cpu_baseline": {"value": val, "unit": "term-elements/s", "cores": workers, "kind": "port", "sample": desc,
                         "host": cpu_info()},
        "e2e": {"value": val, "unit": "term-elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extras": extras,
    }
    print(json.dumps(line), flush=True)


def headline_config(n, world, accumulation):
    V, E = cloth_sizes(n, n * world)
    F = 2 * (n - 1) * (n * world - 1)
    return {"workload": (f"cloth grid {n}x{n * world} (V={V}, E={E}, F={F}) Newton-step "
                         "eval_terms(psd_floor=1e-9), inertia+spring+gravity, 2 pins"),
            "accumulation": accumulation,
            "l2": "inputs+outputs 2.6 GB per GPU > 126 MB L2; no flush",
            "parallelism": (f"vertex-partitioned shards x{world} (halo all_to_all + energy all_reduce)"
                            if world > 1 else "1 GPU")}


def run_engine(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # MG_BENCH_DIST=1: the sharded path (NCCL, halo exchange, energy all_reduce)
    # even at one rank, so a one-GPU box runs the N > 1 code end to end
    sharded = world > 1 or os.environ.get("MG_BENCH_DIST") == "1"
    dist = None
    if sharded:
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
    if not sharded:
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
    if not sharded:
        roofline = roofline_obj(label, kms, cloth_bytes(V, E, nnzb_local), peak, peak_kind,
                                "24V x + 24V target + 8V masses + 8E rest lengths + 8E edge ids + 24V grad + 72 nnzb H",
                                workload=f"grid{n}")
        roofline["kernel_share_of_step"] = kms / ms
    else:
        roofline = {"bound": "hbm", "kernel": label, "kernel_ms": kms, "note": "per-rank shard; see the N=1 line"}

    # e2e through the public API with host buffers
    extras = {}
    if not sharded:
        x_host = torch.from_numpy(x).pin_memory()
        g_host = torch.empty(p.num_dofs, dtype=torch.float64).pin_memory()
        e_host = torch.empty(1, dtype=torch.float64).pin_memory()
        h_host = torch.empty_like(p.hess.values_device, device="cpu").pin_memory()

        def e2e_step(with_h=True):
            p.x_device.copy_(x_host, non_blocking=True)
            p.eval_terms(psd_floor=FLOOR, sync=False)
            g_host.copy_(p.grad_device, non_blocking=True)
            e_host.copy_(p.energy_device, non_blocking=True)
            if with_h:
                h_host.copy_(p.hess.values_device, non_blocking=True)
        d2h = int(g_host.numel() * 8 + 8 + h_host.numel() * 8)
        path = "Problem.x (pinned H2D) -> eval_terms(psd_floor) -> energy + grad + Hessian values D2H (pinned)"
    else:
        own = len(dp.plan.owned_global)
        x_host = torch.from_numpy(dp.problem.x.reshape(-1, 3)[np.flatnonzero(dp.plan.owned)].ravel()).pin_memory()
        x_dev = torch.empty(own * 3, dtype=torch.float64, device="cuda")
        g_host = torch.empty(own * 3, dtype=torch.float64).pin_memory()
        e_host = torch.empty(1, dtype=torch.float64).pin_memory()

        def e2e_step(with_h=False):
            x_dev.copy_(x_host, non_blocking=True)
            dp.set_x_owned(x_dev)
            dp.eval_terms(psd_floor=FLOOR, sync=False)
            g_host.copy_(dp.grad_owned().reshape(-1), non_blocking=True)
            e_host.copy_(dp.energy_device, non_blocking=True)
        d2h = int(g_host.numel() * 8 + 8)
        path = "owned x (pinned H2D) -> halo -> eval_terms(psd_floor) -> energy + owned grad D2H"

    ms_e2e, _ = time_device(e2e_step, max(3, steps // 2), 2, dist)
    e2e = {"value": units / (ms_e2e * 1e-3), "unit": "term-elements/s",
           "h2d_bytes_per_step": int(x_host.numel() * 8), "d2h_bytes_per_step": d2h,
           "ms_per_step": ms_e2e, "path": path}
    if not sharded:
        ms_dev_h, _ = time_device(lambda: e2e_step(False), max(3, steps // 2), 2, dist)
        extras["cloth_e2e_h_on_device"] = {
            "ms": ms_dev_h, "term_elements_per_s": units / (ms_dev_h * 1e-3),
            "h2d_bytes_per_step": int(x_host.numel() * 8), "d2h_bytes_per_step": int(g_host.numel() * 8 + 8),
            "path": "as e2e, but the Hessian stays on the device"}
        del h_host

    if not args.no_extras and not sharded:
        extras.update(run_extras(p, v, V, E, nnzb_local, steps, peak, peak_kind))
        for k, r in run_traced(n, max(5, steps // 2), peak, peak_kind).items():
            r["vs_builtin_newton_step"] = r["newton_step_ms"] / ms
            extras[k] = r
        extras.update(run_fp32(n, max(5, steps // 2), peak, peak_kind))
    if not args.no_configs and not sharded:
        del p
        gc_cuda()
        extras.update(run_configs(peak, peak_kind, args.sub))
        if not args.no_cpu:
            extras["configs_cpu_baseline"] = cpu_config_rates()
        if not args.no_config5:
            extras.update(run_config5(peak, peak_kind, args.grid5))
    if sharded and not args.no_config5:
        del p, dp
        gc_cuda()
        extras.update(run_config5_dist(world, rank, dist, args.grid5))
    cpu = None
    if rank == 0 and not sharded and not args.no_cpu:
        cpu = cpu_baseline_line(n)
    if rank == 0:
        cfg = headline_config(n, world, args.accumulation)
        cfg.update({"nnzb_per_rank": nnzb_local, "faces_per_s": 2 * (n - 1) * (n * world - 1) / (ms * 1e-3),
                    "setup_s": t_setup})
        line = {
            "metric": METRIC,
            "value": value, "unit": "term-elements/s", "n_gpus": world, "steps": steps, "warmup": warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": cfg,
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


def gc_cuda():
    import gc

    import torch

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def call_record(p, fn, units, unit, nbytes, label, peak, peak_kind, steps=10, extra=None, workload="grid2048"):
    ms, kms = time_with_kernel(p, fn, steps, 3)
    t = kms if kms else ms
    r = {"ms": ms, "kernel_ms": kms, unit + "_per_s": units / (ms * 1e-3), "algorithmic_bytes": nbytes,
         "hbm_frac": nbytes / (t * 1e-3) / 1e9 / peak,
         "roofline": roofline_obj(label, t, nbytes, peak, peak_kind, workload=workload)}
    if extra:
        r.update(extra)
    return r


def run_extras(p, v, V, E, nnzb, steps, peak, peak_kind):
    """The headline problem's other calls, each with its kernel time and roofline."""
    import torch

    xd = p.x_device
    vd = torch.from_numpy(v).cuda()
    y = torch.empty_like(vd)
    k = max(5, steps // 2)
    te = 2 * V + E
    return {
        "cloth_grad_hess": call_record(p, lambda: p.eval_terms(sync=False), te, "term_elements",
                                       cloth_bytes(V, E, nnzb), kernel_label(p, "plain"), peak, peak_kind, k, workload="grid2048"),
        "cloth_hvp": call_record(p, lambda: p.hvp(xd, vd, out=y), te, "term_elements", cloth_hvp_bytes(V, E),
                                 kernel_label(p, "hvp"), peak, peak_kind, k, workload="grid2048"),
        "cloth_hvp_psd": call_record(p, lambda: p.hvp(xd, vd, psd_floor=FLOOR, out=y), te, "term_elements",
                                     cloth_hvp_bytes(V, E), kernel_label(p, "hvp_psd"), peak, peak_kind, k, workload="grid2048"),
        "cloth_energy_only": call_record(p, lambda: p.eval_energy_only(xd), te, "term_elements",
                                         cloth_energy_bytes(V, E), "k_elem energy (3 launches)", peak, peak_kind, k, workload="grid2048"),
        "cloth_newton_cg": run_pcg(p, nnzb, V),
    }


def run_fp32(n, steps, peak, peak_kind):
    """The headline problem with fp32 storage (Problem(dtype=torch.float32)):
    x, target, masses, rest lengths, gradient, Hessian values and HVP vectors
    in fp32, the edge row kernels computing in fp64; algorithmic bytes halve
    except the int32 edge ids (12V x + 12V target + 4V masses + 4E l2 + 8E ids
    + 12V grad + 36 nnzb)."""
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import ClothConfig, cloth_problem, default_pins, lumped_masses

    pos, faces, target, x, v = cloth_inputs(n)
    mesh = mg.Mesh(pos, faces)
    cfg = ClothConfig(grid_n=n, spacing=1.0 / (n - 1))
    p = cloth_problem(cfg, mesh, torch.from_numpy(target).cuda(),
                      masses=torch.from_numpy(lumped_masses(mesh, cfg.mass_density)).cuda(), pinned=default_pins(n),
                      dtype=torch.float32, live_host_attrs=False)
    p.precompute_sparsity()
    p.x = x
    V, E = cloth_sizes(n)
    nnzb = p.hess.nnz_blocks
    b_h = 12 * V + 12 * V + 4 * V + 4 * E + 8 * E + 12 * V + 36 * nnzb
    b_v = 12 * V + 12 * V + 4 * V + 4 * E + 8 * E + 12 * V
    vd = torch.from_numpy(v).cuda().to(torch.float32)
    y = torch.empty_like(vd)
    te = 2 * V + E
    out = {}
    for name, fn, nb in (("grad_hess_psd", lambda: p.eval_terms(psd_floor=FLOOR, sync=False), b_h),
                         ("grad_hess", lambda: p.eval_terms(sync=False), b_h),
                         ("hvp", lambda: p.hvp(p.x_device, vd, out=y), b_v),
                         ("hvp_psd", lambda: p.hvp(p.x_device, vd, psd_floor=FLOOR, out=y), b_v)):
        ms, kms = time_with_kernel(p, fn, steps, 3)
        t = kms if kms else ms
        out["cloth_fp32_" + name] = {"ms": ms, "kernel_ms": kms, "term_elements_per_s": te / (ms * 1e-3),
                                     "algorithmic_bytes": nb, "hbm_frac": nb / (t * 1e-3) / 1e9 / peak,
                                     "storage": "fp32 (fp64 arithmetic)", "parity": "tests/test_fp32_gpu.py: 1e-5"}
    del p, vd, y, mesh
    gc_cuda()
    return out


def run_pcg(p, nnzb, V, iters=40):
    """The Newton direction solve on the headline Hessian (newton_solve's inner
    CG, block-Jacobi PCG, a fixed 40 iterations: tol 0): the device PCG
    (mg_pcg, scalars on the GPU) against the reference-structured
    cg_linear_solve on the same device operators (3 host syncs per
    iteration); per-iteration wall time on the host clock (syncs included),
    and the HBM fraction of one iteration's algorithmic bytes (SpMV, the
    fused x / r / z update with the block-Jacobi apply, the p update)."""
    import torch

    import paper_2509_00406_b200.solvers as S

    p.eval_terms(psd_floor=FLOOR)
    b = -p.grad_device.clone()
    cfg = S.SolverConfig(cg_tol=0.0, cg_max_iters=iters)
    out = {}
    for name, fn in (("device_pcg", lambda: S.device_cg(p, b, cfg, hess=p.hess.values_device)),
                     ("host_cg", lambda: S.cg_linear_solve(p.hess.matvec, b, 0.0, iters,
                                                           precond=S._block_jacobi(p)))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            _, info = fn()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / 3
        out[name] = {"ms_per_solve": ms, "iterations": info.iterations, "ms_per_iteration": ms / info.iterations}
    # per iteration: SpMV 72 nnzb + 24V p + 24V y; update p, y, r, x read, the 3x3
    # block-Jacobi inverses read (72V), x, r, z written; p update z, p read, p written
    it_bytes = 72 * nnzb + (48 + 96 + 72 + 72 + 72) * V
    it_ms = out["device_pcg"]["ms_per_iteration"]
    out["device_pcg"]["bytes_per_iteration"] = it_bytes
    out["device_pcg"]["hbm_frac"] = it_bytes / (it_ms * 1e-3) / 1e9 / peaks()[0]
    out["speedup"] = out["host_cg"]["ms_per_solve"] / out["device_pcg"]["ms_per_solve"]
    return out


def run_traced(n, steps, peak, peak_kind):
    """The same cloth Newton step with the terms registered as reference-style
    Python callbacks (the builtin terms' __call__ bodies are the reference
    app's formulas, apps/cloth.py:102-113): traced once, compiled by nvcc for
    sm_100a, assembled (a) by the generated edge row module (jit_rows.cuh:
    the tracer proves the spring radial, phi(r) on a one-variable
    second-order dual), (b) by the problem's generated patch module
    (jit_patch.cuh) and (c) by the element-parallel kernels with fixed-order
    gather. Closure arrays are snapshots (live_host_attrs=False) so the timed
    region holds only device work."""
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import default_pins, lumped_masses, rest_lengths2
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    pos, faces, target, x, v = cloth_inputs(n)
    V, E = cloth_sizes(n)
    out = {}
    for path, env, rows in (("rows", "0", "1"), ("patch", "0", "0"), ("element", str(1 << 62), "0")):
        os.environ["MG_JIT_PATCH_MIN"] = env
        os.environ["MG_JIT_ROWS"] = rows
        t0 = time.perf_counter()
        mesh = mg.Mesh(pos, faces)
        masses = lumped_masses(mesh, 1.0)
        h2 = 0.01 * 0.01
        terms = [Inertia(masses, target), Spring(rest_lengths2(mesh), 0.5 * 1e4 * h2),
                 Gravity(masses, np.array([0.0, -9.8, 0.0]), h2)]
        p = mg.Problem(mesh, 3, fixed_vertices=default_pins(n), live_host_attrs=False)
        for t in terms:
            p.add_term(t.kind, t.op, lambda hd, nb, xx, _t=t: _t(hd, nb, xx))  # plain callbacks: traced
        p.precompute_sparsity()
        p.x = x
        p.eval_terms(psd_floor=FLOOR)
        st = time.perf_counter() - t0
        vd = torch.from_numpy(v).cuda()
        y = torch.empty_like(vd)
        ms, _ = time_device(lambda: p.eval_terms(psd_floor=FLOOR, sync=False), steps, 3)
        ms_h, _ = time_device(lambda: p.hvp(p.x_device, vd, out=y), steps, 3)
        out[f"cloth_traced_{path}"] = {
            "newton_step_ms": ms, "term_elements_per_s": (2 * V + E) / (ms * 1e-3), "hvp_ms": ms_h,
            "setup_and_compile_s": st, "patch_module": p.patch_module, "row_module": p.row_module,
            "hbm_frac_newton_step": cloth_bytes(V, E, p.hess.nnz_blocks) / (ms * 1e-3) / 1e9 / peak}
        del p, vd, y, mesh
        gc_cuda()
    os.environ.pop("MG_JIT_PATCH_MIN", None)
    os.environ.pop("MG_JIT_ROWS", None)
    return out


def run_configs(peak, peak_kind, sub=10):
    """The other BASELINE workloads at their BASELINE sizes, per call: device
    ms, main-kernel ms, rate and a roofline object. Config 2' is the >= 10M
    face cloth (2240^2), config 3 symmetric Dirichlet grad + Hessian on the
    punctured icosphere(10), config 4 the sphere and smoothing HVPs on
    icosphere(10)."""
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import (distortion_problem, edge_length_problem, initial_sphere, rest_geometry,
                                            sphere_problem, tangent_bases)

    out = {}
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    # config 2': cloth 2240^2 (10.03M faces)
    n = 2240
    t0 = time.perf_counter()
    p, x, v = build_engine_cloth(n, "deterministic")
    st = time.perf_counter() - t0
    V, E = cloth_sizes(n)
    vd, y = dev(v), torch.empty(3 * V, dtype=torch.float64, device="cuda")
    ex = {"V": V, "E": E, "F": 2 * (n - 1) ** 2, "setup_s": st}
    out["cloth2240_grad_hess_psd"] = call_record(
        p, lambda: p.eval_terms(psd_floor=FLOOR, sync=False), 2 * V + E, "term_elements",
        cloth_bytes(V, E, p.hess.nnz_blocks), kernel_label(p, "psd"), peak, peak_kind, extra=ex, workload="grid2240")
    out["cloth2240_grad_hess"] = call_record(
        p, lambda: p.eval_terms(sync=False), 2 * V + E, "term_elements", cloth_bytes(V, E, p.hess.nnz_blocks),
        kernel_label(p, "plain"), peak, peak_kind, workload="grid2240")
    out["cloth2240_hvp"] = call_record(p, lambda: p.hvp(p.x_device, vd, out=y), 2 * V + E, "term_elements",
                                       cloth_hvp_bytes(V, E), kernel_label(p, "hvp"), peak, peak_kind, workload="grid2240")
    out["cloth2240_hvp_psd"] = call_record(p, lambda: p.hvp(p.x_device, vd, psd_floor=FLOOR, out=y), 2 * V + E,
                                           "term_elements", cloth_hvp_bytes(V, E), kernel_label(p, "hvp_psd"), peak,
                                           peak_kind, workload="grid2240")
    del p, vd, y
    gc_cuda()
    # config 3: symmetric Dirichlet on the punctured icosphere (stereographic UV, all det J > 0)
    t0 = time.perf_counter()
    pos, faces, uv = mg.punctured_icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    rest_inv, areas = (dev(a) for a in rest_geometry(mesh))
    p = distortion_problem(mesh, rest_inv, areas, with_hessian=True)
    p.precompute_sparsity()
    p.x = uv.ravel()
    V, F, nnzb = len(pos), len(faces), p.hess.nnz_blocks
    st = time.perf_counter() - t0
    vd = dev(np.random.default_rng(1).normal(size=2 * V))
    y = torch.empty_like(vd)
    b_hess = 16 * V + 12 * F + 32 * F + 8 * F + 16 * V + 32 * nnzb
    b_hvp = 16 * V + 16 * V + 12 * F + 32 * F + 8 * F + 16 * V
    ex = {"V": V, "F": F, "nnzb": nnzb, "setup_s": st, "row_order": mesh.row_order_used()[0],
          "bytes_note": "16V uv + 12F faces + 32F rest_inv + 8F areas + 16V grad + 32 nnzb H (HVP: + 16V v, y for grad/H)"}
    pre = f"dirichlet_ico{sub}"
    out[pre + "_grad_hess"] = call_record(p, lambda: p.eval_terms(sync=False), F, "faces", b_hess,
                                          "k_rows_dirichlet<HESS>", peak, peak_kind, extra=ex, workload=f"ico{sub}")
    out[pre + "_grad_hess_psd"] = call_record(p, lambda: p.eval_terms(psd_floor=FLOOR, sync=False), F, "faces",
                                              b_hess, "k_cta_dirichlet<HESS,psd>", peak, peak_kind, workload=f"ico{sub}")
    out[pre + "_hvp"] = call_record(p, lambda: p.hvp(p.x_device, vd, out=y), F, "faces", b_hvp,
                                    "k_cta_dirichlet<HVP>", peak, peak_kind, workload=f"ico{sub}")
    out[pre + "_hvp_psd"] = call_record(p, lambda: p.hvp(p.x_device, vd, psd_floor=FLOOR, out=y), F, "faces", b_hvp,
                                        "k_cta_dirichlet<HVP,psd>", peak, peak_kind, workload=f"ico{sub}")
    del p, vd, y, mesh
    gc_cuda()
    # config 4: sphere manifold HVP (and its gradient), smoothing HVP (and gradient)
    t0 = time.perf_counter()
    pos, faces = mg.icosphere_arrays(sub)
    mesh = mg.Mesh(pos, faces)
    base = initial_sphere(mesh)
    b1, b2 = tangent_bases(base)
    p = sphere_problem(mesh, dev(base), dev(b1), dev(b2))
    V, F = len(pos), len(faces)
    p.x = 1e-5 * np.random.default_rng(0).normal(size=2 * V)  # tangent noise below the 1.1e-3 edge (no flips)
    st = time.perf_counter() - t0
    vd = dev(np.random.default_rng(1).normal(size=2 * V))
    y = torch.empty_like(vd)
    b_grad = 16 * V + 72 * V + 12 * F + 16 * V
    b_hvp = 16 * V + 16 * V + 72 * V + 12 * F + 16 * V
    ex = {"V": V, "F": F, "setup_s": st, "bytes_note": "16V x + 72V base/b1/b2 + 12F faces + 16V out (HVP: + 16V v)"}
    pre = f"sphere_ico{sub}"
    out[pre + "_grad"] = call_record(p, lambda: p.eval_terms(sync=False), F, "faces", b_grad,
                                     "k_rows_sphere<GRAD>", peak, peak_kind, extra=ex, workload=f"ico{sub}")
    out[pre + "_hvp"] = call_record(p, lambda: p.hvp(p.x_device, vd, out=y), F, "faces", b_hvp,
                                    "k_rows_sphere<HVP>", peak, peak_kind, workload=f"ico{sub}")
    out[pre + "_hvp_psd"] = call_record(p, lambda: p.hvp(p.x_device, vd, psd_floor=FLOOR, out=y), F, "faces", b_hvp,
                                        "k_sphere_face_hvp_psd", peak, peak_kind, workload=f"ico{sub}")
    del p, vd, y
    gc_cuda()
    p = edge_length_problem(mesh)
    p.x = pos.ravel()
    E = 3 * F // 2
    vd = dev(np.random.default_rng(1).normal(size=3 * V))
    y = torch.empty_like(vd)
    pre = f"smooth_ico{sub}"
    out[pre + "_grad"] = call_record(p, lambda: p.eval_terms(sync=False), E, "edges", 24 * V + 8 * E + 24 * V,
                                     "k_rows_fast<3,GRAD,EDGE_LENGTH>", peak, peak_kind,
                                     extra={"bytes_note": "24V x + 8E edge ids + 24V grad"}, workload=f"ico{sub}")
    out[pre + "_hvp"] = call_record(p, lambda: p.hvp(p.x_device, vd, out=y), E, "edges", 24 * V + 8 * E + 24 * V,
                                    "k_rows_fast<3,HVP,EDGE_LENGTH>", peak, peak_kind,
                                    extra={"bytes_note": "24V v + 8E edge ids + 24V y (the Hessian is constant)"}, workload=f"ico{sub}")
    del p, vd, y, mesh
    gc_cuda()
    return out


def run_config5(peak, peak_kind, n=7072):
    """BASELINE config 5 at N=1: cloth on generate_grid(7072) (50.0M vertices,
    150M edges, 100M faces), gradient-mode problem: eval_terms (energy +
    gradient) and the Newton-CG HVP, plain and clamped. Inputs are built on
    the device (lumped masses and rest lengths from the device mesh)."""
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import default_pins
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    t0 = time.perf_counter()
    pos, faces = mg.grid_arrays(n, 1.0 / (n - 1))
    mesh = mg.Mesh(pos, faces)
    mesh.to_device()
    pos_d = torch.from_numpy(pos).cuda()
    f_d = torch.from_numpy(faces).cuda()
    del faces
    cr = torch.linalg.cross(pos_d[f_d[:, 1]] - pos_d[f_d[:, 0]], pos_d[f_d[:, 2]] - pos_d[f_d[:, 0]])
    area3 = (0.5 * torch.linalg.vector_norm(cr, dim=1) / 3.0).repeat_interleave(3)
    del cr
    masses = torch.zeros(len(pos), dtype=torch.float64, device="cuda").index_add_(0, f_d.reshape(-1), area3)
    del area3, f_d
    e_d = mesh._edges_device
    dd = pos_d[e_d[:, 1]] - pos_d[e_d[:, 0]]
    l2 = (dd * dd).sum(dim=1)
    del dd
    gen = torch.Generator(device="cuda").manual_seed(0)
    sig = 0.01 / (n - 1)
    target = (pos_d + sig * torch.randn(pos_d.shape, generator=gen, device="cuda", dtype=torch.float64)).contiguous()
    x = (pos_d + sig * torch.randn(pos_d.shape, generator=gen, device="cuda", dtype=torch.float64)).reshape(-1)
    vd = torch.randn(x.numel(), generator=gen, device="cuda", dtype=torch.float64)
    h = 0.01
    p = mg.Problem(mesh, 3, with_hessian=False, fixed_vertices=default_pins(n))
    p.add_term(mg.Element.VERTEX, mg.Op.V, Inertia(masses, target))
    p.add_term(mg.Element.EDGE, mg.Op.EV, Spring(l2, 0.5 * 1e4 * h * h))
    p.add_term(mg.Element.VERTEX, mg.Op.V, Gravity(masses, np.array([0.0, -9.8, 0.0]), h * h))
    p.x = x
    del pos_d
    torch.cuda.synchronize()
    st = time.perf_counter() - t0
    V, E = cloth_sizes(n)
    y = torch.empty_like(vd)
    te = 2 * V + E
    ex = {"V": V, "E": E, "F": 2 * (n - 1) ** 2, "setup_s": st, "problem": "gradient mode (with_hessian=False)",
          "inputs": "device-built (torch seeded generator); masses / rest lengths from the device mesh",
          "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
    out = {
        "cloth7072_grad": call_record(p, lambda: p.eval_terms(sync=False), te, "term_elements",
                                      cloth_energy_bytes(V, E) + 24 * V, "k_rows_fast<3,GRAD,SPRING>", peak,
                                      peak_kind, extra=ex, workload="grid7072"),
        "cloth7072_hvp": call_record(p, lambda: p.hvp(p.x_device, vd, out=y), te, "term_elements",
                                     cloth_hvp_bytes(V, E), "k_rows_fast<3,HVP,SPRING>", peak, peak_kind, workload="grid7072"),
        "cloth7072_hvp_psd": call_record(p, lambda: p.hvp(p.x_device, vd, psd_floor=FLOOR, out=y), te,
                                         "term_elements", cloth_hvp_bytes(V, E), "k_rows_fast<3,HVP,psd,SPRING>",
                                         peak, peak_kind, workload="grid7072"),
    }
    del p, vd, y, x, target, masses, l2, mesh
    gc_cuda()
    return out


def run_config5_dist(world, rank, dist, n=7072, steps=10):
    """Config 5 on `world` ranks: the same 7072^2 cloth (gradient mode),
    vertex-partitioned (device-built shard plans), interior rows assembled
    while the ribbon exchange is in flight (DistributedProblem overlap);
    strong scaling: the whole-job rate over the max-over-ranks device time."""
    import torch

    import paper_2509_00406_b200 as mg
    from paper_2509_00406_b200.apps import default_pins
    from paper_2509_00406_b200.distributed import DistributedProblem
    from paper_2509_00406_b200.terms import Gravity, Inertia, Spring

    t0 = time.perf_counter()
    pos, faces = mg.grid_arrays(n, 1.0 / (n - 1))
    pos_d = torch.from_numpy(pos).cuda()
    f_d = torch.from_numpy(faces).cuda()
    cr = torch.linalg.cross(pos_d[f_d[:, 1]] - pos_d[f_d[:, 0]], pos_d[f_d[:, 2]] - pos_d[f_d[:, 0]])
    area3 = (0.5 * torch.linalg.vector_norm(cr, dim=1) / 3.0).repeat_interleave(3)
    del cr
    masses = torch.zeros(len(pos), dtype=torch.float64, device="cuda").index_add_(0, f_d.reshape(-1), area3)
    del area3
    sides = torch.cat([f_d[:, [0, 1]], f_d[:, [1, 2]], f_d[:, [2, 0]]])
    keys = torch.unique(sides.min(dim=1).values * len(pos) + sides.max(dim=1).values)
    del sides, f_d
    e0, e1 = keys // len(pos), keys % len(pos)
    dd = pos_d[e1] - pos_d[e0]
    l2 = (dd * dd).sum(dim=1)
    del dd, keys, e0, e1
    gen = torch.Generator(device="cuda").manual_seed(0)
    sig = 0.01 / (n - 1)
    target = (pos_d + sig * torch.randn(pos_d.shape, generator=gen, device="cuda", dtype=torch.float64)).contiguous()
    x = (pos_d + sig * torch.randn(pos_d.shape, generator=gen, device="cuda", dtype=torch.float64)).reshape(-1)
    v = torch.randn(x.numel(), generator=gen, device="cuda", dtype=torch.float64)
    h = 0.01
    terms = [("V", Inertia(masses, target)), ("EV", Spring(l2, 0.5 * 1e4 * h * h)),
             ("V", Gravity(masses, np.array([0.0, -9.8, 0.0]), h * h))]
    # id-range partition: horizontal stripes of the row-major grid (two ribbon
    # rows per cut); owned rows are contiguous slices, so the direction is
    # written straight into the shard's buffer and the result read as a view
    dp = DistributedProblem(pos, faces, 3, terms, fixed_vertices=default_pins(n), with_hessian=False, overlap=True,
                            partition="range")
    dp.set_x_global(x.cpu().numpy())
    own = torch.as_tensor(dp.plan.owned_global, device="cuda")
    v_own = dp.v_owned_buffer()
    v_own.copy_(v.view(-1, 3).index_select(0, own))
    del pos_d, x, v, target, masses, l2
    gc_cuda()
    st = time.perf_counter() - t0
    V, E = cloth_sizes(n)
    te = 2 * V + E
    out = {"setup_s": st, "owned_rows": len(dp.plan.owned_global), "interior_rows": dp.interior_rows,
           "boundary_rows": dp.boundary_rows, "halo_bytes_per_exchange": dp.halo.bytes_per_call,
           "scaling": f"strong (one {n}^2 mesh over all ranks)", "partition": "global id ranges (grid stripes)",
           "host_max_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20}
    ms, _ = time_device(lambda: dp.eval_terms(sync=False), steps, 3, dist)
    out["grad"] = {"ms": ms, "term_elements_per_s": te / (ms * 1e-3)}
    ms, _ = time_device(lambda: dp.hvp_owned(v_own), steps, 3, dist)
    out["hvp"] = {"ms": ms, "term_elements_per_s": te / (ms * 1e-3)}
    del dp
    gc_cuda()
    return {f"cloth{n}_strong": out}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_engine(args)


if __name__ == "__main__":
    main()
