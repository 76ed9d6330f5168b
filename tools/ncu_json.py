"""Collect per-launch ncu facts (DRAM bytes, executed FP64 flops, DRAM% and
FP64-pipe%, duration) from tools/ncu_summary.py outputs into
profiles/ncu_kernels.json, keyed by the labels bench.py reports.

usage: python tools/ncu_json.py <summary.txt> [...]   (merges into the json)
"""
import json
import re
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent.parent / "profiles" / "ncu_kernels.json"
MODES = {"1": "GRAD", "2": "HESS", "3": "HVP"}
EVT = {"2": "SPRING", "4": "EDGE_LENGTH", "0": "ANY"}


def label_of(kernel):
    m = re.search(r"k_rows_fast<(\d), (\d), (\d), (\d)(?:, (double|float))?>", kernel)
    if m:
        n, mode, psd, evt, st = m.groups()
        return (f"k_rows_fast<{n},{MODES[mode]}{',psd' if psd == '1' else ''},{EVT[evt]}"
                f"{',fp32' if st == 'float' else ''}>")
    m = re.search(r"k_rows_dirichlet<(\d), (\d), (\d)>", kernel)
    if m:
        mode, psd, _ = m.groups()
        return f"k_rows_dirichlet<{MODES[mode]}{',psd' if psd == '1' else ''}>"
    m = re.search(r"k_cta_dirichlet<(\d), (\d), (\d)>", kernel)
    if m:
        mode, psd, _ = m.groups()
        return f"k_cta_dirichlet<{MODES[mode]}{',psd' if psd == '1' else ''}>"
    m = re.search(r"k_rows_sphere<(\d)>", kernel)
    if m:
        return f"k_rows_sphere<{MODES[m.group(1)]}>"
    for k in ("k_face_psd", "k_sphere_face_hvp_psd", "k_tile_ev"):
        if k in kernel:
            return k
    return kernel


def parse(path):
    txt = Path(path).read_text()
    kern = re.search(r"kernel: (.*)", txt).group(1)
    num = lambda pat: float(re.search(pat, txt).group(1).replace(",", "")) if re.search(pat, txt) else None
    rd = num(r"dram__bytes_read.sum: ([\d.,]+) Gbyte") or (num(r"dram__bytes_read.sum: ([\d.,]+) Mbyte") or 0) / 1e3
    wr = num(r"dram__bytes_write.sum: ([\d.,]+) Gbyte") or (num(r"dram__bytes_write.sum: ([\d.,]+) Mbyte") or 0) / 1e3
    flops = num(r"fp64 executed flops \(dadd\+dmul\+2 dfma\): ([\d.e+]+)")
    dur_us = num(r"gpu__time_duration.sum: ([\d.,]+) us")
    if dur_us is None:
        ms = num(r"gpu__time_duration.sum: ([\d.,]+) ms")
        dur_us = ms * 1e3 if ms is not None else None
    tag = re.search(r"== (\S+) \((.*)\)", txt)
    cmd = tag.group(2) if tag else ""
    g = re.search(r"--grid (\d+)", cmd)
    sub = re.search(r"--sub (\d+)", cmd)
    workload = f"grid{g.group(1)}" if g else (f"ico{sub.group(1)}" if sub else "grid2048")
    return label_of(kern), {
        "workload": workload,
        "traffic": int(round((rd + wr) * 1e9)), "dram_read": int(round(rd * 1e9)), "dram_write": int(round(wr * 1e9)),
        "fp64_flops": flops, "dram_pct": num(r"DRAM Throughput: ([\d.]+) %"),
        "fp64_pipe_pct": num(r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active: ([\d.]+) %"),
        "ncu_duration_us": dur_us, "registers": num(r"Registers Per Thread: (\d+)"),
        "occupancy_pct": num(r"Achieved Occupancy: ([\d.]+) %"),
        "source": f"{Path(path).name}" + (f" ({tag.group(2)})" if tag else ""),
    }


def composite(d, name, parts):
    ps = [d[p] for p in parts if p in d]
    if len(ps) != len(parts):
        return
    dur = sum(p["ncu_duration_us"] for p in ps)
    d[name] = {
        "traffic": sum(p["traffic"] for p in ps),
        "fp64_flops": sum(p["fp64_flops"] or 0 for p in ps) or None,
        "dram_pct": sum(p["dram_pct"] * p["ncu_duration_us"] for p in ps) / dur,
        "fp64_pipe_pct": sum(p["fp64_pipe_pct"] * p["ncu_duration_us"] for p in ps) / dur,
        "ncu_duration_us": dur, "source": " + ".join(p["source"] for p in ps),
    }


def main(paths):
    d = json.loads(OUT.read_text()) if OUT.exists() else {}
    d = {k: v for k, v in d.items() if isinstance(v, dict)}
    for p in paths:
        k, v = parse(p)
        d[k] = v
    composite(d, "k_face_psd + k_rows_dirichlet<HESS,psd>", ["k_face_psd", "k_rows_dirichlet<HESS,psd>"])
    composite(d, "k_face_psd + k_rows_dirichlet<HVP,psd>", ["k_face_psd", "k_rows_dirichlet<HVP,psd>"])
    OUT.write_text(json.dumps(dict(sorted(d.items())), indent=1) + "\n")
    print(json.dumps(d, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1:])
