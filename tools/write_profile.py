"""Write profiles/<name>.md from one tools/round_gpu.sh pass (bench line, configs,
launch list, ncu summaries) and refresh profiles/ncu_traffic.json.
usage: python tools/write_profile.py <tag> <name>"""
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"


def summary(rep, top):
    return subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep), str(top)],
                          capture_output=True, text=True).stdout.strip()


def main(tag, name):
    d = json.loads((OUT / f"bench_{tag}.json").read_text().strip().splitlines()[-1])
    cfg = [json.loads(l) for l in (OUT / f"configs_{tag}.jsonl").read_text().splitlines() if l.startswith("{")]
    s1, s2, s3 = (summary(OUT / f"prof_{p}{tag}.ncu-rep", n) for p, n in (("", 25), ("hvp_", 15), ("dir_", 15)))
    rd = float(re.search(r"dram__bytes_read.sum: ([\d.]+) Mbyte", s1).group(1)) * 1e6
    wr = re.search(r"dram__bytes_write.sum: ([\d.]+) (\w+)", s1)
    traffic = int(round(rd + float(wr.group(1)) * (1e9 if wr.group(2) == "Gbyte" else 1e6)))
    (ROOT / "profiles" / "ncu_traffic.json").write_text(json.dumps(
        {"k_rows_fast<3,HESS,psd,SPRING>": traffic,
         "_source": f"profiles/{name}.md: ncu --set full, bench.py --profile (cloth 2048^2, psd), "
                    "dram__bytes_read.sum + dram__bytes_write.sum"}, indent=1))
    d["roofline"]["traffic"] = traffic
    ll = subprocess.run([sys.executable, str(ROOT / "tools" / "launch_summary.py"), str(OUT / f"launches_{tag}.csv"),
                         "k_rows_fast"], capture_output=True, text=True).stdout.strip()
    o = ["# Round 1 (final pass): bench line, BASELINE configs, launch list, ncu captures\n",
         f"All numbers from one `gpurun` pass (`bash tools/round_gpu.sh {tag}`), one B200, SM clocks at max with no "
         "throttle reasons during the timed region. Device times by CUDA events; ncu numbers are per-launch, "
         "cold-cache, serialised (only a kernel's SHARE of a step is comparable). `traffic` is this capture's dram "
         "read + write of the headline kernel.\n",
         "## bench.py (default: cloth 2048^2 Newton step, eval_terms(psd_floor=1e-9))\n```",
         json.dumps({k: d[k] for k in ("metric", "value", "unit", "ms_per_step", "roofline", "cpu_baseline", "e2e",
                                       "gpu_launches", "clocks")}, indent=1),
         "```\n\nextras (same run; hbm_frac = algorithmic bytes / kernel time / 6556 GB/s):\n",
         "| call | step ms | kernel ms | HBM frac |\n|---|---|---|---|"]
    for k, v in d["extras"].items():
        km = v.get("kernel_ms")
        o.append(f"| {k} | {v['ms']:.4f} | {km and round(km, 4)} | {v['hbm_frac']:.3f} |")
    o += ["\n## tools/bench_configs.py --sub 10 (icosphere(10): F = 20.97M)\n",
          "| config | call | ms | kernel ms | rate | HBM frac |\n|---|---|---|---|---|---|"]
    for c in cfg:
        rate = c.get("faces_per_s") or c.get("edges_per_s")
        unit = "faces/s" if "faces_per_s" in c else "edges/s"
        km = c.get("kernel_ms")
        o.append(f"| {c['config']} | {c['call']} | {c['ms']:.3f} | {km and round(km, 3)} | {rate:.3g} {unit} | "
                 f"{c['hbm_frac']:.3f} |")
    o += ["\n## launch list of the timed steps (ncu --metrics gpu__time_duration.sum --clock-control none, "
          "bench.py --profile)\n```", ll, "```\n\n## ncu --set full: headline kernel (edge row kernel, Hessian + PSD)\n```",
          s1, "```\n\n## ncu --set full: cloth HVP (staged edge tiles)\n```", s2,
          "```\n\n## ncu --set full: symmetric Dirichlet row kernel (icosphere(8))\n```", s3, "```\n"]
    (ROOT / "profiles" / f"{name}.md").write_text("\n".join(o))
    print(traffic)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
