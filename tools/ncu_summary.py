"""Summarise an ncu report: key throughput/occupancy metrics, DRAM bytes, stall mix, hottest source lines."""
import csv
import subprocess
import sys

FP64_PEAK = 34.116e12  # tools/fp64_peak on this pool's B200 (profiles/fp64_peak.json)


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, top=25):
    det = list(csv.reader(ncu(rep, "--page", "details", "--csv").splitlines()))
    keys = ("Duration", "DRAM Throughput", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
            "Executed Ipc Active", "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem",
            "Compute (SM) Throughput", "L1/TEX Hit Rate", "L2 Hit Rate")
    hdr = det[0]
    iname, iunit, ival = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    name = det[1][hdr.index("Kernel Name")] if len(det) > 1 else "?"
    print("kernel:", name[:120])
    seen = set()
    for r in det[1:]:
        if len(r) > ival and r[iname] in keys and r[iname] not in seen:
            seen.add(r[iname])
            print(f"  {r[iname]}: {r[ival]} {r[iunit]}")
    raw = list(csv.reader(ncu(rep, "--page", "raw", "--csv").splitlines()))
    h, u, v = raw[0], raw[1], raw[2]
    for i, x in enumerate(h):
        if x in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "gpu__time_duration.sum"):
            print(f"  {x}: {v[i]} {u[i]}")
    fp = {}
    for i, x in enumerate(h):
        for op in ("dadd", "dmul", "dfma"):
            if x == f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum":
                fp[op] = float(v[i].replace(",", ""))
        if x == "gpu__time_duration.sum":
            scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
            dur = float(v[i].replace(",", "")) * scale.get(u[i], 1e-3)
    if len(fp) == 3:
        flops = fp["dadd"] + fp["dmul"] + 2 * fp["dfma"]
        print(f"  fp64 executed flops (dadd+dmul+2 dfma): {flops:.4g}; at the kernel's duration "
              f"{flops / dur / 1e12:.2f} TFLOP/s = {flops / dur / FP64_PEAK:.3f} of the measured {FP64_PEAK / 1e12:.1f} TFLOP/s")
    st = []
    for i, x in enumerate(h):
        if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
            try:
                st.append((float(v[i].replace(",", "")), x.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(a for a, _ in st) or 1
    st.sort(reverse=True)
    print("  stalls:", ", ".join(f"{n} {100 * a / tot:.0f}%" for a, n in st[:8]))
    rows = list(csv.reader(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass").splitlines()))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] not in ("", "Function Name") and len(r) >= 5:
            try:
                s = int(r[4])
            except ValueError:
                continue
            k = (cur, int(r[0]), r[1][:90])
            agg[k] = agg.get(k, 0) + s
    tot = sum(agg.values()) or 1
    print("  hottest source lines (share of stall samples):")
    for k, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"   {100 * s / tot:5.1f}% {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
