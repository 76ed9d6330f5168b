"""Per-source-line instruction counts and stall samples of an ncu report (needs -lineinfo).
usage: python tools/ncu_lines.py rep [top] [file-filter]"""
import csv
import subprocess
import sys


def main(rep, top=30, filt=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, rows = None, None, []
    for r in csv.reader(out.splitlines()):
        if len(r) >= 2 and r[0] in ("File Path", "File Name"):
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit() and len(r) == len(hdr) and r[2] == "-":
            try:
                ins = int(r[hdr.index("Instructions Executed")])
                smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            except ValueError:
                continue
            rows.append((ins, smp, cur, int(r[0]), r[1].strip()[:100]))
    ti = sum(x[0] for x in rows) or 1
    ts = sum(x[1] for x in rows) or 1
    print(f"total warp instructions {ti}")
    for ins, smp, f, ln, src in sorted(rows, key=lambda x: -x[0])[:top]:
        if filt in f:
            print(f"{100 * ins / ti:5.1f}% ins {100 * smp / ts:5.1f}% stall  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else "")
