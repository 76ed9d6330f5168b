"""Per-kernel register / spill table from `nvcc -Xptxas -v` output.
usage: python tools/regs.py <file.cu> [filter]   (run from paper_2509_00406_b200/csrc)"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
extra = sys.argv[3:] 
cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-Xcompiler", "-fPIC",
       "--expt-relaxed-constexpr", "-Xptxas", "-v", *extra, "-c", src, "-o", "/dev/null"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur, spill = None, ""
for line in out.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = cur.replace("mg::(anonymous namespace)::", "")
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}" if m.group(1) != "0" or m.group(2) != "0" else ""
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if flt in cur:
            print(f"{m.group(1):>4} regs {spill:>14}  {cur[:140]}")
        cur = None
if " error" in out:
    print(out[-3000:])
