#!/usr/bin/env python
"""Compile holo_plan.cu with -Xptxas -v and print registers / spills per kernel (demangled, short)."""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "paper_2407_20304_b200/csrc/holo_plan.cu"
filt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v",
                      "-c", src, "-o", "/tmp/_ptxas.o"], capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur).replace("void holo::", "").replace("holo::", "")
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k in sorted(rows):
    if filt in k:
        print(f"{k:40s} regs {rows[k].get('regs', '?'):>4}  spill {rows[k].get('spill', '?')}")
errs = [l for l in out.splitlines() if "error" in l]
print("\n".join(errs))
