#!/usr/bin/env python
"""Top stall hot spots (SASS) per kernel from an ncu report: groups stall samples by
instruction opcode class and lists the hottest instructions.
    python tools/ncu_hotspots.py gpurun_out/prof.ncu-rep [kernel-substring]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def main(rep, filt=""):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', txt)
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if filt not in name:
            continue
        rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
        h = rows[0]
        si, ni = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        tot = 0
        byop = Counter()
        hot = []
        for r in rows[1:]:
            if len(r) <= ni:
                continue
            try:
                n = int(r[ni])
            except ValueError:
                continue
            op = r[si].strip().split()[0] if r[si].strip() else "?"
            if op.startswith("@"):
                op = r[si].strip().split()[1]
            op = op.split(".")[0]
            byop[op] += n
            tot += n
            hot.append((n, r[si].strip()[:70]))
        print(f"== {name[:90]}  samples {tot}")
        print("   by opcode:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in byop.most_common(12)))
        for n, src in sorted(hot, reverse=True)[:12]:
            print(f"   {100*n/tot:5.2f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
