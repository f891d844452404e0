#!/usr/bin/env python
"""Per-kernel warp-stall breakdown (pc sampling) from an ncu --set full report.
    python tools/ncu_stalls.py gpurun_out/X.ncu-rep"""
import csv
import io
import subprocess
import sys


def main(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ki = h.index("Kernel Name")
    cols = [i for i, c in enumerate(h) if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
    for r in rows[2:]:
        vals = []
        for i in cols:
            try:
                vals.append((float(r[i].replace(",", "")), h[i].replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1
        vals.sort(reverse=True)
        print(r[ki][:24], " ".join(f"{n}={100 * v / tot:.0f}%" for v, n in vals[:9]))


if __name__ == "__main__":
    main(sys.argv[1])
