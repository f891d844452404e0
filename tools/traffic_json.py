#!/usr/bin/env python
"""From an ncu --set full report, write profiles/traffic.json: per pass (X1..X3) the mean
dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes), plus per-kernel detail.
bench.py puts the dominant pass's value into roofline.traffic."""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
PASS = {"k_x1": "X1", "k_x1s": "X1", "k_y1": "Y1", "k_x2": "X2", "k_y2": "Y2", "k_x3": "X3", "k_x3s": "X3", "k_ref": "ref"}


def main(rep, out, workload="cfg3", batch=8):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units = rows[0], rows[1]
    c = {n: i for i, n in enumerate(head)}
    acc = defaultdict(list)
    for r in rows[2:]:
        name = r[c["Kernel Name"]]
        base = re.sub(r"^void ", "", name).split("<")[0].split("(")[0]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[c[m]]) * UNIT.get(units[c[m]], 1)
        acc[PASS.get(base, base)].append(b)
    res = {k: sum(v) / len(v) for k, v in acc.items()}
    res["_launches"] = {k: len(v) for k, v in acc.items()}
    res["_source"] = rep
    res["_workload"] = workload  # bench.py uses these per-launch bytes only for the same workload
    res["_angle_batch"] = int(batch)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json",
         sys.argv[3] if len(sys.argv) > 3 else "cfg3", sys.argv[4] if len(sys.argv) > 4 else 8)
