"""Build libholo.so (sm_100a) in-tree with nvcc."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libholo.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared"]


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + \
        [os.path.join(HERE, "..", "include", "holo.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile libholo.so; `defines` (e.g. ["-DHOLO_NT_ROWS=256"]) and `out` build tuning variants."""
    if not force and out == LIB and not defines and up_to_date():
        return LIB
    tmp = out + ".tmp%d" % os.getpid()
    cmd = [NVCC] + FLAGS + list(defines) + [os.path.join(CSRC, "holo_plan.cu"), "-o", tmp]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=LIB)
    a, defines = ap.parse_known_args()  # the rest: -DNAME=VALUE tuning knobs
    print(build(force=True, verbose=True, out=a.out, defines=defines))
