"""Build libholo.so (sm_100a) in-tree with nvcc.

The library is split into one translation unit per torus size (csrc/inst_<L>.cu, the
pass kernels instantiated for that L) plus the ABI unit (csrc/holo_plan.cu); they are
compiled in parallel to objects under build/ and linked into libholo.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libholo.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def units():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + \
        [os.path.join(HERE, "..", "include", "holo.h")]


def up_to_date(out=LIB) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=(), jobs=None) -> str:
    """Compile libholo.so; `defines` (e.g. ["-DHOLO_SINGLE_BUF=0"]) and `out` build tuning variants."""
    if not force and out == LIB and not defines and up_to_date():
        return LIB
    tag = "%s_%d" % (os.path.basename(out).replace(".so", ""), os.getpid())
    bdir = os.path.join(os.path.dirname(HERE), "build", tag)
    os.makedirs(bdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [NVCC] + CFLAGS + list(defines) + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        return obj

    srcs = units()
    # the largest units (big tori) first so the pool finishes together
    srcs.sort(key=lambda s: -int(os.path.basename(s)[5:-3]) if os.path.basename(s).startswith("inst_") else 0)
    with cf.ThreadPoolExecutor(max_workers=jobs or min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = out + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs)
    os.replace(tmp, out)
    for o in objs:
        os.remove(o)
    os.rmdir(bdir)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=LIB)
    a, defines = ap.parse_known_args()  # the rest: -DNAME=VALUE tuning knobs
    print(build(force=True, verbose=True, out=a.out, defines=defines))
