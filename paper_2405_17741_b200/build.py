"""Build liblsw.so (the C-ABI library) in-tree with nvcc for sm_100a.

Every .cu under csrc/ is compiled in parallel with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_2405_17741_b200/liblsw.so`` (static cudart; NCCL is bound with dlopen at first use).  The oracle
is pure numpy and needs no build.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "liblsw.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _compile(src: str, verbose: bool, tuning: bool = False) -> str:
    obj = os.path.join(BUILD + ("_tuning" if tuning else ""), os.path.basename(src) + ".o")
    # the source, every header and every .cu (a conservative rebuild rule)
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".cu"))]
    inc = os.path.join(ROOT, "include")
    deps += [os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DLSW_TUNING"] if tuning else []), "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    return obj


def build(verbose: bool = False, tuning: bool = False) -> str:
    """tuning=True: the measurement build (-DLSW_TUNING: probe options that
    produce deliberately wrong results take effect), objects in build_tuning/,
    linked to the same liblsw.so -- for tuning scripts only; rebuild without
    it before tests or the bench."""
    bdir = BUILD + ("_tuning" if tuning else "")
    os.makedirs(bdir, exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, tuning), srcs))
    stamp = LIB + ".flavor"
    flavor = "tuning" if tuning else "release"
    same = os.path.exists(stamp) and open(stamp).read() == flavor
    if same and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(flavor)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, tuning="--tuning" in sys.argv))
