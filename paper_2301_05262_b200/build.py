"""Build the in-tree C-ABI library ``libnsm.so`` with nvcc for sm_100a.

The library is compiled in-tree (``paper_2301_05262_b200/libnsm.so``) so it
travels to the GPU box with the repo snapshot; nothing is JIT-compiled into
``~/.cache``. Sources are recompiled only when a source/header is newer than
the object.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnsm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# Experiment builds (-DNSM_EXPERIMENTS: the NSM_* attribution / tracing
# switches of tools/) go to their own object directory; the library they link
# reports it through nsm_build_flags() and bench.py refuses to time it.
EXPERIMENTS = os.environ.get("NSM_BUILD_EXPERIMENTS", "0") == "1"
if EXPERIMENTS:
    BUILD = os.path.join(HERE, "_build_exp")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--use_fast_math",
         "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "nsm.h")]


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src] + _headers())


def _compile(src):
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    path = os.path.join(CSRC, src)
    if not _stale(obj, path):
        return obj, ""
    # fast-math only where it is harmless: the parity kernels keep IEEE
    # division/sqrt (features.cu, net_f32.cu, producer.cu, abi.cu)
    flags = [f for f in FLAGS if f != "--use_fast_math"] if src in (
        "features.cu", "net_f32.cu", "producer.cu", "abi.cu", "temporal.cu", "feat5.cu") else FLAGS
    if EXPERIMENTS:
        flags = flags + ["-DNSM_EXPERIMENTS"]
    cmd = [NVCC, *ARCH, *flags, "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(f"--- {os.path.basename(o)}\n{log}")
    # relink whenever the objects are newer or the library came from the
    # other build flavour
    stamp = LIB + ".flavour"
    flavour = "experiments" if EXPERIMENTS else "release"
    same = os.path.exists(stamp) and open(stamp).read() == flavour
    if not same or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        with open(stamp, "w") as f:
            f.write(flavour)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
