"""Build the sm_100a shared library paper_1310_3435_b200/_lib/libsddg.so.

Explicit nvcc, in-tree output (it travels to the GPU box with the repo
snapshot).  Translation units that must reproduce the reference's rounding
sequence (walk_ref.cu, solver.cu) are compiled with -fmad=false; the others
may contract to FMA.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
# SDDG_BUILD_TAG / SDDG_EXTRA_NVCC: side-by-side variant builds for A/B timing
_TAG = os.environ.get("SDDG_BUILD_TAG", "")
OBJ_DIR = os.path.join(OUT_DIR, "obj" + (("_" + _TAG) if _TAG else ""))
LIB = os.path.join(OUT_DIR, "libsddg" + (("_" + _TAG) if _TAG else "") + ".so")
EXTRA = os.environ.get("SDDG_EXTRA_NVCC", "").split()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "-I" + os.path.join(ROOT, "include")]
UNITS = {
    "walk_ref.cu": ["-fmad=false"],
    # fp32 walks: no denormal fix-ups around SFU ops.  SDDG_SMEM_ABS: the
    # fastmath tables' offset in the shared window (1 KB reserved, no static
    # shared memory; checked at kernel entry)
    "walk_fast.cu": ["-fmad=true", "-ftz=true", "-DSDDG_SMEM_ABS=0x400"],
    "reduce.cu": ["-fmad=false"],
    "solver.cu": ["-fmad=false"],
    "mesh.cu": ["-fmad=false"],
    "smooth.cu": ["-fmad=false"],
    "probe.cu": [],
    "runtime.cu": [],
    "team.cu": [],
}
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def _compile(unit, flags, verbose):
    src = os.path.join(CSRC, unit)
    obj = os.path.join(OBJ_DIR, unit.replace(".cu", ".o"))
    deps = [src, os.path.abspath(__file__)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(ROOT, "include", "sddg.h")]  # build.py itself: flag changes rebuild
    if _mtime(obj) >= max(_mtime(d) for d in deps):
        return obj, False
    cmd = [NVCC] + ARCH + COMMON + EXTRA + flags + ["-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {unit}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj, True


def build(verbose=False, force=False):
    os.makedirs(OBJ_DIR, exist_ok=True)
    if force:
        for f in os.listdir(OBJ_DIR):
            os.remove(os.path.join(OBJ_DIR, f))
    with cf.ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        results = list(ex.map(lambda kv: _compile(kv[0], kv[1], verbose), UNITS.items()))
    objs = [o for o, _ in results]
    if any(changed for _, changed in results) or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    if not _TAG:
        build_examples()
    return LIB


EXAMPLES = os.path.join(ROOT, "examples")
EXAMPLE_BIN = os.path.join(EXAMPLES, "_bin")


def build_examples():
    """Plain C callers of the C-ABI (examples/*.c), linked against the
    in-tree library with an rpath relative to the binary."""
    if not os.path.isdir(EXAMPLES):
        return
    os.makedirs(EXAMPLE_BIN, exist_ok=True)
    for src in sorted(f for f in os.listdir(EXAMPLES) if f.endswith(".c")):
        out = os.path.join(EXAMPLE_BIN, src[:-2])
        deps = [os.path.join(EXAMPLES, src), LIB, os.path.join(ROOT, "include", "sddg.h")]
        if _mtime(out) >= max(_mtime(d) for d in deps):
            continue
        cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
               os.path.join(EXAMPLES, src), "-o", out, "-L" + OUT_DIR, "-lsddg",
               "-Wl,-rpath,$ORIGIN/../../paper_1310_3435_b200/_lib"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"gcc failed for {src}:\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
