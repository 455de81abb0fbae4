"""In-tree build of libigs_b200.so (sm_100a) with plain nvcc.

Each translation unit under csrc/ is compiled to build/<name>.o and linked
into paper_1809_05471_b200/libigs_b200.so.  The library travels to the GPU
box with the repo snapshot; nothing is JIT-compiled at run time.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
BUILD = os.path.join(REPO, "build")
LIB_NAME = "libigs_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "--expt-relaxed-constexpr"]
# Per-file extra flags: the tabulation must round like the reference's
# Python float arithmetic, so no FMA contraction there.
EXTRA = {"tabulate.cu": ["-fmad=false"], "mmio.cpp": ["-Xcompiler", "-fopenmp"]}

SOURCES = [
    "common.cu",
    "tabulate.cu",
    "pattern.cu",
    "generic.cu",
    "capi.cu",
    "synth.cu",
    "apply3d.cu",
    "assemble3d.cu",
    "geometry.cu",
    "naive.cu",
    "sharded.cu",
    "mmio.cpp",
]


def _sources():
    out = []
    for name in SOURCES:
        path = os.path.join(CSRC, name)
        if os.path.exists(path):
            out.append(name)
    return out


def _headers_mtime():
    m = 0.0
    for d in (CSRC, os.path.join(REPO, "include")):
        for f in os.listdir(d):
            if f.endswith((".cuh", ".h")):
                m = max(m, os.path.getmtime(os.path.join(d, f)))
    return m


def _compile(name, hdr_mtime, verbose):
    src = os.path.join(CSRC, name)
    stem = os.path.splitext(name)[0]
    obj = os.path.join(BUILD, stem + ".o")
    log = os.path.join(BUILD, stem + ".ptxas.txt")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj, False
    cmd = [NVCC, *ARCH, *COMMON, *EXTRA.get(name, []), "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{res.stderr[-6000:]}")
    if verbose:
        print(f"[build] compiled {name}", file=sys.stderr)
    return obj, True


def build(verbose=False, force=False):
    """Compile every CUDA translation unit for sm_100a and link the library."""
    os.makedirs(BUILD, exist_ok=True)
    hdr = _headers_mtime()
    if force:
        hdr = float("inf")
    names = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(names))) as ex:
        results = list(ex.map(lambda n: _compile(n, hdr if not force else 1e300, verbose), names))
    objs = [r[0] for r in results]
    changed = any(r[1] for r in results)
    if changed or not os.path.exists(LIB_PATH) or force:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB_PATH, *objs, "-lcudart", "-lcuda", "-lgomp", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
        if verbose:
            print(f"[build] linked {LIB_PATH}", file=sys.stderr)
    return LIB_PATH


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
