"""Build libsurge.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python paper_2605_01060_b200/build.py          # or __graft_entry__.build()

Objects go to paper_2605_01060_b200/_build/, the library to paper_2605_01060_b200/libsurge.so.
cudart is linked statically; the TMA encoder is resolved at run time through
cudaGetDriverEntryPoint, so the library loads on a machine without a GPU (the
"-m 'not gpu'" ABI test) and fails loudly at surge_create instead.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.environ.get("SURGE_BUILD_OUT") or os.path.join(PKG, "libsurge.so")   # variants: scripts/ experiments
BUILD = os.environ.get("SURGE_BUILD_DIR") or os.path.join(PKG, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall,-Wno-unused-function",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
FLAGS += os.environ.get("NVCC_EXTRA", "").split()   # tuning experiments (scripts/gpu_*_sweep.sh)


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "surge.h"))
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cc = nvcc()
    jobs = []
    objs = []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, src):
            cmd = [cc, *ARCH, *FLAGS, "-c", src, "-o", obj]
            if src.endswith(".cpp"):
                cmd = [cc, *FLAGS, "-x", "cu", *ARCH, "-c", src, "-o", obj]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if jobs or not os.path.exists(OUT) or force:
        run([cc, *ARCH, "-shared", "-o", OUT, *objs, "-lpthread", "-ldl",
             *os.environ.get("NVCC_LINK_EXTRA", "").split()])   # e.g. the TSAN runtime (scripts/sanitize.sh)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
