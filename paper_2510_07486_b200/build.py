"""In-tree build of the sm_100a libraries (nvcc cross-compiles without a GPU).

  libasyncspade.so  -- the product: the C ABI of include/asyncspade.h
  libasp_synth.so   -- seeded device input generator (bench/test support)

Both link the CUDA runtime statically, so the .so files that travel to the
GPU box with the repo snapshot are self-contained.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libasyncspade.so")
SYNTH_LIB = os.path.join(PKG, "libasp_synth.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]
PRODUCT_SOURCES = ["abi.cu", "append.cu", "predict.cu", "score.cu", "select.cu", "select_short.cu",
                   "decode.cu",
                   "score_cc.cu", "decode_cc.cu",
                   "quest.cu", "gather.cu"]
SYNTH_SOURCES = ["synth.cu"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, log: list) -> str:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")] + \
        [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)]
    if _stale(obj, deps):
        cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append((src, r.stderr))
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def _link(objs: list[str], out: str) -> None:
    if _stale(out, objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", out, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed for {out}:\n{r.stderr}")


def build(verbose: bool = False) -> list[str]:
    os.makedirs(BUILD, exist_ok=True)
    log: list = []
    srcs = [os.path.join(CSRC, f) for f in PRODUCT_SOURCES + SYNTH_SOURCES]
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, log), srcs))
    n = len(PRODUCT_SOURCES)
    _link(objs[:n], LIB)
    _link(objs[n:], SYNTH_LIB)
    if verbose:
        for src, err in log:
            print(f"== {os.path.basename(src)}\n{err}")
    return [LIB, SYNTH_LIB]


def build_profiling(defines: list[str], tag: str = "prof") -> str:
    """Instrumented variant (e.g. -DASP_PROFILE_SCORE) at build/<tag>/ -- dev only."""
    out_dir = os.path.join(BUILD, tag)
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "libasyncspade_prof.so")
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    if os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(f) for f in srcs):
        return out                                   # prebuilt (e.g. here, before a gpurun call)
    objs = []
    for f in PRODUCT_SOURCES:
        obj = os.path.join(out_dir, f + ".o")
        cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *defines, "-c", os.path.join(CSRC, f), "-o", obj]
        subprocess.run(cmd, check=True, capture_output=True)
        objs.append(obj)
    out = os.path.join(out_dir, "libasyncspade_prof.so")
    subprocess.run([_nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", out, *objs], check=True)
    return out


if __name__ == "__main__":
    import sys
    for p in build(verbose="-v" in sys.argv):
        print(p)
