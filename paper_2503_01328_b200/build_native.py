"""Build ``libppo_b200.so`` in-tree with nvcc for sm_100a (no JIT cache, no torch types).

Each ``csrc/*.cu`` compiles to an object under ``build/`` (in parallel, re-built only
when the source or a header is newer), then one link step writes the shared library
next to this file.  The library travels to the GPU box with the repo snapshot; the
product path loads it with ``ctypes`` (``runtime.native``) and fails loudly if it is
missing -- there is no CPU fallback.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libppo_b200.so")
SOURCES = ["ppo_runtime.cu", "ppo_kernels.cu", "ppo_layernorm.cu", "ppo_comm.cu", "ppo_gemm_fwd.cu", "ppo_gemm_bwd.cu", "ppo_gemm_wgrad.cu",
           "ppo_attention.cu", "ppo_attention_bwd.cu", "ppo_attention_fwd.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (need CUDA 12.9 for sm_100a)")


def _site_dir(mod: str, rel: str) -> str | None:
    try:
        import importlib.util

        spec = importlib.util.find_spec(mod)
        for base in list(spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(base, rel)
            if os.path.exists(cand):
                return cand
    except Exception:
        pass
    return None


def nccl_dir() -> str | None:
    try:
        import nvidia.nccl  # type: ignore

        base = list(nvidia.nccl.__path__)[0]
    except Exception:
        return None
    if os.path.exists(os.path.join(base, "include", "nccl.h")) and os.path.exists(os.path.join(base, "lib", "libnccl.so.2")):
        return base
    return None


def cutlass_include() -> str | None:
    """CUTLASS/CuTe 4.x headers vendored in the image (flashinfer's copy, found
    without importing flashinfer)."""
    cand = os.environ.get("CUTLASS_INCLUDE") or _site_dir("flashinfer", os.path.join("data", "cutlass", "include"))
    if cand and os.path.exists(os.path.join(cand, "cutlass", "cutlass.h")):
        return cand
    return None


def fmha_include() -> str | None:
    """Blackwell FMHA collectives (CUTLASS example 77) vendored in flashinfer's header tree."""
    cand = os.environ.get("FMHA_INCLUDE") or _site_dir("flashinfer", os.path.join("data", "include"))
    if cand and os.path.exists(os.path.join(cand, "flashinfer", "attention", "blackwell", "device", "fmha.hpp")):
        return cand
    return None


def _flags(src: str) -> list[str]:
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", f"-I{os.path.join(ROOT, 'include')}"]
    flags += ["-Xptxas", "-v"] if os.environ.get("PPO_PTXAS_VERBOSE") else []
    nd = nccl_dir()
    if nd:
        flags += ["-DPPO_WITH_NCCL", f"-I{os.path.join(nd, 'include')}"]
    if src.startswith("ppo_gemm") or src == "ppo_attention.cu":
        inc = cutlass_include()
        if not inc:
            raise RuntimeError("CUTLASS headers not found (set CUTLASS_INCLUDE)")
        util = os.path.join(os.path.dirname(inc), "tools", "util", "include")
        # CUTLASS_ENABLE_GDC_FOR_SM100: the kernels' griddepcontrol.wait / launch_dependents
        # are compiled in, so they may be launched with programmatic dependent launch
        flags += [f"-I{inc}", f"-I{util}", "--expt-relaxed-constexpr", "-DNDEBUG", "-DCUTLASS_ENABLE_GDC_FOR_SM100=1"]
    if src == "ppo_attention.cu":
        fi = fmha_include()
        if not fi:
            raise RuntimeError("Blackwell FMHA headers not found (set FMHA_INCLUDE)")
        flags += [f"-I{os.path.join(fi, 'flashinfer', 'attention', 'blackwell')}", f"-I{fi}"]
    return flags


def _headers() -> list[str]:
    return glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "ppo_b200.h")]


def _compile(src: str, force: bool, verbose: bool) -> str:
    os.makedirs(OBJ, exist_ok=True)
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    if not force and os.path.exists(obj):
        newest = max(os.path.getmtime(p) for p in [path, __file__] + _headers())
        if os.path.getmtime(obj) >= newest:
            return obj
    cmd = [nvcc_path(), *_flags(src), "-c", path, "-o", obj + ".tmp"]
    if verbose:
        print("[build] " + " ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src} ({res.returncode}):\n{res.stdout}\n{res.stderr[-8000:]}")
    if verbose and res.stderr.strip():
        print(res.stderr if os.environ.get("PPO_PTXAS_VERBOSE") else res.stderr[-2000:], file=sys.stderr)
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        objs = list(pool.map(lambda s: _compile(s, force, verbose), SOURCES))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    cmd = [nvcc_path(), *ARCH, "-shared", "-o", LIB + ".tmp", *objs]
    nd = nccl_dir()
    if nd:
        cmd += [f"-L{os.path.join(nd, 'lib')}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{os.path.join(nd, 'lib')}"]
    if verbose:
        print("[build] " + " ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
