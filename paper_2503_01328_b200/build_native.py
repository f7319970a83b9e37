"""Build ``libppo_b200.so`` in-tree with nvcc for sm_100a (no JIT cache, no torch types).

The shared library travels to the GPU box with the repo snapshot; the product
path loads it with ``ctypes`` (``runtime.native``) and fails loudly if it is
missing -- there is no CPU fallback.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libppo_b200.so")
SOURCES = ["ppo_runtime.cu", "ppo_kernels.cu", "ppo_layernorm.cu", "ppo_comm.cu", "ppo_gemm.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (need CUDA 12.9 for sm_100a)")


def nccl_dir() -> str | None:
    try:
        import nvidia.nccl  # type: ignore

        base = list(nvidia.nccl.__path__)[0]
    except Exception:
        return None
    if os.path.exists(os.path.join(base, "include", "nccl.h")) and os.path.exists(os.path.join(base, "lib", "libnccl.so.2")):
        return base
    return None


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    built = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "ppo_b200.h")]
    return any(os.path.getmtime(p) > built for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not _stale():
        return LIB
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
           "-Xptxas", "-v" if os.environ.get("PPO_PTXAS_VERBOSE") else "-O3",
           f"-I{os.path.join(ROOT, 'include')}", "-o", LIB + ".tmp"]
    nd = nccl_dir()
    if nd:
        cmd += ["-DPPO_WITH_NCCL", f"-I{os.path.join(nd, 'include')}", f"-L{os.path.join(nd, 'lib')}",
                "-l:libnccl.so.2", "-Xlinker", f"-rpath,{os.path.join(nd, 'lib')}"]
    cmd += [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if verbose:
        print("[build] " + " ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr.strip():
        print(res.stderr if os.environ.get("PPO_PTXAS_VERBOSE") else res.stderr[-4000:], file=sys.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(LIB)
