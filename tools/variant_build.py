"""A/B builds of libppo_b200.so: recompile ONE translation unit with extra nvcc flags
(e.g. -DPPO_FWD_POLY=2) and link it with the in-tree objects of the others into
abtest/<name>/libppo_b200.so (git-ignored, travels to the GPU box).  Load a variant with
PPO_LIB_PATH=abtest/<name>/libppo_b200.so.

    python tools/variant_build.py NAME SOURCE.cu [-DFOO=1 ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_01328_b200 import build_native as bn  # noqa: E402


def main():
    name, src, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
    bn.build(verbose=False)  # the in-tree objects of every other unit
    out = os.path.join(ROOT, "abtest", name)
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, src.replace(".cu", ".o"))
    subprocess.run([bn.nvcc_path(), *bn._flags(src), *extra, "-c", os.path.join(bn.CSRC, src), "-o", obj], check=True)
    objs = [obj if s == src else os.path.join(bn.OBJ, s.replace(".cu", ".o")) for s in bn.SOURCES]
    cmd = [bn.nvcc_path(), *bn.ARCH, "-shared", "-o", os.path.join(out, "libppo_b200.so"), *objs]
    nd = bn.nccl_dir()
    if nd:
        cmd += [f"-L{os.path.join(nd, 'lib')}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{os.path.join(nd, 'lib')}"]
    subprocess.run(cmd, check=True)
    print(os.path.join(out, "libppo_b200.so"))


if __name__ == "__main__":
    main()
