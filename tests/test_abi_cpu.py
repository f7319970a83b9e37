"""The C ABI (include/ppo_b200.h) on a machine without a GPU: the library loads,
exports every declared entry point, the ctypes binding covers exactly the header,
the ABI version agrees, and argument errors come back as PPO_E* codes with a
message -- no compute call is made."""
import ctypes
import os
import re

import pytest

from paper_2503_01328_b200 import build_native
from paper_2503_01328_b200.runtime import native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ppo_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"^\s*(?:int|int64_t|const char\*|uint64_t|void\*)\s+(ppo_\w+)\s*\(", text, flags=re.M))


def macro(name):
    m = re.search(rf"#define {name} \(?(-?\d+)\)?", open(HEADER).read())
    return int(m.group(1))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(native.LIB_PATH):
        build_native.build()
    return ctypes.CDLL(native.LIB_PATH)


def test_header_declares_the_bound_entry_points():
    names = declared()
    assert len(names) >= 25
    assert names == set(native.SIGNATURES), (names ^ set(native.SIGNATURES))


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in sorted(declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_abi_version_and_binding_load(lib):
    lib.ppo_abi_version.restype = ctypes.c_int
    assert lib.ppo_abi_version() == macro("PPO_ABI_VERSION")
    assert native.load() is not None  # the ctypes binding accepts this library


def test_argument_errors_are_codes_not_crashes():
    lib = native.load()
    einval = macro("PPO_EINVAL")
    assert lib.ppo_pack(None, -1, None, None) == einval
    assert b"ppo_pack" in lib.ppo_last_error()
    assert lib.ppo_dropout(None, None, 7, ctypes.c_float(0.1), 0, 0, None, None) == einval
    assert lib.ppo_transfer(7, None, 0, None, None, None) == einval
    assert lib.ppo_embed_fwd(None, None, None, None, 4, 12, 10, None) == einval
    assert lib.ppo_pool_create(0, None) == einval
    assert lib.ppo_pool_destroy(None) == 0
    assert lib.ppo_pool_bytes(None) == 0


def test_product_path_refuses_to_run_without_cuda():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():  # pragma: no cover
        pytest.skip("a GPU is present")
    with pytest.raises(native.NativeUnavailable):
        native.require_cuda()


def test_row_kernels_do_not_spill(lib):
    """Resource usage of the built sm_100a cubins (cuobjdump -res-usage): the LayerNorm
    backward kernels, at every (warps per row, rows per CTA) the dispatch can pick, keep
    their double-buffered rows in registers -- a spill cost 4x at h = 5120
    (profiles/r1_ln_bwd_spill_fix.txt).  The forward kernels at the default 4 vectors
    per lane spill at most a word."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-res-usage", native.LIB_PATH], capture_output=True, text=True).stdout
    usage = dict(re.findall(r"Function (\S+):\s*\n\s*(REG:.*)", out))
    # the default dispatch (next-row prefetch): no spill without the LN recompute output,
    # at most two words with it (the ln_out kernels of the unsplit backward)
    bwd = {f: u for f, u in usage.items() if "ln_bwd_kernel" in f and re.search(r"ELb0ELb1EE", f)}
    assert len(bwd) >= 10
    for f, u in bwd.items():
        assert "STACK:0 " in u and "LOCAL:0 " in u, (f, u)
    bwd_ln = {f: u for f, u in usage.items() if "ln_bwd_kernel" in f and re.search(r"ELb1ELb1EE", f)}
    assert len(bwd_ln) >= 10
    for f, u in bwd_ln.items():
        assert int(re.search(r"STACK:(\d+)", u).group(1)) <= 8, (f, u)
    # default build of the forward kernels (kMinBlocks = 1; the PPO_LN_FWD_MINB=4 A/B variants may spill)
    fwd4 = {f: u for f, u in usage.items() if re.search(r"ln_fwd_kernelILb[01]ELi\d+ELi4ELi\d+ELb[01]ELi1EE", f)}
    assert fwd4
    for f, u in fwd4.items():
        assert int(re.search(r"STACK:(\d+)", u).group(1)) <= 8, (f, u)
