"""ctypes binding of ``libppo_b200.so`` (ABI: ``include/ppo_b200.h``).

This is the only door from Python into the device code.  It loads the in-tree
library and raises ``NativeUnavailable`` when it is missing or the process has
no CUDA device -- the runtime has no CPU fallback.

Tensor-level helpers take torch tensors (device memory + the current stream are
PyTorch's; the library only sees raw pointers, sizes and stream handles).
"""

from __future__ import annotations

import collections
import ctypes
import os
import threading

PKG = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.environ.get("PPO_LIB_PATH") or os.path.join(PKG, "libppo_b200.so")  # override: A/B builds only

PPO_D2H, PPO_H2D = 0, 1
PPO_NCCL_BASE = 10000


class NativeUnavailable(RuntimeError):
    """libppo_b200.so (or a CUDA device) is not available: nothing to fall back to."""


class PpoError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed with code {code}: {msg}")
        self.code = code


class Segment(ctypes.Structure):
    _fields_ = [("dev", ctypes.c_void_p), ("host", ctypes.c_void_p), ("bytes", ctypes.c_uint64)]


class GatherItem(ctypes.Structure):
    _fields_ = [
        ("src", ctypes.c_void_p),
        ("dst_off", ctypes.c_uint64),
        ("rows", ctypes.c_uint64),
        ("row_bytes", ctypes.c_uint64),
        ("src_pitch", ctypes.c_uint64),
        ("dst_pitch", ctypes.c_uint64),
    ]


class P2POp(ctypes.Structure):
    _fields_ = [("is_send", ctypes.c_int), ("peer", ctypes.c_int), ("buf", ctypes.c_void_p), ("bytes", ctypes.c_uint64)]


_VP, _U64, _I64, _F32, _I32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_float, ctypes.c_int
ABI_VERSION = 9  # include/ppo_b200.h PPO_ABI_VERSION
_FP = ctypes.POINTER(ctypes.c_float)

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "ppo_abi_version": [],
    "ppo_last_error": [],
    "ppo_timestamp": [_VP, _VP],
    "ppo_stream_write_u32": [_VP, _VP, ctypes.c_uint32],
    "ppo_stream_wait_u32": [_VP, _VP, ctypes.c_uint32],
    "ppo_host_register": [_VP, _U64, ctypes.POINTER(_VP)],
    "ppo_host_unregister": [_VP],
    "ppo_gemm_set_swizzle": [_I32, _I64, _I64, _I64, _I32],
    "ppo_kernel_launches": [],
    "ppo_device_info": [_I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32)],
    "ppo_pool_create": [_U64, ctypes.POINTER(_VP)],
    "ppo_pool_create_numa": [_U64, _I32, _I32, ctypes.POINTER(_VP), ctypes.POINTER(_I32)],
    "ppo_pool_numa_node": [_VP],
    "ppo_pool_destroy": [_VP],
    "ppo_pool_base": [_VP],
    "ppo_pool_bytes": [_VP],
    "ppo_transfer": [_I32, ctypes.POINTER(Segment), _I32, _VP, _VP, _VP],
    "ppo_pack": [ctypes.POINTER(GatherItem), _I32, _VP, _VP],
    "ppo_layernorm_fwd": [_VP, _VP, _VP, _VP, _I64, _I64, _F32, _VP],
    "ppo_residual_dropout_ln_fwd": [_VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _F32, _F32, _U64, _U64, _VP, _VP],
    "ppo_layernorm_bwd": [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _F32, _VP, _F32, _U64, _U64, _VP, _VP, _VP,
                          _VP],
    "ppo_layernorm_fwd2": [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _F32, _VP],
    "ppo_dropout": [_VP, _VP, _I64, _F32, _U64, _U64, _VP, _VP],
    "ppo_gelu_fwd": [_VP, _VP, _I64, _VP],
    "ppo_gelu_bwd": [_VP, _VP, _VP, _VP, _I64, _VP],
    "ppo_colsum": [_VP, _VP, _I64, _I64, _VP],
    "ppo_embed_fwd": [_VP, _VP, _VP, _VP, _I64, _I64, _I64, _VP],
    "ppo_embed_bwd": [_VP, _VP, _VP, _VP, _I64, _I64, _I64, _VP],
    "ppo_gemm_tn": [_VP, _VP, _VP, _I64, _I64, _I64, _VP],
    "ppo_gemm_tn_gelu": [_VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _VP],
    "ppo_gemm_nn": [_VP, _VP, _VP, _I64, _I64, _I64, _F32, _VP],
    "ppo_gemm_nn_dgelu": [_VP, _VP, _VP, _VP, _I64, _I64, _I64, _VP],
    "ppo_gemm_wgrad": [_VP, _VP, _VP, _I64, _I64, _I64, _F32, _VP],
    "ppo_attn_fwd": [_VP, _VP, _VP, _I64, _I64, _I64, _F32, _VP],
    "ppo_attn_fwd_trace": [_VP],
    "ppo_attn_bwd_workspace_bytes": [_I64, _I64, _I64],
    "ppo_attn_bwd_trace": [_VP],
    "ppo_attn_bwd": [_VP, _VP, _VP, _VP, _VP, _VP, _I64, _I64, _I64, _F32, _VP],
    "ppo_comm_unique_id": [ctypes.POINTER(ctypes.c_uint8)],
    "ppo_comm_init": [ctypes.POINTER(ctypes.c_uint8), _I32, _I32, _I32, ctypes.POINTER(_VP)],
    "ppo_comm_destroy": [_VP],
    "ppo_p2p": [_VP, ctypes.POINTER(P2POp), _I32, _VP],
}
_RESTYPES = {
    "ppo_last_error": ctypes.c_char_p,
    "ppo_kernel_launches": ctypes.c_uint64,
    "ppo_pool_base": ctypes.c_void_p,
    "ppo_pool_bytes": ctypes.c_uint64,
    "ppo_attn_bwd_workspace_bytes": ctypes.c_int64,
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the library (no CUDA device needed to load; calls need one)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: run __graft_entry__.build() (nvcc, sm_100a); there is no CPU fallback"
            )
        lib = ctypes.CDLL(path)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        if lib.ppo_abi_version() != ABI_VERSION:
            raise NativeUnavailable("libppo_b200.so ABI version mismatch")
        _lib = lib
        return lib


def check(fn: str, rc: int) -> None:
    if rc != 0:
        msg = load().ppo_last_error()
        raise PpoError(fn, rc, msg.decode() if msg else "")


CALLS: collections.Counter = collections.Counter()  # ABI entry point -> calls (launch accounting)
SHAPES: collections.Counter = collections.Counter()  # (GEMM entry point, M, N, K) -> calls


def call(fn: str, *args) -> None:
    CALLS[fn] += 1
    check(fn, getattr(load(), fn)(*args))


def call_counts():
    """Snapshot of (CALLS, SHAPES), for crediting CUDA-graph replays (see credit)."""
    return collections.Counter(CALLS), collections.Counter(SHAPES)


def since(snap):
    """Calls made after ``snap`` (a call_counts() result)."""
    c, sh = snap
    return CALLS - c, SHAPES - sh


def credit(delta, sign: int = 1):
    """Add (sign=1) or remove (sign=-1) a block of calls: a graph capture records
    launches that do not execute; each replay executes them."""
    c, sh = delta
    for k, v in c.items():
        CALLS[k] += sign * v
    for k, v in sh.items():
        SHAPES[k] += sign * v


def kernel_launches() -> int:
    return int(load().ppo_kernel_launches())


# ---------------------------------------------------------------- torch helpers


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 runtime has no CPU fallback")
    load()
    return torch


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _check_bf16(*ts):
    import torch

    for t in ts:
        if t is not None and (t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous()):
            raise ValueError("expected a contiguous bf16 CUDA tensor")


def layernorm_fwd(x, gamma, beta, y, eps=1e-5, stream=None):
    _check_bf16(x, y)
    h = x.shape[-1]
    call("ppo_layernorm_fwd", _ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), x.numel() // h, h, eps, _stream(stream))


def residual_dropout_ln_fwd(resid, branch, out, gamma, beta, ln, p, seed, offset, eps=1e-5, stream=None,
                            offset_base=None):
    """offset_base: optional 1-element uint64/int64 device tensor added to ``offset``."""
    _check_bf16(resid, branch, out, ln)
    h = resid.shape[-1]
    call(
        "ppo_residual_dropout_ln_fwd", _ptr(resid), _ptr(branch), _ptr(out), _ptr(gamma), _ptr(beta), _ptr(ln),
        resid.numel() // h, h, eps, p, seed, offset, _ptr(offset_base), _stream(stream),
    )


def layernorm_bwd(x, gamma, dy, resid_grad, dx, dgamma, dbeta, drop_out=None, p=0.0, drop_seed=0,
                  drop_offset=0, eps=1e-5, stream=None, offset_base=None, beta=None, ln_out=None):
    """dx = resid_grad + LN_bwd(dy; x); dgamma/dbeta += ...; drop_out = dropout_bwd(dx);
    ln_out = LN(x)*gamma + beta (the recompute, when given)."""
    _check_bf16(x, dy, resid_grad, dx, drop_out, ln_out)
    h = x.shape[-1]
    call(
        "ppo_layernorm_bwd", _ptr(x), _ptr(gamma), _ptr(dy), _ptr(resid_grad), _ptr(dx), _ptr(dgamma),
        _ptr(dbeta), x.numel() // h, h, eps, _ptr(drop_out), p, drop_seed, drop_offset, _ptr(offset_base),
        _ptr(beta), _ptr(ln_out), _stream(stream),
    )


def layernorm_fwd2(x_a, gamma_a, beta_a, y_a, x_b, gamma_b, beta_b, y_b, eps=1e-5, stream=None):
    """Two LayerNorms of equal shape in one launch (W-pass LN1 + LN2 recompute)."""
    _check_bf16(x_a, y_a, x_b, y_b)
    h = x_a.shape[-1]
    if x_b.shape != x_a.shape:
        raise ValueError("layernorm_fwd2: both inputs must have one shape")
    call("ppo_layernorm_fwd2", _ptr(x_a), _ptr(gamma_a), _ptr(beta_a), _ptr(y_a), _ptr(x_b), _ptr(gamma_b),
         _ptr(beta_b), _ptr(y_b), x_a.numel() // h, h, eps, _stream(stream))


def dropout(x, y, p, seed, offset, stream=None, offset_base=None):
    _check_bf16(x, y)
    call("ppo_dropout", _ptr(x), _ptr(y), x.numel(), p, seed, offset, _ptr(offset_base), _stream(stream))


def gelu_fwd(f, g, stream=None):
    _check_bf16(f, g)
    call("ppo_gelu_fwd", _ptr(f), _ptr(g), f.numel(), _stream(stream))


def gelu_bwd(f, dg, g, df, stream=None):
    _check_bf16(f, dg, g, df)
    call("ppo_gelu_bwd", _ptr(f), _ptr(dg), _ptr(g), _ptr(df), f.numel(), _stream(stream))


def gemm_tn(a, b, d, stream=None):
    """d[M,N] = a[M,K] @ b[N,K]^T on tcgen05 (bf16 in/out, fp32 accumulation in TMEM)."""
    _check_bf16(a, b, d)
    M, K = a.shape
    N = b.shape[0]
    if b.shape[1] != K or tuple(d.shape) != (M, N):
        raise ValueError(f"gemm_tn shapes: a {tuple(a.shape)} b {tuple(b.shape)} d {tuple(d.shape)}")
    SHAPES[("ppo_gemm_tn", M, N, K)] += 1
    call("ppo_gemm_tn", _ptr(a), _ptr(b), _ptr(d), M, N, K, _stream(stream))


def gemm_tn_gelu(a, b, g, f, zero_bias, stream=None):
    """f = a @ b^T (pre-activation, bf16) and g = gelu_tanh(f) from one tcgen05 GEMM."""
    _check_bf16(a, b, g, f)
    M, K = a.shape
    N = b.shape[0]
    if b.shape[1] != K or tuple(g.shape) != (M, N) or tuple(f.shape) != (M, N) or zero_bias.numel() != N:
        raise ValueError("gemm_tn_gelu shapes")
    SHAPES[("ppo_gemm_tn_gelu", M, N, K)] += 1
    call("ppo_gemm_tn_gelu", _ptr(a), _ptr(b), _ptr(g), _ptr(f), _ptr(zero_bias), M, N, K, _stream(stream))


def attn_fwd(qkv, o, lse, heads, scale=None, stream=None):
    """Causal attention forward on tcgen05 (K7): qkv[s, 3h] bf16 -> o[s, h] bf16 and
    lse[heads, s] fp32 (natural log), both writable views into the activation slab."""
    _check_bf16(qkv, o)
    s, h3 = qkv.shape
    h = h3 // 3
    D = h // heads
    if h3 != 3 * h or tuple(o.shape) != (s, h) or lse.dtype != _torch().float32 or not lse.is_cuda or lse.numel() != heads * s:
        raise ValueError(f"attn_fwd shapes: qkv {tuple(qkv.shape)} o {tuple(o.shape)} lse {tuple(lse.shape)}")
    if not (qkv.is_contiguous() and o.is_contiguous() and lse.is_contiguous()):
        raise ValueError("attn_fwd: qkv, o and lse must be contiguous")
    scale = D ** -0.5 if scale is None else scale
    SHAPES[("ppo_attn_fwd", s, heads, D)] += 1
    call("ppo_attn_fwd", _ptr(qkv), _ptr(o), _ptr(lse), s, heads, D, scale, _stream(stream))


def attn_bwd_workspace_bytes(seq, heads, head_dim=128):
    return int(load().ppo_attn_bwd_workspace_bytes(seq, heads, head_dim))


def attn_bwd(qkv, o, do, lse, dqkv, heads, workspace, scale=None, stream=None):
    """Causal attention backward on tcgen05 (K7b): dqkv[s, 3h] = [dq | dk | dv] (bf16) from
    qkv[s, 3h], the saved o[s, h] and lse[heads, s] and the output gradient do[s, h].
    ``workspace``: a CUDA buffer of at least ``attn_bwd_workspace_bytes`` (fp32 dq
    accumulator + row statistics)."""
    _check_bf16(qkv, o, do, dqkv)
    s, h3 = qkv.shape
    h = h3 // 3
    D = h // heads
    if (h3 != 3 * h or tuple(o.shape) != (s, h) or tuple(do.shape) != (s, h) or tuple(dqkv.shape) != (s, h3)
            or lse.dtype != _torch().float32 or not lse.is_cuda or lse.numel() != heads * s):
        raise ValueError(f"attn_bwd shapes: qkv {tuple(qkv.shape)} o {tuple(o.shape)} do {tuple(do.shape)} "
                         f"dqkv {tuple(dqkv.shape)} lse {tuple(lse.shape)}")
    if not all(t.is_contiguous() for t in (qkv, o, do, lse, dqkv)):
        raise ValueError("attn_bwd: operands must be contiguous")
    need = attn_bwd_workspace_bytes(s, heads, D)
    if not workspace.is_cuda or workspace.numel() * workspace.element_size() < need:
        raise ValueError(f"attn_bwd: workspace needs {need} bytes")
    scale = D ** -0.5 if scale is None else scale
    SHAPES[("ppo_attn_bwd", s, heads, D)] += 1
    call("ppo_attn_bwd", _ptr(qkv), _ptr(o), _ptr(do), _ptr(lse), _ptr(dqkv), _ptr(workspace), s, heads, D, scale,
         _stream(stream))


def gemm_nn(a, b, d, beta=0.0, stream=None):
    """d[M,N] = a[M,K] @ b[K,N] + beta * d on tcgen05 (activation gradients: dX = dY @ W)."""
    _check_bf16(a, b, d)
    M, K = a.shape
    N = b.shape[1]
    if b.shape[0] != K or tuple(d.shape) != (M, N):
        raise ValueError(f"gemm_nn shapes: a {tuple(a.shape)} b {tuple(b.shape)} d {tuple(d.shape)}")
    SHAPES[("ppo_gemm_nn", M, N, K)] += 1
    call("ppo_gemm_nn", _ptr(a), _ptr(b), _ptr(d), M, N, K, beta, _stream(stream))


def gemm_nn_dgelu(a, b, z, d, stream=None):
    """d = (a @ b) * gelu_tanh'(z): fc2 dgrad fused with the GeLU backward."""
    _check_bf16(a, b, z, d)
    M, K = a.shape
    N = b.shape[1]
    if b.shape[0] != K or tuple(d.shape) != (M, N) or tuple(z.shape) != (M, N):
        raise ValueError("gemm_nn_dgelu shapes")
    SHAPES[("ppo_gemm_nn_dgelu", M, N, K)] += 1
    call("ppo_gemm_nn_dgelu", _ptr(a), _ptr(b), _ptr(z), _ptr(d), M, N, K, _stream(stream))


def gemm_wgrad(dy, x, dw, beta=1.0, stream=None):
    """dw[M,N] (fp32) = beta * dw + dy[K,M]^T @ x[K,N] on tcgen05 (K = tokens)."""
    _check_bf16(dy, x)
    K, M = dy.shape
    N = x.shape[1]
    if x.shape[0] != K or tuple(dw.shape) != (M, N) or dw.dtype != _torch().float32 or not dw.is_contiguous():
        raise ValueError(f"gemm_wgrad shapes: dy {tuple(dy.shape)} x {tuple(x.shape)} dw {tuple(dw.shape)}")
    SHAPES[("ppo_gemm_wgrad", M, N, K)] += 1
    call("ppo_gemm_wgrad", _ptr(dy), _ptr(x), _ptr(dw), M, N, K, beta, _stream(stream))


def _torch():
    import torch

    return torch


def embed_fwd(tokens, wte, wpe, x, stream=None):
    """x[r] = wte[tokens[r]] + wpe[r] (first stage input; tokens: int64 [rows] on device)."""
    _check_bf16(wte, wpe, x)
    rows, h = x.shape
    if tokens.dtype != _torch().int64 or tokens.numel() != rows or wte.shape[1] != h or tuple(wpe.shape) != (rows, h):
        raise ValueError("embed_fwd shapes")
    call("ppo_embed_fwd", _ptr(tokens), _ptr(wte), _ptr(wpe), _ptr(x), rows, h, wte.shape[0], _stream(stream))


def embed_bwd(tokens, dy, gwte, gwpe, stream=None):
    """gwte[tokens[r]] += dy[r]; gwpe[r] += dy[r] (fp32 accumulators, bf16 dy)."""
    _check_bf16(dy)
    rows, h = dy.shape
    t = _torch()
    if (tokens.dtype != t.int64 or tokens.numel() != rows or gwte.dtype != t.float32 or gwpe.dtype != t.float32
            or gwte.shape[1] != h or tuple(gwpe.shape) != (rows, h)):
        raise ValueError("embed_bwd shapes")
    call("ppo_embed_bwd", _ptr(tokens), _ptr(dy), _ptr(gwte), _ptr(gwpe), rows, h, gwte.shape[0], _stream(stream))


def colsum(x, acc, stream=None):
    _check_bf16(x)
    call("ppo_colsum", _ptr(x), _ptr(acc), x.numel() // x.shape[-1], x.shape[-1], _stream(stream))


def pack(items, dst, stream=None):
    """items: list of (src_tensor_or_ptr, dst_offset, rows, row_bytes, src_pitch[, dst_pitch])."""
    arr = (GatherItem * len(items))()
    for i, it in enumerate(items):
        src, off, rows, row_bytes, pitch = it[:5]
        dpitch = it[5] if len(it) > 5 else 0
        arr[i] = GatherItem(src if isinstance(src, int) else src.data_ptr(), off, rows, row_bytes, pitch, dpitch)
    call("ppo_pack", arr, len(items), dst if isinstance(dst, int) else dst.data_ptr(), _stream(stream))


def transfer(direction, segments, copy_stream, wait_event=None, done_event=None):
    """segments: list of (device_ptr, host_ptr, nbytes); events: raw cudaEvent_t ints or None."""
    arr = (Segment * len(segments))()
    for i, (d, h, n) in enumerate(segments):
        arr[i] = Segment(d, h, n)
    call("ppo_transfer", direction, arr, len(segments), copy_stream, wait_event, done_event)


GEMM_OPS = {"tn": 0, "tn_gelu": 1, "nn": 2, "nn_acc": 2, "nn_dgelu": 3, "wgrad": 4}


def gemm_set_swizzle(kind: str, M: int, N: int, K: int, swizzle: int) -> None:
    """Tile-scheduler swizzle for libppo_b200 GEMM ``kind`` at M x N x K (tuner hook)."""
    call("ppo_gemm_set_swizzle", GEMM_OPS[kind], M, N, K, swizzle)


def stream_write_u32(stream, addr: int, value: int) -> None:
    """Stream-ordered 32-bit store (cuStreamWriteValue32): signal a sync-edge flag."""
    call("ppo_stream_write_u32", stream.cuda_stream, addr, value)


def stream_wait_u32(stream, addr: int, value: int) -> None:
    """Block ``stream`` until *addr == value (cuStreamWaitValue32): wait on a sync-edge flag."""
    call("ppo_stream_wait_u32", stream.cuda_stream, addr, value)


def host_register(ptr: int, nbytes: int) -> int:
    """Pin and map host memory (e.g. POSIX shared memory) into the GPU; returns the device pointer."""
    out = ctypes.c_void_p()
    call("ppo_host_register", ptr, nbytes, ctypes.byref(out))
    return int(out.value)


def host_unregister(ptr: int) -> None:
    call("ppo_host_unregister", ptr)


def timestamp(slot_ptr: int, stream) -> None:
    """Stream-ordered GPU global-timer write (ns, uint64) to device address slot_ptr."""
    call("ppo_timestamp", slot_ptr, stream.cuda_stream)


class PinnedPool:
    """Preallocated page-locked host arena carved into host bins (no per-step alloc).

    ``numa_node`` -1 (default): pages bound to the NUMA node of ``device``'s PCI
    function before first touch (``ppo_pool_create_numa``); -2: no binding; >= 0: that
    node.  ``self.numa_node`` is the node the pages are bound to (-1: single-node host
    or unbound)."""

    def __init__(self, nbytes: int, device: int | None = None, numa_node: int = -1):
        self._h = ctypes.c_void_p()
        if device is None:
            import torch

            device = torch.cuda.current_device()
        node = _I32(-1)
        call("ppo_pool_create_numa", int(nbytes), int(device), int(numa_node), ctypes.byref(self._h),
             ctypes.byref(node))
        self.numa_node = int(node.value)
        self.base = int(load().ppo_pool_base(self._h))
        self.nbytes = int(nbytes)
        self._cursor = 0

    def carve(self, nbytes: int, align: int = 4096) -> int:
        start = (self._cursor + align - 1) // align * align
        if start + nbytes > self.nbytes:
            raise MemoryError(f"pinned pool exhausted: need {nbytes} at {start}, pool {self.nbytes}")
        self._cursor = start + nbytes
        return self.base + start

    def close(self):
        if self._h:
            call("ppo_pool_destroy", self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NcclComm:
    """Point-to-point communicator (K8) created from a unique id shared by the host runtime."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        call("ppo_comm_unique_id", buf)
        return bytes(buf)

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        self._h = ctypes.c_void_p()
        call("ppo_comm_init", buf, nranks, rank, device, ctypes.byref(self._h))
        self.nranks, self.rank = nranks, rank

    def p2p(self, ops, stream):
        """ops: list of (is_send, peer, ptr, nbytes); one NCCL group on ``stream`` (raw handle)."""
        arr = (P2POp * len(ops))()
        for i, (is_send, peer, ptr, n) in enumerate(ops):
            arr[i] = P2POp(1 if is_send else 0, peer, ptr, n)
        call("ppo_p2p", self._h, arr, len(ops), stream)

    def close(self):
        if self._h:
            call("ppo_comm_destroy", self._h)
            self._h = ctypes.c_void_p()
