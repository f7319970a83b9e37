"""tcgen05 GEMMs of libppo_b200 vs cuBLAS (torch.mm) at the C2 layer shapes:
correctness (relative error vs fp32 reference) and TFLOP/s (CUDA-graph replay)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_01328_b200.runtime import native  # noqa: E402

dev = torch.device("cuda:0")
torch.manual_seed(0)
s, h = int(os.environ.get("S", 4096)), int(os.environ.get("H", 2048))
shapes = {"qkv": (s, 3 * h, h), "proj": (s, h, h), "fc1": (s, 4 * h, h), "fc2": (s, h, 4 * h)}


def timeit(fn, reps=20):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / reps)
    return best * 1e-3


for name, (M, N, K) in shapes.items():
    a = (torch.randn(M, K, device=dev) * 0.5).bfloat16()
    b = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
    d = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ref = a.float() @ b.float().t()
    native.gemm_tn(a, b, d)
    torch.cuda.synchronize()
    err = float((d.float() - ref).norm() / ref.norm())
    t_ours = timeit(lambda: native.gemm_tn(a, b, d))
    out = torch.empty_like(d)
    t_cublas = timeit(lambda: torch.mm(a, b.t(), out=out))
    fl = 2 * M * N * K
    print(f"{name:5s} M={M} N={N} K={K}: rel_err {err:.2e}  ours {fl / t_ours / 1e12:7.1f} TF/s  cuBLAS {fl / t_cublas / 1e12:7.1f} TF/s")
    if name == "fc1":
        f = torch.empty_like(d)
        g = torch.empty_like(d)
        zb = torch.zeros(N, device=dev)
        native.gemm_tn_gelu(a, b, g, f, zb)
        torch.cuda.synchronize()
        errf = float((f.float() - ref).norm() / ref.norm())
        gref = 0.5 * ref * (1 + torch.tanh(0.7978845608028654 * (ref + 0.044715 * ref ** 3)))
        errg = float((g.float() - gref).norm() / gref.norm())
        t_f = timeit(lambda: native.gemm_tn_gelu(a, b, g, f, zb))
        print(f"      fc1+gelu fused: rel_err f {errf:.2e} g {errg:.2e}  {fl / t_f / 1e12:7.1f} TF/s "
              f"(vs cuBLAS + gelu kernel {t_cublas * 1e6:.1f} us + separate gelu)")

# ---- backward GEMMs: dgrad (NN), fused fc2-dgrad + dGeLU, weight gradient (fp32 accumulate)
for name, (M, N, K) in {"dgrad_fc1": (s, h, 4 * h), "dgrad_qkv": (s, h, 3 * h), "dgrad_fc2": (s, 4 * h, h),
                        "dgrad_proj": (s, h, h)}.items():
    a = (torch.randn(M, K, device=dev) * 0.5).bfloat16()
    b = (torch.randn(K, N, device=dev) * 0.02).bfloat16()
    d = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ref = a.float() @ b.float()
    native.gemm_nn(a, b, d)
    torch.cuda.synchronize()
    err = float((d.float() - ref).norm() / ref.norm())
    t_ours = timeit(lambda: native.gemm_nn(a, b, d))
    out = torch.empty_like(d)
    t_cublas = timeit(lambda: torch.mm(a, b, out=out))
    fl = 2 * M * N * K
    print(f"{name:10s} NN M={M} N={N} K={K}: rel_err {err:.2e}  ours {fl / t_ours / 1e12:7.1f}  cuBLAS {fl / t_cublas / 1e12:7.1f} TF/s")
    if name == "dgrad_fc2":
        z = (torch.randn(M, N, device=dev)).bfloat16()
        native.gemm_nn_dgelu(a, b, z, d)
        torch.cuda.synchronize()
        zf = z.float()
        th = torch.tanh(0.7978845608028654 * zf * (1 + 0.044715 * zf * zf))
        dgl = 0.5 * zf * (1 - th * th) * (0.7978845608028654 + 0.1070322243 * zf * zf) + 0.5 * (1 + th)
        want = ref * dgl
        err = float((d.float() - want).norm() / want.norm())
        t_f = timeit(lambda: native.gemm_nn_dgelu(a, b, z, d))
        print(f"           fused dGeLU: rel_err {err:.2e}  {fl / t_f / 1e12:7.1f} TF/s")
for name, (M, N, K) in {"wgrad_qkv": (3 * h, h, s), "wgrad_proj": (h, h, s), "wgrad_fc1": (4 * h, h, s),
                        "wgrad_fc2": (h, 4 * h, s)}.items():
    dy = (torch.randn(K, M, device=dev) * 0.5).bfloat16()
    x = (torch.randn(K, N, device=dev) * 0.5).bfloat16()
    dw = torch.randn(M, N, device=dev)
    ref = dw + dy.float().t() @ x.float()
    native.gemm_wgrad(dy, x, dw, 1.0)
    torch.cuda.synchronize()
    err = float((dw - ref).norm() / ref.norm())
    dw2 = torch.zeros(M, N, device=dev)
    t_ours = timeit(lambda: native.gemm_wgrad(dy, x, dw2, 1.0))
    t_cublas = timeit(lambda: torch.addmm(dw2, dy.t(), x, out_dtype=torch.float32, out=dw2))
    fl = 2 * M * N * K
    print(f"{name:10s} M={M} N={N} K={K}: rel_err {err:.2e}  ours {fl / t_ours / 1e12:7.1f}  cuBLAS(addmm fp32) {fl / t_cublas / 1e12:7.1f} TF/s")
