"""tcgen05 GEMM throughput vs the tile-scheduler swizzle (PPO_GEMM_SWIZZLE) at the
C2 and C4 layer shapes, next to cuBLAS.  CUDA-graph replay, TFLOP/s."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_01328_b200.runtime import native  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)


def timeit(fn, reps=10):
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
    return best * 1e3  # us


out = {}
for s, h in ((4096, 2048), (16384, 5120)):
    shapes = {"tn qkv": ("tn", s, 3 * h, h), "tn fc1": ("tn", s, 4 * h, h), "tn fc2": ("tn", s, h, 4 * h),
              "nn fc2-dgrad": ("nn", s, 4 * h, h), "nn fc1-dgrad": ("nn", s, h, 4 * h),
              "wgrad fc1": ("wgrad", 4 * h, h, s), "wgrad proj": ("wgrad", h, h, s)}
    for name, (kind, M, N, K) in shapes.items():
        flops = 2 * M * N * K
        if kind == "tn":
            a, b, d = (torch.randn(M, K, device=dev).bfloat16(), torch.randn(N, K, device=dev).bfloat16(),
                       torch.empty(M, N, device=dev, dtype=torch.bfloat16))
            ours = lambda: native.gemm_tn(a, b, d)  # noqa: E731
            cub = lambda: torch.mm(a, b.t(), out=d)  # noqa: E731
        elif kind == "nn":
            a, b, d = (torch.randn(M, K, device=dev).bfloat16(), torch.randn(K, N, device=dev).bfloat16(),
                       torch.empty(M, N, device=dev, dtype=torch.bfloat16))
            ours = lambda: native.gemm_nn(a, b, d, 0.0)  # noqa: E731
            cub = lambda: torch.mm(a, b, out=d)  # noqa: E731
        else:  # wgrad: acc[M,N] += dy[K,M]^T x[K,N]
            dy, x = torch.randn(K, M, device=dev).bfloat16(), torch.randn(K, N, device=dev).bfloat16()
            acc = torch.zeros(M, N, device=dev)
            ours = lambda: native.gemm_wgrad(dy, x, acc, 1.0)  # noqa: E731
            cub = lambda: torch.addmm(acc, dy.t(), x, out_dtype=torch.float32, out=acc)  # noqa: E731
        row = {"cublas": round(flops / timeit(cub) / 1e6, 1)}
        for sw in (1, 2, 4, 8, 16):
            os.environ["PPO_GEMM_SWIZZLE"] = str(sw)
            row[f"sw{sw}"] = round(flops / timeit(ours) / 1e6, 1)
        os.environ.pop("PPO_GEMM_SWIZZLE")
        out[f"s{s} h{h} {name} {M}x{N}x{K}"] = row
        print(f"s{s} h{h} {name:14s} {M}x{N}x{K}", row, flush=True)

        torch.cuda.empty_cache()
print(json.dumps(out))
