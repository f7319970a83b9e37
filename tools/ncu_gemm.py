"""Launch one tcgen05 GEMM of libppo_b200 a few times at a given shape, for
`ncu --set full -k regex:device_kernel --launch-skip 2 -c 1`.

usage: python tools/ncu_gemm.py ENTRY M N K     (ENTRY: tn | tn_gelu | nn | nn_dgelu | wgrad)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_01328_b200.runtime import native  # noqa: E402

entry, M, N, K = sys.argv[1], *map(int, sys.argv[2:5])
dev = torch.device("cuda:0")
bf = dict(device=dev, dtype=torch.bfloat16)
if entry == "wgrad":
    dy, x, dw = torch.randn(K, M, **bf), torch.randn(K, N, **bf), torch.zeros(M, N, device=dev)
    fn = lambda: native.gemm_wgrad(dy, x, dw, 1.0)  # noqa: E731
elif entry in ("tn", "tn_gelu"):
    a, b, d, f = torch.randn(M, K, **bf), torch.randn(N, K, **bf), torch.empty(M, N, **bf), torch.empty(M, N, **bf)
    z = torch.zeros(N, device=dev)
    fn = (lambda: native.gemm_tn(a, b, d)) if entry == "tn" else (lambda: native.gemm_tn_gelu(a, b, d, f, z))
else:
    a, b, d, z = torch.randn(M, K, **bf), torch.randn(K, N, **bf), torch.empty(M, N, **bf), torch.randn(M, N, **bf)
    fn = (lambda: native.gemm_nn(a, b, d, 0.0)) if entry == "nn" else (lambda: native.gemm_nn_dgelu(a, b, z, d))
for _ in range(4):
    fn()
torch.cuda.synchronize()
print("ok", entry, M, N, K)
