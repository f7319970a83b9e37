"""A few eager launches of our attention forward and backward at one shape (for ncu):
    python tools/attn_eager.py [--s 4096 --heads 16 --n 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=4096)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--n", type=int, default=3)
    a = ap.parse_args()
    import torch

    from paper_2503_01328_b200.runtime import native

    dev = torch.device("cuda:0")
    s, H, D = a.s, a.heads, 128
    qkv = torch.randn(s, 3 * H * D, device=dev).bfloat16()
    do = torch.randn(s, H * D, device=dev).bfloat16()
    o = torch.empty(s, H * D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(H, s, device=dev)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(native.attn_bwd_workspace_bytes(s, H, D), device=dev, dtype=torch.uint8)
    for _ in range(a.n):
        native.attn_fwd(qkv, o, lse, H)
        native.attn_bwd(qkv, o, do, lse, dqkv, H, ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
