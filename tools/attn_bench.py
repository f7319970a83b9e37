"""K7 attention forward: ours (tcgen05, libppo_b200) vs cuDNN's fused kernel (+ the K1
pack into the slab that cuDNN's separate output needs), device time per launch from a
CUDA-graph replay.  FLOPs are causal-effective (2 s^2 h).  PPO_ATTN_ORDER selects the
tile-deal order of our persistent scheduler (0 snake LPT, 1 cyclic LPT, 2 shortest first).

    python tools/attn_bench.py [--shapes 4096x16,8192x32,16384x40] [--orders 0,1,2]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one(s, H, D, order):
    import torch

    from bench import _graph_time_us
    from paper_2503_01328_b200.runtime import native

    dev = torch.device("cuda:0")
    h = H * D
    sets = []
    for _ in range(2):
        qkv = torch.randn(s, 3 * h, device=dev, dtype=torch.bfloat16)
        sets.append((qkv, torch.empty(s, h, device=dev, dtype=torch.bfloat16), torch.empty(H, s, device=dev),
                     torch.empty(2 * s * h + 4 * H * s, device=dev, dtype=torch.uint8)))
    ours = [lambda t=t: native.attn_fwd(t[0], t[1], t[2], H) for t in sets]

    def cudnn(t):
        q, k, v = [x.transpose(1, 2) for x in t[0].view(1, s, 3, H, D).unbind(2)]
        r = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
        native.pack([(r[0], 0, 1, 2 * s * h, 0), (r[1], 2 * s * h, 1, 4 * H * s, 0)], t[3])

    def cudnn_only(t):
        q, k, v = [x.transpose(1, 2) for x in t[0].view(1, s, 3, H, D).unbind(2)]
        torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)

    flops = 2 * s * s * h
    out = {"s": s, "heads": H, "head_dim": D, "order": order}
    for name, fns in (("ours", ours), ("cudnn+pack", [lambda t=t: cudnn(t) for t in sets]),
                      ("cudnn", [lambda t=t: cudnn_only(t) for t in sets])):
        if name != "ours" and order != 0:
            continue
        us = _graph_time_us(fns, dev, torch, launches=8)
        out[name] = {"us": round(us, 2), "tflops": round(flops / us / 1e6, 1)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x16,8192x32,16384x40")
    ap.add_argument("--orders", default="0,1,2")
    ap.add_argument("--one", default=None, help=argparse.SUPPRESS)
    a = ap.parse_args()
    if a.one:
        s, H, D, order = map(int, a.one.split(","))
        print(json.dumps(run_one(s, H, D, order)))
        return
    for shp in a.shapes.split(","):
        s, H = map(int, shp.split("x"))
        for order in map(int, a.orders.split(",")):
            env = dict(os.environ, PPO_ATTN_ORDER=str(order))
            p = subprocess.run([sys.executable, __file__, "--one", f"{s},{H},128,{order}"], env=env,
                               capture_output=True, text=True)
            print(p.stdout.strip() or p.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()
