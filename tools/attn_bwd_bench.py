"""K7b attention backward: ours (hand-written tcgen05, libppo_b200) vs cuDNN's fused
backward, device µs per launch from a CUDA-graph replay over 2 rotating input sets, and
causal-effective TFLOP/s (5 GEMMs over the lower triangle: 5 * 2 * s^2/2 * h = 5 s^2 h;
cuDNN is credited the same FLOPs).  Ours includes its prep (delta, dq zero) and dq-cast
kernels.

    python tools/attn_bwd_bench.py [--shapes 4096x16,8192x32,16384x40]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one(s, H, D=128, eager=0, profile=0):
    import torch

    from bench import _graph_time_us
    from paper_2503_01328_b200.runtime import native

    dev = torch.device("cuda:0")
    h = H * D
    sets = []
    for i in range(2):
        g = torch.Generator(device=dev).manual_seed(i)
        qkv = torch.randn(s, 3 * h, device=dev, generator=g).bfloat16()
        do = torch.randn(s, h, device=dev, generator=g).bfloat16()
        q, k, v = [t.transpose(1, 2) for t in qkv.view(1, s, 3, H, D).unbind(2)]
        res = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False)
        o = res[0].transpose(1, 2).reshape(s, h).contiguous()
        lse = res[1].reshape(H, s).contiguous()
        dqkv = torch.empty_like(qkv)
        ws = torch.empty(native.attn_bwd_workspace_bytes(s, H, D), device=dev, dtype=torch.uint8)
        sets.append(dict(qkv=qkv, do=do, q=q, k=k, v=v, res=res, o=o, lse=lse, dqkv=dqkv, ws=ws,
                         do4=do.view(1, s, H, D).transpose(1, 2)))

    def ours(t):
        native.attn_bwd(t["qkv"], t["o"], t["do"], t["lse"], t["dqkv"], H, t["ws"])

    def cudnn(t):
        r = t["res"]
        torch.ops.aten._scaled_dot_product_cudnn_attention_backward(
            t["do4"], t["q"], t["k"], t["v"], r[0], r[1], r[6], r[7], None, r[2], r[3], r[4], r[5], 0.0, True)

    if profile:  # per-kernel device time (CUPTI via torch.profiler), eager launches
        from torch.profiler import ProfilerActivity, profile as prof
        res = {}
        for name, fn in (("ours", ours), ("cudnn", cudnn)):
            for i in range(4):
                fn(sets[i % 2])
            torch.cuda.synchronize()
            with prof(activities=[ProfilerActivity.CUDA]) as p:
                for i in range(profile):
                    fn(sets[i % 2])
                torch.cuda.synchronize()
            per = {}
            for e in p.events():
                if e.device_type.name == "CUDA" and e.device_time_total > 0:
                    per.setdefault(e.name[:60], []).append(e.device_time_total)
            res[name] = {k: round(sum(v) / len(v), 2) for k, v in per.items() if len(v) >= profile}
        return {"s": s, "heads": H, "per_kernel_us": res}
    if eager:  # for ncu: plain launches of ours only
        for i in range(eager):
            ours(sets[i % 2])
        torch.cuda.synchronize()
        return {"s": s, "heads": H, "eager_launches": eager}
    flops = 5 * s * s * h
    out = {"s": s, "heads": H, "head_dim": D}
    for name, fn in (("ours", ours), ("cudnn", cudnn)):
        us = _graph_time_us([lambda t=t: fn(t) for t in sets], dev, torch, launches=8)
        out[name] = {"us": round(us, 2), "tflops": round(flops / us / 1e6, 1)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x16,8192x32,16384x40")
    ap.add_argument("--eager", type=int, default=0, help="only launch ours N times (for ncu)")
    ap.add_argument("--profile", type=int, default=0, help="per-kernel times over N eager launches")
    a = ap.parse_args()
    for shp in a.shapes.split(","):
        s, H = map(int, shp.split("x"))
        print(json.dumps(run_one(s, H, eager=a.eager, profile=a.profile)), flush=True)


if __name__ == "__main__":
    main()
