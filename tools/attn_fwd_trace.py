"""Pipeline timeline of the hand-written attention forward (K7) for the heaviest CTA of
head 0 (the last q-block pair, work item 0), from the kernel's diagnostic SM-clock events
(ppo_attn_fwd_trace): per kv step, when the UMMA thread reached / passed the P waits of
q block 0 and 1, and when each softmax warpgroup saw S, finished the exponentials and
released P.

    python tools/variant_build.py trace ppo_attention_fwd.cu -DPPO_ATTN_TRACE=1
    PPO_LIB_PATH=abtest/trace/libppo_b200.so python tools/attn_fwd_trace.py [--s 4096 --heads 16]

(the probes are compiled out of the default build)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EVENTS = {0: "m_pv0_at", 1: "m_pv0_go", 2: "m_pv1_at", 3: "m_pv1_go", 10: "s0_S", 13: "s0_ld", 20: "s0_max",
          11: "s0_exp", 12: "s0_P", 14: "s1_S", 17: "s1_ld", 21: "s1_max", 15: "s1_exp", 16: "s1_P",
          24: "s0_exp_w0", 25: "s0_exp_w1", 26: "s0_exp_w2", 27: "s0_exp_w3", 28: "s1_exp_w4", 29: "s1_exp_w5",
          30: "s1_exp_w6", 31: "s1_exp_w7"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=4096)
    ap.add_argument("--heads", type=int, default=16)
    a = ap.parse_args()
    import torch

    from paper_2503_01328_b200.runtime import native

    dev = torch.device("cuda:0")
    s, H, D = a.s, a.heads, 128
    qkv = torch.randn(s, 3 * H * D, device=dev).bfloat16()
    o = torch.empty(s, H * D, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(H, s, device=dev)
    native.attn_fwd(qkv, o, lse, H)
    tr = torch.zeros(32 * 256, device=dev, dtype=torch.int64)
    native.load().ppo_attn_fwd_trace(tr.data_ptr())
    native.attn_fwd(qkv, o, lse, H)
    torch.cuda.synchronize()
    native.load().ppo_attn_fwd_trace(None)
    t = tr.view(32, 256).cpu()
    kv = 128  # rows per kv step
    n = s // kv
    t0 = int(t[10, 0])
    ev = {name: [int(t[e, j]) - t0 for j in range(n)] for e, name in EVENTS.items()}
    for j in list(range(4)) + [n - 2]:
        print(j, {k: v[j] for k, v in ev.items()})
    per = lambda a_, b_: round(sum(ev[b_][j] - ev[a_][j] for j in range(2, n - 2)) / (n - 4), 1)  # noqa: E731
    print(json.dumps({"step_clk": round((ev["s0_S"][n - 2] - ev["s0_S"][2]) / (n - 4), 1),
                      "ideal_clk": 4 * 4 * kv, "wait_P0": per("m_pv0_at", "m_pv0_go"),
                      "wait_P1": per("m_pv1_at", "m_pv1_go"), "sm0_S_to_ld": per("s0_S", "s0_ld"),
                      "sm0_ld_to_max": per("s0_ld", "s0_max"), "sm0_max_to_exp": per("s0_max", "s0_exp"),
                      "sm0_exp_to_P": per("s0_exp", "s0_P"), "sm1_S_to_ld": per("s1_S", "s1_ld"),
                      "sm1_ld_to_max": per("s1_ld", "s1_max"), "sm1_max_to_exp": per("s1_max", "s1_exp"),
                      "sm1_exp_to_P": per("s1_exp", "s1_P"),
                      "exp_done_per_warp_vs_w0": [per("s0_S", f"s0_exp_w{w}") for w in range(4)] +
                      [per("s1_S", f"s1_exp_w{w}") for w in range(4, 8)]}))


if __name__ == "__main__":
    main()
