"""Pipeline timeline of the K7b attention backward for CTA (head 0, kv block 0) -- the
longest walk -- from the kernel's diagnostic SM-clock events (ppo_attn_bwd_trace).
Prints, per q step, the clocks (relative to the first S issue) at which the UMMA thread
passed each wait and commit, and when the softmax-gradient and dQ-drain warps did, plus
a summary of where the issuing thread waited.

    python tools/attn_bwd_trace.py [--s 4096 --heads 16]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EVENTS = {0: "m_qf", 1: "m_S", 2: "m_dsf", 3: "m_dk", 4: "m_dof", 5: "m_dqe", 6: "m_dP", 7: "m_pf", 8: "m_dV",
          16: "g_S0", 17: "g_S1", 18: "g_dQ0", 19: "g_dQ1", 23: "g_dK1", 24: "g_dP0", 25: "g_dP1", 26: "g_dV0",
          27: "g_dV1", 28: "p_qe", 29: "p_doe", 10: "c_sf", 40: "c_ldS", 41: "c_exp", 42: "c_bar", 43: "c_stP", 11: "c_pa", 12: "c_dpf", 13: "c_dse", 44: "c_ldP", 45: "c_dS", 46: "c_fence", 14: "c_dsa", 20: "r_dqf", 21: "r_dqe"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=4096)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--rows", type=int, default=8)
    a = ap.parse_args()
    import torch

    from paper_2503_01328_b200.runtime import native

    dev = torch.device("cuda:0")
    s, H, D = a.s, a.heads, 128
    h = H * D
    qkv = torch.randn(s, 3 * h, device=dev).bfloat16()
    do = torch.randn(s, h, device=dev).bfloat16()
    o = torch.empty(s, h, device=dev, dtype=torch.bfloat16)
    lse = torch.empty(H, s, device=dev)
    native.attn_fwd(qkv, o, lse, H)
    dqkv = torch.empty_like(qkv)
    ws = torch.empty(native.attn_bwd_workspace_bytes(s, H, D), device=dev, dtype=torch.uint8)
    n_cta = H * (s // 128)
    tr = torch.zeros(64 * 256 + 4 * n_cta, device=dev, dtype=torch.int64)
    native.attn_bwd(qkv, o, do, lse, dqkv, H, ws)  # warm
    native.load().ppo_attn_bwd_trace(tr.data_ptr())
    native.attn_bwd(qkv, o, do, lse, dqkv, H, ws)
    torch.cuda.synchronize()
    native.load().ppo_attn_bwd_trace(None)
    cta = [c for c in tr[64 * 256:].view(n_cta, 4).cpu().tolist() if c[0] > 0]  # persistent grid: <= n_cta
    t = tr[:64 * 256].view(64, 256).cpu()
    n = s // 128
    t0 = int(t[0, 0])
    ev = {name: [int(t[e, i]) - t0 for i in range(n)] for e, name in EVENTS.items()}
    if ev["g_S1"][1] < 0:
        ev = {k: v for k, v in ev.items() if not k.startswith("g_")}
    print("step " + " ".join(f"{k:>7}" for k in ev))
    for i in list(range(min(a.rows, n))) + [n - 1]:
        print(f"{i:4d} " + " ".join(f"{ev[k][i]:7d}" for k in ev))
    # issuing-thread waits per step (clocks): q, dS, dO, dQ drained, P
    waits = {"dS": [], "dQ_drained": [], "P": [], "period": [], "q_wait": [], "q_tma_latency": [],
             "do_tma_latency": []}
    for i in range(1, n):
        waits["dS"].append(ev["m_dsf"][i - 1] - ev["m_S"][i])
        waits["dQ_drained"].append(ev["m_dqe"][i] - ev["m_dof"][i])
        waits["P"].append(ev["m_pf"][i] - ev["m_dP"][i])
        waits["period"].append(ev["m_S"][i] - ev["m_S"][i - 1])
        waits["q_wait"].append(ev["m_qf"][i] - ev["m_dV"][i - 1])
        waits["q_tma_latency"].append(ev["m_qf"][i] - ev["p_qe"][i])
        waits["do_tma_latency"].append(ev["m_dof"][i] - ev["p_doe"][i])
    if "g_S1" in ev and ev["g_S1"][1] > 0:  # PPO_ATB_EXP bit 2: each GEMM serialised and timed
        for name, a0, a1 in (("S", "g_S0", "g_S1"), ("dK", "g_dQ0", "g_dQ1"), ("dQ", "g_dQ1", "g_dK1"),
                             ("dP", "g_dP0", "g_dP1"), ("dV", "g_dV0", "g_dV1")):
            d = [ev[a1][i] - ev[a0][i] for i in range(1, n - 1)]
            waits["gemm_" + name] = d
    for a0, a1 in (("c_sf", "c_ldS"), ("c_ldS", "c_exp"), ("c_exp", "c_bar"), ("c_bar", "c_stP"), ("c_stP", "c_pa"),
                   ("c_dse", "c_ldP"), ("c_ldP", "c_dS"), ("c_dS", "c_fence"), ("c_fence", "c_dsa"), ("c_dpf", "c_dse")):
        waits[a0 + "->" + a1] = [ev[a1][i] - ev[a0][i] for i in range(1, n)]
    summ = {k: round(sum(v) / len(v), 1) for k, v in waits.items()}
    if int(t[30, 0]) > 0:  # PPO_ATB_EXP bit 3: clocks per 128^3 GEMM, 16 back to back
        summ["gemm_form_clk"] = dict(zip(["S_KK", "dQ_MNMN", "dK_KMN", "dV_TMN", "T_K", "KK_acc"],
                                         [int(t[30, i]) for i in range(6)]))
    life = [int(t[48, i]) - t0 for i in range(5)]  # start, K/V landed, dK/dV done, stores issued, all done
    summ["cta00_clk"] = {"start_to_kv": life[1] - life[0], "kv_to_first_q": -life[1],
                         "last_step_to_dkdv": life[2] - ev["m_dk"][n - 1], "epilogue": life[3] - life[2],
                         "to_exit": life[4] - life[3]}
    summ["ideal_period_clk"] = 5 * 512
    summ["total_clk"] = ev["m_dk"][n - 1]
    # CTA residency: busy time per SM vs the kernel's span, gaps between CTAs on an SM
    t_lo = min(c[0] for c in cta)
    t_hi = max(c[1] for c in cta)
    per_sm = {}
    for c in cta:
        per_sm.setdefault(c[2], []).append((c[0] - t_lo, c[1] - t_lo))
    busy = [sum(b - a for a, b in v) for v in per_sm.values()]
    gaps = [b2[0] - a1[1] for v in per_sm.values() for a1, b2 in zip(sorted(v), sorted(v)[1:])]
    ends = [max(b for _, b in v) for v in per_sm.values()]
    import numpy as np
    A = np.array([[1.0, c[3]] for c in cta])
    y = np.array([(c[1] - c[0]) / 1e3 for c in cta])
    fit = np.linalg.lstsq(A, y, rcond=None)[0]
    summ["cta_fit_us"] = {"fixed": round(float(fit[0]), 2), "per_step": round(float(fit[1]), 3)}
    summ["cta"] = {"span_us": round((t_hi - t_lo) / 1e3, 1), "sms": len(per_sm),
                   "mean_busy_frac": round(sum(busy) / len(busy) / (t_hi - t_lo), 3),
                   "mean_gap_us": round(sum(gaps) / max(1, len(gaps)) / 1e3, 2),
                   "first_sm_done_us": round(min(ends) / 1e3, 1), "mean_cta_us": round(
                       sum(b - a for v in per_sm.values() for a, b in v) / len(cta) / 1e3, 2)}
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
