"""Observed parity errors of the B200 path against the fp32 CPU oracle (diagnostic).

Prints one JSON line per case: loss relative error and the max / per-parameter
relative-L2 gradient error, so the test tolerances can be set from measurements.
usage: python tools/parity_errors.py
"""
import json
import os
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_01328_b200 as po  # noqa: E402
from oracle import gpt as og  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402


def rel(a, b):
    return float((a - b).norm() / (b.norm() + 1e-12))


def grads(res):
    return {k: g.float().cpu() for r in res.runners for st in r.stages.values() for k, g in st.g.items()}


def report(name, loss, want_loss, got, want, **extra):
    errs = {k: rel(got[k], g) for k, g in want.items()}
    worst = max(errs, key=errs.get)
    mat = {k: e for k, e in errs.items() if want[k].dim() == 2}
    vec = {k: e for k, e in errs.items() if want[k].dim() == 1}
    print(json.dumps(dict(case=name, loss=loss, oracle_loss=want_loss, loss_rel=abs(loss - want_loss) / abs(want_loss),
                          grad_rel_max=errs[worst], grad_rel_worst=worst,
                          matrix_max=max(mat.values()), matrix_worst=max(mat, key=mat.get),
                          vector_max=max(vec.values()), vector_worst=max(vec, key=vec.get),
                          grad_rel_median=sorted(errs.values())[len(errs) // 2], **extra)), flush=True)


def main():
    cfg = ModelConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)
    ocfg = og.GPTConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)
    tokens = og.make_tokens(ocfg, 8, seed=0)
    for bf16 in (False, True):
        want_loss, _, want = og.forward_backward(ocfg, og.init_params(ocfg), tokens, bf16=bf16) if bf16 else \
            og.forward_backward(ocfg, og.init_params(ocfg), tokens)
        U = po.PassCosts.unit()
        sched, plan = po.build_1f1b_full_offload(4, 8, U, Fraction(3, 2))
        for gemm, attn in (("tcgen05", "tcgen05"), ("cublas", "cudnn"), ("tcgen05", "cudnn")):
            res = ex.execute(sched, plan, model=cfg, mode="virtual", tokens=tokens, optimizer="none", gemm=gemm, attn=attn)
            report(f"c1_full_offload gemm={gemm} attn={attn} oracle_bf16={bf16}", res.losses[-1], want_loss, grads(res), want)
            res.close()
        for kind in ("gis-h", "po"):
            sv = (po.build_gis_h if kind == "gis-h" else po.build_po)(2, 2, 8, U)
            pl = po.plan_slots(sv, po.select_offload_stages(po.po_block(2, 2, U), 1), Fraction(1))
            res = ex.execute(sv, pl, model=cfg, mode="virtual", tokens=tokens, optimizer="none", gemm="tcgen05",
                             attn="tcgen05")
            report(f"{kind} oracle_bf16={bf16}", res.losses[-1], want_loss, grads(res), want)
            res.close()


if __name__ == "__main__":
    main()
