"""Must-fail tests: the parity bars (tests/helpers/parity.py) are tight enough to
catch the bugs a recompute / offload engine can plausibly have.

Each test first runs the unmodified path (must pass the bars), then injects one
fault and requires the SAME checker to reject it:
* the backward replays one dropout site with a wrong Philox offset (mask of the
  forward != mask of the backward);
* the backward skips one LayerNorm recompute (LN2 of the top layer, emitted by
  the LN2 backward: the fc1 weight gradient then reads a stale workspace);
* a reload lands in the wrong slab (the lowered program's RELOAD and its B disagree).
"""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2503_01328_b200 as po  # noqa: E402
from helpers.parity import violations  # noqa: E402
from oracle import gpt as oracle_gpt  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402
from paper_2503_01328_b200.runtime import model as rt  # noqa: E402

DEV = torch.device("cuda:0")
CFG = rt.ModelConfig(n_layers=2, hidden=256, heads=4, seq=512, vocab=1024)
OCFG = oracle_gpt.GPTConfig(n_layers=2, hidden=256, heads=4, seq=512, vocab=1024)
M = 2


@pytest.fixture(scope="module")
def oracle():
    tokens = oracle_gpt.make_tokens(OCFG, M, seed=0)
    loss, _, grads = oracle_gpt.forward_backward(OCFG, oracle_gpt.init_params(OCFG, seed=1234), tokens)
    return tokens, loss, grads


def _stage_run(tokens):
    st = rt.Stage(CFG, 0, 1, M, DEV, gemm="tcgen05", attn="tcgen05")
    slab = rt.SlabView(st.layout, torch.empty(st.layout.slab_bytes, dtype=torch.uint8, device=DEV))
    st.zero_grad()
    for mb in range(M):
        tok = tokens[mb].to(DEV)
        st.embed(slab, tok)
        st.forward(slab, mb, 0, tokens=tok)
        st.backward(slab, mb, 0, tokens=tok)
    torch.cuda.synchronize()
    return float(st.loss_sum) / M, {k: v.cpu() for k, v in st.g.items()}


def test_wrong_dropout_offset_in_backward_is_caught(oracle, monkeypatch):
    tokens, want_loss, want = oracle
    loss, grads = _stage_run(tokens)
    assert violations(loss, want_loss, grads, want) == []
    real_offsets = rt.Stage._offsets
    real_bwd = rt.Stage.backward_body
    state = {"bwd": False}

    def offsets(self, l):
        a, m = real_offsets(self, l)
        return (a + 2, m) if (state["bwd"] and l == 1) else (a, m)  # layer 1, attention branch

    def backward_body(self, *a, **k):
        state["bwd"] = True
        try:
            return real_bwd(self, *a, **k)
        finally:
            state["bwd"] = False

    monkeypatch.setattr(rt.Stage, "_offsets", offsets)
    monkeypatch.setattr(rt.Stage, "backward_body", backward_body)
    loss, grads = _stage_run(tokens)
    bad = violations(loss, want_loss, grads, want)
    assert bad, "a backward replaying the wrong dropout mask passed the parity bars"
    assert any(k.startswith("l1.") or k.startswith("l0.") for k, _ in bad)


def test_skipped_ln2_recompute_is_caught(oracle, monkeypatch):
    tokens, want_loss, want = oracle
    real_k = rt.Stage._k
    seen = {"n": 0}

    def k(self, name, nbytes, fn, *args, **kw):
        # the LN2 recompute rides in the LN2 backward (ln_out): drop it once -- the fc1
        # weight gradient of the top layer, first microbatch, then reads a stale workspace
        if name == "layernorm_bwd" and kw.get("ln_out") is not None:
            seen["n"] += 1
            if seen["n"] == 1:
                kw = dict(kw, ln_out=None, beta=None)
        return real_k(self, name, nbytes, fn, *args, **kw)

    monkeypatch.setattr(rt.Stage, "_k", k)
    loss, grads = _stage_run(tokens)
    assert seen["n"] >= 2
    bad = violations(loss, want_loss, grads, want)
    assert bad, "a skipped LN2 recompute passed the parity bars"
    assert any(name == "l1.w_fc1" for name, _ in bad), bad


def test_reload_into_wrong_slab_is_caught(monkeypatch):
    cfg = rt.ModelConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)
    ocfg = oracle_gpt.GPTConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)
    tokens = oracle_gpt.make_tokens(ocfg, 8, seed=0)
    want_loss, _, want = oracle_gpt.forward_backward(ocfg, oracle_gpt.init_params(ocfg, seed=1234), tokens)
    sched, plan = po.build_1f1b_full_offload(4, 8, po.PassCosts.unit(), Fraction(3, 2))
    kw = dict(model=cfg, mode="virtual", tokens=tokens, optimizer="none", verify_roundtrip=True, gemm="tcgen05",
              attn="tcgen05", use_graphs=False)
    good = ex.execute(sched, plan, **kw)
    assert ex.roundtrip_mismatches(good.runners) == []
    g_good = {k: v.float().cpu() for r in good.runners for st in r.stages.values() for k, v in st.g.items()}
    assert violations(good.losses[-1], want_loss, g_good, want) == []
    good.close()

    real_lower = ex.lower

    def lower(sched_, plan_, rank, **k):
        prog = real_lower(sched_, plan_, rank, **k)
        if rank == 0 and prog.n_slabs > 1:
            for op in prog.ops:
                if op.kind == "RELOAD":
                    # the reload of the first reloaded pair goes to another slab; its B
                    # (and the digest at B start) still read the planned one
                    op.slab = (op.slab + 1) % prog.n_slabs
                    break
        return prog

    monkeypatch.setattr(ex, "lower", lower)
    bad = ex.execute(sched, plan, **kw)
    mism = ex.roundtrip_mismatches(bad.runners)
    g_bad = {k: v.float().cpu() for r in bad.runners for st in r.stages.values() for k, v in st.g.items()}
    # the in-situ digests (slab at B start vs slab at F end) or the oracle bars must see it
    assert mism or violations(bad.losses[-1], want_loss, g_bad, want), "a reload into the wrong slab went unnoticed"
    bad.close()
