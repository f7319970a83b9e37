"""One stage (no pipeline) of the runtime model vs the serial fp32 oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from helpers.parity import violations  # noqa: E402
from oracle import gpt as oracle_gpt  # noqa: E402
from paper_2503_01328_b200.runtime import model as rt  # noqa: E402

DEV = torch.device("cuda:0")


def rel_err(a, b):
    return float((a - b).norm() / (b.norm() + 1e-12))


@pytest.mark.parametrize("attn", ["tcgen05", "cudnn"])
def test_single_stage_loss_and_grads_match_oracle(attn):
    cfg = rt.ModelConfig(n_layers=2, hidden=256, heads=4, seq=512, vocab=1024)
    ocfg = oracle_gpt.GPTConfig(n_layers=2, hidden=256, heads=4, seq=512, vocab=1024)
    m = 2
    tokens = oracle_gpt.make_tokens(ocfg, m, seed=0)
    params = oracle_gpt.init_params(ocfg, seed=1234)
    ref_params = rt.init_params(cfg, seed=1234)
    assert all(torch.equal(params[k], ref_params[k]) for k in params)
    want_loss, _, want_grads = oracle_gpt.forward_backward(ocfg, params, tokens)

    st = rt.Stage(cfg, 0, 1, m, DEV, attn=attn)
    assert st.attn_ours == (attn == "tcgen05")
    slab_mem = torch.empty(st.layout.slab_bytes, dtype=torch.uint8, device=DEV)
    slab = rt.SlabView(st.layout, slab_mem)
    st.zero_grad()
    for mb in range(m):
        tok = tokens[mb].to(DEV)
        st.embed(slab, tok)
        st.forward(slab, mb, 0, tokens=tok)
        st.backward(slab, mb, 0, tokens=tok)
    torch.cuda.synchronize()
    loss = float(st.loss_sum) / m
    assert violations(loss, want_loss, {k: v.cpu() for k, v in st.g.items()}, want_grads) == []
