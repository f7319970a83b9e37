"""NCCL stage-boundary traffic inside the whole-iteration CUDA graph.

Every gpurun box has one GPU, so the boundary runs over a 1-rank NCCL communicator
(``mode="nccl_loopback"``: each message a grouped self send/recv, neighbours
emulated exactly as ``mode="emulate"`` does).  Checked: the NCCL p2p kernels are
captured into the one-graph-per-iteration replay (the path ``mode="nccl"`` takes
under torchrun), numerics equal the emulated boundary's bit for bit, and the
captured replay equals the host-issued iterations.
"""

from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2503_01328_b200 as po  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

CFG = ModelConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)


def _grads(res):
    return {k: g.float().cpu().clone() for r in res.runners for st in r.stages.values() for k, g in st.g.items()}


@pytest.mark.parametrize("rank", [0, 1])
def test_nccl_loopback_in_iteration_graph(rank):
    sched, plan = po.build_1f1b_full_offload(2, 4, po.PassCosts.unit(), Fraction(1))
    tokens = torch.randint(0, CFG.vocab, (4, CFG.seq + 1), generator=torch.Generator().manual_seed(0))
    kw = dict(model=CFG, rank=rank, tokens=tokens, optimizer="none", iters=2, warmup=1, gemm="tcgen05",
              attn="tcgen05", verify_roundtrip=True)
    emu = ex.execute(sched, plan, mode="emulate", **kw)
    g_emu = _grads(emu)
    emu.close()
    eager = ex.execute(sched, plan, mode="nccl_loopback", **kw)
    g_eager = _grads(eager)
    ops = [op.kind for op in eager.programs[rank].ops]
    assert ("SEND_ACT" in ops) if rank == 0 else ("RECV_ACT" in ops)
    eager.close()
    graph = ex.execute(sched, plan, mode="nccl_loopback", iteration_graph=True, **kw)
    assert "iteration" in graph.runners[0].graph_native_launches  # replayed as one CUDA graph
    assert ex.roundtrip_mismatches(graph.runners) == []
    g_graph = _grads(graph)
    for k in g_emu:  # optimizer "none": every iteration recomputes the same gradients
        # (equal up to the order of the LN / embedding float atomics)
        assert torch.allclose(g_eager[k], g_emu[k], rtol=1e-5, atol=1e-9), k
        assert torch.allclose(g_graph[k], g_emu[k], rtol=1e-5, atol=1e-9), k
    if rank == 1:
        assert graph.losses[-1] == eager.losses[-1] == emu.losses[-1]
    graph.close()
