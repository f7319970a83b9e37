"""Multi-process pipeline runs on one GPU (torchrun, one process per rank).

NCCL refuses two ranks on one device, and gpurun boxes have one GPU, so the
boundary here goes over gloo host copies (``executor.HostTransport``).  What is
checked is everything else of the N>1 path: per-rank lowering from the same
schedule, rank-local slab arenas / pinned pools / copy streams, message order
across processes (incl. the interleaved wrap edge), MAX-over-ranks timing, the
last-stage loss reaching every rank -- and that the result equals the
single-process virtual run of the same schedule bit for bit in the first step.
"""
import json
import os
import socket
import subprocess
import sys
from fractions import Fraction

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers.dist_worker import CFG, build  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(nproc, args, env=None, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}"] + args
    e = dict(os.environ, **(env or {}))
    return subprocess.run(cmd, cwd=ROOT, env=e, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("kind", ["1f1b", "1f1b-i", "1f1b-i-sync"])
def test_two_process_pipeline_matches_virtual(kind, tmp_path):
    out = tmp_path / "r.json"
    p = _torchrun(2, ["tests/helpers/dist_worker.py", kind, str(out)])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    reports = json.loads(out.read_text())
    assert [r["rank"] for r in reports] == [0, 1]
    # loss of the last stage reaches every rank; times are MAX over ranks (identical)
    assert reports[0]["losses"] == reports[1]["losses"]
    assert reports[0]["secs"] == reports[1]["secs"]
    for r in reports:
        assert r["mismatches"] == []
    assert sum(r["offloaded"] for r in reports) > 0

    sched, plan = build(kind, 2)
    tokens = torch.randint(0, CFG.vocab, (8, CFG.seq + 1), generator=torch.Generator().manual_seed(0))
    res = ex.execute(sched, plan, model=CFG, mode="virtual", iters=2, warmup=0, tokens=tokens, optimizer="sgd",
                     lr=1e-2, gemm="tcgen05", attn="tcgen05")  # the workers' pinned backends
    for r in res.runners:
        rep = reports[r.rank]
        assert rep["compute_order"] == [list(k) for k in r.prog.compute_order]
        assert rep["n_slabs"] == r.prog.n_slabs
    # step 1 is a pure function of (params, tokens, seeds): bit-identical
    assert reports[0]["losses"][0] == res.losses[0]
    # step 2 sees weights updated with gradients that used float atomics (LN dgamma/dbeta)
    assert reports[0]["losses"][1] == pytest.approx(res.losses[1], rel=1e-3)


def test_two_process_auto_backends_agree(tmp_path):
    """gemm="auto" / attn="auto" under torchrun: rank 0 tunes the decision table and
    broadcasts it (gemm_tune.ensure), so both ranks run identical kernels; the
    single-process run replays the same table and matches the first step bit for bit."""
    out = tmp_path / "r.json"
    p = _torchrun(2, ["tests/helpers/dist_worker.py", "1f1b", str(out), "auto", "auto"])
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    reports = json.loads(out.read_text())
    assert reports[0]["table_digest"] == reports[1]["table_digest"]
    assert reports[0]["table"] and reports[0]["losses"] == reports[1]["losses"]
    from paper_2503_01328_b200.runtime import gemm_tune

    saved = dict(gemm_tune.TABLE)
    try:
        gemm_tune.reset()
        sched, plan = build("1f1b", 2)
        tokens = torch.randint(0, CFG.vocab, (8, CFG.seq + 1), generator=torch.Generator().manual_seed(0))
        res = ex.execute(sched, plan, model=CFG, mode="virtual", iters=1, warmup=0, tokens=tokens, optimizer="sgd",
                         lr=1e-2, tune_table=reports[0]["table"])
        assert gemm_tune.digest() == reports[0]["table_digest"]  # nothing re-tuned
        assert reports[0]["losses"][0] == res.losses[0]
    finally:
        gemm_tune.reset()
        gemm_tune.install(saved)


def test_bench_two_ranks(tmp_path):
    """bench.py's N>1 path end to end (rank 0 prints one JSON line)."""
    p = _torchrun(2, ["bench.py", "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3",
                      "--no-cpu-baseline"], env={"PPO_DIST_BACKEND": "gloo"})
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert abs(line["value"] - 2 * line["pipeline_tokens_per_s"]) < 1e-6 * line["value"]
    full = line["offload"]["full"]
    assert len(full["peak_act_gb_per_rank"]) == 2
    assert full["peak_act_gb"] == max(full["peak_act_gb_per_rank"])
