"""One rank of a multi-process pipeline run (launched by torchrun from
tests/test_multiproc_gpu.py).  All ranks may share one GPU: the boundary goes
over gloo host copies (executor.HostTransport), everything else is the product
path (lowered per-rank program, slab arena, pinned pool, copy streams, kernels).

usage: torchrun --nproc-per-node D tests/helpers/dist_worker.py KIND OUT.json [GEMM ATTN]
KIND: 1f1b (build_1f1b_full_offload(D, 8, unit, 3/2)), 1f1b-i (v=2, selective n=1) or
1f1b-i-sync (the same plan through apply_topology_sync: cross-rank sync-edge flags)
GEMM/ATTN: backends (default tcgen05/tcgen05, pinned so the single-process comparison
run uses the same kernels; "auto" exercises the collective decision table)
"""
import json
import os
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2503_01328_b200 as po  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402
from paper_2503_01328_b200.runtime import gemm_tune  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

CFG = ModelConfig(n_layers=4, hidden=256, heads=4, seq=512, vocab=1024)


def build(kind: str, d: int):
    U = po.PassCosts.unit()
    if kind == "1f1b":
        return po.build_1f1b_full_offload(d, 8, U, Fraction(3, 2))
    if kind == "1f1b-i-sync":  # topology-synchronised plan: cross-process flags in shared memory
        sched = po.build_interleaved_1f1b(d, 2, 8, U)
        plan = po.plan_slots(sched, po.select_offload_stages(po.po_block(d, 2, U), 1), Fraction(1, 2) * U.total)
        hw = po.HardwareSpec(compute_bandwidth=1.0, transfer_bandwidth=1.0, devices_per_switch=2)
        return sched, po.apply_topology_sync(plan, hw)
    sched = po.build_interleaved_1f1b(d, 2, 8, U)
    stages = po.select_offload_stages(po.po_block(d, 2, U), 1)
    return sched, po.plan_slots(sched, stages, Fraction(1, 2) * U.total)


def main():
    kind, out = sys.argv[1], sys.argv[2]
    gemm, attn = (sys.argv[3], sys.argv[4]) if len(sys.argv) > 4 else ("tcgen05", "tcgen05")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    sched, plan = build(kind, world)
    tokens = torch.randint(0, CFG.vocab, (8, CFG.seq + 1), generator=torch.Generator().manual_seed(0))
    res = ex.execute(sched, plan, model=CFG, mode="gloo", rank=rank, device=dev, iters=2, warmup=0, tokens=tokens,
                     optimizer="sgd", lr=1e-2, verify_roundtrip=True, gemm=gemm, attn=attn)
    r = res.runners[0]
    report = {"rank": rank, "losses": res.losses, "secs": res.iteration_seconds,
              "mismatches": ex.roundtrip_mismatches(res.runners), "offloaded": len(r.prog.offloaded),
              "compute_order": [list(k) for k in r.prog.compute_order], "n_slabs": r.prog.n_slabs,
              "table_digest": gemm_tune.digest(), "table": gemm_tune.decisions()}
    reports = [None] * world
    dist.all_gather_object(reports, report)
    if rank == 0:
        with open(out, "w") as f:
            json.dump(reports, f)
    r.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
