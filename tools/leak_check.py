"""Device-memory accounting across repeated calibrate / execute calls (the sweep
tools run many in one process): prints torch.cuda.memory_allocated after each step
and who still references a finished runner, if anything does."""
import gc
import sys
import weakref

import torch

sys.path.insert(0, ".")
import paper_2503_01328_b200 as po  # noqa: E402
from paper_2503_01328_b200.runtime.calibrate import calibrate_costs  # noqa: E402
from paper_2503_01328_b200.runtime.executor import execute  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402


def mem(tag):
    gc.collect()
    torch.cuda.empty_cache()
    print(f"{tag:28s} allocated {torch.cuda.memory_allocated() / 1e9:8.3f} GB  reserved "
          f"{torch.cuda.memory_reserved() / 1e9:8.3f} GB", flush=True)


dev = torch.device("cuda:0")
cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=1024)
mem("start")
for d in (2, 4):
    lps = 24 // d
    costs, t_o, cal = calibrate_costs(cfg, d, 8, dev, units=lps)
    mem(f"d={d} after calibrate")
    sched = po.build_1f1b(d, lps, 8, costs)
    for name, plan in (("none", None), ("full", po.plan_slots(sched, (0,), t_o / 8))):
        res = execute(sched, plan, model=cfg, mode="emulate", rank=0, device=dev, iters=1, warmup=1)
        mem(f"d={d} {name} after run")
        wr = weakref.ref(res.runners[0])
        ws = weakref.ref(next(iter(res.runners[0].stages.values())))
        res.close()
        del res
        mem(f"d={d} {name} after del")
        for ref_, what in ((wr, "runner"), (ws, "stage")):
            obj = ref_()
            if obj is not None:
                print("  ", what, "alive; referrers:")
                for rr in gc.get_referrers(obj):
                    print("     ", type(rr).__name__, (list(rr.keys())[:8] if isinstance(rr, dict) else str(rr)[:160]))
                del obj
