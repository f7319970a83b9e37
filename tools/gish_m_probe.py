"""GIS-H (v = 3 one-layer chunks) vs 1F1B without offload at the C2 shape, rank 0
emulated, for several microbatch counts and vocabularies in ONE process (one backend
table): is the split-backward overhead a property of the schedule or of the run?
usage: python tools/gish_m_probe.py > profiles/r2_gish_m_probe.jsonl"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2503_01328_b200 as po  # noqa: E402
from paper_2503_01328_b200.runtime import executor as ex  # noqa: E402
from paper_2503_01328_b200.runtime import gemm_tune  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig  # noqa: E402

dev = torch.device("cuda:0")
for vocab in (50304, 1024):
    cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=vocab)
    gemm_tune.ensure(cfg, dev)
    for m in (16, 32):
        c3 = po.measured_pass_costs(0.35e-3, 0.8e-3, 0.0, 30e-6)
        c1 = po.measured_pass_costs(0.39e-3, 0.53e-3, 0.35e-3, 30e-6)
        for name, sched in (("1f1b", po.build_1f1b(8, 3, m, c3)), ("gis-h", po.build_gis_h(8, 3, m, c1)),
                            ("po", po.build_po(8, 3, m, c1))):
            res = ex.execute(sched, None, model=cfg, mode="emulate", rank=0, device=dev, iters=10, warmup=3,
                             iteration_graph=True, optimizer="sgd")
            it = statistics.median(res.iteration_seconds)
            kinds = {}
            for p in res.trace.compute_passes():
                kinds.setdefault(str(p.kind), []).append(float(p.duration) * 1e3)
            print(json.dumps({"vocab": vocab, "m": m, "schedule": name, "ms_per_step": round(it * 1e3, 3),
                              "tokens_per_s": round(m * cfg.seq / it), "peak_act_gb": res.mem["alloc_peak_bytes"] / 1e9,
                              "pass_ms": {k: round(statistics.mean(v), 4) for k, v in kinds.items()},
                              "iters_ms": [round(x * 1e3, 2) for x in res.iteration_seconds]}), flush=True)
            res.close()
            torch.cuda.empty_cache()
