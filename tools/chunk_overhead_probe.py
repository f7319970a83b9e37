"""Where a 1-layer chunk pass (GIS-H / PO at v = layers per stage) loses time against
the same layer inside a 3-layer stage: pass time per layer (CUDA events, CUDA-graph
replay) and the kernel list of one pass (torch.profiler / CUPTI, device times).

usage: python tools/chunk_overhead_probe.py > profiles/r2_chunk_overhead.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_01328_b200.runtime import gemm_tune  # noqa: E402
from paper_2503_01328_b200.runtime.model import ModelConfig, SlabView, Stage  # noqa: E402

DEV = torch.device("cuda:0")
cfg = ModelConfig(n_layers=24, hidden=2048, heads=16, seq=4096, vocab=50304)
gemm_tune.ensure(cfg, DEV)


def graph_ms(fn, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
        b.synchronize()
    return a.elapsed_time(b) / reps


def kernels(fn, label):
    from torch.profiler import ProfilerActivity, profile

    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    tot = sum(e.device_time for e in evs)
    print(f"--- {label}: {len(evs)} device ops, {tot / 1e3:.3f} ms device time")
    agg = {}
    for e in evs:
        k = e.name[:70]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {t / 1e3:8.3f} ms  x{n:3d}  {k}")


def probe(n_layers, split):
    st = Stage(cfg, 8, 24, 32, DEV, layers=list(range(8, 8 + n_layers)))  # a middle stage
    slab = SlabView(st.layout, torch.empty(st.layout.slab_bytes, dtype=torch.uint8, device=DEV))
    x_in = (torch.randn(cfg.seq, cfg.hidden, device=DEV) * 0.5).bfloat16()
    out = torch.empty_like(x_in)
    dy = (torch.randn(cfg.seq, cfg.hidden, device=DEV) * 1e-3).bfloat16()
    dx = torch.empty_like(x_in)
    wbuf = st.new_wbuffer() if split else None
    st.set_pass_context(0, 0)

    def fwd():
        slab.get(0, "x").copy_(x_in)
        st.forward_body(slab, out)

    def bwd():
        st.backward_body(slab, dy, dx, wbuf)

    def w():
        st.wgrad_body(slab, wbuf)

    fwd()
    res = {"F": graph_ms(fwd), "B": graph_ms(bwd)}
    if split:
        res["W"] = graph_ms(w)
    per_layer = {k: round(v / n_layers, 4) for k, v in res.items()}
    print(f"=== {n_layers}-layer stage, split={split}: pass ms {dict((k, round(v, 4)) for k, v in res.items())}, "
          f"per layer {per_layer}")
    kernels(fwd, f"F ({n_layers} layers)")
    kernels(bwd, f"B ({n_layers} layers, split={split})")
    if split:
        kernels(w, f"W ({n_layers} layers)")
    del st, slab
    torch.cuda.empty_cache()


for n, split in ((3, False), (3, True), (1, True), (1, False)):
    probe(n, split)
