#!/bin/bash
# C2 shape (24 layers, h=2048, s=4096, PP=8, m=32), rank 0 emulated: 1F1B vs the
# split-backward schedules (GIS-H, PO) and interleaved 1F1B at v=3 (1-layer chunks),
# without offload and with the reference's selective n=1 on duplex copy streams.
# One summary JSON per run under $OUT/<name>/.
OUT=${OUT:-gpurun_out/sched_c2}
COMMON="--d 8 --m 32 --layers 24 --hidden 2048 --heads 16 --seq 4096 --vocab 50304 --mode emulate --iters 3 --warmup 2 ${EXTRA:-}"
run() { name=$1; shift; timeout 600 python -m paper_2503_01328_b200 run $COMMON "$@" --out $OUT/$name > $OUT.$name.log 2>&1; echo "$name rc=$?"; }
mkdir -p $OUT
run 1f1b_none --schedule 1f1b --offload none
run po3_none --schedule po --v 3 --offload none
run po3_n1_duplex --schedule po --v 3 --offload 1 --planner duplex --stream-mode dual
run gish3_none --schedule gis-h --v 3 --offload none
run gish3_n1_duplex --schedule gis-h --v 3 --offload 1 --planner duplex --stream-mode dual
run i3_none --schedule 1f1b-i --v 3 --offload none
run i3_n1_duplex --schedule 1f1b-i --v 3 --offload 1 --planner duplex --stream-mode dual
python - <<'PY'
import glob, json, os
out = os.environ.get("OUT", "gpurun_out/sched_c2")
for f in sorted(glob.glob(f"{out}/*/*-summary.json")):
    d = json.load(open(f))
    print(os.path.basename(os.path.dirname(f)), "tok/s %.0f" % d["tokens_per_s"], "ms %.1f" % d["ms_per_step"],
          "arena_gb", d["arena_gb"], "model_peak", d["modelled_peak_units"][0], "pred_ms %.1f" % (d["predicted_makespan_s"] * 1e3))
PY
