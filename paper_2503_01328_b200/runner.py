"""Drop-in measured runner with the reference's ``simulate`` signature.

Reference boundary (``pkg/src/ppoff/sim.py:141-149``)::

    simulate(sched, plan=None, costs=None, hw=None, contention=None, model=None,
             stream_mode="single") -> SimTrace

``execute`` takes the same arguments and returns a ``MeasuredTrace`` -- a ``SimTrace``
(same fields, so ``peak_memory``, ``bubble_time``, ``summary()``, ``to_csv()`` and the
reference's ``analysis`` / ``render`` consume it unchanged) whose pass times are CUDA
measurements in seconds on the B200, plus:

* ``run``: the runtime's ``RunResult`` (per-iteration times, losses, measured
  activation memory, lowered programs);
* ``predicted``: the reference runner model's trace for the same inputs (``simulate``
  with the given ``costs`` / ``hw`` / ``contention``), for predicted-vs-measured.

``costs`` / ``hw`` / ``contention`` only feed ``predicted``: the measured run has
the machine's real compute rates and link contention.  ``model`` (a ``ModelSpec``:
hidden h, sequence s, microbatch b, layers per stage) sizes the transformer the
run trains (b must be 1, bf16); pass ``config=ModelConfig(...)`` to set heads /
vocabulary / dropout explicitly.  Runtime options (``mode``, ``iters``, ``warmup``,
``gemm``, ``attn``, ``iteration_graph``, ...) are keywords of
``runtime.executor.execute``.

``runner(**fixed)`` returns a callable with exactly ``simulate``'s signature, so code
written against the reference -- e.g. ``ppoff.analysis.reduction_curve``, which calls
``simulate(sched)`` / ``simulate(sched, plan)`` (analysis.py:161-165) -- runs over
measured traces by rebinding one name.
"""

from __future__ import annotations

from dataclasses import dataclass

from .costs import ModelSpec
from .sim import SimTrace, simulate

DEFAULT_VOCAB = 50304


@dataclass(frozen=True)
class MeasuredTrace(SimTrace):
    run: object = None
    predicted: SimTrace | None = None


def config_from_spec(model: ModelSpec, num_stages: int, heads: int | None = None, vocab: int = DEFAULT_VOCAB):
    """ModelConfig of the GPT the run trains, from the reference's ``ModelSpec``."""
    from .runtime.model import ModelConfig

    if model.microbatch_size != 1:
        raise ValueError("the B200 runtime runs microbatch_size 1 (b=1, SURVEY 8(d))")
    if model.bytes_per_element != 2:
        raise ValueError("the B200 runtime stores activations in bf16 (bytes_per_element=2)")
    h = model.hidden_size
    if heads is None:
        heads = h // 128 if h % 128 == 0 else max(1, h // 64)
    return ModelConfig(n_layers=model.layers_per_stage * num_stages, hidden=h, heads=heads,
                       seq=model.sequence_length, vocab=vocab)


def execute(sched, plan=None, costs=None, hw=None, contention=None, model: ModelSpec | None = None,
            stream_mode: str = "single", *, config=None, predict: bool = True, **runtime) -> MeasuredTrace:
    """Run ``sched`` (+ ``plan``) on the GPU and return its measured trace (see module doc)."""
    from .runtime import executor

    if config is None:
        if model is None:
            raise ValueError("execute needs model=ModelSpec(...) or config=ModelConfig(...)")
        config = config_from_spec(model, sched.num_stages)
    runtime.setdefault("mode", "virtual")
    res = executor.execute(sched, plan, model=config, stream_mode=stream_mode, **runtime)
    predicted = simulate(sched, plan, costs, hw, contention, model, stream_mode) if predict else None
    t = res.trace
    return MeasuredTrace(schedule=t.schedule, passes=t.passes, makespan=t.makespan, device_busy=t.device_busy,
                         memory=t.memory, host_events=t.host_events, contention_log=t.contention_log,
                         bytes_per_unit=t.bytes_per_unit, run=res, predicted=predicted)


def runner(**fixed):
    """A ``simulate``-signature callable bound to runtime options (``config=``, ``mode=``,
    ``iters=``, ...): ``analysis.simulate = runner(config=cfg)`` points the reference's
    analysis layer at measured traces."""

    def simulate_measured(sched, plan=None, costs=None, hw=None, contention=None, model=None, stream_mode="single"):
        tr = execute(sched, plan, costs, hw, contention, model, stream_mode, **fixed)
        tr.run.close()  # release pinned pools / arenas; the trace keeps the measurements
        return tr

    return simulate_measured
