"""Per-launch device times of a compiled forward, measured inside the real
step: the whole forward is captured as one CUDA graph with an external
event-record node between consecutive launches, so every kernel runs in its
true context (same L2 state, no host gaps, no repetition) and the events
bracket exactly one launch each."""

from __future__ import annotations

import numpy as np


def _rt():
    from cuda.bindings import runtime as rt
    return rt


def _check(res):
    err = res[0] if isinstance(res, tuple) else res
    if int(err) != 0:
        raise RuntimeError(f"CUDA runtime error {err}")
    return res[1] if isinstance(res, tuple) and len(res) > 1 else None


def timed_launches(prog, reps: int = 3, flush=None) -> np.ndarray:
    """Median per-launch milliseconds of ``prog.launches`` over ``reps``
    graph replays (``flush``: optional zero-arg callable run on the program
    stream before each replay, e.g. an L2 flush)."""
    import torch
    from . import device as D
    rt = _rt()
    n = len(prog.launches)
    evs = [_check(rt.cudaEventCreate()) for _ in range(n + 1)]
    st = rt.cudaStream_t(prog.stream.cuda_stream)
    ext = rt.cudaEventRecordExternal

    def body():
        _check(rt.cudaEventRecordWithFlags(evs[0], st, ext))
        for i, fn in enumerate(prog.launches):
            fn()
            _check(rt.cudaEventRecordWithFlags(evs[i + 1], st, ext))

    graph = D.capture(body, prog.stream)
    out = []
    try:
        for r in range(reps + 1):
            if flush is not None:
                with torch.cuda.stream(prog.stream):
                    flush()
            graph.launch(prog.stream)
            prog.stream.synchronize()
            if r:
                out.append([_check(rt.cudaEventElapsedTime(evs[i], evs[i + 1]))
                            for i in range(n)])
    finally:
        del graph
        for e in evs:
            rt.cudaEventDestroy(e)
    return np.median(np.asarray(out, dtype=np.float64), axis=0)


def graph_time(prog, select, reps: int = 3, flush=None) -> float:
    """Median device seconds of one CUDA-graph replay of the launches whose
    index ``select(i)`` accepts, in program order (events around the graph
    launch only: no extra nodes inside)."""
    import torch
    from . import device as D
    fns = [fn for i, fn in enumerate(prog.launches) if select(i)]
    graph = D.capture(lambda: [fn() for fn in fns], prog.stream)
    out = []
    for r in range(reps + 1):
        if flush is not None:
            with torch.cuda.stream(prog.stream):
                flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(prog.stream)
        graph.launch(prog.stream)
        b.record(prog.stream)
        b.synchronize()
        if r:
            out.append(a.elapsed_time(b) * 1e-3)
    del graph
    return float(np.median(out))


__all__ = ["timed_launches", "graph_time"]
