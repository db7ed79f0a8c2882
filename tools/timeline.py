#!/usr/bin/env python
"""In-graph per-launch timelines of the tensor-core convs of one graphed
forward (debug build flag NEOB200_DBG=256: every conv CTA stamps globaltimer
at entry, past griddepcontrol.wait, first MMA, last MMA commit and exit).
Prints per launch: start (first CTA entry), wait release, first/last MMA,
exit spread, and the gap to the next launch -- where a step's time goes
between and inside kernels.

  NEOB200_DBG=256 python tools/timeline.py [--model resnet50 --batch 64]
"""

from __future__ import annotations

import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--untuned", action="store_true")
    args = ap.parse_args()
    assert int(os.environ.get("NEOB200_DBG", "0")) & 256, "set NEOB200_DBG=256"
    import numpy as np
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model(args.model, batch=args.batch)
    db = None if args.untuned else ScheduleDb(DEFAULT_DB)
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode="bf16", db=db)), 0, "bf16")
    prog.set_inputs(model_input(g))
    names = [n for n in prog.launch_names if n.startswith("conv") and "simt" not in n]
    C = len(names)
    assert C <= 64
    flush = torch.empty(64 << 20, device="cuda")
    prog.launch()                 # warm-up (slots 0..C-1) + capture (slots C..2C-1)
    for _ in range(3):
        with torch.cuda.stream(prog.stream):
            flush.fill_(1.0)
        prog.launch()
    prog.stream.synchronize()
    lib = L.load()
    n = 64 * 160 * 5
    buf = (ctypes.c_ulonglong * n)()
    lib.neo_dbg_timeline(buf, n)
    tl = np.frombuffer(buf, dtype=np.uint64).reshape(64, 160, 5).astype(np.float64)
    rows = []
    for j, name in enumerate(names):
        s = (C + j) % 64
        v = tl[s]
        ok = v[:, 0] > 0
        v = v[ok]
        rows.append((name, v))
    t0 = min(r[1][:, 0].min() for r in rows)
    print(f"{'launch':>14s} {'ctas':>4s} {'entry':>8s} {'wait_out':>8s} {'mma0':>8s} "
          f"{'mma_end_med':>11s} {'exit_min':>8s} {'exit_max':>8s} {'span':>6s} {'gap':>6s}")
    prev_exit = None
    tot_gap = 0.0
    for name, v in rows:
        us = (v - t0) / 1000.0
        entry, wait, m0, m1, ex = us[:, 0], us[:, 1], us[:, 2], us[:, 3], us[:, 4]
        m0v = m0[us[:, 2] > 0] if (us[:, 2] > 0).any() else m0
        gap = (wait.min() - prev_exit) if prev_exit is not None else 0.0
        tot_gap += max(gap, 0.0)
        print(f"{name:>14s} {len(v):4d} {entry.min():8.2f} {wait.min():8.2f} {m0v.min():8.2f} "
              f"{np.median(m1):11.2f} {ex.min():8.2f} {ex.max():8.2f} {ex.max() - wait.min():6.2f} "
              f"{gap:6.2f}")
        prev_exit = ex.max()
    print(f"sum of gaps (prev launch's last exit -> this launch's wait release): {tot_gap:.1f} us")


if __name__ == "__main__":
    main()
