#!/usr/bin/env python
"""Graphed-step time of the bench program (tuned tile DB, L2 flushed before
every replay, median of 30) in each requested mode:

  python tools/step_times.py --model resnet50 --batch 64 --modes bf16,tf32,fp8
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--modes", default="bf16,tf32,fp8")
    ap.add_argument("--untuned", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model(args.model, batch=args.batch)
    db = None if args.untuned else ScheduleDb(DEFAULT_DB)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    for mode in args.modes.split(","):
        prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=mode, db=db)), 0, mode)
        prog.set_inputs(model_input(g))
        for _ in range(3):
            prog.launch()
        ts = []
        for _ in range(30):
            with torch.cuda.stream(prog.stream):
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(prog.stream)
            prog.launch()
            b.record(prog.stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        print(f"{args.model} b{args.batch} {mode}: {ms:.4f} ms/step, {args.batch / ms * 1e3:.0f} img/s")
        del prog


if __name__ == "__main__":
    main()
