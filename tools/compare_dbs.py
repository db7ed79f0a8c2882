#!/usr/bin/env python
"""Graphed-step time of a model compiled with each of several schedule DBs
(L2 flushed before every replay; medians of 30):

  python tools/compare_dbs.py --model resnet50 --batch 64 a.npsd b.npsd
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
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("dbs", nargs="+")
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    g = build_model(args.model, batch=args.batch)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    for name in args.dbs * 2:
        prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=args.mode,
                                                                  db=ScheduleDb(name))),
                             0, args.mode)
        prog.set_inputs(model_input(g))
        for _ in range(5):
            prog.launch()
        prog.stream.synchronize()
        ts = []
        for _ in range(30):
            with torch.cuda.stream(prog.stream):
                flush.fill_(0.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(prog.stream)
            prog.launch()
            b.record(prog.stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{name}: median {ts[len(ts) // 2]:.4f} ms, min {ts[0]:.4f} ms")
        del prog


if __name__ == "__main__":
    main()
