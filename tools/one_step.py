#!/usr/bin/env python
"""Run exactly (warmup + 1) un-graphed forwards of the bench workload so an
ncu launch list can capture one step: ``ncu -s <launches> -c <launches>``.
Prints the number of launches per step."""

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
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--untuned", action="store_true")
    ap.add_argument("--dump", default="", help="write launch names / bytes / flops as JSON")
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model(args.model, batch=args.batch)
    db = None if args.untuned else ScheduleDb(DEFAULT_DB)      # same program as bench.py
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=args.mode, db=db)), 0,
                         args.mode, use_graph=False)
    prog.set_inputs(model_input(g))
    for _ in range(args.warmup):
        prog.launch()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("step")       # ncu --nvtx --nvtx-include "step/"
    prog.launch()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(f"launches_per_step={prog.kernel_launches}")
    if args.dump:
        import json
        with open(args.dump, "w") as fh:
            json.dump([{"name": n, "bytes": b, "flops": f, "desc": d} for n, b, f, d in
                       zip(prog.launch_names, prog.launch_bytes, prog.launch_flops,
                           prog.launch_desc)], fh, indent=1)
    for i, n in enumerate(prog.launch_names):
        print(i, n)


if __name__ == "__main__":
    main()
