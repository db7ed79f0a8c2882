#!/usr/bin/env python
"""Device-resident images/s of every BASELINE model family at its configured
batch sizes (one GPU, CUDA events around CUDA-graph replays, L2 flushed
between steps).  Writes a JSON table (``--out``)."""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CONFIGS = [("resnet18", 1), ("resnet18", 64), ("resnet50", 1), ("resnet50", 64),
           ("vgg16", 1), ("vgg16", 128), ("inception_v3", 1), ("inception_v3", 128),
           ("densenet201", 1), ("densenet201", 32), ("ssd_resnet50", 1), ("ssd_resnet50", 32)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default="")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.models import conv_flops
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    db = ScheduleDb(DEFAULT_DB)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    rows = []
    for name, batch in CONFIGS:
        if args.only and name not in args.only.split(","):
            continue
        g = build_model(name, batch=batch)
        prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=args.mode, db=db)), 0,
                             args.mode)
        prog.set_inputs(model_input(g))
        for _ in range(3):
            prog.launch()
        prog.stream.synchronize()
        total = 0.0
        for _ in range(args.steps):
            with torch.cuda.stream(prog.stream):
                flush.fill_(0.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(prog.stream)
            prog.launch()
            b.record(prog.stream)
            b.synchronize()
            total += a.elapsed_time(b) * 1e-3
        ms = 1e3 * total / args.steps
        fl = conv_flops(g)
        row = {"model": name, "batch": batch, "mode": args.mode, "ms_per_batch": ms,
               "images_per_s": batch / (ms * 1e-3), "conv_tflops": fl / (ms * 1e-3) / 1e12,
               "launches": prog.kernel_launches, "arena_mb": prog.arena_bytes / 1e6}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del prog
        torch.cuda.empty_cache()
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
