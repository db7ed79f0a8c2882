#!/usr/bin/env python
"""Per-launch in-graph times (timing.timed_launches, L2 flushed) as JSON:
  python tools/per_launch.py --model resnet50 --batch 64 [--untuned] > out.json
Used to compare kernel modes launch by launch (e.g. NEOB200_HALF=1)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--untuned", action="store_true")
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.timing import timed_launches
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model(args.model, batch=args.batch)
    db = None if args.untuned else ScheduleDb(DEFAULT_DB)
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=args.mode, db=db)), 0,
                         args.mode)
    prog.set_inputs(model_input(g))
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    ms = timed_launches(prog, args.reps, lambda: flush.zero_())
    print(json.dumps({"names": prog.launch_names, "desc": prog.launch_desc,
                      "us": [t * 1e3 for t in ms]}))


if __name__ == "__main__":
    main()
