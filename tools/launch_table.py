#!/usr/bin/env python
"""In-graph per-launch times of any model / mode (event-bracketed graph
replays, L2 flushed before each replay), grouped by launch kind:

  python tools/launch_table.py --model densenet201 --batch 32 --mode fp8
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--top", type=int, default=12)
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.timing import timed_launches
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model(args.model, batch=args.batch)
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=args.mode,
                                                              db=ScheduleDb(DEFAULT_DB))),
                         0, args.mode)
    prog.set_inputs(model_input(g))
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    ms = timed_launches(prog, 5, lambda: flush.zero_())
    groups = collections.defaultdict(lambda: [0, 0.0, 0])
    for name, t, nb in zip(prog.launch_names, ms, prog.launch_bytes):
        kind = name.rstrip("0123456789_").split("_")[0].rstrip("0123456789+>")
        gk = groups[kind]
        gk[0] += 1
        gk[1] += t * 1e3
        gk[2] += nb
    tot = sum(v[1] for v in groups.values())
    print(f"{args.model} b{args.batch} {args.mode}: {len(prog.launches)} launches, "
          f"{tot:.1f} us event-bracketed")
    for k, (n, us, nb) in sorted(groups.items(), key=lambda kv: -kv[1][1]):
        print(f"  {k:10s} {n:4d} launches {us:8.1f} us  {nb / max(us, 1e-9) / 1e3:7.0f} GB/s alg")
    rows = sorted(zip(ms, prog.launch_names, prog.launch_desc), reverse=True)[:args.top]
    for t, name, desc in rows:
        print(f"    {name:18s} {t * 1e3:7.1f} us  {desc}")


if __name__ == "__main__":
    main()
