#!/usr/bin/env python
"""Per-layer block-size planning on the GPU (north_star piece 3, reference
planning.py:360-383 fed with B200-measured costs):

  1. search_pairs: time every GPU-legal (ic_bn, oc_bn) pair of every conv
     workload (plus a few tile variants) -> schedule DB;
  2. planning.plan: exact DP (PBQP on state explosion) over those costs and
     CUDA-event-timed device retiles;
  3. compile the planned graph and compare its graphed step time with the
     default (blocked_assignment + tuned tiles) program.

  python tools/plan_model.py --model inception_v3 --batch 128 --out plan.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def step_ms(prog, flush, reps=20):
    import torch
    for _ in range(3):
        prog.launch()
    prog.stream.synchronize()
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(prog.stream):
            flush.fill_(0.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(prog.stream)
        prog.launch()
        b.record(prog.stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="inception_v3")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--db", default=None, help="schedule DB (default: a scratch file)")
    ap.add_argument("--tiles-per-pair", type=int, default=6)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input, simplify)
    from paper_1809_02697_b200.planning import TransformCostTable, plan
    from paper_1809_02697_b200.tuning import DEFAULT_DB, search_pairs
    g = build_model(args.model, batch=args.batch)
    db = ScheduleDb(args.db or os.path.join("gpurun_out", f"plan_{args.model}_b{args.batch}.npsd"))
    t0 = time.time()
    key = search_pairs(g, db, args.mode, args.batch, tiles_per_pair=args.tiles_per_pair)
    t1 = time.time()
    sg = simplify(g)
    sp = plan(sg, db, costs=TransformCostTable(mode=args.mode), cpu=key)
    t2 = time.time()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    feeds = model_input(g)
    planned = DeviceProgram(ExecutablePlan.compile(compile_graph(g, assign=sp.schedules(),
                                                                 mode=args.mode)), 0, args.mode)
    planned.set_inputs(feeds)
    ms_plan = step_ms(planned, flush)
    del planned
    default = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=args.mode,
                                                                 db=ScheduleDb(DEFAULT_DB))),
                            0, args.mode)
    default.set_inputs(feeds)
    ms_default = step_ms(default, flush)
    pairs = {}
    for cand in sp.assignment.values():
        k = f"{cand.schedule.ic_bn}/{cand.schedule.oc_bn}"
        pairs[k] = pairs.get(k, 0) + 1
    row = {"model": args.model, "batch": args.batch, "mode": args.mode, "solver": sp.solver,
           "planned_conv_ns": sp.total_ns, "search_s": round(t1 - t0, 1),
           "plan_s": round(t2 - t1, 2), "step_ms_planned": ms_plan,
           "step_ms_default": ms_default, "pairs": pairs}
    print(json.dumps(row))
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(sp.to_json())


if __name__ == "__main__":
    main()
