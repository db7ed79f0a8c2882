#!/usr/bin/env python
"""Per-layer block-size planning on the GPU (north_star piece 3, reference
planning.py:360-383 fed with B200-measured costs):

  1. search_pairs: time every GPU-legal (ic_bn, oc_bn) pair of every conv
     workload (plus a few tile variants) -> schedule DB;
  2. planning.plan: exact DP (PBQP on state explosion) over those costs and
     CUDA-event-timed device retiles;
  3. in-context refinement (planning.refine_in_context): the planned and the
     default (blocked_assignment + tuned tiles) programs are timed as whole
     graphed forwards, the faster one is kept and per-workload groups are
     flipped to the other's choice while that makes the forward faster --
     the result is never slower than the default.

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
    ap.add_argument("--trials", type=int, default=16, help="in-context flips to try")
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input, simplify)
    from paper_1809_02697_b200.planning import (SchemeCandidate, SchemePlan, TransformCostTable,
                                                plan)
    from paper_1809_02697_b200.tuning import DEFAULT_DB, search_pairs
    g = build_model(args.model, batch=args.batch)
    db = ScheduleDb(args.db or os.path.join("gpurun_out", f"plan_{args.model}_b{args.batch}.npsd"))
    t0 = time.time()
    key = search_pairs(g, db, args.mode, args.batch, tiles_per_pair=args.tiles_per_pair)
    t1 = time.time()
    sg = simplify(g)
    sp = plan(sg, db, costs=TransformCostTable(mode=args.mode), cpu=key)
    t2 = time.time()
    from paper_1809_02697_b200.planning import refine_in_context
    from paper_1809_02697_b200.passes import blocked_assignment
    from paper_1809_02697_b200.tuning import tuned_assignment
    from paper_1809_02697_b200.kernels import ConvSchedule
    base = tuned_assignment(g, ScheduleDb(DEFAULT_DB), args.mode)
    if base is None:
        base = {nid: (v if isinstance(v, ConvSchedule) else ConvSchedule(v[0], v[1], 8, True))
                for nid, v in blocked_assignment(sg, mode=args.mode).items()}
    best, ms_best, log = refine_in_context(g, sp.schedules(), base, args.mode,
                                          max_trials=args.trials)
    ms_plan, ms_default = log[0][1], log[1][1]
    pairs = {}
    for cand in sp.assignment.values():
        k = f"{cand.schedule.ic_bn}/{cand.schedule.oc_bn}"
        pairs[k] = pairs.get(k, 0) + 1
    row = {"model": args.model, "batch": args.batch, "mode": args.mode, "solver": sp.solver,
           "planned_conv_ns": sp.total_ns, "search_s": round(t1 - t0, 1),
           "plan_s": round(t2 - t1, 2), "step_ms_planned": ms_plan,
           "step_ms_default": ms_default, "step_ms_refined": ms_best,
           "refine_log": log, "pairs": pairs}
    print(json.dumps(row))
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(SchemePlan({nid: SchemeCandidate(nid, sch, 0.0) for nid, sch in best.items()},
                                ms_best * 1e6, sp.solver + "+in-context").to_json())


if __name__ == "__main__":
    main()
