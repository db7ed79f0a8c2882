#!/usr/bin/env python
"""In-context tile selection: per distinct conv workload, the top-K tile
configurations of the isolated per-layer search (tools/tune_model.py) are
re-timed inside the whole graphed forward (L2 flushed before every replay)
and the fastest kept -- greedy coordinate descent over workloads, since a
layer's best tile in isolation is often not its best next to its neighbours
(PDL overlap, L2 state, tile-count interplay).  The winner of each workload is
written back as the first (lowest mean_ns) entry of its block pair:

  python tools/tune_in_context.py --model resnet50 --batch 64 --db schedules.npsd [--k 6]
"""

from __future__ import annotations

import argparse
import copy
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--db", required=True)
    ap.add_argument("--k", type=int, default=6, help="isolated top-K candidates per workload")
    ap.add_argument("--reps", type=int, default=25)
    ap.add_argument("--min-gain", type=float, default=0.002, help="relative step-time gain to accept")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.passes import blocked_assignment, simplify
    from paper_1809_02697_b200.planning import conv_workloads
    from paper_1809_02697_b200.tuning import tuning_key

    db = ScheduleDb(args.db)
    g = build_model(args.model, batch=args.batch)
    s = simplify(g)
    pairs = blocked_assignment(s, mode=args.mode)
    key = tuning_key(args.mode, args.batch)
    wls = {}
    for nid, wl in conv_workloads(s).items():
        wls.setdefault((wl, pairs[nid]), []).append(nid)
    feeds = model_input(g)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")

    def schemes_of(d, wl, pair):
        return [m for m in (d.get(key, wl) or []) if (m.schedule.ic_bn, m.schedule.oc_bn) == pair]

    def with_choice(base, wl, pair, chosen):
        """copy of ``base`` whose best entry for (wl, pair) is ``chosen``"""
        d = ScheduleDb(None)
        d._data = copy.deepcopy(base._data)
        ms = schemes_of(d, wl, pair)
        lo = min(m.mean_ns for m in ms)
        others = [m for m in (d.get(key, wl) or []) if m not in ms]
        for m in ms:
            if m.schedule == chosen.schedule:
                m.mean_ns = lo * 0.999
        d._data[(key, __import__("json").dumps(wl.key()))] = sorted(ms + others,
                                                                     key=lambda m: m.mean_ns)
        return d

    # fp8: calibrate once, every trial program reuses the scales
    scales = None
    if args.mode == "fp8":
        from paper_1809_02697_b200.quant import calibrate
        scales = calibrate(g)

    from paper_1809_02697_b200.errors import ScheduleInvalid

    def step_ms(d) -> float:
        kw = {"fp8_scales": scales} if scales is not None else {}
        prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=args.mode, db=d, **kw)),
                             0, args.mode)
        prog.set_inputs(feeds)
        try:
            prog.launch()
        except ScheduleInvalid as exc:
            # a stored candidate the kernel no longer accepts (e.g. measured as a
            # plain tile before its row format joined the halo mainloop)
            print(f"  skipped: {str(exc)[:120]}")
            del prog
            return float("inf")
        for _ in range(2):
            prog.launch()
        prog.stream.synchronize()
        ts = []
        for _ in range(args.reps):
            with torch.cuda.stream(prog.stream):
                flush.fill_(0.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(prog.stream)
            prog.launch()
            b.record(prog.stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        del prog
        return float(np.median(ts))

    t0 = time.time()
    cur = db
    best = min(step_ms(cur) for _ in range(2))
    print(f"start: {best:.4f} ms")
    # largest layers first (most time at stake): order by isolated best time x count
    order = sorted(wls, key=lambda kp: -min((m.mean_ns for m in schemes_of(db, *kp)), default=0)
                   * len(wls[kp]))
    for wl, pair in order:
        ms = sorted(schemes_of(cur, wl, pair), key=lambda m: m.mean_ns)
        if len(ms) < 2:
            continue
        incumbent = ms[0]
        for cand in ms[1:args.k]:
            trial = with_choice(cur, wl, pair, cand)
            t = min(step_ms(trial) for _ in range(2))
            if t < best * (1 - args.min_gain):
                print(f"  {wl.key()} {pair}: {cand.schedule.tile()} {best:.4f} -> {t:.4f} ms")
                best, cur, incumbent = t, trial, cand
        torch.cuda.empty_cache()
    print(f"final: {best:.4f} ms after {time.time() - t0:.0f}s")
    out = ScheduleDb(args.db)
    out._data = cur._data
    out._save()


if __name__ == "__main__":
    main()
