#!/usr/bin/env python
"""Concurrent sub-batch chains: split the batch into ``--chains`` independent
sub-batches, each a whole graphed forward on its own stream, and time the
group (CUDA events on a third stream that forks to / joins the chains, L2
flushed between iterations).  With NEOB200_HALF=1 every conv CTA takes half
an SM, so CTAs of two chains are co-resident and one chain's launch fill /
drain phases overlap the other's MMA phases.

  NEOB200_HALF=1 python tools/dual_chain.py --chains 2 --batch 64
  python tools/dual_chain.py --chains 1 --batch 64 --tuned      # the shipped program
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64, help="total batch over all chains")
    ap.add_argument("--chains", type=int, default=2)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--tuned", action="store_true")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--check", action="store_true", help="compare chain outputs with a 1-chain run")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    db = ScheduleDb(DEFAULT_DB) if args.tuned else None
    assert args.batch % args.chains == 0
    sub = args.batch // args.chains
    g = build_model(args.model, batch=sub)
    plan = ExecutablePlan.compile(compile_graph(g, mode=args.mode, db=db))
    progs = [DeviceProgram(plan, 0, args.mode) for _ in range(args.chains)]
    feeds = model_input(g)
    for p in progs:
        p.set_inputs(feeds)
        p.launch()
        p.stream.synchronize()
    main_s = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    times = []
    for it in range(args.iters + 3):
        with torch.cuda.stream(main_s):
            flush.fill_(it & 1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main_s)
        for p in progs:
            p.stream.wait_event(a)
            p.launch()
            done = torch.cuda.Event()
            done.record(p.stream)
            main_s.wait_event(done)
        b.record(main_s)
        b.synchronize()
        if it >= 3:
            times.append(a.elapsed_time(b))
    ms = float(np.median(times))
    print(f"{args.model} b{args.batch} {args.mode} chains={args.chains} (sub-batch {sub}) "
          f"half={os.environ.get('NEOB200_HALF', '0')} tuned={args.tuned}: "
          f"{ms:.4f} ms/step (min {min(times):.4f}), {args.batch / ms * 1e3:.0f} img/s, "
          f"{progs[0].kernel_launches} launches per chain", flush=True)
    if args.check:
        outs = [p.output_tensors()[0].float().cpu().numpy() for p in progs]
        for o in outs[1:]:
            assert np.array_equal(o, outs[0]), "chains disagree"
        print("chains agree bitwise; top-1 of image 0:", int(outs[0][0].argmax()))


if __name__ == "__main__":
    main()
