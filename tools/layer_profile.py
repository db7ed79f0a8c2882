#!/usr/bin/env python
"""Per-launch device-time breakdown of one compiled forward (CUDA events
around every launch on the executor stream).  Prints one row per launch
with the conv workload, tile config, time, TFLOP/s and algorithmic GB/s,
and writes the table as JSON (``--out``)."""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="")
    ap.add_argument("--untuned", action="store_true")
    ap.add_argument("--isolated", action="store_true",
                    help="time each launch alone (repeated, L2-warm) instead of in the step")
    args = ap.parse_args()

    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200 import device as D
    from paper_1809_02697_b200.graph import hw_pair, infer_shapes

    from paper_1809_02697_b200 import ScheduleDb
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    g = build_model(args.model, batch=args.batch)
    planned = compile_graph(g, mode=args.mode, db=None if args.untuned else ScheduleDb(DEFAULT_DB))
    prog = DeviceProgram(ExecutablePlan.compile(planned), 0, args.mode, use_graph=False)
    prog.set_inputs(model_input(g))
    specs = infer_shapes(planned)
    es = 2 if args.mode == "bf16" else 4
    info = {}
    for nid, node in planned.nodes.items():
        if node.kind.value != "Conv2d":
            continue
        _, c, h, w = specs[node.inputs[0][0]].logical_nchw
        _, k, oh, ow = specs[nid].logical_nchw
        wt = planned.nodes[node.inputs[1][0]].attrs["value"]
        r, s = wt.shape[2], wt.shape[3]
        n = args.batch
        flops = 2 * n * k * c * r * s * oh * ow
        byts = es * (n * c * h * w + k * c * r * s + n * k * oh * ow *
                     (2 if (node.attrs.get("epilogue") or {}).get("residual") else 1))
        sch = node.attrs.get("schedule") or {}
        tile = "/".join(str(sch.get(f, 0)) for f in ("tile_n", "slices_per_stage", "stages"))
        info[f"conv{nid}"] = dict(c=c, k=k, h=h, w=w, r=r, s=s, tile=tile,
                                  stride=hw_pair(node.attrs["stride"])[0], flops=flops,
                                  bytes=byts)
    # tile config the kernel picks
    prog.launch()
    prog.stream.synchronize()
    if args.isolated:
        # each launch timed as a CUDA graph of `inner` back-to-back copies (no
        # host overhead; operands L2-warm after the first copy)
        inner = 10
        times = np.zeros((args.reps, len(prog.launches)))
        graphs = [D.capture(lambda fn=fn: [fn() for _ in range(inner)], prog.stream)
                  for fn in prog.launches]
        for rep in range(args.reps + 1):
            evs = []
            for gr in graphs:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(prog.stream)
                gr.launch(prog.stream)
                b.record(prog.stream)
                evs.append((a, b))
            prog.stream.synchronize()
            if rep:
                times[rep - 1] = [a.elapsed_time(b) * 1e3 / inner for a, b in evs]
        med = np.median(times, axis=0)
    else:
        # in the real step: one graph of the whole forward with event-record
        # nodes between launches, L2 flushed before each replay
        from paper_1809_02697_b200.timing import timed_launches
        flush = torch.empty(64 * 1024 * 1024, device=prog.device)
        med = timed_launches(prog, args.reps, flush=lambda: flush.fill_(0.0)) * 1e3
    rows = []
    total = med.sum()
    for name, t in zip(prog.launch_names, med):
        row = {"launch": name, "us": float(t)}
        if name in info:
            d = info[name]
            row.update(d)
            row["tflops"] = d["flops"] / (t * 1e-6) / 1e12
            row["gbs"] = d["bytes"] / (t * 1e-6) / 1e9
        rows.append(row)
    print(f"total {total:.1f} us over {len(rows)} launches")
    agg = {}
    for row in rows:
        key = row["launch"].rstrip("0123456789_simt").rstrip("0123456789")
        kind = "conv" if row["launch"].startswith("conv") else row["launch"].rstrip("0123456789")
        agg[kind] = agg.get(kind, 0.0) + row["us"]
    print("by kind:", {k: round(v, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])})
    for row in rows:
        if "flops" in row:
            print(f"{row['launch']:>10} C{row['c']:>5} K{row['k']:>5} {row['h']:>3}x{row['w']:<3} "
                  f"{row['r']}x{row['s']} s{row['stride']} {row['us']:8.1f} us "
                  f"{row['tflops']:7.1f} TF/s {row['gbs']:7.0f} GB/s {row.get('tile', '')}")
        else:
            print(f"{row['launch']:>10} {row['us']:8.1f} us")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"model": args.model, "batch": args.batch, "mode": args.mode,
                       "total_us": float(total), "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
