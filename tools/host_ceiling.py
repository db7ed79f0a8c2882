#!/usr/bin/env python
"""Host-side ceiling of the end-to-end serving loop at 1..8 ranks on one box.

Every rank of an 8-GPU run feeds its GPU from the same host: with host
rounding (bench.py --upload bf16) each rank reads 38.5 MB of f32 and writes
19.3 MB of bf16 per 64-image batch on the CPU before its DMA; with --upload
f32 the host does no compute and the DMA reads 38.5 MB.  This tool measures,
with P = 1, 2, 4, 8 concurrent processes:

  * host rounding: pinned f32 batch -> pinned bf16 (torch, RN), batches/s per
    process and aggregate;
  * pinned host -> device copies of one batch (f32 and bf16) from rank 0 to
    GPU 0 (the single-GPU link; on an 8-GPU box every GPU has its own link).

and prints the images/s each P could sustain per rank through host rounding,
next to the device step rate -- the number that says whether host rounding
caps multi-GPU e2e scaling.

  python tools/host_ceiling.py [--seconds 3]
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import time

SHAPE = (64, 3, 224, 224)


def _rounder(seconds: float, threads: int, q):
    import torch
    torch.set_num_threads(threads)
    src = torch.randn(SHAPE).pin_memory()
    dst = torch.empty(SHAPE, dtype=torch.bfloat16).pin_memory()
    dst.copy_(src)
    n = 0
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        dst.copy_(src)
        n += 1
    q.put(n / (time.perf_counter() - t0))


def copy_bandwidth(dtype, reps: int = 20) -> float:
    import torch
    src = torch.randn(SHAPE).to(dtype).pin_memory()
    dst = torch.empty(SHAPE, dtype=dtype, device="cuda")
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    b.record()
    b.synchronize()
    return src.numel() * src.element_size() * reps / (a.elapsed_time(b) * 1e-3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    args = ap.parse_args()
    ctx = mp.get_context("spawn")
    out = {"batch": list(SHAPE), "rounding": {}}
    for p in (1, 2, 4, 8):
        q = ctx.Queue()
        import os
        threads = max(1, (os.cpu_count() or 2) // 2 // p)     # physical cores split over ranks
        procs = [ctx.Process(target=_rounder, args=(args.seconds, threads, q)) for _ in range(p)]
        for pr in procs:
            pr.start()
        rates = [q.get(timeout=120) for _ in procs]
        for pr in procs:
            pr.join()
        out["rounding"][p] = {"threads_per_rank": threads,
                              "batches_per_s_per_rank": min(rates),
                              "images_per_s_per_rank": 64 * min(rates),
                              "host_GBps_aggregate": sum(rates) * (38.5 + 19.3) / 1e3}
    try:
        out["h2d_GBps_f32"] = copy_bandwidth(__import__("torch").float32)
        out["h2d_GBps_bf16"] = copy_bandwidth(__import__("torch").bfloat16)
    except Exception as exc:       # no GPU
        out["h2d"] = f"unavailable: {type(exc).__name__}"
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
