#!/usr/bin/env python
"""Time one pooling configuration on the blocked layout (CUDA events).

  python tools/pool_bench.py --n 128 --c 192 --hw 35 --x 16 --win 3 --stride 1 --pad 1 --mode avg
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--c", type=int, default=192)
    ap.add_argument("--hw", type=int, default=35)
    ap.add_argument("--x", type=int, default=16)
    ap.add_argument("--win", type=int, default=3)
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--pad", type=int, default=1)
    ap.add_argument("--mode", default="avg")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_1809_02697_b200 import device as D
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    n, cb, hw, x = args.n, args.c // args.x, args.hw, args.x
    oh = (hw + 2 * args.pad - args.win) // args.stride + 1
    src = torch.randn((n, cb, hw, hw, x), device="cuda").to(dt)
    out = torch.empty((n, cb, oh, oh, x), device="cuda", dtype=dt)
    run = lambda: D.pool2d(src, out, n, cb, hw, hw, x, args.win, args.stride, args.pad, args.mode)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.iters):
        run()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) * 1e3 / args.iters
    byts = (src.numel() + out.numel()) * src.element_size()
    print(f"{args.mode}pool n{n} c{args.c} {hw}x{hw} x{x} win{args.win}/s{args.stride}/p{args.pad}: "
          f"{us:.1f} us  {byts / us / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
