#!/usr/bin/env python
"""Time one tensor-core conv configuration (CUDA events), optionally sweeping
tile configurations.  Used for ncu captures and tile exploration.

  python tools/conv_bench.py --n 64 --c 64 --k 256 --hw 56 --r 1 [--res] [--sweep]
"""

from __future__ import annotations

import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--c", type=int, default=64)
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--hw", type=int, default=56)
    ap.add_argument("--r", type=int, default=1)
    ap.add_argument("--s", type=int, default=0, help="kernel width (default = r)")
    ap.add_argument("--h", type=int, default=0, help="input height (default = hw)")
    ap.add_argument("--w", type=int, default=0, help="input width (default = hw)")
    ap.add_argument("--stride-w", type=int, default=0)
    ap.add_argument("--pad-h", type=int, default=-1)
    ap.add_argument("--pad-w", type=int, default=-1)
    ap.add_argument("--stride", type=int, default=1)
    ap.add_argument("--x", type=int, default=64)
    ap.add_argument("--y", type=int, default=64)
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--res", action="store_true")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--tile", default="", help="json dict of tile fields")
    ap.add_argument("--flat", action="store_true", help="1x1 conv as a 1 x (H*W) image")
    ap.add_argument("--once", action="store_true", help="one plain launch (tracing)")
    ap.add_argument("--prologue", action="store_true", help="BN-ReLU prologue on the input")
    ap.add_argument("--strips", action="store_true",
                    help="explicit --tile geometry is a halo strip (tile_w = band width)")
    args = ap.parse_args()

    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D

    dev = torch.device("cuda:0")
    act = {"bf16": torch.bfloat16, "fp8": torch.float8_e4m3fn}.get(args.mode, torch.float32)
    lmode = {"bf16": L.MODE_BF16, "fp8": L.MODE_FP8}.get(args.mode, L.MODE_TF32)
    n, c, k, hw, r, st = args.n, args.c, args.k, args.hw, args.r, args.stride
    s_ = args.s or r
    H, W = args.h or hw, args.w or hw
    sw = args.stride_w or st
    ph = args.pad_h if args.pad_h >= 0 else r // 2
    pw = args.pad_w if args.pad_w >= 0 else s_ // 2
    oh = (H + 2 * ph - r) // st + 1
    ow = (W + 2 * pw - s_) // sw + 1
    x = torch.randn((n, -(-c // args.x), H, W, args.x), device=dev).to(act)
    w = torch.randn((k, c, r, s_), device=dev) * 0.05
    if args.mode == "fp8":
        wd = D.pack_weights_umma_fp8(w, torch.full((k,), 0.05 / 8, device=dev), args.x,
                                     pad_channels=c % args.x != 0)
    else:
        wd = D.pack_weights_umma(w, args.x, lmode, pad_channels=c % args.x != 0)
    out = torch.empty((n, k // args.y, oh, ow, args.y), dtype=act, device=dev)
    res = torch.randn(out.shape, device=dev).to(act) if args.res else None
    bias = torch.randn(k, device=dev)
    flops = 2 * n * k * c * r * s_ * oh * ow
    byts = (x.numel() + out.numel() * (2 if args.res else 1)) * x.element_size()

    hh, ww = (1, H * W) if args.flat else (H, W)

    def run(tile):
        from paper_1809_02697_b200 import _lib as L2
        pro = (torch.ones(c, device=dev), torch.zeros(c, device=dev), True) if args.prologue else None
        p = D.conv_params(lmode, x, wd, out, n, c, hh, ww, k, r, s_, (st, sw), (ph, pw), args.x,
                          args.y, bias=bias, residual=res, relu=True, tile=tile,
                          flags=(L2.FLAG_PAD_CHANNELS if c % args.x else 0)
                          | (L2.FLAG_HALO_STRIPS if args.strips else 0), prologue=pro)
        cfg = D.default_tiles(p)
        ws = torch.zeros(max(D.conv_workspace_bytes(p), 4) // 4, device=dev)
        D.set_workspace(p, ws)
        if args.once:
            D.conv2d(p)
            torch.cuda.synchronize()
            return 1e-9, cfg
        cs = torch.cuda.Stream()
        for _ in range(3):
            D.conv2d(p, cs)
        torch.cuda.synchronize()
        # back-to-back launches replayed from a CUDA graph: no host overhead
        graph = D.capture(lambda: [D.conv2d(p, cs) for _ in range(args.iters)], cs)
        graph.launch(cs)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        graph.launch(cs)
        b.record(cs)
        b.synchronize()
        us = a.elapsed_time(b) * 1e3 / args.iters
        return us, cfg

    tiles = [json.loads(args.tile) if args.tile else None]
    if args.sweep:
        from paper_1809_02697_b200.kernels import ConvWorkload
        from paper_1809_02697_b200.tuning import tile_variants
        wl = ConvWorkload(c, k, H, W, r, s_, (st, sw), (ph, pw))
        tiles = [None] + [t for t in tile_variants(wl, args.mode, n, pair=True) if t]
    for tile in tiles:
        try:
            us, cfg = run(tile)
        except Exception as exc:
            print(f"{tile}: {type(exc).__name__}: {exc}")
            continue
        print(f"{json.dumps(cfg)} {us:8.1f} us  {flops / us / 1e6:7.1f} TF/s  "
              f"{byts / us / 1e3:7.0f} GB/s")


if __name__ == "__main__":
    main()
