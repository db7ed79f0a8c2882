#!/usr/bin/env python
"""M-tile geometry sweep for one or more conv shapes (CUDA events over a
graph of back-to-back launches, like tools/conv_bench.py).  Answers: does the
kernel's own geometry pick (maximal useful MMA rows, which at batch 128 on odd
maps is one pixel x 128 images) lose to tiles that keep pixels of ONE image
together?

  python tools/geo_sweep.py --shapes inception        # the Inception-v3 b128 shapes
  python tools/geo_sweep.py --shape 128,32,32,149,149,3,3,1,0,0,32,32
      (n,c,k,h,w,r,s,stride,pad_h,pad_w,x,y)
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

INCEPTION = [
    # n, c, k, h, w, r, s, stride, ph, pw, x, y
    (128, 32, 32, 149, 149, 3, 3, 1, 0, 0, 32, 32),
    (128, 32, 64, 147, 147, 3, 3, 1, 1, 1, 32, 64),
    (128, 64, 80, 73, 73, 1, 1, 1, 0, 0, 64, 16),
    (128, 80, 192, 73, 73, 3, 3, 1, 0, 0, 16, 64),
    (128, 64, 96, 35, 35, 3, 3, 1, 1, 1, 64, 32),
    (128, 96, 96, 35, 35, 3, 3, 1, 1, 1, 32, 32),
    (128, 48, 64, 35, 35, 5, 5, 1, 2, 2, 16, 32),
    (128, 288, 64, 35, 35, 1, 1, 1, 0, 0, 32, 32),
    (128, 288, 384, 35, 35, 3, 3, 2, 0, 0, 32, 32),
    (128, 768, 192, 17, 17, 1, 1, 1, 0, 0, 64, 64),
    (128, 192, 192, 17, 17, 1, 7, 1, 0, 3, 64, 64),
    (128, 160, 160, 17, 17, 7, 1, 1, 3, 0, 32, 32),
]


def exact_geometries(n, oh, ow, min_eff=0.93):
    """Every (bw, bh, bni) box of <= 128 pixels with >= min_eff useful rows,
    image-spanning boxes included (``--exact``)."""
    out = [None]
    for bw in range(1, min(ow, 128) + 1):
        for bh in range(1, min(oh, 128 // bw) + 1):
            for bni in range(1, min(n, 128 // (bw * bh)) + 1):
                eff = n * oh * ow / (-(-ow // bw) * -(-oh // bh) * -(-n // bni) * 128)
                if eff >= min_eff:
                    out.append({"tile_w": bw, "tile_h": bh, "tile_img": bni})
    return out


def geometries(n, oh, ow):
    out = [None]
    seen = set()
    for bw in sorted({ow, min(ow, 128), 64, 32, 16, 8, -(-ow // 2), -(-ow // 3), -(-ow // 4),
                      -(-ow // 5), -(-ow // 8), -(-ow // 10)}):
        if bw < 1 or bw > min(ow, 128):
            continue
        for bh in sorted({1, 2, 3, 4, 5, 6, 7, 8, 16, oh}):
            if bh > oh or bw * bh > 128:
                continue
            bni = 1
            if bw == ow and bh == oh:
                bni = max(1, min(n, 128 // (bw * bh)))
            eff = n * oh * ow / (-(-ow // bw) * -(-oh // bh) * -(-n // bni) * 128)
            if eff < 0.75 or (bw, bh, bni) in seen:
                continue
            seen.add((bw, bh, bni))
            out.append({"tile_w": bw, "tile_h": bh, "tile_img": bni})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="")
    ap.add_argument("--shape", action="append", default=[])
    ap.add_argument("--mode", default="bf16")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--extra", default="", help="json dict merged into every explicit tile")
    ap.add_argument("--exact", action="store_true",
                    help="sweep every box with >= 93%% useful rows (image-spanning included)")
    ap.add_argument("--res", action="store_true", help="fused residual + relu epilogue")
    args = ap.parse_args()
    shapes = [tuple(int(v) for v in s.split(",")) for s in args.shape]
    if args.shapes == "inception":
        shapes += INCEPTION

    import torch
    from paper_1809_02697_b200 import _lib as L
    from paper_1809_02697_b200 import device as D

    dev = torch.device("cuda:0")
    act = {"bf16": torch.bfloat16, "fp8": torch.float8_e4m3fn}.get(args.mode, torch.float32)
    lmode = {"bf16": L.MODE_BF16, "fp8": L.MODE_FP8}.get(args.mode, L.MODE_TF32)
    extra = json.loads(args.extra) if args.extra else {}
    for (n, c, k, H, W, r, s, st, ph, pw, bx, by) in shapes:
        oh = (H + 2 * ph - r) // st + 1
        ow = (W + 2 * pw - s) // st + 1
        x = torch.randn((n, -(-c // bx), H, W, bx), device=dev).to(act)
        w = torch.randn((k, c, r, s), device=dev) * 0.05
        wd = D.pack_weights_umma(w, bx, lmode, pad_channels=c % bx != 0)
        out = torch.empty((n, k // by, oh, ow, by), dtype=act, device=dev)
        bias = torch.randn(k, device=dev)
        res = torch.randn(out.shape, device=dev).to(act) if args.res else None
        flops = 2 * n * k * c * r * s * oh * ow
        byts = (x.numel() + out.numel()) * x.element_size()
        print(f"== n{n} C{c} K{k} {H}x{W} {r}x{s}/{st} pad({ph},{pw}) x{bx} y{by}: "
              f"{flops / 1e9:.1f} GFLOP, {byts / 1e6:.0f} MB "
              f"(hbm {byts / 6.5e6:.0f} us, tensor {flops / 1.65e9:.0f} us)", flush=True)
        rows = []
        for geo in (exact_geometries(n, oh, ow) if args.exact else geometries(n, oh, ow)):
            tile = None if geo is None else {**geo, **extra}
            try:
                p = D.conv_params(lmode, x, wd, out, n, c, H, W, k, r, s, (st, st), (ph, pw), bx,
                                  by, bias=bias, residual=res, relu=True, tile=tile,
                                  flags=L.FLAG_PAD_CHANNELS if c % bx else 0)
                cfg = D.default_tiles(p)
                ws = torch.zeros(max(D.conv_workspace_bytes(p), 4) // 4, device=dev)
                D.set_workspace(p, ws)
                cs = torch.cuda.Stream()
                for _ in range(2):
                    D.conv2d(p, cs)
                torch.cuda.synchronize()
                graph = D.capture(lambda: [D.conv2d(p, cs) for _ in range(args.iters)], cs)
                graph.launch(cs)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(cs)
                graph.launch(cs)
                b.record(cs)
                b.synchronize()
                us = a.elapsed_time(b) * 1e3 / args.iters
            except Exception as exc:
                print(f"   {tile}: {type(exc).__name__}: {str(exc)[:100]}")
                continue
            rows.append((us, geo is None, cfg))
        for us, dflt, cfg in sorted(rows, key=lambda r: r[0])[:8] + [r for r in rows if r[1]]:
            print(f"   {us:8.1f} us {flops / us / 1e6:6.0f} TF/s {byts / us / 1e3:6.0f} GB/s "
                  f"{'DEFAULT ' if dflt else ''}{json.dumps(cfg)}", flush=True)


if __name__ == "__main__":
    main()
