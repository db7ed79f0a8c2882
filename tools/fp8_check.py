#!/usr/bin/env python
"""FP8 (e4m3) conv mode: op-level and whole-network checks against the
oracle's e4m3 arithmetic model, plus graphed-step timings (exploration
script; the pinned checks live in tests/test_gpu_fp8.py)."""

from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import oracle
from oracle.ops import (conv2d_fp8, e4m3_from_bytes, e4m3_to_bytes, pack_nchw, round_e4m3,
                        unpack_nchw)
from paper_1809_02697_b200 import _lib as L
from paper_1809_02697_b200 import device as D


def to_dev_fp8(vals_e4m3: np.ndarray, x: int):
    b = pack_nchw(e4m3_to_bytes(vals_e4m3), x)
    return torch.from_numpy(np.ascontiguousarray(b)).cuda().view(torch.float8_e4m3fn)


def from_dev_fp8(t) -> np.ndarray:
    return unpack_nchw(e4m3_from_bytes(t.view(torch.uint8).cpu().numpy()))


def conv_case(n, c, h, w, k, r, s, stride, pad, ic_bn, oc_bn, res=False, relu=True, seed=0,
              tile=None):
    rng = np.random.default_rng(seed)
    xs, os_, rs = 2.0 ** -6, 2.0 ** -4, 2.0 ** -5
    xq = round_e4m3(rng.standard_normal((n, c, h, w)).astype(np.float32) / np.float32(xs))
    wt = (rng.standard_normal((k, c, r, s)) * np.sqrt(2 / (c * r * s))).astype(np.float32)
    bias = rng.normal(0, 0.1, k).astype(np.float32)
    oh = (h + 2 * pad - r) // stride + 1
    ow = (w + 2 * pad - s) // stride + 1
    rq = round_e4m3(rng.standard_normal((n, k, oh, ow)).astype(np.float32)) if res else None
    ref = conv2d_fp8(xq, wt, xs, os_, stride, pad, None, None, bias,
                     rq * np.float32(rs) if res else None, relu)
    xd = to_dev_fp8(xq, ic_bn)
    ws = torch.from_numpy(oracle.ops.fp8_weight_scales(wt)).cuda()
    wd = D.pack_weights_umma_fp8(torch.from_numpy(wt).cuda(), ws, ic_bn)
    out = torch.empty((n, k // oc_bn, oh, ow, oc_bn), dtype=torch.float8_e4m3fn, device="cuda")
    sc = torch.from_numpy((np.float32(xs) * oracle.ops.fp8_weight_scales(wt)).astype(np.float32)).cuda()
    rd = to_dev_fp8(rq, oc_bn) if res else None
    p = D.conv_params(L.MODE_FP8, xd, wd, out, n, c, h, w, k, r, s, (stride, stride), (pad, pad),
                      ic_bn, oc_bn, sc, None, torch.from_numpy(bias).cuda(), rd, relu,
                      qscales=(rs, os_, 0.0), tile=tile)
    D.conv2d(p)
    torch.cuda.synchronize()
    got = from_dev_fp8(out)
    diff = got != ref
    spacing = np.maximum(np.abs(ref), 2.0 ** -6) * 2.0 ** -3
    worst = float(np.max(np.abs(got - ref) / spacing)) if diff.any() else 0.0
    print(f"conv {n}x{c}x{h}x{w} k{k} {r}x{s}/{stride} x{ic_bn}/{oc_bn} res={res}: "
          f"mismatch {diff.mean():.2e}, worst {worst:.2f} ulp, nonzero {np.mean(ref != 0):.2f}")
    return diff.mean(), worst


def main():
    torch.cuda.init()
    cases = [
        (1, 64, 56, 56, 64, 3, 3, 1, 1, 64, 64, False),
        (2, 64, 56, 56, 256, 1, 1, 1, 0, 64, 128, True),
        (2, 256, 56, 56, 64, 1, 1, 1, 0, 128, 64, False),
        (2, 128, 28, 28, 128, 3, 3, 1, 1, 128, 128, False),
        (4, 256, 14, 14, 256, 3, 3, 1, 1, 128, 128, False),
        (2, 512, 28, 28, 256, 1, 1, 2, 0, 128, 128, False),
        (2, 512, 7, 7, 2048, 1, 1, 1, 0, 128, 128, True),
    ]
    for cs in cases:
        conv_case(*cs)
    # whole network
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, build_model, compile_graph,
                                       model_input)
    for model, batch in (("resnet18", 4), ("resnet50", 4)):
        g = build_model(model, batch=batch, softmax=False)
        feeds = model_input(g)
        t0 = time.time()
        cg = compile_graph(g, mode="fp8")
        t1 = time.time()
        prog = DeviceProgram(ExecutablePlan.compile(cg), 0, "fp8")
        out = prog.run(feeds)[0]
        model8 = oracle.execute_reference(cg, feeds, arith="fp8")[0]
        ref = oracle.execute_reference(g, feeds)[0]
        print(f"{model} b{batch} fp8: calib+compile {t1 - t0:.1f}s, vs fp8 model "
              f"{oracle.rel_err(out, model8):.3e}, model vs f32 {oracle.rel_err(model8, ref):.3e}, "
              f"device vs f32 {oracle.rel_err(out, ref):.3e}, top1 {np.mean(out.argmax(1) == ref.argmax(1)):.2f} "
              f"(model {np.mean(model8.argmax(1) == ref.argmax(1)):.2f})")
    # timing at b64
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    for mode in ("bf16", "fp8"):
        g = build_model("resnet50", batch=64)
        cg = compile_graph(g, mode=mode)
        prog = DeviceProgram(ExecutablePlan.compile(cg), 0, mode)
        prog.set_inputs(model_input(g))
        ts = []
        for i in range(30):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(prog.stream)
            prog.launch()
            b.record(prog.stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts[5:]))
        print(f"resnet50 b64 {mode}: {ms:.3f} ms/step, {64 / ms * 1e3:.0f} img/s, "
              f"{len(prog.launches)} launches")
        if mode == "fp8" and os.environ.get("PER_LAUNCH"):
            from paper_1809_02697_b200.timing import timed_launches
            ms_l = timed_launches(prog)
            for name, t, desc, fl in zip(prog.launch_names, ms_l, prog.launch_desc,
                                          prog.launch_flops):
                print(f"  {name:16s} {t * 1e3:7.1f} us {fl / t / 1e9 if t else 0:7.0f} TF/s {desc}")


if __name__ == "__main__":
    main()
