#!/usr/bin/env python
"""Where the end-to-end (public-API) step goes: times K steps of
(a) DeviceProgram.pipeline as bench.py runs it (bf16 host rounding or f32
upload), (b) the device-side part alone -- staging copy + graphed forward +
result readback -- with the inputs already on the device, (c) the graphed
forward alone."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, ScheduleDb, build_model,
                                       compile_graph, model_input)
    from paper_1809_02697_b200.tuning import DEFAULT_DB
    K = 40
    g = build_model("resnet50", batch=64)
    cg = compile_graph(g, mode="bf16", db=ScheduleDb(DEFAULT_DB))
    for host_round in (True, False):
        prog = DeviceProgram(ExecutablePlan.compile(cg), 0, "bf16", host_round=host_round)
        feeds = [model_input(g, seed=1 + j) for j in range(3)]
        name = prog.input_names()[0]
        pinned = [torch.from_numpy(f[name]).pin_memory() for f in feeds]
        out_t = prog.output_tensors()[0]
        outs = [torch.empty(out_t.shape, dtype=out_t.dtype).pin_memory() for _ in range(K + 5)]
        rot = lambda k: [pinned[i % 3] for i in range(k)]
        prog.pipeline(rot(5), outs[:5])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(prog._copy_stream)
        prog.pipeline(rot(K), outs[5:])
        t_enq = time.perf_counter() - t0
        e1.record(prog._d2h_stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / K
        print(f"pipeline host_round={host_round}: {ms:.4f} ms/step ({64 / ms * 1e3:.0f} img/s), "
              f"host enqueue {t_enq / K * 1e3:.3f} ms/step, H2D bytes {prog.upload_bytes}")
        # device part only
        dst = prog.vals[prog.plan.input_ids[0]].tensor
        stg = torch.empty_like(dst)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(prog.stream)
        for i in range(K):
            with torch.cuda.stream(prog.stream):
                dst.copy_(stg, non_blocking=True)
            prog.launch()
            with torch.cuda.stream(prog.stream):
                outs[i].copy_(out_t, non_blocking=True)
        b.record(prog.stream)
        b.synchronize()
        ms2 = a.elapsed_time(b) / K
        a.record(prog.stream)
        for i in range(K):
            prog.launch()
        b.record(prog.stream)
        b.synchronize()
        ms3 = a.elapsed_time(b) / K
        print(f"  device part (staging copy + forward + readback): {ms2:.4f} ms/step; "
              f"forward alone {ms3:.4f} ms/step (no L2 flush)")
        # H2D alone
        src = pinned[0] if not host_round else torch.empty(dst.shape, dtype=dst.dtype).pin_memory()
        a.record(prog._copy_stream)
        for i in range(K):
            with torch.cuda.stream(prog._copy_stream):
                stg.copy_(src if src.dtype == stg.dtype else src.to(stg.dtype), non_blocking=True)
        b.record(prog._copy_stream)
        b.synchronize()
        print(f"  H2D alone: {a.elapsed_time(b) / K:.4f} ms/step "
              f"({stg.numel() * stg.element_size() / (a.elapsed_time(b) / K) / 1e6:.1f} GB/s)")
        del prog


if __name__ == "__main__":
    main()
