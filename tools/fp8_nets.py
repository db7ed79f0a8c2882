#!/usr/bin/env python
"""FP8 whole-network check for every family (device vs the oracle's e4m3
model of the same compiled graph and scales, and vs the f32 oracle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle


def main():
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, build_model, compile_graph,
                                       model_input)
    cases = [("densenet201", 2, 64), ("inception_v3", 2, 139), ("ssd_resnet50", 1, 256),
             ("resnet50", 2, 224), ("vgg16", 2, 64)]
    only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
    for model, batch, image in cases:
        if only and model not in only:
            continue
        kw = {} if model == "ssd_resnet50" else {"softmax": False}
        g = build_model(model, batch=batch, image=image, **kw)
        try:
            cg = compile_graph(g, mode="fp8")
            prog = DeviceProgram(ExecutablePlan.compile(cg), 0, "fp8")
        except Exception as exc:
            print(f"{model}: {type(exc).__name__}: {exc}")
            continue
        feeds = model_input(g)
        try:
            got = prog.run(feeds)
        except Exception as exc:
            print(f"{model}: {type(exc).__name__}: {exc}")
            continue
        m8 = oracle.execute_reference(cg, feeds, arith="fp8")
        ref = oracle.execute_reference(g, feeds)
        errs = [oracle.rel_err(a, b) for a, b in zip(got, m8)]
        rms = [float(np.sqrt(np.mean((a - b) ** 2)) / max(1e-30, np.sqrt(np.mean(b ** 2))))
               for a, b in zip(got, m8)]
        errf = [oracle.rel_err(a, b) for a, b in zip(m8, ref)]
        print(f"{model} b{batch} {image}: {prog.kernel_launches} launches; device vs e4m3 model "
              f"max {max(errs):.3e} rms {max(rms):.3e}; model vs f32 {max(errf):.3e}")


if __name__ == "__main__":
    main()
