#!/usr/bin/env python
"""Where does a model's device error come from?  Exposes intermediate values
(the residual-block outputs / every ReLU) as extra graph outputs, runs the
device program and the CPU oracle on the same seeded input and prints, per
exposed value in topological order, rel_err = max|a-b| / max(1, max|b|) and
the value's magnitude.

  python tools/layer_error.py --model ssd_resnet50 --mode tf32 [--every relu|add]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="ssd_resnet50")
    ap.add_argument("--mode", default="tf32")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--every", default="add", choices=["add", "relu"])
    args = ap.parse_args()

    import numpy as np
    import oracle
    from paper_1809_02697_b200 import DevicePool, build_model, compile_graph, execute, model_input
    from paper_1809_02697_b200.graph import OpKind, topo_sort

    g = build_model(args.model, batch=args.batch)
    order = topo_sort(g)
    users = {n: [] for n in g.nodes}
    for node in g.nodes.values():
        for i, _ in node.inputs:
            users[i].append(node.id)
    picks = []
    for nid in order:
        node = g.nodes[nid]
        if node.kind != OpKind.ReLU:
            continue
        src = g.nodes[node.inputs[0][0]]
        if args.every == "relu" or src.kind == OpKind.ElementwiseAdd:
            picks.append(nid)
    h = g.copy()
    h.outputs = list(g.outputs) + picks
    feeds = model_input(g, seed=1)
    t0 = time.time()
    ref = oracle.execute_reference(h, feeds)
    t1 = time.time()
    got = execute(compile_graph(h, mode=args.mode), feeds, DevicePool(0, args.mode))
    t2 = time.time()
    print(f"oracle {t1 - t0:.1f} s, device {t2 - t1:.1f} s")
    nout = len(g.outputs)
    for i, nid in enumerate(picks):
        a, b = got[nout + i], ref[nout + i]
        print(f"relu{nid:5d} shape {tuple(b.shape)} max|b| {np.abs(b).max():9.3f} "
              f"rel_err {oracle.rel_err(a, b):.3e} rel_to_max {np.abs(a - b).max() / np.abs(b).max():.3e}")
    for i in range(nout):
        a, b = got[i], ref[i]
        print(f"output{i:2d} shape {tuple(b.shape)} max|b| {np.abs(b).max():9.3f} "
              f"rel_err {oracle.rel_err(a, b):.3e}")


if __name__ == "__main__":
    main()
