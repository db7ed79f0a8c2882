#!/usr/bin/env python
"""Per-layer device vs e4m3-model differences of an fp8 program (debug):
every conv / pool output of the compiled graph is kept on the device and
compared with the oracle's e4m3 model of the same graph and scales."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from oracle.ops import unpack_nchw


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
    batch = 1 if model.startswith("ssd") else 2
    image = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, build_model, compile_graph,
                                       model_input)
    from paper_1809_02697_b200.graph import OpKind, topo_sort
    g = build_model(model, batch=batch, image=image, **({} if model.startswith("ssd") else {"softmax": False}))
    cg = compile_graph(g, mode="fp8")
    users = cg.consumers()
    # (a conv feeding only a max pool is the fused image stem: keeping it
    # would unfuse the stem and change the program)
    ids = [nid for nid in topo_sort(cg) if cg.nodes[nid].kind in (OpKind.Conv2d, OpKind.MaxPool)
           and not (cg.nodes[nid].kind == OpKind.Conv2d and users.get(nid)
                    and all(cg.nodes[u].kind == OpKind.MaxPool for u in users[nid]))]
    prog = DeviceProgram(ExecutablePlan.compile(cg), 0, "fp8", keep=ids)
    feeds = model_input(g)
    outs = prog.run(feeds)
    dev = dict(zip(list(cg.outputs) + ids, outs))
    h = cg.copy()
    h.outputs = list(cg.outputs) + ids
    ref = dict(zip(h.outputs, oracle.execute_reference(h, feeds, arith="fp8")))
    for nid in ids:
        d = dev[nid]
        s = cg.nodes[nid].attrs.get("fp8_scale")
        v = prog.vals[nid]
        if str(v.tensor.dtype) == "torch.float8_e4m3fn" and s is not None:
            d = d * np.float32(s)
        if d.ndim == 5:
            d = unpack_nchw(d)
        r = ref[nid]
        if r.ndim == 5:
            r = unpack_nchw(r)
        print(f"{cg.nodes[nid].kind.value:8s} {nid:4d} {str(v.tensor.dtype):22s} scale {s} "
              f"rel_err {oracle.rel_err(d, r):.3e} max|ref| {np.abs(r).max():.3e}")


if __name__ == "__main__":
    main()
