"""Whole-graph CPU interpreter -- TEST INFRASTRUCTURE ONLY.

Restates the reference executor (executor.py:131-218) for graphs in the
reference IR (graph.py:82-126: nodes with ``kind``, ``attrs``, ``inputs``
edges, ``outputs``).  It is duck-typed: it reads the graph structure but
imports nothing from the product package.  Conv nodes may carry an
asymmetric ``pad=(ph, pw)`` / ``stride=(sh, sw)`` (the Inception-v3
extension the reference cannot express); blocked
layouts and LayoutTransform nodes are honoured like the reference does.
"""

from __future__ import annotations

import heapq

import numpy as np

from . import ops


def _topo(graph) -> list[int]:
    """graph.py:129-152: Kahn order, ties broken by ascending id."""
    indeg = {nid: 0 for nid in graph.nodes}
    succ = {nid: [] for nid in graph.nodes}
    for n in graph.nodes.values():
        seen = set()
        for i, _ in n.inputs:
            if i in indeg and i not in seen:
                seen.add(i)
                indeg[n.id] += 1
                succ[i].append(n.id)
    ready = [nid for nid, d in indeg.items() if d == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        nid = heapq.heappop(ready)
        order.append(nid)
        for s in succ[nid]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(ready, s)
    return order


def _kind(n) -> str:
    return getattr(n.kind, "value", n.kind)


def _conv(n, vals, arith=None):
    data = vals[n.inputs[0][0]]
    weight = vals[n.inputs[1][0]]
    epi = dict(n.attrs.get("epilogue") or {})
    ins = [vals[i] for i, _ in n.inputs]
    residual = None
    extra = 0
    if epi.get("residual"):
        residual = ins[-1]
        extra += 1
    bias = epi.get("bias")
    if len(n.inputs) - extra >= 3:  # executor.py:63-66 explicit bias input
        b = ins[2]
        bias = b if bias is None else bias + b
    stride, pad = n.attrs["stride"], n.attrs["pad"]
    blocked = data.ndim == 5
    if blocked:
        data = ops.unpack_nchw(data)
        if weight.ndim == 6:
            weight = ops.unpack_kcrs(weight)
        if residual is not None:
            residual = ops.unpack_nchw(residual)
    args = (data, weight, stride, pad, epi.get("scale"), epi.get("shift"), bias, residual,
            bool(epi.get("relu", False)))
    out = ops.conv2d(*args) if arith is None else ops.conv2d_rounded(arith, *args)
    if blocked:
        sch = n.attrs.get("schedule") or {}
        y = sch.get("oc_bn") or (vals[n.inputs[1][0]].shape[5]
                                 if vals[n.inputs[1][0]].ndim == 6 else 1)
        out = ops.pack_nchw(out, y)
    return out


def _conv_fp8(n, vals, q8: set, scales: dict, feeds_pool: set):
    """FP8-mode conv of a compiled graph (node attr ``fp8_scale`` = scale of
    its stored e4m3 output): an e4m3 input gives an e4m3 conv
    (ops.conv2d_fp8); the image stem (input not e4m3) runs in bf16 like the
    device's fused stem and leaves its output unquantized."""
    data_id = n.inputs[0][0]
    if data_id not in q8:
        # bf16 operands (the image stem); its output is stored as e4m3 unless
        # a max pool fused with it (the ResNet stem) quantizes the pooled map
        if n.attrs.get("fp8_scale") is None or n.id in feeds_pool:
            return _conv(n, vals, "bf16"), False
        data, weight = vals[data_id], vals[n.inputs[1][0]]
        epi = dict(n.attrs.get("epilogue") or {})
        ins = [vals[i] for i, _ in n.inputs]
        bias = epi.get("bias")
        if len(n.inputs) >= 3:
            bias = ins[2] if bias is None else bias + ins[2]
        blocked = data.ndim == 5
        if blocked:
            data = ops.unpack_nchw(data)
        if weight.ndim == 6:
            weight = ops.unpack_kcrs(weight)
        s8 = np.float32(n.attrs["fp8_scale"])
        out = ops.conv2d(ops.round_rn(data, "bf16"), ops.round_rn(weight, "bf16"), n.attrs["stride"],
                         n.attrs["pad"], epi.get("scale"), epi.get("shift"), bias, None,
                         bool(epi.get("relu", False)))
        out = (ops.round_e4m3(out / s8) * s8).astype(np.float32)
        if blocked:
            sch = n.attrs.get("schedule") or {}
            y = sch.get("oc_bn") or (vals[n.inputs[1][0]].shape[5]
                                     if vals[n.inputs[1][0]].ndim == 6 else 1)
            out = ops.pack_nchw(out, y)
        return out, True
    epi = dict(n.attrs.get("epilogue") or {})
    ins = [vals[i] for i, _ in n.inputs]
    extra = 1 if epi.get("residual") else 0
    residual = ins[-1] if extra else None
    bias = epi.get("bias")
    if len(n.inputs) - extra >= 3:
        bias = ins[2] if bias is None else bias + ins[2]
    data, weight = vals[data_id], vals[n.inputs[1][0]]
    if data.ndim == 5:
        data = ops.unpack_nchw(data)
        if residual is not None:
            residual = ops.unpack_nchw(residual)
    if weight.ndim == 6:
        weight = ops.unpack_kcrs(weight)
    xs = np.float32(scales[data_id])
    out_scale = n.attrs["fp8_scale"]
    sch = n.attrs.get("schedule") or {}
    bf16_out = (sch.get("oc_bn") or 16) < 16      # rows under 16 bytes: stored bf16
    stored = ops.conv2d_fp8(data / xs, weight, xs, None if bf16_out else out_scale,
                            n.attrs["stride"], n.attrs["pad"], epi.get("scale"), epi.get("shift"),
                            bias, residual, bool(epi.get("relu", False)))
    out = ops.round_rn(stored, "bf16") if bf16_out else \
        (stored * np.float32(out_scale)).astype(np.float32)
    if vals[data_id].ndim == 5:
        sch = n.attrs.get("schedule") or {}
        y = sch.get("oc_bn") or (vals[n.inputs[1][0]].shape[5]
                                 if vals[n.inputs[1][0]].ndim == 6 else 1)
        out = ops.pack_nchw(out, y)
    return out, not bf16_out


def _q8(a, scale) -> np.ndarray:
    """Store f32 values as e4m3 at ``scale`` (the dequantized result)."""
    s8 = np.float32(scale)
    return (ops.round_e4m3(np.asarray(a, np.float32) / s8) * s8).astype(np.float32)


def execute_reference(graph, inputs: dict, arith: str | None = None) -> list[np.ndarray]:
    """Run ``graph`` on numpy ``inputs`` (name -> array); outputs in
    ``graph.outputs`` order.  ``arith`` ("bf16" / "tf32") models the
    roundings of a single-pass tensor-core mode in every conv
    (ops.conv2d_rounded); "fp8" models the FP8 mode on a graph compiled with
    e4m3 scales (node attr ``fp8_scale``): e4m3 maps are the dequantized
    stored values; None is the reference's f32 arithmetic."""
    vals: dict[int, np.ndarray] = {}
    q8: set = set()                       # nodes whose values are e4m3 maps
    scales = {nid: float(nd.attrs["fp8_scale"]) for nid, nd in graph.nodes.items()
              if "fp8_scale" in nd.attrs} if arith == "fp8" else {}
    return _execute(graph, inputs, arith, vals, q8, scales)


def _execute(graph, inputs, arith, vals, q8, scales):
    # convs whose only consumers are max pools: the device fuses an image
    # stem with its pool and stores the pooled map, not the conv output
    users: dict[int, list] = {}
    for nd in graph.nodes.values():
        for src, _ in nd.inputs:
            users.setdefault(src, []).append(nd)
    feeds_pool = {nid for nid, nd in graph.nodes.items() if _kind(nd) == "Conv2d" and users.get(nid)
                  and all(_kind(u) == "MaxPool" for u in users[nid])}
    for nid in _topo(graph):
        n = graph.nodes[nid]
        k = _kind(n)
        src = [vals[i] for i, _ in n.inputs]
        if k == "Input":
            name = n.attrs.get("name", f"input{nid}")
            a = np.ascontiguousarray(inputs[name], dtype=np.float32)
            if n.attrs.get("layout", "NCHW") == "NHWC":
                a = ops.nhwc_to_nchw(a)
            vals[nid] = a
        elif k == "Constant":
            vals[nid] = np.asarray(n.attrs["value"], dtype=np.float32)
        elif k == "Conv2d" and arith == "fp8":
            vals[nid], quant = _conv_fp8(n, vals, q8, scales, feeds_pool)
            if quant:
                q8.add(nid)
        elif k == "Conv2d":
            vals[nid] = _conv(n, vals, arith)
        elif k == "ReLU":
            vals[nid] = ops.relu(src[0])
            if arith == "fp8" and nid in scales:
                vals[nid] = _q8(vals[nid], scales[nid])       # e4m3 BN-ReLU output
                q8.add(nid)
        elif k == "Softmax":
            vals[nid] = ops.softmax(src[0])
        elif k == "BatchNorm":
            if len(n.inputs) == 5:
                # executor.py:176-181 computes in the constants' dtype (f32)
                g, b, m, v = (np.asarray(t, np.float32) for t in src[1:])
                scale = g / np.sqrt(v + np.float32(n.attrs.get("eps", 1e-5)))
                shift = b - m * scale
            else:
                scale, shift = n.attrs["scale"], n.attrs["shift"]
            vals[nid] = ops.batchnorm(src[0], scale, shift)
        elif k in ("MaxPool", "AvgPool"):
            vals[nid] = ops.pool2d(src[0], n.attrs["window"], n.attrs["stride"],
                                   n.attrs.get("pad", 0), "max" if k == "MaxPool" else "avg")
            if arith == "fp8" and nid in scales and vals[nid].ndim == 5:
                # e4m3 pooled map (a max pool at its input's scale is exact;
                # the fused stem's pooled bf16 maxima and averages round once)
                vals[nid] = _q8(vals[nid], scales[nid])
                q8.add(nid)
        elif k == "ElementwiseAdd":
            vals[nid] = ops.add(src[0], src[1])
        elif k == "Concat":
            vals[nid] = ops.concat(src, n.attrs.get("axis", 1))
            if arith == "fp8" and all(i in q8 for i, _ in n.inputs):
                q8.add(nid)           # members share the group's scale: exact
        elif k == "Flatten":
            vals[nid] = ops.flatten(src[0])
        elif k == "Dense":
            vals[nid] = ops.dense(src[0], src[1], src[2] if len(src) == 3 else None)
        elif k == "LayoutTransform":
            vals[nid] = ops.transform(src[0], n.attrs["src_layout"], n.attrs["dst_layout"])
        else:
            raise ValueError(f"oracle cannot execute node kind {k}")
    return [vals[o] for o in graph.outputs]
