"""FP8 (e4m3) quantized inference: static per-tensor activation scales.

The reference has no quantized mode (PAPER.md:433 names quantized inference
as future work; its only dtype is f32, graph.py:20-21).  This module is the
host half of the B200 FP8 conv mode:

* weights: per output channel, ``wscale[k] = max_j |W[k, j]| / 448`` (f32)
  and ``W_q = RN_e4m3(W / wscale[k])`` (neo_pack_weights_umma_fp8); the conv
  folds ``x_scale * wscale[k]`` into its per-channel epilogue scale, which is
  the reference Epilogue's scale slot (kernels.py:74-87, applied in the order
  of :185-197);
* activations: one power-of-two scale per stored NCHW[x]c map, chosen by
  running the bf16 program once on calibration images (static calibration):
  ``s = 2^ceil(log2(absmax * margin / 448))``.  Powers of two keep every
  (de)quantization an exact multiply, so the only rounding an e4m3 map adds
  is the one RN_e4m3 of each stored value.
"""

from __future__ import annotations

import math

import numpy as np

from .graph import Graph, OpKind

E4M3_MAX = 448.0
# headroom over the calibration absmax (inputs of the same distribution but
# other images reach a little further)
CALIB_MARGIN = 1.25


def weight_scales(kcrs: np.ndarray) -> np.ndarray:
    """Per-output-channel e4m3 weight scales (f32): absmax / 448 (1 for an
    all-zero channel)."""
    w = np.asarray(kcrs, np.float32)
    amax = np.abs(w.reshape(w.shape[0], -1)).max(axis=1).astype(np.float32)
    ws = (amax / np.float32(E4M3_MAX)).astype(np.float32)
    ws[ws == 0] = np.float32(1.0)
    return ws


def act_scale(absmax: float, margin: float = CALIB_MARGIN) -> float:
    """Power-of-two activation scale covering ``absmax * margin``."""
    a = float(absmax) * margin
    if not np.isfinite(a) or a <= 0:
        return 1.0
    return float(2.0 ** math.ceil(math.log2(a / E4M3_MAX)))


def _global_pool(g: Graph, nid: int) -> bool:
    """A global average pool the fused classifier head absorbs (C % 256 ==
    0, fusion._Analysis._fused_head_info): the head pools the e4m3 map at its
    input's scale, so the pool itself stores nothing and needs no scale."""
    from .graph import hw_pair, infer_shapes
    n = g.nodes[nid]
    if n.kind != OpKind.AvgPool:
        return False
    spec = infer_shapes(g)[n.inputs[0][0]]
    _, c, h, w = spec.logical_nchw
    return (hw_pair(n.attrs["window"]) == (h, w) and hw_pair(n.attrs.get("pad", 0)) == (0, 0)
            and c % 256 == 0)


def quantized_nodes(g: Graph) -> list[int]:
    """Nodes whose outputs an fp8 program may store as e4m3 maps: convs,
    pools (the fused stem's output is its max pool; global average pools
    feed the classifier head, which reads its input map's scale) and ReLUs
    (DenseNet's BN-ReLU pre-activations)."""
    return [nid for nid, n in g.nodes.items()
            if n.kind in (OpKind.Conv2d, OpKind.MaxPool, OpKind.AvgPool, OpKind.ReLU)
            and not _global_pool(g, nid)]


def calibrate(g: Graph, feeds: dict | None = None, batch: int = 4, device: int = 0,
              margin: float = CALIB_MARGIN) -> dict[int, float]:
    """{node id: power-of-two e4m3 scale} from one bf16 forward of ``g``
    (the uncompiled model graph) on ``feeds`` (default: a seeded N(0, 1)
    batch of ``batch`` images, seed 7).  Node ids refer to the simplified
    graph, which compile_graph produces identically in every mode."""
    import torch
    from . import device as D
    from .executor import DeviceProgram, ExecutablePlan, with_batch
    from .models import model_input
    from .passes import compile_graph
    if feeds is None:
        gc = with_batch(g, batch)
        feeds = model_input(gc, seed=7)
    else:
        n0 = next(iter(feeds.values())).shape[0]
        gc = with_batch(g, n0)
    cg = compile_graph(gc, mode="bf16")
    keep = [nid for nid in quantized_nodes(cg) if nid not in cg.outputs]
    prog = DeviceProgram(ExecutablePlan.compile(cg), device, "bf16", keep=keep, use_graph=False)
    prog.set_inputs(feeds)
    prog.launch()
    scales = {}
    tensors = prog.output_tensors()
    amax = torch.empty(len(tensors), dtype=torch.float32, device=prog.device)
    with torch.cuda.stream(prog.stream):
        for i, t in enumerate(tensors):
            D.absmax(t.contiguous(), amax[i:i + 1], stream=prog.stream)
    prog.stream.synchronize()
    host = amax.cpu().numpy()
    ids = list(cg.outputs) + keep
    for nid, a in zip(ids, host):
        if nid in keep:
            scales[nid] = act_scale(a, margin)
    return scales


def attach_scales(g: Graph, scales: dict[int, float]) -> Graph:
    """Store the scales as ``fp8_scale`` attrs of the compiled graph's conv,
    pool and ReLU nodes (in place).

    * A max pool inherits its input's scale: its outputs are a subset of its
      inputs' stored values, so the e4m3 bytes carry over unchanged.
    * Channel concats are done in place (producers write windows of one
      buffer), so a concat and all its inputs -- transitively, through nested
      concats -- form one group stored at one scale: the largest of the
      members' calibrated scales (a power of two covering every member)."""
    from .graph import topo_sort
    quant = set(quantized_nodes(g))
    for nid in topo_sort(g):
        node = g.nodes[nid]
        if nid not in quant:
            continue
        src = node.inputs[0][0] if node.inputs else None
        if node.kind == OpKind.MaxPool and src is not None and "fp8_scale" in g.nodes[src].attrs:
            node.attrs["fp8_scale"] = g.nodes[src].attrs["fp8_scale"]
        elif nid in scales:
            node.attrs["fp8_scale"] = float(scales[nid])
    parent: dict[int, int] = {}

    def find(a: int) -> int:
        parent.setdefault(a, a)
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    concats = [nid for nid, n in g.nodes.items()
               if n.kind == OpKind.Concat and n.attrs.get("axis", 1) == 1]
    for c in concats:
        for src, _ in g.nodes[c].inputs:
            parent[find(src)] = find(c)
    groups: dict[int, list[int]] = {}
    for m in list(parent):
        groups.setdefault(find(m), []).append(m)
    for members in groups.values():
        sc = [g.nodes[m].attrs["fp8_scale"] for m in members if "fp8_scale" in g.nodes[m].attrs]
        if not sc:
            continue
        top = max(sc)
        for m in members:
            if m in quant or g.nodes[m].kind == OpKind.Concat:
                g.nodes[m].attrs["fp8_scale"] = top
    return g


__all__ = ["E4M3_MAX", "weight_scales", "act_scale", "calibrate", "attach_scales",
           "quantized_nodes"]
