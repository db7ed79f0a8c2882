"""Graph executor: lowers a (planned or unplanned) graph onto libneob200.

Reference surface kept (executor.py): ``ExecutablePlan.compile`` (:25-45),
``execute(plan|graph, inputs, pool=None)`` (:131-218), ``benchmark`` (:221-236)
and ``scalability_report`` (:239-247).  The reference interprets the graph in
Python and allocates every intermediate in NumPy; here ``DeviceProgram``
compiles it once per (device, mode):

* every operator becomes one pre-bound libneob200 launch (conv with fused
  epilogue, pool, eltwise, concat copy, dense, softmax, layout transform),
  except where fusion.py's plan merges several into one launch (image stem,
  classifier head, sibling 1x1 convs, BN-ReLU, Dense-ReLU);
* standalone BatchNorm followed by its only consumer ReLU runs as one fused
  scale-shift-relu launch (DenseNet's pre-activations);
* all intermediates live in one static arena with liveness-based reuse
  (reference executor.py:211-216 only frees buffers; SPEC.md asks for a
  planned arena);
* the whole forward is captured once as a CUDA graph and replayed;
* dtype rule: NCHW[x]c feature maps are stored in the mode's activation type
  (bf16 in "bf16", tf32-rounded f32 in "tf32", f32 in "fp32", e4m3 with a
  static per-tensor scale in "fp8"); everything else (NCHW maps, matrices,
  logits, graph outputs) is f32;
* "fp8" (quantized inference, quant.py) covers graphs whose blocked maps are
  all produced by tensor-core convs or the fused image stem and read by
  tensor-core convs or the fused classifier head (the ResNet family); other
  operators on e4m3 maps raise InputMismatch;
* a 3-channel (or otherwise tensor-core-illegal) packed graph input that
  only feeds convs is physically packed with zero-padded lanes to the
  smallest legal block (8 bf16 / 4 tf32 lanes), so the stem runs on the
  tensor cores too.

There is no CPU path: without libneob200 or a CUDA device every entry point
raises.
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import InputMismatch, ShapeMismatch
from .fusion import FusionOptions, conv_kcrs, dense_block, plan_fusions
from .graph import Graph, OpKind, hw_pair, infer_shapes, topo_sort, validate
from .kernels import bytes_per_elem, tc_legal_block
from .layout import Layout, host_unpack_kcrs
from .runtime import DevicePool, resolve_pool


@dataclass
class ExecutablePlan:
    """Validated graph + deterministic order + use counts (executor.py:25-45)."""

    graph: Graph
    order: list
    refcounts: dict
    input_ids: list
    programs: dict = field(default_factory=dict, repr=False)

    @classmethod
    def compile(cls, g: Graph) -> "ExecutablePlan":
        problems = validate(g)
        if problems:
            raise InputMismatch("invalid graph: " + "; ".join(problems))
        order = topo_sort(g)
        uses = {nid: 0 for nid in g.nodes}
        for node in g.nodes.values():
            for src, _ in node.inputs:
                uses[src] += 1
        for o in g.outputs:
            uses[o] += 1
        inputs = [nid for nid in order if g.nodes[nid].kind == OpKind.Input]
        return cls(g, order, uses, inputs)


# ---------------------------------------------------------------------------
# device values and the arena

@dataclass
class _Val:
    nid: int
    shape: tuple          # physical storage shape
    dtype: object         # torch dtype
    layout: Layout        # logical layout
    px: int = 0           # physical block size of an NCHW[x]c value
    alias: int | None = None  # value whose storage this one views (Flatten)
    win: tuple | None = None  # (root nid, block offset) inside a concat buffer
    first: int = 0
    last: int = 0
    offset: int = -1
    tensor: object = None

    @property
    def nbytes(self) -> int:
        import torch
        return int(np.prod(self.shape)) * torch.empty((), dtype=self.dtype).element_size()


def _plan_arena(vals: list[_Val], align: int = 256) -> int:
    """Greedy first-fit offsets for non-overlapping lifetimes; returns size."""
    placed: list[_Val] = []
    for v in sorted(vals, key=lambda v: (-v.nbytes, v.first)):
        size = -(-v.nbytes // align) * align
        busy = sorted((p.offset, p.offset + (-(-p.nbytes // align) * align)) for p in placed
                      if not (p.last < v.first or v.last < p.first))
        off = 0
        for lo, hi in busy:
            if off + size <= lo:
                break
            off = max(off, hi)
        v.offset = off
        placed.append(v)
    return max((p.offset + p.nbytes for p in placed), default=0)


def _nb(t) -> int:
    """Bytes of a device tensor."""
    return int(t.numel()) * t.element_size()


def _vb(v) -> int:
    """Bytes of a value's own elements (its window, for concat windows)."""
    import torch
    return int(np.prod(v.shape)) * torch.empty((), dtype=v.dtype).element_size()


class DeviceProgram:
    """One compiled forward of ``plan`` on ``device`` in ``mode``."""

    def __init__(self, plan: ExecutablePlan, device: int = 0, mode: str = "bf16",
                 keep=(), use_graph: bool = True, host_round: bool | None = None,
                 fusion: FusionOptions | None = None):
        """``host_round``: an image read only by fused stems is uploaded as
        bf16 rounded on the host (half the PCIe bytes, host CPU work per
        batch) when True (default), or as f32 and rounded by the stem's
        loader (bit-identical, no host compute: what several ranks sharing one
        host want) when False; NEOB200_HOST_ROUND=0 flips the default.
        ``fusion``: fusion planner switches (fusion.FusionOptions; default
        the shipped configuration with the NEOB200_* experiment overrides)."""
        import torch
        from . import _lib as L
        L.load()
        if not torch.cuda.is_available():
            raise InputMismatch("DeviceProgram needs a CUDA device")
        self.plan = plan
        self.g = plan.graph
        self.mode = mode
        self.device = torch.device("cuda", device)
        self.keep = list(keep)
        self.act_dtype = {"bf16": torch.bfloat16, "fp8": torch.float8_e4m3fn}.get(mode, torch.float32)
        # dense layers (and their non-blocked inputs) and folded image stems
        # run bf16 in fp8 mode: only the blocked conv chain is e4m3
        self.dense_mode = "bf16" if mode == "fp8" else mode
        self.dense_dtype = torch.bfloat16 if mode == "fp8" else self.act_dtype
        # fp8: static e4m3 scale of every stored map (quant.py, node attr)
        self.qscale = {nid: float(n.attrs["fp8_scale"]) for nid, n in self.g.nodes.items()
                       if "fp8_scale" in n.attrs}
        self.round_flag = L.FLAG_ROUND_TF32 if mode == "tf32" else 0
        self.launches: list = []        # zero-arg callables, in order
        self.tc_params: list = []       # tensor-core conv params (split-K workspace)
        self.launch_names: list[str] = []
        self.launch_bytes: list[int] = []
        self.launch_flops: list[int] = []
        self.launch_desc: list[str] = []
        self.vals: dict[int, _Val] = {}
        self.weights: list = []         # device tensors kept alive
        self._pinned_inputs: dict = {}  # input id -> (pinned staging, upload-done event)
        self.graph_exec = None
        # serving input slots: slot 0 is each input's own buffer, slot 1 an
        # alternate buffer pipeline() uploads into while slot 0 is read;
        # launches reading a graph input resolve it at launch time, and one
        # CUDA graph is captured per slot (no device-side staging copy)
        self._input_slot = 0
        self._alt_inputs: dict = {}
        self._graphs: dict = {}
        self.input_readers: dict = {}   # input nid -> launch names reading it
        self.use_graph = use_graph and not os.environ.get("NEOB200_NO_GRAPH")
        self.host_round = (os.environ.get("NEOB200_HOST_ROUND", "1") != "0") if host_round is None \
            else bool(host_round)
        self.fusion_options = fusion if fusion is not None else \
            FusionOptions.from_env(host_round=self.host_round)
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(self.device)
            self._lower()
            self._allocate()
            self._bind()
            torch.cuda.synchronize(self.device)   # weight images built on the side stream

    # -- analysis ------------------------------------------------------------
    def _lower(self):
        g = self.g
        self.specs = infer_shapes(g)
        self.users = g.consumers()
        order = self.plan.order
        self.step = {nid: i for i, nid in enumerate(order)}
        # which operators share a launch: fusion.py owns the decisions
        self.fusion = fp = plan_fusions(g, self.mode, self.keep, self.fusion_options,
                                        specs=self.specs, users=self.users, order=order)
        self.skip = fp.skip
        self.fused_bn_relu, self.prologue, self.pro_src = fp.fused_bn_relu, fp.prologue, fp.pro_src
        self.tc_dense, self.fused_dense_relu = fp.tc_dense, fp.fused_dense_relu
        self.stem_fold, self.fused_stem, self.bf16_inputs = fp.stem_fold, fp.fused_stem, fp.bf16_inputs
        self.fused_head = fp.fused_head
        self.sibling, self.sibling_of = fp.sibling, fp.sibling_of
        self.junction, self.junction_of = fp.junction, fp.junction_of
        self.phys_x = fp.phys_x
        for nid in order:
            if nid in self.skip:
                continue
            node = g.nodes[nid]
            if node.kind == OpKind.Constant:
                continue
            self.vals[nid] = self._make_val(nid)
        # NCHW[x]c -> NCHW of an H = W = 1 map is the identity on memory: alias
        for nid in order:
            node = g.nodes[nid]
            if node.kind != OpKind.LayoutTransform or nid not in self.vals:
                continue
            src = self.vals.get(node.inputs[0][0])
            out = self.vals[nid]
            if (src is not None and src.layout.tag == "NCHWc" and out.layout.tag == "NCHW"
                    and src.shape[2] == 1 and src.shape[3] == 1 and src.dtype == out.dtype
                    and src.px == src.layout.x and not node.attrs.get("pad_channels")):
                out.alias = node.inputs[0][0]
        self._plan_concat_windows()
        # lifetimes
        last_step = len(order)
        for nid, v in self.vals.items():
            v.first = self.step[nid]
            v.last = self.step[nid]
        for nid in order:
            node = self.g.nodes[nid]
            for src, _ in node.inputs:
                tgt = self._storage(self.pro_src.get(src, src))
                if tgt is not None:
                    tgt.last = max(tgt.last, self.step[nid])
            if nid in self.fused_head:      # the fused head reads the pool's input
                tgt = self._storage(self.fused_head[nid]["src"])
                if tgt is not None:
                    tgt.last = max(tgt.last, self.step[nid])
            if nid in self.fused_stem:      # the fused stem reads the graph input
                tgt = self._storage(self.fused_stem[nid][1])
                if tgt is not None:
                    tgt.last = max(tgt.last, self.step[nid])
            fused_src = self.fused_bn_relu.get(nid, self.fused_dense_relu.get(nid))
            if fused_src is not None:
                for src, _ in self.g.nodes[fused_src].inputs:
                    tgt = self._storage(src)
                    if tgt is not None:
                        tgt.last = max(tgt.last, self.step[nid])
        for o in list(self.g.outputs) + self.keep:
            tgt = self._storage(o)
            if tgt is not None:
                tgt.last = last_step
        for nid in self.plan.input_ids:
            self.vals[nid].first = -1
        for second, first in list(self.sibling_of.items()) + list(self.junction_of.items()):
            tgt = self._storage(second)                # written by the first's launch
            if tgt is not None:
                tgt.first = min(tgt.first, self.step[first])
        # a concat buffer lives as long as any of its windows
        for v in self.vals.values():
            if v.win is not None:
                root = self.vals[v.win[0]]
                root.first = min(root.first, v.first)
                root.last = max(root.last, v.last)

    # -- concat in place ---------------------------------------------------------
    def _plan_concat_windows(self):
        """Channel-axis concats of NCHW[x]c maps are done in place: every
        eligible input is produced straight into its channel-block window of
        the concat's buffer (conv epilogues, pools and scale-shift launches
        all take a window), so the concat launch copies only the rest.
        Nested concats (DenseNet's growing feature stack) compose: processing
        in reverse order gives each inner concat its window in the outer
        buffer first, and its own inputs then land in sub-windows of that."""
        g = self.g
        self.concat_windowed: dict[int, set] = {}
        for nid in reversed(self.plan.order):
            node = g.nodes[nid]
            if node.kind != OpKind.Concat or nid not in self.vals:
                continue
            out = self.vals[nid]
            if (node.attrs.get("axis", 1) != 1 or out.layout.tag != "NCHWc"
                    or out.alias is not None or out.px != out.layout.x):
                continue
            root, base = out.win if out.win is not None else (nid, 0)
            srcs = [src for src, _ in node.inputs]
            done = set()
            off = 0
            for src in srcs:
                v = self.vals.get(src)
                if v is None:
                    break
                if srcs.count(src) == 1 and self._window_eligible(src, nid):
                    v.win = (root, base + off)
                    done.add(src)
                off += v.shape[1]
            self.concat_windowed[nid] = done

    def _window_eligible(self, nid: int, concat: int) -> bool:
        g = self.g
        v, out = self.vals[nid], self.vals[concat]
        node = g.nodes[nid]
        if (v.alias is not None or v.win is not None or nid in g.outputs or nid in self.keep
                or v.layout.tag != "NCHWc" or v.px != v.layout.x or v.px != out.px
                or v.dtype != out.dtype or v.shape[0] != out.shape[0]
                or v.shape[2:] != out.shape[2:] or nid in self.phys_x
                or nid in self.stem_fold):
            return False
        if self.mode != "fp32" and not tc_legal_block(v.px, self.mode):
            return False
        kind = node.kind
        if kind == OpKind.ReLU:
            if nid in self.fused_dense_relu:
                return False
        elif kind not in (OpKind.Conv2d, OpKind.MaxPool, OpKind.AvgPool, OpKind.Concat,
                          OpKind.BatchNorm):
            return False
        if kind == OpKind.Conv2d and g.nodes[node.inputs[0][0]].kind == OpKind.Input:
            return False
        for u in self.users[nid]:
            un = g.nodes[u]
            if u == concat:
                continue
            pos = [i for i, (s, _) in enumerate(un.inputs) if s == nid]
            if un.kind == OpKind.Conv2d:
                if pos != [0]:
                    return False
            elif un.kind in (OpKind.MaxPool, OpKind.AvgPool, OpKind.ReLU, OpKind.BatchNorm):
                if pos != [0] or u in self.fused_dense_relu:
                    return False
            else:
                return False
        return True

    def _window(self, v: _Val) -> tuple:
        """(block offset, blocks in the buffer) of a value's storage."""
        if v.win is None:
            return 0, v.shape[1]
        return v.win[1], self.vals[v.win[0]].shape[1]

    def _conv_kcrs(self, nid: int) -> np.ndarray:
        return conv_kcrs(self.g, nid)

    def _storage(self, nid) -> _Val | None:
        v = self.vals.get(nid)
        while v is not None and v.alias is not None:
            v = self.vals[v.alias]
        return v

    def _make_val(self, nid) -> _Val:
        import torch
        spec = self.specs[nid]
        node = self.g.nodes[nid]
        layout = spec.layout
        if nid in self.bf16_inputs:
            return _Val(nid, tuple(spec.shape), torch.bfloat16, layout)
        if node.kind == OpKind.Input and layout.tag == "NHWC":
            layout = Layout("NCHW")
            n, h, w, c = spec.shape
            return _Val(nid, (n, c, h, w), torch.float32, layout)
        if node.kind == OpKind.Flatten:
            return _Val(nid, spec.shape, self.vals[node.inputs[0][0]].dtype, layout,
                        alias=node.inputs[0][0])
        if nid in self.stem_fold:
            f = self.stem_fold[nid]
            shape = (f["n"], -(-f["F"] // f["xf"]), f["h"], f["ow"], f["xf"])
            return _Val(nid, shape, self.dense_dtype, layout, px=f["xf"])
        if layout.tag == "NCHWc":
            px = self.phys_x.get(nid, layout.x)
            n, c, h, w = spec.logical_nchw
            if nid in self.phys_x:
                shape = (n, -(-c // px), h, w, px)
            else:
                shape = spec.shape
            dtype = self.act_dtype
            if self.mode == "fp8" and px < 16:
                # an e4m3 row under 16 bytes has no TMA store: such maps (the
                # SSD heads' 2-8 channel blocks) are kept in bf16
                dtype = torch.bfloat16
            return _Val(nid, tuple(shape), dtype, layout, px=px)
        dtype = self.dense_dtype if self._feeds_tc_dense(nid) else torch.float32
        return _Val(nid, tuple(spec.shape), dtype, layout)

    def _dense_block(self, width: int) -> int:
        return dense_block(width, self.dense_mode)

    def _feeds_tc_dense(self, nid: int) -> bool:
        """A non-blocked value is kept in the activation type when every use
        is the data input of a tensor-core Dense (directly or via Flatten)."""
        g = self.g
        if nid in g.outputs or nid in self.keep:
            return False
        us = self.users[nid]
        if not us:
            return False
        for u in us:
            node = g.nodes[u]
            if node.kind == OpKind.Dense:
                if u not in self.tc_dense or node.inputs[0][0] != nid:
                    return False
            elif node.kind == OpKind.Flatten:
                if not self._feeds_tc_dense(u):
                    return False
            elif node.kind == OpKind.ReLU and nid in self.fused_dense_relu.values():
                if not self._feeds_tc_dense(u):
                    return False
            else:
                return False
        return True

    # -- memory ----------------------------------------------------------------
    def _allocate(self):
        import torch
        owners = [v for v in self.vals.values() if v.alias is None and v.win is None]
        inputs = [v for v in owners if v.first < 0]
        arena_vals = [v for v in owners if v.first >= 0]
        size = _plan_arena(arena_vals)
        self.arena = torch.empty(max(size, 256), dtype=torch.uint8, device=self.device)
        self.arena_bytes = size
        for v in arena_vals:
            nb = v.nbytes
            v.tensor = self.arena[v.offset:v.offset + nb].view(v.dtype).view(v.shape)
        for v in inputs:
            v.tensor = torch.empty(v.shape, dtype=v.dtype, device=self.device)
        for v in self.vals.values():
            if v.win is not None:
                # kernels take the root buffer plus the (offset, total) window
                v.tensor = self.vals[v.win[0]].tensor
        for v in self.vals.values():
            if v.alias is not None:
                base = self._storage(v.nid)
                v.tensor = base.tensor.reshape(v.shape)

    # -- launches --------------------------------------------------------------
    def _emit(self, name, fn, nbytes: int = 0, flops: int = 0, desc: str = ""):
        """Append a launch; ``nbytes`` = its algorithmic HBM bytes (what the
        kernel must read and write once), ``flops`` its algorithmic FLOPs
        (2 per MAC; convs / dense), ``desc`` a shape summary."""
        self.launches.append(fn)
        self.launch_names.append(name)
        self.launch_bytes.append(int(nbytes))
        self.launch_flops.append(int(flops))
        self.launch_desc.append(desc)

    def _conv_work(self, n, c, h, w, k, r, s, stride, pad, es, residual=False, kb=None):
        """(flops, algorithmic bytes, desc) of one conv:
        FLOP = 2 N K C R S OH OW; bytes = (in + weights + out [+ residual])."""
        sh, sw = stride
        ph, pw = pad
        oh = (h + 2 * ph - r) // sh + 1
        ow = (w + 2 * pw - s) // sw + 1
        flops = 2 * n * k * c * r * s * oh * ow
        out = n * k * oh * ow
        nbytes = es * (n * c * h * w + k * c * r * s + out * (2 if residual else 1))
        desc = (f"{r}x{s}/{sh} C{c} K{k if kb is None else kb} {h}x{w}->{oh}x{ow} n{n}"
                + (" +res" if residual else ""))
        return flops, nbytes, desc

    def _upload(self, arr, dtype=None):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(self.device)
        if dtype is not None and dtype != torch.float32:
            t = t.to(dtype)
        self.weights.append(t)
        return t

    def _bind(self):
        from . import device as D
        g = self.g
        self.junction_bound: set[int] = set()
        for nid in self.plan.order:
            node = g.nodes[nid]
            kind = node.kind
            if nid in self.skip or kind in (OpKind.Input, OpKind.Constant, OpKind.Flatten):
                continue
            out = self.vals[nid]
            ins = [self.vals.get(src) for src, _ in node.inputs]
            if kind == OpKind.Conv2d and nid in self.sibling_of:
                continue                      # launched with its sibling
            if kind == OpKind.Conv2d and nid in self.junction_of and \
                    self.junction_of[nid] in self.junction_bound:
                continue                      # launched with its expand conv
            if kind == OpKind.Conv2d and nid in self.junction:
                if self._bind_junction(node, g.nodes[self.junction[nid]]):
                    self.junction_bound.add(nid)
                    continue
            if kind == OpKind.Conv2d and nid in self.sibling:
                self._bind_conv_pair(node, g.nodes[self.sibling[nid][0]], self.sibling[nid][1])
            elif kind == OpKind.Conv2d:
                self._bind_conv(node, out)
            elif kind == OpKind.LayoutTransform:
                if out.alias is None:
                    self._bind_transform(node, ins[0], out)
            elif nid in self.fused_head:
                self._bind_head(self.fused_head[nid], out)
            elif nid in self.fused_stem:
                self._bind_stem(node, out)
            elif kind in (OpKind.MaxPool, OpKind.AvgPool):
                self._bind_pool(node, ins[0], out)
            elif kind == OpKind.ReLU and nid in self.fused_dense_relu:
                dn = g.nodes[self.fused_dense_relu[nid]]
                self._bind_dense(dn, self.vals[dn.inputs[0][0]], out, relu=True)
            elif kind == OpKind.ReLU:
                if nid in self.fused_bn_relu:
                    bn = g.nodes[self.fused_bn_relu[nid]]
                    self._bind_scale_shift(bn, self.vals[bn.inputs[0][0]], out, relu=True)
                else:
                    self._bind_eltwise(D_ELT_RELU, ins[0], None, out)
            elif kind == OpKind.BatchNorm:
                self._bind_scale_shift(node, ins[0], out, relu=False)
            elif kind == OpKind.ElementwiseAdd:
                if ins[0].shape != ins[1].shape:
                    raise ShapeMismatch(f"add {nid}: {ins[0].shape} vs {ins[1].shape}",
                                        node_id=nid)
                self._bind_eltwise(D_ELT_ADD, ins[0], ins[1], out)
            elif kind == OpKind.Concat:
                self._bind_concat(node, ins, out)
            elif kind == OpKind.Dense:
                self._bind_dense(node, ins[0], out)
            elif kind == OpKind.Softmax:
                self._bind_softmax(ins[0], out)
            else:
                raise InputMismatch(f"cannot execute node kind {kind}")
        self._bind_workspace()
        # graph outputs / kept values that ended up in bf16 get an f32 copy
        self.out_vals = []
        for o in list(g.outputs) + self.keep:
            v = self.vals[o]
            self.out_vals.append(v)
        del D

    def _bind_workspace(self):
        """One split-K workspace shared by every tensor-core conv (they run
        in order on one stream), sized for the largest."""
        import torch
        from . import device as D
        need = max((D.conv_workspace_bytes(p) for p in self.tc_params), default=0)
        self.workspace_bytes = need
        self.workspace = None
        if need:
            self.workspace = torch.zeros(need // 4 + 1, dtype=torch.float32, device=self.device)
            for p in self.tc_params:
                D.set_workspace(p, self.workspace)

    # conv ---------------------------------------------------------------------
    def _bind_conv_pair(self, na, nb, tile_n: int):
        """Two sibling 1x1 convs over one input as one tensor-core launch:
        weights and epilogue vectors concatenated along the output channels,
        channels [0, K_a) -> a's map, [K_a, K_a + K_b) -> b's map, each with its
        own relu (kernels.py:185-197 order per channel)."""
        from . import _lib as L
        from . import device as D
        g = self.g
        data = self.vals[na.inputs[0][0]]
        oa, ob = self.vals[na.id], self.vals[nb.id]
        parts = []
        for node in (na, nb):
            epi = dict(node.attrs.get("epilogue") or {})
            kcrs = self._conv_kcrs(node.id)
            k = kcrs.shape[0]
            bias = epi.get("bias")
            if len(node.inputs) >= 3:
                bb = g.nodes[node.inputs[2][0]].attrs["value"]
                bias = bb if bias is None else bias + bb
            scale, shift = epi.get("scale"), epi.get("shift")
            parts.append({"w": kcrs, "k": k, "bias": bias, "scale": scale, "shift": shift,
                          "relu": bool(epi.get("relu"))})
        ka = parts[0]["k"]
        cat = lambda key, fill: (None if all(p_[key] is None for p_ in parts) else np.concatenate(
            [np.asarray(p_[key], np.float32) if p_[key] is not None
             else np.full(p_["k"], fill, np.float32) for p_ in parts]))
        scale, shift, bias = cat("scale", 1.0), cat("shift", 0.0), cat("bias", 0.0)
        if scale is not None and shift is None:
            shift = np.zeros(scale.shape, np.float32)
        if shift is not None and scale is None:
            scale = np.ones(shift.shape, np.float32)
        vec = lambda v: None if v is None else self._upload(v)
        w = np.concatenate([parts[0]["w"], parts[1]["w"]])
        k, c = w.shape[0], w.shape[1]
        n, _, h, wd = self.specs[na.inputs[0][0]].logical_nchw
        ic_bn, oc_bn = data.px, oa.layout.x
        mode = self._lib_mode()
        qscales = None
        if self.mode == "fp8":
            wdev, scale = self._pack_fp8(w, ic_bn, self._scale_of(na.inputs[0][0]), scale)
            qscales = (0.0, self._scale_of(na.id), self._scale_of(nb.id))
        else:
            wdev = D.pack_weights_umma(self._upload(w), ic_bn, mode)
        self.weights.append(wdev)
        flags = self.round_flag | L.FLAG_STATIC_WEIGHTS
        p = D.conv_params(mode, data.tensor, wdev, oa.tensor, n, c, h, wd, k, 1, 1,
                          hw_pair(na.attrs["stride"]), (0, 0), ic_bn, oc_bn, vec(scale),
                          vec(shift), vec(bias), None, parts[0]["relu"],
                          x_cb=self._window(data), out_cb=self._window(oa), flags=flags,
                          tile=self._sibling_tile_params(tile_n, c, ic_bn),
                          second=(ob.tensor, ka, parts[1]["relu"], self._window(ob)),
                          qscales=qscales)
        self.tc_params.append(p)
        es = bytes_per_elem(self.mode)
        fl, nbytes, desc = self._conv_work(n, c, h, wd, k, 1, 1, hw_pair(na.attrs["stride"]),
                                           (0, 0), es, kb=f"{ka}+{k - ka}")
        self._emit(f"conv{na.id}+{nb.id}", lambda p=p: D.conv2d(p, self.stream), nbytes, fl, desc)

    def _sibling_tile_params(self, tile_n: int, c: int, ic_bn: int) -> dict:
        """Tile parameters of a merged sibling launch (it has no schedule-DB
        entry of its own).  Short reductions (<= 4 channel-block slices: the
        56x56 stride-2 pair of ResNet-50, C = 256) get two slices per stage
        and two stages: the kernel's own choice keeps the full four-group
        epilogue staging and squeezes the ring to 2 x 32 KB (42.5 us isolated
        at b64 against 30.1 us; `tools/conv_bench.py --sweep` on the merged
        C256 -> K640 workload); longer reductions keep the kernel's choice,
        which the same sweep finds best."""
        tile = {"tile_n": tile_n}
        if self.mode == "bf16" and tile_n <= 128 and -(-c // ic_bn) <= 4:
            tile.update({"slices_per_stage": 2, "stages": 2})
        return tile

    def _bind_junction(self, ne, nr) -> bool:
        """Expand conv ``ne`` (+ residual) and reduce conv ``nr`` as one
        neo_conv_junction launch; False (bind them separately) when a window
        or the kernel's shape limits rule it out."""
        from . import _lib as L
        from . import device as D
        g = self.g
        x, y1, y2 = self.vals[ne.inputs[0][0]], self.vals[ne.id], self.vals[nr.id]
        res = self.vals[ne.inputs[-1][0]]
        if any(v.win is not None or v.alias is not None for v in (x, y1, y2, res)):
            return False
        if any(v.px != 64 for v in (x, y1, y2, res)):
            return False
        w1, w2 = self._conv_kcrs(ne.id), self._conv_kcrs(nr.id)
        n1, c1 = w1.shape[:2]
        n2 = w2.shape[0]
        n, _, h, w = self.specs[ne.inputs[0][0]].logical_nchw

        def bias_of(node, k):
            epi = node.attrs.get("epilogue") or {}
            b = epi.get("bias")
            extra = 1 if epi.get("residual") else 0
            if len(node.inputs) - extra >= 3:
                bb = g.nodes[node.inputs[2][0]].attrs["value"]
                b = bb if b is None else b + bb
            return None if b is None else self._upload(np.asarray(b, np.float32))

        b1, b2 = bias_of(ne, n1), bias_of(nr, n2)
        wd1 = D.pack_weights_umma(self._upload(w1), 64, L.MODE_BF16)
        wd2 = D.pack_weights_umma(self._upload(w2), 64, L.MODE_BF16)
        self.weights += [wd1, wd2]
        relu1 = bool((ne.attrs.get("epilogue") or {}).get("relu"))
        relu2 = bool((nr.attrs.get("epilogue") or {}).get("relu"))
        xt, rt, y1t, y2t = x.tensor, res.tensor, y1.tensor, y2.tensor
        fl1, nb1, d1 = self._conv_work(n, c1, h, w, n1, 1, 1, (1, 1), (0, 0), 2, residual=True)
        fl2, nb2, d2 = self._conv_work(n, n1, h, w, n2, 1, 1, (1, 1), (0, 0), 2)
        self._emit(f"conv{ne.id}>{nr.id}", lambda: D.conv_junction(
            xt, wd1, b1, rt, y1t, wd2, b2, y2t, n, c1, h, w, n1, n2, relu1, relu2, self.stream),
            nb1 + nb2 - _nb(y1t), fl1 + fl2, f"junction [{d1}] > [{d2}]")
        return True

    def _bind_conv(self, node, out: _Val):
        import torch
        from . import _lib as L
        from . import device as D
        g = self.g
        data_id = self.pro_src.get(node.inputs[0][0], node.inputs[0][0])
        data = self.vals[data_id]
        wv = g.nodes[node.inputs[1][0]].attrs["value"]
        epi = dict(node.attrs.get("epilogue") or {})
        extra = 1 if epi.get("residual") else 0
        res = self.vals[node.inputs[-1][0]] if extra else None
        bias = epi.get("bias")
        if len(node.inputs) - extra >= 3:   # executor.py:63-66: explicit bias input
            b = g.nodes[node.inputs[2][0]].attrs["value"]
            bias = b if bias is None else bias + b
        sh, sw = hw_pair(node.attrs["stride"])
        ph, pw = hw_pair(node.attrs["pad"])
        dspec = self.specs[data_id]
        n, c, h, w = dspec.logical_nchw
        if wv.ndim == 6:
            kcrs = host_unpack_kcrs(wv)
        else:
            kcrs = np.asarray(wv, np.float32)
        k, wc, r, s = kcrs.shape
        fold = self.stem_fold.get(node.inputs[0][0])
        if fold is not None:
            # W'[k, s*C + c, r, 0] = W[k, c, r, s]; width taps became channels
            kcrs = np.ascontiguousarray(
                kcrs.transpose(0, 3, 1, 2).reshape(k, s * wc, r, 1), dtype=np.float32)
            k, wc, r, s = kcrs.shape
            c, w, sw, pw = fold["F"], fold["ow"], 1, 0
        if data.layout.tag == "NCHWc":
            ic_bn = data.px
            oc_bn = out.layout.x
        else:   # NCHW data: the naive path, NCHW == NCHW[1]c
            ic_bn, oc_bn = 1, 1
        c = min(c, wc)              # channel-padded input: only wc real channels
        pad_c = c % ic_bn != 0
        use_tc = data.layout.tag == "NCHWc" and tc_legal_block(ic_bn, self.mode)
        scale, shift = epi.get("scale"), epi.get("shift")
        if scale is None and shift is not None:
            scale = np.ones(k, np.float32)
        if scale is not None and shift is None:
            shift = np.zeros(k, np.float32)
        vec = lambda v: None if v is None else self._upload(np.asarray(v, np.float32))
        t_scale, t_shift, t_bias = vec(scale), vec(shift), vec(bias)
        sched = node.attrs.get("schedule") or {}
        from .kernels import TILE_FIELDS
        tile = {f: sched.get(f, 0) for f in TILE_FIELDS}
        if fold is not None:      # tuned for the unfolded workload: let the kernel pick
            tile = {}
        if use_tc:
            mode = self._lib_mode()
            qscales = None
            if self.mode == "fp8" and data.tensor.dtype == torch.float8_e4m3fn:
                wd, scale = self._pack_fp8(kcrs, ic_bn, self._scale_of(data_id), scale,
                                           pad_channels=pad_c)
                t_scale = vec(scale)
                qscales = (self._scale_of(node.inputs[-1][0]) if res is not None else 0.0,
                           self._scale_of(node.id), 0.0)
            elif self.mode == "fp8":
                # a bf16 input (the folded 3-channel image of a VGG-style
                # stem): bf16 operands, e4m3 output entering the fp8 chain
                mode = L.MODE_BF16
                if res is not None:
                    raise InputMismatch(f"fp8 mode: conv {node.id} on a bf16 input with a residual")
                wd = D.pack_weights_umma(self._upload(kcrs), ic_bn, mode, pad_channels=pad_c)
                qscales = (0.0, self._scale_of(node.id), 0.0)
            else:
                wk = self._upload(kcrs)
                wd = D.pack_weights_umma(wk, ic_bn, mode, pad_channels=pad_c)
            self.weights.append(wd)
            x_t, o_t = data.tensor, out.tensor
            r_t = None
            if res is not None:
                r_t = res.tensor if res.tensor.dtype == o_t.dtype else self._as_f32(res)
            # weights are packed here, at load time: the conv may prefetch its
            # resident weight image before waiting on the previous kernel
            flags = self.round_flag | (L.FLAG_PAD_CHANNELS if pad_c else 0) | L.FLAG_STATIC_WEIGHTS
            pro = None
            if node.id in self.prologue:      # BN -> ReLU applied on the smem tiles
                ps, pt = self._bn_scale_shift(g.nodes[self.prologue[node.id]])
                pro = (self._upload(ps), self._upload(pt), True)
                tile["tile_n"] = min(tile.get("tile_n") or 0, 128)
                tile["cta_pair"] = 0
            p = D.conv_params(mode, x_t, wd, o_t, n, c, h, w, k, r, s, (sh, sw), (ph, pw),
                              ic_bn, oc_bn, t_scale, t_shift, t_bias, r_t,
                              bool(epi.get("relu")), x_cb=self._window(data),
                              out_cb=self._window(out), flags=flags,
                              tile=tile if any(tile.values()) else None, prologue=pro,
                              qscales=qscales)
            self.tc_params.append(p)
            es = bytes_per_elem(self.mode)
            fl, nbytes, desc = self._conv_work(n, c, h, w, k, r, s, (sh, sw), (ph, pw), es,
                                               residual=res is not None)
            self._emit(f"conv{node.id}", lambda p=p: D.conv2d(p, self.stream), nbytes, fl, desc)
            return
        # SIMT fp32 path (fp32 mode, NCHW data, or tensor-core-illegal blocks)
        if ic_bn > 1 or oc_bn > 1:
            wpk = wv if wv.ndim == 6 else None
            if wpk is None or wpk.shape[4] != ic_bn or wpk.shape[5] != oc_bn:
                from .layout import host_pack_kcrs
                wpk = host_pack_kcrs(kcrs, ic_bn, oc_bn)
        else:
            wpk = kcrs
        wdev = self._upload(wpk)
        x_t = self._as_f32(data)
        r_t = self._as_f32(res) if res is not None else None
        o_t = out.tensor if out.tensor.dtype == torch.float32 else torch.empty(
            out.shape, dtype=torch.float32, device=self.device)
        if o_t is not out.tensor:
            self.weights.append(o_t)
        p = D.conv_params(L.MODE_FP32, x_t, wdev, o_t, n, c, h, w, k, r, s, (sh, sw), (ph, pw),
                          ic_bn, oc_bn, t_scale, t_shift, t_bias, r_t, bool(epi.get("relu")),
                          x_cb=self._window(data) if x_t is data.tensor else (0, 0),
                          out_cb=self._window(out) if o_t is out.tensor else (0, 0),
                          flags=self.round_flag)
        fl, nbytes, desc = self._conv_work(n, c, h, w, k, r, s, (sh, sw), (ph, pw), 4,
                                           residual=res is not None)
        self._emit(f"conv{node.id}_simt", lambda p=p: D.conv2d(p, self.stream), nbytes, fl, desc)
        if o_t is not out.tensor:
            self._emit_convert(o_t, out.tensor)

    def _lib_mode(self) -> int:
        from . import _lib as L
        return {"bf16": L.MODE_BF16, "tf32": L.MODE_TF32, "fp8": L.MODE_FP8}[self.mode]

    def _scale_of(self, nid: int) -> float:
        """e4m3 scale of the map node ``nid`` stores (fp8 mode); a concat
        window stores at its buffer's scale (quant.attach_scales gives every
        member of a concat group the group's scale)."""
        v = self._storage(nid)
        key = v.nid if v is not None else nid
        if v is not None and v.win is not None:
            key = v.win[0]
        if key not in self.qscale:
            raise InputMismatch(f"fp8 mode: node {key} has no e4m3 scale (compile the graph "
                                f"with compile_graph(..., mode='fp8'))")
        return self.qscale[key]

    def _pack_fp8(self, kcrs, ic_bn: int, x_scale: float, bn_scale, pad_channels=False):
        """e4m3 weight image (per-output-channel scales, quant.weight_scales)
        and the epilogue scale vector x_scale * wscale[k] (* BN scale)."""
        from . import device as D
        from .quant import weight_scales
        ws = weight_scales(kcrs)
        wd = D.pack_weights_umma_fp8(self._upload(kcrs), self._upload(ws), ic_bn,
                                     pad_channels=pad_channels)
        sc = np.float32(x_scale) * ws
        if bn_scale is not None:
            sc = sc * np.asarray(bn_scale, np.float32)
        return wd, sc.astype(np.float32)

    def _no_fp8(self, what: str, *tensors):
        import torch
        if any(t is not None and t.dtype == torch.float8_e4m3fn for t in tensors):
            raise InputMismatch(f"fp8 mode: {what} on e4m3 maps is not supported (the fp8 "
                                f"mode covers conv / fused-stem / fused-head graphs)")

    def _as_f32(self, v: _Val):
        import torch
        self._no_fp8("conversion to f32", v.tensor)
        if v.tensor.dtype == torch.float32:
            return v.tensor
        t = torch.empty(v.shape, dtype=torch.float32, device=self.device)
        self.weights.append(t)
        self._emit_convert(v.tensor, t)
        return t

    def _emit_convert(self, src, dst):
        from . import _lib as L
        from . import device as D
        self._no_fp8("dtype conversion", src, dst)
        numel = src.numel()
        self._emit("convert", lambda: L.call(
            "neo_layout_transform", D.dtype_code(src), D.dtype_code(dst), src.data_ptr(),
            dst.data_ptr(), 1, numel, 1, 1, L.NCHW_TAG, 1, L.NCHW_TAG, 1, 0,
            D.stream_handle(self.stream)), _nb(src) + _nb(dst))

    def _bind_stem(self, pool_node, out: _Val):
        """conv 7x7/2 (+ epilogue) -> max pool 3x3/2 of a <=4-channel image as
        one neo_stem_conv_pool launch (reference: conv_blocked + _pool2d)."""
        from . import device as D
        g = self.g
        cv_id, src_id = self.fused_stem[pool_node.id]
        node = g.nodes[cv_id]
        src = self.vals[src_id]
        epi = dict(node.attrs.get("epilogue") or {})
        bias = epi.get("bias")
        if len(node.inputs) >= 3:           # executor.py:63-66: explicit bias input
            b = g.nodes[node.inputs[2][0]].attrs["value"]
            bias = b if bias is None else bias + b
        scale, shift = epi.get("scale"), epi.get("shift")
        if scale is None and shift is not None:
            scale = np.ones(64, np.float32)
        vec = lambda v: None if v is None else self._upload(np.asarray(v, np.float32))
        t_scale, t_shift, t_bias = vec(scale), vec(shift), vec(bias)
        w = g.nodes[node.inputs[1][0]].attrs["value"]
        w = np.asarray(host_unpack_kcrs(w) if w.ndim == 6 else w, np.float32)
        wimg = D.pack_stem_weights(self._upload(w))
        self.weights.append(wimg)
        n, c, h, wd = src.shape
        x_t, o_t = src.tensor, out.tensor
        y = out.layout.x
        cb = self._window(out)
        relu = bool(epi.get("relu"))
        self.input_readers.setdefault(src_id, []).append("stem")
        kr, ks = w.shape[2], w.shape[3]
        fl, _, desc = self._conv_work(n, c, h, wd, w.shape[0], kr, ks,
                                      hw_pair(node.attrs["stride"]), hw_pair(node.attrs["pad"]), 2)
        qs = self._scale_of(pool_node.id) if self.mode == "fp8" else 1.0
        self._emit(f"stem{cv_id}_pool{pool_node.id}", lambda: D.stem_conv_pool(
            self._input_of(src_id, x_t), wimg, o_t, n, c, h, wd, y, t_scale, t_shift, t_bias,
            relu, cb, self.stream, out_scale=qs),
            _nb(x_t) + _vb(out) + _nb(wimg), fl, desc + " + maxpool 3x3/2")

    def _bind_head(self, info: dict, out: _Val):
        """Global avg pool -> dense (+bias) -> softmax as one
        neo_classifier_head launch (reference: _pool2d, Dense, Softmax)."""
        import torch
        from . import device as D
        g = self.g
        src = self.vals[info["src"]]
        if src.win is not None or src.tensor.dtype not in (torch.bfloat16, torch.float8_e4m3fn) \
                or out.tensor.dtype != torch.float32:
            raise InputMismatch(f"fused head {info['anchor']}: unsupported operand storage")
        dn = g.nodes[info["dense"]]
        w = np.asarray(g.nodes[dn.inputs[1][0]].attrs["value"], np.float32)
        units, c = w.shape
        w_t = self._upload(w, torch.bfloat16)
        b_t = self._upload(g.nodes[dn.inputs[2][0]].attrs["value"]) if len(dn.inputs) == 3 else None
        n, cb, h, wd, y = src.shape
        scratch = D.HeadScratch(n, c, units, self.device)
        self.weights.append(scratch)
        x_t, o_t, sm = src.tensor, out.tensor, info["softmax"]
        xs = self._scale_of(info["src"]) if self.mode == "fp8" else 1.0
        self._emit(f"head{info['anchor']}", lambda: D.classifier_head(
            x_t, w_t, b_t, o_t, n, c, h * wd, y, units, sm, scratch, self.stream, x_scale=xs),
            _nb(x_t) + _nb(w_t) + _nb(o_t), 2 * n * units * c,
            f"avgpool {h}x{wd} + dense {c}->{units}" + (" + softmax" if sm else "") + f" n{n}")

    # other operators ---------------------------------------------------------
    def _bind_transform(self, node, src: _Val, out: _Val):
        import torch
        from . import _lib as L
        from . import device as D
        if src.tensor.dtype == torch.float8_e4m3fn and out.layout.tag == "NCHW" \
                and src.layout.tag == "NCHWc" and out.tensor.dtype != torch.float8_e4m3fn:
            # the fp8 chain's exit: decode e4m3 * scale into NCHW f32 / bf16
            n, c, h, w = self.specs[node.inputs[0][0]].logical_nchw
            s8 = self._scale_of(node.inputs[0][0])
            s_t, d_t, cbw = src.tensor, out.tensor, self._window(src)
            self._emit(f"dequant{node.id}", lambda: D.dequant_fp8(
                s_t, d_t, s8, n, c, h, w, src.px, cbw, self.stream), _vb(src) + _nb(d_t))
            return
        self._no_fp8("layout transform", src.tensor, out.tensor)
        if node.id in self.stem_fold:
            f = self.stem_fold[node.id]
            s_t, d_t = src.tensor, out.tensor
            self._emit(f"stemfold{node.id}", lambda: D.stem_fold(
                s_t, d_t, f["n"], f["C"], f["h"], f["w"], f["S"], f["sw"], f["pw"], f["ow"],
                f["xf"], self.round_flag, self.stream), _nb(s_t) + _nb(d_t))
            return
        n, c, h, w = self.specs[node.inputs[0][0]].logical_nchw
        src_layout = src.layout
        dst_layout = Layout.parse(node.attrs["dst_layout"])
        s_tag = src_layout if src_layout.tag != "NCHWc" else Layout("NCHWc", x=src.px)
        d_tag = dst_layout if dst_layout.tag != "NCHWc" else Layout("NCHWc", x=out.px)
        flags = 0
        if node.attrs.get("pad_channels") or out.nid in self.phys_x:
            flags |= L.FLAG_PAD_CHANNELS
        if out.tensor.dtype.is_floating_point and out.layout.tag == "NCHWc":
            flags |= self.round_flag
        s_t, d_t = src.tensor, out.tensor
        self._emit(f"transform{node.id}", lambda: D.layout_transform(
            s_t, d_t, n, c, h, w, s_tag, d_tag, flags, self.stream), _nb(s_t) + _nb(d_t))

    def _geom(self, v: _Val):
        """(n, channel blocks, h, w, lanes) of a feature-map value."""
        if v.layout.tag == "NCHWc":
            n, cb, h, w, x = v.shape
            return n, cb, h, w, x
        if len(v.shape) == 4:
            n, c, h, w = v.shape
            return n, c, h, w, 1
        # matrices / vectors: channel-free elementwise over all elements
        return 1, 1, 1, int(np.prod(v.shape)), 1

    def _bind_pool(self, node, src: _Val, out: _Val):
        import torch
        from . import device as D
        if src.tensor.dtype == torch.float8_e4m3fn:
            # e4m3 pooling: dequantize, pool (max / reference-order average),
            # requantize at the output's scale (a max pool that keeps its
            # input's scale copies the winning bytes)
            if out.tensor.dtype != torch.float8_e4m3fn:
                self._no_fp8("pooling into a non-e4m3 map", src.tensor)
            n, cb, h, w, x = self._geom(src)
            mode = "max" if node.kind == OpKind.MaxPool else "avg"
            win, st, pad = node.attrs["window"], node.attrs["stride"], node.attrs.get("pad", 0)
            s_t, d_t, iw, ow = src.tensor, out.tensor, self._window(src), self._window(out)
            si, so = self._scale_of(src.nid), self._scale_of(node.id)
            self._emit(f"{mode}pool{node.id}", lambda: D.pool2d_q(
                s_t, d_t, n, cb, h, w, x, win, st, pad, mode, iw, ow, si, so, self.stream),
                _vb(src) + _vb(out))
            return
        self._no_fp8("pooling", src.tensor, out.tensor)
        n, cb, h, w, x = self._geom(src)
        mode = "max" if node.kind == OpKind.MaxPool else "avg"
        win, st, pad = node.attrs["window"], node.attrs["stride"], node.attrs.get("pad", 0)
        flags = self.round_flag if src.layout.tag == "NCHWc" else 0
        s_t, d_t = src.tensor, out.tensor
        nb = _vb(src) + _vb(out)
        if src.win is not None or out.win is not None:
            iw, ow = self._window(src), self._window(out)
            self._emit(f"{mode}pool{node.id}", lambda: D.pool2d_window(
                s_t, d_t, n, cb, h, w, x, win, st, pad, mode, iw, ow, flags, self.stream), nb)
            return
        self._emit(f"{mode}pool{node.id}", lambda: D.pool2d(
            s_t, d_t, n, cb, h, w, x, win, st, pad, mode, flags, self.stream), nb)

    def _bind_eltwise(self, op, a: _Val, b: _Val | None, out: _Val):
        import torch
        from . import device as D
        if a.tensor.dtype == torch.float8_e4m3fn and b is None and op == D_ELT_RELU \
                and out.tensor.dtype == torch.float8_e4m3fn:
            n, cb, h, w, x = self._geom(a)
            a_t, o_t, aw, ow = a.tensor, out.tensor, self._window(a), self._window(out)
            sa, so = self._scale_of(a.nid), self._scale_of(out.nid)
            self._emit(f"relu{out.nid}", lambda: D.eltwise_q(
                D_ELT_RELU, a_t, o_t, n, cb, h * w, x, aw, ow, sa, so, stream=self.stream),
                _vb(a) + _vb(out))
            return
        self._no_fp8("elementwise op", a.tensor, b.tensor if b is not None else None, out.tensor)
        n, cb, h, w, x = self._geom(a)
        flags = self.round_flag if a.layout.tag == "NCHWc" else 0
        a_t, b_t, o_t = a.tensor, (b.tensor if b is not None else None), out.tensor
        nb = _vb(a) + _vb(out) + (_vb(b) if b is not None else 0)
        if b is None and (a.win is not None or out.win is not None):
            aw, ow = self._window(a), self._window(out)
            self._emit(f"eltwise{out.nid}", lambda: D.eltwise_window(
                op, a_t, o_t, n, cb, h * w, x, aw, ow, None, None, flags, self.stream), nb)
            return
        if (b is not None and b.win is not None) or a.win is not None or out.win is not None:
            raise InputMismatch(f"eltwise {out.nid}: windowed add")
        self._emit(f"eltwise{out.nid}", lambda: D.eltwise(
            op, a_t, b_t, o_t, n, cb, h * w, x, None, None, flags, self.stream), nb)

    def _bn_scale_shift(self, node):
        """Per-channel (scale, shift) of a standalone BatchNorm."""
        if len(node.inputs) == 5:   # unfolded BN (executor.py:174-178, f32 arithmetic)
            gamma, beta, mean, var = (np.asarray(self.g.nodes[s].attrs["value"], np.float32)
                                      for s, _ in node.inputs[1:])
            scale = gamma / np.sqrt(var + np.float32(node.attrs.get("eps", 1e-5)))
            shift = beta - mean * scale
        else:
            scale, shift = node.attrs["scale"], node.attrs["shift"]
        return np.asarray(scale, np.float32), np.asarray(shift, np.float32)

    def _bind_scale_shift(self, node, src: _Val, out: _Val, relu: bool):
        import torch
        from . import device as D
        from . import _lib as L
        scale, shift = self._bn_scale_shift(node)
        t_scale, t_shift = self._upload(scale), self._upload(shift)
        n, cb, h, w, x = self._geom(src)
        op = L.ELT_SCALE_SHIFT_RELU if relu else L.ELT_SCALE_SHIFT
        if src.tensor.dtype == torch.float8_e4m3fn and out.tensor.dtype == torch.float8_e4m3fn:
            # e4m3 BN(-ReLU), e.g. DenseNet's pre-activations over a concat
            # window: dequantize, a*scale+shift, relu, requantize
            a_t, o_t, aw, ow = src.tensor, out.tensor, self._window(src), self._window(out)
            sa, so = self._scale_of(src.nid), self._scale_of(out.nid)
            self._emit(f"bn{node.id}{'_relu' if relu else ''}", lambda: D.eltwise_q(
                op, a_t, o_t, n, cb, h * w, x, aw, ow, sa, so, t_scale, t_shift, self.stream),
                _vb(src) + _vb(out))
            return
        self._no_fp8("batch norm", src.tensor, out.tensor)
        flags = self.round_flag if src.layout.tag == "NCHWc" else 0
        a_t, o_t = src.tensor, out.tensor
        nb = _vb(src) + _vb(out)
        if src.win is not None or out.win is not None:
            aw, ow = self._window(src), self._window(out)
            self._emit(f"bn{node.id}{'_relu' if relu else ''}", lambda: D.eltwise_window(
                op, a_t, o_t, n, cb, h * w, x, aw, ow, t_scale, t_shift, flags, self.stream), nb)
            return
        self._emit(f"bn{node.id}{'_relu' if relu else ''}", lambda: D.eltwise(
            op, a_t, None, o_t, n, cb, h * w, x, t_scale, t_shift, flags, self.stream), nb)

    def _bind_concat(self, node, ins, out: _Val):
        import torch
        from . import device as D
        if out.tensor.dtype == torch.float8_e4m3fn:
            # e4m3 concat: every input is stored at the concat group's scale
            # (quant.attach_scales), so copies are byte copies
            so = self._scale_of(node.id)
            for (src, _), v in zip(node.inputs, ins):
                if self._scale_of(src) != so:
                    raise InputMismatch(f"fp8 concat {node.id}: input {src} has another scale")
        axis = node.attrs.get("axis", 1)
        done = self.concat_windowed.get(node.id, set())
        dst = out
        base_blocks = 0
        if out.win is not None:     # this concat is itself a window of a wider one
            dst = self.vals[out.win[0]]
            base_blocks = out.win[1]
        outer = int(np.prod(dst.shape[:axis]))
        row = int(np.prod(dst.shape[axis:]))
        plane = int(np.prod(dst.shape[2:])) if axis == 1 else 0
        off = base_blocks * plane
        for (src, _), v in zip(node.inputs, ins):
            if v.tensor.dtype != out.tensor.dtype:
                raise InputMismatch(f"concat {node.id}: mixed storage types")
            chunk = int(np.prod(v.shape[axis:]))
            if src not in done:
                if v.win is not None:
                    raise InputMismatch(f"concat {node.id}: input {src} is a foreign window")
                s_t, d_t = v.tensor, dst.tensor
                self._emit(f"concat{node.id}", lambda s_t=s_t, d_t=d_t, chunk=chunk, off=off:
                           D.concat_copy(s_t, d_t, outer, chunk, row, off, self.stream),
                           2 * _nb(s_t))
            off += chunk

    def _bind_dense(self, node, src: _Val, out: _Val, relu: bool = False):
        self._no_fp8("dense", src.tensor)    # fp8 mode: dense inputs are bf16
        import torch
        from . import _lib as L
        from . import device as D
        w = np.asarray(self.g.nodes[node.inputs[1][0]].attrs["value"], np.float32)
        units, width = w.shape
        b_t = None
        if len(node.inputs) == 3:
            b_t = self._upload(self.g.nodes[node.inputs[2][0]].attrs["value"])
        n = src.shape[0]
        if node.id in self.tc_dense and src.tensor.dtype == self.dense_dtype:
            # tensor cores: (n, width) row-major == NCHW[x]c with H = W = 1, so
            # the dense is a 1x1 conv; the output (n, units) is NCHW[y]c with
            # H = W = 1 for any y dividing units.
            x = self._dense_block(width)
            mode = L.MODE_BF16 if self.dense_mode == "bf16" else L.MODE_TF32
            wd = D.pack_weights_umma(self._upload(w.reshape(units, width, 1, 1)), x, mode)
            self.weights.append(wd)
            o_t = out.tensor
            y = next(d for d in (32, 16, 8, 4, 2, 1) if units % d == 0)
            tile = {"tile_w": 1, "tile_h": 1, "tile_img": min(n, 128),
                    "tile_n": max(16, min(256, -(-units // 148 // 16) * 16))}
            p = D.conv_params(mode, src.tensor.reshape(-1), wd, o_t.reshape(-1), n, width, 1, 1,
                              units, 1, 1, (1, 1), (0, 0), x, y, bias=b_t, relu=relu,
                              flags=self.round_flag if o_t.dtype == torch.float32 and
                              self._feeds_tc_dense(out.nid) else 0, tile=tile)
            self.tc_params.append(p)
            self._emit(f"dense{node.id}_tc", lambda p=p: D.conv2d(p, self.stream),
                       _nb(wd) + _nb(src.tensor) + _nb(o_t), 2 * n * units * width,
                       f"dense {width}->{units} n{n}")
            return
        a_t = self._as_f32(src) if self.dense_mode != "bf16" or src.tensor.dtype != torch.bfloat16 \
            else src.tensor
        w_t = self._upload(w, a_t.dtype)
        o_t = out.tensor if out.tensor.dtype == torch.float32 else torch.empty(
            out.shape, dtype=torch.float32, device=self.device)
        self._emit(f"dense{node.id}", lambda: D.dense(a_t, w_t, b_t, o_t, n, width, units,
                                                      self.stream),
                   _nb(w_t) + _nb(a_t) + _nb(o_t), 2 * n * units * width,
                   f"dense {width}->{units} n{n}")
        if relu:
            from . import _lib as L2
            self._emit(f"relu{out.nid}", lambda: D.eltwise(
                L2.ELT_RELU, o_t, None, o_t, 1, 1, o_t.numel(), 1, flags=0, stream=self.stream),
                2 * _nb(o_t))
        if o_t is not out.tensor:
            self.weights.append(o_t)
            self._emit_convert(o_t, out.tensor)

    def _bind_softmax(self, src: _Val, out: _Val):
        from . import device as D
        cols = src.shape[-1]
        rows = int(np.prod(src.shape[:-1]))
        a_t = self._as_f32(src)
        o_t = out.tensor
        self._emit(f"softmax{out.nid}", lambda: D.softmax(a_t, o_t, rows, cols, self.stream),
                   _nb(a_t) + _nb(o_t))

    # -- running -----------------------------------------------------------------
    @property
    def upload_bytes(self) -> int:
        """Host->device bytes of one batch of inputs as stored on the device."""
        return sum(_nb(self.vals[nid].tensor) for nid in self.plan.input_ids)

    def input_names(self) -> list[str]:
        return [self.g.nodes[nid].attrs.get("name", f"input{nid}") for nid in self.plan.input_ids]

    def input_tensor(self, name: str):
        for nid in self.plan.input_ids:
            if self.g.nodes[nid].attrs.get("name", f"input{nid}") == name:
                return self.vals[nid].tensor
        raise InputMismatch(f"missing input {name!r}")

    def output_tensors(self) -> list:
        return [v.tensor for v in self.out_vals]

    def _input_of(self, nid: int, default):
        """The buffer a launch reads graph input ``nid`` from in the active
        input slot (resolved when the launch is issued or captured)."""
        if self._input_slot:
            return self._alt_inputs[nid]
        return default

    def _launch_all(self):
        for i, fn in enumerate(self.launches):
            try:
                fn()
            except Exception as exc:
                # name the launch ("conv123", "bn45_relu", ...) in the error
                exc.args = (f"{self.launch_names[i]} [{self.launch_desc[i]}]: "
                            f"{exc.args[0] if exc.args else exc}",) + tuple(exc.args[1:])
                raise

    def launch(self):
        """Run the forward on ``self.stream`` (inputs already in place)."""
        import torch
        from . import device as D
        if self.use_graph and self._graphs.get(self._input_slot) is None:
            with torch.cuda.device(self.device):
                self._launch_all()                 # warm-up: sets kernel attributes
                self.stream.synchronize()
                with torch.cuda.stream(self.stream):
                    self._graphs[self._input_slot] = D.capture(self._launch_all, self.stream)
            if self._input_slot == 0:
                self.graph_exec = self._graphs[0]
        if self.use_graph:
            self._graphs[self._input_slot].launch(self.stream)
        else:
            with torch.cuda.device(self.device):
                self._launch_all()

    @property
    def kernel_launches(self) -> int:
        return len(self.launches)

    def set_inputs(self, inputs: dict):
        import torch
        for nid in self.plan.input_ids:
            node = self.g.nodes[nid]
            name = node.attrs.get("name", f"input{nid}")
            if name not in inputs:
                raise InputMismatch(f"missing input {name!r}")
            a = inputs[name]
            declared = tuple(node.attrs["shape"])
            if tuple(a.shape) != declared:
                raise InputMismatch(f"input {name!r}: shape {tuple(a.shape)} vs {declared}")
            dst = self.vals[nid].tensor
            if node.attrs.get("layout", "NCHW") == "NHWC":
                self._ingest_nhwc(a, dst)
                continue
            src = a if isinstance(a, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(a, dtype=np.float32))
            if src.is_cuda or (src.is_pinned() and src.dtype == dst.dtype):
                with torch.cuda.stream(self.stream):
                    dst.copy_(src, non_blocking=True)
                continue
            # pageable host data goes through a pinned staging buffer so the
            # upload is asynchronous (the shards of a multi-device execute()
            # upload concurrently); a bf16 input is rounded RN on the host
            # while it is copied into the staging buffer
            pin, done = self._pinned_inputs.get(nid, (None, None))
            if pin is None:
                pin = torch.empty(dst.shape, dtype=dst.dtype).pin_memory()
                done = torch.cuda.Event()
                done.record(self.stream)
                self._pinned_inputs[nid] = (pin, done)
            done.synchronize()                  # its previous upload has finished
            pin.copy_(src)
            with torch.cuda.stream(self.stream):
                dst.copy_(pin, non_blocking=True)
            done.record(self.stream)

    def _ingest_nhwc(self, a, dst):
        import torch
        from . import device as D
        src = a if isinstance(a, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(a, dtype=np.float32))
        # one staging buffer per NHWC input, reused by every call (the copy
        # and the transform are both ordered on self.stream)
        if not hasattr(self, "_nhwc_staging"):
            self._nhwc_staging = {}
        key = dst.data_ptr()
        staging = self._nhwc_staging.get(key)
        if staging is None or tuple(staging.shape) != tuple(src.shape):
            staging = torch.empty(tuple(src.shape), dtype=torch.float32, device=self.device)
            self._nhwc_staging[key] = staging
        with torch.cuda.stream(self.stream):
            staging.copy_(src, non_blocking=True)
        n, h, w, c = src.shape
        D.layout_transform(staging, dst, n, c, h, w, "NHWC", "NCHW", 0, self.stream)

    def run(self, inputs: dict) -> list[np.ndarray]:
        """Host in, host out: inputs -> device, forward, outputs -> host f32."""
        self.set_inputs(inputs)
        self.launch()
        self.stream.synchronize()
        return [t.float().cpu().numpy() for t in self.output_tensors()]

    def pipeline(self, batches, outputs):
        """Serving loop over pinned host batches: the upload of batch i+1 (a
        separate copy stream into the other of two device input buffers)
        overlaps the forward of batch i; each forward's first-output tensor
        is read back into ``outputs[i]`` (pinned host tensors).  Every copy
        is part of the loop; returns after all work is enqueued.  Inputs must
        be NCHW f32 and the graph must have a single input.  When the input is
        stored as bf16 (read only by fused stems), each batch is rounded to
        bf16 on the host into a pinned buffer before its upload.

        When the input is read only by fused stems (which resolve their input
        buffer at launch time), the two input buffers are the graph's own
        inputs -- one captured CUDA graph per buffer -- so no device-side
        staging copy runs; the result is copied to a small device staging
        buffer on the compute stream and read back on a third stream, off the
        forward's critical path.  ``upload_bytes`` is the host->device byte
        count per batch."""
        import torch
        if len(self.plan.input_ids) != 1:
            raise InputMismatch("pipeline() needs a single-input graph")
        in_id = self.plan.input_ids[0]
        dst = self.vals[in_id].tensor
        zero_copy = (self.use_graph and bool(self.input_readers.get(in_id))
                     and all(u in self.skip for u in self.users[in_id]))
        if not hasattr(self, "_staging"):
            if zero_copy:
                self._alt_inputs[in_id] = torch.empty_like(dst)
                self._staging = [dst, self._alt_inputs[in_id]]
            else:
                self._staging = [torch.empty_like(dst) for _ in range(2)]
            self._copy_stream = torch.cuda.Stream(self.device)
            self._d2h_stream = torch.cuda.Stream(self.device)
            self._copied = [torch.cuda.Event() for _ in range(2)]
            self._consumed = [torch.cuda.Event() for _ in range(2)]
            self._out_ready = [torch.cuda.Event() for _ in range(2)]
            self._out_read = [torch.cuda.Event() for _ in range(2)]
            for ev in self._consumed + self._out_read:
                ev.record(self.stream)
        out_dev = self.output_tensors()[0]
        if not hasattr(self, "_out_stage"):
            self._out_stage = [torch.empty_like(out_dev) for _ in range(2)]
        convert = dst.dtype != torch.float32
        if convert and not hasattr(self, "_host_stage"):
            # f32 host batch -> pinned bf16 (RN, multi-threaded on the host)
            # while the GPU runs the previous forward; half the PCIe bytes
            # three host buffers: the rounding of a batch may run up to three
            # batches ahead of the GPU, which absorbs host scheduling hiccups
            self._host_stage = [torch.empty(dst.shape, dtype=dst.dtype).pin_memory()
                                for _ in range(3)]
            self._host_done = [torch.cuda.Event() for _ in range(3)]
            self._host_used = [False, False, False]
        n = dst.shape[0]
        chunks = [(lo, min(n, lo + max(1, n // 4))) for lo in range(0, n, max(1, n // 4))]
        # a collector pause inside the loop would stall the uploads behind it
        import gc
        gc_was = gc.isenabled()
        gc.disable()
        try:
            self._pipeline_loop(batches, outputs, dst, out_dev, convert, chunks, zero_copy)
        finally:
            self._input_slot = 0
            if gc_was:
                gc.enable()

    def _pipeline_loop(self, batches, outputs, dst, out_dev, convert, chunks, zero_copy):
        import torch
        for i, host in enumerate(batches):
            slot = i & 1
            with torch.cuda.stream(self._copy_stream):
                self._copy_stream.wait_event(self._consumed[slot])
            if convert:
                hs = i % 3
                if self._host_used[hs]:
                    self._host_done[hs].synchronize()       # its previous upload finished
                # round and upload in batch chunks: the upload of one chunk
                # overlaps the host rounding of the next
                for lo, hi in chunks:
                    self._host_stage[hs][lo:hi].copy_(host[lo:hi])
                    with torch.cuda.stream(self._copy_stream):
                        self._staging[slot][lo:hi].copy_(self._host_stage[hs][lo:hi],
                                                         non_blocking=True)
                self._host_done[hs].record(self._copy_stream)
                self._host_used[hs] = True
            else:
                with torch.cuda.stream(self._copy_stream):
                    self._staging[slot].copy_(host, non_blocking=True)
            with torch.cuda.stream(self._copy_stream):
                self._copied[slot].record(self._copy_stream)
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(self._copied[slot])
                if zero_copy:
                    self._input_slot = slot            # the graph reading this buffer
                else:
                    dst.copy_(self._staging[slot], non_blocking=True)
            self.launch()
            with torch.cuda.stream(self.stream):
                self._consumed[slot].record(self.stream)
                # result -> small device stage (its previous readback done),
                # read back on the third stream while the next forward runs
                self.stream.wait_event(self._out_read[slot])
                self._out_stage[slot].copy_(out_dev, non_blocking=True)
                self._out_ready[slot].record(self.stream)
            with torch.cuda.stream(self._d2h_stream):
                self._d2h_stream.wait_event(self._out_ready[slot])
                outputs[i].copy_(self._out_stage[slot], non_blocking=True)
                self._out_read[slot].record(self._d2h_stream)


# ---------------------------------------------------------------------------
# reference-compatible entry points

D_ELT_RELU, D_ELT_ADD = 0, 1


def _program(plan: ExecutablePlan, device: int, mode: str, keep=()) -> DeviceProgram:
    key = (device, mode, tuple(keep))
    prog = plan.programs.get(key)
    if prog is None:
        prog = DeviceProgram(plan, device, mode, keep)
        plan.programs[key] = prog
    return prog


def with_batch(g: Graph, batch: int) -> Graph:
    """Copy of ``g`` whose Input nodes have leading dimension ``batch``."""
    h = g.copy()
    for node in h.nodes.values():
        if node.kind == OpKind.Input:
            shape = list(node.attrs["shape"])
            shape[0] = batch
            node.attrs["shape"] = tuple(shape)
    return h


def execute(plan, inputs: dict, pool=None, keep=()) -> list[np.ndarray]:
    """Run the graph; outputs in ``graph.outputs`` order (then ``keep``), in
    the default layout as host f32 arrays (executor.py:131-218).

    ``pool``: a DevicePool (devices + mode), a mode string or None.  With
    several devices the batch is split contiguously across them and each
    shard runs the same compiled graph independently (no collective)."""
    if isinstance(plan, Graph):
        plan = ExecutablePlan.compile(plan)
    dp = resolve_pool(pool)
    if dp.size == 1:
        return _program(plan, dp.device, dp.mode, keep).run(inputs)
    batch = plan.graph.nodes[plan.input_ids[0]].attrs["shape"][0]
    shards = dp.shards(batch)
    progs = []
    for dev, (lo, hi) in shards:
        sub = plan.programs.get(("shard", dev, lo, hi, dp.mode, tuple(keep)))
        if sub is None:
            sub = DeviceProgram(ExecutablePlan.compile(with_batch(plan.graph, hi - lo)), dev,
                                dp.mode, keep)
            plan.programs[("shard", dev, lo, hi, dp.mode, tuple(keep))] = sub
        import torch
        with torch.cuda.device(sub.device):
            sub.set_inputs({k: v[lo:hi] for k, v in inputs.items()})   # async (pinned)
            sub.launch()
        progs.append(sub)
    parts = []
    for sub in progs:
        sub.stream.synchronize()
        parts.append([t.float().cpu().numpy() for t in sub.output_tensors()])
    return [np.concatenate([p[i] for p in parts], axis=0) for i in range(len(parts[0]))]


def benchmark(plan, pool, inputs: dict, samples: int = 1000,
              warmups: int = 3) -> tuple[float, float]:
    """(mean_ns, stderr_ns) of end-to-end forwards (executor.py:221-236):
    each sample = inputs to device + forward + outputs to host, timed with
    CUDA events on the program's stream."""
    import torch
    if isinstance(plan, Graph):
        plan = ExecutablePlan.compile(plan)
    dp = resolve_pool(pool)
    if dp.size > 1:
        # the reference times execute(plan, inputs, pool) with the given pool
        for _ in range(max(1, warmups)):
            execute(plan, inputs, dp)
        times = np.empty(samples, dtype=np.float64)
        for i in range(samples):
            t0 = time.perf_counter_ns()
            execute(plan, inputs, dp)
            times[i] = time.perf_counter_ns() - t0
        mean = float(times.mean())
        stderr = float(times.std(ddof=1) / math.sqrt(samples)) if samples > 1 else 0.0
        return mean, stderr
    prog = _program(plan, dp.device, dp.mode)
    for _ in range(max(1, warmups)):
        prog.run(inputs)
    host = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in prog.output_tensors()]
    times = np.empty(samples, dtype=np.float64)
    for i in range(samples):
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(prog.stream)
        prog.set_inputs(inputs)
        prog.launch()
        # readback enqueued on the program stream, inside the timed window
        with torch.cuda.stream(prog.stream):
            for t, h in zip(prog.output_tensors(), host):
                h.copy_(t, non_blocking=True)
        end.record(prog.stream)
        end.synchronize()
        times[i] = start.elapsed_time(end) * 1e6
    mean = float(times.mean())
    stderr = float(times.std(ddof=1) / math.sqrt(samples)) if samples > 1 else 0.0
    return mean, stderr


def scalability_report(g: Graph, inputs: dict, samples: int, device_counts,
                       mode: str = "bf16") -> list[str]:
    """CSV lines ``gpus,samples,mean_ns,stderr_ns`` (executor.py:239-247 with
    device counts in place of thread counts); the batch is sharded."""
    import torch
    lines = []
    plan = ExecutablePlan.compile(g)
    for count in device_counts:
        count = min(count, max(1, torch.cuda.device_count()))
        pool = DevicePool(list(range(count)), mode)
        execute(plan, inputs, pool)
        times = []
        for _ in range(samples):
            t0 = time.perf_counter_ns()
            execute(plan, inputs, pool)
            times.append(time.perf_counter_ns() - t0)
        arr = np.asarray(times, np.float64)
        se = float(arr.std(ddof=1) / math.sqrt(len(arr))) if len(arr) > 1 else 0.0
        lines.append(f"{count},{samples},{arr.mean():.0f},{se:.0f}")
    return lines
