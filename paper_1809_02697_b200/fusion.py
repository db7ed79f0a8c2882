"""Fusion planning: which operators of a compiled graph share a launch.

The reference executes every operator on its own (executor.py:131-218; its
only fusion is the conv epilogue built by passes.py:119-157).  On B200 the
per-launch fill / drain and the HBM round trip of each intermediate cost more
than the math of the small operators around the convs, so the device
executor merges them.  This module owns those decisions as a pure analysis
of the compiled graph -- no device, no torch -- so they can be inspected and
tested on a CPU host (``plan_fusions``) and switched by explicit options
(``FusionOptions``) instead of scattered environment reads.

Decisions (each records node ids; ``skip`` = nodes that get no launch and no
buffer of their own):

* ``fused_bn_relu``   standalone BatchNorm whose only consumer is a ReLU: one
                      scale-shift-relu launch (DenseNet pre-activations);
* ``prologue``        such a BN-ReLU feeding only an unpadded 1x1 tensor-core
                      conv becomes that conv's shared-memory prologue
                      (opt-in: measured slower on B200);
* ``tc_dense`` / ``fused_dense_relu``  Dense layers on the tensor cores, a
                      Dense->ReLU pair as one launch;
* ``stem_fold``       a few-channel graph input packed with the stem conv's
                      horizontal taps folded into channels (neo_stem_fold);
* ``fused_stem``      7x7/2 conv + 3x3/2 max pool over the image as one
                      launch (neo_stem_conv_pool);
* ``bf16_inputs``     graph inputs read only by fused stems, uploaded as bf16;
* ``fused_head``      global avg pool -> flatten -> dense -> softmax as one
                      launch (neo_classifier_head);
* ``sibling``         two 1x1 convs over one input as one two-output launch;
* ``junction``        expand 1x1 + next reduce 1x1 in one launch (opt-in);
* ``phys_x``          physical block for tensor-core-illegal packed inputs.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from .graph import Graph, OpKind, hw_pair, infer_shapes, topo_sort
from .kernels import bytes_per_elem, tc_legal_block
from .layout import Layout, host_unpack_kcrs


@dataclass(frozen=True)
class FusionOptions:
    """Switches of the fusion planner.  Defaults are the shipped B200
    configuration; ``from_env`` reads the experiment overrides
    (NEOB200_PROLOGUE=1, NEOB200_NO_FUSED_STEM, NEOB200_NO_FUSED_HEAD,
    NEOB200_NO_SIBLING, NEOB200_JUNCTION=1, NEOB200_JUNCTION_MIN_HW)."""
    prologue: bool = False
    fused_stem: bool = True
    fused_head: bool = True
    sibling: bool = True
    junction: bool = False
    junction_min_hw: int = 0
    host_round: bool = True

    @classmethod
    def from_env(cls, host_round: bool = True) -> "FusionOptions":
        env = os.environ
        return cls(prologue=bool(env.get("NEOB200_PROLOGUE")),
                   fused_stem=not env.get("NEOB200_NO_FUSED_STEM"),
                   fused_head=not env.get("NEOB200_NO_FUSED_HEAD"),
                   sibling=not env.get("NEOB200_NO_SIBLING"),
                   junction=env.get("NEOB200_JUNCTION") == "1",
                   junction_min_hw=int(env.get("NEOB200_JUNCTION_MIN_HW", "0")),
                   host_round=host_round)


@dataclass
class FusionPlan:
    mode: str
    fused_bn_relu: dict = field(default_factory=dict)     # relu id -> bn id
    prologue: dict = field(default_factory=dict)          # conv id -> bn id
    pro_src: dict = field(default_factory=dict)           # relu id -> the BN's input
    tc_dense: set = field(default_factory=set)
    fused_dense_relu: dict = field(default_factory=dict)  # relu id -> dense id
    stem_fold: dict = field(default_factory=dict)         # transform id -> fold params
    fused_stem: dict = field(default_factory=dict)        # pool id -> (conv, input)
    bf16_inputs: set = field(default_factory=set)
    fused_head: dict = field(default_factory=dict)        # anchor id -> info
    sibling: dict = field(default_factory=dict)           # first conv -> (second, tile_n)
    sibling_of: dict = field(default_factory=dict)        # second -> first
    junction: dict = field(default_factory=dict)          # expand conv -> reduce conv
    junction_of: dict = field(default_factory=dict)       # reduce conv -> expand conv
    phys_x: dict = field(default_factory=dict)            # transform id -> physical block
    skip: set = field(default_factory=set)

    def summary(self) -> dict:
        """Counts per decision (reported by the CLI / tests)."""
        return {"bn_relu": len(self.fused_bn_relu), "prologue": len(self.prologue),
                "tc_dense": len(self.tc_dense), "dense_relu": len(self.fused_dense_relu),
                "stem_fold": len(self.stem_fold), "fused_stem": len(self.fused_stem),
                "bf16_inputs": len(self.bf16_inputs), "fused_head": len(self.fused_head),
                "sibling": len(self.sibling), "junction": len(self.junction),
                "phys_x": len(self.phys_x), "skipped": len(self.skip)}


def dense_mode_of(mode: str) -> str:
    """Dense layers and folded image stems run bf16 in fp8 mode."""
    return "bf16" if mode == "fp8" else mode


def conv_kcrs(g: Graph, nid: int) -> np.ndarray:
    """The conv's logical KCRS f32 weights (unpacking a pre-packed image)."""
    wv = g.nodes[g.nodes[nid].inputs[1][0]].attrs["value"]
    return host_unpack_kcrs(wv) if wv.ndim == 6 else np.asarray(wv, np.float32)


def dense_block(width: int, dense_mode: str) -> int:
    """Legal tensor-core block dividing a dense input width (0 if none)."""
    for x in (64, 32, 16, 8, 4):
        if width % x == 0 and tc_legal_block(x, dense_mode):
            return x
    return 0


def plan_fusions(g: Graph, mode: str, keep=(), options: FusionOptions | None = None,
                 specs: dict | None = None, users: dict | None = None,
                 order: list | None = None) -> FusionPlan:
    """Fusion decisions for compiled graph ``g`` run in ``mode`` ("bf16",
    "tf32", "fp32", "fp8").  Nodes in ``keep`` (and graph outputs) are never
    fused away: their values stay readable."""
    a = _Analysis(g, mode, keep, options or FusionOptions(),
                  specs if specs is not None else infer_shapes(g),
                  users if users is not None else g.consumers(),
                  order if order is not None else topo_sort(g))
    a.run()
    return a.plan


class _Analysis:
    def __init__(self, g, mode, keep, opts, specs, users, order):
        self.g, self.mode, self.keep, self.opts = g, mode, list(keep), opts
        self.specs, self.users, self.order = specs, users, order
        self.dense_mode = dense_mode_of(mode)
        self.plan = p = FusionPlan(mode)
        # the rules below read each other's decisions through these names
        self.skip, self.prologue, self.pro_src = p.skip, p.prologue, p.pro_src
        self.fused_dense_relu, self.stem_fold = p.fused_dense_relu, p.stem_fold
        self.sibling, self.sibling_of = p.sibling, p.sibling_of

    def run(self):
        g, p, order, users = self.g, self.plan, self.order, self.users
        tc_mode = self.mode in ("bf16", "tf32", "fp8")
        for nid in order:
            node = g.nodes[nid]
            if node.kind == OpKind.BatchNorm and len(node.inputs) == 1:
                us = users[nid]
                if (len(us) == 1 and g.nodes[us[0]].kind == OpKind.ReLU
                        and nid not in g.outputs and nid not in self.keep):
                    p.fused_bn_relu[us[0]] = nid
                    p.skip.add(nid)
        # BN -> ReLU feeding only the data input of an unpadded 1x1 conv on the
        # tensor cores can become the conv's shared-memory prologue (DenseNet
        # pre-activation; neither the BN nor the ReLU value is materialised).
        # Opt-in: on B200 the in-smem rewrite sits on the critical path of
        # every pipeline stage and costs more than the HBM-speed
        # scale-shift-relu launches it removes (DenseNet-201 b32: 2.75 ms
        # without, 4.25 ms with the round-2 rewrite -- per-slice parameters in
        # registers, bit-identical to the unfused path; 5.2 ms with the
        # round-1 rewrite).
        if self.mode in ("bf16", "tf32") and self.opts.prologue:
            self._plan_prologues()
        # Dense layers run as 1x1 tensor-core convs over their row-major input
        # ((N, F) == NCHW[x]c with H = W = 1); a Dense whose only consumer is a
        # ReLU writes the ReLU's value with the relu fused into the epilogue.
        if tc_mode:
            for nid in order:
                node = g.nodes[nid]
                if node.kind != OpKind.Dense:
                    continue
                width = g.nodes[node.inputs[1][0]].attrs["value"].shape[1]
                if dense_block(width, self.dense_mode):
                    p.tc_dense.add(nid)
                us = users[nid]
                if (len(us) == 1 and g.nodes[us[0]].kind == OpKind.ReLU
                        and nid not in g.outputs and nid not in self.keep):
                    p.fused_dense_relu[us[0]] = nid
                    p.skip.add(nid)
        # 3-channel image stems: fold the kernel's horizontal taps into
        # channels (neo_stem_fold) so the first conv reads 64-byte rows
        if tc_mode:
            for nid in order:
                info = self._stem_fold_info(nid)
                if info:
                    p.stem_fold[nid] = info
        # image stem (7x7/2 conv + relu + 3x3/2 max pool over a <=4-channel
        # input) as one fused launch: neither the packed input nor the conv
        # map is materialised (neo_stem_conv_pool)
        if self.mode in ("bf16", "fp8") and self.opts.fused_stem:
            for t, info in list(p.stem_fold.items()):
                found = self._fused_stem_info(t, info)
                if found:
                    cv, mp, src = found
                    p.fused_stem[mp] = (cv, src)
                    p.skip.update((t, cv))
                    del p.stem_fold[t]
        # a graph input read only by fused stems is stored as bf16: the stem
        # rounds it RN to bf16 anyway, so rounding on the host before the
        # upload gives identical results with half the host->device bytes
        stem_srcs = {src for _, src in p.fused_stem.values()} if self.opts.host_round else set()
        for src in stem_srcs:
            if all(u in p.skip for u in users[src]) and src not in g.outputs \
                    and g.nodes[src].attrs.get("layout", "NCHW") == "NCHW" \
                    and self.specs[src].logical_nchw[3] % 8 == 0:
                p.bf16_inputs.add(src)
        # classifier head (global avg pool -> flatten -> dense -> softmax) as
        # one fused launch (neo_classifier_head)
        if self.mode in ("bf16", "fp8") and self.opts.fused_head:
            for nid in order:
                info = self._fused_head_info(nid)
                if info:
                    p.fused_head[info["anchor"]] = info
                    p.skip.update(info["skip"])
        # sibling 1x1 convs over one input (a bottleneck's reduce conv and its
        # projection shortcut, Inception's branch reducers) run as one
        # two-output launch over concatenated weights
        if tc_mode and self.opts.sibling:
            self._plan_siblings()
        # junctions between bottleneck blocks: an expand conv (1x1, fused
        # shortcut) and the next block's reduce conv (1x1) reading its output
        # run as one neo_conv_junction launch; the reduce conv takes the
        # expand's output from shared memory (both maps are still written).
        # Opt-in: bit-identical and faster per launch in isolation, but
        # measured slower inside the graphed ResNet-50 b64 step (1.190 vs
        # 1.183 ms with only the 56x56 junctions, 1.235 ms with all): one tile
        # in flight per SM drains its chunks serially, while the two tuned
        # stand-alone convs overlap tiles and neighbouring launches
        if self.mode == "bf16" and self.opts.junction:
            for nid in order:
                r = self._junction_partner(nid)
                if r is not None and r not in p.junction_of and nid not in p.junction_of:
                    p.junction[nid] = r
                    p.junction_of[r] = nid
        if self.mode in ("bf16", "tf32"):
            self._plan_phys_blocks()

    # -- rules -------------------------------------------------------------------
    def _plan_prologues(self):
        g, p = self.g, self.plan
        for relu, bn in list(p.fused_bn_relu.items()):
            us = self.users[relu]
            if len(us) != 1 or relu in g.outputs or relu in self.keep:
                continue
            cv = g.nodes[us[0]]
            if cv.kind != OpKind.Conv2d or cv.inputs[0][0] != relu:
                continue
            if any(s == relu for s, _ in cv.inputs[1:]):
                continue
            wt = g.nodes[cv.inputs[1][0]].attrs["value"]
            kh, kw = wt.shape[2], wt.shape[3]
            spec = self.specs[relu]
            if (kh, kw) != (1, 1) or hw_pair(cv.attrs["pad"]) != (0, 0):
                continue
            if spec.layout.tag != "NCHWc" or not tc_legal_block(spec.layout.x, self.mode):
                continue
            if spec.logical_nchw[1] % spec.layout.x:
                continue
            p.prologue[cv.id] = bn
            p.pro_src[relu] = g.nodes[bn].inputs[0][0]
            p.skip.add(relu)
            del p.fused_bn_relu[relu]

    def _plan_siblings(self):
        g, p = self.g, self.plan
        groups: dict[int, list[int]] = {}
        for nid in self.order:
            if self._sibling_eligible(nid):
                groups.setdefault(g.nodes[nid].inputs[0][0], []).append(nid)
        for convs in groups.values():
            convs = list(convs)
            while len(convs) >= 2:
                a = convs.pop(0)
                pick = None
                for b in convs:
                    tn = self._sibling_tile(a, b)
                    if tn:
                        pick = (b, tn)
                        break
                if pick:
                    convs.remove(pick[0])
                    p.sibling[a] = pick
                    p.sibling_of[pick[0]] = a

    def _plan_phys_blocks(self):
        """Physical block size for tensor-core-illegal packed inputs."""
        g, p = self.g, self.plan
        min_lanes = 16 // bytes_per_elem(self.mode)
        for nid in self.order:
            node = g.nodes[nid]
            if node.kind != OpKind.LayoutTransform:
                continue
            dst = Layout.parse(node.attrs["dst_layout"])
            if dst.tag != "NCHWc" or tc_legal_block(dst.x, self.mode):
                continue
            src_layout = Layout.parse(node.attrs["src_layout"])
            us = self.users[nid]
            if nid in p.stem_fold or nid in p.skip:
                continue
            if (src_layout.tag == "NCHW" and us and nid not in g.outputs
                    and all(g.nodes[u].kind == OpKind.Conv2d and g.nodes[u].inputs[0][0] == nid
                            for u in us)):
                px = min_lanes
                while px < dst.x:
                    px *= 2
                if tc_legal_block(px, self.mode):
                    p.phys_x[nid] = px

    def _conv_kcrs(self, nid: int) -> np.ndarray:
        return conv_kcrs(self.g, nid)

    def _fused_stem_info(self, t: int, info: dict):
        """(conv, pool, input) if stem transform ``t`` feeds exactly one
        7x7/2 pad-3 conv with 64 outputs and no residual whose only consumer
        is a 3x3/2 pad-1 max pool writing NCHW[y]c."""
        g = self.g
        if info["S"] != 7 or info["sw"] != 2 or info["pw"] != 3 or info["w"] % 4:
            return None
        us = self.users[t]
        if len(us) != 1:
            return None
        cv = g.nodes[us[0]]
        wt = g.nodes[cv.inputs[1][0]].attrs["value"]
        if wt.ndim == 6:                    # pre-packed KCRS[x]c[y]k
            wt = host_unpack_kcrs(wt)
        epi = cv.attrs.get("epilogue") or {}
        if (wt.ndim != 4 or tuple(wt.shape) != (64, info["C"], 7, 7) or epi.get("residual")
                or len(cv.inputs) > 3 or hw_pair(cv.attrs["stride"]) != (2, 2)
                or hw_pair(cv.attrs["pad"]) != (3, 3)):
            return None
        cus = self.users[cv.id]
        if len(cus) != 1 or cv.id in g.outputs or cv.id in self.keep:
            return None
        mp = g.nodes[cus[0]]
        if (mp.kind != OpKind.MaxPool or hw_pair(mp.attrs["window"]) != (3, 3)
                or hw_pair(mp.attrs["stride"]) != (2, 2)
                or hw_pair(mp.attrs.get("pad", 0)) != (1, 1)):
            return None
        lay = self.specs[mp.id].layout
        if lay.tag != "NCHWc" or lay.x not in (8, 16, 32, 64):
            return None
        return cv.id, mp.id, g.nodes[t].inputs[0][0]

    def _sibling_eligible(self, nid: int) -> bool:
        """Unpadded 1x1 tensor-core conv without residual or prologue over a
        blocked input, writing a blocked map whose rows suit the TMA-store
        epilogue."""
        g = self.g
        node = g.nodes[nid]
        if node.kind != OpKind.Conv2d or nid in self.prologue or nid in self.skip:
            return False
        epi = node.attrs.get("epilogue") or {}
        if epi.get("residual") or hw_pair(node.attrs["pad"]) != (0, 0):
            return False
        src = node.inputs[0][0]
        if src in self.stem_fold or src in self.skip:
            return False
        k, c, r, s = self._conv_kcrs(nid).shape
        if (r, s) != (1, 1):
            return False
        dl, ol = self.specs[src].layout, self.specs[nid].layout
        if dl.tag != "NCHWc" or ol.tag != "NCHWc" or not tc_legal_block(dl.x, self.mode):
            return False
        if c % dl.x or k % ol.x or (ol.x * bytes_per_elem(self.mode)) not in (32, 64, 128):
            return False
        return True

    def _sibling_tile(self, a: int, b: int) -> int:
        """N tile of the merged launch (k_split = K of ``a`` must be a whole
        number of tiles), or 0 when the pair should not merge."""
        g = self.g
        na, nb = g.nodes[a], g.nodes[b]
        if hw_pair(na.attrs["stride"]) != hw_pair(nb.attrs["stride"]):
            return 0
        if self.specs[a].layout.x != self.specs[b].layout.x:
            return 0
        ka, kb = self._conv_kcrs(a).shape[0], self._conv_kcrs(b).shape[0]
        # measured (B200, b64): merging pays when both halves fill 128-256
        # wide N tiles; 64-wide tiles (the 56x56 64 -> 64 reducer) lose
        for tn in (256, 128):
            if ka % tn == 0 and kb >= tn:
                return tn
        return 0

    def _junction_conv_ok(self, nid: int, residual: bool) -> bool:
        """Unpadded stride-1 1x1 bf16 conv over NCHW[64]c into NCHW[64]c,
        bias-only epilogue (BN folded), with / without a fused residual."""
        g = self.g
        node = g.nodes[nid]
        if node.kind != OpKind.Conv2d or nid in self.skip or nid in self.prologue:
            return False
        if nid in self.sibling or nid in self.sibling_of or nid in self.stem_fold:
            return False
        epi = node.attrs.get("epilogue") or {}
        if bool(epi.get("residual")) != residual or epi.get("scale") is not None \
                or epi.get("shift") is not None:
            return False
        if hw_pair(node.attrs["stride"]) != (1, 1) or hw_pair(node.attrs["pad"]) != (0, 0):
            return False
        k, c, r, s_ = self._conv_kcrs(nid).shape
        src = node.inputs[0][0]
        dl, ol = self.specs[src].layout, self.specs[nid].layout
        if (r, s_) != (1, 1) or dl.tag != "NCHWc" or ol.tag != "NCHWc":
            return False
        if dl.x != 64 or ol.x != 64 or c % 64 or k % 64 or src in self.stem_fold:
            return False
        if residual and self.specs[node.inputs[-1][0]].layout.x != 64:
            return False
        return True

    def _junction_partner(self, nid: int) -> int | None:
        """Reduce conv R that can share a launch with expand conv ``nid``."""
        if not self._junction_conv_ok(nid, residual=True):
            return None
        n1 = self._conv_kcrs(nid).shape[0]
        if n1 % 128:
            return None
        _, _, h, w = self.specs[nid].logical_nchw
        if h * w < self.opts.junction_min_hw:
            return None
        for u in self.users[nid]:
            if u == nid or self.g.nodes[u].inputs[0][0] != nid:
                continue
            if not self._junction_conv_ok(u, residual=False):
                continue
            if self.pro_src.get(nid) is not None:
                continue
            n2 = self._conv_kcrs(u).shape[0]
            if n2 <= 256:
                return u
        return None

    def _fused_head_info(self, nid: int) -> dict | None:
        """Chain global AvgPool -> (NCHW transform) -> Flatten -> Dense ->
        (Softmax) with single consumers, over a bf16 / e4m3 NCHW[y]c map."""
        g = self.g
        node = g.nodes[nid]
        if node.kind != OpKind.AvgPool or hw_pair(node.attrs.get("pad", 0)) != (0, 0):
            return None
        src = node.inputs[0][0]
        sspec = self.specs[src]
        n, c, h, w = sspec.logical_nchw
        if hw_pair(node.attrs["window"]) != (h, w) or sspec.layout.tag != "NCHWc":
            return None
        if sspec.layout.x % 8 or c % 256 or c % sspec.layout.x:
            return None
        chain, cur = [nid], nid
        protected = set(g.outputs) | set(self.keep)
        while True:
            us = self.users[cur]
            if len(us) != 1 or cur in protected:
                break
            nxt = g.nodes[us[0]]
            if nxt.kind in (OpKind.LayoutTransform, OpKind.Flatten) and len(chain) < 3:
                chain.append(nxt.id)
                cur = nxt.id
                continue
            if nxt.kind == OpKind.Dense and nxt.inputs[0][0] == cur:
                if nxt.id in self.skip or nxt.id in self.fused_dense_relu.values():
                    return None       # the Dense is already fused into its ReLU
                chain.append(nxt.id)
                cur = nxt.id
                if len(self.users[cur]) == 1 and cur not in protected:
                    sm = g.nodes[self.users[cur][0]]
                    if sm.kind == OpKind.Softmax:
                        chain.append(sm.id)
                break
            break
        kinds = [g.nodes[i].kind for i in chain]
        if OpKind.Dense not in kinds or kinds[-2 if kinds[-1] == OpKind.Softmax else -1] != OpKind.Dense:
            return None
        if OpKind.Flatten not in kinds:
            return None
        dense = next(i for i in chain if g.nodes[i].kind == OpKind.Dense)
        wt = g.nodes[g.nodes[dense].inputs[1][0]].attrs["value"]
        if wt.ndim != 2 or wt.shape[1] != c:
            return None
        return {"anchor": chain[-1], "skip": chain[:-1], "src": src, "dense": dense,
                "softmax": kinds[-1] == OpKind.Softmax}

    def _stem_fold_info(self, nid) -> dict | None:
        """Fold parameters if ``nid`` packs a few-channel graph input that
        only feeds convs sharing one kernel width / stride / pad along w."""
        g = self.g
        node = g.nodes[nid]
        if node.kind != OpKind.LayoutTransform or nid in g.outputs or nid in self.keep:
            return None
        if Layout.parse(node.attrs["src_layout"]).tag != "NCHW" or \
                Layout.parse(node.attrs["dst_layout"]).tag != "NCHWc":
            return None
        src = node.inputs[0][0]
        if g.nodes[src].kind != OpKind.Input:
            return None
        n, c, h, w = self.specs[src].logical_nchw
        us = self.users[nid]
        if not us or c > 4:
            return None
        geo = set()
        for u in us:
            un = g.nodes[u]
            if un.kind != OpKind.Conv2d or un.inputs[0][0] != nid:
                return None
            wt = g.nodes[un.inputs[1][0]].attrs["value"]
            geo.add((wt.shape[3], hw_pair(un.attrs["stride"])[1], hw_pair(un.attrs["pad"])[1]))
        if len(geo) != 1:
            return None
        S, sw, pw = geo.pop()
        F = S * c
        lanes = [x for x in (8, 16, 32, 64, 4) if tc_legal_block(x, self.dense_mode)]
        fits = [x for x in sorted(lanes) if x >= F]
        if S == 1 or not fits:
            return None
        ow = (w + 2 * pw - S) // sw + 1
        return {"S": S, "sw": sw, "pw": pw, "ow": ow, "C": c, "F": F, "xf": fits[0],
                "n": n, "h": h, "w": w}


__all__ = ["FusionOptions", "FusionPlan", "plan_fusions", "conv_kcrs", "dense_block",
           "dense_mode_of"]
