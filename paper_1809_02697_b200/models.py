"""Seeded, random-init graph builders for the BASELINE.json configurations,
written against the reference Graph API (graph.py:82-126).

The reference ships only four toy generators (models.py:10); the benchmark
families (ResNet-18/50 v1, VGG-16, Inception-v3, DenseNet-201, SSD with a
ResNet-50 backbone) are defined here.  Initialisation follows BASELINE.json /
SURVEY.md 8(d): conv weights He-normal std = sqrt(2 / (C R S)); BN gamma
U(0.5, 1.5), beta N(0, 0.1), mean N(0, 0.1), var U(0.5, 1.5), eps 1e-5
(Inception: 1e-3); dense weights He-normal, zero bias; conv biases (VGG) zero.
Weights are drawn from ``default_rng(seed)`` in construction order.
"""

from __future__ import annotations

import numpy as np

from .graph import Graph, OpKind


class NetBuilder:
    """Small helper that threads a Graph and an RNG through a network."""

    def __init__(self, name: str, batch: int, channels: int, size: int, seed: int = 0,
                 bn_eps: float = 1e-5):
        self.g = Graph(name)
        self.rng = np.random.default_rng(seed)
        self.bn_eps = bn_eps
        self.data = self.g.add(OpKind.Input, shape=(batch, channels, size, size),
                               layout="NCHW", name="data")

    # -- layers ------------------------------------------------------------
    def conv(self, x, c_in, c_out, kernel, stride=1, pad=None, bias=False):
        kh, kw = (kernel, kernel) if isinstance(kernel, int) else kernel
        if pad is None:
            pad = (kh // 2, kw // 2) if kh != kw else kh // 2
        std = np.sqrt(2.0 / (c_in * kh * kw))
        w = self.g.constant((self.rng.standard_normal((c_out, c_in, kh, kw)) * std)
                            .astype(np.float32))
        ins = [x, w]
        if bias:
            ins.append(self.g.constant(np.zeros(c_out, np.float32)))
        return self.g.add(OpKind.Conv2d, inputs=ins, stride=stride, pad=pad)

    def bn(self, x, c):
        r = self.rng
        consts = [r.uniform(0.5, 1.5, c), r.normal(0.0, 0.1, c), r.normal(0.0, 0.1, c),
                  r.uniform(0.5, 1.5, c)]
        ids = [self.g.constant(np.asarray(v, np.float32)) for v in consts]
        return self.g.add(OpKind.BatchNorm, inputs=[x, *ids], eps=self.bn_eps)

    def relu(self, x):
        return self.g.add(OpKind.ReLU, inputs=[x])

    def conv_bn_relu(self, x, c_in, c_out, kernel, stride=1, pad=None, relu=True):
        y = self.bn(self.conv(x, c_in, c_out, kernel, stride, pad), c_out)
        return self.relu(y) if relu else y

    def maxpool(self, x, win, stride, pad=0):
        return self.g.add(OpKind.MaxPool, inputs=[x], window=win, stride=stride, pad=pad)

    def avgpool(self, x, win, stride, pad=0):
        return self.g.add(OpKind.AvgPool, inputs=[x], window=win, stride=stride, pad=pad)

    def add(self, a, b):
        return self.g.add(OpKind.ElementwiseAdd, inputs=[a, b])

    def concat(self, xs):
        return self.g.add(OpKind.Concat, inputs=list(xs), axis=1)

    def classifier(self, x, c_in, units=1000, softmax=True):
        x = self.g.add(OpKind.Flatten, inputs=[x])
        w = self.g.constant((self.rng.standard_normal((units, c_in)) * np.sqrt(2.0 / c_in))
                            .astype(np.float32))
        b = self.g.constant(np.zeros(units, np.float32))
        logits = self.g.add(OpKind.Dense, inputs=[x, w, b], name="logits")
        self.logits = logits
        return self.g.add(OpKind.Softmax, inputs=[logits]) if softmax else logits

    def dense_relu(self, x, c_in, units):
        w = self.g.constant((self.rng.standard_normal((units, c_in)) * np.sqrt(2.0 / c_in))
                            .astype(np.float32))
        b = self.g.constant(np.zeros(units, np.float32))
        return self.relu(self.g.add(OpKind.Dense, inputs=[x, w, b]))

    def finish(self, *outputs) -> Graph:
        self.g.outputs = list(outputs)
        self.g.logits_id = getattr(self, "logits", None)
        return self.g


# ---------------------------------------------------------------------------
# ResNet v1 (He et al. 2016): BASELINE configs 1 and 2

def _basic_block(b: NetBuilder, x, c_in, c_out, stride):
    y = b.conv_bn_relu(x, c_in, c_out, 3, stride, 1)
    y = b.conv_bn_relu(y, c_out, c_out, 3, 1, 1, relu=False)
    short = x
    if stride != 1 or c_in != c_out:
        short = b.conv_bn_relu(x, c_in, c_out, 1, stride, 0, relu=False)
    return b.relu(b.add(y, short))


def _bottleneck(b: NetBuilder, x, c_in, width, stride):
    c_out = 4 * width
    y = b.conv_bn_relu(x, c_in, width, 1, stride, 0)       # v1: stride on the 1x1
    y = b.conv_bn_relu(y, width, width, 3, 1, 1)
    y = b.conv_bn_relu(y, width, c_out, 1, 1, 0, relu=False)
    short = x
    if stride != 1 or c_in != c_out:
        short = b.conv_bn_relu(x, c_in, c_out, 1, stride, 0, relu=False)
    return b.relu(b.add(y, short))


def resnet_trunk(b: NetBuilder, x, depth: int, stages: int = 4):
    """Stem + the first ``stages`` residual stages; returns (node, channels,
    per-stage outputs)."""
    x = b.conv_bn_relu(x, 3, 64, 7, 2, 3)
    x = b.maxpool(x, 3, 2, 1)
    if depth == 18:
        counts, block, expand = (2, 2, 2, 2), _basic_block, 1
    elif depth == 34:
        counts, block, expand = (3, 4, 6, 3), _basic_block, 1
    elif depth == 50:
        counts, block, expand = (3, 4, 6, 3), _bottleneck, 4
    elif depth == 101:
        counts, block, expand = (3, 4, 23, 3), _bottleneck, 4
    else:
        raise ValueError(f"unsupported ResNet depth {depth}")
    c = 64
    feats = []
    for stage, (count, width) in enumerate(zip(counts[:stages], (64, 128, 256, 512))):
        for i in range(count):
            stride = 2 if (i == 0 and stage > 0) else 1
            x = block(b, x, c, width, stride)
            c = width * expand
        feats.append((x, c))
    return x, c, feats


def resnet(depth: int = 50, batch: int = 1, image: int = 224, num_classes: int = 1000,
           seed: int = 0, softmax: bool = True) -> Graph:
    b = NetBuilder(f"resnet{depth}_v1", batch, 3, image, seed)
    x, c, _ = resnet_trunk(b, b.data, depth)
    x = b.avgpool(x, image // 32, 1)
    return b.finish(b.classifier(x, c, num_classes, softmax))


# ---------------------------------------------------------------------------
# VGG-16 (config D): BASELINE config 3

def vgg16(batch: int = 1, image: int = 224, num_classes: int = 1000, seed: int = 0,
          softmax: bool = True) -> Graph:
    b = NetBuilder("vgg16", batch, 3, image, seed)
    x, c = b.data, 3
    for item in (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
                 512, 512, 512, "M"):
        if item == "M":
            x = b.maxpool(x, 2, 2)
        else:
            x = b.relu(b.conv(x, c, item, 3, 1, 1, bias=True))
            c = item
    side = image // 32
    x = b.g.add(OpKind.Flatten, inputs=[x])
    x = b.dense_relu(x, c * side * side, 4096)
    x = b.dense_relu(x, 4096, 4096)
    w = b.g.constant((b.rng.standard_normal((num_classes, 4096)) * np.sqrt(2.0 / 4096))
                     .astype(np.float32))
    bias = b.g.constant(np.zeros(num_classes, np.float32))
    logits = b.g.add(OpKind.Dense, inputs=[x, w, bias], name="logits")
    b.logits = logits
    out = b.g.add(OpKind.Softmax, inputs=[logits]) if softmax else logits
    return b.finish(out)


# ---------------------------------------------------------------------------
# DenseNet-201 (growth 32, bn_size 4): BASELINE config 4

def densenet(blocks=(6, 12, 48, 32), growth: int = 32, batch: int = 1, image: int = 224,
             num_classes: int = 1000, seed: int = 0, softmax: bool = True,
             name: str = "densenet201") -> Graph:
    b = NetBuilder(name, batch, 3, image, seed)
    x = b.conv_bn_relu(b.data, 3, 2 * growth, 7, 2, 3)
    x = b.maxpool(x, 3, 2, 1)
    c = 2 * growth
    for bi, layers in enumerate(blocks):
        for _ in range(layers):
            y = b.relu(b.bn(x, c))
            y = b.conv_bn_relu(y, c, 4 * growth, 1, 1, 0)
            y = b.conv(y, 4 * growth, growth, 3, 1, 1)
            x = b.concat([x, y])
            c += growth
        if bi != len(blocks) - 1:
            y = b.relu(b.bn(x, c))
            y = b.conv(y, c, c // 2, 1, 1, 0)
            x = b.avgpool(y, 2, 2)
            c //= 2
    x = b.relu(b.bn(x, c))
    from .graph import infer_shapes
    b.g.outputs = [x]
    x = b.avgpool(x, infer_shapes(b.g)[x].shape[2], 1)
    return b.finish(b.classifier(x, c, num_classes, softmax))


def densenet201(batch: int = 1, **kw) -> Graph:
    return densenet((6, 12, 48, 32), 32, batch, **kw)


# ---------------------------------------------------------------------------
# Inception-v3 (Szegedy et al. 2016, no aux head): BASELINE config 3

def _incA(b, x, c, pool_feat):
    b1 = b.conv_bn_relu(x, c, 64, 1, 1, 0)
    b5 = b.conv_bn_relu(b.conv_bn_relu(x, c, 48, 1, 1, 0), 48, 64, 5, 1, 2)
    b3 = b.conv_bn_relu(x, c, 64, 1, 1, 0)
    b3 = b.conv_bn_relu(b.conv_bn_relu(b3, 64, 96, 3, 1, 1), 96, 96, 3, 1, 1)
    bp = b.conv_bn_relu(b.avgpool(x, 3, 1, 1), c, pool_feat, 1, 1, 0)
    return b.concat([b1, b5, b3, bp]), 64 + 64 + 96 + pool_feat


def _incB(b, x, c):
    b3 = b.conv_bn_relu(x, c, 384, 3, 2, 0)
    bd = b.conv_bn_relu(x, c, 64, 1, 1, 0)
    bd = b.conv_bn_relu(b.conv_bn_relu(bd, 64, 96, 3, 1, 1), 96, 96, 3, 2, 0)
    bp = b.maxpool(x, 3, 2)
    return b.concat([b3, bd, bp]), 384 + 96 + c


def _incC(b, x, c, c7):
    b1 = b.conv_bn_relu(x, c, 192, 1, 1, 0)
    b7 = b.conv_bn_relu(x, c, c7, 1, 1, 0)
    b7 = b.conv_bn_relu(b7, c7, c7, (1, 7), 1, (0, 3))
    b7 = b.conv_bn_relu(b7, c7, 192, (7, 1), 1, (3, 0))
    bd = b.conv_bn_relu(x, c, c7, 1, 1, 0)
    bd = b.conv_bn_relu(bd, c7, c7, (7, 1), 1, (3, 0))
    bd = b.conv_bn_relu(bd, c7, c7, (1, 7), 1, (0, 3))
    bd = b.conv_bn_relu(bd, c7, c7, (7, 1), 1, (3, 0))
    bd = b.conv_bn_relu(bd, c7, 192, (1, 7), 1, (0, 3))
    bp = b.conv_bn_relu(b.avgpool(x, 3, 1, 1), c, 192, 1, 1, 0)
    return b.concat([b1, b7, bd, bp]), 768


def _incD(b, x, c):
    b3 = b.conv_bn_relu(b.conv_bn_relu(x, c, 192, 1, 1, 0), 192, 320, 3, 2, 0)
    b7 = b.conv_bn_relu(x, c, 192, 1, 1, 0)
    b7 = b.conv_bn_relu(b7, 192, 192, (1, 7), 1, (0, 3))
    b7 = b.conv_bn_relu(b7, 192, 192, (7, 1), 1, (3, 0))
    b7 = b.conv_bn_relu(b7, 192, 192, 3, 2, 0)
    bp = b.maxpool(x, 3, 2)
    return b.concat([b3, b7, bp]), 320 + 192 + c


def _incE(b, x, c):
    b1 = b.conv_bn_relu(x, c, 320, 1, 1, 0)
    b3 = b.conv_bn_relu(x, c, 384, 1, 1, 0)
    b3 = b.concat([b.conv_bn_relu(b3, 384, 384, (1, 3), 1, (0, 1)),
                   b.conv_bn_relu(b3, 384, 384, (3, 1), 1, (1, 0))])
    bd = b.conv_bn_relu(x, c, 448, 1, 1, 0)
    bd = b.conv_bn_relu(bd, 448, 384, 3, 1, 1)
    bd = b.concat([b.conv_bn_relu(bd, 384, 384, (1, 3), 1, (0, 1)),
                   b.conv_bn_relu(bd, 384, 384, (3, 1), 1, (1, 0))])
    bp = b.conv_bn_relu(b.avgpool(x, 3, 1, 1), c, 192, 1, 1, 0)
    return b.concat([b1, b3, bd, bp]), 320 + 768 + 768 + 192


def inception_v3(batch: int = 1, image: int = 299, num_classes: int = 1000, seed: int = 0,
                 softmax: bool = True) -> Graph:
    b = NetBuilder("inception_v3", batch, 3, image, seed, bn_eps=1e-3)
    x = b.conv_bn_relu(b.data, 3, 32, 3, 2, 0)
    x = b.conv_bn_relu(x, 32, 32, 3, 1, 0)
    x = b.conv_bn_relu(x, 32, 64, 3, 1, 1)
    x = b.maxpool(x, 3, 2)
    x = b.conv_bn_relu(x, 64, 80, 1, 1, 0)
    x = b.conv_bn_relu(x, 80, 192, 3, 1, 0)
    x = b.maxpool(x, 3, 2)
    c = 192
    for pf in (32, 64, 64):
        x, c = _incA(b, x, c, pf)
    x, c = _incB(b, x, c)
    for c7 in (128, 160, 160, 192):
        x, c = _incC(b, x, c, c7)
    x, c = _incD(b, x, c)
    for _ in range(2):
        x, c = _incE(b, x, c)
    from .graph import infer_shapes
    b.g.outputs = [x]
    side = infer_shapes(b.g)[x].shape[2]
    x = b.avgpool(x, side, 1)
    return b.finish(b.classifier(x, c, num_classes, softmax))


# ---------------------------------------------------------------------------
# SSD-512 with a ResNet-50 v1 backbone: BASELINE config 4

SSD_ANCHORS = (4, 6, 6, 6, 4, 4)


def ssd_resnet50(batch: int = 1, image: int = 512, num_classes: int = 21, seed: int = 0) -> Graph:
    """Six feature maps (ResNet-50 stage 3 and 4 + four extra stride-2
    blocks); per map a 3x3 class head (anchors x classes) and a 3x3 box head
    (anchors x 4).  Outputs are the 12 raw head maps (pre-NMS)."""
    b = NetBuilder("ssd512_resnet50_v1", batch, 3, image, seed)
    _, c, feats = resnet_trunk(b, b.data, 50, stages=4)
    maps = [feats[2], feats[3]]
    x, c = feats[3]
    for mid, out in ((256, 512), (256, 512), (128, 256), (128, 256)):
        y = b.conv_bn_relu(x, c, mid, 1, 1, 0)
        x = b.conv_bn_relu(y, mid, out, 3, 2, 1)
        c = out
        maps.append((x, c))
    outs = []
    for (fm, fc), anchors in zip(maps, SSD_ANCHORS):
        outs.append(b.conv(fm, fc, anchors * num_classes, 3, 1, 1, bias=True))
        outs.append(b.conv(fm, fc, anchors * 4, 3, 1, 1, bias=True))
    return b.finish(*outs)


# ---------------------------------------------------------------------------

MODELS = {
    "resnet18": lambda batch=1, **kw: resnet(18, batch, **kw),
    "resnet50": lambda batch=1, **kw: resnet(50, batch, **kw),
    "vgg16": vgg16,
    "inception_v3": inception_v3,
    "densenet201": densenet201,
    "ssd_resnet50": ssd_resnet50,
}


def build_model(name: str, batch: int = 1, seed: int = 0, **kw) -> Graph:
    if name not in MODELS:
        raise ValueError(f"unknown model {name!r}; choose from {sorted(MODELS)}")
    return MODELS[name](batch=batch, seed=seed, **kw)


def model_input(g: Graph, seed: int = 1) -> dict:
    """N(0, 1) input for every Input node, drawn from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    feeds = {}
    for nid in sorted(g.nodes):
        node = g.nodes[nid]
        if node.kind == OpKind.Input:
            name = node.attrs.get("name", f"input{nid}")
            feeds[name] = rng.standard_normal(node.attrs["shape"]).astype(np.float32)
    return feeds


def conv_flops(g: Graph, batch: int | None = None) -> int:
    """Sum of 2*N*K*C*R*S*OH*OW over the graph's convs."""
    from .graph import infer_shapes
    specs = infer_shapes(g)
    total = 0
    for node in g.nodes.values():
        if node.kind != OpKind.Conv2d:
            continue
        n, c = specs[node.inputs[0][0]].logical_nchw[:2]
        w = g.nodes[node.inputs[1][0]].attrs["value"]
        k, r, s = (w.shape[0], w.shape[2], w.shape[3]) if w.ndim == 4 else (
            w.shape[0] * w.shape[5], w.shape[2], w.shape[3])
        _, _, oh, ow = specs[node.id].logical_nchw
        total += 2 * (batch or n) * k * c * r * s * oh * ow
    return total


# ---------------------------------------------------------------------------
# The reference's four seeded toy families (models.py:10-95), kept so a user
# of ``neoplan gen`` / ``gen_model`` gets the same graphs and weights here:
# the random draws happen in the same order, so a given (kind, depth,
# channels, hw, seed) yields bit-identical constants (pinned against the
# reference in tests/test_modelio.py).

KINDS = ("chain", "vgg-ish", "resnet-block", "diamond-concat")


class _Toy:
    """Seeded builder for the toy families: He-like scaled convs without
    bias and BatchNorms with random statistics."""

    def __init__(self, g: Graph, seed: int):
        self.g = g
        self.rng = np.random.default_rng(seed)

    def conv(self, x, c_in, c_out, k, stride=1, pad=None, gain=0.2):
        w = self.rng.standard_normal((c_out, c_in, k, k)) * gain / np.sqrt(c_in * k * k)
        wid = self.g.constant(w.astype(np.float32))
        return self.g.add(OpKind.Conv2d, inputs=[x, wid], stride=stride,
                          pad=k // 2 if pad is None else pad)

    def bn(self, x, c):
        draws = [(0.5, 1.5), (-0.2, 0.2), (-0.1, 0.1), (0.5, 1.5)]   # gamma beta mean var
        stats = [self.g.constant(self.rng.uniform(lo, hi, c).astype(np.float32))
                 for lo, hi in draws]
        return self.g.add(OpKind.BatchNorm, inputs=[x, *stats], eps=1e-5)

    def relu(self, x):
        return self.g.add(OpKind.ReLU, inputs=[x])


def gen_model(kind: str, depth: int = 3, channels: int = 16, hw: int = 16,
              seed: int = 0) -> Graph:
    """Toy CNN of one of ``KINDS`` (reference models.py:29-95)."""
    if kind not in KINDS:
        raise ValueError(f"unknown model kind {kind!r}; choose from {KINDS}")
    if min(depth, channels, hw) < 1:
        raise ValueError("depth, channels and hw must be positive")
    g = Graph(f"{kind}-d{depth}-c{channels}")
    t = _Toy(g, seed)
    x = g.add(OpKind.Input, shape=(1, channels, hw, hw), layout="NCHW", name="data")
    c = channels
    if kind == "chain":
        for _ in range(depth):
            x = t.relu(t.bn(t.conv(x, c, c, 3), c))
    elif kind == "vgg-ish":
        size = hw
        for _ in range(depth):
            x = t.relu(t.conv(x, c, 2 * c, 3))
            c *= 2
            if size >= 4:
                x = g.add(OpKind.MaxPool, inputs=[x], window=2, stride=2)
                size //= 2
        x = g.add(OpKind.Flatten, inputs=[x])
        w = g.constant((t.rng.standard_normal((10, c * size * size)) * 0.05).astype(np.float32))
        x = g.add(OpKind.Softmax, inputs=[g.add(OpKind.Dense, inputs=[x, w])])
    elif kind == "resnet-block":
        for _ in range(depth):
            y = t.relu(t.bn(t.conv(x, c, c, 3), c))
            y = t.bn(t.conv(y, c, c, 3), c)
            x = t.relu(g.add(OpKind.ElementwiseAdd, inputs=[y, x]))
    else:   # diamond-concat: a 3x3 and a 1x1 branch joined on the channel axis
        for _ in range(depth):
            half = max(1, c // 2)
            a = t.relu(t.conv(x, c, half, 3))
            b = t.relu(t.conv(x, c, half, 1))
            x = g.add(OpKind.Concat, inputs=[a, b], axis=1)
            c = 2 * half
        x = t.conv(x, c, c, 1)
    g.outputs = [x]
    return g
