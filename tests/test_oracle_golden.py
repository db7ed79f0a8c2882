"""Pin the CPU oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py).  Layout and pooling restatements
must be bit-exact; conv / graph outputs within the reference's own bounds
(tests/test_kernels.py:31-32 rel_err, Acceptance 1: 1e-5, Acceptance 3: 1e-4)."""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from oracle import ops as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def test_layouts_bitexact():
    d = load("layouts.npz")
    a = d["a"]
    for x in (1, 2, 3, 4, 6, 12):
        assert np.array_equal(O.pack_nchw(a, x).view(np.uint32), d[f"pack_x{x}"].view(np.uint32))
        assert np.array_equal(O.unpack_nchw(d[f"pack_x{x}"]), d[f"unpack_x{x}"])
    p4 = d["pack_x4"]
    for b in (2, 3, 6, 12):
        assert np.array_equal(O.retile_nchw(p4, b), d[f"retile_4_{b}"])
    assert np.array_equal(O.pack_nchw(d["big"], 16), d["big_pack16"])
    assert np.array_equal(O.pack_nchw(d["big"], 64), d["big_pack64"])
    assert np.array_equal(O.nhwc_to_nchw(d["nhwc"]), d["nhwc_to_nchw"])
    for x, y in ((1, 1), (2, 4), (4, 8), (4, 2)):
        assert np.array_equal(O.pack_kcrs(d["w"], x, y), d[f"wpack_{x}_{y}"])
        assert np.array_equal(O.unpack_kcrs(d[f"wpack_{x}_{y}"]), d["w"])


def _conv_cases(d):
    i = 0
    while f"{i}/wl" in d:
        yield i
        i += 1


def test_conv_matches_reference():
    d = load("conv.npz")
    n = 0
    for i in _conv_cases(d):
        c, k, h, w, r, s, st, pd = (int(v) for v in d[f"{i}/wl"])
        get = lambda key: d[f"{i}/{key}"] if f"{i}/{key}" in d else None
        out = O.conv2d(d[f"{i}/x"], d[f"{i}/w"], st, pd, get("scale"), get("shift"),
                       get("bias"), get("residual"), bool(d[f"{i}/relu"]))
        assert O.rel_err(out, d[f"{i}/reference"]) < 1e-5
        assert O.rel_err(d[f"{i}/blocked"], d[f"{i}/reference"]) < 1e-5
        n += 1
    assert n == 8


def test_config0_conv():
    """BASELINE config 0: 3x3 64->64 on NCHW16c + BN + ReLU."""
    d = load("conv.npz")
    x = O.unpack_nchw(d["c0/x16"])
    out = O.conv2d(x, d["c0/w"], 1, 1, d["c0/scale"], d["c0/shift"], relu=True)
    assert O.rel_err(out, d["c0/reference"]) < 1e-5
    assert O.rel_err(O.pack_nchw(out, 16), d["c0/blocked16"]) < 1e-5
    assert (out >= 0).all()


def test_pool_bitexact():
    d = load("pool.npz")
    a = d["a"]
    for mode in ("max", "avg"):
        for win, st, pd in ((2, 2, 0), (3, 2, 1), (3, 1, 1), (9, 1, 0)):
            key = f"{mode}_{win}_{st}_{pd}"
            assert np.array_equal(O.pool2d(a, win, st, pd, mode), d[key]), key
            assert np.array_equal(O.pool2d(O.pack_nchw(a, 4), win, st, pd, mode),
                                  d[key + "_b4"]), key


def _toy_graphs():
    import sys
    sys.path.insert(0, GOLD)
    import graphio
    from paper_1809_02697_b200 import Graph, Node, OpKind
    doc = json.load(open(os.path.join(GOLD, "graphs.json")))
    arrays = np.load(os.path.join(GOLD, "graphs.npz"))
    for case in doc["cases"]:
        g = graphio.load_graph(case["graph"], arrays, Graph, Node, OpKind)
        yield case, g, arrays


def test_toy_graphs_oracle():
    """Whole-graph oracle == reference executor on the four toy model kinds
    (unoptimized and optimized reference runs)."""
    count = 0
    for case, g, arrays in _toy_graphs():
        tag = case["tag"]
        outs = oracle.execute_reference(g, {"data": arrays[f"{tag}/input"]})
        for i, o in enumerate(outs):
            assert O.rel_err(o, arrays[f"{tag}/plain{i}"]) < 1e-5, tag
            assert O.rel_err(o, arrays[f"{tag}/opt{i}"]) < 1e-4, tag
        count += 1
    assert count == 8


@pytest.mark.parametrize("tag,name,batch,kw", [
    ("resnet18_b2_small", "resnet18", 2, {"image": 64, "num_classes": 10}),
    ("resnet18_b1", "resnet18", 1, {}),
])
def test_model_logits_oracle(tag, name, batch, kw):
    """The oracle on this repo's seeded ResNet builders reproduces the
    reference executor's logits (weights regenerated from the seed; digests
    guard against RNG drift)."""
    from paper_1809_02697_b200 import build_model, model_input
    d = load("models.npz")
    g = build_model(name, batch=batch, softmax=False, **kw)
    feeds = model_input(g)
    h = hashlib.sha256()
    for nid in sorted(g.nodes):
        v = g.nodes[nid].attrs.get("value")
        if v is not None:
            h.update(np.ascontiguousarray(v, np.float32).tobytes())
    assert h.digest() == d[f"{tag}/weight_digest"].tobytes()
    assert hashlib.sha256(feeds["data"].tobytes()).digest() == d[f"{tag}/input_digest"].tobytes()
    logits = oracle.execute_reference(g, feeds)[0]
    assert O.rel_err(logits, d[f"{tag}/logits"]) < 1e-4
    assert (logits.argmax(1) == d[f"{tag}/logits"].argmax(1)).all()


def test_oracle_known_answers():
    """Reference known-answer properties restated (tests/test_layout.py:74-117,
    tests/test_kernels.py:175-186)."""
    rng = np.random.default_rng(0)
    a = rng.standard_normal((2, 8, 3, 4)).astype(np.float32)
    p = O.pack_nchw(a, 4)
    for c in range(8):
        assert np.array_equal(p[:, c // 4, :, :, c % 4], a[:, c])
    w = rng.standard_normal((8, 4, 3, 3)).astype(np.float32)
    pw = O.pack_kcrs(w, 2, 4)
    for k in range(8):
        for c in range(4):
            assert np.array_equal(pw[k // 4, c // 2, :, :, c % 2, k % 4], w[k, c])
    x = rng.standard_normal((1, 8, 8, 8)).astype(np.float32)
    wt = rng.standard_normal((8, 8, 3, 3)).astype(np.float32)
    plain = O.conv2d(x, wt, 1, 1)
    got = O.conv2d(x, wt, 1, 1, np.full(8, 2.0, np.float32), np.full(8, -1.0, np.float32),
                   np.full(8, 0.25, np.float32), relu=True)
    assert O.rel_err(got, np.maximum(plain * 2.0 - 1.0 + 0.25, 0.0)) < 1e-6
