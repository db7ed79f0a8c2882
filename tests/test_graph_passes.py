"""Host IR and compile passes (CPU).  Mirrors the reference's
tests/test_graph.py (topo ties, cycles, validation, shape inference) and
tests/test_passes.py (BN folding, fusion, transform minimality, weight
packing), plus agreement with the reference's own pass results on the toy
models (golden graphs.json) and the B200 extensions."""

import json
import os
import sys

import numpy as np
import pytest

import oracle
from paper_1809_02697_b200 import (Graph, Node, OpKind, alter_and_insert_transforms,
                                   count_transforms, fold_batchnorm, fuse_elementwise,
                                   infer_shapes, nchwc, per_conv_packing, pretransform_weights,
                                   simplify, topo_sort, uniform_assignment, validate)
from paper_1809_02697_b200.errors import (AssignmentIncomplete, CycleDetected,
                                          NonConstantStatistics, ShapeMismatch)
from paper_1809_02697_b200.layout import Layout, host_pack_kcrs, host_unpack_kcrs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def conv_chain(depth=3, c=16, hw=8, bn=True, relu=True, seed=0):
    rng = np.random.default_rng(seed)
    g = Graph("chain")
    x = g.add(OpKind.Input, shape=(1, c, hw, hw), layout="NCHW", name="data")
    for _ in range(depth):
        w = g.constant(rng.standard_normal((c, c, 3, 3)).astype(np.float32) * 0.2)
        x = g.add(OpKind.Conv2d, inputs=[x, w], stride=1, pad=1)
        if bn:
            stats = [g.constant(rng.uniform(0.5, 1.5, c).astype(np.float32)) for _ in range(4)]
            x = g.add(OpKind.BatchNorm, inputs=[x, *stats], eps=1e-5)
        if relu:
            x = g.add(OpKind.ReLU, inputs=[x])
    g.outputs = [x]
    return g


class TestGraph:
    def test_topo_ties_by_id(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 1, 2, 2))
        b = g.add(OpKind.ReLU, inputs=[a])
        c = g.add(OpKind.ReLU, inputs=[a])
        d = g.add(OpKind.ElementwiseAdd, inputs=[c, b])
        g.outputs = [d]
        assert topo_sort(g) == [a, b, c, d]

    def test_cycle(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 1, 2, 2))
        b = g.add(OpKind.ReLU, inputs=[a])
        g.nodes[b].inputs.append((b + 1, 0))
        c = g.add(OpKind.ReLU, inputs=[b])
        g.outputs = [c]
        with pytest.raises(CycleDetected):
            topo_sort(g)
        assert any("cycle" in p for p in validate(g))

    def test_validate_messages(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 1, 2, 2))
        r = g.add(OpKind.ReLU, inputs=[a, a])
        assert any("arity" in p for p in validate(g))
        g.outputs = [r, 99]
        assert any("missing node 99" in p for p in validate(g))
        assert "graph has no outputs" in validate(Graph())

    def test_infer_blocked_and_default(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(2, 3, 4, 32, 16), layout="NCHW16c")
        w = g.constant(np.zeros((2, 3, 3, 3, 16, 8), np.float32))
        c = g.add(OpKind.Conv2d, inputs=[a, w], stride=2, pad=1)
        p = g.add(OpKind.MaxPool, inputs=[c], window=2, stride=2)
        t = g.add(OpKind.LayoutTransform, inputs=[p], src_layout="NCHW8c", dst_layout="NCHW")
        f = g.add(OpKind.Flatten, inputs=[t])
        g.outputs = [f]
        sp = infer_shapes(g)
        assert sp[c].shape == (2, 2, 2, 16, 8) and sp[c].layout == nchwc(8)
        assert sp[p].shape == (2, 2, 1, 8, 8)
        assert sp[t].shape == (2, 16, 1, 8)
        assert sp[f].shape == (2, 128)

    def test_flatten_rejects_blocked(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 1, 2, 2, 4), layout="NCHW4c")
        f = g.add(OpKind.Flatten, inputs=[a])
        g.outputs = [f]
        with pytest.raises(ShapeMismatch) as e:
            infer_shapes(g)
        assert e.value.node_id == f

    def test_asymmetric_pad_extension(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 8, 17, 17))
        w = g.constant(np.zeros((8, 8, 1, 7), np.float32))
        c = g.add(OpKind.Conv2d, inputs=[a, w], stride=1, pad=(0, 3))
        g.outputs = [c]
        assert infer_shapes(g)[c].shape == (1, 8, 17, 17)

    def test_pad_channels_transform(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 3, 8, 8))
        t = g.add(OpKind.LayoutTransform, inputs=[a], src_layout="NCHW", dst_layout="NCHW8c",
                  pad_channels=True)
        g.outputs = [t]
        assert infer_shapes(g)[t].shape == (1, 1, 8, 8, 8)
        del g.nodes[t].attrs["pad_channels"]
        with pytest.raises(ShapeMismatch):
            infer_shapes(g)

    def test_nhwc_input_is_ingested(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 8, 8, 3), layout="NHWC")
        w = g.constant(np.zeros((4, 3, 3, 3), np.float32))
        c = g.add(OpKind.Conv2d, inputs=[a, w], stride=1, pad=1)
        g.outputs = [c]
        assert infer_shapes(g)[c].shape == (1, 4, 8, 8)


class TestPasses:
    def test_fold_batchnorm_preserves_values(self):
        g = conv_chain(depth=2, relu=False)
        feeds = {"data": np.random.default_rng(1).standard_normal((1, 16, 8, 8)).astype(np.float32)}
        ref = oracle.execute_reference(g, feeds)[0]
        f = fold_batchnorm(g)
        assert not any(n.kind == OpKind.BatchNorm for n in f.nodes.values())
        assert oracle.rel_err(oracle.execute_reference(f, feeds)[0], ref) < 1e-5

    def test_fold_fanout_canonicalises(self):
        g = conv_chain(depth=1, relu=False)
        conv = next(n.id for n in g.nodes.values() if n.kind == OpKind.Conv2d)
        extra = g.add(OpKind.ReLU, inputs=[conv])
        g.outputs.append(extra)
        f = fold_batchnorm(g)
        bns = [n for n in f.nodes.values() if n.kind == OpKind.BatchNorm]
        assert len(bns) == 1 and set(bns[0].attrs) == {"scale", "shift"}

    def test_nonconstant_statistics(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 2, 2, 2))
        b = g.add(OpKind.BatchNorm, inputs=[a, a, a, a, a])
        g.outputs = [b]
        with pytest.raises(NonConstantStatistics):
            fold_batchnorm(g)

    def test_fusion_and_transform_minimality(self):
        g = conv_chain(depth=3)
        s = simplify(g)
        convs = [n for n in s.nodes.values() if n.kind == OpKind.Conv2d]
        assert len(convs) == 3 and all(n.attrs["epilogue"]["relu"] for n in convs)
        assert not any(n.kind in (OpKind.ReLU, OpKind.BatchNorm) for n in s.nodes.values())
        opt = alter_and_insert_transforms(s, uniform_assignment(s, x=16))
        assert count_transforms(opt) == 2          # graph entry and exit only
        ablation = per_conv_packing(s, uniform_assignment(s, x=16))
        assert count_transforms(ablation) == 2 * 3

    def test_residual_fusion(self):
        from paper_1809_02697_b200.models import resnet
        g = resnet(18, batch=1, image=32, num_classes=10)
        s = simplify(g)
        res = [n for n in s.nodes.values() if n.kind == OpKind.Conv2d
               and n.attrs["epilogue"]["residual"]]
        assert len(res) == 8                       # one per basic block
        assert all(n.attrs["epilogue"]["relu"] for n in res)

    def test_pretransform_packs_and_duplicates_shared(self):
        g = Graph()
        a = g.add(OpKind.Input, shape=(1, 8, 4, 4))
        w = g.constant(np.arange(8 * 8 * 9, dtype=np.float32).reshape(8, 8, 3, 3))
        c1 = g.add(OpKind.Conv2d, inputs=[a, w], stride=1, pad=1)
        c2 = g.add(OpKind.Conv2d, inputs=[c1, w], stride=1, pad=1)
        g.outputs = [c2]
        with pytest.raises(AssignmentIncomplete):
            pretransform_weights(g)
        p = pretransform_weights(g, {c1: (4, 8), c2: (8, 2)})
        w1 = p.nodes[p.nodes[c1].inputs[1][0]].attrs
        w2 = p.nodes[p.nodes[c2].inputs[1][0]].attrs
        assert w1["layout"] == "KCRS4c8k" and w2["layout"] == "KCRS8c2k"
        assert p.nodes[c1].inputs[1][0] != p.nodes[c2].inputs[1][0]
        assert np.array_equal(host_unpack_kcrs(w2["value"]), g.nodes[w].attrs["value"])

    def test_host_weight_pack_matches_oracle(self):
        w = np.random.default_rng(3).standard_normal((12, 8, 3, 3)).astype(np.float32)
        for x, y in ((1, 1), (2, 3), (4, 6), (8, 12)):
            assert np.array_equal(host_pack_kcrs(w, x, y), oracle.pack_kcrs(w, x, y))


def _golden_cases():
    sys.path.insert(0, GOLD)
    import graphio
    doc = json.load(open(os.path.join(GOLD, "graphs.json")))
    arrays = np.load(os.path.join(GOLD, "graphs.npz"))
    for case in doc["cases"]:
        yield case, graphio.load_graph(case["graph"], arrays, Graph, Node, OpKind), arrays


def test_passes_agree_with_reference_on_toy_models():
    """Same simplified size, same uniform assignment for the reference's split
    factor, same transform count, and the optimized graph computes the
    reference's outputs (oracle interpreter)."""
    for case, g, arrays in _golden_cases():
        s = simplify(g)
        assert len(s.nodes) == case["simplified_nodes"], case["tag"]
        assign = uniform_assignment(s, x=case["split_factor"])
        assert {str(k): list(v) for k, v in assign.items()} == case["assignment"]
        opt = pretransform_weights(alter_and_insert_transforms(s, assign))
        assert count_transforms(opt) == case["transforms"], case["tag"]
        assert len(opt.nodes) == case["optimized_nodes"], case["tag"]
        outs = oracle.execute_reference(opt, {"data": arrays[f"{case['tag']}/input"]})
        for i, o in enumerate(outs):
            assert oracle.rel_err(o, arrays[f"{case['tag']}/opt{i}"]) < 1e-4


def test_gpu_split_factor_on_baseline_models():
    from paper_1809_02697_b200 import build_model
    from paper_1809_02697_b200.passes import uniform_split_factor
    expect = {"resnet50": 64, "vgg16": 64, "inception_v3": 16, "densenet201": 32,
              "ssd_resnet50": 64}
    for name, x in expect.items():
        g = simplify(build_model(name, batch=1))
        assert uniform_split_factor(g, "bf16") == x, name
        assert uniform_split_factor(g, "tf32") == min(x, 32), name
        opt = alter_and_insert_transforms(g, uniform_assignment(g, mode="bf16"))
        heads = 12 if name == "ssd_resnet50" else 1
        assert count_transforms(opt) == 1 + heads, name
