"""Fusion planner (fusion.py) on the BASELINE model graphs -- host logic, no
GPU: which operators the device executor merges in each mode, and that the
switches and ``keep`` are honoured."""
import pytest

from paper_1809_02697_b200 import models
from paper_1809_02697_b200.fusion import FusionOptions, plan_fusions
from paper_1809_02697_b200.graph import OpKind, hw_pair
from paper_1809_02697_b200.passes import compile_graph

_CACHE: dict = {}


def _compiled(name, mode):
    key = (name, mode)
    if key not in _CACHE:
        g = models.build_model(name, batch=1)
        _CACHE[key] = compile_graph(g, mode=mode, fp8_scales={} if mode == "fp8" else None)
    return _CACHE[key]


def _kind(cg, nid):
    return cg.nodes[nid].kind


def _check_invariants(cg, fp):
    outs = set(cg.outputs)
    assert not (fp.skip & outs), "a graph output was fused away"
    for a, (b, tn) in fp.sibling.items():
        assert fp.sibling_of[b] == a and tn in (128, 256)
        na, nb = cg.nodes[a], cg.nodes[b]
        assert na.inputs[0][0] == nb.inputs[0][0]                 # one shared input
        assert _kind(cg, a) == _kind(cg, b) == OpKind.Conv2d
        assert hw_pair(na.attrs["pad"]) == hw_pair(nb.attrs["pad"]) == (0, 0)
    assert not (set(fp.sibling) & set(fp.sibling_of))
    for relu, bn in fp.fused_bn_relu.items():
        assert _kind(cg, relu) == OpKind.ReLU and _kind(cg, bn) == OpKind.BatchNorm
        assert bn in fp.skip and relu not in fp.skip
    for pool, (conv, src) in fp.fused_stem.items():
        assert _kind(cg, pool) == OpKind.MaxPool and _kind(cg, conv) == OpKind.Conv2d
        assert _kind(cg, src) == OpKind.Input and conv in fp.skip
    for anchor, info in fp.fused_head.items():
        assert info["dense"] in info["skip"] or info["dense"] == anchor
        assert all(s in fp.skip for s in info["skip"]) and anchor not in fp.skip


@pytest.mark.parametrize("name", ["resnet50", "resnet18", "densenet201", "inception_v3",
                                  "vgg16", "ssd_resnet50"])
@pytest.mark.parametrize("mode", ["bf16", "tf32", "fp8", "fp32"])
def test_plan_invariants_every_family(name, mode):
    cg = _compiled(name, mode)
    fp = plan_fusions(cg, mode)
    _check_invariants(cg, fp)
    if mode == "fp32":                 # the CUDA-core path fuses only BN-ReLU
        assert not (fp.fused_stem or fp.fused_head or fp.sibling or fp.tc_dense)


def test_resnet50_bf16_plan():
    cg = _compiled("resnet50", "bf16")
    fp = plan_fusions(cg, "bf16")
    assert len(fp.fused_stem) == 1 and not fp.stem_fold
    (pool, (conv, src)), = fp.fused_stem.items()
    assert fp.bf16_inputs == {src}                 # host-rounded image upload
    (anchor, info), = fp.fused_head.items()
    assert _kind(cg, anchor) == OpKind.Softmax and info["softmax"]
    assert _kind(cg, info["src"]) == OpKind.Conv2d
    # the projection shortcut and reduce conv of stages 2-4 share a launch
    assert len(fp.sibling) == 3
    assert not fp.fused_bn_relu and not fp.prologue and not fp.junction


def test_tf32_keeps_stem_and_head_unfused():
    fp = plan_fusions(_compiled("resnet50", "tf32"), "tf32")
    assert not fp.fused_stem and not fp.fused_head and len(fp.stem_fold) == 1
    assert fp.stem_fold[next(iter(fp.stem_fold))]["S"] == 7


def test_options_switch_fusions_off():
    cg = _compiled("resnet50", "bf16")
    fp = plan_fusions(cg, "bf16", options=FusionOptions(fused_stem=False, fused_head=False,
                                                         sibling=False))
    assert not fp.fused_stem and not fp.fused_head and not fp.sibling
    assert len(fp.stem_fold) == 1              # the stem falls back to the folded conv
    assert not plan_fusions(cg, "bf16", options=FusionOptions(host_round=False)).bf16_inputs


def test_keep_blocks_fusion_of_kept_values():
    cg = _compiled("resnet50", "bf16")
    fp = plan_fusions(cg, "bf16")
    (pool, (conv, _)), = fp.fused_stem.items()
    (anchor, info), = fp.fused_head.items()
    pool = info["skip"][0]                       # the global average pool
    kept = plan_fusions(cg, "bf16", keep=[conv, pool])
    assert not kept.fused_stem and not kept.fused_head
    assert conv not in kept.skip and pool not in kept.skip
    # a kept Dense stays readable: the head then ends at the Dense (softmax apart)
    dense_kept = plan_fusions(cg, "bf16", keep=[info["dense"]])
    (anchor2, info2), = dense_kept.fused_head.items()
    assert anchor2 == info["dense"] and not info2["softmax"]


def test_densenet_prologue_option():
    cg = _compiled("densenet201", "bf16")
    base = plan_fusions(cg, "bf16")
    assert len(base.fused_bn_relu) > 90 and not base.prologue
    pro = plan_fusions(cg, "bf16", options=FusionOptions(prologue=True))
    assert pro.prologue
    assert len(pro.prologue) + len(pro.fused_bn_relu) == len(base.fused_bn_relu)
    for conv, bn in pro.prologue.items():
        node = cg.nodes[conv]
        relu = node.inputs[0][0]
        assert _kind(cg, relu) == OpKind.ReLU and relu in pro.skip
        assert pro.pro_src[relu] == cg.nodes[bn].inputs[0][0]
        assert hw_pair(node.attrs["pad"]) == (0, 0)
    # the reference keeps its graph: a kept ReLU is never absorbed
    relu0 = next(iter(base.fused_bn_relu))
    assert relu0 in plan_fusions(cg, "bf16", keep=[relu0],
                                 options=FusionOptions(prologue=True)).fused_bn_relu


def test_junction_option_pairs_bottlenecks():
    cg = _compiled("resnet50", "bf16")
    fp = plan_fusions(cg, "bf16", options=FusionOptions(junction=True))
    assert fp.junction
    for e, r in fp.junction.items():
        assert cg.nodes[r].inputs[0][0] == e and fp.junction_of[r] == e
        assert (cg.nodes[e].attrs.get("epilogue") or {}).get("residual")
    big = plan_fusions(cg, "bf16", options=FusionOptions(junction=True, junction_min_hw=56 * 56))
    assert 0 < len(big.junction) < len(fp.junction)


def test_options_from_env(monkeypatch):
    for k in ("NEOB200_PROLOGUE", "NEOB200_NO_FUSED_STEM", "NEOB200_NO_FUSED_HEAD",
              "NEOB200_NO_SIBLING", "NEOB200_JUNCTION", "NEOB200_JUNCTION_MIN_HW"):
        monkeypatch.delenv(k, raising=False)
    assert FusionOptions.from_env() == FusionOptions()
    monkeypatch.setenv("NEOB200_NO_SIBLING", "1")
    monkeypatch.setenv("NEOB200_JUNCTION", "1")
    monkeypatch.setenv("NEOB200_JUNCTION_MIN_HW", "784")
    o = FusionOptions.from_env(host_round=False)
    assert not o.sibling and o.junction and o.junction_min_hw == 784 and not o.host_round
