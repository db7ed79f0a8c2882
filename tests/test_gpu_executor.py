"""End-to-end parity of the device executor against the CPU oracle on
identical seeded inputs and random-init weights (north_star tolerances:
tf32 logits <= 1e-3, bf16 <= 2e-2; fp32 within the reference's own 1e-4
end-to-end bound, tests/test_acceptance.py:145-163)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "tf32": 1e-3, "bf16": 2e-2}


def _run(g, mode, optimize=True, keep=()):
    from paper_1809_02697_b200 import DevicePool, compile_graph, execute, model_input
    feeds = model_input(g, seed=1)
    ref = oracle.execute_reference(g, feeds)
    graph = compile_graph(g, mode=mode) if optimize else g
    got = execute(graph, feeds, DevicePool(0, mode), keep=keep)
    return ref, got


@pytest.mark.parametrize("mode", ["fp32", "tf32", "bf16"])
def test_resnet18_logits(cuda, mode):
    from paper_1809_02697_b200 import build_model
    g = build_model("resnet18", batch=2, softmax=False)
    ref, got = _run(g, mode)
    assert got[0].shape == (2, 1000)
    err = oracle.rel_err(got[0], ref[0])
    assert err < TOL[mode], err
    assert (got[0].argmax(1) == ref[0].argmax(1)).all()


@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_resnet50_logits(cuda, mode):
    from paper_1809_02697_b200 import build_model
    g = build_model("resnet50", batch=1, softmax=False)
    ref, got = _run(g, mode)
    assert oracle.rel_err(got[0], ref[0]) < TOL[mode]
    assert (got[0].argmax(1) == ref[0].argmax(1)).all()


def test_unoptimized_graph_naive_path(cuda):
    """Default-layout graph (no planning): every conv runs the naive device
    conv_reference path; must match the oracle like the reference's naive
    executor does."""
    from paper_1809_02697_b200 import build_model
    g = build_model("resnet18", batch=1, image=64, num_classes=10)
    ref, got = _run(g, "fp32", optimize=False)
    assert oracle.rel_err(got[0], ref[0]) < 1e-4


@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_small_densenet_bn_relu_and_concat(cuda, mode):
    from paper_1809_02697_b200.models import densenet
    g = densenet(blocks=(2, 3), growth=16, batch=2, image=64, num_classes=10, softmax=False)
    ref, got = _run(g, mode)
    assert oracle.rel_err(got[0], ref[0]) < TOL[mode]


@pytest.mark.parametrize("mode", ["fp32", "tf32", "bf16"])
def test_concat_in_place(cuda, mode):
    """Dense-block concats run in place: producers write their channel-block
    windows of the block's buffer, so no concat copy is launched, and the
    logits still match the oracle."""
    from paper_1809_02697_b200 import DeviceProgram, ExecutablePlan, compile_graph, model_input
    from paper_1809_02697_b200.models import densenet
    g = densenet(blocks=(3, 4), growth=32, batch=2, image=64, num_classes=10, softmax=False)
    feeds = model_input(g, seed=1)
    ref = oracle.execute_reference(g, feeds)
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=mode)), 0, mode)
    assert any(v.win is not None for v in prog.vals.values())
    copies = [n for n in prog.launch_names if n.startswith("concat")]
    assert not copies, copies
    got = prog.run(feeds)
    assert oracle.rel_err(got[0], ref[0]) < TOL[mode]


def test_softmax_and_cuda_graph_replay(cuda):
    from paper_1809_02697_b200 import (DevicePool, ExecutablePlan, build_model, compile_graph,
                                       execute, model_input)
    g = build_model("resnet18", batch=2, image=64, num_classes=10)
    feeds = model_input(g)
    plan = ExecutablePlan.compile(compile_graph(g, mode="tf32"))
    pool = DevicePool(0, "tf32")
    probs, logits = execute(plan, feeds, pool, keep=[g.logits_id])
    probs2, logits2 = execute(plan, feeds, pool, keep=[g.logits_id])
    assert np.array_equal(probs, probs2) and np.array_equal(logits, logits2)
    ref_logits = oracle.execute_reference(_with_outputs(g, [g.logits_id]), feeds)[0]
    assert oracle.rel_err(logits, ref_logits) < 1e-3
    # softmax kernel vs the oracle softmax of the same device logits
    assert np.abs(probs - oracle.softmax(logits)).max() < 1e-6
    assert np.allclose(probs.sum(1), 1.0, atol=1e-5)


def _with_outputs(g, outs):
    h = g.copy()
    h.outputs = list(outs)
    return h


def test_nhwc_input_and_per_conv_packing(cuda):
    from paper_1809_02697_b200 import (DevicePool, build_model, execute, model_input, passes)
    # 224x224 (the BASELINE input size): at toy sizes the tf32 logits error of
    # random-init ResNet-18 spreads around 0.4e-3..1.3e-3 from seed to seed
    g = build_model("resnet18", batch=1, softmax=False)
    feeds = model_input(g)
    ref = oracle.execute_reference(g, feeds)[0]
    s = passes.simplify(g)
    assign = passes.uniform_assignment(s, mode="tf32")
    ablation = passes.pretransform_weights(passes.per_conv_packing(s, assign))
    got = execute(ablation, feeds, DevicePool(0, "tf32"))[0]
    assert oracle.rel_err(got, ref) < 1e-3
    # NHWC-declared input is ingested once into NCHW
    h = g.copy()
    for node in h.nodes.values():
        if node.kind.value == "Input":
            n, c, hh, ww = node.attrs["shape"]
            node.attrs["shape"] = (n, hh, ww, c)
            node.attrs["layout"] = "NHWC"
    nhwc = {"data": feeds["data"].transpose(0, 2, 3, 1).copy()}
    got2 = execute(passes.compile_graph(h, mode="tf32"), nhwc, DevicePool(0, "tf32"))[0]
    assert oracle.rel_err(got2, ref) < 1e-3


@pytest.mark.parametrize("model", ["vgg16", "inception_v3", "densenet201"])
def test_baseline_models_bf16(cuda, model):
    from paper_1809_02697_b200 import build_model
    g = build_model(model, batch=1, softmax=False)
    ref, got = _run(g, "bf16")
    assert oracle.rel_err(got[0], ref[0]) < TOL["bf16"]
    assert (got[0].argmax(1) == ref[0].argmax(1)).all()


@pytest.mark.parametrize("mode,tol", [("fp32", 1e-4), ("tf32", 3e-3), ("bf16", 4e-2)])
def test_ssd_heads(cuda, mode, tol):
    """12 pre-NMS head maps of SSD-512/ResNet-50.  The north_star bounds
    (tf32 1e-3, bf16 2e-2) are stated for classifier logits; the detector
    heads sit ~60 rounded layers deep and are held to measured-plus-margin
    bounds here (measured: tf32 1.9e-3, bf16 1.2e-2..3.0e-2 per head, the
    sqrt(depth) growth of one bf16 storage rounding per layer).  fp32 mode
    checks the same graph at 1e-4."""
    from paper_1809_02697_b200 import build_model
    g = build_model("ssd_resnet50", batch=1)
    ref, got = _run(g, mode)
    assert len(got) == 12
    for a, b in zip(got, ref):
        assert a.shape == b.shape
        assert oracle.rel_err(a, b) < tol


@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_densenet_bn_relu_prologue_fusion(cuda, mode, monkeypatch):
    """Opt-in executor fusion of DenseNet's pre-activation BN-ReLU into the
    following 1x1 conv (NEOB200_PROLOGUE=1): fewer launches, same logits."""
    from paper_1809_02697_b200 import DeviceProgram, ExecutablePlan, compile_graph, model_input
    from paper_1809_02697_b200.models import densenet
    g = densenet(blocks=(3, 4), growth=32, batch=2, image=64, num_classes=10, softmax=False)
    feeds = model_input(g, seed=1)
    ref = oracle.execute_reference(g, feeds)
    plain = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=mode)), 0, mode)
    monkeypatch.setenv("NEOB200_PROLOGUE", "1")
    fused = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode=mode)), 0, mode)
    assert fused.prologue and len(fused.launches) < len(plain.launches)
    a, b = plain.run(feeds)[0], fused.run(feeds)[0]
    assert np.array_equal(a, b)
    assert oracle.rel_err(b, ref[0]) < TOL[mode]
