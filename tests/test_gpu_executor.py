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


def test_ssd_heads_fp32_path(cuda):
    """C4 (SSD-512/ResNet-50, 12 pre-NMS head maps) on the fp32 path: every
    head within 1e-4 of the oracle (the reference's own end-to-end bound,
    tests/test_acceptance.py:145-163, tighter than north_star's 1e-3)."""
    from paper_1809_02697_b200 import build_model
    g = build_model("ssd_resnet50", batch=1)
    ref, got = _run(g, "fp32")
    assert len(got) == 12
    for a, b in zip(got, ref):
        assert a.shape == b.shape
        assert oracle.rel_err(a, b) < 1e-4


@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_ssd_heads_single_pass_modes(cuda, mode):
    """SSD heads in the single-pass tensor-core modes.  The heads sit ~60
    conv layers deep in a random-init ResNet-50 whose activations grow to
    ~6e4; the f32 oracle with nothing but the mode's RN operand / storage
    roundings (oracle.ops.conv2d_rounded: no kernel, no reordering) already
    lands at tf32 ~3e-3 and bf16 ~2.5e-2 on these heads -- the number
    formats, not the kernels, set the error, so the device is held to its
    own arithmetic: worst head within 1.25x the modelled worst head, and the
    logits-level bounds of north_star are met where they are stated
    (test_resnet50_logits, test_bench_program_logits_vs_oracle)."""
    from paper_1809_02697_b200 import build_model, compile_graph, model_input
    g = build_model("ssd_resnet50", batch=1)
    ref, got = _run(g, mode)
    model = oracle.execute_reference(compile_graph(g, mode=mode), model_input(g, seed=1),
                                     arith=mode)
    assert len(got) == 12
    e_dev = max(oracle.rel_err(a, b) for a, b in zip(got, ref))
    e_model = max(oracle.rel_err(m, b) for m, b in zip(model, ref))
    # the device and the model are two realisations of the same rounding
    # noise: per head they differ by tens of percent either way, so the
    # bound is on the worst head
    assert e_dev < 1.25 * e_model, (e_dev, e_model)


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
