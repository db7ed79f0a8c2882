#!/usr/bin/env python
"""Generate the golden fixtures by running the UNMODIFIED reference package
(neoplan, /root/reference/pkg/src or baseline/_ref) on seeded inputs.

Run in the build container (the reference does not exist on the GPU box):
    python tests/golden/make_golden.py
Fixtures written next to this script:
  layouts.npz        pack/unpack/retile/NHWC/weight-pack outputs (bit patterns)
  conv.npz           conv_reference and conv_blocked outputs incl. epilogues and
                     BASELINE config 0 (3x3 64->64 56x56 + BN + ReLU, NCHW16c)
  pool.npz           _pool2d outputs on NCHW and NCHW[x]c
  graphs.json/.npz   the four reference toy models + their unoptimized and
                     optimized executor outputs, assignment and transform count
  models.npz         ResNet-18/50 logits (this repo's seeded builders, run by
                     the reference executor) + weight digests
  planner.json/.npz  DP / PBQP results on random layout problems
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle.refbridge import import_reference, reference_optimized, to_reference_graph  # noqa: E402
import graphio  # noqa: E402


def layouts(neo):
    from neoplan import layout as L
    rng = np.random.default_rng(100)
    out = {}
    a = rng.standard_normal((2, 12, 5, 7)).astype(np.float32)
    out["a"] = a
    for x in (1, 2, 3, 4, 6, 12):
        p = L.pack_nchw_array(a, x)
        out[f"pack_x{x}"] = p
        out[f"unpack_x{x}"] = L.unpack_nchw_array(p)
    p4 = L.pack_nchw_array(a, 4)
    for b in (2, 3, 6, 12):
        out[f"retile_4_{b}"] = L.retile_nchw_array(p4, b)
    big = rng.standard_normal((1, 64, 9, 9)).astype(np.float32)
    out["big"] = big
    out["big_pack16"] = L.pack_nchw_array(big, 16)
    out["big_pack64"] = L.pack_nchw_array(big, 64)
    nhwc = rng.standard_normal((2, 5, 6, 3)).astype(np.float32)
    out["nhwc"] = nhwc
    out["nhwc_to_nchw"] = L.nhwc_to_nchw_array(nhwc)
    w = rng.standard_normal((8, 4, 3, 3)).astype(np.float32)
    out["w"] = w
    for x, y in ((1, 1), (2, 4), (4, 8), (4, 2)):
        pk = L.pack_kcrs_array(w, x, y)
        out[f"wpack_{x}_{y}"] = pk
        out[f"wunpack_{x}_{y}"] = L.unpack_kcrs_array(pk)
    np.savez_compressed(os.path.join(HERE, "layouts.npz"), **out)


CONV_CASES = [
    # (C, K, H, W, R, S, stride, pad), (ic_bn, oc_bn, reg_n, unroll), epilogue kind
    ((3, 5, 9, 9, 3, 3, 1, 1), (1, 5, 4, True), "none"),
    ((4, 4, 8, 10, 1, 1, 1, 0), (2, 4, 8, True), "bias_relu"),
    ((2, 7, 11, 11, 5, 5, 1, 2), (1, 7, 8, True), "scale_shift"),
    ((6, 3, 12, 12, 3, 3, 2, 1), (3, 3, 5, True), "all"),
    ((1, 1, 7, 7, 7, 7, 1, 3), (1, 1, 4, False), "none"),
    ((8, 16, 7, 7, 1, 1, 1, 0), (8, 16, 7, True), "residual"),
    ((8, 8, 10, 10, 3, 3, 1, 1), (2, 8, 4, True), "all"),
    ((16, 32, 6, 6, 3, 3, 2, 1), (16, 16, 8, True), "all"),
]


def _epilogue(neo, kind, k, rng, out_shape):
    epi = neo.Epilogue()
    arrays = {}
    if kind in ("scale_shift", "all"):
        arrays["scale"] = rng.uniform(0.5, 1.5, k).astype(np.float32)
        arrays["shift"] = rng.uniform(-1, 1, k).astype(np.float32)
    if kind in ("bias_relu", "all"):
        arrays["bias"] = rng.uniform(-1, 1, k).astype(np.float32)
    if kind in ("residual", "all"):
        arrays["residual"] = rng.standard_normal(out_shape).astype(np.float32)
    relu = kind in ("bias_relu", "all")
    return arrays, relu


def conv(neo):
    from neoplan.layout import pack_data, pack_weights, unpack_data
    out = {}
    for i, (wl_t, sch_t, ekind) in enumerate(CONV_CASES):
        c, k, h, w, r, s, st, pd = wl_t
        wl = neo.ConvWorkload(c, k, h, w, r, s, st, pd)
        sch = neo.ConvSchedule(*sch_t)
        rng = np.random.default_rng(200 + i)
        x = rng.standard_normal((1, c, h, w)).astype(np.float32)
        wt = rng.standard_normal((k, c, r, s)).astype(np.float32)
        arrays, relu = _epilogue(neo, ekind, k, rng, (1, k, wl.out_h, wl.out_w))
        epi_ref = neo.Epilogue(arrays.get("scale"), arrays.get("shift"), arrays.get("bias"),
                               relu, arrays.get("residual"))
        ref = neo.conv_reference(neo.Tensor(x), neo.Tensor(wt, neo.KCRS), wl, epi_ref).data
        res_b = None
        if "residual" in arrays:
            res_b = pack_data(neo.Tensor(arrays["residual"]), sch.oc_bn).data
        epi_blk = neo.Epilogue(arrays.get("scale"), arrays.get("shift"), arrays.get("bias"),
                               relu, res_b)
        blk = unpack_data(neo.conv_blocked(pack_data(neo.Tensor(x), sch.ic_bn),
                                           pack_weights(neo.Tensor(wt, neo.KCRS), sch.ic_bn,
                                                        sch.oc_bn), wl, sch, epi_blk)).data
        out[f"{i}/wl"] = np.array(wl_t, np.int64)
        out[f"{i}/sch"] = np.array(sch_t, np.int64)
        out[f"{i}/x"] = x
        out[f"{i}/w"] = wt
        out[f"{i}/relu"] = np.array(relu)
        for key, v in arrays.items():
            out[f"{i}/{key}"] = v
        out[f"{i}/reference"] = ref
        out[f"{i}/blocked"] = blk
    # BASELINE config 0: NCHW16c input N(0,1), He weights, BN(gamma U, beta N(0,.1),
    # mean N(0,.1), var U) folded into scale/shift, ReLU
    rng = np.random.default_rng(0)
    x16 = rng.standard_normal((1, 4, 56, 56, 16)).astype(np.float32)
    wt = (rng.standard_normal((64, 64, 3, 3)) * np.sqrt(2.0 / 576)).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, 64)
    beta = rng.normal(0, 0.1, 64)
    mean = rng.normal(0, 0.1, 64)
    var = rng.uniform(0.5, 1.5, 64)
    scale = (gamma / np.sqrt(var + 1e-5)).astype(np.float32)
    shift = (beta - mean * gamma / np.sqrt(var + 1e-5)).astype(np.float32)
    wl = neo.ConvWorkload(64, 64, 56, 56, 3, 3, 1, 1)
    sch = neo.ConvSchedule(16, 16, 8, True)
    x = unpack_data(neo.Tensor(x16, neo.nchwc(16))).data
    ref = neo.conv_reference(neo.Tensor(x), neo.Tensor(wt, neo.KCRS), wl,
                             neo.Epilogue(scale=scale, shift=shift, relu=True)).data
    blk = neo.conv_blocked(neo.Tensor(x16, neo.nchwc(16)),
                           pack_weights(neo.Tensor(wt, neo.KCRS), 16, 16), wl, sch,
                           neo.Epilogue(scale=scale, shift=shift, relu=True)).data
    out.update({"c0/x16": x16, "c0/w": wt, "c0/scale": scale, "c0/shift": shift,
                "c0/reference": ref, "c0/blocked16": blk})
    np.savez_compressed(os.path.join(HERE, "conv.npz"), **out)


def pool(neo):
    from neoplan.executor import _pool2d
    from neoplan.layout import pack_nchw_array
    rng = np.random.default_rng(300)
    a = rng.standard_normal((2, 8, 9, 9)).astype(np.float32)
    out = {"a": a}
    for mode in ("max", "avg"):
        for win, st, pd in ((2, 2, 0), (3, 2, 1), (3, 1, 1), (9, 1, 0)):
            out[f"{mode}_{win}_{st}_{pd}"] = _pool2d(a, win, st, pd, mode)
            out[f"{mode}_{win}_{st}_{pd}_b4"] = _pool2d(pack_nchw_array(a, 4), win, st, pd, mode)
    np.savez_compressed(os.path.join(HERE, "pool.npz"), **out)


def graphs(neo):
    doc = {"cases": []}
    arrays = {}
    for kind in neo.models.KINDS:
        for seed in (0, 1):
            g = neo.gen_model(kind, depth=2, channels=8, hw=8, seed=seed)
            rng = np.random.default_rng(400 + seed)
            inp = rng.standard_normal((1, 8, 8, 8)).astype(np.float32)
            plain = neo.execute(g, {"data": inp})
            s = neo.simplify(g)
            assign = neo.uniform_assignment(s)
            opt = neo.pretransform_weights(neo.alter_and_insert_transforms(s, assign))
            optimized = neo.execute(opt, {"data": inp})
            tag = f"{kind}-{seed}"
            arrays[f"{tag}/input"] = inp
            for i, o in enumerate(plain):
                arrays[f"{tag}/plain{i}"] = o
            for i, o in enumerate(optimized):
                arrays[f"{tag}/opt{i}"] = o
            doc["cases"].append({
                "tag": tag, "graph": graphio.dump_graph(g, tag, arrays),
                "n_outputs": len(plain),
                "assignment": {str(k): list(v) for k, v in assign.items()},
                "split_factor": neo.passes.uniform_split_factor(s),
                "transforms": neo.count_transforms(opt),
                "simplified_nodes": len(s.nodes), "optimized_nodes": len(opt.nodes)})
    graphio.save(os.path.join(HERE, "graphs.json"), os.path.join(HERE, "graphs.npz"), doc, arrays)


def digest(g) -> str:
    h = hashlib.sha256()
    for nid in sorted(g.nodes):
        v = g.nodes[nid].attrs.get("value")
        if v is not None:
            h.update(np.ascontiguousarray(v, np.float32).tobytes())
    return h.hexdigest()


def models(neo):
    from paper_1809_02697_b200 import build_model, model_input
    out = {}
    cases = [("resnet18", 1, {}), ("resnet50", 1, {}),
             ("resnet18", 2, {"image": 64, "num_classes": 10})]
    for name, batch, kw in cases:
        g = build_model(name, batch=batch, softmax=False, **kw)
        feeds = model_input(g)
        ng = to_reference_graph(g, neo)
        with neo.ThreadPool(neo.physical_cores()) as pool:
            logits = neo.execute(reference_optimized(ng, neo), feeds, pool)[0]
        tag = f"{name}_b{batch}" + ("_small" if kw else "")
        out[f"{tag}/input_digest"] = np.frombuffer(
            hashlib.sha256(feeds["data"].tobytes()).digest(), np.uint8)
        out[f"{tag}/weight_digest"] = np.frombuffer(bytes.fromhex(digest(g)), np.uint8)
        out[f"{tag}/logits"] = logits
    np.savez_compressed(os.path.join(HERE, "models.npz"), **out)


def planner(neo):
    sys.path.insert(0, "/root/reference/pkg/tests")
    import helpers  # reference test helpers (random graphs, candidates, stub costs)
    doc = {"cases": []}
    arrays = {}
    for seed in range(8):
        g = helpers.random_conv_graph(seed)
        cands = helpers.random_candidates(g, seed) if hasattr(helpers, "random_candidates") \
            else None
        costs = helpers.StubCosts()
        prob = neo.planning.build_problem(g, cands, costs)
        dp_assign, dp_cost = neo.solve_dp(prob.instance)
        pb_assign, pb_cost = neo.pbqp_solve(prob.instance)
        tag = f"rand{seed}"
        doc["cases"].append({
            "tag": tag, "graph": graphio.dump_graph(g, tag, arrays),
            "candidates": {str(cid): [m.to_dict() for m in ms] for cid, ms in cands.items()},
            "dp_cost": dp_cost, "dp_assign": {str(k): v for k, v in dp_assign.items()},
            "pbqp_cost": pb_cost, "pbqp_assign": {str(k): v for k, v in pb_assign.items()},
            "n_nodes": len(prob.nodes)})
    graphio.save(os.path.join(HERE, "planner.json"), os.path.join(HERE, "planner.npz"), doc,
                 arrays)


def modelfiles(neo):
    """Model container files written by the reference (modelio.py): a raw
    toy graph and an optimized one (packed weights, epilogue dicts), to pin
    byte compatibility of save_model / load_model / read_weights."""
    g = neo.gen_model("resnet-block", depth=2, channels=8, hw=8, seed=4)
    neo.save_model(g, os.path.join(HERE, "model_toy.json"), os.path.join(HERE, "model_toy.npwt"))
    s = neo.simplify(neo.gen_model("diamond-concat", depth=2, channels=16, hw=8, seed=5))
    opt = neo.pretransform_weights(neo.alter_and_insert_transforms(s, neo.uniform_assignment(s, 8)))
    neo.save_model(opt, os.path.join(HERE, "model_opt.json"), os.path.join(HERE, "model_opt.npwt"))


def main(only=None):
    neo = import_reference()
    print("reference:", neo.__file__)
    steps = [layouts, conv, pool, graphs, models, planner, modelfiles]
    for step in steps:
        if only is None or step.__name__ in only:
            step(neo)
    print("fixtures written to", HERE)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
