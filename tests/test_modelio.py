"""Model container, toy generators, CLI and runtime compatibility names
(CPU).  Mirrors the reference's tests/test_modelio.py (round trips, CRC and
truncation errors) and pins byte compatibility against files the reference
itself wrote (tests/golden/model_*.json/.npwt, from make_golden.py)."""

import filecmp
import json
import os
import struct
import sys

import numpy as np
import pytest

from paper_1809_02697_b200 import (Graph, Node, OpKind, ThreadPool, gen_model, load_model,
                                   parallel_for, read_weights, save_model, split_ranges,
                                   write_weights)
from paper_1809_02697_b200 import cli
from paper_1809_02697_b200.errors import CorruptModel

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _same_graph(a, b):
    assert a.name == b.name and list(a.outputs) == list(b.outputs)
    assert sorted(a.nodes) == sorted(b.nodes)
    for nid in a.nodes:
        na, nb = a.nodes[nid], b.nodes[nid]
        assert na.kind == nb.kind and [tuple(e) for e in na.inputs] == [tuple(e) for e in nb.inputs]
        assert set(na.attrs) == set(nb.attrs)
        for k, va in na.attrs.items():
            vb = nb.attrs[k]
            if isinstance(va, np.ndarray):
                assert va.dtype == vb.dtype and np.array_equal(va, vb)
            elif isinstance(va, dict):
                assert set(va) == set(vb)
                for kk in va:
                    if isinstance(va[kk], np.ndarray):
                        assert np.array_equal(va[kk], vb[kk])
                    else:
                        assert va[kk] == vb[kk]
            else:
                assert va == vb, (nid, k)


@pytest.mark.parametrize("tag", ["toy", "opt"])
def test_reference_files_load_and_resave_bit_identical(tmp_path, tag):
    js, wt = os.path.join(GOLD, f"model_{tag}.json"), os.path.join(GOLD, f"model_{tag}.npwt")
    g = load_model(js, wt)
    save_model(g, tmp_path / "m.json", tmp_path / "m.npwt")
    assert filecmp.cmp(js, tmp_path / "m.json", shallow=False)
    assert filecmp.cmp(wt, tmp_path / "m.npwt", shallow=False)
    _same_graph(g, load_model(tmp_path / "m.json", tmp_path / "m.npwt"))


def test_gen_model_matches_reference_toys():
    """gen_model draws the reference's seeded constants in the same order:
    the golden toy graphs (written by the reference) are reproduced exactly."""
    sys.path.insert(0, GOLD)
    import graphio
    doc = json.load(open(os.path.join(GOLD, "graphs.json")))
    arrays = np.load(os.path.join(GOLD, "graphs.npz"))
    for case in doc["cases"]:
        kind, seed = case["tag"].rsplit("-", 1)
        ref = graphio.load_graph(case["graph"], arrays, Graph, Node, OpKind)
        _same_graph(gen_model(kind, depth=2, channels=8, hw=8, seed=int(seed)), ref)
    g = load_model(os.path.join(GOLD, "model_toy.json"), os.path.join(GOLD, "model_toy.npwt"))
    _same_graph(gen_model("resnet-block", depth=2, channels=8, hw=8, seed=4), g)


def test_gen_model_rejects_bad_arguments():
    with pytest.raises(ValueError):
        gen_model("unet")
    with pytest.raises(ValueError):
        gen_model("chain", depth=0)


def test_weights_round_trip_and_alignment(tmp_path):
    rng = np.random.default_rng(0)
    t = {"b": rng.standard_normal((3, 5)).astype(np.float32), "a": np.float32(2.5) * np.ones(()),
         "c": rng.standard_normal((2, 1, 4, 4)).astype(np.float32)}
    write_weights(tmp_path / "w.npwt", t)
    raw = open(tmp_path / "w.npwt", "rb").read()
    assert raw[:4] == b"NPWT" and struct.unpack_from("<II", raw, 4) == (1, 3)
    back = read_weights(tmp_path / "w.npwt")
    assert sorted(back) == ["a", "b", "c"]
    for k in t:
        assert np.array_equal(back[k], np.asarray(t[k], np.float32))


def _corrupt(tmp_path, fn):
    src = os.path.join(GOLD, "model_toy.npwt")
    raw = bytearray(open(src, "rb").read())
    fn(raw)
    p = tmp_path / "bad.npwt"
    p.write_bytes(bytes(raw))
    return p


@pytest.mark.parametrize("damage", [
    lambda r: r.__setitem__(0, ord("X")),                  # magic
    lambda r: r.__setitem__(4, 2),                         # version
    lambda r: r.__setitem__(20, r[20] ^ 0xFF),             # header byte -> CRC mismatch
    lambda r: r.__delitem__(slice(40, None)),              # truncated header
    lambda r: r.__delitem__(slice(len(r) - 64, None)),     # payload past the end
])
def test_corrupt_weights_raise(tmp_path, damage):
    with pytest.raises(CorruptModel):
        read_weights(_corrupt(tmp_path, damage))


def test_corrupt_graph_json_raises(tmp_path):
    wt = os.path.join(GOLD, "model_toy.npwt")
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(CorruptModel):
        load_model(tmp_path / "bad.json", wt)
    doc = json.load(open(os.path.join(GOLD, "model_toy.json")))
    doc["nodes"][0]["kind"] = "Deconv"
    (tmp_path / "kind.json").write_text(json.dumps(doc))
    with pytest.raises(CorruptModel):
        load_model(tmp_path / "kind.json", wt)
    doc = json.load(open(os.path.join(GOLD, "model_toy.json")))
    write_weights(tmp_path / "empty.npwt", {})
    (tmp_path / "ok.json").write_text(json.dumps(doc))
    with pytest.raises(CorruptModel):
        load_model(tmp_path / "ok.json", tmp_path / "empty.npwt")


def test_cli_gen_and_exit_codes(tmp_path, capsys):
    js, wt = str(tmp_path / "m.json"), str(tmp_path / "m.npwt")
    assert cli.main(["gen", "--kind", "diamond-concat", "--depth", "2", "--channels", "8",
                     "--out", js, "--weights", wt]) == 0
    _same_graph(load_model(js, wt), gen_model("diamond-concat", depth=2, channels=8))
    # plan against an empty schedule DB: missing schedules -> 4
    assert cli.main(["plan", "--model", js, "--weights", wt, "--schedule-db",
                     str(tmp_path / "db.npsd"), "--machine", "nobody"]) == 4
    # corrupt weights -> 3
    (tmp_path / "bad.npwt").write_bytes(b"XXXX" + bytes(20))
    assert cli.main(["run", "--model", js, "--weights", str(tmp_path / "bad.npwt")]) == 3
    # invalid graph (dangling edge) -> 2
    doc = json.load(open(js))
    doc["nodes"][-1]["inputs"] = [[999, 0]]
    (tmp_path / "dangling.json").write_text(json.dumps(doc))
    assert cli.main(["run", "--model", str(tmp_path / "dangling.json"), "--weights", wt]) == 2


def test_threadpool_and_parallel_for():
    seen = []
    with ThreadPool(4) as pool:
        assert pool.num_threads == 4 and pool.devices == [0]
        parallel_for(pool, 10, lambda lo, hi: seen.extend(range(lo, hi)))
    assert sorted(seen) == list(range(10))
    assert split_ranges(10, 4) == [(0, 3), (3, 6), (6, 9), (9, 10)]

    def boom(lo, hi):
        if lo > 0:
            raise RuntimeError("worker failed")
    with pytest.raises(RuntimeError):
        parallel_for(ThreadPool(3), 9, boom)
