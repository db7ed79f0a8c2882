"""Host-side logic that needs no GPU: schedule database (reference
tests/test_tuning.py:49-133), candidate space, runtime / batch split
(tests/test_runtime.py:9-29), workload & schedule types
(tests/test_kernels.py:36-68), model builders, the executor's arena planner,
and the C-ABI library (loads; exports every symbol include/neob200.h
declares; no compute calls)."""

import os
import re
import struct

import numpy as np
import pytest

from paper_1809_02697_b200 import (ConvSchedule, ConvWorkload, DevicePool, Epilogue,
                                   MeasuredScheme, ScheduleDb, build_model, split_ranges)
from paper_1809_02697_b200.errors import CorruptDb, ScheduleInvalid, ShapeMismatch
from paper_1809_02697_b200.tuning import generate_candidates, local_search

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class TestTypes:
    def test_workload_dims(self):
        wl = ConvWorkload(8, 16, 56, 56, 3, 3, 1, 1)
        assert (wl.out_h, wl.out_w) == (56, 56)
        assert ConvWorkload(8, 16, 56, 56, 3, 3, 2, 1).out_h == 28
        assert ConvWorkload(8, 8, 17, 17, 1, 7, 1, (0, 3)).out_w == 17
        with pytest.raises(ShapeMismatch):
            ConvWorkload(4, 4, 2, 2, 5, 5, 1, 0)
        assert ConvWorkload(64, 64, 56, 56, 3, 3, 1, 1).flops() == 231211008  # BASELINE C0

    def test_schedule_check_and_dict(self):
        wl = ConvWorkload(8, 12, 8, 8, 3, 3, 1, 1)
        ConvSchedule(4, 6, 8).check(wl)
        for bad in (ConvSchedule(3, 6, 8), ConvSchedule(4, 5, 8), ConvSchedule(0, 6, 8)):
            with pytest.raises(ScheduleInvalid):
                bad.check(wl)
        s = ConvSchedule(4, 8, 16, True, tile_n=128, stages=3)
        assert ConvSchedule.from_dict(s.as_dict()) == s
        # reference-format dicts (4 keys) still load
        assert ConvSchedule.from_dict({"ic_bn": 4, "oc_bn": 8, "reg_n": 16,
                                       "unroll_ker": True}) == ConvSchedule(4, 8, 16, True)
        assert Epilogue().is_empty() and not Epilogue(relu=True).is_empty()


class TestScheduleDb:
    def make(self):
        wl = ConvWorkload(8, 8, 8, 8, 3, 3, 1, 1)
        ms = [MeasuredScheme(ConvSchedule(4, 4, 8, True, tile_n=64), 5.0, 0.1, 3),
              MeasuredScheme(ConvSchedule(8, 8, 8, True), 2.0, 0.1, 3)]
        return wl, ms

    def test_round_trip_sorted(self, tmp_path):
        wl, ms = self.make()
        path = str(tmp_path / "db.npsd")
        db = ScheduleDb(path)
        db.put("gpu", wl, ms)
        again = ScheduleDb(path)
        got = again.get("gpu", wl)
        assert [m.mean_ns for m in got] == [2.0, 5.0]
        assert got[1].schedule.tile_n == 64
        assert again.workloads("gpu") == [wl] and len(again) == 1
        assert not os.path.exists(path + ".tmp")

    def test_corruption_detected(self, tmp_path):
        wl, ms = self.make()
        path = str(tmp_path / "db.npsd")
        ScheduleDb(path).put("gpu", wl, ms)
        raw = bytearray(open(path, "rb").read())
        raw[20] ^= 0xFF
        open(path, "wb").write(bytes(raw))
        with pytest.raises(CorruptDb):
            ScheduleDb(path)
        open(path, "wb").write(b"XXXX" + struct.pack("<I", 1))
        with pytest.raises(CorruptDb):
            ScheduleDb(path)
        open(path, "wb").write(b"NPSD" + struct.pack("<I", 9))
        with pytest.raises(CorruptDb):
            ScheduleDb(path)
        open(path, "wb").write(b"NPSD" + struct.pack("<I", 1) + struct.pack("<I", 100) + b"{}")
        with pytest.raises(CorruptDb):
            ScheduleDb(path)

    def test_cache_hit_skips_measurement(self, monkeypatch):
        wl, ms = self.make()
        db = ScheduleDb()
        db.put("gpu", wl, ms)

        def boom(*a, **k):
            raise AssertionError("measured despite cache hit")
        monkeypatch.setattr("paper_1809_02697_b200.tuning.measure", boom)
        assert local_search(wl, db=db, cpu="gpu") == db.get("gpu", wl)

    def test_candidates_are_tensor_core_legal(self):
        space = generate_candidates(ConvWorkload(256, 512, 14, 14, 3, 3, 1, 1), "bf16")
        assert set(space.ic_bn_list) == {8, 16, 32, 64}
        assert all(t.get("tile_n", 16) % 16 == 0 for t in space.tile_list)
        stem = generate_candidates(ConvWorkload(3, 64, 224, 224, 7, 7, 2, 3), "bf16")
        assert stem.ic_bn_list == (1,)
        head = generate_candidates(ConvWorkload(512, 84, 32, 32, 3, 3, 1, 1), "bf16")
        assert head.oc_bn_list == (42,)
        tf = generate_candidates(ConvWorkload(64, 64, 8, 8, 1, 1, 1, 0), "tf32")
        assert set(tf.ic_bn_list) == {4, 8, 16, 32}


class TestRuntime:
    @pytest.mark.parametrize("n,parts", [(10, 3), (7, 7), (3, 8), (64, 8), (512, 8), (1, 1)])
    def test_split_ranges_cover(self, n, parts):
        r = split_ranges(n, parts)
        assert r[0][0] == 0 and r[-1][1] == n
        assert all(a < b for a, b in r) and all(r[i][1] == r[i + 1][0] for i in range(len(r) - 1))
        assert len(r) <= parts

    def test_device_pool(self):
        p = DevicePool([0, 1, 2, 3], "bf16")
        assert p.shards(512) == [(0, (0, 128)), (1, (128, 256)), (2, (256, 384)),
                                 (3, (384, 512))]
        assert DevicePool(2, "tf32").devices == [2]
        with pytest.raises(ValueError):
            DevicePool([0], "fp16")
        assert split_ranges(0, 4) == []


class TestModels:
    @pytest.mark.parametrize("name,gflop", [("resnet18", 3.627), ("resnet50", 7.712),
                                           ("vgg16", 30.693), ("densenet201", 8.579)])
    def test_conv_flops(self, name, gflop):
        from paper_1809_02697_b200.models import conv_flops
        g = build_model(name, batch=1)
        assert conv_flops(g) / 1e9 == pytest.approx(gflop, abs=5e-3)

    def test_inception_and_ssd_shapes(self):
        from paper_1809_02697_b200 import infer_shapes, validate
        g = build_model("inception_v3", batch=2)
        assert not validate(g)
        assert infer_shapes(g)[g.outputs[0]].shape == (2, 1000)
        asym = [n for n in g.nodes.values() if n.kind.value == "Conv2d"
                and isinstance(n.attrs["pad"], tuple) and n.attrs["pad"][0] != n.attrs["pad"][1]]
        assert len(asym) > 10
        ssd = build_model("ssd_resnet50", batch=1)
        shapes = [infer_shapes(ssd)[o].shape for o in ssd.outputs]
        assert [s[2] for s in shapes[::2]] == [32, 16, 8, 4, 2, 1]
        assert [s[1] for s in shapes[::2]] == [84, 126, 126, 126, 84, 84]


def test_arena_planner_never_overlaps_live_buffers():
    from paper_1809_02697_b200.executor import _plan_arena, _Val
    rng = np.random.default_rng(0)
    vals = []
    for i in range(200):
        first = int(rng.integers(0, 100))
        v = _Val(i, (int(rng.integers(1, 5000)),), _dtype(), None)
        v.first, v.last = first, first + int(rng.integers(0, 20))
        vals.append(v)
    size = _plan_arena(vals)
    for a in vals:
        for b in vals:
            if a is b or a.last < b.first or b.last < a.first:
                continue
            assert a.offset + a.nbytes <= b.offset or b.offset + b.nbytes <= a.offset
    assert size >= max(v.offset + v.nbytes for v in vals)
    assert size < sum(v.nbytes for v in vals)      # reuse happened


def _dtype():
    import torch
    return torch.float32


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "neob200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(neo_[a-z0-9_]+)\s*\(", text)))


def test_native_library_exports_every_declared_symbol():
    import ctypes
    from paper_1809_02697_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    loaded = _lib.load()
    assert loaded.neo_abi_version() == 3
    assert loaded.neo_last_error() is not None
    assert loaded.neo_conv_params_size() == ctypes.sizeof(_lib.ConvParams)


def test_integration_doc_binding_matches_the_abi():
    """The ctypes ConvParams a maintainer would copy from INTEGRATION.md has
    the library's layout (same fields, same size), and a struct built for an
    older, shorter layout is rejected by the library instead of being read
    past its end (no GPU needed: the size check precedes any device call)."""
    import ctypes
    from paper_1809_02697_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = text.split("# neoplan/b200.py")[1].split("```")[0]
    code = block.split("class ConvParams", 1)[1].split("\nassert ", 1)[0]
    ns = {"ctypes": ctypes}
    exec("class ConvParams" + code, ns)
    Doc = ns["ConvParams"]
    assert [f[0] for f in Doc._fields_] == [f[0] for f in _lib.ConvParams._fields_]
    lib = _lib.load()
    assert ctypes.sizeof(Doc) == lib.neo_conv_params_size()
    p = Doc(mode=2)
    assert p.struct_size == ctypes.sizeof(Doc)
    p.struct_size = ctypes.sizeof(Doc) - 40          # a v1-era binding
    st = lib.neo_conv_default_tiles(ctypes.cast(ctypes.byref(p), ctypes.POINTER(_lib.ConvParams)))
    assert st == 7 or st != 0          # NEO_ERR_INVALID_ARG
    assert b"struct_size" in lib.neo_last_error()


def test_library_errors_map_to_reference_exceptions():
    """A CPU-side argument check (no kernel launch) surfaces as the reference
    exception type."""
    from paper_1809_02697_b200 import _lib
    from paper_1809_02697_b200.errors import IndivisibleChannel, ShapeMismatch as SM
    lib = _lib.load()
    st = lib.neo_layout_transform(0, 0, 16, 16, 1, 6, 2, 2, 0, 1, 2, 4, 0, None)
    with pytest.raises(IndivisibleChannel):
        _lib.check(st)
    st = lib.neo_layout_transform(0, 0, 16, 16, 0, 6, 2, 2, 0, 1, 2, 3, 0, None)
    with pytest.raises(SM):
        _lib.check(st)


def _rn_f32(fr):
    """Exact round-to-nearest-even of a Fraction to binary32 (as a float)."""
    from fractions import Fraction
    if fr == 0:
        return 0.0
    sign = -1.0 if fr < 0 else 1.0
    v = abs(fr)
    e = v.numerator.bit_length() - v.denominator.bit_length()
    if Fraction(2) ** e > v:
        e -= 1
    e = max(e, -126)                       # subnormals share the minimum exponent
    scale = Fraction(2) ** (e - 23)
    m = v / scale
    n = m.numerator // m.denominator
    rem = m - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return sign * float(n * scale)


def test_pool_division_by_constant_is_correctly_rounded():
    """ops.cu div_rn_const (avg pool /9): q = RN(a r), rem = fma(-q, d, a),
    RN(q + rem r) with r = RN(1/d) equals IEEE a / d for random f32 sums and
    for quotients crafted next to rounding midpoints, so the fast path stays
    bit-identical to the reference's numpy division (executor.py:125)."""
    from fractions import Fraction as F
    rng = np.random.default_rng(7)
    d = 9.0
    r = float(np.float32(1.0) / np.float32(9.0))
    a = list((rng.standard_normal(3000) * np.exp2(rng.integers(-60, 60, 3000))).astype(np.float32))
    for _ in range(3000):                   # a / 9 within an ulp of a midpoint
        mid = F(int(rng.integers(1 << 24, 1 << 25)) * 2 + 1, 1 << int(rng.integers(20, 30)))
        base = np.float32(float(mid * 9))
        a += [base, np.nextafter(base, np.float32(np.inf)), np.nextafter(base, np.float32(-np.inf))]
    for x in a:
        x = float(x)
        q = _rn_f32(F(x) * F(r))
        rem = _rn_f32(F(x) - F(d) * F(q))
        q1 = _rn_f32(F(rem) * F(r) + F(q))
        assert q1 == float(np.float32(x) / np.float32(d)), x


def test_fp8_scale_groups_and_pools():
    """quant.attach_scales (host logic, no GPU): a max pool keeps its
    input's scale, every member of an in-place concat group (transitively
    through nested concats) takes the group's largest scale, and a global
    average pool the fused head absorbs gets none."""
    from paper_1809_02697_b200.graph import OpKind
    from paper_1809_02697_b200.models import NetBuilder
    from paper_1809_02697_b200.passes import compile_graph
    from paper_1809_02697_b200.quant import attach_scales, quantized_nodes
    b = NetBuilder("groups", 1, 3, 32)
    x = b.conv_bn_relu(b.data, 3, 64, 3)
    p = b.maxpool(x, 2, 2)
    c1 = b.conv_bn_relu(p, 64, 64, 1)
    c2 = b.conv_bn_relu(p, 64, 64, 3)
    cat1 = b.concat([p, c1])
    cat2 = b.concat([cat1, c2])
    head = b.avgpool(b.conv_bn_relu(cat2, 192, 256, 1), 16, 1)
    b.g.outputs = [b.classifier(head, 256, 10, softmax=False)]
    cg = compile_graph(b.g, mode="bf16")
    q = quantized_nodes(cg)
    kinds = {cg.nodes[n].kind for n in q}
    assert OpKind.Conv2d in kinds and OpKind.MaxPool in kinds
    assert not any(cg.nodes[n].kind == OpKind.AvgPool for n in q)   # global, C % 256 == 0
    scales = {n: 2.0 ** (i % 5 - 2) for i, n in enumerate(sorted(q))}
    attach_scales(cg, scales)
    sc = lambda n: cg.nodes[n].attrs.get("fp8_scale")
    pools = [n for n in q if cg.nodes[n].kind == OpKind.MaxPool]
    cats = [n for n, nd in cg.nodes.items() if nd.kind == OpKind.Concat]
    assert len(pools) == 1 and len(cats) == 2
    members = set(cats)
    for c in cats:
        members |= {s for s, _ in cg.nodes[c].inputs}
    group = {sc(m) for m in members}
    assert len(group) == 1 and None not in group            # one scale for the group
    top = group.pop()
    assert top == max(scales[m] for m in members if m in scales)
    # the pool is a group member: its scale was raised to the group's
    assert sc(pools[0]) == top
