"""Global planner and PBQP (CPU).  Mirrors reference tests/test_planning.py
and tests/test_pbqp.py: DP equals brute force, PBQP never beats DP, state
explosion falls back, plan JSON round trips -- and reproduces the
reference's own DP/PBQP costs and assignments on the golden instances."""

import itertools
import json
import os
import sys

import numpy as np
import pytest

from paper_1809_02697_b200 import (ConvSchedule, Graph, MeasuredScheme, Node, OpKind,
                                   PbqpInstance, ScheduleDb, SchemePlan, dp_plan, pbqp_solve,
                                   plan, solve_dp)
from paper_1809_02697_b200.errors import Infeasible, MissingSchedule, StateExplosion
from paper_1809_02697_b200.planning import build_problem, conv_workloads, prune_candidates

GOLD = os.path.join(os.path.dirname(__file__), "golden")


class StubCosts:
    """Deterministic stand-in for the measured retile table (restates the
    reference test helper tests/helpers.py:12-20)."""

    def cost(self, shape, from_x, to_x):
        if from_x == to_x:
            return 0.0
        return ((from_x * 31 + to_x * 17 + sum(shape)) % 7 + 1) * 1e5


def brute_force(inst):
    nodes = sorted(inst.costs)
    best = (np.inf, None)
    for combo in itertools.product(*[range(len(inst.costs[n])) for n in nodes]):
        a = dict(zip(nodes, combo))
        c = inst.objective(a)
        if c < best[0]:
            best = (c, a)
    return best


def random_instance(seed, n=6, k=3, density=0.5):
    rng = np.random.default_rng(seed)
    inst = PbqpInstance()
    for i in range(n):
        inst.add_node(i, rng.uniform(0, 10, k))
    for u in range(n):
        for v in range(u + 1, n):
            if rng.random() < density:
                inst.add_edge(u, v, rng.uniform(0, 10, (k, k)))
    return inst


def golden_cases():
    sys.path.insert(0, GOLD)
    import graphio
    doc = json.load(open(os.path.join(GOLD, "planner.json")))
    arrays = np.load(os.path.join(GOLD, "planner.npz"))
    for case in doc["cases"]:
        g = graphio.load_graph(case["graph"], arrays, Graph, Node, OpKind)
        cands = {int(cid): [MeasuredScheme.from_dict(m) for m in ms]
                 for cid, ms in case["candidates"].items()}
        yield case, g, cands


def test_matches_reference_planner_on_golden_instances():
    n = 0
    for case, g, cands in golden_cases():
        prob = build_problem(g, cands, StubCosts())
        assert len(prob.nodes) == case["n_nodes"]
        dp_assign, dp_cost = solve_dp(prob.instance)
        assert dp_cost == pytest.approx(case["dp_cost"], rel=1e-12)
        assert {str(k): v for k, v in dp_assign.items()} == case["dp_assign"]
        pb_assign, pb_cost = pbqp_solve(prob.instance)
        assert pb_cost == pytest.approx(case["pbqp_cost"], rel=1e-12)
        assert {str(k): v for k, v in pb_assign.items()} == case["pbqp_assign"]
        assert pb_cost >= dp_cost - 1e-6
        n += 1
    assert n == 8


@pytest.mark.parametrize("seed", range(10))
def test_dp_equals_brute_force(seed):
    inst = random_instance(seed, n=5, k=3)
    assign, cost = solve_dp(inst)
    bf_cost, _ = brute_force(inst)
    assert cost == pytest.approx(bf_cost)
    assert inst.objective(assign) == pytest.approx(cost)


@pytest.mark.parametrize("seed", range(10))
def test_pbqp_quality(seed):
    inst = random_instance(seed, n=7, k=3, density=0.6)
    _, dp_cost = solve_dp(inst)
    _, pb_cost = pbqp_solve(inst)
    assert pb_cost >= dp_cost - 1e-9
    assert dp_cost / pb_cost >= 0.5


def test_pbqp_exact_on_chains_and_infeasible():
    inst = PbqpInstance()
    for i in range(5):
        inst.add_node(i, [1.0, 2.0, 0.5])
    for i in range(4):
        m = np.full((3, 3), 3.0)
        np.fill_diagonal(m, 0.0)
        inst.add_edge(i, i + 1, m)
    _, cost = pbqp_solve(inst)
    assert cost == pytest.approx(brute_force(inst)[0])
    bad = PbqpInstance()
    bad.add_node(0, [1.0, 1.0])
    bad.add_node(1, [1.0, 1.0])
    bad.add_edge(0, 1, np.full((2, 2), np.inf))
    with pytest.raises(Infeasible):
        pbqp_solve(bad)


def test_state_explosion_and_fallback(monkeypatch):
    inst = random_instance(1, n=8, k=4, density=1.0)
    with pytest.raises(StateExplosion):
        solve_dp(inst, state_cap=3)


def test_plan_entry_point_and_json(tmp_path):
    case, g, cands = next(golden_cases())
    db = ScheduleDb(str(tmp_path / "s.npsd"))
    key = "test-machine"
    for nid, wl in conv_workloads(g).items():
        db.put(key, wl, cands[nid])
    p = plan(g, db, costs=StubCosts(), cpu=key)
    assert p.solver == "DP"
    again = SchemePlan.from_json(p.to_json())
    assert again.schedules() == p.schedules() and again.total_ns == p.total_ns
    pb = plan(g, db, costs=StubCosts(), cpu=key, state_cap=1)
    assert pb.solver == "PBQP" and pb.total_ns >= p.total_ns - 1e-6
    with pytest.raises(MissingSchedule):
        plan(g, ScheduleDb(), costs=StubCosts(), cpu=key)
    via_dp = dp_plan(g, {nid: prune_candidates(db.get(key, wl))
                         for nid, wl in conv_workloads(g).items()}, StubCosts())
    assert via_dp.total_ns == pytest.approx(p.total_ns)


def test_prune_keeps_best_per_pair():
    ms = [MeasuredScheme(ConvSchedule(4, 8, r, True), t, 0.0, 1)
          for r, t in ((8, 5.0), (4, 3.0), (2, 9.0))]
    ms.append(MeasuredScheme(ConvSchedule(8, 8, 4, True), 4.0, 0.0, 1))
    best = prune_candidates(ms)
    assert [(m.schedule.ic_bn, m.schedule.reg_n, m.mean_ns) for m in best] == \
        [(4, 4, 3.0), (8, 4, 4.0)]


class DividingCosts(StubCosts):
    """StubCosts that, like the device table, refuses splits that do not
    divide the tensor's channels."""

    def cost(self, shape, from_x, to_x):
        from paper_1809_02697_b200.errors import IndivisibleChannel
        if shape[1] % from_x or shape[1] % to_x:
            raise IndivisibleChannel(f"C={shape[1]} vs {from_x}->{to_x}")
        return super().cost(shape, from_x, to_x)


def _dense_block_graph(layers=4, growth=32, c0=64):
    """A DenseNet-style block: x0 -> [conv -> concat]* with growth-channel
    convs (oc 32 only) joined onto a running concat whose first input may
    sit in 64-lane blocks."""
    rng = np.random.default_rng(0)
    g = Graph("dense")
    x = g.add(OpKind.Input, shape=(1, 3, 16, 16), layout="NCHW", name="data")
    w = g.constant(rng.standard_normal((c0, 3, 3, 3)).astype(np.float32))
    cur = g.add(OpKind.Conv2d, inputs=[x, w], stride=1, pad=1)
    c = c0
    for _ in range(layers):
        wg = g.constant(rng.standard_normal((growth, c, 1, 1)).astype(np.float32))
        br = g.add(OpKind.Conv2d, inputs=[cur, wg], stride=1, pad=0)
        cur = g.add(OpKind.Concat, inputs=[cur, br], axis=1)
        c += growth
    g.outputs = [cur]
    return g


def test_nested_concat_joins_degrade_per_join():
    """DenseNet's nested concats: a 64-lane first input next to a 32-channel
    branch cannot share a split.  Each such join costs the NCHW round trip
    (reference passes.py:222-227) instead of infinity, so both the DP and
    PBQP find a finite plan and PBQP is not Infeasible."""
    g = _dense_block_graph()
    cands = {}
    for nid, wl in conv_workloads(g).items():
        # the block's first conv only offers 64-lane outputs: every join
        # mirrors it, and every 32-channel branch needs the fallback
        ocs = [64] if wl.in_channel == 3 else [x for x in (64, 32) if wl.out_channel % x == 0]
        ics = [x for x in (64, 32) if wl.in_channel % x == 0] or [1]
        cands[nid] = [MeasuredScheme(ConvSchedule(ic, oc, 8, True), 1e4 + 100 * ic + oc, 0.0, 1)
                      for ic in ics for oc in ocs]
    prob = build_problem(g, cands, DividingCosts())
    picks, cost = pbqp_solve(prob.instance)
    assert np.isfinite(cost)
    dp_picks, dp_cost = solve_dp(prob.instance)
    assert np.isfinite(dp_cost) and dp_cost <= cost + 1e-6
    assert dp_cost == pytest.approx(brute_force(prob.instance)[0])
    # the same instance with the pre-fallback semantics (indivisible = inf)
    # has no finite assignment at all
    from paper_1809_02697_b200 import planning
    orig = planning.join_fallback_ns
    try:
        planning.join_fallback_ns = lambda costs, shape, fx: np.inf
        hard = build_problem(g, cands, DividingCosts())
        with pytest.raises((Infeasible, StateExplosion)):
            solve_dp(hard.instance)
    finally:
        planning.join_fallback_ns = orig
