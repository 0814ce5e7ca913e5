"""Bit-exact parity of the host solver / predictor / fit (libmgwfbp.so,
through the C ABI) with the reference.

Three independent sources agree on every case:
  golden.json  — outputs of the UNMODIFIED reference headers (tools/make_golden.py)
  oracle C     — the literal O(L^2) restatement (oracle/mgw_oracle.c)
  oracle/_ref  — the reference compiled in place (when built)
Known answers are the reference tests' own golden values
(test_planner.cpp:221-280, test_timeline.cpp:146-172, test_cli.cpp:145-153).
"""
import math
import os
import random

import pytest

from conftest import GOLDEN
from oracle import pyoracle
from paper_1912_09268_b200 import gradsched as gs


def _trace(params, t_b, t_f, bpe=4):
    return gs.trace_from_arrays(params, t_b, t_f, bpe)


def _tags(plan):
    return "".join(str(int(t)) for t in plan.tags)


def test_golden_cases_bit_exact(golden):
    assert len(golden["cases"]) >= 100
    for c in golden["cases"]:
        t_b = [float.fromhex(x) for x in c["t_b"]]
        tr = _trace(c["params"], t_b, float.fromhex(c["t_f"]), c["bpe"])
        m = gs.AllReduceModel(float.fromhex(c["a"]), float.fromhex(c["b"]))
        opt = gs.optimal_plan(tr, m)
        gr = gs.greedy_plan(tr, m)
        assert _tags(opt) == c["optimal"], c["name"]
        assert _tags(gr) == c["greedy"], c["name"]
        assert gs.iteration_time(tr, opt, m).iteration_time.hex() == c["t_optimal"], c["name"]
        assert gs.iteration_time(tr, gr, m).iteration_time.hex() == c["t_greedy"], c["name"]
        L = len(c["params"])
        assert gs.iteration_time(tr, gs.MergePlan.all_normal(L), m).iteration_time.hex() == c["t_wfbp"]
        single = gs.iteration_time(tr, gs.MergePlan.all_merged(L), m).iteration_time
        assert single.hex() == c["t_single"]
        assert gs.synceasgd_time(tr, m) == single  # timeline.hpp:218-221 bitwise identity


def _random_case(rng):
    L = rng.randint(1, 300)
    params = [0 if rng.random() < 0.1 else int(math.exp(rng.uniform(0, math.log(3e7)))) for _ in range(L)]
    if not any(params):
        params[0] = 1
    t_b = [0.0 if rng.random() < 0.1 else math.exp(rng.uniform(math.log(1e-6), math.log(1e-2))) for _ in range(L)]
    t_f = rng.choice([0.0, math.exp(rng.uniform(math.log(1e-5), math.log(1e-1)))])
    a = rng.choice([1e-9, math.exp(rng.uniform(math.log(1e-6), math.log(1e-2)))])
    b = rng.choice([0.0, math.exp(rng.uniform(math.log(1e-12), math.log(1e-8)))])
    return params, t_b, t_f, a, b


def test_optimal_and_greedy_match_literal_restatement():
    rng = random.Random(8675309)
    for _ in range(300):
        params, t_b, t_f, a, b = _random_case(rng)
        bpe = rng.choice([2, 4])
        tr = _trace(params, t_b, t_f, bpe)
        m = gs.AllReduceModel(a, b)
        opt = [int(t) for t in gs.optimal_plan(tr, m).tags]
        assert opt == pyoracle.orc_optimal(params, t_b, t_f, bpe, a, b)
        gr = [int(t) for t in gs.greedy_plan(tr, m).tags]
        assert gr == pyoracle.orc_greedy(params, t_b, t_f, bpe, a, b)
        assert gs.iteration_time(tr, gs.MergePlan([gs.LayerTag(x) for x in opt]), m).iteration_time == \
            pyoracle.orc_iteration_time(params, t_b, t_f, bpe, a, b, opt)


@pytest.mark.skipif(pyoracle.REF is None, reason="oracle/_ref not built")
def test_optimal_and_greedy_match_reference_build_live():
    rng = random.Random(424242)
    for _ in range(300):
        params, t_b, t_f, a, b = _random_case(rng)
        tr = _trace(params, t_b, t_f)
        m = gs.AllReduceModel(a, b)
        assert [int(t) for t in gs.optimal_plan(tr, m).tags] == pyoracle.ref_optimal(params, t_b, t_f, 4, a, b)
        assert [int(t) for t in gs.greedy_plan(tr, m).tags] == pyoracle.ref_greedy(params, t_b, t_f, 4, a, b)


def test_optimal_equals_brute_force_small():
    # reference test_planner.cpp:126-155 (ties, zeros, degenerate models)
    rng = random.Random(555777)
    for _ in range(400):
        L = rng.randint(1, 9)
        params = [rng.choice([0, rng.randint(1, 4), int(math.exp(rng.uniform(math.log(25), math.log(2.5e7))))])
                  for _ in range(L)]
        if not any(params):
            params[0] = 1
        t_b = [rng.choice([0.0, math.exp(rng.uniform(math.log(1e-6), math.log(1e-2)))]) for _ in range(L)]
        tr = _trace(params, t_b, rng.choice([0.0, 1e-3]))
        m = gs.AllReduceModel(rng.choice([1e-9, 1e-4, 1e-2]), rng.choice([0.0, 1e-9]))
        plan = gs.optimal_plan(tr, m)
        assert gs.iteration_time(tr, plan, m).iteration_time == gs.brute_force_plan(tr, m).iteration_time


def test_known_answers_three_layer_and_counterexample():
    m = gs.AllReduceModel(1e-3, 1e-9)
    tr = gs.load_trace(os.path.join(GOLDEN, "three_layer.json"))
    plan = gs.optimal_plan(tr, m)
    assert [int(t) for t in plan.tags] == [0, 0, 1]
    assert plan.groups() == [[0], [1, 2]]
    assert abs(gs.iteration_time(tr, plan, m).iteration_time - 6.5e-3) < 1e-9
    ce = gs.load_trace(os.path.join(GOLDEN, "greedy_counterexample.json"))
    g = gs.greedy_plan(ce, m)
    o = gs.optimal_plan(ce, m)
    assert [int(t) for t in g.tags] == [0, 0, 1]
    assert [int(t) for t in o.tags] == [0, 1, 0]
    assert gs.iteration_time(ce, o, m).iteration_time == 0.055000000000000007
    assert gs.iteration_time(ce, g, m).iteration_time == 0.055500000000000008
    assert gs.iteration_time(ce, o, m).iteration_time == gs.brute_force_plan(ce, m).iteration_time


def test_timeline_goldens():
    # test_timeline.cpp:146-156 two-layer golden and :164-172 zero-param head
    tl = gs.iteration_time(_trace([10, 10], [1.0, 1.0], 0.0), gs.MergePlan.all_normal(2), gs.AllReduceModel(0.1, 0.0))
    assert abs(tl.tau_c[1] - 1.0) < 1e-9 and abs(tl.tau_c[0] - 2.0) < 1e-9
    assert abs(tl.iteration_time - 2.1) < 1e-9 and abs(tl.comm_nonoverlap - 0.1) < 1e-9
    tl = gs.iteration_time(_trace([0, 1000], [1e-3, 1e-3], 0.0), gs.MergePlan.all_normal(2), gs.AllReduceModel(0.5, 0.0))
    assert tl.t_c[0] == 0.5 and abs(tl.iteration_time - 1.001) < 1e-12


def test_fit_cluster1_bits(golden):
    meas = gs.load_measurements_csv(os.path.join(GOLDEN, "cluster1_allreduce.csv"))
    assert len(meas) == 40
    m = gs.fit_model(meas)
    assert m.a.hex() == golden["cluster1_fit"]["a"]
    assert m.b.hex() == golden["cluster1_fit"]["b"]
    assert m.a == 9.6743922885256055e-4 and m.b == 1.9857165404367356e-9  # SURVEY §8c probe bits
    a, b = pyoracle.orc_fit([x.size_bytes for x in meas], [x.time_sec for x in meas])
    assert (a, b) == (m.a, m.b)


def test_fit_noiseless_exact_and_errors():
    truth = gs.AllReduceModel(9.72e-4, 1.97e-9)
    ms = [gs.CommMeasurement(int(s), truth.a + truth.b * s) for s in (1e3, 1e5, 1e6, 1e7, 1e8)]
    m = gs.fit_model(ms)
    assert abs(m.a - truth.a) <= 1e-12 and abs(m.b - truth.b) <= 1e-12
    with pytest.raises(gs.FitError):
        gs.fit_model([gs.CommMeasurement(1024, 1e-3)])
    with pytest.raises(gs.FitError, match="b="):
        gs.fit_model([gs.CommMeasurement(1000, 1e-2), gs.CommMeasurement(1000000, 1e-3)])
    with pytest.raises(gs.FitError, match="a="):
        gs.fit_model([gs.CommMeasurement(1000000, 1e-3), gs.CommMeasurement(2000000, 3e-3)])
    with pytest.raises(gs.ValidationError):
        gs.fit_model([gs.CommMeasurement(1024, 0.0), gs.CommMeasurement(2048, 1e-3)])


def test_planner_errors_map_to_reference_classes():
    tr = _trace([100, 100], [1e-3, 1e-3], 0.0)
    for a, b in ((0.0, 1e-9), (-1e-3, 1e-9), (1e-3, -1e-9)):
        with pytest.raises(gs.PlannerError):
            gs.optimal_plan(tr, gs.AllReduceModel(a, b))
        with pytest.raises(gs.PlannerError):
            gs.greedy_plan(tr, gs.AllReduceModel(a, b))
    big = _trace([1000] * 25, [1e-3] * 25, 0.0)
    with pytest.raises(gs.GuardError, match=r"2\^24"):
        gs.brute_force_plan(big, gs.AllReduceModel(1e-3, 1e-9))
    with pytest.raises(gs.ValidationError):
        gs.optimal_plan(_trace([0, 0], [1e-3, 1e-3], 0.0), gs.AllReduceModel(1e-3, 1e-9))


def test_skewed_161_regenerates_byte_for_byte():
    text = gs.synth_trace_json(gs.SynthSpec(161, 25_500_000, 0.25, 0.125, 8.0, 4, 20))
    with open(os.path.join(GOLDEN, "skewed_161.json")) as f:
        assert text == f.read()


def test_named_traces_load_and_plan():
    tdir = os.path.join(os.path.dirname(GOLDEN), "..", "traces")
    names = [f for f in os.listdir(tdir) if f.endswith(".json") and f != "META.json"] if os.path.isdir(tdir) else []
    if not names:
        pytest.skip("traces/ not generated yet")
    expect = {"googlenet": 173, "resnet50": 161, "resnet152": 467, "densenet201": 604, "bert_large": 398,
              "inception_v4": 449}
    for fn in names:
        tr = gs.load_trace(os.path.join(tdir, fn))
        key = fn[:-5]
        if key in expect:
            assert tr.n_layers() == expect[key]
        m = gs.AllReduceModel(10e-6, 1 / 600e9)
        plan = gs.optimal_plan(tr, m)
        t = gs.iteration_time(tr, plan, m).iteration_time
        assert t <= gs.iteration_time(tr, gs.MergePlan.all_normal(tr.n_layers()), m).iteration_time
        assert t <= gs.synceasgd_time(tr, m)
