"""B200 extension: merge planning with the measured (piecewise) cost curve
(mgw_plan_optimal_table / mgw_predict_table). Not a reference API — checked
against the reference model where they must agree, and against exhaustive
search where they must be optimal."""
import itertools

import numpy as np

from paper_1912_09268_b200 import gradsched as gs


def _trace(rng, L):
    params = [int(x) for x in rng.integers(1, 3_000_000, L)]
    t_b = [float(x) for x in rng.uniform(1e-5, 3e-4, L)]
    return gs.trace_from_arrays(params, t_b, 1e-3)


def test_table_from_a_linear_model_reproduces_the_reference():
    rng = np.random.default_rng(5)
    model = gs.AllReduceModel(2e-5, 1e-9)
    sizes = [0] + [2 ** k for k in range(8, 36)]
    meas = [gs.CommMeasurement(s, model.a + model.b * s) for s in sizes]
    for _ in range(20):
        tr = _trace(rng, int(rng.integers(2, 60)))
        ref_plan = gs.optimal_plan(tr, model)
        tab_plan = gs.optimal_plan_table(tr, meas)
        t_ref = gs.iteration_time(tr, ref_plan, model).iteration_time
        t_tab = gs.iteration_time(tr, tab_plan, model).iteration_time
        assert abs(t_tab - t_ref) <= 1e-9 * t_ref
        assert abs(gs.iteration_time_table(tr, ref_plan, meas) - t_ref) <= 1e-9 * t_ref


def test_table_plan_is_optimal_by_exhaustive_search():
    rng = np.random.default_rng(7)
    # a piecewise, non-linear (but monotone) cost curve like the fused kernel's
    meas = [gs.CommMeasurement(4096, 5e-6), gs.CommMeasurement(512 << 10, 8e-6),
            gs.CommMeasurement(1 << 20, 13e-6), gs.CommMeasurement(8 << 20, 26e-6),
            gs.CommMeasurement(64 << 20, 130e-6)]
    for _ in range(40):
        L = int(rng.integers(2, 11))
        tr = _trace(rng, L)
        best = min(
            gs.iteration_time_table(tr, gs.MergePlan([gs.LayerTag(0)] + [gs.LayerTag(t) for t in tags]), meas)
            for tags in itertools.product([0, 1], repeat=L - 1))
        plan = gs.optimal_plan_table(tr, meas)
        assert gs.iteration_time_table(tr, plan, meas) <= best * (1 + 1e-12)


def test_table_api_rejects_bad_measurements():
    tr = gs.trace_from_arrays([100, 200], [1e-4, 1e-4], 1e-3)
    import pytest

    with pytest.raises(gs.ValidationError):
        gs.optimal_plan_table(tr, [])
    with pytest.raises(gs.ValidationError):
        gs.optimal_plan_table(tr, [gs.CommMeasurement(1024, 0.0)])
    # a single point is a flat (latency-only) curve: merging everything is optimal
    plan = gs.optimal_plan_table(tr, [gs.CommMeasurement(1024, 1e-3)])
    assert [int(t) for t in plan.tags] == [0, 1]
