"""The C++ schedule model (p3_simulate) against the reference simulator's timelines
(tests/golden: figure scenarios, shipped scenario files, 50+ seeded random scenarios, the
slice-size sweep) and the reference's own golden numbers (tests/test_sim.py:56-136)."""

import pytest

from paper_1905_03960_b200.sim import (
    AGGRESSIVE_COARSE,
    PRIORITY_SLICED,
    DOWNLINK,
    UPDATE,
    UPLINK,
    Scenario,
    ScenarioError,
    StageCost,
    scenario_from_dict,
    scenario_to_dict,
    simulate,
    sweep_slice_size,
)
from paper_1905_03960_b200.model import LayerSpec, ModelProfile


def test_all_golden_timelines(golden):
    assert len(golden["sim_cases"]) >= 50
    for case in golden["sim_cases"]:
        sc = scenario_from_dict(case["scenario"])
        tl = simulate(sc)
        assert tl.to_csv() == case["csv"], case["scenario"]
        assert tl.summary() == case["summary"]
        assert scenario_to_dict(sc) == case["scenario"]


def test_sweep_interior_optimum(golden):
    sw = scenario_from_dict(golden["sweep"]["scenario"])
    got = sweep_slice_size(sw, golden["sweep"]["sizes"])
    assert [list(x) for x in got] == golden["sweep"]["result"]
    best = min(got, key=lambda x: x[1])[0]
    assert best not in (golden["sweep"]["sizes"][0], golden["sweep"]["sizes"][-1])


def _tick(fwd, bwd, n):
    return ModelProfile("sc", 0, tuple(LayerSpec(i, f"L{i}", 1, fwd, bwd) for i in range(n)))


def test_reference_figure_numbers():
    # tests/test_sim.py:88-136 of the reference: Fig.4 delay 4 -> 2, Fig.6 makespan 10 -> 7
    f4 = lambda p: Scenario(_tick(1, 1, 3), (StageCost(2, 0, 0),) * 3, p, 1, 1)
    assert simulate(f4(AGGRESSIVE_COARSE)).inter_iteration_delay() == 4
    pri = simulate(f4(PRIORITY_SLICED))
    assert pri.inter_iteration_delay() == 2
    assert [(e.start, e.end) for e in pri.entries_for("compute") if e.item.startswith("fwd:1")] == [(5, 6), (6, 7), (7, 8)]
    assert pri.busy_intervals(UPLINK) == [(1, 7)]
    f6 = Scenario(_tick(0, 0, 3), (StageCost(1, 1, 1), StageCost(3, 3, 3), StageCost(1, 1, 1)), AGGRESSIVE_COARSE, 1, 1)
    tl = simulate(f6)
    assert tl.makespan == 10
    upd = {e.item: (e.start, e.end) for e in tl.entries_for(UPDATE)}
    assert upd["upd:0:L1:s0"] == (4, 7) and upd["upd:0:L0:s0"] == (5, 6)
    assert tl.busy_intervals(DOWNLINK)[-1][1] == 10


def test_validation_errors():
    with pytest.raises(ScenarioError):
        simulate(Scenario(_tick(1, 1, 2), (StageCost(3, 0, 0),) * 2, PRIORITY_SLICED, slice_ticks=2))
    with pytest.raises(ScenarioError):
        simulate(Scenario(_tick(1, 1, 2), (StageCost(2, 0, 0),), PRIORITY_SLICED))
