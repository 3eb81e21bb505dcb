"""Metrics mirror: the reference's throughput / idle_fraction definitions (metrics.py:113-169)
and its known answers (tests/test_metrics.py of the reference)."""

import pytest

from paper_1905_03960_b200.metrics import Sample, NetSampler, idle_fraction, samples_from_csv, samples_to_csv, throughput


def test_throughput_formula():
    r = throughput([100.0] * 5 + [50.0] * 4, batch_size=32, num_workers=4, skip_iterations=5)
    assert r.measure_iterations == 4
    assert r.window_seconds == pytest.approx(0.2)
    assert r.samples_per_second == pytest.approx(4 * 32 * 4 / 0.2)
    with pytest.raises(ValueError):
        throughput([1.0] * 5, 32, 1, skip_iterations=5)


def test_idle_fraction():
    s = [Sample(0, 0, 0), Sample(10, 0, 0), Sample(20, 100, 0), Sample(30, 100, 0), Sample(40, 300, 50), Sample(50, 300, 50)]
    # active window: intervals 1..3 -> deltas [100, 0, 250]; below 10 -> 1 of 3
    assert idle_fraction(s, 10) == pytest.approx(1 / 3)
    assert idle_fraction([Sample(0, 0, 0), Sample(10, 0, 0)], 1) == 1.0
    assert samples_from_csv(samples_to_csv(s)) == s


def test_sampler_monotone():
    class C:
        n = 0

        def totals(self):
            self.n += 1
            return self.n, 2 * self.n

    smp = NetSampler(C(), period_ms=5)
    smp.start()
    import time

    time.sleep(0.06)
    smp.stop()
    ts = [x.t_ms for x in smp.samples]
    assert len(ts) >= 5 and ts == sorted(ts)
    assert all(b.bytes_in >= a.bytes_in for a, b in zip(smp.samples, smp.samples[1:]))


def test_samples_and_timeline_from_device_trace():
    # link bytes from trace records: pushes of slices owned elsewhere leave the pusher and
    # enter the owner; a broadcast leaves the owner N-1 times and enters every other rank
    from dataclasses import dataclass

    from paper_1905_03960_b200.metrics import iteration_timeline, link_bytes, samples_from_trace
    from paper_1905_03960_b200.model import LayerSpec, ModelProfile
    from paper_1905_03960_b200.plan import make_p3_plan

    @dataclass
    class R:
        t_ns: int
        iteration: int
        layer: int
        slice: int
        rank: int
        event: int

    plan = make_p3_plan(ModelProfile("m", 0, (LayerSpec(0, "a", 10, 0, 0), LayerSpec(1, "b", 30, 0, 0))), 2, 20)
    owner = {(s.key.layer_index, s.key.slice_index): s.server for s in plan.slices}
    assert owner == {(0, 0): 0, (1, 0): 1, (1, 1): 0}
    ms = 1_000_000
    traces = {
        0: [R(0, 0, 0, 0, 0, 5), R(1 * ms, 0, 1, 0, 0, 0), R(2 * ms, 0, 0, 0, 0, 0), R(12 * ms, 0, 0, 0, 0, 1),
            R(15 * ms, 0, 1, 1, 0, 1), R(31 * ms, 0, 0, 0, 0, 6)],
        1: [R(0, 0, 0, 0, 1, 5), R(3 * ms, 0, 0, 0, 1, 0), R(4 * ms, 0, 1, 1, 1, 0), R(25 * ms, 0, 1, 0, 1, 1),
            R(30 * ms, 0, 0, 0, 1, 6)],
    }
    rows = link_bytes(traces, plan, 0)
    assert sum(r[2] for r in rows) == 4 * 20 + 4 * 10 + 4 * 10  # push (1,0) + bcasts of (0,0), (1,1)
    assert sum(r[1] for r in rows) == 4 * 10 + 4 * 10 + 4 * 20  # push of (0,0), (1,1) from rank 1 + bcast (1,0)
    smp = samples_from_trace(traces, plan, 0, 0, 31 * ms)
    assert [s.t_ms for s in smp] == [0, 10, 20, 30, 40]
    assert smp[-1].bytes_out == 160 and smp[1].bytes_out == 80 and smp[2].bytes_out == 160
    walls, starts = iteration_timeline(traces[0], 0)
    assert walls == [31.0] and starts == [0.0]
