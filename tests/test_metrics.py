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
