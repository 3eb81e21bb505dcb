"""Host token bucket (the K7 rule with the reference's transport API): the behaviours the
reference's transport tests pin (tests/test_transport.py: bad rate, free first burst, rate
over a short window, one bucket shared by threads, pass-through shaper)."""

import threading
import time

import pytest

from paper_1905_03960_b200.shaping import Shaper, TokenBucket


def test_rejects_bad_rate():
    with pytest.raises(ValueError):
        TokenBucket(0)


def test_first_burst_is_free():
    b = TokenBucket(8_000_000, burst_bytes=10_000)
    t0 = time.perf_counter()
    b.consume(10_000)
    assert time.perf_counter() - t0 < 0.05


def test_rate_over_a_short_window():
    b = TokenBucket(800_000, burst_bytes=10_000)  # 100 KB/s
    b.consume(10_000)
    t0 = time.perf_counter()
    b.consume(20_000)  # 20 KB beyond the burst: ~0.2 s
    assert 0.15 <= time.perf_counter() - t0 <= 0.35


def test_shared_across_threads():
    b = TokenBucket(1_600_000, burst_bytes=5_000)  # 200 KB/s
    def send():
        for _ in range(6):
            b.consume(5_000)
    t0 = time.perf_counter()
    ts = [threading.Thread(target=send) for _ in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    # 60 KB combined, 5 KB free: ~0.275 s
    assert 0.2 <= time.perf_counter() - t0 <= 0.45


def test_shaper_pass_through():
    s = Shaper(None)
    t0 = time.perf_counter()
    s.consume(10**9)
    assert time.perf_counter() - t0 < 0.01 and s.bucket is None
