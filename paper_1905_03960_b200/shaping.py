"""Link shaping: the token bucket of the reference transport (transport.py:22-66).

On the GPU path shaping is K7 inside the comm kernel (``pace()``, csrc/p3_kernels.cu): one
bucket per rank's egress, charged per job, as a virtual clock on %globaltimer — configured
with ``SyncContext(throttle_bps=..., throttle_burst=...)``. ``TokenBucket`` / ``Shaper`` are
the same rule on the host, with the reference's names and behaviour (rate in bits/s, burst
in bytes, the first burst free, blocking ``consume``, shared by threads) for code that
shapes host-side traffic.
"""

from __future__ import annotations

import threading
import time

DEFAULT_BURST_BYTES = 50 * 1024


class TokenBucket:
    """Blocking token bucket; the virtual-clock form of K7: a grant of n bytes moves the
    clock V (the time the bucket has paid for) to max(V, now - burst/rate) + n/rate and
    returns once now >= V — when all n tokens are taken, as transport.py:42-55 does."""

    def __init__(self, rate_bps: float, burst_bytes: int = DEFAULT_BURST_BYTES) -> None:
        if rate_bps <= 0:
            raise ValueError("rate must be positive; use None for no shaping")
        self.rate_bytes = rate_bps / 8.0
        self.burst = float(burst_bytes)
        self._slack = self.burst / self.rate_bytes  # seconds of burst
        self._v = time.monotonic() - self._slack    # a full bucket at creation
        self._lock = threading.Lock()

    def consume(self, n: int) -> None:
        """Block until n bytes may pass (n may exceed the burst)."""
        with self._lock:
            now = time.monotonic()
            self._v = max(self._v, now - self._slack) + n / self.rate_bytes
            due = self._v
        while True:
            wait = due - time.monotonic()
            if wait <= 0:
                return
            time.sleep(min(wait, 0.05))


class Shaper:
    """Optional bucket (transport.py:58-66): None means pass-through."""

    def __init__(self, rate_bps: float | None, burst_bytes: int = DEFAULT_BURST_BYTES) -> None:
        self.bucket = TokenBucket(rate_bps, burst_bytes) if rate_bps else None

    def consume(self, n: int) -> None:
        if self.bucket is not None:
            self.bucket.consume(n)
