"""CPU oracle of the P3 sync path — TEST INFRASTRUCTURE ONLY.

A plain numpy / pure-Python restatement of the reference algorithm (``p3sync``, mounted
read-only at /root/reference/pkg/src/p3sync during development; absent on the GPU box).
It is imported only by ``tests/``, by ``__graft_entry__.smoke()`` and by ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs, and only as the checker or the CPU
baseline — never as a fallback of the product path.

Parity pinning: every function here is checked against the golden vectors of the
reference's own tests and against fixtures produced by running the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/golden.json``; see
``tests/test_oracle.py``). Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import hashlib
import heapq
from dataclasses import dataclass

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15           # hashing.py:15
MUL_ITER = 0x9E3779B97F4A7C15        # hashing.py:16
MUL_LAYER = 0xC2B2AE3D27D4EB4F       # hashing.py:17
MUL_ELEM = 0x165667B19E3779F9        # hashing.py:18
FNV_BASIS = 0xCBF29CE484222325       # hashing.py:20
FNV_MUL = 0x100000001B3              # hashing.py:21


# ------------------------------------------------------------------ hashing.py


def mix(x: int) -> int:
    """splitmix64 finaliser, hashing.py:24-29."""
    x &= M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def stream(seed: int, i: int) -> int:
    """splitmix64_stream, hashing.py:32-35."""
    return mix(seed + (i + 1) * GAMMA)


def grad_one(seed: int, it: int, layer: int, e: int) -> np.float32:
    """gradient_value, hashing.py:45-52 (scalar, arbitrary-precision ints)."""
    x = seed ^ ((it * MUL_ITER) & M64) ^ ((layer * MUL_LAYER) & M64) ^ ((e * MUL_ELEM) & M64)
    return np.float32(float(mix(x) >> 40) * 2.0**-23 - 1.0)


def grad_block(seed: int, it: int, layer: int, start: int, count: int) -> np.ndarray:
    """gradient_block, hashing.py:55-63 (vectorised over uint64 with wraparound)."""
    base = np.uint64((seed ^ ((it * MUL_ITER) & M64) ^ ((layer * MUL_LAYER) & M64)) & M64)
    e = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = base ^ (e * np.uint64(MUL_ELEM))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    top = (z >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (top.astype(np.float64) * 2.0**-23).astype(np.float32)


def fnv(data: bytes, h: int = FNV_BASIS) -> int:
    """fnv1a64, hashing.py:79-83 (pure Python: keep inputs small)."""
    for b in data:
        h = ((h ^ b) * FNV_MUL) & M64
    return h


# ------------------------------------------------------------------ plan.py


@dataclass(frozen=True)
class Row:
    layer: int
    slice: int
    offset: int
    length: int
    priority: int
    server: int


def p3_rows(counts: list[int], servers: int, max_slice: int) -> list[Row]:
    """make_p3_plan, plan.py:94-119 (+ _chunk_layer :82-91)."""
    rows, owner = [], 0
    for layer, c in enumerate(counts):
        starts = list(range(0, c, max_slice))
        for s, off in enumerate(starts):
            rows.append(Row(layer, s, off, min(max_slice, c - off), layer, owner % servers))
            owner += 1
    return rows


def baseline_rows(counts: list[int], servers: int, big: int, seed: int) -> list[Row]:
    """make_baseline_plan, plan.py:122-164."""
    rows = []
    for layer, c in enumerate(counts):
        if c < big:
            rows.append(Row(layer, 0, 0, c, layer, stream(seed, layer) % servers))
            continue
        part = c // servers
        for s in range(servers):
            off = s * part
            rows.append(Row(layer, s, off, part if s < servers - 1 else c - off, layer, s))
    return rows


def plan_csv(mode: str, rows: list[Row], servers: int, max_slice=50_000, big=1_000_000, seed=0) -> str:
    """plan_to_csv, plan.py:196-206."""
    head = f"# p3sync-plan mode={mode} num_servers={servers} max_slice={max_slice} big_threshold={big} rng_seed={seed}\n"
    body = "".join(f"{r.layer},{r.slice},{r.offset},{r.length},{r.priority},{r.server}\n" for r in sorted(rows, key=lambda r: (r.layer, r.slice)))
    return head + "layer,slice,offset,len,priority,server\n" + body


# ------------------------------------------------------------------ server.py


def shard_update(params: np.ndarray, grads_by_rank: dict[int, np.ndarray], lr: float) -> np.ndarray:
    """ShardState.aggregate_and_update, server.py:55-68: zero-initialised fp32 sum in
    ascending rank order, divide by fp32 N, params - fp32(lr) * grad."""
    acc = np.zeros(len(params), dtype=np.float32)
    for r in sorted(grads_by_rank):
        acc = acc + grads_by_rank[r]
    g = acc / np.float32(len(grads_by_rank))
    return params - np.float32(lr) * g


def shard_update_scalar(params: np.ndarray, grads_by_rank: dict[int, np.ndarray], lr: float) -> np.ndarray:
    """Element-by-element fp32 replay (tests/test_server.py:14-25), for pinning shard_update."""
    out = np.empty_like(params)
    n = np.float32(len(grads_by_rank))
    lr32 = np.float32(lr)
    for i in range(len(params)):
        a = np.float32(0.0)
        for r in sorted(grads_by_rank):
            a = np.float32(a + grads_by_rank[r][i])
        out[i] = np.float32(params[i] - np.float32(lr32 * np.float32(a / n)))
    return out


# ------------------------------------------------------------------ worker.py / runtime


def rank_seed(seed: int, rank: int, distinct: bool) -> int:
    """Seed of a rank's GradGen: the profile seed for every rank in the reference
    (worker.py:71); with ``distinct`` a splitmix-salted per-rank seed (extension)."""
    return seed if (not distinct or rank == 0) else seed ^ stream(0x5EED, rank)


def replay_params(counts: list[int], seed: int, world: int, iterations: int, lr: float,
                  distinct: bool = False) -> list[np.ndarray]:
    """Parameters after ``iterations`` synchronous P3 iterations, by direct arithmetic:
    the formula of tests/test_runtime.py:157-177 generalised to per-rank gradients.
    Slicing never changes values (each element is aggregated independently), so the
    replay runs per layer."""
    params = [np.zeros(c, dtype=np.float32) for c in counts]
    for k in range(iterations):
        for layer, c in enumerate(counts):
            grads = {r: grad_block(rank_seed(seed, r, distinct), k, layer, 0, c) for r in range(world)}
            params[layer] = shard_update(params[layer], grads, lr)
    return params


def replay_params_momentum(counts: list[int], seed: int, world: int, iterations: int, lr: float, mu: float,
                           distinct: bool = True, bf16: bool = False) -> list[np.ndarray]:
    """replay_params with heavy-ball momentum (extension; the reference has plain SGD; with
    ``bf16`` every contribution rounded to bf16 first, the declared bf16 push transport):
    g = rank-ordered fp32 sum / N; v = fp32(mu * v) + g; p = p - fp32(lr * v) — each
    operation rounded to fp32 separately, as the kernel does (no FMA)."""
    params = [np.zeros(c, dtype=np.float32) for c in counts]
    vel = [np.zeros(c, dtype=np.float32) for c in counts]
    n, lr32, mu32 = np.float32(world), np.float32(lr), np.float32(mu)
    for k in range(iterations):
        for layer, c in enumerate(counts):
            acc = np.zeros(c, dtype=np.float32)
            for r in range(world):
                gr = grad_block(rank_seed(seed, r, distinct), k, layer, 0, c)
                acc = acc + (to_bf16(gr) if bf16 else gr)
            g = acc / n
            vel[layer] = mu32 * vel[layer] + g
            params[layer] = params[layer] - lr32 * vel[layer]
    return params


def to_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 -> fp32, round to nearest even (finite inputs): the declared lossy
    transport of the B200 path (not in the reference)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def replay_params_bf16(counts: list[int], seed: int, world: int, iterations: int, lr: float,
                       distinct: bool = True) -> list[np.ndarray]:
    """replay_params with every rank's contribution rounded to bf16 before the fp32 sum."""
    params = [np.zeros(c, dtype=np.float32) for c in counts]
    for k in range(iterations):
        for layer, c in enumerate(counts):
            grads = {r: to_bf16(grad_block(rank_seed(seed, r, distinct), k, layer, 0, c)) for r in range(world)}
            params[layer] = shard_update(params[layer], grads, lr)
    return params


def digest(params: list[np.ndarray]) -> int:
    """TrainingWorker.params_digest, worker.py:372-376."""
    h = FNV_BASIS
    for v in params:
        h = fnv(v.astype("<f4").tobytes(), h)
    return h


# ------------------------------------------------------------------ queues.py


class HeapQueue:
    """FrameQueue order (queues.py:20-62): priority mode pops the minimum of
    (priority, layer, slice) with arrival as the final tie-break; FIFO pops arrivals."""

    def __init__(self, priority_mode: bool = True) -> None:
        self.priority_mode = priority_mode
        self._h: list = []
        self._n = 0

    def put_layer(self, layer: int, nslices: int) -> None:
        for s in range(nslices):
            key = (layer, layer, s) if self.priority_mode else ()
            heapq.heappush(self._h, (key, self._n, (layer, s)))
            self._n += 1

    def poll(self):
        return heapq.heappop(self._h)[2] if self._h else None

    def __len__(self) -> int:
        return len(self._h)


# Live-trace replay (the transmission-order contract of SPEC.md:435 on a recorded run).
# Trace events, in device append order: (event, iteration, layer, slice, t_ns, t0_ns) with the
# codes of include/p3.h (PUSH 0, BCAST 1, PUBLISH 2, COMPLETE 3, PICK 4).
EV_PUSH, EV_BCAST, EV_PUBLISH, EV_COMPLETE, EV_PICK = 0, 1, 2, 3, 4


def replay_live(events, nslices: list[int], priority_mode: bool = True) -> tuple[list, list]:
    """Feed one rank's recorded publish / pop interleaving of one iteration through the
    FrameQueue order: PUBLISH = put_batch of every slice of the layer (worker.py:173-182,
    queues.py:44-50; FIFO arrival = the publish sequence number), PUSH = poll (queues.py:
    52-62). Returns (expected pops, recorded pops) as (layer, slice) lists; with a single
    consumer they must be equal."""
    heap: list = []
    expect, got = [], []
    for ev, _it, layer, sl, _t, _t0 in events:
        if ev == EV_PUBLISH:
            for s in range(nslices[layer]):
                key = (layer, layer, s) if priority_mode else ()
                heapq.heappush(heap, (key, (sl, s), (layer, s)))
        elif ev == EV_PUSH:
            got.append((layer, sl))
            expect.append(heapq.heappop(heap)[2] if heap else None)
    return expect, got


def relaxation(events, avail_event: int, take_event: int, owner: int | None = None) -> int:
    """Largest number of distinct layers more urgent than a claimed slice's layer that certainly
    held an available slice at the claim: made available (avail_event record) before the
    claim's queue snapshot started (t0) and claimed (own snapshot start) after the claim
    completed (t). A strict FrameQueue consumer gives 0; C consumers popping at once give < C
    (bounded relaxation of queues.py:52-62). avail/take = PUBLISH/PUSH for one worker's
    outbox (availability per layer), COMPLETE/PICK for one server's inbox (availability per
    slice; records carry the owner as a 7th field, selected by ``owner``)."""
    avail: dict = {}
    claims = []
    for rec in events:
        ev, _it, layer, sl, t, t0 = rec[:6]
        if owner is not None and len(rec) > 6 and rec[6] != owner:
            continue
        if ev == avail_event:
            key = layer if avail_event == EV_PUBLISH else (layer, sl)
            avail[key] = min(avail.get(key, t), t)
        elif ev == take_event:
            claims.append((layer, sl, t, t0))
    worst = 0
    for layer, sl, t, t0 in claims:
        ahead = set()
        for l2, s2, t2, t02 in claims:
            if l2 >= layer or t02 <= t:
                continue
            ta = avail.get(l2) if avail_event == EV_PUBLISH else avail.get((l2, s2))
            if ta is not None and ta < t0:
                ahead.add(l2)
        worst = max(worst, len(ahead))
    return worst


# ------------------------------------------------------------------ sim.py (tick model)


def tick_uplink_sequence(fwd: list[int], bwd: list[int], nslices: list[int], slice_ticks: int,
                         iterations: int, priority: bool, pop=None, put=None) -> tuple[list[str], int]:
    """Uplink transmission order of the discrete-event model of sim.py:241-365 for the
    scenario family used by the schedule goldens: per-layer uplink cost nslices*T split
    into T-tick slices, zero update and downlink cost. Returns the uplink items
    ("up:k:Ll:ss" in start order) and the last inter-iteration delay (sim.py:181-185).

    ``put(layer, k)`` / ``pop() -> (layer, slice)`` may replace the internal queue (the
    device queue is driven through them in tests); the default is ``HeapQueue``.
    """
    L = len(fwd)
    q = HeapQueue(priority)
    put = put or (lambda l, k: q.put_layer(l, nslices[l]))
    pop = pop or q.poll
    ev: list = [(0, 0, 0, 0, 0)]  # (tick, kind, k, l, s); kinds: 0 boot, 1 fwd, 2 bwd, 3 up
    items, fwd_start, bwd_end = [], {}, {}
    bwd_ready: set = set()
    chain_ok: set = set()
    params_ok: set = set()
    started: set = set()
    remaining = {(k, l): nslices[l] for k in range(iterations) for l in range(L)}
    link_busy = False

    def start_compute(t):
        while bwd_ready:
            k, l = min(bwd_ready)
            bwd_ready.discard((k, l))
            heapq.heappush(ev, (t + bwd[l], 2, k, l, 0))
            bwd_end[(k, l)] = t + bwd[l]
            if bwd[l] > 0:
                break
        for k in range(1, iterations + 1):
            for l in range(L):
                if (k, l) in started or (k, l) not in chain_ok or (k, l) not in params_ok:
                    continue
                started.add((k, l))
                fwd_start[(k, l)] = t
                heapq.heappush(ev, (t + fwd[l], 1, k, l, 0))

    def on_event(t, kind, k, l, s):
        nonlocal link_busy
        if kind == 0:
            bwd_ready.add((0, L - 1))
        elif kind == 2:  # backward of (k, l) finished: publish its slices
            put(l, k)
            if l:
                bwd_ready.add((k, l - 1))
            else:
                chain_ok.add((k + 1, 0))
        elif kind == 1:
            if l < L - 1:
                chain_ok.add((k, l + 1))
            elif k < iterations:
                bwd_ready.add((k, L - 1))
        else:  # uplink slice delivered; update and downlink are free in this family
            link_busy = False
            remaining[(k, l)] -= 1
            if remaining[(k, l)] == 0:
                params_ok.add((k + 1, l))

    cur_k = 0
    while ev:
        t = ev[0][0]
        while ev and ev[0][0] == t:
            batch = []
            while ev and ev[0][0] == t:
                batch.append(heapq.heappop(ev))
            for e in batch:
                if e[1] == 2:
                    cur_k = e[2]
                on_event(*e)
            start_compute(t)
        if not link_busy:
            got = pop()
            if got is not None:
                l, s = got
                link_busy = True
                items.append(f"up:{cur_k}:L{l}:s{s}")
                heapq.heappush(ev, (t + slice_ticks, 3, cur_k, l, s))
    delays = []
    k = 0
    while (k, 0) in bwd_end and (k + 1, 0) in fwd_start:
        delays.append(fwd_start[(k + 1, 0)] - bwd_end[(k, 0)])
        k += 1
    return items, (delays[-1] if delays else -1)


def seq_hash(items: list[str]) -> str:
    return hashlib.sha256(" ".join(items).encode()).hexdigest()[:16]
