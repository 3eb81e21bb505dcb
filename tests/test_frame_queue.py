"""FrameQueue for host frames (queues.py:20-75 API; ordering in libp3's native heap): priority
and FIFO order with arrival tie-break, atomic batches under a racing consumer, blocking poll
with DeadlockError, close -> drain -> None, snapshot in dequeue order. CPU only."""

import random
import threading
import time

import pytest

from paper_1905_03960_b200.proto import Frame, MsgType
from paper_1905_03960_b200.queues import DeadlockError, FrameQueue, frame_order_key


def push(p, layer=0, sl=0, rank=0):
    return Frame(MsgType.PUSH, p, 0, rank, layer, sl, 0)


def test_priority_and_fifo_order():
    rng = random.Random(3)
    frames = [push(rng.randrange(5), rng.randrange(4), rng.randrange(3), i) for i in range(200)]
    q = FrameQueue(priority_mode=True)
    for f in frames:
        q.put(f)
    got = [q.poll(0.1) for _ in frames]
    # minimum key first; equal keys in arrival order (queues.py:34-38)
    assert got == sorted(frames, key=lambda f: (frame_order_key(f), frames.index(f)))
    q = FrameQueue(priority_mode=False)
    q.put_batch(frames)
    assert [q.poll(0.1) for _ in frames] == frames


def test_blocking_close_and_snapshot():
    q = FrameQueue()
    with pytest.raises(DeadlockError):
        q.poll(0.05)
    threading.Timer(0.05, lambda: q.put(push(2))).start()
    assert q.poll(2.0).priority == 2
    q.put_batch([push(5), push(1), push(3)])
    assert [f.priority for f in q.snapshot()] == [1, 3, 5]
    q.close()
    with pytest.raises(RuntimeError):
        q.put(push(0))
    assert [q.poll(0.1).priority for _ in range(3)] == [1, 3, 5]
    t0 = time.monotonic()
    assert q.poll(1.0) is None and time.monotonic() - t0 < 0.5
    assert len(q) == 0


def test_batch_atomic_under_racing_consumer():
    # a consumer never sees part of a batch: each batch lists its slices in DESCENDING order,
    # so a consumer that could see a partial batch would take a later slice of a layer before
    # an earlier one; with atomic batches the slices of every layer leave in ascending order
    q = FrameQueue()
    seen = []
    stop = threading.Event()

    def consume():
        while not stop.is_set() or len(q):
            try:
                seen.append(q.poll(0.05))
            except DeadlockError:
                pass

    t = threading.Thread(target=consume)
    t.start()
    for layer in reversed(range(50)):
        q.put_batch([push(layer, layer, s) for s in reversed(range(8))])
    stop.set()
    t.join()
    assert len(seen) == 400
    for layer in range(50):
        assert [f.slice_index for f in seen if f.layer_index == layer] == list(range(8))
