"""Pin the CPU oracle (oracle/p3_oracle.py) to the reference's golden vectors and to
fixtures produced by running the reference itself (tests/golden/make_golden.py)."""

import hashlib

import numpy as np
import pytest

import p3_oracle as O


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


# tests/test_hashing.py:19-27 of the reference, frozen
REF_GOLDEN = [
    ((0, 0, 0, 0), -1.0),
    ((0, 0, 0, 1), 0.402935266494751),
    ((0, 0, 1, 0), -0.1834399700164795),
    ((0, 1, 0, 0), 0.7666215896606445),
    ((1, 0, 0, 0), -0.3236668109893799),
    ((42, 3, 2, 7), 0.17637872695922852),
    ((2**64 - 1, 9, 17, 123456), -0.8298367261886597),
]


@pytest.mark.parametrize("args,expected", REF_GOLDEN)
def test_reference_gradgen_vectors(args, expected):
    assert O.grad_one(*args) == np.float32(expected)
    assert O.grad_block(args[0], args[1], args[2], args[3], 1)[0] == np.float32(expected)


def test_gradient_values_fixture(golden):
    for args, bits in golden["gradient_values"]:
        assert int(np.float32(O.grad_one(*args)).view(np.uint32)) == bits
        assert int(O.grad_block(*args, 1).view(np.uint32)[0]) == bits


def test_gradient_blocks_fixture(golden):
    for args, h in golden["gradient_blocks"]:
        assert sha(O.grad_block(*args).astype("<f4").tobytes()) == h


def test_fnv_and_splitmix(golden):
    for s, h in golden["fnv"]:
        assert O.fnv(s.encode()) == h
    assert O.fnv(b" world", O.fnv(b"hello")) == O.fnv(b"hello world")
    for seed, i, v in golden["splitmix_stream"]:
        assert O.stream(seed, i) == v
    assert O.mix(0) == 0


def test_plans_fixture(golden):
    counts = {"toy3": [1024] * 3}
    counts.update(golden["real_counts"])
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    from paper_1905_03960_b200.model import builtin_profile

    for n in ("resnet50-like", "vgg19-like", "sockeye-like"):
        counts[n] = builtin_profile(n).param_counts()
    checked = 0
    for row in golden["plans"]:
        if row[0] == "p3":
            _, name, servers, ms, nslices, h = row
            if name in golden["real_counts"] and ms == 1000:
                continue  # large; covered by the libp3 plan test
            rows = O.p3_rows(counts[name], servers, ms)
            assert len(rows) == nslices
            assert sha(O.plan_csv("p3", rows, servers, max_slice=ms).encode()) == h, row
        else:
            _, name, servers, big, seed, h = row
            rows = O.baseline_rows(counts[name], servers, big, seed)
            assert sha(O.plan_csv("baseline", rows, servers, big=big, seed=seed).encode()) == h, row
        checked += 1
    assert checked > 100


def _update_case(case):
    rng = np.random.RandomState(1000 + case)
    n = int(rng.randint(1, 70_000)) if case % 4 == 0 else int(rng.randint(1, 300))
    nw = int(rng.randint(1, 9))
    lr = float(rng.uniform(0.0, 1.0))
    params = rng.uniform(-5, 5, n).astype(np.float32)
    grads = {r: rng.uniform(-3, 3, n).astype(np.float32) for r in range(nw)}
    return n, nw, lr, params, grads


def test_shard_update_fixture(golden):
    for case, n, nw, lr, h in golden["shard_updates"]:
        n2, nw2, lr2, params, grads = _update_case(case)
        assert (n2, nw2, lr2) == (n, nw, lr)
        out = O.shard_update(params, grads, lr)
        assert sha(out.astype("<f4").tobytes()) == h
        if n < 300:
            assert O.shard_update_scalar(params, grads, lr).tobytes() == out.tobytes()


def test_server_known_answers():
    # tests/test_server.py:72-85 of the reference
    assert O.shard_update(np.array([1.0], np.float32), {0: np.array([2.0], np.float32)}, 0.5).tolist() == [0.0]
    g = {0: np.array([1.0], np.float32), 1: np.array([3.0], np.float32)}
    assert O.shard_update(np.array([0.0], np.float32), g, 1.0).tolist() == [-2.0]


@pytest.mark.parametrize("name", ["toy3", "resnet50-like", "sockeye-like"])
def test_digest_fixture(golden, name):
    from paper_1905_03960_b200.model import builtin_profile

    prof = builtin_profile(name)
    rows = [d for d in golden["digests"] if d[0] == name and d[2] <= 10]
    for _, world, iters, lr, kind, h in rows:
        if world > 4 and name != "toy3":
            continue  # keep the CPU suite short; N=8 covered on the GPU
        params = O.replay_params(prof.param_counts(), prof.seed, world, iters, lr, distinct=kind == "distinct")
        assert f"{O.digest(params):016x}" == h, (name, world, kind)


def test_schedule_fixture(golden):
    for s in golden["schedules"]:
        items, delay = O.tick_uplink_sequence(s["fwd"], s["bwd"], s["nslices"], s["T"], 2,
                                              priority=s["policy"] == "priority-sliced")
        items = [i for i in items if i.startswith("up:0:")]
        assert items == s["items"], (s["profile"], s["T"], s["policy"])
        assert O.seq_hash(items) == s["hash"]
        assert delay == s["delay"]


def test_fig4_fixture(golden):
    for f in golden["fig4"]:
        coarse = f["policy"] == "aggressive-coarse"
        items, delay = O.tick_uplink_sequence([1, 1, 1], [1, 1, 1], f["nslices"], 2 if coarse else 1, 1,
                                              priority=not coarse)
        assert items == f["items"]
        assert delay == f["delay"]


def test_heap_queue_order():
    q = O.HeapQueue(True)
    q.put_layer(2, 2)
    q.put_layer(0, 1)
    q.put_layer(1, 2)
    assert [q.poll() for _ in range(5)] == [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1)]
    f = O.HeapQueue(False)
    f.put_layer(2, 1)
    f.put_layer(0, 1)
    assert [f.poll(), f.poll(), f.poll()] == [(2, 0), (0, 0), None]


def test_bf16_rounding_matches_torch():
    # pin the oracle's RNE bf16 rounding against torch's conversion
    import torch

    rng = np.random.RandomState(0)
    x = np.concatenate([rng.uniform(-3, 3, 100_000), rng.standard_normal(10_000) * 1e-30,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 65504.0, 3.4e38])]).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert O.to_bf16(x).tobytes() == want.tobytes()


def test_replay_live_and_relaxation():
    # the live-trace checkers used by tests/test_gpu_live_order.py, on hand-made traces:
    # PUBLISH = put_batch of a layer, PUSH = poll (queues.py:44-62)
    P, U = O.EV_PUBLISH, O.EV_PUSH
    nsl = [2, 1, 3]
    ev = [(P, 0, 2, 0, 10, 0), (U, 0, 2, 0, 11, 10), (P, 0, 0, 1, 12, 0), (U, 0, 0, 0, 13, 12),
          (U, 0, 0, 1, 14, 13), (P, 0, 1, 2, 15, 0), (U, 0, 1, 0, 16, 15), (U, 0, 2, 1, 17, 16),
          (U, 0, 2, 2, 18, 17)]
    expect, got = O.replay_live(ev, nsl, priority_mode=True)
    assert got == expect
    assert O.relaxation(ev, P, U) == 0
    # a pop that passes over a layer published before its snapshot and popped after it
    bad = [(P, 0, 2, 0, 10, 0), (P, 0, 0, 1, 11, 0), (U, 0, 2, 0, 20, 12), (U, 0, 0, 0, 22, 21),
           (U, 0, 0, 1, 23, 22), (U, 0, 2, 1, 24, 23), (U, 0, 2, 2, 25, 24)]
    e2, g2 = O.replay_live(bad, nsl, priority_mode=True)
    assert g2 != e2 and e2[0] == (0, 0)
    assert O.relaxation(bad, P, U) == 1
    # FIFO: arrival = publish sequence (slice field of PUBLISH)
    fifo = [(P, 0, 2, 0, 10, 0), (P, 0, 0, 1, 11, 0), (U, 0, 2, 0, 12, 11), (U, 0, 2, 1, 13, 12),
            (U, 0, 2, 2, 14, 13), (U, 0, 0, 0, 15, 14), (U, 0, 0, 1, 16, 15)]
    e3, g3 = O.replay_live(fifo, nsl, priority_mode=False)
    assert g3 == e3
    # server inbox: COMPLETE / PICK per slice, filtered by owner
    C, K = O.EV_COMPLETE, O.EV_PICK
    srv = [(C, 0, 1, 0, 5, 0, 0), (C, 0, 0, 0, 6, 0, 0), (K, 0, 1, 0, 9, 7, 0), (K, 0, 0, 0, 12, 10, 0),
           (C, 0, 0, 1, 6, 0, 1), (K, 0, 2, 0, 3, 1, 1)]
    assert O.relaxation(srv, C, K, owner=0) == 1
    assert O.relaxation(srv, C, K, owner=1) == 0
