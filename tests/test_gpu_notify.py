"""The baseline's NOTIFY -> PULL -> BCAST round trip on the device (server.py:227-247,
worker.py:226-239; SPEC.md:442 keeps it to reproduce the baseline's extra round trip).

In notify mode the owner updates only its own replica and NOTIFYs every other rank; each
replica queues a PULL (behind its pushes) at the owner, and the owner answers it with the
slice. Checked on emulated worlds: the parameters are the reference's (cross-mode bit
equality with P3, SPEC acceptance #3), and the trace shows, for every rank and every slice
it does not own, exactly one NOTIFY -> PULL -> answer chain in causal order."""

import pytest

import p3_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", ["vgg19-like", "resnet50-like"])
def test_notify_pull_round_trip(cuda, golden, world, name):
    from paper_1905_03960_b200 import _lib
    from paper_1905_03960_b200.model import builtin_profile
    from paper_1905_03960_b200.runtime import TrainingWorker, WorkerConfig

    prof = builtin_profile(name)
    iters = 3
    cfg = WorkerConfig(rank=0, mode="baseline", servers=world, iterations=iters, emulate_compute=True, comm_ctas=8,
                       trace_cap=100_000, rank_distinct_grads=True, big_threshold=100_000)
    w = TrainingWorker(cfg, prof, ranks=list(range(world)))
    assert w.ctx.fingerprint  # (notify mode is part of the plan fingerprint)
    w.run()
    want = O.replay_params(prof.param_counts(), prof.seed, world, iters, 0.1, distinct=True)
    for li in range(world):
        for a, b in zip(w.params(li), want):
            assert a.tobytes() == b.tobytes()
    owner = {(s.key.layer_index, s.key.slice_index): s.server for s in w.plan.slices}
    traces = {li: w.ctx.trace(li) for li in range(world)}
    for k in range(iters):
        notify, pull, answer = {}, {}, {}
        for li, tr in traces.items():
            for e in tr:
                if e.iteration != k:
                    continue
                key = (e.layer, e.slice)
                if e.event == _lib.P3_EV_NOTIFY:  # at the owner li, to rank e.rank
                    assert owner[key] == li
                    notify[(e.rank, key)] = e.t_ns
                elif e.event == _lib.P3_EV_PULL:  # at the requester li, to owner e.rank
                    assert owner[key] == e.rank
                    pull[(li, key)] = e.t_ns
                elif e.event == _lib.P3_EV_BCAST and e.rank != li:  # answer at the owner to e.rank
                    answer[(e.rank, key)] = e.t_ns
        expect = {(q, key) for key, o in owner.items() for q in range(world) if q != o}
        assert set(notify) == set(pull) == set(answer) == expect
        for x in expect:
            assert notify[x] <= pull[x] <= answer[x]
    # the forward gates opened only on answered data: every replica holds the final values (above)
    w.close()
