"""Single-rank FINISH as one streaming update (k_update_stream): with every layer published
and no other consumer, tiles of the priority-ordered element space go to the CTAs
round-robin, cut at layer and slice ends; a slice is complete when all its elements are.
Bit-exact against the oracle's ShardState replay (server.py:55-68) with words written
directly (sync-only phase) or through the publication ring (training: no DRAIN launch at
N=1), odd slice sizes, momentum, the declared bf16 push; every slice popped and completed
once per iteration; and the slice-pop comm kernel (P3_STREAM=0) gives the same values."""

import os

import pytest

import p3_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["1", "0"], ids=["stream", "slice_pops"])
def _stream(request, monkeypatch):
    monkeypatch.setenv("P3_STREAM", request.param)  # read by p3_ctx_create

COUNTS = [5, 1023, 70_001, 9, 200_000, 64, 64, 2_359_296, 1000, 2_048_000]


@pytest.mark.parametrize("max_slice", [7, 1000, 50_000, 333_333])
@pytest.mark.parametrize("ring", [False, True])
def test_single_rank_finish_matches_oracle(cuda, max_slice, ring):
    import torch

    from paper_1905_03960_b200 import _lib
    from paper_1905_03960_b200.runtime import SyncContext

    counts = COUNTS if max_slice >= 1000 else COUNTS[:6]
    seed, lr, iters = 77, 0.3, 3
    ctx = SyncContext(counts, 1, [0], max_slice=max_slice, lr=lr, comm_ctas=148, finish_ctas=148, emulate_grads=True,
                      drain_bytes=1 << 62, pub_batch_bytes=1 << 62, trace_cap=400_000, timeout_s=30.0)
    st = torch.cuda.Stream()
    nsl = [-(-c // max_slice) for c in counts]
    for k in range(iters):
        for l in range(len(counts)):
            ctx.gradgen_layer(0, seed, k, l, st)
        if not ring:  # sync-only phase: words written before the iteration opens
            for l in range(len(counts)):
                ctx.layer_ready(0, l, k, None, st)
            st.synchronize()
        ctx.iteration_begin(k, st)
        if ring:  # training: the hooks publish through the ring during the open iteration
            for l in reversed(range(len(counts))):
                ctx.layer_ready(0, l, k, None, st)
        n0 = ctx.launches()
        ctx.iteration_end(k)
        assert ctx.launches() == n0 + 1
        ctx.sync_all(k + 1)
    st.synchronize()
    want = O.replay_params(counts, seed, 1, iters, lr)
    for a, b in zip(ctx.params_numpy(0), want):
        assert a.tobytes() == b.tobytes()
    tr = ctx.trace(0)
    for k in range(iters):
        pops = [(e.layer, e.slice) for e in tr if e.iteration == k and e.event == _lib.P3_EV_PUSH]
        done = [(e.layer, e.slice) for e in tr if e.iteration == k and e.event == _lib.P3_EV_BCAST]
        every = [(l, s) for l in range(len(counts)) for s in range(nsl[l])]
        assert sorted(pops) == every and sorted(done) == every
    ctx.close()


def test_single_rank_finish_momentum(cuda):
    import torch

    from paper_1905_03960_b200.runtime import SyncContext

    counts = COUNTS
    seed, lr, mu, iters = 5, 0.05, 0.9, 3
    ctx = SyncContext(counts, 1, [0], lr=lr, momentum=mu, comm_ctas=148, finish_ctas=148, emulate_grads=True,
                      drain_bytes=1 << 62, timeout_s=30.0)
    st = torch.cuda.Stream()
    for k in range(iters):
        for l in range(len(counts)):
            ctx.gradgen_layer(0, seed, k, l, st)
            ctx.layer_ready(0, l, k, None, st)
        st.synchronize()
        ctx.iteration_begin(k, st)
        ctx.iteration_end(k)
        ctx.sync_all(k + 1)
    want = O.replay_params_momentum(counts, seed, 1, iters, lr, mu, distinct=False)
    for a, b in zip(ctx.params_numpy(0), want):
        assert a.tobytes() == b.tobytes()
    ctx.close()


def test_single_rank_finish_bf16_push(cuda):
    # declared bf16 push at N=1: the own contribution rounded to bf16 before the update
    import torch

    from paper_1905_03960_b200.runtime import SyncContext

    counts = COUNTS[:8]
    seed, lr, iters = 9, 0.25, 2
    ctx = SyncContext(counts, 1, [0], lr=lr, comm_ctas=148, finish_ctas=148, emulate_grads=True,
                      drain_bytes=1 << 62, timeout_s=30.0, push_dtype="bf16")
    st = torch.cuda.Stream()
    for k in range(iters):
        for l in range(len(counts)):
            ctx.gradgen_layer(0, seed, k, l, st)
            ctx.layer_ready(0, l, k, None, st)
        st.synchronize()
        ctx.iteration_begin(k, st)
        ctx.iteration_end(k)
        ctx.sync_all(k + 1)
    want = O.replay_params_bf16(counts, seed, 1, iters, lr, distinct=False)
    for a, b in zip(ctx.params_numpy(0), want):
        assert a.tobytes() == b.tobytes()
    ctx.close()
