"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Run in the development container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything here calls ``p3sync`` (the reference) only; the fixtures pin both the oracle
(oracle/p3_oracle.py) and the CUDA path. The GPU box has no /root/reference, so the
tests read only the committed JSON.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
from dataclasses import replace as dataclasses_replace

import p3sync
from p3sync import hashing, plan as rplan, sim as rsim
from p3sync.model import LayerSpec, ModelProfile
from p3sync.plan import SliceKey
from p3sync.server import ShardState

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()[:16]


def real_counts() -> dict[str, list[int]]:
    from paper_1905_03960_b200.torch_models import real_counts as rc

    return {n: rc(n) for n in ("resnet50", "vgg19", "seq2seq")}


def counts_profile(name: str, counts: list[int]) -> ModelProfile:
    return ModelProfile(name, 0, tuple(LayerSpec(i, f"t{i}", c, 0, 0) for i, c in enumerate(counts)))


def main() -> None:
    out: dict = {"reference": "p3sync " + p3sync.__version__}

    # 1. GradGen golden vectors (tests/test_hashing.py:19-27) + extra blocks
    vals = [(0, 0, 0, 0), (0, 0, 0, 1), (0, 0, 1, 0), (0, 1, 0, 0), (1, 0, 0, 0), (42, 3, 2, 7),
            (2**64 - 1, 9, 17, 123456), (50, 19, 49, 59_999), (7, 2**32 - 1, 2**31, 2**40)]
    out["gradient_values"] = [[list(a), int(np.float32(hashing.gradient_value(*a)).view(np.uint32))] for a in vals]
    blocks = [(42, 0, 0, 0, 1024), (50, 3, 49, 0, 60_000), (19, 7, 16, 650_000, 65_000), (2**64 - 1, 1, 3, 1, 4099),
              (12345, 0, 0, 0, 1_000_003)]
    out["gradient_blocks"] = [[list(b), sha(hashing.gradient_block(*b).astype("<f4").tobytes())] for b in blocks]

    # 2. FNV-1a vectors (tests/test_hashing.py:79-94)
    out["fnv"] = [["", hashing.fnv1a64(b"")], ["a", hashing.fnv1a64(b"a")], ["foobar", hashing.fnv1a64(b"foobar")],
                  ["hello world", hashing.fnv1a64(b"hello world")]]
    out["splitmix_stream"] = [[s, i, hashing.splitmix64_stream(s, i)] for s, i in [(0, 0), (9, 3), (77, 5), (2**64 - 1, 10)]]

    # 3. Plans: every builtin and real profile x servers x max_slice (sha of plan_to_csv)
    reals = real_counts()
    out["real_counts"] = reals
    plans = []
    profiles = {n: p3sync.builtin_profile(n) for n in p3sync.BUILTIN_NAMES}
    profiles.update({n: counts_profile(n, c) for n, c in reals.items()})
    for name, prof in profiles.items():
        for servers in (1, 2, 3, 4, 8):
            for ms in (1_000, 10_000, 50_000, 100_000, 1_000_000):
                if name in reals and ms == 1_000 and servers not in (1, 8):
                    continue
                csv = rplan.plan_to_csv(rplan.make_p3_plan(prof, servers, ms))
                plans.append(["p3", name, servers, ms, len(rplan.make_p3_plan(prof, servers, ms).slices), sha(csv.encode())])
            for big, seed in ((1_000_000, 0), (10_000, 5)):
                csv = rplan.plan_to_csv(rplan.make_baseline_plan(prof, servers, big, seed))
                plans.append(["baseline", name, servers, big, seed, sha(csv.encode())])
    out["plans"] = plans
    # small full CSV for eyeballing
    out["plan_csv_toy3_2"] = rplan.plan_to_csv(rplan.make_p3_plan(profiles["toy3"], 2))

    # 4. aggregate_and_update through the reference ShardState (seeded inputs)
    upd = []
    for case in range(40):
        rng = np.random.RandomState(1000 + case)
        n = int(rng.randint(1, 70_000)) if case % 4 == 0 else int(rng.randint(1, 300))
        nw = int(rng.randint(1, 9))
        lr = float(rng.uniform(0.0, 1.0))
        params = rng.uniform(-5, 5, n).astype(np.float32)
        grads = {r: rng.uniform(-3, 3, n).astype(np.float32) for r in range(nw)}
        s = ShardState(SliceKey(0, 0), params.copy(), nw, lr)
        for r in range(nw):
            s.on_push(r, 0, grads[r])
        got = s.aggregate_and_update()
        upd.append([case, n, nw, lr, sha(got.astype("<f4").tobytes())])
    out["shard_updates"] = upd

    # 5. Runtime digests after 10 iterations (direct arithmetic replay, test_runtime.py:157-177,
    #    identical gradients on every rank as in the reference runtime, worker.py:71)
    def replay(prof, world, iters, lr, seeds):
        params = [np.zeros(l.param_count, dtype=np.float32) for l in prof.layers]
        for k in range(iters):
            for l in prof.layers:
                sh = ShardState(SliceKey(l.index, 0), params[l.index], world, lr, iteration=k)
                for r in range(world):
                    sh.on_push(r, k, hashing.gradient_block(seeds[r], k, l.index, 0, l.param_count))
                params[l.index] = sh.aggregate_and_update()
        h = hashing.FNV_OFFSET
        for v in params:
            h = hashing.fnv1a64(v.astype("<f4").tobytes(), h)
        return h

    def salted(seed, r):
        return seed if r == 0 else seed ^ hashing.splitmix64_stream(0x5EED, r)

    digests = []
    for name in p3sync.BUILTIN_NAMES:
        prof = profiles[name]
        for world in (1, 2, 3, 4, 8):
            digests.append([name, world, 10, 0.1, "same", f"{replay(prof, world, 10, 0.1, [prof.seed] * world):016x}"])
        for world in (2, 4, 8):
            seeds = [salted(prof.seed, r) for r in range(world)]
            digests.append([name, world, 4, 0.1, "distinct", f"{replay(prof, world, 4, 0.1, seeds):016x}"])
    # the C0 oracle config: resnet50-like, 4 workers, 20 iterations
    digests.append(["resnet50-like", 4, 20, 0.1, "same", f"{replay(profiles['resnet50-like'], 4, 20, 0.1, [50] * 4):016x}"])
    out["digests"] = digests

    # 6. Schedule goldens from the reference simulator (SURVEY §8(c) recipe)
    sched = []
    for name in ("resnet50-like", "vgg19-like", "sockeye-like"):
        prof = profiles[name]
        ns = [len(rplan.make_p3_plan(prof, 4).slices_of_layer(l.index)) for l in prof.layers]
        tick_prof = ModelProfile(name, prof.seed, tuple(
            LayerSpec(l.index, l.name, l.param_count, l.fwd_time // 100, l.bwd_time // 100) for l in prof.layers))
        for T in (30, 3):
            for policy in (rsim.PRIORITY_SLICED, rsim.AGGRESSIVE_SLICED):
                sc = rsim.Scenario(profile=tick_prof, stages=tuple(rsim.StageCost(n * T, 0, 0) for n in ns),
                                   policy=policy, slice_ticks=T, num_iterations=2)
                tl = rsim.simulate(sc)
                items = [e.item for e in sorted(tl.entries_for(rsim.UPLINK), key=lambda e: e.start)
                         if e.item.startswith("up:0:")]
                seq = " ".join(items)
                sched.append({"profile": name, "T": T, "policy": policy, "nslices": ns,
                              "fwd": [l.fwd_time for l in tick_prof.layers], "bwd": [l.bwd_time for l in tick_prof.layers],
                              "hash": hashlib.sha256(seq.encode()).hexdigest()[:16], "items": items,
                              "delay": tl.inter_iteration_delay()})
    out["schedules"] = sched

    # 7. Fig.4 / Fig.6 (tests/test_sim.py:35-136) — as tick-model scenarios
    fig4 = []
    for policy in (rsim.AGGRESSIVE_COARSE, rsim.PRIORITY_SLICED):
        sc = rsim.Scenario(profile=ModelProfile("sc", 0, tuple(LayerSpec(i, f"L{i}", 1, 1, 1) for i in range(3))),
                           stages=(rsim.StageCost(2, 0, 0),) * 3, policy=policy, slice_ticks=1, num_iterations=1)
        tl = rsim.simulate(sc)
        fig4.append({"policy": policy, "nslices": [sc.num_slices(i) for i in range(3)],
                     "items": [e.item for e in sorted(tl.entries_for(rsim.UPLINK), key=lambda e: e.start)],
                     "delay": tl.inter_iteration_delay()})
    out["fig4"] = fig4

    # 8. Full simulator timelines (sim.py) for the figure scenarios, the shipped scenario files
    #    and seeded random scenarios (every policy, serial update, per-slice overhead)
    import random

    cases = []

    def add(sc):
        tl = rsim.simulate(sc)
        cases.append({"scenario": rsim.scenario_to_dict(sc), "csv": tl.to_csv(), "summary": tl.summary()})

    for policy in (rsim.AGGRESSIVE_COARSE, rsim.AGGRESSIVE_SLICED, rsim.PRIORITY_SLICED):
        add(rsim.Scenario(profile=ModelProfile("fig4", 0, tuple(LayerSpec(i, f"L{i}", 1, 1, 1) for i in range(3))),
                          stages=(rsim.StageCost(2, 0, 0),) * 3, policy=policy, slice_ticks=1, num_iterations=1))
        add(rsim.Scenario(profile=ModelProfile("fig6", 0, tuple(LayerSpec(i, f"L{i}", 1, 0, 0) for i in range(3))),
                          stages=(rsim.StageCost(1, 1, 1), rsim.StageCost(3, 3, 3), rsim.StageCost(1, 1, 1)),
                          policy=policy, slice_ticks=1, num_iterations=1))
    for f in ("fig4.json", "fig6.json"):
        path = Path("/root/reference/pkg/scenarios") / f
        if path.exists():
            sc = rsim.load_scenario(path)
            for policy in rsim.POLICIES:
                add(dataclasses_replace(sc, policy=policy))
    rng = random.Random(1905)
    while len(cases) < 60:
        n = rng.randint(2, 7)
        T = rng.choice([1, 2, 3])
        layers, stages = [], []
        for i in range(n):
            layers.append(LayerSpec(i, f"L{i}", 1, rng.randint(0, 4), rng.randint(0, 4)))
            k = rng.randint(1, 4)
            stages.append(rsim.StageCost(k * T * rng.choice([0, 1, 1, 2]), k * rng.randint(0, 2), k * rng.randint(0, 2)))
        sc = rsim.Scenario(profile=ModelProfile("rnd", 0, tuple(layers)), stages=tuple(stages),
                           policy=rng.choice(rsim.POLICIES), slice_ticks=T, num_iterations=rng.randint(1, 3),
                           per_slice_overhead=rng.choice([0, 0, 1]), serial_update=rng.random() < 0.4)
        try:
            sc.validate()
        except rsim.ScenarioError:
            continue
        add(sc)
    out["sim_cases"] = cases
    sw = rsim.Scenario(profile=ModelProfile("sw", 0, tuple(LayerSpec(i, f"L{i}", 1, 2, 3) for i in range(4))),
                       stages=tuple(rsim.StageCost(24, 0, 24) for _ in range(4)), policy=rsim.PRIORITY_SLICED,
                       slice_ticks=1, num_iterations=2, per_slice_overhead=1)
    out["sweep"] = {"scenario": rsim.scenario_to_dict(sw), "sizes": [1, 2, 3, 4, 6, 8, 12, 24],
                    "result": rsim.sweep_slice_size(sw, [1, 2, 3, 4, 6, 8, 12, 24])}

    # wire frames (proto.py): reference encodings of random frames, and the reference's
    # verdict on malformed / truncated buffers
    from p3sync import proto as rproto
    import random as _random

    rr = _random.Random(1905)
    frames = []
    for i in range(40):
        mt = rproto.MsgType(rr.randrange(6))
        pay = b""
        if mt in (rproto.MsgType.PUSH, rproto.MsgType.BCAST):
            vals = np.array([rr.uniform(-4, 4) for _ in range(rr.randrange(0, 9))], dtype=np.float32)
            pay = rproto.pack_f32(vals)
        fr = rproto.Frame(msg_type=mt, priority=rr.randrange(2**32), iteration=rr.randrange(2**64),
                          worker_rank=rr.randrange(2**16), layer_index=rr.randrange(2**32),
                          slice_index=rr.randrange(2**32), offset=rr.randrange(2**64), payload=pay)
        frames.append({"msg_type": int(mt), "priority": fr.priority, "iteration": fr.iteration,
                       "worker_rank": fr.worker_rank, "layer_index": fr.layer_index, "slice_index": fr.slice_index,
                       "offset": fr.offset, "payload": pay.hex(), "wire": rproto.encode_frame(fr).hex()})
    bad = []
    hello = rproto.encode_frame(rproto.Frame(msg_type=rproto.MsgType.HELLO, worker_rank=3))
    push = rproto.encode_frame(rproto.Frame(msg_type=rproto.MsgType.PUSH, payload=rproto.pack_f32(np.ones(4, np.float32))))
    import struct as _struct
    cases = {
        "short_header": hello[:10], "short_payload": push[:-3], "bad_magic": b"XXXX" + hello[4:],
        "bad_type": hello[:4] + bytes([99]) + hello[5:],
        "oversize": _struct.pack("<4sBIQHIIQI", rproto.MAGIC, 0, 0, 0, 0, 0, 0, 0, rproto.DEFAULT_MAX_PAYLOAD + 4),
        "control_payload": _struct.pack("<4sBIQHIIQI", rproto.MAGIC, 2, 0, 0, 0, 0, 0, 0, 4) + b"\0" * 4,
        "two_frames": push + hello,
    }
    for name, buf in cases.items():
        try:
            fr, n = rproto.try_decode(buf)
            bad.append({"name": name, "buf": buf.hex(), "ok": fr is not None, "n": n})
        except rproto.ProtocolError as e:
            bad.append({"name": name, "buf": buf.hex(), "error": str(e)})
    out["frames"] = {"frames": frames, "decode_cases": bad}

    (HERE / "golden.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()
