"""The reference's bench outputs and summary (cli.py:241-398) from an emulated world on one
GPU; SPEC acceptance #4 (throttled P3 >= 1.05x the baseline and a lower idle fraction); the
reference worker's public entry points (enqueue_layer, on_bcast, the plan/mode check)."""

import json

import numpy as np
import pytest

import p3_oracle as O

pytestmark = pytest.mark.gpu


def test_bench_outputs_and_summary(cuda, tmp_path, golden):
    from paper_1905_03960_b200.bench_run import RunConfig, run_bench

    cfg = RunConfig(mode="p3", profile="resnet50-like", num_workers=4, iterations=20, skip_iterations=5,
                    output_dir=str(tmp_path))
    summary = run_bench(cfg)
    # BASELINE configs[0] (C0): the reference's digest of this exact run
    assert summary["digest"] == "720d9a1a5872f34c"
    assert set(summary) == {"mode", "profile", "num_workers", "num_servers", "iterations", "batch_size",
                            "skip_iterations", "idle_threshold", "samples_per_second", "idle_fraction", "digest",
                            "server_slices_verified"}
    assert summary["server_slices_verified"] == 51  # every slice of resnet50-like, once
    assert json.loads((tmp_path / "summary.json").read_text()) == summary
    # compute floor: 90.5 ms of emulated fwd+bwd per iteration -> at most 4*32/0.0905 samples/s
    assert 0.5 * 4 * 32 / 0.0905 < summary["samples_per_second"] <= 4 * 32 / 0.0905 * 1.01
    assert 0.0 <= summary["idle_fraction"] <= 1.0
    rows = (tmp_path / "throughput_worker0.csv").read_text().splitlines()
    assert rows[0] == "iteration,wall_ms,start_ms" and len(rows) == 21
    util = (tmp_path / "net_util_worker1.csv").read_text().splitlines()
    last = [int(x) for x in util[-1].split(",")]
    # link bytes of rank 1: pushes of slices it does not own + broadcasts of the ones it owns
    from paper_1905_03960_b200.model import builtin_profile
    from paper_1905_03960_b200.plan import make_p3_plan

    plan = make_p3_plan(builtin_profile("resnet50-like"), 4)
    out = 20 * 4 * (sum(s.length for s in plan.slices if s.server != 1) +
                    3 * sum(s.length for s in plan.slices if s.server == 1))
    assert last[2] == out


def test_server_digest_mismatch_is_reported(cuda, tmp_path):
    from paper_1905_03960_b200.bench_run import RunConfig, run_bench, summarize_run
    from paper_1905_03960_b200.model import builtin_profile
    from paper_1905_03960_b200.proto import ProtocolError

    cfg = RunConfig(profile="toy3", num_workers=2, iterations=6, output_dir=str(tmp_path))
    run_bench(cfg)
    dump = tmp_path / "params_worker0.bin"
    b = bytearray(dump.read_bytes())
    b[5] ^= 1
    dump.write_bytes(bytes(b))
    with pytest.raises(ProtocolError):
        summarize_run(cfg, tmp_path, builtin_profile("toy3"))


def test_throttled_p3_beats_baseline_with_less_idle(cuda, tmp_path):
    """SPEC.md:678 acceptance #4: vgg19-like, 2 workers, token-bucket throttle with
    communication ~2x the emulated compute, >= 30 measured iterations: P3 throughput >= 1.05x
    the baseline's (KVStore placement, FIFO) and P3 idle fraction < the baseline's. The same
    run must also give the same parameters in both modes (acceptance #3)."""
    from paper_1905_03960_b200.bench_run import RunConfig, run_bench

    res = {}
    for mode in ("p3", "baseline"):
        cfg = RunConfig(mode=mode, profile="vgg19-like", num_workers=2, iterations=35, skip_iterations=5,
                        throttle_rate=300e6, comm_ctas=4, output_dir=str(tmp_path / mode))
        res[mode] = run_bench(cfg)
    p3, base = res["p3"], res["baseline"]
    print("ACCEPTANCE4", json.dumps({"p3": p3, "baseline": base, "ratio": p3["samples_per_second"] / base["samples_per_second"]}))
    assert p3["digest"] == base["digest"]
    assert p3["samples_per_second"] >= 1.05 * base["samples_per_second"]
    assert p3["idle_fraction"] < base["idle_fraction"]


def test_worker_entry_points(cuda):
    import torch

    from paper_1905_03960_b200.model import builtin_profile
    from paper_1905_03960_b200.plan import PlanError, make_baseline_plan, make_p3_plan
    from paper_1905_03960_b200.proto import Frame, MsgType, ProtocolError
    from paper_1905_03960_b200.runtime import TrainingWorker, WorkerConfig

    prof = builtin_profile("vgg19-like")
    cfg = WorkerConfig(0, "p3", [("gpu", 0), ("gpu", 1)], 2, emulate_compute=False, comm_ctas=4)
    assert cfg.world == 2
    with pytest.raises(ValueError):  # worker.py:65-67
        TrainingWorker(cfg, prof, make_baseline_plan(prof, 2))
    with pytest.raises(PlanError):  # a plan the device would not run
        TrainingWorker(WorkerConfig(0, "p3", 2, 2), prof, make_p3_plan(prof, 3))
    # a plan with a different slice size is adopted (the device builds the same one)
    w = TrainingWorker(WorkerConfig(0, "p3", 1, 1, emulate_compute=False), prof, make_p3_plan(prof, 1, 20_000))
    assert w.cfg.max_slice == 20_000 and len(w.plan.slices) == len(make_p3_plan(prof, 1, 20_000).slices)
    # on_bcast: a host BCAST frame lands in the replica and opens the layer's gate
    layer = 16  # 5 slices of 20K
    sl = w.plan.slices_of_layer(layer)
    rng = np.random.default_rng(0)
    vals = [rng.standard_normal(s.length).astype(np.float32) for s in sl]
    frames = [Frame(MsgType.BCAST, s.priority, 0, 0, layer, s.key.slice_index, s.offset, v.tobytes())
              for s, v in zip(sl, vals)]
    with pytest.raises(ProtocolError):
        w.on_bcast(Frame(MsgType.BCAST, layer, 1, 0, layer, 0, 0, vals[0].tobytes()))  # wrong iteration
    with pytest.raises(ProtocolError):
        w.on_bcast(Frame(MsgType.BCAST, layer, 0, 0, layer, 0, 0, vals[0][:-1].tobytes()))  # length
    for f in frames[:-1]:
        w.on_bcast(f)
    with pytest.raises(ProtocolError):
        w.on_bcast(frames[0])  # duplicate
    assert w.flag(layer) == 0
    w.on_bcast(frames[-1])
    torch.cuda.synchronize()
    assert w.flag(layer) == 1
    assert np.array_equal(w.params()[layer], np.concatenate(vals))
    w.close()
    # enqueue_layer drives one iteration by hand (the run_iteration loop, worker.py:312-325)
    w = TrainingWorker(WorkerConfig(0, "p3", 1, 1, emulate_compute=False, comm_ctas=4), prof)
    w.ctx.iteration_begin(0, w.comm_stream)
    for layer in reversed(range(prof.num_layers)):
        w.enqueue_layer(layer, 0)
    w.ctx.iteration_end(0)
    w.wait_all(1)
    want = O.replay_params(prof.param_counts(), prof.seed, 1, 1, 0.1)
    for a, b in zip(w.params(), want):
        assert a.tobytes() == b.tobytes()
    w.close()
