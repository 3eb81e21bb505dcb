#!/usr/bin/env python
"""Benchmark of the P3 sync path on B200 (BASELINE.json metric: samples/s of P3 vs
layer-wise sync; slice-sync GB/s; roofline fraction).

One step = one data-parallel training iteration of the named model on synthetic input:
forward (each layer gated on its synced parameters), backward (each layer's gradient
published by a hook), and the sliced, priority-scheduled reduce + SGD + broadcast done by
the persistent comm kernel, overlapped with compute. Launch:

    python bench.py [--gpus 1] [--steps K] [--warmup W]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N
    python bench.py --impl reference   # the reference P3 path on host cores (oracle port)

Rank 0 prints ONE JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "samples/sec P3 vs layer-wise sync at 1/2/4/8 B200; slice-sync NVLink GB/s"  # BASELINE.json metric
DEFAULT_BATCH = {"resnet50": 256, "vgg19": 128, "seq2seq": 128}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", choices=["resnet50", "vgg19", "seq2seq"], default="resnet50")
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (default per model)")
    ap.add_argument("--max-slice", type=int, default=50_000)
    ap.add_argument("--comm-ctas", type=int, default=8)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--skip-layerwise", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-sync", action="store_true")
    ap.add_argument("--sync-reps", type=int, default=10)
    ap.add_argument("--throttle-gbps", type=float, default=10.0,
                    help="emulated per-GPU egress for the P3 vs layer-wise comparison on the same kernels "
                         "(N>1 only; 0 skips it)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers


class ClockSampler:
    FIELDS = ("clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int) -> None:
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(device_index), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 2 + i and r[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


class NvlinkCounters:
    """NVLink data bytes sent / received by this GPU (NVML field values THROUGHPUT_DATA_TX/RX,
    KiB, summed over the links), read around a measured phase: the traffic of the transfers."""

    FIELDS = (138, 139)  # NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (KiB)

    def __init__(self, device_index: int) -> None:
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.links = [l for l in range(18) if self._link_up(l)]
            self.ok = bool(self.links)
        except Exception:  # noqa: BLE001 - no NVML / no NVLink: traffic stays null
            self.ok = False

    def _link_up(self, link: int) -> bool:
        try:
            return bool(self._nvml.nvmlDeviceGetNvLinkState(self.h, link))
        except Exception:  # noqa: BLE001
            return False

    def read(self) -> tuple[int, int] | None:
        if not self.ok:
            return None
        ids = [(f, l) for f in self.FIELDS for l in self.links]
        vals = self._nvml.nvmlDeviceGetFieldValues(self.h, ids)
        tot = [0, 0]
        for (f, _), v in zip(ids, vals):
            if v.nvmlReturn == 0:
                tot[self.FIELDS.index(f)] += int(v.value.ullVal)
        return tot[0] * 1024, tot[1] * 1024


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # (gloo: the CPU tests of these helpers)
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int) -> None:
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def build(args, rank):
    import torch

    from paper_1905_03960_b200.torch_models import build_model

    torch.manual_seed(1234)
    m = build_model(args.model).cuda()
    if args.model in ("resnet50", "vgg19"):
        m = m.to(memory_format=torch.channels_last)
    return m


def time_training(args, world, rank, ddp, x, y, steps, warmup, e2e=None):
    """Device time of `steps` training steps (max over ranks), after `warmup` steps."""
    import torch

    from paper_1905_03960_b200.torch_models import loss_fn

    from paper_1905_03960_b200.loader import DevicePrefetcher

    feed = None

    def step(i):
        if e2e is None:
            loss = loss_fn(args.model, ddp, x, y)
            loss.backward()
            return loss
        xd, yd = next(feed)  # pinned host batch, copied in on the copy stream
        loss = loss_fn(args.model, ddp, xd, yd)
        loss.backward()
        lh[i % len(lh)].copy_(loss.detach(), non_blocking=True)
        return loss

    if e2e is not None:
        xh, yh, lh = e2e
        feed = DevicePrefetcher([(xh, yh)] * warmup)
    for i in range(warmup):
        step(i)
    ddp.synchronize()
    barrier(world)
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    if e2e is not None:  # every timed step's input copy is issued inside the timed region
        feed = DevicePrefetcher([(xh, yh)] * steps)
    for i in range(steps):
        step(i)
    ddp.synchronize()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    ck = clocks.stop() if clocks else None
    return max_over_ranks(ms, world), ck


# ----------------------------------------------------------------------------- arms


def sync_only_roofline(args, world, rank, counts):
    """Slice-sync kernel alone: every layer's gradient already in HBM and published, the
    comm kernel (K3 + K4) launched over the whole GPU. Returns per-launch device ms."""
    import torch

    from paper_1905_03960_b200 import _lib
    from paper_1905_03960_b200.runtime import SyncContext, connect

    props = torch.cuda.get_device_properties(0)
    ctas = props.multi_processor_count  # one 512-thread comm CTA per SM (126 registers)
    ctx = SyncContext(counts, world, [rank], max_slice=args.max_slice, lr=args.lr, comm_ctas=ctas,
                      comm_threads=512, timeout_s=60.0, emulate_grads=True)
    connect(ctx)
    stream = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    # a read sweep of another buffer after the flush write retires the flush's dirty lines
    # before the timed region (else their write-back lands inside the kernel: ~60 MB of extra
    # DRAM writes, ~8 us at N=1 — tools/stream_gap.py under ncu --cache-control none)
    sweep = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
    align = torch.zeros(1, device="cuda")
    for l in range(len(counts)):
        ctx.gradgen_layer(0, 7, 0, l, stream)
    stream.synchronize()
    times = []
    reps = args.sync_reps
    nvl = NvlinkCounters(torch.cuda.current_device()) if world > 1 else None
    nvl0 = dev0 = None
    for k in range(reps + 2):
        if k == 2 and nvl is not None:
            torch.cuda.synchronize()
            nvl0 = nvl.read()
            dev0 = ctx.counters(0)
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
            sweep.sum(dtype=torch.int32)
        for l in range(len(counts)):  # published before the iteration opens: no DRAIN launches
            ctx.layer_ready(0, l, k, None, stream)
        stream.synchronize()
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(200_000)  # ~0.1 ms: the host enqueues the launch before the GPU gets there
            if world > 1:  # align the ranks on the device: a late peer is not this kernel's time
                import torch.distributed as dist

                dist.all_reduce(align)
        ctx.iteration_begin(k, stream)  # per-iteration counter reset (memset) — not the kernel
        s.record(stream)
        ctx.iteration_end(k)  # one FINISH launch does the whole iteration
        e.record(stream)
        ctx.sync_all(k + 1, 60.0)
        stream.synchronize()
        if k >= 2:
            times.append(max_over_ranks(s.elapsed_time(e), world))
    traffic = None
    if dev0 is not None:
        nvl1, dev1 = nvl.read(), ctx.counters(0)
        traffic = {"device_counted_out_bytes_per_launch": (dev1[1] - dev0[1]) / reps,
                   "device_counted_in_bytes_per_launch": (dev1[0] - dev0[0]) / reps,
                   "device_counted": "the comm kernel's own byte counters (p3_counters: payload it stored over "
                                     "NVLink / received), per timed launch"}
        if nvl1 is not None and nvl0 is not None and nvl1[0] > nvl0[0]:
            traffic.update({"nvlink_tx_bytes_per_launch": (nvl1[0] - nvl0[0]) / reps,
                            "nvlink_rx_bytes_per_launch": (nvl1[1] - nvl0[1]) / reps})
        else:  # NVML returns NOT_SUPPORTED for every NVLink counter field on this pool
            traffic["nvlink_hw_counters"] = ("unavailable: NVML NVLink throughput/count fields return NOT_SUPPORTED "
                                             "here (profiles/r02/nvml_nvlink_probe.txt); ncu cannot replay a "
                                             "cross-rank kernel")
    ctx.close()
    return statistics.mean(times), ctas, traffic


def training_sync_profile(args, world, rank, x, y, steps=4, warmup=3):
    """The comm kernel inside training, from its device trace (a traced P3DataParallel run of
    `steps` steps): per iteration, the bytes this rank moved over its link and when — how much
    of the sync overlapped the backward pass (before the last publication) and the exposed
    tail after it, with that tail's throughput (the FINISH phase of the shipped launch policy)."""
    import torch

    from paper_1905_03960_b200 import _lib
    from paper_1905_03960_b200.ddp import P3DataParallel
    from paper_1905_03960_b200.torch_models import loss_fn

    model = build(args, rank)
    P = sum(p.numel() for p in model.parameters())
    d = P3DataParallel(model, lr=args.lr, max_slice=args.max_slice, comm_ctas=args.comm_ctas,
                       trace_cap=(steps + warmup + 1) * 8 * (P // args.max_slice + 400))
    for _ in range(warmup + steps):
        loss_fn(args.model, d, x, y).backward()
    d.synchronize()
    torch.cuda.synchronize()
    tr = d.ctx.trace(0)
    plan_counts = d.ctx.layer_counts
    from paper_1905_03960_b200.model import LayerSpec, ModelProfile
    from paper_1905_03960_b200.plan import make_p3_plan

    plan = make_p3_plan(ModelProfile("m", 0, tuple(LayerSpec(i, "t", c, 0, 0) for i, c in enumerate(plan_counts))),
                        world, args.max_slice)
    rows = []
    for k in range(warmup, warmup + steps):
        ev = [e for e in tr if e.iteration == k]
        pubs = [e.t_ns for e in ev if e.event == _lib.P3_EV_PUBLISH]
        moves = [e for e in ev if e.event in (_lib.P3_EV_PUSH, _lib.P3_EV_BCAST)]
        if not pubs or not moves:
            continue
        t_last = max(pubs)
        # N > 1: this rank's NVLink egress — pushes of slices it does not own + (N-1) broadcast
        # copies of owned ones; N = 1: the update's HBM bytes (read g, read p, write p)
        own = {(s.key.layer_index, s.key.slice_index): s for s in plan.slices}
        egress_before = egress_after = 0
        for e in moves:
            sl = own[(e.layer, e.slice)]
            if world == 1:
                nb = 12 * sl.length if e.event == _lib.P3_EV_BCAST else 0
            elif e.event == _lib.P3_EV_PUSH and sl.server != rank:
                nb = 4 * sl.length
            elif e.event == _lib.P3_EV_BCAST:
                nb = 4 * sl.length * (world - 1)
            else:
                continue
            if e.t_ns <= t_last:
                egress_before += nb
            else:
                egress_after += nb
        t_end = max(e.t_ns for e in moves)
        rows.append((egress_before, egress_after, (t_end - t_last) / 1e6))
    d.close()
    if not rows:
        return None
    eb = statistics.mean(r[0] for r in rows)
    ea = statistics.mean(r[1] for r in rows)
    tail_ms = statistics.mean(r[2] for r in rows)
    return {
        "bytes_per_iteration": eb + ea,
        "bytes": "NVLink egress of this rank" if world > 1 else "HBM bytes of the update (12 B/param)",
        "overlapped_fraction": eb / (eb + ea) if eb + ea else None,
        "exposed_tail_ms": tail_ms,
        "tail_GBps": ea / (tail_ms * 1e-3) / 1e9 if tail_ms > 0 and ea else None,
        "steps": len(rows),
        "how": "device trace of a P3DataParallel training run: PUBLISH / PUSH / BCAST records on %globaltimer; "
               "egress = pushes of slices owned elsewhere + (N-1) broadcast copies of owned slices",
    }


def cpu_reference(counts, world, batch, steps, warmup, seconds_budget=20.0):
    """The reference's P3 sync iteration on host cores, bounded sample: the reference's own
    code from baseline/_ref (kind "reference": FrameQueue, GradGen, ShardState) when it is
    installed, else the numpy restatement (kind "port")."""
    sys.path.insert(0, str(REPO / "oracle"))
    import ref_p3
    from cpu_p3 import CpuP3

    kind = "reference" if ref_p3.available() else "port"
    cpu = ref_p3.RefP3(counts, world) if kind == "reference" else CpuP3(counts, world)
    n_slices = len(cpu.rows)
    dt, frac = cpu.time_iteration(0, sample_slices=min(n_slices, 32))  # calibrate
    per_iter = dt / frac
    sample = n_slices if per_iter * max(steps, 1) < seconds_budget else max(8, int(n_slices * seconds_budget / (per_iter * max(steps, 1))))
    sample = min(sample, n_slices)
    for k in range(warmup):
        cpu.time_iteration(1 + k, sample_slices=min(sample, 16))
    tot, cov = 0.0, 0.0
    for k in range(steps):
        dt, frac = cpu.time_iteration(100 + k, sample_slices=sample)
        tot += dt
        cov += frac
    iter_s = tot / cov  # seconds per full iteration
    cpu.close()
    return {
        "value": batch * world / iter_s,
        "unit": "samples/sec",
        "cores": cpu.threads,
        "kind": kind,
        "sample": f"{sample} of {n_slices} slices per step (priority pop order), {steps} steps, scaled to a full "
                  f"iteration; sync path only (GradGen materialise + rank-ordered aggregate + SGD + replica apply), "
                  f"compute excluded; " + ("the reference's own p3sync objects (baseline/_ref)" if kind == "reference"
                                           else "numpy restatement (oracle/cpu_p3.py)") +
                  f"; {cpu.threads} threads of nproc {os.cpu_count()}",
        "seconds_per_iteration": iter_s,
    }


def run_reference(args):
    from paper_1905_03960_b200.torch_models import real_counts

    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    batch = args.batch or DEFAULT_BATCH[args.model]
    counts = real_counts(args.model)
    cb = cpu_reference(counts, world, batch, args.steps, args.warmup)
    ms = 1000.0 * batch * world / cb["value"]
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "samples/sec", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (GradGen gradients)",
        "config": {"workload": f"{args.model} P3 sync path, {world} ranks, {args.max_slice}-param slices",
                   "global_batch": batch * world, "max_slice": args.max_slice},
        "note": "the reference computes no model (its compute is emulated by sleeps, worker.py:299-310): this is its "
                "sync path per iteration at the model's shapes, converted with the training batch; compare it with "
                "our line's sync_path (same work on the GPU), not with the training value",
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "samples/sec", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ours(args):
    import torch

    from paper_1905_03960_b200 import _lib
    from paper_1905_03960_b200.ddp import LayerwiseDataParallel, P3DataParallel
    from paper_1905_03960_b200.torch_models import real_counts, synthetic_batch

    world, rank, local = dist_setup(args)
    batch = args.batch or DEFAULT_BATCH[args.model]
    counts = real_counts(args.model)
    P = sum(counts)
    torch.backends.cudnn.benchmark = False

    # --- process warm-up (cuDNN/cuBLAS handles, autotuning caches, clocks) before any timing
    from paper_1905_03960_b200.torch_models import loss_fn

    x, y = synthetic_batch(args.model, batch, seed=1234 + rank)
    model = build(args, rank)
    for _ in range(3):
        loss_fn(args.model, model, x, y).backward()
    torch.cuda.synchronize()
    del model

    # --- P3: device-resident inputs
    model = build(args, rank)
    ddp = P3DataParallel(model, lr=args.lr, max_slice=args.max_slice, comm_ctas=args.comm_ctas)
    launches0 = ddp.launches()
    ms, clocks = time_training(args, world, rank, ddp, x, y, args.steps, args.warmup)
    value = args.steps * batch * world / (ms / 1000.0)
    # comm kernel launches (DRAIN per layer + FINISH per iteration) of the timed steps
    gpu_launches = (ddp.launches() - launches0) * args.steps // (args.steps + args.warmup)

    # --- e2e through the public API: pinned host batch copied in, loss copied out, every step
    e2e_value, h2d = None, 0
    if not args.skip_e2e:
        xh, yh = synthetic_batch(args.model, batch, seed=1234 + rank, pinned_host=True)
        lh = [torch.empty((), dtype=torch.float32).pin_memory() for _ in range(args.steps)]
        ms_e2e, _ = time_training(args, world, rank, ddp, None, None, args.steps, 1, e2e=(xh, yh, lh))
        e2e_value = args.steps * batch * world / (ms_e2e / 1000.0)
        h2d = xh.numel() * xh.element_size() + yh.numel() * yh.element_size()
    ddp.close()
    del ddp, model
    torch.cuda.empty_cache()

    # --- layer-wise baseline (NCCL all-reduce per tensor, FIFO) on the same box
    layerwise = None
    if not args.skip_layerwise:
        model = build(args, rank)
        lw = LayerwiseDataParallel(model, lr=args.lr)
        ms_lw, _ = time_training(args, world, rank, lw, x, y, args.steps, args.warmup)
        layerwise = {"value": args.steps * batch * world / (ms_lw / 1000.0), "ms_per_step": ms_lw / args.steps,
                     "impl": "per-tensor NCCL all_reduce in backward-hook order + SGD" if world > 1 else
                             "SGD only (no communication at N=1)"}
        lw.close()
        del lw, model
        torch.cuda.empty_cache()

    # --- the paper's experiment: emulated slow links (K7 token bucket, SPEC/PAPER tc shaping),
    #     P3 (50K slices, priority) vs aggressive layer-wise sync (KVStore placement, FIFO) on the
    #     same comm kernel, same gates, same fused SGD
    throttled = None
    if world > 1 and args.throttle_gbps > 0:
        throttled = {"gbps": args.throttle_gbps, "burst_bytes": 50 * 1024}
        for arm, kw in (("p3", {}), ("layerwise_fifo", {"plan_mode": "baseline", "priority_mode": False}),
                        ("p3_bf16_push", {"push_dtype": "bf16"}), ("p3_bf16_params", {})):
            model = build(args, rank)
            if arm == "p3_bf16_params":  # bf16 parameters: bf16 replicas on the wire, fp32 masters
                model = model.bfloat16()
            d = P3DataParallel(model, lr=args.lr, max_slice=args.max_slice, comm_ctas=4, pub_batch_bytes=0,
                               throttle_bps=args.throttle_gbps * 1e9, **kw)
            ms_t, _ = time_training(args, world, rank, d, x, y, max(5, args.steps), 3)
            throttled[arm] = max(5, args.steps) * batch * world / (ms_t / 1000.0)
            d.close()
            del d, model
            torch.cuda.empty_cache()
        throttled["p3_vs_layerwise"] = throttled["p3"] / throttled["layerwise_fifo"]

    # --- the comm kernel inside training (device trace): overlap and exposed tail
    # (N>1 only: at N=1 the whole update is one FINISH launch after the backward pass)
    train_sync = training_sync_profile(args, world, rank, x, y) if world > 1 and not args.skip_sync else None
    torch.cuda.empty_cache()

    # --- slice-sync kernel roofline
    sync_ms, ctas, nvl_traffic = (sync_only_roofline(args, world, rank, counts) if not args.skip_sync
                                  else (float("nan"), 0, None))
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
    if world == 1:
        alg = 12 * P  # read G + read W + write W per element (SURVEY §8(d), K4 with N=1)
        peak = peaks.get("hbm_gbs", 6650.0)
        roof = {"bound": "hbm", "achieved": alg / (sync_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}
    else:
        alg = 2 * (world - 1) / world * P * 4  # NVLink egress per GPU: pushes + broadcasts
        peak = 770.0
        roof = {"bound": "nvlink", "achieved": alg / (sync_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"}
    # DRAM bytes per launch of the same kernel configuration from the committed ncu --set full
    # capture (profiles/ncu_traffic.json), when one exists for this model and world size
    traffic = None
    tf = REPO / "profiles" / "ncu_traffic.json"
    if tf.exists() and world == 1:
        t = json.loads(tf.read_text()).get(args.model)
        if t and t["world"] == world and t["max_slice"] == args.max_slice:
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    if world > 1 and nvl_traffic is not None:  # hardware NVLink bytes when NVML has them, else null
        traffic = nvl_traffic.get("nvlink_tx_bytes_per_launch")
        roof["traffic_detail"] = nvl_traffic
    roof.update({"frac": roof["achieved"] / peak, "traffic": traffic,
                 "kernel": ("k_update_stream (single-rank FINISH: the fused SGD update of every slice in "
                            "priority order, one streaming pass)" if world == 1 and os.environ.get("P3_STREAM", "1") != "0"
                            else "k_comm (K3 push + K4 reduce/SGD/bcast)"),
                 "algorithmic_bytes_per_launch": alg, "launch_ms": sync_ms, "ctas": ctas,
                 "measured_in": "sync-only phase: all layers' gradients in HBM and published, one launch per "
                                "iteration over the whole GPU, L2 flushed between launches (256 MB write, then a 256 MB "
                                "read of another buffer so no dirty flush lines are written back inside the kernel)"})

    out = None
    if rank == 0:
        cpu = None
        if not args.skip_cpu:
            cb = cpu_reference(counts, world, batch, 3, 1)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        # like-for-like: the same sync work per iteration (every slice of the model through
        # aggregate + SGD + replica apply) on the GPU (sync-only launch) and on the host cores
        gpu_sync = batch * world / (sync_ms * 1e-3) if sync_ms == sync_ms else None
        sync_path = {"gpu_samples_per_s": gpu_sync, "gpu_ms_per_iteration": sync_ms,
                     "cpu_samples_per_s": cpu["value"] if cpu else None,
                     "cpu_ms_per_iteration": 1000.0 * batch * world / cpu["value"] if cpu else None,
                     "gpu_over_cpu": gpu_sync / cpu["value"] if (cpu and gpu_sync) else None,
                     "what": "one iteration of the P3 sync path at the model's shapes (aggregate in rank order + SGD "
                             "+ apply to every replica; the CPU side also materialises GradGen gradients) — the "
                             "reference arm measures this; the training value above adds the model's compute"}
        out = {
            "metric": METRIC, "value": value, "unit": "samples/sec", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",  # the sync path's arithmetic (fp32 sum / SGD / broadcast)
            "data": "synthetic (random-init weights, N(0,1) bf16 images / uniform labels)",
            "config": {"workload": f"{args.model} bf16-autocast training, P3 sliced priority sync",
                       "model": args.model, "per_gpu_batch": batch, "global_batch": batch * world,
                       "max_slice": args.max_slice,
                       "comm_launches": (f"{args.comm_ctas}-CTA DRAIN launches during the backward pass + one "
                                         f"{args.comm_ctas}-CTA FINISH launch per step" if world > 1 else
                                         f"one {torch.cuda.get_device_properties(0).multi_processor_count}-CTA FINISH "
                                         "launch per step (SWEEP mode: nothing to overlap at N=1)"),
                       "pop_order": ("bounded relaxation: each pop among the C most urgent available layers, C = CTAs "
                                     "of its launch; strict FrameQueue order is the strict_order mode (tests)"
                                     if world > 1 else "guided chunk claims of the priority-ordered element space, "
                                     "in order (bounded by the concurrent CTAs)"),
                       "parallelism": f"dp{world}",
                       "model_compute": "bf16 autocast (fp32 master parameters)",
                       "params": P, "tensors": len(counts), "l2": "activations >> 126 MB L2 each step"},
            "e2e": {"value": e2e_value, "unit": "samples/sec", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4}
                   if e2e_value else None,
            "layerwise": layerwise,
            "p3_vs_layerwise": (value / layerwise["value"]) if layerwise else None,
            "throttled": throttled,
            "roofline": roof,
            "slice_sync": {"ms": sync_ms, "GBps_per_gpu": roof["achieved"], "bound": roof["bound"]},
            "sync_path": sync_path,
            "training_sync": train_sync,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": gpu_launches,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
