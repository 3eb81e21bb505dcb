"""Device runtime of the P3 sync path: the sync context and the emulated training worker.

``SyncContext`` wraps one ``p3_ctx_t`` (csrc/p3_ctx.cu): the plan tables on the GPU, the
per-rank parameter replica ``W`` (peer-writable), the receive slots ``R``, the flags, and
the per-iteration launch of the persistent comm kernel (K3). It hosts either one rank
(one process per GPU, peers opened through CUDA IPC) or all ranks of a world on one GPU
(single-launch emulation for tests).

``TrainingWorker`` mirrors ``p3sync.worker.TrainingWorker`` (reference
``pkg/src/p3sync/worker.py:64-392``) in emulate mode: per-layer forward gating
(_wait_layer), sleep-emulated fwd/bwd compute on the device, synthetic GradGen gradients
(K1) and atomic per-layer publication (enqueue_layer), with the comm kernel doing the
priority send, the owner-side aggregate/update and the broadcast.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .hashing import FNV_OFFSET, fnv1a64
from .model import ModelProfile
from .plan import BASELINE_MODE, P3_MODE, DEFAULT_MAX_SLICE, SliceKey, make_baseline_plan, make_p3_plan


class _DeviceArray:
    """Zero-copy __cuda_array_interface__ view so torch can alias libp3-owned memory."""

    def __init__(self, ptr: int, n: int, owner, typestr: str = "<f4") -> None:
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 2}
        self._owner = owner


@dataclass
class TraceEvent:
    t_ns: int
    iteration: int
    layer: int
    slice: int
    rank: int
    event: int  # _lib.P3_EV_PUSH / BCAST / PUBLISH / COMPLETE / PICK
    t0_ns: int = 0  # PUSH / PICK: before the queue snapshot the claim came from


def plan_fingerprint(layer_counts, world, max_slice, plan_mode, big_threshold, rng_seed, priority_mode, lr, momentum,
                     push_dtype, notify_pull=False, param_dtype="fp32") -> str:
    """What every rank of one sync group must agree on: the plan (layer sizes, world, slice
    size, placement), the discipline and the update rule. Ranks that disagree would wait on
    each other forever (a slice one rank never pushes), so ``connect`` refuses them."""
    key = repr((list(map(int, layer_counts)), int(world), int(max_slice), plan_mode, int(big_threshold), int(rng_seed),
                bool(priority_mode), float(lr), float(momentum), push_dtype, bool(notify_pull), param_dtype))
    return f"{fnv1a64(key.encode()):016x}"


def exchange_peer_handles(handle: bytes, fingerprint: str, group=None) -> list[bytes]:
    """All-gather (torch.distributed, any backend) of every rank's IPC handle, in rank order,
    after checking that all ranks built the same plan (``plan_fingerprint``): the host side of
    TrainingWorker._connect_all (worker.py:136), which dials every server."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if len(handle) != _lib.P3_IPC_BYTES:
        raise ValueError(f"IPC handle must be {_lib.P3_IPC_BYTES} bytes")
    rows = [None] * world
    dist.all_gather_object(rows, (rank, fingerprint, bytes(handle)), group=group)
    prints = sorted({r[1] for r in rows})
    if len(prints) != 1:
        from .plan import PlanError

        raise PlanError(f"ranks built different sync plans (fingerprints {prints}): same model, world, "
                        "max_slice, plan mode and update rule are required on every rank")
    if [r[0] for r in rows] != list(range(world)):
        raise RuntimeError("handle exchange out of rank order")
    return [r[2] for r in rows]


def connect(ctx: "SyncContext", group=None) -> None:
    """Open every peer's arena (NVLink / CUDA IPC) for a one-rank-per-process context; with
    ``nvls`` the arenas travel as file descriptors and the replicas join one multicast object
    (connect_nvls)."""
    if ctx.world > 1 and ctx.nvls:
        connect_nvls(ctx, group)
    elif ctx.world > 1:
        ctx.open_peers(exchange_peer_handles(ctx.ipc_handle(0), ctx.fingerprint, group))


def connect_nvls(ctx: "SyncContext", group=None) -> None:
    """NVLS bootstrap (include/p3.h, p3_ctx_export_fd .. p3_nvls_bind): every rank serves its
    arena's file descriptor (rank 0 also the multicast object's) on a Unix socket, the paths
    go around with torch.distributed, each rank receives its peers' descriptors (SCM_RIGHTS)
    and maps their arenas; then every rank adds its GPU to the multicast object, and once all
    have, binds its replica to it."""
    import os
    import socket
    import tempfile
    import threading
    import uuid

    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine, err = [], None
    try:  # (a failure on one rank must not leave the others waiting in the exchange)
        mine.append(ctx.export_fd(0))
        if rank == 0:
            mine.append(ctx.nvls_create())
    except Exception as e:  # noqa: BLE001
        err = f"rank {rank}: {e}"
    errs = [None] * world
    dist.all_gather_object(errs, err, group=group)
    if any(errs):
        for f in mine:
            os.close(f)
        raise RuntimeError("nvls bootstrap failed: " + "; ".join(e for e in errs if e))
    path = os.path.join(tempfile.gettempdir(), f"p3_nvls_{uuid.uuid4().hex}_{rank}.sock")
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(path)
    srv.listen(world)

    def serve() -> None:
        for _ in range(world - 1):
            conn, _ = srv.accept()
            with conn:
                socket.send_fds(conn, [b"p3"], mine)
                conn.recv(1)  # the peer holds its copies: the descriptors may close

    t = threading.Thread(target=serve, daemon=True)
    t.start()
    rows = [None] * world
    dist.all_gather_object(rows, (rank, ctx.fingerprint, path), group=group)
    if len({r[1] for r in rows}) != 1:
        from .plan import PlanError

        raise PlanError("ranks built different sync plans (fingerprints differ)")
    fds, mc = [-1] * world, -1
    try:
        for r in range(world):
            if r == rank:
                continue
            with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as cl:
                cl.connect(rows[r][2])
                _, got, _, _ = socket.recv_fds(cl, 16, 2)
                cl.sendall(b"k")
            fds[r] = got[0]
            if r == 0:
                mc = got[1]
        t.join()
        ctx.open_peers_fd(fds)
        ctx.nvls_attach(mc)
        dist.barrier(group)  # every GPU added before any bind
        ctx.nvls_bind()
        dist.barrier(group)
    finally:
        srv.close()
        os.unlink(path)
        for f in mine + [x for x in fds if x >= 0] + ([mc] if mc >= 0 else []):
            os.close(f)


class SyncContext:
    """One p3 sync context (see include/p3.h, p3_ctx_create)."""

    def __init__(
        self,
        layer_counts: list[int],
        world: int,
        local_ranks: list[int],
        max_slice: int = DEFAULT_MAX_SLICE,
        lr: float = 0.1,
        momentum: float = 0.0,
        priority_mode: bool = True,
        comm_ctas: int = 16,
        comm_threads: int = 512,
        timeout_s: float = 60.0,
        trace_cap: int = 0,
        emulate_grads: bool = False,
        drain_bytes: int = 0,
        plan_mode: str = "p3",
        big_threshold: int = 1_000_000,
        rng_seed: int = 0,
        throttle_bps: float = 0.0,
        throttle_burst: int = 50 * 1024,
        gate_groups: list[int] | None = None,
        pub_batch_bytes: int = 0,
        drain_linger_us: int = 0,
        finish_ctas: int = 0,
        pop_relax: int = 0,
        pop_run: int = 0,
        pop_multi: int = 0,
        push_dtype: str = "fp32",
        drain_streams: int = 0,
        notify_pull: bool = False,
        param_dtype: str = "fp32",
        nvls: bool = False,
    ) -> None:
        import torch

        torch.cuda.init()
        self.lib = _lib.load()
        self.layer_counts = [int(c) for c in layer_counts]
        self.world = world
        self.local_ranks = list(local_ranks)
        self.max_slice = max_slice
        self.lr = lr
        self.trace_cap = trace_cap
        self.timeout_s = timeout_s
        cfg = _lib.Config()
        cfg.world = world
        cfg.n_local = len(self.local_ranks)
        for i, r in enumerate(self.local_ranks):
            cfg.local_ranks[i] = r
        cfg.n_layers = len(self.layer_counts)
        self._counts = _lib.u64_array(self.layer_counts)
        cfg.layer_counts = ctypes.cast(self._counts, ctypes.POINTER(ctypes.c_uint64))
        cfg.max_slice = max_slice
        if plan_mode not in (P3_MODE, BASELINE_MODE):
            raise ValueError(f"plan_mode must be {P3_MODE!r} or {BASELINE_MODE!r}")
        cfg.plan_mode = _lib.P3_PLAN_P3 if plan_mode == P3_MODE else _lib.P3_PLAN_BASELINE
        cfg.big_threshold = big_threshold
        cfg.rng_seed = rng_seed
        cfg.throttle_bps = throttle_bps or 0.0
        cfg.throttle_burst = throttle_burst
        cfg.pub_batch_bytes = pub_batch_bytes
        cfg.drain_linger_us = drain_linger_us
        cfg.finish_ctas = finish_ctas
        cfg.pop_relax = pop_relax
        cfg.pop_run = pop_run
        cfg.pop_multi = pop_multi
        if push_dtype not in ("fp32", "bf16"):
            raise ValueError("push_dtype must be 'fp32' or 'bf16'")
        cfg.push_bf16 = 1 if push_dtype == "bf16" else 0
        self.push_dtype = push_dtype
        if gate_groups is not None:
            if len(gate_groups) != len(self.layer_counts):
                raise ValueError("gate_groups needs one group id per layer")
            self._groups = (ctypes.c_uint32 * len(gate_groups))(*gate_groups)
            cfg.gate_groups = ctypes.cast(self._groups, ctypes.POINTER(ctypes.c_uint32))
        cfg.sched = _lib.P3_SCHED_PRIORITY if priority_mode else _lib.P3_SCHED_FIFO
        cfg.lr = lr
        cfg.momentum = momentum
        cfg.comm_ctas = comm_ctas
        cfg.comm_threads = comm_threads
        cfg.timeout_s = timeout_s
        cfg.trace_cap = trace_cap
        cfg.emulate_grads = 1 if emulate_grads else 0
        cfg.drain_bytes = drain_bytes
        cfg.drain_streams = drain_streams
        cfg.notify_pull = 1 if notify_pull else 0
        if param_dtype not in ("fp32", "bf16"):
            raise ValueError("param_dtype must be 'fp32' or 'bf16'")
        cfg.param_bf16 = 1 if param_dtype == "bf16" else 0
        self.param_dtype = param_dtype
        cfg.nvls = 1 if nvls else 0
        self.nvls = bool(nvls)
        self.strict = comm_ctas == 1 and (finish_ctas or comm_ctas) == 1 and pop_relax == 1 and drain_streams == 1
        h = ctypes.c_void_p()
        _lib.check(self.lib.p3_ctx_create(ctypes.byref(cfg), ctypes.byref(h)), what="p3_ctx_create")
        self._h = h
        self.layer_offsets = []
        off = ctypes.c_uint64()
        for l in range(len(self.layer_counts)):
            self._check(self.lib.p3_ctx_layer_offset(self._h, l, ctypes.byref(off)), "p3_ctx_layer_offset")
            self.layer_offsets.append(int(off.value))
        self.arena_elems = self.layer_offsets[-1] + self.layer_counts[-1]
        self.plan_mode = plan_mode
        self.fingerprint = plan_fingerprint(self.layer_counts, world, max_slice, plan_mode, big_threshold, rng_seed,
                                            priority_mode, lr, momentum, push_dtype, notify_pull, param_dtype)

    # ------------------------------------------------------------------ plumbing
    def _check(self, rc: int, what: str) -> None:
        _lib.check(rc, self._h, what)

    @property
    def handle(self):
        return self._h

    def _ptr(self, fn, li: int) -> int:
        p = ctypes.c_void_p()
        self._check(fn(self._h, li, ctypes.byref(p)), fn.__name__)
        return int(p.value)

    def params_arena(self, li: int = 0):
        """torch view (float32, or bfloat16 with param_dtype="bf16") over the whole parameter
        replica W of local rank ``li``."""
        import torch

        ptr = self._ptr(self.lib.p3_ctx_params, li)
        if self.param_dtype == "bf16":
            raw = torch.as_tensor(_DeviceArray(ptr, self.arena_elems, self, "<i2"), device="cuda")
            return raw.view(torch.bfloat16)
        return torch.as_tensor(_DeviceArray(ptr, self.arena_elems, self), device="cuda")

    def master_init(self, li: int = 0, stream=None) -> None:
        """param_bf16: the owned slices' fp32 master from the replica (once, after the initial
        parameters are in W)."""
        self._check(self.lib.p3_master_init(self._h, li, _lib.stream_handle(stream)), "p3_master_init")

    def grads_arena(self, li: int = 0):
        import torch

        return torch.as_tensor(_DeviceArray(self._ptr(self.lib.p3_ctx_grads, li), self.arena_elems, self), device="cuda")

    def layer_params(self, li: int, layer: int):
        off = self.layer_offsets[layer]
        return self.params_arena(li)[off : off + self.layer_counts[layer]]

    def ipc_handle(self, li: int = 0) -> bytes:
        buf = ctypes.create_string_buffer(_lib.P3_IPC_BYTES)
        self._check(self.lib.p3_ctx_ipc_handle(self._h, li, buf), "p3_ctx_ipc_handle")
        return buf.raw

    def export_fd(self, li: int = 0) -> int:
        fd = ctypes.c_int(-1)
        self._check(self.lib.p3_ctx_export_fd(self._h, li, ctypes.byref(fd)), "p3_ctx_export_fd")
        return fd.value

    def open_peers_fd(self, fds: list[int]) -> None:
        arr = (ctypes.c_int * len(fds))(*fds)
        self._check(self.lib.p3_ctx_open_peers_fd(self._h, arr), "p3_ctx_open_peers_fd")

    def nvls_create(self) -> int:
        fd = ctypes.c_int(-1)
        self._check(self.lib.p3_nvls_create(self._h, ctypes.byref(fd)), "p3_nvls_create")
        return fd.value

    def nvls_attach(self, fd: int) -> None:
        self._check(self.lib.p3_nvls_attach(self._h, fd), "p3_nvls_attach")

    def nvls_bind(self) -> None:
        self._check(self.lib.p3_nvls_bind(self._h), "p3_nvls_bind")

    def open_peers(self, handles: list[bytes]) -> None:
        blob = b"".join(h.ljust(_lib.P3_IPC_BYTES, b"\0") for h in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        self._check(self.lib.p3_ctx_open_peers(self._h, buf), "p3_ctx_open_peers")

    # ------------------------------------------------------------------ hot calls
    def iteration_begin(self, k: int, stream=None) -> None:
        self._check(self.lib.p3_iteration_begin(self._h, k, _lib.stream_handle(stream)), "p3_iteration_begin")

    def iteration_end(self, k: int) -> None:
        self._check(self.lib.p3_iteration_end(self._h, k), "p3_iteration_end")

    def launches(self) -> int:
        n = ctypes.c_uint64()
        self._check(self.lib.p3_comm_launches(self._h, ctypes.byref(n)), "p3_comm_launches")
        return int(n.value)

    def layer_ready(self, li: int, layer: int, k: int, grad=None, stream=None) -> None:
        ptr = grad.data_ptr() if grad is not None else None
        self._check(self.lib.p3_layer_ready(self._h, li, layer, k, ptr, _lib.stream_handle(stream)), "p3_layer_ready")

    def gradgen_layer(self, li: int, seed: int, k: int, layer: int, stream=None) -> None:
        self._check(
            self.lib.p3_gradgen_layer(self._h, li, seed & 0xFFFFFFFFFFFFFFFF, k, layer, _lib.stream_handle(stream)),
            "p3_gradgen_layer",
        )

    def wait_layer(self, li: int, layer: int, k: int, stream=None) -> None:
        self._check(self.lib.p3_wait_layer(self._h, li, layer, k, _lib.stream_handle(stream)), "p3_wait_layer")

    def wait_group(self, li: int, group: int, k: int, stream=None) -> None:
        self._check(self.lib.p3_wait_group(self._h, li, group, k, _lib.stream_handle(stream)), "p3_wait_group")

    def sync_all(self, k: int, timeout_s: float | None = None) -> None:
        self._check(self.lib.p3_sync_all(self._h, k, self.timeout_s if timeout_s is None else timeout_s), "p3_sync_all")

    # ------------------------------------------------------------------ outputs
    def trace(self, li: int = 0) -> list[TraceEvent]:
        n = ctypes.c_uint64()
        self._check(self.lib.p3_trace_read(self._h, li, None, 0, ctypes.byref(n)), "p3_trace_read")
        if n.value == 0:
            return []
        recs = (_lib.TraceRec * n.value)()
        self._check(self.lib.p3_trace_read(self._h, li, recs, n.value, ctypes.byref(n)), "p3_trace_read")
        return [TraceEvent(r.t_ns, r.iteration, r.layer, r.slice, r.rank, r.event, r.t0_ns) for r in recs[: n.value]]

    def debug_snapshot(self, li: int = 0) -> dict:
        n = ctypes.c_uint64()
        self._check(self.lib.p3_debug_snapshot(self._h, li, None, 0, ctypes.byref(n)), "p3_debug_snapshot")
        buf = (ctypes.c_uint32 * n.value)()
        self._check(self.lib.p3_debug_snapshot(self._h, li, buf, n.value, ctypes.byref(n)), "p3_debug_snapshot")
        L = len(self.layer_counts)
        arr = list(buf)
        names = ("ready", "cursor", "srv_taken", "hint", "done")
        out = {nm: arr[i * L : (i + 1) * L] for i, nm in enumerate(names)}
        out["pushed"], out["reduced"], out["exited"], out["jobs"] = arr[5 * L : 5 * L + 4]
        t = arr[5 * L + 4 : 5 * L + 12]
        for i, nm in enumerate(("t_pick_ns", "t_slot_wait_ns", "t_move_ns", "t_signal_ns")):
            out[nm] = t[2 * i] | (t[2 * i + 1] << 32)
        base = 5 * L + 12 + 512
        S = (len(arr) - base) // 2
        out["cta_phase"] = arr[5 * L + 12 : base]
        out["arrivals"] = arr[base : base + S]
        out["claim"] = arr[base + S :]
        return out

    def clear_trace(self) -> None:
        self._check(self.lib.p3_trace_clear(self._h), "p3_trace_clear")

    def counters(self, li: int = 0) -> tuple[int, int]:
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(self.lib.p3_counters(self._h, li, ctypes.byref(a), ctypes.byref(b)), "p3_counters")
        return int(a.value), int(b.value)

    def params_numpy(self, li: int = 0) -> list[np.ndarray]:
        flat = self.params_arena(li).float().cpu().numpy()
        return [flat[o : o + c].copy() for o, c in zip(self.layer_offsets, self.layer_counts)]

    def params_digest(self, li: int = 0) -> int:
        """params_digest (worker.py:372-376): chained FNV-1a over fp32 LE layer bytes."""
        h = FNV_OFFSET
        for vec in self.params_numpy(li):
            h = fnv1a64(vec.astype("<f4").tobytes(), h)
        return h

    def close(self) -> None:
        if getattr(self, "_h", None):
            self.lib.p3_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


@dataclass
class WorkerConfig:
    """Worker settings (worker.py:39-50). ``servers`` keeps the reference's meaning — the
    parameter servers a worker pushes to, one per rank (cli.py:81-82) — given as the peer
    list or just its length; ``world`` is that count. The fields after ``sample_period_ms``
    configure the device path."""

    rank: int
    mode: str
    servers: object = None             # list of peers (host, port) / GPUs, or their count
    iterations: int = 1
    lr: float = 0.1
    batch_size: int = 32
    throttle_rate: float | None = None  # bit/s per rank egress (worker.py:46); None = full NVLink
    throttle_burst: int = 50 * 1024
    deadlock_timeout: float = 60.0
    sample_period_ms: int = 10
    world: int = 0                      # = number of servers (derived from ``servers``)
    max_slice: int = DEFAULT_MAX_SLICE
    emulate_compute: bool = True
    comm_ctas: int = 16
    comm_threads: int = 512
    trace_cap: int = 0
    rank_distinct_grads: bool = False
    big_threshold: int = 1_000_000     # baseline plan (cli.py:68)
    seed: int = 0                      # baseline plan placement seed (cli.py:74)
    push_dtype: str = "fp32"           # "bf16": declared lossy transport of pushes
    finish_ctas: int = 0               # CTAs of the FINISH launch (0: comm_ctas)
    pop_relax: int = 0                 # bounded pop relaxation (0: the launch's CTA count)
    drain_streams: int = 0             # side streams of DRAIN launches (0: 4)
    strict_order: bool = False         # one consumer at a time: 1 CTA per launch, 1 DRAIN stream,
                                       # strict FrameQueue order (the reference's single sender)
    notify_pull: bool | None = None    # owners NOTIFY, replicas PULL (None: in baseline mode, as the
                                       # reference's baseline does, server.py:227-247)

    def __post_init__(self) -> None:
        n = None if self.servers is None else (self.servers if isinstance(self.servers, int) else len(self.servers))
        if self.world == 0:
            if n is None:
                raise ValueError("WorkerConfig needs servers (or world)")
            self.world = n
        elif n is None:
            self.servers = self.world
        elif n != self.world:
            raise ValueError(f"{n} servers but world={self.world}")
        if not 0 <= self.rank < self.world:
            raise ValueError(f"rank {self.rank} outside [0, {self.world})")


def rank_seed(seed: int, rank: int, distinct: bool) -> int:
    """GradGen seed of a rank: the reference's seed for every rank (worker.py:71), or a
    splitmix-salted seed per rank when distinct gradients are requested."""
    if not distinct or rank == 0:
        return seed
    from .hashing import splitmix64_stream

    return seed ^ splitmix64_stream(0x5EED, rank)


class TrainingWorker:
    """Emulate-mode worker(s) on one GPU; ``ranks`` > 1 emulates a whole world in one process.

    ``run_iteration`` issues, per hosted rank and on that rank's compute stream:
    forward: ``_wait_layer`` gate (stream memory wait) + device sleep per layer;
    backward: device sleep, K1 gradient generation and ``enqueue_layer`` per layer in
    reverse order (worker.py:312-325); each publication is followed on the comm stream by
    a DRAIN launch of the comm kernel, and the iteration ends with a FINISH launch.
    """

    def __init__(self, config: WorkerConfig, profile: ModelProfile, plan=None, ranks: list[int] | None = None,
                 ctx: SyncContext | None = None) -> None:
        import torch

        if plan is not None and not hasattr(plan, "slices"):  # (round-1 call form: ranks third)
            plan, ranks = None, plan
        if config.mode not in (P3_MODE, BASELINE_MODE):
            raise ValueError(f"mode must be {P3_MODE!r} or {BASELINE_MODE!r}, not {config.mode!r}")
        if plan is not None and plan.mode != config.mode:
            raise ValueError(f"plan mode {plan.mode!r} != worker mode {config.mode!r}")  # worker.py:65-67
        self.cfg = config
        self.profile = profile
        self.ranks = list(ranks) if ranks is not None else [config.rank]
        # p3: sliced plan + priority queue; baseline: KVStore placement + FIFO (the reference's
        # two modes, worker.py:84-93, plan.py:94-164). The device builds its plan from the
        # same inputs; a caller's plan must be that plan.
        if plan is not None and config.mode == P3_MODE:
            multi = [s.length for s in plan.slices if s.key.slice_index == 0 and len(plan.slices_of_layer(s.key.layer_index)) > 1]
            if multi:
                config.max_slice = max(multi)
        if config.mode == P3_MODE:
            self.plan = make_p3_plan(profile, config.world, config.max_slice)
        else:
            self.plan = make_baseline_plan(profile, config.world, config.big_threshold, config.seed)
        if plan is not None:
            from .plan import PlanError, plan_to_csv

            if plan_to_csv(plan) != plan_to_csv(self.plan):
                raise PlanError("the plan differs from the one the device builds for this profile, server count, "
                                "slice size and placement (make_p3_plan / make_baseline_plan)")
        self.ctx = ctx or SyncContext(
            profile.param_counts(),
            config.world,
            self.ranks,
            max_slice=config.max_slice,
            lr=config.lr,
            priority_mode=config.mode == P3_MODE,
            comm_ctas=1 if config.strict_order else config.comm_ctas,
            comm_threads=config.comm_threads,
            timeout_s=config.deadlock_timeout,
            trace_cap=config.trace_cap,
            emulate_grads=True,
            plan_mode=config.mode,
            big_threshold=config.big_threshold,
            rng_seed=config.seed,
            throttle_bps=config.throttle_rate or 0.0,
            throttle_burst=config.throttle_burst,
            push_dtype=config.push_dtype,
            finish_ctas=1 if config.strict_order else config.finish_ctas,
            pop_relax=1 if config.strict_order else config.pop_relax,
            drain_streams=1 if config.strict_order else config.drain_streams,
            notify_pull=(config.mode == BASELINE_MODE) if config.notify_pull is None else config.notify_pull,
        )
        self.comm_stream = torch.cuda.Stream()
        self.streams = [torch.cuda.Stream() for _ in self.ranks]
        self.mark_stream = torch.cuda.Stream()
        self.iterations_done = 0
        self.iter_events: list = []
        self._nslices = [len(self.plan.slices_of_layer(l.index)) for l in profile.layers]
        self._recv_seen: dict = {}

    def run_iteration(self, k: int) -> None:
        import torch

        lib = self.ctx.lib
        ctx = self.ctx
        ctx.iteration_begin(k, self.comm_stream)
        marks = ctx.trace_cap > 0
        for li, rank in enumerate(self.ranks):
            s = self.streams[li]
            sh = _lib.stream_handle(s)
            seed = rank_seed(self.profile.seed, rank, self.cfg.rank_distinct_grads)
            if marks:  # IterationRecord.start (worker.py:312-313) on the device clock
                ctx._check(lib.p3_trace_mark(ctx.handle, li, k, _lib.P3_EV_ITER_START, sh), "p3_trace_mark")
            for layer in self.profile.layers:
                ctx._check(lib.p3_wait_layer(ctx.handle, li, layer.index, k, sh), "p3_wait_layer")
                if self.cfg.emulate_compute and layer.fwd_time:
                    _lib.check(lib.p3_emulate_compute(layer.fwd_time, sh), what="p3_emulate_compute")
            if li == 0:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s)
                self.iter_events.append(ev)
            for layer in reversed(self.profile.layers):
                if self.cfg.emulate_compute and layer.bwd_time:
                    _lib.check(lib.p3_emulate_compute(layer.bwd_time, sh), what="p3_emulate_compute")
                ctx._check(lib.p3_gradgen_layer(ctx.handle, li, seed & 0xFFFFFFFFFFFFFFFF, k, layer.index, sh), "p3_gradgen_layer")
                ctx._check(lib.p3_layer_ready(ctx.handle, li, layer.index, k, None, sh), "p3_layer_ready")
        ctx.iteration_end(k)
        if marks:  # sync_end (worker.py:265-268): every layer of the rank holds iteration k+1
            mh = _lib.stream_handle(self.mark_stream)
            for li in range(len(self.ranks)):
                for layer in self.profile.layers:
                    ctx._check(lib.p3_wait_layer(ctx.handle, li, layer.index, k + 1, mh), "p3_wait_layer")
                ctx._check(lib.p3_trace_mark(ctx.handle, li, k, _lib.P3_EV_SYNCED, mh), "p3_trace_mark")
        self.iterations_done = k + 1

    # -- the reference worker's public entry points -----------------------------------

    def enqueue_layer(self, layer_index: int, iteration: int, li: int = 0, grad=None, stream=None) -> None:
        """TrainingWorker.enqueue_layer (worker.py:173-182): publish every slice of the layer for
        ``iteration`` atomically. Emulate mode (``grad`` None) first materialises the rank's
        GradGen gradient (K1, worker.py:166-171) on ``stream``; the iteration must be open
        (``ctx.iteration_begin``) for the comm kernel to pick it up."""
        s = stream if stream is not None else self.streams[li]
        if grad is None:
            seed = rank_seed(self.profile.seed, self.ranks[li], self.cfg.rank_distinct_grads)
            self.ctx.gradgen_layer(li, seed & 0xFFFFFFFFFFFFFFFF, iteration, layer_index, s)
        self.ctx.layer_ready(li, layer_index, iteration, grad, s)

    def flag(self, layer_index: int, li: int = 0) -> int:
        """flags[layer] (worker.py:74-75): the forward pass whose parameters the layer holds."""
        it = ctypes.c_uint64()
        self.ctx._check(self.ctx.lib.p3_layer_flag(self.ctx.handle, li, layer_index, ctypes.byref(it)), "p3_layer_flag")
        return int(it.value)

    def on_bcast(self, frame, li: int = 0) -> None:
        """TrainingWorker.on_bcast (worker.py:241-269) for a BCAST frame that reached the host
        (the wire path beyond the NVSwitch domain): same checks and ProtocolErrors, then the
        slice goes into the device replica and counts towards the layer's forward gate."""
        from .proto import ProtocolError

        key = SliceKey(frame.layer_index, frame.slice_index)
        layer = key.layer_index
        if not 0 <= layer < len(self._nslices) or not 0 <= key.slice_index < self._nslices[layer]:
            raise ProtocolError(f"BCAST for unknown key {key}")
        held = self.flag(layer, li)
        if frame.iteration != held:
            raise ProtocolError(f"layer {layer}: BCAST for iteration {frame.iteration}, "
                                f"worker holds parameters of iteration {held}")
        seen = self._recv_seen.setdefault((li, layer, held), set())
        if key in seen:
            raise ProtocolError(f"duplicate BCAST slice {key} at iteration {frame.iteration}")
        values = np.ascontiguousarray(frame.payload_f32(), dtype=np.float32)
        sl = self.plan.slices_of_layer(layer)[key.slice_index]
        if len(values) != sl.length:
            raise ProtocolError(f"slice {key}: payload holds {len(values)} values, expected {sl.length}")
        stream = self.streams[li]
        self.ctx._check(self.ctx.lib.p3_apply_slice(self.ctx.handle, li, layer, key.slice_index,
                                                    values.ctypes.data_as(ctypes.c_void_p), len(values),
                                                    _lib.stream_handle(stream)), "p3_apply_slice")
        stream.synchronize()  # the host payload buffer may be released after return
        seen.add(key)
        if len(seen) == self._nslices[layer]:
            del self._recv_seen[(li, layer, held)]

    def run(self) -> None:
        for k in range(self.cfg.iterations):
            self.run_iteration(k)
        self.wait_all(self.cfg.iterations)

    def wait_all(self, iteration: int) -> None:
        self.ctx.sync_all(iteration, self.cfg.deadlock_timeout)
        import torch

        for s in self.streams:
            s.synchronize()

    def params(self, li: int = 0) -> list[np.ndarray]:
        return self.ctx.params_numpy(li)

    def params_digest(self, li: int = 0) -> int:
        return self.ctx.params_digest(li)

    def transmission_sequence(self, li: int = 0, iteration: int | None = None) -> list[SliceKey]:
        ev = [e for e in self.ctx.trace(li) if e.event == _lib.P3_EV_PUSH and (iteration is None or e.iteration == iteration)]
        return [SliceKey(e.layer, e.slice) for e in ev]

    def close(self) -> None:
        self.ctx.close()
