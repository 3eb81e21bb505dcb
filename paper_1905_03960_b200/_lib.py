"""ctypes binding of libp3.so, the C ABI declared in include/p3.h.

The library is built in-tree by ``paper_1905_03960_b200/csrc/build.sh`` (see
``__graft_entry__.build``). There is no fallback: if the shared object is missing every
entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

P3_OK = 0
P3_EUSAGE = 1
P3_EPROTOCOL = 2
P3_ETIMEOUT = 3
P3_ECUDA = 4
P3_EMORE = 5
P3_FRAME_HEADER_BYTES = 39

P3_PLAN_P3 = 0
P3_PLAN_BASELINE = 1
P3_SCHED_PRIORITY = 0
P3_SCHED_FIFO = 1
P3_MAX_RANKS = 16
P3_IPC_BYTES = 64
P3_EV_PUSH = 0
P3_EV_BCAST = 1
P3_EV_PUBLISH = 2
P3_EV_COMPLETE = 3
P3_EV_PICK = 4
P3_EV_ITER_START = 5
P3_EV_SYNCED = 6
P3_EV_NOTIFY = 7
P3_EV_PULL = 8

LIB_PATH = Path(__file__).resolve().parent / "libp3.so"


class SliceRow(ctypes.Structure):
    _fields_ = [
        ("layer", ctypes.c_uint32),
        ("slice", ctypes.c_uint32),
        ("offset", ctypes.c_uint64),
        ("length", ctypes.c_uint64),
        ("priority", ctypes.c_uint32),
        ("server", ctypes.c_uint32),
    ]


class TraceRec(ctypes.Structure):
    _fields_ = [
        ("t_ns", ctypes.c_uint64),
        ("t0_ns", ctypes.c_uint64),
        ("iteration", ctypes.c_uint32),
        ("layer", ctypes.c_uint32),
        ("slice", ctypes.c_uint32),
        ("rank", ctypes.c_uint16),
        ("event", ctypes.c_uint16),
    ]


class FrameT(ctypes.Structure):
    _fields_ = [
        ("msg_type", ctypes.c_uint32),
        ("priority", ctypes.c_uint32),
        ("iteration", ctypes.c_uint64),
        ("worker_rank", ctypes.c_uint32),
        ("layer", ctypes.c_uint32),
        ("slice", ctypes.c_uint32),
        ("offset", ctypes.c_uint64),
        ("payload_len", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
    ]


class Config(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_uint32),
        ("n_local", ctypes.c_uint32),
        ("local_ranks", ctypes.c_uint32 * P3_MAX_RANKS),
        ("n_layers", ctypes.c_uint32),
        ("layer_counts", ctypes.POINTER(ctypes.c_uint64)),
        ("max_slice", ctypes.c_uint64),
        ("plan_mode", ctypes.c_uint32),
        ("sched", ctypes.c_uint32),
        ("lr", ctypes.c_float),
        ("momentum", ctypes.c_float),
        ("comm_ctas", ctypes.c_uint32),
        ("comm_threads", ctypes.c_uint32),
        ("timeout_s", ctypes.c_double),
        ("trace_cap", ctypes.c_uint32),
        ("emulate_grads", ctypes.c_uint32),
        ("drain_bytes", ctypes.c_uint64),
        ("big_threshold", ctypes.c_uint64),
        ("rng_seed", ctypes.c_uint64),
        ("throttle_bps", ctypes.c_double),
        ("throttle_burst", ctypes.c_uint64),
        ("pub_batch_bytes", ctypes.c_uint64),
        ("drain_linger_us", ctypes.c_uint32),
        ("finish_ctas", ctypes.c_uint32),
        ("pop_relax", ctypes.c_uint32),
        ("pop_run", ctypes.c_uint32),
        ("pop_multi", ctypes.c_uint32),
        ("push_bf16", ctypes.c_uint32),
        ("gate_groups", ctypes.POINTER(ctypes.c_uint32)),
        ("drain_streams", ctypes.c_uint32),
        ("notify_pull", ctypes.c_uint32),
        ("param_bf16", ctypes.c_uint32),
        ("nvls", ctypes.c_uint32),
    ]


_P = ctypes.c_void_p
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_PU32 = ctypes.POINTER(ctypes.c_uint32)
_PU64 = ctypes.POINTER(ctypes.c_uint64)

# name -> (restype, argtypes); exactly the symbols include/p3.h declares
SIGNATURES = {
    "p3_plan_p3": (ctypes.c_int, [_PU64, _U32, _U32, _U64, ctypes.POINTER(SliceRow), _U64, _PU64]),
    "p3_plan_baseline": (ctypes.c_int, [_PU64, _U32, _U32, _U64, _U64, ctypes.POINTER(SliceRow), _U64, _PU64]),
    "p3_splitmix64_stream": (_U64, [_U64, _U64]),
    "p3_fnv1a64": (_U64, [_P, _U64, _U64]),
    "p3_gradient_block": (ctypes.c_int, [_U64, _U64, _U64, _U64, _U64, _P, _P]),
    "p3_shard_update": (ctypes.c_int, [_P, ctypes.POINTER(_P), _U32, _U64, ctypes.c_float, ctypes.c_float, _P, _P]),
    "p3_emulate_compute": (ctypes.c_int, [_U64, _P]),
    "p3_simulate": (ctypes.c_int, [_P, _P, _U64, _PU64]),
    "p3_queue_create": (ctypes.c_int, [_PU32, _U32, _U32, ctypes.POINTER(_P)]),
    "p3_queue_put_layer": (ctypes.c_int, [_P, _U32, _U32]),
    "p3_queue_poll": (ctypes.c_int, [_P, _PU32, _PU32]),
    "p3_queue_destroy": (ctypes.c_int, [_P]),
    "p3_ctx_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(_P)]),
    "p3_ctx_destroy": (ctypes.c_int, [_P]),
    "p3_ctx_ipc_handle": (ctypes.c_int, [_P, _U32, _P]),
    "p3_ctx_open_peers": (ctypes.c_int, [_P, _P]),
    "p3_ctx_export_fd": (ctypes.c_int, [_P, _U32, ctypes.POINTER(ctypes.c_int)]),
    "p3_ctx_open_peers_fd": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
    "p3_nvls_create": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
    "p3_nvls_attach": (ctypes.c_int, [_P, ctypes.c_int]),
    "p3_nvls_bind": (ctypes.c_int, [_P]),
    "p3_ctx_params": (ctypes.c_int, [_P, _U32, ctypes.POINTER(_P)]),
    "p3_ctx_layer_offset": (ctypes.c_int, [_P, _U32, _PU64]),
    "p3_ctx_grads": (ctypes.c_int, [_P, _U32, ctypes.POINTER(_P)]),
    "p3_iteration_begin": (ctypes.c_int, [_P, _U64, _P]),
    "p3_iteration_end": (ctypes.c_int, [_P, _U64]),
    "p3_comm_launches": (ctypes.c_int, [_P, _PU64]),
    "p3_layer_ready": (ctypes.c_int, [_P, _U32, _U32, _U64, _P, _P]),
    "p3_gradgen_layer": (ctypes.c_int, [_P, _U32, _U64, _U64, _U32, _P]),
    "p3_wait_layer": (ctypes.c_int, [_P, _U32, _U32, _U64, _P]),
    "p3_wait_group": (ctypes.c_int, [_P, _U32, _U32, _U64, _P]),
    "p3_sync_all": (ctypes.c_int, [_P, _U64, ctypes.c_double]),
    "p3_trace_read": (ctypes.c_int, [_P, _U32, ctypes.POINTER(TraceRec), _U64, _PU64]),
    "p3_trace_clear": (ctypes.c_int, [_P]),
    "p3_apply_slice": (ctypes.c_int, [_P, _U32, _U32, _U32, _P, _U64, _P]),
    "p3_master_init": (ctypes.c_int, [_P, _U32, _P]),
    "p3_layer_flag": (ctypes.c_int, [_P, _U32, _U32, _PU64]),
    "p3_fq_create": (ctypes.c_int, [_U32, ctypes.POINTER(_P)]),
    "p3_fq_put_batch": (ctypes.c_int, [_P, _PU64, _PU64, _U64]),
    "p3_fq_poll": (ctypes.c_int, [_P, _PU64]),
    "p3_fq_size": (_U64, [_P]),
    "p3_fq_snapshot": (ctypes.c_int, [_P, _PU64, _U64, _PU64]),
    "p3_fq_destroy": (ctypes.c_int, [_P]),
    "p3_trace_mark": (ctypes.c_int, [_P, _U32, _U64, _U32, _P]),
    "p3_counters": (ctypes.c_int, [_P, _U32, _PU64, _PU64]),
    "p3_debug_snapshot": (ctypes.c_int, [_P, _U32, _PU32, _U64, _PU64]),
    "p3_last_error": (ctypes.c_char_p, [_P]),
    "p3_device_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)] * 4),
    "p3_frame_encode": (ctypes.c_int, [ctypes.POINTER(FrameT), _P, _P, _U64, _PU64]),
    "p3_frame_decode": (ctypes.c_int, [_P, _U64, _U64, ctypes.POINTER(FrameT), _PU64]),
    "p3_frames_pack": (ctypes.c_int, [_P, _P, _P, _U32, _P, _P]),
    "p3_frames_unpack": (ctypes.c_int, [_P, _P, _U32, _U64, _P, _P, _P, _P]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libp3.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("P3_LIB") or LIB_PATH)
    if not path.exists():
        raise RuntimeError(
            f"{path} is missing: build the sm_100a extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = ctypes.CDLL(str(path))
    variant = bool(os.environ.get("P3_LIB"))  # an experiment build (older variants may lack newer entries)
    for name, (res, args) in SIGNATURES.items():
        if variant and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class P3Error(RuntimeError):
    """A libp3 call failed; ``code`` is the P3_* return code."""

    def __init__(self, code: int, msg: str) -> None:
        super().__init__(msg)
        self.code = code


def last_error(ctx=None) -> str:
    raw = load().p3_last_error(ctx)
    return raw.decode() if raw else ""


def check(rc: int, ctx=None, what: str = "") -> None:
    """Map a P3_* return code onto the reference's exception types."""
    if rc == P3_OK:
        return
    msg = last_error(ctx) or f"libp3 error {rc}"
    if what:
        msg = f"{what}: {msg}"
    # imported lazily: these modules import this one
    if rc == P3_EUSAGE:
        from .plan import PlanError

        raise PlanError(msg)
    if rc == P3_EPROTOCOL:
        from .proto import ProtocolError

        raise ProtocolError(msg)
    if rc == P3_ETIMEOUT:
        from .queues import DeadlockError

        raise DeadlockError(msg)
    raise P3Error(rc, msg)


def u64_array(values) -> ctypes.Array:
    vals = list(values)
    return (ctypes.c_uint64 * max(len(vals), 1))(*vals)


def stream_handle(stream=None) -> int:
    """Raw cudaStream_t of a torch stream (current stream when None)."""
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)
