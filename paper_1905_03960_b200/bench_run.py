"""``p3sync bench`` on one GPU: a whole emulated world, its output files and summary.json.

The reference's bench (cli.py:241-376) spawns N server and N worker processes over loopback
TCP, then summarises their output files. Here all N ranks run as one TrainingWorker on one
GPU (emulate mode: device-sleep compute, K1 GradGen gradients, the comm kernel for the
sync), and the run leaves the same files in ``output_dir``:

  throughput_worker{r}.csv   iteration,wall_ms,start_ms   (device-clock ITER_START marks)
  net_util_worker{r}.csv     t_ms,bytes_in,bytes_out      (10 ms buckets of the trace)
  digest_worker{r}.txt       FNV-1a of rank r's parameters (worker.py:372-376)
  params_worker0.bin         rank 0's parameters, fp32 LE, layer order (worker.py:378-379)
  digest_server{r}.csv       layer,slice,offset,len,digest of every slice rank r owns
                             (ServerEngine.digests_csv, server.py:283-292)
  summary.json               the schema of cli.py:361-375

``summarize_run`` reads those files back like cli.py:331-376 does: digests must agree,
samples/s = measured iterations x batch x workers / the longest worker window, idle
fraction of worker 0's link over the post-warm-up window, and every server slice digest
checked against worker 0's parameter dump (cli.py:379-398).
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, fields
from pathlib import Path

import numpy as np

from .hashing import fnv1a64
from .metrics import (
    clip_samples,
    idle_fraction,
    iteration_starts_from_csv,
    iteration_timeline,
    iterations_from_csv,
    iterations_to_csv,
    samples_from_csv,
    samples_from_trace,
    samples_to_csv,
    throughput,
    write_text,
)
from .model import ModelProfile, resolve_profile
from .plan import DEFAULT_MAX_SLICE, P3_MODE
from .proto import ProtocolError


@dataclass
class RunConfig:
    """RunConfig of cli.py:61-82 (same field names and defaults) plus the device knobs."""

    mode: str = P3_MODE
    profile: str = "toy3"
    num_workers: int = 2
    num_servers: int = 0  # 0 -> num_workers; the device path has one server per worker
    max_slice: int = DEFAULT_MAX_SLICE
    big_threshold: int = 1_000_000
    lr: float = 0.1
    iterations: int = 10
    batch_size: int = 32
    throttle_rate: float = 0.0  # bit/s per rank egress; 0 disables shaping
    throttle_burst: int = 50 * 1024
    seed: int = 0
    output_dir: str = "bench-out"
    skip_iterations: int = 5
    idle_threshold: int = 4096
    timeout: float = 240.0
    dump_params: bool = True
    comm_ctas: int = 16
    strict_order: bool = False

    def resolved_servers(self) -> int:
        return self.num_servers if self.num_servers > 0 else self.num_workers

    @classmethod
    def from_json(cls, text: str, **overrides) -> "RunConfig":
        raw = json.loads(text)
        unknown = set(raw) - {f.name for f in fields(cls)}
        if unknown:
            raise ValueError(f"unknown config keys: {sorted(unknown)}")  # cli.py:89-92
        return cls(**{**raw, **{k: v for k, v in overrides.items() if v is not None}})


def server_digests_csv(worker, li: int) -> str:
    """digests_csv (server.py:283-292) of local rank ``li`` as a server: FNV-1a of every slice
    it owns, in key order, read from its parameter replica (the owner's copy is the master)."""
    rank = worker.ranks[li]
    params = worker.params(li)
    rows = ["layer,slice,offset,len,digest"]
    for s in sorted(worker.plan.slices_on_server(rank), key=lambda s: (s.key.layer_index, s.key.slice_index)):
        blob = params[s.key.layer_index][s.offset : s.offset + s.length].astype("<f4").tobytes()
        rows.append(f"{s.key.layer_index},{s.key.slice_index},{s.offset},{s.length},{fnv1a64(blob):016x}")
    return "\n".join(rows) + "\n"


def verify_server_digests(profile: ModelProfile, servers: int, outdir: Path, blob: bytes) -> int:
    """Every server slice digest against the same bytes of worker 0's parameter dump
    (cli.py:379-398); returns the number of slices checked, ProtocolError on a mismatch."""
    base = np.cumsum([0] + [l.param_count for l in profile.layers])
    checked = 0
    for r in range(servers):
        for line in (outdir / f"digest_server{r}.csv").read_text().splitlines()[1:]:
            layer, sl, offset, length, digest = line.split(",")
            lo = 4 * (int(base[int(layer)]) + int(offset))
            want = f"{fnv1a64(blob[lo : lo + 4 * int(length)]):016x}"
            if want != digest:
                raise ProtocolError(f"server {r} slice {layer}/{sl} digest {digest} != worker-side {want}")
            checked += 1
    return checked


def run_bench(cfg: RunConfig, profile: ModelProfile | None = None) -> dict:
    """Run the emulated world on the current GPU, write the output files, summarise."""
    from .runtime import TrainingWorker, WorkerConfig

    if cfg.resolved_servers() != cfg.num_workers:
        raise ValueError("the device path runs one server per worker (num_servers == num_workers)")
    profile = profile or resolve_profile(cfg.profile)
    outdir = Path(cfg.output_dir)
    N = cfg.num_workers
    S_est = sum(-(-l.param_count // cfg.max_slice) + N for l in profile.layers)
    wcfg = WorkerConfig(rank=0, mode=cfg.mode, servers=N, iterations=cfg.iterations, lr=cfg.lr,
                        batch_size=cfg.batch_size, throttle_rate=cfg.throttle_rate or None,
                        throttle_burst=cfg.throttle_burst, deadlock_timeout=cfg.timeout, max_slice=cfg.max_slice,
                        emulate_compute=True, comm_ctas=cfg.comm_ctas,
                        trace_cap=cfg.iterations * (6 * S_est + profile.num_layers + 8) + 64,
                        big_threshold=cfg.big_threshold, seed=cfg.seed, strict_order=cfg.strict_order)
    w = TrainingWorker(wcfg, profile, ranks=list(range(N)))
    try:
        w.run()
        traces = {li: w.ctx.trace(li) for li in range(N)}
        for li in range(N):
            if len(traces[li]) >= w.ctx.trace_cap:
                raise RuntimeError("trace ring overflowed")
        origin = min(e.t_ns for recs in traces.values() for e in recs if e.event == 5)  # first ITER_START
        end = max(e.t_ns for recs in traces.values() for e in recs)
        for li in range(N):
            walls, starts = iteration_timeline(traces[li], origin)
            write_text(outdir / f"throughput_worker{li}.csv", iterations_to_csv(walls, starts))
            write_text(outdir / f"net_util_worker{li}.csv",
                       samples_to_csv(samples_from_trace(traces, w.plan, li, origin, end)))
            write_text(outdir / f"digest_worker{li}.txt", f"{w.params_digest(li):016x}\n")
            write_text(outdir / f"digest_server{li}.csv", server_digests_csv(w, li))
        if cfg.dump_params:
            (outdir / "params_worker0.bin").write_bytes(b"".join(v.astype("<f4").tobytes() for v in w.params(0)))
    finally:
        w.close()
    return summarize_run(cfg, outdir, profile)


def summarize_run(cfg: RunConfig, outdir: Path, profile: ModelProfile) -> dict:
    """summary.json (cli.py:331-376) from the files of a run."""
    outdir = Path(outdir)
    digests, windows = [], []
    walls0 = starts0 = None
    for r in range(cfg.num_workers):
        digests.append((outdir / f"digest_worker{r}.txt").read_text().strip())
        text = (outdir / f"throughput_worker{r}.csv").read_text()
        walls = iterations_from_csv(text)
        if r == 0:
            walls0, starts0 = walls, iteration_starts_from_csv(text)
        windows.append(throughput(walls, cfg.batch_size, cfg.num_workers, cfg.skip_iterations).window_seconds)
    if len(set(digests)) != 1:
        raise ProtocolError(f"worker digests disagree: {digests}")
    rate = (len(walls0) - cfg.skip_iterations) * cfg.batch_size * cfg.num_workers / max(windows)
    samples = samples_from_csv((outdir / "net_util_worker0.csv").read_text())
    window = clip_samples(samples, starts0[cfg.skip_iterations], starts0[-1] + walls0[-1])
    idle = idle_fraction(window if len(window) >= 2 else samples, cfg.idle_threshold)
    dump = outdir / "params_worker0.bin"
    checked = verify_server_digests(profile, cfg.resolved_servers(), outdir, dump.read_bytes()) if dump.exists() else 0
    summary = {
        "mode": cfg.mode,
        "profile": profile.name,
        "num_workers": cfg.num_workers,
        "num_servers": cfg.resolved_servers(),
        "iterations": cfg.iterations,
        "batch_size": cfg.batch_size,
        "skip_iterations": cfg.skip_iterations,
        "idle_threshold": cfg.idle_threshold,
        "samples_per_second": rate,
        "idle_fraction": idle,
        "digest": digests[0],
        "server_slices_verified": checked,
    }
    write_text(outdir / "summary.json", json.dumps(summary, indent=2) + "\n")
    return summary


def main(argv=None) -> int:
    """``python -m paper_1905_03960_b200.bench_run [config.json] [--key value ...]``."""
    import sys

    args = list(sys.argv[1:] if argv is None else argv)
    text = "{}"
    if args and not args[0].startswith("--"):
        text = Path(args.pop(0)).read_text()
    over = {}
    types = {f.name: f.type for f in fields(RunConfig)}
    while args:
        k = args.pop(0).lstrip("-").replace("-", "_")
        v = args.pop(0)
        t = types.get(k)
        over[k] = v if t in ("str",) else (v.lower() in ("1", "true") if t == "bool" else (float(v) if t == "float" else int(v)))
    print(json.dumps(run_bench(RunConfig.from_json(text, **over)), indent=2))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
