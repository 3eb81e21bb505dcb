"""Timeline of one sync-only FINISH launch at N=1 from the device trace (pick = PUSH event,
signal = BCAST event, %globaltimer ns): when the first / median / last jobs complete, the
bytes completed per 5 us bin, and the kernel's event-timed duration.
python tools/exp_timeline.py resnet50 '{"pop_relax":148}'"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1905_03960_b200.runtime import SyncContext
from paper_1905_03960_b200.torch_models import real_counts
from paper_1905_03960_b200.plan import make_p3_plan
from paper_1905_03960_b200.model import ModelProfile, LayerSpec


def main():
    m = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    counts = [1024] if m == "tiny" else real_counts(m)
    plan = make_p3_plan(ModelProfile("x", 0, tuple(LayerSpec(i, "l", c, 0, 0) for i, c in enumerate(counts))), 1, 50_000)
    first = {}
    for i, s in enumerate(plan.slices):
        first.setdefault(s.key.layer_index, i)
    lens = [s.length for s in plan.slices]
    ctx = SyncContext(counts, 1, [0], comm_ctas=148, comm_threads=512, timeout_s=30.0, emulate_grads=True,
                      trace_cap=1 << 16, **extra)
    st = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush2 = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
    for l in range(len(counts)):
        ctx.gradgen_layer(0, 7, 0, l, st)
    st.synchronize()
    for k in range(4):
        with torch.cuda.stream(st):
            flush.fill_(k)
            if os.environ.get("P3_CLEAN_FLUSH"):
                torch.sum(flush2, dtype=torch.int64)  # read pass: the L2 ends clean
        for l in range(len(counts)):
            ctx.layer_ready(0, l, k, None, st)
        st.synchronize()
        ctx.clear_trace()
        s, e, s1 = torch.cuda.Event(True), torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(st):
            torch.cuda._sleep(200_000)  # the host enqueues everything below before the GPU gets there
        s.record(st)
        ctx.iteration_begin(k, st)
        s1.record(st)
        ctx.iteration_end(k)
        e.record(st)
        ctx.sync_all(k + 1, 30.0)
        st.synchronize()
        tr_all = [r for r in ctx.trace(0) if r.iteration == k]
        starts_ev = [r.t_ns for r in tr_all if r.event == 16]
        exits_ev = [r.t_ns for r in tr_all if r.event == 17]
        tr = [r for r in tr_all if r.event in (0, 1)]
        picks = sorted(r.t_ns for r in tr if r.event == 0)
        sig = sorted((r.t_ns, lens[first[r.layer] + r.slice]) for r in tr if r.event == 1)
        t0 = picks[0]
        tot = sum(b for _, b in sig)
        bins = {}
        for t, n in sig:
            bins[(t - t0) // 5000] = bins.get((t - t0) // 5000, 0) + n
        if os.environ.get("P3_TRACE_CTA") and k == 3:
            per = {}
            for r in tr:
                per.setdefault(r.rank, []).append((r.t_ns - t0, r.event, lens[first[r.layer] + r.slice]))
            ends = sorted(max(t for t, ev, _ in v) for v in per.values())
            starts = sorted(min(t for t, ev, _ in v) for v in per.values())
            busy_elems = sorted(sum(n for _, ev, n in v if ev == 1) for v in per.values())
            njobs = sorted(sum(1 for _, ev, _ in v if ev == 1) for v in per.values())
            q = lambda a, f: round(a[min(len(a) - 1, int(f * len(a)))] / 1e3, 1)
            print("CTA", json.dumps({"ctas": len(per), "first_pick_us": [q(starts, 0), q(starts, .5), q(starts, 1)],
                                     "last_signal_us": [q(ends, 0), q(ends, .1), q(ends, .5), q(ends, .9), q(ends, 1)],
                                     "elems_per_cta_M": [round(busy_elems[0] / 1e6, 3), round(busy_elems[len(busy_elems) // 2] / 1e6, 3), round(busy_elems[-1] / 1e6, 3)],
                                     "jobs_per_cta": [njobs[0], njobs[len(njobs) // 2], njobs[-1]]}), flush=True)
            # SM-time accounting: the share of (CTAs x span) each CTA spends after its last signal
            # (tail), and each CTA's element rate between its first pick and its last signal
            span = max(ends) - min(starts)
            tail = sum(max(ends) - max(t for t, ev, _ in v) for v in per.values()) / (len(per) * span)
            rates = sorted(sum(n for _, ev, n in v if ev == 1) * 12 / max(1, (max(t for t, ev, _ in v) - min(t for t, ev, _ in v))) for v in per.values())
            print("SMTIME", json.dumps({"span_us": round(span / 1e3, 1), "tail_share": round(tail, 3),
                                        "GBps_per_cta_p10_p50_p90": [round(rates[int(f * (len(rates) - 1))], 1) for f in (.1, .5, .9)]}), flush=True)
            # the CTA that finished last: its job sequence
            last = max(per, key=lambda c: max(t for t, ev, _ in per[c]))
            print("LAST", [(round(t / 1e3, 1), ev, n) for t, ev, n in sorted(per[last])], flush=True)
        if starts_ev:
            print("EDGES", json.dumps({"first_cta_start_to_first_pick_us": round((t0 - min(starts_ev)) / 1e3, 2),
                                       "cta_start_spread_us": round((max(starts_ev) - min(starts_ev)) / 1e3, 2),
                                       "last_signal_to_last_exit_us": round((max(exits_ev) - max(t for t, _ in sig)) / 1e3, 2),
                                       "first_start_to_last_exit_us": round((max(exits_ev) - min(starts_ev)) / 1e3, 2)}))
        print(json.dumps({"model": m, "k": k, "event_ms": round(s.elapsed_time(e), 4), "launch_ms": round(s1.elapsed_time(e), 4), "jobs": len(sig),
                          "first_pick_to_last_signal_us": round((sig[-1][0] - t0) / 1e3, 1),
                          "first_signal_us": round((sig[0][0] - t0) / 1e3, 1),
                          "half_bytes_us": round((next(t for t, c in _cum(sig) if c >= tot / 2) - t0) / 1e3, 1),
                          "p90_bytes_us": round((next(t for t, c in _cum(sig) if c >= 0.9 * tot) - t0) / 1e3, 1),
                          "elems_per_5us_bin_M": [round(bins.get(i, 0) / 1e6, 2) for i in range(max(bins) + 1)]}),
              flush=True)
    ctx.close()


def _cum(sig):
    c = 0
    for t, n in sig:
        c += n
        yield t, c


main()
