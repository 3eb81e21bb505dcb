"""Sync-only timeline at N>1 (torchrun): every rank's gradients resident and published, one
FINISH launch; rank 0's device trace (P3_TRACE_CTA=1: trace rank field = CTA index) gives
when pushes are popped and reduces broadcast, and when each CTA finishes.
torchrun --nproc-per-node 2 tools/exp_timeline_mp.py resnet50"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_1905_03960_b200.runtime import SyncContext
from paper_1905_03960_b200.torch_models import real_counts


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    m = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    extra = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
    counts = real_counts(m)
    ctx = SyncContext(counts, world, [rank], comm_ctas=148, comm_threads=512, timeout_s=30.0, emulate_grads=True,
                      trace_cap=1 << 18, **extra)
    hs = [None] * world
    dist.all_gather_object(hs, ctx.ipc_handle(0))
    ctx.open_peers(hs)
    st = torch.cuda.Stream()
    for l in range(len(counts)):
        ctx.gradgen_layer(0, 7 + rank, 0, l, st)
    st.synchronize()
    for k in range(4):
        for l in range(len(counts)):
            ctx.layer_ready(0, l, k, None, st)
        st.synchronize()
        ctx.clear_trace()
        dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(st):
            torch.cuda._sleep(200_000)
        ctx.iteration_begin(k, st)
        s.record(st)
        ctx.iteration_end(k)
        e.record(st)
        ctx.sync_all(k + 1, 30.0)
        st.synchronize()
        if k == 3 and os.environ.get("P3_TL_DUMP"):  # raw records of every rank (analysed offline)
            recs = [(r.t_ns, r.t0_ns, r.event, r.layer, r.slice, r.rank) for r in ctx.trace(0) if r.iteration == k]
            with open(os.path.join(os.environ["P3_TL_DUMP"], f"tl_{m}_rank{rank}.json"), "w") as f:
                json.dump(recs, f)
        if rank == 0 and k == 3:
            tr_all = [r for r in ctx.trace(0) if r.iteration == k]
            tr = [r for r in tr_all if r.event in (0, 1)]
            t0 = min(r.t_ns for r in tr_all)
            push = sorted((r.t_ns - t0) / 1e3 for r in tr if r.event == 0)
            bc = sorted((r.t_ns - t0) / 1e3 for r in tr if r.event == 1)
            per = {}
            for r in tr:
                per.setdefault(r.rank, []).append((r.t_ns - t0) / 1e3)
            ends = sorted(max(v) for v in per.values())
            q = lambda a, f: round(a[min(len(a) - 1, int(f * len(a)))], 1) if a else None
            bins = lambda a: [sum(1 for x in a if i * 10 <= x < (i + 1) * 10) for i in range(int(max(a) // 10) + 1)]
            if os.environ.get("P3_TL_DETAIL"):
                late = [r for r in tr if r.event == 0 and (r.t_ns - t0) / 1e3 > 60]
                print("LATE_POPS", len(late), "layers", sorted({r.layer for r in late})[:40], flush=True)
                for c in sorted(per)[:3]:
                    seq = sorted((round((r.t_ns - t0) / 1e3, 1), r.event, r.layer, r.slice) for r in tr_all if r.rank == c)
                    print("CTA", c, seq[:400], flush=True)
                sig = {}
                for r in sorted(tr_all, key=lambda r: r.t_ns):
                    if r.event == 4: sig[r.rank] = r.t_ns
                    elif r.event == 5 and r.rank in sig: sig.setdefault("d", []).append((r.t_ns - sig.pop(r.rank)) / 1e3)
                idle = [r for r in tr_all if r.event == 8]
                if idle:
                    print("IDLE", len(idle), "first/last us", round((min(r.t_ns for r in idle) - t0) / 1e3, 1),
                          round((max(r.t_ns for r in idle) - t0) / 1e3, 1), "pushed seen (min,max)",
                          min(r.layer for r in idle), max(r.layer for r in idle),
                          "idle with pops left", sum(1 for r in idle if r.layer < 643), flush=True)
                    c2 = [(round((r.t_ns - t0) / 1e3, 1), r.layer) for r in sorted(idle, key=lambda r: r.t_ns) if r.rank == 2]
                    print("IDLE_CTA2", c2[:30], flush=True)
                d = sorted(sig.get("d", []))
                if d: print("SIGNAL_US", len(d), [round(d[int(f * (len(d) - 1))], 1) for f in (0, .5, .9, .99, 1)], flush=True)
            print(json.dumps({"model": m, "world": world, "kernel_ms": round(s.elapsed_time(e), 4),
                              "pushes": len(push), "bcasts": len(bc),
                              "push_pop_us_q": [q(push, f) for f in (0, .25, .5, .75, 1)],
                              "bcast_us_q": [q(bc, f) for f in (0, .25, .5, .75, 1)],
                              "cta_end_us_q": [q(ends, f) for f in (0, .1, .5, .9, 1)],
                              "push_per_10us": bins(push), "bcast_per_10us": bins(bc)}), flush=True)
    ctx.close()
    dist.destroy_process_group()


main()
