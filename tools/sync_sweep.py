"""Sync-only comm-kernel timing over NVLink: every rank's gradients resident and published,
one FINISH launch per iteration; max over ranks. torchrun --nproc-per-node N tools/sync_sweep.py"""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1905_03960_b200.runtime import SyncContext, connect
from paper_1905_03960_b200.torch_models import real_counts

def main():
    world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    models = sys.argv[1].split(",") if len(sys.argv) > 1 else ["resnet50", "vgg19", "seq2seq"]
    ctas_list = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148]
    slices = [int(c) for c in sys.argv[3].split(",")] if len(sys.argv) > 3 else [50_000]
    threads = int(sys.argv[4]) if len(sys.argv) > 4 else 512
    extra = json.loads(sys.argv[5]) if len(sys.argv) > 5 else {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sweep = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")  # retires the flush's dirty lines (bench.py)
    rows = []
    for m in models:
        if m.endswith("-notiny"):  # experiment: the model without its layers under 8K parameters
            counts = [c for c in real_counts(m[:-7]) if c >= 8192]
        elif m.endswith("-merged"):  # experiment: tiny layers merged into runs of >= 8K parameters
            counts, acc = [], 0
            for c in real_counts(m[:-7]):
                if c >= 8192:
                    if acc: counts.append(acc); acc = 0
                    counts.append(c)
                else:
                    acc += c
                    if acc >= 8192: counts.append(acc); acc = 0
            if acc: counts.append(acc)
        else:
            counts = real_counts(m)
        P = sum(counts)
        for ms in slices:
            for ctas in ctas_list:
                ctx = SyncContext(counts, world, [rank], max_slice=ms, comm_ctas=ctas, comm_threads=threads,
                                  timeout_s=60.0, emulate_grads=True, **extra)
                if world > 1:
                    connect(ctx)  # (CUDA IPC, or fd + multicast with extra {"nvls": true})
                st = torch.cuda.Stream()
                for l in range(len(counts)): ctx.gradgen_layer(0, 7 + rank, 0, l, st)
                st.synchronize()
                ts = []
                for k in range(8):
                    with torch.cuda.stream(st): flush.fill_(k); sweep.sum(dtype=torch.int32)
                    for l in range(len(counts)): ctx.layer_ready(0, l, k, None, st)
                    st.synchronize()
                    if world > 1: dist.barrier()
                    torch.cuda.synchronize()
                    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                    with torch.cuda.stream(st):
                        torch.cuda._sleep(200_000)  # the host enqueues the launch ahead of the GPU
                        if world > 1: dist.all_reduce(torch.zeros(1, device="cuda"))  # ranks aligned on the device
                    ctx.iteration_begin(k, st); s.record(st); ctx.iteration_end(k); e.record(st)
                    try:
                        ctx.sync_all(k + 1, 20.0)
                    except Exception as ex:
                        d = ctx.debug_snapshot(0)
                        from paper_1905_03960_b200.plan import make_p3_plan
                        from paper_1905_03960_b200.model import ModelProfile, LayerSpec
                        plan = make_p3_plan(ModelProfile("x", 0, tuple(LayerSpec(i, "l", c, 0, 0) for i, c in enumerate(counts))), world, ms)
                        bad = [l for l in range(len(counts)) if d["done"][l] < (k + 1) * len(plan.slices_of_layer(l))]
                        print(f"HANG rank {rank} k {k} ctas {ctas}: {ex}", flush=True)
                        print(f"HANG rank {rank} pushed {d['pushed']} reduced {d['reduced']} exited {d['exited']} jobs {d['jobs']}", flush=True)
                        for l in bad[:3] + [32]:
                            sl = plan.slices_of_layer(l); first = plan.slices.index(sl[0])
                            print(f"HANG rank {rank} layer {l}: done {d['done'][l]} hint {d['hint'][l]} taken {d['srv_taken'][l]} cursor {d['cursor'][l]} tag {d['ready'][l]}", flush=True)
                            print(f"HANG rank {rank}   slices(owner,arr,claim): " + " ".join(f"{s.server},{d['arrivals'][first+i]},{d['claim'][first+i]}" for i, s in enumerate(sl)), flush=True)
                        from collections import Counter
                        ph = d["cta_phase"][:ctas]
                        print(f"HANG rank {rank} phases {Counter((p >> 20) & 0xf for p in ph)} {[hex(p) for p in ph if (p >> 20) & 0xf != 5][:8]}", flush=True)
                        raise
                    st.synchronize()
                    t = torch.tensor([s.elapsed_time(e)], device="cuda")
                    if world > 1: dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    if k >= 2: ts.append(float(t.item()))
                ms_ = statistics.mean(ts)
                dsn = ctx.debug_snapshot(0)
                jobs = max(dsn["jobs"], 1)
                stats = {k2: round(dsn[k2] / jobs / 1000, 2) for k2 in ("t_pick_ns", "t_slot_wait_ns", "t_move_ns", "t_signal_ns")}
                stats["jobs"] = dsn["jobs"]
                stats["exited"] = dsn["exited"]
                nvl = 2 * (world - 1) / world * P * 4 / (ms_ * 1e-3) / 1e9 if world > 1 else None
                hbm = 12 * P / (ms_ * 1e-3) / 1e9 if world == 1 else None
                rows.append({"extra": extra, "model": m, "world": world, "max_slice": ms, "ctas": ctas, "threads": threads, "ms": round(ms_, 4),
                             "nvlink_GBps": nvl and round(nvl, 1), "hbm_GBps": hbm and round(hbm, 1), "us_per_job": stats})
                ctx.close()
                if world > 1: dist.barrier()
    if rank == 0:
        for r in rows: print("SWEEP " + json.dumps(r), flush=True)
    if world > 1: dist.destroy_process_group()

main()
