"""BASELINE configs[4]: slice-size sweep x link-throttle sweep, P3 vs layer-wise FIFO on the
same comm kernel. torchrun --nproc-per-node N tools/sweep.py MODEL [BATCH] [SLICES] [GBPS]
Rank 0 prints one `SWEEP {...}` JSON line per point (samples/s, max over ranks)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1905_03960_b200.ddp import P3DataParallel
from paper_1905_03960_b200.torch_models import build_model, synthetic_batch, loss_fn

def main():
    world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    name = sys.argv[1]
    B = (int(sys.argv[2]) if len(sys.argv) > 2 else 0) or {"resnet50": 256, "vgg19": 128, "seq2seq": 128}[name]
    slices = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "1000,10000,50000,100000,1000000").split(",")]
    rates = [float(v) for v in (sys.argv[4] if len(sys.argv) > 4 else "10,25,0").split(",")]
    x, y = synthetic_batch(name, B, seed=7 + rank)
    torch.manual_seed(0)
    model = build_model(name).cuda()
    if name != "seq2seq":
        model = model.to(memory_format=torch.channels_last)
    base = {k: v.detach().clone() for k, v in model.state_dict().items()}

    def measure(**kw):
        model.load_state_dict(base)
        d = P3DataParallel(model, lr=0.01, comm_ctas=8, pub_batch_bytes=0, timeout_s=300.0, **kw)
        rate = kw.get("throttle_bps", 0)
        steps = 6 if rate and rate < 50e9 else 10
        for _ in range(3):
            loss_fn(name, d, x, y).backward()
        d.synchronize(); torch.cuda.synchronize()
        if world > 1: dist.barrier()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record()
        for _ in range(steps):
            loss_fn(name, d, x, y).backward()
        d.synchronize(); e.record(); torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / steps], device="cuda")
        if world > 1: dist.all_reduce(t, op=dist.ReduceOp.MAX)
        d.close()
        return float(t.item())

    for gbps in rates:
        thr = gbps * 1e9
        ms_lw = measure(plan_mode="baseline", priority_mode=False, throttle_bps=thr)
        for ms_ in slices:
            ms_p3 = measure(max_slice=ms_, throttle_bps=thr)
            if rank == 0:
                print("SWEEP " + json.dumps({
                    "model": name, "world": world, "per_gpu_batch": B, "link_gbps": gbps or "nvlink",
                    "max_slice": ms_, "p3_ms_per_step": round(ms_p3, 3), "layerwise_fifo_ms_per_step": round(ms_lw, 3),
                    "p3_samples_s": round(B * world / ms_p3 * 1e3, 1), "layerwise_samples_s": round(B * world / ms_lw * 1e3, 1),
                    "p3_speedup": round(ms_lw / ms_p3, 3)}), flush=True)
    if world > 1:
        dist.destroy_process_group()

main()
