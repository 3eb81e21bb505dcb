"""Per-variant P3 step time (torchrun, N ranks): isolates publication/drain/gate settings."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1905_03960_b200.ddp import P3DataParallel, _HookedDataParallel
from paper_1905_03960_b200.torch_models import build_model, synthetic_batch, loss_fn
world = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
if world > 1: dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
name = sys.argv[1]; B = int(sys.argv[2])
x, y = synthetic_batch(name, B, seed=1 + rank)
def model():
    torch.manual_seed(0); m = build_model(name).cuda()
    return m.to(memory_format=torch.channels_last) if name != "seq2seq" else m
variants = {
    "default": {},
    "nosync": {},
    "pub0": {"pub_batch_bytes": 0},
    "drain0": {"drain_bytes": 0},
    "pub0_drain0": {"pub_batch_bytes": 0, "drain_bytes": 0},
    "drain64M": {"drain_bytes": 64 << 20},
    "ctas32": {"comm_ctas": 32},
    "linger0": {"drain_linger_us": 0},
    "t256c16": {"comm_threads": 256, "comm_ctas": 16},
    "t128c32": {"comm_threads": 128, "comm_ctas": 32},
    "t128c16": {"comm_threads": 128, "comm_ctas": 16},
    "t256c32": {"comm_threads": 256, "comm_ctas": 32},
    "linger1000": {"drain_linger_us": 1000},
    "fin148": {"finish_ctas": 148},
    "fin148_linger0": {"finish_ctas": 148, "drain_linger_us": 0},
    "fin64_linger1000": {"finish_ctas": 64, "drain_linger_us": 1000},
}
for vn in sys.argv[3].split(","):
    kw = dict(variants[vn.replace("+layergate", "")])
    d = P3DataParallel(model(), lr=0.01, **kw)
    if vn == "nosync":  # diagnostic: no comm kernel work at all (gates pass, nothing published)
        d.ctx.iteration_begin = lambda k, stream=None: None
        d.ctx.iteration_end = lambda k: None
        d.ctx.layer_ready = lambda *a, **k: None
        d._gate = lambda l: None
        d.ctx.wait_group = lambda *a, **k: None
        d.synchronize = lambda *a, **k: torch.cuda.synchronize()
    if vn.endswith("+layergate"):
        d._make_gate = lambda layers: _HookedDataParallel._make_gate(d, layers)
        d.remove_hooks(); d._install()
    for _ in range(4): loss_fn(name, d, x, y).backward()
    d.synchronize(); torch.cuda.synchronize()
    a0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    if world > 1: dist.barrier()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record()
    for _ in range(6): loss_fn(name, d, x, y).backward()
    d.synchronize(); e.record(); torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / 6], device="cuda")
    if world > 1: dist.all_reduce(t, op=dist.ReduceOp.MAX)
    a1 = torch.cuda.memory_stats().get("num_device_alloc", 0)
    if rank == 0 and vn != "nosync":
        sn = d.ctx.debug_snapshot(0)
        print("STATS", vn, {k2: sn[k2] for k2 in ("pushed", "reduced", "jobs", "t_pick_ns", "t_slot_wait_ns", "t_move_ns", "t_signal_ns")}, flush=True)
    if rank == 0: print("VARIANT", vn, round(float(t.item()), 3), "ms/step", d.ctx.launches(), "launches", a1 - a0, "cudaMallocs", flush=True)
    d.close(); del d; torch.cuda.empty_cache()
if world > 1: dist.destroy_process_group()
