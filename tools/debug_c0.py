import sys, time, os, threading
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import torch
from paper_1905_03960_b200.model import builtin_profile
from paper_1905_03960_b200.runtime import TrainingWorker, WorkerConfig
variant = sys.argv[1]
world = int(sys.argv[2]); iters = int(sys.argv[3])
cfg = WorkerConfig(rank=0, mode="p3", world=world, iterations=iters, deadlock_timeout=6.0, emulate_compute=True, comm_ctas=16)
w = TrainingWorker(cfg, builtin_profile("resnet50-like"), ranks=list(range(world)))
if variant == "prio":
    w.comm_stream = torch.cuda.Stream(priority=-1)
t = time.time()
try:
    for k in range(iters):
        w.run_iteration(k)
    snap_t = threading.Timer(3.0, lambda: print("snapshot@3s", {k: (v if not isinstance(v, list) else v[:8] + ['...'] + v[-4:]) for k, v in w.ctx.debug_snapshot(0).items()}, flush=True))
    snap_t.start()
    w.wait_all(iters)
    snap_t.cancel()
    print(variant, world, iters, "ok", f"{w.params_digest(0):016x}", time.time() - t, flush=True)
except Exception as e:
    print(variant, world, iters, "FAIL", e, time.time() - t, flush=True)
