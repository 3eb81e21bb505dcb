"""Multi-process P3 check, one process per GPU (launched by tests/test_multigpu.py under
torchrun). Emulate-mode digests vs the reference goldens, then torch-mode training parity."""

import json
import os
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    golden = json.loads((REPO / "tests" / "golden" / "golden.json").read_text())
    out = {"rank": rank, "world": world, "digests": {}, "errors": []}

    from paper_1905_03960_b200.model import builtin_profile
    from paper_1905_03960_b200.runtime import SyncContext, TrainingWorker, WorkerConfig

    want = {(d[0], d[1], d[4]): d[5] for d in golden["digests"] if d[2] in (10, 4)}
    for name in ("toy3", "resnet50-like", "vgg19-like", "sockeye-like"):
        for kind, iters in (("same", 10), ("distinct", 4)):
            if (name, world, kind) not in want:
                continue
            prof = builtin_profile(name)
            cfg = WorkerConfig(rank=rank, mode="p3", world=world, iterations=iters, deadlock_timeout=60.0,
                               emulate_compute=kind == "same", comm_ctas=16, rank_distinct_grads=kind == "distinct",
                               trace_cap=20_000)
            ctx = SyncContext(prof.param_counts(), world, [rank], lr=cfg.lr, comm_ctas=16, timeout_s=60.0,
                              emulate_grads=True, trace_cap=20_000)
            hs = [None] * world
            dist.all_gather_object(hs, ctx.ipc_handle(0))
            ctx.open_peers(hs)
            dist.barrier()
            w = TrainingWorker(cfg, prof, ranks=[rank], ctx=ctx)
            try:
                w.run()
                got = f"{w.params_digest(0):016x}"
            except Exception as e:  # noqa: BLE001
                got = f"error: {e}"
            out["digests"][f"{name}/{kind}"] = [got, want[(name, world, kind)]]
            dist.barrier()
            w.close()

    # full ResNet-50 shapes over NVLink, rank-distinct gradients, 148-CTA FINISH launches:
    # every replica equals the oracle's replay (computed once, on rank 0)
    sys.path.insert(0, str(REPO / "oracle"))
    import p3_oracle as O
    from paper_1905_03960_b200.model import LayerSpec, ModelProfile
    from paper_1905_03960_b200.torch_models import real_counts

    counts = real_counts("resnet50")
    prof = ModelProfile("resnet50", 1905, tuple(LayerSpec(i, f"t{i}", c, 0, 0) for i, c in enumerate(counts)))
    cfg = WorkerConfig(rank=rank, mode="p3", world=world, iterations=2, deadlock_timeout=60.0, emulate_compute=False,
                       comm_ctas=148, rank_distinct_grads=True)
    ctx = SyncContext(counts, world, [rank], lr=cfg.lr, comm_ctas=148, timeout_s=60.0, emulate_grads=True)
    hs = [None] * world
    dist.all_gather_object(hs, ctx.ipc_handle(0))
    ctx.open_peers(hs)
    dist.barrier()
    w = TrainingWorker(cfg, prof, ranks=[rank], ctx=ctx)
    try:
        w.run()
        got = f"{w.params_digest(0):016x}"
    except Exception as e:  # noqa: BLE001
        got = f"error: {e}"
    ref = [f"{O.digest(O.replay_params(counts, 1905, world, 2, cfg.lr, distinct=True)):016x}" if rank == 0 else None]
    dist.broadcast_object_list(ref, src=0)
    out["digests"]["resnet50-real/distinct"] = [got, ref[0]]
    dist.barrier()
    w.close()

    # NVLS multicast broadcasts (one multimem.st per element reaches every replica; arenas
    # shared by file descriptor): the same digests, where the GPUs support multicast objects
    from paper_1905_03960_b200.runtime import connect

    out["nvls"] = "ok"
    for name, kind, iters, counts_, seed in (("resnet50-like", "distinct", 4, None, None),
                                              ("vgg19-like", "same", 10, None, None),
                                              ("resnet50-real", "distinct", 2, counts, 1905)):
        if counts_ is None and (name, world, kind) not in want:
            continue
        prof = builtin_profile(name) if counts_ is None else ModelProfile(name, seed, tuple(
            LayerSpec(i, f"t{i}", c, 0, 0) for i, c in enumerate(counts_)))
        ctas = 148 if counts_ is not None else 16
        cfg = WorkerConfig(rank=rank, mode="p3", world=world, iterations=iters, deadlock_timeout=60.0,
                           emulate_compute=kind == "same", comm_ctas=ctas, rank_distinct_grads=kind == "distinct")
        try:
            ctx = SyncContext(prof.param_counts(), world, [rank], lr=cfg.lr, comm_ctas=ctas, timeout_s=60.0,
                              emulate_grads=True, nvls=True)
        except Exception as e:  # noqa: BLE001  (no multicast support on this box)
            out["nvls"] = f"unavailable: {e}"
            break
        connect(ctx)
        w = TrainingWorker(cfg, prof, ranks=[rank], ctx=ctx)
        try:
            w.run()
            got = f"{w.params_digest(0):016x}"
        except Exception as e:  # noqa: BLE001
            got = f"error: {e}"
        want_d = want[(name, world, kind)] if counts_ is None else ref[0]
        out["digests"][f"{name}/{kind}/nvls"] = [got, want_d]
        dist.barrier()
        w.close()

    # the layer-wise baseline (KVStore placement + FIFO) on the same kernels across processes:
    # bit-identical to P3 (SPEC acceptance #3)
    for name in ("toy3", "vgg19-like"):
        if (name, world, "same") not in want:
            continue
        prof = builtin_profile(name)
        cfg = WorkerConfig(rank=rank, mode="baseline", world=world, iterations=10, deadlock_timeout=60.0,
                           emulate_compute=False, comm_ctas=8, big_threshold=100_000)
        ctx = SyncContext(prof.param_counts(), world, [rank], lr=cfg.lr, comm_ctas=8, timeout_s=60.0,
                          emulate_grads=True, plan_mode="baseline", priority_mode=False, big_threshold=100_000,
                          notify_pull=True)  # the reference baseline's NOTIFY -> PULL round trip
        hs = [None] * world
        dist.all_gather_object(hs, ctx.ipc_handle(0))
        ctx.open_peers(hs)
        dist.barrier()
        w = TrainingWorker(cfg, prof, ranks=[rank], ctx=ctx)
        try:
            w.run()
            got = f"{w.params_digest(0):016x}"
        except Exception as e:  # noqa: BLE001
            got = f"error: {e}"
        out["digests"][f"{name}/baseline"] = [got, want[(name, world, "same")]]
        dist.barrier()
        w.close()

    # torch mode: identical data on every rank -> mean gradient == local gradient, so the
    # result must equal single-GPU fp32 SGD bit for bit
    from paper_1905_03960_b200.ddp import LayerwiseDataParallel, P3DataParallel

    def mlp():
        torch.manual_seed(0)
        return torch.nn.Sequential(torch.nn.Linear(64, 300), torch.nn.ReLU(), torch.nn.Linear(300, 233),
                                   torch.nn.ReLU(), torch.nn.Linear(233, 10)).cuda()

    lr = 0.05
    ref, mod, mod2 = mlp(), mlp(), mlp()
    ddp = P3DataParallel(mod, lr=lr, max_slice=1000, comm_ctas=4, timeout_s=30.0)
    lw = LayerwiseDataParallel(mod2, lr=lr)
    g = torch.Generator(device="cuda").manual_seed(1)
    for it in range(5):
        x = torch.randn(32, 64, device="cuda", generator=g)
        y = torch.randint(0, 10, (32,), device="cuda", generator=g)
        torch.nn.functional.cross_entropy(ddp(x), y).backward()
        torch.nn.functional.cross_entropy(lw(x), y).backward()
        torch.nn.functional.cross_entropy(ref(x), y).backward()
        with torch.no_grad():
            for p in ref.parameters():
                p.sub_(p.grad.mul(lr))
                p.grad = None
    ddp.synchronize()
    lw.synchronize()
    out["torch_p3_exact"] = all(torch.equal(a, b) for a, b in zip(mod.parameters(), ref.parameters()))
    out["torch_layerwise_close"] = all(torch.allclose(a, b, atol=1e-5) for a, b in zip(mod2.parameters(), ref.parameters()))
    ddp.close()
    lw.close()

    # torch mode on real shapes with DIFFERENT data on every rank: after every step each
    # replica must hold p - lr * ((g_0 + ... + g_{N-1}) / N), the rank-ordered fp32 sum of the
    # ranks' own autograd gradients (gathered here), separately rounded (server.py:55-68)
    from paper_1905_03960_b200.torch_models import build_model, loss_fn, synthetic_batch

    for name, batch, nvls in (("resnet50", 8, False), ("seq2seq", 8, False), ("resnet50", 8, True)):
        if nvls and out["nvls"] != "ok":
            continue  # (NVLS: the same check with multicast broadcasts, where the box has them)
        torch.manual_seed(7)
        m = build_model(name).cuda()
        if name == "resnet50":
            m = m.to(memory_format=torch.channels_last)
        d = P3DataParallel(m, lr=lr, comm_ctas=8, timeout_s=60.0, nvls=nvls)
        names = [n for n, p in m.named_parameters() if p.requires_grad]
        exact, differs = True, False
        for it in range(3):
            old = {n: p.detach().clone() for n, p in m.named_parameters() if p.requires_grad}
            x, y = synthetic_batch(name, batch, seed=1000 * it + rank)
            loss_fn(name, d, x, y).backward()
            grads = {n: p.grad.detach().clone() for n, p in m.named_parameters() if p.requires_grad}
            d.synchronize()
            torch.cuda.synchronize()
            params = dict(m.named_parameters())
            for n in names:
                gs = [torch.empty(grads[n].shape, dtype=grads[n].dtype, device="cuda") for _ in range(world)]
                dist.all_gather(gs, grads[n].contiguous())
                acc = torch.zeros_like(old[n])
                for r in range(world):
                    acc = acc + gs[r].view_as(acc)
                want = old[n] - (acc / torch.full_like(acc, world)).mul(lr)
                exact &= bool(torch.equal(params[n].detach(), want))
                differs |= not torch.equal(gs[0], gs[-1])
        out[f"torch_p3_distinct_{name}" + ("_nvls" if nvls else "")] = exact and differs
        d.close()
        del d, m
        torch.cuda.empty_cache()
    # bf16 replicas (param_dtype bf16) over NVLink, different data per rank: each replica equals
    # bf16(master), the fp32 master updated from the ranks' own bf16 gradients in rank order
    torch.manual_seed(7)
    m = build_model("resnet50").cuda().to(memory_format=torch.channels_last).bfloat16()
    d = P3DataParallel(m, lr=lr, comm_ctas=8, timeout_s=60.0)
    names = [n for n, p in m.named_parameters() if p.requires_grad]
    master = {n: p.detach().float().clone() for n, p in m.named_parameters() if p.requires_grad}
    exact, differs = d.param_dtype == "bf16", False
    for it in range(2):
        x, y = synthetic_batch("resnet50", 8, seed=2000 * it + rank)
        loss_fn("resnet50", d, x, y).backward()
        grads = {n: p.grad.detach().clone() for n, p in m.named_parameters() if p.requires_grad}
        d.synchronize()
        torch.cuda.synchronize()
        params = dict(m.named_parameters())
        for n in names:
            gs = [torch.empty(grads[n].shape, dtype=grads[n].dtype, device="cuda") for _ in range(world)]
            dist.all_gather(gs, grads[n].contiguous())
            acc = torch.zeros_like(master[n])
            for r in range(world):
                acc = acc + gs[r].view_as(acc).float()
            master[n] = master[n] - (acc / torch.full_like(acc, world)).mul(lr)
            exact &= bool(torch.equal(params[n].detach(), master[n].bfloat16()))
            differs |= not torch.equal(gs[0], gs[-1])
    out["torch_p3_bf16_replicas"] = exact and differs
    d.close()
    del d, m
    torch.cuda.empty_cache()
    out_dir = os.environ.get("P3_MP_OUT")
    if out_dir:
        Path(out_dir, f"rank{rank}.json").write_text(json.dumps(out))
    print("MPRESULT " + json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
