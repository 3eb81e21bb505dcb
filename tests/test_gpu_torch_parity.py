"""Torch-mode parity of P3DataParallel at N > 1 on real shapes, on one GPU.

``P3LocalWorld`` hosts all N ranks of a world in one process: N replicas of the model share
one sync context with N local ranks, each trains on DIFFERENT data, and the comm kernel
sums the N autograd gradients of every slice in ascending rank order, divides by N and
applies SGD (ShardState.aggregate_and_update, server.py:55-68). After every iteration each
replica must hold exactly p - lr * ((g_0 + ... + g_{N-1}) / N), computed here with separately
rounded fp32 torch ops from the gradients the replicas produced — bit for bit, for ResNet-50
(161 tensors, 25.6M parameters) and for the seq2seq model with its tied embedding.
Also: forward-order priorities and the tied-parameter gate."""

import pytest

pytestmark = pytest.mark.gpu


def _model(name, seed):
    import torch

    from paper_1905_03960_b200.torch_models import build_model

    torch.manual_seed(seed)
    if name == "mlp":
        m = torch.nn.Sequential(torch.nn.Embedding(1000, 64), torch.nn.Flatten(), torch.nn.Linear(64 * 8, 300),
                                torch.nn.ReLU(), torch.nn.Linear(300, 10))
        return m.cuda()
    m = build_model(name).cuda()
    if name in ("resnet50", "vgg19"):
        m = m.to(memory_format=torch.channels_last)
    return m


def _batch(name, batch, seed):
    import torch

    from paper_1905_03960_b200.torch_models import synthetic_batch

    if name == "mlp":
        g = torch.Generator(device="cuda").manual_seed(seed)
        return (torch.randint(0, 1000, (batch, 8), device="cuda", generator=g),
                torch.randint(0, 10, (batch,), device="cuda", generator=g))
    return synthetic_batch(name, batch, seed=seed)


def _loss(name, model, x, y):
    import torch

    from paper_1905_03960_b200.torch_models import loss_fn

    if name == "mlp":
        return torch.nn.functional.cross_entropy(model(x), y)
    return loss_fn(name, model, x, y)


@pytest.mark.parametrize("name,world,batch", [("mlp", 3, 16), ("resnet50", 2, 4), ("resnet50", 4, 2),
                                              ("seq2seq", 2, 4)])
def test_local_world_equals_rank_ordered_sgd(cuda, name, world, batch):
    import torch

    from paper_1905_03960_b200.ddp import P3DataParallel, P3LocalWorld

    lr = 0.05
    models = [_model(name, 7) for _ in range(world)]
    lw = P3LocalWorld(world, timeout_s=60.0)
    reps = [P3DataParallel(m, lr=lr, local_world=lw, comm_ctas=8, max_slice=50_000) for m in models]
    names = [n for n, p in models[0].named_parameters() if p.requires_grad]
    for it in range(3):
        old = {n: p.detach().clone() for n, p in models[0].named_parameters() if p.requires_grad}
        grads = []
        for r, (rep, m) in enumerate(zip(reps, models)):
            x, y = _batch(name, batch, seed=1000 * it + r)  # different data on every rank
            _loss(name, rep, x, y).backward()
            grads.append({n: p.grad.detach().clone() for n, p in m.named_parameters() if p.requires_grad})
        reps[0].synchronize()
        torch.cuda.synchronize()
        for n in names:
            acc = torch.zeros_like(old[n])
            for r in range(world):  # ascending rank order from +0.0 (server.py:60-63)
                acc = acc + grads[r][n]
            # separately rounded div, mul, sub (server.py:64-65); the divisor is a tensor: torch
            # turns division by a Python scalar into a multiply by its reciprocal
            want = old[n] - (acc / torch.full_like(acc, world)).mul(lr)
            for r, m in enumerate(models):
                got = dict(m.named_parameters())[n]
                assert torch.equal(got, want), f"{name} it {it} rank {r} {n}"
        assert len({d[names[0]].sum().item() for d in grads}) == world  # the data did differ
    for rep in reps:
        rep.close()


class _Reordered:
    """Registers its layers in the reverse of the order the forward uses them, with an
    output projection tied to the embedding (own bias) registered BEFORE the embedding."""

    @staticmethod
    def build():
        import torch

        class TiedOut(torch.nn.Module):
            def __init__(self, emb):
                super().__init__()
                self.weight = emb.weight  # shared Parameter, owned here AND by the embedding
                self.bias = torch.nn.Parameter(torch.zeros(emb.num_embeddings))

            def forward(self, h):
                return torch.nn.functional.linear(h, self.weight, self.bias)

        class M(torch.nn.Module):
            def __init__(self):
                super().__init__()
                emb = torch.nn.Embedding(500, 32)
                self.out = TiedOut(emb)           # registered first, used last
                self.mid = torch.nn.Linear(32, 32)
                self.emb = emb                    # registered last, used first

            def forward(self, x):
                return self.out(torch.tanh(self.mid(self.emb(x).mean(1))))

        torch.manual_seed(3)
        return M().cuda()


def test_forward_order_priorities_and_tied_gate(cuda):
    import torch

    from paper_1905_03960_b200.ddp import P3DataParallel

    lr = 0.1
    ref, mod = _Reordered.build(), _Reordered.build()
    ddp = P3DataParallel(mod, lr=lr, comm_ctas=4, timeout_s=20.0)
    g = torch.Generator(device="cuda").manual_seed(5)
    for it in range(5):
        x = torch.randint(0, 500, (16, 6), device="cuda", generator=g)
        y = torch.randint(0, 500, (16,), device="cuda", generator=g)
        loss = torch.nn.functional.cross_entropy(ddp(x), y)
        loss.backward()
        lref = torch.nn.functional.cross_entropy(ref(x), y)
        lref.backward()
        with torch.no_grad():
            for p in ref.parameters():
                p.sub_(p.grad.mul(lr))
                p.grad = None
        assert loss.item() == lref.item(), it
    # priorities follow the forward: the embedding (shared with the output) first, the
    # output bias last — not the registration order (out.weight, out.bias, mid.*, emb.weight)
    assert ddp.layer_names() == ["out.weight", "mid.weight", "mid.bias", "out.bias"]
    # the shared tensor is gated by the embedding, its first user in the forward
    gated_by = {id(m): ls for m, ls in ddp._module_layers}
    assert gated_by[id(mod.emb)] == [0]
    ddp.synchronize()
    for a, b in zip(mod.parameters(), ref.parameters()):
        assert torch.equal(a, b)
    ddp.close()


@pytest.mark.parametrize("name,world,batch", [("mlp", 1, 16), ("mlp", 3, 16), ("resnet50", 2, 4)])
def test_bf16_parameters_fp32_masters(cuda, name, world, batch):
    """Declared bf16 replicas (param_dtype bf16, chosen from the model's bf16 parameters): bf16
    gradients are pushed as they are, the owner sums them in fp32 in rank order, updates its
    fp32 master with the fp32 path's arithmetic and broadcasts bf16(master) (round to nearest
    even). Each replica must equal that, computed here with torch from the replicas' own bf16
    gradients — bit for bit; no copy / cast kernels on the sync path (the gradients are
    published in place)."""
    import torch

    from paper_1905_03960_b200.ddp import P3DataParallel, P3LocalWorld

    lr = 0.05
    models = [_model(name, 11).bfloat16() for _ in range(world)]
    lw = P3LocalWorld(world, timeout_s=60.0) if world > 1 else None
    reps = [P3DataParallel(m, lr=lr, local_world=lw, comm_ctas=8) for m in models]
    assert reps[0].param_dtype == "bf16"
    names = [n for n, p in models[0].named_parameters() if p.requires_grad]
    master = {n: p.detach().float().clone() for n, p in models[0].named_parameters() if p.requires_grad}
    for it in range(3):
        grads = []
        for r, (rep, m) in enumerate(zip(reps, models)):
            x, y = _batch(name, batch, seed=500 * it + r)
            if name == "resnet50":
                x = x.bfloat16()
            _loss(name, rep, x, y).backward()
            grads.append({n: p.grad.detach().clone() for n, p in m.named_parameters() if p.requires_grad})
        reps[0].synchronize()
        torch.cuda.synchronize()
        for n in names:
            acc = torch.zeros_like(master[n])
            for r in range(world):
                acc = acc + grads[r][n].float()
            master[n] = master[n] - (acc / torch.full_like(acc, world)).mul(lr)
            want = master[n].bfloat16()
            for r, m in enumerate(models):
                got = dict(m.named_parameters())[n]
                assert got.dtype == torch.bfloat16
                assert torch.equal(got, want), f"{name} it {it} rank {r} {n}"
    for rep in reps:
        rep.close()
