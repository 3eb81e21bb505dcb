"""The three real model shapes of the benchmark configs (BASELINE.json configs[1..3]).

- ResNet-50 and VGG-19: torchvision definitions (161 / 38 parameter tensors,
  25,557,032 / 143,667,240 parameters), random init, synthetic ImageNet-shape input.
- A Sockeye-style seq2seq translation model (builder-defined):
  a 32000x512 embedding shared by source, target and the output softmax at forward
  index 0 (the reference pins only "heaviest layer first", model.py:146-153), a
  bidirectional LSTM + 3 LSTM encoder layers, a 4-layer LSTM decoder whose first layer
  reads [target embedding; encoder summary] (1024 inputs), bilinear attention, an
  attention-combine layer and the softmax bias: 41 tensors, 34,537,216 parameters.

Each parameter tensor is one P3 "layer" (one KVStore key) and its
priority is its forward index (registration order here).
"""

from __future__ import annotations

from .model import ModelProfile, profile_from_module

REAL_MODELS = ("resnet50", "vgg19", "seq2seq")
VOCAB = 32000
HIDDEN = 512
SEQ_LEN = 50


def _torch():
    import torch
    import torch.nn as nn

    return torch, nn


def build_seq2seq():
    torch, nn = _torch()

    class TiedSoftmax(nn.Module):
        # output projection sharing the embedding matrix; owns only the softmax bias so the
        # bias is gated (and prioritised) at its point of use, last in the forward pass
        def __init__(self, embed) -> None:
            super().__init__()
            self.bias = nn.Parameter(torch.zeros(VOCAB))
            self._embed = [embed]  # not a submodule: the weight stays owned by `embed`

        def forward(self, x):
            return torch.nn.functional.linear(x, self._embed[0].weight, self.bias)

    class Seq2Seq(nn.Module):
        def __init__(self) -> None:
            super().__init__()
            self.embed = nn.Embedding(VOCAB, HIDDEN)
            self.enc_bi = nn.LSTM(HIDDEN, HIDDEN // 2, bidirectional=True, batch_first=True)
            self.enc = nn.LSTM(HIDDEN, HIDDEN, num_layers=3, batch_first=True)
            self.dec = nn.LSTM(2 * HIDDEN, HIDDEN, num_layers=4, batch_first=True)
            self.att = nn.Linear(HIDDEN, HIDDEN, bias=False)
            self.combine = nn.Linear(2 * HIDDEN, HIDDEN)
            self.softmax = TiedSoftmax(self.embed)

        def forward(self, src, trg):
            e = self.embed(src)
            h, _ = self.enc_bi(e)
            h, _ = self.enc(h)  # [B, S, H]
            summary = h.mean(dim=1, keepdim=True).expand(-1, trg.shape[1], -1)
            d, _ = self.dec(torch.cat([self.embed(trg), summary], dim=-1))  # [B, T, H]
            scores = torch.bmm(self.att(d), h.transpose(1, 2))  # [B, T, S]
            ctx = torch.bmm(torch.softmax(scores, dim=-1), h)
            o = torch.tanh(self.combine(torch.cat([d, ctx], dim=-1)))
            return self.softmax(o)

    return Seq2Seq()


def build_model(name: str):
    torch, nn = _torch()
    import torchvision

    if name == "resnet50":
        return torchvision.models.resnet50()
    if name == "vgg19":
        return torchvision.models.vgg19()
    if name == "seq2seq":
        return build_seq2seq()
    raise ValueError(f"unknown model {name!r}; have {REAL_MODELS}")


# Parameter counts per tensor (forward order), so profiles need no model construction.
_COUNTS_CACHE: dict[str, list[int]] = {}


def real_counts(name: str) -> list[int]:
    if name not in _COUNTS_CACHE:
        torch, _ = _torch()
        with torch.device("meta"):
            m = build_model(name)
        _COUNTS_CACHE[name] = [int(p.numel()) for p in m.parameters() if p.requires_grad]
    return _COUNTS_CACHE[name]


def real_profile(name: str, seed: int = 0) -> ModelProfile:
    torch, _ = _torch()
    with torch.device("meta"):
        m = build_model(name)
    return profile_from_module(m, name, seed=seed)


def synthetic_batch(name: str, batch: int, device="cuda", seed: int = 1234, pinned_host: bool = False):
    """Synthetic inputs of the configs: x ~ N(0,1) bf16
    [B,3,224,224] channels_last with labels in [0,1000), or token ids in [0,32000)."""
    torch, _ = _torch()
    g = torch.Generator().manual_seed(seed)
    dev = "cpu" if pinned_host else device
    if name in ("resnet50", "vgg19"):
        x = torch.randn(batch, 3, 224, 224, generator=g).to(torch.bfloat16)
        x = x.contiguous(memory_format=torch.channels_last)
        y = torch.randint(0, 1000, (batch,), generator=g)
    else:
        x = torch.randint(0, VOCAB, (batch, 2, SEQ_LEN), generator=g)
        y = torch.randint(0, VOCAB, (batch, SEQ_LEN), generator=g)
    if pinned_host:
        return x.pin_memory(), y.pin_memory()
    return x.to(dev), y.to(dev)


def loss_fn(name: str, model, x, y):
    torch, _ = _torch()
    if name in ("resnet50", "vgg19"):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = model(x)
        return torch.nn.functional.cross_entropy(out.float(), y)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = model(x[:, 0], x[:, 1])
    return torch.nn.functional.cross_entropy(logits.float().reshape(-1, VOCAB), y.reshape(-1))
