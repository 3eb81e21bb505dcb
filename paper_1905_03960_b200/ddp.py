"""P3 for real PyTorch models: backward hooks publish layers, forward hooks gate them.

``P3DataParallel`` is the torch-mode driver of the sync path. Every trainable parameter
tensor is one P3 layer (one KVStore key) whose priority is its forward index
(registration order). Its storage is moved into the context's peer-writable parameter
arena ``W`` so the comm kernel's broadcast stores land directly in the tensors the next
forward reads.

Per iteration k:
  - root forward pre-hook: the gradients of iteration k-1 are released to the allocator
    only after the comm stream's current work (record_stream), and iteration k is opened
    on a high-priority comm stream;
  - per-module forward pre-hook: ``p3_wait_layer`` (a stream memory wait, no SM) gates the
    module on its parameters having been updated by iteration k-1 (worker.py:277-285);
  - post-accumulate-grad hook: ``p3_layer_ready`` publishes the layer's gradient pointer
    and iteration tag with stream-ordered writes (enqueue_layer, worker.py:173-182) and
    queues a DRAIN launch of the comm kernel behind that point;
  - end-of-backward callback: publishes layers that got no gradient (zeros), queues the
    iteration's FINISH launch and advances k.
The optimizer step is fused into the comm kernel (SGD, optional momentum): do not run a
torch optimizer on these parameters.

``LayerwiseDataParallel`` is the baseline the paper compares against (aggressive,
non-sliced, FIFO layer-wise sync): per-tensor NCCL all-reduce issued in backward-hook
order, the SGD step applied in the next forward's pre-hook behind the same gates.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .plan import DEFAULT_MAX_SLICE
from .runtime import SyncContext, connect


def _dist_info() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def _param_modules(module: torch.nn.Module, params: list) -> list[tuple[torch.nn.Module, list[int]]]:
    index = {id(p): i for i, p in enumerate(params)}
    out = []
    for m in module.modules():
        own = [index[id(p)] for p in m._parameters.values() if p is not None and id(p) in index]
        if own:
            out.append((m, own))
    return out


class _HookedDataParallel:
    def __init__(self, module: torch.nn.Module) -> None:
        self.module = module
        self.params = [p for p in module.parameters() if p.requires_grad]
        self.world, self.rank = _dist_info()
        self.k = 0
        self._handles = []
        self._gated: set[int] = set()
        self._ready: set[int] = set()

    def __call__(self, *args, **kwargs):
        return self.module(*args, **kwargs)

    def _install(self) -> None:
        self._handles.append(self.module.register_forward_pre_hook(self._root_pre_hook))
        for m, layers in _param_modules(self.module, self.params):
            self._handles.append(m.register_forward_pre_hook(self._make_gate(layers)))
        for l, p in enumerate(self.params):
            self._handles.append(p.register_post_accumulate_grad_hook(self._make_ready(l)))

    def _make_gate(self, layers):
        def hook(mod, inputs):
            for l in layers:
                if l not in self._gated:
                    self._gate(l)
                    self._gated.add(l)

        return hook

    def _make_ready(self, l):
        def hook(p):
            if not self._ready:
                torch.autograd.Variable._execution_engine.queue_callback(self._end_backward)
            self._ready.add(l)
            self._publish(l, p.grad)

        return hook

    def _end_backward(self) -> None:
        for l, p in enumerate(self.params):
            if l not in self._ready:  # no gradient this iteration: sync zeros
                if l not in self._gated:
                    self._gate(l)
                    self._gated.add(l)
                p.grad = torch.zeros_like(p)
                self._publish(l, p.grad)
        self._after_backward()
        self._ready.clear()
        self._gated.clear()
        self.k += 1

    def _root_pre_hook(self, mod, inputs):
        self._begin_iteration()

    def remove_hooks(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles.clear()


class P3DataParallel(_HookedDataParallel):
    """Sliced, priority-scheduled parameter sync of ``module`` on the local GPU."""

    def __init__(
        self,
        module: torch.nn.Module,
        lr: float,
        momentum: float = 0.0,
        max_slice: int = DEFAULT_MAX_SLICE,
        comm_ctas: int = 8,
        comm_threads: int = 512,
        timeout_s: float = 120.0,
        trace_cap: int = 0,
        priority_mode: bool = True,
        drain_bytes: int | None = None,
        pub_batch_bytes: int = 1 << 20,
        drain_linger_us: int = 200,
        finish_ctas: int | None = None,
        push_dtype: str = "fp32",
        plan_mode: str = "p3",
        throttle_bps: float = 0.0,
        throttle_burst: int = 50 * 1024,
        big_threshold: int = 1_000_000,
    ) -> None:
        super().__init__(module)
        self.lr = lr
        counts = [p.numel() for p in self.params]
        # one forward gate per module: all parameters a module owns share a gate group
        self._module_layers = _param_modules(module, self.params)
        groups = [0] * len(self.params)
        for gi, (_, layers) in enumerate(self._module_layers):
            for l in layers:
                groups[l] = gi
        self._group_of = groups
        if drain_bytes is None:
            # N>1: sync overlaps the backward pass (a DRAIN launch per 4 MB of gradients).
            # N=1 there is nothing to overlap: no DRAIN launches (the backward keeps every SM)
            # and one FINISH launch over the whole GPU updates the parameters in priority order
            drain_bytes = 4 << 20 if self.world > 1 else 1 << 62
        if finish_ctas is None:
            finish_ctas = 0 if self.world > 1 else torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        self.ctx = SyncContext(
            counts, self.world, [self.rank], max_slice=max_slice, lr=lr, momentum=momentum,
            priority_mode=priority_mode, comm_ctas=comm_ctas, comm_threads=comm_threads,
            timeout_s=timeout_s, trace_cap=trace_cap, drain_bytes=drain_bytes, plan_mode=plan_mode,
            throttle_bps=throttle_bps, throttle_burst=throttle_burst, big_threshold=big_threshold,
            gate_groups=groups, pub_batch_bytes=pub_batch_bytes, drain_linger_us=drain_linger_us,
            finish_ctas=finish_ctas, push_dtype=push_dtype,
        )
        connect(self.ctx)  # every rank's arena, after checking all ranks built the same plan
        arena = self.ctx.params_arena(0)
        with torch.no_grad():
            for l, p in enumerate(self.params):
                if self.world > 1:
                    dist.broadcast(p.data, src=0)
                off = self.ctx.layer_offsets[l]
                flat = arena[off : off + p.numel()]
                if p.is_contiguous() or not _dense(p):
                    view = flat.view(p.shape)
                else:  # keep e.g. channels_last weights in their memory order
                    view = flat.as_strided(p.shape, p.stride())
                view.copy_(p.data)
                p.data = view
        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        self.comm_stream = torch.cuda.Stream(priority=-1)
        self._grads: list = []
        self._launched = -1
        self._install()

    # -- hooks
    def _begin_iteration(self) -> None:
        if self._launched == self.k:
            return
        for p in self.params:
            if p.grad is not None:
                # the comm kernel of the previous iteration may still read this gradient
                p.grad.record_stream(self.comm_stream)
                p.grad = None
        self.ctx.iteration_begin(self.k, self.comm_stream)
        self._launched = self.k

    def _gate(self, l: int) -> None:
        self.ctx.wait_layer(0, l, self.k)

    def _make_gate(self, layers):
        group = self._group_of[layers[0]]

        def hook(mod, inputs):
            if layers[0] not in self._gated:
                self.ctx.wait_group(0, group, self.k)
                self._gated.update(layers)

        return hook

    def _publish(self, l: int, grad) -> None:
        p = self.params[l]
        if grad.dtype != torch.float32 or grad.stride() != p.stride():
            grad = _relayout(grad, p)
            p.grad = grad
        self.ctx.layer_ready(0, l, self.k, grad)

    def _after_backward(self) -> None:
        self.ctx.iteration_end(self.k)

    # -- API
    def synchronize(self, timeout_s: float | None = None) -> None:
        """Block until every layer holds the parameters of the last finished iteration."""
        self.ctx.sync_all(self.k, timeout_s)
        torch.cuda.current_stream().wait_stream(self.comm_stream)

    def close(self) -> None:
        """Detach: parameters get their own storage again (a copy of the synced values)
        before the context (and its parameter arena) is destroyed."""
        self.remove_hooks()
        try:
            self.synchronize()
        except Exception:  # noqa: BLE001 - detach anyway
            pass
        with torch.no_grad():
            for p in self.params:
                p.data = p.data.clone(memory_format=torch.preserve_format)
                p.grad = None
        torch.cuda.synchronize()
        self.ctx.close()


def _dense(t: torch.Tensor) -> bool:
    """Non-overlapping and dense (some permutation of a contiguous layout)."""
    expect = 1
    for size, stride in sorted(zip(t.shape, t.stride()), key=lambda d: d[1]):
        if size == 1:
            continue
        if stride != expect:
            return False
        expect *= size
    return True


def _relayout(grad: torch.Tensor, p: torch.Tensor) -> torch.Tensor:
    out = torch.empty_strided(p.shape, p.stride(), dtype=torch.float32, device=p.device)
    out.copy_(grad)
    return out


class LayerwiseDataParallel(_HookedDataParallel):
    """Baseline: per-tensor NCCL all-reduce (FIFO in backward order) + SGD before reuse."""

    def __init__(self, module: torch.nn.Module, lr: float) -> None:
        super().__init__(module)
        self.lr = lr
        if self.world > 1:
            with torch.no_grad():
                for p in self.params:
                    dist.broadcast(p.data, src=0)
        self._work: dict[int, object] = {}
        self._install()

    def _begin_iteration(self) -> None:
        pass

    def _publish(self, l: int, grad) -> None:
        if self.world > 1:
            self._work[l] = dist.all_reduce(grad, async_op=True)

    def _gate(self, l: int) -> None:
        p = self.params[l]
        if p.grad is None:
            return
        w = self._work.pop(l, None)
        if w is not None:
            w.wait()
        with torch.no_grad():
            p.add_(p.grad, alpha=-self.lr / self.world)
        p.grad = None

    def _after_backward(self) -> None:
        pass

    def synchronize(self, timeout_s: float | None = None) -> None:
        for l in range(len(self.params)):
            self._gate(l)
        torch.cuda.current_stream().synchronize()

    def close(self) -> None:
        self.remove_hooks()
