"""P3 for real PyTorch models: backward hooks publish layers, forward hooks gate them.

``P3DataParallel`` is the torch-mode driver of the sync path. Every trainable parameter
tensor is one P3 layer (one KVStore key). Its priority is its FORWARD index:
the order in which the first forward pass uses the tensors (recorded by forward pre-hooks,
SURVEY §7 hard part 6), so the layer the next forward needs first is synced first whatever
order the module registered its parameters in (``order="registration"`` keeps the
``parameters()`` order). The layer's storage is moved into the context's peer-writable
parameter arena ``W`` so the comm kernel's broadcast stores land directly in the tensors
the next forward reads. The context is built at the end of the first forward (once the
order is known); that forward reads the initial parameters, which need no gate.

Per iteration k:
  - root forward pre-hook: the gradients of iteration k-1 are released to the allocator
    only after the comm stream's current work (record_stream), and iteration k is opened
    on a high-priority comm stream;
  - per-module forward pre-hook: ``p3_wait_group`` (a stream memory wait, no SM) gates the
    module on every parameter it owns having been updated by iteration k-1
    (worker.py:277-285); a tensor shared by several modules is gated by its first user;
    tensors owned by modules the forward never calls are gated at the root;
  - post-accumulate-grad hook: ``p3_layer_ready`` publishes the layer's gradient pointer
    and iteration tag (enqueue_layer, worker.py:173-182) and queues a DRAIN launch of the
    comm kernel behind that point;
  - end-of-backward callback: publishes layers that got no gradient (zeros), queues the
    iteration's FINISH launch and advances k.
The optimizer step is fused into the comm kernel (SGD, optional momentum): do not run a
torch optimizer on these parameters.

One process normally hosts one rank (torchrun, one GPU each). ``P3LocalWorld`` hosts every
rank of a world in one process instead — N replicas of the model sharing one context with
N local ranks on one GPU — which is how torch-mode parity at N > 1 is tested on one device.

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


class _ForwardOrder:
    """Records, during one forward pass, the order in which parameter-owning modules are
    first called; a parameter's forward index is the position of its first use."""

    def __init__(self, module: torch.nn.Module, params: list) -> None:
        self.ids = {id(p): i for i, p in enumerate(params)}
        self.seen: list[int] = []
        self.called: list[torch.nn.Module] = []  # parameter-owning modules, in first-call order
        self._h = []
        for m in module.modules():
            if any(p is not None and id(p) in self.ids for p in m._parameters.values()):
                self._h.append(m.register_forward_pre_hook(self._hook))

    def _hook(self, mod, inputs):
        if not any(m is mod for m in self.called):
            self.called.append(mod)
        for p in mod._parameters.values():
            if p is not None and id(p) in self.ids and self.ids[id(p)] not in self.seen:
                self.seen.append(self.ids[id(p)])

    def finish(self, n: int) -> list[int]:
        for h in self._h:
            h.remove()
        self._h.clear()
        rest = [i for i in range(n) if i not in set(self.seen)]
        return self.seen + rest


def _gate_groups(module: torch.nn.Module, params: list, called: list | None):
    """(module, layers) pairs for the forward gates, and the layers no called module owns.
    A tensor shared by several modules (tied weights) belongs to the first of them the
    forward calls (module order without a trace), so each tensor is gated exactly once,
    before its first use; tensors of modules the traced forward never called are gated at
    the root (they may still be read functionally)."""
    index = {id(p): i for i, p in enumerate(params)}
    taken: set[int] = set()
    out = []
    for m in (called if called is not None else module.modules()):
        own = [index[id(p)] for p in m._parameters.values() if p is not None and id(p) in index]
        own = [l for l in own if l not in taken]
        if own:
            taken.update(own)
            out.append((m, own))
    orphans = [l for l in range(len(params)) if l not in taken]
    return out, orphans


class _HookedDataParallel:
    def __init__(self, module: torch.nn.Module, order: str = "forward") -> None:
        if order not in ("forward", "registration"):
            raise ValueError("order must be 'forward' or 'registration'")
        self.module = module
        self.params = [p for p in module.parameters() if p.requires_grad]
        self.world, self.rank = _dist_info()
        self.order = order
        self.k = 0
        self._handles = []
        self._gated: set[int] = set()
        self._ready: set[int] = set()
        self._tracer: _ForwardOrder | None = None
        self._called: list | None = None
        self._set_up = False

    def __call__(self, *args, **kwargs):
        return self.module(*args, **kwargs)

    # -- construction: at once (registration order) or after the first forward (forward order)
    def _start(self) -> None:
        if self.order == "registration":
            self._finish_setup(list(range(len(self.params))))
            return
        self._tracer = _ForwardOrder(self.module, self.params)
        self._trace_handle = self.module.register_forward_hook(self._end_trace)

    def _end_trace(self, mod, inputs, output):
        self._trace_handle.remove()
        perm = self._tracer.finish(len(self.params))
        self._called = self._tracer.called
        self._tracer = None
        self._finish_setup(perm)
        self._begin_iteration()  # iteration 0 (its forward read the initial parameters)

    def _finish_setup(self, perm: list[int]) -> None:
        self.params = [self.params[i] for i in perm]
        self._module_layers, self._orphans = _gate_groups(self.module, self.params, self._called)
        self._setup()
        self._install()
        self._set_up = True

    def _setup(self) -> None:  # subclass: build the sync state once the layer order is known
        pass

    def _install(self) -> None:
        self._handles.append(self.module.register_forward_pre_hook(self._root_pre_hook))
        for m, layers in self._module_layers:
            self._handles.append(m.register_forward_pre_hook(self._make_gate(layers)))
        for l, p in enumerate(self.params):
            self._handles.append(p.register_post_accumulate_grad_hook(self._make_ready(l)))

    def _make_gate(self, layers):
        def hook(mod, inputs):
            todo = [l for l in layers if l not in self._gated]
            if todo:
                self._gate_layers(todo)
                self._gated.update(todo)

        return hook

    def _gate_layers(self, layers) -> None:
        for l in layers:
            self._gate(l)

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
                    self._gate_layers([l])
                    self._gated.add(l)
                p.grad = torch.zeros_like(p)
                self._publish(l, p.grad)
        self._after_backward()
        self._ready.clear()
        self._gated.clear()
        self.k += 1

    def _root_pre_hook(self, mod, inputs):
        self._begin_iteration()
        todo = [l for l in self._orphans if l not in self._gated]
        if todo:
            self._gate_layers(todo)
            self._gated.update(todo)

    def remove_hooks(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles.clear()
        if self._tracer is not None:
            self._tracer.finish(len(self.params))
            self._trace_handle.remove()
            self._tracer = None


class P3LocalWorld:
    """Every rank of a P3 world hosted in THIS process: one SyncContext with ``world`` local
    ranks on the current GPU, shared by ``world`` model replicas (``P3DataParallel(...,
    local_world=lw)`` in rank order). The replicas train one after the other inside each
    iteration; the iteration opens at the first replica's forward and its FINISH launch is
    queued after the last replica's backward. The replicas must be constructed from equal
    initial parameters (replica r copies replica 0's values, the broadcast of a real run)."""

    def __init__(self, world: int, **ctx_kwargs) -> None:
        if world < 1:
            raise ValueError("world must be >= 1")
        self.world = world
        self.ctx_kwargs = ctx_kwargs
        self.ctx: SyncContext | None = None
        self.replicas: list[P3DataParallel] = []
        self.comm_stream = None
        self._begun = -1
        self._ended: dict[int, set[int]] = {}
        self._perm: list[int] | None = None

    def _join(self, rep: "P3DataParallel") -> int:
        if len(self.replicas) >= self.world:
            raise ValueError(f"local world of {self.world} ranks is full")
        self.replicas.append(rep)
        return len(self.replicas) - 1

    def begin(self, k: int) -> None:
        if self._begun < k:
            self.ctx.iteration_begin(k, self.comm_stream)
            self._begun = k

    def end(self, li: int, k: int) -> None:
        done = self._ended.setdefault(k, set())
        done.add(li)
        if len(done) == self.world:
            self.ctx.iteration_end(k)
            del self._ended[k]


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
        order: str = "forward",
        local_world: P3LocalWorld | None = None,
        notify_pull: bool | None = None,
        nvls: bool = False,
    ) -> None:
        super().__init__(module, order)
        dtypes = {p.dtype for p in self.params}
        if dtypes - {torch.float32, torch.bfloat16} or len(dtypes) > 1:
            raise ValueError(f"parameters must be all float32 or all bfloat16 (have {sorted(map(str, dtypes))})")
        # bf16 parameters: bf16 replicas and gradients on the wire, fp32 masters at the owners
        self.param_dtype = "bf16" if dtypes == {torch.bfloat16} else "fp32"
        self.lr = lr
        self.lw = local_world
        if local_world is not None:
            if self.world > 1:
                raise ValueError("local_world hosts a whole world in one process: do not combine with torch.distributed")
            self.world = local_world.world
            self.li = local_world._join(self)
            self.rank = self.li
            if self.li > 0:  # the broadcast of the initial parameters
                with torch.no_grad():
                    for p, p0 in zip(self.params, local_world.replicas[0].params_registration):
                        p.data.copy_(p0.data)
        else:
            self.li = 0
        self.params_registration = list(self.params)
        if self.world > 1 and local_world is None:
            with torch.no_grad():  # every rank starts from rank 0's values (before any forward)
                for p in self.params:
                    dist.broadcast(p.data, src=0)
        if drain_bytes is None:
            # N>1: sync overlaps the backward pass (a DRAIN launch per 4 MB of gradients).
            # N=1 there is nothing to overlap: no DRAIN launches (the backward keeps every SM)
            # and one FINISH launch over the whole GPU updates the parameters in priority order
            drain_bytes = 4 << 20 if self.world > 1 else 1 << 62
        if finish_ctas is None:
            finish_ctas = 0 if self.world > 1 else torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        self._ctx_kwargs = dict(
            max_slice=max_slice, lr=lr, momentum=momentum, priority_mode=priority_mode, comm_ctas=comm_ctas,
            comm_threads=comm_threads, timeout_s=timeout_s, trace_cap=trace_cap, drain_bytes=drain_bytes,
            plan_mode=plan_mode, throttle_bps=throttle_bps, throttle_burst=throttle_burst,
            big_threshold=big_threshold, pub_batch_bytes=pub_batch_bytes, drain_linger_us=drain_linger_us,
            finish_ctas=finish_ctas, push_dtype=push_dtype,
            notify_pull=(plan_mode == "baseline") if notify_pull is None else notify_pull,
            param_dtype=self.param_dtype,
            nvls=nvls,  # opt-in multicast broadcasts (one process per GPU; include/p3.h cfg.nvls)
        )
        self.ctx: SyncContext | None = None
        self.comm_stream = None
        self._launched = -1
        self._start()

    # -- lazy construction (once the layer order is known)
    def _finish_setup(self, perm: list[int]) -> None:
        lw = self.lw
        if lw is not None and self.li > 0:
            if lw._perm is None:
                raise RuntimeError("replica 0 of a local world must run its first forward first")
            perm = lw._perm  # every replica uses replica 0's layer order
        elif lw is not None:
            lw._perm = perm
        super()._finish_setup(perm)

    def _setup(self) -> None:
        counts = [p.numel() for p in self.params]
        groups = [0] * len(self.params)
        for gi, (_, layers) in enumerate(self._module_layers):
            for l in layers:
                groups[l] = gi
        for j, l in enumerate(self._orphans):
            groups[l] = len(self._module_layers) + j
        self._group_of = groups
        lw = self.lw
        if lw is None:
            self.ctx = SyncContext(counts, self.world, [self.rank], gate_groups=groups, **self._ctx_kwargs)
            connect(self.ctx)  # every rank's arena, after checking all ranks built the same plan
            self.comm_stream = torch.cuda.Stream(priority=-1)
        else:
            if lw.ctx is None:
                kw = dict(self._ctx_kwargs)
                kw.update(lw.ctx_kwargs)
                lw.ctx = SyncContext(counts, lw.world, list(range(lw.world)), gate_groups=groups, **kw)
                lw.comm_stream = torch.cuda.Stream(priority=-1)
            self.ctx = lw.ctx
            self.comm_stream = lw.comm_stream
        arena = self.ctx.params_arena(self.li)
        with torch.no_grad():
            for l, p in enumerate(self.params):
                off = self.ctx.layer_offsets[l]
                flat = arena[off : off + p.numel()]
                if p.is_contiguous() or not _dense(p):
                    view = flat.view(p.shape)
                else:  # keep e.g. channels_last weights in their memory order
                    view = flat.as_strided(p.shape, p.stride())
                view.copy_(p.data)
                p.data = view
        if self.param_dtype == "bf16":  # the owners' fp32 masters start from the replica's values
            self.ctx.master_init(self.li, torch.cuda.current_stream())
        torch.cuda.synchronize()
        if self.world > 1 and lw is None:
            dist.barrier()
        self._grads: list = []

    # -- hooks
    def _begin_iteration(self) -> None:
        if not self._set_up or self._launched == self.k:
            return
        for p in self.params:
            if p.grad is not None:
                # the comm kernel of the previous iteration may still read this gradient
                p.grad.record_stream(self.comm_stream)
                p.grad = None
        if self.lw is not None:
            self.lw.begin(self.k)
        else:
            self.ctx.iteration_begin(self.k, self.comm_stream)
        self._launched = self.k

    def _gate(self, l: int) -> None:
        self.ctx.wait_layer(self.li, l, self.k)

    def _gate_layers(self, layers) -> None:
        # one stream memory wait per gate group (every layer of a group is in one module)
        for g in sorted({self._group_of[l] for l in layers}):
            self.ctx.wait_group(self.li, g, self.k)

    def _publish(self, l: int, grad) -> None:
        p = self.params[l]
        if grad.dtype != p.dtype or grad.stride() != p.stride():
            grad = _relayout(grad, p)
            p.grad = grad
        self.ctx.layer_ready(self.li, l, self.k, grad)

    def _after_backward(self) -> None:
        if self.lw is not None:
            self.lw.end(self.li, self.k)
        else:
            self.ctx.iteration_end(self.k)

    # -- API
    def launches(self) -> int:
        """Comm kernel launches so far (0 before the first forward built the context)."""
        return self.ctx.launches() if self.ctx is not None else 0

    def layer_names(self) -> list[str]:
        """Parameter names in priority (forward) order: layer index i = priority i."""
        names = {id(p): n for n, p in self.module.named_parameters()}
        return [names.get(id(p), "?") for p in self.params]

    def synchronize(self, timeout_s: float | None = None) -> None:
        """Block until every layer holds the parameters of the last finished iteration."""
        if self.ctx is None:
            return
        self.ctx.sync_all(self.k, timeout_s)
        torch.cuda.current_stream().wait_stream(self.comm_stream)

    def close(self) -> None:
        """Detach: parameters get their own storage again (a copy of the synced values)
        before the context (and its parameter arena) is destroyed."""
        self.remove_hooks()
        if self.ctx is None:
            return
        try:
            self.synchronize()
        except Exception:  # noqa: BLE001 - detach anyway
            pass
        with torch.no_grad():
            for p in self.params:
                p.data = p.data.clone(memory_format=torch.preserve_format)
                p.grad = None
        torch.cuda.synchronize()
        if self.lw is None:
            self.ctx.close()
        else:
            self.lw.replicas[self.li] = None
            if all(r is None for r in self.lw.replicas):
                self.ctx.close()
                self.lw.ctx = None


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
    out = torch.empty_strided(p.shape, p.stride(), dtype=p.dtype, device=p.device)
    out.copy_(grad)
    return out


class LayerwiseDataParallel(_HookedDataParallel):
    """Baseline: per-tensor NCCL all-reduce (FIFO in backward order) + SGD before reuse."""

    def __init__(self, module: torch.nn.Module, lr: float, order: str = "forward") -> None:
        super().__init__(module, order)
        self.lr = lr
        if self.world > 1:
            with torch.no_grad():
                for p in self.params:
                    dist.broadcast(p.data, src=0)
        self._work: dict[int, object] = {}
        self._start()

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
        if not self._set_up:
            return
        for l in range(len(self.params)):
            self._gate(l)
        torch.cuda.current_stream().synchronize()

    def close(self) -> None:
        self.remove_hooks()
