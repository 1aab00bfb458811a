"""One updater's captured training step (the grad_block half of a6/a10).

``StepProgram`` binds an objective to a stream-private replica arena
(parameters) and gradient arena, and captures, per block id the updater can
be assigned, one CUDA graph that does

    gather batch (index_select from device data, or a staged host batch)
    -> forward -> loss -> autograd.grad over the block's leaf tensors
    -> one multi-tensor copy of those gradients into the gradient arena

so the block gradient lands in ``grads[block.start:block.stop]`` — exactly
the range the apply kernel then reads.  This is ``Objective.grad_block``
(objectives.py:286-308) with autograd doing the truncated backward
("specifying the leaf tensors ... w.r.t. which gradients are
needed").  The snapshot (K3) and the apply (K1/K2) are launched around the
replay by the engine through the C ABI.
"""

from __future__ import annotations

import gc
import threading

import torch

from .conv import mark_weight_grads
from .partition import Block

# kernels of this library launched from inside replayed step graphs (the
# conv_f32.cu convolutions): counted per graph at capture, summed per replay
# here and by the native loop (lpp_updater_stats.graph_kernels)
_GRAPH_KERNELS = [0]
_GK_LOCK = threading.Lock()


def add_graph_kernels(n: int) -> None:
    with _GK_LOCK:
        _GRAPH_KERNELS[0] += int(n)


def graph_kernel_count() -> int:
    """Library kernels run inside step-graph replays so far (process-wide)."""
    return _GRAPH_KERNELS[0]


def _lib_launches() -> int:
    from . import _native

    return _native.launch_count()


class StepProgram:
    def __init__(self, obj, device: torch.device, replica: torch.Tensor, grads: torch.Tensor,
                 blocks: dict[int, Block], batch_size: int, stream: torch.cuda.Stream,
                 input_mode: str = "index", use_graphs: bool = True, warmup: int = 2,
                 seed: int = 0, nbuf: int = 1, grad_mode: str = "copy",
                 epoch: tuple[int, int, int] | None = None):
        if input_mode not in ("index", "batch", "random"):
            raise ValueError(f"unknown input mode {input_mode!r}")
        self.obj = obj
        self.device = device
        self.stream = stream
        self.input_mode = input_mode
        self.grads = grads
        self.bound = obj.bind(replica, grads)
        self.feats = obj.features_on(device)
        self.labels = obj.labels_on(device)
        B = int(batch_size)
        self.batch_size = B
        self.idx = torch.zeros(B, dtype=torch.long, device=device)
        # "batch" mode: nbuf static input buffers, one captured graph variant per
        # buffer, so the next step's H2D can land in the buffer the running
        # step is not reading (no device-side staging copy)
        self.nbuf = nbuf if input_mode == "batch" else 1
        if input_mode == "batch":
            self.xbs = [torch.zeros((B, *self.feats.shape[1:]), dtype=self.feats.dtype, device=device)
                        for _ in range(self.nbuf)]
            self.ybs = [torch.zeros(B, dtype=self.labels.dtype, device=device) for _ in range(self.nbuf)]
            self.xb, self.yb = self.xbs[0], self.ybs[0]
        # the step's loss, one slot per input buffer so a D2H of step t's loss
        # can overlap step t+1 (which writes the other slot)
        self.losses = [torch.zeros((), dtype=torch.float32, device=device) for _ in range(self.nbuf)]
        self.loss = self.losses[0]
        # "random": the batch indices are drawn on the device inside the
        # captured graph (lpp_sample_indices: a splitmix64 stream keyed by
        # seed, advanced by a device-side step counter on every replay)
        self.sample_key = int(seed)
        self.sample_step = torch.zeros(1, dtype=torch.long, device=device)
        # epoch = (shard base, stride, length): the epoch-partition walk over
        # the worker's shard (lpp_sample_epoch) instead of i.i.d. draws
        self.epoch = epoch
        if input_mode == "random":
            from . import _native
            self._native_mod = _native
        self.blocks = dict(blocks)
        self.leaves = {}
        self.grad_views = {}
        for bid, blk in self.blocks.items():
            first, last = obj.tensors_of_block(blk)
            self.leaves[bid] = self.bound.params[first:last + 1]
            self.grad_views[bid] = self.bound.grad_views[first:last + 1]
        # "copy": autograd.grad over the block's leaves, then one multi-tensor
        # copy into the gradient arena's views; "accumulate": zero the block's
        # slice and let backward() accumulate into the views (one add kernel
        # per tensor) — same values, ~45 fewer launches per step for "copy"
        self.grad_mode = grad_mode
        if grad_mode == "accumulate" and not self.bound.mixed:
            raise ValueError("grad_mode='accumulate' needs fp32 parameters (bf16 shadow weights "
                             "have no arena .grad views)")
        self.graphs: dict[int, torch.cuda.CUDAGraph] = {}
        self.graph_kernels: dict[tuple[int, int], int] = {}
        self.use_graphs = use_graphs
        with torch.cuda.stream(stream):
            for _ in range(max(warmup, 1)):
                for bid in self.blocks:
                    self._body(bid)
            stream.synchronize()
            if use_graphs:
                # a cyclic-GC pass during capture may finalise an earlier run's
                # arenas or graphs (cudaFree / cudaGraphExecDestroy), which
                # invalidates the capture; torch 2.11 no longer collects before
                # capturing, so collect now and keep the collector off until done
                gc.collect()
                was_enabled = gc.isenabled()
                gc.disable()
                try:
                    pool = None
                    for bid in self.blocks:
                        for buf in range(self.nbuf):
                            g = torch.cuda.CUDAGraph()
                            l0 = _lib_launches()
                            # thread_local: a CUDA call on another thread (NCCL's
                            # watchdog polling its events on multi-GPU jobs)
                            # must not invalidate this capture
                            with torch.cuda.graph(g, pool=pool, stream=stream,
                                                  capture_error_mode="thread_local"):
                                self._body(bid, buf)
                            self.graph_kernels[(bid, buf)] = _lib_launches() - l0
                            pool = g.pool()
                            self.graphs[(bid, buf)] = g
                finally:
                    if was_enabled:
                        gc.enable()
                stream.synchronize()
        # the batch stream starts at step 0 on the first replay (warm-up
        # draws do not count), and the native loop's host-drawn batches
        # (end-to-end input) continue the same stream from host_step
        self.sample_step.zero_()
        self.host_step = 0
        # raw cudaGraphExec_t handles, launched straight through the C ABI
        # (no framework generator state to advance: sampling is our kernel)
        self.execs = {}
        if use_graphs:
            from . import _native

            self._native = _native
            for key, g in self.graphs.items():
                self.execs[key] = int(g.raw_cuda_graph_exec())

    def _body(self, bid: int, buf: int = 0) -> None:
        blk = self.blocks[bid]
        if self.input_mode == "random":
            sp = torch.cuda.current_stream().cuda_stream
            if self.epoch is not None:
                self._native_mod.sample_epoch(self.idx.data_ptr(), self.sample_step.data_ptr(),
                                              self.batch_size, *self.epoch, self.sample_key, sp)
            else:
                self._native_mod.sample_indices(self.idx.data_ptr(), self.sample_step.data_ptr(),
                                                self.batch_size, self.feats.shape[0],
                                                self.sample_key, sp)
        if self.input_mode == "batch":
            xb, yb = self.xbs[buf], self.ybs[buf]
        else:
            xb = self.feats.index_select(0, self.idx)
            yb = self.labels.index_select(0, self.idx)
        module = getattr(self.bound, "module", None)
        if module is not None:
            mark_weight_grads(module, self.leaves[bid])
        loss = self.obj.loss_on(self.bound, xb, yb)
        if self.grad_mode == "copy":
            grads = torch.autograd.grad(loss, self.leaves[bid])
            torch._foreach_copy_(self.grad_views[bid], list(grads))
        else:
            self.grads[blk.start:blk.stop].zero_()
            loss.backward(inputs=self.leaves[bid])
        self.losses[buf].copy_(loss.detach())

    def loss_of(self, buf: int) -> torch.Tensor:
        return self.losses[buf % self.nbuf]

    def run(self, bid: int, buf: int = 0) -> None:
        """Enqueue block ``bid``'s fwd+bwd (reading input buffer ``buf``)."""
        buf %= self.nbuf
        if self.execs:
            self._native.graph_launch(self.execs[(bid, buf)], self.stream.cuda_stream)
            add_graph_kernels(self.graph_kernels.get((bid, buf), 0))
        elif self.use_graphs:
            self.graphs[(bid, buf)].replay()
            add_graph_kernels(self.graph_kernels.get((bid, buf), 0))
        else:
            with torch.cuda.stream(self.stream):
                self._body(bid, buf)

    def close(self) -> None:
        """Release the captured graphs now (not whenever the collector
        reaches this object, which may be inside another capture)."""
        self.execs = {}
        for g in self.graphs.values():
            g.reset()
        self.graphs = {}
