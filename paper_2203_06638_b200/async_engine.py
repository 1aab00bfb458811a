"""The asynchronous engine: LPP-SGD / LAP-SGD on CUDA streams (a10-a12).

worker q = one GPU (or, in one process, one arena on a device) holding the
shared fp32 arena x_q; updater r = one CUDA stream driven by one host
thread (engine.py:315-383); averager = one host thread + a high-priority
stream running the round protocol of ``rounds.py`` and the K4 / NVLS data
plane (engine.py:385-453).  Both threads run either the Python loops
below (records, host-sampled reference rng, host batches, quiescent
pauses, eval points) or their native forms (``native_loops``: the whole
loop in one GIL-free C call).  ``run_serialized`` is the canonical
deterministic interleaving used as the parity mode.
"""

from __future__ import annotations

import os
import threading
import time

import numpy as np
import torch

from . import _native as N
from .arena import Arena, enable_peer_access
from .paramstore import AtomicCounter, ParamStore
from .partition import BlockChoice, SelectionReason, select_block
from .records import AveragerStamp, RunConfig, UpdateRecord
from .rounds import RoundControl, averager_loop
from .sampling import worker_sampler
from .schedules import lr_at, sync_every
from .native_loops import NativeLoops
from .step import StepProgram


def shard_bounds(dim: int, workers: int) -> list[tuple[int, int]]:
    """Owner shards [lo, hi), boundaries rounded to 4 elements (16 bytes)."""
    cuts = [0]
    for q in range(1, workers):
        c = (dim * q // workers) // 4 * 4
        cuts.append(max(cuts[-1], min(c, dim)))
    cuts.append(dim)
    return [(cuts[q], cuts[q + 1]) for q in range(workers)]


# ---------------------------------------------------------------------------
# quiescent mode (test-only, engine.py:153-196)


class PauseGate:
    """Lets an averager fence its worker's updaters between two steps.

    Same contract as the reference's gate (engine.py:153-196): updaters
    pass ``checkpoint`` before claiming a slot; ``pause`` returns once every
    registered updater is parked there.  On the GPU the averager then also
    drains the updater streams, so no device write overlaps the round."""

    def __init__(self):
        self._cv = threading.Condition()
        self._active = 0
        self._idle = 0
        self._paused = False

    def register(self) -> None:
        with self._cv:
            self._active += 1

    def leave(self) -> None:
        with self._cv:
            self._active -= 1
            self._cv.notify_all()

    def checkpoint(self) -> None:
        with self._cv:
            if not self._paused:
                return
            self._idle += 1
            self._cv.notify_all()
            while self._paused:
                self._cv.wait()
            self._idle -= 1
            self._cv.notify_all()

    def pause(self) -> None:
        with self._cv:
            self._paused = True
            while self._idle < self._active:
                self._cv.wait()

    def resume(self) -> None:
        with self._cv:
            self._paused = False
            self._cv.notify_all()


# ---------------------------------------------------------------------------
# workers


class _Worker:
    def __init__(self, engine: "_Engine", q: int, device: int, x0: torch.Tensor):
        cfg = engine.cfg
        self.q = q
        self.device = device
        self.dev = torch.device("cuda", device)
        self.store = ParamStore(x0, device=device, mode=cfg.apply_mode)
        self.exited = AtomicCounter(0)
        self.synced_at = AtomicCounter(0)
        self.gate = PauseGate() if cfg.quiescent else None
        d = engine.dim
        U = cfg.updaters
        with torch.cuda.device(device):
            self.streams = [torch.cuda.Stream(device=device) for _ in range(U)]
            self.avg_stream = torch.cuda.Stream(device=device, priority=-1)
            # optional: the apply of every updater on its own high-priority
            # stream, so parameter updates are not queued behind other
            # streams' convolutions (less staleness); ordered by events
            self.apply_streams = [torch.cuda.Stream(device=device, priority=-1) for _ in range(U)]
            self.graph_done = [torch.cuda.Event() for _ in range(U)]
            self.apply_done = [torch.cuda.Event() for _ in range(U)]
        self.replicas = [Arena(d, device) for _ in range(U)]
        self.grads = [Arena(d, device) for _ in range(U)]
        self.moms = [Arena(d, device) for _ in range(U)] if cfg.momentum else [None] * U
        self.mean_out = torch.zeros(d + 4, dtype=torch.float32, device=self.dev)
        # K5 write tags (int32 stamps, an arena reinterpreted)
        self.tag_arena = Arena(d, device) if cfg.tracks else None
        self.tags = self.tag_arena.tensor.view(torch.int32) if cfg.tracks else None
        depth = cfg.in_flight + 2
        self.tag_pick = min(cfg.tag_sample, d)
        k = max(self.tag_pick, 1)
        # the worker's round-stamp cell on the device: the stamp of the last
        # round applied to this arena, written by the averager (lpp_set_i64)
        # before the host cell last_avg_stamp moves; the apply kernels read it
        # as k_claim and as the tag floor
        # Where the kernels read it: "device" (default) — a device mirror the
        # averager sets with a one-thread launch per round before the host
        # cell moves; "host" — the host cell itself in mapped pinned memory
        # (no device work per round, but every read is a PCIe round trip:
        # in-situ apply median 33 vs 20 us on ResNet-20, tools/exp_insitu_variants.py).
        # With more than 8 streams per device set CUDA_DEVICE_MAX_CONNECTIONS
        # >= 16 (bench.py does): at 8 hardware queues the averager's stream
        # shares one with a compute stream and the apply's p99 reaches ms
        self.round_cell_mode = os.environ.get("LPP_ROUND_CELL", "device")
        if self.round_cell_mode == "host":
            self.round_mem = N.HostBuffer(64)
            self.last_avg_stamp = AtomicCounter(0, cell=self.round_mem.view(np.int64, (1,)), index=0)
            self.round_cell = None
            self.avg_dev = self.round_mem.dev
        else:
            self.round_mem = None
            self.last_avg_stamp = AtomicCounter(0)
            self.round_cell = torch.zeros(1, dtype=torch.int64, device=self.dev)
            self.avg_dev = self.round_cell.data_ptr()
        # K5 step records, per updater and in-flight slot: {k_claim, clean,
        # tags[k] (int32)} — written on the device by the kernels (the tags at
        # the step's snapshot, (k_claim, clean) by its apply), copied to the
        # pinned ring after the apply; the sampled-tag indices go the other
        # way (pinned ring -> device ring, before the step's graph)
        self.rec_cols = 2 + (k + 1) // 2
        if cfg.tracks:
            self.tag_idx_pinned = torch.zeros((U, depth, k), dtype=torch.long, pin_memory=True)
            self.tag_idx_np = self.tag_idx_pinned.numpy()
            self.tag_idx_ring = torch.zeros((U, depth, k), dtype=torch.long, device=self.dev)
            self.rec_dev = torch.zeros((U, depth, self.rec_cols), dtype=torch.long, device=self.dev)
            self.rec_pinned = torch.zeros((U, depth, self.rec_cols), dtype=torch.long, pin_memory=True)
            rec_np = self.rec_pinned.numpy()
            self.claim_np = rec_np[:, :, :2]
            self.tag_np = rec_np[:, :, 2:].view(np.int32)
            # fused runs: per-block write stamps (an update writes one block
            # range) and the block boundaries, on the device
            nb = cfg.partition.num_blocks
            self.block_stamps = torch.zeros(nb + 1, dtype=torch.int32, device=self.dev)
            self.block_bounds = torch.tensor(cfg.partition.boundaries, dtype=torch.long,
                                             device=self.dev)
            self.block_bounds_host = np.ascontiguousarray(cfg.partition.boundaries, dtype=np.int64)
            self.min_dev = torch.zeros((U, depth), dtype=torch.int32, device=self.dev)
        # full record mode keeps every update's whole tag snapshot (reference
        # full mode, engine.py:343-344); one buffer per in-flight slot
        self.snap_tags = None
        if cfg.tracks and cfg.record_mode == "full" and cfg.record_tensors:
            self.snap_tags = [[torch.zeros(d, dtype=torch.int32, device=self.dev)
                               for _ in range(depth)] for _ in range(U)]
        self.programs: list[StepProgram] = []
        self.idx_pinned = None
        self.batch_pinned = None

    def stage_idx(self, r: int, slot: int, idx, stream_ptr: int) -> int:
        """Sampled-tag indices of (updater r, slot): pinned ring -> device
        ring on ``stream_ptr``; returns the device address."""
        k = self.tag_pick
        self.tag_idx_np[r, slot, :k] = idx
        N.copy_async(self.tag_idx_ring[r, slot].data_ptr(), self.tag_idx_pinned[r, slot].data_ptr(),
                     8 * k, stream_ptr)
        return self.tag_idx_ring[r, slot].data_ptr()

    def rec_claim(self, r: int, slot: int) -> int:
        """Device address of step record (r, slot): (k_claim, clean)."""
        return self.rec_dev[r, slot].data_ptr()

    def rec_tags(self, r: int, slot: int) -> int:
        """Device address of step record (r, slot): its sampled tags (int32)."""
        return self.rec_dev[r, slot].data_ptr() + 16

    def copy_rec(self, r: int, slot: int, stream_ptr: int) -> None:
        N.copy_async(self.rec_pinned[r, slot].data_ptr(), self.rec_dev[r, slot].data_ptr(),
                     8 * self.rec_cols, stream_ptr)

    def publish_round(self, u: int, stream: torch.cuda.Stream) -> None:
        """The round with stamp u is applied to this arena: the device cell
        the kernels read as k_claim / tag floor (enqueued on the averager's
        stream) and the host cell."""
        if self.round_cell is not None:
            N.set_i64(self.avg_dev, u, stream.cuda_stream)
            # the Python averager serves the serialized / quiescent / record
            # modes, where the next steps must see the new stamp: wait (the
            # native averager, the throughput path, does not)
            stream.synchronize()
        self.last_avg_stamp.store(u)

    def build_programs(self, engine: "_Engine", block_ids_per_rank: list[list[int]]) -> None:
        cfg = engine.cfg
        obj = cfg.objective
        input_mode = "random" if cfg.sampling == "device" else "index"
        if engine.host_batches:
            input_mode = "batch"
        with torch.cuda.device(self.device):
            for r in range(cfg.updaters):
                # replica starts as a snapshot of the shared arena
                N.snapshot(self.store.arena.ptr, self.replicas[r].ptr, engine.dim,
                           self.streams[r].cuda_stream)
                blocks = {b: cfg.partition.block(b) for b in block_ids_per_rank[r]}
                self.programs.append(StepProgram(
                    obj, self.dev, self.replicas[r].tensor, self.grads[r].tensor, blocks,
                    cfg.batch_size, self.streams[r], input_mode=input_mode,
                    use_graphs=cfg.use_graphs, seed=cfg.seed * 7919 + self.q * 101 + r + 1,
                    epoch=self.epoch_shard(engine) if cfg.epoch_partition else None,
                    nbuf=2))
            depth = cfg.in_flight + 2
            self.loss_pinned = torch.zeros((cfg.updaters, depth), dtype=torch.float32, pin_memory=True)
            self.idx_pinned = torch.zeros((cfg.updaters, depth, cfg.batch_size), dtype=torch.long,
                                          pin_memory=True)
            if engine.host_batches:
                shape = obj.features.shape[1:]
                self.batch_pinned = torch.zeros((cfg.updaters, depth, cfg.batch_size, *shape),
                                                dtype=obj.features.dtype, pin_memory=True)
                self.label_pinned = torch.zeros((cfg.updaters, depth, cfg.batch_size),
                                                dtype=obj.labels.dtype, pin_memory=True)
                # H2D prefetch: a copy stream per updater fills a device ring,
                # overlapping the previous step's compute; the step then does
                # a D2D into the captured graph's static input
                U_ = cfg.updaters
                self.copy_streams = [torch.cuda.Stream(device=self.device) for _ in range(U_)]
                self.copied = [[torch.cuda.Event() for _ in range(depth)] for _ in range(U_)]
                self.buf_free = [[torch.cuda.Event() for _ in range(2)] for _ in range(U_)]
            # numpy views of the pinned staging rings: the per-step host
            # writes/reads skip the framework's dispatch
            self.idx_np = self.idx_pinned.numpy()
            # the warm-up passes touched the replica/grad arenas and BN stats
            # only; re-snapshot so every replica starts at x0
            for r in range(cfg.updaters):
                N.snapshot(self.store.arena.ptr, self.replicas[r].ptr, engine.dim,
                           self.streams[r].cuda_stream)
            torch.cuda.synchronize(self.device)

    def epoch_shard(self, engine: "_Engine") -> tuple[int, int, int]:
        """This worker's index shard arange(n)[q::Q] as (base, stride, length)
        (engine.py:294-296)."""
        n, Q = engine.cfg.objective.n_samples, engine.cfg.workers
        return self.q, Q, (n - self.q + Q - 1) // Q

    def close(self):
        """Free every device resource now: captured graphs first, then the
        arenas (a failed run may leave this worker in a reference cycle, and
        a later collector pass must not free device memory mid-capture)."""
        torch.cuda.synchronize(self.device)
        for p in self.programs:
            p.close()
        self.programs = []
        extra = [self.tag_arena] if self.tag_arena is not None else []
        for a in (self.replicas + self.grads + [m for m in self.moms if m is not None] + extra
                  + [self.store.arena]):
            a.close()
        if self.store.tag_arena is not None:
            self.store.tag_arena.close()
        self.tags = None
        if self.round_mem is not None:
            self.round_mem.close()


class _Engine(NativeLoops):
    """Shared machinery of the asynchronous run (in-process workers)."""

    def __init__(self, cfg: RunConfig, host_batches: bool = False, time_apply: bool = False,
                 group=None):
        self.cfg = cfg
        obj = cfg.objective
        self.dim = obj.dim
        self.host_batches = host_batches
        self.time_apply = time_apply
        self.group = group  # multi-process attachment (None: all workers in this process)
        # K5: rounds write their stamp into every element's tag only in full
        # record mode (whole-vector tag snapshots); otherwise the round floor
        # stands for it — the updaters' tag gathers read max(tag, last round
        # stamp), so averaging writes no tags and takes no stamp fence
        self.round_tags = cfg.tracks and cfg.record_mode == "full"
        self.x0_host = np.asarray(obj.init_params(cfg.seed), dtype=np.float64)
        x0 = torch.from_numpy(self.x0_host.astype(np.float32))
        if group is None:
            devs = cfg.devices or (torch.cuda.current_device(),)
            self.local_workers = list(range(cfg.workers))
            dev_of = [devs[q % len(devs)] for q in range(cfg.workers)]
        else:
            self.local_workers = [group.rank]
            dev_of = {group.rank: torch.cuda.current_device()}
        self.workers: dict[int, _Worker] = {}
        for q in self.local_workers:
            self.workers[q] = _Worker(self, q, dev_of[q], x0)
        if group is None:
            for a in self.local_workers:
                for b in self.local_workers:
                    if self.workers[a].device != self.workers[b].device:
                        if not enable_peer_access(self.workers[a].device, self.workers[b].device):
                            raise RuntimeError("averaging needs peer access between worker devices")
            self.arena_ptrs = [self.workers[q].store.arena.ptr for q in range(cfg.workers)]
            self.tag_ptrs = ([self.workers[q].tag_arena.ptr for q in range(cfg.workers)]
                             if self.round_tags else None)
            self.ctrl = RoundControl(cfg.workers)
        else:
            group.reset_control()
            n_peers = len(group.peers)
            self.arena_ptrs = group.attach_arenas(self.workers[group.rank].store.arena)
            self.tag_ptrs = (group.attach_arenas(self.workers[group.rank].tag_arena)
                             if self.round_tags else None)
            # this engine's IPC mappings of the peers' arenas (closed with it)
            self._peer_maps = group.peers[n_peers:]
            self.ctrl = group.control
        self.shards = shard_bounds(self.dim, cfg.workers)
        self.nvls = {}
        if cfg.averaging == "nvls" and cfg.algo in ("lap_sgd", "lpp_sgd"):
            from .nvls import NvlsGroup

            for q in self.local_workers:
                self.nvls[q] = NvlsGroup(self.dim, cfg.workers, self.workers[q].device, group=group)
        lpp = cfg.algo == "lpp_sgd"
        ids = [[0] + ([r + 1] if lpp else []) for r in range(cfg.updaters)]
        for w in self.workers.values():
            w.build_programs(self, ids)
        self.flops = AtomicCounter(0)
        self.clean_count = AtomicCounter(0)
        self.classified_count = AtomicCounter(0)
        self.updates: list[list[UpdateRecord]] = [[] for _ in range(cfg.workers * cfg.updaters)]
        self.stamps: list[list[AveragerStamp]] = [[] for _ in range(cfg.workers)]
        self.errors: list[BaseException] = []
        self.err_lock = threading.Lock()
        self.apply_events: list = []
        self.native_apply = [0, 0.0, 0.0]   # launches, ms, bytes (native loop, time_apply)
        self.apply_ms_samples: list = []    # per-launch ms (native loop, time_apply)
        self._apply_logs: dict = {}
        self._records: dict = {}             # native loop record buffers per (worker, updater)
        self.side_apply = False             # applies on the high-priority stream (set per run)
        self.k4_timing = [0, 0.0]           # in-situ K4 rounds, summed ms (native averager, time_apply)
        self.native_lock = threading.Lock()
        self.t0 = 0.0
        self.budget = cfg.budget
        self.read_loss = False
        self.loss_log: list = []
        self.nvtx: str | None = None   # per-thread NVTX range name for profiling a phase
        self.eval_points: list = []
        mu, wd = cfg.momentum, cfg.weight_decay
        # algorithmic bytes per element of K1/K2: read g, read +
        # write x (the weight-decay read of x is that same read), + read and
        # write the per-stream momentum buffer, + the int32 write tag (K5)
        # (fused runs keep per-BLOCK stamps: no per-element tag bytes)
        self.apply_bytes_per_elem = 12 + (8 if mu else 0) + (4 if cfg.tracks and not self.fused() else 0)
        fwd = obj.forward_cost()
        self._flops_of = {b: cfg.batch_size * (fwd + obj.backward_cost(cfg.partition.block(b)))
                          for b in range(cfg.partition.num_blocks + 1)}
        self._bflops_of = {b: cfg.batch_size * obj.backward_cost(cfg.partition.block(b))
                           for b in range(cfg.partition.num_blocks + 1)}

    def reset(self, budget: int) -> None:
        """Start a new phase of ``budget`` slots per worker on the same
        arenas and captured graphs (counters, control block and logs reset)."""
        self.budget = int(budget)
        for w in self.workers.values():
            for c in (w.store.sample_counter, w.store.update_order_counter, w.exited,
                      w.last_avg_stamp, w.synced_at):
                c.store(0)
        if self.group is None:
            self.ctrl.buf[:] = 0
        else:
            self.group.reset_control()
        self.flops.store(0)
        self.clean_count.store(0)
        self.classified_count.store(0)
        for w in self.workers.values():
            if w.round_cell is not None:
                w.round_cell.zero_()
            if w.tags is not None:
                w.tags.zero_()
                w.block_stamps.zero_()
        torch.cuda.synchronize()
        self.updates = [[] for _ in range(self.cfg.workers * self.cfg.updaters)]
        self.stamps = [[] for _ in range(self.cfg.workers)]
        self.errors = []
        self.apply_events = []
        self.native_apply = [0, 0.0, 0.0]
        self.apply_ms_samples = []
        self.k4_timing = [0, 0.0]
        self.loss_log = []
        self.eval_points = []

    # -- one updater step: K3 -> graph -> K1/K2, all on the updater stream --

    def step(self, w: _Worker, r: int, s: int, block_id: int, lr: float, batch, slot: int,
             u: int = 0, tag_idx=None, rec=None, buf: int = 0):
        cfg = self.cfg
        stream = w.streams[r]
        prog = w.programs[r]
        blk = cfg.partition.block(block_id)
        sp = stream.cuda_stream
        tracks = w.tags is not None
        with torch.cuda.stream(stream):
            if batch is not None:
                if self.host_batches:
                    self.stage_host_batch(w, r, batch, slot, buf)
                else:
                    w.idx_np[r, slot] = batch
                    N.copy_async(prog.idx.data_ptr(), w.idx_pinned[r, slot].data_ptr(),
                                 8 * cfg.batch_size, sp)
            if not tracks:
                N.snapshot(w.store.arena.ptr, w.replicas[r].ptr, self.dim, sp)       # K3
            elif cfg.record_mode == "full":
                # K5: full tagged snapshot; the min tag decides "clean"
                w.min_dev[r, slot].fill_(2**31 - 1)
                out_tags = None
                if w.snap_tags is not None and rec is not None:
                    out_tags = w.snap_tags[r][slot].data_ptr()
                N.snapshot_tagged(w.store.arena.ptr, w.tag_arena.ptr, w.replicas[r].ptr, out_tags,
                                  self.dim, w.min_dev[r, slot].data_ptr(), sp)
            else:
                # K5: sampled tags are gathered BEFORE the value copy (paramstore.py:108-112)
                self.gather_tags(w, r, slot, tag_idx)
                N.snapshot(w.store.arena.ptr, w.replicas[r].ptr, self.dim, sp)       # K3
            prog.run(block_id, buf)                                                   # fwd+bwd
            if self.host_batches:
                w.buf_free[r][buf].record(stream)
            if rec is not None and cfg.record_mode == "full" and cfg.record_tensors:
                rec.grad = w.grads[r].tensor[blk.start:blk.stop].clone()
                rec.snapshot = w.replicas[r].tensor.clone()
            off = 4 * blk.start
            mom = w.moms[r]
            astream = stream
            if self.side_apply:
                astream = w.apply_streams[r]
                w.graph_done[r].record(stream)
                astream.wait_event(w.graph_done[r])
                sp = astream.cuda_stream
            if self.time_apply:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(astream)
            if tracks:                                                                # K1/K2 + K5
                self.classify_on_device(w, r, slot, sp)
                N.apply_sgd_tagged(w.store.arena.ptr + off, w.grads[r].ptr + off,
                                   (mom.ptr + off) if mom is not None else None, blk.length,
                                   float(lr), None, cfg.momentum, cfg.weight_decay,
                                   N.MODES[cfg.apply_mode], w.tag_arena.ptr + off, u, sp)
            else:
                N.apply_sgd(w.store.arena.ptr + off, w.grads[r].ptr + off,          # K1/K2
                            (mom.ptr + off) if mom is not None else None, blk.length, float(lr),
                            None, cfg.momentum, cfg.weight_decay, N.MODES[cfg.apply_mode], sp)
            if self.time_apply:
                e1.record(astream)
                self.apply_events.append((e0, e1, self.apply_bytes_per_elem * blk.length))
            if astream is not stream:
                w.apply_done[r].record(astream)
                stream.wait_event(w.apply_done[r])
            if tracks:   # (k_claim, clean) + tags -> host, on the updater stream
                w.copy_rec(r, slot, stream.cuda_stream)
            if self.read_loss:
                self.read_back_loss(w, r, slot, buf)

    def stage_host_batch(self, w: _Worker, r: int, batch, slot: int, buf: int) -> None:
        """End-to-end input: gather the batch on the host into a pinned slot,
        H2D on the updater's copy stream straight into the graph's input
        buffer ``buf`` once the step that last read it is done (overlapping
        the previous step's compute), then make the compute stream wait."""
        cfg = self.cfg
        stream = w.streams[r]
        prog = w.programs[r]
        feats, labs = cfg.objective.features, cfg.objective.labels
        xs, ls = w.batch_pinned[r, slot], w.label_pinned[r, slot]
        n = feats.shape[0]
        N.host_gather_rows(xs.data_ptr(), feats.data_ptr(), n, xs[0].numel() * xs.element_size(), batch)
        N.host_gather_rows(ls.data_ptr(), labs.data_ptr(), n, ls.element_size(), batch)
        cs = w.copy_streams[r]
        cs.wait_event(w.buf_free[r][buf])
        with torch.cuda.stream(cs):
            prog.xbs[buf].copy_(w.batch_pinned[r, slot], non_blocking=True)
            prog.ybs[buf].copy_(w.label_pinned[r, slot], non_blocking=True)
            w.copied[r][slot].record(cs)
        stream.wait_event(w.copied[r][slot])

    def read_back_loss(self, w: _Worker, r: int, slot: int, buf: int) -> None:
        """The step's loss back to the host (end-to-end measurement).  In the
        compute stream: a separate out stream + event waits measured slower
        (146k vs 151k images/s on ResNet-20)."""
        prog = w.programs[r]
        w.loss_pinned[r, slot].copy_(prog.loss_of(buf), non_blocking=True)

    def loss_value(self, w: _Worker, r: int, slot: int, buf: int) -> float:
        return float(w.loss_pinned[r, slot])

    def fused(self) -> bool:
        """Whether async steps use the fused apply+next-snapshot kernel."""
        cfg = self.cfg
        # the fused K5 plan carries at most 32 sampled tags (and block ids
        # < 128) in its launch parameters; larger ones take the unfused
        # per-element path
        return (cfg.fuse_snapshot and cfg.schedule == "async" and not cfg.quiescent
                and cfg.record_mode != "full" and cfg.apply_mode != "plain"
                and (not cfg.tracks or (min(cfg.tag_sample, self.dim) <= 32
                                        and cfg.partition.num_blocks <= 127)))

    def gather_tags(self, w: _Worker, r: int, slot: int, tag_idx) -> None:
        """K5: the step's sampled tags, raised to the round floor, into slot
        (the step's device record); on the updater stream before the
        snapshot values it describes (paramstore.py:108-112).  The indices are
        copied to a device ring first, in stream order."""
        k = w.tag_pick
        sp = w.streams[r].cuda_stream
        idx_dev = w.stage_idx(r, slot, tag_idx, sp)
        if self.fused():   # fused runs stamp blocks, not elements
            N.gather_block_stamps(w.block_stamps.data_ptr(), w.block_bounds.data_ptr(),
                                  self.cfg.partition.num_blocks, idx_dev, k, w.avg_dev,
                                  w.rec_tags(r, slot), None, sp)
        else:
            N.gather_tags_floor(w.tag_arena.ptr, idx_dev, k, w.avg_dev, w.rec_tags(r, slot), None, sp)

    def classify_on_device(self, w: _Worker, r: int, slot: int, stream_ptr: int) -> None:
        """K5 classification at apply time (engine.py:353-362): k_claim is
        read by the kernel when it runs, i.e. after the step's gradient."""
        if self.cfg.record_mode == "full":
            N.classify(w.min_dev[r, slot].data_ptr(), 1, w.avg_dev, w.rec_claim(r, slot), stream_ptr)
        else:
            N.classify(w.rec_tags(r, slot), w.tag_pick, w.avg_dev, w.rec_claim(r, slot), stream_ptr)

    def step_fused(self, w: _Worker, r: int, block_id: int, lr: float, batch, slot: int,
                   next_slot: int, u: int, first: bool, tag_idx, next_tag_idx,
                   buf: int = 0) -> None:
        """One async step with K1+K3 fused: [first: gather + K3] -> graph ->
        apply(this) fused with snapshot(next) and the K5 plan (classify this
        step, read the next step's sampled tags) -> block stamp + record."""
        cfg = self.cfg
        stream = w.streams[r]
        prog = w.programs[r]
        blk = cfg.partition.block(block_id)
        sp = stream.cuda_stream
        tracks = w.tags is not None
        with torch.cuda.stream(stream):
            if batch is not None:
                if self.host_batches:
                    self.stage_host_batch(w, r, batch, slot, buf)
                else:
                    w.idx_np[r, slot] = batch
                    N.copy_async(prog.idx.data_ptr(), w.idx_pinned[r, slot].data_ptr(),
                                 8 * cfg.batch_size, sp)
            if first:
                if tracks:
                    self.gather_tags(w, r, slot, tag_idx)
                N.snapshot(w.store.arena.ptr, w.replicas[r].ptr, self.dim, sp)          # K3
            if tracks:   # the next step's indices: host ring, passed to the apply by value
                w.tag_idx_np[r, next_slot, :w.tag_pick] = next_tag_idx
            prog.run(block_id, buf)                                                      # fwd+bwd
            if self.host_batches:
                w.buf_free[r][buf].record(stream)
            plan = None
            if tracks:
                # K5 inside the apply: classify this step (k_claim read after
                # its gradient) and read the next step's sampled tags before
                # their values, after this apply's own reductions
                # (engine.py:343-362 order)
                k = w.tag_pick
                plan = N.TagPlan(w.tag_idx_pinned[r, next_slot].data_ptr(), w.rec_tags(r, next_slot),
                                 None, w.rec_tags(r, slot),
                                 w.rec_claim(r, slot), w.avg_dev, w.block_stamps.data_ptr(),
                                 w.block_bounds_host.ctypes.data,
                                 cfg.partition.num_blocks, block_id, k)
            mom = w.moms[r]
            astream = stream
            if self.side_apply:
                astream = w.apply_streams[r]
                w.graph_done[r].record(stream)
                astream.wait_event(w.graph_done[r])
                sp = astream.cuda_stream
            if self.time_apply:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(astream)
            if plan is not None:                                                         # K1+K3+K5
                N.apply_snapshot_plan(w.store.arena.ptr, w.grads[r].ptr,
                                      mom.ptr if mom is not None else None, w.replicas[r].ptr,
                                      None, self.dim, blk.start, blk.stop, float(lr), None,
                                      cfg.momentum, cfg.weight_decay, u, plan, sp)
            else:                                                                         # K1+K3
                N.apply_snapshot(w.store.arena.ptr, w.grads[r].ptr,
                                 mom.ptr if mom is not None else None, w.replicas[r].ptr,
                                 None, self.dim, blk.start, blk.stop,
                                 float(lr), None, cfg.momentum, cfg.weight_decay, u, sp)
            if self.time_apply:
                e1.record(astream)
                # block: read g, RMW x, (+m), (+tag); whole arena: read x outside
                # the block, write the replica
                nbytes = self.apply_bytes_per_elem * blk.length + 4 * (self.dim - blk.length) \
                    + 4 * self.dim
                self.apply_events.append((e0, e1, nbytes))
            if astream is not stream:
                w.apply_done[r].record(astream)
                stream.wait_event(w.apply_done[r])
            # K5 bookkeeping on the updater stream, after the apply: this
            # update's block stamp, then (k_claim, clean) + tags -> host
            if plan is not None:
                N.publish_stamp(w.block_stamps.data_ptr(), block_id, u, stream.cuda_stream)
            if tracks:
                w.copy_rec(r, slot, stream.cuda_stream)
            if self.read_loss:
                self.read_back_loss(w, r, slot, buf)

    def average(self, owner: int, stream: torch.cuda.Stream, final: bool, stamps=None) -> None:
        lo, hi = self.shards[owner]
        w = self.workers[owner]
        if self.cfg.workers == 1:
            # a single worker's mean is itself: the correction is exactly 0
            # (test_engine.py:169-182), so only the final mean is copied out
            # (and the round's stamp written into the tags, add_assign's tagging)
            if final:
                N.snapshot(w.store.arena.ptr, w.mean_out.data_ptr(), self.dim, stream.cuda_stream)
            if self.round_tags:
                with torch.cuda.stream(stream):
                    w.tags.fill_(int(stamps[0]))
            return
        mean_ptr = w.mean_out.data_ptr() + 4 * lo if final else None
        if self.tag_ptrs is not None:
            N.average_shard_tagged(self.arena_ptrs, self.tag_ptrs, stamps, lo, hi, mean_ptr,
                                   N.MODE_RED, stream.cuda_stream)
        else:
            N.average_shard(self.arena_ptrs, lo, hi, mean_ptr, N.MODE_RED, stream.cuda_stream)

    def nvls_round(self, q: int, u: int, final: bool, fence=None) -> None:
        """One NVLS round for worker q: stage -> (all staged) -> in-switch
        mean of the owned shard -> (all broadcast) -> local add of
        (mean - stage).  ``fence(i)`` is the group barrier between phases."""
        w = self.workers[q]
        nv = self.nvls[q]
        st = w.avg_stream
        sp = st.cuda_stream
        nv.stage_copy(w.store.arena.ptr, sp)
        st.synchronize()
        if fence is not None and not fence(0):
            return
        lo, hi = self.shards[q]
        nv.reduce_mean(lo, hi, sp)
        st.synchronize()
        if fence is not None and not fence(1):
            return
        nv.apply(w.store.arena.ptr, w.tag_arena.ptr if self.round_tags else None, u, sp)
        if final:
            with torch.cuda.stream(st):
                w.mean_out[: self.dim].copy_(nv.mean_tensor)
        st.synchronize()

    def fail(self, exc: BaseException) -> None:
        with self.err_lock:
            self.errors.append(exc)
        self.ctrl.abort.store(1)
        self.ctrl.stop.store(1)
        for w in self.workers.values():
            if w.gate is not None:
                w.gate.resume()

    def record_update(self, q, r, s, u, k_claim, choice: BlockChoice, lr, tag_idx=None):
        b = choice.block_id
        rec = UpdateRecord(
            worker=q, rank=r + 1, s=s, u=u, k_claim=k_claim, block_id=b, reason=choice.reason.value,
            lr=lr, flops=self._flops_of[b], backward_flops=self._bflops_of[b], clean=None,
            tag_indices=tag_idx)
        if self.cfg.record_mode != "off":
            self.updates[q * self.cfg.updaters + r].append(rec)
        return rec

    def classify(self, w: _Worker, r: int, slot: int, rec: UpdateRecord) -> None:
        """Clean iff every sampled (or every, in full mode) tag is at or after
        the last averaging stamp at apply time (engine.py:357-362).  The
        apply-side kernel already compared them; called once the step's
        event completed, this reads its (k_claim, clean) record."""
        if w.tags is None:
            return
        kc, cl = (int(v) for v in w.claim_np[r, slot])
        rec.k_claim = kc
        clean = bool(cl)
        if self.cfg.record_mode == "full":
            if self.cfg.record_tensors and rec.snapshot is not None and rec.tags is None:
                rec.tags = w.snap_tags[r][slot].cpu().numpy().astype(np.int64)
        else:
            rec.tags = w.tag_np[r, slot, :w.tag_pick].astype(np.int64)
        rec.clean = clean
        self.classified_count.add(1)
        if clean:
            self.clean_count.add(1)

    def p_hat(self) -> float:
        total = self.classified_count.read()
        return self.clean_count.read() / total if total else 1.0

    def choose(self, s: int, rank: int) -> BlockChoice:
        cfg = self.cfg
        if cfg.algo == "lpp_sgd":
            return select_block(s, cfg.warm_start_budget, cfg.partition.num_blocks, rank)
        return BlockChoice(0, SelectionReason.WARM_START)

    # -- asynchronous threads -------------------------------------------------

    def updater(self, q: int, r: int) -> None:
        cfg = self.cfg
        w = self.workers[q]
        torch.cuda.set_device(w.device)
        rank = r + 1
        gen = np.random.default_rng(np.random.SeedSequence([cfg.seed, q, rank]))
        n = cfg.objective.n_samples
        sampler = (worker_sampler(n, cfg.workers, q, rank, cfg.seed)
                   if cfg.epoch_partition and cfg.sampling == "host" else None)
        depth = cfg.in_flight + 2
        events = [torch.cuda.Event() for _ in range(cfg.in_flight)]
        used = [False] * cfg.in_flight
        pending = [None] * cfg.in_flight
        ctrl = self.ctrl
        sampled_tags = w.tags is not None and cfg.record_mode != "full"
        fused = self.fused()
        next_tag_idx = None

        def draw_tags():
            if not sampled_tags:
                return None
            return np.sort(gen.choice(self.dim, size=w.tag_pick, replace=False))

        s, t = 0, 0
        if w.gate is not None:
            w.gate.register()
        if self.nvtx:
            torch.cuda.nvtx.range_push(self.nvtx)
        try:
            while s < self.budget and not ctrl.stop.read():
                if w.gate is not None:
                    w.gate.checkpoint()
                s = w.store.read_and_inc()
                lr = lr_at(cfg.lr, s)
                choice = self.choose(s, rank)
                k = t % cfg.in_flight
                if used[k]:
                    events[k].synchronize()
                    old_slot = (t - cfg.in_flight) % depth
                    if self.read_loss:
                        self.loss_log.append(self.loss_value(w, r, old_slot, (t - cfg.in_flight) % 2))
                    self.classify(w, r, old_slot, pending[k])
                # reference rng order: sampled tag indices first, then the batch
                # (engine.py:343-351); the fused path draws the NEXT step's tag
                # indices right after this batch, which keeps that order
                if fused:
                    tag_idx = next_tag_idx if t else draw_tags()
                else:
                    tag_idx = draw_tags()
                batch = None
                if sampler is not None:
                    batch = sampler.next_batch(cfg.batch_size)
                elif cfg.sampling == "host":
                    batch = gen.integers(0, n, cfg.batch_size)
                k_claim = w.last_avg_stamp.read()
                u = w.store.claim_update_order()
                rec = self.record_update(q, r, s, u, k_claim, choice, lr, tag_idx)
                if fused:
                    next_tag_idx = draw_tags()
                    self.step_fused(w, r, choice.block_id, lr, batch, t % depth, (t + 1) % depth,
                                    u, t == 0, tag_idx, next_tag_idx, buf=t % 2)
                else:
                    self.step(w, r, s, choice.block_id, lr, batch, t % depth, u=u, tag_idx=tag_idx,
                              rec=rec, buf=t % 2)
                events[k].record(w.streams[r])
                used[k] = True
                pending[k] = rec
                self.flops.add(self._flops_of[choice.block_id])
                t += 1
            w.streams[r].synchronize()
            for tt in range(max(t - cfg.in_flight, 0), t):     # the last steps, in step order
                if used[tt % cfg.in_flight]:
                    if self.read_loss:
                        self.loss_log.append(self.loss_value(w, r, tt % depth, tt % 2))
                    self.classify(w, r, tt % depth, pending[tt % cfg.in_flight])
        except BaseException as exc:  # surfaced after join (engine.py:456-463)
            self.fail(exc)
        finally:
            if self.nvtx:
                torch.cuda.nvtx.range_pop()
            if w.gate is not None:
                w.gate.leave()
            if w.exited.add(1) + 1 == cfg.updaters:
                ctrl.drained.add(1)

    def averager(self, q: int) -> None:
        cfg = self.cfg
        w = self.workers[q]
        torch.cuda.set_device(w.device)
        store = w.store
        u_of = {}

        def do_round(r, final, s_cur):
            quiet = w.gate is not None
            evalm = cfg.eval_interval > 0
            # fence 0: every worker's stamp is published before owners write it
            # into the tags (full records) / every updater parked (quiescent);
            # fence 1: every owner is done with this worker's arena before the
            # round counts as applied (the updaters' k_claim and tag floor) and
            # before worker 0 reads the owners' round means (eval points)
            fenced0 = quiet or self.round_tags
            fenced1 = quiet or w.tags is not None or evalm
            if quiet:
                # quiescent: every worker's updaters parked and their streams
                # drained before any owner touches the arenas
                w.gate.pause()
                for st in w.streams:
                    st.synchronize()
            try:
                u_of[r] = store.claim_update_order()
                full = cfg.record_mode == "full" and cfg.record_tensors
                # the worker's own view before any owner corrects it (quiescent: exact)
                snap = w.store.arena.tensor.clone() if full else None
                if self.nvls:
                    self.nvls_round(q, u_of[r], final or full or evalm,
                                    fence=lambda i: self.ctrl.fence(i, r))
                    w.publish_round(u_of[r], w.avg_stream)
                    w.synced_at.store(s_cur)
                    if full:
                        snaps[r] = (snap, self.nvls[q].mean_tensor.clone() if q == 0 else None)
                    return
                stamps = None
                if fenced0:
                    # every worker's round stamp is published before the owners
                    # write them into the tags (K5); the round counts as applied
                    # to this worker's arena only when every owner is done
                    self.ctrl.publish_stamp(q, u_of[r])
                    if not self.ctrl.fence(0, r):
                        return
                    stamps = self.ctrl.stamps()
                self.average(q, w.avg_stream, final=final or full or evalm, stamps=stamps)
                w.avg_stream.synchronize()
                if fenced1 and not self.ctrl.fence(1, r):
                    return
                if full:
                    # the round mean, assembled from every owner's shard
                    # (engine.py:441 keeps it for worker 0 only)
                    mean = self.gather_round_mean() if q == 0 else None
                    snaps[r] = (snap, mean)
                w.publish_round(u_of[r], w.avg_stream)
                w.synced_at.store(s_cur)
            finally:
                if quiet:
                    w.gate.resume()

        snaps = {}
        next_eval = [cfg.eval_interval if cfg.eval_interval else self.budget + 1]

        def on_round(r, s_cur, k_delta, unanimous):
            snap, mean = snaps.pop(r, (None, None))
            wall = (time.perf_counter() - self.t0) * 1e3
            self.stamps[q].append(AveragerStamp(
                worker=q, round=r, u=u_of.pop(r), s_cur=s_cur, k_delta=k_delta,
                wall_ms=wall, snapshot=snap, mean=mean))
            # engine.py:445-451: worker 0 keeps the round mean at eval points
            if q == 0 and cfg.eval_interval and not unanimous and s_cur >= next_eval[0]:
                m = self.round_mean(q)
                self.eval_points.append((s_cur, r, wall, self.flops.read(), self.p_hat(), m))
                while next_eval[0] <= s_cur:
                    next_eval[0] += cfg.eval_interval

        if self.nvtx:
            torch.cuda.nvtx.range_push(self.nvtx)
        try:
            averager_loop(self.ctrl, workers=cfg.workers,
                          read_counter=store.sample_counter.read,
                          local_drained=lambda: w.exited.read() == cfg.updaters,
                          sync_period=lambda s: sync_every(cfg.sync, s),
                          do_round=do_round, on_round=on_round, stop_after=cfg.round_budget)
        except BaseException as exc:
            self.fail(exc)
        finally:
            if self.nvtx:
                torch.cuda.nvtx.range_pop()

    # -- drivers ------------------------------------------------------------------

    def _device_span_start(self):
        evs = {}
        for q, w in self.workers.items():
            with torch.cuda.device(w.device):
                torch.cuda.synchronize(w.device)
                e = torch.cuda.Event(enable_timing=True)
                e.record(torch.cuda.current_stream(w.device))
                evs[q] = e
        return evs

    def _device_span_end(self, starts) -> float:
        ms = 0.0
        for q, w in self.workers.items():
            with torch.cuda.device(w.device):
                cur = torch.cuda.current_stream(w.device)
                side = getattr(w, "copy_streams", None) or []
                for s in w.streams + [w.avg_stream] + side:
                    cur.wait_stream(s)
                e = torch.cuda.Event(enable_timing=True)
                e.record(cur)
                e.synchronize()
                ms = max(ms, starts[q].elapsed_time(e))
        return ms

    def run_async(self) -> float:
        cfg = self.cfg
        if self.host_batches and cfg.sampling == "device" and not self.native_loop():
            raise ValueError("host batches drawn from the device sampler's stream need the native "
                             "loop (record_mode='off', host_loop != 'python'); the Python loop "
                             "samples host batches with sampling='host'")
        self.side_apply = self.apply_on_side()
        starts = self._device_span_start()
        threads = []
        for q in self.local_workers:
            target = self.averager_native if self.native_averager() else self.averager
            threads.append(threading.Thread(target=target, args=(q,), daemon=True,
                                            name=f"averager-{q}"))
        for q in self.local_workers:
            for r in range(cfg.updaters):
                target = self.updater_native if self.native_loop() else self.updater
                threads.append(threading.Thread(target=target, args=(q, r), daemon=True,
                                                name=f"updater-{q}-{r + 1}"))
        if self.group is not None:
            self.group.barrier()
        self.t0 = time.perf_counter()
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        self.wall_ms = (time.perf_counter() - self.t0) * 1e3
        dev_ms = self._device_span_end(starts)
        if self.group is not None:
            # peers may not release or reuse arenas until every owner is done
            self.group.barrier()
        if self.errors:
            # drop the engine's references to the failures before raising, so
            # engine -> errors -> traceback -> thread frame -> engine is no cycle
            first, self.errors = self.errors[0], []
            raise RuntimeError("engine thread failed") from first
        return dev_ms

    def run_serialized(self) -> float:
        """Canonical deterministic schedule (oracle/schedule.py)."""
        cfg = self.cfg
        self.side_apply = bool(cfg.apply_priority)
        if self.group is not None:
            raise ValueError("the serialized schedule runs in one process")
        n = cfg.objective.n_samples
        gens = {(q, r): np.random.default_rng(np.random.SeedSequence([cfg.seed, q, r + 1]))
                for q in range(cfg.workers) for r in range(cfg.updaters)}
        samplers = ({(q, r): worker_sampler(n, cfg.workers, q, r + 1, cfg.seed)
                     for q in range(cfg.workers) for r in range(cfg.updaters)}
                    if cfg.epoch_partition else None)
        active = {(q, r): True for q in range(cfg.workers) for r in range(cfg.updaters)}
        s_pre = [0] * cfg.workers
        self.round_trace = []
        next_eval = cfg.eval_interval if cfg.eval_interval else self.budget + 1
        starts = self._device_span_start()
        self.t0 = time.perf_counter()
        sweep, t = 0, 0
        while True:
            for q in range(cfg.workers):
                w = self.workers[q]
                for r in range(cfg.updaters):
                    if not active[(q, r)]:
                        continue
                    s = w.store.read_and_inc()
                    lr = lr_at(cfg.lr, s)
                    choice = self.choose(s, r + 1)
                    tag_idx = None
                    if w.tags is not None and cfg.record_mode != "full":
                        tag_idx = np.sort(gens[(q, r)].choice(self.dim, size=w.tag_pick,
                                                              replace=False))
                    if samplers is not None:
                        batch = samplers[(q, r)].next_batch(cfg.batch_size)
                    else:
                        batch = gens[(q, r)].integers(0, n, cfg.batch_size)
                    k_claim = w.last_avg_stamp.read()
                    u = w.store.claim_update_order()
                    slot = t % (cfg.in_flight + 2)
                    rec = self.record_update(q, r, s, u, k_claim, choice, lr, tag_idx)
                    self.step(w, r, s, choice.block_id, lr, batch, slot, u=u, tag_idx=tag_idx,
                              rec=rec, buf=t % 2)
                    w.streams[r].synchronize()
                    for st_ in getattr(w, "copy_streams", None) or []:
                        st_.synchronize()
                    self.classify(w, r, slot, rec)
                    self.flops.add(self._flops_of[choice.block_id])
                    t += 1
                    if s >= self.budget:
                        active[(q, r)] = False
            sweep += 1
            drained = not any(active.values())
            counts = [self.workers[q].store.sample_counter.read() for q in range(cfg.workers)]
            fresh = any(counts[q] - s_pre[q] >= sync_every(cfg.sync, counts[q])
                        for q in range(cfg.workers))
            if fresh or drained:
                rnd = len(self.round_trace) + 1
                u_avgs = [self.workers[q].store.claim_update_order() for q in range(cfg.workers)]
                full = cfg.record_mode == "full" and cfg.record_tensors
                snaps = [self.workers[q].store.arena.tensor.clone() if full else None
                         for q in range(cfg.workers)]
                for q in range(cfg.workers):
                    w = self.workers[q]
                    if self.nvls:
                        self.nvls_round(q, u_avgs[q], drained or full)
                    else:
                        self.average(q, w.avg_stream, final=drained or full or cfg.eval_interval > 0,
                                 stamps=u_avgs)
                    w.avg_stream.synchronize()
                mean = (self.gather_round_mean() if not self.nvls else
                        self.nvls[0].mean_tensor.clone()) if full else None
                if cfg.eval_interval and not drained and counts[0] >= next_eval:
                    m = mean if mean is not None else self.round_mean(0)
                    self.eval_points.append((counts[0], rnd, (time.perf_counter() - self.t0) * 1e3,
                                             self.flops.read(), self.p_hat(), m))
                    while next_eval <= counts[0]:
                        next_eval += cfg.eval_interval
                for q in range(cfg.workers):
                    w = self.workers[q]
                    u_avg = u_avgs[q]
                    w.publish_round(u_avg, w.avg_stream)
                    self.stamps[q].append(AveragerStamp(
                        worker=q, round=rnd, u=u_avg, s_cur=counts[q], k_delta=counts[q] - s_pre[q],
                        wall_ms=(time.perf_counter() - self.t0) * 1e3, snapshot=snaps[q],
                        mean=mean if q == 0 else None))
                    s_pre[q] = counts[q]
                self.round_trace.append((rnd, sweep, *counts))
            if drained:
                break
        self.wall_ms = (time.perf_counter() - self.t0) * 1e3
        return self._device_span_end(starts)

    def round_mean(self, q: int) -> torch.Tensor:
        """The just-finished round's mean as seen by worker q (a device copy)."""
        if self.nvls:
            return self.nvls[q].mean_tensor.clone()
        m = self.gather_round_mean()
        if m is None:
            # multi-process P2P: the other shards' means live in the peers;
            # use this worker's arena right after the round (mean + racing updates)
            m = self.workers[q].store.arena.tensor.clone()
        return m

    def gather_round_mean(self):
        """The current round's mean from the owners' mean_out shards (one process)."""
        if self.group is not None:
            return None
        parts = [self.workers[q].mean_out[lo:hi] for q, (lo, hi) in enumerate(self.shards)]
        return torch.cat(parts).clone()

    def final_values(self) -> np.ndarray:
        """The last round's mean, gathered shard by shard from the owners."""
        if self.nvls:
            # every worker holds the whole broadcast mean
            q = self.local_workers[0]
            return self.workers[q].mean_out[: self.dim].cpu().numpy()
        if self.group is not None:
            return self.group.gather_mean(self.workers[self.group.rank].mean_out, self.shards)
        out = np.empty(self.dim, dtype=np.float32)
        for q, (lo, hi) in enumerate(self.shards):
            out[lo:hi] = self.workers[q].mean_out[lo:hi].cpu().numpy()
        return out

    def apply_timing(self):
        n, ms, nbytes = self.native_apply
        if not self.apply_events and not n:
            return ()
        ms += sum(e0.elapsed_time(e1) for e0, e1, _ in self.apply_events)
        nbytes += sum(b for _, _, b in self.apply_events)
        return (n + len(self.apply_events), ms, nbytes)

    def close(self):
        for nv in self.nvls.values():
            nv.close()
        self.nvls = {}
        if self.group is not None:
            # every rank is past its run (run_async ends on a group barrier):
            # drop this engine's peer mappings before the arenas go
            for pm in getattr(self, "_peer_maps", []):
                pm.close()
                if pm in self.group.peers:
                    self.group.peers.remove(pm)
            self._peer_maps = []
        for w in self.workers.values():
            w.close()
        self.errors = []
        self.apply_events = []
