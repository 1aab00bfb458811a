"""Native (C++) updater and averager loops of the asynchronous engine.

``lpp_updater_run`` / ``lpp_averager_run`` (``csrc/updater.cu``) run one
updater's step loop (a10, engine.py:289-383) and one worker's averager
(a11, engine.py:385-453) GIL-free; this mixin decides when they apply
(updaters: async, record mode off / light, the in-graph device sampler
or the reference's numpy stream restated in csrc/nprng.cu, with or without
end-to-end host batches; averagers: p2p averaging without quiescent pauses
or full records, eval points included) and builds their C configuration
structs from the engine's arenas, streams, captured graphs and host
counters.  The Python loops in ``async_engine`` remain the full-record /
quiescent / parity paths; both drive the same kernels through the same C
ABI, and the two averagers share one round protocol.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N
from .records import AveragerStamp, UpdateRecord
from .step import add_graph_kernels


class NativeLoops:
    """Mixin of ``async_engine._Engine``."""

    def native_loop(self) -> bool:
        """Whether updaters run the C++ loop (lpp_updater_run): the
        throughput configuration — async, device-stream sampling (drawn in
        the captured graph, or on the host for end-to-end host batches), no
        per-update records, no quiescent pauses."""
        cfg = self.cfg
        ok = (cfg.schedule == "async" and not cfg.quiescent and cfg.record_mode in ("off", "light")
              and cfg.use_graphs)
        if cfg.host_loop == "native" and not ok:
            raise ValueError("host_loop='native' needs schedule='async', record_mode 'off' or "
                             "'light', CUDA graphs, no quiescent pauses")
        return ok and cfg.host_loop != "python"

    def apply_on_side(self) -> bool:
        """Whether applies run on the per-updater high-priority stream.

        Auto (``apply_priority=None``): native loop and at most ~8 streams
        per worker.  The side stream doubles a worker's streams; past the
        device's 8 hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS) streams
        share queues and serialise — measured -12 % images/s at U = 6 and
        -13 % end to end at U = 4 (3 streams per updater with the copy
        stream), neutral at U = 4 device-resident; raising the queue count
        to 32 costs 2-3 % everywhere (tools/ab_priority_streams.py)."""
        p = self.cfg.apply_priority
        if p is None:
            # updater + apply (+ copy, end to end) streams per updater, + the averager's
            streams = self.cfg.updaters * (3 if self.host_batches else 2) + 1
            return self.native_loop() and streams <= 9
        return bool(p)

    def updater_cfg(self, w: _Worker, r: int) -> tuple:
        """The ``lpp_updater_cfg`` of updater r of worker w (+ the arrays it
        points into, which the caller keeps alive for the run)."""
        cfg = self.cfg
        sched = cfg.lr
        nb = cfg.partition.num_blocks
        prog = w.programs[r]
        lo = np.zeros(nb + 1, dtype=np.int64)
        hi = np.zeros(nb + 1, dtype=np.int64)
        execs = (ctypes.c_void_p * (2 * (nb + 1)))()       # [block][input buffer]
        flops = np.zeros(nb + 1, dtype=np.int64)
        gk = np.zeros(nb + 1, dtype=np.int64)
        for b in range(nb + 1):
            blk = cfg.partition.block(b)
            lo[b], hi[b] = blk.start, blk.stop
            flops[b] = self._flops_of[b]
            gk[b] = prog.graph_kernels.get((b, 0), 0)
            for buf in (0, 1):
                key = (b, buf % prog.nbuf)
                if key in prog.execs:
                    execs[2 * b + buf] = prog.execs[key]
        ms = np.ascontiguousarray(sched.milestones, dtype=np.int64)
        tracks = w.tags is not None
        k = w.tag_pick if tracks else 0
        c = N.UpdaterCfg()
        c.sample_counter = w.store.sample_counter._a
        c.update_order = w.store.update_order_counter._a
        c.stop = self.ctrl.stop._a
        c.last_avg_stamp = w.last_avg_stamp._a
        c.budget = self.budget
        c.lr_kind = 0 if sched.kind == "cosine" else 1
        c.n_milestones = len(ms)
        c.alpha0, c.peak, c.gamma = sched.alpha0, sched.peak, sched.gamma
        c.warmup, c.total = sched.warmup, sched.total
        c.milestones = ms.ctypes.data if len(ms) else None
        c.lpp = int(cfg.algo == "lpp_sgd")
        c.num_blocks, c.rank = nb, r + 1
        c.fused = int(self.fused())
        c.warm_start = cfg.warm_start_budget
        c.block_lo, c.block_hi = lo.ctypes.data, hi.ctypes.data
        c.graph_exec = ctypes.addressof(execs)
        c.flops_of = flops.ctypes.data
        c.graph_kernels_of = gk.ctypes.data
        c.x, c.g = w.store.arena.ptr, w.grads[r].ptr
        c.m = w.moms[r].ptr if w.moms[r] is not None else None
        c.replica = w.replicas[r].ptr
        c.tags = w.tag_arena.ptr if tracks else None
        c.n = self.dim
        c.mu, c.wd = cfg.momentum, cfg.weight_decay
        c.apply_mode = N.MODES[cfg.apply_mode]
        c.in_flight = cfg.in_flight
        c.tag_pick = k
        c.time_apply = int(self.time_apply)
        c.tag_seed = (cfg.seed * 1_000_003 + w.q * 1009 + r + 1) & (2**64 - 1)
        if tracks:
            # K5: sampled-index rings (pinned -> device), step records
            # (device -> pinned after each apply), round cell, block stamps
            c.tag_idx_dev = w.tag_idx_ring[r].data_ptr()
            c.tag_idx_pinned = w.tag_idx_pinned[r].data_ptr()
            c.rec_dev = w.rec_dev[r].data_ptr()
            c.rec_pinned = w.rec_pinned[r].data_ptr()
            c.rec_cols = w.rec_cols
            c.avg_cell_dev = w.avg_dev
            c.block_stamps = w.block_stamps.data_ptr()
            c.block_bounds_dev = w.block_bounds.data_ptr()
        c.classified = self.classified_count._a
        c.clean = self.clean_count._a
        c.apply_bytes_per_elem = float(self.apply_bytes_per_elem)
        if self.time_apply:
            # per-launch apply times (distribution beside the bench's average)
            alog = np.zeros(self.budget + 2, dtype=np.float32)
            c.apply_ms_log, c.apply_ms_cap = alog.ctypes.data, len(alog)
            self._apply_logs[(w.q, r)] = alog
        c.stream = w.streams[r].cuda_stream
        c.apply_stream = w.apply_streams[r].cuda_stream if self.side_apply else None
        keep = [lo, hi, execs, flops, ms, gk]
        if cfg.sampling == "host":
            # the reference's numpy stream (engine.py:293-296), restated natively
            c.host_rng = 1
            c.n_entropy = 3
            c.rng_entropy[0], c.rng_entropy[1], c.rng_entropy[2] = cfg.seed, w.q, r + 1
            c.batch = cfg.batch_size
            c.n_rows = cfg.objective.n_samples
            c.epoch_seed = (cfg.seed * 1000 + w.q * 10 + r + 1) if cfg.epoch_partition else -1
            if cfg.epoch_partition:
                c.epoch_base, c.epoch_stride, c.epoch_len = w.epoch_shard(self)
            if not self.host_batches:
                c.idx_pinned = w.idx_pinned[r].data_ptr()
                c.idx_dev = prog.idx.data_ptr()
        else:
            c.epoch_seed = -1
        if self.host_batches:
            obj = cfg.objective
            feats, labs = obj.features, obj.labels
            c.host_feats, c.host_labels = feats.data_ptr(), labs.data_ptr()
            c.n_rows = feats.shape[0]
            c.row_bytes = feats[0].numel() * feats.element_size()
            c.label_bytes = labs.element_size()
            c.batch = cfg.batch_size
            c.sample_key = prog.sample_key & (2**64 - 1)
            c.sample_step0 = prog.host_step
            if prog.epoch is not None:
                c.epoch_base, c.epoch_stride, c.epoch_len = prog.epoch
            c.feat_pinned = w.batch_pinned[r].data_ptr()
            c.label_pinned = w.label_pinned[r].data_ptr()
            c.xbuf[0], c.xbuf[1] = prog.xbs[0].data_ptr(), prog.xbs[1 % prog.nbuf].data_ptr()
            c.ybuf[0], c.ybuf[1] = prog.ybs[0].data_ptr(), prog.ybs[1 % prog.nbuf].data_ptr()
            c.copy_stream = w.copy_streams[r].cuda_stream
        if cfg.record_mode == "light":
            rcap = self.budget + 2           # an updater processes at most budget + 1 slots
            rec = np.zeros((rcap, 6), dtype=np.int64)
            rlr = np.zeros(rcap, dtype=np.float64)
            kk = max(k, 1)
            rti = np.zeros((rcap, kk), dtype=np.int64)
            rtg = np.zeros((rcap, kk), dtype=np.int32)
            rcount = np.zeros(1, dtype=np.int64)
            c.rec_i64, c.rec_lr = rec.ctypes.data, rlr.ctypes.data
            c.rec_tag_idx = rti.ctypes.data if k else None
            c.rec_tags = rtg.ctypes.data if k else None
            c.rec_cap, c.rec_count = rcap, rcount.ctypes.data
            self._records[(w.q, r)] = (rec, rlr, rti, rtg, rcount, k)
        if self.read_loss:
            cap = self.budget + cfg.updaters + 8
            log = np.zeros(cap, dtype=np.float32)
            count = np.zeros(1, dtype=np.int64)
            c.read_loss = 1
            c.loss_dev[0] = prog.loss_of(0).data_ptr()
            c.loss_dev[1] = prog.loss_of(1).data_ptr()
            c.loss_pinned = w.loss_pinned[r].data_ptr()
            c.loss_log, c.loss_cap, c.loss_count = log.ctypes.data, cap, count.ctypes.data
            keep += [log, count]
        return c, keep

    def updater_native(self, q: int, r: int) -> None:
        """a10 in native code: the whole loop is one GIL-free C call."""
        w = self.workers[q]
        torch.cuda.set_device(w.device)
        if self.nvtx:
            torch.cuda.nvtx.range_push(self.nvtx)
        try:
            c, keep = self.updater_cfg(w, r)
            st = N.updater_run(c)
            w.programs[r].host_step += int(st.steps)
            if (q, r) in self._records:
                self._collect_records(q, r)
            if self.read_loss:
                log, count = keep[-2], int(keep[-1][0])
                with self.native_lock:
                    self.loss_log.extend(float(v) for v in log[:min(count, len(log))])
            del keep
            self.flops.add(int(st.flops))
            add_graph_kernels(int(st.graph_kernels))
            if self.time_apply:
                alog = self._apply_logs.pop((q, r), None)
                with self.native_lock:
                    if alog is not None:
                        self.apply_ms_samples.extend(alog[:int(st.apply_launches)].tolist())
                    self.native_apply[0] += int(st.apply_launches)
                    self.native_apply[1] += float(st.apply_ms)
                    self.native_apply[2] += float(st.apply_bytes)
        except BaseException as exc:  # surfaced after join (engine.py:456-463)
            self.fail(exc)
        finally:
            if self.nvtx:
                torch.cuda.nvtx.range_pop()
            if w.exited.add(1) + 1 == self.cfg.updaters:
                self.ctrl.drained.add(1)

    def native_averager(self) -> bool:
        """Whether averagers run the C++ round loop (lpp_averager_run): p2p
        averaging without quiescent pauses or full records."""
        cfg = self.cfg
        return (cfg.host_loop != "python" and cfg.schedule == "async" and not cfg.quiescent
                and not self.nvls and cfg.record_mode != "full")

    def averager_native(self, q: int) -> None:
        """a11 in native code: the round protocol + K4 in one GIL-free call."""
        cfg = self.cfg
        w = self.workers[q]
        torch.cuda.set_device(w.device)
        ctrl = self.ctrl
        Q = cfg.workers
        if self.nvtx:
            torch.cuda.nvtx.range_push(self.nvtx)
        try:
            arenas = (ctypes.c_void_p * Q)(*self.arena_ptrs)
            tags = (ctypes.c_void_p * Q)(*self.tag_ptrs) if self.tag_ptrs is not None else None
            # per-round records: at most one round per slot claimed (+ drain)
            cap = Q * (self.budget + cfg.updaters) + 8
            if cfg.round_budget is not None:
                cap = min(cap, cfg.round_budget + 8)
            cap = min(cap, 1 << 20)
            rec = np.zeros((cap, 5), dtype=np.int64)
            wall = np.zeros(cap, dtype=np.float64)
            lo, hi = self.shards[q]
            c = N.AveragerCfg()
            c.ctrl = ctrl.buf.ctypes.data
            c.max_rounds = 0
            c.workers, c.q, c.updaters = Q, q, cfg.updaters
            c.tagged = int(self.tag_ptrs is not None)
            c.stamp_floor = int(cfg.tracks)
            c.round_cell = w.avg_dev if w.round_cell is not None else None
            c.sample_counter = w.store.sample_counter._a
            c.update_order = w.store.update_order_counter._a
            c.exited = w.exited._a
            c.last_avg_stamp = w.last_avg_stamp._a
            c.synced_at = w.synced_at._a
            c.switch_point, c.period = cfg.sync.switch_point, cfg.sync.period
            c.stop_after = cfg.round_budget or 0
            c.arenas = ctypes.addressof(arenas)
            c.tags = ctypes.addressof(tags) if tags is not None else None
            c.lo, c.hi, c.n = lo, hi, self.dim
            c.mean_out = w.mean_out.data_ptr()
            c.stream = w.avg_stream.cuda_stream
            c.t0 = self.t0
            c.rec, c.rec_wall_ms, c.max_records = rec.ctypes.data, wall.ctypes.data, cap
            keep = []
            if cfg.eval_interval > 0:
                # eval points (engine.py:445-451): worker 0 keeps round means
                ecap = (self.budget // cfg.eval_interval + 2) if q == 0 else 0
                ebuf = torch.empty((max(ecap, 1), self.dim), dtype=torch.float32, device=w.dev)
                erec = np.zeros((max(ecap, 1), 5), dtype=np.int64)
                ewall = np.zeros(max(ecap, 1), dtype=np.float64)
                ecount = np.zeros(1, dtype=np.int64)
                bounds = np.array([lo_ for lo_, _ in self.shards] + [self.shards[-1][1]], dtype=np.int64)
                parts = None
                if self.group is None:
                    parts = (ctypes.c_void_p * Q)(*[self.workers[o].mean_out.data_ptr() for o in range(Q)])
                c.eval_interval = cfg.eval_interval
                c.mean_parts = ctypes.addressof(parts) if parts is not None else None
                c.shard_bounds = bounds.ctypes.data
                c.eval_buf, c.eval_cap = ebuf.data_ptr(), ecap
                c.eval_rec, c.eval_wall_ms, c.eval_count = erec.ctypes.data, ewall.ctypes.data, ecount.ctypes.data
                c.flops_cell = self.flops._a
                c.classified_cell, c.clean_cell = self.classified_count._a, self.clean_count._a
                keep = [ebuf, erec, ewall, ecount, bounds, parts]
            k4_ms = np.zeros(1, dtype=np.float64)
            k4_n = np.zeros(1, dtype=np.int64)
            if self.time_apply:
                c.time_rounds, c.k4_ms, c.k4_rounds = 1, k4_ms.ctypes.data, k4_n.ctypes.data
            n = N.averager_run(c)
            if self.time_apply:
                with self.native_lock:
                    self.k4_timing[0] += int(k4_n[0])
                    self.k4_timing[1] += float(k4_ms[0])
            if keep:
                ebuf, erec, ewall, ecount = keep[:4]
                for i in range(int(ecount[0])):
                    s_cur, r_, fl, classified, clean = (int(v) for v in erec[i])
                    ph = clean / classified if classified else 1.0
                    self.eval_points.append((s_cur, r_, float(ewall[i]), fl, ph, ebuf[i].clone()))
            for i in range(min(n, cap)):
                r, u, s_cur, k_delta, _ = (int(v) for v in rec[i])
                self.stamps[q].append(AveragerStamp(worker=q, round=r, u=u, s_cur=s_cur,
                                                    k_delta=k_delta, wall_ms=float(wall[i])))
        except BaseException as exc:  # surfaced after join (engine.py:456-463)
            self.fail(exc)
        finally:
            if self.nvtx:
                torch.cuda.nvtx.range_pop()

    _REASONS = ("warm_start", "alternate_full", "alternate_partial")

    def _collect_records(self, q: int, r: int) -> None:
        """UpdateRecords of one native updater run (record_mode "light")."""
        rec, rlr, rti, rtg, rcount, k = self._records.pop((q, r))
        out = self.updates[q * self.cfg.updaters + r]
        for i in range(int(rcount[0])):
            s_, u, k_claim, b, reason, clean = (int(v) for v in rec[i])
            out.append(UpdateRecord(
                worker=q, rank=r + 1, s=s_, u=u, k_claim=k_claim, block_id=b,
                reason=self._REASONS[reason], lr=float(rlr[i]), flops=self._flops_of[b],
                backward_flops=self._bflops_of[b], clean=None if clean < 0 else bool(clean),
                tag_indices=rti[i, :k].copy() if k else None,
                tags=rtg[i, :k].astype(np.int64) if k else None))
