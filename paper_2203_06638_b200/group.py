"""One-process-per-GPU worker groups.

Each rank is worker q = rank: it owns its arena (``lpp_arena_create``,
plain cudaMalloc) and exports it with a CUDA IPC handle; every rank maps
all peers' arenas (``lpp_ipc_open``; P2P over NVLink / NVSwitch) so that
its averager can run the owner-computes K4 over its shard against all Q
arenas with plain loads and ``red.add`` — no NCCL on the averaging path.

Plumbing uses ``torch.distributed`` (any backend; NCCL on the box, gloo in
the CPU tests): the control block name and the IPC handles are exchanged
with object collectives, and the round-control cells live in POSIX shared
memory on the node (host atomics, K6).  NCCL collectives are used only by
the synchronous baselines (``allreduce_mean``: B1 MB-SGD gradients, B2
L-SGD parameters) and to gather the final mean once at the end.
"""

from __future__ import annotations

from multiprocessing import shared_memory

import numpy as np
import torch
import torch.distributed as dist

from .rounds import RoundControl


class ProcessGroup:
    def __init__(self, workers: int | None = None, max_rounds: int = 1 << 16,
                 map_arenas: bool = True):
        if not dist.is_initialized():
            raise RuntimeError("ProcessGroup needs torch.distributed to be initialised")
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        if workers is not None and workers != self.world:
            raise ValueError(f"group of {workers} workers needs world_size {workers}, got {self.world}")
        self.workers = self.world
        self.max_rounds = int(max_rounds)
        nbytes = RoundControl.nbytes(self.max_rounds)
        name = [None]
        if self.rank == 0:
            self._shm = shared_memory.SharedMemory(create=True, size=nbytes)
            name[0] = self._shm.name
        dist.broadcast_object_list(name, src=0)
        if self.rank != 0:
            self._shm = shared_memory.SharedMemory(name=name[0])
            # only the creator (rank 0) owns the segment's lifetime; attached
            # ranks must not let their resource tracker unlink it at exit
            try:
                from multiprocessing import resource_tracker

                resource_tracker.unregister(self._shm._name, "shared_memory")
            except Exception:
                pass
        self._buf = np.ndarray((RoundControl.cells(self.max_rounds),), dtype=np.int64,
                               buffer=self._shm.buf)
        if self.rank == 0:
            self._buf[:] = 0
        dist.barrier()
        self.control = RoundControl(self.workers, self.max_rounds, self._buf)
        self.peers = []
        self.map_arenas = map_arenas

    # -- arenas ------------------------------------------------------------

    def attach_arenas(self, arena) -> list[int]:
        """Exchange IPC handles; return the Q arena pointers as seen from here."""
        from .arena import PeerMapping

        handle = arena.export_ipc()
        handles = [None] * self.world
        dist.all_gather_object(handles, (handle, arena.n))
        ptrs = []
        for q, (h, n) in enumerate(handles):
            if n != arena.n:
                raise ValueError("all workers must hold arenas of the same size")
            if q == self.rank:
                ptrs.append(arena.ptr)
            else:
                pm = PeerMapping(arena.device, h, n)
                self.peers.append(pm)
                ptrs.append(pm.ptr)
        dist.barrier()
        return ptrs

    # -- control -------------------------------------------------------------

    def reset_control(self) -> None:
        dist.barrier()
        if self.rank == 0:
            self._buf[:] = 0
        dist.barrier()

    def barrier(self) -> None:
        dist.barrier()

    # -- baselines / gathers (NCCL) --------------------------------------------

    def allreduce_mean(self, t: torch.Tensor) -> None:
        if dist.get_backend() == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.AVG)
            return
        # gloo (tests): no AVG, stage through the host
        h = t.detach().cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM)
        t.copy_(h / self.world)

    def gather_mean(self, mean_out: torch.Tensor, shards) -> np.ndarray:
        lo, hi = shards[self.rank]
        width = max(h - l for l, h in shards)
        dev = mean_out.device if dist.get_backend() == "nccl" else torch.device("cpu")
        mean_out = mean_out.to(dev)
        mine = torch.zeros(width, dtype=torch.float32, device=dev)
        mine[: hi - lo] = mean_out[lo:hi]
        out = torch.empty(width * self.world, dtype=torch.float32, device=dev)
        dist.all_gather_into_tensor(out, mine)
        host = out.cpu().numpy()
        dim = shards[-1][1]
        res = np.empty(dim, dtype=np.float32)
        for q, (l, h) in enumerate(shards):
            res[l:h] = host[q * width: q * width + (h - l)]
        return res

    def close(self) -> None:
        try:
            dist.barrier()
        except Exception:
            pass
        for pm in self.peers:
            try:
                pm.close()
            except Exception:
                pass
        self.peers = []
        self.control = None
        self._buf = None
        try:
            self._shm.close()
            if self.rank == 0:
                self._shm.unlink()
        except Exception:
            pass
