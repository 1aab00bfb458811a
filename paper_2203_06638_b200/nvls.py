"""NVLS (in-NVSwitch) averaging state: SURVEY §8f rank 1.

Two multicast objects span the group's GPUs: ``stage`` (each worker's round
snapshot) and ``mean`` (the broadcast round mean).  Every worker owns one
VMM buffer bound into each object (its "unicast" copy) and maps the objects'
multicast address.  A round (engine.py:418-421, snapshot -> mean all-reduce
-> add_assign(mean - snapshot)) is then:

    stage_q = x_q                              local copy (K3)
    -- all staged --
    owner o: mean[shard o] = ld_reduce(stage)/Q  in the switch, multimem.st to all
    -- all means broadcast --
    x_q += mean_q - stage_q                    local, element-atomic (updaters keep writing)

One process per GPU: rank 0 creates the objects and hands their POSIX file
descriptors to the peers over an abstract-namespace Unix socket
(SCM_RIGHTS); every rank adds its device, then (after a barrier) binds its
buffers and maps the multicast VA.  In one process only a single-device
group is supported (used by the functional test); multi-device NVLS runs as
one process per GPU.
"""

from __future__ import annotations

import ctypes
import os
import socket
import uuid

import torch

from . import _native as N


def _ck(rc, what):
    N.check(rc, what)


class _Vmm:
    def __init__(self, device: int, nbytes: int):
        h = ctypes.c_void_p()
        _ck(N.lib.lpp_vmm_create(int(device), int(nbytes), ctypes.byref(h)), "vmm_create")
        self.h = h
        self.ptr = int(N.lib.lpp_vmm_ptr(h))
        self.size = int(N.lib.lpp_vmm_size(h))

    def close(self):
        if self.h is not None:
            _ck(N.lib.lpp_vmm_destroy(self.h), "vmm_destroy")
            self.h = None


class _Mc:
    def __init__(self, h: ctypes.c_void_p):
        self.h = h
        self.ptr = 0

    @classmethod
    def create(cls, q: int, nbytes: int) -> "_Mc":
        h = ctypes.c_void_p()
        _ck(N.lib.lpp_mc_create(int(q), int(nbytes), ctypes.byref(h)), "mc_create")
        return cls(h)

    @classmethod
    def import_fd(cls, fd: int, nbytes: int) -> "_Mc":
        h = ctypes.c_void_p()
        _ck(N.lib.lpp_mc_import_fd(int(fd), int(nbytes), ctypes.byref(h)), "mc_import_fd")
        return cls(h)

    def export_fd(self) -> int:
        fd = ctypes.c_int(-1)
        _ck(N.lib.lpp_mc_export_fd(self.h, ctypes.byref(fd)), "mc_export_fd")
        return fd.value

    def add_device(self, device: int):
        _ck(N.lib.lpp_mc_add_device(self.h, int(device)), "mc_add_device")

    def bind(self, mem: _Vmm):
        _ck(N.lib.lpp_mc_bind(self.h, mem.h, 0), "mc_bind")

    def map(self, device: int) -> int:
        p = ctypes.c_void_p()
        _ck(N.lib.lpp_mc_map(self.h, int(device), ctypes.byref(p)), "mc_map")
        self.ptr = int(p.value)
        return self.ptr

    def close(self):
        if self.h is not None:
            _ck(N.lib.lpp_mc_destroy(self.h), "mc_destroy")
            self.h = None


def share_fds(group, fds: list[int] | None, count: int | None = None) -> list[int]:
    """Hand rank 0's file descriptors to every other rank of the group.

    Rank 0 passes ``fds`` (it keeps its own copies and gets them back); the
    others pass None and ``count``, and receive duplicates of the same open
    files over an abstract-namespace Unix socket (SCM_RIGHTS) whose name
    travels over ``torch.distributed``.  Used for the multicast-object
    handles, which are POSIX file descriptors."""
    import torch.distributed as dist

    name = [None]
    srv = None
    if group.rank == 0:
        name[0] = f"lpp-fds-{uuid.uuid4().hex}"
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind("\0" + name[0])
        srv.listen(max(group.world - 1, 1))
    dist.broadcast_object_list(name, src=0)
    if group.rank == 0:
        for _ in range(group.world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"fds"], fds)
            conn.close()
        srv.close()
        return list(fds)
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.connect("\0" + name[0])
    _, got, _, _ = socket.recv_fds(cli, 16, count)
    cli.close()
    if len(got) != count:
        raise RuntimeError(f"expected {count} file descriptors, received {len(got)}")
    return list(got)


def supported(device: int, workers: int = 1) -> bool:
    """Multicast attribute AND a multicast object can actually be created
    (containers that expose one GPU without fabric-manager access report the
    attribute but refuse cuMulticastCreate)."""
    return probe(device, workers)[0]


def probe(device: int, workers: int = 1) -> tuple[bool, str]:
    out = ctypes.c_int(0)
    try:
        _ck(N.lib.lpp_mc_supported(int(device), ctypes.byref(out)), "mc_supported")
    except Exception as exc:  # no driver
        return False, str(exc)
    if not out.value:
        return False, "CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0"
    gran = ctypes.c_size_t(0)
    try:
        _ck(N.lib.lpp_mc_granularity(int(device), int(workers), ctypes.byref(gran)), "mc_granularity")
        _Mc.create(workers, int(gran.value)).close()
    except Exception as exc:
        return False, str(exc)
    return True, "ok"


class NvlsGroup:
    """The staging / mean buffers of this process's worker and their multicast VAs."""

    def __init__(self, dim: int, workers: int, device: int, group=None):
        ok, why = probe(device, workers)
        if not ok:
            raise RuntimeError(f"NVLS averaging needs NVSwitch multicast, unavailable here: {why}")
        self.dim = int(dim)
        self.workers = int(workers)
        self.device = int(device)
        gran = ctypes.c_size_t(0)
        _ck(N.lib.lpp_mc_granularity(self.device, self.workers, ctypes.byref(gran)), "mc_granularity")
        g = int(gran.value)
        self.nbytes = ((4 * max(self.dim, 1) + g - 1) // g) * g
        if group is None:
            if workers != 1:
                raise NotImplementedError(
                    "in one process NVLS averaging spans a single device; run one process per GPU")
            self.mc_stage, self.mc_mean = _Mc.create(1, self.nbytes), _Mc.create(1, self.nbytes)
            for mc in (self.mc_stage, self.mc_mean):
                mc.add_device(self.device)
        else:
            self._exchange(group)
        self.stage, self.mean = _Vmm(self.device, self.nbytes), _Vmm(self.device, self.nbytes)
        self.mc_stage.bind(self.stage)
        self.mc_mean.bind(self.mean)
        if group is not None:
            group.barrier()
        self.mc_stage.map(self.device)
        self.mc_mean.map(self.device)
        self.mean_tensor = _view(self.mean.ptr, self.dim, self.device)

    def _exchange(self, group) -> None:
        if group.rank == 0:
            self.mc_stage = _Mc.create(self.workers, self.nbytes)
            self.mc_mean = _Mc.create(self.workers, self.nbytes)
            fds = share_fds(group, [self.mc_stage.export_fd(), self.mc_mean.export_fd()])
        else:
            fds = share_fds(group, None, count=2)
            self.mc_stage = _Mc.import_fd(fds[0], self.nbytes)
            self.mc_mean = _Mc.import_fd(fds[1], self.nbytes)
        for fd in fds:
            os.close(fd)
        for mc in (self.mc_stage, self.mc_mean):
            mc.add_device(self.device)
        group.barrier()   # every device added before anyone binds

    # -- the round's three device phases --------------------------------------

    def stage_copy(self, arena_ptr: int, stream: int) -> None:
        N.snapshot(arena_ptr, self.stage.ptr, self.dim, stream)

    def reduce_mean(self, lo: int, hi: int, stream: int) -> None:
        _ck(N.lib.lpp_nvls_mean_shard(self.mc_stage.ptr, self.mc_mean.ptr, lo, hi, self.workers,
                                      stream), "nvls_mean_shard")

    def apply(self, arena_ptr: int, tags_ptr: int | None, stamp: int, stream: int) -> None:
        _ck(N.lib.lpp_nvls_apply(arena_ptr, self.stage.ptr, self.mean.ptr, self.dim, tags_ptr,
                                 int(stamp), stream), "nvls_apply")

    def close(self) -> None:
        for mc in (getattr(self, "mc_stage", None), getattr(self, "mc_mean", None)):
            if mc is not None:
                mc.close()
        for v in (getattr(self, "stage", None), getattr(self, "mean", None)):
            if v is not None:
                v.close()


def _view(ptr: int, n: int, device: int) -> torch.Tensor:
    from .arena import _CAI

    with torch.cuda.device(device):
        t = torch.as_tensor(_CAI(ptr, max(n, 1)), device=f"cuda:{device}")
    return t[:n]
