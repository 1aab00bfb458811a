"""Flat fp32 device arenas owned by the C ABI, viewed as torch tensors.

An arena is the B200 replacement of ``ParamStore.values``
(``paramstore.py:68-70``): one C-contiguous 1-D parameter vector.  It is
allocated by ``lpp_arena_create`` (plain ``cudaMalloc``, so it can be
exported over CUDA IPC to the peer processes of a multi-GPU group) and
exposed to PyTorch zero-copy through ``__cuda_array_interface__``, so that
model parameters and gradients can be views into it.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N


class _CAI:
    """Minimal ``__cuda_array_interface__`` carrier for torch.as_tensor."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {
            "shape": (n,),
            "typestr": "<f4",
            "data": (ptr, False),
            "version": 3,
            "strides": None,
            "stream": None,
        }


class Arena:
    """Owned fp32[n] device buffer; ``.tensor`` is a torch view of it."""

    def __init__(self, n: int, device: int):
        if n < 0:
            raise ValueError("arena size must be non-negative")
        handle = ctypes.c_void_p()
        N.check(N.lib.lpp_arena_create(int(device), int(n), ctypes.byref(handle)), "arena_create")
        self._h = handle
        self.n = int(n)
        self.device = int(device)
        self.ptr = int(N.lib.lpp_arena_data(handle))
        with torch.cuda.device(self.device):
            t = torch.as_tensor(_CAI(self.ptr, max(self.n, 1)), device=f"cuda:{self.device}")
        self.tensor = t[: self.n]

    def export_ipc(self) -> bytes:
        buf = (ctypes.c_char * N.IPC_HANDLE_BYTES)()
        N.check(N.lib.lpp_arena_export_ipc(self._h, buf), "arena_export_ipc")
        return bytes(buf)

    def close(self) -> None:
        if self._h is not None and self._h.value:
            # drop torch views first; the caller must not use .tensor afterwards
            self.tensor = None
            N.check(N.lib.lpp_arena_destroy(self._h), "arena_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PeerMapping:
    """A peer arena opened from a CUDA IPC handle (one process per GPU)."""

    def __init__(self, device: int, handle: bytes, n: int):
        if len(handle) != N.IPC_HANDLE_BYTES:
            raise ValueError("bad IPC handle length")
        out = ctypes.c_void_p()
        hb = (ctypes.c_char * N.IPC_HANDLE_BYTES).from_buffer_copy(handle)
        N.check(N.lib.lpp_ipc_open(int(device), hb, ctypes.byref(out)), "ipc_open")
        self.device = int(device)
        self.ptr = int(out.value)
        self.n = int(n)

    def close(self) -> None:
        if self.ptr:
            N.check(N.lib.lpp_ipc_close(self.device, self.ptr), "ipc_close")
            self.ptr = 0


def enable_peer_access(device: int, peer: int) -> bool:
    ok = ctypes.c_int(0)
    N.check(N.lib.lpp_can_access_peer(int(device), int(peer), ctypes.byref(ok)), "can_access_peer")
    if not ok.value:
        return False
    N.check(N.lib.lpp_enable_peer_access(int(device), int(peer)), "enable_peer_access")
    return True


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
