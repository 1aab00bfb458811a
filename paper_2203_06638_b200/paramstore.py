"""Arena-backed shared parameter store with the reference ``ParamStore`` API.

Drop-in for ``asyncsgd.paramstore`` (``/root/reference/pkg/src/asyncsgd/paramstore.py``):

* ``AtomicCounter`` (``paramstore.py:19-39``): a host int64 cell updated
  with the C ABI's acquire/release/acq_rel atomics (K6); the cell can live
  in a numpy array or in a POSIX shared-memory control block (multi-process
  groups).
* ``ParamStore`` (``paramstore.py:59-136``): ``values`` is an fp32 device
  arena (``Arena``) instead of an fp64 numpy vector; ``snapshot`` is K3,
  ``sub_assign``/``add_assign`` are K1 (``lpp_accum``) — element-atomic
  device reductions, so concurrent updates from many CUDA streams are never
  lost (``_atomics.c:58-74``).  Device ops are asynchronous on the current
  torch stream (or the ``stream=`` given); ``read``/``write`` synchronise.

``track_writes=True`` keeps int32 write tags (K5): ``sub_assign`` /
``add_assign`` stamp every written element after its value
(``accum_cas_tagged_f64``), and ``snapshot`` returns tags read before the
values — sampled at ``tag_indices`` or for the whole vector
(``paramstore.py:97-117``).  Tags are device tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .arena import Arena, stream_ptr


class AtomicCounter:
    """A shared int64 with atomic fetch-and-add (``paramstore.py:19-39``)."""

    __slots__ = ("_cell", "_i", "_a")

    def __init__(self, initial: int = 0, cell: np.ndarray | None = None, index: int = 0):
        if cell is None:
            cell = np.array([initial], dtype=np.int64)
            index = 0
        else:
            N.atomic_store(cell, index, initial)
        self._cell = cell                  # keeps the cell's buffer alive
        self._i = index
        self._a = N.cell_address(cell, index)

    def read_and_inc(self) -> int:
        return N.lib.lpp_atomic_fetch_add_i64(self._a, 1)

    def read(self) -> int:
        return N.lib.lpp_atomic_load_i64(self._a)

    def add(self, delta: int) -> int:
        return N.lib.lpp_atomic_fetch_add_i64(self._a, delta)

    def store(self, value: int) -> None:
        N.lib.lpp_atomic_store_i64(self._a, value)

    def cas(self, expected: int, desired: int) -> bool:
        return bool(N.lib.lpp_atomic_cas_i64(self._a, expected, desired))

    def wait_ge(self, target: int, abort: "AtomicCounter | None" = None) -> int | None:
        """Block without the GIL until the value is >= target (None: aborted)."""
        if abort is None:
            return N.atomic_wait_ge(self._cell, self._i, target)
        return N.atomic_wait_ge(self._cell, self._i, target, abort._cell, abort._i)


@dataclass(frozen=True)
class Snapshot:
    """Per-element copy of a store (``paramstore.py:42-56``); values on device."""

    values: torch.Tensor
    order: int
    tags: np.ndarray | None = None
    tag_indices: np.ndarray | None = None


def _as_device_f32(delta, device: int) -> torch.Tensor:
    t = torch.as_tensor(delta)
    if t.dim() != 1:
        t = t.reshape(-1)
    return t.to(device=f"cuda:{device}", dtype=torch.float32).contiguous()


class ParamStore:
    """One worker's shared arena plus its two shared counters."""

    def __init__(self, initial, track_writes: bool = False, device: int | None = None,
                 mode: str = "red"):
        arr = torch.as_tensor(np.asarray(initial) if not torch.is_tensor(initial) else initial)
        if arr.dim() != 1:
            raise ValueError("parameter vector must be one-dimensional")
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.dim = int(arr.shape[0])
        self.arena = Arena(self.dim, self.device)
        if self.dim:
            self.arena.tensor.copy_(arr.to(torch.float32))
        self.mode = N.MODES[mode]
        self.sample_counter = AtomicCounter(0)
        self.update_order_counter = AtomicCounter(0)
        self.tag_arena = Arena(self.dim, self.device) if track_writes else None
        self.tags = self.tag_arena.tensor.view(torch.int32) if track_writes else None

    @property
    def values(self) -> torch.Tensor:
        return self.arena.tensor

    # -- element access ---------------------------------------------------

    def read(self, index: int, stream: torch.cuda.Stream | None = None) -> float:
        """One element, acquire-loaded (``_atomics.load_f64``, _atomics.c:41-48)."""
        if not 0 <= index < self.dim:
            raise IndexError(f"index {index} out of range [0, {self.dim})")
        with torch.cuda.device(self.device):
            return N.load_f32(self.arena.ptr, self.dim, int(index), stream_ptr(stream))

    def write(self, index: int, value: float, stream: torch.cuda.Stream | None = None) -> None:
        """One element, release-stored (``_atomics.store_f64``, _atomics.c:50-56)."""
        if not 0 <= index < self.dim:
            raise IndexError(f"index {index} out of range [0, {self.dim})")
        with torch.cuda.device(self.device):
            N.store_f32(self.arena.ptr, self.dim, int(index), float(value), stream_ptr(stream))

    # -- counters -----------------------------------------------------------

    def read_and_inc(self) -> int:
        return self.sample_counter.read_and_inc()

    def claim_update_order(self) -> int:
        return self.update_order_counter.read_and_inc() + 1

    # -- snapshots (K3) -----------------------------------------------------

    def snapshot(self, tag_indices=None, out: torch.Tensor | None = None,
                 stream: torch.cuda.Stream | None = None) -> Snapshot:
        order = self.sample_counter.read()
        if out is None:
            out = torch.empty(self.dim, dtype=torch.float32, device=f"cuda:{self.device}")
        elif out.numel() != self.dim or out.dtype != torch.float32 or not out.is_contiguous():
            raise ValueError("snapshot out must be a contiguous fp32 vector of the store's length")
        sp = stream_ptr(stream)
        if self.tags is None:
            if self.dim:
                N.snapshot(self.arena.ptr, out.data_ptr(), self.dim, sp)
            return Snapshot(out, order)
        dev = f"cuda:{self.device}"
        if tag_indices is not None:
            idx_np = np.asarray(tag_indices, dtype=np.int64)
            if idx_np.size and (idx_np.min() < 0 or idx_np.max() >= self.dim):
                raise IndexError("tag index out of range")
            idx = torch.as_tensor(idx_np, device=dev)
            out_tags = torch.empty(idx.numel(), dtype=torch.int32, device=dev)
            # tags gathered before the value copy (paramstore.py:108-112)
            N.gather_tags(self.tag_arena.ptr, idx.data_ptr(), idx.numel(), out_tags.data_ptr(), sp)
            if self.dim:
                N.snapshot(self.arena.ptr, out.data_ptr(), self.dim, sp)
            if stream is not None:
                idx.record_stream(stream)
            return Snapshot(out, order, out_tags, idx_np)
        out_tags = torch.empty(self.dim, dtype=torch.int32, device=dev)
        if self.dim:
            N.snapshot_tagged(self.arena.ptr, self.tag_arena.ptr, out.data_ptr(), out_tags.data_ptr(),
                              self.dim, None, sp)
        return Snapshot(out, order, out_tags)

    # -- range updates (K1) -------------------------------------------------

    def sub_assign(self, start: int, delta, stamp: int = 0,
                   stream: torch.cuda.Stream | None = None) -> None:
        self._accum(start, delta, -1.0, stamp, stream)

    def add_assign(self, start: int, delta, stamp: int = 0,
                   stream: torch.cuda.Stream | None = None) -> None:
        self._accum(start, delta, 1.0, stamp, stream)

    def _accum(self, start: int, delta, scale: float, stamp: int, stream) -> None:
        d = _as_device_f32(delta, self.device)
        n = d.numel()
        if stream is not None:
            # `d` was produced (uploaded / converted) on the current stream:
            # the kernel on `stream` must not read it before that finished
            stream.wait_stream(torch.cuda.current_stream(self.device))
        if start < 0 or start + n > self.dim:
            raise IndexError("update range out of bounds")
        mode = self.mode if self.mode != N.MODE_BULK else N.MODE_RED
        if self.tags is None:
            N.accum(self.arena.ptr, self.dim, int(start), d.data_ptr(), n, scale, mode,
                    stream_ptr(stream))
        else:
            N.accum_tagged(self.arena.ptr, self.tag_arena.ptr, self.dim, int(start), d.data_ptr(),
                           n, scale, int(stamp), mode, stream_ptr(stream))
        if stream is not None:
            # `d` may be a temporary of the current stream: keep its block
            # reserved until the kernel on `stream` has consumed it
            d.record_stream(stream)
