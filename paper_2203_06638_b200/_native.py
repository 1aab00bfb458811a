"""ctypes binding of the C-ABI CUDA library ``lib/liblpp_b200.so``.

The library is the product: there is no CPU fallback.  Importing this
module fails loudly (ImportError) when the library has not been built, and
every call that returns a non-zero status raises, mirroring the reference's
exception contract for ``asyncsgd._atomics`` (``_atomics.c:26-36`` ValueError,
``:76-84,328-333`` IndexError).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = LIB_DIR / "liblpp_b200.so"

MODE_PLAIN = 0
MODE_RED = 1
MODE_BULK = 2
MODES = {"plain": MODE_PLAIN, "red": MODE_RED, "bulk": MODE_BULK}
MAX_WORKERS = 8
IPC_HANDLE_BYTES = 64

E_VALUE, E_INDEX, E_CUDA, E_NOMEM = -1, -2, -3, -4


class LppError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


def _load() -> ctypes.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA extension is required; there is no CPU fallback)"
        )
    return ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)


lib = _load()

_c = ctypes
_size = _c.c_size_t
_vp = _c.c_void_p
_i64p = _c.POINTER(_c.c_int64)

class UpdaterCfg(ctypes.Structure):
    """``lpp_updater_cfg`` (include/lpp_b200.h), field for field."""

    _fields_ = [
        ("sample_counter", _vp), ("update_order", _vp), ("stop", _vp), ("last_avg_stamp", _vp),
        ("budget", _c.c_int64),
        ("lr_kind", _c.c_int32), ("n_milestones", _c.c_int32),
        ("alpha0", _c.c_double), ("peak", _c.c_double), ("gamma", _c.c_double),
        ("warmup", _c.c_int64), ("total", _c.c_int64), ("milestones", _vp),
        ("lpp", _c.c_int32), ("num_blocks", _c.c_int32), ("rank", _c.c_int32),
        ("fused", _c.c_int32), ("warm_start", _c.c_int64),
        ("block_lo", _vp), ("block_hi", _vp), ("graph_exec", _vp), ("flops_of", _vp),
        ("x", _vp), ("g", _vp), ("m", _vp), ("replica", _vp), ("tags", _vp), ("n", _size),
        ("mu", _c.c_float), ("wd", _c.c_float), ("apply_mode", _c.c_int32),
        ("in_flight", _c.c_int32),
        ("tag_pick", _c.c_int32), ("time_apply", _c.c_int32), ("tag_seed", _c.c_uint64),
        ("tag_idx_pinned", _vp), ("tag_idx_dev", _vp), ("classified", _vp), ("clean", _vp),
        ("apply_bytes_per_elem", _c.c_double), ("stream", _vp), ("apply_stream", _vp),
        ("host_feats", _vp), ("host_labels", _vp), ("n_rows", _c.c_int64), ("row_bytes", _c.c_int64),
        ("label_bytes", _c.c_int64), ("batch", _c.c_int32), ("read_loss", _c.c_int32),
        ("sample_key", _c.c_uint64), ("feat_pinned", _vp), ("label_pinned", _vp),
        ("xbuf", _vp * 2), ("ybuf", _vp * 2), ("copy_stream", _vp), ("loss_dev", _vp * 2),
        ("loss_pinned", _vp), ("loss_log", _vp), ("loss_cap", _c.c_int64), ("loss_count", _vp),
        ("sample_step0", _c.c_int64), ("epoch_base", _c.c_int64), ("epoch_stride", _c.c_int64),
        ("epoch_len", _c.c_int64), ("rec_i64", _vp), ("rec_lr", _vp), ("rec_tag_idx", _vp),
        ("rec_tags", _vp), ("rec_cap", _c.c_int64), ("rec_count", _vp),
        ("host_rng", _c.c_int32), ("n_entropy", _c.c_int32), ("rng_entropy", _c.c_uint64 * 4),
        ("epoch_seed", _c.c_int64), ("idx_pinned", _vp), ("idx_dev", _vp),
        ("rec_dev", _vp), ("rec_pinned", _vp), ("rec_cols", _c.c_int32), ("avg_cell_dev", _vp),
        ("block_stamps", _vp), ("block_bounds_dev", _vp), ("apply_ms_log", _vp),
        ("apply_ms_cap", _c.c_int64), ("graph_kernels_of", _vp),
    ]


class TagPlan(ctypes.Structure):
    """``lpp_tag_plan`` (include/lpp_b200.h)."""

    _fields_ = [("next_idx", _vp), ("next_dev", _vp), ("next_host", _vp), ("cur_dev", _vp),
                ("cur_claim", _vp), ("avg_cell", _vp), ("block_stamps", _vp),
                ("block_bounds", _vp), ("num_blocks", _c.c_int32), ("block_id", _c.c_int32),
                ("k", _c.c_int32)]


class AveragerCfg(ctypes.Structure):
    """``lpp_averager_cfg`` (include/lpp_b200.h), field for field."""

    _fields_ = [
        ("ctrl", _vp), ("max_rounds", _c.c_int64),
        ("workers", _c.c_int32), ("q", _c.c_int32), ("updaters", _c.c_int32), ("tagged", _c.c_int32),
        ("sample_counter", _vp), ("update_order", _vp), ("exited", _vp), ("last_avg_stamp", _vp),
        ("synced_at", _vp), ("switch_point", _c.c_int64), ("period", _c.c_int64),
        ("stop_after", _c.c_int64), ("arenas", _vp), ("tags", _vp), ("lo", _size), ("hi", _size),
        ("n", _size), ("mean_out", _vp), ("stream", _vp), ("t0", _c.c_double), ("rec", _vp),
        ("rec_wall_ms", _vp), ("max_records", _c.c_int64),
        ("eval_interval", _c.c_int64), ("mean_parts", _vp), ("shard_bounds", _vp), ("eval_buf", _vp),
        ("eval_cap", _c.c_int64), ("eval_rec", _vp), ("eval_wall_ms", _vp), ("eval_count", _vp),
        ("flops_cell", _vp), ("classified_cell", _vp), ("clean_cell", _vp),
        ("time_rounds", _c.c_int32), ("k4_ms", _vp), ("k4_rounds", _vp),
        ("stamp_floor", _c.c_int32), ("round_cell", _vp),
    ]


class UpdaterStats(ctypes.Structure):
    """``lpp_updater_stats``."""

    _fields_ = [("steps", _c.c_int64), ("flops", _c.c_int64), ("apply_launches", _c.c_int64),
                ("apply_ms", _c.c_double), ("apply_bytes", _c.c_double),
                ("graph_kernels", _c.c_int64)]


_SIGS = {
    "lpp_abi_version": (_c.c_int, []),
    "lpp_last_error": (_c.c_char_p, []),
    "lpp_launch_count": (_c.c_ulonglong, []),
    "lpp_atomic_load_i64": (_c.c_int64, [_vp]),
    "lpp_atomic_store_i64": (None, [_vp, _c.c_int64]),
    "lpp_atomic_fetch_add_i64": (_c.c_int64, [_vp, _c.c_int64]),
    "lpp_atomic_cas_i64": (_c.c_int, [_vp, _c.c_int64, _c.c_int64]),
    "lpp_atomic_wait_ge_i64": (_c.c_int64, [_vp, _c.c_int64, _vp, _c.c_int]),
    "lpp_arena_create": (_c.c_int, [_c.c_int, _size, _c.POINTER(_vp)]),
    "lpp_arena_destroy": (_c.c_int, [_vp]),
    "lpp_arena_data": (_vp, [_vp]),
    "lpp_arena_size": (_size, [_vp]),
    "lpp_arena_device": (_c.c_int, [_vp]),
    "lpp_arena_export_ipc": (_c.c_int, [_vp, _vp]),
    "lpp_ipc_open": (_c.c_int, [_c.c_int, _vp, _c.POINTER(_vp)]),
    "lpp_ipc_close": (_c.c_int, [_c.c_int, _vp]),
    "lpp_enable_peer_access": (_c.c_int, [_c.c_int, _c.c_int]),
    "lpp_can_access_peer": (_c.c_int, [_c.c_int, _c.c_int, _c.POINTER(_c.c_int)]),
    "lpp_apply_sgd": (
        _c.c_int,
        [_vp, _vp, _vp, _size, _c.c_float, _vp, _c.c_float, _c.c_float, _c.c_int, _vp],
    ),
    "lpp_accum": (_c.c_int, [_vp, _size, _size, _vp, _size, _c.c_float, _c.c_int, _vp]),
    "lpp_apply_snapshot": (
        _c.c_int,
        [_vp, _vp, _vp, _vp, _vp, _size, _size, _size, _c.c_float, _vp, _c.c_float, _c.c_float,
         _c.c_int32, _vp],
    ),
    "lpp_apply_snapshot_plan": (
        _c.c_int,
        [_vp, _vp, _vp, _vp, _vp, _size, _size, _size, _c.c_float, _vp, _c.c_float, _c.c_float,
         _c.c_int32, _c.POINTER(TagPlan), _vp],
    ),
    "lpp_gather_tags_floor": (_c.c_int, [_vp, _vp, _size, _vp, _vp, _vp, _vp]),
    "lpp_classify": (_c.c_int, [_vp, _size, _vp, _vp, _vp]),
    "lpp_set_i64": (_c.c_int, [_vp, _c.c_int64, _vp]),
    "lpp_publish_stamp": (_c.c_int, [_vp, _c.c_int, _c.c_int32, _vp]),
    "lpp_gather_block_stamps": (_c.c_int, [_vp, _vp, _c.c_int, _vp, _size, _vp, _vp, _vp, _vp]),
    "lpp_host_alloc": (_c.c_int, [_size, _c.POINTER(_vp), _c.POINTER(_vp)]),
    "lpp_host_free": (_c.c_int, [_vp]),
    "lpp_load_f32": (_c.c_int, [_vp, _size, _size, _c.POINTER(_c.c_float), _vp]),
    "lpp_store_f32": (_c.c_int, [_vp, _size, _size, _c.c_float, _vp]),
    "lpp_snapshot": (_c.c_int, [_vp, _vp, _size, _vp]),
    "lpp_average_shard": (
        _c.c_int,
        [_c.POINTER(_vp), _c.c_int, _size, _size, _vp, _c.c_int, _vp],
    ),
    "lpp_apply_sgd_tagged": (
        _c.c_int,
        [_vp, _vp, _vp, _size, _c.c_float, _vp, _c.c_float, _c.c_float, _c.c_int, _vp,
         _c.c_int32, _vp],
    ),
    "lpp_accum_tagged": (
        _c.c_int, [_vp, _vp, _size, _size, _vp, _size, _c.c_float, _c.c_int32, _c.c_int, _vp]),
    "lpp_snapshot_tagged": (_c.c_int, [_vp, _vp, _vp, _vp, _size, _vp, _vp]),
    "lpp_gather_tags": (_c.c_int, [_vp, _vp, _size, _vp, _vp]),
    "lpp_average_shard_tagged": (
        _c.c_int,
        [_c.POINTER(_vp), _c.POINTER(_vp), _c.POINTER(_c.c_int32), _c.c_int, _size, _size, _vp,
         _c.c_int, _vp],
    ),
    "lpp_mc_supported": (_c.c_int, [_c.c_int, _c.POINTER(_c.c_int)]),
    "lpp_mc_granularity": (_c.c_int, [_c.c_int, _c.c_int, _c.POINTER(_size)]),
    "lpp_vmm_create": (_c.c_int, [_c.c_int, _size, _c.POINTER(_vp)]),
    "lpp_vmm_ptr": (_vp, [_vp]),
    "lpp_vmm_size": (_size, [_vp]),
    "lpp_vmm_destroy": (_c.c_int, [_vp]),
    "lpp_mc_create": (_c.c_int, [_c.c_int, _size, _c.POINTER(_vp)]),
    "lpp_mc_export_fd": (_c.c_int, [_vp, _c.POINTER(_c.c_int)]),
    "lpp_mc_import_fd": (_c.c_int, [_c.c_int, _size, _c.POINTER(_vp)]),
    "lpp_mc_add_device": (_c.c_int, [_vp, _c.c_int]),
    "lpp_mc_bind": (_c.c_int, [_vp, _vp, _size]),
    "lpp_mc_map": (_c.c_int, [_vp, _c.c_int, _c.POINTER(_vp)]),
    "lpp_mc_destroy": (_c.c_int, [_vp]),
    "lpp_nvls_mean_shard": (_c.c_int, [_vp, _vp, _size, _size, _c.c_int, _vp]),
    "lpp_nvls_apply": (_c.c_int, [_vp, _vp, _vp, _size, _vp, _c.c_int32, _vp]),
    "lpp_copy_async": (_c.c_int, [_vp, _vp, _size, _vp]),
    "lpp_graph_launch": (_c.c_int, [_vp, _vp]),
    "lpp_host_gather_rows": (_c.c_int, [_vp, _vp, _size, _size, _vp, _size]),
    "lpp_l2_flush": (_c.c_int, [_vp, _size, _vp]),
    "lpp_sm_count": (_c.c_int, [_c.c_int, _c.POINTER(_c.c_int)]),
    "lpp_lr_at": (_c.c_double, [_c.c_int, _c.c_double, _c.c_double, _c.c_int64, _c.c_int64, _vp,
                                _c.c_int, _c.c_double, _c.c_int64]),
    "lpp_select_block": (_c.c_int, [_c.c_int64, _c.c_int64, _c.c_int, _c.c_int]),
    "lpp_sample_indices": (_c.c_int, [_vp, _vp, _c.c_int32, _c.c_int64, _c.c_uint64, _vp]),
    "lpp_sample_indices_host": (_c.c_int, [_vp, _c.c_int32, _c.c_int64, _c.c_uint64, _c.c_int64]),
    "lpp_sample_epoch": (_c.c_int, [_vp, _vp, _c.c_int32, _c.c_int64, _c.c_int64, _c.c_int64,
                                    _c.c_uint64, _vp]),
    "lpp_sample_epoch_host": (_c.c_int, [_vp, _c.c_int32, _c.c_int64, _c.c_int64, _c.c_int64,
                                         _c.c_uint64, _c.c_int64]),
    "lpp_updater_run": (_c.c_int, [_c.POINTER(UpdaterCfg), _c.POINTER(UpdaterStats)]),
    "lpp_nprng_create": (_c.c_int, [_vp, _c.c_int, _c.POINTER(_vp)]),
    "lpp_nprng_destroy": (_c.c_int, [_vp]),
    "lpp_nprng_integers": (_c.c_int, [_vp, _c.c_int64, _c.c_int32, _vp]),
    "lpp_nprng_choice": (_c.c_int, [_vp, _c.c_int64, _c.c_int32, _vp]),
    "lpp_nprng_permutation": (_c.c_int, [_vp, _c.c_int64, _vp]),
    "lpp_averager_run": (_c.c_int, [_c.POINTER(AveragerCfg), _c.POINTER(_c.c_int64)]),
    "lpp_fill_i32": (_c.c_int, [_vp, _size, _c.c_int32, _vp]),
    "lpp_conv3x3_supported": (_c.c_int, [_c.c_int, _c.c_int]),
    "lpp_fma_probe": (_c.c_int, [_vp, _c.c_int, _c.c_int, _vp]),
    "lpp_conv1x1s2_supported": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int]),
    "lpp_conv3x3s2_supported": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int]),
    "lpp_conv3x3s2_wgrad_workspace": (_size, [_c.c_int, _c.c_int, _c.c_int, _c.c_int]),
    "lpp_conv3x3s2_f32": (_c.c_int, [_vp, _vp, _vp, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _vp, _size,
                                      _vp, _vp, _vp]),
    "lpp_conv1x1s2_wgrad_workspace": (_size, [_c.c_int, _c.c_int, _c.c_int, _c.c_int]),
    "lpp_conv1x1s2_f32": (_c.c_int, [_vp, _vp, _vp, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _vp, _size,
                                      _vp, _vp, _vp]),
    "lpp_conv3x3_f32": (_c.c_int, [_vp, _vp, _vp, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _vp, _size, _vp, _vp,
                                    _vp]),
    "lpp_conv3x3_stats_workspace": (_size, [_c.c_int, _c.c_int, _c.c_int]),
    "lpp_conv3x3_tapmajor": (_c.c_int, [_vp, _vp, _c.c_int, _vp]),
    "lpp_conv1x1s2_stats_workspace": (_size, [_c.c_int, _c.c_int, _c.c_int, _c.c_int]),
    "lpp_conv3x3s2_stats_workspace": (_size, [_c.c_int, _c.c_int, _c.c_int, _c.c_int]),
    "lpp_bn_backward_workspace": (_size, [_c.c_int64, _c.c_int]),
    "lpp_bn_backward_f32": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _size, _vp, _c.c_int64,
                                        _c.c_int, _c.c_int, _vp]),
    "lpp_stem_workspace": (_size, [_c.c_int]),
    "lpp_stem_f32": (_c.c_int, [_vp, _vp, _vp, _c.c_int, _c.c_int, _vp, _size, _vp, _vp, _vp]),
    "lpp_bn_apply_f32": (_c.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c.c_int64, _c.c_int,
                                     _c.c_float, _c.c_float, _c.c_int, _vp]),
    "lpp_conv3x3_wgrad_workspace": (_size, [_c.c_int, _c.c_int, _c.c_int]),
    "lpp_conv3x3_wgrad_f32": (_c.c_int, [_vp, _vp, _vp, _vp, _size, _vp, _c.c_int, _c.c_int, _c.c_int, _vp]),
}

EXPORTED = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def launch_count() -> int:
    """Kernels launched by the library so far (an atomic counter in C; the
    bench reports its delta over the timed region)."""
    return int(lib.lpp_launch_count())


def last_error() -> str:
    msg = lib.lpp_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    if status == 0:
        return
    err = last_error()
    # the C side names the entry point already; do not repeat it
    msg = err if err.startswith(what.split("(")[0] + ":") else f"{what}: {err}"
    if status == E_VALUE:
        raise ValueError(msg)
    if status == E_INDEX:
        raise IndexError(msg)
    if status == E_NOMEM:
        raise MemoryError(msg)
    raise LppError(msg)


# ---------------------------------------------------------------------------
# host atomics on numpy int64 cells (K6)


def _cell_ptr(buf: np.ndarray, i: int) -> int:
    if buf.dtype != np.int64 or not buf.flags.c_contiguous:
        raise ValueError("counter buffer must be C-contiguous int64")
    if not 0 <= i < buf.shape[0]:
        raise IndexError(f"index {i} out of range [0, {buf.shape[0]})")
    return buf.ctypes.data + 8 * i


def cell_address(buf: np.ndarray, i: int) -> int:
    """Address of int64 cell i (validated); the caller keeps ``buf`` alive."""
    return _cell_ptr(buf, i)


def atomic_load(buf: np.ndarray, i: int = 0) -> int:
    return int(lib.lpp_atomic_load_i64(_cell_ptr(buf, i)))


def atomic_store(buf: np.ndarray, i: int, v: int) -> None:
    lib.lpp_atomic_store_i64(_cell_ptr(buf, i), int(v))


def atomic_fetch_add(buf: np.ndarray, i: int, delta: int) -> int:
    return int(lib.lpp_atomic_fetch_add_i64(_cell_ptr(buf, i), int(delta)))


def atomic_cas(buf: np.ndarray, i: int, expected: int, desired: int) -> bool:
    return bool(lib.lpp_atomic_cas_i64(_cell_ptr(buf, i), int(expected), int(desired)))


def atomic_wait_ge(buf: np.ndarray, i: int, target: int, abort: np.ndarray | None = None,
                   abort_i: int = 0, max_sleep_us: int = 200) -> int | None:
    """Block (GIL released) until buf[i] >= target; None if aborted."""
    ap = _cell_ptr(abort, abort_i) if abort is not None else None
    v = int(lib.lpp_atomic_wait_ge_i64(_cell_ptr(buf, i), int(target), ap, int(max_sleep_us)))
    return None if v == -(2**63) else v


# ---------------------------------------------------------------------------
# device-side wrappers (raw pointers; the torch layer lives in arena.py)


def sm_count(device: int) -> int:
    out = _c.c_int(0)
    check(lib.lpp_sm_count(int(device), _c.byref(out)), "sm_count")
    return out.value


def apply_sgd(x_ptr: int, g_ptr: int, m_ptr: int | None, n: int, lr: float,
              lr_dev_ptr: int | None, mu: float, wd: float, mode: int, stream: int) -> None:
    check(
        lib.lpp_apply_sgd(x_ptr, g_ptr, m_ptr, n, lr, lr_dev_ptr, mu, wd, mode, stream),
        "apply_sgd",
    )


def apply_snapshot(x_ptr, g_ptr, m_ptr, replica_ptr, tags_ptr, n, lo, hi, lr, lr_dev_ptr, mu, wd,
                   stamp, stream) -> None:
    check(lib.lpp_apply_snapshot(x_ptr, g_ptr, m_ptr, replica_ptr, tags_ptr, n, lo, hi, lr,
                                 lr_dev_ptr, mu, wd, int(stamp), stream), "apply_snapshot")


def apply_snapshot_plan(x_ptr, g_ptr, m_ptr, replica_ptr, tags_ptr, n, lo, hi, lr, lr_dev_ptr, mu,
                        wd, stamp, plan: TagPlan, stream) -> None:
    check(lib.lpp_apply_snapshot_plan(x_ptr, g_ptr, m_ptr, replica_ptr, tags_ptr, n, lo, hi, lr,
                                      lr_dev_ptr, mu, wd, stamp, ctypes.byref(plan), stream),
          "apply_snapshot_plan")


def gather_tags_floor(tags_ptr, idx_ptr, k, floor_ptr, out_dev_ptr, out_host_ptr, stream) -> None:
    check(lib.lpp_gather_tags_floor(tags_ptr, idx_ptr, k, floor_ptr, out_dev_ptr, out_host_ptr, stream),
          "gather_tags_floor")


def classify(tags_ptr, k, claim_ptr, out_ptr, stream) -> None:
    check(lib.lpp_classify(tags_ptr, k, claim_ptr, out_ptr, stream), "classify")


def gather_block_stamps(stamps_ptr, bounds_ptr, nb, idx_ptr, k, floor_ptr, out_dev_ptr, out_host_ptr,
                        stream) -> None:
    check(lib.lpp_gather_block_stamps(stamps_ptr, bounds_ptr, nb, idx_ptr, k, floor_ptr, out_dev_ptr,
                                      out_host_ptr, stream), "gather_block_stamps")


def publish_stamp(stamps_ptr: int, block_id: int, stamp: int, stream: int) -> None:
    check(lib.lpp_publish_stamp(stamps_ptr, block_id, stamp, stream), "publish_stamp")


def set_i64(dev_ptr: int, v: int, stream: int) -> None:
    check(lib.lpp_set_i64(dev_ptr, int(v), stream), "set_i64")


def load_f32(arena_ptr: int, length: int, i: int, stream: int = 0) -> float:
    out = ctypes.c_float()
    check(lib.lpp_load_f32(arena_ptr, length, i, ctypes.byref(out), stream), "load_f32")
    return float(out.value)


def store_f32(arena_ptr: int, length: int, i: int, v: float, stream: int = 0) -> None:
    check(lib.lpp_store_f32(arena_ptr, length, i, float(v), stream), "store_f32")


class HostBuffer:
    """Mapped, portable host memory (``lpp_host_alloc``) that kernels read
    and write directly; ``view(dtype, shape)`` gives numpy views, ``dev`` the
    device address of the first byte."""

    def __init__(self, nbytes: int):
        h, d = ctypes.c_void_p(), ctypes.c_void_p()
        check(lib.lpp_host_alloc(int(nbytes), ctypes.byref(h), ctypes.byref(d)), "host_alloc")
        self.ptr, self.dev, self.nbytes = int(h.value), int(d.value), int(nbytes)
        self._raw = (ctypes.c_char * self.nbytes).from_address(self.ptr)

    def view(self, dtype, shape, offset: int = 0) -> np.ndarray:
        dt = np.dtype(dtype)
        count = int(np.prod(shape))
        if offset + count * dt.itemsize > self.nbytes:
            raise ValueError("view exceeds the host buffer")
        return np.frombuffer(self._raw, dtype=dt, count=count, offset=offset).reshape(shape)

    def close(self) -> None:
        if self.ptr:
            self._raw = None
            check(lib.lpp_host_free(self.ptr), "host_free")
            self.ptr = self.dev = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def accum(dst_ptr: int, dst_len: int, start: int, delta_ptr: int, n: int, scale: float,
          mode: int, stream: int) -> None:
    check(lib.lpp_accum(dst_ptr, dst_len, start, delta_ptr, n, scale, mode, stream), "accum")


def snapshot(src_ptr: int, out_ptr: int, n: int, stream: int) -> None:
    check(lib.lpp_snapshot(src_ptr, out_ptr, n, stream), "snapshot")


def average_shard(arena_ptrs, lo: int, hi: int, mean_out_ptr: int | None, mode: int,
                  stream: int) -> None:
    q = len(arena_ptrs)
    table = (_vp * max(q, 1))(*arena_ptrs)
    check(lib.lpp_average_shard(table, q, lo, hi, mean_out_ptr, mode, stream), "average_shard")


def apply_sgd_tagged(x_ptr, g_ptr, m_ptr, n, lr, lr_dev_ptr, mu, wd, mode, tags_ptr, stamp,
                     stream) -> None:
    check(lib.lpp_apply_sgd_tagged(x_ptr, g_ptr, m_ptr, n, lr, lr_dev_ptr, mu, wd, mode, tags_ptr,
                                   int(stamp), stream), "apply_sgd_tagged")


def accum_tagged(dst_ptr, tags_ptr, dst_len, start, delta_ptr, n, scale, stamp, mode,
                 stream) -> None:
    check(lib.lpp_accum_tagged(dst_ptr, tags_ptr, dst_len, start, delta_ptr, n, scale,
                               int(stamp), mode, stream), "accum_tagged")


def snapshot_tagged(src_ptr, tags_ptr, out_ptr, out_tags_ptr, n, min_tag_ptr, stream) -> None:
    check(lib.lpp_snapshot_tagged(src_ptr, tags_ptr, out_ptr, out_tags_ptr, n, min_tag_ptr,
                                  stream), "snapshot_tagged")


def gather_tags(tags_ptr, idx_ptr, k, out_ptr, stream) -> None:
    check(lib.lpp_gather_tags(tags_ptr, idx_ptr, k, out_ptr, stream), "gather_tags")


def average_shard_tagged(arena_ptrs, tag_ptrs, stamps, lo, hi, mean_out_ptr, mode,
                         stream) -> None:
    q = len(arena_ptrs)
    a = (_vp * q)(*arena_ptrs)
    t = (_vp * q)(*tag_ptrs)
    st = (_c.c_int32 * q)(*[int(v) for v in stamps])
    check(lib.lpp_average_shard_tagged(a, t, st, q, lo, hi, mean_out_ptr, mode, stream),
          "average_shard_tagged")


def graph_launch(exec_ptr: int, stream: int) -> None:
    rc = lib.lpp_graph_launch(exec_ptr, stream)
    if rc:
        check(rc, "graph_launch")


def copy_async(dst_ptr: int, src_ptr: int, nbytes: int, stream: int) -> None:
    rc = lib.lpp_copy_async(dst_ptr, src_ptr, nbytes, stream)
    if rc:
        check(rc, "copy_async")


def l2_flush(ptr: int, nbytes: int, stream: int) -> None:
    check(lib.lpp_l2_flush(ptr, nbytes, stream), "l2_flush")


# -- native updater loop helpers ---------------------------------------------


def lr_at_native(sched, s: int) -> float:
    """``lpp_lr_at`` for an ``LrSchedule`` (the native loop's lr)."""
    ms = np.ascontiguousarray(sched.milestones, dtype=np.int64)
    return float(lib.lpp_lr_at(0 if sched.kind == "cosine" else 1, sched.alpha0, sched.peak,
                               sched.warmup, sched.total, ms.ctypes.data if len(ms) else None,
                               len(ms), sched.gamma, int(s)))


def select_block_native(s: int, warm_start: int, num_blocks: int, rank: int) -> int:
    b = int(lib.lpp_select_block(int(s), int(warm_start), int(num_blocks), int(rank)))
    if b < 0:
        raise ValueError(last_error())
    return b


def sample_indices(idx_ptr: int, step_ptr: int, batch: int, n: int, key: int, stream: int) -> None:
    check(lib.lpp_sample_indices(idx_ptr, step_ptr, batch, n, key & (2**64 - 1), stream),
          "sample_indices")


def sample_indices_host(batch: int, n: int, key: int, step: int) -> np.ndarray:
    out = np.zeros(batch, dtype=np.int64)
    check(lib.lpp_sample_indices_host(out.ctypes.data, batch, n, key & (2**64 - 1), step),
          "sample_indices_host")
    return out


def updater_run(cfg: UpdaterCfg) -> UpdaterStats:
    """Run one updater's loop natively (ctypes drops the GIL for the call)."""
    st = UpdaterStats()
    check(lib.lpp_updater_run(ctypes.byref(cfg), ctypes.byref(st)), "updater_run")
    return st


def host_gather_rows(dst_ptr: int, src_ptr: int, n_rows: int, row_bytes: int, idx: np.ndarray) -> None:
    """dst row i = src row idx[i] (host memory, GIL released)."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    check(lib.lpp_host_gather_rows(dst_ptr, src_ptr, n_rows, row_bytes, idx.ctypes.data, len(idx)),
          "host_gather_rows")


def averager_run(cfg: AveragerCfg) -> int:
    """Run one worker's averager natively (GIL released); returns rounds."""
    n = ctypes.c_int64(0)
    check(lib.lpp_averager_run(ctypes.byref(cfg), ctypes.byref(n)), "averager_run")
    return int(n.value)


def fill_i32(ptr: int, n: int, value: int, stream: int) -> None:
    check(lib.lpp_fill_i32(ptr, n, int(value), stream), "fill_i32")


def sample_epoch(idx_ptr: int, step_ptr: int, batch: int, base: int, stride: int, length: int,
                 key: int, stream: int) -> None:
    check(lib.lpp_sample_epoch(idx_ptr, step_ptr, batch, base, stride, length, key & (2**64 - 1),
                               stream), "sample_epoch")


def sample_epoch_host(batch: int, base: int, stride: int, length: int, key: int, step: int) -> np.ndarray:
    out = np.zeros(batch, dtype=np.int64)
    check(lib.lpp_sample_epoch_host(out.ctypes.data, batch, base, stride, length, key & (2**64 - 1),
                                    step), "sample_epoch_host")
    return out


class NpRng:
    """The reference's numpy sampling stream, restated natively (tests)."""

    def __init__(self, *entropy: int):
        ent = np.array(entropy, dtype=np.uint64)
        h = ctypes.c_void_p()
        check(lib.lpp_nprng_create(ent.ctypes.data, len(ent), ctypes.byref(h)), "nprng_create")
        self._h = h

    def integers(self, n: int, b: int) -> np.ndarray:
        out = np.zeros(b, dtype=np.int64)
        check(lib.lpp_nprng_integers(self._h, n, b, out.ctypes.data), "nprng_integers")
        return out

    def choice(self, pop: int, k: int) -> np.ndarray:
        out = np.zeros(k, dtype=np.int64)
        check(lib.lpp_nprng_choice(self._h, pop, k, out.ctypes.data), "nprng_choice")
        return out

    def permutation(self, m: int) -> np.ndarray:
        out = np.zeros(m, dtype=np.int64)
        check(lib.lpp_nprng_permutation(self._h, m, out.ctypes.data), "nprng_permutation")
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib.lpp_nprng_destroy(self._h)
            self._h = None
