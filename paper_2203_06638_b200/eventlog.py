"""NDJSON event log of a GPU run, in the reference's schema.

``save_event_log(path, result)`` writes one JSON object per update and per
averaging stamp with exactly the keys of the reference's
``save_event_log`` (/root/reference/pkg/src/asyncsgd/instrumentation.py:371-421),
so the reference's ``load_event_log`` / ``replay_rounds`` (and
``oracle/replay.py``) can audit a GPU run: replayed round means vs the
means the run measured.  Device tensors (grads, snapshots, tags) are
copied to the host here, after the run — nothing is logged on the hot path.
"""

from __future__ import annotations

import gzip
import json
from pathlib import Path

import numpy as np


def _host(a):
    if a is None:
        return None
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.asarray(a).tolist()


def save_event_log(path, result) -> None:
    path = Path(path)
    opener = gzip.open if path.suffix == ".gz" else open
    with opener(path, "wt") as fh:
        for rec in result.updates:
            fh.write(json.dumps({
                "kind": "update", "worker": rec.worker, "rank": rec.rank, "s": rec.s, "u": rec.u,
                "k_claim": rec.k_claim, "block_id": rec.block_id, "reason": rec.reason,
                "lr": rec.lr, "flops": rec.flops, "backward_flops": rec.backward_flops,
                "clean": rec.clean, "tag_indices": _host(rec.tag_indices), "tags": _host(rec.tags),
                "grad": _host(rec.grad), "snapshot": _host(rec.snapshot)}) + "\n")
        for st in result.stamps:
            fh.write(json.dumps({
                "kind": "average", "worker": st.worker, "round": st.round, "u": st.u,
                "s_cur": st.s_cur, "k_delta": st.k_delta, "wall_ms": st.wall_ms,
                "snapshot": _host(st.snapshot), "mean": _host(st.mean)}) + "\n")
