"""Block partition of the arena and the per-slot block scheduler (a4, a5).

Same names, argument meaning and error behaviour as the reference
``asyncsgd.partition`` (``/root/reference/pkg/src/asyncsgd/partition.py``):

* block 0 is the whole vector; block i >= 1 is ``[b_{i-1}, b_i)``
  (``partition.py:40-59``);
* ``select_block`` is the PASSM+ rule (``partition.py:132-145``);
* ``balanced_boundaries`` returns exactly the split the reference's brute
  force returns (``partition.py:86-129``), but is exact and fast for any
  layer count (the reference enumerates C(n-1, U-1) splits, which is
  infeasible for ResNet-50's 161 tensors at U=8).

Why the fast path is exact: the reference key is
``(worst suffix cost, worst block size, bounds)`` minimised
lexicographically.  Block 1 always starts at layer 0, so with non-negative
layer costs the worst suffix cost is ``suffix[0]`` for *every* split; the key
reduces to (worst size, bounds).  The minimum worst size ``W`` is found by
binary search over the feasibility test, and the lexicographically smallest
bounds with worst size ``W`` by choosing each cut as early as the remaining
layers still allow.  Negative costs (allowed by the reference's signature)
fall back to exhaustive enumeration.
"""

from __future__ import annotations

import enum
import itertools
from dataclasses import dataclass
from typing import NamedTuple, Sequence


class Block(NamedTuple):
    """Element range [start, stop) of the flat arena (a K1/K2 apply range)."""

    start: int
    stop: int

    @property
    def length(self) -> int:
        return self.stop - self.start


class SelectionReason(enum.Enum):
    """Why a slot trains the block it trains (partition.py:132-145)."""

    WARM_START = "warm_start"                # s <= T_st: everyone trains the full model
    ALTERNATE_FULL = "alternate_full"        # odd distance past T_st: full model
    ALTERNATE_PARTIAL = "alternate_partial"  # even distance: the updater's own block


@dataclass(frozen=True)
class BlockChoice:
    block_id: int
    reason: SelectionReason


@dataclass(frozen=True)
class BlockPartition:
    """Boundaries 0 = b_0 < ... < b_U = dim; block 0 is the whole arena,
    block i in 1..U the slice [b_{i-1}, b_i)."""

    dim: int
    boundaries: tuple[int, ...]

    @property
    def num_blocks(self) -> int:
        return len(self.boundaries) - 1

    def block(self, block_id: int) -> Block:
        u = self.num_blocks
        if block_id == 0:
            return Block(0, self.dim)
        if 0 < block_id <= u:
            return Block(*self.boundaries[block_id - 1:block_id + 1])
        raise ValueError(f"block id {block_id} outside [0, {u}]")

    def blocks(self) -> list[Block]:
        return [Block(a, b) for a, b in zip(self.boundaries, self.boundaries[1:])]


def _partition_error(dim: int, b: tuple[int, ...]) -> str | None:
    if dim < 0:
        return "dimension must be non-negative"
    if len(b) < 2 or b[0] != 0 or b[-1] != dim:
        return f"boundaries must run from 0 to {dim}, got {b}"
    if not all(x < y for x, y in zip(b, b[1:])):
        return f"boundaries must be strictly ascending, got {b}"
    return None


def make_partition(dim: int, boundaries: Sequence[int]) -> BlockPartition:
    b = tuple(map(int, boundaries))
    err = _partition_error(dim, b)
    if err is not None:
        raise ValueError(err)
    return BlockPartition(dim, b)


def even_boundaries(dim: int, num_blocks: int) -> tuple[int, ...]:
    """Near-equal contiguous slices (unlayered objectives): the first
    ``dim % num_blocks`` slices hold one extra element."""
    if not 1 <= num_blocks <= dim:
        raise ValueError(f"cannot split {dim} elements into {num_blocks} blocks")
    base, extra = divmod(dim, num_blocks)
    sizes = [base + 1] * extra + [base] * (num_blocks - extra)
    return (0, *itertools.accumulate(sizes))


def _min_blocks_from(sizes: list[int], start: int, cap: int) -> int:
    """Fewest contiguous blocks covering sizes[start:] with each sum <= cap."""
    count, acc = 0, None
    for s in sizes[start:]:
        if s > cap:
            return 1 << 60
        if acc is None or acc + s > cap:
            count += 1
            acc = s
        else:
            acc += s
    return count


def _balanced_fast(sizes: list[int], k: int) -> tuple[int, ...]:
    n = len(sizes)
    prefix = [0]
    for s in sizes:
        prefix.append(prefix[-1] + s)
    lo, hi = max(sizes), prefix[-1]
    while lo < hi:  # smallest cap W with a feasible k-split (k <= n always holds)
        mid = (lo + hi) // 2
        if _min_blocks_from(sizes, 0, mid) <= k:
            hi = mid
        else:
            lo = mid + 1
    cap = lo
    cuts = [0]
    start = 0
    for remaining in range(k, 1, -1):
        # earliest cut c > start leaving layers [c, n) splittable into
        # `remaining - 1` blocks of size <= cap (each non-empty)
        chosen = None
        for c in range(start + 1, n - (remaining - 1) + 1):
            if prefix[c] - prefix[start] > cap:
                break
            if _min_blocks_from(sizes, c, cap) <= remaining - 1:
                chosen = c
                break
        assert chosen is not None
        cuts.append(chosen)
        start = chosen
    cuts.append(n)
    return tuple(prefix[c] for c in cuts)


def _balanced_exhaustive(sizes: list[int], k: int, costs: list[float]) -> tuple[int, ...]:
    n = len(sizes)
    suffix = [0.0] * (n + 1)
    for i in range(n - 1, -1, -1):
        suffix[i] = suffix[i + 1] + costs[i]
    prefix = [0]
    for s in sizes:
        prefix.append(prefix[-1] + s)
    best = None
    for cut in itertools.combinations(range(1, n), k - 1):
        sp = (0, *cut, n)
        key = (
            max(suffix[sp[i]] for i in range(k)),
            max(prefix[sp[i + 1]] - prefix[sp[i]] for i in range(k)),
            tuple(prefix[c] for c in sp),
        )
        if best is None or key < best:
            best = key
    return best[2]


def balanced_boundaries(
    layer_sizes: Sequence[int],
    num_blocks: int,
    layer_costs: Sequence[float] | None = None,
) -> tuple[int, ...]:
    """Layer-aligned boundaries minimising the worst block cost (see module doc)."""
    sizes = [int(s) for s in layer_sizes]
    if not sizes or any(s <= 0 for s in sizes):
        raise ValueError("layer sizes must be positive")
    if num_blocks < 1 or num_blocks > len(sizes):
        raise ValueError(f"cannot split {len(sizes)} layers into {num_blocks} blocks")
    costs = [float(c) for c in layer_costs] if layer_costs is not None else [float(s) for s in sizes]
    if len(costs) != len(sizes):
        raise ValueError("layer_costs length must match layer_sizes")
    if all(c >= 0 for c in costs):
        return _balanced_fast(sizes, num_blocks)
    return _balanced_exhaustive(sizes, num_blocks, costs)


def select_block(s: int, warm_start_budget: int, num_blocks: int, rank: int) -> BlockChoice:
    """PASSM+ block for slot ``s`` and updater ``rank`` (1-based)."""
    if rank < 1 or rank > num_blocks:
        raise ValueError(f"rank {rank} outside [1, {num_blocks}]")
    if s <= warm_start_budget:
        return BlockChoice(0, SelectionReason.WARM_START)
    if (s - warm_start_budget) & 1:
        return BlockChoice(0, SelectionReason.ALTERNATE_FULL)
    return BlockChoice(rank, SelectionReason.ALTERNATE_PARTIAL)
