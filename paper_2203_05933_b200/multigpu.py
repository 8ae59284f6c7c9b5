"""Multi-GPU target sharding (one process per GPU).

Every rank builds the same plan (identical tree and lists: the build is
deterministic), keeps the whole upward pass, and evaluates the target side
(M2L, L2L, L2P + near-field P2P) only for a Morton-contiguous range of target
leaves.  Ranges are balanced by estimated work -- near-field pairs plus M2L
translations of the leaf, not point counts (a uniform 4M grid and the star
strip have very different per-leaf costs).  Non-owned outputs are 0.0, so one
all-reduce(SUM) assembles the full potential vector bit-identically to the
single-GPU result; inside the timed step there is no collective at all.

Only host logic lives here; it is exercised on CPU with gloo (tests/test_multigpu_cpu.py).
"""
from __future__ import annotations

import numpy as np


def _squash(v):
    v = v & 0x55555555
    v = (v | (v >> 1)) & 0x33333333
    v = (v | (v >> 2)) & 0x0F0F0F0F
    v = (v | (v >> 4)) & 0x00FF00FF
    v = (v | (v >> 8)) & 0x0000FFFF
    return v


def _spread(v):
    v = (v | (v << 8)) & 0x00FF00FF
    v = (v | (v << 4)) & 0x0F0F0F0F
    v = (v | (v << 2)) & 0x33333333
    v = (v | (v << 1)) & 0x55555555
    return v


def leaf_costs(src_off, tgt_off, levels, order, m2l_per_leaf=None):
    """Work estimate per target leaf (Morton order), in FP64 instructions.

    near field: ntgt * (sources in the 3x3 neighbourhood) * 14
    (summation.cpp:330-344); local evaluation ntgt * 4(P+1); M2L of the leaf
    box ~ 4P(P+1) per list entry (27 in the interior).
    """
    src_off = np.asarray(src_off, np.int64)
    tgt_off = np.asarray(tgt_off, np.int64)
    nb = 1 << levels
    nleaf = nb * nb
    b = np.arange(nleaf, dtype=np.int64)
    ix, iy = _squash(b), _squash(b >> 1)
    scnt = np.diff(src_off)
    ntgt = np.diff(tgt_off)
    nsrc = np.zeros(nleaf, np.int64)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            jx, jy = ix + dx, iy + dy
            ok = (jx >= 0) & (jx < nb) & (jy >= 0) & (jy < nb)
            sid = _spread(np.where(ok, jx, 0)) | (_spread(np.where(ok, jy, 0)) << 1)
            nsrc += np.where(ok, scnt[sid], 0)
    m2l = np.full(nleaf, 27, np.int64) if m2l_per_leaf is None else np.asarray(m2l_per_leaf)
    cost = ntgt * nsrc * 14.0 + ntgt * 4.0 * (order + 1) + np.where(ntgt > 0, m2l, 0) * 4.0 * order * (order + 1)
    return cost


def balanced_ranges(costs, world):
    """Contiguous [begin, end) leaf ranges with near-equal cumulative cost."""
    costs = np.asarray(costs, float)
    n = costs.size
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def shard_plan(plan, rank, world):
    """Restricts ``plan`` to this rank's balanced unit range; returns the range.

    Reference-mode (uniform) trees are balanced with ``leaf_costs`` from the
    dumped tree; adaptive (native-mode) trees with the library's per-unit
    estimates (vpg_plan_shard_units: their units are the target leaves)."""
    if plan.info()["mode"] == 1 and plan.info()["family"] == 0:
        costs = plan.shard_units()
        lo, hi = balanced_ranges(costs, world)[rank]
        plan.set_shard(lo, hi)
        return lo, hi
    t = plan.dump_tree()
    costs = leaf_costs(t["src_off"], t["tgt_off"], plan.levels(), plan.expansion_order())
    lo, hi = balanced_ranges(costs, world)[rank]
    plan.set_shard(lo, hi)
    return lo, hi


def owned_targets(tgt_off, tgt_ids, leaf_range):
    """Original target indices owned by a leaf range."""
    lo, hi = leaf_range
    return np.asarray(tgt_ids)[int(tgt_off[lo]):int(tgt_off[hi])]


def assemble(local_out, group=None):
    """Sums the ranks' outputs (non-owned entries are 0.0): exact assembly."""
    import torch
    import torch.distributed as dist
    t = local_out if isinstance(local_out, torch.Tensor) else torch.from_numpy(np.asarray(local_out))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t
