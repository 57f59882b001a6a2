"""Multi-GPU layout of the hot path.

The volume update and the wall-distance/compaction pass are independent per
volume node, so N ranks (one process per GPU) take contiguous node ranges and
need no data-path collective: each rank runs the whole per-level pipeline on
its shard against a replicated control set (<= 5000 controls, 240 KB).  The
only collectives are the benchmark's barrier and the max-over-ranks device
time; an optional gather reassembles the sparse update in ascending node order
(wall_distance.hpp:36-38), which works because the shards are contiguous and
ordered by rank.

The greedy selection is NOT sharded here: its factorisation is a sequential
chain (rbf.cpp:114-120) and the per-step exchange would be a 16-byte
(norm, index) max-reduction, far too small for a collective to pay.  Ranks
that need the control set run it redundantly ("replicas only") or receive it
from rank 0 by broadcast.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n units for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank/world")
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi


def merge_sparse_updates(parts):
    """Concatenate per-rank (global_node_ids, values) in rank order; the result
    is ascending because shards are contiguous and ranked."""
    idx = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.int64)
    val = np.concatenate([p[1] for p in parts]) if parts else np.zeros((0, 3))
    return idx, val


def sharded_update_volume(update_fn, nodes, dist, rank, world, gather=None, **kw):
    """Run `update_fn(nodes_shard, dist_shard, **kw) -> (idx, val)` on this
    rank's shard and return global (idx, val); with `gather` (e.g.
    torch.distributed.all_gather_object) the full update is returned on every
    rank."""
    lo, hi = shard_range(len(nodes), rank, world)
    idx, val = update_fn(nodes[lo:hi], dist[lo:hi], **kw)
    mine = (np.asarray(idx, dtype=np.int64) + lo, np.asarray(val))
    if gather is None:
        return mine
    parts = [None] * world
    gather(parts, mine)
    return merge_sparse_updates(parts)
