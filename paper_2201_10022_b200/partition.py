"""Partitioning for multi-GPU steps, host-side logic.

Implemented on the device (csrc/comm.cu, csrc/k_broad.cu): the per-pair work is
split by OVERLAP BODY PAIR -- the sorted overlap list is identical on every
rank and rank r takes pairs r, r + W, r + 2W, ... (`pair_owner` /
`rows_of_owned_pairs` restate it for the CPU tests); the system, energies and
CCD bound are all-reduced, the solve is replicated.  Every candidate belongs to
exactly one overlap pair, so the ranks' candidate sets are disjoint and their
union is the single-GPU set.

The body-slab helpers below are the alternative SURVEY §8(e) sketches (slab
ownership with halo bodies); they are kept for slab-sharded scenes.

One process per GPU.  Each step, dynamic bodies are sorted by centroid along
the longest scene axis and cut into contiguous slabs balanced by primitive
count; kinematic bodies (ground slabs, walls) are replicated.  Geometry is
replicated on every GPU so only q / dq cross ranks.

Per rank:
  * halo bodies  = bodies owned elsewhere whose swept box overlaps a box of an
                   owned body (from the body-pair overlap list);
  * owned pairs  = candidate rows with at least one owned body (a cross-slab
                   pair is evaluated on both owners, each keeps its own rows of
                   the gradient / BSR, so no reverse reduction is needed);
  * counted pairs = the subset whose scalar contribution (energy, counts) this
                   rank adds: owner of min(body_a, body_b), or of the dynamic
                   side when the other is kinematic — every pair exactly once;
  * scalars are combined in rank order after an all-gather so `e < e0`
    decisions are identical on every rank and for every world size.
"""
from __future__ import annotations

import numpy as np

__all__ = ["pair_owner", "rows_of_owned_pairs", "slab_partition", "halo_bodies", "owned_rows", "counted_rows",
           "dedup_union", "ordered_sum"]


def pair_owner(n_pairs, world):
    """Owning rank of each overlap pair (index order of the sorted overlap list)."""
    return np.arange(n_pairs, dtype=np.int64) % max(int(world), 1)


def rows_of_owned_pairs(rows, overlap_pairs, rank, world):
    """Candidate rows (body_a, prim_a, body_b, prim_b) whose overlap pair `rank` owns."""
    r = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
    ov = np.asarray(overlap_pairs, dtype=np.int64).reshape(-1, 2)
    owner = pair_owner(len(ov), world)
    index = {(int(a), int(b)): k for k, (a, b) in enumerate(ov)}
    keep = [owner[index[(min(int(x[0]), int(x[2])), max(int(x[0]), int(x[2])))]] == rank for x in r]
    return r[np.array(keep, dtype=bool)] if len(r) else r


def slab_partition(centroids, weights, dynamic, n_parts, axis=None):
    """owner[b] in [0, n_parts) for dynamic bodies, -1 (replicated) for kinematic."""
    c = np.asarray(centroids, dtype=float).reshape(-1, 3)
    w = np.asarray(weights, dtype=float).reshape(-1)
    dyn = np.asarray(dynamic, dtype=bool).reshape(-1)
    owner = np.full(len(c), -1, dtype=np.int64)
    idx = np.nonzero(dyn)[0]
    if len(idx) == 0 or n_parts <= 1:
        owner[idx] = 0
        return owner
    if axis is None:
        ext = c[idx].max(axis=0) - c[idx].min(axis=0)
        axis = int(np.argmax(ext))
    order = idx[np.lexsort((idx, c[idx, axis]))]  # stable, ties by body id
    cum = np.cumsum(w[order])
    total = cum[-1]
    # slab k takes bodies whose cumulative weight falls in (k/n, (k+1)/n]
    part = np.minimum((cum - 0.5 * w[order]) * n_parts // max(total, 1e-300), n_parts - 1).astype(np.int64)
    owner[order] = part
    return owner


def halo_bodies(overlap_pairs, owner, rank):
    """Bodies owned by other ranks that overlap (body boxes) an owned body."""
    ov = np.asarray(overlap_pairs, dtype=np.int64).reshape(-1, 2)
    oi, oj = owner[ov[:, 0]], owner[ov[:, 1]]
    h = set(ov[(oi == rank) & (oj != rank) & (oj >= 0), 1].tolist())
    h |= set(ov[(oj == rank) & (oi != rank) & (oi >= 0), 0].tolist())
    return np.array(sorted(h), dtype=np.int64)


def owned_rows(rows, owner, rank):
    """Candidate rows (body_a, prim_a, body_b, prim_b) with >= 1 body owned by `rank`."""
    r = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
    return r[(owner[r[:, 0]] == rank) | (owner[r[:, 2]] == rank)]


def counted_rows(rows, owner, rank):
    """Rows whose scalar contribution `rank` adds (exactly one rank per pair)."""
    r = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
    a, b = r[:, 0], r[:, 2]
    lo = np.minimum(a, b)
    hi = np.maximum(a, b)
    resp = np.where(owner[lo] >= 0, owner[lo], owner[hi])
    return r[resp == rank]


def dedup_union(per_rank_rows):
    """Deduplicated, canonically sorted (c0, c2, c1, c3) union of per-rank rows."""
    parts = [np.asarray(x, dtype=np.int64).reshape(-1, 4) for x in per_rank_rows]
    allr = np.concatenate(parts) if parts else np.zeros((0, 4), dtype=np.int64)
    if len(allr) == 0:
        return allr
    u = np.unique(allr, axis=0)
    return u[np.lexsort((u[:, 3], u[:, 1], u[:, 2], u[:, 0]))]


def ordered_sum(values_by_rank):
    """Sum of per-rank partial scalars in rank order (identical on all ranks)."""
    total = 0.0
    for v in values_by_rank:
        total += float(v)
    return total
