"""Body-slab partition of a multi-GPU Newton step, host-side restatement.

Implemented on the device (csrc/comm.cu `slab_partition`, csrc/k_broad.cu,
csrc/k_chol.cu `slab_pcg`); these functions restate it for the CPU / gloo tests.

One process per GPU.  Each step the dynamic bodies are sorted by position along
the longest axis of their positions (ties by body id) and cut into W contiguous
slabs balanced by primitive count (V + E + T per body); kinematic bodies are
replicated (owner -1).  Geometry is replicated on every GPU, only q / dq move.

  * a body pair (and every candidate row of it) belongs to the slab of its lower
    body, or of its higher body when the lower one is kinematic (`counted_rows`):
    pairs across a slab face are the halo pairs of exactly one rank, so the ranks'
    candidate sets are disjoint and their union is the single-GPU set;
  * that rank evaluates the pair's blocks, CCD query and energy; the partial
    systems are all-reduced, so every rank holds complete rows for its bodies;
  * the Newton system is solved by a distributed PCG: rows by slab, each rank's
    preconditioner the Cholesky of its slab block, the search direction's slab
    segments exchanged (a superset of the halo of `halo_bodies`), dot products,
    energies and the CCD bound all-reduced.
"""
from __future__ import annotations

import numpy as np

__all__ = ["slab_partition", "slab_owner_of_q", "halo_bodies", "owned_rows", "counted_rows", "dedup_union",
           "ordered_sum"]


def slab_partition(centroids, weights, dynamic, n_parts, axis=None):
    """owner[b] in [0, n_parts) for dynamic bodies, -1 (replicated) for kinematic.

    Dynamic bodies sorted by (centroid[axis], id); slab k takes those whose weight
    midpoint lies in [k/n, (k+1)/n) of the total, in integer arithmetic:
    owner = (2 cum - w) n // (2 total) (csrc/comm.cu slab_partition)."""
    c = np.asarray(centroids, dtype=float).reshape(-1, 3)
    w = np.rint(np.asarray(weights, dtype=float).reshape(-1)).astype(np.int64)
    dyn = np.asarray(dynamic, dtype=bool).reshape(-1)
    owner = np.full(len(c), -1, dtype=np.int64)
    idx = np.nonzero(dyn)[0]
    if len(idx) == 0 or n_parts <= 1:
        owner[idx] = 0
        return owner
    if axis is None:
        ext = c[idx].max(axis=0) - c[idx].min(axis=0)
        axis = int(np.argmax(ext))
    order = idx[np.lexsort((idx, c[idx, axis]))]
    cum = np.cumsum(w[order])
    total = int(cum[-1])
    if total <= 0:
        owner[order] = 0
        return owner
    owner[order] = np.minimum((2 * cum - w[order]) * n_parts // (2 * total), n_parts - 1)
    return owner


def slab_owner_of_q(q_all, prim_counts, dynamic, n_parts):
    """The device's partition of a state: centroids = body positions p = q[:, :3]."""
    return slab_partition(np.asarray(q_all, dtype=float).reshape(-1, 12)[:, :3], prim_counts, dynamic, n_parts)


def halo_bodies(overlap_pairs, owner, rank):
    """Bodies owned by other ranks that overlap (body boxes) an owned body."""
    ov = np.asarray(overlap_pairs, dtype=np.int64).reshape(-1, 2)
    oi, oj = owner[ov[:, 0]], owner[ov[:, 1]]
    h = set(ov[(oi == rank) & (oj != rank) & (oj >= 0), 1].tolist())
    h |= set(ov[(oj == rank) & (oi != rank) & (oi >= 0), 0].tolist())
    return np.array(sorted(h), dtype=np.int64)


def owned_rows(rows, owner, rank):
    """Candidate rows (body_a, prim_a, body_b, prim_b) with >= 1 body owned by `rank` (the
    rows whose blocks touch its rows of the system)."""
    r = np.asarray(rows, dtype=np.int64).reshape(-1, 4)
    return r[(owner[r[:, 0]] == rank) | (owner[r[:, 2]] == rank)]


def counted_rows(rows, owner, rank):
    """Rows of the body pairs `rank` evaluates: the slab of the lower body, or of the higher
    one when the lower is kinematic (exactly one rank per pair; k_prim_pairs2's rule)."""
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
