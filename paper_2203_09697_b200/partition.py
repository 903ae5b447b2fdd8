"""Edge/triplet/node partitions across graph-parallel ranks and the
analytic communication model.

``partition_graph`` / ``split_range`` / ``comm_volume`` keep the reference
interface and results (egn/partition.py:19-95): contiguous, +-1-balanced
shards of the sorted triplet, edge and node orders ("balanced" policy).

``partition_centers`` is the B200 policy used by the NCCL runtime
(runtime.py): ranks own contiguous ranges of centre atoms, hence their
out-edges (contiguous, edges are sorted by source) and whole triplet tiles
(contiguous, sorted by out-edge), balanced on the triplet count
sum_j deg_j (deg_j - 1).  Triplet aggregation is then rank-local, and the
per-block exchange is an all-gather of owned edge/node rows, whose size is
independent of the triplet count and dimension (criterion of PAPER.md
section 3 / egn/partition.py:85-95).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import GEMNET, ModelConfig


@dataclass(frozen=True)
class GraphPartition:
    workers: int
    triplet_shards: list
    edge_shards: list
    node_shards: list
    topology: object


def split_range(n: int, workers: int) -> list[np.ndarray]:
    """Contiguous index ranges whose sizes differ by at most one (partition.py:28-37)."""
    base, extra = divmod(n, workers)
    out, start = [], 0
    for p in range(workers):
        size = base + (1 if p < extra else 0)
        out.append(np.arange(start, start + size, dtype=np.int64))
        start += size
    return out


def partition_graph(topology, workers: int) -> GraphPartition:
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return GraphPartition(workers, split_range(topology.num_triplets, workers),
                          split_range(topology.num_edges, workers),
                          split_range(topology.num_nodes, workers), topology)


@dataclass(frozen=True)
class CenterPartition:
    """Per-rank ranges: centres [node_lo, node_hi), edges [edge_lo, edge_hi),
    triplets [trip_lo, trip_hi) -- all contiguous."""

    workers: int
    node_bounds: np.ndarray  # [P+1]
    edge_bounds: np.ndarray  # [P+1]
    trip_bounds: np.ndarray  # [P+1]

    def rank(self, r: int):
        return (int(self.node_bounds[r]), int(self.node_bounds[r + 1]),
                int(self.edge_bounds[r]), int(self.edge_bounds[r + 1]),
                int(self.trip_bounds[r]), int(self.trip_bounds[r + 1]))


def partition_centers(deg: np.ndarray, workers: int, weight: str = "triplets",
                      candidates: np.ndarray | None = None) -> CenterPartition:
    """Split centre atoms into contiguous ranges balancing sum deg(deg-1) (+ edges).

    The cost of a centre is its triplet count plus its out-edge count (the
    per-edge dense work), so edge-heavy but triplet-light graphs still
    balance.  ``candidates`` (e.g. the graph offsets of a batch) restricts the
    split points; a partition aligned to graph boundaries has no cross-rank
    edges, so its edge/node exchanges are empty."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    deg = np.asarray(deg, dtype=np.int64)
    n = deg.shape[0]
    edge_ptr = np.zeros(n + 1, dtype=np.int64)
    edge_ptr[1:] = np.cumsum(deg)
    tri_ptr = np.zeros(n + 1, dtype=np.int64)
    tri_ptr[1:] = np.cumsum(deg * (deg - 1))
    cost = deg * (deg - 1) + deg if weight == "triplets" else deg
    cum = np.concatenate([[0], np.cumsum(cost)])
    total = cum[-1]
    bounds = np.zeros(workers + 1, dtype=np.int64)
    cand = None if candidates is None else np.unique(np.asarray(candidates, dtype=np.int64))
    for r in range(1, workers):
        target = total * r / workers
        if cand is None:
            bounds[r] = int(np.searchsorted(cum, target, side="left"))
        else:
            bounds[r] = int(cand[np.argmin(np.abs(cum[cand] - target))])
        bounds[r] = max(bounds[r], bounds[r - 1])
    bounds[workers] = n
    bounds = np.minimum(bounds, n)
    return CenterPartition(workers, bounds, edge_ptr[bounds], tri_ptr[bounds])


@dataclass(frozen=True)
class ReferencePartition:
    """The reference's balanced shards (egn/partition.py:28-49: split_range of the sorted
    triplet, edge and node orders) for the graph-parallel reference schedule, plus the centre
    range that covers each rank's triplet shard and the window into its first / last centre
    (egn_triplet_fwd_window: a shard may cut through a centre's tile)."""

    workers: int
    trip_bounds: np.ndarray  # [P+1]
    edge_bounds: np.ndarray  # [P+1]
    node_bounds: np.ndarray  # [P+1]
    centre_lo: np.ndarray  # [P] first centre of the triplet shard
    centre_hi: np.ndarray  # [P] one past the last centre
    first_lo: np.ndarray  # [P] centre-local triplet index where the shard starts (first centre)
    last_hi: np.ndarray  # [P] centre-local index where it ends (last centre)

    def triplet_shards(self) -> list:
        return [np.arange(a, b, dtype=np.int64) for a, b in zip(self.trip_bounds[:-1], self.trip_bounds[1:])]


def _bounds(n: int, workers: int) -> np.ndarray:
    sizes = [s.size for s in split_range(n, workers)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def partition_reference(tri_ptr: np.ndarray, num_edges: int, num_nodes: int, workers: int) -> ReferencePartition:
    """split_range shards (identical to partition_graph) and the centre windows of the triplet
    shards; tri_ptr [V+1] = triplet offsets per centre (sorted (out, in) order)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    tri_ptr = np.asarray(tri_ptr, dtype=np.int64)
    nt = int(tri_ptr[-1]) if tri_ptr.size else 0
    tb = _bounds(nt, workers)
    lo = np.zeros(workers, dtype=np.int64)
    hi = np.zeros(workers, dtype=np.int64)
    flo = np.zeros(workers, dtype=np.int64)
    lhi = np.zeros(workers, dtype=np.int64)
    for r in range(workers):
        t0, t1 = int(tb[r]), int(tb[r + 1])
        if t1 <= t0:
            continue
        jlo = int(np.searchsorted(tri_ptr, t0, side="right")) - 1
        jhi = int(np.searchsorted(tri_ptr, t1 - 1, side="right")) - 1
        lo[r], hi[r] = jlo, jhi + 1
        flo[r], lhi[r] = t0 - tri_ptr[jlo], t1 - tri_ptr[jhi]
    return ReferencePartition(workers, tb, _bounds(int(num_edges), workers), _bounds(int(num_nodes), workers),
                              lo, hi, flo, lhi)


@dataclass(frozen=True)
class CommModel:
    n_v: int
    n_e: int
    n_t: int
    d_v: int
    d_e: int
    d_t: int
    d_u: int
    variant: str

    @classmethod
    def from_graph(cls, topology, config: ModelConfig) -> "CommModel":
        return cls(topology.num_nodes, topology.num_edges, topology.num_triplets, config.d_v,
                   config.d_e, config.d_t, config.d_u, config.variant)


@dataclass(frozen=True)
class CommVolume:
    per_block: int
    total: int


def comm_volume(model: CommModel, blocks: int) -> CommVolume:
    """Forward elements exchanged per block: N_e d_e + N_v d_v + d_u (+ N_e d_e for gemnet)."""
    per_block = model.n_e * model.d_e + model.n_v * model.d_v + model.d_u
    if model.variant == GEMNET:
        per_block += model.n_e * model.d_e
    return CommVolume(per_block, blocks * per_block)
