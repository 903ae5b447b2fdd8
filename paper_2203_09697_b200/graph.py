"""Cutoff graphs on the GPU: neighbour list, triplets, reverse edges, geometry.

``build_graph(system, cutoff)`` mirrors egn/graph.py:82-103 and returns the
same two containers (GraphTopology, Geometry) holding CUDA tensors; the
index arrays are bit-identical to the reference's (int64 at this API, int32
inside the kernels).  ``BatchGraph`` is the model's device-resident form of
a batch of graphs (disjoint union, graphs concatenated): it never
materialises per-triplet arrays -- triplets are implicit in the centre
tiles (see include/egn_b200.h).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops


@dataclass
class BatchGraph:
    """Device-resident topology + packed geometry of G concatenated graphs."""

    num_graphs: int
    num_nodes: int
    num_edges: int
    num_triplets: int
    cutoff: float
    pos: torch.Tensor  # f64 [V, 3]
    graph_ptr: torch.Tensor  # i64 [G+1]
    node_graph: torch.Tensor  # i32 [V]
    deg: torch.Tensor  # i32 [V]
    edge_ptr: torch.Tensor  # i64 [V+1]  CSR of out-edges by source
    src: torch.Tensor  # i32 [E]
    recv: torch.Tensor  # i32 [E]
    rev: torch.Tensor  # i32 [E]
    tri_ptr: torch.Tensor  # i64 [V+1]  triplet offsets per centre
    geo: torch.Tensor  # f32 [E, 4]  (ux, uy, uz, d)
    graph_sizes: list  # host: atoms per graph
    edge_counts: list | None = None  # host: edges per graph (lazily)
    max_deg: int = 0  # host: max out-degree (sizes the backward tile)
    # periodic batches: per-edge image index and shift ((x_recv - x_src)
    # + shift is the edge vector), per-graph cell / image ranges; None when non-periodic
    img: torch.Tensor | None = None  # i32 [E]
    shift: torch.Tensor | None = None  # f64 [E, 3]
    cell: torch.Tensor | None = None  # f64 [G, 3, 3]
    nimg: torch.Tensor | None = None  # i32 [G, 3]

    @property
    def device(self):
        return self.pos.device

    def edge_graph_ptr(self) -> torch.Tensor:
        return self.edge_ptr[self.graph_ptr]

    def update_positions(self, pos: torch.Tensor) -> None:
        """Copy new positions into this batch and recompute the packed geometry in
        place, keeping the topology (edges, triplets): a training pass over a fixed
        dataset (train_simple, egn/tasks.py:187-209) revisits the same graphs, so the
        neighbour list is built once per batch and its buffers stay valid for a
        captured step."""
        self.pos.copy_(pos, non_blocking=True)
        if self.shift is None:
            ops.call("egn_geometry", ops.ptr(self.pos), ops.ptr(self.src), ops.ptr(self.recv), self.num_edges,
                     ops.ptr(self.geo), None, None, ops.stream())
        else:
            ops.call("egn_geometry_shift", ops.ptr(self.pos), ops.ptr(self.src), ops.ptr(self.recv),
                     ops.ptr(self.shift), self.num_edges, ops.ptr(self.geo), None, None, ops.stream())


def _as_positions(systems) -> tuple[np.ndarray, list[int]]:
    if hasattr(systems, "positions") or (isinstance(systems, np.ndarray) and systems.ndim == 2):
        systems = [systems]
    pos = [np.asarray(s.positions if hasattr(s, "positions") else s, dtype=np.float64) for s in systems]
    return (np.concatenate(pos, axis=0) if pos else np.zeros((0, 3))), [p.shape[0] for p in pos]


def image_ranges(cell, pbc, cutoff: float, span=None) -> np.ndarray:
    """Images per axis that can hold a neighbour within the cutoff: max(ceil(r), floor(r +
    span_a)) with r = cutoff / h_a, h_a = |det C| / |c_b x c_c| the cell height normal to
    face a and span_a the extent of the atoms' fractional coordinates along a (< 1 when
    all atoms sit in one cell, where this is ceil(r)); 0 on non-periodic axes."""
    cell = np.asarray(cell, dtype=np.float64)
    vol = abs(np.linalg.det(cell))
    span = np.zeros(3) if span is None else np.asarray(span, dtype=np.float64)
    out = np.zeros(3, dtype=np.int32)
    for a in range(3):
        if pbc[a]:
            r = cutoff / (vol / np.linalg.norm(np.cross(cell[(a + 1) % 3], cell[(a + 2) % 3])))
            out[a] = max(int(np.ceil(r)), int(np.floor(r + span[a])))
    return out


def _frac_spans(pos: torch.Tensor, sizes, cells, pbc) -> np.ndarray:
    """Extent of the fractional coordinates of every periodic graph ([G, 3], one sync)."""
    g = len(sizes)
    spans = []
    off = 0
    for i in range(g):
        n = sizes[i]
        if n and bool(np.any(pbc[i])):
            inv = torch.from_numpy(np.linalg.inv(cells[i])).to(pos.device)
            frac = pos[off:off + n] @ inv
            spans.append(frac.max(dim=0).values - frac.min(dim=0).values)
        else:
            spans.append(torch.zeros(3, dtype=torch.float64, device=pos.device))
        off += n
    return torch.stack(spans).cpu().numpy() if spans else np.zeros((0, 3))


def _periodic_info(systems, g):
    """(cells [G,3,3], nimg-ready pbc [G,3]) when any system is periodic, else None."""
    if systems is None:
        return None
    if hasattr(systems, "positions"):
        systems = [systems]
    if not isinstance(systems, (list, tuple)) or not any(getattr(s, "periodic", False) for s in systems):
        return None
    cells = np.zeros((g, 3, 3))
    pbc = np.zeros((g, 3), dtype=bool)
    for i, s in enumerate(systems):
        if getattr(s, "periodic", False):
            cells[i] = s.cell
            pbc[i] = s.pbc
    return cells, pbc


def _cap(pos, graph_ptr, node_graph, deg, edge_ptr, src, recv, rev, img, shift, max_neighbors):
    """Keep the mutual max_neighbors-nearest edges (egn_cap_keep / egn_cap_compact)."""
    nv, ne = pos.shape[0], src.shape[0]
    dev = pos.device
    _, d64, _ = ops.geometry(pos, src, recv, want_fp64=True, shift=shift)
    keep1 = torch.empty(ne, dtype=torch.int32, device=dev)
    keep = torch.empty(ne, dtype=torch.int32, device=dev)
    ndeg = torch.empty(nv, dtype=torch.int32, device=dev)
    ops.call("egn_cap_keep", ops.ptr(edge_ptr), ops.ptr(d64), ops.ptr(rev), nv, int(max_neighbors), ops.ptr(keep1),
             ops.ptr(keep), ops.ptr(ndeg), ops.stream())
    nptr = ops.scan_counts(ndeg)
    ntri = ops.scan_counts(ndeg, square_minus_one=True)
    dmax = ndeg.max().to(torch.int64) if nv else nptr[-1]
    counts = torch.stack([nptr[-1], ntri[-1], dmax]).cpu()
    nne, nnt, nmax = int(counts[0]), int(counts[1]), int(counts[2])
    new_id = torch.empty(ne, dtype=torch.int32, device=dev)
    nsrc = torch.empty(nne, dtype=torch.int32, device=dev)
    nrecv = torch.empty(nne, dtype=torch.int32, device=dev)
    nimg = torch.empty(nne, dtype=torch.int32, device=dev) if img is not None else None
    nshift = torch.empty((nne, 3), dtype=torch.float64, device=dev) if shift is not None else None
    nrev = torch.empty(nne, dtype=torch.int32, device=dev)
    ops.call("egn_cap_compact", ops.ptr(edge_ptr), ops.ptr(nptr), nv, ne, ops.ptr(keep), ops.ptr(src), ops.ptr(recv),
             ops.ptr(img), ops.ptr(shift), ops.ptr(rev), ops.ptr(new_id), ops.ptr(nsrc), ops.ptr(nrecv),
             ops.ptr(nimg), ops.ptr(nshift), ops.ptr(nrev), ops.stream())
    return ndeg, nptr, ntri, nne, nnt, nmax, nsrc, nrecv, nrev, nimg, nshift


def build_batch(systems, cutoff: float, device="cuda", positions: torch.Tensor | None = None,
                sizes: list[int] | None = None, cells=None, pbc=None, max_neighbors: int | None = None) -> BatchGraph:
    """Build the batched device graph.  ``systems``: an AtomicSystem, a list of
    them, or raw (n,3) position arrays; alternatively pass device ``positions``
    (f64 [V,3]) and ``sizes`` directly (no host->device copy of positions).
    Periodic systems (AtomicSystem.cell / pbc, or ``cells`` [G,3,3] with ``pbc`` [G,3])
    get edges to every periodic image within the cutoff.  max_neighbors:
    keep an edge only if it is among the max_neighbors nearest of its source and its reverse
    is among those of its receiver (OC20-style cap, kept symmetric; ties by edge order)."""
    if cutoff <= 0:
        raise ValueError("cutoff must be positive")
    if positions is None:
        pos_np, sizes = _as_positions(systems)
        pos = torch.from_numpy(pos_np).to(device)
    else:
        pos = positions.to(torch.float64).contiguous()
        if sizes is None:
            sizes = [pos.shape[0]]
    dev = pos.device
    g = len(sizes)
    gp = np.zeros(g + 1, dtype=np.int64)
    gp[1:] = np.cumsum(sizes)
    graph_ptr = torch.from_numpy(gp).to(dev)
    node_graph = torch.from_numpy(np.repeat(np.arange(g, dtype=np.int32), sizes)).to(dev)
    per = None
    if cells is not None:
        per = (np.broadcast_to(np.asarray(cells, dtype=np.float64), (g, 3, 3)),
               np.broadcast_to(np.asarray(pbc if pbc is not None else True, dtype=bool), (g, 3)))
    else:
        per = _periodic_info(systems, g)
    if per is not None:
        cells_np, pbc_np = per
        spans = _frac_spans(pos, sizes, cells_np, pbc_np)
        nimg_np = np.stack([image_ranges(cells_np[i], pbc_np[i], cutoff, spans[i]) for i in range(g)]).astype(np.int32)
        cell_t = torch.from_numpy(np.ascontiguousarray(cells_np)).to(dev)
        nimg_t = torch.from_numpy(nimg_np).to(dev)
        deg = ops.neighbors_count_pbc(pos, graph_ptr, node_graph, cell_t, nimg_t, cutoff)
    else:
        deg = ops.neighbors_count(pos, graph_ptr, node_graph, cutoff)
    edge_ptr = ops.scan_counts(deg)
    tri_ptr = ops.scan_counts(deg, square_minus_one=True)
    dmax = deg.max().to(torch.int64) if pos.shape[0] else edge_ptr[-1]
    counts = torch.stack([edge_ptr[-1], tri_ptr[-1], dmax]).cpu()  # host sync 1: sizes
    ne, nt, max_deg = int(counts[0]), int(counts[1]), int(counts[2])
    img = shift = cell_keep = nimg_keep = None
    if per is not None:
        src, recv, img, shift = ops.neighbors_fill_pbc(pos, graph_ptr, node_graph, cell_t, nimg_t, cutoff, edge_ptr,
                                                       ne)
        rev, missing = ops.reverse_edges_pbc(edge_ptr, src, recv, img, node_graph, nimg_t)
        cell_keep, nimg_keep = cell_t, nimg_t
    else:
        src, recv = ops.neighbors_fill(pos, graph_ptr, node_graph, cutoff, edge_ptr, ne)
        rev, missing = ops.reverse_edges(edge_ptr, src, recv)
    # host sync 2: every edge must have its reverse (egn/graph.py:52-53 raises otherwise);
    # rev = -1 would index row -1 in every gather / scatter downstream
    if ne and int(missing.item()):
        bad = int(torch.nonzero(rev < 0)[0].item())
        raise ValueError(f"edge {bad} ({int(src[bad])} -> {int(recv[bad])}) has no reverse edge")
    if max_neighbors is not None:
        if max_neighbors < 0:
            raise ValueError("max_neighbors must be >= 0")
        if max_deg > max_neighbors:
            deg, edge_ptr, tri_ptr, ne, nt, max_deg, src, recv, rev, img, shift = _cap(
                pos, graph_ptr, node_graph, deg, edge_ptr, src, recv, rev, img, shift, max_neighbors)
    geo, _, _ = ops.geometry(pos, src, recv, shift=shift)
    return BatchGraph(g, int(pos.shape[0]), ne, nt, float(cutoff), pos, graph_ptr, node_graph, deg,
                      edge_ptr, src, recv, rev, tri_ptr, geo, list(sizes), max_deg=max_deg, img=img, shift=shift,
                      cell=cell_keep, nimg=nimg_keep)


# ---------------------------------------------------------------------------
# reference-shaped API (egn/graph.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class GraphTopology:
    """Directed edges and triplets (egn/graph.py:22-70), CUDA int64 tensors."""

    num_nodes: int
    edge_src: torch.Tensor
    edge_recv: torch.Tensor
    trip_in: torch.Tensor  # id3_kj
    trip_out: torch.Tensor  # id3_ji
    _rev: torch.Tensor | None = None

    @property
    def num_edges(self) -> int:
        return int(self.edge_src.shape[0])

    @property
    def num_triplets(self) -> int:
        return int(self.trip_in.shape[0])

    def reverse_edges(self) -> torch.Tensor:
        """rev with edges[rev[k]] == (recv_k, src_k); ValueError if some edge has no partner."""
        if self._rev is not None:
            return self._rev
        src = self.edge_src.to(torch.int32)
        recv = self.edge_recv.to(torch.int32)
        edge_ptr = ops.csr_ptr(self.edge_src, self.num_nodes)  # edges sorted by source
        rev, missing = ops.reverse_edges(edge_ptr, src, recv)
        if int(missing.item()):
            bad = int(torch.nonzero(rev < 0)[0].item())
            raise ValueError(f"edge {bad} has no reverse edge "
                             f"{(int(self.edge_recv[bad]), int(self.edge_src[bad]))}")
        return rev.to(torch.int64)

    def validate(self) -> None:
        s, r = self.edge_src, self.edge_recv
        if self.num_edges and bool(((s == r) | (s < 0) | (r >= self.num_nodes)).any()):
            raise ValueError("malformed edge list")
        if self.num_triplets:
            if bool(((self.trip_in >= self.num_edges) | (self.trip_out >= self.num_edges)).any()):
                raise ValueError("triplet references edge out of range")
            if bool((r[self.trip_in] != s[self.trip_out]).any()):
                raise ValueError("triplet edges do not share a middle atom")
            if bool((s[self.trip_in] == r[self.trip_out]).any()):
                raise ValueError("triplet with k == i")


@dataclass(frozen=True)
class Geometry:
    distances: torch.Tensor  # f64 [E]
    unit_vectors: torch.Tensor  # f64 [E, 3]
    angles: torch.Tensor  # f64 [N_t]


def build_graph(system, cutoff: float, device="cuda") -> tuple[GraphTopology, Geometry]:
    """Directed cutoff graph + geometry of one system (egn/graph.py:82-103)."""
    bg = build_batch(system, cutoff, device)
    return topology_of(bg), geometry_of(bg)


def topology_of(bg: BatchGraph) -> GraphTopology:
    kj, ji = ops.triplets_fill(bg.edge_ptr, bg.rev, bg.tri_ptr, bg.num_triplets)
    return GraphTopology(bg.num_nodes, bg.src.to(torch.int64), bg.recv.to(torch.int64), kj, ji,
                         bg.rev.to(torch.int64))


def geometry_of(bg: BatchGraph) -> Geometry:
    _, d64, u64 = ops.geometry(bg.pos, bg.src, bg.recv, want_fp64=True, shift=bg.shift)
    ang = ops.triplet_angles(bg.pos, bg.edge_ptr, bg.recv, bg.tri_ptr, bg.num_triplets, shift=bg.shift)
    return Geometry(d64, u64, ang)


def enumerate_triplets(num_nodes, edge_src=None, edge_recv=None):
    """((k->j),(j->i)) pairs with k != i sorted by (out, in) (egn/graph.py:106-139).

    Accepts (num_nodes, edge_src, edge_recv) or a GraphTopology; edges must be
    sorted by (src, recv) as build_graph produces them."""
    if isinstance(num_nodes, GraphTopology):
        t = num_nodes
        num_nodes, edge_src, edge_recv = t.num_nodes, t.edge_src, t.edge_recv
    edge_src = torch.as_tensor(edge_src, device="cuda")
    edge_recv = torch.as_tensor(edge_recv, device="cuda")
    if edge_src.numel() == 0:
        e = torch.empty(0, dtype=torch.int64, device="cuda")
        return e, e
    edge_ptr = ops.csr_ptr(edge_src.to(torch.int64), int(num_nodes))  # edges sorted by source
    deg = (edge_ptr[1:] - edge_ptr[:-1]).to(torch.int32)
    tri_ptr = ops.scan_counts(deg, square_minus_one=True)
    rev, missing = ops.reverse_edges(edge_ptr, edge_src.to(torch.int32), edge_recv.to(torch.int32))
    if int(missing.item()):
        raise ValueError("edge list is not symmetric; triplets are defined on cutoff graphs")
    return ops.triplets_fill(edge_ptr, rev, tri_ptr, int(tri_ptr[-1].item()))
