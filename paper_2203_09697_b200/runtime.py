"""Graph-parallel execution: one rank per GPU (torch.distributed / NCCL), or P
in-process ranks on one device (threads) for testing and the WorkerGroup API.

Reference: egn/runtime.py (Collective :131-200, WorkerGroup :265-683).  The
reference shards triplets/edges/nodes with contiguous +-1-balanced ranges and
all-reduces zero-padded full buffers after every stage.  Here ranks own
contiguous ranges of CENTRE atoms (partition.partition_centers): their
out-edges (contiguous, edges are sorted by source) and their complete triplet
tiles, so the triplet aggregation (TA) never crosses a rank.  Per block:

  forward                                   exchange (this module)
  X = m W_down^T [A^T]   all rows (redundant, m replicated)
  S, TU, EU              own edges
  m_new                  -> all-gather rows            (edge,  N_e d_e)
  EA + NU                own nodes (in-edges read from the gathered m_new)
  gemnet: v              -> all-gather rows            (node,  N_v d_v)
          EU2 own edges, m2 -> all-gather rows         (edge,  N_e d_e)
          sym            all rows (redundant)
  GU head: per-graph node sums of own nodes -> all-reduce (global, G d_v)

Forward volume per block: N_e d_e + G d_v (dimenet) and 2 N_e d_e + N_v d_v
+ G d_v (gemnet) -- independent of N_t and d_t (sec. 3; compare
egn/partition.py:85-95).  The backward is the adjoint: every all-gather
becomes a reduce-scatter of partial row adjoints; parameter and position
gradients are all-reduced once at the end (egn/runtime.py:674-676).
Quantities computed redundantly from replicated inputs with replicated
adjoints (the per-graph GU/energy tail) contribute their parameter
gradients on rank 0 only, so the final sum counts them once.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from . import ops
from .config import GEMNET
from .engine import DeviceWeights, ForwardResult, _silu_bwd
from .graph import BatchGraph
from .partition import CenterPartition, partition_centers

ALLOWED_LEVELS = frozenset({"edge", "node", "global", "position", "param", "replica"})


class CollectiveError(RuntimeError):
    pass


class CollectiveShapeError(CollectiveError):
    pass


class CollectiveTimeoutError(CollectiveError):
    pass


class WorkerGroupError(RuntimeError):
    def __init__(self, stage: str, rank: int, cause: BaseException):
        super().__init__(f"worker {rank} failed during stage {stage!r}: {cause!r}")
        self.stage = stage
        self.rank = rank


@dataclass(frozen=True)
class CommRecord:
    phase: str
    block: int
    stage: str
    level: str
    elements: int
    op: str = "all_reduce"


@dataclass
class CommLog:
    """Collective accounting (egn/runtime.py:89-128); bytes = elements * 4 (fp32)."""

    records: list = field(default_factory=list)

    def elements(self, phase=None, block=None) -> int:
        return sum(r.elements for r in self.records
                   if (phase is None or r.phase == phase) and (block is None or r.block == block))

    def forward_blocks(self) -> dict:
        out: dict = {}
        for r in self.records:
            if r.phase == "forward" and r.block >= 0:
                out[r.block] = out.get(r.block, 0) + r.elements
        return out

    def levels(self) -> set:
        return {r.level for r in self.records}

    def to_csv_rows(self) -> list:
        rows = ["phase,block,stage,level,op,elements,bytes"]
        rows += [f"{r.phase},{r.block},{r.stage},{r.level},{r.op},{r.elements},{r.elements * 4}" for r in self.records]
        return rows


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class Comm:
    """Row-range collectives over P ranks; rank r owns rows [bounds[r], bounds[r+1])."""

    def __init__(self, rank: int, world: int, log: CommLog | None = None):
        self.rank, self.world = rank, world
        self.log = log if log is not None else CommLog()

    def _tag(self, t: torch.Tensor, op: str, phase="forward", block=-1, stage="", level="edge"):
        if level not in ALLOWED_LEVELS:
            raise ValueError(f"buffers of level {level!r} must never enter a collective")
        if self.rank == 0:
            self.log.records.append(CommRecord(phase, block, stage, level, int(t.numel()), op))

    # subclasses implement the three primitives
    def all_reduce_(self, t, **tag):  # pragma: no cover - interface
        raise NotImplementedError

    def all_gather_rows(self, full, bounds, **tag):  # pragma: no cover - interface
        raise NotImplementedError

    def reduce_scatter_rows(self, full, bounds, **tag):  # pragma: no cover - interface
        raise NotImplementedError


class LocalComm(Comm):
    """P = 1: every collective is the identity (still logged)."""

    def __init__(self, log=None):
        super().__init__(0, 1, log)

    def all_reduce_(self, t, **tag):
        self._tag(t, "all_reduce", **tag)
        return t

    def all_gather_rows(self, full, bounds, **tag):
        self._tag(full, "all_gather", **tag)
        return full

    def reduce_scatter_rows(self, full, bounds, **tag):
        self._tag(full, "reduce_scatter", **tag)
        return full[int(bounds[0]):int(bounds[1])]


def gp_dp_layout(world: int, gp: int) -> tuple[list, list]:
    """GP x DP composition (pkg/README.md "Scaling notes"): `world` ranks
    as world / gp data-parallel replicas of `gp` graph-parallel workers.  Replica k owns ranks
    [k gp, (k + 1) gp); the DP group of worker index i is {i, i + gp, i + 2 gp, ...}.
    Returns (gp_groups, dp_groups) as rank lists."""
    if gp < 1 or world % gp:
        raise ValueError(f"world size {world} is not a multiple of the graph-parallel size {gp}")
    gp_groups = [list(range(k * gp, (k + 1) * gp)) for k in range(world // gp)]
    dp_groups = [list(range(i, world, gp)) for i in range(gp)]
    return gp_groups, dp_groups


class DistComm(Comm):
    """torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    @classmethod
    def gp_dp(cls, gp: int, log=None) -> tuple["DistComm", "DistComm"]:
        """This rank's (graph-parallel, data-parallel) communicators of gp_dp_layout; every rank
        must call it (torch.distributed.new_group is collective)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        gp_groups, dp_groups = gp_dp_layout(world, gp)
        mine_gp = mine_dp = None
        for ranks in gp_groups:
            g = dist.new_group(ranks)
            if rank in ranks:
                mine_gp = g
        for ranks in dp_groups:
            g = dist.new_group(ranks)
            if rank in ranks:
                mine_dp = g
        return cls(mine_gp, log), cls(mine_dp, log)

    def __init__(self, group=None, log=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        super().__init__(dist.get_rank(group), dist.get_world_size(group), log)
        self.backend = dist.get_backend(group)

    def all_reduce_(self, t, **tag):
        self._tag(t, "all_reduce", **tag)
        self.dist.all_reduce(t, group=self.group)
        return t

    def _padded(self, full, bounds):
        rows = np.diff(np.asarray(bounds))
        mr = int(rows.max()) if rows.size else 0
        return rows, mr

    def all_gather_rows(self, full, bounds, **tag):
        self._tag(full, "all_gather", **tag)
        rows, mr = self._padded(full, bounds)
        if mr == 0:
            return full
        lo, hi = int(bounds[self.rank]), int(bounds[self.rank + 1])
        send = torch.zeros((mr,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        send[: hi - lo] = full[lo:hi]
        if self.backend == "nccl":
            recv = torch.empty((self.world * mr,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
            self.dist.all_gather_into_tensor(recv, send, group=self.group)
            chunks = recv.view(self.world, mr, *full.shape[1:])
        else:
            lst = [torch.empty_like(send) for _ in range(self.world)]
            self.dist.all_gather(lst, send, group=self.group)
            chunks = lst
        for r in range(self.world):
            a, b = int(bounds[r]), int(bounds[r + 1])
            if r != self.rank and b > a:
                full[a:b] = chunks[r][: b - a]
        return full

    def reduce_scatter_rows(self, full, bounds, **tag):
        self._tag(full, "reduce_scatter", **tag)
        rows, mr = self._padded(full, bounds)
        lo, hi = int(bounds[self.rank]), int(bounds[self.rank + 1])
        if self.backend != "nccl" or mr == 0:
            self.dist.all_reduce(full, group=self.group)
            return full[lo:hi]
        send = torch.zeros((self.world * mr,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        sv = send.view(self.world, mr, *full.shape[1:])
        for r in range(self.world):
            a, b = int(bounds[r]), int(bounds[r + 1])
            if b > a:
                sv[r, : b - a] = full[a:b]
        out = torch.empty((mr,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
        self.dist.reduce_scatter_tensor(out, send, group=self.group)
        full[lo:hi] = out[: hi - lo]
        return full[lo:hi]


class _ThreadShared:
    def __init__(self, world: int, timeout: float, fault: str | None):
        self.world = world
        self.timeout = timeout
        self.fault = fault
        self.slots: list = [None] * world
        self.enter = threading.Barrier(world)
        self.exit = threading.Barrier(world)

    def abort(self):
        self.enter.abort()
        self.exit.abort()

    def wait(self, barrier):
        try:
            barrier.wait(timeout=self.timeout)
        except threading.BrokenBarrierError:
            raise CollectiveTimeoutError(
                f"collective did not complete within {self.timeout}s (missing participant or aborted group)"
            ) from None


class ThreadComm(Comm):
    """P ranks as threads of one process on one device (the reference's
    execution model, egn/runtime.py:131-200): rank-ordered sums, identical
    results on every rank.  All ranks share torch's current stream, so the
    host barrier orders the device work."""

    def __init__(self, rank: int, shared: _ThreadShared, log: CommLog):
        super().__init__(rank, shared.world, log)
        self.sh = shared

    def _exchange(self, t):
        self.sh.slots[self.rank] = t
        self.sh.wait(self.sh.enter)
        shapes = {tuple(s.shape) for s in self.sh.slots}
        if len(shapes) != 1:
            raise CollectiveShapeError(f"shape mismatch across workers: {sorted(shapes)}")
        return list(self.sh.slots)

    def _done(self):
        self.sh.wait(self.sh.exit)

    def all_reduce_(self, t, **tag):
        self._tag(t, "all_reduce", **tag)
        slots = self._exchange(t)
        last = self.world - 1 if self.sh.fault == "drop-last" and self.world > 1 else None
        total = slots[0].clone()
        for r in range(1, self.world):
            if r != last:
                total += slots[r]
        self._done()
        t.copy_(total)
        return t

    def all_gather_rows(self, full, bounds, **tag):
        self._tag(full, "all_gather", **tag)
        slots = self._exchange(full)
        pieces = [(int(bounds[r]), int(bounds[r + 1]), slots[r][int(bounds[r]):int(bounds[r + 1])].clone())
                  for r in range(self.world) if r != self.rank]
        self._done()
        for a, b, p in pieces:
            full[a:b] = p
        return full

    def reduce_scatter_rows(self, full, bounds, **tag):
        self._tag(full, "reduce_scatter", **tag)
        slots = self._exchange(full)
        lo, hi = int(bounds[self.rank]), int(bounds[self.rank + 1])
        total = slots[0][lo:hi].clone()
        for r in range(1, self.world):
            total += slots[r][lo:hi]
        self._done()
        full[lo:hi] = total
        return full[lo:hi]


# ---------------------------------------------------------------------------
# graph-parallel engine (one rank)
# ---------------------------------------------------------------------------
class GraphParallelEngine:
    """Forward/backward of one rank's centre shard; P = 1 reproduces Engine.

    When no edge crosses a rank boundary (a partition aligned to graph
    boundaries of a batch: the "halo" is empty) the edge/node exchanges are
    skipped and the redundant all-row products are restricted to the owned
    rows; only the per-graph GU sums, the loss and the gradients are reduced
    (graph parallelism degenerates to data parallelism over whole graphs)."""

    def __init__(self, weights: DeviceWeights, comm: Comm, part: CenterPartition):
        self.weights, self.comm, self.part = weights, comm, part
        self.config = weights.config
        r = comm.rank
        self.n0, self.n1, self.e0, self.e1, self.t0, self.t1 = part.rank(r)
        self._halo = {}

    def halo_free(self, bg: BatchGraph) -> bool:
        key = id(bg)
        if key not in self._halo:
            rv = bg.rev[self.e0:self.e1]
            local = bool(((rv >= self.e0) & (rv < self.e1)).all()) if self.e1 > self.e0 else True
            flag = torch.tensor([0.0 if local else 1.0], device=bg.device)
            self.comm.all_reduce_(flag, phase="setup", block=-1, stage="halo", level="global")
            self._halo = {key: bool(flag.item() == 0.0)}
        return self._halo[key]

    def _slices(self, bg: BatchGraph):
        n0, n1 = self.n0, self.n1
        ep_own = bg.edge_ptr[n0:n1 + 1]
        gp_own = (bg.graph_ptr.clamp(n0, n1) - n0).contiguous()
        return ep_own, gp_own

    def _sbf_weight(self, b):
        c, w = self.config, self.weights.w
        p = f"block{b}.tu."
        wp = w[p + "sbf_gate"]
        if c.variant == GEMNET:
            wp = w[p + "bilinear_b"] @ wp
        return wp.view(wp.shape[0], c.k_rbf, c.l_sbf).permute(1, 2, 0).contiguous()

    def forward(self, bg: BatchGraph) -> ForwardResult:
        c, w, cm = self.config, self.weights.w, self.comm
        gem = c.variant == GEMNET
        e0, e1, n0, n1 = self.e0, self.e1, self.n0, self.n1
        eb, nb = self.part.edge_bounds, self.part.node_bounds
        hf = self.halo_free(bg)
        lo, hi = (e0, e1) if hf else (0, bg.num_edges)  # rows of the redundant products
        ep_own, gp_own = self._slices(bg)
        E, V, dev = bg.num_edges, bg.num_nodes, bg.device
        rbf = ops.rbf(bg.geo, c.k_rbf, c.cutoff)
        m = torch.zeros((E, c.d_e), dtype=torch.float32, device=dev)
        torch.addmm(w["edge_init.b"], rbf[lo:hi], w["edge_init.w"].t(), out=m[lo:hi])
        u = torch.zeros((bg.num_graphs, c.d_u), dtype=torch.float32, device=dev)
        blocks, v_own = [], None
        dg = c.triplet_width
        for b in range(c.blocks):
            p = f"block{b}."
            st = {"m": m}
            down = torch.zeros((E, c.d_t), dtype=torch.float32, device=dev)
            torch.mm(m[lo:hi], w[p + "tu.down"].t(), out=down[lo:hi])
            if gem:
                X = torch.zeros((E, dg), dtype=torch.float32, device=dev)
                torch.mm(down[lo:hi], w[p + "tu.bilinear_a"].t(), out=X[lo:hi])
            else:
                X = down
            Wk = self._sbf_weight(b)
            S = torch.zeros_like(X)
            if n1 > n0:
                _triplet_fwd_into(ep_own, bg, X, Wk, c.cutoff, S)
            S_o = S[e0:e1]
            g = rbf[e0:e1] @ w[p + "tu.rbf_gate"].t()
            if gem:
                Z = S_o @ w[p + "tu.bilinear_proj"].t()
                Y = Z * g
                st["Z"] = Z
            else:
                Y = S_o * g
            ta = Y @ w[p + "tu.up"].t()
            m_o = m[e0:e1]
            xcat = torch.cat([m_o, ta], dim=1)
            h = torch.addmm(w[p + "eu.b1"], xcat, w[p + "eu.w1"].t())
            a1 = F.silu(h)
            m_new = torch.zeros((E, c.d_e), dtype=torch.float32, device=dev)
            torch.addmm(w[p + "eu.b2"], a1, w[p + "eu.w2"].t(), out=m_new[e0:e1])
            m_new[e0:e1] += m_o
            if not hf:
                cm.all_gather_rows(m_new, eb, phase="forward", block=b, stage="m_new", level="edge")
            agg = ops.aggregate_in_edges(ep_own, bg.rev, m_new)
            hv = torch.addmm(w[p + "nu.b1"], agg, w[p + "nu.w1"].t())
            av = F.silu(hv)
            v_own = torch.addmm(w[p + "nu.b2"], av, w[p + "nu.w2"].t())
            st.update(down=down, X=X, Wk=Wk, S=S, g=g, Y=Y, xcat=xcat, h=h, a1=a1, m_new=m_new, agg=agg, hv=hv,
                      av=av, v_own=v_own)
            if gem:
                v_full = torch.zeros((V, c.d_v), dtype=torch.float32, device=dev)
                v_full[n0:n1] = v_own
                if not hf:
                    cm.all_gather_rows(v_full, nb, phase="forward", block=b, stage="v", level="node")
                w1 = w[p + "eu2.w1"]
                pv = v_full @ w1[:, c.d_e:].t()
                h2 = torch.addmm(w[p + "eu2.b1"], m_new[e0:e1], w1[:, :c.d_e].t())
                ops.gather_rows(bg.recv[e0:e1], pv, out=h2, accumulate=True)
                a2 = F.silu(h2)
                m2 = torch.zeros((E, c.d_e), dtype=torch.float32, device=dev)
                torch.addmm(w[p + "eu2.b2"], a2, w[p + "eu2.w2"].t(), out=m2[e0:e1])
                m2[e0:e1] += m_new[e0:e1]
                if not hf:
                    cm.all_gather_rows(m2, eb, phase="forward", block=b, stage="m2", level="edge")
                m2r = torch.zeros_like(m2)
                ops.gather_rows(bg.rev[lo:hi], m2, out=m2r[lo:hi])
                m = torch.zeros_like(m2)
                torch.addmm(m2[lo:hi], m2r[lo:hi], w[p + "sym.w"].t(), out=m[lo:hi])
                st.update(v_full=v_full, h2=h2, a2=a2, m2r=m2r)
            else:
                m = m_new
            s = ops.graph_sum(gp_own, v_own) if n1 > n0 else torch.zeros((bg.num_graphs, c.d_v), device=dev)
            cm.all_reduce_(s, phase="forward", block=b, stage="gu", level="global")
            pre = torch.addmm(w[p + "gu.b1"], s, w[p + "gu.w1"].t())
            act = F.silu(pre)
            u = torch.addmm(w[p + "gu.b2"], act, w[p + "gu.w2"].t()).add_(u)
            st.update(s=s, pre=pre, act=act)
            blocks.append(st)
        energy = torch.addmm(w["energy_head.b"], u, w["energy_head.w"].t()).view(-1)
        forces = scale = None
        if gem:
            scale, forces = ops.force_head_fwd(ep_own, bg.rev, bg.geo, m, w["force_head.w"].view(-1))
        return ForwardResult(energy, forces, m, v_own, u, rbf, blocks, scale)

    def backward(self, bg: BatchGraph, fw: ForwardResult, d_energy: torch.Tensor,
                 d_forces_own: torch.Tensor | None = None) -> torch.Tensor:
        """Sets weights.grad_flat to the all-reduced dL/dW; returns the all-reduced dL/dx (f64 [V,3])."""
        c, w, gr, cm = self.config, self.weights.w, self.weights.g, self.comm
        gem = c.variant == GEMNET
        de = c.d_e
        e0, e1, n0, n1 = self.e0, self.e1, self.n0, self.n1
        eb, nb = self.part.edge_bounds, self.part.node_bounds
        hf = self.halo_free(bg)
        lo, hi = (e0, e1) if hf else (0, bg.num_edges)
        ep_own, gp_own = self._slices(bg)
        E, V, dev = bg.num_edges, bg.num_nodes, bg.device
        lead = cm.rank == 0
        wg, cs = ops.wgrad, ops.column_sum
        self.weights.grad_flat.zero_()
        eg = torch.zeros((E, 4), dtype=torch.float32, device=dev)
        dE = d_energy.to(torch.float32).view(-1, 1)
        if lead:
            torch.mm(dE.t(), fw.u, out=gr["energy_head.w"])
            gr["energy_head.b"].copy_(dE.sum(0))
        u_bar = dE @ w["energy_head.w"]
        m_bar = torch.zeros((E, de), dtype=torch.float32, device=dev)  # partial adjoint
        if gem and d_forces_own is not None:
            f_bar = torch.zeros((V, 3), dtype=torch.float32, device=dev)
            f_bar[n0:n1] = d_forces_own.to(torch.float32)
            ops.force_head_bwd(bg.recv, bg.geo, fw.m, w["force_head.w"].view(-1), fw.scale, f_bar, m_bar, eg,
                               w_bar=gr["force_head.w"].view(-1))
        rbf_bar = torch.zeros_like(fw.rbf)
        for b in range(c.blocks - 1, -1, -1):
            p = f"block{b}."
            st = fw.blocks[b]
            # GU (replicated): parameter grads from rank 0 only
            pre_bar = _silu_bwd(u_bar @ w[p + "gu.w2"], st["pre"])
            if lead:
                torch.mm(u_bar.t(), st["act"], out=gr[p + "gu.w2"])
                gr[p + "gu.b2"].copy_(u_bar.sum(0))
                gr[p + "gu.b1"].copy_(pre_bar.sum(0))
                torch.mm(pre_bar.t(), st["s"], out=gr[p + "gu.w1"])
            s_bar = pre_bar @ w[p + "gu.w1"]
            v_bar = ops.gather_rows(bg.node_graph[n0:n1], s_bar)
            if gem:
                # sym (rows lo:hi) and its adjoint
                wg(m_bar[lo:hi], st["m2r"][lo:hi], out=gr[p + "sym.w"])
                t = m_bar[lo:hi] @ w[p + "sym.w"]
                m2_bar = m_bar.clone()
                ops.scatter_rows(bg.rev[lo:hi], torch.arange(hi - lo, dtype=torch.int32, device=dev), t, m2_bar)
                if hf:
                    m2_bar_o = m2_bar[e0:e1]
                else:
                    m2_bar_o = cm.reduce_scatter_rows(m2_bar, eb, phase="backward", block=b, stage="m2",
                                                      level="edge")
                wg(m2_bar_o, st["a2"], out=gr[p + "eu2.w2"])
                cs(m2_bar_o, out=gr[p + "eu2.b2"])
                h2_bar = _silu_bwd(m2_bar_o @ w[p + "eu2.w2"], st["h2"])
                cs(h2_bar, out=gr[p + "eu2.b1"])
                w1 = w[p + "eu2.w1"]
                gr[p + "eu2.w1"][:, :de].copy_(wg(h2_bar, st["m_new"][e0:e1]))
                h2_full = torch.zeros((E, de), dtype=torch.float32, device=dev)
                h2_full[e0:e1] = h2_bar
                if hf:
                    pv_bar = ops.aggregate_in_edges(ep_own, bg.rev, h2_full)  # own nodes, complete
                    gr[p + "eu2.w1"][:, de:].copy_(pv_bar.t() @ st["v_own"])
                    v_bar = v_bar + pv_bar @ w1[:, de:]
                else:
                    pv_bar = ops.aggregate_in_edges(bg.edge_ptr, bg.rev, h2_full)  # all nodes, partial
                    gr[p + "eu2.w1"][:, de:].copy_(pv_bar.t() @ st["v_full"])
                    v_bar_full = pv_bar @ w1[:, de:]
                    v_bar = v_bar + cm.reduce_scatter_rows(v_bar_full, nb, phase="backward", block=b, stage="v",
                                                           level="node")
                mnb = torch.zeros((E, de), dtype=torch.float32, device=dev)
                torch.addmm(m2_bar_o, h2_bar, w1[:, :de], out=mnb[e0:e1])
            else:
                mnb = m_bar
            # NU (own nodes)
            wg(v_bar, st["av"], out=gr[p + "nu.w2"])
            cs(v_bar, out=gr[p + "nu.b2"])
            hv_bar = _silu_bwd(v_bar @ w[p + "nu.w2"], st["hv"])
            cs(hv_bar, out=gr[p + "nu.b1"])
            wg(hv_bar, st["agg"], out=gr[p + "nu.w1"])
            agg_bar = hv_bar @ w[p + "nu.w1"]
            # in-edges of own nodes are rev(own edges): rows rev[e] += agg_bar[src(e) - n0]
            if e1 > e0:
                src_local = (bg.src[e0:e1] - n0).to(torch.int32)
                ops.scatter_rows(bg.rev[e0:e1], src_local, agg_bar, mnb, accumulate=True)
            if hf:
                m_new_bar = mnb[e0:e1]
            else:
                m_new_bar = cm.reduce_scatter_rows(mnb, eb, phase="backward", block=b, stage="m_new", level="edge")
            # EU (own edges)
            wg(m_new_bar, st["a1"], out=gr[p + "eu.w2"])
            cs(m_new_bar, out=gr[p + "eu.b2"])
            h_bar = _silu_bwd(m_new_bar @ w[p + "eu.w2"], st["h"])
            cs(h_bar, out=gr[p + "eu.b1"])
            wg(h_bar, st["xcat"], out=gr[p + "eu.w1"])
            x_bar = h_bar @ w[p + "eu.w1"]
            m_in_o = m_new_bar + x_bar[:, :de]
            ta_bar = x_bar[:, de:]
            # TU (own centres)
            wg(ta_bar, st["Y"], out=gr[p + "tu.up"])
            Y_bar = ta_bar @ w[p + "tu.up"]
            if gem:
                Z_bar = Y_bar * st["g"]
                g_bar = Y_bar * st["Z"]
                wg(Z_bar, st["S"][e0:e1], out=gr[p + "tu.bilinear_proj"])
                S_bar_o = Z_bar @ w[p + "tu.bilinear_proj"]
            else:
                S_bar_o = Y_bar * st["g"]
                g_bar = Y_bar * st["S"][e0:e1]
            wg(g_bar, fw.rbf[e0:e1], out=gr[p + "tu.rbf_gate"])
            rbf_bar[e0:e1].addmm_(g_bar, w[p + "tu.rbf_gate"])
            S_bar = torch.zeros_like(st["S"])
            S_bar[e0:e1] = S_bar_o
            X_bar = torch.zeros_like(st["X"])
            Wk_bar = torch.zeros_like(st["Wk"])
            if n1 > n0:
                ops.triplet_bwd(ep_own, bg.rev, bg.geo, st["X"], st["Wk"], c.cutoff, S_bar, eg, X_bar=X_bar,
                                W_bar=Wk_bar, max_degree=bg.max_deg)
            wp_bar = Wk_bar.permute(2, 0, 1).reshape(Wk_bar.shape[2], -1)
            Xb = X_bar[lo:hi]
            if gem:
                torch.mm(wp_bar, w[p + "tu.sbf_gate"].t(), out=gr[p + "tu.bilinear_b"])
                torch.mm(w[p + "tu.bilinear_b"].t(), wp_bar, out=gr[p + "tu.sbf_gate"])
                wg(Xb, st["down"][lo:hi], out=gr[p + "tu.bilinear_a"])
                down_bar = Xb @ w[p + "tu.bilinear_a"]
            else:
                gr[p + "tu.sbf_gate"].copy_(wp_bar)
                down_bar = Xb
            wg(down_bar, st["m"][lo:hi], out=gr[p + "tu.down"])
            m_bar = torch.zeros((E, de), dtype=torch.float32, device=dev)
            torch.mm(down_bar, w[p + "tu.down"], out=m_bar[lo:hi])  # partial, rows rev(own)
            m_bar[e0:e1] += m_in_o
        # edge init (rows lo:hi; partial adjoint)
        wg(m_bar[lo:hi], fw.rbf[lo:hi], out=gr["edge_init.w"])
        cs(m_bar[lo:hi], out=gr["edge_init.b"])
        rbf_bar[lo:hi].addmm_(m_bar[lo:hi], w["edge_init.w"])
        ops.rbf_bwd(bg.geo, rbf_bar, c.cutoff, eg)
        pos_bar = ops.positions_bwd(bg.edge_ptr, bg.rev, bg.geo, eg)
        cm.all_reduce_(pos_bar, phase="backward", block=-1, stage="positions", level="position")
        cm.all_reduce_(self.weights.grad_flat, phase="backward", block=-1, stage="params", level="param")
        return pos_bar


def _triplet_fwd_into(ep_own, bg, X, Wk, cutoff, S):
    """Triplet forward over a centre range, writing the owned rows of a full-size S."""
    from ._lib import call, ptr, stream

    k, l, dg = Wk.shape
    call("egn_triplet_fwd", ptr(ep_own), ptr(bg.rev), ptr(bg.geo), ep_own.shape[0] - 1, int(bg.max_deg),
         ptr(X.contiguous()), ptr(Wk), k, l, dg, float(cutoff), ptr(S), stream())
    return S


class GPTrainer:
    """Graph-parallel SGD step for one rank over a replicated BatchGraph
    (tasks.loss_and_grads semantics, egn/tasks.py:131-185): energies are
    replicated, force residuals and seeds are rank-local for the owned atoms,
    the loss value is all-reduced for reporting."""

    def __init__(self, params, bg: BatchGraph, e_target, f_target, w_energy: float, w_forces: float, comm: Comm,
                 part: CenterPartition, device="cuda", dp_comm: Comm | None = None, global_graphs: int | None = None):
        """dp_comm / global_graphs: GP x DP composition -- this replica's graphs are part of a
        global batch of `global_graphs`; after the graph-parallel backward the parameter
        gradient and the loss are all-reduced across the replicas (gp_dp_layout)."""
        self.config = params.config
        self.bg, self.comm, self.part = bg, comm, part
        self.dp_comm = dp_comm
        self.weights = DeviceWeights.from_params(params, device)
        self.engine = GraphParallelEngine(self.weights, comm, part)
        self.n = bg.num_graphs if global_graphs is None else int(global_graphs)
        self.e_target = torch.as_tensor(np.asarray(e_target), dtype=torch.float64, device=bg.device)
        n0, n1 = self.engine.n0, self.engine.n1
        self.f_target = (torch.as_tensor(np.asarray(f_target), dtype=torch.float64, device=bg.device)[n0:n1]
                         if f_target is not None else None)
        sizes = torch.as_tensor(bg.graph_sizes, dtype=torch.float64, device=bg.device)
        self.atom_count = sizes.repeat_interleave(torch.as_tensor(bg.graph_sizes, device=bg.device))[n0:n1]
        self.w_energy, self.w_forces = float(w_energy), float(w_forces)

    def step(self, lr: float) -> torch.Tensor:
        fw = self.engine.forward(self.bg)
        res = fw.energy.double() - self.e_target
        loss = torch.zeros(1, dtype=torch.float64, device=self.bg.device)
        if self.comm.rank == 0:
            loss += (self.w_energy * res * res).sum() / self.n
        d_e = 2.0 * self.w_energy * res / self.n
        d_f = None
        if self.w_forces != 0.0:
            delta = fw.forces.double() - self.f_target
            loss += self.w_forces * ((delta * delta).sum(dim=1) / self.atom_count).sum() / self.n
            d_f = 2.0 * self.w_forces * delta / (self.n * self.atom_count[:, None])
        self.engine.backward(self.bg, fw, d_e, d_f)
        self.comm.all_reduce_(loss, phase="backward", block=-1, stage="loss", level="global")
        if self.dp_comm is not None:
            self.dp_comm.all_reduce_(self.weights.grad_flat, phase="backward", block=-1, stage="params",
                                     level="replica")
            self.dp_comm.all_reduce_(loss, phase="backward", block=-1, stage="loss", level="replica")
        if lr != 0.0:
            self.weights.sgd_(lr)
        return loss


# ---------------------------------------------------------------------------
# reference-shaped API: WorkerGroup (egn/runtime.py:265-683) on one device
# ---------------------------------------------------------------------------
@dataclass
class ParallelRunResult:
    energy: float
    forces: np.ndarray | None
    comm_log: CommLog
    partition: CenterPartition
    stage_seconds: dict = field(default_factory=dict)


@dataclass
class GradientBundle:
    d_params: dict
    d_positions: np.ndarray


class WorkerGroup:
    """P graph-parallel ranks over one system, run as threads on one GPU.

    Same surface as egn.runtime.WorkerGroup: forward() and
    forward_backward(d_energy, d_forces) -> (ParallelRunResult, GradientBundle);
    worker failures surface as WorkerGroupError(stage, rank)."""

    def __init__(self, system, params, timeout: float = 60.0, fault: str | None = None, device="cuda",
                 align_graphs: bool = False):
        from .graph import build_batch

        self.params = params
        self.config = params.config
        self.workers = self.config.workers
        self.timeout, self.fault, self.device = timeout, fault, device
        self.bg = build_batch(system, self.config.cutoff, device)
        cand = self.bg.graph_ptr.cpu().numpy() if align_graphs else None
        self.partition = partition_centers(self.bg.deg.cpu().numpy(), self.workers, candidates=cand)

    def forward(self) -> ParallelRunResult:
        res, _ = self._run(False, 0.0, None)
        return res

    def forward_backward(self, d_energy: float = 1.0, d_forces=None):
        if d_forces is not None and self.config.variant != GEMNET:
            raise ValueError("force seeds require the force-centric variant")
        return self._run(True, d_energy, d_forces)

    def _run(self, backward: bool, d_energy: float, d_forces):
        P = self.workers
        log = CommLog()
        shared = _ThreadShared(P, self.timeout, self.fault)
        outs: list = [None] * P
        errors: list = [None] * P
        stages = ["setup"] * P
        dev = torch.device(self.device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev)

        def body(rank):
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(stream):
                    comm = ThreadComm(rank, shared, log) if P > 1 else LocalComm(log)
                    eng = GraphParallelEngine(DeviceWeights.from_params(self.params, self.device), comm,
                                              self.partition)
                    stages[rank] = "forward"
                    fw = eng.forward(self.bg)
                    bundle = None
                    if backward:
                        stages[rank] = "backward"
                        df = None
                        if d_forces is not None:
                            df = torch.as_tensor(np.asarray(d_forces), device=dev)[eng.n0:eng.n1]
                        de = torch.as_tensor(np.broadcast_to(np.asarray(d_energy, dtype=np.float64),
                                                             (self.bg.num_graphs,)).copy(), device=dev)
                        pos_bar = eng.backward(self.bg, fw, de, df)
                        bundle = (eng.weights.to_numpy(grads=True), pos_bar.cpu().numpy())
                    outs[rank] = (fw, eng, bundle)
            except BaseException as exc:  # noqa: BLE001 - reported to the caller
                errors[rank] = exc
                shared.abort()

        if P == 1:
            body(0)
        else:
            threads = [threading.Thread(target=body, args=(r,), name=f"egn-gp-{r}") for r in range(P)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
        primary = None
        for r, exc in enumerate(errors):
            if exc is not None and (primary is None or (isinstance(primary[1], CollectiveTimeoutError)
                                                        and not isinstance(exc, CollectiveTimeoutError))):
                primary = (r, exc)
        if primary is not None:
            raise WorkerGroupError(stages[primary[0]], primary[0], primary[1]) from primary[1]
        fw0 = outs[0][0]
        energies = {tuple(o[0].energy.tolist()) for o in outs}
        if len(energies) != 1:
            raise WorkerGroupError("finalize", 0, AssertionError("worker outputs diverged"))
        forces = None
        if self.config.variant == GEMNET:
            forces = np.concatenate([o[0].forces.double().cpu().numpy() for o in outs], axis=0)
        energy = float(fw0.energy[0]) if fw0.energy.numel() == 1 else fw0.energy.double().cpu().numpy()
        result = ParallelRunResult(energy, forces, log, self.partition)
        bundle = None
        if backward:
            grads, pos = outs[0][2]
            bundle = GradientBundle(grads, pos)
        return result, bundle
