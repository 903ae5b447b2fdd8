"""Graph-parallel execution: one rank per GPU (torch.distributed / NCCL), or P
in-process ranks on one device (threads) for testing and the WorkerGroup API.

Reference: egn/runtime.py (Collective :131-200, WorkerGroup :265-683).  Two
schedules, both on the native kernels (tcgen05 GEMMs with fused epilogues, the
centre-tile triplet kernels, native gathers / segment sums / GU / heads):

``ReferenceScheduleEngine`` ("reference", the WorkerGroup default) is the
reference's own schedule (egn/runtime.py:392-683): split_range shards of the
sorted triplet, edge and node lists (a triplet shard may cut through a centre's
tile: egn_triplet_fwd_window keeps exactly its triplets) and, per block, an
all-reduce of full-size zero-padded buffers after every aggregation level --
ta (edge), v (node), m2 (edge, GemNet), z = (sum v) W1^T (global) -- so the
forward CommLog equals comm_volume() exactly (egn/partition.py:85-95).  EU and
sym are recomputed on all rows by every rank, as the reference does.

``GraphParallelEngine`` ("centre", the B200 performance schedule) gives each
rank a contiguous range of CENTRE atoms (partition.partition_centers): their
out-edges (contiguous, edges are sorted by source) and complete triplet tiles,
so the triplet aggregation never crosses a rank and nothing is recomputed.  Per
block every rank computes only its own rows and all-gathers what its
neighbours read:

  forward                                       exchange
  X = m W_down^T [A^T]     own rows             -> all-gather rows   (edge, N_e d_t)
  S, TU, EU                own edges             (in-edges of own centres read from X)
  m_new                    own rows             -> all-gather rows   (edge, N_e d_e)
  EA + NU                  own nodes             (in-edges read from m_new)
  gemnet: pv = v W1b^T     own nodes            -> all-gather rows   (node, N_v d_e)
          EU2 own edges, m2                     -> all-gather rows   (edge, N_e d_e)
          sym              own edges             (m2[rev] read from the gathered m2)
  GU head: per-graph sums of own nodes          -> all-reduce        (global, G d_v)
  force head: s_e = m_e . w own edges           -> all-gather        (edge, N_e)

The backward is the adjoint: every all-gather becomes a reduce-scatter of
partial row adjoints; parameter and position gradients are all-reduced once at
the end.  Collectives are asynchronous (NCCL on its own stream): each producing
GEMM is split in row chunks and the all-gather of chunk i runs while chunk i+1
is computed; the GU all-reduces run under the following blocks' edge work; each
backward reduce-scatter runs under the weight-gradient products that do not
depend on it.  When no edge crosses a rank boundary (a partition aligned to the
graphs of a batch) every edge / node exchange is skipped.
"""

from __future__ import annotations

import hashlib
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .config import GEMNET
from .engine import DeviceWeights, Engine, ForwardResult
from .graph import BatchGraph
from .partition import CenterPartition, ReferencePartition, partition_centers, partition_reference

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
def _ranges(spec) -> np.ndarray:
    """Per-rank row ranges [P, 2] from bounds [P+1] (contiguous) or explicit (lo, hi) pairs."""
    a = np.asarray(spec, dtype=np.int64)
    if a.ndim == 1:
        return np.stack([a[:-1], a[1:]], axis=1)
    return a.reshape(-1, 2)


class _Handle:
    """A collective in flight: wait() makes the current stream (or host) wait and returns its
    result.  Synchronous transports return completed handles."""

    def __init__(self, value=None, work=None, finish=None):
        self._value, self._work, self._finish = value, work, finish

    def wait(self):
        if self._work is not None:
            self._work.wait()
            self._work = None
        if self._finish is not None:
            self._value = self._finish()
            self._finish = None
        return self._value


class Comm:
    """Row-range collectives over P ranks.  all_gather_rows / reduce_scatter_rows take the
    per-rank row ranges as bounds [P+1] or (lo, hi) pairs [P, 2]; async_op=True returns a
    handle whose wait() completes the collective (NCCL overlaps it with later kernels)."""

    def __init__(self, rank: int, world: int, log: CommLog | None = None, track: bool = False):
        self.rank, self.world = rank, world
        self.log = log if log is not None else CommLog()
        self.track = track  # replica digests (egn/runtime.py:397-401, track_replicas)
        self.digests: list = []

    def _tag(self, t: torch.Tensor, op: str, phase="forward", block=-1, stage="", level="edge", rows=None,
             width=None, elements=None):
        """CommLog record.  Row collectives count the rows they move (a chunked all-gather logs
        each chunk).  width / elements: the reference-layout size when the device buffer has
        zero-padded feature columns (DeviceWeights padding), so the log stays comparable with
        comm_volume()."""
        if level not in ALLOWED_LEVELS:
            raise ValueError(f"buffers of level {level!r} must never enter a collective")
        if self.rank == 0:
            if elements is None and rows is None and width is None:
                elements = int(t.numel())
            elif elements is None:
                r = t.shape[0] if rows is None else int(rows)
                w = int(np.prod(t.shape[1:])) if width is None else int(width)
                elements = r * w
            self.log.records.append(CommRecord(phase, block, stage, level, int(elements), op))

    def _digest(self, t: torch.Tensor) -> torch.Tensor:
        if self.track:
            self.digests.append(hashlib.sha256(t.detach().float().cpu().numpy().tobytes()).hexdigest())
        return t

    def _done(self, h: _Handle, async_op: bool):
        if self.track:
            inner = h
            h = _Handle(finish=lambda: self._digest(inner.wait()))
        return h if async_op else h.wait()

    def all_reduce_(self, t, async_op=False, **tag):
        self._tag(t, "all_reduce", **tag)
        return self._done(self._all_reduce(t), async_op)

    def all_gather_rows(self, full, bounds, async_op=False, **tag):
        rg = _ranges(bounds)
        self._tag(full, "all_gather", rows=int((rg[:, 1] - rg[:, 0]).sum()), **tag)
        return self._done(self._all_gather(full, rg), async_op)

    def reduce_scatter_rows(self, full, bounds, async_op=False, **tag):
        """Sum over ranks of each rank's partial full-size buffer; returns the own rows."""
        rg = _ranges(bounds)
        self._tag(full, "reduce_scatter", rows=int((rg[:, 1] - rg[:, 0]).sum()), **tag)
        return self._done(self._reduce_scatter(full, rg), async_op)

    # transports implement the three primitives, each returning a _Handle
    def _all_reduce(self, t):  # pragma: no cover - interface
        raise NotImplementedError

    def _all_gather(self, full, rg):  # pragma: no cover - interface
        raise NotImplementedError

    def _reduce_scatter(self, full, rg):  # pragma: no cover - interface
        raise NotImplementedError


class LocalComm(Comm):
    """P = 1: every collective is the identity (still logged)."""

    def __init__(self, log=None, track=False):
        super().__init__(0, 1, log, track)

    def _all_reduce(self, t):
        return _Handle(t)

    def _all_gather(self, full, rg):
        return _Handle(full)

    def _reduce_scatter(self, full, rg):
        return _Handle(full[int(rg[0, 0]):int(rg[0, 1])])


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
    """torch.distributed process group.  NCCL: asynchronous collectives straight on the
    device buffers -- uneven row ranges go through all_gather / reduce_scatter with per-rank
    views (grouped broadcasts / reduces inside NCCL), equal contiguous ranges through the
    single-call all_gather_into_tensor / reduce_scatter_tensor, in place.  gloo (CPU tests,
    or CUDA tensors staged through host memory): padded equal-size exchanges."""

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

    def __init__(self, group=None, log=None, track=False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        super().__init__(dist.get_rank(group), dist.get_world_size(group), log, track)
        self.backend = dist.get_backend(group)

    @staticmethod
    def _regular(full, rg):
        sizes = rg[:, 1] - rg[:, 0]
        return (rg[0, 0] == 0 and rg[-1, 1] == full.shape[0] and bool(np.all(rg[1:, 0] == rg[:-1, 1]))
                and bool(np.all(sizes == sizes[0])))

    def _all_reduce(self, t):
        if self.backend != "nccl" and t.is_cuda:
            host = t.cpu()
            self.dist.all_reduce(host, group=self.group)
            t.copy_(host)
            return _Handle(t)
        return _Handle(t, self.dist.all_reduce(t, group=self.group, async_op=True))

    def _all_gather(self, full, rg):
        lo, hi = (int(x) for x in rg[self.rank])
        if self.backend == "nccl":
            if self._regular(full, rg):
                w = self.dist.all_gather_into_tensor(full, full[lo:hi], group=self.group, async_op=True)
            else:
                views = [full[int(a):int(b)] for a, b in rg]
                w = self.dist.all_gather(views, views[self.rank], group=self.group, async_op=True)
            return _Handle(full, w)
        host = full.cpu() if full.is_cuda else full
        sizes = rg[:, 1] - rg[:, 0]
        mr = max(int(sizes.max()), 1)
        send = torch.zeros((mr,) + tuple(full.shape[1:]), dtype=full.dtype)
        send[: hi - lo] = host[lo:hi]
        lst = [torch.empty_like(send) for _ in range(self.world)]
        self.dist.all_gather(lst, send, group=self.group)
        for r, (a, b) in enumerate(rg):
            a, b = int(a), int(b)
            if r != self.rank and b > a:
                host[a:b] = lst[r][: b - a]
        if full.is_cuda:
            full.copy_(host)
        return _Handle(full)

    def _reduce_scatter(self, full, rg):
        lo, hi = (int(x) for x in rg[self.rank])
        if self.backend == "nccl":
            out = torch.empty((hi - lo,) + tuple(full.shape[1:]), dtype=full.dtype, device=full.device)
            if self._regular(full, rg):
                w = self.dist.reduce_scatter_tensor(out, full, group=self.group, async_op=True)
            else:
                w = self.dist.reduce_scatter(out, [full[int(a):int(b)] for a, b in rg], group=self.group,
                                             async_op=True)
            return _Handle(out, w)
        host = full.cpu() if full.is_cuda else full.clone()
        self.dist.all_reduce(host, group=self.group)
        own = host[lo:hi]
        return _Handle(own.to(full.device) if full.is_cuda else own)


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
    """P ranks as threads of one process on one device (the reference's execution model,
    egn/runtime.py:131-200): rank-ordered sums, identical results on every rank.  All ranks
    share torch's current stream, so the host barrier orders the device work."""

    def __init__(self, rank: int, shared: _ThreadShared, log: CommLog, track: bool = False):
        super().__init__(rank, shared.world, log, track)
        self.sh = shared

    def _exchange(self, t):
        self.sh.slots[self.rank] = t
        self.sh.wait(self.sh.enter)
        shapes = {tuple(s.shape) for s in self.sh.slots}
        if len(shapes) != 1:
            raise CollectiveShapeError(f"shape mismatch across workers: {sorted(shapes)}")
        return list(self.sh.slots)

    def _leave(self):
        self.sh.wait(self.sh.exit)

    def _all_reduce(self, t):
        slots = self._exchange(t)
        last = self.world - 1 if self.sh.fault == "drop-last" and self.world > 1 else None
        total = slots[0].clone()
        for r in range(1, self.world):
            if r != last:
                total += slots[r]
        self._leave()
        t.copy_(total)
        return _Handle(t)

    def _all_gather(self, full, rg):
        slots = self._exchange(full)
        pieces = [(int(a), int(b), slots[r][int(a):int(b)].clone()) for r, (a, b) in enumerate(rg)
                  if r != self.rank and b > a]
        self._leave()
        for a, b, p in pieces:
            full[a:b] = p
        return _Handle(full)

    def _reduce_scatter(self, full, rg):
        slots = self._exchange(full)
        lo, hi = (int(x) for x in rg[self.rank])
        total = slots[0][lo:hi].clone()
        for r in range(1, self.world):
            total += slots[r][lo:hi]
        self._leave()
        return _Handle(total)


class Collective:
    """egn/runtime.py:131-200 surface: P thread workers, allreduce_sum(rank, buffer, *, phase,
    block, stage, level) -> rank-ordered sum identical on every worker, barrier(rank), abort();
    CollectiveShapeError / CollectiveTimeoutError / level guard as the reference.  Buffers may
    be numpy arrays (fp64, returned as numpy) or tensors (CPU or CUDA)."""

    def __init__(self, workers: int, log: CommLog, timeout: float = 30.0, fault: str | None = None):
        self.workers, self.log, self.timeout, self.fault = workers, log, timeout, fault
        self._sh = _ThreadShared(workers, timeout, fault)
        self._comms = [ThreadComm(r, self._sh, log) for r in range(workers)]

    def abort(self) -> None:
        self._sh.abort()

    def barrier(self, rank: int) -> None:
        self._sh.wait(self._sh.enter)
        self._sh.wait(self._sh.exit)

    def allreduce_sum(self, rank: int, buffer, *, phase: str, block: int, stage: str, level: str):
        if level not in ALLOWED_LEVELS:
            raise ValueError(f"buffers of level {level!r} must never enter a collective")
        as_np = not isinstance(buffer, torch.Tensor)
        t = torch.from_numpy(np.array(buffer, dtype=np.float64)) if as_np else buffer.clone()
        out = self._comms[rank].all_reduce_(t, phase=phase, block=block, stage=stage, level=level)
        return out.numpy() if as_np else out


# ---------------------------------------------------------------------------
# shared helpers
# ---------------------------------------------------------------------------
class _StageClock:
    """Per-stage device time on rank 0 (ParallelRunResult.stage_seconds, egn/runtime.py:
    219-262): CUDA events at every stage boundary, read once at the end (no syncs in between).
    Also names the current stage for WorkerGroupError."""

    def __init__(self, timed: bool):
        self.timed = timed
        self.stage = "setup"
        self.marks: list = []

    def mark(self, name: str):
        self.stage = name
        if self.timed:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.marks.append((name, ev))

    def seconds(self) -> dict:
        if not self.marks:
            return {}
        self.mark("done")
        torch.cuda.synchronize()
        out: dict = {}
        for (name, a), (_, b) in zip(self.marks[:-1], self.marks[1:]):
            if name != "setup":
                out[name] = out.get(name, 0.0) + a.elapsed_time(b) / 1000.0
        return out


_NO_CLOCK = _StageClock(False)


def _wg(g, x, out, bias_out=None):
    return ops.linear_wgrad(g, x, out, bias_out)


def _rows_add(dst, src, ident):
    """dst += src (row-major, same shape) on the native gather kernel (identity index)."""
    return ops.gather_rows(ident[: src.shape[0]], src, out=dst, accumulate=True)


def _lead_grads(weights: DeviceWeights, lead: bool, cache: dict) -> dict:
    """Gradient views for the replicated tail (energy head, GU): the real buffer on rank 0, a
    scratch copy elsewhere, so the final all-reduce counts them once."""
    if lead:
        return weights.g
    if "junk" not in cache:
        junk = torch.empty_like(weights.grad_flat)
        cache["junk"] = {s.name: junk[a:b].view(s.shape)
                         for s, a, b in zip(weights.specs, weights.offsets[:-1], weights.offsets[1:])}
    return cache["junk"]


# ---------------------------------------------------------------------------
# performance schedule: centre partition, own rows, all-gathers / reduce-scatters
# ---------------------------------------------------------------------------
class GraphParallelEngine:
    """Forward/backward of one rank's centre shard; P = 1 reproduces Engine."""

    def __init__(self, weights: DeviceWeights, comm: Comm, part: CenterPartition, chunks: int = 2,
                 clock: _StageClock | None = None):
        self.weights, self.comm, self.part = weights, comm, part
        self.config = weights.config
        self._helper = Engine(weights)  # folded weights (one batched launch per step)
        self.n0, self.n1, self.e0, self.e1, self.t0, self.t1 = part.rank(comm.rank)
        self.R = weights.ref_config  # CommLog widths in the reference layout
        self.nparam = sum(int(np.prod(s.shape)) for s in weights.ref_specs)
        self.chunks = max(1, int(chunks))
        self.clock = clock or _NO_CLOCK
        self._cache: dict = {}
        self._prep_key = None
        self._prep_val = None

    def _prep(self, bg: BatchGraph) -> dict:
        if self._prep_key == id(bg):
            return self._prep_val
        e0, e1, n0, n1 = self.e0, self.e1, self.n0, self.n1
        dev = bg.device
        rv = bg.rev[e0:e1]
        local = bool(((rv >= e0) & (rv < e1)).all()) if e1 > e0 else True
        flag = torch.tensor([0.0 if local else 1.0], device=dev)
        self.comm.all_reduce_(flag, phase="setup", block=-1, stage="halo", level="global")
        hf = bool(flag.item() == 0.0)
        eb = _ranges(self.part.edge_bounds)
        nb = _ranges(self.part.node_bounds)
        ident = torch.arange(max(bg.num_edges, bg.num_nodes, 1), dtype=torch.int32, device=dev)
        d = dict(hf=hf, eb=eb, nb=nb, ident=ident,
                 ep_own=bg.edge_ptr[n0:n1 + 1], gp_own=(bg.graph_ptr.clamp(n0, n1) - n0).contiguous(),
                 rev_own=rv, recv_own=bg.recv[e0:e1], geo_own=bg.geo[e0:e1],
                 node_graph_own=bg.node_graph[n0:n1],
                 src_local=(bg.src[e0:e1] - n0).to(torch.int32),
                 rev_local=(rv - e0).to(torch.int32) if hf else None,
                 recv_local=(bg.recv[e0:e1] - n0).to(torch.int32) if hf else None)
        self._prep_key, self._prep_val = id(bg), d
        return d

    def halo_free(self, bg: BatchGraph) -> bool:
        return self._prep(bg)["hf"]

    def _chunked(self, rg):
        """Split every rank's range into self.chunks near-equal row ranges (same on all ranks)."""
        out = []
        for i in range(self.chunks):
            a = rg[:, 0] + (rg[:, 1] - rg[:, 0]) * i // self.chunks
            b = rg[:, 0] + (rg[:, 1] - rg[:, 0]) * (i + 1) // self.chunks
            out.append(np.stack([a, b], axis=1))
        return out

    def _produce(self, d, full, rg, fn, **tag):
        """Own rows of `full` by fn(lo, hi, out) in row chunks (relative to the own range), each
        chunk's all-gather in flight while the next one is computed."""
        me = rg[self.comm.rank]
        if d["hf"] or self.comm.world == 1:
            fn(0, int(me[1] - me[0]), full[int(me[0]):int(me[1])])
            return full
        handles = []
        for piece in self._chunked(rg):
            a, b = int(piece[self.comm.rank, 0]), int(piece[self.comm.rank, 1])
            if b > a:
                fn(a - int(me[0]), b - int(me[0]), full[a:b])
            handles.append(self.comm.all_gather_rows(full, piece, async_op=True, **tag))
        for h in handles:
            h.wait()
        return full

    def forward(self, bg: BatchGraph) -> ForwardResult:
        c, w, cm = self.config, self.weights.w, self.comm
        gem = c.variant == GEMNET
        L = ops.linear
        ops.refresh_weight_lo(self.weights.flat)  # the weights may have changed since the last pass
        d = self._prep(bg)
        hf = d["hf"]
        e0, e1, n0, n1 = self.e0, self.e1, self.n0, self.n1
        E, V, G, dev = bg.num_edges, bg.num_nodes, bg.num_graphs, bg.device
        de, dg = c.d_e, c.triplet_width
        f32 = torch.float32
        self.clock.mark("init")
        folded = self._helper._folded_weights()
        rbf = ops.rbf(d["geo_own"], c.k_rbf, c.cutoff, c.basis_code)
        m = ops.rbf_linear(rbf, w["edge_init.w"], w["edge_init.b"])
        gates = [ops.rbf_linear(rbf, w[f"block{b}.tu.rbf_gate"]) for b in range(c.blocks)]
        u = ops.zeros((G, c.d_u), dev)
        blocks, pending, v = [], [], None
        for b in range(c.blocks):
            p = f"block{b}."
            self.clock.mark(f"block{b}.tu")
            st = {"m": m}
            Wx = folded[b]["Wda"] if gem else w[p + "tu.down"]
            X = torch.empty((E, dg), dtype=f32, device=dev)
            mm = m
            self._produce(d, X, d["eb"], lambda a, z, out: L(mm[a:z], Wx, out=out),
                          phase="forward", block=b, stage="X", level="edge", width=self.R.triplet_width)
            Wk = folded[b]["Wk"]
            S = ops.triplet_fwd(d["ep_own"], bg.rev, bg.geo, X, Wk, c.cutoff, max_degree=bg.max_deg,
                                basis=c.basis_code)
            S_o, g = S[e0:e1], gates[b]
            self.clock.mark(f"block{b}.eu")
            if gem:
                Y, Z = L(S_o, w[p + "tu.bilinear_proj"], aux=g, flags=ops.EPI_MUL_AUX)
                st["Z"] = Z
            else:
                Y = ops.hadamard(S_o, g)
            w1 = w[p + "eu.w1"]
            W1u = folded[b]["W1u"]
            h, a1 = L(m, w1[:, :de], a2=Y, w2=W1u, bias=w[p + "eu.b1"], flags=ops.EPI_SILU_OUT2)
            m_new_full = torch.empty((E, de), dtype=f32, device=dev)
            self._produce(d, m_new_full, d["eb"],
                          lambda a, z, out: L(a1[a:z], w[p + "eu.w2"], bias=w[p + "eu.b2"], resid=mm[a:z], out=out),
                          phase="forward", block=b, stage="m_new", level="edge", width=self.R.d_e)
            m_new = m_new_full[e0:e1]
            self.clock.mark(f"block{b}.nu")
            agg = ops.aggregate_in_edges(d["ep_own"], bg.rev, m_new_full)
            hv, av = L(agg, w[p + "nu.w1"], bias=w[p + "nu.b1"], flags=ops.EPI_SILU_OUT2)
            v = L(av, w[p + "nu.w2"], bias=w[p + "nu.b2"])
            st.update(X=X, Wx=Wx, Wk=Wk, S=S, g=g, Y=Y, W1u=W1u, h=h, a1=a1, m_new=m_new, agg=agg, hv=hv, av=av, v=v)
            if gem:
                self.clock.mark(f"block{b}.eu2")
                w1 = w[p + "eu2.w1"]
                pv = torch.empty((V, de), dtype=f32, device=dev)
                vv = v
                self._produce(d, pv, d["nb"], lambda a, z, out: L(vv[a:z], w1[:, de:], out=out),
                              phase="forward", block=b, stage="pv", level="node", width=self.R.d_e)
                h2, a2 = L(m_new, w1[:, :de], bias=w[p + "eu2.b1"], gather=(pv, d["recv_own"]),
                           flags=ops.EPI_SILU_OUT2)
                m2_full = torch.empty((E, de), dtype=f32, device=dev)
                self._produce(d, m2_full, d["eb"],
                              lambda a, z, out: L(a2[a:z], w[p + "eu2.w2"], bias=w[p + "eu2.b2"],
                                                  resid=m_new[a:z], out=out),
                              phase="forward", block=b, stage="m2", level="edge", width=self.R.d_e)
                self.clock.mark(f"block{b}.sym")
                m2r = ops.gather_rows(d["rev_own"], m2_full)
                m = L(m2r, w[p + "sym.w"], resid=m2_full[e0:e1])
                st.update(h2=h2, a2=a2, m2r=m2r)
            else:
                m = m_new
            # GU head: per-graph sums of own nodes, all-reduced under the next blocks' edge work
            s = ops.graph_sum(d["gp_own"], v) if n1 > n0 else ops.zeros((G, c.d_v), dev)
            pending.append((b, s, cm.all_reduce_(s, async_op=True, phase="forward", block=b, stage="gu",
                                                 level="global", width=self.R.d_v)))
            blocks.append(st)
        self.clock.mark("readout")
        for b, s, hnd in pending:
            hnd.wait()
            p = f"block{b}."
            pre, act = ops.graph_mlp_fwd(s, w[p + "gu.w1"], w[p + "gu.b1"], w[p + "gu.w2"], w[p + "gu.b2"], u)
            blocks[b].update(s=s, pre=pre, act=act)
        energy = ops.graph_linear(u, w["energy_head.w"], w["energy_head.b"]).view(-1)
        forces = scale = None
        if gem:
            scale_full = torch.empty((E, 1), dtype=f32, device=dev)
            wf = w["force_head.w"].view(-1)
            self._produce(d, scale_full, d["eb"], lambda a, z, out: ops.force_head_scale(m[a:z], wf, out.view(-1)),
                          phase="forward", block=-1, stage="force", level="edge")
            scale = scale_full.view(-1)
            forces = ops.force_head_gather(d["ep_own"], bg.rev, bg.geo, scale, de)
        return ForwardResult(energy, forces, m, v, u, rbf, blocks, scale)

    def backward(self, bg: BatchGraph, fw: ForwardResult, d_energy: torch.Tensor,
                 d_forces_own: torch.Tensor | None = None) -> torch.Tensor:
        """Sets weights.grad_flat to the all-reduced dL/dW; returns the all-reduced dL/dx (f64 [V,3])."""
        c, w, gr, cm = self.config, self.weights.w, self.weights.g, self.comm
        gem = c.variant == GEMNET
        L = ops.linear
        d = self._prep(bg)
        hf = d["hf"]
        de = c.d_e
        e0, e1, n0, n1 = self.e0, self.e1, self.n0, self.n1
        E, V, dev = bg.num_edges, bg.num_nodes, bg.device
        f32 = torch.float32
        ident = d["ident"]
        lead = cm.rank == 0
        gL = _lead_grads(self.weights, lead, self._cache)
        self.clock.mark("backward.readout")
        ops.zero_(self.weights.grad_flat)
        eg = ops.zeros((E, 4), dev)
        dE = d_energy.to(f32).view(-1, 1).contiguous()
        u_bar = ops.graph_linear_bwd(dE, fw.u, w["energy_head.w"], w_bar=gL["energy_head.w"],
                                     b_bar=gL["energy_head.b"])
        m_bar = ops.zeros((e1 - e0, de), dev)
        if gem and d_forces_own is not None:
            f_full = ops.zeros((V, 3), dev)
            f_full[n0:n1] = d_forces_own.to(f32)
            if not hf:
                cm.all_gather_rows(f_full, d["nb"], phase="backward", block=-1, stage="forces", level="node")
            ops.force_head_bwd(d["recv_own"], d["geo_own"], fw.m, w["force_head.w"].view(-1), fw.scale[e0:e1],
                               f_full, m_bar, eg[e0:e1], w_bar=gr["force_head.w"].view(-1))
        rbf_bar = ops.zeros(tuple(fw.rbf.shape), dev)
        # GU adjoints of every block first: u_bar passes unchanged through the residual updates
        v_bar_gu = []
        for b in range(c.blocks):
            p, st = f"block{b}.", fw.blocks[b]
            s_bar = ops.graph_mlp_bwd(u_bar, st["s"], st["pre"], st["act"], w[p + "gu.w1"], w[p + "gu.w2"],
                                      gL[p + "gu.w1"], gL[p + "gu.b1"], gL[p + "gu.w2"], gL[p + "gu.b2"])
            v_bar_gu.append(ops.gather_rows(d["node_graph_own"], s_bar))
        post = []
        for b in range(c.blocks - 1, -1, -1):
            p, st = f"block{b}.", fw.blocks[b]
            if gem:
                # sym: m = m2 + m2[rev] Wsym^T
                self.clock.mark(f"backward.block{b}.sym")
                t = L(m_bar, w[p + "sym.w"], w_mn=True)
                if hf:
                    _wg(m_bar, st["m2r"], gr[p + "sym.w"])
                    m2_bar = ops.gather_rows(d["rev_local"], t, out=m_bar, accumulate=True)
                else:
                    part = ops.zeros((E, de), dev)
                    ops.scatter_rows(d["rev_own"], ident[: e1 - e0], t, part)
                    hnd = cm.reduce_scatter_rows(part, d["eb"], async_op=True, phase="backward", block=b,
                                                 stage="m2", level="edge", width=self.R.d_e)
                    _wg(m_bar, st["m2r"], gr[p + "sym.w"])  # under the reduce-scatter
                    m2_bar = _rows_add(hnd.wait(), m_bar, ident)
                # EU2
                self.clock.mark(f"backward.block{b}.eu2")
                _wg(m2_bar, st["a2"], gr[p + "eu2.w2"], gr[p + "eu2.b2"])
                h2_full = torch.empty((E, de), dtype=f32, device=dev) if hf else ops.zeros((E, de), dev)
                h2_bar = L(m2_bar, w[p + "eu2.w2"], w_mn=True, aux=st["h2"], flags=ops.EPI_DSILU_AUX,
                           out=h2_full[e0:e1])
                w1 = w[p + "eu2.w1"]
                if hf:
                    pv_bar = ops.aggregate_in_edges(d["ep_own"], bg.rev, h2_full)
                else:
                    pv_part = ops.aggregate_in_edges(bg.edge_ptr, bg.rev, h2_full)
                    hnd = cm.reduce_scatter_rows(pv_part, d["nb"], async_op=True, phase="backward", block=b,
                                                 stage="pv", level="node", width=self.R.d_e)
                _wg(h2_bar, st["m_new"], gr[p + "eu2.w1"][:, :de], gr[p + "eu2.b1"])
                m_new_bar = L(h2_bar, w1[:, :de], w_mn=True, resid=m2_bar)
                if not hf:
                    pv_bar = hnd.wait()
                v_bar = L(pv_bar, w1[:, de:], w_mn=True, resid=v_bar_gu[b])
                _wg(pv_bar, st["v"], gr[p + "eu2.w1"][:, de:])
            else:
                m_new_bar, v_bar = m_bar, v_bar_gu[b]
            # EA + NU (own nodes); EA adjoint = rows rev(e) of own out-edges
            self.clock.mark(f"backward.block{b}.nu")
            hv_bar = L(v_bar, w[p + "nu.w2"], w_mn=True, aux=st["hv"], flags=ops.EPI_DSILU_AUX)
            agg_bar = L(hv_bar, w[p + "nu.w1"], w_mn=True)
            if hf:
                ops.gather_rows(d["recv_local"], agg_bar, out=m_new_bar, accumulate=True)
                _wg(v_bar, st["av"], gr[p + "nu.w2"], gr[p + "nu.b2"])
                _wg(hv_bar, st["agg"], gr[p + "nu.w1"], gr[p + "nu.b1"])
            else:
                part = ops.zeros((E, de), dev)
                ops.scatter_rows(d["rev_own"], d["src_local"], agg_bar, part)
                hnd = cm.reduce_scatter_rows(part, d["eb"], async_op=True, phase="backward", block=b,
                                             stage="m_new", level="edge", width=self.R.d_e)
                _wg(v_bar, st["av"], gr[p + "nu.w2"], gr[p + "nu.b2"])
                _wg(hv_bar, st["agg"], gr[p + "nu.w1"], gr[p + "nu.b1"])
                m_new_bar = _rows_add(hnd.wait(), m_new_bar, ident)
            # EU (own edges)
            self.clock.mark(f"backward.block{b}.eu")
            _wg(m_new_bar, st["a1"], gr[p + "eu.w2"], gr[p + "eu.b2"])
            h_bar = L(m_new_bar, w[p + "eu.w2"], w_mn=True, aux=st["h"], flags=ops.EPI_DSILU_AUX)
            w1 = w[p + "eu.w1"]
            _wg(h_bar, st["m"], gr[p + "eu.w1"][:, :de], gr[p + "eu.b1"])
            T2 = _wg(h_bar, st["Y"], torch.empty((de, st["Y"].shape[1]), dtype=f32, device=dev))
            post.append((T2, w[p + "tu.up"], gr[p + "eu.w1"][:, de:], 0, 1, 0))
            post.append((w1[:, de:], T2, gr[p + "tu.up"], 1, 0, 0))
            m_in_bar = L(h_bar, w1[:, :de], w_mn=True, resid=m_new_bar)
            # TU (own centres)
            self.clock.mark(f"backward.block{b}.tu")
            S_bar = torch.empty((E, st["X"].shape[1]), dtype=f32, device=dev)
            if gem:
                Z_bar, Y_bar = L(h_bar, st["W1u"], w_mn=True, aux=st["g"], flags=ops.EPI_MUL_AUX)
                _wg(Z_bar, st["S"][e0:e1], gr[p + "tu.bilinear_proj"])
                L(Z_bar, w[p + "tu.bilinear_proj"], w_mn=True, out=S_bar[e0:e1])
                g_prod = (Y_bar, st["Z"])
            else:
                Y_bar = L(h_bar, st["W1u"], w_mn=True)
                ops.hadamard(Y_bar, st["g"], out=S_bar[e0:e1])
                g_prod = (Y_bar, st["S"][e0:e1])
            X_bar_full = torch.empty_like(st["X"]) if hf else ops.zeros(tuple(st["X"].shape), dev)
            X_bar_full, Wk_bar = ops.triplet_bwd(d["ep_own"], bg.rev, bg.geo, st["X"], st["Wk"], c.cutoff, S_bar, eg,
                                                 X_bar=X_bar_full, max_degree=bg.max_deg,
                                                 basis=c.basis_code)
            if not hf:
                hnd = cm.reduce_scatter_rows(X_bar_full, d["eb"], async_op=True, phase="backward", block=b,
                                             stage="X", level="edge", width=self.R.triplet_width)
            ops.rbf_linear_bwd(fw.rbf, w[p + "tu.rbf_gate"], g_prod[0], rbf_bar, gr[p + "tu.rbf_gate"], g2=g_prod[1])
            X_bar = X_bar_full[e0:e1] if hf else hnd.wait()
            if gem:
                wkb = Wk_bar.view(-1, Wk_bar.shape[2])
                post.append((wkb, w[p + "tu.sbf_gate"], gr[p + "tu.bilinear_b"], 1, 1, 0))
                post.append((w[p + "tu.bilinear_b"], wkb, gr[p + "tu.sbf_gate"], 1, 1, 0))
                T = _wg(X_bar, st["m"], torch.empty((X_bar.shape[1], de), dtype=f32, device=dev))
                post.append((T, w[p + "tu.down"], gr[p + "tu.bilinear_a"], 0, 1, 0))
                post.append((w[p + "tu.bilinear_a"], T, gr[p + "tu.down"], 1, 0, 0))
                m_bar = L(X_bar, st["Wx"], w_mn=True, resid=m_in_bar)
            else:
                ops.transpose_into(Wk_bar.view(-1, Wk_bar.shape[2]), gr[p + "tu.sbf_gate"])
                _wg(X_bar, st["m"], gr[p + "tu.down"])
                m_bar = L(X_bar, w[p + "tu.down"], w_mn=True, resid=m_in_bar)
        self.clock.mark("backward.init")
        ops.small_gemms(post)
        ops.rbf_linear_bwd(fw.rbf, w["edge_init.w"], m_bar, rbf_bar, gr["edge_init.w"], gr["edge_init.b"])
        self.clock.mark("backward.geometry")
        ops.rbf_bwd(d["geo_own"], rbf_bar, c.cutoff, eg[e0:e1], c.basis_code)
        pos_bar = ops.positions_bwd(bg.edge_ptr, bg.rev, bg.geo, eg)
        self.clock.mark("backward.reduce")
        cm.all_reduce_(pos_bar, phase="backward", block=-1, stage="positions", level="position")
        cm.all_reduce_(self.weights.grad_flat, phase="backward", block=-1, stage="params", level="param",
                       elements=self.nparam)
        return pos_bar


# ---------------------------------------------------------------------------
# reference schedule: split_range shards, full-buffer all-reduces (comm_volume exact)
# ---------------------------------------------------------------------------
class ReferenceScheduleEngine:
    """egn/runtime.py:392-683 on the native kernels.  Rank r owns the split_range shards of
    the triplets (through a centre window), edges and nodes; after every aggregation level the
    zero-padded full buffer is all-reduced, so the buffers are replicated and the CommLog
    equals comm_volume."""

    def __init__(self, weights: DeviceWeights, comm: Comm, part: ReferencePartition,
                 clock: _StageClock | None = None):
        self.weights, self.comm, self.part = weights, comm, part
        self.config = weights.config
        if self.config.basis_code:
            raise ValueError("the reference schedule implements the reference's Gaussian basis only; "
                             "use schedule='centre' for basis='bessel'")
        self._helper = Engine(weights)
        r = comm.rank
        self.t0, self.t1 = int(part.trip_bounds[r]), int(part.trip_bounds[r + 1])
        self.e0, self.e1 = int(part.edge_bounds[r]), int(part.edge_bounds[r + 1])
        self.n0, self.n1 = int(part.node_bounds[r]), int(part.node_bounds[r + 1])
        self.j0, self.j1 = int(part.centre_lo[r]), int(part.centre_hi[r])
        self.flo, self.lhi = int(part.first_lo[r]), int(part.last_hi[r])
        self.R = weights.ref_config  # CommLog widths in the reference layout
        self.nparam = sum(int(np.prod(s.shape)) for s in weights.ref_specs)
        self.clock = clock or _NO_CLOCK
        self._cache: dict = {}
        self._prep_key = None
        self._prep_val = None

    def _prep(self, bg):
        if self._prep_key == id(bg):
            return self._prep_val
        ep = bg.edge_ptr.cpu().numpy()
        n0, n1, j0, j1 = self.n0, self.n1, self.j0, self.j1
        d = dict(ra=int(ep[j0]), rb=int(ep[j1]), na=int(ep[n0]), nb=int(ep[n1]),
                 ep_t=bg.edge_ptr[j0:j1 + 1], ep_n=bg.edge_ptr[n0:n1 + 1],
                 gp_own=(bg.graph_ptr.clamp(n0, n1) - n0).contiguous(),
                 ident=torch.arange(max(bg.num_edges, bg.num_nodes, 1), dtype=torch.int32, device=bg.device))
        d["src_local"] = (bg.src[d["na"]:d["nb"]] - n0).to(torch.int32)
        self._prep_key, self._prep_val = id(bg), d
        return d

    def forward(self, bg: BatchGraph) -> ForwardResult:
        c, w, cm = self.config, self.weights.w, self.comm
        gem = c.variant == GEMNET
        L = ops.linear
        ops.refresh_weight_lo(self.weights.flat)  # the weights may have changed since the last pass
        d = self._prep(bg)
        E, V, G, dev = bg.num_edges, bg.num_nodes, bg.num_graphs, bg.device
        de, dg = c.d_e, c.triplet_width
        e0, e1, n0, n1 = self.e0, self.e1, self.n0, self.n1
        ra, rb = d["ra"], d["rb"]
        has_t = self.j1 > self.j0
        f32 = torch.float32
        self.clock.mark("init")
        folded = self._helper._folded_weights()
        rbf = ops.rbf(bg.geo, c.k_rbf, c.cutoff, c.basis_code)
        m = ops.rbf_linear(rbf, w["edge_init.w"], w["edge_init.b"])
        u = ops.zeros((G, c.d_u), dev)
        blocks, v = [], None
        for b in range(c.blocks):
            p = f"block{b}."
            self.clock.mark(f"block{b}.tu")
            st = {"m": m}
            Wx = folded[b]["Wda"] if gem else w[p + "tu.down"]
            X = L(m, Wx)
            Wk = folded[b]["Wk"]
            S = ops.zeros((E, dg), dev)
            ta = ops.zeros((E, de), dev)
            g = ops.rbf_linear(rbf[ra:rb], w[p + "tu.rbf_gate"]) if has_t else None
            Y = Z = None
            if has_t:
                ops.triplet_fwd_window(d["ep_t"], bg.rev, bg.geo, X, Wk, c.cutoff, self.flo, self.lhi, S)
                if gem:
                    Y, Z = L(S[ra:rb], w[p + "tu.bilinear_proj"], aux=g, flags=ops.EPI_MUL_AUX)
                else:
                    Y = ops.hadamard(S[ra:rb], g)
                L(Y, w[p + "tu.up"], out=ta[ra:rb])
            cm.all_reduce_(ta, phase="forward", block=b, stage="ta", level="edge", width=self.R.d_e)
            self.clock.mark(f"block{b}.eu")
            w1 = w[p + "eu.w1"]
            h, a1 = L(m, w1[:, :de], a2=ta, w2=w1[:, de:], bias=w[p + "eu.b1"], flags=ops.EPI_SILU_OUT2)
            m_new = L(a1, w[p + "eu.w2"], bias=w[p + "eu.b2"], resid=m)
            self.clock.mark(f"block{b}.nu")
            v_part = ops.zeros((V, c.d_v), dev)
            agg = hv = av = None
            if n1 > n0:
                agg = ops.aggregate_in_edges(d["ep_n"], bg.rev, m_new)
                hv, av = L(agg, w[p + "nu.w1"], bias=w[p + "nu.b1"], flags=ops.EPI_SILU_OUT2)
                L(av, w[p + "nu.w2"], bias=w[p + "nu.b2"], out=v_part[n0:n1])
            v = cm.all_reduce_(v_part, phase="forward", block=b, stage="nu", level="node", width=self.R.d_v)
            st.update(X=X, Wx=Wx, Wk=Wk, S=S, g=g, Y=Y, Z=Z, ta=ta, h=h, a1=a1, m_new=m_new, agg=agg, hv=hv, av=av, v=v)
            if gem:
                self.clock.mark(f"block{b}.eu2")
                m2 = ops.zeros((E, de), dev)
                h2 = a2 = None
                if e1 > e0:
                    w1 = w[p + "eu2.w1"]
                    pv = L(v, w1[:, de:])
                    h2, a2 = L(m_new[e0:e1], w1[:, :de], bias=w[p + "eu2.b1"], gather=(pv, bg.recv[e0:e1]),
                               flags=ops.EPI_SILU_OUT2)
                    L(a2, w[p + "eu2.w2"], bias=w[p + "eu2.b2"], resid=m_new[e0:e1], out=m2[e0:e1])
                cm.all_reduce_(m2, phase="forward", block=b, stage="eu2", level="edge", width=self.R.d_e)
                self.clock.mark(f"block{b}.sym")
                m2r = ops.gather_rows(bg.rev, m2)
                m = L(m2r, w[p + "sym.w"], resid=m2)
                st.update(h2=h2, a2=a2, m2r=m2r)
            else:
                m = m_new
            self.clock.mark(f"block{b}.gu")
            s = (ops.graph_sum(d["gp_own"], v[n0:n1]) if n1 > n0
                 else ops.zeros((G, c.d_v), dev))
            z = ops.graph_linear(s, w[p + "gu.w1"])
            cm.all_reduce_(z, phase="forward", block=b, stage="gu", level="global", width=self.R.d_u)
            pre, act = ops.graph_mlp_fwd(z, None, w[p + "gu.b1"], w[p + "gu.w2"], w[p + "gu.b2"], u)
            st.update(s=s, z=z, pre=pre, act=act)
            blocks.append(st)
        self.clock.mark("readout")
        energy = ops.graph_linear(u, w["energy_head.w"], w["energy_head.b"]).view(-1)
        forces = scale = None
        if gem:
            scale, forces = ops.force_head_fwd(bg.edge_ptr, bg.rev, bg.geo, m, w["force_head.w"].view(-1))
        return ForwardResult(energy, forces, m, v, u, rbf, blocks, scale)

    def triplet_shard_features(self, bg: BatchGraph, fw: ForwardResult, block: int) -> torch.Tensor:
        """t_feat rows of this rank's triplet shard (ParallelRunResult.triplet_shards,
        egn/runtime.py:430-431: the last block's own-triplet features)."""
        c, w = self.config, self.weights.w
        dev = bg.device
        if self.j1 <= self.j0:
            return ops.zeros((0, c.d_t), dev)
        st = fw.blocks[block]
        tp = bg.tri_ptr[self.j0:self.j1 + 1]
        tp = (tp - tp[0]).contiguous()
        nt = int(tp[-1])
        P = ops.triplet_terms(bg.edge_ptr[self.j0:self.j1 + 1], bg.rev, bg.geo, tp, nt, st["X"], st["Wk"], c.cutoff)
        _, ji = ops.triplets_fill(bg.edge_ptr[self.j0:self.j1 + 1], bg.rev, tp, nt)
        gate = ops.rbf_linear(fw.rbf, w[f"block{block}.tu.rbf_gate"]).index_select(0, ji)
        if c.variant == GEMNET:
            P = ops.linear(P, w[f"block{block}.tu.bilinear_proj"])
        t = P * gate
        return t[self.flo:self.flo + (self.t1 - self.t0)]

    def backward(self, bg: BatchGraph, fw: ForwardResult, d_energy: torch.Tensor,
                 d_forces: torch.Tensor | None = None) -> torch.Tensor:
        """egn/runtime.py:516-683: rank-partial adjoints all-reduced per stage; returns dL/dx."""
        c, w, gr, cm = self.config, self.weights.w, self.weights.g, self.comm
        gem = c.variant == GEMNET
        L = ops.linear
        d = self._prep(bg)
        E, V, G, dev = bg.num_edges, bg.num_nodes, bg.num_graphs, bg.device
        de = c.d_e
        e0, e1, n0, n1 = self.e0, self.e1, self.n0, self.n1
        ra, rb = d["ra"], d["rb"]
        has_t = self.j1 > self.j0
        ident = d["ident"]
        f32 = torch.float32
        lead = cm.rank == 0
        self.clock.mark("backward.readout")
        ops.zero_(self.weights.grad_flat)
        eg = ops.zeros((E, 4), dev)
        rbf_bar = ops.zeros(tuple(fw.rbf.shape), dev)
        dE = d_energy.to(f32).view(-1, 1).contiguous()
        if lead:
            u_bar = ops.graph_linear_bwd(dE, fw.u, w["energy_head.w"], w_bar=gr["energy_head.w"],
                                         b_bar=gr["energy_head.b"])
        else:
            u_bar = ops.zeros((G, c.d_u), dev)
        cm.all_reduce_(u_bar, phase="backward", block=-1, stage="energy", level="global", width=self.R.d_u)
        m_bar = ops.zeros((E, de), dev)
        if gem and d_forces is not None:
            f_part = ops.zeros((V, 3), dev)
            f_part[n0:n1] = d_forces.to(f32)[n0:n1]
            ops.force_head_bwd(bg.recv, bg.geo, fw.m, w["force_head.w"].view(-1), fw.scale, f_part, m_bar, eg,
                               w_bar=gr["force_head.w"].view(-1))
            cm.all_reduce_(m_bar, phase="backward", block=-1, stage="force", level="edge", width=self.R.d_e)
        post = []
        for b in range(c.blocks - 1, -1, -1):
            p, st = f"block{b}.", fw.blocks[b]
            self.clock.mark(f"backward.block{b}.gu")
            if lead:
                z_bar = ops.graph_mlp_bwd(u_bar, st["z"], st["pre"], st["act"], None, w[p + "gu.w2"], None,
                                          gr[p + "gu.b1"], gr[p + "gu.w2"], gr[p + "gu.b2"])
            else:
                z_bar = ops.zeros((G, c.d_u), dev)
            cm.all_reduce_(z_bar, phase="backward", block=b, stage="gu", level="global", width=self.R.d_u)
            s_bar = ops.graph_linear_bwd(z_bar, st["s"], w[p + "gu.w1"], w_bar=gr[p + "gu.w1"])
            v_bar = ops.zeros((V, c.d_v), dev)
            if n1 > n0:
                ops.gather_rows(bg.node_graph[n0:n1], s_bar, out=v_bar[n0:n1])
            if gem:
                self.clock.mark(f"backward.block{b}.sym")
                m2_bar = ops.zeros((E, de), dev)
                if e1 > e0:
                    mb = m_bar[e0:e1]
                    _wg(mb, st["m2r"][e0:e1], gr[p + "sym.w"])
                    t = L(mb, w[p + "sym.w"], w_mn=True)
                    ops.gather_rows(ident[: e1 - e0], mb, out=m2_bar[e0:e1])
                    ops.scatter_rows(bg.rev[e0:e1], ident[: e1 - e0], t, m2_bar)
                cm.all_reduce_(m2_bar, phase="backward", block=b, stage="sym", level="edge", width=self.R.d_e)
                self.clock.mark(f"backward.block{b}.eu2")
                mn_bar = ops.zeros((E, de), dev)
                if e1 > e0:
                    g2 = m2_bar[e0:e1]
                    w1 = w[p + "eu2.w1"]
                    _wg(g2, st["a2"], gr[p + "eu2.w2"], gr[p + "eu2.b2"])
                    h2_full = ops.zeros((E, de), dev)
                    h2_bar = L(g2, w[p + "eu2.w2"], w_mn=True, aux=st["h2"], flags=ops.EPI_DSILU_AUX,
                               out=h2_full[e0:e1])
                    _wg(h2_bar, st["m_new"][e0:e1], gr[p + "eu2.w1"][:, :de], gr[p + "eu2.b1"])
                    L(h2_bar, w1[:, :de], w_mn=True, resid=g2, out=mn_bar[e0:e1])
                    pv_bar = ops.aggregate_in_edges(bg.edge_ptr, bg.rev, h2_full)
                    _wg(pv_bar, st["v"], gr[p + "eu2.w1"][:, de:])
                    v_bar = L(pv_bar, w1[:, de:], w_mn=True, resid=v_bar)
            else:
                mn_bar = ops.zeros((E, de), dev)
            self.clock.mark(f"backward.block{b}.nu")
            cm.all_reduce_(v_bar, phase="backward", block=b, stage="nu", level="node", width=self.R.d_v)
            if n1 > n0:
                vb = v_bar[n0:n1]
                _wg(vb, st["av"], gr[p + "nu.w2"], gr[p + "nu.b2"])
                hv_bar = L(vb, w[p + "nu.w2"], w_mn=True, aux=st["hv"], flags=ops.EPI_DSILU_AUX)
                _wg(hv_bar, st["agg"], gr[p + "nu.w1"], gr[p + "nu.b1"])
                agg_bar = L(hv_bar, w[p + "nu.w1"], w_mn=True)
                ops.scatter_rows(bg.rev[d["na"]:d["nb"]], d["src_local"], agg_bar, mn_bar)
            cm.all_reduce_(mn_bar, phase="backward", block=b, stage="m_new", level="edge", width=self.R.d_e)
            if not gem:
                _rows_add(mn_bar, m_bar, ident)
            m_new_bar = mn_bar
            self.clock.mark(f"backward.block{b}.eu")
            ta_bar = ops.zeros((E, de), dev)
            m_in = ops.zeros((E, de), dev)
            if e1 > e0:
                g1 = m_new_bar[e0:e1]
                w1 = w[p + "eu.w1"]
                _wg(g1, st["a1"][e0:e1], gr[p + "eu.w2"], gr[p + "eu.b2"])
                h_bar = L(g1, w[p + "eu.w2"], w_mn=True, aux=st["h"][e0:e1], flags=ops.EPI_DSILU_AUX)
                _wg(h_bar, st["m"][e0:e1], gr[p + "eu.w1"][:, :de], gr[p + "eu.b1"])
                _wg(h_bar, st["ta"][e0:e1], gr[p + "eu.w1"][:, de:])
                L(h_bar, w1[:, :de], w_mn=True, resid=g1, out=m_in[e0:e1])
                L(h_bar, w1[:, de:], w_mn=True, out=ta_bar[e0:e1])
            cm.all_reduce_(ta_bar, phase="backward", block=b, stage="ta", level="edge", width=self.R.d_e)
            self.clock.mark(f"backward.block{b}.tu")
            if has_t:
                tb = ta_bar[ra:rb]
                _wg(tb, st["Y"], gr[p + "tu.up"])
                S_bar = ops.zeros(tuple(st["S"].shape), dev)
                if gem:
                    Z_bar, Y_bar = L(tb, w[p + "tu.up"], w_mn=True, aux=st["g"], flags=ops.EPI_MUL_AUX)
                    _wg(Z_bar, st["S"][ra:rb], gr[p + "tu.bilinear_proj"])
                    L(Z_bar, w[p + "tu.bilinear_proj"], w_mn=True, out=S_bar[ra:rb])
                    g_prod = (Y_bar, st["Z"])
                else:
                    Y_bar = L(tb, w[p + "tu.up"], w_mn=True)
                    ops.hadamard(Y_bar, st["g"], out=S_bar[ra:rb])
                    g_prod = (Y_bar, st["S"][ra:rb])
                ops.rbf_linear_bwd(fw.rbf[ra:rb], w[p + "tu.rbf_gate"], g_prod[0], rbf_bar[ra:rb],
                                   gr[p + "tu.rbf_gate"], g2=g_prod[1])
                X_bar = ops.zeros(tuple(st["X"].shape), dev)
                Wk_bar = ops.triplet_bwd_window(d["ep_t"], bg.rev, bg.geo, st["X"], st["Wk"], c.cutoff, self.flo,
                                                self.lhi, S_bar, eg, X_bar, bg.max_deg)
                if gem:
                    wkb = Wk_bar.view(-1, Wk_bar.shape[2])
                    post.append((wkb, w[p + "tu.sbf_gate"], gr[p + "tu.bilinear_b"], 1, 1, 0))
                    post.append((w[p + "tu.bilinear_b"], wkb, gr[p + "tu.sbf_gate"], 1, 1, 0))
                    T = _wg(X_bar, st["m"], torch.empty((X_bar.shape[1], de), dtype=f32, device=dev))
                    post.append((T, w[p + "tu.down"], gr[p + "tu.bilinear_a"], 0, 1, 0))
                    post.append((w[p + "tu.bilinear_a"], T, gr[p + "tu.down"], 1, 0, 0))
                    m_in = L(X_bar, st["Wx"], w_mn=True, resid=m_in)
                else:
                    ops.transpose_into(Wk_bar.view(-1, Wk_bar.shape[2]), gr[p + "tu.sbf_gate"])
                    _wg(X_bar, st["m"], gr[p + "tu.down"])
                    m_in = L(X_bar, w[p + "tu.down"], w_mn=True, resid=m_in)
            m_bar = cm.all_reduce_(m_in, phase="backward", block=b, stage="m_in", level="edge", width=self.R.d_e)
        self.clock.mark("backward.init")
        ops.small_gemms(post)
        if e1 > e0:
            ops.rbf_linear_bwd(fw.rbf[e0:e1], w["edge_init.w"], m_bar[e0:e1], rbf_bar[e0:e1], gr["edge_init.w"],
                               gr["edge_init.b"])
        self.clock.mark("backward.geometry")
        ops.rbf_bwd(bg.geo, rbf_bar, c.cutoff, eg, c.basis_code)
        pos_bar = ops.positions_bwd(bg.edge_ptr, bg.rev, bg.geo, eg)
        self.clock.mark("backward.reduce")
        cm.all_reduce_(pos_bar, phase="backward", block=-1, stage="positions", level="position")
        cm.all_reduce_(self.weights.grad_flat, phase="backward", block=-1, stage="params", level="param",
                       elements=self.nparam)
        return pos_bar


# ---------------------------------------------------------------------------
# training step of one rank
# ---------------------------------------------------------------------------
class GPTrainer:
    """Graph-parallel SGD step for one rank over a replicated BatchGraph
    (tasks.loss_and_grads semantics, egn/tasks.py:131-185): energies are replicated, force
    residuals and seeds are rank-local for the owned atoms (centre schedule) or computed for
    the rank's node shard (reference schedule); the loss value is all-reduced."""

    def __init__(self, params, bg: BatchGraph, e_target, f_target, w_energy: float, w_forces: float, comm: Comm,
                 part, device="cuda", dp_comm: Comm | None = None, global_graphs: int | None = None,
                 chunks: int = 2, cuda_graph: bool = False):
        """part: CenterPartition (centre schedule) or ReferencePartition (reference schedule).
        dp_comm / global_graphs: GP x DP composition -- this replica's graphs are part of a
        global batch of `global_graphs`; after the graph-parallel backward the parameter
        gradient and the loss are all-reduced across the replicas (gp_dp_layout)."""
        self.config = params.config
        self.bg, self.comm, self.part = bg, comm, part
        self.dp_comm = dp_comm
        self.weights = DeviceWeights.from_params(params, device)
        self.reference = isinstance(part, ReferencePartition)
        if self.reference:
            self.engine = ReferenceScheduleEngine(self.weights, comm, part)
        else:
            self.engine = GraphParallelEngine(self.weights, comm, part, chunks=chunks)
        self.n = bg.num_graphs if global_graphs is None else int(global_graphs)
        self.n0, self.n1 = self.engine.n0, self.engine.n1
        self.e_target = torch.as_tensor(np.asarray(e_target), dtype=torch.float64, device=bg.device)
        self.f_target = (torch.as_tensor(np.asarray(f_target), dtype=torch.float64, device=bg.device)[self.n0:self.n1]
                         if f_target is not None else None)
        sizes = torch.as_tensor(bg.graph_sizes, dtype=torch.float64, device=bg.device)
        self.atom_count = sizes.repeat_interleave(torch.as_tensor(bg.graph_sizes, device=bg.device))[self.n0:self.n1]
        self.w_energy, self.w_forces = float(w_energy), float(w_forces)
        # cuda_graph: the whole graph-parallel step -- compute and its NCCL collectives -- is
        # captured once and replayed (NCCL communicators can be captured; gloo ones cannot,
        # and a failed capture falls back to eager steps)
        self.cuda_graph = bool(cuda_graph)
        self._graph = None
        self._graph_loss = None

    def loss_and_grads(self) -> torch.Tensor:
        fw = self.engine.forward(self.bg)
        lead = self.comm.rank == 0
        # energies are replicated: the energy seed on every rank, its loss term on rank 0 only;
        # force terms per owned atom
        loss, d_e, _ = ops.loss_seeds(fw.energy, self.e_target, None, None, None, self.w_energy, 0.0, self.n)
        if not lead:
            loss = ops.loss_seeds(fw.energy, self.e_target, None, None, None, 0.0, 0.0, self.n)[0]
        d_f = None
        if self.w_forces != 0.0:
            f_own = fw.forces[self.n0:self.n1] if self.reference else fw.forces
            lf, _, d_f = ops.loss_seeds(fw.energy, self.e_target, f_own, self.f_target, self.atom_count, 0.0,
                                        self.w_forces, self.n)
            loss = loss + lf
            if self.reference:
                full = ops.zeros((self.bg.num_nodes, 3), self.bg.device)
                full[self.n0:self.n1] = d_f
                d_f = full
        self.engine.backward(self.bg, fw, d_e, d_f)
        loss = loss.reshape(1)
        self.comm.all_reduce_(loss, phase="backward", block=-1, stage="loss", level="global")
        if self.dp_comm is not None:
            self.dp_comm.all_reduce_(self.weights.grad_flat, phase="backward", block=-1, stage="params",
                                     level="replica")
            self.dp_comm.all_reduce_(loss, phase="backward", block=-1, stage="loss", level="replica")
        return loss

    def step(self, lr: float) -> torch.Tensor:
        if self.cuda_graph and self._graph is not None:
            self._graph.replay()
            loss = self._graph_loss
        else:
            loss = self.loss_and_grads()
            if self.cuda_graph:
                self._capture()
        if lr != 0.0:
            self.weights.sgd_(lr)
        return loss

    def _capture(self):
        """Capture loss_and_grads (after one eager step sized every workspace and cached the
        partition's host-side prep)."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.stream(side):
                with torch.cuda.graph(graph, stream=side):
                    self._graph_loss = self.loss_and_grads()
        except Exception as exc:  # noqa: BLE001 (e.g. a gloo communicator)
            import sys

            torch.cuda.synchronize()
            print(f"[egn] CUDA-graph capture of the graph-parallel step failed ({exc!r}); running eagerly",
                  file=sys.stderr)
            self.cuda_graph = False
            return
        torch.cuda.current_stream().wait_stream(side)
        self._graph = graph


# ---------------------------------------------------------------------------
# reference-shaped API: WorkerGroup (egn/runtime.py:203-683) on one device
# ---------------------------------------------------------------------------
@dataclass
class FeatureState:
    """egn/engine.py FeatureState: final features of one forward (host arrays)."""

    global_features: np.ndarray
    node_features: np.ndarray
    edge_features: np.ndarray
    triplet_features: np.ndarray | None
    topology: object
    geometry: object
    basis: object = None


@dataclass
class ParallelRunResult:
    """egn/runtime.py:203-217."""

    energy: float
    forces: np.ndarray | None
    state: FeatureState | None = None
    triplet_shards: list = field(default_factory=list)
    comm_log: CommLog = field(default_factory=CommLog)
    replica_digests: list = field(default_factory=list)
    stage_seconds: dict = field(default_factory=dict)
    partition: object = None

    def timing_csv_rows(self) -> list:
        rows = ["stage,seconds"]
        for stage, seconds in self.stage_seconds.items():
            rows.append(f"{stage},{seconds!r}")
        return rows


@dataclass
class GradientBundle:
    d_params: dict
    d_positions: np.ndarray


class WorkerGroup:
    """P graph-parallel ranks over one system, run as threads on one GPU.

    Same surface as egn.runtime.WorkerGroup(system, params, timeout, fault, track_replicas):
    forward() and forward_backward(d_energy, d_forces) -> (ParallelRunResult, GradientBundle);
    worker failures surface as WorkerGroupError(stage, rank).  schedule="reference" (default)
    runs the reference's split_range shards and full-buffer all-reduces (CommLog ==
    comm_volume); schedule="centre" runs the B200 performance schedule (centre partition,
    row all-gathers / reduce-scatters)."""

    def __init__(self, system, params, timeout: float = 60.0, fault: str | None = None,
                 track_replicas: bool = False, device="cuda", schedule: str = "reference",
                 align_graphs: bool = False):
        from .graph import build_batch, geometry_of, topology_of

        # SURVEY 8(e) names: "balanced" (the parity mode) and "center-aligned" (the performance mode)
        schedule = {"balanced": "reference", "center-aligned": "centre"}.get(schedule, schedule)
        if schedule not in ("reference", "centre"):
            raise ValueError(f"schedule must be 'reference' or 'centre', got {schedule!r}")
        self.system = system
        self.params = params
        self.config = params.config
        self.workers = self.config.workers
        self.timeout, self.fault, self.device = timeout, fault, device
        self.track_replicas = track_replicas
        self.schedule = schedule
        if schedule == "reference" and self.config.basis_code:
            raise ValueError("the reference schedule implements the reference's Gaussian basis only; "
                             "use schedule='centre' for basis='bessel'")
        self.bg = build_batch(system, self.config.cutoff, device)
        self.topology = topology_of(self.bg)
        self.geometry = geometry_of(self.bg)
        if schedule == "reference":
            self.partition = partition_reference(self.bg.tri_ptr.cpu().numpy(), self.bg.num_edges,
                                                 self.bg.num_nodes, self.workers)
        else:
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
        clocks = [_StageClock(timed=(r == 0)) for r in range(P)]
        comms: list = [None] * P
        dev = torch.device(self.device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev)
        bg = self.bg

        def body(rank):
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(stream):
                    comm = (ThreadComm(rank, shared, log, self.track_replicas) if P > 1
                            else LocalComm(log, self.track_replicas))
                    comms[rank] = comm
                    weights = DeviceWeights.from_params(self.params, self.device)
                    if self.schedule == "reference":
                        eng = ReferenceScheduleEngine(weights, comm, self.partition, clocks[rank])
                    else:
                        eng = GraphParallelEngine(weights, comm, self.partition, clock=clocks[rank])
                    fw = eng.forward(bg)
                    t_own = (eng.triplet_shard_features(bg, fw, self.config.blocks - 1)
                             if self.schedule == "reference" else None)
                    bundle = None
                    if backward:
                        df = None
                        if d_forces is not None:
                            df = torch.as_tensor(np.asarray(d_forces), dtype=torch.float64, device=dev)
                            if self.schedule == "centre":
                                df = df[eng.n0:eng.n1]
                        de = torch.as_tensor(np.broadcast_to(np.asarray(d_energy, dtype=np.float64),
                                                             (bg.num_graphs,)).copy(), device=dev)
                        pos_bar = eng.backward(bg, fw, de, df)
                        bundle = (weights.to_numpy(grads=True), pos_bar.cpu().numpy())
                    outs[rank] = (fw, eng, bundle, t_own)
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
            raise WorkerGroupError(clocks[primary[0]].stage, primary[0], primary[1]) from primary[1]
        energies = {tuple(o[0].energy.tolist()) for o in outs}
        if len(energies) != 1:
            raise WorkerGroupError("finalize", 0, AssertionError("worker outputs diverged"))
        fw0 = outs[0][0]
        to_np = lambda t: t.double().cpu().numpy()  # noqa: E731
        dw = outs[0][1].weights
        un = lambda t, dim: to_np(dw.unpad_rows(t, dim))  # noqa: E731
        if self.schedule == "reference":
            m, v = un(fw0.m, "d_e"), un(fw0.v, "d_v")
            forces = to_np(fw0.forces) if fw0.forces is not None else None
        else:
            m = np.concatenate([un(o[0].m, "d_e") for o in outs], axis=0)
            v = np.concatenate([un(o[0].v, "d_v") for o in outs], axis=0)
            forces = (np.concatenate([to_np(o[0].forces) for o in outs], axis=0)
                      if self.config.variant == GEMNET else None)
        energy = float(fw0.energy[0]) if fw0.energy.numel() == 1 else to_np(fw0.energy)
        state = FeatureState(un(fw0.u, "d_u"), v, m, None, self.topology, self.geometry)
        shards = [un(o[3], "d_t") for o in outs] if self.schedule == "reference" else []
        result = ParallelRunResult(energy, forces, state, shards, log, [c.digests for c in comms],
                                   clocks[0].seconds(), self.partition)
        bundle = None
        if backward:
            grads, pos = outs[0][2]
            bundle = GradientBundle(grads, pos)
        return result, bundle
