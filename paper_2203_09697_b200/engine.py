"""Batched EGN forward/backward on the GPU (DimeNet++-style and GemNet-T-style).

This is the device counterpart of egn/engine.py (ModelTape :320-438, stage
recorders :99-261) and the adjoints its tape applies (egn/tape.py).  The
graph is a BatchGraph (G graphs concatenated); every per-graph quantity of
the reference (global state u, energy) becomes a [G, .] tensor, so one call
reproduces the reference's per-graph loop (tasks.py:158-183).

Schedule per block (engine.py:118-217), with the algebraic reorder that is
exact in real arithmetic:
  X  = m W_down^T [A^T] (GemNet: m (A W_down)^T, one GEMM; gather id3_kj commutes with linear)
  S  = triplet_fwd(X)                      (centre-tile kernel, triplet.cu)
  ta = ((S [P^T]) * (rbf W_rbf^T)) W_up^T  (up/P/rbf-gate commute with segment_sum;
                                           W_up is folded into the EU weight, ta is never formed)
  EU, EA+NU, [EU2 + sym], GU               (dense MLPs; EA = in-edge gather-sum)
The backward is written out explicitly (no autograd), mirroring the
reference's reverse walk; geometry adjoints accumulate into one per-edge
float4 (dE/dv_e, dE/dd_e) that a final CSR gather turns into dE/dx.

Edge- and node-sized dense products run on the native tcgen05 3xTF32 GEMM
(ops.linear / ops.linear_wgrad, fused epilogues, bias adjoints folded into the
weight-gradient kernel); the K = k_rbf (6) products, the G-row global stage and
the energy head run on dedicated native kernels.  The graph-structured work (neighbour list, basis,
triplet interaction, segment sums, force head, geometry adjoints, SGD) runs in
the native library.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import contextlib
import os
import threading

import numpy as np
import torch

from . import ops
from .config import GEMNET, ModelConfig
from .graph import BatchGraph
from .params import ModelParams, param_specs

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def _segments(name: str, c: ModelConfig) -> tuple[list, list]:
    """Row and column segments (widths) of a weight of config c.  A concatenated input
    ([m, ta] for eu.w1, [m_new, v] for eu2.w1) has one segment per operand, each padded on
    its own, so the operands keep their own zero-padded layouts."""
    leaf = name.split(".", 1)[1] if name.startswith("block") else name
    K, KL = c.k_rbf, c.k_rbf * c.l_sbf
    table = {
        "atom_embedding": ([118], [c.d_v]), "edge_init.w": ([c.d_e], [K]), "edge_init.b": ([c.d_e], []),
        "tu.down": ([c.d_t], [c.d_e]), "tu.rbf_gate": ([c.d_t], [K]), "tu.sbf_gate": ([c.d_t], [KL]),
        "tu.bilinear_a": ([c.d_bil], [c.d_t]), "tu.bilinear_b": ([c.d_bil], [c.d_t]),
        "tu.bilinear_proj": ([c.d_t], [c.d_bil]), "tu.up": ([c.d_e], [c.d_t]),
        "eu.w1": ([c.d_e], [c.d_e, c.d_e]), "eu.b1": ([c.d_e], []), "eu.w2": ([c.d_e], [c.d_e]),
        "eu.b2": ([c.d_e], []), "nu.w1": ([c.d_v], [c.d_e]), "nu.b1": ([c.d_v], []), "nu.w2": ([c.d_v], [c.d_v]),
        "nu.b2": ([c.d_v], []), "eu2.w1": ([c.d_e], [c.d_e, c.d_v]), "eu2.b1": ([c.d_e], []),
        "eu2.w2": ([c.d_e], [c.d_e]), "eu2.b2": ([c.d_e], []), "sym.w": ([c.d_e], [c.d_e]),
        "gu.w1": ([c.d_u], [c.d_v]), "gu.b1": ([c.d_u], []), "gu.w2": ([c.d_u], [c.d_u]), "gu.b2": ([c.d_u], []),
        "energy_head.w": ([1], [c.d_u]), "energy_head.b": ([1], []), "force_head.w": ([1], [c.d_e]),
    }
    return table[leaf]


def _seg_index(real: list, padded: list) -> np.ndarray:
    """Positions of the real entries of a segmented axis inside its padded layout."""
    out, off = [], 0
    for r, p in zip(real, padded):
        out.append(np.arange(off, off + r))
        off += p
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


class DeviceWeights:
    """fp32 device copy of ModelParams in one flat buffer (+ a grad buffer of
    the same layout), so the SGD update is a single native kernel.

    Feature widths that do not map onto the tcgen05 GEMM tiling (e.g. GemNet-XL d_e = 1302)
    are zero-padded to a multiple of 16 (ModelConfig.padded): ``config`` is the padded
    config the engine runs, ``ref_config`` the reference one; load() / to_numpy() convert
    between the reference layout and the padded device layout (exact: see padded())."""

    def __init__(self, config: ModelConfig, device="cuda", pad: int | None = 16):
        self.ref_config = config
        self.config = config.padded(pad) if pad else config
        self.is_padded = self.config != config
        self.ref_specs = param_specs(config)
        self.specs = param_specs(self.config)
        sizes = [int(np.prod(s.shape)) for s in self.specs]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        total = int(self.offsets[-1])
        self.flat = torch.zeros(total, dtype=torch.float32, device=device)
        self.grad_flat = torch.zeros(total, dtype=torch.float32, device=device)
        # tf32 lo parts of the weights for the GEMMs' B operands (ops.refresh_weight_lo at the
        # start of every forward pass)
        self._lo = ops.register_weight_lo(self.flat) if self.flat.is_cuda else None
        self.w = {}
        self.g = {}
        for s, a, b in zip(self.specs, self.offsets[:-1], self.offsets[1:]):
            self.w[s.name] = self.flat[a:b].view(s.shape)
            self.g[s.name] = self.grad_flat[a:b].view(s.shape)
        self._index = {}
        if self.is_padded:
            for s in self.specs:
                rr, rc = _segments(s.name, config)
                pr, pc = _segments(s.name, self.config)
                self._index[s.name] = (_seg_index(rr, pr), _seg_index(rc, pc) if rc else None)

    @classmethod
    def from_params(cls, params: ModelParams, device="cuda") -> "DeviceWeights":
        dw = cls(params.config, device)
        dw.load(params)
        return dw

    def _pad(self, name: str, a: np.ndarray, shape) -> np.ndarray:
        if not self.is_padded:
            return a
        out = np.zeros(shape, dtype=np.float64)
        ri, ci = self._index[name]
        if ci is None:
            out[ri] = a
        else:
            out[np.ix_(ri, ci)] = a
        return out

    def _unpad(self, name: str, a: np.ndarray) -> np.ndarray:
        if not self.is_padded:
            return a
        ri, ci = self._index[name]
        return a[ri] if ci is None else a[np.ix_(ri, ci)]

    def load(self, params: ModelParams) -> None:
        host = np.concatenate([self._pad(s.name, np.asarray(params.arrays[s.name], dtype=np.float64), s.shape).ravel()
                               for s in self.specs])
        self.flat.copy_(torch.from_numpy(host.astype(np.float32)))

    def to_numpy(self, grads: bool = False) -> dict:
        """Reference-layout host arrays (padding removed)."""
        src = (self.grad_flat if grads else self.flat).detach().double().cpu().numpy()
        return {s.name: self._unpad(s.name, src[a:b].reshape(s.shape)).copy()
                for s, a, b in zip(self.specs, self.offsets[:-1], self.offsets[1:])}

    def unpad(self, name: str, a: np.ndarray) -> np.ndarray:
        """Reference-layout view of a padded parameter-shaped host array."""
        return self._unpad(name, a)

    def unpad_rows(self, x: torch.Tensor, dim: str) -> torch.Tensor:
        """Reference channels of a padded activation (columns [0, d) of [rows, d_padded])."""
        return x[:, : getattr(self.ref_config, dim)]

    def sgd_(self, lr: float) -> None:
        """w -= lr * g (tasks.py:207-208)."""
        ops.sgd_(self.flat, self.grad_flat, lr)

    def adamw_(self, lr: float, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 1e-2) -> None:
        """One AdamW step over the flat buffer (moments allocated on first use)."""
        if not hasattr(self, "_adam_m"):
            self._adam_m = torch.zeros_like(self.flat)
            self._adam_v = torch.zeros_like(self.flat)
            self._adam_t = 0
        self._adam_t += 1
        ops.adamw_(self.flat, self.grad_flat, self._adam_m, self._adam_v, lr, self._adam_t, betas, eps, weight_decay)


@dataclass
class ForwardResult:
    energy: torch.Tensor  # [G]
    forces: torch.Tensor | None  # [V, 3] (gemnet direct head)
    m: torch.Tensor  # final edge features [E, d_e]
    v: torch.Tensor  # final node features [V, d_v]
    u: torch.Tensor  # final global features [G, d_u]
    rbf: torch.Tensor
    blocks: list = field(default_factory=list)
    scale: torch.Tensor | None = None


class Engine:
    """Forward/backward of one model configuration over BatchGraphs."""

    def __init__(self, weights: DeviceWeights):
        self.weights = weights
        self.config = weights.config
        self._side = {}  # per host thread: the stream weight gradients run on (backward)

    def _side_stream(self, bg, index: int = 0):
        """Side stream `index` of this host thread (0: weight gradients and graph-level work,
        1: the node-level adjoint chain, 2: the triplet angle adjoint), or None: EGN_WGRAD_STREAM=0, or a batch below
        EGN_SIDE_MIN_EDGES edges (default 16384) launched eagerly, whose kernels are too short
        for the fork / join to pay (relaxation of one small system)."""
        device = bg.device
        if device.type != "cuda" or os.environ.get("EGN_WGRAD_STREAM", "1") == "0":
            return None
        # (a captured step pays no launch cost for the fork / join: any size)
        if (bg.num_edges < int(os.environ.get("EGN_SIDE_MIN_EDGES", "16384"))
                and not torch.cuda.is_current_stream_capturing()):
            return None
        key = (threading.get_ident(), index)
        if key not in self._side:
            self._side[key] = torch.cuda.Stream(device=device)
        return self._side[key]

    # -- helpers -----------------------------------------------------------
    def _folded_weights(self) -> list:
        """Per block: the folded weights of this step, all from one batched launch
        (egn_small_gemm_batched): Wda = A W_down (GemNet), W1u = W1b W_up, and the
        SBF weight W[k, l, c] = (B W_sbf)[c, k L + l] (GemNet; DimeNet: W_sbf permuted)."""
        c, w = self.config, self.weights.w
        gem = c.variant == GEMNET
        de, dev = c.d_e, self.weights.flat.device
        dt = c.triplet_width
        shapes = [("W1u", (de, c.d_t))] + ([("Wda", (c.d_bil, de)), ("Wk", (c.k_rbf, c.l_sbf, c.d_bil))] if gem
                                           else [("Wk", (c.k_rbf, c.l_sbf, dt))])
        per = [int(np.prod(sh)) for _, sh in shapes]
        per = [(n + 3) // 4 * 4 for n in per]  # 16-byte aligned views
        # one persistent buffer per thread (in-process graph-parallel ranks run forward passes
        # concurrently), registered for tf32 lo parts: the folded weights are GEMM B operands too
        bufs = self.__dict__.setdefault("_fold_bufs", {})
        key = threading.get_ident()
        if key not in bufs or bufs[key][0].device != dev:
            flat = torch.zeros(c.blocks * sum(per), dtype=torch.float32, device=dev)
            bufs[key] = (flat, ops.register_weight_lo(flat) if flat.is_cuda else None)
        flat = bufs[key][0]
        out, probs, o = [], [], 0
        for b in range(c.blocks):
            p = f"block{b}."
            f = {}
            for (name, sh), n in zip(shapes, per):
                f[name] = flat[o:o + int(np.prod(sh))].view(sh)
                o += n
            w1b = w[p + "eu.w1"][:, de:]
            probs.append((w1b, w[p + "tu.up"], f["W1u"], 0, 0, 0))
            if gem:
                probs.append((w[p + "tu.bilinear_a"], w[p + "tu.down"], f["Wda"], 0, 0, 0))
                probs.append((w[p + "tu.bilinear_b"], w[p + "tu.sbf_gate"],
                              f["Wk"].view(c.k_rbf * c.l_sbf, c.d_bil), 0, 0, 1))
            else:  # W[k, l, c] = W_sbf[c, k L + l]: a native transpose into [K L, d_t]
                ops.transpose_into(w[p + "tu.sbf_gate"], f["Wk"].view(c.k_rbf * c.l_sbf, dt))
            out.append(f)
        ops.small_gemms(probs)
        ops.refresh_weight_lo(flat)
        return out

    # -- forward -------------------------------------------------------------
    def forward(self, bg: BatchGraph, m0: torch.Tensor | None = None, u0: torch.Tensor | None = None,
                blocks: list | None = None) -> ForwardResult:
        """Full forward; m0 / u0 / blocks (the reference's block_forward, egn/engine.py:281-317):
        start from given edge / global features and run only the listed blocks."""
        c, w = self.config, self.weights.w
        gem = c.variant == GEMNET
        de = c.d_e
        L = ops.linear
        ops.refresh_weight_lo(self.weights.flat)  # the weights may have changed since the last pass
        folded = self._folded_weights()
        side = self._side_stream(bg)
        rbf = ops.rbf(bg.geo, c.k_rbf, c.cutoff, c.basis_code)
        m = ops.rbf_linear(rbf, w["edge_init.w"], w["edge_init.b"]) if m0 is None else m0  # K = k_rbf (6)
        u = ops.zeros((bg.num_graphs, c.d_u), bg.device) if u0 is None else u0.clone()
        v = None
        order = list(range(c.blocks)) if blocks is None else list(blocks)
        blocks = []
        # the rbf gates of every block (K = k_rbf (6)) depend on the geometry only: side stream,
        # overlapping block 0's down-projection and triplet interaction
        gates_ready = None
        if side is not None:
            side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side) if side is not None else contextlib.nullcontext():
            gates = [ops.rbf_linear(rbf, w[f"block{b}.tu.rbf_gate"]) for b in range(c.blocks)]
        if side is not None:
            gates_ready = torch.cuda.Event()
            gates_ready.record(side)
        for b in order:
            p = f"block{b}."
            st = {"m": m}
            if gem:
                # X = (m W_down^T) A^T = m (A W_down)^T: one edge-sized GEMM with the
                # folded [d_bil, d_e] weight (the [E, d_t] intermediate is never formed)
                Wda = folded[b]["Wda"]
                X = L(m, Wda)
                down = None
                st["Wda"] = Wda
            else:
                down = X = L(m, w[p + "tu.down"])
            Wk = folded[b]["Wk"]
            S = ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X, Wk, c.cutoff, max_degree=bg.max_deg, basis=c.basis_code)
            g = gates[b]
            if gates_ready is not None:
                torch.cuda.current_stream().wait_event(gates_ready)
                gates_ready = None
            if gem:
                Y, Z = L(S, w[p + "tu.bilinear_proj"], aux=g, flags=ops.EPI_MUL_AUX)  # Y = (S P^T) * g
                st["Z"] = Z
            else:
                Y = ops.hadamard(S, g)
            w1 = w[p + "eu.w1"]
            # h = [m, ta] W1^T + b1 with ta = Y W_up^T folded into the second segment:
            # h = m W1a^T + Y (W1b W_up)^T + b1 (no concat, no [E, d_e] ta); a1 = silu(h)
            W1u = folded[b]["W1u"]
            h, a1 = L(m, w1[:, :de], a2=Y, w2=W1u, bias=w[p + "eu.b1"], flags=ops.EPI_SILU_OUT2)
            m_new = L(a1, w[p + "eu.w2"], bias=w[p + "eu.b2"], resid=m)
            st.update(down=down, X=X, Wk=Wk, S=S, g=g, Y=Y, W1u=W1u, h=h, a1=a1, m_new=m_new)
            agg = ops.aggregate_in_edges(bg.edge_ptr, bg.rev, m_new)
            hv, av = L(agg, w[p + "nu.w1"], bias=w[p + "nu.b1"], flags=ops.EPI_SILU_OUT2)
            v = L(av, w[p + "nu.w2"], bias=w[p + "nu.b2"])
            st.update(agg=agg, hv=hv, av=av, v=v)
            if gem:
                w1 = w[p + "eu2.w1"]
                pv = L(v, w1[:, de:])
                h2, a2 = L(m_new, w1[:, :de], bias=w[p + "eu2.b1"], gather=(pv, bg.recv), flags=ops.EPI_SILU_OUT2)
                m2 = L(a2, w[p + "eu2.w2"], bias=w[p + "eu2.b2"], resid=m_new)
                m2r = ops.gather_rows(bg.rev, m2)
                m = L(m2r, w[p + "sym.w"], resid=m2)
                st.update(h2=h2, a2=a2, m2r=m2r)
            else:
                m = m_new
            # GU (engine.py:207-217): u += silu(s W1^T + b1) W2^T + b2, one fused launch over G rows.
            # Only the energy head reads u, so the graph update runs on the side stream,
            # overlapping the next block's edge work (joined before the energy head).
            if side is not None:
                side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side) if side is not None else contextlib.nullcontext():
                s = ops.graph_sum(bg.graph_ptr, v)
                pre, act = ops.graph_mlp_fwd(s, w[p + "gu.w1"], w[p + "gu.b1"], w[p + "gu.w2"], w[p + "gu.b2"], u)
            st.update(s=s, pre=pre, act=act)
            blocks.append(st)
        if side is not None:
            torch.cuda.current_stream().wait_stream(side)
        energy = ops.graph_linear(u, w["energy_head.w"], w["energy_head.b"]).view(-1)
        forces = scale = None
        if gem:
            scale, forces = ops.force_head_fwd(bg.edge_ptr, bg.rev, bg.geo, m, w["force_head.w"].view(-1))
        if v is None:
            v = ops.zeros((bg.num_nodes, c.d_v), bg.device)
        return ForwardResult(energy, forces, m, v, u, rbf, blocks, scale)

    # -- backward ------------------------------------------------------------
    def backward(self, bg: BatchGraph, fw: ForwardResult, d_energy: torch.Tensor,
                 d_forces: torch.Tensor | None = None) -> torch.Tensor:
        """Overwrite weights.grad_flat with dL/dW; return dL/dpositions (f64 [V,3])."""
        c, w, gr = self.config, self.weights.w, self.weights.g
        gem = c.variant == GEMNET
        if d_forces is not None and not gem:
            raise ValueError("force seed given but this variant has no force head")
        de = c.d_e
        L, cs = ops.linear, ops.column_sum
        # Weight gradients (g^T x) depend on nothing the data gradients produce later in the
        # block, so they run on a side stream and overlap the data-gradient products and
        # gathers of the main stream (each fills the other's wave tail and launch latency).
        # Same kernels, same order per stream: results are unchanged.  Their operands stay
        # referenced until the join at the next block, so no buffer is recycled under them.
        main = torch.cuda.current_stream() if bg.device.type == "cuda" else None
        side = self._side_stream(bg)
        side2 = self._side_stream(bg, 1)
        # the angle adjoint of the triplet interaction (edge_grad x, y, z) feeds only the final
        # positions adjoint: it runs on a third stream, overlapping the rest of the backward,
        # and is joined before the first later writer of edge_grad (rbf_bwd)
        angle = self._side_stream(bg, 2)
        angle_keep = []
        pending = []

        def wg(g, x, out, bias_out=None):
            if side is None or not (ops._tc_ok(4, x.shape[1], g, x) and out.stride(1) == 1):
                return ops.linear_wgrad(g, x, out, bias_out)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                ops.gemm_wgrad(g, x, out=out, colsum=bias_out)
            pending.append((g, x, out, bias_out))
            return out

        def join():
            if side is not None and pending:
                main.wait_stream(side)
                pending.clear()

        ops.zero_(self.weights.grad_flat)
        eg = ops.zeros((bg.num_edges, 4), bg.device)
        dE = d_energy.to(torch.float32).view(-1, 1)
        u_bar = ops.graph_linear_bwd(dE, fw.u, w["energy_head.w"], w_bar=gr["energy_head.w"],
                                     b_bar=gr["energy_head.b"])
        m_bar = ops.zeros((bg.num_edges, de), bg.device)
        if gem and d_forces is not None:
            ops.force_head_bwd(bg.recv, bg.geo, fw.m, w["force_head.w"].view(-1), fw.scale,
                               d_forces.to(torch.float32).contiguous(), m_bar, eg,
                               w_bar=gr["force_head.w"].view(-1))
        rbf_bar = ops.zeros(tuple(fw.rbf.shape), bg.device)
        post = []  # weight-sized gradient products, batched after the block loop
        for b in range(c.blocks - 1, -1, -1):
            join()
            p = f"block{b}."
            st = fw.blocks[b]
            # GU (engine.py:207-217): fused adjoint over G rows (data and weight gradients)
            # (node-level: on the side stream, overlapping the edge-level adjoints below; the
            # main stream waits for v_ready before its first use of v_bar)
            v_ready = None
            if side is not None:
                side.wait_stream(main)
            with torch.cuda.stream(side) if side is not None else contextlib.nullcontext():
                s_bar = ops.graph_mlp_bwd(u_bar, st["s"], st["pre"], st["act"], w[p + "gu.w1"], w[p + "gu.w2"],
                                          gr[p + "gu.w1"], gr[p + "gu.b1"], gr[p + "gu.w2"], gr[p + "gu.b2"])
                v_bar = ops.gather_rows(bg.node_graph, s_bar)
            if side is not None:
                v_ready = torch.cuda.Event()
                v_ready.record(side)
                pending.append((s_bar, v_bar))
            if gem:
                # sym (engine.py:195-200): m = m2 + m2[rev] Wsym^T
                wg(m_bar, st["m2r"], gr[p + "sym.w"])
                t = L(m_bar, w[p + "sym.w"], w_mn=True)
                # m_bar is dead after this point of the block: accumulate in place (once the
                # side-stream weight gradient above has read it)
                join()
                m2_bar = ops.gather_rows(bg.rev, t, out=m_bar, accumulate=True)
                # EU2 (engine.py:180-192)
                wg(m2_bar, st["a2"], gr[p + "eu2.w2"], gr[p + "eu2.b2"])
                h2_bar = L(m2_bar, w[p + "eu2.w2"], w_mn=True, aux=st["h2"], flags=ops.EPI_DSILU_AUX)
                w1 = w[p + "eu2.w1"]
                wg(h2_bar, st["m_new"], gr[p + "eu2.w1"][:, :de], gr[p + "eu2.b1"])
                # The node-level chain (EA + NU adjoints, engine.py:166-177: pv_bar -> v_bar ->
                # hv_bar -> agg_bar) runs on a second side stream, overlapping the edge-sized
                # m_new_bar product; the main stream joins it before the gather into m_new_bar.
                if side2 is not None:
                    side2.wait_stream(main)
                with torch.cuda.stream(side2) if side2 is not None else contextlib.nullcontext():
                    pv_bar = ops.aggregate_in_edges(bg.edge_ptr, bg.rev, h2_bar)
                    if v_ready is not None:
                        side2.wait_event(v_ready)
                    v_bar = L(pv_bar, w1[:, de:], w_mn=True, resid=v_bar)
                    hv_bar = L(v_bar, w[p + "nu.w2"], w_mn=True, aux=st["hv"], flags=ops.EPI_DSILU_AUX)
                    agg_bar = L(hv_bar, w[p + "nu.w1"], w_mn=True)
                node_ready = None
                if side2 is not None:
                    node_ready = torch.cuda.Event()
                    node_ready.record(side2)
                    pending.append((h2_bar, pv_bar, v_bar, hv_bar, agg_bar))
                m_new_bar = L(h2_bar, w1[:, :de], w_mn=True, resid=m2_bar)
                if node_ready is not None:
                    main.wait_event(node_ready)
                wg(pv_bar, st["v"], gr[p + "eu2.w1"][:, de:])
                wg(v_bar, st["av"], gr[p + "nu.w2"], gr[p + "nu.b2"])
                wg(hv_bar, st["agg"], gr[p + "nu.w1"], gr[p + "nu.b1"])
                ops.gather_rows(bg.recv, agg_bar, out=m_new_bar, accumulate=True)
            else:
                m_new_bar = m_bar  # dead after this point of the block
                # EA + NU (engine.py:166-177)
                wg(v_bar, st["av"], gr[p + "nu.w2"], gr[p + "nu.b2"])
                if v_ready is not None:
                    main.wait_event(v_ready)
                hv_bar = L(v_bar, w[p + "nu.w2"], w_mn=True, aux=st["hv"], flags=ops.EPI_DSILU_AUX)
                wg(hv_bar, st["agg"], gr[p + "nu.w1"], gr[p + "nu.b1"])
                agg_bar = L(hv_bar, w[p + "nu.w1"], w_mn=True)
                ops.gather_rows(bg.recv, agg_bar, out=m_new_bar, accumulate=True)
            # EU (engine.py:152-158)
            wg(m_new_bar, st["a1"], gr[p + "eu.w2"], gr[p + "eu.b2"])
            h_bar = L(m_new_bar, w[p + "eu.w2"], w_mn=True, aux=st["h"], flags=ops.EPI_DSILU_AUX)
            w1 = w[p + "eu.w1"]
            wg(h_bar, st["m"], gr[p + "eu.w1"][:, :de], gr[p + "eu.b1"])
            # ta = Y W_up^T was folded into W1u = W1b W_up: both weight gradients come from
            # T2 = h_bar^T Y  (W1b_bar = T2 W_up^T, W_up_bar = W1b^T T2)
            T2 = wg(h_bar, st["Y"], torch.empty((de, st["Y"].shape[1]), dtype=torch.float32, device=bg.device))
            post.append((T2, w[p + "tu.up"], gr[p + "eu.w1"][:, de:], 0, 1, 0))  # W1b_bar = T2 W_up^T
            post.append((w1[:, de:], T2, gr[p + "tu.up"], 1, 0, 0))  # W_up_bar = W1b^T T2
            m_in_bar = L(h_bar, w1[:, :de], w_mn=True, resid=m_new_bar)
            # TU (engine.py:118-149): Y_bar = ta_bar W_up = h_bar W1u
            if gem:
                # Z_bar = Y_bar * g fused into the GEMM epilogue (second output Y_bar)
                Z_bar, Y_bar = L(h_bar, st["W1u"], w_mn=True, aux=st["g"], flags=ops.EPI_MUL_AUX)
                g_prod = (Y_bar, st["Z"])  # g_bar = Y_bar * Z, formed inside the adjoint kernel
                wg(Z_bar, st["S"], gr[p + "tu.bilinear_proj"])
                S_bar = L(Z_bar, w[p + "tu.bilinear_proj"], w_mn=True)
            else:
                # S_bar = Y_bar * g fused into the GEMM epilogue (second output Y_bar)
                S_bar, Y_bar = L(h_bar, st["W1u"], w_mn=True, aux=st["g"], flags=ops.EPI_MUL_AUX)
                g_prod = (Y_bar, st["S"])  # g_bar = Y_bar * S
            # rbf_bar is read only after the block loop: the gate adjoint runs on the side stream
            if side is not None:
                side.wait_stream(main)
            with torch.cuda.stream(side) if side is not None else contextlib.nullcontext():
                ops.rbf_linear_bwd(fw.rbf, w[p + "tu.rbf_gate"], g_prod[0], rbf_bar, gr[p + "tu.rbf_gate"],
                                   g2=g_prod[1])
            if side is not None:
                pending.append(g_prod)
            if angle is not None:
                angle.wait_stream(main)
                with torch.cuda.stream(angle):
                    ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, st["X"], st["Wk"], c.cutoff, S_bar, eg,
                                    max_degree=bg.max_deg, basis=c.basis_code, phases=1)
                angle_keep.append(S_bar)  # read on the angle stream: alive until the join
            X_bar, Wk_bar = ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, st["X"], st["Wk"], c.cutoff,
                                            S_bar, eg, max_degree=bg.max_deg, basis=c.basis_code,
                                            phases=2 if angle is not None else 3)
            if gem:
                # wp_bar[c, kl] = Wk_bar[kl, c]: read transposed in place
                wkb = Wk_bar.view(-1, Wk_bar.shape[2])
                post.append((wkb, w[p + "tu.sbf_gate"], gr[p + "tu.bilinear_b"], 1, 1, 0))
                post.append((w[p + "tu.bilinear_b"], wkb, gr[p + "tu.sbf_gate"], 1, 1, 0))
                # T = X_bar^T m; A_bar = T W_down^T, W_down_bar = A^T T (weight-sized products)
                T = wg(X_bar, st["m"], torch.empty((X_bar.shape[1], de), dtype=torch.float32, device=bg.device))
                post.append((T, w[p + "tu.down"], gr[p + "tu.bilinear_a"], 0, 1, 0))
                post.append((w[p + "tu.bilinear_a"], T, gr[p + "tu.down"], 1, 0, 0))
                m_bar = L(X_bar, st["Wda"], w_mn=True, resid=m_in_bar)
                continue
            else:
                ops.transpose_into(Wk_bar.view(-1, Wk_bar.shape[2]), gr[p + "tu.sbf_gate"])  # [dg, K*L]
                down_bar = X_bar
            wg(down_bar, st["m"], gr[p + "tu.down"])
            m_bar = L(down_bar, w[p + "tu.down"], w_mn=True, resid=m_in_bar)
        join()
        # every deferred weight-sized gradient product in one launch, on the side stream next to
        # the edge-init / geometry adjoints
        if side is not None:
            side.wait_stream(main)
        with torch.cuda.stream(side) if side is not None else contextlib.nullcontext():
            ops.small_gemms(post)
        # edge init (engine.py:109-111), K = k_rbf
        ops.rbf_linear_bwd(fw.rbf, w["edge_init.w"], m_bar, rbf_bar, gr["edge_init.w"], gr["edge_init.b"])
        if angle is not None:
            main.wait_stream(angle)
            angle_keep.clear()
        ops.rbf_bwd(bg.geo, rbf_bar, c.cutoff, eg, c.basis_code)
        pos_bar = ops.positions_bwd(bg.edge_ptr, bg.rev, bg.geo, eg)
        if side is not None:
            main.wait_stream(side)
        return pos_bar

    # -- debug / parity ------------------------------------------------------
    def triplet_features(self, bg: BatchGraph, fw: ForwardResult, block: int, index: int | None = None) -> torch.Tensor:
        """t_feat of one block for every triplet in (out, in) order (engine.py:146,149); index:
        position of that block in fw.blocks when the forward ran a subset of blocks."""
        c, w = self.config, self.weights.w
        if c.basis_code:
            raise ValueError("per-triplet features are materialised for the reference's Gaussian basis only")
        st = fw.blocks[block if index is None else index]
        P = ops.triplet_terms(bg.edge_ptr, bg.rev, bg.geo, bg.tri_ptr, bg.num_triplets, st["X"], st["Wk"],
                              c.cutoff)
        _, ji = ops.triplets_fill(bg.edge_ptr, bg.rev, bg.tri_ptr, bg.num_triplets)
        gt = st["g"].index_select(0, ji)
        if c.variant == GEMNET:
            return (P @ w[f"block{block}.tu.bilinear_proj"].t()) * gt
        return P * gt
