"""torch custom-op layer over the C ABI: ``torch.ops.egn.*``.

Every op is a ``torch.library.custom_op`` whose implementation calls the native library
(libegn_b200.so) through ops.py, with a fake (meta) implementation for the shape-static ops
so the dispatcher, FakeTensor tracing and ``torch.compile`` see them as opaque graph nodes.
Two levels:

* kernel ops -- ``egn::rbf``, ``egn::rbf_linear``, ``egn::linear``, ``egn::triplet_fwd``,
  ``egn::triplet_bwd`` (mutates edge_grad), ``egn::aggregate_in_edges``, ``egn::gather_rows``,
  ``egn::graph_sum``, ``egn::force_head``, ``egn::positions_bwd``;
* the model op ``egn::energy_forces(params, positions, graph_ptr, key)`` -> (energy [G], forces [V, 3])
  with its autograd formula ``egn::energy_forces_backward`` (the explicit adjoint of
  engine.Engine), which EGNModel calls.  `key` names a registered (Engine, BatchGraph) pair:
  graph topology is data-dependent, so it is built outside the traced region and looked up
  by key inside the op (its sizes make the fake implementation shape-static).
"""

from __future__ import annotations

import itertools
import threading

import torch
from torch import Tensor

from . import ops

_LOCK = threading.Lock()
_KEYS = itertools.count(1)
_MODELS: dict = {}  # key -> {"engine", "bg", "fw"}


def register_model(engine, bg) -> int:
    """Register an (Engine, BatchGraph) pair for egn::energy_forces; returns its key."""
    with _LOCK:
        key = next(_KEYS)
        _MODELS[key] = {"engine": engine, "bg": bg, "fw": None}
    return key


def release_model(key: int) -> None:
    with _LOCK:
        _MODELS.pop(key, None)


# ---------------------------------------------------------------------------
# kernel ops
# ---------------------------------------------------------------------------
@torch.library.custom_op("egn::rbf", mutates_args=())
def rbf(geo: Tensor, k_rbf: int, cutoff: float) -> Tensor:
    """Radial basis of the packed per-edge (u, d) (egn/basis.py:35-42, fp32)."""
    return ops.rbf(geo, k_rbf, cutoff)


@rbf.register_fake
def _(geo, k_rbf, cutoff):
    return geo.new_empty((geo.shape[0], k_rbf))


@torch.library.custom_op("egn::rbf_linear", mutates_args=())
def rbf_linear(rbf_t: Tensor, w: Tensor, b: Tensor | None = None) -> Tensor:
    return ops.rbf_linear(rbf_t, w, b)


@rbf_linear.register_fake
def _(rbf_t, w, b=None):
    return rbf_t.new_empty((rbf_t.shape[0], w.shape[0]))


@torch.library.custom_op("egn::linear", mutates_args=())
def linear(a: Tensor, w: Tensor, bias: Tensor | None = None, resid: Tensor | None = None, w_mn: bool = False,
           dsilu_aux: Tensor | None = None) -> Tensor:
    """a w^T (+ bias, + resid; w_mn: a w; dsilu_aux: times silu'(aux)) on the tcgen05 GEMM."""
    flags = ops.EPI_DSILU_AUX if dsilu_aux is not None else 0
    return ops.linear(a, w, bias=bias, resid=resid, aux=dsilu_aux, flags=flags, w_mn=w_mn)


@linear.register_fake
def _(a, w, bias=None, resid=None, w_mn=False, dsilu_aux=None):
    return a.new_empty((a.shape[0], w.shape[1] if w_mn else w.shape[0]))


@torch.library.custom_op("egn::triplet_fwd", mutates_args=())
def triplet_fwd(edge_ptr: Tensor, rev: Tensor, geo: Tensor, X: Tensor, Wk: Tensor, cutoff: float,
                max_degree: int) -> Tensor:
    """S of the centre-tile triplet interaction (egn/engine.py:118-149)."""
    return ops.triplet_fwd(edge_ptr, rev, geo, X, Wk, cutoff, max_degree=max_degree)


@triplet_fwd.register_fake
def _(edge_ptr, rev, geo, X, Wk, cutoff, max_degree):
    return torch.empty_like(X)


@torch.library.custom_op("egn::triplet_bwd", mutates_args=("edge_grad",))
def triplet_bwd(edge_ptr: Tensor, rev: Tensor, geo: Tensor, X: Tensor, Wk: Tensor, cutoff: float, S_bar: Tensor,
                edge_grad: Tensor, max_degree: int) -> tuple[Tensor, Tensor]:
    X_bar, W_bar = ops.triplet_bwd(edge_ptr, rev, geo, X, Wk, cutoff, S_bar, edge_grad, max_degree=max_degree)
    return X_bar, W_bar


@triplet_bwd.register_fake
def _(edge_ptr, rev, geo, X, Wk, cutoff, S_bar, edge_grad, max_degree):
    return torch.empty_like(X), torch.empty_like(Wk)


@torch.library.custom_op("egn::aggregate_in_edges", mutates_args=())
def aggregate_in_edges(edge_ptr: Tensor, rev: Tensor, x: Tensor) -> Tensor:
    return ops.aggregate_in_edges(edge_ptr, rev, x)


@aggregate_in_edges.register_fake
def _(edge_ptr, rev, x):
    return x.new_empty((edge_ptr.shape[0] - 1, x.shape[1]))


@torch.library.custom_op("egn::gather_rows", mutates_args=())
def gather_rows(idx: Tensor, x: Tensor) -> Tensor:
    return ops.gather_rows(idx, x)


@gather_rows.register_fake
def _(idx, x):
    return x.new_empty((idx.shape[0], x.shape[1]))


@torch.library.custom_op("egn::graph_sum", mutates_args=())
def graph_sum(graph_ptr: Tensor, x: Tensor) -> Tensor:
    return ops.graph_sum(graph_ptr, x)


@graph_sum.register_fake
def _(graph_ptr, x):
    return x.new_empty((graph_ptr.shape[0] - 1, x.shape[1]))


@torch.library.custom_op("egn::force_head", mutates_args=())
def force_head(edge_ptr: Tensor, rev: Tensor, geo: Tensor, m: Tensor, w: Tensor) -> tuple[Tensor, Tensor]:
    return ops.force_head_fwd(edge_ptr, rev, geo, m, w)


@force_head.register_fake
def _(edge_ptr, rev, geo, m, w):
    return m.new_empty((m.shape[0],)), m.new_empty((edge_ptr.shape[0] - 1, 3))


@torch.library.custom_op("egn::positions_bwd", mutates_args=())
def positions_bwd(edge_ptr: Tensor, rev: Tensor, geo: Tensor, edge_grad: Tensor) -> Tensor:
    return ops.positions_bwd(edge_ptr, rev, geo, edge_grad)


@positions_bwd.register_fake
def _(edge_ptr, rev, geo, edge_grad):
    return geo.new_empty((edge_ptr.shape[0] - 1, 3), dtype=torch.float64)


# ---------------------------------------------------------------------------
# model op with its autograd formula
# ---------------------------------------------------------------------------
@torch.library.custom_op("egn::energy_forces", mutates_args=())
def energy_forces(params: list[Tensor], positions: Tensor, graph_ptr: Tensor, key: int) -> tuple[Tensor, Tensor]:
    """Energies [G] and forces [V, 3] of the registered batch (egn/engine.py:320-438); params
    are the views of the engine's flat weight buffer (state_dict order); positions [V, 3] and
    graph_ptr [G+1] give the output shapes (the fake implementation never reads `key`, which
    torch.compile may turn symbolic).  Energy-centric
    variants return F = -dE/dx at fixed topology (egn/tasks.py:54-59)."""
    ent = _MODELS[key]
    eng, bg = ent["engine"], ent["bg"]
    fw = eng.forward(bg)
    ent["fw"] = fw
    if fw.forces is not None:
        forces = fw.forces
    else:
        ones = torch.ones(bg.num_graphs, device=bg.device)
        forces = (-eng.backward(bg, fw, ones)).to(torch.float32)
    return fw.energy.clone(), forces.clone()


@energy_forces.register_fake
def _(params, positions, graph_ptr, key):
    g, v = graph_ptr.shape[0] - 1, positions.shape[0]
    return positions.new_empty((g,), dtype=torch.float32), positions.new_empty((v, 3), dtype=torch.float32)


@torch.library.custom_op("egn::energy_forces_backward", mutates_args=())
def energy_forces_backward(params: list[Tensor], g_energy: Tensor, g_forces: Tensor, key: int) -> list[Tensor]:
    """Parameter gradients of <g_energy, E> + <g_forces, F> (force-centric: F is differentiable;
    energy-centric: F is not, as tasks.py:147-151)."""
    ent = _MODELS[key]
    eng, bg = ent["engine"], ent["bg"]
    fw = ent["fw"] if ent["fw"] is not None else eng.forward(bg)
    gf = g_forces if fw.forces is not None else None
    eng.backward(bg, fw, g_energy, gf)
    w = eng.weights
    return [w.g[s.name].clone() for s in w.specs]


@energy_forces_backward.register_fake
def _(params, g_energy, g_forces, key):
    return [torch.empty_like(p) for p in params]


def _setup(ctx, inputs, output):
    params, positions, graph_ptr, key = inputs
    ctx.key = key
    ctx.g, ctx.v = graph_ptr.shape[0] - 1, positions.shape[0]
    ctx.save_for_backward(*params)


def _backward(ctx, g_energy, g_forces):
    params = list(ctx.saved_tensors)
    g, v = ctx.g, ctx.v
    dev = params[0].device
    if g_energy is None:
        g_energy = torch.zeros(g, device=dev)
    if g_forces is None:
        g_forces = torch.zeros((v, 3), device=dev)
    grads = torch.ops.egn.energy_forces_backward(params, g_energy.contiguous(), g_forces.contiguous(), ctx.key)
    return list(grads), None, None, None


energy_forces.register_autograd(_backward, setup_context=_setup)
