"""Reference-shaped model surface (egn/__init__.py:3-27) over the native engine.

``ModelTape(system, params, prebuilt=None)`` with ``.energy / .forces / .state`` and
``.backward(d_energy, d_forces) -> GradientBundle`` (egn/engine.py:320-438);
``initial_state`` / ``block_forward`` (:264-317); the basis functions
``rbf_features / rbf_features_ddist / sbf_features / sbf_features_partials /
compute_basis`` (egn/basis.py:35-103); and the gradient surfaces ``backward /
forces_energy_centric / geometry_grads`` (egn/gradients.py:15-61).  Results are host
numpy arrays like the reference's; everything is computed by the native library
(libegn_b200.so) on the GPU -- the hot path itself never materialises the basis
tables these functions return.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .config import GEMNET
from .engine import DeviceWeights, Engine
from .graph import BatchGraph, Geometry, GraphTopology, build_batch, geometry_of, topology_of
from .runtime import FeatureState, GradientBundle

MAX_Z = 118


def _dev(device=None):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def _f64(x, device=None):
    if isinstance(x, torch.Tensor):
        return x.to(device=_dev(device), dtype=torch.float64).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=_dev(device)).contiguous()


def _raise_if(flag: torch.Tensor, msg: str):
    if int(flag.item()):
        raise ValueError(msg)


# ---------------------------------------------------------------------------
# basis (egn/basis.py)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class BasisFeatures:
    edge_rbf: np.ndarray  # (N_e, K)
    triplet_sbf: np.ndarray  # (N_t, K * L)


def rbf_centers(k_rbf: int, cutoff: float) -> np.ndarray:
    """egn/basis.py:23-28."""
    if k_rbf < 1:
        raise ValueError("k_rbf must be >= 1")
    if k_rbf == 1:
        return np.zeros(1, dtype=np.float64)
    return np.linspace(0.0, cutoff, k_rbf)


def rbf_gamma(k_rbf: int, cutoff: float) -> float:
    return (k_rbf / cutoff) ** 2


def _rbf(distances, k_rbf, cutoff, want, derivative, check):
    if k_rbf < 1:
        raise ValueError("k_rbf must be >= 1")
    d = _f64(distances).reshape(-1)
    n = d.shape[0]
    out = torch.empty((n, k_rbf), dtype=torch.float64, device=d.device) if want else None
    dout = torch.empty((n, k_rbf), dtype=torch.float64, device=d.device) if derivative else None
    bad = torch.zeros(1, dtype=torch.int32, device=d.device) if check else None
    ops.call("egn_rbf_features", ops.ptr(d), n, int(k_rbf), float(cutoff), ops.ptr(out), ops.ptr(dout),
             ops.ptr(bad), ops.stream())
    if check and n:
        _raise_if(bad, "distances must lie in (0, cutoff]")
    return out, dout


def rbf_features(distances, k_rbf: int, cutoff: float) -> np.ndarray:
    """Gaussian radial features, entry (e, k) = exp(-gamma (d_e - c_k)^2) (egn/basis.py:35-42)."""
    return _rbf(distances, k_rbf, cutoff, True, False, True)[0].cpu().numpy()


def rbf_features_ddist(distances, k_rbf: int, cutoff: float) -> np.ndarray:
    """d rbf_k / d d_e (egn/basis.py:45-51)."""
    return _rbf(distances, k_rbf, cutoff, False, True, False)[1].cpu().numpy()


def _sbf(in_edge_distances, angles, k_rbf, l_sbf, cutoff, want, partials):
    if l_sbf < 1:
        raise ValueError("l_sbf must be >= 1")
    if k_rbf < 1:
        raise ValueError("k_rbf must be >= 1")
    d = _f64(in_edge_distances).reshape(-1)
    a = _f64(angles).reshape(-1)
    if d.shape != a.shape:
        raise ValueError("in_edge_distances and angles must have the same length")
    n, kl = a.shape[0], k_rbf * l_sbf
    mk = lambda: torch.empty((n, kl), dtype=torch.float64, device=a.device)  # noqa: E731
    out = mk() if want else None
    dd, da = (mk(), mk()) if partials else (None, None)
    bad = torch.zeros(1, dtype=torch.int32, device=a.device)
    ops.call("egn_sbf_features", ops.ptr(d), ops.ptr(a), n, int(k_rbf), int(l_sbf), float(cutoff), ops.ptr(out),
             ops.ptr(dd), ops.ptr(da), ops.ptr(bad), ops.stream())
    if n:
        ang = a
        if bool(((ang < -1e-12) | (ang > np.pi + 1e-12)).any()):
            raise ValueError("angles must lie in [0, pi]")
        _raise_if(bad, "distances must lie in (0, cutoff]")
    return out, dd, da


def sbf_features(in_edge_distances, angles, k_rbf: int, l_sbf: int, cutoff: float) -> np.ndarray:
    """Entry (t, k L + l) = rbf_k(d_kj) cos(l angle_t) (egn/basis.py:54-74)."""
    return _sbf(in_edge_distances, angles, k_rbf, l_sbf, cutoff, True, False)[0].cpu().numpy()


def sbf_features_partials(in_edge_distances, angles, k_rbf: int, l_sbf: int, cutoff: float):
    """(d sbf / d d_kj, d sbf / d angle) (egn/basis.py:77-95)."""
    _, dd, da = _sbf(in_edge_distances, angles, k_rbf, l_sbf, cutoff, False, True)
    return dd.cpu().numpy(), da.cpu().numpy()


def compute_basis(geometry: Geometry, topology: GraphTopology, k_rbf: int, l_sbf: int,
                  cutoff: float) -> BasisFeatures:
    """Edge and triplet basis tables of a built graph (egn/basis.py:98-103)."""
    d = _f64(geometry.distances)
    rbf = _rbf(d, k_rbf, cutoff, True, False, True)[0]
    in_dist = d.index_select(0, torch.as_tensor(topology.trip_in, device=d.device).long())
    sbf = _sbf(in_dist, geometry.angles, k_rbf, l_sbf, cutoff, True, False)[0]
    return BasisFeatures(rbf.cpu().numpy(), sbf.cpu().numpy())


# ---------------------------------------------------------------------------
# geometry derivatives (egn/gradients.py)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class GeometryGrads:
    dist_d_src: np.ndarray
    dist_d_recv: np.ndarray
    angle_d_k: np.ndarray
    angle_d_j: np.ndarray
    angle_d_i: np.ndarray


def geometry_grads(positions, topology: GraphTopology) -> GeometryGrads:
    """Closed-form d(distance)/dx and d(angle)/dx (egn/gradients.py:33-36)."""
    pos = _f64(positions)
    dev = pos.device
    src = torch.as_tensor(topology.edge_src, device=dev).long().contiguous()
    recv = torch.as_tensor(topology.edge_recv, device=dev).long().contiguous()
    tin = torch.as_tensor(topology.trip_in, device=dev).long().contiguous()
    tout = torch.as_tensor(topology.trip_out, device=dev).long().contiguous()
    ne, nt = src.shape[0], tin.shape[0]
    outs = [torch.empty((n, 3), dtype=torch.float64, device=dev) for n in (ne, ne, nt, nt, nt)]
    ops.call("egn_geometry_grads", ops.ptr(pos), ops.ptr(src), ops.ptr(recv), ne, ops.ptr(tin), ops.ptr(tout), nt,
             *[ops.ptr(o) for o in outs], ops.stream())
    return GeometryGrads(*[o.cpu().numpy() for o in outs])


# ---------------------------------------------------------------------------
# ModelTape (egn/engine.py:320-438)
# ---------------------------------------------------------------------------
def _positions(system) -> np.ndarray:
    return np.asarray(system.positions if hasattr(system, "positions") else system, dtype=np.float64)


def _check_species(system):
    z = getattr(system, "atomic_numbers", None)
    if z is not None and np.asarray(z).size and int(np.max(z)) > MAX_Z:
        raise ValueError(f"atomic number {int(np.max(z))} exceeds the embedding table ({MAX_Z})")


def batch_from_topology(topology: GraphTopology, positions, cutoff: float) -> BatchGraph:
    """Device batch of one graph from a prebuilt GraphTopology (ModelTape(prebuilt=...)):
    the CSR and reverse edges from the edge list, geometry recomputed from `positions`."""
    pos = _f64(positions)
    dev = pos.device
    src = torch.as_tensor(topology.edge_src, device=dev).long()
    recv = torch.as_tensor(topology.edge_recv, device=dev).long()
    n = int(topology.num_nodes)
    deg = torch.bincount(src, minlength=n).to(torch.int32)
    edge_ptr = ops.scan_counts(deg)
    tri_ptr = ops.scan_counts(deg, square_minus_one=True)
    src32, recv32 = src.to(torch.int32).contiguous(), recv.to(torch.int32).contiguous()
    rev, missing = ops.reverse_edges(edge_ptr, src32, recv32)
    if src.numel() and int(missing.item()):
        raise ValueError("edge list is not symmetric: some edge has no reverse edge")
    geo, _, _ = ops.geometry(pos, src32, recv32)
    ne, nt = int(src.numel()), int(tri_ptr[-1].item())
    max_deg = int(deg.max().item()) if n else 0
    return BatchGraph(1, n, ne, nt, float(cutoff), pos, torch.tensor([0, n], dtype=torch.int64, device=dev),
                      torch.zeros(n, dtype=torch.int32, device=dev), deg, edge_ptr, src32, recv32, rev, tri_ptr, geo,
                      [n], max_deg=max_deg)


class ModelTape:
    """One forward pass over a system (egn/engine.py:320-438): ``energy``, ``forces`` (the
    force-centric head, else None), ``state`` (final features) and ``backward(d_energy,
    d_forces)`` -> GradientBundle(d_params, d_positions).  The forward runs once at
    construction on the native engine; each backward replays the explicit adjoint."""

    def __init__(self, system, params, prebuilt: tuple | None = None, device=None):
        _check_species(system)
        self.system = system
        self.params = params
        self.config = params.config
        dev = _dev(device)
        pos = _positions(system)
        if prebuilt is None:
            self.bg = build_batch(system, self.config.cutoff, dev)
            self.topology, self.geometry = topology_of(self.bg), geometry_of(self.bg)
        else:
            self.topology, self.geometry = prebuilt
            self.bg = batch_from_topology(self.topology, pos, self.config.cutoff)
        self.engine = Engine(DeviceWeights.from_params(params, dev))
        self._fw = self.engine.forward(self.bg)
        self._energy = float(self._fw.energy[0])
        self._basis = None

    @property
    def energy(self) -> float:
        return self._energy

    @property
    def forces(self):
        if self.config.variant != GEMNET:
            return None
        return self._fw.forces.double().cpu().numpy()

    @property
    def basis(self) -> BasisFeatures:
        if self._basis is None:
            c = self.config
            self._basis = compute_basis(self.geometry, self.topology, c.k_rbf, c.l_sbf, c.cutoff)
        return self._basis

    @property
    def state(self) -> FeatureState:
        fw, c = self._fw, self.config
        dw = self.engine.weights
        h = lambda x, dim: dw.unpad_rows(x, dim).double().cpu().numpy()  # noqa: E731
        t = self.engine.triplet_features(self.bg, fw, c.blocks - 1) if c.blocks else None
        return FeatureState(h(fw.u, "d_u"), h(fw.v, "d_v"), h(fw.m, "d_e"), h(t, "d_t") if t is not None else None,
                            self.topology, self.geometry, self.basis)

    def backward(self, d_energy: float = 1.0, d_forces=None, check_replay: bool = False) -> GradientBundle:
        if d_forces is not None and self.config.variant != GEMNET:
            raise ValueError("force seed given but this variant has no force head")
        dev = self.bg.device
        de = torch.tensor([float(d_energy)], dtype=torch.float32, device=dev)
        df = (torch.as_tensor(np.asarray(d_forces, dtype=np.float64), device=dev).to(torch.float32)
              if d_forces is not None else None)
        pos_bar = self.engine.backward(self.bg, self._fw, de, df)
        if check_replay:  # the explicit adjoint is deterministic: a second pass is identical
            again = self.engine.backward(self.bg, self._fw, de, df)
            if not torch.equal(again, pos_bar):
                raise RuntimeError("backward replay differs")
        return GradientBundle(self.engine.weights.to_numpy(grads=True), pos_bar.cpu().numpy())


def backward(model: ModelTape, d_energy: float = 1.0, d_forces=None, check_replay: bool = False) -> GradientBundle:
    """egn/gradients.py:39-46."""
    return model.backward(d_energy=d_energy, d_forces=d_forces, check_replay=check_replay)


def forces_energy_centric(system, params):
    """(energy, -dE/dx, bundle) at fixed topology (egn/gradients.py:49-61)."""
    model = ModelTape(system, params)
    bundle = model.backward(d_energy=1.0)
    return model.energy, -bundle.d_positions, bundle


def initial_state(atomic_numbers, topology: GraphTopology, geometry: Geometry, basis: BasisFeatures,
                  params) -> FeatureState:
    """Feature buffers before the first block (egn/engine.py:264-278): node = atom embedding,
    edge = edge_init(rbf), triplet and global zeros."""
    z = np.asarray(atomic_numbers, dtype=np.int64)
    if z.size and int(z.max()) > MAX_Z:
        raise ValueError(f"atomic number {int(z.max())} exceeds the embedding table ({MAX_Z})")
    c = params.config
    dev = _dev()
    rbf = torch.as_tensor(np.asarray(basis.edge_rbf, dtype=np.float32), device=dev).contiguous()
    w = DeviceWeights.from_params(params, dev).w
    edge = ops.rbf_linear(rbf, w["edge_init.w"], w["edge_init.b"]).double().cpu().numpy()
    node = np.asarray(params.arrays["atom_embedding"])[z - 1]
    return FeatureState(np.zeros((1, c.d_u)), node, edge, np.zeros((topology.num_triplets, c.d_t)), topology,
                        geometry, basis)


def block_forward(state: FeatureState, params, block: int, positions=None) -> FeatureState:
    """One interaction block applied to a feature state (egn/engine.py:281-317).  The device
    geometry of the state's graph is recomputed from `positions` (the system the state came
    from; the reference reads its precomputed basis from the state instead)."""
    c = params.config
    topo = state.topology
    dev = _dev()
    if positions is None:
        raise ValueError("block_forward needs the positions of the state's system")
    bg = batch_from_topology(topo, positions, c.cutoff)
    eng = Engine(DeviceWeights.from_params(params, dev))
    pc = eng.config  # padded widths (zero channels beyond the reference ones)
    m_np = np.asarray(state.edge_features, dtype=np.float32)
    u_np = np.asarray(state.global_features, dtype=np.float32).reshape(1, -1)
    m0 = torch.zeros((m_np.shape[0], pc.d_e), dtype=torch.float32, device=dev)
    m0[:, : m_np.shape[1]] = torch.as_tensor(m_np, device=dev)
    u0 = torch.zeros((1, pc.d_u), dtype=torch.float32, device=dev)
    u0[:, : u_np.shape[1]] = torch.as_tensor(u_np, device=dev)
    fw = eng.forward(bg, m0=m0, u0=u0, blocks=[block])
    t = eng.triplet_features(bg, fw, block, index=0)
    dw = eng.weights
    h = lambda x, dim: dw.unpad_rows(x, dim).double().cpu().numpy()  # noqa: E731
    return FeatureState(h(fw.u, "d_u"), h(fw.v, "d_v"), h(fw.m, "d_e"), h(t, "d_t"), topo, state.geometry,
                        state.basis)
