"""DimeNet++ / GemNet-T bases on the native kernels vs the fp64 oracle.

basis="bessel": radial Bessel RBF with the p=6 polynomial envelope on every edge; triplet basis
DimeNet SBF  sqrt(2/c^3)/|j_{l+1}(z_ln)| u(d/c) j_l(z_ln d/c) Y_l0(angle)  (basis code 2) or
GemNet CBF   e_k(d) Y_l0(angle)                                             (basis code 1),
restated in oracle/egn_oracle.py (bessel_rbf, sbf_bessel). The native kernels are segment.cu
(egn_rbf_bessel[_bwd]) and triplet_sh.cu (egn_triplet_fwd_basis / egn_triplet_bwd_basis).
Tolerance: fp32 kernels vs fp64 oracle, max-relative <= 1e-4 (TOL).
"""

import numpy as np
import pytest
import torch

from conftest import TOL, max_rel
from oracle import egn_oracle as O

pytestmark = pytest.mark.gpu

VARIANTS = {"dimenet-style": 2, "gemnet-style": 1}


def _ref(pos, cutoff, X, W, B, variant):
    """S = sum_t X[kj] * (basis_t @ W); adjoints of J = sum(S * B) in fp64 (oracle primitives)."""
    g = O.build_graph(pos, cutoff)
    K, L, dg = W.shape
    Wmat = W.reshape(K * L, dg)
    d_in = g.dist[g.trip_in]
    sb = O.sbf_bessel(d_in, g.angles, K, L, cutoff, variant)
    gt = sb @ Wmat
    S = O.segment_sum(X[g.trip_in] * gt, g.trip_out, g.src.size)
    Bt = B[g.trip_out]
    X_bar = O.scatter_rows(gt * Bt, g.trip_in, g.src.size)
    W_bar = (sb.T @ (X[g.trip_in] * Bt)).reshape(K, L, dg)
    sb_bar = (X[g.trip_in] * Bt) @ Wmat.T
    dd, da = O.sbf_bessel_partials(d_in, g.angles, K, L, cutoff, variant)
    dist_bar = np.zeros(g.src.size)
    np.add.at(dist_bar, g.trip_in, (sb_bar * dd).sum(1))
    ang_bar = (sb_bar * da).sum(1)
    pos_bar = np.zeros_like(pos)
    gk, gj, gi = O.angle_gradients(pos, g.src, g.recv, g.trip_in, g.trip_out)
    k, j, i = g.src[g.trip_in], g.recv[g.trip_in], g.recv[g.trip_out]
    np.add.at(pos_bar, k, ang_bar[:, None] * gk)
    np.add.at(pos_bar, i, ang_bar[:, None] * gi)
    np.add.at(pos_bar, j, ang_bar[:, None] * gj)
    c = dist_bar[:, None] * g.units
    np.add.at(pos_bar, g.recv, c)
    np.add.at(pos_bar, g.src, -c)
    return S, X_bar, W_bar, pos_bar


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("n,density,dg", [(40, 0.06, 64), (30, 0.06, 16), (24, 0.5, 8), (60, 0.3, 32)])
def test_triplet_basis_kernels_vs_oracle(variant, n, density, dg):
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    cutoff, K, L = 6.0, 6, 7
    rng = np.random.default_rng(n + dg)
    pos, _ = O.random_cloud(n, density, rng)
    bg = build_batch([pos], cutoff)
    X = rng.standard_normal((bg.num_edges, dg))
    W = rng.standard_normal((K, L, dg)) / np.sqrt(K * L)
    B = rng.standard_normal((bg.num_edges, dg))
    S_ref, Xb_ref, Wb_ref, pb_ref = _ref(pos, cutoff, X, W, B, variant)
    code = VARIANTS[variant]
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    Wd = torch.tensor(W, dtype=torch.float32, device="cuda")
    S = ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, Xd, Wd, cutoff, max_degree=bg.max_deg, basis=code)
    eg = torch.zeros((bg.num_edges, 4), device="cuda")
    Xb, Wb = ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, Xd, Wd, cutoff,
                             torch.tensor(B, dtype=torch.float32, device="cuda"), eg, max_degree=bg.max_deg,
                             basis=code)
    pb = ops.positions_bwd(bg.edge_ptr, bg.rev, bg.geo, eg)
    torch.cuda.synchronize()
    assert max_rel(S.cpu().numpy(), S_ref) < TOL
    assert max_rel(Xb.cpu().numpy(), Xb_ref) < TOL
    assert max_rel(Wb.cpu().numpy(), Wb_ref) < TOL
    assert max_rel(pb.cpu().numpy(), pb_ref) < TOL


def test_triplet_basis_dimension_errors():
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    rng = np.random.default_rng(0)
    pos, _ = O.random_cloud(12, 0.3, rng)
    bg = build_batch([pos], 6.0)
    X = torch.zeros((bg.num_edges, 8), device="cuda")
    with pytest.raises(ValueError, match="k_rbf = 6, l_sbf = 7"):
        ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X, torch.zeros((6, 4, 8), device="cuda"), 6.0,
                        max_degree=bg.max_deg, basis=2)
    with pytest.raises(ValueError, match="basis must be"):
        ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X, torch.zeros((6, 7, 8), device="cuda"), 6.0,
                        max_degree=bg.max_deg, basis=5)


@pytest.mark.parametrize("k", [6, 8])
def test_bessel_rbf_and_adjoint_vs_oracle(k):
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    cutoff = 5.0
    rng = np.random.default_rng(k)
    pos, _ = O.random_cloud(50, 0.2, rng)
    bg = build_batch([pos], cutoff)
    g = O.build_graph(pos, cutoff)
    r = ops.rbf(bg.geo, k, cutoff, basis=1).cpu().numpy()
    assert max_rel(r, O.bessel_rbf(g.dist, k, cutoff)) < TOL
    rb = rng.standard_normal((bg.num_edges, k))
    eg = torch.zeros((bg.num_edges, 4), device="cuda")
    ops.rbf_bwd(bg.geo, torch.tensor(rb, dtype=torch.float32, device="cuda"), cutoff, eg, basis=1)
    pb = ops.positions_bwd(bg.edge_ptr, bg.rev, bg.geo, eg).cpu().numpy()
    dist_bar = (rb * O.bessel_rbf_ddist(g.dist, k, cutoff)).sum(1)
    ref = np.zeros_like(pos)
    c = dist_bar[:, None] * g.units
    np.add.at(ref, g.recv, c)
    np.add.at(ref, g.src, -c)
    assert max_rel(pb, ref) < TOL


def _model_vs_oracle(cfg, systems, rng, eng_factory):
    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.graph import build_batch

    params = init_params(cfg)
    eng = eng_factory(params)
    bg = build_batch([s[0] for s in systems], cfg.cutoff)
    fw = eng.forward(bg)
    de = rng.standard_normal(len(systems))
    dfs = [rng.standard_normal(s[0].shape) for s in systems] if cfg.variant == "gemnet-style" else None
    pos_bar = eng.backward(bg, fw, torch.tensor(de, dtype=torch.float32, device="cuda"),
                           torch.tensor(np.concatenate(dfs), device="cuda") if dfs else None).cpu().numpy()
    grads = eng.weights.to_numpy(grads=True)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    ref_g = {k: np.zeros_like(v) for k, v in params.arrays.items()}
    off = 0
    for i, (pos, z) in enumerate(systems):
        f = O.forward(oc, params.arrays, pos, z)
        G, dp = O.backward(f, params.arrays, float(de[i]), dfs[i] if dfs else None)
        n = pos.shape[0]
        assert abs(float(fw.energy[i]) - f.energy) <= TOL * max(abs(f.energy), 1e-8)
        assert max_rel(pos_bar[off:off + n], dp) < TOL
        if cfg.variant == "gemnet-style":
            assert max_rel(fw.forces[off:off + n].cpu().numpy(), f.forces) < TOL
        for k in ref_g:
            ref_g[k] += G[k]
        off += n
    for k, g in ref_g.items():
        assert max_rel(grads[k], g) < TOL, k


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_model_on_bessel_bases_vs_oracle(variant):
    """The whole DimeNet++ / GemNet-T-style model on the published bases: energy, forces, dL/dx
    and every parameter gradient vs the fp64 oracle (O.forward / O.backward, basis="bessel")."""
    from paper_2203_09697_b200 import ModelConfig
    from paper_2203_09697_b200.engine import DeviceWeights, Engine

    cfg = ModelConfig(variant=variant, blocks=2, d_u=32, d_v=32, d_e=64, d_t=32, d_bil=64, k_rbf=6, l_sbf=7,
                      cutoff=6.0, seed=3, basis="bessel")
    rng = np.random.default_rng(29)
    systems = [O.random_cloud(n, 0.06, rng) for n in (21, 34, 16)]
    _model_vs_oracle(cfg, systems, rng, lambda p: Engine(DeviceWeights.from_params(p)))


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_bessel_model_padded_widths_vs_oracle(variant):
    """Unaligned widths (zero-padded to 16 inside DeviceWeights) on the bessel bases."""
    from paper_2203_09697_b200 import ModelConfig
    from paper_2203_09697_b200.engine import DeviceWeights, Engine

    cfg = ModelConfig(variant=variant, blocks=1, d_u=20, d_v=24, d_e=40, d_t=18, d_bil=24, k_rbf=6, l_sbf=7,
                      cutoff=5.0, seed=5, basis="bessel")
    rng = np.random.default_rng(31)
    systems = [O.random_cloud(n, 0.1, rng) for n in (19, 25)]
    _model_vs_oracle(cfg, systems, rng, lambda p: Engine(DeviceWeights.from_params(p)))


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_bessel_centre_schedule_two_ranks_vs_oracle(variant):
    """The graph-parallel centre schedule (two in-process ranks) on the bessel bases."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg = ModelConfig(variant=variant, blocks=2, d_u=32, d_v=32, d_e=32, d_t=32, d_bil=32, k_rbf=6, l_sbf=7,
                      cutoff=6.0, seed=8, basis="bessel", workers=2)
    params = init_params(cfg)
    rng = np.random.default_rng(41)
    pos, z = O.random_cloud(30, 0.06, rng)
    from paper_2203_09697_b200.system import AtomicSystem

    wg = WorkerGroup(AtomicSystem(pos, z), params, schedule="centre")
    res = wg.forward()
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    f = O.forward(oc, params.arrays, pos, z)
    assert abs(float(res.energy) - f.energy) <= TOL * max(abs(f.energy), 1e-8)
    if variant == "gemnet-style":
        assert max_rel(np.asarray(res.forces), f.forces) < TOL
    de = 0.7
    df = rng.standard_normal(pos.shape) if variant == "gemnet-style" else None
    res, gb = wg.forward_backward(de, df)
    G, _ = O.backward(f, params.arrays, de, df)
    for k, g in G.items():
        assert max_rel(np.asarray(gb.d_params[k]), g) < TOL, k
    with pytest.raises(ValueError, match="Gaussian basis only"):
        WorkerGroup(AtomicSystem(pos, z), params, schedule="reference")


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_bessel_bases_on_periodic_cells_vs_oracle(variant):
    """The Bessel bases on periodic graphs (edges to images, §8(f) f1 x f2): energies, forces,
    every d_param and d_positions vs the oracle on the same periodic graph."""
    from paper_2203_09697_b200 import AtomicSystem, ModelConfig, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig(variant=variant, blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, k_rbf=6, l_sbf=7,
                      cutoff=3.0, seed=4, basis="bessel")
    params = init_params(cfg)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    rng = np.random.default_rng(23)
    cells = [np.array([[4.2, 0, 0], [0.5, 4.0, 0], [0.3, 0.2, 4.4]]), np.array([[5.0, 0, 0], [0, 5.0, 0], [0, 0, 30.0]])]
    pbcs = [(True, True, True), (True, True, False)]
    systems = []
    for cell, pbc, n in zip(cells, pbcs, (5, 8)):
        systems.append(AtomicSystem(rng.uniform(0, 1, (n, 3)) @ cell, np.full(n, 6), cell=cell, pbc=pbc))
    eng = Engine(DeviceWeights.from_params(params))
    bg = build_batch(systems, cfg.cutoff)
    fw = eng.forward(bg)
    d_e = torch.tensor([0.6, -0.9], device="cuda")
    df_np = [rng.standard_normal((s.n, 3)) for s in systems] if variant == "gemnet-style" else None
    pos_bar = eng.backward(bg, fw, d_e, torch.tensor(np.concatenate(df_np), device="cuda") if df_np else None)
    pos_bar = pos_bar.cpu().numpy()
    grads = eng.weights.to_numpy(grads=True)
    ref_g = {k: np.zeros_like(v) for k, v in params.arrays.items()}
    off = 0
    for i, s in enumerate(systems):
        f = O.forward(oc, params.arrays, s.positions, s.atomic_numbers,
                      graph=O.build_graph_pbc(s.positions, s.cell, s.pbc, cfg.cutoff))
        G, dp = O.backward(f, params.arrays, float(d_e[i]), df_np[i] if df_np else None)
        assert abs(float(fw.energy[i]) - f.energy) <= TOL * max(abs(f.energy), 1e-8)
        assert max_rel(pos_bar[off:off + s.n], dp) < TOL
        for k in ref_g:
            ref_g[k] += G[k]
        off += s.n
    for k, g in ref_g.items():
        assert max_rel(grads[k], g) < TOL, k


def test_bessel_captured_trainer_with_isolated_atoms(monkeypatch):
    """The captured multi-stream training step (bench path) on the Bessel bases over a batch
    with an isolated atom and a two-atom graph (no triplets) next to an ordinary graph: the
    loss and every gradient equal the oracle's loss_and_grads."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    monkeypatch.setenv("EGN_SIDE_MIN_EDGES", "0")
    cfg = ModelConfig(variant="gemnet-style", blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, k_rbf=6,
                      l_sbf=7, cutoff=5.0, seed=6, basis="bessel")
    params = init_params(cfg)
    rng = np.random.default_rng(5)
    systems = [np.zeros((1, 3)), np.array([[0.0, 0.0, 0.0], [1.1, 0.2, -0.3]]), O.random_cloud(20, 0.1, rng)[0]]
    e_t = rng.standard_normal(3)
    f_t = np.concatenate([rng.standard_normal((s.shape[0], 3)) for s in systems])
    tr = Trainer(params, None, e_t, f_t, 1.0, 0.5, graph=build_batch(systems, cfg.cutoff), cuda_graph=True)
    tr.step(0.0)
    loss = float(tr.step(0.0))
    grads = tr.weights.to_numpy(grads=True)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    z = [np.full(s.shape[0], 6) for s in systems]
    loss_ref, g_ref = O.loss_and_grads(oc, params.arrays, [(s, zz, e, f) for s, zz, e, f in
                                                           zip(systems, z, e_t, np.split(f_t, np.cumsum(
                                                               [s.shape[0] for s in systems])[:-1]))],
                                       w_energy=1.0, w_forces=0.5)
    assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
    for k, g in g_ref.items():
        assert max_rel(grads[k], g) < TOL, k
