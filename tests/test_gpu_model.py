"""Whole-model parity on the GPU: energies, forces, every parameter gradient and
the position gradient vs the reference (golden fixtures) and the fp64 oracle.

Tolerance (north star): per tensor max|a-b| / max(max|b|, 1e-8) <= 1e-4.
"""

import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN, TOL, load_golden, max_rel
from oracle import egn_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["default", "tcgen05"], autouse=True)
def gemm_path(request, monkeypatch):
    """Every model test runs twice: the default dispatch (node-row and small products on the
    SIMT GEMM, one stream below EGN_SIDE_MIN_EDGES edges) and with every product forced onto
    the tcgen05 3xTF32 GEMM (egn_gemm_simt_max_m = 0) and the three-stream schedule forced on
    (EGN_SIDE_MIN_EDGES = 0) -- the code path the bench step runs at M = 58,644."""
    from paper_2203_09697_b200 import _lib

    if request.param == "default":
        yield request.param
        return
    monkeypatch.setenv("EGN_SIDE_MIN_EDGES", "0")
    old = _lib.call("egn_gemm_simt_max_m", 0)
    try:
        yield request.param
    finally:
        _lib.call("egn_gemm_simt_max_m", old)

SMALL = ["model_dimenet_small.npz", "model_gemnet_small.npz", "model_gemnet_odd.npz", "model_dimenet_chain.npz"]
LARGE = ["model_dimenet_c1dims.npz", "model_gemnet_c2dims.npz"]


def _setup(gd):
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig.from_json(str(gd["config"]))
    params = init_params(cfg)
    eng = Engine(DeviceWeights.from_params(params))
    bg = build_batch([gd["pos"]], cfg.cutoff)
    return cfg, params, eng, bg


@pytest.mark.parametrize("fname", SMALL + LARGE)
def test_model_matches_reference_golden(fname):
    gd = load_golden(fname)
    cfg, params, eng, bg = _setup(gd)
    fw = eng.forward(bg)
    d_forces = gd.get("d_forces")
    df = torch.tensor(d_forces, device="cuda") if d_forces is not None else None
    pos_bar = eng.backward(bg, fw, torch.tensor([0.7], device="cuda"), df)
    grads = eng.weights.to_numpy(grads=True)
    e_ref = float(gd["energy"])
    assert abs(float(fw.energy[0]) - e_ref) <= TOL * max(abs(e_ref), 1e-8)
    dw = eng.weights  # padded widths (non-tile dims) -> reference channels
    assert max_rel(dw.unpad_rows(fw.m, "d_e").cpu().numpy(), gd["m"]) < TOL
    assert max_rel(dw.unpad_rows(fw.v, "d_v").cpu().numpy(), gd["v"]) < TOL
    assert max_rel(dw.unpad_rows(fw.u, "d_u").cpu().numpy(), gd["u"]) < TOL
    assert max_rel(pos_bar.cpu().numpy(), gd["d_positions"]) < TOL
    if cfg.variant == "gemnet-style":
        assert max_rel(fw.forces.cpu().numpy(), gd["forces"]) < TOL
    t_feat = dw.unpad_rows(eng.triplet_features(bg, fw, cfg.blocks - 1), "d_t").cpu().numpy()
    assert max_rel(t_feat, gd["t_feat"]) < TOL
    for name in gd["param_names"]:
        name = str(name)
        if f"dp/{name}" in gd:
            assert max_rel(grads[name], gd[f"dp/{name}"]) < TOL, name
        else:
            ref_head = gd[f"dphead/{name}"]
            scale = max(float(gd[f"dpnorm/{name}"]), 1e-8)
            assert np.abs(grads[name].ravel()[:64] - ref_head).max() / scale < TOL, name


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_full_dims_batched_vs_oracle(variant):
    """C1/C2 model dims, a batch of 3 OC20-density graphs; every d_param vs the live oracle."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig(variant=variant, blocks=4, d_u=128, d_v=128, d_e=128, d_t=64, d_bil=64, k_rbf=6,
                      l_sbf=7, cutoff=6.0, seed=0)
    params = init_params(cfg)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    rng = np.random.default_rng(11)
    systems = [O.random_cloud(n, 0.06, rng) for n in (20, 33, 27)]
    eng = Engine(DeviceWeights.from_params(params))
    bg = build_batch([s[0] for s in systems], cfg.cutoff)
    fw = eng.forward(bg)
    d_e = torch.tensor([0.3, -1.1, 0.6], device="cuda")
    df = None
    df_np = []
    if variant == "gemnet-style":
        df_np = [rng.standard_normal((s[0].shape[0], 3)) for s in systems]
        df = torch.tensor(np.concatenate(df_np), device="cuda")
    pos_bar = eng.backward(bg, fw, d_e, df).cpu().numpy()
    grads = eng.weights.to_numpy(grads=True)
    ref_g = {k: np.zeros_like(v) for k, v in params.arrays.items()}
    off = 0
    for i, (pos, z) in enumerate(systems):
        f = O.forward(oc, params.arrays, pos, z)
        G, dp = O.backward(f, params.arrays, float(d_e[i]), df_np[i] if df_np else None)
        n = pos.shape[0]
        assert abs(float(fw.energy[i]) - f.energy) <= TOL * max(abs(f.energy), 1e-8)
        assert max_rel(pos_bar[off:off + n], dp) < TOL
        if variant == "gemnet-style":
            assert max_rel(fw.forces[off:off + n].cpu().numpy(), f.forces) < TOL
        for k in ref_g:
            ref_g[k] += G[k]
        off += n
    for k in ref_g:
        assert max_rel(grads[k], ref_g[k]) < TOL, k


def test_nn_module_autograd_path():
    from paper_2203_09697_b200 import EGNModel, ModelConfig, init_params

    cfg = ModelConfig(variant="gemnet-style", blocks=2, seed=2)
    params = init_params(cfg)
    model = EGNModel(cfg, params)
    assert list(model.state_dict().keys()) == [s for s in params.arrays]
    pos, z = O.random_cloud(12, 0.9, np.random.default_rng(2))
    energy, forces = model([pos])
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    f = O.forward(oc, params.arrays, pos, z)
    assert abs(float(energy[0].detach()) - f.energy) <= TOL * max(1.0, abs(f.energy))
    w = torch.tensor(np.random.default_rng(1).standard_normal((12, 3)), device="cuda", dtype=torch.float32)
    loss = 0.5 * energy.sum() + (forces * w).sum()
    loss.backward()
    G, _ = O.backward(f, params.arrays, 0.5, w.double().cpu().numpy())
    for name, p in model.named_parameters():
        assert max_rel(model.weights.unpad(name, p.grad.double().cpu().numpy()), G[name]) < TOL, name


def test_dimenet_predict_forces_and_force_loss_error():
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.tasks import loss_and_grads, predict

    cfg = ModelConfig(variant="dimenet-style", blocks=2, seed=1)
    params = init_params(cfg)
    pos, z = O.random_cloud(10, 0.9, np.random.default_rng(4))
    e, f = predict(pos, params)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    e_ref, f_ref = O.predict(oc, params.arrays, pos, z)
    assert abs(e - e_ref) <= TOL * max(1.0, abs(e_ref))
    assert max_rel(f, f_ref) < TOL
    # net force and torque vanish (translation/rotation invariance, test_gradients.py:128-135)
    assert np.abs(f.sum(0)).max() < 1e-4 * np.abs(f).max()
    with pytest.raises(ValueError):
        loss_and_grads([(pos, 0.0, np.zeros((10, 3)))], params, w_forces=1.0)


@pytest.mark.parametrize("variant", ["dimenet", "gemnet"])
def test_loss_and_grads_and_training_match_reference(variant):
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.tasks import loss_and_grads, train_simple

    gd = load_golden(f"train_{variant}.npz")
    cfg = ModelConfig.from_json(str(gd["config"]))
    params = init_params(cfg)
    data = [(gd[f"pos{i}"], float(gd[f"e{i}"]), gd[f"f{i}"]) for i in range(3)]
    w_f = float(gd["w_forces"])
    loss, grads = loss_and_grads(data, params, 1.0, w_f)
    assert abs(loss - float(gd["loss"])) <= TOL * abs(float(gd["loss"]))
    for k, g in grads.items():
        assert max_rel(g, gd[f"grad/{k}"]) < TOL, k
    _, hist = train_simple(data, params, lr=0.002, epochs=4, w_energy=1.0, w_forces=w_f)
    assert max_rel(np.array(hist), gd["history"]) < 1e-3
    assert hist[-1] < hist[0]


def test_rigid_motion_invariance():
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.tasks import predict

    cfg = ModelConfig(variant="gemnet-style", blocks=2, seed=3)
    params = init_params(cfg)
    rng = np.random.default_rng(9)
    pos, _ = O.random_cloud(14, 0.9, rng)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    e0, f0 = predict(pos, params)
    e1, f1 = predict(pos @ q.T + 3.0, params)
    assert abs(e0 - e1) < 1e-4 * max(1.0, abs(e0))
    assert max_rel(f1, f0 @ q.T) < 1e-3


XL = {
    # C3 DimeNet++-XL (d_e 2048, d_v = d_u 1536, d_t 256) and C4 GemNet-XL
    # (d_v = d_u 2320, d_e 1302 -> zero-padded to 1312 for the tcgen05 tiling, d_t 512,
    # d_bil 288 > 256: channel-chunked triplet kernels), 2 blocks, small graph
    "c3-dimenet-xl": dict(variant="dimenet-style", blocks=2, d_u=1536, d_v=1536, d_e=2048, d_t=256, d_bil=64),
    "c4-gemnet-xl": dict(variant="gemnet-style", blocks=2, d_u=2320, d_v=2320, d_e=1302, d_t=512, d_bil=288),
}


@pytest.mark.parametrize("name", sorted(XL))
def test_xl_dims_batch_over_8k_edges(name):
    """C3/C4 widths on a batch above the SIMT threshold (> 8192 edges: every edge product on
    the tcgen05 GEMM, d_e = 1302 padded), one block, vs the fp64 oracle per graph."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig(k_rbf=6, l_sbf=7, cutoff=6.0, seed=9, **{**XL[name], "blocks": 1})
    params = init_params(cfg)
    rng = np.random.default_rng(31)
    systems = [O.random_cloud(80, 0.06, rng) for _ in range(6)]
    eng = Engine(DeviceWeights.from_params(params))
    assert eng.weights.config.d_e % 16 == 0
    bg = build_batch([s[0] for s in systems], cfg.cutoff)
    assert bg.num_edges > 8192
    fw = eng.forward(bg)
    gem = cfg.variant == "gemnet-style"
    de = rng.standard_normal(len(systems))
    dfs = [rng.standard_normal(s[0].shape) for s in systems] if gem else None
    pos_bar = eng.backward(bg, fw, torch.tensor(de, device="cuda"),
                           torch.tensor(np.concatenate(dfs), device="cuda") if gem else None).cpu().numpy()
    grads = eng.weights.to_numpy(grads=True)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    ref_g = {k: np.zeros_like(v) for k, v in params.arrays.items()}
    off = 0
    for i, (pos, z) in enumerate(systems):
        f = O.forward(oc, params.arrays, pos, z)
        G, dp = O.backward(f, params.arrays, float(de[i]), dfs[i] if gem else None)
        n = pos.shape[0]
        assert abs(float(fw.energy[i]) - f.energy) <= TOL * max(abs(f.energy), 1e-8)
        assert max_rel(pos_bar[off:off + n], dp) < TOL
        if gem:
            assert max_rel(fw.forces[off:off + n].double().cpu().numpy(), f.forces) < TOL
        for k in ref_g:
            ref_g[k] += G[k]
        off += n
    for k, g in ref_g.items():
        assert max_rel(grads[k], g) < TOL, k


@pytest.mark.parametrize("name", sorted(XL))
def test_xl_dims_match_oracle(name):
    """SURVEY 8(d) C3/C4 widths on a 14-atom graph vs the fp64 oracle (energy, forces,
    every parameter gradient, position gradient)."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig(k_rbf=6, l_sbf=7, cutoff=6.0, seed=4, **XL[name])
    params = init_params(cfg)
    pos, z = O.random_cloud(14, 0.06, np.random.default_rng(21))
    eng = Engine(DeviceWeights.from_params(params))
    bg = build_batch([pos], cfg.cutoff)
    fw = eng.forward(bg)
    gem = cfg.variant == "gemnet-style"
    df = np.random.default_rng(3).standard_normal(pos.shape) if gem else None
    pos_bar = eng.backward(bg, fw, torch.tensor([0.9], device="cuda"),
                           torch.tensor(df, device="cuda") if gem else None)
    grads = eng.weights.to_numpy(grads=True)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    ofw = O.forward(oc, params.arrays, pos, z)
    G, dpos = O.backward(ofw, params.arrays, 0.9, df)
    assert abs(float(fw.energy[0]) - ofw.energy) <= TOL * max(abs(ofw.energy), 1e-8)
    if gem:
        assert max_rel(fw.forces.double().cpu().numpy(), ofw.forces) < TOL
    assert max_rel(pos_bar.cpu().numpy(), dpos) < TOL
    for k, g in G.items():
        assert max_rel(grads[k], g) < TOL, k


def test_cuda_graph_step_equals_eager_step():
    """Trainer(cuda_graph=True) captures the whole SGD step once and replays it; four
    steps must reproduce the eager trainer bit for bit (same kernels, same order),
    including after update_inputs() swaps positions/targets in place."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    cfg = ModelConfig(variant="gemnet-style", blocks=2, d_u=32, d_v=32, d_e=64, d_t=64, d_bil=64, k_rbf=6,
                      l_sbf=7, cutoff=6.0, seed=6)
    params = init_params(cfg)
    rng = np.random.default_rng(12)
    systems = [O.random_cloud(n, 0.06, rng)[0] for n in (22, 31)]
    e_t = rng.standard_normal(2)
    f_t = np.concatenate([rng.standard_normal((s.shape[0], 3)) for s in systems])
    runs = []
    for graph_mode in (False, True):
        tr = Trainer(params, None, e_t, f_t, 1.0, 0.3, graph=build_batch(systems, cfg.cutoff), cuda_graph=graph_mode)
        losses = [float(tr.step(1e-6)) for _ in range(3)]
        pos = tr.bg.pos.clone() * 1.01
        tr.update_inputs(pos, tr.e_target * 0.5, tr.f_target)
        losses.append(float(tr.step(1e-6)))
        runs.append((losses, tr.weights.flat.clone()))
    (l0, w0), (l1, w1) = runs
    assert all(np.isfinite(l0)) and l0[1] != l0[0] and l0[3] != l0[2]
    assert l0 == l1
    assert torch.equal(w0, w1)


@pytest.mark.parametrize("variant", ["dimenet", "gemnet"])
def test_relax_matches_reference(variant):
    """GPU relax (graph rebuilt on the device per evaluation) vs the reference trajectory:
    same accept / reject decisions and step count, positions / energies / max |F| within
    the parity tolerance."""
    from paper_2203_09697_b200 import AtomicSystem, ModelConfig, init_params
    from paper_2203_09697_b200.tasks import relax

    gd = load_golden(f"relax_{variant}.npz")
    cfg = ModelConfig.from_json(str(gd["config"]))
    params = init_params(cfg)
    system = AtomicSystem(gd["pos"], gd["z"])
    res = relax(system, params, float(gd["fmax_threshold"]), int(gd["max_steps"]), float(gd["step_size"]))
    assert res.steps == int(gd["steps"]) and res.converged == bool(gd["converged"])
    traj = np.stack(res.trajectory)
    assert traj.shape == gd["trajectory"].shape
    assert max_rel(traj, gd["trajectory"]) < TOL
    assert max_rel(np.array(res.energies), gd["energies"]) < TOL
    assert max_rel(np.array(res.max_forces), gd["max_forces"]) < TOL
    if variant == "dimenet":  # energy guard: rejected steps repeat the energy exactly
        e = np.array(res.energies)
        assert np.sum(np.diff(e) == 0) == int(np.sum(np.diff(gd["energies"]) == 0))
        assert np.all(np.diff(e) <= 0)


def test_relax_edge_cases():
    from paper_2203_09697_b200 import AtomicSystem, ModelConfig, init_params
    from paper_2203_09697_b200.tasks import relax

    gd = load_golden("relax_gemnet.npz")
    params = init_params(ModelConfig.from_json(str(gd["config"])))
    system = AtomicSystem(gd["pos"], gd["z"])
    with pytest.raises(ValueError):
        relax(system, params, 0.0)
    with pytest.raises(ValueError):
        relax(system, params, 1e-3, max_steps=-1)
    done = relax(system, params, 1e9)  # already converged: zero steps
    assert done.converged and done.steps == 0 and len(done.trajectory) == 1
    capped = relax(system, params, 1e-12, max_steps=2)
    assert not capped.converged and capped.steps == 2 and len(capped.trajectory) == 3
    with pytest.raises(ValueError):
        relax(system, init_params(ModelConfig(diagnostic=True)), 1e-3)


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_periodic_model_vs_oracle(variant):
    """Model on periodic graphs (images within the cutoff): energies, forces,
    every d_param and d_positions vs the fp64 oracle run on the same periodic graph."""
    from paper_2203_09697_b200 import AtomicSystem, ModelConfig, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig(variant=variant, blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, k_rbf=6, l_sbf=7,
                      cutoff=3.0, seed=2)
    params = init_params(cfg)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    rng = np.random.default_rng(21)
    cells = [np.array([[4.0, 0, 0], [0.6, 3.9, 0], [0.2, 0.4, 4.1]]), np.array([[5.0, 0, 0], [0, 5.0, 0], [0, 0, 30.0]])]
    pbcs = [(True, True, True), (True, True, False)]
    systems = []
    for cell, pbc, n in zip(cells, pbcs, (6, 9)):
        pos = rng.uniform(0, 1, (n, 3)) @ cell
        systems.append(AtomicSystem(pos, np.full(n, 6), cell=cell, pbc=pbc))
    eng = Engine(DeviceWeights.from_params(params))
    bg = build_batch(systems, cfg.cutoff)
    fw = eng.forward(bg)
    d_e = torch.tensor([0.8, -0.4], device="cuda")
    df_np = [rng.standard_normal((s.n, 3)) for s in systems] if variant == "gemnet-style" else None
    df = torch.tensor(np.concatenate(df_np), device="cuda") if df_np else None
    pos_bar = eng.backward(bg, fw, d_e, df).cpu().numpy()
    grads = eng.weights.to_numpy(grads=True)
    ref_g = {k: np.zeros_like(v) for k, v in params.arrays.items()}
    off = 0
    for i, s in enumerate(systems):
        g = O.build_graph_pbc(s.positions, s.cell, s.pbc, cfg.cutoff)
        f = O.forward(oc, params.arrays, s.positions, s.atomic_numbers, graph=g)
        G, dp = O.backward(f, params.arrays, float(d_e[i]), df_np[i] if df_np else None)
        n = s.n
        assert abs(float(fw.energy[i]) - f.energy) <= TOL * max(abs(f.energy), 1e-8)
        assert max_rel(pos_bar[off:off + n], dp) < TOL
        if variant == "gemnet-style":
            assert max_rel(fw.forces[off:off + n].cpu().numpy(), f.forces) < TOL
        for k in ref_g:
            ref_g[k] += G[k]
        off += n
    for k in ref_g:
        assert max_rel(grads[k], ref_g[k]) < TOL, k


def test_periodic_lattice_translation_invariance():
    """Moving an atom by a lattice vector changes nothing physical."""
    from paper_2203_09697_b200 import AtomicSystem, ModelConfig, init_params
    from paper_2203_09697_b200.tasks import predict

    cfg = ModelConfig(variant="gemnet-style", blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, k_rbf=6, l_sbf=7,
                      cutoff=3.0, seed=3)
    params = init_params(cfg)
    cell = np.array([[4.2, 0, 0], [0.5, 4.0, 0], [0.3, 0.2, 4.4]])
    pos = np.random.default_rng(8).uniform(0, 1, (7, 3)) @ cell
    e0, f0 = predict(AtomicSystem(pos, np.full(7, 6), cell=cell, pbc=(True, True, True)), params)
    moved = pos.copy()
    moved[2] += cell[0] - cell[2]
    moved[5] -= cell[1]
    e1, f1 = predict(AtomicSystem(moved, np.full(7, 6), cell=cell, pbc=(True, True, True)), params)
    assert abs(e1 - e0) <= 1e-5 * max(abs(e0), 1.0)
    assert max_rel(f1, f0) < 1e-4


def test_adamw_step_matches_torch_and_numpy():
    """egn_adamw vs torch.optim.AdamW (fp32) and an fp64 numpy restatement over 5 steps."""
    from paper_2203_09697_b200 import ops

    g0 = torch.Generator(device="cuda").manual_seed(5)
    n = 100_003
    w = torch.randn(n, device="cuda", generator=g0)
    w_ref = w.clone().requires_grad_(True)
    m = torch.zeros_like(w)
    v = torch.zeros_like(w)
    opt = torch.optim.AdamW([w_ref], lr=3e-3, betas=(0.9, 0.99), eps=1e-7, weight_decay=0.05)
    wn = w.double().cpu().numpy()
    mn = np.zeros(n)
    vn = np.zeros(n)
    for t in range(1, 6):
        grad = torch.randn(n, device="cuda", generator=g0)
        ops.adamw_(w, grad, m, v, 3e-3, t, (0.9, 0.99), 1e-7, 0.05)
        w_ref.grad = grad.clone()
        opt.step()
        gn = grad.double().cpu().numpy()
        wn = wn * (1 - 3e-3 * 0.05)
        mn = 0.9 * mn + 0.1 * gn
        vn = 0.99 * vn + 0.01 * gn * gn
        wn = wn - 3e-3 / (1 - 0.9 ** t) * mn / (np.sqrt(vn) / np.sqrt(1 - 0.99 ** t) + 1e-7)
    assert max_rel(w.cpu().numpy(), w_ref.detach().cpu().numpy()) < 1e-6
    assert max_rel(w.cpu().numpy(), wn) < 1e-5


def test_trainer_adamw_reduces_loss():
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.tasks import Trainer

    gd = load_golden("train_gemnet.npz")
    cfg = ModelConfig.from_json(str(gd["config"]))
    systems = [gd[f"pos{i}"] for i in range(3)]
    e_t = [float(gd[f"e{i}"]) for i in range(3)]
    f_t = np.concatenate([gd[f"f{i}"] for i in range(3)])
    tr = Trainer(init_params(cfg), systems, e_t, f_t, 1.0, 0.5, optimizer="adamw", adamw={"weight_decay": 0.0})
    losses = [float(tr.step(1e-3)) for _ in range(8)]
    assert losses[-1] < losses[0]
    with pytest.raises(ValueError):
        Trainer(init_params(cfg), systems, e_t, f_t, 1.0, 0.5, optimizer="lamb")


def test_capped_graph_model_vs_oracle():
    """Model on a max_neighbors-capped graph vs the fp64 oracle on the same capped graph."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig(variant="gemnet-style", blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, k_rbf=6, l_sbf=7,
                      cutoff=4.5, seed=6)
    params = init_params(cfg)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    pos, z = O.random_cloud(30, 0.2, np.random.default_rng(17))
    g = O.cap_graph(O.build_graph(pos, cfg.cutoff), pos, 6)
    f = O.forward(oc, params.arrays, pos, z, graph=g)
    df = np.random.default_rng(1).standard_normal((30, 3))
    G, dp = O.backward(f, params.arrays, 0.7, df)
    eng = Engine(DeviceWeights.from_params(params))
    bg = build_batch(pos, cfg.cutoff, max_neighbors=6)
    fw = eng.forward(bg)
    pos_bar = eng.backward(bg, fw, torch.tensor([0.7], device="cuda"), torch.tensor(df, device="cuda"))
    grads = eng.weights.to_numpy(grads=True)
    assert abs(float(fw.energy[0]) - f.energy) <= TOL * max(abs(f.energy), 1e-8)
    assert max_rel(fw.forces.cpu().numpy(), f.forces) < TOL
    assert max_rel(pos_bar.cpu().numpy(), dp) < TOL
    for k in G:
        assert max_rel(grads[k], G[k]) < TOL, k


@pytest.mark.gpu
@pytest.mark.parametrize("with_forces", [False, True])
def test_loss_seeds_match_reference_formula(with_forces):
    """egn_loss_seeds against egn/tasks.py:166-176 evaluated in numpy fp64."""
    from paper_2203_09697_b200 import ops

    rng = np.random.default_rng(5)
    sizes = [7, 12, 3, 30]
    G, V = len(sizes), sum(sizes)
    e = rng.standard_normal(G).astype(np.float32)
    e_t = rng.standard_normal(G)
    f = rng.standard_normal((V, 3)).astype(np.float32)
    f_t = rng.standard_normal((V, 3))
    cnt = np.repeat(np.asarray(sizes, dtype=np.float64), sizes)
    w_e, w_f, n = 0.7, (1.3 if with_forces else 0.0), 6.0
    dev = "cuda"
    loss, d_e, d_f = ops.loss_seeds(torch.tensor(e, device=dev), torch.tensor(e_t, device=dev),
                                    torch.tensor(f, device=dev) if with_forces else None,
                                    torch.tensor(f_t, device=dev), torch.tensor(cnt, device=dev), w_e, w_f, n)
    res = e.astype(np.float64) - e_t
    ref_loss = (w_e * res * res).sum() / n
    np.testing.assert_array_equal(d_e.cpu().numpy(), (2.0 * w_e * res / n).astype(np.float32))
    if with_forces:
        delta = f.astype(np.float64) - f_t
        ref_loss += w_f * ((delta * delta).sum(1) / cnt).sum() / n
        np.testing.assert_array_equal(d_f.cpu().numpy(), (2.0 * w_f * delta / (n * cnt[:, None])).astype(np.float32))
    else:
        assert d_f is None
    assert abs(float(loss) - ref_loss) <= 1e-12 * abs(ref_loss)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_side_streams_bit_identical(variant, monkeypatch):
    """The side-stream schedule of Engine.forward/backward (weight gradients, graph update,
    rbf gates, node-level adjoint chain) forced on for a small batch: eager and captured
    steps reproduce the single-stream trainer bit for bit, and the gradients still match
    the live oracle."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    cfg = ModelConfig(variant=variant, blocks=2, d_u=32, d_v=32, d_e=64, d_t=64, d_bil=64, k_rbf=6,
                      l_sbf=7, cutoff=6.0, seed=8)
    params = init_params(cfg)
    rng = np.random.default_rng(21)
    systems = [O.random_cloud(n, 0.06, rng)[0] for n in (25, 18, 30)]
    e_t = rng.standard_normal(3)
    gem = variant == "gemnet-style"
    f_t = np.concatenate([rng.standard_normal((s.shape[0], 3)) for s in systems]) if gem else None
    w_f = 0.3 if gem else 0.0
    runs = []
    for streams, graph_mode in (("0", False), ("1", False), ("1", True)):
        monkeypatch.setenv("EGN_WGRAD_STREAM", streams)
        monkeypatch.setenv("EGN_SIDE_MIN_EDGES", "0")
        tr = Trainer(params, None, e_t, f_t, 1.0, w_f, graph=build_batch(systems, cfg.cutoff), cuda_graph=graph_mode)
        losses = [float(tr.step(1e-6)) for _ in range(3)]
        runs.append((losses, tr.weights.flat.clone()))
    (l0, w0) = runs[0]
    for l1, w1 in runs[1:]:
        assert l0 == l1
        assert torch.equal(w0, w1)
    # the multi-stream gradient against the live oracle
    from paper_2203_09697_b200.tasks import loss_and_grads

    data = [(s, float(e), f_t[sum(len(x) for x in systems[:i]):][:len(s)] if gem else None)
            for i, (s, e) in enumerate(zip(systems, e_t))]
    loss, grads = loss_and_grads(data, params, 1.0, w_f)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    odata = [(s, np.zeros(len(s), dtype=np.int64), e, f) for s, e, f in data]
    ref_loss, ref_grads = O.loss_and_grads(oc, params.arrays, odata, 1.0, w_f)[:2]
    assert abs(loss - ref_loss) <= TOL * abs(ref_loss)
    for k, g in grads.items():
        assert max_rel(g, ref_grads[k]) < TOL, k


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_egn_model_custom_op_under_torch_compile(variant):
    """EGNModel calls torch.ops.egn.energy_forces (custom op + registered autograd): the module
    runs under torch.compile(fullgraph=False) with results identical to eager mode, and both
    match the fp64 oracle."""
    from paper_2203_09697_b200 import EGNModel, ModelConfig, init_params

    cfg = ModelConfig(variant=variant, blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, cutoff=6.0, seed=6)
    params = init_params(cfg)
    pos, z = O.random_cloud(16, 0.06, np.random.default_rng(12))
    model = EGNModel(cfg, params)
    bg = model.batch([pos])
    w = torch.tensor(np.random.default_rng(3).standard_normal((16, 3)), device="cuda", dtype=torch.float32)

    def run(fn):
        model.zero_grad(set_to_none=True)
        e, f = fn(bg)
        loss = 0.5 * e.sum() + ((f * w).sum() if variant == "gemnet-style" else 0.0)
        loss.backward()
        return e.detach().clone(), f.detach().clone(), {n: p.grad.clone() for n, p in model.named_parameters()}

    e0, f0, g0 = run(model)
    compiled = torch.compile(model, backend="aot_eager", fullgraph=False)
    e1, f1, g1 = run(compiled)
    assert torch.equal(e0, e1) and torch.equal(f0, f1)
    for n in g0:
        assert torch.equal(g0[n], g1[n]), n
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    fr = O.forward(oc, params.arrays, pos, z)
    G, _ = O.backward(fr, params.arrays, 0.5, w.double().cpu().numpy() if variant == "gemnet-style" else None)
    assert abs(float(e0[0]) - fr.energy) <= TOL * max(1.0, abs(fr.energy))
    for n, g in G.items():
        assert max_rel(model.weights.unpad(n, g0[n].double().cpu().numpy()), g) < TOL, n


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_model_on_spherical_harmonic_triplet_kernels(variant):
    """The whole model with the linear-in-degree spherical-harmonic triplet kernels for every
    centre (egn_triplet_path 1) vs the fp64 oracle: energies, forces, all gradients."""
    from paper_2203_09697_b200 import ModelConfig, _lib, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    cfg = ModelConfig(variant=variant, blocks=2, d_u=32, d_v=32, d_e=64, d_t=32, d_bil=64, k_rbf=6, l_sbf=7,
                      cutoff=6.0, seed=13)
    params = init_params(cfg)
    rng = np.random.default_rng(17)
    systems = [O.random_cloud(n, 0.06, rng) for n in (22, 35)]
    old = _lib.call("egn_triplet_path", 1)
    try:
        eng = Engine(DeviceWeights.from_params(params))
        bg = build_batch([s[0] for s in systems], cfg.cutoff)
        fw = eng.forward(bg)
        de = np.array([0.4, -0.9])
        dfs = [rng.standard_normal(s[0].shape) for s in systems] if variant == "gemnet-style" else None
        pos_bar = eng.backward(bg, fw, torch.tensor(de, device="cuda"),
                               torch.tensor(np.concatenate(dfs), device="cuda") if dfs else None).cpu().numpy()
    finally:
        _lib.call("egn_triplet_path", old)
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
        for k in ref_g:
            ref_g[k] += G[k]
        off += n
    for k, g in ref_g.items():
        assert max_rel(grads[k], g) < TOL, k


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_captured_step_with_degenerate_graphs(variant, monkeypatch):
    """The captured multi-stream training step over a batch holding an isolated atom, a dimer
    (no triplets) and an ordinary graph: loss and every gradient equal the oracle's
    loss_and_grads (the bench path on the graphs the kernels special-case)."""
    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    monkeypatch.setenv("EGN_SIDE_MIN_EDGES", "0")
    cfg = ModelConfig(variant=variant, blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, k_rbf=6, l_sbf=7,
                      cutoff=5.0, seed=9)
    params = init_params(cfg)
    rng = np.random.default_rng(8)
    systems = [np.zeros((1, 3)), np.array([[0.0, 0.0, 0.0], [0.9, -0.4, 0.5]]), O.random_cloud(24, 0.1, rng)[0]]
    w_f = 0.5 if variant == "gemnet-style" else 0.0
    e_t = rng.standard_normal(3)
    f_t = np.concatenate([rng.standard_normal((s.shape[0], 3)) for s in systems])
    tr = Trainer(params, None, e_t, f_t if w_f else None, 1.0, w_f, graph=build_batch(systems, cfg.cutoff),
                 cuda_graph=True)
    tr.step(0.0)
    loss = float(tr.step(0.0))
    grads = tr.weights.to_numpy(grads=True)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    f_split = np.split(f_t, np.cumsum([s.shape[0] for s in systems])[:-1])
    data = [(s, np.full(s.shape[0], 6), e, f) for s, e, f in zip(systems, e_t, f_split)]
    loss_ref, g_ref = O.loss_and_grads(oc, params.arrays, data, w_energy=1.0, w_forces=w_f)
    assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
    for k, g in g_ref.items():
        assert max_rel(grads[k], g) < TOL, k
