"""Pin the CPU oracle (oracle/egn_oracle.py) to the reference's own outputs.

The golden fixtures were produced by running the reference package in this
container (tests/golden/make_golden.py).  Topology must be bit-exact;
floating-point outputs and all gradients agree to 1e-10 relative (the
oracle is a restatement in the same fp64 operation order).
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, max_rel
from oracle import egn_oracle as O

MODEL_FILES = sorted(p.name for p in GOLDEN.glob("model_*.npz"))


def _cfg(js):
    d = json.loads(str(js))
    return O.Config(**{k: d[k] for k in O.Config.__dataclass_fields__ if k in d})


def test_graph_topology_bit_exact(graphs_golden):
    data, names = graphs_golden
    assert len(names) >= 15
    for name in names:
        g = O.build_graph(data[f"{name}/pos"], float(data[f"{name}/cutoff"]))
        for key, val in (("src", g.src), ("recv", g.recv), ("trip_in", g.trip_in), ("trip_out", g.trip_out),
                         ("rev", g.rev)):
            np.testing.assert_array_equal(val, data[f"{name}/{key}"], err_msg=f"{name}/{key}")
        np.testing.assert_array_equal(g.dist, data[f"{name}/dist"])
        np.testing.assert_array_equal(g.units, data[f"{name}/units"])
        np.testing.assert_array_equal(g.angles, data[f"{name}/angles"])


def test_graph_edge_cases(graphs_golden):
    data, _ = graphs_golden
    assert data["dimer/src"].size == 2 and data["dimer/trip_in"].size == 0
    assert data["collinear_chain/trip_in"].size == 2
    np.testing.assert_allclose(data["collinear_chain/angles"], np.pi)
    assert data["triangle/trip_in"].size == 6
    assert data["zero_edge/src"].size == 0
    assert data["single_atom/src"].size == 0
    # spacing == cutoff: the 6 axis neighbours of an interior lattice point are edges
    assert data["lattice_at_cutoff/src"].size == 2 * 3 * 4 * 4 * 3


@pytest.mark.parametrize("fname", MODEL_FILES)
def test_model_forward_backward_matches_reference(fname):
    gd = load_golden(fname)
    cfg = _cfg(gd["config"])
    P = O.init_params(cfg)
    np.testing.assert_allclose([float(np.sum(a)) for a in P.values()], gd["param_checksum"], rtol=0, atol=0)
    fw = O.forward(cfg, P, gd["pos"], gd["z"])
    d_forces = gd.get("d_forces")
    G, d_pos = O.backward(fw, P, 0.7, d_forces)
    assert abs(fw.energy - float(gd["energy"])) <= 1e-10 * max(abs(float(gd["energy"])), 1.0)
    assert max_rel(fw.m, gd["m"]) < (1e-6 if gd["m"].dtype == np.float32 else 1e-10)
    assert max_rel(fw.t_feat, gd["t_feat"]) < (1e-6 if gd["t_feat"].dtype == np.float32 else 1e-10)
    assert max_rel(fw.v, gd["v"]) < 1e-10
    assert max_rel(d_pos, gd["d_positions"]) < 1e-10
    if cfg.variant == O.GEMNET:
        assert max_rel(fw.forces, gd["forces"]) < 1e-10
    else:
        _, dp1 = O.backward(fw, P, 1.0)
        assert max_rel(-dp1, gd["forces"]) < 1e-10
    for name in gd["param_names"]:
        name = str(name)
        if f"dp/{name}" in gd:
            assert max_rel(G[name], gd[f"dp/{name}"]) < 1e-10, name
        else:
            assert max_rel(G[name].ravel()[:64], gd[f"dphead/{name}"]) < 1e-10, name
            assert abs(np.abs(G[name]).max() - float(gd[f"dpnorm/{name}"])) <= 1e-10 * max(float(gd[f"dpnorm/{name}"]), 1e-300)


@pytest.mark.parametrize("variant", ["dimenet", "gemnet"])
def test_loss_and_grads_matches_reference(variant):
    gd = load_golden(f"train_{variant}.npz")
    cfg = _cfg(gd["config"])
    P = O.init_params(cfg)
    data = [(gd[f"pos{i}"], gd[f"z{i}"], float(gd[f"e{i}"]), gd[f"f{i}"]) for i in range(3)]
    w_f = float(gd["w_forces"])
    loss, grads = O.loss_and_grads(cfg, P, data, 1.0, w_f)
    assert abs(loss - float(gd["loss"])) <= 1e-10 * abs(float(gd["loss"]))
    for k, g in grads.items():
        assert max_rel(g, gd[f"grad/{k}"]) < 1e-10, k
    # train_simple history
    hist, cur = [], P
    for _ in range(4):
        l, g = O.loss_and_grads(cfg, cur, data, 1.0, w_f)
        hist.append(l)
        cur = O.sgd_step(cur, g, 0.002)
    np.testing.assert_allclose(hist, gd["history"], rtol=1e-9)


@pytest.mark.parametrize("variant", ["dimenet", "gemnet"])
def test_relax_matches_reference(variant):
    """relax (tasks.py:79-128): graph rebuilt per evaluation; the dimenet case rejects
    five proposals (energy guard, eta halved), the gemnet case has no guard."""
    gd = load_golden(f"relax_{variant}.npz")
    cfg = _cfg(gd["config"])
    P = O.init_params(cfg)
    traj, fmax, energies, converged, steps = O.relax(cfg, P, gd["pos"], gd["z"], float(gd["fmax_threshold"]),
                                                     int(gd["max_steps"]), float(gd["step_size"]))
    assert steps == int(gd["steps"]) and converged == bool(gd["converged"])
    assert max_rel(np.stack(traj), gd["trajectory"]) < 1e-10
    assert max_rel(np.array(energies), gd["energies"]) < 1e-10
    assert max_rel(np.array(fmax), gd["max_forces"]) < 1e-10
    if variant == "dimenet":
        assert np.sum(np.diff(energies) == 0) == 5
        assert np.all(np.diff(energies) <= 0)
    with pytest.raises(ValueError):
        O.relax(cfg, P, gd["pos"], gd["z"], 0.0)
    with pytest.raises(ValueError):
        O.relax(cfg, P, gd["pos"], gd["z"], 1e-3, max_steps=-1)


PBC_NAMES = ["cubic4", "triclinic5", "slab6", "self_image1", "unwrapped5"]


@pytest.mark.parametrize("name", PBC_NAMES)
def test_periodic_graph_matches_reference_supercell(name):
    """Periodic neighbour list vs the reference build_graph on an explicit
    supercell (tests/golden/pbc.npz): same (a, b, image) edges; distances within a few ulp of the coordinates (the
    supercell materialises x_b + s before subtracting x_a, the kernels form (x_b - x_a) + s,
    which is exactly antisymmetric so every edge has its reverse)."""
    gd = load_golden("pbc.npz")
    g = O.build_graph_pbc(gd[f"{name}/pos"], gd[f"{name}/cell"], gd[f"{name}/pbc"], float(gd[f"{name}/cutoff"]))
    np.testing.assert_array_equal(O.image_ranges(gd[f"{name}/cell"], gd[f"{name}/pbc"], float(gd[f"{name}/cutoff"]),
                                                 gd[f"{name}/pos"]), gd[f"{name}/nimg"])
    for key, val in (("src", g.src), ("recv", g.recv), ("img", g.img)):
        np.testing.assert_array_equal(val, gd[f"{name}/{key}"], err_msg=f"{name}/{key}")
    # the two operation orders round differently at the scale of the coordinates (unwrapped
    # inputs sit several cells out): a few ulp of max |x|
    ref_d = gd[f"{name}/dist"]
    scale = max(float(np.abs(gd[f"{name}/pos"]).max()) + float(np.abs(gd[f"{name}/cell"]).sum(0).max()), 1.0)
    assert np.abs(g.dist - ref_d).max(initial=0.0) <= 8 * np.finfo(np.float64).eps * scale, name
    # reverse edges mirror the image; triplets never pair an edge with its own reverse
    n_img = int(np.prod(2 * gd[f"{name}/nimg"] + 1))
    assert np.array_equal(g.src[g.rev], g.recv) and np.array_equal(g.img[g.rev], n_img - 1 - g.img)
    assert not np.any(g.rev[g.trip_out] == g.trip_in)
    assert np.array_equal(g.recv[g.trip_in], g.src[g.trip_out])


def test_periodic_graph_symmetric_at_cutoff_boundary():
    """An atom's own +-2-cell images sit exactly at the cutoff (cell 3, cutoff 6): with the
    antisymmetric edge vector (x_b - x_a) + s both directions pass or fail together, so the
    graph always has every reverse edge (the oracle raises ValueError otherwise)."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        pos = rng.uniform(0.0, 3.0, size=(2, 3))
        g = O.build_graph_pbc(pos, np.eye(3) * 3.0, (True, True, True), 6.0)
        assert np.array_equal(g.src[g.rev], g.recv) and np.array_equal(g.rev[g.rev], np.arange(g.src.size))
        assert np.array_equal(g.dist[g.rev], g.dist)


def test_periodic_graph_without_images_is_the_reference_graph():
    rng = np.random.default_rng(5)
    pos, _ = O.random_cloud(30, 0.2, rng)
    a = O.build_graph(pos, 3.0)
    b = O.build_graph_pbc(pos, np.eye(3) * 1e3, (True, True, True), 3.0)
    for key in ("src", "recv", "trip_in", "trip_out", "rev", "dist", "units", "angles"):
        np.testing.assert_array_equal(getattr(a, key), getattr(b, key), err_msg=key)


def test_oracle_fd_gradient_spot_check():
    """Independent of the fixtures: central differences of the oracle energy."""
    cfg = O.Config(variant=O.DIMENET, blocks=1)
    rng = np.random.default_rng(3)
    pos, z = O.random_cloud(6, 0.9, rng)
    P = O.init_params(cfg)
    fw = O.forward(cfg, P, pos, z)
    G, dpos = O.backward(fw, P, 1.0)
    h = 1e-6
    for name in ("block0.tu.sbf_gate", "block0.tu.down", "edge_init.w"):
        i = 1
        a = P[name].ravel()
        orig = a[i]
        a[i] = orig + h
        ep = O.forward(cfg, P, pos, z).energy
        a[i] = orig - h
        em = O.forward(cfg, P, pos, z).energy
        a[i] = orig
        fd = (ep - em) / (2 * h)
        assert abs(fd - G[name].ravel()[i]) < 1e-6 * max(1.0, abs(fd))


def test_neighbour_cap_restatement():
    """Cap rule: mutual k-nearest edges; symmetric, degree <= k, identity when
    k >= max degree, and every kept edge is within both endpoints' k nearest."""
    rng = np.random.default_rng(3)
    pos, _ = O.random_cloud(40, 0.2, rng)
    g = O.build_graph(pos, 4.0)
    for k in (1, 5, 8, 20):
        c = O.cap_graph(g, pos, k)
        assert np.array_equal(c.src[c.rev], c.recv) and np.array_equal(c.recv[c.rev], c.src)
        assert np.bincount(c.src, minlength=40).max() <= k
        for a, b, d in zip(c.src, c.recv, c.dist):
            for x, y in ((a, b), (b, a)):
                row = g.dist[g.src == x]
                assert np.sum(row < d) < k  # (ties resolved by edge order)
    full = O.cap_graph(g, pos, 1000)
    for key in ("src", "recv", "trip_in", "trip_out", "rev", "dist", "angles"):
        assert np.array_equal(getattr(full, key), getattr(g, key)), key


@pytest.mark.parametrize("variant", [O.DIMENET, O.GEMNET])
def test_bessel_bases_restatement(variant):
    """DimeNet++ / GemNet bases (no reference counterpart, parity unpinned):
    known answers and finite-difference checks of the fp64 restatement."""
    from scipy.special import spherical_jn

    z = O.spherical_bessel_zeros(7, 6)
    for l in range(7):
        assert np.abs(spherical_jn(l, z[l])).max() < 1e-12
    np.testing.assert_allclose(z[0], np.pi * np.arange(1, 7), rtol=1e-13)
    # envelope: smooth cutoff, u(1) = u'(1) = 0
    assert abs(O.envelope(1.0 - 1e-12) - 0.0) < 1e-9 and abs(O.envelope_dx(1.0 - 1e-12)) < 1e-8
    rng = np.random.default_rng(0)
    d = rng.uniform(0.5, 5.9, 30)
    ang = rng.uniform(0.05, np.pi - 0.05, 30)
    h = 1e-6
    fd = (O.bessel_rbf(d + h, 6, 6.0) - O.bessel_rbf(d - h, 6, 6.0)) / (2 * h)
    np.testing.assert_allclose(O.bessel_rbf_ddist(d, 6, 6.0), fd, rtol=1e-6, atol=1e-8)
    dd, da = O.sbf_bessel_partials(d, ang, 6, 7, 6.0, variant)
    fdd = (O.sbf_bessel(d + h, ang, 6, 7, 6.0, variant) - O.sbf_bessel(d - h, ang, 6, 7, 6.0, variant)) / (2 * h)
    fda = (O.sbf_bessel(d, ang + h, 6, 7, 6.0, variant) - O.sbf_bessel(d, ang - h, 6, 7, 6.0, variant)) / (2 * h)
    np.testing.assert_allclose(dd, fdd, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(da, fda, rtol=1e-5, atol=1e-7)
    # the whole model on the bessel bases: position and parameter gradients vs central differences
    cfg = O.Config(variant=variant, blocks=2, d_u=4, d_v=5, d_e=6, d_t=4, d_bil=3, k_rbf=6, l_sbf=7, cutoff=6.0,
                   basis="bessel")
    pos, zz = O.random_cloud(7, 0.06, np.random.default_rng(5))
    P = O.init_params(cfg)
    fw = O.forward(cfg, P, pos, zz)
    df = rng.standard_normal(pos.shape) if variant == O.GEMNET else None

    def objective(p_, P_):
        f = O.forward(cfg, P_, p_, zz)
        val = 0.7 * f.energy
        if df is not None:
            val += float((f.forces * df).sum())
        return val

    G, dpos = O.backward(fw, P, 0.7, df)
    for a in range(3):
        for ax in range(3):
            e = np.zeros_like(pos)
            e[a, ax] = 1e-5
            fdv = (objective(pos + e, P) - objective(pos - e, P)) / 2e-5
            assert abs(fdv - dpos[a, ax]) < 1e-6 * max(1.0, abs(fdv)), (a, ax, fdv, dpos[a, ax])
    for name in ("block0.tu.sbf_gate", "block1.tu.rbf_gate", "edge_init.w"):
        arr = P[name].ravel()
        i = 2
        orig = arr[i]
        arr[i] = orig + 1e-6
        fp = objective(pos, P)
        arr[i] = orig - 1e-6
        fm = objective(pos, P)
        arr[i] = orig
        fdv = (fp - fm) / 2e-6
        assert abs(fdv - G[name].ravel()[i]) < 1e-6 * max(1.0, abs(fdv)), name
