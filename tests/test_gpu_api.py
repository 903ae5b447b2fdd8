"""The reference's public model surface with only the import swapped (egn/__init__.py:3-27):
ModelTape, basis functions, gradient surfaces, predict / loss_and_grads / train_simple with
workers > 1 (egn/tasks.py routes them through WorkerGroup).  Known answers follow the
reference's own tests (tests/test_basis.py, tests/test_gradients.py, tests/test_engine.py);
values are checked against the fp64 oracle.
"""

import numpy as np
import pytest

import paper_2203_09697_b200 as egn
from paper_2203_09697_b200 import api as egn_api
from conftest import TOL, max_rel
from oracle import egn_oracle as O

pytestmark = pytest.mark.gpu


def _oc(cfg):
    return O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})


# -- egn/basis.py (tests/test_basis.py) -------------------------------------------------
def test_rbf_known_answers_and_errors():
    centers = egn_api.rbf_centers(6, 1.5)
    assert egn.rbf_features(np.array([centers[2]]), 6, 1.5)[0, 2] == pytest.approx(1.0)
    f = egn.rbf_features(np.array([1.0]), 1, 1.0)
    assert f.shape == (1, 1) and f[0, 0] == pytest.approx(np.exp(-1.0), abs=1e-15)
    c4 = egn_api.rbf_centers(4, 2.0)
    vals = egn.rbf_features(c4[1] + np.array([0.05, 0.1, 0.2, 0.4]), 4, 2.0)[:, 1]
    assert np.all(np.diff(vals) < 0)
    d = np.linspace(0.1, 1.5, 20)
    feats = egn.rbf_features(d, 5, 1.5)
    assert np.all(feats > 0) and np.all(feats <= 1.0)
    np.testing.assert_allclose(feats, O.rbf(d, 5, 1.5), rtol=1e-14, atol=0)
    np.testing.assert_allclose(egn_api.rbf_features_ddist(d, 5, 1.5), O.rbf_ddist(d, 5, 1.5), rtol=1e-13, atol=1e-15)
    for bad in ((np.array([1.0]), 0, 1.5), (np.array([2.0]), 3, 1.5), (np.array([0.0]), 3, 1.5)):
        with pytest.raises(ValueError):
            egn.rbf_features(*bad)


def test_sbf_known_answers_and_errors():
    d, ang = np.array([0.7, 1.1]), np.array([0.3, 2.0])
    np.testing.assert_allclose(egn.sbf_features(d, ang, 3, 2, 1.5)[:, 0::2], egn.rbf_features(d, 3, 1.5), atol=1e-15)
    np.testing.assert_allclose(egn.sbf_features(np.array([1.0]), np.array([np.pi / 2]), 2, 2, 1.5)[0, 1::2], 0.0,
                               atol=1e-15)
    c = egn_api.rbf_centers(3, 1.5)
    assert egn.sbf_features(np.array([c[1]]), np.array([np.pi / 3]), 3, 3, 1.5)[0, 1 * 3 + 2] == pytest.approx(
        -0.5, abs=1e-12)
    rng = np.random.default_rng(0)
    dd, aa = rng.uniform(0.2, 1.5, 50), rng.uniform(0, np.pi, 50)
    np.testing.assert_allclose(egn.sbf_features(dd, aa, 4, 5, 1.5), O.sbf(dd, aa, 4, 5, 1.5), rtol=1e-13,
                               atol=1e-15)
    p_d, p_a = egn_api.sbf_features_partials(dd, aa, 4, 5, 1.5)
    r_d, r_a = O.sbf_partials(dd, aa, 4, 5, 1.5)
    np.testing.assert_allclose(p_d, r_d, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(p_a, r_a, rtol=1e-12, atol=1e-14)
    with pytest.raises(ValueError):
        egn.sbf_features(np.array([1.0]), np.array([0.5]), 3, 0, 1.5)
    with pytest.raises(ValueError):
        egn.sbf_features(np.array([1.0]), np.array([4.0]), 3, 2, 1.5)


def test_compute_basis_matches_oracle():
    pos, _ = O.random_cloud(20, 0.2, np.random.default_rng(1))
    topo, geom = egn.build_graph(pos, 3.0)
    b = egn.compute_basis(geom, topo, 6, 7, 3.0)
    g = O.build_graph(pos, 3.0)
    np.testing.assert_allclose(b.edge_rbf, O.rbf(g.dist, 6, 3.0), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(b.triplet_sbf, O.sbf(g.dist[g.trip_in], g.angles, 6, 7, 3.0), rtol=1e-9, atol=1e-12)


# -- egn/gradients.py (tests/test_gradients.py) -----------------------------------------
def test_geometry_grads_known_answers_and_oracle():
    dimer = np.array([[0.0, 0, 0], [0.0, 0, 1.0]])
    topo, _ = egn.build_graph(dimer, 1.5)
    g = egn.geometry_grads(dimer, topo)
    np.testing.assert_allclose(g.dist_d_recv[0], [0, 0, 1.0], atol=1e-14)
    np.testing.assert_allclose(g.dist_d_src[0], [0, 0, -1.0], atol=1e-14)
    tri = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, np.sqrt(3) / 2, 0]])
    topo, _ = egn.build_graph(tri, 1.5)
    g = egn.geometry_grads(tri, topo)
    np.testing.assert_allclose(g.angle_d_k + g.angle_d_j + g.angle_d_i, 0.0, atol=1e-14)
    pos, _ = O.random_cloud(15, 0.3, np.random.default_rng(4))
    topo, _ = egn.build_graph(pos, 3.0)
    g = egn.geometry_grads(pos, topo)
    r = O.build_graph(pos, 3.0)
    gk, gj, gi = O.angle_gradients(pos, r.src, r.recv, r.trip_in, r.trip_out)
    np.testing.assert_allclose(g.angle_d_k, gk, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g.angle_d_j, gj, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g.angle_d_i, gi, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(g.dist_d_recv, r.units, rtol=1e-14, atol=1e-15)


# -- egn/engine.py ModelTape (tests/test_engine.py, tests/test_gradients.py) ---------------
@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_model_tape_matches_oracle(variant):
    cfg = egn.ModelConfig(variant=variant, blocks=2, d_u=16, d_v=24, d_e=32, d_t=16, d_bil=8, k_rbf=6, l_sbf=7,
                          cutoff=6.0, seed=5)
    params = egn.init_params(cfg)
    pos, z = O.random_cloud(18, 0.06, np.random.default_rng(8))
    system = egn.AtomicSystem(pos, z)
    tape = egn.ModelTape(system, params)
    f = O.forward(_oc(cfg), params.arrays, pos, z)
    assert abs(tape.energy - f.energy) <= TOL * max(1.0, abs(f.energy))
    st = tape.state
    assert max_rel(st.edge_features, f.m) < TOL and max_rel(st.global_features, f.u) < TOL
    assert max_rel(st.triplet_features, f.t_feat) < TOL
    rng = np.random.default_rng(2)
    df = rng.standard_normal(pos.shape) if variant == "gemnet-style" else None
    bundle = egn.backward(tape, d_energy=0.6, d_forces=df, check_replay=True)
    G, dp = O.backward(f, params.arrays, 0.6, df)
    assert max_rel(bundle.d_positions, dp) < TOL
    for k in G:
        assert max_rel(bundle.d_params[k], G[k]) < TOL, k
    if variant == "gemnet-style":
        assert max_rel(tape.forces, f.forces) < TOL
    else:
        assert tape.forces is None
        with pytest.raises(ValueError):
            tape.backward(d_forces=np.zeros(pos.shape))
        e, forces, b2 = egn.forces_energy_centric(system, params)
        _, f_ref = O.predict(_oc(cfg), params.arrays, pos, z)
        assert max_rel(forces, f_ref) < TOL and abs(e - f.energy) <= TOL * max(1.0, abs(f.energy))
    # prebuilt topology / geometry (egn/engine.py:331-341) gives the same model
    again = egn.ModelTape(system, params, prebuilt=(tape.topology, tape.geometry))
    assert again.energy == pytest.approx(tape.energy, rel=1e-6)
    with pytest.raises(ValueError):
        egn.ModelTape(egn.AtomicSystem(pos, np.full(pos.shape[0], 119)), params)


def test_block_forward_equals_second_block():
    cfg = egn.ModelConfig(variant="gemnet-style", blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, cutoff=6.0,
                          seed=1)
    params = egn.init_params(cfg)
    pos, z = O.random_cloud(14, 0.06, np.random.default_rng(3))
    tape = egn.ModelTape(egn.AtomicSystem(pos, z), params)
    full = tape.state
    cfg1 = cfg.replace(blocks=1)
    p1 = egn.ModelParams(cfg1, {k: v for k, v in params.arrays.items() if not k.startswith("block1.")})
    st1 = egn.ModelTape(egn.AtomicSystem(pos, z), p1).state
    nxt = egn.block_forward(st1, params, 1, positions=pos)
    assert max_rel(nxt.edge_features, full.edge_features) < TOL
    assert max_rel(nxt.global_features, full.global_features) < TOL


# -- egn/tasks.py with workers > 1 -------------------------------------------------------
@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_predict_and_loss_with_workers(variant):
    cfg = egn.ModelConfig(variant=variant, blocks=2, d_u=16, d_v=16, d_e=32, d_t=16, d_bil=16, cutoff=6.0, seed=3)
    params = egn.init_params(cfg)
    rng = np.random.default_rng(6)
    systems = [O.random_cloud(n, 0.06, rng) for n in (16, 21)]
    e1, f1 = egn.predict(systems[0][0], params)
    e3, f3 = egn.predict(systems[0][0], params, workers=3)
    assert abs(e3 - e1) <= 1e-5 * max(1.0, abs(e1)) and max_rel(f3, f1) < 1e-5
    w_f = 0.5 if variant == "gemnet-style" else 0.0
    data = [(p, float(rng.standard_normal()), rng.standard_normal((p.shape[0], 3))) for p, _ in systems]
    l1, g1 = egn.loss_and_grads(data, params, 1.0, w_f)
    l2, g2 = egn.loss_and_grads(data, params, 1.0, w_f, workers=2)
    ref_l, ref_g = O.loss_and_grads(_oc(cfg), params.arrays, [(p, z, e, f) for (p, z), (_, e, f) in zip(systems, data)],
                                    1.0, w_f)
    assert abs(l2 - ref_l) <= TOL * abs(ref_l) and abs(l1 - l2) <= 1e-5 * abs(l1)
    for k in ref_g:
        assert max_rel(g2[k], ref_g[k]) < TOL, k
    p_out, hist = egn.train_simple(data, params, lr=1e-3, epochs=2, w_forces=w_f, workers=2)
    assert len(hist) == 2 and hist[0] == pytest.approx(l2, rel=1e-6)


def test_collective_surface():
    """egn.runtime.Collective (tests/test_runtime.py:51-96): rank-ordered sums, level guard."""
    import threading

    log = egn.CommLog()
    col = egn.Collective(2, log, timeout=10.0)
    out = [None, None]

    def body(r):
        out[r] = col.allreduce_sum(r, np.full(3, r + 1.0), phase="forward", block=0, stage="x", level="edge")

    ts = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert np.array_equal(out[0], np.full(3, 3.0)) and np.array_equal(out[1], out[0])
    assert log.records[0].elements == 3
    with pytest.raises(ValueError):
        col.allreduce_sum(0, np.zeros(1), phase="forward", block=0, stage="t", level="triplet")
