"""Generate golden fixtures by running the REFERENCE package (egn) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [graphs models training relax]

The reference is not available on the GPU box, so its outputs are frozen
here as small .npz files.  Inputs (positions) are stored explicitly;
weights are regenerated from init_params(seed) (checked by checksum).
Every file records the numpy version used.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("EGN_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from egn import ModelConfig, ModelTape, build_graph, init_params  # noqa: E402
from egn.system import AtomicSystem, random_cloud  # noqa: E402
from egn.tasks import loss_and_grads, relax, train_simple  # noqa: E402

OUT = Path(__file__).resolve().parent


def fixture_systems():
    """Named (system, cutoff) cases: reference test fixtures + random + boundary cases."""
    cases = {}
    cases["dimer"] = (AtomicSystem(np.array([[0.0, 0, 0], [0, 0, 1.0]]), np.array([1, 1])), 1.5)
    chain = np.zeros((3, 3))
    chain[:, 2] = np.arange(3.0)
    cases["collinear_chain"] = (AtomicSystem(chain, np.full(3, 6)), 1.5)
    tri = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, np.sqrt(3) / 2, 0]])
    cases["triangle"] = (AtomicSystem(tri, np.full(3, 6)), 1.5)
    star = np.array([[0.0, 0, 0], [1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0]])
    cases["star"] = (AtomicSystem(star, np.array([6, 1, 1, 1])), 1.2)
    cases["zero_edge"] = (AtomicSystem(np.array([[0.0, 0, 0], [10.0, 0, 0]]), np.array([1, 1])), 1.0)
    cases["single_atom"] = (AtomicSystem(np.array([[0.0, 0, 0]]), np.array([8])), 1.5)
    # cubic lattice with spacing == cutoff: axis neighbours at exactly d == cutoff
    g = np.arange(4) * 1.5
    lat = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    cases["lattice_at_cutoff"] = (AtomicSystem(lat, np.full(len(lat), 6)), 1.5)
    # shell of atoms at |x - c| == cutoff up to rounding around a centre
    rng = np.random.default_rng(99)
    dirs = rng.standard_normal((40, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    shell = np.concatenate([[[0.3, 0.2, 0.1]], np.array([0.3, 0.2, 0.1]) + 1.5 * dirs])
    cases["shell_at_cutoff"] = (AtomicSystem(shell, np.full(len(shell), 6)), 1.5)
    for s in range(10):
        r = np.random.default_rng(s)
        n = int(r.integers(2, 41))
        cases[f"cloud{s}"] = (random_cloud(n, 0.9, r), 1.5)
    cases["oc20_80"] = (random_cloud(80, 0.06, np.random.default_rng(0)), 6.0)
    cases["oc20_64"] = (random_cloud(64, 0.06, np.random.default_rng(1)), 6.0)
    return cases


def make_graphs():
    data = {}
    for name, (system, cutoff) in fixture_systems().items():
        topo, geom = build_graph(system, cutoff)
        data[f"{name}/pos"] = system.positions
        data[f"{name}/z"] = system.atomic_numbers
        data[f"{name}/cutoff"] = np.array(cutoff)
        data[f"{name}/src"] = topo.edge_src
        data[f"{name}/recv"] = topo.edge_recv
        data[f"{name}/trip_in"] = topo.trip_in
        data[f"{name}/trip_out"] = topo.trip_out
        data[f"{name}/rev"] = topo.reverse_edges() if topo.num_edges else np.zeros(0, np.int64)
        data[f"{name}/dist"] = geom.distances
        data[f"{name}/units"] = geom.unit_vectors
        data[f"{name}/angles"] = geom.angles
    data["numpy_version"] = np.array(np.__version__)
    np.savez_compressed(OUT / "graphs.npz", **data)
    print("graphs.npz:", len(data), "arrays")


MODEL_CASES = {
    # name: (config kwargs, system generator, full d_params?)
    "dimenet_small": (dict(variant="dimenet-style", blocks=2, seed=3), ("cloud", 14, 0.9, 7), True),
    "gemnet_small": (dict(variant="gemnet-style", blocks=2, seed=4), ("cloud", 14, 0.9, 8), True),
    "gemnet_odd": (dict(variant="gemnet-style", blocks=3, d_u=5, d_v=7, d_e=9, d_t=3, d_bil=5, k_rbf=3,
                        l_sbf=3, cutoff=1.7, seed=5), ("cloud", 20, 0.9, 9), True),
    "dimenet_chain": (dict(variant="dimenet-style", blocks=2, seed=6), ("chain",), True),
    "dimenet_c1dims": (dict(variant="dimenet-style", blocks=4, d_u=128, d_v=128, d_e=128, d_t=64,
                            k_rbf=6, l_sbf=7, cutoff=6.0, seed=0), ("cloud", 24, 0.06, 0), False),
    "gemnet_c2dims": (dict(variant="gemnet-style", blocks=4, d_u=128, d_v=128, d_e=128, d_t=64,
                           d_bil=64, k_rbf=6, l_sbf=7, cutoff=6.0, seed=0), ("cloud", 24, 0.06, 1), False),
}


def _system(spec):
    if spec[0] == "chain":
        pos = np.zeros((3, 3))
        pos[:, 2] = np.arange(3.0)
        return AtomicSystem(pos, np.full(3, 6))
    _, n, rho, seed = spec
    return random_cloud(n, rho, np.random.default_rng(seed))


def make_models():
    for name, (kw, spec, full) in MODEL_CASES.items():
        cfg = ModelConfig(**kw)
        params = init_params(cfg)
        system = _system(spec)
        model = ModelTape(system, params)
        rng = np.random.default_rng(1000)
        d_forces = rng.standard_normal((system.n, 3)) if cfg.variant == "gemnet-style" else None
        bundle = model.backward(d_energy=0.7, d_forces=d_forces)
        out = {
            "config": np.array(cfg.to_json()),
            "pos": system.positions,
            "z": system.atomic_numbers,
            "energy": np.array(model.energy),
            "m": model.state.edge_features.astype(np.float32 if not full else np.float64),
            "v": model.state.node_features,
            "u": model.state.global_features,
            "t_feat": model.state.triplet_features.astype(np.float32 if not full else np.float64),
            "d_positions": bundle.d_positions,
            "param_checksum": np.array([float(np.sum(a)) for a in params.arrays.values()]),
            "numpy_version": np.array(np.__version__),
        }
        if d_forces is not None:
            out["d_forces"] = d_forces
            out["forces"] = model.forces
        else:
            out["forces"] = -model.backward(d_energy=1.0).d_positions
        names = list(bundle.d_params)
        out["param_names"] = np.array(names)
        if full:
            for k in names:
                out[f"dp/{k}"] = bundle.d_params[k]
        else:
            for k in names:
                g = bundle.d_params[k]
                out[f"dpnorm/{k}"] = np.array(np.abs(g).max())
                out[f"dphead/{k}"] = g.ravel()[:64]
        np.savez_compressed(OUT / f"model_{name}.npz", **out)
        print(f"model_{name}.npz", system.n, "atoms")


def make_training():
    """loss_and_grads / train_simple over a 3-sample dataset with a teacher (cli.py:153-160 style)."""
    for variant, w_f in (("dimenet-style", 0.0), ("gemnet-style", 0.5)):
        cfg = ModelConfig(variant=variant, blocks=2, seed=0)
        teacher = init_params(cfg.replace(seed=1))
        params = init_params(cfg)
        data, pos_all = [], []
        for s in range(3):
            system = random_cloud(8 + 3 * s, 0.9, np.random.default_rng(50 + s))
            t = ModelTape(system, teacher)
            e = t.energy
            f = t.forces if variant == "gemnet-style" else -t.backward(1.0).d_positions
            data.append((system, e, f))
        loss, grads = loss_and_grads(data, params, w_energy=1.0, w_forces=w_f)
        _, hist = train_simple(data, params, lr=0.002, epochs=4, w_energy=1.0, w_forces=w_f)
        out = {"config": np.array(cfg.to_json()), "w_forces": np.array(w_f), "loss": np.array(loss),
               "history": np.array(hist), "numpy_version": np.array(np.__version__)}
        for i, (system, e, f) in enumerate(data):
            out[f"pos{i}"] = system.positions
            out[f"z{i}"] = system.atomic_numbers
            out[f"e{i}"] = np.array(e)
            out[f"f{i}"] = f
        for k, g in grads.items():
            out[f"grad/{k}"] = g
        np.savez_compressed(OUT / f"train_{variant.split('-')[0]}.npz", **out)
        print("train", variant, loss, hist)


RELAX_CASES = {
    # name: (config kwargs, (n atoms, density, seed), fmax_threshold, max_steps, step_size)
    "dimenet": (dict(variant="dimenet-style", blocks=2, seed=7), (10, 0.9, 60), 1e-3, 8, 1.0),
    "gemnet": (dict(variant="gemnet-style", blocks=2, seed=8), (10, 0.9, 61), 1e-3, 6, 0.05),
}


def make_relax():
    """relax() trajectories (tasks.py:79-128): graph rebuilt per evaluation, energy guard
    with step halving for the energy-centric variant."""
    for name, (kw, (n, rho, seed), fmax, steps, eta) in RELAX_CASES.items():
        cfg = ModelConfig(**kw)
        params = init_params(cfg)
        system = random_cloud(n, rho, np.random.default_rng(seed))
        res = relax(system, params, fmax_threshold=fmax, max_steps=steps, step_size=eta)
        out = {"config": np.array(cfg.to_json()), "pos": system.positions, "z": system.atomic_numbers,
               "fmax_threshold": np.array(fmax), "max_steps": np.array(steps), "step_size": np.array(eta),
               "trajectory": np.stack(res.trajectory), "energies": np.array(res.energies),
               "max_forces": np.array(res.max_forces), "converged": np.array(res.converged),
               "steps": np.array(res.steps), "numpy_version": np.array(np.__version__)}
        np.savez_compressed(OUT / f"relax_{name}.npz", **out)
        print(f"relax_{name}.npz steps", res.steps, "converged", res.converged, "energies", res.energies)


PBC_CASES = {
    # name: (n atoms, box-fill seed, cell rows, pbc, cutoff)
    "cubic4": (4, 70, [[3.0, 0, 0], [0, 3.0, 0], [0, 0, 3.0]], (True, True, True), 2.5),
    "triclinic5": (5, 71, [[3.2, 0, 0], [0.8, 2.9, 0], [0.5, 0.6, 3.1]], (True, True, True), 2.8),
    "slab6": (6, 72, [[3.5, 0, 0], [0, 3.5, 0], [0, 0, 20.0]], (True, True, False), 3.0),
    "self_image1": (1, 73, [[1.6, 0, 0], [0, 1.7, 0], [0, 0, 1.8]], (True, True, True), 2.0),
    # atoms spread over three cells along c0 (unwrapped coordinates): wider image range
    "unwrapped5": (5, 74, [[3.0, 0, 0], [0.4, 3.1, 0], [0, 0.5, 3.3]], (True, True, True), 2.6),
}


def _image_shifts(cell, pbc, cutoff, pos):
    """Image ranges max(ceil(r), floor(r + span)) (r = cutoff / cell height, span = extent of
    the fractional coordinates) and shifts (i c0 + j c1) + k c2 in image-index order
    ((i, j, k) lexicographic) -- the convention of include/egn_b200.h."""
    cell = np.asarray(cell, dtype=np.float64)
    vol = abs(np.linalg.det(cell))
    frac = pos @ np.linalg.inv(cell)
    span = frac.max(axis=0) - frac.min(axis=0)
    nimg = []
    for a in range(3):
        r = cutoff / (vol / np.linalg.norm(np.cross(cell[(a + 1) % 3], cell[(a + 2) % 3])))
        nimg.append(max(int(np.ceil(r)), int(np.floor(r + span[a]))) if pbc[a] else 0)
    ijk = np.array([(i, j, k) for i in range(-nimg[0], nimg[0] + 1) for j in range(-nimg[1], nimg[1] + 1)
                    for k in range(-nimg[2], nimg[2] + 1)], dtype=np.float64)
    return np.array(nimg), (ijk[:, 0:1] * cell[0] + ijk[:, 1:2] * cell[1]) + ijk[:, 2:3] * cell[2]


def make_pbc():
    """Periodic neighbour lists from the REFERENCE build_graph on an explicit supercell: every
    image within range is materialised as atoms x_b + s_img; the neighbours of the home-image
    atoms are the periodic edges (a, b, img) with their distances."""
    out = {}
    for name, (n, seed, cell, pbc, cutoff) in PBC_CASES.items():
        cell = np.asarray(cell, dtype=np.float64)
        frac = np.random.default_rng(seed).uniform(0.0, 1.0, (n, 3))
        if name == "unwrapped5":
            frac[:, 0] += np.array([0.0, 1.0, -1.0, 2.0, 0.0])
        pos = frac @ cell
        nimg, shifts = _image_shifts(cell, pbc, cutoff, pos)
        n_img = shifts.shape[0]
        centre = n_img // 2
        sc = (pos[None, :, :] + shifts[:, None, :]).reshape(-1, 3)  # supercell atom img * n + b
        topo, geom = build_graph(AtomicSystem(sc, np.full(sc.shape[0], 6)), cutoff)
        home = (topo.edge_src >= centre * n) & (topo.edge_src < (centre + 1) * n)
        a = topo.edge_src[home] - centre * n
        b = topo.edge_recv[home] % n
        img = topo.edge_recv[home] // n
        d = geom.distances[home]
        order = np.lexsort((img, b, a))  # rows ordered by (a, b, img)
        out[f"{name}/pos"] = pos
        out[f"{name}/cell"] = cell
        out[f"{name}/pbc"] = np.array(pbc)
        out[f"{name}/cutoff"] = np.array(cutoff)
        out[f"{name}/nimg"] = nimg
        out[f"{name}/src"] = a[order]
        out[f"{name}/recv"] = b[order]
        out[f"{name}/img"] = img[order]
        out[f"{name}/dist"] = d[order]
        print(name, "edges", len(order), "images", nimg.tolist())
    out["numpy_version"] = np.array(np.__version__)
    np.savez_compressed(OUT / "pbc.npz", **out)


if __name__ == "__main__":
    parts = sys.argv[1:] or ["graphs", "models", "training", "relax", "pbc"]
    if "pbc" in parts:
        make_pbc()
    if "graphs" in parts:
        make_graphs()
    if "models" in parts:
        make_models()
    if "training" in parts:
        make_training()
    if "relax" in parts:
        make_relax()
    (OUT / "README.md").write_text(
        "Golden fixtures produced by `make_golden.py` from the reference package egn "
        "(/root/reference/pkg/src) with numpy " + np.__version__ + ".\n"
    )
