"""Neighbour list / triplets / reverse edges / geometry on the GPU vs the reference.

Topology is compared bit-exactly against the golden fixtures (reference
outputs) and against the oracle on extra random systems, including batched
(disjoint-union) builds."""

import numpy as np
import pytest
import torch

from conftest import max_rel
from oracle import egn_oracle as O

pytestmark = pytest.mark.gpu


def _gpu_graph(pos, cutoff):
    from paper_2203_09697_b200.graph import build_graph

    topo, geom = build_graph(pos, cutoff)
    return topo, geom


def test_graph_fixtures_bit_exact(graphs_golden):
    data, names = graphs_golden
    for name in names:
        pos = data[f"{name}/pos"]
        topo, geom = _gpu_graph(pos, float(data[f"{name}/cutoff"]))
        for key, val in (("src", topo.edge_src), ("recv", topo.edge_recv), ("trip_in", topo.trip_in),
                         ("trip_out", topo.trip_out), ("rev", topo.reverse_edges())):
            np.testing.assert_array_equal(val.cpu().numpy(), data[f"{name}/{key}"], err_msg=f"{name}/{key}")
        np.testing.assert_array_equal(geom.distances.cpu().numpy(), data[f"{name}/dist"], err_msg=name)
        np.testing.assert_array_equal(geom.unit_vectors.cpu().numpy(), data[f"{name}/units"], err_msg=name)
        np.testing.assert_allclose(geom.angles.cpu().numpy(), data[f"{name}/angles"], rtol=0, atol=1e-12)
        topo.validate()


@pytest.mark.parametrize("seed", range(50))
def test_random_clouds_bit_exact_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 120))
    rho = float(rng.choice([0.06, 0.2, 0.9]))
    pos, _ = O.random_cloud(n, rho, rng)
    cutoff = float(rng.choice([1.5, 3.0, 6.0]))
    ref = O.build_graph(pos, cutoff)
    topo, geom = _gpu_graph(pos, cutoff)
    np.testing.assert_array_equal(topo.edge_src.cpu().numpy(), ref.src)
    np.testing.assert_array_equal(topo.edge_recv.cpu().numpy(), ref.recv)
    np.testing.assert_array_equal(topo.trip_in.cpu().numpy(), ref.trip_in)
    np.testing.assert_array_equal(topo.trip_out.cpu().numpy(), ref.trip_out)
    np.testing.assert_array_equal(topo.reverse_edges().cpu().numpy(), ref.rev)
    np.testing.assert_array_equal(geom.distances.cpu().numpy(), ref.dist)


def test_batched_union_equals_per_graph():
    from paper_2203_09697_b200.graph import build_batch, topology_of

    rng = np.random.default_rng(7)
    systems = [O.random_cloud(int(k), 0.06, rng)[0] for k in (30, 1, 45, 2, 64)]
    bg = build_batch(systems, 6.0)
    topo = topology_of(bg)
    e_off = t_off = n_off = 0
    src = topo.edge_src.cpu().numpy()
    kj = topo.trip_in.cpu().numpy()
    ji = topo.trip_out.cpu().numpy()
    for pos in systems:
        ref = O.build_graph(pos, 6.0)
        ne, nt = ref.src.size, ref.trip_in.size
        np.testing.assert_array_equal(src[e_off:e_off + ne], ref.src + n_off)
        np.testing.assert_array_equal(kj[t_off:t_off + nt], ref.trip_in + e_off)
        np.testing.assert_array_equal(ji[t_off:t_off + nt], ref.trip_out + e_off)
        e_off += ne
        t_off += nt
        n_off += pos.shape[0]
    assert (bg.num_edges, bg.num_triplets) == (e_off, t_off)


def test_enumerate_triplets_api_and_errors():
    from paper_2203_09697_b200.graph import GraphTopology, build_graph, enumerate_triplets

    tri = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, np.sqrt(3) / 2, 0]])
    topo, _ = build_graph(tri, 1.5)
    kj, ji = enumerate_triplets(topo)
    assert torch.equal(kj, topo.trip_in) and torch.equal(ji, topo.trip_out)
    e = torch.empty(0, dtype=torch.int64, device="cuda")
    a, b = enumerate_triplets(3, e, e)
    assert a.numel() == 0 and b.numel() == 0
    lop = GraphTopology(2, torch.tensor([0], device="cuda"), torch.tensor([1], device="cuda"), e, e)
    with pytest.raises(ValueError):
        lop.reverse_edges()
    with pytest.raises(ValueError):
        build_graph(tri, 0.0)


def test_large_graph_neighbor_counts():
    """1k atoms, mean degree ~50: bit-exact edges and triplet count."""
    rng = np.random.default_rng(5)
    pos, _ = O.random_cloud(1000, 0.1, rng)
    ref_src, ref_recv = O.neighbor_list(pos, 5.0)
    topo, geom = _gpu_graph(pos, 5.0)
    np.testing.assert_array_equal(topo.edge_src.cpu().numpy(), ref_src)
    np.testing.assert_array_equal(topo.edge_recv.cpu().numpy(), ref_recv)
    deg = np.bincount(ref_src, minlength=1000)
    assert topo.num_triplets == int((deg * (deg - 1)).sum())
    assert max_rel(geom.distances.cpu().numpy(), np.sqrt(((pos[ref_recv] - pos[ref_src]) ** 2).sum(1))) == 0.0


@pytest.mark.parametrize("name", ["cubic4", "triclinic5", "slab6", "self_image1", "unwrapped5"])
def test_periodic_graph_bit_exact(name):
    """GPU periodic neighbour list / reverse edges / triplets / geometry vs the oracle
    restatement (itself pinned to the reference on an explicit supercell)."""
    from conftest import load_golden
    from paper_2203_09697_b200 import AtomicSystem
    from paper_2203_09697_b200.graph import build_batch, geometry_of, topology_of

    gd = load_golden("pbc.npz")
    pos, cell, pbc, cutoff = gd[f"{name}/pos"], gd[f"{name}/cell"], gd[f"{name}/pbc"], float(gd[f"{name}/cutoff"])
    ref = O.build_graph_pbc(pos, cell, pbc, cutoff)
    bg = build_batch(AtomicSystem(pos, np.full(pos.shape[0], 6), cell=cell, pbc=tuple(pbc)), cutoff)
    topo, geom = topology_of(bg), geometry_of(bg)
    np.testing.assert_array_equal(bg.img.cpu().numpy(), ref.img)
    for key, val in (("src", topo.edge_src), ("recv", topo.edge_recv), ("trip_in", topo.trip_in),
                     ("trip_out", topo.trip_out), ("rev", topo.reverse_edges())):
        np.testing.assert_array_equal(val.cpu().numpy(), getattr(ref, key), err_msg=key)
    np.testing.assert_array_equal(geom.distances.cpu().numpy(), ref.dist)
    np.testing.assert_array_equal(geom.unit_vectors.cpu().numpy(), ref.units)
    np.testing.assert_allclose(geom.angles.cpu().numpy(), ref.angles, rtol=0, atol=1e-12)


def test_periodic_graph_symmetric_at_cutoff_boundary():
    """Own +-2-cell images exactly at the cutoff (cell 3, cutoff 6): every edge has its reverse
    (no rev = -1 reaches the model), and the GPU graph equals the oracle bit for bit."""
    from paper_2203_09697_b200 import AtomicSystem
    from paper_2203_09697_b200.graph import build_batch

    rng = np.random.default_rng(7)
    cell = np.eye(3) * 3.0
    for _ in range(20):
        pos = rng.uniform(0.0, 3.0, size=(2, 3))
        ref = O.build_graph_pbc(pos, cell, (True, True, True), 6.0)
        bg = build_batch(AtomicSystem(pos, np.full(2, 6), cell=cell, pbc=(True, True, True)), 6.0)
        rev = bg.rev.cpu().numpy()
        assert rev.min() >= 0
        np.testing.assert_array_equal(rev, ref.rev)
        np.testing.assert_array_equal(bg.src.cpu().numpy(), ref.src)
        np.testing.assert_array_equal(bg.img.cpu().numpy(), ref.img)


def test_periodic_batch_mixes_periodic_and_open_graphs():
    from paper_2203_09697_b200 import AtomicSystem
    from paper_2203_09697_b200.graph import build_batch, topology_of

    rng = np.random.default_rng(3)
    cell = np.array([[4.0, 0, 0], [0.5, 3.8, 0], [0, 0.3, 4.2]])
    p1 = rng.uniform(0, 1, (7, 3)) @ cell
    p2, _ = O.random_cloud(12, 0.2, rng)
    systems = [AtomicSystem(p1, np.full(7, 6), cell=cell, pbc=(True, True, True)), AtomicSystem(p2, np.full(12, 6))]
    bg = build_batch(systems, 3.0)
    t = topology_of(bg)
    r1 = O.build_graph_pbc(p1, cell, (True, True, True), 3.0)
    r2 = O.build_graph(p2, 3.0)
    e1 = r1.src.size
    np.testing.assert_array_equal(t.edge_src.cpu().numpy()[:e1], r1.src)
    np.testing.assert_array_equal(t.edge_recv.cpu().numpy()[:e1], r1.recv)
    np.testing.assert_array_equal(t.edge_src.cpu().numpy()[e1:], r2.src + 7)
    np.testing.assert_array_equal(t.edge_recv.cpu().numpy()[e1:], r2.recv + 7)
    np.testing.assert_array_equal(bg.geo[:, 3].cpu().numpy(), np.concatenate([r1.dist, r2.dist]).astype(np.float32))


@pytest.mark.parametrize("d", [128, 64, 8, 6, 200])
def test_aggregate_in_edges_vs_numpy(d):
    """out[v] = sum over the in-edges of v (reverse of v's out-edges) of x rows, in CSR order
    (16-byte path for d % 4 == 0, scalar path otherwise; two 128-column chunks at d = 200)."""
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    rng = np.random.default_rng(d)
    systems = [O.random_cloud(n, 0.06, rng)[0] for n in (40, 1, 57)]
    bg = build_batch(systems, 6.0)
    x = torch.randn((bg.num_edges, d), device="cuda", dtype=torch.float32)
    out = ops.aggregate_in_edges(bg.edge_ptr, bg.rev, x).cpu().numpy()
    xe = x.cpu().numpy().astype(np.float64)
    ptr, rev = bg.edge_ptr.cpu().numpy(), bg.rev.cpu().numpy()
    ref = np.stack([xe[rev[ptr[v]:ptr[v + 1]]].sum(axis=0) if ptr[v + 1] > ptr[v] else np.zeros(d)
                    for v in range(bg.num_nodes)])
    assert max_rel(out, ref) < 1e-5


@pytest.mark.parametrize("d,rows,acc", [(128, 1001, False), (128, 1000, True), (64, 7, True), (6, 33, False)])
def test_gather_rows_vs_torch(d, rows, acc):
    """out[r] (+)= x[idx[r]] (16-byte path for d % 4 == 0, odd row counts, accumulate)."""
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(d + rows)
    x = torch.randn((500, d), device="cuda", generator=g)
    idx = torch.randint(0, 500, (rows,), device="cuda", generator=g, dtype=torch.int32)
    base = torch.randn((rows, d), device="cuda", generator=g)
    out = base.clone()
    ops.gather_rows(idx, x, out=out, accumulate=acc)
    ref = (base if acc else 0) + x[idx.long()]
    assert torch.equal(out, ref)


@pytest.mark.parametrize("seed,k", [(0, 4), (1, 8), (2, 12), (3, 1000)])
def test_neighbour_cap_bit_exact(seed, k):
    """GPU max_neighbors cap vs the oracle restatement: edges, reverse edges, triplets, geometry."""
    from paper_2203_09697_b200.graph import build_batch, geometry_of, topology_of

    rng = np.random.default_rng(700 + seed)
    pos, _ = O.random_cloud(int(rng.integers(20, 70)), 0.2, rng)
    ref = O.cap_graph(O.build_graph(pos, 4.5), pos, k)
    bg = build_batch(pos, 4.5, max_neighbors=k)
    topo, geom = topology_of(bg), geometry_of(bg)
    for key, val in (("src", topo.edge_src), ("recv", topo.edge_recv), ("trip_in", topo.trip_in),
                     ("trip_out", topo.trip_out), ("rev", topo.reverse_edges())):
        np.testing.assert_array_equal(val.cpu().numpy(), getattr(ref, key), err_msg=key)
    np.testing.assert_array_equal(geom.distances.cpu().numpy(), ref.dist)
    assert bg.max_deg <= k


def test_neighbour_cap_periodic():
    from conftest import load_golden
    from paper_2203_09697_b200 import AtomicSystem
    from paper_2203_09697_b200.graph import build_batch, topology_of

    gd = load_golden("pbc.npz")
    pos, cell, cutoff = gd["triclinic5/pos"], gd["triclinic5/cell"], float(gd["triclinic5/cutoff"])
    ref = O.cap_graph(O.build_graph_pbc(pos, cell, (True, True, True), cutoff), pos, 6)
    bg = build_batch(AtomicSystem(pos, np.full(5, 6), cell=cell, pbc=(True, True, True)), cutoff, max_neighbors=6)
    t = topology_of(bg)
    np.testing.assert_array_equal(t.edge_src.cpu().numpy(), ref.src)
    np.testing.assert_array_equal(t.edge_recv.cpu().numpy(), ref.recv)
    np.testing.assert_array_equal(bg.img.cpu().numpy(), ref.img)
    np.testing.assert_array_equal(t.reverse_edges().cpu().numpy(), ref.rev)


def test_device_utilities():
    """egn_zero / egn_hadamard / egn_transpose / egn_csr_ptr (the step's non-framework
    elementwise work) against torch."""
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(3)
    for n in (0, 1, 7, 4096, 4099):
        a = torch.randn(n, device="cuda", generator=g)
        b = torch.randn(n, device="cuda", generator=g)
        assert torch.equal(ops.hadamard(a, b), a * b)
    t = torch.randn((1000, 64), device="cuda", generator=g)
    ops.zero_(t)
    assert not t.any()
    src = torch.randn((42, 70), device="cuda", generator=g)
    big = torch.full((70, 50), float("nan"), device="cuda")
    ops.transpose_into(src, big[:, 3:45])
    assert torch.equal(big[:, 3:45], src.t())
    assert torch.isnan(big[:, :3]).all() and torch.isnan(big[:, 45:]).all()
    keys = torch.tensor([0, 0, 1, 3, 3, 3, 6], dtype=torch.int64, device="cuda")
    assert ops.csr_ptr(keys, 8).cpu().tolist() == [0, 2, 3, 3, 6, 6, 6, 7, 7]
    with pytest.raises(ValueError):
        ops.hadamard(a, torch.randn(n + 1, device="cuda"))
