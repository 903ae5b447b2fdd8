"""Triplet-interaction kernels vs the reference's per-triplet formulation.

Reference formulation (record_tu, engine.py:118-149): per triplet t,
g_t = sbf_t @ Wmat with sbf from basis.py:54-73 and the fp64 angles of
graph.py:162-170; S[ji] = sum_t X[kj] * g_t.  The adjoints are computed with
the oracle's primitives (sbf_partials, angle_gradients) in fp64.
Tolerance: fp32 kernel vs fp64 reference, max-relative <= 1e-4.
"""

import numpy as np
import pytest
import torch

from conftest import TOL, max_rel
from oracle import egn_oracle as O

pytestmark = pytest.mark.gpu


def _ref(pos, cutoff, X, W, B):
    g = O.build_graph(pos, cutoff)
    K, L, dg = W.shape
    Wmat = W.reshape(K * L, dg)
    d_in = g.dist[g.trip_in]
    sbf = O.sbf(d_in, g.angles, K, L, cutoff) if g.trip_in.size else np.zeros((0, K * L))
    gt = sbf @ Wmat
    term = X[g.trip_in] * gt
    S = O.segment_sum(term, g.trip_out, g.src.size)
    # adjoint of J = sum(S * B)
    Bt = B[g.trip_out]
    X_bar = O.scatter_rows(gt * Bt, g.trip_in, g.src.size)
    W_bar = (sbf.T @ (X[g.trip_in] * Bt)).reshape(K, L, dg)
    sbf_bar = (X[g.trip_in] * Bt) @ Wmat.T
    pos_bar = np.zeros_like(pos)
    if g.trip_in.size:
        dd, da = O.sbf_partials(d_in, g.angles, K, L, cutoff)
        dist_bar = np.zeros(g.src.size)
        np.add.at(dist_bar, g.trip_in, (sbf_bar * dd).sum(1))
        ang_bar = (sbf_bar * da).sum(1)
        gk, gj, gi = O.angle_gradients(pos, g.src, g.recv, g.trip_in, g.trip_out)
        k, j, i = g.src[g.trip_in], g.recv[g.trip_in], g.recv[g.trip_out]
        np.add.at(pos_bar, k, ang_bar[:, None] * gk)
        np.add.at(pos_bar, i, ang_bar[:, None] * gi)
        np.add.at(pos_bar, j, ang_bar[:, None] * gj)
        c = dist_bar[:, None] * g.units
        np.add.at(pos_bar, g.recv, c)
        np.add.at(pos_bar, g.src, -c)
    return g, S, X_bar, W_bar, pos_bar


def _run(pos, cutoff, K, L, dg, seed=0):
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    bg = build_batch([pos], cutoff)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((bg.num_edges, dg))
    W = rng.standard_normal((K, L, dg)) / np.sqrt(K * L)
    B = rng.standard_normal((bg.num_edges, dg))
    g, S_ref, Xb_ref, Wb_ref, pb_ref = _ref(pos, cutoff, X, W, B)
    Xd = torch.tensor(X, dtype=torch.float32, device="cuda")
    Wd = torch.tensor(W, dtype=torch.float32, device="cuda")
    # max_degree known: tensor-core forward when d_g % 64 == 0 (triplet_tc.cu); unknown: CUDA-core kernels
    S = ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, Xd, Wd, cutoff, max_degree=bg.max_deg)
    S_cc = ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, Xd, Wd, cutoff)
    assert max_rel(S_cc.cpu().numpy(), S_ref) < TOL
    eg = torch.zeros((bg.num_edges, 4), device="cuda")
    Bd = torch.tensor(B, dtype=torch.float32, device="cuda")
    Xb, Wb = ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, Xd, Wd, cutoff, Bd, eg)
    pb = ops.positions_bwd(bg.edge_ptr, bg.rev, bg.geo, eg)
    torch.cuda.synchronize()
    return (S.cpu().numpy(), S_ref), (Xb.cpu().numpy(), Xb_ref), (Wb.cpu().numpy(), Wb_ref), (pb.cpu().numpy(), pb_ref), g


CASES = [
    # (n atoms, density, cutoff, K, L, dg)
    (20, 0.9, 1.5, 6, 4, 4),
    (30, 0.9, 1.5, 3, 2, 3),
    (40, 0.06, 6.0, 6, 7, 64),
    (40, 0.06, 6.0, 6, 7, 16),
    (40, 0.06, 6.0, 6, 7, 32),
    (30, 0.06, 6.0, 6, 7, 128),
    (24, 0.06, 6.0, 5, 7, 100),
    (30, 0.06, 6.0, 1, 1, 8),
    (60, 0.06, 6.0, 6, 8, 5),
    (150, 0.3, 6.0, 6, 7, 64),   # degree ~ 100: multiple row blocks and q tiles
    (120, 0.3, 6.0, 4, 7, 256),
]


@pytest.fixture(params=["auto", "sh", "pairwise"])
def triplet_path(request):
    """Every kernel test on each path: auto (pairwise centre tiles up to deg 64, the
    spherical-harmonic factorised kernels above), spherical-harmonic kernels for every
    centre, pairwise only (tensor-core kernels above deg 64)."""
    from paper_2203_09697_b200 import _lib

    old = _lib.call("egn_triplet_path", {"auto": 0, "sh": 1, "pairwise": 2}[request.param])
    yield request.param
    _lib.call("egn_triplet_path", old)


CASES += [
    (120, 0.8, 6.0, 6, 7, 64),   # near-complete graph, degree ~ 119: four 32-edge tiles per centre
    (200, 0.6, 6.0, 6, 7, 96),   # channel blocks 32 + 32 + 32
]


@pytest.mark.parametrize("case", CASES)
def test_triplet_fwd_bwd_matches_reference(case, triplet_path):
    n, rho, cutoff, K, L, dg = case
    pos, _ = O.random_cloud(n, rho, np.random.default_rng(n + dg))
    (S, Sr), (Xb, Xbr), (Wb, Wbr), (pb, pbr), g = _run(pos, cutoff, K, L, dg)
    assert g.trip_in.size > 0
    assert max_rel(S, Sr) < TOL
    assert max_rel(Xb, Xbr) < TOL
    assert max_rel(Wb, Wbr) < TOL
    assert max_rel(pb, pbr) < TOL


def test_triplet_collinear_and_low_degree():
    # collinear chain (zero angle subgradient), dimer (no triplets), isolated atom
    chain = np.zeros((4, 3))
    chain[:, 2] = np.arange(4.0)
    for pos, cutoff in ((chain, 1.5), (np.array([[0.0, 0, 0], [0, 0, 1.0]]), 1.5),
                        (np.array([[0.0, 0, 0], [5.0, 0, 0], [5.0, 1.0, 0]]), 1.5)):
        (S, Sr), (Xb, Xbr), (Wb, Wbr), (pb, pbr), g = _run(pos, cutoff, 6, 4, 8)
        assert max_rel(S, Sr) < TOL and max_rel(Xb, Xbr) < TOL and max_rel(Wb, Wbr) < TOL
        assert np.abs(pb - pbr).max() < 1e-4 * max(1.0, np.abs(pbr).max())


def test_degree_one_centres_zero_their_in_edge_gradient():
    """A centre of degree 1 has no triplets; its in-edge must get X_bar == 0 even
    when the output buffer starts as garbage."""
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    # atom 3 is bonded only to atom 2 (degree 1); the rest form a triangle
    pos = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, 0.8, 0], [0.5, 2.0, 0.0]])
    bg = build_batch([pos], 1.3)
    dg = 8
    X = torch.randn((bg.num_edges, dg), device="cuda")
    W = torch.randn((6, 4, dg), device="cuda")
    B = torch.randn((bg.num_edges, dg), device="cuda")
    eg = torch.zeros((bg.num_edges, 4), device="cuda")
    Xb = torch.full_like(X, float("nan"))
    ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, X, W, 1.3, B, eg, X_bar=Xb)
    assert torch.isfinite(Xb).all()
    _, _, Xb_ref, _, _ = _ref(pos, 1.3, X.double().cpu().numpy(), W.double().cpu().numpy(), B.double().cpu().numpy())
    assert max_rel(Xb.cpu().numpy(), Xb_ref) < TOL


def test_triplet_terms_and_sbf_debug_outputs():
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    pos, _ = O.random_cloud(25, 0.9, np.random.default_rng(3))
    bg = build_batch([pos], 1.5)
    g = O.build_graph(pos, 1.5)
    K, L, dg = 6, 4, 8
    rng = np.random.default_rng(0)
    X = rng.standard_normal((bg.num_edges, dg))
    W = rng.standard_normal((K, L, dg))
    sbf = O.sbf(g.dist[g.trip_in], g.angles, K, L, 1.5)
    P_ref = X[g.trip_in] * (sbf @ W.reshape(K * L, dg))
    P = ops.triplet_terms(bg.edge_ptr, bg.rev, bg.geo, bg.tri_ptr, bg.num_triplets,
                          torch.tensor(X, dtype=torch.float32, device="cuda"),
                          torch.tensor(W, dtype=torch.float32, device="cuda"), 1.5)
    assert max_rel(P.cpu().numpy(), P_ref) < TOL
    sb = ops.sbf(bg.geo, bg.edge_ptr, bg.tri_ptr, bg.num_triplets, K, L, 1.5)
    assert max_rel(sb.cpu().numpy(), sbf) < TOL
    rb = ops.rbf(bg.geo, K, 1.5)
    assert max_rel(rb.cpu().numpy(), O.rbf(g.dist, K, 1.5)) < TOL


def test_triplet_dimension_errors():
    from paper_2203_09697_b200 import ops
    from paper_2203_09697_b200.graph import build_batch

    bg = build_batch([np.array([[0.0, 0, 0], [0, 0, 1.0], [0, 1.0, 0]])], 1.5)
    X = torch.zeros((bg.num_edges, 8), device="cuda")
    with pytest.raises(ValueError):
        ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X, torch.zeros((6, 9, 8), device="cuda"), 1.5)
    with pytest.raises(ValueError):  # the C ABI takes <= 256 channels per call
        from paper_2203_09697_b200._lib import call, ptr, stream
        X3, W3 = torch.zeros((bg.num_edges, 300), device="cuda"), torch.zeros((6, 4, 300), device="cuda")
        S3 = torch.empty_like(X3)
        call("egn_triplet_fwd", ptr(bg.edge_ptr), ptr(bg.rev), ptr(bg.geo), bg.num_nodes, -1, ptr(X3), ptr(W3), 6, 4,
             300, 1.5, ptr(S3), None, stream())
    # ... and ops.triplet_fwd chunks wider embeddings exactly (per-channel independence)
    X3 = torch.randn((bg.num_edges, 300), device="cuda")
    W3 = torch.randn((6, 4, 300), device="cuda")
    S3 = ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X3, W3, 1.5)
    S_lo = ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X3[:, :256].contiguous(), W3[:, :, :256].contiguous(), 1.5)
    assert torch.equal(S3[:, :256], S_lo)


@pytest.mark.parametrize("n,k,ne,strided,prod", [(128, 6, 5000, False, False), (64, 6, 3001, True, False),
                                                 (32, 8, 777, False, False), (48, 3, 1000, False, True),
                                                 (8, 6, 513, False, False), (128, 1, 2, False, False),
                                                 (64, 6, 4000, False, True)])
def test_rbf_linear_bwd_vs_fp64(n, k, ne, strided, prod):
    """Basis-linear adjoint (warp-per-edge path for N = 32, 64, 128; tiled path otherwise):
    rbf_bar += g W, W_bar = g^T rbf, b_bar = column sums of g, vs fp64 torch."""
    from paper_2203_09697_b200 import ops

    gen = torch.Generator(device="cuda").manual_seed(ne)
    rbf_t = torch.rand((ne, k), device="cuda", generator=gen)
    w = torch.randn((n, k), device="cuda", generator=gen)
    gfull = torch.randn((ne, n + (16 if strided else 0)), device="cuda", generator=gen)
    g = gfull[:, :n]
    rbf_bar0 = torch.randn((ne, k), device="cuda", generator=gen)
    rbf_bar = rbf_bar0.clone()
    w_bar = torch.empty((n, k), device="cuda")
    b_bar = torch.empty((n,), device="cuda")
    g2 = torch.randn_like(g) if prod else None
    ops.rbf_linear_bwd(rbf_t, w, g, rbf_bar, w_bar, b_bar, g2=g2)
    gd, rd, wd = g.double(), rbf_t.double(), w.double()
    if prod:
        gd = gd * g2.double()
    ref_rb = rbf_bar0.double() + gd @ wd
    assert max_rel(rbf_bar.cpu().numpy(), ref_rb.cpu().numpy()) < 1e-5
    assert max_rel(w_bar.cpu().numpy(), (gd.t() @ rd).cpu().numpy()) < 1e-5
    assert max_rel(b_bar.cpu().numpy(), gd.sum(0).cpu().numpy()) < 1e-5


@pytest.mark.parametrize("g,dv,du", [(32, 128, 128), (1, 16, 24), (33, 7, 5), (5, 200, 96)])
def test_graph_mlp_vs_fp64(g, dv, du):
    """Fused GU block (egn_graph_mlp_fwd / _bwd) vs fp64 torch: u += silu(s W1^T + b1) W2^T + b2
    and every adjoint."""
    from paper_2203_09697_b200 import ops

    gen = torch.Generator(device="cuda").manual_seed(g * 1000 + dv)
    s = torch.randn((g, dv), device="cuda", generator=gen)
    w1 = torch.randn((du, dv), device="cuda", generator=gen) * dv ** -0.5
    b1 = torch.randn((du,), device="cuda", generator=gen)
    w2 = torch.randn((du, du), device="cuda", generator=gen) * du ** -0.5
    b2 = torch.randn((du,), device="cuda", generator=gen)
    u0 = torch.randn((g, du), device="cuda", generator=gen)
    u = u0.clone()
    pre, act = ops.graph_mlp_fwd(s, w1, b1, w2, b2, u)
    sd, w1d, b1d, w2d, b2d = (t.double() for t in (s, w1, b1, w2, b2))
    pre_r = sd @ w1d.t() + b1d
    act_r = torch.nn.functional.silu(pre_r)
    u_r = u0.double() + act_r @ w2d.t() + b2d
    assert max_rel(pre.cpu().numpy(), pre_r.cpu().numpy()) < 1e-5
    assert max_rel(act.cpu().numpy(), act_r.cpu().numpy()) < 1e-5
    assert max_rel(u.cpu().numpy(), u_r.cpu().numpy()) < 1e-5
    u_bar = torch.randn((g, du), device="cuda", generator=gen)
    gw1, gb1 = torch.empty_like(w1), torch.empty_like(b1)
    gw2, gb2 = torch.empty_like(w2), torch.empty_like(b2)
    s_bar = ops.graph_mlp_bwd(u_bar, s, pre, act, w1, w2, gw1, gb1, gw2, gb2)
    ub = u_bar.double()
    sg = torch.sigmoid(pre_r)
    pb = (ub @ w2d) * sg * (1 + pre_r * (1 - sg))
    for got, ref in ((s_bar, pb @ w1d), (gw1, pb.t() @ sd), (gb1, pb.sum(0)), (gw2, ub.t() @ act_r),
                     (gb2, ub.sum(0))):
        assert max_rel(got.cpu().numpy(), ref.cpu().numpy()) < 1e-5


@pytest.mark.parametrize("basis", [0, 1, 2])
@pytest.mark.parametrize("n,density,dg,mode", [(40, 0.06, 64, 0), (300, 0.9, 64, 0), (40, 0.06, 320, 0),
                                                (40, 0.06, 64, 2)])
def test_triplet_bwd_phases_match_single_call(n, density, dg, mode, basis):
    """egn_triplet_bwd_ex / egn_triplet_bwd_basis_ex: the angle phase (1) and the rest (2), run
    on two streams, give the bit-identical X_bar, W_bar and edge_grad of the single call (3);
    includes centres above the small-degree range (dense cloud), a width above 256 (channel
    chunks), the pairwise path and every basis (0 Gaussian, 1 GemNet CBF, 2 DimeNet SBF)."""
    from paper_2203_09697_b200 import _lib, ops
    from paper_2203_09697_b200.graph import build_batch

    rng = np.random.default_rng(n + dg)
    pos, _ = O.random_cloud(n, density, rng)
    old = _lib.call("egn_triplet_path", mode)
    try:
        bg = build_batch([pos], 6.0)
        X = torch.randn((bg.num_edges, dg), device="cuda")
        W = torch.randn((6, 7, dg), device="cuda") / 6.5
        Sb = torch.randn((bg.num_edges, dg), device="cuda")
        eg0 = torch.randn((bg.num_edges, 4), device="cuda")
        eg1 = eg0.clone()
        xb, wb = ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, X, W, 6.0, Sb, eg0, max_degree=bg.max_deg,
                                 basis=basis)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            assert ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, X, W, 6.0, Sb, eg1, max_degree=bg.max_deg,
                                   basis=basis, phases=1) == (None, None)
        xb2, wb2 = ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, X, W, 6.0, Sb, eg1, max_degree=bg.max_deg,
                                   basis=basis, phases=2)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
    finally:
        _lib.call("egn_triplet_path", old)
    assert torch.equal(xb, xb2) and torch.equal(wb, wb2)
    assert torch.equal(eg0, eg1)
