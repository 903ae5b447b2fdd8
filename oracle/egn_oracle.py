"""CPU fp64 oracle for the EGN (DimeNet++/GemNet-T style) training hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, and only as the checker
or as the timed CPU baseline.

This is a plain-numpy restatement of the reference package ``egn``
(``/root/reference/pkg/src/egn``; paths below are relative to it).  The
reference runs its model through a recorded tape of primitives
(``tape.py``); here the same primitive sequence is written out explicitly
with hand-derived adjoints, in the same order, so that it follows the
reference algorithm (per-triplet gathers, ``np.add.at`` scatters, dense
``x @ W.T`` linears, branch-stable SiLU).

Parity pin: ``tests/golden/make_golden.py`` runs the reference itself
(``ModelTape``, ``build_graph``, ``init_params``) in this container and
writes fixtures under ``tests/golden/``; ``tests/test_oracle.py`` checks
this module against every fixture (bit-exact topology, 1e-10 relative for
floating-point outputs and gradients).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DIMENET = "dimenet-style"
GEMNET = "gemnet-style"
MAX_Z = 118
COLLINEAR_EPS = 1e-14  # graph.py:17-19


# ---------------------------------------------------------------------------
# config / params  (config.py:13-64, params.py:30-108)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Config:
    variant: str = DIMENET
    blocks: int = 2
    d_u: int = 4
    d_v: int = 6
    d_e: int = 8
    d_t: int = 4
    d_bil: int = 4
    k_rbf: int = 6
    l_sbf: int = 4
    cutoff: float = 1.5
    seed: int = 0
    # "gaussian": the reference's surrogate bases (egn/basis.py); "bessel": the DimeNet++ / GemNet
    # bases (no reference counterpart -- restated below from the published
    # definitions with scipy.special, independent of the CUDA kernels)
    basis: str = "gaussian"


def param_specs(c: Config) -> list[tuple[str, tuple[int, ...], int]]:
    """(name, shape, fan_in) in declaration order; params.py:30-70."""
    s = [
        ("atom_embedding", (MAX_Z, c.d_v), 1),
        ("edge_init.w", (c.d_e, c.k_rbf), c.k_rbf),
        ("edge_init.b", (c.d_e,), c.k_rbf),
    ]
    kl = c.k_rbf * c.l_sbf
    for b in range(c.blocks):
        p = f"block{b}."
        s += [
            (p + "tu.down", (c.d_t, c.d_e), c.d_e),
            (p + "tu.rbf_gate", (c.d_t, c.k_rbf), c.k_rbf),
            (p + "tu.sbf_gate", (c.d_t, kl), kl),
        ]
        if c.variant == GEMNET:
            s += [
                (p + "tu.bilinear_a", (c.d_bil, c.d_t), c.d_t),
                (p + "tu.bilinear_b", (c.d_bil, c.d_t), c.d_t),
                (p + "tu.bilinear_proj", (c.d_t, c.d_bil), c.d_bil),
            ]
        s += [
            (p + "tu.up", (c.d_e, c.d_t), c.d_t),
            (p + "eu.w1", (c.d_e, 2 * c.d_e), 2 * c.d_e),
            (p + "eu.b1", (c.d_e,), 2 * c.d_e),
            (p + "eu.w2", (c.d_e, c.d_e), c.d_e),
            (p + "eu.b2", (c.d_e,), c.d_e),
            (p + "nu.w1", (c.d_v, c.d_e), c.d_e),
            (p + "nu.b1", (c.d_v,), c.d_e),
            (p + "nu.w2", (c.d_v, c.d_v), c.d_v),
            (p + "nu.b2", (c.d_v,), c.d_v),
        ]
        if c.variant == GEMNET:
            s += [
                (p + "eu2.w1", (c.d_e, c.d_e + c.d_v), c.d_e + c.d_v),
                (p + "eu2.b1", (c.d_e,), c.d_e + c.d_v),
                (p + "eu2.w2", (c.d_e, c.d_e), c.d_e),
                (p + "eu2.b2", (c.d_e,), c.d_e),
                (p + "sym.w", (c.d_e, c.d_e), c.d_e),
            ]
        s += [
            (p + "gu.w1", (c.d_u, c.d_v), c.d_v),
            (p + "gu.b1", (c.d_u,), c.d_v),
            (p + "gu.w2", (c.d_u, c.d_u), c.d_u),
            (p + "gu.b2", (c.d_u,), c.d_u),
        ]
    s += [("energy_head.w", (1, c.d_u), c.d_u), ("energy_head.b", (1,), c.d_u)]
    if c.variant == GEMNET:
        s.append(("force_head.w", (1, c.d_e), c.d_e))
    return s


def init_params(c: Config) -> dict[str, np.ndarray]:
    """U(+-1/sqrt(fan_in)) per array from SeedSequence(seed).spawn; params.py:94-108."""
    specs = param_specs(c)
    children = np.random.SeedSequence(c.seed).spawn(len(specs))
    out = {}
    for (name, shape, fan_in), child in zip(specs, children):
        rng = np.random.default_rng(child)
        bound = 1.0 / np.sqrt(fan_in)
        out[name] = rng.uniform(-bound, bound, size=shape)
    return out


# ---------------------------------------------------------------------------
# synthetic systems (system.py:129-166) -- input generator for the harness
# ---------------------------------------------------------------------------

CLOUD_SPECIES = (1, 6, 7, 8, 14, 29)


def random_cloud(n: int, density: float, rng: np.random.Generator, max_tries_per_atom: int = 500):
    """Rejection-sampled cube cloud, min pair distance 0.8*density^(-1/3)."""
    spacing = density ** (-1.0 / 3.0)
    min_dist = 0.8 * spacing
    side = (n / density) ** (1.0 / 3.0)
    placed = np.empty((n, 3), dtype=np.float64)
    for i in range(n):
        for _ in range(max_tries_per_atom):
            cand = rng.uniform(0.0, side, size=3)
            if i == 0:
                placed[0] = cand
                break
            d = np.sqrt(((placed[:i] - cand) ** 2).sum(axis=1))
            if d.min() >= min_dist:
                placed[i] = cand
                break
        else:
            raise RuntimeError(f"could not place atom {i + 1}/{n} at density {density}")
    z = rng.choice(CLOUD_SPECIES, size=n).astype(np.int64)
    return placed, z


# ---------------------------------------------------------------------------
# graph (graph.py:82-203)
# ---------------------------------------------------------------------------


@dataclass
class Graph:
    n: int
    src: np.ndarray
    recv: np.ndarray
    trip_in: np.ndarray  # id3_kj
    trip_out: np.ndarray  # id3_ji
    dist: np.ndarray
    units: np.ndarray
    angles: np.ndarray
    rev: np.ndarray = field(default=None)
    # periodic graphs: edge vectors (x_recv - x_src) + shift and the
    # image index per edge; None for the reference's non-periodic graphs
    vec: np.ndarray = field(default=None)
    img: np.ndarray = field(default=None)


def neighbor_list(pos: np.ndarray, cutoff: float):
    """Dense fp64 distances, mask (0, cutoff], row-major nonzero; graph.py:89-96."""
    diff = pos[None, :, :] - pos[:, None, :]
    dist = np.sqrt((diff * diff).sum(axis=2))
    mask = (dist > 0.0) & (dist <= cutoff)
    np.fill_diagonal(mask, False)
    src, recv = np.nonzero(mask)
    return src.astype(np.int64), recv.astype(np.int64)


def enumerate_triplets(n: int, src: np.ndarray, recv: np.ndarray):
    """((k->j),(j->i)), k != i, sorted by (out, in); graph.py:106-139."""
    if src.size == 0:
        e = np.empty(0, dtype=np.int64)
        return e, e
    order = np.argsort(recv, kind="stable").astype(np.int64)
    bounds = np.searchsorted(recv[order], np.arange(n + 1))
    ins, outs = [], []
    for out_edge in range(src.size):
        j = src[out_edge]
        cand = order[bounds[j] : bounds[j + 1]]
        cand = cand[src[cand] != recv[out_edge]]
        if cand.size:
            ins.append(cand)
            outs.append(np.full(cand.size, out_edge, dtype=np.int64))
    if not ins:
        e = np.empty(0, dtype=np.int64)
        return e, e
    return np.concatenate(ins), np.concatenate(outs)


def reverse_edges(src: np.ndarray, recv: np.ndarray) -> np.ndarray:
    """rev[e] = index of (recv_e, src_e); graph.py:40-55 (dict restated as a sort)."""
    n_e = src.size
    if n_e == 0:
        return np.empty(0, dtype=np.int64)
    key = {(int(a), int(b)): i for i, (a, b) in enumerate(zip(src, recv))}
    rev = np.empty(n_e, dtype=np.int64)
    for i in range(n_e):
        pair = (int(recv[i]), int(src[i]))
        if pair not in key:
            raise ValueError(f"edge {i} has no reverse edge {pair}")
        rev[i] = key[pair]
    return rev


def triplet_vectors(pos, src, recv, trip_in, trip_out, vec=None, rev=None):
    """graph.py:153-159.  Periodic graphs: v1 = vector of the out-edge j -> k' (the reverse of
    the in-edge), v2 = vector of the out-edge j -> i', i.e. the images the edges connect."""
    k = src[trip_in]
    j = recv[trip_in]
    i = recv[trip_out]
    if vec is not None:
        return k, j, i, vec[rev[trip_in]], vec[trip_out]
    return k, j, i, pos[k] - pos[j], pos[i] - pos[j]


def triplet_angles(pos, src, recv, trip_in, trip_out, vec=None, rev=None):
    """atan2(|v1 x v2|, v1.v2); graph.py:162-170."""
    if trip_in.size == 0:
        return np.empty(0, dtype=np.float64)
    _, _, _, v1, v2 = triplet_vectors(pos, src, recv, trip_in, trip_out, vec, rev)
    cross = np.cross(v1, v2)
    s = np.sqrt((cross * cross).sum(axis=1))
    c = (v1 * v2).sum(axis=1)
    return np.arctan2(s, c)


def angle_gradients(pos, src, recv, trip_in, trip_out, vec=None, rev=None):
    """Closed-form d(angle)/d(x_k, x_j, x_i), zero subgradient when collinear; graph.py:173-197."""
    if trip_in.size == 0:
        z = np.zeros((0, 3))
        return z, z, z
    _, _, _, v1, v2 = triplet_vectors(pos, src, recv, trip_in, trip_out, vec, rev)
    cross = np.cross(v1, v2)
    s = np.sqrt((cross * cross).sum(axis=1))
    ok = s > COLLINEAR_EPS
    safe = np.where(ok, s, 1.0)
    nhat = cross / safe[:, None]
    n1 = np.sqrt((v1 * v1).sum(axis=1))
    n2 = np.sqrt((v2 * v2).sum(axis=1))
    g_k = np.cross(v1 / n1[:, None], nhat) / n1[:, None]
    g_i = np.cross(nhat, v2 / n2[:, None]) / n2[:, None]
    g_k[~ok] = 0.0
    g_i[~ok] = 0.0
    return g_k, -(g_k + g_i), g_i


def build_graph(pos: np.ndarray, cutoff: float) -> Graph:
    """graph.py:82-103 (+ reverse edges, graph.py:40-55)."""
    if cutoff <= 0:
        raise ValueError("cutoff must be positive")
    pos = np.asarray(pos, dtype=np.float64)
    n = pos.shape[0]
    src, recv = neighbor_list(pos, cutoff)
    trip_in, trip_out = enumerate_triplets(n, src, recv)
    diff = pos[recv] - pos[src]
    dist = np.sqrt((diff * diff).sum(axis=1))
    units = diff / dist[:, None] if src.size else np.zeros((0, 3))
    angles = triplet_angles(pos, src, recv, trip_in, trip_out)
    rev = reverse_edges(src, recv)
    return Graph(n, src, recv, trip_in, trip_out, dist, units, angles, rev)


# ---------------------------------------------------------------------------
# periodic cells (no reference counterpart -- pinned against the
# reference build_graph on an explicit supercell, tests/golden/pbc.npz)
# ---------------------------------------------------------------------------


def image_ranges(cell, pbc, cutoff, pos=None):
    """Images per periodic axis: max(ceil(r), floor(r + span)), r = cutoff / h_a with
    h_a = |det C| / |c_b x c_c| and span the extent of the fractional coordinates along a
    (< 1 for atoms inside one cell, where this is ceil(r))."""
    cell = np.asarray(cell, dtype=np.float64)
    vol = abs(np.linalg.det(cell))
    span = np.zeros(3)
    if pos is not None and len(pos):
        frac = np.asarray(pos, dtype=np.float64) @ np.linalg.inv(cell)
        span = frac.max(axis=0) - frac.min(axis=0)
    out = np.zeros(3, dtype=np.int64)
    for a in range(3):
        if pbc[a]:
            r = cutoff / (vol / np.linalg.norm(np.cross(cell[(a + 1) % 3], cell[(a + 2) % 3])))
            out[a] = max(int(np.ceil(r)), int(np.floor(r + span[a])))
    return out


def image_shifts(cell, nimg):
    """Shift of every image index img = ((i+na)(2nb+1) + (j+nb))(2nc+1) + (k+nc):
    s = (i c0 + j c1) + k c2, evaluated left to right in fp64."""
    cell = np.asarray(cell, dtype=np.float64)
    na, nb, nc = (int(x) for x in nimg)
    ijk = np.array([(i, j, k) for i in range(-na, na + 1) for j in range(-nb, nb + 1) for k in range(-nc, nc + 1)],
                   dtype=np.float64)
    return (ijk[:, 0:1] * cell[0] + ijk[:, 1:2] * cell[1]) + ijk[:, 2:3] * cell[2]


def build_graph_pbc(pos, cell, pbc, cutoff) -> Graph:
    """Periodic cutoff graph: edges (a, b, img) with 0 < |(x_b - x_a) + s_img| <= cutoff
    (not b == a in the home image), rows ordered by (b, img); reverse = (b, a, mirrored
    img); triplets of out-edge (j -> i') pair it with every in-edge (k -> j) that is not its
    own reverse, in the order of the centre's out-edges (for a non-periodic cell this is
    the reference's enumerate_triplets order)."""
    if cutoff <= 0:
        raise ValueError("cutoff must be positive")
    pos = np.asarray(pos, dtype=np.float64)
    n = pos.shape[0]
    nimg = image_ranges(cell, pbc, cutoff, pos)
    shifts = image_shifts(cell, nimg)
    n_img = shifts.shape[0]
    centre = n_img // 2
    # candidate (a, b, img): vector (x_b - x_a) + s, same operation order as the kernels.  This
    # form is exactly antisymmetric under (a, b, s) -> (b, a, -s), so every edge has its
    # reverse; it equals the supercell reference's (x_b + s) - x_a to within an ulp
    diff = (pos[None, None, :, :] - pos[:, None, None, :]) + shifts[None, :, None, :]  # [a, img, b, 3]
    dist = np.sqrt((diff * diff).sum(axis=3))
    mask = (dist > 0.0) & (dist <= cutoff)
    mask[np.arange(n), centre, np.arange(n)] = False
    mask = mask.transpose(0, 2, 1)  # [a, b, img]: row-major nonzero = (a, b, img) order
    src, recv, img = (x.astype(np.int64) for x in np.nonzero(mask))
    shift = shifts[img]
    vec = (pos[recv] - pos[src]) + shift
    d = np.sqrt((vec * vec).sum(axis=1))
    units = vec / d[:, None] if src.size else np.zeros((0, 3))
    key = {(int(a), int(b), int(m)): e for e, (a, b, m) in enumerate(zip(src, recv, img))}
    rev = np.empty(src.size, dtype=np.int64)
    for e in range(src.size):
        pair = (int(recv[e]), int(src[e]), n_img - 1 - int(img[e]))
        if pair not in key:
            raise ValueError(f"edge {e} has no reverse edge {pair}")
        rev[e] = key[pair]
    ptr = np.searchsorted(src, np.arange(n + 1))
    ins, outs = [], []
    for j in range(n):
        row = np.arange(ptr[j], ptr[j + 1])
        for p in row:
            q = row[row != p]
            if q.size:
                ins.append(rev[q])
                outs.append(np.full(q.size, p, dtype=np.int64))
    trip_in = np.concatenate(ins) if ins else np.empty(0, dtype=np.int64)
    trip_out = np.concatenate(outs) if outs else np.empty(0, dtype=np.int64)
    angles = triplet_angles(pos, src, recv, trip_in, trip_out, vec, rev)
    return Graph(n, src, recv, trip_in, trip_out, d, units, angles, rev, vec, img)


def cap_graph(g: Graph, pos, max_nb: int) -> Graph:
    """Neighbour cap (no reference counterpart): an out-edge survives when it
    is among the max_nb nearest of its source (fp64 distance, ties by edge index) and so is its
    reverse at the other end; survivors keep their row order; triplets and angles follow from
    the capped graph as in build_graph_pbc."""
    n = g.n
    ptr = np.searchsorted(g.src, np.arange(n + 1))
    keep1 = np.zeros(g.src.size, dtype=bool)
    for v in range(n):
        row = np.arange(ptr[v], ptr[v + 1])
        order = row[np.argsort(g.dist[row], kind="stable")]
        keep1[order[:max_nb]] = True
    keep = keep1 & keep1[g.rev]
    new_id = np.full(g.src.size, -1, dtype=np.int64)
    new_id[keep] = np.arange(int(keep.sum()))
    src, recv = g.src[keep], g.recv[keep]
    rev = new_id[g.rev[keep]]
    vec = (g.vec[keep] if g.vec is not None else np.asarray(pos)[recv] - np.asarray(pos)[src])
    img = g.img[keep] if g.img is not None else None
    d = g.dist[keep]
    units = g.units[keep]
    nptr = np.searchsorted(src, np.arange(n + 1))
    ins, outs = [], []
    for j in range(n):
        row = np.arange(nptr[j], nptr[j + 1])
        for p in row:
            q = row[row != p]
            if q.size:
                ins.append(rev[q])
                outs.append(np.full(q.size, p, dtype=np.int64))
    trip_in = np.concatenate(ins) if ins else np.empty(0, dtype=np.int64)
    trip_out = np.concatenate(outs) if outs else np.empty(0, dtype=np.int64)
    angles = triplet_angles(pos, src, recv, trip_in, trip_out, vec, rev)
    return Graph(n, src, recv, trip_in, trip_out, d, units, angles, rev, vec, img)


# ---------------------------------------------------------------------------
# basis (basis.py:23-93)
# ---------------------------------------------------------------------------


def rbf_centers(k: int, cutoff: float) -> np.ndarray:
    if k < 1:
        raise ValueError("k_rbf must be >= 1")
    return np.zeros(1) if k == 1 else np.linspace(0.0, cutoff, k)


def rbf_gamma(k: int, cutoff: float) -> float:
    return (k / cutoff) ** 2


def rbf(d: np.ndarray, k: int, cutoff: float) -> np.ndarray:
    d = np.asarray(d, dtype=np.float64)
    if d.size and (np.any(d <= 0.0) or np.any(d > cutoff)):
        raise ValueError("distances must lie in (0, cutoff]")
    return np.exp(-rbf_gamma(k, cutoff) * (d[:, None] - rbf_centers(k, cutoff)[None, :]) ** 2)


def rbf_ddist(d: np.ndarray, k: int, cutoff: float) -> np.ndarray:
    g = rbf_gamma(k, cutoff)
    delta = np.asarray(d)[:, None] - rbf_centers(k, cutoff)[None, :]
    return -2.0 * g * delta * np.exp(-g * delta**2)


def sbf(d_in: np.ndarray, ang: np.ndarray, k: int, l: int, cutoff: float) -> np.ndarray:
    """(t, k*L + l) = rbf_k(d_kj) * cos(l * angle); basis.py:54-73."""
    radial = rbf(d_in, k, cutoff)
    orders = np.arange(l, dtype=np.float64)
    angular = np.cos(ang[:, None] * orders[None, :])
    return (radial[:, :, None] * angular[:, None, :]).reshape(ang.shape[0], k * l)


def sbf_partials(d_in, ang, k, l, cutoff):
    """basis.py:76-93."""
    n = ang.shape[0]
    radial = rbf(d_in, k, cutoff) if n else np.zeros((0, k))
    dradial = rbf_ddist(d_in, k, cutoff)
    orders = np.arange(l, dtype=np.float64)
    angular = np.cos(ang[:, None] * orders[None, :])
    dangular = -orders[None, :] * np.sin(ang[:, None] * orders[None, :])
    d_dist = (dradial[:, :, None] * angular[:, None, :]).reshape(n, k * l)
    d_ang = (radial[:, :, None] * dangular[:, None, :]).reshape(n, k * l)
    return d_dist, d_ang


# ---------------------------------------------------------------------------
# DimeNet++ / GemNet bases.  No reference counterpart: restated from the
# published definitions (DimeNet, Klicpera et al. 2020, eqs. 7-8 and the polynomial envelope;
# GemNet, Gasteiger et al. 2021, the radial Bessel basis and the circular basis Y_l0), with
# scipy.special for the spherical Bessel functions and Legendre polynomials.  Parity unpinned
# (no reference output exists); checked by finite differences (tests/test_oracle.py).
# ---------------------------------------------------------------------------
ENVELOPE_P = 6  # DimeNet's envelope exponent 5 -> p = exponent + 1


def envelope(x, p: int = ENVELOPE_P):
    """u(x) = 1/x + a x^(p-1) + b x^p + c x^(p+1) on (0, 1), 0 beyond (DimeNet Envelope)."""
    a, b, c = -(p + 1) * (p + 2) / 2.0, p * (p + 2.0), -p * (p + 1) / 2.0
    x = np.asarray(x, dtype=np.float64)
    u = 1.0 / x + a * x ** (p - 1) + b * x ** p + c * x ** (p + 1)
    return np.where(x < 1.0, u, 0.0)


def envelope_dx(x, p: int = ENVELOPE_P):
    a, b, c = -(p + 1) * (p + 2) / 2.0, p * (p + 2.0), -p * (p + 1) / 2.0
    x = np.asarray(x, dtype=np.float64)
    du = -1.0 / x ** 2 + a * (p - 1) * x ** (p - 2) + b * p * x ** (p - 1) + c * (p + 1) * x ** p
    return np.where(x < 1.0, du, 0.0)


def bessel_rbf(d, k: int, cutoff: float):
    """e_n(d) = sqrt(2/c) u(d/c) sin(n pi d/c), n = 1..k (GemNet / DimeNet radial basis)."""
    d = np.asarray(d, dtype=np.float64)
    if d.size and (np.any(d <= 0.0) or np.any(d > cutoff)):
        raise ValueError("distances must lie in (0, cutoff]")
    x = d[:, None] / cutoff
    n = np.arange(1, k + 1, dtype=np.float64)[None, :]
    return np.sqrt(2.0 / cutoff) * envelope(x) * np.sin(n * np.pi * x)


def bessel_rbf_ddist(d, k: int, cutoff: float):
    x = np.asarray(d, dtype=np.float64)[:, None] / cutoff
    n = np.arange(1, k + 1, dtype=np.float64)[None, :]
    return np.sqrt(2.0 / cutoff) * (envelope_dx(x) * np.sin(n * np.pi * x)
                                     + envelope(x) * n * np.pi * np.cos(n * np.pi * x)) / cutoff


def spherical_bessel_zeros(l_max: int, k: int) -> np.ndarray:
    """z[l, n]: the first k positive zeros of j_l, l < l_max (scipy, bracket + brentq)."""
    from scipy.optimize import brentq
    from scipy.special import spherical_jn

    z = np.zeros((l_max, k))
    xs = np.linspace(0.1, 20.0 + 4.0 * (k + l_max), 40000)
    for l in range(l_max):
        f = spherical_jn(l, xs)
        roots = []
        for i in range(xs.size - 1):
            if f[i] * f[i + 1] < 0:
                roots.append(brentq(lambda t: spherical_jn(l, t), xs[i], xs[i + 1], xtol=1e-15))
                if len(roots) == k:
                    break
        z[l] = roots
    return z


def _y_l0(ang, l_max):
    """Y_l0(angle) = sqrt((2l+1)/(4 pi)) P_l(cos angle) and its derivative w.r.t. the angle."""
    from scipy.special import eval_legendre

    x = np.cos(np.asarray(ang, dtype=np.float64))
    s = np.sin(np.asarray(ang, dtype=np.float64))
    out = np.zeros((x.size, l_max))
    dout = np.zeros((x.size, l_max))
    for l in range(l_max):
        nrm = np.sqrt((2 * l + 1) / (4 * np.pi))
        out[:, l] = nrm * eval_legendre(l, x)
        # P_l'(x) = l (x P_l - P_{l-1}) / (x^2 - 1);  d/dangle = -sin(angle) P_l'(cos angle)
        dp = np.polynomial.legendre.legval(x, np.polynomial.legendre.legder(np.eye(l_max)[l]))
        dout[:, l] = -nrm * s * dp
    return out, dout


def _sbf_bessel_parts(d_in, ang, k, l, cutoff, variant):
    """Radial [n, k, l] and its d-derivative, angular [n, l] and its angle derivative."""
    from scipy.special import spherical_jn

    d = np.asarray(d_in, dtype=np.float64)
    if d.size and (np.any(d <= 0.0) or np.any(d > cutoff)):
        raise ValueError("distances must lie in (0, cutoff]")
    ang_v, ang_d = _y_l0(ang, l)
    if variant == GEMNET:  # GemNet: radial Bessel basis of d_kj times the circular basis Y_l0
        rad = np.repeat(bessel_rbf(d, k, cutoff)[:, :, None], l, axis=2)
        drad = np.repeat(bessel_rbf_ddist(d, k, cutoff)[:, :, None], l, axis=2)
        return rad, drad, ang_v, ang_d
    # DimeNet: sqrt(2/c^3) / |j_{l+1}(z_ln)| u(d/c) j_l(z_ln d/c)
    z = spherical_bessel_zeros(l, k)  # [l, k]
    x = d[:, None, None] / cutoff
    zz = z.T[None, :, :]  # [1, k, l]
    orders = np.arange(l)[None, None, :]
    norm = np.sqrt(2.0 / cutoff ** 3) / np.abs(spherical_jn(orders + 1, zz))
    j = spherical_jn(orders, zz * x)
    dj = spherical_jn(orders, zz * x, derivative=True) * zz / cutoff
    u, du = envelope(x), envelope_dx(x) / cutoff
    return norm * u * j, norm * (du * j + u * dj), ang_v, ang_d


def sbf_bessel(d_in, ang, k, l, cutoff, variant):
    """(t, k*L + l) = radial_{k,l}(d_kj) * Y_l0(angle)."""
    rad, _, ang_v, _ = _sbf_bessel_parts(d_in, ang, k, l, cutoff, variant)
    return (rad * ang_v[:, None, :]).reshape(ang_v.shape[0], k * l)


def sbf_bessel_partials(d_in, ang, k, l, cutoff, variant):
    rad, drad, ang_v, ang_d = _sbf_bessel_parts(d_in, ang, k, l, cutoff, variant)
    n = ang_v.shape[0]
    return (drad * ang_v[:, None, :]).reshape(n, k * l), (rad * ang_d[:, None, :]).reshape(n, k * l)


def edge_basis(c, d):
    return bessel_rbf(d, c.k_rbf, c.cutoff) if c.basis == "bessel" else rbf(d, c.k_rbf, c.cutoff)


def edge_basis_ddist(c, d):
    return bessel_rbf_ddist(d, c.k_rbf, c.cutoff) if c.basis == "bessel" else rbf_ddist(d, c.k_rbf, c.cutoff)


def triplet_basis(c, d_in, ang):
    if c.basis == "bessel":
        return sbf_bessel(d_in, ang, c.k_rbf, c.l_sbf, c.cutoff, c.variant)
    return sbf(d_in, ang, c.k_rbf, c.l_sbf, c.cutoff)


def triplet_basis_partials(c, d_in, ang):
    if c.basis == "bessel":
        return sbf_bessel_partials(d_in, ang, c.k_rbf, c.l_sbf, c.cutoff, c.variant)
    return sbf_partials(d_in, ang, c.k_rbf, c.l_sbf, c.cutoff)


# ---------------------------------------------------------------------------
# primitives (tape.py:27-154)
# ---------------------------------------------------------------------------


def sigmoid(x):
    """Branch-stable sigmoid; tape.py:31-38."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def silu(x):
    return x * sigmoid(x)


def silu_grad(x):
    s = sigmoid(x)
    return s * (1.0 + x * (1.0 - s))


def segment_sum(x, seg, num):
    out = np.zeros((num,) + x.shape[1:], dtype=x.dtype)
    np.add.at(out, seg, x)
    return out


def scatter_rows(g, idx, num):
    """Adjoint of a row gather (tape.py:133-139)."""
    out = np.zeros((num,) + g.shape[1:], dtype=g.dtype)
    np.add.at(out, idx, g)
    return out


def receiver_plan(recv: np.ndarray, n: int):
    """Edges grouped by receiver (stable); engine.py:78-90."""
    order = np.argsort(recv, kind="stable").astype(np.int64)
    return order, recv[order]


# ---------------------------------------------------------------------------
# model forward (engine.py:99-261, 328-390)
# ---------------------------------------------------------------------------


def _mlp2_fwd(x, P, prefix):
    h = x @ P[prefix + ".w1"].T + P[prefix + ".b1"]
    a = silu(h)
    return a @ P[prefix + ".w2"].T + P[prefix + ".b2"], (x, h, a)


def _mlp2_bwd(g, cache, P, G, prefix):
    x, h, a = cache
    G[prefix + ".w2"] += g.T @ a
    G[prefix + ".b2"] += g.sum(axis=0)
    gh = (g @ P[prefix + ".w2"]) * silu_grad(h)
    G[prefix + ".w1"] += gh.T @ x
    G[prefix + ".b1"] += gh.sum(axis=0)
    return gh @ P[prefix + ".w1"]


@dataclass
class Forward:
    config: Config
    graph: Graph
    pos: np.ndarray
    energy: float
    forces: np.ndarray | None
    m: np.ndarray
    v: np.ndarray
    u: np.ndarray
    t_feat: np.ndarray
    rbf: np.ndarray
    sbf: np.ndarray
    cache: list


def forward(c: Config, P: dict, pos: np.ndarray, z: np.ndarray, graph: Graph | None = None) -> Forward:
    """Sequential forward of ModelTape (engine.py:328-390)."""
    z = np.asarray(z, dtype=np.int64)
    if np.any(z > MAX_Z):  # engine.py:71-75
        raise ValueError("atomic number exceeds the embedding table")
    g = graph if graph is not None else build_graph(pos, c.cutoff)
    n_e, n_v = g.src.size, g.n
    gem = c.variant == GEMNET
    R = edge_basis(c, g.dist) if n_e else np.zeros((0, c.k_rbf))
    S = triplet_basis(c, g.dist[g.trip_in], g.angles) if g.trip_in.size else np.zeros((0, c.k_rbf * c.l_sbf))
    sel, seg = receiver_plan(g.recv, n_v)

    m = R @ P["edge_init.w"].T + P["edge_init.b"]
    u = np.zeros((1, c.d_u))
    v = P["atom_embedding"][z - 1]
    t_feat = np.zeros((g.trip_in.size, c.d_t))
    cache = []
    for b in range(c.blocks):
        p = f"block{b}."
        blk = {"m": m, "u": u}
        # TU (engine.py:118-149)
        m_in = m[g.trip_in]
        down = m_in @ P[p + "tu.down"].T
        rb = R[g.trip_out]
        grbf = rb @ P[p + "tu.rbf_gate"].T
        gsbf = S @ P[p + "tu.sbf_gate"].T
        blk.update(m_in=m_in, down=down, rb=rb, grbf=grbf, gsbf=gsbf)
        if gem:
            a = down @ P[p + "tu.bilinear_a"].T
            bb = gsbf @ P[p + "tu.bilinear_b"].T
            ab = a * bb
            mixed = ab @ P[p + "tu.bilinear_proj"].T
            t_feat = mixed * grbf
            blk.update(a=a, bb=bb, ab=ab, mixed=mixed)
        else:
            dg = down * gsbf
            t_feat = dg * grbf
            blk.update(dg=dg)
        up = t_feat @ P[p + "tu.up"].T
        ta = segment_sum(up, g.trip_out, n_e)
        blk["t"] = t_feat
        # EU (engine.py:152-158)
        mlp, blk["eu"] = _mlp2_fwd(np.concatenate([m, ta], axis=1), P, p + "eu")
        m_new = m + mlp
        # EA + NU (engine.py:166-177)
        agg = segment_sum(m_new[sel], seg, n_v)
        v, blk["nu"] = _mlp2_fwd(agg, P, p + "nu")
        if gem:
            # EU2 + sym (engine.py:180-200)
            mlp2, blk["eu2"] = _mlp2_fwd(np.concatenate([m_new, v[g.recv]], axis=1), P, p + "eu2")
            m2 = m_new + mlp2
            m = m2 + m2[g.rev] @ P[p + "sym.w"].T
            blk["m2"] = m2
        else:
            m = m_new
        # GU (engine.py:207-217)
        s = v.sum(axis=0, keepdims=True)
        zz = s @ P[p + "gu.w1"].T
        pre = zz + P[p + "gu.b1"][None, :]
        act = silu(pre)
        u = u + (act @ P[p + "gu.w2"].T + P[p + "gu.b2"])
        blk.update(v=v, s=s, pre=pre, act=act)
        cache.append(blk)
    energy = float((u @ P["energy_head.w"].T + P["energy_head.b"])[0, 0])
    forces = None
    if gem:  # engine.py:234-246
        scale = m[sel] @ P["force_head.w"].T
        forces = segment_sum(scale * g.units[sel], seg, n_v)
    return Forward(c, g, np.asarray(pos, np.float64), energy, forces, m, v, u, t_feat, R, S, cache)


# ---------------------------------------------------------------------------
# model backward (tape.py:348-383 walking the recorded sequence in reverse;
# geometry adjoints tape.py:164-242, runtime.py:626-671)
# ---------------------------------------------------------------------------


def backward(fw: Forward, P: dict, d_energy: float = 1.0, d_forces: np.ndarray | None = None):
    """Returns (d_params dict in declaration order, d_positions)."""
    c, g = fw.config, fw.graph
    gem = c.variant == GEMNET
    n_e, n_v, n_t = g.src.size, g.n, g.trip_in.size
    G = {name: np.zeros(shape) for name, shape, _ in param_specs(c)}
    if d_forces is not None and not gem:
        raise ValueError("force seed given but this variant has no force head")
    sel, seg = receiver_plan(g.recv, n_v)

    # readout
    u_bar = np.array([[d_energy]]) @ P["energy_head.w"]
    G["energy_head.w"] += d_energy * fw.u
    G["energy_head.b"] += d_energy
    m_bar = np.zeros((n_e, c.d_e))
    units_bar = np.zeros((n_e, 3))
    if gem and d_forces is not None:
        fb = np.asarray(d_forces, dtype=np.float64)
        f_rows = fb[seg]  # segment_sum adjoint = gather
        m_rows = fw.m[sel]
        scale = m_rows @ P["force_head.w"].T
        scale_bar = (f_rows * g.units[sel]).sum(axis=1, keepdims=True)
        units_bar += scatter_rows(scale * f_rows, sel, n_e)
        G["force_head.w"] += scale_bar.T @ m_rows
        m_bar += scatter_rows(scale_bar @ P["force_head.w"], sel, n_e)

    R_bar = np.zeros_like(fw.rbf)
    S_bar = np.zeros_like(fw.sbf)
    for b in range(c.blocks - 1, -1, -1):
        p = f"block{b}."
        blk = fw.cache[b]
        # GU
        G[p + "gu.w2"] += u_bar.T @ blk["act"]
        G[p + "gu.b2"] += u_bar.sum(axis=0)
        pre_bar = (u_bar @ P[p + "gu.w2"]) * silu_grad(blk["pre"])
        G[p + "gu.b1"] += pre_bar.sum(axis=0)
        G[p + "gu.w1"] += pre_bar.T @ blk["s"]
        s_bar = pre_bar @ P[p + "gu.w1"]
        v_bar = np.broadcast_to(s_bar, (n_v, c.d_v)).copy()
        # u_bar flows unchanged through the residual
        if gem:
            m2 = blk["m2"]
            m2_bar = m_bar.copy()
            G[p + "sym.w"] += m_bar.T @ m2[g.rev]
            m2_bar += scatter_rows(m_bar @ P[p + "sym.w"], g.rev, n_e)
            x_bar = _mlp2_bwd(m2_bar, blk["eu2"], P, G, p + "eu2")
            m_new_bar = m2_bar + x_bar[:, : c.d_e]
            v_bar += scatter_rows(x_bar[:, c.d_e :], g.recv, n_v)
        else:
            m_new_bar = m_bar
        agg_bar = _mlp2_bwd(v_bar, blk["nu"], P, G, p + "nu")
        m_new_bar = m_new_bar + scatter_rows(agg_bar[seg], sel, n_e)
        x_bar = _mlp2_bwd(m_new_bar, blk["eu"], P, G, p + "eu")
        m_bar = m_new_bar + x_bar[:, : c.d_e]
        ta_bar = x_bar[:, c.d_e :]
        # TU backward
        up_bar = ta_bar[g.trip_out]
        G[p + "tu.up"] += up_bar.T @ blk["t"]
        t_bar = up_bar @ P[p + "tu.up"]
        if gem:
            mixed_bar = t_bar * blk["grbf"]
            grbf_bar = t_bar * blk["mixed"]
            G[p + "tu.bilinear_proj"] += mixed_bar.T @ blk["ab"]
            ab_bar = mixed_bar @ P[p + "tu.bilinear_proj"]
            a_bar = ab_bar * blk["bb"]
            bb_bar = ab_bar * blk["a"]
            G[p + "tu.bilinear_b"] += bb_bar.T @ blk["gsbf"]
            gsbf_bar = bb_bar @ P[p + "tu.bilinear_b"]
            G[p + "tu.bilinear_a"] += a_bar.T @ blk["down"]
            down_bar = a_bar @ P[p + "tu.bilinear_a"]
        else:
            dg_bar = t_bar * blk["grbf"]
            grbf_bar = t_bar * blk["dg"]
            down_bar = dg_bar * blk["gsbf"]
            gsbf_bar = dg_bar * blk["down"]
        G[p + "tu.sbf_gate"] += gsbf_bar.T @ fw.sbf
        S_bar += gsbf_bar @ P[p + "tu.sbf_gate"]
        G[p + "tu.rbf_gate"] += grbf_bar.T @ blk["rb"]
        R_bar += scatter_rows(grbf_bar @ P[p + "tu.rbf_gate"], g.trip_out, n_e)
        G[p + "tu.down"] += down_bar.T @ blk["m_in"]
        m_bar = m_bar + scatter_rows(down_bar @ P[p + "tu.down"], g.trip_in, n_e)

    # edge init
    G["edge_init.w"] += m_bar.T @ fw.rbf
    G["edge_init.b"] += m_bar.sum(axis=0)
    R_bar += m_bar @ P["edge_init.w"]

    # geometry (runtime.py:626-671 ordering: angles, units, distances)
    pos = fw.pos
    dist_bar = np.zeros(n_e)
    pos_bar = np.zeros_like(pos)
    if n_t:
        d_in = g.dist[g.trip_in]
        dd, da = triplet_basis_partials(c, d_in, g.angles)
        np.add.at(dist_bar, g.trip_in, (S_bar * dd).sum(axis=1))
        ang_bar = (S_bar * da).sum(axis=1)
        g_k, g_j, g_i = angle_gradients(pos, g.src, g.recv, g.trip_in, g.trip_out, g.vec, g.rev)
        k = g.src[g.trip_in]
        j = g.recv[g.trip_in]
        i = g.recv[g.trip_out]
        buf = np.zeros_like(pos)
        np.add.at(buf, k, ang_bar[:, None] * g_k)
        np.add.at(buf, i, ang_bar[:, None] * g_i)
        np.add.at(buf, j, ang_bar[:, None] * g_j)
        pos_bar = pos_bar + buf
    if n_e:
        dist_bar += (R_bar * edge_basis_ddist(c, g.dist)).sum(axis=1)
        if gem:
            diff = g.vec if g.vec is not None else pos[g.recv] - pos[g.src]
            unit = diff / g.dist[:, None]
            proj = (units_bar * unit).sum(axis=1, keepdims=True)
            contrib = (units_bar - proj * unit) / g.dist[:, None]
            buf = np.zeros_like(pos)
            np.add.at(buf, g.recv, contrib)
            np.add.at(buf, g.src, -contrib)
            pos_bar = pos_bar + buf
        contrib = dist_bar[:, None] * g.units
        buf = np.zeros_like(pos)
        np.add.at(buf, g.recv, contrib)
        np.add.at(buf, g.src, -contrib)
        pos_bar = pos_bar + buf
    return G, pos_bar


# ---------------------------------------------------------------------------
# drivers (tasks.py:37-67, 79-128, 131-209)
# ---------------------------------------------------------------------------


def predict(c: Config, P: dict, pos, z):
    """Energy and forces; tasks.py:37-67 (P == 1 path)."""
    fw = forward(c, P, pos, z)
    if c.variant == GEMNET:
        return fw.energy, fw.forces
    _, d_pos = backward(fw, P, d_energy=1.0)
    return fw.energy, -d_pos


def relax(c: Config, P: dict, pos, z, fmax_threshold: float, max_steps: int = 200, step_size: float = 0.05):
    """Steepest-descent relaxation x <- x + eta F with the energy guard of energy-centric
    models (reject and halve eta when the energy rises); tasks.py:79-128.  Returns
    (trajectory, max_forces, energies, converged, steps)."""
    if fmax_threshold <= 0:
        raise ValueError("fmax_threshold must be positive")
    if max_steps < 0:
        raise ValueError("max_steps must be >= 0")
    guard = c.variant == DIMENET  # energy_centric (config.py:46-47); the diagnostic model is not restated
    eta = step_size
    x = np.array(pos, dtype=np.float64)
    trajectory = [x.copy()]
    energies, max_forces = [], []
    steps, converged = 0, False
    energy, forces = predict(c, P, x, z)
    while True:
        if not (np.isfinite(energy) and np.all(np.isfinite(forces))):
            raise RuntimeError(f"non-finite prediction at step {steps}")
        fmax = float(np.sqrt((forces * forces).sum(axis=1)).max())
        energies.append(energy)
        max_forces.append(fmax)
        if fmax < fmax_threshold:
            converged = True
            break
        if steps >= max_steps:
            break
        proposal = x + eta * forces
        steps += 1
        new_energy, new_forces = predict(c, P, proposal, z)
        if guard and new_energy > energy:
            eta *= 0.5
        else:
            x = proposal
            energy, forces = new_energy, new_forces
        trajectory.append(x.copy())
    return trajectory, max_forces, energies, converged, steps


def loss_and_grads(c: Config, P: dict, dataset, w_energy=1.0, w_forces=0.0):
    """Mean squared loss and exact gradient over a list of (pos, z, E*, F*); tasks.py:131-185."""
    if w_forces != 0.0 and c.variant != GEMNET:
        raise ValueError("force-loss gradients require the force-centric variant")
    n = len(dataset)
    if n == 0:
        raise ValueError("dataset is empty")
    total = 0.0
    grad_sum = {name: np.zeros(shape) for name, shape, _ in param_specs(c)}
    for pos, z, e_t, f_t in dataset:
        fw = forward(c, P, pos, z)
        res = np.float64(fw.energy - e_t)
        d_energy = float(2.0 * w_energy * res / n)
        loss = float(w_energy * res * res)
        d_forces = None
        if w_forces != 0.0:
            delta = fw.forces - np.asarray(f_t, dtype=np.float64)
            n_at = pos.shape[0]
            loss += w_forces * float((delta * delta).sum()) / n_at
            d_forces = 2.0 * w_forces * delta / (n * n_at)
        G, _ = backward(fw, P, d_energy, d_forces)
        for k in grad_sum:
            grad_sum[k] += G[k]
        total += loss / n
    return total, grad_sum


def sgd_step(P: dict, grads: dict, lr: float) -> dict:
    """tasks.py:207-208."""
    return {k: P[k] - lr * grads[k] for k in P}
