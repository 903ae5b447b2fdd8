"""Torch-tensor wrappers over the C ABI (include/egn_b200.h).

Each function allocates its outputs with torch (device memory + the
caching allocator are the only things torch provides here), launches the
native kernels on the current stream and returns.  Inputs must be CUDA
tensors of the documented dtype; there is no CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import torch

from ._lib import call, ptr, stream


def _c(t: torch.Tensor, dtype) -> torch.Tensor:
    if t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    return t.contiguous()


def neighbors_count(pos, graph_ptr, node_graph, cutoff):
    n = pos.shape[0]
    deg = torch.empty(n, dtype=torch.int32, device=pos.device)
    call("egn_neighbors_count", ptr(pos), ptr(graph_ptr), ptr(node_graph), n, float(cutoff), ptr(deg), stream())
    return deg


def scan_counts(counts, square_minus_one=False):
    out = torch.empty(counts.shape[0] + 1, dtype=torch.int64, device=counts.device)
    call("egn_scan_counts", ptr(counts), counts.shape[0], int(square_minus_one), ptr(out), stream())
    return out


def neighbors_fill(pos, graph_ptr, node_graph, cutoff, edge_ptr, num_edges):
    src = torch.empty(num_edges, dtype=torch.int32, device=pos.device)
    recv = torch.empty(num_edges, dtype=torch.int32, device=pos.device)
    call("egn_neighbors_fill", ptr(pos), ptr(graph_ptr), ptr(node_graph), pos.shape[0], float(cutoff),
         ptr(edge_ptr), ptr(src), ptr(recv), stream())
    return src, recv


def reverse_edges(edge_ptr, src, recv, missing=None):
    rev = torch.empty_like(src)
    if missing is None:
        missing = zeros((1,), src.device, torch.int32)
    call("egn_reverse_edges", ptr(edge_ptr), ptr(src), ptr(recv), src.shape[0], ptr(rev), ptr(missing), stream())
    return rev, missing


def triplets_fill(edge_ptr, rev, tri_ptr, num_triplets):
    n = edge_ptr.shape[0] - 1
    kj = torch.empty(num_triplets, dtype=torch.int64, device=rev.device)
    ji = torch.empty(num_triplets, dtype=torch.int64, device=rev.device)
    call("egn_triplets_fill", ptr(edge_ptr), ptr(rev), ptr(tri_ptr), n, ptr(kj), ptr(ji), stream())
    return kj, ji


def neighbors_count_pbc(pos, graph_ptr, node_graph, cell, nimg, cutoff):
    n = pos.shape[0]
    deg = torch.empty(n, dtype=torch.int32, device=pos.device)
    call("egn_neighbors_count_pbc", ptr(pos), ptr(graph_ptr), ptr(node_graph), n, ptr(cell), ptr(nimg),
         float(cutoff), ptr(deg), stream())
    return deg


def neighbors_fill_pbc(pos, graph_ptr, node_graph, cell, nimg, cutoff, edge_ptr, num_edges):
    dev = pos.device
    src = torch.empty(num_edges, dtype=torch.int32, device=dev)
    recv = torch.empty(num_edges, dtype=torch.int32, device=dev)
    img = torch.empty(num_edges, dtype=torch.int32, device=dev)
    shift = torch.empty((num_edges, 3), dtype=torch.float64, device=dev)
    call("egn_neighbors_fill_pbc", ptr(pos), ptr(graph_ptr), ptr(node_graph), pos.shape[0], ptr(cell), ptr(nimg),
         float(cutoff), ptr(edge_ptr), ptr(src), ptr(recv), ptr(img), ptr(shift), stream())
    return src, recv, img, shift


def reverse_edges_pbc(edge_ptr, src, recv, img, node_graph, nimg):
    rev = torch.empty_like(src)
    missing = torch.zeros(1, dtype=torch.int32, device=src.device)
    call("egn_reverse_edges_pbc", ptr(edge_ptr), ptr(src), ptr(recv), ptr(img), ptr(node_graph), ptr(nimg),
         src.shape[0], ptr(rev), ptr(missing), stream())
    return rev, missing


def geometry(pos, src, recv, want_fp64=False, shift=None):
    """Packed fp32 (u, d) per edge (+ fp64 d and u); edge vector (x_recv - x_src) + shift."""
    e = src.shape[0]
    geo = torch.empty((e, 4), dtype=torch.float32, device=pos.device)
    d64 = u64 = None
    if want_fp64:
        d64 = torch.empty(e, dtype=torch.float64, device=pos.device)
        u64 = torch.empty((e, 3), dtype=torch.float64, device=pos.device)
    if shift is None:
        call("egn_geometry", ptr(pos), ptr(src), ptr(recv), e, ptr(geo), ptr(d64), ptr(u64), stream())
    else:
        call("egn_geometry_shift", ptr(pos), ptr(src), ptr(recv), ptr(shift), e, ptr(geo), ptr(d64), ptr(u64),
             stream())
    return geo, d64, u64


def triplet_angles(pos, edge_ptr, recv, tri_ptr, num_triplets, shift=None):
    out = torch.empty(num_triplets, dtype=torch.float64, device=pos.device)
    if shift is None:
        call("egn_triplet_angles", ptr(pos), ptr(edge_ptr), ptr(recv), ptr(tri_ptr), pos.shape[0], ptr(out),
             stream())
    else:
        call("egn_triplet_angles_shift", ptr(pos), ptr(edge_ptr), ptr(recv), ptr(shift), ptr(tri_ptr),
             pos.shape[0], ptr(out), stream())
    return out


def rbf(geo, k_rbf, cutoff, basis=0):
    """Edge radial basis [E, K]: Gaussian (basis 0, the reference) or the radial Bessel basis
    with the polynomial envelope (basis 1 / 2, DimeNet++ / GemNet)."""
    out = torch.empty((geo.shape[0], k_rbf), dtype=torch.float32, device=geo.device)
    if basis:
        call("egn_rbf_bessel", ptr(geo), geo.shape[0], int(k_rbf), float(cutoff), ptr(out), stream())
    else:
        call("egn_rbf", ptr(geo), geo.shape[0], int(k_rbf), float(cutoff), ptr(out), stream())
    return out


def rbf_linear(rbf_t, w, b=None, out=None):
    """out = rbf w^T (+ b) for a K <= 8 basis (egn_rbf_linear)."""
    e, k = rbf_t.shape
    n = w.shape[0]
    if out is None:
        out = torch.empty((e, n), dtype=torch.float32, device=rbf_t.device)
    if k > 8 or n % 4 or out.stride(0) % 4 or out.stride(1) != 1 or out.data_ptr() % 16:
        raise ValueError(f"rbf_linear: K = {k} <= 8, N = {n} % 4 == 0 and 16-byte aligned rows required "
                         "(the engine pads feature widths to multiples of 16)")
    call("egn_rbf_linear", ptr(_c(rbf_t, torch.float32)), e, k, ptr(_c(w, torch.float32)),
         ptr(_c(b, torch.float32)) if b is not None else None, n, ptr(out), out.stride(0), stream())
    return out


def graph_mlp_fwd(s, w1, b1, w2, b2, u):
    """GU block over G graphs (egn_graph_mlp_fwd): returns (pre, act); u updated in place.
    w1 None: identity first layer (s is the already projected z = s W1^T)."""
    g, dv = s.shape
    du = w1.shape[0] if w1 is not None else dv
    pre = torch.empty((g, du), dtype=torch.float32, device=s.device)
    act = torch.empty_like(pre)
    call("egn_graph_mlp_fwd", g, dv, du, ptr(_c(s, torch.float32)),
         ptr(_c(w1, torch.float32)) if w1 is not None else None,
         ptr(_c(b1, torch.float32)), ptr(_c(w2, torch.float32)), ptr(_c(b2, torch.float32)), ptr(pre), ptr(act),
         ptr(u), stream())
    return pre, act


def graph_mlp_bwd(u_bar, s, pre, act, w1, w2, w1_bar, b1_bar, w2_bar, b2_bar):
    """Adjoint of graph_mlp_fwd (egn_graph_mlp_bwd): returns s_bar [G, dv]; weight / bias
    adjoints written into the given (contiguous) views.  w1 None: identity first layer
    (s is the projected z; s_bar = pre_bar, w1_bar unused)."""
    g, dv = s.shape
    du = w1.shape[0] if w1 is not None else dv
    pre_bar = torch.empty((g, du), dtype=torch.float32, device=s.device)
    s_bar = torch.empty((g, dv), dtype=torch.float32, device=s.device)
    for t in (w1_bar, b1_bar, w2_bar, b2_bar):
        if t is not None and not t.is_contiguous():
            raise ValueError("graph_mlp_bwd outputs must be contiguous")
    call("egn_graph_mlp_bwd", g, dv, du, ptr(_c(u_bar, torch.float32)), ptr(_c(s, torch.float32)),
         ptr(_c(pre, torch.float32)), ptr(_c(act, torch.float32)),
         ptr(_c(w1, torch.float32)) if w1 is not None else None,
         ptr(_c(w2, torch.float32)), ptr(pre_bar), ptr(s_bar), ptr(w1_bar) if w1 is not None else None, ptr(b1_bar),
         ptr(w2_bar), ptr(b2_bar), stream())
    return s_bar


def graph_linear(x, w, b=None):
    """z = x w^T (+ b) over G rows (egn_graph_linear)."""
    g, din = x.shape
    dout = w.shape[0]
    y = torch.empty((g, dout), dtype=torch.float32, device=x.device)
    call("egn_graph_linear", g, din, dout, ptr(_c(x, torch.float32)), ptr(_c(w, torch.float32)),
         ptr(_c(b, torch.float32)) if b is not None else None, ptr(y), stream())
    return y


def graph_linear_bwd(y_bar, x, w, x_bar=True, w_bar=None, b_bar=None):
    """Adjoint of graph_linear: returns x_bar = y_bar w (or None); w_bar = y_bar^T x and
    b_bar = column sums of y_bar written into the given contiguous views."""
    g, din = x.shape
    dout = w.shape[0]
    xb = torch.empty((g, din), dtype=torch.float32, device=x.device) if x_bar else None
    call("egn_graph_linear_bwd", g, din, dout, ptr(_c(y_bar, torch.float32)), ptr(_c(x, torch.float32)),
         ptr(_c(w, torch.float32)), ptr(xb), ptr(w_bar), ptr(b_bar), stream())
    return xb


def rbf_linear_bwd(rbf_t, w, g, rbf_bar, w_bar, b_bar=None, g2=None):
    """Adjoint of rbf_linear: rbf_bar += g w; w_bar = g^T rbf; b_bar = column sums of g.
    g2 (same shape): the adjoint arrives as a product g * g2 (a gate's VJP), fused."""
    e, k = rbf_t.shape
    n = w.shape[0]
    if g.stride(1) != 1:
        g = g.contiguous()
    if g2 is not None and (g2.stride(1) != 1 or g2.stride(0) != g.stride(0)):
        g, g2 = (g * g2).contiguous(), None
    if k > 8:
        raise ValueError(f"rbf_linear_bwd: k_rbf = {k} > 8 is outside the native kernel")
    if n > 128:
        # wide outputs (XL edge_init d_e = 2048, C3 rbf gate d_t = 256): 128-column chunks of the
        # same kernel; rbf_bar accumulates over chunks, W_bar / b_bar rows per chunk
        for c0 in range(0, n, 128):
            c1 = min(n, c0 + 128)
            rbf_linear_bwd(rbf_t, w[c0:c1], g[:, c0:c1], rbf_bar, w_bar[c0:c1],
                           b_bar[c0:c1] if b_bar is not None else None,
                           g2[:, c0:c1] if g2 is not None else None)
        return
    nbytes = call("egn_rbf_linear_bwd_workspace_bytes", e, k, n)
    ws = _workspace_named("rbflin", nbytes, g.device)
    call("egn_rbf_linear_bwd", ptr(_c(rbf_t, torch.float32)), e, k, ptr(_c(w, torch.float32)), n, ptr(g),
         ptr(g2) if g2 is not None else None, g.stride(0), ptr(rbf_bar), ptr(w_bar),
         ptr(b_bar) if b_bar is not None else None, ptr(ws), stream())


def sbf(geo, edge_ptr, tri_ptr, num_triplets, k_rbf, l_sbf, cutoff):
    out = torch.empty((num_triplets, k_rbf * l_sbf), dtype=torch.float32, device=geo.device)
    call("egn_sbf", ptr(geo), ptr(edge_ptr), ptr(tri_ptr), edge_ptr.shape[0] - 1, int(k_rbf), int(l_sbf),
         float(cutoff), ptr(out), stream())
    return out


# the native triplet kernels take up to 256 channels per call; wider triplet
# embeddings (GemNet-XL d_bil = 288) are processed in channel chunks, which is
# exact because the contraction is independent per channel (the geometry
# adjoint edge_grad accumulates over chunks).
MAX_TRIPLET_WIDTH = 256


def _channel_chunks(dg):
    return [(c0, min(dg, c0 + MAX_TRIPLET_WIDTH)) for c0 in range(0, dg, MAX_TRIPLET_WIDTH)]


def triplet_fwd(edge_ptr, rev, geo, X, Wk, cutoff, max_degree=-1, basis=0):
    """S = sum over the centre tile (see include/egn_b200.h egn_triplet_fwd; basis 1 / 2:
    egn_triplet_fwd_basis, the DimeNet++ / GemNet triplet bases)."""
    X = _c(X, torch.float32)
    Wk = _c(Wk, torch.float32)
    k, l, dg = Wk.shape
    if dg > MAX_TRIPLET_WIDTH:
        S = torch.empty_like(X)
        for c0, c1 in _channel_chunks(dg):
            S[:, c0:c1] = triplet_fwd(edge_ptr, rev, geo, X[:, c0:c1].contiguous(), Wk[:, :, c0:c1].contiguous(),
                                      cutoff, max_degree, basis)
        return S
    S = torch.empty_like(X)
    nv = edge_ptr.shape[0] - 1
    if basis:
        ne = X.shape[0]
        nbytes = call("egn_triplet_fwd_basis_workspace_bytes", nv, ne, int(max_degree), k, l, dg, int(basis))
        ws = _workspace_named("tfwd", nbytes, X.device)
        call("egn_triplet_fwd_basis", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ne, int(max_degree), ptr(X), ptr(Wk), k,
             l, dg, float(cutoff), int(basis), ptr(S), ptr(ws), stream())
        return S
    nbytes = call("egn_triplet_fwd_workspace_bytes", nv, int(max_degree), k, l, dg)
    ws = _workspace_named("tfwd", nbytes, X.device) if nbytes > 0 else None
    call("egn_triplet_fwd", ptr(edge_ptr), ptr(rev), ptr(geo), nv, int(max_degree), ptr(X),
         ptr(Wk), k, l, dg, float(cutoff), ptr(S), ptr(ws), stream())
    return S


_WS: dict = {}
# Workspaces that were outgrown are retired, never freed: a captured CUDA graph (Trainer.step)
# holds raw pointers into the buffer that was current at capture time, and its replays must
# keep writing valid memory even after a later, larger call replaced that buffer.
_WS_RETIRED: list = []


def _workspace_named(name: str, nbytes: int, device, minimum: int = 1 << 16) -> torch.Tensor:
    # per thread: in-process graph-parallel ranks (runtime.ThreadComm) share a stream
    key = (str(device), name, threading.get_ident())
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            _WS_RETIRED.append(buf)
        buf = torch.empty(max(nbytes, minimum), dtype=torch.uint8, device=device)
        _WS[key] = buf
    return buf


def _workspace(nbytes: int, device) -> torch.Tensor:
    return _workspace_named("ws", nbytes, device, 1 << 20)


def triplet_bwd(edge_ptr, rev, geo, X, Wk, cutoff, S_bar, edge_grad, X_bar=None, W_bar=None, max_degree=None,
                basis=0, phases=3):
    """Adjoint of triplet_fwd (egn_triplet_bwd).  phases (egn_triplet_bwd_ex): 1 = the angle
    adjoint only (edge_grad x, y, z of the small-degree centres; returns (None, None)), 2 = the
    rest, 3 = all.  Phases 1 and 2 write disjoint outputs and may run on two streams."""
    X = _c(X, torch.float32)
    Wk = _c(Wk, torch.float32)
    S_bar = _c(S_bar, torch.float32)
    k, l, dg = Wk.shape
    nv = edge_ptr.shape[0] - 1
    if X_bar is None:
        X_bar = torch.empty_like(X)
    if W_bar is None:
        W_bar = torch.empty_like(Wk)
    if max_degree is None:
        max_degree = int((edge_ptr[1:] - edge_ptr[:-1]).max().item()) if nv else 0
    if dg > MAX_TRIPLET_WIDTH:
        for c0, c1 in _channel_chunks(dg):
            xb, wb = triplet_bwd(edge_ptr, rev, geo, X[:, c0:c1].contiguous(), Wk[:, :, c0:c1].contiguous(), cutoff,
                                 S_bar[:, c0:c1].contiguous(), edge_grad, max_degree=max_degree, basis=basis,
                                 phases=phases)
            if phases != 1:
                X_bar[:, c0:c1] = xb
                W_bar[:, :, c0:c1] = wb
        return (None, None) if phases == 1 else (X_bar, W_bar)
    ne = X.shape[0]
    if phases == 1 and basis:  # its own radial table, no X_bar / W_bar writes
        ws = _workspace_named("tbw_angle", call("egn_triplet_bwd_angle_workspace_bytes", ne, int(basis)), X.device)
        call("egn_triplet_bwd_basis_ex", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ne, int(max_degree), ptr(X), ptr(Wk),
             k, l, dg, float(cutoff), int(basis), 1, ptr(S_bar), None, None, ptr(edge_grad), ptr(ws), stream())
        return None, None
    if phases == 1:  # no workspace, no X_bar / W_bar writes
        call("egn_triplet_bwd_ex", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ne, int(max_degree), ptr(X), ptr(Wk), k, l,
             dg, float(cutoff), ptr(S_bar), None, None, ptr(edge_grad), 1, None, stream())
        return None, None
    if basis:
        nbytes = call("egn_triplet_bwd_basis_workspace_bytes", nv, ne, int(max_degree), k, l, dg, int(basis))
    else:
        nbytes = call("egn_triplet_bwd_workspace_bytes", nv, ne, int(max_degree), k, l, dg)
    ws = _workspace(nbytes, X.device)
    if basis:
        call("egn_triplet_bwd_basis_ex", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ne, int(max_degree), ptr(X), ptr(Wk),
             k, l, dg, float(cutoff), int(basis), int(phases), ptr(S_bar), ptr(X_bar), ptr(W_bar), ptr(edge_grad),
             ptr(ws), stream())
        return X_bar, W_bar
    if phases == 2:
        call("egn_triplet_bwd_ex", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ne, int(max_degree), ptr(X), ptr(Wk), k, l,
             dg, float(cutoff), ptr(S_bar), ptr(X_bar), ptr(W_bar), ptr(edge_grad), 2, ptr(ws), stream())
        return X_bar, W_bar
    call("egn_triplet_bwd", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ne, int(max_degree), ptr(X), ptr(Wk), k, l, dg,
         float(cutoff), ptr(S_bar), ptr(X_bar), ptr(W_bar), ptr(edge_grad), ptr(ws), stream())
    return X_bar, W_bar


def triplet_fwd_window(edge_ptr, rev, geo, X, Wk, cutoff, first_lo, last_hi, S):
    """Triplet forward over the centres of edge_ptr restricted to a contiguous triplet window
    (egn_triplet_fwd_window); writes the covered centres' rows of the full-size S."""
    k, l, dg = Wk.shape
    if dg > MAX_TRIPLET_WIDTH:
        for c0, c1 in _channel_chunks(dg):
            part = torch.zeros((S.shape[0], c1 - c0), dtype=torch.float32, device=S.device)
            triplet_fwd_window(edge_ptr, rev, geo, X[:, c0:c1].contiguous(), Wk[:, :, c0:c1].contiguous(), cutoff,
                               first_lo, last_hi, part)
            S[:, c0:c1] += part
        return S
    call("egn_triplet_fwd_window", ptr(edge_ptr), ptr(rev), ptr(geo), edge_ptr.shape[0] - 1, int(first_lo),
         int(last_hi), ptr(_c(X, torch.float32)), ptr(_c(Wk, torch.float32)), k, l, dg, float(cutoff), ptr(S),
         stream())
    return S


def triplet_bwd_window(edge_ptr, rev, geo, X, Wk, cutoff, first_lo, last_hi, S_bar, edge_grad, X_bar, max_degree):
    """Adjoint of triplet_fwd_window: X_bar rows rev(q) of the covered centres overwritten (the
    caller zeroes the rest), returns W_bar; edge_grad accumulated."""
    k, l, dg = Wk.shape
    W_bar = torch.empty_like(Wk)
    if dg > MAX_TRIPLET_WIDTH:
        for c0, c1 in _channel_chunks(dg):
            xb = torch.zeros((X.shape[0], c1 - c0), dtype=torch.float32, device=X.device)
            W_bar[:, :, c0:c1] = triplet_bwd_window(edge_ptr, rev, geo, X[:, c0:c1].contiguous(),
                                                    Wk[:, :, c0:c1].contiguous(), cutoff, first_lo, last_hi,
                                                    S_bar[:, c0:c1].contiguous(), edge_grad, xb, max_degree)
            X_bar[:, c0:c1] += xb
        return W_bar
    nv, ne = edge_ptr.shape[0] - 1, X.shape[0]
    nbytes = call("egn_triplet_bwd_workspace_bytes", nv, ne, int(max_degree), k, l, dg)
    ws = _workspace(nbytes, X.device)
    call("egn_triplet_bwd_window", ptr(edge_ptr), ptr(rev), ptr(geo), nv, int(first_lo), int(last_hi),
         int(max_degree), ptr(_c(X, torch.float32)), ptr(_c(Wk, torch.float32)), k, l, dg, float(cutoff),
         ptr(_c(S_bar, torch.float32)), ptr(X_bar), ptr(W_bar), ptr(edge_grad), ptr(ws), stream())
    return W_bar


def triplet_terms(edge_ptr, rev, geo, tri_ptr, num_triplets, X, Wk, cutoff):
    k, l, dg = Wk.shape
    out = torch.empty((num_triplets, dg), dtype=torch.float32, device=X.device)
    call("egn_triplet_terms", ptr(edge_ptr), ptr(rev), ptr(geo), ptr(tri_ptr), edge_ptr.shape[0] - 1,
         ptr(_c(X, torch.float32)), ptr(_c(Wk, torch.float32)), k, l, dg, float(cutoff), ptr(out), stream())
    return out


def aggregate_in_edges(edge_ptr, rev, x, out=None):
    nv = edge_ptr.shape[0] - 1
    d = x.shape[1]
    if out is None:
        out = torch.empty((nv, d), dtype=torch.float32, device=x.device)
    call("egn_aggregate_in_edges", ptr(edge_ptr), ptr(rev), nv, ptr(x), x.stride(0), d, ptr(out), stream())
    return out


def gather_rows(idx, x, out=None, accumulate=False):
    rows = idx.shape[0]
    d = x.shape[1]
    if out is None:
        out = torch.empty((rows, d), dtype=torch.float32, device=x.device)
    call("egn_gather_rows", ptr(idx), rows, ptr(x), x.stride(0), d, ptr(out), out.stride(0), int(accumulate),
         stream())
    return out


def scatter_rows(dst, src, x, out, accumulate=True):
    """out[dst[r]] (+)= x[src[r]] (distinct dst)."""
    rows = dst.shape[0]
    call("egn_scatter_rows", ptr(dst), ptr(src), rows, ptr(x), x.stride(0), x.shape[1], ptr(out), out.stride(0),
         int(accumulate), stream())
    return out


def graph_sum(graph_ptr, x):
    g = graph_ptr.shape[0] - 1
    out = torch.empty((g, x.shape[1]), dtype=torch.float32, device=x.device)
    call("egn_graph_sum", ptr(graph_ptr), g, ptr(_c(x, torch.float32)), x.shape[1], ptr(out), stream())
    return out


def force_head_fwd(edge_ptr, rev, geo, m, w):
    nv = edge_ptr.shape[0] - 1
    ne = m.shape[0]
    scale = torch.empty(ne, dtype=torch.float32, device=m.device)
    forces = torch.empty((nv, 3), dtype=torch.float32, device=m.device)
    call("egn_force_head_fwd", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ne, ptr(_c(m, torch.float32)), m.shape[1],
         ptr(_c(w, torch.float32)), ptr(scale), ptr(forces), stream())
    return scale, forces


def force_head_scale(m, w, out):
    """s_e = m_e . w into out [rows] (first half of egn_force_head_fwd)."""
    call("egn_force_head_fwd", None, None, None, 0, m.shape[0], ptr(_c(m, torch.float32)), m.shape[1],
         ptr(_c(w, torch.float32)), ptr(out), None, stream())
    return out


def force_head_gather(edge_ptr, rev, geo, scale, d):
    """f[v] = sum over v's in-edges of s_e u_e for the centres of edge_ptr (second half)."""
    nv = edge_ptr.shape[0] - 1
    forces = torch.empty((nv, 3), dtype=torch.float32, device=scale.device)
    call("egn_force_head_fwd", ptr(edge_ptr), ptr(rev), ptr(geo), nv, 0, None, int(d), None, ptr(scale),
         ptr(forces), stream())
    return forces


def force_head_bwd(recv, geo, m, w, scale, f_bar, m_bar, edge_grad, w_bar=None):
    ne, d = m.shape
    if w_bar is None:
        w_bar = torch.empty(d, dtype=torch.float32, device=m.device)
    nbytes = call("egn_force_head_bwd_workspace_bytes", ne, d)
    ws = _workspace(nbytes, m.device)
    call("egn_force_head_bwd", ptr(recv), ptr(geo), ne, ptr(m), d, ptr(w), ptr(scale), ptr(_c(f_bar, torch.float32)),
         ptr(m_bar), ptr(w_bar), ptr(edge_grad), ptr(ws), stream())
    return w_bar


def rbf_bwd(geo, rbf_bar, cutoff, edge_grad, basis=0):
    ne, k = rbf_bar.shape
    name = "egn_rbf_bessel_bwd" if basis else "egn_rbf_bwd"
    call(name, ptr(geo), ptr(_c(rbf_bar, torch.float32)), ne, k, float(cutoff), ptr(edge_grad), stream())


def positions_bwd(edge_ptr, rev, geo, edge_grad):
    nv = edge_ptr.shape[0] - 1
    out = torch.empty((nv, 3), dtype=torch.float64, device=geo.device)
    call("egn_positions_bwd", ptr(edge_ptr), ptr(rev), ptr(geo), nv, ptr(edge_grad), ptr(out), stream())
    return out


def column_sum(x, out=None):
    """out[c] = sum_r x[r, c] (deterministic)."""
    rows, d = x.shape
    if x.stride(1) != 1:
        x = x.contiguous()
    if out is None:
        out = torch.empty(d, dtype=torch.float32, device=x.device)
    nbytes = call("egn_column_sum_workspace_bytes", rows, d)
    ws = _workspace_named("colsum", nbytes, x.device)
    call("egn_column_sum", ptr(x), rows, d, x.stride(0), ptr(out), ptr(ws), stream())
    return out


EPI_BIAS, EPI_RESID, EPI_GATHER, EPI_SILU_OUT2, EPI_MUL_AUX, EPI_DSILU_AUX = 1, 2, 4, 8, 16, 32


def _rowmajor(t):
    return t if t.stride(1) == 1 else t.contiguous()


def gemm(a, b, a2=None, b2=None, bias=None, resid=None, gather=None, aux=None, flags=0, out=None, out2=None,
         b_mn=False, b_lo=None, b2_lo=None):
    """out = a b^T (+ a2 b2^T) with the fused epilogue of egn_gemm (tcgen05, 3xTF32).

    a: [M, K] rows, b: [N, K] (weights stored (out, in)), or with b_mn=True b: [K, N]
    (so a @ W for a weight W [K, N] needs no transpose); gather = (src [*, N], idx int32 [M])."""
    a, b = _rowmajor(a), _rowmajor(b)
    M, K = a.shape
    N = b.shape[1] if b_mn else b.shape[0]
    nseg = 1 if a2 is None else 2
    if nseg == 2:
        a2, b2 = _rowmajor(a2), _rowmajor(b2)
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=a.device)
    if bias is not None:
        flags |= EPI_BIAS
    if resid is not None:
        flags |= EPI_RESID
    gsrc = gidx = None
    if gather is not None:
        gsrc, gidx = gather
        flags |= EPI_GATHER
    need2 = flags & (EPI_SILU_OUT2 | EPI_MUL_AUX)
    if need2 and out2 is None:
        out2 = torch.empty((M, N), dtype=torch.float32, device=a.device)
    args = (M, N, nseg, ptr(a), a.stride(0), ptr(b), b.stride(0), K,
            ptr(a2) if nseg == 2 else None, a2.stride(0) if nseg == 2 else 0,
            ptr(b2) if nseg == 2 else None, b2.stride(0) if nseg == 2 else 0, a2.shape[1] if nseg == 2 else 0,
            ptr(bias), ptr(resid), resid.stride(0) if resid is not None else 0,
            ptr(gsrc), ptr(gidx), gsrc.stride(0) if gsrc is not None else 0,
            ptr(aux), aux.stride(0) if aux is not None else 0, int(flags),
            ptr(out), out.stride(0), ptr(out2), out2.stride(0) if out2 is not None else 0, int(b_mn))
    if (b_lo is not None and b_lo.stride(-1) == 1 and b.stride(-1) == 1
            and (nseg == 1 or (b2_lo is not None and b2_lo.stride(-1) == 1 and b2.stride(-1) == 1))):
        call("egn_gemm_blo", *args, ptr(b_lo), b_lo.stride(0), ptr(b2_lo) if nseg == 2 else None,
             b2_lo.stride(0) if nseg == 2 else 0, stream())
    else:
        call("egn_gemm", *args, stream())
    return (out, out2) if need2 else out


# ---- tf32 lo parts of the weights (egn_gemm_blo) -------------------------------------------
# A flat weight buffer registers a same-shaped lo buffer; refresh_weight_lo recomputes it
# (every forward pass starts with it, so the lo parts always match the weights the pass reads;
# inside a captured step the refresh is part of the graph).  linear() passes the lo view of any
# weight that is a view of a registered buffer; other B operands keep the in-kernel split.
class _LoPair:
    __slots__ = ("flat", "lo", "__weakref__")

    def __init__(self, flat, lo):
        self.flat, self.lo = flat, lo


_LO_REG = weakref.WeakValueDictionary()
_LO_OFF = os.environ.get("EGN_GEMM_BLO", "1") == "0"  # A/B switch: in-kernel split only


def register_weight_lo(flat):
    """Allocate the lo buffer of a flat fp32 weight buffer and register it; returns the holder
    (keep it alive as long as the buffer: the registry holds it weakly)."""
    pair = _LoPair(flat, torch.empty_like(flat))
    _LO_REG[flat.untyped_storage().data_ptr()] = pair
    return pair


def refresh_weight_lo(flat):
    """Recompute the registered lo buffer of flat (one egn_tf32_lo launch; no-op if unregistered)."""
    pair = _LO_REG.get(flat.untyped_storage().data_ptr())
    if pair is None:
        return
    n = flat.numel()
    call("egn_tf32_lo", ptr(pair.flat), 1, n, n, ptr(pair.lo), n, stream())


def _weight_lo(w):
    if w is None or _LO_OFF or not _LO_REG or w.device.type != "cuda":
        return None
    pair = _LO_REG.get(w.untyped_storage().data_ptr())
    if pair is None:
        return None
    return pair.lo.as_strided(w.shape, w.stride(), w.storage_offset())


def gemm_wgrad(g, x, out=None, accumulate=False, colsum=None):
    """out[M, N] (+)= g^T x for g [R, M], x [R, N] on the tensor cores (split over R);
    out may be a row-strided view.  colsum [M] (+)= column sums of g (the bias adjoint)."""
    g, x = _rowmajor(g), _rowmajor(x)
    R, M = g.shape
    N = x.shape[1]
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=g.device)
    if out.stride(1) != 1:
        raise ValueError("gemm_wgrad output rows must be contiguous")
    if colsum is not None and not colsum.is_contiguous():
        raise ValueError("gemm_wgrad column-sum output must be contiguous")
    nbytes = call("egn_gemm_wgrad_workspace_bytes", R, M, N)
    ws = _workspace_named("wgrad", nbytes, g.device)
    call("egn_gemm_wgrad", R, M, N, ptr(g), g.stride(0), ptr(x), x.stride(0), ptr(out), out.stride(0),
         ptr(colsum) if colsum is not None else None, int(accumulate), ptr(ws), stream())
    return out


def _tc_ok(k, n, *ts):
    """Shapes the tcgen05 GEMM tiles (K % 4, N % 16, 16-byte aligned rows)."""
    if k % 4 or n % 16 or n < 16:
        return False
    for t in ts:
        if t is not None and (t.data_ptr() % 16 or (t.dim() == 2 and t.stride(0) % 4) or t.stride(-1) != 1):
            return False
    return True


def linear(a, w, a2=None, w2=None, bias=None, resid=None, gather=None, aux=None, flags=0, w_mn=False, out=None):
    """Dense layer y = a w^T (+ a2 w2^T) (+ bias, resid, gathered rows; SiLU / gate / SiLU' epilogues).

    w is stored (out, in) as in the reference (egn/tape.py:104-119); w_mn=True
    computes a @ w instead (the data gradient).  Always the tcgen05 3xTF32 GEMM (or its
    small-M SIMT sibling inside egn_gemm): shapes must map onto the UMMA tiling (N % 16 == 0,
    K % 4 == 0, 16-byte aligned rows) -- the engine pads every feature width to a multiple
    of 16 (DeviceWeights / ModelConfig.padded), so no model product ever needs a fallback.
    out: optional row-major destination (e.g. the owned rows of a full-size buffer).
    Returns y, or (y, out2) for EPI_SILU_OUT2 / EPI_MUL_AUX."""
    k = a.shape[1]
    n = w.shape[1] if w_mn else w.shape[0]
    ok = _tc_ok(k, n, a, w, a2, w2, resid, aux, out)
    if a2 is not None:
        ok = ok and a2.shape[1] % 4 == 0 and not w_mn
    if gather is not None:
        ok = ok and gather[0].stride(-1) == 1
    if not ok:
        raise ValueError(f"linear: [{a.shape[0]} x {k}] x [{k} x {n}] does not map onto the tcgen05 tiling "
                         "(N % 16, K % 4, 16-byte aligned rows)")
    return gemm(a, w, a2=a2, b2=w2, bias=bias, resid=resid, gather=gather, aux=aux, flags=flags, b_mn=w_mn, out=out,
                b_lo=_weight_lo(w), b2_lo=_weight_lo(w2))


def linear_wgrad(g, x, out, bias_out=None):
    """out = g^T x (weight gradient over all rows); bias_out = column sums of g."""
    if not (_tc_ok(4, x.shape[1], g, x) and out.stride(1) == 1):
        raise ValueError(f"linear_wgrad: N = {x.shape[1]} does not map onto the tcgen05 tiling")
    return gemm_wgrad(g, x, out=out, colsum=bias_out)


def small_gemms(problems):
    """One launch for many weight-sized products C = op(A) op(B) (egn_small_gemm_batched).

    problems: (A, B, C, trans_a, trans_b, trans_c) with 2-D tensors whose rows are
    contiguous; op(A) is [m, k] (A is [k, m] when trans_a), op(B) is [k, n] (B is [n, k]
    when trans_b), C is [m, n] ([n, m] when trans_c)."""
    from ._lib import SmallGemm

    if not problems:
        return
    arr = (SmallGemm * len(problems))()
    for i, (A, B, C, ta, tb, tc) in enumerate(problems):
        for t in (A, B, C):
            if t.dtype != torch.float32 or t.dim() != 2 or t.stride(1) != 1:
                raise ValueError("small_gemms takes fp32 2-D tensors with contiguous rows")
        m, k = (A.shape[1], A.shape[0]) if ta else (A.shape[0], A.shape[1])
        kb, n = (B.shape[1], B.shape[0]) if tb else (B.shape[0], B.shape[1])
        cm, cn = (C.shape[1], C.shape[0]) if tc else (C.shape[0], C.shape[1])
        if kb != k or cm != m or cn != n:
            raise ValueError(f"small_gemms: shape mismatch {tuple(A.shape)} {tuple(B.shape)} {tuple(C.shape)}")
        arr[i] = SmallGemm(ptr(A), ptr(B), ptr(C), m, n, k, A.stride(0), B.stride(0), C.stride(0), int(ta), int(tb),
                           int(tc))
    call("egn_small_gemm_batched", ctypes.addressof(arr), len(problems), stream())


def zero_(t):
    """t[:] = 0 on the device (egn_zero: a memset, no framework fill kernel)."""
    if not t.is_contiguous():
        raise ValueError("zero_ takes contiguous tensors")
    call("egn_zero", ptr(t), t.numel() * t.element_size(), stream())
    return t


def zeros(shape, device, dtype=torch.float32):
    return zero_(torch.empty(shape, dtype=dtype, device=device))


def hadamard(a, b, out=None):
    """out = a * b elementwise (egn_hadamard)."""
    a, b = _c(a, torch.float32), _c(b, torch.float32)
    if a.shape != b.shape:
        raise ValueError(f"hadamard: shapes {tuple(a.shape)} and {tuple(b.shape)} differ")
    if out is None:
        out = torch.empty_like(a)
    call("egn_hadamard", ptr(a), ptr(b), ptr(out), a.numel(), stream())
    return out


def transpose_into(src, dst):
    """dst[c, r] = src[r, c] for 2-D fp32 views with contiguous rows (egn_transpose)."""
    if src.dim() != 2 or dst.dim() != 2 or src.stride(1) != 1 or dst.stride(1) != 1:
        raise ValueError("transpose_into takes 2-D views with contiguous rows")
    if dst.shape[0] != src.shape[1] or dst.shape[1] != src.shape[0]:
        raise ValueError("transpose_into: shape mismatch")
    call("egn_transpose", ptr(src), src.shape[0], src.shape[1], src.stride(0), ptr(dst), dst.stride(0), stream())
    return dst


def csr_ptr(keys, num_rows):
    """CSR offsets [num_rows + 1] of sorted int64 row keys (egn_csr_ptr)."""
    keys = _c(keys, torch.int64)
    out = torch.empty(int(num_rows) + 1, dtype=torch.int64, device=keys.device)
    call("egn_csr_ptr", ptr(keys), keys.numel(), int(num_rows), ptr(out), stream())
    return out


def sgd_(w, g, lr):
    call("egn_sgd", ptr(w), ptr(g), w.numel(), float(lr), stream())


def loss_seeds(energy, e_target, forces, f_target, atom_count, w_energy, w_forces, n):
    """(loss f64 [], d_energy f32 [G], d_forces f32 [V, 3] or None) in one launch
    (egn_loss_seeds; egn/tasks.py:166-176).  forces=None: energy terms only."""
    G = energy.shape[0]
    dev = energy.device
    loss = torch.empty((), dtype=torch.float64, device=dev)
    d_e = torch.empty(G, dtype=torch.float32, device=dev)
    d_f = None
    V = 0
    if forces is not None:
        forces, f_target = _c(forces, torch.float32), _c(f_target, torch.float64)
        V = forces.shape[0]
        d_f = torch.empty((V, 3), dtype=torch.float32, device=dev)
    call("egn_loss_seeds", ptr(_c(energy, torch.float32)), ptr(_c(e_target, torch.float64)), G,
         ptr(forces) if forces is not None else None, ptr(f_target) if forces is not None else None,
         ptr(_c(atom_count, torch.float64)) if forces is not None else None, V, float(w_energy),
         float(w_forces), float(n), ptr(loss), ptr(d_e), ptr(d_f) if d_f is not None else None, stream())
    return loss, d_e, d_f


def adamw_(w, g, m, v, lr, step, betas=(0.9, 0.999), eps=1e-8, weight_decay=1e-2):
    """In-place AdamW step `step` (>= 1) on flat fp32 buffers (egn_adamw)."""
    call("egn_adamw", ptr(w), ptr(g), ptr(m), ptr(v), w.numel(), float(lr), float(betas[0]), float(betas[1]),
         float(eps), float(weight_decay), int(step), stream())
