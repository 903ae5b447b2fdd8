/*
 * egn_b200.h -- C ABI of the B200-native EGN (DimeNet++/GemNet-T) hot path.
 *
 * Every entry point takes raw device pointers, element counts and a CUDA
 * stream (passed as void*), launches its kernels on that stream and returns
 * 0 on success or a nonzero status; egn_last_error() then returns a
 * thread-local message.  Outputs are caller-allocated; nothing here
 * allocates device memory.  There is no CPU fallback: every call launches
 * sm_100a kernels.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src):
 * each declaration names the egn function (file:line) whose array result it
 * produces.  Index conventions:
 *   - edges are sorted by (source, receiver) inside each graph and graphs
 *     are concatenated (graph.py:93 row-major nonzero);
 *   - edge_ptr[V+1] is the CSR of out-edges by source node;
 *   - triplets of centre atom j occupy the contiguous range
 *     [tri_ptr[j], tri_ptr[j+1]) with tri_ptr[j+1]-tri_ptr[j] = deg(j)(deg(j)-1),
 *     ordered by (out-edge, in-edge) exactly as enumerate_triplets
 *     (graph.py:106-139) orders them.
 */
#ifndef EGN_B200_H
#define EGN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* egn_stream_t; /* cudaStream_t */

/* Thread-local description of the last failure (never NULL). */
const char* egn_last_error(void);
/* ABI version (bumped on any signature change). */
int egn_abi_version(void);

/* ------------------------------------------------------------------ */
/* Graph construction: build_graph (graph.py:82-103)                   */
/* ------------------------------------------------------------------ */

/* Out-degree of every node: count of b in the node's graph with
 * 0 < |x_b - x_a| <= cutoff, distances in fp64 as ((dx*dx+dy*dy)+dz*dz)
 * without FMA contraction (graph.py:89-92).  node_graph[a] is a's graph;
 * graph_ptr[G+1] the node offsets. */
int egn_neighbors_count(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                        int64_t num_nodes, double cutoff, int32_t* deg, egn_stream_t stream);

/* Exclusive scan out[0]=0, out[i+1]=out[i]+in[i] (int32 in, int64 out, n+1 outputs).
 * If square_minus_one is nonzero, scans in[i]*(in[i]-1) instead (triplet
 * offsets tri_ptr from out-degrees, graph.py:124-139). */
int egn_scan_counts(const int32_t* in, int64_t n, int square_minus_one, int64_t* out,
                    egn_stream_t stream);

/* Fill src/recv of every edge, row-major order (graph.py:93); edge_ptr from
 * egn_scan_counts(deg). */
int egn_neighbors_fill(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                       int64_t num_nodes, double cutoff, const int64_t* edge_ptr, int32_t* src,
                       int32_t* recv, egn_stream_t stream);

/* rev[e] = index of the edge (recv_e, src_e)  (GraphTopology.reverse_edges,
 * graph.py:40-55).  *missing (device int32) receives the count of edges
 * without a reverse partner. */
int egn_reverse_edges(const int64_t* edge_ptr, const int32_t* src, const int32_t* recv,
                      int64_t num_edges, int32_t* rev, int32_t* missing, egn_stream_t stream);

/* Materialise id3_kj (trip_in) and id3_ji (trip_out) as int64 (enumerate_triplets,
 * graph.py:106-139); tri_ptr from egn_scan_counts(deg, square_minus_one=1). */
int egn_triplets_fill(const int64_t* edge_ptr, const int32_t* rev, const int64_t* tri_ptr,
                      int64_t num_nodes, int64_t* id3_kj, int64_t* id3_ji, egn_stream_t stream);

/* Per-edge geometry (edge_distances / edge_unit_vectors, graph.py:142-150).
 * geo[e] = (ux, uy, uz, d) in fp32 (the model's packed layout); dist64 [E]
 * and unit64 [E,3] optional (NULL to skip) in fp64. */
int egn_geometry(const double* pos, const int32_t* src, const int32_t* recv, int64_t num_edges,
                 float* geo, double* dist64, double* unit64, egn_stream_t stream);

/* Triplet angles atan2(|v1 x v2|, v1.v2) in fp64 (triplet_angles, graph.py:162-170). */
int egn_triplet_angles(const double* pos, const int64_t* edge_ptr, const int32_t* recv,
                       const int64_t* tri_ptr, int64_t num_nodes, double* angles,
                       egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Periodic cells (no counterpart in the reference,  */
/* which is non-periodic: parity is pinned by an explicit supercell     */
/* expansion through the reference build_graph, tests/golden/pbc.npz)   */
/* ------------------------------------------------------------------ */
/*
 * Per graph g: cell[9g..9g+8] = lattice vectors c0, c1, c2 (rows, fp64) and
 * nimg[3g..3g+2] = (na, nb, nc) images per axis (0 on a non-periodic axis).
 * Image index img = ((i+na)(2nb+1) + (j+nb))(2nc+1) + (k+nc) for i in [-na, na] ...;
 * shift s = (i c0 + j c1) + k c2 per component (fp64, round-to-nearest, no FMA).
 * An edge (a, b, img) has the vector (x_b - x_a) + s (exactly antisymmetric, so
 * every edge has its reverse) and exists iff
 * 0 < |v| <= cutoff (and not (b == a, s == 0)); each row is ordered by (b, img),
 * so a row is sorted by (recv, img) and the reverse of (a, b, img) is
 * (b, a, n_img - 1 - img).  Degrees/counts/triplets then follow the
 * non-periodic CSR conventions above (triplet exclusion is by edge: the
 * in-edge is never the reverse of the out-edge).
 */
int egn_neighbors_count_pbc(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                            int64_t num_nodes, const double* cell, const int32_t* nimg, double cutoff, int32_t* deg,
                            egn_stream_t stream);
/* src/recv/img [E] and shift [E,3] (fp64) of every periodic edge, rows ordered by (recv, img). */
int egn_neighbors_fill_pbc(const double* pos, const int64_t* graph_ptr, const int32_t* node_graph,
                           int64_t num_nodes, const double* cell, const int32_t* nimg, double cutoff,
                           const int64_t* edge_ptr, int32_t* src, int32_t* recv, int32_t* img, double* shift,
                           egn_stream_t stream);
/* rev[e] = index of (recv_e, src_e, mirrored image); *missing counts edges without one. */
int egn_reverse_edges_pbc(const int64_t* edge_ptr, const int32_t* src, const int32_t* recv, const int32_t* img,
                          const int32_t* node_graph, const int32_t* nimg, int64_t num_edges, int32_t* rev,
                          int32_t* missing, egn_stream_t stream);
/* Neighbour cap (OC20 max-neighbours; reference-free, pinned to the
 * oracle restatement): keep1[e] = e is among the max_neighbors nearest out-edges of its
 * source (fp64 distance, then edge index); keep[e] = keep1[e] && keep1[rev[e]] (mutual, so the
 * graph stays symmetric); deg[v] = kept out-degree. */
int egn_cap_keep(const int64_t* edge_ptr, const double* dist, const int32_t* rev, int64_t num_nodes, int max_neighbors,
                 int32_t* keep1, int32_t* keep, int32_t* deg, egn_stream_t stream);
/* Compact the kept edges in row order into new_ptr (egn_scan_counts of the kept degrees):
 * new_id[e] (-1 if dropped), src/recv (+ img / shift of periodic graphs, NULL otherwise) and the
 * remapped reverse edges nrev. */
int egn_cap_compact(const int64_t* edge_ptr, const int64_t* new_ptr, int64_t num_nodes, int64_t num_edges,
                    const int32_t* keep, const int32_t* src, const int32_t* recv, const int32_t* img,
                    const double* shift, const int32_t* rev, int32_t* new_id, int32_t* nsrc, int32_t* nrecv,
                    int32_t* nimg, double* nshift, int32_t* nrev, egn_stream_t stream);
/* egn_geometry / egn_triplet_angles on edge vectors (x_recv - x_src) + shift; shift NULL
 * gives the non-periodic results bit for bit. */
int egn_geometry_shift(const double* pos, const int32_t* src, const int32_t* recv, const double* shift,
                       int64_t num_edges, float* geo, double* dist64, double* unit64, egn_stream_t stream);
int egn_triplet_angles_shift(const double* pos, const int64_t* edge_ptr, const int32_t* recv, const double* shift,
                             const int64_t* tri_ptr, int64_t num_nodes, double* angles, egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Basis: rbf_features / rbf_features_ddist (basis.py:35-51)           */
/* ------------------------------------------------------------------ */

/* rbf[e,k] = exp(-gamma (d_e - c_k)^2), c = linspace(0, cutoff, K) (c=[0] if K=1),
 * gamma = (K/cutoff)^2; fp32 [E,K]. */
int egn_rbf(const float* geo, int64_t num_edges, int k_rbf, double cutoff, float* rbf,
            egn_stream_t stream);

/* SBF rows (t, k*L+l) = rbf_k(d_kj) cos(l alpha_t) for every triplet (sbf_features,
 * basis.py:54-73), fp32 [N_t, K*L].  Debug/parity only: the model never
 * materialises per-triplet basis rows. */
int egn_sbf(const float* geo, const int64_t* edge_ptr, const int64_t* tri_ptr, int64_t num_nodes,
            int k_rbf, int l_sbf, double cutoff, float* sbf, egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Triplet interaction: record_tu (engine.py:118-149)                  */
/* ------------------------------------------------------------------ */
/*
 * With rq = rev(off_j + q) the in-edge (k->j) of centre j and x_pq = u_p . u_q
 * (= cos alpha of triplet (q -> p)):
 *   S[off_j+p, c] = sum_{q != p} X[rq, c] * sum_l T_l(x_pq) * Rw[rq, l, c],
 *   Rw[e, l, c]   = sum_k rbf_k(d_e) * W[k, l, c].
 * X is the per-edge down projection (dimenet: m W_down^T; gemnet:
 * m W_down^T A^T), W the sbf gate reshaped to [K, L, dg] (gemnet: B W_sbf).
 * The gate by rbf(d_ji) and the up projection are applied by the caller on
 * the per-edge result, which is exact because both are constant or linear
 * inside a triplet segment (engine.py:138,147-148).
 * max_degree: max deg(j) if known (selects the deg<=64 fast path alone, and sizes the
 * spherical-harmonic path's per-chunk moments), -1 if not.
 * workspace: egn_triplet_fwd_workspace_bytes(...) bytes (NULL: the spherical-harmonic path is
 * not used).
 */
int64_t egn_triplet_fwd_workspace_bytes(int64_t num_nodes, int max_degree, int k_rbf, int l_sbf, int dg);
int egn_triplet_fwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                    int64_t num_nodes, int max_degree, const float* X, const float* W, int k_rbf,
                    int l_sbf, int dg, double cutoff, float* S, void* workspace, egn_stream_t stream);

/* DimeNet++ / GemNet bases (no reference counterpart): basis 0 = the
 * reference's Gaussian rbf x cos(l angle) (= egn_triplet_fwd / _bwd), 1 = GemNet CBF (radial
 * Bessel basis e_k(d_kj) x Y_l0(angle)), 2 = DimeNet SBF (sqrt(2/c^3) / |j_{l+1}(z_lk)|
 * u(d_kj/c) j_l(z_lk d_kj / c) x Y_l0(angle)); the radial Bessel basis is
 * e_k(d) = sqrt(2/c) u(d/c) sin((k+1) pi d/c) with the polynomial envelope u (p = 6).  Bases 1
 * and 2 run the spherical-harmonic kernels (k_rbf = 6, l_sbf = 7) and need max_degree and the
 * workspace of egn_triplet_fwd_basis_workspace_bytes / egn_triplet_bwd_basis_workspace_bytes
 * (which includes the per-call radial table of the edges: the Bessel rows depend on the
 * geometry only and are tabulated once, one thread per element, instead of per lane). */
int64_t egn_triplet_fwd_basis_workspace_bytes(int64_t num_nodes, int64_t num_edges, int max_degree, int k_rbf,
                                              int l_sbf, int dg, int basis);
int64_t egn_triplet_bwd_basis_workspace_bytes(int64_t num_nodes, int64_t num_edges, int max_degree, int k_rbf,
                                              int l_sbf, int dg, int basis);
int egn_triplet_fwd_basis(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                          int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                          int dg, double cutoff, int basis, float* S, void* workspace, egn_stream_t stream);
int egn_triplet_bwd_basis(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                          int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                          int dg, double cutoff, int basis, const float* S_bar, float* X_bar, float* W_bar,
                          float* edge_grad, void* workspace, egn_stream_t stream);
/* egn_triplet_bwd_basis in the phases of egn_triplet_bwd_ex (centres of degree <= 64, both
 * bases; on the forced spherical-harmonic path phase 1 does nothing and phase 2 all).  Phase 1 needs its own workspace of
 * egn_triplet_bwd_angle_workspace_bytes (its radial table), so both phases can run at once. */
int64_t egn_triplet_bwd_angle_workspace_bytes(int64_t num_edges, int basis);
int egn_triplet_bwd_basis_ex(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                             int64_t num_edges, int max_degree, const float* X, const float* W, int k_rbf, int l_sbf,
                             int dg, double cutoff, int basis, int phases, const float* S_bar, float* X_bar,
                             float* W_bar, float* edge_grad, void* workspace, egn_stream_t stream);
/* Edge radial Bessel basis [E, K] of the packed geometry and its adjoint (edge_grad.w +=). */
int egn_rbf_bessel(const float* geo, int64_t num_edges, int k_rbf, double cutoff, float* rbf, egn_stream_t stream);
int egn_rbf_bessel_bwd(const float* geo, const float* rbf_bar, int64_t num_edges, int k_rbf, double cutoff,
                       float* edge_grad, egn_stream_t stream);
/* Triplet kernel selection (returns the previous mode; -1 queries): 0 = auto (deg <= 64:
 * pairwise centre tiles; larger centres: linear-in-degree spherical-harmonic kernels, the
 * angular sum factorised by the addition theorem -- triplet_sh.cu), 1 = spherical-harmonic
 * kernels for every centre, 2 = pairwise kernels only (tensor-core kernels above deg 64). */
int egn_triplet_path(int mode);
/* Triplet window (graph-parallel reference schedule: one split_range shard of the triplet
 * list, egn/partition.py:28-37, egn/runtime.py:425-431).  The launch covers the centres of
 * edge_ptr[0 .. num_nodes] and keeps only triplets whose centre-local index
 * k = p (n-1) + (q < p ? q : q-1) is >= first_lo at the first centre and < last_hi at the last;
 * the kept terms are summed exactly as egn_triplet_fwd does (rows of every covered centre are
 * written, zero where no triplet of the row is kept). */
int egn_triplet_fwd_window(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                           int64_t first_lo, int64_t last_hi, const float* X, const float* W, int k_rbf, int l_sbf,
                           int dg, double cutoff, float* S, egn_stream_t stream);
/* Adjoint of egn_triplet_fwd_window: X_bar rows rev(q) of the covered centres overwritten,
 * W_bar overwritten, edge_grad accumulated (workspace: egn_triplet_bwd_workspace_bytes). */
int egn_triplet_bwd_window(const int64_t* edge_ptr, const int32_t* rev, const float* geo, int64_t num_nodes,
                           int64_t first_lo, int64_t last_hi, int max_degree, const float* X, const float* W,
                           int k_rbf, int l_sbf, int dg, double cutoff, const float* S_bar, float* X_bar,
                           float* W_bar, float* edge_grad, void* workspace, egn_stream_t stream);
/* Adjoint of egn_triplet_fwd (tape.py gather/segment_sum/linear/angular_sbf VJPs).
 * Inputs S_bar [E,dg].  Outputs:
 *   X_bar [E, dg]            (overwritten),
 *   W_bar [K, L, dg]          (overwritten; reduced over all centres),
 *   edge_grad [E, 4] float   (+=): (dE/dv_e (3), dE/dd_e) for the edge
 *                              vector v_e = x_recv - x_src from the angles and the
 *                              in-edge distance of the basis.
 * max_degree bounds deg(j) over all centres (sizes shared memory).
 * workspace: egn_triplet_bwd_workspace_bytes(...) bytes of device memory. */
int64_t egn_triplet_bwd_workspace_bytes(int64_t num_nodes, int64_t num_edges, int max_degree, int k_rbf,
                                        int l_sbf, int dg);
int egn_triplet_bwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                    int64_t num_nodes, int64_t num_edges, int max_degree, const float* X,
                    const float* W, int k_rbf, int l_sbf, int dg, double cutoff, const float* S_bar,
                    float* X_bar, float* W_bar, float* edge_grad, void* workspace,
                    egn_stream_t stream);
/* egn_triplet_bwd in two phases that touch disjoint outputs, so they can run on two streams:
 *   phases = 1: the angle adjoint of the small-degree centres (edge_grad x, y, z only);
 *   phases = 2: everything else (X_bar, W_bar, edge_grad.w, and all of the larger centres);
 *   phases = 3: both (== egn_triplet_bwd).
 * Where the split does not apply (other triplet paths), phases = 1 does nothing and
 * phases = 2 does the whole adjoint.  Phase 1 uses no workspace. */
int egn_triplet_bwd_ex(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                       int64_t num_nodes, int64_t num_edges, int max_degree, const float* X,
                       const float* W, int k_rbf, int l_sbf, int dg, double cutoff, const float* S_bar,
                       float* X_bar, float* W_bar, float* edge_grad, int phases, void* workspace,
                       egn_stream_t stream);

/* Per-triplet feature debug output t_feat-like rows for parity tests:
 * P[t, c] = X[rq, c] * sum_l T_l(x_pq) Rw[rq, l, c] for every triplet t in
 * (out, in) order (the summand of egn_triplet_fwd). */
int egn_triplet_terms(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                      const int64_t* tri_ptr, int64_t num_nodes, const float* X, const float* W,
                      int k_rbf, int l_sbf, int dg, double cutoff, float* P, egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Edge/node aggregation: segment_sum / gather (tape.py:129-154)       */
/* ------------------------------------------------------------------ */

/* out[v, c] = sum over in-edges e of v (recv(e) = v, ascending e) of x[e, c];
 * in-edges of v are rev(out-edges of v).  (record_ea_nu, engine.py:166-177) */
int egn_aggregate_in_edges(const int64_t* edge_ptr, const int32_t* rev, int64_t num_nodes,
                           const float* x, int64_t ld_x, int d, float* out, egn_stream_t stream);

/* out[e, c] (+)= x[idx[e], c]: row gather with optional accumulate (gather, tape.py:129-139). */
int egn_gather_rows(const int32_t* idx, int64_t rows, const float* x, int64_t ld_x, int d,
                    float* out, int64_t ld_out, int accumulate, egn_stream_t stream);

/* out[dst[r], c] (+)= x[src[r], c] with distinct dst within one call: the adjoint of a
 * row gather restricted to one rank's rows (graph-parallel backward, runtime.py). */
int egn_scatter_rows(const int32_t* dst, const int32_t* src, int64_t rows, const float* x,
                     int64_t ld_x, int d, float* out, int64_t ld_out, int accumulate,
                     egn_stream_t stream);

/* out[g, c] = sum_{v in graph g} x[v, c]  (sum_rows in record_gu_head, engine.py:207-211). */
int egn_graph_sum(const int64_t* graph_ptr, int64_t num_graphs, const float* x, int d,
                  float* out, egn_stream_t stream);

/* GemNet direct force head (record_force_head, engine.py:234-246):
 *   s_e = m_e . w ; f[v] = sum_{recv(e)=v} s_e u_e.  scale [E] is an output.
 * m NULL: scale is an input (the graph-parallel runtime all-gathers it between the two
 * halves); forces NULL: only the per-edge dot products s_e. */
int egn_force_head_fwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                       int64_t num_nodes, int64_t num_edges, const float* m, int d,
                       const float* w, float* scale, float* forces, egn_stream_t stream);
/* Adjoint: m_bar[e] += (f_bar[recv e] . u_e) w ; edge_grad[e].xyz += unit-vector adjoint
 * (tape.py:197-209 edge_units VJP folded into dE/dv_e); w_bar_partial [blocks, d]. */
int egn_force_head_bwd(const int32_t* recv, const float* geo, int64_t num_edges, const float* m,
                       int d, const float* w, const float* scale, const float* f_bar,
                       float* m_bar, float* w_bar, float* edge_grad, void* workspace,
                       egn_stream_t stream);
int64_t egn_force_head_bwd_workspace_bytes(int64_t num_edges, int d);

/* K <= 8 linears of the radial basis (edge_init engine.py:109-111, rbf gate engine.py:138):
 * out[e, n] (row stride ldo) = sum_k rbf[e, k] w[n, k] (+ b[n] if b != NULL); N % 4 == 0. */
int egn_rbf_linear(const float* rbf, int64_t num_edges, int k, const float* w, const float* b, int n, float* out,
                   int64_t ldo, egn_stream_t stream);
/* Adjoint (linear VJP, tape.py:104-119) for N <= 128: rbf_bar[e,k] += sum_n g[e,n] w[n,k];
 * w_bar = g^T rbf (overwritten), b_bar = column sums of g (overwritten; NULL to skip);
 * deterministic (fixed-order partial reduction).  g2 (NULL to skip, same row stride ldg):
 * the adjoint of a gate product, g := g * g2 elementwise (engine.py:138/146 mul VJP). */
int64_t egn_rbf_linear_bwd_workspace_bytes(int64_t num_edges, int k, int n);
int egn_rbf_linear_bwd(const float* rbf, int64_t num_edges, int k, const float* w, int n, const float* g,
                       const float* g2,
                       int64_t ldg, float* rbf_bar, float* w_bar, float* b_bar, void* workspace,
                       egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Geometry adjoints (tape.py:164-242, runtime.py:626-671)             */
/* ------------------------------------------------------------------ */

/* edge_grad[e].w += sum_k rbf_bar[e,k] d rbf_k/dd (gaussian_rbf VJP, tape.py:219-228). */
int egn_rbf_bwd(const float* geo, const float* rbf_bar, int64_t num_edges, int k_rbf,
                double cutoff, float* edge_grad, egn_stream_t stream);

/* pos_bar[a] = sum_{recv(e)=a} g_e - sum_{src(e)=a} g_e with
 * g_e = edge_grad[e].xyz + edge_grad[e].w * u_e  (fp64 output). */
int egn_positions_bwd(const int64_t* edge_ptr, const int32_t* rev, const float* geo,
                      int64_t num_nodes, const float* edge_grad, double* pos_bar,
                      egn_stream_t stream);

/* Column sums out[c] = sum_r x[r*ld + c] (bias adjoints of linear, tape.py:113-119),
 * deterministic two-stage reduction; workspace from egn_column_sum_workspace_bytes. */
int64_t egn_column_sum_workspace_bytes(int64_t rows, int d);
int egn_column_sum(const float* x, int64_t rows, int d, int64_t ld, float* out, void* workspace,
                   egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Dense layers: linear (tape.py:104-119) on tcgen05 tensor cores      */
/* ------------------------------------------------------------------ */
/* out[M, N] = sum over nseg (1 or 2) segments of A_s[M, K_s] B_s[N, K_s]^T, fp32-accurate
 * (3 x TF32 split on tcgen05.mma kind::tf32, TMEM accumulator), then the fused epilogue
 * selected by flags (applied in this order):
 *   1  += bias[n]            2  += resid[m*ldr + n]     4  += gsrc[gidx[m]*ldg + n]
 *   32 *= silu'(aux[m*ldaux + n])
 *   16 out2 = value; value *= aux[m*ldaux + n]
 *   8  out2 = silu(value) after storing value to out.
 * A is row-major with K contiguous; B is row-major [N, K] (weights stored (out, in)) or,
 * with b_mn != 0, [K, N] with N contiguous (the weight of a data-gradient product);
 * K_s % 4 == 0, N % 16 == 0, pointers 16-byte aligned, row strides multiples of 4. */
/* Products with M <= egn_gemm_simt_max_m (default 8192, env EGN_GEMM_SIMT_MAX_M) run as an
 * fp32 SIMT GEMM with the same epilogue (too few 128-row tiles to fill the GPU); value >= 0
 * sets the threshold, the previous one is returned (value < 0: query only). */
int64_t egn_gemm_simt_max_m(int64_t value);
int egn_gemm(int64_t M, int N, int nseg, const float* a0, int64_t lda0, const float* b0, int64_t ldb0,
             int k0, const float* a1, int64_t lda1, const float* b1, int64_t ldb1, int k1,
             const float* bias, const float* resid, int64_t ldr, const float* gsrc,
             const int32_t* gidx, int64_t ldg, const float* aux, int64_t ldaux, int flags,
             float* out, int64_t ldo, float* out2, int64_t ldo2, int b_mn, egn_stream_t stream);
/* egn_gemm with the tf32 lo parts of B precomputed (b*_lo, from egn_tf32_lo; both segments,
 * 16-byte aligned rows): the tensor-core path loads them by TMA instead of forming them per tile
 * (bit-identical results).  For weights, whose lo parts change only when the weights do
 * (egn/tape.py:104-119 linear). */
int egn_gemm_blo(int64_t M, int N, int nseg, const float* a0, int64_t lda0, const float* b0, int64_t ldb0,
                 int k0, const float* a1, int64_t lda1, const float* b1, int64_t ldb1, int k1,
                 const float* bias, const float* resid, int64_t ldr, const float* gsrc,
                 const int32_t* gidx, int64_t ldg, const float* aux, int64_t ldaux, int flags,
                 float* out, int64_t ldo, float* out2, int64_t ldo2, int b_mn, const float* b0_lo,
                 int64_t ldb0_lo, const float* b1_lo, int64_t ldb1_lo, egn_stream_t stream);
/* lo[r, c] = tf32 lo part of x[r, c] (x - trunc_tf32(x), rounded to tf32) of a row-strided array. */
int egn_tf32_lo(const float* x, int64_t rows, int cols, int64_t ldx, float* lo, int64_t ldl, egn_stream_t stream);

/* Weight gradient out[M, N] (row stride ldo) (+)= g^T x with g [krows, M], x [krows, N] (both
 * MN-major on the tensor cores), split over krows across CTAs; partial tiles reduced in a fixed
 * order.  If g_colsum is non-NULL it also receives (+=) the column sums of g, i.e. the bias
 * adjoint of the same linear (tape.py:113-119), read from the operand tiles already on chip. */
int64_t egn_gemm_wgrad_workspace_bytes(int64_t krows, int M, int N);
int egn_gemm_wgrad(int64_t krows, int M, int N, const float* g, int64_t ldg, const float* x,
                   int64_t ldx, float* out, int64_t ldo, float* g_colsum, int accumulate,
                   void* workspace, egn_stream_t stream);

/* Batched small products C = op(A) op(B) (op = transpose if the flag is set; C stored
 * transposed if trans_c): the weight-sized products of the folded projections
 * (A W_down, W1b W_up, B W_sbf) and their adjoints, all in one launch.  fp32. */
typedef struct {
  const float* a;
  const float* b;
  float* c;
  int m, n, k;
  int lda, ldb, ldc;
  int trans_a, trans_b, trans_c;
} egn_small_gemm_t;
int egn_small_gemm_batched(const egn_small_gemm_t* problems, int count, egn_stream_t stream);

/* Graph-level update block GU (record_gu_head/tail, engine.py:207-217), G graphs:
 *   pre = s W1^T + b1, act = silu(pre), u += act W2^T + b2
 * s [G, dv] (per-graph sum of node features), W1 [du, dv], W2 [du, du]; pre/act [G, du]
 * written, u [G, du] updated in place (two launches, activation / bias / residual fused). */
int egn_graph_mlp_fwd(int64_t num_graphs, int dv, int du, const float* s, const float* w1, const float* b1,
                      const float* w2, const float* b2, float* pre, float* act, float* u, egn_stream_t stream);
/* Adjoint: pre_bar = silu'(pre) (u_bar W2), s_bar = pre_bar W1 [G, dv]; W1_bar = pre_bar^T s,
 * b1_bar = column sums of pre_bar, W2_bar = u_bar^T act, b2_bar = column sums of u_bar
 * (all overwritten; sums over graphs in order). */
int egn_graph_mlp_bwd(int64_t num_graphs, int dv, int du, const float* u_bar, const float* s, const float* pre,
                      const float* act, const float* w1, const float* w2, float* pre_bar, float* s_bar,
                      float* w1_bar, float* b1_bar, float* w2_bar, float* b2_bar, egn_stream_t stream);
/* w1 NULL in egn_graph_mlp_fwd / _bwd: the first layer is the identity (dv == du; its input
 * is the already projected, all-reduced z of the graph-parallel reference schedule,
 * egn/runtime.py:477-484 + egn/engine.py:214-217); w1_bar may then be NULL. */
/* GU head z = x W^T (+ b) over G rows (egn/engine.py:207-211, record_gu_head); w NULL = identity. */
int egn_graph_linear(int64_t num_graphs, int din, int dout, const float* x, const float* w, const float* b, float* y,
                     egn_stream_t stream);
/* Adjoint: x_bar = y_bar W, w_bar = y_bar^T x, b_bar = column sums of y_bar (each optional). */
int egn_graph_linear_bwd(int64_t num_graphs, int din, int dout, const float* y_bar, const float* x, const float* w,
                         float* x_bar, float* w_bar, float* b_bar, egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Basis tables and geometry derivatives at the public API (fp64)      */
/* ------------------------------------------------------------------ */
/* rbf_features (egn/basis.py:35-42): out[e, k] = exp(-gamma (d_e - c_k)^2), c = linspace(0,
 * cutoff, K), gamma = (K / cutoff)^2; d_out (optional) = d/dd (rbf_features_ddist :45-51).
 * invalid (optional device int32) is set to 1 when some d lies outside (0, cutoff] (the
 * reference raises ValueError; the binding checks the flag). */
int egn_rbf_features(const double* distances, int64_t n, int k_rbf, double cutoff, double* out, double* d_out,
                     int32_t* invalid, egn_stream_t stream);
/* sbf_features (egn/basis.py:54-74): out[t, k L + l] = rbf_k(d_t) cos(l a_t); d_dist / d_ang
 * (optional) = sbf_features_partials (:77-95); invalid also flags angles outside [0, pi]. */
int egn_sbf_features(const double* in_edge_distances, const double* angles, int64_t n, int k_rbf, int l_sbf,
                     double cutoff, double* out, double* d_dist, double* d_ang, int32_t* invalid,
                     egn_stream_t stream);
/* geometry_grads (egn/gradients.py:33-36): distance gradients -u / +u per edge [E, 3] and the
 * closed-form angle gradients at k, j, i per triplet [N_t, 3] (egn/graph.py:173-203; zero for
 * collinear triplets, |v1 x v2| <= 1e-14).  Indices int64 as in GraphTopology. */
int egn_geometry_grads(const double* pos, const int64_t* src, const int64_t* recv, int64_t num_edges,
                       const int64_t* trip_in, const int64_t* trip_out, int64_t num_triplets, double* dist_d_src,
                       double* dist_d_recv, double* angle_d_k, double* angle_d_j, double* angle_d_i,
                       egn_stream_t stream);

/* ------------------------------------------------------------------ */
/* Optimizer: train_simple SGD update (tasks.py:207-208)               */
/* ------------------------------------------------------------------ */
/* Loss of one step and its seeds (reference egn/tasks.py:166-176, per sample, fp64):
 * d_energy[g] = 2 w_e (E_g - E*_g) / n, d_forces[v] = 2 w_f (F_v - F*_v) / (n count_v),
 * loss[0] = (sum_g w_e (E_g - E*_g)^2 + w_f sum_v |F_v - F*_v|^2 / count_v) / n.
 * forces == NULL: energy terms only.  One launch; seeds are written as fp32. */
int egn_loss_seeds(const float* energy, const double* e_target, int64_t num_graphs, const float* forces,
                   const double* f_target, const double* atom_count, int64_t num_nodes, double w_energy,
                   double w_forces, double n, double* loss, float* d_energy, float* d_forces, egn_stream_t stream);
int egn_sgd(float* w, const float* g, int64_t n, float lr, egn_stream_t stream);
/* Device utilities of the training step (no framework elementwise kernels on the path):
 * egn_zero: bytes of zeros (cudaMemsetAsync); egn_hadamard: out = a * b elementwise
 * (16-byte aligned); egn_transpose: out[c][r] = in[r][c] (row strides ld_in, ld_out);
 * egn_csr_ptr: ptr[v] = lower_bound(keys, v) for v in [0, nv] over keys sorted ascending
 * (the CSR offsets of a sorted user edge list, egn/graph.py:106-139's enumerate_triplets input). */
int egn_zero(void* ptr, int64_t bytes, egn_stream_t stream);
int egn_hadamard(const float* a, const float* b, float* out, int64_t n, egn_stream_t stream);
int egn_transpose(const float* in, int64_t rows, int64_t cols, int64_t ld_in, float* out, int64_t ld_out,
                  egn_stream_t stream);
int egn_csr_ptr(const int64_t* keys, int64_t n, int64_t nv, int64_t* ptr, egn_stream_t stream);
/* AdamW step t >= 1 over a flat parameter buffer (the
 * reference documents it only): decoupled weight decay, bias-corrected first / second moments
 * m, v (caller-owned, zero before step 1), torch.optim.AdamW's update order. */
int egn_adamw(float* w, const float* g, float* m, float* v, int64_t n, float lr, float beta1, float beta2,
              float eps, float weight_decay, int64_t step, egn_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* EGN_B200_H */
