"""tcgen05 3xTF32 GEMM with fused epilogues vs a float64 torch reference.

The dense layers of the model (linear, egn/tape.py:104-119) must be fp32-accurate:
tolerance 2e-6 relative to max|ref| (plain TF32 would be ~1e-3)."""

import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 2e-6


def _rel(a, b):
    return float((a.double() - b).abs().max() / max(b.abs().max().item(), 1e-30))


@pytest.fixture(params=["tcgen05", "simt"], autouse=True)
def gemm_path(request):
    """Run every product test on both paths: the tcgen05 3xTF32 GEMM and the small-M fp32
    SIMT GEMM (egn_gemm_simt_max_m threshold forced to 0 / infinity)."""
    from paper_2203_09697_b200 import _lib

    old = _lib.call("egn_gemm_simt_max_m", 0 if request.param == "tcgen05" else 1 << 40)
    yield request.param
    _lib.call("egn_gemm_simt_max_m", old)


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (1000, 64, 128), (4097, 128, 256), (300, 256, 64),
                                   (77, 384, 96), (2560, 16, 128), (58644, 128, 128), (5000, 1312, 640)])
def test_plain_gemm(M, N, K):
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn((M, K), device="cuda", generator=g)
    b = torch.randn((N, K), device="cuda", generator=g) / K ** 0.5
    out = ops.gemm(a, b)
    ref = a.double() @ b.double().t()
    assert _rel(out, ref) < TOL


def test_two_segments_and_epilogues():
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(0)
    M, N, K0, K1 = 3000, 128, 128, 128
    a0 = torch.randn((M, K0), device="cuda", generator=g)
    a1 = torch.randn((M, K1), device="cuda", generator=g)
    w = torch.randn((N, K0 + K1), device="cuda", generator=g) / 16
    bias = torch.randn(N, device="cuda", generator=g)
    resid = torch.randn((M, N), device="cuda", generator=g)
    # concat-free linear with bias and SiLU side output: h = [a0, a1] W^T + b, a = silu(h)
    h, act = ops.gemm(a0, w[:, :K0], a2=a1, b2=w[:, K0:], bias=bias, flags=ops.EPI_SILU_OUT2)
    ref = torch.cat([a0, a1], 1).double() @ w.double().t() + bias.double()
    assert _rel(h, ref) < TOL
    assert _rel(act, torch.nn.functional.silu(ref)) < 1e-5
    # residual
    out = ops.gemm(a0, w[:, :K0], bias=bias, resid=resid)
    assert _rel(out, a0.double() @ w[:, :K0].double().t() + bias.double() + resid.double()) < TOL
    # gathered-row add
    src = torch.randn((500, N), device="cuda", generator=g)
    idx = torch.randint(0, 500, (M,), device="cuda", generator=g, dtype=torch.int32)
    out = ops.gemm(a0, w[:, :K0], gather=(src, idx))
    assert _rel(out, a0.double() @ w[:, :K0].double().t() + src.double()[idx.long()]) < TOL
    # gate multiply with pre-gate side output
    aux = torch.randn((M, N), device="cuda", generator=g)
    y, z = ops.gemm(a0, w[:, :K0], aux=aux, flags=ops.EPI_MUL_AUX)
    zr = a0.double() @ w[:, :K0].double().t()
    assert _rel(z, zr) < TOL and _rel(y, zr * aux.double()) < TOL
    # SiLU backward
    out = ops.gemm(a0, w[:, :K0], aux=aux, flags=ops.EPI_DSILU_AUX)
    s = torch.sigmoid(aux.double())
    assert _rel(out, zr * s * (1 + aux.double() * (1 - s))) < 1e-5


@pytest.mark.parametrize("M,N,K", [(1000, 128, 64), (3001, 64, 128), (500, 256, 128), (77, 128, 256)])
def test_mn_major_b_dgrad(M, N, K):
    """a @ W with W [K, N] (the data gradient of a linear layer) without a transpose copy."""
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(M)
    a = torch.randn((M, K), device="cuda", generator=g)
    w = torch.randn((K, N), device="cuda", generator=g) / K ** 0.5
    aux = torch.randn((M, N), device="cuda", generator=g)
    out = ops.gemm(a, w, b_mn=True)
    assert _rel(out, a.double() @ w.double()) < TOL
    out = ops.gemm(a, w, b_mn=True, aux=aux, flags=ops.EPI_DSILU_AUX)
    s = torch.sigmoid(aux.double())
    assert _rel(out, (a.double() @ w.double()) * s * (1 + aux.double() * (1 - s))) < 1e-5


@pytest.mark.parametrize("R,M,N", [(58644, 128, 128), (58644, 64, 256), (1000, 128, 64), (37, 64, 64),
                                   (2560, 128, 128), (20000, 256, 128), (14792, 1312, 1312), (640, 1536, 2048)])
def test_wgrad_split_k(R, M, N):
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(R + M)
    gr = torch.randn((R, M), device="cuda", generator=g)
    x = torch.randn((R, N), device="cuda", generator=g)
    out = ops.gemm_wgrad(gr, x)
    ref = gr.double().t() @ x.double()
    assert _rel(out, ref) < TOL
    prev = torch.randn((M, N), device="cuda", generator=g)
    out2 = ops.gemm_wgrad(gr, x, out=prev.clone(), accumulate=True)
    assert _rel(out2, ref + prev.double()) < TOL
    # strided operand (a column block of a wider matrix)
    wide = torch.randn((R, 2 * N), device="cuda", generator=g)
    out3 = ops.gemm_wgrad(gr, wide[:, N:])
    assert _rel(out3, gr.double().t() @ wide[:, N:].double()) < TOL


def test_strided_operands_and_errors():
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(1)
    big = torch.randn((1000, 256), device="cuda", generator=g)
    w = torch.randn((64, 256), device="cuda", generator=g)
    out = ops.gemm(big[:, 128:], w[:, 128:])  # row stride 256, K = 128
    assert _rel(out, big[:, 128:].double() @ w[:, 128:].double().t()) < TOL
    with pytest.raises(ValueError):
        ops.gemm(torch.randn((10, 6), device="cuda"), torch.randn((16, 6), device="cuda"))  # K % 4
    with pytest.raises(ValueError):
        ops.gemm(torch.randn((10, 8), device="cuda"), torch.randn((12, 8), device="cuda"))  # N % 16


@pytest.mark.parametrize("R,M,N", [(58644, 128, 128), (1000, 64, 256), (77, 32, 16), (14792, 1312, 1312)])
def test_wgrad_fused_column_sums_and_strided_out(R, M, N):
    """egn_gemm_wgrad with g_colsum (bias adjoint from the same operand tiles) and a
    row-strided destination (a column block of a wider weight gradient)."""
    from paper_2203_09697_b200 import ops

    torch.manual_seed(R)
    gr = torch.randn((R, M), device="cuda")
    x = torch.randn((R, N), device="cuda")
    big = torch.full((M, N + 48), float("nan"), device="cuda")
    cs = torch.full((M,), float("nan"), device="cuda")
    ops.gemm_wgrad(gr, x, out=big[:, 16:16 + N], colsum=cs)
    ref = gr.double().t() @ x.double()
    assert _rel(big[:, 16:16 + N], ref) < TOL
    assert torch.isnan(big[:, :16]).all() and torch.isnan(big[:, 16 + N:]).all()
    assert _rel(cs, gr.double().sum(0)) < TOL
    prev = cs.clone()
    ops.gemm_wgrad(gr, x, out=big[:, 16:16 + N], colsum=cs, accumulate=True)
    assert _rel(cs, prev.double() + gr.double().sum(0)) < TOL


@pytest.mark.parametrize("scale", ["small", "xl"])
def test_small_gemms_batched_all_layouts(scale):
    """egn_small_gemm_batched (the weight-sized folds of the backward) for every transpose
    combination in one batch; 'xl' sizes select the 64 x 64 register-blocked kernel."""
    from paper_2203_09697_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(7)
    dims = [(64, 128, 96), (37, 70, 129)] if scale == "small" else [(2048, 256, 2048), (1312, 288, 1312)]
    probs, refs = [], []
    for m, n, k in dims:
        for ta in (0, 1):
            for tb in (0, 1):
                for tc in (0, 1):
                    A = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
                    B = torch.randn((n, k) if tb else (k, n), device="cuda", generator=g)
                    C = torch.empty((n, m) if tc else (m, n), device="cuda")
                    ref = (A.double().t() if ta else A.double()) @ (B.double().t() if tb else B.double())
                    probs.append((A, B, C, ta, tb, tc))
                    refs.append(ref.t() if tc else ref)
    ops.small_gemms(probs)
    torch.cuda.synchronize()
    for (A, B, C, ta, tb, tc), ref in zip(probs, refs):
        # plain fp32 FMA chains of length K (up to 2048): ~sqrt(K) ulp, not the 3xTF32 bound
        assert _rel(C, ref) < 1e-5, (A.shape, B.shape, ta, tb, tc)


@pytest.mark.parametrize("M,N,K,b_mn,two", [(8192, 128, 128, False, False), (8192, 128, 128, True, False),
                                            (9000, 64, 192, False, False), (8192, 128, 64, False, True),
                                            (5000, 1312, 640, False, False), (6000, 256, 512, True, False)])
def test_gemm_precomputed_b_lo_bit_identical(M, N, K, b_mn, two):
    """egn_gemm_blo (B's tf32 lo parts from egn_tf32_lo, loaded by TMA) gives exactly the
    products of egn_gemm (lo parts formed by the split warps)."""
    from paper_2203_09697_b200 import ops

    torch.manual_seed(M + N + K)
    a = torch.randn((M, K), device="cuda")
    full = torch.randn((K + 64, N + 32) if b_mn else (N + 32, K + 64), device="cuda")
    b = full[:K, :N] if b_mn else full[:N, :K]  # row-strided weight view
    lo_full = torch.empty_like(full)
    ops.call("egn_tf32_lo", ops.ptr(full), full.shape[0], full.shape[1], full.stride(0), ops.ptr(lo_full),
             lo_full.stride(0), ops.stream())
    b_lo = lo_full[:K, :N] if b_mn else lo_full[:N, :K]
    kw = {}
    if two:
        a2 = torch.randn((M, 32), device="cuda")
        b2 = torch.randn((N, 32), device="cuda")
        b2_lo = torch.empty_like(b2)
        ops.call("egn_tf32_lo", ops.ptr(b2), N, 32, 32, ops.ptr(b2_lo), 32, ops.stream())
        kw = dict(a2=a2, b2=b2)
    resid = torch.randn((M, N), device="cuda")
    ref = ops.gemm(a, b, resid=resid, b_mn=b_mn, **kw)
    got = ops.gemm(a, b, resid=resid, b_mn=b_mn, b_lo=b_lo, b2_lo=b2_lo if two else None, **kw)
    torch.cuda.synchronize()
    assert torch.equal(ref, got)
