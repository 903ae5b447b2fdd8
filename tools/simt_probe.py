"""Warm device time of the node-sized products (M = 2560) alone: gemm (both B layouts,
resid epilogue) and gemm_wgrad, 200 calls captured in one CUDA graph.

    EGN_GEMM_PANEL=0|1 python tools/simt_probe.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2203_09697_b200 import ops  # noqa: E402


def timed(fn, reps=200):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1000 / reps


def sweep():
    """M x N x K grid of plain products (EGN_GEMM_PANEL selects the kernel)."""
    for M in (256, 1280, 2560, 5120):
        for N, K in ((128, 32), (128, 128), (64, 128), (128, 256)):
            a = torch.randn(M, K, device="cuda")
            w = torch.randn(N, K, device="cuda")
            out = torch.empty(M, N, device="cuda")
            print(f"M={M:5d} N={N:3d} K={K:3d}  {timed(lambda: ops.gemm(a, w, out=out)):6.2f} us")


if __name__ == "__main__" and os.environ.get("SWEEP"):
    sweep()
    sys.exit(0)

torch.manual_seed(0)
M = int(os.environ.get("M", "2560"))
a = torch.randn(M, 128, device="cuda")
w = torch.randn(128, 128, device="cuda")
r = torch.randn(M, 128, device="cuda")
a2 = torch.randn(M, 64, device="cuda")
w2 = torch.randn(128, 64, device="cuda")
out = torch.empty(M, 128, device="cuda")
tag = "panel=" + os.environ.get("EGN_GEMM_PANEL", "1")
small = torch.empty(1024, device="cuda")
print(tag, "floor (1 KB fill) %.2f us" % timed(lambda: small.fill_(1.0)))
print(tag, "warm-up long run %.2f us" % timed(lambda: ops.gemm(a, w, out=out), reps=5000))
print(tag, "gemm          %.2f us" % timed(lambda: ops.gemm(a, w, out=out)))
print(tag, "gemm Bmn resid %.2f us" % timed(lambda: ops.gemm(a, w, resid=r, out=out, b_mn=True)))
print(tag, "gemm K=128+64 %.2f us" % timed(lambda: ops.gemm(a, w, a2=a2, b2=w2, out=out)))
wo = torch.empty(128, 128, device="cuda")
cs = torch.empty(128, device="cuda")
print(tag, "wgrad colsum  %.2f us" % timed(lambda: ops.gemm_wgrad(a, r, out=wo, colsum=cs)))
ref = a.double() @ w.double().t()
print(tag, "max err", (ops.gemm(a, w) - ref).abs().max().item())
