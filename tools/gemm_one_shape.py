"""Cold-L2 device time of one GEMM shape (for A/B experiments with env switches).

    EGN_GEMM_FLUSH_SHORT=4 python tools/gemm_one_shape.py [M N K] [--kind fwd|dgrad|wgrad]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2203_09697_b200 import ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", nargs="*", type=int, default=[58644, 128, 128])
    ap.add_argument("--kind", default="fwd")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    M, N, K = a.shape
    torch.manual_seed(0)
    A = torch.randn((M, K), device="cuda")
    W = torch.randn((N, K), device="cuda")
    R = torch.randn((M, N), device="cuda")
    G = torch.randn((M, N), device="cuda")
    Wt = torch.randn((K, N), device="cuda")
    # the weight's tf32 lo parts precomputed, as in the model's products (egn_gemm_blo); EGN_GEMM_BLO=0: split warps
    W_lo = Wt_lo = None
    if os.environ.get("EGN_GEMM_BLO", "1") != "0":
        W_lo, Wt_lo = torch.empty_like(W), torch.empty_like(Wt)
        for src, dst in ((W, W_lo), (Wt, Wt_lo)):
            ops.call("egn_tf32_lo", ops.ptr(src), src.shape[0], src.shape[1], src.shape[1], ops.ptr(dst), dst.shape[1],
                     ops.stream())
    fn = {"fwd": lambda: ops.gemm(A, W, resid=R, b_lo=W_lo), "dgrad": lambda: ops.gemm(A, Wt, b_mn=True, b_lo=Wt_lo),
          "wgrad": lambda: ops.gemm_wgrad(G, A), "copy": lambda: R.copy_(G),
          "copy3": lambda: torch.add(G, R, out=A if K == N else R)}[a.kind]
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    x = torch.randn((4096, 4096), device="cuda")
    for _ in range(50):
        x = (x @ x).tanh_()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()

    def graph(body):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(a.reps):
                    flush.zero_()
                    body()
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1000 / a.reps

    t0 = graph(lambda: None)
    t1 = graph(fn)
    print(f"{a.kind} M={M} N={N} K={K}: {t1 - t0:.1f} us (flush {t0:.1f})")


if __name__ == "__main__":
    main()
