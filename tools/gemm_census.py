"""Every tcgen05 GEMM call of one bench training step, timed one by one.

Records the (M, N, K, segments, epilogue, operand layout) of each ops.gemm /
ops.gemm_wgrad call in a step, then replays each call alone in a CUDA graph with
an L2 flush (256 MB write) between repetitions and subtracts the flush time, so
every figure is a cold-L2 device time.  Prints per call: us, algorithmic bytes
(operands read once + outputs written once) and the implied GB/s.

    python tools/gemm_census.py [--workload gemnet-t-oc20] [--out gpurun_out/gemm_census.txt]
"""

from __future__ import annotations

import argparse
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2203_09697_b200 import ops  # noqa: E402


def _bytes(t):
    return 0 if t is None else t.shape[0] * (t.shape[1] if t.dim() > 1 else 1) * 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gemnet-t-oc20")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "gemm_census.txt"))
    args = ap.parse_args()
    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    wl = bench.WORKLOADS[args.workload]
    cfg = bench._config(wl)
    bg = build_batch(bench._systems(wl, wl["graphs"]), cfg.cutoff)
    e_t = np.zeros(bg.num_graphs)
    f_t = np.zeros((bg.num_nodes, 3)) if wl["w_forces"] else None
    tr = Trainer(init_params(cfg), None, e_t, f_t, 1.0, wl["w_forces"], graph=bg, cuda_graph=False)
    tr.step(1e-6)
    torch.cuda.synchronize()

    calls = []
    g0, w0 = ops.gemm, ops.gemm_wgrad

    def gemm_hook(a, b, *x, **kw):
        out = g0(a, b, *x, **kw)
        kw2 = dict(kw)
        calls.append(("gemm", (a, b) + x, kw2, out))
        return out

    def wgrad_hook(g, x, *y, **kw):
        out = w0(g, x, *y, **kw)
        calls.append(("wgrad", (g, x) + y, dict(kw), out))
        return out

    ops.gemm, ops.gemm_wgrad = gemm_hook, wgrad_hook
    tr.step(1e-6)
    torch.cuda.synchronize()
    ops.gemm, ops.gemm_wgrad = g0, w0

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(args.reps):
                    flush.zero_()
                    fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay()
        torch.cuda.synchronize()
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1000 / args.reps

    t_flush = timed(lambda: None)
    rows, agg = [], defaultdict(lambda: [0, 0.0, 0])
    for kind, a, kw, out in calls:
        if kind == "gemm":
            A, B = a[0], a[1]
            M, K = A.shape
            b_mn = kw.get("b_mn", False)
            N = B.shape[1] if b_mn else B.shape[0]
            a2 = kw.get("a2")
            flags = kw.get("flags", 0)
            desc = (f"gemm M={M} N={N} K={K}" + (f"+{a2.shape[1]}" if a2 is not None else "") +
                    (" Bmn" if b_mn else "") + (" bias" if kw.get("bias") is not None else "") +
                    (" resid" if kw.get("resid") is not None else "") +
                    (" gather" if kw.get("gather") is not None else "") +
                    (" aux" if kw.get("aux") is not None else "") + f" f={flags}")
            outs = out if isinstance(out, tuple) else (out,)
            byt = _bytes(A) + _bytes(B) + _bytes(a2) + _bytes(kw.get("b2")) + _bytes(kw.get("resid")) + \
                _bytes(kw.get("aux")) + sum(_bytes(o) for o in outs)
            if kw.get("gather") is not None:
                byt += M * N * 4
            fn = lambda a=a, kw=kw: g0(*a, **kw)  # noqa: E731
        else:
            G, X = a[0], a[1]
            desc = f"wgrad R={G.shape[0]} M={G.shape[1]} N={X.shape[1]}" + (" colsum" if kw.get("colsum") is not None else "")
            byt = _bytes(G) + _bytes(X) + G.shape[1] * X.shape[1] * 4
            fn = lambda a=a, kw=kw: w0(*a, **kw)  # noqa: E731
        us = timed(fn) - t_flush
        rows.append((desc, us, byt))
        agg[desc][0] += 1
        agg[desc][1] += us
        agg[desc][2] = byt
    lines = [f"GEMM census: {len(rows)} calls per step, cold-L2 device time (flush {t_flush:.1f} us subtracted)",
             f"{'call':62s} {'n':>3s} {'us/call':>8s} {'MB':>7s} {'GB/s':>7s} {'us total':>9s}"]
    for desc, (n, us, byt) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{desc:62s} {n:3d} {us / n:8.1f} {byt / 1e6:7.1f} {byt / (us / n) / 1e3:7.0f} {us:9.1f}")
    tot_us = sum(r[1] for r in rows)
    tot_b = sum(r[2] for r in rows)
    lines.append(f"total {tot_us:.1f} us per step, {tot_b / 1e6:.1f} MB algorithmic, {tot_b / tot_us / 1e3:.0f} GB/s")
    text = "\n".join(lines)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
