"""C5 triplet-kernel sweep: one 1000-atom graph whose density is
tuned for a mean degree in {32, 64, 128, 256, 500}, d_g in {64, 128, 256}, K=6, L=7.

For each point it reports:
* the edge and triplet counts and the maximum degree;
* forward and backward kernel times (CUDA events, L2 flushed between launches);
* G triplets/s and FP32 TF/s;
* the HBM fraction of the algorithmic bytes B_fwd = 12 N_t + (8 d_g + 4) N_e and
  B_bwd = 16 N_t + (12 d_g + 8) N_e.

Under torchrun each rank takes a contiguous centre range balanced on deg(deg-1)
(partition_centers). It runs the kernels on its own centres only, with no exchange
(the triplet aggregation is rank-local), and the max over ranks is reported.

    python tools/c5_sweep.py [--degrees 32,64,128] [--dg 64,128] [--out profiles/r1_c5_sweep.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def cloud(n, deg, cutoff, seed):
    """Uniform random atoms in a cube sized for the target mean degree (bulk estimate)."""
    rho = (deg + 1) / (4.0 / 3.0 * np.pi * cutoff ** 3)
    side = (n / rho) ** (1.0 / 3.0)
    return np.random.default_rng(seed).uniform(0.0, side, size=(n, 3))


def time_it(fn, iters, flush):
    times = []
    for i in range(iters + 2):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i >= 2:
            times.append(s.elapsed_time(e) / 1000.0)
    return float(np.median(times))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--degrees", default="32,64,128,256,500")
    ap.add_argument("--dg", default="64,128,256")
    ap.add_argument("--atoms", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--path", default="auto", choices=["auto", "sh", "pairwise"],
                    help="triplet kernels: auto (pairwise <= deg 64, spherical-harmonic above), sh, pairwise")
    args = ap.parse_args()
    import torch.distributed as dist

    from paper_2203_09697_b200 import _lib, ops
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.partition import partition_centers

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
    if world > 1:
        dist.init_process_group(os.environ.get("EGN_DIST_BACKEND", "nccl"))
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    hbm = peaks["hbm_gbs"] * 1e9
    fp32 = 148 * 128 * 2 * 1.965e9
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    _lib.call("egn_triplet_path", {"auto": 0, "sh": 1, "pairwise": 2}[args.path])
    cutoff, K, L = 6.0, 6, 7
    rows = []
    for deg in [int(x) for x in args.degrees.split(",")]:
        pos = cloud(args.atoms, deg, cutoff, seed=deg)
        bg = build_batch([pos], cutoff)
        degs = bg.deg.cpu().numpy()
        part = partition_centers(degs, world)
        n0, n1, e0, e1, t0, t1 = part.rank(rank)
        ep_own = bg.edge_ptr[n0:n1 + 1]
        for dg in [int(x) for x in args.dg.split(",")]:
            g = torch.Generator(device="cuda").manual_seed(deg + dg)
            X = torch.randn((bg.num_edges, dg), device="cuda", generator=g)
            W = torch.randn((K, L, dg), device="cuda", generator=g) / np.sqrt(K * L)
            Sb = torch.randn((bg.num_edges, dg), device="cuda", generator=g)
            eg = torch.zeros((bg.num_edges, 4), device="cuda")
            Xb = torch.empty_like(X)
            Wb = torch.empty_like(W)
            md = int(degs.max())

            def fwd():
                ops.triplet_fwd(ep_own, bg.rev, bg.geo, X, W, cutoff, md)

            def bwd():
                ops.triplet_bwd(ep_own, bg.rev, bg.geo, X, W, cutoff, Sb, eg, X_bar=Xb, W_bar=Wb, max_degree=md)

            t_f = time_it(fwd, args.iters, flush)
            t_b = time_it(bwd, args.iters, flush)
            tt = torch.tensor([t_f, t_b], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_f, t_b = float(tt[0]), float(tt[1])
            ne, nt = bg.num_edges, bg.num_triplets
            b_f = 12 * nt + (8 * dg + 4) * ne
            b_b = 16 * nt + (12 * dg + 8) * ne
            flops = 2.0 * nt * L * dg
            # bytes the implicit-triplet kernels must move: X rows gathered + S written (+ geometry)
            b_impl_f = (8 * dg + 20) * ne
            b_impl_b = (16 * dg + 36) * ne  # S_bar, X read; X_bar written; geometry, edge_grad
            row = {"path": args.path, "target_deg": deg, "mean_deg": ne / args.atoms, "max_deg": md, "edges": ne,
                   "triplets": nt, "dg": dg, "gpus": world, "fwd_us": t_f * 1e6, "bwd_us": t_b * 1e6,
                   "fwd_hbm_frac_implicit": b_impl_f / t_f / hbm, "bwd_hbm_frac_implicit": b_impl_b / t_b / hbm,
                   "fwd_gtrip_s": nt / t_f / 1e9, "bwd_gtrip_s": nt / t_b / 1e9,
                   "fwd_fp32_frac": flops / t_f / fp32, "bwd_fp32_frac": 2 * flops / t_b / fp32,
                   "fwd_hbm_frac": b_f / t_f / hbm, "bwd_hbm_frac": b_b / t_b / hbm}
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
            del X, Sb, eg, Xb
        del bg
        torch.cuda.empty_cache()
    if rank == 0 and args.out:
        Path(args.out).write_text(json.dumps(rows, indent=1))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
