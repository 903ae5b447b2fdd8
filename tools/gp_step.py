"""Graph-parallel training step of the bench batch with P in-process ranks on one GPU (ThreadComm),
for launch lists: which kernels the centre / reference schedules launch per forward+backward.

    python tools/gp_step.py [--workload gemnet-t-oc20] [--workers 2] [--schedule centre] [--steps 1]

Only for kernel inventories (ncu --metrics gpu__time_duration.sum): the ranks share one GPU, so
times are not a multi-GPU measurement.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gemnet-t-oc20")
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--schedule", default="centre", choices=["centre", "reference"])
    ap.add_argument("--graphs", type=int, default=8)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    from dataclasses import replace

    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.runtime import WorkerGroup

    wl = bench.WORKLOADS[args.workload]
    cfg = replace(bench._config(wl), workers=args.workers)
    systems = bench._systems(wl, args.graphs)
    params = init_params(cfg)
    wg = WorkerGroup(systems, params, schedule=args.schedule)
    df = np.zeros((wg.bg.num_nodes, 3)) if cfg.variant == "gemnet-style" else None
    for _ in range(2 + args.steps):
        res, _ = wg.forward_backward(1.0, df)
    torch.cuda.synchronize()
    print(f"ok energy[0]={float(np.asarray(res.energy).ravel()[0]):.6g} E={wg.bg.num_edges} "
          f"stages={sorted(res.stage_seconds)}")


if __name__ == "__main__":
    main()
