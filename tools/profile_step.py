"""Per-kernel device-time breakdown of the bench training step (torch.profiler / CUPTI).

    python tools/profile_step.py [--workload gemnet-t-oc20] [--steps 3] [--out gpurun_out/step_kernels.txt]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gemnet-t-oc20")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--graphs", type=int, default=None)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "step_kernels.txt"))
    ap.add_argument("--plain", action="store_true", help="run the steps without torch.profiler")
    ap.add_argument("--basis", default="gaussian")
    args = ap.parse_args()
    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    wl = dict(bench.WORKLOADS[args.workload], basis=args.basis)
    cfg = bench._config(wl)
    systems = bench._systems(wl, args.graphs or wl["graphs"])
    bg = build_batch(systems, cfg.cutoff)
    import numpy as np

    e_t = np.zeros(bg.num_graphs)
    f_t = np.zeros((bg.num_nodes, 3)) if wl["w_forces"] else None
    tr = Trainer(init_params(cfg), None, e_t, f_t, 1.0, wl["w_forces"], graph=bg)
    for _ in range(3):
        tr.step(1e-6)
    torch.cuda.synchronize()
    if args.plain:  # no CUPTI subscriber (for ncu runs)
        for _ in range(args.steps):
            tr.step(1e-6)
        torch.cuda.synchronize()
        return
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            tr.step(1e-6)
        torch.cuda.synchronize()
    table = prof.key_averages().table(sort_by="cuda_time_total", row_limit=60, max_name_column_width=90)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(table)
    print(table)
    total = sum(e.device_time_total for e in prof.key_averages()) / args.steps
    print(f"device time per step (sum of kernels): {total / 1000:.3f} ms; E={bg.num_edges} T={bg.num_triplets}")


if __name__ == "__main__":
    main()
