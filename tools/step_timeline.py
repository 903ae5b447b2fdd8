"""Per-stream device timeline of the bench training step (torch.profiler / CUPTI kernel events).

    python tools/step_timeline.py [--workload gemnet-t-oc20] [--steps 3] [--eager]

Prints, per CUDA stream: kernels and busy time per step and the idle time between the
stream's own kernels (waiting on another stream or on the host), then each stream's top
kernels.  Default: CUDA-graph replay of the step, as bench.py times it.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gemnet-t-oc20")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--basis", default="gaussian")
    args = ap.parse_args()
    from torch.profiler import ProfilerActivity, profile

    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    wl = dict(bench.WORKLOADS[args.workload], basis=args.basis)
    cfg = bench._config(wl)
    systems = bench._systems(wl, wl["graphs"])
    bg = build_batch(systems, cfg.cutoff)
    e_t = np.zeros(bg.num_graphs)
    f_t = np.zeros((bg.num_nodes, 3)) if wl["w_forces"] else None
    tr = Trainer(init_params(cfg), None, e_t, f_t, 1.0, wl["w_forces"], graph=bg, cuda_graph=not args.eager)
    for _ in range(3):
        tr.step(1e-6)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            tr.step(1e-6)
        torch.cuda.synchronize()
    ev = [e for e in prof.events()
          if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0
          and "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
    by_stream = defaultdict(list)
    for e in ev:
        by_stream[getattr(e, "device_resource_id", 0)].append(e)
    t0 = min(e.time_range.start for e in ev)
    t1 = max(e.time_range.end for e in ev)
    print(f"span per step {(t1 - t0) / args.steps:.1f} us over {args.steps} steps; E={bg.num_edges}")
    # device occupancy: time with >= 1 kernel running, and with >= 2
    pts = sorted([(e.time_range.start, 1) for e in ev] + [(e.time_range.end, -1) for e in ev])
    level, last, cover = 0, None, defaultdict(float)
    for t, d in pts:
        if last is not None and level > 0:
            cover[min(level, 3)] += t - last
        level += d
        last = t
    print("time with 1 / 2 / >=3 kernels running per step: " +
          " / ".join(f"{cover[i] / args.steps:.1f}" for i in (1, 2, 3)) + " us")
    if not args.eager:
        return
    for sid, es in sorted(by_stream.items(), key=lambda kv: -len(kv[1])):
        es.sort(key=lambda e: e.time_range.start)
        busy = sum(e.time_range.elapsed_us() for e in es) / args.steps
        gaps = sum(max(0, b.time_range.start - a.time_range.end) for a, b in zip(es, es[1:])) / args.steps
        print(f"stream {sid}: {len(es) / args.steps:.0f} kernels/step, busy {busy:.1f} us/step, idle between "
              f"own kernels {gaps:.1f} us/step")
        tot = defaultdict(float)
        for e in es:
            tot[e.name.split("(")[0][:80]] += e.time_range.elapsed_us() / args.steps
        for k in sorted(tot, key=lambda k: -tot[k])[:14]:
            print(f"    {tot[k]:8.1f}  {k}")


if __name__ == "__main__":
    main()
