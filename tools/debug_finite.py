"""Check every intermediate of the bench workload's training step for non-finite values."""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def report(name, t):
    if t is None:
        return
    bad = (~torch.isfinite(t)).sum().item()
    print(f"{name:28s} shape={tuple(t.shape)} nonfinite={bad} absmax={t.abs().max().item() if t.numel() else 0:.3e}")


def main():
    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    wl = bench.WORKLOADS["gemnet-t-oc20"]
    cfg = bench._config(wl)
    systems = bench._systems(wl, 32)
    bg = build_batch(systems, cfg.cutoff)
    print("E", bg.num_edges, "T", bg.num_triplets, "maxdeg", bg.max_deg,
          "min deg", int(bg.deg.min()), "isolated", int((bg.deg == 0).sum()))
    report("geo", bg.geo)
    eng = Engine(DeviceWeights.from_params(init_params(cfg)))
    fw = eng.forward(bg)
    for b, st in enumerate(fw.blocks):
        for k, v in st.items():
            report(f"block{b}.{k}", v)
    report("energy", fw.energy)
    report("forces", fw.forces)
    pb = eng.backward(bg, fw, torch.ones(bg.num_graphs, device="cuda"), torch.ones_like(fw.forces))
    report("pos_bar", pb)
    g = eng.weights.to_numpy(grads=True)
    for k, v in g.items():
        if not np.all(np.isfinite(v)):
            print("NONFINITE grad", k)


if __name__ == "__main__":
    main()
