"""Structure relaxation: GPU relax() with the neighbour graph rebuilt on
the device at every evaluation, timed per evaluation, beside the fp64 oracle's predict.

    python tools/relax_bench.py [--atoms 80] [--steps 50]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--atoms", type=int, default=80)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--variant", default="gemnet-style")
    a = ap.parse_args()
    from oracle import egn_oracle as O
    from paper_2203_09697_b200 import ModelConfig, init_params, random_cloud
    from paper_2203_09697_b200.tasks import relax

    cfg = ModelConfig(variant=a.variant, blocks=4, d_u=128, d_v=128, d_e=128, d_t=64, d_bil=64, k_rbf=6, l_sbf=7,
                      cutoff=6.0, seed=0)
    params = init_params(cfg)
    system = random_cloud(a.atoms, 0.06, np.random.default_rng(0))
    relax(system, params, 1e-12, max_steps=3, step_size=1e-3)  # warm-up (library load, workspaces)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = relax(system, params, 1e-12, max_steps=a.steps, step_size=1e-3)
    torch.cuda.synchronize()
    gpu_s = (time.perf_counter() - t0) / (res.steps + 1)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    P = O.init_params(oc)
    t0 = time.perf_counter()
    for _ in range(2):
        O.predict(oc, P, system.positions, system.atomic_numbers)
    cpu_s = (time.perf_counter() - t0) / 2
    out = {"atoms": a.atoms, "variant": a.variant, "evaluations": res.steps + 1,
           "gpu_ms_per_evaluation": gpu_s * 1e3, "oracle_ms_per_evaluation": cpu_s * 1e3,
           "speedup": cpu_s / gpu_s, "final_energy": res.energies[-1], "final_fmax": res.max_forces[-1]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
