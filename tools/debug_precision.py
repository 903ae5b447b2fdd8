"""Model-level error vs the fp64 oracle with the tcgen05 GEMM path on / off (cuBLAS fp32 composite)."""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import egn_oracle as O  # noqa: E402
from paper_2203_09697_b200 import ModelConfig, init_params, ops  # noqa: E402
from paper_2203_09697_b200.engine import DeviceWeights, Engine  # noqa: E402
from paper_2203_09697_b200.graph import build_batch  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-8))


def run(tc: bool, variant):
    orig = ops._tc_ok
    if not tc:
        ops._tc_ok = lambda *a, **k: False
    try:
        cfg = ModelConfig(variant=variant, blocks=4, d_u=128, d_v=128, d_e=128, d_t=64, d_bil=64, k_rbf=6, l_sbf=7,
                          cutoff=6.0, seed=0)
        params = init_params(cfg)
        oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
        rng = np.random.default_rng(11)
        systems = [O.random_cloud(n, 0.06, rng) for n in (20, 33, 27)]
        eng = Engine(DeviceWeights.from_params(params))
        bg = build_batch([s[0] for s in systems], cfg.cutoff)
        fw = eng.forward(bg)
        d_e = torch.tensor([0.3, -1.1, 0.6], device="cuda")
        df_np = [rng.standard_normal((s[0].shape[0], 3)) for s in systems] if variant == "gemnet-style" else None
        df = torch.tensor(np.concatenate(df_np), device="cuda") if df_np else None
        eng.backward(bg, fw, d_e, df)
        grads = eng.weights.to_numpy(grads=True)
        ref = {k: np.zeros_like(v) for k, v in params.arrays.items()}
        es = []
        for i, (pos, z) in enumerate(systems):
            f = O.forward(oc, params.arrays, pos, z)
            G, _ = O.backward(f, params.arrays, float(d_e[i]), df_np[i] if df_np else None)
            es.append(f.energy)
            for k in ref:
                ref[k] += G[k]
        worst = sorted(((rel(grads[k], ref[k]), k) for k in ref), reverse=True)[:6]
        print(f"{variant} tc={tc} energy rel {rel(fw.energy.double().cpu().numpy(), np.array(es)):.2e} worst grads:",
              [(k, f'{e:.1e}') for e, k in worst])
    finally:
        ops._tc_ok = orig


for v in ("gemnet-style", "dimenet-style"):
    run(True, v)
    run(False, v)
