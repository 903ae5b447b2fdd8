"""Parity at exactly the configurations bench.py times (VERDICT r1 "Next" 1).

The bench step is GemNet-T C2 (BASELINE configs[1]): 32 graphs x 80 atoms, dims
128/64/64, 4 blocks, loss w_E = w_F = 1 against teacher targets, run by
``Trainer(cuda_graph=True)`` -- captured step, three-stream schedule, tcgen05 3xTF32
GEMMs at M = 58,644 edges.  Here that same Trainer (same systems, same weights, same
targets) is replayed and its loss, every parameter gradient and the position gradient
are compared with the fp64 oracle's per-graph loop (egn/tasks.py:131-185 restated in
oracle.loss_and_grads; egn/engine.py:320-438 for the backward).

DimeNet++ C1 (BASELINE configs[0], ``--workload dimenet-pp-small``): 4 graphs x 64
atoms, energy loss; checked on both GEMM paths (its 5.3k-edge batch runs the SIMT GEMM
by default, the tcgen05 GEMM when the SIMT threshold is forced to 0).

Tolerance (north star): per tensor max|a-b| / max|b| <= 1e-4.
"""

import numpy as np
import pytest
import torch

import bench
from conftest import TOL, max_rel
from oracle import egn_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_loss_grads(cfg, params, systems, e_t, f_t, w_e, w_f):
    """Per-graph fp64 loop: loss, summed parameter gradients and the position gradient of
    every graph (the seeds of tasks.py:166-176)."""
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    n = len(systems)
    total = 0.0
    grads = {k: np.zeros_like(v) for k, v in params.arrays.items()}
    dpos, energies = [], []
    off = 0
    for i, s in enumerate(systems):
        fw = O.forward(oc, params.arrays, s.positions, s.atomic_numbers)
        na = s.positions.shape[0]
        res = fw.energy - e_t[i]
        total += w_e * res * res / n
        d_f = None
        if w_f:
            delta = fw.forces - f_t[off:off + na]
            total += w_f * float((delta * delta).sum()) / na / n
            d_f = 2.0 * w_f * delta / (n * na)
        G, dp = O.backward(fw, params.arrays, 2.0 * w_e * res / n, d_f)
        for k in grads:
            grads[k] += G[k]
        dpos.append(dp)
        energies.append(fw.energy)
        off += na
    return total, grads, np.concatenate(dpos), np.asarray(energies)


def _bench_setup(workload):
    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch

    wl = bench.WORKLOADS[workload]
    cfg = bench._config(wl)
    systems = bench._systems(wl, wl["graphs"])
    params = init_params(cfg)
    bg = build_batch(systems, cfg.cutoff)
    teacher = Engine(DeviceWeights.from_params(init_params(cfg.replace(seed=1))))
    tf = teacher.forward(bg)
    e_t = tf.energy.double().cpu().numpy()
    f_t = tf.forces.double().cpu().numpy() if wl["w_forces"] else None
    return wl, cfg, systems, params, bg, e_t, f_t


def _check(tr, cfg, systems, params, e_t, f_t, w_f, loss):
    from paper_2203_09697_b200.tasks import _seeds

    grads = tr.weights.to_numpy(grads=True)
    # the position gradient of the same seeds (eager forward + backward on the same engine)
    fw = tr.engine.forward(tr.bg)
    _, d_e, d_f = _seeds(fw.energy, fw.forces, tr.e_target, tr.f_target, tr.atom_count, tr.w_energy,
                         tr.w_forces, tr.n)
    pos_bar = tr.engine.backward(tr.bg, fw, d_e, d_f).cpu().numpy()
    ref_loss, ref_g, ref_dp, ref_e = _oracle_loss_grads(cfg, params, systems, e_t, f_t, 1.0, w_f)
    assert abs(loss - ref_loss) <= TOL * abs(ref_loss)
    assert max_rel(fw.energy.double().cpu().numpy(), ref_e) < TOL
    assert max_rel(pos_bar, ref_dp) < TOL
    worst = max((max_rel(grads[k], ref_g[k]), k) for k in ref_g)
    assert worst[0] < TOL, worst


def test_gemnet_c2_bench_step_matches_oracle():
    """The exact bench step: captured Trainer, side streams, tcgen05 GEMMs at M = 58,644."""
    from paper_2203_09697_b200 import _lib
    from paper_2203_09697_b200.tasks import Trainer

    wl, cfg, systems, params, bg, e_t, f_t = _bench_setup("gemnet-t-oc20")
    assert bg.num_edges > 16384 > 8192  # side streams on, every edge product on tcgen05
    assert _lib.call("egn_gemm_simt_max_m", -1) <= 8192 < bg.num_edges
    tr = Trainer(params, None, e_t, f_t, 1.0, wl["w_forces"], graph=bg, cuda_graph=True)
    tr.step(0.0)  # eager step + capture
    assert tr._graph is not None, "the bench step must be the captured graph"
    loss = float(tr.step(0.0))  # replay of the captured step (lr 0: weights unchanged)
    _check(tr, cfg, systems, params, e_t, f_t, wl["w_forces"], loss)


@pytest.mark.parametrize("gemm_path", ["default", "tcgen05"])
def test_dimenet_c1_bench_step_matches_oracle(gemm_path):
    from paper_2203_09697_b200 import _lib
    from paper_2203_09697_b200.tasks import Trainer

    wl, cfg, systems, params, bg, e_t, f_t = _bench_setup("dimenet-pp-small")
    old = _lib.call("egn_gemm_simt_max_m", 0 if gemm_path == "tcgen05" else -1)  # -1: query only
    try:
        tr = Trainer(params, None, e_t, None, 1.0, 0.0, graph=bg, cuda_graph=True)
        tr.step(0.0)
        loss = float(tr.step(0.0))
        _check(tr, cfg, systems, params, e_t, None, 0.0, loss)
    finally:
        _lib.call("egn_gemm_simt_max_m", old)


@pytest.mark.parametrize("args", [["--workload", "dimenet-pp-small"],
                                  ["--workload", "dimenet-pp-small", "--basis", "bessel"]])
def test_bench_line_contract(args):
    """bench.py's JSON line (the driver's contract): metric, value, e2e with its copy sizes,
    gpu_launches, roofline with its bound / achieved / peak / frac, clocks, config naming the
    workload (and the basis when it is not the reference's)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), *args, "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=str(root))
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    assert line["higher_is_better"] is True and line["scaling"] == "weak" and line["dtype"] == "f32"
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 100
    roof = line["roofline"]
    assert roof["bound"] in ("hbm", "tensor") and 0 < roof["frac"] <= 1.2 and roof["peak"] > 0
    assert line["config"]["workload"] == "dimenet-pp-small"
    assert ("basis" in line["config"]) == ("bessel" in args)
    assert "sm_mhz" in line["clocks"]
