"""Graph-parallel runtime on one GPU: P in-process ranks vs the single-rank engine
and vs the fp64 oracle (egn/runtime.py parallel == sequential, tests/test_runtime.py:115-175)."""

import numpy as np
import pytest
import torch

from conftest import TOL, max_rel
from oracle import egn_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["default", "tcgen05"], autouse=True)
def gemm_path(request, monkeypatch):
    """Every model test runs twice: the default dispatch (node-row and small products on the
    SIMT GEMM, one stream below EGN_SIDE_MIN_EDGES edges) and with every product forced onto
    the tcgen05 3xTF32 GEMM (egn_gemm_simt_max_m = 0) and the three-stream schedule forced on
    (EGN_SIDE_MIN_EDGES = 0) -- the code path the bench step runs at M = 58,644."""
    from paper_2203_09697_b200 import _lib

    if request.param == "default":
        yield request.param
        return
    monkeypatch.setenv("EGN_SIDE_MIN_EDGES", "0")
    old = _lib.call("egn_gemm_simt_max_m", 0)
    try:
        yield request.param
    finally:
        _lib.call("egn_gemm_simt_max_m", old)


def _case(variant, n=40, seed=3):
    from paper_2203_09697_b200 import ModelConfig, init_params

    cfg = ModelConfig(variant=variant, blocks=3, d_u=16, d_v=24, d_e=32, d_t=32, d_bil=32, k_rbf=6, l_sbf=7,
                      cutoff=6.0, seed=seed)
    pos, z = O.random_cloud(n, 0.06, np.random.default_rng(seed))
    return cfg, init_params(cfg), pos, z


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
@pytest.mark.parametrize("workers", [1, 2, 3, 4])
def test_parallel_matches_oracle(variant, workers):
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, z = _case(variant)
    run = ModelParams(cfg.replace(workers=workers), params.arrays)
    rng = np.random.default_rng(5)
    df = rng.standard_normal((pos.shape[0], 3)) if variant == "gemnet-style" else None
    res, bundle = WorkerGroup(pos, run).forward_backward(d_energy=0.8, d_forces=df)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    fw = O.forward(oc, params.arrays, pos, z)
    G, dpos = O.backward(fw, params.arrays, 0.8, df)
    assert abs(res.energy - fw.energy) <= TOL * max(1.0, abs(fw.energy))
    if variant == "gemnet-style":
        assert max_rel(res.forces, fw.forces) < TOL
    assert max_rel(bundle.d_positions, dpos) < TOL
    for k, g in G.items():
        assert max_rel(bundle.d_params[k], g) < TOL, k


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_parallel_equals_single_rank_engine(variant):
    """P = 1, 2, 4 agree with each other to fp32 summation-order noise."""
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, _ = _case(variant, n=60, seed=7)
    outs = {}
    for p in (1, 2, 4):
        run = ModelParams(cfg.replace(workers=p), params.arrays)
        outs[p] = WorkerGroup(pos, run).forward_backward(d_energy=1.0)
    r1, b1 = outs[1]
    for p in (2, 4):
        rp, bp = outs[p]
        assert abs(rp.energy - r1.energy) <= 1e-5 * max(1.0, abs(r1.energy))
        assert max_rel(bp.d_positions, b1.d_positions) < 1e-5
        for k in b1.d_params:
            assert max_rel(bp.d_params[k], b1.d_params[k]) < 1e-5, k


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_comm_volume_independent_of_triplets(variant):
    """Forward exchange per block: N_e d_e + G d_v (+ N_e d_e + N_v d_v for gemnet); no triplet level."""
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, _ = _case(variant)
    for d_t in (16, 48):
        c2 = cfg.replace(workers=3, d_t=d_t)
        from paper_2203_09697_b200 import init_params

        wg = WorkerGroup(pos, init_params(c2))
        res = wg.forward()
        ne, nv = wg.bg.num_edges, wg.bg.num_nodes
        expect = ne * c2.d_e + c2.d_v
        if variant == "gemnet-style":
            expect += ne * c2.d_e + nv * c2.d_v
        assert res.comm_log.forward_blocks() == {b: expect for b in range(c2.blocks)}
        assert "triplet" not in res.comm_log.levels()


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_graph_aligned_partition_is_halo_free_and_exact(variant):
    """A batch split at graph boundaries needs no edge/node exchange; results equal the
    single-rank engine over the same batch."""
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, _, _ = _case(variant)
    rng = np.random.default_rng(21)
    systems = [O.random_cloud(n, 0.06, rng)[0] for n in (30, 41, 25, 37)]
    wg = WorkerGroup(systems, ModelParams(cfg.replace(workers=2), params.arrays), align_graphs=True)
    de = np.array([0.5, -1.0, 0.25, 2.0])
    df = rng.standard_normal((sum(s.shape[0] for s in systems), 3)) if variant == "gemnet-style" else None
    res, bundle = wg.forward_backward(d_energy=de, d_forces=df)
    assert {r.level for r in res.comm_log.records} <= {"global", "position", "param"}
    eng = Engine(DeviceWeights.from_params(params))
    fw = eng.forward(wg.bg)
    pos = eng.backward(wg.bg, fw, torch.tensor(de, device="cuda"),
                       torch.tensor(df, device="cuda") if df is not None else None).cpu().numpy()
    g = eng.weights.to_numpy(grads=True)
    assert max_rel(res.energy, fw.energy.double().cpu().numpy()) < 1e-5
    assert max_rel(bundle.d_positions, pos) < 1e-5
    for k in g:
        assert max_rel(bundle.d_params[k], g[k]) < 1e-5, k


def test_fault_injection_and_errors():
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, _ = _case("dimenet-style")
    good = WorkerGroup(pos, ModelParams(cfg.replace(workers=2), params.arrays)).forward()
    bad = WorkerGroup(pos, ModelParams(cfg.replace(workers=2), params.arrays), fault="drop-last")
    # a dropped contribution is either detected as diverged replicas or yields a different energy
    try:
        res = bad.forward()
        assert abs(res.energy - good.energy) > 1e-6
    except Exception as exc:  # noqa: BLE001
        assert "WorkerGroupError" in type(exc).__name__
    with pytest.raises(ValueError):
        WorkerGroup(pos, ModelParams(cfg.replace(workers=2), params.arrays)).forward_backward(
            d_forces=np.zeros((pos.shape[0], 3)))


def test_graph_aligned_trainer_equals_union_batch():
    """Graph-aligned graph parallelism (bench --gpus N): each rank owns whole graphs,
    the loss is normalised over the global batch and the flat gradient and loss are
    all-reduced -- one step must equal the single-device step over the union batch."""
    import threading

    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.runtime import CommLog, ThreadComm, _ThreadShared
    from paper_2203_09697_b200.tasks import Trainer

    cfg = ModelConfig(variant="gemnet-style", blocks=2, d_u=16, d_v=16, d_e=32, d_t=32, d_bil=32, k_rbf=6,
                      l_sbf=7, cutoff=6.0, seed=2)
    params = init_params(cfg)
    rng = np.random.default_rng(9)
    systems = [O.random_cloud(n, 0.06, rng)[0] for n in (20, 26, 23, 30)]
    e_t = rng.standard_normal(4)
    f_t = [rng.standard_normal((s.shape[0], 3)) for s in systems]
    ref = Trainer(params, None, e_t, np.concatenate(f_t), 1.0, 0.5, graph=build_batch(systems, cfg.cutoff))
    loss_ref = float(ref.step(0.0))
    g_ref = ref.weights.grad_flat.double().cpu().numpy()

    world, per = 2, 2
    shared, log = _ThreadShared(world, 60.0, None), CommLog()
    out = {}

    def body(r):
        sl = slice(r * per, (r + 1) * per)
        bg = build_batch(systems[sl], cfg.cutoff)
        tr = Trainer(params, None, e_t[sl], np.concatenate(f_t[sl]), 1.0, 0.5, graph=bg,
                     comm=ThreadComm(r, shared, log), global_graphs=world * per)
        loss = float(tr.step(0.0))
        torch.cuda.synchronize()
        out[r] = (loss, tr.weights.grad_flat.double().cpu().numpy())

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for r in range(world):
        loss, g = out[r]
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
        assert max_rel(g, g_ref) < 1e-5


def test_gp_dp_composition_equals_union_batch():
    """GP x DP: 2 data-parallel replicas x 2 graph-parallel workers (threads
    on one GPU, ThreadComm per GP group and per DP group).  Each replica runs its own graphs
    through the graph-parallel engine; the replica gradients are all-reduced -- one step
    must equal the single-device step over the union batch."""
    import threading

    from paper_2203_09697_b200 import ModelConfig, init_params
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.partition import partition_centers
    from paper_2203_09697_b200.runtime import CommLog, GPTrainer, ThreadComm, _ThreadShared, gp_dp_layout
    from paper_2203_09697_b200.tasks import Trainer

    cfg = ModelConfig(variant="gemnet-style", blocks=2, d_u=16, d_v=16, d_e=32, d_t=32, d_bil=32, k_rbf=6,
                      l_sbf=7, cutoff=6.0, seed=4)
    params = init_params(cfg)
    rng = np.random.default_rng(12)
    systems = [O.random_cloud(n, 0.06, rng)[0] for n in (21, 27, 24, 19)]
    e_t = rng.standard_normal(4)
    f_t = [rng.standard_normal((s.shape[0], 3)) for s in systems]
    ref = Trainer(params, None, e_t, np.concatenate(f_t), 1.0, 0.5, graph=build_batch(systems, cfg.cutoff))
    loss_ref = float(ref.step(0.0))
    g_ref = ref.weights.grad_flat.double().cpu().numpy()

    world, gp = 4, 2
    gp_groups, dp_groups = gp_dp_layout(world, gp)
    log = CommLog()
    gp_shared = [_ThreadShared(gp, 60.0, None) for _ in gp_groups]
    dp_shared = [_ThreadShared(len(dp_groups[0]), 60.0, None) for _ in dp_groups]
    per = len(systems) // len(gp_groups)
    bgs = [build_batch(systems[k * per:(k + 1) * per], cfg.cutoff) for k in range(len(gp_groups))]
    parts = [partition_centers(bg.deg.cpu().numpy(), gp) for bg in bgs]
    out, errs = {}, []
    stream = torch.cuda.current_stream()

    def body(rank):
        try:
            with torch.cuda.stream(stream):
                k, i = rank // gp, rank % gp  # replica, worker index
                sl = slice(k * per, (k + 1) * per)
                tr = GPTrainer(params, bgs[k], e_t[sl], np.concatenate(f_t[sl]), 1.0, 0.5,
                               ThreadComm(i, gp_shared[k], log), parts[k],
                               dp_comm=ThreadComm(k, dp_shared[i], log), global_graphs=len(systems))
                loss = float(tr.step(0.0))
                torch.cuda.synchronize()
                out[rank] = (loss, tr.weights.grad_flat.double().cpu().numpy())
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            for sh in gp_shared + dp_shared:
                sh.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for r in range(world):
        loss, g = out[r]
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
        assert max_rel(g, g_ref) < 1e-4
    assert "replica" in log.levels()
