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


@pytest.mark.parametrize("schedule", ["reference", "centre"])
@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
@pytest.mark.parametrize("workers", [1, 2, 3, 4])
def test_parallel_matches_oracle(variant, workers, schedule):
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, z = _case(variant)
    run = ModelParams(cfg.replace(workers=workers), params.arrays)
    rng = np.random.default_rng(5)
    df = rng.standard_normal((pos.shape[0], 3)) if variant == "gemnet-style" else None
    res, bundle = WorkerGroup(pos, run, schedule=schedule).forward_backward(d_energy=0.8, d_forces=df)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    fw = O.forward(oc, params.arrays, pos, z)
    G, dpos = O.backward(fw, params.arrays, 0.8, df)
    assert abs(res.energy - fw.energy) <= TOL * max(1.0, abs(fw.energy))
    if variant == "gemnet-style":
        assert max_rel(res.forces, fw.forces) < TOL
    assert max_rel(bundle.d_positions, dpos) < TOL
    for k, g in G.items():
        assert max_rel(bundle.d_params[k], g) < TOL, k


@pytest.mark.parametrize("schedule", ["reference", "centre"])
@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_parallel_equals_single_rank_engine(variant, schedule):
    """P = 1, 2, 4 agree with each other to fp32 summation-order noise."""
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, _ = _case(variant, n=60, seed=7)
    outs = {}
    for p in (1, 2, 4):
        run = ModelParams(cfg.replace(workers=p), params.arrays)
        outs[p] = WorkerGroup(pos, run, schedule=schedule).forward_backward(d_energy=1.0)
    r1, b1 = outs[1]
    for p in (2, 4):
        rp, bp = outs[p]
        assert abs(rp.energy - r1.energy) <= 1e-5 * max(1.0, abs(r1.energy))
        assert max_rel(bp.d_positions, b1.d_positions) < 1e-5
        for k in b1.d_params:
            assert max_rel(bp.d_params[k], b1.d_params[k]) < 1e-5, k


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_centre_schedule_comm_volume(variant):
    """Centre schedule, forward rows moved per block: X (N_e d_g) + m_new (N_e d_e) + G d_v
    (+ pv (N_v d_e) + m2 (N_e d_e) for gemnet) -- independent of the triplet count; no
    triplet-level buffer."""
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, _ = _case(variant)
    for d_t in (16, 48):
        c2 = cfg.replace(workers=3, d_t=d_t)
        from paper_2203_09697_b200 import init_params

        wg = WorkerGroup(pos, init_params(c2), schedule="centre")
        res = wg.forward()
        ne, nv = wg.bg.num_edges, wg.bg.num_nodes
        expect = ne * c2.triplet_width + ne * c2.d_e + c2.d_v
        if variant == "gemnet-style":
            expect += ne * c2.d_e + nv * c2.d_e
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
    wg = WorkerGroup(systems, ModelParams(cfg.replace(workers=2), params.arrays), schedule="centre",
                     align_graphs=True)
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


# ---------------------------------------------------------------------------
# reference schedule: the reference's own runtime tests (tests/test_runtime.py) on the GPU
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
@pytest.mark.parametrize("workers", [1, 2, 5])
def test_forward_comm_matches_prediction_exactly(variant, workers):
    """tests/test_runtime.py:202-212: forward CommLog == comm_volume, per block and total."""
    from paper_2203_09697_b200 import CommModel, comm_volume, init_params
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, _, pos, _ = _case(variant)
    cfg = cfg.replace(workers=workers)
    group = WorkerGroup(pos, init_params(cfg))
    result, _ = group.forward_backward(d_energy=1.0)
    expected = comm_volume(CommModel.from_graph(group.topology, cfg), cfg.blocks)
    per_block = result.comm_log.forward_blocks()
    assert sorted(per_block) == list(range(cfg.blocks))
    for elements in per_block.values():
        assert elements == expected.per_block
    assert result.comm_log.elements(phase="forward") == expected.total
    # tests/test_runtime.py:225-240: only replicated-buffer sizes, never a triplet buffer
    assert {r.level for r in result.comm_log.records if r.phase == "forward"} == {"edge", "node", "global"}
    sizes = {group.topology.num_edges * cfg.d_e, group.topology.num_nodes * cfg.d_v, cfg.d_u}
    assert all(r.elements in sizes for r in result.comm_log.records if r.phase == "forward")


def test_forward_comm_invariant_under_triplet_dim():
    """tests/test_runtime.py:215-222."""
    from paper_2203_09697_b200 import init_params
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, _, pos, _ = _case("gemnet-style")
    counts = {}
    for d_t in (8, 24):
        c2 = cfg.replace(workers=2, d_t=d_t, d_bil=d_t)
        counts[d_t] = WorkerGroup(pos, init_params(c2)).forward().comm_log.elements(phase="forward")
    assert counts[8] == counts[24]


@pytest.mark.parametrize("variant", ["dimenet-style", "gemnet-style"])
def test_triplet_shards_are_split_range_and_match_oracle(variant):
    """ParallelRunResult.triplet_shards (egn/runtime.py:430-431): rank r holds the last block's
    t_feat rows of split_range(N_t, P)[r] -- shards cut through centre tiles (window kernel)."""
    from paper_2203_09697_b200 import ModelParams, split_range
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, z = _case(variant)
    run = ModelParams(cfg.replace(workers=3), params.arrays)
    group = WorkerGroup(pos, run)
    res = group.forward()
    nt = group.topology.num_triplets
    shards = split_range(nt, 3)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    ref = O.forward(oc, params.arrays, pos, z).t_feat
    assert [s.shape[0] for s in res.triplet_shards] == [s.size for s in shards]
    for got, idx in zip(res.triplet_shards, shards):
        assert max_rel(got, ref[idx]) < TOL
    # a shard boundary strictly inside a centre's tile exists in this graph
    tp = group.bg.tri_ptr.cpu().numpy()
    assert any(int(s[0]) not in set(tp.tolist()) for s in shards[1:] if s.size)


def test_replicas_identical_and_stage_timing():
    """tests/test_runtime.py:243-252 (replica digests agree after every collective) and
    :318-328 (stage timing CSV)."""
    from paper_2203_09697_b200 import ModelParams
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg, params, pos, _ = _case("gemnet-style")
    group = WorkerGroup(pos, ModelParams(cfg.replace(workers=3), params.arrays), track_replicas=True)
    res, _ = group.forward_backward(d_energy=1.0)
    assert len(res.replica_digests) == 3 and len(res.replica_digests[0]) > 0
    assert res.replica_digests[0] == res.replica_digests[1] == res.replica_digests[2]
    assert {"init", "block0.tu", "block0.eu", "block0.nu", "backward.reduce"} <= set(res.stage_seconds)
    assert all(v >= 0.0 for v in res.stage_seconds.values())
    rows = res.timing_csv_rows()
    assert rows[0] == "stage,seconds" and len(rows) == len(res.stage_seconds) + 1


def test_zero_edge_and_more_workers_than_triplets():
    """tests/test_runtime.py:178-199: empty shards contribute zeros."""
    from paper_2203_09697_b200 import ModelConfig, ModelParams, init_params
    from paper_2203_09697_b200.runtime import WorkerGroup

    cfg = ModelConfig(variant="gemnet-style", blocks=1, workers=3)
    params = init_params(cfg)
    far = np.array([[0.0, 0, 0], [40.0, 0, 0]])
    res, _ = WorkerGroup(far, params).forward_backward(d_energy=1.0)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    f = O.forward(oc, params.arrays, far, np.ones(2, dtype=np.int64))
    assert abs(res.energy - f.energy) <= TOL * max(1.0, abs(f.energy))
    np.testing.assert_array_equal(res.forces, np.zeros((2, 3)))
    tri = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1.2, 0]])
    cfg6 = ModelConfig(variant="dimenet-style", blocks=2, workers=8)
    p6 = init_params(cfg6)
    res6, b6 = WorkerGroup(tri, p6).forward_backward(d_energy=1.0)
    oc6 = O.Config(**{k: getattr(cfg6, k) for k in O.Config.__dataclass_fields__})
    f6 = O.forward(oc6, p6.arrays, tri, np.ones(3, dtype=np.int64))
    G6, dp6 = O.backward(f6, p6.arrays, 1.0)
    assert abs(res6.energy - f6.energy) <= TOL * max(1.0, abs(f6.energy))
    assert max_rel(b6.d_positions, dp6) < TOL
