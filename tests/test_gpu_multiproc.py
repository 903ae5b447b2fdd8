"""Graph parallelism through real process groups: 2 processes on cuda:0, torch.distributed
gloo (NCCL refuses two ranks on one device; gloo stages the CUDA buffers through host
memory, so no rank's kernel ever waits on another rank's kernel on the device).

Each rank runs GPTrainer on a batch whose partition cuts through graphs (halo edges and
nodes): the centre schedule (row all-gathers / reduce-scatters through DistComm) and the
reference schedule (split_range shards, full-buffer all-reduces).  One step must equal the
single-process Trainer step over the same batch (egn/runtime.py parallel == sequential,
tests/test_runtime.py:135-160), and bench.py's multi-rank path must run end to end.
"""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import max_rel

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    sys.path.insert(0, str(ROOT))
    from oracle import egn_oracle as O
    from paper_2203_09697_b200 import ModelConfig, init_params

    cfg = ModelConfig(variant="gemnet-style", blocks=2, d_u=16, d_v=32, d_e=32, d_t=32, d_bil=16, k_rbf=6,
                      l_sbf=7, cutoff=6.0, seed=3)
    rng = np.random.default_rng(17)
    systems = [O.random_cloud(n, 0.06, rng)[0] for n in (30, 44, 37)]
    e_t = rng.standard_normal(3)
    f_t = np.concatenate([rng.standard_normal((s.shape[0], 3)) for s in systems])
    return cfg, init_params(cfg), systems, e_t, f_t


def _worker(rank, world, port, schedule, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2203_09697_b200.graph import build_batch
        from paper_2203_09697_b200.partition import partition_centers, partition_reference
        from paper_2203_09697_b200.runtime import DistComm, GPTrainer

        cfg, params, systems, e_t, f_t = _case()
        bg = build_batch(systems, cfg.cutoff)
        if schedule == "centre":
            part = partition_centers(bg.deg.cpu().numpy(), world)  # splits inside graphs: halo rows
        else:
            part = partition_reference(bg.tri_ptr.cpu().numpy(), bg.num_edges, bg.num_nodes, world)
        comm = DistComm()
        tr = GPTrainer(params, bg, e_t, f_t, 1.0, 0.5, comm, part)
        if schedule == "centre":
            assert not tr.engine.halo_free(bg)
        loss = float(tr.step(0.0))
        torch.cuda.synchronize()
        g = tr.weights.grad_flat.double().cpu().numpy()
        levels = sorted({r.level for r in comm.log.records})
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", loss, g, levels))
    except BaseException as exc:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc(), None, None, None))


@pytest.mark.parametrize("schedule", ["centre", "reference"])
def test_two_process_gp_step_equals_single_process(schedule):
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    cfg, params, systems, e_t, f_t = _case()
    ref = Trainer(params, None, e_t, f_t, 1.0, 0.5, graph=build_batch(systems, cfg.cutoff))
    loss_ref = float(ref.step(0.0))
    g_ref = ref.weights.grad_flat.double().cpu().numpy()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, schedule, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, status, loss, g, levels in sorted(res, key=lambda x: x[0]):
        assert status == "ok", status
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref), (rank, loss, loss_ref)
        assert max_rel(g, g_ref) < 1e-5, rank
        if rank == 0:  # rank 0 keeps the CommLog
            assert "edge" in levels and "node" in levels  # real halo exchanges happened


@pytest.mark.parametrize("partition", ["centre", "aligned", "balanced"])
def test_bench_multi_rank_path_runs(partition):
    """bench.py under torchrun with 2 ranks (gloo on one GPU): the centre partition with halos,
    the default graph-aligned data parallelism (captured step + gradient all-reduce) and the
    reference parity schedule ("balanced")."""
    env = dict(os.environ, EGN_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "1", "--graphs", "2", "--partition", partition, "--no-cpu-baseline",
           "--no-kernel-timing"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    expect = {"centre": "centre", "aligned": "graph-aligned", "balanced": "reference schedule"}[partition]
    assert expect in line["config"]["parallelism"]


def _nccl_worker(port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        from paper_2203_09697_b200.graph import build_batch
        from paper_2203_09697_b200.partition import partition_centers, partition_reference
        from paper_2203_09697_b200.runtime import DistComm, GPTrainer
        from paper_2203_09697_b200.tasks import Trainer

        cfg, params, systems, e_t, f_t = _case()
        bg = build_batch(systems, cfg.cutoff)
        out = {}
        for name in ("centre", "reference"):
            part = (partition_centers(bg.deg.cpu().numpy(), 1) if name == "centre"
                    else partition_reference(bg.tri_ptr.cpu().numpy(), bg.num_edges, bg.num_nodes, 1))
            tr = GPTrainer(params, bg, e_t, f_t, 1.0, 0.5, DistComm(), part)
            out[name] = (float(tr.step(0.0)), tr.weights.grad_flat.double().cpu().numpy())
            # the captured step (compute + NCCL collectives in one CUDA graph), replayed
            trg = GPTrainer(params, bg, e_t, f_t, 1.0, 0.5, DistComm(), part, cuda_graph=True)
            trg.step(0.0)
            assert trg._graph is not None, "capture failed"
            out[name + "-graph"] = (float(trg.step(0.0)), trg.weights.grad_flat.double().cpu().numpy())
        # graph-aligned data parallelism (bench.py's default N > 1 path): gradient all-reduce
        tr = Trainer(params, None, e_t, f_t, 1.0, 0.5, graph=bg, comm=DistComm(), global_graphs=len(systems),
                     cuda_graph=True)
        tr.step(0.0)
        out["aligned"] = (float(tr.step(0.0)), tr.weights.grad_flat.double().cpu().numpy())
        torch.cuda.synchronize()
        dist.destroy_process_group()
        q.put(("ok", out))
    except BaseException:  # noqa: BLE001
        import traceback

        q.put((traceback.format_exc(), None))


def test_nccl_process_group_paths_world1():
    """The NCCL code paths of DistComm (async all_reduce, all_gather_into_tensor,
    reduce_scatter_tensor on device buffers) inside GPTrainer (both schedules) and the
    graph-aligned Trainer with a captured step, through a real NCCL process group of one rank
    (one GPU per rank is all NCCL allows); results equal the communicator-free Trainer."""
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.tasks import Trainer

    cfg, params, systems, e_t, f_t = _case()
    ref = Trainer(params, None, e_t, f_t, 1.0, 0.5, graph=build_batch(systems, cfg.cutoff))
    loss_ref = float(ref.step(0.0))
    g_ref = ref.weights.grad_flat.double().cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    status, out = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", status
    for name, (loss, g) in out.items():
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref), (name, loss, loss_ref)
        assert max_rel(g, g_ref) < 1e-5, name
