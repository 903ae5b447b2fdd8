"""Graph-parallel collectives on CPU: torch.distributed gloo, world size 2 and 3.

Covers the host-side runtime (row-range all-gather / reduce-scatter /
all-reduce semantics with uneven ownership, CommLog accounting, the level
guard) without a GPU; the device math of the schedule is covered by
tests/test_gpu_runtime.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2203_09697_b200.runtime import DistComm

        comm = DistComm()
        bounds = np.array([0, 3, 7, 8][: world + 1]) if world == 3 else np.array([0, 5, 8])
        n = int(bounds[-1])
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        # all-gather rows: every rank fills its own rows with (rank+1)*row index
        full = torch.full((n, 4), -1.0)
        full[lo:hi] = (rank + 1) * torch.arange(lo, hi, dtype=torch.float32)[:, None]
        comm.all_gather_rows(full, bounds, phase="forward", block=0, stage="m_new", level="edge")
        expect = torch.zeros((n, 4))
        for r in range(world):
            a, b = int(bounds[r]), int(bounds[r + 1])
            expect[a:b] = (r + 1) * torch.arange(a, b, dtype=torch.float32)[:, None]
        assert torch.equal(full, expect)
        # reduce-scatter: each rank contributes rank+1 everywhere; own rows receive the sum
        part = torch.full((n, 3), float(rank + 1))
        own = comm.reduce_scatter_rows(part, bounds, phase="backward", block=0, stage="m_new", level="edge")
        assert own.shape == (hi - lo, 3)
        assert torch.allclose(own, torch.full((hi - lo, 3), float(sum(range(1, world + 1)))))
        # all-reduce
        t = torch.tensor([float(rank)])
        comm.all_reduce_(t, phase="forward", block=0, stage="gu", level="global")
        assert float(t) == float(sum(range(world)))
        # level guard: triplet buffers never enter a collective
        try:
            comm.all_reduce_(torch.zeros(1), level="triplet")
            raise AssertionError("triplet level accepted")
        except ValueError:
            pass
        if rank == 0:
            recs = comm.log.records
            assert [r.op for r in recs] == ["all_gather", "reduce_scatter", "all_reduce"]
            assert recs[0].elements == n * 4 and recs[2].level == "global"
            assert comm.log.elements(phase="forward") == n * 4 + 1
            assert comm.log.to_csv_rows()[0].startswith("phase,block")
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))


@pytest.mark.parametrize("world", [2, 3])
def test_dist_comm_row_collectives_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(results) == [(r, "ok") for r in range(world)], results


def test_thread_comm_semantics_cpu():
    """In-process ranks (threads): rank-ordered sums, identical results, fault hook, shape check."""
    import threading

    from paper_2203_09697_b200.runtime import CollectiveShapeError, CommLog, ThreadComm, _ThreadShared

    for fault in (None, "drop-last"):
        sh = _ThreadShared(3, timeout=10.0, fault=fault)
        log = CommLog()
        out = [None] * 3

        def body(r):
            c = ThreadComm(r, sh, log)
            t = torch.tensor([float(r + 1)])
            c.all_reduce_(t, level="global")
            full = torch.zeros((6, 2))
            b = np.array([0, 2, 4, 6])
            full[b[r]:b[r + 1]] = r + 1
            c.all_gather_rows(full, b, level="edge")
            out[r] = (float(t), full.clone())

        ts = [threading.Thread(target=body, args=(r,)) for r in range(3)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        expect = 3.0 if fault else 6.0
        assert all(o[0] == expect for o in out)
        assert all(torch.equal(o[1], out[0][1]) for o in out)
        assert len(log.records) == 2
    sh = _ThreadShared(2, timeout=10.0, fault=None)
    errs = [None, None]

    def bad(r):
        try:
            ThreadComm(r, sh, CommLog()).all_reduce_(torch.zeros(r + 1), level="edge")
        except CollectiveShapeError as e:
            errs[r] = e

    ts = [threading.Thread(target=bad, args=(r,)) for r in range(2)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert all(isinstance(e, CollectiveShapeError) for e in errs)


def test_thread_comm_timeout():
    from paper_2203_09697_b200.runtime import CollectiveTimeoutError, CommLog, ThreadComm, _ThreadShared

    sh = _ThreadShared(2, timeout=0.5, fault=None)
    with pytest.raises(CollectiveTimeoutError):
        ThreadComm(0, sh, CommLog()).all_reduce_(torch.zeros(1), level="global")


def test_gp_dp_layout():
    from paper_2203_09697_b200.runtime import gp_dp_layout

    gp, dp = gp_dp_layout(8, 2)
    assert gp == [[0, 1], [2, 3], [4, 5], [6, 7]]
    assert dp == [[0, 2, 4, 6], [1, 3, 5, 7]]
    gp, dp = gp_dp_layout(6, 3)
    assert gp == [[0, 1, 2], [3, 4, 5]] and dp == [[0, 3], [1, 4], [2, 5]]
    with pytest.raises(ValueError):
        gp_dp_layout(6, 4)


def _gp_dp_worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2203_09697_b200.runtime import DistComm

        gp_comm, dp_comm = DistComm.gp_dp(2)
        t = torch.tensor([float(rank)])
        gp_comm.all_reduce_(t.clone(), level="param")
        a = gp_comm.all_reduce_(torch.tensor([float(rank)]), level="param")
        b = dp_comm.all_reduce_(torch.tensor([float(rank)]), level="replica")
        k, i = rank // 2, rank % 2
        assert float(a) == float(2 * k + 2 * k + 1), (rank, float(a))  # ranks 2k, 2k+1
        assert float(b) == float(i + (i + 2)), (rank, float(b))        # ranks i, i+2
        assert gp_comm.rank == i and dp_comm.rank == k and gp_comm.world == 2 and dp_comm.world == 2
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))


def test_gp_dp_groups_gloo():
    """GP x DP communicators (world 4 = 2 replicas x 2 graph-parallel workers) on gloo."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 4
    procs = [ctx.Process(target=_gp_dp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(results) == [(r, "ok") for r in range(world)], results
