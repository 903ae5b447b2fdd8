#!/usr/bin/env python
"""Benchmark of the graph-parallel EGN training step (BASELINE.json metric:
triplet-interactions/s and train steps/s, GemNet-T / DimeNet++).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One step = one SGD training step (forward + backward + update) over one
synthetic batch.  Default workload = BASELINE configs[1]: GemNet-T default
dims (emb 128, triplet emb 64, bilinear 64, 4 blocks), 32 graphs x 80 atoms
per GPU at OC20-like density (random_cloud rho=0.06, cutoff 6 A, <=50
neighbours), loss w_E = w_F = 1 against a teacher model (init_params(seed=1)).

N > 1 (weak scaling, 32 graphs per GPU): graph parallelism over the global
batch (NCCL).  ``--partition aligned`` (default) gives every rank whole graphs
(its own batch), so only the gradient and the loss are all-reduced;
``--partition centre`` splits the centre range by triplet count inside graphs
(runtime.GraphParallelEngine: own-row compute, asynchronous row all-gathers /
reduce-scatters every block); ``--partition reference`` runs the reference's
schedule (split_range shards, full-buffer all-reduces; runtime.ReferenceScheduleEngine).

Prints ONE JSON line (rank 0).  ``value`` = triplet-interactions/s of the
whole job = N_t(global batch) * blocks / t_step, device-timed (CUDA events,
max over ranks) with inputs resident; ``e2e`` = the same metric through Trainer.update_inputs / step
with host buffers: H2D of positions + targets, geometry recomputed on the
resident topology (a pass over a fixed dataset revisits the same graphs, as
train_simple does; the neighbour list is built once per batch), the step, and
the D2H of the loss inside the timed region.  ``--impl reference`` times the CPU reference path
(the fp64 numpy oracle, a restatement of egn.ModelTape; oracle/egn_oracle.py)
on the host cores for a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # BASELINE configs[1]
    "gemnet-t-oc20": dict(variant="gemnet-style", blocks=4, d_u=128, d_v=128, d_e=128, d_t=64, d_bil=64,
                          k_rbf=6, l_sbf=7, cutoff=6.0, atoms=80, density=0.06, graphs=32, w_forces=1.0),
    # BASELINE configs[0] (the reference's own CPU-runnable case)
    "dimenet-pp-small": dict(variant="dimenet-style", blocks=4, d_u=128, d_v=128, d_e=128, d_t=64, d_bil=64,
                             k_rbf=6, l_sbf=7, cutoff=6.0, atoms=64, density=0.06, graphs=4, w_forces=0.0),
    # BASELINE configs[2] / [3] on one GPU: DimeNet++-XL and
    # GemNet-XL (d_e = 1302 zero-padded to 1312 for the tcgen05 tiling)
    "dimenet-pp-xl": dict(variant="dimenet-style", blocks=4, d_u=1536, d_v=1536, d_e=2048, d_t=256, d_bil=64,
                          k_rbf=6, l_sbf=7, cutoff=6.0, atoms=80, density=0.06, graphs=8, w_forces=0.0),
    "gemnet-xl": dict(variant="gemnet-style", blocks=8, d_u=2320, d_v=2320, d_e=1302, d_t=512, d_bil=288,
                      k_rbf=6, l_sbf=7, cutoff=6.0, atoms=80, density=0.06, graphs=8, w_forces=1.0),
}


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="gemnet-t-oc20")
    ap.add_argument("--graphs", type=int, default=None, help="override graphs per GPU")
    ap.add_argument("--partition", choices=["aligned", "centre", "center-aligned", "reference", "balanced"],
                    default="aligned",
                    help="aligned: whole graphs per rank (data parallel); centre (SURVEY 8(e) 'center-aligned', "
                         "the performance mode): centre ranges balanced by triplet count inside graphs, halo "
                         "exchanges every block; reference (SURVEY 8(e) 'balanced', the parity mode): the "
                         "reference's split_range shards and full-buffer all-reduces (CommLog == comm_volume)")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU oracle sampling")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--basis", choices=["gaussian", "bessel"], default="gaussian",
                    help="gaussian: the reference's bases; bessel: DimeNet++ / GemNet-T bases (SURVEY 8(f) f2)")
    ap.add_argument("--no-kernel-timing", action="store_true")
    ap.add_argument("--eager", action="store_true", help="no CUDA-graph replay of the training step")
    return ap.parse_args()


def _config(wl):
    from paper_2203_09697_b200 import ModelConfig

    keys = ("variant", "blocks", "d_u", "d_v", "d_e", "d_t", "d_bil", "k_rbf", "l_sbf", "cutoff")
    return ModelConfig(**{k: wl[k] for k in keys}, seed=0, basis=wl.get("basis", "gaussian"))


def _systems(wl, graphs, rank=0):
    from paper_2203_09697_b200.system import random_cloud

    base = 1000 * rank
    return [random_cloud(wl["atoms"], wl["density"], np.random.default_rng(base + s)) for s in range(graphs)]


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event reasons polled through NVML every ~10 ms while the
    timed region runs (nvidia-smi's own -lms loop starts too slowly for a region of
    well under a second); falls back to one nvidia-smi query per poll."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int, period_s: float = 0.01):
        self.period = period_s
        self.sm, self.smax, self.reasons, self.err = [], None, set(), None
        self._stop = threading.Event()
        self._t = None
        self.h = None
        try:
            import pynvml as N
            import torch

            N.nvmlInit()
            p = torch.cuda.get_device_properties(index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            self.h = N.nvmlDeviceGetHandleByPciBusId(bus)
            self.N = N
            self.bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self.smax = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001 - report, never fail the bench on telemetry
            self.h, self.err = None, f"nvml: {e}"
            self.index = index

    def _poll_once(self):
        if self.h is not None:
            N = self.N
            self.sm.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
            r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for nm, bit in self.bits.items():
                if r & bit:
                    self.reasons.add(nm)
            return
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
        parts = [p.strip() for p in out.split(",")]
        if len(parts) >= 2:
            self.sm.append(float(parts[0]))
            self.smax = float(parts[1])

    def _run(self):
        while not self._stop.is_set():
            try:
                self._poll_once()
            except Exception as e:  # noqa: BLE001
                self.err = str(e)
                return
            self._stop.wait(self.period)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=15)
        out = {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.smax,
               "reasons": sorted(self.reasons), "samples": len(self.sm),
               "source": "nvml" if self.h is not None else "nvidia-smi"}
        if self.err:
            out["error"] = self.err
        return out


# ---------------------------------------------------------------------------
# CPU reference (fp64 numpy oracle, restatement of egn.ModelTape)
# ---------------------------------------------------------------------------
def cpu_reference(wl, systems, budget_s, min_graphs=1):
    from oracle import egn_oracle as O

    cfg = _config(wl)
    oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
    params = O.init_params(oc)
    trip, secs, done = 0, 0.0, 0
    for s in systems:
        g = O.build_graph(s.positions, oc.cutoff)  # graph build excluded (egn/bench.py:294-296)
        t0 = time.perf_counter()
        fw = O.forward(oc, params, s.positions, s.atomic_numbers, graph=g)
        d_f = np.zeros_like(s.positions) if wl["w_forces"] else None
        O.backward(fw, params, 1.0, d_f)
        secs += time.perf_counter() - t0
        trip += g.trip_in.size * oc.blocks
        done += 1
        if done >= min_graphs and secs >= budget_s:
            break
    return {"triplets_per_s": trip / secs, "graphs": done, "seconds": secs, "sec_per_graph": secs / done}


def host_info() -> dict:
    """CPU model, core count and the BLAS threads the numpy oracle runs with."""
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info

        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads"), "version": i.get("version")}
                for i in threadpool_info() if i.get("user_api") == "blas"]
    except Exception:  # noqa: BLE001 - informational only
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset (all cores)"), "blas": blas}


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    graphs = args.graphs or wl["graphs"]
    systems = _systems(wl, graphs)
    cores = os.cpu_count()
    for i in range(args.warmup):
        cpu_reference(wl, [systems[i % graphs]], 0.0)
    trip, secs = 0.0, 0.0
    for i in range(args.steps):  # each step = one graph of the batch, forward + backward (bounded sample)
        r = cpu_reference(wl, [systems[(args.warmup + i) % graphs]], 0.0)
        trip += r["triplets_per_s"] * r["seconds"]
        secs += r["seconds"]
    value = trip / secs
    ms_graph = 1000 * secs / args.steps
    line = {
        "impl": "reference", "metric": "triplet-interactions/s (train step, fwd+bwd+SGD)", "value": value,
        "unit": "triplets/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_graph * graphs * args.gpus, "ms_per_step_kind": "extrapolated: ms per graph x graphs",
        "timed": "forward + backward per graph (the fp64 oracle port of egn.ModelTape + backward); the SGD update "
                 "(one axpy over the parameters) and the graph build are outside the timed region, as in "
                 "egn/bench.py:294-296",
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "variant": wl["variant"], "graphs_per_gpu": graphs,
                   "atoms_per_graph": wl["atoms"], "cutoff": wl["cutoff"],
                   "sample": "one graph of the batch per step (fwd+bwd), host cores"},
        "cpu_baseline": {"value": value, "unit": "triplets/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} graphs x fwd+bwd of the {graphs}-graph batch, fp64 numpy oracle",
                         "host": host_info()},
        "e2e": {"value": value, "unit": "triplets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "steps_per_s": 1000.0 / (ms_graph * graphs * args.gpus),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU path
# ---------------------------------------------------------------------------
def _time_kernel(fn, iters, flush):
    """Device time of one launch of fn with a cold L2: `iters` (256 MB flush, fn) pairs captured
    in one CUDA graph, minus a graph of the flushes alone, timed with CUDA events on the
    capturing stream.  No host launch gap enters the interval."""
    import torch

    fn()
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        g_run, g_flush = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_run, stream=st):
            for _ in range(iters):
                flush.zero_()
                fn()
        with torch.cuda.graph(g_flush, stream=st):
            for _ in range(iters):
                flush.zero_()
    torch.cuda.current_stream().wait_stream(st)

    def replay(g):
        with torch.cuda.stream(st):
            g.replay()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            g.replay()
            e.record(st)
        torch.cuda.synchronize()
        return s.elapsed_time(e) / 1000.0

    t = (replay(g_run) - replay(g_flush)) / iters
    del g_run, g_flush
    return float(t)


def _kernel_roofline(tr, bg, cfg):
    """Roofline of the dominant kernel, measured live with the L2 flushed between launches.

    The dominant kernel by share of the step is the tcgen05 GEMM (~55% of
    the step over 128 calls); its representative launch is the E x 128 x 128 product with a
    residual epilogue (the most frequent wide shape).  Algorithmic bytes = A + W + residual
    read once + output written once.  The triplet-interaction kernels (SURVEY.md 8(d)
    bytes per triplet / edge) are reported alongside under "triplet"."""
    import torch

    from paper_2203_09697_b200 import ops

    eng = tr.engine
    cfg = eng.config  # padded widths (what the kernels run)
    fw = eng.forward(bg)
    st0 = fw.blocks[0]
    dg = cfg.triplet_width
    S_bar = torch.randn_like(st0["S"])
    eg = torch.zeros((bg.num_edges, 4), device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    X, Wk = st0["X"], st0["Wk"]
    t_f = _time_kernel(lambda: ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X, Wk, cfg.cutoff, bg.max_deg), 20,
                       flush)
    t_b = _time_kernel(lambda: ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, X, Wk, cfg.cutoff, S_bar, eg,
                                               max_degree=bg.max_deg), 20, flush)
    ne, nt = bg.num_edges, bg.num_triplets
    b_fwd = 12 * nt + (8 * dg + 4) * ne  # SURVEY.md 8(d) algorithmic bytes
    b_bwd = 16 * nt + (12 * dg + 8) * ne
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    fma = 2.0 * nt * cfg.l_sbf * dg
    fp32_peak = 148 * 128 * 2 * 1.965e9  # FFMA pipe
    # dominant kernel: the E x d_e x d_e GEMM with residual epilogue
    de = cfg.d_e
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn((ne, de), device="cuda", generator=g)
    W = torch.randn((de, de), device="cuda", generator=g) * de ** -0.5
    R = torch.randn((ne, de), device="cuda", generator=g)
    # as in the step: the weight's tf32 lo parts precomputed (egn_gemm_blo; EGN_GEMM_BLO=0: split warps)
    W_lo = None
    if os.environ.get("EGN_GEMM_BLO", "1") != "0":
        W_lo = torch.empty_like(W)
        ops.call("egn_tf32_lo", ops.ptr(W), de, de, de, ops.ptr(W_lo), de, ops.stream())
    t_g = _time_kernel(lambda: ops.gemm(A, W, resid=R, b_lo=W_lo), 20, flush)
    b_gemm = 4 * (3 * ne * de + de * de)
    ach = b_gemm / t_g / 1e9
    traffic = None
    tpath = ROOT / "profiles" / "r2_traffic.json"
    key = f"gemm_fwd_resid_{de}"
    if tpath.exists():
        tj = json.loads(tpath.read_text())
        if tj.get("workload", {}).get("edges") == ne:
            rec = tj.get(key, {})
            traffic = (rec.get("dram_read", 0) + rec.get("dram_write", 0)) or None
    bf16 = peaks.get("bf16_tflops", 1640.8)
    tf32_peak = bf16 / 2  # TF32 = half the bf16 tensor rate
    flops = 2.0 * ne * de * de
    # fp32-accurate products cost 3 TF32 MMAs: the attainable rate is tf32_peak / 3; the kernel is
    # tensor-bound when its intensity (fp32 FLOP per algorithmic byte) exceeds that rate / HBM
    tensor_bound = flops / b_gemm > (tf32_peak / 3) * 1e12 / (hbm * 1e9)
    base = {"kernel": f"gemm_tf32x3 E x {de} x {de} (+residual), 3xTF32 on tcgen05"
                      + (", B lo parts by TMA (egn_gemm_blo)" if W_lo is not None else ""),
            "traffic": traffic, "traffic_source": f"profiles/r2_traffic.json:{key} (ncu --set full)" if traffic else None,
            "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback",
            "launch_us": t_g * 1e6, "algorithmic_bytes": b_gemm, "algorithmic_flops": flops,
            "tensor_frac": 3 * flops / t_g / 1e12 / tf32_peak, "hbm_frac": ach / hbm}
    if tensor_bound:
        base.update(bound="tensor", achieved=flops / t_g / 1e12, unit="TFLOP/s", peak=tf32_peak / 3,
                    frac=flops / t_g / 1e12 / (tf32_peak / 3),
                    peak_derivation=f"measured dense bf16 {bf16:.0f} TF/s / 2 (TF32) / 3 (3xTF32 per fp32 product)")
    else:
        base.update(bound="hbm", achieved=ach, peak=hbm, unit="GB/s", frac=ach / hbm)
    return {**base,
            "triplet": {"fwd_us": t_f * 1e6, "bwd_us": t_b * 1e6,
                        "fwd_gbs": b_fwd / t_f / 1e9, "bwd_gbs": b_bwd / t_b / 1e9,
                        "fwd_hbm_frac": b_fwd / t_f / 1e9 / hbm, "bwd_hbm_frac": b_bwd / t_b / 1e9 / hbm,
                        "fwd_gtrip_s": nt / t_f / 1e9, "bwd_gtrip_s": nt / t_b / 1e9,
                        "fwd_fp32_pipe_frac": fma / t_f / fp32_peak, "bwd_fp32_pipe_frac": 2 * fma / t_b / fp32_peak,
                        "algorithmic_bytes": {"fwd": b_fwd, "bwd": b_bwd}}}


def dense_flops_per_step(cfg, ne, nv):
    """SURVEY.md 8(d) dense algorithmic FLOPs (after the reorder) of one training step:
    forward per block 2[N_e(d_e d_t + K d_t + K L d_t + d_t d_e + 3 d_e^2) + N_v(d_e d_v + d_v^2)]
    (+ GemNet 2 N_e(d_t d_bil + K L d_bil + d_bil d_t + (d_e + d_v) d_e + 2 d_e^2)); backward ~2x."""
    c = cfg
    K, KL = c.k_rbf, c.k_rbf * c.l_sbf
    f = 2 * (ne * (c.d_e * c.d_t + K * c.d_t + KL * c.d_t + c.d_t * c.d_e + 3 * c.d_e ** 2)
             + nv * (c.d_e * c.d_v + c.d_v ** 2))
    if c.variant == "gemnet-style":
        f += 2 * ne * (c.d_t * c.d_bil + KL * c.d_bil + c.d_bil * c.d_t + (c.d_e + c.d_v) * c.d_e + 2 * c.d_e ** 2)
    return 3.0 * f * c.blocks


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    from paper_2203_09697_b200 import _lib, init_params
    from paper_2203_09697_b200.engine import DeviceWeights, Engine
    from paper_2203_09697_b200.graph import build_batch
    from paper_2203_09697_b200.partition import partition_centers, partition_reference
    from paper_2203_09697_b200.runtime import DistComm, GPTrainer
    from paper_2203_09697_b200.tasks import Trainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("EGN_DIST_BACKEND", "nccl")  # gloo: single-GPU smoke test of the N>1 path
    ndev = torch.cuda.device_count()
    torch.cuda.set_device(local % ndev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = _config(wl)
    graphs = args.graphs or wl["graphs"]
    aligned = world == 1 or args.partition == "aligned"
    use_graph = not args.eager
    # weak scaling: every rank contributes `graphs` graphs to the global batch.  With the
    # graph-aligned partition a rank builds and owns only its own graphs.
    if aligned:
        systems = _systems(wl, graphs, rank)
    else:
        systems = [s for r in range(world) for s in _systems(wl, graphs, r)]
    params = init_params(cfg)
    bg = build_batch(systems, cfg.cutoff)
    teacher = Engine(DeviceWeights.from_params(init_params(cfg.replace(seed=1))))
    tf = teacher.forward(bg)
    e_t = tf.energy.double().cpu().numpy()
    f_t = tf.forces.double().cpu().numpy() if wl["w_forces"] else None
    del tf, teacher
    if world == 1:
        tr = Trainer(params, None, e_t, f_t, 1.0, wl["w_forces"], graph=bg, cuda_graph=use_graph)
        comm = None
        parallelism = "single"
    elif aligned:
        # graph-aligned centre partition: no halo, one gradient all-reduce per step
        comm = DistComm()
        tr = Trainer(params, None, e_t, f_t, 1.0, wl["w_forces"], graph=bg, comm=comm,
                     global_graphs=graphs * world, cuda_graph=use_graph)
        parallelism = f"gp{world} (graph-aligned centre partition: no halo, gradient all-reduce, {backend})"
    else:
        comm = DistComm()
        if args.partition == "centre":
            part = partition_centers(bg.deg.cpu().numpy(), world)
        else:
            part = partition_reference(bg.tri_ptr.cpu().numpy(), bg.num_edges, bg.num_nodes, world)
        tr = GPTrainer(params, bg, e_t, f_t, 1.0, wl["w_forces"], comm, part,
                       cuda_graph=use_graph and backend == "nccl")
        parallelism = f"gp{world} ({args.partition} schedule, halo exchanges every block, {backend})"

    def barrier():
        if world > 1:
            dist.barrier()

    # SGD step size from the first gradient (keeps the synthetic run finite); lr=0 step is outside timing
    loss0 = float(tr.step(0.0))
    gnorm = float(tr.weights.grad_flat.norm())
    lr = 1e-2 / max(gnorm, 1.0)
    for _ in range(args.warmup):
        tr.step(lr)
    torch.cuda.synchronize()
    barrier()
    clocks = ClockSampler(torch.cuda.current_device()) if rank == 0 else None
    if clocks:
        clocks.start()
    _lib.LAUNCH_COUNTER.update(calls=0, kernels=0)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    st.record()
    for _ in range(args.steps):
        loss = tr.step(lr)
    en.record()
    torch.cuda.synchronize()
    t_dev = st.elapsed_time(en) / 1000.0 / args.steps
    launches = _lib.LAUNCH_COUNTER["kernels"] // args.steps
    if getattr(tr, "cuda_graph", False) and getattr(tr, "kernels_per_step", None):
        launches = tr.kernels_per_step  # replayed from the captured step graph
    loss_last = float(loss)
    # ---- end to end: host buffers -> device -> step -> loss back to host
    pos_host = torch.from_numpy(np.concatenate([s.positions for s in systems])).pin_memory()
    et_host = torch.from_numpy(e_t).pin_memory()
    ft_host = torch.from_numpy(f_t).pin_memory() if f_t is not None else None
    h2d = pos_host.numel() * 8 + et_host.numel() * 8 + (ft_host.numel() * 8 if ft_host is not None else 0)
    sizes = [s.positions.shape[0] for s in systems]

    # every step's loss comes back to pinned host memory asynchronously (the next step's
    # inputs are queued behind it, as a training loop that logs its loss does); the timed
    # region ends with a synchronize, so every copy is inside it
    loss_host = torch.zeros(args.steps + 2, dtype=torch.float64).pin_memory()

    def e2e_step(i):
        pos = pos_host.to("cuda", non_blocking=True)
        et = et_host.to("cuda", non_blocking=True)
        ft = ft_host.to("cuda", non_blocking=True) if ft_host is not None else None
        if aligned:
            # same batch every step (a pass over a fixed dataset): copy this step's
            # positions and targets into the resident batch, recompute its geometry
            tr.update_inputs(pos, et, ft)
        else:
            tr.bg.update_positions(pos)
            tr.e_target = et
            tr.f_target = ft[tr.n0:tr.n1] if ft is not None else None
        loss_host[i].copy_(tr.step(lr).reshape(()), non_blocking=True)

    for i in range(2):
        e2e_step(args.steps + i)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        e2e_step(i)
    torch.cuda.synchronize()
    t_e2e = (time.perf_counter() - t0) / args.steps
    if not bool(torch.isfinite(loss_host[:args.steps]).all()):
        raise RuntimeError("non-finite loss in the end-to-end steps")
    clk = clocks.stop() if clocks else None

    tt = torch.tensor([t_dev, t_e2e], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_dev, t_e2e = float(tt[0]), float(tt[1])
    nt = torch.tensor([float(bg.num_triplets), float(bg.num_edges)], dtype=torch.float64, device="cuda")
    if world > 1 and aligned:
        dist.all_reduce(nt)  # each rank holds its own graphs
    total_trip = float(nt[0]) * cfg.blocks  # global batch (all ranks)
    value = total_trip / t_dev
    roof = None
    if rank == 0 and not args.no_kernel_timing:
        rb = bg if aligned else build_batch(systems[:graphs], cfg.cutoff)
        if not aligned:
            rtr = Trainer(params, None, e_t[:graphs], None, 1.0, 0.0, graph=rb)
        else:
            rtr = tr
        roof = _kernel_roofline(rtr, rb, cfg)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        r = cpu_reference(wl, systems[:graphs], args.cpu_budget)
        cpu = {"value": r["triplets_per_s"], "unit": "triplets/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"{r['graphs']} graph(s) of the batch, fwd+bwd, fp64 numpy oracle, {r['seconds']:.1f}s",
               "host": host_info()}
    if rank == 0:
        line = {
            "metric": "triplet-interactions/s (train step, fwd+bwd+SGD)", "value": value, "unit": "triplets/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random_cloud OC20-density graphs, random-init weights, teacher targets)",
            "config": {"workload": args.workload, "variant": wl["variant"], "graphs_per_gpu": graphs,
                       **({"basis": cfg.basis} if cfg.basis != "gaussian" else {}),
                       "atoms_per_graph": wl["atoms"], "cutoff": wl["cutoff"], "blocks": cfg.blocks,
                       "d_e": cfg.d_e, "d_t": cfg.d_t, "d_bil": cfg.d_bil, "edges_total": int(nt[1]),
                       "triplets_total": int(nt[0]), "parallelism": parallelism,
                       "l2": "step working set > L2 (126 MB); kernel timings flush L2 with a 256 MB write"},
            "steps_per_s": 1.0 / t_dev,
            "dense": {"tflop_per_step": dense_flops_per_step(cfg, int(nt[1]), sum(len(s.positions) for s in systems)
                                                             * (world if aligned else 1)) / 1e12,
                      "achieved_tflops": dense_flops_per_step(cfg, int(nt[1]), sum(len(s.positions) for s in systems)
                                                              * (world if aligned else 1)) / t_dev / 1e12,
                      "source": "SURVEY.md 8(d) formula, reference widths, fwd + 2x bwd"},
            "e2e": {"value": total_trip / t_e2e, "unit": "triplets/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8, "ms_per_step": t_e2e * 1e3},
            "gpu_launches": launches,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk,
            "loss": {"first": loss0, "last": loss_last, "lr": lr},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = _args()
    args.partition = {"balanced": "reference", "center-aligned": "centre"}.get(args.partition, args.partition)
    wl = dict(WORKLOADS[args.workload], basis=args.basis)
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
