"""B200-native graph-parallel DimeNet++/GemNet-T training hot path.

A drop-in for the reference package ``egn`` (arXiv 2203.09697, "Graph
Parallelism"): same configuration, weight names, graph/partition interface
and drivers, executed by hand-written sm_100a kernels behind the C ABI in
include/egn_b200.h (libegn_b200.so).  See DESIGN.md.
"""

from .config import DIMENET, GEMNET, ModelConfig
from .params import ModelParams, ParamSpec, init_params, load_params, param_specs, save_params, zero_params
from .partition import (CenterPartition, CommModel, CommVolume, GraphPartition, ReferencePartition, comm_volume,
                        partition_centers, partition_graph, partition_reference, split_range)
from .system import AtomicSystem, random_cloud

__all__ = [
    "DIMENET", "GEMNET", "ModelConfig", "ModelParams", "ParamSpec", "init_params", "load_params",
    "param_specs", "save_params", "zero_params", "CenterPartition", "CommModel", "CommVolume",
    "GraphPartition", "comm_volume", "partition_centers", "partition_graph", "split_range",
    "AtomicSystem", "random_cloud", "build_graph", "build_batch", "EGNModel", "predict", "relax", "RelaxationResult",
    "loss_and_grads", "train_simple", "Trainer", "enumerate_triplets", "WorkerGroup", "ParallelRunResult",
    "GradientBundle", "CollectiveShapeError", "CollectiveTimeoutError", "WorkerGroupError",
    "ModelTape", "BasisFeatures", "compute_basis", "rbf_features", "sbf_features", "initial_state", "block_forward",
    "GeometryGrads", "backward", "forces_energy_centric", "geometry_grads", "FeatureState", "Collective", "CommLog",
    "partition_reference", "ReferencePartition",
]


def __getattr__(name):
    # GPU-facing pieces load the native library lazily (CPU-only hosts can
    # still import the config/params/partition surface).
    if name in ("build_graph", "build_batch", "enumerate_triplets", "BatchGraph", "GraphTopology", "Geometry"):
        from . import graph
        return getattr(graph, name)
    if name in ("EGNModel",):
        from .model import EGNModel
        return EGNModel
    if name in ("predict", "relax", "RelaxationResult", "loss_and_grads", "train_simple", "Trainer"):
        from . import tasks
        return getattr(tasks, name)
    if name in ("ModelTape", "BasisFeatures", "compute_basis", "rbf_features", "rbf_features_ddist", "sbf_features",
                "sbf_features_partials", "initial_state", "block_forward", "GeometryGrads", "backward",
                "forces_energy_centric", "geometry_grads"):
        from . import api
        return getattr(api, name)
    if name in ("WorkerGroup", "ParallelRunResult", "GradientBundle", "CollectiveError", "CollectiveShapeError",
                "CollectiveTimeoutError", "WorkerGroupError", "GraphParallelEngine", "GPTrainer", "FeatureState",
                "Collective", "CommLog", "ReferenceScheduleEngine"):
        from . import runtime
        return getattr(runtime, name)
    if name in ("Engine", "DeviceWeights"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
