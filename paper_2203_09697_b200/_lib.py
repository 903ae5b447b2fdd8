"""ctypes binding of ``libegn_b200.so`` (the C ABI declared in include/egn_b200.h).

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
and is the only compute path: importing an op without the library raises,
there is no CPU fallback.  Tensors are passed as raw device pointers; every
call runs on torch's current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("EGN_LIB", _HERE / "libegn_b200.so"))  # EGN_LIB: same-box A/B builds

_p = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_f32 = ctypes.c_float
_f64 = ctypes.c_double

class SmallGemm(ctypes.Structure):
    """egn_small_gemm_t (include/egn_b200.h)."""

    _fields_ = [("a", _p), ("b", _p), ("c", _p), ("m", _i32), ("n", _i32), ("k", _i32), ("lda", _i32),
                ("ldb", _i32), ("ldc", _i32), ("trans_a", _i32), ("trans_b", _i32), ("trans_c", _i32)]


# name -> (restype, argtypes); mirrors include/egn_b200.h
SIGNATURES: dict[str, tuple] = {
    "egn_last_error": (ctypes.c_char_p, []),
    "egn_abi_version": (_i32, []),
    "egn_neighbors_count": (_i32, [_p, _p, _p, _i64, _f64, _p, _p]),
    "egn_scan_counts": (_i32, [_p, _i64, _i32, _p, _p]),
    "egn_neighbors_fill": (_i32, [_p, _p, _p, _i64, _f64, _p, _p, _p, _p]),
    "egn_reverse_edges": (_i32, [_p, _p, _p, _i64, _p, _p, _p]),
    "egn_triplets_fill": (_i32, [_p, _p, _p, _i64, _p, _p, _p]),
    "egn_geometry": (_i32, [_p, _p, _p, _i64, _p, _p, _p, _p]),
    "egn_neighbors_count_pbc": (_i32, [_p, _p, _p, _i64, _p, _p, _f64, _p, _p]),
    "egn_gemm_simt_max_m": (_i64, [_i64]),
    "egn_adamw": (_i32, [_p, _p, _p, _p, _i64, _f32, _f32, _f32, _f32, _f32, _i64, _p]),
    "egn_loss_seeds": (_i32, [_p, _p, _i64, _p, _p, _p, _i64, _f64, _f64, _f64, _p, _p, _p, _p]),
    "egn_cap_keep": (_i32, [_p, _p, _p, _i64, _i32, _p, _p, _p, _p]),
    "egn_cap_compact": (_i32, [_p, _p, _i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "egn_graph_mlp_fwd": (_i32, [_i64, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "egn_graph_mlp_bwd": (_i32, [_i64, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "egn_neighbors_fill_pbc": (_i32, [_p, _p, _p, _i64, _p, _p, _f64, _p, _p, _p, _p, _p, _p]),
    "egn_reverse_edges_pbc": (_i32, [_p, _p, _p, _p, _p, _p, _i64, _p, _p, _p]),
    "egn_geometry_shift": (_i32, [_p, _p, _p, _p, _i64, _p, _p, _p, _p]),
    "egn_triplet_angles_shift": (_i32, [_p, _p, _p, _p, _p, _i64, _p, _p]),
    "egn_triplet_angles": (_i32, [_p, _p, _p, _p, _i64, _p, _p]),
    "egn_rbf": (_i32, [_p, _i64, _i32, _f64, _p, _p]),
    "egn_sbf": (_i32, [_p, _p, _p, _i64, _i32, _i32, _f64, _p, _p]),
    "egn_triplet_fwd_workspace_bytes": (_i64, [_i64, _i32, _i32, _i32, _i32]),
    "egn_triplet_fwd": (_i32, [_p, _p, _p, _i64, _i32, _p, _p, _i32, _i32, _i32, _f64, _p, _p, _p]),
    "egn_triplet_bwd_workspace_bytes": (_i64, [_i64, _i64, _i32, _i32, _i32, _i32]),
    "egn_triplet_bwd": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p, _p, _i32, _i32, _i32, _f64, _p, _p, _p, _p, _p,
                               _p]),
    "egn_triplet_bwd_ex": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p, _p, _i32, _i32, _i32, _f64, _p, _p, _p, _p,
                                  _i32, _p, _p]),
    "egn_triplet_path": (_i32, [_i32]),
    "egn_triplet_fwd_basis_workspace_bytes": (_i64, [_i64, _i64, _i32, _i32, _i32, _i32, _i32]),
    "egn_triplet_bwd_basis_workspace_bytes": (_i64, [_i64, _i64, _i32, _i32, _i32, _i32, _i32]),
    "egn_triplet_fwd_basis": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p, _p, _i32, _i32, _i32, _f64, _i32, _p, _p,
                                     _p]),
    "egn_triplet_bwd_basis": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p, _p, _i32, _i32, _i32, _f64, _i32, _p, _p, _p,
                                     _p, _p, _p]),
    "egn_triplet_bwd_angle_workspace_bytes": (_i64, [_i64, _i32]),
    "egn_triplet_bwd_basis_ex": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p, _p, _i32, _i32, _i32, _f64, _i32, _i32, _p, _p,
                                        _p, _p, _p, _p]),
    "egn_rbf_bessel": (_i32, [_p, _i64, _i32, _f64, _p, _p]),
    "egn_rbf_bessel_bwd": (_i32, [_p, _p, _i64, _i32, _f64, _p, _p]),
    "egn_triplet_fwd_window": (_i32, [_p, _p, _p, _i64, _i64, _i64, _p, _p, _i32, _i32, _i32, _f64, _p, _p]),
    "egn_triplet_bwd_window": (_i32, [_p, _p, _p, _i64, _i64, _i64, _i32, _p, _p, _i32, _i32, _i32, _f64, _p, _p,
                                      _p, _p, _p, _p]),
    "egn_graph_linear": (_i32, [_i64, _i32, _i32, _p, _p, _p, _p, _p]),
    "egn_graph_linear_bwd": (_i32, [_i64, _i32, _i32, _p, _p, _p, _p, _p, _p, _p]),
    "egn_rbf_features": (_i32, [_p, _i64, _i32, _f64, _p, _p, _p, _p]),
    "egn_sbf_features": (_i32, [_p, _p, _i64, _i32, _i32, _f64, _p, _p, _p, _p, _p]),
    "egn_geometry_grads": (_i32, [_p, _p, _p, _i64, _p, _p, _i64, _p, _p, _p, _p, _p, _p]),
    "egn_triplet_terms": (_i32, [_p, _p, _p, _p, _i64, _p, _p, _i32, _i32, _i32, _f64, _p, _p]),
    "egn_aggregate_in_edges": (_i32, [_p, _p, _i64, _p, _i64, _i32, _p, _p]),
    "egn_gather_rows": (_i32, [_p, _i64, _p, _i64, _i32, _p, _i64, _i32, _p]),
    "egn_scatter_rows": (_i32, [_p, _p, _i64, _p, _i64, _i32, _p, _i64, _i32, _p]),
    "egn_graph_sum": (_i32, [_p, _i64, _p, _i32, _p, _p]),
    "egn_force_head_fwd": (_i32, [_p, _p, _p, _i64, _i64, _p, _i32, _p, _p, _p, _p]),
    "egn_force_head_bwd_workspace_bytes": (_i64, [_i64, _i32]),
    "egn_force_head_bwd": (_i32, [_p, _p, _i64, _p, _i32, _p, _p, _p, _p, _p, _p, _p, _p]),
    "egn_rbf_linear": (_i32, [_p, _i64, _i32, _p, _p, _i32, _p, _i64, _p]),
    "egn_rbf_linear_bwd_workspace_bytes": (_i64, [_i64, _i32, _i32]),
    "egn_rbf_linear_bwd": (_i32, [_p, _i64, _i32, _p, _i32, _p, _p, _i64, _p, _p, _p, _p, _p]),
    "egn_rbf_bwd": (_i32, [_p, _p, _i64, _i32, _f64, _p, _p]),
    "egn_positions_bwd": (_i32, [_p, _p, _p, _i64, _p, _p, _p]),
    "egn_column_sum_workspace_bytes": (_i64, [_i64, _i32]),
    "egn_column_sum": (_i32, [_p, _i64, _i32, _i64, _p, _p, _p]),
    "egn_gemm": (_i32, [_i64, _i32, _i32, _p, _i64, _p, _i64, _i32, _p, _i64, _p, _i64, _i32, _p, _p, _i64, _p,
                        _p, _i64, _p, _i64, _i32, _p, _i64, _p, _i64, _i32, _p]),
    "egn_gemm_blo": (_i32, [_i64, _i32, _i32, _p, _i64, _p, _i64, _i32, _p, _i64, _p, _i64, _i32, _p, _p, _i64, _p,
                            _p, _i64, _p, _i64, _i32, _p, _i64, _p, _i64, _i32, _p, _i64, _p, _i64, _p]),
    "egn_tf32_lo": (_i32, [_p, _i64, _i32, _i64, _p, _i64, _p]),
    "egn_gemm_wgrad_workspace_bytes": (_i64, [_i64, _i32, _i32]),
    "egn_gemm_wgrad": (_i32, [_i64, _i32, _i32, _p, _i64, _p, _i64, _p, _i64, _p, _i32, _p, _p]),
    "egn_small_gemm_batched": (_i32, [_p, _i32, _p]),
    "egn_sgd": (_i32, [_p, _p, _i64, _f32, _p]),
    "egn_zero": (_i32, [_p, _i64, _p]),
    "egn_hadamard": (_i32, [_p, _p, _p, _i64, _p]),
    "egn_transpose": (_i32, [_p, _i64, _i64, _i64, _p, _i64, _p]),
    "egn_csr_ptr": (_i32, [_p, _i64, _i64, _p, _p]),
}


class EgnNativeError(RuntimeError):
    """A C-ABI call returned a nonzero status."""


_LIB = None


def lib() -> ctypes.CDLL:
    """Load the native library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                "there is no CPU fallback for the EGN hot path"
            )
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("EGN kernels take CUDA tensors only (no CPU fallback)")
    return t.data_ptr()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# Kernels launched per successful ABI call (for the bench's gpu_launches count).
KERNELS_PER_CALL = {
    "egn_triplet_bwd": 4, "egn_triplet_bwd_ex": 2, "egn_triplet_fwd": 2, "egn_triplet_fwd_basis": 3, "egn_triplet_bwd_basis": 4, "egn_triplet_bwd_basis_ex": 2, "egn_triplet_bwd_window": 2, "egn_graph_linear_bwd": 2, "egn_geometry_grads": 2, "egn_force_head_fwd": 2, "egn_force_head_bwd": 2, "egn_column_sum": 2, "egn_gemm_wgrad": 2, "egn_rbf_linear_bwd": 2, "egn_graph_mlp_fwd": 2, "egn_graph_mlp_bwd": 3, "egn_cap_keep": 2, "egn_cap_compact": 2,
}
LAUNCH_COUNTER = {"calls": 0, "kernels": 0}
_NOT_LAUNCHES = {"egn_triplet_path", "egn_abi_version"}
_NO_KERNEL = {"egn_zero"}  # a memset: checked, not counted as a kernel


def call(name: str, *args) -> int:
    """Invoke an ABI function; raise EgnNativeError with the library message on failure."""
    fn = getattr(lib(), name)
    rc = fn(*args)
    if (SIGNATURES[name][0] is _i32 and not name.endswith("_bytes") and name not in _NOT_LAUNCHES
            and name not in _NO_KERNEL):
        LAUNCH_COUNTER["calls"] += 1
        LAUNCH_COUNTER["kernels"] += KERNELS_PER_CALL.get(name, 1)
    if SIGNATURES[name][0] is _i32 and rc != 0 and name not in _NOT_LAUNCHES:
        msg = lib().egn_last_error().decode(errors="replace")
        if rc == 2:
            raise ValueError(f"{name}: {msg}")
        raise EgnNativeError(f"{name} failed ({rc}): {msg}")
    return rc


def exported_symbols() -> list[str]:
    return [n for n in SIGNATURES]


def header_symbols() -> list[str]:
    """Function names declared in include/egn_b200.h (for the ABI coverage test)."""
    import re

    text = (_HERE.parent / "include" / "egn_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|int)\s+(egn_\w+)\s*\(", text, re.M)))


def env_flag(name: str) -> bool:
    return os.environ.get(name, "0") not in ("", "0", "false", "False")
