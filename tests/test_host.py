"""Host-side logic on CPU: config, parameters, partitions, comm model, C-ABI symbols."""

import json
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle import egn_oracle as O
from paper_2203_09697_b200 import (CommModel, ModelConfig, comm_volume, init_params, load_params,
                                   param_specs, partition_centers, save_params, split_range)


def test_config_validation_and_json_roundtrip():
    c = ModelConfig(variant="gemnet-style", blocks=3, d_e=16)
    assert ModelConfig.from_json(c.to_json()) == c
    with pytest.raises(ValueError):
        ModelConfig(variant="bogus")
    with pytest.raises(ValueError):
        ModelConfig(d_t=0)
    with pytest.raises(ValueError):
        ModelConfig(cutoff=0.0)
    with pytest.raises(ValueError):
        ModelConfig.from_json(json.dumps({"bogus": 1}))
    assert c.triplet_width == c.d_bil and ModelConfig().triplet_width == ModelConfig().d_t


def test_config_basis_selection():
    """basis="bessel" selects the DimeNet++ / GemNet-T bases (native code 2 / 1); the
    reference's Gaussian surrogate stays the default and keeps the reference's JSON keys."""
    assert ModelConfig().basis_code == 0 and "basis" not in json.loads(ModelConfig().to_json())
    d = ModelConfig(variant="dimenet-style", k_rbf=6, l_sbf=7, basis="bessel")
    g = ModelConfig(variant="gemnet-style", k_rbf=6, l_sbf=7, basis="bessel")
    assert (d.basis_code, g.basis_code) == (2, 1)
    assert ModelConfig.from_json(g.to_json()) == g
    with pytest.raises(ValueError, match="k_rbf = 6 and l_sbf = 7"):
        ModelConfig(k_rbf=8, l_sbf=7, basis="bessel")
    with pytest.raises(ValueError, match="basis must be"):
        ModelConfig(basis="legendre")


@pytest.mark.parametrize("fname", ["model_dimenet_small.npz", "model_gemnet_odd.npz", "model_gemnet_c2dims.npz"])
def test_init_params_matches_reference_checksums(fname):
    gd = load_golden(fname)
    cfg = ModelConfig.from_json(str(gd["config"]))
    p = init_params(cfg)
    assert [s.name for s in param_specs(cfg)] == [str(n) for n in gd["param_names"]]
    np.testing.assert_array_equal([float(np.sum(a)) for a in p.arrays.values()], gd["param_checksum"])


def test_param_specs_match_oracle():
    for variant in ("dimenet-style", "gemnet-style"):
        cfg = ModelConfig(variant=variant, blocks=2, d_bil=5)
        oc = O.Config(**{k: getattr(cfg, k) for k in O.Config.__dataclass_fields__})
        assert [(s.name, s.shape, s.fan_in) for s in param_specs(cfg)] == O.param_specs(oc)


def test_egn1_container_roundtrip(tmp_path):
    cfg = ModelConfig(variant="gemnet-style", blocks=2)
    p = init_params(cfg)
    save_params(p, tmp_path / "w.egn")
    q = load_params(tmp_path / "w.egn", cutoff=cfg.cutoff)
    assert q.config == cfg
    for k in p.arrays:
        np.testing.assert_array_equal(p.arrays[k], q.arrays[k])
    blob = (tmp_path / "w.egn").read_bytes()
    (tmp_path / "bad.egn").write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(ValueError):
        load_params(tmp_path / "bad.egn")
    (tmp_path / "trunc.egn").write_bytes(blob[:-8])
    with pytest.raises(ValueError):
        load_params(tmp_path / "trunc.egn")


def test_split_range_and_comm_volume_known_answers():
    assert [s.size for s in split_range(7, 3)] == [3, 2, 2]
    assert comm_volume(CommModel(10, 40, 999, 4, 8, 16, 1, "dimenet-style"), 1).per_block == 361
    assert comm_volume(CommModel(10, 40, 999, 4, 8, 16, 1, "gemnet-style"), 1).per_block == 681
    m = CommModel(5, 12, 50, 3, 4, 2, 2, "gemnet-style")
    assert comm_volume(m, 4).total == 4 * comm_volume(m, 1).per_block


@pytest.mark.parametrize("workers", [1, 2, 3, 4, 8])
def test_partition_centers_contiguous_and_balanced(workers):
    rng = np.random.default_rng(workers)
    deg = rng.integers(0, 60, size=500)
    part = partition_centers(deg, workers)
    assert part.node_bounds[0] == 0 and part.node_bounds[-1] == deg.size
    assert np.all(np.diff(part.node_bounds) >= 0)
    edge_ptr = np.concatenate([[0], np.cumsum(deg)])
    tri_ptr = np.concatenate([[0], np.cumsum(deg * (deg - 1))])
    np.testing.assert_array_equal(part.edge_bounds, edge_ptr[part.node_bounds])
    np.testing.assert_array_equal(part.trip_bounds, tri_ptr[part.node_bounds])
    cost = deg * (deg - 1) + deg
    per = [cost[part.node_bounds[r]:part.node_bounds[r + 1]].sum() for r in range(workers)]
    assert max(per) - min(per) <= 2 * cost.max()


def test_abi_header_lists_every_bound_symbol():
    from paper_2203_09697_b200 import _lib

    header = set(_lib.header_symbols())
    bound = set(_lib.SIGNATURES)
    assert header == bound, (header ^ bound)


def test_native_library_loads_and_exports_all_symbols():
    """No GPU needed: dlopen the built library and resolve every declared entry point."""
    from paper_2203_09697_b200 import _lib

    if not _lib.LIB_PATH.exists():
        pytest.skip("libegn_b200.so not built (run make)")
    lib = _lib.lib()
    for name in _lib.header_symbols():
        assert hasattr(lib, name), name
    assert lib.egn_abi_version() == 3
    assert isinstance(lib.egn_last_error(), bytes)
    # pure host entry point: workspace sizing
    assert lib.egn_triplet_bwd_workspace_bytes(1000, 20000, 40, 6, 7, 64) > 0


def test_product_path_does_not_import_oracle():
    pkg = ROOT / "paper_2203_09697_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), f
        assert "egn_oracle" not in text, f


def test_torch_custom_ops_registered_with_fake_kernels():
    """torch.ops.egn.* exist and their fake (meta) implementations give shapes without a GPU
    (FakeTensor tracing / torch.compile see them as opaque graph nodes)."""
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode

    import paper_2203_09697_b200.torch_ops as T

    names = {"rbf", "rbf_linear", "linear", "triplet_fwd", "triplet_bwd", "aggregate_in_edges", "gather_rows",
             "graph_sum", "force_head", "positions_bwd", "energy_forces", "energy_forces_backward"}
    assert names <= set(dir(torch.ops.egn))
    with FakeTensorMode():
        E, V, dg = 50, 7, 16
        geo = torch.empty((E, 4))
        X = torch.empty((E, dg))
        Wk = torch.empty((6, 7, dg))
        ep = torch.empty(V + 1, dtype=torch.int64)
        rev = torch.empty(E, dtype=torch.int32)
        assert torch.ops.egn.rbf(geo, 6, 6.0).shape == (E, 6)
        assert torch.ops.egn.triplet_fwd(ep, rev, geo, X, Wk, 6.0, 10).shape == (E, dg)
        xb, wb = torch.ops.egn.triplet_bwd(ep, rev, geo, X, Wk, 6.0, X, torch.empty((E, 4)), 10)
        assert xb.shape == X.shape and wb.shape == Wk.shape
        assert torch.ops.egn.linear(X, torch.empty((32, dg))).shape == (E, 32)
        assert torch.ops.egn.linear(X, torch.empty((dg, 8)), w_mn=True).shape == (E, 8)
        assert torch.ops.egn.aggregate_in_edges(ep, rev, X).shape == (V, dg)
        assert torch.ops.egn.positions_bwd(ep, rev, geo, torch.empty((E, 4))).dtype == torch.float64
        s, f = torch.ops.egn.force_head(ep, rev, geo, X, torch.empty(dg))
        assert s.shape == (E,) and f.shape == (V, 3)


def test_bench_reference_arm_contract():
    """bench.py --impl reference on the host (no GPU): one JSON line with the contract keys the
    driver reads (impl, metric, value, unit, e2e, cpu_baseline with cores / kind / sample)."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--workload",
                          "dimenet-pp-small", "--steps", "1", "--warmup", "0", "--graphs", "1"],
                         capture_output=True, text=True, timeout=600, cwd=str(root))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["metric"].startswith("triplet-interactions/s") and line["unit"] == "triplets/s"
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == line["value"]
