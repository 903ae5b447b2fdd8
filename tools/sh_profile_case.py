"""One forward + backward of the triplet kernels on a C5-style graph (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_09697_b200 import _lib, ops  # noqa: E402
from paper_2203_09697_b200.graph import build_batch  # noqa: E402

deg = int(sys.argv[1]) if len(sys.argv) > 1 else 500
dg = int(sys.argv[2]) if len(sys.argv) > 2 else 64
path = {"auto": 0, "sh": 1, "pairwise": 2}[sys.argv[3] if len(sys.argv) > 3 else "sh"]
_lib.call("egn_triplet_path", path)
cutoff, n = 6.0, 1000
rho = (deg + 1) / (4.0 / 3.0 * np.pi * cutoff ** 3)
pos = np.random.default_rng(deg).uniform(0.0, (n / rho) ** (1 / 3), size=(n, 3))
bg = build_batch([pos], cutoff)
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((bg.num_edges, dg), device="cuda", generator=g)
W = torch.randn((6, 7, dg), device="cuda", generator=g) / 6.5
Sb = torch.randn((bg.num_edges, dg), device="cuda", generator=g)
eg = torch.zeros((bg.num_edges, 4), device="cuda")
md = int(bg.deg.max())
for _ in range(2):
    ops.triplet_fwd(bg.edge_ptr, bg.rev, bg.geo, X, W, cutoff, md)
    ops.triplet_bwd(bg.edge_ptr, bg.rev, bg.geo, X, W, cutoff, Sb, eg, max_degree=md)
torch.cuda.synchronize()
print("ok", bg.num_edges, md)
