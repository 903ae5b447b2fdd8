"""Probe the tcgen05 GEMM variants on small shapes (NaN-prefilled outputs, explicit sync)."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2203_09697_b200 import ops  # noqa: E402


def show(name, out, ref):
    torch.cuda.synchronize()
    o = out.double()
    print(f"{name:28s} nan={torch.isnan(o).sum().item():6d} zero={int((o == 0).sum())} "
          f"maxerr={float((o - ref).abs().nan_to_num(1e9).max()):.3e} refmax={float(ref.abs().max()):.3e}")
    print("   out[0,:6]", [round(x, 4) for x in o[0, :6].tolist()], " ref[0,:6]", [round(x, 4) for x in ref[0, :6].tolist()])


M, N, K = 128, 64, 32
a = torch.randn((M, K), device="cuda")
w = torch.randn((N, K), device="cuda")
out = torch.full((M, N), float("nan"), device="cuda")
ops.gemm(a, w, out=out)
show("K-major", out, a.double() @ w.double().t())
wt = w.t().contiguous()  # [K, N]
out = torch.full((M, N), float("nan"), device="cuda")
ops.gemm(a, wt, out=out, b_mn=True)
show("B MN-major", out, a.double() @ wt.double())
g = torch.randn((256, 128), device="cuda")
x = torch.randn((256, 64), device="cuda")
out = torch.full((128, 64), float("nan"), device="cuda")
ops.gemm_wgrad(g, x, out=out)
show("wgrad", out, g.double().t() @ x.double())
print(torch.cuda.synchronize(), "sync ok")
