"""Run one large fused GEMM a few times (ncu target)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2203_09697_b200 import ops  # noqa: E402
a = torch.randn((58644, 128), device="cuda")
w = torch.randn((128, 128), device="cuda")
r = torch.randn((58644, 128), device="cuda")
for _ in range(3):
    ops.gemm(a, w, resid=r)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    ops.gemm(a, w, resid=r)
e.record()
torch.cuda.synchronize()
print("gemm 58644x128x128 resid: %.1f us" % (s.elapsed_time(e) * 100))
