"""Run one large fused GEMM a few times (ncu target).  python tools/gemm_one.py [fwd|dgrad|wgrad]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2203_09697_b200 import ops  # noqa: E402
kind = sys.argv[1] if len(sys.argv) > 1 else "fwd"
a = torch.randn((58644, 128), device="cuda")
w = torch.randn((128, 128), device="cuda")
r = torch.randn((58644, 128), device="cuda")
fn = {"fwd": lambda: ops.gemm(a, w, resid=r), "dgrad": lambda: ops.gemm(a, w, b_mn=True),
      "wgrad": lambda: ops.gemm_wgrad(r, a)}[kind]
for _ in range(3):
    fn()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    fn()
e.record()
torch.cuda.synchronize()
print("gemm 58644x128x128 %s: %.1f us" % (kind, s.elapsed_time(e) * 100))
