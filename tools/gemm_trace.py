"""Print the CTA-0 role timeline (ns) of one tcgen05 GEMM launch per shape (EGN_GEMM_TRACE)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2203_09697_b200 import ops  # noqa: E402

E = 58644
a = torch.randn((E, 128), device="cuda")
w = torch.randn((128, 128), device="cuda")
r = torch.randn((E, 128), device="cuda")
g = torch.randn((E, 128), device="cuda")
import time  # noqa: E402
x = torch.randn((4096, 4096), device="cuda")
t0 = time.time()
while time.time() - t0 < 2.0:  # bring the SM clock to boost
    for _ in range(20):
        x = (x @ x).tanh_()
    torch.cuda.synchronize()
for _ in range(3):
    ops.gemm(a, w, resid=r)
    ops.gemm(a, w, b_mn=True)
torch.cuda.synchronize()
os.environ["EGN_GEMM_TRACE"] = "1"
bias = torch.randn((128,), device="cuda")
for name, fn in (("silu2 bias", lambda: ops.gemm(a, w, bias=bias, flags=ops.EPI_SILU_OUT2)),
                 ("dgrad (no operand)", lambda: ops.gemm(a, w, b_mn=True)),
                 ("fwd resid", lambda: ops.gemm(a, w, resid=r)),
                 ("wgrad", lambda: ops.gemm_wgrad(g, a))):
    print("==", name, flush=True)
    fn()
    torch.cuda.synchronize()
    os.environ.pop("EGN_GEMM_TRACE")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    fn()
    ev[1].record()
    fn()
    fn()
    fn()
    ev[2].record()
    torch.cuda.synchronize()
    print(f"   one call {ev[0].elapsed_time(ev[1]) * 1000:.1f} us, three calls {ev[1].elapsed_time(ev[2]) * 1000:.1f} us",
          flush=True)
    os.environ["EGN_GEMM_TRACE"] = "1"
