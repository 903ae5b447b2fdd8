"""CTA-0 role timeline (EGN_GEMM_TRACE) of one XL-width GEMM launch (14,792 x 2048 x 2048 by default):
the per-k-block hand-off times of the producer / split / MMA roles in the long-K steady state.

    python tools/gemm_trace_xl.py [M N K]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2203_09697_b200 import ops  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (14792, 2048, 2048)
a = torch.randn((M, K), device="cuda")
w = torch.randn((N, K), device="cuda")
for _ in range(3):
    ops.gemm(a, w)
torch.cuda.synchronize()
os.environ["EGN_GEMM_TRACE"] = "1"
ops.gemm(a, w)
torch.cuda.synchronize()
