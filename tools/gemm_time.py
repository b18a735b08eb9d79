"""Time the NEXT-3 tcgen05 GEMM (dmha_linear) at the layer shapes: CUDA events,
TF/s and the clock (A/B helper; DMHA_LIB selects a variant build)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2302_06218_b200 import dmha  # noqa: E402

dmha.init(1, 0, None, 0, "bf16", "contiguous")
for M, K, N in ((262144, 2048, 6144), (262144, 2048, 2048), (65536, 2048, 2048)):
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        dmha.linear(x, w, y)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    n = 20
    for _ in range(n):
        dmha.linear(x, w, y)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    print(f"M={M} K={K} N={N}: {ms:.3f} ms  {2 * M * K * N / ms / 1e9:.0f} TF/s")
dmha.finalize()
