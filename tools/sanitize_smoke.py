"""Tiny end-to-end run of every CUDA entry point, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_06218_b200 import dmha  # noqa: E402

dmha.init(1, 0, None, 0, "bf16", "contiguous")
for D in (64, 128):
    for causal in (False, True):
        L, H = 300, 2
        q, k, v = (torch.randn(L, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
        dmha.forward(q, k, v, L, causal)
        for kern in ("cluster", "pair"):
            if kern == "pair" and D != 128:
                continue
            os.environ["DMHA_KERNEL"] = kern
            dmha.forward(q, k, v, L, causal)
        os.environ.pop("DMHA_KERNEL", None)
P, L, H, D = 2, 512, 2, 64
q, k, v = (torch.randn(P, L // P, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
dmha.forward_emulated(P, "zigzag", q, k, v, L, True)
dmha.forward_headpar_emulated(P, "zigzag", q, k, v, L, True)
torch.cuda.synchronize()
dmha.finalize()
dmha.init(1, 0, None, 0, "fp32", "contiguous")
q, k, v = (torch.randn(128, 2, 64, device="cuda") for _ in range(3))
dmha.forward(q, k, v, 128, True)
torch.cuda.synchronize()
dmha.finalize()
print("sanitize smoke done")
