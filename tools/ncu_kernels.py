"""Run ONE of the secondary kernels a few times so ncu can capture it alone.

  python tools/ncu_kernels.py tf32      # 3xTF32 attention, C2's shape in fp32
  python tools/ncu_kernels.py gemm      # NEXT-3 projection GEMM (C4 row count, 128 -> 3*128)
  python tools/ncu_kernels.py headpar   # NEXT-1 pack/unpack at C4, P=8 (emulated exchange)
  python tools/ncu_kernels.py combine   # a4 separate LSE combine at a C4 P=8 shard

Used by tools/gpu_runs/gpu_r2z.sh as `ncu --set full -k regex:<kernel> -s 2 -c 1 python tools/ncu_kernels.py X`.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2302_06218_b200 import dmha  # noqa: E402


def main():
    what = sys.argv[1]
    torch.manual_seed(0)
    if what == "tf32":
        dmha.init(1, 0, None, 0, "fp32", "contiguous")
        L, H, D = 16384, 8, 64
        q, k, v = (torch.randn(L, H, D, device="cuda") for _ in range(3))
        out, lse = torch.empty_like(q), torch.empty(H, L, device="cuda")
        for _ in range(4):
            dmha.forward(q, k, v, L, False, out, lse)
    elif what == "gemm":
        dmha.init(1, 0, None, 0, "bf16", "contiguous")
        M, K, N = 262144, 2048, 3 * 2048
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for _ in range(4):
            dmha.linear(x, w, y)
    elif what == "headpar":
        dmha.init(1, 0, None, 0, "bf16", "contiguous")
        P, L, H, D = 8, 262144, 16, 128
        q, k, v = (torch.randn(P, L // P, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
        out, lse = None, None
        for _ in range(2):
            out, lse = dmha.forward_headpar_emulated(P, "contiguous", q, k, v, L, False, out, lse)
    elif what == "combine":
        dmha.init(1, 0, None, 0, "bf16", "contiguous")
        rows, H, D = 262144 // 8, 16, 128
        acc = torch.randn(rows, H, D, device="cuda")
        part = torch.randn(rows, H, D, device="cuda")
        la, lp = torch.randn(H, rows, device="cuda"), torch.randn(H, rows, device="cuda")
        for _ in range(4):
            dmha.lse_combine(acc, la, part, lp)
    else:
        raise SystemExit(f"unknown kernel family {what}")
    torch.cuda.synchronize()
    dmha.finalize()


if __name__ == "__main__":
    main()
