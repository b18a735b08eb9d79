"""Per-step measurements of the hot path on one GPU.

    python tools/bench_steps.py [--out profiles/r01_steps.json]

a2  attention kernel: TFLOP/s per config (C2, C2 causal, C3@P=1, C4@P=1, C5@P=1),
    CUDA-event timed on the launch stream; the fp32 path (3xTF32) at C1 and
    at C2's shape
NEXT-1 head-parallel pack/unpack kernels: HBM GB/s (library profiling events)
NEXT-3 projection GEMM (tcgen05): TFLOP/s at the layer's shapes
a4  LSE combine kernel: HBM GB/s (12 B/elem + 12 B/row) at C4 P=8 shard size
a1+a2+a4 through the single-GPU ring emulation (P = 2, 4, 8) at C3 size:
    the per-rank compute of the real ring without NCCL (the exchange step,
    a3, needs >1 GPU and is not measurable here)
Each line also records the SM clock seen during the run.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2302_06218_b200 import dmha  # noqa: E402

PEAKS = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {
    "hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def time_cuda(fn, iters=5, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def attn_flops(L, D, H, causal):
    f = 4.0 * L * L * D * H
    return f / 2 if causal else f


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "steps.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    res = {"gpu": torch.cuda.get_device_name(0), "peaks": PEAKS, "a2_attention": [], "a4_combine": [],
           "ring_emulated": []}
    dmha.init(1, 0, None, 0, "bf16", "contiguous")
    configs = [("C2", 16384, 64, 8, False), ("C2c", 16384, 64, 8, True), ("C3@P1", 131072, 128, 8, False),
               ("C4@P1", 262144, 128, 16, False), ("C5@P1", 1048576, 64, 16, True)]
    if args.quick:
        configs = configs[:3]
    for name, L, D, H, causal in configs:
        q, k, v = (torch.randn(L, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
        out = torch.empty_like(q)
        lse = torch.empty(H, L, device="cuda")
        for kern in ("default",):
            iters = 2 if L >= 262144 else 10
            ms = time_cuda(lambda: dmha.forward(q, k, v, L, causal, out, lse), iters=iters, warmup=2)
            tf = attn_flops(L, D, H, causal) / ms / 1e9
            res["a2_attention"].append({"config": name, "kernel": kern, "L": L, "D": D, "H": H, "causal": causal,
                                        "ms": ms, "tflops": tf,
                                        "frac_sustained": tf / PEAKS["bf16_tflops_sustained"],
                                        "frac_burst": tf / PEAKS["bf16_tflops"], "frac_datasheet": tf / 2250.0})
            print(json.dumps(res["a2_attention"][-1]), flush=True)
        del q, k, v, out, lse
        torch.cuda.empty_cache()

    dmha.finalize()
    # fp32 path (3xTF32 tcgen05): C1 and C2's shape in fp32
    res["fp32_path"] = []
    dmha.init(1, 0, None, 0, "fp32", "contiguous")
    for name, L, D, H, causal in (("C1", 512, 64, 4, False), ("C2-fp32", 16384, 64, 8, False)):
        q, k, v = (torch.randn(L, H, D, device="cuda") for _ in range(3))
        out = torch.empty_like(q)
        lse = torch.empty(H, L, device="cuda")
        ms = time_cuda(lambda: dmha.forward(q, k, v, L, causal, out, lse), iters=10)
        tf = attn_flops(L, D, H, causal) / ms / 1e9
        rec = {"config": name, "L": L, "D": D, "H": H, "ms": ms, "tflops": tf,
               "frac_tf32_datasheet_1125": tf / 1125.0,
               "note": "3xTF32: 3 tensor-core passes per GEMM (counted once, algorithmic FLOP)"}
        res["fp32_path"].append(rec)
        print(json.dumps(rec), flush=True)
    dmha.finalize()
    dmha.init(1, 0, None, 0, "bf16", "contiguous")

    # NEXT-3 projection GEMM: x [L_loc, d_model] @ W [d_model, H*D]
    res["gemm"] = []
    for M, N, K in ((32768, 2048, 2048), (131072, 2048, 2048), (262144, 2048, 2048), (16384, 1024, 1024)):
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(K, N, device="cuda") / K ** 0.5).to(torch.bfloat16)
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ms = time_cuda(lambda: dmha.linear(x, w, y), iters=20)
        tf = 2.0 * M * N * K / ms / 1e9
        ms_cb = time_cuda(lambda: torch.matmul(x, w, out=y), iters=20)
        rec = {"M": M, "N": N, "K": K, "ms": ms, "tflops": tf,
               "frac_sustained": tf / PEAKS["bf16_tflops_sustained"], "frac_burst": tf / PEAKS["bf16_tflops"],
               "context_torch_matmul_tflops": 2.0 * M * N * K / ms_cb / 1e9}
        res["gemm"].append(rec)
        print(json.dumps(rec), flush=True)
        del x, w, y

    # NEXT-1 pack/unpack kernels (head-parallel exchange) at C4 P=8 / C5 P=8 shard sizes
    res["headpar_pack"] = []
    for L, D, H, P, layout in ((262144, 128, 16, 8, "contiguous"), (1 << 20, 64, 16, 8, "zigzag")):
        Ll = L // P
        q, k, v = (torch.randn(P, Ll, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
        out = torch.empty_like(q)
        lse = torch.empty(P, H, Ll, device="cuda")
        dmha.forward_headpar_emulated(P, layout, q, k, v, L, layout == "zigzag", out, lse)
        torch.cuda.synchronize()
        dmha.set_profiling(True)
        dmha.forward_headpar_emulated(P, layout, q, k, v, L, layout == "zigzag", out, lse)
        torch.cuda.synchronize()
        st = dmha.get_stats()
        dmha.set_profiling(False)
        gbs = st["pack_bytes"] / (st["pack_ms"] / 1e3) / 1e9
        rec = {"L": L, "D": D, "H": H, "P": P, "layout": layout, "launches": st["pack_launches"],
               "ms_total": st["pack_ms"], "bytes": st["pack_bytes"], "gbs": gbs,
               "frac_hbm": gbs / PEAKS["hbm_gbs"]}
        res["headpar_pack"].append(rec)
        print(json.dumps(rec), flush=True)
        del q, k, v, out, lse
        torch.cuda.empty_cache()

    # a4: combine kernel at C4 P=8 shard size (L_loc = 32768, H = 16, D = 128)
    for (Lq, H, D) in ((32768, 16, 128), (131072, 16, 64)):
        oa, op = (torch.randn(Lq, H, D, device="cuda") for _ in range(2))
        la, lp = (torch.randn(H, Lq, device="cuda") for _ in range(2))
        out = torch.empty(Lq, H, D, device="cuda", dtype=torch.bfloat16)
        lo = torch.empty(H, Lq, device="cuda")
        ms = time_cuda(lambda: dmha.lse_combine(oa, la, op, lp, final=False), iters=20)
        by = 12.0 * Lq * H * D + 12.0 * Lq * H
        ms_f = time_cuda(lambda: dmha.lse_combine(oa, la, op, lp, out, lo, final=True), iters=20)
        by_f = 10.0 * Lq * H * D + 12.0 * Lq * H
        rec = {"Lq": Lq, "H": H, "D": D, "ms_accumulate": ms, "gbs_accumulate": by / ms / 1e6,
               "ms_final_bf16": ms_f, "gbs_final_bf16": by_f / ms_f / 1e6, "hbm_peak_gbs": PEAKS["hbm_gbs"]}
        rec["frac_accumulate"] = rec["gbs_accumulate"] / PEAKS["hbm_gbs"]
        res["a4_combine"].append(rec)
        print(json.dumps(rec), flush=True)
        del oa, op, la, lp, out, lo

    # NEXT-4 selector: X = C5's P=8 shard as rows of width H*D (131072 x 1024
    # bf16, 256 MiB) and C4's P=1 (262144 x 2048), tau at the median score
    res["selector"] = []
    for n, w in ((131072, 1024), (262144, 2048)):
        x = torch.randn(n, w, device="cuda").to(torch.bfloat16)
        xo = torch.empty_like(x)
        idx = torch.empty(n, dtype=torch.int64, device="cuda")
        sc = torch.empty(n, dtype=torch.float64, device="cuda")
        _, kept, _ = dmha.select(x, 0.0, "l2", None, xo, idx, sc)
        tau = float(sc.median())
        kept_n = [0]

        def run():
            kept_n[0] = dmha.select(x, tau, "l2", None, xo, idx, sc)[1].shape[0]
        ms = time_cuda(run, iters=10)
        k = kept_n[0]
        by = n * w * 2 + 2 * k * w * 2 + 8 * n + n + 8 * k  # score read, row copy r+w, scores, flags, idx
        rec = {"n": n, "width": w, "kept": k, "ms": ms, "gbs": by / ms / 1e6,
               "frac_hbm": by / ms / 1e6 / PEAKS["hbm_gbs"], "note": "includes the host sync for n_kept"}
        res["selector"].append(rec)
        print(json.dumps(rec), flush=True)
        del x, xo, idx, sc

    # whole per-rank ring compute through the emulation (C3 size P = 2, 4, 8;
    # C4 P = 8), with the NEXT-2 fused combine (default) and the separate pass
    cases = [(131072, 128, 8, P) for P in (2, 4, 8)] + [(262144, 128, 16, 8), (1 << 20, 64, 16, 8)]
    for L, D, H, P in cases:
        for layout, causal in (("contiguous", False), ("zigzag", True)):
            if L == 262144 and causal:
                continue
            if L == (1 << 20) and not causal:  # C5 is causal, zigzag
                continue
            Ll = L // P
            q, k, v = (torch.randn(P, Ll, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
            out = torch.empty_like(q)
            lse = torch.empty(P, H, Ll, device="cuda")
            for fused in ("1", "0"):
                os.environ["DMHA_FUSED_COMBINE"] = fused
                ms = time_cuda(lambda: dmha.forward_emulated(P, layout, q, k, v, L, causal, out, lse),
                               iters=3 if L < 262144 else (2 if L < (1 << 20) else 1), warmup=1)
                tf = attn_flops(L, D, H, causal) / ms / 1e9  # all P ranks' work, serialised on one GPU
                rec = {"P": P, "layout": layout, "causal": causal, "L": L, "D": D, "H": H,
                       "fused_combine": fused == "1", "ms_all_ranks_serial": ms, "tflops_serial": tf,
                       "projected_ms_per_rank_if_perfectly_parallel": ms / P}
                res["ring_emulated"].append(rec)
                print(json.dumps(rec), flush=True)
            os.environ.pop("DMHA_FUSED_COMBINE", None)
            del q, k, v, out, lse
            torch.cuda.empty_cache()
    dmha.finalize()
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
