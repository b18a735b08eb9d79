"""Maximum sequence length per SURVEY §8(d) (BASELINE.json metric "max seq len").

    python tools/max_len.py [--cap-s 300] [--out gpurun_out/max_len.json]

For each family — (D=128, H=16, non-causal) and (D=64, H=16, causal) — at
P = 1 on this GPU: double L from 2^16 running a FULL dmha_forward each time
(CUDA-event timed), until the next doubling would exceed either the HBM
capacity bound or the per-forward time cap (300 s).  Then refine once: the
largest multiple of 256 below both bounds, predicted from the last measured
forward (time ~ L^2), is run in full and must finish under the cap.  Each
L_max is reported as "time-bound" or "capacity-bound".

Every run is checked by a closed form that holds at any size:
a few sampled query rows are set to zero, so their output is the mean of the
V rows they may see (causal: the prefix 0..g) and their lse is ln(#keys);
the means are accumulated in fp64 on the device from the same bf16 V.

P > 1 figures are capacity-derived (H*(20*D+8) bytes per local token with the
fused combine, dmha_ring_workspace_bytes) and labelled so: one GPU per call.
Paper context: ~2K vanilla on 1x RTX 3090, ~80K distributed on 4x RTX 3090
(P:679).
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2302_06218_b200 import dmha  # noqa: E402

N_ZERO_ROWS = 12


def bytes_per_token_p1(D, H):
    return H * (8 * D + 4)  # q, k, v, out (bf16) + lse (fp32); no workspace at P = 1


def zero_rows(L, seed):
    g = torch.Generator().manual_seed(seed)
    r = set(torch.randint(0, L, (N_ZERO_ROWS - 3,), generator=g).tolist()) | {0, L // 2, L - 1}
    return sorted(r)


def closed_form_check(v, out, lse, rows, causal):
    """Zero query rows: out = mean of the visible V rows, lse = ln(#visible)."""
    L, H, D = v.shape
    acc = torch.zeros((H, D), dtype=torch.float64, device=v.device)
    total = None
    if not causal:
        for s in range(0, L, 1 << 16):
            acc += v[s:s + (1 << 16)].double().sum(0)
        total = acc / L
    max_abs, max_lse = 0.0, 0.0
    pos = 0
    for g in rows:
        if causal:  # prefix 0..g
            while pos <= g:
                e = min(g + 1, (pos // (1 << 16) + 1) << 16)
                acc += v[pos:e].double().sum(0)
                pos = e
            ref, n = acc / (g + 1), g + 1
        else:
            ref, n = total, L
        max_abs = max(max_abs, (out[g].double() - ref).abs().max().item())
        max_lse = max(max_lse, (lse[:, g].double() - math.log(n)).abs().max().item())
    return max_abs, max_lse


def run_forward(L, D, H, causal, seed):
    """Allocate, fill, run ONE full forward; returns (ms, check)."""
    q, k, v = (torch.empty((L, H, D), device="cuda", dtype=torch.bfloat16) for _ in range(3))
    gen = torch.Generator(device="cuda").manual_seed(seed)
    for x in (q, k, v):
        for s in range(0, L, 1 << 20):
            x[s:s + (1 << 20)].normal_(generator=gen)
    rows = zero_rows(L, seed)
    q[torch.tensor(rows, device="cuda")] = 0
    out = torch.empty_like(q)
    lse = torch.empty((H, L), device="cuda", dtype=torch.float32)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dmha.forward(q, k, v, L, causal, out, lse)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    del q, k
    err, lerr = closed_form_check(v, out, lse, rows, causal)
    del v, out, lse
    torch.cuda.empty_cache()
    return ms, {"zero_rows": len(rows), "max_abs_err": err, "max_lse_err": lerr,
                "ok": bool(err <= 2e-2 and lerr <= 1e-3)}


def family(D, H, causal, cap_s, start_log2=16):
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    per_tok = bytes_per_token_p1(D, H)
    L_cap = int(0.97 * free // per_tok) // 256 * 256
    flop = lambda L: 4.0 * L * L * D * H / (2 if causal else 1)  # noqa: E731
    runs = []
    L = 1 << start_log2
    while True:
        ms, chk = run_forward(L, D, H, causal, seed=L % 9973)
        runs.append({"L": L, "forward_s": ms / 1e3, "tflops": flop(L) / (ms / 1e3) / 1e12, "check": chk})
        print(json.dumps(runs[-1]), flush=True)
        if ms / 1e3 > cap_s:
            break
        nxt = 2 * L
        if nxt > L_cap or 4 * ms / 1e3 > cap_s:
            break
        L = nxt
    last = max((r for r in runs if r["forward_s"] <= cap_s), key=lambda r: r["L"])
    # refine: largest multiple of 256 under both bounds (time ~ L^2 from the last run)
    L_time = int(last["L"] * math.sqrt(0.97 * cap_s / last["forward_s"])) // 256 * 256
    L_try = min(L_time, L_cap)
    bound = "time" if L_time < L_cap else "capacity"
    final = last
    if L_try > last["L"]:
        ms, chk = run_forward(L_try, D, H, causal, seed=L_try % 9973)
        rec = {"L": L_try, "forward_s": ms / 1e3, "tflops": flop(L_try) / (ms / 1e3) / 1e12, "check": chk}
        runs.append(rec)
        print(json.dumps(rec), flush=True)
        if ms / 1e3 <= cap_s:
            final = rec
    cap_by_p = {}
    for P in (2, 4, 8):
        pt = H * (20 * D + 8)
        lp = P * int(0.96 * free // pt)
        cap_by_p[str(P)] = lp - lp % (2 * P * 256)
    return {"D": D, "H": H, "causal": causal, "P": 1, "cap_s": cap_s,
            "L_max_P1": final["L"], "L_max_P1_bound": bound if final is not last or L_try <= last["L"] else "time",
            "forward_s_at_L_max": final["forward_s"], "tflops_at_L_max": final["tflops"],
            "check_at_L_max": final["check"],
            "L_capacity_P1": L_cap, "bytes_per_token_P1": per_tok, "free_bytes": free,
            "L_time_bound_P1_predicted": L_time,
            "doubling_runs": runs,
            "L_capacity_by_P_derived": cap_by_p,
            "note": "P > 1: capacity-derived (H*(20D+8) B per local token, fused combine); "
                    "the time bound at P ranks is ~ sqrt(P) x the P = 1 one if strong scaling holds",
            "paper_context": "paper: ~2K vanilla on 1x RTX 3090, ~80K distributed on 4x RTX 3090 (P:679, P:689)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cap-s", type=float, default=300.0)
    ap.add_argument("--families", default="128,64")
    ap.add_argument("--start-log2", type=int, default=16)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "max_len.json"))
    args = ap.parse_args()
    dmha.init(1, 0, None, 0, "bf16", "contiguous")
    res = []
    t0 = time.time()
    for d in args.families.split(","):
        D = int(d)
        r = family(D, 16, D == 64, args.cap_s, args.start_log2)
        r["wall_s"] = time.time() - t0
        print(json.dumps({k: v for k, v in r.items() if k != "doubling_runs"}), flush=True)
        res.append(r)
        Path(args.out).write_text(json.dumps(res, indent=1))
    dmha.finalize()


if __name__ == "__main__":
    main()
