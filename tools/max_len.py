"""Maximum sequence length that fits (BASELINE.json metric).

    python tools/max_len.py [--out gpurun_out/max_len.json]

Per local token the library needs (bf16):
  P = 1:  H*(8*D + 4) bytes       (q, k, v, out + lse; no workspace)
  P > 1:  H*(20*D + 8) bytes      (+ two K/V ring buffers, fp32 O_acc, lse_acc; the
                                   combine is fused, NEXT-2 — H*(24*D + 12) without)
so L_max(P) = P * floor(free_HBM / bytes_per_token) (rounded to 2P*256).

On this single GPU the P = 1 bound is demonstrated, not only computed: q, k, v,
out and lse are allocated at L_max, and the attention kernel runs a 256-row
query block against all L_max keys with Q = 0, whose exact result is known in
closed form (out = mean of V over all keys, lse = ln L) — checked on the GPU
output.  The full-forward time at L_max is extrapolated from that launch
(labelled "extrapolated").  The P > 1 figures are capacity-derived.
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


def run_family(D, H, causal, free_bytes, rows=256):
    per_tok = H * (8 * D + 4)
    L = int(0.95 * free_bytes // per_tok)
    L -= L % 256
    t0 = time.time()
    q_full = torch.empty((L, H, D), device="cuda", dtype=torch.bfloat16)  # the whole q shard fits
    q = q_full[L - rows:]
    q.zero_()
    k = torch.empty((L, H, D), device="cuda", dtype=torch.bfloat16)
    v = torch.empty((L, H, D), device="cuda", dtype=torch.bfloat16)
    out_full = torch.empty((L, H, D), device="cuda", dtype=torch.bfloat16)  # proves `out` fits too
    lse_full = torch.empty((H, L), device="cuda", dtype=torch.float32)
    chunk = 1 << 22
    for s in range(0, L, chunk):
        k[s:s + chunk].normal_()
        v[s:s + chunk].normal_()
    alloc_s = time.time() - t0
    out = torch.empty((rows, H, D), device="cuda", dtype=torch.bfloat16)
    lse = torch.empty((H, rows), device="cuda", dtype=torch.float32)
    # the query block sits at the END of the sequence so that, causal or not,
    # it attends to all L keys
    qmap = (L - rows, L, rows)
    kmap = (0, L, L)
    dmha.attention_local(q, k, v, out, lse, causal, qmap, kmap, 0)
    torch.cuda.synchronize()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_ev.record()
    dmha.attention_local(q, k, v, out, lse, causal, qmap, kmap, 0)
    e_ev.record()
    torch.cuda.synchronize()
    ms = s_ev.elapsed_time(e_ev)
    # closed form: Q = 0 -> uniform softmax over all keys of the block
    vmean = torch.zeros((H, D), device="cuda", dtype=torch.float64)
    for s in range(0, L, 1 << 15):
        vmean += v[s:s + (1 << 15)].double().sum(0)
    vmean /= L
    if causal:  # row i (global L-rows+i) sees keys 0..L-rows+i
        ok_rows = rows - 1
        ref_last = vmean  # last row sees all keys
        err = (out[ok_rows].double() - ref_last).abs().max().item()
        lse_err = abs(lse[:, ok_rows].double() - math.log(L)).max().item()
    else:
        err = (out.double() - vmean[None]).abs().max().item()
        lse_err = (lse.double() - math.log(L)).abs().max().item()
    # The block ran one 256-row CTA per head (H CTAs, one wave); the full
    # forward is (L/256)*H such CTAs, i.e. ceil(L/256*H/148) waves of ~the
    # same per-CTA time (extrapolated; causal halves the average CTA work).
    waves = math.ceil((L / 256) * H / 148)
    full_ms = ms * waves
    if causal:
        full_ms /= 2
    flops = 4.0 * L * L * D * H / (2 if causal else 1)
    res = {"D": D, "H": H, "causal": causal, "L_max_P1": L, "bytes_per_token_P1": per_tok,
           "free_bytes": free_bytes, "allocated_bytes": torch.cuda.memory_allocated(),
           "fraction_of_capacity_bound": L * per_tok / free_bytes,
           "alloc_and_fill_s": alloc_s, "block_rows": rows, "block_ms": ms,
           "closed_form_max_abs_err": err, "closed_form_lse_err": lse_err,
           "full_forward_s_extrapolated": full_ms / 1e3,
           "full_forward_tflops_extrapolated": flops / (full_ms / 1e3) / 1e12}
    cap = {}
    for P in (1, 2, 4, 8):
        pt = H * (8 * D + 4) if P == 1 else H * (20 * D + 8)
        lp = P * int(0.96 * free_bytes // pt)
        lp -= lp % (2 * P * 256)
        cap[str(P)] = lp
    res["L_max_capacity_by_P"] = cap
    res["paper_context"] = "paper: ~2K vanilla on 1x RTX 3090, ~80K distributed on 4x RTX 3090 (P:679, P:689)"
    del q, q_full, k, v, out_full, lse_full, out, lse
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "max_len.json"))
    args = ap.parse_args()
    dmha.init(1, 0, None, 0, "bf16", "contiguous")
    out = []
    for D, H, causal in ((128, 16, False), (64, 16, True)):
        torch.cuda.empty_cache()
        free, total = torch.cuda.mem_get_info()
        r = run_family(D, H, causal, free)
        print(json.dumps(r), flush=True)
        out.append(r)
    dmha.finalize()
    Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
