"""Soak the default kernels: many seeded random configurations (P = 1 and the
emulated ring up to P = 8, both layouts, D = 64 / 128, causal or not, ragged
lengths, kv-split small grids) checked against the fp64 oracle.  Reports the
worst errors; any hang shows up as the caller's timeout.

    python tools/soak.py [n_cases] [seed] [bf16|fp32]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402  (test infrastructure: checking only)
from paper_2302_06218_b200 import dmha  # noqa: E402
from synth import inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
dt = sys.argv[3] if len(sys.argv) > 3 else "bf16"
tdt = torch.bfloat16 if dt == "bf16" else torch.float32
tol = (2e-2, 5e-3, 1e-3) if dt == "bf16" else (1e-3, 1e-4, 1e-5)
dmha.init(1, 0, None, 0, dt, "contiguous")
worst_abs = worst_rel = 0.0
t0 = time.time()
for i in range(n):
    P = int(rng.choice([1, 1, 2, 3, 4, 5, 8]))
    layout = str(rng.choice(["contiguous", "zigzag"])) if P > 1 else "contiguous"
    div = 2 * P if layout == "zigzag" else P
    L = int(rng.integers(1, 4096 // div + 1)) * div
    H = int(rng.integers(1, 4))
    D = int(rng.choice([64, 128]))
    causal = bool(rng.integers(0, 2))
    q, k, v = inputs.qkv(L, H, D, seed=10000 + i, dtype=dt)
    if P == 1:
        dq, dk, dv = (torch.from_numpy(x).to(tdt).cuda() for x in (q, k, v))
        out, lse = dmha.forward(dq, dk, dv, L, causal)
        torch.cuda.synchronize()
        o, l = out.float().cpu().numpy(), lse.cpu().numpy()
    else:
        parts = [np.stack([dmha.shard(x, P, r, layout) for r in range(P)]) for x in (q, k, v)]
        dq, dk, dv = (torch.from_numpy(x).to(tdt).cuda() for x in parts)
        out, lse = dmha.forward_emulated(P, layout, dq, dk, dv, L, causal)
        torch.cuda.synchronize()
        o = dmha.unshard(list(out.float().cpu().numpy()), L, layout)
        l = dmha.unshard([x.T for x in lse.cpu().numpy()], L, layout).T
    ref_o, ref_l = oracle.attention(q, k, v, causal)
    err = float(np.abs(o - ref_o).max())
    rel = float(np.linalg.norm(o - ref_o) / max(np.linalg.norm(ref_o), 1e-30))
    lerr = float(np.abs(l - ref_l).max())
    ok = np.isfinite(o).all() and err <= tol[0] and rel <= tol[1] and lerr <= tol[2]
    worst_abs, worst_rel = max(worst_abs, err), max(worst_rel, rel)
    if not ok:
        print(f"FAIL case {i}: L={L} H={H} D={D} causal={causal} P={P} {layout}: "
              f"max abs {err:.3e} rel {rel:.3e} lse {lerr:.3e}", flush=True)
print(f"{n} cases in {time.time() - t0:.0f} s; worst max abs {worst_abs:.3e}, worst rel L2 {worst_rel:.3e}")
dmha.finalize()
