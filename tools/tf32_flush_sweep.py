"""Accuracy and time of the 3xTF32 kernel vs its O flush interval (variant
builds -DDMHA_TF32_FLUSH_KEYS=K under paper_2302_06218_b200/ab/<name>/, loaded via
DMHA_LIB): sampled rows of a C2-shaped fp32 forward against the fp64 oracle.
Usage (one variant per process): DMHA_LIB=... python tools/tf32_flush_sweep.py L H D causal"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import oracle  # noqa: E402  (test infrastructure only)
from paper_2302_06218_b200 import dmha  # noqa: E402
from synth import inputs  # noqa: E402
from tests.parity import metrics  # noqa: E402

L, H, D, causal = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), bool(int(sys.argv[4]))
dmha.init(1, 0, None, 0, "fp32", "contiguous")
q, k, v = inputs.qkv(L, H, D, seed=3100 + D + int(causal), dtype="fp32")
dq, dk, dv = (torch.from_numpy(x).cuda() for x in (q, k, v))
out, lse = dmha.forward(dq, dk, dv, L, causal)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    dmha.forward(dq, dk, dv, L, causal, out, lse)
s.record()
for _ in range(10):
    dmha.forward(dq, dk, dv, L, causal, out, lse)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
rows = np.array(sorted(set(range(64)) | set(range(L - 64, L)) |
                       set(np.random.default_rng(7).integers(0, L, 64).tolist())), dtype=np.int64)
ref_o, ref_l = oracle.attention(q, k, v, causal, rows=rows)
o = out.cpu().numpy()[rows]
ma, rel = metrics(o, ref_o)
print(f"L={L} H={H} D={D} causal={int(causal)} ms={ms:.3f} max_abs={ma:.3e} rel_l2={rel:.3e}")
dmha.finalize()
