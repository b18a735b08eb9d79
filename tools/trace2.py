"""Timeline of the dbuf kernel (attn_fwd_sm100_v2.cu): per 64-key tile,
softmax and issuer phase times (SM cycles) for the first traced CTA."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_06218_b200 import dmha  # noqa: E402

os.environ["DMHA_KERNEL"] = "dbuf"
L = int(os.environ.get("TL", 65536)); H = 16; D = int(os.environ.get("TD", 128))
dmha.init(1, 0, None, 0, "bf16", "contiguous")
q, k, v = (torch.randn(L, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
buf = torch.zeros(dmha.TRACE_WORDS, dtype=torch.int64, device="cuda")
dmha.forward(q, k, v, L, False)
dmha.debug_set_trace(buf)
dmha.forward(q, k, v, L, False)
torch.cuda.synchronize()
dmha.debug_set_trace(None)
t = buf[:4 * 9 * 64].view(4, 9, 64).cpu().numpy().astype(np.int64)
tc = t[0] - t[0][0][0]
print("cols: 0 WG0 saw S | 1 WG0 P | 2 WG1 saw S | 3 WG1 P | 4 S0,S1 issued | 5 PV saw P0 | 6 PV saw P1 | 7 WG0 S loaded | 8 WG0 exps start")
for j in range(16, 26):
    print(j, " ".join(f"{tc[e][j]:8d}" for e in range(9)))
js = range(16, 60)
per = np.diff(tc[0][16:60]).mean()
sm0 = np.mean([tc[1][j] - tc[0][j] for j in js]); sm1 = np.mean([tc[3][j] - tc[2][j] for j in js])
w0 = np.mean([tc[0][j + 1] - tc[1][j] for j in js]); w1 = np.mean([tc[2][j + 1] - tc[3][j] for j in js])
ld = np.mean([tc[7][j] - tc[0][j] for j in js]); mx = np.mean([tc[8][j] - tc[7][j] for j in js])
ex = np.mean([tc[1][j] - tc[8][j] for j in js])
slack = np.mean([tc[0][j] - tc[4][j] for j in js])
print(f"period/64-key tile {per:.0f} (x2 = {2 * per:.0f} per 128 keys)  softmax WG0 {sm0:.0f} WG1 {sm1:.0f}  "
      f"wait-S WG0 {w0:.0f} WG1 {w1:.0f}")
print(f"WG0: S load {ld:.0f}  max {mx:.0f}  exp+store+arrive {ex:.0f};  S issued -> WG0 saw S {slack:.0f}")
dmha.finalize()
