"""Kernel timeline: run one forward with the trace hook and print per-tile
softmax / MMA phase durations (SM cycles) for the first traced CTA."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_06218_b200 import build, dmha  # noqa: E402

if "DMHA_LIB" not in os.environ:  # the stamps exist only in a -DDMHA_TRACE=1 build
    dmha._LIB_PATH = build.build(defines=["DMHA_TRACE=1"], variant="trace")

L = int(os.environ.get("TL", 262144 // 8)); H = 16; D = int(os.environ.get("TD", 128))
dmha.init(1, 0, None, 0, "bf16", "contiguous")
q, k, v = (torch.randn(L, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
buf = torch.zeros(dmha.TRACE_WORDS, dtype=torch.int64, device="cuda")
dmha.forward(q, k, v, L, False)
dmha.debug_set_trace(buf)
dmha.forward(q, k, v, L, False)
torch.cuda.synchronize()
dmha.debug_set_trace(None)
t = buf[:4 * 9 * 64].view(4, 9, 64).cpu().numpy().astype(np.int64)
for c in range(int(os.environ.get("TCTAS", 2))):
    tc = t[c] - t[c][0][0]
    print(f"CTA {c}: rows = tile j; cols = 0:WG0 saw S 1:WG0 P 2:WG1 saw S 3:WG1 P 4:mma saw P 5:mma PV issued 6:mma S issued 7:mma saw V landed 8:producer issued V load")
    for j in range(8, 16):
        print(j, " ".join(f"{tc[e][j]:8d}" if t[c][e][j] else "       -" for e in range(9)))
    # steady-state stats over tiles 8..60
    js = range(8, 60)
    per = np.diff(tc[0][8:60]).mean()
    sm0 = np.mean([tc[1][j] - tc[0][j] for j in js]); sm1 = np.mean([tc[3][j] - tc[2][j] for j in js])
    w0 = np.mean([tc[0][j + 1] - tc[1][j] for j in js]); w1 = np.mean([tc[2][j + 1] - tc[3][j] for j in js])
    lat0 = np.mean([tc[4][j] - max(tc[1][j], tc[3][j]) for j in js])
    if t[c][7][10] and t[c][8][10]:
        ld = np.mean([tc[7][j] - tc[0][j] for j in js]); mx = np.mean([tc[8][j] - tc[7][j] for j in js])
        ex = np.mean([tc[1][j] - tc[8][j] for j in js])
        print(f"  WG0 per tile: S load {ld:.0f}  max+decision {mx:.0f}  exp+store+arrive {ex:.0f}")
    print(f"  period/tile {per:.0f}  softmax WG0 {sm0:.0f}  WG1 {sm1:.0f}  wait-S WG0 {w0:.0f}  WG1 {w1:.0f}  P->mma-sees {lat0:.0f}")
dmha.finalize()
# Extra events of CTA 0 (D = 64 kernel): per issuer g (base 9g):
#  0 before K_j wait, 1 K_j landed, 2 s_free seen, 3 V_{j-1} landed, 4 PV_{j-1} committed;
#  producer: 5/14 before kv_empty wait for K_j / V_j, 6/15 slot free
x = buf.view(-1)[18 * 64: 36 * 64].view(18, 64).cpu().numpy().astype(np.int64)
if D == 128 and x[0][10]:
    # in-place D = 128 softmax sub-phases per WG g (base 9g): 0 max done, 1 turn
    # granted, 2 exps done, 3 P stored; relative to that WG's "saw S" (t[0][2g])
    for g in range(2):
        js = range(8, 60)
        saw = t[0][2 * g]
        ph = [np.mean([x[9 * g + e][j] - (saw[j] if e == 0 else x[9 * g + e - 1][j]) for j in js]) for e in range(4)]
        pr = np.mean([t[0][2 * g + 1][j] - x[9 * g + 3][j] for j in js])
        print(f"  WG{g}: load+max {ph[0]:.0f}  turn-wait {ph[1]:.0f}  exps {ph[2]:.0f}  pack+store {ph[3]:.0f}  ->P-ready {pr:.0f}")
elif D == 64 and os.environ.get("TPHASES") and x[0][10]:
    # split-softmax sub-phases (measurement build -DDMHA_TRACE_PHASES=1): WG (g0,h0)
    js = range(8, 60)
    saw = t[0][0]
    seg = [("S load", lambda j: x[0][j] - saw[j]), ("mask+max+smem", lambda j: x[1][j] - x[0][j]),
           ("bar.sync", lambda j: x[2][j] - x[1][j]), ("decision+exps", lambda j: x[3][j] - x[2][j]),
           ("pv_done wait", lambda j: x[4][j] - x[3][j]), ("store P+sum", lambda j: x[5][j] - x[4][j]),
           ("-> next S", lambda j: saw[j + 1] - x[5][j])]
    print("  split softmax (g0 h0) per tile: " + "  ".join(f"{n} {np.mean([f(j) for j in js]):.0f}" for n, f in seg))
elif x[0][10]:
    x0 = t[0][0][0]
    names = ["g0 preK", "g0 Kland", "g0 sfree", "g0 Vland", "g0 PVdone", "prodK pre", "prodK free", "", "",
             "g1 preK", "g1 Kland", "g1 sfree", "g1 Vland", "g1 PVdone", "prodV pre", "prodV free", "", ""]
    print("extra events (CTA 0, relative to WG0 first S):")
    print("  j " + " ".join(f"{n:>10s}" for n in names if n))
    for j in range(8, 16):
        print(f"{j:3d} " + " ".join(f"{x[e][j] - x0:10d}" if x[e][j] else "         -" for e in range(18) if names[e]))
