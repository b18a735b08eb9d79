"""Per-CTA wall-clock timeline of one attention launch (%globaltimer stamps at
CTA start / end, dmha_debug_set_trace): CTA durations, launch gaps on an SM
slot, and the steady-state time per KV tile — separates per-CTA fixed cost
from the tile loop.

    python -m paper_2302_06218_b200.build --variant tr -DDMHA_TRACE_PHASES=1 -DDMHA_CTA_STAMPS=1
    DMHA_LIB=paper_2302_06218_b200/ab/tr/libdmha.so TL=16384 TH=8 TD=64 [TC=0] python tools/cta_timeline.py

The stamps exist only in a measurement build (-DDMHA_CTA_STAMPS=1): in the
product they cost the 96-register D = 64 kernel 20 %.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_06218_b200 import dmha  # noqa: E402

L = int(os.environ.get("TL", 16384)); H = int(os.environ.get("TH", 8)); D = int(os.environ.get("TD", 64))
causal = os.environ.get("TC", "0") == "1"
dmha.init(1, 0, None, 0, "bf16", "contiguous")
q, k, v = (torch.randn(L, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
buf = torch.zeros(dmha.TRACE_WORDS, dtype=torch.int64, device="cuda")
for _ in range(2):
    dmha.forward(q, k, v, L, causal)
torch.cuda.synchronize()
dmha.debug_set_trace(buf)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
dmha.forward(q, k, v, L, causal)
b.record()
torch.cuda.synchronize()
dmha.debug_set_trace(None)
ms = a.elapsed_time(b)
t = buf[4096:].view(-1, 2).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3  # us
dur = en - st
n = len(t)
print(f"L={L} H={H} D={D} causal={causal}: {n} CTAs, event time {ms*1e3:.1f} us, "
      f"first start -> last end {en.max():.1f} us")
print(f"CTA duration us: min {dur.min():.1f} median {np.median(dur):.1f} max {dur.max():.1f}")
# the first wave: CTAs that start within 5 us of t0
w1 = st < 5.0
print(f"first wave: {w1.sum()} CTAs, start spread {st[w1].max():.2f} us, end spread "
      f"{en[w1].min():.1f}-{en[w1].max():.1f} us")
# gaps: for each CTA starting after the first wave, distance to the closest earlier end
ends = np.sort(en)
later = np.sort(st[~w1])
gaps = [s_ - ends[np.searchsorted(ends, s_) - 1] for s_ in later if np.searchsorted(ends, s_) > 0]
if gaps:
    print(f"relaunch gap (start - latest earlier CTA end) us: median {np.median(gaps):.2f} max {np.max(gaps):.2f}")
dmha.finalize()
