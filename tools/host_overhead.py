"""Host cost of one small forward (C1: L=512, H=4, D=64, fp32): the Python
binding vs the raw C-ABI call, and CUDA-graph replay of the same forward."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2302_06218_b200 import dmha  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "fp32"
L, H, D = 512, 4, 64
dmha.init(1, 0, None, 0, dt, "contiguous")
tdt = torch.float32 if dt == "fp32" else torch.bfloat16
q, k, v = (torch.randn(L, H, D, device="cuda").to(tdt) for _ in range(3))
out, lse = torch.empty_like(q), torch.empty(H, L, device="cuda")
lib = dmha.lib()
args = [q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr(), L, D, H, 0]


def host_us(fn, n=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t) / n * 1e6, (t2 - t) / n * 1e6


print("binding  host/total us", host_us(lambda: dmha.forward(q, k, v, L, False, out, lse)))
print("raw ABI  host/total us", host_us(lambda: lib.dmha_forward(*args)))
print("1 ctypes call (stats) us", host_us(lambda: lib.dmha_set_stream(torch.cuda.current_stream().cuda_stream)))
dmha.reserve(L, D, H)
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    dmha.forward(q, k, v, L, False, out, lse)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        dmha.forward(q, k, v, L, False, out, lse)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(20):
    g.replay()
s.record()
for _ in range(300):
    g.replay()
e.record()
torch.cuda.synchronize()
print("graph replay us per forward", s.elapsed_time(e) / 300 * 1e3)
dmha.finalize()
