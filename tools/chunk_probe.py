import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2302_06218_b200 import dmha
L, H, D, causal = 1 << 20, 16, 64, True
dmha.init(1, 0, None, 0, "bf16", "zigzag")
q, k, v = (torch.randn(L, H, D, device="cuda").to(torch.bfloat16) for _ in range(3))
hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
ho = torch.empty_like(hq).pin_memory(); hl = torch.empty(H, L).pin_memory()
dmha.set_profiling(True)
for name, fn in [("device", lambda: dmha.forward(q, k, v, L, causal)),
                 ("host", lambda: dmha.forward_host(hq, hk, hv, L, causal, ho, hl))]:
    fn(); torch.cuda.synchronize()
    s0 = dmha.get_stats()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); t = time.perf_counter() - t
    s1 = dmha.get_stats()
    print(name, f"wall {t*1e3:.1f} ms  attn kernels {s1['attn_ms']-s0['attn_ms']:.1f} ms  launches {s1['attn_launches']-s0['attn_launches']}", flush=True)
dmha.finalize()
