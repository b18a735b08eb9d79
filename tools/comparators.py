"""Context only: library attention kernels timed on the
same box and shapes as the bench, so the "1 kW power cap" argument has a number.
Never on the product path.

    python tools/comparators.py [C4 C5 C2 C2c ...]

Backends: torch SDPA forced to cuDNN (cuDNN 9.22 sm100 fMHA), and flashinfer's
trtllm-gen context kernels (precompiled Blackwell FMHA cubins; K/V viewed as a
paged NHD cache with one page table).  Same [L, H, D] bf16 layout, N(0,1)
inputs, CUDA-event timing, algorithmic FLOP 4*L^2*D*H (/2 causal).
"""
import json
import sys
import threading

import torch

W = {
    "C4": (262144, 128, 16, False),
    "C5": (1 << 20, 64, 16, True),
    "C5s": (1 << 17, 64, 16, True),
    "C3": (131072, 128, 8, False),
    "C2": (16384, 64, 8, False),
    "C2c": (16384, 64, 8, True),
}


def clocks(stop, out):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        while not stop.is_set():
            out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            stop.wait(0.05)
    except Exception as e:  # noqa: BLE001
        out.append(("err", str(e)))


def timeit(fn, steps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    stop, samp = threading.Event(), []
    th = threading.Thread(target=clocks, args=(stop, samp))
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ok = [s for s in samp if s[0] != "err"]
    clk = sorted(s[0] for s in ok)[len(ok) // 2] if ok else None
    pw = sorted(s[1] for s in ok)[len(ok) // 2] if ok else None
    return a.elapsed_time(b) / steps, clk, pw


def main():
    names = sys.argv[1:] or ["C4", "C5", "C2", "C2c"]
    for name in names:
        L, D, H, causal = W[name]
        flop = 4.0 * L * L * D * H / (2 if causal else 1)
        steps = max(2, min(20, int(3e15 / flop)))
        g = torch.Generator(device="cuda").manual_seed(7)
        q, k, v = (torch.randn(L, H, D, device="cuda", dtype=torch.bfloat16, generator=g) for _ in range(3))
        res = {"workload": name, "L": L, "D": D, "H": H, "causal": causal}
        # cuDNN through SDPA ([1, H, L, D] strided views of the [L, H, D] tensors)
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel
            qt, kt, vt = (x.permute(1, 0, 2).unsqueeze(0) for x in (q, k, v))

            def f():
                with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                    return torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=causal)
            ms, clk, pw = timeit(f, steps)
            res["cudnn"] = {"ms": ms, "tflops": flop / ms / 1e9, "sm_mhz": clk, "power_w": pw}
        except Exception as e:  # noqa: BLE001
            res["cudnn"] = {"error": repr(e)[:300]}
        torch.cuda.empty_cache()
        # flashinfer trtllm-gen (precompiled sm100 cubins)
        try:
            import flashinfer
            ps = 64
            npg = L // ps
            kc = k.view(npg, ps, H, D)
            vc = v.view(npg, ps, H, D)
            bt = torch.arange(npg, device="cuda", dtype=torch.int32).view(1, npg)
            sl = torch.tensor([L], device="cuda", dtype=torch.int32)
            cu = torch.tensor([0, L], device="cuda", dtype=torch.int32)
            ws = torch.zeros(256 << 20, device="cuda", dtype=torch.uint8)
            outb = torch.empty_like(q)

            def f2():
                return flashinfer.prefill.trtllm_batch_context_with_kv_cache(
                    q, (kc, vc), ws, bt, sl, L, L, 1.0 / D ** 0.5, 1.0, 1, cu, cu,
                    out=outb, kv_layout="NHD", causal=causal)
            ms, clk, pw = timeit(f2, steps)
            ref = None
            if L <= 16384:  # sanity against SDPA math on a slice
                qs = q[:256].permute(1, 0, 2).unsqueeze(0).float()
                ref = torch.nn.functional.scaled_dot_product_attention(
                    qs, k.permute(1, 0, 2).unsqueeze(0).float(), v.permute(1, 0, 2).unsqueeze(0).float(),
                    attn_mask=None if not causal else
                    (torch.arange(L, device="cuda")[None, :] <= torch.arange(256, device="cuda")[:, None]))
                err = (outb[:256].permute(1, 0, 2).float() - ref[0]).abs().max().item()
            res["trtllm_gen"] = {"ms": ms, "tflops": flop / ms / 1e9, "sm_mhz": clk, "power_w": pw,
                                 "max_abs_vs_sdpa_rows0_255": None if ref is None else err}
        except Exception as e:  # noqa: BLE001
            res["trtllm_gen"] = {"error": repr(e)[:400]}
        print(json.dumps(res), flush=True)
        del q, k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
