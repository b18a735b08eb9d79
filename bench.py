#!/usr/bin/env python
"""bench.py — throughput of the distributed multi-head attention forward.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (N > 1)

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py re-launches
itself under torch.distributed.run with N ranks on 127.0.0.1 (one per GPU).

A step is one full dmha_forward (every hot-path row of SURVEY §8(a): shard
map, ring K/V exchange, tcgen05 attention, LSE combine) over one batch of
synthetic input.  Default workload C4 (BASELINE.json configs[3]): L=262144,
D=128, H=16, bf16, non-causal, the sequence sharded over the N ranks
(strong scaling; at N=1 it is the largest single-GPU config of the sweep).
Metric: attention TFLOP/s = 4 L^2 D H (/2 causal) / time, whole job.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU fp64 oracle
(oracle/, the tier's reference arm) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "C1": dict(L=512, D=64, H=4, causal=False, dtype="fp32", layout="contiguous",
               desc="C1 single-head-group MHA L=512 D=64 H=4 fp32 non-causal"),
    "C2": dict(L=16384, D=64, H=8, causal=False, dtype="bf16", layout="contiguous",
               desc="C2 MHA L=16384 D=64 H=8 bf16 non-causal"),
    "C2c": dict(L=16384, D=64, H=8, causal=True, dtype="bf16", layout="zigzag",
                desc="C2 MHA L=16384 D=64 H=8 bf16 causal"),
    "C3": dict(L=131072, D=128, H=8, causal=False, dtype="bf16", layout="contiguous",
               desc="C3 MHA L=131072 D=128 H=8 bf16 sequence-sharded"),
    "C4": dict(L=262144, D=128, H=16, causal=False, dtype="bf16", layout="contiguous",
               desc="C4 MHA L=262144 D=128 H=16 bf16 strong-scaling sweep"),
    "C5": dict(L=1048576, D=64, H=16, causal=True, dtype="bf16", layout="zigzag",
               desc="C5 million-scale MHA L=1048576 D=64 H=16 bf16 causal"),
    # A/B-only: C5's head shape at 1/8 of its length (tuning runs, not a bench line)
    "C5s": dict(L=131072, D=64, H=16, causal=True, dtype="bf16", layout="zigzag",
                desc="C5-shaped A/B workload L=131072 D=64 H=16 bf16 causal"),
    "C5nc": dict(L=131072, D=64, H=16, causal=False, dtype="bf16", layout="contiguous",
                 desc="A/B workload L=131072 D=64 H=16 bf16 non-causal"),
    "C2f": dict(L=16384, D=64, H=8, causal=False, dtype="fp32", layout="contiguous",
                desc="A/B workload L=16384 D=64 H=8 fp32 non-causal (C2's shape on the fp32 path)"),
    "C2x4": dict(L=65536, D=64, H=8, causal=False, dtype="bf16", layout="contiguous",
                 desc="A/B workload L=65536 D=64 H=8 bf16 non-causal (C2 heads, 4x longer)"),
}
METRIC = "attention TFLOP/s (4*L^2*D*H, /2 causal)"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def flops(w) -> float:
    f = 4.0 * w["L"] * w["L"] * w["D"] * w["H"]
    return f / 2 if w["causal"] else f


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured (MEASURED_PEAKS.json)"
    return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock / throttle reasons with NVML during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, torch_device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            pr = torch.cuda.get_device_properties(torch_device)
            try:
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(torch_device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nv = pynvml
        except Exception:
            self._h = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self._h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._h is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def spawn_ranks_if_needed(args) -> int | None:
    """--gpus N > 1 without a torchrun environment: re-launch this script under
    torch.distributed.run (N ranks, 127.0.0.1, a free port) and return its
    exit code; None when already inside a launched rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# ----------------------------------------------------------------- CPU oracle baseline
def cpu_oracle_sample(w, target_s: float = 12.0, seed: int = 4321):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload:
    `n` query rows of one head against all L keys (same L, D; the per-row cost
    is what the full job would pay L*H times).  Returns (TFLOP/s, cores, desc)."""
    import numpy as np
    # all of this process's host cores for the OpenMP oracle (torchrun sets
    # OMP_NUM_THREADS=1 for its ranks; libgomp reads it when the oracle loads)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    from oracle import oracle
    from synth import inputs
    L, D = w["L"], w["D"]
    q = inputs.normal((L, 1, D), seed, 0, w["dtype"])
    k = inputs.normal((L, 1, D), seed, 1, w["dtype"])
    v = inputs.normal((L, 1, D), seed, 2, w["dtype"])
    q64, k64, v64 = (x.astype(np.float64) for x in (q, k, v))
    rng = np.random.default_rng(seed)

    def run(n):
        rows = np.sort(rng.integers(0, L, n))
        t0 = time.perf_counter()
        oracle.attention(q64, k64, v64, w["causal"], rows=rows)
        dt = time.perf_counter() - t0
        keys = (rows + 1).sum() if w["causal"] else n * L
        return 4.0 * keys * D / dt, dt

    n = 16
    rate, dt = run(n)
    while dt < 0.5 and n < (1 << 20):
        n *= 4
        rate, dt = run(n)
    n = max(1, int(n * target_s / max(dt, 1e-3)))
    n = min(n, 1 << 22)
    rate, dt = run(n)
    desc = (f"{n} query rows x 1 head against all L={L} keys (D={D}, causal={w['causal']}), "
            f"fp64 C/OpenMP oracle, {dt:.1f} s, CPU: {cpu_model()}")
    return rate / 1e12, oracle.num_threads(), desc, dt


# ----------------------------------------------------------------- reference arm
def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    from oracle import oracle
    oracle.build()
    times, rates, desc, cores = [], [], "", 1
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for i in range(args.warmup + args.steps):
        r, cores, desc, dt = cpu_oracle_sample(w, target_s=per_step, seed=9000 + i)
        if i >= args.warmup:
            rates.append(r)
            times.append(dt)
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, w),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": desc, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(args, w):
    return {"workload": w["desc"], "L": w["L"], "D": w["D"], "H": w["H"], "causal": w["causal"],
            "layout": w["layout"], "batch": 1,
            "parallelism": (f"seq-ring-cp{args.gpus}" if getattr(args, "exchange", "ring") == "ring"
                            else f"seq-a2a-headpar{args.gpus}"),
            "l2": "inputs larger than L2 (q,k,v each >= 126 MB per rank)"
            if w["L"] // args.gpus * w["H"] * w["D"] * 2 > 126e6 else
            "L2 flushed (256 MB write) between timed steps"}


# ----------------------------------------------------------------- our arm
NVLINK_DATASHEET_GBS = 900.0  # NVLink 5, per direction per GPU (B200 datasheet)


def measure_nccl_sendrecv(dist, dev, world, rank, nbytes=256 << 20, iters=5):
    """Measured ring send/recv ceiling on this box (torch.distributed NCCL,
    CUDA-event timed, max over ranks): bytes sent per rank per second."""
    import torch
    send = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    recv = torch.empty_like(send)

    def once():
        ops = [dist.P2POp(dist.isend, send, (rank + 1) % world),
               dist.P2POp(dist.irecv, recv, (rank - 1) % world)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    once()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        once()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return nbytes / (float(t.item()) / 1e3) / 1e9


def roofline_of(w, st, steps, world, step_ms_local, peaks, peak_src):
    """Roofline of the dominant kernel (attention): algorithmic FLOP per
    launch / its CUDA-event launch time (library events on its own stream)."""
    L, D = w["L"], w["D"]
    total_flops = flops(w)
    attn_ms_avg = st["attn_ms"] / max(1, st["attn_launches"])
    launches_per_step = st["attn_launches"] / steps
    flops_per_launch = total_flops / world / max(1.0, launches_per_step)
    achieved = flops_per_launch / (attn_ms_avg / 1e3) / 1e12
    attn_share = st["attn_ms"] / steps / step_ms_local if step_ms_local > 0 else None
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(w["name"])
        except Exception:
            traffic = None
    if w["dtype"] == "fp32":
        # 3xTF32 on tcgen05 kind::tf32 (attn_fwd_tf32.cu): tensor-bound at the
        # TF32 rate = the measured bf16 peak x the nominal tf32/bf16 ratio
        # (1.125 / 2.25 PF dense); algorithmic FLOP counted once, although
        # each product takes three tensor passes
        bf = float(peaks.get("bf16_tflops", 1590.0))
        peak = bf * 0.5
        return {"bound": "tensor", "kernel": "attn_fwd_tf32x3_kernel", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "peak_kind": f"TF32 dense = measured bf16 burst {bf:.0f} x 0.5 (nominal ratio), {peak_src}",
                "frac_of_3pass_work": 3 * achieved / peak,
                "flops_per_launch": flops_per_launch, "launch_ms": attn_ms_avg,
                "share_of_step": attn_share}
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    r = {"bound": "tensor", "kernel": f"attn_fwd_sm100_kernel<{D}>", "achieved": achieved,
         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
         "peak_kind": f"bf16 dense sustained, {peak_src}",
         "frac_of_burst": achieved / float(peaks.get("bf16_tflops", peak)),
         "frac_of_datasheet_2250": achieved / 2250.0,
         "flops_per_launch": flops_per_launch, "launch_ms": attn_ms_avg,
         "share_of_step": attn_share}
    if D == 64:
        # At D = 64 one exponential (MUFU, 16/clk/SM) per score binds before
        # the tensor pipe: ceiling = 148 SMs x 16 x 4*D FLOP per clock
        # (DESIGN.md §5 a2) at the maximum SM clock.
        mx = float(peaks.get("sm_max_mhz", 1965.0))
        cap = 148 * 16 * 4 * D * mx * 1e6 / 1e12
        r["exp_ceiling"] = {"peak_at_max_clock": cap, "frac_at_max_clock": achieved / cap,
                            "unit": "TFLOP/s",
                            "pipe": "MUFU ex2, 16/clk/SM (measured, tools/mufu_rate.cu)"}
    return r


def run_ours(args, w):
    import torch
    import torch.distributed as dist
    from paper_2302_06218_b200 import dmha

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launch_check:  # CPU test hook: which ranks did the launcher start?
        print(json.dumps({"rank": rank, "world": world, "gpus": args.gpus}), flush=True)
        return 0
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    if world > 1:
        dmha.init_distributed(w["dtype"], w["layout"], local)
    else:
        dmha.init(1, 0, None, local, w["dtype"], w["layout"], stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def make_inputs(wl):
        L, D, H = wl["L"], wl["D"], wl["H"]
        if L % (2 * world if wl["layout"] == "zigzag" else world):
            raise SystemExit("L not divisible for this world size")
        Lloc = L // world
        tdt = torch.bfloat16 if wl["dtype"] == "bf16" else torch.float32
        gen = torch.Generator(device=dev)
        shards = []
        for tid in range(3):  # synthetic N(0,1) shards, seeded per (rank, tensor)
            gen.manual_seed(1234 * 1000003 + rank * 101 + tid)
            shards.append(torch.randn((Lloc, H, D), generator=gen, device=dev,
                                      dtype=torch.float32).to(tdt))
        out = torch.empty_like(shards[0])
        lse = torch.empty((H, Lloc), dtype=torch.float32, device=dev)
        return (*shards, out, lse)

    fwd = dmha.forward if args.exchange == "ring" else dmha.forward_headpar

    def timed_run(wl, steps, warmup):
        """W untimed warmups, then exactly K device-timed steps (CUDA events on
        the launch stream, barrier + synchronize on both sides, max over
        ranks); returns (step_ms, local step_ms, stats delta, clocks, inputs)."""
        q, k, v, out, lse = make_inputs(wl)
        Lloc = q.shape[0]
        need_flush = Lloc * wl["H"] * wl["D"] * q.element_size() <= 126e6
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if need_flush else None
        for _ in range(warmup):
            fwd(q, k, v, wl["L"], wl["causal"], out, lse)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        st0 = dmha.get_stats()
        dmha.set_profiling(True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        with ClockSampler(local) as clk:
            for i in range(steps):
                if flush is not None:
                    flush.fill_(i & 0xFF)
                evs[i][0].record(stream)
                fwd(q, k, v, wl["L"], wl["causal"], out, lse)
                evs[i][1].record(stream)
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        st1 = dmha.get_stats()
        dmha.set_profiling(False)
        delta = {key: st1[key] - st0[key] for key in ("kernel_launches", "bytes_sent")}
        for key in ("attn_ms", "attn_launches", "combine_ms", "combine_launches", "exchange_ms",
                    "exchanges", "last_bytes_sent", "last_exchanges"):
            delta[key] = st1[key]  # profiling counters were reset by set_profiling(True)
        local_ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        return max_over_ranks(local_ms), local_ms, delta, clk.summary(), (q, k, v, out, lse)

    w = dict(w, name=args.workload)
    xpeak = measure_nccl_sendrecv(dist, dev, world, rank) if world > 1 else None
    step_ms, step_ms_local, st, clocks, (q, k, v, out, lse) = timed_run(w, args.steps, args.warmup)
    L, D, H = w["L"], w["D"], w["H"]
    Lloc = L // world
    total_flops = flops(w)
    value = total_flops / (step_ms / 1e3) / 1e12
    peaks, peak_src = load_peaks()
    roofline = roofline_of(w, st, args.steps, world, step_ms_local, peaks, peak_src)
    peak = roofline["peak"]
    secondary = {}
    if st["combine_launches"]:
        cm = st["combine_ms"] / st["combine_launches"]
        cbytes = 12.0 * Lloc * H * D + 12.0 * Lloc * H
        secondary["combine"] = {"bound": "hbm", "achieved": cbytes / (cm / 1e3) / 1e9,
                                "peak": float(peaks.get("hbm_gbs", 6551.7)), "unit": "GB/s",
                                "launch_ms": cm}
        secondary["combine"]["frac"] = secondary["combine"]["achieved"] / secondary["combine"]["peak"]
    if st["exchanges"]:
        xm = st["exchange_ms"] / st["exchanges"]
        xbytes = 2.0 * Lloc * H * D * q.element_size()
        ach = xbytes / (xm / 1e3) / 1e9
        secondary["exchange"] = {
            "bound": "nvlink", "achieved": ach, "unit": "GB/s", "launch_ms": xm,
            "peak": NVLINK_DATASHEET_GBS, "frac": ach / NVLINK_DATASHEET_GBS,
            "peak_kind": "NVLink 5 datasheet, 900 GB/s per direction per GPU",
            "peak_measured_nccl_sendrecv": xpeak,
            "frac_of_measured": (ach / xpeak) if xpeak else None,
            "note": "bytes sent per ring step / CUDA-event time of the exchange on the comm stream"}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
        hout = torch.empty(hq.shape, dtype=hq.dtype).pin_memory()
        hlse = torch.empty((H, Lloc), dtype=torch.float32).pin_memory()
        dmha.forward_host(hq, hk, hv, L, w["causal"], hout, hlse)  # warm the staging buffers
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dmha.forward_host(hq, hk, hv, L, w["causal"], hout, hlse)
        t_e2e = (time.perf_counter() - t0) / args.steps
        barrier()
        t_e2e = max_over_ranks(t_e2e)
        e2e = {"value": total_flops / t_e2e / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": 3 * hq.numel() * hq.element_size(),
               "d2h_bytes_per_step": hout.numel() * hout.element_size() + hlse.numel() * 4,
               "ms_per_step": 1e3 * t_e2e}
        del hq, hk, hv, hout, hlse
    del q, k, v, out, lse

    # ---- the north-star head shape (C5, D = 64 causal) device-timed at N = 1
    if world == 1 and args.workload != "C5" and w["dtype"] == "bf16" and not args.no_secondary:
        w5 = dict(WORKLOADS["C5"], name="C5")
        torch.cuda.empty_cache()
        ms5, ms5_local, st5, clk5, _ = timed_run(w5, 3, 1)
        torch.cuda.empty_cache()
        secondary["C5"] = {"workload": w5["desc"], "value": flops(w5) / (ms5 / 1e3) / 1e12,
                           "unit": "TFLOP/s", "ms_per_step": ms5, "steps": 3, "warmup": 1,
                           "roofline": roofline_of(w5, st5, 3, 1, ms5_local, peaks, peak_src),
                           "clocks": clk5}

    # ---- CPU oracle baseline (rank 0, every N; the other ranks wait at a barrier)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rate, cores, desc, _ = cpu_oracle_sample(w)
        cpu = {"value": rate, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": desc,
               "cpu_model": cpu_model()}
    barrier()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": w["dtype"], "data": "synthetic", "config": config_of(args, w),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(st["kernel_launches"]), "clocks": clocks,
            "pct_of_peak": {"measured_sustained": value / (peak * world),
                            "datasheet_2250": value / (2250.0 * world)},
            "secondary": secondary or None,
            "bytes_sent_per_step": st["bytes_sent"] / args.steps,
            "bytes_sent_last_forward": st["last_bytes_sent"],
        }
        print(json.dumps(line), flush=True)
    dmha.finalize()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--exchange", default="ring", choices=["ring", "headpar"],
                    help="ring (north_star, default) or the paper's all-to-all head-parallel exchange")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary C5 line (N=1)")
    ap.add_argument("--launch-check", action="store_true",
                    help="(test hook) each launched rank prints its rank/world and exits")
    args = ap.parse_args()
    rc = spawn_ranks_if_needed(args)
    if rc is not None:
        return rc
    if args.warmup < 3 and args.impl == "ours" and not os.environ.get("BENCH_ALLOW_SHORT_WARMUP"):
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)
    return run_ours(args, w)


if __name__ == "__main__":
    sys.exit(main())
