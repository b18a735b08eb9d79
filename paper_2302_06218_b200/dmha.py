"""Thin Python binding of the dmha C ABI (include/dmha.h).

Argument marshalling only: every step of the hot path (shard index math for
the kernels, attention, ring exchange, LSE combine) runs inside libdmha.so.
PyTorch supplies device memory, the current CUDA stream and, for world size
> 1, the process group that broadcasts the NCCL unique id.

There is no fallback: if libdmha.so is missing or cannot be loaded, every
call raises ``DmhaError``.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "libdmha.so"
# A/B tooling only: DMHA_LIB names another in-tree build of the same library
# (e.g. paper_2302_06218_b200/build_ab/libdmha.so compiled with other flags).
if os.environ.get("DMHA_LIB"):
    _LIB_PATH = Path(os.environ["DMHA_LIB"]).resolve()

OK, ERR_INVALID, ERR_UNSUPPORTED, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_STATE = 0, -1, -2, -3, -4, -5, -6
BF16, FP32 = 0, 1
CONTIGUOUS, ZIGZAG = 0, 1
UNIQUE_ID_BYTES = 128

EXPORTED_SYMBOLS = (
    "dmha_get_unique_id", "dmha_init", "dmha_set_stream", "dmha_finalize", "dmha_last_error",
    "dmha_forward", "dmha_forward_host", "dmha_forward_emulated", "dmha_workspace_bytes",
    "dmha_get_stats", "dmha_local_to_global", "dmha_attention_local", "dmha_lse_combine",
    "dmha_synchronize", "dmha_set_profiling", "dmha_debug_set_trace", "dmha_ring_plan_step",
    "dmha_forward_headpar", "dmha_forward_headpar_emulated", "dmha_mha_forward", "dmha_linear",
    "dmha_reserve", "dmha_shard_rows",
    "dmha_select", "dmha_scatter_rows", "dmha_ring_workspace_bytes",
)


class DmhaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"dmha error {code}: {msg}")
        self.code = code


class Stats(ctypes.Structure):
    _fields_ = [("bytes_sent", ctypes.c_uint64), ("ring_steps", ctypes.c_uint64),
                ("forwards", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("workspace_bytes", ctypes.c_uint64), ("attn_launches", ctypes.c_uint64),
                ("combine_launches", ctypes.c_uint64), ("exchanges", ctypes.c_uint64),
                ("attn_ms", ctypes.c_double), ("combine_ms", ctypes.c_double),
                ("exchange_ms", ctypes.c_double), ("last_bytes_sent", ctypes.c_uint64),
                ("last_exchanges", ctypes.c_uint64), ("pack_launches", ctypes.c_uint64),
                ("pack_ms", ctypes.c_double), ("pack_bytes", ctypes.c_uint64),
                ("gemm_launches", ctypes.c_uint64), ("gemm_ms", ctypes.c_double),
                ("gemm_flop", ctypes.c_double)]


class RingPlan(ctypes.Structure):
    _fields_ = [("src", ctypes.c_int), ("send_to", ctypes.c_int), ("recv_from", ctypes.c_int),
                ("compute_buf", ctypes.c_int), ("recv_buf", ctypes.c_int),
                ("recv_after_compute_of", ctypes.c_int), ("output", ctypes.c_int),
                ("q_base0", ctypes.c_int64), ("q_base1", ctypes.c_int64), ("q_chunk", ctypes.c_int64),
                ("k_base0", ctypes.c_int64), ("k_base1", ctypes.c_int64), ("k_chunk", ctypes.c_int64)]


PLAN_FINAL, PLAN_ACC, PLAN_COMBINE, PLAN_COMBINE_FINAL = 0, 1, 2, 3

_lib = None


def lib():
    """Load libdmha.so (raises DmhaError if it is missing: no fallback path)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise DmhaError(ERR_STATE, f"{_LIB_PATH} not built; run `python -m paper_2302_06218_b200.build`")
        L = ctypes.CDLL(str(_LIB_PATH))
        P, I, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
        sig = {
            "dmha_get_unique_id": [P],
            "dmha_init": [I, I, P, I, I, I, P],
            "dmha_set_stream": [P],
            "dmha_finalize": [],
            "dmha_forward": [P, P, P, P, P, I64, I, I, I],
            "dmha_forward_host": [P, P, P, P, P, I64, I, I, I],
            "dmha_forward_emulated": [I, I, P, P, P, P, P, I64, I, I, I],
            "dmha_workspace_bytes": [I64, I, I, ctypes.POINTER(SZ)],
            "dmha_ring_workspace_bytes": [I, I64, I, I, ctypes.POINTER(SZ)],
            "dmha_get_stats": [ctypes.POINTER(Stats)],
            "dmha_local_to_global": [I64, I, I, I, I64, ctypes.POINTER(I64)],
            "dmha_attention_local": [P, P, P, P, P, I64, I64, I, I, I, I64, I64, I64, I64, I64, I64, I],
            "dmha_lse_combine": [P, P, P, P, P, P, I64, I, I, I],
            "dmha_synchronize": [],
            "dmha_set_profiling": [I],
            "dmha_debug_set_trace": [P],
            "dmha_ring_plan_step": [I, I, I, I, I64, ctypes.POINTER(RingPlan)],
            "dmha_forward_headpar": [P, P, P, P, P, I64, I, I, I],
            "dmha_forward_headpar_emulated": [I, I, P, P, P, P, P, I64, I, I, I],
            "dmha_mha_forward": [P, P, P, P, P, P, P, I64, I, I, I, I],
            "dmha_linear": [P, P, P, I64, I, I],
            "dmha_reserve": [I, I64, I, I],
            "dmha_shard_rows": [I64, I, I, I, ctypes.POINTER(I64)],
            "dmha_select": [P, I64, I, I, P, ctypes.c_double, P, P, P, ctypes.POINTER(I64)],
            "dmha_scatter_rows": [P, P, I64, I, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.dmha_last_error.argtypes = []
        L.dmha_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        raise DmhaError(rc, lib().dmha_last_error().decode(errors="replace"))


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


_STATE = {"dtype": None}  # dtype given to init() (the library fixes it per process)


def _need(cond: bool, msg: str):
    if not cond:
        raise DmhaError(ERR_INVALID, msg)


def _check_tensors(tensors: dict, shapes: dict, dtypes: dict, device=None, pinned: bool = False):
    """Argument checks the kernels rely on (they assume contiguous rows of
    H*D elements and write exactly the documented sizes): every tensor is
    contiguous, has the expected shape and dtype, and lives on one CUDA
    device (or in host memory for the host path).  Messages are formatted
    only on failure (this runs on every call; small forwards are host-bound)."""
    dev = None
    for name, t in tensors.items():
        if t is None:
            continue
        if not t.is_contiguous():
            raise DmhaError(ERR_INVALID, f"{name} must be contiguous (got strides {tuple(t.stride())})")
        want = shapes.get(name)
        if want is not None and t.shape != want:
            raise DmhaError(ERR_INVALID, f"{name} has shape {tuple(t.shape)}, expected {tuple(want)}")
        want = dtypes.get(name)
        if want is not None and t.dtype != want:
            raise DmhaError(ERR_INVALID, f"{name} has dtype {t.dtype}, expected {want}")
        if pinned:
            if t.is_cuda:
                raise DmhaError(ERR_INVALID, f"{name} must be a host tensor for the host path")
        else:
            if not t.is_cuda:
                raise DmhaError(ERR_INVALID, f"{name} must be a CUDA tensor")
            d = t.get_device()
            if dev is None:
                dev = d
            elif d != dev:
                raise DmhaError(ERR_INVALID, f"{name} is on cuda:{d}, other arguments on cuda:{dev}")


def _elem_dtype():
    import torch
    d = _STATE["dtype"]
    _need(d is not None, "dmha.init() has not been called")
    return torch.bfloat16 if d == BF16 else torch.float32


def _cur_stream() -> int:
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:  # no Stream object per call
        return int(raw(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


_DT = {"bf16": BF16, "fp32": FP32}
_LAY = {"contiguous": CONTIGUOUS, "zigzag": ZIGZAG}


def dtype_code(dtype) -> int:
    return _DT[dtype] if isinstance(dtype, str) else int(dtype)


def layout_code(layout) -> int:
    return _LAY[layout] if isinstance(layout, str) else int(layout)


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(UNIQUE_ID_BYTES)
    _check(lib().dmha_get_unique_id(ctypes.addressof(buf)))
    return buf.raw


def init(world_size: int = 1, rank: int = 0, unique_id: bytes | None = None, device: int = 0,
         dtype="bf16", layout="contiguous", stream: int | None = None):
    uid = None
    if unique_id is not None:
        uid = ctypes.create_string_buffer(bytes(unique_id), UNIQUE_ID_BYTES)
    s = _cur_stream() if stream is None else int(stream)
    _check(lib().dmha_init(world_size, rank, None if uid is None else ctypes.addressof(uid), device,
                           dtype_code(dtype), layout_code(layout), s))
    _STATE["dtype"] = dtype_code(dtype)
    _STATE["world"] = int(world_size)
    _STATE["stream"] = s  # the stream dmha_init was given


def init_distributed(dtype="bf16", layout="contiguous", device: int | None = None):
    """init() over an initialised torch.distributed process group: rank 0 makes
    the NCCL unique id and the group broadcasts it."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.cuda.current_device() if device is None else device
    if world == 1:
        return init(1, 0, None, dev, dtype, layout)
    obj = [get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    init(world, rank, obj[0], dev, dtype, layout)


def set_stream(stream: int):
    """The stream every later call launches on (cached: the C call is made
    only when it changes)."""
    stream = int(stream)
    if _STATE.get("stream") != stream:
        _check(lib().dmha_set_stream(stream))
        _STATE["stream"] = stream


def finalize():
    _check(lib().dmha_finalize())
    _STATE["dtype"] = None
    _STATE["stream"] = None


def synchronize():
    _check(lib().dmha_synchronize())


def forward(q, k, v, L: int, causal: bool = False, out=None, lse=None):
    """Distributed forward on this rank's [L/P, H, D] device shards; returns (out, lse)."""
    import torch
    Lloc, H, D = q.shape
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((H, Lloc), dtype=torch.float32, device=q.device)
    et = _elem_dtype()
    _check_tensors(dict(q=q, k=k, v=v, out=out, lse=lse),
                   dict(k=q.shape, v=q.shape, out=q.shape, lse=(H, Lloc)),
                   dict(q=et, k=et, v=et, out=et, lse=torch.float32))
    set_stream(_cur_stream())
    _check(lib().dmha_forward(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), int(L), D, H,
                              int(bool(causal))))
    return out, lse


def forward_host(q, k, v, L: int, causal: bool = False, out=None, lse=None):
    """Same as forward() but with host (pinned) tensors; copies in, runs, copies
    out and synchronises (the end-to-end path)."""
    import torch
    Lloc, H, D = q.shape
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((H, Lloc), dtype=torch.float32, pin_memory=q.is_pinned())
    et = _elem_dtype()
    _check_tensors(dict(q=q, k=k, v=v, out=out, lse=lse),
                   dict(k=q.shape, v=q.shape, out=q.shape, lse=(H, Lloc)),
                   dict(q=et, k=et, v=et, out=et, lse=torch.float32), pinned=True)
    set_stream(_cur_stream())
    _check(lib().dmha_forward_host(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), int(L), D, H,
                                   int(bool(causal))))
    return out, lse


def forward_emulated(world_size: int, layout, q, k, v, L: int, causal: bool = False, out=None,
                     lse=None):
    """Single-GPU emulation of the P-rank ring; q/k/v are [P, L/P, H, D] device tensors."""
    import torch
    P, Lloc, H, D = q.shape
    _need(P == world_size, f"q has {P} shards, world_size {world_size}")
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((P, H, Lloc), dtype=torch.float32, device=q.device)
    et = _elem_dtype()
    _check_tensors(dict(q=q, k=k, v=v, out=out, lse=lse),
                   dict(k=q.shape, v=q.shape, out=q.shape, lse=(P, H, Lloc)),
                   dict(q=et, k=et, v=et, out=et, lse=torch.float32))
    set_stream(_cur_stream())
    _check(lib().dmha_forward_emulated(world_size, layout_code(layout), _ptr(q), _ptr(k), _ptr(v),
                                       _ptr(out), _ptr(lse), int(L), D, H, int(bool(causal))))
    return out, lse


def forward_headpar(q, k, v, L: int, causal: bool = False, out=None, lse=None):
    """The paper's head-parallel algorithm (two all-to-alls); same
    contract as forward()."""
    import torch
    Lloc, H, D = q.shape
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((H, Lloc), dtype=torch.float32, device=q.device)
    et = _elem_dtype()
    _check_tensors(dict(q=q, k=k, v=v, out=out, lse=lse),
                   dict(k=q.shape, v=q.shape, out=q.shape, lse=(H, Lloc)),
                   dict(q=et, k=et, v=et, out=et, lse=torch.float32))
    set_stream(_cur_stream())
    _check(lib().dmha_forward_headpar(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), int(L), D, H,
                                      int(bool(causal))))
    return out, lse


def forward_headpar_emulated(world_size: int, layout, q, k, v, L: int, causal: bool = False,
                             out=None, lse=None):
    """Single-GPU emulation of forward_headpar; q/k/v are [P, L/P, H, D]."""
    import torch
    P, Lloc, H, D = q.shape
    _need(P == world_size, f"q has {P} shards, world_size {world_size}")
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((P, H, Lloc), dtype=torch.float32, device=q.device)
    et = _elem_dtype()
    _check_tensors(dict(q=q, k=k, v=v, out=out, lse=lse),
                   dict(k=q.shape, v=q.shape, out=q.shape, lse=(P, H, Lloc)),
                   dict(q=et, k=et, v=et, out=et, lse=torch.float32))
    set_stream(_cur_stream())
    _check(lib().dmha_forward_headpar_emulated(world_size, layout_code(layout), _ptr(q), _ptr(k),
                                               _ptr(v), _ptr(out), _ptr(lse), int(L), D, H,
                                               int(bool(causal))))
    return out, lse


def mha_forward(x, wq, wk, wv, wo, L: int, H: int, D: int, causal: bool = False, y=None, lse=None):
    """NEXT-3: distributed MHA layer y = Attn(x W_Q, x W_K, x W_V) W_0 on this
    rank's rows x [L/P, d_model] (weights replicated)."""
    import torch
    Lloc, d_model = x.shape
    if y is None:
        y = torch.empty((Lloc, d_model), dtype=x.dtype, device=x.device)
    bf = torch.bfloat16
    _check_tensors(dict(x=x, wq=wq, wk=wk, wv=wv, wo=wo, y=y, lse=lse),
                   dict(wq=(d_model, H * D), wk=(d_model, H * D), wv=(d_model, H * D),
                        wo=(H * D, d_model), y=(Lloc, d_model), lse=(H, Lloc)),
                   dict(x=bf, wq=bf, wk=bf, wv=bf, wo=bf, y=bf, lse=torch.float32))
    set_stream(_cur_stream())
    _check(lib().dmha_mha_forward(_ptr(x), _ptr(wq), _ptr(wk), _ptr(wv), _ptr(wo), _ptr(y), _ptr(lse),
                                  int(L), int(d_model), int(D), int(H), int(bool(causal))))
    return y


def linear(x, w, y=None):
    """NEXT-3 projection step y = x @ w (bf16 [M, K] x [K, N], tcgen05 GEMM)."""
    import torch
    M, K = x.shape
    N = w.shape[1]
    if y is None:
        y = torch.empty((M, N), dtype=x.dtype, device=x.device)
    bf = torch.bfloat16
    _check_tensors(dict(x=x, w=w, y=y), dict(w=(K, N), y=(M, N)), dict(x=bf, w=bf, y=bf))
    set_stream(_cur_stream())
    _check(lib().dmha_linear(_ptr(x), _ptr(w), _ptr(y), int(M), int(N), int(K)))
    return y


def attention_local(q, k, v, out, lse, causal=False, qmap=None, kmap=None, out_mode: int = 0):
    """One local attention pass (hot-path step a2).  qmap/kmap = (base0, base1, chunk)."""
    Lq, H, D = q.shape
    Lk = k.shape[0]
    qm = qmap if qmap is not None else (0, Lq, Lq)
    km = kmap if kmap is not None else (0, Lk, Lk)
    set_stream(_cur_stream())
    _check(lib().dmha_attention_local(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), Lq, Lk, D, H,
                                      int(bool(causal)), *map(int, qm), *map(int, km), int(out_mode)))
    return out, lse


def lse_combine(o_acc, lse_acc, o_part, lse_part, out=None, lse_out=None, final: bool = False):
    """Hot-path step a4/a5: merge a partial into the accumulator (in place), or
    with final=True write the merged result to out/lse_out."""
    Lq, H, D = o_acc.shape
    set_stream(_cur_stream())
    _check(lib().dmha_lse_combine(_ptr(o_acc), _ptr(lse_acc), _ptr(o_part), _ptr(lse_part),
                                  _ptr(out), _ptr(lse_out), Lq, D, H, int(bool(final))))


SCORERS = {"l2": 0, "proj": 1}


def select(x, tau: float, scorer: str = "l2", psi=None, x_out=None, idx_out=None, scores=None):
    """NEXT-4 token Selector s_{psi,tau} (Eq. `selector`) on this rank's rows
    x [n, width] (bf16 device tensor).  Returns (x_out[:n_kept] view,
    idx_out[:n_kept] view of LOCAL row indices, scores [n] fp64)."""
    import torch
    n, w = x.shape
    if x_out is None:
        x_out = torch.empty_like(x)
    if idx_out is None:
        idx_out = torch.empty(n, dtype=torch.int64, device=x.device)
    if scores is None:
        scores = torch.empty(n, dtype=torch.float64, device=x.device)
    k = ctypes.c_int64(0)
    set_stream(_cur_stream())
    _check(lib().dmha_select(_ptr(x), int(n), int(w), SCORERS[scorer], _ptr(psi), float(tau),
                             _ptr(x_out), _ptr(idx_out), _ptr(scores), ctypes.byref(k)))
    return x_out[:k.value], idx_out[:k.value], scores


def scatter_rows(y_sel, idx, y_full):
    """Re-aggregation: y_full[idx[i]] = y_sel[i] in place."""
    k = int(idx.shape[0])
    w = int(y_full.shape[1])
    set_stream(_cur_stream())
    _check(lib().dmha_scatter_rows(_ptr(y_sel), _ptr(idx), k, w, _ptr(y_full)))
    return y_full


def workspace_bytes(L: int, D: int, H: int, world_size: int | None = None) -> int:
    """Library workspace of a forward (dmha_workspace_bytes; with world_size,
    dmha_ring_workspace_bytes — what forward_emulated at that size holds)."""
    n = ctypes.c_size_t(0)
    if world_size is None:
        _check(lib().dmha_workspace_bytes(int(L), D, H, ctypes.byref(n)))
    else:
        _check(lib().dmha_ring_workspace_bytes(int(world_size), int(L), D, H, ctypes.byref(n)))
    return n.value


def get_stats() -> dict:
    s = Stats()
    _check(lib().dmha_get_stats(ctypes.byref(s)))
    return {f: (float if t is ctypes.c_double else int)(getattr(s, f)) for f, t in Stats._fields_}


TRACE_WORDS = 4096 + 2 * 16384  # DMHA_TRACE_WORDS (dmha.h)


def debug_set_trace(buf):
    """Timeline hook: buf = device uint64 tensor of >= TRACE_WORDS entries, or None."""
    _check(lib().dmha_debug_set_trace(None if buf is None else _ptr(buf)))


def reserve(L: int, D: int, H: int, world_size: int | None = None):
    """Pre-allocate the workspace of a forward of this size (CUDA-graph capture)."""
    ws = world_size if world_size is not None else _STATE.get("world", 1)
    _check(lib().dmha_reserve(int(ws), int(L), int(D), int(H)))


def set_profiling(enable: bool):
    _check(lib().dmha_set_profiling(int(bool(enable))))


def local_to_global(L: int, world_size: int, rank: int, layout, i: int) -> int:
    g = ctypes.c_int64(0)
    _check(lib().dmha_local_to_global(int(L), int(world_size), int(rank), layout_code(layout),
                                      int(i), ctypes.byref(g)))
    return g.value


def ring_plan(world_size: int, rank: int, step: int, layout, L: int) -> dict:
    """The library's ring schedule for (rank, step): a plain dict of RingPlan fields."""
    pl = RingPlan()
    _check(lib().dmha_ring_plan_step(int(world_size), int(rank), int(step), layout_code(layout),
                                     int(L), ctypes.byref(pl)))
    return {f: int(getattr(pl, f)) for f, _ in RingPlan._fields_}


def shard_rows(L: int, world_size: int, rank: int, layout) -> int:
    """Rows rank `rank` owns (dmha_shard_rows: uneven contiguous shards allowed)."""
    n = ctypes.c_int64(0)
    _check(lib().dmha_shard_rows(int(L), int(world_size), int(rank), layout_code(layout),
                                 ctypes.byref(n)))
    return n.value


def global_rows(L: int, world_size: int, rank: int, layout) -> np.ndarray:
    """Global positions of rank `rank`'s local rows, from the library's own
    position map (the q map of dmha_ring_plan_step: two increasing pieces,
    i < chunk -> base0 + i, else base1 + i - chunk; tests check it against
    dmha_local_to_global row by row)."""
    pl = ring_plan(world_size, rank, 0, layout, L)
    n = shard_rows(L, world_size, rank, layout)
    c = pl["q_chunk"]
    return np.concatenate([np.arange(pl["q_base0"], pl["q_base0"] + min(c, n)),
                           np.arange(pl["q_base1"], pl["q_base1"] + max(0, n - c))]).astype(np.int64)


def shard(x, world_size: int, rank: int, layout):
    """Rows of the global [L, ...] tensor that rank `rank` owns, in local order."""
    idx = global_rows(x.shape[0], world_size, rank, layout)
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x[torch.from_numpy(idx).to(x.device)]
    except ImportError:  # pragma: no cover
        pass
    return x[idx]


def unshard(parts, L: int, layout):
    """Inverse of shard: list of per-rank [L/P, ...] blocks -> global [L, ...]."""
    P = len(parts)
    first = parts[0]
    try:
        import torch
        if isinstance(first, torch.Tensor):
            outp = torch.empty((L,) + tuple(first.shape[1:]), dtype=first.dtype, device=first.device)
            for r, p in enumerate(parts):
                idx = global_rows(L, P, r, layout)
                outp[torch.from_numpy(idx).to(first.device)] = p[:len(idx)]
            return outp
    except ImportError:  # pragma: no cover
        pass
    outp = np.empty((L,) + tuple(first.shape[1:]), dtype=first.dtype)
    for r, p in enumerate(parts):
        idx = global_rows(L, P, r, layout)
        outp[idx] = p[:len(idx)]  # a padded slot (uneven shards) keeps its rows first
    return outp


def stack_shards(x, world_size: int, layout):
    """Global [L, ...] -> [P, Lm, ...] rank-major shard slots (Lm = the largest
    shard; short slots zero-padded at the end), the layout dmha_forward_emulated
    takes."""
    parts = [shard(x, world_size, r, layout) for r in range(world_size)]
    Lm = max(len(p) for p in parts)
    try:
        import torch
        if isinstance(x, torch.Tensor):
            outp = torch.zeros((world_size, Lm) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
            for r, p in enumerate(parts):
                outp[r, :len(p)] = p
            return outp
    except ImportError:  # pragma: no cover
        pass
    outp = np.zeros((world_size, Lm) + tuple(x.shape[1:]), dtype=x.dtype)
    for r, p in enumerate(parts):
        outp[r, :len(p)] = p
    return outp


def unstack_emulated(out, lse, L: int, layout):
    """dmha_forward_emulated results -> global out [L, H, D] and lse [H, L]
    (slot r: its rows first; lse packed as [H, rows] from the slot start)."""
    P, Lm, H = out.shape[0], out.shape[1], out.shape[2]
    rows = [shard_rows(L, P, r, layout) for r in range(P)]
    o_parts = [out[r][:rows[r]] for r in range(P)]
    flat = lse.reshape(P, -1)
    l_parts = [flat[r][:H * rows[r]].reshape(H, rows[r]).T for r in range(P)]
    return unshard(o_parts, L, layout), unshard(l_parts, L, layout).T


def attention_flops(L: int, D: int, H: int, causal: bool) -> float:
    """north_star metric FLOPs: 4*L^2*D*H, halved for causal."""
    f = 4.0 * L * L * D * H
    return f / 2 if causal else f
