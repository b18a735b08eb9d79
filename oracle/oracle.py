"""CPU fp64 oracle for the distributed MHA forward of arXiv 2302.06218.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code with ``paper_2302_06218_b200`` (the product) and
never imports it.

Three independent implementations of the same definition:

* ``attention`` — the C OpenMP oracle (``attention_oracle.c``), fp64, plain
  left-to-right sums.  This is "the oracle" that parity tests and the CPU
  baseline use.
* ``attention_np`` — a numpy fp64 twin (row-blocked ``q @ k.T``) used to
  cross-check the C oracle on mid-size inputs.
* ``attention_decimal`` — a 50-digit ``decimal`` brute force for tiny
  inputs, evaluated straight from the paper's three steps WITHOUT the
  max-subtraction, to pin the other two.

Definition followed (§4 "Self-Attention"):
  P:193-196 Eq. ``unnormalized``  A'_t = Q_t K^T      (+ 1/sqrt(D), reading R1)
  P:198-201 row softmax over keys
  P:203-211 Eq. ``attn-sum``      Z_t = sum_j A_{t,j} V_j   (reading R2)
  lse_t = ln sum_j exp(A'_{t,j}/sqrt(D))                  (reading R9)
Causal (north_star): keys j <= t on GLOBAL positions.

Layouts: q, k, v are ``[L, H, D]`` in global sequence order; ``out`` is
``[n_rows, H, D]`` and ``lse`` is ``[H, n_rows]``.
"""
from __future__ import annotations

import ctypes
import decimal
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "attention_oracle.c"
_BODY = _HERE / "attention_oracle_body.h"
_LIB_PATH = _HERE / "build" / "liboracle.so"
_lib = None


def build(force: bool = False) -> Path:
    """Compile the C oracle with gcc -O2 -fopenmp (plain C, fp64)."""
    _LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
    newest = max(_SRC.stat().st_mtime, _BODY.stat().st_mtime)
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < newest:
        # -fno-fast-math: keep IEEE fp64 semantics; no -ffast-math reassociation.
        cmd = ["gcc", "-O2", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               str(_SRC), "-o", str(_LIB_PATH), "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(_LIB_PATH))
        lib.oracle_attention_f64.restype = ctypes.c_int
        P = ctypes.c_void_p
        lib.oracle_attention_f64.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, P, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int64, P, P]
        lib.oracle_attention_f32in.restype = ctypes.c_int
        lib.oracle_attention_f32in.argtypes = lib.oracle_attention_f64.argtypes
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def attention(q, k, v, causal: bool = False, rows=None, key_range=None):
    """C fp64 oracle.  Returns (out [n,H,D] fp64, lse [H,n] fp64)."""
    lib = _load()
    # fp32 inputs (the bf16-valued test tensors) are read as fp32 and widened
    # to fp64 on load; anything else is converted to fp64 first.  The
    # arithmetic is fp64 either way and the results are identical.
    f32 = all(isinstance(x, np.ndarray) and x.dtype == np.float32 for x in (q, k, v))
    dt = np.float32 if f32 else np.float64
    q = np.ascontiguousarray(q, dtype=dt)
    k = np.ascontiguousarray(k, dtype=dt)
    v = np.ascontiguousarray(v, dtype=dt)
    L, H, D = q.shape
    assert k.shape == (L, H, D) and v.shape == (L, H, D)
    if rows is None:
        rows_arr = None
        n = L
    else:
        rows_arr = np.ascontiguousarray(rows, dtype=np.int64)
        n = rows_arr.shape[0]
    kb, ke = (0, L) if key_range is None else key_range
    out = np.empty((n, H, D), dtype=np.float64)
    lse = np.empty((H, n), dtype=np.float64)
    fn = lib.oracle_attention_f32in if f32 else lib.oracle_attention_f64
    rc = fn(q.ctypes.data, k.ctypes.data, v.ctypes.data, L, D, H,
                                  int(bool(causal)),
                                  None if rows_arr is None else rows_arr.ctypes.data, n,
                                  int(kb), int(ke), out.ctypes.data, lse.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_attention_f64: bad arguments")
    return out, lse


def attention_np(q, k, v, causal: bool = False, rows=None, key_range=None, block: int = 256):
    """numpy fp64 twin of ``attention`` (same definition, row-blocked matmuls)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    L, H, D = q.shape
    rows = np.arange(L) if rows is None else np.asarray(rows, dtype=np.int64)
    kb, ke = (0, L) if key_range is None else key_range
    n = rows.shape[0]
    out = np.zeros((n, H, D))
    lse = np.full((H, n), -np.inf)
    keys = np.arange(kb, ke)
    scale = 1.0 / np.sqrt(D)
    for h in range(H):
        Kh = k[kb:ke, h, :]
        Vh = v[kb:ke, h, :]
        for s in range(0, n, block):
            rb = rows[s:s + block]
            x = (q[rb, h, :] @ Kh.T) * scale           # A'_t / sqrt(D)
            if causal:
                x = np.where(keys[None, :] <= rb[:, None], x, -np.inf)
            m = x.max(axis=1, initial=-np.inf)
            ok = np.isfinite(m)
            msafe = np.where(ok, m, 0.0)
            e = np.exp(x - msafe[:, None])               # exp(-inf) = 0 for masked
            l = e.sum(axis=1)
            with np.errstate(invalid="ignore", divide="ignore"):
                a = np.where(ok[:, None], e / np.where(ok, l, 1.0)[:, None], 0.0)
                out[s:s + block, h, :] = a @ Vh
                lse[h, s:s + block] = np.where(ok, m + np.log(np.where(ok, l, 1.0)), -np.inf)
    return out, lse


def attention_decimal(q, k, v, causal: bool = False, digits: int = 50):
    """Brute force in ``digits``-digit decimal arithmetic, straight from
    P:193-211: scores, exp, normalise, weighted sum (no max-subtraction).
    For tiny inputs only (pure-Python loops)."""
    ctx = decimal.Context(prec=digits)
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    L, H, D = q.shape
    Dd = decimal.Decimal
    inv_sqrt_d = ctx.divide(Dd(1), ctx.sqrt(Dd(D)))
    out = np.zeros((L, H, D))
    lse = np.zeros((H, L))
    for h in range(H):
        for t in range(L):
            keys = range(0, t + 1) if causal else range(0, L)
            ex = []
            for j in keys:
                s = Dd(0)
                for d in range(D):
                    s = ctx.add(s, ctx.multiply(Dd(float(q[t, h, d])), Dd(float(k[j, h, d]))))
                ex.append(ctx.exp(ctx.multiply(s, inv_sqrt_d)))
            den = Dd(0)
            for e in ex:
                den = ctx.add(den, e)
            for d in range(D):
                z = Dd(0)
                for e, j in zip(ex, keys):
                    z = ctx.add(z, ctx.multiply(ctx.divide(e, den), Dd(float(v[j, h, d]))))
                out[t, h, d] = float(z)
            lse[h, t] = float(ctx.ln(den))
    return out, lse


def round_bf16(a):
    """Round to the nearest bf16 (ties to even) — the storage format of the
    layer's activations (reading R17).  Written here, independent of
    the product and of synth/."""
    a32 = np.ascontiguousarray(a, dtype=np.float32)
    b = a32.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64).reshape(a32.shape)


def mha_layer(x, wq, wk, wv, wo, H: int, D: int, causal: bool = False):
    """The distributed MHA layer of P:670-675 on one device (NEXT-3):
    Q, K, V = X W_Q, X W_K, X W_V (fp64 products stored as bf16),
    Z = attention(Q, K, V) (this oracle; stored as bf16),
    Y = concat_h(Z) W_0, in fp64.  Returns (Y, lse)."""
    x = np.asarray(x, dtype=np.float64)
    L = x.shape[0]
    q = round_bf16(x @ np.asarray(wq, np.float64)).reshape(L, H, D)
    k = round_bf16(x @ np.asarray(wk, np.float64)).reshape(L, H, D)
    v = round_bf16(x @ np.asarray(wv, np.float64)).reshape(L, H, D)
    z, lse = attention(q, k, v, causal)
    z = round_bf16(z).reshape(L, H * D)
    return z @ np.asarray(wo, np.float64), lse


def attention_flops(L: int, D: int, H: int, causal: bool) -> float:
    """Algorithmic FLOP count of the north_star metric: 4*L^2*D*H, halved if causal."""
    f = 4.0 * L * L * D * H
    return f / 2 if causal else f


if __name__ == "__main__":  # pragma: no cover - manual timing helper
    import time
    rng = np.random.default_rng(0)
    L, H, D = 2048, 4, 64
    q, k, v = (rng.standard_normal((L, H, D)) for _ in range(3))
    t = time.time(); attention(q, k, v); print("C oracle", time.time() - t, "s", num_threads(), "threads")
    t = time.time(); attention_np(q, k, v); print("numpy twin", time.time() - t, "s")
    os._exit(0)
