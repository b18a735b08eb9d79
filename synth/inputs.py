"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no scores, softmax, mask or
combine): it only draws random numbers and rounds them to the storage dtype,
so both the oracle and the product see the same bits.

Recipe: q, k, v ~ N(0, 1) i.i.d. per element,
drawn with numpy's PCG64 from ``seed`` and a per-tensor id (q=0, k=1, v=2),
then rounded to bf16 (round-to-nearest-even) for the bf16 path, or kept as
fp32 for the fp32 path.  Layout is the paper's X_{L x ...} sequence-major
[L, H, D] in GLOBAL sequence order (PAPER.md:21 nomenclature; §10.4).
"""
from __future__ import annotations

import numpy as np


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """fp32 -> nearest bf16 (ties to even), returned as fp32 holding bf16 values."""
    x = np.array(x, dtype=np.float32, copy=True, order="C")
    b = x.view(np.uint32)  # in place, uint32: no overflow for finite inputs
    lsb = (b >> 16) & 1
    b += np.uint32(0x7FFF)
    b += lsb
    b &= np.uint32(0xFFFF0000)
    return x


def normal(shape, seed: int, tensor_id: int, dtype: str = "bf16", scale: float = 1.0) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64([int(seed), int(tensor_id)]))
    x = (rng.standard_normal(shape, dtype=np.float32) * np.float32(scale)).astype(np.float32)
    return round_to_bf16(x) if dtype == "bf16" else x


def qkv(L: int, H: int, D: int, seed: int = 1234, dtype: str = "bf16", q_scale: float = 1.0):
    """The contract parity inputs: N(0,1) q, k, v of shape [L, H, D]."""
    q = normal((L, H, D), seed, 0, dtype, q_scale)
    k = normal((L, H, D), seed, 1, dtype)
    v = normal((L, H, D), seed, 2, dtype)
    return q, k, v


def one_hot_selector(L: int, H: int, D: int, targets, q_mag: float = 8.0, k_mag: float = 40.0,
                     seed: int = 7, dtype: str = "bf16"):
    """Structured input for the one-hot closed form.

    Query row t of every head is ``q_mag * e_{a(t)}`` with a(t) = t mod D.
    Key rows are zero except the D selector keys ``targets[a]`` which are
    ``k_mag * e_a``.  Values are N(0,1) (bf16-rounded).  All magnitudes are
    bf16-exact powers/small integers.
    """
    targets = np.asarray(targets, dtype=np.int64)
    assert targets.shape == (D,) and len(set(targets.tolist())) == D
    q = np.zeros((L, H, D), np.float32)
    a = np.arange(L) % D
    q[np.arange(L), :, a] = q_mag
    k = np.zeros((L, H, D), np.float32)
    k[targets, :, np.arange(D)] = k_mag
    v = normal((L, H, D), seed, 2, dtype)
    return q, k, v


def mha_layer(L: int, d_model: int, H: int, D: int, seed: int = 99):
    """x ~ N(0,1) [L, d_model]; W_Q, W_K, W_V ~ N(0, 1/d_model) [d_model, H*D];
    W_0 ~ N(0, 1/(H*D)) [H*D, d_model]; all rounded to bf16."""
    x = normal((L, d_model), seed, 10)
    wq = normal((d_model, H * D), seed, 11, scale=d_model ** -0.5)
    wk = normal((d_model, H * D), seed, 12, scale=d_model ** -0.5)
    wv = normal((d_model, H * D), seed, 13, scale=d_model ** -0.5)
    wo = normal((H * D, d_model), seed, 14, scale=(H * D) ** -0.5)
    return x, wq, wk, wv, wo
