"""Pins for the CPU oracle (oracle/), checked against things other than itself.

Every test here is CPU-only (``-m "not gpu"``).  The pins follow SURVEY.md
§8(c): hand-derived worked examples (tests/golden/hand_cases.txt), a 50-digit
brute force of PAPER.md P:193-211, a library routine (torch SDPA in fp64),
closed forms (Q=0 mean / prefix mean, one-hot selection, constant V column,
L=1), and invariants (joint K/V permutation, Q permutation equivariance,
key shift, linearity in V, rows of A summing to one).
"""
import math
from pathlib import Path

import numpy as np
import pytest
import torch

from synth import inputs

GOLDEN = Path(__file__).parent / "golden" / "hand_cases.txt"


def _cases():
    for line in GOLDEN.read_text().splitlines():
        if not line.strip() or line.startswith("#"):
            continue
        f = [s.strip() for s in line.split("|")]
        name = f[0]
        L, H, D, causal = (int(x) for x in f[1].split())
        arr = [np.array([float(x) for x in s.split()]) for s in f[2:7]]
        yield name, L, H, D, bool(causal), arr


@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: c[0])
def test_hand_worked_examples(oracle_mod, case):
    name, L, H, D, causal, (q, k, v, out, lse) = case
    shp = (L, H, D)
    o, l = oracle_mod.attention(q.reshape(shp), k.reshape(shp), v.reshape(shp), causal=causal)
    np.testing.assert_allclose(o.reshape(-1), out, rtol=0, atol=1e-12)
    np.testing.assert_allclose(l.reshape(-1), lse, rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("L,H,D", [(1, 1, 1), (5, 2, 3), (8, 2, 4), (7, 1, 4)])
def test_decimal_brute_force(oracle_mod, L, H, D, causal):
    rng = np.random.default_rng(L * 100 + H * 10 + D + causal)
    q, k, v = (rng.standard_normal((L, H, D)) * 2 for _ in range(3))
    ref_o, ref_l = oracle_mod.attention_decimal(q, k, v, causal=causal)
    o, l = oracle_mod.attention(q, k, v, causal=causal)
    np.testing.assert_allclose(o, ref_o, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(l, ref_l, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("L,H,D", [(300, 3, 64), (129, 2, 128), (64, 1, 8)])
def test_matches_torch_sdpa_fp64(oracle_mod, L, H, D, causal):
    """A library routine (torch SDPA, CPU fp64) pins scale, mask and operand order."""
    q, k, v = (x.astype(np.float64) for x in inputs.qkv(L, H, D, seed=11 + L, dtype="fp32"))
    o, l = oracle_mod.attention(q, k, v, causal=causal)
    t = [torch.from_numpy(x).permute(1, 0, 2) for x in (q, k, v)]
    ref = torch.nn.functional.scaled_dot_product_attention(*t, is_causal=causal)
    np.testing.assert_allclose(o, ref.permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)
    # lse against torch.logsumexp of explicitly scaled scores
    s = torch.einsum("hid,hjd->hij", t[0], t[1]) / math.sqrt(D)
    if causal:
        s = s.masked_fill(torch.ones(L, L, dtype=torch.bool).triu(1), float("-inf"))
    np.testing.assert_allclose(l, torch.logsumexp(s, dim=-1).numpy(), rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
def test_numpy_twin_agrees_rows_and_key_ranges(oracle_mod, causal):
    L, H, D = 700, 2, 64
    q, k, v = inputs.qkv(L, H, D, seed=5)
    rows = np.array([0, 1, 127, 128, 300, 699])
    for kr in (None, (0, 128), (128, 600), (650, 700)):
        o, l = oracle_mod.attention(q, k, v, causal, rows=rows, key_range=kr)
        o2, l2 = oracle_mod.attention_np(q, k, v, causal, rows=rows, key_range=kr)
        np.testing.assert_allclose(o, o2, rtol=0, atol=1e-12)
        np.testing.assert_allclose(l, l2, rtol=0, atol=1e-12)


def test_empty_key_range_gives_neg_inf_and_zero(oracle_mod):
    q, k, v = inputs.qkv(64, 2, 8, seed=3)
    o, l = oracle_mod.attention(q, k, v, causal=True, rows=np.array([5, 10]), key_range=(20, 40))
    assert np.all(l == -np.inf) and np.all(o == 0)
    o, l = oracle_mod.attention(q, k, v, causal=False, key_range=(7, 7))
    assert np.all(l == -np.inf) and np.all(o == 0)


@pytest.mark.parametrize("causal", [False, True])
def test_zero_query_gives_mean_of_values(oracle_mod, causal):
    """Q=0 -> uniform softmax: out = mean of V (prefix mean if causal), lse = ln(#keys)."""
    L, H, D = 200, 2, 16
    _, k, v = inputs.qkv(L, H, D, seed=9)
    q = np.zeros_like(k)
    o, l = oracle_mod.attention(q, k, v, causal=causal)
    v64 = v.astype(np.float64)
    if causal:
        cnt = np.arange(1, L + 1)
        ref = np.cumsum(v64, axis=0) / cnt[:, None, None]
        ref_l = np.log(cnt)[None, :].repeat(H, 0)
    else:
        ref = np.broadcast_to(v64.mean(axis=0), v.shape)
        ref_l = np.full((H, L), math.log(L))
    np.testing.assert_allclose(o, ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(l, ref_l, rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
def test_one_hot_scores_select_value_row(oracle_mod, causal):
    L, H, D = 256, 2, 64
    targets = np.random.default_rng(1).permutation(L)[:D]
    q, k, v = inputs.one_hot_selector(L, H, D, targets)
    o, _ = oracle_mod.attention(q, k, v, causal=causal)
    a = np.arange(L) % D
    tgt = targets[a]
    # scaled winning score = 8*40/sqrt(64) = 40; others 0 -> error <= L*e^-40*max|v|
    for t in range(L):
        if not causal or tgt[t] <= t:
            np.testing.assert_allclose(o[t], v[tgt[t]], rtol=0, atol=1e-12)
        else:  # target not visible -> all visible scores are 0 -> prefix mean
            np.testing.assert_allclose(o[t], v[: t + 1].astype(np.float64).mean(0), rtol=0, atol=1e-12)


def test_constant_value_column_and_rows_sum_to_one(oracle_mod):
    L, H, D = 96, 2, 128
    q, k, v = inputs.qkv(L, H, D, seed=21, q_scale=3.0)
    v = v.copy()
    v[:, :, 5] = 0.75
    o, _ = oracle_mod.attention(q, k, v, causal=False)
    np.testing.assert_allclose(o[:, :, 5], 0.75, rtol=0, atol=1e-13)
    # V = identity (L <= D): out row t is the attention row A_t itself
    vi = np.zeros((L, H, D))
    vi[np.arange(L), :, np.arange(L)] = 1.0
    for causal in (False, True):
        A, _ = oracle_mod.attention(q, k, vi, causal=causal)
        A = A[:, :, :L]
        assert np.all(A >= 0)
        np.testing.assert_allclose(A.sum(-1), 1.0, rtol=0, atol=1e-13)
        if causal:
            assert np.all(A[np.triu_indices(L, 1)[0], :, np.triu_indices(L, 1)[1]] == 0)


def test_single_token_returns_value_row(oracle_mod):
    q, k, v = inputs.qkv(1, 3, 64, seed=2)
    for causal in (False, True):
        o, l = oracle_mod.attention(q, k, v, causal=causal)
        np.testing.assert_array_equal(o, v.astype(np.float64))
        s = (q.astype(np.float64) * k).sum(-1) / 8.0
        np.testing.assert_allclose(l, s.T, rtol=0, atol=1e-12)


def test_permutation_invariances(oracle_mod):
    L, H, D = 160, 2, 32
    q, k, v = inputs.qkv(L, H, D, seed=4)
    o, l = oracle_mod.attention(q, k, v)
    p = np.random.default_rng(0).permutation(L)
    o2, l2 = oracle_mod.attention(q, k[p], v[p])          # joint (K,V) row permutation
    np.testing.assert_allclose(o2, o, rtol=0, atol=1e-12)
    np.testing.assert_allclose(l2, l, rtol=0, atol=1e-12)
    o3, l3 = oracle_mod.attention(q[p], k, v)             # Q permutation -> output permuted
    np.testing.assert_allclose(o3, o[p], rtol=0, atol=1e-12)
    np.testing.assert_allclose(l3, l[:, p], rtol=0, atol=1e-12)


def test_key_shift_and_value_linearity(oracle_mod):
    L, H, D = 128, 2, 64
    q, k, v = (x.astype(np.float64) for x in inputs.qkv(L, H, D, seed=6))
    o, l = oracle_mod.attention(q, k, v, causal=True)
    c = np.random.default_rng(1).standard_normal((H, D))
    o2, l2 = oracle_mod.attention(q, k + c[None], v, causal=True)
    np.testing.assert_allclose(o2, o, rtol=0, atol=1e-11)
    shift = np.einsum("thd,hd->ht", q, c) / math.sqrt(D)
    np.testing.assert_allclose(l2, l + shift, rtol=0, atol=1e-11)
    v2 = np.random.default_rng(2).standard_normal(v.shape)
    oa, _ = oracle_mod.attention(q, k, 2.0 * v - 3.0 * v2, causal=True)
    ob, _ = oracle_mod.attention(q, k, v2, causal=True)
    np.testing.assert_allclose(oa, 2.0 * o - 3.0 * ob, rtol=0, atol=1e-11)


def test_large_scores_stay_finite(oracle_mod):
    """|scores| ~ 1e3: max-subtraction keeps fp64 finite; compare with the
    decimal brute force (which has no overflow at 50 digits)."""
    L, H, D = 6, 1, 4
    rng = np.random.default_rng(3)
    q, k, v = rng.standard_normal((L, H, D)) * 40, rng.standard_normal((L, H, D)) * 40, rng.standard_normal((L, H, D))
    o, l = oracle_mod.attention(q, k, v)
    assert np.all(np.isfinite(o)) and np.all(np.isfinite(l))
    ro, rl = oracle_mod.attention_decimal(q, k, v)
    np.testing.assert_allclose(o, ro, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(l, rl, rtol=1e-13, atol=0)


def test_input_generator_is_bf16_exact_and_seeded():
    q, k, v = inputs.qkv(33, 2, 64, seed=99)
    for x in (q, k, v):
        assert np.all((x.view(np.uint32) & 0xFFFF) == 0)
        t = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
        np.testing.assert_array_equal(t, x)
    q2, _, _ = inputs.qkv(33, 2, 64, seed=99)
    np.testing.assert_array_equal(q, q2)
    assert abs(float(q.std()) - 1.0) < 0.05


def test_mha_layer_oracle_reduces_to_attention_with_identity_weights(oracle_mod):
    """NEXT-3 oracle pin: with W_Q = W_K = W_V = W_0 = I (d_model = H*D) the
    layer is the attention of X with itself, up to the bf16 storage of Z."""
    L, H, D = 64, 2, 8
    x = inputs.normal((L, H * D), 5, 0)
    I = np.eye(H * D)
    y, lse = oracle_mod.mha_layer(x, I, I, I, I, H, D, causal=True)
    xr = x.astype(np.float64).reshape(L, H, D)
    z, l2 = oracle_mod.attention(xr, xr, xr, True)
    np.testing.assert_allclose(y, oracle_mod.round_bf16(z).reshape(L, H * D), rtol=0, atol=0)
    np.testing.assert_allclose(lse, l2, rtol=0, atol=0)
    # W_V = 0 -> Y = 0 exactly; W_0 linear: Y(2 W_0) = 2 Y(W_0)
    y0, _ = oracle_mod.mha_layer(x, I, I, 0 * I, I, H, D)
    assert np.all(y0 == 0)
    wo = np.random.default_rng(0).standard_normal((H * D, 5))
    ya, _ = oracle_mod.mha_layer(x, I, I, I, wo, H, D)
    yb, _ = oracle_mod.mha_layer(x, I, I, I, 2 * wo, H, D)
    np.testing.assert_allclose(yb, 2 * ya, rtol=0, atol=1e-12)


def test_round_bf16_matches_torch():
    from oracle import oracle
    a = np.random.default_rng(1).standard_normal(1000).astype(np.float32) * 100
    np.testing.assert_array_equal(oracle.round_bf16(a),
                                  torch.from_numpy(a).to(torch.bfloat16).double().numpy())


def test_fp32_input_entry_identical_to_fp64(oracle_mod):
    """oracle_attention_f32in (fp32 inputs widened on load, used for the
    GiB-sized sampled-parity configs) gives the same bits as the fp64 entry."""
    q, k, v = inputs.qkv(333, 3, 64, seed=21)
    rows = np.array([0, 5, 100, 332], dtype=np.int64)
    for causal in (False, True):
        a = oracle_mod.attention(q, k, v, causal, rows=rows, key_range=(7, 300))
        b = oracle_mod.attention(*(x.astype(np.float64) for x in (q, k, v)), causal, rows=rows,
                                 key_range=(7, 300))
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
