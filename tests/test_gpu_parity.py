"""GPU parity of the CUDA path (through the C ABI) against the fp64 CPU oracle.

Run on a B200 with ``pytest -m gpu``.  Inputs are the seeded synthetic
generators of synth/inputs.py; the oracle is oracle/ (never the CUDA path).
"""
import math

import numpy as np
import pytest

from synth import inputs
from tests.parity import TOL, assert_parity, metrics

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2302_06218_b200 import dmha  # noqa: E402


_STATE = {"dtype": None}


def ensure_lib(dtype):
    """(Re)initialise the library for `dtype` (it holds one global state)."""
    if _STATE["dtype"] != dtype:
        if _STATE["dtype"] is not None:
            dmha.finalize()
        dmha.init(1, 0, None, 0, dtype, "contiguous")
        _STATE["dtype"] = dtype


@pytest.fixture(scope="module", autouse=True)
def _teardown():
    yield
    if _STATE["dtype"] is not None:
        dmha.finalize()
        _STATE["dtype"] = None


@pytest.fixture
def lib_bf16():
    ensure_lib("bf16")


def to_dev(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dtype).cuda()


def run_p1(q, k, v, causal, dtype=torch.bfloat16):
    L = q.shape[0]
    out, lse = dmha.forward(to_dev(q, dtype), to_dev(k, dtype), to_dev(v, dtype), L, causal)
    torch.cuda.synchronize()
    return out.float().cpu().numpy(), lse.cpu().numpy()


SMALL = [  # (L, H, D): ragged tails, single tile, several tiles, L=1
    (1, 1, 64), (1, 2, 128), (37, 2, 64), (128, 1, 64), (200, 3, 128), (256, 2, 64),
    (300, 1, 128), (777, 2, 64), (1000, 2, 128), (2085, 2, 64), (4096, 1, 128),
]


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("L,H,D", SMALL)
def test_p1_small_full_oracle(lib_bf16, oracle_mod, L, H, D, causal):
    q, k, v = inputs.qkv(L, H, D, seed=1000 + L + D)
    out, lse = run_p1(q, k, v, causal)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(out, lse, ref_o, ref_l, "bf16", f"L={L} H={H} D={D} causal={causal}")


def _sample_rows(L, bounds, n_rand=128, seed=0):
    rows = set(range(0, min(64, L))) | set(range(max(0, L - 64), L))
    for b in bounds:
        rows |= set(range(max(0, b - 32), min(L, b + 32)))
    rows |= set(np.random.default_rng(seed).integers(0, L, n_rand).tolist())
    return np.array(sorted(rows), dtype=np.int64)


@pytest.mark.parametrize("causal", [False, True])
def test_config_c2_sampled(lib_bf16, oracle_mod, causal):
    """C2: L=16384, D=64, H=8, bf16, P=1 (BASELINE.json configs[1])."""
    L, H, D = 16384, 8, 64
    q, k, v = inputs.qkv(L, H, D, seed=1235)
    out, lse = run_p1(q, k, v, causal)
    rows = _sample_rows(L, [128 * i for i in range(1, L // 128, 17)], 256)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal, rows=rows)
    assert_parity(out[rows], lse[:, rows], ref_o, ref_l, "bf16", f"C2 causal={causal}")


def test_zero_query_prefix_mean_and_one_hot(lib_bf16, oracle_mod):
    L, H, D = 1000, 2, 64
    _, k, v = inputs.qkv(L, H, D, seed=3)
    out, lse = run_p1(np.zeros_like(k), k, v, True)
    cnt = np.arange(1, L + 1)
    ref = np.cumsum(v.astype(np.float64), 0) / cnt[:, None, None]
    ma, rel = metrics(out, ref)
    assert ma <= 2e-2 and rel <= 5e-3
    np.testing.assert_allclose(lse, np.log(cnt)[None].repeat(H, 0), atol=1e-4)
    targets = np.random.default_rng(5).permutation(L)[:D]
    q1, k1, v1 = inputs.one_hot_selector(L, H, D, targets)
    out1, _ = run_p1(q1, k1, v1, False)
    sel = v1[targets[np.arange(L) % D]]
    # selected value row, up to bf16 output rounding (|v| < 8 -> half-ulp <= 2^-6)
    np.testing.assert_allclose(out1, sel, atol=2 ** -6 + 1e-6, rtol=0)


def test_peaky_scores_finite_and_ulp_bound(lib_bf16, oracle_mod):
    """Large scores (q x 16): no NaN/Inf; |err| <= 2^-8 |ref| + 2^-8 max|v|."""
    L, H, D = 1500, 2, 128
    q, k, v = inputs.qkv(L, H, D, seed=8, q_scale=16.0)
    for causal in (False, True):
        out, lse = run_p1(q, k, v, causal)
        ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
        assert np.all(np.isfinite(out)) and np.all(np.isfinite(lse))
        bound = 2 ** -8 * np.abs(ref_o) + 2 ** -8 * np.abs(v).max()
        assert np.all(np.abs(out - ref_o) <= bound)
        assert np.max(np.abs(lse - ref_l)) <= 1e-3  # reading R15


def test_deterministic_and_host_path_identical(lib_bf16):
    L, H, D = 3000, 2, 128
    q, k, v = inputs.qkv(L, H, D, seed=77)
    a_o, a_l = run_p1(q, k, v, True)
    b_o, b_l = run_p1(q, k, v, True)
    np.testing.assert_array_equal(a_o, b_o)
    np.testing.assert_array_equal(a_l, b_l)
    hq, hk, hv = (torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in (q, k, v))
    ho, hl = dmha.forward_host(hq, hk, hv, L, True)
    np.testing.assert_array_equal(ho.float().numpy(), a_o)
    np.testing.assert_array_equal(hl.numpy(), a_l)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("layout", ["contiguous", "zigzag"])
@pytest.mark.parametrize("causal", [False, True])
def test_emulated_ring_matches_oracle(lib_bf16, oracle_mod, P, layout, causal):
    L, H, D = 2048 + 64 * P, 2, 64 if P != 4 else 128
    q, k, v = inputs.qkv(L, H, D, seed=500 + P)
    parts = [[dmha.shard(x, P, r, layout) for r in range(P)] for x in (q, k, v)]
    dq, dk, dv = (to_dev(np.stack(p)) for p in parts)
    out, lse = dmha.forward_emulated(P, layout, dq, dk, dv, L, causal)
    torch.cuda.synchronize()
    out_g = dmha.unshard([o for o in out.float().cpu().numpy()], L, layout)
    lse_g = dmha.unshard([l.T for l in lse.cpu().numpy()], L, layout).T
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(out_g, lse_g, ref_o, ref_l, "bf16", f"ring P={P} {layout} causal={causal}")
    # SURVEY §8(c) accounting, exact and per forward: each of the P emulated
    # ranks sends (P-1) K/V blocks of 2 * L_loc*H*D*2 bytes, one exchange per step
    st = dmha.get_stats()
    assert st["last_bytes_sent"] == P * (P - 1) * 2 * (L // P) * H * D * 2
    assert st["last_exchanges"] == P * (P - 1)


def _ring_by_steps(P, layout, dq, dk, dv, L, causal, monkeypatch):
    """The ring composed step by step from the exported a2 / a4 entry points,
    in Python: rank r at step s attends its q to rank (r - s) mod P's K/V
    IN PLACE (no ring buffers, no comm stream) with the global position maps
    of dmha_ring_plan_step, writes an fp32 partial and merges it with
    dmha_lse_combine (final at the last step)."""
    Pn, Lloc, H, D = dq.shape
    out = torch.empty_like(dq)
    lse = torch.empty((P, H, Lloc), dtype=torch.float32, device="cuda")
    o_acc = torch.empty((Lloc, H, D), dtype=torch.float32, device="cuda")
    l_acc = torch.empty((H, Lloc), dtype=torch.float32, device="cuda")
    o_p = torch.empty_like(o_acc)
    l_p = torch.empty_like(l_acc)
    for r in range(P):
        for s in range(P):
            pl = dmha.ring_plan(P, r, s, layout, L)
            qm = (pl["q_base0"], pl["q_base1"], pl["q_chunk"])
            km = (pl["k_base0"], pl["k_base1"], pl["k_chunk"])
            src = (r - s) % P
            assert pl["src"] == src
            dst_o, dst_l = (o_acc, l_acc) if s == 0 else (o_p, l_p)
            dmha.attention_local(dq[r], dk[src], dv[src], dst_o, dst_l, causal, qm, km, out_mode=1)
            if s > 0:
                dmha.lse_combine(o_acc, l_acc, o_p, l_p, out[r], lse[r], final=(s == P - 1))
    torch.cuda.synchronize()
    return out, lse


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("layout", ["contiguous", "zigzag"])
@pytest.mark.parametrize("causal", [False, True])
def test_buffered_ring_bit_identical_to_in_place_steps(lib_bf16, monkeypatch, P, layout, causal):
    """a3: dmha_forward_emulated runs the real ring loop (two K/V ring buffers,
    comm stream, recv / compute events, one cudaMemcpyAsync per K and V block)
    and must give exactly the bits of the same steps composed in Python on the
    source shards read in place (unfused combine == fused combine bit for bit,
    test_fused_combine_bit_identical_to_separate_pass)."""
    L, H, D = 2 * P * 300 + (0 if layout == "zigzag" else P * 37), 2, 64 if P != 4 else 128
    q, k, v = inputs.qkv(L, H, D, seed=5150 + P)
    parts = [[dmha.shard(x, P, r, layout) for r in range(P)] for x in (q, k, v)]
    dq, dk, dv = (to_dev(np.stack(p)) for p in parts)
    ring_o, ring_l = dmha.forward_emulated(P, layout, dq, dk, dv, L, causal)
    torch.cuda.synchronize()
    step_o, step_l = _ring_by_steps(P, layout, dq, dk, dv, L, causal, monkeypatch)
    np.testing.assert_array_equal(ring_o.float().cpu().numpy(), step_o.float().cpu().numpy())
    np.testing.assert_array_equal(ring_l.cpu().numpy(), step_l.cpu().numpy())


def test_fault_injection_turns_parity_red(lib_bf16, oracle_mod, monkeypatch):
    """DMHA_FAULT=perturb_lse adds 0.5 to each partial lse inside the combine
    (SURVEY §5 fault hook): the parity check must fail, then pass again."""
    P, layout, L, H, D = 4, "zigzag", 2048, 2, 64
    q, k, v = inputs.qkv(L, H, D, seed=4242)
    parts = [np.stack([dmha.shard(x, P, r, layout) for r in range(P)]) for x in (q, k, v)]
    dq, dk, dv = (to_dev(p) for p in parts)
    ref_o, ref_l = oracle_mod.attention(q, k, v, True)

    def run():
        o, l = dmha.forward_emulated(P, layout, dq, dk, dv, L, True)
        torch.cuda.synchronize()
        return (dmha.unshard(list(o.float().cpu().numpy()), L, layout),
                dmha.unshard([x.T for x in l.cpu().numpy()], L, layout).T)

    monkeypatch.setenv("DMHA_FAULT", "perturb_lse")
    bad_o, bad_l = run()
    with pytest.raises(AssertionError):
        assert_parity(bad_o, bad_l, ref_o, ref_l, "bf16", "faulty combine")
    ma, rel = metrics(bad_o, ref_o)
    assert rel > 5e-3  # the output itself is wrong, not just lse
    monkeypatch.delenv("DMHA_FAULT")
    good_o, good_l = run()
    assert_parity(good_o, good_l, ref_o, ref_l, "bf16", "fault removed")


@pytest.mark.parametrize("case", ["p1_split", "p1_nosplit", "emulated_p4", "emulated_p3_fp32"])
def test_workspace_bytes_equal_what_is_held(oracle_mod, case):
    """dmha_workspace_bytes is exactly what a fresh library holds after one
    forward (SURVEY §8(c) accounting; the P = 1 split-KV partials included)."""
    if _STATE["dtype"] is not None:
        dmha.finalize()
        _STATE["dtype"] = None
    dtype = "fp32" if case.endswith("fp32") else "bf16"
    tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
    dmha.init(1, 0, None, 0, dtype, "contiguous")
    try:
        if case.startswith("p1"):
            L, H, D = (16384, 8, 64) if case == "p1_split" else (65536, 16, 128)
            q = torch.randn((L, H, D), device="cuda").to(tdt)
            dmha.forward(q, q.clone(), q.clone(), L, False)
            torch.cuda.synchronize()
            want = dmha.workspace_bytes(L, D, H)
            assert (want > 0) == (case == "p1_split")
        else:
            P = 4 if case == "emulated_p4" else 3
            L, H, D = P * 1000, 2, 64
            q = torch.randn((P, L // P, H, D), device="cuda").to(tdt)
            dmha.forward_emulated(P, "contiguous", q, q.clone(), q.clone(), L, True)
            torch.cuda.synchronize()
            want = dmha.workspace_bytes(L, D, H, world_size=P)
            e = 2 if dtype == "bf16" else 4
            Ll = L // P
            parts = 1 if dtype == "bf16" else 2  # fused combine only on the bf16 path
            # fp32: + the 3xTF32 split K hi/lo [Ll, H, D] and V^T hi/lo [H, D, Ll up to x4]
            tf32 = 0 if dtype == "bf16" else 2 * Ll * H * D * 4 + 2 * H * D * (-(-Ll // 4) * 4) * 4
            assert want == 4 * Ll * H * D * e + parts * (Ll * H * D * 4 + Ll * H * 4) + tf32
        assert dmha.get_stats()["workspace_bytes"] == want
    finally:
        dmha.finalize()


def test_emulated_p1_bit_identical_to_forward(lib_bf16):
    L, H, D = 1024, 2, 128
    q, k, v = inputs.qkv(L, H, D, seed=9)
    a_o, a_l = run_p1(q, k, v, True)
    o, l = dmha.forward_emulated(1, "contiguous", to_dev(q[None]), to_dev(k[None]), to_dev(v[None]), L, True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(o[0].float().cpu().numpy(), a_o)
    np.testing.assert_array_equal(l[0].cpu().numpy(), a_l)


@pytest.mark.parametrize("D", [64, 128])
def test_lse_combine_kernel_against_oracle_partials(lib_bf16, oracle_mod, D):
    """Step a4/a5 alone: oracle partials over disjoint key ranges, merged on the
    GPU, must equal the oracle over all keys (includes -inf partials)."""
    L, H = 500, 3
    q, k, v = inputs.qkv(L, H, D, seed=31)
    cuts = [0, 100, 101, 350, L]
    parts = [oracle_mod.attention(q, k, v, True, key_range=(a, b)) for a, b in zip(cuts[:-1], cuts[1:])]
    o_acc = torch.from_numpy(parts[0][0].astype(np.float32)).cuda()
    l_acc = torch.from_numpy(parts[0][1].astype(np.float32)).cuda()
    out = torch.empty((L, H, D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((H, L), dtype=torch.float32, device="cuda")
    for i, (po, pl) in enumerate(parts[1:], start=1):
        dmha.lse_combine(o_acc, l_acc, torch.from_numpy(po.astype(np.float32)).cuda(),
                         torch.from_numpy(pl.astype(np.float32)).cuda(), out, lse,
                         final=(i == len(parts) - 1))
    torch.cuda.synchronize()
    ref_o, ref_l = oracle_mod.attention(q, k, v, True)
    assert_parity(out.float().cpu().numpy(), lse.cpu().numpy(), ref_o, ref_l, "bf16", "combine")


def test_attention_local_partial_with_global_positions(lib_bf16, oracle_mod):
    """Step a2 alone on a (query chunk, key chunk) pair with zigzag-style maps:
    fp32 partial output and -inf rows where no key is visible."""
    L, H, D = 1024, 2, 64
    q, k, v = inputs.qkv(L, H, D, seed=41)
    # query rows: global [128,256) then [768,896); keys: global [256,512)
    qidx = np.r_[128:256, 768:896]
    kidx = np.r_[256:512]
    out = torch.empty((len(qidx), H, D), dtype=torch.float32, device="cuda")
    lse = torch.empty((H, len(qidx)), dtype=torch.float32, device="cuda")
    dmha.attention_local(to_dev(q[qidx]), to_dev(k[kidx]), to_dev(v[kidx]), out, lse, causal=True,
                         qmap=(128, 768, 128), kmap=(256, 512, 256), out_mode=1)
    torch.cuda.synchronize()
    ref_o, ref_l = oracle_mod.attention(q, k, v, True, rows=qidx, key_range=(256, 512))
    o = out.cpu().numpy()
    l = lse.cpu().numpy()
    assert np.all(l[:, :128] == -np.inf) and np.all(o[:128] == 0)
    assert_parity(o, l, ref_o, ref_l, "bf16", "local partial")


@pytest.mark.parametrize("causal", [False, True])
def test_fp32_path_config_c1(oracle_mod, causal):
    """C1: L=512, D=64, H=4, fp32, rel L2 <= 1e-4 (BASELINE.json configs[0])."""
    ensure_lib("fp32")
    if True:
        L, H, D = 512, 4, 64
        q, k, v = inputs.qkv(L, H, D, seed=1234, dtype="fp32")
        out, lse = run_p1(q, k, v, causal, torch.float32)
        ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
        assert_parity(out, lse, ref_o, ref_l, "fp32", f"C1 causal={causal}")
        # fp32 ring emulation at P=4 as well
        P = 4
        parts = [np.stack([dmha.shard(x, P, r, "zigzag") for r in range(P)]) for x in (q, k, v)]
        o4, l4 = dmha.forward_emulated(P, "zigzag", *(to_dev(p, torch.float32) for p in parts), L, causal)
        torch.cuda.synchronize()
        og = dmha.unshard(list(o4.cpu().numpy()), L, "zigzag")
        lg = dmha.unshard([x.T for x in l4.cpu().numpy()], L, "zigzag").T
        assert_parity(og, lg, ref_o, ref_l, "fp32", "C1 ring P=4")


def test_error_codes(lib_bf16):
    x = torch.zeros((64, 2, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(dmha.DmhaError) as e:
        dmha.forward(x, x, x, 64, False, out=x)  # out aliases q
    assert e.value.code == dmha.ERR_INVALID
    y = torch.zeros((64, 2, 96), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(dmha.DmhaError) as e:
        dmha.forward(y, y, y, 64, False)
    assert e.value.code == dmha.ERR_UNSUPPORTED
    with pytest.raises(dmha.DmhaError) as e:
        dmha.forward_emulated(3, "contiguous", *(torch.zeros((3, 10, 2, 64), dtype=torch.bfloat16,
                                                            device="cuda") for _ in range(3)), 31, False)
    assert e.value.code == dmha.ERR_INVALID


# (P, H, D): row segments of H/P heads x D bf16 = 16 vectors (flat copy path),
# 64 vectors and 24 vectors (not a power of two: warp-per-row path)
@pytest.mark.parametrize("P,H,D", [(2, 4, 64), (4, 4, 128), (2, 8, 128), (2, 6, 64)])
@pytest.mark.parametrize("layout", ["contiguous", "zigzag"])
@pytest.mark.parametrize("causal", [False, True])
def test_headpar_emulated_matches_oracle_and_ring(lib_bf16, oracle_mod, P, H, D, layout, causal):
    """NEXT-1, the paper's own exchange: head-parallel all-to-all
    path vs the oracle, and vs the ring (two distributions, one result)."""
    L = 2048 + 128 * P
    q, k, v = inputs.qkv(L, H, D, seed=600 + P)
    parts = [np.stack([dmha.shard(x, P, r, layout) for r in range(P)]) for x in (q, k, v)]
    dq, dk, dv = (to_dev(p) for p in parts)
    out, lse = dmha.forward_headpar_emulated(P, layout, dq, dk, dv, L, causal)
    torch.cuda.synchronize()
    og = dmha.unshard(list(out.float().cpu().numpy()), L, layout)
    lg = dmha.unshard([x.T for x in lse.cpu().numpy()], L, layout).T
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(og, lg, ref_o, ref_l, "bf16", f"headpar P={P} {layout} causal={causal}")
    ro, rl = dmha.forward_emulated(P, layout, dq, dk, dv, L, causal)
    torch.cuda.synchronize()
    ma, rel = metrics(out.float().cpu().numpy(), ro.float().cpu().numpy())
    assert ma <= 2e-2 and rel <= 5e-3


def test_headpar_requires_divisible_heads(lib_bf16):
    x = torch.zeros((2, 64, 3, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(dmha.DmhaError) as e:
        dmha.forward_headpar_emulated(2, "contiguous", x, x.clone(), x.clone(), 128, False)
    assert e.value.code == dmha.ERR_INVALID


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("D", [64, 128])
def test_mha_layer_matches_oracle(lib_bf16, oracle_mod, causal, D):
    """NEXT-3: the full layer (tcgen05 projection GEMMs + our attention) vs the
    oracle layer with the same bf16 storage points (reading R17)."""
    L, H, d_model = 1000, 4, 256
    x, wq, wk, wv, wo = inputs.mha_layer(L, d_model, H, D)
    dev = [to_dev(a) for a in (x, wq, wk, wv, wo)]
    lse = torch.empty((H, L), dtype=torch.float32, device="cuda")
    y = dmha.mha_forward(*dev, L, H, D, causal, lse=lse)
    torch.cuda.synchronize()
    ref_y, ref_l = oracle_mod.mha_layer(x, wq, wk, wv, wo, H, D, causal)
    yo = y.float().cpu().numpy()
    ma, rel = metrics(yo, ref_y)
    assert rel <= 5e-3 and ma <= 2e-2, (ma, rel)
    assert np.max(np.abs(lse.cpu().numpy() - ref_l)) <= 1e-3  # reading R15


@pytest.mark.parametrize("P,layout,causal,D", [(2, "contiguous", False, 128), (4, "zigzag", True, 64),
                                               (8, "zigzag", True, 128), (3, "contiguous", True, 64)])
def test_fused_combine_bit_identical_to_separate_pass(lib_bf16, oracle_mod, monkeypatch, P,
                                                      layout, causal, D):
    """NEXT-2: the epilogue-fused LSE combine (default) gives exactly the bits
    of the separate lse_combine pass (shared combine_math.cuh, _rn arithmetic),
    and both match the oracle."""
    H = 2
    L = P * 777 if layout == "contiguous" else 2 * P * 389  # ragged shards
    q, k, v = inputs.qkv(L, H, D, seed=900 + P)
    parts = [[dmha.shard(x, P, r, layout) for r in range(P)] for x in (q, k, v)]
    dq, dk, dv = (to_dev(np.stack(p)) for p in parts)
    res = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("DMHA_FUSED_COMBINE", fused)
        o, l = dmha.forward_emulated(P, layout, dq, dk, dv, L, causal)
        torch.cuda.synchronize()
        res[fused] = (o.float().cpu().numpy(), l.cpu().numpy())
    np.testing.assert_array_equal(res["1"][0], res["0"][0])
    np.testing.assert_array_equal(res["1"][1], res["0"][1])
    out_g = dmha.unshard(list(res["1"][0]), L, layout)
    lse_g = dmha.unshard([x.T for x in res["1"][1]], L, layout).T
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(out_g, lse_g, ref_o, ref_l, "bf16", f"fused ring P={P} {layout} causal={causal}")



@pytest.mark.parametrize("causal", [False, True])
def test_host_path_pipelined(lib_bf16, oracle_mod, monkeypatch, causal):
    """dmha_forward_host at world size 1 and L >= 65536 pipelines the copies:
    Q chunk 0 (all of Q when causal) is attended over K/V blocks as they land
    (the ring's fused combine), later chunks over all keys.  Later chunks must
    carry the bits of the device path; every sampled row must match the
    oracle."""
    L, H, D = 70000, 2, 64
    monkeypatch.setenv("DMHA_KV_SPLIT", "0")  # compare with the one-launch device path
    q, k, v = inputs.qkv(L, H, D, seed=71)
    a_o, a_l = run_p1(q, k, v, causal)
    hq, hk, hv = (torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in (q, k, v))
    ho, hl = dmha.forward_host(hq, hk, hv, L, causal)
    ho = ho.float().numpy()
    hl = hl.numpy()
    half = L // 2 + 256  # past the first chunk (at most ceil(L/2) rounded up to 256 rows)
    if not causal:  # causal runs split only the keys (all rows combined), see dmha.h
        np.testing.assert_array_equal(ho[half:], a_o[half:])
        np.testing.assert_array_equal(hl[:, half:], a_l[:, half:])
    rows = _sample_rows(L, [17408, 35072, half], 128, seed=2)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal, rows=rows)
    assert_parity(ho[rows], hl[:, rows], ref_o, ref_l, "bf16", f"host pipelined causal={causal}")


@pytest.mark.parametrize("env", [{"DMHA_ISSUERS": "1"}, {"DMHA_ISSUERS": "2"}, {"DMHA_ISSUERS": "4"},
                                 {"DMHA_EMU": "1"}, {"DMHA_EMU": "2"}, {"DMHA_EMU": "3"},
                                 {"DMHA_SPLIT": "1"}, {"DMHA_SPLIT": "0"}, {"DMHA_PS": "0"},
                                 {"DMHA_PS": "1"}, {"DMHA_PS": "1", "DMHA_ISSUERS": "2"},
                                 {"DMHA_PS": "1", "DMHA_ISSUERS": "3"}, {"DMHA_PS": "1", "DMHA_ISSUERS": "4"},
                                 {"DMHA_PS": "1", "DMHA_EMU": "2"}])
@pytest.mark.parametrize("L,H,D,causal", [(777, 2, 64, True), (1000, 2, 128, False), (2085, 1, 64, False)])
def test_measurement_knobs_keep_parity(lib_bf16, oracle_mod, monkeypatch, env, L, H, D, causal):
    """Every kernel knob DESIGN.md reports a measurement for stays correct."""
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    q, k, v = inputs.qkv(L, H, D, seed=31 + L)
    out, lse = run_p1(q, k, v, causal)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(out, lse, ref_o, ref_l, "bf16", f"{env} L={L} D={D} causal={causal}")


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("D", [64, 128])
def test_kv_split_small_grid(lib_bf16, oracle_mod, monkeypatch, causal, D):
    """Small grids split each row block's keys over two CTAs and merge the fp32
    partials (log-sum-exp combine); the result matches the oracle and, within
    the tolerance, the unsplit launch."""
    L, H = 5000, 3
    q, k, v = inputs.qkv(L, H, D, seed=41 + D)
    a_o, a_l = run_p1(q, k, v, causal)  # split (L*H small)
    monkeypatch.setenv("DMHA_KV_SPLIT", "0")
    b_o, b_l = run_p1(q, k, v, causal)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(a_o, a_l, ref_o, ref_l, "bf16", f"kv split D={D} causal={causal}")
    assert_parity(b_o, b_l, ref_o, ref_l, "bf16", f"unsplit D={D} causal={causal}")


@pytest.mark.parametrize("env", [{"DMHA_PS": "0"}, {"DMHA_PS": "1"}, {"DMHA_PS": "1", "DMHA_ISSUERS": "2"}])
@pytest.mark.parametrize("P,layout,causal", [(4, "zigzag", True), (3, "contiguous", False)])
def test_d128_schedules_on_the_ring(lib_bf16, oracle_mod, monkeypatch, env, P, layout, causal):
    """The D = 128 schedules (P over S in TMEM, or P in shared memory) on the
    ring path: global-position masks, fused combine, ragged shards."""
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    H, D = 2, 128
    L = 2 * P * 389 if layout == "zigzag" else P * 777
    q, k, v = inputs.qkv(L, H, D, seed=1700 + P)
    parts = [np.stack([dmha.shard(x, P, r, layout) for r in range(P)]) for x in (q, k, v)]
    out, lse = dmha.forward_emulated(P, layout, *(to_dev(x) for x in parts), L, causal)
    torch.cuda.synchronize()
    og = dmha.unshard(list(out.float().cpu().numpy()), L, layout)
    lg = dmha.unshard([x.T for x in lse.cpu().numpy()], L, layout).T
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(og, lg, ref_o, ref_l, "bf16", f"{env} ring P={P} {layout} causal={causal}")


FP32_SHAPES = [(1, 1, 64), (37, 2, 64), (128, 1, 128), (200, 3, 128), (512, 4, 64), (777, 2, 64),
               (1000, 2, 128), (4133, 2, 64), (2085, 2, 128), (1, 2, 128), (33, 64, 64)]


@pytest.mark.parametrize("simt", [False, True])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("L,H,D", FP32_SHAPES)
def test_fp32_path_tf32x3_and_simt(oracle_mod, monkeypatch, simt, causal, L, H, D):
    """The fp32 path: 3xTF32 tcgen05 kernel (default) and the SIMT fp32
    cross-check (DMHA_FP32_SIMT=1), ragged and tiny shapes, both head dims,
    against the fp64 oracle at the fp32 tolerance (rel L2 <= 1e-4)."""
    ensure_lib("fp32")
    if simt:
        monkeypatch.setenv("DMHA_FP32_SIMT", "1")
    q, k, v = inputs.qkv(L, H, D, seed=2100 + L + D, dtype="fp32")
    out, lse = run_p1(q, k, v, causal, torch.float32)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(out, lse, ref_o, ref_l, "fp32", f"fp32 simt={simt} L={L} H={H} D={D} causal={causal}")


@pytest.mark.parametrize("L,H,D,causal", [(16384, 8, 64, False), (16384, 8, 64, True),
                                          (8269, 4, 128, True)])
def test_fp32_path_large_sampled(oracle_mod, L, H, D, causal):
    """The fp32 path at C2's shape in fp32 (and D = 128 with a ragged tail):
    hundreds of key tiles through the 3xTF32 kernel's K / V^T rings, the
    double-buffered S / P and the lazy rescale; sampled rows (first / last
    128, CTA boundaries, random) against the fp64 oracle over all keys at the
    fp32 tolerance."""
    ensure_lib("fp32")
    q, k, v = inputs.qkv(L, H, D, seed=3100 + D + int(causal), dtype="fp32")
    out, lse = run_p1(q, k, v, causal, torch.float32)
    rows = set(range(128)) | set(range(L - 128, L))
    for b in range(128, L, 128 * 13):
        rows |= {b - 1, b}
    rows |= set(np.random.default_rng(7).integers(0, L, 64).tolist())
    rows = np.array(sorted(rows), dtype=np.int64)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal, rows=rows)
    assert_parity(out[rows], lse[:, rows], ref_o, ref_l, "fp32", f"fp32 L={L} H={H} D={D} causal={causal}")


def test_fp32_tf32x3_beats_one_pass_tf32_bound(oracle_mod):
    """3xTF32 is what makes rel L2 <= 1e-4 reachable (R13: one-pass
    TF32 measured 4.3e-4 in SURVEY's emulation); the kernel's error must sit
    near fp32 rounding, far below one-pass TF32."""
    ensure_lib("fp32")
    L, H, D = 512, 4, 64
    q, k, v = inputs.qkv(L, H, D, seed=1234, dtype="fp32")
    out, _ = run_p1(q, k, v, False, torch.float32)
    ref_o, _ = oracle_mod.attention(q, k, v, False)
    _, rel = metrics(out, ref_o)
    assert rel <= 1e-5, rel


@pytest.mark.parametrize("case", ["p1_split", "p1_large_grid", "emulated_p4"])
def test_forward_captures_into_cuda_graph(lib_bf16, case):
    """After dmha_reserve, a forward allocates nothing and is stream-ordered
    only, so it captures into a CUDA graph — at P = 1 (split-KV small grid:
    attention + combine; large grid: one launch) and the emulated P = 4 ring
    (comm stream, copies and events join the capture).  Replays on new input
    values equal eager forwards bit for bit."""
    if case == "p1_split":
        P, L, H, D, causal, layout = 1, 5000, 3, 64, False, "contiguous"
    elif case == "p1_large_grid":
        P, L, H, D, causal, layout = 1, 65536, 4, 128, True, "contiguous"
    else:
        P, L, H, D, causal, layout = 4, 4096, 2, 128, True, "zigzag"
    _graph_capture_case(P, L, H, D, causal, layout, torch.bfloat16, case)


@pytest.mark.parametrize("P,L,H,D,causal,layout", [(1, 3000, 3, 64, True, "contiguous"),
                                                   (3, 3001, 2, 128, False, "contiguous")])
def test_fp32_forward_captures_into_cuda_graph(P, L, H, D, causal, layout):
    """The fp32 path in a CUDA graph: dmha_reserve also pre-allocates the
    3xTF32 split-operand scratch, so the split pre-pass + attention (+ the
    ring's copies and combines) capture and replay bit-identically."""
    ensure_lib("fp32")
    _graph_capture_case(P, L, H, D, causal, layout, torch.float32, f"fp32 P={P}")


def _graph_capture_case(P, L, H, D, causal, layout, tdt, case):
    if P == 1:
        shape, lshape = (L, H, D), (H, L)
    else:
        rows = max(dmha.shard_rows(L, P, r, layout) for r in range(P))
        shape, lshape = (P, rows, H, D), (P, H, rows)
    q, k, v = (torch.empty(shape, dtype=tdt, device="cuda") for _ in range(3))
    out = torch.empty_like(q)
    lse = torch.empty(lshape, dtype=torch.float32, device="cuda")
    dmha.reserve(L, D, H, world_size=P)

    def fwd():
        if P == 1:
            dmha.forward(q, k, v, L, causal, out, lse)
        else:
            dmha.forward_emulated(P, layout, q, k, v, L, causal, out, lse)

    gen = torch.Generator(device="cuda").manual_seed(17)
    for x in (q, k, v):
        x.copy_(torch.randn(shape, generator=gen, device="cuda"))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fwd()  # warm-up outside the capture (function attributes, descriptors)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        fwd()
    for seed in (21, 22):
        for x in (q, k, v):
            x.copy_(torch.randn(shape, generator=gen.manual_seed(seed), device="cuda"))
        graph.replay()
        torch.cuda.synchronize()
        g_o, g_l = out.clone(), lse.clone()
        fwd()
        torch.cuda.synchronize()
        assert torch.equal(g_o, out) and torch.equal(g_l, lse), f"{case} seed {seed}"


@pytest.mark.parametrize("P,extra,causal,D", [(3, 1, False, 64), (4, 3, True, 128), (5, 2, True, 64),
                                               (8, 5, False, 128), (2, 1, True, 64)])
def test_emulated_ring_uneven_shards(lib_bf16, oracle_mod, P, extra, causal, D):
    """Uneven contiguous shards (L % P != 0; SPEC S:438-446 equal-as-possible:
    the first L % P ranks hold one row more): the ring moves each block at its
    owner's size, ragged query/key tiles and global-position masks — against
    the oracle, and the exact per-forward byte count."""
    L, H = 300 * P + extra, 2
    q, k, v = inputs.qkv(L, H, D, seed=1900 + P + extra)
    parts = [dmha.stack_shards(x, P, "contiguous") for x in (q, k, v)]
    dmha.get_stats()
    out, lse = dmha.forward_emulated(P, "contiguous", *(to_dev(x) for x in parts), L, causal)
    torch.cuda.synchronize()
    og, lg = dmha.unstack_emulated(out.float().cpu().numpy(), lse.cpu().numpy(), L, "contiguous")
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(og, lg, ref_o, ref_l, "bf16", f"uneven ring P={P} L={L} causal={causal} D={D}")
    rows = [dmha.shard_rows(L, P, r, "contiguous") for r in range(P)]
    assert sorted(set(rows)) == sorted({L // P, L // P + 1})
    # the emulation sums every rank's sends: (P-1) blocks per rank, each block
    # sized by its owner
    sent = sum(rows[(r - s) % P] for r in range(P) for s in range(P - 1)) * H * D * 2 * 2
    assert dmha.get_stats()["last_bytes_sent"] == sent


@pytest.mark.parametrize("P,layout,causal,D,extra", [(4, "zigzag", True, 64, 0),
                                                     (3, "contiguous", True, 128, 2),
                                                     (2, "contiguous", False, 64, 1)])
def test_fp32_ring_emulated_many_tiles(oracle_mod, P, layout, causal, D, extra):
    """The fp32 path (3xTF32 kernel + separate log-sum-exp combine) through the
    emulated ring at sizes with many key tiles per step: zigzag key blocks
    (two chunks per block, global-position causal limits inside a tile),
    uneven contiguous shards, every step's split-operand pre-pass — against
    the fp64 oracle at the fp32 tolerance."""
    ensure_lib("fp32")
    L, H = 1024 * P + extra, 2
    q, k, v = inputs.qkv(L, H, D, seed=2700 + P + D, dtype="fp32")
    parts = [dmha.stack_shards(x, P, layout) for x in (q, k, v)]
    out, lse = dmha.forward_emulated(P, layout, *(to_dev(x, torch.float32) for x in parts), L, causal)
    torch.cuda.synchronize()
    og, lg = dmha.unstack_emulated(out.cpu().numpy(), lse.cpu().numpy(), L, layout)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(og, lg, ref_o, ref_l, "fp32", f"fp32 ring P={P} {layout} causal={causal} D={D}")


@pytest.mark.parametrize("P,layout,causal,D", [(2, "contiguous", False, 64), (4, "zigzag", True, 128)])
def test_headpar_emulated_fp32(oracle_mod, P, layout, causal, D):
    """NEXT-1 on the fp32 path: the pack / all-to-all / unpack kernels move
    4-byte elements and each rank's local attention (all L keys, H/P heads)
    runs the 3xTF32 kernel with its split-operand scratch sized for L keys —
    against the oracle at the fp32 tolerance."""
    ensure_lib("fp32")
    L, H = 1024 * P, 2 * P
    q, k, v = inputs.qkv(L, H, D, seed=650 + P, dtype="fp32")
    parts = [np.stack([dmha.shard(x, P, r, layout) for r in range(P)]) for x in (q, k, v)]
    out, lse = dmha.forward_headpar_emulated(P, layout, *(to_dev(p, torch.float32) for p in parts),
                                             L, causal)
    torch.cuda.synchronize()
    og = dmha.unshard(list(out.cpu().numpy()), L, layout)
    lg = dmha.unshard([x.T for x in lse.cpu().numpy()], L, layout).T
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(og, lg, ref_o, ref_l, "fp32", f"fp32 headpar P={P} {layout} causal={causal} D={D}")


@pytest.mark.parametrize("causal", [False, True])
def test_fp32_host_path_pipelined(oracle_mod, causal):
    """dmha_forward_host on the fp32 path at L >= 65536 (copies pipelined with
    Q row chunks; one K/V block, as the fp32 path has no fused combine): every
    row is attended over all keys in one launch, so the result equals the
    device path bit for bit; sampled rows against the oracle."""
    ensure_lib("fp32")
    L, H, D = 70000, 2, 64
    q, k, v = inputs.qkv(L, H, D, seed=72, dtype="fp32")
    a_o, a_l = run_p1(q, k, v, causal, torch.float32)
    hq, hk, hv = (torch.from_numpy(x).pin_memory() for x in (q, k, v))
    ho, hl = dmha.forward_host(hq, hk, hv, L, causal)
    ho, hl = ho.numpy(), hl.numpy()
    np.testing.assert_array_equal(ho, a_o)
    np.testing.assert_array_equal(hl, a_l)
    rows = _sample_rows(L, [17408, 35072], 64, seed=3)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal, rows=rows)
    assert_parity(ho[rows], hl[:, rows], ref_o, ref_l, "fp32", f"fp32 host pipelined causal={causal}")


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("L,P,causal", [(3, 4, False), (3, 4, True), (5, 8, True), (1, 2, False)])
def test_emulated_ring_empty_shards(oracle_mod, dtype, L, P, causal):
    """Fewer rows than ranks (SPEC's equal-as-possible partition leaves some
    contiguous shards empty): ring steps with zero query rows or zero keys
    must produce the exact result for the rows that exist."""
    ensure_lib(dtype)
    H, D = 2, 64
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q, k, v = inputs.qkv(L, H, D, seed=2900 + L * 10 + P, dtype=dtype)
    rows = [dmha.shard_rows(L, P, r, "contiguous") for r in range(P)]
    assert 0 in rows
    parts = [dmha.stack_shards(x, P, "contiguous") for x in (q, k, v)]
    out, lse = dmha.forward_emulated(P, "contiguous", *(to_dev(x, tdt) for x in parts), L, causal)
    torch.cuda.synchronize()
    og, lg = dmha.unstack_emulated(out.float().cpu().numpy(), lse.cpu().numpy(), L, "contiguous")
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(og, lg, ref_o, ref_l, dtype, f"empty shards {dtype} L={L} P={P} causal={causal}")
