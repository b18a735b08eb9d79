"""Seeded random sweep of the whole path against the fp64 oracle.

Each case draws (L, H, D, causal, P, layout) from a fixed seed — ragged
lengths, single-row and single-tile cases, odd world sizes, both layouts — and
runs the default kernels through the C ABI: one dmha_forward at P = 1 (which
may take the split-KV route on small grids), or the P-rank ring schedule
emulated on one GPU (same kernels, position maps and fused combine as the
NCCL ring).  Every output row and lse is compared with the oracle at the
north_star bf16 tolerance.
"""
import numpy as np
import pytest

from synth import inputs
from tests.parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2302_06218_b200 import dmha  # noqa: E402


def _cases(n=48, seed=20261018):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        P = int(rng.choice([1, 1, 2, 3, 4]))
        layout = str(rng.choice(["contiguous", "zigzag"])) if P > 1 else "contiguous"
        div = 2 * P if layout == "zigzag" else P
        L = int(rng.integers(1, 6000 // div + 1)) * div
        H = int(rng.integers(1, 5))
        D = int(rng.choice([64, 128]))
        causal = bool(rng.integers(0, 2))
        out.append((i, L, H, D, causal, P, layout))
    return out


@pytest.fixture(scope="module", autouse=True)
def _lib():
    dmha.init(1, 0, None, 0, "bf16", "contiguous")
    yield
    dmha.finalize()


@pytest.mark.parametrize("i,L,H,D,causal,P,layout", _cases())
def test_random_configuration(oracle_mod, i, L, H, D, causal, P, layout):
    q, k, v = inputs.qkv(L, H, D, seed=7000 + i)
    if P == 1:
        dq, dk, dv = (torch.from_numpy(x).to(torch.bfloat16).cuda() for x in (q, k, v))
        out, lse = dmha.forward(dq, dk, dv, L, causal)
        torch.cuda.synchronize()
        got_o, got_l = out.float().cpu().numpy(), lse.cpu().numpy()
    else:
        parts = [np.stack([dmha.shard(x, P, r, layout) for r in range(P)]) for x in (q, k, v)]
        dq, dk, dv = (torch.from_numpy(x).to(torch.bfloat16).cuda() for x in parts)
        out, lse = dmha.forward_emulated(P, layout, dq, dk, dv, L, causal)
        torch.cuda.synchronize()
        got_o = dmha.unshard(list(out.float().cpu().numpy()), L, layout)
        got_l = dmha.unshard([x.T for x in lse.cpu().numpy()], L, layout).T
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(got_o, got_l, ref_o, ref_l, "bf16",
                  f"case {i}: L={L} H={H} D={D} causal={causal} P={P} {layout}")
