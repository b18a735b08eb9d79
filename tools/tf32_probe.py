"""Isolation probe for the fp32 path: one case per process (run each under
`timeout`), printing the max error against a torch fp64 reference.

    python tools/tf32_probe.py <case>     cases: see CASES
"""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2302_06218_b200 import dmha  # noqa: E402

# name: (dtype, P, L, H, D, causal)
CASES = {
    "p1_small": ("fp32", 1, 128, 1, 64, False),
    "p1_c1": ("fp32", 1, 512, 4, 64, False),
    "p1_ragged_causal": ("fp32", 1, 1000, 2, 64, True),
    "p1_d128": ("fp32", 1, 256, 2, 128, False),
    "p1_d128_causal": ("fp32", 1, 300, 2, 128, True),
    "emu_p3": ("fp32", 3, 3000, 2, 64, True),
    "emu_p2": ("fp32", 2, 512, 2, 64, False),
    "bf16_emu_p3": ("bf16", 3, 3000, 2, 64, True),
}


def ref(q, k, v, causal):
    L, H, D = q.shape
    qd, kd, vd = (x.double().permute(1, 0, 2) for x in (q, k, v))
    s = qd @ kd.transpose(1, 2) / D ** 0.5
    if causal:
        s = s.masked_fill(torch.ones(L, L, dtype=torch.bool, device=q.device).triu(1), float("-inf"))
    return (torch.softmax(s, -1) @ vd).permute(1, 0, 2), torch.logsumexp(s, -1)


def main():
    name = sys.argv[1]
    dt, P, L, H, D, causal = CASES[name]
    dmha.init(1, 0, None, 0, dt, "contiguous")
    tdt = torch.float32 if dt == "fp32" else torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v = (torch.randn((L, H, D), generator=g, device="cuda").to(tdt) for _ in range(3))
    if P == 1:
        out, lse = dmha.forward(q, k, v, L, causal)
    else:
        sh = lambda x: x.view(P, L // P, H, D)  # noqa: E731  contiguous shards
        out, lse = dmha.forward_emulated(P, "contiguous", sh(q), sh(k), sh(v), L, causal)
        out = out.reshape(L, H, D)
        lse = lse.permute(1, 0, 2).reshape(H, L)
    torch.cuda.synchronize()
    ro, rl = ref(q, k, v, causal)
    err = (out.double() - ro).abs().max().item()
    rel = ((out.double() - ro).norm() / ro.norm()).item()
    lerr = (lse.double() - rl).abs().max().item()
    print(json.dumps({"case": name, "max_abs": err, "rel_l2": rel, "lse_err": lerr}), flush=True)
    dmha.finalize()


if __name__ == "__main__":
    main()
