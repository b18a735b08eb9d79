"""Parity helpers shared by the GPU tests (tolerances from BASELINE.json north_star).

bf16 path : max |out - oracle| <= 2e-2 and rel L2 <= 5e-3   (north_star)
fp32 path : rel L2 <= 1e-4                                 (north_star)
lse       : |lse - oracle| <= 1e-3 (bf16) / 1e-5 (fp32)     (reading R15)
The oracle runs in fp64 on the exact (bf16-rounded) values the GPU sees.
"""
from __future__ import annotations

import numpy as np

TOL = {
    "bf16": dict(max_abs=2e-2, rel_l2=5e-3, lse_abs=1e-3),
    "fp32": dict(max_abs=1e-3, rel_l2=1e-4, lse_abs=1e-5),
}


def metrics(out, ref):
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    diff = out - ref
    max_abs = float(np.max(np.abs(diff))) if diff.size else 0.0
    den = float(np.linalg.norm(ref))
    rel = float(np.linalg.norm(diff) / den) if den > 0 else float(np.linalg.norm(diff))
    return max_abs, rel


def assert_parity(out, lse, ref_out, ref_lse, dtype="bf16", what=""):
    t = TOL[dtype]
    out = np.asarray(out, dtype=np.float64)
    lse = np.asarray(lse, dtype=np.float64)
    assert np.all(np.isfinite(out)), f"{what}: non-finite output"
    max_abs, rel = metrics(out, ref_out)
    assert max_abs <= t["max_abs"], f"{what}: max abs {max_abs:.3e} > {t['max_abs']}"
    assert rel <= t["rel_l2"], f"{what}: rel L2 {rel:.3e} > {t['rel_l2']}"
    fin = np.isfinite(ref_lse)
    assert np.array_equal(np.isfinite(lse), fin), f"{what}: lse -inf pattern differs"
    if fin.any():
        lerr = float(np.max(np.abs(lse[fin] - ref_lse[fin])))
        assert lerr <= t["lse_abs"], f"{what}: lse abs err {lerr:.3e} > {t['lse_abs']}"
    return max_abs, rel
