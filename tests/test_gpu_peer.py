"""NEXT-2 peer-memory K/V transport (DMHA_TRANSPORT=peer): P real processes,
one library instance each, exchanging K/V by copy-engine pulls from CUDA-IPC
shared buffers with interprocess events and a shared-memory host barrier.

Run here with all ranks on ONE GPU (the pool gives one per call): the
processes never wait on each other inside a kernel — only streams wait on
events — so this is the multi-process protocol for real, just without
NVLink.  Checks: the output equals the single-GPU emulation of the same ring
bit for bit (same kernels, same block order), matches the fp64 oracle, and
the per-forward byte accounting is exact.
"""
import os
import socket
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

from synth import inputs
from tests.parity import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2302_06218_b200 import dmha  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_ranks(P, L, H, D, causal, layout, nfwd=3):
    d = tempfile.mkdtemp(prefix="dmha_peer_")
    port = _free_port()
    procs = []
    for r in range(P):
        env = dict(os.environ, DMHA_TRANSPORT="peer", RANK=str(r), WORLD_SIZE=str(P),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS="1")
        procs.append(subprocess.Popen(
            [sys.executable, str(ROOT / "tests" / "peer_rank.py"), d, str(L), str(H), str(D),
             str(int(causal)), layout, str(nfwd)], env=env, stdout=subprocess.PIPE,
            stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            pytest.fail("peer ranks timed out")
        outs.append(o)
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    res = [(np.load(f"{d}/out{r}.npy"), np.load(f"{d}/lse{r}.npy"), np.load(f"{d}/bytes{r}.npy"))
           for r in range(P)]
    return res


@pytest.mark.parametrize("P,layout,causal,D,extra", [(2, "contiguous", False, 128, 0),
                                                     (2, "zigzag", True, 64, 0),
                                                     (3, "contiguous", True, 64, 0),
                                                     (4, "zigzag", True, 128, 0),
                                                     (3, "contiguous", True, 128, 2)])
def test_peer_transport_processes(oracle_mod, P, layout, causal, D, extra):
    """extra > 0: uneven contiguous shards (L % P == extra)."""
    L, H = 256 * P * 2 + (0 if layout == "zigzag" else 64 * P) + extra, 2
    if layout == "zigzag":
        L -= L % (2 * P)
    res = _run_ranks(P, L, H, D, causal, layout)
    q, k, v = inputs.qkv(L, H, D, seed=4242)
    # reference 1: the single-GPU emulation of the same ring (bit-identical)
    dmha.init(1, 0, None, 0, "bf16", layout)
    try:
        parts = [dmha.stack_shards(x, P, layout) for x in (q, k, v)]
        dq, dk, dv = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in parts)
        eo, el = dmha.forward_emulated(P, layout, dq, dk, dv, L, causal)
        torch.cuda.synchronize()
        eo, el = eo.float().cpu().numpy(), el.cpu().numpy().reshape(P, -1)
        rows = [dmha.shard_rows(L, P, r, layout) for r in range(P)]
    finally:
        dmha.finalize()
    for r in range(P):
        np.testing.assert_array_equal(res[r][0], eo[r][:rows[r]])
        np.testing.assert_array_equal(res[r][1], el[r][:H * rows[r]].reshape(H, rows[r]))
        # exact accounting: P-1 sends, each of the block the rank holds at that
        # step (its owner's rows x H x D bf16, K and V)
        sent = sum(rows[(r - s) % P] for s in range(P - 1)) * H * D * 2 * 2
        assert int(res[r][2][0]) == sent and int(res[r][2][1]) == P - 1
    # reference 2: the fp64 oracle
    out = dmha.unshard([res[r][0] for r in range(P)], L, layout)
    lse = dmha.unshard([res[r][1].T for r in range(P)], L, layout).T
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    assert_parity(out, lse, ref_o, ref_l, "bf16", f"peer P={P} {layout} causal={causal} D={D}")
