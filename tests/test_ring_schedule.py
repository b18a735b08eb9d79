"""Multi-process CPU test of the ring distribution.

Real processes (torch.distributed, gloo, world size 2 and 4) follow the
library's own schedule (`dmha_ring_plan_step`, the function dmha_forward and
the GPU emulation execute) to pass K/V blocks around the ring with
send/recv, compute each step's partial with the CPU oracle over the block's
keys at the plan's GLOBAL positions, and merge the partials with the
log-sum-exp rule.  The merged result must equal the oracle over all keys —
this checks the schedule (who sends what to whom, which block is used at
each step, buffer reuse order) and the shard/position maps without a GPU.
The LSE merge written here is test code (north_star (3)), not the CUDA
combine, which is checked against oracle partials in test_gpu_parity.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rows_of(base0, base1, chunk, n):
    i = np.arange(n)
    return np.where(i < chunk, base0 + i, base1 + (i - chunk))


def _worker(rank, world, port, L, H, D, layout, causal, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2302_06218_b200 import dmha

    q, k, v = inputs.qkv(L, H, D, seed=4242)
    my_rows = dmha.global_rows(L, world, rank, layout)
    Lloc = len(my_rows)  # uneven contiguous shards: L/P or L/P + 1 rows
    assert Lloc == dmha.shard_rows(L, world, rank, layout)
    kv_cur = np.concatenate([k[my_rows], v[my_rows]]).astype(np.float32)  # step 0: own block
    ring = [None, None]
    o_acc = lse_acc = None
    for s in range(world):
        pl = dmha.ring_plan(world, rank, s, layout, L)
        q_glob = _rows_of(pl["q_base0"], pl["q_base1"], pl["q_chunk"], Lloc)
        assert np.array_equal(q_glob, my_rows)
        nk = dmha.shard_rows(L, world, pl["src"], layout)  # the block's owner's rows
        k_glob = _rows_of(pl["k_base0"], pl["k_base1"], pl["k_chunk"], nk)
        assert np.array_equal(k_glob, dmha.global_rows(L, world, pl["src"], layout))
        kv_use = kv_cur if pl["compute_buf"] < 0 else ring[pl["compute_buf"]]
        # the block really is the src rank's keys (data arrived through the ring)
        np.testing.assert_array_equal(kv_use[:nk], k[k_glob])
        # exchange for the next step (send current block, receive the next,
        # sized by ITS owner's rows)
        if pl["recv_buf"] >= 0:
            nxt = dmha.ring_plan(world, rank, s + 1, layout, L)["src"]
            recv = torch.empty(2 * dmha.shard_rows(L, world, nxt, layout), H, D)
            reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(kv_use)), pl["send_to"]),
                    dist.irecv(recv, pl["recv_from"])]
            for r_ in reqs:
                r_.wait()
            assert pl["recv_buf"] != pl["compute_buf"]  # never overwrite the block in use
            ring[pl["recv_buf"]] = recv.numpy()
        # partial over this block's keys at global positions (oracle on a gathered view)
        kk = np.zeros((L, H, D), np.float32)
        vv = np.zeros((L, H, D), np.float32)
        kk[k_glob] = kv_use[:nk]
        vv[k_glob] = kv_use[nk:]
        mask_keys = np.zeros(L, bool)
        mask_keys[k_glob] = True
        # contiguous key ranges of the block (one or two chunks)
        parts = []
        for a, b in _ranges(k_glob):
            parts.append(oracle.attention(q, kk, vv, causal, rows=my_rows, key_range=(a, b)))
        o_s, l_s = _merge_list(parts)
        if pl["output"] == dmha.PLAN_FINAL or pl["output"] == dmha.PLAN_ACC:
            o_acc, lse_acc = o_s, l_s
        else:
            o_acc, lse_acc = _merge(o_acc, lse_acc, o_s, l_s)
    np.save(os.path.join(out_dir, f"o{rank}.npy"), o_acc)
    np.save(os.path.join(out_dir, f"l{rank}.npy"), lse_acc)
    dist.destroy_process_group()


def _ranges(idx):
    idx = np.asarray(idx)
    cuts = np.where(np.diff(idx) != 1)[0]
    starts = np.r_[idx[0], idx[cuts + 1]]
    ends = np.r_[idx[cuts] + 1, idx[-1] + 1]
    return list(zip(starts.tolist(), ends.tolist()))


def _merge(oa, la, ob, lb):
    """log-sum-exp merge of two normalised partials; -inf weighs 0."""
    m = np.maximum(la, lb)
    safe = np.where(np.isfinite(m), m, 0.0)
    wa = np.where(np.isfinite(la), np.exp(la - safe), 0.0)
    wb = np.where(np.isfinite(lb), np.exp(lb - safe), 0.0)
    tot = wa + wb
    l = np.where(tot > 0, safe + np.log(np.where(tot > 0, tot, 1.0)), -np.inf)
    a = np.where(tot > 0, wa / np.where(tot > 0, tot, 1.0), 0.0)
    b = np.where(tot > 0, wb / np.where(tot > 0, tot, 1.0), 0.0)
    o = oa * a.T[:, :, None] + ob * b.T[:, :, None]
    return o, l


def _merge_list(parts):
    o, l = parts[0]
    for ob, lb in parts[1:]:
        o, l = _merge(o, l, ob, lb)
    return o, l


@pytest.mark.parametrize("world,layout,causal,extra", [(2, "contiguous", False, 0), (2, "zigzag", True, 0),
                                                        (4, "zigzag", True, 0), (4, "contiguous", True, 0),
                                                        (4, "contiguous", True, 3), (3, "contiguous", False, 1)])
def test_ring_over_gloo_matches_oracle(tmp_path, oracle_mod, world, layout, causal, extra):
    """extra > 0: L % P == extra, uneven contiguous shards."""
    L, H, D = 96 * world + extra, 2, 8
    port = _free_port()
    mp.spawn(_worker, args=(world, port, L, H, D, layout, causal, str(tmp_path)), nprocs=world, join=True)
    from paper_2302_06218_b200 import dmha
    q, k, v = inputs.qkv(L, H, D, seed=4242)
    ref_o, ref_l = oracle_mod.attention(q, k, v, causal)
    for r in range(world):
        rows = dmha.global_rows(L, world, r, layout)
        o = np.load(tmp_path / f"o{r}.npy")
        l = np.load(tmp_path / f"l{r}.npy")
        np.testing.assert_allclose(o, ref_o[rows], rtol=0, atol=1e-10)
        np.testing.assert_allclose(l, ref_l[:, rows], rtol=0, atol=1e-10)


def test_plan_structure_and_bytes():
    """Schedule invariants: every rank attends to every block exactly once,
    sends go to r+1 / receives come from r-1 on steps < P-1, a receive never
    targets the buffer being computed on, and the byte count is (P-1)*2*blk."""
    from paper_2302_06218_b200 import dmha
    for P in (1, 2, 3, 8):
        for layout in ("contiguous", "zigzag"):
            L = 16 * P
            for r in range(P):
                srcs = []
                for s in range(P):
                    pl = dmha.ring_plan(P, r, s, layout, L)
                    srcs.append(pl["src"])
                    if s < P - 1:
                        assert pl["send_to"] == (r + 1) % P and pl["recv_from"] == (r - 1) % P
                        assert pl["recv_buf"] != pl["compute_buf"]
                    else:
                        assert pl["send_to"] == -1 and pl["recv_buf"] == -1
                    exp_out = (dmha.PLAN_FINAL if P == 1 else dmha.PLAN_ACC if s == 0 else
                               dmha.PLAN_COMBINE_FINAL if s == P - 1 else dmha.PLAN_COMBINE)
                    assert pl["output"] == exp_out
                assert sorted(srcs) == list(range(P))
                # the block used at step s+1 is the one received at step s
                for s in range(P - 1):
                    a = dmha.ring_plan(P, r, s, layout, L)
                    b = dmha.ring_plan(P, r, s + 1, layout, L)
                    assert b["compute_buf"] == a["recv_buf"]
                    assert b["src"] == (a["src"] - 1) % P


def test_bench_gpus2_launches_two_ranks():
    """bench.py --gpus 2 without a torchrun environment re-launches itself
    under torch.distributed.run with two ranks (the driver's plain
    `python bench.py --gpus N` invocation); --launch-check makes every rank
    report and exit before touching a GPU."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["gpus"] == 2 for d in lines)
