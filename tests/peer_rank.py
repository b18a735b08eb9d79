"""One rank of the peer-transport test (tests/test_gpu_peer.py): run as a
separate process per rank, all on the same GPU (CUDA IPC works within one
device), DMHA_TRANSPORT=peer.  torch.distributed (gloo, 127.0.0.1) only
broadcasts the 128-byte unique id; no NCCL communicator is created.

    python tests/peer_rank.py <outdir> <L> <H> <D> <causal> <layout> <forwards>
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2302_06218_b200 import dmha  # noqa: E402
from synth import inputs  # noqa: E402


def main():
    outdir, L, H, D, causal, layout, nfwd = sys.argv[1:8]
    L, H, D, causal, nfwd = int(L), int(H), int(D), bool(int(causal)), int(nfwd)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    dmha.init_distributed("bf16", layout, 0)
    q, k, v = inputs.qkv(L, H, D, seed=4242)
    dq, dk, dv = (torch.from_numpy(dmha.shard(x, world, rank, layout)).cuda().to(torch.bfloat16)
                  for x in (q, k, v))
    for i in range(nfwd):  # repeated forwards exercise the published-buffer reuse protocol
        out, lse = dmha.forward(dq, dk, dv, L, causal)
    torch.cuda.synchronize()
    st = dmha.get_stats()
    np.save(os.path.join(outdir, f"out{rank}.npy"), out.float().cpu().numpy())
    np.save(os.path.join(outdir, f"lse{rank}.npy"), lse.cpu().numpy())
    np.save(os.path.join(outdir, f"bytes{rank}.npy"), np.array([st["last_bytes_sent"], st["last_exchanges"]]))
    dmha.finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
