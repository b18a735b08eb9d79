// peer_link.h — single-node peer-memory plumbing for the NEXT-2 K/V transport
// ("the devices exchange ... NCCL").
//
// Each rank publishes its K/V block in a library-owned buffer shared with the
// other processes through CUDA IPC; a peer PULLS the block it needs with the
// copy engine (cudaMemcpyAsync from the IPC-mapped pointer, over NVLink when
// the ranks sit on different GPUs).  No SMs are used for the transfer, no
// kernel waits on another rank, and every block crosses the link once,
// straight from its owner (no relay around the ring).
//
// Ordering between processes uses interprocess CUDA events ("published",
// "done pulling") whose record calls are made to precede the peers' waits by
// a host barrier in POSIX shared memory (ranks share one node).
// Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

namespace dmha {

struct PeerLink;

// Collective over the `world` ranks of one node: creates/opens the shared
// segment named after the 128-byte unique id, exchanges interprocess event
// handles.  Returns 0 or a negative DMHA_ERR_* code with *err set.
int peer_open(PeerLink** out, const void* unique_id, int world, int rank, int device,
              std::string* err);
// Collective: barrier, close peer mappings, free the published buffer.
void peer_close(PeerLink* pl);
// Host barrier over all ranks (bounded: fails after `timeout_s`).
int peer_barrier(PeerLink* pl, std::string* err, double timeout_s = 300.0);
// Collective: make the published buffer at least `bytes` (re-sharing it when
// it grows).  The same `bytes` on every rank.
int peer_ensure_pub(PeerLink* pl, size_t bytes, std::string* err);
// This rank's published buffer / rank r's buffer mapped into this process.
void* peer_local_pub(PeerLink* pl);
void* peer_pub(PeerLink* pl, int r);
// Interprocess events: rank r's "published" / "done pulling" (own if r == rank).
cudaEvent_t peer_pub_event(PeerLink* pl, int r);
cudaEvent_t peer_done_event(PeerLink* pl, int r);
size_t peer_pub_bytes(PeerLink* pl);

}  // namespace dmha
