// peer_link.cu — see peer_link.h (NEXT-2 peer-memory K/V transport plumbing).
#include "peer_link.h"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "dmha.h"

namespace dmha {

namespace {
constexpr int kMaxRanks = 64;

struct Slot {
  cudaIpcMemHandle_t mem;       // published buffer
  cudaIpcEventHandle_t ev_pub;  // "my block is published"
  cudaIpcEventHandle_t ev_done; // "I finished pulling"
  uint64_t pub_bytes;
  uint32_t mem_version;
  int device;
};

struct Shm {
  std::atomic<uint32_t> count;
  std::atomic<uint32_t> gen;
  Slot slot[kMaxRanks];
};
static_assert(std::atomic<uint32_t>::is_always_lock_free, "lock-free atomics needed in shared memory");
}  // namespace

struct PeerLink {
  int world = 1, rank = 0, device = 0;
  std::string name;
  Shm* shm = nullptr;
  void* pub = nullptr;  // own published buffer
  size_t pub_bytes = 0;
  uint32_t version = 0;
  std::vector<void*> peer_pub;        // mapped peer buffers (nullptr for self)
  std::vector<cudaEvent_t> ev_pub;    // own at [rank], opened handles otherwise
  std::vector<cudaEvent_t> ev_done;
};

namespace {
int failf(std::string* err, int code, const char* what, cudaError_t e = cudaSuccess) {
  char buf[256];
  snprintf(buf, sizeof(buf), "dmha peer link: %s%s%s", what, e != cudaSuccess ? ": " : "",
           e != cudaSuccess ? cudaGetErrorString(e) : "");
  if (err) *err = buf;
  return code;
}

void close_peer_maps(PeerLink* pl) {
  for (int r = 0; r < pl->world; ++r)
    if (r != pl->rank && pl->peer_pub[r]) {
      cudaIpcCloseMemHandle(pl->peer_pub[r]);
      pl->peer_pub[r] = nullptr;
    }
}
}  // namespace

int peer_barrier(PeerLink* pl, std::string* err, double timeout_s) {
  Shm* s = pl->shm;
  const uint32_t g0 = s->gen.load(std::memory_order_acquire);
  if (s->count.fetch_add(1, std::memory_order_acq_rel) == static_cast<uint32_t>(pl->world - 1)) {
    s->count.store(0, std::memory_order_relaxed);
    s->gen.fetch_add(1, std::memory_order_release);
    return DMHA_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t it = 0; s->gen.load(std::memory_order_acquire) == g0; ++it) {
    if ((it & 1023) == 0) {
      sched_yield();
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > timeout_s) return failf(err, DMHA_ERR_STATE, "host barrier timed out (a rank is missing)");
    }
  }
  return DMHA_OK;
}

int peer_open(PeerLink** out, const void* unique_id, int world, int rank, int device,
              std::string* err) {
  if (world > kMaxRanks) return failf(err, DMHA_ERR_UNSUPPORTED, "more than 64 ranks");
  auto* pl = new PeerLink();
  pl->world = world;
  pl->rank = rank;
  pl->device = device;
  // segment name from the unique id (identical on every rank, fresh per job)
  uint64_t h = 1469598103934665603ull;
  const auto* b = static_cast<const uint8_t*>(unique_id);
  for (int i = 0; i < 128; ++i) h = (h ^ b[i]) * 1099511628211ull;
  char nm[64];
  snprintf(nm, sizeof(nm), "/dmha_peer_%016llx", static_cast<unsigned long long>(h));
  pl->name = nm;
  const int fd = shm_open(nm, O_CREAT | O_RDWR, 0600);
  if (fd < 0) {
    delete pl;
    return failf(err, DMHA_ERR_STATE, "shm_open failed");
  }
  if (ftruncate(fd, sizeof(Shm)) != 0) {
    close(fd);
    delete pl;
    return failf(err, DMHA_ERR_STATE, "ftruncate of the shared segment failed");
  }
  void* m = mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) {
    delete pl;
    return failf(err, DMHA_ERR_STATE, "mmap of the shared segment failed");
  }
  pl->shm = static_cast<Shm*>(m);  // zero-filled on creation
  pl->peer_pub.assign(world, nullptr);
  pl->ev_pub.assign(world, nullptr);
  pl->ev_done.assign(world, nullptr);
  const unsigned flags = cudaEventDisableTiming | cudaEventInterprocess;
  cudaError_t e;
  if ((e = cudaEventCreateWithFlags(&pl->ev_pub[rank], flags)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&pl->ev_done[rank], flags)) != cudaSuccess) {
    peer_close(pl);
    return failf(err, DMHA_ERR_CUDA, "interprocess event creation", e);
  }
  Slot& me = pl->shm->slot[rank];
  if ((e = cudaIpcGetEventHandle(&me.ev_pub, pl->ev_pub[rank])) != cudaSuccess ||
      (e = cudaIpcGetEventHandle(&me.ev_done, pl->ev_done[rank])) != cudaSuccess) {
    peer_close(pl);
    return failf(err, DMHA_ERR_CUDA, "cudaIpcGetEventHandle", e);
  }
  me.device = device;
  if (int rc = peer_barrier(pl, err)) {
    peer_close(pl);
    return rc;
  }
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    if ((e = cudaIpcOpenEventHandle(&pl->ev_pub[r], pl->shm->slot[r].ev_pub)) != cudaSuccess ||
        (e = cudaIpcOpenEventHandle(&pl->ev_done[r], pl->shm->slot[r].ev_done)) != cudaSuccess) {
      peer_close(pl);
      return failf(err, DMHA_ERR_CUDA, "cudaIpcOpenEventHandle", e);
    }
  }
  if (int rc = peer_barrier(pl, err)) {
    peer_close(pl);
    return rc;
  }
  *out = pl;
  return DMHA_OK;
}

int peer_ensure_pub(PeerLink* pl, size_t bytes, std::string* err) {
  if (bytes <= pl->pub_bytes) return DMHA_OK;
  // every rank grows at the same call (collective contract): drop the old
  // mappings, wait until nobody reads the old buffers, re-publish
  close_peer_maps(pl);
  if (int rc = peer_barrier(pl, err)) return rc;
  if (pl->pub) cudaFree(pl->pub);
  pl->pub = nullptr;
  pl->pub_bytes = 0;
  cudaError_t e = cudaMalloc(&pl->pub, bytes);
  if (e != cudaSuccess) {
    pl->pub = nullptr;
    return failf(err, DMHA_ERR_OOM, "published K/V buffer", e);
  }
  pl->pub_bytes = bytes;
  Slot& me = pl->shm->slot[pl->rank];
  if ((e = cudaIpcGetMemHandle(&me.mem, pl->pub)) != cudaSuccess)
    return failf(err, DMHA_ERR_CUDA, "cudaIpcGetMemHandle", e);
  me.pub_bytes = bytes;
  me.mem_version = ++pl->version;
  if (int rc = peer_barrier(pl, err)) return rc;
  for (int r = 0; r < pl->world; ++r) {
    if (r == pl->rank) continue;
    if (pl->shm->slot[r].pub_bytes < bytes)
      return failf(err, DMHA_ERR_STATE, "ranks disagree on the published buffer size");
    if ((e = cudaIpcOpenMemHandle(&pl->peer_pub[r], pl->shm->slot[r].mem,
                                  cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess)
      return failf(err, DMHA_ERR_CUDA, "cudaIpcOpenMemHandle", e);
  }
  return peer_barrier(pl, err);
}

void peer_close(PeerLink* pl) {
  if (!pl) return;
  if (pl->shm) {
    close_peer_maps(pl);
    std::string ignore;
    peer_barrier(pl, &ignore, 60.0);
  }
  for (int r = 0; r < pl->world && r < static_cast<int>(pl->ev_pub.size()); ++r) {
    if (pl->ev_pub[r]) cudaEventDestroy(pl->ev_pub[r]);
    if (pl->ev_done[r]) cudaEventDestroy(pl->ev_done[r]);
  }
  if (pl->pub) cudaFree(pl->pub);
  if (pl->shm) {
    munmap(pl->shm, sizeof(Shm));
    if (pl->rank == 0) shm_unlink(pl->name.c_str());
  }
  delete pl;
}

void* peer_local_pub(PeerLink* pl) { return pl->pub; }
void* peer_pub(PeerLink* pl, int r) { return r == pl->rank ? pl->pub : pl->peer_pub[r]; }
cudaEvent_t peer_pub_event(PeerLink* pl, int r) { return pl->ev_pub[r]; }
cudaEvent_t peer_done_event(PeerLink* pl, int r) { return pl->ev_done[r]; }
size_t peer_pub_bytes(PeerLink* pl) { return pl->pub_bytes; }

}  // namespace dmha
