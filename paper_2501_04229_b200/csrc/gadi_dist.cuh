// gadi_dist.cuh — the collectives of a sharded (z-slab) solve, SURVEY §8(e).
//
// A sharded solve splits the stencil grid into `world` z-slabs of the slowest
// index (row = i*n^2 + j*n + k, problems.cpp:14): rank r owns planes
// [r*n/world, (r+1)*n/world), a contiguous, aligned power-of-two block of
// every pairwise-sum tree. Each device holds its slab plus one ghost plane on
// each side of every vector an operator pass reads. Two collectives are used:
//
//  * allgather of the 4-word reduction record (gadi_kernels.cuh finish_red):
//    every rank gets every rank's subtree sums and flag / max words, and
//    k_dist_finish folds them in rank order -- bit for bit the single-device
//    value -- and applies the reduction's epilogue identically on all ranks,
//    so every rank takes the same control-flow decisions;
//  * halo: a vector's first / last owned entries (one plane of a z-slab,
//    the band of a CSR row block) into the neighbours' ghost entries before
//    an operator pass reads them.
//
// Two transports implement them: LocalComm (ranks are threads of one
// process, on one or several devices: device copies ordered by CUDA events,
// a host barrier per collective -- no kernel ever waits on another rank, so
// several ranks may share one GPU) and NcclComm (one rank per process;
// ncclAllGather and grouped ncclSend/ncclRecv, libnccl loaded at run time).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace gadi_host {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // dst[4*r + k] = rank r's src[k], k < 4 (device pointers, stream ordered)
  virtual void allgather4(const double* src, double* dst, cudaStream_t s) = 0;
  // ghost entries of a shard vector (len bytes of owned entries, `ghost`
  // bytes of ghosts on each side, ghost <= len): interior - ghost <- rank-1's
  // last ghost bytes, interior + len <- rank+1's first ghost bytes. Stencil
  // slabs exchange one plane; CSR row blocks the band of x entries.
  virtual void halo(char* interior, int64_t ghost, int64_t len, cudaStream_t s) = 0;
};

// ------------------------------------------------------------ local group
// Ranks are threads of this process. Each collective publishes (pointer,
// event) per rank, meets at a host barrier, then pulls from the peers on the
// caller's stream after waiting on their events. A rank rewrites a published
// buffer only after a later collective in which it waited on every peer's
// event recorded after that peer's pull, so the pulls never race the writes
// (the reduction record is double-buffered by the caller for the same reason).
struct LocalGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;
  struct Slot {
    const void* p = nullptr;
    cudaEvent_t ev = nullptr;
  };
  std::vector<Slot> slots;
  explicit LocalGroup(int w) : world(w), slots(w) {}

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw std::runtime_error("sharded solve aborted by another rank");
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      if (aborted && gen == g) throw std::runtime_error("sharded solve aborted by another rank");
    }
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct LocalComm final : Comm {
  LocalGroup* g;
  cudaEvent_t ev = nullptr;
  LocalComm(LocalGroup* grp, int r) : g(grp) {
    rank = r;
    world = grp->world;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
      throw std::runtime_error("cudaEventCreate failed");
  }
  ~LocalComm() override {
    if (ev) cudaEventDestroy(ev);
  }
  void publish(const void* p, cudaStream_t s) {
    if (cudaEventRecord(ev, s) != cudaSuccess) throw std::runtime_error("cudaEventRecord failed");
    g->slots[rank] = {p, ev};
    g->barrier();
  }
  void allgather4(const double* src, double* dst, cudaStream_t s) override {
    publish(src, s);
    for (int r = 0; r < world; ++r) {
      const LocalGroup::Slot sl = g->slots[r];
      if (r != rank) cudaStreamWaitEvent(s, sl.ev, 0);
      cudaMemcpyAsync(dst + 4 * r, sl.p, 4 * sizeof(double), cudaMemcpyDefault, s);
    }
    g->barrier();  // every rank has read the slots before they are republished
  }
  void halo(char* interior, int64_t ghost, int64_t len, cudaStream_t s) override {
    publish(interior, s);
    if (rank > 0) {
      const LocalGroup::Slot sl = g->slots[rank - 1];
      cudaStreamWaitEvent(s, sl.ev, 0);
      cudaMemcpyAsync(interior - ghost, static_cast<const char*>(sl.p) + len - ghost, ghost, cudaMemcpyDefault, s);
    }
    if (rank + 1 < world) {
      const LocalGroup::Slot sl = g->slots[rank + 1];
      cudaStreamWaitEvent(s, sl.ev, 0);
      cudaMemcpyAsync(interior + len, sl.p, ghost, cudaMemcpyDefault, s);
    }
    g->barrier();
  }
};

// ------------------------------------------------------------ NCCL
// The few NCCL entry points used, resolved from libnccl.so.2 at run time (the
// library does not link NCCL; torch's process already has one loaded).
struct NcclApi {
  typedef int (*GetUniqueId)(void*);
  typedef int (*CommInitRank)(void**, int, const char* /* by value: 128 bytes */, int);
  typedef int (*CommDestroy)(void*);
  typedef int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t);
  typedef int (*SendRecv)(const void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*Group)();
  typedef const char* (*ErrStr)(int);
  void* lib = nullptr;
  GetUniqueId get_unique_id = nullptr;
  void* comm_init_rank = nullptr;
  CommDestroy comm_destroy = nullptr;
  AllGather all_gather = nullptr;
  SendRecv send = nullptr, recv = nullptr;
  Group group_start = nullptr, group_end = nullptr;
  ErrStr err = nullptr;

  static NcclApi& get() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
      for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
        a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (a.lib) break;
      }
      if (!a.lib) return;
      a.get_unique_id = (GetUniqueId)dlsym(a.lib, "ncclGetUniqueId");
      a.comm_init_rank = dlsym(a.lib, "ncclCommInitRank");
      a.comm_destroy = (CommDestroy)dlsym(a.lib, "ncclCommDestroy");
      a.all_gather = (AllGather)dlsym(a.lib, "ncclAllGather");
      a.send = (SendRecv)dlsym(a.lib, "ncclSend");
      a.recv = (SendRecv)dlsym(a.lib, "ncclRecv");
      a.group_start = (Group)dlsym(a.lib, "ncclGroupStart");
      a.group_end = (Group)dlsym(a.lib, "ncclGroupEnd");
      a.err = (ErrStr)dlsym(a.lib, "ncclGetErrorString");
    });
    if (!a.lib || !a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.send || !a.recv)
      throw std::runtime_error("libnccl.so.2 not loadable");
    return a;
  }
};

struct NcclId {
  char b[128];
};
typedef int (*NcclInitFn)(void**, int, NcclId, int);  // ncclCommInitRank(comm*, nranks, id by value, rank)

struct NcclComm final : Comm {
  void* comm = nullptr;
  static constexpr int kDouble = 8, kChar = 0;  // ncclDouble, ncclInt8
  NcclComm(int w, int r, const NcclId& id) {
    rank = r;
    world = w;
    NcclApi& a = NcclApi::get();
    const int rc = reinterpret_cast<NcclInitFn>(a.comm_init_rank)(&comm, w, id, r);
    if (rc != 0) throw std::runtime_error(std::string("ncclCommInitRank: ") + (a.err ? a.err(rc) : "error"));
  }
  ~NcclComm() override {
    if (comm) NcclApi::get().comm_destroy(comm);
  }
  void check(int rc, const char* what) {
    if (rc != 0) {
      NcclApi& a = NcclApi::get();
      throw std::runtime_error(std::string(what) + ": " + (a.err ? a.err(rc) : "error"));
    }
  }
  void allgather4(const double* src, double* dst, cudaStream_t s) override {
    check(NcclApi::get().all_gather(src, dst, 4, kDouble, comm, s), "ncclAllGather");
  }
  void halo(char* interior, int64_t ghost, int64_t len, cudaStream_t s) override {
    NcclApi& a = NcclApi::get();
    check(a.group_start(), "ncclGroupStart");
    if (rank > 0) {
      check(a.send(interior, (size_t)ghost, kChar, rank - 1, comm, s), "ncclSend");
      check(a.recv(interior - ghost, (size_t)ghost, kChar, rank - 1, comm, s), "ncclRecv");
    }
    if (rank + 1 < world) {
      check(a.send(interior + len - ghost, (size_t)ghost, kChar, rank + 1, comm, s), "ncclSend");
      check(a.recv(interior + len, (size_t)ghost, kChar, rank + 1, comm, s), "ncclRecv");
    }
    check(a.group_end(), "ncclGroupEnd");
  }
};

}  // namespace gadi_host

// The opaque group handle of the C ABI: a local (threads) group, or one
// process's NCCL membership.
struct gadi_group {
  int world = 1;
  int nccl_rank = -1;  // >= 0: NCCL (one rank per process)
  std::unique_ptr<gadi_host::LocalGroup> local;
  gadi_host::NcclId id{};
};
