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
// Three transports implement them: LocalComm (ranks are threads of one
// process, on one or several devices: device copies ordered by CUDA events,
// a host barrier per collective -- no kernel ever waits on another rank, so
// several ranks may share one GPU), IpcComm (one rank per process on one node:
// the same protocol across processes -- CUDA IPC memory and interprocess
// events, a barrier in POSIX shared memory, peer loads over NVLink / NVSwitch;
// again no kernel waits on another rank) and NcclComm (one rank per process;
// ncclAllGather and grouped ncclSend/ncclRecv, libnccl loaded at run time).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
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


// ------------------------------------------------------------ CUDA IPC
// One rank per process, all on one node (the torchrun launch of bench.py
// --gpus N). Each rank owns a staging buffer (cudaMalloc, exported with
// cudaIpcGetMemHandle and mapped by every peer) holding, per collective
// parity p, its 4-word reduction record and its first / last `ghost` bytes,
// and two interprocess events per parity: ready[p] (my staging[p] is written)
// and pulled[p] (my reads of the peers' staging[p] are done). A collective:
//   1. wait (stream) on every peer's pulled[p] of two collectives ago, write
//      my staging[p], record ready[p];
//   2. host barrier in shared memory (every rank has RECORDED ready[p]: a
//      cudaStreamWaitEvent captures the event's latest record at call time);
//   3. wait (stream) on the peers' ready[p], read their staging[p] through the
//      mapped pointers (a halo pulls two chunks with device copies, a record
//      all-gather reads every peer in ONE kernel: the one-shot exchange over
//      NVLink / NVSwitch peer loads), record pulled[p].
// The wait in step 1 of collective c + 2 follows the barrier of collective
// c + 1, which every rank passes only after recording pulled[p] in c, so it
// sees that record. No kernel ever spins on another rank's progress: ranks
// may share a GPU (the 2- and 4-process tests do).
struct IpcShared {
  std::atomic<uint32_t> bar_count, bar_gen, attached;
  uint32_t world;
  struct Slot {
    cudaIpcMemHandle_t mem;
    cudaIpcEventHandle_t ev[4];  // ready[0], ready[1], pulled[0], pulled[1]
    uint64_t stage_bytes;
  } slot[64];
};

struct IpcGroup {
  std::string name;
  int world = 1, rank = 0;
  IpcShared* sh = nullptr;
  IpcGroup(int w, int r, const std::string& nm) : name(nm), world(w), rank(r) {
    int fd = -1;
    if (r == 0) {
      shm_unlink(name.c_str());
      fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0 || ftruncate(fd, sizeof(IpcShared)) != 0) throw std::runtime_error("ipc group: shm_open failed: " + name);
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      while ((fd = shm_open(name.c_str(), O_RDWR, 0600)) < 0) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          throw std::runtime_error("ipc group: rank 0 never created " + name);
        usleep(1000);
      }
      // wait until rank 0 sized the segment
      for (;;) {
        const off_t sz = lseek(fd, 0, SEEK_END);
        if (sz >= (off_t)sizeof(IpcShared)) break;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          throw std::runtime_error("ipc group: segment never sized: " + name);
        usleep(1000);
      }
    }
    void* p = mmap(nullptr, sizeof(IpcShared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) throw std::runtime_error("ipc group: mmap failed");
    sh = static_cast<IpcShared*>(p);
    if (r == 0) sh->world = (uint32_t)w;  // the fresh segment is zero-filled: counters start at 0
    sh->attached.fetch_add(1, std::memory_order_acq_rel);
    const auto t0 = std::chrono::steady_clock::now();
    while (sh->attached.load(std::memory_order_acquire) < (uint32_t)w) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
        throw std::runtime_error("ipc group: not every rank attached");
      sched_yield();
    }
  }
  ~IpcGroup() {
    if (sh) munmap(sh, sizeof(IpcShared));
    if (rank == 0) shm_unlink(name.c_str());
  }
  void barrier() {
    const uint32_t gen = sh->bar_gen.load(std::memory_order_acquire);
    if (sh->bar_count.fetch_add(1, std::memory_order_acq_rel) + 1 == (uint32_t)world) {
      sh->bar_count.store(0, std::memory_order_relaxed);
      sh->bar_gen.fetch_add(1, std::memory_order_release);
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spins = 0; sh->bar_gen.load(std::memory_order_acquire) == gen; ++spins) {
      if ((spins & 1023u) == 1023u) {
        sched_yield();
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300))
          throw std::runtime_error("ipc group: a rank did not reach the barrier (300 s)");
      }
    }
  }
};

struct IpcPeers {
  const double* rec[64];
};
// dst[4 r + k] = rank r's record: one launch reads every peer (mapped pointers)
static __global__ void k_ipc_gather(IpcPeers pp, int world, double* __restrict__ dst) {
  const int t = threadIdx.x;
  if (t < 4 * world) dst[t] = pp.rec[t >> 2][t & 3];
}

struct IpcComm final : Comm {
  IpcGroup* g;
  size_t ghost_max = 0, par_bytes = 0;
  char* stage = nullptr;                 // [2 parities][256 B record | ghost_max | ghost_max]
  cudaEvent_t ev[4] = {};                // ready[0], ready[1], pulled[0], pulled[1]
  std::vector<char*> peer_stage;
  std::vector<cudaEvent_t> peer_ev;      // [rank][4]
  uint64_t seq = 0;
  static void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
  IpcComm(IpcGroup* grp, size_t ghost_bytes_max) : g(grp) {
    rank = grp->rank;
    world = grp->world;
    ghost_max = (ghost_bytes_max + 255) & ~size_t(255);
    par_bytes = 256 + 2 * ghost_max;
    ck(cudaMalloc((void**)&stage, 2 * par_bytes), "ipc: cudaMalloc");
    ck(cudaMemset(stage, 0, 2 * par_bytes), "ipc: cudaMemset");
    IpcShared::Slot& me = g->sh->slot[rank];
    ck(cudaIpcGetMemHandle(&me.mem, stage), "cudaIpcGetMemHandle");
    for (int k = 0; k < 4; ++k) {
      ck(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming | cudaEventInterprocess), "ipc: cudaEventCreate");
      ck(cudaIpcGetEventHandle(&me.ev[k], ev[k]), "cudaIpcGetEventHandle");
    }
    me.stage_bytes = 2 * par_bytes;
    ck(cudaDeviceSynchronize(), "ipc: sync");
    g->barrier();  // every slot is published
    peer_stage.assign(world, nullptr);
    peer_ev.assign((size_t)world * 4, nullptr);
    for (int r = 0; r < world; ++r) {
      if (r == rank) {
        peer_stage[r] = stage;
        for (int k = 0; k < 4; ++k) peer_ev[(size_t)r * 4 + k] = ev[k];
        continue;
      }
      const IpcShared::Slot& sl = g->sh->slot[r];
      if (sl.stage_bytes != 2 * par_bytes) throw std::runtime_error("ipc: ranks disagree on the ghost size");
      void* p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, sl.mem, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      peer_stage[r] = static_cast<char*>(p);
      for (int k = 0; k < 4; ++k) ck(cudaIpcOpenEventHandle(&peer_ev[(size_t)r * 4 + k], sl.ev[k]), "cudaIpcOpenEventHandle");
    }
    g->barrier();  // every rank has opened every slot before a slot is reused by the next IpcComm
  }
  ~IpcComm() override {
    cudaDeviceSynchronize();
    try {
      g->barrier();  // no peer still reads my staging buffer
    } catch (...) {
    }
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      if (peer_stage[r]) cudaIpcCloseMemHandle(peer_stage[r]);
      for (int k = 0; k < 4; ++k)
        if (peer_ev[(size_t)r * 4 + k]) cudaEventDestroy(peer_ev[(size_t)r * 4 + k]);
    }
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (stage) cudaFree(stage);
  }
  char* rec_of(int r, int p) const { return peer_stage[r] + (size_t)p * par_bytes; }
  char* lo_of(int r, int p) const { return rec_of(r, p) + 256; }
  char* hi_of(int r, int p) const { return lo_of(r, p) + ghost_max; }
  int begin(cudaStream_t s) {  // step 1's waits; returns the parity
    const int p = (int)(seq++ & 1);
    for (int r = 0; r < world; ++r)
      if (r != rank) ck(cudaStreamWaitEvent(s, peer_ev[(size_t)r * 4 + 2 + p], 0), "ipc: wait pulled");
    return p;
  }
  void allgather4(const double* src, double* dst, cudaStream_t s) override {
    const int p = begin(s);
    ck(cudaMemcpyAsync(rec_of(rank, p), src, 4 * sizeof(double), cudaMemcpyDeviceToDevice, s), "ipc: record copy");
    ck(cudaEventRecord(ev[p], s), "ipc: record ready");
    g->barrier();
    IpcPeers pp;
    for (int r = 0; r < world; ++r) {
      if (r != rank) ck(cudaStreamWaitEvent(s, peer_ev[(size_t)r * 4 + p], 0), "ipc: wait ready");
      pp.rec[r] = reinterpret_cast<const double*>(rec_of(r, p));
    }
    k_ipc_gather<<<1, 256, 0, s>>>(pp, world, dst);
    ck(cudaGetLastError(), "k_ipc_gather");
    ck(cudaEventRecord(ev[2 + p], s), "ipc: record pulled");
  }
  void halo(char* interior, int64_t ghost, int64_t len, cudaStream_t s) override {
    if ((size_t)ghost > ghost_max) throw std::runtime_error("ipc: ghost larger than the staging buffer");
    const int p = begin(s);
    if (rank > 0) ck(cudaMemcpyAsync(lo_of(rank, p), interior, ghost, cudaMemcpyDeviceToDevice, s), "ipc: stage lo");
    if (rank + 1 < world)
      ck(cudaMemcpyAsync(hi_of(rank, p), interior + len - ghost, ghost, cudaMemcpyDeviceToDevice, s), "ipc: stage hi");
    ck(cudaEventRecord(ev[p], s), "ipc: record ready");
    g->barrier();
    if (rank > 0) {
      ck(cudaStreamWaitEvent(s, peer_ev[(size_t)(rank - 1) * 4 + p], 0), "ipc: wait ready");
      ck(cudaMemcpyAsync(interior - ghost, hi_of(rank - 1, p), ghost, cudaMemcpyDefault, s), "ipc: pull lower");
    }
    if (rank + 1 < world) {
      ck(cudaStreamWaitEvent(s, peer_ev[(size_t)(rank + 1) * 4 + p], 0), "ipc: wait ready");
      ck(cudaMemcpyAsync(interior + len, lo_of(rank + 1, p), ghost, cudaMemcpyDefault, s), "ipc: pull upper");
    }
    ck(cudaEventRecord(ev[2 + p], s), "ipc: record pulled");
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
  int nccl_rank = -1;  // >= 0: one rank per process (NCCL, or CUDA IPC when `ipc` is set)
  std::unique_ptr<gadi_host::LocalGroup> local;
  std::unique_ptr<gadi_host::IpcGroup> ipc;
  gadi_host::NcclId id{};
};
