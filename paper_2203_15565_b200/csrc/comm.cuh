// comm.cuh — the step's collectives behind one interface: NCCL between the GPUs
// of a box (one process per GPU), or a loopback communicator that runs R ranks as R contexts
// of ONE process (R host threads, any devices, typically all on one GPU).
//
// The loopback exists so that the library's own rank code (rank-local shards, foreign
// positives, the stats exchange, per-row offset max, dX reduce-scatter / all-reduce) executes
// and is checked where only one GPU is available.  It is host-synchronised: at each collective
// the R threads rendezvous (condition-variable barrier) to publish their buffers and CUDA
// events; every device-side dependency is a cudaStreamWaitEvent on a peer's event, so no kernel
// ever waits on another rank's kernel.  Reductions run in ascending rank order (deterministic),
// in-place operations go through a per-rank scratch buffer that is copied back only after every
// peer finished reading.  Not capturable into a CUDA graph (contexts using it run eagerly).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace pfc {

// ------------------------------------------------------------------ NCCL (dlopen'ed lazily)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { ncclInt8 = 0, ncclInt32 = 2, ncclInt64 = 4, ncclUint64 = 5, ncclFloat32 = 7, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };
struct Nccl {
  void* h = nullptr;
  int (*GetUniqueId)(ncclUniqueId*) = nullptr;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*ReduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool load(std::string& err) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* hh = nullptr;
    for (const char* n : names)
      if ((hh = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!hh) {
      err = "NCCL not found (dlopen libnccl.so.2 failed)";
      return false;
    }
    GetUniqueId = (decltype(GetUniqueId))dlsym(hh, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(hh, "ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))dlsym(hh, "ncclCommDestroy");
    AllGather = (decltype(AllGather))dlsym(hh, "ncclAllGather");
    AllReduce = (decltype(AllReduce))dlsym(hh, "ncclAllReduce");
    ReduceScatter = (decltype(ReduceScatter))dlsym(hh, "ncclReduceScatter");
    GetErrorString = (decltype(GetErrorString))dlsym(hh, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !AllGather || !AllReduce || !ReduceScatter) {
      err = "NCCL symbols missing";
      return false;
    }
    h = hh;
    return true;
  }
};
inline Nccl g_nccl;

enum CommDt { kI32 = 0, kI64 = 1, kU64 = 2, kF32 = 3, kF64 = 4 };
enum CommOp { kSum = 0, kMax = 1 };
inline size_t dt_size(CommDt t) { return t == kI32 || t == kF32 ? 4 : 8; }
inline int nccl_dt(CommDt t) {
  switch (t) {
    case kI32: return ncclInt32;
    case kI64: return ncclInt64;
    case kU64: return ncclUint64;
    case kF32: return ncclFloat32;
    default: return ncclFloat64;
  }
}
inline int nccl_op(CommOp o) { return o == kSum ? ncclSum : ncclMax; }

// ------------------------------------------------------------------ loopback
constexpr int kLoopMaxRanks = 16;
constexpr char kLoopMagic[8] = {'P', 'F', 'C', 'L', 'O', 'O', 'P', 0};

struct LoopPtrs {
  const void* p[kLoopMaxRanks];
};

// out[i] = op over ranks 0..R-1 (ascending) of src_r[off + i]
template <typename T>
__global__ void loop_reduce_kernel(LoopPtrs src, int R, size_t off, size_t n, int op,
                                   T* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    T a = static_cast<const T*>(src.p[0])[off + i];
    for (int r = 1; r < R; ++r) {
      const T v = static_cast<const T*>(src.p[r])[off + i];
      a = op == kSum ? a + v : (a < v ? v : a);
    }
    out[i] = a;
  }
}

struct LoopGroup {
  int R = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  int alive = 0;
  struct Slot {
    const void* send = nullptr;
    void* recv = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    int device = 0;
  };
  std::vector<Slot> slot;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == R) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LoopRegistry {
  std::mutex mu;
  std::map<std::string, std::shared_ptr<LoopGroup>> groups;
  uint64_t next = 1;
};
inline LoopRegistry g_loop;

inline bool is_loop_id(const uint8_t* id) { return id && std::memcmp(id, kLoopMagic, 8) == 0; }

inline void loop_new_id(uint8_t out[128]) {
  std::lock_guard<std::mutex> lk(g_loop.mu);
  std::memset(out, 0, 128);
  std::memcpy(out, kLoopMagic, 8);
  const uint64_t n = g_loop.next++;
  std::memcpy(out + 8, &n, 8);
}

// join (or create) the group named by id as `rank` of R; scratch_bytes per rank
inline std::shared_ptr<LoopGroup> loop_join(const uint8_t* id, int R, int rank, int device,
                                            size_t scratch_bytes, std::string& err) {
  std::shared_ptr<LoopGroup> g;
  {
    std::lock_guard<std::mutex> lk(g_loop.mu);
    const std::string key(reinterpret_cast<const char*>(id), 128);
    auto it = g_loop.groups.find(key);
    if (it == g_loop.groups.end()) {
      g = std::make_shared<LoopGroup>();
      g->R = R;
      g->slot.resize((size_t)R);
      g_loop.groups[key] = g;
    } else {
      g = it->second;
    }
    if (g->R != R || R > kLoopMaxRanks) {
      err = "loopback group: world_size mismatch or more than 16 ranks";
      return nullptr;
    }
    g->alive++;
  }
  LoopGroup::Slot& s = g->slot[(size_t)rank];
  s.device = device;
  if (cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&s.scratch, scratch_bytes) != cudaSuccess) {
    err = "loopback group: CUDA allocation failed";
    return nullptr;
  }
  s.scratch_bytes = scratch_bytes;
  g->barrier();  // every rank joined (its events exist) before any collective
  // ranks on other devices read this one's buffers in the reduce kernels
  for (int r = 0; r < R; ++r)
    if (g->slot[(size_t)r].device != device) {
      cudaDeviceEnablePeerAccess(g->slot[(size_t)r].device, 0);
      cudaGetLastError();
    }
  return g;
}

inline void loop_leave(const std::shared_ptr<LoopGroup>& g, const uint8_t* id, int rank) {
  if (!g) return;
  LoopGroup::Slot& s = g->slot[(size_t)rank];
  if (s.ready) cudaEventDestroy(s.ready);
  if (s.done) cudaEventDestroy(s.done);
  if (s.scratch) cudaFree(s.scratch);
  s = LoopGroup::Slot{};
  std::lock_guard<std::mutex> lk(g_loop.mu);
  if (--g->alive == 0) g_loop.groups.erase(std::string(reinterpret_cast<const char*>(id), 128));
}

template <typename T>
cudaError_t loop_reduce_launch(const LoopPtrs& src, int R, size_t off, size_t n, CommOp op, void* out,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<size_t>((n + 255) / 256, 1184);
  loop_reduce_kernel<T><<<grid, 256, 0, s>>>(src, R, off, n, (int)op, static_cast<T*>(out));
  return cudaGetLastError();
}

inline cudaError_t loop_reduce(CommDt dt, const LoopPtrs& src, int R, size_t off, size_t n, CommOp op,
                               void* out, cudaStream_t s) {
  switch (dt) {
    case kI32: return loop_reduce_launch<int32_t>(src, R, off, n, op, out, s);
    case kI64: return loop_reduce_launch<long long>(src, R, off, n, op, out, s);
    case kU64: return loop_reduce_launch<unsigned long long>(src, R, off, n, op, out, s);
    case kF32: return loop_reduce_launch<float>(src, R, off, n, op, out, s);
    default: return loop_reduce_launch<double>(src, R, off, n, op, out, s);
  }
}

// kind 0: all-gather (count per rank), 1: all-reduce (count), 2: reduce-scatter (count per rank)
inline cudaError_t loop_collective(LoopGroup& g, int rank, int kind, const void* send, void* recv,
                                   size_t count, CommDt dt, CommOp op, cudaStream_t s) {
  const int R = g.R;
  const size_t es = dt_size(dt), bytes = count * es;
  LoopGroup::Slot& me = g.slot[(size_t)rank];
  cudaError_t e = cudaSuccess;
  auto keep = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  if (kind != 0 && bytes > me.scratch_bytes) return cudaErrorMemoryAllocation;
  me.send = send;
  me.recv = recv;
  keep(cudaEventRecord(me.ready, s));
  g.barrier();  // 1: buffers published, ready events recorded
  for (int p = 0; p < R; ++p) keep(cudaStreamWaitEvent(s, g.slot[(size_t)p].ready, 0));
  LoopPtrs src{};
  for (int p = 0; p < R; ++p) src.p[p] = g.slot[(size_t)p].send;
  if (kind == 0) {
    for (int p = 0; p < R; ++p) {
      char* dst = static_cast<char*>(recv) + (size_t)p * bytes;
      if (dst != g.slot[(size_t)p].send && bytes)
        keep(cudaMemcpyAsync(dst, g.slot[(size_t)p].send, bytes, cudaMemcpyDeviceToDevice, s));
    }
  } else {
    const size_t off = kind == 2 ? (size_t)rank * count : 0;
    keep(loop_reduce(dt, src, R, off, count, op, me.scratch, s));
  }
  keep(cudaEventRecord(me.done, s));
  g.barrier();  // 2: every rank enqueued its reads of the peers' buffers
  for (int p = 0; p < R; ++p) keep(cudaStreamWaitEvent(s, g.slot[(size_t)p].done, 0));
  if (kind != 0 && bytes) keep(cudaMemcpyAsync(recv, me.scratch, bytes, cudaMemcpyDeviceToDevice, s));
  g.barrier();  // 3: nobody re-records ready / done before every rank has waited on them
  return e;
}

}  // namespace pfc
