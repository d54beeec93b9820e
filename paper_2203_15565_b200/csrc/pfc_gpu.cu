// pfc_gpu.cu — host orchestration of the B200-native Partial-FC step and the C ABI of
// include/pfc_gpu.h.  One context = one rank = one GPU; it owns the fp32 row-major W and
// momentum of its reference shards and runs
//
//   [NCCL all-gather labels, X]  (world > 1)
//   sampler (bit-exact build_buffers)                 sampler.cu
//   normalise X, gather+normalise sampled W rows      kernels.cuh
//   logits GEMM + margin -> E = exp(z - o) + row sums  tcgen05 GEMM, FwdEpi
//   row sums [NCCL all-gather, all-reduce z_pos] -> loss, rowscale, positive correction
//   dX = rowscale E W^ (split-K) + corrections [NCCL reduce-scatter]  tcgen05 GEMM, DxPartEpi
//   dW = E^T (rowscale X^) -> center_proj (2-CTA DSMEM) -> fused sparse momentum-SGD
//                                                      tcgen05 GEMM, DwUpdateEpi
//
// mirroring pfc::distributed_partial_step (proj/include/pfc/shardsim.hpp:166-420).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pfc_gpu.h"
#include "common.cuh"
#include "comm.cuh"
#include "epilogues.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "diag.cuh"
#include "sampler.cu"

namespace pfc {
namespace {

thread_local std::string g_create_error;

// cudaFuncAttributeMaxDynamicSharedMemorySize is per (device, kernel): a process may hold
// contexts on several devices (and create them from several threads), so the attribute is
// set once per pair under a lock rather than once per process.
cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, fn})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({dev, fn});
  return e;
}


// ------------------------------------------------------------------ TMA descriptor encode
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled_t get_encode() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

// 2-D bf16 tensor [outer][inner] with row stride ld (elements); box {box_inner, box_outer}.
// Loads use {64, rows} with 128B swizzle (UMMA operand atoms); the G^T store uses {32, 128}
// with 64B swizzle (matching the epilogue's smem staging).
// elem: 2 (bf16) or 4 (fp32 operands of the tf32 engine; box_inner then 32 for 128 B rows).
bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_outer, uint32_t box_inner = 64,
              CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B, int elem = 2) {
  PFN_encodeTiled_t enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * (uint64_t)elem};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapDataType dt =
      elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  return enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

constexpr int kBN = 256;  // tcgen05 tile 128 x 256
#ifndef PFC_FWD_BN
#define PFC_FWD_BN 256
#endif
#ifndef PFC_FWD_NWG
#define PFC_FWD_NWG 2
#endif
constexpr int kFwdBN = PFC_FWD_BN;    // logits GEMM tile width (classes)
constexpr int kNarrowBN = 128;        // ... when kFwdBN-wide tiles would fill at most half the SMs
constexpr int kFwdNWG = PFC_FWD_NWG;  // logits GEMM epilogue warpgroups (kFwdBN / 64 / kFwdNWG chunks)
#ifndef PFC_FWD_CG
#define PFC_FWD_CG 1
#endif
#ifndef PFC_DX_CG
#define PFC_DX_CG 1
#endif
#ifndef PFC_FWD_STAGES
#define PFC_FWD_STAGES 4
#endif
constexpr int kFwdStages = PFC_FWD_STAGES;  // logits GEMM operand ring depth
constexpr int kFwdCG = PFC_FWD_CG;  // logits GEMM: 1 = one CTA per 128-row tile, 2 = CTA pair
constexpr int kDxCG = PFC_DX_CG;    // dX GEMM likewise
#ifndef PFC_DIAG_CG
#define PFC_DIAG_CG 1
#endif
constexpr int kDiagCG = PFC_DIAG_CG;  // diagnostics / mics screening GEMMs likewise
constexpr int64_t kDwDeepBatch = 1024;  // dW GEMM: 3 operand stages + 3 KB ring above 2 KB of E^T per row
#ifndef PFC_DW_STAGES
#define PFC_DW_STAGES 2
#endif  // dW GEMM operand ring depth (2: leaves shared memory to the W / momentum ring)
constexpr int kSimtBN = 64;

struct PhaseTimer {
  bool enabled = false;
  static constexpr int kMax = 16;
  cudaEvent_t ev[kMax + 1] = {};
  const char* names[kMax] = {};
  int n = 0;
  float ms[kMax] = {};
};

struct Ctx {
  pfc_gpu_desc d{};
  std::string err;
  int64_t C, D, K, Dp, blk, cap, k0, nk, cls_lo, cls_hi, rows, ncols, ncols_pad, ldg;
  int64_t pool_stride, maxB;
  int R, rank;
  bool coll = false;  // R > 1, or PFC_FLAG_FORCE_COLLECTIVES: the collectives run (1-rank group)
  bool bf16;          // tcgen05 kind::f16 engine (bf16 operands)
  bool tf32 = false;  // tcgen05 kind::tf32 engine (fp32 operands)
  bool umma = false;  // either tcgen05 engine (else the fp32 SIMT validation engine)
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t s2 = nullptr;                      // forked stream inside the step
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  MarginDev mg{};
  // state
  float* W = nullptr;
  float* M = nullptr;
  // sampler
  int64_t* labels = nullptr;  // global batch labels (world > 1 / host path)
  int64_t* labs = nullptr;    // the step's labels as the sampler copied them (device)
  uint32_t* bits = nullptr;   // [nwords] label bitmap over all C classes (all-zero between steps)
  int32_t* ccnt = nullptr;    // [nchunk] set bits per chunk of chunk_words words (zero between steps)
  int32_t* rej = nullptr;     // [nk] a draw of the shard saw a modulo rejection
  long long* oobs = nullptr;  // [2] smallest negative / >= C label of the step (LLONG_MAX: none)
  int64_t nwords = 0;
  int chunk_words = 32, nchunk = 1;
  ShardMeta* meta = nullptr;
  int32_t* buf_cls = nullptr;
  int32_t* pos_col = nullptr;
  int32_t* head = nullptr;
  int32_t* nxt = nullptr;
  int32_t* jv = nullptr;
  int32_t* pool_scratch = nullptr;
  // features / centres
  float* X = nullptr;  // global batch rows [B][D] fp32 (world > 1 / host path)
  uint64_t step_nccl_bytes = 0;  // bytes handed to NCCL by the last step (pfc_gpu_step_out)
  uint64_t step_wire_bytes = 0;  // the same collectives under the ring model (all ranks)
  // diagnostics (pfc_gpu_diagnostics), allocated on first use
  void* dwall = nullptr;  // w^ of every local class, operand dtype [rows_pad][Dp]
  double *dwinv = nullptr, *dxinv = nullptr, *dapcs = nullptr;
  uint32_t* drmax = nullptr;
  unsigned long long* demax = nullptr;
  int* dhasc = nullptr;
  int64_t *dcid = nullptr, *dsid = nullptr;
  int64_t diag_rows_pad = 0;
  DiagCand* dcand = nullptr;
  unsigned long long* dncand = nullptr;
  int64_t dcand_cap = 0;
  CUtensorMap tm_wall;
  float* xnorm = nullptr;
  void* xh = nullptr;  // [maxB][Dp] bf16 or fp32
  void* wh = nullptr;  // [ncols_pad][Dp]
  float* wnorm = nullptr;
  int32_t* lrow = nullptr;
  // softmax statistics (fixed-offset form, see epilogues.cuh)
  void* part_s = nullptr;  // [T * NWG][maxB] sums of E per column slice
  void* ls = nullptr;      // [R][maxB] rank-local sums
  void* rowscale = nullptr;
  void* delta = nullptr;
  double* zpos = nullptr;
  double* cpos = nullptr;
  float* epos = nullptr;
  int* hasval = nullptr;
  double* loss_row = nullptr;
  float* offr = nullptr;      // [maxB] per-row softmax offsets (exact mode)
  float* dbgz = nullptr;      // [maxB][ncols] debug logits (PFC_FLAG_DEBUG_LOGITS)
  bool exact = false;         // per-row offsets on every step (s > kFixedOffsetMaxScale or forced)
  bool exact_retry = false;   // this step reruns a fixed-offset step that underflowed
  bool underflowed = false;   // the last checked step failed with a fixed-offset underflow
  // backward
  void* G = nullptr;       // E^T [ncols_pad][ldg]: exp(z - o) (bf16 / fp32), class-major
  void* xs = nullptr;      // [maxB][Dp] rowscale * x^
  float* poscorr = nullptr;  // [nk * pmax][D]
  int32_t* pslot = nullptr;  // [ncols]
  float* dwt = nullptr;      // fp32 validation path: [ncols][D]
  int64_t pmax = 1;
  int64_t cap_alloc = 0;     // capacity the column buffers were allocated for
  float* dx_part = nullptr;  // [S][maxB][D]
  float* dX = nullptr;       // [maxB][D]
  int max_splits = 1;
  // host-path scratch
  double* xdb = nullptr;  // D x maxB fp64
  StepStatus* st = nullptr;
  StepStatus* st_host = nullptr;
  StepParams* sp = nullptr;
  bool reset_status = true;  // false while asynchronous device steps are in flight
  // CUDA graph of the device step (one per batch size); sampler_kernel (which opens the step)
  // is the node whose arguments change per step
  // captured steps: slot 0 = device-resident I/O (pfc_gpu_step_device), slot 1 = the host
  // drop-in with its copies inside the graph (pfc_gpu_step with pinned host buffers)
  struct GraphSlot {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaGraphNode_t gbegin = nullptr;
    cudaGraphNode_t cp_x = nullptr, cp_dx = nullptr;  // slot 1 memcpy nodes
    const void* cp_ptr[3] = {nullptr, nullptr, nullptr};  // host pointers the nodes hold
    int64_t gB = -1;
    int64_t glaunches = 0;
    uint64_t gbytes = 0, gwire = 0;  // collective bytes per replay
  } gs[4];  // + 2: the per-row offset (exact) variants
  // host drop-in with overlapped copies: X upload + conversion + normalisation run on s2 while
  // the sampler and gather run; dX conversion + download on s2 while the dW GEMM runs
  struct E2E {
    bool on = false;
    const double* xdb_h = nullptr;
    const int64_t* lab_h = nullptr;
    double* dxdb_h = nullptr;
  } e2e;
  cudaEvent_t ev_s = nullptr, ev_x = nullptr, ev_dx = nullptr, ev_out = nullptr;
  // tensor maps cached per batch
  int64_t tm_B = -1;
  CUtensorMap tm_x_k, tm_w_k, tm_w_k128, tm_e_st, tm_e_k, tm_e_k16, tm_w_mn, tm_e_mn, tm_xs_mn;
  // collectives: NCCL communicator, or the loopback group (comm.cuh)
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopGroup> loop;
  uint8_t loop_id[128] = {};
  // bookkeeping
  int64_t lastB = 0;
  int64_t launches = 0;
  PhaseTimer pt;
  bool pdl = true;  // launch the step's kernels with programmatic stream serialisation
  std::vector<void*> allocs;
  struct Guard {
    uint8_t* base;  // [kGuardBytes guard][user bytes][kGuardBytes guard] (PFC_FLAG_GUARD)
    size_t user;
  };
  std::vector<Guard> guards;
};

// PFC_FLAG_GUARD (the out-of-bounds write check that stands in for compute-sanitizer, which
// this pool does not allow): every context buffer sits between two guard regions
constexpr size_t kGuardBytes = 4096;
constexpr int kGuardByte = 0xA5;

// Largest margin scale that keeps the fixed softmax offset o = max(0, s - 40): above it every
// step takes per-row offsets from a max-only pass (epilogues.cuh header).
constexpr double kFixedOffsetMaxScale = 64.0;
inline bool exact_now(const Ctx* c) { return c->exact || c->exact_retry; }

int fail(Ctx* c, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_create_error = buf;
  return code;
}

#define CUDA_TRY(c, expr)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail((c), PFC_ERR_CUDA, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),    \
                  __FILE__, __LINE__, cudaGetErrorString(e_));                              \
  } while (0)

#define NCCL_TRY(c, expr)                                                                   \
  do {                                                                                      \
    int r_ = (expr);                                                                        \
    if (r_ != 0)                                                                            \
      return fail((c), PFC_ERR_NCCL, "NCCL error %d (%s) at %s:%d", r_,                     \
                  g_nccl.GetErrorString ? g_nccl.GetErrorString(r_) : "?", __FILE__, __LINE__); \
  } while (0)

// One collective through the context's communicator.  kind 0: all-gather (count per rank),
// 1: all-reduce (count), 2: reduce-scatter (count per rank).  The bytes this rank hands to it
// (the larger of its send and receive buffers) are added to the step's accounting.
int comm_call(Ctx* c, int kind, const void* send, void* recv, size_t count, CommDt dt, CommOp op,
              cudaStream_t s) {
  const uint64_t es = dt_size(dt);
  const uint64_t S = (kind == 1 ? 1 : (uint64_t)c->R) * (uint64_t)count * es;  // whole buffer
  c->step_nccl_bytes += S;
  c->step_wire_bytes += (kind == 1 ? 2 : 1) * (uint64_t)(c->R - 1) * S;
  if (c->loop) {
    const cudaError_t e = loop_collective(*c->loop, c->rank, kind, send, recv, count, dt, op, s);
    if (e != cudaSuccess)
      return fail(c, PFC_ERR_CUDA, "loopback collective failed: %s", cudaGetErrorString(e));
    return PFC_OK;
  }
  int r;
  if (kind == 0) r = g_nccl.AllGather(send, recv, count, nccl_dt(dt), c->comm, s);
  else if (kind == 1) r = g_nccl.AllReduce(send, recv, count, nccl_dt(dt), nccl_op(op), c->comm, s);
  else r = g_nccl.ReduceScatter(send, recv, count, nccl_dt(dt), nccl_op(op), c->comm, s);
  if (r != 0)
    return fail(c, PFC_ERR_NCCL, "NCCL error %d (%s)", r,
                g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
  return PFC_OK;
}
inline int comm_all_gather(Ctx* c, const void* send, void* recv, size_t count, CommDt dt,
                           cudaStream_t s) {
  return comm_call(c, 0, send, recv, count, dt, kSum, s);
}
inline int comm_all_reduce(Ctx* c, const void* send, void* recv, size_t count, CommDt dt,
                           CommOp op, cudaStream_t s) {
  return comm_call(c, 1, send, recv, count, dt, op, s);
}
inline int comm_reduce_scatter(Ctx* c, const void* send, void* recv, size_t count, CommDt dt,
                               CommOp op, cudaStream_t s) {
  return comm_call(c, 2, send, recv, count, dt, op, s);
}
#define COMM_TRY(expr)               \
  do {                               \
    if (int rc_ = (expr)) return rc_; \
  } while (0)

template <typename T>
cudaError_t dalloc(Ctx* c, T** p, size_t n) {
  void* q = nullptr;
  const size_t user = n * sizeof(T) + 256;
  if (c->d.flags & PFC_FLAG_GUARD) {  // [guard][buffer][guard], guards filled with the pattern
    cudaError_t e = cudaMalloc(&q, user + 2 * kGuardBytes);
    if (e != cudaSuccess) return e;
    c->allocs.push_back(q);
    uint8_t* b = static_cast<uint8_t*>(q);
    cudaMemset(b, kGuardByte, kGuardBytes);
    cudaMemset(b + kGuardBytes, 0, user);
    cudaMemset(b + kGuardBytes + user, kGuardByte, kGuardBytes);
    c->guards.push_back({b, user});
    *p = reinterpret_cast<T*>(b + kGuardBytes);
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc(&q, user);
  if (e == cudaSuccess) {
    c->allocs.push_back(q);
    cudaMemset(q, 0, user);
  }
  *p = static_cast<T*>(q);
  return e;
}

void phase(Ctx* c, const char* name) {
  if (!c->pt.enabled || c->pt.n >= PhaseTimer::kMax) return;
  c->pt.names[c->pt.n] = name;
  cudaEventRecord(c->pt.ev[c->pt.n + 1], c->stream);
  c->pt.n++;
}

// PDL on the device path only: with the host drop-in's copy nodes forked around the kernels,
// programmatic edges measured slower end to end (360k: 0.39 vs 0.31 ms per step).
inline bool use_pdl(const Ctx* c) { return c->pdl && !c->e2e.on; }

// Launch a step kernel with programmatic stream serialisation (PDL, common.cuh pdl_entry):
// its CTAs may be scheduled while the previous kernel on the stream drains.
template <typename... KArgs, typename... Args>
cudaError_t klaunch(Ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                    cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = use_pdl(c) ? 1 : 0;
  c->launches++;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------ GEMM launchers
template <int BN, int STAGES, int NWG, bool A_MN, bool B_MN, class Epi, int CG = 1,
          class OT = __nv_bfloat16>
cudaError_t launch_umma(Ctx* c, const CUtensorMap& ta, const CUtensorMap& tb, const GemmGeom& g,
                        const Epi& epi) {
  auto kern = umma_gemm_kernel<BN, STAGES, NWG, A_MN, B_MN, Epi, CG, OT>;
  constexpr int smem = umma_smem_bytes<BN, STAGES, NWG, Epi, CG>();
  static_assert(smem <= 232448, "shared memory budget");
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem)) return e;
  const int total = g.total();
  if (total <= 0) return cudaSuccess;
  constexpr int kCl = CG > Epi::kCluster ? CG : Epi::kCluster;
  if constexpr (kCl > 1) {
    // clusters of kCl CTAs: the grid (the tile stride of the persistent schedule) is a multiple
    // of the cluster size.  Epilogue clusters (kCluster) own the dim blocks of one class block,
    // one tile per CTA; CTA pairs (CG = 2) own one pair tile per cluster.
    int grid = (c->num_sms / kCl) * kCl;
    const int need = CG == 2 ? total * 2 : total;
    if (grid > need) grid = need;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(32 * PFC_CTRL_WARPS + 128 * NWG);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = use_pdl(c) ? 2 : 1;
    c->launches++;
    return cudaLaunchKernelEx(&cfg, kern, ta, tb, g, epi);
  } else {
    const int grid = total < c->num_sms ? total : c->num_sms;
    return klaunch(c, kern, dim3(grid), dim3(32 * PFC_CTRL_WARPS + 128 * NWG), smem, c->stream,
                   ta, tb, g, epi);
  }
}

template <bool A_MN, bool B_MN, class Epi>
cudaError_t launch_simt(Ctx* c, const float* A, int lda, const float* Bm, int ldb,
                        const GemmGeom& g, const Epi& epi) {
  auto kern = simt_gemm_kernel<A_MN, B_MN, Epi>;
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), kSimtSmemBytes))
    return e;
  if (g.total() <= 0) return cudaSuccess;
  return klaunch(c, kern, dim3(g.total()), dim3(128), kSimtSmemBytes, c->stream, A, lda, Bm, ldb,
                 g, epi);
}

int ensure_maps(Ctx* c, int64_t B) {
  if (!c->umma || c->tm_B == B) return PFC_OK;
  bool ok = true;
  const int el = c->tf32 ? 4 : 2;       // operand bytes
  const uint32_t kb = 128 / (uint32_t)el;  // elements per 128-byte swizzle row
  const auto sw = CU_TENSOR_MAP_SWIZZLE_128B;
  // MN-major operands: tf32 needs the 32-byte-atom variant (gemm.cuh make_sdesc_sw128_32b)
  const auto swm = c->tf32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  // logits GEMM (M = b, N = classes): A = X^ [B][Dp], B = W^ [ncols][Dp], both K-major;
  // its epilogue stores E^T [ncols][ldg] (bf16: per-warp box 32 b x 32 classes, 64B swizzle)
  ok &= make_map(&c->tm_x_k, c->xh, c->Dp, B, c->Dp, 128, kb, sw, el);
  ok &= make_map(&c->tm_w_k, c->wh, c->Dp, c->ncols, c->Dp, kFwdBN / kFwdCG, kb, sw, el);
  ok &= make_map(&c->tm_w_k128, c->wh, c->Dp, c->ncols, c->Dp, kNarrowBN / kFwdCG, kb, sw, el);
  if (c->bf16)
    ok &= make_map(&c->tm_e_st, c->G, B, c->ncols, c->ldg, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  // dX GEMM (M = b, N = d, K = classes): A = E^T read MN-major (b contiguous); B = W^ MN-major
  ok &= make_map(&c->tm_e_mn, c->G, B, c->ncols, c->ldg, kb, kb, swm, el);
  ok &= make_map(&c->tm_w_mn, c->wh, c->Dp, c->ncols, c->Dp, kb, kb, swm, el);
  // dW GEMM (M = classes, N = d, K = b): A = E^T K-major (whole class blocks contiguous);
  // B = rowscale * x^ MN-major
  ok &= make_map(&c->tm_e_k, c->G, B, c->ncols, c->ldg, 128, kb, sw, el);
  ok &= make_map(&c->tm_e_k16, c->G, B, c->ncols, c->ldg, 16, kb, sw, el);  // dW half tiles
  ok &= make_map(&c->tm_xs_mn, c->xs, c->Dp, B, c->Dp, kb, kb, swm, el);
  if (!ok) return fail(c, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  c->tm_B = B;
  return PFC_OK;
}

// The sampler's arguments for this step (sampler.cu SamplerArgs).
SamplerArgs sampler_args(Ctx* c, const pfc_gpu_step_args* a, const float* x, const int64_t* lab,
                         float* dx_full, int64_t B, int normalize) {
  SamplerArgs sa{};
  sa.st = c->st;
  sa.sp = c->sp;
  sa.seed = a->seed;
  sa.stream = a->stream_id;
  sa.lr = (float)a->lr;
  sa.reset = c->reset_status ? 1 : 0;
  sa.x = x;
  sa.labels_in = lab;
  sa.dx = dx_full;
  sa.B = (int)B;
  sa.C = c->C;
  sa.K = (int)c->K;
  sa.blk = c->blk;
  sa.cap = (int)c->cap;
  sa.k0 = (int)c->k0;
  sa.nk = (int)c->nk;
  sa.force_sequential = (c->d.flags & PFC_FLAG_FORCE_SEQUENTIAL_SAMPLER) ? 1 : 0;
  sa.normalize = normalize;
  sa.D = (int)c->D;
  sa.Dp = (int)c->Dp;
  sa.xh = c->xh;
  sa.xnorm = c->xnorm;
  sa.bits = c->bits;
  sa.ccnt = c->ccnt;
  sa.chunk_words = c->chunk_words;
  sa.nchunk = c->nchunk;
  sa.oobs = c->oobs;
  sa.rej = c->rej;
  sa.labs = c->labs;
  sa.zpos = c->zpos;
  sa.hasval = c->d.has_filter ? c->hasval : nullptr;
  sa.meta = c->meta;
  sa.buf_cls = c->buf_cls;
  sa.pos_col = c->pos_col;
  sa.head = c->head;
  sa.nxt = c->nxt;
  sa.jv = c->jv;
  sa.pool_scratch = c->pool_scratch;
  sa.pool_stride = c->pool_stride;
  return sa;
}

// The three sampler kernels (sampler.cu): mark opens the step (no programmatic edge: it
// follows work outside the step), fill and walk follow it with PDL.  Grid-stride loops over one
// CTA of 1024 threads per SM.
cudaError_t launch_sampler(Ctx* c, SamplerArgs& sa) {
  const size_t smem = sampler_smem_bytes(c->nchunk, (int)c->nk);
  const size_t wsmem = walk_smem_bytes((int)c->nk);
  const int smax = (int)sampler_smem_bytes(kMaxSamplerChunks, kMaxSamplerLocalShards);
  const int wmax = (int)walk_smem_bytes(kMaxSamplerLocalShards);
  const void* fill = c->bf16   ? reinterpret_cast<const void*>(fill_kernel<__nv_bfloat16>)
                     : c->tf32 ? reinterpret_cast<const void*>(fill_kernel<tf32_t>)
                               : reinterpret_cast<const void*>(fill_kernel<float>);
  if (cudaError_t e = ensure_smem_attr(fill, smax)) return e;
  if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(walk_kernel), wmax)) return e;
  const dim3 grid((unsigned)c->num_sms), blk(kSamplerThreads);
  mark_kernel<<<grid, blk, 0, c->stream>>>(sa);
  c->launches++;
  if (cudaError_t e = cudaGetLastError()) return e;
  cudaError_t e = c->bf16   ? klaunch(c, fill_kernel<__nv_bfloat16>, grid, blk, smem, c->stream, sa)
                  : c->tf32 ? klaunch(c, fill_kernel<tf32_t>, grid, blk, smem, c->stream, sa)
                            : klaunch(c, fill_kernel<float>, grid, blk, smem, c->stream, sa);
  if (e != cudaSuccess) return e;
  return klaunch(c, walk_kernel, grid, blk, wsmem, c->stream, sa);
}

int dx_splits(Ctx* c, int64_t B) {
  if (c->umma) {
    const int64_t tiles = ceil_div(B, 128 * kDxCG) * kDxCG * ceil_div(c->D, kBN);  // CTAs per split
    int64_t s = c->num_sms / (tiles > 0 ? tiles : 1);
    if (s < 1) s = 1;
    return (int)std::min<int64_t>(s, c->max_splits);
  }
  const int64_t tiles = ceil_div(B, 128) * ceil_div(c->D, kSimtBN);
  int64_t s = (2 * c->num_sms) / (tiles > 0 ? tiles : 1);
  if (s < 1) s = 1;
  return (int)std::min<int64_t>(s, c->max_splits);
}

// The logits GEMM with kFwdBN-wide tiles fills at most half the SMs: use kNarrowBN tiles.
bool logits_narrow(const Ctx* c, int64_t B) {
  return ceil_div(B, 128) * ceil_div(c->ncols, kFwdBN) * 2 <= c->num_sms;
}

// Small column counts leave most clusters idle in the dW GEMM (one per 128-class block): when
// even twice as many blocks fit in one round, every block becomes two half tiles (64 rows, 16 per
// TMEM lane quadrant, 4 per warp), which halves the round (10k: 0.077 -> 0.073 ms per step).  A
// half tail on a longer schedule measured slower (2M: +1%), so it is not used there.
void dw_half_tail(Ctx* c, GemmGeom& g) {
  const int64_t nb = g.m_tiles;
  const int64_t W = std::max(c->num_sms / g.n_tiles, 1);  // clusters (CTAs per block: n_tiles)
  if (2 * nb > W) return;
  g.half_m0 = 0;
  g.m_tiles = (int)ceil_div(c->ncols, 64);
}

// The device pipeline for one step on a gathered global batch of B rows.
// x: [B][D] fp32 rows; lab: [B] int64 (device).  Writes the rank-local partial dX into
// dx_full ([B][D]).
template <typename ST, typename OT, bool kUmma>
int run_pipeline(Ctx* c, const float* x, const int64_t* lab, int64_t B,
                 const pfc_gpu_step_args* a, float* dx_full) {
  // tcgen05 engine: bf16 operands (kind::f16) or fp32 operands (kind::tf32, the TF32 mode)
  constexpr bool kTf = kUmma && sizeof(OT) == 4;
  constexpr int BKU = kUmma ? 128 / (int)sizeof(OT) : 64;  // K elements per GEMM stage
  constexpr int FCG = kTf ? 1 : kFwdCG;
  constexpr int XCG = kTf ? 1 : kDxCG;
  cudaStream_t s = c->stream;
  const int bs = 256;
  if (int rc = ensure_maps(c, B)) return rc;
  const bool e2e = c->e2e.on;
  if (e2e) {  // features: upload (D x B fp64), -> [B][D] fp32, normalise; joined before the GEMM.
    // Needs nothing from the step's first kernel, so it forks before it.
    CUDA_TRY(c, cudaEventRecord(c->ev_s, s));
    CUDA_TRY(c, cudaStreamWaitEvent(c->s2, c->ev_s, 0));
    CUDA_TRY(c, cudaMemcpyAsync(c->xdb, c->e2e.xdb_h, sizeof(double) * B * c->D,
                                cudaMemcpyHostToDevice, c->s2));
    dim3 grid((unsigned)ceil_div(B, 32), (unsigned)ceil_div(c->D, 32)), blk(32, 8);
    x_from_dxb_kernel<<<grid, blk, 0, c->s2>>>(c->xdb, (int)c->D, (int)B, c->X);
    normalize_x_kernel<OT><<<(unsigned)ceil_div(B * 32, bs), bs, 0, c->s2>>>(
        c->X, (int)B, (int)c->D, (int)c->Dp, static_cast<OT*>(c->xh), c->xnorm);
    c->launches += 2;
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaEventRecord(c->ev_x, c->s2));
  }
  // ---- sampler (build_buffers, sampler.hpp:63-126); its first kernel also opens the step.
  // (host drop-in: `lab` is the caller's page-locked labels, read once over PCIe by the sampler)
  {
    SamplerArgs sa = sampler_args(c, a, x, lab, dx_full, B, e2e ? 0 : 1);
    CUDA_TRY(c, launch_sampler(c, sa));
  }
  phase(c, "sampler");
  // ---- gather + normalise sampled centres
  OT* wh = static_cast<OT*>(c->wh);
  CUDA_TRY(c, klaunch(c, gather_w_kernel<OT>, dim3((unsigned)ceil_div(c->ncols_pad * 32, bs)),
                      dim3(bs), 0, s, c->W, (int)c->D, (int)c->Dp, c->buf_cls, (int)c->ncols,
                      (int)c->ncols_pad, c->cls_lo, c->rows, wh, c->wnorm, c->lrow, c->pslot,
                      (const StepStatus*)c->st));
  phase(c, "gather");

  constexpr int BN = kUmma ? kBN : kSimtBN;
  constexpr int FBN = kUmma ? kFwdBN : kSimtBN;  // logits GEMM tile width
  constexpr int NWG = kUmma ? kFwdNWG : 1;         // logits GEMM epilogue warpgroups
  ST* ps = static_cast<ST*>(c->part_s);
  OT* E = static_cast<OT*>(c->G);
  const float tau = (float)c->d.filter_threshold;
  const bool filt = c->d.has_filter != 0;
  if (e2e) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_x, 0));
  // small problems (the 10k CPU-reference workload: 4 tiles) take narrow tiles: twice the CTAs
  const bool narrow = kUmma && logits_narrow(c, B);
  const GemmGeom gf = make_geom((int)B, (int)c->ncols, (int)c->Dp, narrow ? kNarrowBN : FBN, 1, 0,
                                kUmma ? 128 * FCG : 128, BKU);
  const bool exact = exact_now(c);
  if (exact) {
    // ---- per-row offsets: max-only pass of the logits GEMM -> o_b (rank max: collective 1,
    // shardsim.hpp:270-299).  Its slice maxima reuse the row-sum slices (consumed before the
    // logits pass rewrites them).
    float* pm = reinterpret_cast<float*>(c->part_s);
    cudaError_t err;
    auto go = [&](auto e) {
      if constexpr (kUmma) {
        if (narrow)
          return launch_umma<kNarrowBN, kFwdStages, kFwdNWG, false, false, decltype(e), FCG, OT>(c, c->tm_x_k, c->tm_w_k128, gf, e);
        return launch_umma<kFwdBN, kFwdStages, kFwdNWG, false, false, decltype(e), FCG, OT>(c, c->tm_x_k, c->tm_w_k, gf, e);
      } else return launch_simt<false, false>(c, (const float*)c->xh, (int)c->Dp,
                                              (const float*)c->wh, (int)c->Dp, gf, e);
    };
    if (filt) err = go(MaxEpi<true>{{}, (int)B, (int)c->ncols, c->pos_col, c->mg, tau, pm, c->zpos});
    else err = go(MaxEpi<false>{{}, (int)B, (int)c->ncols, c->pos_col, c->mg, tau, pm, c->zpos});
    CUDA_TRY(c, err);
    CUDA_TRY(c, klaunch(c, row_offset_kernel, dim3((unsigned)ceil_div(B, bs)), dim3(bs), 0, s,
                        pm, gf.n_tiles * NWG, (int)B, c->pos_col, c->zpos, c->mg, c->offr));
    if (c->coll) COMM_TRY(comm_all_reduce(c, c->offr, c->offr, B, kF32, kMax, s));
    phase(c, "row_offsets");
  }
  const float* offr = exact ? c->offr : nullptr;
  // ---- logits GEMM + margin + E = exp(z - o) and its per-slice row sums (shardsim.hpp:249-318)
  {
    cudaError_t err;
    auto go = [&](auto e) {
      if constexpr (kUmma) {
        if (narrow)
          return launch_umma<kNarrowBN, kFwdStages, kFwdNWG, false, false, decltype(e), FCG, OT>(c, c->tm_x_k, c->tm_w_k128, gf, e);
        return launch_umma<kFwdBN, kFwdStages, kFwdNWG, false, false, decltype(e), FCG, OT>(c, c->tm_x_k, c->tm_w_k, gf, e);
      } else return launch_simt<false, false>(c, (const float*)c->xh, (int)c->Dp,
                                              (const float*)c->wh, (int)c->Dp, gf, e);
    };
    if (filt)
      err = go(FwdEpi<ST, OT, true, kUmma && !kTf>{{}, c->tm_e_st, (int)B, (int)c->ncols, (int)c->ldg, c->pos_col,
                                           c->mg, tau, ps, c->zpos, c->cpos, c->epos, c->hasval, E,
                                           offr, c->dbgz});
    else
      err = go(FwdEpi<ST, OT, false, kUmma && !kTf>{{}, c->tm_e_st, (int)B, (int)c->ncols, (int)c->ldg, c->pos_col,
                                            c->mg, tau, ps, c->zpos, c->cpos, c->epos, c->hasval, E,
                                            offr, c->dbgz});
    CUDA_TRY(c, err);
  }
  phase(c, "logits_gemm");
  // ---- softmax statistics: slices -> rank-local sum -> ranks (collectives 1 + 2) -> loss
  const int T = gf.n_tiles * NWG;
  ST* ls = static_cast<ST*>(c->ls);
  const unsigned nrb = (unsigned)ceil_div(B, kRowsPerBlk);
  if (c->coll) {  // the rank-local sums are exchanged; with one rank finalize forms them
    CUDA_TRY(c, klaunch(c, local_sums_kernel<ST>, dim3(nrb), dim3(kStatsThreads), 0, s, ps, T, (int)B,
                        ls + c->rank * B));
    const CommDt dt = sizeof(ST) == 8 ? kF64 : kF32;
    COMM_TRY(comm_all_gather(c, ls + c->rank * B, ls, B, dt, s));
    COMM_TRY(comm_all_reduce(c, c->zpos, c->zpos, B, kF64, kSum, s));
    if (filt) COMM_TRY(comm_all_reduce(c, c->hasval, c->hasval, B, kI32, kSum, s));
  }
  ST* rsc = static_cast<ST*>(c->rowscale);
  ST* dlt = static_cast<ST*>(c->delta);
  CUDA_TRY(c, klaunch(c, finalize_stats_kernel<ST>, dim3(nrb), dim3(kStatsThreads), 0, s, (const ST*)ls,
                      (int)c->R, (const ST*)(c->coll ? nullptr : ps), T, (int)B,
                      (const double*)c->zpos, (const double*)c->cpos, (const float*)c->epos,
                      (const int32_t*)c->pos_col, (const int*)c->hasval, filt ? 1 : 0, c->mg,
                      offr, rsc, dlt, c->loss_row, c->st));
  CUDA_TRY(c, cudaGetLastError());
  phase(c, "softmax_stats");
  // X^s and the positive corrections feed only the dW GEMM: they run on a forked stream,
  // concurrently with the dX GEMM (which leaves SMs free: split-K grid of 144 CTAs)
  CUDA_TRY(c, cudaEventRecord(c->ev_fork, s));
  CUDA_TRY(c, cudaStreamWaitEvent(c->s2, c->ev_fork, 0));
  xs_kernel<ST, OT><<<(unsigned)B, 128, 0, c->s2>>>(c->sp, c->xnorm, rsc, (int)B, (int)c->D,
                                                    (int)c->Dp, static_cast<OT*>(c->xs), c->meta,
                                                    (int)c->nk, (int)c->cap, c->jv, c->head,
                                                    c->pool_stride, c->st);
  poscorr_kernel<<<dim3((unsigned)c->pmax, (unsigned)c->nk), 256, 0, c->s2>>>(
      c->meta, (int)c->cap, (int)c->pmax, c->pos_col, (int)B, c->sp, c->xnorm, (int)c->D,
      std::is_same<ST, float>::value ? reinterpret_cast<const float*>(dlt) : nullptr,
      std::is_same<ST, double>::value ? reinterpret_cast<const double*>(dlt) : nullptr,
      c->poscorr, c->pslot, c->st);
  c->launches += 2;
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaEventRecord(c->ev_join, c->s2));
  // ---- dX = rowscale * E W^ + delta w^_pos (split-K), tangent projection (shardsim.hpp:363-376)
  {
    const int S = dx_splits(c, B);
    const GemmGeom gx = make_geom((int)B, (int)c->D, (int)c->ncols, BN, S, 0, kUmma ? 128 * XCG : 128, BKU);
    DxPartEpi e{{}, (int)B, (int)c->D, c->dx_part};
    cudaError_t err;
    if constexpr (kUmma) err = launch_umma<kBN, 4, 1, true, true, DxPartEpi, XCG, OT>(c, c->tm_e_mn, c->tm_w_mn, gx, e);
    else err = launch_simt<true, true>(c, (const float*)c->G, (int)c->ldg, (const float*)c->wh,
                                       (int)c->Dp, gx, e);
    CUDA_TRY(c, err);
    const int dpt = (int)ceil_div(c->D, 256);
#define PFC_FIN(N)                                                                           \
  klaunch(c, dx_finalize_kernel<N, ST>, dim3((unsigned)B), dim3(256), 0, s,                 \
          (const float*)c->dx_part, gx.splits, (const StepParams*)c->sp,                     \
          (const float*)c->xnorm, (const ST*)rsc, (const ST*)dlt, (const int32_t*)c->pos_col, \
          (const int32_t*)c->lrow, (const float*)c->wnorm, (const float*)c->W, (int)B,        \
          (int)c->D, c->st)
    if (dpt <= 1) CUDA_TRY(c, PFC_FIN(1));
    else if (dpt <= 2) CUDA_TRY(c, PFC_FIN(2));
    else if (dpt <= 4) CUDA_TRY(c, PFC_FIN(4));
    else CUDA_TRY(c, PFC_FIN(8));
#undef PFC_FIN
  }
  if (e2e) {  // d_features: [sum over ranks], -> D x B fp64, download; overlaps the dW GEMM
    CUDA_TRY(c, cudaEventRecord(c->ev_dx, s));
    CUDA_TRY(c, cudaStreamWaitEvent(c->s2, c->ev_dx, 0));
    if (c->coll)  // the drop-in returns the FULL summed d_features on every rank
      COMM_TRY(comm_all_reduce(c, c->dX, c->dX, B * c->D, kF32, kSum, c->s2));
    dim3 grid((unsigned)ceil_div(B, 32), (unsigned)ceil_div(c->D, 32)), blk(32, 8);
    dx_to_dxb_kernel<<<grid, blk, 0, c->s2>>>(c->dX, (int)c->D, (int)B, c->xdb);
    c->launches++;
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaMemcpyAsync(c->e2e.dxdb_h, c->xdb, sizeof(double) * B * c->D,
                                cudaMemcpyDeviceToHost, c->s2));
    // the step status is final after dx_finalize (the dW GEMM only reads it): its download rides
    // the same copy stream instead of trailing the step
    CUDA_TRY(c, cudaMemcpyAsync(c->st_host, c->st, sizeof(StepStatus), cudaMemcpyDeviceToHost,
                                c->s2));
    CUDA_TRY(c, cudaEventRecord(c->ev_out, c->s2));
  }
  phase(c, "dx_gemm");
  CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_join, 0));  // X^s and the positive corrections
  // ---- dwt = E^T (rowscale x^) + positive corrections; center_proj; fused momentum-SGD
  {
    GemmGeom gw = make_geom((int)c->ncols, (int)c->D, (int)B, BN, 1, 1, 128, BKU);
    if constexpr (kUmma) dw_half_tail(c, gw);
    cudaError_t err;
    if constexpr (kUmma) {
      // one cluster CTA per 256-dim block of a class block (tile order n fastest)
      // operand pipeline vs W / momentum ring: the GEMM's K is the batch, so past 2 KB of E^T
      // per class row (bf16 B > 1024, tf32 B > 512) its operand stream needs a third stage
      // (10M / B = 2048: dW 3.26 vs 3.52 ms; tf32 2M: 0.612 vs 0.675 ms), paid for with a 3 KB
      // ring (bf16 2M / B = 1024 keeps 2 stages + 6 KB: 0.475 vs 0.488 ms)
      const bool deep = B * (int64_t)sizeof(OT) > kDwDeepBatch * 2;  // K bytes per E^T row
      auto dw = [&](auto nc) {
        constexpr int NC = decltype(nc)::value;
        auto go = [&](auto e) {
          using E = decltype(e);
          constexpr int S = E::R::kCap == PFC_DW_CAP ? PFC_DW_STAGES : 3;
          return launch_umma<kBN, S, 4, false, true, E, 1, OT>(c, c->tm_e_k, c->tm_xs_mn, gw, e);
        };
        auto make = [&](auto e) {
          e.ncols = (int)c->ncols;
          e.D = (int)c->D;
          e.wnorm = c->wnorm;
          e.lrow = c->lrow;
          e.pslot = c->pslot;
          e.poscorr = c->poscorr;
          e.W = c->W;
          e.Mom = c->M;
          e.sp = c->sp;
          e.mu = (float)c->d.momentum;
          e.wd = (float)c->d.weight_decay;
          e.st = c->st;
          if constexpr (decltype(e)::kHalfTiles) e.tm_a16 = c->tm_e_k16;
          return go(e);
        };
        const bool halves = gw.half_m0 < gw.m_tiles;
        if (deep) return halves ? make(DwUpdateEpi<NC, 3, true>{}) : make(DwUpdateEpi<NC, 3>{});
        return halves ? make(DwUpdateEpi<NC, PFC_DW_CAP, true>{}) : make(DwUpdateEpi<NC>{});
      };
      switch (gw.n_tiles) {
        case 1: err = dw(std::integral_constant<int, 1>{}); break;
        case 2: err = dw(std::integral_constant<int, 2>{}); break;
        case 3: err = dw(std::integral_constant<int, 3>{}); break;
        default: err = dw(std::integral_constant<int, 4>{}); break;
      }
    } else {
      err = launch_simt<false, true>(c, (const float*)c->G, (int)c->ldg, (const float*)c->xs,
                                     (int)c->Dp, gw, DwStoreEpi{{}, (int)c->ncols, (int)c->D, c->dwt});
      if (err == cudaSuccess) {
        err = klaunch(c, dw_rows_update_kernel, dim3((unsigned)ceil_div(c->ncols * 32, bs)),
                      dim3(bs), 0, s, (const float*)c->dwt, (const int32_t*)c->lrow,
                      (const float*)c->wnorm, (const int32_t*)c->pslot, (const float*)c->poscorr,
                      (int)c->ncols, (int)c->D, c->W, c->M, (const StepParams*)c->sp,
                      (float)c->d.momentum, (float)c->d.weight_decay, (const StepStatus*)c->st);
      }
    }
    CUDA_TRY(c, err);
  }
  phase(c, "dw_update_gemm");
  if (e2e) CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_out, 0));
  return PFC_OK;
}

int run_step(Ctx* c, const float* x, const int64_t* lab, int64_t B, const pfc_gpu_step_args* a,
             float* dx_full) {
  c->lastB = B;
  // the loopback communicator synchronises host threads: it cannot be captured
  const bool graph = !(c->d.flags & PFC_FLAG_NO_GRAPH) && !c->pt.enabled && !c->loop;
  auto pipeline = [&]() {
    c->launches = 0;
    if (c->bf16) return run_pipeline<float, __nv_bfloat16, true>(c, x, lab, B, a, dx_full);
    if (c->tf32) return run_pipeline<float, tf32_t, true>(c, x, lab, B, a, dx_full);
    return run_pipeline<double, float, false>(c, x, lab, B, a, dx_full);
  };
  if (!graph) {
    if (c->pt.enabled) {
      c->pt.n = 0;
      cudaEventRecord(c->pt.ev[0], c->stream);
    }
    return pipeline();
  }
  Ctx::GraphSlot& G = c->gs[(c->e2e.on ? 1 : 0) + (exact_now(c) ? 2 : 0)];
  if (!G.gexec || G.gB != B) {  // capture the step once per batch size
    const uint64_t bytes0 = c->step_nccl_bytes, wire0 = c->step_wire_bytes;
    if (G.gexec) {
      cudaGraphExecDestroy(G.gexec);
      cudaGraphDestroy(G.graph);
      G.gexec = nullptr;
    }
    CUDA_TRY(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = pipeline();
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    CUDA_TRY(c, ce);
    CUDA_TRY(c, cudaGraphInstantiate(&G.gexec, g, 0));
    G.graph = g;
    size_t n = 0;
    CUDA_TRY(c, cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CUDA_TRY(c, cudaGraphGetNodes(g, nodes.data(), &n));
    G.gbegin = G.cp_x = G.cp_dx = nullptr;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      cudaGraphNodeGetType(nd, &ty);
      if (ty == cudaGraphNodeTypeMemcpy) {  // the host drop-in's copies (slot 1)
        cudaMemcpy3DParms mp{};
        if (cudaGraphMemcpyNodeGetParams(nd, &mp) != cudaSuccess) continue;
        if (mp.dstPtr.ptr == c->xdb) G.cp_x = nd;
        else if (mp.srcPtr.ptr == c->xdb) G.cp_dx = nd;
        continue;
      }
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp{};
      if (cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess &&
          kp.func == reinterpret_cast<void*>(mark_kernel))
        G.gbegin = nd;
    }
    if (!G.gbegin) return fail(c, PFC_ERR_CUDA, "graph capture lost the step-opening node");
    if (c->e2e.on && (!G.cp_x || !G.cp_dx))
      return fail(c, PFC_ERR_CUDA, "graph capture lost a host copy node");
    G.gB = B;
    G.glaunches = c->launches;
    G.gbytes = c->step_nccl_bytes - bytes0;
    G.gwire = c->step_wire_bytes - wire0;
    c->step_nccl_bytes = bytes0;
    c->step_wire_bytes = wire0;
    G.cp_ptr[0] = G.cp_ptr[1] = G.cp_ptr[2] = nullptr;
  }
  // per step, only the step-opening kernel's arguments (and the host drop-in's host pointers)
  // change; the other arguments and the launch shape are the captured ones
  // the fill / walk nodes read the per-step values from the StepParams block mark_kernel
  // writes, so only the opening node's arguments change (the captured SamplerArgs of the other
  // two nodes are identical for every step of this batch size except the fields below, which
  // they do not use: seed, stream, lr, reset, labels_in)
  SamplerArgs sa = sampler_args(c, a, x, lab, dx_full, B, c->e2e.on ? 0 : 1);
  void* args[] = {&sa};
  cudaKernelNodeParams kp{};
  kp.func = reinterpret_cast<void*>(mark_kernel);
  kp.gridDim = dim3((unsigned)c->num_sms);
  kp.blockDim = dim3(kSamplerThreads);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  kp.extra = nullptr;
  CUDA_TRY(c, cudaGraphExecKernelNodeSetParams(G.gexec, G.gbegin, &kp));
  if (c->e2e.on) {  // re-point the copy nodes when the caller's host buffers changed
    if (G.cp_ptr[1] != c->e2e.xdb_h)
      CUDA_TRY(c, cudaGraphExecMemcpyNodeSetParams1D(G.gexec, G.cp_x, c->xdb, c->e2e.xdb_h,
                                                     sizeof(double) * B * c->D,
                                                     cudaMemcpyHostToDevice));
    if (G.cp_ptr[2] != c->e2e.dxdb_h)
      CUDA_TRY(c, cudaGraphExecMemcpyNodeSetParams1D(G.gexec, G.cp_dx, c->e2e.dxdb_h, c->xdb,
                                                     sizeof(double) * B * c->D,
                                                     cudaMemcpyDeviceToHost));
    G.cp_ptr[1] = c->e2e.xdb_h;
    G.cp_ptr[2] = c->e2e.dxdb_h;
  }
  CUDA_TRY(c, cudaGraphLaunch(G.gexec, c->stream));
  c->launches = G.glaunches;
  c->step_nccl_bytes += G.gbytes;  // the collectives the graph replays
  c->step_wire_bytes += G.gwire;
  return PFC_OK;
}

void trace_closed_form(Ctx* c, int64_t B, pfc_gpu_step_out* o) {
  // reference accounting (shardsim.hpp:192-193, 327-328, 395-398)
  const uint64_t K = (uint64_t)c->K, b = (uint64_t)B, dd = (uint64_t)c->D;
  o->allgather_bytes = (K - 1) * b * dd * 8;
  o->reduce_scalar_bytes = (K - 1) * b * 2 * 2 * 8;
  o->reduce_grad_bytes = (K - 1) * b * dd * 2 * 8;
  o->reduce_ops = 3;
  o->capacity = c->cap;
}

// Check the device status block; map to the reference's error types and messages.
int check_status(Ctx* c, int64_t step_index, int64_t B, pfc_gpu_step_out* out) {
  const StepStatus& st = *c->st_host;
  c->underflowed = false;
  if (st.label_oob)
    return fail(c, PFC_ERR_CONTRACT, "build_buffers: label %lld outside [0, %lld)",
                (long long)st.oob_label, (long long)c->C);
  if (st.capacity_shard >= 0) {
    const int64_t k = st.capacity_shard;
    const int64_t lo = std::min(k * c->blk, c->C), hi = std::min((k + 1) * c->blk, c->C);
    if (st.capacity_npos > c->cap)
      return fail(c, PFC_ERR_CAPACITY,
                  "build_buffers: shard %lld received %d distinct positives but capacity is %lld; "
                  "increase the sampling ratio r or the shard count",
                  (long long)k, st.capacity_npos, (long long)c->cap);
    return fail(c, PFC_ERR_CAPACITY,
                "build_buffers: shard %lld owns only %lld classes but capacity is %lld (C must "
                "divide evenly enough across K at this r)",
                (long long)k, (long long)(hi - lo), (long long)c->cap);
  }
  if (st.masked_row != 0x7fffffff)
    return fail(c, PFC_ERR_CONTRACT,
                "distributed_partial_step: all buffer columns masked for row %d", st.masked_row);
  if (st.underflow_row != 0x7fffffff) {
    c->underflowed = !exact_now(c);
    return fail(c, PFC_ERR_NUMERICAL,
                "pfc_gpu: row %d: every logit lies far below the fixed softmax offset "
                "max(0, s - 40) (no update was applied); the synchronous step calls rerun such a "
                "step with per-row offsets, asynchronous device steps report it (create the "
                "context with PFC_FLAG_EXACT_SOFTMAX to always use per-row offsets)",
                st.underflow_row);
  }
  if (st.nonfinite_loss)
    return fail(c, PFC_ERR_NUMERICAL, "distributed_partial_step: non-finite loss at step %lld",
                (long long)step_index);
  if (st.nonfinite_dx)
    return fail(c, PFC_ERR_NUMERICAL,
                "distributed_partial_step d_features: non-finite entry in %lldx%lld result",
                (long long)c->D, (long long)B);
  if (out) {
    out->loss = st.loss;
    out->rejection_shards = st.rejection_shards;
  out->nccl_bytes = c->step_nccl_bytes;
    out->wire_bytes = c->step_wire_bytes;
    trace_closed_form(c, B, out);
  }
  return PFC_OK;
}

// Runs a synchronous step; when it failed only because the fixed softmax offset underflowed
// (nothing was updated), reruns it with per-row offsets.  Every rank sees the same global row
// sums, so all ranks take the same branch (their collectives stay matched).
template <class F>
int with_exact_retry(Ctx* c, F&& once) {
  int rc = once();
  if (rc == PFC_ERR_NUMERICAL && c->underflowed) {
    c->exact_retry = true;
    c->reset_status = true;
    rc = once();
    c->exact_retry = false;
  }
  return rc;
}

int finish_phase_timing(Ctx* c) {
  if (!c->pt.enabled) return PFC_OK;
  CUDA_TRY(c, cudaEventSynchronize(c->pt.ev[c->pt.n]));
  for (int i = 0; i < c->pt.n; ++i) cudaEventElapsedTime(&c->pt.ms[i], c->pt.ev[i], c->pt.ev[i + 1]);
  return PFC_OK;
}

// Host-side replica of build_buffers' validation (sampler.hpp:68-98) for the host-buffer
// path, so errors are raised with the reference's text before any device work.
int host_validate(Ctx* c, const int64_t* labels, int64_t B) {
  std::vector<int64_t> s(labels, labels + B);
  std::sort(s.begin(), s.end());
  s.erase(std::unique(s.begin(), s.end()), s.end());
  for (int64_t v : s)
    if (v < 0 || v >= c->C)
      return fail(c, PFC_ERR_CONTRACT, "build_buffers: label %lld outside [0, %lld)", (long long)v,
                  (long long)c->C);
  size_t p = 0;
  for (int64_t k = 0; k < c->K; ++k) {
    const int64_t lo = std::min(k * c->blk, c->C), hi = std::min((k + 1) * c->blk, c->C);
    int64_t np = 0;
    while (p < s.size() && s[p] < hi) {
      ++np;
      ++p;
    }
    if (np > c->cap)
      return fail(c, PFC_ERR_CAPACITY,
                  "build_buffers: shard %lld received %lld distinct positives but capacity is "
                  "%lld; increase the sampling ratio r or the shard count",
                  (long long)k, (long long)np, (long long)c->cap);
    if (hi - lo < c->cap)
      return fail(c, PFC_ERR_CAPACITY,
                  "build_buffers: shard %lld owns only %lld classes but capacity is %lld (C must "
                  "divide evenly enough across K at this r)",
                  (long long)k, (long long)(hi - lo), (long long)c->cap);
  }
  return PFC_OK;
}

// buffer_capacity (sampler.hpp:50-57): ceil(C r - 1e-9) columns spread over K shards
int64_t capacity_for(int64_t C, int64_t K, double r) {
  const double want = (double)C * r;
  const int64_t total = (int64_t)std::ceil(want - 1e-9);
  return (total + K - 1) / K;
}

// the step-invariant margin state of c->d (softmax offset mode included)
void set_margin_state(Ctx* c) {
  c->mg.kind = c->d.margin_kind;
  c->mg.s = (float)c->d.margin_scale;
  c->mg.sd = c->d.margin_scale;
  c->mg.md = c->d.margin_m;
  const bool comb = c->d.margin_kind == PFC_MARGIN_COMBINED;
  c->mg.m1d = comb ? c->d.margin_m1 : 1.0;
  c->mg.m3d = comb ? c->d.margin_m3 : 0.0;
  c->mg.offd = std::max(0.0, c->d.margin_scale - 40.0);  // E = exp(z - o) <= e^40
  c->mg.off = (float)c->mg.offd;
  c->exact = c->d.margin_scale > kFixedOffsetMaxScale || (c->d.flags & PFC_FLAG_EXACT_SOFTMAX);
}

// capacity-derived geometry of c->cap
void set_cap_geometry(Ctx* c) {
  c->ncols = c->nk * c->cap;
  c->ncols_pad = round_up(std::max<int64_t>(c->ncols, 1), 256);
  c->pmax = std::max<int64_t>(1, std::min<int64_t>(c->cap, c->maxB));
}

void dfree(Ctx* c, void* p) {
  if (!p) return;
  for (size_t i = 0; i < c->guards.size(); ++i)
    if (c->guards[i].base + kGuardBytes == p) {
      p = c->guards[i].base;
      c->guards.erase(c->guards.begin() + (long)i);
      break;
    }
  for (size_t i = 0; i < c->allocs.size(); ++i)
    if (c->allocs[i] == p) {
      c->allocs.erase(c->allocs.begin() + (long)i);
      cudaFree(p);
      return;
    }
}

// The buffers whose size follows the buffer capacity (c->ncols / c->ncols_pad / c->pmax);
// (re)allocated at creation and when a later StepConfig needs more columns than allocated.
cudaError_t alloc_cap_buffers(Ctx* c) {
  void** old[] = {reinterpret_cast<void**>(&c->buf_cls), reinterpret_cast<void**>(&c->nxt),
                  reinterpret_cast<void**>(&c->jv), &c->wh,
                  reinterpret_cast<void**>(&c->wnorm), reinterpret_cast<void**>(&c->lrow),
                  &c->part_s, reinterpret_cast<void**>(&c->dbgz), &c->G,
                  reinterpret_cast<void**>(&c->poscorr), reinterpret_cast<void**>(&c->pslot),
                  reinterpret_cast<void**>(&c->dwt)};
  for (void** p : old) {
    dfree(c, *p);
    *p = nullptr;
  }
  const size_t ob = c->bf16 ? 2 : 4;  // operand bytes
  const size_t sb = c->umma ? 4 : 8;  // statistics bytes
  const int64_t B = c->maxB;
  const int64_t n1 = std::max<int64_t>(c->ncols, 1);
  const int BN = c->umma ? kBN : kSimtBN;
  // (narrow logits tiles, logits_narrow, need the finer slice count)
  const int64_t Tf = c->umma ? ceil_div(n1, kNarrowBN) * kFwdNWG : ceil_div(n1, BN);
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  A(dalloc(c, &c->buf_cls, (size_t)n1));
  A(dalloc(c, &c->nxt, (size_t)n1));
  A(dalloc(c, &c->jv, (size_t)n1));
  A(dalloc(c, reinterpret_cast<uint8_t**>(&c->wh), (size_t)c->ncols_pad * c->Dp * ob));
  A(dalloc(c, &c->wnorm, (size_t)c->ncols_pad));
  A(dalloc(c, &c->lrow, (size_t)c->ncols_pad));
  A(dalloc(c, reinterpret_cast<uint8_t**>(&c->part_s), (size_t)(Tf * B) * sb));
  if (c->d.flags & PFC_FLAG_DEBUG_LOGITS) A(dalloc(c, &c->dbgz, (size_t)B * n1));
  A(dalloc(c, reinterpret_cast<uint8_t**>(&c->G), (size_t)c->ncols_pad * c->ldg * ob));
  A(dalloc(c, &c->poscorr, (size_t)(c->nk * c->pmax * c->D)));
  A(dalloc(c, &c->pslot, (size_t)n1));
  if (!c->umma) A(dalloc(c, &c->dwt, (size_t)n1 * c->D));
  c->cap_alloc = c->cap;
  return e;
}

void drop_graphs(Ctx* c) {
  for (Ctx::GraphSlot& G : c->gs) {
    if (G.gexec) cudaGraphExecDestroy(G.gexec);
    if (G.graph) cudaGraphDestroy(G.graph);
    G = Ctx::GraphSlot{};
  }
  c->tm_B = -1;  // tensor maps over the column buffers are re-encoded
}

int validate_desc(const pfc_gpu_desc* d) {
  if (!d) return fail(nullptr, PFC_ERR_CONTRACT, "pfc_gpu_create: null descriptor");
  if (d->num_classes < 1 || d->num_shards < 1)
    return fail(nullptr, PFC_ERR_CONTRACT, "ShardLayout: need at least one class and one shard");
  if (!(d->r > 0.0 && d->r <= 1.0))
    return fail(nullptr, PFC_ERR_CONTRACT, "buffer_capacity: sampling ratio must lie in (0, 1]");
  if (!(d->margin_scale > 0.0))
    return fail(nullptr, PFC_ERR_CONFIG, "margin: scale must be positive");
  if (d->margin_m < 0.0 || d->margin_m >= 1.0)
    return fail(nullptr, PFC_ERR_CONFIG, "margin: m must be in [0, 1)");
  if (d->margin_kind == PFC_MARGIN_PLAIN && (d->margin_scale != 1.0 || d->margin_m != 0.0))
    return fail(nullptr, PFC_ERR_CONFIG, "margin: plain kind requires s=1, m=0");
  if (d->margin_kind < 0 || d->margin_kind > 3)
    return fail(nullptr, PFC_ERR_CONTRACT, "apply_margin: unknown kind");
  if (d->margin_kind == PFC_MARGIN_COMBINED) {  // extension (pfc_gpu.h)
    if (!(d->margin_m1 > 0.0 && d->margin_m1 <= 2.0))
      return fail(nullptr, PFC_ERR_CONFIG, "margin: m1 must be in (0, 2]");
    if (!(d->margin_m3 >= 0.0 && d->margin_m3 < 1.0))
      return fail(nullptr, PFC_ERR_CONFIG, "margin: m3 must be in [0, 1)");
  }
  if (d->dim < 1) return fail(nullptr, PFC_ERR_SHAPE, "pfc_gpu_create: dim must be >= 1");
  if (d->max_batch < 1 || d->max_batch > kMaxBatch)
    return fail(nullptr, PFC_ERR_CONTRACT, "pfc_gpu_create: max_batch must be in [1, %d]",
                kMaxBatch);
  if (d->world_size < 1 || d->rank < 0 || d->rank >= d->world_size ||
      d->num_shards % d->world_size != 0)
    return fail(nullptr, PFC_ERR_CONTRACT,
                "pfc_gpu_create: world_size must divide num_shards and 0 <= rank < world_size");
  if (d->num_shards / d->world_size > kMaxSamplerLocalShards)
    return fail(nullptr, PFC_ERR_CONTRACT,
                "pfc_gpu_create: at most %d reference shards per rank (num_shards / world_size)",
                kMaxSamplerLocalShards);
  if (d->precision < PFC_PRECISION_BF16 || d->precision > PFC_PRECISION_TF32)
    return fail(nullptr, PFC_ERR_CONFIG, "pfc_gpu_create: unknown precision %d", d->precision);
  if (d->precision != PFC_PRECISION_FP32 && (d->dim % 4 != 0 || d->dim > 1024))
    return fail(nullptr, PFC_ERR_CONFIG,
                "pfc_gpu: the tcgen05 paths (bf16, tf32) need dim %% 4 == 0 and dim <= 1024 "
                "(use PFC_PRECISION_FP32 otherwise)");
  if (d->num_classes >= (int64_t)INT32_MAX)
    return fail(nullptr, PFC_ERR_CONTRACT, "pfc_gpu_create: num_classes must be < 2^31");
  return PFC_OK;
}

}  // namespace
}  // namespace pfc

using namespace pfc;

__global__ void diag_fill_kernel(uint32_t* rmax, unsigned long long* emax, int* hasc, int n3,
                                 int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n3) {
    rmax[i] = pfc::enc_f32(-INFINITY);
    emax[i] = pfc::enc_f64(-INFINITY);
  }
  if (i < n) hasc[i] = 0;
}

int diag_alloc(Ctx* c) {
  if (c->dwall) return PFC_OK;  // w^ of every local class + per-row scratch, kept across calls
  c->diag_rows_pad = round_up(std::max<int64_t>(c->rows, 1), 256);
  const size_t ob = c->bf16 ? 2 : 4;
  CUDA_TRY(c, dalloc(c, reinterpret_cast<uint8_t**>(&c->dwall), (size_t)c->diag_rows_pad * c->Dp * ob));
  CUDA_TRY(c, dalloc(c, &c->dwinv, (size_t)c->diag_rows_pad));
  CUDA_TRY(c, dalloc(c, &c->dxinv, (size_t)c->maxB));
  CUDA_TRY(c, dalloc(c, &c->dapcs, (size_t)c->maxB));
  CUDA_TRY(c, dalloc(c, &c->drmax, (size_t)c->maxB * 3));
  CUDA_TRY(c, dalloc(c, &c->demax, (size_t)c->maxB * 3));
  CUDA_TRY(c, dalloc(c, &c->dhasc, (size_t)c->maxB));
  CUDA_TRY(c, dalloc(c, &c->dcid, (size_t)std::max<int64_t>(c->rows, 1)));
  CUDA_TRY(c, dalloc(c, &c->dsid, (size_t)c->maxB));
  c->dcand_cap = (int64_t)1 << 22;  // 4M candidates (64 MB)
  CUDA_TRY(c, dalloc(c, &c->dcand, (size_t)c->dcand_cap));
  CUDA_TRY(c, dalloc(c, &c->dncand, (size_t)1));
  if (c->bf16 && !make_map(&c->tm_wall, c->dwall, c->Dp, c->rows, c->Dp, kBN / kDiagCG))
    return fail(c, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return PFC_OK;
}

// mics over rows [r0, r0 + nr) of the local classes against all of them (one screening launch
// + exact pass); per-row maxima in emax[3 * r] (bucket 0)
template <typename OT, bool kUmma>
int run_mics_block(Ctx* c, int64_t r0, int64_t nr, uint32_t* rmax, unsigned long long* emax,
                   int* hasc) {
  cudaStream_t s = c->stream;
  OT* wall = static_cast<OT*>(c->dwall);
  DiagMaxEpi e{};
  e.B = (int)nr;
  e.rows = c->rows;
  e.cls_lo = c->cls_lo;
  e.labels = nullptr;
  e.row_base = r0;
  e.cid = nullptr;
  e.sid = nullptr;
  e.rmax = rmax;
  e.hasc = hasc;
  e.cand = c->dcand;
  e.ncand = c->dncand;
  e.cap = (unsigned long long)c->dcand_cap;
  for (int pass = 0; pass < 2; ++pass) {
    CUDA_TRY(c, cudaMemsetAsync(c->dncand, 0, sizeof(unsigned long long), s));
    cudaError_t err;
    if constexpr (kUmma) {
      CUtensorMap ta;
      if (!make_map(&ta, wall + (size_t)r0 * c->Dp, c->Dp, nr, c->Dp, 128))
        return fail(c, PFC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
      // n fastest: all CTAs sweep the columns of the same 128 rows together, so the running
      // maxima converge within the first wave and later tiles yield few candidates
      const GemmGeom g = make_geom((int)nr, (int)c->rows, (int)c->Dp, kBN, 1, 1, 128 * kDiagCG);
      err = launch_umma<kBN, 4, 2, false, false, DiagMaxEpi, kDiagCG>(c, ta, c->tm_wall, g, e);
    } else {
      const GemmGeom g = make_geom((int)nr, (int)c->rows, (int)c->Dp, kSimtBN, 1, 1);
      err = launch_simt<false, false>(c, (const float*)(wall + (size_t)r0 * c->Dp), (int)c->Dp,
                                      (const float*)wall, (int)c->Dp, g, e);
    }
    CUDA_TRY(c, err);
    unsigned long long n = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&n, c->dncand, sizeof(n), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    if (n <= (unsigned long long)c->dcand_cap) break;
    if (pass == 1) return fail(c, PFC_ERR_CUDA, "pfc_gpu_mics: candidate list overflow");
  }
  // rows of this block are the "samples": X = the W rows, xinv = their 1/|w|
  diag_exact_kernel<<<(unsigned)(c->num_sms * 8), 256, 0, s>>>(
      c->dcand, c->dncand, (unsigned long long)c->dcand_cap, rmax, c->W + (size_t)r0 * c->D,
      c->dwinv + r0, c->W, c->dwinv, (int)c->D, emax);
  CUDA_TRY(c, cudaGetLastError());
  return PFC_OK;
}

template <typename OT, bool kUmma>
int run_diagnostics(Ctx* c, int64_t B, bool split) {
  cudaStream_t s = c->stream;
  const int bs = 256;
  OT* xh = static_cast<OT*>(c->xh);
  OT* wall = static_cast<OT*>(c->dwall);
  diag_norm_x_kernel<OT><<<(unsigned)ceil_div(B * 32, bs), bs, 0, s>>>(c->X, (int)B, (int)c->D,
                                                                       (int)c->Dp, xh, c->dxinv);
  diag_norm_w_kernel<OT><<<(unsigned)ceil_div(c->diag_rows_pad * 32, bs), bs, 0, s>>>(
      c->W, c->rows, c->diag_rows_pad, (int)c->D, (int)c->Dp, wall, c->dwinv);
  diag_fill_kernel<<<(unsigned)ceil_div(B * 3, bs), bs, 0, s>>>(c->drmax, c->demax, c->dhasc,
                                                                (int)(B * 3), (int)B);
  CUDA_TRY(c, cudaGetLastError());
  DiagMaxEpi e{};
  e.B = (int)B;
  e.rows = c->rows;
  e.cls_lo = c->cls_lo;
  e.labels = c->labels;
  e.cid = split ? c->dcid : nullptr;
  e.sid = split ? c->dsid : nullptr;
  e.rmax = c->drmax;
  e.hasc = c->dhasc;
  e.cand = c->dcand;
  e.ncand = c->dncand;
  e.cap = (unsigned long long)c->dcand_cap;
  // screening GEMM; if the candidate list overflowed (running maxima still low early on), screen
  // again from the final maxima, which keeps only near-maximal classes
  for (int pass = 0; pass < 2; ++pass) {
    CUDA_TRY(c, cudaMemsetAsync(c->dncand, 0, sizeof(unsigned long long), s));
    cudaError_t err;
    if constexpr (kUmma) {
      if (int rc = ensure_maps(c, B)) return rc;
      const GemmGeom g = make_geom((int)B, (int)c->rows, (int)c->Dp, kBN, 1, 0, 128 * kDiagCG);
      err = launch_umma<kBN, 4, 2, false, false, DiagMaxEpi, kDiagCG>(c, c->tm_x_k, c->tm_wall, g, e);
    } else {
      const GemmGeom g = make_geom((int)B, (int)c->rows, (int)c->Dp, kSimtBN, 1, 0);
      err = launch_simt<false, false>(c, (const float*)xh, (int)c->Dp, (const float*)wall,
                                      (int)c->Dp, g, e);
    }
    CUDA_TRY(c, err);
    unsigned long long n = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&n, c->dncand, sizeof(n), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    if (n <= (unsigned long long)c->dcand_cap) break;
    if (pass == 1) return fail(c, PFC_ERR_CUDA, "pfc_gpu_diagnostics: candidate list overflow");
  }
  diag_exact_kernel<<<(unsigned)(c->num_sms * 8), 256, 0, s>>>(
      c->dcand, c->dncand, (unsigned long long)c->dcand_cap, c->drmax, c->X, c->dxinv, c->W,
      c->dwinv, (int)c->D, c->demax);
  CUDA_TRY(c, cudaGetLastError());
  diag_apcs_kernel<<<(unsigned)ceil_div(B * 32, bs), bs, 0, s>>>(c->X, c->dxinv, c->W, c->dwinv,
                                                           c->labels, (int)B, (int)c->D,
                                                           c->cls_lo, c->rows, c->dapcs);
  CUDA_TRY(c, cudaGetLastError());
  return PFC_OK;
}

extern "C" {

const char* pfc_gpu_version(void) { return "pfc_gpu 0.1 (sm_100a tcgen05)"; }

const char* pfc_gpu_last_error(const void* ctx) {
  if (!ctx) return g_create_error.c_str();
  return static_cast<const Ctx*>(ctx)->err.c_str();
}

int pfc_gpu_loopback_id(uint8_t out[128]) {
  loop_new_id(out);
  return PFC_OK;
}

int pfc_gpu_debug_logits(void* ctx, float* out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!c->dbgz)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_debug_logits: create with PFC_FLAG_DEBUG_LOGITS");
  CUDA_TRY(c, cudaMemcpyAsync(out, c->dbgz, sizeof(float) * c->lastB * c->ncols,
                              cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PFC_OK;
}

int pfc_gpu_nccl_unique_id(uint8_t out[128]) {
  std::string e;
  if (!g_nccl.load(e)) return fail(nullptr, PFC_ERR_NCCL, "%s", e.c_str());
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != 0) return fail(nullptr, PFC_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(out, id.internal, 128);
  return PFC_OK;
}

int pfc_gpu_create(const pfc_gpu_desc* desc, void** ctx_out) {
  if (int rc = validate_desc(desc)) return rc;
  Ctx* c = new Ctx();
  c->d = *desc;
  c->C = desc->num_classes;
  c->D = desc->dim;
  c->K = desc->num_shards;
  c->R = desc->world_size;
  c->coll = c->R > 1 || (desc->flags & PFC_FLAG_FORCE_COLLECTIVES);
  c->rank = desc->rank;
  c->bf16 = desc->precision == PFC_PRECISION_BF16;
  c->tf32 = desc->precision == PFC_PRECISION_TF32;
  c->umma = c->bf16 || c->tf32;
  c->Dp = round_up(c->D, 64);
  c->blk = ceil_div(c->C, c->K);
  c->cap = capacity_for(c->C, c->K, desc->r);
  c->nk = c->K / c->R;
  c->k0 = (int64_t)c->rank * c->nk;
  c->cls_lo = std::min(c->k0 * c->blk, c->C);
  c->cls_hi = std::min((c->k0 + c->nk) * c->blk, c->C);
  c->rows = c->cls_hi - c->cls_lo;
  c->ldg = round_up(desc->max_batch, 8);  // E^T row stride
  c->pool_stride = std::max<int64_t>(c->blk, 1);
  c->maxB = desc->max_batch;
  set_cap_geometry(c);
  set_margin_state(c);
  c->pdl = !(desc->flags & PFC_FLAG_NO_PDL);
  int64_t B = c->maxB;
  auto bail = [&](int rc) {
    g_create_error = c->err;
    pfc_gpu_destroy(c);
    return rc;
  };
#define CT(expr)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return bail(fail(c, PFC_ERR_CUDA, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), \
                       __FILE__, __LINE__, cudaGetErrorString(e_)));                     \
  } while (0)
  CT(cudaSetDevice(desc->device));
  {
    int major = 0, minor = 0;
    CT(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, desc->device));
    CT(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, desc->device));
    if (major != 10 || minor != 0)
      return bail(fail(c, PFC_ERR_CUDA, "pfc_gpu requires an sm_100 (B200) device, got sm_%d%d",
                       major, minor));
    CT(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, desc->device));
  }
  CT(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CT(cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking));
  CT(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CT(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&c->ev_s, &c->ev_x, &c->ev_dx, &c->ev_out})
    CT(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  const size_t ob = c->bf16 ? 2 : 4;  // operand bytes
  const size_t sb = c->umma ? 4 : 8;  // statistics bytes
  c->max_splits = c->umma ? 32 : 64;
  CT(dalloc(c, &c->W, (size_t)std::max<int64_t>(c->rows, 1) * c->D));
  CT(dalloc(c, &c->M, (size_t)std::max<int64_t>(c->rows, 1) * c->D));
  CT(dalloc(c, &c->labels, (size_t)B));
  c->nwords = c->C / 32 + 1;  // covers bit C itself: bits_below(C) is the total count
  if (c->d.flags & PFC_FLAG_WIDE_SAMPLER_CHUNKS) c->chunk_words = 1024;
  while (ceil_div(c->nwords, c->chunk_words) > kMaxSamplerChunks) c->chunk_words *= 2;
  c->nchunk = (int)ceil_div(c->nwords, c->chunk_words);
  CT(dalloc(c, &c->labs, (size_t)B));
  CT(dalloc(c, &c->bits, (size_t)c->nwords));
  CT(dalloc(c, &c->ccnt, (size_t)c->nchunk));
  CT(dalloc(c, &c->rej, (size_t)c->nk));
  CT(dalloc(c, &c->oobs, 2));
  {
    const long long none[2] = {LLONG_MAX, LLONG_MAX};
    CT(cudaMemcpy(c->oobs, none, sizeof none, cudaMemcpyHostToDevice));
  }
  CT(dalloc(c, &c->meta, (size_t)c->nk));
  CT(dalloc(c, &c->pos_col, (size_t)B));
  CT(dalloc(c, &c->head, (size_t)(c->nk * c->pool_stride)));
  CT(cudaMemset(c->head, 0xFF, sizeof(int32_t) * c->nk * c->pool_stride));  // reset per draw after
  CT(dalloc(c, &c->pool_scratch, (size_t)(c->nk * c->pool_stride)));
  CT(dalloc(c, &c->X, (size_t)B * c->D));
  CT(dalloc(c, &c->xnorm, (size_t)B));
  CT(dalloc(c, reinterpret_cast<uint8_t**>(&c->xh), (size_t)B * c->Dp * ob));
  CT(dalloc(c, reinterpret_cast<uint8_t**>(&c->ls), (size_t)(c->R * B) * sb));
  CT(dalloc(c, reinterpret_cast<uint8_t**>(&c->rowscale), (size_t)B * sb));
  CT(dalloc(c, reinterpret_cast<uint8_t**>(&c->delta), (size_t)B * sb));
  CT(dalloc(c, &c->zpos, (size_t)B));
  CT(dalloc(c, &c->cpos, (size_t)B));
  CT(dalloc(c, &c->epos, (size_t)B));
  CT(dalloc(c, &c->hasval, (size_t)B));
  CT(dalloc(c, &c->loss_row, (size_t)B));
  CT(dalloc(c, &c->offr, (size_t)B));
  CT(dalloc(c, reinterpret_cast<uint8_t**>(&c->xs), (size_t)B * c->Dp * ob));
  CT(alloc_cap_buffers(c));
  CT(dalloc(c, &c->dx_part, (size_t)c->max_splits * B * c->D));
  CT(dalloc(c, &c->dX, (size_t)B * c->D));
  CT(dalloc(c, &c->xdb, (size_t)B * c->D));
  CT(dalloc(c, &c->st, 1));
  CT(dalloc(c, &c->sp, 1));
  CT(cudaMallocHost(&c->st_host, sizeof(StepStatus)));
  for (int i = 0; i <= PhaseTimer::kMax; ++i) CT(cudaEventCreate(&c->pt.ev[i]));
  if (c->coll) {
    if (!desc->nccl_id) return bail(fail(c, PFC_ERR_NCCL, "world_size > 1 needs nccl_id"));
    std::string e;
    if (is_loop_id(desc->nccl_id)) {  // R ranks as R contexts of this process (comm.cuh)
      std::memcpy(c->loop_id, desc->nccl_id, 128);
      const size_t scratch = (size_t)B * (size_t)std::max<int64_t>(c->D * 4, 3 * 8);
      c->loop = loop_join(c->loop_id, c->R, c->rank, desc->device, scratch, e);
      if (!c->loop) return bail(fail(c, PFC_ERR_NCCL, "%s", e.c_str()));
    } else {
      if (!g_nccl.load(e)) return bail(fail(c, PFC_ERR_NCCL, "%s", e.c_str()));
      ncclUniqueId id;
      std::memcpy(id.internal, desc->nccl_id, 128);
      const int r = g_nccl.CommInitRank(&c->comm, c->R, id, c->rank);
      if (r != 0) return bail(fail(c, PFC_ERR_NCCL, "ncclCommInitRank failed (%d)", r));
    }
    // one collective outside any graph capture: NCCL may set up its connections lazily at the
    // first collective, which the step's captured graph must not be the one to trigger
    if (comm_all_reduce(c, c->st, c->st, 1, kI32, kMax, c->stream) != PFC_OK)
      return bail(fail(c, PFC_ERR_NCCL, "warm-up all-reduce failed: %s", c->err.c_str()));
    c->step_nccl_bytes = c->step_wire_bytes = 0;
  }
  CT(cudaStreamSynchronize(c->stream));
#undef CT
  *ctx_out = c;
  return PFC_OK;
}

int pfc_gpu_destroy(void* ctx) {
  if (!ctx) return PFC_OK;
  Ctx* c = static_cast<Ctx*>(ctx);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graphs(c);
  for (cudaEvent_t e : {c->ev_s, c->ev_x, c->ev_dx, c->ev_out})
    if (e) cudaEventDestroy(e);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->loop) loop_leave(c->loop, c->loop_id, c->rank);
  for (void* p : c->allocs) cudaFree(p);
  if (c->st_host) cudaFreeHost(c->st_host);
  for (int i = 0; i <= PhaseTimer::kMax; ++i)
    if (c->pt.ev[i]) cudaEventDestroy(c->pt.ev[i]);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->s2) cudaStreamDestroy(c->s2);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
  return PFC_OK;
}

int64_t pfc_gpu_capacity(const void* ctx) { return static_cast<const Ctx*>(ctx)->cap; }

int pfc_gpu_set_step_config(void* ctx, const pfc_gpu_step_config* sc) {
  Ctx* c = static_cast<Ctx*>(ctx);
  pfc_gpu_desc d = c->d;
  d.r = sc->r;
  d.margin_kind = sc->margin_kind;
  d.margin_scale = sc->margin_scale;
  d.margin_m = sc->margin_m;
  d.margin_m1 = sc->margin_m1;
  d.margin_m3 = sc->margin_m3;
  d.has_filter = sc->has_filter ? 1 : 0;
  d.filter_threshold = sc->has_filter ? sc->filter_threshold : 0.0;
  d.momentum = sc->momentum;
  d.weight_decay = sc->weight_decay;
  if (int rc = validate_desc(&d)) return fail(c, rc, "%s", g_create_error.c_str());
  const pfc_gpu_desc& o = c->d;
  if (d.r == o.r && d.margin_kind == o.margin_kind && d.margin_scale == o.margin_scale &&
      d.margin_m == o.margin_m && d.margin_m1 == o.margin_m1 && d.margin_m3 == o.margin_m3 &&
      d.has_filter == o.has_filter &&
      d.filter_threshold == o.filter_threshold && d.momentum == o.momentum &&
      d.weight_decay == o.weight_decay)
    return PFC_OK;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));  // no step in flight uses the old state
  CUDA_TRY(c, cudaStreamSynchronize(c->s2));
  c->d = d;
  set_margin_state(c);
  const int64_t cap = capacity_for(c->C, c->K, d.r);
  if (cap != c->cap) {
    c->cap = cap;
    set_cap_geometry(c);
    if (cap > c->cap_alloc) CUDA_TRY(c, alloc_cap_buffers(c));
  }
  drop_graphs(c);  // the captured epilogue parameters and column geometry are stale
  return PFC_OK;
}

int pfc_gpu_local_shards(const void* ctx, int64_t* first, int64_t* n) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  *first = c->k0;
  *n = c->nk;
  return PFC_OK;
}

int pfc_gpu_shard_range(const void* ctx, int64_t k, int64_t* b, int64_t* e) {
  const Ctx* c = static_cast<const Ctx*>(ctx);
  *b = std::min(k * c->blk, c->C);
  *e = std::min((k + 1) * c->blk, c->C);
  return PFC_OK;
}

static int shard_local(Ctx* c, int64_t k, int64_t* row0, int64_t* n) {
  if (k < c->k0 || k >= c->k0 + c->nk)
    return fail(c, PFC_ERR_CONTRACT, "shard %lld is not local to rank %d", (long long)k, c->rank);
  const int64_t lo = std::min(k * c->blk, c->C), hi = std::min((k + 1) * c->blk, c->C);
  *row0 = lo - c->cls_lo;
  *n = hi - lo;
  return PFC_OK;
}

// D x owned fp64 (CenterShard layout) <-> rows fp32, staged through a bounded scratch.
static int shard_io(Ctx* c, int64_t k, double* wbuf, double* mbuf, bool in) {
  int64_t row0, n;
  if (int rc = shard_local(c, k, &row0, &n)) return rc;
  if (n == 0) return PFC_OK;
  const int64_t chunk = std::max<int64_t>(1, (int64_t)(64ll << 20) / (8 * c->D));  // 64 MB
  double* scratch = nullptr;
  CUDA_TRY(c, cudaMalloc(&scratch, (size_t)std::min(chunk, n) * c->D * sizeof(double)));
  for (int which = 0; which < 2; ++which) {
    double* hb = which == 0 ? wbuf : mbuf;
    float* dev = which == 0 ? c->W : c->M;
    if (!hb) {
      if (in && which == 1) {
        CUDA_TRY(c, cudaMemsetAsync(dev + row0 * c->D, 0, sizeof(float) * n * c->D, c->stream));
      }
      continue;
    }
    for (int64_t j0 = 0; j0 < n; j0 += chunk) {
      const int64_t m = std::min(chunk, n - j0);
      dim3 grid((unsigned)ceil_div(m, 32), (unsigned)ceil_div(c->D, 32)), blk(32, 8);
      if (in) {
        CUDA_TRY(c, cudaMemcpy2DAsync(scratch, m * sizeof(double), hb + j0, n * sizeof(double),
                                      m * sizeof(double), c->D, cudaMemcpyHostToDevice, c->stream));
        shard_in_kernel<<<grid, blk, 0, c->stream>>>(scratch, (int)c->D, (int)m, row0 + j0, dev);
      } else {
        shard_out_kernel<<<grid, blk, 0, c->stream>>>(dev, (int)c->D, (int)m, row0 + j0, scratch);
        CUDA_TRY(c, cudaMemcpy2DAsync(hb + j0, n * sizeof(double), scratch, m * sizeof(double),
                                      m * sizeof(double), c->D, cudaMemcpyDeviceToHost, c->stream));
      }
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
  }
  cudaFree(scratch);
  return PFC_OK;
}

// ---- checkpoint streams (trainer.hpp:235-338 shard section, io.hpp:18-91 encoding) ---------
// One matrix (int64 rows = D, int64 cols = n, then D x n fp64 row-major) moved in dim-row chunks:
// chunk [d0, d0 + dn) is a contiguous span of the file.
static int ckpt_matrix(Ctx* c, FILE* f, float* dev, int64_t row0, int64_t n, bool write,
                       double* dstage, double* hstage, int64_t stage_elems) {
  const int64_t D = c->D;
  if (write) {
    const int64_t hdr[2] = {D, n};
    if (fwrite(hdr, sizeof(int64_t), 2, f) != 2) return fail(c, PFC_ERR_IO, "write failed");
  } else {
    int64_t hdr[2];
    if (fread(hdr, sizeof(int64_t), 2, f) != 2) return fail(c, PFC_ERR_IO, "truncated checkpoint");
    // the reference caps rows * cols at 2^32 (io.hpp:78); the device reader does not
    if (hdr[0] != D || hdr[1] != n)
      return fail(c, PFC_ERR_IO, "checkpoint matrix %lldx%lld does not match the shard (%lldx%lld)",
                  (long long)hdr[0], (long long)hdr[1], (long long)D, (long long)n);
  }
  if (n == 0) return PFC_OK;
  const int64_t dn = std::max<int64_t>(1, std::min<int64_t>(D, stage_elems / n));
  for (int64_t d0 = 0; d0 < D; d0 += dn) {
    const int64_t m = std::min(dn, D - d0);
    dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(m, 32)), blk(32, 8);
    if (write) {
      dims_out_kernel<<<grid, blk, 0, c->stream>>>(dev, (int)D, (int)n, row0, (int)d0, (int)m, dstage);
      CUDA_TRY(c, cudaMemcpyAsync(hstage, dstage, sizeof(double) * m * n, cudaMemcpyDeviceToHost,
                                  c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      if (fwrite(hstage, sizeof(double), (size_t)(m * n), f) != (size_t)(m * n))
        return fail(c, PFC_ERR_IO, "write failed");
    } else {
      if (fread(hstage, sizeof(double), (size_t)(m * n), f) != (size_t)(m * n))
        return fail(c, PFC_ERR_IO, "truncated checkpoint");
      CUDA_TRY(c, cudaMemcpyAsync(dstage, hstage, sizeof(double) * m * n, cudaMemcpyHostToDevice,
                                  c->stream));
      dims_in_kernel<<<grid, blk, 0, c->stream>>>(dstage, (int)D, (int)n, row0, (int)d0, (int)m, dev);
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
  }
  return PFC_OK;
}

static int ckpt_shards(Ctx* c, const char* path, int64_t offset, int mode, int64_t* end_offset) {
  // mode 0: write (truncate), 1: write (append), 2: read at offset
  const bool write = mode != 2;
  FILE* f = fopen(path, mode == 0 ? "wb" : (mode == 1 ? "ab" : "rb"));
  if (!f) return fail(c, PFC_ERR_IO, write ? "cannot open for writing: %s" : "cannot open: %s", path);
  const int64_t stage_elems = (int64_t)(32ll << 20) / 8;  // 32 MB staging
  double *dstage = nullptr, *hstage = nullptr;
  int rc = PFC_OK;
  auto done = [&](int r) {
    if (dstage) cudaFree(dstage);
    if (hstage) cudaFreeHost(hstage);
    fclose(f);
    return r;
  };
  if (cudaMalloc(&dstage, sizeof(double) * stage_elems) != cudaSuccess ||
      cudaMallocHost(&hstage, sizeof(double) * stage_elems) != cudaSuccess)
    return done(fail(c, PFC_ERR_CUDA, "checkpoint staging allocation failed"));
  if (write) {
    const int64_t count = c->nk;
    if (fwrite(&count, sizeof(int64_t), 1, f) != 1) return done(fail(c, PFC_ERR_IO, "write failed"));
    for (int64_t kk = 0; kk < c->nk; ++kk) {
      const int64_t k = c->k0 + kk;
      const int64_t lo = std::min(k * c->blk, c->C), hi = std::min((k + 1) * c->blk, c->C);
      const int64_t hdr[3] = {k, lo, hi};
      if (fwrite(hdr, sizeof(int64_t), 3, f) != 3) return done(fail(c, PFC_ERR_IO, "write failed"));
      for (float* dev : {c->W, c->M})
        if ((rc = ckpt_matrix(c, f, dev, lo - c->cls_lo, hi - lo, true, dstage, hstage, stage_elems)))
          return done(rc);
    }
  } else {
    if (fseeko(f, (off_t)offset, SEEK_SET) != 0) return done(fail(c, PFC_ERR_IO, "truncated checkpoint"));
    int64_t count = 0;
    if (fread(&count, sizeof(int64_t), 1, f) != 1) return done(fail(c, PFC_ERR_IO, "truncated checkpoint"));
    for (int64_t i = 0; i < count; ++i) {
      int64_t hdr[3];
      if (fread(hdr, sizeof(int64_t), 3, f) != 3) return done(fail(c, PFC_ERR_IO, "truncated checkpoint"));
      const int64_t k = hdr[0], lo = hdr[1], hi = hdr[2];
      if (k < 0 || k >= c->K || lo != std::min(k * c->blk, c->C) || hi != std::min((k + 1) * c->blk, c->C))
        return done(fail(c, PFC_ERR_CONTRACT,
                         "checkpoint shard %lld [%lld, %lld) does not match the contiguous equal "
                         "partition", (long long)k, (long long)lo, (long long)hi));
      const bool local = k >= c->k0 && k < c->k0 + c->nk;
      for (float* dev : {c->W, c->M}) {
        if (local) {
          if ((rc = ckpt_matrix(c, f, dev, lo - c->cls_lo, hi - lo, false, dstage, hstage, stage_elems)))
            return done(rc);
        } else {  // another rank's shard: skip its matrix
          int64_t mh[2];
          if (fread(mh, sizeof(int64_t), 2, f) != 2 ||
              fseeko(f, (off_t)(mh[0] * mh[1] * (int64_t)sizeof(double)), SEEK_CUR) != 0)
            return done(fail(c, PFC_ERR_IO, "truncated checkpoint"));
        }
      }
    }
  }
  if (end_offset) *end_offset = (int64_t)ftello(f);
  if (write && fflush(f) != 0) return done(fail(c, PFC_ERR_IO, "write failed"));
  return done(PFC_OK);
}

int pfc_gpu_mics(void* ctx, double* out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (c->C < 2) return fail(c, PFC_ERR_CONTRACT, "mics: needs at least two classes");
  if (c->R > 1) return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_mics: single-rank contexts only");
  if (int rc = diag_alloc(c)) return rc;
  cudaStream_t s = c->stream;
  const int bs = 256;
  // w^ of every class (bf16 operand rows + fp64 1/|w|)
  if (c->bf16)
    diag_norm_w_kernel<__nv_bfloat16><<<(unsigned)ceil_div(c->diag_rows_pad * 32, bs), bs, 0, s>>>(
        c->W, c->rows, c->diag_rows_pad, (int)c->D, (int)c->Dp, static_cast<__nv_bfloat16*>(c->dwall),
        c->dwinv);
  else
    diag_norm_w_kernel<float><<<(unsigned)ceil_div(c->diag_rows_pad * 32, bs), bs, 0, s>>>(
        c->W, c->rows, c->diag_rows_pad, (int)c->D, (int)c->Dp, static_cast<float*>(c->dwall), c->dwinv);
  CUDA_TRY(c, cudaGetLastError());
  const int64_t blk = std::min<int64_t>(c->rows, 1 << 17);  // rows per screening launch
  uint32_t* rmax = nullptr;
  unsigned long long* emax = nullptr;
  int* hasc = nullptr;
  CUDA_TRY(c, cudaMalloc(&rmax, sizeof(uint32_t) * blk * 3));
  CUDA_TRY(c, cudaMalloc(&emax, sizeof(unsigned long long) * blk * 3));
  CUDA_TRY(c, cudaMalloc(&hasc, sizeof(int) * blk));
  std::vector<unsigned long long> em((size_t)blk * 3);
  int rc = PFC_OK;
  for (int64_t r0 = 0; r0 < c->rows && rc == PFC_OK; r0 += blk) {
    const int64_t nr = std::min(blk, c->rows - r0);
    diag_fill_kernel<<<(unsigned)ceil_div(nr * 3, bs), bs, 0, s>>>(rmax, emax, hasc, (int)(nr * 3), (int)nr);
    rc = c->bf16 ? run_mics_block<__nv_bfloat16, true>(c, r0, nr, rmax, emax, hasc)
                 : run_mics_block<float, false>(c, r0, nr, rmax, emax, hasc);
    if (rc) break;
    // on the context stream: the legacy default stream does not wait for a non-blocking stream
    if (cudaMemcpyAsync(em.data(), emax, sizeof(unsigned long long) * nr * 3, cudaMemcpyDeviceToHost,
                        s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
      rc = fail(c, PFC_ERR_CUDA, "pfc_gpu_mics: copy failed");
      break;
    }
    for (int64_t r = 0; r < nr; ++r) out[c->cls_lo + r0 + r] = dec_f64(em[(size_t)r * 3]);
  }
  cudaFree(rmax);
  cudaFree(emax);
  cudaFree(hasc);
  return rc;
}

int pfc_gpu_write_shards(void* ctx, const char* path, int append) {
  return ckpt_shards(static_cast<Ctx*>(ctx), path, 0, append ? 1 : 0, nullptr);
}

int pfc_gpu_read_shards(void* ctx, const char* path, int64_t offset, int64_t* end_offset) {
  return ckpt_shards(static_cast<Ctx*>(ctx), path, offset, 2, end_offset);
}

int pfc_gpu_set_shard(void* ctx, int64_t k, const double* w, const double* m) {
  return shard_io(static_cast<Ctx*>(ctx), k, const_cast<double*>(w), const_cast<double*>(m), true);
}

int pfc_gpu_get_shard(void* ctx, int64_t k, double* w, double* m) {
  return shard_io(static_cast<Ctx*>(ctx), k, w, m, false);
}

int pfc_gpu_init_shards(void* ctx, uint64_t seed) {
  Ctx* c = static_cast<Ctx*>(ctx);
  uint64_t h = 0xcbf29ce484222325ULL;  // fnv1a("center-init") (rng.hpp:26-32)
  for (const char* p = "center-init"; *p; ++p) {
    h ^= (unsigned char)*p;
    h *= 0x100000001b3ULL;
  }
  if (c->rows > 0) {
    init_centers_kernel<<<(unsigned)ceil_div(c->rows * 32, 256), 256, 0, c->stream>>>(
        c->W, c->M, c->rows, (int)c->D, c->cls_lo, seed, h);
    CUDA_TRY(c, cudaGetLastError());
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return PFC_OK;
}

int pfc_gpu_device_state(void* ctx, float** w, float** m, int64_t* rows) {
  Ctx* c = static_cast<Ctx*>(ctx);
  *w = c->W;
  *m = c->M;
  *rows = c->rows;
  return PFC_OK;
}

void* pfc_gpu_stream(void* ctx) { return static_cast<Ctx*>(ctx)->stream; }

// the device-side address of page-locked host memory (the same address under UVA)
static const int64_t* dev_view(const int64_t* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess || !at.devicePointer) {
    cudaGetLastError();
    return h;
  }
  return static_cast<const int64_t*>(at.devicePointer);
}

// page-locked (or registered) host memory: eligible for copies inside the captured step
static bool pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// The step on a FeatureBatch already on the device: D x B fp64 features in c->xdb, labels in
// c->labels.  Leaves the summed D x B fp64 d_features in c->xdb; synchronous.
static int step_from_X(Ctx* c, int64_t B, const pfc_gpu_step_args* a, pfc_gpu_step_out* out) {
  cudaStream_t s = c->stream;
  dim3 grid((unsigned)ceil_div(B, 32), (unsigned)ceil_div(c->D, 32)), blk(32, 8);
  if (int rc = run_step(c, c->X, c->labels, B, a, c->dX)) return rc;
  c->reset_status = true;
  if (c->coll) {  // the drop-in returns the FULL summed d_features on every rank
    COMM_TRY(comm_all_reduce(c, c->dX, c->dX, B * c->D, kF32, kSum, s));
  }
  dx_to_dxb_kernel<<<grid, blk, 0, s>>>(c->dX, (int)c->D, (int)B, c->xdb);
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaMemcpyAsync(c->st_host, c->st, sizeof(StepStatus), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  if (int rc = finish_phase_timing(c)) return rc;
  return check_status(c, a->step_index, B, out);
}
static int step_from_xdb(Ctx* c, int64_t B, const pfc_gpu_step_args* a, pfc_gpu_step_out* out) {
  dim3 grid((unsigned)ceil_div(B, 32), (unsigned)ceil_div(c->D, 32)), blk(32, 8);
  x_from_dxb_kernel<<<grid, blk, 0, c->stream>>>(c->xdb, (int)c->D, (int)B, c->X);
  CUDA_TRY(c, cudaGetLastError());
  c->step_nccl_bytes = c->step_wire_bytes = 0;
  // the features stay in c->X (c->xdb receives d_features), so a rerun starts from there
  return with_exact_retry(c, [&] { return step_from_X(c, B, a, out); });
}

int pfc_gpu_step(void* ctx, const double* xdb, const int64_t* labels, int64_t B,
                 const pfc_gpu_step_args* a, double* dxdb, pfc_gpu_step_out* out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!(a->lr >= 0.0)) return fail(c, PFC_ERR_CONTRACT, "distributed_partial_step: lr must be >= 0");
  if (B < 0) return fail(c, PFC_ERR_SHAPE, "FeatureBatch: label count != feature columns");
  cudaStream_t s = c->stream;
  if (B > 0 && B <= c->maxB && pinned(xdb) && pinned(labels) && pinned(dxdb)) {
    // copies inside the step: X upload overlaps the sampler + gather, dX download the dW GEMM.
    // The host-side label / capacity check runs while the GPU works: the device sampler makes
    // the same checks and skips every update on failure, so launching first is safe.
    // On an error the contents of dxdb are unspecified (the reference throws instead).
    c->step_nccl_bytes = c->step_wire_bytes = 0;
    return with_exact_retry(c, [&]() -> int {
      c->e2e = {true, xdb, labels, dxdb};
      const int rc = run_step(c, c->X, dev_view(labels), B, a, c->dX);
      c->e2e.on = false;
      if (rc) return rc;
      c->reset_status = true;  // the status download is part of the step (run_pipeline)
      const int vrc = host_validate(c, labels, B);
      CUDA_TRY(c, cudaStreamSynchronize(s));
      if (int rc2 = finish_phase_timing(c)) return rc2;
      if (vrc) return vrc;
      return check_status(c, a->step_index, B, out);
    });
  }
  if (int rc = host_validate(c, labels, B)) return rc;
  if (B == 0)
    return fail(c, PFC_ERR_NUMERICAL, "distributed_partial_step: non-finite loss at step %lld",
                (long long)a->step_index);
  if (B > c->maxB)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu: batch %lld exceeds max_batch %lld", (long long)B,
                (long long)c->maxB);
  CUDA_TRY(c, cudaMemcpyAsync(c->xdb, xdb, sizeof(double) * B * c->D, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(c->labels, labels, sizeof(int64_t) * B, cudaMemcpyHostToDevice, s));
  if (int rc = step_from_xdb(c, B, a, out)) return rc;
  CUDA_TRY(c, cudaMemcpy(dxdb, c->xdb, sizeof(double) * B * c->D, cudaMemcpyDeviceToHost));
  return PFC_OK;
}

static int step_device_once(Ctx* c, const float* x_local, const int64_t* labels_local,
                            int64_t b_local, const pfc_gpu_step_args* a, float* dx_local,
                            pfc_gpu_step_out* out);

int pfc_gpu_step_device(void* ctx, const float* x_local, const int64_t* labels_local,
                        int64_t b_local, const pfc_gpu_step_args* a, float* dx_local,
                        pfc_gpu_step_out* out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!(a->lr >= 0.0)) return fail(c, PFC_ERR_CONTRACT, "distributed_partial_step: lr must be >= 0");
  const int64_t B = b_local * c->R;
  if (B < 1 || B > c->maxB)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu: global batch %lld outside [1, max_batch=%lld]",
                (long long)B, (long long)c->maxB);
  c->step_nccl_bytes = c->step_wire_bytes = 0;
  if (!out) return step_device_once(c, x_local, labels_local, b_local, a, dx_local, out);
  return with_exact_retry(
      c, [&] { return step_device_once(c, x_local, labels_local, b_local, a, dx_local, out); });
}

static int step_device_once(Ctx* c, const float* x_local, const int64_t* labels_local,
                            int64_t b_local, const pfc_gpu_step_args* a, float* dx_local,
                            pfc_gpu_step_out* out) {
  const int64_t B = b_local * c->R;
  cudaStream_t s = c->stream;
  const float* x = x_local;
  const int64_t* lab = labels_local;
  float* dxf = dx_local;
  if (c->coll) {  // feature all-gather (rank-major, all_gather_features shardsim.hpp:86-115)
    COMM_TRY(comm_all_gather(c, x_local, c->X, b_local * c->D, kF32, s));
    COMM_TRY(comm_all_gather(c, labels_local, c->labels, b_local, kI64, s));
    x = c->X;
    lab = c->labels;
    dxf = c->dX;
  }
  if (int rc = run_step(c, x, lab, B, a, dxf)) return rc;
  c->reset_status = false;  // errors stay on the device until a synchronous check
  if (c->coll)  // collective 3 (shardsim.hpp:387-399) as a reduce-scatter to the owners
    COMM_TRY(comm_reduce_scatter(c, c->dX, dx_local, b_local * c->D, kF32, kSum, s));
  if (!out) return PFC_OK;
  CUDA_TRY(c, cudaMemcpyAsync(c->st_host, c->st, sizeof(StepStatus), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  c->reset_status = true;
  if (int rc = finish_phase_timing(c)) return rc;
  return check_status(c, a->step_index, B, out);
}

// the reference's checks ahead of apcs / amncs (metrics.hpp:56-79, 91-146)
static int diag_validate(Ctx* c, const int64_t* labels, int64_t B, const int64_t* class_identity,
                         const int64_t* sample_identity) {
  if (B < 1 || B > c->maxB)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu: batch %lld outside [1, max_batch=%lld]", (long long)B,
                (long long)c->maxB);
  if ((class_identity == nullptr) != (sample_identity == nullptr))
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_diagnostics: give both identities or neither");
  // apcs (metrics.hpp:56-79) validates the labels first, then l2_normalize_columns (matrix.hpp:141)
  for (int64_t b = 0; b < B; ++b)
    if (labels[b] < 0 || labels[b] >= c->C)
      return fail(c, PFC_ERR_CONTRACT, "apcs: label %lld owned by no shard", (long long)labels[b]);
  return PFC_OK;
}

// apcs / amncs of the batch whose D x B fp64 features are in c->xdb and labels in c->labels
// (device), identities (split) in c->dcid / c->dsid; the labels were validated by the caller.
static int diagnostics_device(Ctx* c, int64_t B, bool split, pfc_gpu_diag_out* out) {
  cudaStream_t s = c->stream;
  dim3 grid((unsigned)ceil_div(B, 32), (unsigned)ceil_div(c->D, 32)), blk(32, 8);
  x_from_dxb_kernel<<<grid, blk, 0, s>>>(c->xdb, (int)c->D, (int)B, c->X);
  const int rc = c->bf16 ? run_diagnostics<__nv_bfloat16, true>(c, B, split)
                         : run_diagnostics<float, false>(c, B, split);
  if (rc) return rc;
  if (c->coll) {  // merge over ranks: maxima, sibling flags, the owner's apcs term
    COMM_TRY(comm_all_reduce(c, c->demax, c->demax, B * 3, kU64, kMax, s));
    COMM_TRY(comm_all_reduce(c, c->dhasc, c->dhasc, B, kI32, kMax, s));
    COMM_TRY(comm_all_reduce(c, c->dapcs, c->dapcs, B, kF64, kSum, s));
  }
  std::vector<unsigned long long> em((size_t)B * 3);
  std::vector<int> hc((size_t)B);
  std::vector<double> ap((size_t)B);
  CUDA_TRY(c, cudaMemcpyAsync(em.data(), c->demax, sizeof(unsigned long long) * B * 3,
                              cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(hc.data(), c->dhasc, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(ap.data(), c->dapcs, sizeof(double) * B, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  // means in the reference's order (b ascending, metrics.hpp:76-78, 118-146)
  double apcs = 0.0, total = 0.0, hard = 0.0, conf = 0.0;
  int64_t conf_rows = 0;
  for (int64_t b = 0; b < B; ++b) {
    apcs += ap[b];
    const double m0 = dec_f64(em[b * 3]), m1 = dec_f64(em[b * 3 + 1]), m2 = dec_f64(em[b * 3 + 2]);
    total += split ? std::max(m1, m2) : m0;
    if (split) {
      hard += m2;
      if (hc[b]) {
        conf += m1;
        ++conf_rows;
      }
    }
  }
  *out = pfc_gpu_diag_out{};
  out->apcs = apcs / (double)B;
  out->amncs = total / (double)B;
  out->has_split = split ? 1 : 0;
  if (split) {
    out->amncs_hard = hard / (double)B;
    if (conf_rows > 0) {
      out->amncs_conflicted = conf / (double)conf_rows;
      out->has_conflicted = 1;
    }
  }
  return PFC_OK;
}

int pfc_gpu_diagnostics(void* ctx, const double* xdb, const int64_t* labels, int64_t B,
                        const int64_t* class_identity, const int64_t* sample_identity,
                        pfc_gpu_diag_out* out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (int rc = diag_validate(c, labels, B, class_identity, sample_identity)) return rc;
  for (int64_t i = 0; i < B * c->D; ++i)
    if (!std::isfinite(xdb[i]))
      return fail(c, PFC_ERR_NUMERICAL, "l2_normalize_columns: non-finite entry in %lldx%lld result",
                  (long long)c->D, (long long)B);
  if (c->C < 2) return fail(c, PFC_ERR_CONTRACT, "amncs: needs at least two classes");
  const bool split = class_identity != nullptr;
  cudaStream_t s = c->stream;
  if (int rc = diag_alloc(c)) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(c->xdb, xdb, sizeof(double) * B * c->D, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(c->labels, labels, sizeof(int64_t) * B, cudaMemcpyHostToDevice, s));
  if (split) {
    CUDA_TRY(c, cudaMemcpyAsync(c->dcid, class_identity + c->cls_lo, sizeof(int64_t) * c->rows,
                                cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(c->dsid, sample_identity, sizeof(int64_t) * B,
                                cudaMemcpyHostToDevice, s));
  }
  return diagnostics_device(c, B, split, out);
}

int pfc_gpu_sync(void* ctx, pfc_gpu_step_out* out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  CUDA_TRY(c, cudaMemcpyAsync(c->st_host, c->st, sizeof(StepStatus), cudaMemcpyDeviceToHost,
                              c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->reset_status = true;
  if (int rc = finish_phase_timing(c)) return rc;
  return check_status(c, -1, c->lastB, out);
}

int pfc_gpu_get_buffers(void* ctx, int64_t k, int64_t* cls, int64_t* npos) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (k < c->k0 || k >= c->k0 + c->nk)
    return fail(c, PFC_ERR_CONTRACT, "shard %lld is not local to rank %d", (long long)k, c->rank);
  const int64_t kk = k - c->k0;
  int64_t* tmp = nullptr;
  CUDA_TRY(c, cudaMalloc(&tmp, sizeof(int64_t) * std::max<int64_t>(c->cap, 1)));
  buffers_out_kernel<<<(unsigned)ceil_div(std::max<int64_t>(c->cap, 1), 256), 256, 0, c->stream>>>(
      c->buf_cls + kk * c->cap, (int)c->cap, tmp);
  CUDA_TRY(c, cudaMemcpyAsync(cls, tmp, sizeof(int64_t) * c->cap, cudaMemcpyDeviceToHost, c->stream));
  ShardMeta m;
  CUDA_TRY(c, cudaMemcpyAsync(&m, c->meta + kk, sizeof(ShardMeta), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  cudaFree(tmp);
  if (npos) *npos = m.npos;
  return PFC_OK;
}

int pfc_gpu_bench_inputs(void* ctx, uint64_t seed, uint64_t step, int64_t B, float* x,
                         int64_t* labels) {
  Ctx* c = static_cast<Ctx*>(ctx);
  auto stream_of = [](const char* tag, uint64_t a) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (const char* p = tag; *p; ++p) {
      h ^= (unsigned char)*p;
      h *= 0x100000001b3ULL;
    }
    h = mix64(h ^ mix64(a + kPhi));
    h = mix64(h ^ mix64(0 + 0x2545f4914f6cdd1dULL));
    return h;  // make_stream(tag, a, 0)  (rng.hpp:91-96)
  };
  int* rej = nullptr;
  CUDA_TRY(c, cudaMalloc(&rej, sizeof(int)));
  CUDA_TRY(c, cudaMemsetAsync(rej, 0, sizeof(int), c->stream));
  const uint64_t kl = rng_key(seed, stream_of("bench-labels", step));
  const uint64_t kx = rng_key(seed, stream_of("bench-x", step));
  bench_labels_kernel<<<(unsigned)ceil_div(B, 256), 256, 0, c->stream>>>(kl, (int)B, c->C, labels, rej);
  bench_x_kernel<<<(unsigned)ceil_div(B * c->D, 256), 256, 0, c->stream>>>(kx, B * c->D, x);
  int hrej = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&hrej, rej, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  cudaFree(rej);
  if (hrej) {  // exact sequential next_below (rng.hpp:67-73) on the host; astronomically rare
    std::vector<int64_t> h((size_t)B);
    uint64_t ctr = 0;
    const uint64_t n = (uint64_t)c->C, limit = UINT64_MAX - UINT64_MAX % n;
    for (int64_t b = 0; b < B; ++b) {
      uint64_t r = rng_draw(kl, ++ctr);
      while (r >= limit) r = rng_draw(kl, ++ctr);
      h[(size_t)b] = (int64_t)(r % n);
    }
    CUDA_TRY(c, cudaMemcpy(labels, h.data(), sizeof(int64_t) * B, cudaMemcpyHostToDevice));
  }
  return PFC_OK;
}

int pfc_gpu_set_phase_timing(void* ctx, int enabled) {
  static_cast<Ctx*>(ctx)->pt.enabled = enabled != 0;
  return PFC_OK;
}

int pfc_gpu_phase_times(void* ctx, float* ms, const char** names, int n) {
  Ctx* c = static_cast<Ctx*>(ctx);
  const int m = std::min(n, c->pt.n);
  for (int i = 0; i < m; ++i) {
    ms[i] = c->pt.ms[i];
    if (names) names[i] = c->pt.names[i];
  }
  return m;
}

int64_t pfc_gpu_launches_per_step(void* ctx) { return static_cast<Ctx*>(ctx)->launches; }

}  // extern "C"

// ====================================================================== trainer integration
// the reference's training loop (trainer.hpp:362-581) drives the step with a
// backbone in front of it.  Here the dataset points, the backbone (trainer.hpp:51-126, fp64), the
// step's features X and its d_features dX all live on the device; per step the host sends the
// batch's point ids and reads back the step status (loss).  The loop itself (split, shuffle,
// schedule, checkpoints, final metrics) is include/pfc/gpu_trainer.hpp.
#include "backbone.cuh"

namespace {

struct Trainer {
  Ctx* c = nullptr;
  int64_t in_dim = 0, npts = 0, H = 0, E = 0, maxB = 0;
  std::vector<void*> allocs;
  std::vector<int64_t> plabels_h;          // observed labels (host copy: validation, diagnostics)
  double* points = nullptr;                // in_dim x npts (device, the dataset)
  int64_t* plabels = nullptr;              // npts
  double *w1 = nullptr, *b1 = nullptr, *w2 = nullptr, *b2 = nullptr;  // H x in, H, E x H, E
  double *inputs = nullptr, *hidden = nullptr, *feat = nullptr;        // in x B, H x B, E x B
  double *dw2 = nullptr, *dhid = nullptr, *dw1 = nullptr;              // E x H, H x B, H x in
  int64_t* ids = nullptr;                  // maxB (device)
  int64_t* ids_h = nullptr;                // maxB (pinned)
  int* flag = nullptr;                     // non-finite product bits (device)
  int* flag_h = nullptr;                   // pinned
  std::vector<int64_t> batch_labels;       // labels of the last forward batch
  int64_t B = 0;                           // batch of the cached activations (0: none)
  bool stepped = false;                    // the cached batch has a d_features in c->xdb

  template <typename T>
  cudaError_t alloc(T** p, size_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) allocs.push_back(q);
    *p = static_cast<T*>(q);
    return e;
  }
};

// the reference's shape strings of the products whose require_finite failed (matrix.hpp:103)
int trainer_flag_error(Trainer* t, int bits, int64_t B) {
  const int64_t shapes[5][2] = {{t->H, B}, {t->E, B}, {t->E, t->H}, {t->H, B}, {t->H, t->in_dim}};
  for (int w = 0; w < 5; ++w)
    if (bits & (1 << w))
      return fail(t->c, PFC_ERR_NUMERICAL, "matmul: non-finite entry in %lldx%lld result",
                  (long long)shapes[w][0], (long long)shapes[w][1]);
  return PFC_OK;
}

// reads and clears the device flag (synchronises the context stream)
int trainer_check(Trainer* t, int64_t B) {
  Ctx* c = t->c;
  CUDA_TRY(c, cudaMemcpyAsync(t->flag_h, t->flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  const int bits = *t->flag_h;
  if (bits) {
    CUDA_TRY(c, cudaMemsetAsync(t->flag, 0, sizeof(int), c->stream));
    return trainer_flag_error(t, bits, B);
  }
  return PFC_OK;
}

template <int EPI>
cudaError_t bb_matmul(Trainer* t, const double* A, int64_t a_i, int64_t a_k, const double* Bm,
                      int64_t b_k, int64_t b_j, double* C, int64_t rows, int64_t cols,
                      int64_t inner, const double* aux, int which) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  dim3 grid((unsigned)ceil_div(cols, 128), (unsigned)rows);
  bb_matmul_kernel<EPI><<<grid, 128, 0, t->c->stream>>>(A, a_i, a_k, Bm, b_k, b_j, C, (int)rows,
                                                        (int)cols, (int)inner, aux, t->flag, which);
  t->c->launches++;
  return cudaGetLastError();
}

// Backbone::forward (trainer.hpp:79-96) of `n` dataset points into t->feat (E x n, the step's
// FeatureBatch layout); caches inputs and hidden for apply_gradient.
int trainer_forward(Trainer* t, const int64_t* ids, int64_t n) {
  Ctx* c = t->c;
  cudaStream_t s = c->stream;
  for (int64_t b = 0; b < n; ++b)
    if (ids[b] < 0 || ids[b] >= t->npts)
      return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_trainer: point id %lld outside [0, %lld)",
                  (long long)ids[b], (long long)t->npts);
  std::memcpy(t->ids_h, ids, sizeof(int64_t) * n);
  CUDA_TRY(c, cudaMemcpyAsync(t->ids, t->ids_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
  bb_gather_kernel<<<dim3((unsigned)ceil_div(n, 128), (unsigned)t->in_dim), 128, 0, s>>>(
      t->points, t->npts, (int)t->in_dim, t->ids, (int)n, t->plabels, t->inputs, c->labels);
  c->launches++;
  CUDA_TRY(c, cudaGetLastError());
  // hidden = tanh(w1 inputs + b1); output = w2 hidden + b2
  CUDA_TRY(c, bb_matmul<kBbTanhBias>(t, t->w1, t->in_dim, 1, t->inputs, n, 1, t->hidden, t->H, n,
                                     t->in_dim, t->b1, 0));
  CUDA_TRY(c, bb_matmul<kBbBias>(t, t->w2, t->H, 1, t->hidden, n, 1, t->feat, t->E, n, t->H,
                                 t->b2, 1));
  t->batch_labels.resize((size_t)n);
  for (int64_t b = 0; b < n; ++b) t->batch_labels[(size_t)b] = t->plabels_h[(size_t)ids[b]];
  t->B = n;
  t->stepped = false;
  return PFC_OK;
}

// Backbone::init (trainer.hpp:65-77) on the host: the same counter-based streams and Box-Muller
// (rng.hpp:77-81) with the host libm, so the initial weights equal the reference's bit for bit.
void backbone_init_host(int64_t rows, int64_t cols, uint64_t seed, const char* tag,
                        std::vector<double>& w) {
  uint64_t h = 0xcbf29ce484222325ULL;  // fnv1a(tag) (rng.hpp:26-32)
  for (const char* p = tag; *p; ++p) {
    h ^= (unsigned char)*p;
    h *= 0x100000001b3ULL;
  }
  h = mix64(h ^ mix64(0 + kPhi));  // make_stream(tag, 0, 0) (rng.hpp:91-96)
  h = mix64(h ^ mix64(0 + 0x2545f4914f6cdd1dULL));
  const uint64_t key = rng_key(seed, h);
  const double sc = 1.0 / std::sqrt((double)cols);
  w.assign((size_t)(rows * cols), 0.0);
  uint64_t ctr = 0;
  for (double& v : w) {
    const double u1 = ((double)(rng_draw(key, ++ctr) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = (double)(rng_draw(key, ++ctr) >> 11) * 0x1.0p-53;
    v = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793 * u2) * sc;
  }
}

}  // namespace

extern "C" {

int pfc_gpu_step_features(void* ctx, const double* xdb_dev, const int64_t* labels_dev, int64_t B,
                          const pfc_gpu_step_args* a, double* dxdb_dev, pfc_gpu_step_out* out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  if (!(a->lr >= 0.0)) return fail(c, PFC_ERR_CONTRACT, "distributed_partial_step: lr must be >= 0");
  if (B < 0) return fail(c, PFC_ERR_SHAPE, "FeatureBatch: label count != feature columns");
  if (B == 0)
    return fail(c, PFC_ERR_NUMERICAL, "distributed_partial_step: non-finite loss at step %lld",
                (long long)a->step_index);
  if (B > c->maxB)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu: batch %lld exceeds max_batch %lld", (long long)B,
                (long long)c->maxB);
  cudaStream_t s = c->stream;
  // labels are checked on the device by the sampler (same errors as build_buffers)
  if (xdb_dev != c->xdb)
    CUDA_TRY(c, cudaMemcpyAsync(c->xdb, xdb_dev, sizeof(double) * B * c->D, cudaMemcpyDeviceToDevice, s));
  if (labels_dev != c->labels)
    CUDA_TRY(c, cudaMemcpyAsync(c->labels, labels_dev, sizeof(int64_t) * B, cudaMemcpyDeviceToDevice, s));
  if (int rc = step_from_xdb(c, B, a, out)) return rc;
  if (dxdb_dev && dxdb_dev != c->xdb)
    CUDA_TRY(c, cudaMemcpyAsync(dxdb_dev, c->xdb, sizeof(double) * B * c->D, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  return PFC_OK;
}

int pfc_gpu_check_guards(void* ctx, int64_t* corrupted) {
  Ctx* c = static_cast<Ctx*>(ctx);
  *corrupted = 0;
  if (!(c->d.flags & PFC_FLAG_GUARD))
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_check_guards: context created without PFC_FLAG_GUARD");
  CUDA_TRY(c, cudaDeviceSynchronize());
  std::vector<uint8_t> h(kGuardBytes);
  std::string where;
  for (size_t i = 0; i < c->guards.size(); ++i) {
    const Ctx::Guard& g = c->guards[i];
    for (int side = 0; side < 2; ++side) {
      const uint8_t* at = side ? g.base + kGuardBytes + g.user : g.base;
      CUDA_TRY(c, cudaMemcpy(h.data(), at, kGuardBytes, cudaMemcpyDeviceToHost));
      size_t bad = 0, first = kGuardBytes;
      for (size_t j = 0; j < kGuardBytes; ++j)
        if (h[j] != (uint8_t)kGuardByte) {
          ++bad;
          if (first == kGuardBytes) first = j;
        }
      if (bad) {
        ++*corrupted;
        char buf[160];
        snprintf(buf, sizeof buf, "%sbuffer #%zu (%zu bytes): %zu guard bytes %s it changed, first at %zu",
                 where.empty() ? "" : "; ", i, g.user, bad, side ? "after" : "before", first);
        where += buf;
      }
    }
  }
  if (*corrupted) return fail(c, PFC_ERR_CUDA, "out-of-bounds writes: %s", where.c_str());
  return PFC_OK;
}

int pfc_gpu_trainer_create(void* ctx, const double* points, int64_t input_dim, int64_t num_points,
                           const int64_t* observed_labels, int64_t hidden_dim, int64_t embed_dim,
                           uint64_t seed, void** trainer_out) {
  Ctx* c = static_cast<Ctx*>(ctx);
  *trainer_out = nullptr;
  if (c->R > 1)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_trainer: single-rank contexts only");
  if (input_dim < 1 || num_points < 1 || hidden_dim < 1 || embed_dim < 2)
    return fail(c, PFC_ERR_CONFIG, "train: bad backbone dims");
  if (embed_dim != c->D)
    return fail(c, PFC_ERR_SHAPE, "pfc_gpu_trainer: embed_dim %lld != the context's dim %lld",
                (long long)embed_dim, (long long)c->D);
  auto* t = new Trainer();
  t->c = c;
  t->in_dim = input_dim;
  t->npts = num_points;
  t->H = hidden_dim;
  t->E = embed_dim;
  t->maxB = c->maxB;
  t->plabels_h.assign(observed_labels, observed_labels + num_points);
  const size_t mb = (size_t)t->maxB;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  A(t->alloc(&t->points, (size_t)(input_dim * num_points)));
  A(t->alloc(&t->plabels, (size_t)num_points));
  A(t->alloc(&t->w1, (size_t)(hidden_dim * input_dim)));
  A(t->alloc(&t->b1, (size_t)hidden_dim));
  A(t->alloc(&t->w2, (size_t)(embed_dim * hidden_dim)));
  A(t->alloc(&t->b2, (size_t)embed_dim));
  A(t->alloc(&t->inputs, (size_t)input_dim * mb));
  A(t->alloc(&t->hidden, (size_t)hidden_dim * mb));
  A(t->alloc(&t->feat, (size_t)embed_dim * mb));
  A(t->alloc(&t->dw2, (size_t)(embed_dim * hidden_dim)));
  A(t->alloc(&t->dhid, (size_t)hidden_dim * mb));
  A(t->alloc(&t->dw1, (size_t)(hidden_dim * input_dim)));
  A(t->alloc(&t->ids, mb));
  A(t->alloc(&t->flag, 1));
  A(cudaMallocHost(&t->ids_h, sizeof(int64_t) * mb));
  A(cudaMallocHost(&t->flag_h, sizeof(int)));
  if (e == cudaSuccess) {
    cudaStream_t s = c->stream;
    std::vector<double> w1, w2, zh((size_t)hidden_dim, 0.0), ze((size_t)embed_dim, 0.0);
    backbone_init_host(hidden_dim, input_dim, seed, "backbone-w1", w1);
    backbone_init_host(embed_dim, hidden_dim, seed, "backbone-w2", w2);
    A(cudaMemcpyAsync(t->points, points, sizeof(double) * input_dim * num_points, cudaMemcpyHostToDevice, s));
    A(cudaMemcpyAsync(t->plabels, observed_labels, sizeof(int64_t) * num_points, cudaMemcpyHostToDevice, s));
    A(cudaMemcpyAsync(t->w1, w1.data(), sizeof(double) * w1.size(), cudaMemcpyHostToDevice, s));
    A(cudaMemcpyAsync(t->w2, w2.data(), sizeof(double) * w2.size(), cudaMemcpyHostToDevice, s));
    A(cudaMemcpyAsync(t->b1, zh.data(), sizeof(double) * zh.size(), cudaMemcpyHostToDevice, s));
    A(cudaMemcpyAsync(t->b2, ze.data(), sizeof(double) * ze.size(), cudaMemcpyHostToDevice, s));
    A(cudaMemsetAsync(t->flag, 0, sizeof(int), s));
    A(cudaStreamSynchronize(s));
  }
  if (e != cudaSuccess) {
    for (void* p : t->allocs) cudaFree(p);
    if (t->ids_h) cudaFreeHost(t->ids_h);
    if (t->flag_h) cudaFreeHost(t->flag_h);
    delete t;
    return fail(c, PFC_ERR_CUDA, "pfc_gpu_trainer_create: %s", cudaGetErrorString(e));
  }
  *trainer_out = t;
  return PFC_OK;
}

int pfc_gpu_trainer_destroy(void* tr) {
  if (!tr) return PFC_OK;
  auto* t = static_cast<Trainer*>(tr);
  cudaStreamSynchronize(t->c->stream);
  for (void* p : t->allocs) cudaFree(p);
  if (t->ids_h) cudaFreeHost(t->ids_h);
  if (t->flag_h) cudaFreeHost(t->flag_h);
  delete t;
  return PFC_OK;
}

int pfc_gpu_trainer_get_backbone(void* tr, double* w1, double* b1, double* w2, double* b2) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  cudaStream_t s = c->stream;
  // a pending non-finite product surfaces here, before anything (a checkpoint) is written
  if (int rc = trainer_check(t, t->B)) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(w1, t->w1, sizeof(double) * t->H * t->in_dim, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(b1, t->b1, sizeof(double) * t->H, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(w2, t->w2, sizeof(double) * t->E * t->H, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(b2, t->b2, sizeof(double) * t->E, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  return PFC_OK;
}

int pfc_gpu_trainer_set_backbone(void* tr, const double* w1, const double* b1, const double* w2,
                                 const double* b2) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  cudaStream_t s = c->stream;
  CUDA_TRY(c, cudaMemcpyAsync(t->w1, w1, sizeof(double) * t->H * t->in_dim, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(t->b1, b1, sizeof(double) * t->H, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(t->w2, w2, sizeof(double) * t->E * t->H, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(t->b2, b2, sizeof(double) * t->E, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  t->B = 0;
  return PFC_OK;
}

int pfc_gpu_trainer_forward(void* tr, const int64_t* point_ids, int64_t batch) {
  auto* t = static_cast<Trainer*>(tr);
  if (batch < 1 || batch > t->maxB)
    return fail(t->c, PFC_ERR_CONTRACT, "pfc_gpu_trainer: batch %lld outside [1, max_batch=%lld]",
                (long long)batch, (long long)t->maxB);
  return trainer_forward(t, point_ids, batch);
}

int pfc_gpu_trainer_diagnostics(void* tr, const int64_t* class_identity,
                                const int64_t* sample_identity, pfc_gpu_diag_out* out) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  if (t->B < 1 || t->stepped)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_trainer_diagnostics: call after forward, before step");
  const int64_t B = t->B;
  if (int rc = diag_validate(c, t->batch_labels.data(), B, class_identity, sample_identity)) return rc;
  if (int rc = trainer_check(t, B)) return rc;  // the features are finite (matmul checks)
  if (c->C < 2) return fail(c, PFC_ERR_CONTRACT, "amncs: needs at least two classes");
  const bool split = class_identity != nullptr;
  cudaStream_t s = c->stream;
  if (int rc = diag_alloc(c)) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(c->xdb, t->feat, sizeof(double) * B * c->D, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(c->labels, t->batch_labels.data(), sizeof(int64_t) * B,
                              cudaMemcpyHostToDevice, s));
  if (split) {
    CUDA_TRY(c, cudaMemcpyAsync(c->dcid, class_identity + c->cls_lo, sizeof(int64_t) * c->rows,
                                cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(c->dsid, sample_identity, sizeof(int64_t) * B,
                                cudaMemcpyHostToDevice, s));
  }
  return diagnostics_device(c, B, split, out);
}

int pfc_gpu_trainer_step(void* tr, const pfc_gpu_step_args* a, pfc_gpu_step_out* out) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  if (t->B < 1 || t->stepped)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_trainer_step: call after forward");
  if (!(a->lr >= 0.0)) return fail(c, PFC_ERR_CONTRACT, "distributed_partial_step: lr must be >= 0");
  const int64_t B = t->B;
  if (int rc = host_validate(c, t->batch_labels.data(), B)) return rc;
  cudaStream_t s = c->stream;
  // the batch labels were gathered into c->labels by the forward
  CUDA_TRY(c, cudaMemcpyAsync(c->xdb, t->feat, sizeof(double) * B * c->D, cudaMemcpyDeviceToDevice, s));
  if (int rc = trainer_check(t, B)) return rc;  // Backbone::forward's matmul checks come first
  if (int rc = step_from_xdb(c, B, a, out)) return rc;
  t->stepped = true;  // d_features (D x B fp64) are in c->xdb
  return PFC_OK;
}

int pfc_gpu_trainer_apply_gradient(void* tr, double lr) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  if (!t->stepped)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_trainer_apply_gradient: call after a successful step");
  const int64_t B = t->B, H = t->H, E = t->E, I = t->in_dim;
  const double* dout = c->xdb;  // E x B
  // d_w2 = d_out hidden^T; d_hidden = (w2^T d_out) * (1 - h^2); d_w1 = d_hidden inputs^T
  CUDA_TRY(c, bb_matmul<kBbPlain>(t, dout, B, 1, t->hidden, 1, B, t->dw2, E, H, B, nullptr, 2));
  CUDA_TRY(c, bb_matmul<kBbTanhGrad>(t, t->w2, 1, H, dout, B, 1, t->dhid, H, B, E, t->hidden, 3));
  CUDA_TRY(c, bb_matmul<kBbPlain>(t, t->dhid, B, 1, t->inputs, 1, B, t->dw1, H, I, B, nullptr, 4));
  // matmul's require_finite throws before apply_gradient touches w1/w2 (matrix.hpp:103,
  // trainer.hpp:98-124): the products' flags are read before the SGD rows run
  if (int rc = trainer_check(t, B)) return rc;
  // SGD, w2 rows then w1 rows (trainer.hpp:113-124)
  bb_sgd_rows_kernel<<<(unsigned)E, 128, 0, c->stream>>>(t->w2, t->b2, t->dw2, dout, (int)H, (int)B, lr);
  bb_sgd_rows_kernel<<<(unsigned)H, 128, 0, c->stream>>>(t->w1, t->b1, t->dw1, t->dhid, (int)I, (int)B, lr);
  c->launches += 2;
  CUDA_TRY(c, cudaGetLastError());
  t->stepped = false;
  t->B = 0;
  return PFC_OK;
}

// normalised embeddings [n][E] of the points into a device buffer (chunked forward)
int trainer_embed_device(Trainer* t, const int64_t* point_ids, int64_t n, double* emb) {
  Ctx* c = t->c;
  for (int64_t at = 0; at < n; at += t->maxB) {
    const int64_t m = std::min<int64_t>(t->maxB, n - at);
    if (int rc = trainer_forward(t, point_ids + at, m)) return rc;
    if (int rc = trainer_check(t, m)) return rc;
    eval_normalize_kernel<<<(unsigned)ceil_div(m, 128), 128, 0, c->stream>>>(
        t->feat, (int)t->E, (int)m, emb + at * t->E);
    CUDA_TRY(c, cudaGetLastError());
  }
  t->B = 0;  // the cached activations are not a training batch
  return PFC_OK;
}

int pfc_gpu_trainer_nearest_center(void* tr, const int64_t* point_ids, int64_t n,
                                   int64_t* best_class) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  if (n <= 0) return PFC_OK;
  if (t->E > 512)
    return fail(c, PFC_ERR_CONTRACT, "pfc_gpu_trainer_nearest_center: embed_dim %lld > 512",
                (long long)t->E);
  double *emb = nullptr, *winv = nullptr;
  int64_t* best = nullptr;
  cudaStream_t s = c->stream;
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    cudaFree(emb);
    cudaFree(winv);
    cudaFree(best);
  };
  cudaError_t e = cudaMalloc(&emb, sizeof(double) * n * t->E);
  if (e == cudaSuccess) e = cudaMalloc(&winv, sizeof(double) * std::max<int64_t>(c->rows, 1));
  if (e == cudaSuccess) e = cudaMalloc(&best, sizeof(int64_t) * n);
  if (e != cudaSuccess) {
    cleanup();
    return fail(c, PFC_ERR_CUDA, "pfc_gpu_trainer_nearest_center: %s", cudaGetErrorString(e));
  }
  int rc = trainer_embed_device(t, point_ids, n, emb);
  if (rc == PFC_OK) {
    eval_center_inv_kernel<<<(unsigned)ceil_div(std::max<int64_t>(c->rows, 1), 128), 128, 0, s>>>(
        c->W, c->rows, (int)c->D, winv);
    eval_argmax_kernel<<<(unsigned)n, 256, 0, s>>>(emb, (int)t->E, c->W, winv, c->rows, best);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(best_class, best, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail(c, PFC_ERR_CUDA, "pfc_gpu_trainer_nearest_center: %s", cudaGetErrorString(e));
  }
  cleanup();
  return rc;
}

int pfc_gpu_trainer_pair_cosines(void* tr, const int64_t* point_ids, int64_t n, double* cos_out) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  if (n < 2) return PFC_OK;
  const int64_t np = n * (n - 1) / 2;
  double *emb = nullptr, *out = nullptr;
  cudaStream_t s = c->stream;
  auto cleanup = [&]() {
    cudaStreamSynchronize(s);
    cudaFree(emb);
    cudaFree(out);
  };
  cudaError_t e = cudaMalloc(&emb, sizeof(double) * n * t->E);
  if (e == cudaSuccess) e = cudaMalloc(&out, sizeof(double) * np);
  if (e != cudaSuccess) {
    cleanup();
    return fail(c, PFC_ERR_CUDA, "pfc_gpu_trainer_pair_cosines: %s", cudaGetErrorString(e));
  }
  int rc = trainer_embed_device(t, point_ids, n, emb);
  if (rc == PFC_OK) {
    for (int64_t i0 = 0; i0 < n && e == cudaSuccess; i0 += 65535) {  // rows i0.. (grid.y limit)
      const int64_t ni = std::min<int64_t>(65535, n - i0);
      dim3 grid((unsigned)ceil_div(n, 128), (unsigned)ni);
      eval_pairs_kernel<<<grid, 128, 0, s>>>(emb, (int)t->E, n, i0, out);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(cos_out, out, sizeof(double) * np, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = fail(c, PFC_ERR_CUDA, "pfc_gpu_trainer_pair_cosines: %s", cudaGetErrorString(e));
  }
  cleanup();
  return rc;
}

int pfc_gpu_trainer_embed(void* tr, const int64_t* point_ids, int64_t n, double* emb) {
  auto* t = static_cast<Trainer*>(tr);
  Ctx* c = t->c;
  for (int64_t at = 0; at < n; at += t->maxB) {
    const int64_t m = std::min<int64_t>(t->maxB, n - at);
    if (int rc = trainer_forward(t, point_ids + at, m)) return rc;
    if (int rc = trainer_check(t, m)) return rc;
    std::vector<double> blk((size_t)(t->E * m));
    CUDA_TRY(c, cudaMemcpyAsync(blk.data(), t->feat, sizeof(double) * t->E * m,
                                cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (int64_t e = 0; e < t->E; ++e)
      std::memcpy(emb + e * n + at, blk.data() + e * m, sizeof(double) * m);
  }
  t->B = 0;  // the cached activations are not a training batch
  return PFC_OK;
}

}  // extern "C"
