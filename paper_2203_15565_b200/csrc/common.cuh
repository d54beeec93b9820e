// common.cuh — device-side definitions shared by the PFC hot-path kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace pfc {

// Operand type of the TF32 precision mode: fp32 storage holding values already rounded to tf32
// (cvt.rna), so the tensor core's tf32 read of the operand is exact and unbiased.
struct alignas(4) tf32_t {
  float v;
};
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ULL;

// reference rng.hpp:17-24 (murmur3 finaliser)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
// rng.hpp:49-51: stream id of SeededRng::fork(label)
__host__ __device__ __forceinline__ uint64_t fork_stream(uint64_t stream, uint64_t label) {
  return mix64(stream ^ mix64(label + kPhi));
}
// rng.hpp:53-56: draw number `counter` (1-based) of stream (seed, stream), as a pure function.
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
  return mix64(seed + kPhi) ^ mix64(stream);
}
__host__ __device__ __forceinline__ uint64_t rng_draw(uint64_t key, uint64_t counter) {
  return mix64(key + kPhi * counter);
}

// Programmatic dependent launch (PDL): the step's kernels are launched with programmatic
// stream serialisation, so kernel N+1's CTAs may be scheduled while kernel N drains.  Every
// kernel first waits for its predecessor grid to complete (griddepcontrol.wait: completion and
// memory visibility; a no-op without the launch attribute), then lets its own dependents start
// launching.  Only launch latency and prologues overlap; no data is read early.
__device__ __forceinline__ void pdl_entry() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Device status block, read back once per step (SURVEY.md §5 failure detection).
struct StepStatus {
  double loss;
  int32_t label_oob;          // 1 when some label is outside [0, C)
  int32_t capacity_shard;     // first shard (global id) with npos > cap, else -1
  int64_t oob_label;          // smallest out-of-range label (sorted order, as the reference)
  int32_t capacity_npos;
  int32_t masked_row;         // first row whose buffer columns are all masked, else INT32_MAX
  int32_t nonfinite_loss;
  int32_t nonfinite_dx;
  int32_t rejection_shards;   // count of shards that needed the sequential sampler
  int32_t reserved0;
  int32_t underflow_row;      // first row whose exp(z - offset) sum underflowed, else INT32_MAX
  uint32_t fin_blocks;        // finalize_stats blocks done (last one reduces the loss)
};

// Per-step scalars, written on the device by step_begin (thread 0 of mark_kernel, the only
// graph node whose arguments change between steps) and read by the kernels that need them.
struct StepParams {
  uint64_t seed;    // iteration_rng.seed()
  uint64_t stream;  // iteration_rng.stream_id()
  float lr;
  uint32_t step_id;        // incremented by every step_begin
  const float* x;          // [B][D] fp32 features of this step
  const int64_t* labels;   // [B]
  float* dx;               // [B][D] rank-local partial d_features
};

struct ShardMeta {        // per local shard
  int64_t lo, hi;         // owned range [lo, hi)
  int32_t npos;           // distinct positives
  int32_t need;           // cap - npos negatives to draw
  int32_t pool;           // N = owned - npos
  int32_t full;           // 1 -> full-sampling branch (ascending complement, no RNG)
  int32_t ustart;         // set label bits below the shard (its positives start at rank 0)
  int32_t reject;         // 1 -> a modulo rejection happened: sequential fallback
};

enum MarginKindDev : int { kPlain = 0, kAddCos = 1, kAddAng = 2, kComb = 3 };

struct MarginDev {
  int kind;
  float s;       // scale (1 for plain)
  double sd, md; // scale, margin in fp64 for the positive logit
  double m1d, m3d;  // combined margin (kComb): s (cos(m1 theta + m) - m3); 1 and 0 otherwise
  float off;     // fixed softmax offset o = max(0, s - 40): exp(z - o) never overflows (z <= s)
  double offd;
};

constexpr double kAngularClamp = 1e-7;  // margin.hpp:15

// apply_margin for the positive entry (margin.hpp:41-54), fp64 like the reference.
__device__ __forceinline__ double margin_pos(const MarginDev& mg, double c) {
  if (mg.kind == kPlain) return c;
  if (mg.kind == kAddCos) return mg.sd * (c - mg.md);
  const double lo = -1.0 + kAngularClamp, hi = 1.0 - kAngularClamp;
  const double cc = c < lo ? lo : (hi < c ? hi : c);
  if (mg.kind == kComb) return mg.sd * (cos(mg.m1d * acos(cc) + mg.md) - mg.m3d);
  return mg.sd * cos(acos(cc) + mg.md);
}
// margin_derivative for the positive entry (margin.hpp:58-72).
__device__ __forceinline__ double margin_deriv_pos(const MarginDev& mg, double c) {
  if (mg.kind == kPlain) return 1.0;
  if (mg.kind == kAddCos) return mg.sd;
  if (c <= -1.0 + kAngularClamp || c >= 1.0 - kAngularClamp) return 0.0;
  const double th = acos(c);
  if (mg.kind == kComb) return mg.sd * mg.m1d * sin(mg.m1d * th + mg.md) / sqrt(1.0 - c * c);
  return mg.sd * sin(th + mg.md) / sqrt(1.0 - c * c);
}

__device__ __forceinline__ float fast_exp(float x) { return __expf(x); }
__device__ __forceinline__ double fast_exp(double x) { return exp(x); }

}  // namespace pfc
