// kernels.cuh — bandwidth-bound kernels of the step (everything that is not a GEMM).
#pragma once
#include "common.cuh"

namespace pfc {

__device__ __forceinline__ bool sampler_failed(const StepStatus* st) {
  return st->label_oob || st->capacity_shard >= 0 || st->batch_too_large;
}
__device__ __forceinline__ bool step_failed(const StepStatus* st) {
  return sampler_failed(st) || st->masked_row != 0x7fffffff || st->nonfinite_loss || st->nonfinite_dx;
}

// First node of every step: per-step scalars + a fresh status block.  Errors are sticky
// across asynchronous steps (pfc_gpu_sync reports and clears them), like the reference,
// which stops at the first throwing step.
__global__ void step_begin_kernel(StepStatus* st, StepParams* sp, uint64_t seed, uint64_t stream,
                                  float lr, int reset, const float* x, const int64_t* labels,
                                  float* dx) {
  if (threadIdx.x != 0) return;
  sp->x = x;
  sp->labels = labels;
  sp->dx = dx;
  const bool sticky = !reset && (sampler_failed(st) || st->masked_row != 0x7fffffff ||
                                 st->nonfinite_loss || st->nonfinite_dx);
  sp->seed = seed;
  sp->stream = stream;
  sp->lr = sticky ? 0.f : lr;
  if (sticky) return;
  StepStatus s{};
  s.capacity_shard = -1;
  s.masked_row = 0x7fffffff;
  *st = s;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void store_out(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ void store_out(float* p, float v) { *p = v; }

// FeatureBatch layout (D x B fp64, types.hpp:14-26) -> rows [B][D] fp32.  32x32 tiles.
__global__ void x_from_dxb_kernel(const double* __restrict__ xdb, int D, int B,
                                  float* __restrict__ X) {
  __shared__ float tile[32][33];
  const int b0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int d = d0 + i, b = b0 + threadIdx.x;
    tile[i][threadIdx.x] = (d < D && b < B) ? (float)xdb[(size_t)d * B + b] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int b = b0 + i, d = d0 + threadIdx.x;
    if (b < B && d < D) X[(size_t)b * D + d] = tile[threadIdx.x][i];
  }
}

// rows [B][D] fp32 -> D x B fp64 (StepResult::d_features layout).
__global__ void dx_to_dxb_kernel(const float* __restrict__ dX, int D, int B,
                                 double* __restrict__ out) {
  __shared__ float tile[32][33];
  const int b0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int b = b0 + i, d = d0 + threadIdx.x;
    tile[i][threadIdx.x] = (b < B && d < D) ? dX[(size_t)b * D + d] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int d = d0 + i, b = b0 + threadIdx.x;
    if (d < D && b < B) out[(size_t)d * B + b] = (double)tile[threadIdx.x][i];
  }
}

// Feature normalisation (shardsim.hpp:196-204): |x| (fp64 accumulate), x^ = x * 1/max(|x|,1e-12),
// written zero-padded to Dp columns in the GEMM operand type.  One warp per row.
template <typename OT>
__global__ void normalize_x_kernel(const StepParams* __restrict__ sp, int B, int D, int Dp,
                                   OT* __restrict__ xh, float* __restrict__ xnorm) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B) return;
  const float* x = sp->x + (size_t)warp * D;
  double ss = 0.0;
  for (int d = lane; d < D; d += 32) ss += (double)x[d] * (double)x[d];
  ss = warp_sum(ss);
  const double n = sqrt(ss);
  const float inv = (float)(1.0 / (n > 1e-12 ? n : 1e-12));
  if (lane == 0) xnorm[warp] = (float)n;
  OT* o = xh + (size_t)warp * Dp;
  for (int d = lane; d < Dp; d += 32) store_out(o + d, d < D ? x[d] * inv : 0.f);
}

// Centre gather + normalisation (shardsim.hpp:234-247).  One warp per sampled column; W is
// fp32 row-major [local classes][D] so each class is one contiguous row (128-bit loads).
template <typename OT>
__global__ void gather_w_kernel(const float* __restrict__ W, int D, int Dp,
                                const int32_t* __restrict__ buf_cls, int ncols, int ncols_pad,
                                int64_t cls_lo, int64_t rows, OT* __restrict__ wh,
                                float* __restrict__ wnorm, int32_t* __restrict__ lrow,
                                const StepStatus* st) {
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= ncols_pad) return;
  OT* o = wh + (size_t)c * Dp;
  int64_t r = -1;
  if (c < ncols && !sampler_failed(st)) {
    r = (int64_t)buf_cls[c] - cls_lo;
    if (r < 0 || r >= rows) r = -1;
  }
  if (r < 0) {
    for (int d = lane; d < Dp; d += 32) store_out(o + d, 0.f);
    if (lane == 0 && c < ncols) {
      wnorm[c] = 0.f;
      lrow[c] = -1;
    }
    return;
  }
  const float* w = W + (size_t)r * D;
  if ((D & 127) == 0 && D <= 1024) {
    float4 v[8];
    const int nv = D / 128;  // float4 per lane
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nv) {
        v[i] = reinterpret_cast<const float4*>(w)[i * 32 + lane];
        ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
      }
    ss = warp_sum(ss);
    const float n = sqrtf(ss);
    const float inv = 1.0f / (n > 1e-12f ? n : 1e-12f);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < nv) {
        const int d = (i * 32 + lane) * 4;
        store_out(o + d, v[i].x * inv);
        store_out(o + d + 1, v[i].y * inv);
        store_out(o + d + 2, v[i].z * inv);
        store_out(o + d + 3, v[i].w * inv);
      }
    for (int d = D + lane; d < Dp; d += 32) store_out(o + d, 0.f);
    if (lane == 0) {
      wnorm[c] = n;
      lrow[c] = (int32_t)r;
    }
  } else {
    double ss = 0.0;
    for (int d = lane; d < D; d += 32) ss += (double)w[d] * (double)w[d];
    ss = warp_sum(ss);
    const double n = sqrt(ss);
    const float inv = (float)(1.0 / (n > 1e-12 ? n : 1e-12));
    for (int d = lane; d < Dp; d += 32) store_out(o + d, d < D ? w[d] * inv : 0.f);
    if (lane == 0) {
      wnorm[c] = (float)n;
      lrow[c] = (int32_t)r;
    }
  }
}

// Merge the per-column-tile (max, sumexp) partials of each row into one (max, sum) pair.
// Pass 1: grid (rows/128, segments); thread = row b, coalesced over b, loops its segment of
// tiles.  Pass 2: thread = row, folds the segments in order.
constexpr int kMergeSegs = 64;
template <typename ST>
__global__ void __launch_bounds__(128) merge_tiles_kernel(const ST* __restrict__ pm,
                                                          const ST* __restrict__ ps, int T, int B,
                                                          ST* __restrict__ sm, ST* __restrict__ ss) {
  const int b = blockIdx.x * 128 + threadIdx.x;
  if (b >= B) return;
  const int per = (T + gridDim.y - 1) / gridDim.y;
  const int t0 = blockIdx.y * per, t1 = min(T, t0 + per);
  ST m = -INFINITY;
  // pass A: max (independent loads, 4 in flight)
  int t = t0;
  for (; t + 4 <= t1; t += 4) {
    const ST a0 = pm[(size_t)t * B + b], a1 = pm[(size_t)(t + 1) * B + b];
    const ST a2 = pm[(size_t)(t + 2) * B + b], a3 = pm[(size_t)(t + 3) * B + b];
    m = fmax(m, fmax(fmax(a0, a1), fmax(a2, a3)));
  }
  for (; t < t1; ++t) m = fmax(m, pm[(size_t)t * B + b]);
  ST s = 0;
  if (m != (ST)-INFINITY) {
    for (t = t0; t + 4 <= t1; t += 4) {
      ST acc = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const ST mt = pm[(size_t)(t + u) * B + b], st = ps[(size_t)(t + u) * B + b];
        acc += (mt == (ST)-INFINITY) ? ST(0) : st * fast_exp(mt - m);
      }
      s += acc;
    }
    for (; t < t1; ++t) {
      const ST mt = pm[(size_t)t * B + b];
      if (mt != (ST)-INFINITY) s += ps[(size_t)t * B + b] * fast_exp(mt - m);
    }
  }
  sm[(size_t)blockIdx.y * B + b] = m;
  ss[(size_t)blockIdx.y * B + b] = s;
}
// warp per row: lanes over segments, then a warp reduction
template <typename ST>
__global__ void merge_segments_kernel(const ST* __restrict__ sm, const ST* __restrict__ ss,
                                      int nseg, int B, ST* __restrict__ lm, ST* __restrict__ ls) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (b >= B) return;
  ST m = -INFINITY;
  for (int i = lane; i < nseg; i += 32) m = fmax(m, sm[(size_t)i * B + b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  ST s = 0;
  if (m != (ST)-INFINITY)
    for (int i = lane; i < nseg; i += 32) {
      const ST mi = sm[(size_t)i * B + b];
      if (mi != (ST)-INFINITY) s += ss[(size_t)i * B + b] * fast_exp(mi - m);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    lm[b] = m;
    ls[b] = s;
  }
}

// Cross-rank merge in ascending rank order (collectives 1 and 2, shardsim.hpp:284-338),
// per-row loss terms, and the "all columns masked" contract check.
template <typename ST>
__global__ void merge_ranks_kernel(const ST* __restrict__ lm, const ST* __restrict__ ls, int R,
                                   int B, const double* __restrict__ zpos, ST* __restrict__ gmax,
                                   ST* __restrict__ inv_gsum, double* __restrict__ loss_row,
                                   StepStatus* st) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (sampler_failed(st)) return;
  ST m = -INFINITY;
  for (int r = 0; r < R; ++r) m = fmax(m, lm[(size_t)r * B + b]);
  if (!(m > (ST)-INFINITY)) {
    atomicMin(&st->masked_row, b);
    gmax[b] = 0;
    inv_gsum[b] = 0;
    loss_row[b] = 0;
    return;
  }
  double s = 0.0;
  for (int r = 0; r < R; ++r) {
    const ST mr = lm[(size_t)r * B + b];
    if (mr != (ST)-INFINITY) s += (double)ls[(size_t)r * B + b] * exp((double)mr - (double)m);
  }
  gmax[b] = m;
  inv_gsum[b] = (ST)(1.0 / s);
  loss_row[b] = log(s) + (double)m - zpos[b];
}

// loss = mean_b loss_row[b] in a fixed order (one CTA, deterministic).
__global__ void loss_reduce_kernel(const double* __restrict__ loss_row, int B, StepStatus* st) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) acc += loss_row[b];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      if (sampler_failed(st) || st->masked_row != 0x7fffffff) return;
      const double loss = v / (double)B;
      st->loss = loss;
      if (!isfinite(loss)) st->nonfinite_loss = 1;
    }
  }
}

// dX = (r - feat_proj * x^) / max(|x|, 1e-12)  (shardsim.hpp:371-375), r = sum_split part.
// feat_proj_b = sum_j g_bj c_bj = x^_b . r_b since c_bj = x^_b . w^_j (exact identity).
template <int D_PER_THREAD>
__global__ void __launch_bounds__(256) dx_finalize_kernel(const float* __restrict__ part, int S,
                                                          const StepParams* __restrict__ sp,
                                                          const float* __restrict__ xnorm, int B,
                                                          int D, StepStatus* st) {
  const int b = blockIdx.x;
  const float* __restrict__ X = sp->x;
  float* __restrict__ dX = sp->dx;
  __shared__ double red[8];
  const float n = xnorm[b];
  const float inv = 1.0f / (n > 1e-12f ? n : 1e-12f);
  float r[D_PER_THREAD], xh[D_PER_THREAD];
  double dot = 0.0;
#pragma unroll
  for (int i = 0; i < D_PER_THREAD; ++i) {
    const int d = threadIdx.x + i * 256;
    float acc = 0.f;
    xh[i] = 0.f;
    if (d < D) {
      for (int s = 0; s < S; ++s) acc += part[((size_t)s * B + b) * D + d];
      xh[i] = X[(size_t)b * D + d] * inv;
    }
    r[i] = acc;
    dot += (double)acc * (double)xh[i];
  }
  dot = warp_sum(dot);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
  __syncthreads();
  double fp = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) fp += red[w];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < D_PER_THREAD; ++i) {
    const int d = threadIdx.x + i * 256;
    if (d < D) {
      const float v = (r[i] - (float)fp * xh[i]) * inv;
      dX[(size_t)b * D + d] = v;
      bad |= !isfinite(v);
    }
  }
  if (bad && !sampler_failed(st)) st->nonfinite_dx = 1;
}

// SeededRng::next_normal (rng.hpp:77-81) from its two draws.
__device__ __forceinline__ double box_muller(uint64_t a, uint64_t b) {
  const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = (double)(b >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

// init_center_shards on the device (shardsim.hpp:56-82): class c's column is D draws of
// next_normal() from SeededRng(seed, make_stream("center-init", c)), unit-normalised (fp64).
__global__ void init_centers_kernel(float* __restrict__ W, float* __restrict__ M, int64_t rows,
                                    int D, int64_t cls_lo, uint64_t seed, uint64_t tag_hash) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const uint64_t cls = (uint64_t)(cls_lo + r);
  uint64_t h = mix64(tag_hash ^ mix64(cls + kPhi));
  h = mix64(h ^ mix64(0 + 0x2545f4914f6cdd1dULL));
  const uint64_t key = rng_key(seed, h);
  double ss = 0.0;
  for (int d = lane; d < D; d += 32) {
    const double v = box_muller(rng_draw(key, 2 * (uint64_t)d + 1), rng_draw(key, 2 * (uint64_t)d + 2));
    ss += v * v;
  }
  ss = warp_sum(ss);
  const double n = sqrt(ss);
  const double inv = 1.0 / (n > 1e-12 ? n : 1e-12);
  for (int d = lane; d < D; d += 32) {
    const double v = box_muller(rng_draw(key, 2 * (uint64_t)d + 1), rng_draw(key, 2 * (uint64_t)d + 2));
    W[r * D + d] = (float)(v * inv);
    M[r * D + d] = 0.f;
  }
}

// Bench inputs: labels via next_below(C) (draw b+1; a modulo rejection is flagged and the
// host redoes the labels sequentially), X via next_normal (draws 2i+1, 2i+2, i = b*D + d).
__global__ void bench_labels_kernel(uint64_t key, int B, int64_t C, int64_t* labels,
                                    int* rejected) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const uint64_t n = (uint64_t)C;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  const uint64_t r = rng_draw(key, (uint64_t)b + 1);
  if (r >= limit) atomicExch(rejected, 1);
  labels[b] = (int64_t)(r % n);
}
__global__ void bench_x_kernel(uint64_t key, int64_t n, float* X) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  X[i] = (float)box_muller(rng_draw(key, 2 * (uint64_t)i + 1), rng_draw(key, 2 * (uint64_t)i + 2));
}

// CenterShard (D x owned fp64, a column block [j0, j0+n)) <-> W rows [owned][D] fp32.
__global__ void shard_in_kernel(const double* __restrict__ blk, int D, int n, int64_t row0,
                                float* __restrict__ W) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int d = d0 + i, j = j0 + threadIdx.x;
    tile[i][threadIdx.x] = (d < D && j < n) ? (float)blk[(size_t)d * n + j] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int j = j0 + i, d = d0 + threadIdx.x;
    if (j < n && d < D) W[(size_t)(row0 + j) * D + d] = tile[threadIdx.x][i];
  }
}
__global__ void shard_out_kernel(const float* __restrict__ W, int D, int n, int64_t row0,
                                 double* __restrict__ blk) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int j = j0 + i, d = d0 + threadIdx.x;
    tile[i][threadIdx.x] = (j < n && d < D) ? W[(size_t)(row0 + j) * D + d] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int d = d0 + i, j = j0 + threadIdx.x;
    if (d < D && j < n) blk[(size_t)d * n + j] = (double)tile[threadIdx.x][i];
  }
}

__global__ void buffers_out_kernel(const int32_t* __restrict__ buf, int n, int64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = buf[i];
}

}  // namespace pfc
