// kernels.cuh — bandwidth-bound kernels of the step (everything that is not a GEMM).
#pragma once
#include "common.cuh"

namespace pfc {

__device__ __forceinline__ bool sampler_failed(const StepStatus* st) {
  return st->label_oob || st->capacity_shard >= 0;
}
__device__ __forceinline__ bool step_failed(const StepStatus* st) {
  return sampler_failed(st) || st->masked_row != 0x7fffffff || st->nonfinite_loss || st->nonfinite_dx;
}

// Opens a step (thread 0 of the sampler's first kernel): per-step scalars + a fresh status block.
// Errors are sticky across asynchronous steps (pfc_gpu_sync reports and clears them), like the
// reference, which stops at the first throwing step: the status is kept and lr = 0 skips every
// update.
__device__ __forceinline__ void step_begin(StepStatus* st, StepParams* sp, uint64_t seed,
                                           uint64_t stream, float lr, int reset, const float* x,
                                           const int64_t* labels, float* dx) {
  sp->x = x;
  sp->labels = labels;
  sp->dx = dx;
  const bool sticky = !reset && (sampler_failed(st) || st->masked_row != 0x7fffffff ||
                                 st->nonfinite_loss || st->nonfinite_dx ||
                                 st->underflow_row != 0x7fffffff);
  sp->seed = seed;
  sp->stream = stream;
  sp->step_id += 1;
  sp->lr = sticky ? 0.f : lr;
  if (sticky) return;
  StepStatus s{};
  s.capacity_shard = -1;
  s.masked_row = 0x7fffffff;
  s.underflow_row = 0x7fffffff;
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
__device__ __forceinline__ void store_out(tf32_t* p, float v) { p->v = to_tf32(v); }

// FeatureBatch layout (D x B fp64, types.hpp:14-26) -> rows [B][D] fp32.  32x32 tiles.
__global__ void x_from_dxb_kernel(const double* __restrict__ xdb, int D, int B,
                                  float* __restrict__ X) {
  pdl_entry();
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
  pdl_entry();
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
__device__ __forceinline__ void normalize_x_rows(const float* __restrict__ xs, int B, int D,
                                                 int Dp, OT* __restrict__ xh,
                                                 float* __restrict__ xnorm, int blk) {
  const int warp = (blk * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B) return;
  const float* x = xs + (size_t)warp * D;
  double ss = 0.0;
  for (int d = lane; d < D; d += 32) ss += (double)x[d] * (double)x[d];
  ss = warp_sum(ss);
  const double n = sqrt(ss);
  const float inv = (float)(1.0 / (n > 1e-12 ? n : 1e-12));
  if (lane == 0) xnorm[warp] = (float)n;
  OT* o = xh + (size_t)warp * Dp;
  for (int d = lane; d < Dp; d += 32) store_out(o + d, d < D ? x[d] * inv : 0.f);
}

template <typename OT>
__global__ void normalize_x_kernel(const float* __restrict__ x, int B, int D, int Dp,
                                   OT* __restrict__ xh, float* __restrict__ xnorm) {
  pdl_entry();
  normalize_x_rows(x, B, D, Dp, xh, xnorm, (int)blockIdx.x);
}

// Centre gather + normalisation (shardsim.hpp:234-247).  One warp per sampled column; W is
// fp32 row-major [local classes][D] so each class is one contiguous row (128-bit loads).
template <typename OT>
__global__ void gather_w_kernel(const float* __restrict__ W, int D, int Dp,
                                const int32_t* __restrict__ buf_cls, int ncols, int ncols_pad,
                                int64_t cls_lo, int64_t rows, OT* __restrict__ wh,
                                float* __restrict__ wnorm, int32_t* __restrict__ lrow,
                                int32_t* __restrict__ pslot, const StepStatus* st) {
  pdl_entry();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= ncols_pad) return;
  if (lane == 0 && c < ncols) pslot[c] = -1;
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
        if constexpr (std::is_same<OT, __nv_bfloat16>::value) {  // one 8-byte store per lane
          __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * inv, v[i].y * inv);
          __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * inv, v[i].w * inv);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&lo);
          u.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(o + d) = u;
        } else {
          store_out(o + d, v[i].x * inv);
          store_out(o + d + 1, v[i].y * inv);
          store_out(o + d + 2, v[i].z * inv);
          store_out(o + d + 3, v[i].w * inv);
        }
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

// Sum the per-(column slice) sums of E = exp(z - o) of each row, in a fixed order: a block owns
// kRowsPerBlk rows; thread (g, r) sums slices t = g, g + kSliceGroups, ... of row r (coalesced over
// the rows of one slice, loads batched 8 deep, one fp32/fp64 running sum per thread), then the
// kSliceGroups partials are added in ascending g in fp64.  One launch replaces the former
// slices -> segments -> row kernels.
constexpr int kRowsPerBlk = 16, kSliceGroups = 64;  // 1024 threads: ~T / 64 loads per thread
constexpr int kStatsThreads = kRowsPerBlk * kSliceGroups;
template <typename ST>
__device__ __forceinline__ double row_slice_sum(const ST* __restrict__ ps, int T, int B, int b0,
                                                double* red /* [kSliceGroups][kRowsPerBlk] */) {
  const int r = threadIdx.x % kRowsPerBlk, g = threadIdx.x / kRowsPerBlk;
  const int b = b0 + r;
  ST acc = 0;
  if (b < B) {
    int t = g;
    for (; t + 7 * kSliceGroups < T; t += 8 * kSliceGroups) {
      ST v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ps[(size_t)(t + u * kSliceGroups) * B + b];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; t < T; t += kSliceGroups) acc += ps[(size_t)t * B + b];
  }
  red[g * kRowsPerBlk + r] = (double)acc;
  __syncthreads();
  double S = 0.0;
  if (g == 0) {
#pragma unroll
    for (int q = 0; q < kSliceGroups; ++q) S += red[q * kRowsPerBlk + r];
  }
  return S;  // valid in threads g == 0
}

// Rank-local row sums for the cross-rank exchange (world > 1): ls[b] = sum over this rank's slices.
template <typename ST>
__global__ void __launch_bounds__(kStatsThreads) local_sums_kernel(const ST* __restrict__ ps, int T, int B,
                                                         ST* __restrict__ ls) {
  pdl_entry();
  __shared__ double red[kSliceGroups * kRowsPerBlk];
  const int b0 = blockIdx.x * kRowsPerBlk;
  const double S = row_slice_sum(ps, T, B, b0, red);
  const int b = b0 + (int)threadIdx.x;
  if (threadIdx.x < kRowsPerBlk && b < B) ls[b] = (ST)S;
}

// Per-row softmax offset of the exact mode: o_b = max over the row's unmasked logits on this
// rank (s * the largest negative cosine of the MaxEpi slices, the local positive's z_pos), the
// rank-local max of shardsim.hpp:270-281; ranks then take the maximum (collective 1, 284-299).
// A row with nothing unmasked here gets -1e30 (its E values are all masked to 0).
__global__ void row_offset_kernel(const float* __restrict__ part_m, int T, int B,
                                  const int32_t* __restrict__ pos_col,
                                  const double* __restrict__ zpos, MarginDev mg,
                                  float* __restrict__ offr) {
  pdl_entry();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float m = -INFINITY;
  for (int t = 0; t < T; ++t) m = fmaxf(m, part_m[(size_t)t * B + b]);
  double o = (double)mg.s * (double)m;
  if (pos_col[b] >= 0) o = fmax(o, zpos[b]);
  offr[b] = isfinite(o) ? (float)o : -1e30f;
}

// Cross-rank sum in ascending rank order (collectives 1 + 2, shardsim.hpp:284-338), the loss
// terms, the row scale of G and the positive's correction:
//   S = sum_r ls[r];  loss_b = log S + o - z_pos;  rowscale = s / (B S)
//   delta_b = ((p_pos - 1)/B) margin'(c_pos) - rowscale * E_pos(stored)   (owner rank only)
// With one rank (ps != nullptr) the rank-local sum is formed here from the T slice sums
// (row_slice_sum).  A block owns kRowsPerBlk rows; the last block to finish reduces loss_row in
// a fixed order into the step's loss.
template <typename ST>
__global__ void __launch_bounds__(kStatsThreads) finalize_stats_kernel(
    const ST* __restrict__ ls, int R, const ST* __restrict__ ps, int T, int B,
    const double* __restrict__ zpos, const double* __restrict__ cpos,
    const float* __restrict__ epos, const int32_t* __restrict__ pos_col,
    const int* __restrict__ hasval, int has_filter, MarginDev mg, const float* __restrict__ offr,
    ST* __restrict__ rowscale, ST* __restrict__ delta, double* __restrict__ loss_row,
    StepStatus* st) {
  pdl_entry();
  __shared__ double red[kSliceGroups * kRowsPerBlk];
  const int b0 = blockIdx.x * kRowsPerBlk;
  const bool ok = !sampler_failed(st);
  double S = 0.0;
  if (ps) {
    S = row_slice_sum(ps, T, B, b0, red);
    S = (double)(ST)S;  // the rank-local sum in the statistics type, as exchanged with R > 1
  } else if (threadIdx.x < kRowsPerBlk && b0 + (int)threadIdx.x < B) {
    for (int r = 0; r < R; ++r) S += (double)ls[(size_t)r * B + b0 + threadIdx.x];
  }
  const int b = b0 + (int)threadIdx.x;
  if (ok && threadIdx.x < kRowsPerBlk && b < B) {
    [&] {
      rowscale[b] = 0;
      delta[b] = 0;
      loss_row[b] = 0;
      if (has_filter && hasval[b] == 0) {  // every buffer column masked (shardsim.hpp:294-297)
        atomicMin(&st->masked_row, b);
        return;
      }
      // S_b >= 1 with a per-row offset; with the fixed one, a tiny S_b means every logit of the
      // row sits far below the offset (terms under 2^-126 were flushed): flagged, so the host
      // drop-in reruns the step with per-row offsets
      if (!(S > 1e-20) || !isfinite(S)) {
        atomicMin(&st->underflow_row, b);
        return;
      }
      const double off = offr ? (double)offr[b] : mg.offd;
      const double invB = 1.0 / (double)B;
      const double rs = mg.sd * invB / S;
      rowscale[b] = (ST)rs;
      loss_row[b] = log(S) + off - zpos[b];
      if (pos_col[b] >= 0) {
        const double p = exp(zpos[b] - off) / S;
        const double g = (p - 1.0) * invB * margin_deriv_pos(mg, cpos[b]);
        delta[b] = (ST)(g - (double)(ST)rs * (double)epos[b]);
      }
    }();
  }
  __threadfence();
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&st->fin_blocks, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) acc += ((volatile double*)loss_row)[i];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
    st->fin_blocks = 0;
    if (sampler_failed(st) || st->masked_row != 0x7fffffff || st->underflow_row != 0x7fffffff)
      return;
    const double loss = v / (double)B;
    st->loss = loss;
    if (!isfinite(loss)) st->nonfinite_loss = 1;
  }
}

// rowscale_b * x^_b in the GEMM operand type: the dW GEMM's B operand (G = diag(rowscale) E).
// Also resets the draws' per-position list heads (off the critical path, on the forked stream):
// the walk no longer reads them, and resetting only the entries this step's draws set keeps them
// all -1 between steps without a memset over every pool position.
template <typename ST, typename OT>
__global__ void xs_kernel(const StepParams* __restrict__ sp, const float* __restrict__ xnorm,
                          const ST* __restrict__ rowscale, int B, int D, int Dp,
                          OT* __restrict__ xs, const ShardMeta* __restrict__ meta, int nk, int cap,
                          const int32_t* __restrict__ jv, int32_t* __restrict__ head,
                          int64_t pool_stride, const StepStatus* st) {
  pdl_entry();
  if (!sampler_failed(st)) {
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < (int64_t)nk * cap;
         g += (int64_t)gridDim.x * blockDim.x) {
      const int kk = (int)(g / cap), i = (int)(g % cap);
      const ShardMeta& m = meta[kk];
      if (!m.full && i < m.need) head[(int64_t)kk * pool_stride + jv[g]] = -1;
    }
  }
  const int b = blockIdx.x;
  const float* x = sp->x + (size_t)b * D;
  const float n = xnorm[b];
  const float inv = (float)(1.0 / (double)(n > 1e-12f ? n : 1e-12f));
  const ST rs = rowscale[b];
  OT* o = xs + (size_t)b * Dp;
  for (int d = threadIdx.x; d < Dp; d += blockDim.x)
    store_out(o + d, d < D ? (float)(rs * (ST)(x[d] * inv)) : 0.f);
}

// Positive corrections of dwt: poscorr[slot(j)] = sum over EVERY row b with pos_col[b] == j (in
// ascending b, like the reference's dwt accumulation, shardsim.hpp:349-376) of delta_b x^_b;
// pslot[j] = slot for this step's positive columns.  The batch is scanned in 256-row chunks;
// each chunk's matching rows are compacted in order and added to the running sums (kept in the
// output row between chunks, so a label may repeat any number of times).
__global__ void __launch_bounds__(256) poscorr_kernel(
    const ShardMeta* __restrict__ meta, int cap, int pmax, const int32_t* __restrict__ pos_col,
    int B, const StepParams* __restrict__ sp, const float* __restrict__ xnorm, int D,
    const float* __restrict__ delta_f, const double* __restrict__ delta_d,
    float* __restrict__ poscorr, int32_t* __restrict__ pslot, const StepStatus* st) {
  pdl_entry();
  const int kk = blockIdx.y, i = blockIdx.x;
  if (sampler_failed(st)) return;
  if (i >= meta[kk].npos) return;
  const int col = kk * cap + i, slot = kk * pmax + i;
  __shared__ int rows[256];
  __shared__ int warp_cnt[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* out = poscorr + (size_t)slot * D;
  bool first = true;  // no rows accumulated yet (every positive column has at least one row)
  for (int b0 = 0; b0 < B; b0 += 256) {
    const int b = b0 + threadIdx.x;
    const bool hit = b < B && pos_col[b] == col;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) warp_cnt[w] = __popc(m);
    __syncthreads();
    int before = 0, nr = 0;
    for (int q = 0; q < 8; ++q) {
      before += q < w ? warp_cnt[q] : 0;
      nr += warp_cnt[q];
    }
    if (hit) rows[before + __popc(m & ((1u << lane) - 1))] = b;
    __syncthreads();
    if (nr > 0) {  // uniform across the block
      for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float acc = first ? 0.f : out[d];
        for (int q = 0; q < nr; ++q) {
          const int bb = rows[q];
          const float n = xnorm[bb];
          const float xh = sp->x[(size_t)bb * D + d] * (1.0f / (n > 1e-12f ? n : 1e-12f));
          const float dl = delta_f ? delta_f[bb] : (float)delta_d[bb];
          acc += dl * xh;
        }
        out[d] = acc;
      }
      first = false;
    }
    __syncthreads();  // rows[] / warp_cnt[] are rewritten by the next chunk
  }
  if (threadIdx.x == 0) pslot[col] = slot;
}

// dX = (r - feat_proj * x^) / max(|x|, 1e-12)  (shardsim.hpp:371-375) with
//   r = rowscale_b * sum_split part + delta_b w^_pos(b)    (G = diag(rowscale) E + positive)
//   feat_proj_b = sum_j g_bj c_bj = x^_b . r_b              (c_bj = x^_b . w^_j, exact identity)
template <int D_PER_THREAD, typename ST>
__global__ void __launch_bounds__(256) dx_finalize_kernel(
    const float* __restrict__ part, int S, const StepParams* __restrict__ sp,
    const float* __restrict__ xnorm, const ST* __restrict__ rowscale,
    const ST* __restrict__ delta, const int32_t* __restrict__ pos_col,
    const int32_t* __restrict__ lrow, const float* __restrict__ wnorm,
    const float* __restrict__ W, int B, int D, StepStatus* st) {
  pdl_entry();
  const int b = blockIdx.x;
  __shared__ double red[8];
  const float* __restrict__ X = sp->x;
  float* __restrict__ dX = sp->dx;
  const float n = xnorm[b];
  const float inv = 1.0f / (n > 1e-12f ? n : 1e-12f);
  const float rs = (float)rowscale[b];
  const float dl = (float)delta[b];
  const int pc = pos_col[b];
  const float* wpos = nullptr;
  float winv = 0.f;
  if (pc >= 0 && dl != 0.f) {
    const int r = lrow[pc];
    if (r >= 0) {
      wpos = W + (size_t)r * D;
      const float wn = wnorm[pc];
      winv = 1.0f / (wn > 1e-12f ? wn : 1e-12f);
    }
  }
  float r[D_PER_THREAD], xh[D_PER_THREAD];
  double dot = 0.0;
#pragma unroll
  for (int i = 0; i < D_PER_THREAD; ++i) {
    const int d = threadIdx.x + i * 256;
    float acc = 0.f;
    xh[i] = 0.f;
    if (d < D) {
      // ascending splits; loads issued 8 at a time (independent L2 round trips)
      const float* p = part + (size_t)b * D + d;
      const size_t stride = (size_t)B * D;
      int s = 0;
      for (; s + 8 <= S; s += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = p[(size_t)(s + u) * stride];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      for (; s < S; ++s) acc += p[(size_t)s * stride];
      acc *= rs;
      if (wpos) acc += dl * (wpos[d] * winv);
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

// fp32 validation path: finish the sampled rows from the stored dwt (warp per class):
// center_proj = w^ . dwt, dW = (dwt - center_proj w^)/|w|, momentum-SGD (shardsim.hpp:139-159).
__global__ void dw_rows_update_kernel(const float* __restrict__ dwt, const int32_t* __restrict__ lrow,
                                      const float* __restrict__ wnorm,
                                      const int32_t* __restrict__ pslot,
                                      const float* __restrict__ poscorr, int ncols, int D,
                                      float* __restrict__ W, float* __restrict__ Mom,
                                      const StepParams* __restrict__ sp, float mu, float wd,
                                      const StepStatus* st) {
  pdl_entry();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= ncols) return;
  if (sampler_failed(st) || st->masked_row != 0x7fffffff || st->nonfinite_loss ||
      st->nonfinite_dx || st->underflow_row != 0x7fffffff)
    return;
  const int r = lrow[c];
  if (r < 0) return;
  const int ps = pslot[c];
  const float n = wnorm[c];
  const double inv = 1.0 / (double)(n > 1e-12f ? n : 1e-12f);
  float* w = W + (size_t)r * D;
  float* m = Mom + (size_t)r * D;
  double dot = 0.0;
  for (int d = lane; d < D; d += 32) {
    double a = dwt[(size_t)c * D + d];
    if (ps >= 0) a += poscorr[(size_t)ps * D + d];
    dot += a * (double)w[d];
  }
  dot = warp_sum(dot);
  const double cp = dot * inv;
  const float lr = sp->lr;
  for (int d = lane; d < D; d += 32) {
    double a = dwt[(size_t)c * D + d];
    if (ps >= 0) a += poscorr[(size_t)ps * D + d];
    const float wv = w[d];
    const float dw = (float)((a - cp * ((double)wv * inv)) * inv);
    const float g = dw + wd * wv;
    const float vv = mu * m[d] + g;
    m[d] = vv;
    w[d] = wv - lr * vv;
  }
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

// Dim-row block [d0, d0 + dn) x n classes of the reference's D x owned layout <-> rows
// [row0, row0 + n) of the fp32 row-major state (checkpoint streams, io.hpp put_matrix order).
__global__ void dims_out_kernel(const float* __restrict__ W, int D, int n, int64_t row0, int d0,
                                int dn, double* __restrict__ blk) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int j = j0 + i, dd = i0 + threadIdx.x;
    tile[i][threadIdx.x] = (j < n && dd < dn) ? W[(size_t)(row0 + j) * D + d0 + dd] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int dd = i0 + i, j = j0 + threadIdx.x;
    if (dd < dn && j < n) blk[(size_t)dd * n + j] = (double)tile[threadIdx.x][i];
  }
}
__global__ void dims_in_kernel(const double* __restrict__ blk, int D, int n, int64_t row0, int d0,
                               int dn, float* __restrict__ W) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int dd = i0 + i, j = j0 + threadIdx.x;
    tile[i][threadIdx.x] = (dd < dn && j < n) ? (float)blk[(size_t)dd * n + j] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int j = j0 + i, dd = i0 + threadIdx.x;
    if (j < n && dd < dn) W[(size_t)(row0 + j) * D + d0 + dd] = tile[threadIdx.x][i];
  }
}

__global__ void buffers_out_kernel(const int32_t* __restrict__ buf, int n, int64_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = buf[i];
}

}  // namespace pfc
