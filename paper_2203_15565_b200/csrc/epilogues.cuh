// epilogues.cuh — fused GEMM epilogues of the Partial-FC step.  Each functor is run by 128
// threads; thread `tid` owns accumulator row (row0 + tid) and pulls 32-column chunks from the
// accumulator source (TMEM on the tcgen05 engine, shared memory on the SIMT engine).
//
//   FwdStatsEpi  : cos tile -> margin (margin.hpp:41-54) + filter mask (shardsim.hpp:258-268)
//                  -> per (row, column-tile) online (max, sum exp) partials and z_pos
//                  (shardsim.hpp:270-318 restated flash-style; nothing B x cap hits HBM)
//   GradEpi      : recomputed cos tile -> g = ((p - onehot)/B) * margin'(c) (shardsim.hpp:352-362)
//                  -> G (bf16/fp32) + partial feat_proj (row) and center_proj (column) sums
//   DwUpdateEpi  : dwt tile (sum_b g x^) -> dW = (dwt - center_proj w^)/|w| (shardsim.hpp:377-384)
//                  -> fused sparse momentum-SGD of the sampled rows (update_centers, 139-159)
//   DxPartEpi    : split-K partial of sum_j g w^_j -> fp32 partials (reduced in fixed order)
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace pfc {

template <typename T>
__device__ __forceinline__ T neg_inf();
template <>
__device__ __forceinline__ float neg_inf<float>() {
  return -INFINITY;
}
template <>
__device__ __forceinline__ double neg_inf<double>() {
  return -INFINITY;
}

// Transpose-reduce: lane l ends with sum over the warp's 32 lanes of v[l].
__device__ __forceinline__ float warp_transpose_sum32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

template <typename ST>
struct FwdStatsEpi {
  int B, ncols;
  const int32_t* pos_col;
  MarginDev mg;
  int has_filter;
  float tau;
  ST* part_m;  // [n_tiles][B]
  ST* part_s;  // [n_tiles][B]
  double* zpos;

  template <int BN, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int tid, uint8_t*) const {
    const int b = t.row0 + tid;
    const bool rv = b < B;
    const int pc = rv ? pos_col[b] : -1;
    ST m = neg_inf<ST>(), s = ST(0);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      src.load(c0, v);
      const int colb = t.col0 + c0;
      if (!rv || colb >= ncols) continue;
      ST z[32];
      ST cmax = neg_inf<ST>();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = colb + j;
        ST zz;
        bool masked = col >= ncols;
        if (col == pc) {
          const double zp = margin_pos(mg, (double)v[j]);
          zpos[b] = zp;
          zz = (ST)zp;
        } else {
          zz = (ST)mg.s * (ST)v[j];
          masked = masked || (has_filter && v[j] > tau);
        }
        z[j] = masked ? neg_inf<ST>() : zz;
        cmax = z[j] > cmax ? z[j] : cmax;
      }
      if (cmax == neg_inf<ST>()) continue;
      const ST mn = m > cmax ? m : cmax;
      ST acc = (m == neg_inf<ST>()) ? ST(0) : s * fast_exp(m - mn);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += fast_exp(z[j] - mn);
      s = acc;
      m = mn;
    }
    if (rv) {
      part_m[(size_t)t.n_tile * B + b] = m;
      part_s[(size_t)t.n_tile * B + b] = s;
    }
  }
};

__device__ __forceinline__ void store_g32(__nv_bfloat16* dst, const float (&g)[32]) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
}
__device__ __forceinline__ void store_g32(float* dst, const float (&g)[32]) {
  float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i] = make_float4(g[4 * i], g[4 * i + 1], g[4 * i + 2], g[4 * i + 3]);
}
__device__ __forceinline__ void store_g1(__nv_bfloat16* dst, float g) { *dst = __float2bfloat16_rn(g); }
__device__ __forceinline__ void store_g1(float* dst, float g) { *dst = g; }

template <typename ST, typename GT>
struct GradEpi {
  int B, ncols, ldg;
  const int32_t* pos_col;
  MarginDev mg;
  int has_filter;
  float tau;
  const ST* gmax;
  const ST* inv_gsum;
  ST inv_batch;
  GT* G;              // [B][ldg]
  ST* fproj_part;     // [n_tiles][B]
  ST* cproj_part;     // [m_tiles][ncols]

  template <int BN, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int tid,
                                      uint8_t* smem) const {
    float* red = reinterpret_cast<float*>(smem);  // [4][32]
    const int b = t.row0 + tid;
    const bool rv = b < B;
    const int pc = rv ? pos_col[b] : -1;
    const ST gm = rv ? gmax[b] : ST(0);
    const ST ig = rv ? inv_gsum[b] : ST(0);
    ST fp = ST(0);
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      src.load(c0, v);
      const int colb = t.col0 + c0;
      if (colb >= ldg) continue;  // uniform across the CTA
      float gf[32], gc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = colb + j;
        ST g = ST(0);
        if (rv && col < ncols) {
          const bool ip = col == pc;
          if (ip || !(has_filter && v[j] > tau)) {
            const ST z = ip ? (ST)margin_pos(mg, (double)v[j]) : (ST)mg.s * (ST)v[j];
            const ST p = fast_exp(z - gm) * ig;
            const ST gz = (p - (ip ? ST(1) : ST(0))) * inv_batch;
            const ST d = ip ? (ST)margin_deriv_pos(mg, (double)v[j]) : (ST)mg.s;
            g = gz * d;
          }
        }
        gf[j] = (float)g;
        const ST prod = g * (ST)v[j];
        fp += prod;
        gc[j] = (float)prod;
      }
      if (rv) {
        GT* dst = G + (size_t)b * ldg + colb;
        if (colb + 32 <= ldg) {
          store_g32(dst, gf);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (colb + j < ldg) store_g1(dst + j, gf[j]);
        }
      }
      const float colsum = warp_transpose_sum32(gc);
      red[warp * 32 + lane] = colsum;
      pfc_sm100::named_bar_sync(1, 128);
      if (tid < 32) {
        const int col = colb + tid;
        if (col < ncols)
          cproj_part[(size_t)t.m_tile * ncols + col] =
              (ST)red[tid] + (ST)red[32 + tid] + (ST)red[64 + tid] + (ST)red[96 + tid];
      }
      pfc_sm100::named_bar_sync(1, 128);
    }
    if (rv) fproj_part[(size_t)t.n_tile * B + b] = fp;
  }
};

template <typename ST>
struct DwUpdateEpi {
  int ncols, D, n_mparts;
  const float* wnorm;       // [ncols]
  const int32_t* lrow;      // [ncols] local row of W
  const ST* cproj_part;     // [n_mparts][ncols]
  float* W;
  float* Mom;
  float lr, mu, wd;
  const StepStatus* st;  // no update when the step failed (the reference throws before 412)

  template <int BN, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int tid,
                                      uint8_t* smem) const {
    float* stage = reinterpret_cast<float*>(smem);  // [128][33]
    float* s_inv = stage + 128 * 33;
    float* s_cp = s_inv + 128;
    int* s_row = reinterpret_cast<int*>(s_cp + 128);
    const int warp = tid >> 5, lane = tid & 31;
    pfc_sm100::named_bar_sync(1, 128);  // previous tile's readers are done with smem
    const bool failed = st->label_oob || st->capacity_shard >= 0 || st->batch_too_large ||
                        st->masked_row != 0x7fffffff || st->nonfinite_loss || st->nonfinite_dx;
    {
      const int c = t.row0 + tid;
      float inv = 0.f, cp = 0.f;
      int r = -1;
      if (c < ncols && !failed) {
        const float n = wnorm[c];
        inv = 1.0f / (n > 1e-12f ? n : 1e-12f);
        ST acc = ST(0);
        for (int p = 0; p < n_mparts; ++p) acc += cproj_part[(size_t)p * ncols + c];
        cp = (float)acc;
        r = lrow[c];
      }
      s_inv[tid] = inv;
      s_cp[tid] = cp;
      s_row[tid] = r;
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      src.load(c0, v);
      pfc_sm100::named_bar_sync(1, 128);
#pragma unroll
      for (int j = 0; j < 32; ++j) stage[tid * 33 + j] = v[j];
      pfc_sm100::named_bar_sync(1, 128);
      const int d = t.col0 + c0 + lane;
      if (d < D) {
#pragma unroll 1
        for (int rr = 0; rr < 32; rr += 8) {
          float w[8], mo[8];
          int rw[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            rw[u] = s_row[warp * 32 + rr + u];
            if (rw[u] >= 0) {
              w[u] = W[(size_t)rw[u] * D + d];
              mo[u] = Mom[(size_t)rw[u] * D + d];
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (rw[u] >= 0) {
              const int r = warp * 32 + rr + u;
              const float inv = s_inv[r];
              const float dw = (stage[r * 33 + lane] - s_cp[r] * (w[u] * inv)) * inv;
              const float g = dw + wd * w[u];
              const float vv = mu * mo[u] + g;
              Mom[(size_t)rw[u] * D + d] = vv;
              W[(size_t)rw[u] * D + d] = w[u] - lr * vv;
            }
          }
        }
      }
    }
  }
};

struct DxPartEpi {
  int B, D;
  float* part;  // [splits][B][D]
  template <int BN, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int tid, uint8_t*) const {
    const int b = t.row0 + tid;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      src.load(c0, v);
      const int d0 = t.col0 + c0;
      if (b >= B || d0 >= D) continue;
      float* dst = part + ((size_t)t.split * B + b) * D + d0;
      if (d0 + 32 <= D && (D & 3) == 0) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (d0 + j < D) dst[j] = v[j];
      }
    }
  }
};

}  // namespace pfc
