// epilogues.cuh — fused GEMM epilogues of the Partial-FC step.  Each epilogue warpgroup (128
// threads) runs the functor; thread `row` owns accumulator row (row0 + row) and pulls 32-column
// chunks from the accumulator source (TMEM on the tcgen05 engine, shared memory on the SIMT
// engine).  With NWG warpgroups, warpgroup wg owns columns [wg*BN/NWG, (wg+1)*BN/NWG).
//
//   FwdStatsEpi  rows = batch rows b, cols = buffered classes j.
//                cos tile -> margin (margin.hpp:41-54) + filter mask (shardsim.hpp:258-268)
//                -> per (row, column-slice) online (max, sum exp) partials and z_pos
//                (shardsim.hpp:270-318 restated flash-style: nothing B x cap reaches HBM).
//   GradEpi      rows = buffered classes j, cols = batch rows b (the recomputed cos tile).
//                g = ((p - onehot)/B) * margin'(c)  (shardsim.hpp:352-362) -> G^T (bf16 via
//                swizzled smem + TMA store, or fp32) and center_proj_j = sum_b g c partials,
//                thread-local in this orientation.
//   DwUpdateEpi  rows = classes, cols = dims: dW = (sum_b g x^ - center_proj w^)/|w|
//                (shardsim.hpp:377-384) fused with the sparse momentum-SGD of the sampled rows
//                (update_centers, shardsim.hpp:139-159); W / momentum of the next tile are
//                prefetched into L2 while this tile is processed.
//   DxPartEpi    rows = batch rows, cols = dims: split-K partials of sum_j g w^_j.
// feat_proj_b = sum_j g c_bj equals x^_b . (sum_j g w^_j) because c_bj = x^_b . w^_j, so it is
// formed in dx_finalize_kernel from the dX GEMM result instead of being reduced here.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "gemm.cuh"

namespace pfc {

constexpr float kLog2e = 1.4426950408889634f;

template <typename T>
__device__ __forceinline__ T neg_inf() {
  return -INFINITY;
}

__device__ __forceinline__ bool status_failed(const StepStatus* st) {
  return st->label_oob || st->capacity_shard >= 0 || st->batch_too_large ||
         st->masked_row != 0x7fffffff || st->nonfinite_loss || st->nonfinite_dx;
}

template <typename ST, bool kFilter>
struct FwdStatsEpi {
  static constexpr int kSmem = 0;
  int B, ncols;
  const int32_t* pos_col;
  MarginDev mg;
  float tau;
  ST* part_m;  // [n_tiles * NWG][B]
  ST* part_s;
  double* zpos;

  __device__ __forceinline__ void prefetch(const TileInfo&, int, int) const {}
  __device__ __forceinline__ void finish(int, int) const {}

  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t*) const {
    constexpr int CW = BN / NWG;
    const int b = t.row0 + row;
    const bool rv = b < B;
    const int pc = rv ? pos_col[b] : -1;
    ST m = neg_inf<ST>(), s = ST(0);
    const float A = mg.s * kLog2e;
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32) {
      float v[32];
      src.load(c0, v);
      const int colb = t.col0 + c0;
      if (!rv || colb >= ncols) continue;
      const int jp = pc - colb;
      if constexpr (std::is_same<ST, float>::value && !kFilter) {
        if (colb + 32 <= ncols && (unsigned)jp >= 32u) {
          // fast path: 32 valid negatives, z = s * c (s > 0 keeps the order of c)
          float vmax = v[0];
#pragma unroll
          for (int j = 1; j < 32; ++j) vmax = fmaxf(vmax, v[j]);
          const float mn = fmaxf(m, mg.s * vmax);
          float acc = (m == -INFINITY) ? 0.f : s * pfc_sm100::ex2_approx((m - mn) * kLog2e);
          const float off = mn * kLog2e;
          float acc2 = 0.f;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            acc += pfc_sm100::ex2_approx(fmaf(v[j], A, -off));
            acc2 += pfc_sm100::ex2_approx(fmaf(v[j + 1], A, -off));
          }
          s = acc + acc2;
          m = mn;
          continue;
        }
      }
      // general path: bounds, filter mask, the positive's margin (fp64, margin.hpp:41-54)
      ST z[32];
      ST cmax = neg_inf<ST>();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool masked = (colb + j >= ncols) || (kFilter && j != jp && v[j] > tau);
        z[j] = masked ? neg_inf<ST>() : (ST)mg.s * (ST)v[j];
      }
      if ((unsigned)jp < 32u) {
        float vp = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) vp = (j == jp) ? v[j] : vp;
        const double zp = margin_pos(mg, (double)vp);
        zpos[b] = zp;
#pragma unroll
        for (int j = 0; j < 32; ++j) z[j] = (j == jp) ? (ST)zp : z[j];
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) cmax = z[j] > cmax ? z[j] : cmax;
      if (cmax == neg_inf<ST>()) continue;
      const ST mn = m > cmax ? m : cmax;
      ST acc = (m == neg_inf<ST>()) ? ST(0) : s * fast_exp(m - mn);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += fast_exp(z[j] - mn);
      s = acc;
      m = mn;
    }
    if (rv) {
      const size_t slot = (size_t)(t.n_tile * NWG + wg) * B + b;
      part_m[slot] = m;
      part_s[slot] = s;
    }
  }
};

__device__ __forceinline__ void pack_bf16x32(const float (&g)[32], uint32_t (&w)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
}
__device__ __forceinline__ void store_g32(__nv_bfloat16* dst, const float (&g)[32]) {
  uint32_t w[16];
  pack_bf16x32(g, w);
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

// rows = buffered classes j (M), cols = batch rows b (N).  Writes G^T[j][b].
template <typename ST, typename GT, bool kFilter, bool kTma>
struct alignas(64) GradEpi {
  static constexpr int kSmem = 36 * 1024;  // 4 KB column constants + 4 x 8 KB G^T staging
  CUtensorMap tm;     // G^T store map: inner = b (box 32, SWIZZLE_64B), outer = classes (box 128)
  int B, ncols, ldgt;
  const int32_t* pos_col;
  MarginDev mg;
  float tau;
  const ST* gmax;
  const ST* inv_gsum;
  ST inv_batch;
  GT* Gt;             // [ncols_pad][ldgt]
  ST* cproj_part;     // [n_tiles(b) * NWG][ncols]

  __device__ __forceinline__ void prefetch(const TileInfo&, int, int) const {}
  __device__ __forceinline__ void finish(int row, int) const {
    if constexpr (kTma) {
      if (row == 0) pfc_sm100::bulk_wait_all();
    }
  }

  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t* smem) const {
    constexpr int CW = BN / NWG;
    static_assert(CW <= 128, "column slice");
    const int cb = wg * CW;
    const uint32_t bar = 1 + wg;
    // per-column (b) constants of this warpgroup's slice
    float2* cf = reinterpret_cast<float2*>(smem);          // [CW] {gmax*log2e, s*ig/B}
    ST* cg = reinterpret_cast<ST*>(cf + CW);               // [CW] gmax
    ST* ci = cg + CW;                                      // [CW] inv_gsum
    uint8_t* prow = reinterpret_cast<uint8_t*>(ci + CW);   // [CW] positive's row in tile or 0xFF
    uint8_t* stage = smem + 4096;                          // CW/32 x [128][64 B], 64B-swizzled
    if (kTma && row == 0) pfc_sm100::bulk_wait_read<0>();  // last tile's stores left smem
    pfc_sm100::named_bar_sync(bar, 128);
    for (int i = row; i < CW; i += 128) {
      const int b = t.col0 + cb + i;
      float2 k = make_float2(0.f, 0.f);
      ST gm = ST(0), ig = ST(0);
      uint8_t pr = 0xFF;
      if (b < B) {
        gm = gmax[b];
        ig = inv_gsum[b];
        k = make_float2((float)gm * kLog2e, (float)(mg.sd * (double)ig * (double)inv_batch));
        const int pc = pos_col[b] - t.row0;
        if ((unsigned)pc < 128u) pr = (uint8_t)pc;
      }
      cf[i] = k;
      cg[i] = gm;
      ci[i] = ig;
      prow[i] = pr;
    }
    pfc_sm100::named_bar_sync(bar, 128);
    const int j = t.row0 + row;
    const bool rv = j < ncols;
    const float A = mg.s * kLog2e;
    const uint32_t rowx4 = 0x01010101u * (uint32_t)row;
    ST cp = ST(0);
    bool staged = false;
#pragma unroll 1
    for (int c0 = cb; c0 < cb + CW; c0 += 32) {
      float v[32];
      src.load(c0, v);
      const int colb = t.col0 + c0;
      if (colb >= B) continue;  // uniform across the warpgroup
      const int lc = c0 - cb;
      float g[32];
      if constexpr (std::is_same<ST, float>::value) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const float2 k = cf[lc + q];
          float gq = pfc_sm100::ex2_approx(fmaf(v[q], A, -k.x)) * k.y;
          if (kFilter) gq = v[q] > tau ? 0.f : gq;
          g[q] = gq;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int b = colb + q;
          double gq = 0.0;
          if (b < B && !(kFilter && v[q] > tau)) {
            const double p = exp((double)mg.s * (double)v[q] - (double)cg[lc + q]) * (double)ci[lc + q];
            gq = p * (double)inv_batch * mg.sd;
          }
          g[q] = (float)gq;
        }
      }
      // positives in this chunk: columns b whose label is this thread's class j
      {
        const uint4* pw = reinterpret_cast<const uint4*>(prow + lc);
        const uint4 p0 = pw[0], p1 = pw[1];
        const uint32_t hit = __vcmpeq4(p0.x, rowx4) | __vcmpeq4(p0.y, rowx4) |
                             __vcmpeq4(p0.z, rowx4) | __vcmpeq4(p0.w, rowx4) |
                             __vcmpeq4(p1.x, rowx4) | __vcmpeq4(p1.y, rowx4) |
                             __vcmpeq4(p1.z, rowx4) | __vcmpeq4(p1.w, rowx4);
        if (hit) {
#pragma unroll 1
          for (int q = 0; q < 32; ++q) {
            if (prow[lc + q] != (uint8_t)row) continue;
            float vq = 0.f;
#pragma unroll
            for (int u = 0; u < 32; ++u) vq = (u == q) ? v[u] : vq;
            const double z = margin_pos(mg, (double)vq);
            const double p = exp(z - (double)cg[lc + q]) * (double)ci[lc + q];
            const double gq = (p - 1.0) * (double)inv_batch * margin_deriv_pos(mg, (double)vq);
#pragma unroll
            for (int u = 0; u < 32; ++u) g[u] = (u == q) ? (float)gq : g[u];
          }
        }
      }
      if (!rv) {
#pragma unroll
        for (int q = 0; q < 32; ++q) g[q] = 0.f;
      }
      ST c1 = ST(0), c2 = ST(0);
#pragma unroll
      for (int q = 0; q < 32; q += 2) {
        c1 += (ST)g[q] * (ST)v[q];
        c2 += (ST)g[q + 1] * (ST)v[q + 1];
      }
      cp += c1 + c2;
      if constexpr (kTma) {
        // 64B-swizzled staging of the 128 x 32 chunk; TMA stores after the slice is complete
        uint8_t* sb = stage + (lc >> 5) * 8192;
        uint32_t w[16];
        pack_bf16x32(g, w);
        const int sw = (row >> 1) & 3;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
          *reinterpret_cast<uint4*>(sb + row * 64 + ((qq ^ sw) << 4)) =
              make_uint4(w[4 * qq], w[4 * qq + 1], w[4 * qq + 2], w[4 * qq + 3]);
        staged = true;
      } else {
        GT* dst = Gt + (size_t)j * ldgt + colb;
        if (colb + 32 <= B) {
          store_g32(dst, g);
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (colb + q < B) store_g1(dst + q, g[q]);
        }
      }
    }
    if constexpr (kTma) {
      if (staged) {  // uniform
        pfc_sm100::fence_proxy_async_smem();
        pfc_sm100::named_bar_sync(bar, 128);
        if (row == 0) {
          for (int c0 = cb; c0 < cb + CW && t.col0 + c0 < B; c0 += 32)
            pfc_sm100::tma_store_2d(&tm, stage + ((c0 - cb) >> 5) * 8192, t.col0 + c0, t.row0);
          pfc_sm100::bulk_commit();
        }
      }
    }
    if (rv) cproj_part[(size_t)(t.n_tile * NWG + wg) * ncols + j] = cp;
  }
};

template <typename ST>
struct DwUpdateEpi {
  static constexpr int kSmem = 18 * 1024;
  int ncols, D, n_parts;
  const float* wnorm;       // [ncols]
  const int32_t* lrow;      // [ncols] local row of W
  const ST* cproj_part;     // [n_parts][ncols]
  float* W;
  float* Mom;
  float lr, mu, wd;
  const StepStatus* st;  // no update when the step failed (the reference throws before 412)
  int cw;                // columns per warpgroup (BN / NWG), for prefetch
  int pf_mode;           // 0 none, 1 current tile at epilogue start, 2 one tile ahead

  // Pull a tile's W / momentum row segments toward L2.
  __device__ __forceinline__ void prefetch(const TileInfo& t, int row, int wg) const {
    if (pf_mode == 2) prefetch_rows(t, row, wg);
  }
  __device__ __forceinline__ void prefetch_rows(const TileInfo& t, int row, int wg) const {
    const int c = t.row0 + row;
    if (c >= ncols) return;
    const int r = lrow[c];
    if (r < 0) return;
    const int d0 = t.col0 + wg * cw;
    if (d0 >= D) return;
    const int dn = min(cw, D - d0);
    const char* w = reinterpret_cast<const char*>(W + (size_t)r * D + d0);
    const char* m = reinterpret_cast<const char*>(Mom + (size_t)r * D + d0);
    for (int off = 0; off < dn * 4; off += 128) {
      pfc_sm100::prefetch_l2(w + off);
      pfc_sm100::prefetch_l2(m + off);
    }
  }
  __device__ __forceinline__ void finish(int, int) const {}

  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t* smem) const {
    constexpr int CW = BN / NWG;
    const uint32_t bar = 1 + wg;
    float* stage = reinterpret_cast<float*>(smem);  // [128][33]
    float* s_inv = stage + 128 * 33;
    float* s_cp = s_inv + 128;
    int* s_row = reinterpret_cast<int*>(s_cp + 128);
    const int warp = row >> 5, lane = row & 31;
    if (pf_mode == 1) prefetch_rows(t, row, wg);
    pfc_sm100::named_bar_sync(bar, 128);  // previous tile's readers are done with smem
    const bool failed = status_failed(st);
    {
      const int c = t.row0 + row;
      float inv = 0.f, cp = 0.f;
      int r = -1;
      if (c < ncols && !failed) {
        const float n = wnorm[c];
        inv = 1.0f / (n > 1e-12f ? n : 1e-12f);
        ST acc = ST(0);
        for (int p = 0; p < n_parts; ++p) acc += cproj_part[(size_t)p * ncols + c];
        cp = (float)acc;
        r = lrow[c];
      }
      s_inv[row] = inv;
      s_cp[row] = cp;
      s_row[row] = r;
    }
    const int sub = lane >> 3, q4 = (lane & 7) * 4;  // 4 rows x 8 lanes x float4 per warp op
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32) {
      float v[32];
      src.load(c0, v);
      pfc_sm100::named_bar_sync(bar, 128);
#pragma unroll
      for (int q = 0; q < 32; ++q) stage[row * 33 + q] = v[q];
      pfc_sm100::named_bar_sync(bar, 128);
      const int d = t.col0 + c0 + q4;
      if (d >= D) continue;
      const bool vec = (d + 4 <= D) && ((D & 3) == 0);
      float4 w[8], mo[8];
      int rw[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        rw[u] = s_row[warp * 32 + u * 4 + sub];
        if (rw[u] >= 0) {
          const size_t o = (size_t)rw[u] * D + d;
          if (vec) {
            w[u] = *reinterpret_cast<const float4*>(W + o);
            mo[u] = *reinterpret_cast<const float4*>(Mom + o);
          } else {
            w[u] = make_float4(W[o], d + 1 < D ? W[o + 1] : 0.f, d + 2 < D ? W[o + 2] : 0.f,
                               d + 3 < D ? W[o + 3] : 0.f);
            mo[u] = make_float4(Mom[o], d + 1 < D ? Mom[o + 1] : 0.f,
                                d + 2 < D ? Mom[o + 2] : 0.f, d + 3 < D ? Mom[o + 3] : 0.f);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (rw[u] < 0) continue;
        const int r = warp * 32 + u * 4 + sub;
        const float inv = s_inv[r], cpj = s_cp[r];
        const float* a = stage + r * 33 + q4;
        float wv[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
        float mv[4] = {mo[u].x, mo[u].y, mo[u].z, mo[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float dw = (a[e] - cpj * (wv[e] * inv)) * inv;
          const float g = dw + wd * wv[e];
          const float vv = mu * mv[e] + g;
          mv[e] = vv;
          wv[e] = wv[e] - lr * vv;
        }
        const size_t o = (size_t)rw[u] * D + d;
        if (vec) {
          *reinterpret_cast<float4*>(Mom + o) = make_float4(mv[0], mv[1], mv[2], mv[3]);
          *reinterpret_cast<float4*>(W + o) = make_float4(wv[0], wv[1], wv[2], wv[3]);
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (d + e < D) {
              Mom[o + e] = mv[e];
              W[o + e] = wv[e];
            }
        }
      }
    }
  }
};

struct DxPartEpi {
  static constexpr int kSmem = 0;
  int B, D;
  float* part;  // [splits][B][D]
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int) const {}
  __device__ __forceinline__ void finish(int, int) const {}
  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t*) const {
    constexpr int CW = BN / NWG;
    const int b = t.row0 + row;
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32) {
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
