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

  struct Pre {};
  __device__ __forceinline__ Pre preload(const TileInfo&, int, int) const { return {}; }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int) const {}
  __device__ __forceinline__ void finish(int, int) const {}

  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t*, const Pre&) const {
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
// kTma (tcgen05 engine): per-column constants arrive one tile ahead in registers (Pre); every
// warp stages its 32 rows x 32 columns chunks (64B-swizzled) in a private 4-deep ring and
// TMA-stores them itself, so the epilogue needs no cross-warp barrier.
template <typename ST, typename GT, bool kFilter, bool kTma>
struct alignas(64) GradEpi {
  static constexpr int kWarpBytes = 9728;  // 4 x 2 KB staging + 1 KB constants + 128 B rows
  static constexpr int kSmem = kTma ? 4 * kWarpBytes : 20 * 1024;
  CUtensorMap tm;     // G^T store map: inner = b (box 32, SWIZZLE_64B), outer = classes (box 32)
  int B, ncols, ldgt;
  const int32_t* pos_col;
  MarginDev mg;
  float tau;
  const ST* gmax;
  const ST* inv_gsum;
  ST inv_batch;
  GT* Gt;             // [ncols_pad][ldgt]
  ST* cproj_part;     // [n_tiles(b) * NWG][ncols]

  struct Pre {
    float2 k[4];
    int pc[4];
  };
  __device__ __forceinline__ Pre preload(const TileInfo& t, int row, int wg) const {
    Pre p{};
    if constexpr (kTma) {
      const int lane = row & 31;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int b = t.col0 + wg * 128 + lane + 32 * i;
        p.k[i] = make_float2(0.f, 0.f);
        p.pc[i] = -1;
        if (b < B) {
          const float gm = (float)gmax[b];
          const float ig = (float)inv_gsum[b];
          p.k[i] = make_float2(gm * kLog2e, (float)(mg.sd * (double)ig * (double)inv_batch));
          p.pc[i] = pos_col[b];
        }
      }
    }
    return p;
  }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int) const {}
  __device__ __forceinline__ void finish(int row, int) const {
    if constexpr (kTma) {
      if ((row & 31) == 0) pfc_sm100::bulk_wait_all();
    }
  }

  // g for 32 columns from the cosines v and per-column constants (gmax*log2e, s*ig/B)
  __device__ __forceinline__ void grad32(const float (&v)[32], const float2* cf, float (&g)[32]) const {
    const float A = mg.s * kLog2e;
    const float4* cf4 = reinterpret_cast<const float4*>(cf);  // two columns per 128-bit load
#pragma unroll
    for (int q = 0; q < 32; q += 2) {
      const float4 k = cf4[q >> 1];
      float g0 = pfc_sm100::ex2_approx(fmaf(v[q], A, -k.x)) * k.y;
      float g1 = pfc_sm100::ex2_approx(fmaf(v[q + 1], A, -k.z)) * k.w;
      if (kFilter) {
        g0 = v[q] > tau ? 0.f : g0;
        g1 = v[q + 1] > tau ? 0.f : g1;
      }
      g[q] = g0;
      g[q + 1] = g1;
    }
  }
  // the positive entry q of this chunk: margin form (margin.hpp:41-72), fp64
  __device__ __forceinline__ void patch_positive(const float (&v)[32], float (&g)[32], int q,
                                                 double gm, double ig) const {
    float vq = 0.f;
#pragma unroll
    for (int u = 0; u < 32; ++u) vq = (u == q) ? v[u] : vq;
    const double z = margin_pos(mg, (double)vq);
    const double p = exp(z - gm) * ig;
    const double gq = (p - 1.0) * (double)inv_batch * margin_deriv_pos(mg, (double)vq);
#pragma unroll
    for (int u = 0; u < 32; ++u) g[u] = (u == q) ? (float)gq : g[u];
  }

  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t* smem, const Pre& pre) const {
    constexpr int CW = BN / NWG;
    const int cb = wg * CW;
    const int j = t.row0 + row;
    const bool rv = j < ncols;
    ST cp = ST(0);
    if constexpr (kTma) {
      static_assert(CW == 128, "warp-private staging assumes 128 columns per warpgroup");
      const int wig = row >> 5, lane = row & 31;
      uint8_t* ws = smem + wig * kWarpBytes;
      uint8_t* stage = ws;                                   // 4 x [32 rows][64 B]
      float2* cf = reinterpret_cast<float2*>(ws + 8192);     // [128]
      uint8_t* prow = ws + 9216;                             // [128]
      __syncwarp();  // lanes finished reading the previous tile's constants
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        cf[lane + 32 * i] = pre.k[i];
        const int pr = pre.pc[i] - t.row0;
        prow[lane + 32 * i] = (uint8_t)((unsigned)pr < 128u ? pr : 0xFF);
      }
      __syncwarp();
      const uint32_t rowx4 = 0x01010101u * (uint32_t)row;
#pragma unroll 1
      for (int kk = 0; kk < CW / 32; ++kk) {
        const int c0 = cb + kk * 32;
        float v[32];
        src.load(c0, v);
        const int colb = t.col0 + c0;
        uint8_t* sb = stage + kk * 2048;
        if (colb < B) {  // uniform
          float g[32];
          grad32(v, cf + kk * 32, g);
          const uint4* pw = reinterpret_cast<const uint4*>(prow + kk * 32);
          const uint4 p0 = pw[0], p1 = pw[1];
          const uint32_t hit = __vcmpeq4(p0.x, rowx4) | __vcmpeq4(p0.y, rowx4) |
                               __vcmpeq4(p0.z, rowx4) | __vcmpeq4(p0.w, rowx4) |
                               __vcmpeq4(p1.x, rowx4) | __vcmpeq4(p1.y, rowx4) |
                               __vcmpeq4(p1.z, rowx4) | __vcmpeq4(p1.w, rowx4);
          if (hit) {
#pragma unroll 1
            for (int q = 0; q < 32; ++q)
              if (prow[kk * 32 + q] == (uint8_t)row)
                patch_positive(v, g, q, (double)gmax[colb + q], (double)inv_gsum[colb + q]);
          }
          // rows j >= ncols (last class tile) are clipped by the TMA store and not accumulated
          float c1 = 0.f, c2 = 0.f;
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            c1 = fmaf(g[q], v[q], c1);
            c2 = fmaf(g[q + 1], v[q + 1], c2);
          }
          cp += (ST)(c1 + c2);
          uint32_t w[16];
          pack_bf16x32(g, w);
          if (lane == 0) pfc_sm100::bulk_wait_read<3>();  // this buffer's store, 4 groups ago
          __syncwarp();
          const int sw = (lane >> 1) & 3;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            *reinterpret_cast<uint4*>(sb + lane * 64 + ((qq ^ sw) << 4)) =
                make_uint4(w[4 * qq], w[4 * qq + 1], w[4 * qq + 2], w[4 * qq + 3]);
          pfc_sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) pfc_sm100::tma_store_2d(&tm, sb, colb, t.row0 + wig * 32);
        }
        if (lane == 0) pfc_sm100::bulk_commit();  // one group per chunk (possibly empty)
      }
    } else {
      // SIMT engine (fp32 validation): block-wide constants, plain stores
      const uint32_t bar = 1 + wg;
      float2* cf = reinterpret_cast<float2*>(smem);
      ST* cg = reinterpret_cast<ST*>(cf + CW);
      ST* ci = cg + CW;
      int* pcs = reinterpret_cast<int*>(ci + CW);
      pfc_sm100::named_bar_sync(bar, 128);
      for (int i = row; i < CW; i += 128) {
        const int b = t.col0 + cb + i;
        ST gm = ST(0), ig = ST(0);
        int pc = -1;
        if (b < B) {
          gm = gmax[b];
          ig = inv_gsum[b];
          pc = pos_col[b];
        }
        cf[i] = make_float2((float)gm * kLog2e, (float)(mg.sd * (double)ig * (double)inv_batch));
        cg[i] = gm;
        ci[i] = ig;
        pcs[i] = pc;
      }
      pfc_sm100::named_bar_sync(bar, 128);
#pragma unroll 1
      for (int c0 = cb; c0 < cb + CW; c0 += 32) {
        float v[32];
        src.load(c0, v);
        const int colb = t.col0 + c0;
        if (colb >= B) continue;
        const int lc = c0 - cb;
        float g[32];
        if constexpr (std::is_same<ST, float>::value) {
          grad32(v, cf + lc, g);
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            double gq = 0.0;
            if (colb + q < B && !(kFilter && v[q] > tau)) {
              const double p = exp((double)mg.s * (double)v[q] - (double)cg[lc + q]) * (double)ci[lc + q];
              gq = p * (double)inv_batch * mg.sd;
            }
            g[q] = (float)gq;
          }
        }
        for (int q = 0; q < 32; ++q)
          if (pcs[lc + q] == j) patch_positive(v, g, q, (double)cg[lc + q], (double)ci[lc + q]);
        if (!rv) {
#pragma unroll
          for (int q = 0; q < 32; ++q) g[q] = 0.f;
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) cp += (ST)g[q] * (ST)v[q];
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
    if (rv) cproj_part[(size_t)(t.n_tile * NWG + wg) * ncols + j] = cp;
  }
};

template <typename ST, bool kVecD>
struct DwUpdateEpi {
  // per warp: transposed 32 x 32 chunk (stride 33) + 3 x 32 row scalars
  static constexpr int kWarpFloats = 32 * 33 + 3 * 32;
  static constexpr int kSmem = 4 * kWarpFloats * 4;
  int ncols, D, n_parts;
  const float* wnorm;       // [ncols]
  const int32_t* lrow;      // [ncols] local row of W
  const ST* cproj_part;     // [n_parts][ncols]
  float* W;
  float* Mom;
  const StepParams* sp;  // lr of this step
  float mu, wd;
  const StepStatus* st;  // no update when the step failed (the reference throws before 412)
  int cw;                // columns per warpgroup (BN / NWG), for prefetch
  int pf_mode;           // 0 none, 1 current tile at epilogue start, 2 one tile ahead

  struct Pre {
    float inv, cp;
    int r;
  };
  // the tile's per-row scalars: 1/|w|, center_proj (sum of partials), local W row
  __device__ __forceinline__ Pre preload(const TileInfo& t, int row, int) const {
    Pre p{0.f, 0.f, -1};
    const int c = t.row0 + row;
    if (c < ncols) {
      const float n = wnorm[c];
      p.inv = 1.0f / (n > 1e-12f ? n : 1e-12f);
      ST acc = ST(0);
      for (int q = 0; q < n_parts; ++q) acc += cproj_part[(size_t)q * ncols + c];
      p.cp = (float)acc;
      p.r = lrow[c];
    }
    return p;
  }
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

  __device__ __forceinline__ void update4(float4& w, float4& m, const float* a, float inv,
                                          float cpj, float lr) const {
    float wv[4] = {w.x, w.y, w.z, w.w};
    float mv[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float dw = (a[e] - cpj * (wv[e] * inv)) * inv;  // shardsim.hpp:382
      const float g = dw + wd * wv[e];                      // shardsim.hpp:152-153
      const float vv = mu * mv[e] + g;                      // shardsim.hpp:154
      mv[e] = vv;
      wv[e] = wv[e] - lr * vv;                              // shardsim.hpp:156
    }
    w = make_float4(wv[0], wv[1], wv[2], wv[3]);
    m = make_float4(mv[0], mv[1], mv[2], mv[3]);
  }

  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t* smem, const Pre& pre) const {
    constexpr int CW = BN / NWG;
    const int wig = row >> 5, lane = row & 31;
    float* ws = reinterpret_cast<float*>(smem) + wig * kWarpFloats;
    float* stage = ws;                 // [32][33]: row-of-warp x dim
    float* s_inv = ws + 32 * 33;
    float* s_cp = s_inv + 32;
    int* s_row = reinterpret_cast<int*>(s_cp + 32);
    if (pf_mode == 1) prefetch_rows(t, row, wg);
    const bool failed = status_failed(st);
    const float lr = sp->lr;
    __syncwarp();  // the warp finished reading the previous tile's scalars
    s_inv[lane] = pre.inv;
    s_cp[lane] = pre.cp;
    s_row[lane] = failed ? -1 : pre.r;
    __syncwarp();
    const int sub = lane >> 3, q4 = (lane & 7) * 4;  // 4 rows x 8 lanes x float4 per warp op
    int rw[8];
    float rinv[8], rcp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = u * 4 + sub;
      rw[u] = s_row[r];
      rinv[u] = s_inv[r];
      rcp[u] = s_cp[r];
    }
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32) {
      float v[32];
      src.load(c0, v);
      const int d = t.col0 + c0 + q4;
      if (kVecD && t.col0 + c0 >= D) continue;  // uniform
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 32; ++q) stage[lane * 33 + q] = v[q];
      __syncwarp();
      if constexpr (kVecD) {
        float4 w[8], mo[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (rw[u] >= 0) {
            const size_t o = (size_t)rw[u] * D + d;
            w[u] = *reinterpret_cast<const float4*>(W + o);
            mo[u] = *reinterpret_cast<const float4*>(Mom + o);
          }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (rw[u] >= 0) {
            update4(w[u], mo[u], stage + (u * 4 + sub) * 33 + q4, rinv[u], rcp[u], lr);
            const size_t o = (size_t)rw[u] * D + d;
            *reinterpret_cast<float4*>(Mom + o) = mo[u];
            *reinterpret_cast<float4*>(W + o) = w[u];
          }
      } else {
        // generic D: scalar lanes over the chunk's 32 dims, one row per iteration
        const int dd = t.col0 + c0 + lane;
        if (dd < D) {
          for (int r = 0; r < 32; ++r) {
            const int wr = s_row[r];
            if (wr < 0) continue;
            const size_t o = (size_t)wr * D + dd;
            float4 w4 = make_float4(W[o], 0.f, 0.f, 0.f), m4 = make_float4(Mom[o], 0.f, 0.f, 0.f);
            float a[4] = {stage[r * 33 + lane], 0.f, 0.f, 0.f};
            update4(w4, m4, a, s_inv[r], s_cp[r], lr);
            Mom[o] = m4.x;
            W[o] = w4.x;
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
  struct Pre {};
  __device__ __forceinline__ Pre preload(const TileInfo&, int, int) const { return {}; }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int) const {}
  __device__ __forceinline__ void finish(int, int) const {}
  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t*, const Pre&) const {
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
