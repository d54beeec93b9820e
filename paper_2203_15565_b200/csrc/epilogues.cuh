// epilogues.cuh — fused GEMM epilogues of the Partial-FC step.  Each epilogue warpgroup (128
// threads) runs the functor; thread `row` owns accumulator row (row0 + row) and pulls 32-column
// chunks from the accumulator source (TMEM on the tcgen05 engine, shared memory on the SIMT
// engine).  With NWG warpgroups, warpgroup wg owns columns [wg*BN/NWG, (wg+1)*BN/NWG).
//
// Softmax in a fixed-offset form.  Every logit satisfies z <= s (|cos| <= 1, margins only lower
// the positive), so with o = max(0, s - 40) the quantity E = exp(z - o) lies in [0, e^40] and
// never overflows.  Then, with S_b = sum_j E_bj (the rank-local and cross-rank sums):
//   loss_b = log S_b + o - z_pos                 (shardsim.hpp:330-334: log gsum + gmax - z_pos)
//   g_bj   = (s / (B S_b)) E_bj                  for negatives   (shardsim.hpp:356-359)
//   g_bpos = ((p_pos - 1)/B) margin'(c_pos)       for the positive
// so G = diag(rowscale) E + (sparse positive correction) and no B x cap gradient matrix or
// logits recompute is needed: the logits GEMM writes E once (bf16), the dX GEMM consumes E
// (row scale applied in its finalize), and the dW GEMM consumes E against rowscale * x^.
// The offset is either fixed (s <= 64: o = max(0, s - 40), no extra pass) or per row (s > 64, or
// after a fixed-offset underflow, or forced): o_b = max over the row's unmasked logits across all
// ranks, taken by a preceding max-only pass of the same GEMM (MaxEpi) -- the reference's own
// max-subtracted form (shardsim.hpp:270-318), valid for any s > 0.  A fixed-offset row whose sum
// S_b falls below 1e-20 (every logit far below o) is flagged; the host drop-in then reruns the
// step with per-row offsets (no update was applied: the dW epilogue skips a failed step).
//
//   FwdEpi       rows = batch rows b, cols = buffered classes j: cos tile -> margin + filter
//                mask -> E (bf16, per-warp TMA stores) + per-(row, column slice) sums of E.
//   DxPartEpi    rows = batch rows, cols = dims: split-K partials of sum_j E_bj w^_j.
//   DwUpdateEpi  rows = classes, cols = dims (2-CTA cluster owns both 256-dim halves of a class
//                block): dwt = sum_b E_bj (rowscale_b x^_b) + positive correction;
//                center_proj = w^ . dwt (half-dots exchanged through DSMEM); dW and the fused
//                momentum-SGD of the sampled rows (shardsim.hpp:139-159, 377-384).
//   DwStoreEpi   fp32 validation engine: stores dwt; dw_rows_update_kernel finishes the rows.
#pragma once
#include <utility>
#include <type_traits>

#include "common.cuh"
#include "gemm.cuh"

namespace pfc {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ bool status_failed(const StepStatus* st) {
  return st->label_oob || st->capacity_shard >= 0 ||
         st->masked_row != 0x7fffffff || st->nonfinite_loss || st->nonfinite_dx ||
         st->underflow_row != 0x7fffffff;
}

__device__ __forceinline__ void pack_bf16x32(const float (&g)[32], uint32_t (&w)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
    w[i] = *reinterpret_cast<const uint32_t*>(&h);
  }
}
__device__ __forceinline__ float round_to(const __nv_bfloat16*, float v) {
  return __bfloat162float(__float2bfloat16_rn(v));
}
__device__ __forceinline__ float round_to(const float*, float v) { return v; }
__device__ __forceinline__ float round_to(const tf32_t*, float v) { return to_tf32(v); }
__device__ __forceinline__ void store_out1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ void store_out1(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_out1(tf32_t* p, float v) { p->v = to_tf32(v); }

struct NoSetup {
  static constexpr int kCluster = 1;
  static constexpr int kExtraSmem = 0;  // CTA-shared epilogue bytes past the NWG per-WG areas
  static constexpr bool kNext = false;  // true: run_next() also receives the next tile's Pre
  __device__ __forceinline__ void setup(uint8_t*) const {}
};

// ------------------------------------------------------------------------------------ FwdEpi
#ifndef PFC_FWD_STBUF
#define PFC_FWD_STBUF 1
#endif
template <typename ST, typename OT, bool kFilter, bool kTma>
struct alignas(64) FwdEpi : NoSetup {
  static constexpr int kStageBufs = PFC_FWD_STBUF;  // E^T staging buffers per warp (TMA store in flight)
  static constexpr int kWarpBytes = kStageBufs * 2048;  // [32 classes][64 B] each
  static constexpr int kSmem = kTma ? 4 * kWarpBytes : 0;
  CUtensorMap tm;   // E^T store map: inner = b (box 32, SWIZZLE_64B), outer = classes (box 32)
  int B, ncols, lde;  // lde = row stride of E^T (>= B)
  const int32_t* pos_col;
  MarginDev mg;
  float tau;
  ST* part_s;       // [n_tiles * NWG][B]: sum of E per row and column slice
  double* zpos;     // [B] margined positive logit (rows whose positive is local)
  double* cpos;     // [B] cosine of the positive
  float* epos;      // [B] E of the positive as stored (after OT rounding)
  int* hasval;      // [B] 1 when the row has an unmasked column (filter only)
  OT* E;            // E^T [ncols][lde]: class-major, so the dW GEMM streams whole class blocks
  const float* offr;  // [B] per-row softmax offset o_b (exact mode), nullptr: the fixed mg.off
  float* dbgz;      // [B][ncols] debug export of z (masked: -inf), nullptr: off

  struct Pre {};
  __device__ __forceinline__ Pre preload(const TileInfo&, int, int) const { return {}; }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int, const Pre&) const {}
  __device__ __forceinline__ void finish(int row, int) const {
    if constexpr (kTma) {
      if ((row & 31) == 0) pfc_sm100::bulk_wait_all();
    }
  }

  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t* smem, const Pre&) const {
    constexpr int CW = BN / NWG;
    const int b = t.row0 + row;
    const bool rv = b < B;
    const int pc = rv ? pos_col[b] : -1;
    const float A = mg.s * kLog2e;
    const float O = (offr && rv ? offr[b] : mg.off) * kLog2e;  // this thread's row
    const double offd = offr && rv ? (double)offr[b] : mg.offd;
    const int wig = row >> 5, lane = row & 31;
    // fragment-path rows of this thread: t/4 + 8h (ra) and 16 + t/4 + 8h (rb) of the warp's 32
    float Of[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int bf = t.row0 + wig * 32 + (k >> 1) * 16 + (lane >> 2) + (k & 1) * 8;
      Of[k] = (offr && bf < B ? offr[bf] : mg.off) * kLog2e;
    }
    uint8_t* stage = smem + wig * kWarpBytes;
    ST sum = ST(0);
    bool any = false;
    int kk = 0;
    // fragment path (tcgen05 engine, no filter): per-thread partial sums of rows t/4, t/4 + 8,
    // 16 + t/4, 24 + t/4 of the warp's 32 rows (t = lane)
    float qs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32, ++kk) {
      const int colb = t.col0 + c0;
      if (colb >= ncols) {  // uniform: past the buffer (an empty group keeps the TMA ring even)
        if (kTma && lane == 0) pfc_sm100::bulk_commit();
        continue;
      }
      if constexpr (kTma && std::is_same<ST, float>::value && !kFilter) {
        // 32 valid negatives in every row of the warp: read the accumulator in the MMA-fragment
        // layout (tcgen05.ld 16x256b), whose bf16x2 pairs are stmatrix.trans operands, so the
        // E^T staging needs no shuffles (stmatrix stores class rows of 8 b values)
        if (__all_sync(0xffffffffu, dbgz == nullptr && colb + 32 <= ncols && (unsigned)(pc - colb) >= 32u)) {
          uint32_t ra[16], rb[16];
          pfc_sm100::tmem_ld_16x256b_x4(src.taddr + (uint32_t)c0, ra);
          pfc_sm100::tmem_ld_16x256b_x4(src.taddr + (16u << 16) + (uint32_t)c0, rb);
          pfc_sm100::tmem_wait_ld();
          uint32_t pa[8], pb[8];  // [2j + h]: rows (h ? t/4 + 8 : t/4) (+16 for pb), classes 8j..
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int j = i >> 1, h = i & 1;
            const float a0 = pfc_sm100::ex2_approx(fmaf(__uint_as_float(ra[4 * j + 2 * h]), A, -Of[h]));
            const float a1 = pfc_sm100::ex2_approx(fmaf(__uint_as_float(ra[4 * j + 2 * h + 1]), A, -Of[h]));
            const float b0 = pfc_sm100::ex2_approx(fmaf(__uint_as_float(rb[4 * j + 2 * h]), A, -Of[2 + h]));
            const float b1 = pfc_sm100::ex2_approx(fmaf(__uint_as_float(rb[4 * j + 2 * h + 1]), A, -Of[2 + h]));
            qs[h] += a0 + a1;
            qs[2 + h] += b0 + b1;
            __nv_bfloat162 x = __floats2bfloat162_rn(a0, a1), y = __floats2bfloat162_rn(b0, b1);
            pa[i] = *reinterpret_cast<uint32_t*>(&x);
            pb[i] = *reinterpret_cast<uint32_t*>(&y);
          }
          uint8_t* sb = stage + (kk % kStageBufs) * 2048;
          if (lane == 0) pfc_sm100::bulk_wait_read<kStageBufs - 1>();  // this buffer's last store
          __syncwarp();
          // stmatrix j: matrices i = (rows 0-7, 8-15, 16-23, 24-31) x classes 8j..8j+7; thread
          // 8i + r addresses class row 8j + r, b chunk i (16 B, swizzled by the class row)
          const int mi = lane >> 3, mr = lane & 7;
          const uint32_t sbase = pfc_sm100::smem_u32(sb);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int q = 8 * j + mr;
            pfc_sm100::stmatrix_x4_trans(sbase + q * 64 + ((mi ^ ((q >> 1) & 3)) << 4), pa[2 * j],
                                         pa[2 * j + 1], pb[2 * j], pb[2 * j + 1]);
          }
          pfc_sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            pfc_sm100::tma_store_2d(&tm, sb, t.row0 + wig * 32, colb);
            pfc_sm100::bulk_commit();
          }
          any = true;
          continue;
        }
      }
      float v[32];
      src.load(c0, v);
      float e[32];
      const int jp = pc - colb;
      bool done = false;
      if constexpr (std::is_same<ST, float>::value && !kFilter) {
        if (dbgz == nullptr && colb + 32 <= ncols && (unsigned)jp >= 32u) {  // 32 valid negatives
          float s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int q = 0; q < 32; q += 2) {
            e[q] = pfc_sm100::ex2_approx(fmaf(v[q], A, -O));
            e[q + 1] = pfc_sm100::ex2_approx(fmaf(v[q + 1], A, -O));
            s1 += e[q];
            s2 += e[q + 1];
          }
          sum += s1 + s2;
          any = true;
          done = true;
        }
      }
      if (!done) {
        // bounds, filter mask (shardsim.hpp:258-268), the positive's margin (margin.hpp:41-54)
        ST acc = ST(0);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const bool masked = (colb + q >= ncols) || (kFilter && q != jp && v[q] > tau);
          ST eq;
          if constexpr (std::is_same<ST, float>::value)
            eq = pfc_sm100::ex2_approx(fmaf(v[q], A, -O));
          else
            eq = exp((double)mg.s * (double)v[q] - offd);
          eq = masked ? ST(0) : eq;
          if (dbgz && rv && colb + q < ncols)  // debug export of the logit the softmax used
            dbgz[(size_t)b * ncols + colb + q] = masked ? -INFINITY : mg.s * v[q];
          any = any || !masked;
          e[q] = (float)eq;
          if (q != jp) acc += eq;
        }
        if ((unsigned)jp < 32u) {
          float vp = 0.f;
#pragma unroll
          for (int q = 0; q < 32; ++q) vp = (q == jp) ? v[q] : vp;
          const double zp = margin_pos(mg, (double)vp);
          const double ep = exp(zp - offd);
          if (dbgz && rv) dbgz[(size_t)b * ncols + colb + jp] = (float)zp;
          const float eps = round_to(E, (float)ep);
          zpos[b] = zp;
          cpos[b] = (double)vp;
          epos[b] = eps;
          acc += (ST)ep;
#pragma unroll
          for (int q = 0; q < 32; ++q) e[q] = (q == jp) ? (float)ep : e[q];
        }
        sum += acc;
      }
      if constexpr (kTma) {
        // transposed staging: E^T chunk [32 classes][32 rows b] (64 B per class, 64B swizzle)
        uint8_t* sb = stage + (kk % kStageBufs) * 2048;
        if (lane == 0) pfc_sm100::bulk_wait_read<kStageBufs - 1>();  // this buffer's last store
        __syncwarp();
        // element (class q, row b) lives at byte q*64 + b*2, its 16-byte chunk swizzled by q.
        // Lanes b, b^1 swap halves of their packed (q, q+1) pairs so that each stores one
        // 4-byte (rows b&~1, b|1) pair: the even lane class q, the odd lane class q+1.
        const bool odd = lane & 1;
        const int b0 = lane & ~1;
#pragma unroll
        for (int q = 0; q < 32; q += 2) {
          __nv_bfloat162 own = __floats2bfloat162_rn(rv ? e[q] : 0.f, rv ? e[q + 1] : 0.f);
          const uint32_t ou = *reinterpret_cast<uint32_t*>(&own);
          const uint32_t nu = __shfl_xor_sync(0xffffffffu, ou, 1);
          // even: (own.lo, nb.lo) = class q rows (b, b+1); odd: (nb.hi, own.hi) = class q+1
          const uint32_t packed = odd ? __byte_perm(nu, ou, 0x7632) : __byte_perm(ou, nu, 0x5410);
          const int qq = q + (odd ? 1 : 0);
          const int chunk = (b0 >> 3) ^ ((qq >> 1) & 3);
          *reinterpret_cast<uint32_t*>(sb + qq * 64 + chunk * 16 + (b0 & 7) * 2) = packed;
        }
        pfc_sm100::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          pfc_sm100::tma_store_2d(&tm, sb, t.row0 + wig * 32, colb);
          pfc_sm100::bulk_commit();
        }
      } else if (rv) {
        // E^T[class][b] (fp32 validation engine)
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (colb + q < ncols) store_out1(E + (size_t)(colb + q) * lde + b, e[q]);
      }
    }
    if constexpr (kTma && std::is_same<ST, float>::value && !kFilter) {
      // fragment-path sums: reduce over the quad, then row r (lane r) takes slot r / 8 of quad r % 8
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        qs[k] += __shfl_xor_sync(0xffffffffu, qs[k], 1);
        qs[k] += __shfl_xor_sync(0xffffffffu, qs[k], 2);
      }
      float mine = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float v = __shfl_sync(0xffffffffu, qs[k], (lane & 7) * 4);
        mine = (lane >> 3) == k ? v : mine;
      }
      sum += mine;
    }
    if (rv) {
      part_s[(size_t)(t.n_tile * NWG + wg) * B + b] = sum;
      if (kFilter && any) hasval[b] = 1;
    }
  }
};

// ------------------------------------------------------------------------------------ MaxEpi
// Max-only pass of the per-row offset mode (same GEMM geometry as FwdEpi): per (row, column
// slice) the largest unmasked negative cosine (fp32, -inf if none; the filter rule of
// shardsim.hpp:258-268), and for a local positive its margined logit z_pos (fp64,
// margin.hpp:41-54) -- the local max of shardsim.hpp:270-281 up to the scale s.
template <bool kFilter>
struct MaxEpi : NoSetup {
  static constexpr int kSmem = 0;
  int B, ncols;
  const int32_t* pos_col;
  MarginDev mg;
  float tau;
  float* part_m;  // [n_tiles * NWG][B]
  double* zpos;   // [B]
  struct Pre {};
  __device__ __forceinline__ Pre preload(const TileInfo&, int, int) const { return {}; }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int, const Pre&) const {}
  __device__ __forceinline__ void finish(int, int) const {}
  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t*, const Pre&) const {
    constexpr int CW = BN / NWG;
    const int b = t.row0 + row;
    const bool rv = b < B;
    const int pc = rv ? pos_col[b] : -1;
    float mx = -INFINITY;
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32) {
      const int colb = t.col0 + c0;
      if (colb >= ncols) continue;  // uniform
      float v[32];
      src.load(c0, v);
      const int jp = pc - colb;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const bool use = colb + q < ncols && q != jp && !(kFilter && v[q] > tau);
        mx = use ? fmaxf(mx, v[q]) : mx;
      }
      if ((unsigned)jp < 32u) {
        float vp = 0.f;
#pragma unroll
        for (int q = 0; q < 32; ++q) vp = (q == jp) ? v[q] : vp;
        zpos[b] = margin_pos(mg, (double)vp);
      }
    }
    if (rv) part_m[(size_t)(t.n_tile * NWG + wg) * B + b] = mx;
  }
};

// --------------------------------------------------------------------------------- DxPartEpi
struct DxPartEpi : NoSetup {
  static constexpr int kSmem = 0;
  int B, D;
  float* part;  // [splits][B][D]
  struct Pre {};
  __device__ __forceinline__ Pre preload(const TileInfo&, int, int) const { return {}; }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int, const Pre&) const {}
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

// ------------------------------------------------------------------------------- DwUpdateEpi
// Four epilogue warpgroups (16 warps).  The update is a gathered-row stream (W and momentum read
// + write) whose speed is set by the bytes in flight per SM (profiles/micro/rowupd.cu: 16 warps
// with 6 KB each in flight reach 6.2 TB/s, 8 warps with 1.5 KB 3.3 TB/s).  Registers cannot hold
// that much next to the TMEM chunk, so each warp streams its rows through a 6 KB cp.async ring
// in shared memory: a compile-time greedy schedule keeps it full across both passes of a tile
// (the update pass's loads are in flight during the dot pass and the half-dot exchange).
//
// Each CTA owns a 256-dim half of a 128-class block; warp (g, q) owns the 8 rows 32q + 8g .. +7
// of TMEM lane quadrant q over all 256 dims, so a row's CTA-local half-dot is warp-local.  With
// kPair (D = 512) the two CTAs of a 2-CTA cluster own the two halves and swap half-dots warp by
// warp (st.async into the peer's shared memory, completing its per-warp mbarrier).
#ifndef PFC_DW_CAP
#define PFC_DW_CAP 6
#endif
#ifndef PFC_DW_EXP
#define PFC_DW_EXP 0  // timing probes of the update epilogue (profiles/micro/dwexp.sh); 0 = product
#endif
namespace dw_ring {
constexpr int kNC = 8;                      // 32-dim chunks per 256-dim tile half
constexpr int kItems = 2 * kNC;             // W chunk c (dot pass), then W + momentum chunk c
constexpr int kTileSlots = kNC * 1 + kNC * 2;
__host__ __device__ constexpr int size(int i) { return (i % kItems) < kNC ? 1 : 2; }
// Cap: ring capacity in 1 KB sub-slots (8 rows x 128 B)
template <int Cap>
struct Ring {
  static constexpr int kCap = Cap;
  static_assert(kTileSlots % kCap == 0, "ring positions must repeat every tile");
  __host__ __device__ static constexpr int pos(int i) {  // first sub-slot of item i
    int p = 0;
    for (int j = 0; j < i % kItems; ++j) p += size(j);
    return p % kCap;
  }
  // Greedy issue over the endless item stream (tile after tile): items issued before item k is
  // consumed, in steady state (the previous tile already issued this tile's first items).
  __host__ __device__ static constexpr int issued_before(int k) {
    int issued = 0, used = 0;
    for (int c = 0;; ++c) {
      while (issued < 3 * kItems && used + size(issued) <= kCap) used += size(issued++);
      if (c == kItems + k) return issued - kItems;
      used -= size(c);
    }
  }
  static constexpr int kHead = issued_before(0);  // items of a tile in flight when it starts
  static_assert(issued_before(kItems) - kItems == kHead, "periodic steady state");
};
// compile-time loop: f(std::integral_constant<int, I>) for I in [A, B)
template <int A, int B, class F>
__device__ __forceinline__ void static_range(F&& f) {
  if constexpr (A < B) {
    f(std::integral_constant<int, A>{});
    static_range<A + 1, B>(f);
  }
}
}  // namespace dw_ring

// NC: CTAs per class block (a cluster): the dim blocks of 256 (D <= 256 * NC, up to 1024).  Each
// CTA sends its rows' partial dots to the other NC - 1 and sums all NC in cluster-rank order, so
// every CTA of the cluster forms the same center_proj.
// Cap: the W / momentum ring per warp in KB (6 with 2 operand stages at B <= 1024; 3 with 3
// stages when the GEMM's K = B is larger and its operand stream needs the deeper pipeline).
struct DwHalfMap {
  CUtensorMap tm_a16;  // E^T K-major, 16-row boxes (the producer's half-tile A loads)
};
struct DwNoHalfMap {};
template <int NC, int Cap = PFC_DW_CAP, bool Half = false>
struct DwUpdateEpi : std::conditional_t<Half, DwHalfMap, DwNoHalfMap> {
  static_assert(NC >= 1 && NC <= 4, "DwUpdateEpi: 1-4 dim blocks");
  static constexpr bool kPair = NC > 1;
  // half tiles (the schedule's tail, GemmGeom::half_m0): 64 class rows, 16 at the top of each
  // TMEM lane quadrant, 4 per warp (lanes 4 wg .. 4 wg + 3) instead of 8
  // (a separate instantiation: the full-tile schedule keeps the plain 8-rows-per-warp path)
  static constexpr bool kHalfTiles = Half;
  static constexpr int kCluster = NC;
  static constexpr bool kNext = true;
  static constexpr int kStageFloats = 8 * 36;             // TMEM chunk of the warp's 8 rows
  using R = dw_ring::Ring<Cap>;
  static constexpr int kRingFloats = Cap * 256;  // Cap x 1 KB
  static constexpr int kWarpFloats = kStageFloats + kRingFloats + 2 * 3 * 8;  // + [2][inv|row|pslot]
  static constexpr int kWarpBytes = kWarpFloats * 4;
  // CTA-shared (in warpgroup 0's scratch): hrem[2 parity][NC source rank][128 rows] + mbarriers
  // [2][16 warps]
  static constexpr int kHremFloats = 2 * NC * 128;
  static constexpr int kSharedBytes = kHremFloats * 4 + 2 * 16 * 8;
  static constexpr int kSmem = ((4 * kWarpBytes + 127) / 128) * 128;  // per warpgroup
  static constexpr int kExtraSmem = ((kSharedBytes + 127) / 128) * 128;  // once, after all 4
  int ncols, D;
  const float* wnorm;       // [ncols]
  const int32_t* lrow;      // [ncols] local row of W
  const int32_t* pslot;     // [ncols] positive-correction slot or -1
  const float* poscorr;     // [slots][D]: sum over rows with this label of delta_b x^_b
  float* W;
  float* Mom;
  const StepParams* sp;     // lr of this step
  float mu, wd;
  const StepStatus* st;     // no update when the step failed (the reference throws before 412)

  struct Pre {
    float inv;
    int r, ps;
    int li;  // this lane's row slot among the warp's rows, -1: not one of them
  };
  // lane -> row of a tile: full tiles 32 q + lane (warp wg: lanes 8 wg ..), half tiles 16 q + lane
  // for lane < 16 (warp wg: lanes 4 wg ..)
  __device__ __forceinline__ static int slot_of(const TileInfo& t, int lane, int wg) {
    if (!Half || t.h == 128) return (lane >> 3) == wg ? (lane & 7) : -1;
    return (lane < 16 && (lane >> 2) == wg) ? (lane & 3) : -1;
  }
  __device__ __forceinline__ Pre preload(const TileInfo& t, int row, int wg) const {
    Pre p{0.f, -1, -1, -1};
    const int lane = row & 31, q = row >> 5;
    const int c = t.row0 + ((!Half || t.h == 128) ? 32 : 16) * q + lane;
    p.li = slot_of(t, lane, wg);
    if (p.li >= 0 && c < ncols) {  // only this warp's rows
      const float n = wnorm[c];
      p.inv = 1.0f / (n > 1e-12f ? n : 1e-12f);
      p.r = lrow[c];
      p.ps = pslot[c];
    }
    return p;
  }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int, const Pre&) const {}
  __device__ __forceinline__ void finish(int, int) const {}

  __device__ __forceinline__ static uint8_t* shared_area(uint8_t* wg0) { return wg0 + 4 * kSmem; }
  __device__ __forceinline__ void setup(uint8_t* epi_base) const {
    if constexpr (kPair) {
      uint64_t* mb = reinterpret_cast<uint64_t*>(shared_area(epi_base) + kHremFloats * 4);
      for (int k = 0; k < 32; ++k) pfc_sm100::mbar_init(&mb[k], 1);  // local arrive + tx bytes
    }
  }

  // The ring runs across tiles: the end of tile i issues tile i+1's first loads (its rows come
  // from pre_next), so the ring never drains at a tile boundary.  The CTA's dims half (col0) is
  // the same for all its tiles (the tile stride is a multiple of n_tiles).
  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run_next(const TileInfo& t, const Src& src, int row, int wg,
                                           uint8_t* smem, const Pre& pre, const Pre& pre_next,
                                           bool has_next) const {
    static_assert(NWG == 4 && BN == 256, "DwUpdateEpi: 4 warpgroups, 256-dim tiles");
    using namespace dw_ring;
    constexpr int kCap = R::kCap, kHead = R::kHead;
    const int q = row >> 5, lane = row & 31;
    uint8_t* wg0 = smem - wg * kSmem;
    float* ws = reinterpret_cast<float*>(smem + q * kWarpBytes);
    float* stage = ws;                          // [8 rows][36]
    float* ring = ws + kStageFloats;            // [6 sub-slots][8 rows][32]
    float* sc = ring + kRingFloats;             // [2 tile parity][inv 8 | row 8 | pslot 8]
    float* s_inv = sc + (t.iter & 1) * 24;
    int* s_row = reinterpret_cast<int*>(s_inv + 8);
    int* s_ps = s_row + 8;
    int* s_row_n = reinterpret_cast<int*>(sc + ((t.iter & 1) ^ 1) * 24 + 8);
    float* hrem = reinterpret_cast<float*>(shared_area(wg0));                      // [2][NC][128]
    uint64_t* mb = reinterpret_cast<uint64_t*>(shared_area(wg0) + kHremFloats * 4);  // [2][16]
    const bool failed = status_failed(st);
    const float lr = sp->lr;
    const int li = slot_of(t, lane, wg);
    const bool mine = li >= 0;  // this lane's TMEM row is one of the warp's rows
    float* sn = sc + ((t.iter & 1) ^ 1) * 24;
    __syncwarp();  // the warp finished with the previous tile's scalars
    if constexpr (Half) {
      if (lane < 8) {  // slots a half tile leaves empty stay invalid rows
        if (t.iter == 0) {
          s_inv[lane] = 0.f;
          s_row[lane] = -1;
          s_ps[lane] = -1;
        }
        sn[lane] = 0.f;
        reinterpret_cast<int*>(sn)[8 + lane] = -1;
        reinterpret_cast<int*>(sn)[16 + lane] = -1;
      }
      __syncwarp();
    }
    if constexpr (Half) {  // each tile's own lane -> slot map (the slots were cleared above)
      if (t.iter == 0 && pre.li >= 0) {  // later tiles' scalars were stored by the tile before
        s_inv[pre.li] = pre.inv;
        s_row[pre.li] = failed ? -1 : pre.r;
        s_ps[pre.li] = pre.ps;
      }
      if (has_next && pre_next.li >= 0) {
        sn[pre_next.li] = pre_next.inv;
        reinterpret_cast<int*>(sn)[8 + pre_next.li] = failed ? -1 : pre_next.r;
        reinterpret_cast<int*>(sn)[16 + pre_next.li] = pre_next.ps;
      }
    } else if (mine) {  // full tiles only: one map, every slot of the warp written
      if (t.iter == 0) {  // later tiles' scalars were stored by the tile before them
        s_inv[li] = pre.inv;
        s_row[li] = failed ? -1 : pre.r;
        s_ps[li] = pre.ps;
      }
      sn[li] = pre_next.inv;
      reinterpret_cast<int*>(sn)[8 + li] = (failed || !has_next) ? -1 : pre_next.r;
      reinterpret_cast<int*>(sn)[16 + li] = pre_next.ps;
    }
    __syncwarp();
    // lanes run along dims: 8 lanes x float4 per row, rows u*4 + sub (u = 0, 1)
    const int sub = lane >> 3, q4 = (lane & 7) * 4;
    int rw[2], ps[2], rwn[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      rw[u] = s_row[u * 4 + sub];
      ps[u] = s_ps[u * 4 + sub];
      rwn[u] = s_row_n[u * 4 + sub];
    }
    const int dbase = t.col0 + q4;
#if PFC_DW_EXP == 3  // timing probe: no positive corrections (wrong values)
    const bool anyp = false;
#else
    const bool anyp = __any_sync(0xffffffffu, ps[0] >= 0 || ps[1] >= 0);  // positives are rare
#endif
    if constexpr (kPair) {  // this tile's exchange: each peer's 8 partial dots arrive as 32 tx bytes
      if (lane == 0)
        pfc_sm100::mbar_arrive_expect_tx(&mb[(t.iter & 1) * 16 + wg * 4 + q], 32u * (NC - 1));
    }
    // this lane's 16-byte piece of row (u*4+sub) in ring sub-slot p
    const uint32_t ring_s = pfc_sm100::smem_u32(ring);
    auto slot_off = [&](int p, int u) { return (uint32_t)((p * 256 + (u * 4 + sub) * 32 + q4) * 4); };
    // item i of the stream: W chunk c (i % 16 < 8) or W + momentum chunk c of this tile
    // (i < 16) or of the next one (i >= 16; an empty group when there is none)
    auto issue = [&](auto ic) {
      constexpr int i = decltype(ic)::value;
      constexpr int ii = i % kItems;
      constexpr int c = ii < kNC ? ii : ii - kNC;
      constexpr int p = R::pos(i);
      const int d = dbase + c * 32;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = i < kItems ? rw[u] : rwn[u];
        if (r >= 0 && d < D) {
          const size_t o = (size_t)r * D + d;
          pfc_sm100::cp_async16(ring_s + slot_off(p, u), W + o);
          if (ii >= kNC) pfc_sm100::cp_async16(ring_s + slot_off((p + 1) % kCap, u), Mom + o);
        }
      }
      pfc_sm100::cp_async_commit();
    };
    auto ring4 = [&](int p, int u) {
      return *reinterpret_cast<const float4*>(ring + p * 256 + (u * 4 + sub) * 32 + q4);
    };
    auto stage_chunk = [&](int c0) {
      __syncwarp();
      float v0[16], v1[16];
      src.load16x2(c0, v0, v1);  // 32 columns, one TMEM round trip
#if PFC_DW_EXP != 6  // timing probe 6: no staging stores (wrong values)
      if (mine) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          *reinterpret_cast<float4*>(stage + li * 36 + 4 * j) =
              make_float4(v0[4 * j], v0[4 * j + 1], v0[4 * j + 2], v0[4 * j + 3]);
          *reinterpret_cast<float4*>(stage + li * 36 + 16 + 4 * j) =
              make_float4(v1[4 * j], v1[4 * j + 1], v1[4 * j + 2], v1[4 * j + 3]);
        }
      }
#else
      if (v0[0] == 1234.5f && v1[3] == 7.f) stage[li] = 0.f;
#endif
      __syncwarp();
    };
    auto dwt4 = [&](int u, int d) {
      float4 r = *reinterpret_cast<const float4*>(stage + (u * 4 + sub) * 36 + q4);
      if (anyp) {
        if (ps[u] >= 0) {
          const float4 pc = *reinterpret_cast<const float4*>(poscorr + (size_t)ps[u] * D + d);
          r.x += pc.x; r.y += pc.y; r.z += pc.z; r.w += pc.w;
        }
      }
      return r;
    };

    if (t.iter == 0) static_range<0, kHead>(issue);  // otherwise issued by the previous tile
    float dot[2] = {0.f, 0.f}, rcp[2] = {0.f, 0.f}, rinv[2] = {0.f, 0.f};
    static_range<0, kItems>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      constexpr int c = k < kNC ? k : k - kNC;
      const int d = dbase + c * 32;
      if constexpr (k == kNC) {
        // ---- dot pass done: reduce, exchange half-dots with the peer CTA, center_proj
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], 1);
          dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], 2);
          dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], 4);
        }
        if constexpr (kPair) {
          const int it = t.iter, par = it & 1, e = wg * 4 + q;
          const uint32_t me = pfc_sm100::cluster_ctarank();
          // this warp's 8 rows in the slot of source rank r: hrem[par][r][q*32 + wg*8 + ...]
          auto slot = [&](uint32_t r) { return hrem + (par * NC + (int)r) * 128 + q * 32 + wg * 8; };
          if ((lane & 7) == 0) {
#pragma unroll
            for (int pr = 1; pr < NC; ++pr) {
              const uint32_t peer = (me + (uint32_t)pr) % (uint32_t)NC;
              const uint32_t rbar = pfc_sm100::mapa_shared(pfc_sm100::smem_u32(&mb[par * 16 + e]), peer);
#pragma unroll
              for (int u = 0; u < 2; ++u)
                pfc_sm100::st_async_f32(pfc_sm100::mapa_shared(pfc_sm100::smem_u32(slot(me) + u * 4 + sub), peer),
                                        dot[u], rbar);
            }
          }
#if PFC_DW_EXP != 4  // timing probe 4: no wait for the peers' partial dots (wrong values)
          pfc_sm100::mbar_wait_cluster(&mb[par * 16 + e], (uint32_t)((it >> 1) & 1));
#endif
          // every CTA sums the NC partial dots in rank order: the same center_proj everywhere
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            float tot = 0.f;
#pragma unroll
            for (int r = 0; r < NC; ++r) tot += r == (int)me ? dot[u] : slot((uint32_t)r)[u * 4 + sub];
            dot[u] = tot;
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          rinv[u] = s_inv[u * 4 + sub];
          rcp[u] = dot[u] * rinv[u];  // center_proj_j = w^_j . dwt_j (shardsim.hpp:361-362)
        }
      }
      pfc_sm100::cp_async_wait<R::issued_before(k) - k - 1>();  // item k landed (this lane's pieces)
      stage_chunk(c * 32);
      if (d < D) {
        if constexpr (k < kNC) {  // dot pass: half-dot w . dwt over this CTA's dims
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const float4 a = dwt4(u, d);
            const float4 w = ring4(R::pos(k), u);
            dot[u] += a.x * w.x + a.y * w.y + a.z * w.z + a.w * w.w;
          }
        } else {  // update pass: dW and the momentum-SGD update of the sampled rows
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (rw[u] < 0) continue;
            const float4 a4 = dwt4(u, d);
            const float4 w4 = ring4(R::pos(k), u), m4 = ring4((R::pos(k) + 1) % kCap, u);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w};
            float wv[4] = {w4.x, w4.y, w4.z, w4.w};
            float mv[4] = {m4.x, m4.y, m4.z, m4.w};
            const float inv = rinv[u], cpj = rcp[u];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float dw = (av[e] - cpj * (wv[e] * inv)) * inv;  // shardsim.hpp:382
              const float g = dw + wd * wv[e];                      // shardsim.hpp:152-153
              const float vv = mu * mv[e] + g;                      // shardsim.hpp:154
              mv[e] = vv;
              wv[e] = wv[e] - lr * vv;                              // shardsim.hpp:156
            }
            const size_t o = (size_t)rw[u] * D + d;
#if PFC_DW_EXP == 2  // timing probe: no W / momentum stores
            if (mv[0] == 1234.5f)
#endif
            {
#if PFC_DW_EXP == 5  // probe: streaming (evict-first) stores
            __stcs(reinterpret_cast<float4*>(Mom + o), make_float4(mv[0], mv[1], mv[2], mv[3]));
            __stcs(reinterpret_cast<float4*>(W + o), make_float4(wv[0], wv[1], wv[2], wv[3]));
#else
            *reinterpret_cast<float4*>(Mom + o) = make_float4(mv[0], mv[1], mv[2], mv[3]);
            *reinterpret_cast<float4*>(W + o) = make_float4(wv[0], wv[1], wv[2], wv[3]);
#endif
            }
          }
        }
      }
      // refill the ring (reads of item k's sub-slots were consumed above: in-order issue)
      static_range<R::issued_before(k), R::issued_before(k + 1)>(issue);
    });
  }
};

// -------------------------------------------------------------------- DwStoreEpi (SIMT path)
struct DwStoreEpi : NoSetup {
  static constexpr int kSmem = 0;
  int ncols, D;
  float* dwt;  // [ncols][D]
  struct Pre {};
  __device__ __forceinline__ Pre preload(const TileInfo&, int, int) const { return {}; }
  __device__ __forceinline__ void prefetch(const TileInfo&, int, int, const Pre&) const {}
  __device__ __forceinline__ void finish(int, int) const {}
  template <int BN, int NWG, class Src>
  __device__ __forceinline__ void run(const TileInfo& t, const Src& src, int row, int wg,
                                      uint8_t*, const Pre&) const {
    constexpr int CW = BN / NWG;
    const int j = t.row0 + row;
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32) {
      float v[32];
      src.load(c0, v);
      const int d0 = t.col0 + c0;
      if (j >= ncols || d0 >= D) continue;
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (d0 + q < D) dwt[(size_t)j * D + d0 + q] = v[q];
    }
  }
};

}  // namespace pfc
