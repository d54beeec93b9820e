// gemm.cuh — the two GEMM engines of the hot path.
//
//  * umma_gemm_kernel: persistent, warp-specialised tcgen05 GEMM for sm_100a.
//      warp 0      : TMA producer (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier complete_tx)
//      warp 1      : single-thread tcgen05.mma issuer (kind::f16, bf16 in, fp32 accum in TMEM)
//                    and TMEM allocator (2 x BN columns: double-buffered accumulators)
//      warps 2..   : NWG epilogue warpgroups; warp w reads TMEM lane quadrant w % 4
//                    (tcgen05.ld 32x32b -> registers -> fused epilogue functor)
//    Tile = 128 x BN, BK = 64, STAGES-deep smem ring.  A and B may each be K-major or
//    MN-major (UMMA descriptor transpose bits), so one gathered centre block and one
//    normalised feature block serve all three GEMMs of the step without transposes.
//  * simt_gemm_kernel: fp32 CUDA-core GEMM used by the fp32 validation mode; it feeds the
//    SAME epilogue functors (thread = accumulator row, 32-column chunks), BN = 64.
#pragma once
#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace pfc {

struct TileInfo {
  int m_tile, n_tile, split;
  int row0, col0;
  int kb0, kb1;
  int iter;  // this CTA's tile counter (0, 1, 2, ...)
  int h;     // valid rows: BM, or BM / 2 for a half tile (16 rows at the top of each TMEM
             // lane quadrant; the dW GEMM's tail, GemmGeom::half_m0)
};

// Epi::kHalfTiles (optional, false when absent): the GEMM may be given half tiles, whose A rows
// the producer loads through Epi::tm_a16 (16-row boxes)
template <class E, class = void>
struct kHalfTilesOf : std::false_type {};
template <class E>
struct kHalfTilesOf<E, std::void_t<decltype(E::kHalfTiles)>> : std::bool_constant<E::kHalfTiles> {};

struct GemmGeom {
  int M, N, K;
  int m_tiles, n_tiles, splits, kb_per_split, kb_total;
  int n_fastest;  // tile order: 0 -> m fastest, 1 -> n fastest
  int BN, BK;
  int BM;         // 128, or 256 for a CTA-pair GEMM (the kernel adds 128 x cluster rank)
  int half_m0;    // m tiles from here on are half tiles of BM / 2 rows (m_tiles: none)
  __host__ __device__ int total() const { return m_tiles * n_tiles * splits; }
  // kHalf: the GEMM may have half tiles (half_m0 < m_tiles); without it every tile is BM rows
  template <bool kHalf = false>
  __host__ __device__ TileInfo tile(int t) const {
    TileInfo ti;
    const int mn = m_tiles * n_tiles;
    ti.split = t / mn;
    const int r = t % mn;
    if (n_fastest) {
      ti.n_tile = r % n_tiles;
      ti.m_tile = r / n_tiles;
    } else {
      ti.m_tile = r % m_tiles;
      ti.n_tile = r / m_tiles;
    }
    if constexpr (kHalf) {
      ti.h = ti.m_tile < half_m0 ? BM : BM / 2;
      ti.row0 = ti.m_tile < half_m0 ? ti.m_tile * BM : half_m0 * BM + (ti.m_tile - half_m0) * (BM / 2);
    } else {
      ti.h = BM;
      ti.row0 = ti.m_tile * BM;
    }
    ti.col0 = ti.n_tile * BN;
    ti.kb0 = ti.split * kb_per_split;
    ti.kb1 = ti.kb0 + kb_per_split < kb_total ? ti.kb0 + kb_per_split : kb_total;
    ti.iter = 0;
    return ti;
  }
};

// BK: K elements per stage (one 128-byte swizzle row: 64 bf16 or 32 tf32 operands)
inline GemmGeom make_geom(int M, int N, int K, int BN, int splits, int n_fastest, int BM = 128,
                          int BK = 64) {
  GemmGeom g{};
  g.BM = BM;
  g.M = M;
  g.N = N;
  g.K = K;
  g.BN = BN;
  g.BK = BK;
  g.m_tiles = (M + BM - 1) / BM;
  g.n_tiles = (N + BN - 1) / BN;
  g.kb_total = (K + BK - 1) / BK;
  if (splits < 1) splits = 1;
  if (splits > g.kb_total) splits = g.kb_total;
  g.kb_per_split = (g.kb_total + splits - 1) / splits;
  g.splits = (g.kb_total + g.kb_per_split - 1) / g.kb_per_split;  // no empty split
  g.n_fastest = n_fastest;
  g.half_m0 = g.m_tiles;
  return g;
}

constexpr int kEpiSmemBytes = 20 * 1024;  // SIMT engine epilogue scratch

template <int BN, int STAGES, int NWG, class Epi, int CG = 1>
constexpr int umma_smem_bytes() {
  return 1024 /*align slack*/ + STAGES * (128 * 64 * 2 + (BN / CG) * 64 * 2) + 1024 /*barriers*/ +
         NWG * Epi::kSmem + Epi::kExtraSmem;
}

struct TmemSrc {
  uint32_t taddr;  // lane field already set for this warp
  __device__ __forceinline__ void load(int c0, float (&v)[32]) const {
    pfc_sm100::tmem_ld32(taddr + (uint32_t)c0, v);
  }
  __device__ __forceinline__ void load16(int c0, float (&v)[16]) const {
    pfc_sm100::tmem_ld16(taddr + (uint32_t)c0, v);
  }
  // 32 columns as two x16 loads behind one wait
  __device__ __forceinline__ void load16x2(int c0, float (&v0)[16], float (&v1)[16]) const {
    uint32_t r0[16], r1[16];
    pfc_sm100::tmem_ld16_nowait(taddr + (uint32_t)c0, r0);
    pfc_sm100::tmem_ld16_nowait(taddr + (uint32_t)c0 + 16u, r1);
    pfc_sm100::tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v0[i] = __uint_as_float(r0[i]);
      v1[i] = __uint_as_float(r1[i]);
    }
  }
};

#ifndef PFC_CTRL_WARPS
#define PFC_CTRL_WARPS 2
#endif
// CG = 1: one CTA per 128 x BN tile.  CG = 2: a CTA pair (2-CTA cluster) per 256 x BN tile with
// tcgen05.mma.cta_group::2 issued by the leader: each CTA loads its own 128 rows of A and BN/2
// rows of B (both signal the leader's full barrier), so per CTA the operand bytes per FLOP drop
// by a third (A 128 + B 128 rows per 128 x BN block instead of 128 + BN); each CTA's TMEM holds
// its 128 accumulator rows, so the epilogue functors are the same as for CG = 1.
// OT: operand type -- __nv_bfloat16 (kind::f16) or float (kind::tf32; the TF32 precision mode).
// Every stage holds one 128-byte swizzle row of K per operand row either way (64 bf16 or 32 fp32
// elements), so the shared-memory layout and the descriptors' byte strides are the same; an
// MN-major atom is 128 B of M/N by one stage of K (8 KB bf16, 4 KB tf32).
template <int BN, int STAGES, int NWG, bool A_MN, bool B_MN, class Epi, int CG = 1,
          class OT = __nv_bfloat16>
__global__ void __launch_bounds__(32 * PFC_CTRL_WARPS + 128 * NWG, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, const GemmGeom g,
                     const __grid_constant__ Epi epi) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using namespace pfc_sm100;
  constexpr bool kTf32 = sizeof(OT) == 4;
  constexpr int KB = 128 / (int)sizeof(OT);          // K elements per stage
  constexpr uint32_t ATOM = 128u * (uint32_t)KB;     // MN-major atom bytes (128 B x KB rows)
  constexpr uint32_t KSTEP = 32u / sizeof(OT) * 128u;  // MN-major bytes per MMA K step
  static_assert(CG == 1 || CG == 2, "CG");
  static_assert(!kTf32 || CG == 1, "the tf32 engine runs single-CTA MMAs");
  static_assert(CG == 1 || Epi::kCluster == 1, "a CTA-pair GEMM has no epilogue cluster");
  constexpr int BNL = BN / CG;  // rows of B this CTA loads
  constexpr uint32_t A_BYTES = 128 * 64 * 2;
  constexpr uint32_t B_BYTES = BNL * 64 * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  // two accumulator buffers at columns 0 and BN; the allocation is a power of two >= 2 BN
  constexpr uint32_t TMEM_COLS = 2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512);
  static_assert(BN % 64 == 0 && BN >= 64 && BN <= 256 && BNL % 64 == 0, "BN");

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B, by pointer arithmetic (keeps the shared state space)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* epi_smem = smem + STAGES * STAGE_BYTES + 1024;  // 1024-aligned per-WG scratch

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      // CG = 1: every epilogue thread arrives locally.  CG = 2: both CTAs' epilogues release the
      // leader, one remote arrive per warp (a cluster-scope release per thread costs a fence each)
      mbar_init(&tempty[i], CG == 2 ? 2 * 4 * NWG : 128 * NWG);
    }
    epi.setup(epi_smem);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair(tmem_slot, TMEM_COLS);
    else tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if constexpr (Epi::kCluster > 1 || CG == 2) cluster_sync_all();  // peer barriers initialised
  pdl_entry();  // the prologue above overlapped the previous kernel's drain
  const uint32_t tmem_base = *tmem_slot;
  const int total = g.total();
  // persistent schedule over tiles (CG = 2: over pair tiles, one per cluster)
  const int first = (int)blockIdx.x / CG, stride = (int)gridDim.x / CG;
  auto tile_at = [&](int t) {
    TileInfo ti = g.template tile<kHalfTilesOf<Epi>::value>(t);
    ti.row0 += (int)rank * 128;
    return ti;
  };

  if (warp == 0) {
    if (lane == 0) {
      uint32_t kbc = 0;
      // CG = 2: the leader expects both CTAs' bytes; the peer's loads complete on it remotely
      const uint32_t full_c = CG == 2 ? mapa_shared(smem_u32(full), 0) : 0u;
      for (int t = first; t < total; t += stride) {
        const TileInfo ti = tile_at(t);
        const int bcol = ti.col0 + (int)rank * BNL;
        const bool half = kHalfTilesOf<Epi>::value && ti.h != g.BM;  // (Epi::kHalfTiles GEMMs only)
        for (int kb = ti.kb0; kb < ti.kb1; ++kb, ++kbc) {
          const uint32_t s = kbc % STAGES, ph = (kbc / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[s], (half ? STAGE_BYTES - A_BYTES / 2 : STAGE_BYTES) * CG);
          const int k0 = kb * KB;
          uint8_t* a = sA + s * A_BYTES;
          uint8_t* b = sB + s * B_BYTES;
          auto load = [&](const CUtensorMap* m, void* dst, int c0, int c1) {
            if constexpr (CG == 2) tma_load_2d_pair(m, full_c + s * 8u, dst, c0, c1);
            else tma_load_2d(m, &full[s], dst, c0, c1);
          };
          if constexpr (kHalfTilesOf<Epi>::value) {
            if (half) {  // 16 class rows at the top of each 32-row TMEM lane quadrant
#pragma unroll
              for (int q = 0; q < 4; ++q) load(&epi.tm_a16, a + q * 32 * 128, k0, ti.row0 + 16 * q);
            } else {
              load(&tmA, a, k0, ti.row0);
            }
          } else if (!A_MN) {
            load(&tmA, a, k0, ti.row0);
          } else {
#pragma unroll
            for (int i = 0; i < 128 / KB; ++i) load(&tmA, a + i * ATOM, ti.row0 + KB * i, k0);
          }
          if (!B_MN) {
            load(&tmB, b, k0, bcol);
          } else {
#pragma unroll
            for (int i = 0; i < BNL / KB; ++i) load(&tmB, b + i * ATOM, bcol + KB * i, k0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = kTf32 ? make_idesc_tf32(128, BN, A_MN, B_MN)
                                       : make_idesc_bf16(128 * CG, BN, A_MN, B_MN);
      uint32_t kbc = 0, it = 0;
      for (int t = first; t < total; t += stride, ++it) {
        const TileInfo ti = g.template tile<kHalfTilesOf<Epi>::value>(t);
        const uint32_t as = it & 1, aph = (it >> 1) & 1;
        mbar_wait(&tempty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = ti.kb0; kb < ti.kb1; ++kb, ++kbc) {
          const uint32_t s = kbc % STAGES, ph = (kbc / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 4 MMAs of 32 bytes of K each
            // MN-major tf32 operands use the 32-byte-atom 128B swizzle (4-row K groups, SBO
            // 512 B); everything else the 16-byte-atom one (8-row groups, SBO 1024 B)
            auto mn_desc = [&](uint32_t base) {
              return kTf32 ? make_sdesc_sw128_32b(base + k * KSTEP, ATOM, 512)
                           : make_sdesc_sw128(base + k * KSTEP, ATOM, 1024);
            };
            const uint64_t ad = A_MN ? mn_desc(a_base) : make_sdesc_sw128(a_base + k * 32, 0, 1024);
            const uint64_t bd = B_MN ? mn_desc(b_base) : make_sdesc_sw128(b_base + k * 32, 0, 1024);
            const uint32_t acc = (kb > ti.kb0 || k > 0) ? 1u : 0u;
            if constexpr (kTf32) umma_tf32(d_tmem, ad, bd, idesc, acc);
            else if constexpr (CG == 2) umma_bf16_pair(d_tmem, ad, bd, idesc, acc);
            else umma_bf16(d_tmem, ad, bd, idesc, acc);
          }
          if constexpr (CG == 2) umma_commit_pair(&empty[s]);
          else umma_commit(&empty[s]);
        }
        if constexpr (CG == 2) umma_commit_pair(&tfull[as]);
        else umma_commit(&tfull[as]);
      }
    }
  } else if (warp >= PFC_CTRL_WARPS) {
    // epilogue warpgroups: warp w reads TMEM lanes 32*(w%4).. (row = accumulator row);
    // warpgroup wg takes columns [wg*BN/NWG, (wg+1)*BN/NWG) of every tile.
    const int wg = (warp - PFC_CTRL_WARPS) >> 2;
    const int row = ((warp & 3) << 5) | lane;
    uint8_t* wsm = epi_smem + wg * Epi::kSmem;
    uint32_t it = 0;
    const uint32_t tempty_c = CG == 2 ? mapa_shared(smem_u32(tempty), 0) : 0u;
    // per-tile operands of the epilogue are loaded two tiles ahead (registers), so their
    // global-memory latency hides behind the current tile; epi.prefetch(next tile) runs on values
    // that have already arrived (e.g. bulk L2 prefetch of the rows the next tile updates)
    typename Epi::Pre pre{}, pre_n{};
    if (first < total) pre = epi.preload(tile_at(first), row, wg);
    if (first + stride < total) pre_n = epi.preload(tile_at(first + stride), row, wg);
    if (first < total) epi.prefetch(tile_at(first), row, wg, pre);
    for (int t = first; t < total; t += stride, ++it) {
      TileInfo ti = tile_at(t);
      ti.iter = (int)it;
      const uint32_t as = it & 1, aph = (it >> 1) & 1;
      if (t + stride < total) epi.prefetch(tile_at(t + stride), row, wg, pre_n);
      typename Epi::Pre pre_n2{};
      if (t + 2 * stride < total) pre_n2 = epi.preload(tile_at(t + 2 * stride), row, wg);
      mbar_wait(&tfull[as], aph);
      tc_fence_after();
      const TmemSrc src{tmem_base + as * BN + ((uint32_t)((warp & 3) * 32) << 16)};
      if constexpr (Epi::kNext)  // the epilogue also starts the next tile's loads
        epi.template run_next<BN, NWG>(ti, src, row, wg, wsm, pre, pre_n, t + stride < total);
      else
        epi.template run<BN, NWG>(ti, src, row, wg, wsm, pre);
      tc_fence_before();
      if constexpr (CG == 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_c + as * 8u);
      } else {
        mbar_arrive(&tempty[as]);
      }
      pre = pre_n;
      pre_n = pre_n2;
    }
    epi.finish(row, wg);
  }
  __syncthreads();
  if constexpr (Epi::kCluster > 1 || CG == 2) cluster_sync_all();  // no CTA leaves while its partner writes
  if (warp == 1) {
    if constexpr (CG == 2) tmem_dealloc_pair(tmem_base, TMEM_COLS);
    else tmem_dealloc(tmem_base, TMEM_COLS);
  }
#endif
}

// ---------------------------------------------------------------- SIMT fp32 engine
struct SmemRowSrc {  // accumulator row of this thread, staged in shared memory (stride 65)
  const float* row;
  __device__ __forceinline__ void load(int c0, float (&v)[32]) const {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = row[c0 + j];
  }
};

// A(m,k) = A_MN ? A[k*lda + m] : A[m*lda + k];  B(n,k) = B_MN ? B[k*ldb + n] : B[n*ldb + k].
template <bool A_MN, bool B_MN, class Epi>
__global__ void __launch_bounds__(128)
    simt_gemm_kernel(const float* __restrict__ A, int lda, const float* __restrict__ Bm, int ldb,
                     const GemmGeom g, const Epi epi) {
  constexpr int BN = 64, KC = 32;
  extern __shared__ uint8_t smem_raw[];
  float* sA = reinterpret_cast<float*>(smem_raw);  // [KC][129]
  float* sB = sA + KC * 129;                        // [KC][BN]
  float* sAcc = sB + KC * BN;                       // [128][65]
  uint8_t* epi_smem = reinterpret_cast<uint8_t*>(sAcc + 128 * 65);
  pdl_entry();
  const int tid = threadIdx.x;
  TileInfo ti = g.tile(blockIdx.x);
  float acc[BN];
#pragma unroll
  for (int j = 0; j < BN; ++j) acc[j] = 0.f;
  const int k_begin = ti.kb0 * 64;
  const int k_end = min(g.K, ti.kb1 * 64);
  for (int kc = k_begin; kc < k_end; kc += KC) {
    for (int e = tid; e < KC * 128; e += 128) {
      const int kk = A_MN ? e / 128 : e % KC;
      const int mm = A_MN ? e % 128 : e / KC;
      const int m = ti.row0 + mm, k = kc + kk;
      float v = 0.f;
      if (m < g.M && k < k_end) v = A_MN ? A[(int64_t)k * lda + m] : A[(int64_t)m * lda + k];
      sA[kk * 129 + mm] = v;
    }
    for (int e = tid; e < KC * BN; e += 128) {
      const int kk = B_MN ? e / BN : e % KC;
      const int nn = B_MN ? e % BN : e / KC;
      const int n = ti.col0 + nn, k = kc + kk;
      float v = 0.f;
      if (n < g.N && k < k_end) v = B_MN ? Bm[(int64_t)k * ldb + n] : Bm[(int64_t)n * ldb + k];
      sB[kk * BN + nn] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < KC; ++kk) {
      const float a = sA[kk * 129 + tid];
#pragma unroll
      for (int j = 0; j < BN; ++j) acc[j] = fmaf(a, sB[kk * BN + j], acc[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < BN; ++j) sAcc[tid * 65 + j] = acc[j];
  const SmemRowSrc src{sAcc + tid * 65};
  const typename Epi::Pre pre = epi.preload(ti, tid, 0);
  epi.template run<BN, 1>(ti, src, tid, 0, epi_smem, pre);
  epi.finish(tid, 0);
}

constexpr int kSimtSmemBytes = (32 * 129 + 32 * 64 + 128 * 65) * 4 + kEpiSmemBytes;

}  // namespace pfc
