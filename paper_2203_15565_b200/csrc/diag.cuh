// diag.cuh — the step's diagnostics on the device (metrics.hpp:56-146, computed by the reference
// step when cfg.with_diagnostics, shardsim.hpp:401-410, on the PRE-update shards):
//
//   apcs  = mean_b  cos(x^_b, w^_label(b))                     exact fp64 dot of fp32 inputs
//   amncs = mean_b  max_{j != label(b)} cos(x^_b, w^_j)        over ALL C classes
//   split (conflict ground truth): max over siblings (class_identity[j] == sample_identity[b])
//   and over the rest, averaged over the rows that have siblings / over all rows.
//
// amncs is a full-C cosine GEMM (2 B D C flop) on the tcgen05 engine with bf16 operands and a
// max epilogue.  To return the EXACT maximum, the epilogue keeps a running bf16 maximum per (row,
// bucket) and re-evaluates in fp64 every class whose bf16 cosine is within kBand of it: the bf16
// error of a unit-vector cosine is at most 2^-8 + fp32 accumulation (|x^| = |w^| = 1), so the
// true argmax is always re-evaluated.  Maxima are merged with integer atomics on an
// order-preserving encoding, so the result does not depend on scheduling.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "gemm.cuh"

namespace pfc {

__device__ __forceinline__ uint32_t enc_f32(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float dec_f32(uint32_t e) {
  return __uint_as_float((e & 0x80000000u) ? (e & 0x7fffffffu) : ~e);
}
__host__ __device__ __forceinline__ unsigned long long enc_f64(double f) {
  unsigned long long u;
  memcpy(&u, &f, 8);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double dec_f64(unsigned long long e) {
  const unsigned long long u = (e & 0x8000000000000000ull) ? (e & 0x7fffffffffffffffull) : ~e;
  double f;
  memcpy(&f, &u, 8);
  return f;
}

// x^ in bf16 for the GEMM and 1/max(|x|, 1e-12) in fp64 for the exact dots (matrix.hpp:130-143)
template <typename OT>
__global__ void diag_norm_x_kernel(const float* __restrict__ X, int B, int D, int Dp,
                                   OT* __restrict__ xh, double* __restrict__ xinv) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (b >= B) return;
  const float* x = X + (size_t)b * D;
  double ss = 0.0;
  for (int d = lane; d < D; d += 32) ss += (double)x[d] * (double)x[d];
  ss = warp_sum(ss);
  const double n = sqrt(ss);
  const double inv = 1.0 / (n > 1e-12 ? n : 1e-12);
  if (lane == 0) xinv[b] = inv;
  for (int d = lane; d < Dp; d += 32) store_out(xh + (size_t)b * Dp + d, d < D ? (float)(x[d] * inv) : 0.f);
}

// every local class: w^ in bf16 rows [rows_pad][Dp] and 1/max(|w|, 1e-12) in fp64 (metrics.hpp:20-31)
template <typename OT>
__global__ void diag_norm_w_kernel(const float* __restrict__ W, int64_t rows, int64_t rows_pad,
                                   int D, int Dp, OT* __restrict__ wall, double* __restrict__ winv) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows_pad) return;
  OT* o = wall + (size_t)r * Dp;
  if (r >= rows) {
    for (int d = lane; d < Dp; d += 32) store_out(o + d, 0.f);
    return;
  }
  const float* w = W + (size_t)r * D;
  double ss = 0.0;
  for (int d = lane; d < D; d += 32) ss += (double)w[d] * (double)w[d];
  ss = warp_sum(ss);
  const double n = sqrt(ss);
  const double inv = 1.0 / (n > 1e-12 ? n : 1e-12);
  if (lane == 0) winv[r] = inv;
  for (int d = lane; d < Dp; d += 32) store_out(o + d, d < D ? (float)(w[d] * inv) : 0.f);
}

// exact cos(x^_b, w^_r) in fp64 from the fp32 inputs, in the reference's order (d ascending)
__device__ __forceinline__ double diag_dot_exact(const float* __restrict__ X, double xinv,
                                                 const float* __restrict__ W, double winv, int D) {
  double s = 0.0;
  for (int d = 0; d < D; ++d) s += ((double)X[d] * xinv) * ((double)W[d] * winv);
  return s;
}

// apcs rows: the owner rank's exact cosine to the sample's own centre, 0 elsewhere (warp/row)
__global__ void diag_apcs_kernel(const float* __restrict__ X, const double* __restrict__ xinv,
                                 const float* __restrict__ W, const double* __restrict__ winv,
                                 const int64_t* __restrict__ labels, int B, int D, int64_t cls_lo,
                                 int64_t rows, double* __restrict__ apcs_row) {
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (b >= B) return;
  const int64_t r = labels[b] - cls_lo;
  double s = 0.0;
  if (r >= 0 && r < rows) {
    const float* x = X + (size_t)b * D;
    const float* w = W + (size_t)r * D;
    const double xi = xinv[b], wi = winv[r];
    for (int d = lane; d < D; d += 32) s += ((double)x[d] * xi) * ((double)w[d] * wi);
    s = warp_sum(s);
  }
  if (lane == 0) apcs_row[b] = s;
}

struct DiagCand {  // a class within kBand of its bucket's running maximum when it was seen
  int32_t b, k;
  int64_t j;
  float v, pad;
};

struct DiagMaxEpi : NoSetup {
  static constexpr int kSmem = 0;
  static constexpr float kBand = 1.0f / 64.0f;  // > 2 x (2^-8 + fp32 accumulation)
  int B;
  int64_t rows, cls_lo;
  const int64_t* labels;   // [B] global; nullptr: mics mode, row r excludes column row_base + r
  int64_t row_base;        // mics mode: local class of the first row of this launch
  const int64_t* cid;      // [rows] class identity of the local classes, or nullptr (no split)
  const int64_t* sid;      // [B] sample identity, or nullptr
  uint32_t* rmax;          // [B][3] running bf16 maximum per bucket (enc_f32)
  int* hasc;               // [B] a sibling class exists
  DiagCand* cand;          // candidate list for the exact pass
  unsigned long long* ncand;
  unsigned long long cap;

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
    const int64_t lab = !rv ? -1 : (labels ? labels[b] - cls_lo : row_base + b);
    const int64_t sb = (rv && sid) ? sid[b] : 0;
    float rm[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) rm[k] = rv ? dec_f32(rmax[b * 3 + k]) : 0.f;
#pragma unroll 1
    for (int c0 = wg * CW; c0 < (wg + 1) * CW; c0 += 32) {
      float v[32];
      src.load(c0, v);  // all lanes: tcgen05.ld is warp-collective
      const int64_t colb = t.col0 + c0;
      if (!rv || colb >= rows) continue;
      if (!cid) {  // no split: one bucket; the per-column work runs only near the maximum
        float cm = -INFINITY;
        if (colb + 32 <= rows && (lab < colb || lab >= colb + 32)) {
          // every column valid (the common case): a plain 32-way max, no per-column index tests
          float m4[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
          for (int q = 4; q < 32; ++q) m4[q & 3] = fmaxf(m4[q & 3], v[q]);
          cm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        } else {
          const int nv = (int)(rows - colb < 32 ? rows - colb : 32);
          const int lq = (lab >= colb && lab < colb + 32) ? (int)(lab - colb) : -1;
#pragma unroll
          for (int q = 0; q < 32; ++q) cm = (q < nv && q != lq) ? fmaxf(cm, v[q]) : cm;
        }
        if (cm > rm[0]) {
          rm[0] = cm;
          atomicMax(rmax + b * 3, enc_f32(cm));
        }
        if (cm < rm[0] - kBand) continue;
#pragma unroll 1
        for (int q = 0; q < 32; ++q) {
          const int64_t j = colb + q;
          float vq = v[0];
#pragma unroll
          for (int u = 1; u < 32; ++u) vq = (u == q) ? v[u] : vq;
          if (j >= rows || j == lab || vq < rm[0] - kBand) continue;
          const unsigned long long i = atomicAdd(ncand, 1ull);
          if (i < cap) cand[i] = DiagCand{b, 0, j, vq, 0.f};
        }
        continue;
      }
      // per-column bucket: 1 = sibling, 2 = other (with the conflict split); -1 = excluded
      int bk[32];
      float cm[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int64_t j = colb + q;
        int k = -1;
        if (j < rows && j != lab) k = cid ? (cid[j] == sb ? 1 : 2) : 0;
        bk[q] = k;
        if (k >= 0) cm[k] = fmaxf(cm[k], v[q]);
      }
      if (cid && cm[1] > -INFINITY && !hasc[b]) hasc[b] = 1;
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (cm[k] > rm[k]) {
          rm[k] = cm[k];
          atomicMax(rmax + b * 3 + k, enc_f32(cm[k]));
        }
      // candidates: within kBand of the running maximum of their bucket; evaluated exactly by
      // diag_exact_kernel (which drops those below the FINAL maximum minus kBand)
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int k = bk[q];
        if (k < 0 || v[q] < rm[k] - kBand) continue;
        const unsigned long long i = atomicAdd(ncand, 1ull);
        if (i < cap) cand[i] = DiagCand{b, k, colb + q, v[q], 0.f};
      }
    }
  }
};

// One warp per candidate: exact fp64 cosine (lanes stride d, fixed-order warp reduction) of the
// candidates within kBand of their row's final bf16 maximum; atomic max into emax.
__global__ void diag_exact_kernel(const DiagCand* __restrict__ cand,
                                  const unsigned long long* __restrict__ ncand,
                                  unsigned long long cap, const uint32_t* __restrict__ rmax,
                                  const float* __restrict__ X, const double* __restrict__ xinv,
                                  const float* __restrict__ W, const double* __restrict__ winv,
                                  int D, unsigned long long* __restrict__ emax) {
  const unsigned long long n = min(*ncand, cap);
  const int lane = threadIdx.x & 31;
  for (unsigned long long i = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((unsigned long long)gridDim.x * blockDim.x) >> 5) {
    const DiagCand c = cand[i];
    if (c.v < dec_f32(rmax[c.b * 3 + c.k]) - DiagMaxEpi::kBand) continue;  // warp-uniform
    const float* x = X + (size_t)c.b * D;
    const float* w = W + (size_t)c.j * D;
    const double xi = xinv[c.b], wi = winv[c.j];
    double s = 0.0;
    for (int d = lane; d < D; d += 32) s += ((double)x[d] * xi) * ((double)w[d] * wi);
    s = warp_sum(s);
    if (lane == 0) atomicMax(emax + c.b * 3 + c.k, enc_f64(s));
  }
}

}  // namespace pfc
