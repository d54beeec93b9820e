// backbone.cuh — device side of the trainer integration: the reference's
// two-layer tanh perceptron (trainer.hpp:51-126) in fp64, fed from a device-resident dataset, so
// the features X and their gradient dX of every training step stay in HBM.
//
// The products follow matmul (matrix.hpp:83-105): each output cell sums its k terms in ascending
// order with separate multiply and add (the reference builds with -ffp-contract=off), so every
// cell of every product equals the reference's bit for bit; only tanh (CUDA libdevice vs glibc)
// may differ in the last place.  These are tiny products (hidden 96, embed 64, batch 48 in the
// reference defaults): one thread per output cell, latency-bound, not a roofline kernel.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace pfc {

enum BbEpi { kBbPlain = 0, kBbTanhBias = 1, kBbBias = 2, kBbTanhGrad = 3 };

// C[i][j] = epi(sum_k A(i,k) B(k,j)), A(i,k) = A[i*a_i + k*a_k], B(k,j) = B[k*b_k + j*b_j],
// C row-major [rows][cols].  A non-finite product sets bit `which` of *nonfinite (require_finite
// of matmul, matrix.hpp:103) before the epilogue is applied, as in the reference.
//   kBbTanhBias: tanh(acc + bias[i])                 (Backbone::forward hidden, trainer.hpp:86-90)
//   kBbBias:     acc + bias[i]                       (Backbone::forward output, 91-94)
//   kBbTanhGrad: acc * (1 - h[i][j] * h[i][j])       (apply_gradient d_hidden, 105-111)
template <int EPI>
__global__ void bb_matmul_kernel(const double* __restrict__ A, int64_t a_i, int64_t a_k,
                                 const double* __restrict__ Bm, int64_t b_k, int64_t b_j,
                                 double* __restrict__ C, int rows, int cols, int inner,
                                 const double* __restrict__ aux, int* nonfinite, int which) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= cols || i >= rows) return;
  double acc = 0.0;
  for (int k = 0; k < inner; ++k)
    acc = __dadd_rn(acc, __dmul_rn(A[(int64_t)i * a_i + (int64_t)k * a_k],
                                   Bm[(int64_t)k * b_k + (int64_t)j * b_j]));
  if (!isfinite(acc)) atomicOr(nonfinite, 1 << which);
  if (EPI == kBbTanhBias) acc = tanh(__dadd_rn(acc, aux[i]));
  if (EPI == kBbBias) acc = __dadd_rn(acc, aux[i]);
  if (EPI == kBbTanhGrad) {
    const double h = aux[(int64_t)i * cols + j];
    acc = __dmul_rn(acc, __dsub_rn(1.0, __dmul_rn(h, h)));
  }
  C[(int64_t)i * cols + j] = acc;
}

// One row i of an SGD step (apply_gradient, trainer.hpp:113-124): db = sum_b dsrc[i][b]
// (b ascending), bias[i] -= lr * db, w[i][j] -= lr * g[i][j].  Block per row.
__global__ void bb_sgd_rows_kernel(double* __restrict__ w, double* __restrict__ bias,
                                   const double* __restrict__ g, const double* __restrict__ dsrc,
                                   int cols, int batch, double lr) {
  const int i = blockIdx.x;
  if (threadIdx.x == 0) {
    double db = 0.0;
    for (int b = 0; b < batch; ++b) db = __dadd_rn(db, dsrc[(int64_t)i * batch + b]);
    bias[i] = __dsub_rn(bias[i], __dmul_rn(lr, db));
  }
  for (int j = threadIdx.x; j < cols; j += blockDim.x) {
    const int64_t o = (int64_t)i * cols + j;
    w[o] = __dsub_rn(w[o], __dmul_rn(lr, g[o]));
  }
}

// The step's inputs from the device-resident dataset (trainer.hpp:451-459): column b of the
// batch is point ids[b]; its label is observed_labels[ids[b]].
__global__ void bb_gather_kernel(const double* __restrict__ points, int64_t npts, int in_dim,
                                 const int64_t* __restrict__ ids, int batch,
                                 const int64_t* __restrict__ plabels, double* __restrict__ inputs,
                                 int64_t* __restrict__ labels) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int d = blockIdx.y;
  if (b >= batch) return;
  const int64_t p = ids[b];
  inputs[(int64_t)d * batch + b] = points[(int64_t)d * npts + p];
  if (d == 0 && labels) labels[b] = plabels[p];
}

// ---- evaluation of the trained model (trainer.hpp:519-577) on the device, in fp64 with the
// reference's operation order (products and sums as separate IEEE operations, d ascending), so
// the cosines equal the reference's host loops bit for bit on the same embeddings and centres.

// l2_normalize_columns (matrix.hpp:118-143) of a chunk of embeddings: feat is E x m (the step's
// FeatureBatch layout); out rows [m][E] (row-major per point).
__global__ void eval_normalize_kernel(const double* __restrict__ feat, int E, int m,
                                      double* __restrict__ out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= m) return;
  double s = 0.0;
  for (int d = 0; d < E; ++d) {
    const double x = feat[(int64_t)d * m + b];
    s = __dadd_rn(s, __dmul_rn(x, x));
  }
  const double inv = 1.0 / fmax(sqrt(s), 1e-12);
  for (int d = 0; d < E; ++d) out[(int64_t)b * E + d] = __dmul_rn(feat[(int64_t)d * m + b], inv);
}

// unit_center (metrics.hpp:20-31): per class, 1 / max(|w|, 1e-12) of its fp32 row (as fp64)
__global__ void eval_center_inv_kernel(const float* __restrict__ W, int64_t C, int D,
                                       double* __restrict__ winv) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= C) return;
  double s = 0.0;
  for (int d = 0; d < D; ++d) {
    const double x = (double)W[r * D + d];
    s = __dadd_rn(s, __dmul_rn(x, x));
  }
  winv[r] = 1.0 / fmax(sqrt(s), 1e-12);
}

// Nearest unit centre of each point (trainer.hpp:532-545): one block per point, threads over
// classes, cos = sum_d emb_d (w_d inv) in d order; the first class with the largest cosine wins
// (the reference's strict > scan from best = -2); NaN never wins.
__global__ void __launch_bounds__(256) eval_argmax_kernel(const double* __restrict__ emb, int E,
                                                          const float* __restrict__ W,
                                                          const double* __restrict__ winv,
                                                          int64_t C, int64_t* __restrict__ best) {
  __shared__ double se[512];
  __shared__ double bv[256];
  __shared__ int64_t bc[256];
  const int b = blockIdx.x;
  for (int d = threadIdx.x; d < E; d += blockDim.x) se[d] = emb[(int64_t)b * E + d];
  __syncthreads();
  double v = -2.0;
  int64_t c_best = -1;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
    const float* w = W + c * E;
    const double inv = winv[c];
    double cs = 0.0;
    for (int d = 0; d < E; ++d) cs = __dadd_rn(cs, __dmul_rn(se[d], __dmul_rn((double)w[d], inv)));
    if (cs > v) {  // classes ascend within the thread: strict > keeps the first
      v = cs;
      c_best = c;
    }
  }
  bv[threadIdx.x] = v;
  bc[threadIdx.x] = c_best;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double ov = bv[threadIdx.x + o];
      const int64_t oc = bc[threadIdx.x + o];
      const bool take = oc >= 0 && (ov > bv[threadIdx.x] ||
                                    (ov == bv[threadIdx.x] && (bc[threadIdx.x] < 0 || oc < bc[threadIdx.x])));
      if (take) {
        bv[threadIdx.x] = ov;
        bc[threadIdx.x] = oc;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) best[b] = bc[0];
}

// Cosines of all pairs i < j (trainer.hpp:553-561), in (i, j) lexicographic order.
__global__ void eval_pairs_kernel(const double* __restrict__ emb, int E, int64_t n, int64_t i0,
                                  double* __restrict__ out) {
  const int64_t i = i0 + blockIdx.y;
  const int64_t j = i + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double cs = 0.0;
  for (int d = 0; d < E; ++d) cs = __dadd_rn(cs, __dmul_rn(emb[i * E + d], emb[j * E + d]));
  out[i * n - i * (i + 1) / 2 + (j - i - 1)] = cs;
}

}  // namespace pfc
