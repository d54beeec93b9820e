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

}  // namespace pfc
