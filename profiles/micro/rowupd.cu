// Microbenchmark: gathered-row momentum-SGD update (the dW epilogue's HBM pattern) at different
// access granularities.  200k random rows of a [2M][512] fp32 table (W and momentum), plus a
// dense [200k][512] fp32 "dwt" source.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int D = 512;
// (a) epilogue pattern: warp = 32 rows x 128 dims; per step 8 lanes x float4 per row, 4 rows/op
template <int RPI>
__global__ void upd_a(float* W, float* M, const float* src, const int* rows, int n, float lr) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  constexpr int LPR = 32 / RPI;          // lanes per row
  const int sub = lane / LPR, q = (lane % LPR) * 4;
  for (int blk = warp; blk < n / 32 * (D / 128); blk += nw) {
    const int r0 = (blk / (D / 128)) * 32, d0 = (blk % (D / 128)) * 128;
    for (int c = 0; c < 128; c += LPR * 4) {
#pragma unroll
      for (int u = 0; u < 32 / RPI; ++u) {
        const int rr = r0 + u * RPI + sub;
        const int r = rows[rr];
        const size_t o = (size_t)r * D + d0 + c + q;
        float4 w = *reinterpret_cast<float4*>(W + o), m = *reinterpret_cast<float4*>(M + o);
        const float4 a = *reinterpret_cast<const float4*>(src + (size_t)rr * D + d0 + c + q);
        m.x = 0.9f * m.x + a.x; m.y = 0.9f * m.y + a.y; m.z = 0.9f * m.z + a.z; m.w = 0.9f * m.w + a.w;
        w.x -= lr * m.x; w.y -= lr * m.y; w.z -= lr * m.z; w.w -= lr * m.w;
        *reinterpret_cast<float4*>(W + o) = w;
        *reinterpret_cast<float4*>(M + o) = m;
      }
    }
  }
}

// (b) loads grouped ahead of all stores: U row groups x (W, M, src) float4 in flight per lane
template <int U>
__global__ void upd_b(float* __restrict__ W, float* __restrict__ M, const float* __restrict__ src,
                      const int* __restrict__ rows, int n, float lr) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int sub = lane >> 3, q = (lane & 7) * 4;  // 4 rows x 128 B per op
  constexpr int RB = 4 * U;                       // rows per block step
  for (int blk = warp; blk < n / RB * (D / 32); blk += nw) {
    const int r0 = (blk / (D / 32)) * RB, d = (blk % (D / 32)) * 32 + q;
    float4 w[U], m[U], a[U];
    size_t o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int rr = r0 + u * 4 + sub;
      o[u] = (size_t)__ldg(rows + rr) * D + d;
      w[u] = *reinterpret_cast<const float4*>(W + o[u]);
      m[u] = *reinterpret_cast<const float4*>(M + o[u]);
      a[u] = __ldg(reinterpret_cast<const float4*>(src + (size_t)rr * D + d));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      m[u].x = 0.9f * m[u].x + a[u].x; m[u].y = 0.9f * m[u].y + a[u].y;
      m[u].z = 0.9f * m[u].z + a[u].z; m[u].w = 0.9f * m[u].w + a[u].w;
      w[u].x -= lr * m[u].x; w[u].y -= lr * m[u].y; w[u].z -= lr * m[u].z; w[u].w -= lr * m[u].w;
      *reinterpret_cast<float4*>(W + o[u]) = w[u];
      *reinterpret_cast<float4*>(M + o[u]) = m[u];
    }
  }
}

// (d) temporal spread: a warp owns G*4 rows x 256 dims; chunk-major order (c outer, row groups
// inner, 4 row groups per batch of loads): a row's consecutive 128 B chunks are G/4 batches apart
template <int G>
__global__ void upd_d(float* __restrict__ W, float* __restrict__ M, const float* __restrict__ src,
                      const int* __restrict__ rows, int n, float lr) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int sub = lane >> 3, q = (lane & 7) * 4;
  constexpr int RB = 4 * G;
  for (int blk = warp; blk < n / RB * 2; blk += nw) {
    const int r0 = (blk >> 1) * RB, h = (blk & 1) * 256;
    for (int c = 0; c < 8; ++c) {
      const int d = h + c * 32 + q;
      for (int g0 = 0; g0 < G; g0 += 4) {
        float4 w[4], m[4], a[4];
        size_t o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = r0 + (g0 + u) * 4 + sub;
          o[u] = (size_t)__ldg(rows + rr) * D + d;
          w[u] = *reinterpret_cast<const float4*>(W + o[u]);
          m[u] = *reinterpret_cast<const float4*>(M + o[u]);
          a[u] = __ldg(reinterpret_cast<const float4*>(src + (size_t)rr * D + d));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          m[u].x = 0.9f * m[u].x + a[u].x; m[u].y = 0.9f * m[u].y + a[u].y;
          m[u].z = 0.9f * m[u].z + a[u].z; m[u].w = 0.9f * m[u].w + a[u].w;
          w[u].x -= lr * m[u].x; w[u].y -= lr * m[u].y; w[u].z -= lr * m[u].z; w[u].w -= lr * m[u].w;
          *reinterpret_cast<float4*>(W + o[u]) = w[u];
          *reinterpret_cast<float4*>(M + o[u]) = m[u];
        }
      }
    }
  }
}

// (e) W and momentum interleaved per row: WM[r][2][D] (one 4 KB span per row), grouped loads
template <int U, bool kF4>  // kF4: float4-interleaved WM[r][D/4][2] instead
__global__ void upd_e(float* __restrict__ WM, const float* __restrict__ src,
                      const int* __restrict__ rows, int n, float lr) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int sub = lane >> 3, q = (lane & 7) * 4;
  constexpr int RB = 4 * U;
  for (int blk = warp; blk < n / RB * (D / 32); blk += nw) {
    const int r0 = (blk / (D / 32)) * RB, d = (blk % (D / 32)) * 32 + q;
    float4 w[U], m[U], a[U];
    size_t ow[U], om[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int rr = r0 + u * 4 + sub;
      const size_t base = (size_t)__ldg(rows + rr) * 2 * D;
      ow[u] = kF4 ? base + (size_t)d * 2 : base + d;
      om[u] = kF4 ? ow[u] + 4 : base + D + d;
      w[u] = *reinterpret_cast<const float4*>(WM + ow[u]);
      m[u] = *reinterpret_cast<const float4*>(WM + om[u]);
      a[u] = __ldg(reinterpret_cast<const float4*>(src + (size_t)rr * D + d));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      m[u].x = 0.9f * m[u].x + a[u].x; m[u].y = 0.9f * m[u].y + a[u].y;
      m[u].z = 0.9f * m[u].z + a[u].z; m[u].w = 0.9f * m[u].w + a[u].w;
      w[u].x -= lr * m[u].x; w[u].y -= lr * m[u].y; w[u].z -= lr * m[u].z; w[u].w -= lr * m[u].w;
      *reinterpret_cast<float4*>(WM + ow[u]) = w[u];
      *reinterpret_cast<float4*>(WM + om[u]) = m[u];
    }
  }
}

// (f) the dW epilogue's ownership: a warp owns 8 rows x 256 dims (one CTA's half of each row; the
// other half is the adjacent warp's).  kRowMajor = false: chunk-major (all 8 rows' 128 B chunk c,
// then c+1: the current epilogue order, NR rows per batch of loads); true: row-major (a row's
// whole 1 KB span per step: lanes cover 256 dims with 2 float4 each, NR rows per batch).
template <bool kRowMajor, int NR>
__global__ void upd_f(float* __restrict__ W, float* __restrict__ M, const float* __restrict__ src,
                      const int* __restrict__ rows, int n, float lr) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int blk = warp; blk < n / 8 * 2; blk += nw) {
    const int r0 = (blk >> 1) * 8, h = (blk & 1) * 256;
    if (!kRowMajor) {
      const int sub = lane >> 3, q = (lane & 7) * 4;  // 4 rows x 32 dims per op
      for (int c = 0; c < 8; ++c) {
        const int d = h + c * 32 + q;
        float4 w[2], m[2], a[2];
        size_t o[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int rr = r0 + u * 4 + sub;
          o[u] = (size_t)__ldg(rows + rr) * D + d;
          w[u] = *reinterpret_cast<const float4*>(W + o[u]);
          m[u] = *reinterpret_cast<const float4*>(M + o[u]);
          a[u] = __ldg(reinterpret_cast<const float4*>(src + (size_t)rr * D + d));
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          m[u].x = 0.9f * m[u].x + a[u].x; m[u].y = 0.9f * m[u].y + a[u].y;
          m[u].z = 0.9f * m[u].z + a[u].z; m[u].w = 0.9f * m[u].w + a[u].w;
          w[u].x -= lr * m[u].x; w[u].y -= lr * m[u].y; w[u].z -= lr * m[u].z; w[u].w -= lr * m[u].w;
          *reinterpret_cast<float4*>(W + o[u]) = w[u];
          *reinterpret_cast<float4*>(M + o[u]) = m[u];
        }
      }
    } else {
      for (int r1 = 0; r1 < 8; r1 += NR) {
        float4 w[NR][2], m[NR][2], a[NR][2];
        size_t o[NR][2];
#pragma unroll
        for (int u = 0; u < NR; ++u) {
          const int rr = r0 + r1 + u;
          const size_t base = (size_t)__ldg(rows + rr) * D + h;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int d = k * 128 + lane * 4;
            o[u][k] = base + d;
            w[u][k] = *reinterpret_cast<const float4*>(W + o[u][k]);
            m[u][k] = *reinterpret_cast<const float4*>(M + o[u][k]);
            a[u][k] = __ldg(reinterpret_cast<const float4*>(src + (size_t)rr * D + h + d));
          }
        }
#pragma unroll
        for (int u = 0; u < NR; ++u)
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            float4& mm = m[u][k];
            float4& ww = w[u][k];
            const float4& aa = a[u][k];
            mm.x = 0.9f * mm.x + aa.x; mm.y = 0.9f * mm.y + aa.y; mm.z = 0.9f * mm.z + aa.z; mm.w = 0.9f * mm.w + aa.w;
            ww.x -= lr * mm.x; ww.y -= lr * mm.y; ww.z -= lr * mm.z; ww.w -= lr * mm.w;
            *reinterpret_cast<float4*>(W + o[u][k]) = ww;
            *reinterpret_cast<float4*>(M + o[u][k]) = mm;
          }
      }
    }
  }
}

// (g) the epilogue's actual ring depth: a warp owns 8 rows x 256 dims, chunk-major, with NC
// consecutive 128 B chunks of its 8 rows in flight (the cp.async ring holds ~6), W and momentum
// only (dwt comes from TMEM in the kernel); traffic counted as 4 streams
template <int NC>
__global__ void upd_g(float* __restrict__ W, float* __restrict__ M, const int* __restrict__ rows,
                      int n, float lr) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int sub = lane >> 3, q = (lane & 7) * 4;
  for (int blk = warp; blk < n / 8 * 2; blk += nw) {
    const int r0 = (blk >> 1) * 8, h = (blk & 1) * 256;
    size_t rb[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) rb[u] = (size_t)__ldg(rows + r0 + u * 4 + sub) * D + h + q;
    for (int c0 = 0; c0 < 8; c0 += NC) {
      float4 w[NC][2], m[NC][2];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (c0 + c < 8) {
            w[c][u] = *reinterpret_cast<const float4*>(W + rb[u] + (c0 + c) * 32);
            m[c][u] = *reinterpret_cast<const float4*>(M + rb[u] + (c0 + c) * 32);
          }
        }
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (c0 + c < 8) {
            float4& mm = m[c][u];
            float4& ww = w[c][u];
            mm.x = 0.9f * mm.x + 1e-3f; mm.y = 0.9f * mm.y + 1e-3f; mm.z = 0.9f * mm.z + 1e-3f; mm.w = 0.9f * mm.w + 1e-3f;
            ww.x -= lr * mm.x; ww.y -= lr * mm.y; ww.z -= lr * mm.z; ww.w -= lr * mm.w;
            *reinterpret_cast<float4*>(W + rb[u] + (c0 + c) * 32) = ww;
            *reinterpret_cast<float4*>(M + rb[u] + (c0 + c) * 32) = mm;
          }
        }
    }
  }
}

int main() {
  const int C = 2000000, n = 200000;
  float *W, *M, *src;
  int* rows;
  cudaMalloc(&W, (size_t)C * D * 4);
  cudaMalloc(&M, (size_t)C * D * 4);
  cudaMalloc(&src, (size_t)n * D * 4);
  cudaMalloc(&rows, n * 4);
  float* WM;  // interleaved W + momentum for (e): same 8.2 GB as W and M together
  cudaMalloc(&WM, (size_t)C * 2 * D * 4);
  cudaMemset(WM, 0, (size_t)C * 2 * D * 4);
  cudaMemset(W, 0, (size_t)C * D * 4);
  cudaMemset(M, 0, (size_t)C * D * 4);
  cudaMemset(src, 0, (size_t)n * D * 4);
  std::vector<int> h(C);
  for (int i = 0; i < C; ++i) h[i] = i;
  std::mt19937 g(1);
  std::shuffle(h.begin(), h.end(), g);
  h.resize(n);
  for (int sorted = 0; sorted < 1; ++sorted) {
    std::vector<int> hh = h;
    if (sorted) std::sort(hh.begin(), hh.end());
    cudaMemcpy(rows, hh.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = (double)n * D * 4 * 5;
    auto run = [&](const char* name, auto kern, int blocks, int threads) {
      for (int i = 0; i < 3; ++i) kern<<<blocks, threads>>>(W, M, src, rows, n, 0.1f);
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) kern<<<blocks, threads>>>(W, M, src, rows, n, 0.1f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      printf("%s sorted=%d blocks=%d threads=%d: %.1f us  %.0f GB/s\n", name, sorted, blocks, threads,
             ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    for (int th : {512}) {
      run("rows/op=4 (128B/row)", upd_a<4>, 148 * (2048 / th), th);
      run("rows/op=2 (256B/row)", upd_a<2>, 148 * (2048 / th), th);
      run("rows/op=1 (512B/row)", upd_a<1>, 148 * (2048 / th), th);
    }
    run("rows/op=4 8warps/SM", upd_a<4>, 148, 256);
    run("rows/op=1 8warps/SM", upd_a<1>, 148, 256);
    run("grouped U=2 8warps/SM", upd_b<2>, 148, 256);
    run("grouped U=4 8warps/SM", upd_b<4>, 148, 256);
    run("grouped U=8 8warps/SM", upd_b<8>, 148, 256);
    run("grouped U=4 16warps/SM", upd_b<4>, 148, 512);
    run("grouped U=8 16warps/SM", upd_b<8>, 148, 512);
    run("grouped U=4 64warps/SM", upd_b<4>, 148 * 4, 512);
    run("spread G=4 16warps/SM", upd_d<4>, 148, 512);
    run("spread G=8 16warps/SM", upd_d<8>, 148, 512);
    run("spread G=32 16warps/SM", upd_d<32>, 148, 512);
    run("spread G=128 16warps/SM", upd_d<128>, 148, 512);
    run("dW ownership chunk-major 16warps/SM", upd_f<false, 1>, 148, 512);
    run("dW ownership row-major NR=1 16warps/SM", upd_f<true, 1>, 148, 512);
    run("dW ownership row-major NR=2 16warps/SM", upd_f<true, 2>, 148, 512);
    run("dW ownership row-major NR=4 16warps/SM", upd_f<true, 4>, 148, 512);
    auto run_g = [&](const char* name, auto kern) {
      const double b4 = (double)n * D * 4 * 4;
      for (int i = 0; i < 3; ++i) kern<<<148, 512>>>(W, M, rows, n, 0.1f);
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) kern<<<148, 512>>>(W, M, rows, n, 0.1f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      printf("%s: %.1f us  %.0f GB/s\n", name, ms * 1e3, b4 / (ms * 1e-3) / 1e9);
    };
    run_g("ring emulation W+M chunk-major NC=1 16warps/SM", upd_g<1>);
    run_g("ring emulation W+M chunk-major NC=2 16warps/SM", upd_g<2>);
    run_g("ring emulation W+M chunk-major NC=4 16warps/SM", upd_g<4>);
    run_g("ring emulation W+M chunk-major NC=8 (whole row) 16warps/SM", upd_g<8>);
    auto run_e = [&](const char* name, auto kern, int blocks, int threads) {
      for (int i = 0; i < 3; ++i) kern<<<blocks, threads>>>(WM, src, rows, n, 0.1f);
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) kern<<<blocks, threads>>>(WM, src, rows, n, 0.1f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      printf("%s: %.1f us  %.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    run_e("interleaved [r][2][D] U=4 16warps/SM", upd_e<4, false>, 148, 512);
    run_e("interleaved [r][2][D] U=8 16warps/SM", upd_e<8, false>, 148, 512);
    run_e("interleaved [r][D/4][2] U=4 16warps/SM", upd_e<4, true>, 148, 512);
    run_e("interleaved [r][D/4][2] U=8 16warps/SM", upd_e<8, true>, 148, 512);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
