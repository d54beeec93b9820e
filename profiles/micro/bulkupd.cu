// Microbenchmark: the dW epilogue's gathered-row momentum-SGD stream fed by TMA bulk copies
// (cp.async.bulk, one 1 KB row half per copy = row-major DRAM order) into a CTA-wide shared-memory
// ring, against the per-lane cp.async chunk-major stream of the shipped epilogue (rowupd.cu).
// 200k random rows of a [2M][512] fp32 W and momentum; a unit = R row halves (W + M, 2R KB).
//   producer warp: waits slot empty, expect_tx, lanes issue the 2R bulk loads
//   NCW consumer warps: row-major float4 reads (lane = dims), update, then either
//     kBulkStore: write back into the slot, fence.proxy.async, bulk store (1 KB per row half)
//     else:       st.global.v4 straight from registers (coalesced 512 B per instruction)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bulkupd bulkupd.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2203_15565_b200/csrc/sm100.cuh"

using namespace pfc_sm100;
constexpr int D = 512;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}

template <int R, int S, int NCW, bool kBulkStore>
__global__ void __launch_bounds__(32 * (NCW + 1)) upd_bulk(float* __restrict__ W, float* __restrict__ M,
                                                           const int* __restrict__ rows, int n, float lr) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kSlot = R * 2 * 1024;  // W halves then M halves
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kSlot);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int units = n / R * 2;  // (row block, half)
  if (warp == NCW) {            // producer
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int s = i % S;
      if (i >= S) mbar_wait(&empty[s], ((i / S) - 1) & 1);
      const int r0 = (u >> 1) * R, h = (u & 1) * 256;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], kSlot);
      __syncwarp();
      if (lane < R) {
        const size_t o = (size_t)__ldg(rows + r0 + lane) * D + h;
        const uint32_t base = smem_u32(smem + s * kSlot);
        bulk_g2s(base + lane * 1024, W + o, 1024, &full[s]);
        bulk_g2s(base + (R + lane) * 1024, M + o, 1024, &full[s]);
      }
    }
    return;
  }
  int i = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
    const int s = i % S;
    mbar_wait(&full[s], (i / S) & 1);
    const int r0 = (u >> 1) * R, h = (u & 1) * 256;
    float* ws = reinterpret_cast<float*>(smem + s * kSlot);
    for (int rr = warp; rr < R; rr += NCW) {
      const size_t o = (size_t)__ldg(rows + r0 + rr) * D + h;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int d = k * 128 + lane * 4;
        float4 w = *reinterpret_cast<const float4*>(ws + rr * 256 + d);
        float4 m = *reinterpret_cast<const float4*>(ws + (R + rr) * 256 + d);
        m.x = 0.9f * m.x + 1e-3f; m.y = 0.9f * m.y + 1e-3f; m.z = 0.9f * m.z + 1e-3f; m.w = 0.9f * m.w + 1e-3f;
        w.x -= lr * m.x; w.y -= lr * m.y; w.z -= lr * m.z; w.w -= lr * m.w;
        if (kBulkStore) {
          *reinterpret_cast<float4*>(ws + rr * 256 + d) = w;
          *reinterpret_cast<float4*>(ws + (R + rr) * 256 + d) = m;
        } else {
          *reinterpret_cast<float4*>(W + o + d) = w;
          *reinterpret_cast<float4*>(M + o + d) = m;
        }
      }
      if (kBulkStore) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const uint32_t base = smem_u32(smem + s * kSlot);
          bulk_s2g(W + o, base + rr * 1024, 1024);
          bulk_s2g(M + o, base + (R + rr) * 1024, 1024);
          bulk_commit();
        }
      }
    }
    if (kBulkStore && lane == 0) bulk_wait_read<0>();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (kBulkStore && lane == 0) bulk_wait_all();
}

// per-lane cp.async reference (the shipped order is in rowupd.cu upd_g); here plain row-major
// register loads with NR rows in flight per warp, 16 warps/SM (rowupd.cu upd_f<true, NR>)
int main() {
  const int C = 2000000, n = 200000;
  float *W, *M;
  int* rows;
  cudaMalloc(&W, (size_t)C * D * 4);
  cudaMalloc(&M, (size_t)C * D * 4);
  cudaMalloc(&rows, n * 4);
  cudaMemset(W, 0, (size_t)C * D * 4);
  cudaMemset(M, 0, (size_t)C * D * 4);
  std::vector<int> h(C);
  for (int i = 0; i < C; ++i) h[i] = i;
  std::mt19937 g(1);
  std::shuffle(h.begin(), h.end(), g);
  h.resize(n);
  cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)n * D * 4 * 4;
  auto run = [&](const char* name, auto kern, int R, int S, int ncw, int blocks) {
    const int smem = S * R * 2048 + 2 * S * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int i = 0; i < 3; ++i) kern<<<blocks, 32 * (ncw + 1), smem>>>(W, M, rows, n, 0.1f);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) kern<<<blocks, 32 * (ncw + 1), smem>>>(W, M, rows, n, 0.1f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-48s R=%2d S=%2d ncw=%2d blocks=%4d smem=%6d: %7.1f us  %6.0f GB/s  (%s)\n", name, R, S,
           ncw, blocks, smem, ms * 1e3, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run("bulk load + st.global", upd_bulk<8, 8, 8, false>, 8, 8, 8, 148);
  run("bulk load + st.global", upd_bulk<8, 6, 8, false>, 8, 6, 8, 148);
  run("bulk load + st.global", upd_bulk<8, 4, 8, false>, 8, 4, 8, 148);
  run("bulk load + st.global", upd_bulk<4, 12, 4, false>, 4, 12, 4, 148);
  run("bulk load + st.global", upd_bulk<4, 8, 4, false>, 4, 8, 4, 148);
  run("bulk load + st.global", upd_bulk<16, 4, 16, false>, 16, 4, 16, 148);
  run("bulk load + st.global", upd_bulk<16, 3, 16, false>, 16, 3, 16, 148);
  run("bulk load + bulk store", upd_bulk<8, 8, 8, true>, 8, 8, 8, 148);
  run("bulk load + bulk store", upd_bulk<8, 6, 8, true>, 8, 6, 8, 148);
  run("bulk load + bulk store", upd_bulk<8, 4, 8, true>, 8, 4, 8, 148);
  run("bulk load + bulk store", upd_bulk<4, 12, 4, true>, 4, 12, 4, 148);
  run("bulk load + bulk store", upd_bulk<16, 4, 16, true>, 16, 4, 16, 148);
  run("bulk load + bulk store", upd_bulk<16, 3, 16, true>, 16, 3, 16, 148);
  run("bulk load + st.global 2 CTA/SM", upd_bulk<8, 3, 8, false>, 8, 3, 8, 296);
  run("bulk load + bulk store 2 CTA/SM", upd_bulk<8, 3, 8, true>, 8, 3, 8, 296);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
