// Calibration microkernel for the ncu tensor-pipe counters ("find the counter that
// tracks UTCHMMA issue on a pure-MMA kernel of known FLOP rate").  Every CTA (one per SM) issues
// `iters` back-to-back tcgen05.mma.cta_group::1.kind::f16 (bf16, M=128, N=256, K=16) from
// shared-memory operands into one TMEM accumulator, then commits once and waits.  No loads, no
// epilogue: the kernel runs at the MMA issue floor, so the FLOP rate is exactly known from the
// instruction count and the event-timed duration, and a tensor-activity counter that tracks
// UTCHMMA must read ~100% of the kernel's elapsed cycles.
//   ./mma_rate [iters]  -> prints TFLOP/s; run under ncu with the candidate metrics
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_rate mma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../../paper_2203_15565_b200/csrc/sm100.cuh"

using namespace pfc_sm100;

__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int iters, int kind_tf32, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                 // 128 x 128 B (K-major, SW128)
  uint8_t* sB = smem + 16384;         // 256 x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 32768);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;  // small finite values
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {
    const uint32_t idesc = kind_tf32 ? make_idesc_tf32(128, 256, false, false)
                                     : make_idesc_bf16(128, 256, false, false);
    const uint32_t a = smem_u32(sA), b = smem_u32(sB);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = make_sdesc_sw128(a + k * 32, 0, 1024);
        const uint64_t bd = make_sdesc_sw128(b + k * 32, 0, 1024);
        if (kind_tf32) umma_tf32(tmem, ad, bd, idesc, (it | k) ? 1u : 0u);
        else umma_bf16(tmem, ad, bd, idesc, (it | k) ? 1u : 0u);
      }
    }
    umma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  __syncthreads();
  if (warp == 0) {
    float v[32];
    tmem_ld32(tmem, v);
    if (v[lane] == 12345.f) sink[blockIdx.x] = v[0];
    tc_fence_before();
    tmem_dealloc(tmem, 256);
  }
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 4096);
  const int smem = 1024 + 16384 + 32768 + 64;
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int tf = 0; tf < 2; ++tf) {
    mma_rate_kernel<<<sms, 128, smem>>>(iters / 10, tf, sink);  // warm-up
    cudaEventRecord(e0);
    mma_rate_kernel<<<sms, 128, smem>>>(iters, tf, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // per MMA: M 128 x N 256 x K (16 bf16 | 8 tf32) x 2 flops; 4 MMAs per iteration
    const double kk = tf ? 8.0 : 16.0;
    const double flops = (double)sms * iters * 4 * 2.0 * 128 * 256 * kk;
    printf("%s: %d SMs x %d iters x 4 MMA (128x256x%d): %.3f ms  %.1f TFLOP/s  (%s)\n",
           tf ? "kind::tf32" : "kind::f16 bf16", sms, iters, (int)kk, ms, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
