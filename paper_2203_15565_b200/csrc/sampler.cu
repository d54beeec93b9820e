// sampler.cu — bit-exact GPU restatement of the reference sampler.
//
// Reference: build_buffers (proj/include/pfc/sampler.hpp:63-126) drawing negatives with
// sample_without_replacement (proj/include/pfc/rng.hpp:101-123) on SeededRng::fork(k)
// (rng.hpp:49-51).  The reference runs a sequential partial Fisher-Yates over the
// materialised complement pool.  Here it is restated in parallel (SURVEY.md §7 hard part 1):
//
//   draw i (counter i+1, no rejection) gives j_i = i + r_i mod (N - i);
//   output slot i = P0[p*] where the chain p = j_i, t = i repeatedly steps to the largest
//   s < t with j_s = p (p = s, t = s) until none exists;
//   P0[p] = lo + p + #{m : pos_m - lo - m <= p}  (p-th element of [lo,hi) \ positives).
//
// A modulo rejection (probability <= n / 2^64 per draw) shifts every later counter; it is
// detected per shard and that shard is redone by an exact sequential kernel on the device.
#include "common.cuh"

namespace pfc {

constexpr int kMaxSortBatch = 8192;

// first index with a[i] >= v in the sorted keys a[0..n)
__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int64_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// minimum over the block (every thread gets it); red: 32 shared slots
__device__ __forceinline__ int64_t block_min_i64(int64_t v, int64_t* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int64_t r = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = red[w] < r ? red[w] : r;
  __syncthreads();
  return r;
}

// Exclusive block scan of one int per thread (blockDim.x == 1024).
__device__ int block_exclusive_scan(int v, int* smem_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = smem_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem_warp[lane] = w;
  }
  __syncthreads();
  const int before = (warp > 0 ? smem_warp[warp - 1] : 0) + x - v;
  if (total) *total = smem_warp[31];
  __syncthreads();
  return before;
}

// One CTA of 1024 threads: sort + unique the global batch labels, validate them, route
// positives to shards (sampler.hpp:68-80), check capacity in the reference's shard order
// (sampler.hpp:84-98), and locate every row's positive column (shardsim.hpp:207-213).
// Its thread 0 first opens the step (step_begin: the step's parameters and a status reset), so
// this kernel is the one node of the step's graph whose arguments change from step to step.
__global__ void __launch_bounds__(1024) positives_kernel(
    StepStatus* st, StepParams* sp, uint64_t seed, uint64_t stream, float lr, int reset,
    const float* x, const int64_t* labels_in, float* dx, int B, int64_t C, int K, int64_t blk,
    int cap, int k0, int nk, int64_t* __restrict__ uniq, ShardMeta* __restrict__ meta,
    int32_t* __restrict__ buf_cls, int32_t* __restrict__ pos_col, int force_sequential) {
  if (threadIdx.x == 0) step_begin(st, sp, seed, stream, lr, reset, x, labels_in, dx);
  __syncthreads();  // the block sees the step's parameters and the reset status
  // dynamic smem: keys[P] and the sorted unique labels us[P] (int32), then the batch labels[P]
  // (int64), staged once: in the host drop-in they are read from the caller's page-locked buffer
  // over PCIe (P = B rounded up to a power of 2)
  extern __shared__ int32_t keys[];
  __shared__ int warp_tmp[32];
  __shared__ int nuniq_s;
  __shared__ int64_t red[32];
  if (B > kMaxSortBatch) {
    if (threadIdx.x == 0) st->batch_too_large = 1;
    return;
  }
  int P = 1;
  while (P < B) P <<= 1;
  int64_t* labels = reinterpret_cast<int64_t*>(keys + 2 * P);
  // validation (sampler.hpp:72-78) reports the first invalid label of the SORTED unique list:
  // the smallest negative one, else the smallest one >= C.  With every label in [0, C),
  // C < 2^31, the sort and the searches below run on 32-bit keys.
  int64_t mn = INT64_MAX, mc = INT64_MAX;
  for (int i = threadIdx.x; i < B; i += blockDim.x) {
    const int64_t y = labels_in[i];
    labels[i] = y;
    mn = y < mn ? y : mn;
    if (y >= C && y < mc) mc = y;
  }
  mn = block_min_i64(mn, red);
  mc = block_min_i64(mc, red);
  if (mn < 0 || mc != INT64_MAX) {
    if (threadIdx.x == 0) {
      st->label_oob = 1;
      st->oob_label = mn < 0 ? mn : mc;
    }
    return;
  }
  if (P <= (int)blockDim.x) {
    // one key per thread: register bitonic sort, warp shuffles for partner distance < 32
    const int i = threadIdx.x;
    int32_t key = i < B ? (int32_t)labels[i] : INT32_MAX;
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        int32_t other;
        if (j >= 32) {
          if (i < P) keys[i] = key;
          __syncthreads();
          other = i < P ? keys[i ^ j] : key;
          __syncthreads();
        } else {
          other = __shfl_xor_sync(0xffffffffu, key, j);
        }
        const bool asc = (i & k) == 0, lower = i < (i ^ j);
        key = (asc == lower) ? min(key, other) : max(key, other);
      }
    }
    if (i < P) keys[i] = key;
    __syncthreads();
  } else {
    for (int i = threadIdx.x; i < P; i += blockDim.x) keys[i] = i < B ? (int32_t)labels[i] : INT32_MAX;
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const int32_t a = keys[i], b = keys[ixj];
            const bool asc = (i & k) == 0;
            if (asc ? (a > b) : (a < b)) {
              keys[i] = b;
              keys[ixj] = a;
            }
          }
        }
        __syncthreads();
      }
    }
  }
  // unique (sorted) into shared memory: each thread owns a contiguous run of keys
  int32_t* us = keys + P;
  __shared__ int bad_shard_s;
  const int per = (B + blockDim.x - 1) / blockDim.x;
  const int beg = threadIdx.x * per, end = min(B, beg + per);
  int cnt = 0;
  for (int i = beg; i < end; ++i) cnt += (i == 0 || keys[i] != keys[i - 1]);
  int total = 0;
  int pos = block_exclusive_scan(cnt, warp_tmp, &total);
  for (int i = beg; i < end; ++i)
    if (i == 0 || keys[i] != keys[i - 1]) us[pos++] = keys[i];
  if (threadIdx.x == 0) {
    nuniq_s = total;
    bad_shard_s = K;
  }
  __syncthreads();
  const int nu = nuniq_s;
  // capacity checks for ALL shards; the first failing shard in ascending order wins
  // (sampler.hpp:84-98)
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const int64_t lo = min((int64_t)k * blk, C), hi = min((int64_t)(k + 1) * blk, C);
    const int np = lower_bound_i32(us, nu, hi) - lower_bound_i32(us, nu, lo);
    if (np > cap || hi - lo < cap) atomicMin(&bad_shard_s, k);
  }
  __syncthreads();
  if (threadIdx.x == 0 && bad_shard_s < K) {
    const int k = bad_shard_s;
    const int64_t lo = min((int64_t)k * blk, C), hi = min((int64_t)(k + 1) * blk, C);
    st->capacity_shard = k;
    st->capacity_npos = lower_bound_i32(us, nu, hi) - lower_bound_i32(us, nu, lo);
  }
  __syncthreads();
  if (bad_shard_s < K) return;
  for (int kk = threadIdx.x; kk < nk; kk += blockDim.x) {
    const int k = k0 + kk;
    const int64_t lo = min((int64_t)k * blk, C), hi = min((int64_t)(k + 1) * blk, C);
    const int us0 = lower_bound_i32(us, nu, lo), ue = lower_bound_i32(us, nu, hi);
    ShardMeta m;
    m.lo = lo;
    m.hi = hi;
    m.npos = ue - us0;
    m.need = cap - m.npos;
    m.pool = (int)(hi - lo) - m.npos;
    m.full = (m.need == m.pool);
    m.ustart = us0;
    m.reject = force_sequential && !m.full && m.need > 0;
    meta[kk] = m;
  }
  // positives first, ascending (sampler.hpp:100-104)
  for (int i = threadIdx.x; i < nu; i += blockDim.x) {
    const int32_t y = us[i];
    const int k = (int)((uint32_t)y / (uint32_t)blk);
    if (k >= k0 && k < k0 + nk) {
      const int64_t lo = min((int64_t)k * blk, C);
      const int u0 = lower_bound_i32(us, nu, lo);
      buf_cls[(int64_t)(k - k0) * cap + (i - u0)] = y;
    }
  }
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int32_t y = (int32_t)labels[b];
    const int k = (int)((uint32_t)y / (uint32_t)blk);
    int col = -1;
    if (k >= k0 && k < k0 + nk) {
      const int64_t lo = min((int64_t)k * blk, C);
      col = (k - k0) * cap + (lower_bound_i32(us, nu, y) - lower_bound_i32(us, nu, lo));
    }
    pos_col[b] = col;
  }
}

// Per-draw counter RNG + modulo-rejection flag + per-position lists (j_s = p).  Blocks past
// the draws (blockIdx.x >= nblk_draws) normalise the features instead (independent work that
// shares the launch).
template <typename OT>
__global__ void draws_kernel(ShardMeta* __restrict__ meta, int nk, int cap,
                             const StepParams* __restrict__ sp, int k0, int64_t pool_stride,
                             int32_t* __restrict__ head, int32_t* __restrict__ nxt,
                             int32_t* __restrict__ jv, const StepStatus* st, int nblk_draws,
                             int B, int D, int Dp, OT* __restrict__ xh, float* __restrict__ xnorm) {
  if ((int)blockIdx.x >= nblk_draws) {
    normalize_x_rows(sp->x, B, D, Dp, xh, xnorm, (int)blockIdx.x - nblk_draws);
    return;
  }
  if (st->label_oob || st->capacity_shard >= 0 || st->batch_too_large) return;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)nk * cap) return;
  const int kk = (int)(gid / cap), i = (int)(gid % cap);
  const ShardMeta m = meta[kk];
  if (m.full || i >= m.need) return;
  const uint64_t key = rng_key(sp->seed, fork_stream(sp->stream, (uint64_t)(k0 + kk)));
  const uint64_t n = (uint64_t)(m.pool - i);
  const uint64_t r = rng_draw(key, (uint64_t)i + 1);
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;  // rng.hpp:69
  if (r >= limit) meta[kk].reject = 1;
  const int32_t j = i + (int32_t)(r % n);
  jv[gid] = j;
  nxt[gid] = atomicExch(&head[(int64_t)kk * pool_stride + j], i);
}

// p-th element of [lo, hi) minus the sorted positives pos[0..npos)
__device__ __forceinline__ int64_t pool_value(int64_t lo, const int32_t* pos, int npos,
                                              int64_t p) {
  // count m with q_m = pos_m - lo - m <= p  (q is non-decreasing)
  int a = 0, b = npos;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if ((int64_t)pos[mid] - lo - mid <= p) a = mid + 1; else b = mid;
  }
  return lo + p + a;
}

__device__ void sequential_fallback(ShardMeta* meta, int cap, const StepParams* sp, int k0,
                                    int64_t pool_stride, int32_t* pool_scratch, int32_t* buf_cls,
                                    StepStatus* st, int kk);

// Chain walk of the parallel Fisher-Yates restatement; the last nk blocks run the exact
// sequential sampler for shards that saw a modulo rejection (disjoint from the walked shards).
__global__ void walk_kernel(ShardMeta* __restrict__ meta, int nk, int cap,
                            int64_t pool_stride, const int32_t* __restrict__ head,
                            const int32_t* __restrict__ nxt, const int32_t* __restrict__ jv,
                            int32_t* __restrict__ buf_cls, StepStatus* st, int nblk_walk,
                            const StepParams* __restrict__ sp, int k0,
                            int32_t* __restrict__ pool_scratch) {
  if (st->label_oob || st->capacity_shard >= 0 || st->batch_too_large) return;
  if ((int)blockIdx.x >= nblk_walk) {
    sequential_fallback(meta, cap, sp, k0, pool_stride, pool_scratch, buf_cls, st,
                        (int)blockIdx.x - nblk_walk);
    return;
  }
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)nk * cap) return;
  const int kk = (int)(gid / cap), i = (int)(gid % cap);
  const ShardMeta m = meta[kk];
  if (m.reject || i >= m.need) return;
  int32_t* row = buf_cls + (int64_t)kk * cap;
  int64_t p;
  if (m.full) {
    p = i;  // full sampling: ascending complement (sampler.hpp:106-115)
  } else {
    const int32_t* hd = head + (int64_t)kk * pool_stride;
    const int32_t* nx = nxt + (int64_t)kk * cap;
    int32_t pp = jv[(int64_t)kk * cap + i], t = i;
    for (;;) {
      int32_t best = -1;
      for (int32_t s = hd[pp]; s >= 0; s = nx[s])
        if (s < t && s > best) best = s;
      if (best < 0) break;
      pp = best;
      t = best;
    }
    p = pp;
  }
  row[m.npos + i] = (int32_t)pool_value(m.lo, row, m.npos, p);
}

// Exact sequential sample_without_replacement for shards that saw a modulo rejection
// (or when forced for testing).  One CTA per local shard (walk_kernel's trailing blocks).
__device__ void sequential_fallback(ShardMeta* meta, int cap, const StepParams* sp, int k0,
                                    int64_t pool_stride, int32_t* pool_scratch, int32_t* buf_cls,
                                    StepStatus* st, int kk) {
  const ShardMeta m = meta[kk];
  if (!m.reject) return;
  int32_t* row = buf_cls + (int64_t)kk * cap;
  int32_t* pool = pool_scratch + (int64_t)kk * pool_stride;
  for (int64_t p = threadIdx.x; p < m.pool; p += blockDim.x)
    pool[p] = (int32_t)pool_value(m.lo, row, m.npos, p);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&st->rejection_shards, 1);
    const uint64_t key = rng_key(sp->seed, fork_stream(sp->stream, (uint64_t)(k0 + kk)));
    uint64_t counter = 0;
    for (int i = 0; i < m.need; ++i) {
      const uint64_t n = (uint64_t)(m.pool - i);
      const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
      uint64_t r = rng_draw(key, ++counter);
      while (r >= limit) r = rng_draw(key, ++counter);
      const int64_t j = i + (int64_t)(r % n);
      const int32_t t = pool[i];
      pool[i] = pool[j];
      pool[j] = t;
      row[m.npos + i] = pool[i];
    }
  }
}

}  // namespace pfc
