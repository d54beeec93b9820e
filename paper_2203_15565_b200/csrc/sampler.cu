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
#include <climits>

#include "common.cuh"

namespace pfc {

constexpr int kMaxBatch = 1 << 20;  // global batch rows (pfc_gpu_desc::max_batch)

// ---- build_buffers (sampler.hpp:63-126) in three kernels: a bitmap over the C classes instead
// of a sort, and the parallel Fisher-Yates restatement.
//   mark_kernel (opens the step): every valid label sets its class bit and, when the bit was new,
//      counts it in its chunk (chunk_words words); the two smallest invalid labels are kept (the
//      reference validates the sorted unique list: the smallest negative one, else the smallest
//      one >= C); the labels are copied to the device (host drop-in: read once over PCIe)
//   fill_kernel, every CTA redundantly: chunk prefixes in shared memory; validation; every
//      shard's distinct-positive count against the capacity in ascending shard order
//      (sampler.hpp:84-98); the local shards' metadata (CTA 0 publishes it); then the positives
//      of the local shards ascending (a class's rank among the set bits of its shard is its
//      buffer slot, sampler.hpp:100-104), each row's positive column (shardsim.hpp:207-213), the
//      draws (counter RNG, rejection flag, per-position lists) and x^ = x / |x|
//   walk_kernel: chain walk; the exact sequential sampler for shards that saw a modulo
//      rejection; the bitmap and chunk counts are cleared again (all-zero between steps: no
//      per-step pass over all C classes)
// Grid-stride loops over one CTA of 1024 threads per SM; the kernels are chained by PDL.
constexpr int kSamplerThreads = 1024;
constexpr int kMaxSamplerChunks = 16384;      // chunk prefixes kept in shared memory
constexpr int kMaxSamplerLocalShards = 2048;  // local shard metadata kept in shared memory

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Set bits of the bitmap below class x (warp-collective): the chunk prefix plus a popcount of
// the words of x's chunk before it (coalesced, 32 words per instruction).
__device__ __forceinline__ int bits_below(const uint32_t* bits, const int32_t* bpre_s,
                                          int chunk_words, int64_t x, int lane) {
  const int64_t w = x >> 5;
  const int64_t ch = w / chunk_words;
  int cnt = 0;
  if (chunk_words == 32) {  // one word per lane: a single round trip
    const int64_t i = ch * 32 + lane;
    if (i <= w) {
      const uint32_t v = bits[i];
      cnt = __popc(i < w ? v : (v & ((1u << (x & 31)) - 1u)));
    }
    return bpre_s[ch] + warp_sum_i(cnt);
  }
  // 8 independent loads in flight per lane (not one dependent L2 round trip per 32 words)
  int64_t i = ch * chunk_words + lane;
  for (; i + 7 * 32 < w; i += 8 * 32) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = bits[i + u * 32];
#pragma unroll
    for (int u = 0; u < 8; ++u) cnt += __popc(v[u]);
  }
  for (; i < w; i += 32) cnt += __popc(bits[i]);
  if (lane == 0) cnt += __popc(bits[w] & ((1u << (x & 31)) - 1u));
  return bpre_s[ch] + warp_sum_i(cnt);
}

// bits_below at two points with both loads in flight together (the capacity check's shard
// bounds); the per-lane counts (<= 32 each) travel packed through one warp sum.
__device__ __forceinline__ int2 bits_below2(const uint32_t* bits, const int32_t* bpre_s,
                                            int chunk_words, int64_t x0, int64_t x1, int lane) {
  if (chunk_words != 32)
    return make_int2(bits_below(bits, bpre_s, chunk_words, x0, lane),
                     bits_below(bits, bpre_s, chunk_words, x1, lane));
  const int64_t w0 = x0 >> 5, w1 = x1 >> 5;
  const int64_t i0 = (w0 & ~31ll) + lane, i1 = (w1 & ~31ll) + lane;
  const uint32_t v0 = i0 <= w0 ? bits[i0] : 0u, v1 = i1 <= w1 ? bits[i1] : 0u;
  const int c0 = __popc(i0 < w0 ? v0 : (v0 & ((1u << (x0 & 31)) - 1u)));
  const int c1 = __popc(i1 < w1 ? v1 : (v1 & ((1u << (x1 & 31)) - 1u)));
  const int t = warp_sum_i(c0 | (c1 << 16));
  return make_int2(bpre_s[w0 >> 5] + (t & 0xffff), bpre_s[w1 >> 5] + (t >> 16));
}

__device__ int block_exclusive_scan(int v, int* smem_warp, int* total);

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

// Exact sequential sample_without_replacement for a shard that saw a modulo rejection (or when
// forced for testing), by one CTA: the complement pool, then the reference's loop.
__device__ void sequential_fallback(const ShardMeta& m, int cap, const StepParams* sp, int k0,
                                    int64_t pool_stride, int32_t* pool_scratch, int32_t* buf_cls,
                                    StepStatus* st, int kk) {
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
  __syncthreads();
}

struct SamplerArgs {
  StepStatus* st;
  StepParams* sp;
  uint64_t seed, stream;
  float lr;
  int reset;
  const float* x;
  const int64_t* labels_in;  // device or page-locked host labels of the global batch
  float* dx;
  int B;
  int64_t C;
  int K;
  int64_t blk;
  int cap, k0, nk;
  int force_sequential;
  int normalize;             // 1: phase D also normalises the features (device path)
  int D, Dp;
  void* xh;                  // x^ in the GEMM operand type
  float* xnorm;
  uint32_t* bits;            // [nwords] class bitmap
  int32_t* ccnt;             // [nchunk] set bits per chunk
  int chunk_words, nchunk;
  long long* oobs;           // [2] smallest negative / >= C label (LLONG_MAX: none)
  int32_t* rej;              // [nk] modulo rejection seen by a draw
  int64_t* labs;
  double* zpos;
  int* hasval;
  ShardMeta* meta;           // [nk] published for the later kernels and pfc_gpu_get_buffers
  int32_t* buf_cls;
  int32_t* pos_col;
  int32_t* head;
  int32_t* nxt;
  int32_t* jv;
  int32_t* pool_scratch;
  int64_t pool_stride;
};

__host__ __device__ constexpr size_t sampler_smem_bytes(int nchunk, int nk) {
  return (size_t)nchunk * sizeof(int32_t) + (size_t)nk * sizeof(ShardMeta);
}

// walk_kernel: shard metadata, each local shard's offset into the staged positives, and the
// positives themselves when they fit (kWalkPositives), for pool_value's binary searches
constexpr int kWalkPositives = 8192;
__host__ __device__ constexpr size_t walk_smem_bytes(int nk) {
  return (size_t)nk * (sizeof(ShardMeta) + sizeof(int32_t)) + (size_t)kWalkPositives * sizeof(int32_t);
}

// Opens the step (thread 0: step_begin) and marks the labels.
__global__ void __launch_bounds__(kSamplerThreads) mark_kernel(const SamplerArgs a) {
  pdl_entry();
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) step_begin(a.st, a.sp, a.seed, a.stream, a.lr, a.reset, a.x, a.labels_in, a.dx);
  for (int64_t b = tid; b < a.B; b += nthr) {
    const int64_t y = a.labels_in[b];
    a.labs[b] = y;
    a.zpos[b] = 0.0;  // the logits epilogue writes the local positives' z_pos; 0 elsewhere
    if (a.hasval) a.hasval[b] = 0;
    if (y < 0) {
      atomicMin(&a.oobs[0], (long long)y);
    } else if (y >= a.C) {
      atomicMin(&a.oobs[1], (long long)y);
    } else {
      const uint32_t bit = 1u << (y & 31);
      if (!(atomicOr(&a.bits[y >> 5], bit) & bit)) atomicAdd(&a.ccnt[(y >> 5) / a.chunk_words], 1);
    }
  }
  for (int64_t kk = tid; kk < a.nk; kk += nthr) a.rej[kk] = 0;
}

// fill_kernel's second half: positives + positive columns (one warp per label), draws (one
// thread per draw)
__device__ __forceinline__ void draw_phase(const SamplerArgs& a, const ShardMeta* meta_s,
                                           const int32_t* bpre_s, int lane, int64_t gwarp,
                                           int64_t nwarp, int64_t tid, int64_t nthr) {
  for (int64_t b = gwarp; b < a.B; b += nwarp) {
    const int64_t y = a.labs[b];
    const int k = (int)(y / a.blk);
    int col = -1;
    if (k >= a.k0 && k < a.k0 + a.nk) {
      const int kk = k - a.k0;
      col = kk * a.cap + (bits_below(a.bits, bpre_s, a.chunk_words, y, lane) - meta_s[kk].ustart);
      if (lane == 0) a.buf_cls[col] = (int32_t)y;
    }
    if (lane == 0) a.pos_col[b] = col;
  }
  const int64_t nd = (int64_t)a.nk * a.cap;
  for (int64_t g = tid; g < nd; g += nthr) {
    const int kk = (int)(g / a.cap), i = (int)(g % a.cap);
    const ShardMeta& m = meta_s[kk];
    if (m.full || i >= m.need) continue;
    // per-step values from the StepParams block (only mark_kernel's arguments change per step)
    const uint64_t key = rng_key(a.sp->seed, fork_stream(a.sp->stream, (uint64_t)(a.k0 + kk)));
    const uint64_t n = (uint64_t)(m.pool - i);
    const uint64_t r = rng_draw(key, (uint64_t)i + 1);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;  // rng.hpp:69
    if (r >= limit) a.rej[kk] = 1;
    const int32_t j = i + (int32_t)(r % n);
    a.jv[g] = j;
    a.nxt[g] = atomicExch(&a.head[(int64_t)kk * a.pool_stride + j], i);
  }
}

template <typename OT>
__global__ void __launch_bounds__(kSamplerThreads, 1) fill_kernel(const SamplerArgs a) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t sampler_smem[];
  ShardMeta* meta_s = reinterpret_cast<ShardMeta*>(sampler_smem);
  int32_t* bpre_s = reinterpret_cast<int32_t*>(sampler_smem + (size_t)a.nk * sizeof(ShardMeta));
  __shared__ int warp_tmp[32];
  __shared__ int bad_shard_s;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t gwarp = tid >> 5, nwarp = nthr >> 5;
  StepStatus* st = a.st;
  // ---- chunk prefixes (each thread a run of up to 16 consecutive chunks, one block scan),
  // validation, capacity, local shard metadata (every CTA)
  {
    const int per = (a.nchunk + kSamplerThreads - 1) / kSamplerThreads;
    const int i0 = (int)threadIdx.x * per;
    int v[kMaxSamplerChunks / kSamplerThreads];
    int run = 0;
#pragma unroll
    for (int u = 0; u < kMaxSamplerChunks / kSamplerThreads; ++u) {
      v[u] = (u < per && i0 + u < a.nchunk) ? a.ccnt[i0 + u] : 0;
      run += v[u];
    }
    int ex = block_exclusive_scan(run, warp_tmp, nullptr);
#pragma unroll
    for (int u = 0; u < kMaxSamplerChunks / kSamplerThreads; ++u) {
      if (u < per && i0 + u < a.nchunk) bpre_s[i0 + u] = ex;
      ex += v[u];
    }
  }
  if (threadIdx.x == 0) bad_shard_s = a.K;
  const long long mn = a.oobs[0], mc = a.oobs[1];
  __syncthreads();
  const bool sticky = sampler_failed(st);  // an earlier asynchronous step's error stays first
  const bool oob = mn != LLONG_MAX || mc != LLONG_MAX;
  if (!sticky && !oob) {
    // capacity checks for ALL shards, one warp per shard; the first failing shard wins
    for (int k = wib; k < a.K; k += blockDim.x >> 5) {
      const int64_t lo = min((int64_t)k * a.blk, a.C), hi = min((int64_t)(k + 1) * a.blk, a.C);
      const int2 pb = bits_below2(a.bits, bpre_s, a.chunk_words, lo, hi, lane);
      const int plo = pb.x, np = pb.y - pb.x;
      if (np > a.cap || hi - lo < a.cap) {
        if (lane == 0) atomicMin(&bad_shard_s, k);
      } else if (k >= a.k0 && k < a.k0 + a.nk && lane == 0) {
        ShardMeta m;
        m.lo = lo;
        m.hi = hi;
        m.ustart = plo;
        m.npos = np;
        m.need = a.cap - np;
        m.pool = (int)(hi - lo) - np;
        m.full = (m.need == m.pool);
        m.reject = a.force_sequential && !m.full && m.need > 0;
        meta_s[k - a.k0] = m;
      }
    }
  }
  __syncthreads();
  const int bad = bad_shard_s;
  const bool ok = !sticky && !oob && bad == a.K;
  if (blockIdx.x == 0) {
    if (!sticky && threadIdx.x == 0) {
      if (oob) {
        st->label_oob = 1;
        st->oob_label = mn != LLONG_MAX ? mn : mc;
      } else if (bad < a.K) {
        st->capacity_shard = bad;
      }
    }
    if (!sticky && !oob && bad < a.K && wib == 0) {  // the failing shard's count, for the message
      const int64_t lo = min((int64_t)bad * a.blk, a.C), hi = min((int64_t)(bad + 1) * a.blk, a.C);
      const int np = bits_below(a.bits, bpre_s, a.chunk_words, hi, lane) -
                     bits_below(a.bits, bpre_s, a.chunk_words, lo, lane);
      if (lane == 0) st->capacity_npos = np;
    }
    if (ok)
      for (int kk = threadIdx.x; kk < a.nk; kk += blockDim.x) a.meta[kk] = meta_s[kk];
  }
  if (ok) draw_phase(a, meta_s, bpre_s, lane, gwarp, nwarp, tid, nthr);
  if (a.normalize) {  // x^ = x / |x| last: only the GEMMs after the sampler read it
    const int nw = (int)nwarp;
    for (int row0 = 0; row0 < a.B; row0 += nw)
      normalize_x_rows(a.sp->x + (size_t)row0 * a.D, a.B - row0, a.D, a.Dp,
                       static_cast<OT*>(a.xh) + (size_t)row0 * a.Dp, a.xnorm + row0,
                       (int)blockIdx.x);
  }
}

// Chain walk (+ the exact sequential fallback of rejected shards); clears the bitmap.
__global__ void __launch_bounds__(kSamplerThreads) walk_kernel(const SamplerArgs a) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t sampler_smem[];
  ShardMeta* meta_s = reinterpret_cast<ShardMeta*>(sampler_smem);
  int32_t* off_s = reinterpret_cast<int32_t*>(sampler_smem + (size_t)a.nk * sizeof(ShardMeta));
  int32_t* pos_s = off_s + a.nk;
  __shared__ int warp_tmp[32];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = tid; b < a.B; b += nthr) {
    const int64_t y = a.labs[b];
    if (y >= 0 && y < a.C) {
      a.bits[y >> 5] = 0u;
      a.ccnt[(y >> 5) / a.chunk_words] = 0;
    }
  }
  if (tid == 0) {
    a.oobs[0] = LLONG_MAX;
    a.oobs[1] = LLONG_MAX;
  }
  if (sampler_failed(a.st)) return;
  for (int kk = threadIdx.x; kk < a.nk; kk += blockDim.x) {
    ShardMeta m = a.meta[kk];
    m.reject = m.reject || a.rej[kk];
    meta_s[kk] = m;
  }
  __syncthreads();
  for (int kk = blockIdx.x; kk < a.nk; kk += gridDim.x)
    if (meta_s[kk].reject)  // block-uniform
      sequential_fallback(meta_s[kk], a.cap, a.sp, a.k0, a.pool_stride, a.pool_scratch,
                          a.buf_cls, a.st, kk);
  // the local shards' positives (fill_kernel wrote them) into shared memory when they fit:
  // pool_value's binary search then costs no dependent global round trips
  int npos_all = 0;
  for (int base = 0; base < a.nk; base += blockDim.x) {
    const int kk = base + (int)threadIdx.x;
    int tot = 0;
    const int ex = block_exclusive_scan(kk < a.nk ? meta_s[kk].npos : 0, warp_tmp, &tot);
    if (kk < a.nk) off_s[kk] = npos_all + ex;
    npos_all += tot;
  }
  const bool staged = npos_all <= kWalkPositives;
  if (staged) {
    const int lane = threadIdx.x & 31;
    for (int kk = threadIdx.x >> 5; kk < a.nk; kk += blockDim.x >> 5) {
      const int32_t* src = a.buf_cls + (int64_t)kk * a.cap;
      for (int i = lane; i < meta_s[kk].npos; i += 32) pos_s[off_s[kk] + i] = src[i];
    }
  }
  __syncthreads();
  const int64_t nd = (int64_t)a.nk * a.cap;
  for (int64_t g = tid; g < nd; g += nthr) {
    const int kk = (int)(g / a.cap), i = (int)(g % a.cap);
    const ShardMeta& m = meta_s[kk];
    if (m.reject || i >= m.need) continue;
    int32_t* row = a.buf_cls + (int64_t)kk * a.cap;
    int64_t p;
    if (m.full) {
      p = i;  // full sampling: ascending complement (sampler.hpp:106-115)
    } else {
      const int32_t* hd = a.head + (int64_t)kk * a.pool_stride;
      const int32_t* nx = a.nxt + (int64_t)kk * a.cap;
      int32_t pp = a.jv[g], t = i;
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
    row[m.npos + i] = (int32_t)pool_value(m.lo, staged ? pos_s + off_s[kk] : row, m.npos, p);
  }
}

}  // namespace pfc
