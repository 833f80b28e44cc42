// dq_stats_alloc.cu — super-group statistics and the fast bit allocator on device.
//
// Statistics (proj/src/stats.cpp:23-54): the reference sums every super-group
// sequentially in fp64; fp64 addition is not associative, so the only way to be
// bit-exact is to keep that order.  k_stats stages a 128-super-group x 32-entry
// tile through shared memory with fully coalesced 128-byte row loads and lets
// each thread run its super-group's sequential fp64 chain from the conflict-free
// (stride 33) tile — HBM-bound, the fp64 adds are ~15% of the issue budget.
//
// Fast allocator (proj/src/allocation.cpp:170-260): payload(u) is a step
// function whose steps sit at the flips 4 - a*log2(F_j) (width 2->4, +2 bits per
// entry) and 8 - a*log2(F_j) (4->8, +4); the reference sorts all 2T flips and
// bisects over plateau midpoints.  Here the crossing flip — the first flip, in
// ascending order, at which the cumulative weight exceeds the budget — is
// found with no sort: each pass histograms the flips of the current key range
// into 1024 bins (order-preserving u64 keys of the doubles, so ranges are exact),
// a one-CTA scan picks the bin where the weight crosses, and the next pass
// narrows to that bin's [min, max] key.  <= 8 passes isolate a single flip value
// (each pass removes >= 9 bits of key range); the plateau midpoint with its
// predecessor is then u exactly as the reference computes it.
#include <cfloat>
#include <cstdint>

#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "dq_internal.h"

namespace dq {

// ------------------------------------------------------------ statistics
constexpr int kStatSG = 128;

// PEER: the statistics all-gather fused into the kernel — every block stores its
// super-groups' (mean, sq) into row `me` of every rank's statistics area over NVLink;
// the last block to finish (system-scope fences before the completion count) raises
// row me's flag on every rank.  The reduction waits for all rows' flags.
template <bool PEER>
__global__ void __launch_bounds__(kStatSG) k_stats(const WorkerPtrs xs, uint64_t d, uint32_t T,
                                                   float* mean, float* sq, StatsPeerArgs sp) {
  __shared__ float tile[kStatSG][33];
  pdl_wait();
  pdl_trigger();
  const float* __restrict__ x = xs.p[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PEER: a persistent grid walks the tiles, so the one system-scope fence per block
  // before the completion count is amortised over many tiles
  const uint32_t ntiles = (T + kStatSG - 1) / kStatSG;
  for (uint32_t tile_i = blockIdx.x; tile_i < ntiles; tile_i += PEER ? gridDim.x : ntiles) {
    const uint32_t sg0 = tile_i * kStatSG;
    double s = 0.0, q = 0.0;
#pragma unroll 1
    for (int part = 0; part < kS / 32; ++part) {
      float v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const uint32_t sg = sg0 + warp * 32 + r;
        const uint64_t idx = static_cast<uint64_t>(sg) * kS + part * 32 + lane;
        v[r] = (sg < T && idx < d) ? __ldcs(x + idx) : 0.0f;  // streaming: read once
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) tile[warp * 32 + r][lane] = v[r];
      __syncthreads();
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double t = tile[threadIdx.x][k];
        s = __dadd_rn(s, t);
        q = __dadd_rn(q, __dmul_rn(t, t));
      }
      __syncthreads();
    }
    const uint32_t sg = sg0 + threadIdx.x;
    if constexpr (!PEER) {
      if (sg < T) {
        mean[static_cast<uint64_t>(blockIdx.y) * T + sg] = static_cast<float>(__ddiv_rn(s, static_cast<double>(kS)));
        sq[static_cast<uint64_t>(blockIdx.y) * T + sg] = static_cast<float>(q);
      }
    } else {
      if (sg < T) {
        const float mv = static_cast<float>(__ddiv_rn(s, static_cast<double>(kS))), qv = static_cast<float>(q);
        for (uint32_t r = 0; r < sp.n; ++r) {
          sp.mean[r][sg] = mv;
          sp.sq[r][sg] = qv;
        }
      }
    }
  }
  if constexpr (PEER) {
    __syncthreads();
    __shared__ unsigned int last;
    if (threadIdx.x == 0) {
      __threadfence_system();
      last = atomicAdd(sp.done, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      *sp.done = 0;  // reset for the next round (stream-ordered before its stats kernel)
      const uint32_t epoch = *sp.epoch + 1;  // this round's epoch, read by its later kernels
      *sp.epoch = epoch;
      __threadfence_system();
      for (uint32_t r = 0; r < sp.n; ++r)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sp.flag[r]), "r"(epoch) : "memory");
    }
  }
}

WorkerPtrs worker_ptrs(const float* const* host_ptrs, uint32_t n) {
  WorkerPtrs w{};
  for (uint32_t r = 0; r < n && r < 64; ++r) w.p[r] = host_ptrs[r];
  return w;
}

void launch_stats(const float* const* xs, uint32_t n_workers, uint64_t d, uint32_t T, float* mean,
                  float* sq, cudaStream_t st) {
  if (T == 0) return;
  launch_pdl(k_stats<false>, dim3((T + kStatSG - 1) / kStatSG, n_workers), dim3(kStatSG), 0, st,
             worker_ptrs(xs, n_workers), d, T, mean, sq, StatsPeerArgs{});
}

void launch_stats_peer(const float* const* xs, uint64_t d, uint32_t T, const StatsPeerArgs& sp, cudaStream_t st) {
  if (T == 0) return;
  // one wave of the persistent grid: exactly the CTAs that are resident at once (register-
  // limited), so every CTA walks the same number of tiles and none waits for a second wave
  static int cache[kMaxDevices] = {};
  const uint32_t cap = static_cast<uint32_t>(per_device(cache, [](int dev) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stats<true>, kStatSG, 0);
    return (sms > 0 ? sms : 148) * (per_sm > 0 ? per_sm : 4);
  }));
  const uint32_t ntiles = (T + kStatSG - 1) / kStatSG;
  launch_pdl(k_stats<true>, dim3(ntiles < cap ? ntiles : cap, 1), dim3(kStatSG), 0, st, worker_ptrs(xs, 1), d, T,
             static_cast<float*>(nullptr), static_cast<float*>(nullptr), sp);
}

__global__ void k_reduce_stats(const float* mean, const float* sq, uint32_t n, uint32_t T,
                               float* gm, float* gs) {
  pdl_wait();
  pdl_trigger();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= T) return;
  double a = 0.0, b = 0.0;
  for (uint32_t r = 0; r < n; ++r) {
    a = __dadd_rn(a, static_cast<double>(mean[static_cast<uint64_t>(r) * T + j]));
    b = __dadd_rn(b, static_cast<double>(sq[static_cast<uint64_t>(r) * T + j]));
  }
  gm[j] = static_cast<float>(__ddiv_rn(a, static_cast<double>(n)));
  gs[j] = static_cast<float>(b);
}

void launch_reduce_stats(const float* mean, const float* sq, uint32_t n, uint32_t T, float* gm,
                         float* gs, cudaStream_t st) {
  if (T == 0) return;
  launch_pdl(k_reduce_stats, dim3((T + 255) / 256), dim3(256), 0, st, mean, sq, n, T, gm, gs);
}

// The rank-ordered reduction over the fused all-gather's rows: each block first waits
// (thread 0, acquire at system scope, g_spin_ns timeout -> trap) for every row's flag.
__global__ void k_reduce_stats_peer(const float* mean, const float* sq, const uint32_t* flags,
                                    const uint32_t* epoch_ptr, uint32_t n, uint32_t T, uint32_t stride, float* gm,
                                    float* gs) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    const uint32_t epoch = *epoch_ptr;
    for (uint32_t r = 0; r < n; ++r) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + r) : "memory");
      if (v == epoch) continue;
      const uint64_t t0 = dq_globaltimer();
      for (;;) {
        __nanosleep(64);
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + r) : "memory");
        if (v == epoch) break;
        if (dq_globaltimer() - t0 > g_spin_ns) __trap();
      }
    }
  }
  __syncthreads();
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= T) return;
  double a = 0.0, b = 0.0;
  for (uint32_t r = 0; r < n; ++r) {
    a = __dadd_rn(a, static_cast<double>(__ldcg(mean + static_cast<uint64_t>(r) * stride + j)));
    b = __dadd_rn(b, static_cast<double>(__ldcg(sq + static_cast<uint64_t>(r) * stride + j)));
  }
  gm[j] = static_cast<float>(__ddiv_rn(a, static_cast<double>(n)));
  gs[j] = static_cast<float>(b);
}

void launch_reduce_stats_peer(const float* mean, const float* sq, const uint32_t* flags, const uint32_t* epoch,
                              uint32_t n, uint32_t T, uint32_t stride, float* gm, float* gs, cudaStream_t st) {
  if (T == 0) return;
  launch_pdl(k_reduce_stats_peer, dim3((T + 255) / 256), dim3(256), 0, st, mean, sq, flags, epoch, n, T, stride, gm, gs);
}

// ------------------------------------------------------------ allocation
__device__ __forceinline__ uint64_t dkey(double f) {
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(f));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Block-wide reduction of one u64 (all threads call; the result is valid in thread 0),
// so each CTA issues one global atomic per quantity instead of one per warp: the
// state words are single addresses and per-warp atomics serialise at L2.
enum RedOp { kRedMin, kRedMax, kRedAdd };
template <RedOp OP>
__device__ __forceinline__ unsigned long long red_op(unsigned long long a, unsigned long long b) {
  return OP == kRedMin ? (a < b ? a : b) : (OP == kRedMax ? (a > b ? a : b) : a + b);
}
template <RedOp OP>
__device__ unsigned long long block_reduce(unsigned long long v) {
  __shared__ unsigned long long part[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_op<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) part[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long id = OP == kRedMin ? ~0ull : 0ull;
    v = lane < nw ? part[lane] : id;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = red_op<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
  }
  __syncthreads();
  return v;
}

__device__ void alloc_init(AllocState* s, uint64_t* bins, uint64_t wmax) {
  const int t = threadIdx.x;
  for (int b = t; b < kAllocBins; b += blockDim.x) {
    bins[4 * b + 0] = 0;
    bins[4 * b + 1] = 0;
    bins[4 * b + 2] = ~0ull;
    bins[4 * b + 3] = 0;
  }
  if (t == 0) {
    const uint32_t epoch = s->epoch;  // the mailbox tag survives the reset (one per round)
    *s = AllocState{};
    s->epoch = epoch;
    s->kmin = ~0ull;
    s->kmax = 0;
    s->wmax = wmax;
  }
}

__device__ void alloc_prep(const float* __restrict__ F, uint32_t T, double alpha, double* level,
                           AllocState* s) {
  uint64_t kmin = ~0ull, kmax = 0;
  uint32_t npos = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const float f = F[j];
    double l = __longlong_as_double(0x7ff8000000000000ll);  // NaN: no flips (allocation.cpp:206)
    if (f > 0.0f) {
      l = __dmul_rn(alpha, log2(static_cast<double>(f)));
      kmin = min(kmin, dkey(__dsub_rn(4.0, l)));
      kmax = max(kmax, dkey(__dsub_rn(8.0, l)));
      ++npos;
    }
    level[j] = l;
  }
  kmin = block_reduce<kRedMin>(kmin);
  kmax = block_reduce<kRedMax>(kmax);
  const unsigned long long np = block_reduce<kRedAdd>(npos);
  if (threadIdx.x == 0 && np) {
    atomicMin(reinterpret_cast<unsigned long long*>(&s->kmin), kmin);
    atomicMax(reinterpret_cast<unsigned long long*>(&s->kmax), kmax);
    atomicAdd(&s->npos, static_cast<uint32_t>(np));
  }
}

__device__ void alloc_start(AllocState* s) {
  if (s->npos == 0) {
    s->status = 3;
  } else {
    s->klo = s->kmin;
    s->khi = s->kmax;
  }
}

// Bins of the current pass: kAllocBins equal slices of [klo, khi] in key space
// (order-preserving u64 keys of the flip doubles).  Only weight and count per bin
// (native 32-bit shared atomics: 64-bit shared min/max would be CAS loops under
// contention); the next pass narrows to the crossing bin's slice.
__device__ __forceinline__ int alloc_shift(const AllocState* s) {
  const uint64_t span = s->khi - s->klo;
  const int bits = span ? 64 - __clzll(static_cast<long long>(span)) : 0;
  return bits > 10 ? bits - 10 : 0;
}

constexpr uint32_t kCollectMax = 256;  // crossing-bin flips finished by rank counting

struct HistSmem {
  uint32_t bw[kAllocBins], bc[kAllocBins];
  unsigned long long bmn[kAllocBins];  // alloc_finish: sort keys
};
__device__ void alloc_hist(const double* __restrict__ level, uint32_t T, const AllocState* s, uint64_t* bins,
                           HistSmem& hs) {
  uint32_t* bw = hs.bw;
  uint32_t* bc = hs.bc;
  for (int b = threadIdx.x; b < kAllocBins; b += blockDim.x) {
    bw[b] = 0;
    bc[b] = 0;
  }
  __syncthreads();
  const uint64_t klo = s->klo, span = s->khi - s->klo;
  const int shift = alloc_shift(s);
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const double l = level[j];
    if (l != l) continue;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint64_t k = dkey(__dsub_rn(t ? 8.0 : 4.0, l));
      if (k - klo <= span) {  // unsigned: k in [klo, khi]
        const uint32_t b = static_cast<uint32_t>((k - klo) >> shift);
        atomicAdd(&bw[b], t ? 4u : 2u);
        atomicAdd(&bc[b], 1u);
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kAllocBins; b += blockDim.x) {
    if (bc[b] == 0) continue;
    unsigned long long* g = reinterpret_cast<unsigned long long*>(bins + 4 * b);
    atomicAdd(g + 0, static_cast<unsigned long long>(bw[b]));
    atomicAdd(g + 1, static_cast<unsigned long long>(bc[b]));
  }
}

__device__ void alloc_scan(AllocState* s, uint64_t* bins) {  // one CTA of kAllocBins threads
  __shared__ uint64_t wsum[32];
  __shared__ uint32_t cross_bin;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint64_t w = bins[4 * t], c = bins[4 * t + 1];
  bins[4 * t] = 0;
  bins[4 * t + 1] = 0;
  if (t == 0) cross_bin = 0xffffffffu;
  // block inclusive scan of the bin weights
  uint64_t incl = w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    wsum[lane] = v - wsum[lane];  // exclusive per warp
  }
  __syncthreads();
  incl += wsum[warp];
  const uint64_t below = s->below_w, wmax = s->wmax;
  if (w > 0 && below + incl > wmax && below + incl - w <= wmax) cross_bin = t;
  __syncthreads();
  const uint32_t cb = cross_bin;
  if (static_cast<uint32_t>(t) == cb) {
    const int shift = alloc_shift(s);
    const uint64_t lo = s->klo + (static_cast<uint64_t>(cb) << shift);
    const uint64_t w_nom = (1ull << shift) - 1;
    const uint64_t hi_nom = lo + w_nom < lo ? ~0ull : lo + w_nom;  // no wrap near the top of key space
    s->below_w = below + incl - w;
    if (shift == 0) {  // a one-key slice: that key is the crossing flip
      s->status = 1;
      s->cross_key = lo;
    } else {
      s->klo = lo;
      s->khi = hi_nom < s->khi ? hi_nom : s->khi;
      s->collect = c <= kCollectMax ? 1u : 0u;  // few enough flips left: rank them instead of another pass
      s->ncoll = 0;
    }
    s->passes += 1;
  }
  if (t == 0 && cb == 0xffffffffu) s->status = s->passes == 0 ? 2 : 4;  // 4: internal error
}

// Collect stage: every flip with key in [klo, khi] (at most kCollectMax of them) into
// bins[0..) (keys) and bins[kAllocBins..) (weights 2 / 4).
__device__ void alloc_collect(const double* __restrict__ level, uint32_t T, AllocState* s, uint64_t* bins) {
  const uint64_t klo = s->klo, span = s->khi - s->klo;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const double l = level[j];
    if (l != l) continue;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint64_t k = dkey(__dsub_rn(t ? 8.0 : 4.0, l));
      if (k - klo <= span) {
        const uint32_t at = atomicAdd(&s->ncoll, 1u);
        if (at < kCollectMax) {
          bins[at] = k;
          bins[kAllocBins + at] = t ? 4u : 2u;
        }
      }
    }
  }
}

// Finish on one CTA: each collected flip's cumulative weight below and through its key
// (rank counting over at most kCollectMax flips) gives the crossing key exactly as
// further histogram passes would: below + w(< key) <= wmax < below + w(<= key).
__device__ void alloc_finish(AllocState* s, uint64_t* bins, HistSmem& hs) {
  unsigned long long* key = hs.bmn;
  uint32_t* w = hs.bw;
  __shared__ unsigned int winner;
  const int t = threadIdx.x;
  const uint32_t n = s->ncoll;
  if (n > kCollectMax) {  // cannot happen (the scan counted them); fail loudly
    if (t == 0) s->status = 4;
    return;
  }
  if (t == 0) winner = 0xffffffffu;
  if (static_cast<uint32_t>(t) < n) {
    key[t] = bins[t];
    w[t] = static_cast<uint32_t>(bins[kAllocBins + t]);
  }
  __syncthreads();
  const uint64_t below = s->below_w, wmax = s->wmax;
  uint64_t lt = 0, le = 0;
  if (static_cast<uint32_t>(t) < n) {
    const unsigned long long k = key[t];
    for (uint32_t i = 0; i < n; ++i) {
      const unsigned long long ki = key[i];
      lt += ki < k ? w[i] : 0u;
      le += ki <= k ? w[i] : 0u;
    }
    if (below + lt <= wmax && below + le > wmax) atomicMin(&winner, static_cast<unsigned int>(t));
  }
  __syncthreads();
  if (static_cast<uint32_t>(t) == winner) {
    s->cross_key = key[t];
    s->below_w = below + lt;
    s->status = 1;
    s->passes += 1;
  }
  __syncthreads();
  if (t == 0 && s->status == 0) s->status = 4;
}

// The crossing flip's predecessor: the largest flip key below it (0 = none; no key is 0).
__device__ void alloc_pred(const double* __restrict__ level, uint32_t T, AllocState* s) {
  const uint64_t ck = s->cross_key;
  unsigned long long mx = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const double l = level[j];
    if (l != l) continue;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint64_t k = dkey(__dsub_rn(t ? 8.0 : 4.0, l));
      if (k < ck && k > mx) mx = k;
    }
  }
  mx = block_reduce<kRedMax>(mx);
  if (threadIdx.x == 0 && mx) atomicMax(reinterpret_cast<unsigned long long*>(&s->pred_key), mx);
}

// Find an F_j behind each flip key the host needs (crossing, predecessor, largest).
// ---- neighbourhood of the chosen plateau (exactness against the reference's
// float-threshold bisection, allocation.cpp:238-251): the crossing flip found in
// exact arithmetic names sample L; the reference evaluates payload(u) with float
// thresholds, which can differ from the exact count when a flip sits within float
// rounding of a threshold.  The candidates L-1, L, L+1 are evaluated the way the
// reference does and the choice is made like its bisection (largest in budget).
__device__ void alloc_slots_init(AllocState* s) {
  for (int i = 0; i < 4; ++i) s->slot[i] = FlipRec{0, 0, 0, 0, 0};
  s->slot[0].key = 0;      // max-below accumulator
  s->slot[3].key = ~0ull;  // min-above accumulator
  if (s->status == 1) {
    s->slot[2].key = s->cross_key;
    s->slot[2].present = 1;
    if (s->has_pred) {
      s->slot[1].key = s->pred_key;
      s->slot[1].present = 1;
    }
  } else if (s->status == 2) {
    s->slot[1].key = s->kmax;
    s->slot[1].present = 1;
  }
}

__device__ void alloc_neighbors(const double* __restrict__ level, uint32_t T, AllocState* s) {
  const bool want_below = s->slot[1].present != 0, want_above = s->status == 1;
  const uint64_t below = s->slot[1].key, above = s->slot[2].key;
  unsigned long long mx = 0, mn = ~0ull;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const double l = level[j];
    if (l != l) continue;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint64_t k = dkey(__dsub_rn(t ? 8.0 : 4.0, l));
      if (want_below && k < below && k > mx) mx = k;
      if (want_above && k > above && k < mn) mn = k;
    }
  }
  mx = block_reduce<kRedMax>(mx);
  mn = block_reduce<kRedMin>(mn);
  if (threadIdx.x == 0) {
    if (mx) atomicMax(reinterpret_cast<unsigned long long*>(&s->slot[0].key), mx);
    if (mn != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(&s->slot[3].key), mn);
  }
}

__device__ void alloc_identify(const double* __restrict__ level, const float* __restrict__ F, uint32_t T,
                               AllocState* s) {
  uint64_t keys[4];
  bool on[4];
  for (int i = 0; i < 4; ++i) {
    keys[i] = s->slot[i].key;
    on[i] = s->slot[i].present != 0;
  }
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const double l = level[j];
    if (l != l) continue;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint64_t k = dkey(__dsub_rn(t ? 8.0 : 4.0, l));
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (on[i] && k == keys[i]) {
          atomicExch(&s->slot[i].fbits, __float_as_uint(F[j]));
          atomicExch(&s->slot[i].type, static_cast<uint32_t>(t));
        }
    }
  }
}

// candidate samples L-1, L, L+1 (fast_sample_points, allocation.cpp:201-224) with
// device-libm values; the host re-derives them with glibc and compares.
__device__ void alloc_candidates(AllocState* s, double alpha) {
  auto flip = [&](int i) {
    return __dsub_rn(s->slot[i].type ? 8.0 : 4.0,
                     __dmul_rn(alpha, log2(static_cast<double>(__uint_as_float(s->slot[i].fbits)))));
  };
  auto mid = [](double a, double b) { return __dmul_rn(0.5, __dadd_rn(a, b)); };
  for (int c = 0; c < 3; ++c) {
    s->cand_present[c] = 0;
    s->cand_u[c] = 0.0;
  }
  if (s->status == 3) {
    s->cand_present[1] = 1;
    s->cand_u[1] = 0.0;
  } else if (s->status == 2) {
    const double f1 = flip(1);
    s->cand_present[1] = 1;
    s->cand_u[1] = __dadd_rn(f1, 1.0);
    s->cand_present[0] = 1;
    s->cand_u[0] = s->slot[0].present ? mid(flip(0), f1) : __dsub_rn(f1, 1.0);
  } else if (s->status == 1) {
    const double f2 = flip(2);
    s->cand_present[1] = 1;
    s->cand_u[1] = s->slot[1].present ? mid(flip(1), f2) : __dsub_rn(f2, 1.0);
    if (s->slot[1].present) {
      const double f1 = flip(1);
      s->cand_present[0] = 1;
      s->cand_u[0] = s->slot[0].present ? mid(flip(0), f1) : __dsub_rn(f1, 1.0);
    }
    s->cand_present[2] = 1;
    s->cand_u[2] = s->slot[3].present ? mid(f2, flip(3)) : __dadd_rn(f2, 1.0);
  }
  // certification: float(d) is the same float for every d' with |d' - d| <= 2^-40 |d|,
  // while glibc's double (log2 and exp2 within ~0.5 ulp, CUDA's within 1-2 ulp, five
  // rounded double operations between them on |log2 F| <= 150) differs from the device
  // double by far less than 2^-43 relative
  // stable: float(d) is certain; otherwise the two possible floats lo < hi are adjacent and
  // the widths (F_j >= t) differ between them only for F_j == lo: certified unless some F_j
  // equals lo (counted by alloc_count, checked by alloc_decide)
  auto stable = [](double d, float* amb) {
    const float lo = __double2float_rn(__dmul_rd(d, 1.0 - 0x1p-40)), hi = __double2float_rn(__dmul_ru(d, 1.0 + 0x1p-40));
    if (__float_as_uint(lo) == __float_as_uint(hi)) {
      *amb = -1.0f;
      return true;
    }
    *amb = lo;
    return nextafterf(lo, INFINITY) == hi && lo > 0.0f;  // else (overflow / underflow edges): uncertified
  };
  uint32_t cert = 1;
  s->namb = 0;
  for (int c = 0; c < 3; ++c) {
    double u = s->cand_u[c];
    u = u < -1e6 ? -1e6 : (u > 1e6 ? 1e6 : u);
    s->cand_u[c] = u;
    const double d24 = exp2(__ddiv_rn(__dsub_rn(4.0, u), alpha)), d48 = exp2(__ddiv_rn(__dsub_rn(8.0, u), alpha));
    s->cand_t24[c] = static_cast<float>(d24);
    s->cand_t48[c] = static_cast<float>(d48);
    const bool st24 = stable(d24, &s->amb[c][0]), st48 = stable(d48, &s->amb[c][1]);
    if (s->cand_present[c]) cert &= (st24 || s->amb[c][0] > 0.0f) && (st48 || s->amb[c][1] > 0.0f) ? 1u : 0u;
    else s->amb[c][0] = s->amb[c][1] = -1.0f;
    s->cand_n8[c] = 0;
    s->cand_n48[c] = 0;
  }
  s->certified = cert;
  s->consulted = 0;
}

// Ambiguous thresholds with an F_j equal to the lower float: ask the host service thread
// for the candidates' glibc u and thresholds (microseconds on the host, instead of handing
// it the whole allocation), then recount.  Block 0 only; the caller grid-syncs.
__device__ void alloc_consult(AllocState* s, HostMsg* m) {
  const uint32_t* src = reinterpret_cast<const uint32_t*>(s);
  uint32_t* dst = reinterpret_cast<uint32_t*>(&m->state);
  for (uint32_t k = threadIdx.x; k < sizeof(AllocState) / 4; k += blockDim.x) dst[k] = src[k];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t tag = s->epoch + 1;
    m->thr_request = tag;
    __threadfence_system();
    const uint64_t t0 = dq_globaltimer();
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(&m->thr_resolved) : "memory");
      if (v == tag) break;
      __nanosleep(500);
      if (dq_globaltimer() - t0 > g_spin_ns) __trap();
    }
    for (int c = 0; c < 3; ++c) {
      if (s->cand_present[c]) {
        s->cand_u[c] = *reinterpret_cast<volatile double*>(&m->thr_u[c]);
        s->cand_t24[c] = *reinterpret_cast<volatile float*>(&m->thr_t24[c]);
        s->cand_t48[c] = *reinterpret_cast<volatile float*>(&m->thr_t48[c]);
      }
      s->amb[c][0] = s->amb[c][1] = -1.0f;
      s->cand_n8[c] = 0;
      s->cand_n48[c] = 0;
    }
    s->consulted = 1;
  }
}

__device__ void alloc_count(const float* __restrict__ F, uint32_t T, AllocState* s) {
  float t24[3], t48[3], amb[6];
  bool any_amb = false;
  for (int c = 0; c < 3; ++c) {
    t24[c] = s->cand_t24[c];
    t48[c] = s->cand_t48[c];
    amb[2 * c] = s->amb[c][0];
    amb[2 * c + 1] = s->amb[c][1];
    any_amb |= amb[2 * c] > 0.0f || amb[2 * c + 1] > 0.0f;
  }
  unsigned long long n8[3] = {0, 0, 0}, n48[3] = {0, 0, 0}, namb = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const float f = F[j];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      n8[c] += f >= t48[c];
      n48[c] += f >= t24[c];
    }
    if (any_amb) {
#pragma unroll
      for (int k = 0; k < 6; ++k) namb += f == amb[k];
    }
  }
  if (__syncthreads_or(any_amb)) {
    namb = block_reduce<kRedAdd>(namb);
    if (threadIdx.x == 0 && namb) atomicAdd(&s->namb, namb);
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    n8[c] = block_reduce<kRedAdd>(n8[c]);
    n48[c] = block_reduce<kRedAdd>(n48[c]);
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) {
      atomicAdd(&s->cand_n8[c], n8[c]);
      atomicAdd(&s->cand_n48[c], n48[c]);
    }
}

__device__ int g_force_host_alloc;  // test hook (set_force_host_alloc): 1 finish on the host, 2 consult

// the reference's choice: the largest sample whose float-threshold payload fits
__device__ void alloc_decide(AllocState* s, double budget, uint32_t S, uint32_t T) {
  auto ok = [&](int c) {
    const unsigned long long pay =
        static_cast<unsigned long long>(S) * (2ull * T + 2ull * s->cand_n48[c] + 4ull * s->cand_n8[c]);
    return s->cand_present[c] && static_cast<double>(pay) <= budget;
  };
  int ch;
  if (ok(1)) ch = (s->cand_present[2] && ok(2)) ? -1 : 1;
  else if (s->cand_present[0]) ch = ok(0) ? 0 : -1;
  else ch = -2;
  s->choice = ch;
  const int c = ch >= 0 ? ch : 1;
  s->u = s->cand_u[c];
  s->t24 = s->cand_t24[c];
  s->t48 = s->cand_t48[c];
  if (s->namb && !s->consulted) s->certified = 0;
  s->need_host = (!s->certified || ch < 0 || g_force_host_alloc == 1) ? 1u : 0u;
}

// The whole search in one cooperative launch: prep -> up to kAllocMaxPasses x
// (histogram on every CTA, scan on CTA 0) -> neighbourhood -> identify -> candidate
// counts -> decision, with grid-wide syncs in between (every CTA reads the same
// state after each sync, so the early exit is uniform).
__global__ void __launch_bounds__(kAllocBins) k_alloc_coop(const float* __restrict__ F, uint32_t T, double alpha,
                                                           uint64_t wmax, double budget, uint32_t S, AllocWork w) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ HistSmem hs;
  AllocState* st = w.state;
  if (blockIdx.x == 0) alloc_init(st, w.bins, wmax);
  grid.sync();
  alloc_prep(F, T, alpha, w.level, st);
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) alloc_start(st);
  grid.sync();
  for (int p = 0; p < kAllocMaxPasses; ++p) {
    if (st->status != 0) break;
    if (st->collect) {
      alloc_collect(w.level, T, st, w.bins);
      grid.sync();
      if (blockIdx.x == 0) alloc_finish(st, w.bins, hs);
      grid.sync();
      break;
    }
    alloc_hist(w.level, T, st, w.bins, hs);
    grid.sync();
    if (blockIdx.x == 0) alloc_scan(st, w.bins);
    grid.sync();
  }
  if (st->status == 1) {
    alloc_pred(w.level, T, st);
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->has_pred = st->status == 1 && st->pred_key != 0;
    alloc_slots_init(st);
  }
  grid.sync();
  alloc_neighbors(w.level, T, st);
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->slot[0].present = st->slot[1].present && st->slot[0].key != 0;
    st->slot[3].present = st->status == 1 && st->slot[3].key != ~0ull;
  }
  grid.sync();
  alloc_identify(w.level, F, T, st);
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) alloc_candidates(st, alpha);
  grid.sync();
  alloc_count(F, T, st);
  grid.sync();
  if (w.hmsg && (st->namb || g_force_host_alloc == 2) && st->certified) {  // uniform: namb is not written again this round
    if (blockIdx.x == 0) alloc_consult(st, w.hmsg);
    grid.sync();
    alloc_count(F, T, st);
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    alloc_decide(st, budget, S, T);
    st->T = T;
    st->S = S;
    st->budget = budget;
    st->alpha = alpha;
    st->epoch += 1;  // per-round tag of the host mailbox (device-side: graph replays advance it too)
  }
  if (!w.hmsg) return;  // synchronous round: the host reads the state after a stream sync
  grid.sync();
  // asynchronous round: export F for the host on need_host rounds, then mirror the state
  if (st->need_host)
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) w.hF[j] = F[j];
  grid.sync();
  if (blockIdx.x == 0) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(st);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&w.hmsg->state);
    for (uint32_t k = threadIdx.x; k < sizeof(AllocState) / 4; k += blockDim.x) dst[k] = src[k];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && st->need_host) {  // wake the host service thread (state and F are visible)
      __threadfence_system();
      w.hmsg->request = st->epoch;
      __threadfence_system();
    }
  }
}

void set_force_host_alloc(int on) { cudaMemcpyToSymbol(g_force_host_alloc, &on, sizeof on); }

constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;
__device__ __forceinline__ double key_double(uint64_t k) {  // inverse of dkey
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}
// float(d) certain: -1 (never equals an F_j >= 0); two adjacent candidates lo < hi: lo (the
// probe stays certified if no F_j equals it, see alloc_candidates); else NaN (uncertified)
__device__ __forceinline__ float ambiguous_float(double d) {
  const float lo = __double2float_rn(__dmul_rd(d, 1.0 - 0x1p-40)), hi = __double2float_rn(__dmul_ru(d, 1.0 + 0x1p-40));
  if (__float_as_uint(lo) == __float_as_uint(hi)) return -1.0f;
  return nextafterf(lo, INFINITY) == hi && lo > 0.0f ? lo : __int_as_float(0x7fc00000);
}

// Shared memory of the one-CTA allocation (N = kSmallThreads * IPT >= T super-groups):
//   Fs[N]   F in original order (the assignment reads it here)
//   SF[N]   the positive F sorted descending (the probes count F_j >= t by binary search)
//   L[N]    alpha log2 F of the super-groups sorted by F descending (flip order), J[N] their index
//   UK[2N]  the merged flips as order-preserving keys, then the unique flips; UV[2N] = j | type << 31
// The CUB sort's temporary storage aliases UK (written only after the sort; the region is
// widened when the sort needs more).
template <int IPT>
struct SmallSmem {
  static constexpr int N = kSmallThreads * IPT;
  using Sort = cub::BlockRadixSort<uint32_t, kSmallThreads, IPT, uint32_t>;
  static constexpr size_t kSortB = sizeof(typename Sort::TempStorage);
  // L / J are padded one slot per 8 (pd8) and the merged flips one slot per 16 (pd16), so the
  // per-thread runs of the merge (stride 8-16 elements across a warp) spread over the banks
  static constexpr size_t NP8 = N + N / 8 + 1, MP16 = 2 * N + (2 * N) / 16 + 1;
  static constexpr size_t kF = 0, kSF = kF + 4ull * N, kL = kSF + 4ull * N, kJ = kL + 8ull * NP8;
  static constexpr size_t kUK = (kJ + 4ull * NP8 + 15) / 16 * 16;
  static constexpr size_t kUV = kUK + ((8ull * MP16 > kSortB ? 8ull * MP16 : kSortB) + 15) / 16 * 16;
  static constexpr size_t bytes = kUV + 4ull * MP16;
};

// #{F_j >= t} from the positive F sorted descending (SF[0, np)) and the count of F_j >= 0
// (a 32-ary warp search measured no faster: the probes are bound by their fp64 math)
__device__ __forceinline__ uint32_t small_count_ge(const float* SF, uint32_t np, uint32_t nonneg, float t) {
  if (!(t > 0.0f)) return nonneg;  // t = 0: every F_j >= 0 (t is never negative or NaN)
  uint32_t lo = 0, hi = np;        // first p with SF[p] < t
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (SF[mid] < t) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}
// Probe of the bisection (allocation.cpp:237: payload with the float thresholds of sample u
// <= budget): bit 0 fits, bit 1 certified (thresholds stable, or ambiguous with no F_j
// equal to the lower float).  payload = S (2 T + 2 #{F >= t24} + 4 #{F >= t48}), t48 >= t24.
__device__ __forceinline__ uint32_t small_probe(double u, const float* SF, uint32_t np, uint32_t nonneg, uint32_t T,
                                                double alpha, double budget, uint32_t S) {
  const double d24 = exp2(__ddiv_rn(__dsub_rn(4.0, u), alpha)), d48 = exp2(__ddiv_rn(__dsub_rn(8.0, u), alpha));
  const float t24 = static_cast<float>(d24), t48 = static_cast<float>(d48);
  const float a24 = ambiguous_float(d24), a48 = ambiguous_float(d48);
  const unsigned long long units = 2ull * T + 2ull * small_count_ge(SF, np, nonneg, t24) +
                                   4ull * small_count_ge(SF, np, nonneg, t48);
  // some F_j == a (a > 0): the first p with SF[p] < a is past an element equal to a
  auto hit = [&](float a) {
    if (!(a > 0.0f)) return false;
    const uint32_t c = small_count_ge(SF, np, nonneg, a);
    return c > 0 && SF[c - 1] == a;
  };
  const bool cert = !(a24 != a24) && !(a48 != a48) && !hit(a24) && !hit(a48);
  const bool fits = static_cast<double>(units * S) <= budget;
  return (fits ? 1u : 0u) | (cert ? 2u : 0u);
}

// ---------------------------------------------- small T: search + assignment in one block
// The latency path of small all-reduces (T <= 4096 super-groups, d <= 1M entries): the
// reference's allocate_fast (allocation.cpp:195-260) restated literally in one CTA.
// * Flip order without a 64-bit sort: both flip families 4 - a log2 F_j and 8 - a log2 F_j
//   are decreasing in F_j, so one stable radix sort of the T float bit patterns (CUB,
//   descending F) orders both; a merge-path merge of the two families (ties broken by
//   super-group then family, the stable order of the flat sort) gives the sorted flips,
//   de-duplicated like std::unique on the doubles.
// * The bisection (allocation.cpp:237-255) evaluated 3-4 levels at a time: every warp
//   evaluates one node of the next levels of the bisection tree from the current (lo, hi)
//   (speculative probes, one warp each, F staged in shared memory), then thread 0 follows
//   the path the sequential bisection takes - same probes, same result, and the
//   certification counts only the probes on that path.
// * widths, the stable 8/4/2 partition and the permuted means, as build_permutation.
// One launch instead of the cooperative search's passes and grid syncs plus three
// assignment kernels.  Uncertified probes hand the round to the host (need_host).
template <int IPT>
__global__ void __launch_bounds__(kSmallThreads) k_alloc_small(const float* __restrict__ F, uint32_t T, double alpha,
                                                               double budget, uint32_t S, AllocWork w,
                                                               uint8_t* widths, uint32_t* perm) {
  using SM = SmallSmem<IPT>;
  constexpr int N = SM::N;
  extern __shared__ __align__(16) uint8_t smem[];
  float* Fs = reinterpret_cast<float*>(smem + SM::kF);
  float* SF = reinterpret_cast<float*>(smem + SM::kSF);
  double* L = reinterpret_cast<double*>(smem + SM::kL);
  uint32_t* J = reinterpret_cast<uint32_t*>(smem + SM::kJ);
  uint64_t* UK = reinterpret_cast<uint64_t*>(smem + SM::kUK);
  uint32_t* UV = reinterpret_cast<uint32_t*>(smem + SM::kUV);
  auto& sort_tmp = *reinterpret_cast<typename SM::Sort::TempStorage*>(smem + SM::kUK);
  __shared__ unsigned long long red[kSmallWarps];
  __shared__ uint32_t node_res[kSmallWarps];
  __shared__ uint32_t m_sh, npos_sh, nonneg_sh;
  __shared__ int ok_sh, lo_sh, hi_sh, cert_sh, feas_sh, done_sh;
  AllocState* st = w.state;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  pdl_wait();
  pdl_trigger();
#if defined(DQ_SMALL_PHASES)
  uint64_t ph[10];
  int nph = 0;
#define DQ_PHASE() do { __syncthreads(); if (t == 0) ph[nph++] = dq_globaltimer(); } while (0)
#else
#define DQ_PHASE() do { } while (0)
#endif
  DQ_PHASE();
  // the statistics reduction folded in (small rounds): wait for every rank's rows (peer
  // exchange), then F_j = the rank-ordered fp64 sum exactly as k_reduce_stats[_peer]
  const StatsReduce& rd = w.red;
  if (rd.mean) {
    if (rd.flags && t == 0) {
      const uint32_t epoch = *rd.epoch_ptr;
      for (uint32_t r = 0; r < rd.n; ++r) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(rd.flags + r) : "memory");
        if (v == epoch) continue;
        const uint64_t t0 = dq_globaltimer();
        for (;;) {
          __nanosleep(64);
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(rd.flags + r) : "memory");
          if (v == epoch) break;
          if (dq_globaltimer() - t0 > g_spin_ns) __trap();
        }
      }
    }
    __syncthreads();
  }
  // stage F; sort keys ~bits (ascending = F descending) of the positive F_j, stable in j
  uint32_t key[IPT], val[IPT];
  uint32_t npos = 0, nonneg = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint32_t j = static_cast<uint32_t>(t * IPT + i);
    float f = -1.0f;
    if (j < T) {
      if (rd.mean) {
        double a = 0.0, b = 0.0;
        for (uint32_t r = 0; r < rd.n; ++r) {
          a = __dadd_rn(a, static_cast<double>(__ldcg(rd.mean + static_cast<uint64_t>(r) * rd.stride + j)));
          b = __dadd_rn(b, static_cast<double>(__ldcg(rd.sq + static_cast<uint64_t>(r) * rd.stride + j)));
        }
        rd.gm[j] = static_cast<float>(__ddiv_rn(a, static_cast<double>(rd.n)));
        f = static_cast<float>(b);
        rd.gs[j] = f;
      } else {
        f = F[j];
      }
    }
    if (j < T) Fs[j] = f;
    const bool pos = f > 0.0f;
    key[i] = pos ? ~__float_as_uint(f) : 0xffffffffu;
    val[i] = j;
    npos += pos;
    nonneg += f >= 0.0f;
  }
  {
    unsigned long long c = static_cast<unsigned long long>(npos) | static_cast<unsigned long long>(nonneg) << 32;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) red[warp] = c;
  }
  __syncthreads();
  if (t == 0) {
    unsigned long long c = 0;
    for (int k = 0; k < kSmallWarps; ++k) c += red[k];
    npos_sh = static_cast<uint32_t>(c);
    nonneg_sh = static_cast<uint32_t>(c >> 32);
  }
  DQ_PHASE();
  typename SM::Sort(sort_tmp).SortBlockedToStriped(key, val);  // item i of thread t: position t + 512 i
  __syncthreads();
  DQ_PHASE();
  const uint32_t np = npos_sh, nonneg_all = nonneg_sh;  // sorted positions [0, np): the positive F_j
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const uint32_t p = static_cast<uint32_t>(t + kSmallThreads * i);
    if (p < np) {
      const float f = __uint_as_float(~key[i]);
      SF[p] = f;
      L[p + (p >> 3)] = __dmul_rn(alpha, log2(static_cast<double>(f)));
      J[p + (p >> 3)] = val[i];
    }
  }
  __syncthreads();
  DQ_PHASE();
  // merge A_p = 4 - L[p] (family 0) and B_q = 8 - L[q] (family 1), both ascending in p:
  // thread t produces outputs [t per, (t + 1) per) - one merge-path binary search for its
  // start, then a sequential two-pointer merge (the rank-per-element variant cost 13
  // dependent shared loads per flip: 18.8 vs 4.3 us at T = 4096)
  const uint32_t M = 2 * np;
  auto pd8 = [](uint32_t p) { return p + (p >> 3); };
  auto pd16 = [](uint32_t r) { return r + (r >> 4); };
  auto a_val = [&](uint32_t p) { return __dsub_rn(4.0, L[pd8(p)]); };
  auto b_val = [&](uint32_t q) { return __dsub_rn(8.0, L[pd8(q)]); };
  // A_p before B_q in the flat stable order (value, then super-group, family 0 first)
  auto a_first = [&](uint32_t p, uint32_t q) {
    const double x = a_val(p), y = b_val(q);
    return x < y || (x == y && J[pd8(p)] <= J[pd8(q)]);
  };
  {
    const uint32_t per = (M + kSmallThreads - 1) / kSmallThreads;
    const uint32_t r0 = min(static_cast<uint32_t>(t) * per, M), r1 = min(r0 + per, M);
    uint32_t lo = r0 > np ? r0 - np : 0, hi = min(r0, np);
    while (lo < hi) {  // a = number of A elements among the first r0 merged
      const uint32_t mid = (lo + hi) >> 1;
      if (a_first(mid, r0 - 1 - mid)) lo = mid + 1;
      else hi = mid;
    }
    uint32_t ia = lo, ib = r0 - lo;
    double va = ia < np ? a_val(ia) : 0.0, vb = ib < np ? b_val(ib) : 0.0;
    uint32_t ja = ia < np ? J[pd8(ia)] : 0, jb = ib < np ? J[pd8(ib)] : 0;
    for (uint32_t r = r0; r < r1; ++r) {
      const bool take_a = ib >= np || (ia < np && (va < vb || (va == vb && ja <= jb)));
      if (take_a) {
        UK[pd16(r)] = dkey(va);
        UV[pd16(r)] = ja;
        if (++ia < np) {
          va = a_val(ia);
          ja = J[pd8(ia)];
        }
      } else {
        UK[pd16(r)] = dkey(vb);
        UV[pd16(r)] = jb | 0x80000000u;
        if (++ib < np) {
          vb = b_val(ib);
          jb = J[pd8(ib)];
        }
      }
    }
  }
  __syncthreads();
  DQ_PHASE();
  // std::unique on the merged flips (padded positions), compacted in place into UK[0, m):
  // warp w owns a segment of `seg` positions, lane l its positions seg w + 32 k + l (held in
  // registers across the barrier)
  {
    constexpr int K = 2 * IPT;  // seg / 32 <= 2 N / (16 * 32)
    const uint32_t seg = ((M + kSmallWarps - 1) / kSmallWarps + 31) / 32 * 32;
    const uint32_t s0 = warp * seg;
    uint64_t k_[K];
    uint32_t v_[K], keep[K];
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const uint32_t r = s0 + 32u * i + lane;
      const bool in = r < M && 32u * i < seg;
      k_[i] = in ? UK[pd16(r)] : 0;
      v_[i] = in ? UV[pd16(r)] : 0;
      const bool kp = in && (r == 0 || k_[i] != UK[pd16(r - 1)]);
      keep[i] = __ballot_sync(0xffffffffu, kp);
      cnt += __popc(keep[i]);
    }
    if (lane == 0) red[warp] = cnt;
    __syncthreads();  // every segment is in registers before the compaction overwrites UK
    uint32_t off = 0, all = 0;
    for (int k = 0; k < kSmallWarps; ++k) {
      if (k < warp) off += static_cast<uint32_t>(red[k]);
      all += static_cast<uint32_t>(red[k]);
    }
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (keep[i] & (1u << lane)) {
        const uint32_t pos = off + __popc(keep[i] & lt);
        UK[pos] = k_[i];
        UV[pos] = v_[i];
      }
      off += __popc(keep[i]);
    }
    if (t == 0) m_sh = all;
  }
  __syncthreads();
  DQ_PHASE();
  const uint32_t m = m_sh;
  const uint32_t ns = m ? m + 1 : 1;  // samples (fast_sample_points)
  auto sample = [&](uint32_t i) {
    double u;
    if (m == 0) u = 0.0;
    else if (i == 0) u = __dsub_rn(key_double(UK[0]), 1.0);
    else if (i == m) u = __dadd_rn(key_double(UK[m - 1]), 1.0);
    else u = __dmul_rn(0.5, __dadd_rn(key_double(UK[i - 1]), key_double(UK[i])));
    return u < -1e6 ? -1e6 : (u > 1e6 ? 1e6 : u);
  };
  // Bisection tree node k (breadth-first, k = 0 the next probe) below the interval
  // (lo, hi): descend by the bits of k + 1 (1 = the probe fitted: lo = mid).  Returns the
  // node's probe index, or -1 where the sequential loop would already have stopped.
  auto node_mid = [](int lo, int hi, int k) {
    int level = 31 - __clz(k + 1);
    for (int l = level - 1; l >= 0; --l) {
      if (lo + 1 >= hi) return -1;
      const int mid = (lo + hi) / 2;
      if (((k + 1) >> l) & 1) lo = mid;
      else hi = mid;
    }
    return lo + 1 >= hi ? -1 : (lo + hi) / 2;
  };
  // round 0: fits(0), fits(ns - 1) and the first 3 tree levels below (0, ns - 1)
  {
    int probe = -1;
    if (warp == 0) probe = 0;
    else if (warp == 1) probe = ns > 1 ? static_cast<int>(ns - 1) : -1;
    else if (warp < 9) probe = node_mid(0, static_cast<int>(ns - 1), warp - 2);
    if (probe >= 0) {
      if (lane == 0)
        node_res[warp] = small_probe(sample(static_cast<uint32_t>(probe)), SF, np, nonneg_all, T, alpha, budget, S) | 4u;
    } else if (lane == 0) {
      node_res[warp] = 0;
    }
  }
  __syncthreads();
  if (t == 0) {
    int lo = 0, hi = static_cast<int>(ns - 1), cert = 1, done = 0;
    const uint32_t r0 = node_res[0];
    cert &= (r0 >> 1) & 1;
    const int feasible = r0 & 1;
    if (!feasible) {
      done = 1;
    } else if (ns == 1) {
      done = 1;  // the single sample fits (lo = 0)
    } else {
      const uint32_t r1 = node_res[1];
      cert &= (r1 >> 1) & 1;
      if (r1 & 1) {
        lo = hi;
        done = 1;
      } else {
        int k = 0;
        for (int l = 0; l < 3; ++l) {
          if (lo + 1 >= hi) break;
          const uint32_t r = node_res[2 + k];
          cert &= (r >> 1) & 1;
          const int mid = (lo + hi) / 2;
          if (r & 1) lo = mid;
          else hi = mid;
          k = 2 * k + 1 + static_cast<int>(r & 1);
        }
        done = lo + 1 >= hi;
      }
    }
    lo_sh = lo;
    hi_sh = hi;
    cert_sh = cert;
    feas_sh = feasible;
    done_sh = done;
  }
  __syncthreads();
  // later rounds: 4 tree levels (15 nodes) per round
  while (!done_sh) {
    const int lo0 = lo_sh, hi0 = hi_sh;
    if (warp < 15) {
      const int probe = node_mid(lo0, hi0, warp);
      if (probe >= 0 && lane == 0)
        node_res[warp] = small_probe(sample(static_cast<uint32_t>(probe)), SF, np, nonneg_all, T, alpha, budget, S) | 4u;
    }
    __syncthreads();
    if (t == 0) {
      int lo = lo0, hi = hi0, cert = cert_sh, k = 0;
      for (int l = 0; l < 4; ++l) {
        if (lo + 1 >= hi) break;
        const uint32_t r = node_res[k];
        cert &= (r >> 1) & 1;
        const int mid = (lo + hi) / 2;
        if (r & 1) lo = mid;
        else hi = mid;
        k = 2 * k + 1 + static_cast<int>(r & 1);
      }
      lo_sh = lo;
      hi_sh = hi;
      cert_sh = cert;
      done_sh = lo + 1 >= hi;
    }
    __syncthreads();
  }
  DQ_PHASE();
  const uint32_t lo = static_cast<uint32_t>(lo_sh);
  const bool feasible = feas_sh != 0;
  // final thresholds (certified) + the state the host reads (u via host_u_of, mailbox)
  if (t == 0) {
    const double u = sample(lo);
    const double d24 = exp2(__ddiv_rn(__dsub_rn(4.0, u), alpha)), d48 = exp2(__ddiv_rn(__dsub_rn(8.0, u), alpha));
    const uint32_t epoch = st->epoch + 1;
    *st = AllocState{};
    st->epoch = epoch;
    auto rec = [&](uint32_t i) {
      FlipRec r{};
      r.key = UK[i];
      r.fbits = __float_as_uint(Fs[UV[i] & 0x7fffffffu]);
      r.type = UV[i] >> 31;
      r.present = 1;
      return r;
    };
    if (m == 0) {
      st->status = 3;
    } else if (lo == m) {
      st->status = 2;
      st->slot[1] = rec(m - 1);
    } else {
      st->status = 1;
      st->slot[2] = rec(lo);
      if (lo > 0) st->slot[1] = rec(lo - 1);
    }
    st->choice = 1;
    st->u = u;
    st->t24 = static_cast<float>(d24);
    st->t48 = static_cast<float>(d48);
    st->certified = cert_sh ? 1u : 0u;  // every probe on the bisection's path certified
    st->need_host = (!st->certified || !feasible || g_force_host_alloc == 1) ? 1u : 0u;
    st->T = T;
    st->S = S;
    st->budget = budget;
    st->alpha = alpha;
    ok_sh = static_cast<int>(st->need_host);
  }
  __syncthreads();
  const bool need_host = ok_sh != 0;
  if (need_host) {  // hand the round to the host: export F, mirror, request, wait for the answer
    for (uint32_t j = t; j < T; j += kSmallThreads) w.hF[j] = Fs[j];
  }
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(st);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&w.hmsg->state);
    for (uint32_t k = t; k < sizeof(AllocState) / 4; k += kSmallThreads) dst[k] = src[k];
  }
  if (need_host) {  // (the common round's mirror is read after the round completes: no fence)
    __threadfence_system();
    __syncthreads();
    if (t == 0) {
      w.hmsg->request = st->epoch;
      __threadfence_system();
      const uint64_t t0 = dq_globaltimer();
      for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(&w.hmsg->resolved) : "memory");
        if (v == st->epoch) break;
        __nanosleep(1000);
        if (dq_globaltimer() - t0 > g_spin_ns) __trap();
      }
      st->t24 = *reinterpret_cast<volatile float*>(&w.hmsg->t24);
      st->t48 = *reinterpret_cast<volatile float*>(&w.hmsg->t48);
    }
  }
  __syncthreads();
  DQ_PHASE();
  const float t24 = st->t24, t48 = st->t48;
  // widths + stable partition 8 | 4 | 2 (build_permutation, allocation.cpp:302-310):
  // super-group j = 512 k + t (position-striped), class ballots per (k, warp), then each
  // element's place = class base + the class count of every (k', warp') before it + its
  // rank in the ballot
  __shared__ uint32_t ccnt[IPT][kSmallWarps];
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t bal[IPT][3];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const uint32_t j = static_cast<uint32_t>(k * kSmallThreads + t);
    int c = 3;
    if (j < T) {
      const float fj = Fs[j];
      c = fj >= t48 ? 0 : (fj >= t24 ? 1 : 2);
      widths[j] = static_cast<uint8_t>(c == 0 ? 8 : (c == 1 ? 4 : 2));
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) bal[k][q] = __ballot_sync(0xffffffffu, c == q);
    if (lane == 0) ccnt[k][warp] = __popc(bal[k][0]) | __popc(bal[k][1]) << 8 | __popc(bal[k][2]) << 16;
  }
  __syncthreads();
  // exclusive prefix of the (k, warp) class counts in element order, by warp 0 (IPT * 16
  // entries, IPT / 2 per lane), as 16-bit fields (T <= 4096)
  __shared__ unsigned long long cpre[IPT * kSmallWarps + 1];
  if (warp == 0) {
    constexpr int E = IPT * kSmallWarps, PL = (E + 31) / 32;
    const uint32_t* cc = &ccnt[0][0];
    unsigned long long v[PL], sum = 0;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int idx = lane * PL + q;
      const uint32_t e = idx < E ? cc[idx] : 0u;
      v[q] = (e & 0xffu) | static_cast<unsigned long long>((e >> 8) & 0xffu) << 16 |
             static_cast<unsigned long long>((e >> 16) & 0xffu) << 32;
      sum += v[q];
    }
    unsigned long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    unsigned long long run = incl - sum;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int idx = lane * PL + q;
      if (idx < E) cpre[idx] = run;
      run += v[q];
    }
    if (lane == 31) cpre[E] = incl;
  }
  __syncthreads();
  unsigned long long pre[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) pre[k] = cpre[k * kSmallWarps + warp];
  const unsigned long long acc = cpre[IPT * kSmallWarps];
  const uint32_t n8 = static_cast<uint32_t>(acc & 0xffffu), n4 = static_cast<uint32_t>((acc >> 16) & 0xffffu);
  const uint32_t cbase[3] = {0, n8, n8 + n4};
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const uint32_t j = static_cast<uint32_t>(k * kSmallThreads + t);
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (bal[k][q] & (1u << lane)) {
        const uint32_t at = cbase[q] + static_cast<uint32_t>((pre[k] >> (16 * q)) & 0xffffu) + __popc(bal[k][q] & lt);
        perm[at] = j;
        if (w.pmean) w.pmean[at] = w.gmean[j];
      }
  }
  if (t == 0) {
    w.counts[0] = n8;
    w.counts[1] = n4;
    w.counts[2] = T - n8 - n4;
    w.hmsg->counts[0] = n8;
    w.hmsg->counts[1] = n4;
    w.hmsg->counts[2] = T - n8 - n4;
  }
  DQ_PHASE();
#if defined(DQ_SMALL_PHASES)
  if (t == 0)
    printf("k_alloc_small T=%u m=%u phases(ns): stage %llu sort %llu log2 %llu merge %llu unique %llu bisect %llu mirror %llu "
           "assign %llu\n",
           T, m, ph[1] - ph[0], ph[2] - ph[1], ph[3] - ph[2], ph[4] - ph[3], ph[5] - ph[4], ph[6] - ph[5], ph[7] - ph[6],
           ph[8] - ph[7]);
#endif
#undef DQ_PHASE
}

bool launch_alloc_small(const float* F, uint32_t T, double alpha, double budget, uint32_t S, AllocWork w,
                        uint8_t* widths, uint32_t* perm, cudaStream_t st) {
  if (!w.hmsg || T == 0 || T > kSmallAllocMaxT) return false;
  auto go = [&](auto ipt) {
    constexpr int IPT = decltype(ipt)::value;
    constexpr size_t bytes = SmallSmem<IPT>::bytes;
    static bool attr[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev]) {
      cudaFuncSetAttribute(k_alloc_small<IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
      attr[dev] = true;
    }
    launch_pdl(k_alloc_small<IPT>, dim3(1), dim3(kSmallThreads), bytes, st, F, T, alpha, budget, S, w, widths, perm);
  };
  if (T <= kSmallThreads) go(std::integral_constant<int, 1>{});
  else if (T <= kSmallThreads * 2) go(std::integral_constant<int, 2>{});
  else if (T <= kSmallThreads * 4) go(std::integral_constant<int, 4>{});
  else go(std::integral_constant<int, 8>{});
  return true;
}

cudaError_t launch_alloc_search(const float* F, uint32_t T, double alpha, uint64_t wmax, double budget,
                                uint32_t S, AllocWork w, cudaStream_t st) {
  static int cache[kMaxDevices] = {};
  const int max_blocks = per_device(cache, [](int dev) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_alloc_coop, kAllocBins, 0);
    return (sms > 0 ? sms : 148) * (per_sm > 0 ? per_sm : 1);
  });
  const uint32_t want = T ? (T + 4 * kAllocBins - 1) / (4 * kAllocBins) : 1;
  const uint32_t grid = want < static_cast<uint32_t>(max_blocks) ? want : static_cast<uint32_t>(max_blocks);
  void* args[] = {const_cast<float**>(&F), &T, &alpha, &wmax, &budget, &S, &w};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_alloc_coop), dim3(grid), dim3(kAllocBins), args, 0, st);
}

// ---- slow exact path helpers (rare: ambiguous neighbourhood or a libm mismatch)
__global__ void k_flip_neighbor(const double* __restrict__ level, const float* __restrict__ F, uint32_t T,
                                uint64_t key, int dir, FlipRec* rec) {
  __shared__ unsigned long long best;
  if (threadIdx.x == 0) best = dir < 0 ? 0ull : ~0ull;
  __syncthreads();
  unsigned long long b = dir < 0 ? 0ull : ~0ull;
  for (uint32_t j = threadIdx.x; j < T; j += blockDim.x) {
    const double l = level[j];
    if (l != l) continue;
    for (int t = 0; t < 2; ++t) {
      const uint64_t k = dkey(__dsub_rn(t ? 8.0 : 4.0, l));
      if (dir < 0 && k < key && k > b) b = k;
      if (dir > 0 && k > key && k < b) b = k;
    }
  }
  if (dir < 0) atomicMax(&best, b);
  else atomicMin(&best, b);
  __syncthreads();
  const unsigned long long found = best;
  if (threadIdx.x == 0) *rec = FlipRec{found, 0, 0, (dir < 0 ? found != 0ull : found != ~0ull) ? 1u : 0u, 0};
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < T; j += blockDim.x) {
    const double l = level[j];
    if (l != l) continue;
    for (int t = 0; t < 2; ++t)
      if (dkey(__dsub_rn(t ? 8.0 : 4.0, l)) == found) {
        atomicExch(&rec->fbits, __float_as_uint(F[j]));
        atomicExch(&rec->type, static_cast<uint32_t>(t));
      }
  }
}

void launch_flip_neighbor(const double* level, const float* F, uint32_t T, double alpha, uint64_t key, int dir,
                          FlipRec* rec, cudaStream_t st) {
  (void)alpha;
  k_flip_neighbor<<<1, 1024, 0, st>>>(level, F, T, key, dir, rec);
}

__global__ void k_threshold_counts(const float* __restrict__ F, uint32_t T, float t24, float t48,
                                   unsigned long long* counts) {
  unsigned long long n8 = 0, n48 = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    n8 += F[j] >= t48;
    n48 += F[j] >= t24;
  }
  for (int o = 16; o > 0; o >>= 1) {
    n8 += __shfl_xor_sync(0xffffffffu, n8, o);
    n48 += __shfl_xor_sync(0xffffffffu, n48, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(counts, n8);
    atomicAdd(counts + 1, n48);
  }
}

void launch_threshold_counts(const float* F, uint32_t T, float t24, float t48, unsigned long long* counts,
                             cudaStream_t st) {
  cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), st);
  k_threshold_counts<<<296, 512, 0, st>>>(F, T, t24, t48, counts);
}

uint32_t alloc_blocks(uint32_t T) { return (T + 2047) / 2048; }

// ---------------------------------------------------- width assignment
// widths (proj/src/allocation.cpp:186-199) and the stable 8,4,2 partition
// (allocation.cpp:302-310).  Block b owns super-groups [2048 b, 2048 b + 2048),
// thread t the 8 consecutive ones starting at 2048 b + 8 t.
__device__ __forceinline__ int cls_of(float f, float t24, float t48) {
  return f >= t48 ? 0 : (f >= t24 ? 1 : 2);
}

__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* tot) {
  __shared__ uint64_t ws[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  uint64_t off = 0, all = 0;
  for (int k = 0; k < 8; ++k) {
    if (k < warp) off += ws[k];
    all += ws[k];
  }
  __syncthreads();
  *tot = all;
  return off + incl - v;
}

// MODE 0: fast allocator (float thresholds, from params or the search state);
// 1: fixed width; 2: general allocator (level by double compares, allocation.cpp:100-105)
template <int MODE>
__device__ __forceinline__ int class_of(const float* F, uint32_t j, float t24, float t48, int fixed_cls, double g0,
                                        double g1) {
  if constexpr (MODE == 1) return fixed_cls;
  else if constexpr (MODE == 2) {
    const double f = static_cast<double>(F[j]);
    return f >= g1 ? 0 : (f >= g0 ? 1 : 2);
  } else return cls_of(F[j], t24, t48);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_assign_count(const float* __restrict__ F, uint32_t T, float t24,
                                                      float t48, const AllocState* st_thr, int fixed_cls,
                                                      double g0, double g1, uint8_t* widths, uint32_t* blockcnt,
                                                      HostMsg* hmsg) {
  if (st_thr) {
    t24 = st_thr->t24;
    t48 = st_thr->t48;
    if (hmsg && st_thr->need_host) {  // asynchronous round the device could not certify: host answer
      __shared__ float ht[2];
      if (threadIdx.x == 0) {
        const uint32_t ep = st_thr->epoch;
        const uint64_t t0 = dq_globaltimer();
        for (;;) {
          uint32_t v;
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(&hmsg->resolved) : "memory");
          if (v == ep) break;
          __nanosleep(1000);
          if (dq_globaltimer() - t0 > g_spin_ns) __trap();
        }
        ht[0] = *reinterpret_cast<volatile float*>(&hmsg->t24);
        ht[1] = *reinterpret_cast<volatile float*>(&hmsg->t48);
        if (blockIdx.x == 0) {  // for the scatter kernel that follows
          AllocState* w = const_cast<AllocState*>(st_thr);
          w->t24 = ht[0];
          w->t48 = ht[1];
        }
      }
      __syncthreads();
      t24 = ht[0];
      t48 = ht[1];
    }
  }
  const uint32_t j0 = blockIdx.x * 2048 + threadIdx.x * 8;
  uint64_t packed = 0;  // 16-bit counts per class
  for (int k = 0; k < 8; ++k) {
    const uint32_t j = j0 + k;
    if (j >= T) break;
    const int c = class_of<MODE>(F, j, t24, t48, fixed_cls, g0, g1);
    widths[j] = static_cast<uint8_t>(c == 0 ? 8 : (c == 1 ? 4 : 2));
    packed += 1ull << (16 * c);
  }
  uint64_t tot;
  block_excl_scan_u64(packed, &tot);
  if (threadIdx.x == 0) {
    blockcnt[4 * blockIdx.x + 0] = static_cast<uint32_t>(tot & 0xffff);
    blockcnt[4 * blockIdx.x + 1] = static_cast<uint32_t>((tot >> 16) & 0xffff);
    blockcnt[4 * blockIdx.x + 2] = static_cast<uint32_t>((tot >> 32) & 0xffff);
  }
}

// exclusive scan of the per-block class counts (one CTA), totals -> counts[0..2]
__global__ void __launch_bounds__(1024) k_assign_scan(uint32_t nb, uint32_t* blockcnt, uint32_t* counts,
                                                      HostMsg* hmsg) {
  __shared__ uint64_t carry[3];
  if (threadIdx.x < 3) carry[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nb; base += blockDim.x) {
    const uint32_t b = base + threadIdx.x;
    uint64_t v[3];
    for (int c = 0; c < 3; ++c) v[c] = b < nb ? blockcnt[4 * b + c] : 0;
    for (int c = 0; c < 3; ++c) {
      // block-wide exclusive scan (1024 threads = 32 warps)
      __shared__ uint64_t ws[32];
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      uint64_t incl = v[c];
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) ws[warp] = incl;
      __syncthreads();
      uint64_t off = 0, all = 0;
      for (int k = 0; k < 32; ++k) {
        if (k < warp) off += ws[k];
        all += ws[k];
      }
      if (b < nb) blockcnt[4 * b + c] = static_cast<uint32_t>(carry[c] + off + incl - v[c]);
      __syncthreads();
      if (threadIdx.x == 0) carry[c] += all;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    counts[0] = static_cast<uint32_t>(carry[0]);
    counts[1] = static_cast<uint32_t>(carry[1]);
    counts[2] = static_cast<uint32_t>(carry[2]);
    if (hmsg) {  // asynchronous round: the host reads the class counts lazily
      hmsg->counts[0] = counts[0];
      hmsg->counts[1] = counts[1];
      hmsg->counts[2] = counts[2];
      __threadfence_system();
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_assign_scatter(const float* __restrict__ F, uint32_t T, float t24,
                                                        float t48, const AllocState* st_thr, int fixed_cls,
                                                        double g0, double g1,
                                                        const uint32_t* blockcnt, const uint32_t* counts,
                                                        uint32_t* perm, const float* gmean, float* pmean) {
  if (st_thr) {
    t24 = st_thr->t24;
    t48 = st_thr->t48;
  }
  const uint32_t j0 = blockIdx.x * 2048 + threadIdx.x * 8;
  int cls[8];
  uint64_t packed = 0;
  for (int k = 0; k < 8; ++k) {
    const uint32_t j = j0 + k;
    cls[k] = j < T ? class_of<MODE>(F, j, t24, t48, fixed_cls, g0, g1) : 3;
    if (cls[k] < 3) packed += 1ull << (16 * cls[k]);
  }
  uint64_t tot;
  const uint64_t excl = block_excl_scan_u64(packed, &tot);
  uint32_t pos[3];
  const uint32_t base[3] = {0, counts[0], counts[0] + counts[1]};
  for (int c = 0; c < 3; ++c)
    pos[c] = base[c] + blockcnt[4 * blockIdx.x + c] + static_cast<uint32_t>((excl >> (16 * c)) & 0xffff);
  for (int k = 0; k < 8; ++k)
    if (cls[k] < 3) {
      const uint32_t at = pos[cls[k]]++;
      perm[at] = j0 + k;
      if (pmean) pmean[at] = gmean[j0 + k];
    }
}

static void assign_impl(int mode, const float* F, uint32_t T, float t24, float t48, const AllocState* thr,
                        int fixed_cls, double g0, double g1, AllocWork w, uint8_t* widths, uint32_t* perm,
                        cudaStream_t st) {
  const uint32_t nb = alloc_blocks(T);
  if (nb == 0) return;
#define DQ_ASSIGN(M)                                                                                     \
  do {                                                                                                   \
    k_assign_count<M><<<nb, 256, 0, st>>>(F, T, t24, t48, thr, fixed_cls, g0, g1, widths, w.blockcnt,     \
                                          w.hmsg);                                                       \
    k_assign_scan<<<1, 1024, 0, st>>>(nb, w.blockcnt, w.counts, w.hmsg);                                 \
    k_assign_scatter<M><<<nb, 256, 0, st>>>(F, T, t24, t48, thr, fixed_cls, g0, g1, w.blockcnt, w.counts, \
                                            perm, w.gmean, w.pmean);                                     \
  } while (0)
  if (mode == 1) DQ_ASSIGN(1);
  else if (mode == 2) DQ_ASSIGN(2);
  else DQ_ASSIGN(0);
#undef DQ_ASSIGN
}

void launch_alloc_assign(const float* F, uint32_t T, float t24, float t48, bool from_state, AllocWork w,
                         uint8_t* widths, uint32_t* perm, cudaStream_t st) {
  assign_impl(0, F, T, t24, t48, from_state ? w.state : nullptr, 0, 0.0, 0.0, w, widths, perm, st);
}

void launch_fixed_assign(uint32_t T, int width, AllocWork w, uint8_t* widths, uint32_t* perm,
                         cudaStream_t st) {
  assign_impl(1, nullptr, T, 0.f, 0.f, nullptr, width == 8 ? 0 : (width == 4 ? 1 : 2), 0.0, 0.0, w, widths, perm,
              st);
}

void launch_general_assign(const float* F, uint32_t T, double g0, double g1, AllocWork w, uint8_t* widths,
                           uint32_t* perm, cudaStream_t st) {
  assign_impl(2, F, T, 0.f, 0.f, nullptr, 0, g0, g1, w, widths, perm, st);
}

// ----------------------------------------------------- general allocator
// allocate_general for W = {2,4,8} (allocation.cpp:121-168; the round path's W,
// engine.cpp:306-307): crossing points F_j / chain[k] (chain = {1, 512/17}) of
// every F_j > 0 as order-preserving u64 keys (positive doubles), sorted and
// de-duplicated with CUB; the host then bisects over the sorted points exactly
// like the reference, evaluating each probe with k_general_counts.  Non-positive
// F_j emit ~0 keys (dropped after the sort); negative or NaN F_j are counted as
// invalid (allocation.cpp:127-128).
__global__ void k_general_points(const float* __restrict__ F, uint32_t T, double c1, uint64_t* keys,
                                 unsigned long long* invalid) {
  unsigned long long bad = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const float f = F[j];
    bad += !(f >= 0.0f);
    uint64_t k0 = ~0ull, k1 = ~0ull;
    if (f > 0.0f) {
      k0 = static_cast<uint64_t>(__double_as_longlong(__ddiv_rn(static_cast<double>(f), 1.0)));
      k1 = static_cast<uint64_t>(__double_as_longlong(__ddiv_rn(static_cast<double>(f), c1)));
    }
    keys[2ull * j] = k0;
    keys[2ull * j + 1] = k1;
  }
  if (bad) atomicAdd(invalid, bad);
}

// payload terms at the probe points[idx] (the all-min plateau 2 * back + 1 at idx == M)
__global__ void k_general_counts(const float* __restrict__ F, uint32_t T, const uint64_t* __restrict__ pts,
                                 uint32_t M, uint32_t idx, double c1, unsigned long long* counts, double* base_out) {
  double base;
  if (idx < M) base = __longlong_as_double(static_cast<long long>(pts[idx]));
  else base = M ? __dadd_rn(__dmul_rn(__longlong_as_double(static_cast<long long>(pts[M - 1])), 2.0), 1.0) : 1.0;
  const double g1 = __dmul_rn(base, c1);
  if (blockIdx.x == 0 && threadIdx.x == 0) *base_out = base;
  unsigned long long n8 = 0, n48 = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < T; j += gridDim.x * blockDim.x) {
    const double f = static_cast<double>(F[j]);
    n8 += f >= g1;
    n48 += f >= base;  // base * chain[0] == base
  }
  for (int o = 16; o > 0; o >>= 1) {
    n8 += __shfl_xor_sync(0xffffffffu, n8, o);
    n48 += __shfl_xor_sync(0xffffffffu, n48, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(counts, n8);
    atomicAdd(counts + 1, n48);
  }
}

size_t general_temp_bytes(uint32_t T) {
  size_t a = 0, b = 0;
  const int n = static_cast<int>(2 * T);
  cub::DeviceRadixSort::SortKeys(nullptr, a, static_cast<const uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr), n);
  cub::DeviceSelect::Unique(nullptr, b, static_cast<const uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                            static_cast<int*>(nullptr), n);
  return a > b ? a : b;
}

cudaError_t launch_general_points(const float* F, uint32_t T, double c1, uint64_t* keys, uint64_t* sorted,
                                  void* temp, size_t temp_bytes, int* n_unique, unsigned long long* invalid,
                                  cudaStream_t st) {
  cudaMemsetAsync(invalid, 0, sizeof(*invalid), st);
  if (T == 0) return cudaMemsetAsync(n_unique, 0, sizeof(int), st);
  k_general_points<<<(T + 255) / 256 < 148u * 8 ? (T + 255) / 256 : 148u * 8, 256, 0, st>>>(F, T, c1, keys, invalid);
  const int n = static_cast<int>(2 * T);
  size_t tb = temp_bytes;
  cudaError_t e = cub::DeviceRadixSort::SortKeys(temp, tb, keys, sorted, n, 0, 64, st);
  if (e != cudaSuccess) return e;
  tb = temp_bytes;
  return cub::DeviceSelect::Unique(temp, tb, sorted, keys, n_unique, n, st);  // unique points back into keys
}

void launch_general_counts(const float* F, uint32_t T, const uint64_t* pts, uint32_t M, uint32_t idx, double c1,
                           unsigned long long* counts, double* base_out, cudaStream_t st) {
  cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), st);
  k_general_counts<<<296, 512, 0, st>>>(F, T, pts, M, idx, c1, counts, base_out);
}

// ------------------------------------------------------------------ vNMSE
__global__ void k_vnmse(const WorkerPtrs xs, uint32_t n, const float* y, uint64_t d, double* acc) {
  double err = 0.0, ref = 0.0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < d;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double e = 0.0;
    for (uint32_t r = 0; r < n; ++r) e += static_cast<double>(xs.p[r][i]);
    const double diff = static_cast<double>(y[i]) - e;
    err += diff * diff;
    ref += e * e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    err += __shfl_xor_sync(0xffffffffu, err, o);
    ref += __shfl_xor_sync(0xffffffffu, ref, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, err);
    atomicAdd(acc + 1, ref);
  }
}

void launch_vnmse(const float* const* xs, uint32_t n, const float* y, uint64_t d, double* acc2,
                  cudaStream_t st) {
  k_vnmse<<<148 * 4, 256, 0, st>>>(worker_ptrs(xs, n), n, y, d, acc2);
}

}  // namespace dq
