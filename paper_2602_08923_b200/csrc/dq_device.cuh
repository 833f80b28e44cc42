// dq_device.cuh — device-side building blocks of the DynamiQ B200 hot path.
//
// Keyed counter-based PRNG (bit-exact with proj/src/random.cpp:10-90), bf16
// helpers (proj/include/dynamiq/bf16.hpp:12-40) and the tiled SoA chunk layout
// used on HBM and on the wire between GPUs.
//
// Floating point: every float/double expression that must round exactly like
// the x86-64 reference uses explicit _rn intrinsics, and the whole library is
// compiled with --fmad=false -prec-div=true -ftz=false as a second guard.
#pragma once
#include <cstdint>
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>

namespace dq {

constexpr int kS = 256;            // super-group size S (entries)
constexpr int kG = 16;             // group size s (entries)
constexpr int kGroups = kS / kG;   // groups per super-group
constexpr int kTileSG = 64;        // super-groups per layout tile
constexpr int kMetaBytes = 18;     // per-SG scale bytes of the default format: 16 u8 codes + bf16 sg_scale
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kSeedSalt = 0x6a09e667f3bcc909ULL;

enum Purpose : uint32_t { kEntryQuant = 1, kScaleQuant = 2, kPermutation = 3 };

// Device-side bounds and invariant checks of the debug build (-DDQ_DEBUG_CHECKS=1, the
// `debug` variant of tools/build_debug.sh): the stand-in for compute-sanitizer, which this
// GPU pool does not run.  A failed check prints its condition and traps the kernel.
#if defined(DQ_DEBUG_CHECKS) && DQ_DEBUG_CHECKS
#define DQ_CHECK(c)                                                                             \
  do {                                                                                          \
    if (!(c)) {                                                                                 \
      printf("DQ_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c,        \
             blockIdx.x, threadIdx.x);                                                          \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define DQ_CHECK(c) \
  do {              \
  } while (0)
#endif

// Spin-wait budget of every kernel that waits on another GPU or on the host (peer flags,
// the statistics exchange, a host allocation answer): a wait longer than this traps the
// kernel instead of hanging the GPU.  Per device; set from DQ_WAIT_TIMEOUT_S (default
// 600 s, the scale of PyTorch's NCCL timeout) when the device is first used.
extern __device__ uint64_t g_spin_ns;

// Programmatic dependent launch (PDL) along a round's kernel chain: each kernel is launched
// with programmatic stream serialization (launch_pdl), so its CTAs are scheduled and run
// their independent prologue (shared-memory tables) while the predecessor drains;
// pdl_wait() (griddepcontrol.wait) blocks until the predecessor grid has completed and its
// memory is visible - before any read of the predecessor's outputs and any store the
// predecessor could still observe - and pdl_trigger() then lets the successor launch.
// Kernels launched without the attribute see both as no-ops.  Env DQ_PDL=0 turns it off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();
template <class... P, class... A>
inline void launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}
__device__ __forceinline__ uint64_t dq_globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- PRNG
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdULL;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ULL;
  return z ^ (z >> 33);
}
// h' = mix64(h ^ (w + golden + (h << 6) + (h >> 2)))   (proj/src/random.cpp:19-21)
__host__ __device__ __forceinline__ uint64_t absorb(uint64_t h, uint64_t w) {
  return mix64(h ^ (w + kGolden + (h << 6) + (h >> 2)));
}
// The absorb of a counter into a fixed h: the (h-dependent) addend is shared by
// every counter, so a Fisher-Yates draw costs one add + xor + mix64.
__host__ __device__ __forceinline__ uint64_t absorb_base(uint64_t h) {
  return kGolden + (h << 6) + (h >> 2);
}
__host__ __device__ __forceinline__ double unit53(uint64_t b) {
  return static_cast<double>(b >> 11) * 0x1.0p-53;
}
// Prefix of keyed_bits up to and including the purpose word
// (proj/src/random.cpp:25-34): the per-round constant of each purpose.
__host__ __device__ inline uint64_t purpose_prefix(uint64_t seed, uint64_t round, uint32_t purpose) {
  uint64_t h = mix64(seed ^ kSeedSalt);
  h = absorb(h, round);
  return absorb(h, purpose);
}

// r % k for the Fisher-Yates draw, k = i+1 <= 64.  Compile-time k lets nvcc
// strength-reduce; the runtime path handles arbitrary worker counts.
// K = 3, 5: 2^32 = 1 (mod K), so r = lo + hi (mod K); lo + hi < 2^33 folds once more into
// 32 bits (its high word is 0 or 1 and the sum cannot overflow again) and the 32-bit
// remainder is one multiply-high - 5 instructions instead of the 64-bit magic division.
// K = 6: from r mod 3 and the parity of r (CRT).
template <int K>
__host__ __device__ __forceinline__ uint32_t mod_const(uint64_t r) {
  if constexpr ((K & (K - 1)) == 0) {
    return static_cast<uint32_t>(r) & (K - 1);
  } else if constexpr (K == 3 || K == 5) {
    const uint64_t s = (r & 0xffffffffull) + (r >> 32);
    const uint32_t t = static_cast<uint32_t>(s) + static_cast<uint32_t>(s >> 32);
    return t % K;
  } else if constexpr (K == 6) {
    const uint32_t a = mod_const<3>(r);
    return a + 3u * ((a ^ static_cast<uint32_t>(r)) & 1u);
  } else {
    return static_cast<uint32_t>(r % K);
  }
}

// ---------------------------------------------------------------- bf16
__host__ __device__ __forceinline__ float bf16_to_float(uint16_t b) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
#else
  union { uint32_t u; float f; } c{static_cast<uint32_t>(b) << 16};
  return c.f;
#endif
}
// Round to nearest even onto bf16; inf/nan pass through truncated, a nan stays a nan
// (bf16.hpp:17-28, the width-16 passthrough record).
__device__ __forceinline__ uint16_t bf16_rne(float v) {
  uint32_t u = __float_as_uint(v);
  if (((u >> 23) & 0xffu) == 0xffu) {
    uint16_t hi = static_cast<uint16_t>(u >> 16);
    if ((u & 0x7fffffu) != 0 && (hi & 0x7f) == 0) hi |= 1;
    return hi;
  }
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// Round toward +inf onto bf16 with clamp below +inf (bf16.hpp:30-40).
__device__ __forceinline__ uint16_t bf16_round_up(float v) {
  const uint32_t u = __float_as_uint(v);
  const uint16_t hi = static_cast<uint16_t>(u >> 16);
  if ((u & 0xffffu) == 0) return hi;
  const uint16_t up = static_cast<uint16_t>(hi + 1);
  return (up & 0x7f80u) == 0x7f80u ? 0x7f7fu : up;
}

// ---------------------------------------------------------------- layout
// A chunk of nsg super-groups in body order: n8 width-8, then n4 width-4, then
// n2 width-2 super-groups (the reference's wire run order 8,4,2).  Super-groups
// are packed in tiles of 64: [payloads][group scales x cnt][bf16 sg_scale x cnt].
// Every tile starts 64-byte aligned (payloads are 64/128/256 B, metadata is
// (gs + ss) x 64 B for full tiles) and a run of whole tiles is one contiguous
// byte range, which is what the transport pipelines on.
// Scale format (codec.cpp:92-116, the record fields of serialize_chunk):
//   hierarchical (default, s = 16): gs = 256/s u8 codes, ss = 2 (bf16 sg_scale);
//   flat bf16 (ablation): gs = 2 * 256/s bytes (one bf16 per group), ss = 0.
// gshift = log2(s / 8): lanes per group when a warp holds a super-group 8 entries per lane.
// Width-16 passthrough super-groups (codec.cpp:82-86: 256 bf16, no scales) form a fourth
// run after the width-2 run, as on the wire (8, 4, 2, 16); their tile metadata slots
// are reserved but unused (zero), so the device chunk is 18 B per such super-group
// larger than its wire body.
struct Layout {
  uint32_t nsg, n8, n4;
  uint32_t gs = 16, ss = 2, gshift = 1;
  uint32_t n16 = 0;
  __host__ __device__ bool hierarchical() const { return ss != 0; }
  __host__ __device__ bool default_format() const { return gs == 16 && ss == 2 && gshift == 1; }
  __host__ __device__ uint32_t n2() const { return nsg - n8 - n4 - n16; }
  __host__ __device__ uint32_t width(uint32_t i) const {
    return i < n8 ? 8 : (i < n8 + n4 ? 4 : (i < nsg - n16 ? 2 : 16));
  }
  // payload bytes of super-groups [0, k)
  __host__ __device__ uint64_t pay_prefix(uint32_t k) const {
    const uint32_t a = k < n8 ? k : n8;
    const uint32_t r = k - a;
    const uint32_t b = r < n4 ? r : n4;
    const uint32_t r2 = r - b;
    if (n16 == 0) return 256ull * a + 128ull * b + 64ull * r2;  // no passthrough run (every round)
    const uint32_t m2 = n2(), c = r2 < m2 ? r2 : m2;
    return 256ull * a + 128ull * b + 64ull * c + 512ull * (r2 - c);
  }
  // scale-metadata bytes of the wire records of super-groups [0, k) (width 16 has none)
  __host__ __device__ uint64_t meta_prefix(uint32_t k) const {
    const uint32_t scaled = nsg - n16;
    return static_cast<uint64_t>(gs + ss) * (k < scaled ? k : scaled);
  }
  // wire body bytes (serialize_chunk after the 24-byte header)
  __host__ __device__ uint64_t wire_body() const { return pay_prefix(nsg) + meta_prefix(nsg); }
  __host__ __device__ uint64_t tile_offset(uint32_t t) const {
    const uint32_t k = t * kTileSG < nsg ? t * kTileSG : nsg;
    return pay_prefix(k) + static_cast<uint64_t>(gs + ss) * k;
  }
  __host__ __device__ uint32_t tiles() const { return (nsg + kTileSG - 1) / kTileSG; }
  __host__ __device__ uint64_t bytes() const { return tile_offset(tiles()); }
  struct SG {
    uint64_t payload, codes, scale;
    uint32_t width;
  };
  // a super-group of the quantized runs (i < nsg - n16): width without the passthrough test
  __host__ __device__ SG locate_q(uint32_t i) const {
    SG s = locate_at(i);
    s.width = i < n8 ? 8 : (i < n8 + n4 ? 4 : 2);
    return s;
  }
  // width runs of the super-groups [lo, lo + nsg) of a round whose permuted order holds
  // n8 width-8 then n4 width-4 super-groups (then width 2): asynchronous rounds read the
  // round's class counts on the device instead of the host
  __host__ __device__ void runs_from_counts(uint32_t lo, uint32_t c8, uint32_t c4) {
    const uint32_t hi = lo + nsg;
    const uint32_t e8 = hi < c8 ? hi : c8, e4 = hi < c8 + c4 ? hi : c8 + c4, s4 = lo > c8 ? lo : c8;
    n8 = e8 > lo ? e8 - lo : 0;
    n4 = e4 > s4 ? e4 - s4 : 0;
  }
  __host__ __device__ SG locate(uint32_t i) const {
    SG s = locate_at(i);
    s.width = width(i);
    return s;
  }
  __host__ __device__ SG locate_at(uint32_t i) const {
    const uint32_t t = i / kTileSG, first = t * kTileSG;
    const uint32_t last = first + kTileSG < nsg ? first + kTileSG : nsg;
    const uint32_t cnt = last - first;
    const uint64_t base = tile_offset(t);
    const uint64_t tp = pay_prefix(last) - pay_prefix(first);
    SG s;
    s.payload = base + (pay_prefix(i) - pay_prefix(first));
    s.codes = base + tp + static_cast<uint64_t>(gs) * (i - first);
    s.scale = base + tp + static_cast<uint64_t>(gs) * cnt + static_cast<uint64_t>(ss) * (i - first);
    return s;
  }
};

}  // namespace dq
