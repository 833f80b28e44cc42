// dq_wire.cu — device-side reference wire format (proj/src/codec.cpp:319-399).
//
// The reference serializes a chunk as a 24-byte header {chunk, count, n8, n4, n2,
// n16} (u32 little-endian) followed by one record per super-group in chunk order:
// bf16 sg_scale | 16 u8 group codes | 32*w payload bytes.  The device layout is
// the tiled SoA of dq_device.cuh; both are closed-form, so each super-group maps
// record <-> SoA independently: one warp per super-group, 16-bit moves (every
// record and SoA field starts at an even offset).  Parsing validates like the
// reference's strict parser: the first offending super-group in chunk order
// decides the message (codec.cpp:380-395), truncation and trailing bytes are
// decided from the header on the host.
#include <cstdint>

#include <cuda_runtime.h>

#include "dq_device.cuh"
#include "dq_internal.h"

namespace dq {

namespace {

constexpr int kWireThreads = 256;
constexpr int kWireWarps = kWireThreads / 32;

// byte offset of super-group i's record after the 24-byte header
__device__ __forceinline__ uint64_t record_offset(const Layout& L, uint32_t i) {
  return L.pay_prefix(i) + L.meta_prefix(i);
}

// scale bytes of a record: none for width-16 passthrough (codec.cpp:331-336)
__device__ __forceinline__ uint32_t record_meta(const Layout& L, uint32_t width) {
  return width == 16 ? 0u : L.gs + L.ss;
}

// SoA offset of halfword k of super-group i's record: [sg_scale (ss bytes)]
// [group scales (gs bytes)][payload] (codec.cpp:331-337)
__device__ __forceinline__ uint64_t soa_half(const Layout& L, const Layout::SG& g, uint32_t k) {
  if (g.width == 16) return g.payload + 2 * k;
  const uint32_t h0 = L.ss / 2, h1 = (L.ss + L.gs) / 2;
  return k < h0 ? g.scale + 2 * k : (k < h1 ? g.codes + 2 * (k - h0) : g.payload + 2 * (k - h1));
}

__global__ void __launch_bounds__(kWireThreads) k_to_wire(const uint8_t* __restrict__ soa, Layout L, uint32_t chunk,
                                                          uint8_t* __restrict__ out) {
  if (blockIdx.x == 0 && threadIdx.x < 6) {
    const uint32_t v[6] = {chunk, L.nsg, L.n8, L.n4, L.n2(), L.n16};
    reinterpret_cast<uint32_t*>(out)[threadIdx.x] = v[threadIdx.x];  // little-endian like BitWriter
  }
  const uint32_t lane = threadIdx.x & 31;
  uint16_t* rec_base = reinterpret_cast<uint16_t*>(out + 24);
  for (uint32_t i = blockIdx.x * kWireWarps + (threadIdx.x >> 5); i < L.nsg; i += gridDim.x * kWireWarps) {
    const Layout::SG g = L.locate(i);
    uint16_t* rec = rec_base + record_offset(L, i) / 2;
    const uint32_t halves = (record_meta(L, g.width) + 32 * g.width) / 2;
    for (uint32_t k = lane; k < halves; k += 32)
      rec[k] = *reinterpret_cast<const uint16_t*>(soa + soa_half(L, g, k));
  }
}

// Copies (soa != nullptr) and validates super-groups [0, fit): bad = min over
// offending super-groups of (i << 1 | kind), kind 0 = zero sg_scale with a
// nonzero group code, 1 = zero sg_scale with a nonzero payload byte.
__global__ void __launch_bounds__(kWireThreads) k_from_wire(const uint8_t* __restrict__ in, Layout L, uint32_t fit,
                                                            uint8_t* __restrict__ soa,
                                                            unsigned long long* __restrict__ bad) {
  const uint32_t lane = threadIdx.x & 31;
  const uint16_t* rec_base = reinterpret_cast<const uint16_t*>(in + 24);
  for (uint32_t i = blockIdx.x * kWireWarps + (threadIdx.x >> 5); i < fit; i += gridDim.x * kWireWarps) {
    const Layout::SG g = L.locate(i);
    const uint16_t* rec = rec_base + record_offset(L, i) / 2;
    const bool w16 = g.width == 16;
    const uint32_t h0 = w16 ? 0u : L.ss / 2, h1 = w16 ? 0u : (L.ss + L.gs) / 2;
    const uint32_t halves = (record_meta(L, g.width) + 32 * g.width) / 2;
    uint32_t codes_or = 0, pay_or = 0;
    for (uint32_t k = lane; k < halves; k += 32) {
      const uint16_t v = rec[k];
      if (soa) *reinterpret_cast<uint16_t*>(soa + soa_half(L, g, k)) = v;
      if (k >= h0 && k < h1) codes_or |= v;
      else if (k >= h1) pay_or |= v;
    }
    if (soa && w16) {  // the reserved (unused) scale slots of a passthrough super-group read as zero
      for (uint32_t k = lane; k < L.gs / 2; k += 32) *reinterpret_cast<uint16_t*>(soa + g.codes + 2 * k) = 0;
      for (uint32_t k = lane; k < L.ss / 2; k += 32) *reinterpret_cast<uint16_t*>(soa + g.scale + 2 * k) = 0;
    }
    const bool zero_scale = !w16 && L.hierarchical() && rec[0] == 0;  // both sg_scale bytes zero (flat / 16: no check)
    const bool codes_nz = __any_sync(0xffffffffu, codes_or != 0);
    const bool pay_nz = __any_sync(0xffffffffu, pay_or != 0);
    if (lane == 0 && zero_scale && (codes_nz || pay_nz))
      atomicMin(bad, (static_cast<unsigned long long>(i) << 1) | (codes_nz ? 0ull : 1ull));
  }
}

uint32_t wire_grid(uint32_t nsg) {
  const uint32_t want = (nsg + kWireWarps - 1) / kWireWarps;
  const uint32_t cap = 148u * 16;
  return want == 0 ? 1 : (want < cap ? want : cap);
}

}  // namespace

void launch_to_wire(const uint8_t* soa, const Layout& L, uint32_t chunk, uint8_t* out, cudaStream_t st) {
  k_to_wire<<<wire_grid(L.nsg), kWireThreads, 0, st>>>(soa, L, chunk, out);
}

void launch_from_wire(const uint8_t* in, const Layout& L, uint32_t fit, uint8_t* soa, unsigned long long* bad,
                      cudaStream_t st) {
  if (fit == 0) return;
  k_from_wire<<<wire_grid(fit), kWireThreads, 0, st>>>(in, L, fit, soa, bad);
}

}  // namespace dq
