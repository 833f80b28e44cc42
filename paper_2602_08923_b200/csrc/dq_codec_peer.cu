// dq_codec_peer.cu — peer-transport kernels (fused hop with NVLink peer stores and
// per-unit flags; DA of a peer-delivered message).
#include "dq_codec.cuh"

namespace dq {
namespace {
template <int NS, bool CORR>
void launch_peer_ns(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  const uint32_t units = (a.L.nsg + a.unit - 1) / a.unit;
  const dim3 grid(persistent_grid(units, 64));  // one unit per warp (not persistent: see per_warp_sgs)
  if constexpr (CORR && NS >= 2) {  // ring permutation slices (leaf writes, later hops read)
    if (a.pc_mode == 3 && src == 0 && !dar) {
      launch_pdl(k_quant_peer<NS, true, 0, false, false, 3>, dim3(grid), dim3(kThreads), 0, st, a);
      return;
    }
    if (a.pc_mode == 4 && src == 0 && dar) {
      launch_pdl(k_quant_peer<NS, true, 0, true, false, 4>, dim3(grid), dim3(kThreads), 0, st, a);
      return;
    }
  }
  if (src == 0) {
    if (dar) launch_pdl(k_quant_peer<NS, CORR, 0, true>, dim3(grid), dim3(kThreads), 0, st, a);
    else launch_pdl(k_quant_peer<NS, CORR, 0, false>, dim3(grid), dim3(kThreads), 0, st, a);
  } else {
    if (dar) launch_pdl(k_quant_peer<NS, CORR, 1, true>, dim3(grid), dim3(kThreads), 0, st, a);
    else launch_pdl(k_quant_peer<NS, CORR, 1, false>, dim3(grid), dim3(kThreads), 0, st, a);
  }
}
template <bool CORR>
void launch_peer_corr(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  switch (CORR ? a.n_slots : 1) {
    case 1: return launch_peer_ns<1, CORR>(a, src, dar, st);
    case 2: return launch_peer_ns<2, CORR>(a, src, dar, st);
    case 3: return launch_peer_ns<3, CORR>(a, src, dar, st);
    case 4: return launch_peer_ns<4, CORR>(a, src, dar, st);
    case 5: return launch_peer_ns<5, CORR>(a, src, dar, st);
    case 6: return launch_peer_ns<6, CORR>(a, src, dar, st);
    case 7: return launch_peer_ns<7, CORR>(a, src, dar, st);
    case 8: return launch_peer_ns<8, CORR>(a, src, dar, st);
    default: return launch_peer_ns<0, CORR>(a, src, dar, st);
  }
}
}  // namespace

void launch_da_peer(const CodecArgs& a, int src, cudaStream_t st) {
  if (a.L.nsg == 0) return;
  const uint32_t units = (a.L.nsg + a.unit - 1) / a.unit;
  const dim3 grid(persistent_grid(units, 64));
  if (src == 0) launch_pdl(k_da_peer<0>, dim3(grid), dim3(kThreads), 0, st, a);
  else launch_pdl(k_da_peer<1>, dim3(grid), dim3(kThreads), 0, st, a);
}

void launch_quant_peer(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  if (a.L.nsg == 0) return;
  if (a.correlated) launch_peer_corr<true>(a, src, dar, st);
  else launch_peer_corr<false>(a, src, dar, st);
}

}  // namespace dq
