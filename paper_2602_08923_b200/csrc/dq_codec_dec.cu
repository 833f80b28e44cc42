// dq_codec_dec.cu — sink hops with the chunk's decode fused in (CodecArgs::dec_out).
// A chunk's sink DAR produces the record every rank decodes into its output
// (engine.cpp:219-229 all-gather, then decompress + unpermute + denormalize,
// allocation.cpp:312-325, stats.cpp:65-78); the rank (or simulated round) that runs
// the sink already holds the record in registers, so it stores the decoded values
// too and the gather decode skips that chunk.  Default scale format only.
#include "dq_codec.cuh"

namespace dq {
namespace {
template <int NS, bool CORR>
void launch_peer_dec(const CodecArgs& a, int src, cudaStream_t st) {
  const uint32_t units = (a.L.nsg + a.unit - 1) / a.unit;
  const dim3 grid(persistent_grid(units, 64));
  if constexpr (CORR && NS >= 2) {
    if (a.pc_mode == 4 && src == 0) {  // ring sink reading its permutation slice
      launch_pdl(k_quant_peer<NS, true, 0, true, true, 4>, dim3(grid), dim3(kThreads), 0, st, a);
      return;
    }
  }
  if (src == 0) launch_pdl(k_quant_peer<NS, CORR, 0, true, true>, dim3(grid), dim3(kThreads), 0, st, a);
  else launch_pdl(k_quant_peer<NS, CORR, 1, true, true>, dim3(grid), dim3(kThreads), 0, st, a);
}

void launch_peer_dec_corr(const CodecArgs& a, int src, cudaStream_t st) {
  switch (a.n_slots) {
    case 1: return launch_peer_dec<1, true>(a, src, st);
    case 2: return launch_peer_dec<2, true>(a, src, st);
    case 3: return launch_peer_dec<3, true>(a, src, st);
    case 4: return launch_peer_dec<4, true>(a, src, st);
    case 5: return launch_peer_dec<5, true>(a, src, st);
    case 6: return launch_peer_dec<6, true>(a, src, st);
    case 7: return launch_peer_dec<7, true>(a, src, st);
    case 8: return launch_peer_dec<8, true>(a, src, st);
    default: return launch_peer_dec<0, true>(a, src, st);
  }
}

template <int NS>
bool launch_pc_dec(const CodecArgs& a, cudaStream_t st, bool launch) {
  if (!launch) return true;
  launch_hop(k_quant<NS, true, 0, true, false, 4, true>, a.L.nsg, a, st);
  return true;
}
}  // namespace

bool launch_quant_dec(const CodecArgs& a, int src, bool peer, cudaStream_t st, bool launch) {
  if (!a.dec_out || a.L.nsg == 0 || !a.L.default_format() || a.L.n16) return false;
  if (peer) {
    if (!launch) return true;
    if (a.correlated) launch_peer_dec_corr(a, src, st);
    else launch_peer_dec<1, false>(a, src, st);
    return true;
  }
  if (!a.correlated) {  // independent rounding: no permutation
    if (!launch) return true;
    if (src == 0) launch_hop(k_quant<1, false, 0, true, false, 0, true>, a.L.nsg, a, st);
    else launch_hop(k_quant<1, false, 1, true, false, 0, true>, a.L.nsg, a, st);
    return true;
  }
  if (a.pc_mode != 4 || src != 0) return false;  // correlated: the slice-reading sink only
  switch (a.n_slots) {
    case 2: return launch_pc_dec<2>(a, st, launch);
    case 3: return launch_pc_dec<3>(a, st, launch);
    case 4: return launch_pc_dec<4>(a, st, launch);
    case 5: return launch_pc_dec<5>(a, st, launch);
    case 6: return launch_pc_dec<6>(a, st, launch);
    case 7: return launch_pc_dec<7>(a, st, launch);
    case 8: return launch_pc_dec<8>(a, st, launch);
    default: return false;
  }
}

}  // namespace dq
