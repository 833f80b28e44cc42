// dq_codec_pc.cu — simulated-round hop kernels with permutation slices (dq_sim_round):
// the chunk's first compression computes every entry's Fisher-Yates permutation and
// stores each later slot's pi, later simulated hops read their slot.  Worker counts
// 2..8, gather operand.
#include "dq_codec.cuh"

namespace dq {
namespace {
template <int NS>
bool launch_pc_ns(const CodecArgs& a, bool dar, cudaStream_t st) {
  if (a.pc_mode == 3 && !dar) {
    launch_hop(k_quant<NS, true, 0, false, false, 3>, a.L.nsg, a, st);
    return true;
  }
  if (a.pc_mode == 4) {
    if (dar) launch_hop(k_quant<NS, true, 0, true, false, 4>, a.L.nsg, a, st);
    else launch_hop(k_quant<NS, true, 0, false, false, 4>, a.L.nsg, a, st);
    return true;
  }
  return false;
}
}  // namespace

bool launch_quant_pc(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  if ((a.pc_mode != 3 && a.pc_mode != 4) || src != 0 || !a.correlated) return false;
  switch (a.n_slots) {
    case 2: return launch_pc_ns<2>(a, dar, st);
    case 3: return launch_pc_ns<3>(a, dar, st);
    case 4: return launch_pc_ns<4>(a, dar, st);
    case 5: return launch_pc_ns<5>(a, dar, st);
    case 6: return launch_pc_ns<6>(a, dar, st);
    case 7: return launch_pc_ns<7>(a, dar, st);
    case 8: return launch_pc_ns<8>(a, dar, st);
    default: return false;
  }
}

}  // namespace dq
