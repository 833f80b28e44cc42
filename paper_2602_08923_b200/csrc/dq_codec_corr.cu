// dq_codec_corr.cu — correlated-rounding hop kernels, default scale format: one
// instantiation per worker count 1..8 (compile-time Fisher-Yates trace) and a runtime
// path for larger counts, x (gather | accumulator) x (leaf | DAR).
#include "dq_codec.cuh"

namespace dq {
namespace {
template <int NS>
void launch_ns(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  if (src == 0) {
    if (dar) launch_hop(k_quant<NS, true, 0, true>, a.L.nsg, a, st);
    else launch_hop(k_quant<NS, true, 0, false>, a.L.nsg, a, st);
  } else {
    if (dar) launch_hop(k_quant<NS, true, 1, true>, a.L.nsg, a, st);
    else launch_hop(k_quant<NS, true, 1, false>, a.L.nsg, a, st);
  }
}
}  // namespace

void launch_quant_corr(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  switch (a.n_slots) {
    case 1: return launch_ns<1>(a, src, dar, st);
    case 2: return launch_ns<2>(a, src, dar, st);
    case 3: return launch_ns<3>(a, src, dar, st);
    case 4: return launch_ns<4>(a, src, dar, st);
    case 5: return launch_ns<5>(a, src, dar, st);
    case 6: return launch_ns<6>(a, src, dar, st);
    case 7: return launch_ns<7>(a, src, dar, st);
    case 8: return launch_ns<8>(a, src, dar, st);
    default: return launch_ns<0>(a, src, dar, st);
  }
}

}  // namespace dq
