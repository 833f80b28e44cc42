// dq_codec_gen.cu — hop kernels for the ablation scale formats (group size 8..128,
// flat bf16 group scales): runtime format and worker count (GEN = true).
#include "dq_codec.cuh"

namespace dq {
namespace {
template <bool CORR>
void launch_gen(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  constexpr int NS = CORR ? 0 : 1;
  if (src == 0) {
    if (dar) launch_hop(k_quant<NS, CORR, 0, true, true>, a.L.nsg, a, st);
    else launch_hop(k_quant<NS, CORR, 0, false, true>, a.L.nsg, a, st);
  } else {
    if (dar) launch_hop(k_quant<NS, CORR, 1, true, true>, a.L.nsg, a, st);
    else launch_hop(k_quant<NS, CORR, 1, false, true>, a.L.nsg, a, st);
  }
}
}  // namespace

void launch_quant_gen(const CodecArgs& a, int src, bool dar, cudaStream_t st) {
  if (a.correlated) launch_gen<true>(a, src, dar, st);
  else launch_gen<false>(a, src, dar, st);
}

}  // namespace dq
