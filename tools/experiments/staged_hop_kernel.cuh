// EXPERIMENT (not built): the fused hop with its operands staged through shared memory by
// cp.async.bulk (TMA) copies one super-group ahead, completing on per-warp mbarriers.
// Bit-exact (276 GPU tests green with it as the default hop kernel) but slower on B200:
// N=1 round 2.11 ms vs 2.02 ms with the register-path kernel (quant_dar 1.19 vs 1.13 ms per
// step at 64 registers, 1.23 ms at 80 registers / 3 CTAs per SM) - see profiles/r2_kernel_log.md.
// Drop-in for dq_codec.cuh (k_hop<NS, CORR, SRC, DAR, PC, DEC>), launched like k_quant.
// ------------------------------------------------------------ staged hop kernel
// The fused hop with its operands staged through shared memory by the bulk-copy (TMA)
// engine: while a warp quantizes super-group k, one lane has already issued
// cp.async.bulk copies of super-group k+1's local fp32 operand (1 KiB, gathered through
// the width permutation), its incoming compressed record (payload + 16 group codes) and
// its permutation-slice words into the warp's other stage buffer, completing on that
// stage's mbarrier.  The dependent address chain (perm -> gradient row, layout -> record)
// therefore leaves the critical path; the 2-byte sg_scale is prefetched into a register.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "DQ_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra DQ_WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <bool DAR, bool PIN>
struct alignas(16) HopStage {
  float x[kS];                  // local operand (raw gradient row or accumulator row)
  uint8_t pay[DAR ? 256 : 16];  // incoming payload (W * 32 bytes)
  uint8_t codes[16];            // incoming group-scale codes
  uint32_t pin[PIN ? 32 : 4];   // permutation-slice words (PC 4)
};
template <bool DAR, bool PIN>
struct WarpStages {
  HopStage<DAR, PIN> st[2];
  uint64_t bar[2];
};

// decode of the staged incoming record (codec.cpp:128-162; same arithmetic as decode8w)
template <int W, class Stage>
__device__ __forceinline__ void decode_staged(const Stage& s, float sgs, int lane, const SmemBooks& sb,
                                              float dec[8]) {
  const float sf = div255(__fmul_rn(static_cast<float>(s.codes[lane >> 1]), sgs));
  uint64_t bits;
  if constexpr (W == 8) bits = *reinterpret_cast<const uint64_t*>(s.pay + lane * 8);
  else if constexpr (W == 4) bits = *reinterpret_cast<const uint32_t*>(s.pay + lane * 4);
  else bits = *reinterpret_cast<const uint16_t*>(s.pay + lane * 2);
  const float* q = sb.book(W);
  constexpr uint32_t mask = (1u << W) - 1u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t c = static_cast<uint32_t>(bits >> (j * W)) & mask;
    float mag;
    if constexpr (W == 2) mag = (c >> 1) ? sf : 0.0f;
    else mag = __fmul_rn(q[c >> 1], sf);
    dec[j] = __uint_as_float(__float_as_uint(mag) ^ (c << 31));
  }
}

// SRC 0: gather from the raw gradient through the permutation (normalize fused), SRC 1:
// chunk-local accumulator.  Default scale format, no passthrough run (launch_quant).
template <int NS, bool CORR, int SRC, bool DAR, int PC = 0, bool DEC = false>
__global__ void __launch_bounds__(kThreads, kHopMinBlocks) k_hop(const CodecArgs a) {
  __shared__ SmemQuant sq;
  __shared__ WarpScratch ws[kWarps];
  __shared__ FYTab<PC == 3 ? NS : 1> fy;
  __shared__ WarpStages<DAR, PC == 4> wst[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if constexpr (PC == 3) build_fy(fy);
  WarpStages<DAR, PC == 4>& W = wst[warp];
  if (lane == 0) {
    mbar_init(&W.bar[0], 1);
    mbar_init(&W.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  load_quant_tables(sq, a);  // ends with __syncthreads (also publishes the barrier init)
  const uint32_t nq = a.L.nsg - a.L.n16;
  const uint32_t stride = gridDim.x * kWarps, i0 = blockIdx.x * kWarps + warp;
  if (i0 >= nq) return;
  const uint64_t slot_hi = static_cast<uint64_t>(a.slot) << 32;

  // batch of up to 10 super-groups: key prefixes + (lanes 0..9) permuted row / mean
  KeyBatch kb{};
  uint32_t b_src = 0;
  float b_mu = 0.0f;
  auto batch = [&](uint32_t ib) {
    kb.compute(a, ib, stride, lane);
    if constexpr (SRC == 0) {
      const uint32_t il = ib + static_cast<uint32_t>(lane < 10 ? lane : 0) * stride;
      if (lane < 10 && il < nq) {
        b_src = __ldg(a.perm + a.first_sg + il);
        b_mu = __ldg(a.gmean + a.first_sg + il);
      }
    }
  };
  // issue super-group i (batch slot kk) into stage s; returns its location and, for the
  // DAR, prefetches its sg_scale
  auto issue = [&](uint32_t i, int kk, int s, Layout::SG& loc, uint16_t& scale, bool& direct) {
    loc = a.L.locate_q(i);
    const float* xrow;
    if constexpr (SRC == 0) {
      const uint32_t src = __shfl_sync(0xffffffffu, b_src, kk);
      xrow = a.x + static_cast<uint64_t>(src) * kS;
      direct = static_cast<uint64_t>(src) * kS + kS > a.d;  // zero-padded tail row: plain loads
    } else {
      xrow = a.acc_in + static_cast<uint64_t>(i) * kS;
      direct = false;
    }
    const uint32_t pay = DAR ? loc.width * 32 : 0;
    const uint32_t bytes = (direct ? 0 : 1024) + (DAR ? pay + 16 : 0) + (PC == 4 ? 128 : 0);
    if (lane == 0) {
      auto& st = W.st[s];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of the stage
      mbar_expect_tx(&W.bar[s], bytes);
      if (!direct) bulk_g2s(st.x, xrow, 1024, &W.bar[s]);
      if constexpr (DAR) {
        bulk_g2s(st.pay, a.in + loc.payload, pay, &W.bar[s]);
        bulk_g2s(st.codes, a.in + loc.codes, 16, &W.bar[s]);
      }
      if constexpr (PC == 4) bulk_g2s(st.pin, a.pin + static_cast<uint64_t>(i) * 32, 128, &W.bar[s]);
    }
    if constexpr (DAR) scale = *reinterpret_cast<const uint16_t*>(a.in + loc.scale);
  };

  batch(i0);
  Layout::SG loc_cur, loc_nxt;
  uint16_t sc_cur = 0, sc_nxt = 0;
  bool dir_cur = false, dir_nxt = false;
  issue(i0, 0, 0, loc_cur, sc_cur, dir_cur);
  uint64_t ub = 0;
  int kk = 0;
  uint32_t k = 0;
  for (uint32_t i = i0; i < nq; i += stride, ++k) {
    SgKeys keys{};
    if ((kk & 1) == 0) ub = pair_scale_bits(kb, kk, slot_hi, lane);
    keys.h4e = kb.get(0, kk);
    if constexpr (CORR && PC != 4) keys.h4p = kb.get(2, kk);
    keys.ugc = unit53(shfl64(ub, (lane & ~1) | (kk & 1)));
    float mu = 0.0f;
    uint32_t src_row = i;
    if constexpr (SRC == 0) {
      mu = __shfl_sync(0xffffffffu, b_mu, kk);
      src_row = __shfl_sync(0xffffffffu, b_src, kk);
    }
    const uint32_t inext = i + stride;
    int kn = kk + 1;
    if (kn == 10) {
      if (inext < nq) batch(inext);
      kn = 0;
    }
    __syncwarp();  // every lane is done with stage (k+1)&1 (super-group k-1)
    if (inext < nq) issue(inext, kn, (k + 1) & 1, loc_nxt, sc_nxt, dir_nxt);
    const int s = k & 1;
    mbar_wait(&W.bar[s], (k >> 1) & 1);
    const auto& st = W.st[s];
    float x[8];
    if (!dir_cur) {
      const float4 v0 = *reinterpret_cast<const float4*>(st.x + lane * 8);
      const float4 v1 = *reinterpret_cast<const float4*>(st.x + lane * 8 + 4);
      x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
      x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
    } else {
      const uint64_t base = static_cast<uint64_t>(src_row) * kS + lane * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = base + j < a.d ? a.x[base + j] : 0.0f;  // zero padding
    }
    if constexpr (SRC == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = __fsub_rn(x[j], mu);
    }
    if constexpr (PC == 4) keys.pin_word = st.pin[lane];
    const float sgs_in = bf16_to_float(sc_cur);
    auto run = [&](auto wc) {
      constexpr int Wd = decltype(wc)::value;
      if constexpr (DAR) {
        float dec[8];
        decode_staged<Wd>(st, sgs_in, lane, sq.b, dec);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __fadd_rn(dec[j], x[j]);  // codec.cpp:259-261
      }
      quantize_sg<Wd, NS, CORR, OutOne, false, PC, DEC, true>(a, sq, ws[warp], OutOne{a.out}, loc_cur, a.first_sg + i,
                                                             lane, x, &fy, keys);
    };
    if (loc_cur.width == 2) run(std::integral_constant<int, 2>{});
    else if (loc_cur.width == 4) run(std::integral_constant<int, 4>{});
    else run(std::integral_constant<int, 8>{});
    loc_cur = loc_nxt;
    sc_cur = sc_nxt;
    dir_cur = dir_nxt;
    kk = kn;
  }
}

