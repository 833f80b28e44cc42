// dynamiq_b200.hpp — header-only C++ drop-in for the reference's hot-path API.
//
// A caller of the reference library (namespace dynamiq, proj/include/dynamiq/)
// switches to the B200 path by including this header and using namespace
// dynamiq_b200: the same function names, argument meaning, return types and
// exception types, implemented over the C-ABI in dynamiq_b200.h (device
// buffers, sm_100a kernels).  Host spans in, host vectors out, exactly like the
// reference; device-resident callers use the C-ABI directly.
//
//   reference                                         here
//   codec.hpp:64  compress_chunk(values, widths, books, cfg, qctx, first_sg)
//   codec.hpp:71  decompress_chunk(chunk, books, cfg, out)
//   codec.hpp:75  decompress_accumulate(chunk, acc, books, cfg)
//   codec.hpp:86  decompress_accumulate_recompress(chunk, local, books, cfg, qctx, first_sg)
//   codec.hpp:94  serialize_chunk(chunk, cfg) / parse_chunk(bytes, cfg)
//   stats.hpp:19  compute_stats / reduce_stats
//   allocation.hpp:63 allocate_fast(sq_norms, spec)
//   allocation.hpp:57 allocate_general(sq_norms, spec), :80 allocate_fast_stateful(sq_norms, spec, state)
//   engine.hpp:63 run_round(worker_values, config)
//
// CompressedChunk keeps the reference's serialized bytes (its wire format), so
// chunks interoperate with the reference library byte for byte.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dynamiq_b200.h"

namespace dynamiq_b200 {

struct InfeasibleBudget : std::runtime_error {  // allocation.hpp:14-16
  explicit InfeasibleBudget(const std::string& w) : std::runtime_error(w) {}
};

namespace detail {
inline void check(int rc) {
  if (rc == DQ_OK) return;
  const std::string msg = dq_last_error();
  if (rc == DQ_EINVAL) throw std::invalid_argument(msg);
  if (rc == DQ_EINFEASIBLE) throw InfeasibleBudget(msg);
  if (rc == DQ_EMALFORMED) throw std::runtime_error(msg);
  throw std::runtime_error("dynamiq_b200: " + msg);
}
inline void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("dynamiq_b200: ") + cudaGetErrorString(e));
}
template <class T>
struct Dev {  // owning device buffer
  T* p = nullptr;
  explicit Dev(size_t n) { cuda(cudaMalloc(&p, sizeof(T) * (n ? n : 1))); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};
struct Runs {
  uint32_t n8 = 0, n4 = 0, n2 = 0, n16 = 0;
  size_t count() const { return static_cast<size_t>(n8) + n4 + n2 + n16; }
};
inline Runs runs_of(std::span<const uint8_t> widths) {  // codec.cpp:298-315 order check
  Runs r;
  int prev = -1;
  for (uint8_t w : widths) {
    const int cls = w == 8 ? 0 : w == 4 ? 1 : w == 2 ? 2 : w == 16 ? 3 : -1;
    if (cls < 0) throw std::invalid_argument("unsupported codec width " + std::to_string(w));
    if (cls < prev) throw std::invalid_argument("chunk body must be ordered by width class 8,4,2,16");
    prev = cls;
    (cls == 0 ? r.n8 : cls == 1 ? r.n4 : cls == 2 ? r.n2 : r.n16)++;
  }
  return r;
}
inline std::vector<uint8_t> widths_of(const Runs& r) {
  std::vector<uint8_t> w(r.n8, 8);
  w.insert(w.end(), r.n4, 4);
  w.insert(w.end(), r.n2, 2);
  w.insert(w.end(), r.n16, 16);
  return w;
}
}  // namespace detail

struct SharedSeed {  // random.hpp:12-15
  std::uint64_t seed = 0;
  std::uint64_t round = 0;
};

struct QuantContext {  // codec.hpp:33-40
  SharedSeed seed;
  std::uint32_t chunk_index = 0;
  std::uint32_t hop_slot = 0;
  std::uint32_t n_slots = 1;
  bool correlated = true;
};

struct CodecConfig {  // codec.hpp:26-31 (device: S = 256, s in {8,16,32,64,128}, hierarchical or flat)
  std::uint32_t group_size = 16;
  std::uint32_t super_group_size = 256;
  bool hierarchical_scales = true;
  void validate() const {
    if (group_size == 0 || super_group_size % group_size != 0)
      throw std::invalid_argument("super-group size must be a positive multiple of the group size");
    if (super_group_size % 4 != 0) throw std::invalid_argument("super-group size must be a multiple of 4 for byte alignment");
    if (super_group_size != 256 ||
        (group_size != 8 && group_size != 16 && group_size != 32 && group_size != 64 && group_size != 128))
      throw std::invalid_argument("device codec supports S=256 with s in {8, 16, 32, 64, 128}");
  }
};

// Stand-in for CodebookSet: which default family (codebook.hpp:46-52).
struct CodebookSet {
  bool non_uniform = true;
  static CodebookSet non_uniform_defaults() { return {true}; }
  static CodebookSet uniform_all() { return {false}; }
};

struct CompressedChunk {  // codec.hpp:20-31, held as the reference's serialized bytes
  std::uint32_t chunk_index = 0;
  std::vector<std::uint8_t> widths;
  std::vector<std::uint8_t> wire;  // serialize_chunk() bytes
};

inline std::uint64_t compressed_size_bits(std::span<const std::uint8_t> widths, std::uint32_t S, std::uint32_t s,
                                          bool hierarchical_scales) {  // codec.cpp:281-291
  std::uint64_t bits = 6 * 32;
  for (std::uint8_t w : widths) {
    if (w != 2 && w != 4 && w != 8 && w != 16) throw std::invalid_argument("unsupported codec width");
    bits += static_cast<std::uint64_t>(S) * w;
    if (w != 16) bits += hierarchical_scales ? 16 + static_cast<std::uint64_t>(S / s) * 8 : static_cast<std::uint64_t>(S / s) * 16;
  }
  return bits;
}

namespace detail {
// reference bytes -> device SoA chunk
inline std::unique_ptr<Dev<uint8_t>> upload(const CompressedChunk& c, Runs* r) {
  std::vector<uint8_t> soa(c.wire.size() * 2 + 64);  // >= device size (passthrough: +18 B per 512 B record)
  uint32_t ci = 0;
  check(dq_from_reference_wire(c.wire.data(), c.wire.size(), soa.data(), soa.size(), &ci, &r->n8, &r->n4, &r->n2,
                               &r->n16));
  const size_t bytes = dq_chunk_bytes(r->n8, r->n4, r->n2, r->n16);
  auto d = std::make_unique<Dev<uint8_t>>(bytes);
  cuda(cudaMemcpy(d->p, soa.data(), bytes, cudaMemcpyHostToDevice));
  return d;
}
inline CompressedChunk download(const uint8_t* dsoa, uint32_t chunk_index, Runs r) {
  const size_t bytes = dq_chunk_bytes(r.n8, r.n4, r.n2, r.n16);
  std::vector<uint8_t> soa(bytes + 1);
  cuda(cudaMemcpy(soa.data(), dsoa, bytes, cudaMemcpyDeviceToHost));
  CompressedChunk c;
  c.chunk_index = chunk_index;
  c.widths = widths_of(r);
  c.wire.resize(dq_wire_bytes(r.n8, r.n4, r.n2, r.n16));
  check(dq_to_reference_wire(soa.data(), chunk_index, r.n8, r.n4, r.n2, r.n16, c.wire.data()));
  return c;
}
inline dq_qctx qctx(const QuantContext& q) {
  return dq_qctx{q.seed.seed, q.seed.round, q.chunk_index, q.hop_slot, q.n_slots, q.correlated ? 1 : 0};
}
// the chunk primitives' scale format (CodecConfig) for the scope of one call
struct FormatScope {
  std::uint32_t gs = 16;
  int hier = 1;
  explicit FormatScope(const CodecConfig& c) {
    check(dq_codec_format_set(c.group_size, c.hierarchical_scales ? 1 : 0, &gs, &hier));
  }
  ~FormatScope() { dq_codec_format_set(gs, hier, nullptr, nullptr); }
  FormatScope(const FormatScope&) = delete;
  FormatScope& operator=(const FormatScope&) = delete;
};
}  // namespace detail

inline CompressedChunk compress_chunk(std::span<const float> values, std::span<const std::uint8_t> widths,
                                      const CodebookSet& books, const CodecConfig& cfg, const QuantContext& q,
                                      std::uint32_t first_sg_index) {
  cfg.validate();
  const detail::FormatScope fmt(cfg);
  if (values.size() != widths.size() * cfg.super_group_size)
    throw std::invalid_argument("chunk length does not match widths");
  const detail::Runs r = detail::runs_of(widths);
  detail::Dev<float> dv(values.size());
  detail::Dev<uint8_t> out(dq_chunk_bytes(r.n8, r.n4, r.n2, r.n16));
  detail::cuda(cudaMemcpy(dv.p, values.data(), values.size_bytes(), cudaMemcpyHostToDevice));
  const dq_qctx c = detail::qctx(q);
  detail::check(dq_compress_chunk(dv.p, r.n8, r.n4, r.n2, r.n16, &c, first_sg_index, books.non_uniform, out.p,
                                  nullptr));
  return detail::download(out.p, q.chunk_index, r);
}

inline CompressedChunk decompress_accumulate_recompress(const CompressedChunk& chunk, std::span<const float> local,
                                                        const CodebookSet& books, const CodecConfig& cfg,
                                                        const QuantContext& q, std::uint32_t first_sg_index) {
  cfg.validate();
  const detail::FormatScope fmt(cfg);
  detail::Runs r;
  auto in = detail::upload(chunk, &r);
  if (local.size() != r.count() * 256) throw std::invalid_argument("local buffer length does not match chunk");
  detail::Dev<float> dl(local.size());
  detail::Dev<uint8_t> out(dq_chunk_bytes(r.n8, r.n4, r.n2, r.n16));
  detail::cuda(cudaMemcpy(dl.p, local.data(), local.size_bytes(), cudaMemcpyHostToDevice));
  const dq_qctx c = detail::qctx(q);
  detail::check(dq_dar_chunk(in->p, dl.p, r.n8, r.n4, r.n2, r.n16, &c, first_sg_index, books.non_uniform, out.p,
                             nullptr));
  return detail::download(out.p, q.chunk_index, r);
}

inline void decompress_chunk(const CompressedChunk& chunk, const CodebookSet& books, const CodecConfig& cfg,
                             std::span<float> out) {
  cfg.validate();
  const detail::FormatScope fmt(cfg);
  detail::Runs r;
  auto in = detail::upload(chunk, &r);
  if (out.size() != r.count() * 256) throw std::invalid_argument("output length does not match chunk");
  detail::Dev<float> d(out.size());
  detail::check(dq_decompress_chunk(in->p, d.p, r.n8, r.n4, r.n2, r.n16, books.non_uniform, nullptr));
  detail::cuda(cudaMemcpy(out.data(), d.p, out.size_bytes(), cudaMemcpyDeviceToHost));
}

inline void decompress_accumulate(const CompressedChunk& chunk, std::span<float> acc, const CodebookSet& books,
                                  const CodecConfig& cfg) {
  cfg.validate();
  const detail::FormatScope fmt(cfg);
  detail::Runs r;
  auto in = detail::upload(chunk, &r);
  if (acc.size() != r.count() * 256) throw std::invalid_argument("accumulator length does not match chunk");
  detail::Dev<float> d(acc.size());
  detail::cuda(cudaMemcpy(d.p, acc.data(), acc.size_bytes(), cudaMemcpyHostToDevice));
  detail::check(dq_da_chunk(in->p, d.p, r.n8, r.n4, r.n2, r.n16, books.non_uniform, nullptr));
  detail::cuda(cudaMemcpy(acc.data(), d.p, acc.size_bytes(), cudaMemcpyDeviceToHost));
}

inline std::vector<std::uint8_t> serialize_chunk(const CompressedChunk& chunk, const CodecConfig& cfg) {
  cfg.validate();
  const detail::FormatScope fmt(cfg);
  return chunk.wire;
}

inline CompressedChunk parse_chunk(std::span<const std::uint8_t> bytes, const CodecConfig& cfg) {  // strict
  cfg.validate();
  const detail::FormatScope fmt(cfg);
  CompressedChunk c;
  c.wire.assign(bytes.begin(), bytes.end());
  std::vector<uint8_t> soa(bytes.size() * 2 + 64);
  detail::Runs r;
  detail::check(dq_from_reference_wire(bytes.data(), bytes.size(), soa.data(), soa.size(), &c.chunk_index, &r.n8,
                                       &r.n4, &r.n2, &r.n16));
  c.widths = detail::widths_of(r);
  return c;
}

struct SuperGroupStats {  // stats.hpp:14-17
  float mean = 0.0f;
  float sq_norm = 0.0f;
};

inline std::vector<SuperGroupStats> compute_stats(std::span<const float> values) {
  const size_t T = (values.size() + 255) / 256;
  detail::Dev<float> x(values.size()), m(T), q(T);
  detail::cuda(cudaMemcpy(x.p, values.data(), values.size_bytes(), cudaMemcpyHostToDevice));
  detail::check(dq_compute_stats(x.p, values.size(), m.p, q.p, nullptr));
  std::vector<float> hm(T), hq(T);
  detail::cuda(cudaMemcpy(hm.data(), m.p, T * 4, cudaMemcpyDeviceToHost));
  detail::cuda(cudaMemcpy(hq.data(), q.p, T * 4, cudaMemcpyDeviceToHost));
  std::vector<SuperGroupStats> s(T);
  for (size_t j = 0; j < T; ++j) s[j] = {hm[j], hq[j]};
  return s;
}

struct BudgetSpec {  // allocation.hpp:24-30 (fast allocator: W = {2,4,8})
  double total_bits_per_coordinate = 5.0;
  std::uint32_t group_size = 16;
  std::uint32_t super_group_size = 256;
  std::vector<int> widths = {2, 4, 8};
  bool hierarchical_scales = true;
};

struct BitAllocation {  // allocation.hpp:40-45
  std::vector<std::uint8_t> widths;
  std::vector<std::uint32_t> permutation;
  std::uint64_t payload_bits = 0;
  double u = 0.0;
};

struct FastAllocatorState {  // allocation.hpp:75-79
  double lo = -1e6;
  double hi = 1e6;
  double u = 0.0;
};

namespace detail {
// upload the norms, run one device allocator on a scratch context, download widths / permutation
template <class Call>
inline BitAllocation run_allocator(std::span<const float> sq_norms, const BudgetSpec& spec, Call&& call) {
  dq_config c;
  dq_config_default(&c);
  c.budget_bits = spec.total_bits_per_coordinate;
  c.group_size = spec.group_size;
  c.super_group_size = spec.super_group_size;
  c.hierarchical_scales = spec.hierarchical_scales;
  dq_ctx* ctx = nullptr;
  check(dq_ctx_create(&c, 0, &ctx));
  std::unique_ptr<dq_ctx, int (*)(dq_ctx*)> guard(ctx, dq_ctx_destroy);
  const size_t T = sq_norms.size();
  Dev<float> F(T);
  Dev<uint8_t> w(T);
  Dev<uint32_t> p(T);
  cuda(cudaMemcpy(F.p, sq_norms.data(), T * 4, cudaMemcpyHostToDevice));
  BitAllocation a;
  uint32_t counts[3];
  check(call(ctx, F.p, T, w.p, p.p, &a.u, &a.payload_bits, counts));
  a.widths.resize(T);
  a.permutation.resize(T);
  cuda(cudaMemcpy(a.widths.data(), w.p, T, cudaMemcpyDeviceToHost));
  cuda(cudaMemcpy(a.permutation.data(), p.p, T * 4, cudaMemcpyDeviceToHost));
  return a;
}
}  // namespace detail

inline BitAllocation allocate_fast(std::span<const float> sq_norms, const BudgetSpec& spec) {
  if (spec.widths != std::vector<int>{2, 4, 8}) throw std::invalid_argument("allocate_fast requires W = {2,4,8}");
  return detail::run_allocator(sq_norms, spec, [&](dq_ctx* ctx, const float* F, size_t T, uint8_t* w, uint32_t* p,
                                                   double* u, uint64_t* pay, uint32_t* counts) {
    return dq_allocate_fast(ctx, F, T, spec.total_bits_per_coordinate, w, p, u, pay, counts, nullptr);
  });
}

// allocation.hpp:57 — the device covers W = {2,4,8}, the set run_round uses (engine.cpp:306-307)
inline BitAllocation allocate_general(std::span<const float> sq_norms, const BudgetSpec& spec) {
  if (spec.widths != std::vector<int>{2, 4, 8})
    throw std::invalid_argument("device allocate_general supports W = {2,4,8}");
  return detail::run_allocator(sq_norms, spec, [&](dq_ctx* ctx, const float* F, size_t T, uint8_t* w, uint32_t* p,
                                                   double* u, uint64_t* pay, uint32_t* counts) {
    return dq_allocate_general(ctx, F, T, spec.total_bits_per_coordinate, w, p, u, pay, counts, nullptr);
  });
}

// allocation.hpp:80-81
inline BitAllocation allocate_fast_stateful(std::span<const float> sq_norms, const BudgetSpec& spec,
                                            FastAllocatorState& state) {
  if (spec.widths != std::vector<int>{2, 4, 8}) throw std::invalid_argument("allocate_fast requires W = {2,4,8}");
  double st[3] = {state.lo, state.hi, state.u};
  BitAllocation a = detail::run_allocator(
      sq_norms, spec, [&](dq_ctx* ctx, const float* F, size_t T, uint8_t* w, uint32_t* p, double* u, uint64_t* pay,
                          uint32_t* counts) {
        return dq_allocate_fast_stateful(ctx, F, T, spec.total_bits_per_coordinate, st, w, p, u, pay, counts,
                                         nullptr);
      });
  state.lo = st[0];
  state.hi = st[1];
  state.u = st[2];
  return a;
}

enum class TopologyKind { kRing, kButterfly };
enum class AllocatorKind { kGeneral, kFast, kFixed };
enum class CodecKind { kQuantized, kLossless };

struct PipelineConfig {  // engine.hpp:22-43
  std::uint32_t n_workers = 4;
  std::uint32_t group_size = 16;
  std::uint32_t super_group_size = 256;
  double budget_bits = 5.0;
  bool non_uniform = true;
  bool variable_width = true;
  bool hierarchical_scales = true;
  bool correlated = true;
  int fixed_width = 4;
  AllocatorKind allocator = AllocatorKind::kFast;
  TopologyKind topology = TopologyKind::kRing;
  CodecKind codec = CodecKind::kQuantized;
  SharedSeed seed{1, 0};
  unsigned threads = 1;
};

// metrics.hpp:20-40 WireVolume: the round's wire accounting by phase and field
struct WireVolume {
  std::uint64_t stats_bits = 0;    // stats all-reduce, 2 x 32 per super-group per hop
  std::uint64_t payload_bits = 0;  // packed entries over all transmissions
  std::uint64_t scale_bits = 0;    // group + super-group scales over all transmissions
  std::uint64_t header_bits = 0;   // chunk headers over all transmissions
  std::uint64_t repr_bits = 0;     // per compression event (forwarded copies excluded)
  std::uint64_t compressed_coordinates = 0;
  std::uint64_t transmitted_coordinates = 0;
  std::uint64_t total_bits() const { return stats_bits + payload_bits + scale_bits + header_bits; }
  // metrics.cpp:39-43 (also as the free function below)
  double bits_per_coordinate() const {
    return compressed_coordinates == 0 ? 0.0
                                       : static_cast<double>(repr_bits) / static_cast<double>(compressed_coordinates);
  }
};
inline double bits_per_coordinate(const WireVolume& w) { return w.bits_per_coordinate(); }
inline double stats_phase_fraction(const WireVolume& w) {  // metrics.cpp:45-49
  return w.transmitted_coordinates == 0 ? 0.0
                                        : static_cast<double>(w.stats_bits) / (16.0 * static_cast<double>(w.transmitted_coordinates));
}

struct RoundResult {  // engine.hpp:45-54 (exact sum / hop errors: reference-side diagnostics)
  std::vector<float> synced;
  double vnmse = 0.0;
  double mse = 0.0;
  WireVolume wire;
  std::uint64_t wire_hash = 0;
  BitAllocation allocation;
  dq_round_info info{};
};

inline RoundResult run_round(const std::vector<std::vector<float>>& worker_values, const PipelineConfig& p,
                             bool collect_wire = true) {
  if (worker_values.empty()) throw std::invalid_argument("no workers");
  for (const auto& v : worker_values)
    if (v.size() != worker_values.front().size()) throw std::invalid_argument("worker gradients must have equal length");
  if (worker_values.front().empty()) throw std::invalid_argument("empty gradient");
  if (worker_values.size() != p.n_workers) throw std::invalid_argument("worker count does not match config");
  dq_config c;
  dq_config_default(&c);
  c.n_workers = p.n_workers;
  c.group_size = p.group_size;
  c.super_group_size = p.super_group_size;
  c.budget_bits = p.budget_bits;
  c.non_uniform = p.non_uniform;
  c.variable_width = p.variable_width;
  c.hierarchical_scales = p.hierarchical_scales;
  c.correlated = p.correlated;
  c.fixed_width = p.fixed_width;
  c.allocator = static_cast<int32_t>(p.allocator);
  c.topology = static_cast<int32_t>(p.topology);
  c.codec = static_cast<int32_t>(p.codec);
  c.seed = p.seed.seed;
  c.round = p.seed.round;
  c.threads = p.threads;
  dq_ctx* ctx = nullptr;
  detail::check(dq_ctx_create(&c, 0, &ctx));
  std::unique_ptr<dq_ctx, int (*)(dq_ctx*)> guard(ctx, dq_ctx_destroy);
  const size_t d = worker_values.front().size(), n = worker_values.size();
  std::vector<std::unique_ptr<detail::Dev<float>>> xs;
  std::vector<const float*> ptrs;
  for (const auto& v : worker_values) {
    xs.push_back(std::make_unique<detail::Dev<float>>(d));
    detail::cuda(cudaMemcpy(xs.back()->p, v.data(), d * 4, cudaMemcpyHostToDevice));
    ptrs.push_back(xs.back()->p);
  }
  detail::Dev<float> y(d);
  RoundResult r;
  detail::check(dq_sim_round(ctx, ptrs.data(), d, y.p, collect_wire ? DQ_SIM_COLLECT_WIRE : 0, &r.info, nullptr));
  r.synced.resize(d);
  detail::cuda(cudaMemcpy(r.synced.data(), y.p, d * 4, cudaMemcpyDeviceToHost));
  r.vnmse = r.info.vnmse;
  r.mse = r.info.mse;
  r.wire_hash = r.info.wire_hash;
  r.wire.stats_bits = r.info.stats_bits;
  r.wire.payload_bits = r.info.wire_payload_bits;
  r.wire.scale_bits = r.info.scale_bits;
  r.wire.header_bits = r.info.header_bits;
  r.wire.repr_bits = r.info.repr_bits;
  r.wire.compressed_coordinates = r.info.compressed_coordinates;
  r.wire.transmitted_coordinates = r.info.transmitted_coordinates;
  r.allocation.u = r.info.u;
  r.allocation.payload_bits = r.info.payload_bits;
  if (n > 1) {
    const size_t T = (d + 255) / 256;
    r.allocation.widths.resize(T);
    r.allocation.permutation.resize(T);
    detail::check(dq_round_allocation(ctx, r.allocation.widths.data(), r.allocation.permutation.data(), T));
  }
  return r;
}

}  // namespace dynamiq_b200
