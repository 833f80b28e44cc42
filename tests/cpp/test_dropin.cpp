// test_dropin.cpp — the reference's own test style (proj/tests/test_codec.cpp,
// test_engine.cpp) run against the B200 drop-in header include/dynamiq_b200.hpp.
// Inputs and expected values come from the CPU oracle (oracle/dq_oracle.h, the
// checker only).  Built and run by tests/test_gpu_cpp.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "../../include/dynamiq_b200.hpp"
#include "../../oracle/dq_oracle.h"

namespace {
int g_fail = 0, g_checks = 0;
std::vector<std::pair<const char*, std::function<void()>>>& registry() {
  static std::vector<std::pair<const char*, std::function<void()>>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, f}); }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name) \
  static void CAT(t_, __LINE__)(); \
  static Reg CAT(r_, __LINE__)(name, CAT(t_, __LINE__)); \
  static void CAT(t_, __LINE__)()
#define CHECK(x)                                                            \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(x)) {                                                             \
      ++g_fail;                                                             \
      std::printf("  CHECK failed: %s (%s:%d)\n", #x, __FILE__, __LINE__); \
    }                                                                       \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                 \
  do {                                           \
    bool thrown_ = false;                        \
    try {                                        \
      expr;                                      \
    } catch (const T&) {                         \
      thrown_ = true;                            \
    } catch (...) {                              \
    }                                            \
    CHECK(thrown_ && #T);                        \
  } while (0)

using namespace dynamiq_b200;

std::vector<float> normal_vector(uint64_t seed, size_t count, double scale) {
  std::vector<float> v(count);
  dqo_generate_worker(0, count, seed, 0.0, 256, 0, v.data());
  for (auto& x : v) x = static_cast<float>(x * scale);
  return v;
}
const CodecConfig kDefault{16, 256, true};
QuantContext ctx(uint64_t seed, uint32_t slot = 0, uint32_t n_slots = 1, bool correlated = true, uint32_t chunk = 0) {
  return QuantContext{SharedSeed{seed, 0}, chunk, slot, n_slots, correlated};
}
std::vector<uint8_t> oracle_compress(const std::vector<float>& v, const std::vector<uint8_t>& w, const QuantContext& q,
                                     uint32_t first) {
  dqo_codec cc{16, 256, 1, 1};
  dqo_qctx oq{q.seed.seed, q.seed.round, q.chunk_index, q.hop_slot, q.n_slots, q.correlated};
  std::vector<uint8_t> out(dqo_compressed_size_bits(w.data(), w.size(), 256, 16, 1) / 8);
  size_t len = 0;
  dqo_compress_chunk(v.data(), w.data(), w.size(), &cc, &oq, first, out.data(), out.size(), &len);
  out.resize(len);
  return out;
}
}  // namespace

TEST_CASE("all-zero super-group encodes and decodes to zeros") {
  std::vector<float> zeros(256, 0.0f);
  std::vector<uint8_t> w = {4};
  auto c = compress_chunk(zeros, w, CodebookSet::non_uniform_defaults(), kDefault, ctx(1), 0);
  for (size_t i = 24; i < c.wire.size(); ++i) CHECK(c.wire[i] == 0);
  std::vector<float> out(256, 1.0f);
  decompress_chunk(c, CodebookSet::non_uniform_defaults(), kDefault, out);
  for (float v : out) CHECK(v == 0.0f);
}

TEST_CASE("compress_chunk is byte-identical to the reference codec") {
  std::vector<uint8_t> w = {8, 8, 4, 4, 4, 2, 2, 2, 2};
  for (uint64_t trial = 0; trial < 20; ++trial) {
    auto v = normal_vector(100 + trial, w.size() * 256, 3.0 + trial);
    auto q = ctx(trial, trial % 4, 4, true, 1);
    auto got = compress_chunk(v, w, CodebookSet::non_uniform_defaults(), kDefault, q, 7);
    CHECK(got.wire == oracle_compress(v, w, q, 7));
  }
}

TEST_CASE("fused recompression is byte-identical to the unfused pipeline") {
  auto books = CodebookSet::non_uniform_defaults();
  std::vector<uint8_t> widths = {8, 4, 4, 2};
  for (uint64_t trial = 0; trial < 100; ++trial) {
    const size_t coords = widths.size() * 256;
    auto base = normal_vector(500 + trial, coords, 3.0);
    auto local = normal_vector(600 + trial, coords, 1.0);
    auto in_chunk = compress_chunk(base, widths, books, kDefault, ctx(trial, 0, 4), 0);
    auto hop = ctx(trial, 1, 4);
    auto fused = decompress_accumulate_recompress(in_chunk, local, books, kDefault, hop, 0);
    std::vector<float> decoded(coords);
    decompress_chunk(in_chunk, books, kDefault, decoded);
    for (size_t i = 0; i < coords; ++i) decoded[i] += local[i];
    auto unfused = compress_chunk(decoded, widths, books, kDefault, hop, 0);
    CHECK(serialize_chunk(fused, kDefault) == serialize_chunk(unfused, kDefault));
  }
}

TEST_CASE("decompress-accumulate equals decompress then add") {
  auto books = CodebookSet::non_uniform_defaults();
  std::vector<uint8_t> widths = {8, 4, 2};
  auto values = normal_vector(5, 3 * 256, 2.0);
  auto chunk = compress_chunk(values, widths, books, kDefault, ctx(5), 0);
  std::vector<float> acc(values.size()), acc2(values.size(), 0.0f);
  decompress_chunk(chunk, books, kDefault, acc);
  decompress_accumulate(chunk, acc2, books, kDefault);
  for (size_t i = 0; i < acc.size(); ++i) CHECK(acc2[i] == acc[i]);
}

TEST_CASE("serialization round trip and malformed buffers") {
  auto books = CodebookSet::non_uniform_defaults();
  std::vector<uint8_t> widths = {8, 8, 4, 2, 2};
  auto values = normal_vector(7, widths.size() * 256, 4.0);
  auto chunk = compress_chunk(values, widths, books, kDefault, ctx(7, 0, 2, true, 3), 0);
  auto bytes = serialize_chunk(chunk, kDefault);
  CHECK(bytes.size() * 8 == compressed_size_bits(widths, 256, 16, true));
  auto parsed = parse_chunk(bytes, kDefault);
  CHECK(parsed.chunk_index == 3);
  CHECK(parsed.widths == chunk.widths);
  auto t = bytes;
  t.push_back(0);
  CHECK_THROWS_AS(parse_chunk(t, kDefault), std::runtime_error);
  t = bytes;
  t[8] += 1;
  CHECK_THROWS_AS(parse_chunk(t, kDefault), std::runtime_error);
  std::vector<uint8_t> bad_w = {4, 8};
  CHECK_THROWS_AS(compress_chunk(normal_vector(1, 512, 1.0), bad_w, books, kDefault, ctx(1), 0), std::invalid_argument);
}

TEST_CASE("run_round pins the reference's wire_hash (SURVEY Appendix A)") {
  const size_t d = 1u << 20;
  std::vector<std::vector<float>> ws(4, std::vector<float>(d));
  for (uint32_t r = 0; r < 4; ++r) dqo_generate_worker(1, d, 1, 4.0, 256, r, ws[r].data());
  PipelineConfig cfg;
  cfg.n_workers = 4;
  cfg.budget_bits = 4.0;
  auto res = run_round(ws, cfg);
  CHECK(res.wire_hash == 0x4a094af6775201daULL);
  cfg.budget_bits = 5.0;
  CHECK(run_round(ws, cfg).wire_hash == 0xae9e4b918ba61cfaULL);
  // identical to the oracle's synced gradient
  std::vector<const float*> ptrs;
  for (auto& w : ws) ptrs.push_back(w.data());
  dqo_round_cfg oc{4, 16, 256, 4.0, 1, 1, 1, 1, 4, 1, 0, 0, 1, 0, 1};
  std::vector<float> synced(d);
  dqo_round_out oo;
  dqo_run_round(ptrs.data(), d, &oc, synced.data(), nullptr, nullptr, &oo);
  CHECK(res.synced == synced);
  CHECK(res.allocation.u == oo.u);
  // RoundResult.wire (engine.hpp:45-54, metrics.hpp:20-40) like the reference's accounting
  CHECK(res.wire.payload_bits == oo.wire_payload_bits);
  CHECK(res.wire.scale_bits == oo.scale_bits);
  CHECK(res.wire.stats_bits == oo.stats_bits);
  CHECK(res.wire.header_bits == oo.header_bits);
  CHECK(res.wire.repr_bits == oo.repr_bits);
  CHECK(res.wire.total_bits() == oo.stats_bits + oo.wire_payload_bits + oo.scale_bits + oo.header_bits);
  CHECK(res.wire.bits_per_coordinate() ==
        static_cast<double>(oo.repr_bits) / static_cast<double>(oo.compressed_coordinates));
  CHECK(bits_per_coordinate(res.wire) == res.wire.bits_per_coordinate());
}

TEST_CASE("single worker is an exact no-op; b=2 is infeasible") {
  auto w = normal_vector(5, 4096, 1.0);
  PipelineConfig cfg;
  cfg.n_workers = 1;
  CHECK(run_round({w}, cfg).synced == w);
  cfg.n_workers = 2;
  cfg.budget_bits = 2.0;
  CHECK_THROWS_AS(run_round({w, w}, cfg), InfeasibleBudget);
}

TEST_CASE("allocate_general and allocate_fast_stateful match the oracle") {
  auto g = normal_vector(21, 6000, 1.0);
  std::vector<float> F(g.size());
  for (size_t j = 0; j < g.size(); ++j) F[j] = static_cast<float>(std::exp(4.0 * g[j]));
  const int W[3] = {2, 4, 8};
  for (double b : {3.0, 4.0, 6.0}) {
    BudgetSpec spec;
    spec.total_bits_per_coordinate = b;
    BitAllocation a = allocate_general(F, spec);
    std::vector<uint8_t> w(F.size());
    std::vector<uint32_t> p(F.size());
    double u = 0;
    uint64_t pay = 0;
    CHECK(dqo_allocate_general(F.data(), F.size(), b, 16, 256, 1, W, 3, w.data(), p.data(), &u, &pay) == 0);
    CHECK(a.widths == w);
    CHECK(a.permutation == p);
    CHECK(a.u == u);
    CHECK(a.payload_bits == pay);
    FastAllocatorState st;
    double ost[3] = {-1e6, 1e6, 0.0};
    for (int round = 0; round < 6; ++round) {
      BitAllocation s = allocate_fast_stateful(F, spec, st);
      CHECK(dqo_allocate_fast_stateful(F.data(), F.size(), b, 16, 256, 1, ost, w.data(), p.data(), &u, &pay) == 0);
      CHECK(s.widths == w);
      CHECK(s.u == u);
      CHECK(s.payload_bits == pay);
      CHECK(st.lo == ost[0] && st.hi == ost[1] && st.u == ost[2]);
    }
  }
  BudgetSpec bad;
  bad.widths = {2, 4, 8, 16};
  CHECK_THROWS_AS(allocate_general(F, bad), std::invalid_argument);
}

int main() {
  for (auto& [name, fn] : registry()) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "ok" : "FAIL", name);
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
