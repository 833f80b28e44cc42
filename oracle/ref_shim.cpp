// ref_shim.cpp — exports the dq_oracle.h entry points (prefix dqref_) on top of
// the REFERENCE library compiled from /root/reference/proj/src by oracle/Makefile.
//
// TEST INFRASTRUCTURE ONLY.  This file contains no algorithm: it converts plain
// pointers to the reference's std::span / std::vector types, calls the
// reference function named in each comment, and maps its exceptions to return
// codes (std::invalid_argument -> 2, InfeasibleBudget -> 3,
// std::runtime_error("malformed ...") -> 4), mirroring the CLI's exit codes
// (proj/tools/dynamiq_cli.cpp:446-458).
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "dq_oracle.h"
#include "dynamiq/allocation.hpp"
#include "dynamiq/codebook.hpp"
#include "dynamiq/codec.hpp"
#include "dynamiq/engine.hpp"
#include "dynamiq/random.hpp"
#include "dynamiq/topology.hpp"
#include "dynamiq/stats.hpp"
#include "dynamiq/synth.hpp"

using namespace dynamiq;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InfeasibleBudget& e) {
    g_err = e.what();
    return DQO_EINFEASIBLE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return DQO_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DQO_EMALFORMED;
  }
}

RandomKey key(uint32_t purpose, uint64_t chunk, uint64_t sg, uint64_t entry) {
  return RandomKey{static_cast<Purpose>(purpose), chunk, sg, entry};
}
CodecConfig codec(const dqo_codec* c) {
  return CodecConfig{c->group_size, c->super_group_size, c->hierarchical != 0};
}
CodebookSet books(const dqo_codec* c) {
  return c->non_uniform ? CodebookSet::non_uniform_defaults() : CodebookSet::uniform_all();
}
QuantContext qctx(const dqo_qctx* q) {
  return QuantContext{SharedSeed{q->seed, q->round}, q->chunk, q->slot, q->n_slots, q->correlated != 0};
}
int emit(const std::vector<uint8_t>& bytes, uint8_t* out, size_t cap, size_t* out_len) {
  if (bytes.size() > cap) {
    g_err = "output capacity";
    return DQO_EINVAL;
  }
  std::memcpy(out, bytes.data(), bytes.size());
  *out_len = bytes.size();
  return 0;
}
}  // namespace

extern "C" {

const char* dqref_last_error(void) { return g_err.c_str(); }

uint64_t dqref_random_bits(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                           uint64_t sg, uint64_t entry) {
  return random_bits(SharedSeed{seed, round}, key(purpose, chunk, sg, entry));
}
double dqref_uniform_at(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                        uint64_t sg, uint64_t entry) {
  return uniform_at(SharedSeed{seed, round}, key(purpose, chunk, sg, entry));
}
int dqref_permutation_slot(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                           uint64_t sg, uint64_t entry, uint32_t slot, uint32_t n, uint32_t* out) {
  return guarded([&] { *out = permutation_slot(SharedSeed{seed, round}, key(purpose, chunk, sg, entry), slot, n); });
}
int dqref_correlated_uniform(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                             uint64_t sg, uint64_t entry, uint32_t slot, uint32_t n, double* out) {
  return guarded([&] { *out = correlated_uniform(SharedSeed{seed, round}, key(purpose, chunk, sg, entry), slot, n); });
}
int dqref_codebook(int width, int non_uniform, float* out) {
  return guarded([&] {
    Codebook cb = non_uniform ? build_codebook(width, default_epsilon(width)) : uniform_codebook(width);
    std::memcpy(out, cb.values.data(), cb.values.size() * sizeof(float));
  });
}
uint64_t dqref_compressed_size_bits(const uint8_t* widths, size_t nsg, uint32_t S, uint32_t s,
                                    int hierarchical) {
  return compressed_size_bits({widths, nsg}, S, s, hierarchical != 0);
}
int dqref_compress_chunk(const float* values, const uint8_t* widths, size_t nsg, const dqo_codec* cc,
                         const dqo_qctx* q, uint32_t first_sg, uint8_t* out, size_t cap,
                         size_t* out_len) {
  int rc2 = 0;
  int rc = guarded([&] {
    CompressedChunk ch = compress_chunk({values, nsg * cc->super_group_size}, {widths, nsg}, books(cc),
                                        codec(cc), qctx(q), first_sg);
    rc2 = emit(serialize_chunk(ch, codec(cc)), out, cap, out_len);
  });
  return rc ? rc : rc2;
}
int dqref_dar_chunk(const uint8_t* in, size_t in_len, const float* local, size_t n_local,
                    const dqo_codec* cc, const dqo_qctx* q, uint32_t first_sg, uint8_t* out,
                    size_t cap, size_t* out_len) {
  int rc2 = 0;
  int rc = guarded([&] {
    CompressedChunk held = parse_chunk({in, in_len}, codec(cc));
    CompressedChunk ch = decompress_accumulate_recompress(held, {local, n_local}, books(cc), codec(cc),
                                                          qctx(q), first_sg);
    rc2 = emit(serialize_chunk(ch, codec(cc)), out, cap, out_len);
  });
  return rc ? rc : rc2;
}
int dqref_decompress_chunk(const uint8_t* in, size_t in_len, const dqo_codec* cc, float* out,
                           size_t n_out) {
  return guarded([&] {
    CompressedChunk ch = parse_chunk({in, in_len}, codec(cc));
    decompress_chunk(ch, books(cc), codec(cc), {out, n_out});
  });
}
int dqref_decompress_accumulate(const uint8_t* in, size_t in_len, const dqo_codec* cc, float* acc,
                                size_t n_acc) {
  return guarded([&] {
    CompressedChunk ch = parse_chunk({in, in_len}, codec(cc));
    decompress_accumulate(ch, {acc, n_acc}, books(cc), codec(cc));
  });
}
int dqref_compute_stats(const float* x, size_t d, uint32_t s, uint32_t S, float* mean, float* sq) {
  return guarded([&] {
    Gradient g = Gradient::from_values(std::vector<float>(x, x + d), s, S);
    auto st = compute_stats(g);
    for (size_t j = 0; j < st.size(); ++j) {
      mean[j] = st[j].mean;
      sq[j] = st[j].sq_norm;
    }
  });
}
int dqref_reduce_stats(const float* means, const float* sqs, uint32_t n, size_t nsg, float* gm,
                       float* gs) {
  return guarded([&] {
    std::vector<std::vector<SuperGroupStats>> per(n, std::vector<SuperGroupStats>(nsg));
    for (uint32_t r = 0; r < n; ++r)
      for (size_t j = 0; j < nsg; ++j) per[r][j] = {means[r * nsg + j], sqs[r * nsg + j]};
    auto g = reduce_stats(per);
    for (size_t j = 0; j < nsg; ++j) {
      gm[j] = g[j].mean;
      gs[j] = g[j].sq_norm;
    }
  });
}
int dqref_allocate_fast(const float* F, size_t nsg, double b, uint32_t s, uint32_t S, int hier,
                        uint8_t* widths, uint32_t* perm, double* u, uint64_t* payload_bits) {
  return guarded([&] {
    BudgetSpec spec{b, s, S, {2, 4, 8}, hier != 0};
    BitAllocation a = allocate_fast({F, nsg}, spec);
    std::memcpy(widths, a.widths.data(), nsg);
    if (perm) std::memcpy(perm, a.permutation.data(), nsg * sizeof(uint32_t));
    *u = a.u;
    *payload_bits = a.payload_bits;
  });
}
int dqref_allocate_general(const float* F, size_t nsg, double b, uint32_t s, uint32_t S, int hier, const int* W,
                           int n_w, uint8_t* widths, uint32_t* perm, double* u, uint64_t* payload_bits) {
  return guarded([&] {
    BudgetSpec spec{b, s, S, std::vector<int>(W, W + (n_w > 0 ? n_w : 0)), hier != 0};
    BitAllocation a = allocate_general({F, nsg}, spec);
    std::memcpy(widths, a.widths.data(), nsg);
    if (perm) std::memcpy(perm, a.permutation.data(), nsg * sizeof(uint32_t));
    *u = a.u;
    *payload_bits = a.payload_bits;
  });
}
int dqref_allocate_fast_stateful(const float* F, size_t nsg, double b, uint32_t s, uint32_t S, int hier,
                                 double state[3], uint8_t* widths, uint32_t* perm, double* u,
                                 uint64_t* payload_bits) {
  return guarded([&] {
    BudgetSpec spec{b, s, S, {2, 4, 8}, hier != 0};
    FastAllocatorState st{state[0], state[1], state[2]};
    BitAllocation a = allocate_fast_stateful({F, nsg}, spec, st);
    std::memcpy(widths, a.widths.data(), nsg);
    if (perm) std::memcpy(perm, a.permutation.data(), nsg * sizeof(uint32_t));
    *u = a.u;
    *payload_bits = a.payload_bits;
    state[0] = st.lo;
    state[1] = st.hi;
    state[2] = st.u;
  });
}
int dqref_schedule(uint32_t n, int topology, uint32_t chunk, uint32_t* events, uint32_t cap, uint32_t* n_events,
                   uint32_t* sink_slot, uint32_t* n_slots, uint32_t* n_gather) {
  return guarded([&] {
    Schedule s = topology == 0 ? ring_schedule(n) : butterfly_schedule(n);
    if (chunk >= s.chunks.size()) throw std::invalid_argument("chunk out of range");
    const ChunkPlan& p = s.chunks[chunk];
    *n_events = static_cast<uint32_t>(p.reduce_events.size());
    *sink_slot = p.sink_compress_slot;
    *n_slots = p.n_slots;
    *n_gather = static_cast<uint32_t>(p.gather_events.size());
    if (events) {
      if (cap < p.reduce_events.size()) throw std::invalid_argument("event capacity");
      for (size_t e = 0; e < p.reduce_events.size(); ++e) {
        events[3 * e] = p.reduce_events[e].sender;
        events[3 * e + 1] = p.reduce_events[e].receiver;
        events[3 * e + 2] = p.reduce_events[e].hop_slot;
      }
    }
    if (!validate_schedule(s).ok) throw std::runtime_error("reference schedule failed validation");
  });
}
int dqref_build_permutation(const uint8_t* widths, size_t nsg, uint32_t* perm) {
  return guarded([&] {
    auto p = build_permutation({widths, nsg});
    std::memcpy(perm, p.data(), nsg * sizeof(uint32_t));
  });
}
int dqref_run_round(const float* const* workers, size_t d, const dqo_round_cfg* c, float* synced,
                    uint8_t* widths, uint32_t* perm, dqo_round_out* out) {
  return guarded([&] {
    std::vector<std::vector<float>> wv(c->n_workers);
    for (uint32_t r = 0; r < c->n_workers; ++r) wv[r].assign(workers[r], workers[r] + d);
    PipelineConfig p;
    p.n_workers = c->n_workers;
    p.group_size = c->group_size;
    p.super_group_size = c->super_group_size;
    p.budget_bits = c->budget_bits;
    p.non_uniform = c->non_uniform;
    p.variable_width = c->variable_width;
    p.hierarchical_scales = c->hierarchical;
    p.correlated = c->correlated;
    p.fixed_width = c->fixed_width;
    p.allocator = static_cast<AllocatorKind>(c->allocator);
    p.topology = static_cast<TopologyKind>(c->topology);
    p.codec = static_cast<CodecKind>(c->codec);
    p.seed = SharedSeed{c->seed, c->round};
    p.threads = c->threads ? c->threads : 1;
    RoundResult r = run_round(wv, p);
    std::memcpy(synced, r.synced.data(), d * sizeof(float));
    std::memset(out, 0, sizeof *out);
    out->wire_hash = r.wire_hash;
    out->vnmse = r.vnmse;
    out->mse = r.mse;
    out->u = r.allocation.u;
    out->payload_bits = r.allocation.payload_bits;
    out->stats_bits = r.wire.stats_bits;
    out->wire_payload_bits = r.wire.payload_bits;
    out->scale_bits = r.wire.scale_bits;
    out->header_bits = r.wire.header_bits;
    out->repr_bits = r.wire.repr_bits;
    out->compressed_coordinates = r.wire.compressed_coordinates;
    out->transmitted_coordinates = r.wire.transmitted_coordinates;
    if (widths && !r.allocation.widths.empty()) std::memcpy(widths, r.allocation.widths.data(), r.allocation.widths.size());
    if (perm && !r.allocation.permutation.empty())
      std::memcpy(perm, r.allocation.permutation.data(), r.allocation.permutation.size() * sizeof(uint32_t));
  });
}
int dqref_generate_worker(int kind, size_t d, uint64_t seed, double sigma_log, uint32_t S,
                          uint32_t rank, float* out) {
  return guarded([&] {
    GeneratorSpec spec{kind == 0 ? GeneratorKind::kIidGaussian : GeneratorKind::kLocality, d, seed,
                       sigma_log, ""};
    auto v = generate_worker(spec, S, rank);
    std::memcpy(out, v.data(), d * sizeof(float));
  });
}

}  // extern "C"
