/*
 * dq_oracle.h — C interface of the CPU ORACLE for the DynamiQ all-reduce hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2602_08923_b200/)
 * may include, link or call this.  Two libraries implement the interface:
 *
 *   oracle/build/libdqoracle.so  (prefix dqo_)  — plain-C restatement of the
 *        reference algorithm, written from the reference sources (proj/src)
 *        (file:line cited per function in dq_oracle.c);
 *   oracle/_ref/libdqref.so      (prefix dqref_) — the reference library itself,
 *        compiled from /root/reference/proj/src by oracle/Makefile, behind a
 *        thin shim (oracle/ref_shim.cpp) exporting the same entry points.
 *
 * tests/test_oracle.py pins dqo_ against dqref_ and against the golden vectors
 * in tests/golden/ (generated from dqref_ by tests/golden/make_golden.py).
 *
 * Conventions: every "chunk" buffer is the REFERENCE wire format
 * (proj/src/codec.cpp:268-343): 24-byte header {chunk, count, n8, n4, n2, n16}
 * (u32 LE) followed by per-super-group records in body order.
 * Return codes: 0 ok, 2 invalid argument, 3 infeasible budget, 4 malformed.
 */
#ifndef DQ_ORACLE_H
#define DQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { DQO_OK = 0, DQO_EINVAL = 2, DQO_EINFEASIBLE = 3, DQO_EMALFORMED = 4 };

/* purpose tags, proj/include/dynamiq/random.hpp:17-24 */
enum { DQO_ENTRY_QUANT = 1, DQO_SCALE_QUANT = 2, DQO_PERMUTATION = 3, DQO_SHUFFLE = 4,
       DQO_GEN_ENTRY = 5, DQO_GEN_SCALE = 6 };

typedef struct {
  uint64_t seed, round;   /* SharedSeed */
  uint32_t chunk;         /* QuantContext.chunk_index */
  uint32_t slot;          /* QuantContext.hop_slot */
  uint32_t n_slots;       /* QuantContext.n_slots */
  int32_t correlated;     /* QuantContext.correlated */
} dqo_qctx;

typedef struct {
  uint32_t group_size;       /* s */
  uint32_t super_group_size; /* S */
  int32_t hierarchical;      /* hierarchical (u8 + bf16) vs flat bf16 scales */
  int32_t non_uniform;       /* default non-uniform codebooks vs uniform */
} dqo_codec;

/* PipelineConfig, proj/include/dynamiq/engine.hpp:22-43 */
typedef struct {
  uint32_t n_workers, group_size, super_group_size;
  double budget_bits;
  int32_t non_uniform, variable_width, hierarchical, correlated, fixed_width;
  int32_t allocator; /* 0 general, 1 fast, 2 fixed */
  int32_t topology;  /* 0 ring, 1 butterfly */
  int32_t codec;     /* 0 quantized, 1 lossless */
  uint64_t seed, round;
  uint32_t threads;
} dqo_round_cfg;

typedef struct {
  uint64_t wire_hash;
  double vnmse, mse, u;
  uint64_t payload_bits;
  uint64_t stats_bits, wire_payload_bits, scale_bits, header_bits;
  uint64_t repr_bits, compressed_coordinates, transmitted_coordinates;
} dqo_round_out;

#define DQO_DECL(P)                                                                         \
  uint64_t P##random_bits(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,  \
                          uint64_t sg, uint64_t entry);                                     \
  double P##uniform_at(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,     \
                       uint64_t sg, uint64_t entry);                                        \
  int P##permutation_slot(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,  \
                          uint64_t sg, uint64_t entry, uint32_t slot, uint32_t n,           \
                          uint32_t* out);                                                   \
  int P##correlated_uniform(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,\
                            uint64_t sg, uint64_t entry, uint32_t slot, uint32_t n,         \
                            double* out);                                                   \
  int P##codebook(int width, int non_uniform, float* out);                                  \
  uint64_t P##compressed_size_bits(const uint8_t* widths, size_t nsg, uint32_t S,           \
                                   uint32_t s, int hierarchical);                           \
  int P##compress_chunk(const float* values, const uint8_t* widths, size_t nsg,             \
                        const dqo_codec* cc, const dqo_qctx* q, uint32_t first_sg,          \
                        uint8_t* out, size_t cap, size_t* out_len);                         \
  int P##dar_chunk(const uint8_t* in, size_t in_len, const float* local, size_t n_local,    \
                   const dqo_codec* cc, const dqo_qctx* q, uint32_t first_sg, uint8_t* out, \
                   size_t cap, size_t* out_len);                                            \
  int P##decompress_chunk(const uint8_t* in, size_t in_len, const dqo_codec* cc, float* out,\
                          size_t n_out);                                                    \
  int P##decompress_accumulate(const uint8_t* in, size_t in_len, const dqo_codec* cc,       \
                               float* acc, size_t n_acc);                                   \
  int P##compute_stats(const float* x, size_t d, uint32_t s, uint32_t S, float* mean,       \
                       float* sq);                                                          \
  int P##reduce_stats(const float* means, const float* sqs, uint32_t n_workers, size_t nsg, \
                      float* gmean, float* gsq);                                            \
  int P##allocate_fast(const float* sq_norms, size_t nsg, double budget_bits, uint32_t s,   \
                       uint32_t S, int hierarchical, uint8_t* widths, uint32_t* perm,       \
                       double* u, uint64_t* payload_bits);                                  \
  int P##allocate_general(const float* sq_norms, size_t nsg, double budget_bits, uint32_t s,\
                          uint32_t S, int hierarchical, const int* W, int n_w,              \
                          uint8_t* widths, uint32_t* perm, double* u, uint64_t* payload_bits);\
  int P##allocate_fast_stateful(const float* sq_norms, size_t nsg, double budget_bits,      \
                                uint32_t s, uint32_t S, int hierarchical, double state[3],  \
                                uint8_t* widths, uint32_t* perm, double* u,                 \
                                uint64_t* payload_bits);                                    \
  int P##build_permutation(const uint8_t* widths, size_t nsg, uint32_t* perm);              \
  int P##schedule(uint32_t n, int topology, uint32_t chunk, uint32_t* events, uint32_t cap,  \
                  uint32_t* n_events, uint32_t* sink_slot, uint32_t* n_slots,                \
                  uint32_t* n_gather);                                                       \
  int P##run_round(const float* const* workers, size_t d, const dqo_round_cfg* cfg,         \
                   float* synced, uint8_t* widths, uint32_t* perm, dqo_round_out* out);     \
  int P##generate_worker(int kind, size_t d, uint64_t seed, double sigma_log, uint32_t S,   \
                         uint32_t rank, float* out);                                        \
  const char* P##last_error(void);

DQO_DECL(dqo_)
DQO_DECL(dqref_)

#ifdef __cplusplus
}
#endif
#endif /* DQ_ORACLE_H */
