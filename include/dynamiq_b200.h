/*
 * dynamiq_b200.h — C-ABI of the B200-native DynamiQ compressed all-reduce.
 *
 * Drop-in boundary for the reference's hot path (run_round and the four codec
 * kernels).  Plain pointers and sizes only: device pointers are CUDA device
 * addresses, streams are cudaStream_t passed as void*.  Every entry point
 * returns a status (DQ_OK = 0) and leaves a thread-local message for
 * dq_last_error().  Status codes mirror the reference's exception types and
 * the CLI's exit codes (proj/tools/dynamiq_cli.cpp:446-458):
 *   DQ_EINVAL      std::invalid_argument         (exit 2)
 *   DQ_EINFEASIBLE dynamiq::InfeasibleBudget     (exit 3)
 *   DQ_EMALFORMED  std::runtime_error("malformed compressed buffer: ...")
 *
 * Device chunk format ("dq tiled SoA"): the super-groups of a
 * chunk in body order (n8 width-8, then n4 width-4, then n2 width-2), packed in
 * tiles of 64 super-groups [payloads | 16 u8 group-scale codes each | bf16
 * super-group scale each].  Bits are identical to the reference record fields
 * (proj/src/codec.cpp:92-124); only the interleaving differs and the 24-byte
 * header is implied by (chunk, n8, n4, n2).  dq_to_reference_wire converts to
 * the reference's serialize_chunk bytes (proj/src/codec.cpp:319-343).
 *
 * Reference interface replaced by each entry point is cited in brackets
 * (paths relative to the reference repository root).
 */
#ifndef DYNAMIQ_B200_H
#define DYNAMIQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DQ_VERSION 1

enum dq_status {
  DQ_OK = 0,
  DQ_EINVAL = 2,
  DQ_EINFEASIBLE = 3,
  DQ_EMALFORMED = 4,
  DQ_ECUDA = 5,
  DQ_ENCCL = 6,
};

enum dq_topology { DQ_RING = 0, DQ_BUTTERFLY = 1 };
enum dq_allocator { DQ_ALLOC_GENERAL = 0, DQ_ALLOC_FAST = 1, DQ_ALLOC_FIXED = 2 };

/* [proj/include/dynamiq/engine.hpp:22-43 PipelineConfig] — same fields and
 * defaults (dq_config_default).  Supported on device by the rounds
 * (dq_sim_round, dq_allreduce): super_group_size 256, group_size 8/16/32/64/128,
 * hierarchical (u8 + bf16) or flat bf16 scales, the quantized codec, the fast,
 * general or fixed allocator, ring or butterfly; non_uniform and correlated may
 * be toggled.  The chunk primitives below use the default format (s = 16,
 * hierarchical). */
typedef struct dq_config {
  uint32_t n_workers;
  uint32_t group_size;
  uint32_t super_group_size;
  double budget_bits;
  int32_t non_uniform;
  int32_t variable_width;
  int32_t hierarchical_scales;
  int32_t correlated;
  int32_t fixed_width;
  int32_t allocator; /* enum dq_allocator */
  int32_t topology;  /* enum dq_topology */
  int32_t codec;     /* 0 quantized (1 = lossless debug codec: not on device) */
  uint64_t seed;     /* SharedSeed.seed */
  uint64_t round;    /* SharedSeed.round */
  uint32_t threads;  /* accepted for API parity; the device ignores it */
} dq_config;

/* [proj/include/dynamiq/codec.hpp:33-40 QuantContext] */
typedef struct dq_qctx {
  uint64_t seed, round;
  uint32_t chunk_index;
  uint32_t hop_slot;
  uint32_t n_slots;
  int32_t correlated;
} dq_qctx;

/* [proj/include/dynamiq/engine.hpp:45-54 RoundResult, metrics.hpp:24-40 WireVolume]
 * (synced goes to the caller's buffer; widths/permutation via dq_round_allocation) */
typedef struct dq_round_info {
  uint64_t wire_hash;   /* only when the round was run with collect_wire = 1 */
  double vnmse, mse;    /* only for dq_sim_round (needs every worker's input) */
  double u;             /* fast-allocator search state (BitAllocation.u) */
  uint64_t payload_bits;
  uint64_t stats_bits, wire_payload_bits, scale_bits, header_bits;
  uint64_t repr_bits, compressed_coordinates, transmitted_coordinates;
  uint32_t n8, n4, n2;  /* width-class counts over all super-groups */
  uint32_t alloc_passes;
  double ms_total;      /* device time of the round (CUDA events) */
} dq_round_info;

typedef struct dq_ctx dq_ctx;

int dq_version(void);
/* Build flags of the loaded library: bit 0 = device-side invariant checks
 * (DQ_CHECK, -DDQ_DEBUG_CHECKS=1), bit 1 = phase timing (-DDQ_SMALL_PHASES=1). */
int dq_build_flags(void);
const char* dq_last_error(void);
void dq_config_default(dq_config* cfg);

/* ---- context: one per GPU; owns scratch sized on demand ------------------ */
int dq_ctx_create(const dq_config* cfg, int device, dq_ctx** out);
int dq_ctx_destroy(dq_ctx* ctx);
int dq_ctx_set_config(dq_ctx* ctx, const dq_config* cfg);

/* ---- codec primitives on device buffers (one chunk) ----------------------
 * Widths are given as run lengths n8, n4, n2, n16 of the width-sorted body
 * (the reference's wire order 8, 4, 2, 16, proj/src/codec.cpp:298-315; width 16
 * is the bf16 passthrough record, codec.cpp:82-86).  Device chunk bytes: */
size_t dq_chunk_bytes(uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16);
/* [codec.cpp:268-291 compressed_size_bits / 8] reference wire bytes incl. the 24-byte
 * header (== dq_chunk_bytes + 24 when n16 == 0; passthrough records carry no scales) */
size_t dq_wire_bytes(uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16);
/* [codec.hpp:26-31 CodecConfig{group_size, hierarchical_scales}] scale format of
 * this thread's chunk primitives (sizes, codec kernels, wire converters) until
 * the next call: group_size 8/16/32/64/128, hierarchical u8 + bf16 or flat bf16
 * group scales (default 16, hierarchical).  prev_* (may be NULL) receive the
 * previous format, so a caller can scope it like cudaSetDevice. */
int dq_codec_format_set(uint32_t group_size, int hierarchical, uint32_t* prev_group_size, int* prev_hierarchical);
/* [codec.hpp:64-69 compress_chunk] values: n_sg*256 fp32 */
int dq_compress_chunk(const float* d_values, uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16,
                      const dq_qctx* q, uint32_t first_sg_index, int non_uniform, void* d_out,
                      void* stream);
/* [codec.hpp:86-91 decompress_accumulate_recompress] */
int dq_dar_chunk(const void* d_in, const float* d_local, uint32_t n8, uint32_t n4, uint32_t n2,
                 uint32_t n16, const dq_qctx* q, uint32_t first_sg_index, int non_uniform, void* d_out,
                 void* stream);
/* [codec.hpp:75-78 decompress_accumulate] acc += decompress(in) */
int dq_da_chunk(const void* d_in, float* d_acc, uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16,
                int non_uniform, void* stream);
/* [codec.hpp:71-73 decompress_chunk] */
int dq_decompress_chunk(const void* d_in, float* d_out, uint32_t n8, uint32_t n4, uint32_t n2,
                        uint32_t n16, int non_uniform, void* stream);
/* [codec.cpp:319-399 serialize_chunk / parse_chunk] host buffers.
 * to: writes dq_wire_bytes bytes.  from: strict parse of reference bytes
 * (DQ_EMALFORMED on any malformed buffer), returns the run lengths. */
int dq_to_reference_wire(const void* h_soa, uint32_t chunk_index, uint32_t n8, uint32_t n4,
                         uint32_t n2, uint32_t n16, void* h_ref);
int dq_from_reference_wire(const void* h_ref, size_t len, void* h_soa, size_t soa_cap,
                           uint32_t* chunk_index, uint32_t* n8, uint32_t* n4, uint32_t* n2,
                           uint32_t* n16);
/* [codec.cpp:319-343 serialize_chunk] device buffers, stream-ordered: d_wire
 * receives dq_wire_bytes bytes (header + records), one warp per record. */
int dq_serialize_chunk(const void* d_soa, uint32_t chunk_index, uint32_t n8, uint32_t n4, uint32_t n2,
                       uint32_t n16, void* d_wire, void* stream);
/* [codec.cpp:345-399 parse_chunk] device buffers: strict parse with the
 * reference's checks and messages (DQ_EMALFORMED).  Reads the header and the
 * validation verdict back, so it synchronizes `stream`.  d_soa may be null
 * (validate only); soa_cap < dq_chunk_bytes -> DQ_EINVAL. */
int dq_parse_chunk(const void* d_wire, size_t len, void* d_soa, size_t soa_cap, uint32_t* chunk_index,
                   uint32_t* n8, uint32_t* n4, uint32_t* n2, uint32_t* n16, void* stream);

/* ---- statistics and allocation ------------------------------------------ */
/* [stats.hpp:19 compute_stats] per super-group fp64-sequential mean / sum of squares */
int dq_compute_stats(const float* d_x, size_t d, float* d_mean, float* d_sq, void* stream);
/* [stats.hpp:23 reduce_stats] d_means/d_sqs: [n_workers][n_sg], rank order */
int dq_reduce_stats(const float* d_means, const float* d_sqs, uint32_t n_workers, size_t n_sg,
                    float* d_gmean, float* d_gsq, void* stream);
/* [allocation.hpp:63-64 allocate_fast + :85 build_permutation].  Synchronizes the
 * stream (the plateau midpoint is finished on the host with the reference's libm). */
int dq_allocate_fast(dq_ctx* ctx, const float* d_sq_norms, size_t n_sg, double budget_bits,
                     uint8_t* d_widths, uint32_t* d_perm, double* u, uint64_t* payload_bits,
                     uint32_t counts[3], void* stream);
/* [allocation.hpp:57 allocate_general], W = {2,4,8} (the width set run_round uses,
 * engine.cpp:306-307): crossing points sorted on the device, the reference's
 * bisection driven from the host (one probe kernel + sync per step).  u = the
 * resolved base threshold.  DQ_EINVAL for negative/NaN norms. */
int dq_allocate_general(dq_ctx* ctx, const float* d_sq_norms, size_t n_sg, double budget_bits,
                        uint8_t* d_widths, uint32_t* d_perm, double* u, uint64_t* payload_bits,
                        uint32_t counts[3], void* stream);
/* [allocation.hpp:75-81 allocate_fast_stateful + FastAllocatorState] state =
 * {lo, hi, u} (defaults {-1e6, 1e6, 0}), updated in place by one bisection step;
 * *u = the carried u this round used. */
int dq_allocate_fast_stateful(dq_ctx* ctx, const float* d_sq_norms, size_t n_sg, double budget_bits,
                              double state[3], uint8_t* d_widths, uint32_t* d_perm, double* u,
                              uint64_t* payload_bits, uint32_t counts[3], void* stream);

/* ---- schedule ------------------------------------------------------------ */
/* [topology.hpp:15-46 ring_schedule / butterfly_schedule, ChunkPlan] the reduce
 * events of chunk `chunk` in execution order (sender, receiver, hop slot, and the
 * stage the multi-GPU executor runs it in: ring = hop index, butterfly = halving
 * stage), the sink's compression slot and the slot count.  Host only (no device). */
typedef struct dq_event {
  uint32_t sender, receiver, slot, stage;
} dq_event;
int dq_schedule(uint32_t n_workers, int topology, uint32_t chunk, dq_event* events, uint32_t cap,
                uint32_t* n_events, uint32_t* sink_slot, uint32_t* n_slots, uint32_t* n_gather);

/* ---- the all-reduce ------------------------------------------------------ */
/* [engine.hpp:63-64 run_round] all cfg.n_workers gradients resident on this
 * GPU (simulated hops, BASELINE config 2).  d_workers: host array of n device
 * pointers.  flags: DQ_SIM_COLLECT_WIRE hashes every message in reference wire
 * format (wire_hash parity; slow, for tests); DQ_SIM_NO_METRICS skips the
 * vNMSE pass against the fp64 sum of the inputs and returns without a host
 * synchronisation (fast allocator: the round allocates on the device; dq_round_wait
 * then fills the allocation and accounting fields). */
enum { DQ_SIM_COLLECT_WIRE = 1, DQ_SIM_NO_METRICS = 2 };
int dq_sim_round(dq_ctx* ctx, const float* const* d_workers, size_t d, float* d_synced,
                 int flags, dq_round_info* info, void* stream);
/* Same with HOST gradients: copies in, runs, copies the sum out (the e2e call). */
int dq_run_round_host(dq_ctx* ctx, const float* const* h_workers, size_t d, float* h_synced,
                      dq_round_info* info, void* stream);
/* After a round: widths (original super-group order) and permutation. */
int dq_round_allocation(dq_ctx* ctx, uint8_t* h_widths, uint32_t* h_perm, size_t n_sg);

/* Per-kernel-family device timing: when enabled, every launch is bracketed by
 * CUDA events on its stream; totals (launch count, ms, algorithmic bytes) are
 * read back per family ("quant_dar", "decode_out", ...). */
typedef struct dq_kernel_profile {
  char name[32];
  uint64_t launches;
  double ms;
  double bytes;
} dq_kernel_profile;
int dq_profile_enable(dq_ctx* ctx, int on);
int dq_profile_read(dq_ctx* ctx, dq_kernel_profile* out, int cap, int* count, int reset);

/* Device self-checks of internal arithmetic (tests only): which = 0 compares
 * the shared-reciprocal division with IEEE div.rn on n hashed pairs; which = 1
 * compares the O(1) codebook bracket with binary search; which = 2 compares the
 * decode's code * sg_scale / 255 fast path with div.rn for every code and every
 * bf16 scale.  *mismatches = count. */
int dq_selftest(int which, uint64_t n, uint64_t seed, uint64_t* mismatches);
/* Test hook: on = 1 makes every asynchronous allocation hand its decision to the
 * host service thread (the path of rounds the device cannot decide); on = 2
 * makes every cooperative search consult the host for its candidates' glibc
 * thresholds (the path of ambiguous float thresholds); 0 = normal. */
int dq_debug_force_host_alloc(int on);
/* Diagnostics.  *finished: rounds of this context whose allocation the host
 * finished (asynchronous rounds the device could not decide, plus the
 * synchronous path's exact walks) - normally 0, each costs a host sort of the
 * flips in the round's critical path.  *consulted (may be NULL): asynchronous
 * rounds that asked the host only for the candidates' glibc thresholds (a float
 * threshold within rounding of an F_j) - a few microseconds of host math and
 * one mapped-memory round trip. */
int dq_ctx_host_allocations(const dq_ctx* ctx, uint64_t* finished, uint64_t* consulted);

/* Multi-GPU: one process per GPU.  Rank 0 creates the id, the caller ships the
 * 128 bytes to every rank (e.g. torch.distributed), every rank joins. */
int dq_comm_unique_id(uint8_t out[128]);
int dq_comm_init(dq_ctx* ctx, int rank, int nranks, const uint8_t id[128]);
/* Transport (ring and butterfly).  PEER (default): the fused hop kernels store
 * compressed units straight into the receiver's memory over NVLink (CUDA IPC
 * mapping of one region per rank, per-unit flags; a flag missing for
 * DQ_WAIT_TIMEOUT_S seconds, default 600, aborts the kernel), and the sink
 * stores into every rank's gather slot.  NCCL: point-to-point sends on a
 * communication stream (ring: tile-aligned pieces; butterfly: per stage).  Same
 * bytes, same result.  Env DQ_TRANSPORT=nccl selects NCCL at context creation;
 * if any rank cannot map its peers, all ranks switch to NCCL at the first
 * round.  The ablation scale formats (group size != 16, flat scales) always use
 * NCCL. */
enum { DQ_TRANSPORT_PEER = 0, DQ_TRANSPORT_NCCL = 1 };
int dq_comm_set_transport(dq_ctx* ctx, int transport);
int dq_comm_get_transport(const dq_ctx* ctx, int* transport);
/* [engine.hpp:63-64 run_round, distributed] d_in: this rank's gradient; d_out:
 * the SUM estimate over ranks (caller divides by n for a mean, as the
 * reference's caller does).  Stream-ordered: with the peer transport and the
 * fast allocator the whole round is enqueued without a host synchronisation
 * (the allocation is decided and certified on the device; the class counts stay
 * on the device) and can be captured in a CUDA graph.  info = NULL returns at
 * once; info != NULL waits for the round and fills the allocation / accounting
 * fields (the reference's RoundResult), as dq_round_wait does later. */
int dq_allreduce(dq_ctx* ctx, const float* d_in, float* d_out, size_t d, dq_round_info* info,
                 void* stream);
/* Wait for the context's last round (dq_allreduce or dq_sim_round) and fill the
 * fields that need its device results: u, payload_bits, n8/n4/n2, the wire
 * accounting and ms_total. */
int dq_round_wait(dq_ctx* ctx, dq_round_info* info);

#ifdef __cplusplus
}
#endif
#endif /* DYNAMIQ_B200_H */
