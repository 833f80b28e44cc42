// dq_internal.h — kernel launch interface shared by the .cu files and the
// host engine (not part of the public C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "dq_device.cuh"

namespace dq {

// Arguments of every codec kernel (passed by value in the param space).
constexpr int kMaxPeers = 8;  // peer transport: ring of up to 8 GPUs (one NVSwitch domain node)

struct CodecArgs {
  Layout L;                 // geometry of the chunk being processed
  // asynchronous rounds: the round's class counts (n8, n4 over all super-groups) in device
  // memory; the kernel derives L.n8 / L.n4 of [first_sg, first_sg + L.nsg) from them
  const uint32_t* counts;
  uint32_t first_sg;        // permuted index of the chunk's first super-group (RNG key, perm lookup)
  const float* x;           // raw gradient, original order (gather source)
  const uint32_t* perm;     // permuted position -> original super-group
  const float* gmean;       // global super-group means, permuted order (gmean[k] = mean of perm[k])
  uint64_t d;               // logical gradient length (zero padding beyond)
  const float* acc_in;      // chunk-local fp32 operand [nsg * 256]
  float* acc_out;           // chunk-local fp32 result, or the output gradient (decode OUT=1)
  const uint8_t* in;        // incoming compressed chunk
  uint8_t* out;             // outgoing compressed chunk
  float n_workers_f;        // float(n) for denormalize
  uint64_t h3_eq, h3_sc, h3_pm;  // keyed prefixes through the chunk word, per purpose
  uint32_t slot, n_slots;
  int correlated;
  int uniform_books;
  float est_c1, est_c2;     // width-8 codebook index estimator (see bracket())
  // peer transport (k_quant_peer): the chunk is produced/consumed in flag units of
  // `unit` consecutive super-groups; a unit of `in` may be read once in_flags[unit]
  // == epoch, and every finished unit is stored to all n_outs destinations (peer
  // memory over NVLink) before its out_flags[o][unit] is set to epoch.  The round's epoch
  // lives in device memory (*epoch_ptr, advanced by the round's statistics kernel), so a
  // round captured in a CUDA graph gets a fresh epoch on every replay.
  const uint32_t* in_flags;
  uint8_t* outs[kMaxPeers];
  uint32_t* out_flags[kMaxPeers];
  int n_outs;
  uint32_t unit;
  const uint32_t* epoch_ptr;
  // permutation slices (pc_mode 3 / 4, correlated, n <= 8): the chunk's leaf stores slot
  // s's pi of every entry into pin_out[s] (null = none): the rank running hop s (ring,
  // peer transport) or the simulated round's slice buffer; hop s reads a.pin.
  int pc_mode;
  // Layout: u32 per (super-group, lane), 4 bits per entry, entry j of the lane at bit 4j.
  uint32_t* pin_out[kMaxPeers];
  const uint32_t* pin;
  // sink DAR only (launch_quant_dec): also decode the finished record into the output
  // gradient (unpermute + denormalize through perm / gmean / n_workers_f / d), i.e. the
  // gather decode of this chunk fused into the hop that produces it
  float* dec_out;
};

// All chunks of a round decoded into the output gradient in one launch.
struct GatherArgs {
  const uint8_t* in[64];     // compressed chunk c (dq tiled SoA)
  uint32_t lo[65];           // chunk c = permuted super-groups [lo[c], lo[c+1]) (or [lo[c], hi[c]))
  uint32_t hi[64];           // explicit end of chunk c when use_hi (non-adjacent chunk lists)
  int use_hi;
  uint32_t n8[64], n4[64];   // width runs of chunk c
  const uint32_t* counts;    // asynchronous rounds: derive n8 / n4 of chunk c from the round's class counts
  const uint32_t* perm;
  const float* gmean;        // permuted order
  float* out;
  uint64_t d;
  float n_workers_f;
  int uniform_books;
  uint32_t gs = 16, ss = 2, gshift = 1;  // scale format of every chunk (see Layout)
  // peer transport: chunk c's unit k may be decoded once flags[c][k] == *epoch_ptr (null: ready)
  const uint32_t* flags[64];
  uint32_t unit[64];
  const uint32_t* epoch_ptr;
};
// max_ctas > 0 caps the grid (CTAs over all chunks; the kernel walks super-groups grid-strided)
void launch_gather_decode(const GatherArgs& g, uint32_t n_chunks, uint32_t max_nsg, cudaStream_t st,
                          uint32_t max_ctas = 0);

void launch_quant(const CodecArgs& a, int src, bool dar, cudaStream_t st);
// reference wire format on the device (dq_wire.cu): SoA chunk -> header + records, and
// records [0, fit) -> SoA (soa may be null: validate only) with the first malformed
// super-group as min(i << 1 | kind) in *bad (initialised to ~0 by the caller)
void launch_to_wire(const uint8_t* soa, const Layout& L, uint32_t chunk, uint8_t* out, cudaStream_t st);
void launch_from_wire(const uint8_t* in, const Layout& L, uint32_t fit, uint8_t* soa, unsigned long long* bad,
                      cudaStream_t st);
// one hop over peer memory (src 0: raw gradient, 1: acc_in); see CodecArgs peer fields
void launch_quant_peer(const CodecArgs& a, int src, bool dar, cudaStream_t st);
// Sink DAR with the chunk's decode fused in (a.dec_out); peer = k_quant_peer, else the
// simulated round's permutation-cache kernel.  Returns false (nothing launched) when the
// configuration has no fused variant: the caller runs the plain sink + gather decode.
// launch = false: only report whether a fused variant exists.
bool launch_quant_dec(const CodecArgs& a, int src, bool peer, cudaStream_t st, bool launch = true);
// decompress-accumulate of a peer-delivered message (waits per unit) into acc_out
void launch_da_peer(const CodecArgs& a, int src, cudaStream_t st);
uint32_t peer_unit(uint32_t nsg);  // super-groups per flag unit of a chunk (same on every rank)
void launch_da(const CodecArgs& a, int src, cudaStream_t st);
void launch_decode(const CodecArgs& a, int out_mode, cudaStream_t st);
cudaError_t upload_codebooks(const float* books);
cudaError_t set_spin_ns(uint64_t ns);  // g_spin_ns of the current device
// Per-device cached attribute (SM counts, occupancy-derived grid caps): the value for the
// current device, computed once per device by `compute` (every device of a process has
// its own cache slot; a second GPU must not inherit the first one's numbers).
constexpr int kMaxDevices = 64;
template <class F>
inline int per_device(int (&cache)[kMaxDevices], F&& compute) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return compute(dev);
  if (!cache[dev]) cache[dev] = compute(dev);
  return cache[dev];
}
void launch_selftest(int which, uint64_t n, uint64_t seed, unsigned long long* bad, float c1, float c2,
                     float* examples, cudaStream_t st);

// ------------------------------------------------------------ statistics
// per-super-group fp64 sequential sum / sum of squares of `n_workers` gradients
// (pointer array in device memory) -> mean[w * T + j], sq[w * T + j]
// worker gradients by value in the kernel parameters (no pointer table in memory: a round
// enqueued far ahead of the GPU, or captured in a graph, carries its own pointers)
struct WorkerPtrs {
  const float* p[64];
};
WorkerPtrs worker_ptrs(const float* const* host_ptrs, uint32_t n);
void launch_stats(const float* const* xs, uint32_t n_workers, uint64_t d, uint32_t T, float* mean,
                  float* sq, cudaStream_t st);
// Statistics all-gather fused into the statistics kernel (peer transport): row `me` of
// every rank's area (mean[r], sq[r] = peer pointers), completion flags flag[r] (row me
// on rank r) set to the new epoch by the last block, which also stores it to *epoch (the
// round's epoch counter in device memory, read by the round's later kernels); done =
// local block-completion counter.
struct StatsPeerArgs {
  float* mean[kMaxPeers];
  float* sq[kMaxPeers];
  uint32_t* flag[kMaxPeers];
  unsigned int* done;
  uint32_t n;
  uint32_t* epoch;
};
void launch_stats_peer(const float* const* xs, uint64_t d, uint32_t T, const StatsPeerArgs& sp, cudaStream_t st);
// reduction of the fused all-gather's rows after waiting for all n row flags == *epoch
void launch_reduce_stats_peer(const float* mean, const float* sq, const uint32_t* flags, const uint32_t* epoch,
                              uint32_t n, uint32_t T, uint32_t stride, float* gm, float* gs, cudaStream_t st);
// rank-ordered fp64 reduction of [n][T] stats -> global [T]
void launch_reduce_stats(const float* mean, const float* sq, uint32_t n, uint32_t T, float* gmean,
                         float* gsq, cudaStream_t st);

// ------------------------------------------------------------ allocation
// Flips around the chosen plateau: slot 0..3 = f_{L-2}, f_{L-1}, f_L, f_{L+1} in the
// sorted unique flip order (sample L lies between f_{L-1} and f_L).
struct FlipRec {
  uint64_t key;
  uint32_t fbits, type, present, pad_;
};
struct AllocState {
  uint64_t klo, khi;       // key range searched by the current pass (inclusive)
  uint64_t below_w;        // total weight of flips with key < klo
  uint64_t pred_key;       // largest flip key below klo (valid when has_pred)
  uint64_t cross_key;      // key of the crossing flip (status 1)
  uint64_t kmin, kmax;     // smallest / largest flip key
  uint64_t wmax;           // largest cumulative flip weight within budget
  uint32_t npos;           // super-groups with F > 0
  uint32_t has_pred;
  uint32_t status;         // 0 searching, 1 crossing found, 2 all flips fit, 3 no flips
  uint32_t passes;
  uint32_t collect;        // the crossing bin holds <= kAllocBins flips: gather and sort them
  uint32_t ncoll;          // flips gathered by the collect stage
  FlipRec slot[4];
  // candidate samples L-1, L, L+1 (present[c]) with device-libm u / thresholds and the
  // float-threshold payload counts (n8, n4 + n8) the reference's bisection would see
  uint32_t cand_present[3];
  double cand_u[3];
  float cand_t24[3], cand_t48[3];
  unsigned long long cand_n8[3], cand_n48[3];
  // a threshold whose float rounding is not stable can only be one of two adjacent floats
  // a < b; the widths differ between them only for an F_j equal to a: amb[c][0/1] = a for
  // the uncertified t24 / t48 of candidate c (else -1), namb = how many F_j equal one
  float amb[3][2];
  unsigned long long namb;
  uint32_t consulted, pad1_;  // the candidates' exact thresholds came from the host (HostMsg::thr_*)
  int32_t choice;          // chosen candidate (0..2); -1 ambiguous (host walk); -2 infeasible
  // chosen u and thresholds (read by the assignment kernels)
  double u;
  float t24, t48;
  // Asynchronous rounds: every present candidate threshold certified equal to glibc's
  // (its float rounding is stable under a relative perturbation of 2^-40, far above the
  // libm error chain; dq_stats_alloc.cu alloc_candidates).  need_host = !certified or no
  // decision among L-1..L+1: the host finishes (host function on a side stream, F
  // exported to mapped host memory) and the assignment waits for its answer.
  uint32_t certified, need_host, epoch, T;
  double budget, alpha;
  uint32_t S, pad2_;
};
// Mapped (zero-copy) host memory shared by the allocation kernels and the host: the
// search mirrors its final state here, the assignment its class counts; on need_host
// rounds the search exports F and raises `request`, the context's host service thread
// answers through `resolved`.
struct HostMsg {
  AllocState state;           // mirror of the search's final state (written by the kernel)
  const float* hF;            // host view of the exported F (set by the host)
  uint32_t counts[4];         // mirror of n8, n4, n2 (written by k_assign_scan)
  volatile uint32_t request;  // epoch of a round that needs the host (written by the search kernel)
  volatile uint32_t resolved; // epoch of the last host answer
  int32_t host_status;        // 0 ok, 3 infeasible budget, 5 internal error (reported at the next sync)
  double u;                   // host answer: u, t24, t48
  float t24, t48;
  // threshold consult (asynchronous rounds whose candidate thresholds are ambiguous and
  // some F_j equals the lower float): the search mirrors its state, raises thr_request;
  // the service thread answers each present candidate's glibc u and float thresholds
  volatile uint32_t thr_request, thr_resolved;
  double thr_u[3];
  float thr_t24[3], thr_t48[3];
};
constexpr int kAllocBins = 1024;
constexpr int kAllocMaxPasses = 8;
// The rank-ordered statistics reduction (k_reduce_stats / k_reduce_stats_peer) folded into
// the one-CTA allocation of small rounds: rows [n][stride] of per-rank means and squares,
// optional per-row flags (peer exchange, compared with *epoch_ptr), outputs gm / gs (= F).
struct StatsReduce {
  const float* mean = nullptr;
  const float* sq = nullptr;
  const uint32_t* flags = nullptr;
  const uint32_t* epoch_ptr = nullptr;
  uint32_t n = 0, stride = 0;
  float* gm = nullptr;
  float* gs = nullptr;
};
struct AllocWork {           // device scratch owned by the context
  double* level;             // alpha * log2(F_j) per super-group (NaN when F_j <= 0)
  AllocState* state;
  uint64_t* bins;            // [kAllocBins][4]: weight, count, min key, max key
  uint32_t* blockcnt;        // [nblocks][4] class counts (8, 4, 2, -)
  uint32_t* counts;          // [4]: n8, n4, n2, payload_units
  const float* gmean;        // global means, original order (input of the permuted copy)
  float* pmean;              // pmean[k] = gmean[perm[k]]
  HostMsg* hmsg;             // asynchronous rounds: mapped host mailbox (null: synchronous rounds)
  float* hF;                 // asynchronous rounds: mapped host copy of F (need_host rounds only)
  StatsReduce red;           // k_alloc_small: reduce the statistics first (red.mean != null)
};
uint32_t alloc_blocks(uint32_t T);
// Search for the crossing flip and the plateau midpoint u, fully on device: one
// cooperative launch (grid-wide syncs between histogram passes), no host sync.
cudaError_t launch_alloc_search(const float* F, uint32_t T, double alpha, uint64_t wmax, double budget,
                                uint32_t S, AllocWork w, cudaStream_t st);
// test hook: make every asynchronous search hand its decision to the host (need_host)
void set_force_host_alloc(int on);
// asynchronous rounds with T <= 4096: search + assignment in one CTA (false: not applicable)
bool launch_alloc_small(const float* F, uint32_t T, double alpha, double budget, uint32_t S, AllocWork w,
                        uint8_t* widths, uint32_t* perm, cudaStream_t st);
constexpr uint32_t kSmallAllocMaxT = 4096;  // launch_alloc_small applies to T <= this
// chunks of at most this many super-groups run one super-group per warp and peer unit
constexpr uint32_t kSmallChunkSGs = 148u * 8 * 2;
// Slow exact path helpers (rare): neighbour flip of `key` (dir -1: largest key below,
// +1: smallest key above) -> rec; float-threshold counts -> counts[0] = #F>=t48,
// counts[1] = #F>=t24.  Both asynchronous on st.
void launch_flip_neighbor(const double* level, const float* F, uint32_t T, double alpha, uint64_t key, int dir,
                          FlipRec* rec, cudaStream_t st);
void launch_threshold_counts(const float* F, uint32_t T, float t24, float t48, unsigned long long* counts,
                             cudaStream_t st);
// Widths from the float thresholds + stable width-class partition (8,4,2).  With
// `from_state` the thresholds are read from w.state (t24/t48 of the search);
// otherwise the given host values are used.
void launch_alloc_assign(const float* F, uint32_t T, float t24, float t48, bool from_state, AllocWork w,
                         uint8_t* widths, uint32_t* perm, cudaStream_t st);
// general allocator, W = {2,4,8} (see dq_stats_alloc.cu): widths by double thresholds
// g0 = base, g1 = base * 512/17; crossing points -> sorted unique u64 keys (back in
// `keys`, count in *n_unique; trailing ~0 = non-positive F); payload counts at a probe.
void launch_general_assign(const float* F, uint32_t T, double g0, double g1, AllocWork w, uint8_t* widths,
                           uint32_t* perm, cudaStream_t st);
size_t general_temp_bytes(uint32_t T);
cudaError_t launch_general_points(const float* F, uint32_t T, double c1, uint64_t* keys, uint64_t* sorted,
                                  void* temp, size_t temp_bytes, int* n_unique, unsigned long long* invalid,
                                  cudaStream_t st);
void launch_general_counts(const float* F, uint32_t T, const uint64_t* pts, uint32_t M, uint32_t idx, double c1,
                           unsigned long long* counts, double* base_out, cudaStream_t st);
void launch_fixed_assign(uint32_t T, int width, AllocWork w, uint8_t* widths, uint32_t* perm,
                         cudaStream_t st);

// vNMSE accumulators (simulation only): err += (y - sum_r x_r)^2, ref += (sum_r x_r)^2
void launch_vnmse(const float* const* xs, uint32_t n, const float* y, uint64_t d, double* acc2,
                  cudaStream_t st);

}  // namespace dq
