// dq_engine.cpp — host runtime of the DynamiQ B200 all-reduce and its C-ABI.
//
// Mirrors the reference's round orchestration (proj/src/engine.cpp:94-418):
// stats -> exact stats reduction -> fast allocation -> width-sorted chunks ->
// per-chunk reduce events (leaf compress / fused DAR / DA, last-parent rule) ->
// sink compression -> all-gather -> decode with unpermute + denormalize.  All
// data stays on the device; every kernel is stream-ordered on the caller's
// stream.  Two executors share the plan: dq_sim_round runs every worker of a
// chunk on one GPU (BASELINE config 2), dq_allreduce runs one rank per GPU and
// moves the compressed chunks over NVLink with NCCL point-to-point.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/dynamiq_b200.h"
#include "dq_internal.h"

namespace dq {
namespace {

thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define DQ_CUDA(x)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw Error(DQ_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));           \
  } while (0)
#define DQ_NCCL(x)                                                                      \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess) throw Error(DQ_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)
[[noreturn]] void invalid(const std::string& m) { throw Error(DQ_EINVAL, m); }

template <class F>
int guarded(F&& f) {
  try {
    f();
    return DQ_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DQ_EINVAL;
  }
}

// ------------------------------------------------------------ codebooks
// f(eps, r) in double, stored as float, strictly increasing (proj/src/codebook.cpp:20-60);
// default eps 0.05 / 0.25 / 0.05 for widths 2 / 4 / 8 (codebook.cpp:63-75).
void fill_book(float* q, int width, bool uniform) {
  const int count = 1 << (width - 1), top = count - 1;
  if (uniform) {
    for (int r = 0; r < count; ++r) q[r] = static_cast<float>(static_cast<double>(r) / top);
    return;
  }
  const double eps = width == 4 ? 0.25 : 0.05;
  const double base = 1.0 + 2.0 * eps * eps;
  for (int r = 0; r < count; ++r)
    q[r] = static_cast<float>(r == 0 ? 0.0 : r == top ? 1.0 : (std::pow(base, r) - 1.0) / (std::pow(base, top) - 1.0));
  for (int r = 1; r < count; ++r)
    if (q[r] <= q[r - 1]) q[r] = std::nextafter(q[r - 1], 2.0f);
}

// The codebooks (__constant__ c_books) and the derived tables (__device__ g_qt, built by
// k_init_tables) exist once per device: upload and build them on the first use of each
// device of the process (the current device of the calling thread).
std::mutex g_books_mu;
int g_books_state[kMaxDevices] = {};  // 0 not yet, 1 ready, 2 failed
void ensure_books() {
  int dev = 0;
  DQ_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) throw Error(DQ_ECUDA, "device index out of range");
  std::lock_guard<std::mutex> lk(g_books_mu);
  if (g_books_state[dev] == 0) {
    float books[2][138];
    for (int u = 0; u < 2; ++u) {
      fill_book(books[u], 2, u);
      fill_book(books[u] + 2, 4, u);
      fill_book(books[u] + 10, 8, u);
    }
    g_books_state[dev] = upload_codebooks(&books[0][0]) == cudaSuccess ? 1 : 2;
    // spin-wait budget of the peer / host waits (DQ_WAIT_TIMEOUT_S seconds, default 600)
    double secs = 600.0;
    if (const char* t = std::getenv("DQ_WAIT_TIMEOUT_S")) secs = std::atof(t) > 0 ? std::atof(t) : secs;
    if (g_books_state[dev] == 1 && set_spin_ns(static_cast<uint64_t>(secs * 1e9)) != cudaSuccess) g_books_state[dev] = 2;
  }
  if (g_books_state[dev] != 1) throw Error(DQ_ECUDA, "codebook upload failed on device " + std::to_string(dev));
}

// alpha = 4 / log2(512/17)  (allocation.cpp:34-35)
const double kAlpha = 4.0 / std::log2(512.0 / 17.0);

double key_to_double(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void reserve(size_t want) {
    if (want <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    DQ_CUDA(cudaMalloc(&p, sizeof(T) * (want ? want : 1)));
    n = want;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct Event {
  uint32_t snd, rcv, slot;
};
struct Plan {  // proj/src/topology.cpp:8-70
  uint32_t sink, sink_slot, n_slots, n_gat;
  std::vector<Event> red;
};
Plan make_plan(uint32_t n, uint32_t c, int topology) {
  Plan p;
  p.sink = c;
  p.n_gat = n - 1;
  if (topology == DQ_RING) {
    for (uint32_t h = 0; h + 1 < n; ++h) p.red.push_back({(c + 1 + h) % n, (c + 2 + h) % n, h});
  } else {
    int stages = 0;
    while ((1u << stages) < n) ++stages;
    uint32_t slot = 0;
    for (int l = 0; l < stages; ++l) {
      const uint32_t bit = 1u << (stages - 1 - l), high = ~(2 * bit - 1);
      for (uint32_t w = 0; w < n; ++w) {
        if ((w & high) != (c & high) || (w & bit) == (c & bit)) continue;
        p.red.push_back({w, w ^ bit, slot++});
      }
    }
  }
  p.sink_slot = static_cast<uint32_t>(p.red.size());
  p.n_slots = p.sink_slot + 1;
  return p;
}

uint64_t fnv1a(const uint8_t* b, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
  return h;
}

}  // namespace
}  // namespace dq

using namespace dq;

// Peer transport region of one rank (cudaMalloc'd, exported by CUDA IPC, mapped by
// every other rank of the node): `ninbox` inboxes (ring: hop h's output lands in the right
// neighbour's inbox h; butterfly: stage s's message for chunk c in the receiver's inbox
// s * n + c) and n gather slots (the sink of chunk c stores its bytes into every rank's slot
// c), then one u32 flag per unit of each, then the ring's permutation slices.  Single-
// buffered: a rank's round k+1 writes into a peer only after its own round k completed,
// which needed every rank's round-k sink output, hence every peer's round-k reads of its
// region; flags carry the round's epoch (device memory, advanced once per round).
struct PeerMem {
  uint8_t* base = nullptr;
  std::vector<uint8_t*> peer;  // rank q's region as mapped here (peer[me] == base)
  size_t cap = 0;              // bytes per chunk slot
  size_t cap_units = 0;        // flags per chunk slot
  uint32_t n = 0, ninbox = 0, npin = 0;
  size_t slots() const { return static_cast<size_t>(ninbox) + n; }
  size_t inbox(uint32_t h) const { return static_cast<size_t>(h) * cap; }
  size_t gather(uint32_t c) const { return (static_cast<size_t>(ninbox) + c) * cap; }
  size_t flags() const { return slots() * cap; }
  size_t iflag(uint32_t h) const { return flags() + 4 * cap_units * h; }
  size_t gflag(uint32_t c) const { return flags() + 4 * cap_units * (static_cast<size_t>(ninbox) + c); }
  // ring permutation slices: npin areas of one u32 per (super-group, lane)
  size_t pins() const { return (flags() + 4 * cap_units * slots() + 255) & ~static_cast<size_t>(255); }
  size_t pin(uint32_t k) const { return pins() + static_cast<size_t>(k) * 128 * cap_units; }
  size_t total() const { return pins() + static_cast<size_t>(npin) * 128 * cap_units; }
};

// Statistics exchange area of one rank (peer transport): the [n][T] mean and sum-of-squares
// rows every rank stores its row into, then n row flags (single-buffered, as PeerMem).
struct StatsMem {
  uint8_t* base = nullptr;
  std::vector<uint8_t*> peer;
  uint32_t n = 0, T = 0;  // T: row capacity (grow-only, headroom): rounds of any T <= it reuse the area
  size_t rows() const { return 4ull * n * T; }  // bytes of one [n][T] float array
  float* mean(uint8_t* b, uint32_t r) const { return reinterpret_cast<float*>(b) + static_cast<size_t>(r) * T; }
  float* sq(uint8_t* b, uint32_t r) const { return reinterpret_cast<float*>(b + rows()) + static_cast<size_t>(r) * T; }
  uint32_t* flags(uint8_t* b) const { return reinterpret_cast<uint32_t*>(b + 2 * rows()); }
  size_t total() const { return 2 * rows() + static_cast<size_t>(n) * sizeof(uint32_t); }
};

struct dq_ctx {
  dq_config cfg{};
  int device = 0;
  // round scratch
  DevBuf<float> mean_all, sq_all, gmean, gsq, pmean;
  DevBuf<uint8_t> widths;
  DevBuf<uint32_t> perm;
  DevBuf<double> level;
  DevBuf<AllocState> astate;
  DevBuf<uint64_t> bins;
  DevBuf<uint32_t> blockcnt, counts;
  DevBuf<FlipRec> nrec;                 // slow allocation path scratch
  DevBuf<unsigned long long> tcount;
  DevBuf<uint64_t> gkeys, gsorted;       // general allocator: crossing points
  DevBuf<uint8_t> gtemp;                 // CUB scratch
  DevBuf<int> gnum;
  DevBuf<double> gbase;
  DevBuf<double> vn;
  DevBuf<uint8_t> msgs;   // message pool
  DevBuf<float> accs;     // per-worker chunk accumulators (butterfly)
  DevBuf<uint32_t> pcache; // simulated round: the chunk's permutation slices (slots 1..n-1)
  DevBuf<float> stage;    // host-round staging of inputs / output
  std::vector<cudaStream_t> cstreams;  // simulated rounds: concurrent chunk chains
  std::vector<cudaEvent_t> cjoin;
  cudaEvent_t cfork = nullptr;
  dq_round_info last_info{};  // the last round's host-known info (dq_round_wait)
  AllocState* h_state = nullptr;
  uint32_t* h_counts = nullptr;
  // asynchronous allocation (no host sync inside a round): per round parity a mapped
  // mailbox the search mirrors its state into, a mapped copy of F for the rare rounds the
  // host must finish, and the service thread that does so
  HostMsg* hmsg = nullptr;   // [2]
  float* hF = nullptr;
  size_t hF_cap = 0;
  std::thread svc;           // answers need_host requests (polls the mailboxes; idle otherwise)
  std::atomic<bool> svc_stop{false};
  uint32_t apar = 0;
  bool async_alloc = true;   // env DQ_SYNC_ALLOC=1: host-synchronous allocation (round-1 behaviour)
  bool no_small_alloc = false;  // env DQ_NO_SMALL_ALLOC=1: the cooperative search at every T
  StatsReduce pending_red;      // small rounds: the statistics reduction handed to k_alloc_small
  // what the last round needs to fill dq_round_info once it has completed
  struct RoundRec {
    bool valid = false, async = false;
    uint32_t par = 0, T = 0, n = 0, S = 256, gs = 16, ss = 2, gshift = 1;
    int topology = 0;
    std::vector<uint32_t> lo;
  } rec;
  double* h_vn = nullptr;
  uint32_t last_T = 0;
  std::atomic<uint64_t> host_allocs{0};    // asynchronous rounds finished by alloc_service
  std::atomic<uint64_t> host_consults{0};  // threshold consults answered by alloc_service
  uint64_t alloc_redos = 0;  // rounds where the device thresholds differed from glibc's
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // round-boundary events of the last asynchronously finished round (measured at the next sync)
  cudaEvent_t lr0 = nullptr, lr1 = nullptr;
  bool lr_pending = false;
  double last_round_ms = 0.0;
  // per-kernel-family device timing (CUDA events bracketing each launch)
  struct Prof {
    int kind;
    double bytes;
    cudaEvent_t a, b;
  };
  int profile = 0;
  std::vector<Prof> pending;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[16] = {}, prof_bytes[16] = {};
  uint64_t prof_launches[16] = {};
  // distributed
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  cudaStream_t cs = nullptr;            // communication stream (NCCL p2p)
  std::vector<cudaEvent_t> pipe_ev;     // per (hop, piece) handshakes compute <-> comm
  int pieces = 4;                       // pipeline pieces per chunk
  int transport = DQ_TRANSPORT_PEER;    // ring transport (butterfly always uses NCCL)
  PeerMem pm;
  StatsMem sm;
  DevBuf<unsigned int> sdone;           // fused stats all-gather: block completion counter
  DevBuf<uint32_t> dev_epoch;           // peer transport: the round's epoch (advanced on the device)
  DevBuf<uint8_t> ipc;                  // IPC handle exchange
  static void close_map(std::vector<uint8_t*>& peer, const uint8_t* base) {
    for (size_t q = 0; q < peer.size(); ++q)
      if (peer[q] && peer[q] != base) cudaIpcCloseMemHandle(peer[q]);
    peer.clear();
  }
  void close_peers() { close_map(pm.peer, pm.base); }
  ~dq_ctx() {
    close_peers();
    close_map(sm.peer, sm.base);
    if (pm.base) cudaFree(pm.base);
    if (sm.base) cudaFree(sm.base);
    if (h_state) cudaFreeHost(h_state);
    for (cudaStream_t s2 : cstreams) cudaStreamDestroy(s2);
    for (cudaEvent_t e2 : cjoin) cudaEventDestroy(e2);
    if (cfork) cudaEventDestroy(cfork);
    if (svc.joinable()) {
      svc_stop = true;
      svc.join();
    }
    if (hmsg) cudaFreeHost(hmsg);
    if (hF) cudaFreeHost(hF);
    if (h_counts) cudaFreeHost(h_counts);
    if (h_vn) cudaFreeHost(h_vn);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (lr0) cudaEventDestroy(lr0);
    if (lr1) cudaEventDestroy(lr1);
    if (comm) ncclCommDestroy(comm);
    if (cs) cudaStreamDestroy(cs);
    for (cudaEvent_t e : pipe_ev) cudaEventDestroy(e);
    for (auto& p : pending) {
      cudaEventDestroy(p.a);
      cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
  }
};

namespace dq {
namespace {

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

enum Kind { K_STATS, K_REDUCE, K_ALLOC_SEARCH, K_ALLOC_ASSIGN, K_LEAF, K_DAR, K_DA, K_DECODE, K_NCCL, K_NKINDS };
const char* const kKindName[K_NKINDS] = {"stats", "reduce_stats", "alloc_search", "alloc_assign", "quant_leaf",
                                         "quant_dar", "decompress_accumulate", "decode_out", "nccl"};
const int kKindLaunches[K_NKINDS] = {1, 1, 1, 3, 1, 1, 1, 1, 0};

cudaEvent_t pool_event(dq_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  DQ_CUDA(cudaEventCreate(&e));
  return e;
}

// run `launch` on st; when profiling, bracket it with events and book its algorithmic bytes
template <class F>
void timed(dq_ctx* ctx, int kind, double bytes, cudaStream_t st, F&& launch) {
  if (!ctx || !ctx->profile) {
    launch();
    if (ctx) ctx->prof_launches[kind] += kKindLaunches[kind];
    return;
  }
  dq_ctx::Prof p{kind, bytes, pool_event(ctx), pool_event(ctx)};
  DQ_CUDA(cudaEventRecord(p.a, st));
  launch();
  DQ_CUDA(cudaEventRecord(p.b, st));
  ctx->pending.push_back(p);
  ctx->prof_launches[kind] += kKindLaunches[kind];
}

// after a stream sync: fold the pending event pairs into the per-kind totals
void harvest(dq_ctx* ctx) {
  if (ctx->lr_pending && cudaEventQuery(ctx->lr1) == cudaSuccess) {
    float ms = 0.f;
    DQ_CUDA(cudaEventElapsedTime(&ms, ctx->lr0, ctx->lr1));
    ctx->last_round_ms = ms;
    ctx->lr_pending = false;
  }
  for (auto& p : ctx->pending) {
    float ms = 0.f;
    DQ_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    ctx->prof_ms[p.kind] += ms;
    ctx->prof_bytes[p.kind] += p.bytes;
    ctx->ev_pool.push_back(p.a);
    ctx->ev_pool.push_back(p.b);
  }
  ctx->pending.clear();
}

// A round returned without a host sync: keep its boundary events for the next sync
// (ev0/ev1 are re-recorded by the next round, so copy them into lr0/lr1 on the GPU
// timeline by recording the copies right here) and report the previous round's time.
void finish_async(dq_ctx* ctx, dq_round_info* info, cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  DQ_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) {  // recorded into a graph: nothing to time on the host
    info->ms_total = 0.0;
    return;
  }
  if (!ctx->lr0) {
    DQ_CUDA(cudaEventCreate(&ctx->lr0));
    DQ_CUDA(cudaEventCreate(&ctx->lr1));
  }
  std::swap(ctx->ev0, ctx->lr0);  // lr0 := this round's start event
  std::swap(ctx->ev1, ctx->lr1);  // lr1 := this round's end event
  ctx->lr_pending = true;
  info->ms_total = ctx->last_round_ms;
}

double quant_bytes(const Layout& L, bool dar) {  // local fp32 + mean/perm + in (DAR) + out
  const double chunk = static_cast<double>(L.bytes());
  return 1024.0 * L.nsg + 8.0 * L.nsg + chunk * (dar ? 2.0 : 1.0);
}

void validate(const dq_config& c) {  // engine.cpp:243-255 + device coverage
  if (c.n_workers == 0 || c.n_workers > 64) invalid("n_workers must be in 1..64");
  if (c.group_size == 0 || c.super_group_size % c.group_size != 0 || c.super_group_size % 4 != 0)
    invalid("super-group size must be a multiple of the group size and of 4");
  if (!c.variable_width && c.fixed_width != 2 && c.fixed_width != 4 && c.fixed_width != 8)
    invalid("fixed width must be one of {2,4,8}");
  if ((c.allocator == DQ_ALLOC_FIXED) != !c.variable_width)
    invalid("fixed-width allocator requires variable_width off and vice versa");
  if (c.threads == 0) invalid("threads must be >= 1");
  if (c.topology == DQ_BUTTERFLY && (c.n_workers & (c.n_workers - 1)) != 0)
    invalid("butterfly topology requires a power-of-two worker count");
  if (c.topology != DQ_RING && c.topology != DQ_BUTTERFLY) invalid("unknown topology");
  if (c.super_group_size != 256) invalid("device codec supports super_group_size 256");
  if (c.group_size != 8 && c.group_size != 16 && c.group_size != 32 && c.group_size != 64 && c.group_size != 128)
    invalid("device codec supports group_size 8, 16, 32, 64 or 128");
  if (c.codec != 0) invalid("device codec supports the quantized codec only");
  if (c.variable_width && c.allocator != DQ_ALLOC_FAST && c.allocator != DQ_ALLOC_GENERAL)
    invalid("unknown allocator");
}

double payload_budget(const dq_config& c) {  // allocation.cpp:45-58
  const double over = c.hierarchical_scales ? 8.0 / c.group_size + 16.0 / c.super_group_size : 16.0 / c.group_size;
  const double bbar = c.budget_bits - over;
  if (!(bbar > 2.0)) {
    char m[160];
    std::snprintf(m, sizeof m, "payload budget %f does not exceed the minimum width 2", bbar);
    throw Error(DQ_EINFEASIBLE, m);
  }
  return bbar;
}

AllocWork work_of(dq_ctx* ctx, uint32_t T) {
  ctx->level.reserve(T);
  if (!ctx->astate.p) {
    ctx->astate.reserve(1);
    DQ_CUDA(cudaMemset(ctx->astate.p, 0, sizeof(AllocState)));  // epoch 0: no mailbox answer matches
  }
  ctx->bins.reserve(4 * kAllocBins);
  ctx->blockcnt.reserve(4 * (alloc_blocks(T) + 1));
  ctx->counts.reserve(4);
  if (!ctx->h_state) DQ_CUDA(cudaMallocHost(&ctx->h_state, sizeof(AllocState)));
  if (!ctx->h_counts) DQ_CUDA(cudaMallocHost(&ctx->h_counts, 4 * sizeof(uint32_t)));
  ctx->pmean.reserve(T);
  const bool have_means = ctx->gmean.n >= T && ctx->gmean.p;  // round path; dq_allocate_fast alone has none
  return AllocWork{ctx->level.p, ctx->astate.p, ctx->bins.p, ctx->blockcnt.p, ctx->counts.p,
                   have_means ? ctx->gmean.p : nullptr, have_means ? ctx->pmean.p : nullptr};
}

struct AllocResult {
  uint32_t gs = 16, ss = 2, gshift = 1;  // scale format of the round's chunks (Layout)
  double u = 0.0;
  uint64_t payload = 0;
  uint32_t n8 = 0, n4 = 0, n2 = 0, passes = 0;
  bool async = false;  // counts live on the device only (ctx->counts), host mailbox parity `par`
  uint32_t par = 0;
};

// allocate_general for W = {2,4,8} (allocation.cpp:121-168), the round path's general
// allocator (engine.cpp:306-307,322-323): crossing points sorted on the device, then the
// reference's bisection over them driven from the host, one probe kernel per step.
AllocResult allocate_general(dq_ctx* ctx, const dq_config& c, const float* dF, uint32_t T, uint8_t* dW,
                             uint32_t* dP, cudaStream_t st) {
  AllocResult r;
  const uint32_t S = c.super_group_size;
  AllocWork w = work_of(ctx, T);
  const double bbar = payload_budget(c);
  const double budget = static_cast<double>(static_cast<uint64_t>(T) * S) * bbar;
  // threshold_chain({2,4,8}) (allocation.cpp:60-90): ratio (4^4-1)(4-2) / (4^4 4 (4^2-1)) = 17/512
  const double c1 = 1.0 / (17.0 / 512.0);
  ctx->gkeys.reserve(2ull * T + 1);
  ctx->gsorted.reserve(2ull * T + 1);
  const size_t tb = general_temp_bytes(T);
  ctx->gtemp.reserve(tb + 1);
  ctx->gnum.reserve(1);
  ctx->gbase.reserve(1);
  ctx->tcount.reserve(2);
  unsigned long long* d_bad = ctx->tcount.p;
  DQ_CUDA(launch_general_points(dF, T, c1, ctx->gkeys.p, ctx->gsorted.p, ctx->gtemp.p, tb, ctx->gnum.p, d_bad, st));
  int nu = 0;
  unsigned long long bad = 0;
  DQ_CUDA(cudaMemcpyAsync(&nu, ctx->gnum.p, sizeof nu, cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaStreamSynchronize(st));
  if (bad) invalid("squared norms must be non-negative");
  uint32_t M = static_cast<uint32_t>(nu);
  if (M) {
    uint64_t last = 0;
    DQ_CUDA(cudaMemcpy(&last, ctx->gkeys.p + M - 1, sizeof last, cudaMemcpyDeviceToHost));
    if (last == ~0ull) --M;  // the non-positive F_j
  }
  // points[0..M) unique ascending, points[M] = the all-min plateau (allocation.cpp:146-147)
  struct Probe {
    double base;
    uint64_t payload;
  };
  auto probe = [&](uint32_t idx) {
    launch_general_counts(dF, T, ctx->gkeys.p, M, idx, c1, ctx->tcount.p, ctx->gbase.p, st);
    unsigned long long cnt[2];
    Probe p;
    DQ_CUDA(cudaMemcpyAsync(cnt, ctx->tcount.p, sizeof cnt, cudaMemcpyDeviceToHost, st));
    DQ_CUDA(cudaMemcpyAsync(&p.base, ctx->gbase.p, sizeof p.base, cudaMemcpyDeviceToHost, st));
    DQ_CUDA(cudaStreamSynchronize(st));
    p.payload = static_cast<uint64_t>(S) * (2ull * T + 2ull * cnt[1] + 4ull * cnt[0]);
    return p;
  };
  uint32_t lo = 0, hi = M;
  Probe p = probe(lo);
  if (static_cast<double>(p.payload) > budget) {
    while (lo + 1 < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;  // == (lo + hi) / 2 without overflow
      if (static_cast<double>(probe(mid).payload) <= budget) hi = mid;
      else lo = mid;
    }
    lo = hi;
    p = probe(lo);
  }
  const double base = p.base;
  timed(ctx, K_ALLOC_ASSIGN, 13.0 * T, st, [&] { launch_general_assign(dF, T, base, base * c1, w, dW, dP, st); });
  DQ_CUDA(cudaGetLastError());
  DQ_CUDA(cudaMemcpyAsync(ctx->h_counts, w.counts, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaStreamSynchronize(st));
  harvest(ctx);
  r.u = base;
  r.n8 = ctx->h_counts[0];
  r.n4 = ctx->h_counts[1];
  r.n2 = ctx->h_counts[2];
  r.payload = static_cast<uint64_t>(S) * (8ull * r.n8 + 4ull * r.n4 + 2ull * r.n2);
  if (static_cast<double>(r.payload) > budget) throw Error(DQ_EINFEASIBLE, "bit allocation infeasible within budget");
  return r;
}

AllocResult allocate_fast(dq_ctx* ctx, const dq_config& c, const float* dF, uint32_t T, uint8_t* dW,
                          uint32_t* dP, cudaStream_t st);

// allocate_fast / allocate_general / fixed width (engine.cpp:308-326) + build_permutation
AllocResult allocate(dq_ctx* ctx, const dq_config& c, const float* dF, uint32_t T, uint8_t* dW,
                     uint32_t* dP, cudaStream_t st) {
  if (c.variable_width && c.allocator == DQ_ALLOC_GENERAL) return allocate_general(ctx, c, dF, T, dW, dP, st);
  return allocate_fast(ctx, c, dF, T, dW, dP, st);
}

// allocate_fast (allocation.cpp:228-260) + build_permutation; see dq_stats_alloc.cu
AllocResult allocate_fast(dq_ctx* ctx, const dq_config& c, const float* dF, uint32_t T, uint8_t* dW,
                          uint32_t* dP, cudaStream_t st) {
  AllocResult r;
  const uint32_t S = c.super_group_size;
  AllocWork w = work_of(ctx, T);
  const double bbar = payload_budget(c);
  if (!c.variable_width) {
    if (c.fixed_width > bbar)
      throw Error(DQ_EINFEASIBLE, "fixed width " + std::to_string(c.fixed_width) + " exceeds the payload budget");
    launch_fixed_assign(T, c.fixed_width, w, dW, dP, st);
    DQ_CUDA(cudaGetLastError());
    r.n8 = c.fixed_width == 8 ? T : 0;
    r.n4 = c.fixed_width == 4 ? T : 0;
    r.n2 = c.fixed_width == 2 ? T : 0;
    r.payload = static_cast<uint64_t>(T) * S * c.fixed_width;
    return r;
  }
  const double budget = static_cast<double>(T) * S * bbar;
  // largest cumulative flip weight W with S * (2T + W) <= budget, compared in double
  auto fits = [&](int64_t W) { return static_cast<double>(static_cast<uint64_t>(S) * (2ull * T + W)) <= budget; };
  int64_t W = static_cast<int64_t>(std::floor(budget / S)) - 2 * static_cast<int64_t>(T);
  if (W < -1) W = -1;
  while (fits(W + 1)) ++W;
  while (W >= 0 && !fits(W)) --W;
  if (W < 0) throw Error(DQ_EINFEASIBLE, "bit allocation infeasible within budget");
  // search + neighbourhood decision on device, assignment with the device thresholds,
  // then ONE sync that brings back the state and the class counts together
  timed(ctx, K_ALLOC_SEARCH, 8.0 * T, st,
        [&] { DQ_CUDA(launch_alloc_search(dF, T, kAlpha, static_cast<uint64_t>(W), budget, S, w, st)); });
  timed(ctx, K_ALLOC_ASSIGN, 13.0 * T, st, [&] { launch_alloc_assign(dF, T, 0.f, 0.f, true, w, dW, dP, st); });
  DQ_CUDA(cudaGetLastError());
  DQ_CUDA(cudaMemcpyAsync(ctx->h_state, w.state, sizeof(AllocState), cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaMemcpyAsync(ctx->h_counts, w.counts, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaStreamSynchronize(st));
  harvest(ctx);  // events of the previous round (finished asynchronously) are complete now
  const AllocState s = *ctx->h_state;
  if (s.status == 0 || s.status > 3)
    throw Error(DQ_ECUDA, "allocation search did not converge (status " + std::to_string(s.status) + ")");
  // Re-derive every candidate with the host libm exactly as fast_sample_points /
  // fast_threshold_* do (allocation.cpp:170-224).  Identical thresholds => identical
  // float-threshold counts => the device's choice is the reference's.
  struct Sample {
    bool has_l = false, has_r = false;
    FlipRec l{}, r{};
    double u() const {
      double v = has_l && has_r ? 0.5 * (hflip_s(l) + hflip_s(r)) : has_r ? hflip_s(r) - 1.0 : has_l ? hflip_s(l) + 1.0 : 0.0;
      return v < -1e6 ? -1e6 : (v > 1e6 ? 1e6 : v);
    }
    static double hflip_s(const FlipRec& q) {
      float f;
      std::memcpy(&f, &q.fbits, 4);
      return (q.type ? 8.0 : 4.0) - kAlpha * std::log2(static_cast<double>(f));
    }
  };
  auto thr = [](double uu, float* a, float* b) {
    *a = static_cast<float>(std::exp2((4.0 - uu) / kAlpha));
    *b = static_cast<float>(std::exp2((8.0 - uu) / kAlpha));
  };
  Sample cand[3];  // L-1, L, L+1 as the device built them
  if (s.status == 2) {
    cand[1].has_l = true;
    cand[1].l = s.slot[1];
    cand[0].has_r = true;
    cand[0].r = s.slot[1];
    if (s.slot[0].present) {
      cand[0].has_l = true;
      cand[0].l = s.slot[0];
    }
  } else if (s.status == 1) {
    cand[1].has_r = true;
    cand[1].r = s.slot[2];
    if (s.slot[1].present) {
      cand[1].has_l = true;
      cand[1].l = s.slot[1];
      cand[0].has_r = true;
      cand[0].r = s.slot[1];
      if (s.slot[0].present) {
        cand[0].has_l = true;
        cand[0].l = s.slot[0];
      }
    }
    cand[2].has_l = true;
    cand[2].l = s.slot[2];
    if (s.slot[3].present) {
      cand[2].has_r = true;
      cand[2].r = s.slot[3];
    }
  }
  bool mismatch = false;
  for (int c = 0; c < 3; ++c) {
    if (!s.cand_present[c]) continue;
    float a, b;
    thr(cand[c].u(), &a, &b);
    // a threshold the device left ambiguous (two adjacent floats, no F_j equal to the lower)
    // gives the same widths with either float
    auto same = [&](float h, float dv, float amb) {
      if (h == dv) return true;
      return s.namb == 0 && amb > 0.0f && std::min(h, dv) == amb && std::nextafter(amb, INFINITY) == std::max(h, dv);
    };
    mismatch |= !same(a, s.cand_t24[c], s.amb[c][0]) || !same(b, s.cand_t48[c], s.amb[c][1]);
  }
  double u;
  float t24, t48;
  if (!mismatch && s.choice == -2) throw Error(DQ_EINFEASIBLE, "bit allocation infeasible within budget");
  if (!mismatch && s.choice >= 0) {
    u = cand[s.choice].u();
    t24 = s.t24;
    t48 = s.t48;
  } else {
    // Exact host-driven walk over the samples (rare): the reference's bisection on a
    // non-decreasing payload(u) ends at the largest sample whose float-threshold
    // payload fits; step from the device's candidate until that boundary.
    ++ctx->alloc_redos;
    ctx->nrec.reserve(1);
    ctx->tcount.reserve(2);
    auto neighbor = [&](const FlipRec& q, int dir) {
      launch_flip_neighbor(w.level, dF, T, kAlpha, q.key, dir, ctx->nrec.p, st);
      FlipRec out;
      DQ_CUDA(cudaMemcpyAsync(&out, ctx->nrec.p, sizeof(FlipRec), cudaMemcpyDeviceToHost, st));
      DQ_CUDA(cudaStreamSynchronize(st));
      return out;
    };
    auto fits = [&](const Sample& sm) {
      float a, b;
      thr(sm.u(), &a, &b);
      launch_threshold_counts(dF, T, a, b, ctx->tcount.p, st);
      unsigned long long cnt[2];
      DQ_CUDA(cudaMemcpyAsync(cnt, ctx->tcount.p, sizeof(cnt), cudaMemcpyDeviceToHost, st));
      DQ_CUDA(cudaStreamSynchronize(st));
      const unsigned long long pay = static_cast<unsigned long long>(S) * (2ull * T + 2ull * cnt[1] + 4ull * cnt[0]);
      return static_cast<double>(pay) <= budget;
    };
    Sample cur = cand[1];
    if (fits(cur)) {
      while (cur.has_r) {
        Sample nx;
        nx.has_l = true;
        nx.l = cur.r;
        const FlipRec q = neighbor(cur.r, +1);
        if (q.present) {
          nx.has_r = true;
          nx.r = q;
        }
        if (!fits(nx)) break;
        cur = nx;
      }
    } else {
      for (;;) {
        if (!cur.has_l) throw Error(DQ_EINFEASIBLE, "bit allocation infeasible within budget");
        Sample pv;
        pv.has_r = true;
        pv.r = cur.l;
        const FlipRec q = neighbor(cur.l, -1);
        if (q.present) {
          pv.has_l = true;
          pv.l = q;
        }
        cur = pv;
        if (fits(cur)) break;
      }
    }
    u = cur.u();
    thr(u, &t24, &t48);
    timed(ctx, K_ALLOC_ASSIGN, 13.0 * T, st, [&] { launch_alloc_assign(dF, T, t24, t48, false, w, dW, dP, st); });
    DQ_CUDA(cudaGetLastError());
    DQ_CUDA(cudaMemcpyAsync(ctx->h_counts, w.counts, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    DQ_CUDA(cudaStreamSynchronize(st));
  }
  r.u = u;
  r.n8 = ctx->h_counts[0];
  r.n4 = ctx->h_counts[1];
  r.n2 = ctx->h_counts[2];
  r.passes = s.passes;
  r.payload = static_cast<uint64_t>(S) * (8ull * r.n8 + 4ull * r.n4 + 2ull * r.n2);
  if (static_cast<double>(r.payload) > budget) {
    char m[512];
    std::snprintf(m, sizeof m,
                  "bit allocation infeasible within budget (T=%u W=%lld status=%u passes=%u has_pred=%u "
                  "u=%.17g t24=%a/%a t48=%a/%a counts=%u,%u,%u payload=%llu budget=%.17g)",
                  T, static_cast<long long>(W), s.status, s.passes, s.has_pred, u, t24, s.t24, t48, s.t48, r.n8,
                  r.n4, r.n2, static_cast<unsigned long long>(r.payload), budget);
    throw Error(DQ_EINFEASIBLE, m);
  }
  return r;
}

// u of the search's chosen candidate, re-derived with the host libm exactly as
// fast_sample_points does (allocation.cpp:201-224) from the flips the search identified.
// glibc u of candidate sample c (0..2 = L-1, L, L+1) from the device's flip records
double host_cand_u(const AllocState& s, int c) {
  auto hflip = [](const FlipRec& q) {
    float f;
    std::memcpy(&f, &q.fbits, 4);
    return (q.type ? 8.0 : 4.0) - kAlpha * std::log2(static_cast<double>(f));
  };
  auto clampu = [](double v) { return v < -1e6 ? -1e6 : (v > 1e6 ? 1e6 : v); };
  const FlipRec* l = nullptr;
  const FlipRec* r = nullptr;
  if (s.status == 2) {
    if (c == 1) l = &s.slot[1];
    else { r = &s.slot[1]; if (s.slot[0].present) l = &s.slot[0]; }
  } else if (s.status == 1) {
    if (c == 1) { r = &s.slot[2]; if (s.slot[1].present) l = &s.slot[1]; }
    else if (c == 0) { r = &s.slot[1]; if (s.slot[0].present) l = &s.slot[0]; }
    else { l = &s.slot[2]; if (s.slot[3].present) r = &s.slot[3]; }
  }
  if (l && r) return clampu(0.5 * (hflip(*l) + hflip(*r)));
  if (r) return clampu(hflip(*r) - 1.0);
  if (l) return clampu(hflip(*l) + 1.0);
  return 0.0;
}
double host_u_of(const AllocState& s) { return host_cand_u(s, s.choice >= 0 ? s.choice : 1); }

// allocate_fast on the host (allocation.cpp:195-260, the same sorted samples and the same
// bisection): the rare asynchronous rounds whose thresholds the device could not certify.
// Returns false when even the first sample is over budget (InfeasibleBudget).
bool host_allocate_fast(const float* F, uint32_t T, uint32_t S, double budget, double* u, float* t24, float* t48) {
  std::vector<double> flips;
  flips.reserve(2ull * T);
  for (uint32_t j = 0; j < T; ++j) {
    if (!(F[j] > 0.0f)) continue;
    const double l = kAlpha * std::log2(static_cast<double>(F[j]));
    flips.push_back(4.0 - l);
    flips.push_back(8.0 - l);
  }
  std::sort(flips.begin(), flips.end());
  flips.erase(std::unique(flips.begin(), flips.end()), flips.end());
  std::vector<double> samples;
  if (flips.empty()) {
    samples.push_back(0.0);
  } else {
    samples.push_back(flips.front() - 1.0);
    for (size_t i = 0; i + 1 < flips.size(); ++i) samples.push_back(0.5 * (flips[i] + flips[i + 1]));
    samples.push_back(flips.back() + 1.0);
  }
  for (double& v : samples) v = v < -1e6 ? -1e6 : (v > 1e6 ? 1e6 : v);
  auto thr = [](double uu, float* a, float* b) {
    *a = static_cast<float>(std::exp2((4.0 - uu) / kAlpha));
    *b = static_cast<float>(std::exp2((8.0 - uu) / kAlpha));
  };
  auto payload = [&](double uu) {
    float a, b;
    thr(uu, &a, &b);
    uint64_t w = 0;
    for (uint32_t j = 0; j < T; ++j) w += F[j] >= b ? 8 : (F[j] >= a ? 4 : 2);
    return static_cast<double>(w * S);
  };
  size_t lo = 0, hi = samples.size() - 1;
  if (payload(samples[lo]) > budget) return false;
  if (payload(samples[hi]) <= budget) {
    lo = hi;
  } else {
    while (lo + 1 < hi) {
      const size_t mid = (lo + hi) / 2;
      if (payload(samples[mid]) <= budget) lo = mid;
      else hi = mid;
    }
  }
  *u = samples[lo];
  thr(*u, t24, t48);
  return true;
}

// The host side of a need_host round: finish the allocation from the exported F and
// release the assignment kernel, which waits for `resolved` to reach the round's epoch.
void host_alloc_resolve(HostMsg* m) {
  const AllocState& s = m->state;
  static const bool verbose = std::getenv("DQ_DEBUG_ALLOC") != nullptr;
  if (verbose) {
    std::fprintf(stderr, "dynamiq_b200: host finish: T=%u certified=%u choice=%d status=%u passes=%u\n", s.T,
                 s.certified, s.choice, s.status, s.passes);
    for (int c = 0; c < 3; ++c) {
      if (!s.cand_present[c]) continue;
      const double uu = s.cand_u[c];
      const double d24 = std::exp2((4.0 - uu) / kAlpha), d48 = std::exp2((8.0 - uu) / kAlpha);
      std::fprintf(stderr, "  cand %d: u=%.17g t24=%a (host %a, d %a) t48=%a (host %a, d %a)\n", c, uu,
                   s.cand_t24[c], static_cast<float>(d24), d24, s.cand_t48[c], static_cast<float>(d48), d48);
    }
    for (int k = 0; k < 4; ++k) {
      float f;
      std::memcpy(&f, &s.slot[k].fbits, 4);
      std::fprintf(stderr, "  slot %d: present=%u type=%u F=%a\n", k, s.slot[k].present, s.slot[k].type, f);
    }
  }
  double u = 0.0;
  float a = INFINITY, b = INFINITY;  // infeasible: all width 2 (the round is reported as failed)
  const bool ok = host_allocate_fast(m->hF, s.T, s.S, s.budget, &u, &a, &b);
  m->u = u;
  m->t24 = a;
  m->t48 = b;
  m->host_status = ok ? 0 : DQ_EINFEASIBLE;
  __atomic_store_n(const_cast<uint32_t*>(&m->resolved), s.epoch, __ATOMIC_RELEASE);
}

// Threshold consult (alloc_consult): the glibc u and float thresholds of each present
// candidate - a few log2 / exp2 calls, the device recounts with them.
void host_thr_resolve(HostMsg* m, uint32_t tag) {
  const AllocState& s = m->state;
  for (int c = 0; c < 3; ++c) {
    if (!s.cand_present[c]) continue;
    const double u = host_cand_u(s, c);
    m->thr_u[c] = u;
    m->thr_t24[c] = static_cast<float>(std::exp2((4.0 - u) / kAlpha));
    m->thr_t48[c] = static_cast<float>(std::exp2((8.0 - u) / kAlpha));
  }
  __atomic_store_n(const_cast<uint32_t*>(&m->thr_resolved), tag, __ATOMIC_RELEASE);
}

// Per-context host service thread: polls both mailboxes for a request newer than its
// answer (no CUDA calls, no per-round callbacks: the common round never involves the host).
void alloc_service(dq_ctx* ctx) {
  while (!ctx->svc_stop.load(std::memory_order_relaxed)) {
    bool busy = false;
    for (int p = 0; p < 2; ++p) {
      HostMsg* m = ctx->hmsg + p;
      const uint32_t treq = __atomic_load_n(const_cast<uint32_t*>(&m->thr_request), __ATOMIC_ACQUIRE);
      if (treq != 0 && treq != m->thr_resolved) {
        host_thr_resolve(m, treq);
        ctx->host_consults.fetch_add(1, std::memory_order_relaxed);
        busy = true;
      }
      const uint32_t req = __atomic_load_n(const_cast<uint32_t*>(&m->request), __ATOMIC_ACQUIRE);
      if (req != 0 && req != m->resolved && req == m->state.epoch) {
        host_alloc_resolve(m);
        ctx->host_allocs.fetch_add(1, std::memory_order_relaxed);
        busy = true;
      }
    }
    if (!busy) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

void ensure_mailbox(dq_ctx* ctx, uint32_t T) {
  if (!ctx->hmsg) {
    DQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->hmsg), 2 * sizeof(HostMsg), cudaHostAllocMapped));
    std::memset(static_cast<void*>(ctx->hmsg), 0, 2 * sizeof(HostMsg));
  }
  if (ctx->hF_cap < T) {
    DQ_CUDA(cudaDeviceSynchronize());  // growing: no round may still write the old copy
    if (ctx->hF) DQ_CUDA(cudaFreeHost(ctx->hF));
    ctx->hF = nullptr;
    const size_t cap = T + T / 4 + 1024;
    DQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->hF), cap * sizeof(float), cudaHostAllocMapped));
    ctx->hF_cap = cap;
    ctx->hmsg[0].hF = ctx->hF;
    ctx->hmsg[1].hF = ctx->hF;
  }
  if (!ctx->svc.joinable()) ctx->svc = std::thread(alloc_service, ctx);
}

// allocate_fast + build_permutation with no host synchronisation: the search decides and
// certifies on the device; the assignment follows in stream order (waiting for the host
// function only on the rare need_host rounds); the class counts stay on the device
// (ctx->counts) for the kernels and are mirrored to the mailbox for dq_round_info.
AllocResult allocate_fast_async(dq_ctx* ctx, const dq_config& c, const float* dF, uint32_t T, uint8_t* dW,
                                uint32_t* dP, cudaStream_t st) {
  const StatsReduce red = ctx->pending_red;  // the round's statistics reduction, not yet launched
  ctx->pending_red = StatsReduce{};
  AllocResult r;
  r.async = true;
  const uint32_t S = c.super_group_size;
  AllocWork w = work_of(ctx, T);
  const double bbar = payload_budget(c);
  const double budget = static_cast<double>(T) * S * bbar;
  auto fits = [&](int64_t W) { return static_cast<double>(static_cast<uint64_t>(S) * (2ull * T + W)) <= budget; };
  int64_t W = static_cast<int64_t>(std::floor(budget / S)) - 2 * static_cast<int64_t>(T);
  if (W < -1) W = -1;
  while (fits(W + 1)) ++W;
  while (W >= 0 && !fits(W)) --W;
  if (W < 0) throw Error(DQ_EINFEASIBLE, "bit allocation infeasible within budget");
  ensure_mailbox(ctx, T);
  const uint32_t par = ctx->apar ^= 1u;
  r.par = par;
  HostMsg* m = ctx->hmsg + par;
  void* dm = nullptr;
  void* dF_host = nullptr;
  DQ_CUDA(cudaHostGetDevicePointer(&dm, m, 0));
  DQ_CUDA(cudaHostGetDevicePointer(&dF_host, ctx->hF, 0));
  w.hmsg = static_cast<HostMsg*>(dm);
  w.hF = static_cast<float*>(dF_host);
  w.red = red;
  if (!ctx->no_small_alloc && launch_alloc_small(dF, T, kAlpha, budget, S, w, dW, dP, st)) {
    DQ_CUDA(cudaGetLastError());
    ctx->prof_launches[K_ALLOC_SEARCH] += 1;  // launch count only (asynchronous rounds are not event-timed)
    return r;
  }
  if (red.mean) {  // (not reached: the caller folds the reduction only into small rounds)
    if (red.flags)
      launch_reduce_stats_peer(red.mean, red.sq, red.flags, red.epoch_ptr, red.n, T, red.stride, red.gm, red.gs, st);
    else
      launch_reduce_stats(red.mean, red.sq, red.n, T, red.gm, red.gs, st);
  }
  DQ_CUDA(launch_alloc_search(dF, T, kAlpha, static_cast<uint64_t>(W), budget, S, w, st));
  launch_alloc_assign(dF, T, 0.f, 0.f, true, w, dW, dP, st);
  DQ_CUDA(cudaGetLastError());
  ctx->prof_launches[K_ALLOC_SEARCH] += kKindLaunches[K_ALLOC_SEARCH];
  ctx->prof_launches[K_ALLOC_ASSIGN] += kKindLaunches[K_ALLOC_ASSIGN];
  return r;
}

// scale format of the codec config (codec.cpp:88-116): s = 8 << gshift entries per
// group; hierarchical: 256/s u8 codes + bf16 sg_scale, flat: 256/s bf16 per super-group
template <class T>
void set_format(T& f, const dq_config& c) {
  uint32_t sh = 0;
  while ((8u << sh) < c.group_size) ++sh;
  f.gshift = sh;
  f.gs = c.hierarchical_scales ? 256 / c.group_size : 2 * 256 / c.group_size;
  f.ss = c.hierarchical_scales ? 2 : 0;
}

Layout chunk_layout(const AllocResult& a, uint32_t lo, uint32_t hi) {
  auto overlap = [](uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
    const uint32_t l = a0 > b0 ? a0 : b0, h = a1 < b1 ? a1 : b1;
    return h > l ? h - l : 0u;
  };
  Layout L;
  L.nsg = hi - lo;
  L.n8 = overlap(lo, hi, 0, a.n8);
  L.n4 = overlap(lo, hi, a.n8, a.n8 + a.n4);
  L.gs = a.gs;
  L.ss = a.ss;
  L.gshift = a.gshift;
  return L;
}

CodecArgs base_args(const dq_config& c, uint32_t chunk) {
  CodecArgs a{};
  a.h3_eq = absorb(purpose_prefix(c.seed, c.round, kEntryQuant), chunk);
  a.h3_sc = absorb(purpose_prefix(c.seed, c.round, kScaleQuant), chunk);
  a.h3_pm = absorb(purpose_prefix(c.seed, c.round, kPermutation), chunk);
  a.correlated = c.correlated;
  a.uniform_books = c.non_uniform ? 0 : 1;
  // width-8 index estimate: q[r] = (B^r - 1) / (B^127 - 1), B = 1 + 2 eps^2 (codebook.cpp:20-48)
  const double B = 1.0 + 2.0 * 0.05 * 0.05;
  a.est_c1 = c.non_uniform ? static_cast<float>(std::pow(B, 127) - 1.0) : 0.0f;
  a.est_c2 = c.non_uniform ? static_cast<float>(1.0 / std::log2(B)) : 127.0f;
  a.n_workers_f = static_cast<float>(c.n_workers);
  return a;
}

// reference-format bytes of a device chunk (serialize_chunk, codec.cpp:319-343)
void to_reference(const uint8_t* soa, uint32_t chunk, const Layout& L, uint8_t* out) {
  auto put32 = [&](size_t at, uint32_t v) {
    for (int i = 0; i < 4; ++i) out[at + i] = static_cast<uint8_t>(v >> (8 * i));
  };
  put32(0, chunk);
  put32(4, L.nsg);
  put32(8, L.n8);
  put32(12, L.n4);
  put32(16, L.n2());
  put32(20, L.n16);
  size_t at = 24;
  for (uint32_t i = 0; i < L.nsg; ++i) {
    const Layout::SG g = L.locate(i);
    if (g.width == 16) {  // passthrough record: payload only (codec.cpp:334-337)
      std::memcpy(out + at, soa + g.payload, 512);
      at += 512;
      continue;
    }
    std::memcpy(out + at, soa + g.scale, L.ss);
    std::memcpy(out + at + L.ss, soa + g.codes, L.gs);
    std::memcpy(out + at + L.ss + L.gs, soa + g.payload, 32 * g.width);
    at += L.ss + L.gs + 32 * g.width;
  }
}

// wire accounting of one message of a chunk (engine.cpp:135-160)
void account(dq_round_info* info, const Layout& L, bool fresh) {
  const uint64_t coords = static_cast<uint64_t>(L.nsg) * 256;
  const uint64_t pay = 256ull * (8ull * L.n8 + 4ull * L.n4 + 2ull * L.n2());
  const uint64_t scl = static_cast<uint64_t>(L.nsg) * 8 * (L.gs + L.ss);  // supergroup_scale_bits (codec.cpp:274-279)
  info->transmitted_coordinates += coords;
  info->header_bits += 192;
  info->wire_payload_bits += pay;
  info->scale_bits += scl;
  if (fresh) {
    info->repr_bits += pay + scl;
    info->compressed_coordinates += coords;
  }
}

struct Prepared {
  uint32_t T;
  AllocResult a;
  std::vector<uint32_t> lo;  // chunk boundaries (engine.cpp:52-62)
  size_t max_chunk_bytes;
};

constexpr uint32_t kChunkStreams = 8;  // worker streams of a simulated round's chunk chains

// Rounds that allocate asynchronously: the fast allocator without the instrumentation or
// wire-hash modes (both read per-chunk sizes on the host); DQ_SYNC_ALLOC=1 turns it off.
bool async_alloc_ok(const dq_ctx* ctx, bool collect_wire) {
  const dq_config& c = ctx->cfg;
  return ctx->async_alloc && !ctx->profile && !collect_wire && c.variable_width && c.allocator == DQ_ALLOC_FAST;
}
// asynchronous rounds whose one-CTA allocation also performs the statistics reduction (one
// kernel less on the latency path of small all-reduces).  Up to 2048 super-groups: at 4096
// the single CTA's reduction of n rows costs more than the separate kernel saves (N = 4,
// 2^20 entries per rank: 0.183 vs 0.174 ms; 2^18: 0.137 vs 0.142 ms).
bool small_alloc_round(const dq_ctx* ctx, uint32_t T, bool async) {
  return async && !ctx->no_small_alloc && T > 0 && T <= 2048 && T <= kSmallAllocMaxT;
}

// stats (already reduced into ctx->gsq / gmean) -> allocation -> chunk plan.  Async: the
// class counts stay on the device, every chunk is sized for the worst case (all width 8)
// and the kernels derive their width runs from ctx->counts.
Prepared prepare(dq_ctx* ctx, uint32_t T, cudaStream_t st, bool async = false) {
  Prepared p;
  p.T = T;
  const dq_config& c = ctx->cfg;
  p.a = async ? allocate_fast_async(ctx, c, ctx->gsq.p, T, ctx->widths.p, ctx->perm.p, st)
              : allocate(ctx, c, ctx->gsq.p, T, ctx->widths.p, ctx->perm.p, st);
  set_format(p.a, c);
  const uint32_t n = c.n_workers;
  p.lo.resize(n + 1);
  for (uint32_t i = 0; i <= n; ++i) p.lo[i] = static_cast<uint32_t>(static_cast<uint64_t>(T) * i / n);
  p.max_chunk_bytes = 0;
  for (uint32_t i = 0; i < n; ++i) {
    Layout L = chunk_layout(p.a, p.lo[i], p.lo[i + 1]);
    if (async) L.n8 = L.nsg;  // worst case
    const size_t b = L.bytes();
    p.max_chunk_bytes = b > p.max_chunk_bytes ? b : p.max_chunk_bytes;
  }
  p.max_chunk_bytes = (p.max_chunk_bytes + 255) / 256 * 256;
  ctx->last_T = T;
  ctx->rec = dq_ctx::RoundRec{};
  ctx->rec.valid = true;
  ctx->rec.async = async;
  ctx->rec.par = p.a.par;
  ctx->rec.T = T;
  ctx->rec.n = n;
  ctx->rec.S = c.super_group_size;
  ctx->rec.gs = p.a.gs;
  ctx->rec.ss = p.a.ss;
  ctx->rec.gshift = p.a.gshift;
  ctx->rec.topology = c.topology;
  ctx->rec.lo = p.lo;
  return p;
}

void reserve_round(dq_ctx* ctx, uint32_t T, uint32_t n) {
  ctx->mean_all.reserve(static_cast<size_t>(n) * T);
  ctx->sq_all.reserve(static_cast<size_t>(n) * T);
  ctx->gmean.reserve(T);
  ctx->gsq.reserve(T);
  ctx->widths.reserve(T);
  ctx->perm.reserve(T);
}

void fill_info_alloc(dq_round_info* info, const Prepared& p) {
  info->u = p.a.u;
  info->payload_bits = p.a.payload;
  info->n8 = p.a.n8;
  info->n4 = p.a.n4;
  info->n2 = p.a.n2;
  info->alloc_passes = p.a.passes;
}

// wire accounting of a whole round (engine.cpp:135-160,368-396): every reduce event sends
// one fresh message of its chunk, the all-gather forwards the sink's bytes n_gat times
void account_round(dq_round_info* info, const AllocResult& a, const std::vector<uint32_t>& lo, uint32_t n,
                   int topology) {
  for (uint32_t ch = 0; ch < n; ++ch) {
    const Plan plan = make_plan(n, ch, topology);
    const Layout L = chunk_layout(a, lo[ch], lo[ch + 1]);
    for (size_t e = 0; e < plan.red.size(); ++e) account(info, L, true);
    for (uint32_t g = 0; g < plan.n_gat; ++g) account(info, L, g == 0);
    info->stats_bits += static_cast<uint64_t>(plan.red.size() + plan.n_gat) * 64ull * L.nsg;
  }
}

// Allocation + accounting fields of the last asynchronous round, from the mailbox it
// filled (call only once the round has completed on the device).
void finish_info(dq_ctx* ctx, dq_round_info* info) {
  const dq_ctx::RoundRec& rec = ctx->rec;
  if (!rec.valid || !rec.async) return;
  const HostMsg& m = ctx->hmsg[rec.par];
  if (m.state.need_host && m.host_status)
    throw Error(m.host_status, "bit allocation infeasible within budget (host finish)");
  AllocResult a;
  a.gs = rec.gs;
  a.ss = rec.ss;
  a.gshift = rec.gshift;
  a.n8 = m.counts[0];
  a.n4 = m.counts[1];
  a.n2 = m.counts[2];
  a.u = m.state.need_host ? m.u : host_u_of(m.state);
  a.passes = m.state.passes;
  a.payload = static_cast<uint64_t>(rec.S) * (8ull * a.n8 + 4ull * a.n4 + 2ull * a.n2);
  info->u = a.u;
  info->payload_bits = a.payload;
  info->n8 = a.n8;
  info->n4 = a.n4;
  info->n2 = a.n2;
  info->alloc_passes = a.passes;
  info->stats_bits = info->wire_payload_bits = info->scale_bits = info->header_bits = 0;
  info->repr_bits = info->compressed_coordinates = info->transmitted_coordinates = 0;
  account_round(info, a, rec.lo, rec.n, rec.topology);
}

// ---------------------------------------------------------- simulation
void sim_round(dq_ctx* ctx, const float* const* xs, size_t d, float* out, int flags,
               dq_round_info* info, cudaStream_t st) {
  const int collect_wire = flags & DQ_SIM_COLLECT_WIRE;
  const dq_config& c = ctx->cfg;
  const uint32_t n = c.n_workers;
  *info = dq_round_info{};
  if (d == 0) invalid("empty gradient");
  if (n == 1) {  // engine.cpp:280-286: nothing to synchronize
    DQ_CUDA(cudaMemcpyAsync(out, xs[0], d * sizeof(float), cudaMemcpyDeviceToDevice, st));
    return;
  }
  for (uint32_t r = 0; r < n; ++r)
    if (reinterpret_cast<uintptr_t>(xs[r]) % 16) invalid("gradients must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(out) % 16) invalid("output must be 16-byte aligned");
  const uint64_t T64 = (d + 255) / 256;
  if (T64 > 0xffffffffull / 2) invalid("gradient too large");
  const uint32_t T = static_cast<uint32_t>(T64);
  ensure_books();
  if (!ctx->ev0) {
    DQ_CUDA(cudaEventCreate(&ctx->ev0));
    DQ_CUDA(cudaEventCreate(&ctx->ev1));
  }
  DQ_CUDA(cudaEventRecord(ctx->ev0, st));
  reserve_round(ctx, T, n);
  ctx->pending_red = StatsReduce{};
  timed(ctx, K_STATS, 4.0 * n * d + 8.0 * n * T, st,
        [&] { launch_stats(xs, n, d, T, ctx->mean_all.p, ctx->sq_all.p, st); });
  const bool async = async_alloc_ok(ctx, collect_wire);
  if (small_alloc_round(ctx, T, async)) {
    StatsReduce& rd = ctx->pending_red;
    rd = StatsReduce{ctx->mean_all.p, ctx->sq_all.p, nullptr, nullptr, n, T, ctx->gmean.p, ctx->gsq.p};
  } else {
    timed(ctx, K_REDUCE, 8.0 * (n + 1) * T, st,
          [&] { launch_reduce_stats(ctx->mean_all.p, ctx->sq_all.p, n, T, ctx->gmean.p, ctx->gsq.p, st); });
  }
  DQ_CUDA(cudaGetLastError());
  Prepared p = prepare(ctx, T, st, async);
  if (!async) fill_info_alloc(info, p);

  // The chunks' event chains are independent: asynchronous rounds run chunk ch on worker
  // stream ch % kChunkStreams (forked after the allocation, joined before the gather decode),
  // so one chunk's kernels fill the others' partial last waves; each chunk then owns its
  // message slots, slices and accumulators.  The wire-hash and profiling modes keep one stream.
  const bool multi = async && n >= 2;
  const uint32_t nstreams = multi ? std::min<uint32_t>(n, kChunkStreams) : 1;
  if (multi) {
    while (ctx->cstreams.size() < nstreams) {
      cudaStream_t s2;
      DQ_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
      ctx->cstreams.push_back(s2);
      cudaEvent_t e2;
      DQ_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      ctx->cjoin.push_back(e2);
    }
    if (!ctx->cfork) DQ_CUDA(cudaEventCreateWithFlags(&ctx->cfork, cudaEventDisableTiming));
    DQ_CUDA(cudaEventRecord(ctx->cfork, st));
    for (uint32_t k = 0; k < nstreams; ++k) DQ_CUDA(cudaStreamWaitEvent(ctx->cstreams[k], ctx->cfork, 0));
  }
  // message pool: per-worker pending slots + scratch (per chunk when the chunks run
  // concurrently, else reused); plus one gather (sink output) buffer per chunk
  const size_t mb = p.max_chunk_bytes;
  const uint32_t scratch_sets = multi ? n : 1;
  ctx->msgs.reserve((scratch_sets * (n + 2) + n) * mb);
  std::vector<int> gslots(n, -1);
  std::vector<char> decoded(n, 0);  // chunk decoded into `out` by its fused sink
  uint32_t max_nsg = 0;
  for (uint32_t i = 0; i < n; ++i) max_nsg = std::max(max_nsg, p.lo[i + 1] - p.lo[i]);
  const bool need_acc = c.topology == DQ_BUTTERFLY;
  if (need_acc) ctx->accs.reserve(static_cast<size_t>(scratch_sets) * n * max_nsg * 256);
  std::vector<uint8_t> host_soa, host_ref;
  uint64_t H = 0xcbf29ce484222325ULL;
  // Permutation slices: every simulated hop of a chunk draws from the same per-entry
  // Fisher-Yates permutation (keyed by chunk, super-group, entry; random.cpp:53-90) and
  // only reads a different slot of it, so the chunk's first compression computes the
  // whole permutation once and stores slot s's pi (4 bits per entry) into slice s, which
  // hop s reads - the same slices the distributed ring ships to the rank running hop s.
  const bool use_pc = c.correlated && n >= 2 && n <= 8 && p.a.gs == 16 && p.a.ss == 2 && p.a.gshift == 1;
  const size_t slice_words = static_cast<size_t>(max_nsg) * 32;  // u32 per (super-group, lane)
  if (use_pc) ctx->pcache.reserve(scratch_sets * (n - 1) * slice_words);

  for (uint32_t ch = 0; ch < n; ++ch) {
    const cudaStream_t cst = multi ? ctx->cstreams[ch % nstreams] : st;  // this chunk's stream
    const size_t set = multi ? ch : 0;                                    // its scratch set
    auto slice = [&](uint32_t s) { return ctx->pcache.p + (set * (n - 1) + s - 1) * slice_words; };
    const Plan plan = make_plan(n, ch, c.topology);
    const Layout L = chunk_layout(p.a, p.lo[ch], p.lo[ch + 1]);
    CodecArgs base = base_args(c, ch);
    base.L = L;
    base.counts = async ? ctx->counts.p : nullptr;
    base.first_sg = p.lo[ch];
    base.perm = ctx->perm.p;
    base.gmean = ctx->pmean.p;
    base.d = d;
    base.n_slots = plan.n_slots;
    std::vector<int> pend_slot(n, -1), last_in(n, -1);
    std::vector<char> has_acc(n, 0);
    for (size_t e = 0; e < plan.red.size(); ++e) last_in[plan.red[e].rcv] = static_cast<int>(e);
    std::vector<int> free_slots;
    for (int k = static_cast<int>(n) + 1; k >= 0; --k) free_slots.push_back(k);
    const int gather_dst = static_cast<int>(scratch_sets * (n + 2) + ch);  // this chunk's sink output lives here
    auto slot_ptr = [&](int k) {
      return ctx->msgs.p + (k < static_cast<int>(n + 2) ? set * (n + 2) + k : static_cast<size_t>(k)) * mb;
    };
    auto acc_ptr = [&](uint32_t w) { return ctx->accs.p + (set * n + w) * max_nsg * 256; };
    uint64_t hsh = 0xcbf29ce484222325ULL;
    auto hash_msg = [&](const uint8_t* dmsg, int times_fresh_first) {
      if (!collect_wire) return;
      const size_t sb = L.bytes();
      host_soa.resize(sb);
      host_ref.resize(sb + 24);
      DQ_CUDA(cudaMemcpyAsync(host_soa.data(), dmsg, sb, cudaMemcpyDeviceToHost, st));
      DQ_CUDA(cudaStreamSynchronize(st));
      to_reference(host_soa.data(), ch, L, host_ref.data());
      for (int t = 0; t < times_fresh_first; ++t) hsh = fnv1a(host_ref.data(), host_ref.size(), hsh);
    };
    auto operand = [&](uint32_t w, CodecArgs& a) -> int {  // 0 gather raw, 1 accumulator
      if (has_acc[w]) {
        a.acc_in = acc_ptr(w);
        return 1;
      }
      a.x = xs[w];
      return 0;
    };
    int gather_slot = -1;
    for (size_t e = 0; e < plan.red.size(); ++e) {
      const Event ev = plan.red[e];
      const int os = free_slots.back();
      free_slots.pop_back();
      CodecArgs a = base;
      a.slot = ev.slot;
      a.out = slot_ptr(os);
      const int src = operand(ev.snd, a);
      const bool dar = pend_slot[ev.snd] >= 0;
      if (dar) a.in = slot_ptr(pend_slot[ev.snd]);
      if (use_pc) {  // event 0 (slot 0) is the chunk's first (leaf) compression
        a.pc_mode = e == 0 ? 3 : 4;
        if (e == 0)
          for (uint32_t s = 1; s < plan.n_slots; ++s) a.pin_out[s] = slice(s);
        else
          a.pin = slice(ev.slot);
      }
      timed(ctx, dar ? K_DAR : K_LEAF, quant_bytes(L, dar), cst, [&] { launch_quant(a, src, dar, cst); });
      if (dar) {
        free_slots.push_back(pend_slot[ev.snd]);
        pend_slot[ev.snd] = -1;
      }
      if (!async) account(info, L, true);
      hash_msg(slot_ptr(os), 1);
      const uint32_t r = ev.rcv;
      if (static_cast<int>(e) == last_in[r] && r != plan.sink) {
        pend_slot[r] = os;
      } else if (static_cast<int>(e) == last_in[r] && r == plan.sink) {
        // fused sink: compress(dec(last) + buf[sink]) at the sink slot (== DA then compress)
        const int gs = gather_dst;
        CodecArgs g = base;
        g.slot = plan.sink_slot;
        g.out = slot_ptr(gs);
        g.in = slot_ptr(os);
        const int gsrc = operand(r, g);
        if (use_pc) {
          g.pc_mode = 4;
          g.pin = slice(plan.sink_slot);
        }
        g.dec_out = out;  // fused decode of the chunk into the output where a variant exists
        decoded[ch] = launch_quant_dec(g, gsrc, false, cst, false);
        timed(ctx, K_DAR, quant_bytes(L, true) + (decoded[ch] ? 1032.0 * L.nsg : 0.0), cst, [&] {
          if (!decoded[ch]) launch_quant(g, gsrc, true, cst);
          else launch_quant_dec(g, gsrc, false, cst);
        });
        free_slots.push_back(os);
        gather_slot = gs;
      } else {
        CodecArgs g = base;
        g.in = slot_ptr(os);
        const int gsrc = operand(r, g);
        g.acc_out = acc_ptr(r);
        timed(ctx, K_DA, 2048.0 * L.nsg + L.bytes(), cst, [&] { launch_da(g, gsrc, cst); });
        has_acc[r] = 1;
        free_slots.push_back(os);
      }
    }
    DQ_CUDA(cudaGetLastError());
    // all-gather of the sink's bytes: hashed once per forward (engine.cpp:219-229)
    if (collect_wire) hash_msg(slot_ptr(gather_slot), static_cast<int>(plan.n_gat));
    if (!async) {
      for (uint32_t g = 0; g < plan.n_gat; ++g) account(info, L, g == 0);
      info->stats_bits += static_cast<uint64_t>(plan.red.size() + plan.n_gat) * 64ull * L.nsg;
    }
    gslots[ch] = gather_slot;
    H ^= hsh + 0x9e3779b97f4a7c15ULL + (H << 6) + (H >> 2);
  }
  if (collect_wire) info->wire_hash = H;
  if (multi) {  // join the chunk streams
    for (uint32_t k = 0; k < nstreams; ++k) {
      DQ_CUDA(cudaEventRecord(ctx->cjoin[k], ctx->cstreams[k]));
      DQ_CUDA(cudaStreamWaitEvent(st, ctx->cjoin[k], 0));
    }
  }
  {  // the chunks whose sink had no fused decode
    GatherArgs g{};
    set_format(g, ctx->cfg);
    g.use_hi = 1;
    g.counts = async ? ctx->counts.p : nullptr;
    uint32_t max_nsg_g = 0, k = 0;
    double gbytes = 0;
    for (uint32_t ch = 0; ch < n; ++ch) {
      if (decoded[ch]) continue;
      const Layout L = chunk_layout(p.a, p.lo[ch], p.lo[ch + 1]);
      g.in[k] = ctx->msgs.p + static_cast<size_t>(gslots[ch]) * mb;
      g.lo[k] = p.lo[ch];
      g.hi[k] = p.lo[ch + 1];
      g.n8[k] = L.n8;
      g.n4[k] = L.n4;
      max_nsg_g = std::max(max_nsg_g, L.nsg);
      gbytes += 1032.0 * L.nsg + L.bytes();
      ++k;
    }
    g.perm = ctx->perm.p;
    g.gmean = ctx->pmean.p;
    g.out = out;
    g.d = d;
    g.n_workers_f = static_cast<float>(n);
    g.uniform_books = c.non_uniform ? 0 : 1;
    if (k) timed(ctx, K_DECODE, gbytes, st, [&] { launch_gather_decode(g, k, max_nsg_g, st); });
    DQ_CUDA(cudaGetLastError());
  }
  DQ_CUDA(cudaEventRecord(ctx->ev1, st));
  if (flags & DQ_SIM_NO_METRICS) {  // asynchronous return: timing resolved at the next sync point
    finish_async(ctx, info, st);
    return;
  }
  // vNMSE against the fp64 sum of the inputs (metrics, not part of the timed path)
  ctx->vn.reserve(2);
  if (!ctx->h_vn) DQ_CUDA(cudaMallocHost(&ctx->h_vn, 2 * sizeof(double)));
  DQ_CUDA(cudaMemsetAsync(ctx->vn.p, 0, 2 * sizeof(double), st));
  launch_vnmse(xs, n, out, d, ctx->vn.p, st);
  DQ_CUDA(cudaMemcpyAsync(ctx->h_vn, ctx->vn.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaStreamSynchronize(st));
  harvest(ctx);
  if (async) finish_info(ctx, info);
  info->mse = ctx->h_vn[0] / static_cast<double>(d);
  info->vnmse = ctx->h_vn[1] > 0 ? ctx->h_vn[0] / ctx->h_vn[1] : 0.0;
  float ms = 0.f;
  DQ_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  info->ms_total = ms;
}

// ---------------------------------------------------------- distributed
// One rank per GPU.  Events of every chunk are grouped into stages (ring: the
// hop index; butterfly: the halving stage) and each stage is one NCCL group of
// point-to-point sends/receives of compressed chunks over NVLink, bracketed by
// the fused codec kernels: outgoing = leaf compress or DAR of the held last
// parent, incoming = held (last parent), DA'd (earlier parents) or, at the
// chunk's sink, fused DAR at the sink slot.  The all-gather forwards the sink
// bytes verbatim (engine.cpp:219-229) as one group of n-1 sends and receives.
// Ring reduce-scatter with per-piece software pipelining (tile-aligned pieces of
// each chunk): at hop h rank r DARs chunk r-1-h piece by piece on the compute
// stream, and the comm stream ships each finished piece to r+1 while receiving
// the same piece of the next hop's chunk from r-1, so NVLink transfers overlap
// the fused kernels.  Returns the device pointer of this rank's sink chunk.
struct Piece {
  uint32_t sg0, sg1;     // super-group range (chunk-local, tile aligned)
  uint64_t b0, b1;       // byte range in the chunk layout
};
std::vector<Piece> split_pieces(const Layout& L, int want) {
  std::vector<Piece> v;
  const uint32_t tiles = L.tiles();
  const uint32_t per = tiles == 0 ? 1 : (tiles + want - 1) / want;
  for (uint32_t t = 0; t < tiles; t += per) {
    const uint32_t t1 = t + per < tiles ? t + per : tiles;
    const uint32_t s0 = t * kTileSG, s1 = t1 * kTileSG < L.nsg ? t1 * kTileSG : L.nsg;
    v.push_back({s0, s1, L.tile_offset(t), L.tile_offset(t1)});
  }
  if (v.empty()) v.push_back({0, 0, 0, 0});
  return v;
}

// A piece as a standalone chunk: its own run lengths, first_sg and base pointers.
CodecArgs piece_args(const CodecArgs& base, const Layout& L, const Piece& p) {
  CodecArgs a = base;
  auto overlap = [](uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
    const uint32_t l = a0 > b0 ? a0 : b0, h = a1 < b1 ? a1 : b1;
    return h > l ? h - l : 0u;
  };
  a.L.nsg = p.sg1 - p.sg0;
  a.L.n8 = overlap(p.sg0, p.sg1, 0, L.n8);
  a.L.n4 = overlap(p.sg0, p.sg1, L.n8, L.n8 + L.n4);
  a.first_sg = base.first_sg + p.sg0;
  return a;
}

uint8_t* ring_pipelined(dq_ctx* ctx, const Prepared& pr, const std::vector<CodecArgs>& bases,
                        const std::vector<Layout>& lays, size_t mb, dq_round_info* info, cudaStream_t st) {
  const uint32_t n = ctx->cfg.n_workers, me = static_cast<uint32_t>(ctx->rank);
  const uint32_t right = (me + 1) % n, left = (me + n - 1) % n;
  if (!ctx->cs) DQ_CUDA(cudaStreamCreateWithFlags(&ctx->cs, cudaStreamNonBlocking));
  // pieces per chunk: enough to overlap transfers with the fused kernels on big
  // chunks, one on small ones (each piece costs a launch + an NCCL group).  Derived
  // from the round-global max chunk size, so every rank splits identically.
  const size_t piece_target = 8u << 20;
  const int P = static_cast<int>(std::max<size_t>(1, std::min<size_t>(ctx->pieces, mb / piece_target)));
  const size_t nev = 2ull * n * ctx->pieces + 2;
  while (ctx->pipe_ev.size() < nev) {
    cudaEvent_t e;
    DQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->pipe_ev.push_back(e);
  }
  // buffers: out[2] (hop parity), in[2], sink
  auto obuf = [&](uint32_t h) { return ctx->msgs.p + static_cast<size_t>(h & 1) * mb; };
  auto ibuf = [&](uint32_t h) { return ctx->msgs.p + static_cast<size_t>(2 + (h & 1)) * mb; };
  uint8_t* sink = ctx->msgs.p + 4ull * mb;
  auto ev_comp = [&](uint32_t h, int p) { return ctx->pipe_ev[(static_cast<size_t>(h) * P + p) * 2]; };
  auto ev_recv = [&](uint32_t h, int p) { return ctx->pipe_ev[(static_cast<size_t>(h) * P + p) * 2 + 1]; };
  cudaEvent_t start = ctx->pipe_ev[nev - 1];
  DQ_CUDA(cudaEventRecord(start, st));
  DQ_CUDA(cudaStreamWaitEvent(ctx->cs, start, 0));  // comm work of this round follows its prologue
  for (uint32_t h = 0; h < n; ++h) {
    const uint32_t ch = (me + 2 * n - 1 - h) % n;  // chunk handled at hop h (sink at h = n-1)
    const Layout& L = lays[ch];
    const std::vector<Piece> pcs = split_pieces(L, P);
    for (int p = 0; p < static_cast<int>(pcs.size()); ++p) {
      CodecArgs a = piece_args(bases[ch], L, pcs[p]);
      a.slot = h;
      a.out = (h + 1 < n ? obuf(h) : sink) + pcs[p].b0;
      if (h > 0) {
        DQ_CUDA(cudaStreamWaitEvent(st, ev_recv(h, p), 0));
        a.in = ibuf(h) + pcs[p].b0;
      }
      const bool dar = h > 0;
      timed(ctx, dar ? K_DAR : K_LEAF, quant_bytes(a.L, dar), st, [&] { launch_quant(a, 0, dar, st); });
      DQ_CUDA(cudaEventRecord(ev_comp(h, p), st));
      if (h + 1 < n) {
        // ship piece p of this hop's result; receive piece p of the next hop's chunk
        const uint32_t nch = (me + 2 * n - 2 - h) % n;
        const std::vector<Piece> npcs = split_pieces(lays[nch], P);
        DQ_CUDA(cudaStreamWaitEvent(ctx->cs, ev_comp(h, p), 0));
        DQ_NCCL(ncclGroupStart());
        DQ_NCCL(ncclSend(obuf(h) + pcs[p].b0, pcs[p].b1 - pcs[p].b0, ncclUint8, right, ctx->comm, ctx->cs));
        if (p < static_cast<int>(npcs.size()))
          DQ_NCCL(ncclRecv(ibuf(h + 1) + npcs[p].b0, npcs[p].b1 - npcs[p].b0, ncclUint8, left, ctx->comm, ctx->cs));
        DQ_NCCL(ncclGroupEnd());
        DQ_CUDA(cudaEventRecord(ev_recv(h + 1, p), ctx->cs));
        // piece counts of consecutive chunks may differ: receive the tail pieces here
        if (p + 1 == static_cast<int>(pcs.size()))
          for (int q = p + 1; q < static_cast<int>(npcs.size()); ++q) {
            DQ_NCCL(ncclRecv(ibuf(h + 1) + npcs[q].b0, npcs[q].b1 - npcs[q].b0, ncclUint8, left, ctx->comm, ctx->cs));
            DQ_CUDA(cudaEventRecord(ev_recv(h + 1, q), ctx->cs));
          }
      }
    }
  }
  // the compute stream must not run ahead of the last sends (buffers are reused next round)
  cudaEvent_t done = ctx->pipe_ev[nev - 2];
  DQ_CUDA(cudaEventRecord(done, ctx->cs));
  DQ_CUDA(cudaStreamWaitEvent(st, done, 0));
  (void)pr;
  return sink;
}

// (Re)build the peer region when this round's chunks do not fit.  Collective: every
// rank takes the same decision from round-global sizes at the same point of the
// same round, after the stats all-gather has ordered all of every peer's previous
// round (its last stores into this rank's region) before it.  If any rank cannot map
// a peer, every rank falls back to the NCCL transport.
// Export `base` by CUDA IPC and map every other rank's region (collective: one NCCL
// all-gather of the 64-byte handles, then an all-reduce of the per-rank success so every
// rank takes the same decision).  peer[me] = base.
bool ipc_map(dq_ctx* ctx, uint8_t* base, std::vector<uint8_t*>& peer, cudaStream_t st) {
  const uint32_t n = ctx->cfg.n_workers, me = static_cast<uint32_t>(ctx->rank);
  ctx->ipc.reserve(static_cast<size_t>(n) * (sizeof(cudaIpcMemHandle_t) + 4));
  cudaIpcMemHandle_t h;
  DQ_CUDA(cudaIpcGetMemHandle(&h, base));
  const size_t hs = sizeof(h);
  DQ_CUDA(cudaMemcpyAsync(ctx->ipc.p + me * hs, &h, hs, cudaMemcpyHostToDevice, st));
  DQ_NCCL(ncclAllGather(ctx->ipc.p + me * hs, ctx->ipc.p, hs, ncclUint8, ctx->comm, st));
  std::vector<uint8_t> all(n * hs);
  DQ_CUDA(cudaMemcpyAsync(all.data(), ctx->ipc.p, n * hs, cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaStreamSynchronize(st));
  peer.assign(n, nullptr);
  int ok = 1;
  for (uint32_t q = 0; q < n; ++q) {
    if (q == me) {
      peer[q] = base;
      continue;
    }
    cudaIpcMemHandle_t hq;
    std::memcpy(&hq, all.data() + q * hs, hs);
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, hq, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    peer[q] = static_cast<uint8_t*>(ptr);
  }
  int* dok = reinterpret_cast<int*>(ctx->ipc.p + n * hs);
  DQ_CUDA(cudaMemcpyAsync(dok, &ok, sizeof ok, cudaMemcpyHostToDevice, st));
  DQ_NCCL(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, ctx->comm, st));
  DQ_CUDA(cudaMemcpyAsync(&ok, dok, sizeof ok, cudaMemcpyDeviceToHost, st));
  DQ_CUDA(cudaStreamSynchronize(st));
  if (!ok) dq_ctx::close_map(peer, base);
  return ok != 0;
}

void peer_fallback(dq_ctx* ctx) {
  ctx->transport = DQ_TRANSPORT_NCCL;
  std::fprintf(stderr, "dynamiq_b200: peer mapping failed on some rank; using NCCL p2p\n");
}

bool peer_setup(dq_ctx* ctx, size_t mb, uint32_t max_nsg, uint32_t ninbox, uint32_t npin, cudaStream_t st) {
  PeerMem& pm = ctx->pm;
  const uint32_t n = ctx->cfg.n_workers;
  if (pm.base && pm.n == n && pm.ninbox == ninbox && pm.npin == npin && mb <= pm.cap && max_nsg <= pm.cap_units)
    return true;
  DQ_CUDA(cudaStreamSynchronize(st));
  ctx->close_peers();
  uint8_t* old = pm.base;
  pm.base = nullptr;
  pm.n = n;
  pm.ninbox = ninbox;
  pm.npin = npin;
  pm.cap = (mb + mb / 4 + 4095) & ~static_cast<size_t>(4095);
  pm.cap_units = max_nsg + max_nsg / 4 + 64;
  DQ_CUDA(cudaMalloc(&pm.base, pm.total()));
  DQ_CUDA(cudaMemsetAsync(pm.base + pm.flags(), 0, pm.pins() - pm.flags(), st));
  const bool ok = ipc_map(ctx, pm.base, pm.peer, st);
  if (old) DQ_CUDA(cudaFree(old));  // every rank closed its mapping of it before the handle all-gather
  if (!ok) {
    DQ_CUDA(cudaFree(pm.base));
    pm.base = nullptr;
    peer_fallback(ctx);
  }
  return ok;
}

// The statistics exchange area (collective, same decision on every rank: T and n are
// round-global).  Sized by capacity with headroom (rows stride sm.T >= the round's T), so
// the varying bucket sizes of a DDP step reuse it; rebuilt only when n changes or T outgrows it.
bool stats_setup(dq_ctx* ctx, uint32_t T, cudaStream_t st) {
  StatsMem& sm = ctx->sm;
  const uint32_t n = ctx->cfg.n_workers;
  if (sm.base && sm.n == n && T <= sm.T) return true;
  DQ_CUDA(cudaStreamSynchronize(st));
  dq_ctx::close_map(sm.peer, sm.base);
  uint8_t* old = sm.base;
  sm.base = nullptr;
  sm.n = n;
  sm.T = std::max<uint32_t>(T + T / 4 + 64, 4096u);
  DQ_CUDA(cudaMalloc(&sm.base, sm.total()));
  DQ_CUDA(cudaMemsetAsync(sm.base + 2 * sm.rows(), 0, sm.total() - 2 * sm.rows(), st));
  ctx->sdone.reserve(1);
  DQ_CUDA(cudaMemsetAsync(ctx->sdone.p, 0, sizeof(unsigned int), st));
  if (!ctx->dev_epoch.p) {  // every rank starts at 0 and advances once per round
    ctx->dev_epoch.reserve(1);
    DQ_CUDA(cudaMemsetAsync(ctx->dev_epoch.p, 0, sizeof(uint32_t), st));
  }
  const bool ok = ipc_map(ctx, sm.base, sm.peer, st);
  if (old) DQ_CUDA(cudaFree(old));
  if (!ok) {
    DQ_CUDA(cudaFree(sm.base));
    sm.base = nullptr;
    peer_fallback(ctx);
  }
  return ok;
}

// Ring over peer memory: at hop h rank r runs the fused kernel on chunk r-1-h, reading
// its inbox h-1 unit by unit as the left neighbour's hop h-1 kernel raises the unit
// flags and storing its own output straight into the right neighbour's inbox h
// (NVLink stores, no staging copy, no NCCL kernel); consecutive hops of neighbouring
// ranks therefore overlap at unit granularity.  The sink (hop n-1) stores its chunk
// into gather slot r of every rank - the all-gather - and one decode launch per rank
// consumes all n gather slots as their units land.
void peer_gather_decode(dq_ctx* ctx, const Prepared& p, const std::vector<Layout>& lays,
                        const std::vector<char>& decoded, float* out, size_t d, cudaStream_t st);


// Fused own-chunk decode in the peer sinks (launch_quant_dec) only up to this many ranks.
// Measured at d = 2^28 per rank (profiles/r1_multi_gpu.md): N = 2 the gather decode is
// HBM-bound and fusing saves 0.07 ms per round (2.73 -> 2.65 ms); N = 4 the gather decode
// is paced by the remote sinks' arrival, the own chunk's decode hides inside that wait,
// and the longer sink costs 0.05 ms (3.15 -> 3.20 ms ring, 3.32 -> 3.36 butterfly).
constexpr uint32_t kFuseDecodeMaxRanks = 2;

// Ring permutation slices (peer transport, correlated rounding, 2 <= n <= 8): every
// entry's Fisher-Yates permutation is computed once per round, by the chunk's leaf (whose
// slot-0 trace draws all n-1 swaps anyway), and hop h's pi[h] is stored into the rank that
// runs hop h; the later hops read 4 bits per entry instead of re-tracing the permutation.
uint32_t ring_pins(const dq_config& c, const Plan& plan) {
  const uint32_t n = c.n_workers;
  return c.topology == DQ_RING && c.correlated && n >= 2 && n <= 8 && plan.n_slots == n ? n - 1 : 0;
}

void ring_peer(dq_ctx* ctx, const Prepared& p, const std::vector<CodecArgs>& bases,
               const std::vector<Layout>& lays, float* out, size_t d, cudaStream_t st) {
  const uint32_t n = ctx->cfg.n_workers, me = static_cast<uint32_t>(ctx->rank);
  const uint32_t right = (me + 1) % n;
  PeerMem& pm = ctx->pm;
  std::vector<char> decoded(n, 0);
  for (uint32_t h = 0; h < n; ++h) {
    const uint32_t ch = (me + 2 * n - 1 - h) % n;  // sink at h = n-1
    CodecArgs a = bases[ch];
    a.slot = h;
    a.unit = peer_unit(lays[ch].nsg);
    a.epoch_ptr = ctx->dev_epoch.p;
    if (h > 0) {
      a.in = pm.base + pm.inbox(h - 1);
      a.in_flags = reinterpret_cast<const uint32_t*>(pm.base + pm.iflag(h - 1));
    }
    if (pm.npin) {  // hop s of this chunk runs on rank me + s - h
      if (h == 0) {
        a.pc_mode = 3;
        for (uint32_t s = 1; s < n; ++s)
          a.pin_out[s] = reinterpret_cast<uint32_t*>(pm.peer[(me + s) % n] + pm.pin(s - 1));
      } else {
        a.pc_mode = 4;
        a.pin = reinterpret_cast<const uint32_t*>(pm.base + pm.pin(h - 1));
      }
    }
    if (h + 1 < n) {
      a.outs[0] = pm.peer[right] + pm.inbox(h);
      a.out_flags[0] = reinterpret_cast<uint32_t*>(pm.peer[right] + pm.iflag(h));
      a.n_outs = 1;
    } else {
      for (uint32_t k = 0; k < n; ++k) {  // remote copies first, own slot last
        const uint32_t q = (me + 1 + k) % n;
        a.outs[k] = pm.peer[q] + pm.gather(me);
        a.out_flags[k] = reinterpret_cast<uint32_t*>(pm.peer[q] + pm.gflag(me));
      }
      a.n_outs = static_cast<int>(n);
    }
    const bool dar = h > 0;
    if (h + 1 == n && n <= kFuseDecodeMaxRanks) {  // the sink also decodes its record into the output
      a.dec_out = out;
      decoded[ch] = launch_quant_dec(a, 0, true, st, false);
    }
    const double ob = (decoded[ch] ? 1032.0 * lays[ch].nsg : 0.0) +
                      (pm.npin ? 128.0 * lays[ch].nsg * (h == 0 ? n - 1 : 1) : 0.0);  // + permutation slices
    timed(ctx, dar ? K_DAR : K_LEAF, quant_bytes(lays[ch], dar) + ob, st, [&] {
      if (!decoded[ch]) launch_quant_peer(a, 0, dar, st);
      else launch_quant_dec(a, 0, true, st);
    });
  }
  peer_gather_decode(ctx, p, lays, decoded, out, d, st);
}

// Every rank decodes the n gather slots of this round's parity into the output, unit by
// unit as the sinks' stores land (its own slot is complete: its sink ran earlier on st),
// except the chunks its own sink already decoded (decoded[c], launch_quant_dec).
void peer_gather_decode(dq_ctx* ctx, const Prepared& p, const std::vector<Layout>& lays,
                        const std::vector<char>& decoded, float* out, size_t d, cudaStream_t st) {
  const uint32_t n = ctx->cfg.n_workers, me = static_cast<uint32_t>(ctx->rank);
  PeerMem& pm = ctx->pm;
  GatherArgs g{};
  set_format(g, ctx->cfg);
  g.use_hi = 1;
  g.counts = p.a.async ? ctx->counts.p : nullptr;
  uint32_t max_nsg = 0, k = 0;
  double gbytes = 0;
  for (uint32_t c = 0; c < n; ++c) {
    if (decoded[c]) continue;
    g.in[k] = pm.base + pm.gather(c);
    g.lo[k] = p.lo[c];
    g.hi[k] = p.lo[c + 1];
    g.n8[k] = lays[c].n8;
    g.n4[k] = lays[c].n4;
    g.flags[k] = c == me ? nullptr : reinterpret_cast<const uint32_t*>(pm.base + pm.gflag(c));
    g.unit[k] = peer_unit(lays[c].nsg);
    max_nsg = std::max(max_nsg, lays[c].nsg);
    gbytes += 1032.0 * lays[c].nsg + lays[c].bytes();
    ++k;
  }
  if (!k) return;
  g.epoch_ptr = ctx->dev_epoch.p;
  g.perm = ctx->perm.p;
  g.gmean = ctx->pmean.p;
  g.out = out;
  g.d = d;
  g.n_workers_f = static_cast<float>(n);
  g.uniform_books = ctx->cfg.non_uniform ? 0 : 1;
  timed(ctx, K_DECODE, gbytes, st, [&] { launch_gather_decode(g, k, max_nsg, st); });
}

// halving stage of a butterfly reduce event (topology.cpp:46-54): partner bit n >> (stage + 1)
uint32_t butterfly_stage(uint32_t n, const Event& ev) {
  const uint32_t bit = ev.snd ^ ev.rcv;
  uint32_t l = 0;
  while ((n >> (l + 1)) != bit) ++l;
  return l;
}

// Butterfly over peer memory: at stage s every sender's fused kernel stores its chunk
// message into the receiver's inbox s * n + c unit by unit; a receiver's last parent is
// "held" (read in place, unit by unit, by its own later DAR), earlier parents are
// decompress-accumulated as their units land (k_da_peer), and the sink's final DAR
// stores into every rank's gather slot c.  Same events, slots and association order as
// the reference schedule (topology.cpp:32-70, engine.cpp:162-216).
void butterfly_peer(dq_ctx* ctx, const Prepared& p, const std::vector<CodecArgs>& bases,
                    const std::vector<Layout>& lays, const std::vector<Plan>& plans, uint32_t max_nsg, float* out,
                    size_t d, cudaStream_t st) {
  const uint32_t n = ctx->cfg.n_workers, me = static_cast<uint32_t>(ctx->rank);
  uint32_t stages = 0;
  while ((1u << stages) < n) ++stages;
  PeerMem& pm = ctx->pm;
  ctx->accs.reserve(static_cast<size_t>(n) * max_nsg * 256);
  auto acc_ptr = [&](uint32_t ch) { return ctx->accs.p + static_cast<size_t>(ch) * max_nsg * 256; };
  std::vector<int> held(n, -1);
  std::vector<char> has_acc(n, 0), decoded(n, 0);
  auto prep = [&](uint32_t ch) {
    CodecArgs a = bases[ch];
    a.unit = peer_unit(lays[ch].nsg);
    a.epoch_ptr = ctx->dev_epoch.p;
    return a;
  };
  auto operand = [&](uint32_t ch, CodecArgs& a) {
    if (!has_acc[ch]) return 0;
    a.acc_in = acc_ptr(ch);
    return 1;
  };
  auto inbox_in = [&](CodecArgs& a, uint32_t k) {
    a.in = pm.base + pm.inbox(k);
    a.in_flags = reinterpret_cast<const uint32_t*>(pm.base + pm.iflag(k));
  };
  for (uint32_t s = 0; s < stages; ++s) {
    for (uint32_t ch = 0; ch < n; ++ch)
      for (size_t e = 0; e < plans[ch].red.size(); ++e) {
        const Event& ev = plans[ch].red[e];
        if (ev.snd != me || butterfly_stage(n, ev) != s) continue;
        CodecArgs a = prep(ch);
        a.slot = ev.slot;
        const int src = operand(ch, a);
        const bool dar = held[ch] >= 0;
        if (dar) inbox_in(a, static_cast<uint32_t>(held[ch]));
        const uint32_t k = s * n + ch;
        a.outs[0] = pm.peer[ev.rcv] + pm.inbox(k);
        a.out_flags[0] = reinterpret_cast<uint32_t*>(pm.peer[ev.rcv] + pm.iflag(k));
        a.n_outs = 1;
        timed(ctx, dar ? K_DAR : K_LEAF, quant_bytes(lays[ch], dar), st, [&] { launch_quant_peer(a, src, dar, st); });
        held[ch] = -1;
      }
    for (uint32_t ch = 0; ch < n; ++ch) {
      const Plan& pl = plans[ch];
      size_t last = 0;
      for (size_t e = 0; e < pl.red.size(); ++e)
        if (pl.red[e].rcv == me) last = e;
      for (size_t e = 0; e < pl.red.size(); ++e) {
        const Event& ev = pl.red[e];
        if (ev.rcv != me || butterfly_stage(n, ev) != s) continue;
        const uint32_t k = s * n + ch;
        if (e == last && me != pl.sink) {
          held[ch] = static_cast<int>(k);  // consumed in place by this rank's next send of ch
          continue;
        }
        CodecArgs a = prep(ch);
        inbox_in(a, k);
        const int src = operand(ch, a);
        if (e == last) {  // sink: final DAR straight into every rank's gather slot ch
          a.slot = pl.sink_slot;
          for (uint32_t j = 0; j < n; ++j) {
            const uint32_t q = (me + 1 + j) % n;
            a.outs[j] = pm.peer[q] + pm.gather(ch);
            a.out_flags[j] = reinterpret_cast<uint32_t*>(pm.peer[q] + pm.gflag(ch));
          }
          a.n_outs = static_cast<int>(n);
          if (n <= kFuseDecodeMaxRanks) a.dec_out = out;  // and decoded into this rank's output
          decoded[ch] = launch_quant_dec(a, src, true, st, false);
          const double ob = decoded[ch] ? 1032.0 * lays[ch].nsg : 0.0;
          timed(ctx, K_DAR, quant_bytes(lays[ch], true) + ob, st, [&] {
            if (!decoded[ch]) launch_quant_peer(a, src, true, st);
            else launch_quant_dec(a, src, true, st);
          });
        } else {
          a.acc_out = acc_ptr(ch);
          timed(ctx, K_DA, 2048.0 * lays[ch].nsg + lays[ch].bytes(), st, [&] { launch_da_peer(a, src, st); });
          has_acc[ch] = 1;
        }
      }
    }
  }
  peer_gather_decode(ctx, p, lays, decoded, out, d, st);
}

// NCCL reports errors of enqueued work (a dead peer, a network failure) asynchronously
// (§5 failure detection): poll the communicator before each round and after the NCCL
// transport's last enqueue.
void check_nccl_async(dq_ctx* ctx) {
  if (!ctx->comm) return;
  ncclResult_t e = ncclSuccess;
  DQ_NCCL(ncclCommGetAsyncError(ctx->comm, &e));
  if (e != ncclSuccess && e != ncclInProgress)
    throw Error(DQ_ENCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(e));
}

void dist_round(dq_ctx* ctx, const float* x, size_t d, float* out, dq_round_info* info, cudaStream_t st) {
  const dq_config& c = ctx->cfg;
  const uint32_t n = c.n_workers, me = static_cast<uint32_t>(ctx->rank);
  *info = dq_round_info{};
  if (d == 0) invalid("empty gradient");
  if (n == 1) {
    if (out != x) DQ_CUDA(cudaMemcpyAsync(out, x, d * sizeof(float), cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (!ctx->comm) invalid("dq_comm_init has not been called");
  if (n != static_cast<uint32_t>(ctx->nranks)) invalid("n_workers must equal the communicator's rank count");
  check_nccl_async(ctx);  // a failure of an earlier round's NCCL work surfaces here
  if (reinterpret_cast<uintptr_t>(x) % 16 || reinterpret_cast<uintptr_t>(out) % 16)
    invalid("buffers must be 16-byte aligned");
  const uint32_t T = static_cast<uint32_t>((d + 255) / 256);
  ensure_books();
  if (!ctx->ev0) {
    DQ_CUDA(cudaEventCreate(&ctx->ev0));
    DQ_CUDA(cudaEventCreate(&ctx->ev1));
  }
  DQ_CUDA(cudaEventRecord(ctx->ev0, st));
  reserve_round(ctx, T, n);
  ctx->pending_red = StatsReduce{};
  const float* const* dxp = &x;
  // peer transport (default scale format): the round allocates asynchronously; the NCCL
  // transport and the ablation formats size their messages on the host (synchronous)
  const bool peer_pre = ctx->transport == DQ_TRANSPORT_PEER && n <= static_cast<uint32_t>(kMaxPeers) &&
                        c.group_size == 16 && c.hierarchical_scales;
  const bool fuse_red = small_alloc_round(ctx, T, peer_pre && async_alloc_ok(ctx, false));
  // (a) local stats into this rank's row, (b) all-gather rows, fixed-order fp64 reduce (H4).
  // Peer transport: the all-gather is fused into the statistics kernel (each block stores
  // its rows into every rank's exchange area over NVLink, the last block raises the row
  // flags) and the reduction waits for all rows' flags; this also orders every peer's
  // previous round before any store of this round into its regions.
  if (ctx->transport == DQ_TRANSPORT_PEER && n <= static_cast<uint32_t>(kMaxPeers) && stats_setup(ctx, T, st)) {
    StatsMem& sm = ctx->sm;
    StatsPeerArgs sp{};
    for (uint32_t q = 0; q < n; ++q) {
      sp.mean[q] = sm.mean(sm.peer[q], me);
      sp.sq[q] = sm.sq(sm.peer[q], me);
      sp.flag[q] = sm.flags(sm.peer[q]) + me;
    }
    sp.done = ctx->sdone.p;
    sp.n = n;
    sp.epoch = ctx->dev_epoch.p;  // advanced by the statistics kernel: this round's epoch
    timed(ctx, K_STATS, 4.0 * d + 8.0 * T * n, st, [&] { launch_stats_peer(dxp, d, T, sp, st); });
    if (fuse_red) {
      ctx->pending_red = StatsReduce{sm.mean(sm.base, 0), sm.sq(sm.base, 0), sm.flags(sm.base), ctx->dev_epoch.p, n,
                                     sm.T, ctx->gmean.p, ctx->gsq.p};
    } else {
      timed(ctx, K_REDUCE, 8.0 * (n + 1) * T, st, [&] {
        launch_reduce_stats_peer(sm.mean(sm.base, 0), sm.sq(sm.base, 0), sm.flags(sm.base), ctx->dev_epoch.p, n, T,
                                 sm.T, ctx->gmean.p, ctx->gsq.p, st);
      });
    }
  } else {
    float* my_mean = ctx->mean_all.p + static_cast<size_t>(me) * T;
    float* my_sq = ctx->sq_all.p + static_cast<size_t>(me) * T;
    timed(ctx, K_STATS, 4.0 * d + 8.0 * T, st, [&] { launch_stats(dxp, 1, d, T, my_mean, my_sq, st); });
    timed(ctx, K_NCCL, 8.0 * T * n, st, [&] {
      DQ_NCCL(ncclGroupStart());
      DQ_NCCL(ncclAllGather(my_mean, ctx->mean_all.p, T, ncclFloat, ctx->comm, st));
      DQ_NCCL(ncclAllGather(my_sq, ctx->sq_all.p, T, ncclFloat, ctx->comm, st));
      DQ_NCCL(ncclGroupEnd());
    });
    if (fuse_red)
      ctx->pending_red = StatsReduce{ctx->mean_all.p, ctx->sq_all.p, nullptr, nullptr, n, T, ctx->gmean.p, ctx->gsq.p};
    else
      timed(ctx, K_REDUCE, 8.0 * (n + 1) * T, st,
            [&] { launch_reduce_stats(ctx->mean_all.p, ctx->sq_all.p, n, T, ctx->gmean.p, ctx->gsq.p, st); });
  }
  DQ_CUDA(cudaGetLastError());
  Prepared p = prepare(ctx, T, st, peer_pre && async_alloc_ok(ctx, false));
  if (!p.a.async) fill_info_alloc(info, p);

  size_t mb = p.max_chunk_bytes;
  uint32_t max_nsg = 0;
  for (uint32_t i = 0; i < n; ++i) max_nsg = std::max(max_nsg, p.lo[i + 1] - p.lo[i]);
  // per chunk: outgoing, incoming, held, gather; accumulators for butterfly receivers

  auto buf = [&](int kind, uint32_t ch) { return ctx->msgs.p + (static_cast<size_t>(kind) * n + ch) * mb; };
  const bool need_acc = c.topology == DQ_BUTTERFLY;
  if (need_acc) ctx->accs.reserve(static_cast<size_t>(n) * max_nsg * 256);
  auto acc_ptr = [&](uint32_t ch) { return ctx->accs.p + static_cast<size_t>(ch) * max_nsg * 256; };

  std::vector<Plan> plans(n);
  std::vector<Layout> lays(n);
  std::vector<CodecArgs> bases(n);
  for (uint32_t ch = 0; ch < n; ++ch) {
    plans[ch] = make_plan(n, ch, c.topology);
    lays[ch] = chunk_layout(p.a, p.lo[ch], p.lo[ch + 1]);
    CodecArgs b = base_args(c, ch);
    b.L = lays[ch];
    b.counts = p.a.async ? ctx->counts.p : nullptr;
    b.first_sg = p.lo[ch];
    b.perm = ctx->perm.p;
    b.gmean = ctx->pmean.p;
    b.d = d;
    b.x = x;
    b.n_slots = plans[ch].n_slots;
    bases[ch] = b;
  }
  // peer transport: default scale format (the ablation formats run their generic kernels over NCCL)
  uint32_t stages = 0;
  while ((1u << stages) < n) ++stages;
  const uint32_t ninbox = c.topology == DQ_RING ? n - 1 : stages * n;
  if (peer_pre && peer_setup(ctx, mb, max_nsg, ninbox, ring_pins(c, plans[0]), st)) {
    if (c.topology == DQ_RING) ring_peer(ctx, p, bases, lays, out, d, st);
    else butterfly_peer(ctx, p, bases, lays, plans, max_nsg, out, d, st);
    if (!p.a.async) account_round(info, p.a, p.lo, n, c.topology);
    DQ_CUDA(cudaGetLastError());
    DQ_CUDA(cudaEventRecord(ctx->ev1, st));
    finish_async(ctx, info, st);
    return;
  }
  if (p.a.async) {  // peer mapping failed on some rank: bring the allocation to the host (NCCL sizes messages)
    DQ_CUDA(cudaStreamSynchronize(st));
    dq_round_info tmp{};
    finish_info(ctx, &tmp);
    p.a.async = false;
    p.a.u = tmp.u;
    p.a.n8 = tmp.n8;
    p.a.n4 = tmp.n4;
    p.a.n2 = tmp.n2;
    p.a.payload = tmp.payload_bits;
    p.a.passes = tmp.alloc_passes;
    ctx->rec.async = false;
    fill_info_alloc(info, p);
    mb = 0;
    for (uint32_t ch = 0; ch < n; ++ch) {
      lays[ch] = chunk_layout(p.a, p.lo[ch], p.lo[ch + 1]);
      bases[ch].L = lays[ch];
      bases[ch].counts = nullptr;
      mb = std::max<size_t>(mb, lays[ch].bytes());
    }
    mb = (mb + 255) / 256 * 256;
  }
  ctx->msgs.reserve(4ull * n * mb);
  uint8_t* mysink = buf(3, me);
  if (c.topology == DQ_RING) {
    mysink = ring_pipelined(ctx, p, bases, lays, mb, info, st);
  } else {
    // stage of event e of a chunk: ring -> e; butterfly -> halving stage
    auto stage_of = [&](uint32_t ch, size_t e) -> uint32_t {
      if (c.topology == DQ_RING) return static_cast<uint32_t>(e);
      const Event& ev = plans[ch].red[e];
      const uint32_t bit = ev.snd ^ ev.rcv;
      uint32_t stages = 0;
      while ((1u << stages) < n) ++stages;
      uint32_t l = 0;
      while ((1u << (stages - 1 - l)) != bit) ++l;
      return l;
    };
    uint32_t n_stages = 0;
    for (uint32_t ch = 0; ch < n; ++ch)
      for (size_t e = 0; e < plans[ch].red.size(); ++e) n_stages = std::max(n_stages, stage_of(ch, e) + 1);
    std::vector<char> held(n, 0), has_acc(n, 0);
    auto operand = [&](uint32_t ch, CodecArgs& a) -> int {
      if (has_acc[ch]) {
        a.acc_in = acc_ptr(ch);
        return 1;
      }
      return 0;
    };
    for (uint32_t s = 0; s < n_stages; ++s) {
      struct Io { uint32_t ch; size_t e; };
      std::vector<Io> sends, recvs;
      for (uint32_t ch = 0; ch < n; ++ch)
        for (size_t e = 0; e < plans[ch].red.size(); ++e) {
          if (stage_of(ch, e) != s) continue;
          if (plans[ch].red[e].snd == me) sends.push_back({ch, e});
          if (plans[ch].red[e].rcv == me) recvs.push_back({ch, e});
        }
      for (const Io& io : sends) {
        CodecArgs a = bases[io.ch];
        a.slot = plans[io.ch].red[io.e].slot;
        a.out = buf(0, io.ch);
        const int src = operand(io.ch, a);
        if (held[io.ch]) a.in = buf(2, io.ch);
        const bool dar = held[io.ch] != 0;
        timed(ctx, dar ? K_DAR : K_LEAF, quant_bytes(lays[io.ch], dar), st, [&] { launch_quant(a, src, dar, st); });
        held[io.ch] = 0;
      }
      DQ_CUDA(cudaGetLastError());
      double xbytes = 0;
      for (const Io& io : sends) xbytes += lays[io.ch].bytes();
      timed(ctx, K_NCCL, xbytes, st, [&] {
        DQ_NCCL(ncclGroupStart());
        for (const Io& io : sends)
          DQ_NCCL(ncclSend(buf(0, io.ch), lays[io.ch].bytes(), ncclUint8, plans[io.ch].red[io.e].rcv, ctx->comm, st));
        for (const Io& io : recvs)
          DQ_NCCL(ncclRecv(buf(1, io.ch), lays[io.ch].bytes(), ncclUint8, plans[io.ch].red[io.e].snd, ctx->comm, st));
        DQ_NCCL(ncclGroupEnd());
      });
      for (const Io& io : recvs) {
        const Plan& pl = plans[io.ch];
        size_t last = 0;
        for (size_t e = 0; e < pl.red.size(); ++e)
          if (pl.red[e].rcv == me) last = e;
        CodecArgs a = bases[io.ch];
        a.in = buf(1, io.ch);
        if (io.e == last && me != pl.sink) {
          DQ_CUDA(cudaMemcpyAsync(buf(2, io.ch), buf(1, io.ch), lays[io.ch].bytes(), cudaMemcpyDeviceToDevice, st));
          held[io.ch] = 1;
        } else if (io.e == last) {
          a.slot = pl.sink_slot;
          a.out = buf(3, io.ch);
          const int src = operand(io.ch, a);
          timed(ctx, K_DAR, quant_bytes(lays[io.ch], true), st, [&] { launch_quant(a, src, true, st); });
        } else {
          const int src = operand(io.ch, a);
          a.acc_out = acc_ptr(io.ch);
          timed(ctx, K_DA, 2048.0 * lays[io.ch].nsg + lays[io.ch].bytes(), st, [&] { launch_da(a, src, st); });
          has_acc[io.ch] = 1;
        }
      }
      DQ_CUDA(cudaGetLastError());
    }
  }
  // all-gather of the sink-compressed chunks (sink of chunk ch is rank ch), overlapped
  // with decode: the bytes are forwarded verbatim (engine.cpp:219-229) peer by peer on
  // the comm stream (step k: send to me+k, receive from me-k over NVSwitch) while the
  // compute stream decodes every chunk that has arrived, fused with unpermute +
  // denormalize into the output.
  if (!ctx->cs) DQ_CUDA(cudaStreamCreateWithFlags(&ctx->cs, cudaStreamNonBlocking));
  while (ctx->pipe_ev.size() < 2ull * n * ctx->pieces + 4 + n) {
    cudaEvent_t e;
    DQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->pipe_ev.push_back(e);
  }
  cudaEvent_t* gev = ctx->pipe_ev.data() + 2ull * n * ctx->pieces + 4;
  auto decode_one = [&](uint32_t ch, const uint8_t* src) {
    GatherArgs g{};
    set_format(g, ctx->cfg);
    g.in[0] = src;
    g.lo[0] = p.lo[ch];
    g.lo[1] = p.lo[ch + 1];
    g.n8[0] = lays[ch].n8;
    g.n4[0] = lays[ch].n4;
    g.perm = ctx->perm.p;
    g.gmean = ctx->pmean.p;
    g.out = out;
    g.d = d;
    g.n_workers_f = static_cast<float>(n);
    g.uniform_books = c.non_uniform ? 0 : 1;
    timed(ctx, K_DECODE, 1032.0 * lays[ch].nsg + lays[ch].bytes(), st,
          [&] { launch_gather_decode(g, 1, lays[ch].nsg, st); });
  };
  DQ_CUDA(cudaEventRecord(gev[0], st));  // this rank's sink chunk is complete
  DQ_CUDA(cudaStreamWaitEvent(ctx->cs, gev[0], 0));
  // one all-to-all group: every peer link of the NVSwitch busy at once
  DQ_NCCL(ncclGroupStart());
  for (uint32_t k = 1; k < n; ++k) {
    const uint32_t to = (me + k) % n, from = (me + n - k) % n;
    DQ_NCCL(ncclSend(mysink, lays[me].bytes(), ncclUint8, to, ctx->comm, ctx->cs));
    DQ_NCCL(ncclRecv(buf(3, from), lays[from].bytes(), ncclUint8, from, ctx->comm, ctx->cs));
  }
  DQ_NCCL(ncclGroupEnd());
  DQ_CUDA(cudaEventRecord(gev[1], ctx->cs));
  decode_one(me, mysink);  // overlaps the exchange
  DQ_CUDA(cudaStreamWaitEvent(st, gev[1], 0));
  {
    GatherArgs g{};
    set_format(g, ctx->cfg);
    uint32_t k = 0, max_nsg_g = 0;
    double gbytes = 0;
    for (uint32_t ch = 0; ch < n; ++ch) {
      if (ch == me) continue;
      g.in[k] = buf(3, ch);
      g.lo[k] = p.lo[ch];  // chunks of this list are not adjacent: explicit ends in hi[]
      g.n8[k] = lays[ch].n8;
      g.n4[k] = lays[ch].n4;
      g.hi[k] = p.lo[ch + 1];
      max_nsg_g = std::max(max_nsg_g, lays[ch].nsg);
      gbytes += 1032.0 * lays[ch].nsg + lays[ch].bytes();
      ++k;
    }
    g.perm = ctx->perm.p;
    g.gmean = ctx->pmean.p;
    g.out = out;
    g.d = d;
    g.n_workers_f = static_cast<float>(n);
    g.uniform_books = c.non_uniform ? 0 : 1;
    g.use_hi = 1;
    timed(ctx, K_DECODE, gbytes, st, [&] { launch_gather_decode(g, k, max_nsg_g, st); });
  }
  for (uint32_t ch = 0; ch < n; ++ch) {
    for (uint32_t g = 0; g < plans[ch].n_gat; ++g) account(info, lays[ch], g == 0);
    for (size_t e = 0; e < plans[ch].red.size(); ++e) account(info, lays[ch], true);
    info->stats_bits += static_cast<uint64_t>(plans[ch].red.size() + plans[ch].n_gat) * 64ull * lays[ch].nsg;
  }
  DQ_CUDA(cudaGetLastError());
  check_nccl_async(ctx);
  DQ_CUDA(cudaEventRecord(ctx->ev1, st));
  finish_async(ctx, info, st);
}

}  // namespace
}  // namespace dq

// ====================================================================== C-ABI
extern "C" {

int dq_version(void) { return DQ_VERSION; }
int dq_build_flags(void) {
  int f = 0;
#if defined(DQ_DEBUG_CHECKS) && DQ_DEBUG_CHECKS
  f |= 1;
#endif
#if defined(DQ_SMALL_PHASES)
  f |= 2;
#endif
  return f;
}
const char* dq_last_error(void) { return g_err.c_str(); }

void dq_config_default(dq_config* c) {  // engine.hpp:22-43 defaults
  *c = dq_config{};
  c->n_workers = 4;
  c->group_size = 16;
  c->super_group_size = 256;
  c->budget_bits = 5.0;
  c->non_uniform = 1;
  c->variable_width = 1;
  c->hierarchical_scales = 1;
  c->correlated = 1;
  c->fixed_width = 4;
  c->allocator = DQ_ALLOC_FAST;
  c->topology = DQ_RING;
  c->codec = 0;
  c->seed = 1;
  c->round = 0;
  c->threads = 1;
}

int dq_ctx_create(const dq_config* cfg, int device, dq_ctx** out) {
  return guarded([&] {
    if (!cfg || !out) invalid("null argument");
    validate(*cfg);
    DQ_CUDA(cudaSetDevice(device));
    auto* c = new dq_ctx;
    c->cfg = *cfg;
    c->device = device;
    if (const char* t = std::getenv("DQ_TRANSPORT"))
      if (std::strcmp(t, "nccl") == 0) c->transport = DQ_TRANSPORT_NCCL;
    if (const char* t = std::getenv("DQ_SYNC_ALLOC"))
      if (std::strcmp(t, "1") == 0) c->async_alloc = false;
    if (const char* t = std::getenv("DQ_NO_SMALL_ALLOC"))
      if (std::strcmp(t, "1") == 0) c->no_small_alloc = true;
    *out = c;
  });
}

int dq_ctx_destroy(dq_ctx* ctx) {
  delete ctx;
  return DQ_OK;
}

int dq_ctx_set_config(dq_ctx* ctx, const dq_config* cfg) {
  return guarded([&] {
    if (!ctx || !cfg) invalid("null argument");
    validate(*cfg);
    // a communicator fixes the worker count: its regions, handles and NCCL ranks are sized by it
    if (ctx->comm && cfg->n_workers != static_cast<uint32_t>(ctx->nranks))
      invalid("n_workers must equal the communicator's rank count");
    ctx->cfg = *cfg;
  });
}

// Scale format of this thread's chunk primitives (dq_codec_format_set; default s = 16,
// hierarchical): the reference's CodecConfig{group_size, hierarchical_scales}.
thread_local uint32_t t_prim_gs = 16;
thread_local int t_prim_hier = 1;

static Layout runs_layout(uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16) {
  if (static_cast<uint64_t>(n8) + n4 + n2 + n16 > 0xffffffffull) invalid("too many super-groups");
  Layout L{n8 + n4 + n2 + n16, n8, n4};
  L.n16 = n16;
  dq_config c;
  dq_config_default(&c);
  c.group_size = t_prim_gs;
  c.hierarchical_scales = t_prim_hier;
  set_format(L, c);
  return L;
}

int dq_codec_format_set(uint32_t group_size, int hierarchical, uint32_t* prev_group_size, int* prev_hierarchical) {
  return guarded([&] {
    if (group_size != 8 && group_size != 16 && group_size != 32 && group_size != 64 && group_size != 128)
      invalid("device codec supports group_size 8, 16, 32, 64 or 128");
    if (prev_group_size) *prev_group_size = t_prim_gs;
    if (prev_hierarchical) *prev_hierarchical = t_prim_hier;
    t_prim_gs = group_size;
    t_prim_hier = hierarchical ? 1 : 0;
  });
}

size_t dq_chunk_bytes(uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16) {
  const Layout L = runs_layout(n8, n4, n2, n16);
  return static_cast<size_t>(L.bytes());
}

size_t dq_wire_bytes(uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16) {
  const Layout L = runs_layout(n8, n4, n2, n16);
  return static_cast<size_t>(24 + L.wire_body());
}

static CodecArgs prim_args(const dq_qctx* q, uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16, uint32_t first,
                           int non_uniform) {
  if (!q) invalid("null qctx");
  if (q->correlated && (q->n_slots == 0 || q->hop_slot >= q->n_slots))
    invalid("correlated_uniform slot out of range");
  if (q->n_slots > 64) invalid("n_slots must be <= 64 on device");
  dq_config c;
  dq_config_default(&c);
  c.seed = q->seed;
  c.round = q->round;
  c.correlated = q->correlated;
  c.non_uniform = non_uniform;
  CodecArgs a = base_args(c, q->chunk_index);
  a.L = runs_layout(n8, n4, n2, n16);
  a.first_sg = first;
  a.slot = q->hop_slot;
  a.n_slots = q->n_slots ? q->n_slots : 1;
  return a;
}

int dq_compress_chunk(const float* d_values, uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16, const dq_qctx* q,
                      uint32_t first, int non_uniform, void* d_out, void* stream) {
  return guarded([&] {
    ensure_books();
    CodecArgs a = prim_args(q, n8, n4, n2, n16, first, non_uniform);
    a.acc_in = d_values;
    a.out = static_cast<uint8_t*>(d_out);
    launch_quant(a, 1, false, S(stream));
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_dar_chunk(const void* d_in, const float* d_local, uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16,
                 const dq_qctx* q, uint32_t first, int non_uniform, void* d_out, void* stream) {
  return guarded([&] {
    ensure_books();
    CodecArgs a = prim_args(q, n8, n4, n2, n16, first, non_uniform);
    a.acc_in = d_local;
    a.in = static_cast<const uint8_t*>(d_in);
    a.out = static_cast<uint8_t*>(d_out);
    launch_quant(a, 1, true, S(stream));
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_da_chunk(const void* d_in, float* d_acc, uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16, int non_uniform,
                void* stream) {
  return guarded([&] {
    ensure_books();
    dq_qctx q{0, 0, 0, 0, 1, 0};
    CodecArgs a = prim_args(&q, n8, n4, n2, n16, 0, non_uniform);
    a.in = static_cast<const uint8_t*>(d_in);
    a.acc_in = d_acc;
    a.acc_out = d_acc;
    launch_da(a, 1, S(stream));
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_decompress_chunk(const void* d_in, float* d_out, uint32_t n8, uint32_t n4, uint32_t n2, uint32_t n16,
                        int non_uniform, void* stream) {
  return guarded([&] {
    ensure_books();
    dq_qctx q{0, 0, 0, 0, 1, 0};
    CodecArgs a = prim_args(&q, n8, n4, n2, n16, 0, non_uniform);
    a.in = static_cast<const uint8_t*>(d_in);
    a.acc_out = d_out;
    launch_decode(a, 0, S(stream));
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_to_reference_wire(const void* h_soa, uint32_t chunk_index, uint32_t n8, uint32_t n4, uint32_t n2,
                         uint32_t n16, void* h_ref) {
  return guarded([&] {
    const Layout L = runs_layout(n8, n4, n2, n16);
    to_reference(static_cast<const uint8_t*>(h_soa), chunk_index, L, static_cast<uint8_t*>(h_ref));
  });
}

int dq_serialize_chunk(const void* d_soa, uint32_t chunk_index, uint32_t n8, uint32_t n4, uint32_t n2,
                       uint32_t n16, void* d_wire, void* stream) {
  return guarded([&] {
    if (!d_wire || (!d_soa && n8 + n4 + n2 + n16)) invalid("null argument");
    if (reinterpret_cast<uintptr_t>(d_wire) % 4 || reinterpret_cast<uintptr_t>(d_soa) % 2)
      invalid("wire buffer must be 4-byte aligned, chunk 2-byte aligned");
    const Layout L = runs_layout(n8, n4, n2, n16);
    launch_to_wire(static_cast<const uint8_t*>(d_soa), L, chunk_index, static_cast<uint8_t*>(d_wire), S(stream));
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_parse_chunk(const void* d_wire, size_t len, void* d_soa, size_t soa_cap, uint32_t* chunk_index,
                   uint32_t* n8, uint32_t* n4, uint32_t* n2, uint32_t* n16, void* stream) {
  return guarded([&] {
    if (!chunk_index || !n8 || !n4 || !n2 || !n16 || (!d_wire && len)) invalid("null argument");
    if (reinterpret_cast<uintptr_t>(d_wire) % 2 || reinterpret_cast<uintptr_t>(d_soa) % 2)
      invalid("buffers must be 2-byte aligned");
    auto mal = [](const char* m) { throw Error(DQ_EMALFORMED, std::string("malformed compressed buffer: ") + m); };
    if (len < 24) mal("truncated header");
    const cudaStream_t st = S(stream);
    const uint8_t* b = static_cast<const uint8_t*>(d_wire);
    uint32_t h[6];
    DQ_CUDA(cudaMemcpyAsync(h, b, 24, cudaMemcpyDeviceToHost, st));
    DQ_CUDA(cudaStreamSynchronize(st));
    const uint32_t count = h[1], r8 = h[2], r4 = h[3], r2 = h[4], r16 = h[5];
    if (static_cast<uint64_t>(r8) + r4 + r2 + r16 != count) mal("width run-lengths do not sum to the super-group count");
    const Layout L = runs_layout(r8, r4, r2, r16);
    // super-groups whose record fits in len (codec.cpp:371-383 checks each before reading it)
    const uint64_t body = len - 24;
    uint32_t fit = count;
    if (L.wire_body() > body) {
      uint32_t lo = 0, hi = count;  // largest k with record_end(k) <= body
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo + 1) / 2;
        if (L.pay_prefix(mid) + L.meta_prefix(mid) <= body) lo = mid;
        else hi = mid - 1;
      }
      fit = lo;
    }
    const bool write = d_soa && soa_cap >= L.bytes();
    unsigned long long* bad = nullptr;
    DQ_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(*bad), st));
    DQ_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(*bad), st));
    launch_from_wire(b, L, fit, write ? static_cast<uint8_t*>(d_soa) : nullptr, bad, st);
    DQ_CUDA(cudaGetLastError());
    unsigned long long hb = 0;
    DQ_CUDA(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, st));
    DQ_CUDA(cudaFreeAsync(bad, st));
    DQ_CUDA(cudaStreamSynchronize(st));
    if (hb != ~0ull) mal(hb & 1 ? "zero super-group scale with nonzero payload" : "zero super-group scale with nonzero group scale");
    if (fit < count) mal(L.width(fit) == 16 ? "truncated width-16 body" : "truncated super-group body");
    if (24 + L.wire_body() != len) mal("trailing bytes after chunk body");
    if (d_soa && !write) invalid("output capacity");
    *chunk_index = h[0];
    *n8 = r8;
    *n4 = r4;
    *n2 = r2;
    *n16 = r16;
  });
}

int dq_from_reference_wire(const void* h_ref, size_t len, void* h_soa, size_t soa_cap,
                           uint32_t* chunk_index, uint32_t* n8, uint32_t* n4, uint32_t* n2, uint32_t* n16) {
  // strict parser with the reference's checks (codec.cpp:345-399), S=256, this thread's scale
  // format (dq_codec_format_set: s, hierarchical u8 + bf16 or flat bf16 group scales)
  return guarded([&] {
    const uint8_t* b = static_cast<const uint8_t*>(h_ref);
    auto mal = [](const char* m) { throw Error(DQ_EMALFORMED, std::string("malformed compressed buffer: ") + m); };
    auto get32 = [&](size_t at) {
      return static_cast<uint32_t>(b[at]) | static_cast<uint32_t>(b[at + 1]) << 8 |
             static_cast<uint32_t>(b[at + 2]) << 16 | static_cast<uint32_t>(b[at + 3]) << 24;
    };
    if (len < 24) mal("truncated header");
    const uint32_t count = get32(4);
    const uint32_t r8 = get32(8), r4 = get32(12), r2 = get32(16), r16 = get32(20);
    if (static_cast<uint64_t>(r8) + r4 + r2 + r16 != count) mal("width run-lengths do not sum to the super-group count");
    const Layout L = runs_layout(r8, r4, r2, r16);
    const size_t meta = L.ss + L.gs;  // 2 + 16 default; flat: 0 + 2 * 256 / s
    size_t at = 24;
    for (uint32_t i = 0; i < count; ++i) {
      const uint32_t w = L.width(i);
      if (w == 16) {
        if (len - at < 512) mal("truncated width-16 body");
        at += 512;
        continue;
      }
      const size_t rec = meta + 32 * w;
      if (len - at < rec) mal("truncated super-group body");
      if (L.ss && (b[at] | b[at + 1] << 8) == 0) {
        for (size_t k = L.ss; k < meta; ++k)
          if (b[at + k]) mal("zero super-group scale with nonzero group scale");
        for (size_t k = meta; k < rec; ++k)
          if (b[at + k]) mal("zero super-group scale with nonzero payload");
      }
      at += rec;
    }
    if (at != len) mal("trailing bytes after chunk body");
    if (soa_cap < L.bytes()) invalid("output capacity");
    uint8_t* o = static_cast<uint8_t*>(h_soa);
    at = 24;
    for (uint32_t i = 0; i < count; ++i) {
      const Layout::SG g = L.locate(i);
      if (g.width == 16) {  // reserved scale slots read as zero
        std::memset(o + g.scale, 0, L.ss);
        std::memset(o + g.codes, 0, L.gs);
        std::memcpy(o + g.payload, b + at, 512);
        at += 512;
        continue;
      }
      std::memcpy(o + g.scale, b + at, L.ss);
      std::memcpy(o + g.codes, b + at + L.ss, L.gs);
      std::memcpy(o + g.payload, b + at + meta, 32 * g.width);
      at += meta + 32 * g.width;
    }
    *chunk_index = get32(0);
    *n8 = r8;
    *n4 = r4;
    *n2 = r2;
    *n16 = r16;
  });
}

int dq_compute_stats(const float* d_x, size_t d, float* d_mean, float* d_sq, void* stream) {
  return guarded([&] {
    const uint32_t T = static_cast<uint32_t>((d + 255) / 256);
    launch_stats(&d_x, 1, d, T, d_mean, d_sq, S(stream));  // the pointer travels in the kernel parameters
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_reduce_stats(const float* d_means, const float* d_sqs, uint32_t n, size_t nsg, float* d_gm,
                    float* d_gs, void* stream) {
  return guarded([&] {
    if (n == 0) invalid("reduce_stats needs at least one worker");
    launch_reduce_stats(d_means, d_sqs, n, static_cast<uint32_t>(nsg), d_gm, d_gs, S(stream));
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_allocate_fast(dq_ctx* ctx, const float* d_F, size_t nsg, double b, uint8_t* d_widths,
                     uint32_t* d_perm, double* u, uint64_t* payload, uint32_t counts[3], void* stream) {
  return guarded([&] {
    if (!ctx) invalid("null context");
    dq_config c = ctx->cfg;
    c.budget_bits = b;
    c.variable_width = 1;
    c.allocator = DQ_ALLOC_FAST;
    AllocResult r = allocate(ctx, c, d_F, static_cast<uint32_t>(nsg), d_widths, d_perm, S(stream));
    if (u) *u = r.u;
    if (payload) *payload = r.payload;
    if (counts) {
      counts[0] = r.n8;
      counts[1] = r.n4;
      counts[2] = r.n2;
    }
  });
}

int dq_allocate_general(dq_ctx* ctx, const float* d_F, size_t nsg, double b, uint8_t* d_widths,
                        uint32_t* d_perm, double* u, uint64_t* payload, uint32_t counts[3], void* stream) {
  return guarded([&] {
    if (!ctx) invalid("null context");
    DQ_CUDA(cudaSetDevice(ctx->device));
    dq_config c = ctx->cfg;
    c.budget_bits = b;
    c.variable_width = 1;
    c.allocator = DQ_ALLOC_GENERAL;
    AllocResult r = allocate_general(ctx, c, d_F, static_cast<uint32_t>(nsg), d_widths, d_perm, S(stream));
    if (u) *u = r.u;
    if (payload) *payload = r.payload;
    if (counts) {
      counts[0] = r.n8;
      counts[1] = r.n4;
      counts[2] = r.n2;
    }
  });
}

int dq_allocate_fast_stateful(dq_ctx* ctx, const float* d_F, size_t nsg, double b, double state[3],
                              uint8_t* d_widths, uint32_t* d_perm, double* u, uint64_t* payload, uint32_t counts[3],
                              void* stream) {
  // allocation.cpp:262-300: widths at the carried u; when over budget, the largest
  // in-budget plateau sample at or below it - payload(u) is non-decreasing, so that is
  // allocate_fast's sample (every sample above the carried u is over budget too)
  return guarded([&] {
    if (!ctx || !state) invalid("null argument");
    DQ_CUDA(cudaSetDevice(ctx->device));
    const cudaStream_t st = S(stream);
    dq_config c = ctx->cfg;
    c.budget_bits = b;
    c.variable_width = 1;
    c.allocator = DQ_ALLOC_FAST;
    const uint32_t T = static_cast<uint32_t>(nsg);
    const uint32_t Sg = c.super_group_size;
    const double budget = static_cast<double>(T) * Sg * payload_budget(c);
    AllocWork w = work_of(ctx, T);
    const float t24 = static_cast<float>(std::exp2((4.0 - state[2]) / kAlpha));
    const float t48 = static_cast<float>(std::exp2((8.0 - state[2]) / kAlpha));
    ctx->tcount.reserve(2);
    launch_threshold_counts(d_F, T, t24, t48, ctx->tcount.p, st);
    unsigned long long cnt[2];
    DQ_CUDA(cudaMemcpyAsync(cnt, ctx->tcount.p, sizeof cnt, cudaMemcpyDeviceToHost, st));
    DQ_CUDA(cudaStreamSynchronize(st));
    const uint64_t pay_u = static_cast<uint64_t>(Sg) * (2ull * T + 2ull * cnt[1] + 4ull * cnt[0]);
    const bool over = static_cast<double>(pay_u) > budget;
    AllocResult r;
    if (over) {
      r = allocate_fast(ctx, c, d_F, T, d_widths, d_perm, st);
    } else {
      launch_alloc_assign(d_F, T, t24, t48, false, w, d_widths, d_perm, st);
      DQ_CUDA(cudaGetLastError());
      DQ_CUDA(cudaMemcpyAsync(ctx->h_counts, w.counts, 3 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      DQ_CUDA(cudaStreamSynchronize(st));
      r.n8 = ctx->h_counts[0];
      r.n4 = ctx->h_counts[1];
      r.n2 = ctx->h_counts[2];
      r.payload = pay_u;
    }
    if (u) *u = state[2];
    if (payload) *payload = r.payload;
    if (counts) {
      counts[0] = r.n8;
      counts[1] = r.n4;
      counts[2] = r.n2;
    }
    if (over) state[1] = state[2];
    else state[0] = state[2];
    state[2] = 0.5 * (state[0] + state[1]);
  });
}

int dq_sim_round(dq_ctx* ctx, const float* const* d_workers, size_t d, float* d_synced, int flags,
                 dq_round_info* info, void* stream) {
  return guarded([&] {
    if (!ctx || !d_workers || !d_synced || !info) invalid("null argument");
    DQ_CUDA(cudaSetDevice(ctx->device));
    sim_round(ctx, d_workers, d, d_synced, flags, info, S(stream));
    ctx->last_info = *info;
  });
}

int dq_run_round_host(dq_ctx* ctx, const float* const* h_workers, size_t d, float* h_synced,
                      dq_round_info* info, void* stream) {
  return guarded([&] {
    if (!ctx || !h_workers || !h_synced || !info) invalid("null argument");
    DQ_CUDA(cudaSetDevice(ctx->device));
    const uint32_t n = ctx->cfg.n_workers;
    const size_t dp = (d + 63) / 64 * 64;
    ctx->stage.reserve((n + 1) * dp);
    std::vector<const float*> xs(n);
    for (uint32_t r = 0; r < n; ++r) {
      float* dst = ctx->stage.p + r * dp;
      DQ_CUDA(cudaMemcpyAsync(dst, h_workers[r], d * sizeof(float), cudaMemcpyHostToDevice, S(stream)));
      xs[r] = dst;
    }
    float* y = ctx->stage.p + n * dp;
    sim_round(ctx, xs.data(), d, y, DQ_SIM_NO_METRICS, info, S(stream));
    DQ_CUDA(cudaMemcpyAsync(h_synced, y, d * sizeof(float), cudaMemcpyDeviceToHost, S(stream)));
    DQ_CUDA(cudaStreamSynchronize(S(stream)));
  });
}

int dq_round_allocation(dq_ctx* ctx, uint8_t* h_widths, uint32_t* h_perm, size_t nsg) {
  return guarded([&] {
    if (!ctx) invalid("null context");
    if (nsg != ctx->last_T) invalid("super-group count does not match the last round");
    if (h_widths) DQ_CUDA(cudaMemcpy(h_widths, ctx->widths.p, nsg, cudaMemcpyDeviceToHost));
    if (h_perm) DQ_CUDA(cudaMemcpy(h_perm, ctx->perm.p, nsg * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  });
}

int dq_allreduce(dq_ctx* ctx, const float* d_in, float* d_out, size_t d, dq_round_info* info, void* stream) {
  return guarded([&] {
    if (!ctx || !d_in || !d_out) invalid("null argument");
    DQ_CUDA(cudaSetDevice(ctx->device));
    dq_round_info scratch{};
    dist_round(ctx, d_in, d, d_out, info ? info : &scratch, S(stream));
    ctx->last_info = info ? *info : scratch;
    if (info) {  // the caller wants the round's allocation and accounting: wait for it
      DQ_CUDA(cudaStreamSynchronize(S(stream)));
      harvest(ctx);
      finish_info(ctx, info);
      info->ms_total = ctx->last_round_ms;
    }
  });
}

int dq_round_wait(dq_ctx* ctx, dq_round_info* info) {
  return guarded([&] {
    if (!ctx || !info) invalid("null argument");
    DQ_CUDA(cudaSetDevice(ctx->device));
    if (ctx->lr_pending) DQ_CUDA(cudaEventSynchronize(ctx->lr1));
    else if (ctx->ev1) DQ_CUDA(cudaEventSynchronize(ctx->ev1));
    harvest(ctx);
    if (!ctx->rec.valid) invalid("no round has been run on this context");
    *info = ctx->last_info;
    if (ctx->rec.async) finish_info(ctx, info);
    info->ms_total = ctx->last_round_ms;
  });
}

int dq_ctx_host_allocations(const dq_ctx* ctx, uint64_t* finished, uint64_t* consulted) {
  return guarded([&] {
    if (!ctx || !finished) invalid("null argument");
    *finished = ctx->host_allocs.load(std::memory_order_relaxed) + ctx->alloc_redos;
    if (consulted) *consulted = ctx->host_consults.load(std::memory_order_relaxed);
  });
}

int dq_debug_force_host_alloc(int on) {
  return guarded([&] {
    ensure_books();
    set_force_host_alloc(on);
    DQ_CUDA(cudaGetLastError());
  });
}

int dq_selftest(int which, uint64_t n, uint64_t seed, uint64_t* mismatches) {
  return guarded([&] {
    if (!mismatches) invalid("null argument");
    ensure_books();
    dq_config c;
    dq_config_default(&c);
    const CodecArgs a = base_args(c, 0);
    unsigned long long* d = nullptr;
    DQ_CUDA(cudaMalloc(&d, 2 * sizeof(*d) + 64 * sizeof(float)));
    DQ_CUDA(cudaMemset(d, 0, 2 * sizeof(*d) + 64 * sizeof(float)));
    float* ex = reinterpret_cast<float*>(d + 2);
    launch_selftest(which, n, seed, d, a.est_c1, a.est_c2, ex, nullptr);
    DQ_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    float hx[64];
    DQ_CUDA(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost));
    DQ_CUDA(cudaMemcpy(hx, ex, sizeof(hx), cudaMemcpyDeviceToHost));
    DQ_CUDA(cudaFree(d));
    *mismatches = h;
    if (h) {  // leave examples in the error string for the test report
      char msg[1024];
      int k = std::snprintf(msg, sizeof msg, "%llu mismatches; a b got want:", h);
      for (int i = 0; i < 4 && k < 900; ++i)
        k += std::snprintf(msg + k, sizeof msg - k, " [%a %a %a %a]", hx[4 * i], hx[4 * i + 1], hx[4 * i + 2], hx[4 * i + 3]);
      g_err = msg;
    }
  });
}

int dq_profile_enable(dq_ctx* ctx, int on) {
  return guarded([&] {
    if (!ctx) invalid("null context");
    ctx->profile = on;
  });
}

int dq_profile_read(dq_ctx* ctx, dq_kernel_profile* out, int cap, int* count, int reset) {
  return guarded([&] {
    if (!ctx) invalid("null context");
    DQ_CUDA(cudaSetDevice(ctx->device));
    DQ_CUDA(cudaDeviceSynchronize());
    harvest(ctx);
    int k = 0;
    for (int i = 0; i < K_NKINDS; ++i) {
      if (!ctx->prof_launches[i] && !ctx->prof_ms[i]) continue;
      if (out && k < cap) {
        dq_kernel_profile& p = out[k];
        std::snprintf(p.name, sizeof p.name, "%s", kKindName[i]);
        p.launches = ctx->prof_launches[i];
        p.ms = ctx->prof_ms[i];
        p.bytes = ctx->prof_bytes[i];
      }
      ++k;
    }
    if (count) *count = k;
    if (reset)
      for (int i = 0; i < K_NKINDS; ++i) ctx->prof_ms[i] = ctx->prof_bytes[i] = 0, ctx->prof_launches[i] = 0;
  });
}

int dq_schedule(uint32_t n_workers, int topology, uint32_t chunk, dq_event* events, uint32_t cap,
                uint32_t* n_events, uint32_t* sink_slot, uint32_t* n_slots, uint32_t* n_gather) {
  return guarded([&] {
    if (!n_events || !sink_slot || !n_slots || !n_gather) invalid("null argument");
    if (topology != DQ_RING && topology != DQ_BUTTERFLY) invalid("unknown topology");
    if (n_workers < 2) invalid(topology == DQ_RING ? "ring schedule requires n >= 2" : "butterfly schedule requires n >= 2");
    if (n_workers > 64) invalid("n_workers must be at most 64");
    if (topology == DQ_BUTTERFLY && (n_workers & (n_workers - 1)))
      invalid("butterfly topology requires a power-of-two worker count");
    if (chunk >= n_workers) invalid("chunk out of range");
    const Plan pl = make_plan(n_workers, chunk, topology);
    *n_events = static_cast<uint32_t>(pl.red.size());
    *sink_slot = pl.sink_slot;
    *n_slots = pl.n_slots;
    *n_gather = pl.n_gat;
    if (events && cap < pl.red.size()) invalid("event capacity");
    for (size_t e = 0; events && e < pl.red.size(); ++e)
      events[e] = dq_event{pl.red[e].snd, pl.red[e].rcv, pl.red[e].slot,
                           topology == DQ_RING ? static_cast<uint32_t>(e) : butterfly_stage(n_workers, pl.red[e])};
  });
}

int dq_comm_unique_id(uint8_t out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    DQ_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, id.internal, 128);
  });
}

int dq_comm_set_transport(dq_ctx* ctx, int transport) {
  return guarded([&] {
    if (!ctx) invalid("null context");
    if (transport != DQ_TRANSPORT_PEER && transport != DQ_TRANSPORT_NCCL) invalid("unknown transport");
    ctx->transport = transport;
  });
}

int dq_comm_get_transport(const dq_ctx* ctx, int* transport) {
  return guarded([&] {
    if (!ctx || !transport) invalid("null argument");
    *transport = ctx->transport;
  });
}

int dq_comm_init(dq_ctx* ctx, int rank, int nranks, const uint8_t id[128]) {
  return guarded([&] {
    if (!ctx) invalid("null context");
    if (static_cast<uint32_t>(nranks) != ctx->cfg.n_workers) invalid("nranks must equal cfg.n_workers");
    DQ_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    DQ_NCCL(ncclCommInitRank(&ctx->comm, nranks, uid, rank));
    ctx->rank = rank;
    ctx->nranks = nranks;
  });
}

}  // extern "C"
