/*
 * dq_oracle.c — plain-C restatement of the DynamiQ reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the thing measured or shipped).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  Each function cites the reference file:line it restates
 * (paths relative to /root/reference/).  Compiled with -ffp-contract=off and
 * no -march flags so float/double expressions round exactly like the reference
 * built for baseline x86-64 (SSE2, no FMA).
 *
 * Parity status: pinned against the reference library itself (oracle/_ref,
 * built from the reference sources by oracle/Makefile) and against the golden
 * vectors in tests/golden/ — see tests/test_oracle.py.
 */
#include "dq_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}
const char* dqo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ PRNG  */
/* proj/src/random.cpp:10-17 (murmur3/splitmix fmix64) */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdULL;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ULL;
  return z ^ (z >> 33);
}
#define GOLDEN 0x9e3779b97f4a7c15ULL
/* proj/src/random.cpp:19-21 */
static inline uint64_t absorb(uint64_t h, uint64_t w) {
  return mix64(h ^ (w + GOLDEN + (h << 6) + (h >> 2)));
}
typedef struct {
  uint64_t seed, round;
  uint32_t purpose;
  uint64_t chunk, sg, entry;
} key_t_;
/* proj/src/random.cpp:25-34: seed, round, purpose, chunk, sg, entry, counter */
static uint64_t keyed(const key_t_* k, uint64_t counter) {
  uint64_t words[6] = {k->round, k->purpose, k->chunk, k->sg, k->entry, counter};
  uint64_t h = mix64(k->seed ^ 0x6a09e667f3bcc909ULL);
  for (int i = 0; i < 6; ++i) h = absorb(h, words[i]);
  return h;
}
/* proj/src/random.cpp:36-38: top 53 bits scaled by 2^-53 */
static inline double unit53(uint64_t b) { return (double)(b >> 11) * 0x1.0p-53; }

/* Fisher-Yates over n slots with r % (i+1): proj/src/random.cpp:53-61,72-81 */
static uint32_t perm_slot(const key_t_* k, uint32_t slot, uint32_t n) {
  uint32_t stack[256];
  uint32_t* pi = n <= 256 ? stack : (uint32_t*)malloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < n; ++i) pi[i] = i;
  for (uint32_t i = n - 1; i > 0; --i) {
    uint32_t j = (uint32_t)(keyed(k, i) % (uint64_t)(i + 1));
    uint32_t t = pi[i];
    pi[i] = pi[j];
    pi[j] = t;
  }
  uint32_t r = pi[slot];
  if (pi != stack) free(pi);
  return r;
}
/* proj/src/random.cpp:83-90: (pi[slot] + gamma) / n, gamma keyed with slot<<32 */
static double corr_uniform(key_t_ k, uint32_t slot, uint32_t n) {
  key_t_ pk = k;
  pk.purpose = DQO_PERMUTATION;
  uint32_t interval = perm_slot(&pk, slot, n);
  k.entry |= (uint64_t)slot << 32; /* with_slot, random.hpp:35-38 */
  double gamma = unit53(keyed(&k, 0));
  return ((double)interval + gamma) / (double)n;
}

uint64_t dqo_random_bits(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                         uint64_t sg, uint64_t entry) {
  key_t_ k = {seed, round, purpose, chunk, sg, entry};
  return keyed(&k, 0);
}
double dqo_uniform_at(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                      uint64_t sg, uint64_t entry) {
  return unit53(dqo_random_bits(seed, round, purpose, chunk, sg, entry));
}
int dqo_permutation_slot(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                         uint64_t sg, uint64_t entry, uint32_t slot, uint32_t n, uint32_t* out) {
  if (n == 0 || slot >= n) return fail(DQO_EINVAL, "permutation_slot out of range");
  key_t_ k = {seed, round, purpose, chunk, sg, entry};
  *out = perm_slot(&k, slot, n);
  return 0;
}
int dqo_correlated_uniform(uint64_t seed, uint64_t round, uint32_t purpose, uint64_t chunk,
                           uint64_t sg, uint64_t entry, uint32_t slot, uint32_t n, double* out) {
  if (n == 0 || slot >= n) return fail(DQO_EINVAL, "correlated_uniform slot out of range");
  key_t_ k = {seed, round, purpose, chunk, sg, entry};
  *out = corr_uniform(k, slot, n);
  return 0;
}

/* --------------------------------------------------------------- bf16     */
static inline float bf16f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint32_t fbits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
/* proj/include/dynamiq/bf16.hpp:30-40 */
static uint16_t bf16_up(float v) {
  uint32_t u = fbits(v);
  uint16_t hi = (uint16_t)(u >> 16);
  if ((u & 0xffffu) == 0) return hi;
  uint16_t up = (uint16_t)(hi + 1);
  return (up & 0x7f80u) == 0x7f80u ? 0x7f7fu : up;
}
/* proj/include/dynamiq/bf16.hpp:16-27 */
static uint16_t bf16_rne(float v) {
  uint32_t u = fbits(v);
  if (((u >> 23) & 0xff) == 0xff) {
    uint16_t hi = (uint16_t)(u >> 16);
    if ((u & 0x7fffffu) != 0 && (hi & 0x7f) == 0) hi |= 1;
    return hi;
  }
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* ------------------------------------------------------------ codebooks   */
/* proj/src/codebook.cpp:20-48 (f(eps,r) in double, stored float, strictly increasing),
 * :50-60 (uniform), :63-75 (default eps 0.05 / 0.25 / 0.05) */
int dqo_codebook(int width, int non_uniform, float* out) {
  if (width != 2 && width != 4 && width != 8) return fail(DQO_EINVAL, "codebook width");
  const int count = 1 << (width - 1), top = count - 1;
  if (!non_uniform) {
    for (int r = 0; r < count; ++r) out[r] = (float)((double)r / top);
    return 0;
  }
  const double eps = width == 4 ? 0.25 : 0.05;
  const double base = 1.0 + 2.0 * eps * eps;
  for (int r = 0; r < count; ++r) {
    double v = r == 0 ? 0.0 : r == top ? 1.0 : (pow(base, r) - 1.0) / (pow(base, top) - 1.0);
    out[r] = (float)v;
  }
  for (int r = 1; r < count; ++r)
    if (out[r] <= out[r - 1]) out[r] = nextafterf(out[r - 1], 2.0f);
  return 0;
}

/* proj/src/codebook.cpp:77-92: lower_bound bracket, float p_up, u < (double)p_up */
static uint32_t sr_index(const float* q, int count, float v, double u) {
  int lo = 0, hi = count; /* first index with q[i] >= v */
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (q[mid] < v) lo = mid + 1; else hi = mid;
  }
  uint32_t h = (uint32_t)lo;
  if (q[h] == v) return h;
  float p_up = (v - q[h - 1]) / (q[h] - q[h - 1]);
  return u < (double)p_up ? h : h - 1;
}

/* ---------------------------------------------------------------- codec   */
/* proj/src/codec.cpp:24-26 */
static inline float group_scale_decode(uint8_t code, float sg) { return (float)code * sg / 255.0f; }
/* proj/src/codec.cpp:28-35 */
static uint8_t group_scale_sr(float ratio, double u) {
  if (ratio >= 255.0f) return 255;
  float lo = floorf(ratio);
  float p_up = ratio - lo;
  return (uint8_t)((u < (double)p_up) ? lo + 1.0f : lo);
}
/* proj/src/codec.cpp:39-47 */
static uint16_t stochastic_bf16(float value, double u) {
  uint32_t bits = fbits(value);
  uint16_t lo = (uint16_t)(bits >> 16);
  if ((bits & 0xffffu) == 0) return lo;
  uint16_t hi = (uint16_t)(lo + 1);
  float flo = bf16f(lo), fhi = bf16f(hi);
  float p_up = (value - flo) / (fhi - flo);
  return (u < (double)p_up) ? hi : lo;
}
/* proj/src/codec.cpp:49-59 */
static double entry_u(const dqo_qctx* q, uint32_t sg, uint32_t e) {
  key_t_ k = {q->seed, q->round, DQO_ENTRY_QUANT, q->chunk, sg, e};
  if (q->correlated) return corr_uniform(k, q->slot, q->n_slots);
  k.entry |= (uint64_t)q->slot << 32;
  return unit53(keyed(&k, 0));
}
static double scale_u(const dqo_qctx* q, uint32_t sg, uint32_t g) {
  key_t_ k = {q->seed, q->round, DQO_SCALE_QUANT, q->chunk, sg, (uint64_t)g | ((uint64_t)q->slot << 32)};
  return unit53(keyed(&k, 0));
}

static int codec_ok(const dqo_codec* c) {
  return c->group_size && c->super_group_size && c->super_group_size % c->group_size == 0 &&
         c->super_group_size % 4 == 0;
}
static int width_ok(int w) { return w == 2 || w == 4 || w == 8 || w == 16; }

/* bytes of one super-group record on the wire, proj/src/codec.cpp:270-281,319-343 */
static size_t sg_record_bytes(int w, const dqo_codec* c) {
  const uint32_t S = c->super_group_size, s = c->group_size;
  if (w == 16) return (size_t)S * 2;
  size_t scales = c->hierarchical ? 2 + S / s : (size_t)(S / s) * 2;
  return scales + (size_t)S * w / 8;
}

/* proj/src/codec.cpp:70-126 — compress one super-group straight into its wire record */
static void compress_sg(const float* x, int w, const float* cb, const dqo_codec* c,
                        const dqo_qctx* q, uint32_t sg, uint8_t* rec) {
  const uint32_t S = c->super_group_size, s = c->group_size;
  if (w == 16) {
    for (uint32_t k = 0; k < S; ++k) {
      uint16_t b = bf16_rne(x[k]);
      rec[2 * k] = (uint8_t)b;
      rec[2 * k + 1] = (uint8_t)(b >> 8);
    }
    return;
  }
  float amax = 0.0f;
  for (uint32_t k = 0; k < S; ++k) amax = fmaxf(amax, fabsf(x[k]));
  float sgs = 0.0f;
  uint8_t* scales = rec;
  if (c->hierarchical) {
    uint16_t b = bf16_up(amax);
    rec[0] = (uint8_t)b;
    rec[1] = (uint8_t)(b >> 8);
    sgs = bf16f(b);
    scales = rec + 2;
  }
  const uint32_t G = S / s;
  uint8_t* payload = scales + (c->hierarchical ? G : 2 * G);
  memset(payload, 0, (size_t)S * w / 8);
  const int count = 1 << (w - 1);
  for (uint32_t g = 0; g < G; ++g) {
    const float* gx = x + (size_t)g * s;
    float m = 0.0f;
    for (uint32_t k = 0; k < s; ++k) m = fmaxf(m, fabsf(gx[k]));
    if (c->hierarchical) {
      uint8_t code = 0;
      if (m > 0.0f && sgs > 0.0f) code = group_scale_sr(m / sgs * 255.0f, scale_u(q, sg, g));
      scales[g] = code;
    } else {
      uint16_t b = m > 0.0f ? stochastic_bf16(m, scale_u(q, sg, g)) : 0;
      scales[2 * g] = (uint8_t)b;
      scales[2 * g + 1] = (uint8_t)(b >> 8);
    }
    for (uint32_t k = 0; k < s; ++k) {
      const float v0 = gx[k];
      uint32_t code = v0 < 0.0f ? 1u : 0u;
      if (m > 0.0f) code |= sr_index(cb, count, fabsf(v0) / m, entry_u(q, sg, g * s + k)) << 1;
      /* LSB-first packing, proj/include/dynamiq/bitio.hpp:13-35 */
      size_t bit = (size_t)(g * s + k) * (size_t)w;
      for (int b = 0; b < w; ++b)
        if (code >> b & 1u) payload[(bit + b) >> 3] |= (uint8_t)(1u << ((bit + b) & 7));
    }
  }
}

/* proj/src/codec.cpp:128-162; add=1 accumulates (proj/src/codec.cpp:198-236) */
static int decode_sg(const uint8_t* rec, int w, const float* cb, const dqo_codec* c, float* out,
                     int add) {
  const uint32_t S = c->super_group_size, s = c->group_size;
  if (w == 16) {
    for (uint32_t k = 0; k < S; ++k) {
      float v = bf16f((uint16_t)(rec[2 * k] | rec[2 * k + 1] << 8));
      out[k] = add ? out[k] + v : v;
    }
    return 0;
  }
  const uint32_t G = S / s;
  const uint8_t* scales = rec + (c->hierarchical ? 2 : 0);
  const float sgs = c->hierarchical ? bf16f((uint16_t)(rec[0] | rec[1] << 8)) : 0.0f;
  const uint8_t* payload = scales + (c->hierarchical ? G : 2 * G);
  const uint32_t count = 1u << (w - 1);
  for (uint32_t g = 0; g < G; ++g) {
    const float sf = c->hierarchical ? group_scale_decode(scales[g], sgs)
                                     : bf16f((uint16_t)(scales[2 * g] | scales[2 * g + 1] << 8));
    for (uint32_t k = 0; k < s; ++k) {
      size_t bit = (size_t)(g * s + k) * (size_t)w;
      uint32_t code = 0;
      for (int b = 0; b < w; ++b) code |= (uint32_t)(payload[(bit + b) >> 3] >> ((bit + b) & 7) & 1u) << b;
      uint32_t idx = code >> 1;
      if (idx >= count) return fail(DQO_EMALFORMED, "malformed compressed buffer: index out of range");
      float mag = cb[idx] * sf;
      float v = (code & 1u) ? -mag : mag;
      out[g * s + k] = add ? out[g * s + k] + v : v;
    }
  }
  return 0;
}

static uint32_t rd32(const uint8_t* p) {
  return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24;
}
static void wr32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

typedef struct {
  float b2[2], b4[8], b8[128];
} books_t;
static void load_books(books_t* b, int non_uniform) {
  dqo_codebook(2, non_uniform, b->b2);
  dqo_codebook(4, non_uniform, b->b4);
  dqo_codebook(8, non_uniform, b->b8);
}
static const float* book_for(const books_t* b, int w) {
  return w == 2 ? b->b2 : w == 4 ? b->b4 : w == 8 ? b->b8 : NULL;
}
static int cls_of(int w) { return w == 8 ? 0 : w == 4 ? 1 : w == 2 ? 2 : w == 16 ? 3 : -1; }

uint64_t dqo_compressed_size_bits(const uint8_t* widths, size_t nsg, uint32_t S, uint32_t s,
                                  int hierarchical) {
  dqo_codec c = {s, S, hierarchical, 1};
  uint64_t bits = 6 * 32; /* header, proj/src/codec.cpp:268 */
  for (size_t i = 0; i < nsg; ++i) bits += (uint64_t)sg_record_bytes(widths[i], &c) * 8;
  return bits;
}

/* serialize: proj/src/codec.cpp:283-343 (header + run-order check 8,4,2,16) */
static int write_header(const uint8_t* widths, size_t nsg, uint32_t chunk, uint8_t* out) {
  uint32_t n[4] = {0, 0, 0, 0};
  int prev = -1;
  for (size_t i = 0; i < nsg; ++i) {
    int c = cls_of(widths[i]);
    if (c < 0) return fail(DQO_EINVAL, "unsupported width on wire");
    if (c < prev) return fail(DQO_EINVAL, "chunk body must be ordered by width class 8,4,2,16");
    prev = c;
    n[c]++;
  }
  wr32(out, chunk);
  wr32(out + 4, (uint32_t)nsg);
  for (int r = 0; r < 4; ++r) wr32(out + 8 + 4 * r, n[r]);
  return 0;
}

/* proj/src/codec.cpp:164-183 then serialize_chunk */
int dqo_compress_chunk(const float* values, const uint8_t* widths, size_t nsg, const dqo_codec* cc,
                       const dqo_qctx* q, uint32_t first_sg, uint8_t* out, size_t cap,
                       size_t* out_len) {
  if (!codec_ok(cc)) return fail(DQO_EINVAL, "invalid codec config");
  for (size_t i = 0; i < nsg; ++i)
    if (!width_ok(widths[i])) return fail(DQO_EINVAL, "unsupported codec width");
  if (q->correlated && (q->n_slots == 0 || q->slot >= q->n_slots))
    return fail(DQO_EINVAL, "correlated_uniform slot out of range");
  size_t need = dqo_compressed_size_bits(widths, nsg, cc->super_group_size, cc->group_size, cc->hierarchical) / 8;
  if (cap < need) return fail(DQO_EINVAL, "output capacity");
  int rc = write_header(widths, nsg, q->chunk, out);
  if (rc) return rc;
  books_t b;
  load_books(&b, cc->non_uniform);
  size_t at = 24;
  for (size_t i = 0; i < nsg; ++i) {
    compress_sg(values + i * cc->super_group_size, widths[i], book_for(&b, widths[i]), cc, q,
                first_sg + (uint32_t)i, out + at);
    at += sg_record_bytes(widths[i], cc);
  }
  *out_len = at;
  return 0;
}

/* strict parser, proj/src/codec.cpp:345-399; returns widths and record offsets */
static int parse(const uint8_t* in, size_t len, const dqo_codec* c, uint8_t** widths_out,
                 size_t** offs_out, size_t* nsg_out, uint32_t* chunk_out) {
  if (len < 24) return fail(DQO_EMALFORMED, "malformed compressed buffer: truncated header");
  uint32_t count = rd32(in + 4);
  uint32_t runs[4] = {rd32(in + 8), rd32(in + 12), rd32(in + 16), rd32(in + 20)};
  if ((uint64_t)runs[0] + runs[1] + runs[2] + runs[3] != count)
    return fail(DQO_EMALFORMED, "malformed compressed buffer: run-lengths");
  const uint32_t S = c->super_group_size, s = c->group_size, G = S / s;
  if ((uint64_t)count * 3 > (uint64_t)len) /* every record is >= 3 bytes */
    return fail(DQO_EMALFORMED, "malformed compressed buffer: truncated super-group body");
  uint8_t* w = (uint8_t*)malloc(count ? count : 1);
  size_t* o = (size_t*)malloc(sizeof(size_t) * (count ? count : 1));
  static const uint8_t kw[4] = {8, 4, 2, 16};
  size_t k = 0, at = 24;
  for (int r = 0; r < 4; ++r)
    for (uint32_t i = 0; i < runs[r]; ++i) w[k++] = kw[r];
  for (size_t i = 0; i < count; ++i) {
    size_t rb = sg_record_bytes(w[i], c);
    if (len - at < rb) {
      free(w); free(o);
      return fail(DQO_EMALFORMED, "malformed compressed buffer: truncated super-group body");
    }
    o[i] = at;
    if (w[i] != 16 && c->hierarchical && (in[at] | in[at + 1] << 8) == 0) {
      for (size_t b = 2; b < rb; ++b)
        if (in[at + b]) {
          free(w); free(o);
          return fail(DQO_EMALFORMED, b < 2 + G ? "malformed compressed buffer: zero super-group scale with nonzero group scale"
                                                : "malformed compressed buffer: zero super-group scale with nonzero payload");
        }
    }
    at += rb;
  }
  if (at != len) {
    free(w); free(o);
    return fail(DQO_EMALFORMED, "malformed compressed buffer: trailing bytes after chunk body");
  }
  *widths_out = w;
  *offs_out = o;
  *nsg_out = count;
  if (chunk_out) *chunk_out = rd32(in);
  return 0;
}

static int decode_chunk(const uint8_t* in, size_t len, const dqo_codec* cc, float* out, size_t n,
                        int add) {
  if (!codec_ok(cc)) return fail(DQO_EINVAL, "invalid codec config");
  uint8_t* w;
  size_t* o;
  size_t nsg;
  int rc = parse(in, len, cc, &w, &o, &nsg, NULL);
  if (rc) return rc;
  if (n != nsg * cc->super_group_size) {
    free(w); free(o);
    return fail(DQO_EINVAL, "output length does not match chunk");
  }
  books_t b;
  load_books(&b, cc->non_uniform);
  for (size_t i = 0; i < nsg && !rc; ++i)
    rc = decode_sg(in + o[i], w[i], book_for(&b, w[i]), cc, out + i * cc->super_group_size, add);
  free(w);
  free(o);
  return rc;
}
int dqo_decompress_chunk(const uint8_t* in, size_t len, const dqo_codec* cc, float* out, size_t n) {
  return decode_chunk(in, len, cc, out, n, 0);
}
int dqo_decompress_accumulate(const uint8_t* in, size_t len, const dqo_codec* cc, float* acc, size_t n) {
  return decode_chunk(in, len, cc, acc, n, 1);
}

/* proj/src/codec.cpp:238-266: per SG decode, sum[k] = dec[k] + local[k], recompress */
int dqo_dar_chunk(const uint8_t* in, size_t len, const float* local, size_t n_local,
                  const dqo_codec* cc, const dqo_qctx* q, uint32_t first_sg, uint8_t* out,
                  size_t cap, size_t* out_len) {
  if (!codec_ok(cc)) return fail(DQO_EINVAL, "invalid codec config");
  uint8_t* w;
  size_t* o;
  size_t nsg;
  int rc = parse(in, len, cc, &w, &o, &nsg, NULL);
  if (rc) return rc;
  const uint32_t S = cc->super_group_size;
  if (n_local != nsg * S) {
    free(w); free(o);
    return fail(DQO_EINVAL, "local buffer length does not match chunk");
  }
  if (cap < len) {
    free(w); free(o);
    return fail(DQO_EINVAL, "output capacity");
  }
  write_header(w, nsg, q->chunk, out);
  books_t b;
  load_books(&b, cc->non_uniform);
  float* sum = (float*)malloc(sizeof(float) * S);
  size_t at = 24;
  for (size_t i = 0; i < nsg && !rc; ++i) {
    rc = decode_sg(in + o[i], w[i], book_for(&b, w[i]), cc, sum, 0);
    for (uint32_t k = 0; k < S; ++k) sum[k] += local[i * S + k];
    compress_sg(sum, w[i], book_for(&b, w[i]), cc, q, first_sg + (uint32_t)i, out + at);
    at += sg_record_bytes(w[i], cc);
  }
  free(sum);
  free(w);
  free(o);
  *out_len = at;
  return rc;
}

/* ---------------------------------------------------------------- stats   */
/* proj/src/stats.cpp:10-35: zero padding to a multiple of S; sequential fp64 per SG */
int dqo_compute_stats(const float* x, size_t d, uint32_t s, uint32_t S, float* mean, float* sq) {
  if (!s || !S || S % s) return fail(DQO_EINVAL, "super-group size must be a positive multiple of the group size");
  size_t nsg = (d + S - 1) / S;
  for (size_t j = 0; j < nsg; ++j) {
    double a = 0.0, b = 0.0;
    for (uint32_t k = 0; k < S; ++k) {
      size_t i = j * S + k;
      float v = i < d ? x[i] : 0.0f;
      a += v;
      b += (double)v * v;
    }
    mean[j] = (float)(a / S);
    sq[j] = (float)b;
  }
  return 0;
}
/* proj/src/stats.cpp:37-54: rank-ordered fp64 sums */
int dqo_reduce_stats(const float* means, const float* sqs, uint32_t n, size_t nsg, float* gm,
                     float* gs) {
  if (!n) return fail(DQO_EINVAL, "reduce_stats needs at least one worker");
  for (size_t j = 0; j < nsg; ++j) {
    double a = 0.0, b = 0.0;
    for (uint32_t r = 0; r < n; ++r) {
      a += means[(size_t)r * nsg + j];
      b += sqs[(size_t)r * nsg + j];
    }
    gm[j] = (float)(a / n);
    gs[j] = (float)b;
  }
  return 0;
}

/* ----------------------------------------------------------- allocation   */
static int cmp_dbl(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : x > y;
}
/* proj/src/allocation.cpp:302-310: stable sort by rank(w) = 16 - w, width 16 last
 * (0x100): class order 8,4,2,1,16 (counting sort over the 513 possible ranks) */
static int perm_rank(uint8_t w) { return (w == 16 ? 0x100 : 16 - (int)w) + 256; }
int dqo_build_permutation(const uint8_t* widths, size_t nsg, uint32_t* perm) {
  size_t cnt[514] = {0};
  for (size_t i = 0; i < nsg; ++i) cnt[perm_rank(widths[i]) + 1]++;
  for (int r = 0; r < 513; ++r) cnt[r + 1] += cnt[r];
  for (size_t i = 0; i < nsg; ++i) perm[cnt[perm_rank(widths[i])]++] = (uint32_t)i;
  return 0;
}
/* proj/src/allocation.cpp:45-58 */
static int bbar_of(double b, uint32_t s, uint32_t S, int hier, double* out) {
  if (!s || S % s) return fail(DQO_EINVAL, "invalid group sizes");
  double over = hier ? 8.0 / s + 16.0 / S : 16.0 / s;
  double bbar = b - over;
  if (!(bbar > 2.0)) return fail(DQO_EINFEASIBLE, "payload budget does not exceed the minimum width 2");
  *out = bbar;
  return 0;
}
/* fast allocator for W={2,4,8}: proj/src/allocation.cpp:34-35,170-260 */
int dqo_allocate_fast(const float* F, size_t nsg, double b, uint32_t s, uint32_t S, int hier,
                      uint8_t* widths, uint32_t* perm, double* u_out, uint64_t* payload_out) {
  double bbar;
  int rc = bbar_of(b, s, S, hier, &bbar);
  if (rc) return rc;
  const double alpha = 4.0 / log2(512.0 / 17.0);
  const double budget = (double)nsg * S * bbar;
  double* flips = (double*)malloc(sizeof(double) * (2 * nsg + 1));
  size_t nf = 0;
  for (size_t j = 0; j < nsg; ++j) {
    if (F[j] <= 0.0f) continue;
    double l = alpha * log2((double)F[j]);
    flips[nf++] = 4.0 - l;
    flips[nf++] = 8.0 - l;
  }
  qsort(flips, nf, sizeof(double), cmp_dbl);
  size_t nu = 0;
  for (size_t i = 0; i < nf; ++i)
    if (nu == 0 || flips[i] != flips[nu - 1]) flips[nu++] = flips[i];
  /* plateau sample points: flips.front()-1, midpoints, flips.back()+1 (or {0}) */
  size_t ns = nu ? nu + 1 : 1;
  double* samp = (double*)malloc(sizeof(double) * ns);
  if (!nu) samp[0] = 0.0;
  else {
    samp[0] = flips[0] - 1.0;
    for (size_t i = 0; i + 1 < nu; ++i) samp[i + 1] = 0.5 * (flips[i] + flips[i + 1]);
    samp[nu] = flips[nu - 1] + 1.0;
    for (size_t i = 0; i < ns; ++i) samp[i] = samp[i] < -1e6 ? -1e6 : samp[i] > 1e6 ? 1e6 : samp[i];
  }
  free(flips);
#define PAYLOAD_AT(uu, res)                                                        \
  do {                                                                             \
    const float t24_ = (float)exp2((4.0 - (uu)) / alpha);                          \
    const float t48_ = (float)exp2((8.0 - (uu)) / alpha);                          \
    uint64_t p_ = 0;                                                               \
    for (size_t j_ = 0; j_ < nsg; ++j_)                                            \
      p_ += (uint64_t)(F[j_] >= t48_ ? 8 : F[j_] >= t24_ ? 4 : 2) * S;              \
    res = p_;                                                                      \
  } while (0)
  size_t lo = 0, hi = ns - 1;
  uint64_t p;
  PAYLOAD_AT(samp[lo], p);
  if ((double)p > budget) {
    free(samp);
    return fail(DQO_EINFEASIBLE, "bit allocation infeasible within budget");
  }
  PAYLOAD_AT(samp[hi], p);
  if ((double)p <= budget) lo = hi;
  else
    while (lo + 1 < hi) {
      size_t mid = (lo + hi) / 2;
      PAYLOAD_AT(samp[mid], p);
      if ((double)p <= budget) lo = mid; else hi = mid;
    }
  const double u = samp[lo];
  free(samp);
  const float t24 = (float)exp2((4.0 - u) / alpha), t48 = (float)exp2((8.0 - u) / alpha);
  uint64_t pay = 0;
  for (size_t j = 0; j < nsg; ++j) {
    widths[j] = F[j] >= t48 ? 8 : F[j] >= t24 ? 4 : 2;
    pay += (uint64_t)widths[j] * S;
  }
  if ((double)pay > budget) return fail(DQO_EINFEASIBLE, "bit allocation infeasible within budget");
  *u_out = u;
  *payload_out = pay;
  if (perm) dqo_build_permutation(widths, nsg, perm);
  return 0;
}

/* general allocator: proj/src/allocation.cpp:14-33 (widths), 44-58 (budget),
 * 60-90 (threshold ratios), 92-115 (chain, widths at a base), 121-168 (search) */
static long long ipow4(int e) {
  long long r = 1;
  for (int i = 0; i < e; ++i) r *= 4;
  return r;
}
static long long gcdll(long long a, long long b) {
  while (b) {
    long long t = a % b;
    a = b;
    b = t;
  }
  return a < 0 ? -a : a;
}
static int gen_level(double f, const double* chain, int nc, double base) {
  int level = 0;
  for (int k = 0; k < nc; ++k)
    if (f >= base * chain[k]) level = k + 1;
  return level;
}
int dqo_allocate_general(const float* F, size_t nsg, double b, uint32_t s, uint32_t S, int hier, const int* W,
                         int n_w, uint8_t* widths, uint32_t* perm, double* u_out, uint64_t* payload_out) {
  static const int allowed[] = {1, 2, 4, 8, 16};
  if (n_w <= 0) return fail(DQO_EINVAL, "width set is empty");
  for (int i = 0; i < n_w; ++i) {
    int ok = 0;
    for (int k = 0; k < 5; ++k) ok |= W[i] == allowed[k];
    if (!ok) return fail(DQO_EINVAL, "unsupported width");
    if (i > 0 && W[i] <= W[i - 1]) return fail(DQO_EINVAL, "width set must be strictly ascending");
  }
  if (!s || S % s) return fail(DQO_EINVAL, "invalid group sizes");
  const double bbar = b - (hier ? 8.0 / s + 16.0 / S : 16.0 / s);
  if (!(bbar > W[0])) return fail(DQO_EINFEASIBLE, "payload budget does not exceed the minimum width");
  const double budget = (double)((uint64_t)nsg * S) * bbar;
  for (size_t j = 0; j < nsg; ++j)
    if (!(F[j] >= 0.0f)) return fail(DQO_EINVAL, "squared norms must be non-negative");
  double u = 0.0;
  if (n_w == 1) {
    for (size_t j = 0; j < nsg; ++j) widths[j] = (uint8_t)W[0];
  } else {
    const int nc = n_w - 1;
    double chain[4];
    chain[0] = 1.0;
    for (int k = 0; k + 1 < nc; ++k) {
      const int a = W[k], bb = W[k + 1], c = W[k + 2];
      long long num = (ipow4(c - bb) - 1) * (bb - a);
      long long den = ipow4(c - bb) * (c - bb) * (ipow4(bb - a) - 1);
      const long long g = gcdll(num, den);
      num /= g;
      den /= g;
      chain[k + 1] = chain[k] / ((double)num / (double)den);
    }
    double* pts = (double*)malloc(sizeof(double) * (nsg * (size_t)nc + 1));
    size_t np = 0;
    for (size_t j = 0; j < nsg; ++j) {
      if (F[j] <= 0.0f) continue;
      for (int k = 0; k < nc; ++k) pts[np++] = (double)F[j] / chain[k];
    }
    qsort(pts, np, sizeof(double), cmp_dbl);
    size_t nu = 0;
    for (size_t i = 0; i < np; ++i)
      if (nu == 0 || pts[i] != pts[nu - 1]) pts[nu++] = pts[i];
    pts[nu] = nu ? pts[nu - 1] * 2.0 + 1.0 : 1.0; /* all-min plateau */
    const size_t M = nu + 1;
#define GEN_PAYLOAD(base, res)                                                   \
  do {                                                                           \
    uint64_t p_ = 0;                                                             \
    for (size_t j_ = 0; j_ < nsg; ++j_)                                          \
      p_ += (uint64_t)W[gen_level((double)F[j_], chain, nc, (base))] * S;        \
    res = p_;                                                                    \
  } while (0)
    size_t lo = 0, hi = M - 1;
    uint64_t p;
    GEN_PAYLOAD(pts[lo], p);
    if ((double)p > budget) {
      while (lo + 1 < hi) {
        const size_t mid = (lo + hi) / 2;
        GEN_PAYLOAD(pts[mid], p);
        if ((double)p <= budget) hi = mid; else lo = mid;
      }
      lo = hi;
    }
#undef GEN_PAYLOAD
    u = pts[lo];
    free(pts);
    for (size_t j = 0; j < nsg; ++j) widths[j] = (uint8_t)W[gen_level((double)F[j], chain, nc, u)];
  }
  uint64_t pay = 0;
  for (size_t j = 0; j < nsg; ++j) pay += (uint64_t)widths[j] * S;
  if ((double)pay > budget) return fail(DQO_EINFEASIBLE, "bit allocation infeasible within budget");
  *u_out = u;
  *payload_out = pay;
  if (perm) dqo_build_permutation(widths, nsg, perm);
  return 0;
}

/* cross-round fast allocator: proj/src/allocation.cpp:262-300.  state = {lo, hi, u}
 * (FastAllocatorState, allocation.hpp:75-79), updated in place. */
int dqo_allocate_fast_stateful(const float* F, size_t nsg, double b, uint32_t s, uint32_t S, int hier,
                               double state[3], uint8_t* widths, uint32_t* perm, double* u_out,
                               uint64_t* payload_out) {
  double bbar;
  int rc = bbar_of(b, s, S, hier, &bbar);
  if (rc) return rc;
  const double alpha = 4.0 / log2(512.0 / 17.0);
  const double budget = (double)nsg * S * bbar;
#define FAST_AT(uu, wout, res)                                                   \
  do {                                                                           \
    const float t24_ = (float)exp2((4.0 - (uu)) / alpha);                        \
    const float t48_ = (float)exp2((8.0 - (uu)) / alpha);                        \
    uint64_t p_ = 0;                                                             \
    for (size_t j_ = 0; j_ < nsg; ++j_) {                                        \
      const uint8_t w_ = F[j_] >= t48_ ? 8 : F[j_] >= t24_ ? 4 : 2;              \
      if (wout) ((uint8_t*)(wout))[j_] = w_;                                     \
      p_ += (uint64_t)w_ * S;                                                    \
    }                                                                            \
    res = p_;                                                                    \
  } while (0)
  uint64_t pay;
  FAST_AT(state[2], widths, pay);
  const int over = (double)pay > budget;
  if (over) {
    /* largest in-budget plateau sample at or below the carried u, scanning down */
    double* flips = (double*)malloc(sizeof(double) * (2 * nsg + 1));
    size_t nf = 0;
    for (size_t j = 0; j < nsg; ++j) {
      if (F[j] <= 0.0f) continue;
      const double l = alpha * log2((double)F[j]);
      flips[nf++] = 4.0 - l;
      flips[nf++] = 8.0 - l;
    }
    qsort(flips, nf, sizeof(double), cmp_dbl);
    size_t nu = 0;
    for (size_t i = 0; i < nf; ++i)
      if (nu == 0 || flips[i] != flips[nu - 1]) flips[nu++] = flips[i];
    size_t ns = nu ? nu + 1 : 1;
    double* samp = (double*)malloc(sizeof(double) * ns);
    if (!nu) samp[0] = 0.0;
    else {
      samp[0] = flips[0] - 1.0;
      for (size_t i = 0; i + 1 < nu; ++i) samp[i + 1] = 0.5 * (flips[i] + flips[i + 1]);
      samp[nu] = flips[nu - 1] + 1.0;
      for (size_t i = 0; i < ns; ++i) samp[i] = samp[i] < -1e6 ? -1e6 : samp[i] > 1e6 ? 1e6 : samp[i];
    }
    free(flips);
    double chosen = -1e6;
    for (size_t i = ns; i-- > 0;) {
      if (samp[i] > state[2]) continue;
      uint64_t p;
      FAST_AT(samp[i], (uint8_t*)NULL, p);
      if ((double)p <= budget) {
        chosen = samp[i];
        break;
      }
    }
    free(samp);
    FAST_AT(chosen, widths, pay);
    if ((double)pay > budget) return fail(DQO_EINFEASIBLE, "bit allocation infeasible within budget");
  }
#undef FAST_AT
  *u_out = state[2];
  *payload_out = pay;
  if (perm) dqo_build_permutation(widths, nsg, perm);
  if (over) state[1] = state[2];
  else state[0] = state[2];
  state[2] = 0.5 * (state[0] + state[1]);
  return 0;
}

/* ------------------------------------------------------------ schedules   */
typedef struct { uint32_t snd, rcv, slot; } rev_t;
typedef struct {
  uint32_t sink, n_red, n_gat, sink_slot, n_slots;
  rev_t red[64 * 8];
} plan_t;
/* proj/src/topology.cpp:8-30 */
static void ring_plan(uint32_t n, uint32_t i, plan_t* p) {
  p->sink = i;
  p->n_red = n - 1;
  for (uint32_t h = 0; h + 1 < n; ++h) p->red[h] = (rev_t){(i + 1 + h) % n, (i + 2 + h) % n, h};
  p->n_gat = n - 1;
  p->sink_slot = n - 1;
  p->n_slots = n;
}
/* proj/src/topology.cpp:32-70 */
static void butterfly_plan(uint32_t n, uint32_t c, plan_t* p) {
  int stages = 0;
  while ((1u << stages) < n) ++stages;
  p->sink = c;
  uint32_t slot = 0;
  for (int l = 0; l < stages; ++l) {
    uint32_t bit = 1u << (stages - 1 - l), high = ~(2 * bit - 1);
    for (uint32_t w = 0; w < n; ++w) {
      if ((w & high) != (c & high) || (w & bit) == (c & bit)) continue;
      p->red[slot] = (rev_t){w, w ^ bit, slot};
      ++slot;
    }
  }
  p->n_red = slot;
  p->n_gat = n - 1;
  p->sink_slot = slot;
  p->n_slots = slot + 1;
}

/* the plans above through the oracle interface: events as (sender, receiver, slot) */
int dqo_schedule(uint32_t n, int topology, uint32_t chunk, uint32_t* events, uint32_t cap, uint32_t* n_events,
                 uint32_t* sink_slot, uint32_t* n_slots, uint32_t* n_gather) {
  if (!n || n > 64 || chunk >= n) return fail(DQO_EINVAL, "bad schedule arguments");
  if (topology == 1 && (n & (n - 1))) return fail(DQO_EINVAL, "butterfly topology requires a power-of-two worker count");
  plan_t p;
  if (topology == 0) ring_plan(n, chunk, &p); else butterfly_plan(n, chunk, &p);
  *n_events = p.n_red;
  *sink_slot = p.sink_slot;
  *n_slots = p.n_slots;
  *n_gather = p.n_gat;
  if (events) {
    if (cap < p.n_red) return fail(DQO_EINVAL, "event capacity");
    for (uint32_t e = 0; e < p.n_red; ++e) {
      events[3 * e] = p.red[e].snd;
      events[3 * e + 1] = p.red[e].rcv;
      events[3 * e + 2] = p.red[e].slot;
    }
  }
  return 0;
}

/* --------------------------------------------------------------- engine   */
static uint64_t fnv(const uint8_t* b, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ULL;
  return h;
}

/* run_round + run_chunk, proj/src/engine.cpp:94-231,269-418 (quantized codec; the
 * lossless debug codec of :24-45 is included for the plumbing tests) */
int dqo_run_round(const float* const* workers, size_t d, const dqo_round_cfg* cfg, float* synced,
                  uint8_t* widths_out, uint32_t* perm_out, dqo_round_out* out) {
  const uint32_t n = cfg->n_workers, s = cfg->group_size, S = cfg->super_group_size;
  memset(out, 0, sizeof *out);
  if (!n || n > 64) return fail(DQO_EINVAL, "n_workers must be in 1..64");
  if (!s || S % s || S % 4) return fail(DQO_EINVAL, "super-group size must be a multiple of the group size and of 4");
  if (!cfg->variable_width && cfg->fixed_width != 2 && cfg->fixed_width != 4 && cfg->fixed_width != 8)
    return fail(DQO_EINVAL, "fixed width must be one of {2,4,8}");
  if ((cfg->allocator == 2) != !cfg->variable_width)
    return fail(DQO_EINVAL, "fixed-width allocator requires variable_width off and vice versa");
  if (cfg->topology == 1 && (n & (n - 1))) return fail(DQO_EINVAL, "butterfly topology requires a power-of-two worker count");
  if (!d) return fail(DQO_EINVAL, "empty gradient");

  double* exact = (double*)calloc(d, sizeof(double));
  for (uint32_t r = 0; r < n; ++r)
    for (size_t i = 0; i < d; ++i) exact[i] += workers[r][i];
  if (n == 1) {
    memcpy(synced, workers[0], d * sizeof(float));
    free(exact);
    return 0;
  }
  const size_t T = (d + S - 1) / S, dp = T * S;
  float* lm = (float*)malloc(sizeof(float) * T * n);
  float* ls = (float*)malloc(sizeof(float) * T * n);
  float *gm = (float*)malloc(sizeof(float) * T), *gs = (float*)malloc(sizeof(float) * T);
  for (uint32_t r = 0; r < n; ++r) dqo_compute_stats(workers[r], d, s, S, lm + r * T, ls + r * T);
  dqo_reduce_stats(lm, ls, n, T, gm, gs);
  free(lm);
  free(ls);

  uint8_t* widths = (uint8_t*)malloc(T);
  uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * T);
  int rc = 0;
  if (cfg->codec == 1) {
    memset(widths, 16, T);
    out->payload_bits = (uint64_t)T * S * 32;
  } else if (!cfg->variable_width) {
    double bbar;
    rc = bbar_of(cfg->budget_bits, s, S, cfg->hierarchical, &bbar);
    if (!rc && cfg->fixed_width > bbar) rc = fail(DQO_EINFEASIBLE, "fixed width exceeds the payload budget");
    memset(widths, cfg->fixed_width, T);
    out->payload_bits = (uint64_t)T * S * cfg->fixed_width;
  } else if (cfg->allocator == 0) {
    static const int W248[3] = {2, 4, 8};  /* engine.cpp:306-307 */
    rc = dqo_allocate_general(gs, T, cfg->budget_bits, s, S, cfg->hierarchical, W248, 3, widths, NULL, &out->u,
                              &out->payload_bits);
  } else {
    rc = dqo_allocate_fast(gs, T, cfg->budget_bits, s, S, cfg->hierarchical, widths, NULL, &out->u,
                           &out->payload_bits);
  }
  if (rc) {
    free(exact); free(gm); free(gs); free(widths); free(perm);
    return rc;
  }
  dqo_build_permutation(widths, T, perm);
  uint8_t* wsorted = (uint8_t*)malloc(T);
  for (size_t k = 0; k < T; ++k) wsorted[k] = widths[perm[k]];

  /* normalized, permuted per-worker data (stats.cpp:56-63, allocation.cpp:319-325) */
  float** P = (float**)malloc(sizeof(float*) * n);
  for (uint32_t r = 0; r < n; ++r) {
    P[r] = (float*)malloc(sizeof(float) * dp);
    for (size_t k = 0; k < T; ++k) {
      size_t src = (size_t)perm[k];
      for (uint32_t e = 0; e < S; ++e) {
        size_t i = src * S + e;
        float v = i < d ? workers[r][i] : 0.0f;
        P[r][k * S + e] = v - gm[src];
      }
    }
  }

  books_t books;
  load_books(&books, cfg->non_uniform);
  dqo_codec cc = {s, S, cfg->hierarchical, cfg->non_uniform};
  float* agg = (float*)malloc(sizeof(float) * dp);
  uint64_t H = 0xcbf29ce484222325ULL;
  for (uint32_t c = 0; c < n && !rc; ++c) {
    plan_t plan;
    if (cfg->topology == 0) ring_plan(n, c, &plan); else butterfly_plan(n, c, &plan);
    const size_t lo = (size_t)((uint64_t)T * c / n), hi = (size_t)((uint64_t)T * (c + 1) / n);
    const size_t nsg = hi - lo, coords = nsg * S;
    const uint8_t* w = wsorted + lo;
    size_t msg_cap = cfg->codec == 1 ? 8 + coords * 4
                                     : dqo_compressed_size_bits(w, nsg, S, s, cfg->hierarchical) / 8;
    uint64_t hsh = 0xcbf29ce484222325ULL;
    float** buf = (float**)malloc(sizeof(float*) * n);
    uint8_t** pend = (uint8_t**)calloc(n, sizeof(uint8_t*));
    int last_in[64 * 8];
    for (uint32_t r = 0; r < n; ++r) {
      buf[r] = (float*)malloc(sizeof(float) * (coords ? coords : 1));
      memcpy(buf[r], P[r] + lo * S, sizeof(float) * coords);
      last_in[r] = -1;
    }
    for (uint32_t e = 0; e < plan.n_red; ++e) last_in[plan.red[e].rcv] = (int)e;
    uint64_t pay = 0, scl = 0;
    for (size_t i = 0; i < nsg; ++i) {
      pay += (uint64_t)S * w[i];
      scl += (uint64_t)(sg_record_bytes(w[i], &cc) - (size_t)S * w[i] / 8) * 8;
    }
    uint8_t* msg = NULL;
    size_t mlen = 0;
    float* tmp = (float*)malloc(sizeof(float) * (coords ? coords : 1));
#define ACCOUNT(bytes, len, fresh)                                            \
  do {                                                                        \
    hsh = fnv((bytes), (len), hsh);                                           \
    out->transmitted_coordinates += coords;                                   \
    if (cfg->codec == 1) {                                                    \
      out->header_bits += 64;                                                 \
      out->wire_payload_bits += (uint64_t)coords * 32;                        \
      if (fresh) { out->repr_bits += (uint64_t)coords * 32; out->compressed_coordinates += coords; } \
    } else {                                                                  \
      out->header_bits += 192;                                                \
      out->wire_payload_bits += pay;                                          \
      out->scale_bits += scl;                                                 \
      if (fresh) { out->repr_bits += pay + scl; out->compressed_coordinates += coords; } \
    }                                                                         \
  } while (0)
    for (uint32_t e = 0; e < plan.n_red && !rc; ++e) {
      const rev_t ev = plan.red[e];
      msg = (uint8_t*)malloc(msg_cap);
      dqo_qctx q = {cfg->seed, cfg->round, c, ev.slot, plan.n_slots, cfg->correlated};
      if (cfg->codec == 1) {
        wr32(msg, c);
        wr32(msg + 4, (uint32_t)coords);
        for (size_t i = 0; i < coords; ++i) {
          float v = buf[ev.snd][i];
          if (pend[ev.snd]) {
            float pv;
            memcpy(&pv, pend[ev.snd] + 8 + 4 * i, 4);
            v = pv + v;
          }
          memcpy(msg + 8 + 4 * i, &v, 4);
        }
        mlen = msg_cap;
      } else if (!pend[ev.snd]) {
        rc = dqo_compress_chunk(buf[ev.snd], w, nsg, &cc, &q, (uint32_t)lo, msg, msg_cap, &mlen);
      } else {
        rc = dqo_dar_chunk(pend[ev.snd], msg_cap, buf[ev.snd], coords, &cc, &q, (uint32_t)lo, msg,
                           msg_cap, &mlen);
      }
      ACCOUNT(msg, mlen, 1);
      const uint32_t r = ev.rcv;
      if ((int)e == last_in[r] && r != plan.sink) {
        free(pend[r]);
        pend[r] = msg;
      } else {
        if (cfg->codec == 1) {
          for (size_t i = 0; i < coords; ++i) {
            float v;
            memcpy(&v, msg + 8 + 4 * i, 4);
            buf[r][i] += v;
          }
        } else if (!rc) {
          rc = dqo_decompress_accumulate(msg, mlen, &cc, buf[r], coords);
        }
        free(msg);
      }
    }
    /* gather: the sink compresses once; the bytes are forwarded n-1 times (engine.cpp:219-229) */
    if (!rc) {
      msg = (uint8_t*)malloc(msg_cap);
      dqo_qctx q = {cfg->seed, cfg->round, c, plan.sink_slot, plan.n_slots, cfg->correlated};
      if (cfg->codec == 1) {
        wr32(msg, c);
        wr32(msg + 4, (uint32_t)coords);
        memcpy(msg + 8, buf[plan.sink], coords * 4);
        mlen = msg_cap;
        memcpy(tmp, buf[plan.sink], coords * 4);
      } else {
        rc = dqo_compress_chunk(buf[plan.sink], w, nsg, &cc, &q, (uint32_t)lo, msg, msg_cap, &mlen);
        if (!rc) rc = dqo_decompress_chunk(msg, mlen, &cc, tmp, coords);
      }
      for (uint32_t g = 0; g < plan.n_gat; ++g) ACCOUNT(msg, mlen, g == 0);
      memcpy(agg + lo * S, tmp, coords * sizeof(float));
      free(msg);
    }
    H ^= hsh + GOLDEN + (H << 6) + (H >> 2);
    out->stats_bits += (uint64_t)(plan.n_red + plan.n_gat) * 64ULL * nsg;
    for (uint32_t r = 0; r < n; ++r) {
      free(buf[r]);
      free(pend[r]);
    }
    free(buf);
    free(pend);
    free(tmp);
  }
  out->wire_hash = H;
  if (!rc) {
    /* unpermute + denormalize, stats.cpp:65-78 */
    for (size_t k = 0; k < T; ++k) {
      size_t j = perm[k];
      float shift = (float)n * gm[j];
      for (uint32_t e = 0; e < S; ++e) {
        size_t i = j * S + e;
        if (i < d) synced[i] = agg[k * S + e] + shift;
      }
    }
    double err = 0.0, ref = 0.0;
    for (size_t i = 0; i < d; ++i) {
      double ee = synced[i] - exact[i];
      err += ee * ee;
      ref += exact[i] * exact[i];
    }
    out->mse = err / (double)d;
    out->vnmse = ref > 0.0 ? err / ref : 0.0;
    if (widths_out) memcpy(widths_out, widths, T);
    if (perm_out) memcpy(perm_out, perm, T * sizeof(uint32_t));
  }
  for (uint32_t r = 0; r < n; ++r) free(P[r]);
  free(P);
  free(agg);
  free(exact);
  free(gm);
  free(gs);
  free(widths);
  free(perm);
  free(wsorted);
  return rc;
}

/* ------------------------------------------------------ synthetic inputs  */
/* proj/src/synth.cpp:19-54: Box-Muller over keyed draws, per-SG log-normal scale */
static double keyed_normal(uint64_t seed, uint32_t purpose, uint64_t stream, uint64_t index) {
  double u1 = dqo_uniform_at(seed, 0, purpose, stream, 0, index);
  double u2 = dqo_uniform_at(seed, 0, purpose, stream, 1, index);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}
int dqo_generate_worker(int kind, size_t d, uint64_t seed, double sigma_log, uint32_t S,
                        uint32_t rank, float* out) {
  if (!d || !S || sigma_log < 0.0) return fail(DQO_EINVAL, "generator arguments");
  if (kind == 0 || sigma_log == 0.0) {
    for (size_t i = 0; i < d; ++i) out[i] = (float)keyed_normal(seed, DQO_GEN_ENTRY, rank, i);
    return 0;
  }
  size_t nsg = (d + S - 1) / S;
  double* sig = (double*)malloc(sizeof(double) * nsg);
  for (size_t j = 0; j < nsg; ++j) sig[j] = exp(sigma_log * keyed_normal(seed, DQO_GEN_SCALE, 0, j));
  for (size_t i = 0; i < d; ++i) out[i] = (float)(sig[i / S] * keyed_normal(seed, DQO_GEN_ENTRY, rank, i));
  free(sig);
  return 0;
}
