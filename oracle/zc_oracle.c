/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the zcomm reference's hot
 * path (see zc_oracle.h).  Each function cites the reference lines it
 * restates (paths relative to /root/reference/proj/core/).  Compiled with
 * -ffp-contract=off so every double operation rounds like the reference's
 * SSE2 build (no FMA contraction).
 */
#include "zc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ frame */
static void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_le(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

/* frame.cpp:35-45 */
void zo_write_header(const zc_frame_header* h, uint8_t* p) {
  put_le(p + 0, h->magic, 4);
  p[4] = h->version;
  p[5] = h->codec;
  put_le(p + 6, h->flags, 2);
  put_le(p + 8, h->raw_bytes, 8);
  put_le(p + 16, h->payload_bytes, 8);
  put_le(p + 24, h->params, 8);
}

/* frame.cpp:47-59 */
int zo_parse_header(const uint8_t* p, uint64_t len, zc_frame_header* h) {
  if (len < ZC_HEADER_BYTES) return 0;
  h->magic = (uint32_t)get_le(p, 4);
  h->version = p[4];
  h->codec = p[5];
  h->flags = (uint16_t)get_le(p + 6, 2);
  h->raw_bytes = get_le(p + 8, 8);
  h->payload_bytes = get_le(p + 16, 8);
  h->params = get_le(p + 24, 8);
  return 1;
}

/* frame.cpp:61-69 */
int zo_validate_header(const zc_frame_header* h, uint64_t region) {
  if (h->magic != ZC_FRAME_MAGIC) return 0;
  if (h->version != ZC_FRAME_VERSION) return 0;
  if (h->codec > ZC_CODEC_HUFFMAN) return 0;
  if (h->raw_bytes == 0) return 0;
  if (region < ZC_HEADER_BYTES || h->payload_bytes > region - ZC_HEADER_BYTES) return 0;
  if (h->codec == ZC_CODEC_RAW && h->payload_bytes != h->raw_bytes) return 0;
  return 1;
}

static void make_header(zc_frame_header* h, int codec, uint16_t flags, uint64_t raw, uint64_t payload,
                        uint64_t params) {
  h->magic = ZC_FRAME_MAGIC;
  h->version = ZC_FRAME_VERSION;
  h->codec = (uint8_t)codec;
  h->flags = flags;
  h->raw_bytes = raw;
  h->payload_bytes = payload;
  h->params = params;
}

/* frame.cpp:71-81 */
uint64_t zo_frame_commit_raw(const uint8_t* raw, uint64_t n, uint8_t* region, uint64_t cap) {
  if (n == 0) return 0;
  if (cap < ZC_HEADER_BYTES || cap - ZC_HEADER_BYTES < n) return 0;
  zc_frame_header h;
  make_header(&h, ZC_CODEC_RAW, 0, n, n, 0);
  zo_write_header(&h, region);
  memmove(region + ZC_HEADER_BYTES, raw, n);
  return ZC_HEADER_BYTES + n;
}

/* ------------------------------------------------------------------ quant */
/* quant.cpp:22-27: half-away-from-zero; |q| >= 2147483647.5 rejected */
static int round_to_symbol(double q, int32_t* out) {
  if (fabs(q) >= 2147483647.5) return ZC_DERR_RANGE;
  *out = (int32_t)llround(q);
  return 0;
}

/* quant.cpp:43-62 (eb_quantize_with_scale / eb_quantize_chunk). The reference checks finiteness of
 * the whole input before quantizing; errors are reported as the OR of what was found. */
int zo_eb_quantize_f64(const double* x, uint64_t n, double scale, int32_t* out) {
  if (!(scale > 0.0) || !isfinite(scale)) return -1;
  int err = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) err |= ZC_DERR_NONFINITE;
  if (err) return err;
  for (uint64_t i = 0; i < n; ++i) {
    int e = round_to_symbol(x[i] / scale, &out[i]);
    if (e) return e;
  }
  return 0;
}

int zo_eb_quantize_f32(const float* x, uint64_t n, double scale, int32_t* out) {
  if (!(scale > 0.0) || !isfinite(scale)) return -1;
  for (uint64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return ZC_DERR_NONFINITE;
  for (uint64_t i = 0; i < n; ++i) {
    int e = round_to_symbol((double)x[i] / scale, &out[i]);
    if (e) return e;
  }
  return 0;
}

/* quant.cpp:13-20 */
int zo_absmax_f32(const float* x, uint64_t n, double* out) {
  double m = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    if (!isfinite(x[i])) return ZC_DERR_NONFINITE;
    double a = fabs((double)x[i]);
    if (a > m) m = a;
  }
  *out = m;
  return 0;
}

/* --------------------------------------------------------------- QSGD (quant.cpp:64-98) */
/* std::mt19937_64 (libstdc++, the reference's generator; C++ [rand.eng.mers] parameters:
 * w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555 s=17 b=0x71D67FFFEDA60000
 * t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005). */
void zo_mt64_seed(zo_mt64* g, uint64_t seed) {
  g->x[0] = seed;
  for (int i = 1; i < 312; ++i) g->x[i] = 6364136223846793005ull * (g->x[i - 1] ^ (g->x[i - 1] >> 62)) + (uint64_t)i;
  g->i = 312;
}
uint64_t zo_mt64_next(zo_mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (g->x[k] & 0xFFFFFFFF80000000ull) | (g->x[(k + 1) % 312] & 0x7FFFFFFFull);
      g->x[k] = g->x[(k + 156) % 312] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ull : 0ull);
    }
    g->i = 0;
  }
  uint64_t z = g->x[g->i++];
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  z ^= z >> 43;
  return z;
}

/* qsgd_quantize_chunk (quant.cpp:64-82) with rng = mt19937_64(seed) advanced by `skip` draws. */
int zo_qsgd_quantize_chunk_f32(const float* x, uint64_t n, uint32_t levels, double norm, uint64_t seed, uint64_t skip,
                               int32_t* out) {
  if (levels == 0 || levels > (1u << 30)) return -1;
  if (!(norm >= 0.0) || !isfinite(norm)) return -1;
  zo_mt64 g;
  zo_mt64_seed(&g, seed);
  for (uint64_t k = 0; k < skip; ++k) zo_mt64_next(&g);
  double scale = norm == 0.0 ? 1.0 : norm;
  for (uint64_t i = 0; i < n; ++i) {
    double v = (double)x[i];
    if (!isfinite(v)) return ZC_DERR_NONFINITE;
    double u = norm == 0.0 ? 0.0 : (double)levels * fabs(v) / scale;
    double fl = floor(u);
    double frac = u - fl;
    double draw = (double)(zo_mt64_next(&g) >> 11) * 0x1.0p-53;
    int64_t mag = (int64_t)fl + (draw < frac ? 1 : 0);
    out[i] = (int32_t)(v < 0.0 ? -mag : mag);
  }
  return 0;
}

/* qsgd_quantize (quant.cpp:84-98): the norm is the sequential double sum of squares. */
int zo_qsgd_quantize_f32(const float* x, uint64_t n, uint32_t levels, uint64_t seed, int32_t* out, double* scale) {
  double sumsq = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    double v = (double)x[i];
    if (!isfinite(v)) return ZC_DERR_NONFINITE;
    sumsq += v * v;
  }
  double norm = sqrt(sumsq);
  *scale = norm == 0.0 ? 1.0 : norm;
  return zo_qsgd_quantize_chunk_f32(x, n, levels, norm, seed, 0, out);
}

/* quant.cpp:107-127 */
void zo_dequantize_f64(const int32_t* s, uint64_t n, int mode, double scale, uint32_t levels, double* out) {
  if (mode == ZC_QUANT_ERROR_BOUNDED) {
    for (uint64_t i = 0; i < n; ++i) out[i] = scale * (double)s[i];
  } else if (mode == ZC_QUANT_QSGD) {
    double k = scale / (double)levels;
    for (uint64_t i = 0; i < n; ++i) out[i] = k * (double)s[i];
  } else {
    for (uint64_t i = 0; i < n; ++i) out[i] = (double)s[i];
  }
}
void zo_dequantize_f32(const int32_t* s, uint64_t n, int mode, double scale, uint32_t levels, float* out) {
  double k = mode == ZC_QUANT_ERROR_BOUNDED ? scale : mode == ZC_QUANT_QSGD ? scale / (double)levels : 1.0;
  for (uint64_t i = 0; i < n; ++i) out[i] = (float)(mode == ZC_QUANT_PREQUANTIZED ? (double)s[i] : k * (double)s[i]);
}

/* --------------------------------------------------------------- fixedlen */
/* fixedlen.hpp:14-19 */
uint32_t zo_zigzag(int32_t v) { return ((uint32_t)v << 1) ^ (uint32_t)(v >> 31); }
static int32_t unzigzag(uint32_t z) { return (int32_t)(z >> 1) ^ -(int32_t)(z & 1); }

static uint32_t bit_width32(uint32_t v) { return v ? 32u - (uint32_t)__builtin_clz(v) : 0u; }

/* fixedlen.cpp:8-13 */
uint32_t zo_fixedlen_width(const int32_t* s, uint64_t n) {
  uint32_t m = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t z = zo_zigzag(s[i]);
    if (z > m) m = z;
  }
  return m == 0 ? 1u : bit_width32(m);
}

/* fixedlen.cpp:15-37 */
uint64_t zo_fixedlen_encode(const int32_t* s, uint64_t n, uint8_t* out, uint64_t cap, uint32_t* w_out) {
  if (n == 0) return 0;
  uint32_t w = zo_fixedlen_width(s, n);
  if (w_out) *w_out = w;
  uint64_t need = (n * w + 7) / 8;
  if (cap < need) return 0;
  uint64_t acc = 0, o = 0;
  unsigned nb = 0;
  for (uint64_t i = 0; i < n; ++i) {
    acc |= (uint64_t)zo_zigzag(s[i]) << nb;
    nb += w;
    while (nb >= 8) {
      out[o++] = (uint8_t)acc;
      acc >>= 8;
      nb -= 8;
    }
  }
  if (nb > 0) out[o++] = (uint8_t)acc;
  return o;
}

/* fixedlen.cpp:39-65 */
int zo_fixedlen_decode(const zc_frame_header* h, const uint8_t* payload, uint64_t plen, uint8_t* dst,
                       uint64_t dlen) {
  uint32_t w = (uint32_t)h->params;
  if (w < 1 || w > 32 || h->params > 32) return 0;
  if (h->raw_bytes == 0 || h->raw_bytes % 4 != 0) return 0;
  if (dlen < h->raw_bytes) return 0;
  uint64_t count = h->raw_bytes / 4;
  uint64_t need = (count * w + 7) / 8;
  if (h->payload_bytes < need || plen < need) return 0;
  uint64_t mask = (1ull << w) - 1, acc = 0, ip = 0;
  unsigned nb = 0;
  for (uint64_t i = 0; i < count; ++i) {
    while (nb < w) {
      acc |= (uint64_t)payload[ip++] << nb;
      nb += 8;
    }
    int32_t v = unzigzag((uint32_t)(acc & mask));
    acc >>= w;
    nb -= w;
    memcpy(dst + 4 * i, &v, 4);
  }
  return 1;
}

/* ---------------------------------------------------------------- huffman */
static uint32_t reverse_bits(uint32_t v, unsigned n) {
  uint32_t r = 0;
  for (unsigned i = 0; i < n; ++i) {
    r = (r << 1) | (v & 1);
    v >>= 1;
  }
  return r;
}

/* huffman.cpp:23-68: pairwise merge; each pick takes the live node of least (weight, creation
 * order); leaves are created in symbol order, merged nodes after them.  Every symbol's length is
 * the number of merges its subtree took part in. */
static void huff_merge_lengths(const uint64_t* freq, uint8_t* lens) {
  uint64_t w[512];
  int32_t ord[512];
  int32_t alive[512];
  int32_t group[256];
  uint32_t depth[256];
  int nn = 0, order = 0, live = 0;
  memset(lens, 0, 256);
  memset(depth, 0, sizeof(depth));
  for (int s = 0; s < 256; ++s) {
    group[s] = -1;
    if (freq[s] > 0) {
      w[nn] = freq[s];
      ord[nn] = order++;
      alive[nn] = 1;
      group[s] = nn;
      ++nn;
      ++live;
    }
  }
  if (live == 0) return;
  if (live == 1) {
    for (int s = 0; s < 256; ++s)
      if (freq[s] > 0) lens[s] = 1;
    return;
  }
  while (live > 1) {
    int pick[2];
    for (int k = 0; k < 2; ++k) {
      int best = -1;
      for (int i = 0; i < nn; ++i) {
        if (!alive[i]) continue;
        if (best < 0 || w[i] < w[best] || (w[i] == w[best] && ord[i] < ord[best])) best = i;
      }
      alive[best] = 0;
      pick[k] = best;
    }
    int m = nn++;
    w[m] = w[pick[0]] + w[pick[1]];
    ord[m] = order++;
    alive[m] = 1;
    --live;
    for (int s = 0; s < 256; ++s) {
      if (group[s] == pick[0] || group[s] == pick[1]) {
        ++depth[s];
        group[s] = m;
      }
    }
  }
  for (int s = 0; s < 256; ++s)
    if (freq[s] > 0) lens[s] = (uint8_t)depth[s];
}

/* huffman.cpp:72-95: cap at 32 and repair Kraft by deepening the deepest (< cap) leaf, highest
 * symbol first among equals. */
static void huff_limit(uint8_t* lens) {
  const unsigned cap = ZC_HUFF_MAX_CODE_LEN;
  uint64_t kraft = 0;
  for (int s = 0; s < 256; ++s) {
    if (lens[s] == 0) continue;
    if (lens[s] > cap) lens[s] = (uint8_t)cap;
    kraft += 1ull << (cap - lens[s]);
  }
  const uint64_t one = 1ull << cap;
  while (kraft > one) {
    int pick = -1;
    unsigned pl = 0;
    for (int s = 0; s < 256; ++s) {
      unsigned l = lens[s];
      if (l > 0 && l < cap && l >= pl) {
        pl = l;
        pick = s;
      }
    }
    if (pick < 0) break;
    lens[pick]++;
    kraft -= 1ull << (cap - pl - 1);
  }
}

void zo_huff_lengths(const uint64_t* hist, uint8_t* lens) {
  huff_merge_lengths(hist, lens);
  huff_limit(lens);
}

/* huffman.cpp:97-161 */
static int huff_finalize(const uint8_t* lens, zo_huff* c) {
  memset(c, 0, sizeof(*c));
  memcpy(c->len, lens, 256);
  uint32_t bl[34] = {0};
  unsigned minl = 0, maxl = 0, nsyms = 0;
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (!l) continue;
    if (l > ZC_HUFF_MAX_CODE_LEN) return 0;
    ++bl[l];
    ++nsyms;
    if (minl == 0 || l < minl) minl = l;
    if (l > maxl) maxl = l;
  }
  if (nsyms == 0) return 0;
  uint64_t kraft = 0;
  for (unsigned l = 1; l <= maxl; ++l) kraft += (uint64_t)bl[l] << (ZC_HUFF_MAX_CODE_LEN - l);
  if (kraft > (1ull << ZC_HUFF_MAX_CODE_LEN)) return 0;
  uint64_t next[34] = {0}, code = 0;
  for (unsigned l = 1; l <= maxl; ++l) {
    code = (code + bl[l - 1]) << 1;
    next[l] = code;
    c->first_code[l] = code;
  }
  uint32_t idx = 0;
  for (unsigned l = 1; l <= maxl; ++l) {
    c->first_index[l] = idx;
    c->count_at_len[l] = bl[l];
    idx += bl[l];
  }
  uint32_t fill[34] = {0};
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (!l) continue;
    c->code[s] = (uint32_t)next[l]++;
    c->sym_order[c->first_index[l] + fill[l]] = (uint8_t)s;
    ++fill[l];
  }
  for (int s = 0; s < 256; ++s)
    if (lens[s]) c->rev[s] = reverse_bits(c->code[s], lens[s]);
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (l == 0 || l > ZC_HUFF_ROOT_BITS) continue;
    uint16_t e = (uint16_t)(s | (l << 8));
    for (uint32_t pad = 0; pad < (1u << (ZC_HUFF_ROOT_BITS - l)); ++pad) c->lut[c->rev[s] | (pad << l)] = e;
  }
  c->min_len = minl;
  c->max_len = maxl;
  c->valid = 1;
  return 1;
}

int zo_huff_build(const uint64_t* hist, zo_huff* out) {
  uint8_t lens[256];
  zo_huff_lengths(hist, lens);
  if (!huff_finalize(lens, out)) {
    memset(out, 0, sizeof(*out));
    return 0;
  }
  return 1;
}

int zo_huff_from_lengths(const uint8_t* lens, zo_huff* out) { return huff_finalize(lens, out); }

/* collectives.cpp:99-106 */
int zo_huff_from_bytes(const uint8_t* sample, uint64_t n, zo_huff* out) {
  uint64_t h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1;
  for (uint64_t i = 0; i < n; ++i) h[sample[i]]++;
  return zo_huff_build(h, out);
}

/* huffman.cpp:200-214 */
int zo_huff_expected_len(const zo_huff* c, const uint64_t* hist, double* bits_out) {
  if (!c || !c->valid) return 0;
  uint64_t total = 0;
  double bits = 0.0;
  for (int s = 0; s < 256; ++s) {
    uint64_t f = hist[s];
    if (!f) continue;
    if (c->len[s] == 0) return 0;
    total += f;
    bits += (double)f * c->len[s];
  }
  if (!total) return 0;
  *bits_out = bits / (double)total;
  return 1;
}

/* huffman.cpp:182-198 */
int zo_huff_self_len(const uint64_t* hist, double* bits_out) {
  uint8_t lens[256];
  zo_huff_lengths(hist, lens);
  uint64_t total = 0;
  double bits = 0.0;
  for (int s = 0; s < 256; ++s) {
    uint64_t f = hist[s];
    if (!f) continue;
    if (lens[s] == 0) return 0;
    total += f;
    bits += (double)f * lens[s];
  }
  if (!total) return 0;
  *bits_out = bits / (double)total;
  return 1;
}

/* huffman.cpp:216-246 */
uint64_t zo_huffman_encode(const uint8_t* raw, uint64_t n, const zo_huff* c, uint8_t* out, uint64_t cap,
                           int embed) {
  if (!c || !c->valid) return 0;
  if (n == 0 && !embed) return 0;
  uint64_t o = 0;
  if (embed) {
    if (cap < ZC_HUFF_CODEBOOK_BYTES) return 0;
    memcpy(out, c->len, 256);
    o = 256;
  }
  uint64_t acc = 0;
  unsigned nb = 0;
  for (uint64_t i = 0; i < n; ++i) {
    unsigned l = c->len[raw[i]];
    if (!l) return 0;
    acc |= (uint64_t)c->rev[raw[i]] << nb;
    nb += l;
    while (nb >= 8) {
      if (o >= cap) return 0;
      out[o++] = (uint8_t)acc;
      acc >>= 8;
      nb -= 8;
    }
  }
  if (nb > 0) {
    if (o >= cap) return 0;
    out[o++] = (uint8_t)acc;
  }
  return o;
}

/* huffman.cpp:248-316 */
int zo_huffman_decode(const zc_frame_header* h, const uint8_t* payload, uint64_t plen, const zo_huff* shared,
                      uint8_t* dst, uint64_t dlen) {
  if (dlen < h->raw_bytes) return 0;
  if (h->payload_bytes > plen) return 0;
  const uint8_t* stream = payload;
  uint64_t slen = h->payload_bytes;
  zo_huff emb;
  const zo_huff* c;
  if (h->flags & ZC_FLAG_EMBEDDED_CODEBOOK) {
    if (h->params != ZC_HUFF_CODEBOOK_BYTES || slen < ZC_HUFF_CODEBOOK_BYTES) return 0;
    if (!huff_finalize(stream, &emb)) return 0;
    c = &emb;
    stream += 256;
    slen -= 256;
  } else {
    if (h->params != 0) return 0;
    if (!shared || !shared->valid) return 0;
    c = shared;
  }
  const uint64_t total_bits = slen * 8;
  uint64_t bitpos = 0, acc = 0, ip = 0;
  unsigned nb = 0;
  for (uint64_t i = 0; i < h->raw_bytes; ++i) {
    while (nb <= 56 && ip < slen) {
      acc |= (uint64_t)stream[ip++] << nb;
      nb += 8;
    }
    uint16_t e = c->lut[acc & ((1u << ZC_HUFF_ROOT_BITS) - 1)];
    unsigned l = e >> 8;
    uint8_t sym = 0;
    if (l) {
      sym = (uint8_t)(e & 0xFF);
    } else {
      uint64_t val = 0;
      unsigned k = 0;
      int found = 0;
      while (k < c->max_len) {
        if (k >= nb) return 0;
        val = (val << 1) | ((acc >> k) & 1);
        ++k;
        if (k >= c->min_len && c->count_at_len[k] > 0 && val >= c->first_code[k] &&
            val < c->first_code[k] + c->count_at_len[k]) {
          sym = c->sym_order[c->first_index[k] + (uint32_t)(val - c->first_code[k])];
          l = k;
          found = 1;
          break;
        }
      }
      if (!found) return 0;
    }
    if (bitpos + l > total_bits || l > nb) return 0;
    acc >>= l;
    nb -= l;
    bitpos += l;
    dst[i] = sym;
  }
  return 1;
}

/* -------------------------------------------------------------------- rea */
/* rea.hpp:64-79, 50-53 */
void zo_default_arb_config(zc_arb_config* c) {
  memset(c, 0, sizeof(*c));
  c->small_batch_threshold_bytes = 4096;
  c->huffman_min_raw_bytes = 65536;
  c->min_gain_permil = 50;
  c->embed_codebook = 0;
  c->lam_enc = 0.25;
  c->lam_dec = 0.25;
  c->cost.fixedlen.alpha_sec = 1.0e-6;
  c->cost.fixedlen.enc_bytes_per_sec = 250.0e9;
  c->cost.fixedlen.dec_bytes_per_sec = 300.0e9;
  c->cost.huffman.alpha_sec = 1.5e-6;
  c->cost.huffman.enc_bytes_per_sec = 120.0e9;
  c->cost.huffman.dec_bytes_per_sec = 150.0e9;
}

/* rea.cpp:93-118 */
void zo_profile_sample(const uint8_t* raw, uint64_t n, const zo_huff* ctx, zc_sample_stats* st) {
  memset(st, 0, sizeof(*st));
  st->sampled_bytes = n < ZC_SAMPLE_WINDOW_BYTES ? n : ZC_SAMPLE_WINDOW_BYTES;
  for (uint64_t i = 0; i < st->sampled_bytes; ++i) st->hist[raw[i]]++;
  for (uint64_t i = 0; i + 4 <= st->sampled_bytes; i += 4) {
    uint32_t u = (uint32_t)get_le(raw + i, 4);
    uint32_t z = zo_zigzag((int32_t)u);
    if (z > st->max_zigzag) st->max_zigzag = z;
  }
  double b;
  if (ctx && ctx->valid && zo_huff_expected_len(ctx, st->hist, &b)) {
    st->ctx_code_len_bits = b;
    st->ctx_code_len_valid = 1;
  }
  if (zo_huff_self_len(st->hist, &b)) {
    st->self_code_len_bits = b;
    st->self_code_len_valid = 1;
  }
}

/* rea.cpp:120-143 */
uint64_t zo_predict_payload(int codec, uint64_t raw, const zc_sample_stats* st, const zc_arb_config* cfg) {
  if (codec == ZC_CODEC_RAW) return raw;
  if (codec == ZC_CODEC_FIXEDLEN) {
    if (raw < 4 || raw % 4 != 0) return 0;
    unsigned w = 1;
    while ((1ull << w) <= st->max_zigzag && w < 32) ++w;
    return (raw / 4 * w + 7) / 8;
  }
  if (codec == ZC_CODEC_HUFFMAN) {
    int valid = cfg->embed_codebook ? st->self_code_len_valid : st->ctx_code_len_valid;
    if (!valid) return 0;
    double el = cfg->embed_codebook ? st->self_code_len_bits : st->ctx_code_len_bits;
    double bits = (double)raw * el;
    uint64_t p = (uint64_t)((bits + 7.0) / 8.0);
    if (cfg->embed_codebook) p += ZC_HUFF_CODEBOOK_BYTES;
    return p;
  }
  return raw;
}

/* rea.cpp:22-25 */
static int gain_ok(uint64_t raw, uint64_t p, uint32_t permil) {
  if (p >= raw) return 0;
  return (raw - p) * 1000ull >= (uint64_t)permil * raw;
}

/* rea.cpp:31-44 */
static void make_estimate(zc_codec_estimate* e, int codec, uint64_t raw, uint64_t p, const zc_transport_hint* hint,
                          const zc_arb_config* cfg) {
  const zc_codec_cost* cc =
      codec == ZC_CODEC_FIXEDLEN ? &cfg->cost.fixedlen : codec == ZC_CODEC_HUFFMAN ? &cfg->cost.huffman : &cfg->cost.raw;
  e->codec = (uint32_t)codec;
  e->predicted_payload = p;
  e->enc_sec = cc->enc_bytes_per_sec > 0.0 ? (double)raw / cc->enc_bytes_per_sec : 0.0;
  e->dec_sec = cc->dec_bytes_per_sec > 0.0 ? (double)raw / cc->dec_bytes_per_sec : 0.0;
  double beta = hint->beta_eff_bytes_per_sec > 0.0 ? hint->beta_eff_bytes_per_sec : INFINITY;
  double t = cc->alpha_sec + cfg->lam_enc * e->enc_sec;
  t = t + (double)p / beta;
  t = t + cfg->lam_dec * e->dec_sec;
  e->predicted_sec = t;
  e->admissible = 0;
}

/* rea.cpp:145-176 */
void zo_arbitrate_plan(uint64_t raw, uint64_t cap, const zc_sample_stats* st, const zc_transport_hint* hint,
                       const zo_huff* ctx, const zc_arb_config* cfg, zc_arbitration_plan* plan) {
  memset(plan, 0, sizeof(*plan));
  make_estimate(&plan->raw, ZC_CODEC_RAW, raw, raw, hint, cfg);
  plan->raw.admissible = raw > 0 && raw <= cap;
  uint64_t pf = zo_predict_payload(ZC_CODEC_FIXEDLEN, raw, st, cfg);
  make_estimate(&plan->fixedlen, ZC_CODEC_FIXEDLEN, raw, pf, hint, cfg);
  plan->fixedlen.admissible = pf > 0 && pf <= cap && gain_ok(raw, pf, cfg->min_gain_permil);
  uint64_t ph = zo_predict_payload(ZC_CODEC_HUFFMAN, raw, st, cfg);
  make_estimate(&plan->huffman, ZC_CODEC_HUFFMAN, raw, ph, hint, cfg);
  int usable = cfg->embed_codebook || (ctx && ctx->valid);
  plan->huffman.admissible =
      ph > 0 && usable && raw >= cfg->huffman_min_raw_bytes && ph <= cap && gain_ok(raw, ph, cfg->min_gain_permil);
  plan->choice = ZC_CODEC_RAW;
  double best = plan->raw.predicted_sec;
  if (plan->fixedlen.admissible && plan->fixedlen.predicted_sec < best) {
    plan->choice = ZC_CODEC_FIXEDLEN;
    best = plan->fixedlen.predicted_sec;
  }
  if (plan->huffman.admissible && plan->huffman.predicted_sec < best) plan->choice = ZC_CODEC_HUFFMAN;
}

static void commit_raw(const uint8_t* raw, uint64_t n, uint8_t* stage, uint64_t cap, zc_encode_result* r) {
  uint64_t t = zo_frame_commit_raw(raw, n, stage, cap);
  memset(r, 0, sizeof(*r));
  if (t == 0) return;
  r->codec = ZC_CODEC_RAW;
  r->payload_bytes = n;
  r->total_bytes = t;
}

static void full_hist(const uint8_t* raw, uint64_t n, uint64_t* h) {
  memset(h, 0, 256 * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) h[raw[i]]++;
}

/* rea.cpp:178-238 (Algorithm 1) */
void zo_encode_best(const uint8_t* raw, uint64_t n, uint8_t* stage, uint64_t cap, const zc_transport_hint* hint,
                    const zo_huff* ctx, const zc_arb_config* cfg, zc_encode_result* r) {
  memset(r, 0, sizeof(*r));
  if (n == 0 || cap <= ZC_HEADER_BYTES) return;
  uint64_t pcap = cap - ZC_HEADER_BYTES;
  if (n <= cfg->small_batch_threshold_bytes) {
    commit_raw(raw, n, stage, cap, r);
    return;
  }
  zc_sample_stats st;
  zo_profile_sample(raw, n, ctx, &st);
  zc_arbitration_plan plan;
  zo_arbitrate_plan(n, pcap, &st, hint, ctx, cfg, &plan);
  uint8_t* pd = stage + ZC_HEADER_BYTES;
  if (plan.choice == ZC_CODEC_FIXEDLEN) {
    int32_t* syms = (int32_t*)malloc((n / 4 ? n / 4 : 1) * 4);
    memcpy(syms, raw, n / 4 * 4);
    uint32_t w = 0;
    uint64_t p = zo_fixedlen_encode(syms, n / 4, pd, pcap, &w);
    free(syms);
    if (p > 0 && p <= pcap && gain_ok(n, p, cfg->min_gain_permil)) {
      zc_frame_header h;
      make_header(&h, ZC_CODEC_FIXEDLEN, 0, n, p, w);
      zo_write_header(&h, stage);
      r->codec = ZC_CODEC_FIXEDLEN;
      r->payload_bytes = p;
      r->total_bytes = ZC_HEADER_BYTES + p;
      return;
    }
  } else if (plan.choice == ZC_CODEC_HUFFMAN) {
    zo_huff own;
    const zo_huff* use = ctx;
    if (cfg->embed_codebook) {
      uint64_t h[256];
      full_hist(raw, n, h);
      zo_huff_build(h, &own);
      use = &own;
    }
    if (use && use->valid) {
      uint64_t p = zo_huffman_encode(raw, n, use, pd, pcap, (int)cfg->embed_codebook);
      if (p > 0 && p <= pcap && gain_ok(n, p, cfg->min_gain_permil)) {
        zc_frame_header h;
        make_header(&h, ZC_CODEC_HUFFMAN, cfg->embed_codebook ? ZC_FLAG_EMBEDDED_CODEBOOK : 0, n, p,
                    cfg->embed_codebook ? ZC_HUFF_CODEBOOK_BYTES : 0);
        zo_write_header(&h, stage);
        r->codec = ZC_CODEC_HUFFMAN;
        r->payload_bytes = p;
        r->total_bytes = ZC_HEADER_BYTES + p;
        return;
      }
    }
  }
  commit_raw(raw, n, stage, cap, r);
}

/* collectives.cpp:213-281 (codec dispatch inside send_batch) */
void zo_send_batch(const uint8_t* raw, uint64_t n, uint8_t* stage, uint64_t cap, int pin,
                   const zc_transport_hint* hint, const zo_huff* ctx, const zc_arb_config* cfg,
                   zc_encode_result* r) {
  memset(r, 0, sizeof(*r));
  if (pin == ZC_PIN_AUTO) {
    zo_encode_best(raw, n, stage, cap, hint, ctx, cfg, r);
    return;
  }
  if (pin == ZC_PIN_FIXEDLEN && n >= 4 && n % 4 == 0 && cap >= ZC_HEADER_BYTES) {
    int32_t* syms = (int32_t*)malloc(n);
    memcpy(syms, raw, n);
    uint32_t w = 0;
    uint64_t p = zo_fixedlen_encode(syms, n / 4, stage + ZC_HEADER_BYTES, cap - ZC_HEADER_BYTES, &w);
    free(syms);
    if (p > 0) {
      zc_frame_header h;
      make_header(&h, ZC_CODEC_FIXEDLEN, 0, n, p, w);
      zo_write_header(&h, stage);
      r->codec = ZC_CODEC_FIXEDLEN;
      r->payload_bytes = p;
      r->total_bytes = ZC_HEADER_BYTES + p;
      return;
    }
  }
  if (pin == ZC_PIN_HUFFMAN && cap >= ZC_HEADER_BYTES) {
    zo_huff own;
    const zo_huff* use = ctx;
    if (cfg->embed_codebook) {
      uint64_t h[256];
      full_hist(raw, n, h);
      zo_huff_build(h, &own);
      use = &own;
    }
    if (use && use->valid) {
      uint64_t p = zo_huffman_encode(raw, n, use, stage + ZC_HEADER_BYTES, cap - ZC_HEADER_BYTES,
                                     (int)cfg->embed_codebook);
      if (p > 0) {
        zc_frame_header h;
        make_header(&h, ZC_CODEC_HUFFMAN, cfg->embed_codebook ? ZC_FLAG_EMBEDDED_CODEBOOK : 0, n, p,
                    cfg->embed_codebook ? ZC_HUFF_CODEBOOK_BYTES : 0);
        zo_write_header(&h, stage);
        r->codec = ZC_CODEC_HUFFMAN;
        r->payload_bytes = p;
        r->total_bytes = ZC_HEADER_BYTES + p;
        return;
      }
    }
  }
  commit_raw(raw, n, stage, cap, r);
}

/* collectives.cpp:304-336 (decode dispatch inside recv_batch) */
int zo_recv_batch(const uint8_t* frame, uint64_t flen, const zo_huff* ctx, uint8_t* dst, uint64_t dlen) {
  zc_frame_header h;
  int decoded = 0, codec = -1;
  if (zo_parse_header(frame, flen, &h) && zo_validate_header(&h, flen) && h.raw_bytes == dlen) {
    const uint8_t* p = frame + ZC_HEADER_BYTES;
    if (h.codec == ZC_CODEC_RAW) {
      memcpy(dst, p, dlen);
      decoded = 1;
    } else if (h.codec == ZC_CODEC_FIXEDLEN) {
      decoded = zo_fixedlen_decode(&h, p, h.payload_bytes, dst, dlen);
    } else {
      decoded = zo_huffman_decode(&h, p, h.payload_bytes, ctx, dst, dlen);
    }
    if (decoded) codec = h.codec;
  }
  if (!decoded) {
    uint64_t have = flen > ZC_HEADER_BYTES ? flen - ZC_HEADER_BYTES : 0;
    memcpy(dst, frame + ZC_HEADER_BYTES, dlen < have ? dlen : have);
    codec = -1;
  }
  return codec;
}

/* ------------------------------------------------------------ collectives */
static void wire_add(zc_wire_stats* w, const zc_encode_result* r, uint64_t raw) {
  if (!w) return;
  w->frames_by_codec[r->codec]++;
  w->raw_bytes += raw;
  w->payload_bytes += r->payload_bytes;
  w->total_bytes += r->total_bytes;
}

/* One lockstep exchange of `bytes` per rank (collectives.cpp:366-396): each rank's outgoing span is
 * cut into chunk_raw_bytes batches (4 MiB, or 512 KiB slots), encoded, and decoded by the successor into scratch.  src[r] is rank r's
 * outgoing span; dst[r] receives what rank r gets from its predecessor.  add != 0 selects the RS
 * sink (int64-checked add into dst). */
/* RankCtx::chunk_raw_bytes (collectives.cpp:197-199): 512 KiB slots under
 * CollectiveConfig::perSlotFraming, else 4 MiB batches.  Every exchange of the ring simulation cuts
 * its spans at this size; the stage capacity stays one bank (kStageBankBytes). */
static uint64_t g_chunk_raw = ZC_BATCH_RAW_BYTES;
void zo_set_per_slot_framing(int on) { g_chunk_raw = on ? ZC_SLOT_BYTES : ZC_BATCH_RAW_BYTES; }

static int ring_exchange(int n, uint8_t** src, uint8_t** dst, uint64_t bytes, int pin, int add,
                         const zc_transport_hint* hint, const zo_huff* ctx, const zc_arb_config* cfg,
                         zc_wire_stats* wire) {
  if (bytes == 0) return 0;
  const uint64_t step = g_chunk_raw;
  uint8_t* stage = (uint8_t*)malloc(ZC_STAGE_BANK_BYTES);
  uint8_t* scratch = (uint8_t*)malloc(ZC_BATCH_RAW_BYTES);
  uint8_t** frames = (uint8_t**)calloc((size_t)n, sizeof(uint8_t*));
  uint64_t* flen = (uint64_t*)calloc((size_t)n, sizeof(uint64_t));
  int rc = 0;
  for (int r = 0; r < n; ++r) frames[r] = (uint8_t*)malloc(ZC_STAGE_BANK_BYTES);
  for (uint64_t off = 0; off < bytes && rc == 0; off += step) {
    uint64_t len = bytes - off < step ? bytes - off : step;
    for (int r = 0; r < n; ++r) {
      zc_encode_result er;
      zo_send_batch(src[r] + off, len, frames[r], ZC_STAGE_BANK_BYTES, pin, hint, ctx, cfg, &er);
      if (er.total_bytes == 0) {
        rc = ZC_ERR_RUNTIME;
        break;
      }
      flen[r] = er.total_bytes;
      wire_add(wire, &er, len);
    }
    for (int r = 0; r < n && rc == 0; ++r) {
      int prev = (r - 1 + n) % n;
      if (add) {
        zo_recv_batch(frames[prev], flen[prev], ctx, scratch, len);
        int32_t* acc = (int32_t*)(dst[r] + off);
        const int32_t* in = (const int32_t*)scratch;
        for (uint64_t i = 0; i < len / 4; ++i) {
          int64_t s = (int64_t)acc[i] + in[i];
          if (s > 2147483647LL || s < -2147483648LL) {
            rc = ZC_ERR_OVERFLOW;
            break;
          }
          acc[i] = (int32_t)s;
        }
      } else {
        zo_recv_batch(frames[prev], flen[prev], ctx, dst[r] + off, len);
      }
    }
  }
  for (int r = 0; r < n; ++r) free(frames[r]);
  free(frames);
  free(flen);
  free(stage);
  free(scratch);
  return rc;
}

/* collectives.cpp:423-503 */
int zo_ring_allreduce(int n, int32_t* syms, uint64_t count, double* scales, int pin, const zc_transport_hint* hint,
                      const zo_huff* ctx, const zc_arb_config* cfg, uint64_t fused_min, zc_wire_stats* wire) {
  if (n == 1 || count == 0) return 0;
  /* meta ring: n-1 raw 24-byte frames sent by every rank (collectives.cpp:440-445) */
  if (wire) {
    wire->frames_by_codec[ZC_CODEC_RAW] += (uint64_t)n * (n - 1);
    wire->raw_bytes += (uint64_t)n * (n - 1) * 24;
    wire->payload_bytes += (uint64_t)n * (n - 1) * 24;
    wire->total_bytes += (uint64_t)n * (n - 1) * (24 + ZC_HEADER_BYTES);
  }
  double shared = scales[0];
  for (int r = 1; r < n; ++r)
    if (scales[r] > shared) shared = scales[r];
  for (int r = 0; r < n; ++r) {
    if (shared != scales[r] && scales[r] > 0.0) {
      double f = scales[r] / shared;
      for (uint64_t i = 0; i < count; ++i) syms[r * count + i] = (int32_t)llround(syms[r * count + i] * f);
      scales[r] = shared;
    }
  }
  int fpin = count * 4 >= fused_min ? pin : ZC_PIN_RAW;
  int rc = 0;
#define CLO(c) ((uint64_t)(c) * count / (uint64_t)n)
  /* reduce-scatter (collectives.cpp:472-492): every rank's step t moves chunk (r - t) to its
   * successor, which folds it into its own copy of that chunk.  All sends of a step read chunks
   * that no receive of the same step writes, so encoding every rank first is equivalent to the
   * lockstep batch interleaving of BatchIo::exchange. */
  for (int t = 0; t < n - 1 && rc == 0; ++t) {
    /* Encode all sends first (they read chunks no receive of this step writes), then receive. */
    {
      uint8_t** sendbuf = (uint8_t**)calloc((size_t)n, sizeof(uint8_t*));
      for (int r = 0; r < n; ++r) {
        int sC = ((r - t) % n + n) % n;
        uint64_t len = (CLO(sC + 1) - CLO(sC)) * 4;
        sendbuf[r] = (uint8_t*)malloc(len ? len : 1);
        memcpy(sendbuf[r], syms + (uint64_t)r * count + CLO(sC), len);
      }
      for (int r = 0; r < n && rc == 0; ++r) {
        int prev = (r - 1 + n) % n;
        int c = ((prev - t) % n + n) % n;
        uint64_t len = (CLO(c + 1) - CLO(c)) * 4;
        /* run a 1-pair exchange: prev's span -> r */
        uint8_t* sp[1] = {sendbuf[prev]};
        uint8_t* dp[1] = {(uint8_t*)(syms + (uint64_t)r * count + CLO(c))};
        rc = ring_exchange(1, sp, dp, len, fpin, 1, hint, ctx, cfg, wire);
      }
      for (int r = 0; r < n; ++r) free(sendbuf[r]);
      free(sendbuf);
    }
  }
  /* allgather of the reduced chunks (collectives.cpp:494-502), cfg pin */
  for (int t = 0; t < n - 1 && rc == 0; ++t) {
    uint8_t** sendbuf = (uint8_t**)calloc((size_t)n, sizeof(uint8_t*));
    for (int r = 0; r < n; ++r) {
      int sC = ((r + 1 - t) % n + n) % n;
      uint64_t len = (CLO(sC + 1) - CLO(sC)) * 4;
      sendbuf[r] = (uint8_t*)malloc(len ? len : 1);
      memcpy(sendbuf[r], syms + (uint64_t)r * count + CLO(sC), len);
    }
    for (int r = 0; r < n && rc == 0; ++r) {
      int prev = (r - 1 + n) % n;
      int c = ((prev + 1 - t) % n + n) % n;
      uint64_t len = (CLO(c + 1) - CLO(c)) * 4;
      uint8_t* sp[1] = {sendbuf[prev]};
      uint8_t* dp[1] = {(uint8_t*)(syms + (uint64_t)r * count + CLO(c))};
      rc = ring_exchange(1, sp, dp, len, pin, 0, hint, ctx, cfg, wire);
    }
    for (int r = 0; r < n; ++r) free(sendbuf[r]);
    free(sendbuf);
  }
#undef CLO
  return rc;
}

/* collectives.cpp:525-544 */
int zo_ring_allgather(int n, const int32_t* blocks, uint64_t block, int pin, const zc_transport_hint* hint,
                      const zo_huff* ctx, const zc_arb_config* cfg, int32_t* out, zc_wire_stats* wire) {
  /* out: n ranks x (n*block) */
  for (int r = 0; r < n; ++r) memcpy(out + ((uint64_t)r * n + r) * block, blocks + (uint64_t)r * block, block * 4);
  if (n == 1 || block == 0) return 0;
  int rc = 0;
  for (int t = 0; t < n - 1 && rc == 0; ++t) {
    for (int r = 0; r < n && rc == 0; ++r) {
      int prev = (r - 1 + n) % n;
      int idx = ((prev - t) % n + n) % n;
      uint8_t* sp[1] = {(uint8_t*)(out + ((uint64_t)prev * n + idx) * block)};
      uint8_t* dp[1] = {(uint8_t*)(out + ((uint64_t)r * n + idx) * block)};
      rc = ring_exchange(1, sp, dp, block * 4, pin, 0, hint, ctx, cfg, wire);
    }
  }
  return rc;
}

/* ------------------------------------------------------------- generators */
/* std::mt19937_64 (the standard's parameters) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}
static uint64_t mt_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* bench.cpp:20-39 */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t chunk_seed(uint64_t seed, int rank, uint64_t chunk) {
  uint64_t rs = mix64(seed ^ mix64(0x724Bull + (uint64_t)rank));
  return mix64(rs ^ mix64(0xC4B2ull + chunk));
}
static double f32r(double v) { return (double)(float)v; }

/* bench.cpp:41-80 */
static int gen_chunk(int dist, double p, uint64_t seed, uint64_t skip, uint64_t n, double* out) {
  mt64 g;
  mt_seed(&g, seed);
#define U01() ((double)(mt_next(&g) >> 11) * 0x1.0p-53)
#define U01P() ((double)((mt_next(&g) >> 11) + 1) * 0x1.0p-53)
  if (dist == 0) {
    for (uint64_t i = 0; i < skip; ++i) mt_next(&g);
    for (uint64_t i = 0; i < n; ++i) out[i] = f32r(2.0 * U01() - 1.0);
  } else if (dist == 1) {
    for (uint64_t i = 0; i < (skip / 2) * 2; ++i) mt_next(&g);
    uint64_t i = 0;
    int drop = (skip & 1) != 0;
    while (i < n) {
      double u1 = U01P();
      double u2 = U01();
      double r = sqrt(-2.0 * log(u1));
      double z0 = r * cos(6.283185307179586 * u2);
      double z1 = r * sin(6.283185307179586 * u2);
      if (!drop) {
        out[i++] = f32r(z0);
        if (i == n) break;
      }
      drop = 0;
      out[i++] = f32r(z1);
    }
  } else if (dist == 2) {
    if (!(p > 0.0) || !(p < 1.0)) return ZC_ERR_INVALID_ARGUMENT;
    for (uint64_t i = 0; i < skip; ++i) mt_next(&g);
    double lp = log(p);
    for (uint64_t i = 0; i < n; ++i) out[i] = f32r(floor(log(U01P()) / lp));
  } else {
    return ZC_ERR_LOGIC;
  }
#undef U01
#undef U01P
  return 0;
}

/* bench.cpp:463-476 */
int zo_gen_data(int dist, double p, uint64_t seed, int rank, uint64_t offset, uint64_t count, double* out) {
  const uint64_t CH = 1ull << 20;
  uint64_t produced = 0;
  while (produced < count) {
    uint64_t idx = offset + produced, chunk = idx / CH, skip = idx % CH;
    uint64_t n = count - produced < CH - skip ? count - produced : CH - skip;
    int rc = gen_chunk(dist, p, chunk_seed(seed, rank, chunk), skip, n, out + produced);
    if (rc) return rc;
    produced += n;
  }
  return 0;
}
