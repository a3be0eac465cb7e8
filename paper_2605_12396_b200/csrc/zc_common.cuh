// zc_common.cuh — shared host/device definitions of the B200 compressed-collective path.
//
// Reference paths are relative to /root/reference/proj/core/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "zcomm_b200.h"

#define ZC_HD __host__ __device__ __forceinline__

namespace zc {

constexpr uint32_t kHeaderBytes = ZC_HEADER_BYTES;
constexpr uint64_t kBatchRawBytes = ZC_BATCH_RAW_BYTES;
constexpr uint64_t kStageBankBytes = ZC_STAGE_BANK_BYTES;
constexpr uint64_t kSampleWindow = ZC_SAMPLE_WINDOW_BYTES;
constexpr uint32_t kIndexGrain = ZC_HUFF_INDEX_GRAIN;

// Device-resident canonical Huffman tables (HuffmanContext, huffman.hpp:20-33).  `enc[s]` packs
// the LSB-first (bit-reversed) code in the low 32 bits and its length in bits 32..39, so the
// encoder fetches both with one 8-byte shared-memory load.
struct DevHuff {
  uint32_t valid;
  uint32_t min_len;
  uint32_t max_len;
  uint32_t _pad;
  uint64_t enc[256];
  uint8_t len[256];
  uint8_t sym_order[256];
  uint32_t count_at_len[33];
  uint32_t first_index[33];
  uint64_t first_code[33];
  uint16_t lut[1u << ZC_HUFF_ROOT_BITS];  // sym | len << 8, len 0 = over-root escape
};

// ------------------------------------------------------------------ frame (frame.cpp:35-69)
ZC_HD void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
ZC_HD uint64_t get_le(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}

// The 32-byte header as four little-endian 64-bit words: word 0 = magic | version<<32 |
// codec<<40 | flags<<48, then rawBytes, payloadBytes, params (frame.hpp:9-10).
ZC_HD void header_words(const zc_frame_header& h, uint64_t w[4]) {
  w[0] = static_cast<uint64_t>(h.magic) | (static_cast<uint64_t>(h.version) << 32) |
         (static_cast<uint64_t>(h.codec) << 40) | (static_cast<uint64_t>(h.flags) << 48);
  w[1] = h.raw_bytes;
  w[2] = h.payload_bytes;
  w[3] = h.params;
}
ZC_HD zc_frame_header header_from_words(const uint64_t w[4]) {
  zc_frame_header h;
  h.magic = static_cast<uint32_t>(w[0]);
  h.version = static_cast<uint8_t>(w[0] >> 32);
  h.codec = static_cast<uint8_t>(w[0] >> 40);
  h.flags = static_cast<uint16_t>(w[0] >> 48);
  h.raw_bytes = w[1];
  h.payload_bytes = w[2];
  h.params = w[3];
  return h;
}
ZC_HD zc_frame_header make_header(uint32_t codec, uint16_t flags, uint64_t raw, uint64_t payload,
                                  uint64_t params) {
  zc_frame_header h;
  h.magic = ZC_FRAME_MAGIC;
  h.version = ZC_FRAME_VERSION;
  h.codec = static_cast<uint8_t>(codec);
  h.flags = flags;
  h.raw_bytes = raw;
  h.payload_bytes = payload;
  h.params = params;
  return h;
}
// validate_header (frame.cpp:61-69)
ZC_HD bool validate_header(const zc_frame_header& h, uint64_t region) {
  if (h.magic != ZC_FRAME_MAGIC) return false;
  if (h.version != ZC_FRAME_VERSION) return false;
  if (h.codec > ZC_CODEC_HUFFMAN) return false;
  if (h.raw_bytes == 0) return false;
  if (region < kHeaderBytes || h.payload_bytes > region - kHeaderBytes) return false;
  if (h.codec == ZC_CODEC_RAW && h.payload_bytes != h.raw_bytes) return false;
  return true;
}

// ------------------------------------------------------------------ zig-zag (fixedlen.hpp:14-19)
ZC_HD uint32_t zigzag32(int32_t v) {
  return (static_cast<uint32_t>(v) << 1) ^ static_cast<uint32_t>(v >> 31);
}
ZC_HD int32_t unzigzag32(uint32_t z) {
  return static_cast<int32_t>(z >> 1) ^ -static_cast<int32_t>(z & 1);
}
ZC_HD uint32_t bit_width32(uint32_t v) {
#ifdef __CUDA_ARCH__
  return 32u - static_cast<uint32_t>(__clz(v));
#else
  return v ? 32u - static_cast<uint32_t>(__builtin_clz(v)) : 0u;
#endif
}
// fixedlen_width (fixedlen.cpp:8-13) from the block's max zig-zag value.
ZC_HD uint32_t width_from_maxzz(uint32_t maxzz) { return maxzz == 0 ? 1u : bit_width32(maxzz); }
ZC_HD uint64_t packed_bytes(uint64_t count, uint32_t w) { return (count * w + 7) / 8; }

// ------------------------------------------------------------------ fp64 helpers
// Bit-exact IEEE double arithmetic on both sides: the device uses explicit _rn intrinsics so
// that nvcc can never contract a*b+c into an FMA (the reference's SSE2 build never does).
ZC_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
ZC_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
ZC_HD double ddiv(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
ZC_HD double u64_to_double(uint64_t v) {
#ifdef __CUDA_ARCH__
  return __ull2double_rn(v);
#else
  return static_cast<double>(v);
#endif
}

// ------------------------------------------------------------------ quantizer (quant.cpp:22-27)
// sym = llround(x / scale) with half-away-from-zero rounding, bit-exact with the reference fed
// (double)x.  Fast path: q' = x * rcp (rcp = RN(1/scale)) differs from RN(x/scale) by < 2^-51 |q|,
// so whenever q' is farther than that from a half-integer both round to the same integer and
// the round-half-even magic-constant conversion equals llround.  Near a tie, or near the int32
// limit, the exact IEEE division decides.  err |= ZC_DERR_* on non-finite input / range.
//
// The fast-path test is integer work on high words: |q| < 2^30 (so |q'-q| < 2^-21, and no int32
// range issue) and |r| < 0.5 - 2^-19 (r = q' - RNE(q'), exact); 2^-19 > 2^-21 keeps the decision
// safe, and only ~4e-6 of inputs take the division.
__device__ __forceinline__ int32_t quantize_one(double x, double scale, double rcp, uint32_t& err) {
  if ((__double2hiint(x) & 0x7ff00000) == 0x7ff00000) {  // Inf / NaN
    err |= ZC_DERR_NONFINITE;
    return 0;
  }
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double q = __dmul_rn(x, rcp);
  const double t = __dadd_rn(q, kMagic);
  const double kd = __dsub_rn(t, kMagic);
  const double r = __dsub_rn(q, kd);  // exact, |r| <= 0.5
  const uint32_t qhi = static_cast<uint32_t>(__double2hiint(q)) & 0x7fffffffu;
  const uint32_t rhi = static_cast<uint32_t>(__double2hiint(r)) & 0x7fffffffu;
  if (qhi < 0x41D00000u && rhi < 0x3FDFFFF0u) {  // |q| < 2^30, |r| < 0.5 - 2^-19
    return static_cast<int32_t>(__double2loint(t));
  }
  double qe = __ddiv_rn(x, scale);
  if (!(fabs(qe) < 2147483647.5)) {
    err |= ZC_DERR_RANGE;
    return 0;
  }
  return static_cast<int32_t>(llround(qe));
}

// fp32 -> fp64 and fp64 -> fp32 (round to nearest even) with integer ops: the F2F conversion
// instructions issue at a fraction of the ALU rate on sm_100 and dominated the codec loops.
// Normal numbers and zeros take the integer path; the rest sets `slow` / falls back.
__device__ __forceinline__ double f2d_bits(uint32_t u, bool& slow) {
  const uint32_t ex = (u >> 23) & 0xffu;
  uint32_t hi, lo;
  if (ex - 1u < 254u) {
    hi = (u & 0x80000000u) | ((ex + 896u) << 20) | ((u >> 3) & 0xfffffu);
    lo = u << 29;
  } else {
    hi = u & 0x80000000u;
    lo = 0;
    slow |= (u & 0x7fffffffu) != 0;  // denormal, Inf, NaN
  }
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

__device__ __forceinline__ float d2f_rn(double d) {
  const uint32_t hi = static_cast<uint32_t>(__double2hiint(d)), lo = static_cast<uint32_t>(__double2loint(d));
  const uint32_t ex = (hi >> 20) & 0x7ffu;
  if (ex - 897u < 254u) {
    uint32_t f = (hi & 0x80000000u) | ((ex - 896u) << 23) | ((hi & 0xfffffu) << 3) | (lo >> 29);
    const uint32_t rb = lo & 0x1fffffffu;
    f += (rb > 0x10000000u || (rb == 0x10000000u && (f & 1u))) ? 1u : 0u;
    return __uint_as_float(f);
  }
  if ((hi & 0x7fffffffu) == 0 && lo == 0) return __uint_as_float(hi & 0x80000000u);
  return __double2float_rn(d);
}

// Branch-free fast path of quantize_one for finite inputs: returns the symbol and sets `slow` when
// this input must instead go through quantize_one (near a tie or |q| >= 2^30).
__device__ __forceinline__ int32_t quantize_fast(double x, double rcp, bool& slow) {
  const double kMagic = 6755399441055744.0;
  const double q = __dmul_rn(x, rcp);
  const double t = __dadd_rn(q, kMagic);
  const double r = __dsub_rn(q, __dsub_rn(t, kMagic));
  const uint32_t qhi = static_cast<uint32_t>(__double2hiint(q)) & 0x7fffffffu;
  const uint32_t rhi = static_cast<uint32_t>(__double2hiint(r)) & 0x7fffffffu;
  slow |= !(qhi < 0x41D00000u && rhi < 0x3FDFFFF0u);
  return static_cast<int32_t>(__double2loint(t));
}

// quantize_one for an fp32 input given as bits: integer widening + branch-free fast path, exact
// fallback only near a tie or for non-normal inputs.
__device__ __forceinline__ int32_t quantize_f32bits(uint32_t u, double scale, double rcp, uint32_t& err) {
  bool slow = false;
  const int32_t r = quantize_fast(f2d_bits(u, slow), rcp, slow);
  if (!slow) return r;
  return quantize_one(static_cast<double>(__uint_as_float(u)), scale, rcp, err);
}

// int32 -> double exactly, without the I2F conversion pipe (magic-number subtraction).
__device__ __forceinline__ double i2d_magic(uint32_t s) {
  return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(s ^ 0x80000000u)), 4503601774854144.0);
}

// ------------------------------------------------------------------ selector (rea.cpp:22-176)
ZC_HD bool gain_ok(uint64_t raw, uint64_t payload, uint32_t permil) {
  if (payload >= raw) return false;
  return (raw - payload) * 1000ull >= static_cast<uint64_t>(permil) * raw;
}

ZC_HD const zc_codec_cost& cost_for(const zc_arb_config& cfg, uint32_t c) {
  return c == ZC_CODEC_FIXEDLEN ? cfg.cost.fixedlen : c == ZC_CODEC_HUFFMAN ? cfg.cost.huffman : cfg.cost.raw;
}

// make_estimate (rea.cpp:31-44): ((alpha + lamEnc*E) + P/beta) + lamDec*D, each op rounded.
ZC_HD zc_codec_estimate make_estimate(uint32_t codec, uint64_t raw, uint64_t payload, const zc_transport_hint& hint,
                                      const zc_arb_config& cfg) {
  const zc_codec_cost& c = cost_for(cfg, codec);
  zc_codec_estimate e;
  e.codec = codec;
  e.admissible = 0;
  e.predicted_payload = payload;
  e.enc_sec = c.enc_bytes_per_sec > 0.0 ? ddiv(u64_to_double(raw), c.enc_bytes_per_sec) : 0.0;
  e.dec_sec = c.dec_bytes_per_sec > 0.0 ? ddiv(u64_to_double(raw), c.dec_bytes_per_sec) : 0.0;
  double beta = hint.beta_eff_bytes_per_sec > 0.0 ? hint.beta_eff_bytes_per_sec : __builtin_huge_val();
  double t = dadd(c.alpha_sec, dmul(cfg.lam_enc, e.enc_sec));
  t = dadd(t, ddiv(u64_to_double(payload), beta));
  t = dadd(t, dmul(cfg.lam_dec, e.dec_sec));
  e.predicted_sec = t;
  return e;
}

// predict_payload (rea.cpp:120-143)
ZC_HD uint64_t predict_payload(uint32_t codec, uint64_t raw, const zc_sample_stats& st, const zc_arb_config& cfg) {
  if (codec == ZC_CODEC_RAW) return raw;
  if (codec == ZC_CODEC_FIXEDLEN) {
    if (raw < 4 || raw % 4 != 0) return 0;
    uint32_t w = 1;
    while ((1ull << w) <= st.max_zigzag && w < 32) ++w;
    return packed_bytes(raw / 4, w);
  }
  if (codec == ZC_CODEC_HUFFMAN) {
    bool valid = cfg.embed_codebook ? st.self_code_len_valid != 0 : st.ctx_code_len_valid != 0;
    if (!valid) return 0;
    double el = cfg.embed_codebook ? st.self_code_len_bits : st.ctx_code_len_bits;
    double bits = dmul(u64_to_double(raw), el);
    uint64_t p = static_cast<uint64_t>(ddiv(dadd(bits, 7.0), 8.0));
    if (cfg.embed_codebook) p += ZC_HUFF_CODEBOOK_BYTES;
    return p;
  }
  return raw;
}

// arbitrate_plan (rea.cpp:145-176).  ctx_usable = (ctx != nullptr && ctx->valid).
ZC_HD zc_arbitration_plan arbitrate_plan(uint64_t raw, uint64_t cap, const zc_sample_stats& st,
                                         const zc_transport_hint& hint, bool ctx_usable, const zc_arb_config& cfg) {
  zc_arbitration_plan p;
  p._pad = 0;
  p.raw = make_estimate(ZC_CODEC_RAW, raw, raw, hint, cfg);
  p.raw.admissible = raw > 0 && raw <= cap;
  uint64_t pf = predict_payload(ZC_CODEC_FIXEDLEN, raw, st, cfg);
  p.fixedlen = make_estimate(ZC_CODEC_FIXEDLEN, raw, pf, hint, cfg);
  p.fixedlen.admissible = pf > 0 && pf <= cap && gain_ok(raw, pf, cfg.min_gain_permil);
  uint64_t ph = predict_payload(ZC_CODEC_HUFFMAN, raw, st, cfg);
  p.huffman = make_estimate(ZC_CODEC_HUFFMAN, raw, ph, hint, cfg);
  bool usable = cfg.embed_codebook || ctx_usable;
  p.huffman.admissible =
      ph > 0 && usable && raw >= cfg.huffman_min_raw_bytes && ph <= cap && gain_ok(raw, ph, cfg.min_gain_permil);
  p.choice = ZC_CODEC_RAW;
  double best = p.raw.predicted_sec;
  if (p.fixedlen.admissible && p.fixedlen.predicted_sec < best) {
    p.choice = ZC_CODEC_FIXEDLEN;
    best = p.fixedlen.predicted_sec;
  }
  if (p.huffman.admissible && p.huffman.predicted_sec < best) p.choice = ZC_CODEC_HUFFMAN;
  return p;
}

}  // namespace zc
