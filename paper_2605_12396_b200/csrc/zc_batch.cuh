// zc_batch.cuh — per-unit state of the batched send-path encoder shared by its kernels
// (zc_batch.cu: profile / scan / emit; zc_fixed.cu: the TMA-pipelined fp32 range and
// FixedLen/RAW emit kernels).  Reference paths are relative to /root/reference/proj/core/.
#pragma once
#include "zc_encode_common.cuh"

namespace zc {
namespace {

constexpr uint32_t BS = 65536;                      // slice: raw symbol bytes
constexpr uint32_t BV = BS / 16;                    // vectors per slice
constexpr uint32_t BMAX = ZC_BATCH_RAW_BYTES / BS;  // slices per full 4 MiB unit

struct BPart {  // per slice (pass 2)
  float fmn, fmx;
  double dmn, dmx;
  uint32_t maxzz, bad, zero, _p;
  unsigned long long bits;
};

struct BUnit {  // per unit, zeroed before every launch
  uint32_t plan;  // selector choice (Auto)
  uint32_t codec, width, scan_done;
  unsigned long long payload;
  uint32_t edone, pdone;
  uint32_t whist[256];  // window histogram (pass 1, merged from PC CTAs)
  uint32_t wmz;         // window max zig-zag
  uint32_t maxzz, bad, hdone;  // hdone: Huffman bit-count slices (scan_kernel, fast mode)
  uint32_t fmin_c, fmax_k;           // fp32 range as order-preserving keys (min complemented)
  unsigned long long dmin_c, dmax_k;  // fp64 range, same encoding
  // speculative FixedLen emit (zc_fixed.cu): guess = window width, redo = decision missed the
  // guess, tdone = tiles done; hdec = Huffman-target decision published (fused Huffman kernel)
  uint32_t guess, redo, tdone, hdec;
  BPart part[BMAX];
  unsigned long long hbase[BMAX];
  unsigned long long head_idx[BMAX], tail_idx[BMAX];
  uint32_t head_val[BMAX], tail_val[BMAX], has_head[BMAX], has_tail[BMAX];
};

struct BGlobal {  // after the BUnit array in the scratch block (zeroed with it)
  uint32_t n_huff;  // units the selector planned as Huffman (Auto)
  uint32_t next_task;  // range kernel work counter (zc_fixed.cu)
  uint32_t n_redo;     // speculative FixedLen units sent to the redo emit (zc_fixed.cu)
  uint32_t huff_task;  // fused Huffman kernel work counter (zc_batch.cu)
  uint32_t pad[60];
};
__device__ __forceinline__ BGlobal* bglobal(BUnit* us, uint32_t nunits) { return reinterpret_cast<BGlobal*>(us + nunits); }

struct BGeom {
  uint32_t s_full;  // slices per full unit
  uint64_t total;   // slices in the message
  uint32_t fast;    // zc_fixed.cu handles the FixedLen / RAW units (range + emit)
  uint32_t spec;    // speculative FixedLen: range pass = window profiles only, emit packs with the window's width
  uint32_t planned;  // Auto: profile_kernel already profiled every window and stored the plans
  __device__ __forceinline__ void unit_of(uint64_t t, uint32_t nunits, uint32_t& u, uint32_t& s) const {
    const uint64_t head = static_cast<uint64_t>(nunits - 1) * s_full;
    if (t < head) {
      u = static_cast<uint32_t>(t / s_full);
      s = static_cast<uint32_t>(t - static_cast<uint64_t>(u) * s_full);
    } else {
      u = nunits - 1;
      s = static_cast<uint32_t>(t - head);
    }
  }
};

__device__ __forceinline__ uint64_t unit_R(const EncParams& p, uint32_t u) {
  const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
  return (p.total_bytes - uoff) < p.unit_bytes ? (p.total_bytes - uoff) : p.unit_bytes;
}
__device__ __forceinline__ uint32_t unit_slices(const EncParams& p, uint32_t u) {
  return static_cast<uint32_t>((unit_R(p, u) + BS - 1) / BS);
}

// The codec pass 2/3 work towards for a unit: Auto -> the plan; pins -> the pin (RAW when the
// pinned codec cannot apply).
__device__ __forceinline__ uint32_t target_codec(const EncParams& p, const BUnit& U, bool ctx_ok) {
  if (p.pin == ZC_PIN_AUTO) return U.plan;
  if (p.pin == ZC_PIN_FIXEDLEN) return ZC_CODEC_FIXEDLEN;
  if (p.pin == ZC_PIN_HUFFMAN) return ctx_ok ? ZC_CODEC_HUFFMAN : ZC_CODEC_RAW;
  return ZC_CODEC_RAW;
}

// Order-preserving u32/u64 keys of fp32/fp64 values, so the unit range merges with atomicMax
// (the minimum is kept as the complement of its key: zero-initialised state works for both).
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); }
__device__ __forceinline__ unsigned long long dkey(double d) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d));
  return (u >> 63) ? ~u : (u | (1ull << 63));
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  return __longlong_as_double(static_cast<long long>((k >> 63) ? (k & ~(1ull << 63)) : ~k));
}

// The unit's final decision once every slice has reported (tid 0 of the CTA that completed it):
// encode_best post-checks (rea.cpp:189-236) or the pinned send_batch fallbacks (collectives.cpp:223-275).
template <int SRC>
__device__ void decide_unit(const EncParams& p, BUnit& U, uint32_t u, bool want_range, bool fast_ok, uint32_t& err) {
  constexpr bool kFloat = SRC != SRC_BYTES;
  const uint64_t R = unit_R(p, u);
  const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
  const uint32_t ns = unit_slices(p, u);
  uint32_t codec = ZC_CODEC_RAW, width = 0;
  unsigned long long pay_b = R;
  const bool gate = p.pin == ZC_PIN_AUTO;  // Auto applies gain_ok; pins do not
  if (want_range) {
    uint32_t maxzz = __ldcg(&U.maxzz);
    if (kFloat && fast_ok) {
      if (__ldcg(&U.bad)) {
        err |= ZC_DERR_NONFINITE;
      } else if (R >= 4) {
        double mn, mx;
        if (SRC == SRC_F32) {
          mn = static_cast<double>(fkey_inv(~__ldcg(&U.fmin_c)));
          mx = static_cast<double>(fkey_inv(__ldcg(&U.fmax_k)));
        } else {
          mn = dkey_inv(~__ldcg(&U.dmin_c));
          mx = dkey_inv(__ldcg(&U.dmax_k));
        }
        maxzz = max(zigzag32(quantize_one(mx, enc_scale(p), enc_rcp(p), err)), zigzag32(quantize_one(mn, enc_scale(p), enc_rcp(p), err)));
      }
    }
    if (R >= 4 && R % 4 == 0) {
      width = width_from_maxzz(maxzz);
      const unsigned long long pay = packed_bytes(R / 4, width);
      if (pay > 0 && pay <= pcap && (!gate || gain_ok(R, pay, p.cfg.min_gain_permil))) {
        codec = ZC_CODEC_FIXEDLEN;
        pay_b = pay;
      }
    }
  } else {
    uint32_t zl = 0;
    unsigned long long bits = 0;
    for (uint32_t r = 0; r < ns; ++r) {
      zl |= __ldcg(&U.part[r].zero);
      U.hbase[r] = bits;
      bits += __ldcg(&U.part[r].bits);
    }
    const unsigned long long pay = (bits + 7) / 8;
    if (!zl && pay > 0 && pay <= pcap && (!gate || gain_ok(R, pay, p.cfg.min_gain_permil))) {
      codec = ZC_CODEC_HUFFMAN;
      pay_b = pay;
    }
  }
  U.codec = codec;
  U.width = width;
  U.payload = pay_b;
}

// The frame a unit ends up with once pass 2 has decided (the emit kernels' common view):
// pins RAW / plan RAW -> RAW if it fits; otherwise the decision of decide_unit.
__device__ __forceinline__ void final_codec(const EncParams& p, const BUnit& U, uint32_t u, bool ctx_ok, uint32_t& codec,
                                            uint32_t& width, uint64_t& P) {
  const uint64_t R = unit_R(p, u);
  const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
  const uint32_t target = target_codec(p, U, ctx_ok);
  width = 0;
  if (p.stage_len <= kHeaderBytes) {
    codec = CODEC_NONE;
    P = 0;
  } else if (target == ZC_CODEC_RAW) {
    codec = R <= pcap ? ZC_CODEC_RAW : CODEC_NONE;
    P = R;
  } else {
    codec = U.codec;
    width = U.width;
    P = U.payload;
    if (codec == ZC_CODEC_RAW && R > pcap) codec = CODEC_NONE;
  }
}

// Writes the 32-byte header (frame.cpp:35-45) and the unit's EncodeResult (one thread).
__device__ __forceinline__ void write_frame_header(const EncParams& p, uint32_t u, uint32_t codec, uint32_t width, uint64_t P) {
  const uint64_t R = unit_R(p, u);
  uint8_t* stage = p.stages + static_cast<uint64_t>(u) * p.stride;
  zc_encode_result res;
  res._pad = 0;
  if (codec == CODEC_NONE) {
    res.codec = ZC_CODEC_RAW;
    res.payload_bytes = 0;
    res.total_bytes = 0;
  } else {
    const zc_frame_header h = make_header(codec, 0, R, P, codec == ZC_CODEC_FIXEDLEN ? width : 0);
    uint64_t hw[4];
    header_words(h, hw);
    uint64_t* hp = reinterpret_cast<uint64_t*>(stage);
    hp[0] = hw[0];
    hp[1] = hw[1];
    hp[2] = hw[2];
    hp[3] = hw[3];
    res.codec = codec;
    res.payload_bytes = P;
    res.total_bytes = kHeaderBytes + P;
  }
  if (p.results) p.results[u] = res;
}

}  // namespace

// zc_fixed.cu: the speculative single-read FixedLen path (see its header comment).
// mode: 0 two-read (range over every slice, then emit), 1 speculative (range = window profiles
// only; emit packs FixedLen units with the window's width and decides), 2 the redo emit of the
// units whose decision differed from the speculation.
cudaError_t launch_fixed_range_m(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                                 int mode, cudaStream_t s);
cudaError_t launch_fixed_emit_m(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                                int mode, cudaStream_t s);
}  // namespace zc
