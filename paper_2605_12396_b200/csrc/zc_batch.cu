// zc_batch.cu — the batched send-path encoder (send_encoded over a whole message,
// collectives.cpp:201-302 for every 4 MiB batch) as three stream-ordered streaming kernels with no
// inter-CTA waiting:
//
//   1. profile   one CTA per unit: the 64 KiB window (rea.cpp:93-118) — histogram, window max
//                zig-zag, expected length under the shared code — and, in Auto mode, the
//                selector's plan (arbitrate_plan, rea.cpp:145-176; bit-exact, zc_common.cuh).
//   2. scan      64 KiB slices, grid-stride: only what the planned codec needs — the value range
//                (FixedLen: max zig-zag = max(zz(q(min x)), zz(q(max x))) since quantization is
//                monotone) or the exact Huffman bit count under the shared code; RAW units are not
//                read at all.  The unit's last slice (atomic counter) finalises the decision:
//                post-checks of encode_best (rea.cpp:189-236) or the pinned send_batch fallbacks
//                (collectives.cpp:223-275), payload size and per-slice Huffman bit offsets.
//   3. emit      64 KiB slices, grid-stride in REVERSE unit order (the tail of pass 2's stream is
//                still in the 126 MB L2): quantize again and materialise RAW / FixedLen (lane-
//                centric packer through a swizzled shared-memory transpose) / Huffman (tile
//                encoder at the slice's exact bit offset; seam words merged by the unit's last
//                slice) plus the 32-byte header (frame.cpp:35-45).
//
// Input is read twice (pass 2 only for FixedLen/Huffman units) instead of once with a cross-CTA
// decision wait: every kernel is a plain HBM stream, robust to co-scheduling and stragglers.
#include <algorithm>
#include <cstdlib>

#include "zc_encode_common.cuh"
#include "zc_huff_device.cuh"

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
  uint32_t maxzz, bad, _q;
  uint32_t fmin_c, fmax_k;           // fp32 range as order-preserving keys (min complemented)
  unsigned long long dmin_c, dmax_k;  // fp64 range, same encoding
  BPart part[BMAX];
  unsigned long long hbase[BMAX];
  unsigned long long head_idx[BMAX], tail_idx[BMAX];
  uint32_t head_val[BMAX], tail_val[BMAX], has_head[BMAX], has_tail[BMAX];
};

struct BGeom {
  uint32_t s_full;  // slices per full unit
  uint64_t total;   // slices in the message
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

// ------------------------------------------------------------------ pass 1: window profile + plan
constexpr uint32_t PC = 16;            // CTAs per unit window (64 KiB / 16 = 4 KiB each)
constexpr uint32_t PT = 256;           // threads per profile CTA: one 16-byte vector each
constexpr uint32_t PV = ZC_SAMPLE_WINDOW_BYTES / 16 / PC;

template <int SRC>
__global__ void __launch_bounds__(PT) profile_kernel(const EncParams p, BUnit* us) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t u = blockIdx.x / PC, part = blockIdx.x % PC;
  __shared__ uint32_t s_hist[256];
  __shared__ uint8_t s_clens[256];
  __shared__ uint32_t s_wmz[PT / 32];
  __shared__ uint32_t s_whist[PT / 32][256];
  __shared__ uint32_t s_last;
  BUnit& U = us[u];
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  const uint64_t R = unit_R(p, u);
  const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
  const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
  if (R <= p.cfg.small_batch_threshold_bytes || p.stage_len <= kHeaderBytes) {
    if (part == 0 && tid == 0) U.plan = ZC_CODEC_RAW;
    return;
  }
  for (int i = tid; i < 256; i += PT) {
    s_hist[i] = 0;
    s_clens[i] = ctx_ok ? p.ctx->len[i] : 0;
  }
  for (int i = tid; i < 256 * (PT / 32); i += PT) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t W = R < kSampleWindow ? R : kSampleWindow;
  const uint64_t v = static_cast<uint64_t>(part) * PV + tid;
  uint32_t wmz = 0, err = 0;
  if (v * 16 < W) {
    RawVec rv;
    fetch<SRC, false>(p, uoff, R, v, rv);
    uint32_t w[4];
    to_words<SRC>(p, rv, w, err);
    const uint32_t nb = static_cast<uint32_t>(W - v * 16 < 16 ? W - v * 16 : 16);
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q)
      if (q < (nb >> 2)) wmz = max(wmz, zigzag32(static_cast<int32_t>(w[q])));
    // per-warp sub-histograms; byte positions rotated across lanes so the (typically few)
    // dominant high-byte values do not hit one bank in the same instruction
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j) {
      const uint32_t jj = (j + static_cast<uint32_t>(lane)) & 15u;
      if (jj < nb) atomicAdd(&s_whist[warp][byte_of(w, jj)], 1u);
    }
  }
  for (int o = 16; o > 0; o >>= 1) wmz = max(wmz, __shfl_xor_sync(FULL, wmz, o));
  if (lane == 0) s_wmz[warp] = wmz;
  __syncthreads();
  for (int i = tid; i < 256; i += PT) {
    uint32_t c = 0;
#pragma unroll
    for (int w2 = 0; w2 < PT / 32; ++w2) c += s_whist[w2][i];
    if (c) atomicAdd(&U.whist[i], c);
  }
  if (tid == 0) {
    uint32_t m = 0;
    for (int i = 0; i < PT / 32; ++i) m = max(m, s_wmz[i]);
    atomicMax(&U.wmz, m);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&U.pdone, 1u) == PC - 1 ? 1u : 0u;
  __syncthreads();
  if (s_last) {  // the unit's last profile CTA: expected code length and the selector's plan
    __threadfence();
    for (int i = tid; i < 256; i += PT) s_hist[i] = __ldcg(&U.whist[i]);
    __syncthreads();
    double el = 0.0;
    bool el_ok = false;
    if (warp == 0) el_ok = ctx_ok && warp_mean_len(s_hist, s_clens, el);
    if (p.stats != nullptr) {
      zc_sample_stats* o = p.stats + u;
      for (int i = tid; i < 256; i += PT) o->hist[i] = s_hist[i];
    }
    if (tid == 0) {
      zc_sample_stats st;
      st.sampled_bytes = W;
      st.max_zigzag = __ldcg(&U.wmz);
      st.ctx_code_len_bits = el_ok ? el : 0.0;
      st.ctx_code_len_valid = el_ok ? 1u : 0u;
      st.self_code_len_bits = 0.0;
      st.self_code_len_valid = 0u;  // only read with embedded codebooks (not on this path)
      if (p.stats != nullptr) {
        zc_sample_stats* o = p.stats + u;
        o->sampled_bytes = st.sampled_bytes;
        o->max_zigzag = st.max_zigzag;
        o->ctx_code_len_bits = st.ctx_code_len_bits;
        o->self_code_len_bits = 0.0;
        o->ctx_code_len_valid = st.ctx_code_len_valid;
        o->self_code_len_valid = 0u;
      }
      U.plan = arbitrate_plan(R, pcap, st, p.hint, ctx_ok, p.cfg).choice;
    }
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}

// ------------------------------------------------------------------ pass 2: ranges / bit counts, decision
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
        maxzz = max(zigzag32(quantize_one(mx, p.scale, p.rcp, err)), zigzag32(quantize_one(mn, p.scale, p.rcp, err)));
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

// Each CTA streams a CONTIGUOUS range of slices (mostly inside one unit), keeps the value range in
// registers across the slices of a unit and merges it into the unit once per unit (one block
// reduction + atomics), so the pass is a plain HBM stream; Huffman units reduce per slice (the
// per-slice bit counts become the slices' bit offsets).
template <int SRC>
__global__ void __launch_bounds__(NT, 1) scan_kernel(const EncParams p, BUnit* us, BGeom g) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint8_t s_clens[256];
  __shared__ uint32_t s_r32[4][NW];
  __shared__ unsigned long long s_r64[2][NW];
  __shared__ uint32_t s_last;
  constexpr bool kFloat = SRC != SRC_BYTES;
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  const bool fast_ok = aligned16(p.src) && (p.unit_bytes % 16) == 0;
  for (int i = tid; i < 256; i += NT) s_clens[i] = ctx_ok ? p.ctx->len[i] : 0;
  __syncthreads();
  uint32_t err = 0;
  const uint64_t t0 = g.total * blockIdx.x / gridDim.x, t1 = g.total * (blockIdx.x + 1) / gridDim.x;
  // running range of the current unit (FixedLen units)
  Range rg;
  uint32_t mz = 0, run_u = 0xffffffffu, run_n = 0;
  auto flush = [&]() {  // merge the running range into unit run_u (all threads)
    if (SRC == SRC_F32) rg.bad = rg.absbits >= 0x7f800000u ? 1u : 0u;
    uint32_t kmn = 0, kmx = 0;
    unsigned long long dmn = 0, dmx = 0;
    if (SRC == SRC_F32) {
      kmn = ~fkey(rg.fmn);
      kmx = fkey(rg.fmx);
    } else if (SRC == SRC_F64) {
      dmn = ~dkey(rg.dmn);
      dmx = dkey(rg.dmx);
    }
    for (int o = 16; o > 0; o >>= 1) {
      mz = max(mz, __shfl_xor_sync(FULL, mz, o));
      rg.bad |= __shfl_xor_sync(FULL, rg.bad, o);
      kmn = max(kmn, __shfl_xor_sync(FULL, kmn, o));
      kmx = max(kmx, __shfl_xor_sync(FULL, kmx, o));
      dmn = max(dmn, __shfl_xor_sync(FULL, dmn, o));
      dmx = max(dmx, __shfl_xor_sync(FULL, dmx, o));
    }
    __syncthreads();
    if (lane == 0) {
      s_r32[0][warp] = mz;
      s_r32[1][warp] = rg.bad;
      s_r32[2][warp] = kmn;
      s_r32[3][warp] = kmx;
      s_r64[0][warp] = dmn;
      s_r64[1][warp] = dmx;
    }
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < NW; ++i) {
        mz = max(mz, s_r32[0][i]);
        rg.bad |= s_r32[1][i];
        kmn = max(kmn, s_r32[2][i]);
        kmx = max(kmx, s_r32[3][i]);
        dmn = max(dmn, s_r64[0][i]);
        dmx = max(dmx, s_r64[1][i]);
      }
      BUnit& U = us[run_u];
      atomicMax(&U.maxzz, mz);
      if (rg.bad) atomicOr(&U.bad, 1u);
      if (SRC == SRC_F32) {
        atomicMax(&U.fmin_c, kmn);
        atomicMax(&U.fmax_k, kmx);
      } else if (SRC == SRC_F64) {
        atomicMax(&U.dmin_c, dmn);
        atomicMax(&U.dmax_k, dmx);
      }
      __threadfence();
      if (atomicAdd(&U.scan_done, run_n) + run_n == unit_slices(p, run_u)) {
        __threadfence();
        decide_unit<SRC>(p, U, run_u, true, fast_ok, err);
      }
    }
    rg = Range();
    mz = 0;
    run_n = 0;
  };
  for (uint64_t t = t0; t < t1; ++t) {
    uint32_t u, s;
    g.unit_of(t, p.nunits, u, s);
    BUnit& U = us[u];
    const uint32_t target = target_codec(p, U, ctx_ok);
    if (target != ZC_CODEC_FIXEDLEN && target != ZC_CODEC_HUFFMAN) continue;  // RAW: decided in pass 3
    const uint64_t R = unit_R(p, u);
    const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
    const uint64_t v0 = static_cast<uint64_t>(s) * BV;
    const uint64_t v1 = min(v0 + BV, (R + 15) / 16);
    const uint64_t vfull = min(v1, R / 16);
    if (target == ZC_CODEC_FIXEDLEN) {
      if (run_n && run_u != u) flush();
      run_u = u;
      ++run_n;
      if (fast_ok) {
        constexpr int UN = 8;
        for (uint64_t base = v0 + static_cast<uint64_t>(warp) * 32; base < vfull; base += NT * UN) {
          RawVec rv[UN];
#pragma unroll
          for (int k = 0; k < UN; ++k) {
            const uint64_t v = base + static_cast<uint64_t>(k) * NT + lane;
            if (v < vfull) fetch_full<SRC, false>(p, uoff, v, rv[k]);
          }
#pragma unroll
          for (int k = 0; k < UN; ++k) {
            const uint64_t v = base + static_cast<uint64_t>(k) * NT + lane;
            if (v < vfull) {
              if (kFloat) {
                minmax_full<SRC>(rv[k], rg);
              } else {
                mz = max(mz, max(max(zigzag32(static_cast<int32_t>(rv[k].a.x)), zigzag32(static_cast<int32_t>(rv[k].a.y))),
                                 max(zigzag32(static_cast<int32_t>(rv[k].a.z)), zigzag32(static_cast<int32_t>(rv[k].a.w)))));
              }
            }
          }
        }
        if (vfull < v1 && tid == 0) {
          RawVec rv;
          fetch<SRC, false>(p, uoff, R, vfull, rv);
          if (kFloat) {
            minmax_vec<SRC>(rv, rg);
          } else {
            uint32_t w[4];
            to_words<SRC>(p, rv, w, err);
            for (uint32_t q = 0; q < (rv.nb >> 2); ++q) mz = max(mz, zigzag32(static_cast<int32_t>(w[q])));
          }
        }
      } else {
        for (uint64_t v = v0 + tid; v < v1; v += NT) {
          RawVec rv;
          fetch<SRC, false>(p, uoff, R, v, rv);
          uint32_t w[4];
          to_words<SRC>(p, rv, w, err);
          for (uint32_t q = 0; q < (rv.nb >> 2); ++q) mz = max(mz, zigzag32(static_cast<int32_t>(w[q])));
        }
      }
      continue;
    }
    // Huffman: exact bit count of this slice under the shared code
    uint32_t zero = 0;
    unsigned long long hb = 0;
    constexpr int UN = 4;
    for (uint64_t base = v0 + static_cast<uint64_t>(warp) * 32; base < v1; base += NT * UN) {
      RawVec rv[UN];
#pragma unroll
      for (int k = 0; k < UN; ++k) {
        const uint64_t v = base + static_cast<uint64_t>(k) * NT + lane;
        rv[k].nb = 0;
        if (v < v1) fetch<SRC, false>(p, uoff, R, v, rv[k]);
      }
#pragma unroll
      for (int k = 0; k < UN; ++k) {
        if (rv[k].nb == 0) continue;
        uint32_t w[4];
        if (rv[k].nb == 16)
          words_full<SRC>(p, rv[k], w, err);
        else
          to_words<SRC>(p, rv[k], w, err);
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j) {
          if (j < rv[k].nb) {
            const uint32_t l = s_clens[byte_of(w, j)];
            hb += l;
            zero |= (l == 0);
          }
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      hb += __shfl_xor_sync(FULL, hb, o);
      zero |= __shfl_xor_sync(FULL, zero, o);
    }
    __syncthreads();
    if (lane == 0) {
      s_r64[0][warp] = hb;
      s_r32[0][warp] = zero;
    }
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < NW; ++i) {
        hb += s_r64[0][i];
        zero |= s_r32[0][i];
      }
      U.part[s].bits = hb;
      U.part[s].zero = zero;
      __threadfence();
      if (atomicAdd(&U.scan_done, 1u) + 1 == unit_slices(p, u)) {
        __threadfence();
        decide_unit<SRC>(p, U, u, false, fast_ok, err);
      }
    }
  }
  if (run_n) flush();
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}

// ------------------------------------------------------------------ pass 3: materialise frames
template <int SRC>
__global__ void __launch_bounds__(NT, 1) emit_kernel(const EncParams p, BUnit* us, BGeom g) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ unsigned long long s_enc[256];
  __shared__ uint32_t s_red32[NW];
  __shared__ uint32_t s_last;
  extern __shared__ __align__(16) uint8_t s_dyn[];
  Scratch& s_x = *reinterpret_cast<Scratch*>(s_dyn);
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  const bool fast_ok = aligned16(p.src) && (p.unit_bytes % 16) == 0;
  const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
  for (int i = tid; i < 256; i += NT) s_enc[i] = ctx_ok ? p.ctx->enc[i] : 0ull;
  __syncthreads();
  uint32_t err = 0;
  for (uint64_t tt = blockIdx.x; tt < g.total; tt += gridDim.x) {
    const uint64_t t = g.total - 1 - tt;  // reverse: pass 2 ended on the last units (L2-resident)
    uint32_t u, s;
    g.unit_of(t, p.nunits, u, s);
    BUnit& U = us[u];
    const uint64_t R = unit_R(p, u);
    const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
    const uint64_t v0 = static_cast<uint64_t>(s) * BV;
    const uint64_t v1 = min(v0 + BV, (R + 15) / 16);
    uint8_t* stage = p.stages + static_cast<uint64_t>(u) * p.stride;
    uint8_t* payload = stage + kHeaderBytes;
    const uint32_t target = target_codec(p, U, ctx_ok);
    uint32_t codec, width = 0;
    uint64_t P;
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
    if (codec == CODEC_NONE) {
      if (s == 0) err |= ZC_DERR_CAPACITY;
    } else if (codec == ZC_CODEC_RAW) {
      constexpr int UN = 4;
      for (uint64_t base = v0 + tid; base < v1; base += NT * UN) {
        RawVec rv[UN];
#pragma unroll
        for (int k = 0; k < UN; ++k) {
          const uint64_t v = base + static_cast<uint64_t>(k) * NT;
          rv[k].nb = 0;
          if (v < v1) fetch<SRC, false>(p, uoff, R, v, rv[k]);
        }
#pragma unroll
        for (int k = 0; k < UN; ++k) {
          const uint64_t v = base + static_cast<uint64_t>(k) * NT;
          if (v >= v1) continue;
          uint32_t w[4];
          if (rv[k].nb == 16)
            words_full<SRC>(p, rv[k], w, err);
          else
            to_words<SRC>(p, rv[k], w, err);
          uint8_t* d = payload + v * 16;
          if (rv[k].nb == 16 && aligned16(d)) {
            *reinterpret_cast<uint4*>(d) = make_uint4(w[0], w[1], w[2], w[3]);
          } else {
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j)
              if (j < rv[k].nb) d[j] = static_cast<uint8_t>(byte_of(w, j));
          }
        }
      }
    } else if (codec == ZC_CODEC_FIXEDLEN) {
      uint4* zz = s_x.zz[warp];
      const uint64_t vfull = min(v1, R / 16);
      for (uint64_t base = v0 + static_cast<uint64_t>(warp) * 256; base < v1; base += static_cast<uint64_t>(NW) * 256) {
        if (fast_ok && base + 256 <= vfull) {
          RawVec rv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) fetch_full<SRC, false>(p, uoff, base + 32 * j + lane, rv[j]);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t w[4];
            words_full<SRC>(p, rv[j], w, err);
            const uint32_t slot = 32 * j + lane;
            zz[slot ^ ((slot >> 3) & 7)] =
                make_uint4(zigzag32(static_cast<int32_t>(w[0])), zigzag32(static_cast<int32_t>(w[1])),
                           zigzag32(static_cast<int32_t>(w[2])), zigzag32(static_cast<int32_t>(w[3])));
          }
        } else {
          RawVec rv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint64_t v = base + 32 * j + lane;
            rv[j].nb = 0;
            if (v < v1) fetch<SRC, false>(p, uoff, R, v, rv[j]);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t w[4] = {0, 0, 0, 0};
            if (rv[j].nb) to_words<SRC>(p, rv[j], w, err);
            uint32_t zq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              zq[q] = (static_cast<uint32_t>(q) < (rv[j].nb >> 2)) ? zigzag32(static_cast<int32_t>(w[q])) : 0u;
            const uint32_t slot = 32 * j + lane;
            zz[slot ^ ((slot >> 3) & 7)] = make_uint4(zq[0], zq[1], zq[2], zq[3]);
          }
        }
        __syncwarp();
        uint32_t z[32];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint32_t slot = 8 * lane + m;
          const uint4 q = zz[slot ^ ((slot >> 3) & 7)];
          z[4 * m] = q.x;
          z[4 * m + 1] = q.y;
          z[4 * m + 2] = q.z;
          z[4 * m + 3] = q.w;
        }
        __syncwarp();
        if ((base + 8 * lane) < v1) pack_store_w(width, z, payload, (base / 8 + lane) * width, P);
      }
    } else {  // Huffman
      uint32_t* tile = s_x.tile;
      uint32_t* uindex = p.index ? p.index + static_cast<uint64_t>(u) * p.index_stride : nullptr;
      unsigned long long base_bits = __ldcg(&U.hbase[s]);
      for (int i = tid; i < TILE_WORDS; i += NT) tile[i] = 0;
      bool first_tile = true, has_head = false;
      unsigned long long head_idx = 0;
      uint32_t head_val = 0, end_mod = 0;
      __syncthreads();
      for (uint64_t t0 = v0; t0 < v1; t0 += NT) {
        const uint64_t v = t0 + tid;
        uint32_t w[4] = {0, 0, 0, 0}, nb = 0;
        if (v < v1) {
          RawVec rv;
          fetch<SRC, false>(p, uoff, R, v, rv);
          to_words<SRC>(p, rv, w, err);
          nb = rv.nb;
        }
        unsigned long long ev[16];
        uint32_t Lb = 0;
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j) {
          ev[j] = j < nb ? s_enc[byte_of(w, j)] : 0ull;
          Lb += static_cast<uint32_t>(ev[j] >> 32);
        }
        uint32_t ttot;
        const uint32_t off = block_excl_scan(Lb, s_red32, &ttot);
        if (v < v1 && uindex != nullptr && (v & 63) == 0) uindex[v >> 6] = static_cast<uint32_t>(base_bits + off);
        {
          const uint32_t lp = static_cast<uint32_t>(base_bits & 31) + off;
          uint32_t wi = lp >> 5, nbit = lp & 31;
          unsigned long long acc = 0;
          bool firstw = true;
#pragma unroll
          for (uint32_t j = 0; j < 16; ++j) {
            const unsigned long long e = ev[j];
            if (!(e >> 32)) continue;
            acc |= (e & 0xffffffffull) << nbit;
            nbit += static_cast<uint32_t>(e >> 32);
            if (nbit >= 32) {
              if (firstw) atomicOr(&tile[wi], static_cast<uint32_t>(acc));
              else tile[wi] = static_cast<uint32_t>(acc);
              firstw = false;
              ++wi;
              acc >>= 32;
              nbit -= 32;
            }
          }
          if (nbit > 0) atomicOr(&tile[wi], static_cast<uint32_t>(acc));
        }
        __syncthreads();
        const uint32_t endb = static_cast<uint32_t>(base_bits & 31) + ttot;
        const uint32_t full = endb >> 5;
        const uint64_t gw0 = base_bits >> 5;
        for (uint32_t i = tid; i < full; i += NT) {
          if (i == 0 && first_tile) {
            if (tid == 0) {
              has_head = true;
              head_idx = gw0;
              head_val = tile[0];
            }
          } else {
            store_word_safe(payload, gw0 + i, tile[i], P);
          }
        }
        const uint32_t carry = (endb & 31) ? tile[full] : 0u;
        __syncthreads();
        for (uint32_t i = tid; i <= full + 1 && i < static_cast<uint32_t>(TILE_WORDS); i += NT) tile[i] = 0;
        __syncthreads();
        if (tid == 0) tile[0] = carry;
        if (full > 0) first_tile = false;
        base_bits += ttot;
        end_mod = static_cast<uint32_t>(base_bits & 31);
        __syncthreads();
      }
      if (tid == 0) {
        U.has_head[s] = has_head ? 1u : 0u;
        U.head_idx[s] = head_idx;
        U.head_val[s] = head_val;
        U.has_tail[s] = (v0 < v1 && end_mod != 0) ? 1u : 0u;
        U.tail_idx[s] = base_bits >> 5;
        U.tail_val[s] = tile[0];
        __threadfence();
        s_last = atomicAdd(&U.edone, 1u) == unit_slices(p, u) - 1 ? 1u : 0u;
        if (s_last) {  // the unit's last slice merges the seam words (OR of head/tail halves)
          __threadfence();
          const uint32_t ns = unit_slices(p, u);
          unsigned long long cur_idx = ~0ull;
          uint32_t cur = 0;
          for (uint32_t r = 0; r < ns; ++r) {
            for (int k = 0; k < 2; ++k) {
              const bool has = k == 0 ? __ldcg(&U.has_head[r]) : __ldcg(&U.has_tail[r]);
              if (!has) continue;
              const unsigned long long idx = k == 0 ? __ldcg(&U.head_idx[r]) : __ldcg(&U.tail_idx[r]);
              const uint32_t val = k == 0 ? __ldcg(&U.head_val[r]) : __ldcg(&U.tail_val[r]);
              if (idx == cur_idx) {
                cur |= val;
              } else {
                if (cur_idx != ~0ull) store_word_safe(payload, cur_idx, cur, P);
                cur_idx = idx;
                cur = val;
              }
            }
          }
          if (cur_idx != ~0ull) store_word_safe(payload, cur_idx, cur, P);
        }
      }
      __syncthreads();
    }
    // header + result: slice 0 of the unit
    if (s == 0 && tid == 0) {
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
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}

template <int SRC>
cudaError_t launch_batch_t(const EncParams& p, void* scratch, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(emit_kernel<SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaMemsetAsync(scratch, 0, sizeof(BUnit) * p.nunits, s);
  BUnit* us = static_cast<BUnit*>(scratch);
  BGeom g;
  g.s_full = static_cast<uint32_t>((p.unit_bytes + BS - 1) / BS);
  const uint64_t last_R = p.total_bytes - static_cast<uint64_t>(p.nunits - 1) * p.unit_bytes;
  g.total = static_cast<uint64_t>(p.nunits - 1) * g.s_full + (last_R + BS - 1) / BS;
  if (p.pin == ZC_PIN_AUTO) {
    note_launch();
    profile_kernel<SRC><<<p.nunits * PC, PT, 0, s>>>(p, us);
  }
  const bool ctx_ok_host = p.ctx != nullptr;  // validity is checked on the device
  if (p.pin == ZC_PIN_AUTO || p.pin == ZC_PIN_FIXEDLEN || (p.pin == ZC_PIN_HUFFMAN && ctx_ok_host)) {
    note_launch();
    scan_kernel<SRC><<<static_cast<uint32_t>(std::min<uint64_t>(g.total, static_cast<uint64_t>(sms))), NT, 0, s>>>(p, us, g);
  }
  note_launch();
  emit_kernel<SRC><<<static_cast<uint32_t>(std::min<uint64_t>(g.total, static_cast<uint64_t>(sms))), NT,
                     sizeof(Scratch), s>>>(p, us, g);
  return cudaGetLastError();
}

}  // namespace

size_t batch_scratch_bytes(uint32_t nunits) { return sizeof(BUnit) * (nunits ? nunits : 1); }

void preload_batch_kernels() {
  cudaFuncSetAttribute(emit_kernel<SRC_BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncSetAttribute(emit_kernel<SRC_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncSetAttribute(emit_kernel<SRC_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, profile_kernel<SRC_BYTES>);
  cudaFuncGetAttributes(&a, profile_kernel<SRC_F32>);
  cudaFuncGetAttributes(&a, profile_kernel<SRC_F64>);
  cudaFuncGetAttributes(&a, scan_kernel<SRC_BYTES>);
  cudaFuncGetAttributes(&a, scan_kernel<SRC_F32>);
  cudaFuncGetAttributes(&a, scan_kernel<SRC_F64>);
  cudaGetLastError();
}

cudaError_t launch_encode_batch(const EncParams& p, void* scratch, cudaStream_t s) {
  if (p.nunits == 0) return cudaSuccess;
  switch (p.src_kind) {
    case SRC_F32:
      return launch_batch_t<SRC_F32>(p, scratch, s);
    case SRC_F64:
      return launch_batch_t<SRC_F64>(p, scratch, s);
    default:
      return launch_batch_t<SRC_BYTES>(p, scratch, s);
  }
}

}  // namespace zc
