// zc_fixed.cu — the fp32 hot path of the batched send encoder (send_encoded over a message,
// collectives.cpp:201-302 for every 4 MiB batch) for units that end up FixedLen or RAW:
//
//   range    one HBM stream over the FixedLen-target units: fp32 min / max (NaN-propagating), so
//            the unit's width is width(max(zz(q(min)), zz(q(max)))) — quantization is monotone —
//            without quantizing anything; the unit's last slice runs decide_unit (the post-checks
//            of encode_best, rea.cpp:189-236, or the pinned send_batch fallbacks,
//            collectives.cpp:223-275).
//   emit     quantize (quant.cpp:22-27) + zig-zag + LSB-first pack (fixedlen.cpp:15-37) or the raw
//            symbol copy, streamed through TMA: each warp owns a ring of 4 KiB tiles (32 rows x 32
//            fp32, 128-byte swizzle) filled by cp.async.bulk.tensor and signalled on mbarriers, so
//            HBM reads run ahead of the arithmetic.  Lane L owns the 32 consecutive symbols of row
//            L, whose packed bits are exactly W whole words (W = width): the pack is compile-time
//            shifts in registers and the words go out as 16/8/4-byte stores.
//
// Huffman units (and every non-fp32 / unaligned source) stay on zc_batch.cu's kernels, which skip
// the units handled here.  Frames are byte-identical to the reference's.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "zc_batch.cuh"
#include "zc_tma.cuh"

namespace zc {
namespace {

constexpr int RT = 512;                  // range kernel threads
constexpr int ET_WARPS = 16;             // emit kernel warps per CTA
constexpr int ET = ET_WARPS * 32;
constexpr int ET_CTAS = 1;               // emit CTAs per SM
constexpr int STAGES = 3;                // tiles in flight per warp
constexpr uint32_t TILE_ELEMS = 1024;    // 32 x 32 fp32
constexpr uint32_t TILE_BYTES = TILE_ELEMS * 4;
// A unit (batch) is 2^ush tiles: 1024 for 4 MiB batches, 128 for 512 KiB slots (per-slot framing).
__host__ __device__ __forceinline__ uint32_t unit_tile_shift(uint64_t unit_bytes) {
  uint32_t s = 0;
  while ((static_cast<uint64_t>(TILE_BYTES) << s) < unit_bytes) ++s;
  return s;
}
constexpr size_t EMIT_SMEM = static_cast<size_t>(ET_WARPS) * STAGES * TILE_BYTES + 1024 + ET_WARPS * STAGES * 8;

__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// ------------------------------------------------------------------ range (+ profile and plan)
// Exact symbols of a 16-byte fp32 vector (fast path, exact division near a tie).
__device__ __noinline__ uint32_t quantize_exact(float x, double scale, double rcp, uint32_t* err);
__device__ __forceinline__ void quantize4(const float4& a, double scale, double rcp, uint32_t (&w)[4], uint32_t& err) {
  const float f[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    bool slow = !(fabsf(f[k]) <= 3.402823466e38f);
    const int32_t q = quantize_fast(static_cast<double>(f[k]), rcp, slow);
    w[k] = slow ? quantize_exact(f[k], scale, rcp, &err) : static_cast<uint32_t>(q);
  }
}

// profile_sample over the window (rea.cpp:93-118; the window is the unit's slice 0): byte
// histogram in per-warp shared bins with warp-aggregated atomics (one atomic per distinct byte
// value per warp instruction), max zig-zag over whole words; then the expected code length
// under the shared context and arbitrate_plan (rea.cpp:145-176).  Whole CTA.
struct ProfSmem {
  uint32_t whist[RT / 32][256];
  uint32_t hist[256];
  uint8_t clens[256];
  uint32_t wmz[RT / 32];
};
template <int SRC>
__device__ __forceinline__ void window_profile(const EncParams& p, BUnit& U, uint32_t u, const float4* src, uint64_t R,
                                               bool ctx_ok, ProfSmem& sm, uint32_t& err) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < (RT / 32) * 256; i += RT) (&sm.whist[0][0])[i] = 0;
  for (int i = tid; i < 256; i += RT) sm.clens[i] = ctx_ok ? p.ctx->len[i] : 0;
  __syncthreads();
  const uint64_t W = R < kSampleWindow ? R : kSampleWindow;  // whole words: R % 4 == 0 on this path
  uint32_t wmz = 0;
  for (uint64_t v0 = 0; v0 * 16 < W; v0 += RT) {
    const uint64_t v = v0 + tid;
    const bool in = v * 16 < W;
    uint32_t w[4] = {0, 0, 0, 0};
    uint32_t nb = 0;
    if (in) {
      nb = static_cast<uint32_t>(W - v * 16 < 16 ? W - v * 16 : 16);
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (nb == 16) {
        a = __ldg(src + v);
      } else {
        const float* fs = reinterpret_cast<const float*>(src + v);
        a.x = nb > 0 ? __ldg(fs) : 0.f;
        a.y = nb > 4 ? __ldg(fs + 1) : 0.f;
        a.z = nb > 8 ? __ldg(fs + 2) : 0.f;
      }
      if (SRC == SRC_F32) {
        quantize4(a, enc_scale(p), enc_rcp(p), w, err);
      } else {  // symbols already
        w[0] = __float_as_uint(a.x);
        w[1] = __float_as_uint(a.y);
        w[2] = __float_as_uint(a.z);
        w[3] = __float_as_uint(a.w);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (static_cast<uint32_t>(k) < nb / 4) wmz = max(wmz, zigzag32(static_cast<int32_t>(w[k])));
    }
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j) {
      const bool act = in && j < nb;
      const uint32_t byte = (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
      const uint32_t key = act ? byte : 0x100u;  // inactive lanes group apart
      const uint32_t peers = __match_any_sync(FULL, key);
      if (act && (__ffs(peers) - 1) == lane) atomicAdd(&sm.whist[warp][byte], static_cast<uint32_t>(__popc(peers)));
    }
  }
  for (int o = 16; o > 0; o >>= 1) wmz = max(wmz, __shfl_xor_sync(FULL, wmz, o));
  if (lane == 0) sm.wmz[warp] = wmz;
  __syncthreads();
  for (int i = tid; i < 256; i += RT) {
    uint32_t c = 0;
#pragma unroll
    for (int w2 = 0; w2 < RT / 32; ++w2) c += sm.whist[w2][i];
    sm.hist[i] = c;
  }
  __syncthreads();
  double el = 0.0;
  bool el_ok = false;
  if (warp == 0) el_ok = ctx_ok && warp_mean_len(sm.hist, sm.clens, el);
  if (p.stats != nullptr)
    for (int i = tid; i < 256; i += RT) p.stats[u].hist[i] = sm.hist[i];
  if (tid == 0) {
    zc_sample_stats st;
    st.sampled_bytes = W;
    uint32_t m = 0;
    for (int i = 0; i < RT / 32; ++i) m = max(m, sm.wmz[i]);
    st.max_zigzag = m;
    U.wmz = m;
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
    const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
    U.plan = arbitrate_plan(R, pcap, st, p.hint, ctx_ok, p.cfg).choice;
  }
}

// One HBM stream over the units that may end up FixedLen: fp32 min / max (NaN-propagating) per
// unit.  Work is claimed dynamically: in Auto the first nunits tasks profile each unit's window
// and store its plan (window_profile), the rest are runs of RCH consecutive 64 KiB slices.  A unit
// is complete when its slices and (Auto) its profile have been counted; the task that completes
// it decides FixedLen units (decide_unit).  Huffman-planned units are decided by scan_kernel's
// bit counts, RAW ones by emit.
constexpr uint32_t RCH = 8;

__device__ __forceinline__ uint32_t zz4(const float4& a) {
  return max(max(zigzag32(__float_as_int(a.x)), zigzag32(__float_as_int(a.y))),
             max(zigzag32(__float_as_int(a.z)), zigzag32(__float_as_int(a.w))));
}

template <int SRC>
__global__ void __launch_bounds__(RT, 2) range_kernel(const __grid_constant__ EncParams p, BUnit* us, BGeom g) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float s_mn[RT / 32], s_mx[RT / 32];
  __shared__ uint32_t s_mz[RT / 32];
  __shared__ ProfSmem s_prof;
  __shared__ uint32_t s_task;
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  const bool automode = p.pin == ZC_PIN_AUTO && !g.planned;  // window profiles are this kernel's tasks
  // symbols whose per-unit max zig-zag the producer already knows (the ring's reduce sink): no
  // slice is read; one task per unit profiles the window (Auto) and decides
  const bool pre = SRC != SRC_F32 && p.maxzz_in != nullptr;
  const uint32_t nprof = (automode || g.spec || pre) ? p.nunits : 0u;
  const uint64_t nchunks = (g.spec || pre) ? 0 : (g.total + RCH - 1) / RCH;
  BGlobal* gl = bglobal(us, p.nunits);
  uint32_t err = 0;
  float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
  uint32_t mz = 0;  // symbol sources: max zig-zag
  uint32_t run_u = 0xffffffffu, run_n = 0;
  // counts `n` finished pieces of unit u (thread 0); the completing one decides
  auto finish = [&](BUnit& U, uint32_t u, uint32_t n) {
    __threadfence();
    if (atomicAdd(&U.scan_done, n) + n == unit_slices(p, u) + (automode ? 1u : 0u)) {
      __threadfence();
      const uint32_t plan = *reinterpret_cast<volatile uint32_t*>(&U.plan);
      if (plan == ZC_CODEC_HUFFMAN && automode) atomicAdd(&gl->n_huff, 1u);
      if (target_codec(p, U, ctx_ok) == ZC_CODEC_FIXEDLEN) decide_unit<SRC>(p, U, u, true, true, err);
    }
  };
  auto flush = [&]() {
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin_nan(mn, __shfl_xor_sync(FULL, mn, o));
      mx = fmax_nan(mx, __shfl_xor_sync(FULL, mx, o));
      mz = max(mz, __shfl_xor_sync(FULL, mz, o));
    }
    __syncthreads();
    if (lane == 0) {
      s_mn[warp] = mn;
      s_mx[warp] = mx;
      s_mz[warp] = mz;
    }
    __syncthreads();
    if (tid == 0) {
      for (int i = 1; i < RT / 32; ++i) {
        mn = fmin_nan(mn, s_mn[i]);
        mx = fmax_nan(mx, s_mx[i]);
        mz = max(mz, s_mz[i]);
      }
      BUnit& U = us[run_u];
      if (SRC == SRC_F32) {
        const bool bad = !(fabsf(mn) <= 3.402823466e38f) || !(fabsf(mx) <= 3.402823466e38f);  // NaN / Inf
        if (bad) atomicOr(&U.bad, 1u);
        atomicMax(&U.fmin_c, ~fkey(mn));
        atomicMax(&U.fmax_k, fkey(mx));
      } else {
        atomicMax(&U.maxzz, mz);
      }
      finish(U, run_u, run_n);
    }
    mn = __int_as_float(0x7f800000);
    mx = -__int_as_float(0x7f800000);
    mz = 0;
    run_n = 0;
  };
  for (;;) {
    __syncthreads();
    if (tid == 0) s_task = atomicAdd(&gl->next_task, 1u);
    __syncthreads();
    const uint32_t task = s_task;
    if (task < nprof) {  // profile + plan of unit `task`
      const uint32_t u = task;
      const uint64_t R = unit_R(p, u);
      if (R <= p.cfg.small_batch_threshold_bytes || p.stage_len <= kHeaderBytes) {
        if (tid == 0) us[u].plan = ZC_CODEC_RAW;
      } else if (automode || g.spec) {
        const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(p.src) + static_cast<uint64_t>(u) * (p.unit_bytes / 4));
        window_profile<SRC>(p, us[u], u, src, R, ctx_ok, s_prof, err);
      }
      __syncthreads();
      if (tid == 0) {
        if (g.spec) {  // the emit decides; here only the plan census and the width guess
          BUnit& U = us[u];
          if (automode && U.plan == ZC_CODEC_HUFFMAN) atomicAdd(&gl->n_huff, 1u);
        } else if (pre) {  // the unit's range is known: complete it at once
          atomicMax(&us[u].maxzz, __ldcg(p.maxzz_in + u));
          finish(us[u], u, unit_slices(p, u) + (automode ? 1u : 0u));
        } else {
          finish(us[u], u, 1u);
        }
      }
      continue;
    }
    const uint64_t ch = task - nprof;
    if (ch >= nchunks) break;
    const uint64_t te = min(g.total, (ch + 1) * RCH);
    for (uint64_t t = ch * RCH; t < te; ++t) {
      uint32_t u, s;
      g.unit_of(t, p.nunits, u, s);
      // Auto: every slice (the plan may not be known yet); FixedLen pin: FixedLen targets only
      if (!automode && target_codec(p, us[u], ctx_ok) != ZC_CODEC_FIXEDLEN) continue;
      if (run_n && run_u != u) flush();
      run_u = u;
      ++run_n;
      const uint64_t R = unit_R(p, u);
      const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(p.src) + static_cast<uint64_t>(u) * (p.unit_bytes / 4));
      const uint64_t nf = R / 16;  // whole 16-byte vectors of the unit
      const uint64_t v0 = static_cast<uint64_t>(s) * BV;
      if (v0 + BV <= nf) {
        const float4* q = src + v0 + tid;
        float4 a[BV / RT];
#pragma unroll
        for (int k = 0; k < static_cast<int>(BV / RT); ++k) a[k] = __ldg(q + k * RT);
#pragma unroll
        for (int k = 0; k < static_cast<int>(BV / RT); ++k) {
          if (SRC == SRC_F32) {
            mn = fmin_nan(mn, fmin_nan(fmin_nan(a[k].x, a[k].y), fmin_nan(a[k].z, a[k].w)));
            mx = fmax_nan(mx, fmax_nan(fmax_nan(a[k].x, a[k].y), fmax_nan(a[k].z, a[k].w)));
          } else {
            mz = max(mz, zz4(a[k]));
          }
        }
      } else {
        const uint64_t v1 = min(v0 + BV, nf);
        for (uint64_t v = v0 + tid; v < v1; v += RT) {
          const float4 a = __ldg(src + v);
          if (SRC == SRC_F32) {
            mn = fmin_nan(mn, fmin_nan(fmin_nan(a.x, a.y), fmin_nan(a.z, a.w)));
            mx = fmax_nan(mx, fmax_nan(fmax_nan(a.x, a.y), fmax_nan(a.z, a.w)));
          } else {
            mz = max(mz, zz4(a));
          }
        }
        if (tid == 0 && v0 * 16 + BS >= R) {  // the unit's last 0..3 elements
          const float* fl = reinterpret_cast<const float*>(src);
          for (uint64_t e = nf * 4; e < R / 4; ++e) {
            const float v = __ldg(fl + e);
            if (SRC == SRC_F32) {
              mn = fmin_nan(mn, v);
              mx = fmax_nan(mx, v);
            } else {
              mz = max(mz, zigzag32(__float_as_int(v)));
            }
          }
        }
      }
    }
    if (run_n) flush();  // a run never outlives its task: units are counted task by task
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}

// ------------------------------------------------------------------ emit
// Quantizes the 32 fp32 values of a row; exact division (quantize_one) for any lane whose row
// holds a value near a rounding tie.  `big` = the unit may hold |q| >= 2^30 (then every value
// takes quantize_one).
// quantize_one out of line: the rare exact path (near a tie, |q| >= 2^30, non-finite) must not
// force the callers' per-row arrays into local memory.
__device__ __noinline__ uint32_t quantize_exact(float x, double scale, double rcp, uint32_t* err) {
  uint32_t e = 0;
  const uint32_t r = static_cast<uint32_t>(quantize_one(static_cast<double>(x), scale, rcp, e));
  *err |= e;
  return r;
}

// |a| max |b| max |c| in one FMNMX3 (three-input max, sm_100+).
__device__ __forceinline__ float absmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(fabsf(b)), "f"(fabsf(c)));
  return r;
}

// The fast path below is exact only while |q| < 2^30 (the low word of t holds the integer and
// |x*rcp - x/scale| < 2^-22).  `xlim` = RZ(2^29 * scale): a row holding any |x| >= xlim takes the
// exact division, which raises the reference's int32-range error (quant.cpp:22-27) where it is
// due.  NaN compares false here, but its residual is NaN and trips the tie test.
__device__ __forceinline__ float fast_xlim(double scale) { return __double2float_rz(__dmul_rn(scale, 536870912.0)); }

__device__ __forceinline__ void quantize_row(const float (&x)[32], double scale, double rcp, float xlim, bool big,
                                             uint32_t (&s)[32], uint32_t& err) {
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  uint32_t rm = 0;  // max over the row of the high word of |r|, r = q - round(q)
  float am = 0.f;   // max |x| over the row
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    // t = RN(x*rcp + M): the nearest integer to x*rcp in its low word; r = RN(x*rcp - k) is the
    // residual to that integer (one rounding), so |x/scale - k| <= |r| + 2^-22 for |q| < 2^30
    const double xd = static_cast<double>(x[i]);
    const double t = __fma_rn(xd, rcp, kMagic);
    const double r = __fma_rn(xd, rcp, -__dsub_rn(t, kMagic));
    rm = max(rm, static_cast<uint32_t>(__double2hiint(r)) & 0x7fffffffu);
    s[i] = static_cast<uint32_t>(__double2loint(t));
    if (i & 1) am = absmax3(am, x[i - 1], x[i]);
  }
  // a value within 2^-18 of a rounding tie (|r| >= 0.5 - 2^-18, high word >= 0x3FDFFFF0), a value
  // outside the fast range, or a unit flagged as such: exact path for the row
  if (big || rm >= 0x3FDFFFF0u || !(am < xlim)) {
#pragma unroll
    for (int i = 0; i < 32; ++i) s[i] = quantize_exact(x[i], scale, rcp, &err);
  }
}

// Packs 32 zig-zag symbols of width W into W words and stores them at word `wb` of the payload
// (no bound: the row lies wholly inside the payload).
template <int W>
__device__ __forceinline__ void pack_store_full(const uint32_t (&z)[32], uint32_t* dst) {
  uint32_t o[W];
#pragma unroll
  for (int k = 0; k < W; ++k) o[k] = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {  // fields are disjoint: + is | (one IMAD per symbol)
    const int bit = i * W, k = bit >> 5, sh = bit & 31;
    o[k] += z[i] << sh;
    if (sh + W > 32) o[k + 1] += z[i] >> (32 - sh);
  }
  if (W % 4 == 0) {
#pragma unroll
    for (int j = 0; j < W / 4; ++j) reinterpret_cast<uint4*>(dst)[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  } else if (W % 2 == 0) {
#pragma unroll
    for (int j = 0; j < W / 2; ++j) reinterpret_cast<uint2*>(dst)[j] = make_uint2(o[2 * j], o[2 * j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j) dst[j] = o[j];
  }
}

__device__ __forceinline__ void store_row(uint32_t codec, uint32_t width, const uint32_t (&s)[32], uint8_t* payload,
                                          uint64_t row_sym) {
  uint32_t* base = reinterpret_cast<uint32_t*>(payload);
  if (codec == ZC_CODEC_RAW) {
    uint4* d = reinterpret_cast<uint4*>(base + row_sym);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j] = make_uint4(s[4 * j], s[4 * j + 1], s[4 * j + 2], s[4 * j + 3]);
    return;
  }
  uint32_t z[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) z[i] = zigzag32(static_cast<int32_t>(s[i]));
  uint32_t* d = base + (row_sym / 32) * width;
  switch (width) {
#define ZC_PS(W)                   \
  case W:                          \
    pack_store_full<W>(z, d);      \
    break;
    ZC_PS(1) ZC_PS(2) ZC_PS(3) ZC_PS(4) ZC_PS(5) ZC_PS(6) ZC_PS(7) ZC_PS(8) ZC_PS(9) ZC_PS(10) ZC_PS(11)
    ZC_PS(12) ZC_PS(13) ZC_PS(14) ZC_PS(15) ZC_PS(16) ZC_PS(17) ZC_PS(18) ZC_PS(19) ZC_PS(20) ZC_PS(21)
    ZC_PS(22) ZC_PS(23) ZC_PS(24) ZC_PS(25) ZC_PS(26) ZC_PS(27) ZC_PS(28) ZC_PS(29) ZC_PS(30) ZC_PS(31)
    ZC_PS(32)
#undef ZC_PS
    default:
      break;
  }
}

// Half a row (16 values): quantize_row's fast path and exactness test on 16 values, so a row is
// quantized and packed in two passes and only half of it is live in registers at a time.
__device__ __forceinline__ void quantize_half(const float (&x)[16], double scale, double rcp, float xlim, bool big,
                                              uint32_t (&s)[16], uint32_t& err) {
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  uint32_t rm = 0;
  float am = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double xd = static_cast<double>(x[i]);
    const double t = __fma_rn(xd, rcp, kMagic);
    const double r = __fma_rn(xd, rcp, -__dsub_rn(t, kMagic));
    rm = max(rm, static_cast<uint32_t>(__double2hiint(r)) & 0x7fffffffu);
    s[i] = static_cast<uint32_t>(__double2loint(t));
    if (i & 1) am = absmax3(am, x[i - 1], x[i]);
  }
  if (big || rm >= 0x3FDFFFF0u || !(am < xlim)) {
#pragma unroll
    for (int i = 0; i < 16; ++i) s[i] = quantize_exact(x[i], scale, rcp, &err);
  }
}

// One row (lane's 32 values of a swizzled fp32 / symbol tile in shared memory) -> its W packed
// words (FixedLen) or 32 symbol words (kRaw), in two 16-value halves; `spec`: the exact symbols'
// max zig-zag into sp_mz.
template <int W, bool kRaw, int SRC>
__device__ __forceinline__ void emit_row(uint32_t row, int lane, double scale, double rcp, float xlim, bool big, bool spec,
                                         uint32_t& sp_mz, uint32_t* dst, uint32_t& err) {
  uint32_t o[W];
#pragma unroll
  for (int k = 0; k < W; ++k) o[k] = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float x[16];
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      const int m = 4 * h + mm;
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(x[4 * mm]), "=f"(x[4 * mm + 1]), "=f"(x[4 * mm + 2]), "=f"(x[4 * mm + 3])
                   : "r"(row + ((m ^ (lane & 7)) << 4)));
    }
    uint32_t sv[16];
    if (SRC == SRC_F32) {
      quantize_half(x, scale, rcp, xlim, big, sv, err);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) sv[i] = __float_as_uint(x[i]);
    }
    if (spec) {
#pragma unroll
      for (int i = 0; i < 16; ++i) sp_mz = max(sp_mz, zigzag32(static_cast<int32_t>(sv[i])));
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int idx = 16 * h + i;
      if (kRaw) {
        o[idx] = sv[i];
      } else {  // fields are disjoint: + is | (one IMAD per symbol)
        const uint32_t z = zigzag32(static_cast<int32_t>(sv[i]));
        const int bit = idx * W, k = bit >> 5, sh = bit & 31;
        o[k] += z << sh;
        if (sh + W > 32) o[k + 1] += z >> (32 - sh);
      }
    }
  }
  if (W % 4 == 0) {
#pragma unroll
    for (int j = 0; j < W / 4; ++j) reinterpret_cast<uint4*>(dst)[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
  } else if (W % 2 == 0) {
#pragma unroll
    for (int j = 0; j < W / 2; ++j) reinterpret_cast<uint2*>(dst)[j] = make_uint2(o[2 * j], o[2 * j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j) dst[j] = o[j];
  }
}

// Grid sizing: a warp's share of the tiles is about CHUNK tiles when the message fills the GPU;
// a small message (the latency regime of small collectives) is spread one tile per warp instead.
constexpr uint64_t CHUNK = 4;
// The decoder's warp tile order: warp gw owns chunks gw, gw + tw, ... of `ch` consecutive tiles
// (ch divides the unit's tiles: chunks never straddle a unit), so the warps in flight write one
// advancing window of the output.
__device__ __forceinline__ uint64_t tile_adv(uint64_t c, uint64_t tw, uint32_t ch) {
  return ((c + 1) % ch) != 0 ? c + 1 : c + 1 + (tw - 1) * ch;
}
// The warp's first tile at or past tile `ue` (a unit boundary), given its current tile c.
__device__ __forceinline__ uint64_t tile_skip_to(uint64_t c, uint64_t ue, uint64_t tw, uint32_t ch) {
  const uint64_t j = c / ch, je = ue / ch;
  return (j + ((je - j + tw - 1) / tw) * tw) * ch;
}
// Tiles per warp chunk for a message of `ntiles` over `slots` warps the GPU can run.
inline uint32_t chunk_for(uint64_t ntiles, uint64_t slots) {
  uint64_t ch = CHUNK;
  while (ch > 1 && ntiles < ch * slots) ch >>= 1;
  return static_cast<uint32_t>(ch);
}

constexpr uint32_t kForeign = 0xFEu;  // unit owned by the general kernels

struct UnitView {
  uint32_t codec, width;
  uint64_t P;
  bool big, spec;
};

// Per-unit view for the emit kernel: owned (RAW / FixedLen) or not, and whether the fast
// quantizer applies (max |q| < 2^30 over the unit, from the range pass).
__device__ __forceinline__ UnitView unit_view(const EncParams& p, const BUnit* us, uint32_t u, bool ctx_ok);

// mode 1: a FixedLen-target unit is packed with the window's width (`spec`; its header waits for
// the decision); mode 2: only the units the decision sent back (redo) are owned.
template <int kMode>
__device__ __forceinline__ UnitView unit_view_m(const EncParams& p, const BUnit* us, uint32_t u, bool ctx_ok) {
  UnitView v = unit_view(p, us, u, ctx_ok);
  v.spec = false;
  if (kMode == 1 && p.stage_len > kHeaderBytes && target_codec(p, us[u], ctx_ok) == ZC_CODEC_FIXEDLEN) {
    v.codec = ZC_CODEC_FIXEDLEN;
    v.width = width_from_maxzz(us[u].wmz);
    v.P = packed_bytes(unit_R(p, u) / 4, v.width);
    v.big = v.width >= 31;
    v.spec = true;
  }
  if (kMode == 2 && !us[u].redo) v.codec = kForeign;
  return v;
}

__device__ __forceinline__ UnitView unit_view(const EncParams& p, const BUnit* us, uint32_t u, bool ctx_ok) {
  UnitView v;
  final_codec(p, us[u], u, ctx_ok, v.codec, v.width, v.P);
  // ownership is by TARGET: a Huffman-target unit (even one that fell back to RAW) belongs to
  // zc_batch.cu's kernels
  if (target_codec(p, us[u], ctx_ok) == ZC_CODEC_HUFFMAN) v.codec = kForeign;
  v.big = true;
  if (v.codec == ZC_CODEC_FIXEDLEN) {
    // the width is < 31 iff max zz < 2^30, i.e. every |q| < 2^29
    v.big = v.width >= 31;
  }
  return v;
}

__device__ __forceinline__ bool owned(uint32_t codec) { return codec == ZC_CODEC_RAW || codec == ZC_CODEC_FIXEDLEN; }

// Speculative FixedLen (mode 1): the tile's value range goes into the unit (the range pass's
// keys), and the unit's last tile decides it (decide_unit: encode_best's post-checks / the pinned
// fallbacks).  When the decision is FixedLen at the speculated width, the frame is complete and
// its header is written; otherwise the unit is marked for the redo emit.  One lane per warp.
template <int SRC>
__device__ __noinline__ void spec_flush(const EncParams& p, BUnit* us, uint32_t u, uint32_t mz, uint32_t ntiles,
                                       uint32_t* err) {
  BUnit& U = us[u];
  atomicMax(&U.maxzz, mz);
  const uint32_t ntu = static_cast<uint32_t>((unit_R(p, u) / 4 + TILE_ELEMS - 1) / TILE_ELEMS);
  uint32_t old;  // release: this warp's range is in before its tiles count
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(&U.tdone), "r"(ntiles) : "memory");
  if (old + ntiles != ntu) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");  // the decider (last arriver) sees every warp's range
  uint32_t e = 0;
  decide_unit<SRC>(p, U, u, true, false, e);  // from the symbols' max zig-zag (U.maxzz)
  *err |= e;
  if (U.codec == ZC_CODEC_FIXEDLEN && U.width == width_from_maxzz(U.wmz)) {
    write_frame_header(p, u, ZC_CODEC_FIXEDLEN, U.width, U.payload);
  } else {
    U.redo = 1;
    atomicAdd(&bglobal(us, p.nunits)->n_redo, 1u);
  }
}

template <int SRC, int kMode>
__global__ void __launch_bounds__(ET, ET_CTAS) emit_kernel(const __grid_constant__ EncParams p, const BUnit* us, BGeom g,
                                                     const __grid_constant__ CUtensorMap tmap, uint64_t ntiles,
                                                     uint64_t nfull) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  uint8_t* s_tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(s_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* my = s_tiles + static_cast<size_t>(warp) * STAGES * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_tiles + static_cast<size_t>(ET_WARPS) * STAGES * TILE_BYTES) + warp * STAGES;
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  uint32_t err = 0;
  // Launched as a programmatic dependent (mode 1 of the window profile, mode 2 of mode 1):
  // everything above ran while the previous kernel drained; units are read only after it completed.
  pdl_trigger();
  pdl_wait();
  // the redo emit has nothing to do unless a speculation missed
  if (kMode == 2 && *reinterpret_cast<const volatile uint32_t*>(&bglobal(const_cast<BUnit*>(us), p.nunits)->n_redo) == 0)
    return;

  // headers / results of every owned unit, and the capacity failures (send_batch throws)
  for (uint32_t u = blockIdx.x * ET + tid; u < p.nunits; u += gridDim.x * ET) {
    const UnitView v = unit_view_m<kMode>(p, us, u, ctx_ok);
    if (v.spec || v.codec == kForeign) continue;  // spec: the decision writes it; foreign: not ours
    if (owned(v.codec) || v.codec == CODEC_NONE) write_frame_header(p, u, v.codec, v.width, v.P);
    if (v.codec == CODEC_NONE) err |= ZC_DERR_CAPACITY;
  }

  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) tma::mbar_init(&bars[i], 1);
    tma::fence_barrier_init();
  }
  __syncwarp();

  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * ET_WARPS + warp, tw = static_cast<uint64_t>(gridDim.x) * ET_WARPS;
  const uint32_t ush = unit_tile_shift(p.unit_bytes);
  const uint64_t umask = (1ull << ush) - 1;
  // The warp's tile sequence: its contiguous share [t_beg, t_end) of the full tiles, owned units
  // only — a warp crosses at most a couple of unit boundaries, so the per-unit view (global loads
  // of the unit's plan / decision) and the speculative range flush happen a few times per warp.
  const uint64_t t_beg = nfull * gw / tw, t_end = nfull * (gw + 1) / tw;
  uint32_t iss_u = 0xffffffffu;
  bool iss_owned = false;
  auto next_tile = [&](uint64_t c) -> uint64_t {
    while (c < t_end) {
      const uint32_t u = static_cast<uint32_t>(c >> ush);
      if (u != iss_u) {
        iss_u = u;
        iss_owned = owned(unit_view_m<kMode>(p, us, u, ctx_ok).codec);
      }
      if (iss_owned) return c;
      c = static_cast<uint64_t>(u + 1) << ush;
    }
    return t_end;
  };
  uint64_t c_issue = next_tile(t_beg);
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      if (c_issue < t_end) {
        tma::mbar_arrive_expect_tx(&bars[i], TILE_BYTES);
        tma::load_2d(my + i * TILE_BYTES, &tmap, &bars[i], 0, static_cast<int32_t>(c_issue * 32));
      }
      c_issue = c_issue < t_end ? next_tile(c_issue + 1) : t_end;
    }
  } else {
    for (int i = 0; i < STAGES; ++i) c_issue = c_issue < t_end ? next_tile(c_issue + 1) : t_end;
  }
  uint32_t k = 0, cur_u = 0xffffffffu;
  UnitView v;
  uint8_t* payload = nullptr;
  const double scale = enc_scale(p), rcp = enc_rcp(p);
  const float xlim = fast_xlim(scale);
  uint64_t c_first = gw;
  {  // the processing sequence restarts from the first tile (its own unit cache)
    iss_u = 0xffffffffu;
    c_first = next_tile(t_beg);
    iss_u = 0xffffffffu;
  }
  uint32_t sp_mz = 0, sp_u = 0xffffffffu, sp_n = 0;
  auto spec_run_flush = [&]() {  // all lanes: the run's max zig-zag and tile count into the unit
    sp_mz = __reduce_max_sync(FULL, sp_mz);
    if (lane == 0) spec_flush<SRC>(p, const_cast<BUnit*>(us), sp_u, sp_mz, sp_n, &err);
    sp_mz = 0;
    sp_n = 0;
  };
  for (uint64_t c = c_first; c < t_end; c = next_tile(c + 1), ++k) {
    const uint32_t st = k % STAGES;
    tma::mbar_wait(&bars[st], (k / STAGES) & 1u);
    const uint8_t* tile = my + st * TILE_BYTES;
    const uint32_t row = tma::smem_u32(tile) + lane * 128;
    const uint32_t u = static_cast<uint32_t>(c >> ush);
    if (u != cur_u) {
      cur_u = u;
      v = unit_view_m<kMode>(p, us, u, ctx_ok);
      payload = p.stages + static_cast<uint64_t>(u) * p.stride + kHeaderBytes;
    }
    if (kMode == 1 && sp_n && sp_u != u) spec_run_flush();
    const bool spec = kMode == 1 && v.spec;  // the exact symbols' max zig-zag (non-finite inputs raised by the quantizer)
    if (spec) {
      sp_u = u;
      ++sp_n;
    }
    {
      const uint64_t row_sym = (c & umask) * TILE_ELEMS + static_cast<uint64_t>(lane) * 32;
      uint32_t* base = reinterpret_cast<uint32_t*>(payload);
      if (v.codec == ZC_CODEC_RAW) {
        emit_row<32, true, SRC>(row, lane, scale, rcp, xlim, v.big, spec, sp_mz, base + row_sym, err);
      } else {
        uint32_t* d = base + (row_sym / 32) * v.width;
        switch (v.width) {
#define ZC_ER(W)                                                                          \
  case W:                                                                                 \
    emit_row<W, false, SRC>(row, lane, scale, rcp, xlim, v.big, spec, sp_mz, d, err); \
    break;
          ZC_ER(1) ZC_ER(2) ZC_ER(3) ZC_ER(4) ZC_ER(5) ZC_ER(6) ZC_ER(7) ZC_ER(8) ZC_ER(9) ZC_ER(10) ZC_ER(11)
          ZC_ER(12) ZC_ER(13) ZC_ER(14) ZC_ER(15) ZC_ER(16) ZC_ER(17) ZC_ER(18) ZC_ER(19) ZC_ER(20) ZC_ER(21)
          ZC_ER(22) ZC_ER(23) ZC_ER(24) ZC_ER(25) ZC_ER(26) ZC_ER(27) ZC_ER(28) ZC_ER(29) ZC_ER(30) ZC_ER(31)
          ZC_ER(32)
#undef ZC_ER
          default:
            break;
        }
      }
    }
    // Refill this stage only now: the row's values have been consumed (stored), so every lane's
    // shared-memory reads of the tile have completed before the async proxy overwrites it (a
    // refill right after the loads raced them when the row work is short, e.g. RAW symbols).
    __syncwarp();
    if (lane == 0 && c_issue < t_end) {
      tma::mbar_arrive_expect_tx(&bars[st], TILE_BYTES);
      tma::load_2d(my + st * TILE_BYTES, &tmap, &bars[st], 0, static_cast<int32_t>(c_issue * 32));
    }
    c_issue = c_issue < t_end ? next_tile(c_issue + 1) : t_end;
  }

  if (kMode == 1 && sp_n) spec_run_flush();
  // the message's last, partial tile (direct guarded loads / byte-exact tail stores)
  if (nfull < ntiles && gw == tw - 1) {
    const uint64_t c = nfull;
    const uint32_t u = static_cast<uint32_t>(c >> ush);
    v = unit_view_m<kMode>(p, us, u, ctx_ok);
    if (owned(v.codec)) {
      const uint64_t R = unit_R(p, u);
      const uint64_t n = R / 4;  // symbols of the unit
      const uint64_t e0 = (c & umask) * TILE_ELEMS + static_cast<uint64_t>(lane) * 32;
      const float* src = static_cast<const float*>(p.src) + static_cast<uint64_t>(u) * (p.unit_bytes / 4);
      uint8_t* payload = p.stages + static_cast<uint64_t>(u) * p.stride + kHeaderBytes;
      uint32_t s[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        s[i] = e0 + i < n ? (SRC == SRC_F32 ? quantize_exact(__ldg(src + e0 + i), enc_scale(p), enc_rcp(p), &err)
                                            : __float_as_uint(__ldg(src + e0 + i)))
                          : 0u;
      if (kMode == 1 && v.spec) {  // the partial tile's max zig-zag (its valid elements only)
        uint32_t mz = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (e0 + i < n) mz = max(mz, zigzag32(static_cast<int32_t>(s[i])));
        mz = __reduce_max_sync(FULL, mz);
        if (lane == 0) spec_flush<SRC>(p, const_cast<BUnit*>(us), u, mz, 1u, &err);
      }
      if (v.codec == ZC_CODEC_RAW) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (e0 + i < n) reinterpret_cast<uint32_t*>(payload)[e0 + i] = s[i];
        // a raw unit of f32 source has R % 4 == 0: no partial word
      } else {
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = zigzag32(static_cast<int32_t>(s[i]));
        if (e0 < n) pack_store_w(v.width, z, payload, (e0 / 32) * v.width, v.P);
      }
    }
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}

// ------------------------------------------------------------------ decode (FixedLen / RAW -> fp32)
// recv_batch's decode dispatch (collectives.cpp:314-336) for valid FixedLen and RAW frames fused
// with dequantize_into (quant.cpp:107-127) into fp32.  Per warp, a ring of STAGES 4 KiB shared
// buffers: a 1-D bulk copy (TMA) brings a tile's packed rows (32 x W words) in, lane L reads the W
// words of row L (its 32 symbols), unpacks them with compile-time shifts, writes its 32 floats
// back into the same buffer in the 128-byte-swizzled layout, and one TMA tensor store moves the
// 4 KiB tile to HBM.  Loads run STAGES-1 tiles ahead.  Everything else (Huffman, the raw-copy
// fallback, other sinks) stays on zc_decode.cu's kernels, which skip these units.
constexpr int DT_WARPS = 16;
constexpr int DT = DT_WARPS * 32;
constexpr int DSTAGES = 3;
// Per-unit views (codec, width) cached in shared memory for the first DEC_VIEWS units: one byte
// each, 0 = not this kernel's, 33 = RAW, else the FixedLen width.
constexpr uint32_t DEC_VIEWS = 4096;
constexpr size_t DEC_SMEM = static_cast<size_t>(DT_WARPS) * DSTAGES * TILE_BYTES + 1024 + DT_WARPS * DSTAGES * 8 + DEC_VIEWS;

struct DecView {
  uint32_t codec;  // ZC_CODEC_RAW / ZC_CODEC_FIXEDLEN when this kernel owns the unit, else kFallback
  uint32_t width;  // FixedLen width; 32 for RAW (the row's words are the symbols)
};

__device__ __forceinline__ DecView dec_view(const DecParams& p, uint32_t u) {
  const uint64_t off = static_cast<uint64_t>(u) * p.unit_bytes;
  const uint64_t R = (p.total_bytes - off) < p.unit_bytes ? (p.total_bytes - off) : p.unit_bytes;
  FrameCheck fc;
  check_frame<false>(p.stages + static_cast<uint64_t>(u) * p.stride, p.frame_len ? p.frame_len[u].total_bytes : p.region,
                     R, nullptr, false, p.ctx, p.index != nullptr, fc);
  DecView v;
  v.codec = (fc.codec == ZC_CODEC_RAW || fc.codec == ZC_CODEC_FIXEDLEN) ? fc.codec : kFallback;
  v.width = fc.codec == ZC_CODEC_FIXEDLEN ? static_cast<uint32_t>(fc.h.params) : 32u;
  return v;
}

// Symbol i (0..31) of a row packed at width W (fixedlen.cpp:49-63), un-zig-zagged.
template <int W, bool kRaw>
__device__ __forceinline__ int32_t row_symbol(const uint32_t (&a)[W], int i) {
  if (kRaw) return static_cast<int32_t>(a[i]);
  const int bit = i * W, k = bit >> 5, sh = bit & 31;
  uint32_t z;
  if (sh + W <= 32) {
    z = a[k] >> sh;
  } else {
    z = __funnelshift_r(a[k], a[k + 1], sh);
  }
  constexpr uint32_t kMask = W < 32 ? (1u << (W & 31)) - 1u : 0xffffffffu;
  z &= kMask;
  return unzigzag32(z);
}

// One tile in shared memory: packed rows in, swizzled fp32 tile out (same buffer).
template <int W, bool kRaw, int OUT>
__device__ __forceinline__ void decode_tile_smem(uint32_t buf, double scale, const int32_t (&acc)[32], int lane,
                                                 uint32_t& mz, uint32_t& err) {
  uint32_t a[W];
  const uint32_t row = buf + lane * W * 4;
  if (W % 4 == 0) {
#pragma unroll
    for (int j = 0; j < W / 4; ++j)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(a[4 * j]), "=r"(a[4 * j + 1]), "=r"(a[4 * j + 2]), "=r"(a[4 * j + 3])
                   : "r"(row + 16 * j));
  } else if (W % 2 == 0) {
#pragma unroll
    for (int j = 0; j < W / 2; ++j)
      asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a[2 * j]), "=r"(a[2 * j + 1]) : "r"(row + 8 * j));
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a[j]) : "r"(row + 4 * j));
  }
  constexpr bool kAdd = OUT == OUT_ADD_I32 || OUT == OUT_ADD_Q;
  __syncwarp();  // every lane holds its row before the output overwrites the buffer
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    uint32_t o[4];
    int32_t ad[4] = {0, 0, 0, 0};
    if (kAdd) {
#pragma unroll
      for (int q = 0; q < 4; ++q) ad[q] = acc[4 * m + q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int32_t sym = row_symbol<W, kRaw>(a, 4 * m + q);
      if (OUT == OUT_F32) {
        o[q] = __float_as_uint(__double2float_rn(__dmul_rn(scale, i2d(static_cast<uint32_t>(sym)))));
      } else if (OUT == OUT_ADD_I32 || OUT == OUT_ADD_Q) {  // RS sink: int64 sum range-checked (collectives.cpp:480-491)
        const long long sum = static_cast<long long>(ad[q]) + sym;
        if (sum != static_cast<int32_t>(sum)) err |= ZC_DERR_OVERFLOW;
        o[q] = static_cast<uint32_t>(static_cast<int32_t>(sum));
        mz = max(mz, zigzag32(static_cast<int32_t>(o[q])));
      } else {
        o[q] = static_cast<uint32_t>(sym);
      }
    }
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 128 + ((m ^ (lane & 7)) << 4)), "r"(o[0]),
                 "r"(o[1]), "r"(o[2]), "r"(o[3])
                 : "memory");
  }
}

template <int OUT>
__device__ __forceinline__ void decode_tile_dispatch(const DecView& v, uint32_t buf, double scale, const int32_t (&acc)[32],
                                                     int lane, uint32_t& mz, uint32_t& err) {
  if (v.codec == ZC_CODEC_RAW) {
    decode_tile_smem<32, true, OUT>(buf, scale, acc, lane, mz, err);
    return;
  }
  switch (v.width) {
#define ZC_DC(W)                                                          \
  case W:                                                                 \
    decode_tile_smem<W, false, OUT>(buf, scale, acc, lane, mz, err); \
    break;
    ZC_DC(1) ZC_DC(2) ZC_DC(3) ZC_DC(4) ZC_DC(5) ZC_DC(6) ZC_DC(7) ZC_DC(8) ZC_DC(9) ZC_DC(10) ZC_DC(11)
    ZC_DC(12) ZC_DC(13) ZC_DC(14) ZC_DC(15) ZC_DC(16) ZC_DC(17) ZC_DC(18) ZC_DC(19) ZC_DC(20) ZC_DC(21)
    ZC_DC(22) ZC_DC(23) ZC_DC(24) ZC_DC(25) ZC_DC(26) ZC_DC(27) ZC_DC(28) ZC_DC(29) ZC_DC(30) ZC_DC(31)
    ZC_DC(32)
#undef ZC_DC
    default:
      break;
  }
}

__device__ __forceinline__ uint8_t pack_view(const DecView& v) {
  return v.codec == kFallback ? 0 : v.codec == ZC_CODEC_RAW ? 33 : static_cast<uint8_t>(v.width);
}
__device__ __forceinline__ DecView unpack_view(uint8_t b) {
  DecView v;
  v.codec = b == 0 ? kFallback : b == 33 ? ZC_CODEC_RAW : ZC_CODEC_FIXEDLEN;
  v.width = b == 33 ? 32u : b;
  return v;
}

// The reduce sinks' accumulator row of lane L (its 32 values of the local chunk): eight 16-byte
// loads in flight at once, then (ADD_Q) the fp32 values quantized with the branch-free fast path
// and, only when some value sits near a rounding tie or out of the fast range, the exact division
// out of line.  Emitted once per kernel, outside the per-width decoders.
template <int OUT>
__device__ __forceinline__ void load_acc_row(const void* accp, int lane, double scale, double rcp, int32_t (&acc)[32],
                                             uint32_t& err) {
  uint32_t b[32];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint4 v = OUT == OUT_ADD_I32 ? __ldcg(reinterpret_cast<const uint4*>(static_cast<const int32_t*>(accp) + lane * 32) + m)
                                       : __ldg(reinterpret_cast<const uint4*>(static_cast<const float*>(accp) + lane * 32) + m);
    b[4 * m] = v.x;
    b[4 * m + 1] = v.y;
    b[4 * m + 2] = v.z;
    b[4 * m + 3] = v.w;
  }
  if (OUT == OUT_ADD_I32) {
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = static_cast<int32_t>(b[i]);
    return;
  }
  bool slow = false;
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = quantize_fast(f2d_bits(b[i], slow), rcp, slow);
  if (slow) {
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = static_cast<int32_t>(quantize_exact(__uint_as_float(b[i]), scale, rcp, &err));
  }
}

struct DecSeq {  // a warp's tile sequence over owned units, with the view of the current unit
  uint64_t nfull, tw;
  uint32_t ush, cu, ch;
  DecView cv;
  const uint8_t* views;  // shared-memory view table (units < DEC_VIEWS)
  __device__ __forceinline__ uint64_t next(const DecParams& p, uint64_t c) {
    while (c < nfull) {
      const uint32_t u = static_cast<uint32_t>(c >> ush);
      if (u != cu) {
        cu = u;
        cv = u < DEC_VIEWS ? unpack_view(views[u]) : dec_view(p, u);
      }
      if (cv.codec != kFallback) return c;
      c = tile_skip_to(c, static_cast<uint64_t>(u + 1) << ush, tw, ch);
    }
    return nfull;
  }
};

template <int OUT>
__global__ void __launch_bounds__(DT, 1) fl_decode_kernel(const __grid_constant__ DecParams p,
                                                          const __grid_constant__ CUtensorMap tmap, uint64_t ntiles,
                                                          uint64_t nfull, uint32_t ch) {
  extern __shared__ __align__(1024) uint8_t s_raw[];
  pdl_trigger();  // the general decoder (its programmatic dependent) may be placed now
  uint8_t* s_tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(s_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* my = s_tiles + static_cast<size_t>(warp) * DSTAGES * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_tiles + static_cast<size_t>(DT_WARPS) * DSTAGES * TILE_BYTES) + warp * DSTAGES;
  uint8_t* views = reinterpret_cast<uint8_t*>(bars + DT_WARPS * DSTAGES - warp * DSTAGES);
  const double scale = dec_scale(p), rcp = OUT == OUT_ADD_Q ? 1.0 / scale : 0.0;
  uint32_t err = 0, mz = 0, mz_u = 0xffffffffu;
  // the sums' max zig-zag per unit (the next send's FixedLen width without a range pass)
  auto mz_flush = [&]() {
    if (OUT != OUT_ADD_I32 && OUT != OUT_ADD_Q) return;
    const uint32_t m = __reduce_max_sync(FULL, mz);
    if (lane == 0 && p.maxzz_out != nullptr && mz_u != 0xffffffffu && m) atomicMax(p.maxzz_out + mz_u, m);
    mz = 0;
  };
  // every unit's view (recv_batch's dispatch result), once per CTA; the decoded codec per owned unit
  for (uint32_t u = tid; u < p.nunits && u < DEC_VIEWS; u += DT) {
    const DecView v = dec_view(p, u);
    views[u] = pack_view(v);
    if (v.codec != kFallback && p.codec_out && u % gridDim.x == blockIdx.x) p.codec_out[u] = v.codec;
  }
  for (uint32_t u = DEC_VIEWS + blockIdx.x * DT + tid; u < p.nunits; u += gridDim.x * DT) {
    const DecView v = dec_view(p, u);
    if (v.codec != kFallback && p.codec_out) p.codec_out[u] = v.codec;
  }
  __syncthreads();
  if (lane == 0) {
    for (int i = 0; i < DSTAGES; ++i) tma::mbar_init(&bars[i], 1);
    tma::fence_barrier_init();
  }
  __syncwarp();
  const uint64_t tw = static_cast<uint64_t>(gridDim.x) * DT_WARPS;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * DT_WARPS + warp;
  const uint32_t ush = unit_tile_shift(p.unit_bytes);
  const uint64_t umask = (1ull << ush) - 1;
  DecSeq iss{nfull, tw, ush, 0xffffffffu, ch, {kFallback, 0}, views},
      prc{nfull, tw, ush, 0xffffffffu, ch, {kFallback, 0}, views};
  auto issue = [&](uint32_t st, uint64_t c) {  // lane 0: the packed rows of tile c into stage st
    const uint32_t u = static_cast<uint32_t>(c >> ush);
    const uint32_t bytes = 128u * iss.cv.width;
    const uint8_t* src = p.stages + static_cast<uint64_t>(u) * p.stride + kHeaderBytes + (c & umask) * bytes;
    tma::mbar_arrive_expect_tx(&bars[st], bytes);
    tma::load_1d(my + st * TILE_BYTES, src, bytes, &bars[st]);
    // the reduce sinks also read the tile's accumulator (the local chunk): into L2 now, so the
    // lane-row loads of the decode hit L2 instead of waiting on HBM
    if (OUT == OUT_ADD_I32) tma::prefetch_l2(static_cast<const int32_t*>(p.out) + c * TILE_ELEMS, TILE_BYTES);
    if (OUT == OUT_ADD_Q) tma::prefetch_l2(p.acc_f32 + c * TILE_ELEMS, TILE_BYTES);
  };
  uint64_t c_issue = iss.next(p, gw * ch);
  for (int i = 0; i < DSTAGES - 1; ++i) {
    if (c_issue < nfull) {
      if (lane == 0) issue(i, c_issue);
      c_issue = iss.next(p, tile_adv(c_issue, tw, ch));
    }
  }
  uint32_t k = 0;
  for (uint64_t c = prc.next(p, gw * ch); c < nfull; c = prc.next(p, tile_adv(c, tw, ch)), ++k) {
    const uint32_t st = k % DSTAGES;
    // refill the stage that tile k-1 used once its store has read the buffer (the ring keeps
    // DSTAGES-1 loads in flight while this tile is decoded)
    if (c_issue < nfull) {
      const uint32_t rs = (k + DSTAGES - 1) % DSTAGES;
      if (lane == 0) {
        tma::bulk_wait_read<0>();
        issue(rs, c_issue);
      }
      c_issue = iss.next(p, tile_adv(c_issue, tw, ch));
    }
    tma::mbar_wait(&bars[st], (k / DSTAGES) & 1u);
    const uint32_t buf = tma::smem_u32(my + st * TILE_BYTES);
    const void* acc = OUT == OUT_ADD_I32 ? static_cast<const void*>(static_cast<const int32_t*>(p.out) + c * TILE_ELEMS)
                      : OUT == OUT_ADD_Q ? static_cast<const void*>(p.acc_f32 + c * TILE_ELEMS)
                                         : nullptr;
    if (static_cast<uint32_t>(c >> ush) != mz_u) {
      mz_flush();
      mz_u = static_cast<uint32_t>(c >> ush);
    }
    int32_t ad[32];
    if (OUT == OUT_ADD_I32 || OUT == OUT_ADD_Q) load_acc_row<OUT>(acc, lane, scale, rcp, ad, err);
    decode_tile_dispatch<OUT>(prc.cv, buf, scale, ad, lane, mz, err);
    tma::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma::store_2d(&tmap, my + st * TILE_BYTES, 0, static_cast<int32_t>(c * 32));
      tma::bulk_commit();
    }
  }
  // the message's last, partial tile: symbol by symbol with byte-exact bounds
  if (nfull < ntiles && gw == (nfull / ch) % tw) {
    const uint32_t u = static_cast<uint32_t>(nfull >> ush);
    const DecView v = dec_view(p, u);
    if (u != mz_u) {
      mz_flush();
      mz_u = u;
    }
    if (v.codec != kFallback) {
      const uint64_t off = static_cast<uint64_t>(u) * p.unit_bytes;
      const uint64_t n = ((p.total_bytes - off) < p.unit_bytes ? (p.total_bytes - off) : p.unit_bytes) / 4;
      const uint8_t* payload = p.stages + static_cast<uint64_t>(u) * p.stride + kHeaderBytes;
      const uint64_t P = v.codec == ZC_CODEC_RAW ? 4 * n : packed_bytes(n, v.width);
      float* out = static_cast<float*>(p.out) + off / 4;
      const uint64_t e0 = (nfull & umask) * TILE_ELEMS + static_cast<uint64_t>(lane) * 32;
      for (uint64_t e = e0; e < e0 + 32 && e < n; ++e) {
        int32_t sym;
        if (v.codec == ZC_CODEC_RAW) {
          sym = static_cast<int32_t>(stream_word<false>(payload, P, e));
        } else {
          const uint64_t bit = e * v.width;
          const unsigned long long x = (static_cast<unsigned long long>(stream_word<false>(payload, P, bit / 32 + 1)) << 32) |
                                       stream_word<false>(payload, P, bit / 32);
          const uint32_t z = static_cast<uint32_t>((x >> (bit & 31)) & (v.width == 32 ? 0xffffffffull : ((1ull << v.width) - 1)));
          sym = unzigzag32(z);
        }
        if (OUT == OUT_F32) {
          out[e] = __double2float_rn(__dmul_rn(scale, i2d(static_cast<uint32_t>(sym))));
        } else if (OUT == OUT_ADD_I32 || OUT == OUT_ADD_Q) {
          int32_t* o = reinterpret_cast<int32_t*>(out) + e;
          const int32_t a = OUT == OUT_ADD_I32 ? *o : quantize_one(static_cast<double>(p.acc_f32[off / 4 + e]), scale, rcp, err);
          const long long sum = static_cast<long long>(a) + sym;
          if (sum != static_cast<int32_t>(sum)) err |= ZC_DERR_OVERFLOW;
          *o = static_cast<int32_t>(sum);
          mz = max(mz, zigzag32(static_cast<int32_t>(sum)));
        } else {
          reinterpret_cast<int32_t*>(out)[e] = sym;
        }
      }
    }
  }
  mz_flush();
  if (lane == 0) tma::bulk_wait<0>();
  __syncwarp();
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}


// ------------------------------------------------------------------ fused ring step (N1)
// One piece of a reduce-scatter step fused with the send of the same chunk at the next step
// (collectives.cpp:472-492 then the next exchange): every unit's tiles are first decoded from the
// predecessor's frame and reduced into the local chunk (phase A: the sums are stored, and the
// unit's max zig-zag and its 64 KiB window's max zig-zag are merged), then, once the unit's phase A
// has completed, decided (arbitrate_plan on the window, encode_best's post-check / the pin on the
// unit range) and packed from the just-written sums — still in L2 — into the successor's region
// (phase B).  Work is an ordered task queue of 8-tile groups, A(0) A(1) B(0) A(2) B(1) ... : a B
// task only waits for A tasks claimed before it by running warps, so it cannot deadlock, and a
// unit's sums are re-read right after they were written.
// Tasks are claimed per WARP (no CTA barriers); within a task the warp double-buffers its tiles
// with cp.async (the next tile's packed rows and accumulator tile load while this one is reduced).
constexpr int FT_WARPS = 4;
constexpr int FT = FT_WARPS * 32;
constexpr int FT_CTAS = 3;   // per SM: 12 warps x 16 KiB of stages
constexpr uint32_t FG = 8;   // tiles per warp task (fewer when the message does not fill the GPU)

struct FusedUnit {
  uint32_t maxzz, wmz, adone, bdone;
  uint32_t codec, width, decided, _pad;
  unsigned long long payload;
};

// Row `lane` of a tile packed at width W (or RAW) in shared memory, as 32 int32 symbols.
template <int W, bool kRaw>
__device__ __forceinline__ void decode_row(uint32_t buf, int lane, int32_t (&sym)[32]) {
  uint32_t a[W];
  const uint32_t row = buf + lane * W * 4;
#pragma unroll
  for (int j = 0; j < W; ++j) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a[j]) : "r"(row + 4 * j));
#pragma unroll
  for (int i = 0; i < 32; ++i) sym[i] = row_symbol<W, kRaw>(a, i);
}
__device__ __forceinline__ void decode_row_dispatch(uint32_t codec, uint32_t width, uint32_t buf, int lane,
                                                    int32_t (&sym)[32]) {
  if (codec == ZC_CODEC_RAW) {
    decode_row<32, true>(buf, lane, sym);
    return;
  }
  switch (width) {
#define ZC_DR(W)                              \
  case W:                                     \
    decode_row<W, false>(buf, lane, sym); \
    break;
    ZC_DR(1) ZC_DR(2) ZC_DR(3) ZC_DR(4) ZC_DR(5) ZC_DR(6) ZC_DR(7) ZC_DR(8) ZC_DR(9) ZC_DR(10) ZC_DR(11)
    ZC_DR(12) ZC_DR(13) ZC_DR(14) ZC_DR(15) ZC_DR(16) ZC_DR(17) ZC_DR(18) ZC_DR(19) ZC_DR(20) ZC_DR(21)
    ZC_DR(22) ZC_DR(23) ZC_DR(24) ZC_DR(25) ZC_DR(26) ZC_DR(27) ZC_DR(28) ZC_DR(29) ZC_DR(30) ZC_DR(31)
    ZC_DR(32)
#undef ZC_DR
    default:
      break;
  }
}

// Task t of the queue -> (phase B?, unit, group).  Units 0..U-2 have G groups, the last GL.  The
// queue runs phase B `lag` units behind phase A — A(0..lag-1), then A(i) B(i-lag), then the last B
// — with lag ~ the warps in flight / G, so a unit's phase A has (almost always) completed when its
// first B task is claimed, and its sums are still in L2.
__device__ __forceinline__ bool fused_task(uint32_t t, uint32_t U, uint32_t G, uint32_t GL, uint32_t lag, uint32_t& u,
                                           uint32_t& g) {
  auto groups = [&](uint32_t v) { return v + 1 == U ? GL : G; };
  uint32_t na = 0, nb = 0;  // next A / B unit
  for (;;) {
    const bool take_a = na < U && (na < lag || nb + lag <= na);
    const uint32_t v = take_a ? na : nb;
    const uint32_t k = groups(v);
    if (t < k) {
      u = v;
      g = t;
      return !take_a;
    }
    t -= k;
    if (take_a) ++na;
    else ++nb;
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int SINK>
__global__ void __launch_bounds__(FT, FT_CTAS) ring_fused_kernel(const __grid_constant__ FusedParams f, BUnit* us,
                                                                 FusedUnit* fu, uint32_t* task_ctr, uint32_t lag,
                                                                 uint32_t fg) {
  extern __shared__ __align__(128) uint8_t s_buf[];
  const EncParams& p = f.enc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // per warp, two stages of {the tile's packed rows, the accumulator / sums tile (swizzled rows)}
  const uint32_t wbase = tma::smem_u32(s_buf) + static_cast<uint32_t>(warp) * 4 * TILE_BYTES;
  auto pk = [&](int st) { return wbase + static_cast<uint32_t>(st) * 2 * TILE_BYTES; };
  auto ac = [&](int st) { return wbase + static_cast<uint32_t>(st) * 2 * TILE_BYTES + TILE_BYTES; };
  const uint32_t U = p.nunits;
  const uint32_t ush = unit_tile_shift(p.unit_bytes);
  const uint32_t unit_tiles = 1u << ush;
  const uint64_t lastR = p.total_bytes - static_cast<uint64_t>(U - 1) * p.unit_bytes;
  const uint32_t last_tiles = static_cast<uint32_t>((lastR / 4 + TILE_ELEMS - 1) / TILE_ELEMS);  // incl. partial
  const uint32_t G = (unit_tiles + fg - 1) / fg, GL = (last_tiles + fg - 1) / fg;
  const uint32_t ntasks = 2 * ((U - 1) * G + GL);
  const double scale = SINK == OUT_ADD_Q ? f.dscale[0] : 1.0, rcp = SINK == OUT_ADD_Q ? f.dscale[1] : 1.0;
  uint32_t err = 0;
  // a 4 KiB tile of int32 / fp32 values into swizzled rows (chunk ch of row r at r*128 + (ch ^ r&7)*16)
  auto issue_tile = [&](uint32_t dst, const void* src) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int c = lane + 32 * k, row = c >> 3, ch = c & 7;
      cp_async16(dst + row * 128 + ((ch ^ (row & 7)) << 4), static_cast<const uint8_t*>(src) + 16 * c);
    }
  };
  auto row_of = [&](uint32_t buf, uint32_t (&v)[32]) {  // lane's row of a swizzled tile
#pragma unroll
    for (int m = 0; m < 8; ++m)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[4 * m]), "=r"(v[4 * m + 1]), "=r"(v[4 * m + 2]), "=r"(v[4 * m + 3])
                   : "r"(buf + lane * 128 + ((m ^ (lane & 7)) << 4)));
  };
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(task_ctr, 1u);
    t = __shfl_sync(FULL, t, 0);
    if (t >= ntasks) break;
    uint32_t u, g;
    const bool isB = fused_task(t, U, G, GL, lag, u, g);
    const uint64_t R = unit_R(p, u);
    const uint64_t n_elem = R / 4;
    const uint32_t tiles_u = static_cast<uint32_t>((n_elem + TILE_ELEMS - 1) / TILE_ELEMS);
    const uint32_t t0 = g * fg, t1 = min(tiles_u, t0 + fg);
    const uint32_t tf1 = min(t1, static_cast<uint32_t>(n_elem / TILE_ELEMS));  // full tiles: [t0, tf1)
    const uint64_t ebase = static_cast<uint64_t>(u) * (p.unit_bytes / 4);  // unit's first element in the piece
    FusedUnit& F = fu[u];
    if (!isB) {  // ---- phase A: decode + reduce
      uint32_t icodec = 0, iw = 0;
      if (lane == 0) {
        FrameCheck fc;
        check_frame<true>(f.in_stages + static_cast<uint64_t>(u) * f.in_stride, f.in_res[u].total_bytes, R, nullptr, false,
                          nullptr, false, fc);
        icodec = fc.codec;
        iw = fc.codec == ZC_CODEC_FIXEDLEN ? static_cast<uint32_t>(fc.h.params) : 32u;
      }
      icodec = __shfl_sync(FULL, icodec, 0);
      iw = __shfl_sync(FULL, iw, 0);
      const uint8_t* payload = f.in_stages + static_cast<uint64_t>(u) * f.in_stride + kHeaderBytes;
      uint32_t mz = 0, wmz = 0;
      if (icodec != ZC_CODEC_RAW && icodec != ZC_CODEC_FIXEDLEN) {
        err |= ZC_DERR_CORRUPT;  // never from this library's encoder; the reduce cannot be replayed
      } else {
        auto issue = [&](uint32_t tl, int st) {
          const uint64_t e0 = static_cast<uint64_t>(tl) * TILE_ELEMS;
          const uint8_t* src = payload + e0 / 8 * iw;  // the tile's 128 * width packed bytes
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t i = lane + 32u * k;
            if (i < 8 * iw) cp_async16(pk(st) + 16 * i, src + 16 * i);
          }
          issue_tile(ac(st), SINK == OUT_ADD_I32 ? static_cast<const void*>(f.sum + ebase + e0)
                                                 : static_cast<const void*>(f.x + ebase + e0));
          cp_async_commit();
        };
        if (t0 < tf1) issue(t0, 0);
        for (uint32_t tl = t0; tl < tf1; ++tl) {
          const int st = (tl - t0) & 1;
          if (tl + 1 < tf1) {
            issue(tl + 1, st ^ 1);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
          __syncwarp();
          int32_t sym[32];
          decode_row_dispatch(icodec, iw, pk(st), lane, sym);
          uint32_t b[32];
          row_of(ac(st), b);
          if (SINK == OUT_ADD_Q) {  // the local fp32, quantized (fast path; exact division near a tie)
            bool slow = false;
            uint32_t q[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) q[i] = static_cast<uint32_t>(quantize_fast(f2d_bits(b[i], slow), rcp, slow));
            if (slow) {
#pragma unroll
              for (int i = 0; i < 32; ++i) q[i] = quantize_exact(__uint_as_float(b[i]), scale, rcp, &err);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) b[i] = q[i];
          }
          const bool win = static_cast<uint64_t>(tl) * TILE_BYTES < kSampleWindow;
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            uint32_t o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const long long sm = static_cast<long long>(static_cast<int32_t>(b[4 * m + q])) + sym[4 * m + q];
              if (sm != static_cast<int32_t>(sm)) err |= ZC_DERR_OVERFLOW;
              o[q] = static_cast<uint32_t>(static_cast<int32_t>(sm));
              const uint32_t z = zigzag32(static_cast<int32_t>(o[q]));
              mz = max(mz, z);
              if (win) wmz = max(wmz, z);
            }
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ac(st) + lane * 128 + ((m ^ (lane & 7)) << 4)),
                         "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3])
                         : "memory");
          }
          __syncwarp();
          int32_t* sumt = f.sum + ebase + static_cast<uint64_t>(tl) * TILE_ELEMS;
#pragma unroll
          for (int m = 0; m < 8; ++m) {  // the sums out, 512 contiguous bytes per instruction
            const int row = 4 * m + (lane >> 3), ch = lane & 7;
            uint32_t o0, o1, o2, o3;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(o0), "=r"(o1), "=r"(o2), "=r"(o3)
                         : "r"(ac(st) + row * 128 + ((ch ^ (row & 7)) << 4))
                         : "memory");
            reinterpret_cast<uint4*>(sumt + row * 32)[ch] = make_uint4(o0, o1, o2, o3);
          }
          __syncwarp();  // the stage's buffers are refilled two tiles later
        }
        if (t1 > tf1) {  // the piece's last, partial tile: element by element
          const uint64_t e0 = static_cast<uint64_t>(tf1) * TILE_ELEMS;
          const uint64_t P = icodec == ZC_CODEC_RAW ? 4 * n_elem : packed_bytes(n_elem, iw);
          for (uint64_t e = e0 + lane; e < n_elem; e += 32) {
            int32_t sy;
            if (icodec == ZC_CODEC_RAW) {
              sy = static_cast<int32_t>(stream_word<true>(payload, P, e));
            } else {
              const uint64_t bit = e * iw;
              const unsigned long long xw = (static_cast<unsigned long long>(stream_word<true>(payload, P, bit / 32 + 1)) << 32) |
                                            stream_word<true>(payload, P, bit / 32);
              sy = unzigzag32(static_cast<uint32_t>((xw >> (bit & 31)) & (iw == 32 ? 0xffffffffull : ((1ull << iw) - 1))));
            }
            const int32_t a = SINK == OUT_ADD_I32 ? f.sum[ebase + e]
                                                  : quantize_one(static_cast<double>(f.x[ebase + e]), scale, rcp, err);
            const long long sm = static_cast<long long>(a) + sy;
            if (sm != static_cast<int32_t>(sm)) err |= ZC_DERR_OVERFLOW;
            f.sum[ebase + e] = static_cast<int32_t>(sm);
            const uint32_t z = zigzag32(static_cast<int32_t>(sm));
            mz = max(mz, z);
            if (e * 4 < kSampleWindow) wmz = max(wmz, z);
          }
        }
      }
      mz = __reduce_max_sync(FULL, mz);
      wmz = __reduce_max_sync(FULL, wmz);
      if (lane == 0) {
        atomicMax(&F.maxzz, mz);
        if (wmz) atomicMax(&F.wmz, wmz);
        uint32_t old;  // acq_rel: this task's sums and ranges before its tiles count; the last sees all
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(&F.adone), "r"(t1 - t0) : "memory");
        if (old + (t1 - t0) == tiles_u) {
          // the unit's last phase-A task decides it (a pure function of the unit's ranges):
          // arbitrate_plan on the window (rea.cpp:145-176) and encode_best's post-check / the pin
          const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
          uint32_t plan = ZC_CODEC_RAW;
          if (!(R <= p.cfg.small_batch_threshold_bytes || p.stage_len <= kHeaderBytes)) {
            zc_sample_stats sst;
            sst.sampled_bytes = R < kSampleWindow ? R : kSampleWindow;
            sst.max_zigzag = __ldcg(&F.wmz);
            sst.ctx_code_len_bits = 0.0;
            sst.ctx_code_len_valid = 0u;
            sst.self_code_len_bits = 0.0;
            sst.self_code_len_valid = 0u;
            plan = arbitrate_plan(R, pcap, sst, p.hint, false, p.cfg).choice;
          }
          BUnit& L = us[u];  // decide_unit / final_codec read only the fields set here
          L.plan = plan;
          L.maxzz = __ldcg(&F.maxzz);
          L.codec = ZC_CODEC_RAW;
          L.width = 0;
          L.payload = R;
          uint32_t e = 0;
          if (target_codec(p, L, false) == ZC_CODEC_FIXEDLEN) decide_unit<SRC_BYTES>(p, L, u, true, true, e);
          err |= e;
          uint32_t codec, width;
          uint64_t P;
          final_codec(p, L, u, false, codec, width, P);
          F.codec = codec;
          F.width = width;
          F.payload = P;
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&F.decided), "r"(1u) : "memory");
        }
      }
      __syncwarp();
      continue;
    }
    // ---- phase B: pack the sums (every phase-A task of the unit was claimed before this one by a
    // running warp, and the last of them decided the unit)
    if (lane == 0) {
      for (;;) {  // relaxed polls (no L1 invalidation per poll), then the acquire below
        uint32_t d;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(&F.decided) : "memory");
        if (d) break;
        __nanosleep(64);
      }
    }
    __syncwarp();
    {
      uint32_t d;  // every lane acquires the decision (and with it the sums)
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(&F.decided) : "memory");
      (void)d;
    }
    const uint32_t codec = __ldcg(&F.codec), width = __ldcg(&F.width);
    const uint64_t P = __ldcg(&F.payload);
    uint8_t* opay = p.stages + static_cast<uint64_t>(u) * p.stride + kHeaderBytes;
    if (codec == ZC_CODEC_RAW || codec == ZC_CODEC_FIXEDLEN) {
      if (t0 < tf1) {
        issue_tile(ac(0), f.sum + ebase + static_cast<uint64_t>(t0) * TILE_ELEMS);
        cp_async_commit();
      }
      for (uint32_t tl = t0; tl < tf1; ++tl) {
        const int st = (tl - t0) & 1;
        if (tl + 1 < tf1) {
          issue_tile(ac(st ^ 1), f.sum + ebase + static_cast<uint64_t>(tl + 1) * TILE_ELEMS);
          cp_async_commit();
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        uint32_t sv[32];
        row_of(ac(st), sv);
        __syncwarp();
        store_row(codec, width, sv, opay, static_cast<uint64_t>(tl) * TILE_ELEMS + static_cast<uint64_t>(lane) * 32);
      }
      if (t1 > tf1) {  // partial tile: the lane's row, guarded
        const uint64_t e0 = static_cast<uint64_t>(tf1) * TILE_ELEMS;
        const uint64_t r0 = e0 + static_cast<uint64_t>(lane) * 32;
        const int32_t* sumt = f.sum + ebase + e0;
        uint32_t sv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) sv[i] = r0 + i < n_elem ? static_cast<uint32_t>(__ldcg(sumt + lane * 32 + i)) : 0u;
        if (codec == ZC_CODEC_RAW) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (r0 + i < n_elem) reinterpret_cast<uint32_t*>(opay)[r0 + i] = sv[i];
        } else {
          uint32_t z[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] = zigzag32(static_cast<int32_t>(sv[i]));
          if (r0 < n_elem) pack_store_w(width, z, opay, (r0 / 32) * width, P);
        }
      }
    } else if (lane == 0) {
      err |= ZC_DERR_CAPACITY;  // cannot ship even raw (collectives.cpp:278-281)
    }
    __syncwarp();
    if (lane == 0) {  // the unit's last phase-B task writes the header and the EncodeResult
      __threadfence();
      if (atomicAdd(&F.bdone, t1 - t0) + (t1 - t0) == tiles_u) write_frame_header(p, u, codec, width, P);
    }
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && f.err) atomicOr(f.err, err);
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

// The fp32 source as a [rows][32] tensor of 4 KiB tiles (32 x 32, 128-byte swizzle).
bool make_row_tensor_map(CUtensorMap* map, const void* base, uint64_t rows) {  // 4-byte elements
  static EncodeTiled fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || f == nullptr)
      return false;
    fn = reinterpret_cast<EncodeTiled>(f);
  }
  const cuuint64_t dims[2] = {32, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Units of 2^k whole tiles, up to one bank: 4 MiB batches and 512 KiB slots.
static bool tiled_unit(uint64_t ub) {
  return ub >= TILE_BYTES && ub <= ZC_BATCH_RAW_BYTES && (ub & (ub - 1)) == 0;
}

bool fixed_path_ok(const EncParams& p) {
  const bool src_ok = p.src_kind == SRC_F32 || (p.src_kind == SRC_BYTES && p.total_bytes % 4 == 0);
  return src_ok && (reinterpret_cast<uintptr_t>(p.src) & 15u) == 0 && tiled_unit(p.unit_bytes) &&
         p.mode == ENC_SEND && !p.link_tx && !p.link_rx_add && !p.cfg.embed_codebook;
}

cudaError_t launch_fixed_range_m(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                                 int mode, cudaStream_t s) {
  BGeom g{};
  g.s_full = s_full;
  g.total = total_slices;
  g.fast = 1;
  g.spec = mode == 1 ? 1u : 0u;
  note_launch();
  g.planned = mode == 3 ? 1u : 0u;
  const uint64_t tasks = (mode == 1 || (p.src_kind != SRC_F32 && p.maxzz_in != nullptr)) ? p.nunits
                         : mode == 3                                                    ? total_slices
                                                                                        : total_slices + p.nunits;
  const uint32_t grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(tasks, 2ull * sms)));
  if (p.src_kind == SRC_F32)
    range_kernel<SRC_F32><<<grid, RT, 0, s>>>(p, static_cast<BUnit*>(scratch), g);
  else
    range_kernel<SRC_BYTES><<<grid, RT, 0, s>>>(p, static_cast<BUnit*>(scratch), g);
  return cudaGetLastError();
}
cudaError_t launch_fixed_range(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                               cudaStream_t s) {
  return launch_fixed_range_m(p, scratch, total_slices, s_full, sms, 0, s);
}
static void set_emit_attrs() {
  cudaFuncSetAttribute(emit_kernel<SRC_F32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(EMIT_SMEM));
  cudaFuncSetAttribute(emit_kernel<SRC_F32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(EMIT_SMEM));
  cudaFuncSetAttribute(emit_kernel<SRC_F32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(EMIT_SMEM));
  cudaFuncSetAttribute(emit_kernel<SRC_BYTES, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(EMIT_SMEM));
}
cudaError_t launch_fixed_emit_m(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                                int mode, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    set_emit_attrs();
  }
  const uint64_t count = p.total_bytes / 4;
  const uint64_t rows = count / 32;
  // tiles of the message (the last unit's may be partial) and the full ones before it
  const uint64_t last_n = (p.total_bytes - static_cast<uint64_t>(p.nunits - 1) * p.unit_bytes) / 4;
  const uint64_t unit_tiles = p.unit_bytes / TILE_BYTES;
  const uint64_t ntiles = static_cast<uint64_t>(p.nunits - 1) * unit_tiles + (last_n + TILE_ELEMS - 1) / TILE_ELEMS;
  const uint64_t nfull = static_cast<uint64_t>(p.nunits - 1) * unit_tiles + last_n / TILE_ELEMS;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (rows > 0 && !make_row_tensor_map(&map, p.src, rows)) return cudaErrorInvalidValue;
  BGeom g{};
  g.s_full = s_full;
  g.total = total_slices;
  g.fast = 1;
  g.spec = mode == 1 ? 1u : 0u;
  const uint64_t ech = chunk_for(ntiles, static_cast<uint64_t>(ET_CTAS) * sms * ET_WARPS);  // warps' shares are contiguous
  const uint64_t want = (ntiles + ET_WARPS * ech - 1) / (ET_WARPS * ech);
  const uint32_t grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(ET_CTAS) * sms)));
  note_launch();
  const BUnit* us = static_cast<const BUnit*>(scratch);
  if (p.src_kind == SRC_F32) {
    if (mode == 1) {  // programmatic dependent launch after profile_kernel (griddepcontrol.wait inside)
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(ET);
      lc.dynamicSmemBytes = EMIT_SMEM;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      if (cudaError_t e = cudaLaunchKernelEx(&lc, emit_kernel<SRC_F32, 1>, p, us, g, map, ntiles, nfull)) return e;
    }
    else if (mode == 2)
      {
        if (cudaError_t e = launch_pdl(emit_kernel<SRC_F32, 2>, dim3(grid), dim3(ET), EMIT_SMEM, s, p, us, g, map, ntiles, nfull))
          return e;
      }
    else
      emit_kernel<SRC_F32, 0><<<grid, ET, EMIT_SMEM, s>>>(p, us, g, map, ntiles, nfull);
  } else {
    emit_kernel<SRC_BYTES, 0><<<grid, ET, EMIT_SMEM, s>>>(p, us, g, map, ntiles, nfull);
  }
  return cudaGetLastError();
}
cudaError_t launch_fixed_emit(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                              cudaStream_t s) {
  return launch_fixed_emit_m(p, scratch, total_slices, s_full, sms, 0, s);
}

bool fixed_decode_ok(const DecParams& p) {
  return !p.bare && (p.out_kind == OUT_F32 || p.out_kind == OUT_ADD_I32 || p.out_kind == OUT_ADD_Q || p.out_kind == OUT_BYTES) &&
         (p.out_kind != OUT_ADD_Q || (reinterpret_cast<uintptr_t>(p.acc_f32) & 15u) == 0) &&
         tiled_unit(p.unit_bytes) && (p.total_bytes % 4) == 0 &&
         (reinterpret_cast<uintptr_t>(p.out) & 15u) == 0 && (p.stride % 16) == 0 &&
         (reinterpret_cast<uintptr_t>(p.stages) & 15u) == 0;
}

cudaError_t launch_fixed_decode(const DecParams& p, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(fl_decode_kernel<OUT_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
    cudaFuncSetAttribute(fl_decode_kernel<OUT_BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
    cudaFuncSetAttribute(fl_decode_kernel<OUT_ADD_I32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
    cudaFuncSetAttribute(fl_decode_kernel<OUT_ADD_Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t count = p.total_bytes / 4;
  const uint64_t rows = count / 32;
  const uint64_t last_n = (p.total_bytes - static_cast<uint64_t>(p.nunits - 1) * p.unit_bytes) / 4;
  const uint64_t unit_tiles = p.unit_bytes / TILE_BYTES;
  const uint64_t ntiles = static_cast<uint64_t>(p.nunits - 1) * unit_tiles + (last_n + TILE_ELEMS - 1) / TILE_ELEMS;
  const uint64_t nfull = static_cast<uint64_t>(p.nunits - 1) * unit_tiles + last_n / TILE_ELEMS;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (rows > 0 && !make_row_tensor_map(&map, p.out, rows)) return cudaErrorInvalidValue;
  const uint32_t ch = chunk_for(ntiles, static_cast<uint64_t>(sms) * DT_WARPS);
  const uint64_t want = (ntiles + DT_WARPS * ch - 1) / (DT_WARPS * ch);
  const uint32_t grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(sms))));
  note_launch();
  if (p.out_kind == OUT_F32)
    fl_decode_kernel<OUT_F32><<<grid, DT, DEC_SMEM, s>>>(p, map, ntiles, nfull, ch);
  else if (p.out_kind == OUT_ADD_I32)
    fl_decode_kernel<OUT_ADD_I32><<<grid, DT, DEC_SMEM, s>>>(p, map, ntiles, nfull, ch);
  else if (p.out_kind == OUT_ADD_Q)
    fl_decode_kernel<OUT_ADD_Q><<<grid, DT, DEC_SMEM, s>>>(p, map, ntiles, nfull, ch);
  else
    fl_decode_kernel<OUT_BYTES><<<grid, DT, DEC_SMEM, s>>>(p, map, ntiles, nfull, ch);
  return cudaGetLastError();
}


constexpr size_t FT_SMEM = static_cast<size_t>(FT_WARPS) * 4 * TILE_BYTES;
size_t ring_fused_scratch_bytes(uint32_t nunits) {
  return sizeof(FusedUnit) * (nunits ? nunits : 1) + 256 + sizeof(BUnit) * (nunits ? nunits : 1);
}

cudaError_t launch_ring_fused(const FusedParams& f, void* scratch, cudaStream_t s) {
  if (f.enc.nunits == 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t fb = sizeof(FusedUnit) * f.enc.nunits;
  if (cudaError_t e = cudaMemsetAsync(scratch, 0, fb + 256, s)) return e;
  FusedUnit* fu = static_cast<FusedUnit*>(scratch);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + fb);
  BUnit* us = reinterpret_cast<BUnit*>(static_cast<uint8_t*>(scratch) + fb + 256);  // written before read
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(ring_fused_kernel<OUT_ADD_Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(FT_SMEM));
    cudaFuncSetAttribute(ring_fused_kernel<OUT_ADD_I32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(FT_SMEM));
  }
  const uint64_t tiles = (f.enc.total_bytes / 4 + TILE_ELEMS - 1) / TILE_ELEMS;
  uint32_t fg = FG;
  while (fg > 1 && tiles < static_cast<uint64_t>(fg) * FT_CTAS * sms * FT_WARPS) fg >>= 1;
  const uint32_t grid = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>((tiles + fg * FT_WARPS - 1) / (fg * FT_WARPS), static_cast<uint64_t>(FT_CTAS) * sms)));
  note_launch();
  const uint32_t G = static_cast<uint32_t>(((f.enc.unit_bytes / TILE_BYTES) + fg - 1) / fg);
  const uint32_t lag = static_cast<uint32_t>(std::max<uint64_t>(1, (static_cast<uint64_t>(grid) * FT_WARPS + G - 1) / G + 1));
  if (f.sink == OUT_ADD_Q)
    ring_fused_kernel<OUT_ADD_Q><<<grid, FT, FT_SMEM, s>>>(f, us, fu, ctr, lag, fg);
  else
    ring_fused_kernel<OUT_ADD_I32><<<grid, FT, FT_SMEM, s>>>(f, us, fu, ctr, lag, fg);
  return cudaGetLastError();
}

void preload_fixed_kernels() {
  cudaFuncAttributes fa;
  cudaFuncSetAttribute(ring_fused_kernel<OUT_ADD_Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(FT_SMEM));
  cudaFuncSetAttribute(ring_fused_kernel<OUT_ADD_I32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(FT_SMEM));
  cudaFuncGetAttributes(&fa, ring_fused_kernel<OUT_ADD_Q>);
  cudaFuncGetAttributes(&fa, ring_fused_kernel<OUT_ADD_I32>);
  set_emit_attrs();
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, range_kernel<SRC_F32>);
  cudaFuncGetAttributes(&a, range_kernel<SRC_BYTES>);
  cudaFuncSetAttribute(fl_decode_kernel<OUT_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
  cudaFuncSetAttribute(fl_decode_kernel<OUT_BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
  cudaFuncSetAttribute(fl_decode_kernel<OUT_ADD_I32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
  cudaFuncSetAttribute(fl_decode_kernel<OUT_ADD_Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(DEC_SMEM));
  cudaGetLastError();
}

}  // namespace zc
