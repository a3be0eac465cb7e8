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

#include "zc_batch.cuh"
#include "zc_huff_device.cuh"

namespace zc {
namespace {

// ------------------------------------------------------------------ pass 1: window profile + plan
constexpr uint32_t PC = 8;             // CTAs per unit window (64 KiB / 8 = 8 KiB each)
constexpr uint32_t PT = 256;           // threads per profile CTA: two 16-byte vectors each
constexpr uint32_t PV = ZC_SAMPLE_WINDOW_BYTES / 16 / PC;

template <int SRC>
__global__ void __launch_bounds__(PT) profile_kernel(const EncParams p, BUnit* us) {
  // the speculative emit may launch now (it waits for this grid's completion before reading units)
  asm volatile("griddepcontrol.launch_dependents;");
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
  // symbols whose per-unit max zig-zag the ring's reduce sink recorded: decided here, no range pass
  auto decide_known = [&](uint32_t& e) {
    if (SRC == SRC_BYTES && p.maxzz_in != nullptr) {
      U.maxzz = __ldcg(p.maxzz_in + u);
      if (target_codec(p, U, ctx_ok) == ZC_CODEC_FIXEDLEN) decide_unit<SRC>(p, U, u, true, true, e);
    }
  };
  if (R <= p.cfg.small_batch_threshold_bytes || p.stage_len <= kHeaderBytes) {
    if (part == 0 && tid == 0) {
      U.plan = ZC_CODEC_RAW;
      uint32_t e = 0;
      decide_known(e);
      if (e && p.err) atomicOr(p.err, e);
    }
    return;
  }
  for (int i = tid; i < 256; i += PT) {
    s_hist[i] = 0;
    s_clens[i] = ctx_ok ? p.ctx->len[i] : 0;
  }
  for (int i = tid; i < 256 * (PT / 32); i += PT) (&s_whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t W = R < kSampleWindow ? R : kSampleWindow;
  uint32_t wmz = 0, err = 0;
  RawVec rvs[PV / PT];
#pragma unroll
  for (uint32_t k = 0; k < PV / PT; ++k) {
    const uint64_t v = static_cast<uint64_t>(part) * PV + k * PT + tid;
    rvs[k].nb = 0;
    if (v * 16 < W) fetch<SRC, false>(p, uoff, R, v, rvs[k]);
  }
#pragma unroll
  for (uint32_t k = 0; k < PV / PT; ++k) {
  const uint64_t v = static_cast<uint64_t>(part) * PV + k * PT + tid;
  if (v * 16 < W) {
    const RawVec& rv = rvs[k];
    uint32_t w[4];
    if (rv.nb == 16)
      words_full<SRC>(p, rv, w, err);
    else
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
      if (U.plan == ZC_CODEC_HUFFMAN) atomicAdd(&bglobal(us, p.nunits)->n_huff, 1u);
      decide_known(err);
    }
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}

// ------------------------------------------------------------------ pass 2: ranges / bit counts, decision
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
  if (g.fast && p.pin == ZC_PIN_AUTO && *reinterpret_cast<volatile uint32_t*>(&bglobal(us, p.nunits)->n_huff) == 0) return;
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
    if (g.fast && target != ZC_CODEC_HUFFMAN) continue;                       // zc_fixed.cu's range pass
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
    if (p.index != nullptr) {
      // per 1 KiB grain (one warp, 32 bytes per lane): the grain's bit count goes to the
      // companion index slot, which huff_emit_kernel turns into the grain's start bit
      uint32_t* uindex = p.index + static_cast<uint64_t>(u) * p.index_stride;
      // GU grains per warp iteration (2*GU x 16 bytes in flight per lane, as registers allow)
      constexpr int GU = SRC == SRC_BYTES ? 4 : SRC == SRC_F32 ? 2 : 1;
      for (uint64_t gv = v0 + static_cast<uint64_t>(warp) * 64; gv < v1; gv += NT * 2 * GU) {
        RawVec rv[2 * GU];
#pragma unroll
        for (int k = 0; k < 2 * GU; ++k) {
          const uint64_t v = gv + (k >> 1) * (NT * 2) + 2 * lane + (k & 1);
          rv[k].nb = 0;
          if (v < v1) fetch<SRC, false>(p, uoff, R, v, rv[k]);
        }
        uint32_t gb[GU];
#pragma unroll
        for (int h = 0; h < GU; ++h) gb[h] = 0;
#pragma unroll
        for (int k = 0; k < 2 * GU; ++k) {
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
              gb[k >> 1] += l;
              zero |= (l == 0);
            }
          }
        }
#pragma unroll
        for (int h = 0; h < GU; ++h) {
          hb += gb[h];
          const uint32_t t2 = __reduce_add_sync(FULL, gb[h]);
          const uint64_t gh = gv + h * (NT * 2);
          if (lane == 0 && gh < v1) uindex[gh / 64] = t2;
        }
      }
    } else
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
      if (atomicAdd(g.fast ? &U.hdone : &U.scan_done, 1u) + 1 == unit_slices(p, u)) {
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
  if (g.fast && p.pin == ZC_PIN_AUTO && *reinterpret_cast<const volatile uint32_t*>(&bglobal(us, p.nunits)->n_huff) == 0) return;
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
    if (g.fast && target != ZC_CODEC_HUFFMAN) continue;  // zc_fixed.cu owns the RAW / FixedLen targets
    if (codec == ZC_CODEC_HUFFMAN && p.index != nullptr) continue;  // huff_emit_kernel
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

// ------------------------------------------------------------------ pass 3b: Huffman frames, one warp per grain
// huffman_encode (huffman.cpp:216-246) for every unit the decision made Huffman, when the companion
// index exists.  scan_kernel left each 1 KiB grain's exact bit count in its index slot; per 64 KiB
// slice the CTA turns the counts into start bits (the index proper).  A warp then encodes a grain
// on its own: two 512-byte steps, lane = 16 bytes; a warp exclusive scan of the lanes' code
// lengths gives each lane its bit offset and the lane packs its codes LSB-first into the warp's
// shared-memory tile (ATOMS.OR only on words it may share with a neighbour).  Every payload word
// has exactly one writer: the grain that starts in it.  The grain ORs in the tail bits of the
// previous grain, recomputed from that grain's last 32 bytes (32 codes >= 32 bits always cover
// the shared word), and leaves its own last partial word to the next grain (the unit's last grain
// writes it, byte-exact at the payload end).  No zeroing pass, no global atomics, no seam merge.
constexpr int HT = 1026;  // tile words per warp: a grain is <= 1024 codes x 32 bits, + shift

template <int SRC, bool kFull>
__device__ __forceinline__ void grain_codes(const EncParams& p, const RawVec& rv, const unsigned long long* s_enc,
                                            unsigned long long ev[16], uint32_t& L, uint32_t& err) {
  uint32_t w[4] = {0, 0, 0, 0};
  if (kFull || rv.nb == 16)
    words_full<SRC>(p, rv, w, err);
  else if (rv.nb)
    to_words<SRC>(p, rv, w, err);
  L = 0;
#pragma unroll
  for (uint32_t j = 0; j < 16; ++j) {
    ev[j] = (kFull || j < rv.nb) ? s_enc[byte_of(w, j)] : 0ull;
    L += static_cast<uint32_t>(ev[j] >> 32);
  }
}

// Packs one lane's codes LSB-first at tile bit `pos`.  Codes are <= 32 bits, so each code flushes
// at most one word.  Only the lane's first and last words may be shared with neighbouring lanes
// (ATOMS.OR into the zeroed tile); the words between are the lane's own (plain stores).
__device__ __forceinline__ void pack_codes(uint32_t* tile, uint32_t pos, const unsigned long long ev[16]) {
  uint32_t wi = pos >> 5, nbit = pos & 31;
  unsigned long long acc = 0;
  bool first = true;
#pragma unroll
  for (uint32_t j = 0; j < 16; ++j) {
    acc |= (ev[j] & 0xffffffffull) << nbit;
    nbit += static_cast<uint32_t>(ev[j] >> 32);
    const bool f = nbit >= 32;
    if (f && first) atomicOr(&tile[wi], static_cast<uint32_t>(acc));
    if (f && !first) tile[wi] = static_cast<uint32_t>(acc);
    first = first && !f;
    acc = f ? (acc >> 32) : acc;
    wi += f ? 1u : 0u;
    nbit -= f ? 32u : 0u;
  }
  if (nbit > 0) atomicOr(&tile[wi], static_cast<uint32_t>(acc));
}

// Codes of <= 24 bits (every context whose longest code fits): one u32 per symbol, code in the low
// 24 bits and length in the top 8, so a lane's 16 codes take 16 registers instead of 32.
template <int SRC>
__device__ __forceinline__ void grain_codes32(const EncParams& p, const RawVec& rv, const uint32_t* s_enc32, uint32_t ev[16],
                                              uint32_t& L, uint32_t& err) {
  uint32_t w[4];
  words_full<SRC>(p, rv, w, err);
  L = 0;
#pragma unroll
  for (uint32_t j = 0; j < 16; ++j) {
    ev[j] = s_enc32[__byte_perm(w[j >> 2], 0u, 0x4440u + (j & 3))];
    L += ev[j] >> 24;
  }
}

__device__ __forceinline__ void pack_codes32(uint32_t* tile, uint32_t pos, const uint32_t ev[16]) {
  uint32_t wi = pos >> 5, nbit = pos & 31;
  unsigned long long acc = 0;
  bool first = true;
#pragma unroll
  for (uint32_t j = 0; j < 16; ++j) {
    acc |= static_cast<unsigned long long>(ev[j] & 0xffffffu) << nbit;
    nbit += ev[j] >> 24;
    const bool f = nbit >= 32;
    if (f && first) atomicOr(&tile[wi], static_cast<uint32_t>(acc));
    if (f && !first) tile[wi] = static_cast<uint32_t>(acc);
    first = first && !f;
    acc = f ? (acc >> 32) : acc;
    wi += f ? 1u : 0u;
    nbit -= f ? 32u : 0u;
  }
  if (nbit > 0) atomicOr(&tile[wi], static_cast<uint32_t>(acc));
}

// grain_pack for full grains with <= 24-bit codes.
template <int SRC>
__device__ __forceinline__ void grain_pack32(const EncParams& p, const RawVec rv[2], const uint32_t* s_enc32, uint32_t* tile,
                                             uint32_t sh0, int lane, uint32_t& err) {
  uint32_t run = sh0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    uint32_t ev[16];
    uint32_t L;
    grain_codes32<SRC>(p, rv[k], s_enc32, ev, L, err);
    uint32_t x = L;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    pack_codes32(tile, run + x - L, ev);
    run += __shfl_sync(FULL, x, 31);
  }
}

template <int SRC, bool kFull>
__device__ __forceinline__ void grain_fetch(const EncParams& p, uint64_t uoff, uint64_t R, uint64_t nvec, uint64_t gv,
                                            int lane, RawVec rv[2]) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint64_t v = gv + 32 * k + lane;
    if (kFull) {
      fetch_full<SRC, false, (SRC == SRC_F32 || SRC == SRC_BYTES) ? kPolDrop : kPolNone>(p, uoff, v, rv[k]);
    } else {
      rv[k].nb = 0;
      if (v < nvec) fetch<SRC, false>(p, uoff, R, v, rv[k]);
    }
  }
}

// Encodes the two 512-byte steps of a grain into `tile` from bit sh0 on.
template <int SRC, bool kFull>
__device__ __forceinline__ void grain_pack(const EncParams& p, const RawVec rv[2], const unsigned long long* s_enc,
                                           uint32_t* tile, uint32_t sh0, int lane, uint32_t& err) {
  uint32_t run = sh0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    unsigned long long ev[16];
    uint32_t L;
    grain_codes<SRC, kFull>(p, rv[k], s_enc, ev, L, err);
    uint32_t x = L;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    pack_codes(tile, run + x - L, ev);
    run += __shfl_sync(FULL, x, 31);
  }
}

// kFused (fast fp32 / byte path with an index): the whole Huffman side of the send path in ONE
// launch — the grain counts and the unit decisions of scan_kernel, the RAW fallbacks of
// emit_kernel and the frames above — as an ordered task queue: every count task is claimed before
// any emit task, and an emit task waits (spinning) only for decisions whose count tasks are
// already held by running CTAs, so no wait can deadlock.  Auto messages with no Huffman plan exit
// at once: one launch instead of three.
template <int SRC, bool kFused>
__global__ void __launch_bounds__(NT, 2) huff_emit_kernel(const EncParams p, BUnit* us, BGeom g) {
  pdl_trigger();
  pdl_wait();  // a programmatic dependent of the FixedLen emit (the units' decisions)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ unsigned long long s_enc[256];
  __shared__ uint32_t s_enc32[256];
  __shared__ uint32_t s_start[BS / kIndexGrain + 1];
  __shared__ uint8_t s_clens[256];
  __shared__ unsigned long long s_r64[NW];
  __shared__ uint32_t s_r32[NW];
  __shared__ uint32_t s_task;
  extern __shared__ __align__(16) uint32_t s_tiles[];
  uint32_t* tile = s_tiles + warp * HT;
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  const bool fast_ok = aligned16(p.src) && (p.unit_bytes % 16) == 0;
  const bool codes24 = ctx_ok && p.ctx->max_len <= 24;
  BGlobal* gl = bglobal(us, p.nunits);
  if (g.fast && p.pin == ZC_PIN_AUTO && *reinterpret_cast<const volatile uint32_t*>(&gl->n_huff) == 0) return;
  if (!ctx_ok) return;
  for (int i = tid; i < 256; i += NT) {
    s_enc[i] = p.ctx->enc[i];
    s_enc32[i] = static_cast<uint32_t>(p.ctx->enc[i] & 0xffffffu) | (static_cast<uint32_t>(p.ctx->len[i]) << 24);
    s_clens[i] = p.ctx->len[i];
  }
  __syncthreads();
  uint32_t err = 0;
  const uint64_t T = g.total;
  for (uint64_t it = blockIdx.x;; it += gridDim.x) {
    uint64_t tsk;
    if (kFused) {
      __syncthreads();
      if (tid == 0) s_task = atomicAdd(&gl->huff_task, 1u);
      __syncthreads();
      tsk = s_task;
      if (tsk >= 2 * T) break;
    } else {
      if (it >= T) break;
      tsk = T + it;
    }
    if (tsk < T) {  // count task (fused): scan_kernel's per-grain Huffman bit counts of slice tsk
      uint32_t u, s;
      g.unit_of(tsk, p.nunits, u, s);
      BUnit& U = us[u];
      if (target_codec(p, U, ctx_ok) != ZC_CODEC_HUFFMAN) continue;
      const uint64_t R = unit_R(p, u);
      const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
      const uint64_t v0 = static_cast<uint64_t>(s) * BV;
      const uint64_t v1 = min(v0 + BV, (R + 15) / 16);
      uint32_t* uindex = p.index + static_cast<uint64_t>(u) * p.index_stride;
      uint32_t zero = 0;
      unsigned long long hb = 0;
      // every vector of the slice full, 16-byte aligned and inside whole grains: no tail checks, and
      // the slice is read with an evict-last hint (the emit task re-reads it)
      if ((SRC == SRC_F32 || SRC == SRC_BYTES) && fast_ok && ((v1 - v0) & 63) == 0 && v1 * 16 <= R) {
        uint32_t lmin = 0xffu;
        for (uint64_t gv = v0 + static_cast<uint64_t>(warp) * 64; gv < v1; gv += NT * 2) {
          RawVec rv[2];
#pragma unroll
          for (int k = 0; k < 2; ++k) fetch_full<SRC, false, kPolKeep>(p, uoff, gv + 2 * lane + k, rv[k]);
          uint32_t gb = 0;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            uint32_t w[4];
            words_full<SRC>(p, rv[k], w, err);
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
              const uint32_t l = s_clens[__byte_perm(w[j >> 2], 0u, 0x4440u + (j & 3))];
              gb += l;
              lmin = min(lmin, l);
            }
          }
          hb += gb;
          gb = __reduce_add_sync(FULL, gb);
          if (lane == 0) uindex[gv / 64] = gb;
        }
        zero = lmin == 0 ? 1u : 0u;
      } else
      for (uint64_t gv = v0 + static_cast<uint64_t>(warp) * 64; gv < v1; gv += NT * 2) {
        RawVec rv[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint64_t v = gv + 2 * lane + k;
          rv[k].nb = 0;
          if (v < v1) fetch<SRC, false>(p, uoff, R, v, rv[k]);
        }
        uint32_t gb = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
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
              gb += l;
              zero |= (l == 0);
            }
          }
        }
        hb += gb;
        gb = __reduce_add_sync(FULL, gb);
        if (lane == 0) uindex[gv / 64] = gb;
      }
      for (int o = 16; o > 0; o >>= 1) hb += __shfl_xor_sync(FULL, hb, o);
      zero = __reduce_or_sync(FULL, zero);
      if (lane == 0) {
        s_r64[warp] = hb;
        s_r32[warp] = zero;
      }
      __syncthreads();
      if (tid == 0) {
        for (int i = 1; i < NW; ++i) {
          hb += s_r64[i];
          zero |= s_r32[i];
        }
        U.part[s].bits = hb;
        U.part[s].zero = zero;
        __threadfence();
        if (atomicAdd(&U.hdone, 1u) + 1 == unit_slices(p, u)) {
          __threadfence();
          decide_unit<SRC>(p, U, u, false, fast_ok, err);
          __threadfence();
          *reinterpret_cast<volatile uint32_t*>(&U.hdec) = 1u;
        }
      }
      continue;
    }
    const uint64_t t = 2 * T - 1 - tsk;  // reverse: the count pass ended on the last units (L2-resident)
    uint32_t u, s;
    g.unit_of(t, p.nunits, u, s);
    BUnit& U = us[u];
    uint32_t codec, width;
    uint64_t P;
    if (kFused) {
      if (target_codec(p, U, ctx_ok) != ZC_CODEC_HUFFMAN) continue;
      if (tid == 0)
        while (*reinterpret_cast<const volatile uint32_t*>(&U.hdec) == 0) __nanosleep(64);
      __syncthreads();
      __threadfence();
      const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
      const uint64_t Ru = unit_R(p, u);
      width = 0;
      if (p.stage_len <= kHeaderBytes) {
        codec = CODEC_NONE;
        P = 0;
      } else {
        codec = __ldcg(&U.codec);
        P = __ldcg(&U.payload);
        if (codec == ZC_CODEC_RAW && Ru > pcap) codec = CODEC_NONE;
      }
      if (codec != ZC_CODEC_HUFFMAN) {  // emit_kernel's RAW fallback of a Huffman target (or capacity failure)
        if (codec == ZC_CODEC_RAW) {
          const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
          uint8_t* payload = p.stages + static_cast<uint64_t>(u) * p.stride + kHeaderBytes;
          const uint64_t v0 = static_cast<uint64_t>(s) * BV;
          const uint64_t v1 = min(v0 + BV, (Ru + 15) / 16);
          for (uint64_t v = v0 + tid; v < v1; v += NT) {
            RawVec rv;
            fetch<SRC, false>(p, uoff, Ru, v, rv);
            uint32_t w[4];
            if (rv.nb == 16)
              words_full<SRC>(p, rv, w, err);
            else
              to_words<SRC>(p, rv, w, err);
            uint8_t* d = payload + v * 16;
            if (rv.nb == 16 && aligned16(d)) {
              *reinterpret_cast<uint4*>(d) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {
              for (uint32_t j = 0; j < 16; ++j)
                if (j < rv.nb) d[j] = static_cast<uint8_t>(byte_of(w, j));
            }
          }
        } else if (s == 0 && tid == 0) {
          err |= ZC_DERR_CAPACITY;
        }
        if (s == 0 && tid == 0) write_frame_header(p, u, codec, 0, P);
        continue;
      }
    } else {
      final_codec(p, U, u, ctx_ok, codec, width, P);
      if (codec != ZC_CODEC_HUFFMAN) continue;
    }
    const uint64_t R = unit_R(p, u);
    const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
    const uint64_t nvec = (R + 15) / 16;
    const uint32_t ngr = static_cast<uint32_t>((R + kIndexGrain - 1) / kIndexGrain);
    const uint32_t gs0 = s * (BS / kIndexGrain);
    const uint32_t n = min(static_cast<uint32_t>(BS / kIndexGrain), ngr - gs0);
    uint8_t* payload = p.stages + static_cast<uint64_t>(u) * p.stride + kHeaderBytes;
    uint32_t* uindex = p.index + static_cast<uint64_t>(u) * p.index_stride;
    if (warp == 0) {  // grain counts -> start bits (the companion index)
      const uint32_t c0 = 2 * lane < n ? __ldcg(uindex + gs0 + 2 * lane) : 0u;
      const uint32_t c1 = 2 * lane + 1 < n ? __ldcg(uindex + gs0 + 2 * lane + 1) : 0u;
      uint32_t x = c0 + c1;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t b0 = static_cast<uint32_t>(__ldcg(&U.hbase[s])) + x - c0 - c1;
      s_start[2 * lane] = b0;
      s_start[2 * lane + 1] = b0 + c0;
      if (lane == 31) s_start[64] = b0 + c0 + c1;
      __syncwarp();
      if (2 * lane < n) uindex[gs0 + 2 * lane] = b0;
      if (2 * lane + 1 < n) uindex[gs0 + 2 * lane + 1] = b0 + c0;
    }
    __syncthreads();
#pragma unroll 1
    for (uint32_t gi = warp; gi < n; gi += NW) {
      const uint32_t gidx = gs0 + gi;
      const uint32_t B = s_start[gi], E = s_start[gi + 1];
      const uint32_t sh0 = B & 31;
      const uint32_t nw = (sh0 + (E - B) + 31) >> 5;  // tile words touched
      const bool last = gidx + 1 == ngr;
      const uint64_t gv = static_cast<uint64_t>(gidx) * 64;
      const bool full = fast_ok && (gidx + 1) * static_cast<uint64_t>(kIndexGrain) <= R;
      RawVec rv[2];
      if (full) grain_fetch<SRC, true>(p, uoff, R, nvec, gv, lane, rv);
      else grain_fetch<SRC, false>(p, uoff, R, nvec, gv, lane, rv);
      // tail bits of the previous grain in this grain's first word
      uint32_t prevtail = 0;
      if (sh0 != 0 && gidx > 0) {
        const uint64_t b = static_cast<uint64_t>(gidx) * kIndexGrain - 32 + lane;
        uint32_t byte;
        if (SRC == SRC_F32) {  // only the lane's own element: one load (4 lanes share it), one quantization
          const uint32_t u = __float_as_uint(__ldg(static_cast<const float*>(p.src) + (uoff + b) / 4));
          const uint32_t q = static_cast<uint32_t>(quantize_f32bits(u, enc_scale(p), enc_rcp(p), err));
          byte = (q >> (8 * static_cast<uint32_t>(b & 3))) & 0xFFu;
        } else {
          RawVec pv;
          fetch<SRC, false>(p, uoff, R, b / 16, pv);
          uint32_t w[4];
          if (pv.nb == 16)
            words_full<SRC>(p, pv, w, err);
          else
            to_words<SRC>(p, pv, w, err);
          byte = byte_of(w, static_cast<uint32_t>(b & 15));
        }
        const unsigned long long e = s_enc[byte];
        const uint32_t l = static_cast<uint32_t>(e >> 32), c = static_cast<uint32_t>(e);
        uint32_t x = l;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, x, o);
          if (lane >= o) x += y;
        }
        const uint32_t T = __shfl_sync(FULL, x, 31);
        // stream positions relative to W0 = B & ~31 (ints: the walk starts up to 1024 bits back)
        const int end = static_cast<int>(sh0) - static_cast<int>(T - x);
        const int start = end - static_cast<int>(l);
        uint32_t part = 0;
        if (end > 0 && l > 0) part = start >= 0 ? (c << start) : (c >> (-start));
        prevtail = __reduce_or_sync(FULL, part);
      }
      for (uint32_t i = lane; i < nw; i += 32) tile[i] = 0;
      __syncwarp();
      if (full && codes24) grain_pack32<SRC>(p, rv, s_enc32, tile, sh0, lane, err);
      else if (full) grain_pack<SRC, true>(p, rv, s_enc, tile, sh0, lane, err);
      else grain_pack<SRC, false>(p, rv, s_enc, tile, sh0, lane, err);
      __syncwarp();
      if (lane == 0 && prevtail) tile[0] |= prevtail;
      __syncwarp();
      const uint64_t wb = B >> 5;
      const uint32_t nout = last ? nw : ((sh0 + (E - B)) >> 5);
      for (uint32_t i = lane; i < nout; i += 32) store_word_safe(payload, wb + i, tile[i], P);
      __syncwarp();
    }
    if (s == 0 && tid == 0) write_frame_header(p, u, codec, width, P);
    __syncthreads();
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
}

constexpr size_t kHuffEmitSmem = sizeof(uint32_t) * NW * HT;

template <int SRC, bool kFused>
void launch_huff_emit(const EncParams& p, BUnit* us, const BGeom& g, int sms, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(huff_emit_kernel<SRC, kFused>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kHuffEmitSmem));
  }
  const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(g.total, static_cast<uint64_t>(2 * sms)));
  note_launch();
  launch_pdl(huff_emit_kernel<SRC, kFused>, dim3(grid), dim3(NT), kHuffEmitSmem, s, p, us, g);
}

template <int SRC>
cudaError_t launch_batch_t(const EncParams& p, void* scratch, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(emit_kernel<SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaMemsetAsync(scratch, 0, sizeof(BUnit) * p.nunits + sizeof(BGlobal), s);
  BUnit* us = static_cast<BUnit*>(scratch);
  BGeom g{};
  g.s_full = static_cast<uint32_t>((p.unit_bytes + BS - 1) / BS);
  const uint64_t last_R = p.total_bytes - static_cast<uint64_t>(p.nunits - 1) * p.unit_bytes;
  g.total = static_cast<uint64_t>(p.nunits - 1) * g.s_full + (last_R + BS - 1) / BS;
  g.fast = ((SRC == SRC_F32 || SRC == SRC_BYTES) && fixed_path_ok(p) && std::getenv("ZC_NO_FIXED") == nullptr) ? 1u : 0u;
  // fp32 FixedLen targets: one read of the input (speculative width, redo on a miss).  The
  // speculative emit stores a unit's payload before its decision is known, so it needs stages
  // that hold any FixedLen payload of a unit (<= the unit's raw bytes); smaller stages take the
  // two-read path, whose decision (capacity check included) precedes every store.
  g.spec = (g.fast && SRC == SRC_F32 && (p.pin == ZC_PIN_AUTO || p.pin == ZC_PIN_FIXEDLEN) &&
            p.stage_len >= kHeaderBytes + p.unit_bytes && !p.no_spec && std::getenv("ZC_NO_SPEC") == nullptr) ? 1u : 0u;
  const int fmode = g.spec ? 1 : 0;
  if (p.pin == ZC_PIN_AUTO && !g.fast) {
    note_launch();
    profile_kernel<SRC><<<p.nunits * PC, PT, 0, s>>>(p, us);
  }
  const bool ctx_ok_host = p.ctx != nullptr;  // validity is checked on the device
  const bool huff_possible = (p.pin == ZC_PIN_AUTO || p.pin == ZC_PIN_HUFFMAN) && ctx_ok_host;
  const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(g.total, static_cast<uint64_t>(sms)));
  if (g.fast) {
    // the range kernel also profiles the window and plans (Auto): no separate profile launch
    if (g.spec || (SRC == SRC_BYTES && p.maxzz_in != nullptr && (p.pin == ZC_PIN_AUTO || p.pin == ZC_PIN_FIXEDLEN))) {
      // window profiles only: the plan and the width guess (speculative fp32), or the plan and the
      // decision from the ranges the ring's reduce sink recorded
      note_launch();
      profile_kernel<SRC><<<p.nunits * PC, PT, 0, s>>>(p, us);
    } else if (p.pin == ZC_PIN_AUTO) {
      // the plans first (8 CTAs per window), then one HBM stream over the FixedLen-planned units
      // only (a window profile as a single task of the range kernel is its critical path)
      note_launch();
      profile_kernel<SRC><<<p.nunits * PC, PT, 0, s>>>(p, us);
      if (cudaError_t e = launch_fixed_range_m(p, scratch, g.total, g.s_full, sms, 3, s)) return e;
    } else if (p.pin == ZC_PIN_FIXEDLEN) {
      if (cudaError_t e = launch_fixed_range_m(p, scratch, g.total, g.s_full, sms, fmode, s)) return e;
    }
    const bool fused = huff_possible && p.index != nullptr;  // one launch for the whole Huffman side
    if (huff_possible && !fused) {
      note_launch();
      scan_kernel<SRC><<<grid, NT, 0, s>>>(p, us, g);
    }
    if (cudaError_t e = launch_fixed_emit_m(p, scratch, g.total, g.s_full, sms, fmode, s)) return e;
    if (g.spec)  // units whose decision differed from the speculated width
      if (cudaError_t e = launch_fixed_emit_m(p, scratch, g.total, g.s_full, sms, 2, s)) return e;
    if (huff_possible && !fused) {  // Huffman targets without an index, and their RAW fallbacks
      note_launch();
      emit_kernel<SRC><<<grid, NT, sizeof(Scratch), s>>>(p, us, g);
    }
    if (fused) launch_huff_emit<SRC, true>(p, us, g, sms, s);
    return cudaGetLastError();
  }
  if (p.pin == ZC_PIN_AUTO || p.pin == ZC_PIN_FIXEDLEN || (p.pin == ZC_PIN_HUFFMAN && ctx_ok_host)) {
    note_launch();
    scan_kernel<SRC><<<grid, NT, 0, s>>>(p, us, g);
  }
  note_launch();
  emit_kernel<SRC><<<grid, NT, sizeof(Scratch), s>>>(p, us, g);
  if (huff_possible && p.index != nullptr) launch_huff_emit<SRC, false>(p, us, g, sms, s);
  return cudaGetLastError();
}

}  // namespace

size_t batch_scratch_bytes(uint32_t nunits) { return sizeof(BUnit) * (nunits ? nunits : 1) + sizeof(BGlobal); }

void preload_batch_kernels() {
  cudaFuncSetAttribute(emit_kernel<SRC_BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncSetAttribute(emit_kernel<SRC_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncSetAttribute(emit_kernel<SRC_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncSetAttribute(huff_emit_kernel<SRC_BYTES, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kHuffEmitSmem));
  cudaFuncSetAttribute(huff_emit_kernel<SRC_F32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kHuffEmitSmem));
  cudaFuncSetAttribute(huff_emit_kernel<SRC_F64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kHuffEmitSmem));
  cudaFuncSetAttribute(huff_emit_kernel<SRC_BYTES, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kHuffEmitSmem));
  cudaFuncSetAttribute(huff_emit_kernel<SRC_F32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kHuffEmitSmem));
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
