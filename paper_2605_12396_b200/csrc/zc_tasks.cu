// zc_tasks.cu — the batched encode hot path (send_encoded over a whole message, collectives.cpp:
// 201-302 per 4 MiB batch) as ONE persistent, cluster-free kernel on every SM.
//
// Reference path (relative to /root/reference/proj/core/): encode_best (rea.cpp:178-238) /
// send_batch pin dispatch (collectives.cpp:213-281) -> profile_sample (rea.cpp:93-118) ->
// arbitrate_plan (rea.cpp:145-176) -> fixedlen_encode (fixedlen.cpp:15-37) / huffman_encode
// (huffman.cpp:216-246) -> write_header (frame.cpp:35-45); optional fused eb_quantize_chunk
// (quant.cpp:54-62).
//
// Every unit (frame) is cut into S = 16 slices; each slice is one task, in two parts:
//   scan(u, s)    one streaming pass over slice s: value range (or zig-zag max), the 64 KiB
//                 profile window's histogram, Huffman bit counts when Huffman is pinned.  The CTA
//                 that completes the unit's last scan runs the bit-exact selector and publishes
//                 the unit's decision (release store).
//   encode(u, s)  acquires the decision and materialises slice s of the frame (FixedLen: the
//                 lane-centric packer; RAW: copy; Huffman: tile encoder at the slice's bit offset,
//                 boundary words merged by the unit's last encode task).
// CTAs claim slices in order from a global counter and run scan(k) then encode(k') where k' is the
// slice the same CTA scanned one claim earlier: the unit's other slices were claimed around the
// same time, so its decision is normally ready, and k' was read ~one task ago (~148 x 256 KiB),
// so the re-read hits the 126 MB L2.  Scans never wait; an encode waits only for scans (and, for
// an auto-selected Huffman unit, for the unit's other encodes' bit counts, which every CTA reaches
// after at most one more scan), so progress needs no co-scheduling.  No cluster barriers: load
// balance is dynamic.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "zc_encode_common.cuh"

namespace zc {
namespace {

constexpr uint32_t S = 16;  // slices (tasks) per unit: 256 KiB of fp32 per 4 MiB batch

struct Part {  // per (unit, slice) scan results
  float fmn, fmx;
  double dmn, dmx;
  uint32_t absbits, bad, maxzz, wmaxzz, zero, _p;
  unsigned long long bits;
};

struct Dec {  // per unit decision
  uint32_t codec, width, pending, dirty;
  unsigned long long payload;
  unsigned long long slice_base[S];
};

struct UnitState {  // per unit, zeroed before every launch
  Part part[S];
  uint32_t hist[256];
  Dec dec;
  unsigned long long hbits[S];
  unsigned long long head_idx[S], tail_idx[S];
  uint32_t head_val[S], tail_val[S], has_head[S], has_tail[S];
  uint32_t scan_done, ready, hdone, edone;
  uint32_t hzero[S];
};

struct TaskHdr {
  unsigned long long next_task;
#ifdef ZC_TASK_TRACE
  unsigned long long tr[8];  // wait, scan, encode, decision ns; ctas done
#endif
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int SRC>
__global__ void __launch_bounds__(NT, 1) task_kernel(const EncParams p, UnitState* us, TaskHdr* th) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t s_hist[256];
  __shared__ unsigned long long s_enc[256];
  __shared__ uint8_t s_clens[256];
  __shared__ zc_sample_stats s_st;
  __shared__ unsigned long long s_red[NW];
  __shared__ double s_redd[NW];
  __shared__ uint32_t s_red32[NW];
  __shared__ unsigned long long s_task;
  __shared__ uint32_t s_last;
  __shared__ Dec s_dec;
  extern __shared__ __align__(16) uint8_t s_dyn[];
  Scratch& s_x = *reinterpret_cast<Scratch*>(s_dyn);

  constexpr bool kFloat = SRC != SRC_BYTES;
  const bool autolike = p.pin == ZC_PIN_AUTO;
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  for (int i = tid; i < 256; i += NT) {
    s_clens[i] = ctx_ok ? p.ctx->len[i] : 0;
    s_enc[i] = ctx_ok ? p.ctx->enc[i] : 0ull;
  }
  const bool fast_ok = aligned16(p.src) && (p.unit_bytes % 16) == 0;
  const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
  const bool stage_ok = p.stage_len > kHeaderBytes;
  const uint64_t total_tasks = static_cast<uint64_t>(p.nunits) * S;
  uint32_t err = 0;

  // Software pipeline per CTA: scan the slice just claimed, then encode the slice this CTA scanned
  // one iteration earlier — the rest of that unit was claimed at about the same time (decision
  // ready) and its input was read one task ago (still in L2).
  uint64_t prev = ~0ull;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_task = atomicAdd(&th->next_task, 1ull);
    __syncthreads();
    const uint64_t t_claim = s_task;
    const bool have = t_claim < total_tasks;
    for (int phase = 0; phase < 2; ++phase) {
    __syncthreads();
    if (phase == 0 && !have) continue;
    if (phase == 1 && prev == ~0ull) continue;
    const bool is_enc = phase == 1;
#ifdef ZC_TASK_TRACE
    const unsigned long long tph0 = globaltimer();
    struct PhaseEnd {
      TaskHdr* th; int tid; bool enc; unsigned long long t0;
      __device__ ~PhaseEnd() { if (tid == 0) atomicAdd(&th->tr[enc ? 2 : 1], globaltimer() - t0); }
    } phase_end{th, tid, is_enc, tph0};
#endif
    const uint64_t t = is_enc ? prev : t_claim;
    const uint32_t u = static_cast<uint32_t>(t / S), s = static_cast<uint32_t>(t % S);
    UnitState& U = us[u];
    const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
    const uint64_t R = (p.total_bytes - uoff) < p.unit_bytes ? (p.total_bytes - uoff) : p.unit_bytes;
    uint64_t v0, v1;
    unit_slice_n(R, s, S, v0, v1);
    const uint64_t W = R < kSampleWindow ? R : kSampleWindow;
    const bool small = autolike && R <= p.cfg.small_batch_threshold_bytes;
    const bool need_profile = autolike && !small;
    const bool need_maxzz = need_profile || p.pin == ZC_PIN_FIXEDLEN;
    const bool p1_hbits = p.pin == ZC_PIN_HUFFMAN && ctx_ok;
    const bool need_syms = p1_hbits;
    uint8_t* stage = p.stages + static_cast<uint64_t>(u) * p.stride;
    uint8_t* payload = stage + kHeaderBytes;
    uint32_t* uindex = p.index ? p.index + static_cast<uint64_t>(u) * p.index_stride : nullptr;

    if (!is_enc) {
      // ================================================================ scan(u, s)
      for (int i = tid; i < 256; i += NT) s_hist[i] = 0;
      __syncthreads();
      uint32_t mz = 0, wmz = 0, zero = 0;
      Range rg;
      unsigned long long hb = 0;
      const uint64_t vfull = min(v1, R / 16);
      const bool bulk = fast_ok && !need_syms && need_maxzz;
      const uint64_t wvec = need_profile ? (W + 15) / 16 : 0;
      // Bulk pass: min/max over the whole slice.  Generic pass: the whole slice when not bulk, else
      // this slice's 1/S share of the unit's profile window (histogram + window zig-zag max), so
      // the window never serialises one scanner while the other slices' encodes wait on it.
      uint64_t gbeg = v0, gend = v1;
      if (bulk) {
        const uint64_t wper = ((wvec + 32 * S - 1) / (32 * S)) * 32;
        gbeg = min(wvec, wper * s);
        gend = min(wvec, wper * (s + 1));
      }
      const bool any_work = stage_ok && (need_maxzz || need_profile || p1_hbits);
      if (any_work && bulk) {
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
      }
      if (any_work) {
        constexpr int UN = 4;
        for (uint64_t base = gbeg + static_cast<uint64_t>(warp) * 32; base < gend; base += NT * UN) {
          RawVec rv[UN];
#pragma unroll
          for (int k = 0; k < UN; ++k) {
            const uint64_t v = base + static_cast<uint64_t>(k) * NT + lane;
            if (v < gend) fetch<SRC, false>(p, uoff, R, v, rv[k]);
          }
#pragma unroll
          for (int k = 0; k < UN; ++k) {
            const uint64_t v = base + static_cast<uint64_t>(k) * NT + lane;
            const bool act = v < gend;
            const bool inwin = need_profile && act && v * 16 < W;
            uint32_t w[4] = {0, 0, 0, 0}, nb = act ? rv[k].nb : 0;
            if (kFloat && !need_syms) {
              if (act) minmax_vec<SRC>(rv[k], rg);
              if (inwin) to_words<SRC>(p, rv[k], w, err);
            } else if (act) {
              to_words<SRC>(p, rv[k], w, err);
            }
            const uint32_t nwhole = nb >> 2;
            if (need_maxzz && (!kFloat || need_syms)) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (static_cast<uint32_t>(q) < nwhole) mz = max(mz, zigzag32(static_cast<int32_t>(w[q])));
            }
            if (need_profile && __any_sync(FULL, inwin)) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (inwin && v * 16 + 4 * q + 4 <= W) wmz = max(wmz, zigzag32(static_cast<int32_t>(w[q])));
#pragma unroll
              for (uint32_t j = 0; j < 16; ++j) {
                const bool in = inwin && j < nb && v * 16 + j < W;
                const uint32_t key = in ? byte_of(w, j) : 256u + lane;
                const uint32_t peers = __match_any_sync(FULL, key);
                if (in && lane == __ffs(peers) - 1) atomicAdd(&s_hist[key], __popc(peers));
              }
            }
            if (p1_hbits && act) {
#pragma unroll
              for (uint32_t j = 0; j < 16; ++j) {
                if (j < nb) {
                  uint32_t l = static_cast<uint32_t>(s_enc[byte_of(w, j)] >> 32);
                  hb += l;
                  zero |= (l == 0);
                }
              }
            }
          }
        }
      }
      // slice partials -> global
      {
        if (SRC == SRC_F32) {
          rg.bad = rg.absbits >= 0x7f800000u ? 1u : 0u;
          rg.dmn = rg.fmn;
          rg.dmx = rg.fmx;
        }
        const uint32_t r1 = block_reduce_max(mz, s_red32);
        const uint32_t r2 = block_reduce_max(wmz, s_red32);
        const uint32_t r3 = block_reduce_max(zero, s_red32);
        const uint32_t r5 = block_reduce_max(rg.bad, s_red32);
        const unsigned long long r4 = block_reduce_sum(hb, s_red);
        const double mn = block_reduce_fmin(rg.dmn, s_redd), mx = block_reduce_fmax(rg.dmx, s_redd);
        if (tid == 0) {
          Part& pt = U.part[s];
          pt.maxzz = r1;
          pt.wmaxzz = r2;
          pt.zero = r3;
          pt.bad = r5;
          pt.bits = r4;
          pt.dmn = mn;
          pt.dmx = mx;
        }
        if (need_profile && gbeg < gend && gbeg * 16 < W)
          for (int i = tid; i < 256; i += NT)
            if (s_hist[i]) atomicAdd(&U.hist[i], s_hist[i]);
        __threadfence();
        __syncthreads();
        if (tid == 0) s_last = atomicAdd(&U.scan_done, 1u) == S - 1 ? 1u : 0u;
        __syncthreads();
      }
      if (!s_last) continue;
      // ---------------- the unit's last scan: decision (bit-exact selector, zc_common.cuh)
      __threadfence();
      for (int i = tid; i < 256; i += NT) s_hist[i] = __ldcg(&U.hist[i]);
      __syncthreads();
      if (need_profile && warp == 0) {
        uint32_t wmaxzz = 0;
        for (uint32_t r = 0; r < S; ++r) wmaxzz = max(wmaxzz, __ldcg(&U.part[r].wmaxzz));
        double el = 0.0;
        const bool v = ctx_ok && warp_mean_len(s_hist, s_clens, el);
        if (lane == 0) {
          s_st.sampled_bytes = W;
          s_st.max_zigzag = wmaxzz;
          s_st.ctx_code_len_bits = v ? el : 0.0;
          s_st.ctx_code_len_valid = v ? 1u : 0u;
          s_st.self_code_len_bits = 0.0;
          s_st.self_code_len_valid = 0u;  // only read with embedded codebooks (not on this path)
        }
      }
      if (need_profile)
        for (int i = tid; i < 256; i += NT) s_st.hist[i] = s_hist[i];
      __syncthreads();
      if (p.stats != nullptr && need_profile) {
        zc_sample_stats* o = p.stats + u;
        for (int i = tid; i < 256; i += NT) o->hist[i] = s_st.hist[i];
        if (tid == 0) {
          o->sampled_bytes = s_st.sampled_bytes;
          o->max_zigzag = s_st.max_zigzag;
          o->ctx_code_len_bits = s_st.ctx_code_len_bits;
          o->self_code_len_bits = s_st.self_code_len_bits;
          o->ctx_code_len_valid = s_st.ctx_code_len_valid;
          o->self_code_len_valid = s_st.self_code_len_valid;
        }
      }
      if (tid == 0) {
        uint32_t maxzz = 0, zl = 0, gbad = 0;
        double gmn = __builtin_huge_val(), gmx = -__builtin_huge_val();
        unsigned long long bits = 0;
        Dec d;
        for (uint32_t r = 0; r < S; ++r) {
          const Part& pt = U.part[r];
          maxzz = max(maxzz, __ldcg(&pt.maxzz));
          zl |= __ldcg(&pt.zero);
          gbad |= __ldcg(&pt.bad);
          gmn = fmin(gmn, __ldcg(&pt.dmn));
          gmx = fmax(gmx, __ldcg(&pt.dmx));
          d.slice_base[r] = bits;
          bits += __ldcg(&pt.bits);
        }
        d.dirty = (kFloat && (!need_maxzz || need_syms || gbad)) ? 1u : 0u;
        if (kFloat && gbad) err |= ZC_DERR_NONFINITE;
        if (kFloat && !need_syms && need_maxzz && R >= 4 && !gbad) {
          const int32_t smax = quantize_one(gmx, p.scale, p.rcp, err);
          const int32_t smin = quantize_one(gmn, p.scale, p.rcp, err);
          maxzz = max(zigzag32(smax), zigzag32(smin));
        }
        uint32_t codec = ZC_CODEC_RAW, width = 0, pending = 0;
        unsigned long long payload_b = R;
        if (!stage_ok) {
          codec = CODEC_NONE;
          err |= ZC_DERR_CAPACITY;
        } else {
          if (autolike) {
            if (!small) {
              const zc_arbitration_plan plan = arbitrate_plan(R, pcap, s_st, p.hint, ctx_ok, p.cfg);
              if (plan.choice == ZC_CODEC_FIXEDLEN) {
                width = width_from_maxzz(maxzz);
                const unsigned long long pay = packed_bytes(R / 4, width);
                if (pay > 0 && pay <= pcap && gain_ok(R, pay, p.cfg.min_gain_permil)) {
                  codec = ZC_CODEC_FIXEDLEN;
                  payload_b = pay;
                }
              } else if (plan.choice == ZC_CODEC_HUFFMAN) {
                pending = 1;
              }
            }
          } else if (p.pin == ZC_PIN_FIXEDLEN) {
            if (R >= 4 && R % 4 == 0) {
              width = width_from_maxzz(maxzz);
              const unsigned long long pay = packed_bytes(R / 4, width);
              if (pay > 0 && pay <= pcap) {
                codec = ZC_CODEC_FIXEDLEN;
                payload_b = pay;
              }
            }
          } else if (p.pin == ZC_PIN_HUFFMAN && ctx_ok) {
            const unsigned long long bytes = (bits + 7) / 8;
            if (!zl && bytes > 0 && bytes <= pcap) {
              codec = ZC_CODEC_HUFFMAN;
              payload_b = bytes;
            }
          }
          if (codec == ZC_CODEC_RAW && !pending && R > pcap) {
            codec = CODEC_NONE;
            err |= ZC_DERR_CAPACITY;
          }
        }
        d.codec = codec;
        d.width = width;
        d.pending = pending;
        d.payload = payload_b;
        U.dec = d;
        __threadfence();
        st_release_gpu(&U.ready, 1u);
      }
      continue;
    }

    // ================================================================ encode(u, s)
    if (tid == 0) {
#ifdef ZC_TASK_TRACE
      const unsigned long long tw0 = globaltimer();
#endif
      while (ld_acquire_gpu(&U.ready) == 0) __nanosleep(64);
#ifdef ZC_TASK_TRACE
      atomicAdd(&th->tr[0], globaltimer() - tw0);
#endif
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&U.dec);
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s_dec);
      for (uint32_t i = 0; i < sizeof(Dec) / 8; ++i) dst[i] = __ldcg(src + i);
    }
    __syncthreads();
    uint32_t codec = s_dec.codec;
    const uint32_t width = s_dec.width;
    unsigned long long P = s_dec.payload;
    unsigned long long base_bits = s_dec.slice_base[s];

    if (s_dec.pending) {
      // auto-selected Huffman: count this slice's bits, then wait for every slice of the unit
      unsigned long long b = 0;
      uint32_t z = 0;
      for (uint64_t base = v0 + static_cast<uint64_t>(warp) * 32; base < v1; base += NT) {
        const uint64_t v = base + lane;
        if (v < v1) {
          RawVec rv;
          fetch<SRC, false>(p, uoff, R, v, rv);
          uint32_t w[4];
          to_words<SRC>(p, rv, w, err);
#pragma unroll
          for (uint32_t j = 0; j < 16; ++j) {
            if (j < rv.nb) {
              const uint32_t l = static_cast<uint32_t>(s_enc[byte_of(w, j)] >> 32);
              b += l;
              z |= (l == 0);
            }
          }
        }
      }
      const unsigned long long tb = block_reduce_sum(b, s_red);
      const uint32_t tz = block_reduce_max(z, s_red32);
      if (tid == 0) {
        U.hbits[s] = tb;
        U.hzero[s] = tz;
        __threadfence();
        atomicAdd(&U.hdone, 1u);
        while (ld_acquire_gpu(&U.hdone) < S) __nanosleep(64);
        unsigned long long bits = 0, mine = 0;
        uint32_t zl = 0;
        for (uint32_t r = 0; r < S; ++r) {
          if (r == s) mine = bits;
          bits += __ldcg(&U.hbits[r]);
          zl |= __ldcg(&U.hzero[r]);
        }
        const unsigned long long bytes = (bits + 7) / 8;
        const bool ok = !zl && bytes > 0 && bytes <= pcap && gain_ok(R, bytes, p.cfg.min_gain_permil);
        s_dec.codec = ok ? ZC_CODEC_HUFFMAN : (R <= pcap ? ZC_CODEC_RAW : CODEC_NONE);
        s_dec.payload = ok ? bytes : R;
        s_dec.slice_base[s] = mine;
        if (!ok && R > pcap) err |= ZC_DERR_CAPACITY;
      }
      __syncthreads();
      codec = s_dec.codec;
      P = s_dec.payload;
      base_bits = s_dec.slice_base[s];
    }

    if (codec == ZC_CODEC_RAW) {
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
      const bool fast = fast_ok && !s_dec.dirty;
      const uint64_t vfull = min(v1, R / 16);
      for (uint64_t base = v0 + static_cast<uint64_t>(warp) * 256; base < v1; base += static_cast<uint64_t>(NW) * 256) {
        if (fast && base + 256 <= vfull) {
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
        const uint64_t wb = (base / 8 + lane) * width;
        if ((base + 8 * lane) < v1) pack_store_w(width, z, payload, wb, P);
      }
    } else if (codec == ZC_CODEC_HUFFMAN) {
      uint32_t* tile = s_x.tile;
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
        const bool has_tail = v0 < v1 && end_mod != 0;
        U.has_tail[s] = has_tail ? 1u : 0u;
        U.tail_idx[s] = base_bits >> 5;
        U.tail_val[s] = tile[0];
        __threadfence();
        s_last = atomicAdd(&U.edone, 1u) == S - 1 ? 1u : 0u;
        if (s_last) {
          __threadfence();
          unsigned long long cur_idx = ~0ull;
          uint32_t cur = 0;
          for (uint32_t r = 0; r < S; ++r) {
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
    }
    // header + result: slice 0 (its decision is the unit's)
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
    }  // phase
    if (!have) break;
    prev = t_claim;
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
#ifdef ZC_TASK_TRACE
  if (tid == 0 && atomicAdd(&th->tr[4], 1ull) == gridDim.x - 1) {
    __threadfence();
    printf("trace pin=%d ctas=%u wait=%.1fus scan=%.1fus enc=%.1fus (sum over ctas; per cta: %.1f %.1f %.1f)\n", p.pin, gridDim.x,
           th->tr[0] * 1e-3, th->tr[1] * 1e-3, th->tr[2] * 1e-3, th->tr[0] * 1e-3 / gridDim.x,
           th->tr[1] * 1e-3 / gridDim.x, th->tr[2] * 1e-3 / gridDim.x);
  }
#endif
}

template <int SRC>
cudaError_t launch_tasks_t(const EncParams& p, void* scratch, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(task_kernel<SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static_assert(sizeof(TaskHdr) <= 256, "task header must fit its slot");
  cudaMemsetAsync(scratch, 0, 256 + sizeof(UnitState) * p.nunits, s);
  TaskHdr* th = static_cast<TaskHdr*>(scratch);
  UnitState* us = reinterpret_cast<UnitState*>(static_cast<uint8_t*>(scratch) + 256);
  const uint32_t ctas = std::min<uint64_t>(static_cast<uint64_t>(sms), static_cast<uint64_t>(p.nunits) * S);
  note_launch();
  task_kernel<SRC><<<ctas, NT, sizeof(Scratch), s>>>(p, us, th);
  return cudaGetLastError();
}

}  // namespace

size_t task_scratch_bytes(uint32_t nunits) { return 256 + sizeof(UnitState) * nunits; }

void preload_task_kernels() {
  cudaFuncSetAttribute(task_kernel<SRC_BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncSetAttribute(task_kernel<SRC_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaFuncSetAttribute(task_kernel<SRC_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sizeof(Scratch)));
  cudaGetLastError();
}

cudaError_t launch_encode_tasks(const EncParams& p, void* scratch, cudaStream_t s) {
  if (p.nunits == 0) return cudaSuccess;
  switch (p.src_kind) {
    case SRC_F32:
      return launch_tasks_t<SRC_F32>(p, scratch, s);
    case SRC_F64:
      return launch_tasks_t<SRC_F64>(p, scratch, s);
    default:
      return launch_tasks_t<SRC_BYTES>(p, scratch, s);
  }
}

}  // namespace zc
