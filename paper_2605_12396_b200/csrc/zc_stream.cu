// zc_stream.cu — the batched send-path encoder (send_encoded over a whole message,
// collectives.cpp:201-302 per 4 MiB batch) as ONE persistent kernel whose input is read from HBM
// exactly once: 64 KiB slices are bulk-copied (TMA, cp.async.bulk) into a ring of shared-memory
// buffers, quantized there in place, and encoded from shared memory once the unit's decision is
// known.
//
// Reference path (relative to /root/reference/proj/core/): encode_best (rea.cpp:178-238) /
// send_batch pin dispatch (collectives.cpp:213-281) -> profile_sample (rea.cpp:93-118) ->
// arbitrate_plan (rea.cpp:145-176) -> fixedlen_encode (fixedlen.cpp:15-37) / huffman_encode
// (huffman.cpp:216-246) / frame_commit_raw (frame.cpp:71-81) -> write_header (frame.cpp:35-45);
// fused eb_quantize_chunk (quant.cpp:43-62) for fp32 sources.
//
// Units (4 MiB frames) are cut into S = 64 slices of 64 KiB; slice 0 is exactly the profile
// window (rea.hpp:16).  Each CTA (one per SM) claims slices in global order and pipelines them
// through NB = 3 buffers:
//   claim k+2 -> TMA load into the freed buffer      (two loads in flight per SM)
//   scan(k)     quantize in place (fp32 -> int32 symbols), exact max zig-zag, Huffman bit count
//               under the shared code, the window histogram (slice 0); the unit's last scanner
//               runs the bit-exact selector and publishes the decision (release store)
//   encode(k-1) materialise the slice from shared memory: RAW copy, FixedLen lane-centric packing
//               through an in-place swizzled transpose, or Huffman tiles at the slice's exact bit
//               offset (the unit's bit counts are known at decision time, so no pending phase)
// A CTA about to wait for a decision first scans its own next claim when that claim belongs to
// the same unit, so a unit's scans never wait behind one of its own encodes (no deadlock).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "zc_encode_common.cuh"
#include "zc_huff_device.cuh"

namespace zc {
namespace {

constexpr uint32_t SB = 65536;                    // slice: raw symbol bytes
constexpr uint32_t SV = SB / 16;                  // 16-byte vectors per slice
constexpr uint32_t NB = 3;                        // shared-memory slice buffers
constexpr uint32_t SMAX = ZC_BATCH_RAW_BYTES / SB;  // slices per full 4 MiB unit
constexpr uint32_t HT_WORDS = NT * 16 / 2 + 64;   // Huffman tile (codes <= 16 bits at NT vectors)

struct SPart {
  uint32_t maxzz, zero;
  unsigned long long bits;
};

struct SDec {
  uint32_t codec, width;
  unsigned long long payload;
};

struct SUnit {  // per unit, zeroed before every launch
  SPart part[SMAX];
  uint32_t hist[256];
  unsigned long long hbase[SMAX];
  unsigned long long head_idx[SMAX], tail_idx[SMAX];
  uint32_t head_val[SMAX], tail_val[SMAX], has_head[SMAX], has_tail[SMAX];
  SDec dec;
  uint32_t scan_done, ready, edone, _p;
};

struct SHdr {
  unsigned long long next;
#ifdef ZC_TASK_TRACE
  unsigned long long tr[8];  // load wait, scan, decision wait, encode, decide ns; ctas done
#endif
};

struct SmemStream {
  uint4 buf[NB][SV];
  uint32_t tile[HT_WORDS];
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(m)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}

// XOR swizzle of 16-byte slots inside one warp's 4 KiB chunk: lane-centric reads (slot 8*l + m)
// and lane-consecutive writes (slot 32*j + l) are both bank-conflict free.
__device__ __forceinline__ uint32_t swz(uint32_t slot) { return slot ^ ((slot >> 3) & 7u); }

template <int SRC>
__global__ void __launch_bounds__(NT, 1) stream_kernel(const EncParams p, SUnit* us, SHdr* th, uint32_t s_full,
                                                       uint64_t total) {
  static_assert(SRC == SRC_F32 || SRC == SRC_BYTES, "stream encoder: fp32 or symbol bytes");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ uint32_t s_hist[256];
  __shared__ unsigned long long s_enc[256];
  __shared__ uint8_t s_clens[256];
  __shared__ unsigned long long s_red[NW];
  __shared__ uint32_t s_red32[NW];
  __shared__ __align__(8) uint64_t s_mbar[NB];
  __shared__ unsigned long long s_claim[NB];
  __shared__ uint32_t s_scanned[NB];
  __shared__ uint32_t s_flag, s_pre;
  __shared__ SDec s_dec;
  extern __shared__ __align__(128) uint8_t s_dyn[];
  SmemStream& sm = *reinterpret_cast<SmemStream*>(s_dyn);

  constexpr bool kFloat = SRC == SRC_F32;
  const bool autolike = p.pin == ZC_PIN_AUTO;
  const bool ctx_ok = p.ctx != nullptr && p.ctx->valid != 0;
  const bool need_hbits = ctx_ok && (autolike || p.pin == ZC_PIN_HUFFMAN);
  const uint64_t pcap = p.stage_len > kHeaderBytes ? p.stage_len - kHeaderBytes : 0;
  const bool stage_ok = p.stage_len > kHeaderBytes;
  for (int i = tid; i < 256; i += NT) {
    s_clens[i] = ctx_ok ? p.ctx->len[i] : 0;
    s_enc[i] = ctx_ok ? p.ctx->enc[i] : 0ull;
  }
  if (tid == 0) {
    for (uint32_t b = 0; b < NB; ++b) mbar_init(&s_mbar[b]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t err = 0;

  auto unit_of = [&](uint64_t t, uint32_t& u, uint32_t& s) {
    const uint64_t head = static_cast<uint64_t>(p.nunits - 1) * s_full;
    if (t < head) {
      u = static_cast<uint32_t>(t / s_full);
      s = static_cast<uint32_t>(t % s_full);
    } else {
      u = p.nunits - 1;
      s = static_cast<uint32_t>(t - head);
    }
  };
  auto unit_R = [&](uint32_t u) {
    const uint64_t uoff = static_cast<uint64_t>(u) * p.unit_bytes;
    return (p.total_bytes - uoff) < p.unit_bytes ? (p.total_bytes - uoff) : p.unit_bytes;
  };
  auto nslices = [&](uint32_t u) { return static_cast<uint32_t>((unit_R(u) + SB - 1) / SB); };

  // tid 0: claim the next slice into buffer b and start its bulk load.
  auto claim = [&](uint32_t b) {
    const unsigned long long t = atomicAdd(&th->next, 1ull);
    s_claim[b] = t;
    s_scanned[b] = 0;
    if (t >= total) return;
    uint32_t u, s;
    unit_of(t, u, s);
    const uint64_t R = unit_R(u);
    const uint64_t off = static_cast<uint64_t>(s) * SB;
    const uint32_t bytes = static_cast<uint32_t>(R - off < SB ? R - off : SB);
    const uint32_t full = bytes & ~15u;
    const uint8_t* src = static_cast<const uint8_t*>(p.src) + static_cast<uint64_t>(u) * p.unit_bytes + off;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&s_mbar[b], full);
    if (full) bulk_g2s(sm.buf[b], src, full, &s_mbar[b]);
  };

  // ---------------------------------------------------------------- scan(t) in buffer b
  auto scan = [&](uint64_t t, uint32_t b, uint32_t parity) {
    uint32_t u, s;
    unit_of(t, u, s);
    SUnit& U = us[u];
    const uint64_t R = unit_R(u);
    const uint64_t off = static_cast<uint64_t>(s) * SB;
    const uint32_t bytes = static_cast<uint32_t>(R - off < SB ? R - off : SB);
    const uint32_t nfull = bytes / 16, nv = (bytes + 15) / 16;
    const bool small = autolike && R <= p.cfg.small_batch_threshold_bytes;
    const bool hist_here = autolike && !small && s == 0;
    uint4* buf = sm.buf[b];
    for (int i = tid; i < 256; i += NT) s_hist[i] = 0;
#ifdef ZC_TASK_TRACE
    const unsigned long long tq0 = (unsigned long long)clock64();
#endif
    mbar_wait(&s_mbar[b], parity);
#ifdef ZC_TASK_TRACE
    if (tid == 0) atomicAdd(&th->tr[0], (unsigned long long)clock64() - tq0);
    const unsigned long long tq1 = (unsigned long long)clock64();
#endif
    if (nfull < nv && tid == 0) {  // message tail (< 16 bytes): plain loads, zero padded
      const uint8_t* src = static_cast<const uint8_t*>(p.src) + static_cast<uint64_t>(u) * p.unit_bytes + off;
      uint32_t w[4] = {0, 0, 0, 0};
      for (uint32_t j = 0; j < bytes - nfull * 16; ++j) w[j >> 2] |= static_cast<uint32_t>(src[nfull * 16 + j]) << (8 * (j & 3));
      buf[nfull] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncthreads();
    uint32_t mz = 0, zero = 0;
    unsigned long long hb = 0;
    const bool any = stage_ok && !small;
    if (any || (kFloat && stage_ok)) {
      for (uint32_t v = tid; v < nv; v += NT) {
        const uint4 x = buf[v];
        const uint32_t nb = v < nfull ? 16u : bytes - nfull * 16;
        uint32_t w[4] = {x.x, x.y, x.z, x.w};
        if (kFloat) {
          RawVec rv;
          rv.a = x;
          rv.nb = nb;
          if (nb == 16)
            words_full<SRC>(p, rv, w, err);
          else
            to_words<SRC>(p, rv, w, err);
          buf[v] = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (any) {
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q)
            if (q < (nb >> 2)) mz = max(mz, zigzag32(static_cast<int32_t>(w[q])));
          if (need_hbits) {
#pragma unroll
            for (uint32_t j = 0; j < 16; ++j) {
              if (j < nb) {
                const uint32_t l = s_clens[byte_of(w, j)];
                hb += l;
                zero |= (l == 0);
              }
            }
          }
        }
        if (hist_here) {
#pragma unroll
          for (uint32_t j = 0; j < 16; ++j) {
            const bool in = j < nb;
            const uint32_t key = in ? byte_of(w, j) : 256u + lane;
            const uint32_t peers = __match_any_sync(__activemask(), key);
            if (in && lane == __ffs(peers) - 1) atomicAdd(&s_hist[key], __popc(peers));
          }
        }
      }
    }
#ifdef ZC_TASK_TRACE
    if (tid == 0) atomicAdd(&th->tr[6], (unsigned long long)clock64() - tq1);
#endif
    // one combined reduction: warp shuffles, one barrier, thread 0 folds the NW partials
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mz = max(mz, __shfl_xor_sync(FULL, mz, o));
      zero |= __shfl_xor_sync(FULL, zero, o);
      hb += __shfl_xor_sync(FULL, hb, o);
    }
    if (lane == 0) {
      s_red32[warp] = mz;
      s_red[warp] = hb | (static_cast<unsigned long long>(zero) << 63);
    }
    if (hist_here) {
      __syncthreads();
      for (int i = tid; i < 256; i += NT) U.hist[i] = s_hist[i];
      __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t r_mz = 0, r_zero = 0;
      unsigned long long r_hb = 0;
      for (int i = 0; i < NW; ++i) {
        r_mz = max(r_mz, s_red32[i]);
        r_zero |= static_cast<uint32_t>(s_red[i] >> 63);
        r_hb += s_red[i] & ~(1ull << 63);
      }
      U.part[s].maxzz = r_mz;
      U.part[s].zero = r_zero;
      U.part[s].bits = r_hb;
      __threadfence();
      s_flag = atomicAdd(&U.scan_done, 1u) == nslices(u) - 1 ? 1u : 0u;
    }
    __syncthreads();
#ifdef ZC_TASK_TRACE
    if (tid == 0) atomicAdd(&th->tr[1], (unsigned long long)clock64() - tq1);
#endif
    if (!s_flag) return;

    // ---------------- the unit's last scan: decision (bit-exact selector, zc_common.cuh)
    __threadfence();
    zc_sample_stats* st_out = p.stats ? p.stats + u : nullptr;
    double el = 0.0;
    bool el_ok = false;
    if (autolike && !small) {
      for (int i = tid; i < 256; i += NT) s_hist[i] = __ldcg(&U.hist[i]);
      __syncthreads();
      if (warp == 0) el_ok = ctx_ok && warp_mean_len(s_hist, s_clens, el);
      if (st_out)
        for (int i = tid; i < 256; i += NT) st_out->hist[i] = s_hist[i];
    }
    if (tid == 0) {
      const uint32_t ns = nslices(u);
      uint32_t maxzz = 0, zl = 0;
      unsigned long long bits = 0;
      for (uint32_t r = 0; r < ns; ++r) {
        maxzz = max(maxzz, __ldcg(&U.part[r].maxzz));
        zl |= __ldcg(&U.part[r].zero);
        U.hbase[r] = bits;
        bits += __ldcg(&U.part[r].bits);
      }
      uint32_t codec = ZC_CODEC_RAW, width = 0;
      unsigned long long payload_b = R;
      if (!stage_ok) {
        codec = CODEC_NONE;
        err |= ZC_DERR_CAPACITY;
      } else {
        const uint64_t W = R < kSampleWindow ? R : kSampleWindow;
        if (autolike) {
          if (!small) {
            zc_sample_stats st;
            st.sampled_bytes = W;
            st.max_zigzag = __ldcg(&U.part[0].maxzz);  // slice 0 == the window: whole words
            st.ctx_code_len_bits = el_ok ? el : 0.0;
            st.ctx_code_len_valid = el_ok ? 1u : 0u;
            st.self_code_len_bits = 0.0;
            st.self_code_len_valid = 0u;
            for (int i = 0; i < 256; ++i) st.hist[i] = 0;  // not read by the selector
            if (st_out) {
              st_out->sampled_bytes = st.sampled_bytes;
              st_out->max_zigzag = st.max_zigzag;
              st_out->ctx_code_len_bits = st.ctx_code_len_bits;
              st_out->self_code_len_bits = 0.0;
              st_out->ctx_code_len_valid = st.ctx_code_len_valid;
              st_out->self_code_len_valid = 0u;
            }
            const zc_arbitration_plan plan = arbitrate_plan(R, pcap, st, p.hint, ctx_ok, p.cfg);
            if (plan.choice == ZC_CODEC_FIXEDLEN) {
              width = width_from_maxzz(maxzz);
              const unsigned long long pay = packed_bytes(R / 4, width);
              if (pay > 0 && pay <= pcap && gain_ok(R, pay, p.cfg.min_gain_permil)) {
                codec = ZC_CODEC_FIXEDLEN;
                payload_b = pay;
              }
            } else if (plan.choice == ZC_CODEC_HUFFMAN && ctx_ok) {
              const unsigned long long pay = (bits + 7) / 8;
              if (!zl && pay > 0 && pay <= pcap && gain_ok(R, pay, p.cfg.min_gain_permil)) {
                codec = ZC_CODEC_HUFFMAN;
                payload_b = pay;
              }
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
          const unsigned long long pay = (bits + 7) / 8;
          if (!zl && pay > 0 && pay <= pcap) {
            codec = ZC_CODEC_HUFFMAN;
            payload_b = pay;
          }
        }
        if (codec == ZC_CODEC_RAW && R > pcap) {
          codec = CODEC_NONE;
          err |= ZC_DERR_CAPACITY;
        }
      }
      U.dec.codec = codec;
      U.dec.width = width;
      U.dec.payload = payload_b;
      __threadfence();
      st_release_gpu(&U.ready, 1u);
    }
  };

  // ---------------------------------------------------------------- encode(t) from buffer b
  auto encode = [&](uint64_t t, uint32_t b) {
    uint32_t u, s;
    unit_of(t, u, s);
    SUnit& U = us[u];
    const uint64_t R = unit_R(u);
    const uint64_t off = static_cast<uint64_t>(s) * SB;
    const uint32_t bytes = static_cast<uint32_t>(R - off < SB ? R - off : SB);
    const uint32_t nfull = bytes / 16, nv = (bytes + 15) / 16;
    uint8_t* stage = p.stages + static_cast<uint64_t>(u) * p.stride;
    uint8_t* payload = stage + kHeaderBytes;
    uint4* buf = sm.buf[b];
#ifdef ZC_TASK_TRACE
    const unsigned long long te0 = (unsigned long long)clock64();
#endif
    if (tid == 0) {
      while (ld_acquire_gpu(&U.ready) == 0) __nanosleep(32);
#ifdef ZC_TASK_TRACE
      atomicAdd(&th->tr[2], (unsigned long long)clock64() - te0);
#endif
      s_dec.codec = __ldcg(&U.dec.codec);
      s_dec.width = __ldcg(&U.dec.width);
      s_dec.payload = __ldcg(&U.dec.payload);
    }
    __syncthreads();
    const uint32_t codec = s_dec.codec;
    const uint64_t P = s_dec.payload;
    if (codec == ZC_CODEC_RAW) {
      uint4* dst = reinterpret_cast<uint4*>(payload + off);
      for (uint32_t v = tid; v < nfull; v += NT) dst[v] = buf[v];
      if (nfull < nv && tid == 0) {
        const uint4 x = buf[nfull];
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
        for (uint32_t j = 0; j < bytes - nfull * 16; ++j) payload[off + nfull * 16 + j] = static_cast<uint8_t>(byte_of(w, j));
      }
    } else if (codec == ZC_CODEC_FIXEDLEN) {
      const uint32_t width = s_dec.width;
      const uint64_t sym0 = off / 4;  // first symbol of the slice (multiple of 16384)
      for (uint32_t c0 = static_cast<uint32_t>(warp) * 256; c0 < nv; c0 += NW * 256) {
        uint4* chunk = buf + c0;
        uint4 q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t v = c0 + 32 * j + lane;
          q[j] = v < nv ? chunk[32 * j + lane] : make_uint4(0, 0, 0, 0);
          if (v == nfull && nfull < nv) {  // tail vector: only whole words are symbols
            const uint32_t nw = (bytes - nfull * 16) >> 2;
            if (nw < 4) q[j].w = 0;
            if (nw < 3) q[j].z = 0;
            if (nw < 2) q[j].y = 0;
            if (nw < 1) q[j].x = 0;
          }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t slot = 32 * j + lane;
          chunk[swz(slot)] = make_uint4(zigzag32(static_cast<int32_t>(q[j].x)), zigzag32(static_cast<int32_t>(q[j].y)),
                                        zigzag32(static_cast<int32_t>(q[j].z)), zigzag32(static_cast<int32_t>(q[j].w)));
        }
        __syncwarp();
        uint32_t z[32];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const uint4 x = chunk[swz(8 * lane + m)];
          z[4 * m] = x.x;
          z[4 * m + 1] = x.y;
          z[4 * m + 2] = x.z;
          z[4 * m + 3] = x.w;
        }
        if (c0 + 8 * lane < nv) pack_store_w(width, z, payload, (sym0 / 32 + c0 / 8 + lane) * width, P);
      }
    } else if (codec == ZC_CODEC_HUFFMAN) {
      // Tiles of NT/2 vectors when some code is longer than 16 bits keep the tile within HT_WORDS.
      const uint32_t maxlen = p.ctx->max_len;
      const uint32_t tv = maxlen <= 16 ? NT : NT / 2;
      uint32_t* tile = sm.tile;
      uint32_t* uindex = p.index ? p.index + static_cast<uint64_t>(u) * p.index_stride : nullptr;
      const uint64_t vbase = off / 16;  // unit-level vector index of the slice start
      unsigned long long base_bits = __ldcg(&U.hbase[s]);
      for (int i = tid; i < static_cast<int>(HT_WORDS); i += NT) tile[i] = 0;
      bool first_tile = true, has_head = false;
      unsigned long long head_idx = 0;
      uint32_t head_val = 0, end_mod = 0;
      __syncthreads();
      for (uint32_t t0 = 0; t0 < nv; t0 += tv) {
        const uint32_t v = t0 + tid;
        const bool act = static_cast<uint32_t>(tid) < tv && v < nv;
        uint32_t w[4] = {0, 0, 0, 0}, nb = 0;
        if (act) {
          const uint4 x = buf[v];
          w[0] = x.x;
          w[1] = x.y;
          w[2] = x.z;
          w[3] = x.w;
          nb = v < nfull ? 16u : bytes - nfull * 16;
        }
        unsigned long long ev[16];
        uint32_t Lb = 0;
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j) {
          ev[j] = j < nb ? s_enc[byte_of(w, j)] : 0ull;
          Lb += static_cast<uint32_t>(ev[j] >> 32);
        }
        uint32_t ttot;
        const uint32_t boff = block_excl_scan(Lb, s_red32, &ttot);
        if (act && uindex != nullptr && ((vbase + v) & 63) == 0) uindex[(vbase + v) >> 6] = static_cast<uint32_t>(base_bits + boff);
        {
          const uint32_t lp = static_cast<uint32_t>(base_bits & 31) + boff;
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
        const uint32_t nfw = endb >> 5;
        const uint64_t gw0 = base_bits >> 5;
        for (uint32_t i = tid; i < nfw; i += NT) {
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
        const uint32_t carry = (endb & 31) ? tile[nfw] : 0u;
        __syncthreads();
        for (uint32_t i = tid; i <= nfw + 1 && i < HT_WORDS; i += NT) tile[i] = 0;
        __syncthreads();
        if (tid == 0) tile[0] = carry;
        if (nfw > 0) first_tile = false;
        base_bits += ttot;
        end_mod = static_cast<uint32_t>(base_bits & 31);
        __syncthreads();
      }
      if (tid == 0) {
        U.has_head[s] = has_head ? 1u : 0u;
        U.head_idx[s] = head_idx;
        U.head_val[s] = head_val;
        const bool has_tail = nv > 0 && end_mod != 0;
        U.has_tail[s] = has_tail ? 1u : 0u;
        U.tail_idx[s] = base_bits >> 5;
        U.tail_val[s] = tile[0];
        __threadfence();
        if (atomicAdd(&U.edone, 1u) == nslices(u) - 1) {  // last encoder merges the slice seams
          __threadfence();
          const uint32_t ns = nslices(u);
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
    }
#ifdef ZC_TASK_TRACE
    if (tid == 0) atomicAdd(&th->tr[3], (unsigned long long)clock64() - te0);
#endif
    // header + result: slice 0 (the decision is the unit's)
    if (s == 0 && tid == 0) {
      zc_encode_result res;
      res._pad = 0;
      if (codec == CODEC_NONE) {
        res.codec = ZC_CODEC_RAW;
        res.payload_bytes = 0;
        res.total_bytes = 0;
      } else {
        const zc_frame_header h = make_header(codec, 0, R, P, codec == ZC_CODEC_FIXEDLEN ? s_dec.width : 0);
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
  };

  // ---------------------------------------------------------------- pipeline
  __syncthreads();
  if (tid == 0)
    for (uint32_t j = 0; j + 1 < NB; ++j) claim(j);
  __syncthreads();
  unsigned long long prev = ~0ull;
  uint32_t prev_b = 0;
  for (uint32_t it = 0;; ++it) {
    const uint32_t b = it % NB;
    const uint32_t parity = (it / NB) & 1u;
    const unsigned long long t = s_claim[b];
    const bool have = t < total;
    if (have && !s_scanned[b]) scan(t, b, parity);
    __syncthreads();
    if (prev != ~0ull) {
      // Before waiting for a decision, scan every claim we hold: then no CTA ever blocks with an
      // unscanned claim, so the oldest unit in flight (fully claimed: a CTA holds NB claims and
      // NB * gridDim >> slices per unit) always completes — no deadlock and no convoy.
      const uint32_t nb2 = (it + 1) % NB;
      const unsigned long long tn = s_claim[nb2];
      if (tn < total && !s_scanned[nb2]) {
        if (tid == 0) {
          uint32_t pu, ps;
          unit_of(prev, pu, ps);
          s_pre = ld_acquire_gpu(&us[pu].ready) == 0 ? 1u : 0u;
        }
        __syncthreads();
        if (s_pre) {
          scan(tn, nb2, ((it + 1) / NB) & 1u);
          __syncthreads();
          if (tid == 0) s_scanned[nb2] = 1;
        }
      }
      encode(prev, prev_b);
      __syncthreads();
      if (tid == 0) claim(prev_b);  // the freed buffer takes claim it + NB - 1
    } else if (it == 0) {
      if (tid == 0) claim(NB - 1);
    }
    __syncthreads();
    if (!have) break;
    prev = t;
    prev_b = b;
  }
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
#ifdef ZC_TASK_TRACE
  if (tid == 0 && atomicAdd(&th->tr[5], 1ull) == gridDim.x - 1) {
    __threadfence();
    const double k = 1.0 / 1965.0 / gridDim.x;
    printf("stream pin=%d ctas=%u per-cta us: loadwait %.1f scan %.1f (loop %.1f) decwait %.1f encode(incl wait) %.1f\n", p.pin,
           gridDim.x, th->tr[0] * k, th->tr[1] * k, th->tr[6] * k, th->tr[2] * k, th->tr[3] * k);
  }
#endif
}

template <int SRC>
cudaError_t launch_stream_t(const EncParams& p, void* scratch, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(stream_kernel<SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(SmemStream)));
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static_assert(sizeof(SHdr) <= 256, "stream header must fit its slot");
  cudaMemsetAsync(scratch, 0, 256 + sizeof(SUnit) * p.nunits, s);
  SHdr* th = static_cast<SHdr*>(scratch);
  SUnit* us = reinterpret_cast<SUnit*>(static_cast<uint8_t*>(scratch) + 256);
  const uint32_t s_full = static_cast<uint32_t>((p.unit_bytes + SB - 1) / SB);
  const uint64_t last_R = p.total_bytes - static_cast<uint64_t>(p.nunits - 1) * p.unit_bytes;
  const uint64_t total = static_cast<uint64_t>(p.nunits - 1) * s_full + (last_R + SB - 1) / SB;
  const uint32_t ctas = static_cast<uint32_t>(std::min<uint64_t>(static_cast<uint64_t>(sms), total));
  note_launch();
  stream_kernel<SRC><<<ctas, NT, sizeof(SmemStream), s>>>(p, us, th, s_full, total);
  return cudaGetLastError();
}

}  // namespace

bool stream_encoder_ok(const EncParams& p) {
  return (p.src_kind == SRC_F32 || p.src_kind == SRC_BYTES) && p.unit_bytes <= ZC_BATCH_RAW_BYTES &&
         p.unit_bytes % SB == 0 && (reinterpret_cast<uintptr_t>(p.src) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(p.stages) & 15) == 0 && p.stride % 16 == 0 && !p.cfg.embed_codebook;
}

size_t stream_scratch_bytes(uint32_t nunits) { return 256 + sizeof(SUnit) * nunits; }

void preload_stream_kernels() {
  cudaFuncSetAttribute(stream_kernel<SRC_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(sizeof(SmemStream)));
  cudaFuncSetAttribute(stream_kernel<SRC_BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(sizeof(SmemStream)));
  cudaGetLastError();
}

cudaError_t launch_encode_stream(const EncParams& p, void* scratch, cudaStream_t s) {
  if (p.nunits == 0) return cudaSuccess;
  return p.src_kind == SRC_F32 ? launch_stream_t<SRC_F32>(p, scratch, s) : launch_stream_t<SRC_BYTES>(p, scratch, s);
}

}  // namespace zc
