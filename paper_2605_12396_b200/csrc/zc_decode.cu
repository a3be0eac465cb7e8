// zc_decode.cu — batched frame decode dispatch fused with the consumer of the symbols.
//
// Reference path (relative to /root/reference/proj/core/): RankCtx::recv_batch
// (collectives.cpp:304-348) -> fixedlen_decode_into (fixedlen.cpp:39-65) /
// huffman_decode_into (huffman.cpp:248-316) -> RS sink (collectives.cpp:480-491) or
// dequantize_into (quant.cpp:107-127).
//
// One launch decodes every unit (4 MiB batch) of a message; each CTA owns a 256 KiB slice of one
// unit's output.  The codec is read from the frame header on the device, so the host never learns
// it.  Huffman frames are decoded chunk-parallel, one thread per 1 KiB grain, from the encoder's
// companion bit-offset index; a grain that does not end exactly where the next one starts (an
// index that does not belong to the payload) sends the unit to the sequential decoder, which is
// also the path for frames that come without an index (e.g. produced by the CPU reference).
#include <cstdlib>

#include "zc_decode.cuh"

namespace zc {
namespace {

// (Measured and dropped: 128-thread CTAs over 128 KiB slices at 7 per SM, for 1.98 waves instead
// of 1.73 — the full shared-memory carveout they need leaves the L1 too small for the Huffman
// window loads, which overlap from round to round: 410 vs 394 us.)
constexpr int DT = 256;                // threads per CTA
constexpr int DT_CTAS = 4;             // resident CTAs per SM (64 registers, ~40 KB shared each)
constexpr uint64_t SLICE_VEC = 16384;  // 16-byte vectors per CTA slice (256 KiB)
constexpr unsigned FULL = 0xffffffffu;
constexpr int kCarveout = 75;           // percent of L1 as shared memory: 4 CTAs x ~40 KB

__device__ __forceinline__ uint64_t unit_raw(const DecParams& p, uint32_t u) {
  if (p.bare) return p.hdr.raw_bytes;
  uint64_t off = static_cast<uint64_t>(u) * p.unit_bytes;
  uint64_t rest = p.total_bytes - off;
  return rest < p.unit_bytes ? rest : p.unit_bytes;
}

__device__ __forceinline__ uint64_t unit_region(const DecParams& p, uint32_t u) {
  return p.frame_len ? p.frame_len[u].total_bytes : p.region;
}


// Index-less Huffman frames (e.g. from the CPU reference: huffman.cpp:281-314 has no sync points),
// decoded by the whole CTA with self-synchronisation.  The stream's bits are split into one
// segment per thread; every thread decodes from a start position to the first code boundary at or
// past its segment's end, counting the codes that start inside.  Round 0 starts every thread at
// its raw segment start (mid-code: garbage at first, but a Huffman decoder falls into step with
// the true code boundaries after a few codes); each later round restarts thread t at the end
// thread t-1 reached.  When no start changes, every thread decoded from a true boundary: the
// counts are exact, an exclusive scan places each thread's symbols, and a last pass writes them.
// Codes crossing the stream end are not decoded (as huff_run); the first n symbols must decode.
// Returns false when they do not (the caller then replays the sequential decoder, which also
// reproduces the reference's partial output).  out: the n raw bytes.  All threads call.
struct SyncScan {
  uint64_t end;       // first code boundary >= the segment end (or where decoding stopped)
  uint32_t count;     // codes starting in [start, segment end)
  uint32_t bad_at;    // codes before an undecodable code / a code crossing the stream end, or ~0
};
__device__ __forceinline__ SyncScan sync_scan(const DevHuff* t, const uint8_t* s, uint64_t slen, uint64_t start,
                                              uint64_t seg_end, uint8_t* out, uint64_t obase, uint64_t n) {
  const uint64_t total = slen * 8;
  SyncScan r{start, 0u, 0xffffffffu};
  uint64_t bitpos = start;
  while (bitpos < seg_end) {
    // a 64-bit window at bitpos (bits past the stream end read as zero)
    const uint64_t w = bitpos >> 5;
    const unsigned long long acc =
        ((static_cast<unsigned long long>(stream_word<false>(s, slen, w + 1)) << 32) | stream_word<false>(s, slen, w)) >>
        (bitpos & 31);
    const uint16_t e = t->lut[acc & ((1u << ZC_HUFF_ROOT_BITS) - 1)];
    uint32_t l = e >> 8, sym = e & 0xFFu;
    if (l == 0) l = huff_long(t, acc, sym);  // acc holds >= 33 valid bits
    if (l == 0 || bitpos + l > total) {
      r.bad_at = r.count;
      break;
    }
    if (out != nullptr && obase + r.count < n) out[obase + r.count] = static_cast<uint8_t>(sym);
    ++r.count;
    bitpos += l;
  }
  r.end = bitpos;
  return r;
}

__device__ bool huff_parallel_sync(const DevHuff* t, const uint8_t* s, uint64_t slen, uint64_t n, uint8_t* out) {
  __shared__ unsigned long long s_end[DT];
  __shared__ uint32_t s_cnt[DT];
  __shared__ uint32_t s_fail;
  const int tid = threadIdx.x;
  const uint64_t total = slen * 8;
  const uint64_t seg0 = total * tid / DT, seg1 = total * (tid + 1) / DT;
  uint64_t start = tid == 0 ? 0 : seg0;
  SyncScan r{};
  for (int round = 0;; ++round) {
    r = sync_scan(t, s, slen, start, seg1, nullptr, 0, 0);
    s_end[tid] = r.end;
    __syncthreads();
    const uint64_t ns = tid == 0 ? 0 : max(static_cast<uint64_t>(s_end[tid - 1]), seg0);
    const bool changed = ns != start;
    start = ns;
    __syncthreads();
    if (!__syncthreads_or(changed)) break;
    if (round >= DT) return false;  // no convergence: let the sequential decoder decide
  }
  // exclusive scan of the counts; the first n symbols must all decode
  s_cnt[tid] = r.count;
  if (tid == 0) s_fail = 0;
  __syncthreads();
  uint64_t off = 0, sum = 0;
  for (int i = 0; i < DT; ++i) {  // DT shared reads per thread: cheap next to the decode
    if (i < tid) off += s_cnt[i];
    sum += s_cnt[i];
  }
  if (r.bad_at != 0xffffffffu && off + r.bad_at < n) atomicOr(&s_fail, 1u);
  __syncthreads();
  if (s_fail || sum < n) return false;
  if (off < n) sync_scan(t, s, slen, start, seg1, out, off, n);
  __syncthreads();
  return true;
}

// The unit's last decode CTA (one per unit, when a flag is set): sequential Huffman decode for units whose index is missing or
// disagrees with the payload (flag bit 0), and the raw-copy fallback for undecodable units.
__device__ void fixup_unit(const DecParams& p, uint32_t u, uint32_t f, FrameCheck& fc, DevHuff& s_t, uint8_t* s_lens,
                           uint32_t& s_flag, uint32_t& s_fail) {
  const uint64_t R = unit_raw(p, u);
  const uint8_t* stage = p.stages + static_cast<uint64_t>(u) * p.stride;
  const uint8_t* payload = p.bare ? stage : stage + kHeaderBytes;
  const uint64_t obase = p.bare ? 0 : static_cast<uint64_t>(u) * p.unit_bytes;
  uint32_t err = 0;
  // Bit 0 makes the sequential decode authoritative; bit 1 alone (a grain hit an undecodable
  // code on a consistent index) is a failure the sequential decoder reaches identically.  A
  // reduction sink cannot be replayed after a partial add, so there the frame is reported corrupt.
  if (threadIdx.x == 0) {
    check_frame<false>(stage, unit_region(p, u), R, p.bare ? &p.hdr : nullptr, p.bare != 0, p.ctx, true, fc);
    s_fail = ((f & 1u) == 0 || is_add_sink(p.out_kind)) ? 1u : 0u;
  }
  __syncthreads();
  const double sc = dec_scale(p);
  Sink sink{p.out_kind, p.out, sc, p.out_kind == OUT_ADD_Q ? 1.0 / sc : 0.0, p.acc_f32, 0u};
  __shared__ uint32_t s_par;
  if (!s_fail && fc.codec == ZC_CODEC_HUFFMAN) {
    const bool ok = load_huff_tables<false>(fc, payload, p.ctx, &s_t, &s_flag, s_lens);
    // byte / fp32 outputs: the CTA-parallel self-synchronising decode into the output's raw bytes,
    // then (fp32) the sink applied in place, 16 bytes at a time (same size)
    if (threadIdx.x == 0) s_par = 0;
    __syncthreads();
    if (ok && (p.out_kind == OUT_BYTES || p.out_kind == OUT_F32)) {
      const bool emb = (fc.h.flags & ZC_FLAG_EMBEDDED_CODEBOOK) != 0;
      const uint8_t* s = payload + (emb ? ZC_HUFF_CODEBOOK_BYTES : 0);
      const uint64_t slen = fc.h.payload_bytes - (emb ? ZC_HUFF_CODEBOOK_BYTES : 0);
      const uint64_t n = fc.h.raw_bytes;
      uint8_t* raw = static_cast<uint8_t*>(p.out) + obase;
      if (huff_parallel_sync(&s_t, s, slen, n, raw)) {
        if (p.out_kind == OUT_F32) {
          for (uint64_t v = threadIdx.x; v * 16 < n; v += DT) {
            const uint32_t nb = static_cast<uint32_t>(n - v * 16 < 16 ? n - v * 16 : 16);
            uint32_t w[4] = {0, 0, 0, 0};
            for (uint32_t j = 0; j < nb; ++j) w[j >> 2] |= static_cast<uint32_t>(raw[v * 16 + j]) << (8 * (j & 3));
            emit16(sink, obase + v * 16, w, nb, err);
          }
        }
        if (threadIdx.x == 0) s_par = 1;
      }
      __syncthreads();
    }
    if (s_par) {
      // decoded
    } else if (!ok) {
      if (threadIdx.x == 0) s_fail = 1;
    } else if (threadIdx.x == 0) {
      const bool emb = (fc.h.flags & ZC_FLAG_EMBEDDED_CODEBOOK) != 0;
      const uint8_t* s = payload + (emb ? ZC_HUFF_CODEBOOK_BYTES : 0);
      const uint64_t slen = fc.h.payload_bytes - (emb ? ZC_HUFF_CODEBOOK_BYTES : 0);
      uint64_t endb;
      unsigned long long lo = 0, hi = 0;
      const uint64_t n = fc.h.raw_bytes;
      bool good = huff_run<false>(&s_t, s, slen, 0, n, &endb, [&](uint64_t j, uint32_t sym) {
        const uint32_t k = static_cast<uint32_t>(j & 15);
        if (k < 8) lo |= static_cast<unsigned long long>(sym) << (8 * k);
        else hi |= static_cast<unsigned long long>(sym) << (8 * (k - 8));
        if (k == 15 || j + 1 == n) {
          uint32_t ww[4] = {static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32), static_cast<uint32_t>(hi),
                            static_cast<uint32_t>(hi >> 32)};
          emit16(sink, obase + (j & ~15ull), ww, k + 1, err);
          lo = hi = 0;
        }
      });
      if (!good) s_fail = 1;
    }
  }
  __syncthreads();
  if (s_fail) {
    if (threadIdx.x == 0) {
      if (p.bare) {
        if (p.ok_out) *p.ok_out = 0;
      } else if (p.codec_out) {
        p.codec_out[u] = kFallback;
      }
      if (is_add_sink(p.out_kind)) err |= ZC_DERR_CORRUPT;
    }
    if (!p.bare && !is_add_sink(p.out_kind)) {
      const uint64_t have = fc.region > kHeaderBytes ? fc.region - kHeaderBytes : 0;
      const uint64_t lim = R < have ? R : have;
      for (uint64_t v = threadIdx.x; v * 16 < lim; v += DT) {
        uint32_t nb = static_cast<uint32_t>(lim - v * 16 < 16 ? lim - v * 16 : 16);
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = stream_word<false>(payload, lim, v * 4 + k);
        emit16(sink, obase + v * 16, w, nb, err);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) p.flags[u] = 0;
  if (err && p.err) atomicOr(p.err, err);
}

__global__ void __launch_bounds__(DT, DT_CTAS) decode_kernel(const DecParams p) {
  pdl_wait();  // a programmatic dependent of the FixedLen decoder (it writes the codecs / outputs first)
  const uint32_t u = blockIdx.y;
  const uint64_t R = unit_raw(p, u);
  const uint64_t nvec = (R + 15) / 16;
  const uint64_t v0 = static_cast<uint64_t>(blockIdx.x) * SLICE_VEC;
  if (v0 >= nvec && blockIdx.x != 0) return;
  const uint64_t v1 = min(nvec, v0 + SLICE_VEC);
  const uint8_t* stage = p.stages + static_cast<uint64_t>(u) * p.stride;
  const uint8_t* payload = p.bare ? stage : stage + kHeaderBytes;
  const uint64_t obase = p.bare ? 0 : static_cast<uint64_t>(u) * p.unit_bytes;
  const int tid = threadIdx.x, lane = tid & 31;

  __shared__ FrameCheck fc;
  // a frame is one codec: the Huffman tables and the FixedLen staging words share the space, which
  // leaves the L1 room for every thread's current 128-byte line of its Huffman grain
  // (Huffman: the tables, then the swizzled root LUT and the warps' stream windows)
  constexpr size_t kWordsBytes = sizeof(uint32_t) * (DT / 32) * 136 * 4;
  constexpr size_t kTabBytes = (sizeof(DevHuff) + 15) / 16 * 16;
  constexpr size_t kHuffBytes =
      kTabBytes + 2u * (1u << ZC_HUFF_ROOT_BITS) + sizeof(uint32_t) * (DT / 32) * kHuffWarpScratchWords;
  __shared__ __align__(16) uint8_t s_pool[kHuffBytes > kWordsBytes ? kHuffBytes : kWordsBytes];
  DevHuff& s_t = *reinterpret_cast<DevHuff*>(s_pool);
  uint32_t* s_words = reinterpret_cast<uint32_t*>(s_pool);
  uint32_t* s_hscratch = p.huff_lane ? nullptr : reinterpret_cast<uint32_t*>(s_pool + kTabBytes);
  __shared__ uint8_t s_lens[256];
  __shared__ uint32_t s_flag;
  uint32_t err = 0;

  if (tid == 0)
    check_frame<false>(stage, unit_region(p, u), R, p.bare ? &p.hdr : nullptr, p.bare != 0, p.ctx, p.index != nullptr, fc);
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    if (p.codec_out && !p.bare && !(p.fast && (fc.codec == ZC_CODEC_RAW || fc.codec == ZC_CODEC_FIXEDLEN)))
      p.codec_out[u] = fc.codec;
    if (p.bare && p.ok_out) *p.ok_out = fc.codec == kFallback ? 0 : 1;
    if (fc.need_seq) atomicOr(&p.flags[u], 1u);
  }
  if (fc.codec == kFallback && p.bare) return;
  if (p.fast && (fc.codec == ZC_CODEC_RAW || fc.codec == ZC_CODEC_FIXEDLEN)) return;  // zc_fixed.cu decoded it
  const double sc = dec_scale(p);
  Sink sink{p.out_kind, p.out, sc, p.out_kind == OUT_ADD_Q ? 1.0 / sc : 0.0, p.acc_f32, 0u};
  const uint32_t* idx = p.index ? p.index + static_cast<uint64_t>(u) * p.index_stride : nullptr;
  uint32_t f = decode_slice<false, 4>(fc, payload, R, v0, v1, sink, obase, idx, p.ctx, &s_t, &s_flag, s_lens, s_words, err,
                                       s_hscratch);
  if (p.maxzz_out != nullptr && is_add_sink(p.out_kind)) {  // the sums' range, for the next send
    const uint32_t m = __reduce_max_sync(FULL, sink.mz);
    if (lane == 0 && m) atomicMax(p.maxzz_out + u, m);
  }
  f = __reduce_or_sync(FULL, f);
  if (lane == 0 && f) atomicOr(&p.flags[u], f);
  err = __reduce_or_sync(FULL, err);
  if (lane == 0 && err && p.err) atomicOr(p.err, err);
  // the unit's CTAs count themselves in the flag word's upper bits; the last one runs the fixup
  // (sequential decode / raw-copy fallback) when a flag is set, after every other CTA's output
  __shared__ uint32_t s_last, s_fail;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const uint64_t nct = (nvec + SLICE_VEC - 1) / SLICE_VEC;
    const uint32_t old = atomicAdd(&p.flags[u], 0x100u);
    s_last = ((old >> 8) + 1 == (nct > 0 ? nct : 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const uint32_t fl = __ldcg(&p.flags[u]) & 0xFFu;
  if (fl == 0) {
    if (tid == 0) p.flags[u] = 0;
    return;
  }
  __syncthreads();
  fixup_unit(p, u, fl, fc, s_t, s_lens, s_flag, s_fail);
}

}  // namespace

void preload_decode_kernels() {
  cudaFuncSetAttribute(decode_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, kCarveout);
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, decode_kernel);
  cudaGetLastError();
}

cudaError_t launch_decode(const DecParams& p0, cudaStream_t s) {
  if (p0.nunits == 0) return cudaSuccess;
  DecParams p = p0;
  p.fast = 0;
  if (fixed_decode_ok(p) && std::getenv("ZC_NO_FIXED") == nullptr) {
    if (cudaError_t e = launch_fixed_decode(p, s)) return e;
    p.fast = 1;
    if (p.own_frames) return cudaSuccess;
  }
  const uint64_t maxR = p.bare ? p.hdr.raw_bytes : (p.unit_bytes < p.total_bytes ? p.unit_bytes : p.total_bytes);
  const uint64_t nvec = (maxR + 15) / 16;
  const uint32_t slices = static_cast<uint32_t>((nvec + SLICE_VEC - 1) / SLICE_VEC);
  dim3 grid(slices > 0 ? slices : 1, p.nunits);
  static std::atomic<uint64_t> carve{0};
  if (first_on_device(carve)) cudaFuncSetAttribute(decode_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, kCarveout);
  static const bool lane_dec = std::getenv("ZC_HUFF_LANE") != nullptr;  // A/B: the per-lane grain decoder
  p.huff_lane = lane_dec ? 1 : 0;
  note_launch();
  if (p.fast) return launch_pdl(decode_kernel, grid, dim3(DT), 0, s, p);
  decode_kernel<<<grid, DT, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace zc
