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

constexpr int DT = 256;                // threads per CTA
constexpr uint64_t SLICE_VEC = 16384;  // 16-byte vectors per CTA slice (256 KiB)
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ uint64_t unit_raw(const DecParams& p, uint32_t u) {
  if (p.bare) return p.hdr.raw_bytes;
  uint64_t off = static_cast<uint64_t>(u) * p.unit_bytes;
  uint64_t rest = p.total_bytes - off;
  return rest < p.unit_bytes ? rest : p.unit_bytes;
}

__device__ __forceinline__ uint64_t unit_region(const DecParams& p, uint32_t u) {
  return p.frame_len ? p.frame_len[u].total_bytes : p.region;
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
  if (!s_fail && fc.codec == ZC_CODEC_HUFFMAN) {
    const bool ok = load_huff_tables<false>(fc, payload, p.ctx, &s_t, &s_flag, s_lens);
    if (!ok) {
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

__global__ void __launch_bounds__(DT) decode_kernel(const DecParams p) {
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
  constexpr size_t kWordsBytes = sizeof(uint32_t) * (DT / 32) * 136 * 4;
  __shared__ __align__(16) uint8_t s_pool[sizeof(DevHuff) > kWordsBytes ? sizeof(DevHuff) : kWordsBytes];
  DevHuff& s_t = *reinterpret_cast<DevHuff*>(s_pool);
  uint32_t* s_words = reinterpret_cast<uint32_t*>(s_pool);
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
  uint32_t f = decode_slice<false, 4>(fc, payload, R, v0, v1, sink, obase, idx, p.ctx, &s_t, &s_flag, s_lens, s_words, err);
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
  cudaFuncSetAttribute(decode_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 40);
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
  if (first_on_device(carve)) cudaFuncSetAttribute(decode_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 40);
  note_launch();
  decode_kernel<<<grid, DT, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace zc
