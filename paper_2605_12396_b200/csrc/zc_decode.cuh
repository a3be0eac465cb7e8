// zc_decode.cuh — device-side frame checks and decoders shared by the standalone decode kernel
// (zc_decode.cu) and the fused ring-step kernels (zc_encode.cu).
//
// Reference (relative to /root/reference/proj/core/):
//   recv_batch header checks + raw-copy fallback   collectives.cpp:304-348
//   fixedlen_decode_into                           fixedlen.cpp:39-65
//   huffman_decode_into                            huffman.cpp:248-316
//   RS sink (int64-checked add)                    collectives.cpp:480-491
//   dequantize_into                                quant.cpp:107-127
#pragma once
#include "zc_huff_device.cuh"
#include "zc_kernels.h"

namespace zc {

constexpr uint32_t kFallback = 0xFFFFFFFFu;

struct FrameCheck {
  zc_frame_header h;
  uint64_t region;
  uint32_t codec;  // codec to run, or kFallback
  uint32_t need_seq;
};

// Loads honour the producer: frames written during this kernel or by a peer GPU are read through
// L2 (ld.global.cg); immutable inputs use the read-only path.
template <bool kCoherent>
__device__ __forceinline__ uint32_t ld32(const uint32_t* p) {
  if (kCoherent) return __ldcg(p);
  return __ldg(p);
}
template <bool kCoherent>
__device__ __forceinline__ uint4 ld128(const uint4* p) {
  if (kCoherent) return __ldcg(p);
  return __ldg(p);
}
template <bool kCoherent>
__device__ __forceinline__ uint8_t ld8(const uint8_t* p) {
  if (kCoherent) return static_cast<uint8_t>(__ldcg(reinterpret_cast<const char*>(p)));
  return __ldg(p);
}

// 32-bit word w of a byte stream of `len` bytes; bytes past the end read as zero.
template <bool kCoherent>
__device__ __forceinline__ uint32_t stream_word(const uint8_t* s, uint64_t len, uint64_t w) {
  uint64_t b = w * 4;
  if (b + 4 <= len) return ld32<kCoherent>(reinterpret_cast<const uint32_t*>(s) + w);
  uint32_t v = 0;
  for (uint32_t j = 0; j < 4; ++j)
    if (b + j < len) v |= static_cast<uint32_t>(ld8<kCoherent>(s + b + j)) << (8 * j);
  return v;
}

// Exact int32 -> double without the conversion pipe: (2^52 + 2^31 + s) - (2^52 + 2^31).
__device__ __forceinline__ double i2d(uint32_t s) {
  return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(s ^ 0x80000000u)), 4503601774854144.0);
}

// Output sink for decoded symbol vectors.
struct Sink {
  int kind;      // OutKind
  void* out;     // base of the whole message (raw byte offsets index it)
  double scale;  // dequantization factor; OUT_ADD_Q: the quantizer's bin width
  double rcp;    // OUT_ADD_Q: 1 / scale
  const float* acc;  // OUT_ADD_Q: the local fp32 chunk (indexed like `out`)
  mutable uint32_t mz;  // OUT_ADD_*: running max zig-zag of the sums this thread wrote
};
__host__ __device__ __forceinline__ bool is_add_sink(int kind) { return kind == OUT_ADD_I32 || kind == OUT_ADD_Q; }

// Writes 4 decoded symbol words (16 raw bytes; nb valid) at raw byte offset `ob` of the output.
__device__ __forceinline__ void emit16(const Sink& k, uint64_t ob, const uint32_t w[4], uint32_t nb, uint32_t& err) {
  switch (k.kind) {
    case OUT_F32: {
      float* o = static_cast<float*>(k.out) + ob / 4;
      float f[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) f[i] = d2f_rn(__dmul_rn(k.scale, i2d(w[i])));
      if (nb == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
        *reinterpret_cast<float4*>(o) = make_float4(f[0], f[1], f[2], f[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (static_cast<uint32_t>(i) < nb / 4) o[i] = f[i];
      }
      break;
    }
    case OUT_F64: {
      double* o = static_cast<double*>(k.out) + ob / 4;
      double d[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) d[i] = __dmul_rn(k.scale, i2d(w[i]));
      if (nb == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
        reinterpret_cast<double2*>(o)[0] = make_double2(d[0], d[1]);
        reinterpret_cast<double2*>(o)[1] = make_double2(d[2], d[3]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (static_cast<uint32_t>(i) < nb / 4) o[i] = d[i];
      }
      break;
    }
    case OUT_ADD_Q: {  // allreduce_eb's RS sink: q(local fp32) + decoded, int64-checked
      int32_t* o = static_cast<int32_t*>(k.out) + ob / 4;
      const float* x = k.acc + ob / 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (static_cast<uint32_t>(i) < nb / 4) {
          const int32_t q = quantize_one(static_cast<double>(x[i]), k.scale, k.rcp, err);
          const long long s = static_cast<long long>(q) + static_cast<int32_t>(w[i]);
          if (s != static_cast<int32_t>(s)) err |= ZC_DERR_OVERFLOW;
          o[i] = static_cast<int32_t>(s);
          k.mz = max(k.mz, zigzag32(static_cast<int32_t>(s)));
        }
      }
      break;
    }
    case OUT_ADD_I32: {
      int32_t* o = static_cast<int32_t*>(k.out) + ob / 4;
      if (nb == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
        int4 a = __ldcg(reinterpret_cast<const int4*>(o));
        long long s0 = static_cast<long long>(a.x) + static_cast<int32_t>(w[0]);
        long long s1 = static_cast<long long>(a.y) + static_cast<int32_t>(w[1]);
        long long s2 = static_cast<long long>(a.z) + static_cast<int32_t>(w[2]);
        long long s3 = static_cast<long long>(a.w) + static_cast<int32_t>(w[3]);
        bool ovf = (s0 != static_cast<int32_t>(s0)) | (s1 != static_cast<int32_t>(s1)) |
                   (s2 != static_cast<int32_t>(s2)) | (s3 != static_cast<int32_t>(s3));
        if (ovf) err |= ZC_DERR_OVERFLOW;
        *reinterpret_cast<int4*>(o) = make_int4(static_cast<int32_t>(s0), static_cast<int32_t>(s1),
                                                static_cast<int32_t>(s2), static_cast<int32_t>(s3));
        k.mz = max(k.mz, max(max(zigzag32(static_cast<int32_t>(s0)), zigzag32(static_cast<int32_t>(s1))),
                             max(zigzag32(static_cast<int32_t>(s2)), zigzag32(static_cast<int32_t>(s3)))));
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (static_cast<uint32_t>(i) < nb / 4) {
            long long s = static_cast<long long>(o[i]) + static_cast<int32_t>(w[i]);
            if (s != static_cast<int32_t>(s)) err |= ZC_DERR_OVERFLOW;
            o[i] = static_cast<int32_t>(s);
            k.mz = max(k.mz, zigzag32(static_cast<int32_t>(s)));
          }
        }
      }
      break;
    }
    default: {
      uint8_t* o = static_cast<uint8_t*>(k.out) + ob;
      if (nb == 16 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
        *reinterpret_cast<uint4*>(o) = make_uint4(w[0], w[1], w[2], w[3]);
      } else {
#pragma unroll
        for (uint32_t j = 0; j < 16; ++j)
          if (j < nb) o[j] = static_cast<uint8_t>(w[j >> 2] >> (8 * (j & 3)));
      }
    }
  }
}

// 32 decoded raw bytes (8 symbol words) at raw offset ob: one 256-bit store per lane for the
// fp32 and byte sinks (a warp store of 32 lanes' rows at different grains touches 32 lines; 32-byte
// rows halve the store wavefronts of two 16-byte ones), emit16 twice otherwise.
__device__ __forceinline__ void emit32(const Sink& k, uint64_t ob, const uint32_t w[8], uint32_t& err) {
  if (k.kind == OUT_F32) {
    float* o = static_cast<float*>(k.out) + ob / 4;
    if ((reinterpret_cast<uintptr_t>(o) & 31) == 0) {
      float f[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = d2f_rn(__dmul_rn(k.scale, i2d(w[i])));
      asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o), "f"(f[0]), "f"(f[1]), "f"(f[2]),
                   "f"(f[3]), "f"(f[4]), "f"(f[5]), "f"(f[6]), "f"(f[7])
                   : "memory");
      return;
    }
  } else if (k.kind == OUT_BYTES) {
    uint8_t* o = static_cast<uint8_t*>(k.out) + ob;
    if ((reinterpret_cast<uintptr_t>(o) & 31) == 0) {
      asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                   "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                   : "memory");
      return;
    }
  }
  emit16(k, ob, w, 16, err);
  emit16(k, ob + 16, w + 4, 16, err);
}

// Header checks of recv_batch (collectives.cpp:313-321) and of the codec decoders' preambles
// (fixedlen.cpp:41-47, huffman.cpp:249-265).  hdr == nullptr: parse the header from the stage.
// bare: `hdr` describes a payload that starts at the stage (no header bytes, no raw fallback).
template <bool kCoherent>
__device__ __forceinline__ void check_frame(const uint8_t* stage, uint64_t region, uint64_t R, const zc_frame_header* hdr,
                                            bool bare, const DevHuff* ctx, bool have_index, FrameCheck& fc) {
  fc.need_seq = 0;
  fc.region = region;
  if (bare) {
    fc.h = *hdr;
  } else {
    if (region < kHeaderBytes) {
      fc.codec = kFallback;
      return;
    }
    uint64_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t lo = ld32<kCoherent>(reinterpret_cast<const uint32_t*>(stage) + 2 * i);
      uint32_t hi = ld32<kCoherent>(reinterpret_cast<const uint32_t*>(stage) + 2 * i + 1);
      w[i] = static_cast<uint64_t>(lo) | (static_cast<uint64_t>(hi) << 32);
    }
    fc.h = header_from_words(w);
    if (!validate_header(fc.h, region) || fc.h.raw_bytes != R) {
      fc.codec = kFallback;
      return;
    }
  }
  const zc_frame_header& h = fc.h;
  const uint64_t plen = bare ? region : h.payload_bytes;
  fc.codec = h.codec;
  if (h.codec == ZC_CODEC_FIXEDLEN) {
    uint32_t w = static_cast<uint32_t>(h.params);
    bool ok = !(w < 1 || w > 32 || h.params > 32) && h.raw_bytes != 0 && h.raw_bytes % 4 == 0 && R >= h.raw_bytes;
    if (ok) {
      uint64_t need = packed_bytes(h.raw_bytes / 4, w);
      ok = h.payload_bytes >= need && plen >= need;
    }
    if (!ok) fc.codec = kFallback;
  } else if (h.codec == ZC_CODEC_HUFFMAN) {
    bool ok = R >= h.raw_bytes && h.payload_bytes <= plen;
    if (ok) {
      if (h.flags & ZC_FLAG_EMBEDDED_CODEBOOK)
        ok = h.params == ZC_HUFF_CODEBOOK_BYTES && h.payload_bytes >= ZC_HUFF_CODEBOOK_BYTES;
      else
        ok = h.params == 0 && ctx != nullptr && ctx->valid;
    }
    if (!ok) fc.codec = kFallback;
    else if (!have_index) fc.need_seq = 1;
  } else if (h.codec == ZC_CODEC_RAW && bare) {
    fc.codec = kFallback;
  }
}

// Decodes a Huffman symbol run starting at `bitpos` into `n` bytes handed to put(j, byte).
// Mirrors huffman.cpp:281-314 with bits past the stream end reading as zero.  Returns false on
// an undecodable code or an overrun; *end receives the final bit position.
template <bool kCoherent, typename Put>
__device__ __forceinline__ bool huff_run(const DevHuff* t, const uint8_t* s, uint64_t slen, uint64_t bitpos, uint64_t n,
                                         uint64_t* end, Put put) {
  const uint64_t total = slen * 8;
  uint64_t wpos = bitpos >> 5;
  const uint32_t sh = static_cast<uint32_t>(bitpos & 31);
  unsigned long long acc = stream_word<kCoherent>(s, slen, wpos++) >> sh;
  uint32_t nbits = 32 - sh;
  for (uint64_t j = 0; j < n; ++j) {
    if (nbits < 32) {
      acc |= static_cast<unsigned long long>(stream_word<kCoherent>(s, slen, wpos++)) << nbits;
      nbits += 32;
    }
    const uint16_t e = t->lut[acc & ((1u << ZC_HUFF_ROOT_BITS) - 1)];
    uint32_t l = e >> 8;
    uint32_t sym = e & 0xFFu;
    if (l == 0) {
      const uint64_t avail = total > bitpos ? total - bitpos : 0;
      unsigned long long val = 0;
      uint32_t k = 0;
      bool found = false;
      while (k < t->max_len) {
        if (k >= avail) return false;
        val = (val << 1) | ((acc >> k) & 1ull);
        ++k;
        if (k >= t->min_len && t->count_at_len[k] > 0 && val >= t->first_code[k] &&
            val < t->first_code[k] + t->count_at_len[k]) {
          sym = t->sym_order[t->first_index[k] + static_cast<uint32_t>(val - t->first_code[k])];
          l = k;
          found = true;
          break;
        }
      }
      if (!found) return false;
    }
    if (bitpos + l > total) return false;
    acc >>= l;
    nbits -= l;
    bitpos += l;
    put(j, sym);
  }
  *end = bitpos;
  return true;
}

// Over-root code (the root LUT escaped): the canonical walk of huffman.cpp:293-306 resumed at
// length ROOT+1 — no code of length <= ROOT matches, or the LUT would have decoded it.  acc holds
// >= 32 valid bits.  Returns the code length (0: undecodable) and the symbol.
__device__ __forceinline__ uint32_t huff_long(const DevHuff* t, unsigned long long acc, uint32_t& sym) {
  unsigned long long val = __brev(static_cast<uint32_t>(acc) & ((1u << ZC_HUFF_ROOT_BITS) - 1)) >> (32 - ZC_HUFF_ROOT_BITS);
  for (uint32_t k = ZC_HUFF_ROOT_BITS + 1; k <= t->max_len; ++k) {
    val = (val << 1) | ((acc >> (k - 1)) & 1ull);
    const uint32_t c = t->count_at_len[k];
    const unsigned long long fc = t->first_code[k];
    if (c > 0 && val >= fc && val < fc + c) {
      sym = t->sym_order[t->first_index[k] + static_cast<uint32_t>(val - fc)];
      return k;
    }
  }
  return 0;
}

// One index grain of a Huffman stream (huffman.cpp:281-314), the throughput path: n raw bytes from
// bit `start`, 16 bytes at a time handed to emit16.  The bit reader keeps a 64-bit window topped
// up to >= 32 bits before every code, from a prefetched next stream word (its load is issued one
// top-up ahead, so no global load sits on the LUT -> shift chain).  The top-up is predicated, not
// a branch: the 32 lanes of a warp refill at different symbols.  The root LUT is read through a
// 32-bit shared-window address.  kChecked (grains near the frame end): stream bytes past the end
// read as zero, as in the reference.  Codes past the stream end are caught by the final position
// check: positions only grow, so any code crossing the end leaves *end > 8*slen.  Returns false
// on an undecodable code or an overrun.  s must be 4-byte aligned.
// kShort: every code fits the root LUT (max_len <= ROOT_BITS), so there is no over-root branch; a
// LUT entry of length 0 can then only be a pattern no code starts with, reported undecodable.
template <bool kCoherent, bool kChecked, bool kShort>
__device__ __forceinline__ bool huff_grain(const DevHuff* t, const uint8_t* s, uint64_t slen, uint64_t start, uint32_t n,
                                           const Sink& sink, uint64_t ob, uint64_t* end, uint32_t& err) {
  const uint32_t* ws = reinterpret_cast<const uint32_t*>(s);
  uint64_t wi = start >> 5;  // next word to prefetch
  auto word = [&](uint64_t i) -> uint32_t {
    if (kChecked) return stream_word<kCoherent>(s, slen, i);
    if (kCoherent) return __ldcg(ws + i);
    uint32_t v;
    asm volatile("ld.global.nc.L2::256B.u32 %0, [%1];" : "=r"(v) : "l"(ws + i));
    return v;
  };
  if (!kChecked) {  // the grain's stream (~1 KiB at most for codes <= 8 bits) into L2 ahead of the reader
    const uint8_t* g0 = s + ((start >> 3) & ~static_cast<uint64_t>(127));
#pragma unroll
    for (int k = 1; k < 8; ++k) asm volatile("prefetch.global.L2 [%0];" ::"l"(g0 + 128 * k));
  }
  const uint32_t lut = static_cast<uint32_t>(__cvta_generic_to_shared(t->lut));
  unsigned long long acc = word(wi++);
  uint32_t nw = word(wi++);
  acc >>= (start & 31);
  uint32_t nb = 32 - static_cast<uint32_t>(start & 31);
  bool ok = true;
  auto sym1 = [&]() -> uint32_t {
    if (nb < 32) {
      acc |= static_cast<unsigned long long>(nw) << nb;
      nb += 32;
      nw = word(wi++);
    }
    uint32_t e;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(e) : "r"(lut + 2u * static_cast<uint32_t>(acc & ((1u << ZC_HUFF_ROOT_BITS) - 1))));
    uint32_t l = e >> 8, sym = e & 0xFFu;
    if (kShort) {
      ok &= l != 0;
      l = l ? l : 1u;  // keep the reader moving; the grain is reported undecodable
    } else if (l == 0) {
      l = huff_long(t, acc, sym);
      if (l == 0) {
        ok = false;
        l = 1;  // keep the reader moving; the grain is reported undecodable
      }
    }
    acc >>= l;
    nb -= l;
    return sym;
  };
  const uint32_t ng = n / 16;
  for (uint32_t gq = 0; gq < ng; ++gq) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t o = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) o |= sym1() << (8 * k);
      w[q] = o;
    }
    emit16(sink, ob + 16ull * gq, w, 16, err);
  }
  if (n & 15) {
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (uint32_t j = 0; j < 16; ++j)
      if (j < (n & 15)) w[j >> 2] |= sym1() << (8 * (j & 3));
    emit16(sink, ob + 16ull * ng, w, n & 15, err);
  }
  // words [start>>5, wi-1) have entered the window; nb of their bits are unconsumed
  const uint64_t pos = (wi - 1) * 32 - nb;
  *end = pos;
  return ok && pos <= slen * 8;
}

// ---- warp-staged short-code grain decoder (max code length <= ROOT_BITS; the throughput path)
//
// huff_grain above reads each lane's stream with its own loads: a warp load touches 32 lines, and
// a predicated refill waits (per-warp scoreboard) on the load another lane issued one symbol ago,
// so L2 latency sits on the chain.  Here the warp decodes its 32 grains in rounds of 32 symbols
// per lane.  Each round first stages every lane's next 16 stream words (>= the 31 + 32 x 12 + 64
// bits a round can touch) into a per-warp shared window with cooperative loads (one warp load =
// two lanes' 64-byte windows), then each lane decodes groups of 4 codes from a 64-bit funnel of
// its window (4 x 12 <= 48 bits: no refill inside a group).  The root LUT is read through a copy
// whose u16 slots are XOR-swizzled by the index's high bits: the low index bits are the next
// code's bits, highly skewed for short codes, and would otherwise pile the warp's lookups onto a
// few banks.
constexpr int kHWinWords = 16;   // staged words per lane and round
constexpr int kHWinPitch = 33;   // words between a window's word k and k+1 (bank = k + lane)
constexpr uint32_t kHuffWarpScratchWords = kHWinWords * kHWinPitch;  // per warp

__device__ __forceinline__ uint32_t lut_swz(uint32_t i) { return i ^ ((i >> 6) & 0x3eu); }

// Swizzled copy of t->lut into slut (all threads call; synchronises).
__device__ __forceinline__ void swizzle_lut(const DevHuff* t, uint16_t* slut) {
  for (uint32_t i = threadIdx.x; i < (1u << ZC_HUFF_ROOT_BITS); i += blockDim.x) slut[lut_swz(i)] = t->lut[i];
  __syncthreads();
}

// All 32 lanes call.  Lanes with n == 0 only help stage windows.  Lanes with n > 0 decode n
// symbols (n a multiple of 32) from bit `start`, handing 16 bytes at a time to emit16 at ob.
// Returns per lane: false on an undecodable code; *end = the final bit position.
template <bool kCoherent>
__device__ __forceinline__ bool huff_grain_warp(const uint16_t* slut, const uint8_t* s, uint64_t slen, uint32_t start,
                                                uint32_t n, const Sink& sink, uint64_t ob, uint32_t* win, uint32_t* end,
                                                uint32_t& err) {
  const int lane = threadIdx.x & 31;
  const uint32_t* ws = reinterpret_cast<const uint32_t*>(s);
  const uint64_t full_words = slen / 4;
  const uint32_t rounds = __reduce_max_sync(0xffffffffu, n) / 32;
  const uint32_t my_rounds = n / 32;
  const uint32_t lut = static_cast<uint32_t>(__cvta_generic_to_shared(slut));
  const uint32_t wsh = static_cast<uint32_t>(__cvta_generic_to_shared(win)) + 4u * lane;
  uint32_t pos = start;
  uint32_t emin = 0xffffu;
  for (uint32_t r = 0; r < rounds; ++r) {
    // stage: load j serves owners j and j+16, word (lane & 15) of each window (shared-memory banks
    // k + owner: the two half-warps' banks are disjoint)
    const uint32_t wbase = pos >> 5;
    uint32_t v[kHWinWords];
    if (__reduce_max_sync(0xffffffffu, wbase) + kHWinWords <= full_words) {  // the whole warp in bounds
      const uint32_t* wl = ws + (lane & 15);
#pragma unroll
      for (int j = 0; j < kHWinWords; ++j) v[j] = ld32<kCoherent>(wl + __shfl_sync(0xffffffffu, wbase, j + 16 * (lane >> 4)));
    } else {
#pragma unroll
      for (int j = 0; j < kHWinWords; ++j) {
        const uint64_t w = static_cast<uint64_t>(__shfl_sync(0xffffffffu, wbase, j + 16 * (lane >> 4))) + (lane & 15);
        v[j] = w < full_words ? ld32<kCoherent>(ws + w) : stream_word<kCoherent>(s, slen, w);
      }
    }
    __syncwarp();  // the previous round's reads of the window are done
#pragma unroll
    for (int j = 0; j < kHWinWords; ++j) win[(lane & 15) * kHWinPitch + j + 16 * (lane >> 4)] = v[j];
    __syncwarp();
    if (r < my_rounds) {
      uint32_t o = pos & 31;  // bit offset from window word 0
      uint32_t w8[8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t* w4 = w8 + 4 * h;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t a = wsh + 4u * kHWinPitch * (o >> 5);
          uint32_t x0, x1, x2;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x0) : "r"(a));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x1) : "r"(a + 4u * kHWinPitch));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x2) : "r"(a + 8u * kHWinPitch));
          const uint32_t sh = o & 31;
          unsigned long long acc = (static_cast<unsigned long long>(__funnelshift_r(x1, x2, sh)) << 32) |
                                   __funnelshift_r(x0, x1, sh);
          uint32_t word = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t e;
            asm volatile("ld.shared.u16 %0, [%1];"
                         : "=r"(e)
                         : "r"(lut + 2u * lut_swz(static_cast<uint32_t>(acc) & ((1u << ZC_HUFF_ROOT_BITS) - 1))));
            const uint32_t l = e >> 8;
            emin = min(emin, e);
            acc >>= l;
            o += l;
            word = __byte_perm(word, e, k == 0 ? 0x3214u : k == 1 ? 0x3240u : k == 2 ? 0x3410u : 0x4210u);
          }
          w4[q] = word;
        }
      }
      emit32(sink, ob + 32ull * r, w8, err);
      pos = (pos & ~31u) + o;
    }
  }
  *end = pos;
  // a LUT entry of length 0 (no code starts with the pattern): undecodable; codes past the
  // stream end (read as zero bits) leave pos beyond it
  return emin >= 256u && pos <= slen * 8;
}

// Decode tables for a Huffman frame into shared memory: the embedded codebook rebuilt (with the
// reference's validation) or a copy of the shared context.  All threads call.
template <bool kCoherent>
__device__ __forceinline__ bool load_huff_tables(const FrameCheck& fc, const uint8_t* payload, const DevHuff* g,
                                                 DevHuff* t, uint32_t* flag, uint8_t* lens_tmp) {
  if (fc.h.flags & ZC_FLAG_EMBEDDED_CODEBOOK) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lens_tmp[i] = ld8<kCoherent>(payload + i);
    __syncthreads();
    return cta_decode_tables(lens_tmp, t, flag);
  }
  for (int i = threadIdx.x; i < (1 << ZC_HUFF_ROOT_BITS); i += blockDim.x) t->lut[i] = g->lut[i];
  if (threadIdx.x < 256) t->sym_order[threadIdx.x] = g->sym_order[threadIdx.x];
  if (threadIdx.x < 33) {
    t->count_at_len[threadIdx.x] = g->count_at_len[threadIdx.x];
    t->first_index[threadIdx.x] = g->first_index[threadIdx.x];
    t->first_code[threadIdx.x] = g->first_code[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    t->min_len = g->min_len;
    t->max_len = g->max_len;
    t->valid = g->valid;
  }
  __syncthreads();
  return true;
}

// Decodes vectors [v0, v1) (16-byte units of raw output) of one checked frame into `sink` at raw
// offset obase.  Every thread of the CTA calls (uniform control flow).  FixedLen/RAW/fallback
// are streaming; Huffman runs one thread per 1 KiB grain from the companion index (v0 must be a
// multiple of 64).  Returns flag bits for the caller: 1 = index inconsistent with the payload,
// 2 = undecodable Huffman stream.  words: >= 32 * nwarps * ... per-warp scratch of 136 words.
template <bool kCoherent, int kDecU>
__device__ inline uint32_t decode_slice(const FrameCheck& fc, const uint8_t* payload, uint64_t R, uint64_t v0, uint64_t v1,
                                 const Sink& sink, uint64_t obase, const uint32_t* idx, const DevHuff* ctx,
                                 DevHuff* s_t, uint32_t* s_flag, uint8_t* s_lens_tmp, uint32_t* s_words,
                                 uint32_t& err, uint32_t* s_hscratch = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  uint32_t flags = 0;
  const uint32_t codec = fc.codec;
  if (codec == kFallback) {
    // raw-copy fallback (collectives.cpp:330-336): the payload region verbatim, min(dst, have)
    const uint64_t have = fc.region > kHeaderBytes ? fc.region - kHeaderBytes : 0;
    const uint64_t lim = R < have ? R : have;
    for (uint64_t v = v0 + tid; v < v1; v += nthr) {
      if (v * 16 >= lim) break;
      uint32_t nb = static_cast<uint32_t>(lim - v * 16 < 16 ? lim - v * 16 : 16);
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = stream_word<kCoherent>(payload, lim, v * 4 + k);
      emit16(sink, obase + v * 16, w, nb, err);
    }
  } else if (codec == ZC_CODEC_RAW) {
    for (uint64_t v = v0 + tid; v < v1; v += nthr) {
      uint32_t nb = static_cast<uint32_t>(R - v * 16 < 16 ? R - v * 16 : 16);
      uint32_t w[4];
      if (nb == 16) {
        uint4 x = ld128<kCoherent>(reinterpret_cast<const uint4*>(payload) + v);
        w[0] = x.x;
        w[1] = x.y;
        w[2] = x.z;
        w[3] = x.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = stream_word<kCoherent>(payload, R, v * 4 + k);
      }
      emit16(sink, obase + v * 16, w, nb, err);
    }
  } else if (codec == ZC_CODEC_FIXEDLEN) {
    // A chunk of 128 symbols occupies exactly 4*width payload words.  Each warp stages U chunks'
    // words in shared memory (every lane issues its <= 5 loads per chunk before any is used),
    // then each lane extracts its 4 symbols per chunk with a 64-bit funnel read.
    const uint32_t width = static_cast<uint32_t>(fc.h.params);
    const uint32_t w4 = 4 * width;
    const uint64_t P = fc.h.payload_bytes;
    const unsigned long long mask = width == 32 ? 0xffffffffull : ((1ull << width) - 1);
    uint32_t* sw = s_words + warp * 136 * kDecU;
    const uint64_t nwarps = nthr / 32;
    for (uint64_t c0 = v0 / 32 + warp; c0 * 32 < v1; c0 += nwarps * kDecU) {
      uint32_t t[kDecU][5];
#pragma unroll
      for (int k = 0; k < kDecU; ++k) {
        const uint64_t gw0 = (c0 + k * nwarps) * w4;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const uint32_t kk = lane + 32 * j;
          const uint64_t g = gw0 + kk;
          t[k][j] = 0;
          if (kk <= w4 && (c0 + k * nwarps) * 32 < v1) {
            if (g * 4 + 4 <= P) t[k][j] = ld32<kCoherent>(reinterpret_cast<const uint32_t*>(payload) + g);
            else t[k][j] = stream_word<kCoherent>(payload, P, g);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kDecU; ++k)
#pragma unroll
        for (int j = 0; j < 5; ++j)
          if (lane + 32 * j <= w4) sw[k * 136 + lane + 32 * j] = t[k][j];
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kDecU; ++k) {
        const uint64_t v = (c0 + k * nwarps) * 32 + lane;
        if (v < v1) {
          const uint32_t* s = sw + k * 136;
          uint32_t w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t bit = (lane * 4 + q) * width;
            const uint32_t wi = bit >> 5, sh = bit & 31;
            unsigned long long x = (static_cast<unsigned long long>(s[wi + 1]) << 32) | s[wi];
            w[q] = static_cast<uint32_t>(unzigzag32(static_cast<uint32_t>((x >> sh) & mask)));
          }
          uint32_t nb = static_cast<uint32_t>(R - v * 16 < 16 ? R - v * 16 : 16);
          emit16(sink, obase + v * 16, w, nb, err);
        }
      }
      __syncwarp();
    }
  } else if (codec == ZC_CODEC_HUFFMAN && !fc.need_seq) {
    const bool ok = load_huff_tables<kCoherent>(fc, payload, ctx, s_t, s_flag, s_lens_tmp);
    const bool emb = (fc.h.flags & ZC_FLAG_EMBEDDED_CODEBOOK) != 0;
    if (!ok) {
      flags |= 2u;
    } else {
      const uint8_t* s = payload + (emb ? ZC_HUFF_CODEBOOK_BYTES : 0);
      const uint64_t slen = fc.h.payload_bytes - (emb ? ZC_HUFF_CODEBOOK_BYTES : 0);
      const uint64_t Rh = fc.h.raw_bytes;
      const uint64_t ngr = (Rh + kIndexGrain - 1) / kIndexGrain;
      const uint64_t g0 = v0 / 64, g1 = min(ngr, (v1 + 63) / 64);
      const bool shortc = s_t->max_len <= ZC_HUFF_ROOT_BITS;
      const bool aligned = (reinterpret_cast<uintptr_t>(s) & 3) == 0;
      uint64_t gseq = g0;  // grains from here on run the per-lane decoder
      if (s_hscratch != nullptr && shortc && aligned) {
        // warp-staged decoder for every full grain; the unit's partial last grain (if any) after
        uint16_t* slut = reinterpret_cast<uint16_t*>(s_hscratch);
        uint32_t* win = s_hscratch + (1u << ZC_HUFF_ROOT_BITS) / 2 + warp * kHuffWarpScratchWords;
        swizzle_lut(s_t, slut);
        const uint64_t gfull = min(g1, Rh / kIndexGrain);
        for (uint64_t gb = g0 + warp * 32; gb < gfull; gb += nthr) {
          const uint64_t g = gb + lane;
          const bool mine = g < gfull;
          const uint32_t start = mine ? ld32<kCoherent>(idx + g) : 0u;
          uint32_t endb = 0;
          const bool good = huff_grain_warp<kCoherent>(slut, s, slen, start, mine ? kIndexGrain : 0u, sink,
                                                       obase + g * kIndexGrain, win, &endb, err);
          if (mine) {
            if (!good) flags |= 2u;
            else if (g + 1 < ngr && endb != ld32<kCoherent>(idx + g + 1)) flags |= 1u;
          }
        }
        gseq = max(g0, gfull);
      }
      for (uint64_t g = gseq + tid; g < g1; g += nthr) {
        const uint64_t b0 = g * kIndexGrain;
        const uint64_t n = Rh - b0 < kIndexGrain ? Rh - b0 : kIndexGrain;
        unsigned long long lo = 0, hi = 0;
        uint64_t endb = 0;
        const uint64_t start = ld32<kCoherent>(idx + g);
        bool good;
        // unchecked 16-byte reads only where even a corrupt grain cannot leave the payload: a
        // grain consumes <= 1024 codes x 32 bits, the reader runs <= 384 bits ahead
        if (aligned && start + 32768 + 1024 <= slen * 8)
          good = shortc ? huff_grain<kCoherent, false, true>(s_t, s, slen, start, static_cast<uint32_t>(n), sink, obase + b0, &endb, err)
                        : huff_grain<kCoherent, false, false>(s_t, s, slen, start, static_cast<uint32_t>(n), sink, obase + b0, &endb, err);
        else if (aligned)
          good = huff_grain<kCoherent, true, false>(s_t, s, slen, start, static_cast<uint32_t>(n), sink, obase + b0, &endb, err);
        else good = huff_run<kCoherent>(s_t, s, slen, start, n, &endb, [&](uint64_t j, uint32_t sym) {
          const uint32_t k = static_cast<uint32_t>(j & 15);
          if (k < 8) lo |= static_cast<unsigned long long>(sym) << (8 * k);
          else hi |= static_cast<unsigned long long>(sym) << (8 * (k - 8));
          if (k == 15 || j + 1 == n) {
            uint32_t ww[4] = {static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32), static_cast<uint32_t>(hi),
                              static_cast<uint32_t>(hi >> 32)};
            emit16(sink, obase + b0 + (j & ~15ull), ww, k + 1, err);
            lo = hi = 0;
          }
        });
        if (!good) flags |= 2u;
        else if (g + 1 < ngr && endb != ld32<kCoherent>(idx + g + 1)) flags |= 1u;
      }
    }
  }
  return flags;
}

}  // namespace zc
