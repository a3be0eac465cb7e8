// zc_encode_common.cuh — device helpers shared by the encode kernels (zc_encode.cu: cluster
// kernels for the ring steps and single-frame API calls; zc_tasks.cu: the persistent task kernel
// of the batched hot path).  Reference paths are relative to /root/reference/proj/core/.
#pragma once
#include <cooperative_groups.h>

#include "zc_decode.cuh"
#include "zc_kernels.h"

namespace zc {
namespace {
constexpr int CL = 8;     // CTAs per cluster (= per frame unit)
constexpr int NT = 512;   // threads per CTA
constexpr int NW = NT / 32;
constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t CODEC_NONE = 0xFFu;
constexpr int TILE_WORDS = NT * 16 + 64;  // Huffman tile: NT vectors x 16 bytes x <= 32 bits
constexpr uint64_t SLICE_ALIGN = 64;      // CTA slices in 16-byte vectors: 1 KiB Huffman grains

struct Bound {
  unsigned long long head_idx, tail_idx;
  uint32_t head_val, tail_val, has_head, has_tail;
};

struct Ctrl {
  uint32_t maxzz, wmaxzz, zero_len, go;  // per-CTA partials; go: CTA 0's wait verdict
  uint32_t bad, dirty;                   // float sources: any Inf/NaN seen (slice; unit, CTA 0)
  double fmin, fmax;                     // float sources: value range of the slice
  unsigned long long bits;
  uint32_t codec, width, pending, _p;    // decision (CTA 0)
  unsigned long long payload;
  unsigned long long rx_len;
  unsigned long long slice_base[CL];
};

union __align__(16) Scratch {
  uint32_t tile[TILE_WORDS];
  uint4 zz[NW][256];  // FixedLen: per warp, 1024 zig-zag symbols as 256 swizzled 16-byte slots
  struct {
    unsigned long long keys[256];
    unsigned long long w[512];
    int parent[512];
    uint8_t depth[512];
  } tree;
  struct {
    DevHuff t;
    uint32_t words[NW * 136 * 2];
  } dec;
};

__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ------------------------------------------------------------------ ring flag protocol
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_err(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Spins until *f >= v.  Gives up (false) when any rank has raised an error bit (the poison of
// transport.cpp:90-95) or after the timeout, which it raises itself.
__device__ bool wait_geq(const unsigned long long* f, unsigned long long v, const Link& L) {
  const unsigned long long t0 = globaltimer();
  for (uint32_t it = 0;; ++it) {
    if (ld_acquire_sys(f) >= v) return true;
    if (ld_err(L.err_self) != 0) return false;
    if ((it & 255) == 255 && globaltimer() - t0 > L.timeout_ns) {
      for (uint32_t r = 0; r < L.nranks; ++r) atomicOr(L.err_all[r], ZC_DERR_TIMEOUT);
      return false;
    }
    __nanosleep(32);
  }
}

__device__ __forceinline__ void broadcast_err(const Link& L, uint32_t err) {
  for (uint32_t r = 0; r < L.nranks; ++r) atomicOr(L.err_all[r], err);
}

__device__ __forceinline__ void wire_add(zc_wire_stats* w, uint32_t codec, uint64_t raw, uint64_t payload,
                                         uint64_t index_bytes) {
  atomicAdd(reinterpret_cast<unsigned long long*>(&w->frames_by_codec[codec]), 1ull);
  atomicAdd(reinterpret_cast<unsigned long long*>(&w->raw_bytes), static_cast<unsigned long long>(raw));
  atomicAdd(reinterpret_cast<unsigned long long*>(&w->payload_bytes), static_cast<unsigned long long>(payload));
  atomicAdd(reinterpret_cast<unsigned long long*>(&w->total_bytes), static_cast<unsigned long long>(payload + kHeaderBytes));
  if (index_bytes) atomicAdd(reinterpret_cast<unsigned long long*>(&w->index_bytes), static_cast<unsigned long long>(index_bytes));
}

// Loads raw vector v (16 bytes) of the unit: bytes [16v, 16v+16) ∩ [0, R).  Float sources are
// quantized here (4 elements -> 4 int32 symbols).  Missing bytes are zero; nb = valid bytes.
// kCoh: the source was written earlier in this kernel (ring mode), so bypass the read-only path.
template <int SRC, bool kCoh>
__device__ __forceinline__ void load_vec(const EncParams& p, uint64_t uoff, uint64_t R, uint64_t v, uint32_t w[4],
                                         uint32_t& nb, uint32_t& err) {
  const uint64_t b0 = v * 16;
  nb = static_cast<uint32_t>(R - b0 < 16 ? R - b0 : 16);
  if (SRC == SRC_BYTES) {
    const uint8_t* s = static_cast<const uint8_t*>(p.src) + uoff + b0;
    if (nb == 16 && aligned16(s)) {
      uint4 x = ld128<kCoh>(reinterpret_cast<const uint4*>(s));
      w[0] = x.x;
      w[1] = x.y;
      w[2] = x.z;
      w[3] = x.w;
    } else {
      w[0] = w[1] = w[2] = w[3] = 0;
#pragma unroll
      for (uint32_t j = 0; j < 16; ++j)
        if (j < nb) w[j >> 2] |= static_cast<uint32_t>(ld8<kCoh>(s + j)) << (8 * (j & 3));
    }
  } else if (SRC == SRC_F32) {
    const float* s = static_cast<const float*>(p.src) + (uoff + b0) / 4;
    float f[4] = {0.f, 0.f, 0.f, 0.f};
    if (nb == 16 && aligned16(s)) {
      float4 x = __ldg(reinterpret_cast<const float4*>(s));
      f[0] = x.x;
      f[1] = x.y;
      f[2] = x.z;
      f[3] = x.w;
    } else {
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j)
        if (j < nb / 4) f[j] = __ldg(s + j);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = (static_cast<uint32_t>(k) < nb / 4)
                 ? static_cast<uint32_t>(quantize_one(static_cast<double>(f[k]), enc_scale(p), enc_rcp(p), err))
                 : 0u;
  } else {
    const double* s = static_cast<const double*>(p.src) + (uoff + b0) / 4;
    double f[4] = {0.0, 0.0, 0.0, 0.0};
    if (nb == 16 && aligned16(s)) {
      double2 a = __ldg(reinterpret_cast<const double2*>(s));
      double2 b = __ldg(reinterpret_cast<const double2*>(s) + 1);
      f[0] = a.x;
      f[1] = a.y;
      f[2] = b.x;
      f[3] = b.y;
    } else {
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j)
        if (j < nb / 4) f[j] = __ldg(s + j);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = (static_cast<uint32_t>(k) < nb / 4) ? static_cast<uint32_t>(quantize_one(f[k], enc_scale(p), enc_rcp(p), err)) : 0u;
  }
}

__device__ __forceinline__ uint32_t byte_of(const uint32_t w[4], uint32_t j) {
  return (w[j >> 2] >> (8 * (j & 3))) & 0xFFu;
}

__device__ __forceinline__ void store_word_safe(uint8_t* payload, uint64_t gw, uint32_t val, uint64_t limit);

// A 16-byte raw-output vector's worth of source data, fetched ahead of use so that several loads
// are in flight per thread (the kernel runs one 16-warp CTA per SM).
struct RawVec {
  uint4 a, b;  // b only for f64 sources (4 doubles)
  uint32_t nb;
};

template <int SRC, bool kCoh>
__device__ __forceinline__ void fetch(const EncParams& p, uint64_t uoff, uint64_t R, uint64_t v, RawVec& rv) {
  const uint64_t b0 = v * 16;
  rv.nb = static_cast<uint32_t>(R - b0 < 16 ? R - b0 : 16);
  if (SRC == SRC_BYTES) {
    const uint8_t* s = static_cast<const uint8_t*>(p.src) + uoff + b0;
    if (rv.nb == 16 && aligned16(s)) {
      rv.a = ld128<kCoh>(reinterpret_cast<const uint4*>(s));
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (uint32_t j = 0; j < 16; ++j)
        if (j < rv.nb) w[j >> 2] |= static_cast<uint32_t>(ld8<kCoh>(s + j)) << (8 * (j & 3));
      rv.a = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else if (SRC == SRC_F32) {
    const float* s = static_cast<const float*>(p.src) + (uoff + b0) / 4;
    if (rv.nb == 16 && aligned16(s)) {
      rv.a = __ldg(reinterpret_cast<const uint4*>(s));
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j)
        if (j < rv.nb / 4) w[j] = __float_as_uint(__ldg(s + j));
      rv.a = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
    const double* s = static_cast<const double*>(p.src) + (uoff + b0) / 4;
    if (rv.nb == 16 && aligned16(s)) {
      rv.a = __ldg(reinterpret_cast<const uint4*>(s));
      rv.b = __ldg(reinterpret_cast<const uint4*>(s) + 1);
    } else {
      double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j)
        if (j < rv.nb / 4) d[j] = __ldg(s + j);
      rv.a = make_uint4(__double2loint(d[0]), __double2hiint(d[0]), __double2loint(d[1]), __double2hiint(d[1]));
      rv.b = make_uint4(__double2loint(d[2]), __double2hiint(d[2]), __double2loint(d[3]), __double2hiint(d[3]));
    }
  }
}

template <int SRC>
__device__ __forceinline__ double element(const RawVec& rv, int k) {
  if (SRC == SRC_F32) {
    const uint32_t u = k == 0 ? rv.a.x : k == 1 ? rv.a.y : k == 2 ? rv.a.z : rv.a.w;
    return static_cast<double>(__uint_as_float(u));
  }
  const uint32_t lo = k == 0 ? rv.a.x : k == 1 ? rv.a.z : k == 2 ? rv.b.x : rv.b.z;
  const uint32_t hi = k == 0 ? rv.a.y : k == 1 ? rv.a.w : k == 2 ? rv.b.y : rv.b.w;
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

// Symbol words of a fetched vector (quantizing float sources; invalid tail elements -> 0).
template <int SRC>
__device__ __forceinline__ void to_words(const EncParams& p, const RawVec& rv, uint32_t w[4], uint32_t& err) {
  if (SRC == SRC_BYTES) {
    w[0] = rv.a.x;
    w[1] = rv.a.y;
    w[2] = rv.a.z;
    w[3] = rv.a.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = static_cast<uint32_t>(k) < rv.nb / 4
                 ? static_cast<uint32_t>(quantize_one(element<SRC>(rv, k), enc_scale(p), enc_rcp(p), err))
                 : 0u;
  }
}

// L2 eviction-priority hints for a read that will be re-read soon (kPolKeep: the scan pass of the
// task kernel) and for its last read (kPolDrop: the encode pass), so the slices in flight between
// the two passes stay resident in L2 instead of competing with the stream.
enum : int { kPolNone = 0, kPolKeep = 1, kPolDrop = 2 };
template <int kPol>
__device__ __forceinline__ uint4 ld128_pol(const uint4* p) {
  if (kPol == kPolNone) return __ldg(p);
  uint64_t pol;
  if (kPol == kPolKeep)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

// Full 16-byte vector at an aligned source (no tail / alignment checks).
template <int SRC, bool kCoh, int kPol = kPolNone>
__device__ __forceinline__ void fetch_full(const EncParams& p, uint64_t uoff, uint64_t v, RawVec& rv) {
  rv.nb = 16;
  if (SRC == SRC_BYTES) {
    if (kCoh)
      rv.a = ld128<kCoh>(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(p.src) + uoff) + v);
    else
      rv.a = ld128_pol<kPol>(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(p.src) + uoff) + v);
  } else if (SRC == SRC_F32) {
    rv.a = ld128_pol<kPol>(reinterpret_cast<const uint4*>(static_cast<const float*>(p.src) + uoff / 4) + v);
  } else {
    const uint4* s = reinterpret_cast<const uint4*>(static_cast<const double*>(p.src) + uoff / 4) + 2 * v;
    rv.a = ld128_pol<kPol>(s);
    rv.b = ld128_pol<kPol>(s + 1);
  }
}

// Symbols of a full vector of FINITE values: branch-free fast quantizer, exact redo (rare) when
// any element sits near a rounding tie.
template <int SRC>
__device__ __forceinline__ void words_full(const EncParams& p, const RawVec& rv, uint32_t w[4], uint32_t& err) {
  if (SRC == SRC_BYTES) {
    w[0] = rv.a.x;
    w[1] = rv.a.y;
    w[2] = rv.a.z;
    w[3] = rv.a.w;
  } else {
    bool slow = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = static_cast<uint32_t>(quantize_fast(element<SRC>(rv, k), enc_rcp(p), slow));
    if (slow) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[k] = static_cast<uint32_t>(quantize_one(element<SRC>(rv, k), enc_scale(p), enc_rcp(p), err));
    }
  }
}

// Running value range of float sources.  fp32: FMNMX in the float domain (no conversion per
// element) and the max of the magnitude bits, which reaches 0x7f800000 iff an Inf/NaN was seen.
struct Range {
  float fmn = __builtin_huge_valf(), fmx = -__builtin_huge_valf();
  uint32_t absbits = 0;
  double dmn = __builtin_huge_val(), dmx = -__builtin_huge_val();
  uint32_t bad = 0;
};

template <int SRC>
__device__ __forceinline__ void minmax_full(const RawVec& rv, Range& g) {
  if (SRC == SRC_F32) {
    const uint32_t u[4] = {rv.a.x, rv.a.y, rv.a.z, rv.a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      g.fmn = fminf(g.fmn, __uint_as_float(u[k]));
      g.fmx = fmaxf(g.fmx, __uint_as_float(u[k]));
      g.absbits = max(g.absbits, u[k] & 0x7fffffffu);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double d = element<SRC>(rv, k);
      g.bad |= (__double2hiint(d) & 0x7ff00000) == 0x7ff00000 ? 1u : 0u;
      g.dmn = fmin(g.dmn, d);
      g.dmx = fmax(g.dmx, d);
    }
  }
}

template <int SRC>
__device__ __forceinline__ void minmax_vec(const RawVec& rv, Range& g) {
  if (SRC == SRC_F32) {
    const uint32_t u[4] = {rv.a.x, rv.a.y, rv.a.z, rv.a.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (static_cast<uint32_t>(k) < rv.nb / 4) {
        const float f = __uint_as_float(u[k]);
        g.fmn = fminf(g.fmn, f);
        g.fmx = fmaxf(g.fmx, f);
        g.absbits = max(g.absbits, u[k] & 0x7fffffffu);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (static_cast<uint32_t>(k) < rv.nb / 4) {
        const double d = element<SRC>(rv, k);
        if ((__double2hiint(d) & 0x7ff00000) == 0x7ff00000) g.bad = 1;
        g.dmn = fmin(g.dmn, d);
        g.dmx = fmax(g.dmx, d);
      }
    }
  }
}

// Packs 32 consecutive zig-zag symbols at compile-time width W into exactly W LSB-first words
// (fixedlen.cpp:26-34) and stores them at payload word `wb`; never writes at or past byte P.
template <int W>
__device__ __forceinline__ void pack_store(const uint32_t (&z)[32], uint8_t* payload, uint64_t wb, uint64_t P) {
  uint32_t o[W];
  unsigned long long acc = 0;
  int nb = 0, k = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    acc |= static_cast<unsigned long long>(z[i]) << nb;
    nb += W;
    if (nb >= 32) {
      o[k++] = static_cast<uint32_t>(acc);
      acc >>= 32;
      nb -= 32;
    }
  }
  uint32_t* dst = reinterpret_cast<uint32_t*>(payload) + wb;
  if ((wb + W) * 4 <= P) {
    if (W % 4 == 0) {
#pragma unroll
      for (int j = 0; j < W / 4; ++j) reinterpret_cast<uint4*>(dst)[j] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
    } else if (W % 2 == 0 && (wb & 1) == 0) {
#pragma unroll
      for (int j = 0; j < W / 2; ++j) reinterpret_cast<uint2*>(dst)[j] = make_uint2(o[2 * j], o[2 * j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) dst[j] = o[j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j)
      if ((wb + j) * 4 < P) store_word_safe(payload, wb + j, o[j], P);
  }
}

__device__ __forceinline__ void pack_store_w(uint32_t width, const uint32_t (&z)[32], uint8_t* payload, uint64_t wb,
                                          uint64_t P) {
  switch (width) {
#define ZC_PACK_CASE(W) \
  case W:               \
    pack_store<W>(z, payload, wb, P); \
    break;
    ZC_PACK_CASE(1) ZC_PACK_CASE(2) ZC_PACK_CASE(3) ZC_PACK_CASE(4) ZC_PACK_CASE(5) ZC_PACK_CASE(6)
    ZC_PACK_CASE(7) ZC_PACK_CASE(8) ZC_PACK_CASE(9) ZC_PACK_CASE(10) ZC_PACK_CASE(11) ZC_PACK_CASE(12)
    ZC_PACK_CASE(13) ZC_PACK_CASE(14) ZC_PACK_CASE(15) ZC_PACK_CASE(16) ZC_PACK_CASE(17) ZC_PACK_CASE(18)
    ZC_PACK_CASE(19) ZC_PACK_CASE(20) ZC_PACK_CASE(21) ZC_PACK_CASE(22) ZC_PACK_CASE(23) ZC_PACK_CASE(24)
    ZC_PACK_CASE(25) ZC_PACK_CASE(26) ZC_PACK_CASE(27) ZC_PACK_CASE(28) ZC_PACK_CASE(29) ZC_PACK_CASE(30)
    ZC_PACK_CASE(31) ZC_PACK_CASE(32)
#undef ZC_PACK_CASE
    default:
      break;
  }
}

// Stores one 32-bit word of the payload at byte offset 4*gw, never past `limit` payload bytes.
__device__ __forceinline__ void store_word_safe(uint8_t* payload, uint64_t gw, uint32_t val, uint64_t limit) {
  uint64_t b = gw * 4;
  if (b + 4 <= limit) {
    reinterpret_cast<uint32_t*>(payload)[gw] = val;
  } else {
    for (uint32_t j = 0; j < 4 && b + j < limit; ++j) payload[b + j] = static_cast<uint8_t>(val >> (8 * j));
  }
}

template <typename T>
__device__ __forceinline__ T block_reduce_max(T v, T* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = red[0];
  for (int i = 1; i < NW; ++i) r = max(r, red[i]);
  return r;
}

__device__ __forceinline__ double block_reduce_fmin(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < NW; ++i) r = fmin(r, red[i]);
  return r;
}

__device__ __forceinline__ double block_reduce_fmax(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = red[0];
  for (int i = 1; i < NW; ++i) r = fmax(r, red[i]);
  return r;
}

__device__ __forceinline__ unsigned long long block_reduce_sum(unsigned long long v, unsigned long long* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  unsigned long long r = 0;
  for (int i = 0; i < NW; ++i) r += red[i];
  return r;
}

// Exclusive scan of a u32 across the CTA; *total receives the sum.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* red, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = x;
  __syncthreads();
  uint32_t before = 0, tot = 0;
  for (int i = 0; i < NW; ++i) {
    uint32_t r = red[i];
    if (i < warp) before += r;
    tot += r;
  }
  *total = tot;
  return before + x - v;
}

// Slice of the unit owned by cluster rank `crank`, in 16-byte vectors; multiples of 64 vectors
// (1 KiB) so FixedLen chunks (128 symbols) and Huffman index grains never straddle CTAs.
__device__ __forceinline__ void unit_slice_n(uint64_t R, uint32_t idx, uint32_t n, uint64_t& v0, uint64_t& v1) {
  const uint64_t nvec = (R + 15) / 16;
  const uint64_t per = ((nvec + SLICE_ALIGN * n - 1) / (SLICE_ALIGN * n)) * SLICE_ALIGN;
  v0 = min(nvec, per * idx);
  v1 = min(nvec, per * (idx + 1));
}
__device__ __forceinline__ void unit_slice(uint64_t R, uint32_t crank, uint64_t& v0, uint64_t& v1) {
  unit_slice_n(R, crank, CL, v0, v1);
}
}  // namespace
}  // namespace zc
