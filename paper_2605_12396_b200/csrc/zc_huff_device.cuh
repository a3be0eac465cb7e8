// zc_huff_device.cuh — CTA-cooperative Huffman table construction on the device.
//
// Used per frame in embedded-codebook mode (rea.cpp:214-221 builds the code from the batch's
// full histogram; huffman.cpp:256-262 rebuilds it from the 256 serialized lengths on decode)
// and for SampleStats::selfCodeLenBits (rea.cpp:113-116).  Same algorithm as the host builder
// (zc_huffman_host.cpp): the reference's pairwise merge realised as a two-queue construction over
// leaves sorted by (weight, symbol), then the 32-bit cap repair and canonical assignment.
#pragma once
#include "zc_common.cuh"

namespace zc {

// Bitonic sort of 256 u64 keys in shared memory by a CTA of >= 256 threads (threads >= 256 idle).
__device__ __forceinline__ void bitonic256(unsigned long long* key) {
  const unsigned t = threadIdx.x;
  for (unsigned k = 2; k <= 256; k <<= 1) {
    for (unsigned j = k >> 1; j > 0; j >>= 1) {
      __syncthreads();
      if (t < 256) {
        unsigned ixj = t ^ j;
        if (ixj > t) {
          unsigned long long a = key[t], b = key[ixj];
          bool up = (t & k) == 0;
          if ((a > b) == up) {
            key[t] = b;
            key[ixj] = a;
          }
        }
      }
    }
  }
  __syncthreads();
}

// Code lengths for hist (u32 bins) into lens[256]; all threads of the CTA must call.
// scratch: >= 256 u64 keys + 512 u32 weights(as u64) + 512 i32 parents + 512 u8 depths.
__device__ inline void cta_huff_lengths(const uint32_t* hist, uint8_t* lens, unsigned long long* keys, unsigned long long* w,
                                 int* parent, uint8_t* depth) {
  const unsigned t = threadIdx.x;
  if (t < 256) {
    // zero-frequency symbols sort first and are skipped; key = freq << 8 | sym
    keys[t] = (static_cast<unsigned long long>(hist[t]) << 8) | t;
    lens[t] = 0;
  }
  bitonic256(keys);
  if (t == 0) {
    int first = 0;
    while (first < 256 && (keys[first] >> 8) == 0) ++first;
    const int L = 256 - first;
    if (L == 1) {
      lens[keys[first] & 0xFF] = 1;
    } else if (L > 1) {
      for (int i = 0; i < L; ++i) {
        w[i] = keys[first + i] >> 8;
        parent[i] = -1;
      }
      int li = 0, mi = L, next = L;
      while (next < 2 * L - 1) {
        int a, b;
        if (li < L && (mi >= next || w[li] <= w[mi])) a = li++; else a = mi++;
        if (li < L && (mi >= next || w[li] <= w[mi])) b = li++; else b = mi++;
        w[next] = w[a] + w[b];
        parent[a] = parent[b] = next;
        parent[next] = -1;
        ++next;
      }
      depth[2 * L - 2] = 0;
      for (int i = 2 * L - 3; i >= 0; --i) depth[i] = static_cast<uint8_t>(depth[parent[i]] + 1);
      for (int i = 0; i < L; ++i) lens[keys[first + i] & 0xFF] = depth[i];
      // cap repair (huffman.cpp:72-95)
      const unsigned cap = ZC_HUFF_MAX_CODE_LEN;
      unsigned long long kraft = 0;
      for (int s = 0; s < 256; ++s) {
        if (!lens[s]) continue;
        if (lens[s] > cap) lens[s] = cap;
        kraft += 1ull << (cap - lens[s]);
      }
      while (kraft > (1ull << cap)) {
        int pick = -1;
        unsigned pl = 0;
        for (int s = 0; s < 256; ++s) {
          unsigned l = lens[s];
          if (l > 0 && l < cap && l >= pl) {
            pl = l;
            pick = s;
          }
        }
        if (pick < 0) break;
        lens[pick]++;
        kraft -= 1ull << (cap - pl - 1);
      }
    }
  }
  __syncthreads();
}

// Mean code length Σf·len/Σf (huffman.cpp:182-214) by warp 0; returns validity (lane 0 result).
__device__ __forceinline__ bool warp_mean_len(const uint32_t* hist, const uint8_t* lens, double& out) {
  const unsigned lane = threadIdx.x & 31;
  unsigned long long bits = 0, total = 0;
  bool bad = false;
  for (int s = lane; s < 256; s += 32) {
    unsigned long long f = hist[s];
    if (!f) continue;
    if (!lens[s]) bad = true;
    total += f;
    bits += f * lens[s];
  }
  for (int o = 16; o > 0; o >>= 1) {
    bits += __shfl_xor_sync(0xffffffffu, bits, o);
    total += __shfl_xor_sync(0xffffffffu, total, o);
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad || total == 0) return false;
  out = __ddiv_rn(__ull2double_rn(bits), __ull2double_rn(total));
  return true;
}

// Canonical encode table from lengths (huffman.cpp:97-161), thread 0 only.  enc[s] = rev | len<<32.
__device__ __forceinline__ void canonical_enc(const uint8_t* lens, unsigned long long* enc) {
  uint32_t bl[34];
  unsigned long long next[34];
  for (int i = 0; i < 34; ++i) bl[i] = 0;
  unsigned maxl = 0;
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (l) {
      ++bl[l];
      if (l > maxl) maxl = l;
    }
  }
  unsigned long long code = 0;
  next[0] = 0;
  for (unsigned l = 1; l <= maxl; ++l) {
    code = (code + bl[l - 1]) << 1;
    next[l] = code;
  }
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (!l) {
      enc[s] = 0;
      continue;
    }
    uint32_t c = static_cast<uint32_t>(next[l]++);
    uint32_t r = __brev(c) >> (32 - l);
    enc[s] = static_cast<unsigned long long>(r) | (static_cast<unsigned long long>(l) << 32);
  }
}

// Full decode tables from 256 lengths with the reference's validation (Kraft, <= 32, non-empty).
// All threads call; returns validity.  Writes d (shared memory DevHuff).
__device__ inline bool cta_decode_tables(const uint8_t* lens_src, DevHuff* d, uint32_t* s_flag) {
  const unsigned t = threadIdx.x;
  if (t < 256) d->len[t] = lens_src[t];
  for (unsigned i = t; i < (1u << ZC_HUFF_ROOT_BITS); i += blockDim.x) d->lut[i] = 0;
  __syncthreads();
  if (t == 0) {
    uint32_t bl[34];
    for (int i = 0; i < 34; ++i) bl[i] = 0;
    unsigned minl = 0, maxl = 0, n = 0;
    bool ok = true;
    for (int s = 0; s < 256; ++s) {
      unsigned l = d->len[s];
      if (!l) continue;
      if (l > ZC_HUFF_MAX_CODE_LEN) {
        ok = false;
        break;
      }
      ++bl[l];
      ++n;
      if (minl == 0 || l < minl) minl = l;
      if (l > maxl) maxl = l;
    }
    if (ok && n == 0) ok = false;
    if (ok) {
      unsigned long long kraft = 0;
      for (unsigned l = 1; l <= maxl; ++l) kraft += static_cast<unsigned long long>(bl[l]) << (ZC_HUFF_MAX_CODE_LEN - l);
      if (kraft > (1ull << ZC_HUFF_MAX_CODE_LEN)) ok = false;
    }
    if (ok) {
      unsigned long long next[34];
      unsigned long long code = 0;
      uint32_t idx = 0;
      for (int l = 0; l < 33; ++l) {
        d->first_code[l] = 0;
        d->first_index[l] = 0;
        d->count_at_len[l] = 0;
      }
      for (unsigned l = 1; l <= maxl; ++l) {
        code = (code + bl[l - 1]) << 1;
        next[l] = d->first_code[l] = code;
        d->first_index[l] = idx;
        d->count_at_len[l] = bl[l];
        idx += bl[l];
      }
      uint32_t fill[34];
      for (int i = 0; i < 34; ++i) fill[i] = 0;
      for (int s = 0; s < 256; ++s) {
        unsigned l = d->len[s];
        if (!l) {
          d->enc[s] = 0;
          continue;
        }
        uint32_t c = static_cast<uint32_t>(next[l]++);
        uint32_t r = __brev(c) >> (32 - l);
        d->enc[s] = static_cast<unsigned long long>(r) | (static_cast<unsigned long long>(l) << 32);
        d->sym_order[d->first_index[l] + fill[l]++] = static_cast<uint8_t>(s);
      }
      d->min_len = minl;
      d->max_len = maxl;
    }
    d->valid = ok ? 1u : 0u;
    *s_flag = ok ? 1u : 0u;
  }
  __syncthreads();
  bool ok = *s_flag != 0;
  if (ok && t < 256) {
    unsigned l = d->len[t];
    if (l && l <= ZC_HUFF_ROOT_BITS) {
      uint32_t r = static_cast<uint32_t>(d->enc[t]);
      uint16_t e = static_cast<uint16_t>(t | (l << 8));
      for (uint32_t pad = 0; pad < (1u << (ZC_HUFF_ROOT_BITS - l)); ++pad) d->lut[r | (pad << l)] = e;
    }
  }
  __syncthreads();
  return ok;
}

}  // namespace zc
