// zc_qsgd.cu — the QSGD quantizer (quant.cpp:64-98) on the device, bit-exact with the reference,
// whose draws come from std::mt19937_64 (one per element, in order, quant.cpp:78).
//
// The generator on the device.  The libstdc++ mt19937_64 sequence is x_{k+312} = x_{k+156} ^
// twist(x_k, x_{k+1}) over the seeded words x_0..x_311 (output j = temper(x_{312+j})); the 19937-bit
// state is the window (x_t .. x_{t+311}) and one step of the window is GF(2)-linear.  To let every
// chunk of a message draw its own stretch of the stream in parallel, chunk c starts from the window
// at t = skip + c*M, reached by jump-ahead (Haramoto et al.): with phi the characteristic polynomial
// of the step, window_{t+D} = g(A) window_t for g = x^D mod phi, evaluated by Horner on the device.
// phi is found once per process on the host by Berlekamp-Massey over one output bit of the
// sequence; x^(2^j) mod phi (j < 64) are precomputed by repeated squaring and uploaded, so a jump
// by D applies the tables of D's set bits.  A chunk then twists its window forward, 312 words per
// round in three dependency phases, tempers, and quantizes its elements with the reference's exact
// double arithmetic (u = levels*|x|/scale, floor, frac, (draw >> 11) * 2^-53 < frac).
//
// The norm is the reference's sequential double sum of squares (quant.cpp:87-91), kept sequential
// (one thread): any parallel summation rounds differently.  qsgd_quantize_chunk with a caller norm
// (zc_qsgd_quantize_chunk_f32) is the parallel path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "zc_api_internal.h"
#include "zc_kernels.h"

namespace zc {
namespace {

constexpr int MTN = 312, MTM = 156;
constexpr uint64_t MATA = 0xB5026F5AA96619E9ull, UPPER = 0xFFFFFFFF80000000ull, LOWER = 0x7FFFFFFFull;
constexpr int DEG = 19937;
constexpr int PW = (DEG + 1 + 63) / 64;  // words of a polynomial of degree < DEG+1 (313)
constexpr int NPOW = 64;                 // x^(2^j) mod phi, j < 64

__host__ __device__ __forceinline__ uint64_t mt_twist(uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t y = (a & UPPER) | (b & LOWER);
  return c ^ (y >> 1) ^ ((y & 1ull) ? MATA : 0ull);
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
  z ^= (z >> 29) & 0x5555555555555555ull;
  z ^= (z << 17) & 0x71D67FFFEDA60000ull;
  z ^= (z << 37) & 0xFFF7EEE000000000ull;
  return z ^ (z >> 43);
}

// ------------------------------------------------------------------ host: phi and x^(2^j) mod phi
struct Poly {
  std::vector<uint64_t> w;
  explicit Poly(size_t bits = 0) : w((bits + 63) / 64, 0) {}
  bool bit(size_t i) const { return (w[i >> 6] >> (i & 63)) & 1ull; }
  void flip(size_t i) { w[i >> 6] ^= 1ull << (i & 63); }
};

// Berlekamp-Massey over GF(2) on bit 0 of the raw sequence: the minimal polynomial of the step.
Poly find_phi() {
  const int N = 2 * DEG + 64;
  std::vector<uint64_t> x(static_cast<size_t>(N) + 2 * MTN);
  x[0] = 5489ull;
  for (int i = 1; i < MTN; ++i) x[i] = 6364136223846793005ull * (x[i - 1] ^ (x[i - 1] >> 62)) + static_cast<uint64_t>(i);
  for (size_t k = 0; k + MTN < x.size(); ++k) x[k + MTN] = mt_twist(x[k], x[k + 1], x[k + MTM]);
  const size_t W = (DEG + 2 + 63) / 64 + 1;
  std::vector<uint64_t> C(W, 0), B(W, 0), T(W, 0), R(W, 0);  // R bit i = s_{n-i}
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  for (int n = 0; n < N; ++n) {
    for (size_t i = W - 1; i > 0; --i) R[i] = (R[i] << 1) | (R[i - 1] >> 63);
    R[0] = (R[0] << 1) | (x[static_cast<size_t>(n) + MTN] & 1ull);  // generated words only
    uint64_t d = 0;
    for (size_t i = 0; i < W; ++i) d ^= C[i] & R[i];
    if (!(__builtin_popcountll(d) & 1)) {
      ++m;
      continue;
    }
    T = C;
    // C ^= B << m
    const size_t ws = static_cast<size_t>(m) >> 6, bs = static_cast<size_t>(m) & 63;
    for (size_t i = W; i-- > ws;) {
      uint64_t v = B[i - ws] << bs;
      if (bs && i - ws > 0) v |= B[i - ws - 1] >> (64 - bs);
      C[i] ^= v;
    }
    if (2 * L <= n) {
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      ++m;
    }
  }
  Poly phi(DEG + 1);
  if (L != DEG) return Poly(0);  // not the full period polynomial: refuse (never expected)
  for (int i = 0; i <= L; ++i)
    if ((C[static_cast<size_t>(i) >> 6] >> (i & 63)) & 1ull) phi.flip(static_cast<size_t>(L - i));
  return phi;
}

// s ^= p << sh (word-level)
void xor_shifted(Poly& s, const Poly& p, size_t sh) {
  const size_t ws = sh >> 6, bs = sh & 63;
  for (size_t i = 0; i < p.w.size(); ++i) {
    const uint64_t v = p.w[i];
    if (!v) continue;
    s.w[i + ws] ^= v << bs;
    if (bs && i + ws + 1 < s.w.size()) s.w[i + ws + 1] ^= v >> (64 - bs);
  }
}

// a^2 mod phi (a of degree < DEG).
Poly sqr_mod(const Poly& a, const Poly& phi) {
  Poly s(2 * DEG + 128);
  for (int i = 0; i < DEG; ++i)
    if (a.bit(static_cast<size_t>(i))) s.flip(2 * static_cast<size_t>(i));
  for (int k = 2 * DEG - 2; k >= DEG; --k)
    if (s.bit(static_cast<size_t>(k))) xor_shifted(s, phi, static_cast<size_t>(k - DEG));
  Poly r(DEG);
  for (int i = 0; i < DEG; ++i)
    if (s.bit(static_cast<size_t>(i))) r.flip(static_cast<size_t>(i));
  return r;
}

struct JumpTables {
  uint64_t* d_pow = nullptr;  // NPOW x PW words: x^(2^j) mod phi
  int device = -1;
  int status = ZC_OK;
};

// Built once per device on first use (a constant of the generator, independent of the seed).
int jump_tables(uint64_t** out) {
  static std::mutex mu;
  static std::vector<uint64_t> host;  // NPOW x PW
  static std::vector<JumpTables> per_dev;
  std::lock_guard<std::mutex> lk(mu);
  if (host.empty()) {
    Poly phi = find_phi();
    if (phi.w.empty()) return set_err(ZC_ERR_RUNTIME, "mt19937_64 characteristic polynomial not found");
    host.assign(static_cast<size_t>(NPOW) * PW, 0);
    Poly p(DEG);
    p.flip(1);  // x
    for (int j = 0; j < NPOW; ++j) {
      for (size_t i = 0; i < p.w.size(); ++i) host[static_cast<size_t>(j) * PW + i] = p.w[i];
      if (j + 1 < NPOW) p = sqr_mod(p, phi);
    }
  }
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto& t : per_dev)
    if (t.device == dev) {
      *out = t.d_pow;
      return t.status;
    }
  JumpTables t;
  t.device = dev;
  t.status = cuda_err(cudaMalloc(&t.d_pow, host.size() * 8), "jump tables");
  if (!t.status) t.status = cuda_err(cudaMemcpy(t.d_pow, host.data(), host.size() * 8, cudaMemcpyHostToDevice), "jump tables");
  per_dev.push_back(t);
  *out = t.d_pow;
  return t.status;
}

// ------------------------------------------------------------------ device: jump + draw + quantize
constexpr int QT = 320;  // threads per chunk CTA (>= 312)

struct QsgdArgs {
  const float* x;       // elements (nullptr: raw draws to `draws`)
  int32_t* sym;
  uint64_t* draws;
  uint64_t n;           // elements / draws
  uint64_t seed, skip;  // the stream: mt19937_64(seed), `skip` draws discarded first
  uint64_t chunk;       // elements per CTA (a power of two)
  uint32_t log2chunk;
  uint32_t levels;
  const double* norm;   // device norm (nullptr: `norm_h`)
  double norm_h;
  const uint64_t* pow;  // jump tables
  uint32_t* err;
};

// ring <- g(A) ring for g = x^(2^j) mod phi, by Horner in blocks of B = 156 coefficients: B steps
// of acc <- A acc ^ g_i s collapse to acc <- A^B acc ^ (+)_{j < B, g_{i0-j}} A^(B-1-j) s.  A^B acc is
// the acc sequence 156 words on (its new words depend only on the current window: parallel), and
// A^p s is the window of the s sequence at offset p (s extended by 156 words once), so a block is
// one parallel twist plus, per output word, a GF(2) convolution of the block's coefficient bits
// with the extended s sequence.  All threads call; smem: ring[312], acc[312], sx[468], nw[156],
// gs[313].
__device__ void apply_pow(uint64_t* ring, uint64_t* acc, uint64_t* sx, uint64_t* nw, uint64_t* gs, const uint64_t* g) {
  const int t = threadIdx.x;
  for (int k = t; k < PW; k += blockDim.x) gs[k] = __ldg(g + k);
  for (int k = t; k < MTN; k += blockDim.x) {
    sx[k] = ring[k];
    acc[k] = 0;
  }
  __syncthreads();
  if (t < MTM) sx[MTN + t] = mt_twist(sx[t], sx[t + 1], sx[t + MTM]);  // s_{312..467}: inputs < 312
  __syncthreads();
  int i0 = DEG - 1;
  int b = DEG % MTM ? DEG % MTM : MTM;
  while (i0 >= 0) {
    if (t < b) nw[t] = mt_twist(acc[t], acc[t + 1], acc[t + MTM]);
    __syncthreads();
    uint64_t v = 0;
    if (t < MTN) {
      v = t + b < MTN ? acc[t + b] : nw[t + b - MTN];
      // coefficient i0-j multiplies s at offset b-1-j
      for (int j = 0; j < b; ++j) {
        const int i = i0 - j;
        if ((gs[i >> 6] >> (i & 63)) & 1ull) v ^= sx[b - 1 - j + t];
      }
    }
    __syncthreads();
    if (t < MTN) acc[t] = v;
    __syncthreads();
    i0 -= b;
    b = MTM;
  }
  for (int k = t; k < MTN; k += blockDim.x) ring[k] = acc[k];
  __syncthreads();
}

__global__ void __launch_bounds__(QT) qsgd_kernel(QsgdArgs a) {
  __shared__ uint64_t ring[MTN], acc[MTN], nxt[MTN], sx[MTN + MTM], gs[PW];
  __shared__ double s_norm;
  const int t = threadIdx.x;
  const uint64_t e0 = static_cast<uint64_t>(blockIdx.x) * a.chunk;
  if (e0 >= a.n) return;
  const uint64_t e1 = min(a.n, e0 + a.chunk);
  // seeded window x_0..x_311 (mersenne_twister_engine::seed)
  if (t == 0) {
    uint64_t v = a.seed;
    ring[0] = v;
    for (int i = 1; i < MTN; ++i) {
      v = 6364136223846793005ull * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
      ring[i] = v;
    }
    s_norm = a.norm ? *a.norm : a.norm_h;
  }
  __syncthreads();
  // jump to t = skip + e0
  const uint64_t D = a.skip + e0;
  for (int j = 0; j < NPOW; ++j)
    if ((D >> j) & 1ull) apply_pow(ring, acc, sx, nxt, gs, a.pow + static_cast<size_t>(j) * PW);
  const double norm = s_norm;
  const double scale = norm == 0.0 ? 1.0 : norm;
  const double lv = static_cast<double>(a.levels);
  uint32_t err = 0;
  for (uint64_t base = e0; base < e1; base += MTN) {
    // x_{t+312+i}, i < 312: three dependency phases of the twist
    if (t < MTM) nxt[t] = mt_twist(ring[t], ring[t + 1], ring[t + MTM]);
    __syncthreads();
    if (t >= MTM && t < MTN - 1) nxt[t] = mt_twist(ring[t], ring[t + 1], nxt[t - MTM]);
    __syncthreads();
    if (t == 0) nxt[MTN - 1] = mt_twist(ring[MTN - 1], nxt[0], nxt[MTM - 1]);
    __syncthreads();
    if (t < MTN) {
      const uint64_t e = base + static_cast<uint64_t>(t);
      if (e < e1) {
        const uint64_t z = mt_temper(nxt[t]);
        if (a.x == nullptr) {
          a.draws[e] = z;
        } else {
          const double v = static_cast<double>(a.x[e]);
          if (!isfinite(v)) err |= ZC_DERR_NONFINITE;
          const double u = norm == 0.0 ? 0.0 : __ddiv_rn(__dmul_rn(lv, fabs(v)), scale);
          const double fl = floor(u);
          const double frac = __dsub_rn(u, fl);
          const double draw = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
          const long long mag = static_cast<long long>(fl) + (draw < frac ? 1 : 0);
          a.sym[e] = static_cast<int32_t>(v < 0.0 ? -mag : mag);
        }
      }
    }
    __syncthreads();
    if (t < MTN) ring[t] = nxt[t];
    __syncthreads();
  }
  if (err && a.err) atomicOr(a.err, err);
}

// quant.cpp:87-91: sumsq += v*v in element order, then sqrt; one thread (the order is the result).
__global__ void qsgd_norm_kernel(const float* x, uint64_t n, double* norm, uint32_t* err) {
  double s = 0.0;
  bool bad = false;
  uint64_t i = 0;
  // The additions are one dependent chain; what must not sit on it is memory latency.  Lines are
  // prefetched into L1 kPre elements ahead (one per 32 elements, so a few hundred misses are in
  // flight from this one thread), and each 32-element step reads them as 16-byte vectors.
  constexpr int U = 32;
  constexpr uint64_t kPre = 16384;  // 64 KiB ahead
  for (; i < n && (reinterpret_cast<uintptr_t>(x + i) & 15) != 0; ++i) {
    const double v = static_cast<double>(x[i]);
    bad |= !isfinite(v);
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  for (uint64_t j = i; j < i + kPre && j < n; j += 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(x + j));
  for (; i + U <= n; i += U) {
    if (i + kPre < n) asm volatile("prefetch.global.L1 [%0];" ::"l"(x + i + kPre));
    float4 q[U / 4];
#pragma unroll
    for (int k = 0; k < U / 4; ++k) q[k] = __ldg(reinterpret_cast<const float4*>(x + i) + k);
#pragma unroll
    for (int k = 0; k < U / 4; ++k) {
      const float f4[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double v = static_cast<double>(f4[e]);
        bad |= !isfinite(v);
        s = __dadd_rn(s, __dmul_rn(v, v));
      }
    }
  }
  for (; i < n; ++i) {
    const double v = static_cast<double>(x[i]);
    bad |= !isfinite(v);
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  *norm = __dsqrt_rn(s);
  if (bad && err) atomicOr(err, ZC_DERR_NONFINITE);
}

int launch_qsgd(const float* x, int32_t* sym, uint64_t* draws, uint64_t n, uint32_t levels, const double* d_norm,
                double norm_h, uint64_t seed, uint64_t skip, uint32_t* d_err, cudaStream_t s) {
  if (n == 0) return ZC_OK;
  uint64_t* pow = nullptr;
  if (int rc = jump_tables(&pow)) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // chunk: a power of two (>= 2^14), at most ~2 CTAs per SM
  uint32_t lg = 14;
  while ((n >> lg) > static_cast<uint64_t>(2 * sms)) ++lg;
  QsgdArgs a;
  std::memset(&a, 0, sizeof(a));
  a.x = x;
  a.sym = sym;
  a.draws = draws;
  a.n = n;
  a.seed = seed;
  a.skip = skip;
  a.chunk = 1ull << lg;
  a.log2chunk = lg;
  a.levels = levels;
  a.norm = d_norm;
  a.norm_h = norm_h;
  a.pow = pow;
  a.err = d_err;
  const uint32_t grid = static_cast<uint32_t>((n + a.chunk - 1) >> lg);
  note_launch();
  qsgd_kernel<<<grid, QT, 0, s>>>(a);
  return cuda_err(cudaGetLastError(), "qsgd");
}

}  // namespace
}  // namespace zc

using namespace zc;

extern "C" {

int zc_mt19937_64(uint64_t seed, uint64_t skip, uint64_t n, uint64_t* d_out, void* stream) {
  if (n > 0 && d_out == nullptr) return set_err(ZC_ERR_INVALID_ARGUMENT, "null output");
  return launch_qsgd(nullptr, nullptr, d_out, n, 1, nullptr, 0.0, seed, skip, nullptr, static_cast<cudaStream_t>(stream));
}

int zc_qsgd_quantize_chunk_f32(const float* d_x, uint64_t n, uint32_t levels, double norm, uint64_t seed, uint64_t skip,
                               int32_t* d_sym, void* stream) {
  if (levels == 0 || levels > (1u << 30))
    return set_err(ZC_ERR_INVALID_ARGUMENT, "qsgd_quantize_chunk: levels must be in [1, 2^30]");
  if (!(norm >= 0.0) || !std::isfinite(norm))
    return set_err(ZC_ERR_INVALID_ARGUMENT, "qsgd_quantize_chunk: norm must be finite and nonnegative");
  if (n == 0) return ZC_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* d_err = nullptr;
  if (int rc = cuda_err(cudaMallocAsync(reinterpret_cast<void**>(&d_err), 4, s), "qsgd scratch")) return rc;
  int rc = cuda_err(cudaMemsetAsync(d_err, 0, 4, s), "qsgd scratch");
  if (!rc) rc = launch_qsgd(d_x, d_sym, nullptr, n, levels, nullptr, norm, seed, skip, d_err, s);
  uint32_t e = 0;
  if (!rc) rc = cuda_err(cudaMemcpyAsync(&e, d_err, 4, cudaMemcpyDeviceToHost, s), "qsgd result");
  if (!rc) rc = cuda_err(cudaStreamSynchronize(s), "qsgd sync");
  cudaFreeAsync(d_err, s);
  if (rc) return rc;
  if (e) return set_err(ZC_ERR_INVALID_ARGUMENT, "qsgd_quantize_chunk: non-finite input");
  return ZC_OK;
}

int zc_qsgd_norm_f32(const float* d_x, uint64_t n, double* d_norm, uint32_t* d_err, void* stream) {
  if (d_norm == nullptr) return set_err(ZC_ERR_INVALID_ARGUMENT, "null output");
  note_launch();
  qsgd_norm_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_x, n, d_norm, d_err);
  return cuda_err(cudaGetLastError(), "qsgd norm");
}

int zc_qsgd_quantize_f32(const float* d_x, uint64_t n, uint32_t levels, uint64_t seed, int32_t* d_sym, double* h_scale,
                         void* stream) {
  if (levels == 0 || levels > (1u << 30))
    return set_err(ZC_ERR_INVALID_ARGUMENT, "qsgd_quantize_chunk: levels must be in [1, 2^30]");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  struct Scratch {
    double norm;
    uint32_t err, _p;
  };
  Scratch* d = nullptr;
  if (int rc = cuda_err(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(Scratch), s), "qsgd scratch")) return rc;
  int rc = cuda_err(cudaMemsetAsync(d, 0, sizeof(Scratch), s), "qsgd scratch");
  if (!rc) rc = zc_qsgd_norm_f32(d_x, n, &d->norm, &d->err, stream);
  if (!rc) rc = launch_qsgd(d_x, d_sym, nullptr, n, levels, &d->norm, 0.0, seed, 0, &d->err, s);
  Scratch h{};
  if (!rc) rc = cuda_err(cudaMemcpyAsync(&h, d, sizeof(Scratch), cudaMemcpyDeviceToHost, s), "qsgd result");
  if (!rc) rc = cuda_err(cudaStreamSynchronize(s), "qsgd sync");
  cudaFreeAsync(d, s);
  if (rc) return rc;
  if (h.err) return set_err(ZC_ERR_INVALID_ARGUMENT, "qsgd_quantize: non-finite input");
  *h_scale = h.norm == 0.0 ? 1.0 : h.norm;
  return ZC_OK;
}

}  // extern "C"
