// zc_quant.cu — interface-layer quantizer kernels (the only lossy step).
//
// Reference (relative to /root/reference/proj/core/):
//   checked_absmax            quant.cpp:13-20
//   eb_quantize_with_scale /
//   eb_quantize_chunk         quant.cpp:43-62  (round_to_symbol quant.cpp:22-27)
//   dequantize_into           quant.cpp:107-127
// Streaming kernels: 128-bit coalesced loads/stores, grid = a multiple of the 148 SMs, grid-stride.
#include "zc_kernels.h"

namespace zc {
namespace {

constexpr int QT = 256;
constexpr unsigned FULL = 0xffffffffu;

int grid_for(uint64_t nvec) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  uint64_t want = (nvec + QT - 1) / QT;
  uint64_t cap = static_cast<uint64_t>(sms) * 8;
  return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

// max|x| as the raw bits of a non-negative double (monotone as unsigned), plus a finiteness flag.
template <typename T>
__global__ void __launch_bounds__(QT) absmax_kernel(const T* __restrict__ x, uint64_t n, unsigned long long* out,
                                                    uint32_t* err) {
  constexpr int V = 16 / sizeof(T);
  const uint64_t nvec = (reinterpret_cast<uintptr_t>(x) & 15) == 0 ? n / V : 0;
  double m = 0.0;
  bool bad = false;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * QT;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(QT) + threadIdx.x; v < nvec; v += stride) {
    if (sizeof(T) == 4) {
      float4 f = __ldg(reinterpret_cast<const float4*>(x) + v);
      float a[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        bad |= !isfinite(a[k]);
        m = fmax(m, fabs(static_cast<double>(a[k])));
      }
    } else {
      double2 d = __ldg(reinterpret_cast<const double2*>(x) + v);
      bad |= !isfinite(d.x) || !isfinite(d.y);
      m = fmax(m, fmax(fabs(d.x), fabs(d.y)));
    }
  }
  for (uint64_t i = nvec * V + blockIdx.x * static_cast<uint64_t>(QT) + threadIdx.x; i < n; i += stride) {
    double a = static_cast<double>(x[i]);
    bad |= !isfinite(a);
    m = fmax(m, fabs(a));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
  bad = __any_sync(FULL, bad);
  if ((threadIdx.x & 31) == 0) {
    if (!isfinite(m)) m = 0.0;  // non-finite input is reported through the error word
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
    if (bad) atomicOr(err, ZC_DERR_NONFINITE);
  }
}

template <typename T>
__global__ void __launch_bounds__(QT) quantize_kernel(const T* __restrict__ x, uint64_t n, double scale, double rcp,
                                                      int32_t* __restrict__ sym, uint32_t* err) {
  const bool al = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(sym)) & 15) == 0;
  const uint64_t nvec = al ? n / 4 : 0;
  uint32_t e = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * QT;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(QT) + threadIdx.x; v < nvec; v += stride) {
    double a[4];
    if (sizeof(T) == 4) {
      const uint4 f = __ldg(reinterpret_cast<const uint4*>(x) + v);
      int4 o;
      o.x = quantize_f32bits(f.x, scale, rcp, e);
      o.y = quantize_f32bits(f.y, scale, rcp, e);
      o.z = quantize_f32bits(f.z, scale, rcp, e);
      o.w = quantize_f32bits(f.w, scale, rcp, e);
      reinterpret_cast<int4*>(sym)[v] = o;
      continue;
    } else {
      double2 d0 = __ldg(reinterpret_cast<const double2*>(x) + 2 * v);
      double2 d1 = __ldg(reinterpret_cast<const double2*>(x) + 2 * v + 1);
      a[0] = d0.x;
      a[1] = d0.y;
      a[2] = d1.x;
      a[3] = d1.y;
    }
    int4 o;
    o.x = quantize_one(a[0], scale, rcp, e);
    o.y = quantize_one(a[1], scale, rcp, e);
    o.z = quantize_one(a[2], scale, rcp, e);
    o.w = quantize_one(a[3], scale, rcp, e);
    reinterpret_cast<int4*>(sym)[v] = o;
  }
  for (uint64_t i = nvec * 4 + blockIdx.x * static_cast<uint64_t>(QT) + threadIdx.x; i < n; i += stride)
    sym[i] = quantize_one(static_cast<double>(x[i]), scale, rcp, e);
  e = __reduce_or_sync(FULL, e);
  if ((threadIdx.x & 31) == 0 && e) atomicOr(err, e);
}

__global__ void __launch_bounds__(QT) dequantize_kernel(const int32_t* __restrict__ sym, uint64_t n, double k,
                                                        void* out, int out_f64) {
  const bool al = ((reinterpret_cast<uintptr_t>(sym) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const uint64_t nvec = al ? n / 4 : 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * QT;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(QT) + threadIdx.x; v < nvec; v += stride) {
    uint4 s = __ldg(reinterpret_cast<const uint4*>(sym) + v);
    double d0 = __dmul_rn(k, i2d_magic(s.x)), d1 = __dmul_rn(k, i2d_magic(s.y));
    double d2 = __dmul_rn(k, i2d_magic(s.z)), d3 = __dmul_rn(k, i2d_magic(s.w));
    if (out_f64) {
      reinterpret_cast<double2*>(out)[2 * v] = make_double2(d0, d1);
      reinterpret_cast<double2*>(out)[2 * v + 1] = make_double2(d2, d3);
    } else {
      reinterpret_cast<float4*>(out)[v] =
          make_float4(d2f_rn(d0), d2f_rn(d1), d2f_rn(d2), d2f_rn(d3));
    }
  }
  for (uint64_t i = nvec * 4 + blockIdx.x * static_cast<uint64_t>(QT) + threadIdx.x; i < n; i += stride) {
    double d = __dmul_rn(k, static_cast<double>(sym[i]));
    if (out_f64) static_cast<double*>(out)[i] = d;
    else static_cast<float*>(out)[i] = __double2float_rn(d);
  }
}

// frame_commit_raw (frame.cpp:71-81) on device.
__global__ void commit_raw_kernel(const uint8_t* raw, uint64_t n, uint8_t* region, uint64_t cap, uint64_t* total) {
  const bool fits = n > 0 && cap >= kHeaderBytes && cap - kHeaderBytes >= n;
  if (!fits) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *total = 0;
    return;
  }
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    region[kHeaderBytes + i] = raw[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    zc_frame_header h = make_header(ZC_CODEC_RAW, 0, n, n, 0);
    uint64_t w[4];
    header_words(h, w);
    for (int i = 0; i < 32; ++i) region[i] = static_cast<uint8_t>(w[i / 8] >> (8 * (i % 8)));
    *total = kHeaderBytes + n;
  }
}

// 256-bin byte histogram (shared-memory privatised bins, warp-aggregated atomics).
__global__ void __launch_bounds__(QT) hist_kernel(const uint8_t* __restrict__ d, uint64_t n, unsigned long long* hist) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += QT) h[i] = 0;
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * QT;
  const uint64_t lim = (n + 31) & ~31ull;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(QT) + threadIdx.x; i < lim; i += stride) {
    const bool in = i < n;
    const uint32_t key = in ? d[i] : 256u + (threadIdx.x & 31);
    const uint32_t peers = __match_any_sync(__activemask(), key);
    if (in && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&h[key], __popc(peers));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += QT)
    if (h[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(h[i]));
}

}  // namespace

void preload_quant_kernels() {
  cudaFuncAttributes a;
  cudaFuncGetAttributes(&a, absmax_kernel<float>);
  cudaFuncGetAttributes(&a, absmax_kernel<double>);
  cudaFuncGetAttributes(&a, quantize_kernel<float>);
  cudaFuncGetAttributes(&a, quantize_kernel<double>);
  cudaFuncGetAttributes(&a, dequantize_kernel);
  cudaFuncGetAttributes(&a, commit_raw_kernel);
  cudaFuncGetAttributes(&a, hist_kernel);
  grid_for(1);
  cudaGetLastError();
}

cudaError_t launch_absmax(const void* x, int src_kind, uint64_t n, double* out, uint32_t* err, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double), s);
  if (n == 0) return cudaGetLastError();
  unsigned long long* o = reinterpret_cast<unsigned long long*>(out);
  if (src_kind == SRC_F64) {
    note_launch();
    absmax_kernel<double><<<grid_for(n / 2), QT, 0, s>>>(static_cast<const double*>(x), n, o, err);
  } else {
    note_launch();
    absmax_kernel<float><<<grid_for(n / 4), QT, 0, s>>>(static_cast<const float*>(x), n, o, err);
  }
  return cudaGetLastError();
}

cudaError_t launch_quantize(const void* x, int src_kind, uint64_t n, double scale, int32_t* sym, uint32_t* err,
                            cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const double rcp = 1.0 / scale;
  if (src_kind == SRC_F64) {
    note_launch();
    quantize_kernel<double><<<grid_for(n / 4), QT, 0, s>>>(static_cast<const double*>(x), n, scale, rcp, sym, err);
  } else {
    note_launch();
    quantize_kernel<float><<<grid_for(n / 4), QT, 0, s>>>(static_cast<const float*>(x), n, scale, rcp, sym, err);
  }
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const int32_t* sym, uint64_t n, double k, int prequant, void* out, int out_f64,
                              cudaStream_t s) {
  if (n == 0) return cudaSuccess; {
  note_launch();
  dequantize_kernel<<<grid_for(n / 4), QT, 0, s>>>(sym, n, prequant ? 1.0 : k, out, out_f64);
}
  return cudaGetLastError();
}

cudaError_t launch_commit_raw(const uint8_t* raw, uint64_t n, uint8_t* region, uint64_t cap, uint64_t* total,
                              cudaStream_t s) {
  note_launch();
  commit_raw_kernel<<<grid_for(n / 16 + 1), QT, 0, s>>>(raw, n, region, cap, total);
  return cudaGetLastError();
}

cudaError_t launch_hist(const uint8_t* d, uint64_t n, uint64_t* hist, cudaStream_t s) {
  cudaMemsetAsync(hist, 0, 256 * sizeof(uint64_t), s);
  if (n == 0) return cudaGetLastError(); {
  note_launch();
  hist_kernel<<<grid_for(n / 4), QT, 0, s>>>(d, n, reinterpret_cast<unsigned long long*>(hist));
}
  return cudaGetLastError();
}

}  // namespace zc
