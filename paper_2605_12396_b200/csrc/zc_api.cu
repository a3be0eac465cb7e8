// zc_api.cu — extern "C" entry points of libzcomm_b200.so (include/zcomm_b200.h).
//
// Host C++ that validates arguments the way the reference does, prepares kernel parameters and
// launches the sm_100a kernels.  Never computes on the CPU: every data-touching entry point
// launches device work and returns ZC_ERR_CUDA when no device is usable.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "zc_api_internal.h"
#include "zc_huffman_host.hpp"
#include "zc_kernels.h"

struct zc_huff_ctx {
  zc::HostHuff h;
  std::mutex mu;
  std::map<int, zc::DevHuff*> dev;  // device ordinal -> uploaded tables
};

namespace zc {

thread_local std::string g_err;

std::atomic<uint64_t>& launch_counter() {
  static std::atomic<uint64_t> n{0};
  return n;
}
void note_launch() { launch_counter().fetch_add(1, std::memory_order_relaxed); }
void note_launches(uint64_t k) { launch_counter().fetch_add(k, std::memory_order_relaxed); }

namespace {
std::atomic<int> g_inflight{0};
std::mutex g_dead_mu;
struct Dead {
  int device;
  void* p;
  bool ipc;
};
std::vector<Dead> g_dead;
void free_now(const Dead& d) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(d.device);
  if (d.ipc) cudaIpcCloseMemHandle(d.p);
  else cudaFree(d.p);
  cudaSetDevice(cur);
}
}  // namespace

InFlight::InFlight() { g_inflight.fetch_add(1); }
InFlight::~InFlight() { g_inflight.fetch_sub(1); }

void release_device_memory(int device, void* p, bool ipc_handle) {
  if (p == nullptr) return;
  if (g_inflight.load() > 0) {
    std::lock_guard<std::mutex> g(g_dead_mu);
    g_dead.push_back(Dead{device, p, ipc_handle});
    return;
  }
  free_now(Dead{device, p, ipc_handle});
}

void flush_deferred_if_idle() {
  std::vector<Dead> v;
  {
    std::lock_guard<std::mutex> g(g_dead_mu);
    if (g_inflight.load() > 0) return;
    v.swap(g_dead);
  }
  for (const Dead& d : v) free_now(d);
}

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_err(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return ZC_OK;
  return set_err(ZC_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

const DevHuff* device_tables(const zc_huff_ctx* c) {
  if (c == nullptr) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  auto* m = const_cast<zc_huff_ctx*>(c);
  std::lock_guard<std::mutex> g(m->mu);
  auto it = m->dev.find(dev);
  if (it != m->dev.end()) return it->second;
  DevHuff host;
  to_device_layout(c->h, host);
  DevHuff* d = nullptr;
  if (cudaMalloc(&d, sizeof(DevHuff)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &host, sizeof(DevHuff), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  m->dev[dev] = d;
  return d;
}

// Per-(device, stream) scratch: decode flags (zero between calls) and an ignorable error word.
struct Scratch {
  uint32_t* flags = nullptr;
  uint64_t nflags = 0;
  uint32_t* sink = nullptr;
  void* task = nullptr;  // batched-encoder unit states
  size_t task_bytes = 0;
};
static std::mutex g_scratch_mu;
static std::map<std::pair<int, void*>, Scratch> g_scratch;

Scratch* scratch_for(cudaStream_t s, uint64_t nflags) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(g_scratch_mu);
  Scratch& sc = g_scratch[{dev, reinterpret_cast<void*>(s)}];
  if (!sc.sink) {
    if (cudaMalloc(&sc.sink, 64) != cudaSuccess) return nullptr;
    cudaMemset(sc.sink, 0, 64);
  }
  if (sc.nflags < nflags) {
    cudaStreamSynchronize(s);
    if (sc.flags) cudaFree(sc.flags);
    uint64_t n = nflags < 1024 ? 1024 : nflags;
    if (cudaMalloc(&sc.flags, n * 4) != cudaSuccess) {
      sc.flags = nullptr;
      sc.nflags = 0;
      return nullptr;
    }
    cudaMemset(sc.flags, 0, n * 4);
    sc.nflags = n;
  }
  return &sc;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int encode_common(EncParams& p, cudaStream_t s) {
  Scratch* sc = scratch_for(s, 1);
  if (!sc) return set_err(ZC_ERR_CUDA, "cannot allocate scratch (no CUDA device?)");
  if (p.err == nullptr) p.err = sc->sink;
  // The batched send path (many frames, shared or no Huffman context) runs on the streaming
  // profile / range / emit kernels (zc_batch.cu, zc_fixed.cu); single frames, bare codecs,
  // profiling and embedded codebooks on the cluster kernels (zc_encode.cu).
  if (p.mode == ENC_SEND && !p.link_tx && !p.link_rx_add && !p.cfg.embed_codebook) {
    const size_t need = batch_scratch_bytes(p.nunits);
    if (sc->task_bytes < need) {
      cudaStreamSynchronize(s);
      if (sc->task) cudaFree(sc->task);
      sc->task = nullptr;
      sc->task_bytes = 0;
      if (int rc = cuda_err(cudaMalloc(&sc->task, need), "encoder scratch")) return rc;
      sc->task_bytes = need;
    }
    return cuda_err(launch_encode_batch(p, sc->task, s), "encode");
  }
  return cuda_err(launch_encode(p, s), "encode");
}

// Pre-sizes the scratch of stream `s` for messages of up to `nunits` batches, so later calls on
// it never allocate (cudaFree / cudaMalloc can wait for the whole device: a ring rank's spinning
// wait kernel would then wait for work not yet enqueued).
int reserve_scratch(cudaStream_t s, uint32_t nunits) {
  Scratch* sc = scratch_for(s, nunits);
  if (!sc) return set_err(ZC_ERR_CUDA, "cannot allocate scratch (no CUDA device?)");
  const size_t need = std::max(batch_scratch_bytes(nunits), ring_fused_scratch_bytes(nunits));
  if (sc->task_bytes < need) {
    cudaStreamSynchronize(s);
    if (sc->task) cudaFree(sc->task);
    sc->task = nullptr;
    sc->task_bytes = 0;
    if (int rc = cuda_err(cudaMalloc(&sc->task, need), "encoder scratch")) return rc;
    sc->task_bytes = need;
  }
  return ZC_OK;
}

int decode_common(DecParams& p, cudaStream_t s) {
  Scratch* sc = scratch_for(s, p.nunits);
  if (!sc) return set_err(ZC_ERR_CUDA, "cannot allocate scratch (no CUDA device?)");
  p.flags = sc->flags;
  if (p.err == nullptr) p.err = sc->sink;
  return cuda_err(launch_decode(p, s), "decode");
}

EncParams base_enc(const zc_transport_hint* hint, const zc_huff_ctx* ctx, const zc_arb_config* cfg) {
  EncParams p;
  std::memset(&p, 0, sizeof(p));
  if (hint) p.hint = *hint;
  else zc_default_transport_hint(&p.hint);
  if (cfg) p.cfg = *cfg;
  else zc_default_arb_config(&p.cfg);
  p.ctx = device_tables(ctx);
  p.scale = 1.0;
  p.rcp = 1.0;
  return p;
}

}  // namespace zc

using namespace zc;

extern "C" {

const char* zc_last_error(void) { return g_err.c_str(); }
const char* zc_version(void) { return "zcomm-b200 0.1 (sm_100a)"; }
uint64_t zc_launch_count(void) { return zc::launch_counter().load(std::memory_order_relaxed); }

int zc_device_count(int* n) {
  cudaError_t e = cudaGetDeviceCount(n);
  if (e != cudaSuccess) {
    *n = 0;
    cudaGetLastError();
    return cuda_err(e, "cudaGetDeviceCount");
  }
  return ZC_OK;
}

int zc_device_malloc(uint64_t bytes, void** d_out) {
  *d_out = nullptr;
  return cuda_err(cudaMalloc(d_out, bytes ? bytes : 1), "cudaMalloc");
}
void zc_device_free(void* d) {
  if (!d) return;
  int dev = 0;
  cudaGetDevice(&dev);
  zc::release_device_memory(dev, d, false);
}
void zc_flush_deferred(void) { zc::flush_deferred_if_idle(); }
int zc_memcpy(void* dst, const void* src, uint64_t bytes) {
  return cuda_err(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault), "cudaMemcpy");
}
int zc_memset(void* d, int value, uint64_t bytes) { return cuda_err(cudaMemset(d, value, bytes), "cudaMemset"); }
int zc_stream_synchronize(void* stream) {
  return cuda_err(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cudaStreamSynchronize");
}

void zc_default_arb_config(zc_arb_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->small_batch_threshold_bytes = 4096;
  c->huffman_min_raw_bytes = 65536;
  c->min_gain_permil = 50;
  c->embed_codebook = 0;
  c->lam_enc = 0.25;
  c->lam_dec = 0.25;
  c->cost.fixedlen = {1.0e-6, 250.0e9, 300.0e9};
  c->cost.huffman = {1.5e-6, 120.0e9, 150.0e9};
}

void zc_default_transport_hint(zc_transport_hint* h) {
  h->regime = ZC_REGIME_INTER;
  h->_pad = 0;
  h->beta_eff_bytes_per_sec = 10.0 * 1073741824.0;
}

void zc_default_collective_config(zc_collective_config* c) {
  std::memset(c, 0, sizeof(*c));
  zc_default_arb_config(&c->arb);
  zc_default_transport_hint(&c->hint);
  c->pin = ZC_PIN_AUTO;
  c->serialized = 0;
  c->fused_codec_min_msg_bytes = ZC_BATCH_RAW_BYTES;
}

// apply_kv (rea.cpp:57-73)
static int apply_kv(zc_arb_config* cfg, const std::string& key, const std::string& value) {
  try {
    size_t pos = 0;
    auto as_u64 = [&] {
      unsigned long long v = std::stoull(value, &pos);
      return static_cast<uint64_t>(v);
    };
    auto as_f64 = [&] { return std::stod(value, &pos); };
    auto as_bool = [&]() -> bool {
      if (value == "1" || value == "true" || value == "on") return true;
      if (value == "0" || value == "false" || value == "off") return false;
      throw std::invalid_argument("expected boolean, got '" + value + "'");
    };
    if (key == "small_batch_threshold") cfg->small_batch_threshold_bytes = as_u64();
    else if (key == "huffman_min_raw_bytes") cfg->huffman_min_raw_bytes = as_u64();
    else if (key == "min_gain_permil") cfg->min_gain_permil = static_cast<uint32_t>(as_u64());
    else if (key == "embed_codebook") cfg->embed_codebook = as_bool() ? 1 : 0;
    else if (key == "lam_enc") cfg->lam_enc = as_f64();
    else if (key == "lam_dec") cfg->lam_dec = as_f64();
    else if (key == "fixedlen_alpha_sec") cfg->cost.fixedlen.alpha_sec = as_f64();
    else if (key == "fixedlen_enc_bps") cfg->cost.fixedlen.enc_bytes_per_sec = as_f64();
    else if (key == "fixedlen_dec_bps") cfg->cost.fixedlen.dec_bytes_per_sec = as_f64();
    else if (key == "huffman_alpha_sec") cfg->cost.huffman.alpha_sec = as_f64();
    else if (key == "huffman_enc_bps") cfg->cost.huffman.enc_bytes_per_sec = as_f64();
    else if (key == "huffman_dec_bps") cfg->cost.huffman.dec_bytes_per_sec = as_f64();
    else return set_err(ZC_ERR_INVALID_ARGUMENT, "unknown config key '" + key + "'");
  } catch (const std::exception& e) {
    return set_err(ZC_ERR_INVALID_ARGUMENT, e.what());
  }
  return ZC_OK;
}

static std::string trim(const std::string& s) {
  size_t b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return {};
  size_t e = s.find_last_not_of(" \t\r\n");
  return s.substr(b, e - b + 1);
}

// load_arbitration_config (rea.cpp:240-263)
int zc_load_arbitration_config(const char* text, zc_arb_config* cfg) {
  std::istringstream in(text ? text : "");
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    size_t hash = line.find('#');
    if (hash != std::string::npos) line.erase(hash);
    line = trim(line);
    if (line.empty()) continue;
    size_t eq = line.find('=');
    if (eq == std::string::npos)
      return set_err(ZC_ERR_INVALID_ARGUMENT, "config line " + std::to_string(lineno) + ": expected key=value");
    int rc = apply_kv(cfg, trim(line.substr(0, eq)), trim(line.substr(eq + 1)));
    if (rc) return set_err(rc, "config line " + std::to_string(lineno) + ": " + g_err);
  }
  return ZC_OK;
}

// apply_env_overrides (rea.cpp:270-279)
int zc_apply_env_overrides(zc_arb_config* cfg) {
  static const char* keys[] = {"small_batch_threshold", "huffman_min_raw_bytes", "min_gain_permil", "embed_codebook",
                               "lam_enc", "lam_dec", "fixedlen_alpha_sec", "fixedlen_enc_bps", "fixedlen_dec_bps",
                               "huffman_alpha_sec", "huffman_enc_bps", "huffman_dec_bps"};
  for (const char* k : keys) {
    std::string env = "ZCOMM_";
    for (const char* p = k; *p; ++p) env += static_cast<char>(std::toupper(static_cast<unsigned char>(*p)));
    const char* v = std::getenv(env.c_str());
    if (v) {
      int rc = apply_kv(cfg, k, v);
      if (rc) return rc;
    }
  }
  return ZC_OK;
}

// ------------------------------------------------------------------ frame
int zc_write_header(const zc_frame_header* h, uint8_t* dst, uint64_t len) {
  if (len < ZC_HEADER_BYTES) return set_err(ZC_ERR_INVALID_ARGUMENT, "write_header: region too small");
  uint64_t w[4];
  header_words(*h, w);
  for (int i = 0; i < 4; ++i) put_le(dst + 8 * i, w[i], 8);
  return ZC_OK;
}

int zc_parse_header(const uint8_t* src, uint64_t len, zc_frame_header* out) {
  if (len < ZC_HEADER_BYTES) return set_err(ZC_ERR_INVALID_ARGUMENT, "parse_header: fewer than 32 bytes");
  uint64_t w[4];
  for (int i = 0; i < 4; ++i) w[i] = get_le(src + 8 * i, 8);
  *out = header_from_words(w);
  return ZC_OK;
}

int zc_validate_header(const zc_frame_header* h, uint64_t region) { return validate_header(*h, region) ? 1 : 0; }

int zc_frame_commit_raw(const uint8_t* d_raw, uint64_t n, uint8_t* d_region, uint64_t cap, uint64_t* d_total,
                        void* stream) {
  return cuda_err(launch_commit_raw(d_raw, n, d_region, cap, d_total, static_cast<cudaStream_t>(stream)),
                  "frame_commit_raw");
}

// ------------------------------------------------------------------ quant
int zc_absmax_f32(const float* d_x, uint64_t n, double* d_out, uint32_t* d_err, void* stream) {
  return cuda_err(launch_absmax(d_x, SRC_F32, n, d_out, d_err, static_cast<cudaStream_t>(stream)), "absmax");
}
int zc_absmax_f64(const double* d_x, uint64_t n, double* d_out, uint32_t* d_err, void* stream) {
  return cuda_err(launch_absmax(d_x, SRC_F64, n, d_out, d_err, static_cast<cudaStream_t>(stream)), "absmax");
}

static int check_scale(double scale, const char* who) {
  if (!(scale > 0.0) || !std::isfinite(scale))
    return set_err(ZC_ERR_INVALID_ARGUMENT, std::string(who) + ": scale must be positive and finite");
  return ZC_OK;
}

int zc_eb_quantize_f32(const float* d_x, uint64_t n, double scale, int32_t* d_sym, uint32_t* d_err, void* stream) {
  if (int rc = check_scale(scale, "eb_quantize_with_scale")) return rc;
  return cuda_err(launch_quantize(d_x, SRC_F32, n, scale, d_sym, d_err, static_cast<cudaStream_t>(stream)), "quantize");
}
int zc_eb_quantize_f64(const double* d_x, uint64_t n, double scale, int32_t* d_sym, uint32_t* d_err, void* stream) {
  if (int rc = check_scale(scale, "eb_quantize_with_scale")) return rc;
  return cuda_err(launch_quantize(d_x, SRC_F64, n, scale, d_sym, d_err, static_cast<cudaStream_t>(stream)), "quantize");
}

int zc_eb_quantize_rel_f32(const float* d_x, uint64_t n, double rel, int32_t* d_sym, double* h_scale, void* stream) {
  if (!(rel > 0.0) || rel > 1.0) return set_err(ZC_ERR_INVALID_ARGUMENT, "eb_quantize: rel must be in (0, 1]");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch* sc = scratch_for(s, 1);
  if (!sc) return set_err(ZC_ERR_CUDA, "no CUDA device");
  double* d_max = reinterpret_cast<double*>(sc->sink + 8);
  uint32_t* d_err = sc->sink + 4;
  cudaMemsetAsync(d_err, 0, 4, s);
  if (int rc = cuda_err(launch_absmax(d_x, SRC_F32, n, d_max, d_err, s), "absmax")) return rc;
  double amax = 0.0;
  uint32_t err = 0;
  cudaMemcpyAsync(&amax, d_max, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, s);
  if (int rc = cuda_err(cudaStreamSynchronize(s), "sync")) return rc;
  if (err & ZC_DERR_NONFINITE) return set_err(ZC_ERR_INVALID_ARGUMENT, "eb_quantize: non-finite input");
  double scale = amax == 0.0 ? 1.0 : 2.0 * rel * amax;
  *h_scale = scale;
  cudaMemsetAsync(d_err, 0, 4, s);
  if (int rc = cuda_err(launch_quantize(d_x, SRC_F32, n, scale, d_sym, d_err, s), "quantize")) return rc;
  cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, s);
  if (int rc = cuda_err(cudaStreamSynchronize(s), "sync")) return rc;
  if (err & ZC_DERR_RANGE) return set_err(ZC_ERR_INVALID_ARGUMENT, "quantize: bin index exceeds int32 range");
  return ZC_OK;
}

static int dequant(const int32_t* d_sym, uint64_t n, int32_t mode, double scale, uint32_t levels, void* out, int f64,
                   void* stream) {
  double k;
  if (mode == ZC_QUANT_ERROR_BOUNDED) k = scale;
  else if (mode == ZC_QUANT_QSGD) {
    if (levels == 0) return set_err(ZC_ERR_INVALID_ARGUMENT, "dequantize: qsgd stream with levels 0");
    k = scale / static_cast<double>(levels);
  } else if (mode == ZC_QUANT_PREQUANTIZED) k = 1.0;
  else return set_err(ZC_ERR_INVALID_ARGUMENT, "dequantize: unknown mode");
  return cuda_err(launch_dequantize(d_sym, n, k, mode == ZC_QUANT_PREQUANTIZED, out, f64, static_cast<cudaStream_t>(stream)),
                  "dequantize");
}
int zc_dequantize_f64(const int32_t* d_sym, uint64_t n, int32_t mode, double scale, uint32_t levels, double* d_out,
                      void* stream) {
  return dequant(d_sym, n, mode, scale, levels, d_out, 1, stream);
}
int zc_dequantize_f32(const int32_t* d_sym, uint64_t n, int32_t mode, double scale, uint32_t levels, float* d_out,
                      void* stream) {
  return dequant(d_sym, n, mode, scale, levels, d_out, 0, stream);
}

// ------------------------------------------------------------------ fixedlen
int zc_fixedlen_encode(const int32_t* d_sym, uint64_t count, uint8_t* d_out, uint64_t out_cap, uint64_t* d_payload,
                       uint32_t* d_width, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (count == 0) return cuda_err(cudaMemsetAsync(d_payload, 0, 8, s), "fixedlen_encode");
  if (!aligned16(d_out)) return set_err(ZC_ERR_INVALID_ARGUMENT, "fixedlen_encode: output must be 16-byte aligned");
  EncParams p = base_enc(nullptr, nullptr, nullptr);
  p.src = d_sym;
  p.src_kind = SRC_BYTES;
  p.mode = ENC_BARE_FL;
  p.total_bytes = p.unit_bytes = count * 4;
  p.nunits = 1;
  p.stages = d_out;
  p.stage_len = out_cap;
  p.bare_payload = d_payload;
  p.bare_width = d_width;
  return encode_common(p, s);
}

int zc_fixedlen_decode(const zc_frame_header* h, const uint8_t* d_payload, uint64_t payload_len, uint8_t* d_dst,
                       uint64_t dst_len, int32_t* d_ok, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (h->raw_bytes == 0 || dst_len < h->raw_bytes) return cuda_err(cudaMemsetAsync(d_ok, 0, 4, s), "fixedlen_decode");
  if (!aligned16(d_payload)) return set_err(ZC_ERR_INVALID_ARGUMENT, "fixedlen_decode: payload must be 16-byte aligned");
  zc_frame_header hh = *h;
  hh.codec = ZC_CODEC_FIXEDLEN;
  DecParams p;
  std::memset(&p, 0, sizeof(p));
  p.stages = d_payload;
  p.region = payload_len;
  p.bare = 1;
  p.hdr = hh;
  p.nunits = 1;
  p.total_bytes = p.unit_bytes = hh.raw_bytes;
  p.out_kind = OUT_BYTES;
  p.out = d_dst;
  p.ok_out = d_ok;
  return decode_common(p, s);
}

// ------------------------------------------------------------------ huffman contexts
static zc_huff_ctx* new_ctx(const HostHuff& h) {
  auto* c = new zc_huff_ctx();
  c->h = h;
  return c;
}

int zc_huff_ctx_create(const uint64_t* hist, zc_huff_ctx** out) {
  *out = new_ctx(huffman_build(hist));
  return ZC_OK;
}

int zc_huff_ctx_create_from_bytes(const uint8_t* sample, uint64_t n, zc_huff_ctx** out) {
  uint64_t h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1;
  for (uint64_t i = 0; i < n; ++i) h[sample[i]]++;
  return zc_huff_ctx_create(h, out);
}

int zc_huff_ctx_create_from_device_bytes(const uint8_t* d_sample, uint64_t n, zc_huff_ctx** out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint64_t* d_h = nullptr;
  if (int rc = cuda_err(cudaMalloc(&d_h, 256 * 8), "malloc")) return rc;
  int rc = cuda_err(launch_hist(d_sample, n, d_h, s), "hist");
  uint64_t h[256];
  if (!rc) rc = cuda_err(cudaMemcpyAsync(h, d_h, sizeof(h), cudaMemcpyDeviceToHost, s), "copy");
  if (!rc) rc = cuda_err(cudaStreamSynchronize(s), "sync");
  cudaFree(d_h);
  if (rc) return rc;
  for (int i = 0; i < 256; ++i) h[i] += 1;  // +1 smoothing (collectives.cpp:102-104)
  return zc_huff_ctx_create(h, out);
}

int zc_huff_ctx_from_lengths(const uint8_t* lens, zc_huff_ctx** out) {
  std::array<uint8_t, 256> l;
  std::memcpy(l.data(), lens, 256);
  auto c = huffman_finalize(l);
  if (!c) {
    *out = nullptr;
    return set_err(ZC_ERR_INVALID_ARGUMENT, "code lengths do not form a valid prefix code");
  }
  *out = new_ctx(*c);
  return ZC_OK;
}

int zc_huff_ctx_valid(const zc_huff_ctx* c) { return c && c->h.valid ? 1 : 0; }

int zc_huff_ctx_code_lengths(const zc_huff_ctx* c, uint8_t* lens) {
  std::memcpy(lens, c->h.len.data(), 256);
  return ZC_OK;
}

int zc_huff_ctx_codes(const zc_huff_ctx* c, uint32_t* code, uint32_t* rev) {
  if (code) std::memcpy(code, c->h.code.data(), 256 * 4);
  if (rev) std::memcpy(rev, c->h.rev.data(), 256 * 4);
  return ZC_OK;
}

void zc_huff_ctx_destroy(zc_huff_ctx* c) {
  if (!c) return;
  for (auto& kv : c->dev) zc::release_device_memory(kv.first, kv.second, false);
  delete c;
}

int zc_huffman_expected_code_len(const zc_huff_ctx* c, const uint64_t* hist, double* bits, int32_t* valid) {
  auto r = c ? huffman_expected_len(c->h, hist) : std::nullopt;
  *valid = r ? 1 : 0;
  *bits = r ? *r : 0.0;
  return ZC_OK;
}

int zc_huffman_self_code_len(const uint64_t* hist, double* bits, int32_t* valid) {
  auto r = huffman_self_len(hist);
  *valid = r ? 1 : 0;
  *bits = r ? *r : 0.0;
  return ZC_OK;
}

int zc_huffman_encode(const uint8_t* d_raw, uint64_t n, const zc_huff_ctx* ctx, uint8_t* d_out, uint64_t out_cap,
                      int32_t embed, uint64_t* d_payload, uint32_t* d_index, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!ctx || !ctx->h.valid || (n == 0 && !embed)) return cuda_err(cudaMemsetAsync(d_payload, 0, 8, s), "huffman_encode");
  if (n == 0) {  // embedded, empty input: the codebook alone (huffman.cpp:219-225)
    if (out_cap < ZC_HUFF_CODEBOOK_BYTES) return cuda_err(cudaMemsetAsync(d_payload, 0, 8, s), "huffman_encode");
    static thread_local uint64_t k256;
    k256 = ZC_HUFF_CODEBOOK_BYTES;
    cudaMemcpyAsync(d_out, ctx->h.len.data(), 256, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_payload, &k256, 8, cudaMemcpyHostToDevice, s);
    return cuda_err(cudaStreamSynchronize(s), "huffman_encode");
  }
  if (!aligned16(d_out)) return set_err(ZC_ERR_INVALID_ARGUMENT, "huffman_encode: output must be 16-byte aligned");
  EncParams p = base_enc(nullptr, ctx, nullptr);
  if (!p.ctx) return set_err(ZC_ERR_CUDA, "cannot upload Huffman tables");
  p.src = d_raw;
  p.src_kind = SRC_BYTES;
  p.mode = ENC_BARE_HF;
  p.embed = embed ? 1 : 0;
  p.total_bytes = p.unit_bytes = n;
  p.nunits = 1;
  p.stages = d_out;
  p.stage_len = out_cap;
  p.bare_payload = d_payload;
  p.index = d_index;
  p.index_stride = (n + ZC_HUFF_INDEX_GRAIN - 1) / ZC_HUFF_INDEX_GRAIN;
  if (n >= (1ull << 27)) p.index = nullptr;  // u32 bit offsets
  return encode_common(p, s);
}

int zc_huffman_decode(const zc_frame_header* h, const uint8_t* d_payload, uint64_t payload_len,
                      const zc_huff_ctx* shared_ctx, const uint32_t* d_index, uint8_t* d_dst, uint64_t dst_len,
                      int32_t* d_ok, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dst_len < h->raw_bytes) return cuda_err(cudaMemsetAsync(d_ok, 0, 4, s), "huffman_decode");
  if (h->raw_bytes == 0) {
    // nothing to decode; the reference returns true after its preamble checks
    zc_frame_header hh = *h;
    bool ok = hh.payload_bytes <= payload_len &&
              ((hh.flags & ZC_FLAG_EMBEDDED_CODEBOOK) ? (hh.params == 256 && hh.payload_bytes >= 256)
                                                      : (hh.params == 0 && shared_ctx && shared_ctx->h.valid));
    static thread_local int32_t v;
    v = ok ? 1 : 0;
    cudaMemcpyAsync(d_ok, &v, 4, cudaMemcpyHostToDevice, s);
    return cuda_err(cudaStreamSynchronize(s), "huffman_decode");
  }
  if (!aligned16(d_payload)) return set_err(ZC_ERR_INVALID_ARGUMENT, "huffman_decode: payload must be 16-byte aligned");
  zc_frame_header hh = *h;
  hh.codec = ZC_CODEC_HUFFMAN;
  DecParams p;
  std::memset(&p, 0, sizeof(p));
  p.stages = d_payload;
  p.region = payload_len;
  p.bare = 1;
  p.hdr = hh;
  p.nunits = 1;
  p.total_bytes = p.unit_bytes = hh.raw_bytes;
  p.out_kind = OUT_BYTES;
  p.out = d_dst;
  p.ok_out = d_ok;
  p.ctx = device_tables(shared_ctx);
  p.index = d_index;
  p.index_stride = (hh.raw_bytes + ZC_HUFF_INDEX_GRAIN - 1) / ZC_HUFF_INDEX_GRAIN;
  return decode_common(p, s);
}

// ------------------------------------------------------------------ rea
int zc_profile_sample(const uint8_t* d_raw, uint64_t n, const zc_huff_ctx* ctx, zc_sample_stats* d_stats, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return cuda_err(cudaMemsetAsync(d_stats, 0, sizeof(zc_sample_stats), s), "profile_sample");
  EncParams p = base_enc(nullptr, ctx, nullptr);
  p.src = d_raw;
  p.src_kind = SRC_BYTES;
  p.mode = ENC_PROFILE;
  p.total_bytes = p.unit_bytes = n;
  p.nunits = 1;
  p.stages = nullptr;
  p.stage_len = ~0ull;
  p.stats = d_stats;
  return encode_common(p, s);
}

uint64_t zc_predict_payload(int32_t codec, uint64_t raw, const zc_sample_stats* st, const zc_arb_config* cfg) {
  return predict_payload(static_cast<uint32_t>(codec), raw, *st, *cfg);
}

int zc_arbitrate_plan(uint64_t raw, uint64_t cap, const zc_sample_stats* st, const zc_transport_hint* hint,
                      const zc_huff_ctx* ctx, const zc_arb_config* cfg, zc_arbitration_plan* out) {
  *out = arbitrate_plan(raw, cap, *st, *hint, ctx != nullptr && ctx->h.valid, *cfg);
  return ZC_OK;
}

int zc_encode_best(const uint8_t* d_raw, uint64_t raw_len, uint8_t* d_stage, uint64_t stage_len,
                   const zc_transport_hint* hint, const zc_huff_ctx* ctx, const zc_arb_config* cfg,
                   zc_encode_result* d_result, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (raw_len == 0 || stage_len <= ZC_HEADER_BYTES)
    return cuda_err(cudaMemsetAsync(d_result, 0, sizeof(zc_encode_result), s), "encode_best");
  if (!aligned16(d_stage)) return set_err(ZC_ERR_INVALID_ARGUMENT, "encode_best: stage must be 16-byte aligned");
  EncParams p = base_enc(hint, ctx, cfg);
  p.src = d_raw;
  p.src_kind = SRC_BYTES;
  p.mode = ENC_BEST;
  p.total_bytes = p.unit_bytes = raw_len;
  p.nunits = 1;
  p.stages = d_stage;
  p.stage_len = stage_len;
  p.results = d_result;
  return encode_common(p, s);
}

// ------------------------------------------------------------------ batched hot path
__attribute__((visibility("hidden"))) int zc_i_reserve_scratch(void* stream, uint32_t nunits) {
  return reserve_scratch(static_cast<cudaStream_t>(stream), nunits);
}

// One fused ring-step piece (zc_fixed.cu ring_fused_kernel): the received piece in `in_region` is
// reduced into `sum` (sink OUT_ADD_I32 in place, or OUT_ADD_Q from the local fp32 `x`) and the sums
// are framed (send_batch semantics, `pin`, no Huffman) into `out_region`.
__attribute__((visibility("hidden"))) int zc_i_ring_fused(const uint8_t* in_region, uint64_t stride,
                                                          const zc_encode_result* in_res, int sink, int32_t* sum,
                                                          const float* x, const double* dscale, uint64_t total,
                                                          uint64_t unit_bytes, uint8_t* out_region,
                                                          zc_encode_result* out_res, int32_t pin,
                                                          const zc_transport_hint* hint, const zc_arb_config* cfg,
                                                          uint32_t* d_err, void* stream) {
  if (total == 0) return ZC_OK;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch* sc = scratch_for(s, 1);
  const uint32_t nunits = static_cast<uint32_t>((total + unit_bytes - 1) / unit_bytes);
  if (!sc || sc->task_bytes < ring_fused_scratch_bytes(nunits))
    return set_err(ZC_ERR_CUDA, "fused ring step: scratch not reserved");
  FusedParams f;
  std::memset(&f, 0, sizeof(f));
  f.in_stages = in_region;
  f.in_stride = stride;
  f.in_res = in_res;
  f.sink = sink;
  f.sum = sum;
  f.x = x;
  f.dscale = dscale;
  f.err = d_err ? d_err : sc->sink;
  EncParams& p = f.enc;
  p = base_enc(hint, nullptr, cfg);
  p.src = sum;
  p.src_kind = SRC_BYTES;
  p.mode = ENC_SEND;
  p.pin = pin;
  p.total_bytes = total;
  p.unit_bytes = unit_bytes;
  p.nunits = nunits;
  p.stages = out_region;
  p.stride = stride;
  p.stage_len = ZC_STAGE_BANK_BYTES;
  p.results = out_res;
  p.err = f.err;
  return cuda_err(launch_ring_fused(f, sc->task, s), "fused ring step");
}

__attribute__((visibility("hidden"))) int zc_i_encode_batches(const void* src, int kind, uint64_t total, double scale, const zc_i_batch_opts* o, uint8_t* d_stages, uint64_t stride,
                          uint64_t stage_len, int32_t pin, const zc_transport_hint* hint, const zc_huff_ctx* ctx,
                          const zc_arb_config* cfg, zc_encode_result* d_results, uint32_t* d_index, uint32_t* d_err,
                          void* stream) {
  if (total == 0) return ZC_OK;
  if (!aligned16(d_stages) || (stride & 15)) return set_err(ZC_ERR_INVALID_ARGUMENT, "stages must be 16-byte aligned");
  if (pin < ZC_PIN_AUTO || pin > ZC_PIN_HUFFMAN) return set_err(ZC_ERR_INVALID_ARGUMENT, "unknown codec pin");
  EncParams p = base_enc(hint, ctx, cfg);
  p.src = src;
  p.src_kind = kind;
  p.mode = ENC_SEND;
  p.pin = pin;
  p.scale = scale;
  p.rcp = 1.0 / scale;
  const uint64_t unit_bytes = o && o->unit_bytes ? o->unit_bytes : ZC_BATCH_RAW_BYTES;
  p.total_bytes = total;
  p.unit_bytes = unit_bytes;
  p.nunits = static_cast<uint32_t>((total + unit_bytes - 1) / unit_bytes);
  p.dscale = o ? o->dscale : nullptr;
  p.maxzz_in = o ? o->maxzz_in : nullptr;
  p.no_spec = o ? o->no_spec : 0;
  p.stages = d_stages;
  p.stride = stride;
  p.stage_len = stage_len;
  p.results = d_results;
  p.index = d_index;
  p.index_stride = ZC_HUFF_INDEX_ENTRIES;
  p.err = d_err;
  return encode_common(p, static_cast<cudaStream_t>(stream));
}

int zc_encode_batches_sym(const int32_t* d_sym, uint64_t raw_bytes, uint8_t* d_stages, uint64_t stride,
                          uint64_t stage_len, int32_t pin, const zc_transport_hint* hint, const zc_huff_ctx* ctx,
                          const zc_arb_config* cfg, zc_encode_result* d_results, uint32_t* d_index, uint32_t* d_err,
                          void* stream) {
  return zc_i_encode_batches(d_sym, SRC_BYTES, raw_bytes, 1.0, nullptr, d_stages, stride, stage_len, pin, hint, ctx, cfg, d_results,
                        d_index, d_err, stream);
}

int zc_encode_batches_f32(const float* d_x, uint64_t count, double scale, uint8_t* d_stages, uint64_t stride,
                          uint64_t stage_len, int32_t pin, const zc_transport_hint* hint, const zc_huff_ctx* ctx,
                          const zc_arb_config* cfg, zc_encode_result* d_results, uint32_t* d_index, uint32_t* d_err,
                          void* stream) {
  if (int rc = check_scale(scale, "eb_quantize_chunk")) return rc;
  if (!aligned16(d_x)) return set_err(ZC_ERR_INVALID_ARGUMENT, "input must be 16-byte aligned");
  return zc_i_encode_batches(d_x, SRC_F32, count * 4, scale, nullptr, d_stages, stride, stage_len, pin, hint, ctx, cfg, d_results,
                        d_index, d_err, stream);
}

__attribute__((visibility("hidden"))) int zc_i_decode_batches(const uint8_t* d_stages, const zc_i_batch_opts* o, uint64_t stride, uint64_t stage_len, const zc_encode_result* d_sent,
                          uint64_t total, const zc_huff_ctx* ctx, const uint32_t* d_index, int out_kind, void* out,
                          double scale, uint32_t* d_codec, uint32_t* d_err, void* stream, int own_frames) {
  if (total == 0) return ZC_OK;
  if (!aligned16(d_stages) || (stride & 15)) return set_err(ZC_ERR_INVALID_ARGUMENT, "stages must be 16-byte aligned");
  DecParams p;
  std::memset(&p, 0, sizeof(p));
  p.stages = d_stages;
  p.stride = stride;
  p.region = stage_len;
  p.frame_len = d_sent;
  const uint64_t unit_bytes = o && o->unit_bytes ? o->unit_bytes : ZC_BATCH_RAW_BYTES;
  p.total_bytes = total;
  p.unit_bytes = unit_bytes;
  p.nunits = static_cast<uint32_t>((total + unit_bytes - 1) / unit_bytes);
  p.dscale = o ? o->dscale : nullptr;
  p.acc_f32 = o ? o->acc_f32 : nullptr;
  p.maxzz_out = o ? o->maxzz_out : nullptr;
  p.out_kind = out_kind;
  p.out = out;
  p.scale = scale;
  p.ctx = device_tables(ctx);
  p.index = d_index;
  p.index_stride = ZC_HUFF_INDEX_ENTRIES;
  p.codec_out = d_codec;
  p.err = d_err;
  p.own_frames = own_frames;
  return decode_common(p, static_cast<cudaStream_t>(stream));
}

int zc_decode_batches_sym(const uint8_t* d_stages, uint64_t stride, uint64_t stage_len, const zc_encode_result* d_sent,
                          uint64_t raw_bytes, const zc_huff_ctx* ctx, const uint32_t* d_index, int32_t* d_sym,
                          uint32_t* d_codec_out, void* stream) {
  return zc_i_decode_batches(d_stages, nullptr, stride, stage_len, d_sent, raw_bytes, ctx, d_index, OUT_BYTES, d_sym, 1.0, d_codec_out,
                        nullptr, stream, 0);
}

int zc_decode_batches_f32(const uint8_t* d_stages, uint64_t stride, uint64_t stage_len, const zc_encode_result* d_sent,
                          uint64_t count, double scale, const zc_huff_ctx* ctx, const uint32_t* d_index, float* d_out,
                          uint32_t* d_codec_out, void* stream) {
  return zc_i_decode_batches(d_stages, nullptr, stride, stage_len, d_sent, count * 4, ctx, d_index, OUT_F32, d_out, scale,
                        d_codec_out, nullptr, stream, 0);
}

int zc_decode_batches_add_sym(const uint8_t* d_stages, uint64_t stride, uint64_t stage_len,
                              const zc_encode_result* d_sent, uint64_t raw_bytes, const zc_huff_ctx* ctx,
                              const uint32_t* d_index, int32_t* d_acc, uint32_t* d_err, void* stream) {
  return zc_i_decode_batches(d_stages, nullptr, stride, stage_len, d_sent, raw_bytes, ctx, d_index, OUT_ADD_I32, d_acc, 1.0, nullptr,
                        d_err, stream, 0);
}

}  // extern "C"

// ------------------------------------------------------------------ host-buffer pipelines
// Three internal streams per device — H2D copies, kernels, D2H copies — chained per group by
// events, so the copy engines stream back to back in both directions (PCIe is full duplex) while
// the kernels of group g run between H2D(g) and D2H(g).  Each stream has its own scratch.
namespace {
constexpr int kEv = 4;
struct Pipe {
  cudaStream_t h2d = nullptr, work = nullptr, d2h = nullptr;
  cudaEvent_t in[kEv] = {}, done[kEv] = {};
  cudaEvent_t start = nullptr, fin_work = nullptr, fin_d2h = nullptr;
  bool ok = false;
};
std::mutex g_pipe_mu;
std::map<int, Pipe> g_pipes;

Pipe* pipe_for_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(g_pipe_mu);
  Pipe& pp = g_pipes[dev];
  if (!pp.ok) {
    for (cudaStream_t* s : {&pp.h2d, &pp.work, &pp.d2h})
      if (cudaStreamCreateWithFlags(s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    for (int i = 0; i < kEv; ++i)
      if (cudaEventCreateWithFlags(&pp.in[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&pp.done[i], cudaEventDisableTiming) != cudaSuccess)
        return nullptr;
    for (cudaEvent_t* e : {&pp.start, &pp.fin_work, &pp.fin_d2h})
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    pp.ok = true;
  }
  return &pp;
}
}  // namespace

extern "C" int zc_codec_roundtrip_host_f32(const float* h_x, uint64_t count, double scale, float* d_work,
                                           uint8_t* d_stages, uint64_t stride, uint64_t stage_len, int32_t pin,
                                           const zc_transport_hint* hint, const zc_huff_ctx* ctx,
                                           const zc_arb_config* cfg, zc_encode_result* d_results, uint32_t* d_index,
                                           uint32_t* d_err, float* h_y, uint32_t group_batches, void* stream) {
  if (count == 0) return ZC_OK;
  if (h_x == nullptr || h_y == nullptr || d_work == nullptr) return set_err(ZC_ERR_INVALID_ARGUMENT, "null buffer");
  if (int rc = check_scale(scale, "eb_quantize_chunk")) return rc;
  if (!aligned16(d_work)) return set_err(ZC_ERR_INVALID_ARGUMENT, "work buffer must be 16-byte aligned");
  Pipe* pp = pipe_for_device();
  if (pp == nullptr) return set_err(ZC_ERR_CUDA, "cannot create pipeline streams (no CUDA device?)");
  const cudaStream_t caller = static_cast<cudaStream_t>(stream);
  const uint64_t per = ZC_BATCH_RAW_BYTES / 4;  // elements per batch
  const uint64_t nb = (count + per - 1) / per;
  const uint64_t gb = group_batches ? group_batches : 4;
  // Group sizes ramp 1, 2, 4, ... up to gb at the start and back down at the end: the first H2D
  // and the last D2H run alone (nothing to overlap them with), so short edge groups keep both copy
  // directions busy for almost the whole call while the middle groups amortise their launches.
  std::vector<uint64_t> sizes;
  {
    std::vector<uint64_t> head, tail;
    uint64_t left = nb;
    for (uint64_t k = 1; k < gb && left > 2 * k; k *= 2) {
      head.push_back(k);
      tail.push_back(k);
      left -= 2 * k;
    }
    sizes = head;
    for (; left >= gb; left -= gb) sizes.push_back(gb);
    if (left) sizes.push_back(left);
    sizes.insert(sizes.end(), tail.rbegin(), tail.rend());
  }
  const uint64_t ngroups = sizes.size();
  // frames of this call's own encoder: without a usable Huffman path every valid frame is
  // FixedLen / RAW and the general decode kernels have nothing to do
  // (embedded codebooks: Auto may pick Huffman without a shared context, rea.cpp:160)
  const bool embed = cfg != nullptr && cfg->embed_codebook != 0;
  const int own = (pin == ZC_PIN_RAW || pin == ZC_PIN_FIXEDLEN || (ctx == nullptr && !embed)) ? 1 : 0;
  if (int rc = cuda_err(cudaEventRecord(pp->start, caller), "pipeline start")) return rc;
  for (cudaStream_t s : {pp->h2d, pp->work, pp->d2h})
    if (int rc = cuda_err(cudaStreamWaitEvent(s, pp->start, 0), "pipeline wait")) return rc;
  uint64_t b0 = 0;
  for (uint64_t g = 0; g < ngroups; b0 += sizes[g], ++g) {
    const uint64_t e0 = b0 * per;
    const uint64_t n = (count - e0) < sizes[g] * per ? (count - e0) : sizes[g] * per;
    cudaEvent_t in = pp->in[g % kEv], done = pp->done[g % kEv];
    if (int rc = cuda_err(cudaMemcpyAsync(d_work + e0, h_x + e0, n * 4, cudaMemcpyHostToDevice, pp->h2d), "H2D")) return rc;
    if (int rc = cuda_err(cudaEventRecord(in, pp->h2d), "H2D event")) return rc;
    if (int rc = cuda_err(cudaStreamWaitEvent(pp->work, in, 0), "H2D wait")) return rc;
    if (int rc = zc_i_encode_batches(d_work + e0, SRC_F32, n * 4, scale, nullptr, d_stages + b0 * stride, stride, stage_len, pin, hint,
                                ctx, cfg, d_results + b0, d_index ? d_index + b0 * ZC_HUFF_INDEX_ENTRIES : nullptr,
                                d_err, pp->work))
      return rc;
    // decoded in place: the group's encode has consumed its input (stream order)
    if (int rc = zc_i_decode_batches(d_stages + b0 * stride, nullptr, stride, stage_len, d_results + b0, n * 4, ctx,
                                d_index ? d_index + b0 * ZC_HUFF_INDEX_ENTRIES : nullptr, OUT_F32, d_work + e0, scale,
                                nullptr, d_err, pp->work, own))
      return rc;
    if (int rc = cuda_err(cudaEventRecord(done, pp->work), "kernel event")) return rc;
    if (int rc = cuda_err(cudaStreamWaitEvent(pp->d2h, done, 0), "kernel wait")) return rc;
    if (int rc = cuda_err(cudaMemcpyAsync(h_y + e0, d_work + e0, n * 4, cudaMemcpyDeviceToHost, pp->d2h), "D2H")) return rc;
  }
  if (int rc = cuda_err(cudaEventRecord(pp->fin_work, pp->work), "pipeline done")) return rc;
  if (int rc = cuda_err(cudaEventRecord(pp->fin_d2h, pp->d2h), "pipeline done")) return rc;
  if (int rc = cuda_err(cudaStreamWaitEvent(caller, pp->fin_work, 0), "pipeline join")) return rc;
  return cuda_err(cudaStreamWaitEvent(caller, pp->fin_d2h, 0), "pipeline join");
}
