// zcomm_b200.hpp — header-only C++17 layer over the C-ABI (zcomm_b200.h) that restores the
// reference's C++ conventions: namespace zcomm, the reference function names, and exceptions of the
// reference's types instead of status codes (std::invalid_argument, std::overflow_error,
// std::runtime_error, std::logic_error).  Data pointers are DEVICE pointers; results that the
// reference returns by value are returned in device memory or, where the reference's caller needs
// them on the host (sizes, decisions), copied back by the *_sync helpers.
//
// Reference headers this replaces (relative to /root/reference/proj/core/include/zcomm/):
// frame.hpp, quant.hpp, fixedlen.hpp, huffman.hpp, rea.hpp, collectives.hpp.
#pragma once
#include <cstdint>
#include <exception>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "zcomm_b200.h"

namespace zcomm {
namespace b200 {

// A peer aborted or timed out (the reference surfaces the root cause through Communicator::run).
struct PeerError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == ZC_OK) return;
  const char* m = zc_last_error();
  std::string msg = m ? m : "";
  switch (rc) {
    case ZC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ZC_ERR_OVERFLOW: throw std::overflow_error(msg);
    case ZC_ERR_LOGIC: throw std::logic_error(msg);
    case ZC_ERR_PEER: throw PeerError(msg);
    case ZC_ERR_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

using FrameHeader = zc_frame_header;
using ArbitrationConfig = zc_arb_config;
using TransportHint = zc_transport_hint;
using SampleStats = zc_sample_stats;
using ArbitrationPlan = zc_arbitration_plan;
using EncodeResult = zc_encode_result;
using WireStats = zc_wire_stats;
using CollectiveConfig = zc_collective_config;

inline ArbitrationConfig default_arbitration_config() {
  ArbitrationConfig c;
  zc_default_arb_config(&c);
  return c;
}
inline TransportHint default_transport_hint() {
  TransportHint h;
  zc_default_transport_hint(&h);
  return h;
}
inline CollectiveConfig default_collective_config() {
  CollectiveConfig c;
  zc_default_collective_config(&c);
  return c;
}
inline FrameHeader make_header(uint8_t codec, uint64_t raw, uint64_t payload, uint64_t params = 0, uint16_t flags = 0) {
  return FrameHeader{ZC_FRAME_MAGIC, ZC_FRAME_VERSION, codec, flags, raw, payload, params};
}

// ---- frame.hpp:38-50 (host)
inline void write_header(const FrameHeader& h, uint8_t* dst, size_t len) { check(zc_write_header(&h, dst, len)); }
inline std::optional<FrameHeader> parse_header(const uint8_t* src, size_t len) {
  FrameHeader h;
  if (zc_parse_header(src, len, &h) != ZC_OK) return std::nullopt;
  return h;
}
inline bool validate_header(const FrameHeader& h, size_t region) { return zc_validate_header(&h, region) == 1; }

// ---- rea.cpp:240-279 (host)
inline void load_arbitration_config(const std::string& text, ArbitrationConfig& cfg) {
  check(zc_load_arbitration_config(text.c_str(), &cfg));
}
inline void apply_env_overrides(ArbitrationConfig& cfg) { check(zc_apply_env_overrides(&cfg)); }

// ---- quant.hpp:29-53 (device pointers, stream-ordered; device-side errors land in d_err)
inline void eb_quantize_chunk(const float* d_x, size_t n, double scale, int32_t* d_sym, uint32_t* d_err,
                              void* stream = nullptr) {
  check(zc_eb_quantize_f32(d_x, n, scale, d_sym, d_err, stream));
}
inline void eb_quantize_chunk(const double* d_x, size_t n, double scale, int32_t* d_sym, uint32_t* d_err,
                              void* stream = nullptr) {
  check(zc_eb_quantize_f64(d_x, n, scale, d_sym, d_err, stream));
}
// eb_quantize (quant.cpp:30-41): returns the scale.
inline double eb_quantize(const float* d_x, size_t n, double rel, int32_t* d_sym, void* stream = nullptr) {
  double s = 0.0;
  check(zc_eb_quantize_rel_f32(d_x, n, rel, d_sym, &s, stream));
  return s;
}
inline void dequantize_into(const int32_t* d_sym, size_t n, int32_t mode, double scale, uint32_t levels,
                            double* d_out, void* stream = nullptr) {
  check(zc_dequantize_f64(d_sym, n, mode, scale, levels, d_out, stream));
}
inline void dequantize_into(const int32_t* d_sym, size_t n, int32_t mode, double scale, uint32_t levels,
                            float* d_out, void* stream = nullptr) {
  check(zc_dequantize_f32(d_sym, n, mode, scale, levels, d_out, stream));
}

// ---- huffman.hpp:20-70: immutable shared context (RAII)
class HuffmanContext {
 public:
  static HuffmanContext build(const uint64_t hist256[256]) {
    zc_huff_ctx* c = nullptr;
    check(zc_huff_ctx_create(hist256, &c));
    return HuffmanContext(c);
  }
  static HuffmanContext from_bytes(const uint8_t* h_sample, size_t n) {
    zc_huff_ctx* c = nullptr;
    check(zc_huff_ctx_create_from_bytes(h_sample, n, &c));
    return HuffmanContext(c);
  }
  static std::optional<HuffmanContext> from_lengths(const uint8_t lens256[256]) {
    zc_huff_ctx* c = nullptr;
    int rc = zc_huff_ctx_from_lengths(lens256, &c);
    if (rc == ZC_ERR_INVALID_ARGUMENT) return std::nullopt;
    check(rc);
    return HuffmanContext(c);
  }
  bool valid() const { return zc_huff_ctx_valid(h_.get()) == 1; }
  std::vector<uint8_t> code_lengths() const {
    std::vector<uint8_t> l(256);
    check(zc_huff_ctx_code_lengths(h_.get(), l.data()));
    return l;
  }
  std::optional<double> expected_code_len(const uint64_t hist256[256]) const {
    double b = 0;
    int32_t v = 0;
    check(zc_huffman_expected_code_len(h_.get(), hist256, &b, &v));
    if (!v) return std::nullopt;
    return b;
  }
  const zc_huff_ctx* get() const { return h_.get(); }

 private:
  explicit HuffmanContext(zc_huff_ctx* c) : h_(c, &zc_huff_ctx_destroy) {}
  std::shared_ptr<zc_huff_ctx> h_;
};

inline std::optional<double> huffman_self_code_len(const uint64_t hist256[256]) {
  double b = 0;
  int32_t v = 0;
  check(zc_huffman_self_code_len(hist256, &b, &v));
  if (!v) return std::nullopt;
  return b;
}

// ---- rea.hpp:114-133
inline uint64_t predict_payload(int32_t codec, uint64_t raw, const SampleStats& st, const ArbitrationConfig& cfg) {
  return zc_predict_payload(codec, raw, &st, &cfg);
}
inline ArbitrationPlan arbitrate_plan(uint64_t raw, uint64_t cap, const SampleStats& st, const TransportHint& hint,
                                      const HuffmanContext* ctx, const ArbitrationConfig& cfg) {
  ArbitrationPlan p;
  check(zc_arbitrate_plan(raw, cap, &st, &hint, ctx ? ctx->get() : nullptr, &cfg, &p));
  return p;
}
// encode_best: result stays on the device (d_result); no host round-trip.
inline void encode_best(const uint8_t* d_raw, size_t n, uint8_t* d_stage, size_t stage_len, const TransportHint& hint,
                        const HuffmanContext* ctx, const ArbitrationConfig& cfg, EncodeResult* d_result,
                        void* stream = nullptr) {
  check(zc_encode_best(d_raw, n, d_stage, stage_len, &hint, ctx ? ctx->get() : nullptr, &cfg, d_result, stream));
}

// Device scratch for the host-returning helpers below (RAII over zc_device_malloc).
class DeviceScratch {
 public:
  explicit DeviceScratch(size_t bytes) {
    void* p = nullptr;
    check(zc_device_malloc(bytes, &p));
    p_ = p;
  }
  ~DeviceScratch() { zc_device_free(p_); }
  DeviceScratch(const DeviceScratch&) = delete;
  DeviceScratch& operator=(const DeviceScratch&) = delete;
  template <class T>
  T* as(size_t byte_off = 0) const {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(p_) + byte_off);
  }

 private:
  void* p_ = nullptr;
};
// A device result of work queued on `stream`, read once that work is complete.
template <class T>
inline T read_back(const T* d_src, void* stream) {
  check(zc_stream_synchronize(stream));
  T v;
  check(zc_memcpy(&v, d_src, sizeof(T)));
  return v;
}

// ---- frame.hpp:52-58: frame_commit_raw on the device; returns the committed frame size (0: no room).
inline size_t frame_commit_raw(const uint8_t* d_raw, size_t n, uint8_t* d_region, size_t region_len,
                               void* stream = nullptr) {
  DeviceScratch s(8);
  check(zc_frame_commit_raw(d_raw, n, d_region, region_len, s.as<uint64_t>(), stream));
  return static_cast<size_t>(read_back(s.as<uint64_t>(), stream));
}

// ---- the coder plugins (fixedlen.hpp:22-42, huffman.hpp:38-70), device spans.  Return values
// follow the reference: encoders return the payload size (0 when it does not fit), decoders
// whether the payload decoded.
inline size_t fixedlen_encode(const int32_t* d_syms, size_t n, uint8_t* d_dst, size_t cap, unsigned* width,
                              void* stream = nullptr) {
  DeviceScratch s(16);
  check(zc_fixedlen_encode(d_syms, n, d_dst, cap, s.as<uint64_t>(), s.as<uint32_t>(8), stream));
  if (width) *width = read_back(s.as<uint32_t>(8), stream);
  return static_cast<size_t>(read_back(s.as<uint64_t>(), stream));
}
inline bool fixedlen_decode_into(const FrameHeader& h, const uint8_t* d_payload, size_t payload_len, uint8_t* d_dst,
                                 size_t dst_len, void* stream = nullptr) {
  DeviceScratch s(4);
  check(zc_fixedlen_decode(&h, d_payload, payload_len, d_dst, dst_len, s.as<int32_t>(), stream));
  return read_back(s.as<int32_t>(), stream) == 1;
}
// huffman_encode: with embed, the payload starts with the 256 code lengths (huffman.cpp:216-246).
// d_index (optional, ZC_HUFF_INDEX_ENTRIES u32): the companion index for the chunk-parallel decode.
inline size_t huffman_encode(const uint8_t* d_raw, size_t n, const HuffmanContext& ctx, uint8_t* d_dst, size_t cap,
                             bool embed, uint32_t* d_index = nullptr, void* stream = nullptr) {
  DeviceScratch s(8);
  check(zc_huffman_encode(d_raw, n, ctx.get(), d_dst, cap, embed ? 1 : 0, s.as<uint64_t>(), d_index, stream));
  return static_cast<size_t>(read_back(s.as<uint64_t>(), stream));
}
inline bool huffman_decode_into(const FrameHeader& h, const uint8_t* d_payload, size_t payload_len,
                                const HuffmanContext* shared, uint8_t* d_dst, size_t dst_len,
                                const uint32_t* d_index = nullptr, void* stream = nullptr) {
  DeviceScratch s(4);
  check(zc_huffman_decode(&h, d_payload, payload_len, shared ? shared->get() : nullptr, d_index, d_dst, dst_len,
                          s.as<int32_t>(), stream));
  return read_back(s.as<int32_t>(), stream) == 1;
}

// ---- rea.cpp:93-118: profile_sample of a device span (the sample window is the first 64 KiB).
inline SampleStats profile_sample(const uint8_t* d_raw, size_t n, const HuffmanContext* ctx, void* stream = nullptr) {
  DeviceScratch s(sizeof(SampleStats));
  check(zc_profile_sample(d_raw, n, ctx ? ctx->get() : nullptr, s.as<SampleStats>(), stream));
  return read_back(s.as<SampleStats>(), stream);
}

// ---- collectives.hpp:48-110: the per-rank face of a communicator (non-owning).  Every call runs
// on the rank's own stream after the caller's `stream` work and returns when complete, like the
// reference's blocking RankCtx methods.  Buffers are device pointers.
class RankCtx {
 public:
  explicit RankCtx(zc_comm* c) : c_(c) {}
  int rank() const { return zc_comm_rank(c_); }
  int nranks() const { return zc_comm_nranks(c_); }
  // point-to-point (collectives.cpp:350-364): batched, framed per send_batch, decoded per recv_batch
  void send_encoded(int peer, const void* d_raw, size_t bytes, void* stream = nullptr) {
    check(zc_comm_send_encoded(c_, peer, d_raw, bytes, stream));
  }
  void recv_decoded(int peer, void* d_dst, size_t bytes, void* stream = nullptr) {
    check(zc_comm_recv_decoded(c_, peer, d_dst, bytes, stream));
  }
  // RankCtx::allreduce(QuantizedStream&): symbols in place; returns the reconciled scale.
  double allreduce(int32_t* d_sym, size_t count, double scale, int32_t mode = ZC_QUANT_ERROR_BOUNDED,
                   uint32_t levels = 0, void* stream = nullptr) {
    check(zc_comm_allreduce_sym(c_, d_sym, count, mode, &scale, levels, stream));
    return scale;
  }
  void allreduce_eb(const float* d_x, float* d_out, size_t count, double rel, void* stream = nullptr) {
    check(zc_comm_allreduce_eb_f32(c_, d_x, d_out, 0, count, rel, stream));
  }
  void allreduce_eb(const float* d_x, double* d_out, size_t count, double rel, void* stream = nullptr) {
    check(zc_comm_allreduce_eb_f32(c_, d_x, d_out, 1, count, rel, stream));
  }
  void reduce_scatter(int32_t* d_sym, size_t count, void* stream = nullptr) {
    check(zc_comm_reduce_scatter_sym(c_, d_sym, count, stream));
  }
  void allgather(int32_t* d_all, size_t block, void* stream = nullptr) {
    check(zc_comm_allgather_sym(c_, d_all, block, stream));
  }
  void alltoall(const int32_t* d_send, int32_t* d_recv, size_t block, void* stream = nullptr) {
    check(zc_comm_alltoall_sym(c_, d_send, d_recv, block, stream));
  }
  void broadcast(int32_t* d_data, size_t count, int root, void* stream = nullptr) {
    check(zc_comm_broadcast_sym(c_, d_data, count, root, stream));
  }
  void group_execute(std::vector<zc_coll_request>& reqs, void* stream = nullptr) {
    check(zc_comm_group_execute(c_, reqs.data(), static_cast<int32_t>(reqs.size()), stream));
  }
  double allreduce_max(double v, void* stream = nullptr) {
    double o = 0;
    check(zc_comm_allreduce_max(c_, v, &o, stream));
    return o;
  }
  zc_comm* get() const { return c_; }

 private:
  zc_comm* c_;
};

// ---- collectives.hpp:111-153, single process: Communicator(n, cfg) + run(fn) with one thread per
// rank (ranks on local devices; several may share one GPU).  A rank whose body throws poisons
// every link (zc_comm_abort), so peers blocked on it fail with PeerError; run() then resets the
// communicator and rethrows the root cause (the first exception that is not a PeerError).
class LocalCommunicator {
 public:
  LocalCommunicator(int nranks, const std::vector<int>& devices, const CollectiveConfig& cfg) : cs_(nranks, nullptr) {
    check(zc_comm_create_group(nranks, devices.data(), &cfg, cs_.data()));
  }
  LocalCommunicator(int nranks, int device, const CollectiveConfig& cfg)
      : LocalCommunicator(nranks, std::vector<int>(static_cast<size_t>(nranks), device), cfg) {}
  ~LocalCommunicator() {
    for (zc_comm* c : cs_) zc_comm_destroy(c);
  }
  LocalCommunicator(const LocalCommunicator&) = delete;
  LocalCommunicator& operator=(const LocalCommunicator&) = delete;
  int nranks() const { return static_cast<int>(cs_.size()); }
  void set_shared_huffman(const HuffmanContext& ctx) {
    for (zc_comm* c : cs_) check(zc_comm_set_shared_huffman(c, ctx.get()));
  }
  template <class F>
  void run(F&& fn) {
    const int n = nranks();
    std::vector<std::exception_ptr> errs(static_cast<size_t>(n));
    std::vector<std::thread> th;
    for (int r = 0; r < n; ++r)
      th.emplace_back([&, r] {
        try {
          RankCtx ctx(cs_[static_cast<size_t>(r)]);
          fn(ctx);
        } catch (...) {
          errs[static_cast<size_t>(r)] = std::current_exception();
          zc_comm_abort(cs_[static_cast<size_t>(r)]);
        }
      });
    for (auto& t : th) t.join();
    zc_flush_deferred();
    std::exception_ptr root, any;
    for (auto& e : errs) {
      if (!e) continue;
      if (!any) any = e;
      if (!root) {
        try {
          std::rethrow_exception(e);
        } catch (const PeerError&) {
        } catch (...) {
          root = e;
        }
      }
    }
    if (!any) return;
    for (zc_comm* c : cs_) zc_comm_reset(c);
    std::rethrow_exception(root ? root : any);
  }
  // Communicator::wire_stats (collectives.cpp:175-186): summed over ranks.
  WireStats wire_stats() const {
    WireStats s{};
    for (zc_comm* c : cs_) {
      WireStats w;
      check(zc_comm_wire_stats(c, &w));
      for (int i = 0; i < 3; ++i) s.frames_by_codec[i] += w.frames_by_codec[i];
      s.raw_bytes += w.raw_bytes;
      s.payload_bytes += w.payload_bytes;
      s.total_bytes += w.total_bytes;
      s.index_bytes += w.index_bytes;
      s.wall_codec_sec += w.wall_codec_sec;
    }
    return s;
  }
  void reset_stats() {
    for (zc_comm* c : cs_) check(zc_comm_reset_stats(c));
  }
  RankCtx rank_ctx(int r) const { return RankCtx(cs_.at(static_cast<size_t>(r))); }

 private:
  std::vector<zc_comm*> cs_;
};

// ---- collectives.hpp:48-153: one rank of a multi-process communicator (RAII)
class Communicator {
 public:
  // Bootstrap: `allgather(blob) -> all ranks' blobs concatenated in rank order` (MPI, torch.distributed,
  // a file, ...).  The data path never uses it.
  template <class AllGather>
  Communicator(int rank, int nranks, int device, const CollectiveConfig& cfg, AllGather&& allgather) {
    zc_comm* c = nullptr;
    check(zc_comm_create(rank, nranks, device, &cfg, &c));
    h_.reset(c);
    std::vector<uint8_t> blob(static_cast<size_t>(zc_comm_export_size()));
    check(zc_comm_export(c, blob.data()));
    std::vector<uint8_t> all = allgather(blob);
    check(zc_comm_connect(c, all.data()));
  }
  void set_shared_huffman(const HuffmanContext& ctx) { check(zc_comm_set_shared_huffman(h_.get(), ctx.get())); }
  // Communicator::run for this process's rank: fn(RankCtx&).
  template <class F>
  void run(F&& fn) {
    RankCtx ctx(h_.get());
    fn(ctx);
  }
  RankCtx rank_ctx() const { return RankCtx(h_.get()); }
  void send_encoded(int peer, const void* d_raw, size_t bytes) { rank_ctx().send_encoded(peer, d_raw, bytes); }
  void recv_decoded(int peer, void* d_dst, size_t bytes) { rank_ctx().recv_decoded(peer, d_dst, bytes); }
  // RankCtx::allreduce(QuantizedStream&): symbols in place; returns the reconciled scale.
  double allreduce(int32_t* d_sym, size_t count, double scale, int32_t mode = ZC_QUANT_ERROR_BOUNDED,
                   uint32_t levels = 0) {
    check(zc_comm_allreduce_sym(h_.get(), d_sym, count, mode, &scale, levels, nullptr));
    return scale;
  }
  void allreduce_eb(const float* d_x, float* d_out, size_t count, double rel) {
    check(zc_comm_allreduce_eb_f32(h_.get(), d_x, d_out, 0, count, rel, nullptr));
  }
  void allreduce_eb(const float* d_x, double* d_out, size_t count, double rel) {
    check(zc_comm_allreduce_eb_f32(h_.get(), d_x, d_out, 1, count, rel, nullptr));
  }
  void reduce_scatter(int32_t* d_sym, size_t count) { check(zc_comm_reduce_scatter_sym(h_.get(), d_sym, count, nullptr)); }
  void allgather(int32_t* d_all, size_t block) { check(zc_comm_allgather_sym(h_.get(), d_all, block, nullptr)); }
  // RankCtx::alltoall / broadcast (collectives.cpp:546-591), device buffers.
  void alltoall(const int32_t* d_send, int32_t* d_recv, size_t block) {
    check(zc_comm_alltoall_sym(h_.get(), d_send, d_recv, block, nullptr));
  }
  void broadcast(int32_t* d_data, size_t count, int root) {
    check(zc_comm_broadcast_sym(h_.get(), d_data, count, root, nullptr));
  }
  // group_execute (collectives.cpp:593-616): requests run in order as one submission.
  void group_execute(std::vector<zc_coll_request>& reqs) {
    check(zc_comm_group_execute(h_.get(), reqs.data(), static_cast<int32_t>(reqs.size()), nullptr));
  }
  double allreduce_max(double v) {
    double o = 0;
    check(zc_comm_allreduce_max(h_.get(), v, &o, nullptr));
    return o;
  }
  WireStats wire_stats() {
    WireStats w;
    check(zc_comm_wire_stats(h_.get(), &w));
    return w;
  }
  void reset() { check(zc_comm_reset(h_.get())); }
  int rank() const { return zc_comm_rank(h_.get()); }
  int nranks() const { return zc_comm_nranks(h_.get()); }
  zc_comm* get() const { return h_.get(); }

 private:
  std::unique_ptr<zc_comm, void (*)(zc_comm*)> h_{nullptr, &zc_comm_destroy};
};

}  // namespace b200
}  // namespace zcomm
