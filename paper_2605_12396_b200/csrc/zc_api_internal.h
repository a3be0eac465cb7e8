// zc_api_internal.h — helpers shared by the C-ABI translation units (not exported).
#pragma once
#include <string>

#include "zc_kernels.h"

namespace zc {
int set_err(int code, const std::string& msg);
// Deferred frees.  cudaFree (and cudaIpcCloseMemHandle) wait for the whole device; called while a
// collective of a single-process group is in flight — e.g. a garbage-collected communicator or
// Huffman context released on a rank thread — it would wait for peer ranks' queued waits that
// the blocked thread itself has to satisfy.  Collectives count themselves in flight; a release
// during that time is queued and performed at the next quiescent point (the end of a group
// collective, communicator creation, zc_flush_deferred).
struct InFlight {
  InFlight();
  ~InFlight();
};
void release_device_memory(int device, void* p, bool ipc_handle);
void flush_deferred_if_idle();
int cuda_err(cudaError_t e, const char* where);
const DevHuff* device_tables(const zc_huff_ctx* c);
}  // namespace zc

// The batched send / receive paths of the C-ABI (zc_api.cu), shared with the staged ring steps of
// zc_comm.cu.  `o` (may be null): the batch size (4 MiB, or 512 KiB slots under per-slot framing)
// and the fused-collective extras.
struct zc_i_batch_opts {
  uint64_t unit_bytes;        // 0 = ZC_BATCH_RAW_BYTES
  const double* dscale;       // float source / sink: {scale, 1/scale} in device memory
  const uint32_t* maxzz_in;   // encode of symbols: per-unit max zig-zag already known
  const float* acc_f32;       // decode OUT_ADD_Q: the local fp32 chunk
  uint32_t* maxzz_out;        // decode OUT_ADD_*: per-unit max zig-zag of the sums (atomicMax)
  int no_spec;                // encode fp32: no speculative width (two reads of the input)
};
extern "C" {
int zc_i_reserve_scratch(void* stream, uint32_t nunits);
int zc_i_ring_fused(const uint8_t* in_region, uint64_t stride, const zc_encode_result* in_res, int sink, int32_t* sum,
                    const float* x, const double* dscale, uint64_t total, uint64_t unit_bytes, uint8_t* out_region,
                    zc_encode_result* out_res, int32_t pin, const zc_transport_hint* hint, const zc_arb_config* cfg,
                    uint32_t* d_err, void* stream);
int zc_i_encode_batches(const void* src, int kind, uint64_t total, double scale, const zc_i_batch_opts* o,
                        uint8_t* d_stages, uint64_t stride, uint64_t stage_len, int32_t pin,
                        const zc_transport_hint* hint, const zc_huff_ctx* ctx, const zc_arb_config* cfg,
                        zc_encode_result* d_results, uint32_t* d_index, uint32_t* d_err, void* stream);
int zc_i_decode_batches(const uint8_t* d_stages, const zc_i_batch_opts* o, uint64_t stride, uint64_t stage_len,
                        const zc_encode_result* d_sent, uint64_t total, const zc_huff_ctx* ctx, const uint32_t* d_index,
                        int out_kind, void* out, double scale, uint32_t* d_codec, uint32_t* d_err, void* stream,
                        int own_frames);
}
