// zc_api_internal.h — helpers shared by the C-ABI translation units (not exported).
#pragma once
#include <string>

#include "zc_kernels.h"

namespace zc {
int set_err(int code, const std::string& msg);
int cuda_err(cudaError_t e, const char* where);
const DevHuff* device_tables(const zc_huff_ctx* c);
}  // namespace zc

// The batched send / receive paths of the C-ABI (zc_api.cu), shared with the staged ring steps of
// zc_comm.cu.  unit_bytes: the batch size (4 MiB, or 512 KiB slots under per-slot framing).  C linkage, hidden visibility.
extern "C" {
int zc_i_reserve_scratch(void* stream, uint32_t nunits);
int zc_i_encode_batches(const void* src, int kind, uint64_t total, double scale, uint64_t unit_bytes, uint8_t* d_stages, uint64_t stride,
                        uint64_t stage_len, int32_t pin, const zc_transport_hint* hint, const zc_huff_ctx* ctx,
                        const zc_arb_config* cfg, zc_encode_result* d_results, uint32_t* d_index, uint32_t* d_err,
                        void* stream);
int zc_i_decode_batches(const uint8_t* d_stages, uint64_t unit_bytes, uint64_t stride, uint64_t stage_len, const zc_encode_result* d_sent,
                        uint64_t total, const zc_huff_ctx* ctx, const uint32_t* d_index, int out_kind, void* out,
                        double scale, uint32_t* d_codec, uint32_t* d_err, void* stream, int own_frames);
}
