// zc_api_internal.h — helpers shared by the C-ABI translation units (not exported).
#pragma once
#include <string>

#include "zc_kernels.h"

namespace zc {
int set_err(int code, const std::string& msg);
int cuda_err(cudaError_t e, const char* where);
const DevHuff* device_tables(const zc_huff_ctx* c);
}  // namespace zc
