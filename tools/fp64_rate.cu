// Micro-benchmark (developer tool): issue rate of the instructions the quantizer uses on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dadd(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
    a0 = __dadd_rn(a0, 1.5); a1 = __dadd_rn(a1, 1.5); a2 = __dadd_rn(a2, 1.5); a3 = __dadd_rn(a3, 1.5);
    a4 = __dadd_rn(a4, 1.5); a5 = __dadd_rn(a5, 1.5); a6 = __dadd_rn(a6, 1.5); a7 = __dadd_rn(a7, 1.5);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_f2d(double* out, int iters) {
  float f = threadIdx.x;
  double a = 0;
  for (int i = 0; i < iters; ++i) {
    a += (double)(f + i) + (double)(f * 2 + i) + (double)(f * 3 + i) + (double)(f * 5 + i);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
__global__ void k_fadd(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
    a0 = __fadd_rn(a0, 1.5f); a1 = __fadd_rn(a1, 1.5f); a2 = __fadd_rn(a2, 1.5f); a3 = __fadd_rn(a3, 1.5f);
    a4 = __fadd_rn(a4, 1.5f); a5 = __fadd_rn(a5, 1.5f); a6 = __fadd_rn(a6, 1.5f); a7 = __fadd_rn(a7, 1.5f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
  double* d; cudaMalloc(&d, 148 * 8 * 1024 * 8);
  int iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a); k_dadd<<<148 * 4, 512>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("DADD: %.1f G inst/s (thread-level)\n", 148.0 * 4 * 512 * iters * 8 / (ms * 1e-3) / 1e9);
    cudaEventRecord(a); k_f2d<<<148 * 4, 512>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("F2F.F64.F32 (+DADD+FADD): %.1f G conversions/s\n", 148.0 * 4 * 512 * iters * 4 / (ms * 1e-3) / 1e9);
    cudaEventRecord(a); k_fadd<<<148 * 4, 512>>>((float*)d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("FADD: %.1f G inst/s\n", 148.0 * 4 * 512 * iters * 8 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
