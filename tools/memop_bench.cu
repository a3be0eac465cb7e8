// Developer microbenchmark: cost of the collective's building blocks on one GPU — a ping-pong of R
// rounds between two streams (kernel, cuStreamWriteValue64 to the peer's flag, cuStreamWaitValue64
// on its own flag), issued eagerly and as a captured CUDA graph; plus R back-to-back tiny kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/memop_bench tools/memop_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

__global__ void tiny(int* p) {
  if (threadIdx.x == 0) p[blockIdx.x] += 1;
}

#define CK(x)                                                         \
  do {                                                                \
    cudaError_t e = (x);                                              \
    if (e != cudaSuccess) {                                           \
      std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const int R = 20;
  cudaStream_t s[2];
  for (auto& x : s) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  unsigned long long* flags;
  int* scratch;
  CK(cudaMalloc(&flags, 64));
  CK(cudaMalloc(&scratch, 4096));
  auto issue = [&](bool with_kernels, bool with_memops) {
    for (int k = 1; k <= R; ++k)
      for (int r = 0; r < 2; ++r) {
        if (with_kernels) tiny<<<1, 32, 0, s[r]>>>(scratch + r);
        if (with_memops) {
          cuStreamWriteValue64(s[r], reinterpret_cast<CUdeviceptr>(flags + (1 - r)), k, 0);
          cuStreamWaitValue64(s[r], reinterpret_cast<CUdeviceptr>(flags + r), k, CU_STREAM_WAIT_VALUE_GEQ);
        }
      }
  };
  cudaEvent_t fork, join;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  for (int variant = 0; variant < 3; ++variant) {
    const bool K = variant != 1, M = variant != 0;
    const char* name = variant == 0 ? "kernels only" : variant == 1 ? "memops only" : "kernel+memops";
    // eager
    double best = 1e30;
    for (int rep = 0; rep < 10; ++rep) {
      CK(cudaMemset(flags, 0, 64));
      CK(cudaDeviceSynchronize());
      const double t0 = now_us();
      issue(K, M);
      CK(cudaStreamSynchronize(s[0]));
      CK(cudaStreamSynchronize(s[1]));
      best = std::min(best, now_us() - t0);
    }
    // graph
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s[0], cudaStreamCaptureModeThreadLocal));
    CK(cudaMemsetAsync(flags, 0, 64, s[0]));
    CK(cudaEventRecord(fork, s[0]));
    CK(cudaStreamWaitEvent(s[1], fork, 0));
    issue(K, M);
    CK(cudaEventRecord(join, s[1]));
    CK(cudaStreamWaitEvent(s[0], join, 0));
    CK(cudaStreamEndCapture(s[0], &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    double gbest = 1e30, lbest = 1e30;
    for (int rep = 0; rep < 10; ++rep) {
      CK(cudaDeviceSynchronize());
      const double t0 = now_us();
      CK(cudaGraphLaunch(ge, s[0]));
      const double t1 = now_us();
      CK(cudaStreamSynchronize(s[0]));
      gbest = std::min(gbest, now_us() - t0);
      lbest = std::min(lbest, t1 - t0);
    }
    std::printf("%-14s x %d rounds x 2 streams: eager %.1f us (%.2f us/round), graph %.1f us (%.2f us/round, "
                "launch call %.1f us)\n",
                name, R, best, best / R, gbest, gbest / R, lbest);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  return 0;
}
