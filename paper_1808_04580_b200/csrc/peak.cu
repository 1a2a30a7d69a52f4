// peak.cu -- fp64 FMA-pipe peak microbenchmark (the roofline denominator of
// the spread / interpolation kernels; MEASURED_PEAKS.json carries HBM and
// bf16 only).  Independent DFMA chains per thread, full-chip grid, CUDA
// events, best of several launches.
#include <algorithm>

#include "common.cuh"

namespace fgsb {

namespace {
constexpr int kChains = 16;
constexpr int kIters = 2048;

__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keep the chains alive
}
}  // namespace

double measure_fp64_peak(int device) {
  FGS_CUDA(cudaSetDevice(device));
  int sms = 0;
  FGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out = nullptr;
  FGS_CUDA(cudaMalloc(&out, 256 * sizeof(double)));
  cudaEvent_t e0, e1;
  FGS_CUDA(cudaEventCreate(&e0));
  FGS_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8;
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    FGS_CUDA(cudaEventRecord(e0));
    dfma_kernel<<<blocks, 256>>>(out, 0.999999, 1e-7);
    FGS_CUDA(cudaEventRecord(e1));
    FGS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FGS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * blocks * 256.0 * kIters * kChains;
    if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

}  // namespace fgsb
