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
// fp64 tensor-core (DMMA m8n8k4) throughput: independent accumulators per warp
constexpr int kMmaChains = 8;
__global__ void __launch_bounds__(256) dmma_kernel(double* out, double a, double b) {
  double c[kMmaChains][2];
#pragma unroll
  for (int k = 0; k < kMmaChains; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9 + k;
  const double av = a + threadIdx.x * 1e-12, bv = b;
  for (int i = 0; i < kIters / 4; ++i) {
#pragma unroll
    for (int k = 0; k < kMmaChains; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(av), "d"(bv));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kMmaChains; ++k) s += c[k][0] + c[k][1];
  if (s == 1234.5678) out[threadIdx.x] = s;
}
}  // namespace

double measure_dmma_peak(int device) {
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
    dmma_kernel<<<blocks, 256>>>(out, 0.999999, 1e-7);
    FGS_CUDA(cudaEventRecord(e1));
    FGS_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FGS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    // per warp per mma: 8*8*4 FMAs = 512 flops
    const double flops = 512.0 * blocks * (256 / 32) * (kIters / 4) * kMmaChains;
    if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return best;
}

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
