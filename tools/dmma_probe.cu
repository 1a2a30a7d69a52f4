// DMMA (mma.sync.m8n8k4.f64) issue/latency probe on the B200: fp64 tensor
// throughput vs warps per SM and independent accumulator chains per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int C>
__global__ void probe(double* out, int iters, double seed) {
  double c[C][2];
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int C>
void run(int warps_per_block, int blocks_per_sm) {
  double* d;
  cudaMalloc(&d, 4096 * 8);
  const int iters = 4096 / C * 4;
  const int blocks = 148 * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<C><<<blocks, 32 * warps_per_block>>>(d, iters, 1.0);
  cudaEventRecord(e0);
  probe<C><<<blocks, 32 * warps_per_block>>>(d, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256.0 * C * iters * (double)blocks * warps_per_block;
  printf("chains %2d  warps/SM %3d  TF %6.2f\n", C, warps_per_block * blocks_per_sm, flops / ms / 1e9);
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<1>(w, 1);
    run<2>(w, 1);
    run<4>(w, 1);
    run<8>(w, 1);
  }
  return 0;
}
