// fp64 pipe probe on the B200: what a DFMA costs next to DMMAs.  Each warp
// repeats G groups of [ND DMMAs, NF DFMAs] (independent accumulators, program
// order pinned with asm volatile) and reports cycles per DMMA-equivalent.
// Answers: is the 2m = 12 spread's 8 + 4 split (3 DMMA + 12 DFMA per K-step)
// cheaper than padded DMMAs, and does grouping the DFMAs matter.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_dfma_probe tools/dmma_dfma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void dfma(double& c, double a, double b) {
  asm volatile("fma.rn.f64 %0, %1, %2, %0;\n" : "+d"(c) : "d"(a), "d"(b));
}

// REP repetitions of [ND DMMA, NF DFMA] per loop iteration
template <int ND, int NF, int REP>
__global__ void mix(double* out, int iters, double seed) {
  double c[ND > 0 ? ND : 1][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = 0.0;
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < REP; ++r) {
#pragma unroll
      for (int i = 0; i < ND; ++i) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
      for (int i = 0; i < NF; ++i) dfma(f[i], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += f[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int ND, int NF, int REP>
void run(int warps, int blocks_per_sm) {
  double* d;
  cudaMalloc(&d, 4096 * 8);
  const int iters = 4096 / REP;
  const int blocks = 148 * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<ND, NF, REP><<<blocks, 32 * warps>>>(d, iters, 1.0);
  cudaEventRecord(e0);
  mix<ND, NF, REP><<<blocks, 32 * warps>>>(d, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // SMSP cycles per [ND, NF] group at 1.965 GHz, warps / 4 per SMSP
  const double groups_per_smsp = static_cast<double>(iters) * REP * warps * blocks_per_sm / 4.0;
  const double cyc = ms * 1e-3 * 1.965e9 / groups_per_smsp;
  const double fl = 2.0 * (256.0 * ND + 32.0 * NF) * iters * REP * static_cast<double>(blocks) * warps;
  printf("DMMA %2d DFMA %2d x%d | warps/SM %2d | %7.1f cycles/group (ideal %3d) | %6.2f TF\n", ND, NF, REP,
         warps * blocks_per_sm, cyc, 16 * ND + 2 * NF, fl / ms / 1e9);
  cudaFree(d);
}

int main() {
  run<8, 0, 1>(8, 2);
  run<0, 16, 1>(8, 2);
  run<3, 12, 1>(8, 2);
  run<3, 12, 1>(6, 3);
  run<3, 12, 4>(8, 2);
  run<6, 24, 1>(8, 2);
  run<12, 48, 1>(4, 2);
  run<3, 4, 1>(8, 2);
  run<3, 1, 1>(8, 2);
  run<8, 6, 1>(8, 2);
  run<8, 1, 1>(8, 2);
  run<8, 2, 1>(8, 2);
  run<1, 4, 1>(8, 2);
  run<1, 1, 1>(8, 2);
  run<1, 8, 1>(8, 2);
  return 0;
}
