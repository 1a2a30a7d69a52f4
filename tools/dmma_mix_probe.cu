// fp64 pipe probe on the B200: DMMA (m8n8k4) throughput when every 8 DMMAs
// of a warp come with NL shared-memory loads feeding the B operands, ND DMULs
// and NI integer ops, at W warps per SM.  Answers what the spread /
// interpolation inner loops can reach.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_mix_probe tools/dmma_mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NL, int ND, int NI>
__global__ void mix(double* out, int iters, double seed) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = seed + i;
  __syncthreads();
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  int idx = threadIdx.x & 31, acc = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    double l[NL > 0 ? NL : 1];
#pragma unroll
    for (int k = 0; k < NL; ++k) l[k] = sm[(idx + 37 * k + (it & 7) * 128) & 4095];
    double m[ND > 0 ? ND : 1];
#pragma unroll
    for (int k = 0; k < ND; ++k) m[k] = (NL ? l[k % (NL ? NL : 1)] : a) * b;
#pragma unroll
    for (int k = 0; k < NI; ++k) acc = acc * 3 + (it ^ k);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double bb = ND ? m[i % (ND ? ND : 1)] : (NL ? l[i % (NL ? NL : 1)] : b);
      dmma(c[i][0], c[i][1], a, bb);
    }
    idx = (idx + (acc & 1)) & 31;
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0 || acc == 7) out[threadIdx.x] = s + acc;
}

// software-pipelined: iteration k+1's loads and products are formed before
// iteration k's DMMAs issue (register double buffer); NI independent int ops
template <int NL, int ND, int NI>
__global__ void mixp(double* out, int iters, double seed) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = seed + i;
  __syncthreads();
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  int idx = threadIdx.x & 31;
  int ac[NI > 0 ? NI : 1];
#pragma unroll
  for (int k = 0; k < NI; ++k) ac[k] = threadIdx.x + k;
  double m[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) m[k] = b;
  for (int it = 0; it < iters; ++it) {
    double l[NL > 0 ? NL : 1];
#pragma unroll
    for (int k = 0; k < NL; ++k) l[k] = sm[(idx + 37 * k + (it & 7) * 128) & 4095];
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, m[i]);
#pragma unroll
    for (int k = 0; k < NI; ++k) ac[k] = ac[k] * 3 + it;
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = k < ND ? l[k % (NL ? NL : 1)] * b : (NL ? l[k % (NL ? NL : 1)] : b);
    idx = (idx + 1) & 31;
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  int t = 0;
#pragma unroll
  for (int k = 0; k < NI; ++k) t += ac[k];
  if (s == 12345.0 || t == 7) out[threadIdx.x] = s + t;
}

template <int NL, int ND, int NI>
void runp(int warps_per_block, int blocks_per_sm) {
  double* d;
  cudaMalloc(&d, 4096 * 8);
  const int iters = 2048;
  const int blocks = 148 * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mixp<NL, ND, NI><<<blocks, 32 * warps_per_block>>>(d, iters, 1.0);
  cudaEventRecord(e0);
  mixp<NL, ND, NI><<<blocks, 32 * warps_per_block>>>(d, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256.0 * 8 * iters * (double)blocks * warps_per_block;
  printf("PIPELINED LDS %d DMUL %d INT %2d per 8 DMMA | warps/SM %3d | DMMA TF %6.2f %s\n", NL, ND, NI,
         warps_per_block * blocks_per_sm, flops / ms / 1e9, cudaGetLastError() == cudaSuccess ? "" : "(launch failed)");
  cudaFree(d);
}

template <int NL, int ND, int NI>
void sweepp() {
  for (int w : {8, 16}) runp<NL, ND, NI>(w, 1);
  runp<NL, ND, NI>(8, 2);
}

template <int NL, int ND, int NI>
void run(int warps_per_block, int blocks_per_sm) {
  double* d;
  cudaMalloc(&d, 4096 * 8);
  const int iters = 2048;
  const int blocks = 148 * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<NL, ND, NI><<<blocks, 32 * warps_per_block>>>(d, iters, 1.0);
  cudaEventRecord(e0);
  mix<NL, ND, NI><<<blocks, 32 * warps_per_block>>>(d, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 256.0 * 8 * iters * (double)blocks * warps_per_block;
  printf("LDS %d DMUL %d INT %2d per 8 DMMA | warps/SM %3d | DMMA TF %6.2f\n", NL, ND, NI,
         warps_per_block * blocks_per_sm, flops / ms / 1e9);
  cudaFree(d);
}

template <int NL, int ND, int NI>
void sweep() {
  for (int w : {8, 12, 16, 24, 32}) run<NL, ND, NI>(w, 1);
}

int main() {
  sweepp<8, 6, 0>();
  sweepp<8, 6, 16>();
  sweepp<8, 6, 32>();
  sweepp<8, 8, 24>();
  sweepp<4, 4, 16>();
  sweep<0, 0, 0>();
  sweep<8, 0, 0>();
  sweep<0, 4, 0>();
  sweep<0, 6, 0>();
  sweep<6, 4, 0>();
  sweep<8, 6, 0>();
  sweep<8, 6, 16>();
  sweep<8, 6, 32>();
  sweep<4, 4, 8>();
  return 0;
}
