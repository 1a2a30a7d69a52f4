// Phase timing of conv2_cluster_kernel (M = 128, N = 64, C2 shape):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DFGS_CONV2_TRACE \
//        -Iinclude -Ipaper_1808_04580_b200/csrc tools/conv2_bench.cu -o tools/conv2_bench
#include <cstdio>
#include <cmath>
#include <vector>

#include "conv2d.cuh"

using namespace fgsb;

int main() {
  const int M = 128, N = 64, H = N / 2 + 1, logM = 7;
  double *g;
  cufftDoubleComplex* mult;
  double2* tw;
  cudaMalloc(&g, sizeof(double) * M * M);
  cudaMalloc(&mult, sizeof(cufftDoubleComplex) * (N + 1) * H);
  cudaMalloc(&tw, sizeof(double2) * M);
  cudaMemset(g, 0, sizeof(double) * M * M);
  cudaMemset(mult, 0, sizeof(cufftDoubleComplex) * (N + 1) * H);
  std::vector<double2> t(M);
  for (int j = 0; j < M; ++j) t[j] = make_double2(cos(2 * M_PI * j / M), -sin(2 * M_PI * j / M));
  cudaMemcpy(tw, t.data(), sizeof(double2) * M, cudaMemcpyHostToDevice);
  Conv2Args a{g, g, mult, tw, M, logM, N, 1, M * M};
  const size_t smem = conv2_smem(M, N);
  cudaFuncSetAttribute(conv2_cluster_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(conv2_cluster_kernel<128>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 10; ++i) conv2_cluster_kernel<128><<<kClusterCtas, kConvThreads, smem>>>(a);
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) conv2_cluster_kernel<128><<<kClusterCtas, kConvThreads, smem>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("avg %.2f us per launch (%s)\n", ms * 10, cudaGetErrorString(cudaGetLastError()));
  unsigned long long tr[16];
  cudaMemcpyFromSymbol(tr, g_conv2_trace, sizeof(tr));
  const char* names[] = {"start", "prefetch", "rowfft", "unpack", "csync1", "colfft", "icolfft", "csync2", "irowfft"};
  for (int i = 1; i < 9; ++i) printf("%-8s %6.2f us\n", names[i], (tr[i] - tr[i - 1]) * 1e-3);
  printf("total    %6.2f us\n", (tr[8] - tr[0]) * 1e-3);
  return 0;
}
