// Host->device for one C2 vector (800 KB): copy engine vs a kernel reading
// pinned host memory directly (zero-copy over UVA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/h2d_probe.cu -o tools/h2d_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pull(const double2* __restrict__ h, double2* __restrict__ d, int n2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += gridDim.x * blockDim.x) d[i] = h[i];
}
__global__ void push(const double2* __restrict__ d, double2* __restrict__ h, int n2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += gridDim.x * blockDim.x) h[i] = d[i];
}

int main() {
  const int n = 100000, n2 = n / 2, reps = 300;
  double *h, *hy, *d;
  cudaHostAlloc(&h, n * 8, cudaHostAllocDefault);
  cudaHostAlloc(&hy, n * 8, cudaHostAllocDefault);
  cudaMalloc(&d, n * 8);
  for (int i = 0; i < n; ++i) h[i] = i;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  auto run = [&](const char* name, auto fn) {
    for (int i = 0; i < 20; ++i) fn();
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) fn();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("%-34s %7.1f us  %5.1f GB/s\n", name, ms * 1000 / reps, 0.8e6 / (ms * 1e6 / reps));
  };
  run("memcpy H2D", [&] { cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice, s); });
  run("memcpy D2H", [&] { cudaMemcpyAsync(hy, d, n * 8, cudaMemcpyDeviceToHost, s); });
  for (int blocks : {148, 296, 592, 1184})
    for (int th : {256, 512}) {
      char name[64];
      snprintf(name, sizeof(name), "kernel pull %d x %d", blocks, th);
      run(name, [&] { pull<<<blocks, th, 0, s>>>(reinterpret_cast<const double2*>(h), reinterpret_cast<double2*>(d), n2); });
    }
  run("kernel push 592 x 256", [&] { push<<<592, 256, 0, s>>>(reinterpret_cast<const double2*>(d), reinterpret_cast<double2*>(hy), n2); });
  printf("check %g %s\n", 0.0, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
