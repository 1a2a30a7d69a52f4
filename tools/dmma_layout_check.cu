// Empirical check of the mma.sync.m8n8k4 f64 fragment layout assumed by
// kernels_v4.cuh: A (8x4 row): lane t holds A[t/4][t%4]; B (4x8 col): lane t
// holds B[t%4][t/4]; C/D (8x8): lane t holds C[t/4][2(t%4)+i], i = 0, 1.
#include <cstdio>
__global__ void k(double* out) {
  int t = threadIdx.x;
  double a = (t / 4 + 1) * 10.0 + (t % 4);          // A[r][k] = (r+1)*10 + k
  double b = ((t % 4) + 1) * 100.0 + (t / 4);       // B[k][n] = (k+1)*100 + n
  double d0 = 0, d1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  out[(t / 4) * 8 + 2 * (t % 4)] = d0;
  out[(t / 4) * 8 + 2 * (t % 4) + 1] = d1;
}
int main() {
  double* d; cudaMalloc(&d, 64 * sizeof(double));
  k<<<1, 32>>>(d);
  double h[64]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 8; ++r) for (int n = 0; n < 8; ++n) {
    double s = 0; for (int kk = 0; kk < 4; ++kk) s += ((r + 1) * 10.0 + kk) * ((kk + 1) * 100.0 + n);
    if (s != h[r * 8 + n]) { ++bad; if (bad < 5) printf("mismatch r=%d n=%d got %g want %g\n", r, n, h[r*8+n], s); }
  }
  printf("dmma layout check: %s\n", bad ? "FAIL" : "OK");
  return bad != 0;
}
