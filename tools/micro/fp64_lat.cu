// Micro-benchmark (experiment only): dependent-latency of FP64 add/mul,
// shared-memory load latency and block barrier cost on one SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* clk, int n, double a, double b) {
  __shared__ int chase[1024];
  __shared__ double sd[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) { chase[i] = (i * 97 + 13) & 1023; sd[i] = i * 0.5; }
  __syncthreads();
  double x = a, y = b;
  long long t0 = clock64();
  if (tid < 32) {
    for (int i = 0; i < n; ++i) { asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(b)); }
  }
  long long t1 = clock64();
  if (tid < 32) {
    for (int i = 0; i < n; ++i) { asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(a)); }
  }
  long long t2 = clock64();
  int p = tid & 1023;
  if (tid < 32) {
    for (int i = 0; i < n; ++i) p = chase[p];
  }
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t4 = clock64();
  if (tid < 32) {
    for (int i = 0; i < n; ++i) { y = sd[(static_cast<int>(y) + i) & 1023] + y * 0.0; }
  }
  long long t5 = clock64();
  if (tid < 32) {  // 4 independent add chains (throughput-ish)
    double x1 = x, x2 = x, x3 = x;
    for (int i = 0; i < n; ++i) {
      asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(b));
      asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x1) : "d"(b));
      asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x2) : "d"(b));
      asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x3) : "d"(b));
    }
    x += x1 + x2 + x3;
  }
  long long t6 = clock64();
  if (tid == 0) {
    clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t4 - t3; clk[4] = t5 - t4; clk[5] = t6 - t5;
  }
  out[tid] = x + y + p;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64);
  const int n = 4096;
  for (int bs : {32, 128}) {
    for (int r = 0; r < 2; ++r) lat<<<1, bs>>>(o, c, n, 1.0000001, 1e-9);
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("block %d: dadd %.2f dmul %.2f lds32-chase %.2f syncthreads %.2f lds64+dmul+dadd %.2f 4xdadd-indep %.2f cycles/iter\n",
           bs, h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
  }
  return 0;
}
