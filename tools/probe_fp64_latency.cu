// Measures dependent-chain latency of FP64 ops on one thread (clock64):
// DADD, DMUL, DFMA-free mul+add pair, and the Floyd-Steinberg carry step
// v = pre + e * c; e = (v >= 0.5) ? v - 1 : v  (speculative form).
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -o build/probe_fp64 tools/probe_fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chains(const double* in, double* out, long long* cyc, int n) {
  double a = in[0], b = in[1], c = in[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a + b;
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) c = c * b;
  long long t2 = clock64();
  double v = a;
  for (int i = 0; i < n; ++i) v = in[3] + v * c;
  long long t3 = clock64();
  double e = 0.3, t = 0.0;
  int emit = 0;
  for (int i = 0; i < n; ++i) {
    double vv = in[4 + (i & 7)] + t;
    t = vv * 0.4375;
    if (vv >= 0.5) { t = (vv - 1.0) * 0.4375; ++emit; }
  }
  long long t4 = clock64();
  out[0] = a + c + v + e + t + emit;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

int main() {
  double h[12] = {1.0, 1e-300, 1.0000001, 0.01, 0.1, 0.2, 0.05, 0.3, 0.01, 0.02, 0.4, 0.15};
  double *din, *dout; long long* dc;
  cudaMalloc(&din, sizeof(h)); cudaMalloc(&dout, 64); cudaMalloc(&dc, 64);
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 1 << 20;
  chains<<<1, 1>>>(din, dout, dc, 1024);
  chains<<<1, 1>>>(din, dout, dc, n);
  long long c[4];
  cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
  printf("cycles per op: DADD %.2f  DMUL %.2f  mul+add %.2f  FS-carry %.2f\n", (double)c[0] / n,
         (double)c[1] / n, (double)c[2] / n, (double)c[3] / n);
  return 0;
}
