// Single-thread FS carry chain v = pre[k] + cr; cr = v * c (speculative form)
// over shared-memory inputs, timed with clock64; variants: immediate vs
// register coefficient, with/without a second warp spinning on shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -o build/probe_fs2 tools/probe_fs_chain2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void chain(const double* in, double* out, long long* cyc, int n, double creg, int spin) {
  __shared__ double pre[4096];
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) pre[i] = in[i & 1023];
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (threadIdx.x >= 32) {
    if (spin) { while (!stop) { } }
    return;
  }
  if (threadIdx.x != 0) return;
  double cr = 0.0, acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    const double* p = pre + ((it * 32) & 4095);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double v = p[k] + cr;
      if (MODE == 0) cr = v * 0.4375; else cr = v * creg;
      acc = (k == 31) ? acc + v : acc;
    }
  }
  long long t1 = clock64();
  stop = 1;
  out[0] = cr + acc;
  cyc[0] = t1 - t0;
}

int main() {
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 0.001 * ((i * 37) % 101);
  double *din, *dout; long long* dc;
  cudaMalloc(&din, sizeof(h)); cudaMalloc(&dout, 64); cudaMalloc(&dc, 64);
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 1 << 15;  // x32 pixels
  for (int spin = 0; spin < 2; ++spin) {
    long long c;
    chain<0><<<1, 64>>>(din, dout, dc, n, 0.4375, spin);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("spin=%d imm: %.2f cycles/pixel\n", spin, (double)c / (32.0 * n));
    chain<1><<<1, 64>>>(din, dout, dc, n, 0.4375, spin);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("spin=%d reg: %.2f cycles/pixel\n", spin, (double)c / (32.0 * n));
  }
  return 0;
}
