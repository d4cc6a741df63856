// Micro-benchmark (experiment only): one warp running the segment sweep's
// 16-pixel group (loads, DADD->DMUL chain, high-word screen, stores) with one
// chain per lane vs two interleaved chains per lane. Cycles per group.
#include <cstdio>
#include <cuda_runtime.h>

template <int NC>
__global__ void groups(const double* __restrict__ pre_g, double* __restrict__ err_g, int n_grp, long long* clk,
                       double cm) {
  __shared__ double pre[2560];
  __shared__ double err[2560];
  const int lane = threadIdx.x;
  for (int i = lane; i < 2560; i += 32) pre[i] = pre_g[i];
  __syncwarp();
  double carry[NC];
  int base[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    carry[c] = 0.0;
    base[c] = (lane + 32 * c) * 31 % 2048;
  }
  unsigned int bigall = 0;
  const long long t0 = clock64();
  for (int g = 0; g < n_grp; ++g) {
    double p[NC][16], v[NC][16];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int k = 0; k < 16; ++k) p[c][k] = pre[base[c] + 16 * (g & 7) + k];
    unsigned int big[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) big[c] = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double vk = p[c][k] + carry[c];
        v[c][k] = vk;
        asm("mul.rn.f64 %0, %1, %2;" : "=d"(carry[c]) : "d"(vk), "d"(cm));
        big[c] |= __double2hiint(vk) >= 0x3FE00000 ? (1u << k) : 0u;
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      bigall |= big[c];
#pragma unroll
      for (int k = 0; k < 16; ++k) err[base[c] + 16 * (g & 7) + k] = v[c][k];
    }
    if (__any_sync(0xffffffffu, bigall == 0xdeadbeefu)) break;
  }
  const long long t1 = clock64();
  __syncwarp();
  for (int i = lane; i < 2560; i += 32) err_g[i] = err[i];
  if (lane == 0) *clk = t1 - t0;
}

int main() {
  double *pre, *err;
  long long* clk;
  cudaMalloc(&pre, 8192 * 8);
  cudaMalloc(&err, 8192 * 8);
  cudaMalloc(&clk, 8);
  cudaMemset(pre, 0, 8192 * 8);
  const int n = 2000;
  long long h;
  for (int r = 0; r < 2; ++r) {
    groups<1><<<1, 32>>>(pre, err, n, clk, 7.0 / 16.0);
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("1 chain/lane: %.1f cycles per group (%.1f per pixel-step)\n", h / (double)n, h / (double)n / 16);
    groups<2><<<1, 32>>>(pre, err, n, clk, 7.0 / 16.0);
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("2 chains/lane: %.1f cycles per double group (%.1f per pixel-step)\n", h / (double)n, h / (double)n / 16);
  }
  return 0;
}
