// Cycles per pixel of k_dither_pipe's speculative 32-pixel group loop on one
// thread (pre/err in scan order, LDS.128/STS.128), optionally with a second
// warp spinning on a shared progress word (as the pre-accumulating helper).
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -o build/probe_fsg tools/probe_fs_group.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define W 1024
#define ROWS 64
__device__ int g_sink[8];

__device__ __forceinline__ void fence_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }

template <int MODE>
__global__ void k(const double* gpre, long long* out, int spin) {
  __shared__ __align__(16) double pre[W + 80], err[W + 80];
  __shared__ unsigned sup[W / 32 + 2];
  __shared__ volatile int progress;
  for (int i = threadIdx.x; i < W + 80; i += blockDim.x) pre[i] = gpre[i % W];
  for (int i = threadIdx.x; i < W / 32 + 2; i += blockDim.x) sup[i] = 0xffffffffu;
  if (threadIdx.x == 0) progress = 0;
  __syncthreads();
  if (threadIdx.x >= 32) {
    if (!spin) return;
    int last = 0;
    double a = pre[threadIdx.x], b = pre[threadIdx.x + 1];
    while (last < ROWS * W) {
      int p = progress;
      if (p < 0) break;
      last += (p > 0);
      if (spin == 2) {  // FP64 work on the helper's lanes
#pragma unroll
        for (int i = 0; i < 8; ++i) { a = a * b + 0.25; }
      }
      if (spin == 3) {  // shared-memory traffic on the helper's lanes
#pragma unroll
        for (int i = 0; i < 4; ++i) err[(threadIdx.x + 64 * i + last) & 1023] = pre[(threadIdx.x + 64 * i) & 1023];
      }
    }
    g_sink[1] = (int)a;
    return;
  }
  if (threadIdx.x) return;
  const double c_mid = 7.0 / 16.0;
  double carry = 0.0;
  int cnt = 0;
  long long t0 = clock64();
  for (int row = 0; row < ROWS; ++row) {
    int q = 1;
    constexpr int G = 32;
    double2 pv[G / 2];
    if (MODE & 2) {
      const double2* p2 = reinterpret_cast<const double2*>(pre + q + 1);
#pragma unroll
      for (int k = 0; k < G / 2; ++k) pv[k] = p2[k];
    }
    for (; q + G <= W - 1; q += G) {
      double2 nx[G / 2];
      if (!(MODE & 2)) {
        const double2* p2 = reinterpret_cast<const double2*>(pre + q + 1);
#pragma unroll
        for (int k = 0; k < G / 2; ++k) pv[k] = p2[k];
      } else {
        const double2* p2 = reinterpret_cast<const double2*>(pre + q + G + 1);
#pragma unroll
        for (int k = 0; k < G / 2; ++k) nx[k] = p2[k];
      }
      int mx = 0;
      double2* e2 = reinterpret_cast<double2*>(err + q + 1);
      const unsigned long long sw = (unsigned long long)sup[q >> 5] | ((unsigned long long)sup[(q >> 5) + 1] << 32);
      const int sh = q & 31;
#pragma unroll
      for (int k = 0; k < 32; k += 2) {
        const double2 in = pv[k / 2];
        const double v0 = in.x + carry;
        asm("mul.rn.f64 %0, %1, %2;" : "=d"(carry) : "d"(v0), "d"(c_mid));
        const double v1 = in.y + carry;
        asm("mul.rn.f64 %0, %1, %2;" : "=d"(carry) : "d"(v1), "d"(c_mid));
        if (MODE & 1) e2[k / 2] = make_double2(v0, v1);
        else { err[q + 1 + k] = v0; err[q + 2 + k] = v1; }
        {
          mx = max(mx, __double2hiint(v0) & -static_cast<int>((sw >> (sh + k)) & 1ull));
          mx = max(mx, __double2hiint(v1) & -static_cast<int>((sw >> (sh + k + 1)) & 1ull));
        }
      }
      if (__builtin_expect(mx >= 0x3FE00000, 0)) { ++cnt; carry = 0.0; }
      if ((MODE & 4) || (((q - 1) / G) % 4 == 3)) {
        fence_cta();
        progress = q + G;
      }
      if (MODE & 2) {
#pragma unroll
        for (int k = 0; k < G / 2; ++k) pv[k] = nx[k];
      }
    }
  }
  long long t1 = clock64();
  progress = -1;
  out[0] = t1 - t0;
  g_sink[0] = cnt + (int)carry + (int)err[5];
}

int main() {
  static double h[W];
  uint64_t x = 1;
  for (int i = 0; i < W; ++i) { x = x * 6364136223846793005ull + 1442695040888963407ull; h[i] = ((x >> 11) * 0x1.0p-53) * 0.001; }
  if (getenv("SUBNORMAL")) for (int i = 0; i < W; ++i) h[i] = (i % 3 == 0) ? 0.0 : h[i] * 1e-305;
  double* d; long long* o;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 64);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int spin = 0; spin < 1; ++spin)
    for (int m = 0; m < 8; m += 5) {
      long long r = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (m) {
          case 0: k<0><<<1, 64>>>(d, o, spin); break;
          case 1: k<1><<<1, 64>>>(d, o, spin); break;
          case 2: k<2><<<1, 64>>>(d, o, spin); break;
          case 3: k<3><<<1, 64>>>(d, o, spin); break;
          case 4: k<4><<<1, 64>>>(d, o, spin); break;
          case 5: k<5><<<1, 64>>>(d, o, spin); break;
          case 6: k<6><<<1, 64>>>(d, o, spin); break;
          case 7: k<7><<<1, 64>>>(d, o, spin); break;
        }
        cudaMemcpy(&r, o, 8, cudaMemcpyDeviceToHost);
      }
      printf("pair=%d prefetch=%d fence/group=%d spin=%d  %.2f cycles/pixel\n", m & 1, (m >> 1) & 1, (m >> 2) & 1, spin, (double)r / (ROWS * 992.0));
    }
  return 0;
}
