// Micro-benchmark (experiment only): cost of the segment sweep's 16-pixel
// group as the real kernel's features are added one by one (one warp).
#include <cstdio>
#include <cuda_runtime.h>

template <int F>  // feature level
__global__ void groups(const double* __restrict__ pre_g, const unsigned* __restrict__ sup_g, double* __restrict__ err_g,
                       int n_grp, long long* clk, double cm, double cf) {
  __shared__ double pre[2560];
  __shared__ double err[2560];
  __shared__ unsigned sup[96];
  const int lane = threadIdx.x;
  for (int i = lane; i < 2560; i += 32) pre[i] = pre_g[i];
  for (int i = lane; i < 96; i += 32) sup[i] = sup_g[i];
  __syncwarp();
  double carry = 0.0;
  const int q0 = lane * 31 % 2048;
  const int qs = q0 + 32, qe = q0 + 31 + 64;
  unsigned int bigall = 0;
  double wu = 0.0;
  const long long t0 = clock64();
  for (int g = 0; g < n_grp; ++g) {
    const int base = q0 + 16 * (g % 5);
    const int valid = (F >= 5 && F < 20) ? max(0, min(16, qe - base)) : 16;
    if (F >= 5 && F < 20) {
      if (!__any_sync(0xffffffffu, valid > 0)) break;
    }
    const double* pb = pre + ((F >= 5 && F < 20) ? (valid > 0 ? base : 0) : base);
    double p[16], v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) p[k] = pb[k];
    unsigned sb = 0xffffu;
    if (F >= 2 && F != 21 && F != 22) {
      const int b = valid > 0 ? base : 0;
      const unsigned long long sw2 = (unsigned long long)sup[b >> 5] | ((unsigned long long)sup[(b >> 5) + 1] << 32);
      sb = (unsigned)(sw2 >> (b & 31)) & (valid >= 16 ? 0xffffu : ((1u << valid) - 1u));
    }
    const bool first = (F >= 3 && F < 20) && base == 0;
    double c = carry;
    unsigned big = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double vk = (F >= 3 && k == 0 && first) ? p[0] : p[k] + c;
      v[k] = vk;
      asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(vk), "d"((F >= 3 && k == 0 && first) ? cf : cm));
      big |= __double2hiint(vk) >= 0x3FE00000 ? (1u << k) : 0u;
    }
    if (F == 22) {
      bigall |= big & sb;
    } else if (F == 23) {  // replay body executed by every lane, results selected by need (no inner branch)
      const bool need = (big & sb) != 0u;
      if (__any_sync(0xffffffffu, need)) {
        double cc = carry;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const double vk = p[k] + cc;
          const bool em = vk >= 0.5 && ((sb >> k) & 1u);
          const double e = em ? vk - 1.0 : vk;
          v[k] = need ? e : v[k];
          asm("mul.rn.f64 %0, %1, %2;" : "=d"(cc) : "d"(e), "d"(cm));
        }
        c = need ? cc : c;
      }
    } else if (F >= 2) {
      const bool need = (big & sb) != 0u;
      if (__any_sync(0xffffffffu, need)) {
        if (need) {
          c = carry;
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const double vk = p[k] + c;
            const bool em = vk >= 0.5 && ((sb >> k) & 1u);
            const double e = em ? vk - 1.0 : vk;
            v[k] = e;
            asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(e), "d"(cm));
          }
        }
      }
    } else {
      bigall |= big;
    }
    carry = c;
    if (F >= 4 && F < 20) {
      const int own = base - qs;
      if (own >= 0) {
        double* eb = err + (valid > 0 ? base : 0);
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < valid) eb[k] = v[k];
      }
      if (own == -16) wu = v[15];
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) err[base + k] = v[k];
    }
    if ((F < 2 || F == 22) && __any_sync(0xffffffffu, bigall == 0xdeadbeefu)) break;
  }
  const long long t1 = clock64();
  __syncwarp();
  for (int i = lane; i < 2560; i += 32) err_g[i] = err[i] + wu;
  if (lane == 0) *clk = t1 - t0;
}


// level 24: level 21 (vote + replay branch, no sup loads) with the next
// group's values loaded before the vote, manually double-buffered (no copies)
__global__ void groups_pf(const double* __restrict__ pre_g, double* __restrict__ err_g, int n_grp, long long* clk,
                          double cm) {
  __shared__ double pre[2560];
  __shared__ double err[2560];
  const int lane = threadIdx.x;
  for (int i = lane; i < 2560; i += 32) pre[i] = pre_g[i];
  __syncwarp();
  double carry = 0.0;
  const int q0 = lane * 31 % 2048;
  const unsigned sb = 0xffffu;
  double pa[16], pb[16], v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) pa[k] = pre[q0 + k];
  auto step = [&](const double (&p)[16], double (&pn)[16], int g) {
    const int base = q0 + 16 * (g % 5);
    double c = carry;
    unsigned big = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double vk = p[k] + c;
      v[k] = vk;
      asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(vk), "d"(cm));
      big |= __double2hiint(vk) >= 0x3FE00000 ? (1u << k) : 0u;
    }
    const int nb = q0 + 16 * ((g + 1) % 5);
#pragma unroll
    for (int k = 0; k < 16; ++k) pn[k] = pre[nb + k];  // the next group's values, before the vote
    const bool need = (big & sb) != 0u;
    if (__any_sync(0xffffffffu, need)) {
      if (need) {
        c = carry;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const double vk = p[k] + c;
          const bool em = vk >= 0.5 && ((sb >> k) & 1u);
          const double e = em ? vk - 1.0 : vk;
          v[k] = e;
          asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(e), "d"(cm));
        }
      }
    }
    carry = c;
#pragma unroll
    for (int k = 0; k < 16; ++k) err[base + k] = v[k];
  };
  const long long t0 = clock64();
  for (int g = 0; g < n_grp; g += 2) {
    step(pa, pb, g);
    step(pb, pa, g + 1);
  }
  const long long t1 = clock64();
  __syncwarp();
  for (int i = lane; i < 2560; i += 32) err_g[i] = err[i];
  if (lane == 0) *clk = t1 - t0;
}

template <int F>
void run(const double* pre, const unsigned* sup, double* err, long long* clk, int n) {
  groups<F><<<1, 32>>>(pre, sup, err, n, clk, 7.0 / 16.0, 7.0 / 16.0);
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  printf("feature level %d: %.1f cycles per group\n", F, h / (double)n);
}

int main() {
  double *pre, *err;
  unsigned* sup;
  long long* clk;
  cudaMalloc(&pre, 2560 * 8);
  cudaMalloc(&err, 2560 * 8);
  cudaMalloc(&sup, 96 * 4);
  cudaMalloc(&clk, 8);
  cudaMemset(pre, 0, 2560 * 8);
  cudaMemset(sup, 0, 96 * 4);
  const int n = 2000;
  for (int r = 0; r < 2; ++r) {
    run<1>(pre, sup, err, clk, n);
    run<2>(pre, sup, err, clk, n);
    run<3>(pre, sup, err, clk, n);
    run<4>(pre, sup, err, clk, n);
    run<5>(pre, sup, err, clk, n);
    run<21>(pre, sup, err, clk, n);
    run<22>(pre, sup, err, clk, n);
    run<23>(pre, sup, err, clk, n);
    {
      groups_pf<<<1, 32>>>(pre, err, n, clk, 7.0 / 16.0);
      long long h;
      cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
      printf("level 24 (21 + next loads before the vote): %.1f cycles per group\n", h / (double)n);
    }
  }
  return 0;
}
