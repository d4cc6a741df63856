// Cycles per pixel of candidate Floyd-Steinberg in-row carry chains on one
// thread, inputs from shared memory in groups of 32 (as k_dither_pipe).
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -o build/probe_fs tools/probe_fs_chain.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 2048
__device__ int g_sink[8];

template <int V>
__device__ __forceinline__ void body(double pv, bool s, double c, double& carry, double* err, int i, int& cnt) {
  const double v = pv + carry;
  if (V == 0) {  // branch + speculative asm multiply
    double next;
    asm("mul.rn.f64 %0, %1, %2;" : "=d"(next) : "d"(v), "d"(c));
    double e = v;
    if (__builtin_expect(v >= 0.5 && s, 0)) { e = v - 1.0; next = e * c; ++cnt; }
    err[i] = e; carry = next;
  } else if (V == 1) {  // branch-free two products + select
    double n0, n1, e1;
    asm("mul.rn.f64 %0, %1, %2;" : "=d"(n0) : "d"(v), "d"(c));
    asm("add.rn.f64 %0, %1, -1.0;" : "=d"(e1) : "d"(v));
    asm("mul.rn.f64 %0, %1, %2;" : "=d"(n1) : "d"(e1), "d"(c));
    const bool em = v >= 0.5 && s;
    cnt += em;
    err[i] = em ? e1 : v; carry = em ? n1 : n0;
  } else if (V == 2) {  // integer threshold compare + branch
    double next;
    asm("mul.rn.f64 %0, %1, %2;" : "=d"(next) : "d"(v), "d"(c));
    double e = v;
    const long long b = __double_as_longlong(v);
    if (__builtin_expect(s && b >= 0x3FE0000000000000ll, 0)) { e = v - 1.0; next = e * c; ++cnt; }
    err[i] = e; carry = next;
  } else if (V == 3) {  // integer compare + select
    double n0, n1, e1;
    asm("mul.rn.f64 %0, %1, %2;" : "=d"(n0) : "d"(v), "d"(c));
    asm("add.rn.f64 %0, %1, -1.0;" : "=d"(e1) : "d"(v));
    asm("mul.rn.f64 %0, %1, %2;" : "=d"(n1) : "d"(e1), "d"(c));
    const long long b = __double_as_longlong(v);
    const bool em = s && b >= 0x3FE0000000000000ll;
    cnt += em;
    err[i] = em ? e1 : v; carry = em ? n1 : n0;
  } else {  // bare dependent add+mul (floor)
    double next;
    asm("mul.rn.f64 %0, %1, %2;" : "=d"(next) : "d"(v), "d"(c));
    err[i] = v; carry = next;
  }
}

template <int V>
__device__ long long run(const double* pre, const unsigned* sup, double* err, double c, int& cnt) {
  double carry = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep)
    for (int q = 0; q < N; q += 32) {
      double pv[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) pv[k] = pre[q + k];
      const unsigned sw = sup[q >> 5];
#pragma unroll
      for (int k = 0; k < 32; ++k) body<V>(pv[k], (sw >> k) & 1u, c, carry, err, q + k, cnt);
      __threadfence_block();
    }
  long long t1 = clock64();
  cnt += carry > 1e300;
  return t1 - t0;
}

__global__ void k(const double* gpre, long long* out) {
  __shared__ double pre[N], err[N];
  __shared__ unsigned sup[N / 32];
  for (int i = threadIdx.x; i < N; i += blockDim.x) pre[i] = gpre[i];
  for (int i = threadIdx.x; i < N / 32; i += blockDim.x) sup[i] = 0xffffffffu;
  __syncthreads();
  if (threadIdx.x) return;
  int cnt = 0;
  const double c = 7.0 / 16.0;
  out[0] = run<0>(pre, sup, err, c, cnt);
  out[1] = run<1>(pre, sup, err, c, cnt);
  out[2] = run<2>(pre, sup, err, c, cnt);
  out[3] = run<3>(pre, sup, err, c, cnt);
  out[4] = run<4>(pre, sup, err, c, cnt);
  g_sink[0] = cnt + (int)err[7];
}

int main() {
  static double h[N];
  uint64_t x = 1;
  for (int i = 0; i < N; ++i) { x = x * 6364136223846793005ull + 1442695040888963407ull; h[i] = ((x >> 11) * 0x1.0p-53) * 0.001; }
  double* d; long long* o;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 64);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  k<<<1, 64>>>(d, o); k<<<1, 64>>>(d, o);
  long long r[5]; cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  const char* nm[5] = {"branch+asm", "select", "int-cmp branch", "int-cmp select", "add+mul floor"};
  for (int i = 0; i < 5; ++i) printf("%-16s %.2f cycles/pixel\n", nm[i], (double)r[i] / (8.0 * N));
  return 0;
}
