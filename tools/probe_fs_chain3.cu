// Which part of the real Floyd-Steinberg group loop costs beyond the bare
// DADD->DMUL chain? Single-thread chain over 32-pixel groups with optional
// (1) STS.128 of the errors, (2) 3-input max screen, (3) a helper warp doing
// FP64 work (DMUL/DADD + LDS/STS) concurrently, (4) mbarrier arrive per group.
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -o build/probe_fs3 tools/probe_fs_chain3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int STS, bool MX, bool ARR>
__global__ void chain(const double* in, double* out, long long* cyc, int n, int helper) {
  __shared__ __align__(16) double pre[2048];
  __shared__ __align__(16) double err[2048];
  __shared__ __align__(16) double hb[1024];
  __shared__ uint64_t bar;
  __shared__ volatile int stop;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) { pre[i] = in[i & 1023]; err[i] = 0.0; if (i < 1024) hb[i] = in[(i * 7) & 1023]; }
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x >= 32) {
    if (helper) {
      const int l = threadIdx.x - 32;
      double a = 0.0;
      while (!stop) {
        for (int b = 0; b < 1024; b += 32) {
          double v = hb[b + l] * 0.3;
          v += err[(b + l + 1) & 2047] * 0.0625;
          v += err[(b + l + 2) & 2047] * 0.3125;
          v += err[(b + l + 3) & 2047] * 0.1875;
          hb[(b + l + 64) & 1023] = v;
          a += v;
        }
      }
      out[8 + threadIdx.x] = a;
    }
    return;
  }
  if (threadIdx.x != 0) return;
  double cr = 0.0;
  int mx = 0;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    const int base = (it * 32) & 2047;
    const double2* p2 = reinterpret_cast<const double2*>(pre + base);
    double2* e2 = reinterpret_cast<double2*>(err + base);
    double vv[32];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 in2 = p2[k];
      const double v0 = in2.x + cr;
      cr = v0 * 0.4375;
      const double v1 = in2.y + cr;
      cr = v1 * 0.4375;
      vv[2 * k] = v0;
      vv[2 * k + 1] = v1;
      if (STS == 1) e2[k] = make_double2(v0, v1);
      if (STS == 2) err[base + 2 * k + 1] = v1;                       // STS.64 every 2 px
      if (STS == 3 && (k & 1)) e2[k] = make_double2(vv[2 * k - 1], v1);  // STS.128 every 4 px
      if (MX) mx = max(mx, max(__double2hiint(v0), __double2hiint(v1)));
    }
    if (STS == 4) {
#pragma unroll
      for (int k = 0; k < 16; ++k) e2[k] = make_double2(vv[2 * k], vv[2 * k + 1]);
    }
    if (MX && mx >= 0x7FF00000) break;
    if (ARR) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
  }
  long long t1 = clock64();
  stop = 1;
  out[0] = cr + mx;
  cyc[0] = t1 - t0;
}

template <int S, bool M, bool A>
void run(const char* name, const double* din, double* dout, long long* dc, int helper) {
  const int n = 1 << 14;
  chain<S, M, A><<<1, 64>>>(din, dout, dc, n, helper);
  long long c;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("%-22s helper=%d: %.2f cycles/pixel\n", name, helper, (double)c / (32.0 * n));
}

int main() {
  double h[1024];
  for (int i = 0; i < 1024; ++i) h[i] = 0.0001 * ((i * 37) % 101);
  double *din, *dout; long long* dc;
  cudaMalloc(&din, sizeof(h)); cudaMalloc(&dout, 1024); cudaMalloc(&dc, 64);
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int helper = 0; helper < 1; ++helper) {
    run<0, false, false>("bare", din, dout, dc, helper);
    run<1, false, false>("+sts128/2px", din, dout, dc, helper);
    run<2, false, false>("+sts64/2px (odd)", din, dout, dc, helper);
    run<3, false, false>("+sts128/4px (odd)", din, dout, dc, helper);
    run<4, false, false>("+sts128 bulk at end", din, dout, dc, helper);
    run<0, true, false>("+max", din, dout, dc, helper);
    run<3, true, true>("+sts128/4px+max+arr", din, dout, dc, helper);
  }
  return 0;
}
