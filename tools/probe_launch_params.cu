// Host cost of a kernel launch vs its parameter block size (B200 driver):
// 20000 back-to-back launches of an empty kernel, wall time per launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/probe_launch tools/probe_launch_params.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
struct P {
  double v[N];
};

template <int N>
__global__ void k(P<N> p, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && p.v[0] == 12345.0) out[0] = p.v[N - 1];
}

template <int N>
void run(double* d) {
  P<N> p{};
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int i = 0; i < 1000; ++i) k<N><<<1, 32, 0, s>>>(p, d);
  cudaStreamSynchronize(s);
  const int n = 20000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < n; ++i) {
    p.v[0] = i;
    k<N><<<1, 32, 0, s>>>(p, d);
  }
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto t2 = std::chrono::steady_clock::now();
  printf("params %6zu B: enqueue %.2f us/launch, total %.2f us/launch\n", sizeof(P<N>),
         std::chrono::duration<double, std::micro>(t1 - t0).count() / n,
         std::chrono::duration<double, std::micro>(t2 - t0).count() / n);
  cudaStreamDestroy(s);
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  run<16>(d);
  run<128>(d);
  run<512>(d);
  run<1024>(d);
  run<2400>(d);
  run<3800>(d);
  cudaEvent_t e;
  cudaEventCreate(&e);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 20000; ++i) cudaEventRecord(e, 0);
  auto t1 = std::chrono::steady_clock::now();
  printf("cudaEventRecord: %.2f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / 20000);
  return 0;
}
