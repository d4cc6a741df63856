// Debug probe: 3-D FP64 TMA box load (the fused step's access pattern) into
// shared memory with an mbarrier, checked against a host reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -o build/probe_tma tools/probe_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const __grid_constant__ CUtensorMap tmap, double* out,
                      int x, int y, int z, int bw, int bh, int mode) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  double* box = reinterpret_cast<double*>(base);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + ((bw * bh * 8 + 127) & ~127));
  if (threadIdx.x == 0) {
    if (mode & 1) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
    if (mode & 2) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bw * bh * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(box)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(0) : "memory");
  } while (!done);
  for (int q = threadIdx.x; q < bw * bh; q += blockDim.x) out[q] = box[q];
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ CUtensorMap g_map;

__global__ void probe_global(double* out, int x, int y, int z, int bw, int bh) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  double* box = reinterpret_cast<double*>(base);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + ((bw * bh * 8 + 127) & ~127));
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(&g_map)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bw * bh * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(box)), "l"(reinterpret_cast<uint64_t>(&g_map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
  }
  __syncthreads();
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(0) : "memory");
  } while (!done);
  for (int q = threadIdx.x; q < bw * bh; q += blockDim.x) out[q] = box[q];
}

int main(int argc, char** argv) {
  const int W = 96, H = 80, C = 4;
  const int mode = argc > 1 ? atoi(argv[1]) : 3;
  const int bw = argc > 2 ? atoi(argv[2]) : 68;
  const int bh = argc > 3 ? atoi(argv[3]) : 19;
  const int dtype = argc > 4 ? atoi(argv[4]) : 0;   // 0 f64, 1 u64, 2 i64
  const int use_global = argc > 5 ? atoi(argv[5]) : 0;
  const int sx = argc > 6 ? atoi(argv[6]) : -3;
  std::vector<double> h(W * H * C);
  for (size_t q = 0; q < h.size(); ++q) h[q] = 1.0 + q;
  double* d;
  cudaMalloc(&d, h.size() * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  double* dout;
  cudaMalloc(&dout, bw * bh * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  printf("entry point: %s qr=%d fn=%p\n", cudaGetErrorString(e), (int)qr, fn);
  CUtensorMap m;
  const cuuint64_t dims[3] = {W, H, C};
  const cuuint64_t strides[2] = {W * 8ull, W * H * 8ull};
  const cuuint32_t box[3] = {bw, bh, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUtensorMapDataType dt = dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : dtype == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_INT64;
  CUresult r = reinterpret_cast<EncodeTiled>(fn)(&m, dt, 3, d, dims, strides, box, es,
                                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  const int x = sx, y = -2, z = 1;
  if (use_global) {
    cudaMemcpyToSymbol(g_map, &m, sizeof(m));
    probe_global<<<1, 64, bw * bh * 8 + 512>>>(dout, x, y, z, bw, bh);
  } else {
    probe<<<1, 64, bw * bh * 8 + 512>>>(m, dout, x, y, z, bw, bh, mode);
  }
  e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<double> o(bw * bh);
  cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int j = 0; j < bh; ++j)
    for (int i = 0; i < bw; ++i) {
      const int gx = x + i, gy = y + j;
      const double want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[(size_t)z * W * H + gy * W + gx] : 0.0;
      bad += o[j * bw + i] != want;
    }
  printf("mismatches: %d\n", bad);
  return bad != 0;
}
