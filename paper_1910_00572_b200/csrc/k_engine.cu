// Device side of the single-process multi-device engine (engine.cpp): the
// peer-memory form of the per-step 8-byte MAX all-reduce, and the belief-map
// MAX combine of a sharded observation. Every read of another device's
// memory goes over NVLink P2P (UVA pointers, peer access enabled by the
// engine); the cross-stream event waits the engine records order them.
#include <cuda_runtime.h>

#include <algorithm>

#include "gl_internal.hpp"

namespace glb {

namespace {

__global__ void k_engine_publish(const unsigned long long* gmax, unsigned long long* mailbox) {
  *mailbox = *reinterpret_cast<const volatile unsigned long long*>(gmax);
}

// uint64 bits of doubles >= 0 order like the values (belief_tensor.cpp:480-481
// takes the max of non-negative channel maxima)
__global__ void k_engine_gather(const PtrList boxes, unsigned long long* gmax) {
  unsigned long long m = 0ull;
  for (int s = 0; s < boxes.n; ++s) {
    const unsigned long long v = *static_cast<const volatile unsigned long long*>(boxes.p[s]);
    m = v > m ? v : m;
  }
  *gmax = m;
}

__global__ void k_plane_max_combine(double* __restrict__ dst, const PtrList srcs, size_t n) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double m = dst[q];
    for (int s = 0; s < srcs.n; ++s) {
      const double v = static_cast<const double*>(srcs.p[s])[q];
      m = (m < v) ? v : m;  // std::max: belief_map is an exact per-cell max
    }
    dst[q] = m;
  }
}

}  // namespace

void launch_engine_publish(gl_context* ctx, const unsigned long long* gmax, unsigned long long* mailbox) {
  k_engine_publish<<<1, 1, 0, ctx->stream>>>(gmax, mailbox);
  ctx->launches++;
}

void launch_engine_gather(gl_context* ctx, const PtrList& mailboxes, unsigned long long* gmax) {
  k_engine_gather<<<1, 1, 0, ctx->stream>>>(mailboxes, gmax);
  ctx->launches++;
}

void launch_plane_max_combine(gl_context* ctx, double* dst, const PtrList& srcs, size_t n) {
  const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 4 * 148));
  k_plane_max_combine<<<blocks > 0 ? blocks : 1, 256, 0, ctx->stream>>>(dst, srcs, n);
  ctx->launches++;
}

}  // namespace glb
