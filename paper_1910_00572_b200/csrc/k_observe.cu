// Observation-path kernels: serpentine Floyd-Steinberg sample extraction
// (observation.cpp:11-71), the likelihood-field scan model over sampled
// states (observation.cpp:73-111) and the sampled multiplicative update
// (observation.cpp:113-170). --fmad=false; reference operand order.
#include <cuda_runtime.h>

#include <cstdint>

#include "gl_internal.hpp"

namespace glb {

namespace {

__device__ __forceinline__ double dmax_ref(double a, double b) {
  return (a < b) ? b : a;
}

// Floyd-Steinberg target weights, in the reference's target order:
// (dir,0) 7/16, (-dir,1) 3/16, (0,1) 5/16, (dir,1) 1/16.
__device__ __forceinline__ double fs_wsum(int i, int j, int w, int h, int dir) {
  double ws = 0.0;
  if (i + dir >= 0 && i + dir < w) ws += 7.0 / 16.0;
  if (j + 1 < h) {
    if (i - dir >= 0 && i - dir < w) ws += 3.0 / 16.0;
    ws += 5.0 / 16.0;
    if (i + dir >= 0 && i + dir < w) ws += 1.0 / 16.0;
  }
  return ws;
}

// dither_samples as a row decomposition that is bit-identical to the
// reference's serial sweep (probe P2):
//   * total: one sequential sum (observation.cpp:16-17), lane 0;
//   * per row, all lanes pre-accumulate the previous row's diffused error
//     into each cell in the reference's arrival order (upstream source,
//     centre, downstream source);
//   * lane 0 runs the in-row carry chain v = pre + e_prev * (7/16)/wsum_prev,
//     thresholds at 0.5 on support cells, emits, and records e = v - q.
// Serpentine order has no inter-row wavefront (row j+1 starts where row j
// ended), so the W*H dependent chain is inherent; see DESIGN.md.
__global__ void __launch_bounds__(32) k_dither(
    const double* __restrict__ bm, int w, int h, int budget,
    int* __restrict__ cells, int cap, int* __restrict__ n_out,
    double* __restrict__ mass_out) {
  extern __shared__ double sh[];
  double* pre = sh;       // w
  double* err = sh + w;   // w: errors of the previous row
  const int lane = threadIdx.x;
  const size_t plane = static_cast<size_t>(w) * h;

  double total = 0.0;
  if (lane == 0) {
#pragma unroll 8
    for (size_t p = 0; p < plane; ++p) total += bm[p];
    *mass_out = total;
  }
  total = __shfl_sync(0xffffffffu, total, 0);
  if (total <= 0.0) {
    if (lane == 0) *n_out = 0;
    return;
  }
  const double scale = budget / total;
  int count = 0;

  for (int j = 0; j < h; ++j) {
    const int dir = (j % 2 == 0) ? 1 : -1;
    const double* brow = bm + static_cast<size_t>(j) * w;
    // 1. pre-accumulate (all lanes)
    for (int t = lane; t < w; t += 32) {
      double v = brow[t] * scale;
      if (j > 0) {
        const int pd = -dir;  // previous row's direction
        const int jp = j - 1;
        const int s1 = t - pd, s3 = t + pd;
        if (s1 >= 0 && s1 < w) v += err[s1] * ((1.0 / 16.0) / fs_wsum(s1, jp, w, h, pd));
        v += err[t] * ((5.0 / 16.0) / fs_wsum(t, jp, w, h, pd));
        if (s3 >= 0 && s3 < w) v += err[s3] * ((3.0 / 16.0) / fs_wsum(s3, jp, w, h, pd));
      }
      pre[t] = v;
    }
    __syncwarp();
    // 2. the serial carry chain (lane 0)
    if (lane == 0) {
      double e_prev = 0.0, c_prev = 0.0;
      bool have_prev = false;
      for (int q = 0; q < w; ++q) {
        const int i = dir == 1 ? q : w - 1 - q;
        double v = pre[i];
        if (have_prev) v += e_prev * c_prev;
        double qv = 0.0;
        if (v >= 0.5 && brow[i] > 0.0) {
          qv = 1.0;
          if (count < cap) {
            cells[2 * count] = i;
            cells[2 * count + 1] = j;
          }
          ++count;
        }
        const double e = v - qv;
        err[i] = e;
        const double ws = fs_wsum(i, j, w, h, dir);
        // in-row target (dir,0) exists iff i+dir is in the grid; when
        // wsum == 0 (bottom corner) the residue is dropped (observation.cpp:44)
        have_prev = (i + dir >= 0 && i + dir < w) && ws > 0.0;
        c_prev = have_prev ? (7.0 / 16.0) / ws : 0.0;
        e_prev = e;
      }
    }
    __syncwarp();
  }
  if (lane == 0) *n_out = count;
}

// scan_likelihood (observation.cpp:73-111) for every (sample s, channel k).
// Host precomputes, with the reference's libm: per-cell beam score
// log((1-f)*exp(-d^2/(2 sigma^2)) + f) (and the out-of-map score), and per
// (channel, scored beam) the (cos, sin) of channel_angle(k) + angle_b. The
// device keeps the endpoint arithmetic and cell lookup in reference order.
// The geometric mean's final exp: with `kind` != nullptr the kernel writes
// the exponent (log_sum / counted) and a case code (0 exp, 1 floor, 2 one)
// so the host applies glibc's exp, exactly like the reference (default);
// otherwise CUDA's exp (<= 1 ulp from glibc).
__global__ void k_likelihoods(const uint8_t* __restrict__ occ,
                              const double* __restrict__ score, double oob_score,
                              int w, int h, double res, double ox, double oy,
                              double cell, double tox, double toy,
                              const int* __restrict__ samples,
                              int n, int c, const double2* __restrict__ dir,
                              int n_scored, const double* __restrict__ reach,
                              double floor_w, double* __restrict__ L,
                              uint8_t* __restrict__ kind) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n * c) return;
  const int s = q / c, k = q % c;
  const double x = tox + (samples[2 * s] + 0.5) * cell;
  const double y = toy + (samples[2 * s + 1] + 0.5) * cell;
  const int pi = static_cast<int>(floor((x - ox) / res));
  const int pj = static_cast<int>(floor((y - oy) / res));
  if (!(pi >= 0 && pi < w && pj >= 0 && pj < h) ||
      occ[static_cast<size_t>(pj) * w + pi]) {
    L[q] = floor_w;
    if (kind) kind[q] = 1;
    return;
  }
  double log_sum = 0.0;
  int counted = 0;
  for (int b = 0; b < n_scored; ++b) {
    const double2 cs = dir[static_cast<size_t>(k) * n_scored + b];
    const double ex = x + reach[b] * cs.x;
    const double ey = y + reach[b] * cs.y;
    const int ci = static_cast<int>(floor((ex - ox) / res));
    const int cj = static_cast<int>(floor((ey - oy) / res));
    const bool in = ci >= 0 && ci < w && cj >= 0 && cj < h;
    log_sum += in ? score[static_cast<size_t>(cj) * w + ci] : oob_score;
    ++counted;
  }
  if (kind) {
    kind[q] = counted == 0 ? 2 : 0;
    L[q] = counted == 0 ? 1.0 : log_sum / counted;
  } else {
    L[q] = counted == 0 ? 1.0 : exp(log_sum / counted);
  }
}

// Sequential mean over all sampled states (observation.cpp:139-141).
__global__ void k_mean(const double* __restrict__ L, int total,
                       double* __restrict__ mean) {
  double m = 0.0;
#pragma unroll 8
  for (int q = 0; q < total; ++q) m += L[q];
  *mean = m / static_cast<double>(total);
}

// B[i,j,k] *= L / mean, quotient first (observation.cpp:145-150).
__global__ void k_observe_apply(double* __restrict__ B, int w, int h, int c,
                                const int* __restrict__ samples, int n,
                                const double* __restrict__ L,
                                const double* __restrict__ mean) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n * c) return;
  const int s = q / c, k = q % c;
  const size_t p = static_cast<size_t>(k) * w * h +
                   static_cast<size_t>(samples[2 * s + 1]) * w + samples[2 * s];
  B[p] *= L[q] / *mean;
}

// Global max -> status + the buffer's pending 1/max rescale
// (observation.cpp:152-169).
__global__ void k_observe_finalize(StepState* st, BufState* buf) {
  const double g = __longlong_as_double(static_cast<long long>(st->gmax_bits));
  st->status = (g <= 0.0) ? GL_E_EXTINGUISHED : GL_OK;
  if (g > 0.0) {
    buf->scaled = 1;
    buf->scale = 1.0 / g;
  }
  st->gmax_bits = 0ull;
}

}  // namespace

void launch_dither(gl_context* ctx, const double* bm, int w, int h, int budget,
                   int* d_cells, int cap, int* d_n, double* d_mass) {
  const size_t smem = static_cast<size_t>(2) * w * sizeof(double);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(k_dither, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  }
  k_dither<<<1, 32, smem, ctx->stream>>>(bm, w, h, budget, d_cells, cap, d_n,
                                        d_mass);
  ctx->launches++;
}

void launch_likelihoods(gl_context* ctx, const uint8_t* occ, const double* score,
                        double oob_score, int w, int h, double res, double ox,
                        double oy, double cell, double tox, double toy,
                        const int* d_samples, int n,
                        int c, const double2* d_dir, int n_scored,
                        const double* d_reach, double floor_w, double* d_L,
                        uint8_t* d_kind) {
  const int total = n * c;
  k_likelihoods<<<(total + 127) / 128, 128, 0, ctx->stream>>>(
      occ, score, oob_score, w, h, res, ox, oy, cell, tox, toy, d_samples, n, c, d_dir,
      n_scored, d_reach, floor_w, d_L, d_kind);
  ctx->launches++;
}

void launch_observe_apply(gl_context* ctx, double* buf, int w, int h, int c,
                          const int* d_samples, int n, const double* d_L,
                          double* d_mean) {
  k_mean<<<1, 1, 0, ctx->stream>>>(d_L, n * c, d_mean);
  const int total = n * c;
  k_observe_apply<<<(total + 127) / 128, 128, 0, ctx->stream>>>(
      buf, w, h, c, d_samples, n, d_L, d_mean);
  ctx->launches += 2;
}

void launch_observe_finalize(gl_context* ctx, StepState* st, BufState* buf) {
  k_observe_finalize<<<1, 1, 0, ctx->stream>>>(st, buf);
  ctx->launches++;
}

}  // namespace glb
