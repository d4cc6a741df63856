// Generic (unfused) sm_100a kernels: the always-available path for every
// KernelSet the reference can build (dense anisotropic kernels with their
// three summation orders, folded angular kernels, any shift), plus the
// tensor-wide reductions. Compiled with --fmad=false: every expression below
// evaluates in the reference's order with separately rounded mul and add,
// which makes the results bit-identical to belief_tensor.cpp.
#include <cuda_runtime.h>

#include <cstdint>

#include "gl_internal.hpp"
#include "wall.hpp"

namespace glb {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double dmax_ref(double a, double b) {
  return (a < b) ? b : a;  // std::max(a, b)
}

__device__ __forceinline__ void atomic_max_pos(unsigned long long* slot,
                                               double v) {
  // Non-negative doubles order like their uint64 bit patterns. Only v > 0 is
  // recorded: the reference's channel max starts at 0.0 and std::max ignores
  // NaN (belief_tensor.cpp:464-474).
  if (v > 0.0) atomicMax(slot, static_cast<unsigned long long>(__double_as_longlong(v)));
}

__device__ __forceinline__ double warp_max_pos(double v) {
  v = v > 0.0 ? v : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = dmax_ref(v, u);
  }
  return v;
}

// shift_plane (belief_tensor.cpp:67-124) for output cell (i, j) of a plane:
// integral (dx, dy) copies (:71-86); otherwise w00, w10, w01, w11 are added
// to 0.0 in that order, skipping taps outside the grid (:107-122). wall !=
// null (the wall-crossing mask extension, wall.hpp): taps whose segment
// crosses an occupied cell are skipped too.
__device__ __forceinline__ double shifted_value(const double* __restrict__ in,
                                                int w, int h, int i, int j,
                                                double dx, double dy,
                                                bool scaled, double sc,
                                                const uint8_t* __restrict__ wall) {
  const double fx = floor(dx), fy = floor(dy);
  if (fx == dx && fy == dy) {
    const long si = i - static_cast<long>(dx), sj = j - static_cast<long>(dy);
    if (si < 0 || si >= w || sj < 0 || sj >= h) return 0.0;
    if (wall && wall_tap_blocked(wall, w, h, si, sj, static_cast<long>(dx), static_cast<long>(dy))) return 0.0;
    double v = in[sj * static_cast<long>(w) + si];
    return scaled ? v * sc : v;
  }
  const long sx = static_cast<long>(fx), sy = static_cast<long>(fy);
  const double ax = dx - fx, ay = dy - fy;
  const double w00 = (1.0 - ax) * (1.0 - ay);
  const double w10 = ax * (1.0 - ay);
  const double w01 = (1.0 - ax) * ay;
  const double w11 = ax * ay;
  const long r0 = j - sy, r1 = j - sy - 1;
  const long c0 = i - sx, c1 = i - sx - 1;
  const bool ok_r0 = r0 >= 0 && r0 < h, ok_r1 = r1 >= 0 && r1 < h;
  const bool ok_c0 = c0 >= 0 && c0 < w, ok_c1 = c1 >= 0 && c1 < w;
  auto ld = [&](long r, long c) {
    const double v = in[r * w + c];
    return scaled ? v * sc : v;
  };
  auto open = [&](long c, long r, long ox, long oy) {
    return wall == nullptr || !wall_tap_blocked(wall, w, h, c, r, ox, oy);
  };
  double acc = 0.0;
  if (ok_r0 && ok_c0 && open(c0, r0, sx, sy)) acc += w00 * ld(r0, c0);
  if (ok_r0 && ok_c1 && open(c1, r0, sx + 1, sy)) acc += w10 * ld(r0, c1);
  if (ok_r1 && ok_c0 && open(c0, r1, sx, sy + 1)) acc += w01 * ld(r1, c0);
  if (ok_r1 && ok_c1 && open(c1, r1, sx + 1, sy + 1)) acc += w11 * ld(r1, c1);
  return acc;
}

// grid: x over columns, y over rows, z over channels. mode 1: step phase 1
// (shift + mask; wall: the wall-crossing mask), 2: apply_motion.
__global__ void k_shift_mask(const double* __restrict__ B,
                             double* __restrict__ S,
                             const double2* __restrict__ motion,
                             const uint8_t* __restrict__ occ,
                             const BufState* __restrict__ st, int w, int h,
                             int mode, int wall) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  if (i >= w) return;
  const size_t plane = static_cast<size_t>(w) * h;
  const bool scaled = st != nullptr && st->scaled;
  const double sc = scaled ? st->scale : 1.0;
  const double2 m = motion[k];
  const double* in = B + plane * k;
  const size_t p = static_cast<size_t>(j) * w + i;
  double v;
  if (mode == 2 && m.x == 0.0 && m.y == 0.0) {
    // apply_motion leaves channels with a zero motion vector untouched
    // (belief_tensor.cpp:346)
    v = in[p];
    if (scaled) v = v * sc;
  } else {
    v = shifted_value(in, w, h, i, j, m.x, m.y, scaled, sc, (mode == 1 && wall) ? occ : nullptr);
  }
  if (mode == 1 && occ[p]) v = 0.0;  // phase-1 mask (:414-416)
  S[plane * k + p] = v;
}

// convolve_plane_separable row pass (belief_tensor.cpp:199-225).
__global__ void k_row_pass(const double* __restrict__ S,
                           double* __restrict__ T, const int w, const int h,
                           const int r, const SepTaps taps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w) return;
  const size_t row = (static_cast<size_t>(blockIdx.z) * h + blockIdx.y) * w;
  double acc = 0.0;
  for (int d = -r; d <= r; ++d) {
    const int s = i + d;
    if (s >= 0 && s < w) acc += taps.t[d + r] * S[row + s];
  }
  T[row + i] = acc;
}

// convolve_plane_separable column pass (belief_tensor.cpp:227-238).
__global__ void k_col_pass(const double* __restrict__ T,
                           double* __restrict__ D, const int w, const int h,
                           const int r, const SepTaps taps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w) return;
  const int j = blockIdx.y;
  const size_t base = static_cast<size_t>(blockIdx.z) * h * w;
  double acc = 0.0;
  for (int d = -r; d <= r; ++d) {
    const int sj = j + d;
    if (sj < 0 || sj >= h) continue;
    acc += taps.t[d + r] * T[base + static_cast<size_t>(sj) * w + i];
  }
  D[base + static_cast<size_t>(j) * w + i] = acc;
}

// convolve_plane (belief_tensor.cpp:126-193) with its three orders.
__global__ void k_conv_dense(const double* __restrict__ S,
                             double* __restrict__ D,
                             const double* __restrict__ kernels, const int w,
                             const int h, const int r, const int c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w) return;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  const int kw = 2 * r + 1;
  const double* kern = kernels + static_cast<size_t>(k % c) * kw * kw;
  const double* in = S + static_cast<size_t>(k) * h * w;
  const bool interior = (j >= r && j < h - r) && (i >= r && i < w - r);
  double acc = 0.0;
  if (!interior) {
    for (int dy = -r; dy <= r; ++dy) {
      const int sj = j + dy;
      if (sj < 0 || sj >= h) continue;
      for (int dx = -r; dx <= r; ++dx) {
        const int si = i + dx;
        if (si < 0 || si >= w) continue;
        acc += kern[(dy + r) * kw + dx + r] * in[static_cast<size_t>(sj) * w + si];
      }
    }
  } else if (r == 2 && w > 4) {
    const double* q = in + static_cast<size_t>(j - 2) * w + (i - 2);
    const double* kk = kern;
    acc = kk[0] * q[0] + kk[1] * q[1] + kk[2] * q[2] + kk[3] * q[3] + kk[4] * q[4];
#pragma unroll
    for (int row = 1; row < 5; ++row) {
      const double* qr = q + static_cast<size_t>(row) * w;
      const double* kr = kk + 5 * row;
      acc += kr[0] * qr[0] + kr[1] * qr[1] + kr[2] * qr[2] + kr[3] * qr[3] + kr[4] * qr[4];
    }
  } else {
    for (int dy = -r; dy <= r; ++dy) {
      const double* qr = in + static_cast<size_t>(j + dy) * w + (i - r);
      const double* kr = kern + (dy + r) * kw;
      for (int dx = 0; dx < kw; ++dx) acc += kr[dx] * qr[dx];
    }
  }
  D[static_cast<size_t>(k) * h * w + static_cast<size_t>(j) * w + i] = acc;
}

// step phase 3 (belief_tensor.cpp:440-475): angular taps (first initialises,
// rest +=), mask, multiply by the activation inverse, global max.
__global__ void k_angular(const double* __restrict__ D, double* __restrict__ out,
                          const uint8_t* __restrict__ occ,
                          const double* __restrict__ inv, const int inv_per_k,
                          const int* __restrict__ off,
                          const double* __restrict__ wt, const int n_ang,
                          const int w, const int h, const int c,
                          unsigned long long* __restrict__ gmax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int k = blockIdx.z;
  const size_t plane = static_cast<size_t>(w) * h;
  const size_t p = static_cast<size_t>(j) * w + i;
  double v = 0.0;
  if (i < w) {
    auto src = [&](int t) {
      const int kk = (k - off[t] % c + c) % c;
      return D[plane * kk + p];
    };
    double acc = wt[0] * src(0);
    for (int t = 1; t < n_ang; ++t) acc += wt[t] * src(t);
    if (occ[p]) {
      acc = 0.0;
    } else {
      acc = acc * inv[inv_per_k ? plane * k + p : p];
      v = acc;
    }
    out[plane * k + p] = acc;
  }
  v = warp_max_pos(v);
  if ((threadIdx.x & 31) == 0) atomic_max_pos(gmax, v);
}

// Turn the step's running max into the status and the output buffer's
// pending rescale (belief_tensor.cpp:480-493); reset the accumulator.
__global__ void k_step_finalize(StepState* st, BufState* dst, int* host_status) {
  const double g = __longlong_as_double(static_cast<long long>(st->gmax_bits));
  publish_status(st, (g <= 0.0) ? GL_E_EXTINGUISHED : GL_OK, host_status);
  if (g > 0.0 && g < 1e-6) {
    dst->scaled = 1;
    dst->scale = 1.0 / g;
  } else {
    dst->scaled = 0;
    dst->scale = 1.0;
  }
  st->gmax_bits = 0ull;
  st->blocks_done = 0u;
}

__global__ void k_apply_scale(double* __restrict__ buf, size_t n,
                              const BufState* __restrict__ st) {
  if (!st->scaled) return;
  const double sc = st->scale;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < n; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    buf[q] = buf[q] * sc;
  }
}

__global__ void k_clear_state(BufState* st) {
  st->scaled = 0;
  st->scale = 1.0;
}

__global__ void k_fill(double* __restrict__ buf, size_t n, double v) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < n; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    buf[q] = v;
  }
}

__global__ void k_init_uniform(double* __restrict__ buf,
                               const uint8_t* __restrict__ occ, size_t plane,
                               int c) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < plane * c; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    buf[q] = occ[q % plane] ? 0.0 : 1.0;
  }
}

__global__ void k_free_indicator(double* __restrict__ base,
                                 const uint8_t* __restrict__ occ,
                                 size_t plane) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < plane; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    base[q] = occ[q] ? 0.0 : 1.0;
  }
}

// make_activation angular part (belief_tensor.cpp:378-392).
__global__ void k_activation(const double* __restrict__ diff, int diff_per_k,
                             double* __restrict__ values,
                             double* __restrict__ inverse,
                             const int* __restrict__ off,
                             const double* __restrict__ wt, int n_ang,
                             size_t plane, int c, int c_out) {
  const size_t total = plane * c_out;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < total; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(q / plane);
    const size_t p = q % plane;
    double acc = 0.0;
    for (int t = 0; t < n_ang; ++t) {
      const int kk = (k - off[t] % c + c) % c;
      acc += wt[t] * diff[(diff_per_k ? plane * kk : 0) + p];
    }
    if (values) values[q] = acc;
    inverse[q] = 1.0 / dmax_ref(acc, 1e-12);
  }
}

// distance_field (occupancy_map.cpp:231-271) on the device, in the
// reference's arithmetic: per-column run lengths by two sweeps (integers),
// min and square; then per row the Felzenszwalb-Huttenlocher lower envelope
// of parabolas (IEEE div/sqrt are correctly rounded on both sides, no FMA
// contraction: bit-identical), sqrt * resolution.
__global__ void k_edt_cols(const uint8_t* __restrict__ occ, double* __restrict__ sq, int w, int h) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w) return;
  const int far = w + h;
  int run = far;
  for (int j = 0; j < h; ++j) {
    const size_t p = static_cast<size_t>(j) * w + i;
    run = occ[p] ? 0 : (run >= far ? far : run + 1);
    sq[p] = run;
  }
  run = far;
  for (int j = h - 1; j >= 0; --j) {
    const size_t p = static_cast<size_t>(j) * w + i;
    run = occ[p] ? 0 : (run >= far ? far : run + 1);
    double c = sq[p];
    c = c < static_cast<double>(run) ? c : static_cast<double>(run);  // std::min(cell, run)
    sq[p] = c * c;
  }
}

// one thread per row; v (int) and z (double) are per-row scratch of w and
// w + 1 entries (occupancy_map.cpp:197-226)
__global__ void k_edt_rows(const double* __restrict__ sq, double* __restrict__ out, int* __restrict__ vs,
                           double* __restrict__ zs, int w, int h, double res) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= h) return;
  const double* f = sq + static_cast<size_t>(j) * w;
  int* v = vs + static_cast<size_t>(j) * w;
  double* z = zs + static_cast<size_t>(j) * (w + 1);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  int k = 0;
  v[0] = 0;
  z[0] = -inf;
  z[1] = inf;
  for (int q = 1; q < w; ++q) {
    double s;
    for (;;) {
      const int p = v[k];
      s = ((f[q] + q * q) - (f[p] + p * p)) / (2.0 * q - 2.0 * p);
      if (s <= z[k]) {
        --k;
      } else {
        break;
      }
    }
    ++k;
    v[k] = q;
    z[k] = s;
    z[k + 1] = inf;
  }
  k = 0;
  double* o = out + static_cast<size_t>(j) * w;
  for (int q = 0; q < w; ++q) {
    while (z[k + 1] < q) ++k;
    const int p = v[k];
    const double d = (q - p) * (q - p) + f[p];
    o[q] = sqrt(d) * res;
  }
}

// belief_map (belief_tensor.cpp:500-510).
// belief_map (belief_tensor.cpp:500-510): out = std::max over channels from
// 0.0. The max of {0.0, v_k} does not depend on the combining order (NaN
// never replaces a value, -0.0 never replaces +0.0), so each thread keeps 4
// independent partial maxima over 2 cells (16-byte loads, 8 loads in flight)
// and merges them: one HBM-speed pass.
__global__ void k_belief_map(const double* __restrict__ B,
                             double* __restrict__ out, size_t plane, int c) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  if ((plane & 1) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0) {
    const size_t p2n = plane / 2;
    const double2* B2 = reinterpret_cast<const double2*>(B);
    double2* out2 = reinterpret_cast<double2*>(out);
    for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < p2n; p += stride) {
      double2 m[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) m[j] = make_double2(0.0, 0.0);
      int k = 0;
      for (; k + 4 <= c; k += 4) {
        double2 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = B2[p2n * (k + j) + p];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          m[j].x = dmax_ref(m[j].x, v[j].x);
          m[j].y = dmax_ref(m[j].y, v[j].y);
        }
      }
      for (; k < c; ++k) {
        const double2 v = B2[p2n * k + p];
        m[0].x = dmax_ref(m[0].x, v.x);
        m[0].y = dmax_ref(m[0].y, v.y);
      }
      double2 r = m[0];
#pragma unroll
      for (int j = 1; j < 4; ++j) {
        r.x = dmax_ref(r.x, m[j].x);
        r.y = dmax_ref(r.y, m[j].y);
      }
      out2[p] = r;
    }
    return;
  }
  for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < plane; p += stride) {
    double m[4] = {0.0, 0.0, 0.0, 0.0};
    int k = 0;
    for (; k + 4 <= c; k += 4) {
      double v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = B[plane * (k + j) + p];
#pragma unroll
      for (int j = 0; j < 4; ++j) m[j] = dmax_ref(m[j], v[j]);
    }
    for (; k < c; ++k) m[0] = dmax_ref(m[0], B[plane * k + p]);
    out[p] = dmax_ref(dmax_ref(m[0], m[1]), dmax_ref(m[2], m[3]));
  }
}

// argmax_state (belief_tensor.cpp:512-541): the first strictly-greater scan
// in (k, j, i) order == the lowest flat index among the maxima (NaN never
// wins, values must exceed -1). Two passes: per-block candidates, then one
// block. (The confidence's total is the reference's sequential sum,
// k_seqsum.cu; the per-block sums here are not used for it.)
struct ArgCand {
  double v;
  long long idx;
  double sum;
};

__device__ __forceinline__ ArgCand better(ArgCand a, ArgCand b) {
  ArgCand r;
  const bool take_b = (b.v > a.v) || (b.v == a.v && b.idx < a.idx);
  r.v = take_b ? b.v : a.v;
  r.idx = take_b ? b.idx : a.idx;
  r.sum = a.sum + b.sum;
  return r;
}

__device__ ArgCand block_reduce(ArgCand c) {
  __shared__ ArgCand sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgCand u;
    u.v = __shfl_down_sync(0xffffffffu, c.v, o);
    u.idx = __shfl_down_sync(0xffffffffu, c.idx, o);
    u.sum = __shfl_down_sync(0xffffffffu, c.sum, o);
    c = better(c, u);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = c;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  if (wid == 0) {
    c = lane < nw ? sh[lane] : ArgCand{-1.0, 0x7fffffffffffffffLL, 0.0};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgCand u;
      u.v = __shfl_down_sync(0xffffffffu, c.v, o);
      u.idx = __shfl_down_sync(0xffffffffu, c.idx, o);
      u.sum = __shfl_down_sync(0xffffffffu, c.sum, o);
      c = better(c, u);
    }
  }
  return c;
}

__global__ void k_argmax_partial(const double* __restrict__ B, size_t n,
                                 ArgCand* __restrict__ part) {
  ArgCand c{-1.0, 0x7fffffffffffffffLL, 0.0};
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < n; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double x = B[q];
    c.sum += x;
    if (x > c.v) {  // strict: keeps the first (lowest) index of a tie
      c.v = x;
      c.idx = static_cast<long long>(q);
    }
  }
  c = block_reduce(c);
  if (threadIdx.x == 0) part[blockIdx.x] = c;
}

__global__ void k_argmax_final(const ArgCand* __restrict__ part, int nparts,
                               ArgCand* __restrict__ out) {
  ArgCand c{-1.0, 0x7fffffffffffffffLL, 0.0};
  for (int q = threadIdx.x; q < nparts; q += blockDim.x) c = better(c, part[q]);
  c = block_reduce(c);
  if (threadIdx.x == 0) *out = c;
}

// Order-independent 64-bit tensor hash: sum over p of splitmix64(bits_p +
// p * golden). Recomputed on the host in tests (numpy) for parity.
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void k_hash(const double* __restrict__ B, size_t n, unsigned long long p0,
                       unsigned long long* out) {
  unsigned long long acc = 0;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < n; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const unsigned long long bits =
        static_cast<unsigned long long>(__double_as_longlong(B[q]));
    acc += mix64(bits + (p0 + static_cast<unsigned long long>(q)) * 0x9e3779b97f4a7c15ull);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

__global__ void k_plane_max(const double* __restrict__ B, size_t n,
                            unsigned long long* gmax) {
  // 16-byte loads over the aligned body (the max is order-independent),
  // scalar head/tail
  double m = 0.0;
  if (n == 0) return;
  const size_t head = (reinterpret_cast<uintptr_t>(B) & 15) ? 1 : 0;
  const size_t n2 = (n - head) / 2;
  const double2* B2 = reinterpret_cast<const double2*>(B + head);
  const size_t tid = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t q = tid; q < n2; q += stride) {
    const double2 v = B2[q];
    m = dmax_ref(m, v.x);
    m = dmax_ref(m, v.y);
  }
  if (tid == 0) {
    if (head && n > 0) m = dmax_ref(m, B[0]);
    if (head + 2 * n2 < n) m = dmax_ref(m, B[n - 1]);
  }
  m = warp_max_pos(m);
  if ((threadIdx.x & 31) == 0) atomic_max_pos(gmax, m);
}

// Sign bit set (negative or -0.0) or exponent all ones (inf/NaN).
__global__ void k_scan_unclean(const double* __restrict__ B, size_t n,
                               unsigned int* flag) {
  unsigned int bad = 0;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < n; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const unsigned long long b =
        static_cast<unsigned long long>(__double_as_longlong(B[q]));
    bad |= ((b >> 63) != 0ull) || ((b & 0x7ff0000000000000ull) == 0x7ff0000000000000ull);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

int grid_for(size_t n, int threads, int max_blocks = 148 * 16) {
  size_t b = (n + threads - 1) / threads;
  if (b > static_cast<size_t>(max_blocks)) b = max_blocks;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

}  // namespace

// ---------------------------------------------------------------- launchers

void launch_shift_mask(gl_context* ctx, const StepArgs& a, double* S, int mode) {
  dim3 grid((a.w + kThreads - 1) / kThreads, a.h, a.c);
  k_shift_mask<<<grid, kThreads, 0, ctx->stream>>>(a.src, S, a.motion, a.occ,
                                                   a.src_state, a.w, a.h, mode, a.wall ? 1 : 0);
  ctx->launches++;
}

void launch_conv_separable(gl_context* ctx, const double* S, double* tmp,
                           double* D, int w, int h, int c, const SepTaps& taps,
                           int r) {
  dim3 grid((w + kThreads - 1) / kThreads, h, c);
  k_row_pass<<<grid, kThreads, 0, ctx->stream>>>(S, tmp, w, h, r, taps);
  k_col_pass<<<grid, kThreads, 0, ctx->stream>>>(tmp, D, w, h, r, taps);
  ctx->launches += 2;
}

void launch_conv_dense(gl_context* ctx, const double* S, double* D, int w,
                       int h, int c, const double* d_spatial, int r,
                       int kernel_channels) {
  dim3 grid((w + kThreads - 1) / kThreads, h, c);
  k_conv_dense<<<grid, kThreads, 0, ctx->stream>>>(S, D, d_spatial, w, h, r,
                                                   kernel_channels);
  ctx->launches++;
}

void launch_angular(gl_context* ctx, const StepArgs& a, const double* D,
                    const int* d_off, const double* d_w, int n_ang) {
  dim3 grid((a.w + kThreads - 1) / kThreads, a.h, a.c);
  k_angular<<<grid, kThreads, 0, ctx->stream>>>(
      D, a.dst, a.occ, a.inv, a.inv_per_channel, d_off, d_w, n_ang, a.w, a.h,
      a.c, &a.step_state->gmax_bits);
  ctx->launches++;
}

void launch_step_finalize(gl_context* ctx, const StepArgs& a) {
  k_step_finalize<<<1, 1, 0, ctx->stream>>>(a.step_state, a.dst_state, a.host_status);
  ctx->launches++;
}

void launch_apply_scale(gl_context* ctx, double* buf, size_t n,
                        BufState* state) {
  k_apply_scale<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(buf, n,
                                                                     state);
  k_clear_state<<<1, 1, 0, ctx->stream>>>(state);
  ctx->launches += 2;
}

// BLF1 snapshot payload (belief_tensor.cpp:555-559, 579-584): float32 <->
// float64, round-to-nearest like static_cast<float>; float -> double exact.
__global__ void k_to_f32(const double* __restrict__ in, float* __restrict__ out, size_t n) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < n; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    out[q] = __double2float_rn(in[q]);
  }
}

__global__ void k_from_f32(const float* __restrict__ in, double* __restrict__ out, size_t n) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < n; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    out[q] = static_cast<double>(in[q]);
  }
}

void launch_to_f32(gl_context* ctx, const double* in, float* out, size_t n) {
  k_to_f32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(in, out, n);
  ctx->launches++;
}

void launch_from_f32(gl_context* ctx, const float* in, double* out, size_t n) {
  k_from_f32<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(in, out, n);
  ctx->launches++;
}

void launch_fill(gl_context* ctx, double* buf, size_t n, double v) {
  k_fill<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(buf, n, v);
  ctx->launches++;
}

void launch_init_uniform(gl_context* ctx, double* buf, const uint8_t* occ,
                         int w, int h, int c) {
  const size_t plane = static_cast<size_t>(w) * h;
  k_init_uniform<<<grid_for(plane * c, kThreads), kThreads, 0, ctx->stream>>>(
      buf, occ, plane, c);
  ctx->launches++;
}

void launch_make_activation(gl_context* ctx, const uint8_t* occ, int w, int h,
                            int c, const gl_kernels* k, double* values,
                            double* inverse, bool k_invariant, double* scratch) {
  // scratch: base plane, row plane(s), diffused plane(s)
  const size_t plane = static_cast<size_t>(w) * h;
  const int r = k->info.radius;
  const int nd = k_invariant ? 1 : c;  // diffused planes needed
  double* base = scratch;
  double* rows = base + plane;
  double* diff = rows + plane * nd;
  k_free_indicator<<<grid_for(plane, kThreads), kThreads, 0, ctx->stream>>>(
      base, occ, plane);
  ctx->launches++;
  dim3 grid1((w + kThreads - 1) / kThreads, h, 1);
  if (k->info.separable) {
    SepTaps taps{};
    for (int t = 0; t < 2 * r + 1; ++t) taps.t[t] = k->sep[t];
    k_row_pass<<<grid1, kThreads, 0, ctx->stream>>>(base, rows, w, h, r, taps);
    k_col_pass<<<grid1, kThreads, 0, ctx->stream>>>(rows, diff, w, h, r, taps);
    ctx->launches += 2;
  } else if (r == 0) {
    cudaMemcpyAsync(diff, base, plane * sizeof(double),
                    cudaMemcpyDeviceToDevice, ctx->stream);
  } else {
    // per-channel dense kernels on the same base plane
    for (int kk = 0; kk < nd; ++kk) {
      k_conv_dense<<<grid1, kThreads, 0, ctx->stream>>>(
          base, diff + plane * kk, k->d_spatial + static_cast<size_t>(kk) * (2 * r + 1) * (2 * r + 1),
          w, h, r, 1);
      ctx->launches++;
    }
  }
  const int c_out = k_invariant ? 1 : c;
  k_activation<<<grid_for(plane * c_out, kThreads), kThreads, 0, ctx->stream>>>(
      diff, k_invariant ? 0 : 1, values, inverse, k->d_ang_off, k->d_ang_w,
      k->info.n_angular, plane, c, c_out);
  ctx->launches++;
}

void launch_distance_field(gl_context* ctx, const uint8_t* d_occ, int w, int h, double res,
                           double* d_out, void* d_scratch) {
  // scratch: sq (w*h doubles) | z (h*(w+1) doubles) | v (h*w ints)
  double* sq = static_cast<double*>(d_scratch);
  double* z = sq + static_cast<size_t>(w) * h;
  int* v = reinterpret_cast<int*>(z + static_cast<size_t>(h) * (w + 1));
  k_edt_cols<<<(w + 127) / 128, 128, 0, ctx->stream>>>(d_occ, sq, w, h);
  k_edt_rows<<<(h + 63) / 64, 64, 0, ctx->stream>>>(sq, d_out, v, z, w, h, res);
  ctx->launches += 2;
}

size_t distance_field_scratch_bytes(int w, int h) {
  return sizeof(double) * (static_cast<size_t>(w) * h + static_cast<size_t>(h) * (w + 1)) +
         sizeof(int) * static_cast<size_t>(w) * h;
}

void launch_belief_map(gl_context* ctx, const double* buf, int w, int h,
                       int c, double* out) {
  const size_t plane = static_cast<size_t>(w) * h;
  k_belief_map<<<grid_for((plane + 1) / 2, kThreads), kThreads, 0, ctx->stream>>>(
      buf, out, plane, c);
  ctx->launches++;
}

size_t argmax_scratch_bytes(size_t) { return sizeof(ArgCand) * (148 * 8 + 1); }

void launch_argmax(gl_context* ctx, const double* buf, size_t n,
                   void* d_scratch, size_t, void* d_out) {
  const int blocks = grid_for(n, kThreads, 148 * 8);
  auto* part = static_cast<ArgCand*>(d_scratch);
  k_argmax_partial<<<blocks, kThreads, 0, ctx->stream>>>(buf, n, part);
  k_argmax_final<<<1, 1024, 0, ctx->stream>>>(part, blocks,
                                              static_cast<ArgCand*>(d_out));
  ctx->launches += 2;
}

__global__ void k_gather_status(StatusPtrs ptrs, int* __restrict__ out) {
  const int i = threadIdx.x;
  if (i < ptrs.n) out[i] = *ptrs.p[i];
}

void launch_gather_status(gl_context* ctx, const StatusPtrs& ptrs, int* d_out) {
  k_gather_status<<<1, kStatusGather, 0, ctx->stream>>>(ptrs, d_out);
  ctx->launches++;
}

void launch_hash(gl_context* ctx, const double* buf, size_t n,
                 unsigned long long* d_out, unsigned long long p0) {
  cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), ctx->stream);
  k_hash<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(buf, n, p0, d_out);
  ctx->launches++;
}

__global__ void k_mask_plane(const double* __restrict__ in,
                             const uint8_t* __restrict__ occ, size_t plane,
                             double* __restrict__ out) {
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
       q < plane; q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    out[q] = occ[q] ? 0.0 : in[q];
  }
}

void launch_mask_plane(gl_context* ctx, const double* in, const uint8_t* occ,
                       size_t plane, double* out) {
  k_mask_plane<<<grid_for(plane, kThreads), kThreads, 0, ctx->stream>>>(in, occ, plane, out);
  ctx->launches++;
}

void launch_scan_unclean(gl_context* ctx, const double* buf, size_t n,
                         unsigned int* d_flag) {
  cudaMemsetAsync(d_flag, 0, sizeof(unsigned int), ctx->stream);
  k_scan_unclean<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(buf, n, d_flag);
  ctx->launches++;
}

void launch_plane_max(gl_context* ctx, const double* buf, size_t n,
                      unsigned long long* d_gmax) {
  k_plane_max<<<grid_for(n, kThreads), kThreads, 0, ctx->stream>>>(buf, n,
                                                                   d_gmax);
  ctx->launches++;
}

}  // namespace glb
