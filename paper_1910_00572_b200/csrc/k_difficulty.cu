// map_difficulty (evaluation.cpp:25-72) on the device: for every query cell,
// a noise-free simulated scan (simulator.cpp:63-94 -> raycast,
// occupancy_map.cpp:273-332), then scan_likelihood (observation.cpp:73-111)
// of that scan at every (candidate cell, test heading), and the first
// maximum. The work is free^2 x theta_bins likelihoods (x beams): the
// reference's largest CPU cost in the evaluation harness.
//
// Exactness. Every transcendental stays on the host where the reference
// evaluates it (glibc): beam directions cos/sin(theta + a_b) and the per-cell
// beam log-score log((1-f) exp(-d^2/2s^2) + f) are tables; the device does the
// reference's FP64 adds/multiplies/divides/floors in its order (--fmad=false),
// so ranges and log sums are bit-identical. The likelihood is
// exp(log_sum / counted) with counted fixed per query, so the argmax of the
// likelihood is the argmax of log_sum except where glibc's exp maps two
// different log sums to the same double: the device counts, per query, the
// earlier candidates whose log sum lies within a tiny window below the max,
// and the host re-decides exactly those queries with glibc exp.
#include <cuda_runtime.h>

#include <cstdint>

#include "gl_internal.hpp"

namespace glb {

namespace {

// raycast (occupancy_map.cpp:273-332): Amanatides-Woo from (x, y) along the
// host-computed direction (dx, dy) = (cos, sin)(angle) (glibc, as the
// reference), with its corner-tie tolerance; every operation in the
// reference's order (--fmad=false). Returns false when the origin is not a
// free in-bounds cell (the reference throws MapParseError kInvalidOrigin).
__device__ __forceinline__ bool raycast_dev(const uint8_t* __restrict__ occ, int w, int h, double res, double ox,
                                            double oy, double x, double y, double dx, double dy, double max_range,
                                            double* out) {
  const double cx = (x - ox) / res;
  const double cy = (y - oy) / res;
  int i = static_cast<int>(floor(cx));
  int j = static_cast<int>(floor(cy));
  if (!(i >= 0 && i < w && j >= 0 && j < h) || occ[static_cast<size_t>(j) * w + i]) return false;
  const double max_cells = max_range / res;
  const int step_x = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
  const int step_y = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const double t_delta_x = step_x != 0 ? fabs(1.0 / dx) : inf;
  const double t_delta_y = step_y != 0 ? fabs(1.0 / dy) : inf;
  double t_max_x = step_x != 0 ? ((step_x > 0 ? (i + 1.0 - cx) : (cx - i)) * t_delta_x) : inf;
  double t_max_y = step_y != 0 ? ((step_y > 0 ? (j + 1.0 - cy) : (cy - j)) * t_delta_y) : inf;
  constexpr double kTieEps = 1e-9;
  double tt = 0.0;
  double r = max_range;
  while (tt <= max_cells) {
    if (t_max_x < t_max_y - kTieEps) {
      tt = t_max_x;
      t_max_x += t_delta_x;
      i += step_x;
    } else if (t_max_y < t_max_x - kTieEps) {
      tt = t_max_y;
      t_max_y += t_delta_y;
      j += step_y;
    } else {
      tt = t_max_x;
      t_max_x += t_delta_x;
      t_max_y += t_delta_y;
      i += step_x;
      j += step_y;
    }
    if (!(i >= 0 && i < w && j >= 0 && j < h)) break;
    if (occ[static_cast<size_t>(j) * w + i]) {
      r = (max_cells < tt ? max_cells : tt) * res;  // std::min(t, max_cells) * res
      break;
    }
  }
  *out = r;
  return true;
}

// map_difficulty's noise-free query scans: from each query cell's centre at
// heading a_b (the query pose has theta = 0, so the beam angle is a_b exactly)
__global__ void k_raycast_queries(const uint8_t* __restrict__ occ, int w, int h, double res,
                                  double ox, double oy, const int2* __restrict__ cells, int n,
                                  const double2* __restrict__ ray, int beams, double max_range,
                                  double* __restrict__ ranges, int* __restrict__ bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * beams) return;
  const int q = t / beams, b = t - q * beams;
  const int2 cl = cells[q];
  const double x = ox + (cl.x + 0.5) * res;  // center_x / center_y
  const double y = oy + (cl.y + 0.5) * res;
  double r = 0.0;
  if (!raycast_dev(occ, w, h, res, ox, oy, x, y, ray[b].x, ray[b].y, max_range, &r)) {
    atomicExch(bad, 1);  // the reference throws (raycast origin not free)
    r = 0.0;
  }
  ranges[t] = r;
}

// A batch of rays (raycast) or scans (simulate_scan, simulator.cpp:63-94):
// ray t = (pose t / beams, beam t % beams) from xy[pose] along dir[t]; with
// noise, r += noise[t] * sigma, clamped to [0, max_range] (std::clamp).
__global__ void k_raycast_batch(const uint8_t* __restrict__ occ, int w, int h, double res, double ox, double oy,
                                const double2* __restrict__ xy, const double2* __restrict__ dir, int n_rays,
                                int beams, double max_range, const double* __restrict__ noise, double sigma,
                                double* __restrict__ ranges, int* __restrict__ bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_rays) return;
  const double2 p = xy[t / beams];
  double r = 0.0;
  if (!raycast_dev(occ, w, h, res, ox, oy, p.x, p.y, dir[t].x, dir[t].y, max_range, &r)) {
    atomicExch(bad, 1);
    ranges[t] = 0.0;
    return;
  }
  if (noise) {
    r += noise[t] * sigma;
    r = r < 0.0 ? 0.0 : (max_range < r ? max_range : r);
  }
  ranges[t] = r;
}

struct QueryBeams {
  int n;                    // scored beams (counted)
  int idx[kMaxDifficultyBeams];  // their indices b (stride, r < max_range - 1e-9)
  double reach[kMaxDifficultyBeams];
};

// log_sum of scan_likelihood for candidate idx = c * bins + a (the reference's
// loop order: cells outer, test headings inner).
__device__ __forceinline__ double cand_log_sum(const QueryBeams& qb, const uint8_t* __restrict__ occ,
                                               const double* __restrict__ score, double oob, int w, int h,
                                               double res, double ox, double oy, const int2* __restrict__ cells,
                                               const double2* __restrict__ dir, int beams, int bins, int idx,
                                               int* __restrict__ bad) {
  const int c = idx / bins, a = idx - c * bins;
  const int2 cl = cells[c];
  const double x = ox + (cl.x + 0.5) * res;
  const double y = oy + (cl.y + 0.5) * res;
  // world_free(pose) (observation.cpp:80): a candidate cell centre always is;
  // flag it if not (the reference would return the weight floor)
  const int pi = static_cast<int>(floor((x - ox) / res));
  const int pj = static_cast<int>(floor((y - oy) / res));
  if (!(pi >= 0 && pi < w && pj >= 0 && pj < h) || occ[static_cast<size_t>(pj) * w + pi]) atomicExch(bad, 2);
  double log_sum = 0.0;
  const double2* da = dir + static_cast<size_t>(a) * beams;
  for (int s = 0; s < qb.n; ++s) {
    const double2 cs = da[qb.idx[s]];
    const double ex = x + qb.reach[s] * cs.x;
    const double ey = y + qb.reach[s] * cs.y;
    const int ci = static_cast<int>(floor((ex - ox) / res));
    const int cj = static_cast<int>(floor((ey - oy) / res));
    const bool in = ci >= 0 && ci < w && cj >= 0 && cj < h;
    log_sum += in ? score[static_cast<size_t>(cj) * w + ci] : oob;
  }
  return log_sum;
}

__device__ __forceinline__ void load_query_beams(QueryBeams& qb, const double* __restrict__ ranges, int q,
                                                 int beams, int stride, double max_range, double half_cell) {
  if (threadIdx.x == 0) {
    int n = 0;
    for (int b = 0; b < beams; b += stride) {
      const double r = ranges[static_cast<size_t>(q) * beams + b];
      if (r >= max_range - 1e-9) continue;  // no-return sentinel (observation.cpp:92)
      qb.idx[n] = b;
      qb.reach[n] = r + half_cell;
      ++n;
    }
    qb.n = n;
  }
  __syncthreads();
}

// One CTA per query: the largest log sum and its first candidate index.
__global__ void __launch_bounds__(256) k_difficulty_argmax(
    const uint8_t* __restrict__ occ, const double* __restrict__ score, double oob, int w, int h, double res,
    double ox, double oy, const int2* __restrict__ cells, int n, const double2* __restrict__ dir, int beams,
    int bins, int stride, double max_range, double half_cell, const double* __restrict__ ranges,
    double* __restrict__ best_ls, int* __restrict__ best_idx, int* __restrict__ counted, int* __restrict__ bad) {
  __shared__ QueryBeams qb;
  __shared__ double s_ls[256];
  __shared__ int s_idx[256];
  const int q = blockIdx.x;
  load_query_beams(qb, ranges, q, beams, stride, max_range, half_cell);
  double bl = -__longlong_as_double(0x7ff0000000000000ll);
  int bi = 0x7fffffff;
  const int total = n * bins;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const double ls = cand_log_sum(qb, occ, score, oob, w, h, res, ox, oy, cells, dir, beams, bins, idx, bad);
    if (ls > bl) {  // strict: a thread's indices ascend, so ties keep the first
      bl = ls;
      bi = idx;
    }
  }
  s_ls[threadIdx.x] = bl;
  s_idx[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double l2 = s_ls[threadIdx.x + o];
      const int i2 = s_idx[threadIdx.x + o];
      if (l2 > s_ls[threadIdx.x] || (l2 == s_ls[threadIdx.x] && i2 < s_idx[threadIdx.x])) {
        s_ls[threadIdx.x] = l2;
        s_idx[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    best_ls[q] = s_ls[0];
    best_idx[q] = s_idx[0];
    counted[q] = qb.n;
  }
}

// Per query: how many candidates BEFORE the first maximum have a log sum
// within `window` below it (only those can tie it after glibc's exp).
__global__ void __launch_bounds__(256) k_difficulty_near(
    const uint8_t* __restrict__ occ, const double* __restrict__ score, double oob, int w, int h, double res,
    double ox, double oy, const int2* __restrict__ cells, int n, const double2* __restrict__ dir, int beams,
    int bins, int stride, double max_range, double half_cell, const double* __restrict__ ranges,
    const double* __restrict__ best_ls, const int* __restrict__ best_idx, int* __restrict__ near,
    int* __restrict__ bad) {
  __shared__ QueryBeams qb;
  const int q = blockIdx.x;
  load_query_beams(qb, ranges, q, beams, stride, max_range, half_cell);
  if (qb.n == 0) return;  // every likelihood is 1.0: the host takes candidate 0
  const double M = best_ls[q];
  const double window = qb.n * (1e-14 + 1e-14 * fabs(M / qb.n));
  int cnt = 0;
  for (int idx = threadIdx.x; idx < best_idx[q]; idx += blockDim.x) {
    const double ls = cand_log_sum(qb, occ, score, oob, w, h, res, ox, oy, cells, dir, beams, bins, idx, bad);
    if (ls >= M - window) ++cnt;
  }
  if (cnt) atomicAdd(&near[q], cnt);
}

}  // namespace

void launch_raycast_batch(gl_context* ctx, const uint8_t* occ, int w, int h, double res, double ox, double oy,
                          const double2* xy, const double2* dir, int n_rays, int beams, double max_range,
                          const double* noise, double sigma, double* ranges, int* bad) {
  k_raycast_batch<<<(n_rays + 127) / 128, 128, 0, ctx->stream>>>(occ, w, h, res, ox, oy, xy, dir, n_rays, beams,
                                                                 max_range, noise, sigma, ranges, bad);
  ctx->launches++;
}

void launch_difficulty(gl_context* ctx, const DifficultyArgs& a) {
  const int rt = a.n * a.beams;
  k_raycast_queries<<<(rt + 127) / 128, 128, 0, ctx->stream>>>(a.occ, a.w, a.h, a.res, a.ox, a.oy, a.cells,
                                                               a.n, a.ray, a.beams, a.max_range, a.ranges, a.bad);
  k_difficulty_argmax<<<a.n, 256, 0, ctx->stream>>>(a.occ, a.score, a.oob, a.w, a.h, a.res, a.ox, a.oy, a.cells,
                                                   a.n, a.dir, a.beams, a.bins, a.stride, a.max_range,
                                                   a.half_cell, a.ranges, a.best_ls, a.best_idx, a.counted, a.bad);
  k_difficulty_near<<<a.n, 256, 0, ctx->stream>>>(a.occ, a.score, a.oob, a.w, a.h, a.res, a.ox, a.oy, a.cells,
                                                 a.n, a.dir, a.beams, a.bins, a.stride, a.max_range, a.half_cell,
                                                 a.ranges, a.best_ls, a.best_idx, a.near, a.bad);
  ctx->launches += 3;
}

}  // namespace glb
