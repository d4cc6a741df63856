// The reference's sequential FP64 sums, bit-exact and parallel:
//   dither_samples' total (observation.cpp:16-17: total = 0.0; total += v
//   over the belief map in row-major order) and argmax_state's confidence
//   denominator (belief_tensor.cpp:517-522: total += pl[p] over the tensor in
//   [k][j][i] order).
// A sequential chain is one dependent DADD per element (8+ M cycles for a
// 1024^2 plane, 600+ M for a 1024^2 x 72 tensor). Here it is a scan.
//
// While the running sum s stays inside one binade [2^e, 2^(e+1)) its ulp U
// is fixed and s = M*U with an integer M < 2^53. For x >= 0, fl(s + x) then
// equals (M + r)*U where r = x/U rounded to nearest, ties to the r that
// makes M + r even (IEEE round-half-even on the result). So inside a binade
// the sequential sum is an INTEGER prefix sum of per-element increments r_i,
// except that a tie's r depends on the parity of the running M: each element
// is a map M -> M + a_{M & 1} with two increments (a_0, a_1) (equal unless
// x/U is exactly half-odd), and such maps compose associatively:
// (f then g)_p = f_p + g_{p ^ (f_p & 1)}. A block-wide scan of these pairs
// gives every element's exact running M; the first element whose M reaches
// 2^53 (the sum leaves the binade) is redone as a real DADD from the exact
// predecessor, and the scan restarts in the new binade. The sum only grows
// (x >= 0), so there are few restarts (one per binade crossed).
//
// Ranges where the sum crosses binades (the chunk could not be taken whole)
// take a segmented walk: an approximate prefix assigns every element the
// binade the running sum is in before it; runs of one binade are composed by
// a segmented block scan, and one thread walks runs and edge elements,
// verifying each run's binade and that M stays below 2^53 (on a failed check
// the rest of the chunk goes element by element as above). Leading chunks of
// zeros are skipped by their chunk sums.
//
// Large inputs (launch_seq_sum): a pass over all chunks of 8192 elements on
// every SM takes approximate chunk sums; their prefix says which binade the
// running sum is in across each chunk (with a 1e-7 relative margin, far
// wider than the sequential sum's error bound n*eps); a second full-GPU pass
// composes each such chunk's map under that binade's U; the final single-CTA
// pass then crosses a verified chunk in O(1) (apply its map, check M < 2^53)
// and scans element by element only the chunks where a binade edge falls or
// the guess was wrong. Elements that are negative, infinite or NaN set
// *invalid (callers then run a sequential chain on the device).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "gl_internal.hpp"

namespace glb {

namespace {

constexpr int kSumT = 1024, kSumK = 8, kSumChunk = kSumT * kSumK;
constexpr long long kSumSat = 1ll << 60;
constexpr int kNoGuess = -100000;  // chunk straddles a binade edge (or unknown)

struct IncPair {
  long long a0, a1;  // increment when the running M is even / odd
};

__device__ __forceinline__ long long sat_add(long long a, long long b) {
  const long long c = a + b;
  return c > kSumSat ? kSumSat : c;
}

__device__ __forceinline__ IncPair compose(IncPair f, IncPair g) {  // f, then g
  IncPair c;
  c.a0 = sat_add(f.a0, (f.a0 & 1) ? g.a1 : g.a0);
  c.a1 = sat_add(f.a1, (f.a1 & 1) ? g.a0 : g.a1);
  return c;
}

__device__ __forceinline__ bool bad_value(double x) {
  const long long xb = __double_as_longlong(x);
  // negative (not -0.0), inf, NaN
  return (xb < 0 && xb != static_cast<long long>(0x8000000000000000ull)) || ((xb >> 52) & 0x7ff) == 0x7ff;
}

// x / U rounded: the increment pair of one element (x finite, >= 0 or -0.0)
__device__ __forceinline__ IncPair inc_of(double x, int ulog) {
  const long long xb = __double_as_longlong(x);
  if (xb < 0) return IncPair{0, 0};  // -0.0 adds nothing to a positive sum (bad values are caught apart)
  const int xe = static_cast<int>((xb >> 52) & 0x7ff);
  const long long mx = xe == 0 ? (xb & 0xfffffffffffffll) : ((xb & 0xfffffffffffffll) | (1ll << 52));
  if (mx == 0) return IncPair{0, 0};
  const int xlog = xe == 0 ? -1074 : xe - 1075;  // x = mx * 2^xlog
  const int d = ulog - xlog;                        // x / U = mx * 2^-d
  if (d <= 0) {
    const long long r = (-d >= 8) ? kSumSat : (mx << (-d));
    return IncPair{r, r};
  }
  if (d >= 55) return IncPair{0, 0};  // below half an ulp: no change, never a tie
  const long long rf = mx >> d;
  const long long rem = mx & ((1ll << d) - 1);
  const long long half = 1ll << (d - 1);
  if (rem != half) {
    const long long r = rf + (rem > half ? 1 : 0);
    return IncPair{r, r};
  }
  return IncPair{rf + (rf & 1), rf + ((1 + rf) & 1)};  // tie: the even result
}

__device__ __forceinline__ long long apply(IncPair f, long long m) { return m + ((m & 1) ? f.a1 : f.a0); }

// binade of a positive double: log2 of its ulp, the integer bound of M, M
__device__ __forceinline__ void binade(double s, int* ulog, long long* mmax, long long* m) {
  const long long sb = __double_as_longlong(s);
  const int se = static_cast<int>((sb >> 52) & 0x7ff);
  *ulog = se == 0 ? -1074 : se - 1075;
  *mmax = se == 0 ? (1ll << 52) : (1ll << 53);
  *m = se == 0 ? (sb & 0xfffffffffffffll) : ((sb & 0xfffffffffffffll) | (1ll << 52));
}

__device__ __forceinline__ double ulp_of(int ulog) {  // 2^ulog (subnormal below 2^-1022)
  return __longlong_as_double(ulog >= -1022 ? (static_cast<long long>(ulog + 1023) << 52) : (1ll << (ulog + 1074)));
}

// block-wide inclusive scan of the threads' maps (every thread gets its
// inclusive prefix; s_warp receives the warps' inclusive totals)
__device__ __forceinline__ IncPair block_scan(IncPair mine, IncPair* s_warp, IncPair* excl) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  IncPair incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    IncPair y;
    y.a0 = __shfl_up_sync(0xffffffffu, incl.a0, o);
    y.a1 = __shfl_up_sync(0xffffffffu, incl.a1, o);
    if (lane >= o) incl = compose(y, incl);
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    IncPair wv = lane < (static_cast<int>(blockDim.x) >> 5) ? s_warp[lane] : IncPair{0, 0};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      IncPair y;
      y.a0 = __shfl_up_sync(0xffffffffu, wv.a0, o);
      y.a1 = __shfl_up_sync(0xffffffffu, wv.a1, o);
      if (lane >= o) wv = compose(y, wv);
    }
    if (lane < (static_cast<int>(blockDim.x) >> 5)) s_warp[lane] = wv;
  }
  __syncthreads();
  IncPair el;
  el.a0 = __shfl_up_sync(0xffffffffu, incl.a0, 1);
  el.a1 = __shfl_up_sync(0xffffffffu, incl.a1, 1);
  if (lane == 0) el = IncPair{0, 0};
  *excl = warp > 0 ? compose(s_warp[warp - 1], el) : el;
  return warp > 0 ? compose(s_warp[warp - 1], incl) : incl;
}

// block-wide exclusive scan of one double per thread (approximate prefix sums)
__device__ __forceinline__ double block_excl_sum(double mine, double* s_w) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    double wv = lane < (static_cast<int>(blockDim.x) >> 5) ? s_w[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= o) wv += y;
    }
    if (lane < (static_cast<int>(blockDim.x) >> 5)) s_w[lane] = wv;
  }
  __syncthreads();
  const double r = (warp > 0 ? s_w[warp - 1] : 0.0) + (incl - mine);
  __syncthreads();
  return r;
}

// segmented composition: f = 1 starts a new segment at B
struct SegMap {
  int f;
  IncPair m;
};
__device__ __forceinline__ SegMap seg_compose(SegMap a, SegMap b) {  // a, then b
  return SegMap{a.f | b.f, b.f ? b.m : compose(a.m, b.m)};
}

// block-wide exclusive segmented scan of one SegMap per thread
__device__ __forceinline__ SegMap block_seg_excl(SegMap mine, SegMap* s_w) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  SegMap incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    SegMap y;
    y.f = __shfl_up_sync(0xffffffffu, incl.f, o);
    y.m.a0 = __shfl_up_sync(0xffffffffu, incl.m.a0, o);
    y.m.a1 = __shfl_up_sync(0xffffffffu, incl.m.a1, o);
    if (lane >= o) incl = seg_compose(y, incl);
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    SegMap wv = lane < (static_cast<int>(blockDim.x) >> 5) ? s_w[lane] : SegMap{0, IncPair{0, 0}};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      SegMap y;
      y.f = __shfl_up_sync(0xffffffffu, wv.f, o);
      y.m.a0 = __shfl_up_sync(0xffffffffu, wv.m.a0, o);
      y.m.a1 = __shfl_up_sync(0xffffffffu, wv.m.a1, o);
      if (lane >= o) wv = seg_compose(y, wv);
    }
    if (lane < (static_cast<int>(blockDim.x) >> 5)) s_w[lane] = wv;
  }
  __syncthreads();
  SegMap el;
  el.f = __shfl_up_sync(0xffffffffu, incl.f, 1);
  el.m.a0 = __shfl_up_sync(0xffffffffu, incl.m.a0, 1);
  el.m.a1 = __shfl_up_sync(0xffffffffu, incl.m.a1, 1);
  if (lane == 0) el = SegMap{0, IncPair{0, 0}};
  const SegMap r = warp > 0 ? seg_compose(s_w[warp - 1], el) : el;
  __syncthreads();
  return r;
}

// Binade of the approximate running sum before one element, when it is
// unambiguous across the element (lo..hi inside one binade): log2 of its ulp,
// else kNoGuess (the element is then added as a real DADD).
__device__ __forceinline__ int guess_binade(double before, double after, double margin) {
  const double lo = before * (1.0 - margin), hi = after * (1.0 + margin);
  if (!(lo > 0.0)) return kNoGuess;
  const int el = static_cast<int>((__double_as_longlong(lo) >> 52) & 0x7ff);
  const int eh = static_cast<int>((__double_as_longlong(hi) >> 52) & 0x7ff);
  if (el != eh || el == 0x7ff) return kNoGuess;
  return el == 0 ? -1074 : el - 1075;
}

// Block-collective (kSumT threads): the segmented structure of len <= kSumChunk
// elements x[0, len) entered with the (approximate) running sum P0, as events
// in order: runs of elements in one guessed binade with their composed map,
// and lone elements at binade edges carrying their value (map.a0 = its bits).
// Zeros met while the sum is still 0 are skipped (0.0 + ±0.0 == 0.0). Stores
// at most `cap` events and returns the count; *bad <- any negative or
// non-finite element.
__device__ int seg_events(const double* __restrict__ x, int len, double P0, double margin, int* evstart, int* evg,
                          IncPair* evmap, int cap, int* bad_out) {
  __shared__ double s_dw[32];
  __shared__ SegMap s_segw[32];
  __shared__ int s_w[32];
  __shared__ int s_nev;
  const int tid = threadIdx.x;
  double xv[kSumK];
  double loc = 0.0;
  int bad = 0;
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const int i = tid * kSumK + k;
    xv[k] = i < len ? x[i] : 0.0;
    bad |= bad_value(xv[k]);
    loc += xv[k];
  }
  *bad_out = __syncthreads_or(bad);
  if (*bad_out) return 0;
  double P = P0 + block_excl_sum(loc, s_dw);
  int g[kSumK];
  IncPair inc[kSumK];
  unsigned int skip = 0;
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const int i = tid * kSumK + k;
    const double after = P + xv[k];
    const bool sk = i >= len || (!(P > 0.0) && xv[k] == 0.0);
    skip |= static_cast<unsigned int>(sk) << k;
    g[k] = sk ? kNoGuess : guess_binade(P, after, margin);
    inc[k] = g[k] != kNoGuess ? inc_of(xv[k], g[k])
                              : IncPair{sk ? 0ll : static_cast<long long>(__double_as_longlong(xv[k])), 0};
    P = after;
  }
  // event starts: a lone element (no guess) or the first of a run
  const int tl = tid & 31, tw = tid >> 5;
  if (tl == 31) s_w[tw] = g[kSumK - 1];
  __syncthreads();
  int prev_g = __shfl_up_sync(0xffffffffu, g[kSumK - 1], 1);
  if (tl == 0) prev_g = tid > 0 ? s_w[tw - 1] : kNoGuess;
  int fl[kSumK];
  int nfl = 0;
  SegMap agg{0, IncPair{0, 0}};
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const int pg = k == 0 ? prev_g : g[k - 1];
    fl[k] = !((skip >> k) & 1u) && (g[k] == kNoGuess || pg == kNoGuess || pg != g[k]);
    nfl += fl[k];
    agg = seg_compose(agg, SegMap{fl[k], inc[k]});
  }
  __syncthreads();  // every prev_g read before s_w is reused
  // event numbers: an exclusive count of the starts
  int incl = nfl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (tl >= o) incl += y;
  }
  if (tl == 31) s_w[tw] = incl;
  __syncthreads();
  if (tid < 32) {
    int wv = s_w[tid];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wv, o);
      if (tid >= o) wv += y;
    }
    s_w[tid] = wv;
  }
  __syncthreads();
  const int ev0 = (tw > 0 ? s_w[tw - 1] : 0) + incl - nfl;
  if (tid == kSumT - 1) s_nev = ev0 + nfl;
  const SegMap before = block_seg_excl(agg, s_segw);  // syncs: s_nev visible, s_w reusable
  const int nev = s_nev;
  // does the next thread's first element start an event (or lie past the range)?
  if (tl == 0) s_w[tw] = fl[0] || ((skip & 1u) && tid * kSumK >= len);
  __syncthreads();
  int next_fl0 = __shfl_down_sync(0xffffffffu, fl[0] || ((skip & 1u) && tid * kSumK >= len), 1);
  if (tl == 31) next_fl0 = tw + 1 < (kSumT >> 5) ? s_w[tw + 1] : 1;
  SegMap run = before;
  int e = ev0 - 1;
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const int i = tid * kSumK + k;
    run = seg_compose(run, SegMap{fl[k], inc[k]});
    if (fl[k]) {
      ++e;
      if (e < cap) {
        evstart[e] = i;
        evg[e] = g[k];
      }
    }
    // the event's last element stores its map (a lone element: its value)
    const bool last = i + 1 >= len || (k + 1 < kSumK ? (fl[k + 1] != 0) : (next_fl0 != 0));
    if (!((skip >> k) & 1u) && last && e >= 0 && e < cap) evmap[e] = run.m;
  }
  __syncthreads();
  return nev;
}

// One thread walks events from the exact running sum s: a run is applied only
// if s is in its guessed binade and M stays below 2^53; a lone element is a
// real DADD. Returns -1, or the first element (relative) of the event where a
// check failed (s then holds the exact sum before it).
__device__ int walk_events(double& s, const int* evstart, const int* evg, const IncPair* evmap, int nev) {
  for (int ev = 0; ev < nev; ++ev) {
    const int gg = evg[ev];
    if (gg == kNoGuess) {
      s = s + __longlong_as_double(evmap[ev].a0);
      continue;
    }
    if (!(s > 0.0)) return evstart[ev];
    int ul;
    long long mm, m0;
    binade(s, &ul, &mm, &m0);
    const long long m1 = apply(evmap[ev], m0);
    if (ul != gg || m1 >= mm) return evstart[ev];
    s = static_cast<double>(m1) * ulp_of(ul);
  }
  return -1;
}

// A thread's K increments under ulp 2^ulog in FP64, when none is a tie: x/U
// is a power-of-two scaling (exact; an underflow only happens far below 1/2),
// (y + 2^52) - 2^52 rounds it half-to-even, and sums of integers below 2^53
// are exact. Returns false on a tie (x/U exactly half an odd integer... any
// half-integer): the increment pair then depends on the running M's parity.
// An increment of 2^52 or more always leaves the binade: saturated.
__device__ __forceinline__ bool inc_sum_fp64(const double (&xv)[kSumK], int ulog, long long* out) {
  const int e1 = -ulog > 1000 ? 1000 : -ulog;  // 2^-ulog (up to 2^1074) in two factors
  const int e2 = -ulog - e1;
  const double f1 = __longlong_as_double(static_cast<long long>(e1 + 1023) << 52);
  const double f2 = __longlong_as_double(static_cast<long long>(e2 + 1023) << 52);
  constexpr double kTwo52 = 4503599627370496.0;
  double sum = 0.0;
  bool tie = false, big = false;
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const double y = (xv[k] * f1) * f2;
    big |= y >= kTwo52;
    const double r = (y + kTwo52) - kTwo52;
    tie |= fabs(y - r) == 0.5;
    sum += r;
  }
  if (tie) return false;
  *out = (big || sum >= 2.0 * kTwo52) ? kSumSat : static_cast<long long>(sum);
  return true;
}

// argmax_state's candidate (the layout launch_argmax writes): the first
// maximum in index order, compared with a strict > from -1.0
struct ArgBest {
  double v;
  long long idx;
  double unused;
};
__device__ __forceinline__ ArgBest arg_better(ArgBest a, ArgBest b) {
  return ((b.v > a.v) || (b.v == a.v && b.idx < a.idx)) ? b : a;
}
__device__ __forceinline__ ArgBest arg_shfl_xor(ArgBest a, int o) {
  ArgBest r;
  r.v = __shfl_xor_sync(0xffffffffu, a.v, o);
  r.idx = __shfl_xor_sync(0xffffffffu, a.idx, o);
  r.unused = 0.0;
  return r;
}

// ---- phase 1: approximate chunk sums (pairwise) + the domain check -------
// (+ argmax_state's per-chunk candidate when `arg` is given: one read of x)
__global__ void __launch_bounds__(256) k_chunk_sums(const double* __restrict__ x, size_t n, double* __restrict__ S,
                                                    int* __restrict__ invalid, ArgBest* __restrict__ arg) {
  __shared__ double ws[8];
  __shared__ ArgBest wa[8];
  const size_t c0 = static_cast<size_t>(blockIdx.x) * kSumChunk;
  double acc = 0.0;
  int bad = 0;
  ArgBest best{-1.0, 0x7fffffffffffffffll, 0.0};
  auto take = [&](double v, size_t q) {
    bad |= bad_value(v);
    acc += v;
    if (v > best.v) {  // strict: the first (lowest) index of a tie
      best.v = v;
      best.idx = static_cast<long long>(q);
    }
  };
  if (c0 + kSumChunk <= n) {  // a full chunk: loads batched, no bounds checks
    constexpr int kU = 8;
    for (int k0 = threadIdx.x; k0 < kSumChunk; k0 += 256 * kU) {
      double v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = x[c0 + k0 + u * 256];
#pragma unroll
      for (int u = 0; u < kU; ++u) take(v[u], c0 + k0 + u * 256);
    }
  } else {
    for (int k = threadIdx.x; k < kSumChunk; k += 256) {
      const size_t q = c0 + k;
      if (q < n) take(x[q], q);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *invalid = 1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  if (arg) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = arg_better(best, arg_shfl_xor(best, o));
    if ((threadIdx.x & 31) == 0) wa[threadIdx.x >> 5] = best;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    S[blockIdx.x] = t;
    if (arg) {
      ArgBest b = wa[0];
      for (int w = 1; w < 8; ++w) b = arg_better(b, wa[w]);
      arg[blockIdx.x] = b;
    }
  }
}

// the chunk candidates' best (argmax_state's result)
__global__ void __launch_bounds__(1024) k_arg_final(const ArgBest* __restrict__ arg, int n_chunks,
                                                    ArgBest* __restrict__ out) {
  __shared__ ArgBest wa[32];
  ArgBest best{-1.0, 0x7fffffffffffffffll, 0.0};
  for (int c = threadIdx.x; c < n_chunks; c += 1024) best = arg_better(best, arg[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = arg_better(best, arg_shfl_xor(best, o));
  if ((threadIdx.x & 31) == 0) wa[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    ArgBest b = wa[0];
    for (int w = 1; w < 32; ++w) b = arg_better(b, wa[w]);
    *out = b;
  }
}

// ---- phase 2: which binade the running sum is in across each chunk -------
__global__ void __launch_bounds__(1024) k_chunk_guess(const double* __restrict__ S, int n_chunks, double s0,
                                                      int* __restrict__ guess, double* __restrict__ Pc) {
  // approximate prefix of the chunk sums (a block scan, tile by tile)
  __shared__ double ws[32];
  __shared__ double carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = s0;  // the running sum enters with s0
  __syncthreads();
  for (int base = 0; base < n_chunks; base += 1024) {
    const int c = base + tid;
    const double v = c < n_chunks ? S[c] : 0.0;
    double incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) ws[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      double wv = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, wv, o);
        if (lane >= o) wv += y;
      }
      ws[lane] = wv;
    }
    __syncthreads();
    const double before = carry + (warp > 0 ? ws[warp - 1] : 0.0) + (incl - v);
    if (c < n_chunks) {
      // the sequential running sum is within n*eps (relative) of the exact
      // prefix; a 1e-7 margin covers any input of < 10^8 elements
      const double lo = before * (1.0 - 1e-7), hi = (before + v) * (1.0 + 1e-7);
      int g = kNoGuess;
      if (lo > 0.0) {
        const int el = static_cast<int>((__double_as_longlong(lo) >> 52) & 0x7ff);
        const int eh = static_cast<int>((__double_as_longlong(hi) >> 52) & 0x7ff);
        if (el == eh && el != 0x7ff) g = el == 0 ? -1074 : el - 1075;
      }
      guess[c] = g;
      Pc[c] = before;
    }
    __syncthreads();
    if (tid == 1023) carry = carry + ws[31];
    __syncthreads();
  }
}

// ---- phase 3a: crossing chunks' events (all SMs) ------------------------
constexpr int kEvCap = 256;   // events per crossing chunk precomputed by the all-SM pass
constexpr int kEvPool = 512;  // crossing chunks that get precomputed events (the rest: the walk's own pass)

// A persistent grid walks the chunks: most are guessed (nothing to do).
__global__ void __launch_bounds__(kSumT) k_chunk_events(const double* __restrict__ x, size_t n, int n_chunks,
                                                        const int* __restrict__ guess, const double* __restrict__ Pc,
                                                        int* __restrict__ ev_n, int* __restrict__ ev_slot,
                                                        int* __restrict__ pool_ctr, int* __restrict__ pool_start,
                                                        int* __restrict__ pool_g, IncPair* __restrict__ pool_map) {
  __shared__ int s_slot;
  for (int c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    if (guess[c] != kNoGuess) {
      if (threadIdx.x == 0) ev_n[c] = -1;
      continue;
    }
    // a chunk where the running sum crosses binades: its events, from the
    // approximate prefix before it (the walk verifies every run)
    if (threadIdx.x == 0) s_slot = atomicAdd(pool_ctr, 1);
    __syncthreads();
    const int slot = s_slot;
    __syncthreads();
    if (slot >= kEvPool) {
      if (threadIdx.x == 0) ev_n[c] = -1;
      continue;
    }
    const size_t c0 = static_cast<size_t>(c) * kSumChunk;
    const int len = static_cast<int>(min(static_cast<size_t>(kSumChunk), n - c0));
    int bad;
    const int nev = seg_events(x + c0, len, Pc[c], 1e-7, pool_start + slot * kEvCap, pool_g + slot * kEvCap,
                               pool_map + static_cast<size_t>(slot) * kEvCap, kEvCap, &bad);
    if (threadIdx.x == 0) {
      ev_n[c] = (bad || nev > kEvCap) ? -1 : nev;
      ev_slot[c] = slot;
    }
  }
}

// ---- phase 3: each guessed chunk's composed map ---------------------------
__global__ void __launch_bounds__(kSumT, 2) k_chunk_maps(const double* __restrict__ x, size_t n,
                                                         const int* __restrict__ guess, IncPair* __restrict__ maps) {
  __shared__ IncPair s_warp[32];
  __shared__ long long s_sum[32];
  const int g = guess[blockIdx.x];
  if (g == kNoGuess) return;
  const size_t c0 = static_cast<size_t>(blockIdx.x) * kSumChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Without ties the chunk's map is {R, R} with R the sum of the increments,
  // and an integer sum has no order: coalesced loads, any association.
  double xv[kSumK];
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const size_t q = c0 + threadIdx.x + static_cast<size_t>(k) * kSumT;
    xv[k] = q < n ? x[q] : 0.0;
  }
  long long r;
  const bool no_tie = inc_sum_fp64(xv, g, &r);
  if (__syncthreads_and(no_tie)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r = sat_add(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (lane == 0) s_sum[warp] = r;
    __syncthreads();
    if (warp == 0) {
      r = s_sum[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) r = sat_add(r, __shfl_xor_sync(0xffffffffu, r, o));
      if (lane == 0) maps[blockIdx.x] = IncPair{r, r};
    }
    return;
  }
  // a tie somewhere: the ordered composition of each thread's K consecutive
  // elements, then of the threads in order (lane l, then l + o)
  const size_t base = c0 + static_cast<size_t>(threadIdx.x) * kSumK;
#pragma unroll
  for (int k = 0; k < kSumK; ++k) xv[k] = base + k < n ? x[base + k] : 0.0;
  IncPair mine{0, 0};
#pragma unroll
  for (int k = 0; k < kSumK; ++k) mine = compose(mine, inc_of(xv[k], g));
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    IncPair y;
    y.a0 = __shfl_down_sync(0xffffffffu, mine.a0, o);
    y.a1 = __shfl_down_sync(0xffffffffu, mine.a1, o);
    if ((lane & (2 * o - 1)) == 0) mine = compose(mine, y);
  }
  if (lane == 0) s_warp[warp] = mine;
  __syncthreads();
  if (warp == 0) {
    mine = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      IncPair y;
      y.a0 = __shfl_down_sync(0xffffffffu, mine.a0, o);
      y.a1 = __shfl_down_sync(0xffffffffu, mine.a1, o);
      if ((lane & (2 * o - 1)) == 0) mine = compose(mine, y);
    }
    if (lane == 0) maps[blockIdx.x] = mine;
  }
}

// ---- phase 3b: runs of consecutive chunks guessed for one binade, composed
// in order (one CTA, a segmented scan over tiles of 1024 chunks): the walk
// then crosses a whole run with one map, checked like a chunk's.
struct RunAcc {
  int f;      // 1: a run starts here (or a non-member breaks the run)
  int start;  // the run's first chunk
  IncPair m;
};
__device__ __forceinline__ RunAcc run_combine(RunAcc a, RunAcc b) {  // a, then b
  return b.f ? b : RunAcc{a.f, a.start, compose(a.m, b.m)};
}
__device__ __forceinline__ RunAcc run_shfl_up(RunAcc a, int o) {
  RunAcc r;
  r.f = __shfl_up_sync(0xffffffffu, a.f, o);
  r.start = __shfl_up_sync(0xffffffffu, a.start, o);
  r.m.a0 = __shfl_up_sync(0xffffffffu, a.m.a0, o);
  r.m.a1 = __shfl_up_sync(0xffffffffu, a.m.a1, o);
  return r;
}

__global__ void __launch_bounds__(1024) k_chunk_runs(const int* __restrict__ guess, const IncPair* __restrict__ maps,
                                                     int n_chunks, int* __restrict__ run_end,
                                                     IncPair* __restrict__ run_map) {
  __shared__ RunAcc s_w[32];
  __shared__ RunAcc s_carry;  // the run still open at the end of the previous tile (f = 1)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = RunAcc{1, -1, IncPair{0, 0}};
  __syncthreads();
  for (int t0 = 0; t0 < n_chunks; t0 += 1024) {
    const int c = t0 + tid;
    const int g = c < n_chunks ? guess[c] : kNoGuess;
    const int gprev = (c > 0 && c - 1 < n_chunks) ? guess[c - 1] : kNoGuess;
    const bool member = g != kNoGuess;
    const bool starts = member && gprev != g;
    RunAcc mine = member ? RunAcc{starts ? 1 : 0, starts ? c : -1, maps[c]} : RunAcc{1, -1, IncPair{0, 0}};
    if (tid == 0 && member && !starts) mine = run_combine(s_carry, mine);  // continues the open run
    // block-wide inclusive segmented scan
    RunAcc incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const RunAcc y = run_shfl_up(incl, o);
      if (lane >= o) incl = run_combine(y, incl);
    }
    if (lane == 31) s_w[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      RunAcc wv = s_w[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const RunAcc y = run_shfl_up(wv, o);
        if (lane >= o) wv = run_combine(y, wv);
      }
      s_w[lane] = wv;
    }
    __syncthreads();
    if (warp > 0) incl = run_combine(s_w[warp - 1], incl);
    const int gnext = c + 1 < n_chunks ? guess[c + 1] : kNoGuess;
    if (member && gnext != g && incl.start >= 0) {  // the run's last chunk
      run_end[incl.start] = c + 1;
      run_map[incl.start] = incl.m;
    }
    __syncthreads();
    if (tid == 1023) s_carry = (member && gnext == g) ? RunAcc{1, incl.start, incl.m} : RunAcc{1, -1, IncPair{0, 0}};
    __syncthreads();
  }
}

// ---- phase 4 (or the whole sum for small inputs): one CTA walks the chunks
#ifdef GL_EXPERIMENT_ENV
__device__ long long g_seq_dbg[8];  // whole-chunk steps, segmented ok, segmented failed, events, element-wise steps, over-cap
#define SEQ_DBG(i, v) do { if (threadIdx.x == 0) g_seq_dbg[i] += (v); } while (0)
#else
#define SEQ_DBG(i, v) do { } while (0)
#endif
constexpr int kSegEv = 2048;  // events (segments + lone elements) per range in the segmented walk
struct SeqSmem {
  IncPair evmap[kSegEv];   // a run's composed map (a lone element: its value's bits)
  int evstart[kSegEv];     // an event's first element (relative)
  int evg[kSegEv];         // its binade (kNoGuess: one element, a real DADD)
};
constexpr size_t kSeqSmem = sizeof(SeqSmem);

__global__ void __launch_bounds__(kSumT) k_seq_sum(const double* __restrict__ x, size_t n, double s0,
                                                   const int* __restrict__ guess, const IncPair* __restrict__ maps,
                                                   const double* __restrict__ S, const int* __restrict__ ev_n,
                                                   const int* __restrict__ ev_slot, const int* __restrict__ pool_start,
                                                   const int* __restrict__ pool_g, const IncPair* __restrict__ pool_map,
                                                   const int* __restrict__ run_end, const IncPair* __restrict__ run_map,
                                                   double* __restrict__ total, int* __restrict__ invalid) {
  extern __shared__ __align__(16) unsigned char seq_dyn[];
  SeqSmem& sm = *reinterpret_cast<SeqSmem*>(seq_dyn);
  __shared__ IncPair s_warp[32];
  __shared__ int s_fail;
  __shared__ double s_walk;
  size_t seg_skip = ~size_t(0);  // a chunk whose segmented walk failed (its rest goes element-wise)
  size_t pre_skip = ~size_t(0);  // a chunk whose precomputed events failed (its rest: the walk's own pass)
  __shared__ unsigned long long s_cross;  // first element whose running M leaves the binade
  __shared__ long long s_mprev;            // its predecessor's M
  __shared__ long long s_mend;             // M at the end of the range (no crossing)
  __shared__ unsigned long long s_first;   // first nonzero element (while s == 0)
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  if (guess && *invalid) return;  // phase 1 found negative / non-finite values
  if (tid == 0) s_bad = 0;
  __syncthreads();
  double s = s0;  // block-uniform running sum (the caller's start: 0.0, or a previous shard's)
  if (!(s >= 0.0) || s == __longlong_as_double(0x7ff0000000000000ll)) {
    if (tid == 0) *invalid = 1;
    return;
  }
  s = s + 0.0;  // -0.0 -> +0.0, as 0.0 + ... would
  size_t pos = 0;
  while (pos < n) {
    // every range ends at the next chunk boundary, so ranges after a binade
    // crossing re-align with the per-chunk maps
    const size_t end = min(n, (pos / kSumChunk + 1) * static_cast<size_t>(kSumChunk));
    // 0.0 + x == x exactly: while the sum is 0 it starts at the first nonzero
    // element. Whole chunks of zeros (chunk sum 0: no negative values here)
    // are skipped 1024 at a time.
    if (s == 0.0 && S && pos % kSumChunk == 0) {
      const size_t c0 = pos / kSumChunk;
      const size_t nch = (n + kSumChunk - 1) / kSumChunk;
      if (tid == 0) s_first = ~0ull;
      __syncthreads();
      if (c0 + tid < nch && S[c0 + tid] != 0.0) atomicMin(&s_first, static_cast<unsigned long long>(c0 + tid));
      __syncthreads();
      const unsigned long long fc = s_first;
      __syncthreads();
      const size_t to = fc == ~0ull ? min(nch, c0 + kSumT) : static_cast<size_t>(fc);
      if (to > c0) {
        pos = min(n, to * static_cast<size_t>(kSumChunk));
        continue;
      }
    }
    // a crossing chunk whose events the all-SM pass precomputed
    if (ev_n && pos % kSumChunk == 0 && pos / kSumChunk != pre_skip) {
      const size_t c = pos / kSumChunk;
      const int ne = ev_n[c];
      if (ne >= 0) {
        const int slot = ev_slot[c];
        for (int i = tid; i < ne; i += kSumT) {
          sm.evstart[i] = pool_start[slot * kEvCap + i];
          sm.evg[i] = pool_g[slot * kEvCap + i];
          sm.evmap[i] = pool_map[static_cast<size_t>(slot) * kEvCap + i];
        }
        __syncthreads();
        if (tid == 0) {
          double sw = s;
          s_fail = walk_events(sw, sm.evstart, sm.evg, sm.evmap, ne);
          s_walk = sw;
        }
        __syncthreads();
        s = s_walk;
        const int fail = s_fail;
        __syncthreads();
        if (fail < 0) {
          pos = end;
        } else {
          pos += fail;  // exact s before element `fail`
          pre_skip = c;
        }
        SEQ_DBG(6, 1);
        continue;
      }
    }
    if (s == 0.0) {
      if (tid == 0) s_first = ~0ull;
      __syncthreads();
      for (size_t q = pos + tid; q < end; q += kSumT)
        if (x[q] != 0.0) atomicMin(&s_first, static_cast<unsigned long long>(q));
      __syncthreads();
      const unsigned long long f = s_first;
      __syncthreads();
      if (f == ~0ull) {
        pos = end;
        continue;
      }
      s = 0.0 + x[f];  // the reference's first effective add
      if (!(s >= 0.0) || s == __longlong_as_double(0x7ff0000000000000ll)) {
        if (tid == 0) *invalid = 1;
        return;
      }
      pos = f + 1;
      continue;
    }
    int ulog;
    long long mmax, m0;
    binade(s, &ulog, &mmax, &m0);
    const double u = ulp_of(ulog);
    // a whole run of chunks guessed for this binade, with its composed map
    if (run_end && pos % kSumChunk == 0) {
      const size_t c0 = pos / kSumChunk;
      if (guess[c0] == ulog) {
        const int re = run_end[c0];
        if (re > static_cast<int>(c0)) {
          const long long m1 = apply(run_map[c0], m0);
          if (m1 < mmax) {
            s = static_cast<double>(m1) * u;
            pos = min(n, static_cast<size_t>(re) * kSumChunk);
            SEQ_DBG(7, 1);
            continue;
          }
        }
      }
    }
    // whole chunks whose maps were composed under this binade, up to 1024
    // at once: the same scan one level up (chunk maps as elements; a chunk
    // guessed for another binade acts as a crossing)
    if (maps && pos % kSumChunk == 0) {
      const size_t c0 = pos / kSumChunk;
      const size_t nch = (n + kSumChunk - 1) / kSumChunk;
      const size_t c = c0 + tid;
      const bool ok = c < nch && guess[c] == ulog;
      const IncPair f = ok ? maps[c] : IncPair{kSumSat, kSumSat};
      if (tid == 0) s_cross = ~0ull;
      IncPair before;
      block_scan(f, s_warp, &before);
      const long long mb = apply(before, m0);
      const long long ma = apply(f, mb);
      if (mb < mmax && ma >= mmax) atomicMin(&s_cross, static_cast<unsigned long long>(tid));
      __syncthreads();
      const unsigned long long stop = s_cross;  // first chunk (relative) that is not taken whole
      if (stop == ~0ull) {                       // all 1024 taken (only if the input ran out)
        if (tid == kSumT - 1) s_mend = ma;
      } else if (tid == static_cast<int>(stop)) {
        s_mend = mb;
      }
      __syncthreads();
      const size_t taken = stop == ~0ull ? kSumT : stop;
      if (taken > 0) {
        SEQ_DBG(0, 1);
        s = static_cast<double>(s_mend) * u;
        pos = min(n, (c0 + taken) * static_cast<size_t>(kSumChunk));
        __syncthreads();
        continue;
      }
      __syncthreads();
    }
    // ---- segmented walk: an approximate prefix gives every element the
    // binade the running sum is in before it; runs of elements in one binade
    // are composed in a segmented scan, and one thread walks the runs (apply
    // the run's map, check the binade and that M stays < 2^53) and adds the
    // elements at binade edges as real DADDs. Many crossings cost one pass.
    if (pos / kSumChunk != seg_skip) {
      const int len = static_cast<int>(end - pos);
      int bad;
      const int nev = seg_events(x + pos, len, s, 1e-9, sm.evstart, sm.evg, sm.evmap, kSegEv, &bad);
      if (bad) {
        if (tid == 0) *invalid = 1;
        return;
      }
      if (nev <= kSegEv) {
        if (tid == 0) {
          double sw = s;
          s_fail = walk_events(sw, sm.evstart, sm.evg, sm.evmap, nev);
          s_walk = sw;
        }
        __syncthreads();
        s = s_walk;
        const int fail = s_fail;
        __syncthreads();
        SEQ_DBG(3, nev);
        if (fail < 0) {
          SEQ_DBG(1, 1);
          pos = end;
          continue;
        }
        SEQ_DBG(2, 1);
        pos += fail;  // exact s before element `fail`; the chunk's rest goes element-wise
        seg_skip = pos / kSumChunk;
        continue;
      }
      SEQ_DBG(5, 1);
      seg_skip = pos / kSumChunk;
      __syncthreads();
    }
    // element by element: this thread's K consecutive elements of [pos, end)
    SEQ_DBG(4, 1);
    const size_t base = pos + static_cast<size_t>(tid) * kSumK;
    IncPair inc[kSumK];
    int bad = 0;
    IncPair mine{0, 0};
#pragma unroll
    for (int k = 0; k < kSumK; ++k) {
      const size_t q = base + k;
      if (q < end) {
        const double v = x[q];
        bad |= bad_value(v);
        inc[k] = inc_of(v, ulog);
      } else {
        inc[k] = IncPair{0, 0};
      }
      mine = compose(mine, inc[k]);
    }
    if (bad) s_bad = 1;
    if (tid == 0) {
      s_cross = ~0ull;
      s_mend = -1;
    }
    IncPair before;
    block_scan(mine, s_warp, &before);  // syncs: s_bad / s_cross / s_mend are visible after it
    if (s_bad) {
      if (tid == 0) *invalid = 1;
      return;
    }
    long long m = apply(before, m0);
    // walk this thread's elements; the first crossing in the block wins
    if (m < mmax) {
#pragma unroll
      for (int k = 0; k < kSumK; ++k) {
        const long long nm = apply(inc[k], m);
        if (nm >= mmax) {
          atomicMin(&s_cross, static_cast<unsigned long long>(base + k));
          break;
        }
        m = nm;
      }
    }
    __syncthreads();
    const unsigned long long cross = s_cross;
    if (cross == ~0ull) {
      if (tid == kSumT - 1) s_mend = m;  // the block's last thread holds the range's end
      __syncthreads();
      s = static_cast<double>(s_mend) * u;
      pos = end;
      __syncthreads();
      continue;
    }
    // the crossing element's thread knows its predecessor's exact M
    if (base <= cross && cross < base + kSumK) {
      long long mp = apply(before, m0);
      for (size_t q = base; q < cross; ++q) mp = apply(inc[q - base], mp);
      s_mprev = mp;
    }
    __syncthreads();
    const double sprev = static_cast<double>(s_mprev) * u;  // exact: M < 2^53
    s = sprev + x[cross];                                     // the real DADD across the binade edge
    pos = cross + 1;
    __syncthreads();
  }
  if (tid == 0) *total = s;
}

// The reference's literal chain on one thread, for inputs outside the scan's
// domain (negative or non-finite values): runs only if *when != 0.
__global__ void k_seq_sum_chain(const double* __restrict__ x, size_t n, double s0, const int* __restrict__ when,
                                double* __restrict__ total) {
  if (when && *when == 0) return;
  double t = s0;
  for (size_t q = 0; q < n; ++q) t += x[q];
  *total = t;
}

}  // namespace

size_t seq_sum_scratch_bytes(size_t n) {
  const size_t chunks = (n + kSumChunk - 1) / kSumChunk;
  return chunks * (2 * sizeof(IncPair) + 2 * sizeof(double) + 4 * sizeof(int) + sizeof(ArgBest)) + 64 +
         static_cast<size_t>(kEvPool) * kEvCap * (sizeof(IncPair) + 2 * sizeof(int)) + 64;
}

static void seq_sum_smem_attr() {
  static const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(k_seq_sum),
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    static_cast<int>(kSeqSmem));
  if (e != cudaSuccess) throw std::runtime_error(std::string("seq-sum shared-memory opt-in: ") + cudaGetErrorString(e));
}

void launch_seq_sum(gl_context* ctx, const double* x, size_t n, double* d_total, int* d_invalid, double s0) {
  seq_sum_smem_attr();
  cudaMemsetAsync(d_invalid, 0, sizeof(int), ctx->stream);
  k_seq_sum<<<1, kSumT, kSeqSmem, ctx->stream>>>(x, n, s0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                 nullptr, nullptr, nullptr, nullptr, d_total, d_invalid);
  ctx->launches++;
}

// From two chunks on, the all-SM passes (chunk maps, crossing chunks' events)
// beat one CTA's own segmented walk.
constexpr size_t kBigMinChunks = 2;
bool seq_sum_fuses_argmax(size_t n) { return (n + kSumChunk - 1) / kSumChunk >= kBigMinChunks; }

void launch_seq_sum_big(gl_context* ctx, const double* x, size_t n, double* d_total, int* d_invalid,
                        void* scratch, double s0, void* d_argmax) {
  const size_t chunks = (n + kSumChunk - 1) / kSumChunk;
  if (d_argmax && !seq_sum_fuses_argmax(n)) throw std::runtime_error("seq-sum: argmax fusion needs 2+ chunks");
  if (chunks < kBigMinChunks) {
    launch_seq_sum(ctx, x, n, d_total, d_invalid, s0);
    return;
  }
  const size_t pool = static_cast<size_t>(kEvPool) * kEvCap;
  auto* maps = static_cast<IncPair*>(scratch);  // 16-byte aligned first
  auto* pool_map = maps + chunks;
  auto* S = reinterpret_cast<double*>(pool_map + pool);
  auto* Pc = S + chunks;
  auto* guess = reinterpret_cast<int*>(Pc + chunks);
  auto* ev_n = guess + chunks;
  auto* ev_slot = ev_n + chunks;
  auto* pool_start = ev_slot + chunks;
  auto* pool_g = pool_start + pool;
  auto* pool_ctr = pool_g + pool;
  auto* arg = reinterpret_cast<ArgBest*>((reinterpret_cast<uintptr_t>(pool_ctr + 1) + 15) & ~uintptr_t(15));
  auto* run_map = reinterpret_cast<IncPair*>(arg + chunks);  // 16-byte aligned (ArgBest is 24 B: realign)
  run_map = reinterpret_cast<IncPair*>((reinterpret_cast<uintptr_t>(run_map) + 15) & ~uintptr_t(15));
  auto* run_end = reinterpret_cast<int*>(run_map + chunks);
  cudaMemsetAsync(run_end, 0, sizeof(int) * chunks, ctx->stream);
  cudaMemsetAsync(d_invalid, 0, sizeof(int), ctx->stream);
  cudaMemsetAsync(pool_ctr, 0, sizeof(int), ctx->stream);
  const int nc = static_cast<int>(chunks);
  k_chunk_sums<<<nc, 256, 0, ctx->stream>>>(x, n, S, d_invalid, d_argmax ? arg : nullptr);
  if (d_argmax) {
    k_arg_final<<<1, 1024, 0, ctx->stream>>>(arg, nc, static_cast<ArgBest*>(d_argmax));
    ctx->launches++;
  }
  k_chunk_guess<<<1, 1024, 0, ctx->stream>>>(S, nc, s0, guess, Pc);
  k_chunk_maps<<<nc, kSumT, 0, ctx->stream>>>(x, n, guess, maps);
  const int ev_grid = min(nc, 2 * (ctx->sm_count > 0 ? ctx->sm_count : 148));
  k_chunk_events<<<ev_grid, kSumT, 0, ctx->stream>>>(x, n, nc, guess, Pc, ev_n, ev_slot, pool_ctr, pool_start, pool_g,
                                                     pool_map);
  seq_sum_smem_attr();
  k_chunk_runs<<<1, 1024, 0, ctx->stream>>>(guess, maps, nc, run_end, run_map);
  k_seq_sum<<<1, kSumT, kSeqSmem, ctx->stream>>>(x, n, s0, guess, maps, S, ev_n, ev_slot, pool_start, pool_g,
                                                 pool_map, run_end, run_map, d_total, d_invalid);
  ctx->launches += 6;
#ifdef GL_EXPERIMENT_ENV
  if (getenv("GL_DEBUG_SEQSUM")) {
    long long h[8];
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpyFromSymbol(h, g_seq_dbg, sizeof(h));
    fprintf(stderr, "seq sum n=%zu chunks=%zu: whole-chunk steps %lld, segmented ok %lld, failed %lld, events %lld, element-wise steps %lld, over cap %lld, precomputed chunks %lld, runs %lld\n",
            n, chunks, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    const long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_seq_dbg, z, sizeof(z));
  }
#endif
}

void launch_seq_sum_chain(gl_context* ctx, const double* x, size_t n, double* d_total, const int* when, double s0) {
  k_seq_sum_chain<<<1, 1, 0, ctx->stream>>>(x, n, s0, when, d_total);
  ctx->launches++;
}

}  // namespace glb
