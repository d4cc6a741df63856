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

// ---- phase 1: approximate chunk sums (pairwise) + the domain check -------
__global__ void __launch_bounds__(256) k_chunk_sums(const double* __restrict__ x, size_t n, double* __restrict__ S,
                                                    int* __restrict__ invalid) {
  __shared__ double ws[8];
  const size_t c0 = static_cast<size_t>(blockIdx.x) * kSumChunk;
  double acc = 0.0;
  int bad = 0;
  for (int k = threadIdx.x; k < kSumChunk; k += 256) {
    const size_t q = c0 + k;
    if (q < n) {
      const double v = x[q];
      bad |= bad_value(v);
      acc += v;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *invalid = 1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    S[blockIdx.x] = t;
  }
}

// ---- phase 2: which binade the running sum is in across each chunk -------
__global__ void __launch_bounds__(1024) k_chunk_guess(const double* __restrict__ S, int n_chunks, double s0,
                                                      int* __restrict__ guess) {
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
    }
    __syncthreads();
    if (tid == 1023) carry = carry + ws[31];
    __syncthreads();
  }
}

// ---- phase 3: each guessed chunk's composed map ---------------------------
__global__ void __launch_bounds__(kSumT) k_chunk_maps(const double* __restrict__ x, size_t n,
                                                      const int* __restrict__ guess, IncPair* __restrict__ maps) {
  __shared__ IncPair s_warp[32];
  const int g = guess[blockIdx.x];
  if (g == kNoGuess) return;
  const size_t base = static_cast<size_t>(blockIdx.x) * kSumChunk + static_cast<size_t>(threadIdx.x) * kSumK;
  IncPair mine{0, 0};
#pragma unroll
  for (int k = 0; k < kSumK; ++k) {
    const size_t q = base + k;
    if (q < n) mine = compose(mine, inc_of(x[q], g));
  }
  IncPair excl;
  const IncPair incl = block_scan(mine, s_warp, &excl);
  if (threadIdx.x == kSumT - 1) maps[blockIdx.x] = incl;
}

// ---- phase 4 (or the whole sum for small inputs): one CTA walks the chunks
__global__ void __launch_bounds__(kSumT) k_seq_sum(const double* __restrict__ x, size_t n, double s0,
                                                   const int* __restrict__ guess, const IncPair* __restrict__ maps,
                                                   double* __restrict__ total, int* __restrict__ invalid) {
  __shared__ IncPair s_warp[32];
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
    if (s == 0.0) {
      // 0.0 + x == x exactly: the sum starts at the first nonzero element
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
        s = static_cast<double>(s_mend) * u;
        pos = min(n, (c0 + taken) * static_cast<size_t>(kSumChunk));
        __syncthreads();
        continue;
      }
      __syncthreads();
    }
    // element by element: this thread's K consecutive elements of [pos, end)
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
  return chunks * (sizeof(double) + sizeof(int) + sizeof(IncPair)) + 64;
}

void launch_seq_sum(gl_context* ctx, const double* x, size_t n, double* d_total, int* d_invalid, double s0) {
  cudaMemsetAsync(d_invalid, 0, sizeof(int), ctx->stream);
  k_seq_sum<<<1, kSumT, 0, ctx->stream>>>(x, n, s0, nullptr, nullptr, d_total, d_invalid);
  ctx->launches++;
}

void launch_seq_sum_big(gl_context* ctx, const double* x, size_t n, double* d_total, int* d_invalid,
                        void* scratch, double s0) {
  const size_t chunks = (n + kSumChunk - 1) / kSumChunk;
  if (chunks <= 4) {
    launch_seq_sum(ctx, x, n, d_total, d_invalid, s0);
    return;
  }
  auto* maps = static_cast<IncPair*>(scratch);  // 16-byte aligned first
  auto* S = reinterpret_cast<double*>(maps + chunks);
  auto* guess = reinterpret_cast<int*>(S + chunks);
  cudaMemsetAsync(d_invalid, 0, sizeof(int), ctx->stream);
  const int nc = static_cast<int>(chunks);
  k_chunk_sums<<<nc, 256, 0, ctx->stream>>>(x, n, S, d_invalid);
  k_chunk_guess<<<1, 1024, 0, ctx->stream>>>(S, nc, s0, guess);
  k_chunk_maps<<<nc, kSumT, 0, ctx->stream>>>(x, n, guess, maps);
  k_seq_sum<<<1, kSumT, 0, ctx->stream>>>(x, n, s0, guess, maps, d_total, d_invalid);
  ctx->launches += 4;
}

void launch_seq_sum_chain(gl_context* ctx, const double* x, size_t n, double* d_total, const int* when, double s0) {
  k_seq_sum_chain<<<1, 1, 0, ctx->stream>>>(x, n, s0, when, d_total);
  ctx->launches++;
}

}  // namespace glb
