// Observation-path kernels: serpentine Floyd-Steinberg sample extraction
// (observation.cpp:11-71), the likelihood-field scan model over sampled
// states (observation.cpp:73-111) and the sampled multiplicative update
// (observation.cpp:113-170). --fmad=false; reference operand order.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "gl_internal.hpp"

namespace glb {

namespace {

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

// In-row carry coefficient (7/16)/wsum of pixel i in row j (direction dir);
// 0 when its (dir,0) target is outside the grid or wsum == 0.
__device__ __forceinline__ double fs_carry_coef(int i, int j, int w, int h, int dir) {
  if (!(i + dir >= 0 && i + dir < w)) return 0.0;
  const double ws = fs_wsum(i, j, w, h, dir);
  if (ws == 1.0) return 7.0 / 16.0;  // interior rows: x / 1 == x, no division
  return ws > 0.0 ? (7.0 / 16.0) / ws : 0.0;
}

// Pipelined serpentine Floyd-Steinberg (observation.cpp:11-71), bit-identical
// to the reference's serial sweep:
//   warp 0, lane 0: the sequential total (observation.cpp:16-17), then the
//     in-row carry chain v = pre + carry; carry = e * (7/16)/wsum, run
//     speculatively in groups that assume no emission (fs_spec_groups; the
//     0.5 threshold on a support cell fires ~once per two rows) and replay a
//     group exactly when one does: ~1 DADD + 1 DMUL latency per pixel;
//   warp 1: pre-accumulates row j+1 (bm*scale plus row j's diffused errors in
//     the reference's arrival order: upstream, centre, downstream source)
//     while the chain is still in row j, a few pixels behind it, via a
//     shared-memory progress counter.
// Serpentine order has no inter-row wavefront (row j+1 starts where row j
// ended), so the W*H chain of dependent FP64 ops is inherent.
// acquire/release fence at CTA scope (MEMBAR.ALL.CTA; __threadfence_block
// is sequentially consistent)
__device__ __forceinline__ void fence_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }
// Speculative in-row sweep of k_dither_pipe, G pixels per group, scan-order
// rows at index q + 1: assumes "no emission in this group", so the chain is a
// pure DADD->DMUL dependency (bit-identical to the exact sweep up to the
// first emission); the threshold tests are reduced once per group:
// v >= 0.5 <=> the high word of v, as a signed int, is >= 0x3FE00000
// (negative v has the sign bit set), so an integer max over the
// support-masked high words keeps predicates off the chain. Returns true,
// with q/carry at the start of the offending group, when a group emits (its
// err values are then rewritten by the exact replay); false at the row tail.
// kConstC: the carry coefficient is 7/16 (every row but the last) and is
// folded into the multiply as an immediate.
template <int G, bool kConstC>
__device__ __forceinline__ bool fs_spec_groups(const double* pre, double* err,
                                               const unsigned int* sup, int& q,
                                               double& carry, double c_reg, int w,
                                               volatile int* /*progress: see the loop end*/) {
  const double c = kConstC ? 7.0 / 16.0 : c_reg;
  for (; q + G <= w - 1; q += G) {
    double2 pv[G / 2];
    const double2* p2 = reinterpret_cast<const double2*>(pre + q + 1);
#pragma unroll
    for (int k = 0; k < G / 2; ++k) pv[k] = p2[k];
    double cr = carry;
    int mx = 0;
    double2* e2 = reinterpret_cast<double2*>(err + q + 1);
    constexpr int GH = G < 32 ? G : 32;
#pragma unroll
    for (int hf = 0; hf < G / GH; ++hf) {
      const int qh = q + 32 * hf;
      const unsigned long long sw =
          static_cast<unsigned long long>(sup[qh >> 5]) |
          (static_cast<unsigned long long>(sup[(qh >> 5) + 1]) << 32);
      const int sh = qh & 31;
#pragma unroll
      for (int k = 0; k < GH; k += 2) {
        const double2 in = pv[(32 * hf + k) / 2];
        const double v0 = in.x + cr;
        cr = v0 * c;
        const double v1 = in.y + cr;
        cr = v1 * c;
        e2[(32 * hf + k) / 2] = make_double2(v0, v1);
        mx = max(mx, __double2hiint(v0) & -static_cast<int>((sw >> (sh + k)) & 1ull));
        mx = max(mx, __double2hiint(v1) & -static_cast<int>((sw >> (sh + k + 1)) & 1ull));
      }
    }
    if (__builtin_expect(mx >= 0x3FE00000, 0)) return true;
    carry = cr;
    // no progress publication: these are the row's tail groups, whose
    // positions only the helper's last chunk reads, after the row end's
    // publication (a CTA fence per tail group cost ~300 cycles per row)
  }
  return false;
}

// Software-pipelined form of the 32-pixel speculative groups (the row's main
// body). Measured on one thread (tools/probe_fs_chain3.cu): the bare
// DADD->DMUL chain costs 17.2 cycles/pixel, but any instruction that
// consumes a value the chain JUST produced (a store of it, an integer max of
// its high word) blocks the in-order issue behind the FP64->store/INT
// forwarding latency (29.5 cycles/pixel with a store per pixel pair). So
// group g's screen (max of its high words) and stores are issued during
// group g+1's chain, from the other register buffer, and group g is
// verified one group late: on an emission in g, g+1's values are dropped
// and the caller replays g exactly. Progress (the shared counter + CTA fence
// of fs_spec_groups) is published every GL_FS_PUBN verified groups.
// Measured (GL_DEBUG_DITHER, 1024^2): sweep 28.3 M cycles with
// fs_spec_groups<32> -> 25.2 M (publishing every 2 groups; 25.9 M every
// group, 26.2 M every 4).
// Returns true with (q, carry) at the start of the group to replay; false at
// the row tail (q then points past the last verified group).
#ifndef GL_FS_PUBN
#define GL_FS_PUBN 2
#endif
template <bool kConstC>
__device__ __forceinline__ bool fs_spec_pipe(const double* __restrict__ pre, double* __restrict__ err,
                                             const unsigned int* __restrict__ sup, int& q,
                                             double& carry, double c_reg, int w,
                                             volatile int* progress) {
  constexpr int G = 32;
  const double c = kConstC ? 7.0 / 16.0 : c_reg;
  if (q + G > w - 1) return false;
  double2 pb[2][G / 2];
  double2 head = *reinterpret_cast<const double2*>(pre + q + 1);
  int q_p = 0;
  double carry_p = 0.0;
  int npub = 0;
  // masked emission test of the pending group (rare: the unmasked screen
  // fires whenever error piles up across non-emitting wall cells)
  auto emits = [&](auto Pt) -> bool {
    constexpr int P = decltype(Pt)::value;
    const unsigned long long sw = static_cast<unsigned long long>(sup[q_p >> 5]) |
                                  (static_cast<unsigned long long>(sup[(q_p >> 5) + 1]) << 32);
    const unsigned int swq = static_cast<unsigned int>(sw >> (q_p & 31));
    int ms = 0;
#pragma unroll
    for (int k = 0; k < G / 2; ++k) {
      ms = max(ms, __double2hiint(pb[P][k].x) & -static_cast<int>((swq >> (2 * k)) & 1u));
      ms = max(ms, __double2hiint(pb[P][k].y) & -static_cast<int>((swq >> (2 * k + 1)) & 1u));
    }
    return ms >= 0x3FE00000;
  };
  // 0 = continue, 1 = replay (q, carry set), 2 = tail reached
  auto group = [&](auto Bt, auto Pendt) -> int {
    constexpr int B = decltype(Bt)::value;
    constexpr int P = 1 - B;
    constexpr bool pend = decltype(Pendt)::value;
    const int qn = q + G;
    const bool more = qn + G <= w - 1;
    {
      const double2* p2 = reinterpret_cast<const double2*>(pre + q + 1);
      pb[B][0] = head;
#pragma unroll
      for (int k = 1; k < G / 2; ++k) pb[B][k] = p2[k];
      if (more) head = *reinterpret_cast<const double2*>(pre + qn + 1);
    }
    double2* ep = reinterpret_cast<double2*>(err + q_p + 1);
    double cr = carry;
    int hm = 0;
#pragma unroll
    for (int k = 0; k < G / 2; ++k) {
      const double2 in = pb[B][k];
      const double v0 = in.x + cr;
      cr = v0 * c;
      const double v1 = in.y + cr;
      cr = v1 * c;
      pb[B][k] = make_double2(v0, v1);
      if constexpr (pend) {  // the previous group: long-ready registers, off the chain
        hm = max(hm, max(__double2hiint(pb[P][k].x), __double2hiint(pb[P][k].y)));
        ep[k] = pb[P][k];
      }
    }
    if constexpr (pend) {
      if (__builtin_expect(hm >= 0x3FE00000, 0) && emits(std::integral_constant<int, P>{})) {
        q = q_p;  // replay the pending group; this group's values are dropped
        carry = carry_p;
        return 1;
      }
      // the pending group is final; published every GL_FS_PUBN groups (a
      // CTA fence per group costs more than the helper gains from it)
      if (++npub == GL_FS_PUBN) {
        npub = 0;
        fence_cta();
        *progress = q;
      }
    }
    q_p = q;
    carry_p = carry;
    carry = cr;
    q = qn;
    if (more) return 0;
    // drain: screen and store the last group
    int hl = 0;
    double2* el = reinterpret_cast<double2*>(err + q_p + 1);
#pragma unroll
    for (int k = 0; k < G / 2; ++k) {
      hl = max(hl, max(__double2hiint(pb[B][k].x), __double2hiint(pb[B][k].y)));
      el[k] = pb[B][k];
    }
    if (__builtin_expect(hl >= 0x3FE00000, 0) && emits(std::integral_constant<int, B>{})) {
      q = q_p;
      carry = carry_p;
      return 1;
    }
    fence_cta();
    *progress = q;
    return 2;
  };
  // the first group has nothing pending; afterwards every group verifies
  // and stores its predecessor
  int r = group(std::integral_constant<int, 0>{}, std::false_type{});
  if (r) return r == 1;
  for (;;) {
    r = group(std::integral_constant<int, 1>{}, std::true_type{});
    if (r) return r == 1;
    r = group(std::integral_constant<int, 0>{}, std::true_type{});
    if (r) return r == 1;
  }
}

__device__ long long g_dither_clk[12];  // phase timestamps (debug read-out)

__global__ void __launch_bounds__(64) k_dither_pipe(
    const double* __restrict__ bm, int w, int h, int budget,
    int* __restrict__ cells, int cap, int* __restrict__ n_out,
    double* __restrict__ mass_out, const int* __restrict__ sum_invalid, const int* __restrict__ seg_done) {
  extern __shared__ double sh2[];
  if (seg_done != nullptr && *seg_done) return;  // k_dither_seg swept this plane
  // rows of RS doubles (scan order at index q + 1; RS even keeps 16-byte
  // alignment)
  const int RS = (w + 3) & ~1;
  double* pre0 = sh2;            // pre-accumulated work of the even rows
  double* pre1 = sh2 + RS;       // odd rows
  double* err = sh2 + 2 * RS;    // errors of the row being swept
  double* nrow = sh2 + 3 * RS;   // w: row j+1 of bm, staged by the helper
  // bm > 0 per pixel as bits in the row's scan order (32 pixels per word)
  unsigned int* sup0 = reinterpret_cast<unsigned int*>(sh2 + 3 * RS + w);
  unsigned int* sup1 = sup0 + (w + 31) / 32 + 1;
  double* ring = sh2;            // phase A: 3 rows of bm staged for the total
  __shared__ volatile int progress;   // pixels of the current row swept
  __shared__ volatile int pre_ready;  // rows whose pre is complete
  __shared__ volatile int filled, consumed;
  __shared__ double s_scale;
  __shared__ int s_stop;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int words = (w + 31) / 32;

  if (tid == 0) {
    progress = 0;
    pre_ready = 0;
    filled = 0;
    consumed = 0;
    g_dither_clk[0] = clock64();
  }
  __syncthreads();
  // ---- phase A: total = sequential sum in row-major order (:16-17) -------
  // The helper warp stages each row's NONZERO values, in order, for the
  // summing thread: total starts at +0.0 and a sum of finite/inf/NaN terms
  // from +0.0 is never -0.0, so adding a +-0.0 term never changes it
  // (x + 0.0 == x for every x except -0.0): skipping zeros (occupied cells)
  // shortens the dependent DADD chain without changing a bit.
  __shared__ int ring_cnt[3];
  // k_seq_sum already produced the bit-exact total into *mass_out unless
  // the plane held negative / non-finite values
  const bool have_total = sum_invalid != nullptr && *sum_invalid == 0;
  if (have_total) {
    if (tid == 0) {
      const double total = *mass_out;
      s_stop = !(total > 0.0);
      s_scale = budget / total;
      g_dither_clk[1] = clock64() - g_dither_clk[0];
    }
  } else if (warp == 1) {
    for (int r = 0; r < h; ++r) {
      while (r - consumed >= 3) {
      }
      double* dst = ring + static_cast<size_t>(r % 3) * w;
      const double* src = bm + static_cast<size_t>(r) * w;
      int n = 0;
      for (int t0 = 0; t0 < w; t0 += 8 * 32) {
        double v[8];  // 8 loads in flight per lane, then the in-order compaction
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int t = t0 + 32 * k + lane;
          v[k] = t < w ? src[t] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const unsigned int nz = __ballot_sync(0xffffffffu, v[k] != 0.0);  // NaN kept, +-0 dropped
          if (v[k] != 0.0) dst[n + __popc(nz & ((1u << lane) - 1u))] = v[k];
          n += __popc(nz);
        }
      }
      if (lane == 0) ring_cnt[r % 3] = n;
      __syncwarp();
      fence_cta();
      if (lane == 0) filled = r + 1;
      __syncwarp();
    }
  } else if (tid == 0) {
    double total = 0.0;
    for (int r = 0; r < h; ++r) {
      while (filled <= r) {
      }
      fence_cta();
      const double* row = ring + static_cast<size_t>(r % 3) * w;
      const int n = ring_cnt[r % 3];
      int t = 0;
      for (; t + 16 <= n; t += 16) {
        double x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = row[t + k];
#pragma unroll
        for (int k = 0; k < 16; ++k) total += x[k];
      }
      for (; t < n; ++t) total += row[t];
      fence_cta();
      consumed = r + 1;
    }
    *mass_out = total;
    s_stop = !(total > 0.0);
    s_scale = budget / total;
    g_dither_clk[1] = clock64() - g_dither_clk[0];
  }
  __syncthreads();
  if (s_stop) {
    if (tid == 0) *n_out = 0;
    return;
  }
  const double scale = s_scale;
  // ---- phase B: row 0's work; the ring is free again ----------------------
  // pre/err rows are kept in the row's SCAN order at index q + 1, so the
  // chain's 32-pixel groups (q = 1 + 32m) are 16-byte aligned and addressed
  // with immediate offsets from one base register
  for (int t = tid; t < w; t += blockDim.x) pre0[t + 1] = bm[t] * scale;
  for (int wd = tid; wd <= words; wd += blockDim.x) {
    unsigned int bits = 0;
    for (int k = 0; k < 32; ++k) {
      const int pos = wd * 32 + k;  // row 0 sweeps left to right
      if (pos < w && bm[pos] > 0.0) bits |= 1u << k;
    }
    sup0[wd] = bits;
  }
  if (tid == 0) pre_ready = 1;
  __syncthreads();

  if (warp == 0) {
    if (lane != 0) return;
    int count = 0;
    long long waited = 0, waited_end = 0;
    const long long t_b = clock64();
    auto record = [&](int i, int j) {
      if (count < cap) {
        cells[2 * count] = i;
        cells[2 * count + 1] = j;
      }
      ++count;
    };
    for (int j = 0; j < h; ++j) {
      const int dir = (j % 2 == 0) ? 1 : -1;
      const double* pre = (j & 1) ? pre1 : pre0;
      const unsigned int* sup = (j & 1) ? sup1 : sup0;
      const long long tw = clock64();
      while (pre_ready < j + 1) {
      }
      waited += clock64() - tw;
      fence_cta();
      const int start = dir == 1 ? 0 : w - 1;
      const double c_first = fs_carry_coef(start, j, w, h, dir);
      const double c_mid = (w > 2) ? fs_carry_coef(start + dir, j, w, h, dir) : 0.0;
      // q = 0: no in-row carry flows into the first pixel
      double carry;
      {
        const double v = pre[1];
        double e = v;
        if (v >= 0.5 && (sup[0] & 1u)) {
          e = v - 1.0;
          record(start, j);
        }
        err[1] = e;
        carry = e * c_first;
      }
      // exact per-pixel step for pixels 1 .. w-2 (carry coefficient c_mid)
      auto body = [&](int q, bool s) {
        const double v = pre[q + 1] + carry;
        double next;
        asm("mul.rn.f64 %0, %1, %2;" : "=d"(next) : "d"(v), "d"(c_mid));
        double e = v;
        if (__builtin_expect(v >= 0.5 && s, 0)) {
          e = v - 1.0;
          next = e * c_mid;
          record(start + q * dir, j);
        }
        err[q + 1] = e;
        carry = next;
      };
      int q = 1;
      // speculative groups (fs_spec_groups) of 32 pixels, then one each of
      // 16, 8, 4, 2 for the row tail; a group with an emission is replayed
      // exactly here, then speculation resumes
      auto sweep = [&](auto gsize) {
        constexpr int G = decltype(gsize)::value;
        auto spec = [&]() {
          if constexpr (G == 32) {
            return c_mid == 7.0 / 16.0 ? fs_spec_pipe<true>(pre, err, sup, q, carry, c_mid, w, &progress)
                                       : fs_spec_pipe<false>(pre, err, sup, q, carry, c_mid, w, &progress);
          } else {
            return c_mid == 7.0 / 16.0 ? fs_spec_groups<G, true>(pre, err, sup, q, carry, c_mid, w, &progress)
                                       : fs_spec_groups<G, false>(pre, err, sup, q, carry, c_mid, w, &progress);
          }
        };
        while (spec()) {
#pragma unroll 1
          for (int k = 0; k < G; ++k) {
            const int qk = q + k;
            body(qk, (sup[qk >> 5] >> (qk & 31)) & 1u);
          }
          q += G;
          fence_cta();
          progress = q;
        }
      };
      sweep(std::integral_constant<int, 32>{});
      sweep(std::integral_constant<int, 16>{});
      sweep(std::integral_constant<int, 8>{});
      sweep(std::integral_constant<int, 4>{});
      sweep(std::integral_constant<int, 2>{});
      for (; q < w - 1; ++q) body(q, (sup[q >> 5] >> (q & 31)) & 1u);
      if (w > 1) {  // last pixel: no in-row target
        const double v = pre[w] + carry;
        double e = v;
        if (v >= 0.5 && ((sup[(w - 1) >> 5] >> ((w - 1) & 31)) & 1u)) {
          e = v - 1.0;
          record(start + (w - 1) * dir, j);
        }
        err[w] = e;
      }
      fence_cta();
      progress = w;
      // the helper resets progress once it has consumed row j
      const long long te = clock64();
      while (progress != 0 && j + 1 < h) {
      }
      waited_end += clock64() - te;
    }
    *n_out = count;
    g_dither_clk[2] = clock64() - t_b;
    g_dither_clk[3] = waited;
    g_dither_clk[0] = waited_end;
    return;
  }

  // warp 1: pre-accumulate row j+1 from row j's errors, behind the chain
  for (int j = 0; j + 1 < h; ++j) {
    const int pd = (j % 2 == 0) ? 1 : -1;  // row j's direction
    const int jn = j + 1;
    double* pre = (jn & 1) ? pre1 : pre0;
    unsigned int* sup = (jn & 1) ? sup1 : sup0;
    const int dn = -pd;                    // row j+1's direction
    const int start_n = dn == 1 ? 0 : w - 1;
    const double* brow = bm + static_cast<size_t>(jn) * w;
    for (int t = lane; t < w; t += 32) nrow[t] = brow[t];
    __syncwarp();
    // support bits of row j+1 in ITS scan order (one ballot per 32 pixels)
    for (int wd = 0; wd <= words; ++wd) {  // + one zero word of padding
      const int qn = wd * 32 + lane;
      const bool s = qn < w && nrow[start_n + qn * dn] > 0.0;
      const unsigned int bits = __ballot_sync(0xffffffffu, s);
      if (lane == 0) sup[wd] = bits;
    }
    // diffusion weights (t.w / wsum) of row j's sources: interior sources
    // have wsum == 1 (the quotients are exact); the two scan ends differ.
    // Their quotients are formed here, before the chain reaches the row: an
    // FP64 division in the row's last chunk sat on the chain's row-end
    // critical path (~880 cycles per row for that chunk, measured).
    const double w_lo = fs_wsum(0, j, w, h, pd), w_hi = fs_wsum(w - 1, j, w, h, pd);
    const double e1[2] = {(1.0 / 16.0) / w_lo, (1.0 / 16.0) / w_hi};
    const double e5[2] = {(5.0 / 16.0) / w_lo, (5.0 / 16.0) / w_hi};
    const double e3[2] = {(3.0 / 16.0) / w_lo, (3.0 / 16.0) / w_hi};
    auto coef = [&](int s, double wt, const double* edge) {
      return s == 0 ? edge[0] : (s == w - 1 ? edge[1] : wt);
    };
    for (int base = 0; base < w; base += 32) {
      const int pos = base + lane;  // scan position in row j
      const int need = min(base + 33, w);  // sources up to pos+1 swept
      while (progress < need) {
      }
      fence_cta();
      if (pos < w) {
        // target pixel t of row j+1 receives, in the reference's arrival
        // order, from row j's pixels t-pd (1/16), t (5/16), t+pd (3/16),
        // i.e. scan positions pos-1, pos, pos+1
        const int t = pd == 1 ? pos : w - 1 - pos;
        double v = nrow[t] * scale;
        if (pos >= 1) v += err[pos] * coef(t - pd, 1.0 / 16.0, e1);
        v += err[pos + 1] * coef(t, 5.0 / 16.0, e5);
        if (pos + 1 < w) v += err[pos + 2] * coef(t + pd, 3.0 / 16.0, e3);
        pre[w - pos] = v;  // row j+1 scans the other way: position w-1-pos
      }
    }
    __syncwarp();
    fence_cta();
    if (lane == 0) {
      progress = 0;
      fence_cta();
      pre_ready = jn + 1;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Segment-parallel serpentine Floyd-Steinberg (round 2). Inside a row the
// reference's carry chain e_q -> v_{q+1} = pre + e_q * (7/16) CONTRACTS: two
// chains started from different carries meet bitwise after ~45-60 pixels
// (the difference shrinks by 7/16 per pixel until one rounding merges them,
// and from then on the same state gives the same future — emissions
// included). So every row is cut into segments, one per lane of the chain
// warps (up to 64). Segment 0 runs [0, F) exactly from the row's first
// pixel; segment l >= 1 runs [s_l, s_l + S) but starts kSegWU pixels early
// with a guessed carry 0 (a warm-up over the previous segment's tail that
// records nothing). Segments are S pixels apart with S odd, so the lanes'
// shared-memory accesses fall in distinct banks. Each lane works in
// 16-pixel groups: values loaded a group ahead, the chain run assuming
// no emission (one DADD and one DMUL per pixel), the group replayed exactly
// by the lanes that need it when any lane's group holds a supported v >= 0.5.
// Emissions are bits of a per-row mask. Then all segments are verified at
// once: segment l is exact iff its warm-up's last error equals, bit for bit,
// segment l-1's error before it; a failing segment reruns from that true
// carry until its values meet its own stored chain (taking the rerun's errors
// and emission bits up to the meeting pixel); a rerun that reaches its
// segment end unmet changed what its successor was checked against, so the
// successor reruns in another round. Every value and every emission is the
// reference's. The row's cells go out in scan order by a warp scan over the
// mask words. The last row (no row below: carry coefficient 1, no
// contraction) and narrow rows run the exact sequential chain on one thread.
// The other two warps stage the next row of the belief map (cp.async) while
// the chains run, build its pre-accumulation while the row is verified, and
// recompute the positions next to errors a rerun rewrote.
#ifndef GL_FS_SEG
#define GL_FS_SEG 1  // the segment-parallel sweep (0: the pipelined chain only)
#endif
constexpr int kSegT = 128;     // threads (4 warps: kSegW chain warps, the rest stage the next row)
constexpr int kSegWU = 64;     // warm-up pixels of segments 1.. (the many-segment layout)
#ifndef GL_SEG_FEW_ROWS
#define GL_SEG_FEW_ROWS 8  // rows the fallback layout holds after 2+ reruns (1: rows alternate)
#endif
constexpr int kSegFewRows = GL_SEG_FEW_ROWS;
#ifndef GL_SEG_FEW_AT
#define GL_SEG_FEW_AT 2  // first-round reruns that switch to the fallback layout
#endif
constexpr int kSegFewAt = GL_SEG_FEW_AT;
#ifndef GL_SEG_FEW_LANES
#define GL_SEG_FEW_LANES 32  // segments of the fallback layout
#endif
#ifndef GL_SEG_WU_FEW
#define GL_SEG_WU_FEW 64
#endif
// the 32-segment layout's warm-up (rows after verification reruns:
// concentrated beliefs). Longer warm-ups there (80, 96) measured within noise
// of 64 (profiles/r02_sweeps.md).
constexpr int kSegWUFew = GL_SEG_WU_FEW;
static_assert(kSegWU % 16 == 0 && kSegWUFew % 16 == 0 && kSegWUFew >= kSegWU,
              "warm-ups are whole 16-pixel groups");
#ifndef GL_SEG_CHAIN_WARPS
#define GL_SEG_CHAIN_WARPS 2
#endif
constexpr int kSegW = GL_SEG_CHAIN_WARPS;  // warps running segment chains (the others stage the next row)
constexpr int kSegLanes = 32 * kSegW;      // segments per row at most
static_assert(kSegW >= 1 && kSegW <= 2, "1 or 2 chain warps (4-warp CTA)");

// a chain lane's segment under one layout (fixed for the kernel)
struct SegLane {
  bool act;           // the lane has a segment
  int qs, qe, q0;     // segment start / end, first pixel it runs
  int n_grp;          // its warp's group count (lanes past their segment: no pixels)
};

struct SegLayout {
  int P, F, S;  // lanes in use, lane 0's length, segment stride (odd)
  int wu;       // warm-up pixels of segments 1..
  __host__ __device__ int start(int l) const { return l == 0 ? 0 : min(w_, F + (l - 1) * S); }
  int w_;
};

__host__ __device__ inline SegLayout seg_layout(int w, int lanes, int wu = kSegWU) {
  SegLayout L{};
  L.w_ = w;
  L.wu = wu;
  if (w < 4 * kSegWU) {
    L.P = 1;
    L.F = w;
    L.S = w;
    return L;
  }
  int S = (w - wu + lanes - 1) / lanes;  // lane 0 takes S + wu (every lane runs ~S + wu pixels)
  S |= 1;
  L.S = S;
  L.F = min(w, S + wu);
  L.P = 1 + (w - L.F + S - 1) / S;
  return L;
}

// support bits of scan positions [base, base + valid) (0 <= valid <= 16), bit k = base + k
__device__ __forceinline__ unsigned int seg_sup_bits(const unsigned int* sup, int base, int valid) {
  // branch-free: lanes without pixels read word 0 under an empty mask
  const int b = valid > 0 ? base : 0;
  const unsigned long long sw2 = static_cast<unsigned long long>(sup[b >> 5]) |
                                 (static_cast<unsigned long long>(sup[(b >> 5) + 1]) << 32);
  return static_cast<unsigned int>(sw2 >> (b & 31)) & (valid >= 16 ? 0xffffu : ((1u << valid) - 1u));
}

__global__ void __launch_bounds__(kSegT) k_dither_seg(const double* __restrict__ bm, int w, int h, int budget,
                                                      int* __restrict__ cells, int cap, int* __restrict__ n_out,
                                                      const double* __restrict__ total_in,
                                                      const int* __restrict__ sum_invalid, int* __restrict__ done) {
  extern __shared__ double segsh[];
  const int WR = ((w + 1) & ~1) + 16, SW = (w + 31) / 32 + 2;  // +16: a lane's last group reads past w
  // buf[j & 1]: row j's pre-accumulated work (scan order); buf[(j + 1) & 1]:
  // row j + 1's, built by the staging warps while row j is verified
  double* buf0 = segsh;
  double* err = segsh + 2 * WR;  // row j's errors, scan order
  double* raw = segsh + 3 * WR;  // row j + 1 of bm in its scan order (cp.async while row j sweeps)
  unsigned int* sup0 = reinterpret_cast<unsigned int*>(segsh + 4 * WR);  // [2][SW] support bits, scan order
  unsigned int* ebits = sup0 + 2 * SW;  // [SW] row j's emission bits, scan order
  __shared__ int s_count;
  __shared__ int s_chg_hi[kSegLanes];  // row j: the last error a lane's verification reruns rewrote (-1: none)
  __shared__ int s_changed[kSegLanes];  // a verification round: the lane's rerun changed its segment end
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (*sum_invalid) {  // negative / non-finite plane: k_dither_pipe's sequential total takes it
    if (tid == 0) *done = 0;
    return;
  }
  const double total = *total_in;
  if (!(total > 0.0)) {
    if (tid == 0) {
      *n_out = 0;
      *done = 1;
    }
    return;
  }
  const double scale = budget / total;
  if (tid == 0) s_count = 0;
  // Two layouts: 32 * kSegW segments (shorter warm-up share per row) and
  // 32 (longer segments). After a row that needed verification reruns on 2+
  // segments (a concentrated belief: steep tails converge slowly, and short
  // segments turn one slow meeting into rounds) the next kSegFewRows rows
  // take the 32-segment layout; the extra chain warp then has no segments and
  // only keeps the barriers.
  const SegLayout L_many = seg_layout(w, kSegLanes), L_few = seg_layout(w, GL_SEG_FEW_LANES, kSegWUFew);
  __shared__ int s_many[2];  // row parity: this row takes L_many
  __shared__ int s_few_left;  // rows the fallback layout still holds (sticky: rows alternate otherwise)
  // per-direction constants of every row but the last (fs_wsum with a row
  // below; [0]: dir +1, [1]: dir -1): carry coefficients and the diffusion
  // quotients of the row-end sources. Computed once into shared memory (in
  // registers the compiler re-derives the divisions inside the row loop).
  __shared__ double s_k[2][8];  // cf, cm, e1 lo/hi, e5 lo/hi, e3 lo/hi
  if (tid < 2) {
    const int dir = tid == 0 ? 1 : -1, st = tid == 0 ? 0 : w - 1;
    const double w_lo = fs_wsum(0, 0, w, 2, dir), w_hi = fs_wsum(w - 1, 0, w, 2, dir);
    s_k[tid][0] = fs_carry_coef(st, 0, w, 2, dir);
    s_k[tid][1] = (w > 2) ? fs_carry_coef(st + dir, 0, w, 2, dir) : 0.0;
    s_k[tid][2] = (1.0 / 16.0) / w_lo;
    s_k[tid][3] = (1.0 / 16.0) / w_hi;
    s_k[tid][4] = (5.0 / 16.0) / w_lo;
    s_k[tid][5] = (5.0 / 16.0) / w_hi;
    s_k[tid][6] = (3.0 / 16.0) / w_lo;
    s_k[tid][7] = (3.0 / 16.0) / w_hi;
  }

  // row 0: pre = work, no error inflow (observation.cpp:23-25)
  for (int pos = tid; pos < w; pos += kSegT) buf0[pos] = bm[pos] * scale;  // dir = +1
  for (int wd = warp; wd <= w / 32; wd += kSegT / 32) {
    const int q = wd * 32 + lane;
    const unsigned int bits = __ballot_sync(0xffffffffu, q < w && bm[q] > 0.0);
    if (lane == 0) sup0[wd] = bits;
  }
  if (tid == 0) {
    sup0[w / 32 + 1] = 0u;
    sup0[SW + w / 32 + 1] = 0u;
  }
  for (int i = tid; i < SW; i += kSegT) ebits[i] = 0u;
  if (tid == 0) {
    s_many[0] = 1;
    s_few_left = 0;
  }
  // each chain lane's segment under both layouts, once: segment 0 takes the
  // row's first pixel itself (no carry in, its own carry coefficient) and its
  // groups start at pixel 1, so no group needs a first-pixel case; the
  // others start kSegWU pixels early (F > kSegWU: inside the row) from the
  // guessed carry 0
  SegLane lane_many{}, lane_few{};
  if (warp < kSegW) {
    auto lane_of = [&](const SegLayout& Ly) {
      SegLane r;
      r.act = tid < Ly.P;
      r.qs = Ly.start(tid);
      r.qe = Ly.start(tid + 1);
      r.q0 = tid == 0 ? 1 : r.qs - Ly.wu;
      r.n_grp = __reduce_max_sync(0xffffffffu, r.act ? (r.qe - r.q0 + 15) / 16 : 0);
      return r;
    };
    lane_many = lane_of(L_many);
    lane_few = lane_of(L_few);
  }
  __syncthreads();
#ifdef GL_EXPERIMENT_ENV
  long long tk_spec = 0, tk_ver = 0, tk_pre = 0, tk_b1 = 0, tk_stage = 0, tk_all = clock64(), tk0 = 0;
  long long tk_g0 = 0, tk_g1 = 0, tk_nrep = 0, n_ovf = 0, n_fix = 0, n_fixpx = 0, n_exact = 0;
  (void)n_ovf;
#define SEG_TICK(acc) do { if (tid == 0) { const long long t_ = clock64(); acc += t_ - tk0; tk0 = t_; } } while (0)
#else
#define SEG_TICK(acc) do { } while (0)
#endif

  for (int j = 0; j < h; ++j) {
#ifdef GL_EXPERIMENT_ENV
    if (tid == 0 || tid == 32) tk0 = clock64();
#endif
    const int dir = (j % 2 == 0) ? 1 : -1;
    const int d = j % 2;
    const int start = dir == 1 ? 0 : w - 1;
    const bool last = j == h - 1;
    double* pre = buf0 + d * WR;            // row j's pre-accumulated work
    double* nbuf = buf0 + (d ^ 1) * WR;     // row j + 1's pre (built by the staging warps during row j)
    const bool nxt = j + 1 < h;
    const SegLayout L = s_many[d] ? L_many : L_few;
    const unsigned int* sup = sup0 + d * SW;
    unsigned int* nsup = sup0 + (d ^ 1) * SW;
    const double c_first = last ? fs_carry_coef(start, j, w, h, dir) : s_k[d][0];
    const double c_mid = last ? ((w > 2) ? fs_carry_coef(start + dir, j, w, h, dir) : 0.0) : s_k[d][1];
    auto supp = [&](int q) { return (sup[q >> 5] >> (q & 31)) & 1u; };
    auto emit_out = [&](int q) {  // lane 0 only, in scan order
      const int c = s_count;
      if (c < cap) {
        cells[2 * c] = start + q * dir;
        cells[2 * c + 1] = j;
      }
      s_count = c + 1;
    };
    // the reference's exact sweep of scan positions [0, w) (lane 0)
    auto exact_row = [&]() {
      double carry = 0.0;
      for (int q = 0; q < w; ++q) {
        const double v = q == 0 ? pre[0] : pre[q] + carry;
        double e = v;
        if (v >= 0.5 && supp(q)) {
          e = v - 1.0;
          emit_out(q);
        }
        err[q] = e;
        carry = e * (q == 0 ? c_first : c_mid);
      }
    };
    if (warp < kSegW) {
      const int sl = tid;  // this thread's segment
      if (last || L.P == 1) {
#ifdef GL_EXPERIMENT_ENV
        ++n_exact;
#endif
        if (tid == 0) {
          exact_row();
          s_many[d ^ 1] = 1;
        }
        s_chg_hi[sl] = -1;
        asm volatile("bar.sync 5, %0;" ::"r"(kSegLanes) : "memory");
        if (nxt) {  // the errors are final: the staging warps take the next row
          asm volatile("bar.arrive 3, %0;" ::"r"(kSegT) : "memory");
          asm volatile("bar.arrive 4, %0;" ::"r"(kSegT) : "memory");
        }
      } else {
        const SegLane& SLn = s_many[d] ? lane_many : lane_few;
        const bool act = SLn.act;
        const int qs = SLn.qs, qe = SLn.qe, q0 = SLn.q0;
        double carry = 0.0;
        double wu = 0.0;
        if (sl == 0) {
          const double v0 = pre[0];
          const bool em0 = v0 >= 0.5 && (sup[0] & 1u);
          const double e0 = em0 ? v0 - 1.0 : v0;
          err[0] = e0;
          if (em0) atomicOr(&ebits[0], 1u);
          carry = e0 * c_first;
        }
        const int n_grp = SLn.n_grp;
        // One group: the chain on values already in registers, then the NEXT
        // group's loads issued before the replay vote (the vote and its
        // branch would otherwise hold them back), double-buffered by hand.
        auto group = [&](const double (&p)[16], double (&pn)[16], int gi) {
#ifdef GL_EXPERIMENT_ENV
          long long tg0 = clock64();
#endif
          const int base = q0 + 16 * gi;
          const int valid = act ? max(0, min(16, qe - base)) : 0;
          const unsigned int sb = seg_sup_bits(sup, base, valid);
          const double c0 = carry;
          double c = c0, v[16];
          unsigned int big = 0;
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const double vk = p[k] + c;
            v[k] = vk;
            asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(vk), "d"(c_mid));
            big |= __double2hiint(vk) >= 0x3FE00000 ? (1u << k) : 0u;
          }
          {
            const int nbase = base + 16;
            const int nvalid = act ? max(0, min(16, qe - nbase)) : 0;
            const double* pb = pre + (nvalid > 0 ? nbase : 0);
#pragma unroll
            for (int k = 0; k < 16; ++k) pn[k] = pb[k];  // past valid: padding / other lanes' values, masked
          }
          unsigned int emask = 0u;
          const bool need = (big & sb) != 0u;
          if (__any_sync(0xffffffffu, need)) {
            if (need) {  // the exact sweep of this group
              c = c0;
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const double vk = p[k] + c;
                const bool em = vk >= 0.5 && ((sb >> k) & 1u);
                const double e = em ? vk - 1.0 : vk;
                emask |= static_cast<unsigned int>(em) << k;
                v[k] = e;
                asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(e), "d"(c_mid));
              }
            }
          }
          carry = c;
          // own-segment errors and emission bits, the warm-up's last error
          // (groups never straddle a segment start: kSegWU is a multiple of 16;
          // segment 0's groups start at pixel 1, inside its segment)
          const int own = base - qs;  // < 0: a warm-up group
          double* eb = err + (valid > 0 ? base : 0);
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            if (own >= 0 && k < valid) eb[k] = v[k];
          }
          if (own >= 0 && emask) {  // neighbouring lanes share boundary words
            const int sh = base & 31;
            atomicOr(&ebits[base >> 5], emask << sh);
            if (sh > 16) atomicOr(&ebits[(base >> 5) + 1], emask >> (32 - sh));
          }
          if (own == -16) wu = v[15];
#ifdef GL_EXPERIMENT_ENV
          if (tid == 0) { const long long t_ = clock64(); tk_g1 += t_ - tg0; }
#endif
        };
        double pa[16], pb2[16];
        {
          const int valid0 = act ? max(0, min(16, qe - q0)) : 0;
          const double* pb = pre + (valid0 > 0 ? q0 : 0);
#pragma unroll
          for (int k = 0; k < 16; ++k) pa[k] = pb[k];
        }
        SEG_TICK(tk_b1);  // row setup
        for (int gi = 0; gi < n_grp; gi += 2) {
          group(pa, pb2, gi);
          if (gi + 1 < n_grp) group(pb2, pa, gi + 1);
        }
        SEG_TICK(tk_g0);  // the groups
        asm volatile("bar.sync 5, %0;" ::"r"(kSegLanes) : "memory");  // every chain's errors stored
        // the staging warps start the next row's pass on these errors now;
        // what the verification below rewrites they recompute after barrier 4
        if (nxt) asm volatile("bar.arrive 3, %0;" ::"r"(kSegT) : "memory");
        SEG_TICK(tk_spec);
        // ---- verification, all lanes at once. Lane l >= 1 is exact if its
        // warm-up's last error equals lane l-1's error before its segment;
        // else it reruns from that true carry until its value meets its own
        // stored chain (same state, same future) and takes the rerun's errors
        // and emissions up to there. This assumes lane l-1's segment end is
        // final; a lane whose rerun reached its segment end without meeting
        // changed that end, and its successor reruns in another round. ----
        bool todo = act && sl > 0, recheck = true;
        int chg_hi = -1;   // the last error this lane's reruns rewrote
        int n_first = 0;   // segments the first round reruns (chooses the next row's layout)
        for (;;) {
          bool run = false;
          double cr = 0.0;
          if (todo) {
            const double et = err[qs - 1];
            run = !recheck || __double_as_longlong(et) != __double_as_longlong(wu);
            cr = et * c_mid;  // qs - 1 >= kSegWU: an interior pixel
          }
          // how many segments rerun, over all chain warps (usually none: one barrier)
          int any;
          asm volatile("{ .reg .pred q; setp.ne.s32 q, %1, 0; bar.red.popc.u32 %0, 5, %2, q; }"
                       : "=r"(any) : "r"(static_cast<int>(run)), "r"(kSegLanes) : "memory");
          if (recheck) n_first = any;
          if (!any) break;
          bool changed = run;  // cleared when the rerun meets the stored chain
#ifdef GL_EXPERIMENT_ENV
          if (run) ++n_fix;
#endif
          int base = qs;
          double rp[16];  // the rerun group's values, loaded one group ahead
          {
            const double* pb = pre + (run ? base : 0);
#pragma unroll
            for (int k = 0; k < 16; ++k) rp[k] = pb[k];
          }
          while (__any_sync(0xffffffffu, run)) {
            const int valid = run ? max(0, min(16, qe - base)) : 0;
            const unsigned int sb = seg_sup_bits(sup, base, valid);
            double v[16], st[16];
            double c = cr;
            unsigned int big = 0u;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const double vk = rp[k] + c;
              v[k] = vk;
              asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(vk), "d"(c_mid));
              big |= __double2hiint(vk) >= 0x3FE00000 ? (1u << k) : 0u;
            }
            // the stored chain to meet, and the next group's values, before the vote
            {
              const double* eb = err + (valid > 0 ? base : 0);
#pragma unroll
              for (int k = 0; k < 16; ++k) st[k] = eb[k];
            }
            double rn[16];
            {
              const int nv = run ? max(0, min(16, qe - base - 16)) : 0;
              const double* pb = pre + (nv > 0 ? base + 16 : 0);
#pragma unroll
              for (int k = 0; k < 16; ++k) rn[k] = pb[k];
            }
            unsigned int emask = 0u;
            const bool need = (big & sb) != 0u;
            if (__any_sync(0xffffffffu, need)) {
              if (need) {  // the exact sweep of this group
                c = cr;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                  const double vk = rp[k] + c;
                  const bool em = vk >= 0.5 && ((sb >> k) & 1u);
                  const double e = em ? vk - 1.0 : vk;
                  emask |= static_cast<unsigned int>(em) << k;
                  v[k] = e;
                  asm("mul.rn.f64 %0, %1, %2;" : "=d"(c) : "d"(e), "d"(c_mid));
                }
              }
            }
            const double cn = c;
#pragma unroll
            for (int k = 0; k < 16; ++k) rp[k] = rn[k];
            if (valid > 0) {
              // the first pixel where the rerun equals the stored chain: the
              // same state from there on. Its emission is the rerun's (equal
              // errors do not imply equal decisions at that pixel).
              unsigned int meet = 0u;
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                if (k < valid && __double_as_longlong(v[k]) == __double_as_longlong(st[k])) meet |= 1u << k;
              }
              const int m = meet ? __ffs(meet) - 1 : valid - 1;  // last pixel taken from the rerun
#ifdef GL_EXPERIMENT_ENV
              n_fixpx += m + 1;
#endif
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                if (k <= m) err[base + k] = v[k];
              }
              chg_hi = max(chg_hi, base + m);
              const unsigned int keep = m >= 15 ? 0xffffu : ((2u << m) - 1u);
              const int sh = base & 31;
              const unsigned long long ow = static_cast<unsigned long long>(ebits[base >> 5]) |
                                            (static_cast<unsigned long long>(ebits[(base >> 5) + 1]) << 32);
              const unsigned int diff = (static_cast<unsigned int>(ow >> sh) ^ emask) & keep;
              if (diff) {  // only this lane's bits change; neighbours share boundary words
                atomicXor(&ebits[base >> 5], diff << sh);
                if (sh > 16) atomicXor(&ebits[(base >> 5) + 1], diff >> (32 - sh));
              }
              if (meet) {
                changed = false;
                run = false;
              } else {
                cr = cn;
                base += 16;
                if (base >= qe) run = false;  // the segment end changed
              }
            }
          }
          recheck = false;  // later rounds rerun unconditionally
          s_changed[sl] = changed;
          asm volatile("bar.sync 5, %0;" ::"r"(kSegLanes) : "memory");
          todo = act && sl > 0 && s_changed[sl - 1];
        }
        s_chg_hi[sl] = chg_hi;
        // reruns rewrote emission bits across the chain warps: warp 0's scan
        // below needs them (n_first is uniform: a barrier reduction)
        if (n_first > 0) asm volatile("bar.sync 5, %0;" ::"r"(kSegLanes) : "memory");
        if (nxt) asm volatile("bar.arrive 4, %0;" ::"r"(kSegT) : "memory");
        if (warp == 0) {
          if (lane == 0) {
            // 2+ reruns: the fallback layout for the next kSegFewRows rows
            if (n_first >= kSegFewAt) s_few_left = kSegFewRows;
            else if (s_few_left > 0) --s_few_left;
            s_many[d ^ 1] = s_few_left == 0;
          }
        // ---- the row's emissions in scan order: a warp scan over the
        // emission words (cleared for the next row) ----
        const int nw = (w + 31) >> 5;
        int c_base = s_count;
        for (int w0 = 0; w0 < nw; w0 += 32) {
          const int wd = w0 + lane;
          unsigned int bits = wd < nw ? ebits[wd] : 0u;
          if (wd < nw) ebits[wd] = 0u;
          const int cnt = __popc(bits);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          int cc = c_base + incl - cnt;
          while (bits) {
            const int q = wd * 32 + __ffs(bits) - 1;
            bits &= bits - 1;
            if (cc < cap) {
              cells[2 * cc] = start + q * dir;
              cells[2 * cc + 1] = j;
            }
            ++cc;
          }
          c_base += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        if (lane == 0) s_count = c_base;
        }
      }
      SEG_TICK(tk_ver);
    } else if (nxt) {
      // ---- the staging warps while the chain warps sweep row j: row j + 1 of bm into raw
      // in its scan order (all loads in flight at once) and its support
      // bits; once the chains are done, row j + 1's pre-accumulation
      // (overlapping the verification); then the positions next to
      // errors the verification rewrote ----
      const double* brow = bm + static_cast<size_t>(j + 1) * w;
      const bool rev = dir == 1;  // row j + 1 scans right to left
      const int t3 = tid - kSegLanes;  // the staging threads
      constexpr int kT3 = kSegT - kSegLanes;
      for (int t = t3; t < w; t += kT3) {
        const unsigned int dst = static_cast<unsigned int>(__cvta_generic_to_shared(raw + (rev ? w - 1 - t : t)));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(brow + t) : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"r"(kT3) : "memory");
      for (int wd = warp - kSegW; wd <= w / 32; wd += kSegT / 32 - kSegW) {
        const int qn = wd * 32 + lane;
        const unsigned int bits = __ballot_sync(0xffffffffu, qn < w && raw[qn] > 0.0);
        if (lane == 0) nsup[wd] = bits;
      }
#ifdef GL_EXPERIMENT_ENV
      if (tid == 32) tk_stage += clock64() - tk0;
#endif
      // the reference's arrival order for a cell of row j+1: upstream,
      // centre, downstream source of row j. Row ends (scan positions 0, 1,
      // w-2, w-1) miss a source or take a row-end quotient: selects (a
      // missing term is not added: not + 0.0, so signed zeros stay the
      // reference's); branch-free batches of 4 (clamped loads, guarded stores)
      const int pd = dir;
      const double E1l = s_k[d][2], E1h = s_k[d][3], E5l = s_k[d][4], E5h = s_k[d][5], E3l = s_k[d][6],
                   E3h = s_k[d][7];
      auto pre_at = [&](int pos) {  // row j+1's pre at its scan position w-1-pos
        const int t = pd == 1 ? pos : w - 1 - pos;  // column of row j at scan position pos
        const double c1 = (t - pd == 0) ? E1l : (t - pd == w - 1 ? E1h : 1.0 / 16.0);
        const double c5 = (t == 0) ? E5l : (t == w - 1 ? E5h : 5.0 / 16.0);
        const double c3 = (t + pd == 0) ? E3l : (t + pd == w - 1 ? E3h : 3.0 / 16.0);
        double x = raw[w - 1 - pos] * scale;  // row j+1 scans the other way
        const double up = x + err[max(pos - 1, 0)] * c1;
        x = pos >= 1 ? up : x;
        x += err[pos] * c5;
        const double dn = x + err[min(pos + 1, w - 1)] * c3;
        return pos + 1 < w ? dn : x;
      };
      asm volatile("bar.sync 3, %0;" ::"r"(kSegT) : "memory");  // the chains are done
      for (int i0 = t3; i0 < w; i0 += 4 * kT3) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = pre_at(min(i0 + u * kT3, w - 1));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (i0 + u * kT3 < w) nbuf[w - 1 - (i0 + u * kT3)] = v[u];
        }
      }
      asm volatile("bar.sync 4, %0;" ::"r"(kSegT) : "memory");  // verification done: s_chg_hi
      // a rewritten error at position p feeds positions p-1..p+1; segment l
      // rewrote [qs_l, s_chg_hi[l]]. 32 read at once, one ballot per word.
#pragma unroll
      for (int wv = 0; wv < kSegW; ++wv) {
        const int my_hi = s_chg_hi[32 * wv + lane];
        unsigned int chg = __ballot_sync(0xffffffffu, my_hi >= 0);
        while (chg) {
          const int l = __ffs(chg) - 1;
          chg &= chg - 1;
          const int hi = __shfl_sync(0xffffffffu, my_hi, l);
          const int lo = max(L.start(32 * wv + l) - 1, 0), top = min(hi + 1, w - 1);
          for (int p = lo + t3; p <= top; p += kT3) nbuf[w - 1 - p] = pre_at(p);
        }
      }
    }
    __syncthreads();
    SEG_TICK(tk_pre);
  }
#ifdef GL_EXPERIMENT_ENV
  if (tid == 32) g_dither_clk[5] = tk_stage;
  if (warp == 0) {
    for (int o = 16; o > 0; o >>= 1) {
      n_fix += __shfl_down_sync(0xffffffffu, n_fix, o);
      n_fixpx += __shfl_down_sync(0xffffffffu, n_fixpx, o);
    }
  }
#endif
  if (tid == 0) {
    *n_out = s_count;
    *done = 1;
#ifdef GL_EXPERIMENT_ENV
    g_dither_clk[0] = tk_spec;
    g_dither_clk[1] = tk_ver;
    g_dither_clk[2] = tk_pre;
    g_dither_clk[4] = tk_b1;
    g_dither_clk[6] = tk_g0;
    g_dither_clk[7] = tk_g1 + (tk_nrep << 40);
    g_dither_clk[8] = n_ovf;
    g_dither_clk[9] = n_fix;
    g_dither_clk[10] = n_fixpx;
    g_dither_clk[11] = n_exact;
    g_dither_clk[3] = clock64() - tk_all;
#endif
  }
#undef SEG_TICK
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
// Row buffers in shared memory, or (gbuf != null, rows wider than shared
// memory holds: W > ~14.5K cells) in global memory.
__global__ void __launch_bounds__(32) k_dither(
    const double* __restrict__ bm, int w, int h, int budget,
    int* __restrict__ cells, int cap, int* __restrict__ n_out,
    double* __restrict__ mass_out, double* gbuf) {
  extern __shared__ double sh[];
  double* base = gbuf ? gbuf : sh;
  double* pre = base;       // w
  double* err = base + w;   // w: errors of the previous row
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
// B[i,j,k] *= L / mean, quotient first (observation.cpp:145-150); mean =
// the sequential sum of all likelihoods (k_seqsum.cu, bit-exact) divided by
// their count (:139-141), formed identically by every thread.
__global__ void k_observe_apply(double* __restrict__ B, int w, int h, int c_local,
                                int k_off, int c_total, const int* __restrict__ samples, int n,
                                const double* __restrict__ L,
                                const double* __restrict__ lsum) {
  const double mean_v = *lsum / static_cast<double>(n * c_total);
  const double* mean = &mean_v;
  // (sample, local channel) pairs; a theta-slab shard holds global channels
  // k_off .. k_off + c_local - 1 of c_total, L is indexed s * c_total + k
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n * c_local) return;
  const int s = q / c_local, kl = q % c_local;
  const size_t p = static_cast<size_t>(kl) * w * h +
                   static_cast<size_t>(samples[2 * s + 1]) * w + samples[2 * s];
  B[p] *= L[static_cast<size_t>(s) * c_total + k_off + kl] / *mean;
}

// Global max -> status + the buffer's pending 1/max rescale
// (observation.cpp:152-169).
__global__ void k_observe_finalize(StepState* st, BufState* buf) {
  const double g = __longlong_as_double(static_cast<long long>(st->gmax_bits));
  publish_status(st, (g <= 0.0) ? GL_E_EXTINGUISHED : GL_OK, nullptr);
  if (g > 0.0) {
    buf->scaled = 1;
    buf->scale = 1.0 / g;
  }
  st->gmax_bits = 0ull;
}

}  // namespace

void launch_dither(gl_context* ctx, const double* bm, int w, int h, int budget,
                   int* d_cells, int cap, int* d_n, double* d_mass, int* d_sum_invalid,
                   void* sum_scratch) {
  const size_t rs = (static_cast<size_t>(w) + 3) & ~static_cast<size_t>(1);
  const size_t smem_pipe = (3 * rs + w) * sizeof(double) + 8 * static_cast<size_t>((w + 31) / 32 + 1) + 16;
  auto attr = [](const void* fn, size_t bytes) {
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(bytes));
    if (e != cudaSuccess) {
      throw std::runtime_error(std::string("dither kernel shared-memory opt-in failed: ") + cudaGetErrorString(e));
    }
  };
  const size_t smem = static_cast<size_t>(2) * w * sizeof(double);
  const size_t smem_seg = (4 * static_cast<size_t>(((w + 1) & ~1) + 16)) * sizeof(double) +
                          3 * 4 * static_cast<size_t>((w + 31) / 32 + 2) + 64;
  if (smem_pipe <= 200 * 1024) {
    if (smem_pipe > 48 * 1024) attr(reinterpret_cast<const void*>(k_dither_pipe), smem_pipe);
    // the total first, as a parallel bit-exact scan (falls back to the
    // pipeline's sequential chain on negative / non-finite planes)
    launch_seq_sum_big(ctx, bm, static_cast<size_t>(w) * h, d_mass, d_sum_invalid, sum_scratch);
    // the segment-parallel sweep where the plane is in the scan's domain;
    // the pipelined kernel then only runs if it could not (a device flag)
    int* d_done = d_sum_invalid + 1;
    const bool seg = GL_FS_SEG && w >= 4 * kSegWU && smem_seg <= 200 * 1024;
    if (seg) {
      if (smem_seg > 48 * 1024) attr(reinterpret_cast<const void*>(k_dither_seg), smem_seg);
      k_dither_seg<<<1, kSegT, smem_seg, ctx->stream>>>(bm, w, h, budget, d_cells, cap, d_n, d_mass, d_sum_invalid,
                                                        d_done);
      ctx->launches++;
    }
    k_dither_pipe<<<1, 64, smem_pipe, ctx->stream>>>(bm, w, h, budget, d_cells, cap, d_n, d_mass, d_sum_invalid,
                                                     seg ? d_done : nullptr);
    ctx->launches++;
  } else if (smem <= 200 * 1024) {
    attr(reinterpret_cast<const void*>(k_dither), smem);
    k_dither<<<1, 32, smem, ctx->stream>>>(bm, w, h, budget, d_cells, cap, d_n, d_mass, nullptr);
  } else {
    // rows wider than shared memory holds: the two row buffers in global
    // memory (stream-ordered allocation around the launch)
    double* gbuf = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&gbuf), smem, ctx->stream);
    if (e != cudaSuccess) throw std::runtime_error(std::string("dither row buffers: ") + cudaGetErrorString(e));
    k_dither<<<1, 32, 0, ctx->stream>>>(bm, w, h, budget, d_cells, cap, d_n, d_mass, gbuf);
    e = cudaFreeAsync(gbuf, ctx->stream);
    if (e != cudaSuccess) throw std::runtime_error(std::string("dither row buffers: ") + cudaGetErrorString(e));
  }
  ctx->launches++;
#ifdef GL_EXPERIMENT_ENV
  if (getenv("GL_DEBUG_DITHER")) {
    long long clk[12];
    cudaStreamSynchronize(ctx->stream);
    cudaMemcpyFromSymbol(clk, g_dither_clk, sizeof(clk));
    fprintf(stderr, "dither clocks: %lld %lld %lld %lld %lld %lld %lld %lld %lld (pipe: row-end wait, total, sweep, row-start wait; seg: spec, verify, pre, all, barrier-1 wait, staging, group chain, group rest, replays) (%d x %d)\n", clk[0], clk[1], clk[2], clk[3], clk[4], clk[5], clk[6], clk[7] & ((1LL << 40) - 1), clk[7] >> 40, w, h);
    fprintf(stderr, "dither events: fixed lanes %lld, fixed pixels %lld, exact rows %lld; setup %lld groups %lld\n", clk[9], clk[10], clk[11], clk[4], clk[6]);
  }
#endif

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

void launch_observe_apply(gl_context* ctx, double* buf, int w, int h, int c_local,
                          int k_off, int c_total, const int* d_samples, int n,
                          const double* d_L, double* d_mean, void* sum_scratch) {
  // d_mean[0]: the likelihoods' sequential sum; d_mean[1]: scan-domain flag
  int* flag = reinterpret_cast<int*>(d_mean + 1);
  launch_seq_sum_big(ctx, d_L, static_cast<size_t>(n) * c_total, d_mean, flag, sum_scratch);
  launch_seq_sum_chain(ctx, d_L, static_cast<size_t>(n) * c_total, d_mean, flag);  // only if flagged
  const int total = n * c_local;
  k_observe_apply<<<(total + 127) / 128, 128, 0, ctx->stream>>>(
      buf, w, h, c_local, k_off, c_total, d_samples, n, d_L, d_mean);
  ctx->launches++;
}

void launch_observe_finalize(gl_context* ctx, StepState* st, BufState* buf) {
  k_observe_finalize<<<1, 1, 0, ctx->stream>>>(st, buf);
  ctx->launches++;
}

}  // namespace glb
