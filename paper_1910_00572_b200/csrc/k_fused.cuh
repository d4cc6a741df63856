// Fused Algorithm-1 step for sm_100a: one launch reads the belief tensor
// once and writes it once (belief_tensor.cpp:396-498 in a single pass).
//
// Work unit = one WARP owning an OW x ROWS output tile (OW = 32 - 2R
// columns) for ALL channels; a CTA holds NWARP independent warps. Lane l
// computes the shifted/masked value S at column x0 - R + l, so the R
// outermost lanes carry the horizontal halo and no shared-memory exchange or
// block barrier is needed inside the channel loop. Per channel m
// (m = -H .. C-1+H, circular):
//   1. TMA (cp.async.bulk.tensor.3d) brings the channel's source box into
//      the warp's shared-memory stage. The box origin absorbs the integer
//      part of the channel's motion vector, so the four bilinear taps sit at
//      fixed offsets; out-of-grid cells arrive as zeros (== the reference's
//      "skip taps outside the grid"). NS-stage mbarrier pipeline per warp.
//   2. Rolling down the rows: S = mask(shift(B)) (2 smem loads per row), the
//      row pass of the separable Gaussian from S(l-R..l+R) via warp shuffles,
//      the column pass over a rolling window of row results -> D_m(row).
//   3. Channels are walked in DESCENDING order, so output channel k's
//      angular sum out = sum_t w_t * D[k - off_t] receives its terms in the
//      reference's order (D[k+H] first) as D_m(row) appears: 2H running
//      sums per row stay live in registers; when D_{k-H}(row) arrives the
//      sum is finished, masked, times the activation inverse, stored,
//      max-reduced. Every tap set is symmetric bitwise, so each D value (and
//      each S and row-pass value) is multiplied by its distinct taps once and
//      the products are shared (same products, same addition order).
// The last CTA turns the global max into the extinguish status and the
// output buffer's pending 1/max rescale (gl_internal.hpp: BufState).
//
// Built with --fmad=false; every arithmetic expression keeps the reference's
// operand order, so the output is bit-identical to step().
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <stdexcept>
#include <string>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <type_traits>

#pragma once
#include "gl_internal.hpp"
#include "wall.hpp"

#ifndef GL_FUSED_ROWS_H1
#define GL_FUSED_ROWS_H1 8   // tile rows for angular half-width H <= 1
#endif
#ifndef GL_FUSED_MINB
#define GL_FUSED_MINB 4      // min resident CTAs/SM -> register cap
#endif
#ifndef GL_FUSED_INVREG_ROWS
#define GL_FUSED_INVREG_ROWS 8  // tiles up to this height keep inv in registers
#endif
#ifndef GL_FUSED_STCS
#define GL_FUSED_STCS 1         // 1: output stores with the evict-first (.cs) hint
#endif
#ifndef GL_FUSED_HIMAX
#define GL_FUSED_HIMAX 1        // high-word max + exact epilogue fallback (FAST steps)
#endif
#ifndef GL_FUSED_INVSMEM
#define GL_FUSED_INVSMEM 1      // the tile's inverse in shared memory (frees 16 registers; measured +2-4% at 1024^2x72)
#endif
#ifndef GL_FUSED_ROT_H
// angular half-widths from which the channel loop is ROLLED with a rotating
// ring of running sums (one channel body of code instead of 2H+1 unrolled
// ones: at H = 3 the unrolled loop is ~4400 SASS instructions and the warps
// stall on instruction fetch); below it the ring slots are indexed at
// compile time in a loop unrolled by 2H+1
#define GL_FUSED_ROT_H 99
#endif
#ifndef GL_FUSED_ROT_UNROLL
#define GL_FUSED_ROT_UNROLL 1   // unroll factor of the rolled channel loop
#endif
#ifndef GL_FUSED_ROWS_H3
#define GL_FUSED_ROWS_H3 4      // tile rows for H >= 2 (Theta = 360: H = 3)
#endif
#ifndef GL_FUSED_MINB_H3
#define GL_FUSED_MINB_H3 4
#endif
#ifndef GL_FUSED_INVREG_ROWS_H3
#define GL_FUSED_INVREG_ROWS_H3 8
#endif


// k_fused.cuh: the fused step kernel templates. Each (R, H) instantiation of
// launch_rh lives in its own translation unit (k_fused_inst_r*_h*.cu, built
// in parallel); k_fused.cu holds the host driver and the epilogue kernel.
namespace glb {
namespace fk {


// HIMAX decision bound: the high word of 1e-6 (0x3EB0C6F7A0B5ED8D) with a
// zero low word. A max whose high word exceeds it is > 1e-6 (no rescale, not
// extinguished); at or below it the exact max is taken.
constexpr int kHiWord1em6 = 0x3EB0C6F7;

__device__ __forceinline__ double dmax_ref(double a, double b) {
  return (a < b) ? b : a;
}

// compile-time loop: f(integral_constant<int, B>), ..., f(<E-1>)
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar,
                                                   uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// Warp-uniform wait: the loop exits for all lanes together, so the code after
// it is provably convergent (shuffles stay plain SHFL).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!__all_sync(0xffffffffu, done));
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map,
                                            int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::"
      "bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z),
      "r"(smem_u32(bar))
      : "memory");
}

// The launch parameters: a fixed header, then the step's per-channel shift
// records and (WALL variants) the wall table. Kernel parameters are copied
// per launch, so their size is host time on every step: windows of up to
// kSmallRec records (Theta <= 90) launch with the ~5 KB FusedParamsSmall,
// larger ones with the ~21 KB FusedParams (384 records + the wall table).
struct FusedHeader {
  double* dst;
  const uint8_t* occ;
  const double* inv;
  const double* inv_masked;  // inv with occupied cells set to 0.0 (FAST)
  int inv_per_k;
  int w, h, c;               // c = output channels (interior planes of a shard)
  int shard;                 // 1: theta-slab storage with halo planes
  int plane_off;             // shard: storage plane of iteration 0 (= halo - H)
  int out_off;               // shard: storage plane of output channel 0 (= halo)
  int defer_finalize;        // shard: leave the local max for a cross-rank all-reduce

  int tiles_x, n_tiles;
  int tiles_y, strip_w;      // tile order: vertical strips strip_w tiles wide (0: row-major)
  int stack, grid_y;         // stack > 1: a CTA's warps take `stack` vertically adjacent tiles
                             // (ordering grid tiles_x x grid_y of such stacks)
  int k_base, k_end;         // this launch's output channels (a window of <= kParamChannels - 2H)
  int k_chunk, n_chunks;     // output channels per warp, chunks per tile
  // wave-tail split: the CTAs from head_ctas on (the last tiles) run their
  // channels in tail_chunks chunks of tail_k, so the grid's last partial wave
  // holds shorter work items (head_ctas = grid size: no split)
  int head_ctas, tail_chunks, tail_k;
  const BufState* src_state;
  BufState* dst_state;
  StepState* step_state;
  int* host_status;          // mapped status word of a synchronous gl_step, or null
  // cp.async load path (widths TMA cannot stride: odd W): storage plane 0 of
  // the own buffer and of the left / right neighbour buffers (peer reads)
  const double* src_base[3];
  double sep[2 * kFusedMaxRadius + 1];
  double ang[2 * kFusedMaxHalf + 1];
};

template <int NREC, int NWALL>
struct FusedParamsT : FusedHeader {
  static constexpr int kRec = NREC;
  static constexpr int kWall = NWALL;
  // the step's shift records (host) for the window's input planes: output
  // channels k_base-H .. k_end-1+H (shard: storage planes from plane_off + k_base)
  ChanRec rec[NREC];
  // wall-crossing mask (WALL variants): the crossed cells of each distinct
  // (floor dx, floor dy) of the window, indexed by ChanRec::wall
  WallEntry wall[NWALL > 0 ? NWALL : 1];
};
constexpr int kSmallRec = 96;
using FusedParams = FusedParamsT<kParamChannels, kWallEntries>;
using FusedParamsSmall = FusedParamsT<kSmallRec, 0>;

template <int R, int ROWS>
struct Geo {
  static constexpr int OW = 32 - 2 * R;     // output columns per warp
  static constexpr int SH = ROWS + 2 * R;   // S rows per tile
  // TMA box: 33 source columns (S columns -R..32-R need c0 and c1) plus one
  // for the even-aligned origin (TMA needs 16-B aligned inner coordinates)
  static constexpr int BW = 34;
  static constexpr int BH = SH + 1;
  static constexpr int B_ELEMS = BW * BH;
  static constexpr uint32_t B_BYTES = B_ELEMS * 8;    // TMA transaction bytes
  static constexpr int STAGE = (B_ELEMS + 15) & ~15;  // 128-B aligned stages
};

// Per-channel bilinear weights (belief_tensor.cpp:87-98) and the integral
// flag (:71-86), from the host-computed record (glb::chan_rec, the
// reference's operations in its order): no per-lane weight arithmetic.
struct ChanShift {
  double w00, w10, w01, w11;
  int sx, sy;
  bool integral;
};

__device__ __forceinline__ ChanShift chan_shift(const ChanRec& r) {
  ChanShift s;
  s.w00 = r.w00;
  s.w10 = r.w10;
  s.w01 = r.w01;
  s.w11 = r.w11;
  s.sx = r.ox;
  s.sy = r.oy;
  s.integral = r.integral != 0;
  return s;
}

// One S value from the four taps: r0 = row j-sy, r1 = j-sy-1, c0 = i-sx,
// c1 = i-sx-1; w00, w10, w01, w11 added to 0.0 in that order
// (belief_tensor.cpp:112-120). Integral shifts copy r0c0 exactly (:71-86);
// both forms are evaluated and selected, so there is no per-cell branch.
//
// FAST (the source buffer is "clean": every value finite and >= +0.0, which
// init_uniform and every step/update on a clean buffer preserve) drops two
// bitwise no-ops: the 0.0 seed of each accumulation (0.0 + x == x unless
// x == -0.0, and a product of non-negative finite values is never -0.0), and
// the integral-copy select (weights (1,0,0,0) give a + (+0) + ... == a).
template <bool FAST>
__device__ __forceinline__ double s_cell(const ChanShift& cs, double r0c0,
                                         double r0c1, double r1c0,
                                         double r1c1) {
  if constexpr (FAST) {
    double acc = cs.w00 * r0c0;
    acc += cs.w10 * r0c1;
    acc += cs.w01 * r1c0;
    acc += cs.w11 * r1c1;
    return acc;
  } else {
    double acc = 0.0;
    acc += cs.w00 * r0c0;
    acc += cs.w10 * r0c1;
    acc += cs.w01 * r1c0;
    acc += cs.w11 * r1c1;
    return cs.integral ? r0c0 : acc;
  }
}

// s_cell with the wall-crossing mask (wall.hpp): a blocked tap adds +0.0
// instead of its product, which equals skipping it — the accumulation starts
// at +0.0 and a sum seeded with +0.0 is never -0.0, so acc + 0.0 == acc
// (FAST: the products of a clean buffer are >= +0.0 as well). Integral
// shifts copy r0c0 unless its tap is blocked.
template <bool FAST>
__device__ __forceinline__ double s_cell_wall(const ChanShift& cs, double r0c0, double r0c1, double r1c0,
                                              double r1c1, uint32_t blk) {
  double acc = (blk & 1u) ? 0.0 : cs.w00 * r0c0;
  if constexpr (!FAST) acc = 0.0 + acc;
  acc += (blk & 2u) ? 0.0 : cs.w10 * r0c1;
  acc += (blk & 4u) ? 0.0 : cs.w01 * r1c0;
  acc += (blk & 8u) ? 0.0 : cs.w11 * r1c1;
  if constexpr (FAST) {
    return acc;
  } else {
    return cs.integral ? ((blk & 1u) ? 0.0 : r0c0) : acc;
  }
}

// sum_t w[t] * x[t] in order from a 0.0 seed (FAST: seeded with the first
// product, bitwise identical on clean data).
template <int N, bool FAST>
__device__ __forceinline__ double dot_seq(const double* w, const double* x) {
  double acc;
  if constexpr (FAST) {
    acc = w[0] * x[0];
  } else {
    acc = 0.0;
    acc += w[0] * x[0];
  }
#pragma unroll
  for (int d = 1; d < N; ++d) acc += w[d] * x[d];
  return acc;
}

// Row pass of the separable Gaussian, acc = 0; acc += t[d+R] * S(i+d),
// d = -R..R (belief_tensor.cpp:211-214). The taps are symmetric bitwise
// (t[R-d] == t[R+d]: build_kernels evaluates exp(-0.5*d*d/..) at d and -d,
// and the host checks it), so the product t[R+d] * S(i+d) that lane i needs
// is the product t[R-|d|] * S(i+d) its neighbour forms for itself: each lane
// multiplies its S by the R+1 distinct taps once and the shuffles move
// products instead of S values (R+1 DMUL per S instead of 2R+1; same values,
// same addition order).
template <int R, bool FAST>
__device__ __forceinline__ double row_pass(const FusedHeader& p, double s) {
  double q[R + 1];
#pragma unroll
  for (int j = 0; j <= R; ++j) q[j] = p.sep[j] * s;
  double acc = __shfl_up_sync(0xffffffffu, q[0], R);  // d = -R
  if constexpr (!FAST) acc = 0.0 + acc;
#pragma unroll
  for (int d = -R + 1; d <= R; ++d) {
    double v;
    if (d < 0) {
      v = __shfl_up_sync(0xffffffffu, q[R + d], -d);
    } else if (d == 0) {
      v = q[R];
    } else {
      v = __shfl_down_sync(0xffffffffu, q[R - d], d);
    }
    acc += v;
  }
  return acc;
}

template <int R, int H, int ROWS, int NS, bool FAST, bool HIMAX, bool TMA, bool WALL, class P>
__device__ __forceinline__ double warp_tile(const CUtensorMap* tmap,
                                            const CUtensorMap* tmap_lo,
                                            const CUtensorMap* tmap_hi,
                                            const P& p, double* Bs,
                                            uint64_t* mbar, int lane, int x0,
                                            int y0, int k0, int n_out,
                                            bool active, double* invs,
                                            uint32_t* colbits) {
  using G = Geo<R, ROWS>;
  constexpr int NG = 2 * H + 1;  // ring depth == angular taps
  const int W = p.w, Hh = p.h;
  const size_t plane = static_cast<size_t>(W) * Hh;
  const int n_iter = n_out + 2 * H;  // this warp's output channels k0 .. k0+n_out-1
  const bool scaled = p.src_state->scaled != 0;  // pending 1/max rescale
  const double sc = p.src_state->scale;

  // Iteration it reads record rec0 + n_iter - 1 - it (the channel walk is
  // descending, see channel() below): the host resolved its source plane
  // (z) and tensor map (own buffer; circular channel walk on one GPU, linear
  // over halo storage for a theta-slab shard, or a neighbour's buffer over
  // peer memory for a shard's halo planes, so no halo exchange step exists).
  const int rec0 = k0 - p.k_base;
  // TMA: lane 0 issues one 3-D box copy. Otherwise (a row pitch TMA cannot
  // stride, i.e. odd W) every lane issues 8-byte cp.async copies of its share
  // of the same box, zero-filled outside the grid, and arrives on the
  // stage's mbarrier (count 32) when they land: same smem layout, same
  // consumer code.
  auto issue = [&](int it, int stage) {
    const ChanRec& rc = p.rec[rec0 + n_iter - 1 - it];  // descending walk
    const int map = rc.map;
    const int bx0 = (x0 - R - rc.ox - 1) & ~1, by0 = y0 - R - rc.oy - 1;
    if constexpr (TMA) {
      const CUtensorMap* m = map == 0 ? tmap : (map == 1 ? tmap_lo : tmap_hi);
      mbar_arrive_expect(&mbar[stage], G::B_BYTES);
      tma_load_3d(Bs + stage * G::STAGE, m, bx0, by0, rc.z, &mbar[stage]);
    } else {
      // row by row: lane l copies box column l (lanes 0, 1 also 32, 33)
      const double* plane_base = p.src_base[map] + plane * static_cast<size_t>(rc.z);
      const uint32_t dst0 = smem_u32(Bs + stage * G::STAGE) + 8u * lane;
      const int gx = bx0 + lane, gx2 = bx0 + 32 + lane;
      const bool xin = gx >= 0 && gx < W;
      const bool xin2 = lane < G::BW - 32 && gx2 >= 0 && gx2 < W;
      ptrdiff_t row = static_cast<ptrdiff_t>(by0) * W;
#pragma unroll
      for (int by = 0; by < G::BH; ++by, row += W) {
        const bool yin = by0 + by >= 0 && by0 + by < Hh;
        const bool in = xin && yin, in2 = xin2 && yin;
        const double* src = in ? plane_base + row + gx : plane_base;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst0 + 8u * by * G::BW), "l"(src),
                     "r"(in ? 8 : 0)
                     : "memory");
        if (lane < G::BW - 32) {
          const double* src2 = in2 ? plane_base + row + gx2 : plane_base;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst0 + 8u * (by * G::BW + 32)),
                       "l"(src2), "r"(in2 ? 8 : 0)
                       : "memory");
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&mbar[stage]))
                   : "memory");
    }
  };

  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&mbar[s], TMA ? 1 : 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (TMA) {
      for (int s = 0; s < NS && s < n_iter; ++s) issue(s, s);
    }
  }
  __syncwarp();
  if constexpr (!TMA) {
    for (int s = 0; s < NS && s < n_iter; ++s) issue(s, s);
  }

  // Per-tile constants of this lane's column: S mask bits (occupied or
  // outside the grid), store-valid bits, and the activation inverse of the
  // output cells (one k-invariant plane on the fused path).
  const int si = x0 - R + lane;
  const bool col_in = si >= 0 && si < W;
  uint32_t smask = 0;
#pragma unroll
  for (int lj = 0; lj < G::SH; ++lj) {
    const int j = y0 - R + lj;
    const bool inside = col_in && j >= 0 && j < Hh;
    const bool occ = !inside || p.occ[static_cast<size_t>(j) * W + si] != 0;
    smask |= static_cast<uint32_t>(occ) << lj;
  }
  if constexpr (WALL) {
    // the wall mask's occupancy window: bit b of colbits[c] is cell
    // (x0 - R - 8 + c, y0 - R - 8 + b), 1 = occupied or outside the grid
    for (int c = lane; c < 32 + 16; c += 32) {
      const int gx = x0 - R - 8 + c;
      uint32_t bitsv = 0;
      for (int b = 0; b < 32; ++b) {
        const int gy = y0 - R - 8 + b;
        const bool o = gx < 0 || gx >= W || gy < 0 || gy >= Hh || p.occ[static_cast<size_t>(gy) * W + gx] != 0;
        bitsv |= static_cast<uint32_t>(o) << b;
      }
      colbits[c] = bitsv;
    }
    __syncwarp();
  }
  const bool out_lane = active && lane >= R && lane < 32 - R && si < W;
  // The inverse is held in registers for short tiles (INVREG) or re-read from
  // L1 per channel for tall ones. FAST folds the output mask into it: for the
  // finite non-negative values of a clean buffer out * 0.0 == +0.0, which is
  // the reference's "out = 0.0" for occupied cells (:466-467).
  constexpr bool INVSM = GL_FUSED_INVSMEM != 0;
  constexpr bool INVREG = !INVSM && ROWS <= (H <= 1 ? GL_FUSED_INVREG_ROWS : GL_FUSED_INVREG_ROWS_H3);
  const double* inv_col = (FAST ? p.inv_masked : p.inv) + (out_lane ? si : 0);
  double invr[INVREG ? ROWS : 1];
  uint32_t store_ok = 0;
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const bool ok = out_lane && (y0 + r) < Hh;
    store_ok |= static_cast<uint32_t>(ok) << r;
    if constexpr (INVREG) invr[r] = ok ? __ldg(inv_col + static_cast<size_t>(y0 + r) * W) : 0.0;
    if constexpr (INVSM) invs[r * 32 + lane] = ok ? __ldg(inv_col + static_cast<size_t>(y0 + r) * W) : 0.0;
  }
  if constexpr (INVSM) __syncwarp();
  [[maybe_unused]] const double* inv_tile = inv_col + static_cast<size_t>(y0) * W;
  double* const out_tile = p.dst + static_cast<size_t>(y0) * W + (out_lane ? si : 0);

  // Angular accumulators: output channel k's sum lives in slot
  // (iteration of its last term) % NG; with the channel walk reversed its
  // terms arrive in the reference's tap order (D[k+H] first).
  double aacc[NG][ROWS];
  double vmax = 0.0;
  unsigned int hmax = 0u;  // HIMAX: max of the outputs' high words

  // One channel: wait for its box, S -> row pass -> column pass -> D_m, whose
  // products with the angular taps go into the output accumulators; with
  // EMIT, output channel m + H (its last term) is finished row by row.
  // Channels are walked DOWNWARD (iteration it reads input channel
  // k0 + n_out - 1 + H - it): output k = sum_t w_t * D[k - (t - H)] adds
  // D[k+H] first (belief_tensor.cpp:449-463), so a descending walk turns the
  // angular stencil into running sums whose symmetric taps (w_t == w_{2H-t}
  // bitwise, host-checked) need H+1 products per D value, not 2H+1.
  // ROT: a rolled channel loop whose ring is rotated instead of indexed:
  // after input channel m, P[i] holds the running sum of output m - H + i
  // (terms 0..i), i = 0..2H-1; the next channel's D finishes P[2H-1] (its
  // last term, emitted), moves every P[i-1] + w_i D into P[i] (in place, top
  // down: no register moves) and starts P[0] = w_0 D. Slots that do not
  // hold a real output yet (the first 2H channels) are never emitted.
  constexpr bool ROT = H >= GL_FUSED_ROT_H;
  auto channel = [&](const int it, auto Ut, auto Et, auto Pt, const bool emit_rt) {
    constexpr int u = decltype(Ut)::value;
    constexpr bool emit_ct = decltype(Et)::value;
    constexpr int tmax = decltype(Pt)::value;  // terms t <= tmax exist (prologue)
    const bool emit = ROT ? emit_rt : emit_ct;
    const int stage = it % NS;
    const int q_in = n_iter - 1 - it;  // relative input channel
    const ChanShift cs = chan_shift(p.rec[rec0 + q_in]);
    double* stage_ptr = Bs + stage * G::STAGE;
    mbar_wait(&mbar[stage], static_cast<uint32_t>((it / NS) & 1));
    if (scaled) {
      // rare: the source buffer carries a pending rescale (stored values
      // times sc are the reference's values), applied to the box in smem
      // (4 loads in flight at a time: few registers in the hot kernels)
      constexpr int kPer = (G::B_ELEMS + 31) / 32;
#pragma unroll 1
      for (int i0 = 0; i0 < kPer; i0 += 4) {
        double bx[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = lane + 32 * (i0 + i);
          bx[i] = q < G::B_ELEMS ? stage_ptr[q] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int q = lane + 32 * (i0 + i);
          if (q < G::B_ELEMS) stage_ptr[q] = bx[i] * sc;
        }
      }
      __syncwarp();
    }
    const double* Bb = stage_ptr + ((x0 - R - cs.sx - 1) & 1) + lane;
    // wall mask: bit lj of wb[t] = tap t of S row lj crosses an occupied cell
    [[maybe_unused]] uint32_t wb[4] = {0u, 0u, 0u, 0u};
    if constexpr (WALL) {
      const WallEntry& we = p.wall[p.rec[rec0 + q_in].wall];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        for (int m = 0; m < we.n[t]; ++m) {
          const int cell = we.cell[t][m];
          const int qx = (cell & 15) - 8, qy = (cell >> 4) - 8;
          wb[t] |= colbits[lane + 8 + qx] >> (qy + 8);
        }
      }
    }
    // emitted output channel k0 + q_in (its last tap reads input q_in = k - H)
    double* orow = out_tile + plane * static_cast<size_t>(p.out_off + k0 + (emit ? q_in : 0));  // += W per row

    double lo_c0 = Bb[1], lo_c1 = Bb[0];
    [[maybe_unused]] double cacc[ROWS];  // column-pass running sums per output row (R > 0)
#pragma unroll
    for (int lj = 0; lj < G::SH; ++lj) {
      const double hi_c0 = Bb[(lj + 1) * G::BW + 1];
      const double hi_c1 = Bb[(lj + 1) * G::BW];
      double s;
      if constexpr (WALL) {
        const uint32_t blk = ((wb[0] >> lj) & 1u) | (((wb[1] >> lj) & 1u) << 1) | (((wb[2] >> lj) & 1u) << 2) |
                             (((wb[3] >> lj) & 1u) << 3);
        s = s_cell_wall<FAST>(cs, hi_c0, hi_c1, lo_c0, lo_c1, blk);
      } else {
        s = s_cell<FAST>(cs, hi_c0, hi_c1, lo_c0, lo_c1);
      }
      s = ((smask >> lj) & 1u) ? 0.0 : s;
      lo_c0 = hi_c0;
      lo_c1 = hi_c1;
      int r = -1;
      double d = 0.0;
      if constexpr (R == 0) {
        r = lj;
        d = s;
      } else {
        // column pass: orow = 0; += t[d] * row(j+d), d = -R..R (:227-238).
        // Row lj is term t = lj - r of output row r (first for r = lj, last
        // for r = lj - 2R); symmetric taps: R+1 products per row result.
        const double x = row_pass<R, FAST>(p, s);
        double cq[R + 1];
#pragma unroll
        for (int j = 0; j <= R; ++j) cq[j] = p.sep[j] * x;
#pragma unroll
        for (int t = 0; t <= 2 * R; ++t) {
          const int rr = lj - t;
          if (rr >= 0 && rr < ROWS) {
            const double v = cq[t <= R ? t : 2 * R - t];
            if (t == 0) {
              if constexpr (FAST) {
                cacc[rr] = v;
              } else {
                cacc[rr] = 0.0 + v;
              }
            } else {
              cacc[rr] += v;
            }
          }
        }
        if (lj >= 2 * R) {
          r = lj - 2 * R;
          d = cacc[r];
        }
      }
      if (r >= 0) {
        // angular taps (belief_tensor.cpp:449-463): D_m is term t of the
        // output finished 2H - t iterations later, slot (u + 2H - t) % NG
        double aq[H + 1];
#pragma unroll
        for (int j = 0; j <= H; ++j) aq[j] = p.ang[j] * d;
        double o = 0.0;
        if constexpr (ROT) {
          if constexpr (H == 0) {
            o = aq[0];
          } else {
            o = aacc[2 * H - 1][r] + aq[0];  // term 2H (w_2H == w_0)
#pragma unroll
            for (int i = 2 * H - 1; i >= 1; --i) aacc[i][r] = aacc[i - 1][r] + aq[i <= H ? i : 2 * H - i];
            aacc[0][r] = aq[0];  // term 0 starts an output (no 0.0 seed: belief_tensor.cpp:454)
          }
        } else {
#pragma unroll
          for (int t = 0; t <= 2 * H; ++t) {
            if (t > tmax) continue;
            const double v = aq[t <= H ? t : 2 * H - t];
            const int slot = (u + 2 * H - t) % NG;
            if (t == 2 * H) {
              o = (H == 0) ? v : aacc[slot][r] + v;
            } else if (t == 0) {
              aacc[slot][r] = v;
            } else {
              aacc[slot][r] += v;
            }
          }
        }
        if (emit) {
          // mask, x inverse, max (belief_tensor.cpp:464-474)
          double iv;
          if constexpr (INVREG) {
            iv = invr[r];
          } else if constexpr (INVSM) {
            iv = invs[r * 32 + lane];
          } else {
            iv = ((store_ok >> r) & 1u) ? __ldg(inv_tile + r * W) : 0.0;
          }
          if constexpr (FAST) {
            o = o * iv;
          } else {
            o = ((smask >> (r + R)) & 1u) ? 0.0 : o * iv;
          }
          // std::max from 0.0 over free cells (belief_tensor.cpp:464-471);
          // masked cells contribute +0.0, which never raises the max
          if constexpr (HIMAX) {
            // clean outputs are finite and >= +0.0: their bit patterns order
            // like their values, so the high word bounds the max (one
            // integer max instead of DSETP + 2 FSEL per output row)
            hmax = max(hmax, static_cast<unsigned int>(__double2hiint(o)));
          } else {
            vmax = dmax_ref(vmax, o);
          }
          const bool ok = (store_ok >> r) & 1u;
#if GL_FUSED_STCS
          if (ok) __stcs(orow, o);  // streaming: the output is not re-read this step
#else
          if (ok) *orow = o;
#endif
          orow += W;
        }
      }
    }
    __syncwarp();  // every lane is done with this stage
    if ((!TMA || lane == 0) && it + NS < n_iter) {
      if (scaled) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(it + NS, stage);
    }
  };

  if constexpr (ROT) {
#pragma unroll
    for (int i = 0; i < NG - 1; ++i)
#pragma unroll
      for (int r = 0; r < ROWS; ++r) aacc[i][r] = 0.0;  // never emitted; keeps the prologue's reads defined
    constexpr int kRotUnroll = GL_FUSED_ROT_UNROLL;
#pragma unroll kRotUnroll
    for (int it = 0; it < n_iter; ++it) {
      channel(it, std::integral_constant<int, 0>{}, std::false_type{}, std::integral_constant<int, 2 * H>{},
              it >= 2 * H);
    }
  } else {
    // channels m = -H .. H-1 only fill the ring (slots 0 .. 2H-1) ...
    static_for<0, 2 * H>([&](auto U) {
      channel(decltype(U)::value, U, std::false_type{}, U, false);
    });
    // ... then every channel emits output channel it - 2H; slot = it % NG
    for (int base = 2 * H; base < n_iter; base += NG) {
      static_for<0, NG>([&](auto V) {
        constexpr int v = decltype(V)::value;
        const int it = base + v;
        if (it < n_iter)
          channel(it, std::integral_constant<int, (2 * H + v) % NG>{}, std::true_type{},
                  std::integral_constant<int, 2 * H>{}, true);
      });
    }
  }
  if constexpr (HIMAX) vmax = __hiloint2double(static_cast<int>(hmax), 0);
  return vmax;
}

// Tile index -> (tile column, tile row). The ordering grid is tiles_x x
// grid_y cells; a cell is one tile, or (stack > 1) `stack` vertically
// adjacent tiles taken by consecutive warps of one CTA, so vertical
// neighbours inside a CTA run in lockstep. Cells go row-major, or in
// vertical strips of strip_w cell columns walked row by row (the last strip
// takes the remaining columns): the cell below then follows strip_w cells
// later instead of a whole grid row later, so a tile's upper / lower
// neighbours run at nearly the same time and the halo rows they share are
// re-read from L2, not DRAM (gl_context_set_tile_order). A tile row past the
// grid (stack padding) comes back >= tiles_y.
__device__ __forceinline__ void tile_coords(const FusedHeader& p, int tile, int* tx, int* ty) {
  int cell = tile, w = 0;
  if (p.stack > 1) {
    cell = tile / p.stack;
    w = tile - cell * p.stack;
  }
  const int sw = p.strip_w;
  int cx, cy;
  if (sw <= 0 || sw >= p.tiles_x) {
    cy = cell / p.tiles_x;
    cx = cell - cy * p.tiles_x;
  } else {
    const int per_strip = sw * p.grid_y;
    const int full = p.tiles_x / sw;
    const int s = cell / per_strip;
    if (s < full) {
      const int q = cell - s * per_strip;
      cy = q / sw;
      cx = s * sw + (q - cy * sw);
    } else {
      const int rem = p.tiles_x - full * sw;
      const int q = cell - full * per_strip;
      cy = q / rem;
      cx = full * sw + (q - cy * rem);
    }
  }
  *tx = cx;
  *ty = cy * (p.stack > 1 ? p.stack : 1) + w;
}

template <int R, int H, int ROWS, int NS, int NWARP, bool FAST, bool HIMAX, bool TMA, bool WALL, class P>
__global__ void __launch_bounds__(32 * NWARP, H <= 1 ? GL_FUSED_MINB : GL_FUSED_MINB_H3)
    k_fused_step(const __grid_constant__ CUtensorMap tmap,
                 const __grid_constant__ CUtensorMap tmap_lo,
                 const __grid_constant__ CUtensorMap tmap_hi,
                 const P p) {
  using G = Geo<R, ROWS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // TMA destinations must be 128-B aligned. Pad by an offset computed from
  // the shared-window address, keeping the pointer in the shared space (so
  // the compiler emits LDS with immediate offsets, not generic loads).
  const uint32_t pad = (128u - (smem_u32(smem_raw) & 127u)) & 127u;
  double* stages = reinterpret_cast<double*>(smem_raw + pad);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* Bs = stages + warp * NS * G::STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NWARP * NS * G::STAGE);
  uint64_t* mbar = bars + warp * NS;
  double* wmax = reinterpret_cast<double*>(bars + NWARP * NS);
  double* invs = wmax + NWARP + warp * ROWS * 32;  // GL_FUSED_INVSMEM: [ROWS][32] per warp
  uint32_t* colbits = reinterpret_cast<uint32_t*>(wmax + NWARP + NWARP * ROWS * 32) + warp * 48;  // WALL

  if (TMA && threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  // Surplus warps of the last CTA redo the last tile with stores disabled,
  // so every warp runs the same control flow (the shuffles then compile to
  // plain SHFL instead of the divergence-safe collective sequence).
  // Work item = (channel chunk, tile). A CTA's warps share one chunk, so the
  // chunk (and every shift-record index) derives from blockIdx alone: the
  // compiler keeps the records in uniform registers. Consecutive warps take
  // neighbouring tiles, so their halo rows meet in L2.
  int tile_raw, k0, n_out;
  if (static_cast<int>(blockIdx.x) < p.head_ctas) {
    const int cta_per_chunk = (p.n_tiles + NWARP - 1) / NWARP;
    const int chunk = blockIdx.x / cta_per_chunk;
    tile_raw = (blockIdx.x - chunk * cta_per_chunk) * NWARP + warp;
    k0 = p.k_base + chunk * p.k_chunk;
    n_out = min(p.k_chunk, p.k_end - k0);
  } else {  // wave tail (n_chunks == 1 here): tiles from head_ctas * NWARP on, channel chunks of tail_k
    const int b = blockIdx.x - p.head_ctas;
    const int first = p.head_ctas * NWARP;
    const int cta_per_chunk = (p.n_tiles - first + NWARP - 1) / NWARP;
    const int chunk = b / cta_per_chunk;
    tile_raw = first + (b - chunk * cta_per_chunk) * NWARP + warp;
    k0 = p.k_base + chunk * p.tail_k;
    n_out = min(p.tail_k, p.k_end - k0);
  }
  bool active = tile_raw < p.n_tiles;
  int tx, ty;
  tile_coords(p, active ? tile_raw : p.n_tiles - 1, &tx, &ty);
  if (ty >= p.tiles_y) {  // stack padding below the grid: redo the last row, stores off
    ty = p.tiles_y - 1;
    active = false;
  }
  const int x0 = tx * G::OW;
  const int y0 = ty * ROWS;
  double vmax = warp_tile<R, H, ROWS, NS, FAST, HIMAX, TMA, WALL, P>(&tmap, &tmap_lo, &tmap_hi, p, Bs, mbar, lane, x0,
                                                             y0, k0, n_out, active, invs, colbits);

  // global max -> the last CTA finalises status and the pending rescale
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vmax = dmax_ref(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  if (lane == 0) wmax[warp] = vmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bm = 0.0;
    for (int q = 0; q < NWARP; ++q) bm = dmax_ref(bm, wmax[q]);
    StepState* st = p.step_state;
    if (bm > 0.0) atomicMax(&st->gmax_bits, static_cast<unsigned long long>(__double_as_longlong(bm)));
    __threadfence();
    const unsigned int prev = atomicAdd(&st->blocks_done, 1u);
    if (prev == gridDim.x - 1 && p.defer_finalize) {
      st->blocks_done = 0u;  // gmax_bits stays for the cross-rank all-reduce
    } else if (prev == gridDim.x - 1) {
      __threadfence();
      const unsigned long long bits = atomicAdd(&st->gmax_bits, 0ull);
      const double g = __longlong_as_double(static_cast<long long>(bits));
      if (HIMAX && g <= __hiloint2double(kHiWord1em6, 0)) {
        // the high word cannot tell max >= 1e-6 (or > 0): the step epilogue
        // kernel takes the exact max of the output and finalises
        st->need_exact = 1;
      } else if (HIMAX) {
        publish_status(st, GL_OK, p.host_status);  // max >= 2^-20 > 1e-6: no rescale
        p.dst_state->scaled = 0;
        p.dst_state->scale = 1.0;
      } else {
      publish_status(st, (g <= 0.0) ? GL_E_EXTINGUISHED : GL_OK, p.host_status);
      if (g > 0.0 && g < 1e-6) {
        p.dst_state->scaled = 1;
        p.dst_state->scale = 1.0 / g;
      } else {
        p.dst_state->scaled = 0;
        p.dst_state->scale = 1.0;
      }
      }
      st->gmax_bits = 0ull;
      st->blocks_done = 0u;
    }
  }
}

#ifndef GL_FUSED_NS
#define GL_FUSED_NS 3  // measured: 3 stages 0.247-0.256 ms vs 2 stages 0.253-0.261 ms at 1024^2 x 72
#endif
constexpr int kNS = GL_FUSED_NS;  // TMA stages per warp
constexpr int kNWARP = 4;  // warps (independent tiles) per CTA

template <int H>
constexpr int rows_for() {
  return H <= 1 ? GL_FUSED_ROWS_H1 : GL_FUSED_ROWS_H3;
}

template <int R, int ROWS, bool WALL>
constexpr size_t smem_bytes() {
  using G = Geo<R, ROWS>;
  return 128 + static_cast<size_t>(kNWARP) * kNS * G::STAGE * 8 + kNWARP * kNS * 8 + kNWARP * 8 +
         static_cast<size_t>(kNWARP) * ROWS * 32 * 8 + (WALL ? kNWARP * 48 * 4 : 0);
}

// Wave-tail default (measured, profiles/r01_sweeps.md "wave tail"): with
// 4 resident CTAs per SM, a grid of more than one wave whose last partial
// wave holds rem CTAs splits its last ~rem/5 CTAs (rounded down to 32) into
// 3 channel chunks. 1024^2 x 72 (1120 CTAs, rem 528 -> 96): 0.2475 ->
// 0.2384 ms; 128 CTAs measured the same, 64 / 160 / 4 chunks gave nothing.
// `slots` = resident CTAs of the instantiated kernel on the whole GPU
// (occupancy API x SMs). Gated to the measured shape class: grids of 1..4
// waves, where the partial last wave is a large share of the run; longer
// grids (4096^2: 59 waves) gain nothing from it and keep one chunk.
inline int auto_tail_ctas(int slots, int blocks) {
  if (slots <= 0 || blocks <= slots || blocks > 4 * slots) return 0;
  return ((blocks % slots) / 5) & ~31;
}

// Tuning-experiment environment overrides (GRIDLOC_B200_CHUNKS,
// GRIDLOC_B200_TAIL = "ctas[,chunks]"): compiled in only with
// -DGL_EXPERIMENT_ENV (tools/build_variants.sh); the shipped library ignores
// the environment and takes only the gl_context_set_* settings.
inline int env_int(const char* name, int dflt) {
#ifdef GL_EXPERIMENT_ENV
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
#else
  (void)name;
  return dflt;
#endif
}
inline int env_tail_chunks() {
#ifdef GL_EXPERIMENT_ENV
  const char* e = std::getenv("GRIDLOC_B200_TAIL");
  const char* c = e ? std::strchr(e, ',') : nullptr;
  return c ? std::atoi(c + 1) : 0;
#else
  return 0;
#endif
}

// Auto tile order (measured, profiles/r02_tile_order.md): grids up to 48
// tiles wide stay row-major (1024^2: a tile row is 35 tiles and its halo rows
// are still in L2 when the row below runs; strips there cost 4%); wider
// grids walk vertical strips of ~35 tiles (4096^2: 137 tiles -> 4 strips of
// 35: DRAM reads 74.1 -> 52.4 GB per step, 48.5 GB algorithmic; kernel
// -2.4..-4%).
inline int auto_strip_tiles(int tiles_x) {
  if (tiles_x <= 48) return 0;
  const int n = (tiles_x + 34) / 35;
  return (tiles_x + n - 1) / n;
}

template <int R, int H, bool FAST, bool HIMAX, bool TMA, bool WALL, class P>
void launch_rhf(gl_context* ctx, const CUtensorMap* const* tmaps, P& fp) {
  const int n_win = fp.k_end - fp.k_base;
  constexpr int ROWS = rows_for<H>();
  using G = Geo<R, ROWS>;
  constexpr size_t smem = smem_bytes<R, ROWS, WALL>();
  auto kern = k_fused_step<R, H, ROWS, kNS, kNWARP, FAST, HIMAX, TMA, WALL, P>;
  // per device (the attribute is per device): the dynamic shared-memory
  // opt-in and the resident CTAs per SM it leaves (grid sizing below)
  static std::atomic<int> per_sm[64] = {};
  const int dslot = ctx->device & 63;
  int cta_per_sm = per_sm[dslot].load(std::memory_order_acquire);
  if (cta_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    int n = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 32 * kNWARP, smem);
    if (e != cudaSuccess || n < 1) {
      throw std::runtime_error(std::string("fused step kernel cannot be configured: ") + cudaGetErrorString(e));
    }
    per_sm[dslot].store(n, std::memory_order_release);
    cta_per_sm = n;
  }
  const int sms = ctx->sm_count > 0 ? ctx->sm_count : 148;
  fp.tiles_x = (fp.w + G::OW - 1) / G::OW;
  fp.tiles_y = (fp.h + ROWS - 1) / ROWS;
  // tile order: strips only pay where a full tile row is long enough that
  // its upper neighbour's halo rows leave L2 before the row below runs
  fp.strip_w = ctx->strip_tiles >= 0 ? ctx->strip_tiles : auto_strip_tiles(fp.tiles_x);
  fp.stack = ctx->tile_stack > 0 ? std::min(ctx->tile_stack, kNWARP) : 1;
  fp.grid_y = (fp.tiles_y + fp.stack - 1) / fp.stack;
  fp.n_tiles = fp.tiles_x * fp.grid_y * fp.stack;  // ordering cells x their stacks (padding rows inactive)
  // Small grids leave SMs idle with one warp per tile: split the channels
  // into chunks (each recomputes its 2H angular neighbours) until one full
  // wave of resident warps (16 per SM) exists, keeping the recompute below
  // 50%. Measured at 1024^2 x 72 (4480 tiles): 1 chunk 0.265 ms, 2 chunks
  // 0.274 ms — chunking only pays when the tiles cannot fill the GPU.
  fp.n_chunks = 1;
  const long wave = static_cast<long>(kNWARP) * cta_per_sm * sms;  // resident warps
  if (fp.n_tiles < wave) {
    // at most one wave: a second, mostly empty wave costs a whole warp
    // lifetime (measured 256^2 x 36: 9 chunks = 1.09 waves 22.7 us, 4 chunks 20.2 us)
    const int want = static_cast<int>(wave / fp.n_tiles);
    const int max_chunks = n_win / (H == 0 ? 2 : 4 * H);
    fp.n_chunks = std::max(1, std::min(want, max_chunks));
  }
  static const int chunk_override = env_int("GRIDLOC_B200_CHUNKS", 0);
  if (ctx->channel_chunks > 0) fp.n_chunks = std::min(ctx->channel_chunks, n_win);
  if (chunk_override > 0) fp.n_chunks = std::min(chunk_override, n_win);
  fp.k_chunk = (n_win + fp.n_chunks - 1) / fp.n_chunks;
  fp.n_chunks = (n_win + fp.k_chunk - 1) / fp.k_chunk;
  int blocks = ((fp.n_tiles + kNWARP - 1) / kNWARP) * fp.n_chunks;
  // Wave tail: with one chunk, the grid's last partial wave of CTAs leaves
  // slots idle while it runs; the last tail CTAs' tiles are split into
  // channel chunks so the tail drains in shorter work items.
  static const int tail_override = env_int("GRIDLOC_B200_TAIL", -1);
  static const int tail_chunks_override = env_tail_chunks();
  fp.head_ctas = blocks;
  fp.tail_chunks = 1;
  fp.tail_k = fp.k_chunk;
  int tail = ctx->tail_ctas >= 0 ? ctx->tail_ctas : auto_tail_ctas(cta_per_sm * sms, blocks);
  if (tail_override >= 0) tail = tail_override;
  tail = fp.n_chunks == 1 ? std::min(tail, blocks) : 0;
  const int tail_chunks = std::max(1, std::min(tail_chunks_override > 0 ? tail_chunks_override : ctx->tail_chunks, n_win));
  if (tail > 0 && tail_chunks > 1) {
    fp.head_ctas = blocks - tail;
    fp.tail_k = (n_win + tail_chunks - 1) / tail_chunks;
    fp.tail_chunks = (n_win + fp.tail_k - 1) / fp.tail_k;
    const int tail_tiles = fp.n_tiles - fp.head_ctas * kNWARP;
    blocks = fp.head_ctas + ((tail_tiles + kNWARP - 1) / kNWARP) * fp.tail_chunks;
  }
  static const CUtensorMap kNoMap{};  // the cp.async path never reads its maps
  kern<<<blocks, 32 * kNWARP, smem, ctx->stream>>>(TMA ? *tmaps[0] : kNoMap, TMA ? *tmaps[1] : kNoMap,
                                                   TMA ? *tmaps[2] : kNoMap, fp);
  ctx->launches++;
}

template <int R, int H, class P>
void launch_rh(gl_context* ctx, const CUtensorMap* const* tmap, P& fp, bool fast, bool himax, bool wall) {
  if (wall) {  // TMA only (odd widths take the generic chain), exact max; the big params carry the table
    if constexpr (P::kWall > 0) {
      if (fast) {
        launch_rhf<R, H, true, false, true, true>(ctx, tmap, fp);
      } else {
        launch_rhf<R, H, false, false, true, true>(ctx, tmap, fp);
      }
    } else {
      throw std::logic_error("wall-mask step routed to parameters without a wall table");
    }
  } else if (tmap[0] == nullptr) {  // cp.async loads (odd widths); no high-word max variant
    if (fast) {
      launch_rhf<R, H, true, false, false, false>(ctx, tmap, fp);
    } else {
      launch_rhf<R, H, false, false, false, false>(ctx, tmap, fp);
    }
  } else if (fast && himax) {
    launch_rhf<R, H, true, true, true, false>(ctx, tmap, fp);
  } else if (fast) {
    launch_rhf<R, H, true, false, true, false>(ctx, tmap, fp);
  } else {
    launch_rhf<R, H, false, false, true, false>(ctx, tmap, fp);
  }
}

}  // namespace fk
}  // namespace glb
