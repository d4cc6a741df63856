// Fused Algorithm-1 step for sm_100a: one launch reads the belief tensor
// once and writes it once (belief_tensor.cpp:396-498 in a single pass).
//
// CTA = 64 threads (2 warps) owning a 64 x ROWS spatial tile and ALL
// channels. Per channel m (m = -H .. C-1+H, circular):
//   1. TMA (cp.async.bulk.tensor.3d) brings the channel's source box into
//      shared memory. The box origin absorbs the integer part of the
//      channel's motion vector, so the bilinear taps sit at fixed smem
//      offsets; out-of-grid cells arrive as zeros (== the reference's
//      "skip taps outside the grid"). NS-stage mbarrier pipeline.
//   2. S = mask(shift(B)) for the tile plus an R-cell halo -> smem.
//   3. Separable Gaussian: row pass from smem, column pass rolled over the
//      thread's column in registers -> D_m (ROWS values per thread).
//   4. D_m enters a (2H+1)-deep register ring; output channel k = m - H is
//      out = sum_t w_t * D[k - off_t] (first tap initialises), masked,
//      multiplied by the activation inverse, stored, and max-reduced.
// The last CTA turns the global max into the extinguish status and the
// output buffer's pending 1/max rescale (see gl_internal.hpp: BufState).
//
// Built with --fmad=false; every arithmetic expression keeps the reference's
// operand order, so the output is bit-identical to step().
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gl_internal.hpp"

namespace glb {

namespace {

constexpr int TW = 64;  // tile width == threads per CTA

__device__ __forceinline__ double dmax_ref(double a, double b) {
  return (a < b) ? b : a;
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
  } while (!done);
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

struct FusedParams {
  double* dst;
  const double2* motion;  // per channel (dx, dy), cells (when C > kParamChannels)
  int param_motion;       // 1: motion vectors are in mv[] below
  const uint8_t* occ;
  const double* inv;
  int inv_per_k;
  int w, h, c;
  const BufState* src_state;
  BufState* dst_state;
  StepState* step_state;
  double sep[2 * kFusedMaxRadius + 1];
  double ang[2 * kFusedMaxHalf + 1];
  double2 mv[kParamChannels];  // the step's motion table, carried by the launch
};

template <int R, int ROWS>
struct Geo {
  static constexpr int SW = TW + 2 * R;          // S tile width
  static constexpr int SH = ROWS + 2 * R;        // S tile height
  // TMA box width: TW+2R+1 source columns plus one for the even-aligned
  // origin (TMA needs 16-B aligned inner coordinates), rounded to 16 B
  static constexpr int BW = (TW + 2 * R + 1 + 1) & ~1;
  static constexpr int BH = ROWS + 2 * R + 1;    // TMA box height
  static constexpr int B_ELEMS = BW * BH;
  static constexpr uint32_t B_BYTES = B_ELEMS * 8;   // TMA transaction bytes
  static constexpr int STAGE = (B_ELEMS + 15) & ~15;  // 128-B aligned stages
  static constexpr int S_ELEMS = SW * SH;
};

// Per-channel bilinear weights from the motion vector (belief_tensor.cpp:
// 87-98); integral shifts copy exactly (:71-86).
struct ChanShift {
  double w00, w10, w01, w11;
  int sx, sy;
  bool integral;
};

__device__ __forceinline__ ChanShift chan_shift(double2 mv) {
  ChanShift s;
  const double fx = floor(mv.x), fy = floor(mv.y);
  s.integral = (fx == mv.x) && (fy == mv.y);
  const double ax = mv.x - fx, ay = mv.y - fy;
  s.w00 = (1.0 - ax) * (1.0 - ay);
  s.w10 = ax * (1.0 - ay);
  s.w01 = (1.0 - ax) * ay;
  s.w11 = ax * ay;
  // far-out shifts only ever read zeros; clamp keeps the int conversion sane
  const double lim = 1073741824.0;
  s.sx = static_cast<int>(fmin(fmax(fx, -lim), lim));
  s.sy = static_cast<int>(fmin(fmax(fy, -lim), lim));
  return s;
}

// One S cell from the four box taps: r0 = (lj+1), r1 = lj, c0 = (li+1),
// c1 = li. Order w00, w10, w01, w11 from 0.0 (belief_tensor.cpp:112-120).
template <bool SCALED>
__device__ __forceinline__ double s_cell(const ChanShift& cs, double sc,
                                         double r0c0, double r0c1, double r1c0,
                                         double r1c1) {
  if (SCALED) {
    r0c0 = r0c0 * sc;
    r0c1 = r0c1 * sc;
    r1c0 = r1c0 * sc;
    r1c1 = r1c1 * sc;
  }
  if (cs.integral) return r0c0;
  double acc = 0.0;
  acc += cs.w00 * r0c0;
  acc += cs.w10 * r0c1;
  acc += cs.w01 * r1c0;
  acc += cs.w11 * r1c1;
  return acc;
}

template <int R, int ROWS, bool SCALED>
__device__ __forceinline__ void compute_s_tile(
    const double* __restrict__ Bb, double* __restrict__ Sb,
    const uint8_t* __restrict__ occ_sh, const ChanShift& cs, double sc,
    uint32_t own_mask, int tid) {
  using G = Geo<R, ROWS>;
  // own column li = tid + R, rolled down the rows: 2 new smem loads per row
  const int li = tid + R;
  double lo_c1 = Bb[li], lo_c0 = Bb[li + 1];  // box row 0 (= r1 of lj = 0)
#pragma unroll
  for (int lj = 0; lj < G::SH; ++lj) {
    const double hi_c1 = Bb[(lj + 1) * G::BW + li];
    const double hi_c0 = Bb[(lj + 1) * G::BW + li + 1];
    double s = s_cell<SCALED>(cs, sc, hi_c0, hi_c1, lo_c0, lo_c1);
    if ((own_mask >> lj) & 1u) s = 0.0;
    Sb[lj * G::SW + li] = s;
    lo_c1 = hi_c1;
    lo_c0 = hi_c0;
  }
  if (R > 0) {
    // halo columns [0, R) and [TW+R, TW+2R): 2R*SH cells, one per thread
    constexpr int NH = 2 * R * G::SH;
    for (int q = tid; q < NH; q += TW) {
      const int side = q / (R * G::SH);
      const int rem = q % (R * G::SH);
      const int hc = rem / G::SH;
      const int lj = rem % G::SH;
      const int col = side == 0 ? hc : TW + R + hc;
      double s = s_cell<SCALED>(cs, sc, Bb[(lj + 1) * G::BW + col + 1],
                                Bb[(lj + 1) * G::BW + col],
                                Bb[lj * G::BW + col + 1], Bb[lj * G::BW + col]);
      if (occ_sh[lj * G::SW + col]) s = 0.0;
      Sb[lj * G::SW + col] = s;
    }
  }
}

template <int R, int H, int ROWS, int NS>
__global__ void __launch_bounds__(TW, 7)
    k_fused_step(const __grid_constant__ CUtensorMap tmap,
                 const FusedParams p) {
  using G = Geo<R, ROWS>;
  constexpr int NG = 2 * H + 1;  // ring depth == angular taps
  extern __shared__ unsigned char smem_raw[];
  // TMA destinations must be 128-B aligned: align the dynamic base by hand
  unsigned char* smem_base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  double* Bs = reinterpret_cast<double*>(smem_base);             // NS boxes
  double* Ss = Bs + NS * G::STAGE;                             // 2 S tiles
  uint8_t* occ_sh = reinterpret_cast<uint8_t*>(Ss + (R > 0 ? 2 * G::S_ELEMS : 0));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(occ_sh + G::S_ELEMS) + 15) & ~uintptr_t(15));
  double* wmax = reinterpret_cast<double*>(mbar + NS);  // TW/32 warp maxima

  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * TW;
  const int y0 = blockIdx.y * ROWS;
  const int W = p.w, Hh = p.h, C = p.c;
  const size_t plane = static_cast<size_t>(W) * Hh;
  const int n_iter = C + 2 * H;

  auto issue = [&](int it, int stage) {
    const int m = it - H;
    const int kc = ((m % C) + C) % C;
    const ChanShift cs = chan_shift(p.param_motion ? p.mv[kc] : p.motion[kc]);
    mbar_arrive_expect(&mbar[stage], G::B_BYTES);
    // the innermost TMA coordinate must be 16-B aligned (an even double
    // index): round the box origin down; the consumer skips the odd column
    tma_load_3d(Bs + stage * G::STAGE, &tmap, (x0 - cs.sx - 1 - R) & ~1,
                y0 - cs.sy - 1 - R, kc, &mbar[stage]);
  };

  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    for (int s = 0; s < NS; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < NS && s < n_iter; ++s) issue(s, s);
  }
  // occupancy of the S tile (outside the grid counts as masked)
  for (int q = tid; q < G::S_ELEMS; q += TW) {
    const int lj = q / G::SW, li = q % G::SW;
    const int i = x0 + li - R, j = y0 + lj - R;
    occ_sh[q] = (i < 0 || i >= W || j < 0 || j >= Hh)
                    ? 1
                    : p.occ[static_cast<size_t>(j) * W + i];
  }
  const bool scaled = p.src_state->scaled != 0;
  const double sc = scaled ? p.src_state->scale : 1.0;
  __syncthreads();

  // own column: S mask bits (lj) and output mask bits (row r = lj - R)
  uint32_t own_mask = 0;
#pragma unroll
  for (int lj = 0; lj < G::SH; ++lj) {
    own_mask |= static_cast<uint32_t>(occ_sh[lj * G::SW + tid + R] != 0) << lj;
  }
  const int gi = x0 + tid;
  const bool col_in = gi < W;

  double ring[NG][ROWS];
  double vmax = 0.0;

  for (int base = 0; base < n_iter; base += NG) {
#pragma unroll
    for (int u = 0; u < NG; ++u) {
      const int it = base + u;
      if (it >= n_iter) break;
      const int stage = it % NS;
      const int m = it - H;
      const int kc = ((m % C) + C) % C;
      const ChanShift cs = chan_shift(p.param_motion ? p.mv[kc] : p.motion[kc]);
      mbar_wait(&mbar[stage], static_cast<uint32_t>((it / NS) & 1));
      const double* Bb = Bs + stage * G::STAGE + ((x0 - cs.sx - 1 - R) & 1);

      if constexpr (R == 0) {
        // rotation-only kernels: no spatial diffusion, S == D
        const int li = tid;
        double lo_c1 = Bb[li], lo_c0 = Bb[li + 1];
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          const double hi_c1 = Bb[(r + 1) * G::BW + li];
          const double hi_c0 = Bb[(r + 1) * G::BW + li + 1];
          double s = scaled ? s_cell<true>(cs, sc, hi_c0, hi_c1, lo_c0, lo_c1)
                            : s_cell<false>(cs, sc, hi_c0, hi_c1, lo_c0, lo_c1);
          if ((own_mask >> r) & 1u) s = 0.0;
          ring[u][r] = s;
          lo_c1 = hi_c1;
          lo_c0 = hi_c0;
        }
        __syncthreads();  // stage fully consumed
        if (tid == 0 && it + NS < n_iter) issue(it + NS, stage);
      } else {
        double* Sb = Ss + (it & 1) * G::S_ELEMS;
        if (scaled) {
          compute_s_tile<R, ROWS, true>(Bb, Sb, occ_sh, cs, sc, own_mask, tid);
        } else {
          compute_s_tile<R, ROWS, false>(Bb, Sb, occ_sh, cs, sc, own_mask, tid);
        }
        __syncthreads();  // S complete; stage fully consumed
        if (tid == 0 && it + NS < n_iter) issue(it + NS, stage);
        // row pass (belief_tensor.cpp:199-225) then column pass (:227-238)
        const int li = tid + R;
        double rr[G::SH];
#pragma unroll
        for (int lj = 0; lj < G::SH; ++lj) {
          const double* srow = Sb + lj * G::SW + li - R;
          double acc = 0.0;
#pragma unroll
          for (int d = 0; d < 2 * R + 1; ++d) acc += p.sep[d] * srow[d];
          rr[lj] = acc;
          if (lj >= 2 * R) {
            const int r = lj - 2 * R;
            double col = 0.0;
#pragma unroll
            for (int d = 0; d < 2 * R + 1; ++d) col += p.sep[d] * rr[r + d];
            ring[u][r] = col;
          }
        }
      }

      // output channel k = m - H (belief_tensor.cpp:440-475)
      if (m >= H) {
        const int k = m - H;
        double* out = p.dst + plane * k;
        const double* inv = p.inv + (p.inv_per_k ? plane * k : 0);
#pragma unroll
        for (int r = 0; r < ROWS; ++r) {
          double o = p.ang[0] * ring[u][r];
#pragma unroll
          for (int t = 1; t < NG; ++t) o += p.ang[t] * ring[(u - t + NG) % NG][r];
          const int gj = y0 + r;
          if (col_in && gj < Hh) {
            const size_t q = static_cast<size_t>(gj) * W + gi;
            if ((own_mask >> (r + R)) & 1u) {
              o = 0.0;
            } else {
              o = o * __ldg(inv + q);
              vmax = (o > 0.0) ? dmax_ref(vmax, o) : vmax;
            }
            out[q] = o;
          }
        }
      }
    }
  }

  // global max -> last CTA finalises status and the pending rescale
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vmax = dmax_ref(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  if ((tid & 31) == 0) wmax[tid >> 5] = vmax;
  __syncthreads();
  if (tid == 0) {
    double bm = 0.0;
    for (int q = 0; q < TW / 32; ++q) bm = dmax_ref(bm, wmax[q]);
    StepState* st = p.step_state;
    if (bm > 0.0) atomicMax(&st->gmax_bits, static_cast<unsigned long long>(__double_as_longlong(bm)));
    __threadfence();
    const unsigned int total = gridDim.x * gridDim.y;
    const unsigned int prev = atomicAdd(&st->blocks_done, 1u);
    if (prev == total - 1) {
      __threadfence();
      const unsigned long long bits = atomicAdd(&st->gmax_bits, 0ull);
      const double g = __longlong_as_double(static_cast<long long>(bits));
      st->status = (g <= 0.0) ? GL_E_EXTINGUISHED : GL_OK;
      if (g > 0.0 && g < 1e-6) {
        p.dst_state->scaled = 1;
        p.dst_state->scale = 1.0 / g;
      } else {
        p.dst_state->scaled = 0;
        p.dst_state->scale = 1.0;
      }
      st->gmax_bits = 0ull;
      st->blocks_done = 0u;
    }
  }
}

template <int R, int ROWS, int NS>
constexpr size_t smem_bytes() {
  using G = Geo<R, ROWS>;
  size_t b = NS * G::STAGE * 8 + (R > 0 ? 2 * G::S_ELEMS * 8 : 0) + G::S_ELEMS;
  b = (b + 15) & ~size_t(15);
  return 128 + b + NS * 8 + (TW / 32) * 8;  // + alignment slack
}

template <int R, int H, int ROWS, int NS>
void launch_variant(gl_context* ctx, const CUtensorMap* tmap,
                    const FusedParams& fp) {
  constexpr size_t smem = smem_bytes<R, ROWS, NS>();
  auto kern = k_fused_step<R, H, ROWS, NS>;
  static uint64_t configured = 0;  // bit per device: the attribute is per device
  const uint64_t bit = 1ull << (ctx->device & 63);
  if (!(configured & bit)) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    configured |= bit;
  }
  dim3 grid((fp.w + TW - 1) / TW, (fp.h + ROWS - 1) / ROWS, 1);
  kern<<<grid, TW, smem, ctx->stream>>>(*tmap, fp);
  ctx->launches++;
}

template <int H>
constexpr int rows_for() {
  return H <= 1 ? 16 : 8;
}

template <int R, int H>
void launch_rh(gl_context* ctx, const CUtensorMap* tmap, const FusedParams& fp) {
  launch_variant<R, H, rows_for<H>(), 2>(ctx, tmap, fp);
}

template <int R>
void launch_r(gl_context* ctx, const CUtensorMap* tmap, const FusedParams& fp,
              int H) {
  switch (H) {
    case 0: launch_rh<R, 0>(ctx, tmap, fp); break;
    case 1: launch_rh<R, 1>(ctx, tmap, fp); break;
    case 2: launch_rh<R, 2>(ctx, tmap, fp); break;
    default: launch_rh<R, 3>(ctx, tmap, fp); break;
  }
}

}  // namespace

// The fused path covers the Localizer's two kernel sets at any channel
// count: separable (isotropic) or impulse spatial kernels with radius <= 2,
// and angular taps that are exactly offsets -H..H in ascending order (the
// unfolded build_kernels output, H <= 3) or the degenerate single tap.
bool fused_supported(int r, const AngTaps& ang, int c) {
  if (r < 0 || r > kFusedMaxRadius) return false;
  if (ang.n < 1 || ang.n > 2 * kFusedMaxHalf + 1 || (ang.n % 2) == 0) return false;
  const int H = ang.n / 2;
  for (int t = 0; t < ang.n; ++t) {
    if (ang.off[t] != t - H) return false;
  }
  return c >= 1;
}

// TMA box (width, height) in doubles for a fused variant; the host encodes
// the tensor map with it.
void fused_box(int r, int H, int* bw, int* bh) {
  const int rows = H <= 1 ? rows_for<1>() : rows_for<3>();
  *bw = (TW + 2 * r + 1 + 1) & ~1;
  *bh = rows + 2 * r + 1;
}

void launch_fused_step(gl_context* ctx, const StepArgs& a,
                       const CUtensorMap* tmap, const double* sep, int r,
                       const AngTaps& ang) {
  FusedParams fp{};
  fp.dst = a.dst;
  fp.motion = a.motion;
  fp.param_motion = (a.c <= kParamChannels && a.h_motion != nullptr) ? 1 : 0;
  if (fp.param_motion) {
    for (int k = 0; k < a.c; ++k) fp.mv[k] = make_double2(a.h_motion[2 * k], a.h_motion[2 * k + 1]);
  }
  fp.occ = a.occ;
  fp.inv = a.inv;
  fp.inv_per_k = a.inv_per_channel;
  fp.w = a.w;
  fp.h = a.h;
  fp.c = a.c;
  fp.src_state = a.src_state;
  fp.dst_state = a.dst_state;
  fp.step_state = a.step_state;
  for (int t = 0; t < 2 * r + 1; ++t) fp.sep[t] = sep[t];
  for (int t = 0; t < ang.n; ++t) fp.ang[t] = ang.w[t];
  const int H = ang.n / 2;
  switch (r) {
    case 0: launch_r<0>(ctx, tmap, fp, H); break;
    case 1: launch_r<1>(ctx, tmap, fp, H); break;
    default: launch_r<2>(ctx, tmap, fp, H); break;
  }
}

}  // namespace glb
