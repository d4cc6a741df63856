// Fused Algorithm-1 step, host side: launch_fused_step (shift records,
// channel windows, the wall table, the HIMAX epilogue) over the kernel
// templates of k_fused.cuh, whose (R, H, params) instantiations are compiled
// in k_fused_inst_r*_h*_{s,l}.cu.
#include "k_fused.cuh"

namespace glb {
namespace fk {
template <int R, int H, class P>
void launch_rh(gl_context* ctx, const CUtensorMap* const* tmap, P& fp, bool fast, bool himax, bool wall);
#define GL_FUSED_EXTERN2(R, H, P) \
  extern template void launch_rh<R, H, P>(gl_context*, const CUtensorMap* const*, P&, bool, bool, bool);
#define GL_FUSED_EXTERN(R, H) GL_FUSED_EXTERN2(R, H, FusedParams) GL_FUSED_EXTERN2(R, H, FusedParamsSmall)
GL_FUSED_EXTERN(0, 0) GL_FUSED_EXTERN(0, 1) GL_FUSED_EXTERN(0, 2) GL_FUSED_EXTERN(0, 3)
GL_FUSED_EXTERN(1, 0) GL_FUSED_EXTERN(1, 1) GL_FUSED_EXTERN(1, 2) GL_FUSED_EXTERN(1, 3)
GL_FUSED_EXTERN(2, 0) GL_FUSED_EXTERN(2, 1) GL_FUSED_EXTERN(2, 2) GL_FUSED_EXTERN(2, 3)
#undef GL_FUSED_EXTERN
#undef GL_FUSED_EXTERN2
}  // namespace fk

using namespace fk;

namespace {

// HIMAX step epilogue (launched after every HIMAX step, one CTA per SM):
// when the high-word max could not decide (max <= ~1e-6: the rescale branch,
// or an extinguished belief — in the cmd_bench stream the rescale fires every
// ~50 steps) it takes the exact max of the output at full HBM bandwidth with
// the reference's std::max-from-0.0 rule and the last CTA finalises status and
// the pending 1/max rescale (belief_tensor.cpp:480-493). Otherwise every CTA
// exits at once. Every CTA reads the flag before it counts itself, so the last
// CTA's reset cannot race a late reader.
__device__ unsigned long long g_fused_counters[4];  // [0] exact HIMAX epilogues run

__global__ void __launch_bounds__(1024) k_himax_epilogue(const double* __restrict__ buf, size_t n,
                                                         StepState* st, BufState* dst,
                                                         int* host_status) {
  __shared__ int need;
  __shared__ double wm[32];
  if (threadIdx.x == 0) need = *static_cast<volatile int*>(&st->need_exact);
  __syncthreads();
  if (!need) return;
  double m = 0.0;
  const double2* b2 = reinterpret_cast<const double2*>(buf);  // n even (TMA needs even W)
  const size_t n2 = n / 2;
  for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n2;
       q += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double2 v = b2[q];
    m = dmax_ref(m, v.x);
    m = dmax_ref(m, v.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = dmax_ref(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double bm = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) bm = dmax_ref(bm, wm[w]);
    if (bm > 0.0) atomicMax(&st->gmax_bits, static_cast<unsigned long long>(__double_as_longlong(bm)));
    __threadfence();
    if (atomicAdd(&st->blocks_done, 1u) == gridDim.x - 1) {
      __threadfence();
      const double g = __longlong_as_double(static_cast<long long>(atomicAdd(&st->gmax_bits, 0ull)));
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
      st->need_exact = 0;
      atomicAdd(&g_fused_counters[0], 1ull);
    }
  }
}

template <int R, class P>
void launch_r(gl_context* ctx, const CUtensorMap* const* tmap, P& fp, int H,
              bool fast, bool himax, bool wall) {
  switch (H) {
    case 0: launch_rh<R, 0, P>(ctx, tmap, fp, fast, himax, wall); break;
    case 1: launch_rh<R, 1, P>(ctx, tmap, fp, fast, himax, wall); break;
    case 2: launch_rh<R, 2, P>(ctx, tmap, fp, fast, himax, wall); break;
    default: launch_rh<R, 3, P>(ctx, tmap, fp, fast, himax, wall); break;
  }
}

// One window's wall table: an entry per distinct (floor dx, floor dy) of its
// records, holding the crossed cells of the four bilinear taps
// (w00: (ox, oy), w10: (ox + 1, oy), w01: (ox, oy + 1), w11: (ox + 1, oy + 1))
// relative to the destination. fused_wall_fits() vetted the sizes.
void wall_table(FusedParams& fp, int n_rec) {
  int n_ent = 0;
  int eox[kWallEntries], eoy[kWallEntries];
  for (int q = 0; q < n_rec; ++q) {
    ChanRec& rc = fp.rec[q];
    int e = 0;
    while (e < n_ent && (eox[e] != rc.ox || eoy[e] != rc.oy)) ++e;
    if (e == n_ent) {
      eox[e] = rc.ox;
      eoy[e] = rc.oy;
      WallEntry& we = fp.wall[e];
      for (int t = 0; t < 4; ++t) {
        int qx[kWallSeg], qy[kWallSeg];
        const int n = wall_seg_cells(rc.ox + (t & 1), rc.oy + (t >> 1), qx, qy, kWallSeg);
        we.n[t] = static_cast<uint8_t>(n);
        for (int m = 0; m < n; ++m) we.cell[t][m] = static_cast<uint8_t>((qx[m] + 8) | ((qy[m] + 8) << 4));
      }
      ++n_ent;
    }
    rc.wall = e;
  }
}

}  // namespace

bool fused_wall_fits(const double* h_motion, int n) {
  // distinct floors over ALL planes bound every window's count
  int n_ent = 0;
  long long eox[kWallEntries], eoy[kWallEntries];
  for (int q = 0; q < n; ++q) {
    const double fx = std::floor(h_motion[2 * q]), fy = std::floor(h_motion[2 * q + 1]);
    if (!(std::fabs(fx) <= kWallReach && std::fabs(fy) <= kWallReach)) return false;
    const long long ox = static_cast<long long>(fx), oy = static_cast<long long>(fy);
    int e = 0;
    while (e < n_ent && (eox[e] != ox || eoy[e] != oy)) ++e;
    if (e < n_ent) continue;
    if (n_ent == kWallEntries) return false;
    eox[n_ent] = ox;
    eoy[n_ent] = oy;
    ++n_ent;
    for (int t = 0; t < 4; ++t) {
      int qx[kWallSeg], qy[kWallSeg];
      const int c = wall_seg_cells(static_cast<int>(ox) + (t & 1), static_cast<int>(oy) + (t >> 1), qx, qy,
                                   kWallSeg);
      if (c > kWallSeg) return false;
      for (int m = 0; m < c; ++m) {
        if (qx[m] < -kWallReach || qx[m] > kWallReach || qy[m] < -kWallReach || qy[m] > kWallReach) return false;
      }
    }
  }
  return true;
}

// The fused path covers the Localizer's two kernel sets at any channel
// count: separable (isotropic) or impulse spatial kernels with radius <= 2,
// and angular taps that are exactly offsets -H..H in ascending order (the
// unfolded build_kernels output, H <= 3) or the degenerate single tap.
// Both tap sets must be symmetric bit for bit (w[t] == w[n-1-t]; always so
// for build_kernels output, which evaluates exp(-0.5*d*d/..) at d and -d):
// the kernel shares each product between the two taps that use it.
bool fused_supported(int r, const double* sep, const AngTaps& ang, int c) {
  if (r < 0 || r > kFusedMaxRadius) return false;
  if (ang.n < 1 || ang.n > 2 * kFusedMaxHalf + 1 || (ang.n % 2) == 0) return false;
  const int H = ang.n / 2;
  for (int t = 0; t < ang.n; ++t) {
    if (ang.off[t] != t - H) return false;
    if (std::memcmp(&ang.w[t], &ang.w[ang.n - 1 - t], sizeof(double)) != 0) return false;
  }
  for (int t = 0; r > 0 && t < 2 * r + 1; ++t) {
    if (std::memcmp(&sep[t], &sep[2 * r - t], sizeof(double)) != 0) return false;
  }
  return c >= 1;
}

// TMA box (width, height) in doubles for a fused variant; the host encodes
// the tensor map with it.
void fused_box(int r, int H, int* bw, int* bh) {
  const int rows = H <= 1 ? rows_for<1>() : rows_for<3>();
  *bw = 34;
  *bh = rows + 2 * r + 1;
}

void fused_counters(unsigned long long* out4) {
  cudaMemcpyFromSymbol(out4, g_fused_counters, sizeof(unsigned long long) * 4);
}

namespace {

// One step's launches with parameter block P (see FusedHeader): records,
// channel windows of P::kRec - 2H output channels, the wall table.
template <class P>
void fused_step_with(gl_context* ctx, const StepArgs& a, const CUtensorMap* tmap, const double* sep, int r,
                     const AngTaps& ang, bool fast) {
  // kept off the stack and not re-zeroed per step (every field the kernel
  // reads is assigned below; unused record slots are never read)
  static thread_local P fp;
  const int H = ang.n / 2;
  fp.dst = a.dst;
  fp.occ = a.occ;
  fp.inv = a.inv;
  fp.inv_masked = a.inv_masked;
  fp.inv_per_k = a.inv_per_channel;
  fp.w = a.w;
  fp.h = a.h;
  fp.c = a.c;
  fp.shard = a.halo >= 0 ? 1 : 0;
  fp.plane_off = a.halo - H;
  fp.out_off = a.halo >= 0 ? a.halo : 0;
  fp.src_state = a.src_state;
  fp.dst_state = a.dst_state;
  fp.step_state = a.step_state;
  fp.host_status = a.host_status;
  // shard with peers: storage planes s < halo are read from the left
  // neighbour's buffer (its plane s + lo_add), planes s >= halo + c from the
  // right neighbour's (plane s - c), through their own tensor maps
  const bool peer_read = a.src_lo != nullptr && a.src_hi != nullptr;
  const int halo = a.halo > 0 ? a.halo : 0;
  // tmap == nullptr: the cp.async load path (a row pitch TMA cannot stride)
  const CUtensorMap* maps[3] = {tmap, peer_read ? a.tmap_lo : tmap, peer_read ? a.tmap_hi : tmap};
  fp.src_base[0] = a.src;
  fp.src_base[1] = peer_read ? a.src_lo : a.src;
  fp.src_base[2] = peer_read ? a.src_hi : a.src;
  for (int t = 0; t < 2 * r + 1; ++t) fp.sep[t] = sep[t];
  for (int t = 0; t < ang.n; ++t) fp.ang[t] = ang.w[t];
  // The shift records ride in the launch parameters; more than
  // P::kRec - 2H output channels take several launches over channel
  // windows. Only the last one finalises the max (a shard never does: its
  // max goes to the cross-rank all-reduce first).
  // high-word max for clean buffers whose step finalises on this device
  // (a partial theta-shard's max goes to the cross-rank all-reduce exact),
  // on tensors large enough that the epilogue launch (~3 us) is noise:
  // measured 4096^2 x 360 25.05 vs 25.78 ms; 1024^2 x 72 0.258 vs 0.255 ms
  const size_t elems = static_cast<size_t>(a.w) * a.h * a.c;
  const bool himax = GL_FUSED_HIMAX && fast && tmap != nullptr && !a.wall && (!fp.shard || a.full_shard) &&
                     (ctx->himax_mode == 1 || (ctx->himax_mode == 0 && elems >= (size_t(1) << 27)));
  const int win = P::kRec - 2 * H;
  for (int kb = 0; kb < a.c; kb += win) {
    const int ke = std::min(a.c, kb + win);
    fp.k_base = kb;
    fp.k_end = ke;
    // a shard holding every channel (one rank) finalises in the kernel too
    fp.defer_finalize = ((fp.shard && !a.full_shard) || ke < a.c) ? 1 : 0;
    for (int q = 0; q < ke - kb + 2 * H; ++q) {
      // h_motion: one (dx, dy) per channel (whole tensor) or per storage
      // plane (shard: plane q <-> channel c_begin - halo + q)
      int src, z, map = 0;
      if (fp.shard) {
        src = z = fp.plane_off + kb + q;  // storage plane
        if (peer_read && z < halo) {
          map = 1;
          z += a.lo_add;
        } else if (peer_read && z >= halo + a.c) {
          map = 2;
          z -= a.c;
        }
      } else {
        src = kb - H + q;  // circular channel
        src = src < 0 ? src + a.c : (src >= a.c ? src - a.c : src);
        z = src;
      }
      chan_rec(a.h_motion[2 * src], a.h_motion[2 * src + 1], &fp.rec[q]);
      fp.rec[q].z = z;
      fp.rec[q].map = map;
    }
    if constexpr (P::kWall > 0) {
      if (a.wall) wall_table(fp, ke - kb + 2 * H);
    }
    switch (r) {
      case 0: launch_r<0>(ctx, maps, fp, H, fast, himax, a.wall); break;
      case 1: launch_r<1>(ctx, maps, fp, H, fast, himax, a.wall); break;
      default: launch_r<2>(ctx, maps, fp, H, fast, himax, a.wall); break;
    }
  }
  if (himax) {
    const size_t plane = static_cast<size_t>(a.w) * a.h;
    k_himax_epilogue<<<ctx->sm_count > 0 ? ctx->sm_count : 148, 1024, 0, ctx->stream>>>(
        a.dst + plane * fp.out_off, plane * a.c, a.step_state, a.dst_state, a.host_status);
    ctx->launches++;
  }
}

}  // namespace

void launch_fused_step(gl_context* ctx, const StepArgs& a,
                       const CUtensorMap* tmap, const double* sep, int r,
                       const AngTaps& ang, bool fast) {
  // the ~5 KB parameter block when one launch holds every record and no
  // wall table is needed (Theta <= 90: configs[0..2] and [4]); launching it
  // costs less host time per step than the ~21 KB block
  const int H = ang.n / 2;
  if (!a.wall && a.c + 2 * H <= kSmallRec) {
    fused_step_with<FusedParamsSmall>(ctx, a, tmap, sep, r, ang, fast);
  } else {
    fused_step_with<FusedParams>(ctx, a, tmap, sep, r, ang, fast);
  }
}

}  // namespace glb
