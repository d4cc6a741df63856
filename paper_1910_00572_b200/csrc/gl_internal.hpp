// Internal types shared by the host runtime (capi.cpp, host_math.cpp) and
// the CUDA kernels (k_*.cu). Not part of the public C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <cuda.h>

#include <cstdint>
#include <string>
#include <vector>

#include "gridloc_b200.h"

namespace glb {

constexpr int kMaxSepTaps = 63;      // separable taps held in kernel params
constexpr int kParamChannels = 384;  // fused path: motion vectors ride in the launch params
constexpr int kFusedMaxHalf = 3;     // fused path: angular offsets in [-3, 3]
constexpr int kFusedMaxRadius = 2;   // fused path: separable radius <= 2 (or 0)

// Per-buffer "pending rescale" (belief_tensor.cpp:486-493). The step that
// produced a buffer records whether its global max fell below 1e-6; the
// multiply by 1/max is folded into the next reader's load (bit-identical:
// the reader computes value*scale exactly where the reference stored it).
struct BufState {
  double scale;  // valid when scaled != 0
  int scaled;
  int pad;
};

// Step reduction scratch on the device. gmax_bits holds the running global
// maximum as uint64 bits (valid ordering for non-negative doubles); the last
// CTA to finish turns it into the status + the next buffer's BufState.
struct StepState {
  unsigned long long gmax_bits;
  unsigned int blocks_done;
  int status;  // GL_OK or GL_E_EXTINGUISHED for the latest step
  // high-word max mode (fused FAST steps): the step kernel tracks only the
  // high 32 bits of the max; when they cannot decide max >= 1e-6 the last
  // CTA sets need_exact and the step epilogue kernel takes the exact max
  int need_exact;
  int pad;
};

// Every step-finalising kernel publishes the status through this; `host` is
// the launching context's mapped pinned status word for a synchronous
// gl_step (it then needs no device-to-host copy), else null.
__device__ __forceinline__ void publish_status(StepState* st, int s, int* host) {
  st->status = s;
  if (host) *reinterpret_cast<volatile int*>(host) = s;
}

struct DeviceBlock {  // one allocation per tensor
  BufState buf[2];
  StepState step;
};

// Per-channel bilinear shift record of one step (belief_tensor.cpp:87-98),
// computed on the host in the reference's operation order: box origin
// (floor of the motion vector), the four weights, and whether the shift is
// integral (the exact-copy branch, :71-86). Fused launches carry the step's
// table in their parameters.
struct ChanRec {
  double w00, w10, w01, w11;
  int ox, oy;             // floor(dx), floor(dy), clamped to +-2^29
  int integral : 8;       // round(dx) == dx && round(dy) == dy
  int map : 8;            // fused launch: 0 own buffer, 1 / 2 left / right neighbour's
  int wall : 8;           // fused launch with the wall-crossing mask: entry of FusedParams::wall
  int z;                  // fused launch: source plane in that buffer
};
void chan_rec(double dx, double dy, ChanRec* r);  // host_math.cpp

// Angular taps (belief_tensor.hpp:82): (offset, weight) in list order.
struct AngTaps {
  int n;
  int off[2 * kFusedMaxHalf + 1];
  double w[2 * kFusedMaxHalf + 1];
};

}  // namespace glb

struct gl_context {
  int device = 0;
  int sm_count = 0;  // multiprocessors of `device` (fused-step grid sizing)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  int path = GL_PATH_AUTO;
  bool allow_fast = true;  // use the FAST fused variant on clean buffers
  int himax_mode = 0;      // high-word step max: 0 auto (large tensors), 1 always, 2 never
  int channel_chunks = 0;  // fused step channel chunks: 0 auto, n >= 1 fixed
  int tail_ctas = -1;      // fused step wave-tail split: -1 auto, 0 off, n CTAs
  int tail_chunks = 3;     // channel chunks of each wave-tail CTA's tiles
  int strip_tiles = -1;    // fused step tile order: -1 auto, 0 row-major, n: vertical strips n tiles wide
  int tile_stack = 0;      // fused step: 0/1 a CTA's warps take side-by-side tiles, n: n stacked vertically
  bool host_exp = true;    // likelihood geometric mean: exp by host glibc (exact)
  bool wall_mask = false;  // step phase 1: also drop taps whose motion segment crosses a wall (extension)
  void* d_kind = nullptr;  // likelihood case codes
  size_t kind_bytes = 0;
  uint64_t launches = 0;
  // generic-path scratch (S and D tensors), grown on demand
  double* d_s = nullptr;
  double* d_d = nullptr;
  size_t scratch_elems = 0;
  // motion-vector upload ring (pinned host -> device), one slot per step
  static constexpr int kRing = 32;
  double* h_motion = nullptr;  // pinned, kRing * cap * 2
  double* d_motion = nullptr;  // device, kRing * cap * 2
  cudaEvent_t ring_ev[kRing] = {};
  int ring_cap = 0;
  int ring_next = 0;
  // pinned scalars for status read-back
  glb::DeviceBlock* h_block = nullptr;
  int* h_status = nullptr;  // mapped pinned status word (host view) ...
  int* d_status = nullptr;  // ... and its device address
  // misc device scratch for reductions / dither
  void* d_misc = nullptr;
  size_t misc_bytes = 0;
  void* h_misc = nullptr;  // pinned mirror of d_misc
  size_t h_misc_bytes = 0;
  // optional per-launch step timing (event pairs)
  static constexpr int kTimers = 8192;
  bool timing = false;
  bool step_events = false;  // begin/end events around every step (t_motion)
  std::vector<cudaEvent_t> tev;  // 2 * kTimers
  int tcount = 0;
  int tstride = 1;     // time every tstride-th step
  unsigned tstep = 0;  // steps since timing was enabled
  cudaEvent_t ev_begin_last = nullptr, ev_end_last = nullptr;
  cudaEvent_t marks[16] = {};
};

struct gl_map {
  int w = 0, h = 0;
  double res = 0.1, ox = 0.0, oy = 0.0;
  int free_count = 0;
  std::vector<uint8_t> occ;  // host copy, 1 = occupied
  uint8_t* d_occ = nullptr;
  int device = 0;
};

struct gl_field {
  int w = 0, h = 0;
  std::vector<double> values;  // meters
  double* d_values = nullptr;
  // per-cell beam log-score table for one LikelihoodParams (host libm),
  // owned by the field so it dies with it
  double score_sigma = -1.0, score_floor = -1.0, score_oob = 0.0;
  double* d_score = nullptr;
};

struct gl_kernels {
  gl_kernel_info info{};
  std::vector<double> sep;
  std::vector<double> spatial;  // channels*(2r+1)^2
  std::vector<int> ang_off;
  std::vector<double> ang_w;
  // device copies (lazily uploaded per device)
  int device = -1;
  double* d_spatial = nullptr;
  int* d_ang_off = nullptr;
  double* d_ang_w = nullptr;
};

struct gl_activation {
  int w = 0, h = 0, channels = 0;
  bool k_invariant = false;  // one W*H plane serves every channel
  double* d_values = nullptr;
  double* d_inverse = nullptr;
  double* d_inverse_masked = nullptr;  // k-invariant: inverse, 0.0 where occupied
};

struct gl_tensor {
  int w = 0, h = 0, c = 0;  // c = channels held (a shard's interior planes)
  // theta-slab shard: this tensor holds global channels
  // [c_begin, c_begin + c) of c_total, stored with `halo` neighbour planes on
  // each side: storage plane q <-> channel (c_begin - halo + q) mod c_total.
  int halo = -1;  // -1: a whole (unsharded) tensor
  int c_total = 0, c_begin = 0;
  double cell = 0.1, ox = 0.0, oy = 0.0;
  double theta_t = 0.0;
  double* d_buf[2] = {nullptr, nullptr};
  int cur = 0;
  // "clean": every value finite and >= +0.0 (no -0.0). init_uniform and a
  // zero tensor are clean; every kernel of this library maps clean input to
  // clean output; uploads are scanned. Enables the FAST fused variant.
  bool clean[2] = {true, true};
  glb::DeviceBlock* d_block = nullptr;
  int device = 0;
  CUtensorMap tmap[2];  // 3-D TMA descriptors over d_buf[0/1]
  bool tmap_ok = false;
  // shard peers (gl_shard_set_peers): the neighbours' ping-pong buffers
  // (storage plane 0) and their interior channel counts
  double* peer_lo_buf[2] = {nullptr, nullptr};
  double* peer_hi_buf[2] = {nullptr, nullptr};
  int peer_lo_count = 0, peer_hi_count = 0;
};

// ---------------------------------------------------------------- launchers
// (defined in the .cu files; all enqueue on ctx->stream)
namespace glb {

struct SepTaps {
  double t[kMaxSepTaps];
};

struct StepArgs {
  const double* src;       // input buffer (C planes)
  double* dst;             // output buffer
  const BufState* src_state;
  BufState* dst_state;
  StepState* step_state;
  const double2* motion;   // per channel (dx, dy) in cells (device)
  const double* h_motion;  // same table on the host (fused path: params)
  const uint8_t* occ;
  const double* inv;       // activation inverse
  const double* inv_masked;  // same with occupied cells 0.0 (k-invariant only)
  int inv_per_channel;     // 0: one plane for all k
  int w, h, c;             // c = output channels (a shard's interior planes)
  int halo = -1;           // theta-slab shard: halo planes per side; -1 = whole tensor
  bool full_shard = false; // the shard holds all channels (one rank): no cross-rank max
  // theta-slab shard with peers: the step reads its halo input planes
  // straight from the neighbours' buffers (TMA over peer memory)
  const CUtensorMap* tmap_lo = nullptr;  // left neighbour's source buffer
  const CUtensorMap* tmap_hi = nullptr;  // right neighbour's source buffer
  int lo_add = 0;                        // left neighbour's interior channel count
  const double* src_lo = nullptr;        // the neighbours' source buffers (storage plane 0)
  const double* src_hi = nullptr;
  int* host_status = nullptr;            // mapped status word (synchronous gl_step)
  bool wall = false;                     // the wall-crossing mask (wall.hpp; an extension, off by default)
};

// k_generic.cu
void launch_shift_mask(gl_context* ctx, const StepArgs& a, double* S, int mode);
void launch_conv_separable(gl_context* ctx, const double* S, double* tmp,
                           double* D, int w, int h, int c, const SepTaps& taps,
                           int r);
void launch_conv_dense(gl_context* ctx, const double* S, double* D, int w,
                       int h, int c, const double* d_spatial, int r,
                       int kernel_channels);
void launch_angular(gl_context* ctx, const StepArgs& a, const double* D,
                    const int* d_off, const double* d_w, int n_ang);
void launch_step_finalize(gl_context* ctx, const StepArgs& a);
void launch_apply_scale(gl_context* ctx, double* buf, size_t n,
                        BufState* state);
void launch_fill(gl_context* ctx, double* buf, size_t n, double v);
void launch_to_f32(gl_context* ctx, const double* in, float* out, size_t n);
void launch_from_f32(gl_context* ctx, const float* in, double* out, size_t n);
void launch_init_uniform(gl_context* ctx, double* buf, const uint8_t* occ,
                         int w, int h, int c);
void launch_make_activation(gl_context* ctx, const uint8_t* occ, int w, int h,
                            int c, const gl_kernels* k, double* values,
                            double* inverse, bool k_invariant, double* scratch);
void launch_distance_field(gl_context* ctx, const uint8_t* d_occ, int w, int h, double res,
                           double* d_out, void* d_scratch);
size_t distance_field_scratch_bytes(int w, int h);
void launch_belief_map(gl_context* ctx, const double* buf, int w, int h,
                       int c, double* out);
void launch_mask_plane(gl_context* ctx, const double* in, const uint8_t* occ,
                       size_t plane, double* out);
size_t argmax_scratch_bytes(size_t n);
void launch_argmax(gl_context* ctx, const double* buf, size_t n,
                   void* d_scratch, size_t scratch_bytes, void* d_out);
// order-independent hash of buf[0..n) as the elements p0 .. p0+n-1 of a
// larger tensor (shard hashes add up to the whole tensor's)
// gl_tensors_status: gather up to kStatusGather tensors' step status words
constexpr int kStatusGather = 64;
struct StatusPtrs {
  const int* p[kStatusGather];
  int n;
};
void launch_gather_status(gl_context* ctx, const StatusPtrs& ptrs, int* d_out);
void launch_hash(gl_context* ctx, const double* buf, size_t n,
                 unsigned long long* d_out, unsigned long long p0);
void launch_plane_max(gl_context* ctx, const double* buf, size_t n,
                      unsigned long long* d_gmax);

// k_fused.cu
bool fused_supported(int r, const double* sep, const AngTaps& ang, int c);
// the wall-crossing mask fits the fused kernel's table for these motion
// vectors (<= kWallEntries distinct floors per window, <= kWallSeg crossed
// cells per tap, within kWallReach); otherwise the generic chain runs it
bool fused_wall_fits(const double* h_motion, int n);
void fused_counters(unsigned long long* out4);  // diagnostics
void fused_box(int r, int H, int* bw, int* bh);
void launch_fused_step(gl_context* ctx, const StepArgs& a,
                       const CUtensorMap* tmap, const double* sep, int r,
                       const AngTaps& ang, bool fast);
// 1 if any value has its sign bit set or is not finite (buffer not "clean")
void launch_scan_unclean(gl_context* ctx, const double* buf, size_t n,
                         unsigned int* d_flag);

// k_engine.cu (the single-process multi-device engine, engine.cpp)
constexpr int kEngineMaxShards = 16;
struct PtrList {
  const void* p[kEngineMaxShards];
  int n;
};
// mailbox[slot] = the shard's step max bits (after its fused step)
void launch_engine_publish(gl_context* ctx, const unsigned long long* gmax, unsigned long long* mailbox);
// gmax = max over the shards' mailboxes (peer reads), for gl_shard_finalize
void launch_engine_gather(gl_context* ctx, const PtrList& mailboxes, unsigned long long* gmax);
// dst[p] = max(dst[p], src_s[p]) over the listed planes (peer reads)
void launch_plane_max_combine(gl_context* ctx, double* dst, const PtrList& srcs, size_t n);
void set_last_error(const std::string& msg);  // capi.cpp

// k_difficulty.cu (map_difficulty, evaluation.cpp:25-72)
constexpr int kMaxDifficultyBeams = 256;
struct DifficultyArgs {
  const uint8_t* occ;
  const double* score;     // per-cell beam log-score (host libm)
  double oob;              // log-score of an out-of-grid endpoint
  int w, h;
  double res, ox, oy;
  const int2* cells;       // query == candidate cells, reference order
  int n;
  const double2* ray;      // beams: (cos, sin) of the scan beam angles (pose theta 0)
  const double2* dir;      // bins x beams: (cos, sin) of test_angle + beam angle
  int beams, bins, stride;
  double max_range, half_cell;
  double* ranges;          // n x beams
  double* best_ls;         // n
  int* best_idx;           // n
  int* counted;            // n
  int* near;               // n (zeroed)
  int* bad;                // 1 (zeroed)
};
void launch_difficulty(gl_context* ctx, const DifficultyArgs& a);
// raycast / simulate_scan batches (occupancy_map.cpp:273-332, simulator.cpp:63-94)
void launch_raycast_batch(gl_context* ctx, const uint8_t* occ, int w, int h, double res, double ox, double oy,
                          const double2* xy, const double2* dir, int n_rays, int beams, double max_range,
                          const double* noise, double sigma, double* ranges, int* bad);

// k_observe.cu
void launch_dither(gl_context* ctx, const double* bm, int w, int h, int budget,
                   int* d_cells, int cap, int* d_n, double* d_mass, int* d_sum_invalid,
                   void* sum_scratch);
// k_seqsum.cu: the reference's sequential FP64 sum of x[0..n) from +0.0
// (observation.cpp:16-17, belief_tensor.cpp:517-522), bit-exact by a
// parallel binade scan; *d_invalid = 1 (and *d_total unspecified) if any x is
// negative or non-finite. _big runs the chunk passes on every SM first
// (scratch: seq_sum_scratch_bytes(n), 16-byte aligned).
// s0: the running sum the chain enters with (0.0; a previous shard's total).
void launch_seq_sum(gl_context* ctx, const double* x, size_t n, double* d_total, int* d_invalid, double s0 = 0.0);
size_t seq_sum_scratch_bytes(size_t n);
// d_argmax (optional, when seq_sum_fuses_argmax(n)): the chunk pass also
// writes argmax_state's candidate {value, flat index, unused} (the first
// maximum, values compared with a strict > from -1.0: k_argmax_partial's rule).
void launch_seq_sum_big(gl_context* ctx, const double* x, size_t n, double* d_total, int* d_invalid,
                        void* scratch, double s0 = 0.0, void* d_argmax = nullptr);
bool seq_sum_fuses_argmax(size_t n);
// the literal chain on one thread (inputs outside the scan's domain); runs
// only when *when != 0 (when == null: always)
void launch_seq_sum_chain(gl_context* ctx, const double* x, size_t n, double* d_total, const int* when,
                          double s0 = 0.0);
void launch_likelihoods(gl_context* ctx, const uint8_t* occ, const double* score,
                        double oob_score, int w, int h, double res, double ox,
                        double oy, double cell, double tox, double toy,
                        const int* d_samples, int n, int c,
                        const double2* d_dir, int n_scored,
                        const double* d_reach, double floor_w, double* d_L,
                        uint8_t* d_kind);
void launch_observe_apply(gl_context* ctx, double* buf, int w, int h, int c_local,
                          int k_off, int c_total, const int* d_samples, int n,
                          const double* d_L, double* d_mean, void* sum_scratch);  // seq_sum_scratch_bytes(n * c_total)
void launch_observe_finalize(gl_context* ctx, StepState* st, BufState* buf);

}  // namespace glb
