/*
 * gridloc_b200 — C-ABI of the B200-native belief-tensor filter.
 *
 * Drop-in boundary for the reference `gridloc` C++ library's hot path
 * (/root/reference/proj/include/gridloc/ *.hpp). The reference has no FFI; its
 * boundary is the C++ API, so each entry point below names the reference
 * function it replaces (file:line). `include/gridloc_b200.hpp` re-exposes the
 * same calls with the reference's C++ signatures, and INTEGRATION.md shows the
 * switch a maintainer makes.
 *
 * Plain C types only (no torch / CUDA types in the signatures). Every call is
 * synchronous unless its name ends in _async; errors map 1:1 onto the
 * reference's exceptions (see gl_status). Objects are single-threaded, like
 * the reference's ThreadPool (thread_pool.hpp:47); distinct objects may be
 * used from different threads and devices.
 *
 * The belief tensor is device-resident FP64, layout [k][j][i] exactly as
 * BeliefTensor (belief_tensor.hpp:55-60,74).
 */
#ifndef GRIDLOC_B200_H
#define GRIDLOC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes <-> reference exceptions. */
typedef enum {
  GL_OK = 0,
  GL_E_EXTINGUISHED = 1, /* gridloc::BeliefExtinguishedError (belief_tensor.hpp:22-25) */
  GL_E_INVALID = 2,      /* std::invalid_argument */
  GL_E_MAP_PARSE = 3,    /* gridloc::MapParseError (occupancy_map.hpp:22-30) */
  GL_E_RUNTIME = 4,      /* std::runtime_error (I/O etc.) */
  GL_E_CUDA = 5,         /* CUDA runtime / driver failure (no reference analogue) */
} gl_status;

typedef struct gl_context gl_context;       /* replaces ThreadPool& + StepScratch& */
typedef struct gl_map gl_map;               /* OccupancyMap (occupancy_map.hpp:35-81) */
typedef struct gl_field gl_field;           /* DistanceField (occupancy_map.hpp:85-101) */
typedef struct gl_kernels gl_kernels;       /* KernelSet (belief_tensor.hpp:79-89) */
typedef struct gl_activation gl_activation; /* Activation (belief_tensor.hpp:93-96) */
typedef struct gl_tensor gl_tensor;         /* BeliefTensor (belief_tensor.hpp:30-75) */

/* Thread-local message for the last non-OK status. */
const char* gl_last_error(void);
/* Library / build identification: "gridloc_b200 <ver> sm_100a". */
const char* gl_version(void);

/* ---- context ------------------------------------------------------------
 * One CUDA device + one stream. Replaces the reference's ThreadPool (the
 * parallel substrate, thread_pool.hpp:15-50) and StepScratch
 * (belief_tensor.hpp:121-128). */
gl_status gl_context_create(int device, gl_context** out);
gl_status gl_context_destroy(gl_context* ctx);
gl_status gl_context_synchronize(gl_context* ctx);
/* Device-time of the last gl_step (ms), measured with CUDA events on the
 * context stream: the fused kernel has no phase boundaries, so the total is
 * reported as t_motion and t_diffusion = t_masking = 0.
 * Off by default (two event records cost ~5 us of host time per step);
 * gl_context_set_step_timing(ctx, 1) turns it on (the C++ ThreadPool does,
 * to fill StepScratch like the reference). */
gl_status gl_context_set_step_timing(gl_context* ctx, int enable);
gl_status gl_context_last_step_ms(gl_context* ctx, double* ms);
/* Path selection (GL_PATH_AUTO = fused when the kernel set allows it). */
enum { GL_PATH_AUTO = 0, GL_PATH_FUSED = 1, GL_PATH_GENERIC = 2 };
gl_status gl_context_set_path(gl_context* ctx, int path);
/* Fused-kernel variant on "clean" tensors (all values finite and >= +0.0,
 * which init_uniform and every library op preserve; uploads are scanned):
 * 1 (default) drops the bitwise no-op 0.0 seeds / copy selects; 0 always
 * runs the literal reference operation sequence. Results are identical. */
gl_status gl_context_set_fast(gl_context* ctx, int enable);
/* Step max in the fused FAST kernel: 0 = auto (high-word max on tensors of
 * >= 2^27 states, with an exact full-grid epilogue when it cannot decide
 * max >= 1e-6), 1 = always, 2 = never (exact max in the kernel). Results are
 * bit-identical in every mode. */
gl_status gl_context_set_himax(gl_context* ctx, int mode);
/* Channel chunks per fused-step launch: 0 = auto (a tensor whose tiles
 * cannot fill one wave of resident warps splits its channels, each chunk
 * recomputing its 2H angular neighbours), n >= 1 = exactly n (capped by the
 * channel count). Batches of small tensors stepped on concurrent streams
 * fill the GPU together: 1 avoids the recompute (64 x 512^2 x 72: 248 vs 239
 * batch-Hz). Results are bit-identical for every setting. */
gl_status gl_context_set_channel_chunks(gl_context* ctx, int n);
/* Wave-tail split of a one-chunk fused-step launch: the last `ctas` CTAs of
 * the grid (the partial last wave of resident CTAs) run their tiles' channels
 * in `chunks` chunks, so the tail drains in shorter work items. ctas = -1:
 * auto (the last ~1/5 of the partial wave, default chunks 3), 0: off.
 * Results are bit-identical for every setting. */
gl_status gl_context_set_wave_tail(gl_context* ctx, int ctas, int chunks);
/* Fused-step tile order: which tiles run side by side. strip_tiles 0 =
 * row-major (tile rows across the whole width); n >= 1 = vertical strips n
 * tiles wide, walked row by row inside a strip, so a tile's upper and lower
 * neighbours run within ~n warps of it and their shared halo rows are still
 * in L2 (at 4096^2 a full tile row is 137 tiles and the neighbour's rows
 * were evicted before it ran); -1 = auto. stack n >= 2: the warps of a CTA
 * take n vertically adjacent tiles (they run in lockstep) instead of n
 * side-by-side ones; 0 = auto. Results are bit-identical for every setting. */
gl_status gl_context_set_tile_order(gl_context* ctx, int strip_tiles, int stack);
/* Wall-crossing mask (an EXTENSION named by the north star, off by default;
 * the reference masks destination cells only, belief_tensor.cpp:414-416):
 * with enable = 1, step() also drops every bilinear tap whose straight
 * segment between source and destination cell centres passes through the
 * interior of an occupied cell (corner touches excepted), so no mass jumps
 * through a wall. Fused into the step kernel's shift stage (a per-warp
 * occupancy bit window; the per-channel crossed-cell lists come from the
 * host); steps whose motion the kernel's table cannot hold (|floor(d)| > 7,
 * > 8 crossed cells per tap, > 64 distinct floors) run the generic chain. Parity for this mode is
 * against the oracle's restatement (oracle/gl_oracle.c glo_step_wall). */
gl_status gl_context_set_wall_mask(gl_context* ctx, int enable);
/* scan_likelihood's final exp (the per-pose geometric mean,
 * observation.cpp:110): 1 (default) evaluates it with the host's libm like the
 * reference (bit-exact; one D2H/H2D of <= 512*Theta doubles per observation),
 * 0 with CUDA's exp on the device (<= 1 ulp). Everything else is device. */
gl_status gl_context_set_host_exp(gl_context* ctx, int enable);
/* Number of kernels this context launched since creation. */
gl_status gl_context_launch_count(gl_context* ctx, uint64_t* n);
/* The context's cudaStream_t, as an opaque pointer (for NCCL / events). */
gl_status gl_context_stream(gl_context* ctx, void** stream);
/* Per-launch device timing of the step kernels: enable = n >= 1 brackets
 * every n-th step kernel with CUDA events on the context stream (an event
 * pair costs ~5 us of host time, which short steps feel: sample them), 0
 * turns it off; *_times synchronises and returns the summed duration and
 * count of the timed kernels since the last call (then resets). */
gl_status gl_context_time_steps(gl_context* ctx, int enable);
gl_status gl_context_step_times(gl_context* ctx, double* total_ms, int* count);
/* Region timing on the context stream: record marker i (0..15), then read
 * the device time between two markers (synchronises). */
gl_status gl_context_mark(gl_context* ctx, int i);
gl_status gl_context_marks_ms(gl_context* ctx, int i, int j, double* ms);

/* ---- maps ------------------------------------------------------------- */
/* load_map (occupancy_map.hpp:106-108, occupancy_map.cpp:148-165): PGM P2/P5
 * decode, gray >= threshold is free, boundary ring forced occupied. Host-only
 * call: with occ == NULL writes dims only. PNG input -> GL_E_MAP_PARSE. */
gl_status gl_load_map(const uint8_t* bytes, size_t n, int threshold, int* width,
                      int* height, uint8_t* occ);
/* OccupancyMap ctor (occupancy_map.cpp:14-42): occ is copied, ring forced. */
gl_status gl_map_create(gl_context* ctx, int width, int height,
                        double resolution, double origin_x, double origin_y,
                        const uint8_t* occ, gl_map** out);
gl_status gl_map_destroy(gl_map* map);
gl_status gl_map_info(const gl_map* map, int* width, int* height,
                      double* resolution, double* origin_x, double* origin_y,
                      int* free_count);
gl_status gl_map_cells(const gl_map* map, uint8_t* occ_out);
/* distance_field (occupancy_map.hpp:117, occupancy_map.cpp:231-271). */
gl_status gl_field_create(gl_context* ctx, const gl_map* map, gl_field** out);
gl_status gl_field_destroy(gl_field* f);
gl_status gl_field_values(const gl_field* f, double* out);

/* ---- kernels / activation ------------------------------------------------
 * build_kernels (belief_tensor.cpp:243-338), evaluated on the host with the
 * same libm calls as the reference. */
typedef struct {
  int channels;   /* number of per-channel spatial kernels */
  int radius;     /* spatial half-width r */
  int separable;  /* isotropic: one 1-D tap vector */
  int degenerate_spatial;
  int degenerate_angular;
  int n_angular;  /* number of (offset, weight) angular taps */
} gl_kernel_info;

gl_status gl_build_kernels(double sigma_x, double sigma_y, double sigma_theta,
                           int channels, double cell_size, double delta_theta,
                           gl_kernels** out);
/* Wrap an explicit KernelSet (e.g. one built by the reference). sep has
 * 2r+1 taps (separable) ; spatial has channels*(2r+1)^2 weights (may be NULL
 * when separable); angular taps in list order. */
gl_status gl_kernels_create(gl_context* ctx, const gl_kernel_info* info,
                            const double* sep, const double* spatial,
                            const int* ang_off, const double* ang_w,
                            gl_kernels** out);
gl_status gl_kernels_destroy(gl_kernels* k);
gl_status gl_kernels_info(const gl_kernels* k, gl_kernel_info* info);
/* Copy taps out (any pointer may be NULL). */
gl_status gl_kernels_get(const gl_kernels* k, double* sep, double* spatial,
                         int* ang_off, double* ang_w);

/* make_activation (belief_tensor.cpp:354-394), computed on the device. */
gl_status gl_make_activation(gl_context* ctx, const gl_map* map,
                             const gl_kernels* kernels, int channels,
                             gl_activation** out);
gl_status gl_activation_destroy(gl_activation* a);
/* values / inverse are channels*W*H (either may be NULL). */
gl_status gl_activation_get(gl_context* ctx, const gl_activation* a,
                            double* values, double* inverse);

/* ---- tensors ---------------------------------------------------------- */
/* BeliefTensor ctor (belief_tensor.cpp:20-33): zero-filled. */
gl_status gl_tensor_create(gl_context* ctx, int width, int height,
                           int channels, double cell_size, double origin_x,
                           double origin_y, gl_tensor** out);
/* init_uniform (belief_tensor.cpp:35-53). */
gl_status gl_init_uniform(gl_context* ctx, const gl_map* map, int channels,
                          gl_tensor** out);
gl_status gl_tensor_destroy(gl_tensor* t);
gl_status gl_tensor_info(const gl_tensor* t, int* width, int* height,
                         int* channels, double* cell_size, double* origin_x,
                         double* origin_y);
gl_status gl_tensor_theta(const gl_tensor* t, double* theta_t);
gl_status gl_tensor_set_theta(gl_tensor* t, double theta_t);
/* Host <-> device copies of the whole tensor, [k][j][i] FP64. */
gl_status gl_tensor_upload(gl_context* ctx, gl_tensor* t, const double* host);
gl_status gl_tensor_download(gl_context* ctx, gl_tensor* t, double* host);
/* Element-range access, flat [k][j][i] offset (BeliefTensor::at / plane()). */
gl_status gl_tensor_read(gl_context* ctx, gl_tensor* t, size_t offset,
                         size_t count, double* host);
gl_status gl_tensor_write(gl_context* ctx, gl_tensor* t, size_t offset,
                          size_t count, const double* host);
/* Deep copy on the device (BeliefTensor is value-semantic in the reference,
 * test_belief_engine.cpp:353,385). */
gl_status gl_tensor_clone(gl_context* ctx, gl_tensor* src, gl_tensor** out);
/* Order-independent 64-bit hash of the tensor's bits, computed on the device:
 * sum over p of splitmix64(bits_p + p * 0x9e3779b97f4a7c15) (parity checks). */
gl_status gl_tensor_hash(gl_context* ctx, gl_tensor* t, uint64_t* hash);
/* The same hash of a theta-slab shard's interior taken as the elements
 * p0 .. p0+n-1 of the whole tensor: the shards' hashes add up (mod 2^64) to
 * the unsharded tensor's gl_tensor_hash. */
gl_status gl_tensor_hash_at(gl_context* ctx, gl_tensor* t, uint64_t p0, uint64_t* hash);
/* argmax_state's building block (belief_tensor.cpp:512-541): the first
 * strict maximum of the (interior) tensor in [k][j][i] order, its flat
 * index, and the reference's sequential total continued from sum_in over
 * this tensor's values (bit-exact: sum_in = 0.0 gives argmax_state's total;
 * theta shards chain their totals in channel order). value <= 0 means no
 * positive mass. */
gl_status gl_tensor_argmax_candidate(gl_context* ctx, gl_tensor* t, double sum_in, double* value, int64_t* flat,
                                     double* sum_out);
/* Raw device pointer of the current buffer (for NCCL halo exchange). */
gl_status gl_tensor_device_ptr(gl_context* ctx, gl_tensor* t, double** dptr);

/* ---- the hot path --------------------------------------------------------
 * step (belief_tensor.hpp:134-136, belief_tensor.cpp:396-498): Algorithm 1
 * in place. Returns GL_E_EXTINGUISHED exactly when the reference throws
 * BeliefExtinguishedError (tensor and theta_t already updated, as there). */
gl_status gl_step(gl_context* ctx, gl_tensor* t, double u, double v, double w,
                  const gl_map* map, const gl_kernels* kernels,
                  const gl_activation* act);
/* Same work, enqueued only: no host sync, no status read-back. The status of
 * the most recent async step is returned by the next gl_tensor_status(). */
gl_status gl_step_async(gl_context* ctx, gl_tensor* t, double u, double v,
                        double w, const gl_map* map, const gl_kernels* kernels,
                        const gl_activation* act);
gl_status gl_tensor_status(gl_context* ctx, gl_tensor* t);
/* The latest step status of n tensors stepped on this context (its stream
 * orders the read after their steps), in one gather launch, one copy and
 * one sync instead of n: statuses[i] = GL_OK or GL_E_EXTINGUISHED; returns
 * GL_E_EXTINGUISHED if any is. (A batch of robots: one call per context.) */
gl_status gl_tensors_status(gl_context* ctx, gl_tensor* const* ts, int n, int* statuses);
/* ---- theta-slab shards ----------------------------------
 * A shard holds global channels [c_begin, c_end) of a c_total-channel belief,
 * stored with `halo` neighbour planes per side: storage plane q is channel
 * (c_begin - halo + q) mod c_total; the user-visible planes (download, hash,
 * argmax, belief_map) are the interior ones. One sharded step is:
 *   gl_step_async                          (fused kernel, local max only)
 *   all-reduce MAX of *gl_tensor_max_ptr   (uint64 bits of a double >= 0)
 *   gl_shard_finalize                      (status + pending 1/max rescale;
 *                                           a no-op for a shard holding
 *                                           every channel: it finalises in
 *                                           the step kernel)
 *   halo exchange of storage planes        (gl_tensor_plane_ptr; NCCL) —
 *                                           or none: gl_shard_set_peers
 * Sharding does not change any per-element operation: results are bitwise
 * those of the unsharded tensor. */
gl_status gl_shard_init_uniform(gl_context* ctx, const gl_map* map, int c_total,
                                int c_begin, int c_end, int halo,
                                gl_tensor** out);
gl_status gl_shard_info(const gl_tensor* t, int* c_total, int* c_begin,
                        int* c_count, int* halo);
gl_status gl_tensor_plane_ptr(gl_context* ctx, gl_tensor* t, int q,
                              double** dptr);
gl_status gl_tensor_max_ptr(gl_context* ctx, gl_tensor* t,
                            unsigned long long** dptr);
gl_status gl_shard_finalize(gl_context* ctx, gl_tensor* t);
/* LIDAR observation on theta-slab shards:
 *   gl_shard_belief_map      local per-cell max over the shard's channels
 *                            into a DEVICE plane (W*H doubles)
 *   all-reduce MAX of that plane (exact) -> the global belief_map
 *   gl_dither_device         (one rank) Floyd-Steinberg on the device plane
 *   broadcast n, source mass and the cells to every rank
 *   gl_shard_observe         likelihoods of ALL c_total channels at the
 *                            samples (every rank forms the reference's
 *                            sequential mean identically), the quotient
 *                            multiply of the shard's own channels, local max
 *                            into *gl_tensor_max_ptr; n == 0 is a no-op (then
 *                            skip the rest, like observation.cpp:117)
 *   all-reduce MAX of *gl_tensor_max_ptr
 *   gl_shard_observe_finalize  the pending 1/max rescale and the extinguish
 *                            status (observation.cpp:152-169)
 *   halo refresh             (exchange mode only; peer reads see it)
 * Bitwise the unsharded dither_samples + observation_update. */
gl_status gl_shard_belief_map(gl_context* ctx, gl_tensor* t, double* d_plane);
/* gl_shard_observe: declared after gl_likelihood, below */
gl_status gl_shard_observe_finalize(gl_context* ctx, gl_tensor* t);
/* Halo exchange fused into the step over peer memory (NVLink P2P): with
 * peers set, the step's TMA reads its lower halo input planes straight from
 * the left neighbour's buffer and its upper ones from the right neighbour's
 * (lo_b / hi_b = the neighbour's buffer b at storage plane 0, lo_count /
 * hi_count = their interior channel counts; same W, H and halo on every
 * shard), so no exchange step exists. Pointers come from
 * gl_tensor_buffer_ptr in this process (same device or peer-enabled
 * devices) or gl_ipc_open across processes. The cross-rank max all-reduce
 * after every step orders the neighbours' writes of a buffer before these
 * reads, and these reads before the neighbours overwrite it. All NULL:
 * read the shard's own halo planes (exchange them yourself). */
gl_status gl_shard_set_peers(gl_context* ctx, gl_tensor* t, void* lo0,
                             void* lo1, int lo_count, void* hi0, void* hi1,
                             int hi_count);
/* storage plane q of ping-pong buffer buf (0/1); the current one is
 * gl_tensor_current_buffer (all shards of one belief flip together) */
gl_status gl_tensor_buffer_ptr(gl_context* ctx, gl_tensor* t, int buf, int q,
                               double** dptr);
gl_status gl_tensor_current_buffer(const gl_tensor* t, int* buf);
/* CUDA IPC of a tensor buffer (64-byte cudaIpcMemHandle_t) for peer planes
 * across processes (one process per GPU) */
gl_status gl_ipc_get_handle(gl_context* ctx, gl_tensor* t, int buf,
                            void* handle64);
gl_status gl_ipc_open(gl_context* ctx, const void* handle64, void** dptr);
gl_status gl_ipc_close(gl_context* ctx, void* dptr);
/* device-to-device plane copy (single-device halo exchange) */
gl_status gl_tensor_copy_planes(gl_context* ctx, gl_tensor* dst, int dst_q,
                                gl_tensor* src, int src_q, int count);

/* write_belief_snapshot / read_belief_snapshot (belief_tensor.hpp:144-148,
 * belief_tensor.cpp:543-587): BLF1 = "BLF1", uint32 W/H/Theta, float32
 * theta_t, W*H*Theta float32 values [k][j][i], little-endian (lossy for the
 * FP64 belief, as in the reference). I/O failures -> GL_E_RUNTIME with the
 * reference's messages; bad dimensions -> GL_E_INVALID. */
gl_status gl_write_belief_snapshot(gl_context* ctx, gl_tensor* t,
                                   const char* path);
gl_status gl_read_belief_snapshot(gl_context* ctx, const char* path,
                                  double cell_size, double origin_x,
                                  double origin_y, gl_tensor** out);

/* apply_motion (belief_tensor.cpp:340-352): shift only, no mask/diffusion. */
gl_status gl_apply_motion(gl_context* ctx, gl_tensor* t, double u, double v,
                          double w);

/* belief_map (belief_tensor.cpp:500-510): W*H doubles to host. */
gl_status gl_belief_map(gl_context* ctx, gl_tensor* t, double* host_out);

/* argmax_state (belief_tensor.cpp:512-541). */
typedef struct {
  double x, y, theta;  /* Pose2 */
  double confidence;   /* max / total mass */
  int i, j, k;
} gl_pose_estimate;
gl_status gl_argmax(gl_context* ctx, gl_tensor* t, gl_pose_estimate* out);

/* dither_samples (observation.cpp:11-71) on a host belief map. cells gets
 * (i, j) pairs in emission order; at most cap pairs are written, *n is the
 * full count. */
gl_status gl_dither(gl_context* ctx, const double* belief_map, int width,
                    int height, int budget, int32_t* cells, int cap, int* n,
                    double* source_mass);
/* dither_samples(belief_map(tensor), budget) without a host round trip. */
/* dither_samples of a belief map already in device memory (W*H doubles,
 * enqueued work on the context's stream orders it) */
gl_status gl_dither_device(gl_context* ctx, const double* d_plane, int width,
                           int height, int budget, int32_t* cells, int cap, int* n,
                           double* source_mass);
gl_status gl_dither_tensor(gl_context* ctx, gl_tensor* t, int budget,
                           int32_t* cells, int cap, int* n,
                           double* source_mass);

/* dither_samples' total (observation.cpp:16-17: total = 0.0; total += v
 * in order), bit-exact, computed on the device by a parallel scan over the
 * running sum's binades (k_observe.cu k_seq_sum). Values must be finite and
 * >= 0 (else GL_E_INVALID). */
gl_status gl_sequential_sum(gl_context* ctx, const double* values, size_t n, double* total);

/* scan_likelihood / observation_update (observation.cpp:73-170). */
typedef struct {
  double sigma_hit;     /* LikelihoodParams (observation.hpp:21-25) */
  double weight_floor;
  int beam_stride;
} gl_likelihood;
gl_status gl_scan_likelihood(gl_context* ctx, const gl_map* map,
                             const gl_field* field, double x, double y,
                             double theta, const double* angles,
                             const double* ranges, int n_beams,
                             double max_range, gl_likelihood params,
                             double* out);
gl_status gl_observation_update(gl_context* ctx, gl_tensor* t,
                                const int32_t* cells, int n,
                                const double* angles, const double* ranges,
                                int n_beams, double max_range,
                                const gl_map* map, const gl_field* field,
                                gl_likelihood params);
/* the theta-slab shard form (sequence: see gl_shard_belief_map above) */
gl_status gl_shard_observe(gl_context* ctx, gl_tensor* t, const int32_t* cells, int n,
                           const double* angles, const double* ranges, int n_beams,
                           double max_range, const gl_map* map, const gl_field* field,
                           gl_likelihood params);

/* raycast (occupancy_map.hpp:123-124, occupancy_map.cpp:273-332) for a batch
 * of rays, rays[3q..3q+2] = (x, y, angle) in world units: ranges[q] in
 * meters, bit-exact (Amanatides-Woo on the device; cos/sin by host glibc).
 * max_range <= 0 -> GL_E_INVALID; an origin outside free space ->
 * GL_E_MAP_PARSE (the reference's MapParseError kInvalidOrigin). */
gl_status gl_raycast(gl_context* ctx, const gl_map* map, const double* rays, int n, double max_range,
                     double* ranges);
/* simulate_scan (simulator.hpp, simulator.cpp:63-94) for n poses
 * (poses[3q..3q+2] = x, y, theta): the beam angles (beam_count, the
 * reference's formula) and ranges[q * beam_count + b]. With
 * range_noise_sigma > 0, noise[q * beam_count + b] must hold the standard
 * normal the reference's Rng would draw for that beam (pose-major, beam
 * order: rng.normal() once per beam); r += noise * sigma, clamped to
 * [0, max_range]. Bit-exact against the reference for the same draws. */
gl_status gl_simulate_scans(gl_context* ctx, const gl_map* map, const double* poses, int n, int beam_count,
                            double fov, double max_range, double range_noise_sigma, const double* noise,
                            double* angles, double* ranges);

/* diagnostics: out4[0] = step epilogues that took the exact max */
gl_status gl_debug_counters(gl_context* ctx, unsigned long long* out4);

/* map_difficulty (evaluation.cpp:25-72; DifficultyConfig evaluation.hpp:
 * 21-29): the fraction of free cells (interior, every `stride`-th) whose
 * noise-free scan is best matched (first maximum over candidate cells x
 * theta_bins headings, scan_likelihood) more than error_threshold meters
 * away. Bit-exact: host-libm tables, device FP64 in reference order, near
 * ties re-decided with glibc exp. beam_count <= 256. */
typedef struct {
  double error_threshold; /* C, meters (1.0) */
  int beam_count;         /* 8 */
  double fov;             /* 2 pi */
  double max_range;       /* 8 m */
  int stride;             /* 1 */
  int theta_bins;         /* 8 */
  gl_likelihood likelihood; /* {0.2, 0.05, 1} */
} gl_difficulty_config;
gl_status gl_map_difficulty(gl_context* ctx, const gl_map* map,
                            const gl_field* field,
                            const gl_difficulty_config* cfg, double* out);

/* ---- multi-device engine (SURVEY.md §8(b) "gl_engine ... device list",
 * §8(e)) -------------------------------------------------------------------
 * ONE process driving a theta-slab sharded belief over a device list — the
 * C++ callers' form of the multi-GPU path (the Python ThetaShard does the
 * same over torch.distributed, one process per GPU). Shard s owns channels
 * [s*C/n, (s+1)*C/n) on devices[s] (a device may repeat: shards then share
 * it). Per step every shard's fused kernel reads its halo input planes
 * straight from its neighbours' buffers over NVLink P2P (no exchange step),
 * then the 8-byte step max is MAX-all-reduced — by NCCL (ncclAllReduce,
 * uint64, ncclMax; needs distinct devices) or by a peer-memory gather
 * kernel on every device after a cross-device event barrier (P2P) — and
 * every shard finalises the extinguish status and the pending 1/max rescale
 * identically. Observation: per-shard belief maps MAX-combined onto shard
 * 0, Floyd-Steinberg there, every shard's likelihoods at the samples, the
 * max all-reduced again. argmax: per-shard candidates, the reference's
 * lowest-flat-index rule. Results are bitwise the unsharded tensor's. */
typedef struct gl_engine gl_engine;
enum { GL_ENGINE_AUTO = 0, GL_ENGINE_NCCL = 1, GL_ENGINE_P2P = 2 };
/* map: W*H occupancy (1 = occupied; ring forced); n_devices <= 16; mode
 * AUTO = NCCL when the devices are distinct and libnccl loads, else P2P. */
gl_status gl_engine_create(const int* devices, int n_devices, int width, int height, double resolution,
                           double origin_x, double origin_y, const uint8_t* occ, int channels, int mode,
                           gl_engine** out);
gl_status gl_engine_destroy(gl_engine* e);
/* shards, the reduction mode in use (NCCL / P2P), halo planes per side */
gl_status gl_engine_info(const gl_engine* e, int* n_shards, int* mode, int* halo);
/* Kernel slot (0 = main, 1 = rotation-only, like Localizer): the taps are
 * copied to every device and the activation built there. Every slot's
 * angular half-width must fit the halo (the first slot set fixes it). */
gl_status gl_engine_set_kernels(gl_engine* e, int slot, const gl_kernels* kernels);
gl_status gl_engine_init_uniform(gl_engine* e);
gl_status gl_engine_step(gl_engine* e, double u, double v, double w, int slot);
gl_status gl_engine_step_async(gl_engine* e, double u, double v, double w, int slot);
gl_status gl_engine_status(gl_engine* e);
gl_status gl_engine_argmax(gl_engine* e, gl_pose_estimate* out);
gl_status gl_engine_belief_map(gl_engine* e, double* host_out);
/* Localizer::observe's update (localizer.cpp:55-58) on the sharded belief:
 * dither_samples(belief_map, budget) + observation_update; the samples in
 * emission order go to cells (at most cap pairs; *n is the full count). */
gl_status gl_engine_observe(gl_engine* e, int budget, const double* angles, const double* ranges,
                            int n_beams, double max_range, gl_likelihood params, int32_t* cells, int cap,
                            int* n, double* source_mass);
gl_status gl_engine_download(gl_engine* e, double* host, double* theta_t);
gl_status gl_engine_upload(gl_engine* e, const double* host, double theta_t);
gl_status gl_engine_hash(gl_engine* e, uint64_t* hash);
/* the shard's context (per-shard tuning / timing), 0 <= s < n_shards */
gl_status gl_engine_context(gl_engine* e, int s, gl_context** ctx);

#ifdef __cplusplus
}
#endif

#endif /* GRIDLOC_B200_H */
