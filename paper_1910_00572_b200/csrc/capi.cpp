// C-ABI implementation (include/gridloc_b200.h): host runtime that owns the
// device objects, computes the per-step host inputs (motion vectors with the
// reference's libm) and dispatches the sm_100a kernels. No CPU compute
// fallback exists: every tensor operation is a kernel launch, and a missing
// or failing device is reported as GL_E_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <chrono>
#include <thread>
#include <fstream>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "gl_internal.hpp"
#include "gridloc_b200.h"
#include "host_math.hpp"

namespace {

thread_local std::string g_err;

struct Fail {
  gl_status code;
  std::string msg;
};

[[noreturn]] void fail(gl_status code, const std::string& msg) {
  throw Fail{code, msg};
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(GL_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(call) cuda_check((call), #call)

template <class F>
gl_status guard(F&& f) {
  try {
    f();
    return GL_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const glb::MapParseFailure& e) {
    g_err = e.what();
    return GL_E_MAP_PARSE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return GL_E_INVALID;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return GL_E_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GL_E_RUNTIME;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void need(bool ok, const char* msg) {
  if (!ok) fail(GL_E_INVALID, msg);
}

// ------------------------------------------------------------ TMA encoding
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t,
                                 void*, const cuuint64_t*, const cuuint64_t*,
                                 const cuuint32_t*, const cuuint32_t*,
                                 CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion,
                                 CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiled>(p);
    }
  });
  return fn;
}

// 3-D [C][H][W] FP64 view of a belief buffer, box (bw, bh, 1), zero OOB fill.
bool make_tmap(CUtensorMap* m, double* base, int w, int h, int c, int bw,
               int bh) {
  EncodeTiled enc = encode_fn();
  if (!enc) return false;
  if ((static_cast<size_t>(w) * sizeof(double)) % 16 != 0) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(w),
                              static_cast<cuuint64_t>(h),
                              static_cast<cuuint64_t>(c)};
  const cuuint64_t strides[2] = {
      static_cast<cuuint64_t>(w) * sizeof(double),
      static_cast<cuuint64_t>(w) * h * sizeof(double)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(bw),
                             static_cast<cuuint32_t>(bh), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor-map cache per (tensor buffer, box) lives on the tensor.
struct TmapCache {
  double* base = nullptr;
  int planes = 0;
  int bw = 0, bh = 0;
  CUtensorMap map;
};

const CUtensorMap* tensor_tmap(gl_tensor* t, int buf, int bw, int bh);

// ------------------------------------------------------------- helpers
size_t plane_of(const gl_tensor* t) { return static_cast<size_t>(t->w) * t->h; }
// user-visible elements: a theta-slab shard's interior planes (its halo
// planes are storage only)
size_t elems_of(const gl_tensor* t) { return plane_of(t) * t->c; }
int halo_of(const gl_tensor* t) { return t->halo > 0 ? t->halo : 0; }
size_t storage_elems(const gl_tensor* t) { return plane_of(t) * (t->c + 2 * halo_of(t)); }
double* interior(const gl_tensor* t) { return t->d_buf[t->cur] + plane_of(t) * halo_of(t); }

// The context's reusable device scratch. Growing it keeps its contents (an
// operation may place data in it and then ask for more room).
void* ensure_misc(gl_context* ctx, size_t bytes) {
  if (ctx->misc_bytes < bytes) {
    void* fresh = nullptr;
    CK(cudaMalloc(&fresh, bytes));
    if (ctx->d_misc) {
      CK(cudaMemcpyAsync(fresh, ctx->d_misc, ctx->misc_bytes, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      CK(cudaFree(ctx->d_misc));
    }
    ctx->d_misc = fresh;
    ctx->misc_bytes = bytes;
  }
  return ctx->d_misc;
}

void ensure_scratch(gl_context* ctx, size_t elems) {
  if (ctx->scratch_elems < elems) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->d_s) CK(cudaFree(ctx->d_s));
    if (ctx->d_d) CK(cudaFree(ctx->d_d));
    ctx->d_s = ctx->d_d = nullptr;
    CK(cudaMalloc(&ctx->d_s, elems * sizeof(double)));
    CK(cudaMalloc(&ctx->d_d, elems * sizeof(double)));
    ctx->scratch_elems = elems;
  }
}

// Host motion vectors for one step -> device ring slot.
const double2* upload_motion(gl_context* ctx, const gl_tensor* t, double u,
                             double v) {
  if (ctx->ring_cap < t->c) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_motion) CK(cudaFreeHost(ctx->h_motion));
    if (ctx->d_motion) CK(cudaFree(ctx->d_motion));
    ctx->h_motion = nullptr;
    ctx->d_motion = nullptr;
    const size_t n = static_cast<size_t>(gl_context::kRing) * t->c * 2;
    CK(cudaMallocHost(&ctx->h_motion, n * sizeof(double)));
    CK(cudaMalloc(&ctx->d_motion, n * sizeof(double)));
    ctx->ring_cap = t->c;
  }
  const int slot = ctx->ring_next;
  ctx->ring_next = (slot + 1) % gl_context::kRing;
  CK(cudaEventSynchronize(ctx->ring_ev[slot]));  // host slot free again
  double* h = ctx->h_motion + static_cast<size_t>(slot) * ctx->ring_cap * 2;
  double* d = ctx->d_motion + static_cast<size_t>(slot) * ctx->ring_cap * 2;
  const double dtheta = 2.0 * M_PI / t->c;
  glb::motion_table(u, v, 0, t->c, t->theta_t, dtheta, t->cell, h);
  CK(cudaMemcpyAsync(d, h, sizeof(double) * 2 * t->c, cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaEventRecord(ctx->ring_ev[slot], ctx->stream));
  return reinterpret_cast<const double2*>(d);
}

void upload_kernels(gl_kernels* k, int device) {
  if (k->device == device && k->d_ang_w) return;
  DeviceGuard g(device);
  if (k->d_spatial) cudaFree(k->d_spatial);
  if (k->d_ang_off) cudaFree(k->d_ang_off);
  if (k->d_ang_w) cudaFree(k->d_ang_w);
  k->d_spatial = nullptr;
  k->d_ang_off = nullptr;
  k->d_ang_w = nullptr;
  if (!k->spatial.empty()) {
    CK(cudaMalloc(&k->d_spatial, k->spatial.size() * sizeof(double)));
    CK(cudaMemcpy(k->d_spatial, k->spatial.data(),
                  k->spatial.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&k->d_ang_off, k->ang_off.size() * sizeof(int)));
  CK(cudaMemcpy(k->d_ang_off, k->ang_off.data(), k->ang_off.size() * sizeof(int),
                cudaMemcpyHostToDevice));
  CK(cudaMalloc(&k->d_ang_w, k->ang_w.size() * sizeof(double)));
  CK(cudaMemcpy(k->d_ang_w, k->ang_w.data(), k->ang_w.size() * sizeof(double),
                cudaMemcpyHostToDevice));
  k->device = device;
}

// Apply a pending 1/max rescale to the current buffer in place (consumers
// other than the step read the tensor as stored).
void materialize(gl_context* ctx, gl_tensor* t) {
  glb::launch_apply_scale(ctx, t->d_buf[t->cur], storage_elems(t),
                          &t->d_block->buf[t->cur]);
}

inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#else
  std::this_thread::yield();
#endif
}

gl_status read_status(gl_context* ctx, gl_tensor* t) {
  CK(cudaMemcpyAsync(&ctx->h_block->step, &t->d_block->step,
                     sizeof(glb::StepState), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return static_cast<gl_status>(ctx->h_block->step.status);
}

}  // namespace

// Per-tensor TMA map cache (stored out of line to keep gl_tensor POD-ish).
namespace {
struct TensorExtra {
  std::deque<TmapCache> maps;  // stable addresses
};
std::mutex g_extra_mu;
std::vector<std::pair<const gl_tensor*, std::unique_ptr<TensorExtra>>> g_extra;

TensorExtra* extra_of(const gl_tensor* t) {
  std::lock_guard<std::mutex> lk(g_extra_mu);
  for (auto& e : g_extra)
    if (e.first == t) return e.second.get();
  g_extra.emplace_back(t, std::make_unique<TensorExtra>());
  return g_extra.back().second.get();
}

void drop_extra(const gl_tensor* t) {
  std::lock_guard<std::mutex> lk(g_extra_mu);
  g_extra.erase(std::remove_if(g_extra.begin(), g_extra.end(),
                               [t](auto& e) { return e.first == t; }),
                g_extra.end());
}

// map over `planes` storage planes at `base` (the tensor's own buffer, or a
// theta-shard neighbour's), cached on the tensor
const CUtensorMap* tensor_tmap_at(gl_tensor* t, double* base, int planes, int bw, int bh) {
  TensorExtra* x = extra_of(t);
  for (auto& m : x->maps)
    if (m.base == base && m.planes == planes && m.bw == bw && m.bh == bh) return &m.map;
  TmapCache c;
  c.base = base;
  c.planes = planes;
  c.bw = bw;
  c.bh = bh;
  if (!make_tmap(&c.map, c.base, t->w, t->h, planes, bw, bh)) return nullptr;
  x->maps.push_back(c);
  return &x->maps.back().map;
}

const CUtensorMap* tensor_tmap(gl_tensor* t, int buf, int bw, int bh) {
  return tensor_tmap_at(t, t->d_buf[buf], t->c + 2 * halo_of(t), bw, bh);
}
}  // namespace

extern "C" {

const char* gl_last_error(void) { return g_err.c_str(); }

extern "C++" {
namespace glb {
void set_last_error(const std::string& msg) { g_err = msg; }  // engine.cpp
}  // namespace glb
}

const char* gl_version(void) { return "gridloc_b200 0.1 sm_100a fp64"; }

// ---------------------------------------------------------------- context
gl_status gl_context_create(int device, gl_context** out) {
  return guard([&] {
    need(out != nullptr, "out is null");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    need(device >= 0 && device < n, "no such CUDA device");
    DeviceGuard g(device);
    auto ctx = std::make_unique<gl_context>();
    ctx->device = device;
    CK(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ctx->ev_begin));
    CK(cudaEventCreate(&ctx->ev_end));
    for (auto& e : ctx->ring_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaMallocHost(&ctx->h_block, sizeof(glb::DeviceBlock)));
    CK(cudaHostAlloc(&ctx->h_status, sizeof(int), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->d_status), ctx->h_status, 0));
    *out = ctx.release();
  });
}

gl_status gl_context_destroy(gl_context* ctx) {
  return guard([&] {
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->d_s) cudaFree(ctx->d_s);
    if (ctx->d_d) cudaFree(ctx->d_d);
    if (ctx->d_motion) cudaFree(ctx->d_motion);
    if (ctx->h_motion) cudaFreeHost(ctx->h_motion);
    if (ctx->h_block) cudaFreeHost(ctx->h_block);
    if (ctx->h_status) cudaFreeHost(ctx->h_status);
    if (ctx->d_misc) cudaFree(ctx->d_misc);
    if (ctx->h_misc) cudaFreeHost(ctx->h_misc);
    if (ctx->d_kind) cudaFree(ctx->d_kind);
    for (auto& e : ctx->marks)
      if (e) cudaEventDestroy(e);
    for (auto& e : ctx->ring_ev) cudaEventDestroy(e);
    for (auto& e : ctx->tev) cudaEventDestroy(e);
    cudaEventDestroy(ctx->ev_begin);
    cudaEventDestroy(ctx->ev_end);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

gl_status gl_context_synchronize(gl_context* ctx) {
  return guard([&] {
    need(ctx, "null context");
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

gl_status gl_context_set_step_timing(gl_context* ctx, int enable) {
  return guard([&] {
    need(ctx, "null context");
    ctx->step_events = enable != 0;
    if (!ctx->step_events) ctx->ev_begin_last = ctx->ev_end_last = nullptr;
  });
}

gl_status gl_context_last_step_ms(gl_context* ctx, double* ms) {
  return guard([&] {
    need(ctx && ms, "null argument");
    need(ctx->ev_end_last != nullptr,
         "no timed step on this context (enable gl_context_set_step_timing before stepping)");
    CK(cudaEventSynchronize(ctx->ev_end_last));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, ctx->ev_begin_last, ctx->ev_end_last));
    *ms = f;
  });
}

gl_status gl_context_mark(gl_context* ctx, int i) {
  return guard([&] {
    need(ctx && i >= 0 && i < 16, "bad marker");
    DeviceGuard g(ctx->device);
    if (!ctx->marks[i]) CK(cudaEventCreate(&ctx->marks[i]));
    CK(cudaEventRecord(ctx->marks[i], ctx->stream));
  });
}

gl_status gl_context_marks_ms(gl_context* ctx, int i, int j, double* ms) {
  return guard([&] {
    need(ctx && ms && i >= 0 && i < 16 && j >= 0 && j < 16, "bad marker");
    need(ctx->marks[i] && ctx->marks[j], "marker not recorded");
    CK(cudaEventSynchronize(ctx->marks[j]));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, ctx->marks[i], ctx->marks[j]));
    *ms = f;
  });
}

gl_status gl_context_stream(gl_context* ctx, void** stream) {
  return guard([&] {
    need(ctx && stream, "null argument");
    *stream = reinterpret_cast<void*>(ctx->stream);
  });
}

gl_status gl_context_time_steps(gl_context* ctx, int enable) {
  return guard([&] {
    need(ctx, "null context");
    DeviceGuard g(ctx->device);
    if (enable && ctx->tev.empty()) {
      ctx->tev.resize(2 * gl_context::kTimers);
      for (auto& e : ctx->tev) CK(cudaEventCreate(&e));
    }
    need(enable >= 0, "enable must be 0 (off) or a step stride >= 1");
    ctx->timing = enable != 0;
    ctx->tstride = enable > 0 ? enable : 1;
    ctx->tstep = 0;
    ctx->tcount = 0;
  });
}

gl_status gl_context_step_times(gl_context* ctx, double* total_ms, int* count) {
  return guard([&] {
    need(ctx && total_ms && count, "null argument");
    DeviceGuard g(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    double tot = 0.0;
    for (int q = 0; q < ctx->tcount; ++q) {
      float f = 0.f;
      CK(cudaEventElapsedTime(&f, ctx->tev[2 * q], ctx->tev[2 * q + 1]));
      tot += f;
    }
    *total_ms = tot;
    *count = ctx->tcount;
    ctx->tcount = 0;
  });
}

gl_status gl_context_set_path(gl_context* ctx, int path) {
  return guard([&] {
    need(ctx, "null context");
    need(path >= GL_PATH_AUTO && path <= GL_PATH_GENERIC, "bad path");
    ctx->path = path;
  });
}

gl_status gl_context_set_host_exp(gl_context* ctx, int enable) {
  return guard([&] {
    need(ctx, "null context");
    ctx->host_exp = enable != 0;
  });
}

gl_status gl_context_set_fast(gl_context* ctx, int enable) {
  return guard([&] {
    need(ctx, "null context");
    ctx->allow_fast = enable != 0;
  });
}

gl_status gl_context_set_himax(gl_context* ctx, int mode) {
  return guard([&] {
    need(ctx, "null context");
    need(mode >= 0 && mode <= 2, "himax mode must be 0 (auto), 1 (always) or 2 (never)");
    ctx->himax_mode = mode;
  });
}

gl_status gl_context_set_channel_chunks(gl_context* ctx, int n) {
  return guard([&] {
    need(ctx, "null context");
    need(n >= 0, "channel chunks must be >= 0 (0 = auto)");
    ctx->channel_chunks = n;
  });
}

gl_status gl_context_set_wave_tail(gl_context* ctx, int ctas, int chunks) {
  return guard([&] {
    need(ctx, "null context");
    need(ctas >= -1, "wave-tail CTAs must be >= -1 (-1 = auto, 0 = off)");
    need(chunks >= 1, "wave-tail chunks must be >= 1");
    ctx->tail_ctas = ctas;
    ctx->tail_chunks = chunks;
  });
}

gl_status gl_context_set_wall_mask(gl_context* ctx, int enable) {
  return guard([&] {
    need(ctx, "null context");
    ctx->wall_mask = enable != 0;
  });
}

gl_status gl_context_set_tile_order(gl_context* ctx, int strip_tiles, int stack) {
  return guard([&] {
    need(ctx, "null context");
    need(strip_tiles >= -1, "tile order must be >= -1 (-1 = auto, 0 = row-major, n = strips of n tiles)");
    need(stack >= 0, "tile stack must be >= 0");
    ctx->strip_tiles = strip_tiles;
    ctx->tile_stack = stack;
  });
}

gl_status gl_context_launch_count(gl_context* ctx, uint64_t* n) {
  return guard([&] {
    need(ctx && n, "null argument");
    *n = ctx->launches;
  });
}

// ------------------------------------------------------------------- maps
gl_status gl_load_map(const uint8_t* bytes, size_t n, int threshold,
                      int* width, int* height, uint8_t* occ) {
  return guard([&] {
    need(bytes && width && height, "null argument");
    glb::MapParse m = glb::parse_pgm_map(bytes, n, threshold);
    *width = m.w;
    *height = m.h;
    if (occ) std::memcpy(occ, m.occ.data(), m.occ.size());
  });
}

gl_status gl_map_create(gl_context* ctx, int width, int height,
                        double resolution, double origin_x, double origin_y,
                        const uint8_t* occ, gl_map** out) {
  return guard([&] {
    need(ctx && occ && out, "null argument");
    if (width < 1 || height < 1) fail(GL_E_MAP_PARSE, "map with zero dimension");
    need(resolution > 0.0, "map resolution must be > 0");
    DeviceGuard g(ctx->device);
    auto m = std::make_unique<gl_map>();
    m->w = width;
    m->h = height;
    m->res = resolution;
    m->ox = origin_x;
    m->oy = origin_y;
    m->occ.assign(occ, occ + static_cast<size_t>(width) * height);
    for (auto& c : m->occ) c = c ? 1 : 0;
    glb::force_ring(m->occ.data(), width, height);
    m->free_count = static_cast<int>(std::count(m->occ.begin(), m->occ.end(), 0));
    m->device = ctx->device;
    CK(cudaMalloc(&m->d_occ, m->occ.size()));
    CK(cudaMemcpy(m->d_occ, m->occ.data(), m->occ.size(), cudaMemcpyHostToDevice));
    *out = m.release();
  });
}

gl_status gl_map_destroy(gl_map* map) {
  return guard([&] {
    if (!map) return;
    DeviceGuard g(map->device);
    cudaFree(map->d_occ);
    delete map;
  });
}

gl_status gl_map_info(const gl_map* m, int* w, int* h, double* res, double* ox,
                      double* oy, int* free_count) {
  return guard([&] {
    need(m, "null map");
    if (w) *w = m->w;
    if (h) *h = m->h;
    if (res) *res = m->res;
    if (ox) *ox = m->ox;
    if (oy) *oy = m->oy;
    if (free_count) *free_count = m->free_count;
  });
}

gl_status gl_map_cells(const gl_map* m, uint8_t* out) {
  return guard([&] {
    need(m && out, "null argument");
    std::memcpy(out, m->occ.data(), m->occ.size());
  });
}

gl_status gl_field_create(gl_context* ctx, const gl_map* map, gl_field** out) {
  return guard([&] {
    need(ctx && map && out, "null argument");
    DeviceGuard g(ctx->device);
    auto f = std::make_unique<gl_field>();
    f->w = map->w;
    f->h = map->h;
    // exact EDT on the device; the host copy feeds the per-cell beam score
    // table, which needs the host libm (obs_tables)
    const size_t cells = static_cast<size_t>(map->w) * map->h;
    f->values.resize(cells);
    CK(cudaMalloc(&f->d_values, cells * sizeof(double)));
    void* scratch = nullptr;
    CK(cudaMalloc(&scratch, glb::distance_field_scratch_bytes(map->w, map->h)));
    glb::launch_distance_field(ctx, map->d_occ, map->w, map->h, map->res, f->d_values, scratch);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(f->values.data(), f->d_values, cells * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaFree(scratch));
    *out = f.release();
  });
}

gl_status gl_field_destroy(gl_field* f) {
  return guard([&] {
    if (!f) return;
    cudaFree(f->d_values);
    if (f->d_score) cudaFree(f->d_score);
    delete f;
  });
}

gl_status gl_field_values(const gl_field* f, double* out) {
  return guard([&] {
    need(f && out, "null argument");
    std::memcpy(out, f->values.data(), f->values.size() * sizeof(double));
  });
}

// ---------------------------------------------------------------- kernels
gl_status gl_build_kernels(double sigma_x, double sigma_y, double sigma_theta,
                           int channels, double cell_size, double delta_theta,
                           gl_kernels** out) {
  return guard([&] {
    need(out != nullptr, "out is null");
    glb::HostKernels hk = glb::build_kernels_host(sigma_x, sigma_y, sigma_theta,
                                                  channels, cell_size, delta_theta);
    auto k = std::make_unique<gl_kernels>();
    k->info.channels = hk.channels;
    k->info.radius = hk.radius;
    k->info.separable = hk.separable;
    k->info.degenerate_spatial = hk.degenerate_spatial;
    k->info.degenerate_angular = hk.degenerate_angular;
    k->info.n_angular = static_cast<int>(hk.ang_w.size());
    k->sep = std::move(hk.sep);
    k->spatial = std::move(hk.spatial);
    k->ang_off = std::move(hk.ang_off);
    k->ang_w = std::move(hk.ang_w);
    *out = k.release();
  });
}

gl_status gl_kernels_create(gl_context*, const gl_kernel_info* info,
                            const double* sep, const double* spatial,
                            const int* ang_off, const double* ang_w,
                            gl_kernels** out) {
  return guard([&] {
    need(info && out && ang_off && ang_w, "null argument");
    need(info->radius >= 0 && info->n_angular >= 1 && info->channels >= 1,
         "bad kernel info");
    const int kw = 2 * info->radius + 1;
    need(!info->separable || (sep && kw <= glb::kMaxSepTaps),
         "separable kernels need 2r+1 <= 63 taps");
    need(info->separable || spatial, "dense kernels need spatial weights");
    auto k = std::make_unique<gl_kernels>();
    k->info = *info;
    if (info->separable) k->sep.assign(sep, sep + kw);
    if (spatial) {
      k->spatial.assign(spatial, spatial + static_cast<size_t>(info->channels) * kw * kw);
    } else {
      k->spatial.resize(static_cast<size_t>(info->channels) * kw * kw);
      for (int c = 0; c < info->channels; ++c)
        for (int a = 0; a < kw; ++a)
          for (int b = 0; b < kw; ++b)
            k->spatial[static_cast<size_t>(c) * kw * kw + a * kw + b] = k->sep[a] * k->sep[b];
    }
    k->ang_off.assign(ang_off, ang_off + info->n_angular);
    k->ang_w.assign(ang_w, ang_w + info->n_angular);
    *out = k.release();
  });
}

gl_status gl_kernels_destroy(gl_kernels* k) {
  return guard([&] {
    if (!k) return;
    if (k->device >= 0) {
      DeviceGuard g(k->device);
      cudaFree(k->d_spatial);
      cudaFree(k->d_ang_off);
      cudaFree(k->d_ang_w);
    }
    delete k;
  });
}

gl_status gl_kernels_info(const gl_kernels* k, gl_kernel_info* info) {
  return guard([&] {
    need(k && info, "null argument");
    *info = k->info;
  });
}

gl_status gl_kernels_get(const gl_kernels* k, double* sep, double* spatial,
                         int* ang_off, double* ang_w) {
  return guard([&] {
    need(k, "null kernels");
    if (sep) std::copy(k->sep.begin(), k->sep.end(), sep);
    if (spatial) std::copy(k->spatial.begin(), k->spatial.end(), spatial);
    if (ang_off) std::copy(k->ang_off.begin(), k->ang_off.end(), ang_off);
    if (ang_w) std::copy(k->ang_w.begin(), k->ang_w.end(), ang_w);
  });
}

gl_status gl_make_activation(gl_context* ctx, const gl_map* map,
                             const gl_kernels* kernels, int channels,
                             gl_activation** out) {
  return guard([&] {
    need(ctx && map && kernels && out, "null argument");
    need(channels >= 1, "channels must be >= 1");
    need(kernels->info.separable || kernels->info.channels >= channels,
         "kernel set has fewer channels than the tensor");
    DeviceGuard g(ctx->device);
    auto* kk = const_cast<gl_kernels*>(kernels);
    upload_kernels(kk, ctx->device);
    auto a = std::make_unique<gl_activation>();
    a->w = map->w;
    a->h = map->h;
    a->channels = channels;
    // isotropic (separable) and impulse kernels make every channel's
    // activation identical (SURVEY.md probe P4): store one plane.
    a->k_invariant = kernels->info.separable || kernels->info.radius == 0;
    const size_t plane = static_cast<size_t>(map->w) * map->h;
    const size_t np = a->k_invariant ? 1 : channels;
    CK(cudaMalloc(&a->d_values, plane * np * sizeof(double)));
    CK(cudaMalloc(&a->d_inverse, plane * np * sizeof(double)));
    const size_t scratch = plane * (2 + 2 * np);
    double* d_scratch = static_cast<double*>(ensure_misc(ctx, scratch * sizeof(double)));
    glb::launch_make_activation(ctx, map->d_occ, map->w, map->h, channels, kk,
                                a->d_values, a->d_inverse, a->k_invariant,
                                d_scratch);
    if (a->k_invariant) {
      CK(cudaMalloc(&a->d_inverse_masked, plane * sizeof(double)));
      glb::launch_mask_plane(ctx, a->d_inverse, map->d_occ, plane, a->d_inverse_masked);
    }
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    *out = a.release();
  });
}

gl_status gl_activation_destroy(gl_activation* a) {
  return guard([&] {
    if (!a) return;
    cudaFree(a->d_values);
    cudaFree(a->d_inverse);
    if (a->d_inverse_masked) cudaFree(a->d_inverse_masked);
    delete a;
  });
}

gl_status gl_activation_get(gl_context* ctx, const gl_activation* a,
                            double* values, double* inverse) {
  return guard([&] {
    need(ctx && a, "null argument");
    DeviceGuard g(ctx->device);
    const size_t plane = static_cast<size_t>(a->w) * a->h;
    for (int k = 0; k < a->channels; ++k) {
      const size_t off = a->k_invariant ? 0 : plane * k;
      if (values)
        CK(cudaMemcpyAsync(values + plane * k, a->d_values + off,
                           plane * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      if (inverse)
        CK(cudaMemcpyAsync(inverse + plane * k, a->d_inverse + off,
                           plane * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

// ---------------------------------------------------------------- tensors
// Owning handle of a tensor under construction: a failure anywhere before
// the caller releases it frees every device buffer allocated so far (at
// 4096^2 x 360 one buffer is 48 GB, which must not leak on an OOM of the
// second).
using TensorPtr = std::unique_ptr<gl_tensor, gl_status (*)(gl_tensor*)>;

static TensorPtr new_tensor(gl_context* ctx, int w, int h, int c, double cell,
                            double ox, double oy, int halo = -1, int c_total = 0,
                            int c_begin = 0) {
  need(w >= 1 && h >= 1 && c >= 1, "belief tensor dimensions must be positive");
  TensorPtr t(new gl_tensor(), gl_tensor_destroy);
  t->w = w;
  t->h = h;
  t->c = c;
  t->cell = cell;
  t->ox = ox;
  t->oy = oy;
  t->device = ctx->device;
  t->halo = halo;
  t->c_total = halo >= 0 ? c_total : c;
  t->c_begin = halo >= 0 ? c_begin : 0;
  const size_t n = storage_elems(t.get());
  CK(cudaMalloc(&t->d_buf[0], n * sizeof(double)));
  CK(cudaMalloc(&t->d_buf[1], n * sizeof(double)));
  CK(cudaMalloc(&t->d_block, sizeof(glb::DeviceBlock)));
  glb::DeviceBlock init{};
  init.buf[0].scale = init.buf[1].scale = 1.0;
  CK(cudaMemcpy(t->d_block, &init, sizeof(init), cudaMemcpyHostToDevice));
  return t;
}

gl_status gl_tensor_create(gl_context* ctx, int width, int height,
                           int channels, double cell_size, double origin_x,
                           double origin_y, gl_tensor** out) {
  return guard([&] {
    need(ctx && out, "null argument");
    DeviceGuard g(ctx->device);
    TensorPtr t = new_tensor(ctx, width, height, channels, cell_size, origin_x, origin_y);
    glb::launch_fill(ctx, t->d_buf[0], elems_of(t.get()), 0.0);
    CK(cudaStreamSynchronize(ctx->stream));
    *out = t.release();
  });
}

gl_status gl_init_uniform(gl_context* ctx, const gl_map* map, int channels,
                          gl_tensor** out) {
  return guard([&] {
    need(ctx && map && out, "null argument");
    need(channels >= 4 && channels % 2 == 0, "channel count must be even and >= 4");
    need(map->free_count > 0, "map has no free cells to initialize from");
    DeviceGuard g(ctx->device);
    TensorPtr t = new_tensor(ctx, map->w, map->h, channels, map->res, map->ox, map->oy);
    glb::launch_init_uniform(ctx, t->d_buf[0], map->d_occ, map->w, map->h, channels);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    *out = t.release();
  });
}

// ------------------------------------------------------------ snapshots
// BLF1 (belief_tensor.hpp:144-148, belief_tensor.cpp:543-587): "BLF1",
// uint32 W/H/Theta, float32 theta_t, W*H*Theta float32 values [k][j][i],
// little-endian. The float32 conversion runs on the device, so half the
// bytes cross PCIe.
gl_status gl_write_belief_snapshot(gl_context* ctx, gl_tensor* t, const char* path) {
  return guard([&] {
    need(ctx && t && path, "null argument");
    need(t->halo < 0, "snapshots are written from whole (unsharded) tensors");
    DeviceGuard g(ctx->device);
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error(std::string("cannot open for writing: ") + path);
    materialize(ctx, t);
    const size_t n = elems_of(t);
    float* d = static_cast<float*>(ensure_misc(ctx, n * sizeof(float)));
    glb::launch_to_f32(ctx, interior(t), d, n);
    std::vector<float> buf(n);
    CK(cudaMemcpyAsync(buf.data(), d, n * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const char magic[4] = {'B', 'L', 'F', '1'};
    out.write(magic, 4);
    const uint32_t dims[3] = {static_cast<uint32_t>(t->w), static_cast<uint32_t>(t->h),
                              static_cast<uint32_t>(t->c)};
    out.write(reinterpret_cast<const char*>(dims), sizeof(dims));
    const float theta = static_cast<float>(t->theta_t);
    out.write(reinterpret_cast<const char*>(&theta), sizeof(theta));
    out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(n * sizeof(float)));
    if (!out) throw std::runtime_error(std::string("write failed: ") + path);
  });
}

gl_status gl_read_belief_snapshot(gl_context* ctx, const char* path, double cell_size,
                                  double origin_x, double origin_y, gl_tensor** out_t) {
  return guard([&] {
    need(ctx && path && out_t, "null argument");
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error(std::string("cannot open snapshot: ") + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "BLF1", 4) != 0) {
      throw std::runtime_error(std::string("bad belief snapshot magic in ") + path);
    }
    uint32_t dims[3];
    float theta;
    in.read(reinterpret_cast<char*>(dims), sizeof(dims));
    in.read(reinterpret_cast<char*>(&theta), sizeof(theta));
    if (!in) throw std::runtime_error(std::string("truncated belief snapshot ") + path);
    // validate the header against the file before allocating (a corrupt
    // header must not request a huge device allocation)
    need(dims[0] >= 1 && dims[1] >= 1 && dims[2] >= 1 && dims[0] <= (1u << 20) && dims[1] <= (1u << 20) &&
             dims[2] <= (1u << 16),
         "belief snapshot dimensions out of range");
    const unsigned long long want = 16ull + 4ull * dims[0] * dims[1] * dims[2];
    const std::streampos here = in.tellg();
    in.seekg(0, std::ios::end);
    const unsigned long long have = static_cast<unsigned long long>(in.tellg());
    in.seekg(here);
    if (have < want) throw std::runtime_error(std::string("truncated belief snapshot ") + path);
    DeviceGuard g(ctx->device);
    TensorPtr t = new_tensor(ctx, static_cast<int>(dims[0]), static_cast<int>(dims[1]), static_cast<int>(dims[2]),
                             cell_size, origin_x, origin_y);
    t->theta_t = theta;
    const size_t n = elems_of(t.get());
    std::vector<float> buf(n);
    in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(n * sizeof(float)));
    if (!in) throw std::runtime_error(std::string("truncated belief snapshot ") + path);
    float* d = static_cast<float*>(ensure_misc(ctx, n * sizeof(float)));
    CK(cudaMemcpyAsync(d, buf.data(), n * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    glb::launch_from_f32(ctx, d, interior(t.get()), n);
    auto* flag = static_cast<unsigned int*>(ensure_misc(ctx, 64));  // the payload is consumed (stream order)
    glb::launch_scan_unclean(ctx, interior(t.get()), n, flag);
    unsigned int unclean = 0;
    CK(cudaMemcpyAsync(&unclean, flag, sizeof(unclean), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    t->clean[t->cur] = unclean == 0;
    *out_t = t.release();
  });
}

gl_status gl_tensor_destroy(gl_tensor* t) {
  return guard([&] {
    if (!t) return;
    DeviceGuard g(t->device);
    cudaFree(t->d_buf[0]);
    cudaFree(t->d_buf[1]);
    cudaFree(t->d_block);
    drop_extra(t);
    delete t;
  });
}

gl_status gl_tensor_info(const gl_tensor* t, int* w, int* h, int* c,
                         double* cell, double* ox, double* oy) {
  return guard([&] {
    need(t, "null tensor");
    if (w) *w = t->w;
    if (h) *h = t->h;
    if (c) *c = t->c;
    if (cell) *cell = t->cell;
    if (ox) *ox = t->ox;
    if (oy) *oy = t->oy;
  });
}

gl_status gl_tensor_theta(const gl_tensor* t, double* theta_t) {
  return guard([&] {
    need(t && theta_t, "null argument");
    *theta_t = t->theta_t;
  });
}

gl_status gl_tensor_set_theta(gl_tensor* t, double theta_t) {
  return guard([&] {
    need(t, "null tensor");
    t->theta_t = theta_t;
  });
}

gl_status gl_tensor_upload(gl_context* ctx, gl_tensor* t, const double* host) {
  return guard([&] {
    need(ctx && t && host, "null argument");
    DeviceGuard g(ctx->device);
    CK(cudaMemcpyAsync(interior(t), host, elems_of(t) * sizeof(double),
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(&t->d_block->buf[t->cur], 0, sizeof(glb::BufState), ctx->stream));
    auto* flag = static_cast<unsigned int*>(ensure_misc(ctx, 64));
    glb::launch_scan_unclean(ctx, interior(t), elems_of(t), flag);
    unsigned int unclean = 0;
    CK(cudaMemcpyAsync(&unclean, flag, sizeof(unclean), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    t->clean[t->cur] = unclean == 0;
  });
}

gl_status gl_tensor_download(gl_context* ctx, gl_tensor* t, double* host) {
  return guard([&] {
    need(ctx && t && host, "null argument");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    CK(cudaMemcpyAsync(host, interior(t), elems_of(t) * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

gl_status gl_tensor_read(gl_context* ctx, gl_tensor* t, size_t offset,
                         size_t count, double* host) {
  return guard([&] {
    need(ctx && t && (host || count == 0), "null argument");
    need(offset <= elems_of(t) && count <= elems_of(t) - offset, "range out of bounds");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    CK(cudaMemcpyAsync(host, interior(t) + offset, count * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

gl_status gl_tensor_write(gl_context* ctx, gl_tensor* t, size_t offset,
                          size_t count, const double* host) {
  return guard([&] {
    need(ctx && t && (host || count == 0), "null argument");
    need(offset <= elems_of(t) && count <= elems_of(t) - offset, "range out of bounds");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    CK(cudaMemcpyAsync(interior(t) + offset, host, count * sizeof(double),
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (size_t q = 0; q < count; ++q) {
      const double v = host[q];
      if (std::signbit(v) || !std::isfinite(v)) t->clean[t->cur] = false;
    }
  });
}

gl_status gl_tensor_clone(gl_context* ctx, gl_tensor* src, gl_tensor** out) {
  return guard([&] {
    need(ctx && src && out, "null argument");
    DeviceGuard g(ctx->device);
    materialize(ctx, src);
    TensorPtr t = new_tensor(ctx, src->w, src->h, src->c, src->cell, src->ox, src->oy,
                             src->halo, src->c_total, src->c_begin);
    CK(cudaMemcpyAsync(t->d_buf[0], src->d_buf[src->cur], storage_elems(src) * sizeof(double),
                       cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    t->theta_t = src->theta_t;
    t->clean[0] = src->clean[src->cur];
    *out = t.release();
  });
}

gl_status gl_tensor_hash(gl_context* ctx, gl_tensor* t, uint64_t* hash) {
  return guard([&] {
    need(ctx && t && hash, "null argument");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    auto* d = static_cast<unsigned long long*>(ensure_misc(ctx, 64));
    glb::launch_hash(ctx, interior(t), elems_of(t), d, 0);
    unsigned long long hv = 0;
    CK(cudaMemcpyAsync(&hv, d, sizeof(hv), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *hash = hv;
  });
}

gl_status gl_tensor_hash_at(gl_context* ctx, gl_tensor* t, uint64_t p0, uint64_t* hash) {
  return guard([&] {
    need(ctx && t && hash, "null argument");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    auto* d = static_cast<unsigned long long*>(ensure_misc(ctx, 64));
    glb::launch_hash(ctx, interior(t), elems_of(t), d, p0);
    unsigned long long hv = 0;
    CK(cudaMemcpyAsync(&hv, d, sizeof(hv), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *hash = hv;
  });
}

// argmax_state's scan (belief_tensor.cpp:512-541): the first strict maximum
// and its flat index (per-block candidates, lowest-index tie rule) and the
// reference's SEQUENTIAL total in [k][j][i] order, bit-exact (k_seqsum.cu:
// parallel binade scan; the literal one-thread chain for tensors holding
// negative / non-finite values). s0: the running total the scan enters with
// (a theta shard continues its left neighbours' sum).
struct ArgmaxExact {
  double v;
  long long idx;
  double total;
};

static ArgmaxExact argmax_exact(gl_context* ctx, gl_tensor* t, double s0) {
  materialize(ctx, t);
  const size_t n = elems_of(t);
  auto al = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  const size_t sb = al(glb::argmax_scratch_bytes(n));
  char* d = static_cast<char*>(ensure_misc(ctx, sb + 256 + glb::seq_sum_scratch_bytes(n)));
  double* d_total = reinterpret_cast<double*>(d + sb + 64);
  int* d_inv = reinterpret_cast<int*>(d + sb + 72);
  if (glb::seq_sum_fuses_argmax(n)) {
    // one read of the tensor: the exact total's chunk pass also takes the
    // argmax candidates ({v, idx, -} at d + sb)
    glb::launch_seq_sum_big(ctx, interior(t), n, d_total, d_inv, d + sb + 256, s0, d + sb);
  } else {
    glb::launch_argmax(ctx, interior(t), n, d, sb, d + sb);  // {v, idx, pairwise sum} at d + sb
    glb::launch_seq_sum_big(ctx, interior(t), n, d_total, d_inv, d + sb + 256, s0);
  }
  glb::launch_seq_sum_chain(ctx, interior(t), n, d_total, d_inv, s0);  // runs only if the scan flagged
  struct {
    double v;
    long long idx;
    double sum;
  } res{};
  double total = 0.0;
  CK(cudaMemcpyAsync(&res, d + sb, sizeof(res), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&total, d_total, sizeof(total), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaGetLastError());
  return ArgmaxExact{res.v, res.idx, total};
}

gl_status gl_tensor_argmax_candidate(gl_context* ctx, gl_tensor* t, double sum_in, double* value, int64_t* flat,
                                     double* sum_out) {
  return guard([&] {
    need(ctx && t && value && flat && sum_out, "null argument");
    DeviceGuard g(ctx->device);
    const ArgmaxExact res = argmax_exact(ctx, t, sum_in);
    *value = res.v;
    *flat = res.idx;
    *sum_out = res.total;
  });
}

gl_status gl_tensor_device_ptr(gl_context* ctx, gl_tensor* t, double** dptr) {
  return guard([&] {
    need(ctx && t && dptr, "null argument");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    CK(cudaStreamSynchronize(ctx->stream));
    *dptr = interior(t);
  });
}

// ----------------------------------------------------------------- step
#ifdef GL_EXPERIMENT_ENV
// host-time sections of enqueue_step (experiment builds; GL_DEBUG_ENQUEUE=1
// prints the per-call means at exit)
struct EnqProf {
  double ns[8] = {};
  long n = 0;
  ~EnqProf() {
    if (n && getenv("GL_DEBUG_ENQUEUE"))
      fprintf(stderr, "enqueue_step host ns/call: checks+guard %.0f | kernels %.0f | fused+tmap %.0f | motion %.0f | launch %.0f | tail %.0f (n=%ld)\n",
              ns[0] / n, ns[1] / n, ns[2] / n, ns[3] / n, ns[4] / n, ns[5] / n, n);
  }
};
static EnqProf g_enq;
#define ENQ_T(i) do { const auto t_ = std::chrono::steady_clock::now(); g_enq.ns[i] += std::chrono::duration<double, std::nano>(t_ - enq_t0).count(); enq_t0 = t_; } while (0)
#else
#define ENQ_T(i) do { } while (0)
#endif
static void enqueue_step(gl_context* ctx, gl_tensor* t, double u, double v,
                         double w, const gl_map* map, const gl_kernels* kernels,
                         const gl_activation* act, bool publish = false) {
#ifdef GL_EXPERIMENT_ENV
  auto enq_t0 = std::chrono::steady_clock::now();
  ++g_enq.n;
#endif
  need(ctx && t && map && kernels && act, "null argument");
  need(map->w == t->w && map->h == t->h, "map and tensor sizes differ");
  need(act->w == t->w && act->h == t->h && act->channels == t->c_total,
       "activation does not match the tensor");
  need(kernels->info.separable || kernels->info.channels >= t->c,
       "kernel set has fewer channels than the tensor");
  DeviceGuard g(ctx->device);
  ENQ_T(0);
  auto* kk = const_cast<gl_kernels*>(kernels);
  upload_kernels(kk, ctx->device);
  ENQ_T(1);

  glb::StepArgs a{};
  const int src = t->cur, dst = 1 - t->cur;
  a.src = t->d_buf[src];
  a.dst = t->d_buf[dst];
  a.src_state = &t->d_block->buf[src];
  a.dst_state = &t->d_block->buf[dst];
  a.step_state = &t->d_block->step;
  a.host_status = publish ? ctx->d_status : nullptr;
  a.occ = map->d_occ;
  a.inv = act->d_inverse;
  a.inv_masked = act->d_inverse_masked;
  a.inv_per_channel = act->k_invariant ? 0 : 1;
  a.w = t->w;
  a.h = t->h;
  a.c = t->c;

  const int r = kernels->info.radius;
  glb::AngTaps ang{};
  bool fused = ctx->path != GL_PATH_GENERIC &&
               (kernels->info.separable || r == 0) &&
               kernels->info.n_angular <= 2 * glb::kFusedMaxHalf + 1;
  if (fused) {
    ang.n = kernels->info.n_angular;
    for (int q = 0; q < ang.n; ++q) {
      ang.off[q] = kernels->ang_off[q];
      ang.w[q] = kernels->ang_w[q];
    }
    fused = glb::fused_supported(r, r > 0 ? kernels->sep.data() : nullptr, ang, t->c) && (t->halo < 0 || ang.n / 2 <= t->halo);
  }
  // TMA descriptor over the source buffer; none for a row pitch TMA cannot
  // stride (odd W: 8*W is not a multiple of 16), where the fused kernel
  // loads its boxes with cp.async instead
  const CUtensorMap* tm = nullptr;
  if (fused) {
    int bw = 0, bh = 0;
    glb::fused_box(r, ang.n / 2, &bw, &bh);
    tm = tensor_tmap(t, src, bw, bh);
  }
  // wall-crossing mask (extension, wall.hpp): the fused kernel takes it when
  // its per-window table holds this step's motion vectors (TMA loads only);
  // anything else runs the generic chain, which tests every tap exactly
  a.wall = ctx->wall_mask;
  if (a.wall && fused) {
    thread_local std::vector<double> wm;
    const int planes = t->halo >= 0 ? t->c + 2 * t->halo : t->c;
    wm.resize(2 * static_cast<size_t>(planes));
    if (t->halo >= 0) {
      const double dtheta = 2.0 * M_PI / t->c_total;
      for (int q = 0; q < planes; ++q) {
        const int k = ((t->c_begin - t->halo + q) % t->c_total + t->c_total) % t->c_total;
        glb::motion_table(u, v, k, 1, t->theta_t, dtheta, t->cell, wm.data() + 2 * q);
      }
    } else {
      glb::motion_table(u, v, 0, t->c, t->theta_t, 2.0 * M_PI / t->c, t->cell, wm.data());
    }
    if (tm == nullptr || !glb::fused_wall_fits(wm.data(), planes)) fused = false;
  }
  if (ctx->path == GL_PATH_FUSED && !fused) {
    fail(GL_E_INVALID, "fused path requested but unsupported for this kernel set/grid");
  }
  ENQ_T(2);
  // motion vectors (host libm): carried in the launch parameters on the
  // fused path, otherwise uploaded through the pinned ring
  thread_local std::vector<double> hm;
  if (t->halo >= 0) {
    // theta-slab shard: one motion vector per storage plane (global channel
    // (c_begin - halo + q) mod c_total), carried in the launch parameters
    if (!fused) fail(GL_E_INVALID, "sharded tensors need the fused path (separable/impulse kernels, H <= halo)");
    const int planes = t->c + 2 * t->halo;
    hm.resize(2 * static_cast<size_t>(planes));
    const double dtheta = 2.0 * M_PI / t->c_total;
    for (int q = 0; q < planes; ++q) {
      const int k = ((t->c_begin - t->halo + q) % t->c_total + t->c_total) % t->c_total;
      glb::motion_table(u, v, k, 1, t->theta_t, dtheta, t->cell, hm.data() + 2 * q);
    }
    a.h_motion = hm.data();
    a.motion = nullptr;
    a.halo = t->halo;
    a.full_shard = t->c == t->c_total;
    if (fused && t->peer_lo_buf[src] != nullptr) {
      if (tm != nullptr) {
        int bw = 0, bh = 0;
        glb::fused_box(r, ang.n / 2, &bw, &bh);
        a.tmap_lo = tensor_tmap_at(t, t->peer_lo_buf[src], t->peer_lo_count + 2 * t->halo, bw, bh);
        a.tmap_hi = tensor_tmap_at(t, t->peer_hi_buf[src], t->peer_hi_count + 2 * t->halo, bw, bh);
        if (a.tmap_lo == nullptr || a.tmap_hi == nullptr) fail(GL_E_CUDA, "tensor map over a peer buffer failed");
      }
      a.src_lo = t->peer_lo_buf[src];
      a.src_hi = t->peer_hi_buf[src];
      a.lo_add = t->peer_lo_count;
    }
  } else if (fused) {
    hm.resize(2 * static_cast<size_t>(t->c));
    glb::motion_table(u, v, 0, t->c, t->theta_t, 2.0 * M_PI / t->c, t->cell, hm.data());
    a.h_motion = hm.data();
    a.motion = nullptr;
  } else {
    a.motion = upload_motion(ctx, t, u, v);
  }
  // per-step device time: cudaEventRecord costs ~2.6 us of host time each
  // (measured, tools/probe_launch_params.cu), so the begin/end pair is only
  // recorded when asked for (gl_context_set_step_timing, gl_context_time_steps)
  ENQ_T(3);
  const bool sampled = ctx->timing && (ctx->tstep++ % static_cast<unsigned>(ctx->tstride)) == 0;
  const int tslot = (sampled && ctx->tcount < gl_context::kTimers) ? ctx->tcount++ : -1;
  const bool events = tslot >= 0 || ctx->step_events;
  if (events) CK(cudaEventRecord(tslot >= 0 ? ctx->tev[2 * tslot] : ctx->ev_begin, ctx->stream));
  if (fused) {
    // r == 0 (impulse) kernels have no separable taps; the fused variant
    // then skips the spatial passes entirely
    const double one = 1.0;
    glb::launch_fused_step(ctx, a, tm, r > 0 ? kernels->sep.data() : &one, r, ang,
                           t->clean[src] && ctx->allow_fast);
    ENQ_T(4);
  } else {
    const size_t n = elems_of(t);
    ensure_scratch(ctx, n);
    glb::launch_shift_mask(ctx, a, ctx->d_s, 1);
    const double* D = ctx->d_s;
    if (kernels->info.separable) {
      glb::SepTaps taps{};
      for (int q = 0; q < 2 * r + 1; ++q) taps.t[q] = kernels->sep[q];
      // rows into d_d, columns back into d_s (S is free after phase 1)
      glb::launch_conv_separable(ctx, ctx->d_s, ctx->d_d, ctx->d_s, t->w, t->h,
                                 t->c, taps, r);
    } else if (r > 0) {
      glb::launch_conv_dense(ctx, ctx->d_s, ctx->d_d, t->w, t->h, t->c,
                             kk->d_spatial, r, kernels->info.channels);
      D = ctx->d_d;
    }
    glb::launch_angular(ctx, a, D, kk->d_ang_off, kk->d_ang_w,
                        kernels->info.n_angular);
    glb::launch_step_finalize(ctx, a);
  }
  CK(cudaGetLastError());
  if (events) {
    CK(cudaEventRecord(tslot >= 0 ? ctx->tev[2 * tslot + 1] : ctx->ev_end, ctx->stream));
    if (tslot >= 0) {
      ctx->ev_begin_last = ctx->tev[2 * tslot];
      ctx->ev_end_last = ctx->tev[2 * tslot + 1];
    } else {
      ctx->ev_begin_last = ctx->ev_begin;
      ctx->ev_end_last = ctx->ev_end;
    }
  }
  t->clean[dst] = t->clean[src];  // clean in -> clean out (non-negative weights)
  t->cur = dst;
  t->theta_t = t->theta_t + w;  // belief_tensor.cpp:478
  ENQ_T(5);
#ifdef GL_EXPERIMENT_ENV
  if (g_enq.n % 1000 == 0 && getenv("GL_DEBUG_ENQUEUE")) {
    const long n = g_enq.n;
    fprintf(stderr, "enqueue_step host ns/call: checks+guard %.0f | kernels %.0f | fused+tmap %.0f | motion %.0f | launch %.0f | tail %.0f (n=%ld)\n",
            g_enq.ns[0] / n, g_enq.ns[1] / n, g_enq.ns[2] / n, g_enq.ns[3] / n, g_enq.ns[4] / n, g_enq.ns[5] / n, n);
  }
#endif
}

gl_status gl_step(gl_context* ctx, gl_tensor* t, double u, double v, double w,
                  const gl_map* map, const gl_kernels* kernels,
                  const gl_activation* act) {
  // The finalising kernel also writes the status into the context's mapped
  // pinned word, so the synchronous call is enqueue + stream sync (a
  // device-to-host copy of the step state costs ~8 us more per step at
  // 256^2; tools/e2e_probe.py). A partial theta shard's status is only final
  // after gl_shard_finalize: it keeps the copy.
  const bool mapped = ctx && t && ctx->h_status && (t->halo < 0 || t->c == t->c_total);
  gl_status st = guard([&] {
    if (mapped) *reinterpret_cast<volatile int*>(ctx->h_status) = -1;  // not yet published
    enqueue_step(ctx, t, u, v, w, map, kernels, act, mapped);
  });
  if (st != GL_OK) return st;
  st = guard([&] {
    gl_status s = GL_E_RUNTIME;
    if (mapped) {
      // wait on the published word itself (the last CTA writes it after every
      // other CTA's output is done; later work stays stream-ordered), with a
      // stream query now and then so a failed launch cannot hang the caller
      DeviceGuard g(ctx->device);
      volatile int* hs = reinterpret_cast<volatile int*>(ctx->h_status);
      for (unsigned spins = 1; *hs == -1; ++spins) {
        if ((spins & 1023u) == 0) {
          const cudaError_t q = cudaStreamQuery(ctx->stream);
          if (q != cudaErrorNotReady) {
            CK(q);
            break;
          }
        }
        cpu_relax();
      }
      s = static_cast<gl_status>(*hs);
    }
    if (!mapped || (s != GL_OK && s != GL_E_EXTINGUISHED)) s = read_status(ctx, t);
    if (s == GL_E_EXTINGUISHED) {
      fail(GL_E_EXTINGUISHED, "belief tensor extinguished: no positive mass after step");
    }
  });
  return st;
}

gl_status gl_step_async(gl_context* ctx, gl_tensor* t, double u, double v,
                        double w, const gl_map* map, const gl_kernels* kernels,
                        const gl_activation* act) {
  return guard([&] { enqueue_step(ctx, t, u, v, w, map, kernels, act); });
}

// ---------------------------------------------------------- theta shards
gl_status gl_shard_init_uniform(gl_context* ctx, const gl_map* map, int c_total,
                                int c_begin, int c_end, int halo, gl_tensor** out) {
  return guard([&] {
    need(ctx && map && out, "null argument");
    need(c_total >= 4 && c_total % 2 == 0, "channel count must be even and >= 4");
    need(0 <= c_begin && c_begin < c_end && c_end <= c_total, "bad channel range");
    need(halo >= 0 && 2 * halo < c_total, "bad halo");
    need(map->free_count > 0, "map has no free cells to initialize from");
    DeviceGuard g(ctx->device);
    TensorPtr t = new_tensor(ctx, map->w, map->h, c_end - c_begin, map->res, map->ox, map->oy, halo,
                             c_total, c_begin);
    // every storage plane (interior and halo) starts as the free indicator
    glb::launch_init_uniform(ctx, t->d_buf[0], map->d_occ, map->w, map->h, t->c + 2 * halo);
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaGetLastError());
    *out = t.release();
  });
}

gl_status gl_shard_info(const gl_tensor* t, int* c_total, int* c_begin, int* c_count, int* halo) {
  return guard([&] {
    need(t, "null tensor");
    if (c_total) *c_total = t->c_total;
    if (c_begin) *c_begin = t->c_begin;
    if (c_count) *c_count = t->c;
    if (halo) *halo = t->halo;
  });
}

gl_status gl_tensor_plane_ptr(gl_context* ctx, gl_tensor* t, int q, double** dptr) {
  return guard([&] {
    need(ctx && t && dptr, "null argument");
    need(q >= 0 && q < t->c + 2 * halo_of(t), "storage plane out of range");
    *dptr = t->d_buf[t->cur] + plane_of(t) * q;  // raw: a pending rescale stays pending
  });
}

gl_status gl_tensor_max_ptr(gl_context* ctx, gl_tensor* t, unsigned long long** dptr) {
  return guard([&] {
    need(ctx && t && dptr, "null argument");
    *dptr = &t->d_block->step.gmax_bits;
  });
}

gl_status gl_shard_finalize(gl_context* ctx, gl_tensor* t) {
  return guard([&] {
    need(ctx && t, "null argument");
    need(t->halo >= 0, "not a sharded tensor");
    if (t->c == t->c_total) return;  // one rank: the step kernel finalised already
    DeviceGuard g(ctx->device);
    glb::StepArgs a{};
    a.step_state = &t->d_block->step;
    a.dst_state = &t->d_block->buf[t->cur];  // the step already flipped cur
    glb::launch_step_finalize(ctx, a);
    CK(cudaGetLastError());
  });
}

gl_status gl_shard_set_peers(gl_context* ctx, gl_tensor* t, void* lo0, void* lo1, int lo_count,
                             void* hi0, void* hi1, int hi_count) {
  return guard([&] {
    need(ctx && t, "null argument");
    need(t->halo >= 0, "not a sharded tensor");
    const bool none = !lo0 && !lo1 && !hi0 && !hi1;
    need(none || (lo0 && lo1 && hi0 && hi1), "peer buffers must be given for both neighbours and buffers");
    need(none || (lo_count >= t->halo && hi_count >= t->halo), "a neighbour holds fewer channels than the halo");
    for (int b = 0; b < 2; ++b) {
      t->peer_lo_buf[b] = static_cast<double*>(b ? lo1 : lo0);
      t->peer_hi_buf[b] = static_cast<double*>(b ? hi1 : hi0);
    }
    t->peer_lo_count = none ? 0 : lo_count;
    t->peer_hi_count = none ? 0 : hi_count;
  });
}

gl_status gl_tensor_buffer_ptr(gl_context* ctx, gl_tensor* t, int buf, int q, double** dptr) {
  return guard([&] {
    need(ctx && t && dptr, "null argument");
    need(buf == 0 || buf == 1, "buffer index must be 0 or 1");
    need(q >= 0 && q < t->c + 2 * halo_of(t), "storage plane out of range");
    *dptr = t->d_buf[buf] + plane_of(t) * q;
  });
}

gl_status gl_tensor_current_buffer(const gl_tensor* t, int* buf) {
  return guard([&] {
    need(t && buf, "null argument");
    *buf = t->cur;
  });
}

gl_status gl_ipc_get_handle(gl_context* ctx, gl_tensor* t, int buf, void* handle64) {
  return guard([&] {
    need(ctx && t && handle64, "null argument");
    need(buf == 0 || buf == 1, "buffer index must be 0 or 1");
    DeviceGuard g(ctx->device);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, t->d_buf[buf]));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof(h));
  });
}

gl_status gl_ipc_open(gl_context* ctx, const void* handle64, void** dptr) {
  return guard([&] {
    need(ctx && handle64 && dptr, "null argument");
    DeviceGuard g(ctx->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    CK(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

gl_status gl_ipc_close(gl_context* ctx, void* dptr) {
  return guard([&] {
    need(ctx && dptr, "null argument");
    DeviceGuard g(ctx->device);
    CK(cudaIpcCloseMemHandle(dptr));
  });
}

gl_status gl_tensor_copy_planes(gl_context* ctx, gl_tensor* dst, int dst_q, gl_tensor* src,
                                int src_q, int count) {
  return guard([&] {
    need(ctx && dst && src, "null argument");
    need(dst->w == src->w && dst->h == src->h, "plane sizes differ");
    need(count >= 0 && dst_q >= 0 && src_q >= 0 && dst_q + count <= dst->c + 2 * halo_of(dst) &&
             src_q + count <= src->c + 2 * halo_of(src),
         "plane range out of bounds");
    DeviceGuard g(ctx->device);
    const size_t plane = plane_of(dst);
    CK(cudaMemcpyAsync(dst->d_buf[dst->cur] + plane * dst_q, src->d_buf[src->cur] + plane * src_q,
                       plane * count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  });
}

gl_status gl_tensor_status(gl_context* ctx, gl_tensor* t) {
  return guard([&] {
    need(ctx && t, "null argument");
    DeviceGuard g(ctx->device);
    if (read_status(ctx, t) == GL_E_EXTINGUISHED) {
      fail(GL_E_EXTINGUISHED, "belief tensor extinguished: no positive mass after step");
    }
  });
}

void* ensure_host_misc(gl_context* ctx, size_t bytes);  // below

gl_status gl_tensors_status(gl_context* ctx, gl_tensor* const* ts, int n, int* statuses) {
  return guard([&] {
    need(ctx && (n == 0 || (ts && statuses)) && n >= 0, "null argument");
    DeviceGuard g(ctx->device);
    if (n == 0) return;
    // one gather kernel per 64 tensors into device scratch, one copy back, one sync
    int* d_out = static_cast<int*>(ensure_misc(ctx, sizeof(int) * static_cast<size_t>(n) + 64));
    int* h_out = static_cast<int*>(ensure_host_misc(ctx, sizeof(int) * static_cast<size_t>(n) + 64));
    for (int i0 = 0; i0 < n; i0 += glb::kStatusGather) {
      glb::StatusPtrs ptrs{};
      ptrs.n = std::min(glb::kStatusGather, n - i0);
      for (int i = 0; i < ptrs.n; ++i) {
        need(ts[i0 + i] != nullptr, "null tensor");
        ptrs.p[i] = &ts[i0 + i]->d_block->step.status;
      }
      glb::launch_gather_status(ctx, ptrs, d_out + i0);
    }
    CK(cudaMemcpyAsync(h_out, d_out, sizeof(int) * static_cast<size_t>(n), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    bool ext = false;
    for (int i = 0; i < n; ++i) {
      statuses[i] = h_out[i];
      ext = ext || h_out[i] == GL_E_EXTINGUISHED;
    }
    if (ext) fail(GL_E_EXTINGUISHED, "a belief tensor extinguished: no positive mass after step");
  });
}

gl_status gl_apply_motion(gl_context* ctx, gl_tensor* t, double u, double v,
                          double w) {
  return guard([&] {
    need(ctx && t, "null argument");
    DeviceGuard g(ctx->device);
    glb::StepArgs a{};
    const int src = t->cur, dst = 1 - t->cur;
    a.src = t->d_buf[src];
    a.src_state = &t->d_block->buf[src];
    a.w = t->w;
    a.h = t->h;
    a.c = t->c;
    a.motion = upload_motion(ctx, t, u, v);
    glb::launch_shift_mask(ctx, a, t->d_buf[dst], 2);
    CK(cudaMemsetAsync(&t->d_block->buf[dst], 0, sizeof(glb::BufState), ctx->stream));
    CK(cudaGetLastError());
    t->clean[dst] = t->clean[src];
    t->cur = dst;
    t->theta_t = t->theta_t + w;
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

// ------------------------------------------------------------ read-outs
static double wrap_angle(double a) {  // geometry.hpp:8-13
  a = std::fmod(a, 2.0 * M_PI);
  if (a < -M_PI) a += 2.0 * M_PI;
  if (a >= M_PI) a -= 2.0 * M_PI;
  return a;
}

gl_status gl_belief_map(gl_context* ctx, gl_tensor* t, double* host_out) {
  return guard([&] {
    need(ctx && t && host_out, "null argument");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    double* d = static_cast<double*>(ensure_misc(ctx, plane_of(t) * sizeof(double)));
    glb::launch_belief_map(ctx, interior(t), t->w, t->h, t->c, d);
    CK(cudaMemcpyAsync(host_out, d, plane_of(t) * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

gl_status gl_argmax(gl_context* ctx, gl_tensor* t, gl_pose_estimate* out) {
  return guard([&] {
    need(ctx && t && out, "null argument");
    DeviceGuard g(ctx->device);
    const ArgmaxExact res = argmax_exact(ctx, t, 0.0);
    if (!(res.v > 0.0)) fail(GL_E_EXTINGUISHED, "argmax on an all-zero belief tensor");
    const size_t plane = plane_of(t);
    const size_t p = static_cast<size_t>(res.idx) % plane;
    out->k = static_cast<int>(static_cast<size_t>(res.idx) / plane);
    out->i = static_cast<int>(p % t->w);
    out->j = static_cast<int>(p / t->w);
    out->x = t->ox + (out->i + 0.5) * t->cell;
    out->y = t->oy + (out->j + 0.5) * t->cell;
    out->theta = wrap_angle(out->k * (2.0 * M_PI / t->c) + t->theta_t);
    out->confidence = res.total > 0.0 ? res.v / res.total : 0.0;  // belief_tensor.cpp:539
  });
}

// misc scratch of a dither call: [bm plane] [n, mass, flag] [cells]
// [sequential-sum scratch]. Callers size it with this BEFORE placing the
// plane in it (ensure_misc reallocates, and a reallocation loses contents).
static size_t dither_cells_bytes(size_t plane, int cap) {
  // device capacity: every cell could emit at most once
  const size_t dcap = std::min<size_t>(plane, static_cast<size_t>(std::max(cap, 1)));
  return (dcap * 8 + 255) & ~static_cast<size_t>(255);
}
static size_t dither_misc_bytes(size_t plane, int cap) {
  return plane * sizeof(double) + 64 + dither_cells_bytes(plane, cap) + glb::seq_sum_scratch_bytes(plane);
}

static void run_dither(gl_context* ctx, const double* d_bm, int w, int h,
                       int budget, int32_t* cells, int cap, int* n,
                       double* mass) {
  need(budget >= 1, "sample budget must be >= 1");
  need(cap >= 0 && n && mass, "bad output arguments");
  const size_t plane = static_cast<size_t>(w) * h;
  const size_t dcap = std::min<size_t>(plane, static_cast<size_t>(std::max(cap, 1)));
  const size_t cells_bytes = dither_cells_bytes(plane, cap);
  need(ctx->misc_bytes >= dither_misc_bytes(plane, cap), "internal: dither scratch not sized by the caller");
  char* base = static_cast<char*>(ctx->d_misc);
  // layout: [bm plane (if copied)] [n, mass, flag] [cells] [sequential-sum scratch]
  int* d_n = reinterpret_cast<int*>(base + plane * sizeof(double));
  double* d_mass = reinterpret_cast<double*>(base + plane * sizeof(double) + 8);
  int* d_inv = reinterpret_cast<int*>(base + plane * sizeof(double) + 16);
  int* d_cells = reinterpret_cast<int*>(base + plane * sizeof(double) + 64);
  void* d_sum = base + plane * sizeof(double) + 64 + cells_bytes;
  glb::launch_dither(ctx, d_bm, w, h, budget, d_cells, static_cast<int>(dcap), d_n, d_mass, d_inv, d_sum);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(n, d_n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(mass, d_mass, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int got = std::min(*n, cap);
  if (got > 0 && cells) {
    CK(cudaMemcpyAsync(cells, d_cells, sizeof(int32_t) * 2 * got,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
}

gl_status gl_dither(gl_context* ctx, const double* belief_map, int width,
                    int height, int budget, int32_t* cells, int cap, int* n,
                    double* source_mass) {
  return guard([&] {
    need(ctx && belief_map, "null argument");
    need(width >= 1 && height >= 1, "bad belief map size");
    DeviceGuard g(ctx->device);
    const size_t plane = static_cast<size_t>(width) * height;
    double* d = static_cast<double*>(ensure_misc(ctx, dither_misc_bytes(plane, cap)));
    CK(cudaMemcpyAsync(d, belief_map, plane * sizeof(double),
                       cudaMemcpyHostToDevice, ctx->stream));
    run_dither(ctx, d, width, height, budget, cells, cap, n, source_mass);
  });
}

gl_status gl_dither_device(gl_context* ctx, const double* d_plane, int width,
                           int height, int budget, int32_t* cells, int cap, int* n,
                           double* source_mass) {
  return guard([&] {
    need(ctx && d_plane, "null argument");
    need(width >= 1 && height >= 1, "bad belief map size");
    DeviceGuard g(ctx->device);
    ensure_misc(ctx, dither_misc_bytes(static_cast<size_t>(width) * height, cap));
    run_dither(ctx, d_plane, width, height, budget, cells, cap, n, source_mass);
  });
}

gl_status gl_dither_tensor(gl_context* ctx, gl_tensor* t, int budget,
                           int32_t* cells, int cap, int* n,
                           double* source_mass) {
  return guard([&] {
    need(ctx && t, "null argument");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    const size_t plane = plane_of(t);
    double* d = static_cast<double*>(ensure_misc(ctx, dither_misc_bytes(plane, cap)));
    glb::launch_belief_map(ctx, interior(t), t->w, t->h, t->c, d);
    run_dither(ctx, d, t->w, t->h, budget, cells, cap, n, source_mass);
  });
}

// ----------------------------------------------------------- observation
namespace {

// Per-cell likelihood-field beam score with the reference's libm:
// log((1 - f) * exp(-d*d*inv2s2) + f) (observation.cpp:101-106), cached on
// the field for the last LikelihoodParams used.
struct ObsTables {
  const double* d_score;
  double oob;
};

void* ensure_kind(gl_context* ctx, size_t n) {
  if (ctx->kind_bytes < n) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->d_kind) CK(cudaFree(ctx->d_kind));
    ctx->d_kind = nullptr;
    CK(cudaMalloc(&ctx->d_kind, n));
    ctx->kind_bytes = n;
  }
  return ctx->d_kind;
}

// The geometric mean's final exp with the host's glibc, like the reference
// (observation.cpp:110): the kernel left the exponent and a case code.
// A few persistent host workers for the glibc exp of an observation's
// likelihoods (<= 512 * Theta values; one thread takes ~0.6 ms for 37K):
// every worker calls the same glibc exp on the same CPU, so the results are
// the single-threaded ones bit for bit.
class HostPool {
 public:
  static HostPool& get() {
    // never destroyed: its detached workers block on its condition variable
    // for the life of the process (destroying it at exit could wait on them)
    static HostPool* pool = new HostPool;
    return *pool;
  }
  // run f(begin, end) over [0, n) in `parts` slices; the caller takes slice 0
  void run(size_t n, int parts, const std::function<void(size_t, size_t)>& f) {
    parts = std::max(1, std::min<int>(parts, static_cast<int>(workers_.size()) + 1));
    if (parts == 1) {
      f(0, n);
      return;
    }
    std::unique_lock<std::mutex> lk(call_mu_);  // one parallel call at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &f;
      n_ = n;
      parts_ = parts;
      next_ = 1;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0, n / parts);
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const int k = static_cast<int>(std::min<unsigned>(hw > 1 ? hw - 1 : 0, 15));
    for (int i = 0; i < k; ++i) workers_.emplace_back([this] { loop(); });
    for (auto& t : workers_) t.detach();  // live for the process
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return gen_ != seen && next_ < parts_; });
      seen = gen_;
      const int part = next_++;
      const auto* f = job_;
      const size_t n = n_;
      const int parts = parts_;
      g.unlock();
      (*f)(n * part / parts, n * (part + 1) / parts);
      g.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t, size_t)>* job_ = nullptr;
  size_t n_ = 0;
  int parts_ = 0, next_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
};

// the context's pinned host scratch (grown on demand; contents not kept)
void* ensure_host_misc(gl_context* ctx, size_t bytes) {
  if (ctx->h_misc_bytes < bytes) {
    if (ctx->h_misc) {
      CK(cudaStreamSynchronize(ctx->stream));
      CK(cudaFreeHost(ctx->h_misc));
      ctx->h_misc = nullptr;
      ctx->h_misc_bytes = 0;
    }
    CK(cudaMallocHost(&ctx->h_misc, bytes));
    ctx->h_misc_bytes = bytes;
  }
  return ctx->h_misc;
}

void finish_likelihoods_on_host(gl_context* ctx, double* d_L, const uint8_t* d_kind, size_t n,
                                double floor_w) {
  // pinned staging: the two copies each way run at full PCIe speed
  char* h = static_cast<char*>(ensure_host_misc(ctx, n * sizeof(double) + n + 64));
  double* l = reinterpret_cast<double*>(h);
  uint8_t* kind = reinterpret_cast<uint8_t*>(h + n * sizeof(double));
  CK(cudaMemcpyAsync(l, d_L, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(kind, d_kind, n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const uint8_t* kd = kind;
  const std::function<void(size_t, size_t)> fin = [=](size_t b, size_t e) {
    for (size_t q = b; q < e; ++q) l[q] = kd[q] == 0 ? std::exp(l[q]) : (kd[q] == 1 ? floor_w : 1.0);
  };
  HostPool::get().run(n, static_cast<int>(n / 4096), fin);
  CK(cudaMemcpyAsync(d_L, l, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
}

ObsTables obs_tables(gl_context* ctx, const gl_field* cf, gl_likelihood p) {
  auto* f = const_cast<gl_field*>(cf);
  if (!(f->score_sigma == p.sigma_hit && f->score_floor == p.weight_floor && f->d_score)) {
    const double fl = p.weight_floor;
    const double inv2s2 = 1.0 / (2.0 * p.sigma_hit * p.sigma_hit);
    // The field takes few distinct values (sqrt(n) * res for the integer
    // squared cell distances n present), so a direct-mapped memo on the
    // value's bits evaluates the host-libm expression once per distinct d
    // (same input, same glibc result: bit-identical to the per-cell loop).
    std::vector<double> score(f->values.size());
    constexpr int kMemoBits = 16;
    std::vector<uint64_t> memo_key(size_t(1) << kMemoBits, ~0ull);
    std::vector<double> memo_val(size_t(1) << kMemoBits);
    for (size_t q = 0; q < f->values.size(); ++q) {
      const double d = f->values[q];
      uint64_t bits;
      std::memcpy(&bits, &d, 8);
      const size_t slot = static_cast<size_t>((bits * 0x9E3779B97F4A7C15ull) >> (64 - kMemoBits));
      if (memo_key[slot] != bits) {
        const double gauss = std::exp(-d * d * inv2s2);  // observation.cpp:101-106
        memo_val[slot] = std::log((1.0 - fl) * gauss + fl);
        memo_key[slot] = bits;
      }
      score[q] = memo_val[slot];
    }
    if (!f->d_score) CK(cudaMalloc(&f->d_score, score.size() * sizeof(double)));
    CK(cudaMemcpy(f->d_score, score.data(), score.size() * sizeof(double), cudaMemcpyHostToDevice));
    f->score_oob = std::log((1.0 - fl) * 0.0 + fl);
    f->score_sigma = p.sigma_hit;
    f->score_floor = p.weight_floor;
  }
  return ObsTables{f->d_score, f->score_oob};
}

}  // namespace

gl_status gl_scan_likelihood(gl_context* ctx, const gl_map* map,
                             const gl_field* field, double x, double y,
                             double theta, const double* angles,
                             const double* ranges, int n_beams,
                             double max_range, gl_likelihood params,
                             double* out) {
  // Single-pose convenience: one (sample, channel) evaluated by the same
  // device kernel as observation_update, with a 1-channel pose table.
  return guard([&] {
    need(ctx && map && field && out, "null argument");
    need(n_beams >= 1 && angles && ranges, "scan must have matching, nonempty beams");
    DeviceGuard g(ctx->device);
    const ObsTables tb = obs_tables(ctx, field, params);
    const int stride = std::max(1, params.beam_stride);
    std::vector<double> dirs, reach;
    const double half = 0.5 * map->res;
    for (int b = 0; b < n_beams; b += stride) {
      if (ranges[b] >= max_range - 1e-9) continue;
      const double a = theta + angles[b];
      dirs.push_back(std::cos(a));
      dirs.push_back(std::sin(a));
      reach.push_back(ranges[b] + half);
    }
    // pose in world coords: pass as a "sample" at fractional cell via origin
    // shift: tox + (0 + 0.5)*cell == x  <=>  tox = x - 0.5*cell with cell = 1
    const int ns = static_cast<int>(reach.size());
    size_t bytes = 64 + (ns + 1) * 24 + 64;
    char* d = static_cast<char*>(ensure_misc(ctx, bytes));
    int* d_s = reinterpret_cast<int*>(d);
    double* d_L = reinterpret_cast<double*>(d + 16);
    double* d_reach = reinterpret_cast<double*>(d + 64);
    double2* d_dir = reinterpret_cast<double2*>(d + 64 + 8 * (ns + 1) + 8);
    d_dir = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(d_dir) + 15) & ~uintptr_t(15));
    const int zero2[2] = {0, 0};
    CK(cudaMemcpyAsync(d_s, zero2, sizeof(zero2), cudaMemcpyHostToDevice, ctx->stream));
    if (ns > 0) {
      CK(cudaMemcpyAsync(d_reach, reach.data(), ns * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(d_dir, dirs.data(), ns * 2 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
    // x = tox + (0 + 0.5) * 0.0 ... use cell = 0 so the pose is exactly (x, y)
    uint8_t* d_kind = ctx->host_exp ? static_cast<uint8_t*>(ensure_kind(ctx, 1)) : nullptr;
    glb::launch_likelihoods(ctx, map->d_occ, tb.d_score, tb.oob, map->w, map->h,
                            map->res, map->ox, map->oy, 0.0, x, y, d_s, 1, 1,
                            d_dir, ns, d_reach, params.weight_floor, d_L, d_kind);
    CK(cudaGetLastError());
    if (ctx->host_exp) finish_likelihoods_on_host(ctx, d_L, d_kind, 1, params.weight_floor);
    CK(cudaMemcpyAsync(out, d_L, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  });
}

// observation_update's device work. shard: likelihoods of ALL c_total
// channels (every rank forms the same sequential mean), multiply only the
// shard's own channels, leave the local max in the max slot for the
// cross-rank all-reduce (gl_shard_observe_finalize finishes).
static void observe_impl(gl_context* ctx, gl_tensor* t, const int32_t* cells, int n,
                         const double* angles, const double* ranges, int n_beams,
                         double max_range, const gl_map* map, const gl_field* field,
                         gl_likelihood params, bool shard) {
  {
    need(ctx && t && map && field, "null argument");
    if (n == 0) return;  // observation.cpp:117
    need(cells != nullptr && n > 0, "bad sample set");
    need(n_beams >= 1 && angles && ranges, "scan must have matching, nonempty beams");
    DeviceGuard g(ctx->device);
    const ObsTables tb = obs_tables(ctx, field, params);
    const int C = shard ? t->c_total : t->c;
    // scored beams and per-(channel, beam) directions with host libm
    const int stride = std::max(1, params.beam_stride);
    std::vector<int> scored;
    for (int b = 0; b < n_beams; b += stride)
      if (!(ranges[b] >= max_range - 1e-9)) scored.push_back(b);
    const int ns = static_cast<int>(scored.size());
    const double half = 0.5 * map->res;
    const double dtheta = 2.0 * M_PI / C;
    std::vector<double> reach(std::max(ns, 1));
    for (int q = 0; q < ns; ++q) reach[q] = ranges[scored[q]] + half;
    std::vector<double> dirs(static_cast<size_t>(C) * std::max(ns, 1) * 2);
    for (int k = 0; k < C; ++k) {
      const double ak = k * dtheta + t->theta_t;  // channel_angle(k)
      for (int q = 0; q < ns; ++q) {
        const double a = ak + angles[scored[q]];
        dirs[(static_cast<size_t>(k) * ns + q) * 2] = std::cos(a);
        dirs[(static_cast<size_t>(k) * ns + q) * 2 + 1] = std::sin(a);
      }
    }
    const size_t nL = static_cast<size_t>(n) * C;
    size_t off_s = 0;
    size_t off_L = (off_s + sizeof(int) * 2 * n + 255) & ~size_t(255);
    size_t off_mean = (off_L + sizeof(double) * nL + 255) & ~size_t(255);
    size_t off_reach = off_mean + 256;
    size_t off_dir = (off_reach + sizeof(double) * reach.size() + 255) & ~size_t(255);
    size_t off_sum = (off_dir + sizeof(double) * dirs.size() + 255) & ~size_t(255);
    size_t total = off_sum + glb::seq_sum_scratch_bytes(nL) + 256;
    char* d = static_cast<char*>(ensure_misc(ctx, total));
    int* d_s = reinterpret_cast<int*>(d + off_s);
    double* d_L = reinterpret_cast<double*>(d + off_L);
    double* d_mean = reinterpret_cast<double*>(d + off_mean);
    double* d_reach = reinterpret_cast<double*>(d + off_reach);
    double2* d_dir = reinterpret_cast<double2*>(d + off_dir);
    CK(cudaMemcpyAsync(d_s, cells, sizeof(int) * 2 * n, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d_reach, reach.data(), sizeof(double) * reach.size(), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(d_dir, dirs.data(), sizeof(double) * dirs.size(), cudaMemcpyHostToDevice, ctx->stream));
    materialize(ctx, t);
    uint8_t* d_kind = ctx->host_exp ? static_cast<uint8_t*>(ensure_kind(ctx, nL)) : nullptr;
    glb::launch_likelihoods(ctx, map->d_occ, tb.d_score, tb.oob, map->w, map->h,
                            map->res, map->ox, map->oy, t->cell, t->ox, t->oy, d_s,
                            n, C, d_dir, ns, d_reach, params.weight_floor, d_L, d_kind);
    if (ctx->host_exp) finish_likelihoods_on_host(ctx, d_L, d_kind, nL, params.weight_floor);
    glb::launch_observe_apply(ctx, interior(t), t->w, t->h, t->c, shard ? t->c_begin : 0, C, d_s, n,
                              d_L, d_mean, d + off_sum);
    glb::launch_plane_max(ctx, interior(t), elems_of(t), &t->d_block->step.gmax_bits);
    if (shard) {
      CK(cudaGetLastError());
      return;
    }
    glb::launch_observe_finalize(ctx, &t->d_block->step, &t->d_block->buf[t->cur]);
    CK(cudaGetLastError());
    if (read_status(ctx, t) == GL_E_EXTINGUISHED) {
      fail(GL_E_EXTINGUISHED, "observation update zeroed the tensor");
    }
  }
}

gl_status gl_observation_update(gl_context* ctx, gl_tensor* t,
                                const int32_t* cells, int n,
                                const double* angles, const double* ranges,
                                int n_beams, double max_range,
                                const gl_map* map, const gl_field* field,
                                gl_likelihood params) {
  return guard([&] {
    observe_impl(ctx, t, cells, n, angles, ranges, n_beams, max_range, map, field, params, false);
  });
}

gl_status gl_shard_observe(gl_context* ctx, gl_tensor* t, const int32_t* cells, int n,
                           const double* angles, const double* ranges, int n_beams,
                           double max_range, const gl_map* map, const gl_field* field,
                           gl_likelihood params) {
  return guard([&] {
    need(t && t->halo >= 0, "not a sharded tensor");
    observe_impl(ctx, t, cells, n, angles, ranges, n_beams, max_range, map, field, params, true);
  });
}

gl_status gl_shard_observe_finalize(gl_context* ctx, gl_tensor* t) {
  return guard([&] {
    need(ctx && t, "null argument");
    need(t->halo >= 0, "not a sharded tensor");
    DeviceGuard g(ctx->device);
    glb::launch_observe_finalize(ctx, &t->d_block->step, &t->d_block->buf[t->cur]);
    CK(cudaGetLastError());
    if (read_status(ctx, t) == GL_E_EXTINGUISHED) {
      fail(GL_E_EXTINGUISHED, "observation update zeroed the tensor");
    }
  });
}

gl_status gl_shard_belief_map(gl_context* ctx, gl_tensor* t, double* d_plane) {
  return guard([&] {
    need(ctx && t && d_plane, "null argument");
    need(t->halo >= 0, "not a sharded tensor");
    DeviceGuard g(ctx->device);
    materialize(ctx, t);
    glb::launch_belief_map(ctx, interior(t), t->w, t->h, t->c, d_plane);
    CK(cudaGetLastError());
  });
}

// diagnostics: [0] step epilogues that took the exact max (HIMAX fallback)
gl_status gl_debug_counters(gl_context* ctx, unsigned long long* out4) {
  return guard([&] {
    need(ctx && out4, "null argument");
    DeviceGuard g(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    glb::fused_counters(out4);
  });
}

// The reference's sequential sum (observation.cpp:16-17 order) of n host
// doubles computed on the device, bit-exact (the parallel binade scan that
// gives dither_samples its total; there the dither kernel's own sequential
// chain covers negative / non-finite planes).
gl_status gl_sequential_sum(gl_context* ctx, const double* host, size_t n, double* total) {
  return guard([&] {
    need(ctx && (host || n == 0) && total, "null argument");
    DeviceGuard g(ctx->device);
    const size_t xb = (n * sizeof(double) + 255) & ~static_cast<size_t>(255);
    char* base = static_cast<char*>(ensure_misc(ctx, 256 + xb + glb::seq_sum_scratch_bytes(n)));
    double* d_t = reinterpret_cast<double*>(base);
    int* d_inv = reinterpret_cast<int*>(base + 8);
    double* d_x = reinterpret_cast<double*>(base + 256);
    if (n) CK(cudaMemcpyAsync(d_x, host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(d_t, 0, sizeof(double), ctx->stream));
    glb::launch_seq_sum_big(ctx, d_x, n, d_t, d_inv, base + 256 + xb);
    int inv = 0;
    CK(cudaMemcpyAsync(total, d_t, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&inv, d_inv, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (inv) fail(GL_E_INVALID, "sequential_sum: values must be finite and >= 0");
  });
}

// ------------------------------------------------- raycast / simulate_scan
// Batches for trace generation: every ray on the device,
// bit-exact against raycast (occupancy_map.cpp:273-332) — the directions are
// glibc cos/sin evaluated on the host, as the reference evaluates them.
namespace {

void run_rays(gl_context* ctx, const gl_map* map, const std::vector<double>& xy, const std::vector<double>& dir,
              int beams, double max_range, const double* noise, double sigma, double* ranges, const char* what) {
  const size_t n_rays = dir.size() / 2, n_pose = xy.size() / 2;
  need(n_rays <= static_cast<size_t>(INT32_MAX), "too many rays in one batch");
  const size_t b_xy = 16 * n_pose, b_dir = 16 * n_rays, b_noise = noise ? 8 * n_rays : 0, b_r = 8 * n_rays;
  auto al = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  char* d = static_cast<char*>(ensure_misc(ctx, al(b_xy) + al(b_dir) + al(b_noise) + al(b_r) + 256));
  auto* d_xy = reinterpret_cast<double2*>(d);
  auto* d_dir = reinterpret_cast<double2*>(d + al(b_xy));
  auto* d_noise = noise ? reinterpret_cast<double*>(d + al(b_xy) + al(b_dir)) : nullptr;
  auto* d_r = reinterpret_cast<double*>(d + al(b_xy) + al(b_dir) + al(b_noise));
  auto* d_bad = reinterpret_cast<int*>(d + al(b_xy) + al(b_dir) + al(b_noise) + al(b_r));
  CK(cudaMemcpyAsync(d_xy, xy.data(), b_xy, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(d_dir, dir.data(), b_dir, cudaMemcpyHostToDevice, ctx->stream));
  if (noise) CK(cudaMemcpyAsync(d_noise, noise, b_noise, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(d_bad, 0, sizeof(int), ctx->stream));
  glb::launch_raycast_batch(ctx, map->d_occ, map->w, map->h, map->res, map->ox, map->oy, d_xy, d_dir,
                            static_cast<int>(n_rays), beams, max_range, d_noise, sigma, d_r, d_bad);
  CK(cudaGetLastError());
  int bad = 0;
  CK(cudaMemcpyAsync(ranges, d_r, b_r, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad) fail(GL_E_MAP_PARSE, what);
}

}  // namespace

gl_status gl_raycast(gl_context* ctx, const gl_map* map, const double* rays, int n, double max_range,
                     double* ranges) {
  return guard([&] {
    need(ctx && map && (n == 0 || (rays && ranges)), "null argument");
    need(n >= 0, "ray count must be >= 0");
    need(max_range > 0.0, "max_range must be > 0");  // occupancy_map.cpp:275
    if (n == 0) return;
    DeviceGuard g(ctx->device);
    std::vector<double> xy(2 * static_cast<size_t>(n)), dir(2 * static_cast<size_t>(n));
    for (int q = 0; q < n; ++q) {
      xy[2 * q] = rays[3 * q];
      xy[2 * q + 1] = rays[3 * q + 1];
      dir[2 * q] = std::cos(rays[3 * q + 2]);
      dir[2 * q + 1] = std::sin(rays[3 * q + 2]);
    }
    run_rays(ctx, map, xy, dir, 1, max_range, nullptr, 0.0, ranges, "raycast origin not in a free cell");
  });
}

gl_status gl_simulate_scans(gl_context* ctx, const gl_map* map, const double* poses, int n, int beam_count,
                            double fov, double max_range, double range_noise_sigma, const double* noise,
                            double* angles, double* ranges) {
  return guard([&] {
    need(ctx && map && (n == 0 || (poses && ranges)), "null argument");
    need(n >= 0, "pose count must be >= 0");
    need(beam_count >= 1, "beam_count must be >= 1");  // simulator.cpp:66
    // world_free(pose) for every pose first (simulator.cpp:67-70)
    for (int q = 0; q < n; ++q) {
      const double x = poses[3 * q], y = poses[3 * q + 1];
      const int i = static_cast<int>(std::floor((x - map->ox) / map->res));
      const int j = static_cast<int>(std::floor((y - map->oy) / map->res));
      if (!(i >= 0 && i < map->w && j >= 0 && j < map->h) || map->occ[static_cast<size_t>(j) * map->w + i]) {
        fail(GL_E_MAP_PARSE, "scan pose is not in free space");
      }
    }
    need(max_range > 0.0, "max_range must be > 0");  // the first raycast (occupancy_map.cpp:275)
    const bool full_circle = fov >= 2.0 * M_PI - 1e-9;
    std::vector<double> a(beam_count);
    for (int b = 0; b < beam_count; ++b) {
      if (beam_count == 1) {
        a[b] = 0.0;
      } else if (full_circle) {
        a[b] = -M_PI + b * (2.0 * M_PI / beam_count);  // endpoint-exclusive
      } else {
        a[b] = -fov / 2.0 + b * (fov / (beam_count - 1));
      }
    }
    if (angles) std::copy(a.begin(), a.end(), angles);
    if (n == 0) return;
    DeviceGuard g(ctx->device);
    const size_t rays = static_cast<size_t>(n) * beam_count;
    std::vector<double> xy(2 * static_cast<size_t>(n)), dir(2 * rays);
    for (int q = 0; q < n; ++q) {
      xy[2 * q] = poses[3 * q];
      xy[2 * q + 1] = poses[3 * q + 1];
      for (int b = 0; b < beam_count; ++b) {
        const double ang = poses[3 * q + 2] + a[b];  // raycast(map, x, y, pose.theta + a, ...)
        dir[2 * (static_cast<size_t>(q) * beam_count + b)] = std::cos(ang);
        dir[2 * (static_cast<size_t>(q) * beam_count + b) + 1] = std::sin(ang);
      }
    }
    const bool noisy = range_noise_sigma > 0.0;
    need(!noisy || noise, "range noise requested without the per-beam normal draws");
    run_rays(ctx, map, xy, dir, beam_count, max_range, noisy ? noise : nullptr, range_noise_sigma, ranges,
             "raycast origin not in a free cell");
  });
}

// -------------------------------------------------------- map difficulty
gl_status gl_map_difficulty(gl_context* ctx, const gl_map* map, const gl_field* field,
                            const gl_difficulty_config* cfg, double* out) {
  return guard([&] {
    need(ctx && map && field && cfg && out, "null argument");
    need(field->w == map->w && field->h == map->h, "field and map sizes differ");
    // simulate_scan / raycast / scan_likelihood argument checks
    need(cfg->beam_count >= 1, "beam_count must be >= 1");
    need(cfg->max_range > 0.0, "max_range must be > 0");
    need(cfg->beam_count <= glb::kMaxDifficultyBeams, "beam_count above 256 is not supported");
    need(cfg->theta_bins >= 0, "theta_bins must be >= 0");
    DeviceGuard g(ctx->device);
    const int W = map->w, H = map->h;
    const double res = map->res, ox = map->ox, oy = map->oy;
    const int stride = std::max(1, cfg->stride);
    std::vector<int> cells;  // (i, j) pairs, evaluation.cpp:28-33 order
    for (int j = 1; j < H - 1; j += stride)
      for (int i = 1; i < W - 1; i += stride)
        if (!map->occ[static_cast<size_t>(j) * W + i]) {
          cells.push_back(i);
          cells.push_back(j);
        }
    const int n = static_cast<int>(cells.size() / 2);
    if (n == 0) {
      *out = 0.0;
      return;
    }
    const int beams = cfg->beam_count, bins = cfg->theta_bins;
    auto cx_of = [&](int i) { return ox + (i + 0.5) * res; };
    auto cy_of = [&](int j) { return oy + (j + 0.5) * res; };
    std::vector<int> winner(n, 0);
    std::vector<double> ranges;
    if (bins > 0) {
      // beam angles (simulator.cpp:75-84) and host-libm direction tables
      std::vector<double> angles(beams);
      const bool full_circle = cfg->fov >= 2.0 * M_PI - 1e-9;
      for (int b = 0; b < beams; ++b) {
        if (beams == 1) {
          angles[b] = 0.0;
        } else if (full_circle) {
          angles[b] = -M_PI + b * (2.0 * M_PI / beams);
        } else {
          angles[b] = -cfg->fov / 2.0 + b * (cfg->fov / (beams - 1));
        }
      }
      std::vector<double> ray(2 * beams), dir(2 * static_cast<size_t>(bins) * beams);
      for (int b = 0; b < beams; ++b) {
        const double a = 0.0 + angles[b];  // query pose theta = 0
        ray[2 * b] = std::cos(a);
        ray[2 * b + 1] = std::sin(a);
      }
      for (int t = 0; t < bins; ++t) {
        const double ta = wrap_angle(2.0 * M_PI * t / bins);  // evaluation.cpp:37-39
        for (int b = 0; b < beams; ++b) {
          const double a = ta + angles[b];
          dir[2 * (static_cast<size_t>(t) * beams + b)] = std::cos(a);
          dir[2 * (static_cast<size_t>(t) * beams + b) + 1] = std::sin(a);
        }
      }
      const ObsTables tb = obs_tables(ctx, field, cfg->likelihood);
      // device buffers (one allocation)
      size_t off = 0;
      auto take = [&](size_t bytes) {
        const size_t o = off;
        off = (off + bytes + 255) & ~size_t(255);
        return o;
      };
      const size_t o_cells = take(sizeof(int) * cells.size()), o_ray = take(sizeof(double) * ray.size()),
                   o_dir = take(sizeof(double) * dir.size()),
                   o_rng = take(sizeof(double) * static_cast<size_t>(n) * beams),
                   o_bls = take(sizeof(double) * n), o_bix = take(sizeof(int) * n), o_cnt = take(sizeof(int) * n),
                   o_near = take(sizeof(int) * n), o_bad = take(sizeof(int));
      char* d = nullptr;
      CK(cudaMalloc(&d, off));
      std::unique_ptr<char, decltype(&cudaFree)> hold(d, &cudaFree);
      CK(cudaMemcpyAsync(d + o_cells, cells.data(), sizeof(int) * cells.size(), cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(d + o_ray, ray.data(), sizeof(double) * ray.size(), cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(d + o_dir, dir.data(), sizeof(double) * dir.size(), cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemsetAsync(d + o_near, 0, sizeof(int) * n, ctx->stream));
      CK(cudaMemsetAsync(d + o_bad, 0, sizeof(int), ctx->stream));
      glb::DifficultyArgs a{};
      a.occ = map->d_occ;
      a.score = tb.d_score;
      a.oob = tb.oob;
      a.w = W;
      a.h = H;
      a.res = res;
      a.ox = ox;
      a.oy = oy;
      a.cells = reinterpret_cast<const int2*>(d + o_cells);
      a.n = n;
      a.ray = reinterpret_cast<const double2*>(d + o_ray);
      a.dir = reinterpret_cast<const double2*>(d + o_dir);
      a.beams = beams;
      a.bins = bins;
      a.stride = std::max(1, cfg->likelihood.beam_stride);
      a.max_range = cfg->max_range;
      a.half_cell = 0.5 * res;
      a.ranges = reinterpret_cast<double*>(d + o_rng);
      a.best_ls = reinterpret_cast<double*>(d + o_bls);
      a.best_idx = reinterpret_cast<int*>(d + o_bix);
      a.counted = reinterpret_cast<int*>(d + o_cnt);
      a.near = reinterpret_cast<int*>(d + o_near);
      a.bad = reinterpret_cast<int*>(d + o_bad);
      glb::launch_difficulty(ctx, a);
      CK(cudaGetLastError());
      ranges.resize(static_cast<size_t>(n) * beams);
      std::vector<double> bls(n);
      std::vector<int> bix(n), cnt(n), nearc(n);
      int bad = 0;
      CK(cudaMemcpyAsync(ranges.data(), a.ranges, sizeof(double) * ranges.size(), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(bls.data(), a.best_ls, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(bix.data(), a.best_idx, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(cnt.data(), a.counted, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(nearc.data(), a.near, sizeof(int) * n, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaMemcpyAsync(&bad, a.bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (bad == 1) fail(GL_E_MAP_PARSE, "raycast origin not in a free cell");
      if (bad == 2) fail(GL_E_RUNTIME, "map_difficulty: a candidate cell centre is not world-free");
      // first maximum of exp(log_sum / counted) (observation.cpp:110), in
      // candidate order with a strict > (evaluation.cpp:51-57)
      std::vector<double> score_h;
      for (int q = 0; q < n; ++q) {
        if (cnt[q] == 0) {  // every likelihood is 1.0: the first candidate wins
          winner[q] = 0;
          continue;
        }
        int best = bix[q];
        if (nearc[q] > 0) {
          // glibc exp may merge log sums just below the maximum: redo this
          // query's earlier candidates on the host (same FP64 sequence)
          if (score_h.empty()) {
            score_h.resize(static_cast<size_t>(W) * H);
            CK(cudaMemcpy(score_h.data(), tb.d_score, sizeof(double) * score_h.size(), cudaMemcpyDeviceToHost));
          }
          std::vector<double> reach;
          std::vector<int> bidx;
          for (int b = 0; b < beams; b += a.stride) {
            const double r = ranges[static_cast<size_t>(q) * beams + b];
            if (r >= cfg->max_range - 1e-9) continue;
            bidx.push_back(b);
            reach.push_back(r + a.half_cell);
          }
          const double lbest = std::exp(bls[q] / cnt[q]);
          for (int idx = 0; idx < bix[q]; ++idx) {
            const int c = idx / bins, t = idx - c * bins;
            const double x = cx_of(cells[2 * c]), y = cy_of(cells[2 * c + 1]);
            double ls = 0.0;
            for (size_t s = 0; s < bidx.size(); ++s) {
              const double* cs = &dir[2 * (static_cast<size_t>(t) * beams + bidx[s])];
              const double ex = x + reach[s] * cs[0];
              const double ey = y + reach[s] * cs[1];
              const int ci = static_cast<int>(std::floor((ex - ox) / res));
              const int cj = static_cast<int>(std::floor((ey - oy) / res));
              const bool in = ci >= 0 && ci < W && cj >= 0 && cj < H;
              ls += in ? score_h[static_cast<size_t>(cj) * W + ci] : tb.oob;
            }
            if (std::exp(ls / cnt[q]) == lbest) {
              best = idx;
              break;
            }
          }
        }
        winner[q] = best / bins;
      }
    }
    size_t n_wrong = 0;
    for (int q = 0; q < n; ++q) {
      const int c = winner[q];
      const double e = std::hypot(cx_of(cells[2 * c]) - cx_of(cells[2 * q]), cy_of(cells[2 * c + 1]) - cy_of(cells[2 * q + 1]));
      n_wrong += e > cfg->error_threshold ? 1 : 0;
    }
    *out = static_cast<double>(n_wrong) / static_cast<double>(n);
  });
}

}  // extern "C"
