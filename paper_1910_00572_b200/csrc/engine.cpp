// Single-process multi-device engine (include/gridloc_b200.h gl_engine_*):
// the theta-slab sharded belief of SURVEY.md §8(e) driven from ONE host
// process over a device list, for the reference's C++ callers
// (localizer.cpp:7-66 owns one tensor; gridloc_b200::ShardedLocalizer in
// gridloc_b200.hpp owns one of these instead). Built entirely from the
// shard entry points of the C-ABI (capi.cpp) plus two peer-memory kernels
// (k_engine.cu); NCCL is loaded at run time (dlopen) only when asked for.
//
// Per step (n shards):
//   1. every shard: the fused step kernel on its slab; its halo input planes
//      are read straight from the neighbours' buffers (gl_shard_set_peers
//      with UVA pointers: TMA over NVLink P2P, or local when a device hosts
//      several shards); local max into its StepState;
//   2. the 8-byte MAX all-reduce (belief_tensor.cpp:480-481):
//        NCCL: ncclAllReduce(uint64, ncclMax) in place, grouped;
//        P2P:  publish the local max into a per-step-parity mailbox, record
//              an event, every stream waits on every other shard's event,
//              a one-thread kernel gathers the mailboxes over peer memory;
//   3. every shard: gl_shard_finalize (status, pending 1/max rescale).
// Ordering of the peer halo reads: shard s's step n+1 reads its neighbours'
// step-n outputs; those kernels precede the all-reduce of step n, which
// precedes s's finalize and hence its step n+1 (stream order). A neighbour
// overwrites that buffer at step n+2, after the all-reduce of step n+1,
// which s joins only after its step n+1. The P2P mailboxes alternate by
// step parity: a mailbox is rewritten two steps later, after every shard
// passed the barrier of the step in between.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gl_internal.hpp"
#include "gridloc_b200.h"

namespace {

struct EFail {
  gl_status code;
  std::string msg;
};

[[noreturn]] void efail(gl_status code, const std::string& msg) { throw EFail{code, msg}; }

void eneed(bool ok, const char* msg) {
  if (!ok) efail(GL_E_INVALID, msg);
}

// a C-ABI call inside the engine: propagate its status and message
void ecall(gl_status s) {
  if (s != GL_OK) efail(s, gl_last_error());
}

void ecuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) efail(GL_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define ECK(call) ecuda((call), #call)

template <class F>
gl_status eguard(F&& f) {
  try {
    f();
    return GL_OK;
  } catch (const EFail& e) {
    glb::set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    glb::set_last_error(e.what());
    return GL_E_RUNTIME;
  }
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) ECK(cudaSetDevice(d));
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// --------------------------------------------------------------- NCCL
// The subset of nccl.h the engine uses, resolved with dlsym so the product
// library links no NCCL and a process that also loads torch's NCCL shares
// whichever libnccl.so.2 is already mapped.
typedef struct ncclComm* ncclComm_t;
enum { kNcclUint64 = 5, kNcclFloat64 = 8, kNcclMax = 2 };  // ncclUint64 / ncclFloat64 / ncclMax (nccl.h)
struct Nccl {
  void* lib = nullptr;
  int (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool load() {
    if (lib) return true;
    lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!lib) return false;
    auto sym = [&](const char* n) { return dlsym(lib, n); };
    CommInitAll = reinterpret_cast<decltype(CommInitAll)>(sym("ncclCommInitAll"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
    return CommInitAll && CommDestroy && AllReduce && GroupStart && GroupEnd && GetErrorString;
  }
  void check(int r, const char* what) const {
    if (r != 0) efail(GL_E_CUDA, std::string(what) + ": " + (GetErrorString ? GetErrorString(r) : "nccl error"));
  }
};

Nccl& nccl() {
  static Nccl n;
  return n;
}

}  // namespace

struct gl_engine {
  int n = 0, W = 0, H = 0, C = 0, halo = -1, mode = GL_ENGINE_P2P;
  std::vector<int> dev;
  std::vector<gl_context*> ctx;
  std::vector<gl_map*> map;
  std::vector<gl_field*> field;            // lazily, for observe
  std::vector<gl_kernels*> kern[2];        // per slot, per shard
  std::vector<gl_activation*> act[2];
  std::vector<gl_tensor*> t;
  std::vector<int> c0, c1;                 // channel ranges
  std::vector<unsigned long long*> mailbox;  // P2P: 2 words per shard (step parity)
  std::vector<cudaEvent_t> ev;
  std::vector<double*> d_plane;            // observation belief maps
  std::vector<ncclComm_t> comms;
  int parity = 0;
  bool stepped = false;
};

namespace {

void engine_release(gl_engine* e) {
  for (int s = 0; s < e->n; ++s) {
    if (s < static_cast<int>(e->ctx.size()) && e->ctx[s]) gl_context_synchronize(e->ctx[s]);
  }
  for (ncclComm_t c : e->comms)
    if (c) nccl().CommDestroy(c);
  for (int s = 0; s < static_cast<int>(e->ctx.size()); ++s) {
    DevGuard g(e->dev[s]);
    if (s < static_cast<int>(e->t.size()) && e->t[s]) gl_tensor_destroy(e->t[s]);
    for (int k = 0; k < 2; ++k) {
      if (s < static_cast<int>(e->act[k].size()) && e->act[k][s]) gl_activation_destroy(e->act[k][s]);
      if (s < static_cast<int>(e->kern[k].size()) && e->kern[k][s]) gl_kernels_destroy(e->kern[k][s]);
    }
    if (s < static_cast<int>(e->field.size()) && e->field[s]) gl_field_destroy(e->field[s]);
    if (s < static_cast<int>(e->map.size()) && e->map[s]) gl_map_destroy(e->map[s]);
    if (s < static_cast<int>(e->mailbox.size()) && e->mailbox[s]) cudaFree(e->mailbox[s]);
    if (s < static_cast<int>(e->d_plane.size()) && e->d_plane[s]) cudaFree(e->d_plane[s]);
    if (s < static_cast<int>(e->ev.size()) && e->ev[s]) cudaEventDestroy(e->ev[s]);
    gl_context_destroy(e->ctx[s]);
  }
  delete e;
}

cudaStream_t stream_of(gl_context* c) {
  void* s = nullptr;
  ecall(gl_context_stream(c, &s));
  return static_cast<cudaStream_t>(s);
}

unsigned long long* max_ptr(gl_engine* e, int s) {
  unsigned long long* p = nullptr;
  ecall(gl_tensor_max_ptr(e->ctx[s], e->t[s], &p));
  return p;
}

// every shard's stream waits for every other shard's latest event
void barrier_all(gl_engine* e) {
  for (int s = 0; s < e->n; ++s) {
    DevGuard g(e->dev[s]);
    ECK(cudaEventRecord(e->ev[s], stream_of(e->ctx[s])));
  }
  for (int s = 0; s < e->n; ++s) {
    DevGuard g(e->dev[s]);
    for (int r = 0; r < e->n; ++r)
      if (r != s) ECK(cudaStreamWaitEvent(stream_of(e->ctx[s]), e->ev[r], 0));
  }
}

// the 8-byte MAX all-reduce of the shards' step maxima
void allreduce_max(gl_engine* e) {
  if (e->n == 1) return;
  if (e->mode == GL_ENGINE_NCCL) {
    Nccl& N = nccl();
    N.check(N.GroupStart(), "ncclGroupStart");
    for (int s = 0; s < e->n; ++s) {
      unsigned long long* p = max_ptr(e, s);
      N.check(N.AllReduce(p, p, 1, kNcclUint64, kNcclMax, e->comms[s], stream_of(e->ctx[s])), "ncclAllReduce");
    }
    N.check(N.GroupEnd(), "ncclGroupEnd");
    return;
  }
  const int slot = e->parity;
  for (int s = 0; s < e->n; ++s) {
    DevGuard g(e->dev[s]);
    glb::launch_engine_publish(e->ctx[s], max_ptr(e, s), e->mailbox[s] + slot);
  }
  barrier_all(e);
  glb::PtrList boxes{};
  boxes.n = e->n;
  for (int s = 0; s < e->n; ++s) boxes.p[s] = e->mailbox[s] + slot;
  for (int s = 0; s < e->n; ++s) {
    DevGuard g(e->dev[s]);
    glb::launch_engine_gather(e->ctx[s], boxes, max_ptr(e, s));
  }
  e->parity ^= 1;
}

void set_peers(gl_engine* e) {
  for (int s = 0; s < e->n; ++s) {
    const int lo = (s - 1 + e->n) % e->n, hi = (s + 1) % e->n;
    double* b[2][2];
    for (int q = 0; q < 2; ++q) {
      const int nb = q == 0 ? lo : hi;
      for (int buf = 0; buf < 2; ++buf) ecall(gl_tensor_buffer_ptr(e->ctx[nb], e->t[nb], buf, 0, &b[q][buf]));
    }
    ecall(gl_shard_set_peers(e->ctx[s], e->t[s], b[0][0], b[0][1], e->c1[lo] - e->c0[lo], b[1][0], b[1][1],
                             e->c1[hi] - e->c0[hi]));
  }
}

void sync_all(gl_engine* e) {
  for (int s = 0; s < e->n; ++s) ecall(gl_context_synchronize(e->ctx[s]));
}

void step_enqueue(gl_engine* e, double u, double v, double w, int slot) {
  eneed(slot == 0 || slot == 1, "kernel slot must be 0 (main) or 1 (rotation-only)");
  eneed(!e->t.empty() && e->t[0] != nullptr, "engine tensor not initialised (gl_engine_init_uniform)");
  eneed(e->kern[slot][0] != nullptr, "kernel slot not set (gl_engine_set_kernels)");
  for (int s = 0; s < e->n; ++s)
    ecall(gl_step_async(e->ctx[s], e->t[s], u, v, w, e->map[s], e->kern[slot][s], e->act[slot][s]));
  allreduce_max(e);
  for (int s = 0; s < e->n; ++s) ecall(gl_shard_finalize(e->ctx[s], e->t[s]));
  e->stepped = true;
}

}  // namespace

extern "C" {

gl_status gl_engine_create(const int* devices, int n_devices, int width, int height, double resolution,
                           double origin_x, double origin_y, const uint8_t* occ, int channels, int mode,
                           gl_engine** out) {
  gl_engine* e = nullptr;
  const gl_status st = eguard([&] {
    eneed(devices && occ && out, "null argument");
    eneed(n_devices >= 1 && n_devices <= glb::kEngineMaxShards, "1..16 devices");
    eneed(channels >= 4 && channels % 2 == 0, "channel count must be even and >= 4");
    eneed(channels >= n_devices, "more shards than channels");
    eneed(mode >= GL_ENGINE_AUTO && mode <= GL_ENGINE_P2P, "mode must be AUTO, NCCL or P2P");
    e = new gl_engine();
    e->n = n_devices;
    e->W = width;
    e->H = height;
    e->C = channels;
    e->dev.assign(devices, devices + n_devices);
    bool distinct = true;
    for (int a = 0; a < n_devices; ++a)
      for (int b = a + 1; b < n_devices; ++b) distinct = distinct && e->dev[a] != e->dev[b];
    if (mode == GL_ENGINE_NCCL) eneed(distinct, "NCCL mode needs distinct devices (one rank per GPU)");
    e->mode = GL_ENGINE_P2P;
    if (n_devices > 1 && (mode == GL_ENGINE_NCCL || (mode == GL_ENGINE_AUTO && distinct))) {
      if (nccl().load()) {
        e->mode = GL_ENGINE_NCCL;
      } else if (mode == GL_ENGINE_NCCL) {
        efail(GL_E_RUNTIME, "libnccl.so.2 could not be loaded");
      }
    }
    if (n_devices == 1 && mode == GL_ENGINE_NCCL) e->mode = GL_ENGINE_NCCL;  // nothing to reduce
    // peer access between every pair of distinct devices (halo reads and the P2P gather)
    for (int a = 0; a < n_devices; ++a) {
      for (int b = 0; b < n_devices; ++b) {
        if (e->dev[a] == e->dev[b]) continue;
        int ok = 0;
        ECK(cudaDeviceCanAccessPeer(&ok, e->dev[a], e->dev[b]));
        eneed(ok != 0, "devices without peer access (the halo planes are read over NVLink P2P)");
        DevGuard g(e->dev[a]);
        const cudaError_t r = cudaDeviceEnablePeerAccess(e->dev[b], 0);
        if (r == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else {
          ECK(r);
        }
      }
    }
    for (int s = 0; s < n_devices; ++s) {
      gl_context* c = nullptr;
      ecall(gl_context_create(e->dev[s], &c));
      e->ctx.push_back(c);
      gl_map* m = nullptr;
      ecall(gl_map_create(c, width, height, resolution, origin_x, origin_y, occ, &m));
      e->map.push_back(m);
      e->c0.push_back(static_cast<int>(static_cast<long long>(s) * channels / n_devices));
      e->c1.push_back(static_cast<int>(static_cast<long long>(s + 1) * channels / n_devices));
      DevGuard g(e->dev[s]);
      unsigned long long* mb = nullptr;
      ECK(cudaMalloc(&mb, 2 * sizeof(unsigned long long)));
      ECK(cudaMemset(mb, 0, 2 * sizeof(unsigned long long)));
      e->mailbox.push_back(mb);
      cudaEvent_t ev = nullptr;
      ECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      e->ev.push_back(ev);
    }
    e->field.assign(n_devices, nullptr);
    e->d_plane.assign(n_devices, nullptr);
    for (int k = 0; k < 2; ++k) {
      e->kern[k].assign(n_devices, nullptr);
      e->act[k].assign(n_devices, nullptr);
    }
    e->t.assign(n_devices, nullptr);
    if (e->mode == GL_ENGINE_NCCL && n_devices > 1) {
      e->comms.assign(n_devices, nullptr);
      nccl().check(nccl().CommInitAll(e->comms.data(), n_devices, e->dev.data()), "ncclCommInitAll");
    }
  });
  if (st != GL_OK) {
    if (e) engine_release(e);
    return st;
  }
  *out = e;
  return GL_OK;
}

gl_status gl_engine_destroy(gl_engine* e) {
  return eguard([&] {
    if (e) engine_release(e);
  });
}

gl_status gl_engine_info(const gl_engine* e, int* n_shards, int* mode, int* halo) {
  return eguard([&] {
    eneed(e, "null engine");
    if (n_shards) *n_shards = e->n;
    if (mode) *mode = e->mode;
    if (halo) *halo = e->halo;
  });
}

gl_status gl_engine_context(gl_engine* e, int s, gl_context** ctx) {
  return eguard([&] {
    eneed(e && ctx && s >= 0 && s < e->n, "bad argument");
    *ctx = e->ctx[s];
  });
}

gl_status gl_engine_set_kernels(gl_engine* e, int slot, const gl_kernels* kernels) {
  return eguard([&] {
    eneed(e && kernels, "null argument");
    eneed(slot == 0 || slot == 1, "kernel slot must be 0 (main) or 1 (rotation-only)");
    gl_kernel_info info{};
    ecall(gl_kernels_info(kernels, &info));
    const int kw = 2 * info.radius + 1;
    std::vector<double> sep(info.separable ? kw : 1), spatial(static_cast<size_t>(info.channels) * kw * kw + 1),
        aw(info.n_angular);
    std::vector<int> ao(info.n_angular);
    ecall(gl_kernels_get(kernels, sep.data(), spatial.data(), ao.data(), aw.data()));
    int hmax = 0;
    for (int q = 0; q < info.n_angular; ++q) hmax = std::max(hmax, std::abs(ao[q]));
    if (e->halo < 0) e->halo = std::max(1, hmax);
    eneed(hmax <= e->halo, "angular half-width exceeds the engine's halo (set the widest slot first)");
    for (int s = 0; s < e->n; ++s) eneed(e->c1[s] - e->c0[s] >= e->halo, "halo wider than a shard");
    for (int s = 0; s < e->n; ++s) {
      if (e->act[slot][s]) gl_activation_destroy(e->act[slot][s]);
      if (e->kern[slot][s]) gl_kernels_destroy(e->kern[slot][s]);
      e->act[slot][s] = nullptr;
      e->kern[slot][s] = nullptr;
      gl_kernels* k = nullptr;
      ecall(gl_kernels_create(e->ctx[s], &info, sep.data(), spatial.data(), ao.data(), aw.data(), &k));
      e->kern[slot][s] = k;
      gl_activation* a = nullptr;
      ecall(gl_make_activation(e->ctx[s], e->map[s], k, e->C, &a));
      e->act[slot][s] = a;
    }
  });
}

gl_status gl_engine_init_uniform(gl_engine* e) {
  return eguard([&] {
    eneed(e, "null engine");
    eneed(e->halo >= 0, "set a kernel slot first (it fixes the halo)");
    sync_all(e);
    for (int s = 0; s < e->n; ++s) {
      if (e->t[s]) gl_tensor_destroy(e->t[s]);
      e->t[s] = nullptr;
    }
    for (int s = 0; s < e->n; ++s) {
      gl_tensor* t = nullptr;
      ecall(gl_shard_init_uniform(e->ctx[s], e->map[s], e->C, e->c0[s], e->c1[s], e->halo, &t));
      e->t[s] = t;
    }
    set_peers(e);
    e->parity = 0;
  });
}

gl_status gl_engine_step_async(gl_engine* e, double u, double v, double w, int slot) {
  return eguard([&] {
    eneed(e, "null engine");
    step_enqueue(e, u, v, w, slot);
  });
}

gl_status gl_engine_status(gl_engine* e) {
  gl_status first = GL_OK;
  const gl_status st = eguard([&] {
    eneed(e, "null engine");
    sync_all(e);
    for (int s = 0; s < e->n; ++s) {
      const gl_status r = gl_tensor_status(e->ctx[s], e->t[s]);
      if (r != GL_OK && first == GL_OK) first = r;
    }
    if (first != GL_OK) efail(first, gl_last_error());
  });
  return st;
}

gl_status gl_engine_step(gl_engine* e, double u, double v, double w, int slot) {
  const gl_status st = gl_engine_step_async(e, u, v, w, slot);
  if (st != GL_OK) return st;
  return gl_engine_status(e);
}

gl_status gl_engine_argmax(gl_engine* e, gl_pose_estimate* out) {
  return eguard([&] {
    eneed(e && out, "null argument");
    const size_t plane = static_cast<size_t>(e->W) * e->H;
    double best = -1.0, total = 0.0;
    long long best_idx = 0;
    for (int s = 0; s < e->n; ++s) {
      double v = 0.0;
      int64_t flat = 0;
      // the reference's sequential total runs through the shards in channel
      // order: each continues the previous one's running sum (bit-exact)
      ecall(gl_tensor_argmax_candidate(e->ctx[s], e->t[s], total, &v, &flat, &total));
      // shards are in channel order: a later shard's equal value has a
      // higher global flat index, so only a strictly larger one wins
      const long long g = static_cast<long long>(e->c0[s]) * static_cast<long long>(plane) + flat;
      if (v > 0.0 && v > best) {
        best = v;
        best_idx = g;
      }
    }
    if (!(best > 0.0)) efail(GL_E_EXTINGUISHED, "argmax on an all-zero belief tensor");
    double theta_t = 0.0, cell = 0.1, ox = 0.0, oy = 0.0;
    int w_ = 0, h_ = 0, c_ = 0;
    ecall(gl_tensor_theta(e->t[0], &theta_t));
    ecall(gl_tensor_info(e->t[0], &w_, &h_, &c_, &cell, &ox, &oy));
    const size_t p = static_cast<size_t>(best_idx) % plane;
    out->k = static_cast<int>(static_cast<size_t>(best_idx) / plane);
    out->i = static_cast<int>(p % e->W);
    out->j = static_cast<int>(p / e->W);
    out->x = ox + (out->i + 0.5) * cell;
    out->y = oy + (out->j + 0.5) * cell;
    double a = std::fmod(out->k * (2.0 * M_PI / e->C) + theta_t, 2.0 * M_PI);  // geometry.hpp:8-13
    if (a < -M_PI) a += 2.0 * M_PI;
    if (a >= M_PI) a -= 2.0 * M_PI;
    out->theta = a;
    out->confidence = total > 0.0 ? best / total : 0.0;
  });
}

namespace {

// per-shard belief maps MAX-combined into shard 0's device plane
double* combined_belief_map(gl_engine* e) {
  const size_t plane = static_cast<size_t>(e->W) * e->H;
  for (int s = 0; s < e->n; ++s) {
    if (!e->d_plane[s]) {
      DevGuard g(e->dev[s]);
      ECK(cudaMalloc(&e->d_plane[s], plane * sizeof(double)));
    }
    ecall(gl_shard_belief_map(e->ctx[s], e->t[s], e->d_plane[s]));
  }
  if (e->n == 1) return e->d_plane[0];
  if (e->mode == GL_ENGINE_NCCL) {
    Nccl& N = nccl();
    N.check(N.GroupStart(), "ncclGroupStart");
    for (int s = 0; s < e->n; ++s)
      N.check(N.AllReduce(e->d_plane[s], e->d_plane[s], plane, kNcclFloat64, kNcclMax, e->comms[s],
                          stream_of(e->ctx[s])),
              "ncclAllReduce");
    N.check(N.GroupEnd(), "ncclGroupEnd");
    return e->d_plane[0];
  }
  barrier_all(e);
  glb::PtrList srcs{};
  srcs.n = e->n - 1;
  for (int s = 1; s < e->n; ++s) srcs.p[s - 1] = e->d_plane[s];
  {
    DevGuard g(e->dev[0]);
    glb::launch_plane_max_combine(e->ctx[0], e->d_plane[0], srcs, plane);
  }
  barrier_all(e);  // shard planes stay untouched until shard 0 has read them
  return e->d_plane[0];
}

}  // namespace

gl_status gl_engine_belief_map(gl_engine* e, double* host_out) {
  return eguard([&] {
    eneed(e && host_out, "null argument");
    double* d = combined_belief_map(e);
    DevGuard g(e->dev[0]);
    ECK(cudaMemcpyAsync(host_out, d, static_cast<size_t>(e->W) * e->H * sizeof(double), cudaMemcpyDeviceToHost,
                        stream_of(e->ctx[0])));
    ECK(cudaStreamSynchronize(stream_of(e->ctx[0])));
  });
}

gl_status gl_engine_observe(gl_engine* e, int budget, const double* angles, const double* ranges, int n_beams,
                            double max_range, gl_likelihood params, int32_t* cells, int cap, int* n,
                            double* source_mass) {
  return eguard([&] {
    eneed(e && n && source_mass, "null argument");
    eneed(cap >= 0 && (cap == 0 || cells), "bad sample buffer");
    double* d = combined_belief_map(e);
    // the whole sample set (the update needs every sample even if the
    // caller's buffer is shorter)
    const int full_cap = static_cast<int>(std::min<size_t>(static_cast<size_t>(e->W) * e->H,
                                                           4 * static_cast<size_t>(std::max(budget, 1)) + 64));
    std::vector<int32_t> all(2 * static_cast<size_t>(std::max(full_cap, 1)));
    int got = 0;
    double mass = 0.0;
    ecall(gl_dither_device(e->ctx[0], d, e->W, e->H, budget, all.data(), full_cap, &got, &mass));
    eneed(got <= full_cap, "sample capacity exceeded");
    *n = got;
    *source_mass = mass;
    for (int q = 0; q < std::min(got, cap); ++q) {
      cells[2 * q] = all[2 * q];
      cells[2 * q + 1] = all[2 * q + 1];
    }
    if (got == 0) return;  // observation.cpp:117: an empty sample set is a no-op
    for (int s = 0; s < e->n; ++s) {
      if (!e->field[s]) ecall(gl_field_create(e->ctx[s], e->map[s], &e->field[s]));
      ecall(gl_shard_observe(e->ctx[s], e->t[s], all.data(), got, angles, ranges, n_beams, max_range, e->map[s],
                             e->field[s], params));
    }
    allreduce_max(e);
    gl_status first = GL_OK;
    std::string msg;
    for (int s = 0; s < e->n; ++s) {
      const gl_status r = gl_shard_observe_finalize(e->ctx[s], e->t[s]);
      if (r != GL_OK && first == GL_OK) {
        first = r;
        msg = gl_last_error();
      }
    }
    if (first != GL_OK) efail(first, msg);
  });
}

gl_status gl_engine_download(gl_engine* e, double* host, double* theta_t) {
  return eguard([&] {
    eneed(e && host, "null argument");
    const size_t plane = static_cast<size_t>(e->W) * e->H;
    for (int s = 0; s < e->n; ++s) ecall(gl_tensor_download(e->ctx[s], e->t[s], host + plane * e->c0[s]));
    if (theta_t) ecall(gl_tensor_theta(e->t[0], theta_t));
  });
}

gl_status gl_engine_upload(gl_engine* e, const double* host, double theta_t) {
  return eguard([&] {
    eneed(e && host, "null argument");
    const size_t plane = static_cast<size_t>(e->W) * e->H;
    sync_all(e);
    bool clean = true;
    for (int s = 0; s < e->n; ++s) {
      ecall(gl_tensor_upload(e->ctx[s], e->t[s], host + plane * e->c0[s]));
      ecall(gl_tensor_set_theta(e->t[s], theta_t));
      clean = clean && e->t[s]->clean[e->t[s]->cur];
    }
    // a shard's step reads its neighbours' planes: the FAST variant is only
    // exact when every shard's buffer is clean
    for (int s = 0; s < e->n; ++s) e->t[s]->clean[e->t[s]->cur] = clean;
    sync_all(e);  // every shard's planes are in place before any neighbour reads them
  });
}

gl_status gl_engine_hash(gl_engine* e, uint64_t* hash) {
  return eguard([&] {
    eneed(e && hash, "null argument");
    sync_all(e);
    const uint64_t plane = static_cast<uint64_t>(e->W) * e->H;
    uint64_t h = 0;
    for (int s = 0; s < e->n; ++s) {
      uint64_t x = 0;
      ecall(gl_tensor_hash_at(e->ctx[s], e->t[s], plane * e->c0[s], &x));
      h += x;
    }
    *hash = h;
  });
}

}  // extern "C"
