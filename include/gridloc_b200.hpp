// gridloc_b200.hpp — header-only C++ mirror of the reference gridloc hot-path
// API (/root/reference/proj/include/gridloc/{belief_tensor,observation,
// localizer,occupancy_map,geometry,grid2d}.hpp) over the C-ABI in
// gridloc_b200.h. Same names, argument meaning and exceptions; the belief
// tensor lives on the GPU. Switching a caller is a namespace change:
//
//     namespace gl = gridloc_b200;   // was: namespace gl = gridloc;
//
// See INTEGRATION.md. Differences a caller can observe:
//   * ThreadPool selects a CUDA device instead of host threads.
//   * BeliefTensor::values() returns a host copy (the tensor is in HBM);
//     write back with set_values(). at(i,j,k) reads/writes one element.
//   * StepScratch::t_motion receives the whole step's device time (the fused
//     kernel has no phase boundaries); t_diffusion = t_masking = 0.
//   (argmax_state().confidence is bit-exact: the reference's sequential
//   total is reproduced by a parallel binade scan.)
#pragma once

#include <cmath>
#include <cstdint>
#include <fstream>
#include <iterator>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gridloc_b200.h"

namespace gridloc_b200 {

// ------------------------------------------------------------ exceptions
class BeliefExtinguishedError : public std::runtime_error {  // belief_tensor.hpp:22-25
 public:
  using std::runtime_error::runtime_error;
};

enum class MapError { kMalformedHeader, kZeroDimensions, kUnsupportedBitDepth, kUnsupportedFormat,
                      kTruncatedData, kNoFreeSpace, kInvalidOrigin };

class MapParseError : public std::runtime_error {  // occupancy_map.hpp:22-30
 public:
  MapParseError(MapError code, const std::string& what) : std::runtime_error(what), code_(code) {}
  MapError code() const { return code_; }

 private:
  MapError code_;
};

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(gl_status s) {
  if (s == GL_OK) return;
  const std::string msg = gl_last_error();
  switch (s) {
    case GL_E_EXTINGUISHED: throw BeliefExtinguishedError(msg);
    case GL_E_INVALID: throw std::invalid_argument(msg);
    case GL_E_MAP_PARSE: throw MapParseError(MapError::kMalformedHeader, msg);
    case GL_E_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// -------------------------------------------------------------- geometry
inline double wrap_angle(double a) {  // geometry.hpp:8-13
  a = std::fmod(a, 2.0 * M_PI);
  if (a < -M_PI) a += 2.0 * M_PI;
  if (a >= M_PI) a -= 2.0 * M_PI;
  return a;
}
struct Pose2 {
  double x = 0.0, y = 0.0, theta = 0.0;
};
struct OdometryDelta {
  double u = 0.0, v = 0.0, w = 0.0;
};
inline Pose2 compose(const Pose2& a, const Pose2& b) {
  const double c = std::cos(a.theta), s = std::sin(a.theta);
  return Pose2{a.x + c * b.x - s * b.y, a.y + s * b.x + c * b.y, wrap_angle(a.theta + b.theta)};
}
inline Pose2 compose(const Pose2& a, const OdometryDelta& d) { return compose(a, Pose2{d.u, d.v, d.w}); }
inline OdometryDelta relative_delta(const Pose2& a, const Pose2& b) {  // geometry.hpp:44-51
  const double c = std::cos(a.theta), s = std::sin(a.theta);
  const double dx = b.x - a.x, dy = b.y - a.y;
  return OdometryDelta{c * dx + s * dy, -s * dx + c * dy, wrap_angle(b.theta - a.theta)};
}
inline OdometryDelta compose_delta(const OdometryDelta& a, const OdometryDelta& b) {
  const double c = std::cos(a.w), s = std::sin(a.w);
  return OdometryDelta{a.u + c * b.u - s * b.v, a.v + s * b.u + c * b.v, a.w + b.w};
}

struct Grid2d {  // grid2d.hpp:9-21
  int width = 0, height = 0;
  std::vector<double> data;
  Grid2d() = default;
  Grid2d(int w, int h, double fill = 0.0) : width(w), height(h), data(static_cast<size_t>(w) * h, fill) {}
  double& at(int i, int j) { return data[static_cast<size_t>(j) * width + i]; }
  double at(int i, int j) const { return data[static_cast<size_t>(j) * width + i]; }
  size_t size() const { return data.size(); }
};

struct MotionNoise {  // belief_tensor.hpp:16-20
  double sigma_x = 0.03, sigma_y = 0.03, sigma_theta = 0.012;
};
struct LikelihoodParams {  // observation.hpp:21-25
  double sigma_hit = 0.2, weight_floor = 0.05;
  int beam_stride = 4;
};
struct LidarScan {
  std::vector<double> angles, ranges;
  double max_range = 0.0;
};
struct SampleSet {
  std::vector<std::pair<int, int>> cells;
  double source_mass = 0.0;
};
struct PoseEstimate {
  Pose2 pose;
  double confidence = 0.0;
  int i = 0, j = 0, k = 0;
};
struct StepScratch {
  double t_motion = 0.0, t_diffusion = 0.0, t_masking = 0.0;
};

// ------------------------------------------------------- device context
// Replaces gridloc::ThreadPool: the parallel substrate is a CUDA device.
class ThreadPool {
 public:
  explicit ThreadPool(int /*threads*/ = 0, int device = 0) {
    gl_context* c = nullptr;
    check(gl_context_create(device, &c));
    ctx_.reset(c, [](gl_context* p) { gl_context_destroy(p); });
    check(gl_context_set_step_timing(c, 1));  // StepScratch::t_motion, as the reference fills it
  }
  int thread_count() const { return 1; }
  gl_context* get() const { return ctx_.get(); }
  // the wall-crossing mask extension for every step on this device context
  // (off by default: the reference masks destination cells only)
  void set_wall_mask(bool enable) { check(gl_context_set_wall_mask(ctx_.get(), enable ? 1 : 0)); }
  static ThreadPool& default_pool() {
    static ThreadPool pool(0, 0);
    return pool;
  }

 private:
  std::shared_ptr<gl_context> ctx_;
};

// ------------------------------------------------------------------ maps
class OccupancyMap {  // occupancy_map.hpp:35-81
 public:
  OccupancyMap(int width, int height, double resolution, std::vector<uint8_t> occupied,
               double origin_x = 0.0, double origin_y = 0.0, ThreadPool& pool = ThreadPool::default_pool())
      : pool_(&pool) {
    gl_map* m = nullptr;
    check(gl_map_create(pool.get(), width, height, resolution, origin_x, origin_y, occupied.data(), &m));
    map_.reset(m, [](gl_map* p) { gl_map_destroy(p); });
    check(gl_map_info(m, &w_, &h_, &res_, &ox_, &oy_, &free_));
    cells_.resize(static_cast<size_t>(w_) * h_);
    check(gl_map_cells(m, cells_.data()));
  }
  int width() const { return w_; }
  int height() const { return h_; }
  double resolution() const { return res_; }
  double origin_x() const { return ox_; }
  double origin_y() const { return oy_; }
  bool in_bounds(int i, int j) const { return i >= 0 && i < w_ && j >= 0 && j < h_; }
  bool occupied(int i, int j) const { return cells_[static_cast<size_t>(j) * w_ + i] != 0; }
  bool free(int i, int j) const { return !occupied(i, j); }
  const std::vector<uint8_t>& cells() const { return cells_; }
  int free_count() const { return free_; }
  int cell_x(double wx) const { return static_cast<int>(std::floor((wx - ox_) / res_)); }
  int cell_y(double wy) const { return static_cast<int>(std::floor((wy - oy_) / res_)); }
  double center_x(int i) const { return ox_ + (i + 0.5) * res_; }
  double center_y(int j) const { return oy_ + (j + 0.5) * res_; }
  bool world_free(double wx, double wy) const {
    const int i = cell_x(wx), j = cell_y(wy);
    return in_bounds(i, j) && free(i, j);
  }
  gl_map* handle() const { return map_.get(); }
  ThreadPool& pool() const { return *pool_; }

 private:
  std::shared_ptr<gl_map> map_;
  ThreadPool* pool_;
  int w_ = 0, h_ = 0, free_ = 0;
  double res_ = 0.1, ox_ = 0.0, oy_ = 0.0;
  std::vector<uint8_t> cells_;
};

inline OccupancyMap load_map(const std::vector<uint8_t>& bytes, int threshold, double resolution,
                             double origin_x = 0.0, double origin_y = 0.0) {  // occupancy_map.hpp:106-108
  int w = 0, h = 0;
  check(gl_load_map(bytes.data(), bytes.size(), threshold, &w, &h, nullptr));
  std::vector<uint8_t> occ(static_cast<size_t>(w) * h);
  check(gl_load_map(bytes.data(), bytes.size(), threshold, &w, &h, occ.data()));
  return OccupancyMap(w, h, resolution, std::move(occ), origin_x, origin_y);
}

inline OccupancyMap load_map_file(const std::string& path, int threshold, double resolution,
                                  double origin_x = 0.0, double origin_y = 0.0) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open map file: " + path);
  std::vector<uint8_t> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return load_map(bytes, threshold, resolution, origin_x, origin_y);
}

class DistanceField {  // occupancy_map.hpp:85-101
 public:
  explicit DistanceField(const OccupancyMap& map) : w_(map.width()), h_(map.height()) {
    gl_field* f = nullptr;
    check(gl_field_create(map.pool().get(), map.handle(), &f));
    field_.reset(f, [](gl_field* p) { gl_field_destroy(p); });
    values_.resize(static_cast<size_t>(w_) * h_);
    check(gl_field_values(f, values_.data()));
  }
  int width() const { return w_; }
  int height() const { return h_; }
  double at(int i, int j) const { return values_[static_cast<size_t>(j) * w_ + i]; }
  const std::vector<double>& values() const { return values_; }
  gl_field* handle() const { return field_.get(); }

 private:
  std::shared_ptr<gl_field> field_;
  int w_, h_;
  std::vector<double> values_;
};

inline DistanceField distance_field(const OccupancyMap& map) { return DistanceField(map); }

// ------------------------------------------------------ kernels / activation
struct KernelSet {  // belief_tensor.hpp:79-89
  int radius = 0;
  std::vector<std::vector<double>> spatial;
  std::vector<std::pair<int, double>> angular;
  bool degenerate_spatial = false;
  bool degenerate_angular = false;
  bool separable = false;
  std::vector<double> sep;
  std::shared_ptr<gl_kernels> handle;  // device copy

  gl_kernels* get(ThreadPool& pool) const {
    if (!handle) {  // built from fields by the caller: wrap them
      gl_kernel_info info{static_cast<int>(spatial.size()), radius, separable ? 1 : 0,
                          degenerate_spatial ? 1 : 0, degenerate_angular ? 1 : 0,
                          static_cast<int>(angular.size())};
      std::vector<double> flat;
      for (const auto& s : spatial) flat.insert(flat.end(), s.begin(), s.end());
      std::vector<int> off;
      std::vector<double> w;
      for (const auto& a : angular) {
        off.push_back(a.first);
        w.push_back(a.second);
      }
      gl_kernels* k = nullptr;
      check(gl_kernels_create(pool.get(), &info, sep.data(), flat.data(), off.data(), w.data(), &k));
      const_cast<KernelSet*>(this)->handle.reset(k, [](gl_kernels* p) { gl_kernels_destroy(p); });
    }
    return handle.get();
  }
};

inline KernelSet build_kernels(const MotionNoise& noise, int channels, double cell_size,
                               double delta_theta) {  // belief_tensor.cpp:243-338
  gl_kernels* k = nullptr;
  check(gl_build_kernels(noise.sigma_x, noise.sigma_y, noise.sigma_theta, channels, cell_size, delta_theta, &k));
  KernelSet ks;
  ks.handle.reset(k, [](gl_kernels* p) { gl_kernels_destroy(p); });
  gl_kernel_info info;
  check(gl_kernels_info(k, &info));
  const int kw = 2 * info.radius + 1;
  std::vector<double> sep(info.separable ? kw : 0), spatial(static_cast<size_t>(info.channels) * kw * kw),
      aw(info.n_angular);
  std::vector<int> ao(info.n_angular);
  check(gl_kernels_get(k, sep.data(), spatial.data(), ao.data(), aw.data()));
  ks.radius = info.radius;
  ks.separable = info.separable != 0;
  ks.degenerate_spatial = info.degenerate_spatial != 0;
  ks.degenerate_angular = info.degenerate_angular != 0;
  ks.sep = sep;
  for (int c = 0; c < info.channels; ++c)
    ks.spatial.emplace_back(spatial.begin() + static_cast<size_t>(c) * kw * kw,
                            spatial.begin() + static_cast<size_t>(c + 1) * kw * kw);
  for (int t = 0; t < info.n_angular; ++t) ks.angular.emplace_back(ao[t], aw[t]);
  return ks;
}

struct Activation {  // belief_tensor.hpp:93-96 (device-resident)
  std::shared_ptr<gl_activation> handle;
  int channels = 0, width = 0, height = 0;
  ThreadPool* pool = nullptr;
  std::vector<double> inverse() const {
    std::vector<double> out(static_cast<size_t>(channels) * width * height);
    check(gl_activation_get(pool->get(), handle.get(), nullptr, out.data()));
    return out;
  }
};

inline Activation make_activation(const OccupancyMap& map, const KernelSet& kernels, int channels,
                                  ThreadPool& pool) {  // belief_tensor.cpp:354-394
  gl_activation* a = nullptr;
  check(gl_make_activation(pool.get(), map.handle(), kernels.get(pool), channels, &a));
  Activation act;
  act.handle.reset(a, [](gl_activation* p) { gl_activation_destroy(p); });
  act.channels = channels;
  act.width = map.width();
  act.height = map.height();
  act.pool = &pool;
  return act;
}

// ---------------------------------------------------------------- tensor
class BeliefTensor {  // belief_tensor.hpp:30-75, values resident in HBM
 public:
  BeliefTensor(int width, int height, int channels, double cell_size, double origin_x, double origin_y,
               ThreadPool& pool = ThreadPool::default_pool())
      : pool_(&pool) {
    gl_tensor* t = nullptr;
    check(gl_tensor_create(pool.get(), width, height, channels, cell_size, origin_x, origin_y, &t));
    adopt(t);
  }
  BeliefTensor(gl_tensor* t, ThreadPool& pool) : pool_(&pool) { adopt(t); }
  BeliefTensor(const BeliefTensor& o) : pool_(o.pool_) {  // value semantics, device copy
    gl_tensor* t = nullptr;
    check(gl_tensor_clone(pool_->get(), o.get(), &t));
    adopt(t);
  }
  BeliefTensor& operator=(const BeliefTensor& o) {
    if (this != &o) {
      BeliefTensor tmp(o);
      std::swap(t_, tmp.t_);
      pool_ = o.pool_;
      w_ = o.w_, h_ = o.h_, c_ = o.c_;
      cell_ = o.cell_, ox_ = o.ox_, oy_ = o.oy_;
    }
    return *this;
  }
  BeliefTensor(BeliefTensor&&) = default;
  BeliefTensor& operator=(BeliefTensor&&) = default;

  int width() const { return w_; }
  int height() const { return h_; }
  int channels() const { return c_; }
  double cell_size() const { return cell_; }
  double delta_theta() const { return 2.0 * M_PI / c_; }
  double theta_t() const {
    double th = 0.0;
    check(gl_tensor_theta(get(), &th));
    return th;
  }
  void set_theta_t(double t) { check(gl_tensor_set_theta(get(), t)); }
  double origin_x() const { return ox_; }
  double origin_y() const { return oy_; }
  double channel_angle(int k) const { return k * delta_theta() + theta_t(); }
  size_t plane_size() const { return static_cast<size_t>(w_) * h_; }
  size_t size() const { return plane_size() * c_; }

  std::vector<double> values() const {  // host copy
    std::vector<double> v(size());
    check(gl_tensor_download(pool_->get(), get(), v.data()));
    return v;
  }
  void set_values(const std::vector<double>& v) {
    if (v.size() != size()) throw std::invalid_argument("value count mismatch");
    check(gl_tensor_upload(pool_->get(), get(), v.data()));
  }
  double at(int i, int j, int k) const {
    double x = 0.0;
    check(gl_tensor_read(pool_->get(), get(), idx(i, j, k), 1, &x));
    return x;
  }
  void set(int i, int j, int k, double x) { check(gl_tensor_write(pool_->get(), get(), idx(i, j, k), 1, &x)); }
  std::vector<double> plane(int k) const {
    std::vector<double> v(plane_size());
    check(gl_tensor_read(pool_->get(), get(), plane_size() * k, plane_size(), v.data()));
    return v;
  }

  gl_tensor* get() const { return t_.get(); }
  ThreadPool& pool() const { return *pool_; }

 private:
  size_t idx(int i, int j, int k) const { return plane_size() * k + static_cast<size_t>(j) * w_ + i; }
  void adopt(gl_tensor* t) {
    t_.reset(t, [](gl_tensor* p) { gl_tensor_destroy(p); });
    check(gl_tensor_info(t, &w_, &h_, &c_, &cell_, &ox_, &oy_));
  }
  std::shared_ptr<gl_tensor> t_;
  ThreadPool* pool_;
  int w_ = 0, h_ = 0, c_ = 0;
  double cell_ = 0.1, ox_ = 0.0, oy_ = 0.0;
};

inline BeliefTensor init_uniform(const OccupancyMap& map, int channels) {  // belief_tensor.cpp:35-53
  gl_tensor* t = nullptr;
  check(gl_init_uniform(map.pool().get(), map.handle(), channels, &t));
  return BeliefTensor(t, map.pool());
}

inline std::pair<double, double> motion_vector(const OdometryDelta& u, int k, double theta_t,
                                               double delta_theta, double cell_size) {  // :55-62
  const double angle = k * delta_theta + theta_t;
  const double c = std::cos(angle), s = std::sin(angle);
  return {(c * u.u - s * u.v) / cell_size, (s * u.u + c * u.v) / cell_size};
}

inline void apply_motion(BeliefTensor& t, const OdometryDelta& u) {  // :340-352
  check(gl_apply_motion(t.pool().get(), t.get(), u.u, u.v, u.w));
}

// belief_tensor.cpp:396-498
inline void step(BeliefTensor& t, const OdometryDelta& u, const OccupancyMap& map, const KernelSet& kernels,
                 const Activation& act, ThreadPool& pool, StepScratch& scratch) {
  const gl_status s =
      gl_step(pool.get(), t.get(), u.u, u.v, u.w, map.handle(), kernels.get(pool), act.handle.get());
  double ms = 0.0;
  if (gl_context_last_step_ms(pool.get(), &ms) == GL_OK) {
    scratch.t_motion = ms * 1e-3;
    scratch.t_diffusion = scratch.t_masking = 0.0;
  }
  check(s);
}

inline Grid2d belief_map(const BeliefTensor& t) {  // :500-510
  Grid2d g(t.width(), t.height());
  check(gl_belief_map(t.pool().get(), t.get(), g.data.data()));
  return g;
}

inline PoseEstimate argmax_state(const BeliefTensor& t) {  // :512-541
  gl_pose_estimate e;
  check(gl_argmax(t.pool().get(), t.get(), &e));
  PoseEstimate p;
  p.pose = Pose2{e.x, e.y, e.theta};
  p.confidence = e.confidence;
  p.i = e.i, p.j = e.j, p.k = e.k;
  return p;
}

// evaluation.hpp:21-36: map_difficulty on the device (bit-exact)
struct DifficultyConfig {
  double error_threshold = 1.0;
  int beam_count = 8;
  double fov = 2.0 * M_PI;
  double max_range = 8.0;
  int stride = 1;
  int theta_bins = 8;
  LikelihoodParams likelihood{0.2, 0.05, 1};
};
inline double map_difficulty(const OccupancyMap& map, const DistanceField& field, const DifficultyConfig& cfg,
                             ThreadPool& pool) {
  gl_difficulty_config c;
  c.error_threshold = cfg.error_threshold;
  c.beam_count = cfg.beam_count;
  c.fov = cfg.fov;
  c.max_range = cfg.max_range;
  c.stride = cfg.stride;
  c.theta_bins = cfg.theta_bins;
  c.likelihood = gl_likelihood{cfg.likelihood.sigma_hit, cfg.likelihood.weight_floor, cfg.likelihood.beam_stride};
  double out = 0.0;
  check(gl_map_difficulty(pool.get(), map.handle(), field.handle(), &c, &out));
  return out;
}

// belief_tensor.hpp:144-148: BLF1 snapshot (float32 payload, lossy)
inline void write_belief_snapshot(const BeliefTensor& t, const std::string& path) {
  check(gl_write_belief_snapshot(t.pool().get(), t.get(), path.c_str()));
}
inline BeliefTensor read_belief_snapshot(const std::string& path, double cell_size, double origin_x,
                                         double origin_y, ThreadPool& pool = ThreadPool::default_pool()) {
  gl_tensor* t = nullptr;
  check(gl_read_belief_snapshot(pool.get(), path.c_str(), cell_size, origin_x, origin_y, &t));
  return BeliefTensor(t, pool);
}

inline SampleSet dither_samples(const Grid2d& bm, int budget,
                                ThreadPool& pool = ThreadPool::default_pool()) {  // observation.cpp:11-71
  const int cap = static_cast<int>(std::min<size_t>(bm.size(), 4 * static_cast<size_t>(std::max(budget, 1)) + 64));
  std::vector<int32_t> cells(2 * static_cast<size_t>(std::max(cap, 1)));
  int n = 0;
  double mass = 0.0;
  check(gl_dither(pool.get(), bm.data.data(), bm.width, bm.height, budget, cells.data(), cap, &n, &mass));
  SampleSet s;
  s.source_mass = mass;
  for (int q = 0; q < n && q < cap; ++q) s.cells.emplace_back(cells[2 * q], cells[2 * q + 1]);
  return s;
}

inline double scan_likelihood(const OccupancyMap& map, const DistanceField& field, const Pose2& pose,
                              const LidarScan& scan, const LikelihoodParams& params) {  // :73-111
  if (scan.angles.empty() || scan.angles.size() != scan.ranges.size())
    throw std::invalid_argument("scan must have matching, nonempty beams");
  double out = 0.0;
  check(gl_scan_likelihood(map.pool().get(), map.handle(), field.handle(), pose.x, pose.y, pose.theta,
                           scan.angles.data(), scan.ranges.data(), static_cast<int>(scan.angles.size()),
                           scan.max_range, gl_likelihood{params.sigma_hit, params.weight_floor, params.beam_stride},
                           &out));
  return out;
}

inline void observation_update(BeliefTensor& t, const SampleSet& samples, const LidarScan& scan,
                               const OccupancyMap& map, const DistanceField& field,
                               const LikelihoodParams& params, ThreadPool& pool) {  // :113-170
  if (samples.cells.empty()) return;
  if (scan.angles.empty() || scan.angles.size() != scan.ranges.size())
    throw std::invalid_argument("scan must have matching, nonempty beams");
  std::vector<int32_t> cells;
  for (const auto& c : samples.cells) {
    cells.push_back(c.first);
    cells.push_back(c.second);
  }
  check(gl_observation_update(pool.get(), t.get(), cells.data(), static_cast<int>(samples.cells.size()),
                              scan.angles.data(), scan.ranges.data(), static_cast<int>(scan.angles.size()),
                              scan.max_range, map.handle(), field.handle(),
                              gl_likelihood{params.sigma_hit, params.weight_floor, params.beam_stride}));
}

// ------------------------------------------------------ raycast / scans
// occupancy_map.hpp:123-124 / simulator.hpp (simulate_scan): on the device,
// bit-exact; the batch forms are for trace generation.
inline double raycast(const OccupancyMap& map, double x, double y, double angle, double max_range) {
  const double ray[3] = {x, y, angle};
  double r = 0.0;
  check(gl_raycast(map.pool().get(), map.handle(), ray, 1, max_range, &r));
  return r;
}
inline std::vector<double> raycast_batch(const OccupancyMap& map, const std::vector<double>& rays_xya,
                                         double max_range) {
  std::vector<double> r(rays_xya.size() / 3);
  check(gl_raycast(map.pool().get(), map.handle(), rays_xya.data(), static_cast<int>(r.size()), max_range,
                   r.data()));
  return r;
}
// Rng: the reference's gridloc::Rng (rng.hpp), or anything with normal():
// one draw per beam when range_noise_sigma > 0, in the reference's order.
template <class Rng>
std::vector<LidarScan> simulate_scans(const OccupancyMap& map, const std::vector<Pose2>& poses, int beam_count,
                                      double fov, double max_range, double range_noise_sigma, Rng& rng) {
  std::vector<double> p;
  for (const auto& q : poses) p.insert(p.end(), {q.x, q.y, q.theta});
  std::vector<double> noise;
  if (range_noise_sigma > 0.0 && beam_count >= 1)
    for (size_t q = 0; q < poses.size() * static_cast<size_t>(beam_count); ++q) noise.push_back(rng.normal());
  std::vector<double> angles(std::max(beam_count, 0)), ranges(poses.size() * std::max(beam_count, 0));
  check(gl_simulate_scans(map.pool().get(), map.handle(), p.data(), static_cast<int>(poses.size()), beam_count,
                          fov, max_range, range_noise_sigma, noise.empty() ? nullptr : noise.data(),
                          angles.data(), ranges.data()));
  std::vector<LidarScan> out(poses.size());
  for (size_t q = 0; q < poses.size(); ++q) {
    out[q].angles = angles;
    out[q].ranges.assign(ranges.begin() + q * beam_count, ranges.begin() + (q + 1) * beam_count);
    out[q].max_range = max_range;
  }
  return out;
}
template <class Rng>
LidarScan simulate_scan(const OccupancyMap& map, const Pose2& pose, int beam_count, double fov, double max_range,
                        double range_noise_sigma, Rng& rng) {  // simulator.cpp:63-94
  return simulate_scans(map, std::vector<Pose2>{pose}, beam_count, fov, max_range, range_noise_sigma, rng)[0];
}

// ------------------------------------------------------------- localizer
struct LocalizerConfig {  // localizer.hpp:17-26
  int channels = 128;
  MotionNoise motion_noise;
  LikelihoodParams likelihood;
  int sample_budget = 512;
  bool use_samples = true;
  double trigger_cells = 1.0;
};

class Localizer {  // localizer.hpp:28-71, localizer.cpp:7-66
 public:
  Localizer(const OccupancyMap& map, const DistanceField& field, const LocalizerConfig& config,
            ThreadPool& pool)
      : map_(map),
        field_(field),
        config_(config),
        pool_(pool),
        kernels_(build_kernels(config.motion_noise, config.channels, map.resolution(),
                               2.0 * M_PI / config.channels)),
        activation_(make_activation(map, kernels_, config.channels, pool)),
        rot_kernels_(build_kernels(MotionNoise{1e-4, 1e-4, config.motion_noise.sigma_theta}, config.channels,
                                   map.resolution(), 2.0 * M_PI / config.channels)),
        rot_activation_(make_activation(map, rot_kernels_, config.channels, pool)),
        tensor_(init_uniform(map, config.channels)),
        trigger_trans_m_(config.trigger_cells * map.resolution()),
        trigger_rot_(M_PI / config.channels) {}

  bool integrate_odometry(const OdometryDelta& delta) {
    pending_ = compose_delta(pending_, delta);
    if (std::hypot(pending_.u, pending_.v) >= trigger_trans_m_ || std::fabs(pending_.w) >= trigger_rot_) {
      flush();
      return true;
    }
    return false;
  }

  void observe(const LidarScan& scan) {
    if (!config_.use_samples) return;
    constexpr double kEps = 1e-12;
    if (std::fabs(pending_.u) > kEps || std::fabs(pending_.v) > kEps || std::fabs(pending_.w) > kEps) flush();
    // belief_map + dither on the device, no host round trip of the plane
    const int cap = config_.sample_budget * 4 + 64;
    std::vector<int32_t> cells(2 * static_cast<size_t>(cap));
    int n = 0;
    double mass = 0.0;
    check(gl_dither_tensor(pool_.get(), tensor_.get(), config_.sample_budget, cells.data(), cap, &n, &mass));
    SampleSet s;
    s.source_mass = mass;
    for (int q = 0; q < n && q < cap; ++q) s.cells.emplace_back(cells[2 * q], cells[2 * q + 1]);
    observation_update(tensor_, s, scan, map_, field_, config_.likelihood, pool_);
  }

  PoseEstimate estimate() const {
    PoseEstimate est = argmax_state(tensor_);
    est.pose = compose(est.pose, pending_);
    est.pose.theta = wrap_angle(est.pose.theta);
    return est;
  }
  const BeliefTensor& belief() const { return tensor_; }
  BeliefTensor& belief() { return tensor_; }
  const KernelSet& kernels() const { return kernels_; }
  const Activation& activation() const { return activation_; }
  const OdometryDelta& pending() const { return pending_; }
  int steps_run() const { return steps_run_; }

  void flush() {
    const bool translated = std::hypot(pending_.u, pending_.v) >= 0.5 * trigger_trans_m_;
    if (translated) {
      step(tensor_, pending_, map_, kernels_, activation_, pool_, scratch_);
    } else {
      step(tensor_, pending_, map_, rot_kernels_, rot_activation_, pool_, scratch_);
    }
    pending_ = OdometryDelta{};
    ++steps_run_;
  }

 private:
  const OccupancyMap& map_;
  const DistanceField& field_;
  LocalizerConfig config_;
  ThreadPool& pool_;
  KernelSet kernels_;
  Activation activation_;
  KernelSet rot_kernels_;
  Activation rot_activation_;
  BeliefTensor tensor_;
  StepScratch scratch_;
  OdometryDelta pending_{};
  double trigger_trans_m_;
  double trigger_rot_;
  int steps_run_ = 0;
};

// ------------------------------------------------- multi-device engine
// one process driving a theta-slab sharded belief over
// a device list (gl_engine_*). Results are bitwise the single-tensor ones.
class ShardedEngine {
 public:
  ShardedEngine(const std::vector<int>& devices, const OccupancyMap& map, int channels, int mode = GL_ENGINE_AUTO)
      : channels_(channels), w_(map.width()), h_(map.height()) {
    gl_engine* e = nullptr;
    check(gl_engine_create(devices.data(), static_cast<int>(devices.size()), map.width(), map.height(),
                           map.resolution(), map.origin_x(), map.origin_y(), map.cells().data(), channels, mode, &e));
    e_.reset(e, [](gl_engine* p) { gl_engine_destroy(p); });
  }
  void set_kernels(int slot, const KernelSet& k, ThreadPool& pool) { check(gl_engine_set_kernels(get(), slot, k.get(pool))); }
  void init_uniform() { check(gl_engine_init_uniform(get())); }
  void step(const OdometryDelta& u, int slot) { check(gl_engine_step(get(), u.u, u.v, u.w, slot)); }
  PoseEstimate argmax() const {
    gl_pose_estimate e;
    check(gl_engine_argmax(get(), &e));
    PoseEstimate p;
    p.pose = Pose2{e.x, e.y, e.theta};
    p.confidence = e.confidence;
    p.i = e.i, p.j = e.j, p.k = e.k;
    return p;
  }
  Grid2d belief_map() const {
    Grid2d g(w_, h_);
    check(gl_engine_belief_map(get(), g.data.data()));
    return g;
  }
  SampleSet observe(int budget, const LidarScan& scan, const LikelihoodParams& params) {
    if (scan.angles.empty() || scan.angles.size() != scan.ranges.size())
      throw std::invalid_argument("scan must have matching, nonempty beams");
    const int cap = budget * 4 + 64;
    std::vector<int32_t> cells(2 * static_cast<size_t>(cap));
    int n = 0;
    double mass = 0.0;
    check(gl_engine_observe(get(), budget, scan.angles.data(), scan.ranges.data(),
                            static_cast<int>(scan.angles.size()), scan.max_range,
                            gl_likelihood{params.sigma_hit, params.weight_floor, params.beam_stride}, cells.data(), cap,
                            &n, &mass));
    SampleSet s;
    s.source_mass = mass;
    for (int q = 0; q < n && q < cap; ++q) s.cells.emplace_back(cells[2 * q], cells[2 * q + 1]);
    return s;
  }
  std::vector<double> values() const {
    std::vector<double> v(static_cast<size_t>(channels_) * w_ * h_);
    check(gl_engine_download(get(), v.data(), nullptr));
    return v;
  }
  double theta_t() const {
    double th = 0.0;
    std::vector<double> v(static_cast<size_t>(channels_) * w_ * h_);
    check(gl_engine_download(get(), v.data(), &th));
    return th;
  }
  uint64_t hash() const {
    uint64_t h = 0;
    check(gl_engine_hash(get(), &h));
    return h;
  }
  int shards() const {
    int n = 0;
    check(gl_engine_info(get(), &n, nullptr, nullptr));
    return n;
  }
  gl_engine* get() const { return e_.get(); }

 private:
  std::shared_ptr<gl_engine> e_;
  int channels_, w_, h_;
};

// Localizer (localizer.hpp:28-71, localizer.cpp:7-66) over a ShardedEngine:
// the same trigger / flush / observe / estimate logic, the belief sharded
// over `devices`.
class ShardedLocalizer {
 public:
  ShardedLocalizer(const OccupancyMap& map, const DistanceField& field, const LocalizerConfig& config,
                   const std::vector<int>& devices, int mode = GL_ENGINE_AUTO,
                   ThreadPool& pool = ThreadPool::default_pool())
      : map_(map),
        field_(field),
        config_(config),
        engine_(devices, map, config.channels, mode),
        trigger_trans_m_(config.trigger_cells * map.resolution()),
        trigger_rot_(M_PI / config.channels) {
    const double dth = 2.0 * M_PI / config.channels;
    const KernelSet k = build_kernels(config.motion_noise, config.channels, map.resolution(), dth);
    const KernelSet rk = build_kernels(MotionNoise{1e-4, 1e-4, config.motion_noise.sigma_theta}, config.channels,
                                       map.resolution(), dth);
    engine_.set_kernels(0, k, pool);
    engine_.set_kernels(1, rk, pool);
    engine_.init_uniform();
  }

  bool integrate_odometry(const OdometryDelta& delta) {
    pending_ = compose_delta(pending_, delta);
    if (std::hypot(pending_.u, pending_.v) >= trigger_trans_m_ || std::fabs(pending_.w) >= trigger_rot_) {
      flush();
      return true;
    }
    return false;
  }
  void observe(const LidarScan& scan) {
    if (!config_.use_samples) return;
    constexpr double kEps = 1e-12;
    if (std::fabs(pending_.u) > kEps || std::fabs(pending_.v) > kEps || std::fabs(pending_.w) > kEps) flush();
    engine_.observe(config_.sample_budget, scan, config_.likelihood);
  }
  PoseEstimate estimate() const {
    PoseEstimate est = engine_.argmax();
    est.pose = compose(est.pose, pending_);
    est.pose.theta = wrap_angle(est.pose.theta);
    return est;
  }
  void flush() {
    const bool translated = std::hypot(pending_.u, pending_.v) >= 0.5 * trigger_trans_m_;
    engine_.step(pending_, translated ? 0 : 1);
    pending_ = OdometryDelta{};
    ++steps_run_;
  }
  std::vector<double> belief_values() const { return engine_.values(); }
  const ShardedEngine& engine() const { return engine_; }
  ShardedEngine& engine() { return engine_; }
  const OdometryDelta& pending() const { return pending_; }
  int steps_run() const { return steps_run_; }

 private:
  const OccupancyMap& map_;
  const DistanceField& field_;
  LocalizerConfig config_;
  ShardedEngine engine_;
  OdometryDelta pending_{};
  double trigger_trans_m_;
  double trigger_rot_;
  int steps_run_ = 0;
};

// ---------------------------------------------------------- wire formats
// the recorded-log inputs that feed the device Localizer.
// Host-side parsing with the reference's record grammar, clamping and
// exceptions (carmen_log.hpp:20-34, carmen_log.cpp:9-69; observation.hpp,
// observation.cpp:172-208); oracle/ref/dropin_parity.cpp checks them field by
// field (bitwise) and byte by byte against the reference.
struct CarmenEvent {  // carmen_log.hpp:13-18
  double timestamp = 0.0;
  Pose2 odom;
  bool has_scan = false;
  LidarScan scan;
};

namespace detail {
// "FLASER n r_1..r_n lx ly lt ox oy ot ts ..." after the tag; false drops
// the record (no beams, short or non-numeric fields)
inline bool carmen_flaser(std::istringstream& in, double fov, double max_range, CarmenEvent* ev) {
  std::size_t n = 0;
  in >> n;
  if (!in || n == 0) return false;
  ev->has_scan = true;
  ev->scan.max_range = max_range;
  ev->scan.ranges.resize(n);
  ev->scan.angles.resize(n);
  for (std::size_t b = 0; b < n; ++b) {
    double& r = ev->scan.ranges[b];
    if (!(in >> r)) return false;
    if (r >= max_range) r = max_range;  // no return: the sentinel
    // beams span [-fov/2, fov/2]; the expression keeps the reference's
    // operation order (bitwise-equal angles)
    ev->scan.angles[b] = n > 1 ? -fov / 2.0 + fov * static_cast<double>(b) / (n - 1) : 0.0;
  }
  double laser_x, laser_y, laser_t;  // laser pose: the filter tracks the robot frame
  in >> laser_x >> laser_y >> laser_t;
  in >> ev->odom.x >> ev->odom.y >> ev->odom.theta >> ev->timestamp;
  return static_cast<bool>(in);
}

// "ODOM x y theta tv rv accel ts ..." after the tag
inline bool carmen_odom(std::istringstream& in, CarmenEvent* ev) {
  double tv, rv, accel;
  in >> ev->odom.x >> ev->odom.y >> ev->odom.theta >> tv >> rv >> accel >> ev->timestamp;
  return static_cast<bool>(in);
}
}  // namespace detail

// FLASER and ODOM records in file order; everything else (comments, PARAM,
// other sensors, malformed records) is skipped.
inline std::vector<CarmenEvent> read_carmen_log(const std::string& path, double fov = M_PI,
                                                double max_range = 10.0) {
  std::ifstream file(path);
  if (!file) throw std::runtime_error("cannot open carmen log: " + path);
  std::vector<CarmenEvent> events;
  for (std::string line; std::getline(file, line);) {
    if (line.empty() || line.front() == '#') continue;
    std::istringstream in(line);
    std::string tag;
    in >> tag;
    CarmenEvent ev;
    const bool keep = tag == "FLASER" ? detail::carmen_flaser(in, fov, max_range, &ev)
                      : tag == "ODOM" ? detail::carmen_odom(in, &ev)
                                      : false;
    if (keep) events.push_back(std::move(ev));
  }
  return events;
}

// Body-frame odometry between consecutive events; the first is zero.
inline std::vector<OdometryDelta> carmen_odometry_deltas(const std::vector<CarmenEvent>& events) {
  std::vector<OdometryDelta> out(events.size());
  for (std::size_t q = 1; q < events.size(); ++q) out[q] = relative_delta(events[q - 1].odom, events[q].odom);
  return out;
}

// One line per scan: "t,n,max_range,a_1..a_n,r_1..r_n" with 9 significant
// digits (observation.cpp:172-183).
inline void write_scan_csv(const std::string& path, const std::vector<std::pair<double, LidarScan>>& scans) {
  std::ofstream file(path);
  if (!file) throw std::runtime_error("cannot open for writing: " + path);
  file.precision(9);
  for (const auto& entry : scans) {
    const LidarScan& sc = entry.second;
    file << entry.first << "," << sc.angles.size() << "," << sc.max_range;
    for (double a : sc.angles) file << "," << a;
    for (double r : sc.ranges) file << "," << r;
    file << "\n";
  }
}

inline std::vector<std::pair<double, LidarScan>> read_scan_csv(const std::string& path) {
  std::ifstream file(path);
  if (!file) throw std::runtime_error("cannot open scan csv: " + path);
  std::vector<std::pair<double, LidarScan>> scans;
  for (std::string line; std::getline(file, line);) {
    if (line.empty()) continue;
    std::vector<double> f;
    std::istringstream in(line);
    for (std::string tok; std::getline(in, tok, ',');) f.push_back(std::stod(tok));  // stod throws on junk
    if (f.size() < 3) throw std::runtime_error("short scan csv line");
    const auto n = static_cast<std::size_t>(f[1]);
    if (f.size() != 3 + 2 * n) throw std::runtime_error("scan csv line length mismatch");
    LidarScan sc;
    sc.max_range = f[2];
    sc.angles.assign(f.begin() + 3, f.begin() + 3 + static_cast<std::ptrdiff_t>(n));
    sc.ranges.assign(f.begin() + 3 + static_cast<std::ptrdiff_t>(n), f.end());
    scans.emplace_back(f[0], std::move(sc));
  }
  return scans;
}

}  // namespace gridloc_b200
