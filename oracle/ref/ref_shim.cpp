// TEST INFRASTRUCTURE ONLY. A thin extern "C" shim over the UNMODIFIED
// reference library (compiled from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libgridloc_ref.so). It lets the Python
// tests and bench.py's CPU arm call the reference's own hot-path functions:
//   gridloc::step            belief_tensor.cpp:396-498
//   gridloc::apply_motion    belief_tensor.cpp:340-352
//   gridloc::build_kernels   belief_tensor.cpp:243-338
//   gridloc::make_activation belief_tensor.cpp:354-394
//   gridloc::belief_map      belief_tensor.cpp:500-510
//   gridloc::argmax_state    belief_tensor.cpp:512-541
//   gridloc::dither_samples  observation.cpp:11-71
//   gridloc::scan_likelihood observation.cpp:73-111
//   gridloc::observation_update observation.cpp:113-170
//   gridloc::distance_field  occupancy_map.cpp:231-271
//   gridloc::load_map        occupancy_map.cpp:148-165
// plus the simulator (simulator.cpp) and Localizer trigger logic
// (localizer.cpp:25-46) to record odometry traces. Nothing in the product
// links this file.
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gridloc/belief_tensor.hpp"
#include "gridloc/evaluation.hpp"
#include "gridloc/worlds.hpp"
#include "gridloc/geometry.hpp"
#include "gridloc/localizer.hpp"
#include "gridloc/observation.hpp"
#include "gridloc/occupancy_map.hpp"
#include "gridloc/rng.hpp"
#include "gridloc/simulator.hpp"
#include "gridloc/thread_pool.hpp"

using namespace gridloc;

namespace {

thread_local std::string g_err;

enum : int {
  kOk = 0,
  kExtinguished = 1,
  kInvalid = 2,
  kMapParse = 3,
  kRuntime = 4,
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const BeliefExtinguishedError& e) {
    g_err = e.what();
    return kExtinguished;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalid;
  } catch (const MapParseError& e) {
    g_err = e.what();
    return kMapParse;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kRuntime;
  }
}

struct Field {
  DistanceField df;
};

LidarScan make_scan(const double* angles, const double* ranges, int nb,
                    double max_range) {
  LidarScan s;
  s.angles.assign(angles, angles + nb);
  s.ranges.assign(ranges, ranges + nb);
  s.max_range = max_range;
  return s;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- thread pool ---------------------------------------------------------
void* ref_pool_new(int threads) { return new ThreadPool(threads); }
void ref_pool_free(void* p) { delete static_cast<ThreadPool*>(p); }
int ref_pool_threads(void* p) {
  return static_cast<ThreadPool*>(p)->thread_count();
}

// ---- maps ----------------------------------------------------------------
int ref_map_new(int w, int h, double res, const uint8_t* occ, double ox,
                double oy, void** out) {
  return guard([&] {
    std::vector<uint8_t> cells(occ, occ + static_cast<std::size_t>(w) * h);
    *out = new OccupancyMap(w, h, res, std::move(cells), ox, oy);
  });
}
int ref_map_load(const uint8_t* bytes, std::size_t n, int threshold,
                 double res, double ox, double oy, void** out) {
  return guard([&] {
    std::vector<uint8_t> b(bytes, bytes + n);
    *out = new OccupancyMap(load_map(b, threshold, res, ox, oy));
  });
}
void ref_map_free(void* m) { delete static_cast<OccupancyMap*>(m); }
void ref_map_dims(void* m, int* w, int* h, int* free_count) {
  auto* map = static_cast<OccupancyMap*>(m);
  *w = map->width();
  *h = map->height();
  *free_count = map->free_count();
}
void ref_map_cells(void* m, uint8_t* out) {
  const auto& c = static_cast<OccupancyMap*>(m)->cells();
  std::memcpy(out, c.data(), c.size());
}
int ref_write_pgm(void* m, uint8_t* out, std::size_t cap, std::size_t* n) {
  return guard([&] {
    const auto bytes = write_pgm(*static_cast<OccupancyMap*>(m));
    *n = bytes.size();
    if (bytes.size() <= cap) std::memcpy(out, bytes.data(), bytes.size());
  });
}

void* ref_field_new(void* m) {
  return new Field{distance_field(*static_cast<OccupancyMap*>(m))};
}
void ref_field_free(void* f) { delete static_cast<Field*>(f); }
void ref_field_values(void* f, double* out) {
  const auto& v = static_cast<Field*>(f)->df.values();
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}

// ---- kernels / activation ------------------------------------------------
int ref_kernels_new(double sx, double sy, double st, int channels,
                    double cell, double dtheta, void** out) {
  return guard([&] {
    *out = new KernelSet(
        build_kernels(MotionNoise{sx, sy, st}, channels, cell, dtheta));
  });
}
void ref_kernels_free(void* k) { delete static_cast<KernelSet*>(k); }
void ref_kernels_info(void* k, int* radius, int* separable, int* n_ang,
                      int* degen_s, int* degen_a, int* n_spatial) {
  auto* ks = static_cast<KernelSet*>(k);
  *radius = ks->radius;
  *separable = ks->separable ? 1 : 0;
  *n_ang = static_cast<int>(ks->angular.size());
  *degen_s = ks->degenerate_spatial ? 1 : 0;
  *degen_a = ks->degenerate_angular ? 1 : 0;
  *n_spatial = static_cast<int>(ks->spatial.size());
}
void ref_kernels_get(void* k, double* sep, double* spatial, int* ang_off,
                     double* ang_w) {
  auto* ks = static_cast<KernelSet*>(k);
  for (std::size_t t = 0; t < ks->sep.size(); ++t) sep[t] = ks->sep[t];
  std::size_t o = 0;
  for (const auto& s : ks->spatial) {
    for (double v : s) spatial[o++] = v;
  }
  for (std::size_t t = 0; t < ks->angular.size(); ++t) {
    ang_off[t] = ks->angular[t].first;
    ang_w[t] = ks->angular[t].second;
  }
}
void* ref_activation_new(void* map, void* kernels, int channels, void* pool) {
  return new Activation(make_activation(*static_cast<OccupancyMap*>(map),
                                        *static_cast<KernelSet*>(kernels),
                                        channels,
                                        *static_cast<ThreadPool*>(pool)));
}
void ref_activation_free(void* a) { delete static_cast<Activation*>(a); }
void ref_activation_get(void* a, double* values, double* inverse) {
  auto* act = static_cast<Activation*>(a);
  if (values) {
    std::memcpy(values, act->values.data(), act->values.size() * sizeof(double));
  }
  if (inverse) {
    std::memcpy(inverse, act->inverse.data(),
                act->inverse.size() * sizeof(double));
  }
}

// ---- tensors -------------------------------------------------------------
int ref_tensor_new(int w, int h, int c, double cell, double ox, double oy,
                   void** out) {
  return guard([&] { *out = new BeliefTensor(w, h, c, cell, ox, oy); });
}
int ref_tensor_init_uniform(void* map, int channels, void** out) {
  return guard([&] {
    *out = new BeliefTensor(
        init_uniform(*static_cast<OccupancyMap*>(map), channels));
  });
}
void ref_tensor_free(void* t) { delete static_cast<BeliefTensor*>(t); }
void ref_tensor_set(void* t, const double* vals, double theta_t) {
  auto* bt = static_cast<BeliefTensor*>(t);
  std::memcpy(bt->values().data(), vals, bt->size() * sizeof(double));
  bt->set_theta_t(theta_t);
}
void ref_tensor_get(void* t, double* vals, double* theta_t) {
  auto* bt = static_cast<BeliefTensor*>(t);
  if (vals) std::memcpy(vals, bt->values().data(), bt->size() * sizeof(double));
  if (theta_t) *theta_t = bt->theta_t();
}

// map_difficulty (evaluation.cpp:25-72) and the fixed synthetic worlds
int ref_map_difficulty(void* map, void* field, double thr, int beams, double fov, double max_range,
                       int stride, int bins, double sigma_hit, double weight_floor, int beam_stride,
                       void* pool, double* out) {
  return guard([&] {
    DifficultyConfig c;
    c.error_threshold = thr;
    c.beam_count = beams;
    c.fov = fov;
    c.max_range = max_range;
    c.stride = stride;
    c.theta_bins = bins;
    c.likelihood = LikelihoodParams{sigma_hit, weight_floor, beam_stride};
    *out = map_difficulty(*static_cast<OccupancyMap*>(map), static_cast<Field*>(field)->df, c,
                          *static_cast<ThreadPool*>(pool));
  });
}
int ref_world(int which, void** out) {
  return guard([&] {
    switch (which) {
      case 0: *out = new OccupancyMap(make_twin_room_map()); break;
      case 1: *out = new OccupancyMap(make_disconnected_twin_rooms()); break;
      case 2: *out = new OccupancyMap(make_asymmetric_office_map()); break;
      case 3: *out = new OccupancyMap(make_loop_corridor_map()); break;
      default: throw std::invalid_argument("no such world");
    }
  });
}

// BLF1 snapshots through the reference's own writer / reader
int ref_write_snapshot(void* t, const char* path) {
  return guard([&] { write_belief_snapshot(*static_cast<BeliefTensor*>(t), path); });
}
int ref_read_snapshot(const char* path, double cell, double ox, double oy, void** out) {
  return guard([&] { *out = new BeliefTensor(read_belief_snapshot(path, cell, ox, oy)); });
}
int ref_tensor_dims(void* t, int* w, int* h, int* c) {
  auto* bt = static_cast<BeliefTensor*>(t);
  *w = bt->width();
  *h = bt->height();
  *c = bt->channels();
  return 0;
}

// Same order-independent hash as gl_tensor_hash: sum of splitmix64(bits_p +
// p * golden) over the tensor.
uint64_t ref_tensor_hash(void* t) {
  const auto& v = static_cast<BeliefTensor*>(t)->values();
  uint64_t acc = 0;
  for (std::size_t p = 0; p < v.size(); ++p) {
    uint64_t bits;
    std::memcpy(&bits, &v[p], 8);
    uint64_t z = bits + static_cast<uint64_t>(p) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    acc += z ^ (z >> 31);
  }
  return acc;
}

void* ref_scratch_new() { return new StepScratch(); }
void ref_scratch_free(void* s) { delete static_cast<StepScratch*>(s); }
void ref_scratch_times(void* s, double* t3) {
  auto* sc = static_cast<StepScratch*>(s);
  t3[0] = sc->t_motion;
  t3[1] = sc->t_diffusion;
  t3[2] = sc->t_masking;
}

int ref_step(void* t, double u, double v, double w, void* map, void* kernels,
             void* act, void* pool, void* scratch) {
  return guard([&] {
    step(*static_cast<BeliefTensor*>(t), OdometryDelta{u, v, w},
         *static_cast<OccupancyMap*>(map), *static_cast<KernelSet*>(kernels),
         *static_cast<Activation*>(act), *static_cast<ThreadPool*>(pool),
         *static_cast<StepScratch*>(scratch));
  });
}
void ref_apply_motion(void* t, double u, double v, double w) {
  apply_motion(*static_cast<BeliefTensor*>(t), OdometryDelta{u, v, w});
}
void ref_motion_vector(double u, double v, double w, int k, double theta_t,
                       double dtheta, double cell, double* dx, double* dy) {
  const auto p = motion_vector(OdometryDelta{u, v, w}, k, theta_t, dtheta, cell);
  *dx = p.first;
  *dy = p.second;
}
void ref_belief_map(void* t, double* out) {
  const Grid2d g = belief_map(*static_cast<BeliefTensor*>(t));
  std::memcpy(out, g.data.data(), g.data.size() * sizeof(double));
}
int ref_argmax(void* t, int* ijk, double* pose, double* conf) {
  return guard([&] {
    const PoseEstimate e = argmax_state(*static_cast<BeliefTensor*>(t));
    ijk[0] = e.i;
    ijk[1] = e.j;
    ijk[2] = e.k;
    pose[0] = e.pose.x;
    pose[1] = e.pose.y;
    pose[2] = e.pose.theta;
    *conf = e.confidence;
  });
}

// ---- observation ---------------------------------------------------------
int ref_dither(const double* bm, int w, int h, int budget, int* cells, int cap,
               int* n, double* mass) {
  return guard([&] {
    Grid2d g(w, h);
    std::memcpy(g.data.data(), bm, g.data.size() * sizeof(double));
    const SampleSet s = dither_samples(g, budget);
    *n = static_cast<int>(s.cells.size());
    *mass = s.source_mass;
    for (int q = 0; q < *n && q < cap; ++q) {
      cells[2 * q] = s.cells[q].first;
      cells[2 * q + 1] = s.cells[q].second;
    }
  });
}
int ref_scan_likelihood(void* map, void* field, double x, double y, double th,
                        const double* angles, const double* ranges, int nb,
                        double max_range, double sigma_hit, double floor_w,
                        int stride, double* out) {
  return guard([&] {
    *out = scan_likelihood(*static_cast<OccupancyMap*>(map),
                           static_cast<Field*>(field)->df, Pose2{x, y, th},
                           make_scan(angles, ranges, nb, max_range),
                           LikelihoodParams{sigma_hit, floor_w, stride});
  });
}
int ref_observation_update(void* t, const int* cells, int n,
                           const double* angles, const double* ranges, int nb,
                           double max_range, void* map, void* field,
                           double sigma_hit, double floor_w, int stride,
                           void* pool) {
  return guard([&] {
    SampleSet s;
    for (int q = 0; q < n; ++q) s.cells.emplace_back(cells[2 * q], cells[2 * q + 1]);
    observation_update(*static_cast<BeliefTensor*>(t), s,
                       make_scan(angles, ranges, nb, max_range),
                       *static_cast<OccupancyMap*>(map),
                       static_cast<Field*>(field)->df,
                       LikelihoodParams{sigma_hit, floor_w, stride},
                       *static_cast<ThreadPool*>(pool));
  });
}
int ref_simulate_scan(void* map, double x, double y, double th, int beams,
                      double fov, double max_range, double noise,
                      uint64_t seed, double* angles, double* ranges) {
  return guard([&] {
    Rng rng(seed);
    const LidarScan s = simulate_scan(*static_cast<OccupancyMap*>(map),
                                      Pose2{x, y, th}, beams, fov, max_range,
                                      noise, rng);
    for (int b = 0; b < beams; ++b) {
      angles[b] = s.angles[b];
      ranges[b] = s.ranges[b];
    }
  });
}

// ---- rng (rng.hpp:10-74): draw sequences for the Python restatement -------
void ref_rng_draws(uint64_t seed, int n, uint64_t* u64, double* uni,
                   double* nrm) {
  Rng a(seed), b(seed), c(seed);
  for (int q = 0; q < n; ++q) {
    u64[q] = a.next_u64();
    uni[q] = b.uniform();
    nrm[q] = c.normal();
  }
}

// ---- trace recorder --------------------------------------------------------
// Runs the reference simulator (RandomWalkPolicy, step_robot,
// odometry_measurement; evaluation.cpp:135-162) from a given start pose and
// applies the Localizer trigger (localizer.cpp:25-46) WITHOUT running the
// filter, recording every step() the Localizer would issue:
//   events[6*e + 0..5] = {kind, u, v, w, slot, t}
// kind 0 = step (slot 0 main kernels, 1 rotation-only kernels),
// kind 1 = observe (u,v,w unused; a scan at the robot's true pose is written
// to scans[beams*2*obs ...]: angles then ranges). observe() first flushes any
// pending motion > 1e-12 (localizer.cpp:51-54), which is recorded as a step.
int ref_gen_trace(void* map_h, int channels, double x0, double y0, double th0,
                  uint64_t seed, int max_steps, double dt, double scan_period,
                  int beams, double fov, double max_range, double* events,
                  int max_events, int* n_events, double* scans, int max_scans,
                  int* n_scans) {
  return guard([&] {
    const auto& map = *static_cast<OccupancyMap*>(map_h);
    Rng rng(seed);
    RobotState robot;
    robot.pose = Pose2{x0, y0, th0};
    RandomWalkPolicy policy;
    const OdometryNoiseModel odom;
    const double trig_t = 1.0 * map.resolution();
    const double trig_r = M_PI / channels;
    OdometryDelta pending{};
    int ne = 0, ns = 0, nsteps = 0;
    double next_scan = scan_period;
    auto emit = [&](int kind, double u, double v, double w, int slot) {
      if (ne >= max_events) return;
      double* e = events + 6 * ne;
      e[0] = kind;
      e[1] = u;
      e[2] = v;
      e[3] = w;
      e[4] = slot;
      e[5] = robot.time;
      ++ne;
    };
    auto flush = [&] {
      const bool translated = std::hypot(pending.u, pending.v) >= 0.5 * trig_t;
      emit(0, pending.u, pending.v, pending.w, translated ? 0 : 1);
      pending = OdometryDelta{};
      ++nsteps;
    };
    while (nsteps < max_steps && ne < max_events) {
      const Command cmd = policy.next(robot, map, rng);
      const RobotState next = step_robot(robot, cmd, dt, map);
      const OdometryDelta true_delta = relative_delta(robot.pose, next.pose);
      const OdometryDelta measured = odometry_measurement(true_delta, odom, rng);
      robot = next;
      pending = compose_delta(pending, measured);
      if (std::hypot(pending.u, pending.v) >= trig_t ||
          std::fabs(pending.w) >= trig_r) {
        flush();
      }
      if (scan_period > 0.0 && robot.time + 1e-9 >= next_scan) {
        next_scan += scan_period;
        const LidarScan scan = simulate_scan(map, robot.pose, beams, fov,
                                             max_range, 0.0, rng);
        if (std::fabs(pending.u) > 1e-12 || std::fabs(pending.v) > 1e-12 ||
            std::fabs(pending.w) > 1e-12) {
          flush();
        }
        if (ns < max_scans) {
          for (int b = 0; b < beams; ++b) {
            scans[2 * beams * ns + b] = scan.angles[b];
            scans[2 * beams * ns + beams + b] = scan.ranges[b];
          }
          emit(1, robot.pose.x, robot.pose.y, robot.pose.theta, ns);
          ++ns;
        }
      }
    }
    *n_events = ne;
    *n_scans = ns;
  });
}

}  // extern "C"
