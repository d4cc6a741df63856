// TEST INFRASTRUCTURE ONLY. Drop-in check: the same driver code is run
// against the reference library (namespace gridloc, compiled from
// /root/reference by oracle/Makefile) and against gridloc_b200 (the C++
// header over our C-ABI). Built here into oracle/_ref/dropin_parity; the GPU
// test (tests/test_gpu_dropin.py) runs the prebuilt binary on the box.
//
// Checks, all against the reference:
//   1. step() bit-exact over random motions, several kernel sets;
//   2. a full Localizer run (reference simulator + trigger logic + sampled
//      LIDAR observations) with both implementations in lockstep: identical
//      estimate() poses, belief bit-exact after every blind step, and
//      relative L1 <= 1e-5 after observations (likelihood exp on the device).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gridloc/belief_tensor.hpp"
#include "gridloc/localizer.hpp"
#include "gridloc/observation.hpp"
#include "gridloc/occupancy_map.hpp"
#include "gridloc/rng.hpp"
#include "gridloc/simulator.hpp"
#include "gridloc/worlds.hpp"
#include "gridloc_b200.hpp"

namespace ref = gridloc;
namespace b2 = gridloc_b200;

static int g_fail = 0;
#define EXPECT(cond, ...)                     \
  do {                                        \
    if (!(cond)) {                            \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);               \
      std::printf("\n");                      \
      ++g_fail;                               \
    }                                         \
  } while (0)

static size_t bit_mismatches(const std::vector<double>& a, const std::vector<double>& b) {
  size_t n = 0;
  for (size_t q = 0; q < a.size(); ++q) n += std::memcmp(&a[q], &b[q], 8) != 0;
  return n;
}

static double rel_l1(const std::vector<double>& g, const std::vector<double>& r) {
  double num = 0.0, den = 0.0;
  for (size_t q = 0; q < g.size(); ++q) {
    num += std::fabs(g[q] - r[q]);
    den += std::fabs(r[q]);
  }
  return den > 0 ? num / den : num;
}

static b2::OccupancyMap to_b2(const ref::OccupancyMap& m, b2::ThreadPool& pool) {
  return b2::OccupancyMap(m.width(), m.height(), m.resolution(), m.cells(), m.origin_x(), m.origin_y(), pool);
}

static void check_steps(const ref::OccupancyMap& rmap, b2::ThreadPool& pool, ref::ThreadPool& rpool,
                        const ref::MotionNoise& rn, int channels) {
  const b2::OccupancyMap bmap = to_b2(rmap, pool);
  const double dth = 2.0 * M_PI / channels;
  const ref::KernelSet rks = ref::build_kernels(rn, channels, rmap.resolution(), dth);
  const b2::KernelSet bks = b2::build_kernels(b2::MotionNoise{rn.sigma_x, rn.sigma_y, rn.sigma_theta}, channels,
                                              bmap.resolution(), dth);
  const ref::Activation ract = ref::make_activation(rmap, rks, channels, rpool);
  const b2::Activation bact = b2::make_activation(bmap, bks, channels, pool);
  ref::BeliefTensor rt = ref::init_uniform(rmap, channels);
  b2::BeliefTensor bt = b2::init_uniform(bmap, channels);
  ref::StepScratch rs;
  b2::StepScratch bs;
  ref::Rng rng(17);
  for (int s = 0; s < 12; ++s) {
    const double u = rng.uniform(-0.15, 0.15), v = rng.uniform(-0.1, 0.1), w = rng.uniform(-0.3, 0.3);
    ref::step(rt, ref::OdometryDelta{u, v, w}, rmap, rks, ract, rpool, rs);
    b2::step(bt, b2::OdometryDelta{u, v, w}, bmap, bks, bact, pool, bs);
    const size_t mm = bit_mismatches(bt.values(), rt.values());
    EXPECT(mm == 0, "step %d (C=%d, noise %.3f/%.3f/%.3f): %zu values differ", s, channels, rn.sigma_x,
           rn.sigma_y, rn.sigma_theta, mm);
    EXPECT(bt.theta_t() == rt.theta_t(), "theta_t differs at step %d", s);
  }
  const ref::PoseEstimate re = ref::argmax_state(rt);
  const b2::PoseEstimate be = b2::argmax_state(bt);
  EXPECT(re.i == be.i && re.j == be.j && re.k == be.k, "argmax differs");
  EXPECT(re.pose.x == be.pose.x && re.pose.y == be.pose.y && re.pose.theta == be.pose.theta, "pose differs");
  EXPECT(std::fabs(re.confidence - be.confidence) <= 1e-12 * re.confidence, "confidence differs");
  const ref::Grid2d rbm = ref::belief_map(rt);
  const b2::Grid2d bbm = b2::belief_map(bt);
  EXPECT(bit_mismatches(bbm.data, rbm.data) == 0, "belief_map differs");
  const ref::SampleSet rsmp = ref::dither_samples(rbm, 64);
  const b2::SampleSet bsmp = b2::dither_samples(bbm, 64, pool);
  EXPECT(rsmp.cells == bsmp.cells && rsmp.source_mass == bsmp.source_mass, "dither differs (%zu vs %zu)",
         rsmp.cells.size(), bsmp.cells.size());
}

static void check_localizer(const ref::OccupancyMap& rmap, b2::ThreadPool& pool, ref::ThreadPool& rpool,
                            int channels, int ticks) {
  const b2::OccupancyMap bmap = to_b2(rmap, pool);
  const ref::DistanceField rfield = ref::distance_field(rmap);
  const b2::DistanceField bfield = b2::distance_field(bmap);
  ref::LocalizerConfig rc;
  rc.channels = channels;
  b2::LocalizerConfig bc;
  bc.channels = channels;
  ref::Localizer rl(rmap, rfield, rc, rpool);
  b2::Localizer bl(bmap, bfield, bc, pool);
  ref::Rng rng(5);
  ref::RobotState robot;
  robot.pose = ref::Pose2{rmap.center_x(12), rmap.center_y(12), 0.3};
  while (!rmap.world_free(robot.pose.x, robot.pose.y)) robot.pose.x += rmap.resolution();
  ref::RandomWalkPolicy policy;
  const ref::OdometryNoiseModel odom;
  int steps = 0, observes = 0, pose_mismatch = 0;
  double worst_l1 = 0.0;
  for (int tick = 0; tick < ticks; ++tick) {
    const ref::Command cmd = policy.next(robot, rmap, rng);
    const ref::RobotState next = ref::step_robot(robot, cmd, 0.05, rmap);
    const ref::OdometryDelta d = ref::relative_delta(robot.pose, next.pose);
    const ref::OdometryDelta meas = ref::odometry_measurement(d, odom, rng);
    robot = next;
    const bool r_step = rl.integrate_odometry(meas);
    const bool b_step = bl.integrate_odometry(b2::OdometryDelta{meas.u, meas.v, meas.w});
    EXPECT(r_step == b_step, "trigger differs at tick %d", tick);
    if (r_step) {
      ++steps;
      const size_t mm = bit_mismatches(bl.belief().values(), rl.belief().values());
      if (observes == 0) EXPECT(mm == 0, "blind step %d: %zu values differ", steps, mm);
      worst_l1 = std::max(worst_l1, rel_l1(bl.belief().values(), rl.belief().values()));
    }
    if (tick % 20 == 19) {
      const ref::LidarScan scan = ref::simulate_scan(rmap, robot.pose, 24, 2.0 * M_PI, 8.0, 0.0, rng);
      rl.observe(scan);
      b2::LidarScan bscan{scan.angles, scan.ranges, scan.max_range};
      bl.observe(bscan);
      ++observes;
      worst_l1 = std::max(worst_l1, rel_l1(bl.belief().values(), rl.belief().values()));
    }
    if (tick % 5 == 0) {
      const ref::PoseEstimate re = rl.estimate();
      const b2::PoseEstimate be = bl.estimate();
      pose_mismatch += !(re.i == be.i && re.j == be.j && re.k == be.k);
    }
  }
  EXPECT(worst_l1 <= 1e-5, "relative L1 %.3e exceeds 1e-5", worst_l1);
  EXPECT(pose_mismatch == 0, "%d estimate() poses differ", pose_mismatch);
  std::printf("{\"localizer\": {\"channels\": %d, \"ticks\": %d, \"steps\": %d, \"observes\": %d, "
              "\"worst_rel_l1\": %.3e, \"pose_mismatch\": %d}}\n",
              channels, ticks, steps, observes, worst_l1, pose_mismatch);
}

int main() {
  b2::ThreadPool pool(0, 0);
  ref::ThreadPool rpool(4);
  const ref::OccupancyMap office = ref::make_asymmetric_office_map();
  const ref::OccupancyMap twin = ref::make_twin_room_map();
  check_steps(office, pool, rpool, ref::MotionNoise{0.03, 0.03, 0.012}, 72);
  check_steps(office, pool, rpool, ref::MotionNoise{1e-4, 1e-4, 0.012}, 72);
  check_steps(twin, pool, rpool, ref::MotionNoise{0.06, 0.05, 0.07}, 8);
  check_steps(twin, pool, rpool, ref::MotionNoise{0.05, 0.05, 2.0}, 8);
  check_localizer(office, pool, rpool, 36, 600);
  check_localizer(ref::make_loop_corridor_map(), pool, rpool, 72, 600);
  std::printf("{\"dropin_parity\": \"%s\", \"failures\": %d}\n", g_fail ? "FAIL" : "ok", g_fail);
  return g_fail ? 1 : 0;
}
