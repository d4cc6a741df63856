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
//      relative L1 <= 1e-5 after observations (likelihood exp on the device);
//   3. (--io-only runs just this, no GPU needed) the wire formats: CARMEN
//      logs (hand-written edge cases + a seeded random log) parsed field by
//      field bitwise-equal, odometry deltas bitwise-equal, scan CSV files
//      byte-identical and read back bitwise-equal, malformed CSV lines
//      rejected by both.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <fstream>
#include <string>
#include <utility>
#include <vector>

#include "gridloc/belief_tensor.hpp"
#include "gridloc/carmen_log.hpp"
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
  EXPECT(re.confidence == be.confidence, "confidence differs");
  const ref::Grid2d rbm = ref::belief_map(rt);
  const b2::Grid2d bbm = b2::belief_map(bt);
  EXPECT(bit_mismatches(bbm.data, rbm.data) == 0, "belief_map differs");
  const ref::SampleSet rsmp = ref::dither_samples(rbm, 64);
  const b2::SampleSet bsmp = b2::dither_samples(bbm, 64, pool);
  EXPECT(rsmp.cells == bsmp.cells && rsmp.source_mass == bsmp.source_mass, "dither differs (%zu vs %zu)",
         rsmp.cells.size(), bsmp.cells.size());
}

static std::vector<double> values_of(const b2::Localizer& l) { return l.belief().values(); }
static std::vector<double> values_of(const b2::ShardedLocalizer& l) { return l.belief_values(); }

template <class B2Localizer, class... Extra>
static void check_localizer(const ref::OccupancyMap& rmap, b2::ThreadPool& pool, ref::ThreadPool& rpool,
                            int channels, int ticks, const char* what, Extra&&... extra) {
  const b2::OccupancyMap bmap = to_b2(rmap, pool);
  const ref::DistanceField rfield = ref::distance_field(rmap);
  const b2::DistanceField bfield = b2::distance_field(bmap);
  ref::LocalizerConfig rc;
  rc.channels = channels;
  b2::LocalizerConfig bc;
  bc.channels = channels;
  ref::Localizer rl(rmap, rfield, rc, rpool);
  B2Localizer bl(bmap, bfield, bc, std::forward<Extra>(extra)...);
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
      const std::vector<double> bv = values_of(bl);
      const size_t mm = bit_mismatches(bv, rl.belief().values());
      if (observes == 0) EXPECT(mm == 0, "blind step %d: %zu values differ", steps, mm);
      worst_l1 = std::max(worst_l1, rel_l1(bv, rl.belief().values()));
    }
    if (tick % 20 == 19) {
      const ref::LidarScan scan = ref::simulate_scan(rmap, robot.pose, 24, 2.0 * M_PI, 8.0, 0.0, rng);
      rl.observe(scan);
      b2::LidarScan bscan{scan.angles, scan.ranges, scan.max_range};
      bl.observe(bscan);
      ++observes;
      worst_l1 = std::max(worst_l1, rel_l1(values_of(bl), rl.belief().values()));
    }
    if (tick % 5 == 0) {
      const ref::PoseEstimate re = rl.estimate();
      const b2::PoseEstimate be = bl.estimate();
      pose_mismatch += !(re.i == be.i && re.j == be.j && re.k == be.k);
    }
  }
  EXPECT(worst_l1 <= 1e-5, "relative L1 %.3e exceeds 1e-5", worst_l1);
  EXPECT(pose_mismatch == 0, "%d estimate() poses differ", pose_mismatch);
  std::printf("{\"%s\": {\"channels\": %d, \"ticks\": %d, \"steps\": %d, \"observes\": %d, "
              "\"worst_rel_l1\": %.3e, \"pose_mismatch\": %d}}\n",
              what, channels, ticks, steps, observes, worst_l1, pose_mismatch);
}


static bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 8 * a.size()) == 0);
}

static std::string slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

static void check_carmen(const std::string& path, double fov, double max_range) {
  const auto re = ref::read_carmen_log(path, fov, max_range);
  const auto be = b2::read_carmen_log(path, fov, max_range);
  EXPECT(re.size() == be.size(), "%s: %zu vs %zu events", path.c_str(), re.size(), be.size());
  size_t bad = 0;
  for (size_t q = 0; q < std::min(re.size(), be.size()); ++q) {
    const auto& a = re[q];
    const auto& b = be[q];
    bad += !(same_bits(a.timestamp, b.timestamp) && same_bits(a.odom.x, b.odom.x) &&
             same_bits(a.odom.y, b.odom.y) && same_bits(a.odom.theta, b.odom.theta) && a.has_scan == b.has_scan &&
             same_bits(a.scan.max_range, b.scan.max_range) && same_bits(a.scan.angles, b.scan.angles) &&
             same_bits(a.scan.ranges, b.scan.ranges));
  }
  EXPECT(bad == 0, "%s: %zu events differ", path.c_str(), bad);
  const auto rd = ref::carmen_odometry_deltas(re);
  const auto bd = b2::carmen_odometry_deltas(be);
  size_t dbad = rd.size() != bd.size();
  for (size_t q = 0; q < std::min(rd.size(), bd.size()); ++q) {
    dbad += !(same_bits(rd[q].u, bd[q].u) && same_bits(rd[q].v, bd[q].v) && same_bits(rd[q].w, bd[q].w));
  }
  EXPECT(dbad == 0, "%s: %zu odometry deltas differ", path.c_str(), dbad);
  std::printf("{\"carmen\": {\"fov\": %.4f, \"max_range\": %.1f, \"events\": %zu, \"scans\": %zu}}\n", fov,
              max_range, re.size(),
              static_cast<size_t>(std::count_if(re.begin(), re.end(), [](const ref::CarmenEvent& e) { return e.has_scan; })));
}

template <class F>
static std::string what_of(F&& f) {
  try {
    f();
  } catch (const std::exception& e) {
    return e.what();
  }
  return "<no exception>";
}

static void check_wire_formats(const std::string& dir) {
  // CARMEN: the reference test's records plus the grammar's edge cases
  const std::string hand = dir + "/dropin_hand.log";
  {
    std::ofstream out(hand);
    out << "# comment line\n";
    out << "PARAM robot_frontlaser_offset 0.08\n";
    out << "FLASER 4 1.0 2.0 3.0 81.9 0.1 0.2 0.05 0.1 0.2 0.05 1000.1 host 1000.1\n";
    out << "ODOM 0.5 0.3 0.10 0.2 0.0 0.0 1000.2 host 1000.2\n";
    out << "\n";
    out << "FLASER 0 0.1 0.2 0.05 0.1 0.2 0.05 1000.3 host 1000.3\n";        // no beams: dropped
    out << "FLASER 3 1.0 2.0\n";                                            // truncated ranges: dropped
    out << "FLASER 2 1.0 2.0 0.1 0.2 0.05 0.1 0.2\n";                        // missing odometry: dropped
    out << "FLASER 1 12.5 0.0 0.0 0.0 -1.5 2.25 3.1 1000.4 host 1000.4\n";   // one beam, clamped
    out << "FLASER 3 1e-3 nan 7.5 0 0 0 1 2 -3.0 1000.5\n";                  // exotic numbers
    out << "ODOM 0.6 0.35\n";                                                // truncated: dropped
    out << "RLASER 2 1.0 1.0 0 0 0 0 0 0 1000.6\n";                         // other sensor: skipped
    out << "ODOM 1.0e1 -2.5 6.0 0 0 0 1000.7\n";
    out << "  ODOM 0.7 0.4 0.2 0 0 0 1000.8 host 1000.8\n";                   // leading blank
  }
  check_carmen(hand, M_PI, 10.0);
  check_carmen(hand, 4.71238898038469, 8.0);
  // a seeded random log (odometry random walk, 181-beam scans)
  const std::string rnd = dir + "/dropin_random.log";
  {
    ref::Rng rng(20191001);
    std::ofstream out(rnd);
    out.precision(17);
    double x = 0, y = 0, th = 0, t = 1000.0;
    for (int q = 0; q < 400; ++q) {
      x += rng.uniform(-0.05, 0.2);
      y += rng.uniform(-0.05, 0.05);
      th += rng.uniform(-0.1, 0.1);
      t += 0.05;
      if (q % 3 == 0) {
        out << "FLASER 181";
        for (int b = 0; b < 181; ++b) out << " " << rng.uniform(0.05, 12.0);
        out << " " << x << " " << y << " " << th << " " << x << " " << y << " " << th << " " << t << " host " << t
            << "\n";
      } else {
        out << "ODOM " << x << " " << y << " " << th << " 0.3 0.1 0 " << t << " host " << t << "\n";
      }
    }
  }
  check_carmen(rnd, M_PI, 10.0);
  EXPECT(what_of([] { ref::read_carmen_log("/nonexistent/x.log"); }) ==
             what_of([] { b2::read_carmen_log("/nonexistent/x.log"); }),
         "missing-file errors differ");

  // scan CSV: byte-identical files, bitwise read-back, same rejections
  std::vector<std::pair<double, ref::LidarScan>> rs;
  std::vector<std::pair<double, b2::LidarScan>> bs;
  ref::Rng rng(7);
  for (int q = 0; q < 50; ++q) {
    ref::LidarScan sc;
    sc.max_range = q % 2 ? 8.0 : 30.0;
    const int n = 1 + q % 37;
    for (int b = 0; b < n; ++b) {
      sc.angles.push_back(-M_PI + 2.0 * M_PI * b / n);
      sc.ranges.push_back(b % 5 == 0 ? sc.max_range : rng.uniform(0.0, sc.max_range));
    }
    const double t = 0.05 * q + rng.uniform(0.0, 1e-6);
    rs.emplace_back(t, sc);
    bs.emplace_back(t, b2::LidarScan{sc.angles, sc.ranges, sc.max_range});
  }
  const std::string rcsv = dir + "/dropin_ref.csv", bcsv = dir + "/dropin_b2.csv";
  ref::write_scan_csv(rcsv, rs);
  b2::write_scan_csv(bcsv, bs);
  const std::string rbytes = slurp(rcsv), bbytes = slurp(bcsv);
  EXPECT(!rbytes.empty() && rbytes == bbytes, "scan csv files differ (%zu vs %zu bytes)", rbytes.size(),
         bbytes.size());
  const auto rb = ref::read_scan_csv(rcsv);
  const auto bb = b2::read_scan_csv(rcsv);
  size_t bad = rb.size() != bb.size();
  for (size_t q = 0; q < std::min(rb.size(), bb.size()); ++q) {
    bad += !(same_bits(rb[q].first, bb[q].first) && same_bits(rb[q].second.max_range, bb[q].second.max_range) &&
             same_bits(rb[q].second.angles, bb[q].second.angles) &&
             same_bits(rb[q].second.ranges, bb[q].second.ranges));
  }
  EXPECT(bad == 0, "%zu scan csv records differ", bad);
  for (const char* line : {"1.0,2\n", "1.0,2,8.0,0.1\n", "1.0,x,8.0\n", "0.5,1,8.0,0.0,1.0\n\n2.0,0,4.0\n"}) {
    const std::string bad_csv = dir + "/dropin_bad.csv";
    {
      std::ofstream out(bad_csv);
      out << line;
    }
    const std::string rw = what_of([&] { ref::read_scan_csv(bad_csv); });
    const std::string bw = what_of([&] { b2::read_scan_csv(bad_csv); });
    EXPECT(rw == bw, "scan csv '%s': reference '%s' vs b200 '%s'", line, rw.c_str(), bw.c_str());
  }
  std::printf("{\"scan_csv\": {\"scans\": %zu, \"bytes\": %zu}}\n", rb.size(), rbytes.size());
}

int main(int argc, char** argv) {
  const char* tmp = std::getenv("TMPDIR");
  const std::string dir = tmp ? tmp : "/tmp";
  check_wire_formats(dir);
  if (argc > 1 && std::strcmp(argv[1], "--io-only") == 0) {
    std::printf("{\"dropin_parity\": \"%s\", \"failures\": %d}\n", g_fail ? "FAIL" : "ok", g_fail);
    return g_fail ? 1 : 0;
  }
  b2::ThreadPool pool(0, 0);
  ref::ThreadPool rpool(4);
  const ref::OccupancyMap office = ref::make_asymmetric_office_map();
  const ref::OccupancyMap twin = ref::make_twin_room_map();
  check_steps(office, pool, rpool, ref::MotionNoise{0.03, 0.03, 0.012}, 72);
  check_steps(office, pool, rpool, ref::MotionNoise{1e-4, 1e-4, 0.012}, 72);
  check_steps(twin, pool, rpool, ref::MotionNoise{0.06, 0.05, 0.07}, 8);
  check_steps(twin, pool, rpool, ref::MotionNoise{0.05, 0.05, 2.0}, 8);
  check_localizer<b2::Localizer>(office, pool, rpool, 36, 600, "localizer", pool);
  check_localizer<b2::Localizer>(ref::make_loop_corridor_map(), pool, rpool, 72, 600, "localizer", pool);
  // the same driver over a theta-sharded belief (gl_engine; three shards on
  // device 0 on a one-GPU box, peer-memory halo reads + P2P max gather)
  const std::vector<int> devs = {0, 0, 0};
  check_localizer<b2::ShardedLocalizer>(office, pool, rpool, 36, 600, "sharded_localizer", devs,
                                        static_cast<int>(GL_ENGINE_P2P), pool);
  check_localizer<b2::ShardedLocalizer>(ref::make_loop_corridor_map(), pool, rpool, 72, 400, "sharded_localizer",
                                        devs, static_cast<int>(GL_ENGINE_P2P), pool);
  std::printf("{\"dropin_parity\": \"%s\", \"failures\": %d}\n", g_fail ? "FAIL" : "ok", g_fail);
  return g_fail ? 1 : 0;
}
