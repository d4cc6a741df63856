// Host-side setup math of the filter: everything that calls libm
// transcendentals (exp, cos, sin) runs here, on the host, exactly where the
// reference evaluates it, so taps, motion vectors and likelihood tables are
// bit-identical to the reference on the same host. Compiled with
// -ffp-contract=off (no FMA contraction), like the reference build.
#include <vector>
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>

#include "gl_internal.hpp"
#include "host_math.hpp"

namespace glb {

// --------------------------------------------------------------- kernels
// Restates build_kernels (belief_tensor.cpp:243-338):
//   spatial: sigma below 0.1 cell -> impulse (r = 0); isotropic -> separable
//   normalised 1-D Gaussian with r = max(1, ceil(3 sigma)); otherwise one
//   rotated anisotropic (2r+1)^2 Gaussian per channel at phi = k*dtheta.
//   angular: sa = sigma_theta/dtheta; impulse below 0.1; h = max(1,ceil(3sa))
//   taps -h..h, folded mod C when 2h+1 >= C.
HostKernels build_kernels_host(double sigma_x, double sigma_y,
                               double sigma_theta, int channels, double cell,
                               double dtheta) {
  if (!(sigma_x > 0.0 && sigma_y > 0.0 && sigma_theta > 0.0)) {
    throw std::invalid_argument("motion noise sigmas must be > 0");
  }
  if (channels < 1) throw std::invalid_argument("channels must be >= 1");
  HostKernels ks;
  ks.channels = channels;
  const double sx = sigma_x / cell;
  const double sy = sigma_y / cell;
  const double smax = std::max(sx, sy);
  auto gauss1 = [](int d, double s) { return std::exp(-0.5 * d * d / (s * s)); };

  if (smax < 0.1) {
    ks.radius = 0;
    ks.degenerate_spatial = true;
    ks.spatial.assign(static_cast<size_t>(channels), 1.0);
  } else if (sx == sy) {
    const int r = std::max(1, static_cast<int>(std::ceil(3.0 * smax)));
    ks.radius = r;
    ks.separable = true;
    ks.sep.resize(2 * r + 1);
    double total = 0.0;
    for (int t = 0; t < 2 * r + 1; ++t) {
      ks.sep[t] = gauss1(t - r, sx);
      total += ks.sep[t];
    }
    for (double& t : ks.sep) t /= total;
    const int kw = 2 * r + 1;
    ks.spatial.resize(static_cast<size_t>(channels) * kw * kw);
    for (int k = 0; k < channels; ++k) {
      double* dst = ks.spatial.data() + static_cast<size_t>(k) * kw * kw;
      for (int a = 0; a < kw; ++a)
        for (int b = 0; b < kw; ++b) dst[a * kw + b] = ks.sep[a] * ks.sep[b];
    }
  } else {
    const int r = std::max(1, static_cast<int>(std::ceil(3.0 * smax)));
    ks.radius = r;
    const int kw = 2 * r + 1;
    ks.spatial.resize(static_cast<size_t>(channels) * kw * kw);
    for (int k = 0; k < channels; ++k) {
      const double phi = k * dtheta;
      const double c = std::cos(phi);
      const double s = std::sin(phi);
      double* dst = ks.spatial.data() + static_cast<size_t>(k) * kw * kw;
      double total = 0.0;
      for (int dy = -r; dy <= r; ++dy) {
        for (int dx = -r; dx <= r; ++dx) {
          const double bu = dx * c + dy * s;
          const double bv = -dx * s + dy * c;
          const double e =
              std::exp(-0.5 * (bu * bu / (sx * sx) + bv * bv / (sy * sy)));
          dst[(dy + r) * kw + (dx + r)] = e;
          total += e;
        }
      }
      for (int t = 0; t < kw * kw; ++t) dst[t] /= total;
    }
  }

  const double sa = sigma_theta / dtheta;
  if (sa < 0.1) {
    ks.degenerate_angular = true;
    ks.ang_off = {0};
    ks.ang_w = {1.0};
  } else {
    const int hh = std::max(1, static_cast<int>(std::ceil(3.0 * sa)));
    if (2 * hh + 1 >= channels) {
      std::vector<double> bins(static_cast<size_t>(channels), 0.0);
      double total = 0.0;
      for (int dk = -hh; dk <= hh; ++dk) {
        const double e = gauss1(dk, sa);
        bins[((dk % channels) + channels) % channels] += e;
        total += e;
      }
      for (int off = 0; off < channels; ++off) {
        ks.ang_off.push_back(off);
        ks.ang_w.push_back(bins[off] / total);
      }
    } else {
      double total = 0.0;
      for (int dk = -hh; dk <= hh; ++dk) total += gauss1(dk, sa);
      for (int dk = -hh; dk <= hh; ++dk) {
        ks.ang_off.push_back(dk);
        ks.ang_w.push_back(gauss1(dk, sa) / total);
      }
    }
  }
  return ks;
}

// motion_vector (belief_tensor.cpp:55-62) for every channel of a step:
// (dx, dy) in cells, with theta_t before the step's rotation is applied.
void motion_table(double u, double v, int c_begin, int count, double theta_t,
                  double dtheta, double cell, double* out_xy) {
  // The table depends only on its arguments; a stream of steps with an
  // unchanged heading offset (translations) reuses the last one instead of
  // 2 * count libm calls (~40 ns each). Per thread, whole tables only.
  struct Memo {
    double u, v, theta_t, dtheta, cell;
    int c_begin = -1, count = 0;
    std::vector<double> xy;
  };
  thread_local Memo memo;
  const bool cacheable = count > 1;
  if (cacheable && memo.count == count && memo.c_begin == c_begin && memo.u == u && memo.v == v &&
      memo.theta_t == theta_t && memo.dtheta == dtheta && memo.cell == cell &&
      std::signbit(memo.u) == std::signbit(u) && std::signbit(memo.v) == std::signbit(v) &&
      std::signbit(memo.theta_t) == std::signbit(theta_t)) {
    std::copy(memo.xy.begin(), memo.xy.end(), out_xy);
    return;
  }
  for (int q = 0; q < count; ++q) {
    const int k = c_begin + q;
    const double angle = k * dtheta + theta_t;
    const double c = std::cos(angle);
    const double s = std::sin(angle);
    out_xy[2 * q] = (c * u - s * v) / cell;
    out_xy[2 * q + 1] = (s * u + c * v) / cell;
  }
  if (cacheable) {
    memo.u = u;
    memo.v = v;
    memo.theta_t = theta_t;
    memo.dtheta = dtheta;
    memo.cell = cell;
    memo.c_begin = c_begin;
    memo.count = count;
    memo.xy.assign(out_xy, out_xy + 2 * static_cast<size_t>(count));
  }
}

// shift_plane's per-channel constants (belief_tensor.cpp:67-98), in the
// reference's operation order on the host (no FMA contraction).
void chan_rec(double dx, double dy, ChanRec* r) {
  const double fx0 = std::floor(dx);
  const double fy0 = std::floor(dy);
  const double ax = dx - fx0;
  const double ay = dy - fy0;
  r->w00 = (1.0 - ax) * (1.0 - ay);
  r->w10 = ax * (1.0 - ay);
  r->w01 = (1.0 - ax) * ay;
  r->w11 = ax * ay;
  // far-out shifts only ever read zeros; the clamp keeps the TMA box-origin
  // arithmetic free of overflow (NaN motion -> origin 0)
  const double lim = static_cast<double>(1 << 29);
  auto clamp = [&](double f) { return f == f ? static_cast<int>(std::min(std::max(f, -lim), lim)) : 0; };
  r->ox = clamp(fx0);
  r->oy = clamp(fy0);
  r->integral = (std::round(dx) == dx && std::round(dy) == dy) ? 1 : 0;
  r->map = 0;
  r->wall = 0;
  r->z = 0;
}

// ------------------------------------------------------------------ maps
namespace {

struct Cursor {
  const uint8_t* b;
  size_t n;
  size_t pos;
  // whitespace and '#' comments between header tokens
  void skip() {
    while (pos < n) {
      if (b[pos] == '#') {
        while (pos < n && b[pos] != '\n') ++pos;
      } else if (std::isspace(b[pos])) {
        ++pos;
      } else {
        break;
      }
    }
  }
  bool integer(long* out) {
    skip();
    if (pos >= n || !std::isdigit(b[pos])) return false;
    long v = 0;
    while (pos < n && std::isdigit(b[pos])) {
      v = v * 10 + (b[pos] - '0');
      if (v > std::numeric_limits<int>::max()) return false;
      ++pos;
    }
    *out = v;
    return true;
  }
};

}  // namespace

// load_map (occupancy_map.cpp:148-165) with decode_pgm (:84-145) or
// decode_png_gray8 (png_decode.cpp) and the OccupancyMap boundary ring
// (:32-40).
MapParse parse_pgm_map(const uint8_t* bytes, size_t n, int threshold) {
  if (threshold <= 0 || threshold >= 255) {
    throw std::invalid_argument("threshold must be in (0, 255)");
  }
  MapParse m;
  auto fail = [](const char* why) { return MapParseFailure(why); };
  if (looks_like_png(bytes, n)) {  // occupancy_map.cpp:154-156
    int pw = 0, ph = 0;
    const std::vector<uint8_t> gray = decode_png_gray8(bytes, n, &pw, &ph);
    m.w = pw;
    m.h = ph;
    m.occ.resize(gray.size());
    for (size_t q = 0; q < gray.size(); ++q) m.occ[q] = gray[q] >= threshold ? 0 : 1;
    force_ring(m.occ.data(), m.w, m.h);
    return m;
  }
  if (n < 2 || bytes[0] != 'P' || (bytes[1] != '2' && bytes[1] != '5')) {
    throw fail("not a P2/P5 PGM (bad magic)");
  }
  Cursor cur{bytes, n, 2};
  long w = 0, h = 0, maxval = 0;
  if (!cur.integer(&w) || !cur.integer(&h) || !cur.integer(&maxval)) {
    throw fail("expected integer in PGM header");
  }
  if (w == 0 || h == 0) throw fail("PGM with zero dimension");
  if (maxval <= 0 || maxval > 255) throw fail("PGM maxval unsupported; need 1..255");
  const size_t cells = static_cast<size_t>(w) * static_cast<size_t>(h);
  std::vector<uint8_t> gray(cells);
  if (bytes[1] == '5') {
    if (cur.pos >= n || !std::isspace(bytes[cur.pos])) {
      throw fail("missing separator before P5 raster");
    }
    ++cur.pos;
    if (n - cur.pos < cells) throw fail("P5 raster truncated");
    std::memcpy(gray.data(), bytes + cur.pos, cells);
  } else {
    for (size_t q = 0; q < cells; ++q) {
      long v = 0;
      if (!cur.integer(&v)) throw fail("P2 raster truncated");
      if (v > maxval) throw fail("P2 sample exceeds maxval");
      gray[q] = static_cast<uint8_t>(v);
    }
  }
  m.w = static_cast<int>(w);
  m.h = static_cast<int>(h);
  m.occ.resize(cells);
  for (size_t q = 0; q < cells; ++q) {
    int g = gray[q];
    if (maxval != 255) g = static_cast<uint8_t>(g * 255L / maxval);
    m.occ[q] = g >= threshold ? 0 : 1;
  }
  force_ring(m.occ.data(), m.w, m.h);
  return m;
}

void force_ring(uint8_t* occ, int w, int h) {
  for (int i = 0; i < w; ++i) {
    occ[i] = 1;
    occ[static_cast<size_t>(h - 1) * w + i] = 1;
  }
  for (int j = 0; j < h; ++j) {
    occ[static_cast<size_t>(j) * w] = 1;
    occ[static_cast<size_t>(j) * w + w - 1] = 1;
  }
}


}  // namespace glb
