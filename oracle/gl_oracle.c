/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the gridloc hot path,
 * used as the checker for the CUDA implementation. See gl_oracle.h for the
 * usage rule and how it is pinned against the real reference.
 *
 * Every floating-point expression follows the reference's evaluation order
 * exactly (no FMA: build with -ffp-contract=off), so results are bit-equal to
 * /root/reference/proj/src/belief_tensor.cpp and observation.cpp.
 */
#define _GNU_SOURCE
#include "gl_oracle.h"

#include <ctype.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* ---------------------------------------------------------------- kernels */

/* build_kernels, belief_tensor.cpp:243-338. */
int glo_build_kernels(double sigma_x, double sigma_y, double sigma_theta,
                      int channels, double cell, double delta_theta,
                      glo_kernels* ks) {
  memset(ks, 0, sizeof(*ks));
  if (channels < 1 || channels > 4096) return GLO_INVALID; /* oracle capacity */
  if (!(sigma_x > 0.0 && sigma_y > 0.0 && sigma_theta > 0.0)) /* :245-247 */
    return GLO_INVALID;
  ks->channels = channels;
  const double sx = sigma_x / cell, sy = sigma_y / cell;
  const double smax = dmax(sx, sy);
  if (smax < 0.1) { /* :253-258 degenerate impulse */
    ks->radius = 0;
    ks->degenerate_spatial = 1;
    ks->spatial = (double*)malloc(sizeof(double) * (size_t)channels);
    for (int k = 0; k < channels; ++k) ks->spatial[k] = 1.0;
  } else if (sx == sy) { /* :259-280 isotropic separable */
    int r = (int)ceil(3.0 * smax);
    if (r < 1) r = 1;
    if (2 * r + 1 > 64) return GLO_INVALID; /* oracle capacity, not a ref rule */
    ks->radius = r;
    ks->separable = 1;
    double sum = 0.0;
    for (int d = -r; d <= r; ++d) {
      ks->sep[d + r] = exp(-0.5 * d * d / (sx * sx));
      sum += ks->sep[d + r];
    }
    for (int t = 0; t < 2 * r + 1; ++t) ks->sep[t] /= sum;
    const int kw = 2 * r + 1;
    ks->spatial = (double*)malloc(sizeof(double) * (size_t)channels * kw * kw);
    for (int k = 0; k < channels; ++k)
      for (int a = 0; a < kw; ++a)
        for (int b = 0; b < kw; ++b)
          ks->spatial[(size_t)k * kw * kw + a * kw + b] = ks->sep[a] * ks->sep[b];
  } else { /* :281-307 anisotropic, rotated by k*delta_theta (no theta_t) */
    int r = (int)ceil(3.0 * smax);
    if (r < 1) r = 1;
    ks->radius = r;
    const int kw = 2 * r + 1;
    ks->spatial = (double*)malloc(sizeof(double) * (size_t)channels * kw * kw);
    for (int k = 0; k < channels; ++k) {
      const double phi = k * delta_theta;
      const double c = cos(phi), s = sin(phi);
      double* wk = ks->spatial + (size_t)k * kw * kw;
      double sum = 0.0;
      for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) {
          const double bu = dx * c + dy * s;
          const double bv = -dx * s + dy * c;
          const double e = exp(-0.5 * (bu * bu / (sx * sx) + bv * bv / (sy * sy)));
          wk[(dy + r) * kw + (dx + r)] = e;
          sum += e;
        }
      for (int t = 0; t < kw * kw; ++t) wk[t] /= sum;
    }
  }
  const double sa = sigma_theta / delta_theta; /* :309-336 angular */
  if (sa < 0.1) {
    ks->degenerate_angular = 1;
    ks->n_ang = 1;
    ks->ang_off[0] = 0;
    ks->ang_w[0] = 1.0;
  } else {
    int hh = (int)ceil(3.0 * sa);
    if (hh < 1) hh = 1;
    if (2 * hh + 1 >= channels) { /* folded onto the circle */
      double* folded = (double*)calloc((size_t)channels, sizeof(double));
      double sum = 0.0;
      for (int dk = -hh; dk <= hh; ++dk) {
        const double e = exp(-0.5 * dk * dk / (sa * sa));
        folded[((dk % channels) + channels) % channels] += e;
        sum += e;
      }
      for (int off = 0; off < channels; ++off) {
        ks->ang_off[off] = off;
        ks->ang_w[off] = folded[off] / sum;
      }
      ks->n_ang = channels;
      free(folded);
    } else {
      double sum = 0.0;
      for (int dk = -hh; dk <= hh; ++dk) sum += exp(-0.5 * dk * dk / (sa * sa));
      for (int dk = -hh; dk <= hh; ++dk) {
        ks->ang_off[ks->n_ang] = dk;
        ks->ang_w[ks->n_ang] = exp(-0.5 * dk * dk / (sa * sa)) / sum;
        ks->n_ang++;
      }
    }
  }
  return GLO_OK;
}

void glo_kernels_free(glo_kernels* k) {
  free(k->spatial);
  k->spatial = NULL;
}

/* motion_vector, belief_tensor.cpp:55-62. */
void glo_motion_vector(double u, double v, int k, double theta_t,
                       double delta_theta, double cell, double* dx,
                       double* dy) {
  const double angle = k * delta_theta + theta_t;
  const double c = cos(angle), s = sin(angle);
  *dx = (c * u - s * v) / cell;
  *dy = (s * u + c * v) / cell;
}

/* ---------------------------------------------------------------- planes */

/* Wall-crossing mask (north-star kernel (2); NOT in the reference, which
 * masks destination cells only, belief_tensor.cpp:414-416). A bilinear tap
 * moves mass from source cell s to destination d = s + o (o integer). It is
 * blocked when the open segment between the two cell centres passes through
 * the open interior of an occupied cell other than s and d (corner touches
 * do not count). Exact integer test: cell c (relative to s) is crossed iff
 * some t in (0,1) has |t*ox - cx| < 1/2 and |t*oy - cy| < 1/2. */
static int seg_crosses(long ox, long oy, long cx, long cy) {
  long lo_n = 0, lo_d = 1, hi_n = 1, hi_d = 1; /* t in (lo, hi) */
  const long o[2] = {ox, oy}, c[2] = {cx, cy};
  for (int a = 0; a < 2; ++a) {
    if (o[a] == 0) {
      if (c[a] != 0) return 0;
      continue;
    }
    const long m = o[a] < 0 ? -o[a] : o[a];
    const long cc = o[a] < 0 ? -c[a] : c[a];
    const long ln = 2 * cc - 1, hn = 2 * cc + 1, d = 2 * m;
    if (ln * lo_d > lo_n * d) { lo_n = ln; lo_d = d; }
    if (hn * hi_d < hi_n * d) { hi_n = hn; hi_d = d; }
  }
  return lo_n * hi_d < hi_n * lo_d;
}

static int tap_blocked(const uint8_t* occ, int w, int h, long si, long sj, long ox, long oy) {
  const long x0 = ox < 0 ? ox : 0, x1 = ox < 0 ? 0 : ox;
  const long y0 = oy < 0 ? oy : 0, y1 = oy < 0 ? 0 : oy;
  for (long cy = y0; cy <= y1; ++cy)
    for (long cx = x0; cx <= x1; ++cx) {
      if ((cx == 0 && cy == 0) || (cx == ox && cy == oy)) continue;
      if (!seg_crosses(ox, oy, cx, cy)) continue;
      const long i = si + cx, j = sj + cy;
      if (i < 0 || i >= w || j < 0 || j >= h || occ[j * w + i]) return 1;
    }
  return 0;
}

/* shift_plane, belief_tensor.cpp:67-124. Integral (dx,dy) copies exactly
 * (:71-86); otherwise the 4-tap blend accumulates w00, w10, w01, w11 from
 * 0.0, skipping taps outside the grid (:107-122). wall != NULL: taps
 * blocked by the wall-crossing rule above are skipped too. */
static void shift(const double* in, double* out, int w, int h, double dx,
                  double dy, const uint8_t* wall) {
  if (round(dx) == dx && round(dy) == dy) {
    const long ix = (long)dx, iy = (long)dy;
    for (long j = 0; j < h; ++j)
      for (long i = 0; i < w; ++i) {
        const long si = i - ix, sj = j - iy;
        const int ok = si >= 0 && si < w && sj >= 0 && sj < h &&
                       !(wall && tap_blocked(wall, w, h, si, sj, ix, iy));
        out[j * w + i] = ok ? in[sj * w + si] : 0.0;
      }
    return;
  }
  const double fx = floor(dx), fy = floor(dy);
  const long sx = (long)fx, sy = (long)fy;
  const double ax = dx - fx, ay = dy - fy;
  const double w00 = (1.0 - ax) * (1.0 - ay), w10 = ax * (1.0 - ay);
  const double w01 = (1.0 - ax) * ay, w11 = ax * ay;
  for (long j = 0; j < h; ++j) {
    const long r0 = j - sy, r1 = j - sy - 1;
    const int ok0 = r0 >= 0 && r0 < h, ok1 = r1 >= 0 && r1 < h;
    for (long i = 0; i < w; ++i) {
      const long c0 = i - sx, c1 = i - sx - 1;
      const int k0 = c0 >= 0 && c0 < w, k1 = c1 >= 0 && c1 < w;
      double acc = 0.0;
      if (ok0 && k0 && !(wall && tap_blocked(wall, w, h, c0, r0, sx, sy))) acc += w00 * in[r0 * w + c0];
      if (ok0 && k1 && !(wall && tap_blocked(wall, w, h, c1, r0, sx + 1, sy))) acc += w10 * in[r0 * w + c1];
      if (ok1 && k0 && !(wall && tap_blocked(wall, w, h, c0, r1, sx, sy + 1))) acc += w01 * in[r1 * w + c0];
      if (ok1 && k1 && !(wall && tap_blocked(wall, w, h, c1, r1, sx + 1, sy + 1))) acc += w11 * in[r1 * w + c1];
      out[j * w + i] = acc;
    }
  }
}

int glo_seg_cells(int ox, int oy, int* qx, int* qy, int cap) {
  const int x0 = ox < 0 ? ox : 0, x1 = ox < 0 ? 0 : ox;
  const int y0 = oy < 0 ? oy : 0, y1 = oy < 0 ? 0 : oy;
  int n = 0;
  for (int cy = y0; cy <= y1; ++cy)
    for (int cx = x0; cx <= x1; ++cx) {
      if ((cx == 0 && cy == 0) || (cx == ox && cy == oy)) continue;
      if (!seg_crosses(ox, oy, cx, cy)) continue;
      if (n < cap) {
        qx[n] = cx - ox;
        qy[n] = cy - oy;
      }
      ++n;
    }
  return n;
}

/* convolve_plane, belief_tensor.cpp:126-193: three summation orders.
 *  - r == 0: copy (:128-131)
 *  - rows/cols within r of the border: sequential acc over in-grid taps
 *    (:135-149)
 *  - interior, r == 2 and w > 4: five per-row partial sums, each a
 *    left-to-right chain starting from the first product, added to acc
 *    (:155-177)
 *  - interior otherwise: one sequential chain from 0.0 (:178-190). */
static double dense_checked(const double* in, int w, int h, int i, int j,
                            const double* kern, int r) {
  const int kw = 2 * r + 1;
  double acc = 0.0;
  for (int dy = -r; dy <= r; ++dy) {
    const int sj = j + dy;
    if (sj < 0 || sj >= h) continue;
    for (int dx = -r; dx <= r; ++dx) {
      const int si = i + dx;
      if (si < 0 || si >= w) continue;
      acc += kern[(dy + r) * kw + dx + r] * in[(size_t)sj * w + si];
    }
  }
  return acc;
}

static void conv_dense(const double* in, double* out, int w, int h,
                       const double* kern, int r) {
  if (r == 0) {
    memcpy(out, in, sizeof(double) * (size_t)w * h);
    return;
  }
  const int kw = 2 * r + 1;
  for (int j = 0; j < h; ++j) {
    const int interior_row = j >= r && j < h - r;
    for (int i = 0; i < w; ++i) {
      /* the reference's interior span is [r, w-r) for rows inside [r, h-r);
       * columns in [0, min(r,w)) and [max(w-r,r), w) use the checked form */
      const int interior = interior_row && i >= r && i < w - r;
      double acc;
      if (!interior) {
        acc = dense_checked(in, w, h, i, j, kern, r);
      } else if (r == 2 && w > 4) {
        const double* k = kern;
        const double* q0 = in + (size_t)(j - 2) * w + (i - 2);
        const double* q1 = q0 + w;
        const double* q2 = q1 + w;
        const double* q3 = q2 + w;
        const double* q4 = q3 + w;
        acc = k[0] * q0[0] + k[1] * q0[1] + k[2] * q0[2] + k[3] * q0[3] + k[4] * q0[4];
        acc += k[5] * q1[0] + k[6] * q1[1] + k[7] * q1[2] + k[8] * q1[3] + k[9] * q1[4];
        acc += k[10] * q2[0] + k[11] * q2[1] + k[12] * q2[2] + k[13] * q2[3] + k[14] * q2[4];
        acc += k[15] * q3[0] + k[16] * q3[1] + k[17] * q3[2] + k[18] * q3[3] + k[19] * q3[4];
        acc += k[20] * q4[0] + k[21] * q4[1] + k[22] * q4[2] + k[23] * q4[3] + k[24] * q4[4];
      } else {
        acc = 0.0;
        for (int dy = -r; dy <= r; ++dy) {
          const double* q = in + (size_t)(j + dy) * w + (i - r);
          for (int dx = 0; dx < kw; ++dx) acc += kern[(dy + r) * kw + dx] * q[dx];
        }
      }
      out[(size_t)j * w + i] = acc;
    }
  }
}

/* convolve_plane_separable, belief_tensor.cpp:197-239: row pass from 0.0 over
 * in-grid taps d = -r..r, then column pass (row starts at 0.0, += tap*row for
 * in-grid rows in ascending d). Zero padding == skipping for finite input. */
static void conv_separable(const double* in, double* out, double* rows, int w,
                           int h, const double* taps, int r) {
  for (int j = 0; j < h; ++j)
    for (int i = 0; i < w; ++i) {
      double acc = 0.0;
      for (int d = -r; d <= r; ++d) {
        const int s = i + d;
        if (s >= 0 && s < w) acc += taps[d + r] * in[(size_t)j * w + s];
      }
      rows[(size_t)j * w + i] = acc;
    }
  for (int j = 0; j < h; ++j)
    for (int i = 0; i < w; ++i) {
      double acc = 0.0;
      for (int d = -r; d <= r; ++d) {
        const int sj = j + d;
        if (sj < 0 || sj >= h) continue;
        acc += taps[d + r] * rows[(size_t)sj * w + i];
      }
      out[(size_t)j * w + i] = acc;
    }
}

static void spatial_conv(const double* in, double* out, double* tmp, int w,
                         int h, const glo_kernels* ks, int k) {
  const int kw = 2 * ks->radius + 1;
  if (ks->separable)
    conv_separable(in, out, tmp, w, h, ks->sep, ks->radius);
  else
    conv_dense(in, out, w, h, ks->spatial + (size_t)k * kw * kw, ks->radius);
}

/* channel that tap t reads for output channel k: (k - off % C + C) % C
 * (belief_tensor.cpp:449-450, :384) */
static int tap_src(int k, int off, int channels) {
  return (k - off % channels + channels) % channels;
}

/* -------------------------------------------------------------- activation */

/* make_activation, belief_tensor.cpp:354-394. */
void glo_make_activation(const uint8_t* occ, int w, int h,
                         const glo_kernels* ks, double* values,
                         double* inverse) {
  const size_t plane = (size_t)w * h;
  const int C = ks->channels;
  double* base = (double*)malloc(sizeof(double) * plane);
  double* tmp = (double*)malloc(sizeof(double) * plane);
  double* diff = (double*)malloc(sizeof(double) * plane * C);
  for (size_t p = 0; p < plane; ++p) base[p] = occ[p] ? 0.0 : 1.0;
  for (int k = 0; k < C; ++k) spatial_conv(base, diff + plane * k, tmp, w, h, ks, k);
  for (int k = 0; k < C; ++k)
    for (size_t p = 0; p < plane; ++p) {
      double acc = 0.0;
      for (int t = 0; t < ks->n_ang; ++t)
        acc += ks->ang_w[t] * diff[plane * tap_src(k, ks->ang_off[t], C) + p];
      if (values) values[plane * k + p] = acc;
      inverse[plane * k + p] = 1.0 / dmax(acc, 1e-12);
    }
  free(base);
  free(tmp);
  free(diff);
}

/* init_uniform, belief_tensor.cpp:35-53. */
int glo_init_uniform(const uint8_t* occ, int w, int h, int channels,
                     double* out) {
  if (channels < 4 || channels % 2 != 0) return GLO_INVALID;
  const size_t plane = (size_t)w * h;
  size_t nfree = 0;
  for (size_t p = 0; p < plane; ++p) nfree += occ[p] == 0;
  if (nfree == 0) return GLO_INVALID;
  for (int k = 0; k < channels; ++k)
    for (size_t p = 0; p < plane; ++p) out[plane * k + p] = occ[p] ? 0.0 : 1.0;
  return GLO_OK;
}

/* -------------------------------------------------------------------- step */

/* step, belief_tensor.cpp:396-498 (Algorithm 1). */
int glo_step(double* B, int w, int h, int C, double cell, double* theta_t,
             double u, double v, double dw, const uint8_t* occ,
             const glo_kernels* ks, const double* inverse) {
  return glo_step_wall(B, w, h, C, cell, theta_t, u, v, dw, occ, ks, inverse, 0);
}

int glo_step_wall(double* B, int w, int h, int C, double cell, double* theta_t,
                  double u, double v, double dw, const uint8_t* occ,
                  const glo_kernels* ks, const double* inverse, int wall_mask) {
  const size_t plane = (size_t)w * h;
  const double dtheta = 2.0 * M_PI / C;
  double* S = (double*)malloc(sizeof(double) * plane * C);
  double* D = (double*)malloc(sizeof(double) * plane * C);
  double* tmp = (double*)malloc(sizeof(double) * plane);
  /* phase 1: shift by the channel's motion vector, mask (:408-417) */
  for (int k = 0; k < C; ++k) {
    double dx, dy;
    glo_motion_vector(u, v, k, *theta_t, dtheta, cell, &dx, &dy);
    double* s = S + plane * k;
    shift(B + plane * k, s, w, h, dx, dy, wall_mask ? occ : NULL);
    for (size_t p = 0; p < plane; ++p)
      if (occ[p]) s[p] = 0.0;
  }
  /* phase 2: spatial diffusion (:423-436) */
  for (int k = 0; k < C; ++k) spatial_conv(S + plane * k, D + plane * k, tmp, w, h, ks, k);
  /* phase 3: circular angular taps (first tap initialises, the rest +=),
   * mask, multiply by the activation inverse, channel max (:440-475) */
  double gmax = 0.0;
  for (int k = 0; k < C; ++k) {
    double* o = B + plane * k;
    const double* inv = inverse + plane * k;
    const double* s0 = D + plane * tap_src(k, ks->ang_off[0], C);
    const double w0 = ks->ang_w[0];
    for (size_t p = 0; p < plane; ++p) o[p] = w0 * s0[p];
    for (int t = 1; t < ks->n_ang; ++t) {
      const double* st = D + plane * tap_src(k, ks->ang_off[t], C);
      const double wt = ks->ang_w[t];
      for (size_t p = 0; p < plane; ++p) o[p] += wt * st[p];
    }
    double mx = 0.0;
    for (size_t p = 0; p < plane; ++p) {
      if (occ[p]) {
        o[p] = 0.0;
      } else {
        o[p] = o[p] * inv[p];
        mx = dmax(mx, o[p]);
      }
    }
    gmax = dmax(gmax, mx);
  }
  free(S);
  free(D);
  free(tmp);
  *theta_t = *theta_t + dw; /* :478 */
  if (gmax <= 0.0) return GLO_EXTINGUISHED; /* :482-485 */
  if (gmax < 1e-6) { /* :486-493 */
    const double sc = 1.0 / gmax;
    for (size_t p = 0; p < plane * C; ++p) B[p] *= sc;
  }
  return GLO_OK;
}

/* apply_motion, belief_tensor.cpp:340-352: shift only, no mask. */
void glo_apply_motion(double* B, int w, int h, int C, double cell,
                      double* theta_t, double u, double v, double dw) {
  const size_t plane = (size_t)w * h;
  const double dtheta = 2.0 * M_PI / C;
  double* tmp = (double*)malloc(sizeof(double) * plane);
  for (int k = 0; k < C; ++k) {
    double dx, dy;
    glo_motion_vector(u, v, k, *theta_t, dtheta, cell, &dx, &dy);
    if (dx == 0.0 && dy == 0.0) continue;
    shift(B + plane * k, tmp, w, h, dx, dy, NULL);
    memcpy(B + plane * k, tmp, sizeof(double) * plane);
  }
  free(tmp);
  *theta_t = *theta_t + dw;
}

/* belief_map, belief_tensor.cpp:500-510. */
void glo_belief_map(const double* B, int w, int h, int C, double* out) {
  const size_t plane = (size_t)w * h;
  for (size_t p = 0; p < plane; ++p) out[p] = 0.0;
  for (int k = 0; k < C; ++k)
    for (size_t p = 0; p < plane; ++p) out[p] = dmax(out[p], B[plane * k + p]);
}

static double wrap_angle(double a) { /* geometry.hpp:8-13 */
  a = fmod(a, 2.0 * M_PI);
  if (a < -M_PI) a += 2.0 * M_PI;
  if (a >= M_PI) a -= 2.0 * M_PI;
  return a;
}

/* argmax_state, belief_tensor.cpp:512-541. */
int glo_argmax(const double* B, int w, int h, int C, double cell, double ox,
               double oy, double theta_t, int* ijk, double* pose,
               double* confidence) {
  const size_t plane = (size_t)w * h;
  double best = -1.0, total = 0.0;
  size_t best_p = 0;
  int best_k = 0;
  for (int k = 0; k < C; ++k)
    for (size_t p = 0; p < plane; ++p) {
      const double x = B[plane * k + p];
      total += x;
      if (x > best) {
        best = x;
        best_p = p;
        best_k = k;
      }
    }
  if (best <= 0.0) return GLO_EXTINGUISHED;
  ijk[0] = (int)(best_p % (size_t)w);
  ijk[1] = (int)(best_p / (size_t)w);
  ijk[2] = best_k;
  pose[0] = ox + (ijk[0] + 0.5) * cell;
  pose[1] = oy + (ijk[1] + 0.5) * cell;
  pose[2] = wrap_angle(best_k * (2.0 * M_PI / C) + theta_t);
  *confidence = total > 0.0 ? best / total : 0.0;
  return GLO_OK;
}

/* ------------------------------------------------------------- observation */

/* dither_samples, observation.cpp:11-71: serpentine Floyd-Steinberg. */
int glo_dither(const double* bm, int w, int h, int budget, int* cells, int cap,
               int* n, double* source_mass) {
  *n = 0;
  if (budget < 1) return GLO_INVALID;
  const size_t plane = (size_t)w * h;
  double total = 0.0;
  for (size_t p = 0; p < plane; ++p) total += bm[p];
  *source_mass = total;
  if (total <= 0.0) return GLO_OK;
  const double scale = budget / total;
  double* work = (double*)malloc(sizeof(double) * plane);
  for (size_t p = 0; p < plane; ++p) work[p] = bm[p] * scale;
  for (int j = 0; j < h; ++j) {
    const int dir = (j % 2 == 0) ? 1 : -1;
    /* the four targets (dir,0) 7/16, (-dir,1) 3/16, (0,1) 5/16, (dir,1) 1/16 */
    const int tdi[4] = {dir, -dir, 0, dir};
    const int tdj[4] = {0, 1, 1, 1};
    const double tw[4] = {7.0 / 16.0, 3.0 / 16.0, 5.0 / 16.0, 1.0 / 16.0};
    for (int i = (dir == 1 ? 0 : w - 1); i >= 0 && i < w; i += dir) {
      const size_t p = (size_t)j * w + i;
      const double val = work[p];
      double q = 0.0;
      if (val >= 0.5 && bm[p] > 0.0) {
        q = 1.0;
        if (*n < cap) {
          cells[2 * *n] = i;
          cells[2 * *n + 1] = j;
        }
        ++*n;
      }
      const double err = val - q;
      double wsum = 0.0;
      int in[4];
      for (int t = 0; t < 4; ++t) {
        const int ti = i + tdi[t], tj = j + tdj[t];
        in[t] = ti >= 0 && ti < w && tj >= 0 && tj < h;
        if (in[t]) wsum += tw[t];
      }
      if (wsum > 0.0)
        for (int t = 0; t < 4; ++t)
          if (in[t]) work[(size_t)(j + tdj[t]) * w + (i + tdi[t])] += err * (tw[t] / wsum);
      work[p] = 0.0;
    }
  }
  free(work);
  return GLO_OK;
}

/* distance_field, occupancy_map.cpp:231-271 (column sweeps + F&H 1D EDT). */
void glo_distance_field(const uint8_t* occ, int w, int h, double res,
                        double* out) {
  const int far = w + h;
  double* sq = out;
  for (int i = 0; i < w; ++i) {
    int run = far;
    for (int j = 0; j < h; ++j) {
      run = occ[(size_t)j * w + i] ? 0 : (run >= far ? far : run + 1);
      sq[(size_t)j * w + i] = run;
    }
    run = far;
    for (int j = h - 1; j >= 0; --j) {
      run = occ[(size_t)j * w + i] ? 0 : (run >= far ? far : run + 1);
      double c = sq[(size_t)j * w + i];
      c = c < (double)run ? c : (double)run; /* std::min(cell, run) */
      sq[(size_t)j * w + i] = c * c;
    }
  }
  double* f = (double*)malloc(sizeof(double) * w);
  double* d = (double*)malloc(sizeof(double) * w);
  double* z = (double*)malloc(sizeof(double) * (w + 1));
  int* v = (int*)malloc(sizeof(int) * w);
  for (int j = 0; j < h; ++j) {
    for (int i = 0; i < w; ++i) f[i] = sq[(size_t)j * w + i];
    int k = 0;
    v[0] = 0;
    z[0] = -INFINITY;
    z[1] = INFINITY;
    for (int q = 1; q < w; ++q) {
      double s;
      for (;;) {
        const int p = v[k];
        s = ((f[q] + q * q) - (f[p] + p * p)) / (2.0 * q - 2.0 * p);
        if (s <= z[k]) --k;
        else break;
      }
      ++k;
      v[k] = q;
      z[k] = s;
      z[k + 1] = INFINITY;
    }
    k = 0;
    for (int q = 0; q < w; ++q) {
      while (z[k + 1] < q) ++k;
      const int p = v[k];
      d[q] = (q - p) * (q - p) + f[p];
    }
    for (int i = 0; i < w; ++i) sq[(size_t)j * w + i] = d[i];
  }
  for (size_t p = 0; p < (size_t)w * h; ++p) out[p] = sqrt(sq[p]) * res;
  free(f);
  free(d);
  free(z);
  free(v);
}

/* scan_likelihood, observation.cpp:73-111. */
int glo_scan_likelihood(const uint8_t* occ, const double* field, int w, int h,
                        double res, double ox, double oy, double px_,
                        double py_, double pth, const double* angles,
                        const double* ranges, int nb, double max_range,
                        double sigma_hit, double weight_floor, int beam_stride,
                        double* out) {
  if (nb <= 0) return GLO_INVALID;
  const double fl = weight_floor;
  {
    const int ci = (int)floor((px_ - ox) / res), cj = (int)floor((py_ - oy) / res);
    if (!(ci >= 0 && ci < w && cj >= 0 && cj < h) || occ[(size_t)cj * w + ci]) {
      *out = fl;
      return GLO_OK;
    }
  }
  const double half_cell = 0.5 * res;
  const double inv2s2 = 1.0 / (2.0 * sigma_hit * sigma_hit);
  double log_sum = 0.0;
  int counted = 0;
  const int stride = beam_stride > 1 ? beam_stride : 1;
  for (int b = 0; b < nb; b += stride) {
    const double r = ranges[b];
    if (r >= max_range - 1e-9) continue;
    const double a = pth + angles[b];
    const double reach = r + half_cell;
    const double ex = px_ + reach * cos(a);
    const double ey = py_ + reach * sin(a);
    const int ci = (int)floor((ex - ox) / res);
    const int cj = (int)floor((ey - oy) / res);
    double gauss = 0.0;
    if (ci >= 0 && ci < w && cj >= 0 && cj < h) {
      const double dd = field[(size_t)cj * w + ci];
      gauss = exp(-dd * dd * inv2s2);
    }
    log_sum += log((1.0 - fl) * gauss + fl);
    ++counted;
  }
  *out = counted == 0 ? 1.0 : exp(log_sum / counted);
  return GLO_OK;
}

/* observation_update, observation.cpp:113-170. */
int glo_observation_update(double* B, int w, int h, int C, double cell,
                           double ox, double oy, double theta_t,
                           const int* cells, int n, const double* angles,
                           const double* ranges, int nb, double max_range,
                           const uint8_t* occ, const double* field,
                           double sigma_hit, double weight_floor,
                           int beam_stride) {
  if (n == 0) return GLO_OK;
  if (nb <= 0) return GLO_INVALID;
  const size_t plane = (size_t)w * h;
  const double dtheta = 2.0 * M_PI / C;
  double* L = (double*)malloc(sizeof(double) * (size_t)n * C);
  for (int s = 0; s < n; ++s) {
    const double x = ox + (cells[2 * s] + 0.5) * cell;
    const double y = oy + (cells[2 * s + 1] + 0.5) * cell;
    for (int k = 0; k < C; ++k)
      glo_scan_likelihood(occ, field, w, h, cell, ox, oy, x, y,
                          k * dtheta + theta_t, angles, ranges, nb, max_range,
                          sigma_hit, weight_floor, beam_stride, &L[(size_t)s * C + k]);
  }
  double mean = 0.0;
  for (size_t q = 0; q < (size_t)n * C; ++q) mean += L[q];
  mean /= (double)((size_t)n * C);
  for (int s = 0; s < n; ++s)
    for (int k = 0; k < C; ++k) {
      double* x = &B[plane * k + (size_t)cells[2 * s + 1] * w + cells[2 * s]];
      *x *= L[(size_t)s * C + k] / mean;
    }
  free(L);
  double gmax = 0.0;
  for (size_t p = 0; p < plane * C; ++p) gmax = dmax(gmax, B[p]);
  if (gmax <= 0.0) return GLO_EXTINGUISHED;
  const double sc = 1.0 / gmax;
  for (size_t p = 0; p < plane * C; ++p) B[p] *= sc;
  return GLO_OK;
}

/* ------------------------------------------------------------------ maps */

/* load_map + decode_pgm, occupancy_map.cpp:84-165 and the boundary ring of
 * the OccupancyMap ctor (:32-40). */
static int pgm_int(const uint8_t* b, size_t n, size_t* pos, long* out) {
  for (;;) {
    while (*pos < n && isspace(b[*pos])) ++*pos;
    if (*pos < n && b[*pos] == '#') {
      while (*pos < n && b[*pos] != '\n') ++*pos;
      continue;
    }
    break;
  }
  if (*pos >= n || !isdigit(b[*pos])) return GLO_MAP_PARSE;
  long v = 0;
  while (*pos < n && isdigit(b[*pos])) {
    v = v * 10 + (b[*pos] - '0');
    if (v > 2147483647L) return GLO_MAP_PARSE;
    ++*pos;
  }
  *out = v;
  return GLO_OK;
}

int glo_load_map(const uint8_t* b, size_t n, int threshold, int* w, int* h,
                 uint8_t* occ) {
  if (threshold <= 0 || threshold >= 255) return GLO_INVALID;
  if (n < 2 || b[0] != 'P' || (b[1] != '2' && b[1] != '5')) return GLO_MAP_PARSE;
  size_t pos = 2;
  long W, H, maxval;
  if (pgm_int(b, n, &pos, &W) || pgm_int(b, n, &pos, &H) || pgm_int(b, n, &pos, &maxval))
    return GLO_MAP_PARSE;
  if (W == 0 || H == 0 || maxval <= 0 || maxval > 255) return GLO_MAP_PARSE;
  *w = (int)W;
  *h = (int)H;
  if (!occ) return GLO_OK;
  const size_t cnt = (size_t)W * H;
  if (b[1] == '5') {
    if (pos >= n || !isspace(b[pos])) return GLO_MAP_PARSE;
    ++pos;
    if (n - pos < cnt) return GLO_MAP_PARSE;
    for (size_t q = 0; q < cnt; ++q) occ[q] = b[pos + q];
  } else {
    for (size_t q = 0; q < cnt; ++q) {
      long v;
      if (pgm_int(b, n, &pos, &v) || v > maxval) return GLO_MAP_PARSE;
      occ[q] = (uint8_t)v;
    }
  }
  for (size_t q = 0; q < cnt; ++q) {
    uint8_t g = occ[q];
    if (maxval != 255) g = (uint8_t)(g * 255L / maxval);
    occ[q] = g >= threshold ? 0 : 1;
  }
  for (long i = 0; i < W; ++i) {
    occ[i] = 1;
    occ[(size_t)(H - 1) * W + i] = 1;
  }
  for (long j = 0; j < H; ++j) {
    occ[(size_t)j * W] = 1;
    occ[(size_t)j * W + W - 1] = 1;
  }
  return GLO_OK;
}
