// Wall-crossing mask (BASELINE north star, kernel (2): "masking by
// traversability and by wall-crossing along the motion segment"). This is an
// EXTENSION: the reference masks destination cells only
// (belief_tensor.cpp:414-416, :466-467), so it is off by default and every
// parity run keeps it off (gl_context_set_wall_mask).
//
// A bilinear tap of shift_plane moves mass from source cell s to destination
// d = s + o, o = (floor(dx) + a, floor(dy) + b), a, b in {0, 1}. The tap is
// dropped (contributes nothing) when the open segment between the two cell
// centres passes through the open interior of an occupied cell other than s
// and d; touching a cell corner does not count. Cell c (relative to s) is
// crossed iff some t in (0, 1) has |t*ox - cx| < 1/2 and |t*oy - cy| < 1/2 —
// decided exactly in integers. Crossed cells always lie inside the bounding
// box of s and d, hence inside the grid whenever both endpoints are.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define GL_HD __host__ __device__ __forceinline__
#else
#define GL_HD inline
#endif

namespace glb {

constexpr int kWallSeg = 8;       // fused path: crossed cells per tap (else the generic chain)
constexpr int kWallEntries = 64;  // fused path: distinct (floor dx, floor dy) per launch window
constexpr int kWallReach = 7;     // fused path: |crossed cell - destination| per axis

GL_HD bool wall_axis(long long o, long long c, long long* lo_n, long long* lo_d, long long* hi_n,
                     long long* hi_d) {
  if (o == 0) return c == 0;  // t unconstrained on this axis iff the cell column holds the segment
  const long long m = o < 0 ? -o : o;
  const long long cc = o < 0 ? -c : c;
  const long long ln = 2 * cc - 1, hn = 2 * cc + 1, d = 2 * m;  // t in (ln/d, hn/d)
  if (ln * *lo_d > *lo_n * d) {
    *lo_n = ln;
    *lo_d = d;
  }
  if (hn * *hi_d < *hi_n * d) {
    *hi_n = hn;
    *hi_d = d;
  }
  return true;
}

// Does the open segment (0,0) -> (ox, oy) (cell centres) cross the open
// interior of cell (cx, cy)?
GL_HD bool wall_seg_crosses(long long ox, long long oy, long long cx, long long cy) {
  long long lo_n = 0, lo_d = 1, hi_n = 1, hi_d = 1;  // t in (0, 1)
  if (!wall_axis(ox, cx, &lo_n, &lo_d, &hi_n, &hi_d)) return false;
  if (!wall_axis(oy, cy, &lo_n, &lo_d, &hi_n, &hi_d)) return false;
  return lo_n * hi_d < hi_n * lo_d;
}

// Is the tap from source (si, sj) by offset (ox, oy) blocked? occ: W*H,
// 1 = occupied. Walks the cells column by column (O(|ox| + |oy|) candidate
// tests, so large in-grid shifts stay cheap on the generic path).
GL_HD bool wall_tap_blocked(const uint8_t* occ, int w, int h, long long si, long long sj, long long ox,
                            long long oy) {
  const long long ax = ox < 0 ? -ox : ox, ay = oy < 0 ? -oy : oy;
  const long long sx = ox < 0 ? -1 : 1, sy = oy < 0 ? -1 : 1;
  for (long long u = 0; u <= ax; ++u) {
    const long long cx = sx * u;
    // y range of the segment inside column cx: t in [(2u-1)/(2ax), (2u+1)/(2ax)] (all t when ox == 0)
    long long v0 = 0, v1 = ay;
    if (ax > 0 && ay > 0) {
      // y*ax spans (u - 1/2)*ay .. (u + 1/2)*ay; candidate rows floor/ceil with a margin of one
      v0 = ((2 * u - 1) * ay) / (2 * ax) - 1;
      v1 = ((2 * u + 1) * ay) / (2 * ax) + 1;
      if (v0 < 0) v0 = 0;
      if (v1 > ay) v1 = ay;
    }
    for (long long v = v0; v <= v1; ++v) {
      const long long cy = sy * v;
      if ((cx == 0 && cy == 0) || (cx == ox && cy == oy)) continue;
      if (!wall_seg_crosses(ox, oy, cx, cy)) continue;
      const long long i = si + cx, j = sj + cy;
      if (i < 0 || i >= w || j < 0 || j >= h || occ[j * w + i]) return true;
    }
  }
  return false;
}

// The crossed cells of offset (ox, oy) relative to the DESTINATION (the
// fused kernel tests them around each output cell). Returns the full count;
// stores at most cap.
GL_HD int wall_seg_cells(int ox, int oy, int* qx, int* qy, int cap) {
  const int x0 = ox < 0 ? ox : 0, x1 = ox < 0 ? 0 : ox;
  const int y0 = oy < 0 ? oy : 0, y1 = oy < 0 ? 0 : oy;
  int n = 0;
  for (int cy = y0; cy <= y1; ++cy) {
    for (int cx = x0; cx <= x1; ++cx) {
      if ((cx == 0 && cy == 0) || (cx == ox && cy == oy)) continue;
      if (!wall_seg_crosses(ox, oy, cx, cy)) continue;
      if (n < cap) {
        qx[n] = cx - ox;
        qy[n] = cy - oy;
      }
      ++n;
    }
  }
  return n;
}

// Fused-path table entry: the four taps' crossed cells for one
// (floor dx, floor dy); a cell is packed as (qx + 8) | (qy + 8) << 4.
struct WallEntry {
  uint8_t n[4];
  uint8_t cell[4][kWallSeg];
};

}  // namespace glb
