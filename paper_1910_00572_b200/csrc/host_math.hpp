// Host-side setup math (see host_math.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace glb {

struct HostKernels {
  int channels = 0;
  int radius = 0;
  bool separable = false;
  bool degenerate_spatial = false;
  bool degenerate_angular = false;
  std::vector<double> sep;
  std::vector<double> spatial;
  std::vector<int> ang_off;
  std::vector<double> ang_w;
};

struct MapParseFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct MapParse {
  int w = 0, h = 0;
  std::vector<uint8_t> occ;
};

HostKernels build_kernels_host(double sigma_x, double sigma_y,
                               double sigma_theta, int channels, double cell,
                               double dtheta);
void motion_table(double u, double v, int c_begin, int count, double theta_t,
                  double dtheta, double cell, double* out_xy);
MapParse parse_pgm_map(const uint8_t* bytes, size_t n, int threshold);
// png_decode.cpp: image_png.cpp:32-100 without libpng
bool looks_like_png(const uint8_t* bytes, size_t n);
std::vector<uint8_t> decode_png_gray8(const uint8_t* bytes, size_t n, int* width, int* height);
void force_ring(uint8_t* occ, int w, int h);


}  // namespace glb
