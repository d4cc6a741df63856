// TEST INFRASTRUCTURE ONLY (oracle/_ref build). libpng is absent from this
// image, so the reference's image_png.cpp cannot compile. This stub provides
// the four symbols declared by /root/reference/proj/include/gridloc/image_png.hpp
// (lines 16-23) so the hot-path translation units link. PGM maps still load
// through the reference's own decoder (occupancy_map.cpp:148-165).
#include <string>
#include <vector>

#include "gridloc/image_png.hpp"
#include "gridloc/occupancy_map.hpp"

namespace gridloc {

bool looks_like_png(const std::vector<uint8_t>&) { return false; }

GrayImage decode_png_gray8(const std::vector<uint8_t>&) {
  throw MapParseError(MapError::kUnsupportedFormat,
                      "PNG decoding unavailable in the oracle build");
}

void write_png_gray8(const std::string&, const GrayImage&) {}

void write_png_rgb8(const std::string&, int, int, const std::vector<uint8_t>&) {}

}  // namespace gridloc
