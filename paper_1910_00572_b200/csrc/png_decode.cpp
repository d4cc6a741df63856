// PNG map ingest: decode_png_gray8 (image_png.cpp:37-100) without libpng.
//
// The reference decodes with libpng: 8-bit grayscale, or 1/2/4-bit
// grayscale expanded to 8 bits (png_set_expand_gray_1_2_4_to_8: v * 255 /
// (2^depth - 1)), or 8-bit gray+alpha with the alpha stripped; 16-bit
// images and every other colour type are rejected; interlaced (Adam7)
// images are de-interlaced by png_read_image. This restatement parses the
// chunk stream (CRC-checked like libpng's critical-chunk default), inflates
// the IDAT stream with zlib, undoes the five row filters and de-interlaces.
// Setup-time host code; the map then goes to the device like a PGM one.
#include <zlib.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "host_math.hpp"

namespace glb {

namespace {

uint32_t be32(const uint8_t* p) {
  return (static_cast<uint32_t>(p[0]) << 24) | (static_cast<uint32_t>(p[1]) << 16) |
         (static_cast<uint32_t>(p[2]) << 8) | static_cast<uint32_t>(p[3]);
}

int paeth(int a, int b, int c) {
  const int p = a + b - c;
  const int pa = p > a ? p - a : a - p;
  const int pb = p > b ? p - b : b - p;
  const int pc = p > c ? p - c : c - p;
  if (pa <= pb && pa <= pc) return a;
  return pb <= pc ? b : c;
}

// Undo the row filters of one (sub)image in place: rows of `stride` bytes
// each preceded by a filter-type byte; bpp = bytes per complete pixel (>= 1).
void unfilter(uint8_t* data, size_t rows, size_t stride, size_t bpp) {
  const uint8_t* prev = nullptr;
  for (size_t r = 0; r < rows; ++r) {
    uint8_t* line = data + r * (stride + 1);
    const int type = line[0];
    uint8_t* x = line + 1;
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= bpp ? x[i - bpp] : 0;
      const int b = prev ? prev[i] : 0;
      const int c = (prev && i >= bpp) ? prev[i - bpp] : 0;
      int v = x[i];
      switch (type) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += b; break;
        case 3: v += (a + b) >> 1; break;
        case 4: v += paeth(a, b, c); break;
        default: throw MapParseFailure("corrupt PNG stream (bad filter type)");
      }
      x[i] = static_cast<uint8_t>(v);
    }
    prev = x;
  }
}

// one 8-bit gray sample of pixel i of an unfiltered row
inline uint8_t sample(const uint8_t* row, size_t i, int depth, int channels) {
  if (depth == 8) return row[i * channels];  // gray (gray+alpha: alpha stripped)
  const int per = 8 / depth;
  const int shift = 8 - depth * (1 + static_cast<int>(i % per));
  const int v = (row[i / per] >> shift) & ((1 << depth) - 1);
  return static_cast<uint8_t>(v * (255 / ((1 << depth) - 1)));  // 1:x255 2:x85 4:x17
}

}  // namespace

bool looks_like_png(const uint8_t* b, size_t n) {  // image_png.cpp:32-35
  static const uint8_t sig[8] = {0x89, 'P', 'N', 'G', '\r', '\n', 0x1a, '\n'};
  return n >= 8 && std::memcmp(b, sig, 8) == 0;
}

std::vector<uint8_t> decode_png_gray8(const uint8_t* b, size_t n, int* width, int* height) {
  if (!looks_like_png(b, n)) throw MapParseFailure("not a PNG stream");
  size_t pos = 8;
  uint32_t w = 0, h = 0;
  int depth = 0, color = -1, interlace = 0;
  bool have_ihdr = false, have_iend = false;
  std::vector<uint8_t> z;  // concatenated IDAT payloads
  while (pos < n && !have_iend) {
    if (n - pos < 12) throw MapParseFailure("truncated PNG stream");
    const uint32_t len = be32(b + pos);
    if (len > 0x7fffffffu || n - pos - 12 < len) throw MapParseFailure("truncated PNG stream");
    const uint8_t* type = b + pos + 4;
    const uint8_t* data = b + pos + 8;
    const bool critical = (type[0] & 0x20) == 0;
    const uint32_t crc = be32(data + len);
    const uint32_t got = static_cast<uint32_t>(crc32(crc32(0L, Z_NULL, 0), type, 4 + len));
    pos += 12 + len;
    if (crc != got) {
      if (critical) throw MapParseFailure("corrupt PNG stream (CRC)");
      continue;  // libpng's default for ancillary chunks: discard
    }
    if (!have_ihdr) {
      if (std::memcmp(type, "IHDR", 4) != 0 || len != 13) throw MapParseFailure("corrupt PNG stream (no IHDR)");
      w = be32(data);
      h = be32(data + 4);
      depth = data[8];
      color = data[9];
      interlace = data[12];
      if (data[10] != 0 || data[11] != 0 || interlace > 1) throw MapParseFailure("corrupt PNG stream (IHDR)");
      if (w == 0 || h == 0) throw MapParseFailure("PNG with zero dimension");
      if (w > 0x7fffffffu || h > 0x7fffffffu) throw MapParseFailure("corrupt PNG stream (IHDR size)");
      if (static_cast<uint64_t>(w) * h > (uint64_t(1) << 32)) throw MapParseFailure("PNG map larger than 2^32 cells");
      if (depth == 16) throw MapParseFailure("16-bit PNG not supported; expected 8-bit grayscale");
      if (color != 0 && color != 4) throw MapParseFailure("PNG is not grayscale");
      const bool ok = color == 0 ? (depth == 1 || depth == 2 || depth == 4 || depth == 8) : depth == 8;
      if (!ok) throw MapParseFailure("corrupt PNG stream (bit depth)");
      have_ihdr = true;
    } else if (std::memcmp(type, "IDAT", 4) == 0) {
      z.insert(z.end(), data, data + len);
    } else if (std::memcmp(type, "IEND", 4) == 0) {
      have_iend = true;
    } else if (critical && std::memcmp(type, "PLTE", 4) != 0) {
      throw MapParseFailure("corrupt PNG stream (unknown critical chunk)");
    }
  }
  if (!have_ihdr || z.empty()) throw MapParseFailure("truncated PNG stream");
  const int channels = color == 4 ? 2 : 1;
  const size_t bits_pp = static_cast<size_t>(channels) * depth;
  const size_t bpp = std::max<size_t>(1, bits_pp / 8);
  auto stride_of = [&](size_t pw) { return (pw * bits_pp + 7) / 8; };
  // the 7 Adam7 passes (x0, y0, dx, dy), or one pass covering the image
  struct Pass {
    int x0, y0, dx, dy;
  };
  static const Pass adam7[7] = {{0, 0, 8, 8}, {4, 0, 8, 8}, {0, 4, 4, 8}, {2, 0, 4, 4},
                                {0, 2, 2, 4}, {1, 0, 2, 2}, {0, 1, 1, 2}};
  static const Pass whole[1] = {{0, 0, 1, 1}};
  const Pass* passes = interlace ? adam7 : whole;
  const int n_pass = interlace ? 7 : 1;
  size_t raw_size = 0;
  for (int q = 0; q < n_pass; ++q) {
    const size_t pw = w > static_cast<uint32_t>(passes[q].x0)
                          ? (w - passes[q].x0 + passes[q].dx - 1) / passes[q].dx : 0;
    const size_t ph = h > static_cast<uint32_t>(passes[q].y0)
                          ? (h - passes[q].y0 + passes[q].dy - 1) / passes[q].dy : 0;
    if (pw && ph) raw_size += ph * (1 + stride_of(pw));
  }
  std::vector<uint8_t> raw(raw_size);
  uLongf out_len = static_cast<uLongf>(raw_size);
  if (uncompress(raw.data(), &out_len, z.data(), static_cast<uLong>(z.size())) != Z_OK || out_len != raw_size) {
    throw MapParseFailure("corrupt PNG stream (image data)");
  }
  std::vector<uint8_t> gray(static_cast<size_t>(w) * h);
  size_t off = 0;
  for (int q = 0; q < n_pass; ++q) {
    const Pass& P = passes[q];
    const size_t pw = w > static_cast<uint32_t>(P.x0) ? (w - P.x0 + P.dx - 1) / P.dx : 0;
    const size_t ph = h > static_cast<uint32_t>(P.y0) ? (h - P.y0 + P.dy - 1) / P.dy : 0;
    if (!pw || !ph) continue;
    const size_t stride = stride_of(pw);
    unfilter(raw.data() + off, ph, stride, bpp);
    for (size_t r = 0; r < ph; ++r) {
      const uint8_t* row = raw.data() + off + r * (stride + 1) + 1;
      const size_t j = P.y0 + r * P.dy;
      for (size_t i = 0; i < pw; ++i) gray[j * w + P.x0 + i * P.dx] = sample(row, i, depth, channels);
    }
    off += ph * (1 + stride);
  }
  *width = static_cast<int>(w);
  *height = static_cast<int>(h);
  return gray;
}

}  // namespace glb
