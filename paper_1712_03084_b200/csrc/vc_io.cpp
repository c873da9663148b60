// SPDX-License-Identifier: Apache-2.0
//
// Host I/O either side of the frame path: PNG depth /
// colour frames in (the reference's image_io.cpp:84-122 over libpng; here a
// zlib-based codec of the PNG format) and the textured mesh out as the
// reference's binary PLY (mesh_io.cpp:104-145 with the channels of
// TexturedMesh::with_channels, texture.cpp:74-91).
//
// Decoding follows the reference's libpng transforms: colour images are
// expanded (palette -> RGB, gray < 8 bit -> 8 bit), 16-bit samples are
// stripped to their high byte, alpha is dropped, gray becomes RGB; depth
// images must be 16-bit grayscale and are returned host-endian.  Writing
// emits non-interlaced 8-bit RGB / 16-bit gray PNGs; the compressed bytes
// differ from libpng's, the decoded pixels are identical.
#include <zlib.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "vc/vc.h"

namespace {

thread_local std::string g_io_err;

vc_status io_fail(vc_status s, const std::string& what, const char* path) {
  g_io_err = what + ": " + (path ? path : "(null)");
  return s;
}

uint32_t be32(const uint8_t* p) { return (uint32_t)p[0] << 24 | (uint32_t)p[1] << 16 | (uint32_t)p[2] << 8 | p[3]; }
void put_be32(std::vector<uint8_t>& o, uint32_t v) {
  o.push_back(v >> 24), o.push_back((v >> 16) & 255), o.push_back((v >> 8) & 255), o.push_back(v & 255);
}

bool read_file(const char* path, std::vector<uint8_t>& out) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  out.resize(n > 0 ? (size_t)n : 0);
  const size_t got = n > 0 ? std::fread(out.data(), 1, (size_t)n, f) : 0;
  std::fclose(f);
  return got == out.size();
}

const uint8_t kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};

struct Png {
  int w = 0, h = 0, depth = 0, ctype = 0, interlace = 0;
  std::vector<uint8_t> plte;  // palette RGB triples
  std::vector<uint8_t> idat;  // concatenated IDAT payload
};

// Chunk walk: IHDR, PLTE, IDAT*, IEND (CRCs are checked).
vc_status parse_png(const char* path, Png& p) {
  std::vector<uint8_t> b;
  if (!read_file(path, b)) return io_fail(VC_ERR_INVALID_ARGUMENT, "cannot open for reading", path);
  if (b.size() < 8 || std::memcmp(b.data(), kSig, 8) != 0) return io_fail(VC_ERR_INVALID_ARGUMENT, "png read error", path);
  size_t o = 8;
  bool have_hdr = false, end = false;
  while (o + 12 <= b.size() && !end) {
    const uint32_t len = be32(&b[o]);
    if (o + 12 + (size_t)len > b.size()) break;
    const uint8_t* type = &b[o + 4];
    const uint8_t* data = &b[o + 8];
    const uint32_t crc = be32(&b[o + 8 + len]);
    if ((uint32_t)crc32(0L, type, 4 + len) != crc) return io_fail(VC_ERR_INVALID_ARGUMENT, "png read error", path);
    if (!std::memcmp(type, "IHDR", 4) && len == 13) {
      p.w = (int)be32(data), p.h = (int)be32(data + 4), p.depth = data[8], p.ctype = data[9];
      p.interlace = data[12];
      have_hdr = data[10] == 0 && data[11] == 0;
    } else if (!std::memcmp(type, "PLTE", 4)) {
      p.plte.assign(data, data + len);
    } else if (!std::memcmp(type, "IDAT", 4)) {
      p.idat.insert(p.idat.end(), data, data + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      end = true;
    }
    o += 12 + len;
  }
  if (!have_hdr || !end || p.w <= 0 || p.h <= 0) return io_fail(VC_ERR_INVALID_ARGUMENT, "png read error", path);
  if (p.interlace != 0) return io_fail(VC_ERR_INVALID_ARGUMENT, "interlaced png not supported", path);
  return VC_OK;
}

int channels_of(int ctype) {
  switch (ctype) {
    case 0: return 1;  // gray
    case 2: return 3;  // RGB
    case 3: return 1;  // palette index
    case 4: return 2;  // gray + alpha
    case 6: return 4;  // RGBA
  }
  return 0;
}

// Inflate + undo the per-row filters (PNG spec 9.2-9.4).  Output: h rows of
// `stride` bytes (samples big-endian as stored).
vc_status inflate_rows(const char* path, const Png& p, std::vector<uint8_t>& rows, size_t* stride_out, int* bpp_out) {
  const int ch = channels_of(p.ctype);
  if (!ch) return io_fail(VC_ERR_INVALID_ARGUMENT, "png read error", path);
  const size_t bits = (size_t)p.w * ch * p.depth;
  const size_t stride = (bits + 7) / 8;
  const int bpp = std::max(1, ch * p.depth / 8);  // filter byte distance
  std::vector<uint8_t> raw((stride + 1) * (size_t)p.h);
  uLongf n = (uLongf)raw.size();
  if (uncompress(raw.data(), &n, p.idat.data(), (uLong)p.idat.size()) != Z_OK || n != raw.size())
    return io_fail(VC_ERR_INVALID_ARGUMENT, "png read error", path);
  rows.assign(stride * (size_t)p.h, 0);
  for (int y = 0; y < p.h; ++y) {
    const uint8_t f = raw[(size_t)y * (stride + 1)];
    const uint8_t* s = &raw[(size_t)y * (stride + 1) + 1];
    uint8_t* d = &rows[(size_t)y * stride];
    const uint8_t* up = y ? &rows[(size_t)(y - 1) * stride] : nullptr;
    for (size_t i = 0; i < stride; ++i) {
      const int a = i >= (size_t)bpp ? d[i - bpp] : 0;
      const int b = up ? up[i] : 0;
      const int c = (up && i >= (size_t)bpp) ? up[i - bpp] : 0;
      int v = s[i];
      switch (f) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += b; break;
        case 3: v += (a + b) >> 1; break;
        case 4: {
          const int pp = a + b - c, pa = std::abs(pp - a), pb = std::abs(pp - b), pc = std::abs(pp - c);
          v += (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
          break;
        }
        default: return io_fail(VC_ERR_INVALID_ARGUMENT, "png read error", path);
      }
      d[i] = (uint8_t)v;
    }
  }
  *stride_out = stride;
  *bpp_out = bpp;
  return VC_OK;
}

// sample s of row r (any depth), as an 8-bit value with the transforms of
// png_set_expand (low bit depths scaled to 8 bits) / png_set_strip_16
int sample8(const uint8_t* row, size_t idx, int depth, bool palette_index) {
  switch (depth) {
    case 16: return row[2 * idx];  // high byte
    case 8: return row[idx];
    default: {
      const int per = 8 / depth;
      const int v = (row[idx / per] >> (8 - depth * (1 + (int)(idx % per)))) & ((1 << depth) - 1);
      if (palette_index) return v;
      return v * 255 / ((1 << depth) - 1);
    }
  }
}

vc_status write_png(const char* path, int w, int h, int depth, int ctype, const uint8_t* rows_be, size_t stride) {
  std::vector<uint8_t> raw;
  raw.reserve((stride + 1) * (size_t)h);
  for (int y = 0; y < h; ++y) {  // filter type 0 (None) per row
    raw.push_back(0);
    raw.insert(raw.end(), rows_be + (size_t)y * stride, rows_be + (size_t)(y + 1) * stride);
  }
  uLongf zn = compressBound((uLong)raw.size());
  std::vector<uint8_t> z(zn);
  if (compress2(z.data(), &zn, raw.data(), (uLong)raw.size(), 6) != Z_OK)
    return io_fail(VC_ERR_INVALID_ARGUMENT, "png write error", path);
  z.resize(zn);
  std::vector<uint8_t> out(kSig, kSig + 8);
  auto chunk = [&](const char* type, const uint8_t* data, uint32_t len) {
    put_be32(out, len);
    const size_t t0 = out.size();
    out.insert(out.end(), type, type + 4);
    out.insert(out.end(), data, data + len);
    put_be32(out, (uint32_t)crc32(0L, &out[t0], 4 + len));
  };
  uint8_t ihdr[13];
  const uint32_t W = (uint32_t)w, H = (uint32_t)h;
  const uint8_t hdr[13] = {(uint8_t)(W >> 24), (uint8_t)(W >> 16), (uint8_t)(W >> 8), (uint8_t)W,
                           (uint8_t)(H >> 24), (uint8_t)(H >> 16), (uint8_t)(H >> 8), (uint8_t)H,
                           (uint8_t)depth, (uint8_t)ctype, 0, 0, 0};
  std::memcpy(ihdr, hdr, 13);
  chunk("IHDR", ihdr, 13);
  chunk("IDAT", z.data(), (uint32_t)z.size());
  chunk("IEND", nullptr, 0);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail(VC_ERR_INVALID_ARGUMENT, "cannot open for writing", path);
  const size_t put = std::fwrite(out.data(), 1, out.size(), f);
  std::fclose(f);
  if (put != out.size()) return io_fail(VC_ERR_INVALID_ARGUMENT, "png write error", path);
  return VC_OK;
}

struct Channel {
  std::string name;
  int comps;
  const float* data;  // comps per vertex
};

// mesh_io.cpp:104-145 write_ply (binary little endian; float vertex data,
// uchar-count int32 faces, comment channel directory)
vc_status write_ply(const char* path, const float* xyz, const float* nrm, int nv, const int32_t* tris, int nt,
                    const std::vector<Channel>& chans) {
  std::string h = "ply\nformat binary_little_endian 1.0\n";
  h += "element vertex " + std::to_string(nv) + "\n";
  h += "property float x\nproperty float y\nproperty float z\n";
  if (nrm) h += "property float nx\nproperty float ny\nproperty float nz\n";
  for (const auto& c : chans)
    for (int k = 0; k < c.comps; ++k) h += "property float " + c.name + "_" + std::to_string(k) + "\n";
  h += "element face " + std::to_string(nt) + "\n";
  h += "property list uchar int vertex_indices\n";
  for (const auto& c : chans) h += "comment channel " + c.name + " " + std::to_string(c.comps) + "\n";
  h += "end_header\n";
  size_t per = 3 + (nrm ? 3 : 0);
  for (const auto& c : chans) per += c.comps;
  std::vector<uint8_t> body((size_t)nv * per * 4 + (size_t)nt * 13);
  uint8_t* o = body.data();
  for (int v = 0; v < nv; ++v) {
    std::memcpy(o, xyz + 3 * (size_t)v, 12), o += 12;
    if (nrm) std::memcpy(o, nrm + 3 * (size_t)v, 12), o += 12;
    for (const auto& c : chans) std::memcpy(o, c.data + (size_t)v * c.comps, 4 * c.comps), o += 4 * c.comps;
  }
  for (int t = 0; t < nt; ++t) {
    *o++ = 3;
    std::memcpy(o, tris + 3 * (size_t)t, 12), o += 12;
  }
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail(VC_ERR_INVALID_ARGUMENT, "cannot open for writing", path);
  bool ok = std::fwrite(h.data(), 1, h.size(), f) == h.size();
  ok = ok && std::fwrite(body.data(), 1, body.size(), f) == body.size();
  std::fclose(f);
  if (!ok) return io_fail(VC_ERR_INVALID_ARGUMENT, "ply write failed", path);
  return VC_OK;
}

}  // namespace

namespace vc_io_detail {
vc_status set_error(vc_status s, const std::string& msg) {  // context-free entry points' last error
  g_io_err = msg;
  return s;
}
}  // namespace vc_io_detail

extern "C" {

const char* vc_io_last_error(void) { return g_io_err.c_str(); }

vc_status vc_png_info(const char* path, vc_png_header* info) {
  if (!path || !info) return io_fail(VC_ERR_INVALID_ARGUMENT, "null argument", path);
  Png p;
  const vc_status s = parse_png(path, p);
  if (s != VC_OK) return s;
  info->width = p.w, info->height = p.h, info->bit_depth = p.depth, info->color_type = p.ctype;
  return VC_OK;
}

// image_io.cpp:105-122 read_depth_png: 16-bit grayscale only, host-endian
vc_status vc_png_read_depth(const char* path, uint16_t* dst, int32_t width, int32_t height) {
  if (!path || !dst) return io_fail(VC_ERR_INVALID_ARGUMENT, "null argument", path);
  Png p;
  vc_status s = parse_png(path, p);
  if (s != VC_OK) return s;
  if (p.ctype != 0 || p.depth != 16) return io_fail(VC_ERR_INVALID_ARGUMENT, "depth png must be 16-bit grayscale", path);
  if (p.w != width || p.h != height) return io_fail(VC_ERR_INVALID_ARGUMENT, "png size mismatch", path);
  std::vector<uint8_t> rows;
  size_t stride;
  int bpp;
  if ((s = inflate_rows(path, p, rows, &stride, &bpp)) != VC_OK) return s;
  for (int y = 0; y < p.h; ++y)
    for (int x = 0; x < p.w; ++x) {
      const uint8_t* q = &rows[(size_t)y * stride + 2 * (size_t)x];
      dst[(size_t)y * p.w + x] = (uint16_t)(q[0] << 8 | q[1]);
    }
  return VC_OK;
}

// image_io.cpp:84-103 read_color_png: expand, strip_16, strip_alpha, gray_to_rgb
vc_status vc_png_read_color(const char* path, uint8_t* rgb, int32_t width, int32_t height) {
  if (!path || !rgb) return io_fail(VC_ERR_INVALID_ARGUMENT, "null argument", path);
  Png p;
  vc_status s = parse_png(path, p);
  if (s != VC_OK) return s;
  if (p.w != width || p.h != height) return io_fail(VC_ERR_INVALID_ARGUMENT, "png size mismatch", path);
  std::vector<uint8_t> rows;
  size_t stride;
  int bpp;
  if ((s = inflate_rows(path, p, rows, &stride, &bpp)) != VC_OK) return s;
  const int ch = channels_of(p.ctype);
  for (int y = 0; y < p.h; ++y) {
    const uint8_t* r = &rows[(size_t)y * stride];
    uint8_t* o = rgb + (size_t)y * p.w * 3;
    for (int x = 0; x < p.w; ++x) {
      if (p.ctype == 3) {
        const int i = sample8(r, (size_t)x, p.depth, true);
        if ((size_t)(3 * i + 2) >= p.plte.size()) return io_fail(VC_ERR_INVALID_ARGUMENT, "png read error", path);
        o[3 * x] = p.plte[3 * i], o[3 * x + 1] = p.plte[3 * i + 1], o[3 * x + 2] = p.plte[3 * i + 2];
      } else if (ch <= 2) {  // gray (+ alpha): the gray sample replicated
        const uint8_t g = (uint8_t)sample8(r, (size_t)x * ch, p.depth, false);
        o[3 * x] = o[3 * x + 1] = o[3 * x + 2] = g;
      } else {  // RGB / RGBA
        for (int c = 0; c < 3; ++c) o[3 * x + c] = (uint8_t)sample8(r, (size_t)x * ch + c, p.depth, false);
      }
    }
  }
  return VC_OK;
}

vc_status vc_png_write_depth(const char* path, const uint16_t* src, int32_t width, int32_t height) {
  if (!path || !src || width <= 0 || height <= 0) return io_fail(VC_ERR_INVALID_ARGUMENT, "bad argument", path);
  std::vector<uint8_t> be((size_t)width * height * 2);
  for (size_t i = 0; i < (size_t)width * height; ++i) be[2 * i] = src[i] >> 8, be[2 * i + 1] = src[i] & 255;
  return write_png(path, width, height, 16, 0, be.data(), (size_t)width * 2);
}

vc_status vc_png_write_color(const char* path, const uint8_t* rgb, int32_t width, int32_t height) {
  if (!path || !rgb || width <= 0 || height <= 0) return io_fail(VC_ERR_INVALID_ARGUMENT, "bad argument", path);
  return write_png(path, width, height, 8, 2, rgb, (size_t)width * 3);
}

vc_status vc_ply_write_mesh(const char* path, const float* xyz, const float* normals, int32_t n_vertices,
                            const int32_t* triangles, int32_t n_triangles, const char* const* channel_names,
                            const int32_t* channel_components, const float* const* channel_data,
                            int32_t n_channels) {
  if (!path || (n_vertices > 0 && !xyz) || (n_triangles > 0 && !triangles) || n_vertices < 0 || n_triangles < 0 ||
      n_channels < 0)
    return io_fail(VC_ERR_INVALID_ARGUMENT, "bad argument", path);
  std::vector<Channel> ch;
  for (int i = 0; i < n_channels; ++i) {
    if (!channel_names || !channel_names[i] || !channel_components || channel_components[i] < 1 || !channel_data ||
        (n_vertices > 0 && !channel_data[i]))
      return io_fail(VC_ERR_INVALID_ARGUMENT, "bad channel", path);
    ch.push_back({channel_names[i], channel_components[i], channel_data[i]});
  }
  return write_ply(path, xyz, normals, n_vertices, triangles, n_triangles, ch);
}

// write_ply(mesh.with_channels()) of the reference CLI (volcap.cpp:312-316):
// cam<k>_vis, cam<k>_uv, cam<k>_w per sensor, then untextured, as floats
vc_status vc_ply_write_textured(const char* path, const vc_textured_mesh* m) {
  if (!path || !m) return io_fail(VC_ERR_INVALID_ARGUMENT, "null argument", path);
  if (m->mem_kind != VC_MEM_HOST) return io_fail(VC_ERR_INVALID_ARGUMENT, "textured mesh must be in host memory", path);
  const int V = m->vertex_count, K = m->sensor_count;
  std::vector<float> xyz(3 * (size_t)V);
  for (size_t i = 0; i < 3 * (size_t)V; ++i) xyz[i] = m->positions_f64 ? (float)m->positions_f64[i] : m->positions[i];
  std::vector<std::vector<float>> store;
  std::vector<Channel> ch;
  store.reserve(3 * (size_t)K + 1);
  for (int k = 0; k < K; ++k) {
    std::vector<float> vis(V), uv(2 * (size_t)V), w(V);
    for (int v = 0; v < V; ++v) {
      vis[v] = (float)m->visible[(size_t)k * V + v];
      uv[2 * (size_t)v] = m->uv[2 * ((size_t)k * V + v)];
      uv[2 * (size_t)v + 1] = m->uv[2 * ((size_t)k * V + v) + 1];
      w[v] = m->weight[(size_t)k * V + v];
    }
    store.push_back(std::move(vis));
    ch.push_back({"cam" + std::to_string(k) + "_vis", 1, store.back().data()});
    store.push_back(std::move(uv));
    ch.push_back({"cam" + std::to_string(k) + "_uv", 2, store.back().data()});
    store.push_back(std::move(w));
    ch.push_back({"cam" + std::to_string(k) + "_w", 1, store.back().data()});
  }
  std::vector<float> un(V);
  for (int v = 0; v < V; ++v) un[v] = (float)m->untextured[v];
  store.push_back(std::move(un));
  ch.push_back({"untextured", 1, store.back().data()});
  return write_ply(path, xyz.data(), m->normals, V, m->triangles, m->triangle_count, ch);
}

}  // extern "C"
