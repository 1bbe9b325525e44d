// io.cpp -- the reference's on-disk tensor format (blob.cpp:29-79,
// SPEC.md:87): four unsigned 64-bit little-endian dims (H, W, C, N), then
// H*W*C*N little-endian IEEE-754 float32 values in flat (height-fastest)
// order.  Host-only; the graph manifest and the trainer checkpoint
// (engine.cu) are built on these.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ck/ck.h"
#include "ck_io.hpp"

namespace ck {

thread_local std::string g_io_err;

static_assert(sizeof(float) == 4, "IEEE-754 float32 required");

static bool little_endian() {
  const uint16_t v = 1;
  uint8_t b;
  std::memcpy(&b, &v, 1);
  return b == 1;
}

static uint64_t le64(uint64_t v) {
  if (little_endian()) return v;
  uint64_t r = 0;
  for (int k = 0; k < 8; ++k) r |= ((v >> (8 * k)) & 0xffULL) << (8 * (7 - k));
  return r;
}

static uint32_t le32(uint32_t v) {
  if (little_endian()) return v;
  return ((v & 0xffu) << 24) | ((v & 0xff00u) << 8) | ((v >> 8) & 0xff00u) | (v >> 24);
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

// blob.cpp:29-51 write_blob
void blob_write(const std::string& path, const float* data, const ck_shape& s) {
  File f;
  f.f = fopen(path.c_str(), "wb");
  if (!f.f) throw IoError("cannot open " + path + " for writing");
  const uint64_t dims[4] = {le64((uint64_t)s.h), le64((uint64_t)s.w), le64((uint64_t)s.c),
                            le64((uint64_t)s.n)};
  bool ok = fwrite(dims, 8, 4, f.f) == 4;
  const int64_t n = s.h * s.w * s.c * s.n;
  if (little_endian()) {
    ok = ok && (int64_t)fwrite(data, 4, (size_t)n, f.f) == n;
  } else {
    for (int64_t k = 0; ok && k < n; ++k) {
      uint32_t b;
      std::memcpy(&b, data + k, 4);
      b = le32(b);
      ok = fwrite(&b, 4, 1, f.f) == 1;
    }
  }
  ok = ok && fflush(f.f) == 0;
  if (!ok) throw IoError("blob write failed");
}

// blob.cpp:53-74 read_blob: header first (shape only when data is null)
ck_shape blob_read(const std::string& path, float* data, const ck_shape* expect) {
  File f;
  f.f = fopen(path.c_str(), "rb");
  if (!f.f) throw IoError("cannot open " + path);
  uint64_t dims[4];
  if (fread(dims, 8, 4, f.f) != 4) throw IoError("truncated blob header in " + path);
  ck_shape s{(int64_t)le64(dims[0]), (int64_t)le64(dims[1]), (int64_t)le64(dims[2]),
             (int64_t)le64(dims[3])};
  const std::string ss = std::to_string(s.h) + "x" + std::to_string(s.w) + "x" +
                         std::to_string(s.c) + "x" + std::to_string(s.n);
  if (s.h < 1 || s.w < 1 || s.c < 1 || s.n < 1 || (double)s.h * s.w * s.c * s.n > (double)(1LL << 34))
    throw IoError("bad blob dimensions in " + path + ": " + ss);
  if (expect && (expect->h != s.h || expect->w != s.w || expect->c != s.c || expect->n != s.n))
    throw IoError("blob " + path + " has shape " + ss + ", expected " +
                  std::to_string(expect->h) + "x" + std::to_string(expect->w) + "x" +
                  std::to_string(expect->c) + "x" + std::to_string(expect->n));
  if (!data) return s;
  const int64_t n = s.h * s.w * s.c * s.n;
  if ((int64_t)fread(data, 4, (size_t)n, f.f) != n) throw IoError("truncated blob data in " + path);
  if (!little_endian())
    for (int64_t k = 0; k < n; ++k) {
      uint32_t b;
      std::memcpy(&b, data + k, 4);
      b = le32(b);
      std::memcpy(data + k, &b, 4);
    }
  return s;
}

}  // namespace ck

using namespace ck;

extern "C" {

const char* ck_io_last_error(void) { return g_io_err.c_str(); }

ck_status ck_blob_write(const char* path, const float* data, ck_shape shape) {
  try {
    if (!path || !data) throw IoError("null argument");
    if (shape.h < 1 || shape.w < 1 || shape.c < 1 || shape.n < 1)
      throw IoError("invalid tensor shape");
    blob_write(path, data, shape);
    return CK_OK;
  } catch (const IoError& e) {
    g_io_err = e.what();
    return CK_ERR_DATA;
  }
}

ck_status ck_blob_read_shape(const char* path, ck_shape* shape) {
  try {
    if (!path || !shape) throw IoError("null argument");
    *shape = blob_read(path, nullptr, nullptr);
    return CK_OK;
  } catch (const IoError& e) {
    g_io_err = e.what();
    return CK_ERR_DATA;
  }
}

ck_status ck_blob_read(const char* path, float* data, ck_shape expect) {
  try {
    if (!path || !data) throw IoError("null argument");
    blob_read(path, data, &expect);
    return CK_OK;
  } catch (const IoError& e) {
    g_io_err = e.what();
    return CK_ERR_DATA;
  }
}

// SPEC.md:721-728 load_idx: IDX files (magic 0x00000803 images /
// 0x00000801 labels, big-endian dims, unsigned bytes).  Images become
// H x W x 1 x N singles scaled to [0, 1]; labels become 1..C (raw + 1, 0 is
// the ignore code).  out == NULL: only the dims (dims[0..3] = H, W, 1, N for
// images; 1, 1, 1, N for labels).
ck_status ck_idx_read(const char* path, float* out, int64_t dims[4]) {
  try {
    if (!path || !dims) throw IoError("null argument");
    File f;
    f.f = fopen(path, "rb");
    if (!f.f) throw IoError(std::string("cannot open ") + path);
    unsigned char hdr[4];
    if (fread(hdr, 1, 4, f.f) != 4) throw IoError(std::string("truncated IDX header in ") + path);
    const uint32_t magic = (uint32_t)hdr[0] << 24 | (uint32_t)hdr[1] << 16 | (uint32_t)hdr[2] << 8 | hdr[3];
    if (magic != 0x00000803u && magic != 0x00000801u)
      throw IoError(std::string("bad IDX magic in ") + path);
    const int nd = magic == 0x00000803u ? 3 : 1;
    uint32_t d[3] = {1, 1, 1};
    for (int k = 0; k < nd; ++k) {
      if (fread(hdr, 1, 4, f.f) != 4) throw IoError(std::string("truncated IDX header in ") + path);
      d[k] = (uint32_t)hdr[0] << 24 | (uint32_t)hdr[1] << 16 | (uint32_t)hdr[2] << 8 | hdr[3];
    }
    const int64_t n = d[0];
    // IDX image bytes are row-major (row r, column c): H = rows along i, W = columns
    const int64_t rows = nd == 3 ? d[1] : 1, cols = nd == 3 ? d[2] : 1;
    dims[0] = rows;
    dims[1] = cols;
    dims[2] = 1;
    dims[3] = n;
    if (!out) return CK_OK;
    std::vector<unsigned char> buf((size_t)(n * rows * cols));
    if (fread(buf.data(), 1, buf.size(), f.f) != buf.size())
      throw IoError(std::string("truncated IDX data in ") + path);
    if (nd == 1) {
      for (int64_t k = 0; k < n; ++k) out[k] = (float)buf[k] + 1.0f;
    } else {
      for (int64_t m = 0; m < n; ++m)
        for (int64_t r = 0; r < rows; ++r)
          for (int64_t c = 0; c < cols; ++c)  // HWCN: i = row, j = column
            out[r + rows * (c + cols * m)] = (float)buf[(m * rows + r) * cols + c] / 255.0f;
    }
    return CK_OK;
  } catch (const IoError& e) {
    g_io_err = e.what();
    return CK_ERR_DATA;
  }
}

}  // extern "C"
