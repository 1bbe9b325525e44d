// Host-side file formats shared by io.cpp and engine.cu: the reference's raw
// tensor blob (blob.cpp:29-79) and the errors they raise (DataError).
#pragma once

#include <stdexcept>
#include <string>

#include "ck/ck.h"

namespace ck {

// convkit::DataError of blob.cpp / the manifest loader
struct IoError : std::runtime_error {
  explicit IoError(const std::string& m) : std::runtime_error(m) {}
};

extern thread_local std::string g_io_err;

void blob_write(const std::string& path, const float* host_data, const ck_shape& shape);
// Reads the header (and, if data != null, the values).  expect != null: the
// stored shape must equal it.
ck_shape blob_read(const std::string& path, float* host_data, const ck_shape* expect);

}  // namespace ck
