// convkit.hpp -- the reference's C++ block API (namespace convkit,
// /root/reference/proj/include/convkit/*.hpp) over device tensors, header-only
// on top of the C ABI in ck.h.
//
// A caller of convkit::conv_forward(x, f, &b, g) switches to
// ck::convkit::conv_forward(x, f, &b, g) with DeviceTensor arguments: same
// names, argument order, shape laws, null-means-skip outputs and exception
// classes (ShapeError / DataError / NumericError, error.hpp:9-24).  Returned
// tensors are freshly allocated as in the reference; the *_into variants of
// ck.h avoid the allocation.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ck/ck.h"

namespace ck {
namespace convkit {

// error.hpp:9-24
struct ShapeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// tensor.hpp:13-32
struct Shape {
  int64_t h = 1, w = 1, c = 1, n = 1;
  Shape() = default;
  Shape(int64_t h_, int64_t w_ = 1, int64_t c_ = 1, int64_t n_ = 1) : h(h_), w(w_), c(c_), n(n_) {}
  int64_t elems() const { return h * w * c * n; }
  bool operator==(const Shape& o) const { return h == o.h && w == o.w && c == o.c && n == o.n; }
  ck_shape c_shape() const { return ck_shape{h, w, c, n}; }
};

using ConvGeom = ck_conv_geom;            // conv.hpp:9-17 (same field order)
using ConvTransposeGeom = ck_convt_geom;  // conv.hpp:21-28
using PoolGeom = ck_pool_geom;            // pool.hpp:13-23
using LrnParams = ck_lrn_params;          // normalize.hpp:11-16
using SpnormParams = ck_spnorm_params;    // normalize.hpp:59-64

// loss.hpp:13-24 (same order as convkit::LossKind)
enum class LossKind : int {
  classerror = CK_LOSS_CLASSERROR,
  topk = CK_LOSS_TOPK,
  log = CK_LOSS_LOG,
  softmaxlog = CK_LOSS_SOFTMAXLOG,
  mhinge = CK_LOSS_MHINGE,
  mshinge = CK_LOSS_MSHINGE,
  binaryerror = CK_LOSS_BINARYERROR,
  binarylog = CK_LOSS_BINARYLOG,
  logistic = CK_LOSS_LOGISTIC,
  hinge = CK_LOSS_HINGE,
};

// loss.hpp:31-36
struct LossOptions {
  int64_t top_k = 5;
  double threshold = 0.0;
  bool random_ties = false;
  uint64_t tie_seed = 0;
  ck_loss_options c() const {
    return ck_loss_options{top_k, threshold, random_ties ? 1 : 0, tie_seed};
  }
};

// normalize.hpp:27-31: per-channel batch mean and (biased) variance
template <class T>
struct BnormMoments {
  std::vector<T> mean;
  std::vector<T> var;
};

inline ConvGeom conv_geom() { return ConvGeom{1, 1, 0, 0, 0, 0, 1}; }

// One handle + stream per host thread (ck.h threading rules).
class Context {
 public:
  explicit Context(int device = 0, cudaStream_t stream = nullptr, ck_math math = CK_MATH_TF32)
      : stream_(stream), math_(math) {
    if (ck_create(&h_, device) != CK_OK) throw CudaError("ck_create failed");
  }
  ~Context() { ck_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ck_handle* handle() const { return h_; }
  cudaStream_t stream() const { return stream_; }
  ck_math math() const { return math_; }
  void set_math(ck_math m) { math_ = m; }
  void check(ck_status s) const {
    if (s == CK_OK) return;
    std::string msg = ck_last_error(h_);
    switch (s) {
      case CK_ERR_SHAPE: throw ShapeError(msg);
      case CK_ERR_DATA: throw DataError(msg);
      case CK_ERR_NUMERIC: throw NumericError(msg);
      default: throw CudaError(msg);
    }
  }
  static Context& current() {
    thread_local Context ctx;
    return ctx;
  }

 private:
  ck_handle* h_ = nullptr;
  cudaStream_t stream_;
  ck_math math_;
};

// Device-resident HWCN fp32 tensor (the reference Tensor<float>, tensor.hpp:36-95).
class DeviceTensor {
 public:
  DeviceTensor() = default;
  explicit DeviceTensor(Shape s) : shape_(s) {
    if (cudaMalloc(&data_, sizeof(float) * (size_t)s.elems()) != cudaSuccess)
      throw CudaError("cudaMalloc failed");
    cudaMemset(data_, 0, sizeof(float) * (size_t)s.elems());  // reference ctor zero-fills
  }
  DeviceTensor(Shape s, const std::vector<float>& host) : DeviceTensor(s) {
    if ((int64_t)host.size() != s.elems()) throw ShapeError("tensor data length mismatch");
    cudaMemcpy(data_, host.data(), sizeof(float) * host.size(), cudaMemcpyHostToDevice);
  }
  ~DeviceTensor() {
    if (data_) cudaFree(data_);
  }
  DeviceTensor(DeviceTensor&& o) noexcept : shape_(o.shape_), data_(std::exchange(o.data_, nullptr)) {}
  DeviceTensor& operator=(DeviceTensor&& o) noexcept {
    if (this != &o) {
      if (data_) cudaFree(data_);
      shape_ = o.shape_;
      data_ = std::exchange(o.data_, nullptr);
    }
    return *this;
  }
  const Shape& shape() const { return shape_; }
  float* data() const { return data_; }
  ck_tensor view() const { return ck_tensor{data_, shape_.c_shape()}; }
  std::vector<float> to_host() const {
    std::vector<float> out((size_t)shape_.elems());
    cudaMemcpy(out.data(), data_, sizeof(float) * out.size(), cudaMemcpyDeviceToHost);
    return out;
  }

 private:
  Shape shape_{1, 1, 1, 1};
  float* data_ = nullptr;
};

inline Shape from_c(const ck_shape& s) { return Shape(s.h, s.w, s.c, s.n); }

// ---- shape laws (conv.cpp:108-154, pool.cpp:35-46) --------------------------
inline Shape conv_output_shape(const Shape& x, const Shape& f, const ConvGeom& g) {
  Context& c = Context::current();
  ck_shape o;
  c.check(ck_conv_output_shape(c.handle(), x.c_shape(), f.c_shape(), &g, &o));
  return from_c(o);
}
inline Shape convt_output_shape(const Shape& x, const Shape& f, const ConvTransposeGeom& g) {
  Context& c = Context::current();
  ck_shape o;
  c.check(ck_convt_output_shape(c.handle(), x.c_shape(), f.c_shape(), &g, &o));
  return from_c(o);
}
inline Shape pool_output_shape(const Shape& x, const PoolGeom& g) {
  Context& c = Context::current();
  ck_shape o;
  c.check(ck_pool_output_shape(c.handle(), x.c_shape(), &g, &o));
  return from_c(o);
}

// ---- vl_nnconv / vl_nnconvt (conv.hpp:60-81) --------------------------------
inline DeviceTensor conv_forward(const DeviceTensor& x, const DeviceTensor& f,
                                 const DeviceTensor* bias, const ConvGeom& g) {
  Context& c = Context::current();
  DeviceTensor y(conv_output_shape(x.shape(), f.shape(), g));
  ck_tensor xv = x.view(), fv = f.view(), yv = y.view(), bv;
  if (bias) bv = bias->view();
  c.check(ck_conv_forward(c.handle(), &xv, &fv, bias ? &bv : nullptr, &g, &yv, c.math(), c.stream()));
  return y;
}

inline void conv_backward(const DeviceTensor& x, const DeviceTensor& f, const ConvGeom& g,
                          const DeviceTensor& dy, DeviceTensor* dx, DeviceTensor* df,
                          DeviceTensor* db) {
  Context& c = Context::current();
  if (dx) *dx = DeviceTensor(x.shape());
  if (df) *df = DeviceTensor(f.shape());
  if (db) *db = DeviceTensor(Shape(1, 1, f.shape().n, 1));
  ck_tensor xv = x.view(), fv = f.view(), dyv = dy.view(), dxv, dfv, dbv;
  if (dx) dxv = dx->view();
  if (df) dfv = df->view();
  if (db) dbv = db->view();
  c.check(ck_conv_backward(c.handle(), &xv, &fv, &g, &dyv, dx ? &dxv : nullptr,
                           df ? &dfv : nullptr, db ? &dbv : nullptr, 0, c.math(), c.stream()));
}

inline DeviceTensor convt_forward(const DeviceTensor& x, const DeviceTensor& f,
                                  const ConvTransposeGeom& g) {
  Context& c = Context::current();
  DeviceTensor y(convt_output_shape(x.shape(), f.shape(), g));
  ck_tensor xv = x.view(), fv = f.view(), yv = y.view();
  c.check(ck_convt_forward(c.handle(), &xv, &fv, &g, &yv, c.math(), c.stream()));
  return y;
}

inline void convt_backward(const DeviceTensor& x, const DeviceTensor& f,
                           const ConvTransposeGeom& g, const DeviceTensor& dy, DeviceTensor* dx,
                           DeviceTensor* df) {
  Context& c = Context::current();
  if (dx) *dx = DeviceTensor(x.shape());
  if (df) *df = DeviceTensor(f.shape());
  ck_tensor xv = x.view(), fv = f.view(), dyv = dy.view(), dxv, dfv;
  if (dx) dxv = dx->view();
  if (df) dfv = df->view();
  c.check(ck_convt_backward(c.handle(), &xv, &fv, &g, &dyv, dx ? &dxv : nullptr,
                            df ? &dfv : nullptr, 0, c.math(), c.stream()));
}

// ---- vl_nnpool (pool.hpp:27-34) -----------------------------------------------
inline DeviceTensor pool_forward(const DeviceTensor& x, const PoolGeom& g) {
  Context& c = Context::current();
  DeviceTensor y(pool_output_shape(x.shape(), g));
  ck_tensor xv = x.view(), yv = y.view();
  c.check(ck_pool_forward(c.handle(), &xv, &g, &yv, c.stream()));
  return y;
}
inline DeviceTensor pool_backward(const DeviceTensor& x, const PoolGeom& g,
                                  const DeviceTensor& dy) {
  Context& c = Context::current();
  DeviceTensor dx(x.shape());
  ck_tensor xv = x.view(), dyv = dy.view(), dxv = dx.view();
  c.check(ck_pool_backward(c.handle(), &xv, &g, &dyv, &dxv, 0, c.stream()));
  return dx;
}

// ---- vl_nnrelu (activation.hpp:7-12) -----------------------------------------
inline DeviceTensor relu_forward(const DeviceTensor& x) {
  Context& c = Context::current();
  DeviceTensor y(x.shape());
  ck_tensor xv = x.view(), yv = y.view();
  c.check(ck_relu_forward(c.handle(), &xv, &yv, c.stream()));
  return y;
}
inline DeviceTensor relu_backward(const DeviceTensor& x, const DeviceTensor& dy) {
  Context& c = Context::current();
  DeviceTensor dx(x.shape());
  ck_tensor xv = x.view(), dyv = dy.view(), dxv = dx.view();
  c.check(ck_relu_backward(c.handle(), &xv, &dyv, &dxv, 0, c.stream()));
  return dx;
}

// ---- vl_nnnormalize / vl_nnbnorm (normalize.hpp:18-49) ----------------------
inline DeviceTensor lrn_forward(const DeviceTensor& x, const LrnParams& p) {
  Context& c = Context::current();
  DeviceTensor y(x.shape());
  ck_tensor xv = x.view(), yv = y.view();
  c.check(ck_lrn_forward(c.handle(), &xv, &p, &yv, c.stream()));
  return y;
}
inline DeviceTensor lrn_backward(const DeviceTensor& x, const LrnParams& p,
                                 const DeviceTensor& dy) {
  Context& c = Context::current();
  DeviceTensor dx(x.shape());
  ck_tensor xv = x.view(), dyv = dy.view(), dxv = dx.view();
  c.check(ck_lrn_backward(c.handle(), &xv, &p, &dyv, &dxv, 0, c.stream()));
  return dx;
}

// moments: K x 2 (mean column, variance column), graph.cpp:259-266
inline DeviceTensor bnorm_forward(const DeviceTensor& x, const DeviceTensor& w,
                                  const DeviceTensor& b, double epsilon,
                                  DeviceTensor* moments) {
  Context& c = Context::current();
  DeviceTensor y(x.shape());
  if (moments) *moments = DeviceTensor(Shape(x.shape().c, 2, 1, 1));
  ck_tensor xv = x.view(), wv = w.view(), bv = b.view(), yv = y.view(), mv;
  if (moments) mv = moments->view();
  c.check(ck_bnorm_forward(c.handle(), &xv, &wv, &bv, epsilon, &yv, moments ? &mv : nullptr,
                           c.stream()));
  return y;
}
inline DeviceTensor bnorm_infer(const DeviceTensor& x, const DeviceTensor& w,
                                const DeviceTensor& b, double epsilon,
                                const DeviceTensor& moments) {
  Context& c = Context::current();
  DeviceTensor y(x.shape());
  ck_tensor xv = x.view(), wv = w.view(), bv = b.view(), mv = moments.view(), yv = y.view();
  c.check(ck_bnorm_infer(c.handle(), &xv, &wv, &bv, epsilon, &mv, &yv, c.stream()));
  return y;
}
// normalize.hpp:35-38 with the reference's BnormMoments<T>* (host vectors)
inline DeviceTensor bnorm_forward(const DeviceTensor& x, const DeviceTensor& w,
                                  const DeviceTensor& b, double epsilon,
                                  BnormMoments<float>* moments = nullptr) {
  if (!moments) return bnorm_forward(x, w, b, epsilon, (DeviceTensor*)nullptr);
  DeviceTensor m;
  DeviceTensor y = bnorm_forward(x, w, b, epsilon, &m);
  std::vector<float> h = m.to_host();
  const size_t K = (size_t)x.shape().c;
  moments->mean.assign(h.begin(), h.begin() + K);
  moments->var.assign(h.begin() + K, h.end());
  return y;
}
// normalize.hpp:41-44 with BnormMoments<T>
inline DeviceTensor bnorm_infer(const DeviceTensor& x, const DeviceTensor& w,
                                const DeviceTensor& b, double epsilon,
                                const BnormMoments<float>& moments) {
  std::vector<float> h(moments.mean);
  h.insert(h.end(), moments.var.begin(), moments.var.end());
  DeviceTensor m(Shape((int64_t)moments.mean.size(), 2, 1, 1), h);
  return bnorm_infer(x, w, b, epsilon, m);
}
inline void bnorm_backward(const DeviceTensor& x, const DeviceTensor& w, const DeviceTensor& b,
                           double epsilon, const DeviceTensor& dy, DeviceTensor* dx,
                           DeviceTensor* dw, DeviceTensor* db) {
  Context& c = Context::current();
  if (dx) *dx = DeviceTensor(x.shape());
  if (dw) *dw = DeviceTensor(w.shape());
  if (db) *db = DeviceTensor(b.shape());
  ck_tensor xv = x.view(), wv = w.view(), bv = b.view(), dyv = dy.view(), dxv, dwv, dbv;
  if (dx) dxv = dx->view();
  if (dw) dwv = dw->view();
  if (db) dbv = db->view();
  c.check(ck_bnorm_backward(c.handle(), &xv, &wv, &bv, epsilon, &dyv, dx ? &dxv : nullptr,
                            dw ? &dwv : nullptr, db ? &dbv : nullptr, 0, c.stream()));
}

// ---- vl_nnsoftmaxloss, kind softmaxlog (loss.hpp:39-49) ---------------------
inline float softmaxlog_forward(const DeviceTensor& x, const DeviceTensor& labels,
                                const DeviceTensor* weights = nullptr) {
  Context& c = Context::current();
  DeviceTensor out(Shape(1, 1, 1, 1));
  ck_tensor xv = x.view(), lv = labels.view(), wv;
  if (weights) wv = weights->view();
  c.check(ck_softmaxlog_forward(c.handle(), &xv, &lv, weights ? &wv : nullptr, out.data(), 1,
                                c.stream()));
  return out.to_host()[0];
}
inline DeviceTensor softmaxlog_backward(const DeviceTensor& x, const DeviceTensor& labels,
                                        const DeviceTensor* weights, float p) {
  Context& c = Context::current();
  DeviceTensor dx(x.shape());
  ck_tensor xv = x.view(), lv = labels.view(), wv, dxv = dx.view();
  if (weights) wv = weights->view();
  c.check(ck_softmaxlog_backward(c.handle(), &xv, &lv, weights ? &wv : nullptr, p, &dxv, 0,
                                 c.stream()));
  return dx;
}


// ---- loss.hpp:39-49: every LossKind ----------------------------------------
// loss_forward: the weighted sum of per-sample penalties (a host scalar, as in
// the reference); label / domain errors raise DataError with its messages.
inline float loss_forward(const DeviceTensor& x, const DeviceTensor& labels, LossKind kind,
                          const DeviceTensor* weights = nullptr, const LossOptions& opts = {}) {
  Context& c = Context::current();
  DeviceTensor out(Shape(1, 1, 1, 1));
  ck_tensor xv = x.view(), lv = labels.view(), wv;
  if (weights) wv = weights->view();
  const ck_loss_options o = opts.c();
  c.check(ck_loss_forward(c.handle(), &xv, &lv, weights ? &wv : nullptr, (ck_loss_kind)kind, &o,
                          out.data(), 1, c.stream()));
  return out.to_host()[0];
}
// loss_backward: projected derivative (p = the scalar projection); error
// kinds return exact zeros (loss.cpp:239)
inline DeviceTensor loss_backward(const DeviceTensor& x, const DeviceTensor& labels,
                                  LossKind kind, const DeviceTensor* weights, float p,
                                  const LossOptions& opts = {}) {
  Context& c = Context::current();
  DeviceTensor dx(x.shape());
  ck_tensor xv = x.view(), lv = labels.view(), wv, dxv = dx.view();
  if (weights) wv = weights->view();
  const ck_loss_options o = opts.c();
  c.check(ck_loss_backward(c.handle(), &xv, &lv, weights ? &wv : nullptr, (ck_loss_kind)kind, &o,
                           p, &dxv, 0, c.stream()));
  return dx;
}
// loss.hpp:52-63 pdist
inline DeviceTensor pdist_forward(const DeviceTensor& x, const DeviceTensor& target, double p,
                                  bool no_root) {
  Context& c = Context::current();
  DeviceTensor y(Shape(x.shape().h, x.shape().w, 1, x.shape().n));
  ck_tensor xv = x.view(), tv = target.view(), yv = y.view();
  c.check(ck_pdist_forward(c.handle(), &xv, &tv, p, no_root ? 1 : 0, &yv, c.stream()));
  return y;
}
inline void pdist_backward(const DeviceTensor& x, const DeviceTensor& target, double p,
                           bool no_root, const DeviceTensor& dy, DeviceTensor* dx,
                           DeviceTensor* dtarget) {
  Context& c = Context::current();
  if (dx) *dx = DeviceTensor(x.shape());
  if (dtarget) *dtarget = DeviceTensor(x.shape());
  ck_tensor xv = x.view(), tv = target.view(), dyv = dy.view(), dxv, dtv;
  if (dx) dxv = dx->view();
  if (dtarget) dtv = dtarget->view();
  c.check(ck_pdist_backward(c.handle(), &xv, &tv, p, no_root ? 1 : 0, &dyv, dx ? &dxv : nullptr,
                            dtarget ? &dtv : nullptr, 0, c.stream()));
}

// ---- activation.hpp:14-19 sigmoid; normalize.hpp:66-76 softmax, spnorm ------
inline DeviceTensor sigmoid_forward(const DeviceTensor& x) {
  Context& c = Context::current();
  DeviceTensor y(x.shape());
  ck_tensor xv = x.view(), yv = y.view();
  c.check(ck_sigmoid_forward(c.handle(), &xv, &yv, c.stream()));
  return y;
}
inline DeviceTensor sigmoid_backward(const DeviceTensor& y, const DeviceTensor& dy) {
  Context& c = Context::current();
  DeviceTensor dx(y.shape());
  ck_tensor yv = y.view(), dyv = dy.view(), dxv = dx.view();
  c.check(ck_sigmoid_backward(c.handle(), &yv, &dyv, &dxv, 0, c.stream()));
  return dx;
}
inline DeviceTensor softmax_forward(const DeviceTensor& x) {
  Context& c = Context::current();
  DeviceTensor y(x.shape());
  ck_tensor xv = x.view(), yv = y.view();
  c.check(ck_softmax_forward(c.handle(), &xv, &yv, c.stream()));
  return y;
}
inline DeviceTensor softmax_backward(const DeviceTensor& y, const DeviceTensor& dy) {
  Context& c = Context::current();
  DeviceTensor dx(y.shape());
  ck_tensor yv = y.view(), dyv = dy.view(), dxv = dx.view();
  c.check(ck_softmax_backward(c.handle(), &yv, &dyv, &dxv, 0, c.stream()));
  return dx;
}
inline DeviceTensor spnorm_forward(const DeviceTensor& x, const SpnormParams& p) {
  Context& c = Context::current();
  DeviceTensor y(x.shape());
  ck_tensor xv = x.view(), yv = y.view();
  c.check(ck_spnorm_forward(c.handle(), &xv, &p, &yv, c.stream()));
  return y;
}
inline DeviceTensor spnorm_backward(const DeviceTensor& x, const SpnormParams& p,
                                   const DeviceTensor& dy) {
  Context& c = Context::current();
  DeviceTensor dx(x.shape());
  ck_tensor xv = x.view(), dyv = dy.view(), dxv = dx.view();
  c.check(ck_spnorm_backward(c.handle(), &xv, &p, &dyv, &dxv, 0, c.stream()));
  return dx;
}

// ---- bilinear.hpp:13-22 ---------------------------------------------------
inline Shape bilinear_output_shape(const Shape& x, const Shape& grid) {
  Context& c = Context::current();
  ck_shape o;
  c.check(ck_bilinear_output_shape(c.handle(), x.c_shape(), grid.c_shape(), &o));
  return from_c(o);
}
inline DeviceTensor bilinear_forward(const DeviceTensor& x, const DeviceTensor& grid) {
  Context& c = Context::current();
  DeviceTensor y(bilinear_output_shape(x.shape(), grid.shape()));
  ck_tensor xv = x.view(), gv = grid.view(), yv = y.view();
  c.check(ck_bilinear_forward(c.handle(), &xv, &gv, &yv, c.stream()));
  return y;
}
inline void bilinear_backward(const DeviceTensor& x, const DeviceTensor& grid,
                              const DeviceTensor& dy, DeviceTensor* dx, DeviceTensor* dgrid) {
  Context& c = Context::current();
  if (dx) *dx = DeviceTensor(x.shape());
  if (dgrid) *dgrid = DeviceTensor(grid.shape());
  ck_tensor xv = x.view(), gv = grid.view(), dyv = dy.view(), dxv, dgv;
  if (dx) dxv = dx->view();
  if (dgrid) dgv = dgrid->view();
  c.check(ck_bilinear_backward(c.handle(), &xv, &gv, &dyv, dx ? &dxv : nullptr,
                               dgrid ? &dgv : nullptr, 0, c.stream()));
}

// ---- blob.hpp:11-18: the raw tensor blob <-> a device tensor ----------------
inline void write_blob(const DeviceTensor& t, const std::string& path) {
  std::vector<float> h = t.to_host();
  if (ck_blob_write(path.c_str(), h.data(), t.shape().c_shape()) != CK_OK)
    throw DataError(ck_io_last_error());
}
inline DeviceTensor read_blob(const std::string& path) {
  ck_shape s;
  if (ck_blob_read_shape(path.c_str(), &s) != CK_OK) throw DataError(ck_io_last_error());
  std::vector<float> h((size_t)(s.h * s.w * s.c * s.n));
  if (ck_blob_read(path.c_str(), h.data(), s) != CK_OK) throw DataError(ck_io_last_error());
  return DeviceTensor(from_c(s), h);
}

}  // namespace convkit
}  // namespace ck
