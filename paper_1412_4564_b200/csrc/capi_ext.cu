// capi_ext.cu -- extern "C" entry points of the rest of the reference block
// set (ck.h): sigmoid, channel softmax, spnorm, bilinear, pdist and every
// loss kind.  Each validates with the reference's rules and messages, then
// launches blocks_ext.cu kernels on the caller's stream.  Citations are to
// /root/reference/proj.
#include <cuda_runtime.h>

#include <string>

#include "ck/ck.h"
#include "ck_handle.hpp"
#include "ck_internal.hpp"

using ck::Err;
using namespace ck;

namespace ck {

// normalize.cpp:29-32 spnorm_pool_geom
static void check_spnorm(const ck_spnorm_params* p) {
  if (!p) throw Err(CK_ERR_ARG, "null spnorm parameters");
  if (p->window_h < 1 || p->window_w < 1) throw Err(CK_ERR_SHAPE, "spnorm window must be positive");
}

// bilinear.cpp:39-51 check_grid + bilinear_output_shape
ck_shape bilinear_output_shape(const ck_shape& xs, const ck_shape& gs) {
  if (gs.h != 2)
    throw Err(CK_ERR_SHAPE, "sampling grid must have two coordinate channels, got " + shape_str(gs));
  if (gs.n != xs.n)
    throw Err(CK_ERR_SHAPE, "sampling grid batch " + std::to_string(gs.n) +
                                " does not match input batch " + std::to_string(xs.n));
  return ck_shape{gs.w, gs.c, xs.c, xs.n};
}

// loss.cpp:349-353
ck_shape pdist_output_shape(const ck_shape& xs, const ck_shape& ts, double p) {
  if (!same(xs, ts))
    throw Err(CK_ERR_SHAPE, "pdist: shapes differ, " + shape_str(xs) + " vs " + shape_str(ts));
  if (!(p > 0)) throw Err(CK_ERR_SHAPE, "pdist exponent must be positive");
  return ck_shape{xs.h, xs.w, 1, xs.n};
}

// loss.cpp:44-53 loss_is_attribute
bool loss_is_attribute(int kind) { return kind >= CK_LOSS_BINARYERROR; }

// loss.cpp:89-94, :35-40, :184-186: weights, label shapes per kind
void check_loss_kind(const ck_tensor* x, const ck_tensor* labels, const ck_tensor* weights,
                     int kind) {
  if (kind < CK_LOSS_CLASSERROR || kind > CK_LOSS_HINGE) throw Err(CK_ERR_DATA, "unknown loss kind");
  check_tensor(x, "x");
  check_tensor(labels, "labels");
  const ck_shape &xs = x->shape, &cs = labels->shape;
  if (weights) {
    check_tensor(weights, "weights");
    if (!same(weights->shape, cs))
      throw Err(CK_ERR_SHAPE, "instance weights must match the label tensor shape");
  }
  if (!loss_is_attribute(kind)) {
    if (cs.h != xs.h || cs.w != xs.w || cs.c != 1 || cs.n != xs.n)
      throw Err(CK_ERR_SHAPE, "classification labels must be " +
                                  shape_str(ck_shape{xs.h, xs.w, 1, xs.n}) + ", got " +
                                  shape_str(cs));
  } else if (!same(cs, xs)) {
    throw Err(CK_ERR_SHAPE, "attribute labels must match the prediction shape");
  }
}

// Launch a loss forward of any kind into the device float `loss`; `site`
// scratch is taken from h->scratch.
void loss_forward_any(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                      const ck_tensor* weights, int kind, const ck_loss_options& o, float* loss,
                      cudaStream_t st) {
  const ck_shape& s = x->shape;
  const int64_t sites = loss_is_attribute(kind) ? elems(s) : s.h * s.w * s.n;
  float* site = (float*)h->scratch.get(sizeof(float) * (size_t)sites, st);
  if (!site) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  h->last_classes = s.c;
  if (kind == CK_LOSS_SOFTMAXLOG) {
    softmaxlog_forward(x->data, labels->data, weights ? weights->data : nullptr, site, loss,
                       h->flag, (int)(s.h * s.w), (int)s.c, (int)s.n, st);
  } else {
    loss_forward_kind(x->data, labels->data, weights ? weights->data : nullptr, kind, o.top_k,
                      o.threshold, (int)o.random_ties, o.tie_seed, site, loss, h->flag, (int)s.h,
                      (int)s.w, (int)s.c, (int)s.n, st);
  }
}

void loss_backward_any(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                       const ck_tensor* weights, int kind, float p, const float* p_dev,
                       float* dx, int acc, cudaStream_t st) {
  const ck_shape& s = x->shape;
  h->last_classes = s.c;
  if (kind == CK_LOSS_SOFTMAXLOG)
    softmaxlog_backward(x->data, labels->data, weights ? weights->data : nullptr, p, p_dev, dx,
                        h->flag, (int)(s.h * s.w), (int)s.c, (int)s.n, acc, st);
  else
    loss_backward_kind(x->data, labels->data, weights ? weights->data : nullptr, kind, p, p_dev,
                       dx, h->flag, (int)s.h, (int)s.w, (int)s.c, (int)s.n, acc, st);
}

ck_loss_options default_loss_options() { return ck_loss_options{5, 0.0, 0, 0}; }

}  // namespace ck

extern "C" {

ck_status ck_sigmoid_forward(ck_handle* h, const ck_tensor* x, ck_tensor* y, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_out(y, x->shape, "y");
  sigmoid_forward(x->data, y->data, elems(x->shape), (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_sigmoid_backward(ck_handle* h, const ck_tensor* y, const ck_tensor* dy, ck_tensor* dx,
                              int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(y, "y");
  check_tensor(dy, "dy");
  if (!same(dy->shape, y->shape))
    throw Err(CK_ERR_SHAPE, "sigmoid backward: projection shape mismatch");
  check_out(dx, y->shape, "dx");
  sigmoid_backward(y->data, dy->data, dx->data, elems(y->shape), accumulate, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_softmax_forward(ck_handle* h, const ck_tensor* x, ck_tensor* y, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_out(y, x->shape, "y");
  const ck_shape& s = x->shape;
  softmax_forward(x->data, y->data, (int)(s.h * s.w), (int)s.c, (int)s.n, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_softmax_backward(ck_handle* h, const ck_tensor* y, const ck_tensor* dy, ck_tensor* dx,
                              int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(y, "y");
  check_tensor(dy, "dy");
  if (!same(dy->shape, y->shape))
    throw Err(CK_ERR_SHAPE, "softmax backward: projection shape mismatch");
  check_out(dx, y->shape, "dx");
  const ck_shape& s = y->shape;
  softmax_backward(y->data, dy->data, dx->data, (int)(s.h * s.w), (int)s.c, (int)s.n, accumulate,
                   (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_spnorm_forward(ck_handle* h, const ck_tensor* x, const ck_spnorm_params* p,
                            ck_tensor* y, ck_stream stream) {
  CK_API_BEGIN(h)
  check_spnorm(p);
  check_tensor(x, "x");
  check_out(y, x->shape, "y");
  const ck_shape& s = x->shape;
  spnorm_forward(x->data, y->data, (int)s.h, (int)s.w, s.c * s.n, (int)p->window_h,
                 (int)p->window_w, (float)p->alpha, (float)p->beta, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_spnorm_backward(ck_handle* h, const ck_tensor* x, const ck_spnorm_params* p,
                             const ck_tensor* dy, ck_tensor* dx, int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_spnorm(p);
  check_tensor(x, "x");
  check_tensor(dy, "dy");
  if (!same(dy->shape, x->shape))
    throw Err(CK_ERR_SHAPE, "spnorm backward: projection shape mismatch");
  check_out(dx, x->shape, "dx");
  const ck_shape& s = x->shape;
  cudaStream_t st = (cudaStream_t)stream;
  float* ws = (float*)h->ws.get(2 * sizeof(float) * (size_t)elems(s), st);
  if (!ws) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  const float a = (float)p->alpha, b = (float)p->beta;
  const float c2ab = (2.0f * a) * b;  // T(2) * alpha * beta (normalize.cpp:302)
  spnorm_backward(x->data, dy->data, dx->data, ws, (int)s.h, (int)s.w, s.c * s.n,
                  (int)p->window_h, (int)p->window_w, a, b, c2ab, accumulate, st);
  after_launch();
  CK_API_END(h)
}

ck_status ck_bilinear_output_shape(ck_handle* h, ck_shape x, ck_shape grid, ck_shape* out) {
  CK_API_BEGIN(h)
  if (!out) throw Err(CK_ERR_ARG, "null output");
  *out = bilinear_output_shape(x, grid);
  CK_API_END(h)
}

ck_status ck_bilinear_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* grid,
                              ck_tensor* y, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(grid, "grid");
  const ck_shape ys = bilinear_output_shape(x->shape, grid->shape);
  check_out(y, ys, "y");
  const ck_shape& s = x->shape;
  bilinear_forward(x->data, grid->data, y->data, (int)s.h, (int)s.w, (int)s.c, (int)s.n,
                   (int)ys.h, (int)ys.w, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_bilinear_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* grid,
                               const ck_tensor* dy, ck_tensor* dx, ck_tensor* dgrid,
                               int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(grid, "grid");
  check_tensor(dy, "dy");
  const ck_shape ys = bilinear_output_shape(x->shape, grid->shape);
  if (!same(dy->shape, ys))
    throw Err(CK_ERR_SHAPE, "bilinear backward: projection " + shape_str(dy->shape) +
                                " does not match output " + shape_str(ys));
  if (dx) check_out(dx, x->shape, "dx");
  if (dgrid) check_out(dgrid, grid->shape, "dgrid");
  const ck_shape& s = x->shape;
  bilinear_backward(x->data, grid->data, dy->data, dx ? dx->data : nullptr,
                    dgrid ? dgrid->data : nullptr, (int)s.h, (int)s.w, (int)s.c, (int)s.n,
                    (int)ys.h, (int)ys.w, accumulate, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_pdist_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* target, double p,
                           int no_root, ck_tensor* y, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(target, "target");
  const ck_shape ys = pdist_output_shape(x->shape, target->shape, p);
  check_out(y, ys, "y");
  const ck_shape& s = x->shape;
  pdist_forward(x->data, target->data, y->data, (int)(s.h * s.w), (int)s.c, (int)s.n, p, no_root,
                (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_pdist_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* target, double p,
                            int no_root, const ck_tensor* dy, ck_tensor* dx, ck_tensor* dtarget,
                            int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(target, "target");
  check_tensor(dy, "dy");
  const ck_shape ys = pdist_output_shape(x->shape, target->shape, p);
  if (!same(dy->shape, ys))
    throw Err(CK_ERR_SHAPE, "pdist backward: projection " + shape_str(dy->shape) +
                                " does not match output " + shape_str(ys));
  if (dx) check_out(dx, x->shape, "dx");
  if (dtarget) check_out(dtarget, x->shape, "dtarget");
  const ck_shape& s = x->shape;
  pdist_backward(x->data, target->data, dy->data, dx ? dx->data : nullptr,
                 dtarget ? dtarget->data : nullptr, (int)(s.h * s.w), (int)s.c, (int)s.n, p,
                 no_root, accumulate, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_loss_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                          const ck_tensor* weights, ck_loss_kind kind, const ck_loss_options* opts,
                          float* loss, int check_labels, ck_stream stream) {
  CK_API_BEGIN(h)
  check_loss_kind(x, labels, weights, kind);
  if (!loss) throw Err(CK_ERR_ARG, "null loss pointer");
  const ck_loss_options o = opts ? *opts : default_loss_options();
  cudaStream_t st = (cudaStream_t)stream;
  if (check_labels) reset_label_flag(h, st);
  loss_forward_any(h, x, labels, weights, kind, o, loss, st);
  after_launch();
  if (check_labels) read_label_flag(h, st);
  CK_API_END(h)
}

ck_status ck_loss_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                           const ck_tensor* weights, ck_loss_kind kind, const ck_loss_options* opts,
                           float p, ck_tensor* dx, int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_loss_kind(x, labels, weights, kind);
  check_out(dx, x->shape, "dx");
  (void)opts;  // loss_backward ignores the options (loss.cpp:234)
  loss_backward_any(h, x, labels, weights, kind, p, nullptr, dx->data, accumulate,
                    (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

}  // extern "C"
