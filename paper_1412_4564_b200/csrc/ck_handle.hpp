// The opaque ck_handle of ck.h and the error plumbing shared by capi.cu,
// graph.cpp and trainer.cpp.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "ck/ck.h"
#include "ck_internal.hpp"

namespace ck {
struct TcState;  // conv_tc.cu: cached tensor maps / layout buffers
}

struct ck_handle {
  int device = 0;
  std::string err;
  ck::LaunchCounter counter;
  ck::Workspace ws;       // conv wgrad partials, bnorm statistics
  ck::Workspace scratch;  // loss per-site values, staging
  int* flag = nullptr;    // device label-error flag (loss.cpp:14-18, :101-106)
  int64_t last_classes = 0;
  ck::TcState* tc = nullptr;
  uint64_t call = 0;      // API call id: scopes transform caches to one call
  ck::ConvCache* conv_cache = nullptr;  // set by the graph engine around conv calls
  float* fuse_relu = nullptr;  // engine: conv forward may also write relu(y) here
  bool fuse_relu_done = false; // ... and reports whether it did
  // engine, conv backward of a fused conv -> relu: dy (the conv output's
  // derivative) is relu_x > 0 ? relu_dy : 0, produced inside the call
  const float* fuse_relu_x = nullptr;
  const float* fuse_relu_dy = nullptr;
  // engine: the conv output's derivative itself need not be stored (only its
  // grid form is consumed); set by ck_conv_backward when it was left pending
  bool fuse_relu_lazy = false;
  bool fuse_relu_pending = false;
  // a dy left unmaterialized by the gated transform: any later reader of dy
  // (a cache miss, a fallback path) first computes it (materialize_pending_dy)
  const float* pending_dy = nullptr;
  const float* pending_rx = nullptr;
  const float* pending_rdy = nullptr;
  int64_t pending_n = 0;
  // engine: a dy grid (and its bias-gradient partials) already built by the
  // layer below's backward (lrn_backward_grid) for the conv backward of this
  // call: used by dy_grid when (source, key) match
  float* pre_dyg = nullptr;
  const float* pre_dyg_src = nullptr;
  int64_t pre_dyg_key = 0;
  const double* pre_bpart = nullptr;
  int pre_rows = 0;
  ck::KernelProfiler prof;
  // engine, conv -> relu -> conv: the forward of the first conv also writes
  // relu(y) into the second conv's x grid (next_xg, laid out by next_xg_plan)
  float* next_xg = nullptr;
  ck::XGridPlan next_xg_plan{};
  bool next_xg_done = false;
  // engine, conv -> relu -> conv backward: the second conv's data-gradient
  // epilogue also writes the first conv's relu-gated dy grid (prev_dyg, laid
  // out by prev_dyg_plan; gate: prev_gate > 0, the second conv's input x)
  // and that grid's bias partials (prev_bpart, [32-pixel warp][Cp] doubles)
  float* prev_dyg = nullptr;
  double* prev_bpart = nullptr;
  const float* prev_gate = nullptr;
  ck::GridPlan prev_dyg_plan{};
  bool prev_dyg_done = false;
  // engine, fused bnorm -> relu: per-channel (mu, inv) of the forward, which
  // the backward uses to recompute the relu gate from x, followed by the
  // forward's w and b (4 floats / channel: [2C] (mu, inv), [C] w, [C] b)
  float* bn_muinv = nullptr;
  // engine, fused bnorm -> relu with the bnorm output read by nothing else:
  // the forward stores only relu(y) (y is recomputed from x on request)
  bool bn_skip_y = false;
  bool bn_y_skipped = false;
};

namespace ck {

// A reference exception (error.hpp:9-24) carried to the C boundary.
struct Err : std::runtime_error {
  ck_status code;
  Err(ck_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Binds the device and the launch counter for the duration of one API call.
struct HandleScope {
  LaunchCounter* prev;
  KernelProfiler* prev_prof;
  explicit HandleScope(ck_handle* h) : prev(g_counter), prev_prof(g_prof) {
    ++h->call;
    cudaSetDevice(h->device);
    g_counter = &h->counter;
    g_prof = &h->prof;
  }
  ~HandleScope() {
    g_counter = prev;
    g_prof = prev_prof;
  }
};

std::string shape_str(const ck_shape& s);
bool same(const ck_shape& a, const ck_shape& b);
int64_t elems(const ck_shape& s);
void check_tensor(const ck_tensor* t, const char* what);
void check_out(const ck_tensor* t, const ck_shape& want, const char* what);
ck_shape conv_output_shape(const ck_shape& x, const ck_shape& f, const ck_conv_geom& g);
ck_shape convt_output_shape(const ck_shape& x, const ck_shape& f, const ck_convt_geom& g);
ck_shape pool_output_shape(const ck_shape& x, const ck_pool_geom& g);
ConvDims conv_dims(const ck_shape& x, const ck_shape& f, const ck_shape& y, const ck_conv_geom& g);
PoolDims pool_dims(const ck_shape& x, const ck_shape& y, const ck_pool_geom& g);
void check_cuda(cudaError_t e, const char* what);
void after_launch();
// the device label/data-error flag of h (2 ints): reset, read (synchronising
// s, throws CK_ERR_DATA with the reference's message), decode a copied value
void reset_label_flag(ck_handle* h, cudaStream_t s);
void read_label_flag(ck_handle* h, cudaStream_t s);
void throw_label_flag(int flag, int label, int64_t classes);
// capi_ext.cu: shape laws / validation / launch of the extended block set
ck_shape bilinear_output_shape(const ck_shape& x, const ck_shape& grid);
ck_shape pdist_output_shape(const ck_shape& x, const ck_shape& target, double p);
bool loss_is_attribute(int kind);
void check_loss_kind(const ck_tensor* x, const ck_tensor* labels, const ck_tensor* weights,
                     int kind);
ck_loss_options default_loss_options();
void loss_forward_any(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                      const ck_tensor* weights, int kind, const ck_loss_options& o, float* loss,
                      cudaStream_t st);
void loss_backward_any(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                       const ck_tensor* weights, int kind, float p, const float* p_dev,
                       float* dx, int acc, cudaStream_t st);

void conv_forward_dispatch(ck_handle* h, const float* x, const float* f, const float* bias,
                           float* y, const ConvDims& d, int relu, ck_math math, cudaStream_t s);
void conv_dgrad_dispatch(ck_handle* h, const float* dy, const float* f, float* dx,
                         const ConvDims& d, int acc, ck_math math, cudaStream_t s);
void conv_wgrad_dispatch(ck_handle* h, const float* x, const float* dy, float* df,
                         const ConvDims& d, int acc, ck_math math, cudaStream_t s);

// conv_tc.cu: the tcgen05 TF32 kernels.  Each returns false (launching
// nothing) when the problem is outside the kernel's envelope.
bool conv_tc_forward(ck_handle* h, const float* x, const float* f, const float* bias, float* y,
                     const ConvDims& d, int relu, cudaStream_t s);
bool conv_tc_dgrad(ck_handle* h, const float* dy, const float* f, float* dx, const ConvDims& d,
                   int acc, cudaStream_t s);
bool conv_tc_wgrad(ck_handle* h, const float* x, const float* dy, float* df, const ConvDims& d,
                   int acc, cudaStream_t s);
bool conv_tc_bias(ck_handle* h, const float* dy, float* db, const ConvDims& d, int acc,
                  cudaStream_t s, const float* relu_x = nullptr, const float* relu_dy = nullptr,
                  bool skip_gout = false);
// The x grid a stride-1 TF32 conv forward (and its weight gradient) reads:
// pixel-major, Cgp channels per group, x at (pt, pl) of an Hg x Wg image grid
// (key: x_grid's cache key).  conv_tc_xgrid_plan says whether conv d reads x
// only through it, so the layer producing x may write it instead.
bool conv_tc_xgrid_plan(const ConvDims& d, XGridPlan* xp);
// capi.cu: bnorm backward writing the conv-below's dy grid (engine bn_grid)
bool bnorm_backward_to_grid(ck_handle* h, const ck_tensor* x, const ck_tensor* w,
                            const ck_tensor* b, double epsilon, const ck_tensor* dy,
                            ck_tensor* dw, ck_tensor* db, int accumulate, const GridPlan& gp,
                            float* grid, double* bpart, cudaStream_t st);
// (GridPlan: ck_internal.hpp)
bool conv_tc_grid_plan(const ConvDims& d, GridPlan* gp);
// capi.cu: compute a dy the gated transform left pending (h->pending_dy == dy)
void materialize_pending_dy(ck_handle* h, const float* dy, cudaStream_t s);
void conv_tc_release(ck_handle* h);

}  // namespace ck

// Entry-point wrapper of every extern "C" function: binds the handle,
// maps reference exceptions to status codes and keeps the message.
#define CK_API_BEGIN(h)                      \
  if (!(h)) return CK_ERR_ARG;               \
  ck::HandleScope _scope(h);                 \
  try {
#define CK_API_END(h)                        \
  return CK_OK;                              \
  }                                          \
  catch (const ck::Err& e) {                 \
    (h)->err = e.what();                     \
    return e.code;                           \
  }                                          \
  catch (const std::exception& e) {          \
    (h)->err = e.what();                     \
    return CK_ERR_ARG;                       \
  }
