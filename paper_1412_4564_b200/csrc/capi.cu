// capi.cu -- the extern "C" block API of ck.h.
//
// Each entry point (1) validates its arguments on the host with the
// reference's rules and messages, (2) maps the reference's exceptions to
// status codes, and (3) launches the device kernels on the caller's stream.
// Citations are to /root/reference/proj.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "ck/ck.h"
#include "ck_internal.hpp"
#include "ck_handle.hpp"

using ck::Err;

namespace ck {

int knob(const char* name, int dflt) {
#ifdef CK_EXPERIMENTS
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

bool experiments_build() {
#ifdef CK_EXPERIMENTS
  return true;
#else
  return false;
#endif
}

static std::atomic<uint64_t> g_ws_gen{0};
uint64_t workspace_generation() { return g_ws_gen.load(std::memory_order_relaxed); }

void* Workspace::get(size_t want, cudaStream_t s) {
  if (want <= bytes) return ptr;
  g_ws_gen.fetch_add(1, std::memory_order_relaxed);
  if (ptr) {
    cudaStreamSynchronize(s);
    cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  size_t cap = want + want / 4;
  if (cudaMalloc(&ptr, cap) != cudaSuccess) {
    ptr = nullptr;
    return nullptr;
  }
  bytes = cap;
  return ptr;
}

void Workspace::release() {
  if (ptr) {
    g_ws_gen.fetch_add(1, std::memory_order_relaxed);
    cudaFree(ptr);
  }
  ptr = nullptr;
  bytes = 0;
}

std::string shape_str(const ck_shape& s) {
  return std::to_string(s.h) + "x" + std::to_string(s.w) + "x" + std::to_string(s.c) + "x" +
         std::to_string(s.n);
}

bool same(const ck_shape& a, const ck_shape& b) {
  return a.h == b.h && a.w == b.w && a.c == b.c && a.n == b.n;
}

int64_t elems(const ck_shape& s) { return s.h * s.w * s.c * s.n; }

// tensor.hpp:88-91 check_shape
void check_tensor(const ck_tensor* t, const char* what) {
  if (!t) throw Err(CK_ERR_ARG, std::string(what) + ": null tensor");
  const ck_shape& s = t->shape;
  if (s.h < 1 || s.w < 1 || s.c < 1 || s.n < 1)
    throw Err(CK_ERR_SHAPE, "invalid tensor shape " + shape_str(s));
  if (elems(s) >= (int64_t(1) << 31))
    throw Err(CK_ERR_ARG, std::string(what) + ": tensor too large (" + shape_str(s) + ")");
  if (!t->data) throw Err(CK_ERR_ARG, std::string(what) + ": null data pointer");
}

void check_out(const ck_tensor* t, const ck_shape& want, const char* what) {
  check_tensor(t, what);
  if (!same(t->shape, want))
    throw Err(CK_ERR_SHAPE, std::string(what) + " tensor " + shape_str(t->shape) +
                                " does not match expected " + shape_str(want));
}

// conv.cpp:108-116
int64_t conv_output_extent(int64_t extent, int64_t window, int64_t stride, int64_t lo,
                           int64_t hi) {
  if (extent + lo + hi < window)
    throw Err(CK_ERR_SHAPE, "window of size " + std::to_string(window) +
                                " larger than padded input of size " +
                                std::to_string(extent + lo + hi));
  return (extent - window + lo + hi) / stride + 1;
}

// conv.cpp:18-23 + :118-135
ck_shape conv_output_shape(const ck_shape& x, const ck_shape& f, const ck_conv_geom& g) {
  if (g.stride_h < 1 || g.stride_w < 1 || g.groups < 1 || g.pad_top < 0 || g.pad_bottom < 0 ||
      g.pad_left < 0 || g.pad_right < 0)
    throw Err(CK_ERR_SHAPE, "invalid convolution geometry");
  if (f.c * g.groups != x.c)
    throw Err(CK_ERR_SHAPE, "filter channels " + std::to_string(f.c) + " x groups " +
                                std::to_string(g.groups) + " do not match input channels " +
                                std::to_string(x.c));
  if (f.n % g.groups != 0)
    throw Err(CK_ERR_SHAPE, "filter count " + std::to_string(f.n) +
                                " not divisible by groups " + std::to_string(g.groups));
  ck_shape o;
  o.h = conv_output_extent(x.h, f.h, g.stride_h, g.pad_top, g.pad_bottom);
  o.w = conv_output_extent(x.w, f.w, g.stride_w, g.pad_left, g.pad_right);
  o.c = f.n;
  o.n = x.n;
  return o;
}

// conv.cpp:25-30 + :137-154
ck_shape convt_output_shape(const ck_shape& x, const ck_shape& f, const ck_convt_geom& g) {
  if (g.up_h < 1 || g.up_w < 1 || g.crop_top < 0 || g.crop_bottom < 0 || g.crop_left < 0 ||
      g.crop_right < 0)
    throw Err(CK_ERR_SHAPE, "invalid convolution-transpose geometry");
  if (f.c != x.c)
    throw Err(CK_ERR_SHAPE, "transposed filter expects " + std::to_string(f.c) +
                                " input channels, got " + std::to_string(x.c));
  ck_shape o;
  o.h = g.up_h * (x.h - 1) + f.h - g.crop_top - g.crop_bottom;
  o.w = g.up_w * (x.w - 1) + f.w - g.crop_left - g.crop_right;
  o.c = f.n;
  o.n = x.n;
  if (o.h < 1 || o.w < 1)
    throw Err(CK_ERR_SHAPE, "transposed convolution output " + shape_str(o) + " is not positive");
  return o;
}

// pool.cpp:9-18 + :35-46
ck_shape pool_output_shape(const ck_shape& x, const ck_pool_geom& g) {
  if (g.window_h < 1 || g.window_w < 1 || g.stride_h < 1 || g.stride_w < 1 || g.pad_top < 0 ||
      g.pad_bottom < 0 || g.pad_left < 0 || g.pad_right < 0)
    throw Err(CK_ERR_SHAPE, "invalid pooling geometry");
  if (g.pad_top > g.window_h - 1 || g.pad_bottom > g.window_h - 1 ||
      g.pad_left > g.window_w - 1 || g.pad_right > g.window_w - 1)
    throw Err(CK_ERR_SHAPE, "pooling pad exceeds window size minus one");
  if (g.mode != CK_POOL_MAX && g.mode != CK_POOL_AVG)
    throw Err(CK_ERR_ARG, "unknown pooling mode");
  ck_shape o;
  o.h = conv_output_extent(x.h, g.window_h, g.stride_h, g.pad_top, g.pad_bottom);
  o.w = conv_output_extent(x.w, g.window_w, g.stride_w, g.pad_left, g.pad_right);
  o.c = x.c;
  o.n = x.n;
  return o;
}

ConvDims conv_dims(const ck_shape& x, const ck_shape& f, const ck_shape& y,
                   const ck_conv_geom& g) {
  ConvDims d;
  d.H = (int)x.h; d.W = (int)x.w; d.C = (int)x.c; d.N = (int)x.n;
  d.fh = (int)f.h; d.fw = (int)f.w; d.Cg = (int)f.c; d.K = (int)f.n;
  d.OH = (int)y.h; d.OW = (int)y.w;
  d.sh = (int)g.stride_h; d.sw = (int)g.stride_w;
  d.pt = (int)g.pad_top; d.pb = (int)g.pad_bottom; d.pl = (int)g.pad_left; d.pr = (int)g.pad_right;
  d.groups = (int)g.groups;
  d.fsc = 1;
  d.fsk = d.Cg;
  return d;
}

PoolDims pool_dims(const ck_shape& x, const ck_shape& y, const ck_pool_geom& g) {
  PoolDims d;
  d.H = (int)x.h; d.W = (int)x.w; d.C = (int)x.c; d.N = (int)x.n;
  d.OH = (int)y.h; d.OW = (int)y.w;
  d.wh = (int)g.window_h; d.ww = (int)g.window_w; d.sh = (int)g.stride_h; d.sw = (int)g.stride_w;
  d.pt = (int)g.pad_top; d.pl = (int)g.pad_left;
  d.mode = (int)g.mode;
  return d;
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Err(CK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void after_launch() { check_cuda(cudaPeekAtLastError(), "kernel launch"); }

// The device label/data flag (kernels.cu read_label): flag[0] bits, flag[1]
// the first offending class label.  Messages are loss.cpp's (:14-18, :101-106,
// :152-154, :201-203, :193-195).
void throw_label_flag(int flag, int label, int64_t classes) {
  // SPEC.md:716, :766 exit code 3: a non-finite objective aborts training
  if (flag & 64) throw Err(CK_ERR_NUMERIC, "non-finite loss (NaN or Inf): training aborted");
  if (flag & 1) throw Err(CK_ERR_DATA, "class label is not an integer");
  if (flag & 2)
    throw Err(CK_ERR_DATA, "class label " + std::to_string(label) + " out of range 1.." +
                               std::to_string(classes));
  if (flag & 4) throw Err(CK_ERR_DATA, "log loss needs a positive ground-truth score");
  if (flag & 8) throw Err(CK_ERR_DATA, "attribute label is not an integer");
  if (flag & 16) throw Err(CK_ERR_DATA, "attribute label must be -1, 0 or +1");
  if (flag & 32) throw Err(CK_ERR_DATA, "binary log loss input must lie in [0,1]");
}

void reset_label_flag(ck_handle* h, cudaStream_t s) {
  check_cuda(cudaMemsetAsync(h->flag, 0, 2 * sizeof(int), s), "flag");
}

void read_label_flag(ck_handle* h, cudaStream_t s) {
  int flag[2] = {0, 0};
  check_cuda(cudaMemcpyAsync(flag, h->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, s), "flag");
  check_cuda(cudaStreamSynchronize(s), "synchronize");
  if (flag[0]) {
    reset_label_flag(h, s);
    throw_label_flag(flag[0], flag[1], h->last_classes);
  }
}


// ---- conv dispatch (shared by the C ABI and the graph engine) ----------------

// a profiler label left by a tensor-core path that declined the shape
static void prof_drop() {
  if (g_prof) g_prof->label.clear();
}

void conv_forward_dispatch(ck_handle* h, const float* x, const float* f, const float* bias,
                           float* y, const ConvDims& d, int relu, ck_math math, cudaStream_t s) {
  if (math == CK_MATH_TF32 && conv_tc_forward(h, x, f, bias, y, d, relu, s)) return;
  prof_drop();
  conv_fwd_fp32(x, f, bias, y, d, relu, s);
}

void materialize_pending_dy(ck_handle* h, const float* dy, cudaStream_t s) {
  if (!h->pending_dy || h->pending_dy != dy) return;
  relu_backward(h->pending_rx, h->pending_rdy, const_cast<float*>(dy), h->pending_n, 0, s);
  h->pending_dy = nullptr;
}

void conv_dgrad_dispatch(ck_handle* h, const float* dy, const float* f, float* dx,
                         const ConvDims& d, int acc, ck_math math, cudaStream_t s) {
  if (math == CK_MATH_TF32 && conv_tc_dgrad(h, dy, f, dx, d, acc, s)) return;
  materialize_pending_dy(h, dy, s);
  prof_drop();
  conv_dgrad_fp32(dy, f, dx, d, acc, s);
}

void conv_wgrad_dispatch(ck_handle* h, const float* x, const float* dy, float* df,
                         const ConvDims& d, int acc, ck_math math, cudaStream_t s) {
  if (math == CK_MATH_TF32 && conv_tc_wgrad(h, x, dy, df, d, acc, s)) return;
  materialize_pending_dy(h, dy, s);
  prof_drop();
  void* ws = h->ws.get(conv_wgrad_ws_bytes(d), s);
  if (!ws) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  conv_wgrad_fp32(x, dy, df, d, acc, ws, s);
}

}  // namespace ck

using namespace ck;

// Engine (conv -> bnorm, TF32 grid path): ck_bnorm_backward with dx written
// as the conv's dy grid + bias partials (bnorm_backward_grid) instead of HWCN;
// dw / db as usual.  False (nothing launched) outside the grid kernel's envelope.
namespace ck {
bool bnorm_backward_to_grid(ck_handle* h, const ck_tensor* x, const ck_tensor* w,
                            const ck_tensor* b, double epsilon, const ck_tensor* dy,
                            ck_tensor* dw, ck_tensor* db, int accumulate, const GridPlan& gp,
                            float* grid, double* bpart, cudaStream_t st) {
  const ck_shape& s = x->shape;
  const int HW = (int)(s.h * s.w), C = (int)s.c, N = (int)s.n;
  if (gp.Kg * gp.groups != C || gp.Kg % 32 || C % 32 || gp.OH != (int)s.h || gp.OW != (int)s.w)
    return false;
  const int splits = bnorm_splits(HW, C, N);
  double* buf = (double*)h->ws.get(sizeof(double) * 4 * (size_t)C * (splits + 1), st);
  if (!buf) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  double* stats = buf + (size_t)4 * C * splits;
  const float* dyp = h->fuse_relu_x ? h->fuse_relu_dy : dy->data;
  BnGate rg;
  if (h->fuse_relu_x && h->bn_muinv) rg = BnGate{w->data, b->data, h->bn_muinv};
  const float* gate = rg.muinv ? nullptr : h->fuse_relu_x;
  if ((int64_t)s.n * gp.Hg * gp.Wg * gp.Kgp * gp.groups >= (1ll << 31)) return false;
  bnorm_stats(x->data, dyp, buf, stats, HW, C, N, splits, st, gate, rg);
  // (dw / db written by the grid kernel's first block)
  return bnorm_backward_grid(x->data, dyp, w->data, stats, epsilon, (int)s.h, (int)s.w, C, N,
                             grid, bpart, gp.Hg, gp.Wg, gp.Kg, gp.Kgp, gp.groups, st, gate, rg,
                             dw ? dw->data : nullptr, db ? db->data : nullptr, accumulate);
}
}  // namespace ck

extern "C" {

const char* ck_version(void) {
  return ck::experiments_build() ? "ck 0.2 (sm_100a, CK_EXPERIMENTS)" : "ck 0.2 (sm_100a)";
}

ck_status ck_create(ck_handle** out, int device) {
  if (!out) return CK_ERR_ARG;
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return CK_ERR_CUDA;
  ck_handle* h = new ck_handle();
  h->device = device;
  if (cudaMalloc(&h->flag, 2 * sizeof(int)) != cudaSuccess) {
    delete h;
    return CK_ERR_CUDA;
  }
  cudaMemset(h->flag, 0, 2 * sizeof(int));
  *out = h;
  return CK_OK;
}

void ck_destroy(ck_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  h->ws.release();
  h->scratch.release();
  if (h->flag) cudaFree(h->flag);
  conv_tc_release(h);
  delete h;
}

const char* ck_last_error(const ck_handle* h) { return h ? h->err.c_str() : "null handle"; }

int64_t ck_tc_launch_count(const ck_handle* h) { return h ? h->counter.tc : 0; }

int64_t ck_launch_count(const ck_handle* h) { return h ? h->counter.n : 0; }

ck_status ck_set_kernel_profiling(ck_handle* h, int on) {
  CK_API_BEGIN(h)
  h->prof.on = on != 0;
  h->prof.label.clear();
  CK_API_END(h)
}

int ck_kernel_profile_count(const ck_handle* h) { return h ? (int)h->prof.recs.size() : 0; }

ck_status ck_kernel_profile_get(ck_handle* h, int i, const char** label, float* ms,
                                double* flops) {
  CK_API_BEGIN(h)
  if (i < 0 || i >= (int)h->prof.recs.size()) throw Err(CK_ERR_ARG, "profile index out of range");
  auto& r = h->prof.recs[(size_t)i];
  check_cuda(cudaEventSynchronize(r.b), "event sync");
  float t = 0;
  check_cuda(cudaEventElapsedTime(&t, r.a, r.b), "event time");
  if (label) *label = r.label.c_str();
  if (ms) *ms = t;
  if (flops) *flops = r.flops;
  CK_API_END(h)
}

ck_status ck_kernel_profile_clear(ck_handle* h) {
  CK_API_BEGIN(h)
  h->prof.clear();
  CK_API_END(h)
}

ck_status ck_memcpy(ck_handle* h, void* dst, const void* src, int64_t bytes, ck_stream stream) {
  CK_API_BEGIN(h)
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) throw Err(CK_ERR_ARG, "memcpy: bad arguments");
  if (bytes)
    check_cuda(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream),
               "cudaMemcpyAsync");
  CK_API_END(h)
}

ck_status ck_conv_output_shape(ck_handle* h, ck_shape x, ck_shape f, const ck_conv_geom* g,
                               ck_shape* out) {
  CK_API_BEGIN(h)
  if (!g || !out) throw Err(CK_ERR_ARG, "null argument");
  *out = conv_output_shape(x, f, *g);
  CK_API_END(h)
}

ck_status ck_convt_output_shape(ck_handle* h, ck_shape x, ck_shape f, const ck_convt_geom* g,
                                ck_shape* out) {
  CK_API_BEGIN(h)
  if (!g || !out) throw Err(CK_ERR_ARG, "null argument");
  *out = convt_output_shape(x, f, *g);
  CK_API_END(h)
}

ck_status ck_pool_output_shape(ck_handle* h, ck_shape x, const ck_pool_geom* g, ck_shape* out) {
  CK_API_BEGIN(h)
  if (!g || !out) throw Err(CK_ERR_ARG, "null argument");
  *out = pool_output_shape(x, *g);
  CK_API_END(h)
}

// conv.cpp:193-226
ck_status ck_conv_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                          const ck_tensor* bias, const ck_conv_geom* g, ck_tensor* y,
                          ck_math math, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(f, "f");
  if (!g) throw Err(CK_ERR_ARG, "null geometry");
  ck_shape ys = conv_output_shape(x->shape, f->shape, *g);
  if (bias) {
    check_tensor(bias, "bias");
    if (elems(bias->shape) != f->shape.n)
      throw Err(CK_ERR_SHAPE, "bias has " + std::to_string(elems(bias->shape)) +
                                  " elements for " + std::to_string(f->shape.n) + " filters");
  }
  check_out(y, ys, "y");
  ConvDims d = conv_dims(x->shape, f->shape, ys, *g);
  conv_forward_dispatch(h, x->data, f->data, bias ? bias->data : nullptr, y->data, d, 0, math,
                        (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

// conv.cpp:229-280
ck_status ck_conv_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                           const ck_conv_geom* g, const ck_tensor* dy, ck_tensor* dx,
                           ck_tensor* df, ck_tensor* db, int accumulate, ck_math math,
                           ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(f, "f");
  check_tensor(dy, "dy");
  if (!g) throw Err(CK_ERR_ARG, "null geometry");
  ck_shape ys = conv_output_shape(x->shape, f->shape, *g);
  if (!same(dy->shape, ys))
    throw Err(CK_ERR_SHAPE, "conv backward: projection " + shape_str(dy->shape) +
                                " does not match output " + shape_str(ys));
  if (dx) check_out(dx, x->shape, "dx");
  if (df) check_out(df, f->shape, "df");
  if (db) {
    check_tensor(db, "db");
    if (elems(db->shape) != f->shape.n)
      throw Err(CK_ERR_SHAPE, "db has " + std::to_string(elems(db->shape)) + " elements for " +
                                  std::to_string(f->shape.n) + " filters");
  }
  cudaStream_t s = (cudaStream_t)stream;
  ConvDims d = conv_dims(x->shape, f->shape, ys, *g);
  // TF32 conv layers with a tensor-core grid path reduce db inside the dy
  // transform their dgrad/wgrad reuse; everything else uses conv_bgrad.
  // With the engine's fused conv -> relu, dy is first produced from the relu
  // output derivative (inside the transform when the grid path runs).
  const float* rx = h->fuse_relu_x;
  const float* rdy = h->fuse_relu_dy;
  // the engine may let the gated transform skip storing dy itself (only its
  // grid form is consumed): dy is then left pending, computed by any reader
  // that needs it, and reported back through fuse_relu_pending
  const bool lazy = h->fuse_relu_lazy && rx;
  h->fuse_relu_pending = false;
  bool gated = false;
  if (db && math == CK_MATH_TF32 && (dx || df) &&
      conv_tc_bias(h, dy->data, db->data, d, accumulate, s, rx, rdy, lazy)) {
    db = nullptr;
    gated = rx != nullptr;
  }
  if (rx && !gated) relu_backward(rx, rdy, dy->data, elems(dy->shape), 0, s);
  if (gated && lazy) {
    h->pending_dy = dy->data;
    h->pending_rx = rx;
    h->pending_rdy = rdy;
    h->pending_n = elems(dy->shape);
  }
  struct PendingReset {
    ck_handle* h;
    ~PendingReset() { h->pending_dy = nullptr; }
  } pending_reset{h};
  if (db) {
    void* bws = h->scratch.get(conv_bgrad_ws_bytes((int)ys.c, (int)ys.n, (int)(ys.h * ys.w)), s);
    if (!bws) throw Err(CK_ERR_CUDA, "workspace allocation failed");
    conv_bgrad(dy->data, db->data, (int)(ys.h * ys.w), (int)ys.c, (int)ys.n, accumulate, bws, s);
  }
  if (df) conv_wgrad_dispatch(h, x->data, dy->data, df->data, d, accumulate, math, s);
  if (dx) conv_dgrad_dispatch(h, dy->data, f->data, dx->data, d, accumulate, math, s);
  h->fuse_relu_pending = h->pending_dy == dy->data;  // still unmaterialized
  after_launch();
  CK_API_END(h)
}

// conv.cpp:283-308: y = M^T x where M is the conv (stride = up, pad = crop)
// mapping y-space (K = f.n channels) onto x-space (D = f.c channels) with the
// swapped bank g[fi,fj,k,d] = f[fi,fj,d,k]; i.e. y = dgrad of that conv.
static ConvDims convt_as_conv(const ck_shape& x, const ck_shape& f, const ck_shape& y,
                              const ck_convt_geom& g) {
  ConvDims d;
  d.H = (int)y.h; d.W = (int)y.w; d.C = (int)f.n; d.N = (int)x.n;
  d.fh = (int)f.h; d.fw = (int)f.w; d.Cg = (int)f.n; d.K = (int)f.c;
  d.OH = (int)x.h; d.OW = (int)x.w;
  d.sh = (int)g.up_h; d.sw = (int)g.up_w;
  d.pt = (int)g.crop_top; d.pb = (int)g.crop_bottom; d.pl = (int)g.crop_left;
  d.pr = (int)g.crop_right;
  d.groups = 1;
  // conv filter (fi,fj,c=k_y,k=d_x) lives at f[fi + fh*(fj + fw*(d_x + D*k_y))]
  d.fsc = f.c;
  d.fsk = 1;
  return d;
}

ck_status ck_convt_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                           const ck_convt_geom* g, ck_tensor* y, ck_math math, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(f, "f");
  if (!g) throw Err(CK_ERR_ARG, "null geometry");
  ck_shape ys = convt_output_shape(x->shape, f->shape, *g);
  check_out(y, ys, "y");
  ConvDims d = convt_as_conv(x->shape, f->shape, ys, *g);
  conv_dgrad_dispatch(h, x->data, f->data, y->data, d, 0, math, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

// conv.cpp:311-365: dx = conv(dy, swapped bank) (stride = up, pad = crop);
// df = wgrad of the same conv with input dy and output-derivative x.
ck_status ck_convt_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                            const ck_convt_geom* g, const ck_tensor* dy, ck_tensor* dx,
                            ck_tensor* df, int accumulate, ck_math math, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(f, "f");
  check_tensor(dy, "dy");
  if (!g) throw Err(CK_ERR_ARG, "null geometry");
  ck_shape ys = convt_output_shape(x->shape, f->shape, *g);
  if (!same(dy->shape, ys))
    throw Err(CK_ERR_SHAPE, "convt backward: projection " + shape_str(dy->shape) +
                                " does not match output " + shape_str(ys));
  if (dx) check_out(dx, x->shape, "dx");
  if (df) check_out(df, f->shape, "df");
  cudaStream_t s = (cudaStream_t)stream;
  ConvDims d = convt_as_conv(x->shape, f->shape, ys, *g);
  if (dx) {
    if (accumulate) {
      // fprop has no accumulate epilogue on the tensor-core path; stage.
      float* tmp = (float*)h->scratch.get(sizeof(float) * elems(x->shape), s);
      if (!tmp) throw Err(CK_ERR_CUDA, "workspace allocation failed");
      conv_forward_dispatch(h, dy->data, f->data, nullptr, tmp, d, 0, math, s);
      axpy_inplace(dx->data, tmp, elems(x->shape), s);
    } else {
      conv_forward_dispatch(h, dy->data, f->data, nullptr, dx->data, d, 0, math, s);
    }
  }
  if (df) conv_wgrad_dispatch(h, dy->data, x->data, df->data, d, accumulate, math, s);
  after_launch();
  CK_API_END(h)
}

// pool.cpp:49-80
ck_status ck_pool_forward(ck_handle* h, const ck_tensor* x, const ck_pool_geom* g, ck_tensor* y,
                          ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  if (!g) throw Err(CK_ERR_ARG, "null geometry");
  ck_shape ys = pool_output_shape(x->shape, *g);
  check_out(y, ys, "y");
  pool_forward(x->data, y->data, pool_dims(x->shape, ys, *g), (cudaStream_t)stream,
               h->conv_cache);
  after_launch();
  CK_API_END(h)
}

// pool.cpp:83-126
ck_status ck_pool_backward(ck_handle* h, const ck_tensor* x, const ck_pool_geom* g,
                           const ck_tensor* dy, ck_tensor* dx, int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(dy, "dy");
  if (!g) throw Err(CK_ERR_ARG, "null geometry");
  ck_shape ys = pool_output_shape(x->shape, *g);
  if (!same(dy->shape, ys))
    throw Err(CK_ERR_SHAPE, "pool backward: projection " + shape_str(dy->shape) +
                                " does not match output " + shape_str(ys));
  check_out(dx, x->shape, "dx");
  pool_backward(x->data, dy->data, dx->data, pool_dims(x->shape, ys, *g), accumulate,
                (cudaStream_t)stream, h->conv_cache);
  after_launch();
  CK_API_END(h)
}

// activation.cpp:8-12
ck_status ck_relu_forward(ck_handle* h, const ck_tensor* x, ck_tensor* y, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_out(y, x->shape, "y");
  relu_forward(x->data, y->data, elems(x->shape), (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

// activation.cpp:15-22
ck_status ck_relu_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* dy, ck_tensor* dx,
                           int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_tensor(x, "x");
  check_tensor(dy, "dy");
  if (!same(dy->shape, x->shape))
    throw Err(CK_ERR_SHAPE, "relu backward: projection shape mismatch");
  check_out(dx, x->shape, "dx");
  relu_backward(x->data, dy->data, dx->data, elems(x->shape), accumulate, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

// normalize.cpp:24-27 check_lrn
static void check_lrn(const ck_lrn_params* p) {
  if (!p) throw Err(CK_ERR_ARG, "null lrn parameters");
  if (p->group_size < 1) throw Err(CK_ERR_SHAPE, "lrn group size must be positive");
  if (p->kappa <= 0) throw Err(CK_ERR_SHAPE, "lrn kappa must be positive");
}

static void check_lrn_channels(int64_t C) {
  if (C * 3 * 32 * 4 > 227 * 1024)
    throw Err(CK_ERR_ARG, "lrn: " + std::to_string(C) + " channels exceed the staging tile");
}

ck_status ck_lrn_forward(ck_handle* h, const ck_tensor* x, const ck_lrn_params* p, ck_tensor* y,
                         ck_stream stream) {
  CK_API_BEGIN(h)
  check_lrn(p);
  check_tensor(x, "x");
  check_out(y, x->shape, "y");
  if (p->group_size > 9) check_lrn_channels(x->shape.c);  // register kernels for n <= 9
  const ck_shape& s = x->shape;
  lrn_forward(x->data, y->data, (int)s.h, (int)s.w, (int)s.c, (int)s.n, (int)p->group_size,
              (float)p->kappa, (float)p->alpha, (float)p->beta, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_lrn_backward(ck_handle* h, const ck_tensor* x, const ck_lrn_params* p,
                          const ck_tensor* dy, ck_tensor* dx, int accumulate, ck_stream stream) {
  CK_API_BEGIN(h)
  check_lrn(p);
  check_tensor(x, "x");
  check_tensor(dy, "dy");
  if (!same(dy->shape, x->shape))
    throw Err(CK_ERR_SHAPE, "lrn backward: projection shape mismatch");
  check_out(dx, x->shape, "dx");
  if (p->group_size > 9) check_lrn_channels(x->shape.c);  // register kernels for n <= 9
  const ck_shape& s = x->shape;
  lrn_backward(x->data, dy->data, dx->data, (int)s.h, (int)s.w, (int)s.c, (int)s.n,
               (int)p->group_size, (float)p->kappa, (float)p->alpha, (float)p->beta, accumulate,
               (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

// normalize.cpp:124-130 check_bnorm_args
static void check_bnorm(const ck_tensor* x, const ck_tensor* w, const ck_tensor* b, double eps) {
  check_tensor(x, "x");
  check_tensor(w, "w");
  check_tensor(b, "b");
  if (elems(w->shape) != x->shape.c || elems(b->shape) != x->shape.c)
    throw Err(CK_ERR_SHAPE, "bnorm expects one multiplier and bias per channel");
  if (!(eps > 0)) throw Err(CK_ERR_SHAPE, "bnorm epsilon must be positive");
}

ck_status ck_bnorm_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* w,
                           const ck_tensor* b, double epsilon, ck_tensor* y, ck_tensor* moments,
                           ck_stream stream) {
  CK_API_BEGIN(h)
  check_bnorm(x, w, b, epsilon);
  check_out(y, x->shape, "y");
  const ck_shape& s = x->shape;
  if (moments) check_out(moments, ck_shape{s.c, 2, 1, 1}, "moments");
  cudaStream_t st = (cudaStream_t)stream;
  int HW = (int)(s.h * s.w), C = (int)s.c, N = (int)s.n;
  int splits = bnorm_splits(HW, C, N);
  double* buf = (double*)h->ws.get(sizeof(double) * 4 * (size_t)C * (splits + 1), st);
  if (!buf) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  double* stats = buf + (size_t)4 * C * splits;
  bnorm_stats(x->data, nullptr, buf, stats, HW, C, N, splits, st);
  // engine (bnorm -> relu): relu(y) written by the same pass
  const bool skip_y = h->fuse_relu && h->bn_muinv && h->bn_skip_y;
  // engine, bnorm -> relu -> conv: relu(y) straight into the conv's x grid
  // (y and the HWCN relu output left unstored, recomputed on request)
  bool gridded = false;
  if (skip_y && h->next_xg) {
    const XGridPlan& xp = h->next_xg_plan;
    gridded = bnorm_apply_grid(x->data, w->data, b->data, stats,
                               moments ? moments->data : nullptr, h->bn_muinv, epsilon, (int)s.h,
                               (int)s.w, C, N, h->next_xg, xp.Hg, xp.Wg, xp.Cg, xp.Cgp, xp.groups,
                               xp.pt, xp.pl, st);
    h->next_xg_done = gridded;
  }
  if (!gridded)
    bnorm_apply(x->data, w->data, b->data, stats, nullptr, skip_y ? nullptr : y->data,
                moments ? moments->data : nullptr, epsilon, HW, C, N, st, h->fuse_relu,
                h->fuse_relu ? h->bn_muinv : nullptr);
  h->bn_y_skipped = skip_y;
  if (h->fuse_relu) h->fuse_relu_done = true;
  after_launch();
  CK_API_END(h)
}

ck_status ck_bnorm_infer(ck_handle* h, const ck_tensor* x, const ck_tensor* w, const ck_tensor* b,
                         double epsilon, const ck_tensor* moments, ck_tensor* y,
                         ck_stream stream) {
  CK_API_BEGIN(h)
  check_bnorm(x, w, b, epsilon);
  check_tensor(moments, "moments");
  if (elems(moments->shape) != 2 * x->shape.c)
    throw Err(CK_ERR_SHAPE, "bnorm moments do not match channel count");
  check_out(y, x->shape, "y");
  const ck_shape& s = x->shape;
  bnorm_apply(x->data, w->data, b->data, nullptr, moments->data, y->data, nullptr, epsilon,
              (int)(s.h * s.w), (int)s.c, (int)s.n, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_bnorm_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* w,
                            const ck_tensor* b, double epsilon, const ck_tensor* dy,
                            ck_tensor* dx, ck_tensor* dw, ck_tensor* db, int accumulate,
                            ck_stream stream) {
  CK_API_BEGIN(h)
  check_bnorm(x, w, b, epsilon);
  check_tensor(dy, "dy");
  if (!same(dy->shape, x->shape))
    throw Err(CK_ERR_SHAPE, "bnorm backward: projection shape mismatch");
  if (dx) check_out(dx, x->shape, "dx");
  if (dw) check_out(dw, w->shape, "dw");
  if (db) check_out(db, b->shape, "db");
  const ck_shape& s = x->shape;
  cudaStream_t st = (cudaStream_t)stream;
  int HW = (int)(s.h * s.w), C = (int)s.c, N = (int)s.n;
  int splits = bnorm_splits(HW, C, N);
  double* buf = (double*)h->ws.get(sizeof(double) * 4 * (size_t)C * (splits + 1), st);
  if (!buf) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  double* stats = buf + (size_t)4 * C * splits;
  // engine (bnorm -> relu, relu backward deferred): the derivative reaching
  // y is fuse_relu_x (= y) > 0 ? fuse_relu_dy : 0, formed inside both passes
  // With the forward's (mu, inv) at hand (h->bn_muinv) the gate y > 0 is
  // recomputed from x -- bit-identical to the forward's y -- instead of read.
  const float* dyp = h->fuse_relu_x ? h->fuse_relu_dy : dy->data;
  BnGate rg;
  if (h->fuse_relu_x && h->bn_muinv) rg = BnGate{w->data, b->data, h->bn_muinv};
  const float* gate = rg.muinv ? nullptr : h->fuse_relu_x;
  bnorm_stats(x->data, dyp, buf, stats, HW, C, N, splits, st, gate, rg);
  bnorm_backward_apply(x->data, dyp, w->data, stats, epsilon, dx ? dx->data : nullptr,
                       dw ? dw->data : nullptr, db ? db->data : nullptr, HW, C, N, accumulate,
                       st, gate, rg);
  after_launch();
  CK_API_END(h)
}


// loss.cpp:35-40 + :92-94
static void check_loss(const ck_tensor* x, const ck_tensor* labels, const ck_tensor* weights) {
  check_tensor(x, "x");
  check_tensor(labels, "labels");
  const ck_shape &xs = x->shape, &cs = labels->shape;
  if (weights) {
    check_tensor(weights, "weights");
    if (!same(weights->shape, cs))
      throw Err(CK_ERR_SHAPE, "instance weights must match the label tensor shape");
  }
  if (cs.h != xs.h || cs.w != xs.w || cs.c != 1 || cs.n != xs.n)
    throw Err(CK_ERR_SHAPE, "classification labels must be " +
                                shape_str(ck_shape{xs.h, xs.w, 1, xs.n}) + ", got " +
                                shape_str(cs));
}

ck_status ck_softmaxlog_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                                const ck_tensor* weights, float* loss, int check_labels,
                                ck_stream stream) {
  CK_API_BEGIN(h)
  check_loss(x, labels, weights);
  if (!loss) throw Err(CK_ERR_ARG, "null loss pointer");
  const ck_shape& s = x->shape;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t sites = s.h * s.w * s.n;
  float* site = (float*)h->scratch.get(sizeof(float) * sites, st);
  if (!site) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  h->last_classes = s.c;
  if (check_labels) reset_label_flag(h, st);  // no stale bit from an unchecked call
  softmaxlog_forward(x->data, labels->data, weights ? weights->data : nullptr, site, loss, h->flag,
                     (int)(s.h * s.w), (int)s.c, (int)s.n, st);
  after_launch();
  if (check_labels) read_label_flag(h, st);
  CK_API_END(h)
}

ck_status ck_softmaxlog_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                                 const ck_tensor* weights, float p, ck_tensor* dx, int accumulate,
                                 ck_stream stream) {
  CK_API_BEGIN(h)
  check_loss(x, labels, weights);
  check_out(dx, x->shape, "dx");
  const ck_shape& s = x->shape;
  h->last_classes = s.c;
  softmaxlog_backward(x->data, labels->data, weights ? weights->data : nullptr, p, nullptr,
                      dx->data, h->flag, (int)(s.h * s.w), (int)s.c, (int)s.n, accumulate,
                      (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

ck_status ck_loss_metrics(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                          const ck_tensor* weights, int64_t top_k, float* top1_err,
                          float* topk_err, ck_stream stream) {
  CK_API_BEGIN(h)
  check_loss(x, labels, weights);
  if (!top1_err || !topk_err) throw Err(CK_ERR_ARG, "null metric pointer");
  const ck_shape& s = x->shape;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t sites = s.h * s.w * s.n;
  float* site = (float*)h->scratch.get(sizeof(float) * 2 * sites, st);
  if (!site) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  h->last_classes = s.c;
  loss_metrics(x->data, labels->data, weights ? weights->data : nullptr, (int)top_k, site,
               top1_err, topk_err, h->flag, (int)(s.h * s.w), (int)s.c, (int)s.n, st);
  after_launch();
  CK_API_END(h)
}

ck_status ck_check_labels(ck_handle* h, ck_stream stream) {
  CK_API_BEGIN(h)
  read_label_flag(h, (cudaStream_t)stream);
  CK_API_END(h)
}

ck_status ck_sgd_step(ck_handle* h, float* w, float* v, const float* g, int64_t n, float lr,
                      float momentum, float weight_decay, ck_stream stream) {
  CK_API_BEGIN(h)
  if (n < 0 || (n > 0 && (!w || !v || !g))) throw Err(CK_ERR_ARG, "sgd: bad arguments");
  sgd_step(w, v, g, n, lr, momentum, weight_decay, (cudaStream_t)stream);
  after_launch();
  CK_API_END(h)
}

}  // extern "C"
