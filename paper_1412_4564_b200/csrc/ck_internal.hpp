// Internal declarations shared by the kernels, the C ABI and the graph
// engine.  Launchers take plain device pointers and pre-validated geometry;
// all argument checking happens in capi.cu before a launcher is called.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "ck/ck.h"

namespace ck {

// Geometry in the reference's terms (conv.hpp:9-17, pool.hpp:13-23).
struct ConvDims {
  int H, W, C, N;      // input x
  int fh, fw, Cg, K;   // filters (Cg = C / groups)
  int OH, OW;          // output
  int sh, sw, pt, pb, pl, pr, groups;
  // Filter element (fi, fj, c, k) lives at f[fi + fh*(fj + fw*(c*fsc + k*fsk))];
  // conv: fsc = 1, fsk = Cg.  convt reuses the conv kernels with the
  // "swapped bank" of conv.cpp:332-342 by exchanging the two strides.
  int64_t fsc, fsk;
#ifdef __CUDACC__
  __host__ __device__
#endif
  int Kg() const { return K / groups; }
};

struct PoolDims {
  int H, W, C, N, OH, OW;
  int wh, ww, sh, sw, pt, pl;
  int mode;  // 0 max, 1 avg
};

// Bumped whenever any Workspace frees or moves its buffer.  A captured CUDA
// graph holds raw pointers into workspaces (and TMA descriptors encoding
// them), so the trainer re-captures when the generation it captured under
// is no longer current.
uint64_t workspace_generation();

#ifdef __CUDACC__
// Programmatic dependent launch (PDL).  Every kernel of the library starts
// with pdl_entry(): it lets the next kernel in the stream be scheduled now
// (griddepcontrol.launch_dependents) and waits until every kernel it depends
// on has completed and its writes are visible (griddepcontrol.wait) -- so a
// kernel launched with the programmatic-serialization attribute (pdl_launch)
// may start, and get its CTAs resident, while its predecessor drains, without
// ever reading that predecessor's output early.  Inside a captured CUDA graph
// these become programmatic edges: the ~100 dependent launches of a training
// step no longer each pay the full launch latency.
__device__ __forceinline__ void pdl_entry() {
#ifdef CK_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
#ifndef CK_NO_PDL
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#else
  (void)attr;
#endif
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

// Tuning / experiment knobs (CK_* environment variables).  Product builds
// ignore the environment and return dflt; only a -DCK_EXPERIMENTS build reads
// them, so no variable can change what a production kernel computes.
int knob(const char* name, int dflt);
bool experiments_build();

// The x grid a stride-1 TF32 conv reads (conv_tc_xgrid_plan, ck_handle.hpp).
struct XGridPlan {
  int Hg, Wg, Cg, Cgp, groups, pt, pl;
  int64_t key;
  size_t bytes;
};

// The dy grid a TF32 conv backward consumes (dy at (0, 0) of an Hg x Wg grid,
// Kgp padded channels per group): conv_tc_grid_plan (ck_handle.hpp) says
// whether BOTH the weight and data gradient of a conv read dy only through
// that grid, and how it is laid out (key: dy_grid's cache key).
struct GridPlan {
  int Hg, Wg, Kg, Kgp, groups, OH, OW;
  int64_t key;
  size_t bytes;
};

// Per-handle scratch owned by the C ABI / engine.
struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* get(size_t want, cudaStream_t s);
  void release();
};

// A conv layer's input in the tensor-core layout (padded pixel-major grid or
// space-to-depth tensor), written by the forward and reused by the weight
// gradient of the same graph step.  Owned by the graph engine, one per conv
// layer; the engine invalidates it at the start of every forward pass.
struct ConvCache {
  Workspace buf;
  const float* src = nullptr;
  int64_t key = 0;
  bool valid = false;
  // the buffer (at zero_ptr) was zero-filled for grid layout zero_key: a
  // producer writing only the interior keeps the halos and channel pads zero
  void* zero_ptr = nullptr;
  int64_t zero_key = 0;
};

struct LaunchCounter {
  int64_t n = 0;
  int64_t tc = 0;  // of which tcgen05 tensor-core GEMM launches (tc_gemm_kernel)
};

// ---- launchers (kernels.cu / conv_simt.cu / conv_tc.cu) -------------------
extern thread_local LaunchCounter* g_counter;  // counts kernel launches

// Optional per-launch timing of the GEMM kernels (ck_set_kernel_profiling).
struct KernelProfiler {
  bool on = false;
  std::string label;  // pending label / FLOP count for the next GEMM launch
  double flops = 0;
  struct Rec {
    std::string label;
    double flops;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  void clear() {
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    recs.clear();
  }
  ~KernelProfiler() { clear(); }
};
extern thread_local KernelProfiler* g_prof;
inline void prof_next(const std::string& label, double flops) {
  if (g_prof && g_prof->on) {
    g_prof->label = label;
    g_prof->flops = flops;
  }
}
inline void count_launch(int k = 1) {
  if (g_counter) g_counter->n += k;
}
inline void count_tc_launch() {
  if (g_counter) g_counter->tc += 1;
}

void relu_forward(const float* x, float* y, int64_t n, cudaStream_t s);
// flag[0] |= bit when any of v[0..n) is not finite (trainer NaN abort)
void flag_nonfinite(const float* v, int64_t n, int* flag, int bit, cudaStream_t s);
void relu_backward(const float* x, const float* dy, float* dx, int64_t n, int acc, cudaStream_t s);
void axpy_inplace(float* y, const float* x, int64_t n, cudaStream_t s);  // y += x
void sgd_step(float* w, float* v, const float* g, int64_t n, float lr, float mom, float wd,
              cudaStream_t s);

struct ConvCache;
void pool_forward(const float* x, float* y, const PoolDims& d, cudaStream_t s,
                  ConvCache* cache = nullptr);
void pool_backward(const float* x, const float* dy, float* dx, const PoolDims& d, int acc,
                   cudaStream_t s, ConvCache* cache = nullptr);

void lrn_forward(const float* x, float* y, int H, int W, int C, int N, int size, float kappa,
                 float alpha, float beta, cudaStream_t s);
// LRN fused with the 3x3 / stride-2 max pool reading it: y = lrn(x), py =
// pool(y) and (cache) the pool's argmax for its backward.  False (nothing
// launched) outside the fused kernel's envelope.
bool lrn_maxpool_forward(const float* x, float* y, float* py, const PoolDims& pd, int size,
                         float kappa, float alpha, float beta, cudaStream_t s, ConvCache* cache);
void lrn_backward(const float* x, const float* dy, float* dx, int H, int W, int C, int N, int size,
                  float kappa, float alpha, float beta, int acc, cudaStream_t s);
// LRN backward whose output goes (ReLU-gated by x > 0) straight into the dy
// grid of the conv below the ReLU that feeds the LRN, with per-warp bias
// partials (bpart: lrn_grid_rows(H, W, N) x Kgp*groups doubles).  False when
// the LRN size has no grid kernel (3 and 5 do).
bool lrn_backward_grid(const float* x, const float* dy, float* grid, double* bpart, int H, int W,
                       int C, int N, int size, float kappa, float alpha, float beta, int Hg, int Wg,
                       int Kg, int Kgp, int groups, cudaStream_t s);
int lrn_grid_rows(int H, int W, int N);

// Per-channel sums in double: out[c] = {sum x, sum x^2, sum dy, sum dy*x}
// (dy may be null).  partial: workspace of splits*C*4 doubles.
// Gate recomputation of a fused bnorm -> relu backward: the bnorm output's
// sign from x with the forward's per-channel (mu, inv) floats (muinv, 2 per
// channel, written by bnorm_apply) and the layer's w, b.
struct BnGate {
  const float* w = nullptr;
  const float* b = nullptr;
  const float* muinv = nullptr;
};
// y = w (x - mu) inv + b from the forward's float (mu, inv) (muinv, 2 per channel)
// (relu != 0: relu of it, the fused relu output)
void bnorm_value(const float* x, const float* w, const float* b, const float* muinv, float* y,
                 int HW, int C, int N, int relu, cudaStream_t s);
// fused bnorm -> relu forward writing relu(y) into the next conv's padded
// pixel-major x grid (XGridPlan layout) instead of HWCN; moments and (mu, inv)
// as bnorm_apply.  False outside the kernel's envelope (nothing launched).
bool bnorm_apply_grid(const float* x, const float* w, const float* b, const double* stats,
                      float* moments_out, float* muinv_out, double eps, int H, int W, int C, int N,
                      float* grid, int Hg, int Wg, int Cg, int Cgp, int groups, int pt, int pl,
                      cudaStream_t s);
// bnorm backward writing dx into the conv-below's dy grid (dy at (0, 0) of an
// Hg x Wg grid, Kgp channels per group) plus 32-pixel bias partials; stats from
// bnorm_stats.  False when the shape is outside the kernel's envelope.
bool bnorm_backward_grid(const float* x, const float* dy, const float* w, const double* stats,
                         double eps, int H, int W, int C, int N, float* grid, double* bpart,
                         int Hg, int Wg, int Kg, int Kgp, int groups, cudaStream_t s,
                         const float* gate, const BnGate& rg, float* dw, float* db, int acc);
void bnorm_stats(const float* x, const float* dy, double* partial, double* out, int HW, int C,
                 int N, int splits, cudaStream_t s, const float* gate = nullptr,
                 const BnGate& rg = BnGate{});
int bnorm_splits(int HW, int C, int N);
// y2 != null: also relu(y) (fused bnorm -> relu); muinv_out: the (mu, inv)
// floats of every channel, for the backward's gate recomputation
void bnorm_apply(const float* x, const float* w, const float* b, const double* stats,
                 const float* fixed_moments, float* y, float* moments_out, double eps, int HW,
                 int C, int N, cudaStream_t s, float* y2 = nullptr, float* muinv_out = nullptr);
// gate != null (fused bnorm -> relu backward): the derivative reaching the
// bnorm output is gate > 0 ? dy : 0 (gate = bnorm output, dy = relu output's);
// rg.muinv != null: the gate recomputed from x instead of read
void bnorm_backward_apply(const float* x, const float* dy, const float* w, const double* stats,
                          double eps, float* dx, float* dw, float* db, int HW, int C, int N,
                          int acc, cudaStream_t s, const float* gate = nullptr,
                          const BnGate& rg = BnGate{});

// softmaxlog: per-site loss into site_loss, then a fixed-order sum into loss.
void softmaxlog_forward(const float* x, const float* labels, const float* weights,
                        float* site_loss, float* loss, int* flag, int HW, int C, int N,
                        cudaStream_t s);
// p_dev (nullable): the projection read on the device instead of p.
void softmaxlog_backward(const float* x, const float* labels, const float* weights, float p,
                         const float* p_dev, float* dx, int* flag, int HW, int C, int N, int acc,
                         cudaStream_t s);
void loss_metrics(const float* x, const float* labels, const float* weights, int top_k,
                  float* site_buf, float* top1, float* topk, int* flag, int HW, int C, int N,
                  cudaStream_t s);

// ---- the rest of the block set (blocks_ext.cu) -----------------------------
void sigmoid_forward(const float* x, float* y, int64_t n, cudaStream_t s);
void sigmoid_backward(const float* y, const float* dy, float* dx, int64_t n, int acc,
                      cudaStream_t s);
void softmax_forward(const float* x, float* y, int HW, int C, int N, cudaStream_t s);
void softmax_backward(const float* y, const float* dy, float* dx, int HW, int C, int N, int acc,
                      cudaStream_t s);
void spnorm_forward(const float* x, float* y, int H, int W, int64_t planes, int wh, int ww,
                    float alpha, float beta, cudaStream_t s);
// ws: 2 * H*W*planes floats
void spnorm_backward(const float* x, const float* dy, float* dx, float* ws, int H, int W,
                     int64_t planes, int wh, int ww, float alpha, float beta, float c2ab, int acc,
                     cudaStream_t s);
void bilinear_forward(const float* x, const float* grid, float* y, int H, int W, int C, int N,
                      int OH, int OW, cudaStream_t s);
void bilinear_backward(const float* x, const float* grid, const float* dy, float* dx, float* dgrid,
                       int H, int W, int C, int N, int OH, int OW, int acc, cudaStream_t s);
void pdist_forward(const float* x, const float* t, float* y, int HW, int C, int N, double p,
                   int no_root, cudaStream_t s);
void pdist_backward(const float* x, const float* t, const float* dy, float* dx, float* dt, int HW,
                    int C, int N, double p, int no_root, int acc, cudaStream_t s);
// every loss kind but softmaxlog (ck_loss_kind numbering); site: per-site
// (classification) or per-element (attribute) scratch
void loss_forward_kind(const float* x, const float* labels, const float* weights, int kind,
                       int64_t top_k, double threshold, int random_ties, uint64_t tie_seed,
                       float* site, float* loss, int* flag, int H, int W, int C, int N,
                       cudaStream_t s);
void loss_backward_kind(const float* x, const float* labels, const float* weights, int kind,
                        float p, const float* p_dev, float* dx, int* flag, int H, int W, int C,
                        int N, int acc, cudaStream_t s);
// dx (+)= sum_k srcs[k] (k < m <= 8), in order
void sum_into(float* dx, const float* const* srcs, int m, int64_t n, int acc, cudaStream_t s);

// ---- convolution -----------------------------------------------------------
// All conv launchers compute the reference semantics of conv.cpp:193-280 on
// HWCN tensors; bias may be null; acc != 0 adds into the destination.
// FP32 (SIMT FFMA) verification path:
void conv_fwd_fp32(const float* x, const float* f, const float* bias, float* y,
                   const ConvDims& d, int relu, cudaStream_t s);
void conv_dgrad_fp32(const float* dy, const float* f, float* dx, const ConvDims& d, int acc,
                     cudaStream_t s);
// wgrad uses `ws` (>= conv_wgrad_ws_bytes) for the split-K partials.
size_t conv_wgrad_ws_bytes(const ConvDims& d);
void conv_wgrad_fp32(const float* x, const float* dy, float* df, const ConvDims& d, int acc,
                     void* ws, cudaStream_t s);
size_t conv_bgrad_ws_bytes(int K, int N, int OHW);
void conv_bgrad(const float* dy, float* db, int OHW, int K, int N, int acc, void* ws,
                cudaStream_t s);

// TF32 tensor-core path (tcgen05).  Returns false when the shape is outside
// the kernel's envelope so the caller can use the FP32 kernel instead.
bool conv_tc_available();

}  // namespace ck
