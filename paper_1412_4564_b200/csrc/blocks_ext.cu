// blocks_ext.cu -- the rest of the reference's block set on the device:
// sigmoid (activation.cpp:25-48), channel softmax (normalize.cpp:309-347),
// spatial normalisation (normalize.cpp:29-42, :268-306), the bilinear grid
// sampler (bilinear.cpp:58-132), pdist (loss.cpp:346-428) and every loss kind
// other than softmaxlog (loss.cpp:86-343).  All tensors are HWCN fp32
// (tensor.hpp:70-72).
//
// These are memory-bound, off the AlexNet hot path.  Layout choices:
//   * element-wise work (sigmoid, attribute losses) is a grid-stride loop;
//   * per-site reductions over channels (softmax, pdist, classification
//     losses) run one thread per site when sites are many and contiguous
//     (H*W >= 32: adjacent threads read adjacent pixels of a channel plane, so
//     every channel step is one coalesced row), one warp per site otherwise
//     (the fc case, H = W = 1: lanes split the channels);
//   * windowed work (spnorm) gathers its window directly: windows are small
//     and overlapping reads hit L1.
// Float operations the reference performs in sequence are issued as
// explicitly rounded intrinsics in the reference's order wherever the
// reference's result is reproducible that way (sigmoid backward, softmax
// backward, spnorm's pooling, bilinear forward and grid gradient, pdist with
// p in {1, 2}); transcendental calls (expf / logf / powf) may differ from
// glibc's in the last ulp.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "ck_handle.hpp"
#include "ck_internal.hpp"

namespace ck {
namespace {

constexpr int kSMs = 148;

inline int grid_for(int64_t n, int threads, int per_sm = 16) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)kSMs * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

#define GRID_STRIDE(i, n)                                                      \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ float warp_maxf(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------- sigmoid ----
// activation.cpp:25-38: split on the sign so the exponential never overflows.
__global__ void sigmoid_fwd_k(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  ck::pdl_entry();
  GRID_STRIDE(k, n) {
    const float v = x[k];
    float r;
    if (v >= 0.f) {
      r = __fdiv_rn(1.f, __fadd_rn(1.f, expf(-v)));
    } else {
      const float e = expf(v);
      r = __fdiv_rn(e, __fadd_rn(1.f, e));
    }
    y[k] = r;
  }
}

// activation.cpp:41-48: dx = dy * y * (1 - y), from the forward OUTPUT.
template <bool kAcc>
__global__ void sigmoid_bwd_k(const float* __restrict__ y, const float* __restrict__ dy, float* dx,
                              int64_t n) {
  ck::pdl_entry();
  GRID_STRIDE(k, n) {
    const float yv = y[k];
    const float r = __fmul_rn(__fmul_rn(dy[k], yv), __fsub_rn(1.f, yv));
    dx[k] = kAcc ? __fadd_rn(dx[k], r) : r;
  }
}

// ------------------------------------------------------------- softmax ----
// normalize.cpp:309-328: per site, y_k = exp(x_k - max) / sum_k exp(x_k - max).
// One thread per site (HW >= 32): the channel loops walk planes HW apart.
__global__ void softmax_fwd_thread_k(const float* __restrict__ x, float* __restrict__ y, int HW,
                                     int C, int64_t sites) {
  ck::pdl_entry();
  GRID_STRIDE(s, sites) {
    const int64_t n = s / HW, p = s % HW;
    const float* xs = x + n * (int64_t)C * HW + p;
    float* ys = y + n * (int64_t)C * HW + p;
    float mx = xs[0];
    for (int k = 1; k < C; ++k) mx = fmaxf(mx, xs[(int64_t)k * HW]);
    float sum = 0.f;
    for (int k = 0; k < C; ++k) {
      const float e = expf(__fsub_rn(xs[(int64_t)k * HW], mx));
      ys[(int64_t)k * HW] = e;
      sum = __fadd_rn(sum, e);
    }
    for (int k = 0; k < C; ++k) ys[(int64_t)k * HW] = __fdiv_rn(ys[(int64_t)k * HW], sum);
  }
}

// One warp per site (few sites, e.g. H = W = 1): lanes split the channels.
__global__ void softmax_fwd_warp_k(const float* __restrict__ x, float* __restrict__ y, int HW,
                                   int C, int64_t sites) {
  ck::pdl_entry();
  const int lane = threadIdx.x % 32;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < sites;
       s += (int64_t)gridDim.x * blockDim.x / 32) {
    const int64_t n = s / HW, p = s % HW;
    const float* xs = x + n * (int64_t)C * HW + p;
    float* ys = y + n * (int64_t)C * HW + p;
    float mx = -INFINITY;
    for (int k = lane; k < C; k += 32) mx = fmaxf(mx, xs[(int64_t)k * HW]);
    mx = warp_maxf(mx);
    float sum = 0.f;
    for (int k = lane; k < C; k += 32) {
      const float e = expf(__fsub_rn(xs[(int64_t)k * HW], mx));
      ys[(int64_t)k * HW] = e;
      sum = __fadd_rn(sum, e);
    }
    sum = warp_sum_f(sum);
    __syncwarp();
    for (int k = lane; k < C; k += 32) ys[(int64_t)k * HW] = __fdiv_rn(ys[(int64_t)k * HW], sum);
  }
}

// normalize.cpp:330-347: dx_k = y_k (dy_k - sum_j dy_j y_j), from the OUTPUT.
template <bool kAcc>
__global__ void softmax_bwd_thread_k(const float* __restrict__ y, const float* __restrict__ dy,
                                     float* dx, int HW, int C, int64_t sites) {
  ck::pdl_entry();
  GRID_STRIDE(s, sites) {
    const int64_t n = s / HW, p = s % HW;
    const int64_t o = n * (int64_t)C * HW + p;
    float dot = 0.f;
    for (int k = 0; k < C; ++k)
      dot = __fadd_rn(dot, __fmul_rn(dy[o + (int64_t)k * HW], y[o + (int64_t)k * HW]));
    for (int k = 0; k < C; ++k) {
      const int64_t e = o + (int64_t)k * HW;
      const float r = __fmul_rn(y[e], __fsub_rn(dy[e], dot));
      dx[e] = kAcc ? __fadd_rn(dx[e], r) : r;
    }
  }
}

template <bool kAcc>
__global__ void softmax_bwd_warp_k(const float* __restrict__ y, const float* __restrict__ dy,
                                   float* dx, int HW, int C, int64_t sites) {
  ck::pdl_entry();
  const int lane = threadIdx.x % 32;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < sites;
       s += (int64_t)gridDim.x * blockDim.x / 32) {
    const int64_t n = s / HW, p = s % HW;
    const int64_t o = n * (int64_t)C * HW + p;
    float dot = 0.f;
    for (int k = lane; k < C; k += 32)
      dot = __fadd_rn(dot, __fmul_rn(dy[o + (int64_t)k * HW], y[o + (int64_t)k * HW]));
    dot = warp_sum_f(dot);
    for (int k = lane; k < C; k += 32) {
      const int64_t e = o + (int64_t)k * HW;
      const float r = __fmul_rn(y[e], __fsub_rn(dy[e], dot));
      dx[e] = kAcc ? __fadd_rn(dx[e], r) : r;
    }
  }
}

// -------------------------------------------------------------- spnorm ----
// normalize.cpp:29-42: a centred avg-pool window (stride 1, pads (w-1)/2 and
// w-1-(w-1)/2), so the energy map has the input's size.  pool.cpp:20-33
// window_at clips it to the image; pool.cpp:67-73 sums j outer, i inner.
__device__ __forceinline__ float spnorm_energy(const float* __restrict__ xp, int H, int W, int i,
                                               int j, int wh, int ww, int pt, int pl) {
  const int i0 = max(0, i - pt), i1 = min(H, i - pt + wh);
  const int j0 = max(0, j - pl), j1 = min(W, j - pl + ww);
  float sum = 0.f;
  for (int jj = j0; jj < j1; ++jj)
    for (int ii = i0; ii < i1; ++ii) {
      const float v = xp[ii + (int64_t)H * jj];
      sum = __fadd_rn(sum, __fmul_rn(v, v));
    }
  return __fdiv_rn(sum, (float)((i1 - i0) * (j1 - j0)));
}

// normalize.cpp:268-281: y = x (1 + alpha E)^-beta.
__global__ void spnorm_fwd_k(const float* __restrict__ x, float* __restrict__ y, int H, int W,
                             int64_t planes, int wh, int ww, int pt, int pl, float alpha,
                             float beta) {
  ck::pdl_entry();
  const int64_t n = (int64_t)H * W * planes;
  GRID_STRIDE(k, n) {
    const int64_t pl_ = k / ((int64_t)H * W);
    const int r = (int)(k - pl_ * H * W), i = r % H, j = r / H;
    const float E = spnorm_energy(x + pl_ * H * W, H, W, i, j, wh, ww, pt, pl);
    y[k] = __fmul_rn(x[k], powf(__fadd_rn(1.f, __fmul_rn(alpha, E)), -beta));
  }
}

// normalize.cpp:284-297, pass 1: eta = dy (1 + alpha E)^(-beta-1) x, stored
// pre-divided by its window's area (pool.cpp:113-118 "share"), and the
// forward scale P = (1 + alpha E)^-beta.
__global__ void spnorm_bwd1_k(const float* __restrict__ x, const float* __restrict__ dy,
                              float* __restrict__ share, float* __restrict__ P, int H, int W,
                              int64_t planes, int wh, int ww, int pt, int pl, float alpha,
                              float beta) {
  ck::pdl_entry();
  const int64_t n = (int64_t)H * W * planes;
  GRID_STRIDE(k, n) {
    const int64_t pl_ = k / ((int64_t)H * W);
    const int r = (int)(k - pl_ * H * W), i = r % H, j = r / H;
    const float E = spnorm_energy(x + pl_ * H * W, H, W, i, j, wh, ww, pt, pl);
    const float base = __fadd_rn(1.f, __fmul_rn(alpha, E));
    P[k] = powf(base, -beta);
    const float eta = __fmul_rn(__fmul_rn(dy[k], powf(base, __fsub_rn(-beta, 1.f))), x[k]);
    const int i0 = max(0, i - pt), i1 = min(H, i - pt + wh);
    const int j0 = max(0, j - pl), j1 = min(W, j - pl + ww);
    share[k] = __fdiv_rn(eta, (float)((i1 - i0) * (j1 - j0)));
  }
}

// Pass 2: spread(i, j) = sum of the shares of every window containing (i, j)
// in the reference's (oj, oi) order -- the adjoint avg-pool as a gather --
// then dx = dy P - 2 alpha beta x spread (normalize.cpp:298-304).
template <bool kAcc>
__global__ void spnorm_bwd2_k(const float* __restrict__ x, const float* __restrict__ dy,
                              const float* __restrict__ share, const float* __restrict__ P,
                              float* dx, int H, int W, int64_t planes, int wh, int ww, int pt,
                              int pl, float c2ab) {
  ck::pdl_entry();
  const int64_t n = (int64_t)H * W * planes;
  GRID_STRIDE(k, n) {
    const int64_t pl_ = k / ((int64_t)H * W);
    const int r = (int)(k - pl_ * H * W), i = r % H, j = r / H;
    const float* sp = share + pl_ * H * W;
    // outputs (oi, oj) whose window [o - p, o - p + w) contains (i, j)
    const int oi0 = max(0, i + pt - wh + 1), oi1 = min(H - 1, i + pt);
    const int oj0 = max(0, j + pl - ww + 1), oj1 = min(W - 1, j + pl);
    float spread = 0.f;
    for (int oj = oj0; oj <= oj1; ++oj)
      for (int oi = oi0; oi <= oi1; ++oi) spread = __fadd_rn(spread, sp[oi + (int64_t)H * oj]);
    const float v = __fsub_rn(__fmul_rn(dy[k], P[k]), __fmul_rn(__fmul_rn(c2ab, x[k]), spread));
    dx[k] = kAcc ? __fadd_rn(dx[k], v) : v;
  }
}

// ------------------------------------------------------------ bilinear ----
// bilinear.cpp:17-37 tent_at: the two integer support points of v and their
// weights max(0, 1 - |v - i|) (0 outside the image) and weight derivatives.
struct Tent {
  int i0, i1;
  float w0, w1, d0, d1;
};
__device__ __forceinline__ void tent_eval(float v, int i, int extent, float& w, float& d) {
  if (i < 0 || i >= extent) {
    w = 0.f;
    d = 0.f;
    return;
  }
  const float t = __fsub_rn(v, (float)i);
  const float a = fabsf(t);
  w = a < 1.f ? __fsub_rn(1.f, a) : 0.f;
  d = (a < 1.f && t != 0.f) ? (t > 0.f ? -1.f : 1.f) : 0.f;
}
__device__ __forceinline__ Tent tent_at(float v, int extent) {
  Tent s;
  const float f = floorf(v);
  // (v is finite on any sensible grid; clamp keeps the int conversion defined)
  s.i0 = (int)fminf(fmaxf(f, -4.f), 2147483000.f);
  s.i1 = s.i0 + 1;
  tent_eval(v, s.i0, extent, s.w0, s.d0);
  tent_eval(v, s.i1, extent, s.w1, s.d1);
  return s;
}

// bilinear.cpp:58-89, one thread per output element (oi, oj, c, n).
__global__ void bilinear_fwd_k(const float* __restrict__ x, const float* __restrict__ grid,
                               float* __restrict__ y, int H, int W, int C, int OH, int OW,
                               int64_t n_out, float av, float au) {
  ck::pdl_entry();
  GRID_STRIDE(e, n_out) {
    const int oi = (int)(e % OH);
    int64_t t = e / OH;
    const int oj = (int)(t % OW);
    t /= OW;
    const int c = (int)(t % C);
    const int64_t n = t / C;
    const int64_t gsite = 2 * (oi + (int64_t)OH * (oj + (int64_t)OW * n));
    const float v = __fmul_rn(av, __fadd_rn(grid[gsite], 1.f));
    const float u = __fmul_rn(au, __fadd_rn(grid[gsite + 1], 1.f));
    const Tent sv = tent_at(v, H), su = tent_at(u, W);
    const float* xp = x + ((int64_t)n * C + c) * H * W;
    float acc = 0.f;
    if (sv.w0 != 0.f && su.w0 != 0.f)
      acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(xp[sv.i0 + (int64_t)H * su.i0], sv.w0), su.w0));
    if (sv.w1 != 0.f && su.w0 != 0.f)
      acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(xp[sv.i1 + (int64_t)H * su.i0], sv.w1), su.w0));
    if (sv.w0 != 0.f && su.w1 != 0.f)
      acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(xp[sv.i0 + (int64_t)H * su.i1], sv.w0), su.w1));
    if (sv.w1 != 0.f && su.w1 != 0.f)
      acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(xp[sv.i1 + (int64_t)H * su.i1], sv.w1), su.w1));
    y[e] = acc;
  }
}

// bilinear.cpp:92-132, one thread per output site (oi, oj, n): the grid
// derivative is a per-site sum over channels (reference order, exact);
// dx is a scatter -- several sites may hit one input pixel -- done with
// atomicAdd into a zeroed (or accumulated) dx, so its summation order is not
// the reference's (within float rounding of it, not bit-exact).
template <bool kAcc>
__global__ void bilinear_bwd_k(const float* __restrict__ x, const float* __restrict__ grid,
                               const float* __restrict__ dy, float* dx, float* dgrid, int H,
                               int W, int C, int OH, int OW, int64_t sites, float av, float au) {
  ck::pdl_entry();
  GRID_STRIDE(s, sites) {
    const int oi = (int)(s % OH);
    const int64_t t = s / OH;
    const int oj = (int)(t % OW);
    const int64_t n = t / OW;
    const int64_t gsite = 2 * s;
    const float v = __fmul_rn(av, __fadd_rn(grid[gsite], 1.f));
    const float u = __fmul_rn(au, __fadd_rn(grid[gsite + 1], 1.f));
    const Tent sv = tent_at(v, H), su = tent_at(u, W);
    float g1 = 0.f, g2 = 0.f;
    for (int c = 0; c < C; ++c) {
      const float p = dy[oi + (int64_t)OH * (oj + (int64_t)OW * (c + (int64_t)C * n))];
      if (p == 0.f && !dgrid) continue;
      const float* xp = x + ((int64_t)n * C + c) * H * W;
      float* dxp = dx ? dx + ((int64_t)n * C + c) * H * W : nullptr;
      auto tap = [&](int i, int j, float wv, float wu, float dv, float du) {
        if (i < 0 || i >= H || j < 0 || j >= W) return;
        const float xv = xp[i + (int64_t)H * j];
        if (dxp) atomicAdd(dxp + i + (int64_t)H * j, __fmul_rn(__fmul_rn(p, wv), wu));
        g1 = __fadd_rn(g1, __fmul_rn(__fmul_rn(__fmul_rn(p, xv), dv), wu));
        g2 = __fadd_rn(g2, __fmul_rn(__fmul_rn(__fmul_rn(p, xv), wv), du));
      };
      tap(sv.i0, su.i0, sv.w0, su.w0, sv.d0, su.d0);
      tap(sv.i1, su.i0, sv.w1, su.w0, sv.d1, su.d0);
      tap(sv.i0, su.i1, sv.w0, su.w1, sv.d0, su.d1);
      tap(sv.i1, su.i1, sv.w1, su.w1, sv.d1, su.d1);
    }
    if (dgrid) {
      const float a = __fmul_rn(av, g1), b = __fmul_rn(au, g2);
      dgrid[gsite] = kAcc ? __fadd_rn(dgrid[gsite], a) : a;
      dgrid[gsite + 1] = kAcc ? __fadd_rn(dgrid[gsite + 1], b) : b;
    }
  }
}

// --------------------------------------------------------------- pdist ----
// loss.cpp:346-371: y = (sum_d |x_d - t_d|^p)^(1/p) per site (no_root: the sum).
__device__ __forceinline__ float pdist_site(const float* __restrict__ x,
                                            const float* __restrict__ t, int64_t o, int HW, int C,
                                            int pk, float tp) {
  float acc = 0.f;
  for (int d = 0; d < C; ++d) {
    const float diff = fabsf(__fsub_rn(x[o + (int64_t)d * HW], t[o + (int64_t)d * HW]));
    if (pk == 1)
      acc = __fadd_rn(acc, diff);
    else if (pk == 2)
      acc = __fadd_rn(acc, __fmul_rn(diff, diff));
    else
      acc = __fadd_rn(acc, powf(diff, tp));
  }
  return acc;
}

__global__ void pdist_fwd_k(const float* __restrict__ x, const float* __restrict__ t,
                            float* __restrict__ y, int HW, int C, int64_t sites, int pk, float tp,
                            float inv_p, int no_root) {
  ck::pdl_entry();
  GRID_STRIDE(s, sites) {
    const int64_t n = s / HW, p = s % HW;
    const float acc = pdist_site(x, t, n * (int64_t)C * HW + p, HW, C, pk, tp);
    y[s] = no_root ? acc : powf(acc, inv_p);
  }
}

// loss.cpp:374-428: the (sub)gradient per element, dtarget = -dx.
template <bool kAcc>
__global__ void pdist_bwd_k(const float* __restrict__ x, const float* __restrict__ t,
                            const float* __restrict__ dy, float* dx, float* dt, int HW, int C,
                            int64_t sites, int pk, float tp, float inv_p, int no_root) {
  ck::pdl_entry();
  GRID_STRIDE(s, sites) {
    const int64_t n = s / HW, p = s % HW;
    const int64_t o = n * (int64_t)C * HW + p;
    const float acc = pdist_site(x, t, o, HW, C, pk, tp);
    const float yv = no_root ? acc : powf(acc, inv_p);
    const float g = dy[s];
    for (int d = 0; d < C; ++d) {
      const int64_t e = o + (int64_t)d * HW;
      const float diff = __fsub_rn(x[e], t[e]);
      const float sgn = diff > 0.f ? 1.f : (diff < 0.f ? -1.f : 0.f);
      const float a = fabsf(diff);
      float v;
      if (no_root) {
        if (pk == 1)
          v = sgn;
        else if (pk == 2)
          v = __fmul_rn(2.f, diff);
        else
          v = __fmul_rn(__fmul_rn(tp, powf(a, __fsub_rn(tp, 1.f))), sgn);
      } else {
        if (yv == 0.f)
          v = 0.f;  // coincident vectors: the zero subgradient
        else if (pk == 1)
          v = sgn;
        else if (pk == 2)
          v = __fdiv_rn(diff, yv);
        else
          v = __fdiv_rn(__fmul_rn(powf(a, __fsub_rn(tp, 1.f)), sgn), powf(yv, __fsub_rn(tp, 1.f)));
      }
      const float gr = __fmul_rn(g, v);
      if (dx) dx[e] = kAcc ? __fadd_rn(dx[e], gr) : gr;
      if (dt) dt[e] = kAcc ? __fsub_rn(dt[e], gr) : -gr;
    }
  }
}

// -------------------------------------------------------------- losses ----
// Label decoding (loss.cpp:14-18 as_label; :101-106 class range; :196-200
// attribute range) with the same device flag bits as kernels.cu read_label:
// 1 non-integer class, 2 class out of range (first label in flag[1]),
// 4 log loss on a non-positive score, 8 non-integer attribute, 16 attribute
// not in {-1, 0, 1}, 32 binarylog input outside [0, 1].
__device__ __forceinline__ int class_label(float v, int C, int* flag) {
  const float r = nearbyintf(v);
  if (r != v) {
    atomicOr(flag, 1);
    return 0;
  }
  if (fabsf(r) > 1e9f) {
    atomicOr(flag, 2);
    atomicCAS(flag + 1, 0, 2147483647);
    return 0;
  }
  const int c = (int)r;
  if (c != 0 && (c < 1 || c > C)) {
    atomicOr(flag, 2);
    atomicCAS(flag + 1, 0, c);
    return 0;
  }
  return c;
}
__device__ __forceinline__ int attr_label(float v, int* flag) {
  const float r = nearbyintf(v);
  if (r != v) {
    atomicOr(flag, 8);
    return 0;
  }
  if (r != 0.f && r != 1.f && r != -1.f) {
    atomicOr(flag, 16);
    return 0;
  }
  return (int)r;
}

// loss.cpp:20-25 (the stateless splitmix64 step used for random ties)
__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Kinds (ck_loss_kind): 0 classerror 1 topk 2 log 3 softmaxlog 4 mhinge
// 5 mshinge 6 binaryerror 7 binarylog 8 logistic 9 hinge.
struct LossOpts {
  int top_k;
  float threshold;
  int random_ties;
  uint64_t tie_seed;
};

// loss.cpp:96-180, one thread per site: the weighted per-site penalty.
__global__ void cls_loss_fwd_k(const float* __restrict__ x, const float* __restrict__ labels,
                               const float* __restrict__ weights, float* site, int* flag, int H,
                               int W, int C, int64_t sites, int kind, LossOpts o) {
  ck::pdl_entry();
  const int HW = H * W;
  GRID_STRIDE(s, sites) {
    const int64_t n = s / HW, pix = s % HW;
    const int c = class_label(labels[s], C, flag);
    float l = 0.f;
    if (c > 0) {
      const float* xs = x + n * (int64_t)C * HW + pix;
      const float xc = xs[(int64_t)(c - 1) * HW];
      switch (kind) {
        case 0: {  // classerror (:111-141)
          int best = 0;
          float bv = xs[0];
          if (o.random_ties) {
            int64_t ties = 1;
            // x.index(i, j, 0, n) = pix + HW * C * n
            uint64_t h = splitmix(o.tie_seed ^ (uint64_t)(pix + (int64_t)HW * C * n));
            for (int k = 1; k < C; ++k) {
              const float v = xs[(int64_t)k * HW];
              if (v > bv) {
                bv = v;
                best = k;
                ties = 1;
              } else if (v == bv) {
                ++ties;
                h = splitmix(h);
                if (h % (uint64_t)ties == 0) best = k;
              }
            }
          } else {
            for (int k = 1; k < C; ++k) {
              const float v = xs[(int64_t)k * HW];
              if (v > bv) {
                bv = v;
                best = k;
              }
            }
          }
          l = best == c - 1 ? 0.f : 1.f;
          break;
        }
        case 1: {  // topk (:142-149)
          int rank = 0;
          for (int k = 0; k < C; ++k) rank += xs[(int64_t)k * HW] >= xc;
          l = rank <= o.top_k ? 0.f : 1.f;
          break;
        }
        case 2:  // log (:150-155)
          if (!(xc > 0.f)) {
            atomicOr(flag, 4);
          } else {
            l = -logf(xc);
          }
          break;
        case 4:  // mhinge (:166-168)
          l = fmaxf(0.f, __fsub_rn(1.f, xc));
          break;
        case 5: {  // mshinge (:169-178)
          float other = -INFINITY;
          for (int k = 0; k < C; ++k)
            if (k != c - 1) other = fmaxf(other, xs[(int64_t)k * HW]);
          if (C == 1) other = 0.f;
          l = fmaxf(0.f, __fadd_rn(__fsub_rn(1.f, xc), other));
          break;
        }
        default:
          break;
      }
      l = __fmul_rn(weights ? weights[s] : 1.f, l);
    }
    site[s] = l;
  }
}

// loss.cpp:187-226, one thread per element: attribute kinds.
__global__ void attr_loss_fwd_k(const float* __restrict__ x, const float* __restrict__ labels,
                                const float* __restrict__ weights, float* site, int* flag,
                                int64_t n, int kind, float threshold) {
  ck::pdl_entry();
  GRID_STRIDE(k, n) {
    const int c = attr_label(labels[k], flag);
    float l = 0.f;
    if (c != 0) {
      const float v = x[k], cv = (float)c;
      switch (kind) {
        case 6: {  // binaryerror
          const float sgn = __fsub_rn(v, threshold) >= 0.f ? 1.f : -1.f;
          l = sgn == cv ? 0.f : 1.f;
          break;
        }
        case 7:  // binarylog
          if (v < 0.f || v > 1.f) {
            atomicOr(flag, 32);
          } else {
            l = -logf(__fadd_rn(__fmul_rn(cv, __fsub_rn(v, 0.5f)), 0.5f));
          }
          break;
        case 8: {  // logistic: stable log1p(exp(-c v)) (:27-31)
          const float t = __fmul_rn(-cv, v);
          l = t > 0.f ? __fadd_rn(t, log1pf(expf(-t))) : log1pf(expf(t));
          break;
        }
        case 9:  // hinge
          l = fmaxf(0.f, __fsub_rn(1.f, __fmul_rn(cv, v)));
          break;
        default:
          break;
      }
      l = __fmul_rn(weights ? weights[k] : 1.f, l);
    }
    site[k] = l;
  }
}

// Deterministic fixed-order sum of per-site values, in double (one block).
__global__ void sum_values_k(const float* __restrict__ v, int64_t n, float* out) {
  ck::pdl_entry();
  __shared__ double red[32];
  double a = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += v[i];
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += red[k];
    *out = (float)t;
  }
}

// loss.cpp:246-302, one thread per site: classification kinds log, mhinge,
// mshinge (error kinds are zero everywhere, :239).  Without accumulation the
// site's channel column is written in full (zeros elsewhere).
template <bool kAcc>
__global__ void cls_loss_bwd_k(const float* __restrict__ x, const float* __restrict__ labels,
                               const float* __restrict__ weights, float pscale,
                               const float* __restrict__ pdev, float* dx, int* flag, int HW, int C,
                               int64_t sites, int kind) {
  ck::pdl_entry();
  if (pdev) pscale = *pdev;
  GRID_STRIDE(s, sites) {
    const int64_t n = s / HW, pix = s % HW;
    const float* xs = x + n * (int64_t)C * HW + pix;
    float* ds = dx + n * (int64_t)C * HW + pix;
    if (!kAcc)
      for (int k = 0; k < C; ++k) ds[(int64_t)k * HW] = 0.f;
    const int c = class_label(labels[s], C, flag);
    if (c == 0) continue;
    const float scale = __fmul_rn(pscale, weights ? weights[s] : 1.f);
    const float xc = xs[(int64_t)(c - 1) * HW];
    float* dc = ds + (int64_t)(c - 1) * HW;
    switch (kind) {
      case 2:  // log (:256-262)
        if (!(xc > 0.f))
          atomicOr(flag, 4);
        else
          *dc = __fsub_rn(*dc, __fdiv_rn(scale, xc));
        break;
      case 4:  // mhinge (:275-276)
        if (xc < 1.f) *dc = __fsub_rn(*dc, scale);
        break;
      case 5: {  // mshinge (:277-293): runner-up = first strict max among the others
        int best = -1;
        float other = -INFINITY;
        for (int k = 0; k < C; ++k) {
          if (k == c - 1) continue;
          const float v = xs[(int64_t)k * HW];
          if (v > other) {
            other = v;
            best = k;
          }
        }
        if (best >= 0 && xc < __fadd_rn(1.f, other)) {
          *dc = __fsub_rn(*dc, scale);
          ds[(int64_t)best * HW] = __fadd_rn(ds[(int64_t)best * HW], scale);
        }
        break;
      }
      default:
        break;
    }
  }
}

// loss.cpp:305-340: attribute kinds binarylog, logistic, hinge.
template <bool kAcc>
__global__ void attr_loss_bwd_k(const float* __restrict__ x, const float* __restrict__ labels,
                                const float* __restrict__ weights, float pscale,
                                const float* __restrict__ pdev, float* dx, int* flag, int64_t n,
                                int kind) {
  ck::pdl_entry();
  if (pdev) pscale = *pdev;
  GRID_STRIDE(k, n) {
    const int c = attr_label(labels[k], flag);
    float r = 0.f;
    if (c != 0) {
      const float scale = __fmul_rn(pscale, weights ? weights[k] : 1.f);
      const float v = x[k], cv = (float)c;
      switch (kind) {
        case 7:  // binarylog
          if (v < 0.f || v > 1.f) {
            atomicOr(flag, 32);
          } else {
            const float q = __fadd_rn(__fmul_rn(cv, __fsub_rn(v, 0.5f)), 0.5f);
            r = __fdiv_rn(__fmul_rn(-scale, cv), q);
          }
          break;
        case 8: {  // logistic: sigma(-c v) without overflow
          const float t = __fmul_rn(-cv, v);
          float sig;
          if (t >= 0.f) {
            sig = __fdiv_rn(1.f, __fadd_rn(1.f, expf(-t)));
          } else {
            const float e = expf(t);
            sig = __fdiv_rn(e, __fadd_rn(1.f, e));
          }
          r = __fmul_rn(__fmul_rn(-scale, cv), sig);
          break;
        }
        case 9:  // hinge
          if (__fmul_rn(cv, v) < 1.f) r = __fmul_rn(-scale, cv);
          break;
        default:
          break;
      }
    }
    dx[k] = kAcc ? __fadd_rn(dx[k], r) : r;
  }
}

// y[i] = sum_k x_k[i] for a split layer's backward (graph.cpp split: dx = sum
// of the projections, in output order) with optional accumulation.
struct SumSrcs {
  const float* p[8];
};
template <bool kAcc>
__global__ void sum_into_k(float* dx, SumSrcs srcs, int m, int64_t n) {
  ck::pdl_entry();
  GRID_STRIDE(i, n) {
    float a = 0.f;
    for (int k = 0; k < m; ++k) a = __fadd_rn(a, srcs.p[k][i]);
    dx[i] = kAcc ? __fadd_rn(dx[i], a) : a;
  }
}

}  // namespace

// ------------------------------------------------------------ launchers ---

void sigmoid_forward(const float* x, float* y, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  count_launch();
  ck::pdl_launch(sigmoid_fwd_k, grid_for(n, 256), 256, 0, s, x, y, n);
}

void sigmoid_backward(const float* y, const float* dy, float* dx, int64_t n, int acc,
                      cudaStream_t s) {
  if (n == 0) return;
  count_launch();
  if (acc)
    ck::pdl_launch(sigmoid_bwd_k<true>, grid_for(n, 256), 256, 0, s, y, dy, dx, n);
  else
    ck::pdl_launch(sigmoid_bwd_k<false>, grid_for(n, 256), 256, 0, s, y, dy, dx, n);
}

void softmax_forward(const float* x, float* y, int HW, int C, int N, cudaStream_t s) {
  const int64_t sites = (int64_t)HW * N;
  if (!sites) return;
  count_launch();
  if (HW >= 32)
    ck::pdl_launch(softmax_fwd_thread_k, grid_for(sites, 128), 128, 0, s, x, y, HW, C, sites);
  else
    ck::pdl_launch(softmax_fwd_warp_k, grid_for(sites * 32, 256), 256, 0, s, x, y, HW, C, sites);
}

void softmax_backward(const float* y, const float* dy, float* dx, int HW, int C, int N, int acc,
                      cudaStream_t s) {
  const int64_t sites = (int64_t)HW * N;
  if (!sites) return;
  count_launch();
  if (HW >= 32) {
    if (acc)
      ck::pdl_launch(softmax_bwd_thread_k<true>, grid_for(sites, 128), 128, 0, s, y, dy, dx, HW, C, sites);
    else
      ck::pdl_launch(softmax_bwd_thread_k<false>, grid_for(sites, 128), 128, 0, s, y, dy, dx, HW, C, sites);
  } else {
    if (acc)
      ck::pdl_launch(softmax_bwd_warp_k<true>, grid_for(sites * 32, 256), 256, 0, s, y, dy, dx, HW, C, sites);
    else
      ck::pdl_launch(softmax_bwd_warp_k<false>, grid_for(sites * 32, 256), 256, 0, s, y, dy, dx, HW, C, sites);
  }
}

void spnorm_forward(const float* x, float* y, int H, int W, int64_t planes, int wh, int ww,
                    float alpha, float beta, cudaStream_t s) {
  const int64_t n = (int64_t)H * W * planes;
  if (!n) return;
  count_launch();
  ck::pdl_launch(spnorm_fwd_k, grid_for(n, 256), 256, 0, s, x, y, H, W, planes, wh, ww, (wh - 1) / 2,
                                                (ww - 1) / 2, alpha, beta);
}

void spnorm_backward(const float* x, const float* dy, float* dx, float* ws, int H, int W,
                     int64_t planes, int wh, int ww, float alpha, float beta, float c2ab, int acc,
                     cudaStream_t s) {
  const int64_t n = (int64_t)H * W * planes;
  if (!n) return;
  count_launch(2);
  float* share = ws;
  float* P = ws + n;
  const int pt = (wh - 1) / 2, pl = (ww - 1) / 2;
  ck::pdl_launch(spnorm_bwd1_k, grid_for(n, 256), 256, 0, s, x, dy, share, P, H, W, planes, wh, ww, pt, pl,
                                                 alpha, beta);
  if (acc)
    ck::pdl_launch(spnorm_bwd2_k<true>, grid_for(n, 256), 256, 0, s, x, dy, share, P, dx, H, W, planes, wh,
                                                         ww, pt, pl, c2ab);
  else
    ck::pdl_launch(spnorm_bwd2_k<false>, grid_for(n, 256), 256, 0, s, x, dy, share, P, dx, H, W, planes, wh,
                                                          ww, pt, pl, c2ab);
}

void bilinear_forward(const float* x, const float* grid, float* y, int H, int W, int C, int N,
                      int OH, int OW, cudaStream_t s) {
  const int64_t n = (int64_t)OH * OW * C * N;
  if (!n) return;
  count_launch();
  ck::pdl_launch(bilinear_fwd_k, grid_for(n, 256), 256, 0, s, x, grid, y, H, W, C, OH, OW, n,
                                                  (float)(H - 1) / 2.f, (float)(W - 1) / 2.f);
}

void bilinear_backward(const float* x, const float* grid, const float* dy, float* dx, float* dgrid,
                       int H, int W, int C, int N, int OH, int OW, int acc, cudaStream_t s) {
  const int64_t sites = (int64_t)OH * OW * N;
  if (dx && !acc) {
    check_cuda(cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)H * W * C * N, s), "memset");
  }
  if (!sites) return;
  count_launch();
  const float av = (float)(H - 1) / 2.f, au = (float)(W - 1) / 2.f;
  if (acc)
    ck::pdl_launch(bilinear_bwd_k<true>, grid_for(sites, 128), 128, 0, s, x, grid, dy, dx, dgrid, H, W, C, OH,
                                                              OW, sites, av, au);
  else
    ck::pdl_launch(bilinear_bwd_k<false>, grid_for(sites, 128), 128, 0, s, x, grid, dy, dx, dgrid, H, W, C, OH,
                                                               OW, sites, av, au);
}

static int pdist_kind(double p) { return p == 1.0 ? 1 : (p == 2.0 ? 2 : 0); }

void pdist_forward(const float* x, const float* t, float* y, int HW, int C, int N, double p,
                   int no_root, cudaStream_t s) {
  const int64_t sites = (int64_t)HW * N;
  if (!sites) return;
  count_launch();
  const float tp = (float)p;
  ck::pdl_launch(pdist_fwd_k, grid_for(sites, 128), 128, 0, s, x, t, y, HW, C, sites, pdist_kind(p), tp,
                                                   1.f / tp, no_root);
}

void pdist_backward(const float* x, const float* t, const float* dy, float* dx, float* dt, int HW,
                    int C, int N, double p, int no_root, int acc, cudaStream_t s) {
  const int64_t sites = (int64_t)HW * N;
  if (!sites) return;
  count_launch();
  const float tp = (float)p;
  if (acc)
    ck::pdl_launch(pdist_bwd_k<true>, grid_for(sites, 128), 128, 0, s, x, t, dy, dx, dt, HW, C, sites,
                                                           pdist_kind(p), tp, 1.f / tp, no_root);
  else
    ck::pdl_launch(pdist_bwd_k<false>, grid_for(sites, 128), 128, 0, s, x, t, dy, dx, dt, HW, C, sites,
                                                            pdist_kind(p), tp, 1.f / tp, no_root);
}

static bool attribute_kind(int kind) { return kind >= 6; }

void loss_forward_kind(const float* x, const float* labels, const float* weights, int kind,
                       int64_t top_k, double threshold, int random_ties, uint64_t tie_seed,
                       float* site, float* loss, int* flag, int H, int W, int C, int N,
                       cudaStream_t s) {
  const LossOpts o{(int)std::min<int64_t>(top_k, 2147483647), (float)threshold, random_ties,
                   tie_seed};
  count_launch(2);
  int64_t n;
  if (attribute_kind(kind)) {
    n = (int64_t)H * W * C * N;
    ck::pdl_launch(attr_loss_fwd_k, grid_for(n, 256), 256, 0, s, x, labels, weights, site, flag, n, kind,
                                                     o.threshold);
  } else {
    n = (int64_t)H * W * N;
    ck::pdl_launch(cls_loss_fwd_k, grid_for(n, 128), 128, 0, s, x, labels, weights, site, flag, H, W, C, n,
                                                    kind, o);
  }
  ck::pdl_launch(sum_values_k, 1, 1024, 0, s, site, n, loss);
}

void loss_backward_kind(const float* x, const float* labels, const float* weights, int kind,
                        float p, const float* p_dev, float* dx, int* flag, int H, int W, int C,
                        int N, int acc, cudaStream_t s) {
  const bool error_kind = kind == 0 || kind == 1 || kind == 6;
  const int64_t total = (int64_t)H * W * C * N;
  if (error_kind) {  // loss.cpp:239: exact zeros
    if (!acc) check_cuda(cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)total, s), "memset");
    return;
  }
  count_launch();
  if (attribute_kind(kind)) {
    if (acc)
      ck::pdl_launch(attr_loss_bwd_k<true>, grid_for(total, 256), 256, 0, s, x, labels, weights, p, p_dev, dx,
                                                                 flag, total, kind);
    else
      ck::pdl_launch(attr_loss_bwd_k<false>, grid_for(total, 256), 256, 0, s, x, labels, weights, p, p_dev,
                                                                  dx, flag, total, kind);
  } else {
    const int64_t sites = (int64_t)H * W * N;
    if (acc)
      ck::pdl_launch(cls_loss_bwd_k<true>, grid_for(sites, 128), 128, 0, s, x, labels, weights, p, p_dev, dx,
                                                                 flag, H * W, C, sites, kind);
    else
      ck::pdl_launch(cls_loss_bwd_k<false>, grid_for(sites, 128), 128, 0, s, x, labels, weights, p, p_dev, dx,
                                                                  flag, H * W, C, sites, kind);
  }
}

void sum_into(float* dx, const float* const* srcs, int m, int64_t n, int acc, cudaStream_t s) {
  if (!n) return;
  if (m > 8) throw Err(CK_ERR_ARG, "split: at most 8 copies");
  SumSrcs a{};
  for (int k = 0; k < m; ++k) a.p[k] = srcs[k];
  count_launch();
  if (acc)
    ck::pdl_launch(sum_into_k<true>, grid_for(n, 256), 256, 0, s, dx, a, m, n);
  else
    ck::pdl_launch(sum_into_k<false>, grid_for(n, 256), 256, 0, s, dx, a, m, n);
}

}  // namespace ck
