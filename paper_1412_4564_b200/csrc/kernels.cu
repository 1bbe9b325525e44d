// Memory-bound block kernels for sm_100a: ReLU, pooling, LRN, batch norm,
// softmaxlog loss, SGD.  All tensors are HWCN fp32 (tensor.hpp:70-72).
//
// Parity notes (see tests/test_gpu_blocks.py):
//  * relu, max/avg pooling, SGD: bit-exact with the reference CPU path.  Every
//    float operation the reference performs is issued as an explicitly
//    rounded intrinsic (__fadd_rn / __fmul_rn / __fdiv_rn) so nvcc cannot
//    contract it into an FMA, and reductions run in the reference's order.
//  * LRN uses the same explicit rounding; powf may differ from glibc's in the
//    last ulp, so parity there is within 1e-6 relative.
//  * bnorm and the loss reduce in double with a fixed, deterministic tree.
#include <cuda_runtime.h>

#include <cstdint>

#include "ck_internal.hpp"

namespace ck {

thread_local LaunchCounter* g_counter = nullptr;
thread_local KernelProfiler* g_prof = nullptr;

namespace {

constexpr int kSMs = 148;

inline int blocks_for(int64_t n, int threads, int per_sm = 16) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)kSMs * per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// x^e as __powf computes it, ex2(e * lg2(x)), minus __powf's subnormal
// argument / result scaling: the same bits whenever x and x^e are normal
// floats.  The LRN kernels below use it only when kappa >= FLT_MIN and
// alpha >= 0 (L = kappa + alpha * sum >= kappa is normal) and beta <= 0.98
// (L^-beta >= 2^-126 for every finite L) -- lrn_pow_fast_ok() on the host.
__device__ __forceinline__ float pow_normal(float x, float e) {
  float l, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fmul_rn(l, e)));
  return r;
}

inline bool lrn_pow_fast_ok(float kappa, float alpha, float beta) {
  return kappa >= 1.17549435e-38f && alpha >= 0.f && beta <= 0.98f;
}

// ---------------------------------------------------------------- ReLU ----
// activation.cpp:8-12 (y = x > 0 ? x : 0) and :15-22 (dx = x > 0 ? dy : 0).

__global__ void relu_fwd_v4(const float4* __restrict__ x, float4* __restrict__ y, int64_t n4) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = x[i];
    v.x = v.x > 0.f ? v.x : 0.f;
    v.y = v.y > 0.f ? v.y : 0.f;
    v.z = v.z > 0.f ? v.z : 0.f;
    v.w = v.w > 0.f ? v.w : 0.f;
    y[i] = v;
  }
}

__global__ void relu_fwd_s(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] > 0.f ? x[i] : 0.f;
}

template <bool kAcc>
__global__ void relu_bwd_v4(const float4* __restrict__ x, const float4* __restrict__ dy,
                            float4* dx, int64_t n4) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = x[i], g = dy[i], r;
    r.x = a.x > 0.f ? g.x : 0.f;
    r.y = a.y > 0.f ? g.y : 0.f;
    r.z = a.z > 0.f ? g.z : 0.f;
    r.w = a.w > 0.f ? g.w : 0.f;
    if (kAcc) {
      float4 o = dx[i];
      r.x = __fadd_rn(o.x, r.x);
      r.y = __fadd_rn(o.y, r.y);
      r.z = __fadd_rn(o.z, r.z);
      r.w = __fadd_rn(o.w, r.w);
    }
    dx[i] = r;
  }
}

template <bool kAcc>
__global__ void relu_bwd_s(const float* __restrict__ x, const float* __restrict__ dy, float* dx,
                           int64_t n) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float r = x[i] > 0.f ? dy[i] : 0.f;
    dx[i] = kAcc ? __fadd_rn(dx[i], r) : r;
  }
}

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// --------------------------------------------------------- axpy / SGD -----

__global__ void axpy_k(float* y, const float* __restrict__ x, int64_t n) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __fadd_rn(y[i], x[i]);
}

// SPEC.md:706 v <- m v - lr (g + wd w); w <- w + v, each product/sum rounded
// exactly as the scalar C++ expression (no FMA contraction).
__global__ void sgd_k(float* w, float* v, const float* __restrict__ g, int64_t n, float lr,
                      float mom, float wd) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float wi = w[i];
    float t = __fadd_rn(g[i], __fmul_rn(wd, wi));
    float vi = __fadd_rn(__fmul_rn(mom, v[i]), -__fmul_rn(lr, t));
    v[i] = vi;
    w[i] = __fadd_rn(wi, vi);
  }
}

// float4 variant (16-byte aligned arrays, n % 4 == 0): same rounding per lane.
__global__ void sgd_v4_k(float4* w, float4* v, const float4* __restrict__ g, int64_t n4,
                         float lr, float mom, float wd) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 wi = w[i], vi0 = v[i], gi = __ldg(g + i);
    float4 vo, wo;
#define CK_SGD_LANE(c)                                                        \
  {                                                                           \
    const float t = __fadd_rn(gi.c, __fmul_rn(wd, wi.c));                     \
    vo.c = __fadd_rn(__fmul_rn(mom, vi0.c), -__fmul_rn(lr, t));               \
    wo.c = __fadd_rn(wi.c, vo.c);                                             \
  }
    CK_SGD_LANE(x) CK_SGD_LANE(y) CK_SGD_LANE(z) CK_SGD_LANE(w)
#undef CK_SGD_LANE
    v[i] = vo;
    w[i] = wo;
  }
}

// ------------------------------------------------------------- pooling ----
// pool.cpp:24-32 window_at: the window is clipped to the real signal.
struct Win {
  int i0, i1, j0, j1;
};
__device__ __forceinline__ Win window_at(const PoolDims& d, int oi, int oj) {
  Win b;
  int si = d.sh * oi - d.pt, sj = d.sw * oj - d.pl;
  b.i0 = max(0, si);
  b.i1 = min(d.H, si + d.wh);
  b.j0 = max(0, sj);
  b.j1 = min(d.W, sj + d.ww);
  return b;
}

// One thread per output element, consecutive threads along H (coalesced).
// max: first strict maximum in j-outer / i-inner order (pool.cpp:58-66).
// avg: sum in the same order, divided by the clipped area (pool.cpp:67-74).
__global__ void pool_fwd_k(const float* __restrict__ x, float* __restrict__ y, PoolDims d) {
  ck::pdl_entry();
  const int64_t total = (int64_t)d.OH * d.OW * d.C * d.N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int oi = (int)(e % d.OH);
    int64_t r = e / d.OH;
    int oj = (int)(r % d.OW);
    int64_t plane = r / d.OW;  // c + C*n
    const float* xp = x + plane * (int64_t)d.H * d.W;
    Win b = window_at(d, oi, oj);
    float out;
    if (d.mode == 0) {
      float best = xp[b.i0 + d.H * b.j0];
      for (int j = b.j0; j < b.j1; ++j)
        for (int i = b.i0; i < b.i1; ++i) {
          float v = xp[i + d.H * j];
          if (v > best) best = v;
        }
      out = best;
    } else {
      float sum = 0.f;
      for (int j = b.j0; j < b.j1; ++j)
        for (int i = b.i0; i < b.i1; ++i) sum = __fadd_rn(sum, xp[i + d.H * j]);
      float area = (float)((b.i1 - b.i0) * (b.j1 - b.j0));
      out = __fdiv_rn(sum, area);
    }
    y[e] = out;
  }
}

// Gather form of pool.cpp:83-126: each input element sums the contributions
// of the windows that route to it, in the reference's (oj, oi) scatter order,
// starting from 0 -- so the float sum is bit-identical and needs no atomics.
template <bool kAcc>
__global__ void pool_bwd_k(const float* __restrict__ x, const float* __restrict__ dy, float* dx,
                           PoolDims d) {
  ck::pdl_entry();
  const int64_t total = (int64_t)d.H * d.W * d.C * d.N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e % d.H);
    int64_t r = e / d.H;
    int j = (int)(r % d.W);
    int64_t plane = r / d.W;
    const float* xp = x + plane * (int64_t)d.H * d.W;
    const float* dyp = dy + plane * (int64_t)d.OH * d.OW;
    // Output windows whose (unclipped) span covers i: s*oi - pt <= i < s*oi - pt + wh.
    int oi_lo = i + d.pt - d.wh + 1;
    oi_lo = oi_lo <= 0 ? 0 : (oi_lo + d.sh - 1) / d.sh;
    int oi_hi = min(d.OH - 1, (i + d.pt) / d.sh);
    int oj_lo = j + d.pl - d.ww + 1;
    oj_lo = oj_lo <= 0 ? 0 : (oj_lo + d.sw - 1) / d.sw;
    int oj_hi = min(d.OW - 1, (j + d.pl) / d.sw);
    float acc = 0.f;
    for (int oj = oj_lo; oj <= oj_hi; ++oj)
      for (int oi = oi_lo; oi <= oi_hi; ++oi) {
        Win b = window_at(d, oi, oj);
        float p = dyp[oi + d.OH * oj];
        if (d.mode == 0) {
          int bi = b.i0, bj = b.j0;
          float best = xp[b.i0 + d.H * b.j0];
          for (int jj = b.j0; jj < b.j1; ++jj)
            for (int ii = b.i0; ii < b.i1; ++ii) {
              float v = xp[ii + d.H * jj];
              if (v > best) {
                best = v;
                bi = ii;
                bj = jj;
              }
            }
          if (bi == i && bj == j) acc = __fadd_rn(acc, p);
        } else {
          float area = (float)((b.i1 - b.i0) * (b.j1 - b.j0));
          acc = __fadd_rn(acc, __fdiv_rn(p, area));
        }
      }
    dx[e] = kAcc ? __fadd_rn(dx[e], acc) : acc;
  }
}

// Plane-tiled variant: one block per (c, n) plane.  The x plane is staged in
// shared memory, each window's argmax (same first-strict-max rule) is
// computed ONCE, then every input element gathers its windows in (oj, oi)
// order -- identical float sums to pool_bwd_k, ~9x fewer loads.
template <bool kAcc>
__global__ void pool_bwd_plane_k(const float* __restrict__ x, const float* __restrict__ dy,
                                 float* dx, PoolDims d) {
  ck::pdl_entry();
  extern __shared__ float psm[];
  const int HW = d.H * d.W, OHW = d.OH * d.OW;
  float* xs = psm;                     // [HW]
  float* ds = xs + HW;                 // [OHW] dy, or dy/area for avg
  int* arg = (int*)(ds + OHW);         // [OHW] argmax (max mode)
  const int64_t plane = blockIdx.x;    // c + C*n
  const float* xp = x + plane * HW;
  const float* dyp = dy + plane * OHW;
  for (int e = threadIdx.x; e < HW; e += blockDim.x) xs[e] = xp[e];
  __syncthreads();
  // (oj, oi) and (j, i) loops: warps over columns, lanes down a column (no
  // per-element division; loads/stores coalesced along H).
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int oj = warp; oj < d.OW; oj += nw)
    for (int oi = lane; oi < d.OH; oi += 32) {
      const int w = oi + d.OH * oj;
      Win b = window_at(d, oi, oj);
      const float p = dyp[w];
      if (d.mode == 0) {
        int best_e = b.i0 + d.H * b.j0;
        float best = xs[best_e];
        for (int j = b.j0; j < b.j1; ++j)
          for (int i = b.i0; i < b.i1; ++i) {
            float v = xs[i + d.H * j];
            if (v > best) {
              best = v;
              best_e = i + d.H * j;
            }
          }
        arg[w] = best_e;
        ds[w] = p;
      } else {
        float area = (float)((b.i1 - b.i0) * (b.j1 - b.j0));
        ds[w] = __fdiv_rn(p, area);
      }
    }
  __syncthreads();
  float* dxp = dx + plane * HW;
  for (int j = warp; j < d.W; j += nw) {
    int oj_lo = j + d.pl - d.ww + 1;
    oj_lo = oj_lo <= 0 ? 0 : (oj_lo + d.sw - 1) / d.sw;
    const int oj_hi = min(d.OW - 1, (j + d.pl) / d.sw);
    for (int i = lane; i < d.H; i += 32) {
      const int e = i + d.H * j;
      int oi_lo = i + d.pt - d.wh + 1;
      oi_lo = oi_lo <= 0 ? 0 : (oi_lo + d.sh - 1) / d.sh;
      const int oi_hi = min(d.OH - 1, (i + d.pt) / d.sh);
      float acc = 0.f;
      for (int oj = oj_lo; oj <= oj_hi; ++oj)
        for (int oi = oi_lo; oi <= oi_hi; ++oi) {
          const int w = oi + d.OH * oj;
          if (d.mode != 0 || arg[w] == e) acc = __fadd_rn(acc, ds[w]);
        }
      dxp[e] = kAcc ? __fadd_rn(dxp[e], acc) : acc;
    }
  }
}

// Compile-time window / stride max pooling (AlexNet 3x3/2, LeNet and VGG
// 2x2/2): unrolled windows; index splits by multiply-shift (FastDiv) instead
// of integer division; INSIDE = every window lies inside the input (no
// padding, no clipping), which drops all bounds tests.  Same rules as
// pool_fwd_k / pool_bwd_plane_k (first strict maximum, (oj, oi) order).
struct FastDiv {  // n / d == (n * m) >> 40 for n * d < 2^39
  uint64_t m;
  explicit FastDiv(int d = 1) : m(((1ull << 40) + (uint64_t)d - 1) / (uint64_t)d) {}
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)n * m) >> 40);
  }
};

// CK_POOL_FWD_W outputs per thread per iteration (e, e + stride, ...): all
// the windows' loads are in flight before the first compare.
#ifndef CK_POOL_FWD_W
#define CK_POOL_FWD_W 2
#endif
template <int WH, int WW, int SH, int SW, bool INSIDE>
__global__ void pool_max_fwd_t(const float* __restrict__ x, float* __restrict__ y, PoolDims d,
                               FastDiv by_ohw, FastDiv by_oh, uint8_t* __restrict__ argout) {
  ck::pdl_entry();
  const int OHW = d.OH * d.OW, HW = d.H * d.W;
  const uint32_t total = (uint32_t)OHW * d.C * d.N;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t e0 = blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += CK_POOL_FWD_W * stride) {
    float v[CK_POOL_FWD_W][WW][WH];
    bool in[CK_POOL_FWD_W][WW][WH];
#pragma unroll
    for (int t = 0; t < CK_POOL_FWD_W; ++t) {
      const uint32_t e = e0 + t * stride;
      const bool live = e < total;
      const uint32_t ee = live ? e : e0;
      const uint32_t plane = by_ohw.div(ee);
      const int w = (int)(ee - plane * OHW);
      const int oj = (int)by_oh.div(w), oi = w - oj * d.OH;
      const int si = oi * SH - d.pt, sj = oj * SW - d.pl;
      const float* xp = x + (size_t)plane * HW;
#pragma unroll
      for (int b = 0; b < WW; ++b) {
        const int j = sj + b;
#pragma unroll
        for (int a = 0; a < WH; ++a) {
          const int i = si + a;
          in[t][b][a] = live && (INSIDE || (i >= 0 && i < d.H && j >= 0 && j < d.W));
          v[t][b][a] = in[t][b][a] ? __ldg(xp + i + d.H * j) : 0.f;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < CK_POOL_FWD_W; ++t) {
      const uint32_t e = e0 + t * stride;
      if (e >= total) break;
      float best = 0.f;
      bool have = false;
      int code = 0;  // window offset a + WH*b of the winner
#pragma unroll
      for (int b = 0; b < WW; ++b)
#pragma unroll
        for (int a = 0; a < WH; ++a)
          if (in[t][b][a]) {
            const float u = v[t][b][a];
            if ((INSIDE && a == 0 && b == 0) || (!INSIDE && !have) || u > best) {
              best = u;
              code = a + WH * b;
            }
            have = true;
          }
      y[e] = best;
      if (argout) argout[e] = (uint8_t)code;
    }
  }
}

// Backward from the argmax the forward recorded (one byte per window): no
// re-read of x, one thread per dx element gathering its <= ceil(W/S)^2
// windows in the reference's (oj, oi) order.
template <int WH, int WW, int SH, int SW, bool kAcc>
__global__ void pool_max_bwd_arg_t(const uint8_t* __restrict__ arg, const float* __restrict__ dy,
                                   float* dx, PoolDims d, FastDiv by_hw, FastDiv by_h) {
  ck::pdl_entry();
  constexpr int NI = (WH + SH - 1) / SH, NJ = (WW + SW - 1) / SW;
  const int HW = d.H * d.W, OHW = d.OH * d.OW;
  const uint32_t total = (uint32_t)HW * d.C * d.N;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += gridDim.x * blockDim.x) {
    const uint32_t plane = by_hw.div(e);
    const int pix = (int)(e - plane * HW);
    const int j = (int)by_h.div(pix), i = pix - j * d.H;
    const int ti = i + d.pt, tj = j + d.pl;
    const int oi_hi = min(d.OH - 1, ti / SH), oj_hi = min(d.OW - 1, tj / SW);
    const int oi_lo = ti - WH + 1 <= 0 ? 0 : (ti - WH + SH) / SH;
    const int oj_lo = tj - WW + 1 <= 0 ? 0 : (tj - WW + SW) / SW;
    const uint8_t* ap = arg + (size_t)plane * OHW;
    const float* dp = dy + (size_t)plane * OHW;
    float acc = 0.f;
#pragma unroll
    for (int b = 0; b < NJ; ++b) {
      const int oj = oj_lo + b;
#pragma unroll
      for (int a = 0; a < NI; ++a) {
        const int oi = oi_lo + a;
        if (oj <= oj_hi && oi <= oi_hi) {
          const int w = oi + d.OH * oj;
          const int code = __ldg(ap + w);
          const int ai = code % WH, bj = code / WH;
          if (oi * SH - d.pt + ai == i && oj * SW - d.pl + bj == j)
            acc = __fadd_rn(acc, __ldg(dp + w));
        }
      }
    }
    dx[e] = kAcc ? __fadd_rn(dx[e], acc) : acc;
  }
}

// 3x3 / stride 2 from the recorded argmax, one thread per 2x2 block of dx in
// padded coordinates (ti, tj) = (2a + di, 2b + dj): the four elements share
// the candidate windows oi in {a-1, a}, oj in {b-1, b}, whose codes and dy
// are loaded once; each element adds the dy of the windows routed to it in
// the reference's (oj, oi) order.
template <bool kAcc>
__global__ void pool_max3s2_bwd_arg_k(const uint8_t* __restrict__ arg,
                                      const float* __restrict__ dy, float* dx, PoolDims d,
                                      int A, int B, FastDiv by_a, FastDiv by_ab) {
  ck::pdl_entry();
  const int HW = d.H * d.W, OHW = d.OH * d.OW;
  const uint32_t total = (uint32_t)A * B * d.C * d.N;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += gridDim.x * blockDim.x) {
    const uint32_t plane = by_ab.div(e);
    const int r = (int)(e - plane * (uint32_t)(A * B));
    const int b = (int)by_a.div(r), a = r - b * A;
    const uint8_t* ap = arg + (size_t)plane * OHW;
    const float* dp = dy + (size_t)plane * OHW;
    int code[2][2];
    float g[2][2];
#pragma unroll
    for (int wb = 0; wb < 2; ++wb)
#pragma unroll
      for (int wa = 0; wa < 2; ++wa) {
        const int oi = a - 1 + wa, oj = b - 1 + wb;
        const bool ok = oi >= 0 && oi < d.OH && oj >= 0 && oj < d.OW;
        code[wb][wa] = ok ? __ldg(ap + oi + d.OH * oj) : -1;
        g[wb][wa] = ok ? __ldg(dp + oi + d.OH * oj) : 0.f;
      }
    float* dxp = dx + (size_t)plane * HW;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int di = 0; di < 2; ++di) {
        const int i = 2 * a + di - d.pt, j = 2 * b + dj - d.pl;
        if (i < 0 || i >= d.H || j < 0 || j >= d.W) continue;
        float acc = 0.f;
#pragma unroll
        for (int wb = 0; wb < 2; ++wb)
#pragma unroll
          for (int wa = 0; wa < 2; ++wa) {
            // window (a-1+wa, b-1+wb) starts at padded (2a-2+2wa, 2b-2+2wb): this
            // element is its offset (di+2-2wa, dj+2-2wb) if that lies in 0..2
            const int ai = di + 2 - 2 * wa, bj = dj + 2 - 2 * wb;
            if (ai <= 2 && bj <= 2 && code[wb][wa] == ai + 3 * bj)
              acc = __fadd_rn(acc, g[wb][wa]);
          }
        float* o = dxp + i + d.H * j;
        *o = kAcc ? __fadd_rn(*o, acc) : acc;
      }
  }
}

// Column-strip form of pool_max3s2_bwd_arg_k (identical matches and adds, in
// the same (oj, oi) order): a segment of SEG lanes owns one plane, lane a
// walks the block column b = 0..B-1.  Per step it loads only window (a, b);
// window (a-1, b) comes from lane a-1 by shuffle and windows (., b-1) from
// the previous step's registers -- 2 loads per 2x2 block instead of 8.  The
// two output rows of a block column are stored as float2 when aligned.
template <bool kAcc, int SEG>
__global__ void __launch_bounds__(256) pool_max3s2_bwd_strip_k(const uint8_t* __restrict__ arg,
                                                               const float* __restrict__ dy,
                                                               float* __restrict__ dx, PoolDims d,
                                                               int A, int B, int planes) {
  ck::pdl_entry();
  const int lane = threadIdx.x & 31;
  const int sub = lane % SEG;  // a
  const int64_t plane = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / SEG;
  const bool pl_ok = plane < planes;
  const int a = sub;
  const bool a_ok = pl_ok && a < A;
  const uint8_t* ap = arg + (pl_ok ? plane : 0) * (int64_t)d.OH * d.OW;
  const float* dp = dy + (pl_ok ? plane : 0) * (int64_t)d.OH * d.OW;
  float* dxp = dx + (pl_ok ? plane : 0) * (int64_t)d.H * d.W;
  const int oi = a;  // this lane's own window row (a, b)
  // windows (a-1, b-1) and (a, b-1) from the previous step
  int c_pl = -1, c_p = -1;
  float g_pl = 0.f, g_p = 0.f;
  const unsigned mask = 0xffffffffu;
  for (int b = 0; b < B; ++b) {
    const int oj = b;
    const bool w_ok = a_ok && oi < d.OH && oj < d.OW;
    const int code = w_ok ? __ldg(ap + oi + d.OH * oj) : -1;
    const float g = w_ok ? __ldg(dp + oi + d.OH * oj) : 0.f;
    // window (a-1, b): the left neighbour's (a = 0: none)
    int code_l = __shfl_up_sync(mask, code, 1, SEG);
    float g_l = __shfl_up_sync(mask, g, 1, SEG);
    if (sub == 0) {
      code_l = -1;
      g_l = 0.f;
    }
    // codes[wb][wa] = window (a-1+wa, b-1+wb)
    const int cd[2][2] = {{c_pl, c_p}, {code_l, code}};
    const float gd[2][2] = {{g_pl, g_p}, {g_l, g}};
    if (a_ok) {
#pragma unroll
      for (int dj = 0; dj < 2; ++dj) {
        const int j = 2 * b + dj - d.pl;
        float out[2];
#pragma unroll
        for (int di = 0; di < 2; ++di) {
          float acc = 0.f;
#pragma unroll
          for (int wb = 0; wb < 2; ++wb)
#pragma unroll
            for (int wa = 0; wa < 2; ++wa) {
              const int ai = di + 2 - 2 * wa, bj = dj + 2 - 2 * wb;
              if (ai <= 2 && bj <= 2 && cd[wb][wa] == ai + 3 * bj) acc = __fadd_rn(acc, gd[wb][wa]);
            }
          out[di] = acc;
        }
        if (j < 0 || j >= d.W) continue;
        const int i0 = 2 * a - d.pt;
        float* o = dxp + (int64_t)d.H * j + i0;
        const bool two = i0 >= 0 && i0 + 1 < d.H;
        if (two && ((reinterpret_cast<uintptr_t>(o) & 7) == 0) && !kAcc) {
          *reinterpret_cast<float2*>(o) = make_float2(out[0], out[1]);
        } else {
#pragma unroll
          for (int di = 0; di < 2; ++di) {
            const int i = i0 + di;
            if (i >= 0 && i < d.H) o[di] = kAcc ? __fadd_rn(o[di], out[di]) : out[di];
          }
        }
      }
    }
    c_pl = code_l;
    g_pl = g_l;
    c_p = code;
    g_p = g;
  }
}

template <int WH, int WW, int SH, int SW, bool INSIDE, bool kAcc>
__global__ void pool_max_bwd_t(const float* __restrict__ x, const float* __restrict__ dy,
                               float* dx, PoolDims d, FastDiv by_oh, FastDiv by_h) {
  ck::pdl_entry();
  extern __shared__ float psm[];
  const int HW = d.H * d.W, OHW = d.OH * d.OW;
  float* xs = psm;              // [HW]
  float* ds = xs + HW;          // [OHW]
  int* arg = (int*)(ds + OHW);  // [OHW]
  const int64_t plane = blockIdx.x;
  const float* xp = x + plane * HW;
  const float* dyp = dy + plane * OHW;
  for (int e = threadIdx.x; e < HW; e += blockDim.x) xs[e] = __ldg(xp + e);
  for (int w = threadIdx.x; w < OHW; w += blockDim.x) ds[w] = __ldg(dyp + w);
  __syncthreads();
  for (int w = threadIdx.x; w < OHW; w += blockDim.x) {
    const int oj = (int)by_oh.div(w), oi = w - oj * d.OH;
    const int si = oi * SH - d.pt, sj = oj * SW - d.pl;
    float best = 0.f;
    int best_e = -1;
#pragma unroll
    for (int b = 0; b < WW; ++b) {
      const int j = sj + b;
#pragma unroll
      for (int a = 0; a < WH; ++a) {
        const int i = si + a;
        if (INSIDE || (i >= 0 && i < d.H && j >= 0 && j < d.W)) {
          const int e = i + d.H * j;
          const float v = xs[e];
          if ((INSIDE && a == 0 && b == 0) || (!INSIDE && best_e < 0) || v > best) {
            best = v;
            best_e = e;
          }
        }
      }
    }
    arg[w] = best_e;
  }
  __syncthreads();
  constexpr int NI = (WH + SH - 1) / SH, NJ = (WW + SW - 1) / SW;
  float* dxp = dx + plane * HW;
  for (int e = threadIdx.x; e < HW; e += blockDim.x) {
    const int j = (int)by_h.div(e), i = e - j * d.H;
    const int ti = i + d.pt, tj = j + d.pl;
    const int oi_hi = min(d.OH - 1, ti / SH), oj_hi = min(d.OW - 1, tj / SW);
    const int oi_lo = ti - WH + 1 <= 0 ? 0 : (ti - WH + SH) / SH;
    const int oj_lo = tj - WW + 1 <= 0 ? 0 : (tj - WW + SW) / SW;
    float acc = 0.f;
#pragma unroll
    for (int b = 0; b < NJ; ++b) {
      const int oj = oj_lo + b;
#pragma unroll
      for (int a = 0; a < NI; ++a) {
        const int oi = oi_lo + a;
        if (oj <= oj_hi && oi <= oi_hi) {
          const int w = oi + d.OH * oj;
          if (arg[w] == e) acc = __fadd_rn(acc, ds[w]);
        }
      }
    }
    dxp[e] = kAcc ? __fadd_rn(dxp[e], acc) : acc;
  }
}

// ----------------------------------------------------------------- LRN ----
// normalize.cpp:18-22 lrn_group: [k - (n-1)/2, k + n-1-(n-1)/2] clipped.
// A block owns kLrnPix consecutive pixels of one image and stages all their
// channels in shared memory (coalesced loads along H), so the channel-window
// sums never re-read HBM.
constexpr int kLrnPix = 32;

__global__ void lrn_fwd_k(const float* __restrict__ x, float* __restrict__ y, int HW, int C,
                          int size, float kappa, float alpha, float nbeta) {
  ck::pdl_entry();
  extern __shared__ float sm[];
  float* sq = sm;  // [C][kLrnPix] squares
  const int n = blockIdx.y;
  const int p0 = blockIdx.x * kLrnPix;
  const int lane = threadIdx.x % kLrnPix;
  const int row = threadIdx.x / kLrnPix, rows = blockDim.x / kLrnPix;
  const int p = p0 + lane;
  const bool ok = p < HW;
  const float* xb = x + (int64_t)n * C * HW;
  float* yb = y + (int64_t)n * C * HW;
  for (int k = row; k < C; k += rows) {
    float v = ok ? xb[(int64_t)k * HW + p] : 0.f;
    sq[k * kLrnPix + lane] = __fmul_rn(v, v);
  }
  __syncthreads();
  const int down = (size - 1) / 2, up = size - 1 - down;
  for (int k = row; k < C; k += rows) {
    int lo = max(0, k - down), hi = min(C - 1, k + up);
    float acc = 0.f;
    for (int t = lo; t <= hi; ++t) acc = __fadd_rn(acc, sq[t * kLrnPix + lane]);
    float scale = powf(__fadd_rn(kappa, __fmul_rn(alpha, acc)), nbeta);
    if (ok) yb[(int64_t)k * HW + p] = __fmul_rn(xb[(int64_t)k * HW + p], scale);
  }
}

// normalize.cpp:74-118: dx_d = dy_d L_d^-b - 2 a b x_d sum_{k: d in G(k)} eta_k,
// eta_k = dy_k L_k^(-b-1) x_k.
template <bool kAcc>
__global__ void lrn_bwd_k(const float* __restrict__ x, const float* __restrict__ dy, float* dx,
                          int HW, int C, int size, float kappa, float alpha, float beta) {
  ck::pdl_entry();
  extern __shared__ float sm[];
  float* xs = sm;                  // [C][P]
  float* Ls = sm + C * kLrnPix;    // [C][P]
  float* eta = Ls + C * kLrnPix;   // [C][P]
  const int n = blockIdx.y;
  const int p0 = blockIdx.x * kLrnPix;
  const int lane = threadIdx.x % kLrnPix;
  const int row = threadIdx.x / kLrnPix, rows = blockDim.x / kLrnPix;
  const int p = p0 + lane;
  const bool ok = p < HW;
  const int64_t base = (int64_t)n * C * HW;
  for (int k = row; k < C; k += rows) xs[k * kLrnPix + lane] = ok ? x[base + (int64_t)k * HW + p] : 0.f;
  __syncthreads();
  const int down = (size - 1) / 2, up = size - 1 - down;
  const float nb1 = -beta - 1.f;
  for (int k = row; k < C; k += rows) {
    int lo = max(0, k - down), hi = min(C - 1, k + up);
    float acc = 0.f;
    for (int t = lo; t <= hi; ++t) {
      float v = xs[t * kLrnPix + lane];
      acc = __fadd_rn(acc, __fmul_rn(v, v));
    }
    float L = __fadd_rn(kappa, __fmul_rn(alpha, acc));
    Ls[k * kLrnPix + lane] = L;
    float g = ok ? dy[base + (int64_t)k * HW + p] : 0.f;
    eta[k * kLrnPix + lane] = __fmul_rn(__fmul_rn(g, powf(L, nb1)), xs[k * kLrnPix + lane]);
  }
  __syncthreads();
  const float c2ab = __fmul_rn(__fmul_rn(2.f, alpha), beta);
  for (int d = row; d < C; d += rows) {
    int klo = max(0, d - up), khi = min(C - 1, d + down);
    float acc = 0.f;
    for (int k = klo; k <= khi; ++k) acc = __fadd_rn(acc, eta[k * kLrnPix + lane]);
    if (ok) {
      int64_t e = base + (int64_t)d * HW + p;
      float g = dy[e];
      float r = __fadd_rn(__fmul_rn(g, powf(Ls[d * kLrnPix + lane], -beta)),
                          -__fmul_rn(__fmul_rn(c2ab, xs[d * kLrnPix + lane]), acc));
      dx[e] = kAcc ? __fadd_rn(dx[e], r) : r;
    }
  }
}

// Register-streaming LRN for group sizes 1..9: one thread per pixel walks the
// channels (coalesced across threads), holding the channel window in
// compile-time-indexed shift registers.  Out-of-range window slots hold 0,
// and 0 + a == a exactly, so every sum is performed in the reference's
// order (normalize.cpp:55-62, :85-111) and matches lrn_fwd_k / lrn_bwd_k.
// LRN with the channel window in registers, one pixel per thread (loads and
// stores coalesced along the pixels of a warp).  Loads run P channels ahead;
// the steady state (all prefetches in range) runs without bounds tests and
// walks the channel planes with pointer increments -- these kernels are
// instruction-bound otherwise.
#ifndef CK_LRN_FWD_P
#define CK_LRN_FWD_P 8
#endif
template <int NW>
__global__ void lrn_fwd_reg_k(const float* __restrict__ x, float* __restrict__ y, int HW, int C,
                              int64_t pixels, float kappa, float alpha, float nbeta) {
  ck::pdl_entry();
  constexpr int DOWN = (NW - 1) / 2, UP = NW - 1 - DOWN;
  constexpr int P = CK_LRN_FWD_P;  // prefetch distance (channels)
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < pixels;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / HW;
    const int p = (int)(e - n * HW);
    const float* xp = x + n * C * HW + p;
    float* yq = y + n * C * HW + p;
    auto ldx = [&](int t) { return (t >= 0 && t < C) ? __ldg(xp + (int64_t)t * HW) : 0.f; };
    float sq[NW], xv[NW];  // window k-DOWN .. k+UP
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      xv[i] = ldx(i - DOWN);
      sq[i] = __fmul_rn(xv[i], xv[i]);
    }
    float xpre[P];  // x[k + UP + 1 + u]
#pragma unroll
    for (int u = 0; u < P; ++u) xpre[u] = ldx(UP + 1 + u);
    const float* lp = xp + (int64_t)(P + UP + 1) * HW;  // prefetch address of step k
    auto step = [&](float v) {
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < NW; ++i) acc = __fadd_rn(acc, sq[i]);
      // fast-math power (MUFU lg2/ex2, a few ulp; normalize.cpp uses std::pow)
      const float scale = pow_normal(__fadd_rn(kappa, __fmul_rn(alpha, acc)), nbeta);
      *yq = __fmul_rn(xv[DOWN], scale);
#pragma unroll
      for (int i = 0; i < NW - 1; ++i) {
        sq[i] = sq[i + 1];
        xv[i] = xv[i + 1];
      }
      xv[NW - 1] = v;
      sq[NW - 1] = __fmul_rn(v, v);
    };
    int k0 = 0;
    for (; k0 + 2 * P + UP + 1 <= C; k0 += P) {  // steady state: no bounds tests
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const float v = xpre[u];
        xpre[u] = __ldg(lp);
        lp += HW;
        step(v);
        yq += HW;
      }
    }
    for (; k0 < C; k0 += P) {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const int k = k0 + u;
        const float v = xpre[u];
        xpre[u] = k + P + UP + 1 < C ? __ldg(lp) : 0.f;
        lp += HW;
        if (k < C) step(v);
        yq += HW;
      }
    }
  }
}

// LRN (normalize.cpp:47-71) fused with the 3x3 / stride-2 max pooling that
// reads it (pool.cpp:49-80; AlexNet norm1 -> pool1, norm2 -> pool2).  A block
// owns TOI x TOJ pool outputs of one image and computes the LRN of the
// (2 TOI + 1) x (2 TOJ + 1) input pixels their windows cover (one thread per
// pixel, the same register channel chain and float operations as
// lrn_fwd_reg_k, so y is bit-identical); every CH channels the values go
// through shared memory to the window maxima (first strict maximum, j outer /
// i inner, the winner's code a + 3b as pool_max_fwd_t records it for the
// backward).  The pool never re-reads the LRN output from HBM; y is still
// written (it is a variable of the tape), by the pixel's owning tile only.
// Requires pad_top = pad_left = 0 and windows covering every input pixel.
template <int NW>
__global__ void __launch_bounds__(320) lrn_maxpool3s2_k(
    const float* __restrict__ x, float* __restrict__ y, float* __restrict__ py,
    uint8_t* __restrict__ arg, int H, int W, int C, int OH, int OW, int TOI, float kappa,
    float alpha, float nbeta) {
  ck::pdl_entry();
  constexpr int DOWN = (NW - 1) / 2, UP = NW - 1 - DOWN;
  constexpr int TOJ = 4, TJ = 2 * TOJ + 1, CH = 8, TIM = 33;
  __shared__ float tile[2][CH][TJ][TIM + 1];  // double-buffered: one barrier per chunk
  const int TI = 2 * TOI + 1;
  const int n = blockIdx.z;
  const int oi0 = blockIdx.x * TOI, oj0 = blockIdx.y * TOJ;
  const int ib = 2 * oi0, jb = 2 * oj0;  // tile origin (pads top/left are 0)
  const int t = threadIdx.x;
  const int ti = t % TI, tj = t / TI;
  const int i = ib + ti, j = jb + tj;
  const bool in_tile = t < TI * TJ;
  const bool active = in_tile && i < H && j < W;
  const bool owned = active && (ti < 2 * TOI || oi0 + TOI >= OH) && (tj < 2 * TOJ || oj0 + TOJ >= OW);
  const int64_t HW = (int64_t)H * W;
  const float* xp = x + (int64_t)n * C * HW + i + (int64_t)H * j;
  float* yq = y + (int64_t)n * C * HW + i + (int64_t)H * j;
  auto ldx = [&](int c) { return (active && c >= 0 && c < C) ? __ldg(xp + (int64_t)c * HW) : 0.f; };
  float sq[NW], xv[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    xv[q] = ldx(q - DOWN);
    sq[q] = __fmul_rn(xv[q], xv[q]);
  }
  float nx[CH];
#pragma unroll
  for (int u = 0; u < CH; ++u) nx[u] = ldx(u + UP + 1);
  // pool-phase assignment: window w = t % 64 of the tile, channels u = t / 64,
  // t / 64 + npu, ... of the chunk
  const int pw = t & 63, pu = t >> 6, npu = max(1, (int)(blockDim.x >> 6));
  const int poi = oi0 + pw % TOI, poj = oj0 + pw / TOI;
  const bool pool_thread = pw < TOI * TOJ && poi < OH && poj < OW;
  const int psi = 2 * (poi - oi0), psj = 2 * (poj - oj0);
  const bool inside = 2 * poi + 2 < H && 2 * poj + 2 < W;
  const int OHW = OH * OW;
  const int64_t po = (int64_t)n * C * OHW + poi + (int64_t)OH * poj;
  for (int k0 = 0, buf = 0; k0 < C; k0 += CH, buf ^= 1) {
    float cur[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) cur[u] = nx[u];
#pragma unroll
    for (int u = 0; u < CH; ++u) nx[u] = ldx(k0 + CH + u + UP + 1);  // next chunk, in flight
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      float acc = 0.f;
#pragma unroll
      for (int q = 0; q < NW; ++q) acc = __fadd_rn(acc, sq[q]);
      const float scale = pow_normal(__fadd_rn(kappa, __fmul_rn(alpha, acc)), nbeta);
      const float v = __fmul_rn(xv[DOWN], scale);
      if (owned && k0 + u < C) yq[(int64_t)(k0 + u) * HW] = v;
      if (in_tile) tile[buf][u][tj][ti] = v;
#pragma unroll
      for (int q = 0; q < NW - 1; ++q) {
        sq[q] = sq[q + 1];
        xv[q] = xv[q + 1];
      }
      xv[NW - 1] = cur[u];
      sq[NW - 1] = __fmul_rn(cur[u], cur[u]);
    }
    __syncthreads();
    if (pool_thread) {
      for (int u = pu; u < CH; u += npu) {
        const int k = k0 + u;
        if (k >= C) break;
        float best;
        int code = 0;
        if (inside) {
          best = tile[buf][u][psj][psi];
#pragma unroll
          for (int bb = 0; bb < 3; ++bb)
#pragma unroll
            for (int aa = 0; aa < 3; ++aa) {
              const float v = tile[buf][u][psj + bb][psi + aa];
              if (v > best) {
                best = v;
                code = aa + 3 * bb;
              }
            }
        } else {  // clipped at the bottom / right edge (pool.cpp:20-33)
          best = 0.f;
          bool have = false;
#pragma unroll
          for (int bb = 0; bb < 3; ++bb)
#pragma unroll
            for (int aa = 0; aa < 3; ++aa) {
              if (2 * poi + aa < H && 2 * poj + bb < W) {
                const float v = tile[buf][u][psj + bb][psi + aa];
                if (!have || v > best) {
                  best = v;
                  code = aa + 3 * bb;
                }
                have = true;
              }
            }
        }
        py[po + (int64_t)k * OHW] = best;
        if (arg) arg[po + (int64_t)k * OHW] = (uint8_t)code;
      }
    }
  }
}

// lrn_bwd_grid_k's output: instead of dx, relu_backward(x, dx) -- x is the
// output of the ReLU feeding this LRN, so x > 0 is that ReLU's mask
// (activation.cpp:14-22) -- straight into the pixel-major dy grid of the conv
// below that ReLU (dy at (0, 0) of an Hg x Wg grid, channel g*Kgp + c of group
// g), with per-warp per-channel sums of the stored values (the conv's bias
// gradient partials).
struct LrnGridOut {
  float* grid;
  double* bpart;  // [pixel warp][Kgp * groups]
  int H, Hg, Wg, Kg, Kgp, Cp;
};

#ifndef CK_LRN_BWD_P
#define CK_LRN_BWD_P 8
#endif
#ifndef CK_LRN_GRID_MINB
#define CK_LRN_GRID_MINB 5
#endif
#ifndef CK_LRN_GRID_P
#define CK_LRN_GRID_P 8
#endif
template <int NW, bool kAcc>
__global__ void __launch_bounds__(128, 6) lrn_bwd_reg_k(const float* __restrict__ x, const float* __restrict__ dy, float* dx,
                              int HW, int C, int64_t pixels, float kappa, float alpha, float beta) {
  ck::pdl_entry();
  constexpr int DOWN = (NW - 1) / 2, UP = NW - 1 - DOWN;
  constexpr int P = CK_LRN_BWD_P;  // prefetch distance (channels): 2P loads in flight per thread
  const float nb = -beta;
  const float c2ab = __fmul_rn(__fmul_rn(2.f, alpha), beta);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < pixels;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / HW;
    const int p = (int)(e - n * HW);
    const int64_t base = n * C * HW + p;
    const float* xp = x + base;
    const float* gp = dy + base;
    auto ldx = [&](int t) { return (t >= 0 && t < C) ? __ldg(xp + (int64_t)t * HW) : 0.f; };
    auto ldg = [&](int t) { return t < C ? __ldg(gp + (int64_t)t * HW) : 0.f; };
    // x window of the lead index j: xw[i] = x[j - DOWN + i], sq = its squares
    float xw[NW], sq[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      xw[i] = ldx(i - DOWN);
      sq[i] = __fmul_rn(xw[i], xw[i]);
    }
    float xpre[P], gpre[P];  // x[j + UP + 1 + u], dy[j + u] for the next P steps
#pragma unroll
    for (int u = 0; u < P; ++u) {
      xpre[u] = ldx(UP + 1 + u);
      gpre[u] = ldg(u);
    }
    const float* lx = xp + (int64_t)(P + UP + 1) * HW;  // prefetch addresses of step j
    const float* lg = gp + (int64_t)P * HW;
    float* dq = dx + base - (int64_t)DOWN * HW;  // store address of step j (d = j - DOWN)
    float eta[NW];  // eta of indices j-NW+1 .. j (0 outside [0, C))
    float Ls[DOWN + 1], xs[DOWN + 1], gs[DOWN + 1];  // L^-beta, x, dy of j-DOWN .. j
    // running window sums (sq over the lead window, eta over its window):
    // one add and one subtract per step instead of NW adds.  They differ from
    // the reference's fresh sums by rounding only, and only inside kappa +
    // alpha * sum and the alpha-scaled correction term (alpha ~ 1e-4).
    float sqsum = 0.f, etasum = 0.f;
#pragma unroll
    for (int i = 0; i < NW; ++i) sqsum = __fadd_rn(sqsum, sq[i]);
#pragma unroll
    for (int i = 0; i < NW; ++i) eta[i] = 0.f;
#pragma unroll
    for (int i = 0; i <= DOWN; ++i) Ls[i] = xs[i] = gs[i] = 0.f;
    // one channel step; `full`: j < C and the store index j - DOWN >= 0
    auto step = [&](int j, float xlead, float gj_in, bool compute, bool store, int slot) {
      float L = 0.f, xj = 0.f, gj = 0.f, et = 0.f;
      if (compute) {
        const float Lj = __fadd_rn(kappa, __fmul_rn(alpha, sqsum));
        L = pow_normal(Lj, nb);  // L^-beta; L^(-beta-1) = L^-beta / L
        xj = xw[DOWN];
        gj = gj_in;
        et = __fmul_rn(__fmul_rn(gj, __fdividef(L, Lj)), xj);
      }
      etasum = __fadd_rn(__fsub_rn(etasum, eta[0]), et);
#pragma unroll
      for (int i = 0; i < NW - 1; ++i) eta[i] = eta[i + 1];
      eta[NW - 1] = et;
#pragma unroll
      for (int i = 0; i < DOWN; ++i) {
        Ls[i] = Ls[i + 1];
        xs[i] = xs[i + 1];
        gs[i] = gs[i + 1];
      }
      Ls[DOWN] = L;
      xs[DOWN] = xj;
      gs[DOWN] = gj;
      if (store) {
        // k in [d-UP, d+DOWN] = [j-NW+1, j]: the whole eta window (etasum)
        const float r = __fadd_rn(__fmul_rn(gs[0], Ls[0]),
                                  -__fmul_rn(__fmul_rn(c2ab, xs[0]), etasum));
        *dq = kAcc ? __fadd_rn(*dq, r) : r;
        (void)slot;
      }
      // advance the x window to lead index j + 1
      const float sqin = __fmul_rn(xlead, xlead);
      sqsum = __fadd_rn(__fsub_rn(sqsum, sq[0]), sqin);
#pragma unroll
      for (int i = 0; i < NW - 1; ++i) {
        xw[i] = xw[i + 1];
        sq[i] = sq[i + 1];
      }
      xw[NW - 1] = xlead;
      sq[NW - 1] = sqin;
      (void)j;
    };
    const int J = C + DOWN;  // steps
    int j0 = 0;
    // head group(s): stores not yet due, checked loads
    for (; j0 < J && (j0 < DOWN || j0 + 2 * P + UP + 1 > C); j0 += P) {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const int j = j0 + u;
        const float xl = xpre[u], gi = gpre[u];
        xpre[u] = j + P + UP + 1 < C ? __ldg(lx) : 0.f;
        gpre[u] = j + P < C ? __ldg(lg) : 0.f;
        lx += HW;
        lg += HW;
        if (j < J) step(j, xl, gi, j < C, j >= DOWN, (u + 8 - DOWN) & 7);
        dq += HW;
      }
    }
    // steady state: every load in range, every step computes and stores
    for (; j0 + 2 * P + UP + 1 <= C; j0 += P) {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const float xl = xpre[u], gi = gpre[u];
        xpre[u] = __ldg(lx);
        gpre[u] = __ldg(lg);
        lx += HW;
        lg += HW;
        step(j0 + u, xl, gi, true, true, (u + 8 - DOWN) & 7);
        dq += HW;
      }
    }
    for (; j0 < J; j0 += P) {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        const int j = j0 + u;
        const float xl = xpre[u], gi = gpre[u];
        xpre[u] = j + P + UP + 1 < C ? __ldg(lx) : 0.f;
        gpre[u] = j + P < C ? __ldg(lg) : 0.f;
        lx += HW;
        lg += HW;
        if (j < J) step(j, xl, gi, j < C, j >= DOWN, (u + 8 - DOWN) & 7);
        dq += HW;
      }
    }
  }
}

// lrn_bwd_reg_k<NW, false, true> restructured around the 32-channel runs of
// the grid store (same per-element float operations, so the grid values are
// bit-identical): the channel loop is unrolled by 32, so the stage slot, the
// prefetch ring slot and the flush point are compile-time constants (no
// per-channel index or branch arithmetic; this kernel was issue-bound at
// ~84 instructions per element), and each flush writes four pixels' 128-byte
// runs per instruction as float4 (lane = 4 channels of one of 4 pixels).
// Every chunk's loads are in range except the last chunk's (CHK variant).
// Bias partials: per warp, per channel, the 32 pixels summed as 8 per lane in
// pixel order and then across the 4 pixel lanes by a fixed xor tree (float),
// stored as [pixel warp][Cp] doubles like the generic kernel.
template <int NW>
__global__ void __launch_bounds__(128, CK_LRN_GRID_MINB)
    lrn_bwd_grid_k(const float* __restrict__ x, const float* __restrict__ dy, int HW, int C,
                   int64_t pixels, float kappa, float alpha, float beta, LrnGridOut go) {
  ck::pdl_entry();
  constexpr int DOWN = (NW - 1) / 2, UP = NW - 1 - DOWN;
  constexpr int P = CK_LRN_GRID_P;  // prefetch distance (channels); divides 32
  const float nb = -beta;
  const float c2ab = __fmul_rn(__fmul_rn(2.f, alpha), beta);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  __shared__ float gsm[4][32][33];  // per warp [pixel][channel of the run]
  __shared__ int grs[4][32];        // per warp: pixel grid row offsets (-1: none)
  const int q4 = lane >> 3, m4 = lane & 7;  // flush role: pixel-in-quad, channel quad
  for (int64_t eb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; eb < pixels;
       eb += (int64_t)gridDim.x * blockDim.x) {
    const bool live = eb + lane < pixels;
    const int64_t e = live ? eb + lane : pixels - 1;
    const int64_t n = e / HW;
    const int p = (int)(e - n * HW);
    {
      const int i = p % go.H, jj = p / go.H;
      const int grow0 = (int)(((int64_t)n * go.Hg * go.Wg + i + (int64_t)go.Hg * jj) * go.Cp);
      __syncwarp();  // the previous pixel group's flushes are done with grs
      grs[wib][lane] = live ? grow0 : -1;
    }
    const int64_t base = n * C * HW + p;
    const float* xp = x + base;
    const float* gp = dy + base;
    auto ldx = [&](int t) { return (t >= 0 && t < C) ? __ldg(xp + (int64_t)t * HW) : 0.f; };
    auto ldg = [&](int t) { return t < C ? __ldg(gp + (int64_t)t * HW) : 0.f; };
    float xw[NW], sq[NW];  // x window of the lead index j: x[j - DOWN + i]
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      xw[i] = ldx(i - DOWN);
      sq[i] = __fmul_rn(xw[i], xw[i]);
    }
    float xpre[P], gpre[P];  // ring slot j % P: x[j + UP + 1], dy[j]
#pragma unroll
    for (int u = 0; u < P; ++u) {
      xpre[u] = ldx(UP + 1 + u);
      gpre[u] = ldg(u);
    }
    const float* lx = xp + (int64_t)(P + UP + 1) * HW;  // next prefetch addresses
    const float* lg = gp + (int64_t)P * HW;
    float eta[NW];
    float Ls[DOWN + 1], xs[DOWN + 1], gs[DOWN + 1];
    float sqsum = 0.f, etasum = 0.f;
#pragma unroll
    for (int i = 0; i < NW; ++i) sqsum = __fadd_rn(sqsum, sq[i]);
#pragma unroll
    for (int i = 0; i < NW; ++i) eta[i] = 0.f;
#pragma unroll
    for (int i = 0; i <= DOWN; ++i) Ls[i] = xs[i] = gs[i] = 0.f;
    float* stage = &gsm[wib][lane][0];
    // step j (ring slot j % P): consume the prefetched lead x / dy, refill the
    // slot with index j + P, compute index j (if j < C), return the value of
    // store index j - DOWN (relu-gated)
    auto step = [&](int j, int slot, bool chk) -> float {
      const float xlead = xpre[slot], gj_in = gpre[slot];
      if (!chk) {
        xpre[slot] = __ldg(lx);
        gpre[slot] = __ldg(lg);
      } else {
        xpre[slot] = j + P + UP + 1 < C ? __ldg(lx) : 0.f;
        gpre[slot] = j + P < C ? __ldg(lg) : 0.f;
      }
      lx += HW;
      lg += HW;
      float L = 0.f, xj = 0.f, gj = 0.f, et = 0.f;
      if (!chk || j < C) {
        const float Lj = __fadd_rn(kappa, __fmul_rn(alpha, sqsum));
        L = pow_normal(Lj, nb);
        xj = xw[DOWN];
        gj = gj_in;
        et = __fmul_rn(__fmul_rn(gj, __fdividef(L, Lj)), xj);
      }
      etasum = __fadd_rn(__fsub_rn(etasum, eta[0]), et);
#pragma unroll
      for (int i = 0; i < NW - 1; ++i) eta[i] = eta[i + 1];
      eta[NW - 1] = et;
#pragma unroll
      for (int i = 0; i < DOWN; ++i) {
        Ls[i] = Ls[i + 1];
        xs[i] = xs[i + 1];
        gs[i] = gs[i + 1];
      }
      Ls[DOWN] = L;
      xs[DOWN] = xj;
      gs[DOWN] = gj;
      const float r = __fadd_rn(__fmul_rn(gs[0], Ls[0]), -__fmul_rn(__fmul_rn(c2ab, xs[0]), etasum));
      const float sqin = __fmul_rn(xlead, xlead);
      sqsum = __fadd_rn(__fsub_rn(sqsum, sq[0]), sqin);
#pragma unroll
      for (int i = 0; i < NW - 1; ++i) {
        xw[i] = xw[i + 1];
        sq[i] = sq[i + 1];
      }
      xw[NW - 1] = xlead;
      sq[NW - 1] = sqin;
      return (live && xs[0] > 0.f) ? r : 0.f;
    };
    // steps 0 .. DOWN-1: nothing to store yet (checked: C may be tiny)
#pragma unroll
    for (int j = 0; j < DOWN; ++j) (void)step(j, j % P, true);
    // run b: stores c = 32 b .. 32 b + 31 (steps j = c + DOWN), then the flush
    auto flush = [&](int c0) {
      __syncwarp();
      const int g = c0 / go.Kg;
      const int cpos = g * go.Kgp + (c0 - g * go.Kg) + 4 * m4;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int q = 4 * it + q4;
        const int rq = grs[wib][q];
        const float* src = &gsm[wib][q][4 * m4];
        const float4 v = make_float4(src[0], src[1], src[2], src[3]);
        s0 += v.x;
        s1 += v.y;
        s2 += v.z;
        s3 += v.w;
        if (rq >= 0) *reinterpret_cast<float4*>(go.grid + rq + cpos) = v;
      }
#pragma unroll
      for (int o = 8; o <= 16; o <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s3 += __shfl_xor_sync(0xffffffffu, s3, o);
      }
      if (q4 == 0) {
        double* bp = go.bpart + (eb >> 5) * go.Cp + cpos;
        bp[0] = s0;
        bp[1] = s1;
        bp[2] = s2;
        bp[3] = s3;
      }
      __syncwarp();
    };
    const int runs = C / 32;
    int b = 0;
    // unchecked runs: every prefetch index < C (max j + P + UP + 1 in the run)
    for (; b < runs && 32 * b + 31 + DOWN + P + UP + 1 < C; ++b) {
#pragma unroll
      for (int u = 0; u < 32; ++u) stage[u] = step(32 * b + u + DOWN, (u + DOWN) % P, false);
      flush(32 * b);
    }
    for (; b < runs; ++b) {
#pragma unroll
      for (int u = 0; u < 32; ++u) stage[u] = step(32 * b + u + DOWN, (u + DOWN) % P, true);
      flush(32 * b);
    }
  }
}

// ---------------------------------------------------------------- bnorm ---
// Per-channel moments over H*W*N (normalize.cpp:132-161).  Grid (C, splits):
// each block reduces a contiguous run of images of one channel in double and
// writes one partial; bnorm_finish sums the partials in a fixed order.
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Element e of a channel's reduction: x, and (backward) the derivative that
// reaches the bnorm output -- dy itself, or, with a fused bnorm -> relu
// (engine), dy = gate > 0 ? relu_dy : 0 (activation.cpp:14-22) computed on
// the fly from the bnorm output `gate` and the relu output's derivative.
// G = 0: plain dy.  G = 1: gate read from the stored bnorm output.  G = 2:
// the bnorm output recomputed from x with the forward's own (mu, inv) floats
// (muinv, written by the fused apply) -- the same float operations as the
// forward's bn_y, so the gate is the forward's exactly, without reading y.
struct BnGateP {
  float w, b, mu, inv;
};
__device__ __forceinline__ float bn_y(float x, float wk, float mu, float inv, float bk) {
  return __fadd_rn(__fmul_rn(__fmul_rn(wk, __fadd_rn(x, -mu)), inv), bk);
}
template <int G>
__device__ __forceinline__ float eff_dy1(float g, float x, const float* gate, int64_t e,
                                         const BnGateP& P) {
  if (G == 1 && !(gate[e] > 0.f)) return 0.f;
  if (G == 2 && !(bn_y(x, P.w, P.mu, P.inv, P.b) > 0.f)) return 0.f;
  return g;
}
template <int G>
__device__ __forceinline__ float4 eff_dy4(const float4* dy, const float4* gate, int64_t q,
                                          const float4& v, const BnGateP& P) {
  float4 g = __ldg(dy + q);
  if (G == 1) {
    const float4 t = __ldg(gate + q);
    g.x = t.x > 0.f ? g.x : 0.f;
    g.y = t.y > 0.f ? g.y : 0.f;
    g.z = t.z > 0.f ? g.z : 0.f;
    g.w = t.w > 0.f ? g.w : 0.f;
  } else if (G == 2) {
    g.x = bn_y(v.x, P.w, P.mu, P.inv, P.b) > 0.f ? g.x : 0.f;
    g.y = bn_y(v.y, P.w, P.mu, P.inv, P.b) > 0.f ? g.y : 0.f;
    g.z = bn_y(v.z, P.w, P.mu, P.inv, P.b) > 0.f ? g.z : 0.f;
    g.w = bn_y(v.w, P.w, P.mu, P.inv, P.b) > 0.f ? g.w : 0.f;
  }
  return g;
}
__device__ __forceinline__ BnGateP bn_gate_params(const float* gw, const float* gb,
                                                  const float* muinv, int c) {
  BnGateP P{0.f, 0.f, 0.f, 0.f};
  if (muinv) P = BnGateP{gw[c], gb[c], muinv[2 * c], muinv[2 * c + 1]};
  return P;
}

// Grid (C, splits): block (c, s) reduces images [n0, n1) of channel c.  The
// planes are contiguous (HWCN), read as float4 with four loads in flight per
// thread; every term is summed in double (the one-pass moments E[x^2] -
// E[x]^2 need it), in a fixed order per thread, a fixed tree per block and a
// fixed split order in bnorm_finish_k: deterministic.  HW % 4 != 0 (or misaligned): scalar loop.
template <bool kGrad, int G>
__global__ void __launch_bounds__(256) bnorm_stats_k(const float* __restrict__ x,
                                                     const float* __restrict__ dy,
                                                     const float* __restrict__ gate,
                                                     const float* __restrict__ gw,
                                                     const float* __restrict__ gb,
                                                     const float* __restrict__ muinv,
                                                     double* partial, int HW, int C, int N,
                                                     int splits, int vec) {
  ck::pdl_entry();
  const int c = blockIdx.x, s = blockIdx.y;
  const BnGateP P = bn_gate_params(gw, gb, muinv, c);
  const int n0 = (int)((int64_t)N * s / splits), n1 = (int)((int64_t)N * (s + 1) / splits);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int n = n0; n < n1; ++n) {
    const int64_t base = ((int64_t)n * C + c) * HW;
    if (vec) {
      const float4* xp = (const float4*)(x + base);
      const float4* gp = (const float4*)(dy + base);
      const float4* tp = (const float4*)(gate + base);
      const int Q = HW / 4;
#pragma unroll 4
      for (int q = threadIdx.x; q < Q; q += 256) {
        const float4 v = __ldg(xp + q);
        const double x0 = v.x, x1 = v.y, x2 = v.z, x3 = v.w;
        a0 += (x0 + x1) + (x2 + x3);
        a1 += (x0 * x0 + x1 * x1) + (x2 * x2 + x3 * x3);
        if (kGrad) {
          const float4 g = eff_dy4<G>(gp, tp, q, v, P);
          const double g0 = g.x, g1 = g.y, g2 = g.z, g3 = g.w;
          a2 += (g0 + g1) + (g2 + g3);
          a3 += (g0 * x0 + g1 * x1) + (g2 * x2 + g3 * x3);
        }
      }
    } else {
      for (int p = threadIdx.x; p < HW; p += 256) {
        const double v = x[base + p];
        a0 += v;
        a1 += v * v;
        if (kGrad) {
          const double g = eff_dy1<G>(dy[base + p], x[base + p], gate, base + p, P);
          a2 += g;
          a3 += g * v;
        }
      }
    }
  }
  __shared__ double red[4][8];
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  if (kGrad) {
    a2 = warp_sum(a2);
    a3 = warp_sum(a3);
  }
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    red[0][w] = a0;
    red[1][w] = a1;
    red[2][w] = a2;
    red[3][w] = a3;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double t = 0;
    for (int k = 0; k < 8; ++k) t += red[threadIdx.x][k];
    partial[((int64_t)s * C + c) * 4 + threadIdx.x] = t;
  }
}

__global__ void bnorm_finish_k(const double* partial, double* out, int C, int splits) {
  ck::pdl_entry();
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double t[4] = {0, 0, 0, 0};
  for (int s = 0; s < splits; ++s)
    for (int q = 0; q < 4; ++q) t[q] += partial[((int64_t)s * C + c) * 4 + q];
  for (int q = 0; q < 4; ++q) out[c * 4 + q] = t[q];
}

// y = w (x - mu) inv + b (normalize.cpp:172-178); moments_out gets the K x 2
// (mean, var) tensor of graph.cpp:259-266.  fixed_moments (bnorm_infer) takes
// precedence over stats.  y2 != null (fused bnorm -> relu): also relu(y).
__global__ void __launch_bounds__(256) bnorm_apply_k(const float* __restrict__ x,
                                                     const float* __restrict__ w,
                                                     const float* __restrict__ b,
                                                     const double* __restrict__ stats,
                                                     const float* __restrict__ fixed,
                                                     float* __restrict__ y, float* __restrict__ y2,
                                                     float* __restrict__ mom_out,
                                                     float* __restrict__ muinv_out, double eps,
                                                     int HW, int C, int N, int vec) {
  ck::pdl_entry();
  const int c = blockIdx.x;
  const double M = (double)HW * N;
  float mu, inv;
  if (fixed) {
    mu = fixed[c];
    inv = (float)(1.0 / sqrt((double)fixed[C + c] + eps));
  } else {
    double m = stats[c * 4] / M;
    double var = stats[c * 4 + 1] / M - m * m;
    if (var < 0) var = 0;
    mu = (float)m;
    inv = (float)(1.0 / sqrt(var + eps));
    if (mom_out && blockIdx.y == 0 && threadIdx.x == 0) {
      mom_out[c] = (float)m;
      mom_out[C + c] = (float)var;
    }
  }
  const float wk = w[c], bk = b[c];
  if (muinv_out && blockIdx.y == 0 && threadIdx.x == 0) {
    muinv_out[2 * c] = mu;  // for the backward's gate recomputation
    muinv_out[2 * c + 1] = inv;
    muinv_out[2 * C + c] = wk;  // the parameter snapshot (engine recomputation)
    muinv_out[3 * C + c] = bk;
  }
  for (int n = blockIdx.y; n < N; n += gridDim.y) {
    const int64_t base = ((int64_t)n * C + c) * HW;
    if (vec) {
      const float4* xp = (const float4*)(x + base);
      float4* yp = (float4*)(y + base);
      float4* rp = (float4*)(y2 + base);
      const int Q = HW / 4;
#pragma unroll 4
      for (int q = threadIdx.x; q < Q; q += 256) {
        const float4 v = __ldg(xp + q);
        float4 o;
        o.x = bn_y(v.x, wk, mu, inv, bk);
        o.y = bn_y(v.y, wk, mu, inv, bk);
        o.z = bn_y(v.z, wk, mu, inv, bk);
        o.w = bn_y(v.w, wk, mu, inv, bk);
        if (y) yp[q] = o;
        if (y2) {
          o.x = o.x > 0.f ? o.x : 0.f;
          o.y = o.y > 0.f ? o.y : 0.f;
          o.z = o.z > 0.f ? o.z : 0.f;
          o.w = o.w > 0.f ? o.w : 0.f;
          rp[q] = o;
        }
      }
    } else {
      for (int p = threadIdx.x; p < HW; p += 256) {
        const float o = bn_y(x[base + p], wk, mu, inv, bk);
        if (y) y[base + p] = o;
        if (y2) y2[base + p] = o > 0.f ? o : 0.f;
      }
    }
  }
}

// normalize.cpp:212-265 with the moments and both reductions taken from
// stats = {sum x, sum x^2, sum dy, sum dy x}:
//   sum dy xhat = inv (sum dy x - mu sum dy)
//   dx = w inv (dy - mean(dy) - xhat mean(dy xhat))
__device__ __forceinline__ float bn_dx(float x, float g, float mu, float inv, float winv, float mdy,
                                       float mdyx) {
  const float xhat = __fmul_rn(__fadd_rn(x, -mu), inv);
  return __fmul_rn(winv, __fadd_rn(__fadd_rn(g, -mdy), -__fmul_rn(xhat, mdyx)));
}

template <bool kAcc, int G>
__global__ void __launch_bounds__(256) bnorm_bwd_k(const float* __restrict__ x,
                                                   const float* __restrict__ dy,
                                                   const float* __restrict__ gate,
                                                   const float* __restrict__ gb,
                                                   const float* __restrict__ muinv,
                                                   const float* __restrict__ w,
                                                   const double* __restrict__ stats, double eps,
                                                   float* dx, float* dw, float* db, int HW, int C,
                                                   int N, int acc_params, int vec) {
  ck::pdl_entry();
  const int c = blockIdx.x;
  const double M = (double)HW * N;
  const double m = stats[c * 4] / M;
  double var = stats[c * 4 + 1] / M - m * m;
  if (var < 0) var = 0;
  const double invd = 1.0 / sqrt(var + eps);
  const double sdy = stats[c * 4 + 2];
  const double sdyx = invd * (stats[c * 4 + 3] - m * sdy);
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    if (dw) dw[c] = acc_params ? dw[c] + (float)sdyx : (float)sdyx;
    if (db) db[c] = acc_params ? db[c] + (float)sdy : (float)sdy;
  }
  if (!dx) return;
  const float mu = (float)m, inv = (float)invd, wk = w[c];
  const float mdy = (float)(sdy / M), mdyx = (float)(sdyx / M);
  const float winv = __fmul_rn(wk, inv);
  const BnGateP P = bn_gate_params(w, gb, muinv, c);
  for (int n = blockIdx.y; n < N; n += gridDim.y) {
    const int64_t base = ((int64_t)n * C + c) * HW;
    if (vec) {
      const float4* xp = (const float4*)(x + base);
      const float4* gp = (const float4*)(dy + base);
      const float4* tp = (const float4*)(gate + base);
      float4* dp = (float4*)(dx + base);
      const int Q = HW / 4;
#pragma unroll 4
      for (int q = threadIdx.x; q < Q; q += 256) {
        const float4 v = __ldg(xp + q);
        const float4 g = eff_dy4<G>(gp, tp, q, v, P);
        float4 r;
        r.x = bn_dx(v.x, g.x, mu, inv, winv, mdy, mdyx);
        r.y = bn_dx(v.y, g.y, mu, inv, winv, mdy, mdyx);
        r.z = bn_dx(v.z, g.z, mu, inv, winv, mdy, mdyx);
        r.w = bn_dx(v.w, g.w, mu, inv, winv, mdy, mdyx);
        if (kAcc) {
          const float4 o = dp[q];
          r.x = __fadd_rn(o.x, r.x);
          r.y = __fadd_rn(o.y, r.y);
          r.z = __fadd_rn(o.z, r.z);
          r.w = __fadd_rn(o.w, r.w);
        }
        dp[q] = r;
      }
    } else {
      for (int p = threadIdx.x; p < HW; p += 256) {
        const float g = eff_dy1<G>(dy[base + p], x[base + p], gate, base + p, P);
        const float r = bn_dx(x[base + p], g, mu, inv, winv, mdy, mdyx);
        dx[base + p] = kAcc ? __fadd_rn(dx[base + p], r) : r;
      }
    }
  }
}

// bnorm backward (normalize.cpp:212-265, bnorm_bwd_k's float operations, so
// the values are bit-identical) writing the conv-below's dy grid instead of dx
// (VGG conv -> bnorm: the engine's bn_grid option): one pixel per thread walks
// the channels (x and dy read coalesced along the warp's 32 pixels, per channel
// plane); every 32 channels the warp's [pixel][channel] stage goes out as
// float4 runs of four pixels' 128-byte grid rows, with the 32-pixel column sums
// (the conv's bias-gradient partials, [pixel warp][Cp] doubles).  The
// per-channel constants come from the stats pass, computed per block in
// bnorm_bwd_k's expressions.  Requires the conv's channels per group % 32 == 0.
#ifndef CK_BN_GRID_BPS
#define CK_BN_GRID_BPS 16
#endif
// channels per block of the pixel-major bnorm grid kernels: all of them when
// the pixels alone fill ~CK_BN_GRID_BPS blocks per SM, else fewer (a multiple
// of 32; sweep on VGG: 16 beats 4 and 8 by ~1% of the step)
static int bn_grid_cchunk(int64_t pixels, int C) {
  const int64_t pblocks = std::min<int64_t>((pixels + 255) / 256, 148 * 8);
  int64_t want = (148 * CK_BN_GRID_BPS + pblocks - 1) / pblocks;  // channel chunks wanted
  int64_t cc = (C + want - 1) / want;
  cc = (cc + 31) / 32 * 32;
  return (int)std::max<int64_t>(32, std::min<int64_t>(C, cc));
}

struct BnGridOut {
  float* grid;
  double* bpart;
  int H, Hg, Wg, Kg, Kgp, Cp;
};

template <int G>
__global__ void __launch_bounds__(256) bnorm_bwd_grid_k(const float* __restrict__ x,
                                                        const float* __restrict__ dy,
                                                        const float* __restrict__ gate,
                                                        const float* __restrict__ gb,
                                                        const float* __restrict__ muinv,
                                                        const float* __restrict__ w,
                                                        const double* __restrict__ stats,
                                                        double eps, int HW, int C,
                                                        int64_t pixels, BnGridOut go,
                                                        float* dw, float* db, int acc_params,
                                                        int cchunk) {
  ck::pdl_entry();
  // blockIdx.y: channels [cb, ce) (a multiple of 32 wide) -- small images with
  // many channels get their parallelism from here
  const int cb = blockIdx.y * cchunk, ce = min(C, cb + cchunk), CC = ce - cb;
  extern __shared__ float bsm[];
  float* cmu = bsm;            // [ce - cb] each, indexed by c - cb
  float* cinv = cmu + CC;
  float* cwinv = cinv + CC;
  float* cmdy = cwinv + CC;
  float* cmdyx = cmdy + CC;
  float* gw = cmdyx + CC;      // G == 2: the gate's (w, b, mu, inv)
  float* gbb = gw + CC;
  float* gmu = gbb + CC;
  float* ginv = gmu + CC;
  float* stage = ginv + CC;    // [8 warps][32 pixels][33]
  int* grs = (int*)(stage + 8 * 32 * 33);  // [8 warps][32]
  const double M = (double)pixels;
  for (int c = cb + threadIdx.x; c < ce; c += blockDim.x) {
    const double m = stats[c * 4] / M;
    double var = stats[c * 4 + 1] / M - m * m;
    if (var < 0) var = 0;
    const double invd = 1.0 / sqrt(var + eps);
    const double sdy = stats[c * 4 + 2];
    const double sdyx = invd * (stats[c * 4 + 3] - m * sdy);
    if (blockIdx.x == 0) {  // bnorm_bwd_k's parameter derivatives
      if (dw) dw[c] = acc_params ? dw[c] + (float)sdyx : (float)sdyx;
      if (db) db[c] = acc_params ? db[c] + (float)sdy : (float)sdy;
    }
    const float inv = (float)invd;
    cmu[c - cb] = (float)m;
    cinv[c - cb] = inv;
    cwinv[c - cb] = __fmul_rn(w[c], inv);
    cmdy[c - cb] = (float)(sdy / M);
    cmdyx[c - cb] = (float)(sdyx / M);
    const BnGateP P = bn_gate_params(w, gb, muinv, c);
    gw[c - cb] = P.w;
    gbb[c - cb] = P.b;
    gmu[c - cb] = P.mu;
    ginv[c - cb] = P.inv;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int q4 = lane >> 3, m4 = lane & 7;
  float* st = stage + wib * 32 * 33;
  for (int64_t eb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; eb < pixels;
       eb += (int64_t)gridDim.x * blockDim.x) {
    const bool live = eb + lane < pixels;
    const int64_t e = live ? eb + lane : pixels - 1;
    const int64_t n = e / HW;
    const int p = (int)(e - n * HW);
    {
      const int i = p % go.H, jj = p / go.H;
      __syncwarp();
      grs[wib * 32 + lane] =
          live ? (int)(((int64_t)n * go.Hg * go.Wg + i + (int64_t)go.Hg * jj) * go.Cp) : -1;
    }
    const float* xp = x + n * C * HW + p;
    const float* dp = dy + n * C * HW + p;
    const float* tp = gate ? gate + n * C * HW + p : nullptr;
    for (int c0 = cb; c0 < ce; c0 += 32) {
#pragma unroll 8
      for (int u = 0; u < 32; ++u) {
        const int c = c0 + u;
        const int64_t off = (int64_t)c * HW;
        const float xv = __ldg(xp + off);
        float g = __ldg(dp + off);
        if (G == 1 && !(__ldg(tp + off) > 0.f)) g = 0.f;
        if (G == 2 && !(bn_y(xv, gw[c - cb], gmu[c - cb], ginv[c - cb], gbb[c - cb]) > 0.f)) g = 0.f;
        const float r = bn_dx(xv, g, cmu[c - cb], cinv[c - cb], cwinv[c - cb], cmdy[c - cb], cmdyx[c - cb]);
        st[lane * 33 + u] = live ? r : 0.f;
      }
      __syncwarp();
      const int grp = c0 / go.Kg;
      const int cpos = grp * go.Kgp + (c0 - grp * go.Kg) + 4 * m4;
      // bias partials in double: in front of a bnorm the conv bias gradient
      // is a sum that cancels to ~0 (sum_p dx_bn = 0), so only double keeps it
      // at the unfused path's accuracy
      double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int q = 4 * it + q4;
        const int rq = grs[wib * 32 + q];
        const float* src = st + q * 33 + 4 * m4;
        const float4 v = make_float4(src[0], src[1], src[2], src[3]);
        s0 += v.x;
        s1 += v.y;
        s2 += v.z;
        s3 += v.w;
        if (rq >= 0) *reinterpret_cast<float4*>(go.grid + rq + cpos) = v;
      }
#pragma unroll
      for (int o = 8; o <= 16; o <<= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s3 += __shfl_xor_sync(0xffffffffu, s3, o);
      }
      if (q4 == 0) {
        double* bp = go.bpart + (eb >> 5) * go.Cp + cpos;
        bp[0] = s0;
        bp[1] = s1;
        bp[2] = s2;
        bp[3] = s3;
      }
      __syncwarp();
    }
  }
}

// ----------------------------------------------------------------- loss ---
// loss.cpp:14-18 as_label, :101-106 range check.  flag bit 1: non-integer
// label, bit 2: out of range (reported by the C ABI as CK_ERR_DATA).
__device__ __forceinline__ int read_label(const float* labels, int64_t e, int C, int* flag) {
  float v = labels[e];
  float r = nearbyintf(v);
  if (r != v) {
    atomicOr(flag, 1);
    return 0;
  }
  int c = (int)r;
  if (c != 0 && (c < 1 || c > C)) {
    atomicOr(flag, 2);
    atomicCAS(flag + 1, 0, c);  // the first offending label, for the message
    return 0;
  }
  return c;
}

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per site (i, j, n); channels are HW apart.  Per-site loss
// w * (-x_c + max + log sum exp(x - max)) (loss.cpp:156-165).
__global__ void softmaxlog_fwd_k(const float* __restrict__ x, const float* __restrict__ labels,
                                 const float* __restrict__ weights, float* site_loss, int* flag,
                                 int HW, int C, int N) {
  ck::pdl_entry();
  const int64_t sites = (int64_t)HW * N;
  const int lane = threadIdx.x % 32;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < sites;
       s += (int64_t)gridDim.x * blockDim.x / 32) {
    int p = (int)(s % HW);
    int64_t n = s / HW;
    int c = read_label(labels, s, C, flag);
    const float* xs = x + n * (int64_t)C * HW + p;
    float mx = -INFINITY;
#pragma unroll 8
    for (int k = lane; k < C; k += 32) mx = fmaxf(mx, xs[(int64_t)k * HW]);
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll 8
    for (int k = lane; k < C; k += 32) sum += expf(xs[(int64_t)k * HW] - mx);
    sum = warp_sumf(sum);
    if (lane == 0) {
      float l = 0.f;
      if (c > 0) {
        float wgt = weights ? weights[s] : 1.f;
        l = wgt * (-xs[(int64_t)(c - 1) * HW] + mx + logf(sum));
      }
      site_loss[s] = l;
    }
  }
}

// Deterministic fixed-order sum of the per-site values (one block).
__global__ void sum_sites_k(const float* __restrict__ v, int64_t n, float* out) {
  ck::pdl_entry();
  __shared__ double red[32];
  double a = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += v[i];
  a = warp_sum(a);
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int k = 0; k < (int)(blockDim.x / 32); ++k) t += red[k];
    *out = (float)t;
  }
}

template <bool kAcc>
__global__ void softmaxlog_bwd_k(const float* __restrict__ x, const float* __restrict__ labels,
                                 const float* __restrict__ weights, float pscale,
                                 const float* __restrict__ pdev, float* dx, int* flag, int HW,
                                 int C, int N) {
  ck::pdl_entry();
  if (pdev) pscale = *pdev;  // the engine's projection, read on the device (graph.cpp:420-425)
  const int64_t sites = (int64_t)HW * N;
  const int lane = threadIdx.x % 32;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < sites;
       s += (int64_t)gridDim.x * blockDim.x / 32) {
    int p = (int)(s % HW);
    int64_t n = s / HW;
    int c = read_label(labels, s, C, flag);
    const float* xs = x + n * (int64_t)C * HW + p;
    float* ds = dx + n * (int64_t)C * HW + p;
    if (c == 0) {  // ignored site: zero derivative (loss.cpp:252)
      if (!kAcc)
        for (int k = lane; k < C; k += 32) ds[(int64_t)k * HW] = 0.f;
      continue;
    }
    float mx = -INFINITY;
#pragma unroll 8
    for (int k = lane; k < C; k += 32) mx = fmaxf(mx, xs[(int64_t)k * HW]);
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll 8
    for (int k = lane; k < C; k += 32) sum += expf(xs[(int64_t)k * HW] - mx);
    sum = warp_sumf(sum);
    const float scale = pscale * (weights ? weights[s] : 1.f);
#pragma unroll 4
    for (int k = lane; k < C; k += 32) {
      float soft = expf(xs[(int64_t)k * HW] - mx) / sum;
      float r = scale * (soft - (k == c - 1 ? 1.f : 0.f));
      ds[(int64_t)k * HW] = kAcc ? ds[(int64_t)k * HW] + r : r;
    }
  }
}

// The same two kernels with a site's C <= 32*R scores held in registers: one
// load pass with every load in flight instead of two (three) dependent
// strided passes.  Per-lane order of the max / exp-sum and the warp
// reductions are those of the kernels above, so results are bit-identical.
template <int R>
__global__ void softmaxlog_fwd_reg_k(const float* __restrict__ x, const float* __restrict__ labels,
                                     const float* __restrict__ weights, float* site_loss,
                                     int* flag, int HW, int C, int N) {
  ck::pdl_entry();
  const int64_t sites = (int64_t)HW * N;
  const int lane = threadIdx.x % 32;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < sites;
       s += (int64_t)gridDim.x * blockDim.x / 32) {
    const int p = (int)(s % HW);
    const int64_t n = s / HW;
    const int c = read_label(labels, s, C, flag);
    const float* xs = x + n * (int64_t)C * HW + p;
    float v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int k = lane + 32 * i;
      v[i] = k < C ? __ldg(xs + (int64_t)k * HW) : -INFINITY;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < R; ++i) mx = fmaxf(mx, v[i]);
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (lane + 32 * i < C) sum += expf(v[i] - mx);
    sum = warp_sumf(sum);
    if (lane == 0) {
      float l = 0.f;
      if (c > 0) {
        float wgt = weights ? weights[s] : 1.f;
        l = wgt * (-xs[(int64_t)(c - 1) * HW] + mx + logf(sum));
      }
      site_loss[s] = l;
    }
  }
}

template <int R, bool kAcc>
__global__ void softmaxlog_bwd_reg_k(const float* __restrict__ x, const float* __restrict__ labels,
                                     const float* __restrict__ weights, float pscale,
                                     const float* __restrict__ pdev, float* dx, int* flag, int HW,
                                     int C, int N) {
  ck::pdl_entry();
  if (pdev) pscale = *pdev;
  const int64_t sites = (int64_t)HW * N;
  const int lane = threadIdx.x % 32;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < sites;
       s += (int64_t)gridDim.x * blockDim.x / 32) {
    const int p = (int)(s % HW);
    const int64_t n = s / HW;
    const int c = read_label(labels, s, C, flag);
    const float* xs = x + n * (int64_t)C * HW + p;
    float* ds = dx + n * (int64_t)C * HW + p;
    if (c == 0) {  // ignored site: zero derivative (loss.cpp:252)
      if (!kAcc)
        for (int k = lane; k < C; k += 32) ds[(int64_t)k * HW] = 0.f;
      continue;
    }
    float v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int k = lane + 32 * i;
      v[i] = k < C ? __ldg(xs + (int64_t)k * HW) : -INFINITY;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < R; ++i) mx = fmaxf(mx, v[i]);
    mx = warp_max(mx);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (lane + 32 * i < C) sum += expf(v[i] - mx);
    sum = warp_sumf(sum);
    const float scale = pscale * (weights ? weights[s] : 1.f);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int k = lane + 32 * i;
      if (k < C) {
        float soft = expf(v[i] - mx) / sum;
        float r = scale * (soft - (k == c - 1 ? 1.f : 0.f));
        ds[(int64_t)k * HW] = kAcc ? ds[(int64_t)k * HW] + r : r;
      }
    }
  }
}

// classerror (loss.cpp:111-141; first strict maximum wins) and topk
// (loss.cpp:142-149; rank = #{k : x_k >= x_c}), weighted, per site.
__global__ void metrics_k(const float* __restrict__ x, const float* __restrict__ labels,
                          const float* __restrict__ weights, int top_k, float* site1,
                          float* sitek, int* flag, int HW, int C, int N) {
  ck::pdl_entry();
  const int64_t sites = (int64_t)HW * N;
  const int lane = threadIdx.x % 32;
  for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < sites;
       s += (int64_t)gridDim.x * blockDim.x / 32) {
    int p = (int)(s % HW);
    int64_t n = s / HW;
    int c = read_label(labels, s, C, flag);
    const float* xs = x + n * (int64_t)C * HW + p;
    if (c == 0) {
      if (lane == 0) site1[s] = sitek[s] = 0.f;
      continue;
    }
    float xc = xs[(int64_t)(c - 1) * HW];
    float bv = -INFINITY;
    int best = 0x7fffffff;
    int rank = 0;
    for (int k = lane; k < C; k += 32) {
      float v = xs[(int64_t)k * HW];
      if (v > bv) {
        bv = v;
        best = k;
      }
      rank += (v >= xc);
    }
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int ob = __shfl_xor_sync(0xffffffffu, best, o);
      if (ov > bv || (ov == bv && ob < best)) {
        bv = ov;
        best = ob;
      }
      rank += __shfl_xor_sync(0xffffffffu, rank, o);
    }
    if (lane == 0) {
      float wgt = weights ? weights[s] : 1.f;
      site1[s] = best == c - 1 ? 0.f : wgt;
      sitek[s] = rank <= top_k ? 0.f : wgt;
    }
  }
}

}  // namespace

// SPEC.md:716 "NaN loss aborts with diagnostic": sets `bit` in the handle's
// flag when any of the n values is NaN or infinite.
__global__ void flag_nonfinite_k(const float* __restrict__ v, int64_t n, int* flag, int bit) {
  ck::pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[i])) atomicOr(flag, bit);
}

// ------------------------------------------------------------ launchers ---

void relu_forward(const float* x, float* y, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  count_launch();
  if (n % 4 == 0 && aligned16(x) && aligned16(y))
    ck::pdl_launch(relu_fwd_v4, blocks_for(n / 4, 256), 256, 0, s, (const float4*)x, (float4*)y, n / 4);
  else
    ck::pdl_launch(relu_fwd_s, blocks_for(n, 256), 256, 0, s, x, y, n);
}

void relu_backward(const float* x, const float* dy, float* dx, int64_t n, int acc,
                   cudaStream_t s) {
  if (n == 0) return;
  count_launch();
  if (n % 4 == 0 && aligned16(x) && aligned16(dy) && aligned16(dx)) {
    if (acc)
      ck::pdl_launch(relu_bwd_v4<true>, blocks_for(n / 4, 256), 256, 0, s, (const float4*)x,
                                                               (const float4*)dy, (float4*)dx, n / 4);
    else
      ck::pdl_launch(relu_bwd_v4<false>, blocks_for(n / 4, 256), 256, 0, s, (const float4*)x,
                                                                (const float4*)dy, (float4*)dx, n / 4);
  } else {
    if (acc)
      ck::pdl_launch(relu_bwd_s<true>, blocks_for(n, 256), 256, 0, s, x, dy, dx, n);
    else
      ck::pdl_launch(relu_bwd_s<false>, blocks_for(n, 256), 256, 0, s, x, dy, dx, n);
  }
}

void axpy_inplace(float* y, const float* x, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  count_launch();
  ck::pdl_launch(axpy_k, blocks_for(n, 256), 256, 0, s, y, x, n);
}

void sgd_step(float* w, float* v, const float* g, int64_t n, float lr, float mom, float wd,
              cudaStream_t s) {
  if (n == 0) return;
  count_launch();
  if (n % 4 == 0 && (((uintptr_t)w | (uintptr_t)v | (uintptr_t)g) & 15) == 0) {
    ck::pdl_launch(sgd_v4_k, blocks_for(n / 4, 256), 256, 0, s, (float4*)w, (float4*)v, (const float4*)g,
                                                     n / 4, lr, mom, wd);
    return;
  }
  ck::pdl_launch(sgd_k, blocks_for(n, 256), 256, 0, s, w, v, g, n, lr, mom, wd);
}

// every window inside the input: no padding and the last window ends in it
static bool pool_inside(const PoolDims& d) {
  return d.pt == 0 && d.pl == 0 && (d.OH - 1) * d.sh + d.wh <= d.H &&
         (d.OW - 1) * d.sw + d.ww <= d.W;
}

template <int WH, int WW, int SH, int SW>
static void pool_max_fwd_launch(const float* x, float* y, const PoolDims& d, uint8_t* arg,
                                cudaStream_t s) {
  const int64_t total = (int64_t)d.OH * d.OW * d.C * d.N;
  const FastDiv a(d.OH * d.OW), b(d.OH);
  if (pool_inside(d))
    ck::pdl_launch(pool_max_fwd_t<WH, WW, SH, SW, true>, blocks_for(total, 256), 256, 0, s, x, y, d, a, b,
                                                                                arg);
  else
    ck::pdl_launch(pool_max_fwd_t<WH, WW, SH, SW, false>, blocks_for(total, 256), 256, 0, s, x, y, d, a, b,
                                                                                 arg);
}

template <int WH, int WW, int SH, int SW>
static void pool_max_bwd_arg_launch(const uint8_t* arg, const float* dy, float* dx,
                                    const PoolDims& d, int acc, cudaStream_t s) {
  const int64_t total = (int64_t)d.H * d.W * d.C * d.N;
  const FastDiv a(d.H * d.W), b(d.H);
  if (acc)
    ck::pdl_launch(pool_max_bwd_arg_t<WH, WW, SH, SW, true>, blocks_for(total, 256), 256, 0, s, arg, dy, dx,
                                                                                     d, a, b);
  else
    ck::pdl_launch(pool_max_bwd_arg_t<WH, WW, SH, SW, false>, blocks_for(total, 256), 256, 0, s, arg, dy, dx,
                                                                                      d, a, b);
}

static int64_t pool_arg_key(const float* x, const PoolDims& d) {
  return (int64_t)(((((((uint64_t)d.H * 4099 + d.W) * 65537 + d.C) * 131071 + d.N) * 31 + d.wh) *
                        31 + d.sh) * 31 + d.pt) ^ (uint64_t)(uintptr_t)x;
}

template <int WH, int WW, int SH, int SW>
static void pool_max_bwd_launch(const float* x, const float* dy, float* dx, const PoolDims& d,
                                int acc, size_t smem, cudaStream_t s) {
  const unsigned planes = (unsigned)((int64_t)d.C * d.N);
  const FastDiv a(d.OH), b(d.H);
  const bool in = pool_inside(d);
  if (in && acc)
    ck::pdl_launch(pool_max_bwd_t<WH, WW, SH, SW, true, true>, planes, 256, smem, s, x, dy, dx, d, a, b);
  else if (in)
    ck::pdl_launch(pool_max_bwd_t<WH, WW, SH, SW, true, false>, planes, 256, smem, s, x, dy, dx, d, a, b);
  else if (acc)
    ck::pdl_launch(pool_max_bwd_t<WH, WW, SH, SW, false, true>, planes, 256, smem, s, x, dy, dx, d, a, b);
  else
    ck::pdl_launch(pool_max_bwd_t<WH, WW, SH, SW, false, false>, planes, 256, smem, s, x, dy, dx, d, a, b);
}

// 2x2 / stride 2 max pooling without padding on even planes (LeNet, VGG):
// windows tile the input exactly, so each input element belongs to ONE
// window.  One thread per window reads its 2x2 block as two float2 rows
// (coalesced along H) and writes the max in the reference's order (j outer,
// i inner, first strict maximum: pool.cpp:59-64) plus the winner's code
// a + 2b; the backward writes the window's four dx elements (dy at the
// argmax, zero elsewhere: pool.cpp:98-110), again as two float2 rows.
// Planes run along grid.y, so no index ever exceeds a plane.
__global__ void pool2_fwd_k(const float* __restrict__ x, float* __restrict__ y,
                            uint8_t* __restrict__ arg, int H, int OH, int OHW, int64_t planes,
                            FastDiv by_oh) {
  ck::pdl_entry();
  for (int64_t pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const float* xp = x + pl * (int64_t)H * (2 * (OHW / OH));
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < OHW; w += gridDim.x * blockDim.x) {
      const int oj = (int)by_oh.div((uint32_t)w), oi = w - oj * OH;
      const float2 r0 = __ldg((const float2*)(xp + 2 * oi + (int64_t)H * (2 * oj)));
      const float2 r1 = __ldg((const float2*)(xp + 2 * oi + (int64_t)H * (2 * oj + 1)));
      float best = r0.x;
      int code = 0;
      if (r0.y > best) { best = r0.y; code = 1; }
      if (r1.x > best) { best = r1.x; code = 2; }
      if (r1.y > best) { best = r1.y; code = 3; }
      y[pl * OHW + w] = best;
      if (arg) arg[pl * OHW + w] = (uint8_t)code;
    }
  }
}

template <bool kAcc, bool kArg>
__global__ void pool2_bwd_k(const float* __restrict__ x, const uint8_t* __restrict__ arg,
                            const float* __restrict__ dy, float* dx, int H, int OH, int OHW,
                            int64_t planes, FastDiv by_oh) {
  ck::pdl_entry();
  for (int64_t pl = blockIdx.y; pl < planes; pl += gridDim.y) {
    const int64_t xo = pl * (int64_t)H * (2 * (OHW / OH));
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < OHW; w += gridDim.x * blockDim.x) {
      const int oj = (int)by_oh.div((uint32_t)w), oi = w - oj * OH;
      const int64_t e0 = xo + 2 * oi + (int64_t)H * (2 * oj), e1 = e0 + H;
      int code;
      if (kArg) {
        code = __ldg(arg + pl * OHW + w);
      } else {
        const float2 r0 = __ldg((const float2*)(x + e0)), r1 = __ldg((const float2*)(x + e1));
        float best = r0.x;
        code = 0;
        if (r0.y > best) { best = r0.y; code = 1; }
        if (r1.x > best) { best = r1.x; code = 2; }
        if (r1.y > best) { best = r1.y; code = 3; }
      }
      const float g = __ldg(dy + pl * OHW + w);
      float2 o0 = make_float2(code == 0 ? g : 0.f, code == 1 ? g : 0.f);
      float2 o1 = make_float2(code == 2 ? g : 0.f, code == 3 ? g : 0.f);
      if (kAcc) {
        const float2 a0 = *(const float2*)(dx + e0), a1 = *(const float2*)(dx + e1);
        o0.x = __fadd_rn(a0.x, o0.x);
        o0.y = __fadd_rn(a0.y, o0.y);
        o1.x = __fadd_rn(a1.x, o1.x);
        o1.y = __fadd_rn(a1.y, o1.y);
      }
      *(float2*)(dx + e0) = o0;
      *(float2*)(dx + e1) = o1;
    }
  }
}

static bool pool2_exact(const PoolDims& d) {
  return d.mode == 0 && d.wh == 2 && d.ww == 2 && d.sh == 2 && d.sw == 2 && d.pt == 0 &&
         d.pl == 0 && d.H % 2 == 0 && d.W % 2 == 0 && d.OH == d.H / 2 && d.OW == d.W / 2 &&
         (int64_t)d.OH * d.OW * d.OH < (1ll << 39);
}

static dim3 pool2_grid(const PoolDims& d) {
  const int64_t planes = (int64_t)d.C * d.N;
  const int OHW = d.OH * d.OW;
  const unsigned gx = (unsigned)std::min<int64_t>((OHW + 255) / 256, 1024);
  const int64_t want = std::max<int64_t>(1, (int64_t)kSMs * 8 / gx);
  return dim3(gx, (unsigned)std::min<int64_t>(std::min<int64_t>(planes, want * 4), 65535));
}

// compile-time window/stride of a max pooling, or 0
static int pool_fixed(const PoolDims& d) {
  if (d.mode != 0) return 0;
  if (d.wh == 3 && d.ww == 3 && d.sh == 2 && d.sw == 2) return 3;
  if (d.wh == 2 && d.ww == 2 && d.sh == 2 && d.sw == 2) return 2;
  return 0;
}

// With a layer cache (graph engine) the fixed-window max path also records
// each window's argmax for the backward of the same step.
void pool_forward(const float* x, float* y, const PoolDims& d, cudaStream_t s, ConvCache* cache) {
  int64_t total = (int64_t)d.OH * d.OW * d.C * d.N;
  if (total == 0) return;
  count_launch();
  // FastDiv and 32-bit indices: total * OH*OW < 2^39
  const int fx = total < (1ll << 31) && total * d.OH * d.OW < (1ll << 39) ? pool_fixed(d) : 0;
  uint8_t* arg = nullptr;
  if (fx && cache) {
    arg = (uint8_t*)cache->buf.get((size_t)total, s);
    if (arg) {
      cache->valid = true;
      cache->src = x;
      cache->key = pool_arg_key(x, d);
    }
  }
  if (pool2_exact(d) && ((uintptr_t)x & 7) == 0) {
    if (!arg && cache && pool_fixed(d)) arg = (uint8_t*)cache->buf.get((size_t)total, s);
    if (arg && cache) {
      cache->valid = true;
      cache->src = x;
      cache->key = pool_arg_key(x, d);
    }
    ck::pdl_launch(pool2_fwd_k, pool2_grid(d), 256, 0, s, x, y, arg, d.H, d.OH, d.OH * d.OW,
                                              (int64_t)d.C * d.N, FastDiv(d.OH));
    return;
  }
  switch (fx) {
    case 3: pool_max_fwd_launch<3, 3, 2, 2>(x, y, d, arg, s); return;
    case 2: pool_max_fwd_launch<2, 2, 2, 2>(x, y, d, arg, s); return;
    default: ck::pdl_launch(pool_fwd_k, blocks_for(total, 256), 256, 0, s, x, y, d);
  }
}

void pool_backward(const float* x, const float* dy, float* dx, const PoolDims& d, int acc,
                   cudaStream_t s, ConvCache* cache) {
  int64_t total = (int64_t)d.H * d.W * d.C * d.N;
  if (total == 0) return;
  count_launch();
  const int fx = pool_fixed(d);
  if (pool2_exact(d) && (((uintptr_t)x | (uintptr_t)dx) & 7) == 0) {
    const bool have_arg = cache && cache->valid && cache->src == x &&
                          cache->key == pool_arg_key(x, d);
    const uint8_t* arg = have_arg ? (const uint8_t*)cache->buf.ptr : nullptr;
    const dim3 grid = pool2_grid(d);
    const int64_t planes = (int64_t)d.C * d.N;
    const FastDiv by(d.OH);
    const int OHW = d.OH * d.OW;
    if (arg) {
      if (acc) ck::pdl_launch(pool2_bwd_k<true, true>, grid, 256, 0, s, x, arg, dy, dx, d.H, d.OH, OHW, planes, by);
      else ck::pdl_launch(pool2_bwd_k<false, true>, grid, 256, 0, s, x, arg, dy, dx, d.H, d.OH, OHW, planes, by);
    } else {
      if (acc) ck::pdl_launch(pool2_bwd_k<true, false>, grid, 256, 0, s, x, arg, dy, dx, d.H, d.OH, OHW, planes, by);
      else ck::pdl_launch(pool2_bwd_k<false, false>, grid, 256, 0, s, x, arg, dy, dx, d.H, d.OH, OHW, planes, by);
    }
    return;
  }
  if (fx && cache && cache->valid && cache->src == x && cache->key == pool_arg_key(x, d) &&
      total < (1ll << 31) && total * d.H * d.W < (1ll << 39)) {
    const uint8_t* arg = (const uint8_t*)cache->buf.ptr;
    if (fx == 3) {
      const int A = (d.H + d.pt + 1) / 2, B = (d.W + d.pl + 1) / 2;
      const int64_t blocks = (int64_t)A * B * d.C * d.N;
      const FastDiv by_a(A), by_ab(A * B);
      if (A <= 31 && !knob("CK_POOL_BWD_FLAT", 0)) {
        // column strips: one lane segment (SEG >= A + 1 lanes) per plane
        const int planes = d.C * d.N;
        const int seg = A < 8 ? 8 : A < 16 ? 16 : 32;
        const int64_t threads = (int64_t)planes * seg;
        const unsigned grid = (unsigned)((threads + 255) / 256);
#define CK_PSB(S)                                                                          \
  do {                                                                                     \
    if (acc) ck::pdl_launch(pool_max3s2_bwd_strip_k<true, S>, grid, 256, 0, s, arg, dy, dx, d, A, B, planes); \
    else ck::pdl_launch(pool_max3s2_bwd_strip_k<false, S>, grid, 256, 0, s, arg, dy, dx, d, A, B, planes);   \
  } while (0)
        if (seg == 8) CK_PSB(8);
        else if (seg == 16) CK_PSB(16);
        else CK_PSB(32);
#undef CK_PSB
        return;
      }
      if (blocks * A * B < (1ll << 39)) {
        if (acc)
          ck::pdl_launch(pool_max3s2_bwd_arg_k<true>, blocks_for(blocks, 256), 256, 0, s, arg, dy, dx, d, A,
                                                                              B, by_a, by_ab);
        else
          ck::pdl_launch(pool_max3s2_bwd_arg_k<false>, blocks_for(blocks, 256), 256, 0, s, arg, dy, dx, d, A,
                                                                               B, by_a, by_ab);
        return;
      }
      pool_max_bwd_arg_launch<3, 3, 2, 2>(arg, dy, dx, d, acc, s);
    } else {
      pool_max_bwd_arg_launch<2, 2, 2, 2>(arg, dy, dx, d, acc, s);
    }
    return;
  }
  const size_t smem = sizeof(float) * ((size_t)d.H * d.W + 2 * (size_t)d.OH * d.OW);
  if (smem <= 96 * 1024) {
    static bool configured = false;
    if (!configured) {
      cudaFuncSetAttribute(pool_bwd_plane_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           96 * 1024);
      cudaFuncSetAttribute(pool_bwd_plane_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           96 * 1024);
      configured = true;
    }
    const unsigned planes = (unsigned)((int64_t)d.C * d.N);
    const int fx = pool_fixed(d);
    // FastDiv needs n * d < 2^39 (n < HW, d <= H)
    if (fx && smem <= 48 * 1024 && (int64_t)d.H * d.W * d.H < (1ll << 39)) {
      if (fx == 3) pool_max_bwd_launch<3, 3, 2, 2>(x, dy, dx, d, acc, smem, s);
      else pool_max_bwd_launch<2, 2, 2, 2>(x, dy, dx, d, acc, smem, s);
      return;
    }
    if (acc)
      ck::pdl_launch(pool_bwd_plane_k<true>, planes, 256, smem, s, x, dy, dx, d);
    else
      ck::pdl_launch(pool_bwd_plane_k<false>, planes, 256, smem, s, x, dy, dx, d);
    return;
  }
  if (acc)
    ck::pdl_launch(pool_bwd_k<true>, blocks_for(total, 256), 256, 0, s, x, dy, dx, d);
  else
    ck::pdl_launch(pool_bwd_k<false>, blocks_for(total, 256), 256, 0, s, x, dy, dx, d);
}

static void lrn_smem_check(int C, int arrays) {
  size_t bytes = (size_t)arrays * C * kLrnPix * sizeof(float);
  static thread_local size_t configured = 0;
  if (bytes > 48 * 1024 && bytes > configured) {
    cudaFuncSetAttribute(lrn_fwd_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(lrn_bwd_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(lrn_bwd_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    configured = 227 * 1024;
  }
}

template <int NW>
static void lrn_fwd_reg(const float* x, float* y, int HW, int C, int N, float kappa, float alpha,
                        float beta, cudaStream_t s) {
  const int64_t pixels = (int64_t)HW * N;
  ck::pdl_launch(lrn_fwd_reg_k<NW>, blocks_for(pixels, 128, 32), 128, 0, s, x, y, HW, C, pixels, kappa, alpha,
                                                                 -beta);
}

template <int NW>
static void lrn_bwd_reg(const float* x, const float* dy, float* dx, int HW, int C, int N,
                        float kappa, float alpha, float beta, int acc, cudaStream_t s) {
  const int64_t pixels = (int64_t)HW * N;
  if (acc)
    ck::pdl_launch(lrn_bwd_reg_k<NW, true>, blocks_for(pixels, 128, 32), 128, 0, s, x, dy, dx, HW, C,
                   pixels, kappa, alpha, beta);
  else
    ck::pdl_launch(lrn_bwd_reg_k<NW, false>, blocks_for(pixels, 128, 32), 128, 0, s, x, dy, dx, HW, C,
                   pixels, kappa, alpha, beta);
}

#define CK_LRN_SWITCH(size, CALL) \
  switch (size) {                 \
    case 1: CALL(1); return;      \
    case 2: CALL(2); return;      \
    case 3: CALL(3); return;      \
    case 4: CALL(4); return;      \
    case 5: CALL(5); return;      \
    case 6: CALL(6); return;      \
    case 7: CALL(7); return;      \
    case 8: CALL(8); return;      \
    case 9: CALL(9); return;      \
    default: break;               \
  }

void lrn_forward(const float* x, float* y, int H, int W, int C, int N, int size, float kappa,
                 float alpha, float beta, cudaStream_t s) {
  const int HW = H * W;
  count_launch();
#define CK_FWD(NW) lrn_fwd_reg<NW>(x, y, HW, C, N, kappa, alpha, beta, s)
  if (lrn_pow_fast_ok(kappa, alpha, beta)) CK_LRN_SWITCH(size, CK_FWD)
#undef CK_FWD
  dim3 grid((HW + kLrnPix - 1) / kLrnPix, N);
  size_t smem = (size_t)C * kLrnPix * sizeof(float);
  lrn_smem_check(C, 1);
  ck::pdl_launch(lrn_fwd_k, grid, 256, smem, s, x, y, HW, C, size, kappa, alpha, -beta);
}

bool lrn_maxpool_forward(const float* x, float* y, float* py, const PoolDims& pd, int size,
                         float kappa, float alpha, float beta, cudaStream_t s, ConvCache* cache) {
  // 3x3 / stride-2 max pooling, pads top/left 0, windows covering the input
  if (!lrn_pow_fast_ok(kappa, alpha, beta)) return false;
  if (pd.mode != 0 || pd.wh != 3 || pd.ww != 3 || pd.sh != 2 || pd.sw != 2 || pd.pt != 0 ||
      pd.pl != 0 || 2 * (pd.OH - 1) + 3 < pd.H || 2 * (pd.OW - 1) + 3 < pd.W)
    return false;
  if (size != 5 && size != 3) return false;
  if (((pd.OH <= 16 ? pd.OH : (pd.OH + 1) / 2)) > 16 || pd.N > 65535) return false;
  uint8_t* arg = nullptr;
  const int64_t total = (int64_t)pd.OH * pd.OW * pd.C * pd.N;
  if (cache) {
    arg = (uint8_t*)cache->buf.get((size_t)total, s);
    if (arg) {
      cache->valid = true;
      cache->src = y;
      cache->key = pool_arg_key(y, pd);
    }
  }
  count_launch();
  // window rows per tile: the whole column when it fits, else halves
  const int TOI = pd.OH <= 16 ? pd.OH : (pd.OH + 1) / 2;
  if (TOI > 16) return false;
  const int threads = ((2 * TOI + 1) * 9 + 31) / 32 * 32;
  const dim3 grid((pd.OH + TOI - 1) / TOI, (pd.OW + 3) / 4, pd.N);
  if (size == 5)
    ck::pdl_launch(lrn_maxpool3s2_k<5>, grid, threads, 0, s, x, y, py, arg, pd.H, pd.W, pd.C, pd.OH, pd.OW,
                                                  TOI, kappa, alpha, -beta);
  else
    ck::pdl_launch(lrn_maxpool3s2_k<3>, grid, threads, 0, s, x, y, py, arg, pd.H, pd.W, pd.C, pd.OH, pd.OW,
                                                  TOI, kappa, alpha, -beta);
  return true;
}

void lrn_backward(const float* x, const float* dy, float* dx, int H, int W, int C, int N, int size,
                  float kappa, float alpha, float beta, int acc, cudaStream_t s) {
  const int HW = H * W;
  count_launch();
#define CK_BWD(NW) lrn_bwd_reg<NW>(x, dy, dx, HW, C, N, kappa, alpha, beta, acc, s)
  if (lrn_pow_fast_ok(kappa, alpha, beta)) CK_LRN_SWITCH(size, CK_BWD)
#undef CK_BWD
  dim3 grid((HW + kLrnPix - 1) / kLrnPix, N);
  size_t smem = (size_t)3 * C * kLrnPix * sizeof(float);
  lrn_smem_check(C, 3);
  if (acc)
    ck::pdl_launch(lrn_bwd_k<true>, grid, 256, smem, s, x, dy, dx, HW, C, size, kappa, alpha, beta);
  else
    ck::pdl_launch(lrn_bwd_k<false>, grid, 256, smem, s, x, dy, dx, HW, C, size, kappa, alpha, beta);
}

bool lrn_backward_grid(const float* x, const float* dy, float* grid, double* bpart, int H, int W,
                       int C, int N, int size, float kappa, float alpha, float beta, int Hg, int Wg,
                       int Kg, int Kgp, int groups, cudaStream_t s) {
  const int HW = H * W;
  const int64_t pixels = (int64_t)HW * N;
  // 32-channel runs never cross a group (and every run completes)
  if (H > Hg || W > Wg || Kg * groups != C || Kg % 32 || C % 32) return false;
  if (!lrn_pow_fast_ok(kappa, alpha, beta)) return false;
  // grid row offsets are kept as 32-bit ints in the kernel
  if ((int64_t)N * Hg * Wg * Kgp * groups >= (1ll << 31)) return false;
  LrnGridOut go{grid, bpart, H, Hg, Wg, Kg, Kgp, Kgp * groups};
  const dim3 grid_dim(blocks_for(pixels, 128, 32));
  switch (size) {
    case 3:
      count_launch();
      ck::pdl_launch(lrn_bwd_grid_k<3>, grid_dim, 128, 0, s, x, dy, HW, C, pixels, kappa, alpha, beta,
                     go);
      return true;
    case 5:
      count_launch();
      ck::pdl_launch(lrn_bwd_grid_k<5>, grid_dim, 128, 0, s, x, dy, HW, C, pixels, kappa, alpha, beta,
                     go);
      return true;
    default:
      return false;
  }
}

int lrn_grid_rows(int H, int W, int N) { return (int)(((int64_t)H * W * N + 31) / 32); }

int bnorm_splits(int HW, int C, int N) {
  // ~4 blocks of 256 threads per SM overall
  int want = (kSMs * 4 + C - 1) / C;
  if (want > N) want = N;
  if (want < 1) want = 1;
  (void)HW;
  return want;
}

static int bnorm_vec(const void* a, const void* b, const void* c, int HW) {
  return HW % 4 == 0 && ((((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 15) == 0);
}

void bnorm_stats(const float* x, const float* dy, double* partial, double* out, int HW, int C,
                 int N, int splits, cudaStream_t s, const float* gate, const BnGate& rg) {
  dim3 grid(C, splits);
  count_launch(2);
  const int vec = bnorm_vec(x, dy, gate, HW);
  if (dy && rg.muinv)
    ck::pdl_launch(bnorm_stats_k<true, 2>, grid, 256, 0, s, x, dy, nullptr, rg.w, rg.b, rg.muinv, partial, HW,
                                                C, N, splits, vec);
  else if (dy && gate)
    ck::pdl_launch(bnorm_stats_k<true, 1>, grid, 256, 0, s, x, dy, gate, nullptr, nullptr, nullptr, partial,
                                                HW, C, N, splits, vec);
  else if (dy)
    ck::pdl_launch(bnorm_stats_k<true, 0>, grid, 256, 0, s, x, dy, nullptr, nullptr, nullptr, nullptr, partial,
                                                HW, C, N, splits, vec);
  else
    ck::pdl_launch(bnorm_stats_k<false, 0>, grid, 256, 0, s, x, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                 partial, HW, C, N, splits, vec);
  ck::pdl_launch(bnorm_finish_k, (C + 127) / 128, 128, 0, s, partial, out, C, splits);
}

static int bnorm_grid_y(int C, int N) {
  int gy = (kSMs * 8 + C - 1) / C;
  if (gy > N) gy = N;
  if (gy < 1) gy = 1;
  return gy;
}

void bnorm_apply(const float* x, const float* w, const float* b, const double* stats,
                 const float* fixed_moments, float* y, float* moments_out, double eps, int HW,
                 int C, int N, cudaStream_t s, float* y2, float* muinv_out) {
  count_launch();
  ck::pdl_launch(bnorm_apply_k, dim3(C, bnorm_grid_y(C, N)), 256, 0, s, 
      x, w, b, stats, fixed_moments, y, y2, moments_out, muinv_out, eps, HW, C, N,
      bnorm_vec(x, y, y2, HW));
}

void bnorm_backward_apply(const float* x, const float* dy, const float* w, const double* stats,
                          double eps, float* dx, float* dw, float* db, int HW, int C, int N,
                          int acc, cudaStream_t s, const float* gate, const BnGate& rg) {
  count_launch();
  const dim3 grid(C, bnorm_grid_y(C, N));
  const int vec = bnorm_vec(x, dy, gate, HW) && bnorm_vec(dx, dx, dx, HW);
#define CK_BNB(A, G)                                                                        \
  ck::pdl_launch(bnorm_bwd_k<A, G>, grid, 256, 0, s, x, dy, gate, rg.b, rg.muinv, w, stats, eps, dx, dw,  \
                                         db, HW, C, N, acc ? 1 : 0, vec)
  const int G = rg.muinv ? 2 : gate ? 1 : 0;
  if (acc) {
    if (G == 2) CK_BNB(true, 2);
    else if (G == 1) CK_BNB(true, 1);
    else CK_BNB(true, 0);
  } else {
    if (G == 2) CK_BNB(false, 2);
    else if (G == 1) CK_BNB(false, 1);
    else CK_BNB(false, 0);
  }
#undef CK_BNB
}

// Fused bnorm -> relu forward for a relu output read only by the next conv
// (VGG bn -> relu -> conv): relu(bn_y(x)) goes straight into that conv's
// padded pixel-major x grid (x at (pt, pl) of an Hg x Wg grid; channel c of
// group g' at g' Cgp + c - g' Cg) instead of HWCN -- the conv skips its input
// transform.  One pixel per thread walks the channels (x read coalesced per
// channel plane); every 32 channels the warp's stage goes out as float4 runs
// of four pixels' 128-byte grid rows.  mu / inv / moments exactly as
// bnorm_apply_k computes them (block 0 writes the moments and (mu, inv)).
struct BnXGridOut {
  float* grid;
  int H, Hg, Wg, Cg, Cgp, Cp, pt, pl;
};

__global__ void __launch_bounds__(256) bnorm_apply_grid_k(const float* __restrict__ x,
                                                          const float* __restrict__ w,
                                                          const float* __restrict__ b,
                                                          const double* __restrict__ stats,
                                                          float* __restrict__ mom_out,
                                                          float* __restrict__ muinv_out,
                                                          double eps, int HW, int C,
                                                          int64_t pixels, BnXGridOut go,
                                                          int cchunk) {
  ck::pdl_entry();
  const int c_b = blockIdx.y * cchunk, c_e = min(C, c_b + cchunk), CC = c_e - c_b;
  extern __shared__ float asm_[];
  float* cw = asm_;  // [c_e - c_b] each, indexed by c - c_b
  float* cmu = cw + CC;
  float* cinv = cmu + CC;
  float* cb = cinv + CC;
  float* stage = cb + CC;  // [8 warps][32][33]
  int* grs = (int*)(stage + 8 * 32 * 33);
  const double M = (double)pixels;
  for (int c = c_b + threadIdx.x; c < c_e; c += blockDim.x) {
    const double m = stats[c * 4] / M;
    double var = stats[c * 4 + 1] / M - m * m;
    if (var < 0) var = 0;
    const float mu = (float)m, inv = (float)(1.0 / sqrt(var + eps));
    cmu[c - c_b] = mu;
    cinv[c - c_b] = inv;
    cw[c - c_b] = w[c];
    cb[c - c_b] = b[c];
    if (blockIdx.x == 0) {
      if (mom_out) {
        mom_out[c] = (float)m;
        mom_out[C + c] = (float)var;
      }
      if (muinv_out) {
        muinv_out[2 * c] = mu;
        muinv_out[2 * c + 1] = inv;
        muinv_out[2 * C + c] = w[c];  // the parameter snapshot (engine recomputation)
        muinv_out[3 * C + c] = b[c];
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int q4 = lane >> 3, m4 = lane & 7;
  float* st = stage + wib * 32 * 33;
  for (int64_t eb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; eb < pixels;
       eb += (int64_t)gridDim.x * blockDim.x) {
    const bool live = eb + lane < pixels;
    const int64_t e = live ? eb + lane : pixels - 1;
    const int64_t n = e / HW;
    const int p = (int)(e - n * HW);
    {
      const int i = p % go.H, jj = p / go.H;
      __syncwarp();
      grs[wib * 32 + lane] =
          live ? (int)(((int64_t)n * go.Wg * go.Hg + (int64_t)(jj + go.pl) * go.Hg + i + go.pt) * go.Cp)
               : -1;
    }
    const float* xp = x + n * C * HW + p;
    for (int c0 = c_b; c0 < c_e; c0 += 32) {
#pragma unroll 8
      for (int u = 0; u < 32; ++u) {
        const int c = c0 + u;
        const float o = bn_y(__ldg(xp + (int64_t)c * HW), cw[c - c_b], cmu[c - c_b], cinv[c - c_b], cb[c - c_b]);
        st[lane * 33 + u] = o > 0.f ? o : 0.f;
      }
      __syncwarp();
      const int grp = c0 / go.Cg;
      const int cpos = grp * go.Cgp + (c0 - grp * go.Cg) + 4 * m4;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int q = 4 * it + q4;
        const int rq = grs[wib * 32 + q];
        const float* src = st + q * 33 + 4 * m4;
        if (rq >= 0)
          *reinterpret_cast<float4*>(go.grid + rq + cpos) = make_float4(src[0], src[1], src[2], src[3]);
      }
      __syncwarp();
    }
  }
}

bool bnorm_apply_grid(const float* x, const float* w, const float* b, const double* stats,
                      float* moments_out, float* muinv_out, double eps, int H, int W, int C, int N,
                      float* grid, int Hg, int Wg, int Cg, int Cgp, int groups, int pt, int pl,
                      cudaStream_t s) {
  const int HW = H * W;
  const int64_t pixels = (int64_t)HW * N;
  if (Cg * groups != C || Cg % 32 || C % 32 || H + pt > Hg || W + pl > Wg) return false;
  if ((int64_t)N * Hg * Wg * Cgp * groups >= (1ll << 31)) return false;
  const int cchunk = bn_grid_cchunk(pixels, C);
  const size_t smem = sizeof(float) * (4 * (size_t)cchunk + 8 * 32 * 33) + sizeof(int) * 8 * 32;
  if (smem > 227 * 1024) return false;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(bnorm_apply_grid_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = 227 * 1024;
  }
  BnXGridOut go{grid, H, Hg, Wg, Cg, Cgp, Cgp * groups, pt, pl};
  count_launch();
  ck::pdl_launch(bnorm_apply_grid_k, dim3(blocks_for(pixels, 256, 8), (C + cchunk - 1) / cchunk), 256,
                 smem, s, x, w, b, stats, moments_out, muinv_out, eps, HW, C, pixels, go, cchunk);
  return true;
}

// y = bn_y(x) with the forward's own float (mu, inv) per channel: the bnorm
// output a fused bnorm -> relu forward did not store (engine bn_lazy_y),
// bit-identical to what bnorm_apply_k would have written.
__global__ void __launch_bounds__(256) bnorm_value_k(const float* __restrict__ x,
                                                     const float* __restrict__ w,
                                                     const float* __restrict__ b,
                                                     const float* __restrict__ muinv,
                                                     float* __restrict__ y, int HW, int C,
                                                     int64_t n_total, int relu) {
  ck::pdl_entry();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)((e / HW) % C);
    const float o = bn_y(x[e], w[c], muinv[2 * c], muinv[2 * c + 1], b[c]);
    y[e] = relu ? (o > 0.f ? o : 0.f) : o;
  }
}

void bnorm_value(const float* x, const float* w, const float* b, const float* muinv, float* y,
                 int HW, int C, int N, int relu, cudaStream_t s) {
  const int64_t n = (int64_t)HW * C * N;
  count_launch();
  ck::pdl_launch(bnorm_value_k, blocks_for(n, 256), 256, 0, s, x, w, b, muinv, y, HW, C, n, relu);
}

bool bnorm_backward_grid(const float* x, const float* dy, const float* w, const double* stats,
                         double eps, int H, int W, int C, int N, float* grid, double* bpart,
                         int Hg, int Wg, int Kg, int Kgp, int groups, cudaStream_t s,
                         const float* gate, const BnGate& rg, float* dw, float* db, int acc) {
  const int HW = H * W;
  const int64_t pixels = (int64_t)HW * N;
  if (H > Hg || W > Wg || Kg * groups != C || Kg % 32 || C % 32) return false;
  if ((int64_t)N * Hg * Wg * Kgp * groups >= (1ll << 31)) return false;
  const int cchunk = bn_grid_cchunk(pixels, C);
  const size_t smem = sizeof(float) * (9 * (size_t)cchunk + 8 * 32 * 33) + sizeof(int) * 8 * 32;
  if (smem > 227 * 1024) return false;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(bnorm_bwd_grid_k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(bnorm_bwd_grid_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(bnorm_bwd_grid_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    configured = 227 * 1024;
  }
  BnGridOut go{grid, bpart, H, Hg, Wg, Kg, Kgp, Kgp * groups};
  const int G = rg.muinv ? 2 : gate ? 1 : 0;
  const dim3 grd(blocks_for(pixels, 256, 8), (C + cchunk - 1) / cchunk);
  count_launch();
  if (G == 2)
    ck::pdl_launch(bnorm_bwd_grid_k<2>, grd, 256, smem, s, x, dy, nullptr, rg.b, rg.muinv, w, stats, eps,
                   HW, C, pixels, go, dw, db, acc, cchunk);
  else if (G == 1)
    ck::pdl_launch(bnorm_bwd_grid_k<1>, grd, 256, smem, s, x, dy, gate, nullptr, nullptr, w, stats, eps,
                   HW, C, pixels, go, dw, db, acc, cchunk);
  else
    ck::pdl_launch(bnorm_bwd_grid_k<0>, grd, 256, smem, s, x, dy, nullptr, nullptr, nullptr, w, stats,
                   eps, HW, C, pixels, go, dw, db, acc, cchunk);
  return true;
}

void softmaxlog_forward(const float* x, const float* labels, const float* weights,
                        float* site_loss, float* loss, int* flag, int HW, int C, int N,
                        cudaStream_t s) {
  int64_t sites = (int64_t)HW * N;
  count_launch(2);
  if (C <= 1024)
    ck::pdl_launch(softmaxlog_fwd_reg_k<32>, blocks_for(sites * 32, 256), 256, 0, s, x, labels, weights,
                                                                         site_loss, flag, HW, C, N);
  else
    ck::pdl_launch(softmaxlog_fwd_k, blocks_for(sites * 32, 256), 256, 0, s, x, labels, weights, site_loss,
                                                                  flag, HW, C, N);
  ck::pdl_launch(sum_sites_k, 1, 1024, 0, s, site_loss, sites, loss);
}

void softmaxlog_backward(const float* x, const float* labels, const float* weights, float p,
                         const float* p_dev, float* dx, int* flag, int HW, int C, int N, int acc,
                         cudaStream_t s) {
  int64_t sites = (int64_t)HW * N;
  count_launch();
  if (C <= 1024) {
    if (acc)
      ck::pdl_launch(softmaxlog_bwd_reg_k<32, true>, blocks_for(sites * 32, 256), 256, 0, s, 
          x, labels, weights, p, p_dev, dx, flag, HW, C, N);
    else
      ck::pdl_launch(softmaxlog_bwd_reg_k<32, false>, blocks_for(sites * 32, 256), 256, 0, s, 
          x, labels, weights, p, p_dev, dx, flag, HW, C, N);
    return;
  }
  if (acc)
    ck::pdl_launch(softmaxlog_bwd_k<true>, blocks_for(sites * 32, 256), 256, 0, s, x, labels, weights, p, p_dev,
                                                                        dx, flag, HW, C, N);
  else
    ck::pdl_launch(softmaxlog_bwd_k<false>, blocks_for(sites * 32, 256), 256, 0, s, x, labels, weights, p,
                                                                         p_dev, dx, flag, HW, C, N);
}

void loss_metrics(const float* x, const float* labels, const float* weights, int top_k,
                  float* site_buf, float* top1, float* topk, int* flag, int HW, int C, int N,
                  cudaStream_t s) {
  int64_t sites = (int64_t)HW * N;
  count_launch(3);
  ck::pdl_launch(metrics_k, blocks_for(sites * 32, 256), 256, 0, s, x, labels, weights, top_k, site_buf,
                                                         site_buf + sites, flag, HW, C, N);
  ck::pdl_launch(sum_sites_k, 1, 1024, 0, s, site_buf, sites, top1);
  ck::pdl_launch(sum_sites_k, 1, 1024, 0, s, site_buf + sites, sites, topk);
}

void flag_nonfinite(const float* v, int64_t n, int* flag, int bit, cudaStream_t s) {
  count_launch();
  ck::pdl_launch(flag_nonfinite_k, blocks_for(n, 256), 256, 0, s, v, n, flag, bit);
}

}  // namespace ck
