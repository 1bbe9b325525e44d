// Exact-FP32 convolution on CUDA cores: the CK_MATH_FP32 "verification" path.
//
// Each pass of conv.cpp:193-280 is an implicit GEMM over HWCN tensors (no
// im2row buffer is ever materialised):
//   fprop : M = output pixels (n, oj, oi), N = filters of a group,
//           K = (c, fj, fi) of the group          -> Y = A F      (conv.cpp:214)
//   dgrad : M = input pixels (n, j, i),  N = channels of a group,
//           K = (k, fj, fi), gather form of row2im -> dX = row2im(P F^T) (conv.cpp:270-278)
//   wgrad : M = (c, fj, fi), N = filters of a group, K = output pixels,
//           split-K with a deterministic reduction  -> dF = sum_n A^T P   (conv.cpp:260-269)
// A 64x64 output tile per 256-thread block, 4x4 per thread, BK = 16 staged in
// shared memory with register double buffering.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "ck_internal.hpp"

namespace ck {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

// ---- gather functors --------------------------------------------------------

struct FpropProb {
  const float* x;
  const float* f;
  const float* bias;
  float* y;
  ConvDims d;
  int relu;
  // per-group bases set by the kernel
  __device__ int64_t M() const { return (int64_t)d.N * d.OH * d.OW; }
  __device__ int64_t N() const { return d.Kg(); }
  __device__ int64_t K() const { return (int64_t)d.fh * d.fw * d.Cg; }
  // Row m -> its pixel; the A operand gathers x through the conv index map
  // (conv.cpp:45-53) with zero padding.
  struct RowCtx {
    const float* xb;
    int bi, bj;  // s*oi - pt, s*oj - pl
    bool valid;
  };
  __device__ RowCtx row(int64_t m, int g) const {
    RowCtx r;
    r.valid = m < M();
    if (!r.valid) m = 0;
    int oi = (int)(m % d.OH);
    int64_t t = m / d.OH;
    int oj = (int)(t % d.OW);
    int n = (int)(t / d.OW);
    r.xb = x + ((int64_t)n * d.C + (int64_t)g * d.Cg) * d.H * d.W;
    r.bi = d.sh * oi - d.pt;
    r.bj = d.sw * oj - d.pl;
    return r;
  }
  __device__ float a(const RowCtx& r, int64_t k) const {
    if (!r.valid || k >= K()) return 0.f;
    int fi = (int)(k % d.fh);
    int64_t t = k / d.fh;
    int fj = (int)(t % d.fw);
    int c = (int)(t / d.fw);
    int ii = r.bi + fi, jj = r.bj + fj;
    if (ii < 0 || ii >= d.H || jj < 0 || jj >= d.W) return 0.f;
    return r.xb[(int64_t)c * d.H * d.W + ii + (int64_t)d.H * jj];
  }
  __device__ float b(int64_t k, int64_t n, int g) const {
    if (k >= K() || n >= N()) return 0.f;
    int fi = (int)(k % d.fh);
    int64_t t = k / d.fh;
    int fj = (int)(t % d.fw);
    int64_t c = t / d.fw;
    int64_t kk = (int64_t)g * d.Kg() + n;
    return f[fi + (int64_t)d.fh * (fj + (int64_t)d.fw * (c * d.fsc + kk * d.fsk))];
  }
  __device__ void store(int64_t m, int64_t n, int g, float v, int acc) const {
    if (m >= M() || n >= N()) return;
    int64_t p = m % ((int64_t)d.OH * d.OW), img = m / ((int64_t)d.OH * d.OW);
    int64_t k = (int64_t)g * d.Kg() + n;
    if (bias) v = __fadd_rn(v, bias[k]);
    if (relu) v = v > 0.f ? v : 0.f;
    float* dst = y + (img * d.K + k) * d.OH * d.OW + p;
    *dst = acc ? __fadd_rn(*dst, v) : v;
  }
};

struct DgradProb {
  const float* dy;
  const float* f;
  float* dx;
  ConvDims d;
  __device__ int64_t M() const { return (int64_t)d.N * d.H * d.W; }
  __device__ int64_t N() const { return d.Cg; }
  __device__ int64_t K() const { return (int64_t)d.fh * d.fw * d.Kg(); }
  struct RowCtx {
    const float* yb;
    int i, j;
    bool valid;
  };
  __device__ RowCtx row(int64_t m, int g) const {
    RowCtx r;
    r.valid = m < M();
    if (!r.valid) m = 0;
    r.i = (int)(m % d.H);
    int64_t t = m / d.H;
    r.j = (int)(t % d.W);
    int n = (int)(t / d.W);
    r.yb = dy + ((int64_t)n * d.K + (int64_t)g * d.Kg()) * d.OH * d.OW;
    return r;
  }
  // A(m, (k, fj, fi)) = dy[oi, oj, k] where s*oi + fi - pt = i (row2im adjoint).
  __device__ float a(const RowCtx& r, int64_t kk) const {
    if (!r.valid || kk >= K()) return 0.f;
    int fi = (int)(kk % d.fh);
    int64_t t = kk / d.fh;
    int fj = (int)(t % d.fw);
    int k = (int)(t / d.fw);
    int ni = r.i + d.pt - fi, nj = r.j + d.pl - fj;
    if (ni < 0 || nj < 0) return 0.f;
    if (ni % d.sh || nj % d.sw) return 0.f;
    int oi = ni / d.sh, oj = nj / d.sw;
    if (oi >= d.OH || oj >= d.OW) return 0.f;
    return r.yb[(int64_t)k * d.OH * d.OW + oi + (int64_t)d.OH * oj];
  }
  __device__ float b(int64_t kk, int64_t n, int g) const {
    if (kk >= K() || n >= N()) return 0.f;
    int fi = (int)(kk % d.fh);
    int64_t t = kk / d.fh;
    int fj = (int)(t % d.fw);
    int64_t k = (int64_t)g * d.Kg() + t / d.fw;
    return f[fi + (int64_t)d.fh * (fj + (int64_t)d.fw * (n * d.fsc + k * d.fsk))];
  }
  __device__ void store(int64_t m, int64_t n, int g, float v, int acc) const {
    if (m >= M() || n >= N()) return;
    int64_t p = m % ((int64_t)d.H * d.W), img = m / ((int64_t)d.H * d.W);
    int64_t c = (int64_t)g * d.Cg + n;
    float* dst = dx + (img * d.C + c) * d.H * d.W + p;
    *dst = acc ? __fadd_rn(*dst, v) : v;
  }
};

// wgrad: rows are (c, fj, fi) of a group, columns filters of the group,
// reduction over output pixels; each z-slice handles a pixel range and
// writes a partial tile (reduced later in fixed order).
struct WgradProb {
  const float* x;
  const float* dy;
  float* part;  // [splits][groups][rows][cols]
  ConvDims d;
  __device__ int64_t M() const { return (int64_t)d.fh * d.fw * d.Cg; }
  __device__ int64_t N() const { return d.Kg(); }
  __device__ int64_t K() const { return (int64_t)d.N * d.OH * d.OW; }
  struct RowCtx {
    const float* xb;
    int fi, fj;
    bool valid;
  };
  __device__ RowCtx row(int64_t m, int g) const {
    RowCtx r;
    r.valid = m < M();
    if (!r.valid) m = 0;
    r.fi = (int)(m % d.fh);
    int64_t t = m / d.fh;
    r.fj = (int)(t % d.fw);
    int c = (int)(t / d.fw);
    r.xb = x + ((int64_t)g * d.Cg + c) * d.H * d.W;
    return r;
  }
  __device__ float a(const RowCtx& r, int64_t kk) const {
    if (!r.valid || kk >= K()) return 0.f;
    int oi = (int)(kk % d.OH);
    int64_t t = kk / d.OH;
    int oj = (int)(t % d.OW);
    int64_t n = t / d.OW;
    int ii = d.sh * oi + r.fi - d.pt, jj = d.sw * oj + r.fj - d.pl;
    if (ii < 0 || ii >= d.H || jj < 0 || jj >= d.W) return 0.f;
    return r.xb[n * d.C * d.H * d.W + ii + (int64_t)d.H * jj];
  }
  __device__ float b(int64_t kk, int64_t n, int g) const {
    if (kk >= K() || n >= N()) return 0.f;
    int64_t p = kk % ((int64_t)d.OH * d.OW), img = kk / ((int64_t)d.OH * d.OW);
    int64_t k = (int64_t)g * d.Kg() + n;
    return dy[(img * d.K + k) * d.OH * d.OW + p];
  }
  int splits;
  __device__ void store_part(int64_t m, int64_t n, int g, int split, float v) const {
    if (m >= M() || n >= N()) return;
    part[(((int64_t)split * d.groups + g) * N() + n) * M() + m] = v;
  }
};

// Fully-connected dgrad (H'' = W'' = 1, no padding): dX[q, n] = sum_k F[q, k] dY[k, n],
// a plain GEMM instead of the 1-valid-tap-in-H*W gather of DgradProb.
struct FcDgradProb {
  const float* dy;
  const float* f;
  float* dx;
  ConvDims d;
  __device__ int64_t Q() const { return (int64_t)d.H * d.W * d.C; }
  __device__ int64_t M() const { return Q(); }
  __device__ int64_t N() const { return d.N; }
  __device__ int64_t K() const { return d.K; }
  struct RowCtx {
    int64_t q;
    bool valid;
  };
  __device__ RowCtx row(int64_t m, int) const { return RowCtx{m, m < M()}; }
  __device__ float a(const RowCtx& r, int64_t k) const {
    return (r.valid && k < K()) ? f[r.q + Q() * k] : 0.f;
  }
  __device__ float b(int64_t k, int64_t n, int) const {
    return (k < K() && n < N()) ? dy[k + (int64_t)d.K * n] : 0.f;
  }
  __device__ void store(int64_t m, int64_t n, int, float v, int acc) const {
    if (m >= M() || n >= N()) return;
    float* dst = dx + m + Q() * n;
    *dst = acc ? __fadd_rn(*dst, v) : v;
  }
};

// ---- the tiled kernel ------------------------------------------------------------

template <class P, bool kSplit>
__global__ void __launch_bounds__(NT) simt_gemm_k(P p, int splits, int acc) {
  ck::pdl_entry();
  __shared__ float As[2][BK][BM];
  __shared__ float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int g = kSplit ? blockIdx.z / splits : blockIdx.z;
  const int split = kSplit ? blockIdx.z % splits : 0;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t Ktot = p.K();
  int64_t kbeg = 0, kend = Ktot;
  if (kSplit) {
    int64_t chunk = (Ktot + splits - 1) / splits;
    chunk = (chunk + BK - 1) / BK * BK;
    kbeg = chunk * split;
    kend = kbeg + chunk < Ktot ? kbeg + chunk : Ktot;
  }
  // loader mapping: element e = tid + NT*r (r<4) -> (row = e % 64, k = e / 64)
  const int lr = tid % 64, lk = tid / 64;  // lk in 0..3, k = lk + 4r
  auto rc = p.row(m0 + lr, g);
  float ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int64_t k = k0 + lk + 4 * r;
      ra[r] = k < kend ? p.a(rc, k) : 0.f;
      rb[r] = k < kend ? p.b(k, n0 + lr, g) : 0.f;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      As[buf][lk + 4 * r][lr] = ra[r];
      Bs[buf][lk + 4 * r][lr] = rb[r];
    }
  };
  float accv[4][4] = {};
  const int tx = tid % 16, ty = tid / 16;
  int buf = 0;
  if (kbeg < kend) {
    load(kbeg);
    stash(0);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[buf][kk][tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][kk][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) accv[i][j] = fmaf(av[i], bv[j], accv[i][j]);
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t m = m0 + tx + 16 * i, n = n0 + ty + 16 * j;
      if constexpr (kSplit)
        p.store_part(m, n, g, split, accv[i][j]);
      else
        p.store(m, n, g, accv[i][j], acc);
    }
}

// df[fi, fj, c, k] (+)= sum_s part[s][g][k][(c,fj,fi)], in split order.
__global__ void wgrad_reduce_k(const float* __restrict__ part, float* df, ConvDims d, int splits,
                               int acc) {
  ck::pdl_entry();
  const int64_t rows = (int64_t)d.fh * d.fw * d.Cg, cols = d.Kg();
  const int64_t per = rows * cols * d.groups;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < per;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = e % rows;
    int64_t t = e / rows;
    int64_t n = t % cols;
    int64_t g = t / cols;
    double s = 0.0;  // the split partials summed in double (FP32 verification path)
    for (int sp = 0; sp < splits; ++sp) s += part[sp * per + (g * cols + n) * rows + m];
    // m = fi + fh*(fj + fw*c)
    int64_t fi = m % d.fh, r = m / d.fh, fj = r % d.fw, c = r / d.fw;
    int64_t k = g * cols + n;
    float* dst = df + fi + (int64_t)d.fh * (fj + (int64_t)d.fw * (c * d.fsc + k * d.fsk));
    *dst = acc ? *dst + (float)s : (float)s;
  }
}

// db[k] = sum_n sum_p dy[p, k, n] (conv.cpp:246-252).  Each image's dy is
// K*OHW contiguous floats, so thread j of [0, K*OHW) sums element j over the
// images of its split (n = s, s+S, ...) with perfectly coalesced loads and
// four images in flight; bgrad_finish_k then reduces the S*OHW partials of
// channel k in a fixed order (deterministic, double accumulation).
__global__ void bgrad_part_k(const float* __restrict__ dy, double* part, int64_t KP, int N) {
  ck::pdl_entry();
  const int s = blockIdx.y, S = gridDim.y;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < KP;
       j += (int64_t)gridDim.x * blockDim.x) {
    const float* p = dy + j;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    int n = s;
    for (; n + 3 * S < N; n += 4 * S) {
      const float v0 = __ldg(p + (int64_t)n * KP), v1 = __ldg(p + (int64_t)(n + S) * KP);
      const float v2 = __ldg(p + (int64_t)(n + 2 * S) * KP), v3 = __ldg(p + (int64_t)(n + 3 * S) * KP);
      a0 += v0; a1 += v1; a2 += v2; a3 += v3;
    }
    for (; n < N; n += S) a0 += __ldg(p + (int64_t)n * KP);
    part[(int64_t)s * KP + j] = (a0 + a1) + (a2 + a3);
  }
}

__global__ void bgrad_finish_k(const double* part, float* db, int K, int OHW, int S, int acc) {
  ck::pdl_entry();
  const int k = blockIdx.x;
  const int64_t KP = (int64_t)K * OHW;
  double t = 0;
  for (int e = threadIdx.x; e < S * OHW; e += blockDim.x) {
    const int sp = e / OHW, q = e - sp * OHW;
    t += part[sp * KP + (int64_t)k * OHW + q];
  }
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __shared__ double red[32];
  if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) u += red[w];
    db[k] = acc ? db[k] + (float)u : (float)u;
  }
}

// Strided dgrad in gather form with the stride-phase decomposition: for dx
// pixel i only taps fi = (i + pt) mod s (+ s, + 2s, ...) hit an output row, so
// each thread visits ceil(fh/s) x ceil(fw/s) taps instead of fh x fw.  One
// thread per dx element, consecutive threads along H.
template <bool kAcc>
__global__ void dgrad_strided_k(const float* __restrict__ dy, const float* __restrict__ f,
                                float* dx, ConvDims d) {
  ck::pdl_entry();
  const int64_t total = (int64_t)d.H * d.W * d.C * d.N;
  const int Kg = d.Kg();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % d.H);
    int64_t r = e / d.H;
    const int j = (int)(r % d.W);
    r /= d.W;
    const int c = (int)(r % d.C);
    const int n = (int)(r / d.C);
    const int g = c / d.Cg, cl = c - g * d.Cg;
    const int ri = (i + d.pt) % d.sh, rj = (j + d.pl) % d.sw;
    float acc = 0.f;
    for (int fj = rj; fj < d.fw; fj += d.sw) {
      const int oj = (j + d.pl - fj) / d.sw;
      if (j + d.pl - fj < 0 || oj >= d.OW) continue;
      for (int fi = ri; fi < d.fh; fi += d.sh) {
        const int oi = (i + d.pt - fi) / d.sh;
        if (i + d.pt - fi < 0 || oi >= d.OH) continue;
        const float* yp = dy + ((int64_t)n * d.K + (int64_t)g * Kg) * d.OH * d.OW + oi +
                          (int64_t)d.OH * oj;
        const float* fp = f + fi + (int64_t)d.fh * (fj + (int64_t)d.fw * (cl * d.fsc));
        const int64_t fstep = (int64_t)d.fh * d.fw * d.fsk;
        const float* fpk = fp + (int64_t)g * Kg * (int64_t)d.fh * d.fw * d.fsk;
        for (int k = 0; k < Kg; ++k)
          acc = fmaf(yp[(int64_t)k * d.OH * d.OW], fpk[k * fstep], acc);
      }
    }
    dx[e] = kAcc ? __fadd_rn(dx[e], acc) : acc;
  }
}

int wgrad_splits(const ConvDims& d) {
  int64_t rows = (int64_t)d.fh * d.fw * d.Cg, cols = d.Kg();
  int64_t tiles = ((rows + BM - 1) / BM) * ((cols + BN - 1) / BN) * d.groups;
  int64_t K = (int64_t)d.N * d.OH * d.OW;
  int64_t want = (148 * 4 + tiles - 1) / tiles;
  int64_t maxs = (K + 255) / 256;  // at least 256 pixels per split
  if (want > maxs) want = maxs;
  // long reductions (b=256 weight gradients: up to 186k pixels) get more,
  // shorter fp32 partial sums (<= 2048 pixels each where the workspace allows)
  const int64_t per = rows * cols * d.groups;
  while (want < 256 && K / want > 2048 && per * want * 2 * sizeof(float) <= (size_t)512 << 20)
    want *= 2;
  if (want > maxs) want = maxs;
  if (want > 256) want = 256;
  if (want < 1) want = 1;
  return (int)want;
}

}  // namespace

void conv_fwd_fp32(const float* x, const float* f, const float* bias, float* y,
                   const ConvDims& d, int relu, cudaStream_t s) {
  FpropProb p{x, f, bias, y, d, relu};
  int64_t M = (int64_t)d.N * d.OH * d.OW;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((d.Kg() + BN - 1) / BN), d.groups);
  count_launch();
  ck::pdl_launch(simt_gemm_k<FpropProb, false>, grid, NT, 0, s, p, 1, 0);
}

void conv_dgrad_fp32(const float* dy, const float* f, float* dx, const ConvDims& d, int acc,
                     cudaStream_t s) {
  const bool fc = d.OH == 1 && d.OW == 1 && d.fh == d.H && d.fw == d.W && d.pt == 0 &&
                  d.pl == 0 && d.groups == 1 && d.fsc == 1;
  if (fc) {
    FcDgradProb p{dy, f, dx, d};
    int64_t Q = (int64_t)d.H * d.W * d.C;
    dim3 grid((unsigned)((Q + BM - 1) / BM), (unsigned)((d.N + BN - 1) / BN), 1);
    count_launch();
    ck::pdl_launch(simt_gemm_k<FcDgradProb, false>, grid, NT, 0, s, p, 1, acc);
    return;
  }
  if (d.sh > 1 || d.sw > 1) {
    int64_t total = (int64_t)d.H * d.W * d.C * d.N;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    count_launch();
    if (acc)
      ck::pdl_launch(dgrad_strided_k<true>, blocks, 256, 0, s, dy, f, dx, d);
    else
      ck::pdl_launch(dgrad_strided_k<false>, blocks, 256, 0, s, dy, f, dx, d);
    return;
  }
  DgradProb p{dy, f, dx, d};
  int64_t M = (int64_t)d.N * d.H * d.W;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((d.Cg + BN - 1) / BN), d.groups);
  count_launch();
  ck::pdl_launch(simt_gemm_k<DgradProb, false>, grid, NT, 0, s, p, 1, acc);
}

size_t conv_wgrad_ws_bytes(const ConvDims& d) {
  int64_t rows = (int64_t)d.fh * d.fw * d.Cg, cols = d.Kg();
  return (size_t)wgrad_splits(d) * rows * cols * d.groups * sizeof(float);
}

void conv_wgrad_fp32(const float* x, const float* dy, float* df, const ConvDims& d, int acc,
                     void* ws, cudaStream_t s) {
  int splits = wgrad_splits(d);
  WgradProb p{x, dy, (float*)ws, d};
  p.splits = splits;
  int64_t rows = (int64_t)d.fh * d.fw * d.Cg;
  dim3 grid((unsigned)((rows + BM - 1) / BM), (unsigned)((d.Kg() + BN - 1) / BN),
            d.groups * splits);
  count_launch(2);
  ck::pdl_launch(simt_gemm_k<WgradProb, true>, grid, NT, 0, s, p, splits, 0);
  int64_t per = rows * d.Kg() * d.groups;
  int blocks = (int)((per + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  ck::pdl_launch(wgrad_reduce_k, blocks, 256, 0, s, (const float*)ws, df, d, splits, acc);
}

static int bgrad_splits(int64_t KP, int N) {
  // ~148 SMs x 2048 threads in flight; at most one image per split
  const int64_t want = (148 * 2048 + KP - 1) / KP;
  return (int)std::max<int64_t>(1, std::min<int64_t>({want, (int64_t)N, 64}));
}

size_t conv_bgrad_ws_bytes(int K, int N, int OHW) {
  const int64_t KP = (int64_t)K * OHW;
  return sizeof(double) * (size_t)KP * bgrad_splits(KP, N);
}

void conv_bgrad(const float* dy, float* db, int OHW, int K, int N, int acc, void* ws,
                cudaStream_t s) {
  const int64_t KP = (int64_t)K * OHW;
  const int S = bgrad_splits(KP, N);
  const int blocks = (int)std::min<int64_t>((KP + 255) / 256, 148 * 8);
  count_launch(2);
  ck::pdl_launch(bgrad_part_k, dim3(blocks, S), 256, 0, s, dy, (double*)ws, KP, N);
  ck::pdl_launch(bgrad_finish_k, K, 256, 0, s, (const double*)ws, db, K, OHW, S, acc);
}

}  // namespace ck
