/*
 * ck_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference block algorithms (convkit, the
 * MatConvNet re-specification under /root/reference/proj) used as the parity
 * checker for the B200 kernels.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as a product path.
 *
 * Parity is pinned: tests/test_oracle_*.py check every function here against
 * (a) the SPEC.md known-answer examples and (b) the reference sources
 * themselves compiled verbatim into oracle/_ref (see oracle/Makefile).
 *
 * Layout: every tensor is dense HWCN, flat index i + H*(j + W*(c + C*n))
 * (reference include/convkit/tensor.hpp:70-72).
 *
 * Precision: the linear blocks (conv, convt, lrn, bnorm, loss) are restated
 * in double, which is the reference's own gradient-check instantiation
 * (conv.cpp:383-384, normalize.cpp:368-369).  Blocks whose parity is
 * bit-exact in single precision (relu, pool, sgd) are restated in float with
 * the reference's exact operation order.
 *
 * Return codes: 0 ok, 1 ShapeError, 2 DataError (reference error.hpp:9-24).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t h, w, c, n;
} cko_shape;

enum { CKO_OK = 0, CKO_SHAPE = 1, CKO_DATA = 2 };

static char g_err[512];
const char* cko_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

#define IDX(S_, I_, J_, C_, N_) ((I_) + (S_).h * ((J_) + (S_).w * ((C_) + (S_).c * (N_))))

static int64_t elems(cko_shape s) { return s.h * s.w * s.c * s.n; }

/* ---- geometry ---------------------------------------------------------- */

/* conv.cpp:108-116 conv_output_extent */
int cko_conv_output_extent(int64_t extent, int64_t window, int64_t stride,
                           int64_t pad_lo, int64_t pad_hi, int64_t* out) {
  if (extent + pad_lo + pad_hi < window) {
    char b[256];
    snprintf(b, sizeof b, "window of size %lld larger than padded input of size %lld",
             (long long)window, (long long)(extent + pad_lo + pad_hi));
    return fail(CKO_SHAPE, b);
  }
  *out = (extent - window + pad_lo + pad_hi) / stride + 1;
  return CKO_OK;
}

/* geom = {stride_h, stride_w, pad_top, pad_bottom, pad_left, pad_right, groups}
 * conv.hpp:9-17; validation conv.cpp:18-23, :118-135 */
int cko_conv_output_shape(cko_shape x, cko_shape f, const int64_t* g, cko_shape* out) {
  if (g[0] < 1 || g[1] < 1 || g[6] < 1 || g[2] < 0 || g[3] < 0 || g[4] < 0 || g[5] < 0)
    return fail(CKO_SHAPE, "invalid convolution geometry");
  if (f.c * g[6] != x.c) return fail(CKO_SHAPE, "filter channels x groups do not match input channels");
  if (f.n % g[6] != 0) return fail(CKO_SHAPE, "filter count not divisible by groups");
  int r;
  if ((r = cko_conv_output_extent(x.h, f.h, g[0], g[2], g[3], &out->h))) return r;
  if ((r = cko_conv_output_extent(x.w, f.w, g[1], g[4], g[5], &out->w))) return r;
  out->c = f.n;
  out->n = x.n;
  return CKO_OK;
}

/* cg = {up_h, up_w, crop_top, crop_bottom, crop_left, crop_right}; conv.cpp:137-154 */
int cko_convt_output_shape(cko_shape x, cko_shape f, const int64_t* cg, cko_shape* out) {
  if (cg[0] < 1 || cg[1] < 1 || cg[2] < 0 || cg[3] < 0 || cg[4] < 0 || cg[5] < 0)
    return fail(CKO_SHAPE, "invalid convolution-transpose geometry");
  if (f.c != x.c) return fail(CKO_SHAPE, "transposed filter input channel mismatch");
  out->h = cg[0] * (x.h - 1) + f.h - cg[2] - cg[3];
  out->w = cg[1] * (x.w - 1) + f.w - cg[4] - cg[5];
  out->c = f.n;
  out->n = x.n;
  if (out->h < 1 || out->w < 1) return fail(CKO_SHAPE, "transposed convolution output is not positive");
  return CKO_OK;
}

/* pg = {window_h, window_w, stride_h, stride_w, pad_top, pad_bottom, pad_left,
 *       pad_right, mode(0=max,1=avg)}; pool.hpp:13-23, pool.cpp:9-46 */
int cko_pool_output_shape(cko_shape x, const int64_t* pg, cko_shape* out) {
  if (pg[0] < 1 || pg[1] < 1 || pg[2] < 1 || pg[3] < 1 || pg[4] < 0 || pg[5] < 0 ||
      pg[6] < 0 || pg[7] < 0)
    return fail(CKO_SHAPE, "invalid pooling geometry");
  if (pg[4] > pg[0] - 1 || pg[5] > pg[0] - 1 || pg[6] > pg[1] - 1 || pg[7] > pg[1] - 1)
    return fail(CKO_SHAPE, "pooling pad exceeds window size minus one");
  int r;
  if ((r = cko_conv_output_extent(x.h, pg[0], pg[2], pg[4], pg[5], &out->h))) return r;
  if ((r = cko_conv_output_extent(x.w, pg[1], pg[3], pg[6], pg[7], &out->w))) return r;
  out->c = x.c;
  out->n = x.n;
  return CKO_OK;
}

/* ---- convolution (conv.cpp:33-84 im2row/row2im, :193-280 fwd/bwd) ------ */

/* Patch matrix of one image, (outH*outW) x (fh*fw*D) column-major
 * (conv.cpp:35-59). */
static void im2row_image(const double* x, int64_t H, int64_t W, int64_t D, int64_t fh,
                         int64_t fw, const int64_t* g, int64_t oH, int64_t oW, double* A) {
  const int64_t rows = oH * oW;
  for (int64_t d = 0; d < D; ++d)
    for (int64_t fj = 0; fj < fw; ++fj)
      for (int64_t fi = 0; fi < fh; ++fi) {
        double* col = A + rows * (fi + fh * (fj + fw * d));
        for (int64_t oj = 0; oj < oW; ++oj) {
          int64_t jj = g[1] * oj + fj - g[4];
          for (int64_t oi = 0; oi < oH; ++oi) {
            int64_t ii = g[0] * oi + fi - g[2];
            col[oi + oH * oj] = (jj >= 0 && jj < W && ii >= 0 && ii < H)
                                    ? x[ii + H * (jj + W * d)] : 0.0;
          }
        }
      }
}

/* Adjoint scatter (conv.cpp:63-84); accumulates into x. */
static void row2im_image(const double* A, int64_t H, int64_t W, int64_t D, int64_t fh,
                         int64_t fw, const int64_t* g, int64_t oH, int64_t oW, double* x) {
  const int64_t rows = oH * oW;
  for (int64_t d = 0; d < D; ++d)
    for (int64_t fj = 0; fj < fw; ++fj)
      for (int64_t fi = 0; fi < fh; ++fi) {
        const double* col = A + rows * (fi + fh * (fj + fw * d));
        for (int64_t oj = 0; oj < oW; ++oj) {
          int64_t jj = g[1] * oj + fj - g[4];
          if (jj < 0 || jj >= W) continue;
          for (int64_t oi = 0; oi < oH; ++oi) {
            int64_t ii = g[0] * oi + fi - g[2];
            if (ii >= 0 && ii < H) x[ii + H * (jj + W * d)] += col[oi + oH * oj];
          }
        }
      }
}

/* Exported for the SPEC im2row/row2im known-answer tests. */
int cko_im2row(const double* x, cko_shape xs, int64_t fh, int64_t fw, const int64_t* g,
               double* A, int64_t* rows, int64_t* cols) {
  int64_t oH, oW;
  int r;
  if ((r = cko_conv_output_extent(xs.h, fh, g[0], g[2], g[3], &oH))) return r;
  if ((r = cko_conv_output_extent(xs.w, fw, g[1], g[4], g[5], &oW))) return r;
  *rows = oH * oW;
  *cols = fh * fw * xs.c;
  if (A) im2row_image(x, xs.h, xs.w, xs.c, fh, fw, g, oH, oW, A);
  return CKO_OK;
}

int cko_row2im(const double* A, cko_shape target, int64_t fh, int64_t fw, const int64_t* g,
               double* x) {
  int64_t oH, oW;
  int r;
  if ((r = cko_conv_output_extent(target.h, fh, g[0], g[2], g[3], &oH))) return r;
  if ((r = cko_conv_output_extent(target.w, fw, g[1], g[4], g[5], &oW))) return r;
  memset(x, 0, sizeof(double) * (size_t)elems(target));
  row2im_image(A, target.h, target.w, target.c, fh, fw, g, oH, oW, x);
  return CKO_OK;
}

/* y = conv(x,f) + bias: per image im2row then one product per group,
 * bias after the product (conv.cpp:193-226). */
int cko_conv_forward(const double* x, cko_shape xs, const double* f, cko_shape fs,
                     const double* bias, const int64_t* g, double* y) {
  cko_shape ys;
  int r = cko_conv_output_shape(xs, fs, g, &ys);
  if (r) return r;
  const int64_t rows = ys.h * ys.w, patch = fs.h * fs.w * xs.c;
  const int64_t gcols = fs.h * fs.w * fs.c, gfil = fs.n / g[6];
  double* A = (double*)malloc(sizeof(double) * (size_t)(rows * patch));
  for (int64_t n = 0; n < xs.n; ++n) {
    im2row_image(x + xs.h * xs.w * xs.c * n, xs.h, xs.w, xs.c, fs.h, fs.w, g, ys.h, ys.w, A);
    double* Y = y + rows * ys.c * n;
    for (int64_t t = 0; t < g[6]; ++t)
      for (int64_t k = 0; k < gfil; ++k) {
        const double* F = f + gcols * (t * gfil + k);
        double* Yc = Y + rows * (t * gfil + k);
        for (int64_t p = 0; p < rows; ++p) {
          double acc = 0.0;
          const double* Ap = A + rows * (t * gcols) + p;
          for (int64_t q = 0; q < gcols; ++q) acc += Ap[rows * q] * F[q];
          Yc[p] = acc;
        }
      }
    if (bias)
      for (int64_t k = 0; k < ys.c; ++k)
        for (int64_t p = 0; p < rows; ++p) Y[p + rows * k] += bias[k];
  }
  free(A);
  return CKO_OK;
}

/* conv.cpp:229-280: db = sum dy; dF += A^T P per image/group; dX = row2im(P F^T). */
int cko_conv_backward(const double* x, cko_shape xs, const double* f, cko_shape fs,
                      const int64_t* g, const double* dy, double* dx, double* df, double* db) {
  cko_shape ys;
  int r = cko_conv_output_shape(xs, fs, g, &ys);
  if (r) return r;
  const int64_t rows = ys.h * ys.w, patch = fs.h * fs.w * xs.c;
  const int64_t gcols = fs.h * fs.w * fs.c, gfil = fs.n / g[6];
  if (dx) memset(dx, 0, sizeof(double) * (size_t)elems(xs));
  if (df) memset(df, 0, sizeof(double) * (size_t)elems(fs));
  if (db) {
    memset(db, 0, sizeof(double) * (size_t)fs.n);
    for (int64_t n = 0; n < ys.n; ++n)
      for (int64_t k = 0; k < ys.c; ++k) {
        double s = 0.0;
        for (int64_t p = 0; p < rows; ++p) s += dy[p + rows * (k + ys.c * n)];
        db[k] += s;
      }
  }
  if (!dx && !df) return CKO_OK;
  double* A = (double*)malloc(sizeof(double) * (size_t)(rows * patch));
  double* M = (double*)malloc(sizeof(double) * (size_t)(rows * patch));
  for (int64_t n = 0; n < xs.n; ++n) {
    const double* P = dy + rows * ys.c * n;
    if (df) {
      im2row_image(x + xs.h * xs.w * xs.c * n, xs.h, xs.w, xs.c, fs.h, fs.w, g, ys.h, ys.w, A);
      for (int64_t t = 0; t < g[6]; ++t)
        for (int64_t k = 0; k < gfil; ++k)
          for (int64_t q = 0; q < gcols; ++q) {
            double acc = 0.0;
            const double* Aq = A + rows * (t * gcols + q);
            const double* Pk = P + rows * (t * gfil + k);
            for (int64_t p = 0; p < rows; ++p) acc += Aq[p] * Pk[p];
            df[q + gcols * (t * gfil + k)] += acc;
          }
    }
    if (dx) {
      for (int64_t t = 0; t < g[6]; ++t)
        for (int64_t q = 0; q < gcols; ++q)
          for (int64_t p = 0; p < rows; ++p) {
            double acc = 0.0;
            for (int64_t k = 0; k < gfil; ++k)
              acc += P[p + rows * (t * gfil + k)] * f[q + gcols * (t * gfil + k)];
            M[p + rows * (t * gcols + q)] = acc;
          }
      row2im_image(M, xs.h, xs.w, xs.c, fs.h, fs.w, g, ys.h, ys.w, dx + xs.h * xs.w * xs.c * n);
    }
  }
  free(A);
  free(M);
  return CKO_OK;
}

static void convt_as_conv(const int64_t* cg, int64_t* g) {
  g[0] = cg[0]; g[1] = cg[1]; g[2] = cg[2]; g[3] = cg[3]; g[4] = cg[4]; g[5] = cg[5]; g[6] = 1;
}

/* convt_forward (conv.cpp:283-308): y = row2im(X Ft^T), Ft((i',j',k),d) = f(i',j',d,k). */
int cko_convt_forward(const double* x, cko_shape xs, const double* f, cko_shape fs,
                      const int64_t* cg, double* y) {
  cko_shape ys;
  int r = cko_convt_output_shape(xs, fs, cg, &ys);
  if (r) return r;
  int64_t g[7];
  convt_as_conv(cg, g);
  const int64_t rows = xs.h * xs.w, ftr = fs.h * fs.w * fs.n, D = fs.c;
  double* M = (double*)malloc(sizeof(double) * (size_t)(rows * ftr));
  memset(y, 0, sizeof(double) * (size_t)elems(ys));
  for (int64_t n = 0; n < xs.n; ++n) {
    const double* X = x + rows * xs.c * n;
    for (int64_t k = 0; k < fs.n; ++k)
      for (int64_t fj = 0; fj < fs.w; ++fj)
        for (int64_t fi = 0; fi < fs.h; ++fi) {
          int64_t col = fi + fs.h * (fj + fs.w * k);
          for (int64_t p = 0; p < rows; ++p) {
            double acc = 0.0;
            for (int64_t d = 0; d < D; ++d)
              acc += X[p + rows * d] * f[fi + fs.h * (fj + fs.w * (d + D * k))];
            M[p + rows * col] = acc;
          }
        }
    row2im_image(M, ys.h, ys.w, ys.c, fs.h, fs.w, g, xs.h, xs.w, y + ys.h * ys.w * ys.c * n);
  }
  free(M);
  return CKO_OK;
}

/* convt_backward (conv.cpp:311-365): dx = conv(dy, swapped bank); df from
 * im2row(dy)^T X. */
int cko_convt_backward(const double* x, cko_shape xs, const double* f, cko_shape fs,
                       const int64_t* cg, const double* dy, double* dx, double* df) {
  cko_shape ys;
  int r = cko_convt_output_shape(xs, fs, cg, &ys);
  if (r) return r;
  int64_t g[7];
  convt_as_conv(cg, g);
  if (dx) {
    cko_shape bs = {fs.h, fs.w, fs.n, fs.c};
    double* bank = (double*)malloc(sizeof(double) * (size_t)elems(fs));
    for (int64_t k = 0; k < fs.n; ++k)
      for (int64_t d = 0; d < fs.c; ++d)
        for (int64_t fj = 0; fj < fs.w; ++fj)
          for (int64_t fi = 0; fi < fs.h; ++fi)
            bank[IDX(bs, fi, fj, k, d)] = f[IDX(fs, fi, fj, d, k)];
    r = cko_conv_forward(dy, ys, bank, bs, NULL, g, dx);
    free(bank);
    if (r) return r;
  }
  if (df) {
    const int64_t rows = xs.h * xs.w, K = fs.h * fs.w * fs.n;
    double* A = (double*)malloc(sizeof(double) * (size_t)(rows * K));
    double* dFt = (double*)calloc((size_t)(K * fs.c), sizeof(double));
    for (int64_t n = 0; n < xs.n; ++n) {
      im2row_image(dy + ys.h * ys.w * ys.c * n, ys.h, ys.w, ys.c, fs.h, fs.w, g, xs.h, xs.w, A);
      const double* X = x + rows * xs.c * n;
      for (int64_t d = 0; d < fs.c; ++d)
        for (int64_t q = 0; q < K; ++q) {
          double acc = 0.0;
          for (int64_t p = 0; p < rows; ++p) acc += A[p + rows * q] * X[p + rows * d];
          dFt[q + K * d] += acc;
        }
    }
    for (int64_t d = 0; d < fs.c; ++d)
      for (int64_t k = 0; k < fs.n; ++k)
        for (int64_t fj = 0; fj < fs.w; ++fj)
          for (int64_t fi = 0; fi < fs.h; ++fi)
            df[IDX(fs, fi, fj, d, k)] = dFt[(fi + fs.h * (fj + fs.w * k)) + K * d];
    free(A);
    free(dFt);
  }
  return CKO_OK;
}

/* ---- pooling (pool.cpp:24-126), float, reference operation order ------- */

static void window_at(cko_shape xs, const int64_t* pg, int64_t oi, int64_t oj, int64_t* b) {
  int64_t i0 = pg[2] * oi - pg[4], j0 = pg[3] * oj - pg[6];
  b[0] = i0 < 0 ? 0 : i0;
  b[1] = i0 + pg[0] < xs.h ? i0 + pg[0] : xs.h;
  b[2] = j0 < 0 ? 0 : j0;
  b[3] = j0 + pg[1] < xs.w ? j0 + pg[1] : xs.w;
}

int cko_pool_forward_f(const float* x, cko_shape xs, const int64_t* pg, float* y) {
  cko_shape ys;
  int r = cko_pool_output_shape(xs, pg, &ys);
  if (r) return r;
  for (int64_t n = 0; n < xs.n; ++n)
    for (int64_t c = 0; c < xs.c; ++c)
      for (int64_t oj = 0; oj < ys.w; ++oj)
        for (int64_t oi = 0; oi < ys.h; ++oi) {
          int64_t b[4];
          window_at(xs, pg, oi, oj, b);
          if (pg[8] == 0) {
            float best = x[IDX(xs, b[0], b[2], c, n)];
            for (int64_t j = b[2]; j < b[3]; ++j)
              for (int64_t i = b[0]; i < b[1]; ++i) {
                float v = x[IDX(xs, i, j, c, n)];
                if (v > best) best = v;
              }
            y[IDX(ys, oi, oj, c, n)] = best;
          } else {
            float sum = 0.0f;
            for (int64_t j = b[2]; j < b[3]; ++j)
              for (int64_t i = b[0]; i < b[1]; ++i) sum += x[IDX(xs, i, j, c, n)];
            float area = (float)((b[1] - b[0]) * (b[3] - b[2]));
            y[IDX(ys, oi, oj, c, n)] = sum / area;
          }
        }
  return CKO_OK;
}

int cko_pool_backward_f(const float* x, cko_shape xs, const int64_t* pg, const float* dy,
                        float* dx) {
  cko_shape ys;
  int r = cko_pool_output_shape(xs, pg, &ys);
  if (r) return r;
  memset(dx, 0, sizeof(float) * (size_t)elems(xs));
  for (int64_t n = 0; n < xs.n; ++n)
    for (int64_t c = 0; c < xs.c; ++c)
      for (int64_t oj = 0; oj < ys.w; ++oj)
        for (int64_t oi = 0; oi < ys.h; ++oi) {
          int64_t b[4];
          window_at(xs, pg, oi, oj, b);
          float p = dy[IDX(ys, oi, oj, c, n)];
          if (pg[8] == 0) {
            int64_t bi = b[0], bj = b[2];
            float best = x[IDX(xs, b[0], b[2], c, n)];
            for (int64_t j = b[2]; j < b[3]; ++j)
              for (int64_t i = b[0]; i < b[1]; ++i) {
                float v = x[IDX(xs, i, j, c, n)];
                if (v > best) { best = v; bi = i; bj = j; }
              }
            dx[IDX(xs, bi, bj, c, n)] += p;
          } else {
            float area = (float)((b[1] - b[0]) * (b[3] - b[2]));
            float share = p / area;
            for (int64_t j = b[2]; j < b[3]; ++j)
              for (int64_t i = b[0]; i < b[1]; ++i) dx[IDX(xs, i, j, c, n)] += share;
          }
        }
  return CKO_OK;
}

/* ---- relu (activation.cpp:8-22), float ---------------------------------- */

void cko_relu_forward_f(const float* x, int64_t n, float* y) {
  for (int64_t k = 0; k < n; ++k) y[k] = x[k] > 0.0f ? x[k] : 0.0f;
}

void cko_relu_backward_f(const float* x, const float* dy, int64_t n, float* dx) {
  for (int64_t k = 0; k < n; ++k) dx[k] = x[k] > 0.0f ? dy[k] : 0.0f;
}

/* ---- LRN (normalize.cpp:18-118) ----------------------------------------- */

static void lrn_group(int64_t k, int64_t size, int64_t count, int64_t* lo, int64_t* hi) {
  int64_t down = (size - 1) / 2, up = size - 1 - down;
  *lo = k - down < 0 ? 0 : k - down;
  *hi = k + up < count - 1 ? k + up : count - 1;
}

static int check_lrn(int64_t size, double kappa) {
  if (size < 1) return fail(CKO_SHAPE, "lrn group size must be positive");
  if (kappa <= 0) return fail(CKO_SHAPE, "lrn kappa must be positive");
  return CKO_OK;
}

int cko_lrn_forward(const double* x, cko_shape s, int64_t size, double kappa, double alpha,
                    double beta, double* y) {
  int r = check_lrn(size, kappa);
  if (r) return r;
  for (int64_t n = 0; n < s.n; ++n)
    for (int64_t j = 0; j < s.w; ++j)
      for (int64_t i = 0; i < s.h; ++i)
        for (int64_t k = 0; k < s.c; ++k) {
          int64_t lo, hi;
          lrn_group(k, size, s.c, &lo, &hi);
          double acc = 0.0;
          for (int64_t t = lo; t <= hi; ++t) {
            double v = x[IDX(s, i, j, t, n)];
            acc += v * v;
          }
          y[IDX(s, i, j, k, n)] = x[IDX(s, i, j, k, n)] * pow(kappa + alpha * acc, -beta);
        }
  return CKO_OK;
}

int cko_lrn_backward(const double* x, cko_shape s, int64_t size, double kappa, double alpha,
                     double beta, const double* dy, double* dx) {
  int r = check_lrn(size, kappa);
  if (r) return r;
  double* L = (double*)malloc(sizeof(double) * (size_t)s.c);
  double* eta = (double*)malloc(sizeof(double) * (size_t)s.c);
  int64_t down = (size - 1) / 2, up = size - 1 - down;
  for (int64_t n = 0; n < s.n; ++n)
    for (int64_t j = 0; j < s.w; ++j)
      for (int64_t i = 0; i < s.h; ++i) {
        for (int64_t k = 0; k < s.c; ++k) {
          int64_t lo, hi;
          lrn_group(k, size, s.c, &lo, &hi);
          double acc = 0.0;
          for (int64_t t = lo; t <= hi; ++t) {
            double v = x[IDX(s, i, j, t, n)];
            acc += v * v;
          }
          L[k] = kappa + alpha * acc;
          eta[k] = dy[IDX(s, i, j, k, n)] * pow(L[k], -beta - 1.0) * x[IDX(s, i, j, k, n)];
        }
        for (int64_t d = 0; d < s.c; ++d) {
          double acc = 0.0;
          int64_t klo = d - up < 0 ? 0 : d - up, khi = d + down < s.c - 1 ? d + down : s.c - 1;
          for (int64_t k = klo; k <= khi; ++k) acc += eta[k];
          dx[IDX(s, i, j, d, n)] = dy[IDX(s, i, j, d, n)] * pow(L[d], -beta) -
                                   2.0 * alpha * beta * x[IDX(s, i, j, d, n)] * acc;
        }
      }
  free(L);
  free(eta);
  return CKO_OK;
}

/* ---- batch normalisation (normalize.cpp:122-265) ------------------------ */

static int check_bnorm(double eps) {
  if (!(eps > 0)) return fail(CKO_SHAPE, "bnorm epsilon must be positive");
  return CKO_OK;
}

/* Two sequential passes: mean, then biased variance (normalize.cpp:132-161). */
static void batch_moments(const double* x, cko_shape s, double* mean, double* var) {
  const double count = (double)(s.h * s.w * s.n);
  for (int64_t k = 0; k < s.c; ++k) mean[k] = var[k] = 0.0;
  for (int64_t n = 0; n < s.n; ++n)
    for (int64_t k = 0; k < s.c; ++k)
      for (int64_t p = 0; p < s.h * s.w; ++p) mean[k] += x[p + s.h * s.w * (k + s.c * n)];
  for (int64_t k = 0; k < s.c; ++k) mean[k] /= count;
  for (int64_t n = 0; n < s.n; ++n)
    for (int64_t k = 0; k < s.c; ++k)
      for (int64_t p = 0; p < s.h * s.w; ++p) {
        double d = x[p + s.h * s.w * (k + s.c * n)] - mean[k];
        var[k] += d * d;
      }
  for (int64_t k = 0; k < s.c; ++k) var[k] /= count;
}

static void bnorm_apply(const double* x, cko_shape s, const double* w, const double* b,
                        double eps, const double* mean, const double* var, double* y) {
  for (int64_t n = 0; n < s.n; ++n)
    for (int64_t k = 0; k < s.c; ++k) {
      double inv = 1.0 / sqrt(var[k] + eps);
      for (int64_t p = 0; p < s.h * s.w; ++p) {
        int64_t e = p + s.h * s.w * (k + s.c * n);
        y[e] = w[k] * (x[e] - mean[k]) * inv + b[k];
      }
    }
}

int cko_bnorm_forward(const double* x, cko_shape s, const double* w, const double* b,
                      double eps, double* y, double* mean, double* var) {
  int r = check_bnorm(eps);
  if (r) return r;
  double* m = (double*)malloc(sizeof(double) * (size_t)s.c * 2);
  batch_moments(x, s, m, m + s.c);
  bnorm_apply(x, s, w, b, eps, m, m + s.c, y);
  if (mean) memcpy(mean, m, sizeof(double) * (size_t)s.c);
  if (var) memcpy(var, m + s.c, sizeof(double) * (size_t)s.c);
  free(m);
  return CKO_OK;
}

int cko_bnorm_infer(const double* x, cko_shape s, const double* w, const double* b, double eps,
                    const double* mean, const double* var, double* y) {
  int r = check_bnorm(eps);
  if (r) return r;
  bnorm_apply(x, s, w, b, eps, mean, var, y);
  return CKO_OK;
}

/* normalize.cpp:212-265: recomputes the moments from x. */
int cko_bnorm_backward(const double* x, cko_shape s, const double* w, const double* b,
                       double eps, const double* dy, double* dx, double* dw, double* db) {
  (void)b;
  int r = check_bnorm(eps);
  if (r) return r;
  const double count = (double)(s.h * s.w * s.n);
  double* m = (double*)malloc(sizeof(double) * (size_t)s.c * 4);
  double *mean = m, *var = m + s.c, *sdy = m + 2 * s.c, *sdyx = m + 3 * s.c;
  batch_moments(x, s, mean, var);
  for (int64_t k = 0; k < s.c; ++k) sdy[k] = sdyx[k] = 0.0;
  for (int64_t n = 0; n < s.n; ++n)
    for (int64_t k = 0; k < s.c; ++k) {
      double inv = 1.0 / sqrt(var[k] + eps);
      for (int64_t p = 0; p < s.h * s.w; ++p) {
        int64_t e = p + s.h * s.w * (k + s.c * n);
        sdy[k] += dy[e];
        sdyx[k] += dy[e] * (x[e] - mean[k]) * inv;
      }
    }
  if (dw) memcpy(dw, sdyx, sizeof(double) * (size_t)s.c);
  if (db) memcpy(db, sdy, sizeof(double) * (size_t)s.c);
  if (dx)
    for (int64_t n = 0; n < s.n; ++n)
      for (int64_t k = 0; k < s.c; ++k) {
        double inv = 1.0 / sqrt(var[k] + eps);
        double mdy = sdy[k] / count, mdyx = sdyx[k] / count;
        for (int64_t p = 0; p < s.h * s.w; ++p) {
          int64_t e = p + s.h * s.w * (k + s.c * n);
          double xhat = (x[e] - mean[k]) * inv;
          dx[e] = w[k] * inv * (dy[e] - mdy - xhat * mdyx);
        }
      }
  free(m);
  return CKO_OK;
}

/* ---- softmaxlog loss and the top-1 / top-k metrics (loss.cpp) ---------- */

/* loss.cpp:14-18 as_label + :35-40 check_classification + :101-106 range. */
static int label_at(const double* labels, int64_t e, int64_t C, int64_t* c) {
  double v = labels[e], rr = nearbyint(v);
  if (rr != v) return fail(CKO_DATA, "class label is not an integer");
  *c = (int64_t)rr;
  if (*c == 0) return CKO_OK;
  if (*c < 1 || *c > C) {
    char b[128];
    snprintf(b, sizeof b, "class label %lld out of range 1..%lld", (long long)*c, (long long)C);
    return fail(CKO_DATA, b);
  }
  return CKO_OK;
}

static int check_cls(cko_shape xs, cko_shape cs) {
  if (cs.h != xs.h || cs.w != xs.w || cs.c != 1 || cs.n != xs.n)
    return fail(CKO_SHAPE, "classification labels must be HxWx1xN");
  return CKO_OK;
}

/* kind: 0 softmaxlog (loss.cpp:156-165), 1 classerror (:111-141, lowest index
 * wins ties), 2 topk (:142-149).  Sum over sites, weighted (:182). */
int cko_loss_forward(const double* x, cko_shape xs, const double* labels, cko_shape cs,
                     const double* weights, int kind, int64_t top_k, double* out) {
  int r = check_cls(xs, cs);
  if (r) return r;
  const int64_t C = xs.c;
  double total = 0.0;
  for (int64_t n = 0; n < xs.n; ++n)
    for (int64_t j = 0; j < xs.w; ++j)
      for (int64_t i = 0; i < xs.h; ++i) {
        int64_t e = IDX(cs, i, j, 0, n), c;
        if ((r = label_at(labels, e, C, &c))) return r;
        if (c == 0) continue;
        double wgt = weights ? weights[e] : 1.0;
        double xc = x[IDX(xs, i, j, c - 1, n)], l = 0.0;
        if (kind == 0) {
          double mx = x[IDX(xs, i, j, 0, n)];
          for (int64_t k = 1; k < C; ++k) {
            double v = x[IDX(xs, i, j, k, n)];
            if (v > mx) mx = v;
          }
          double sum = 0.0;
          for (int64_t k = 0; k < C; ++k) sum += exp(x[IDX(xs, i, j, k, n)] - mx);
          l = -xc + mx + log(sum);
        } else if (kind == 1) {
          int64_t best = 0;
          double bv = x[IDX(xs, i, j, 0, n)];
          for (int64_t k = 1; k < C; ++k) {
            double v = x[IDX(xs, i, j, k, n)];
            if (v > bv) { bv = v; best = k; }
          }
          l = (best == c - 1) ? 0.0 : 1.0;
        } else {
          int64_t rank = 0;
          for (int64_t k = 0; k < C; ++k)
            if (x[IDX(xs, i, j, k, n)] >= xc) ++rank;
          l = rank <= top_k ? 0.0 : 1.0;
        }
        total += wgt * l;
      }
  *out = total;
  return CKO_OK;
}

/* loss.cpp:231-275: dx_k = p * w * (softmax_k - [k == c]). */
int cko_softmaxlog_backward(const double* x, cko_shape xs, const double* labels, cko_shape cs,
                            const double* weights, double p, double* dx) {
  int r = check_cls(xs, cs);
  if (r) return r;
  const int64_t C = xs.c;
  memset(dx, 0, sizeof(double) * (size_t)elems(xs));
  for (int64_t n = 0; n < xs.n; ++n)
    for (int64_t j = 0; j < xs.w; ++j)
      for (int64_t i = 0; i < xs.h; ++i) {
        int64_t e = IDX(cs, i, j, 0, n), c;
        if ((r = label_at(labels, e, C, &c))) return r;
        if (c == 0) continue;
        double scale = p * (weights ? weights[e] : 1.0);
        double mx = x[IDX(xs, i, j, 0, n)];
        for (int64_t k = 1; k < C; ++k) {
          double v = x[IDX(xs, i, j, k, n)];
          if (v > mx) mx = v;
        }
        double sum = 0.0;
        for (int64_t k = 0; k < C; ++k) sum += exp(x[IDX(xs, i, j, k, n)] - mx);
        for (int64_t k = 0; k < C; ++k) {
          double soft = exp(x[IDX(xs, i, j, k, n)] - mx) / sum;
          dx[IDX(xs, i, j, k, n)] += scale * (soft - (k == c - 1 ? 1.0 : 0.0));
        }
      }
  return CKO_OK;
}

/* ---- SGD with momentum (trainer.cpp absent), float --------- */

void cko_sgd_step_f(float* w, float* v, const float* g, int64_t n, float lr, float momentum,
                    float wd) {
  for (int64_t k = 0; k < n; ++k) {
    v[k] = momentum * v[k] - lr * (g[k] + wd * w[k]);
    w[k] = w[k] + v[k];
  }
}

/* ---- xoshiro256** seeded via splitmix64 (rng.cpp:10-59) ----------------- */

typedef struct {
  uint64_t s[4];
} cko_rng;

static uint64_t splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static void rng_seed(cko_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  for (int k = 0; k < 4; ++k) r->s[k] = splitmix64(&sm);
}

static uint64_t rng_next(cko_rng* r) {
  uint64_t* s = r->s;
  uint64_t result = rotl(s[1] * 5, 7) * 9;
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

static double rng_uniform(cko_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_normal(cko_rng* r) {
  double u1 = 1.0 - rng_uniform(r);
  double u2 = rng_uniform(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* A stateful generator handle so several tensors can be drawn from one
 * stream in network order (the bench's weight initialisation). */
cko_rng* cko_rng_new(uint64_t seed) {
  cko_rng* r = (cko_rng*)malloc(sizeof(cko_rng));
  rng_seed(r, seed);
  return r;
}
void cko_rng_free(cko_rng* r) { free(r); }
uint64_t cko_rng_next(cko_rng* r) { return rng_next(r); }

/* oracles.hpp:16-23 random_uniform: lo + (hi-lo) * T(uniform()). */
void cko_rng_fill_uniform_f(cko_rng* r, float* out, int64_t n, float lo, float hi) {
  for (int64_t k = 0; k < n; ++k) out[k] = lo + (hi - lo) * (float)rng_uniform(r);
}
/* SPEC.md:757 weight init: scale * normal(). */
void cko_rng_fill_normal_f(cko_rng* r, float* out, int64_t n, float scale) {
  for (int64_t k = 0; k < n; ++k) out[k] = (float)(scale * rng_normal(r));
}
/* Labels 1 + below(C) (rng.cpp:49). */
void cko_rng_fill_labels_f(cko_rng* r, float* out, int64_t n, uint64_t C) {
  for (int64_t k = 0; k < n; ++k) out[k] = (float)(1 + (C ? rng_next(r) % C : 0));
}
