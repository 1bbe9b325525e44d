// The capi.cpp-style shim of INTEGRATION.md §2 -- the binding a maintainer
// adds to the reference so its C entry points run on libck -- compiled and
// exercised as written there, against a direct ck.h call.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ck/ck.h"

// ---- INTEGRATION.md §2, verbatim ----
extern "C" int convkit_conv_forward(const float* x, const int64_t xs[4], const float* f,
                                    const int64_t fs[4], const float* bias,
                                    const int64_t geom[7], float* y, void* stream) {
  static thread_local ck_handle* h = [] { ck_handle* p; ck_create(&p, 0); return p; }();
  ck_tensor X{(float*)x, {xs[0], xs[1], xs[2], xs[3]}}, F{(float*)f, {fs[0], fs[1], fs[2], fs[3]}};
  ck_tensor B{(float*)bias, {1, 1, fs[3], 1}};
  ck_conv_geom g{geom[0], geom[1], geom[2], geom[3], geom[4], geom[5], geom[6]};
  ck_shape ys;
  if (int s = ck_conv_output_shape(h, X.shape, F.shape, &g, &ys)) return s;
  ck_tensor Y{y, ys};
  return ck_conv_forward(h, &X, &F, bias ? &B : nullptr, &g, &Y, CK_MATH_TF32, stream);
}
// ---- end of the shim ----

int main() {
  const int64_t xs[4] = {27, 27, 96, 4}, fs[4] = {5, 5, 48, 256}, geom[7] = {1, 1, 2, 2, 2, 2, 2};
  const size_t nx = 27 * 27 * 96 * 4, nf = 5 * 5 * 48 * 256, ny = 27 * 27 * 256 * 4;
  std::vector<float> hx(nx), hf(nf), hb(256);
  for (size_t i = 0; i < nx; ++i) hx[i] = (float)((i * 2654435761u) % 1000) / 1000.f - 0.5f;
  for (size_t i = 0; i < nf; ++i) hf[i] = (float)((i * 40503u) % 1000) / 50000.f - 0.01f;
  for (int i = 0; i < 256; ++i) hb[i] = 0.01f * i;
  float *x, *f, *b, *y1, *y2;
  cudaMalloc(&x, nx * 4);
  cudaMalloc(&f, nf * 4);
  cudaMalloc(&b, 256 * 4);
  cudaMalloc(&y1, ny * 4);
  cudaMalloc(&y2, ny * 4);
  cudaMemcpy(x, hx.data(), nx * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(f, hf.data(), nf * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb.data(), 256 * 4, cudaMemcpyHostToDevice);
  if (int s = convkit_conv_forward(x, xs, f, fs, b, geom, y1, nullptr)) {
    std::printf("shim failed: %d\n", s);
    return 1;
  }
  ck_handle* h;
  ck_create(&h, 0);
  ck_tensor X{x, {27, 27, 96, 4}}, F{f, {5, 5, 48, 256}}, B{b, {1, 1, 256, 1}}, Y{y2, {27, 27, 256, 4}};
  ck_conv_geom g{1, 1, 2, 2, 2, 2, 2};
  if (ck_conv_forward(h, &X, &F, &B, &g, &Y, CK_MATH_TF32, nullptr) != CK_OK) return 1;
  std::vector<float> a(ny), c(ny);
  cudaMemcpy(a.data(), y1, ny * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), y2, ny * 4, cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < ny; ++i)
    if (a[i] != c[i]) {
      std::printf("mismatch at %zu\n", i);
      return 1;
    }
  // the shim reports the reference's shape error through its status
  const int64_t bad[4] = {5, 5, 47, 256};
  if (convkit_conv_forward(x, xs, f, bad, b, geom, y1, nullptr) != CK_ERR_SHAPE) return 1;
  std::printf("capi shim ok\n");
  ck_destroy(h);
  return 0;
}
