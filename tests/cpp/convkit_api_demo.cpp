// Exercises the convkit-shaped C++ API (include/ck/convkit.hpp) end to end:
// identity filter bank, relu, pooling, a shape error.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ck/convkit.hpp"

using namespace ck::convkit;

int main() {
  const int H = 7, W = 6, C = 3, N = 2;
  std::vector<float> xh(H * W * C * N);
  for (size_t i = 0; i < xh.size(); ++i) xh[i] = std::sin(0.37f * i);
  DeviceTensor x(Shape(H, W, C, N), xh);
  std::vector<float> fh(C * C, 0.f);
  for (int d = 0; d < C; ++d) fh[d + C * d] = 1.f;  // f[0,0,d,k] = [d == k]
  DeviceTensor f(Shape(1, 1, C, C), fh);
  Context::current().set_math(CK_MATH_FP32);
  DeviceTensor y = conv_forward(x, f, nullptr, conv_geom());
  std::vector<float> yh = y.to_host();
  for (size_t i = 0; i < xh.size(); ++i)
    if (yh[i] != xh[i]) { std::printf("identity conv mismatch at %zu\n", i); return 1; }
  DeviceTensor r = relu_forward(x);
  std::vector<float> rh = r.to_host();
  for (size_t i = 0; i < xh.size(); ++i)
    if (rh[i] != (xh[i] > 0 ? xh[i] : 0.f)) { std::printf("relu mismatch\n"); return 1; }
  PoolGeom pg{3, 3, 2, 2, 0, 1, 0, 1, CK_POOL_MAX};
  DeviceTensor p = pool_forward(x, pg);
  if (!(p.shape() == Shape(3, 3, C, N))) { std::printf("pool shape\n"); return 1; }
  try {
    DeviceTensor bad(Shape(3, 3, 2, 4));
    conv_forward(x, bad, nullptr, conv_geom());
    std::printf("expected ShapeError\n");
    return 1;
  } catch (const ShapeError& e) {
    std::printf("ShapeError ok: %s\n", e.what());
  }
  std::printf("convkit C++ API ok\n");
  return 0;
}
