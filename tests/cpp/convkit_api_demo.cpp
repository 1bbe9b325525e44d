// Exercises the convkit-shaped C++ API (include/ck/convkit.hpp) end to end:
// every block's forward AND backward on the SPEC.md known answers, the
// BnormMoments / LossKind / LossOptions signatures of the reference headers,
// blob round trip and a shape error.  Exit code 0 = all good.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "ck/convkit.hpp"

using namespace ck::convkit;

static int failures = 0;

static void expect(const char* what, const std::vector<float>& got, const std::vector<float>& want,
                   float tol = 1e-5f) {
  bool ok = got.size() == want.size();
  for (size_t i = 0; ok && i < got.size(); ++i) ok = std::fabs(got[i] - want[i]) <= tol;
  if (!ok) {
    ++failures;
    std::printf("FAIL %s: got", what);
    for (float v : got) std::printf(" %g", v);
    std::printf(" want");
    for (float v : want) std::printf(" %g", v);
    std::printf("\n");
  }
}

static DeviceTensor T(Shape s, std::vector<float> v) { return DeviceTensor(s, v); }

int main() {
  Context::current().set_math(CK_MATH_FP32);
  // conv: identity filter bank gives y = x
  {
    const int H = 7, W = 6, C = 3, N = 2;
    std::vector<float> xh(H * W * C * N);
    for (size_t i = 0; i < xh.size(); ++i) xh[i] = std::sin(0.37f * i);
    std::vector<float> fh(C * C, 0.f);
    for (int d = 0; d < C; ++d) fh[d + C * d] = 1.f;
    DeviceTensor y = conv_forward(T(Shape(H, W, C, N), xh), T(Shape(1, 1, C, C), fh), nullptr,
                                  conv_geom());
    expect("conv identity", y.to_host(), xh, 0.f);
  }
  // conv [1,2,3] * [1,1] = [3,5]; backward with dy = [1,1]
  {
    DeviceTensor x = T(Shape(3), {1, 2, 3}), f = T(Shape(2), {1, 1}), b = T(Shape(1), {0.5f});
    expect("conv fwd", conv_forward(x, f, &b, conv_geom()).to_host(), {3.5f, 5.5f});
    DeviceTensor dx, df, db;
    conv_backward(x, f, conv_geom(), T(Shape(2), {1, 1}), &dx, &df, &db);
    expect("conv dx", dx.to_host(), {1, 2, 1});
    expect("conv df", df.to_host(), {3, 5});
    expect("conv db", db.to_host(), {2});
  }
  // convt x = [1,1], f = [1,2,3], U = 2 -> [1,2,4,2,3]
  {
    DeviceTensor x = T(Shape(2), {1, 1}), f = T(Shape(3), {1, 2, 3});
    ConvTransposeGeom g{2, 1, 0, 0, 0, 0};
    expect("convt fwd", convt_forward(x, f, g).to_host(), {1, 2, 4, 2, 3});
    DeviceTensor dx, df;
    convt_backward(x, f, g, T(Shape(5), {1, 1, 1, 1, 1}), &dx, &df);
    expect("convt dx", dx.to_host(), {6, 6});
    expect("convt df", df.to_host(), {2, 2, 2});
  }
  // pool [1,3,2] k2 s1 max -> [3,3], backward routes to the argmax
  {
    DeviceTensor x = T(Shape(3), {1, 3, 2});
    PoolGeom g{2, 1, 1, 1, 0, 0, 0, 0, CK_POOL_MAX};
    expect("pool fwd", pool_forward(x, g).to_host(), {3, 3});
    expect("pool bwd", pool_backward(x, g, T(Shape(2), {1, 1})).to_host(), {0, 2, 0});
    PoolGeom a{2, 1, 1, 1, 0, 1, 0, 0, CK_POOL_AVG};  // [4], k2, pad(0,1) avg -> [4] (:223)
    expect("avg pool cropped area", pool_forward(T(Shape(1), {4}), a).to_host(), {4});
  }
  // relu
  {
    DeviceTensor x = T(Shape(2), {-1, 2});
    expect("relu fwd", relu_forward(x).to_host(), {0, 2});
    expect("relu bwd", relu_backward(x, T(Shape(2), {5, 7})).to_host(), {0, 7});
  }
  // lrn: alpha = 0, kappa = 1 is the identity; D=1, x=1,
  // kappa=alpha=1, beta=0.5 -> 1/sqrt(2) (:323)
  {
    DeviceTensor x = T(Shape(1, 1, 3, 1), {1, -2, 3});
    LrnParams id{5, 1.0, 0.0, 0.75};
    expect("lrn identity", lrn_forward(x, id).to_host(), {1, -2, 3});
    expect("lrn identity bwd", lrn_backward(x, id, T(Shape(1, 1, 3, 1), {4, 5, 6})).to_host(),
           {4, 5, 6});
    LrnParams p{1, 1.0, 1.0, 0.5};
    expect("lrn 1/sqrt2", lrn_forward(T(Shape(1), {1}), p).to_host(), {0.70710678f});
  }
  // bnorm: x = [0, 2] -> mean 1, var 1; constant dy -> dx = 0
  {
    DeviceTensor x = T(Shape(2), {0, 2}), w = T(Shape(1), {1}), b = T(Shape(1), {0.25f});
    BnormMoments<float> m;
    DeviceTensor y = bnorm_forward(x, w, b, 1e-5, &m);
    expect("bnorm moments", {m.mean[0], m.var[0]}, {1, 1});
    const float s = 1.f / std::sqrt(1.f + 1e-5f);
    expect("bnorm fwd", y.to_host(), {0.25f - s, 0.25f + s});
    expect("bnorm infer", bnorm_infer(x, w, b, 1e-5, m).to_host(), {0.25f - s, 0.25f + s});
    DeviceTensor dx, dw, db;
    bnorm_backward(x, w, b, 1e-5, T(Shape(2), {1, 1}), &dx, &dw, &db);
    expect("bnorm dx", dx.to_host(), {0, 0});
    expect("bnorm dw", dw.to_host(), {0});
    expect("bnorm db", db.to_host(), {2});
  }
  // softmaxlog C=2, x=[0,0], c=1 -> log 2, dzdx = [-0.5, 0.5]
  {
    DeviceTensor x = T(Shape(1, 1, 2, 1), {0, 0}), c = T(Shape(1), {1});
    expect("softmaxlog fwd", {loss_forward(x, c, LossKind::softmaxlog)}, {std::log(2.f)});
    expect("softmaxlog bwd", loss_backward(x, c, LossKind::softmaxlog, nullptr, 1.f).to_host(),
           {-0.5f, 0.5f});
    DeviceTensor p = T(Shape(1, 1, 2, 1), {0.2f, 0.8f});
    DeviceTensor c2 = T(Shape(1), {2});
    expect("log loss", {loss_forward(p, c2, LossKind::log)}, {-std::log(0.8f)});
    expect("log loss bwd", loss_backward(p, c2, LossKind::log, nullptr, 1.f).to_host(),
           {0, -1.25f});
    LossOptions o;
    o.top_k = 1;
    expect("topk", {loss_forward(p, T(Shape(1), {1}), LossKind::topk, nullptr, o)}, {1});
    expect("classerror", {loss_forward(p, c2, LossKind::classerror)}, {0});
    expect("hinge", {loss_forward(T(Shape(2), {0.5f, -2}), T(Shape(2), {1, -1}), LossKind::hinge)},
           {0.5f});
    try {
      loss_forward(x, T(Shape(1), {3}), LossKind::softmaxlog);
      std::printf("FAIL expected DataError\n");
      ++failures;
    } catch (const DataError& e) {
      std::printf("DataError ok: %s\n", e.what());
    }
  }
  // sigmoid / softmax / spnorm
  {
    expect("sigmoid fwd", sigmoid_forward(T(Shape(1), {0})).to_host(), {0.5f});
    expect("sigmoid bwd", sigmoid_backward(T(Shape(1), {0.5f}), T(Shape(1), {1})).to_host(),
           {0.25f});
    DeviceTensor y = softmax_forward(T(Shape(1, 1, 2, 1), {0, 0}));
    expect("softmax fwd", y.to_host(), {0.5f, 0.5f});
    expect("softmax bwd", softmax_backward(y, T(Shape(1, 1, 2, 1), {1, 0})).to_host(),
           {0.25f, -0.25f});
    SpnormParams sp{1, 1, 1.0, 0.5};
    expect("spnorm fwd", spnorm_forward(T(Shape(1), {1}), sp).to_host(), {0.70710678f});
    // d/dx x (1 + x^2)^-1/2 at 1 = 2^-1.5
    expect("spnorm bwd", spnorm_backward(T(Shape(1), {1}), sp, T(Shape(1), {1})).to_host(),
           {0.35355339f});
  }
  // bilinear: the identity grid reproduces the input (bilinear.cpp:135-152)
  {
    DeviceTensor x = T(Shape(3, 2, 1, 1), {1, 2, 3, 4, 5, 6});
    DeviceTensor g = T(Shape(2, 3, 2, 1), {-1, -1, 0, -1, 1, -1, -1, 1, 0, 1, 1, 1});
    expect("bilinear identity", bilinear_forward(x, g).to_host(), {1, 2, 3, 4, 5, 6});
    DeviceTensor dx, dg;
    bilinear_backward(x, g, T(Shape(3, 2, 1, 1), {1, 1, 1, 1, 1, 1}), &dx, &dg);
    expect("bilinear dx", dx.to_host(), {1, 1, 1, 1, 1, 1});
  }
  // pdist: |[3,4] - 0|_2 = 5, gradient x / 5, dtarget = -dx (loss.cpp:346-428)
  {
    DeviceTensor x = T(Shape(1, 1, 2, 1), {3, 4}), t = T(Shape(1, 1, 2, 1), {0, 0});
    expect("pdist fwd", pdist_forward(x, t, 2.0, false).to_host(), {5});
    DeviceTensor dx, dt;
    pdist_backward(x, t, 2.0, false, T(Shape(1), {1}), &dx, &dt);
    expect("pdist dx", dx.to_host(), {0.6f, 0.8f});
    expect("pdist dt", dt.to_host(), {-0.6f, -0.8f});
  }
  // blob round trip (blob.cpp:29-79)
  {
    DeviceTensor x = T(Shape(2, 1, 3, 1), {1, -2, 3.5f, 0, 1e-30f, -7});
    const std::string path = "/tmp/ck_demo_blob.bin";
    write_blob(x, path);
    DeviceTensor y = read_blob(path);
    expect("blob round trip", y.to_host(), x.to_host(), 0.f);
    if (!(y.shape() == x.shape())) {
      ++failures;
      std::printf("FAIL blob shape\n");
    }
  }
  try {
    DeviceTensor x(Shape(7, 6, 3, 2)), bad(Shape(3, 3, 2, 4));
    conv_forward(x, bad, nullptr, conv_geom());
    std::printf("FAIL expected ShapeError\n");
    ++failures;
  } catch (const ShapeError& e) {
    std::printf("ShapeError ok: %s\n", e.what());
  }
  if (failures) {
    std::printf("%d failures\n", failures);
    return 1;
  }
  std::printf("convkit C++ API ok\n");
  return 0;
}
