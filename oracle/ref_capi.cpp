// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A small extern "C" surface over the reference convkit library compiled
// verbatim from /root/reference/proj/src (see oracle/Makefile).  It lets the
// Python tests and bench.py's CPU-baseline legs drive the reference's own
// block functions and its DAG engine (graph.cpp:494 forward, :548 backward)
// through ctypes.  Nothing here re-implements reference behaviour: every call
// forwards to the reference symbol named in the comment.
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "convkit/activation.hpp"
#include "convkit/bilinear.hpp"
#include "convkit/blob.hpp"
#include "convkit/conv.hpp"
#include "convkit/graph.hpp"
#include "convkit/loss.hpp"
#include "convkit/normalize.hpp"
#include "convkit/pool.hpp"
#include "convkit/rng.hpp"

using namespace convkit;

namespace {
thread_local std::string g_err;

int guard(const std::function<void()>& fn) {
  try {
    fn();
    return 0;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

Shape shp(const int64_t* s) { return Shape(s[0], s[1], s[2], s[3]); }

TensorF tin(const float* p, const int64_t* s) {
  Shape sh = shp(s);
  return TensorF(sh, std::vector<float>(p, p + sh.elems()));
}

void tout(const TensorF& t, float* p) { std::memcpy(p, t.data(), sizeof(float) * t.size()); }

ConvGeom cgeom(const int64_t* g) {
  ConvGeom c;
  c.stride_h = g[0]; c.stride_w = g[1]; c.pad_top = g[2]; c.pad_bottom = g[3];
  c.pad_left = g[4]; c.pad_right = g[5]; c.groups = g[6];
  return c;
}

PoolGeom pgeom(const int64_t* g) {
  PoolGeom p;
  p.window_h = g[0]; p.window_w = g[1]; p.stride_h = g[2]; p.stride_w = g[3];
  p.pad_top = g[4]; p.pad_bottom = g[5]; p.pad_left = g[6]; p.pad_right = g[7];
  p.mode = g[8] == 0 ? PoolMode::max : PoolMode::avg;
  return p;
}

std::vector<std::string> split_csv(const char* s) {
  std::vector<std::string> out;
  std::stringstream ss(s ? s : "");
  std::string item;
  while (std::getline(ss, item, ',')) if (!item.empty()) out.push_back(item);
  return out;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// conv.cpp:193 conv_forward
int ref_conv_forward(const float* x, const int64_t* xs, const float* f, const int64_t* fs,
                     const float* b, const int64_t* geom, float* y) {
  return guard([&] {
    TensorF X = tin(x, xs), F = tin(f, fs);
    TensorF B;
    if (b) B = TensorF(Shape(1, 1, fs[3], 1), std::vector<float>(b, b + fs[3]));
    tout(conv_forward(X, F, b ? &B : nullptr, cgeom(geom)), y);
  });
}

// conv.cpp:229 conv_backward
int ref_conv_backward(const float* x, const int64_t* xs, const float* f, const int64_t* fs,
                      const int64_t* geom, const float* dy, const int64_t* ys, float* dx,
                      float* df, float* db) {
  return guard([&] {
    TensorF X = tin(x, xs), F = tin(f, fs), DY = tin(dy, ys), DX, DF, DB;
    conv_backward(X, F, cgeom(geom), DY, dx ? &DX : nullptr, df ? &DF : nullptr,
                  db ? &DB : nullptr);
    if (dx) tout(DX, dx);
    if (df) tout(DF, df);
    if (db) tout(DB, db);
  });
}

// conv.cpp:283 / :311 convt_forward / convt_backward (cg = up_h, up_w, crops)
int ref_convt_forward(const float* x, const int64_t* xs, const float* f, const int64_t* fs,
                      const int64_t* cg, float* y) {
  return guard([&] {
    ConvTransposeGeom g;
    g.up_h = cg[0]; g.up_w = cg[1]; g.crop_top = cg[2]; g.crop_bottom = cg[3];
    g.crop_left = cg[4]; g.crop_right = cg[5];
    tout(convt_forward(tin(x, xs), tin(f, fs), g), y);
  });
}

int ref_convt_backward(const float* x, const int64_t* xs, const float* f, const int64_t* fs,
                       const int64_t* cg, const float* dy, const int64_t* ys, float* dx,
                       float* df) {
  return guard([&] {
    ConvTransposeGeom g;
    g.up_h = cg[0]; g.up_w = cg[1]; g.crop_top = cg[2]; g.crop_bottom = cg[3];
    g.crop_left = cg[4]; g.crop_right = cg[5];
    TensorF DX, DF;
    convt_backward(tin(x, xs), tin(f, fs), g, tin(dy, ys), dx ? &DX : nullptr,
                   df ? &DF : nullptr);
    if (dx) tout(DX, dx);
    if (df) tout(DF, df);
  });
}

// pool.cpp:49 / :83
int ref_pool_forward(const float* x, const int64_t* xs, const int64_t* pg, float* y) {
  return guard([&] { tout(pool_forward(tin(x, xs), pgeom(pg)), y); });
}
int ref_pool_backward(const float* x, const int64_t* xs, const int64_t* pg, const float* dy,
                      const int64_t* ys, float* dx) {
  return guard([&] { tout(pool_backward(tin(x, xs), pgeom(pg), tin(dy, ys)), dx); });
}

// activation.cpp:8 / :15
int ref_relu_forward(const float* x, const int64_t* xs, float* y) {
  return guard([&] { tout(relu_forward(tin(x, xs)), y); });
}
int ref_relu_backward(const float* x, const int64_t* xs, const float* dy, float* dx) {
  return guard([&] { tout(relu_backward(tin(x, xs), tin(dy, xs)), dx); });
}

// normalize.cpp:47 / :74
int ref_lrn_forward(const float* x, const int64_t* xs, int64_t n, double kappa, double alpha,
                    double beta, float* y) {
  return guard([&] {
    LrnParams p{n, kappa, alpha, beta};
    tout(lrn_forward(tin(x, xs), p), y);
  });
}
int ref_lrn_backward(const float* x, const int64_t* xs, int64_t n, double kappa, double alpha,
                     double beta, const float* dy, float* dx) {
  return guard([&] {
    LrnParams p{n, kappa, alpha, beta};
    tout(lrn_backward(tin(x, xs), p, tin(dy, xs)), dx);
  });
}

// normalize.cpp:189 / :212
int ref_bnorm_forward(const float* x, const int64_t* xs, const float* w, const float* b,
                      double eps, float* y, float* moments) {
  return guard([&] {
    int64_t cs[4] = {1, 1, xs[2], 1};
    BnormMoments<float> m;
    tout(bnorm_forward(tin(x, xs), tin(w, cs), tin(b, cs), eps, &m), y);
    if (moments) {
      std::memcpy(moments, m.mean.data(), sizeof(float) * xs[2]);
      std::memcpy(moments + xs[2], m.var.data(), sizeof(float) * xs[2]);
    }
  });
}
int ref_bnorm_backward(const float* x, const int64_t* xs, const float* w, const float* b,
                       double eps, const float* dy, float* dx, float* dw, float* db) {
  return guard([&] {
    int64_t cs[4] = {1, 1, xs[2], 1};
    TensorF DX, DW, DB;
    bnorm_backward(tin(x, xs), tin(w, cs), tin(b, cs), eps, tin(dy, xs), dx ? &DX : nullptr,
                   dw ? &DW : nullptr, db ? &DB : nullptr);
    if (dx) tout(DX, dx);
    if (dw) tout(DW, dw);
    if (db) tout(DB, db);
  });
}

// loss.cpp:86 / :231 (kind by name: softmaxlog, classerror, topk, ...)
int ref_loss_forward(const float* x, const int64_t* xs, const float* c, const int64_t* cs,
                     const float* w, const char* kind, int64_t top_k, float* out) {
  return guard([&] {
    LossOptions o;
    o.top_k = top_k;
    TensorF W;
    if (w) W = tin(w, cs);
    *out = loss_forward(tin(x, xs), tin(c, cs), loss_kind_from_name(kind), w ? &W : nullptr, o);
  });
}
int ref_loss_backward(const float* x, const int64_t* xs, const float* c, const int64_t* cs,
                      const float* w, const char* kind, float p, float* dx) {
  return guard([&] {
    TensorF W;
    if (w) W = tin(w, cs);
    tout(loss_backward(tin(x, xs), tin(c, cs), loss_kind_from_name(kind), w ? &W : nullptr, p),
         dx);
  });
}

// loss.cpp:86 / :231 with the full LossOptions; kind as LossKind index.
int ref_loss_forward2(const float* x, const int64_t* xs, const float* c, const int64_t* cs,
                      const float* w, int kind, int64_t top_k, double threshold, int random_ties,
                      uint64_t tie_seed, float* out) {
  return guard([&] {
    LossOptions o;
    o.top_k = top_k;
    o.threshold = threshold;
    o.random_ties = random_ties != 0;
    o.tie_seed = tie_seed;
    TensorF W;
    if (w) W = tin(w, cs);
    *out = loss_forward(tin(x, xs), tin(c, cs), static_cast<LossKind>(kind), w ? &W : nullptr, o);
  });
}
int ref_loss_backward2(const float* x, const int64_t* xs, const float* c, const int64_t* cs,
                       const float* w, int kind, float p, float* dx) {
  return guard([&] {
    TensorF W;
    if (w) W = tin(w, cs);
    tout(loss_backward(tin(x, xs), tin(c, cs), static_cast<LossKind>(kind), w ? &W : nullptr, p),
         dx);
  });
}

// activation.cpp:25 / :41
int ref_sigmoid_forward(const float* x, const int64_t* xs, float* y) {
  return guard([&] { tout(sigmoid_forward(tin(x, xs)), y); });
}
int ref_sigmoid_backward(const float* y, const int64_t* ys, const float* dy, float* dx) {
  return guard([&] { tout(sigmoid_backward(tin(y, ys), tin(dy, ys)), dx); });
}

// normalize.cpp:309 / :330
int ref_softmax_forward(const float* x, const int64_t* xs, float* y) {
  return guard([&] { tout(softmax_forward(tin(x, xs)), y); });
}
int ref_softmax_backward(const float* y, const int64_t* ys, const float* dy, float* dx) {
  return guard([&] { tout(softmax_backward(tin(y, ys), tin(dy, ys)), dx); });
}

// normalize.cpp:268 / :284
int ref_spnorm_forward(const float* x, const int64_t* xs, int64_t wh, int64_t ww, double alpha,
                       double beta, float* y) {
  return guard([&] {
    SpnormParams p{wh, ww, alpha, beta};
    tout(spnorm_forward(tin(x, xs), p), y);
  });
}
int ref_spnorm_backward(const float* x, const int64_t* xs, int64_t wh, int64_t ww, double alpha,
                        double beta, const float* dy, float* dx) {
  return guard([&] {
    SpnormParams p{wh, ww, alpha, beta};
    tout(spnorm_backward(tin(x, xs), p, tin(dy, xs)), dx);
  });
}

// bilinear.cpp:58 / :92
int ref_bilinear_forward(const float* x, const int64_t* xs, const float* g, const int64_t* gs,
                         float* y) {
  return guard([&] { tout(bilinear_forward(tin(x, xs), tin(g, gs)), y); });
}
int ref_bilinear_backward(const float* x, const int64_t* xs, const float* g, const int64_t* gs,
                          const float* dy, const int64_t* ys, float* dx, float* dg) {
  return guard([&] {
    TensorF DX, DG;
    bilinear_backward(tin(x, xs), tin(g, gs), tin(dy, ys), dx ? &DX : nullptr, dg ? &DG : nullptr);
    if (dx) tout(DX, dx);
    if (dg) tout(DG, dg);
  });
}

// loss.cpp:346 / :374
int ref_pdist_forward(const float* x, const float* t, const int64_t* xs, double p, int no_root,
                      float* y) {
  return guard([&] { tout(pdist_forward(tin(x, xs), tin(t, xs), p, no_root != 0), y); });
}
int ref_pdist_backward(const float* x, const float* t, const int64_t* xs, double p, int no_root,
                       const float* dy, const int64_t* ys, float* dx, float* dt) {
  return guard([&] {
    TensorF DX, DT;
    pdist_backward(tin(x, xs), tin(t, xs), p, no_root != 0, tin(dy, ys), dx ? &DX : nullptr,
                   dt ? &DT : nullptr);
    if (dx) tout(DX, dx);
    if (dt) tout(DT, dt);
  });
}

// blob.cpp:29-79 write_blob / read_blob (read: out NULL -> shape only)
int ref_write_blob(const char* path, const float* data, const int64_t* s) {
  return guard([&] { write_blob(tin(data, s), std::string(path)); });
}
int ref_read_blob(const char* path, float* out, int64_t* s) {
  return guard([&] {
    TensorF t = read_blob(std::string(path));
    s[0] = t.shape().h; s[1] = t.shape().w; s[2] = t.shape().c; s[3] = t.shape().n;
    if (out) tout(t, out);
  });
}

// rng.cpp:51-59 Xoshiro256::permutation, and the state after it (rng.hpp:31-32)
int ref_rng_permutation(uint64_t seed, int64_t n, int64_t* out, uint64_t* state) {
  return guard([&] {
    Xoshiro256 r(seed);
    std::vector<int64_t> p = r.permutation(n);
    std::memcpy(out, p.data(), sizeof(int64_t) * (size_t)n);
    auto st = r.state();
    for (int k = 0; k < 4; ++k) state[k] = st[k];
  });
}

// ---- the reference DAG engine (graph.hpp) ---------------------------------

struct RefNet {
  Graph g;
  NamedTensors<float> bind;
  Tape<float> tape;
};

void* ref_graph_new() { return new RefNet(); }
void ref_graph_free(void* h) { delete static_cast<RefNet*>(h); }

int ref_graph_add_input(void* h, const char* name) {
  return guard([&] { static_cast<RefNet*>(h)->g.add_input(name); });
}
int ref_graph_add_param(void* h, const char* name) {
  return guard([&] { static_cast<RefNet*>(h)->g.add_param(name); });
}

// kind: layer_kind_name (graph.cpp:13-31); p: kind-specific parameters.
//   conv: geom[7]; pool: pg[9]; lrn: n,kappa,alpha,beta; bnorm: eps; loss: (softmaxlog)
int ref_graph_add_layer(void* h, const char* kind, const char* name, const char* inputs,
                        const char* outputs, const double* p, int np) {
  return guard([&] {
    LayerDef d;
    d.name = name;
    d.kind = layer_kind_from_name(kind);
    d.inputs = split_csv(inputs);
    d.outputs = split_csv(outputs);
    switch (d.kind) {
      case LayerKind::conv: {
        int64_t g[7];
        for (int k = 0; k < 7; ++k) g[k] = static_cast<int64_t>(p[k]);
        d.hyper = ConvHyper{cgeom(g)};
        break;
      }
      case LayerKind::pool: {
        int64_t g[9];
        for (int k = 0; k < 9; ++k) g[k] = static_cast<int64_t>(p[k]);
        d.hyper = PoolHyper{pgeom(g)};
        break;
      }
      case LayerKind::lrn:
        d.hyper = LrnParams{static_cast<int64_t>(p[0]), p[1], p[2], p[3]};
        break;
      case LayerKind::bnorm:
        d.hyper = BnormHyper{p[0]};
        break;
      case LayerKind::loss: {
        // p: [kind top_k threshold random_ties tie_seed] or NaN-terminated empty
        LossHyper lh;
        if (np > 0) {
          lh.kind = static_cast<LossKind>(static_cast<int>(p[0]));
          if (np > 1) lh.opts.top_k = static_cast<int64_t>(p[1]);
          if (np > 2) lh.opts.threshold = p[2];
          if (np > 3) lh.opts.random_ties = p[3] != 0;
          if (np > 4) lh.opts.tie_seed = static_cast<uint64_t>(p[4]);
        }
        d.hyper = lh;
        break;
      }
      case LayerKind::spnorm:
        d.hyper = SpnormParams{static_cast<int64_t>(p[0]), static_cast<int64_t>(p[1]), p[2], p[3]};
        break;
      case LayerKind::pdist: {
        PdistHyper ph;
        if (np > 0) ph.p = p[0];
        if (np > 1) ph.no_root = p[1] != 0;
        d.hyper = ph;
        break;
      }
      case LayerKind::split:
        d.hyper = SplitHyper{static_cast<int64_t>(d.outputs.size())};
        break;
      default:
        break;
    }
    static_cast<RefNet*>(h)->g.add_layer(std::move(d));
  });
}

int ref_graph_finalize(void* h) { return guard([&] { static_cast<RefNet*>(h)->g.finalize(); }); }

int ref_graph_bind(void* h, const char* name, const float* data, const int64_t* s) {
  return guard([&] {
    auto* n = static_cast<RefNet*>(h);
    n->bind.insert_or_assign(name, tin(data, s));
  });
}

// graph.cpp:494 forward then :548 backward seeded with d(objective) = 1.
int ref_graph_forward_backward(void* h, const char* objective, int do_backward) {
  return guard([&] {
    auto* n = static_cast<RefNet*>(h);
    n->tape = forward(n->g, n->bind, EvalMode::train);
    if (do_backward) {
      NamedTensors<float> seeds;
      seeds[objective] = TensorF::filled(Shape(1, 1, 1, 1), 1.f);
      backward(n->g, n->tape, seeds);
    }
  });
}

// Copies a forward value (which=0) or derivative (which=1) into out; returns
// its shape in s.
int ref_graph_get(void* h, const char* name, int which, float* out, int64_t* s) {
  return guard([&] {
    auto* n = static_cast<RefNet*>(h);
    const TensorF& t = which ? n->tape.derivs.at(name) : n->tape.values.at(name);
    s[0] = t.shape().h; s[1] = t.shape().w; s[2] = t.shape().c; s[3] = t.shape().n;
    if (out) tout(t, out);
  });
}

}  // extern "C"
