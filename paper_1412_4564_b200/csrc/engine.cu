// engine.cu -- the device-resident DAG engine (graph.hpp / graph.cpp) and
// the cnn_train data-parallel training step.
//
// Semantics follow graph.cpp:
//   * layers fire in a stable topological order, ties by declaration order
//     (Graph::finalize);
//   * forward keeps every value resident on the device ("tape");
//   * backward seeds d(objective) = 1, walks layers in reverse and
//     accumulates derivs[in] += d (graph.cpp:548-598).  The zero-init +
//     accumulate of the reference is fused: the first contribution to a
//     derivative is written, later ones are added by the producing kernel
//     (its `acc` epilogue), and derivatives that receive nothing are zeroed
//     at the end -- bit-identical to 0 + a (+ b ...).
// The trainer adds SGD with momentum and NCCL allreduce of the parameter
// derivatives, launched per layer on a communication stream as soon as the
// layer's backward has produced them, overlapping the rest of backward.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <sys/stat.h>

#include <cinttypes>
#include <cmath>
#include <fstream>

#include "ck/ck.h"
#include "ck_handle.hpp"
#include "ck_internal.hpp"
#include "ck_io.hpp"

using ck::Err;

namespace ck {

enum class Kind { conv, convt, pool, relu, lrn, bnorm, loss, sum, sigmoid, softmax, spnorm, bilinear, pdist, split };

static Kind kind_from_name(const std::string& s) {
  if (s == "conv") return Kind::conv;
  if (s == "convt") return Kind::convt;
  if (s == "pool") return Kind::pool;
  if (s == "relu") return Kind::relu;
  if (s == "lrn") return Kind::lrn;
  if (s == "bnorm") return Kind::bnorm;
  if (s == "loss") return Kind::loss;
  if (s == "sum") return Kind::sum;
  if (s == "sigmoid") return Kind::sigmoid;
  if (s == "softmax") return Kind::softmax;
  if (s == "spnorm") return Kind::spnorm;
  if (s == "bilinear") return Kind::bilinear;
  if (s == "pdist") return Kind::pdist;
  if (s == "split") return Kind::split;
  // graph.cpp:33-40 layer_kind_from_name
  throw Err(CK_ERR_ARG, "unknown layer kind '" + s + "'");
}

static const char* kind_name(Kind k) {
  switch (k) {
    case Kind::conv: return "conv";
    case Kind::convt: return "convt";
    case Kind::pool: return "pool";
    case Kind::relu: return "relu";
    case Kind::lrn: return "lrn";
    case Kind::bnorm: return "bnorm";
    case Kind::loss: return "loss";
    case Kind::sum: return "sum";
    case Kind::sigmoid: return "sigmoid";
    case Kind::softmax: return "softmax";
    case Kind::spnorm: return "spnorm";
    case Kind::bilinear: return "bilinear";
    case Kind::pdist: return "pdist";
    case Kind::split: return "split";
  }
  return "?";
}

struct Var {
  std::string name;
  int role = 2;  // 0 input, 1 param, 2 derived
  ck_shape shape{0, 0, 0, 0};
  bool has_shape = false;
  int producer = -1;
  std::vector<std::pair<int, int>> consumers;
  float* value = nullptr;
  float* own_value = nullptr;  // the engine's buffer while an input is bound elsewhere
  float* deriv = nullptr;
  bool deriv_live = false;  // received a contribution in this backward
  // derivative left unmaterialized by a fused conv -> relu backward (only its
  // grid form was consumed): deriv = value(lazy_gate) > 0 ? deriv(lazy_src) : 0,
  // computed when the derivative is requested (ck_graph_var)
  int lazy_gate = -1, lazy_src = -1;
  // derivative left unmaterialized because the LRN layer lazy_lrn wrote its
  // consumer conv's dy grid directly: that LRN backward, computed on request
  int lazy_lrn = -1;
  // derivative left unmaterialized because the bnorm layer lazy_bn wrote its
  // producer conv's dy grid directly: that bnorm backward's dx, on request
  int lazy_bn = -1;
  // value left unstored by the fused bnorm -> relu forward of layer
  // lazy_value (engine option bn_lazy_y): recomputed from x on request
  int lazy_value = -1;
  bool lazy_value_relu = false;  // ... and this var is relu of that bnorm output
};

struct Layer {
  std::string name;
  Kind kind;
  std::vector<int> in, out;
  std::vector<double> p;
  float* aux = nullptr;  // bnorm moments (K x 2), graph.cpp:306
  // bnorm -> relu: the forward's (mu, inv) per channel, then its (w, b)
  // snapshot -- [2C] interleaved (mu, inv), [C] w, [C] b -- so values and
  // derivatives left unstored are recomputed with the parameters of that
  // forward even after the trainer's SGD moved them
  float* muinv = nullptr;
  ConvCache cache;       // conv input transform shared by forward and wgrad
  // conv -> relu fusion: the conv's epilogue also writes relu(y) (the relu
  // layer's output) when its output feeds only that relu; the relu forward
  // then has nothing to do.  fused_by = producing conv layer, or -1.
  int relu_out = -1;     // conv: var index of the fused relu output
  int fused_by = -1;     // relu: index of the conv layer that writes its output
  bool fused_done = false;
  bool fused_bwd = false;  // relu backward may be left to the producing conv's backward
  // conv: its dy grid + bias partials prebuilt by the LRN above (lrn -> relu
  // -> conv chain, see layer_backward), valid for the current backward
  bool pre_grid = false;
  GridPlan plan{};
  Workspace dyg, bpart;
  int pre_rows = 0;
  bool bwd_deferred = false;  // ... and was, in the current backward pass
  // lrn -> max pool (3x3 / 2): the LRN forward also produces the pool's
  // output and argmax (lrn_maxpool_forward); lrn_pool = that pool layer
  int lrn_pool = -1;
};

static std::vector<std::string> split_csv(const char* s) {
  std::vector<std::string> out;
  std::stringstream ss(s ? s : "");
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

}  // namespace ck

struct ck_graph {
  ck_handle* h = nullptr;
  ck_math math = CK_MATH_TF32;
  std::vector<ck::Var> vars;
  std::map<std::string, int> by_name;
  std::vector<ck::Layer> layers;
  std::vector<int> order;
  bool finalized = false;
  std::vector<void*> allocs;
  float* param_deriv_arena = nullptr;
  size_t param_deriv_elems = 0;
  float* one_dev = nullptr;  // the objective seed 1.0f, device-resident (graph-capturable)
  bool has_loss = false;
  bool lrn_grid = true;  // option "lrn_grid": LRN backward writes the conv's dy grid
  // option "lrn_pool": LRN forward also computes the max pool after it.  Off
  // by default: bit-identical but measured slower on AlexNet (norm1+pool1
  // 0.247 vs 0.213 ms, norm2+pool2 0.168 vs 0.149: the per-chunk barrier and
  // the 16% halo recompute cost more than the 297 MB re-read saves)
  bool lrn_pool = false;
  // option "producer_grid": a conv -> relu -> conv forward writes the next
  // conv's x grid from its epilogue (default on)
  bool producer_grid = true;
  // option "dgrad_grid": a conv -> relu -> conv backward writes the first
  // conv's relu-gated dy grid from the second conv's data-gradient epilogue
  // (default on)
  bool dgrad_grid = true;
  // option "bn_grid": a TF32 conv -> bnorm backward writes the conv's dy grid
  // (and bias partials) from the bnorm backward (default on)
  bool bn_grid = true;
  // option "bn_lazy_y": a fused bnorm -> relu forward whose bnorm output has
  // no other reader stores only relu(y) (default on)
  bool bn_lazy_y = true;
  std::vector<std::pair<std::string, std::string>> meta;  // manifest metadata
  std::vector<int> decl;  // input / param vars in declaration order (manifest order)
  int64_t last_launches = 0;
  bool profiling = false;
  // per layer: fwd begin/end, bwd begin/end
  std::vector<cudaEvent_t> prof_ev;
  std::vector<char> prof_fwd_done, prof_bwd_done;

  int var(const std::string& n) const {
    auto it = by_name.find(n);
    if (it == by_name.end()) throw Err(CK_ERR_ARG, "unknown variable '" + n + "'");
    return it->second;
  }
  int intern(const std::string& n, int role) {
    auto it = by_name.find(n);
    if (it != by_name.end()) return it->second;
    ck::Var v;
    v.name = n;
    v.role = role;
    vars.push_back(v);
    by_name[n] = (int)vars.size() - 1;
    return (int)vars.size() - 1;
  }
  ~ck_graph() {
    for (auto& l : layers) {
      l.cache.buf.release();
      l.dyg.release();
      l.bpart.release();
    }
    for (void* p : allocs) cudaFree(p);
    for (auto e : prof_ev) cudaEventDestroy(e);
  }
  void prof(int li, int which, cudaStream_t s) {  // which: 0..3
    if (profiling) cudaEventRecord(prof_ev[4 * li + which], s);
  }
};

namespace ck {

static void need(const Layer& l, size_t nin_lo, size_t nin_hi, size_t nout) {
  if (l.in.size() < nin_lo || l.in.size() > nin_hi || l.out.size() != nout)
    throw Err(CK_ERR_ARG, "layer '" + l.name + "' has wrong arity");
}

static void need_params(const Layer& l, size_t n) {
  if (l.p.size() < n) throw Err(CK_ERR_ARG, "layer '" + l.name + "' needs " + std::to_string(n) + " parameters");
}

static ck_conv_geom conv_geom_of(const Layer& l) {
  need_params(l, 7);
  return ck_conv_geom{(int64_t)l.p[0], (int64_t)l.p[1], (int64_t)l.p[2], (int64_t)l.p[3],
                      (int64_t)l.p[4], (int64_t)l.p[5], (int64_t)l.p[6]};
}
static ck_convt_geom convt_geom_of(const Layer& l) {
  need_params(l, 6);
  return ck_convt_geom{(int64_t)l.p[0], (int64_t)l.p[1], (int64_t)l.p[2],
                       (int64_t)l.p[3], (int64_t)l.p[4], (int64_t)l.p[5]};
}
static ck_pool_geom pool_geom_of(const Layer& l) {
  need_params(l, 9);
  return ck_pool_geom{(int64_t)l.p[0], (int64_t)l.p[1], (int64_t)l.p[2], (int64_t)l.p[3],
                      (int64_t)l.p[4], (int64_t)l.p[5], (int64_t)l.p[6], (int64_t)l.p[7],
                      (int64_t)l.p[8]};
}
static ck_lrn_params lrn_of(const Layer& l) {
  need_params(l, 4);
  return ck_lrn_params{(int64_t)l.p[0], l.p[1], l.p[2], l.p[3]};
}

// graph.hpp:53-62 LossHyper: [kind top_k threshold random_ties tie_seed],
// empty = softmaxlog with the default options
static int loss_kind_of(const Layer& l) {
  const int k = l.p.empty() ? (int)CK_LOSS_SOFTMAXLOG : (int)l.p[0];
  if (k < CK_LOSS_CLASSERROR || k > CK_LOSS_HINGE)
    throw Err(CK_ERR_DATA, "layer '" + l.name + "': unknown loss kind");
  return k;
}
static ck_loss_options loss_opts_of(const Layer& l) {
  ck_loss_options o = default_loss_options();
  if (l.p.size() > 1) o.top_k = (int64_t)l.p[1];
  if (l.p.size() > 2) o.threshold = l.p[2];
  if (l.p.size() > 3) o.random_ties = (int64_t)l.p[3];
  if (l.p.size() > 4) o.tie_seed = (uint64_t)l.p[4];
  return o;
}
static ck_spnorm_params spnorm_of(const Layer& l) {
  need_params(l, 4);
  return ck_spnorm_params{(int64_t)l.p[0], (int64_t)l.p[1], l.p[2], l.p[3]};
}
// graph.hpp:63-66 PdistHyper {p = 2, no_root = false}
static double pdist_p(const Layer& l) { return l.p.empty() ? 2.0 : l.p[0]; }
static int pdist_no_root(const Layer& l) { return l.p.size() > 1 && l.p[1] != 0; }

static ck_tensor tv(Var& v, bool deriv) { return ck_tensor{deriv ? v.deriv : v.value, v.shape}; }

// Graph::finalize: arity, single producer, stable topological order, shapes.
static void finalize(ck_graph* g) {
  std::vector<int> indeg(g->layers.size(), 0);
  for (auto& v : g->vars) {
    v.producer = -1;
    v.consumers.clear();
  }
  for (size_t li = 0; li < g->layers.size(); ++li) {
    Layer& l = g->layers[li];
    for (int o : l.out) {
      if (g->vars[o].producer >= 0)
        throw Err(CK_ERR_ARG, "variable '" + g->vars[o].name + "' has two producers");
      if (g->vars[o].role != 2)
        throw Err(CK_ERR_ARG, "layer '" + l.name + "' writes input/param '" + g->vars[o].name + "'");
      g->vars[o].producer = (int)li;
    }
    for (size_t s = 0; s < l.in.size(); ++s) g->vars[l.in[s]].consumers.push_back({(int)li, (int)s});
  }
  for (size_t li = 0; li < g->layers.size(); ++li)
    for (int i : g->layers[li].in) {
      if (g->vars[i].role == 2 && g->vars[i].producer < 0)
        throw Err(CK_ERR_ARG, "variable '" + g->vars[i].name + "' has no producer");
      if (g->vars[i].producer >= 0) indeg[li]++;
    }
  // Kahn's algorithm, always taking the lowest declared index (stable).
  std::set<int> ready;
  for (size_t li = 0; li < g->layers.size(); ++li)
    if (!indeg[li]) ready.insert((int)li);
  g->order.clear();
  while (!ready.empty()) {
    int li = *ready.begin();
    ready.erase(ready.begin());
    g->order.push_back(li);
    for (int o : g->layers[li].out)
      for (auto [c, s] : g->vars[o].consumers) {
        (void)s;
        if (--indeg[c] == 0) ready.insert(c);
      }
  }
  if (g->order.size() != g->layers.size()) throw Err(CK_ERR_ARG, "graph has a cycle");

  for (auto& v : g->vars)
    if (v.role != 2 && !v.has_shape)
      throw Err(CK_ERR_ARG, "input/param '" + v.name + "' needs a shape on the device path");

  // Shape inference in firing order (the reference's shape laws).
  for (int li : g->order) {
    Layer& l = g->layers[li];
    auto S = [&](int k) -> ck_shape& { return g->vars[l.in[k]].shape; };
    ck_shape out{1, 1, 1, 1};
    switch (l.kind) {
      case Kind::conv: {
        need(l, 2, 3, 1);
        out = conv_output_shape(S(0), S(1), conv_geom_of(l));
        if (l.in.size() > 2 && elems(S(2)) != S(1).n)
          throw Err(CK_ERR_SHAPE, "layer '" + l.name + "': bias has " + std::to_string(elems(S(2))) +
                                      " elements for " + std::to_string(S(1).n) + " filters");
        break;
      }
      case Kind::convt:
        need(l, 2, 2, 1);
        out = convt_output_shape(S(0), S(1), convt_geom_of(l));
        break;
      case Kind::pool:
        need(l, 1, 1, 1);
        out = pool_output_shape(S(0), pool_geom_of(l));
        break;
      case Kind::relu:
        need(l, 1, 1, 1);
        out = S(0);
        break;
      case Kind::lrn: {
        need(l, 1, 1, 1);
        ck_lrn_params p = lrn_of(l);
        if (p.group_size < 1) throw Err(CK_ERR_SHAPE, "lrn group size must be positive");
        if (p.kappa <= 0) throw Err(CK_ERR_SHAPE, "lrn kappa must be positive");
        out = S(0);
        break;
      }
      case Kind::bnorm:
        need(l, 3, 3, 1);
        need_params(l, 1);
        if (elems(S(1)) != S(0).c || elems(S(2)) != S(0).c)
          throw Err(CK_ERR_SHAPE, "layer '" + l.name + "': bnorm expects one multiplier and bias per channel");
        out = S(0);
        break;
      case Kind::loss: {
        need(l, 2, 3, 1);
        const int kind = loss_kind_of(l);
        ck_tensor xt{(float*)1, S(0)}, ct{(float*)1, S(1)}, wt{(float*)1, ck_shape{1, 1, 1, 1}};
        if (l.in.size() > 2) wt.shape = S(2);
        try {
          check_loss_kind(&xt, &ct, l.in.size() > 2 ? &wt : nullptr, kind);
        } catch (const Err& e) {
          throw Err(e.code, "layer '" + l.name + "': " + e.what());
        }
        out = ck_shape{1, 1, 1, 1};
        break;
      }
      case Kind::sigmoid:
      case Kind::softmax:
        need(l, 1, 1, 1);
        out = S(0);
        break;
      case Kind::spnorm: {
        need(l, 1, 1, 1);
        const ck_spnorm_params sp = spnorm_of(l);
        if (sp.window_h < 1 || sp.window_w < 1) throw Err(CK_ERR_SHAPE, "spnorm window must be positive");
        out = S(0);
        break;
      }
      case Kind::bilinear:
        need(l, 2, 2, 1);
        out = bilinear_output_shape(S(0), S(1));
        break;
      case Kind::pdist:
        need(l, 2, 2, 1);
        out = pdist_output_shape(S(0), S(1), pdist_p(l));
        break;
      case Kind::split:
        if (l.in.size() != 1 || l.out.empty() || l.out.size() > 8)
          throw Err(CK_ERR_ARG, "layer '" + l.name + "' has wrong arity");
        out = S(0);
        for (int o : l.out) {
          g->vars[o].shape = out;
          g->vars[o].has_shape = true;
        }
        break;
      case Kind::sum:
        need(l, 1, 64, 1);
        for (size_t k = 1; k < l.in.size(); ++k)
          if (!same(S(k), S(0))) throw Err(CK_ERR_SHAPE, "sum inputs must share one shape");
        out = S(0);
        break;
    }
    g->vars[l.out[0]].shape = out;
    g->vars[l.out[0]].has_shape = true;
  }

  // Allocation: values and derivatives for every variable; parameter
  // derivatives live in one arena ordered by when backward finishes them,
  // so each layer's gradient bucket is contiguous for the allreduce.
  auto alloc = [&](size_t n) -> float* {
    void* p = nullptr;
    check_cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(float)), "cudaMalloc");
    g->allocs.push_back(p);
    return (float*)p;
  };
  // A parameter's derivative is final once the backward of its FIRST
  // consumer in firing order has run (every other consumer comes before it
  // in backward order); the arena follows that completion order, so the
  // parameters one layer finishes (ck_trainer::done) are adjacent.
  std::vector<int> pos(g->layers.size());
  for (size_t k = 0; k < g->order.size(); ++k) pos[g->order[k]] = (int)k;
  std::vector<std::pair<int, int>> fin;  // (-firing position of first consumer, var)
  for (size_t i = 0; i < g->vars.size(); ++i) {
    const Var& v = g->vars[i];
    if (v.role != 1 || v.consumers.empty()) continue;
    int first = (int)g->order.size();
    for (auto [c, sl] : v.consumers) {
      (void)sl;
      first = std::min(first, pos[c]);
    }
    fin.push_back({-first, (int)i});
  }
  std::stable_sort(fin.begin(), fin.end(),
                   [](const std::pair<int, int>& a, const std::pair<int, int>& b) {
                     return a.first < b.first;
                   });
  std::vector<int> param_order;
  for (auto& f : fin) param_order.push_back(f.second);
  for (size_t i = 0; i < g->vars.size(); ++i)  // params nobody consumes
    if (g->vars[i].role == 1 && g->vars[i].consumers.empty()) param_order.push_back((int)i);
  size_t total = 0;
  for (int i : param_order) total += (size_t)((elems(g->vars[i].shape) + 31) / 32 * 32);
  g->param_deriv_arena = alloc(total);
  g->param_deriv_elems = total;
  // zero once: the 32-element pads between parameters are inside allreduce spans
  check_cuda(cudaMemset(g->param_deriv_arena, 0, sizeof(float) * std::max<size_t>(total, 1)),
             "memset");
  g->one_dev = alloc(1);
  {
    const float one = 1.0f;
    check_cuda(cudaMemcpy(g->one_dev, &one, sizeof(float), cudaMemcpyHostToDevice), "seed");
  }
  for (auto& l : g->layers) g->has_loss |= l.kind == Kind::loss;
  size_t off = 0;
  for (int i : param_order) {
    g->vars[i].deriv = g->param_deriv_arena + off;
    off += (size_t)((elems(g->vars[i].shape) + 31) / 32 * 32);
  }
  for (auto& v : g->vars) {
    v.value = alloc((size_t)elems(v.shape));
    if (!v.deriv) v.deriv = alloc((size_t)elems(v.shape));
  }
  for (auto& l : g->layers)
    if (l.kind == Kind::bnorm) {
      l.aux = alloc(2 * (size_t)g->vars[l.in[0]].shape.c);
      l.muinv = alloc(4 * (size_t)g->vars[l.in[0]].shape.c);
    }
  // conv -> relu pairs whose intermediate has no other reader
  for (size_t li = 0; li < g->layers.size(); ++li) {
    Layer& r = g->layers[li];
    if (r.kind != Kind::relu) continue;
    const Var& v = g->vars[r.in[0]];
    if (v.producer < 0 || v.consumers.size() != 1) continue;
    Layer& c = g->layers[v.producer];
    // conv -> relu (fused epilogue) and bnorm -> relu (fused apply / gated
    // backward): the producer writes relu(y) too; the relu layer idles
    if ((c.kind != Kind::conv && c.kind != Kind::bnorm) || c.relu_out >= 0) continue;
    c.relu_out = r.out[0];
    r.fused_by = v.producer;
    r.fused_bwd = true;
  }
  // lrn -> max pool pairs whose intermediate has no other reader
  for (size_t li = 0; li < g->layers.size(); ++li) {
    Layer& pl = g->layers[li];
    if (pl.kind != Kind::pool || pl.p.size() < 9 || pl.p[8] != 0) continue;
    const Var& v = g->vars[pl.in[0]];
    if (v.producer < 0 || v.consumers.size() != 1) continue;
    Layer& l = g->layers[v.producer];
    if (l.kind != Kind::lrn || l.lrn_pool >= 0) continue;
    l.lrn_pool = (int)li;
    pl.fused_by = v.producer;
  }
  g->finalized = true;
}

static void layer_forward(ck_graph* g, Layer& l, cudaStream_t s) {
  ck_handle* h = g->h;
  auto V = [&](int k) { return tv(g->vars[l.in[k]], false); };
  ck_tensor y = tv(g->vars[l.out[0]], false);
  ck_status st = CK_OK;
  switch (l.kind) {
    case Kind::conv: {
      ck_tensor x = V(0), f = V(1), b;
      if (l.in.size() > 2) b = V(2);
      ck_conv_geom cg = conv_geom_of(l);
      h->conv_cache = &l.cache;
      h->fuse_relu = l.relu_out >= 0 ? g->vars[l.relu_out].value : nullptr;
      h->fuse_relu_done = false;
      // conv -> relu -> conv (AlexNet conv3 -> conv4 -> conv5): this forward's
      // epilogue also writes relu(y) into the next conv's x grid, whose
      // forward and weight gradient then skip their input transform
      Layer* nxt = nullptr;
      XGridPlan xp{};
      if (g->producer_grid && g->math == CK_MATH_TF32 && l.relu_out >= 0) {
        const Var& rv = g->vars[l.relu_out];
        if (rv.consumers.size() == 1 && rv.consumers[0].second == 0) {
          Layer& c2 = g->layers[rv.consumers[0].first];
          if (c2.kind == Kind::conv) {
            const ConvDims d2 = conv_dims(rv.shape, g->vars[c2.in[1]].shape,
                                          g->vars[c2.out[0]].shape, conv_geom_of(c2));
            if (conv_tc_xgrid_plan(d2, &xp) && xp.Cg % 32 == 0) {
              float* buf = (float*)c2.cache.buf.get(xp.bytes, s);
              if (!buf) throw Err(CK_ERR_CUDA, "x grid allocation failed");
              if (c2.cache.zero_ptr != buf || c2.cache.zero_key != xp.key) {
                check_cuda(cudaMemsetAsync(buf, 0, c2.cache.buf.bytes, s), "zero");
                c2.cache.zero_ptr = buf;
                c2.cache.zero_key = xp.key;
              }
              h->next_xg = buf;
              h->next_xg_plan = xp;
              h->next_xg_done = false;
              nxt = &c2;
            }
          }
        }
      }
      st = ck_conv_forward(h, &x, &f, l.in.size() > 2 ? &b : nullptr, &cg, &y, g->math, s);
      if (nxt && st == CK_OK && h->next_xg_done) {
        nxt->cache.valid = true;
        nxt->cache.src = g->vars[l.relu_out].value;
        nxt->cache.key = xp.key;
      }
      h->next_xg = nullptr;
      h->next_xg_done = false;
      h->conv_cache = nullptr;
      h->fuse_relu = nullptr;
      if (l.relu_out >= 0) {
        Layer& r = g->layers[g->vars[l.relu_out].producer];
        r.fused_done = st == CK_OK && h->fuse_relu_done;
      }
      break;
    }
    case Kind::convt: {
      ck_tensor x = V(0), f = V(1);
      ck_convt_geom cg = convt_geom_of(l);
      st = ck_convt_forward(h, &x, &f, &cg, &y, g->math, s);
      break;
    }
    case Kind::pool: {
      if (l.fused_by >= 0 && l.fused_done) break;  // produced by the LRN before it
      ck_tensor x = V(0);
      ck_pool_geom pg = pool_geom_of(l);
      h->conv_cache = &l.cache;  // records the argmax for this step's backward
      st = ck_pool_forward(h, &x, &pg, &y, s);
      h->conv_cache = nullptr;
      break;
    }
    case Kind::relu: {
      if (l.fused_by >= 0 && l.fused_done) break;  // written by the conv epilogue
      ck_tensor x = V(0);
      st = ck_relu_forward(h, &x, &y, s);
      break;
    }
    case Kind::lrn: {
      ck_tensor x = V(0);
      ck_lrn_params p = lrn_of(l);
      if (l.lrn_pool >= 0) {
        // lrn -> max pool: one kernel writes y, the pool output and its argmax
        Layer& pl = g->layers[l.lrn_pool];
        pl.fused_done = false;
        const Var& pv = g->vars[pl.out[0]];
        if (g->lrn_pool && p.group_size >= 1 && p.kappa > 0) {
          const PoolDims pd = pool_dims(y.shape, pv.shape, pool_geom_of(pl));
          pl.fused_done = lrn_maxpool_forward(x.data, y.data, pv.value, pd, (int)p.group_size,
                                              (float)p.kappa, (float)p.alpha, (float)p.beta, s,
                                              &pl.cache);
          if (pl.fused_done) {
            after_launch();
            break;
          }
        }
      }
      st = ck_lrn_forward(h, &x, &p, &y, s);
      break;
    }
    case Kind::bnorm: {
      ck_tensor x = V(0), w = V(1), b = V(2);
      ck_tensor m{l.aux, ck_shape{x.shape.c, 2, 1, 1}};
      h->fuse_relu = l.relu_out >= 0 ? g->vars[l.relu_out].value : nullptr;
      h->fuse_relu_done = false;
      h->bn_muinv = l.muinv;
      h->bn_skip_y = g->bn_lazy_y && l.relu_out >= 0 && g->vars[l.out[0]].consumers.size() == 1;
      h->bn_y_skipped = false;
      // bnorm -> relu -> conv (VGG): relu(y) straight into the conv's x grid
      Layer* nxt = nullptr;
      XGridPlan xp{};
      if (h->bn_skip_y && g->producer_grid && g->math == CK_MATH_TF32) {
        const Var& rv = g->vars[l.relu_out];
        if (rv.consumers.size() == 1 && rv.consumers[0].second == 0) {
          Layer& c2 = g->layers[rv.consumers[0].first];
          if (c2.kind == Kind::conv) {
            const ConvDims d2 = conv_dims(rv.shape, g->vars[c2.in[1]].shape,
                                          g->vars[c2.out[0]].shape, conv_geom_of(c2));
            if (conv_tc_xgrid_plan(d2, &xp) && xp.Cg % 32 == 0) {
              float* buf = (float*)c2.cache.buf.get(xp.bytes, s);
              if (!buf) throw Err(CK_ERR_CUDA, "x grid allocation failed");
              if (c2.cache.zero_ptr != buf || c2.cache.zero_key != xp.key) {
                check_cuda(cudaMemsetAsync(buf, 0, c2.cache.buf.bytes, s), "zero");
                c2.cache.zero_ptr = buf;
                c2.cache.zero_key = xp.key;
              }
              h->next_xg = buf;
              h->next_xg_plan = xp;
              h->next_xg_done = false;
              nxt = &c2;
            }
          }
        }
      }
      st = ck_bnorm_forward(h, &x, &w, &b, l.p[0], &y, &m, s);
      const int self = (int)(&l - &g->layers[0]);
      g->vars[l.out[0]].lazy_value = st == CK_OK && h->bn_y_skipped ? self : -1;
      Var& ro = g->vars[l.relu_out >= 0 ? l.relu_out : l.out[0]];
      if (l.relu_out >= 0) ro.lazy_value = -1;
      if (nxt && st == CK_OK && h->next_xg_done) {
        nxt->cache.valid = true;
        nxt->cache.src = ro.value;
        nxt->cache.key = xp.key;
        ro.lazy_value = self;  // the HWCN relu output: relu(bn_y(x)) on request
        ro.lazy_value_relu = true;
      }
      h->next_xg = nullptr;
      h->next_xg_done = false;
      h->fuse_relu = nullptr;
      h->bn_muinv = nullptr;
      h->bn_skip_y = false;
      if (l.relu_out >= 0) {
        Layer& r = g->layers[g->vars[l.relu_out].producer];
        r.fused_done = st == CK_OK && h->fuse_relu_done;
      }
      break;
    }
    case Kind::loss: {
      ck_tensor x = V(0), c = V(1), w;
      if (l.in.size() > 2) w = V(2);
      loss_forward_any(h, &x, &c, l.in.size() > 2 ? &w : nullptr, loss_kind_of(l), loss_opts_of(l),
                       y.data, s);
      after_launch();
      break;
    }
    case Kind::sigmoid:
      sigmoid_forward(V(0).data, y.data, elems(y.shape), s);
      after_launch();
      break;
    case Kind::softmax: {
      const ck_shape& xs = V(0).shape;
      softmax_forward(V(0).data, y.data, (int)(xs.h * xs.w), (int)xs.c, (int)xs.n, s);
      after_launch();
      break;
    }
    case Kind::spnorm: {
      ck_tensor x = V(0);
      const ck_spnorm_params sp = spnorm_of(l);
      st = ck_spnorm_forward(h, &x, &sp, &y, s);
      break;
    }
    case Kind::bilinear: {
      ck_tensor x = V(0), gr = V(1);
      st = ck_bilinear_forward(h, &x, &gr, &y, s);
      break;
    }
    case Kind::pdist: {
      ck_tensor x = V(0), t = V(1);
      st = ck_pdist_forward(h, &x, &t, pdist_p(l), pdist_no_root(l), &y, s);
      break;
    }
    case Kind::split:
      // graph.cpp split: every output is a copy of the input
      for (int o : l.out)
        check_cuda(cudaMemcpyAsync(g->vars[o].value, V(0).data, sizeof(float) * elems(y.shape),
                                   cudaMemcpyDeviceToDevice, s), "copy");
      break;
    case Kind::sum: {
      ck_tensor x0 = V(0);
      check_cuda(cudaMemcpyAsync(y.data, x0.data, sizeof(float) * elems(y.shape),
                                 cudaMemcpyDeviceToDevice, s), "copy");
      for (size_t k = 1; k < l.in.size(); ++k) axpy_inplace(y.data, V((int)k).data, elems(y.shape), s);
      break;
    }
  }
  if (st != CK_OK) throw Err(st, "layer '" + l.name + "': " + h->err);
}

// One layer's backward; contributions for input slot k go to derivs with
// accumulate = deriv_live (graph.cpp:587-596 fused).
// The relu output's derivative an LRN backward skipped (it wrote the conv's
// dy grid instead): the ordinary LRN backward into it, now.
static void materialize_lrn(ck_graph* g, Var& v, cudaStream_t s) {
  if (v.lazy_lrn < 0) return;
  Layer& l = g->layers[v.lazy_lrn];
  ck_tensor x = tv(v, false), dx = tv(v, true), dy = tv(g->vars[l.out[0]], true);
  const ck_lrn_params p = lrn_of(l);
  const ck_status st = ck_lrn_backward(g->h, &x, &p, &dy, &dx, 0, s);
  if (st != CK_OK) throw Err(st, g->h->err);
  v.lazy_lrn = -1;
}

// The bnorm output a fused bnorm -> relu forward did not store: from x with
// the forward's (mu, inv), bit-identical.
static void materialize_value(ck_graph* g, Var& v, cudaStream_t s) {
  if (v.lazy_value < 0) return;
  Layer& l = g->layers[v.lazy_value];
  const Var& x = g->vars[l.in[0]];
  const int64_t C = x.shape.c;  // the forward's (w, b), not the current parameters
  bnorm_value(x.value, l.muinv + 2 * C, l.muinv + 3 * C, l.muinv, v.value,
              (int)(x.shape.h * x.shape.w), (int)x.shape.c, (int)x.shape.n,
              v.lazy_value_relu ? 1 : 0, s);
  v.lazy_value = -1;
  v.lazy_value_relu = false;
}

// The conv output's derivative a bnorm backward skipped (it wrote the conv's
// dy grid instead): that bnorm backward's dx, now, with the same gating.
static void materialize_bn(ck_graph* g, Var& v, cudaStream_t s) {
  if (v.lazy_bn < 0) return;
  Layer& l = g->layers[v.lazy_bn];
  ck_handle* h = g->h;
  ck_tensor x = tv(g->vars[l.in[0]], false), w = tv(g->vars[l.in[1]], false),
            b = tv(g->vars[l.in[2]], false), dx = tv(v, true),
            dy = tv(g->vars[l.out[0]], true);
  if (g->layers[g->vars[l.relu_out].producer].fused_done) {
    // the parameters of the forward this derivative belongs to (the trainer's
    // SGD may have moved w, b since): the snapshot after (mu, inv)
    const int64_t C = x.shape.c;
    w.data = l.muinv + 2 * C;
    b.data = l.muinv + 3 * C;
  }
  const bool fused = l.relu_out >= 0 && g->layers[g->vars[l.relu_out].producer].bwd_deferred;
  if (fused) {
    h->fuse_relu_x = g->vars[l.out[0]].value;
    h->fuse_relu_dy = g->vars[l.relu_out].deriv;
    if (g->layers[g->vars[l.relu_out].producer].fused_done) h->bn_muinv = l.muinv;
  }
  struct ResetM {
    ck_handle* h;
    ~ResetM() {
      h->fuse_relu_x = nullptr;
      h->fuse_relu_dy = nullptr;
      h->bn_muinv = nullptr;
    }
  } reset{h};
  const ck_status st = ck_bnorm_backward(h, &x, &w, &b, l.p[0], &dy, &dx, nullptr, nullptr, 0, s);
  if (st != CK_OK) throw Err(st, h->err);
  v.lazy_bn = -1;
}

static void layer_backward(ck_graph* g, Layer& l, cudaStream_t s) {
  ck_handle* h = g->h;
  auto V = [&](int k) { return tv(g->vars[l.in[k]], false); };
  auto D = [&](int k) { return tv(g->vars[l.in[k]], true); };
  auto acc = [&](int k) { return g->vars[l.in[k]].deriv_live ? 1 : 0; };
  auto mark = [&](int k) { g->vars[l.in[k]].deriv_live = true; };
  ck_tensor dy = tv(g->vars[l.out[0]], true);
  ck_status st = CK_OK;
  switch (l.kind) {
    case Kind::conv: {
      ck_tensor x = V(0), f = V(1), dx = D(0), df = D(1), b, db;
      if (l.in.size() > 2) db = D(2);
      (void)b;
      ck_conv_geom cg = conv_geom_of(l);
      // Independent accumulate flags per output: run the three passes
      // separately when they differ.
      int a0 = acc(0), a1 = acc(1), a2 = l.in.size() > 2 ? acc(2) : a1;
      h->conv_cache = &l.cache;  // the forward's transformed input (valid this step)
      const bool fused = l.relu_out >= 0 && g->layers[g->vars[l.relu_out].producer].bwd_deferred;
      const bool bn_pre = g->vars[l.out[0]].lazy_bn >= 0;
      if (l.pre_grid) {
        l.pre_grid = false;
        if ((fused || bn_pre) && a0 == a1 && a1 == a2 && l.in.size() > 2) {
          h->pre_dyg = (float*)l.dyg.ptr;
          h->pre_dyg_src = dy.data;
          h->pre_dyg_key = l.plan.key;
          h->pre_bpart = (const double*)l.bpart.ptr;
          h->pre_rows = l.pre_rows;
        } else if (bn_pre) {
          // cannot consume the prebuilt grid: materialize dy the bnorm skipped
          materialize_bn(g, g->vars[l.out[0]], s);
        } else {
          // cannot consume the prebuilt grid: materialize the relu output's
          // derivative the LRN skipped, then take the ordinary path
          materialize_lrn(g, g->vars[l.relu_out], s);
        }
      }
      if (fused) {
        // fused relu backward: this call derives dy from the relu output's derivative;
        // dy itself (the conv output's derivative) may stay unmaterialized
        h->fuse_relu_x = g->vars[l.out[0]].value;
        h->fuse_relu_dy = g->vars[l.relu_out].deriv;
        h->fuse_relu_lazy = true;
      }
      // conv -> relu -> this conv (AlexNet conv3 -> conv4 -> conv5): this data
      // gradient's epilogue also writes the conv below's relu-gated dy grid
      // and bias partials; that conv's backward then skips its dy transform
      Layer* below = nullptr;
      GridPlan bgp{};
      int brows = 0;
      if (g->dgrad_grid && g->math == CK_MATH_TF32 && !a0 && a0 == a1 && a1 == a2) {
        const Var& xv = g->vars[l.in[0]];
        if (xv.producer >= 0 && xv.consumers.size() == 1) {
          Layer& r = g->layers[xv.producer];
          if (r.kind == Kind::relu && r.fused_by >= 0 && r.fused_bwd &&
              g->layers[r.fused_by].kind == Kind::conv) {
            Layer& c = g->layers[r.fused_by];
            const ConvDims cd = conv_dims(g->vars[c.in[0]].shape, g->vars[c.in[1]].shape,
                                          g->vars[c.out[0]].shape, conv_geom_of(c));
            if (c.in.size() > 2 && !c.pre_grid && conv_tc_grid_plan(cd, &bgp) &&
                bgp.Kg % 32 == 0) {
              float* old = (float*)c.dyg.ptr;
              float* grid = (float*)c.dyg.get(bgp.bytes, s);
              if (!grid) throw Err(CK_ERR_CUDA, "dy grid allocation failed");
              if (grid != old)  // the grid's junk rows stay zero from here on
                check_cuda(cudaMemsetAsync(grid, 0, c.dyg.bytes, s), "zero");
              brows = (int)(((int64_t)cd.N * cd.OH * cd.OW + 31) / 32);
              double* bp =
                  (double*)c.bpart.get(sizeof(double) * (size_t)brows * bgp.Kgp * bgp.groups, s);
              if (!bp) throw Err(CK_ERR_CUDA, "bias partial allocation failed");
              h->prev_dyg = grid;
              h->prev_bpart = bp;
              h->prev_gate = xv.value;
              h->prev_dyg_plan = bgp;
              h->prev_dyg_done = false;
              below = &c;
            }
          }
        }
      }
      struct Reset {
        ck_handle* h;
        ~Reset() {
          h->conv_cache = nullptr;
          h->fuse_relu_x = nullptr;
          h->fuse_relu_dy = nullptr;
          h->fuse_relu_lazy = false;
          h->fuse_relu_pending = false;
          h->pre_dyg = nullptr;
          h->pre_dyg_src = nullptr;
          h->pre_bpart = nullptr;
          h->prev_dyg = nullptr;
          h->prev_bpart = nullptr;
          h->prev_gate = nullptr;
          h->prev_dyg_done = false;
        }
      } reset{h};
      if (a0 == a1 && a1 == a2) {
        st = ck_conv_backward(h, &x, &f, &cg, &dy, &dx, &df, l.in.size() > 2 ? &db : nullptr, a0,
                              g->math, s);
        if (st == CK_OK && fused && h->fuse_relu_pending) {
          g->vars[l.out[0]].lazy_gate = l.out[0];
          g->vars[l.out[0]].lazy_src = l.relu_out;
        }
        if (st == CK_OK && below && h->prev_dyg_done) {
          below->pre_grid = true;
          below->plan = bgp;
          below->pre_rows = brows;
        }
      } else {
        st = ck_conv_backward(h, &x, &f, &cg, &dy, &dx, nullptr, nullptr, a0, g->math, s);
        if (st == CK_OK) st = ck_conv_backward(h, &x, &f, &cg, &dy, nullptr, &df, nullptr, a1, g->math, s);
        if (st == CK_OK && l.in.size() > 2)
          st = ck_conv_backward(h, &x, &f, &cg, &dy, nullptr, nullptr, &db, a2, g->math, s);
      }
      for (size_t k = 0; k < l.in.size(); ++k) mark((int)k);
      break;
    }
    case Kind::convt: {
      ck_tensor x = V(0), f = V(1), dx = D(0), df = D(1);
      ck_convt_geom cg = convt_geom_of(l);
      int a0 = acc(0), a1 = acc(1);
      if (a0 == a1) {
        st = ck_convt_backward(h, &x, &f, &cg, &dy, &dx, &df, a0, g->math, s);
      } else {
        st = ck_convt_backward(h, &x, &f, &cg, &dy, &dx, nullptr, a0, g->math, s);
        if (st == CK_OK) st = ck_convt_backward(h, &x, &f, &cg, &dy, nullptr, &df, a1, g->math, s);
      }
      mark(0);
      mark(1);
      break;
    }
    case Kind::pool: {
      ck_tensor x = V(0), dx = D(0);
      ck_pool_geom pg = pool_geom_of(l);
      h->conv_cache = &l.cache;
      st = ck_pool_backward(h, &x, &pg, &dy, &dx, acc(0), s);
      h->conv_cache = nullptr;
      mark(0);
      break;
    }
    case Kind::relu: {
      l.bwd_deferred = l.fused_by >= 0 && l.fused_bwd && !acc(0);
      if (l.bwd_deferred) {
        // the producing conv's backward derives this derivative itself
        // (ck_conv_backward with fuse_relu_x / fuse_relu_dy)
        mark(0);
        break;
      }
      materialize_value(g, g->vars[l.in[0]], s);  // (a bnorm output left unstored)
      ck_tensor x = V(0), dx = D(0);
      st = ck_relu_backward(h, &x, &dy, &dx, acc(0), s);
      mark(0);
      break;
    }
    case Kind::lrn: {
      ck_tensor x = V(0), dx = D(0);
      ck_lrn_params p = lrn_of(l);
      // lrn <- relu <- conv with the relu fused into the conv (TF32 grid path):
      // write the conv's ReLU-gated dy grid (+ bias partials) directly; the
      // relu output's derivative is then computed only on request
      Var& xv = g->vars[l.in[0]];
      if (!acc(0) && g->math == CK_MATH_TF32 && xv.producer >= 0 && xv.consumers.size() == 1 &&
          g->lrn_grid) {
        Layer& r = g->layers[xv.producer];
        if (r.kind == Kind::relu && r.fused_by >= 0 && r.fused_bwd &&
            g->layers[r.fused_by].kind == Kind::conv) {
          Layer& c = g->layers[r.fused_by];
          const Var& cx = g->vars[c.in[0]];
          const Var& cf = g->vars[c.in[1]];
          const ConvDims cd = conv_dims(cx.shape, cf.shape, g->vars[c.out[0]].shape,
                                        conv_geom_of(c));
          GridPlan gp;
          if (c.in.size() > 2 && conv_tc_grid_plan(cd, &gp)) {
            float* old = (float*)c.dyg.ptr;
            float* grid = (float*)c.dyg.get(gp.bytes, s);
            if (!grid) throw Err(CK_ERR_CUDA, "dy grid allocation failed");
            if (grid != old)  // the grid's junk rows stay zero from here on
              check_cuda(cudaMemsetAsync(grid, 0, c.dyg.bytes, s), "zero");
            const int rows = lrn_grid_rows((int)x.shape.h, (int)x.shape.w, (int)x.shape.n);
            double* bp = (double*)c.bpart.get(sizeof(double) * (size_t)rows * gp.Kgp * gp.groups, s);
            if (!bp) throw Err(CK_ERR_CUDA, "bias partial allocation failed");
            if (lrn_backward_grid(x.data, dy.data, grid, bp, (int)x.shape.h, (int)x.shape.w,
                                  (int)x.shape.c, (int)x.shape.n, (int)p.group_size,
                                  (float)p.kappa, (float)p.alpha, (float)p.beta, gp.Hg, gp.Wg,
                                  gp.Kg, gp.Kgp, gp.groups, s)) {
              c.pre_grid = true;
              c.plan = gp;
              c.pre_rows = rows;
              xv.lazy_lrn = (int)(&l - &g->layers[0]);
              mark(0);
              break;
            }
          }
        }
      }
      st = ck_lrn_backward(h, &x, &p, &dy, &dx, acc(0), s);
      mark(0);
      break;
    }
    case Kind::bnorm: {
      ck_tensor x = V(0), w = V(1), b = V(2), dx = D(0), dw = D(1), db = D(2);
      int a0 = acc(0), a1 = acc(1), a2 = acc(2);
      // fused bnorm -> relu: the relu backward was deferred; this layer reads
      // the relu output's derivative gated by its own output (> 0), and its
      // output's derivative stays unmaterialized (computed on request)
      const bool fused = l.relu_out >= 0 && g->layers[g->vars[l.relu_out].producer].bwd_deferred;
      if (fused) {
        h->fuse_relu_x = g->vars[l.out[0]].value;
        h->fuse_relu_dy = g->vars[l.relu_out].deriv;
        // (mu, inv) written by this step's fused forward, if it ran fused
        if (g->layers[g->vars[l.relu_out].producer].fused_done) h->bn_muinv = l.muinv;
      }
      struct ResetB {
        ck_handle* h;
        ~ResetB() {
          h->fuse_relu_x = nullptr;
          h->fuse_relu_dy = nullptr;
          h->bn_muinv = nullptr;
        }
      } resetb{h};
      if (fused) {
        g->vars[l.out[0]].lazy_gate = l.out[0];
        g->vars[l.out[0]].lazy_src = l.relu_out;
      }
      // conv -> bnorm (VGG): write the conv's dy grid (+ bias partials) from
      // this backward; the conv output's derivative is computed on request
      Var& xv = g->vars[l.in[0]];
      if (g->bn_grid && g->math == CK_MATH_TF32 && !a0 && a1 == a2 && xv.producer >= 0 &&
          xv.consumers.size() == 1) {
        Layer& c = g->layers[xv.producer];
        if (c.kind == Kind::conv && c.in.size() > 2 && c.relu_out < 0 && !c.pre_grid) {
          const ConvDims cd = conv_dims(g->vars[c.in[0]].shape, g->vars[c.in[1]].shape,
                                        xv.shape, conv_geom_of(c));
          GridPlan gp;
          if (conv_tc_grid_plan(cd, &gp) && gp.Kg % 32 == 0) {
            float* old = (float*)c.dyg.ptr;
            float* grid = (float*)c.dyg.get(gp.bytes, s);
            if (!grid) throw Err(CK_ERR_CUDA, "dy grid allocation failed");
            if (grid != old)  // the grid's junk rows stay zero from here on
              check_cuda(cudaMemsetAsync(grid, 0, c.dyg.bytes, s), "zero");
            const int rows = (int)((elems(xv.shape) / xv.shape.c + 31) / 32);
            double* bp =
                (double*)c.bpart.get(sizeof(double) * (size_t)rows * gp.Kgp * gp.groups, s);
            if (!bp) throw Err(CK_ERR_CUDA, "bias partial allocation failed");
            if (bnorm_backward_to_grid(h, &x, &w, &b, l.p[0], &dy, &dw, &db, a1, gp, grid, bp, s)) {
              c.pre_grid = true;
              c.plan = gp;
              c.pre_rows = rows;
              xv.lazy_bn = (int)(&l - &g->layers[0]);
              mark(0);
              mark(1);
              mark(2);
              break;
            }
          }
        }
      }
      if (a0 == a1 && a1 == a2) {
        st = ck_bnorm_backward(h, &x, &w, &b, l.p[0], &dy, &dx, &dw, &db, a0, s);
      } else {
        st = ck_bnorm_backward(h, &x, &w, &b, l.p[0], &dy, &dx, nullptr, nullptr, a0, s);
        if (st == CK_OK) st = ck_bnorm_backward(h, &x, &w, &b, l.p[0], &dy, nullptr, &dw, nullptr, a1, s);
        if (st == CK_OK) st = ck_bnorm_backward(h, &x, &w, &b, l.p[0], &dy, nullptr, nullptr, &db, a2, s);
      }
      mark(0);
      mark(1);
      mark(2);
      break;
    }
    case Kind::loss: {
      ck_tensor x = V(0), c = V(1), dx = D(0), w;
      if (l.in.size() > 2) w = V(2);
      // the projection (graph.cpp:420-425: proj[0][0], 1 for the objective) is
      // read on the device from the loss output's derivative: no host sync
      loss_backward_any(h, &x, &c, l.in.size() > 2 ? &w : nullptr, loss_kind_of(l), 1.0f,
                        g->vars[l.out[0]].deriv, dx.data, acc(0), s);
      after_launch();
      mark(0);  // labels / weights carry no derivative: left for the final zeroing
      break;
    }
    case Kind::sigmoid: {
      // activation.cpp:41-48 consumes the forward output (graph.cpp:388-389)
      ck_tensor yv = tv(g->vars[l.out[0]], false), dx = D(0);
      st = ck_sigmoid_backward(h, &yv, &dy, &dx, acc(0), s);
      mark(0);
      break;
    }
    case Kind::softmax: {
      ck_tensor yv = tv(g->vars[l.out[0]], false), dx = D(0);
      st = ck_softmax_backward(h, &yv, &dy, &dx, acc(0), s);
      mark(0);
      break;
    }
    case Kind::spnorm: {
      ck_tensor x = V(0), dx = D(0);
      const ck_spnorm_params sp = spnorm_of(l);
      st = ck_spnorm_backward(h, &x, &sp, &dy, &dx, acc(0), s);
      mark(0);
      break;
    }
    case Kind::bilinear: {
      ck_tensor x = V(0), gr = V(1), dx = D(0), dg = D(1);
      if (acc(0) == acc(1)) {
        st = ck_bilinear_backward(h, &x, &gr, &dy, &dx, &dg, acc(0), s);
      } else {
        st = ck_bilinear_backward(h, &x, &gr, &dy, &dx, nullptr, acc(0), s);
        if (st == CK_OK) st = ck_bilinear_backward(h, &x, &gr, &dy, nullptr, &dg, acc(1), s);
      }
      mark(0);
      mark(1);
      break;
    }
    case Kind::pdist: {
      ck_tensor x = V(0), t = V(1), dx = D(0), dt = D(1);
      const double p = pdist_p(l);
      const int nr = pdist_no_root(l);
      if (acc(0) == acc(1)) {
        st = ck_pdist_backward(h, &x, &t, p, nr, &dy, &dx, &dt, acc(0), s);
      } else {
        st = ck_pdist_backward(h, &x, &t, p, nr, &dy, &dx, nullptr, acc(0), s);
        if (st == CK_OK) st = ck_pdist_backward(h, &x, &t, p, nr, &dy, nullptr, &dt, acc(1), s);
      }
      mark(0);
      mark(1);
      break;
    }
    case Kind::split: {
      // graph.cpp split backward: dx = sum of the projections in output order
      // (outputs no live derivative reached are the reference's zeros: skipped)
      std::vector<const float*> src;
      for (int o : l.out)
        if (g->vars[o].deriv_live) src.push_back(g->vars[o].deriv);
      sum_into(D(0).data, src.data(), (int)src.size(), elems(D(0).shape), acc(0), s);
      after_launch();
      mark(0);
      break;
    }
    case Kind::sum: {
      for (size_t k = 0; k < l.in.size(); ++k) {
        ck_tensor dx = D((int)k);
        if (acc((int)k))
          axpy_inplace(dx.data, dy.data, elems(dy.shape), s);
        else
          check_cuda(cudaMemcpyAsync(dx.data, dy.data, sizeof(float) * elems(dy.shape),
                                     cudaMemcpyDeviceToDevice, s), "copy");
        mark((int)k);
      }
      break;
    }
  }
  if (st != CK_OK) throw Err(st, "layer '" + l.name + "': " + h->err);
}

// graph.cpp:494-545 forward (train mode).
// NVTX ranges per layer pass and per gradient bucket (host-side markers for
// nsys / ncu --nvtx; free when no tool is attached).
struct NvtxRange {
  explicit NvtxRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~NvtxRange() { nvtxRangePop(); }
};

static void run_forward(ck_graph* g, cudaStream_t s) {
  for (auto& l : g->layers) l.cache.valid = false;
  // loss layers record label errors (loss.cpp:101-106) in the handle's flag
  if (g->has_loss) reset_label_flag(g->h, s);
  for (int li : g->order) {
    NvtxRange r(g->layers[li].name + " fwd");
    g->prof(li, 0, s);
    layer_forward(g, g->layers[li], s);
    g->prof(li, 1, s);
    if (g->profiling) g->prof_fwd_done[li] = 1;
  }
}

struct LayerDone {
  // Called after each layer's backward with the layer index; used by the
  // trainer to launch the gradient allreduce of finished parameters.
  virtual void done(int li, cudaStream_t s) = 0;
  virtual ~LayerDone() = default;
};

// graph.cpp:548-598 backward with d(objective) = 1.
static void run_backward(ck_graph* g, int objective, cudaStream_t s, LayerDone* cb) {
  for (auto& v : g->vars) {
    v.deriv_live = false;
    v.lazy_gate = v.lazy_src = v.lazy_lrn = v.lazy_bn = -1;
  }
  for (auto& l : g->layers) l.pre_grid = false;
  for (auto& l : g->layers) l.bwd_deferred = false;
  Var& obj = g->vars[objective];
  if (elems(obj.shape) != 1) throw Err(CK_ERR_ARG, "objective '" + obj.name + "' is not a scalar");
  check_cuda(cudaMemcpyAsync(obj.deriv, g->one_dev, sizeof(float), cudaMemcpyDeviceToDevice, s),
             "seed");
  obj.deriv_live = true;
  for (auto it = g->order.rbegin(); it != g->order.rend(); ++it) {
    Layer& l = g->layers[*it];
    bool any = false;
    for (int o : l.out) any |= g->vars[o].deriv_live;
    if (any) {
      NvtxRange r(l.name + " bwd");
      g->prof(*it, 2, s);
      layer_backward(g, l, s);
      g->prof(*it, 3, s);
      if (g->profiling) g->prof_bwd_done[*it] = 1;
    }
    if (cb) cb->done(*it, s);
  }
  // Derivatives nobody wrote are the reference's zero-initialised tensors.
  for (auto& v : g->vars)
    if (!v.deriv_live)
      check_cuda(cudaMemsetAsync(v.deriv, 0, sizeof(float) * elems(v.shape), s), "zero");
}

}  // namespace ck

// ---- trainer ---------------------------------------------------------------

struct ck_trainer : ck::LayerDone {
  ck_graph* g = nullptr;
  int objective = -1;
  float lr = 0.01f, momentum = 0.9f, wd = 5e-4f;
  std::vector<int> params;         // param var indices
  std::vector<float*> mom;         // momentum buffers
  // DP
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> ev;     // per layer "gradient ready"
  cudaEvent_t comm_done = nullptr;
  std::vector<std::vector<int>> layer_params;  // params finished by layer li
  float* loss_dev = nullptr;
  int64_t allreduces = 0;          // NCCL allreduce groups issued (evidence)
  bool update_stream = true;       // single GPU: SGD on a side stream
  // label/data flag of each step, copied to pinned host memory at its end
  // and checked when that copy is known complete (CK_ERR_DATA, loss.cpp:101-106)
  int* flag_host = nullptr;
  cudaEvent_t flag_ev = nullptr;
  bool flag_pending = false;
  // step timing (profiling steps only): forward / backward on the compute
  // stream, and the end of the last allreduce+SGD on the comm stream
  cudaEvent_t t_begin = nullptr, t_fwd = nullptr, t_bwd = nullptr, t_comm = nullptr;
  bool timed = false;
  // single GPU: each layer's SGD runs on an update stream as soon as that
  // layer's backward is done, overlapping the rest of the backward (the
  // streaming update fits beside a persistent GEMM's CTAs on the same SMs)
  cudaStream_t upd_stream = nullptr;
  std::vector<cudaEvent_t> upd_ev;
  cudaEvent_t upd_done = nullptr;
  bool upd_pending = false;
  // CUDA-graph replay of the whole step (ck_trainer_set_graph)
  bool use_graph = false;
  int eager_steps = 0;                 // workspaces are sized by one eager step
  // one captured step per (stream, input bindings): a caller alternating two
  // bound input buffers (ck_graph_bind_input, graph.Feeder) replays two graphs
  struct Captured {
    cudaStream_t stream;
    std::vector<float*> inputs;
    cudaGraphExec_t exec;
    int64_t launches;
    int64_t tc_launches;  // of which tcgen05 GEMMs
    uint64_t gen;  // workspace generation the captured pointers belong to
  };
  uint64_t eager_gen = 0;  // workspace generation after the last eager step
  std::vector<Captured> graphs;

  void done(int li, cudaStream_t s) override {
    const auto& ps = layer_params[li];
    if (ps.empty()) return;
    // a parameter no live derivative reached (its consumers' backward did not
    // run) has the reference's zero derivative (graph.cpp:551-554) -- before
    // the allreduce and the update read it
    for (int p : ps) {
      ck::Var& v = g->vars[p];
      if (!v.deriv_live) {
        ck::check_cuda(cudaMemsetAsync(v.deriv, 0, sizeof(float) * ck::elems(v.shape), s), "zero");
        v.deriv_live = true;
      }
    }
    if (comm) {
      // this layer's finished parameters are adjacent in the arena (finalize):
      // one allreduce per contiguous run (normally exactly one per layer)
      std::vector<std::pair<float*, float*>> runs;
      for (int p : ps) {
        ck::Var& v = g->vars[p];
        runs.push_back({v.deriv, v.deriv + (ck::elems(v.shape) + 31) / 32 * 32});
      }
      std::sort(runs.begin(), runs.end());
      std::vector<std::pair<float*, float*>> merged;
      for (auto& r : runs)
        if (!merged.empty() && r.first <= merged.back().second)
          merged.back().second = std::max(merged.back().second, r.second);
        else
          merged.push_back(r);
      ck::NvtxRange r("allreduce " + g->layers[li].name);
      ck::check_cuda(cudaEventRecord(ev[li], s), "event");
      ck::check_cuda(cudaStreamWaitEvent(comm_stream, ev[li], 0), "wait");
      if (ncclGroupStart() != ncclSuccess) throw Err(CK_ERR_CUDA, "ncclGroupStart failed");
      for (auto& r : merged)
        if (ncclAllReduce(r.first, r.first, (size_t)(r.second - r.first), ncclFloat, ncclSum, comm,
                          comm_stream) != ncclSuccess)
          throw Err(CK_ERR_CUDA, "ncclAllReduce failed");
      if (ncclGroupEnd() != ncclSuccess) throw Err(CK_ERR_CUDA, "ncclGroupEnd failed");
      ++allreduces;
      for (int p : ps) sgd(p, comm_stream);
    } else if (!update_stream) {
      for (int p : ps) sgd(p, s);
    } else {
      if (!upd_stream) {
        ck::check_cuda(cudaStreamCreateWithFlags(&upd_stream, cudaStreamNonBlocking), "stream");
        upd_ev.assign(g->layers.size(), nullptr);
        for (auto& e : upd_ev)
          ck::check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        ck::check_cuda(cudaEventCreateWithFlags(&upd_done, cudaEventDisableTiming), "event");
      }
      ck::check_cuda(cudaEventRecord(upd_ev[li], s), "event");
      ck::check_cuda(cudaStreamWaitEvent(upd_stream, upd_ev[li], 0), "wait");
      for (int p : ps) sgd(p, upd_stream);
      upd_pending = true;
    }
  }
  // the step's parameters are final only after every queued update: join
  void join_updates(cudaStream_t s) {
    if (!upd_pending) return;
    ck::check_cuda(cudaEventRecord(upd_done, upd_stream), "event");
    ck::check_cuda(cudaStreamWaitEvent(s, upd_done, 0), "wait");
    upd_pending = false;
  }
  void sgd(int p, cudaStream_t s) {
    ck::Var& v = g->vars[p];
    size_t k = std::find(params.begin(), params.end(), p) - params.begin();
    ck_status st = ck_sgd_step(g->h, v.value, mom[k], v.deriv, ck::elems(v.shape), lr, momentum,
                               wd, s);
    if (st != CK_OK) throw Err(st, g->h->err);
  }
  void drop_graph() {
    for (auto& c : graphs) cudaGraphExecDestroy(c.exec);
    graphs.clear();
  }
  ~ck_trainer() override {
    drop_graph();
    for (float* m : mom) cudaFree(m);
    for (auto e : ev) cudaEventDestroy(e);
    if (comm_done) cudaEventDestroy(comm_done);
    for (auto e : upd_ev) cudaEventDestroy(e);
    if (upd_done) cudaEventDestroy(upd_done);
    if (upd_stream) cudaStreamDestroy(upd_stream);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (comm) ncclCommDestroy(comm);
    if (loss_dev) cudaFree(loss_dev);
    if (flag_host) cudaFreeHost(flag_host);
    for (auto e : {flag_ev, t_begin, t_fwd, t_bwd, t_comm})
      if (e) cudaEventDestroy(e);
  }
};

using namespace ck;

#define CKG_BEGIN(gr)                     \
  if (!(gr) || !(gr)->h) return CK_ERR_ARG; \
  ck::HandleScope _scope((gr)->h);        \
  try {
#define CKG_END(gr)                       \
  return CK_OK;                           \
  }                                       \
  catch (const ck::Err& e) {              \
    (gr)->h->err = e.what();              \
    return e.code;                        \
  }                                       \
  catch (const std::exception& e) {       \
    (gr)->h->err = e.what();              \
    return CK_ERR_ARG;                    \
  }

extern "C" {

ck_status ck_graph_create(ck_handle* h, ck_graph** out) {
  if (!h || !out) return CK_ERR_ARG;
  *out = new ck_graph();
  (*out)->h = h;
  return CK_OK;
}

void ck_graph_destroy(ck_graph* g) {
  if (!g) return;
  cudaSetDevice(g->h->device);
  cudaDeviceSynchronize();
  delete g;
}

static ck_status add_var(ck_graph* g, const char* name, ck_shape shape, int role) {
  CKG_BEGIN(g)
  if (g->finalized) throw Err(CK_ERR_ARG, "graph already finalized");
  if (!name || !*name) throw Err(CK_ERR_ARG, "empty variable name");
  if (g->by_name.count(name)) throw Err(CK_ERR_ARG, std::string("variable '") + name + "' declared twice");
  if (shape.h < 1 || shape.w < 1 || shape.c < 1 || shape.n < 1)
    throw Err(CK_ERR_SHAPE, "invalid tensor shape " + shape_str(shape));
  for (const char* c = name; *c; ++c)
    if (*c == ' ' || *c == '\t' || *c == '\n' || *c == ',' || *c == '=')
      throw Err(CK_ERR_ARG, std::string("variable name '") + name + "' contains a separator");
  int k = g->intern(name, role);
  g->vars[k].shape = shape;
  g->vars[k].has_shape = true;
  g->decl.push_back(k);
  CKG_END(g)
}

ck_status ck_graph_add_input(ck_graph* g, const char* name, ck_shape shape) {
  return add_var(g, name, shape, 0);
}
ck_status ck_graph_add_param(ck_graph* g, const char* name, ck_shape shape) {
  return add_var(g, name, shape, 1);
}

ck_status ck_graph_add_layer(ck_graph* g, const char* kind, const char* name,
                             const char* inputs_csv, const char* outputs_csv,
                             const double* params, int nparams) {
  CKG_BEGIN(g)
  if (g->finalized) throw Err(CK_ERR_ARG, "graph already finalized");
  Layer l;
  l.name = name ? name : "";
  l.kind = kind_from_name(kind ? kind : "");
  for (auto& n : split_csv(inputs_csv)) l.in.push_back(g->intern(n, 2));
  for (auto& n : split_csv(outputs_csv)) l.out.push_back(g->intern(n, 2));
  if (l.out.empty()) throw Err(CK_ERR_ARG, "layer '" + l.name + "' has no outputs");
  if (params && nparams > 0) l.p.assign(params, params + nparams);
  g->layers.push_back(std::move(l));
  CKG_END(g)
}

ck_status ck_graph_finalize(ck_graph* g, ck_math math) {
  CKG_BEGIN(g)
  if (g->finalized) throw Err(CK_ERR_ARG, "graph already finalized");
  g->math = math;
  finalize(g);
  CKG_END(g)
}

ck_status ck_graph_var(ck_graph* g, const char* name, int deriv, ck_tensor* out) {
  CKG_BEGIN(g)
  if (!g->finalized) throw Err(CK_ERR_ARG, "graph not finalized");
  if (!out) throw Err(CK_ERR_ARG, "null output");
  Var& v = g->vars[g->var(name ? name : "")];
  if (!deriv && v.lazy_value >= 0) {
    check_cuda(cudaDeviceSynchronize(), "synchronize");
    materialize_value(g, v, 0);
    check_cuda(cudaDeviceSynchronize(), "synchronize");
  }
  if (deriv && v.lazy_bn >= 0) {
    check_cuda(cudaDeviceSynchronize(), "synchronize");
    materialize_bn(g, v, 0);
    check_cuda(cudaDeviceSynchronize(), "synchronize");
  }
  if (deriv && v.lazy_lrn >= 0) {
    check_cuda(cudaDeviceSynchronize(), "synchronize");
    materialize_lrn(g, v, 0);
    check_cuda(cudaDeviceSynchronize(), "synchronize");
  }
  if (deriv && v.lazy_gate >= 0 && g->vars[v.lazy_src].lazy_lrn >= 0) {
    check_cuda(cudaDeviceSynchronize(), "synchronize");
    materialize_lrn(g, g->vars[v.lazy_src], 0);
  }
  if (deriv && v.lazy_gate >= 0) {
    // a fused conv -> relu backward left this derivative unmaterialized:
    // relu backward (activation.cpp:14-22) of the relu output's derivative,
    // gated by this var's own value (x > 0), now, in order with all prior work
    check_cuda(cudaDeviceSynchronize(), "synchronize");
    materialize_value(g, g->vars[v.lazy_gate], 0);
    relu_backward(g->vars[v.lazy_gate].value, g->vars[v.lazy_src].deriv, v.deriv,
                  elems(v.shape), 0, 0);
    check_cuda(cudaDeviceSynchronize(), "synchronize");
    v.lazy_gate = v.lazy_src = -1;
  }
  *out = tv(v, deriv != 0);
  CKG_END(g)
}

ck_status ck_graph_bind_input(ck_graph* g, const char* name, float* data) {
  CKG_BEGIN(g)
  if (!g->finalized) throw Err(CK_ERR_ARG, "graph not finalized");
  Var& v = g->vars[g->var(name ? name : "")];
  if (v.role != 0) throw Err(CK_ERR_ARG, "'" + v.name + "' is not a graph input");
  if (!v.own_value) v.own_value = v.value;
  v.value = data ? data : v.own_value;
  CKG_END(g)
}

ck_status ck_graph_forward(ck_graph* g, ck_stream stream) {
  CKG_BEGIN(g)
  if (!g->finalized) throw Err(CK_ERR_ARG, "forward on a non-finalized graph");
  int64_t before = g->h->counter.n;
  run_forward(g, (cudaStream_t)stream);
  g->last_launches = g->h->counter.n - before;
  // the reference throws DataError from the loss layer: read the flag now
  if (g->has_loss) {
    try {
      read_label_flag(g->h, (cudaStream_t)stream);
    } catch (const Err& e) {
      throw Err(e.code, std::string("loss layer: ") + e.what());
    }
  }
  CKG_END(g)
}

ck_status ck_graph_backward(ck_graph* g, const char* objective, ck_stream stream) {
  CKG_BEGIN(g)
  if (!g->finalized) throw Err(CK_ERR_ARG, "backward on a non-finalized graph");
  int64_t before = g->h->counter.n;
  run_backward(g, g->var(objective ? objective : ""), (cudaStream_t)stream, nullptr);
  g->last_launches += g->h->counter.n - before;
  CKG_END(g)
}

int64_t ck_graph_last_launches(const ck_graph* g) { return g ? g->last_launches : 0; }

ck_status ck_graph_set_profiling(ck_graph* g, int enable) {
  CKG_BEGIN(g)
  if (enable && g->prof_ev.empty()) {
    g->prof_ev.resize(4 * g->layers.size());
    for (auto& e : g->prof_ev) check_cuda(cudaEventCreate(&e), "event");
  }
  g->prof_fwd_done.assign(g->layers.size(), 0);
  g->prof_bwd_done.assign(g->layers.size(), 0);
  g->profiling = enable != 0;
  CKG_END(g)
}

ck_status ck_graph_set_option(ck_graph* g, const char* name, int64_t value) {
  CKG_BEGIN(g)
  const std::string n = name ? name : "";
  if (n == "lrn_grid")
    g->lrn_grid = value != 0;
  else if (n == "lrn_pool")
    g->lrn_pool = value != 0;
  else if (n == "producer_grid")
    g->producer_grid = value != 0;
  else if (n == "dgrad_grid")
    g->dgrad_grid = value != 0;
  else if (n == "bn_grid")
    g->bn_grid = value != 0;
  else if (n == "bn_lazy_y")
    g->bn_lazy_y = value != 0;
  else
    throw Err(CK_ERR_ARG, "unknown graph option '" + n + "'");
  CKG_END(g)
}

int ck_graph_layer_count(const ck_graph* g) { return g ? (int)g->layers.size() : 0; }

const char* ck_graph_layer_name(const ck_graph* g, int layer) {
  if (!g || layer < 0 || layer >= (int)g->layers.size()) return "";
  return g->layers[layer].name.c_str();
}

ck_status ck_graph_layer_ms(ck_graph* g, int layer, float* fwd_ms, float* bwd_ms) {
  CKG_BEGIN(g)
  if (layer < 0 || layer >= (int)g->layers.size()) throw Err(CK_ERR_ARG, "bad layer index");
  if (g->prof_ev.empty()) throw Err(CK_ERR_ARG, "profiling was never enabled");
  float a = 0.f, b = 0.f;
  if (g->prof_fwd_done[layer])
    check_cuda(cudaEventElapsedTime(&a, g->prof_ev[4 * layer], g->prof_ev[4 * layer + 1]), "elapsed");
  if (g->prof_bwd_done[layer])
    check_cuda(cudaEventElapsedTime(&b, g->prof_ev[4 * layer + 2], g->prof_ev[4 * layer + 3]), "elapsed");
  if (fwd_ms) *fwd_ms = a;
  if (bwd_ms) *bwd_ms = b;
  CKG_END(g)
}

ck_status ck_nccl_unique_id(char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CK_ERR_CUDA;
  std::memcpy(out, &id, 128);
  return CK_OK;
}

ck_status ck_trainer_create(ck_graph* g, const char* objective, float lr, float momentum,
                            float weight_decay, ck_trainer** out) {
  CKG_BEGIN(g)
  if (!g->finalized) throw Err(CK_ERR_ARG, "trainer needs a finalized graph");
  if (!out) throw Err(CK_ERR_ARG, "null output");
  auto t = std::make_unique<ck_trainer>();
  t->g = g;
  t->objective = g->var(objective ? objective : "");
  t->lr = lr;
  t->momentum = momentum;
  t->wd = weight_decay;
  t->layer_params.assign(g->layers.size(), {});
  // A parameter is final after its last consumer in backward order, i.e.
  // its first consumer in firing order.
  std::vector<int> pos(g->layers.size());
  for (size_t k = 0; k < g->order.size(); ++k) pos[g->order[k]] = (int)k;
  for (size_t i = 0; i < g->vars.size(); ++i) {
    Var& v = g->vars[i];
    if (v.role != 1 || v.consumers.empty()) continue;
    int first = v.consumers[0].first;
    for (auto [c, s] : v.consumers) {
      (void)s;
      if (pos[c] < pos[first]) first = c;
    }
    t->layer_params[first].push_back((int)i);
    t->params.push_back((int)i);
    float* m = nullptr;
    check_cuda(cudaMalloc(&m, sizeof(float) * std::max<int64_t>(1, elems(v.shape))), "cudaMalloc");
    check_cuda(cudaMemset(m, 0, sizeof(float) * elems(v.shape)), "memset");
    t->mom.push_back(m);
  }
  t->ev.resize(g->layers.size());
  for (auto& e : t->ev) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  check_cuda(cudaEventCreateWithFlags(&t->comm_done, cudaEventDisableTiming), "event");
  check_cuda(cudaMalloc(&t->loss_dev, sizeof(float)), "cudaMalloc");
  check_cuda(cudaHostAlloc(&t->flag_host, 2 * sizeof(int), cudaHostAllocDefault), "host alloc");
  t->flag_host[0] = t->flag_host[1] = 0;
  check_cuda(cudaEventCreateWithFlags(&t->flag_ev, cudaEventDisableTiming), "event");
  for (cudaEvent_t* e : {&t->t_begin, &t->t_fwd, &t->t_bwd, &t->t_comm})
    check_cuda(cudaEventCreate(e), "event");
  *out = t.release();
  CKG_END(g)
}

void ck_trainer_destroy(ck_trainer* t) {
  if (!t) return;
  cudaSetDevice(t->g->h->device);
  cudaDeviceSynchronize();
  delete t;
}

ck_status ck_trainer_init_dp(ck_trainer* t, const char id[128], int rank, int world) {
  if (!t) return CK_ERR_ARG;
  ck_graph* g = t->g;
  CKG_BEGIN(g)
  if (world < 1 || rank < 0 || rank >= world) throw Err(CK_ERR_ARG, "bad rank/world");
  if (t->comm) throw Err(CK_ERR_ARG, "data parallelism already initialised");
  t->rank = rank;
  t->world = world;
  // world == 1 still builds a (one-rank) communicator: the step then runs the
  // real DP path -- per-layer allreduce on the comm stream, event hand-off,
  // SGD there, loss allreduce -- which is what the one-GPU tests exercise
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  if (ncclCommInitRank(&t->comm, world, uid, rank) != ncclSuccess)
    throw Err(CK_ERR_CUDA, "ncclCommInitRank failed");
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  check_cuda(cudaStreamCreateWithPriority(&t->comm_stream, cudaStreamNonBlocking, hi), "stream");
  CKG_END(g)
}

// One training step's device work on stream s: forward, backward with the
// per-layer gradient allreduce + SGD, objective to loss_dev, the step's label
// flag to pinned host memory.
static void trainer_body(ck_trainer* t, cudaStream_t s) {
  ck_graph* g = t->g;
  const bool timed = g->profiling;  // profiling steps are always eager
  if (timed) check_cuda(cudaEventRecord(t->t_begin, s), "event");
  if (!g->has_loss) reset_label_flag(g->h, s);  // (run_forward resets it otherwise)
  run_forward(g, s);
  flag_nonfinite(g->vars[t->objective].value, elems(g->vars[t->objective].shape), g->h->flag, 64,
                 s);
  if (timed) check_cuda(cudaEventRecord(t->t_fwd, s), "event");
  run_backward(g, t->objective, s, t);
  if (timed) check_cuda(cudaEventRecord(t->t_bwd, s), "event");
  Var& obj = g->vars[t->objective];
  if (t->comm) {
    // Loss: summed over ranks for reporting only.
    check_cuda(cudaEventRecord(t->ev[0], s), "event");
    check_cuda(cudaStreamWaitEvent(t->comm_stream, t->ev[0], 0), "wait");
    if (ncclAllReduce(obj.value, t->loss_dev, 1, ncclFloat, ncclSum, t->comm, t->comm_stream) !=
        ncclSuccess)
      throw Err(CK_ERR_CUDA, "ncclAllReduce failed");
    if (timed) check_cuda(cudaEventRecord(t->t_comm, t->comm_stream), "event");
    check_cuda(cudaEventRecord(t->comm_done, t->comm_stream), "event");
    check_cuda(cudaStreamWaitEvent(s, t->comm_done, 0), "wait");
  } else {
    check_cuda(cudaMemcpyAsync(t->loss_dev, obj.value, sizeof(float), cudaMemcpyDeviceToDevice, s),
               "copy");
    t->join_updates(s);
    if (timed) check_cuda(cudaEventRecord(t->t_comm, s), "event");
  }
  t->timed = timed;
  check_cuda(cudaMemcpyAsync(t->flag_host, g->h->flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, s),
             "flag");
}

// The label flag of the last step, once its copy is known complete (or
// after a synchronize): CK_ERR_DATA with the reference's message.
static void check_step_flag(ck_trainer* t, bool synced) {
  if (!t->flag_pending) return;
  if (!synced) {
    const cudaError_t q = cudaEventQuery(t->flag_ev);
    if (q == cudaErrorNotReady) return;
    check_cuda(q, "event query");
  }
  t->flag_pending = false;
  const int f = t->flag_host[0], lab = t->flag_host[1];
  if (f) {
    t->flag_host[0] = t->flag_host[1] = 0;
    try {
      throw_label_flag(f, lab, t->g->h->last_classes);
    } catch (const Err& e) {
      throw Err(e.code, std::string("loss layer: ") + e.what());
    }
  }
}

ck_status ck_trainer_set_graph(ck_trainer* t, int on) {
  if (!t) return CK_ERR_ARG;
  ck_graph* g = t->g;
  CKG_BEGIN(g)
  t->use_graph = on != 0;
  t->drop_graph();
  CKG_END(g)
}

ck_status ck_trainer_set_update_stream(ck_trainer* t, int on) {
  if (!t) return CK_ERR_ARG;
  ck_graph* g = t->g;
  CKG_BEGIN(g)
  t->update_stream = on != 0;
  t->drop_graph();
  CKG_END(g)
}

ck_status ck_trainer_step(ck_trainer* t, float* loss_host, ck_stream stream) {
  if (!t) return CK_ERR_ARG;
  ck_graph* g = t->g;
  CKG_BEGIN(g)
  cudaStream_t s = (cudaStream_t)stream;
  check_step_flag(t, false);  // a previous step's label error surfaces here at the latest
  int64_t before = g->h->counter.n, before_tc = g->h->counter.tc;
  // Replay is valid only while every workspace the captured kernels point
  // into is where it was at capture time (Workspace::get/release bump the
  // generation): otherwise drop the graphs and run eagerly, which re-sizes
  // the workspaces; the next step captures again.
  const uint64_t gen = workspace_generation();
  bool replay = t->use_graph && s != nullptr && !g->profiling && !g->h->prof.on &&
                t->eager_steps > 0 && t->eager_gen == gen;
  ck_trainer::Captured* cap = nullptr;
  if (replay) {
    std::vector<float*> inputs;
    for (auto& v : g->vars)
      if (v.role == 0) inputs.push_back(v.value);
    for (auto& c : t->graphs)
      if (c.stream == s && c.inputs == inputs) cap = &c;
    if (cap && cap->gen != gen) {
      t->drop_graph();
      cap = nullptr;
    }
    if (!cap) {
      // (the legacy default stream cannot be captured: such steps stay eager)
      if (t->graphs.size() >= 4) t->drop_graph();
      cudaGraph_t graph;
      check_cuda(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
      try {
        trainer_body(t, s);
      } catch (...) {
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      check_cuda(cudaStreamEndCapture(s, &graph), "end capture");
      cudaGraphExec_t exec = nullptr;
      const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      check_cuda(e, "graph instantiate");
      if (workspace_generation() != gen) {
        // something moved during capture: this graph is not replayable
        cudaGraphExecDestroy(exec);
        throw Err(CK_ERR_CUDA, "workspace reallocated during step capture");
      }
      t->graphs.push_back({s, inputs, exec, g->h->counter.n - before,
                           g->h->counter.tc - before_tc, gen});
      cap = &t->graphs.back();
    } else {
      // a replay launches the captured kernels again: count them
      g->h->counter.n += cap->launches;
      g->h->counter.tc += cap->tc_launches;
    }
    check_cuda(cudaGraphLaunch(cap->exec, s), "graph launch");
  } else {
    trainer_body(t, s);
    ++t->eager_steps;
    t->eager_gen = workspace_generation();
  }
  check_cuda(cudaEventRecord(t->flag_ev, s), "event");
  t->flag_pending = true;
  if (loss_host) {
    check_cuda(cudaMemcpyAsync(loss_host, t->loss_dev, sizeof(float), cudaMemcpyDeviceToHost, s),
               "copy");
    check_cuda(cudaStreamSynchronize(s), "synchronize");
    check_step_flag(t, true);
  }
  g->last_launches = g->h->counter.n - before;
  CKG_END(g)
}

// Timing of the last profiled (eager) step: forward and backward on the
// compute stream, and how long after the backward's last kernel the gradient
// exchange + update finished (the communication NOT hidden behind backward).
ck_status ck_trainer_last_timing(ck_trainer* t, float* fwd_ms, float* bwd_ms, float* tail_ms) {
  if (!t) return CK_ERR_ARG;
  ck_graph* g = t->g;
  CKG_BEGIN(g)
  if (!t->timed) throw Err(CK_ERR_ARG, "no profiled step (ck_graph_set_profiling) has run");
  check_cuda(cudaEventSynchronize(t->t_comm), "synchronize");
  float a = 0, b = 0, c = 0;
  check_cuda(cudaEventElapsedTime(&a, t->t_begin, t->t_fwd), "elapsed");
  check_cuda(cudaEventElapsedTime(&b, t->t_fwd, t->t_bwd), "elapsed");
  check_cuda(cudaEventElapsedTime(&c, t->t_bwd, t->t_comm), "elapsed");
  if (fwd_ms) *fwd_ms = a;
  if (bwd_ms) *bwd_ms = b;
  if (tail_ms) *tail_ms = c;
  CKG_END(g)
}

int64_t ck_trainer_allreduce_count(const ck_trainer* t) { return t ? t->allreduces : 0; }

}  // extern "C"

namespace ck {

// ---- model files: manifest + blobs, checkpoints ----
//
// A model directory holds `manifest.txt` -- line-oriented key/value text:
//   ck-manifest 1
//   var <name> input|param <H> <W> <C> <N>       (declaration order)
//   layer <kind> <name> in=<a,b,..> out=<c,..> p=<v1,v2,..>
//   blob <param> <file>                           (one per parameter)
//   meta <key> <value...>                         (e.g. normalization data)
// -- and one raw tensor blob (blob.cpp:29-79) per parameter.  Hyper-
// parameters are printed with %.17g so a save -> load -> save round trip
// is byte-identical.

static std::string join_names(const ck_graph* g, const std::vector<int>& ids) {
  std::string s;
  for (size_t k = 0; k < ids.size(); ++k) s += (k ? "," : "") + g->vars[ids[k]].name;
  return s;
}

static std::string path_join(const std::string& dir, const std::string& f) {
  return dir.empty() || dir.back() == '/' ? dir + f : dir + "/" + f;
}

static void make_dir(const std::string& dir) {
  if (mkdir(dir.c_str(), 0755) != 0 && errno != EEXIST)
    throw IoError("cannot create directory " + dir);
}

static void save_params(ck_graph* g, const std::string& dir, std::string* manifest) {
  for (int i : g->decl) {
    const Var& v = g->vars[i];
    if (v.role != 1) continue;
    std::vector<float> host((size_t)elems(v.shape));
    check_cuda(cudaMemcpy(host.data(), v.value, sizeof(float) * host.size(), cudaMemcpyDeviceToHost),
               "copy");
    const std::string file = v.name + ".blob";
    blob_write(path_join(dir, file), host.data(), v.shape);
    if (manifest) *manifest += "blob " + v.name + " " + file + "\n";
  }
}

static std::string manifest_text(const ck_graph* g) {
  std::string m = "ck-manifest 1\n";
  char buf[64];
  for (int i : g->decl) {
    const Var& v = g->vars[i];
    snprintf(buf, sizeof(buf), " %" PRId64 " %" PRId64 " %" PRId64 " %" PRId64 "\n", v.shape.h,
             v.shape.w, v.shape.c, v.shape.n);
    m += "var " + v.name + (v.role == 0 ? " input" : " param") + buf;
  }
  for (const Layer& l : g->layers) {
    m += std::string("layer ") + kind_name(l.kind) + " " + l.name + " in=" + join_names(g, l.in) +
         " out=" + join_names(g, l.out) + " p=";
    for (size_t k = 0; k < l.p.size(); ++k) {
      snprintf(buf, sizeof(buf), "%s%.17g", k ? "," : "", l.p[k]);
      m += buf;
    }
    m += "\n";
  }
  return m;
}

static std::vector<std::string> split_ws(const std::string& line) {
  std::vector<std::string> out;
  std::stringstream ss(line);
  std::string t;
  while (ss >> t) out.push_back(t);
  return out;
}

}  // namespace ck

extern "C" {

ck_status ck_graph_set_meta(ck_graph* g, const char* key, const char* value) {
  CKG_BEGIN(g)
  if (!key || !*key || !value) throw Err(CK_ERR_ARG, "null metadata");
  for (const char* c = key; *c; ++c)
    if (*c == ' ' || *c == '\n') throw Err(CK_ERR_ARG, "metadata key contains a separator");
  if (std::strchr(value, '\n')) throw Err(CK_ERR_ARG, "metadata value contains a newline");
  for (auto& kv : g->meta)
    if (kv.first == key) {
      kv.second = value;
      return CK_OK;
    }
  g->meta.push_back({key, value});
  CKG_END(g)
}

const char* ck_graph_get_meta(const ck_graph* g, const char* key) {
  if (!g || !key) return nullptr;
  for (auto& kv : g->meta)
    if (kv.first == key) return kv.second.c_str();
  return nullptr;
}

ck_status ck_graph_save(ck_graph* g, const char* dir) {
  CKG_BEGIN(g)
  if (!g->finalized) throw Err(CK_ERR_ARG, "save needs a finalized graph");
  if (!dir) throw Err(CK_ERR_ARG, "null path");
  try {
    make_dir(dir);
    std::string m = manifest_text(g);
    check_cuda(cudaDeviceSynchronize(), "synchronize");
    save_params(g, dir, &m);
    for (auto& kv : g->meta) m += "meta " + kv.first + " " + kv.second + "\n";
    std::ofstream f(path_join(dir, "manifest.txt"), std::ios::binary);
    f << m;
    if (!f) throw IoError(std::string("cannot write ") + path_join(dir, "manifest.txt"));
  } catch (const IoError& e) {
    throw Err(CK_ERR_DATA, e.what());
  }
  CKG_END(g)
}

// Builds, finalizes and fills a graph from a model directory.
ck_status ck_graph_load(ck_handle* h, const char* dir, ck_math math, ck_graph** out) {
  if (!h || !out) return CK_ERR_ARG;
  *out = nullptr;
  ck_graph* g = nullptr;
  if (ck_graph_create(h, &g) != CK_OK) return CK_ERR_ARG;
  std::unique_ptr<ck_graph, void (*)(ck_graph*)> guard(g, ck_graph_destroy);
  const ck_status st = [&]() -> ck_status {
    CKG_BEGIN(g)
    if (!dir) throw Err(CK_ERR_ARG, "null path");
    const std::string mpath = path_join(dir, "manifest.txt");
    std::ifstream f(mpath);
    if (!f) throw Err(CK_ERR_DATA, "cannot open " + mpath);
    std::string line;
    if (!std::getline(f, line)) throw Err(CK_ERR_DATA, "empty manifest " + mpath);
    const auto head = split_ws(line);
    if (head.size() != 2 || head[0] != "ck-manifest")
      throw Err(CK_ERR_DATA, "not a ck model manifest: " + mpath);
    if (head[1] != "1") throw Err(CK_ERR_DATA, "manifest version " + head[1] + " not supported");
    std::vector<std::pair<std::string, std::string>> blobs;
    int lineno = 1;
    while (std::getline(f, line)) {
      ++lineno;
      if (line.empty() || line[0] == '#') continue;
      const auto t = split_ws(line);
      const std::string where = mpath + ":" + std::to_string(lineno);
      if (t[0] == "var" && t.size() == 7) {
        ck_shape sh{std::stoll(t[3]), std::stoll(t[4]), std::stoll(t[5]), std::stoll(t[6])};
        ck_status r = t[2] == "input" ? ck_graph_add_input(g, t[1].c_str(), sh)
                      : t[2] == "param" ? ck_graph_add_param(g, t[1].c_str(), sh)
                                        : CK_ERR_DATA;
        if (r != CK_OK) throw Err(r, where + ": " + (g->h->err.empty() ? "bad role" : g->h->err));
      } else if (t[0] == "layer" && t.size() == 6 && t[3].rfind("in=", 0) == 0 &&
                 t[4].rfind("out=", 0) == 0 && t[5].rfind("p=", 0) == 0) {
        std::vector<double> p;
        for (auto& v : split_csv(t[5].c_str() + 2)) p.push_back(std::stod(v));
        ck_status r = ck_graph_add_layer(g, t[1].c_str(), t[2].c_str(), t[3].c_str() + 3,
                                         t[4].c_str() + 4, p.data(), (int)p.size());
        if (r != CK_OK) throw Err(r, where + ": " + g->h->err);
      } else if (t[0] == "blob" && t.size() == 3) {
        blobs.push_back({t[1], t[2]});
      } else if (t[0] == "meta" && t.size() >= 2) {
        const size_t at = line.find(t[1]) + t[1].size();
        g->meta.push_back({t[1], at < line.size() ? line.substr(at + 1) : std::string()});
      } else {
        throw Err(CK_ERR_DATA, where + ": malformed line '" + line + "'");
      }
    }
    if (ck_graph_finalize(g, math) != CK_OK) throw Err(CK_ERR_DATA, g->h->err);
    for (int i : g->decl) {
      const Var& v = g->vars[i];
      if (v.role != 1) continue;
      bool found = false;
      for (auto& b : blobs) found |= b.first == v.name;
      if (!found) throw Err(CK_ERR_DATA, "manifest lists no blob for parameter '" + v.name + "'");
    }
    for (auto& b : blobs) {
      Var& v = g->vars[g->var(b.first)];
      if (v.role != 1) throw Err(CK_ERR_DATA, "blob for non-parameter '" + b.first + "'");
      const std::string bp = path_join(dir, b.second);
      FILE* probe = fopen(bp.c_str(), "rb");
      if (!probe) throw Err(CK_ERR_DATA, "manifest references missing blob '" + b.second + "'");
      fclose(probe);
      std::vector<float> host((size_t)elems(v.shape));
      try {
        blob_read(bp, host.data(), &v.shape);
      } catch (const IoError& e) {
        throw Err(CK_ERR_DATA, e.what());
      }
      check_cuda(cudaMemcpy(v.value, host.data(), sizeof(float) * host.size(),
                            cudaMemcpyHostToDevice), "copy");
    }
    CKG_END(g)
  }();
  if (st != CK_OK) {
    h->err = g->h->err;
    return st;
  }
  *out = guard.release();
  return CK_OK;
}

// cnn_train checkpoint: the model directory plus every
// momentum buffer (<param>.momentum.blob) and trainer.txt with the step
// hyper-parameters, the epoch and the shuffling generator's state
// (rng.hpp:31-32), so resuming reproduces straight-through training bitwise.
ck_status ck_trainer_save(ck_trainer* t, const char* dir, const uint64_t rng_state[4],
                          int64_t epoch) {
  if (!t) return CK_ERR_ARG;
  ck_graph* g = t->g;
  ck_status st = ck_graph_save(g, dir);
  if (st != CK_OK) return st;
  CKG_BEGIN(g)
  try {
    for (size_t k = 0; k < t->params.size(); ++k) {
      const Var& v = g->vars[t->params[k]];
      std::vector<float> host((size_t)elems(v.shape));
      check_cuda(cudaMemcpy(host.data(), t->mom[k], sizeof(float) * host.size(),
                            cudaMemcpyDeviceToHost), "copy");
      blob_write(path_join(dir, v.name + ".momentum.blob"), host.data(), v.shape);
    }
    std::ofstream f(path_join(dir, "trainer.txt"), std::ios::binary);
    char buf[256];
    snprintf(buf, sizeof(buf),
             "ck-trainer 1\nlr %.9g\nmomentum %.9g\nweight_decay %.9g\nepoch %" PRId64
             "\nrng %016" PRIx64 " %016" PRIx64 " %016" PRIx64 " %016" PRIx64 "\n",
             (double)t->lr, (double)t->momentum, (double)t->wd, epoch,
             rng_state ? rng_state[0] : 0, rng_state ? rng_state[1] : 0,
             rng_state ? rng_state[2] : 0, rng_state ? rng_state[3] : 0);
    f << buf;
    if (!f) throw IoError("cannot write " + path_join(dir, "trainer.txt"));
  } catch (const IoError& e) {
    throw Err(CK_ERR_DATA, e.what());
  }
  CKG_END(g)
}

// Restores parameters, momentum, epoch and generator state into a trainer
// over the same graph structure.
ck_status ck_trainer_load(ck_trainer* t, const char* dir, uint64_t rng_state[4],
                          int64_t* epoch) {
  if (!t) return CK_ERR_ARG;
  ck_graph* g = t->g;
  CKG_BEGIN(g)
  if (!dir) throw Err(CK_ERR_ARG, "null path");
  check_cuda(cudaDeviceSynchronize(), "synchronize");
  try {
    for (size_t k = 0; k < t->params.size(); ++k) {
      Var& v = g->vars[t->params[k]];
      std::vector<float> host((size_t)elems(v.shape));
      blob_read(path_join(dir, v.name + ".blob"), host.data(), &v.shape);
      check_cuda(cudaMemcpy(v.value, host.data(), sizeof(float) * host.size(),
                            cudaMemcpyHostToDevice), "copy");
      blob_read(path_join(dir, v.name + ".momentum.blob"), host.data(), &v.shape);
      check_cuda(cudaMemcpy(t->mom[k], host.data(), sizeof(float) * host.size(),
                            cudaMemcpyHostToDevice), "copy");
    }
    std::ifstream f(path_join(dir, "trainer.txt"));
    if (!f) throw IoError("cannot open " + path_join(dir, "trainer.txt"));
    std::string line;
    std::getline(f, line);
    if (line != "ck-trainer 1") throw IoError(std::string("not a ck trainer checkpoint: ") + dir);
    while (std::getline(f, line)) {
      const auto tk = split_ws(line);
      if (tk.size() == 2 && tk[0] == "epoch" && epoch) *epoch = std::stoll(tk[1]);
      if (tk.size() == 5 && tk[0] == "rng" && rng_state)
        for (int k = 0; k < 4; ++k) rng_state[k] = std::stoull(tk[1 + k], nullptr, 16);
    }
  } catch (const IoError& e) {
    throw Err(CK_ERR_DATA, e.what());
  }
  CKG_END(g)
}

}  // extern "C"
