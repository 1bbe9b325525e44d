/*
 * ck.h -- C ABI of the B200-native MatConvNet block library (libck.so).
 *
 * This is the drop-in boundary for the reference's computational-block hot
 * path.  The reference (convkit, /root/reference/proj) declares the block API
 * as C++ templates in namespace convkit and intends a shared C ABI over it
 * (proj/src/CMakeLists.txt:25-28, capi.cpp -- source absent, symbol set
 * unknown).  Every entry point below replaces the reference function named in
 * its comment, with the same argument meaning, the same validation rules and
 * the same error messages; the differences are the ones a device library
 * needs:
 *
 *   - tensors are DEVICE pointers in the reference layout: dense HWCN fp32,
 *     flat index i + H*(j + W*(c + C*n))   (tensor.hpp:70-72);
 *   - outputs are caller-allocated and shape-checked (the reference returns
 *     new tensors); a NULL output means "skip", as in conv.hpp:64-65;
 *   - `accumulate` != 0 makes a backward output add into the destination
 *     (the graph engine's derivs[in] += d, graph.cpp:587-596, fused);
 *   - C++ exceptions become status codes (error.hpp:9-24), the message is
 *     kept per handle (ck_last_error);
 *   - every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and validates all arguments on the host before launch.
 *
 * `math` selects the convolution "method" (the reference's cuDNN switch,
 * PAPER.md:112): CK_MATH_TF32 runs the tcgen05 tensor-core kernels,
 * CK_MATH_FP32 the exact-FP32 verification kernels.
 *
 * Threading: one handle per host thread; a handle owns its workspace and is
 * bound to one device.  There is no global mutable state.
 */
#ifndef CK_CK_H
#define CK_CK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ck_status {
  CK_OK = 0,
  CK_ERR_SHAPE = 1,   /* convkit::ShapeError   (error.hpp:9-13)  */
  CK_ERR_DATA = 2,    /* convkit::DataError    (error.hpp:15-19) */
  CK_ERR_NUMERIC = 3, /* convkit::NumericError (error.hpp:21-24) */
  CK_ERR_CUDA = 4,    /* a CUDA runtime / driver / NCCL failure  */
  CK_ERR_ARG = 5      /* NULL handle, bad enum, oversize tensor  */
} ck_status;

typedef enum ck_math { CK_MATH_TF32 = 0, CK_MATH_FP32 = 1 } ck_math;

/* convkit::Shape (tensor.hpp:13-32) */
typedef struct ck_shape {
  int64_t h, w, c, n;
} ck_shape;

/* A device tensor view: HWCN fp32, H fastest. */
typedef struct ck_tensor {
  float* data;
  ck_shape shape;
} ck_tensor;

/* convkit::ConvGeom (conv.hpp:9-17) */
typedef struct ck_conv_geom {
  int64_t stride_h, stride_w, pad_top, pad_bottom, pad_left, pad_right, groups;
} ck_conv_geom;

/* convkit::ConvTransposeGeom (conv.hpp:21-28) */
typedef struct ck_convt_geom {
  int64_t up_h, up_w, crop_top, crop_bottom, crop_left, crop_right;
} ck_convt_geom;

/* convkit::PoolMode / PoolGeom (pool.hpp:7-23) */
typedef enum ck_pool_mode { CK_POOL_MAX = 0, CK_POOL_AVG = 1 } ck_pool_mode;
typedef struct ck_pool_geom {
  int64_t window_h, window_w, stride_h, stride_w, pad_top, pad_bottom, pad_left, pad_right;
  int64_t mode; /* ck_pool_mode */
} ck_pool_geom;

/* convkit::LrnParams (normalize.hpp:11-16) */
typedef struct ck_lrn_params {
  int64_t group_size;
  double kappa, alpha, beta;
} ck_lrn_params;

typedef struct ck_handle ck_handle;
typedef void* ck_stream; /* cudaStream_t */

/* ---- handle ------------------------------------------------------------ */
ck_status ck_create(ck_handle** out, int device);
void ck_destroy(ck_handle* h);
const char* ck_last_error(const ck_handle* h);
const char* ck_version(void);
/* Number of kernels this handle launched since creation (bench evidence). */
int64_t ck_launch_count(const ck_handle* h);
/* Of those, launches of the tcgen05 tensor-core GEMM (tc_gemm_kernel): lets a
 * caller assert that a TF32 call really ran on the tensor cores. */
int64_t ck_tc_launch_count(const ck_handle* h);
/* Per-launch timing of the tensor-core GEMM kernels (bench roofline): while
 * on, every GEMM launch is bracketed by CUDA events on its stream and recorded
 * with a label and its algorithmic FLOP count (2*N*OH*OW*K*fh*fw*C/groups).
 * ck_kernel_profile_get synchronises the record's end event. */
ck_status ck_set_kernel_profiling(ck_handle* h, int on);
int ck_kernel_profile_count(const ck_handle* h);
ck_status ck_kernel_profile_get(ck_handle* h, int i, const char** label, float* ms,
                                double* flops);
ck_status ck_kernel_profile_clear(ck_handle* h);
/* Stream-ordered copy between any host / device pointers (UVA). */
ck_status ck_memcpy(ck_handle* h, void* dst, const void* src, int64_t bytes, ck_stream stream);

/* ---- shape laws --------------------------------------------------------- */
/* conv.cpp:108-135 conv_output_shape */
ck_status ck_conv_output_shape(ck_handle* h, ck_shape x, ck_shape f, const ck_conv_geom* g,
                               ck_shape* out);
/* conv.cpp:137-154 convt_output_shape */
ck_status ck_convt_output_shape(ck_handle* h, ck_shape x, ck_shape f, const ck_convt_geom* g,
                                ck_shape* out);
/* pool.cpp:35-46 pool_output_shape */
ck_status ck_pool_output_shape(ck_handle* h, ck_shape x, const ck_pool_geom* g, ck_shape* out);

/* ---- vl_nnconv: conv.hpp:60-69, conv.cpp:193-280 ----------------------- */
ck_status ck_conv_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                          const ck_tensor* bias /* NULL: no bias */, const ck_conv_geom* g,
                          ck_tensor* y, ck_math math, ck_stream stream);
ck_status ck_conv_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                           const ck_conv_geom* g, const ck_tensor* dy, ck_tensor* dx,
                           ck_tensor* df, ck_tensor* db, int accumulate, ck_math math,
                           ck_stream stream);

/* ---- vl_nnconvt: conv.hpp:74-81, conv.cpp:283-365 ----------------------- */
ck_status ck_convt_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                           const ck_convt_geom* g, ck_tensor* y, ck_math math, ck_stream stream);
ck_status ck_convt_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* f,
                            const ck_convt_geom* g, const ck_tensor* dy, ck_tensor* dx,
                            ck_tensor* df, int accumulate, ck_math math, ck_stream stream);

/* ---- vl_nnpool: pool.hpp:27-34, pool.cpp:49-126 ------------------------- */
ck_status ck_pool_forward(ck_handle* h, const ck_tensor* x, const ck_pool_geom* g, ck_tensor* y,
                          ck_stream stream);
ck_status ck_pool_backward(ck_handle* h, const ck_tensor* x, const ck_pool_geom* g,
                           const ck_tensor* dy, ck_tensor* dx, int accumulate, ck_stream stream);

/* ---- vl_nnrelu: activation.hpp:7-12, activation.cpp:8-22 ---------------- */
ck_status ck_relu_forward(ck_handle* h, const ck_tensor* x, ck_tensor* y, ck_stream stream);
ck_status ck_relu_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* dy, ck_tensor* dx,
                           int accumulate, ck_stream stream);

/* ---- vl_nnnormalize (LRN): normalize.hpp:18-23, normalize.cpp:47-118 ---- */
ck_status ck_lrn_forward(ck_handle* h, const ck_tensor* x, const ck_lrn_params* p, ck_tensor* y,
                         ck_stream stream);
ck_status ck_lrn_backward(ck_handle* h, const ck_tensor* x, const ck_lrn_params* p,
                          const ck_tensor* dy, ck_tensor* dx, int accumulate, ck_stream stream);

/* ---- vl_nnbnorm: normalize.hpp:35-49, normalize.cpp:189-265 ------------- */
/* moments: optional K x 2 tensor (mean column then variance column), the
 * tape.aux layout of graph.cpp:259-266. */
ck_status ck_bnorm_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* w,
                           const ck_tensor* b, double epsilon, ck_tensor* y,
                           ck_tensor* moments, ck_stream stream);
ck_status ck_bnorm_infer(ck_handle* h, const ck_tensor* x, const ck_tensor* w, const ck_tensor* b,
                         double epsilon, const ck_tensor* moments, ck_tensor* y,
                         ck_stream stream);
ck_status ck_bnorm_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* w,
                            const ck_tensor* b, double epsilon, const ck_tensor* dy,
                            ck_tensor* dx, ck_tensor* dw, ck_tensor* db, int accumulate,
                            ck_stream stream);

/* ---- vl_nnsoftmaxloss: loss.hpp:39-49, kind softmaxlog ----------------- */
/* loss: DEVICE scalar receiving sum_sites w * l (loss.cpp:156-165, :182).
 * check_labels != 0 synchronises `stream` and reports malformed labels as
 * CK_ERR_DATA with the reference's message (loss.cpp:14-18, :101-106);
 * otherwise a bad label is recorded on the handle and reported by the next
 * ck_check_labels(). */
ck_status ck_softmaxlog_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                                const ck_tensor* weights /* NULL: all ones */, float* loss,
                                int check_labels, ck_stream stream);
/* dx = p * w * (softmax - onehot)   (loss.cpp:263-275) */
ck_status ck_softmaxlog_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                                 const ck_tensor* weights, float p, ck_tensor* dx,
                                 int accumulate, ck_stream stream);
/* The cnn_train metrics: classerror (loss.cpp:111-141, lowest index wins
 * ties) and topk (loss.cpp:142-149), weighted sums into DEVICE scalars. */
ck_status ck_loss_metrics(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                          const ck_tensor* weights, int64_t top_k, float* top1_err,
                          float* topk_err, ck_stream stream);
ck_status ck_check_labels(ck_handle* h, ck_stream stream);

/* ---- the rest of the reference block set -------------------------------- */
/* activation.cpp:25-38 sigmoid_forward */
ck_status ck_sigmoid_forward(ck_handle* h, const ck_tensor* x, ck_tensor* y, ck_stream stream);
/* activation.cpp:41-48 sigmoid_backward: consumes the forward OUTPUT y */
ck_status ck_sigmoid_backward(ck_handle* h, const ck_tensor* y, const ck_tensor* dy, ck_tensor* dx,
                              int accumulate, ck_stream stream);
/* normalize.cpp:309-328 softmax_forward: channel softmax per site */
ck_status ck_softmax_forward(ck_handle* h, const ck_tensor* x, ck_tensor* y, ck_stream stream);
/* normalize.cpp:330-347 softmax_backward: consumes the forward OUTPUT y */
ck_status ck_softmax_backward(ck_handle* h, const ck_tensor* y, const ck_tensor* dy, ck_tensor* dx,
                              int accumulate, ck_stream stream);

/* convkit::SpnormParams (normalize.hpp:59-64) */
typedef struct ck_spnorm_params {
  int64_t window_h, window_w;
  double alpha, beta;
} ck_spnorm_params;
/* normalize.cpp:268-281 spnorm_forward */
ck_status ck_spnorm_forward(ck_handle* h, const ck_tensor* x, const ck_spnorm_params* p,
                            ck_tensor* y, ck_stream stream);
/* normalize.cpp:284-306 spnorm_backward */
ck_status ck_spnorm_backward(ck_handle* h, const ck_tensor* x, const ck_spnorm_params* p,
                             const ck_tensor* dy, ck_tensor* dx, int accumulate, ck_stream stream);

/* bilinear.cpp:48-51 bilinear_output_shape (grid is 2 x outH x outW x N) */
ck_status ck_bilinear_output_shape(ck_handle* h, ck_shape x, ck_shape grid, ck_shape* out);
/* bilinear.cpp:58-89 bilinear_forward */
ck_status ck_bilinear_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* grid,
                              ck_tensor* y, ck_stream stream);
/* bilinear.cpp:92-132 bilinear_backward (dx or dgrid may be NULL = skip) */
ck_status ck_bilinear_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* grid,
                               const ck_tensor* dy, ck_tensor* dx, ck_tensor* dgrid,
                               int accumulate, ck_stream stream);

/* loss.cpp:346-371 pdist_forward: y is H x W x 1 x N */
ck_status ck_pdist_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* target, double p,
                           int no_root, ck_tensor* y, ck_stream stream);
/* loss.cpp:374-428 pdist_backward (dx or dtarget may be NULL; dtarget = -dx) */
ck_status ck_pdist_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* target, double p,
                            int no_root, const ck_tensor* dy, ck_tensor* dx, ck_tensor* dtarget,
                            int accumulate, ck_stream stream);

/* convkit::LossKind (loss.hpp:13-24), same order */
typedef enum ck_loss_kind {
  CK_LOSS_CLASSERROR = 0,
  CK_LOSS_TOPK = 1,
  CK_LOSS_LOG = 2,
  CK_LOSS_SOFTMAXLOG = 3,
  CK_LOSS_MHINGE = 4,
  CK_LOSS_MSHINGE = 5,
  CK_LOSS_BINARYERROR = 6,
  CK_LOSS_BINARYLOG = 7,
  CK_LOSS_LOGISTIC = 8,
  CK_LOSS_HINGE = 9
} ck_loss_kind;
/* convkit::LossOptions (loss.hpp:31-36) */
typedef struct ck_loss_options {
  int64_t top_k;       /* topk (default 5) */
  double threshold;    /* binaryerror (default 0) */
  int64_t random_ties; /* classerror: break argmax ties randomly */
  uint64_t tie_seed;
} ck_loss_options;
/* loss.cpp:86-228 loss_forward, any kind: the weighted SUM of per-sample
 * penalties into *loss (a DEVICE float).  check_labels != 0 synchronises and
 * reports DataError conditions (non-integer / out-of-range labels, log loss
 * on a non-positive score, binarylog input outside [0,1]).  opts may be NULL
 * (defaults). */
ck_status ck_loss_forward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                          const ck_tensor* weights, ck_loss_kind kind, const ck_loss_options* opts,
                          float* loss, int check_labels, ck_stream stream);
/* loss.cpp:231-343 loss_backward, any kind (error kinds give exact zeros) */
ck_status ck_loss_backward(ck_handle* h, const ck_tensor* x, const ck_tensor* labels,
                           const ck_tensor* weights, ck_loss_kind kind, const ck_loss_options* opts,
                           float p, ck_tensor* dx, int accumulate, ck_stream stream);

/* ---- cnn_train SGD step: v = m v - lr (g + wd w); w += v -- */
ck_status ck_sgd_step(ck_handle* h, float* w, float* v, const float* g, int64_t n, float lr,
                      float momentum, float weight_decay, ck_stream stream);

/* ---- DAG engine (graph.hpp:93-190, graph.cpp:494-598) -------------------- */
typedef struct ck_graph ck_graph;
ck_status ck_graph_create(ck_handle* h, ck_graph** out);
void ck_graph_destroy(ck_graph* g);
/* graph.hpp:96-98 add_input / add_param / add_layer.  `kind` is a
 * layer_kind_name (graph.cpp:13-31); params by kind:
 *   conv  : stride_h stride_w pad_t pad_b pad_l pad_r groups
 *   convt : up_h up_w crop_t crop_b crop_l crop_r
 *   pool  : win_h win_w stride_h stride_w pad_t pad_b pad_l pad_r mode
 *   lrn   : group_size kappa alpha beta
 *   bnorm : epsilon
 *   loss  : [kind top_k threshold random_ties tie_seed] (none: softmaxlog)
 *   spnorm: win_h win_w alpha beta
 *   pdist : p no_root
 *   split : (outputs name the copies)
 *   sigmoid, softmax, relu, sum, bilinear(x, grid): none                 */
ck_status ck_graph_add_input(ck_graph* g, const char* name, ck_shape shape);
ck_status ck_graph_add_param(ck_graph* g, const char* name, ck_shape shape);
ck_status ck_graph_add_layer(ck_graph* g, const char* kind, const char* name,
                             const char* inputs_csv, const char* outputs_csv,
                             const double* params, int nparams);
/* graph.hpp:102 finalize: validates, orders, infers shapes, allocates. */
ck_status ck_graph_finalize(ck_graph* g, ck_math math);
/* Device view of a variable's value (deriv == 0) or derivative (deriv != 0). */
ck_status ck_graph_var(ck_graph* g, const char* name, int deriv, ck_tensor* out);

/* Bind an input variable to caller-owned device memory (elements x 4 bytes,
 * valid while bound; NULL restores the engine's own buffer).  A trainer step
 * replays one captured CUDA graph per set of input bindings, so a caller can
 * alternate two input buffers -- filling one while the step reads the other --
 * with no device-to-device copy (graph.Feeder).  Not a reference entry point. */
ck_status ck_graph_bind_input(ck_graph* g, const char* name, float* data);
/* graph.cpp:494 forward (train mode) */
ck_status ck_graph_forward(ck_graph* g, ck_stream stream);
/* graph.cpp:548 backward with seed d(objective) = 1 */
ck_status ck_graph_backward(ck_graph* g, const char* objective, ck_stream stream);
/* Number of kernels the last forward+backward launched. */
int64_t ck_graph_last_launches(const ck_graph* g);
/* Per-layer CUDA-event timing (on the evaluation stream).  When enabled,
 * every layer's forward and backward is bracketed by events; read the last
 * evaluation's times (ms) after synchronising.  Layers are indexed in
 * declaration order. */
ck_status ck_graph_set_profiling(ck_graph* g, int enable);
int ck_graph_layer_count(const ck_graph* g);
const char* ck_graph_layer_name(const ck_graph* g, int layer);
ck_status ck_graph_layer_ms(ck_graph* g, int layer, float* fwd_ms, float* bwd_ms);
/* Engine options (not reference entry points):
 *   "lrn_grid" (default 1): a TF32 conv -> relu -> lrn chain's LRN backward
 *   writes the conv's ReLU-gated dy grid directly (0: the unfused blocks);
 *   "lrn_pool" (default 0): an lrn -> 3x3/2 max pool pair runs as one kernel
 *   (the pool reads the LRN values from shared memory, not HBM; bit-identical,
 *   measured slower than the two tuned kernels on AlexNet);
 *   "producer_grid" (default 1): a TF32 conv -> relu -> conv forward writes the
 *   second conv's padded x grid from the first conv's epilogue;
 *   "dgrad_grid" (default 1): a TF32 conv -> relu -> conv backward writes the
 *   first conv's ReLU-gated dy grid (and bias partials) from the second conv's
 *   data-gradient epilogue;
 *   "bn_grid" (default 1): a TF32 conv -> bnorm backward writes the conv's dy
 *   grid (and bias partials) from the bnorm backward;
 *   "bn_lazy_y" (default 1): a fused bnorm -> relu forward stores only relu(y).
 * Intermediates these options leave unstored are computed on request
 * (ck_graph_var). */
ck_status ck_graph_set_option(ck_graph* g, const char* name, int64_t value);

/* ---- cnn_train training step with multi-GPU data parallelism ------------ */
typedef struct ck_trainer ck_trainer;
ck_status ck_nccl_unique_id(char out[128]);
ck_status ck_trainer_create(ck_graph* g, const char* objective, float lr, float momentum,
                            float weight_decay, ck_trainer** out);
void ck_trainer_destroy(ck_trainer* t);
/* Join an NCCL data-parallel group (one process per GPU). */
ck_status ck_trainer_init_dp(ck_trainer* t, const char id[128], int rank, int world);
/* forward + backward + gradient allreduce (overlapped) + SGD on `stream`.
 * If loss_host != NULL the step's objective is copied back (synchronising).
 * A label error (CK_ERR_DATA) or a non-finite objective (CK_ERR_NUMERIC,
 * SPEC.md:716 "NaN loss aborts") of a step is reported by that call when it
 * synchronises, else by the next call once the step is complete. */
ck_status ck_trainer_step(ck_trainer* t, float* loss_host, ck_stream stream);
/* Replay each step as one CUDA graph: captured on the first graph step after
 * an eager one (same stream; profiling steps stay eager).  A captured step is
 * dropped and re-captured (after one eager step) whenever any workspace it
 * points into was reallocated since, e.g. by a larger call on the handle. */
ck_status ck_trainer_set_graph(ck_trainer* t, int on);
/* Single GPU: run each layer's SGD on a side stream as soon as its
 * derivatives are final (default 1), or in line on the step's stream (0). */
ck_status ck_trainer_set_update_stream(ck_trainer* t, int on);
/* Timing of the last profiled step (ck_graph_set_profiling on; such steps
 * run eagerly): forward, backward, and the time from the end of backward to
 * the completion of the last gradient allreduce + update (the exchange NOT
 * hidden behind backward). */
ck_status ck_trainer_last_timing(ck_trainer* t, float* fwd_ms, float* bwd_ms, float* tail_ms);
/* NCCL allreduce groups issued by eager / captured steps (DP evidence). */
int64_t ck_trainer_allreduce_count(const ck_trainer* t);

/* ---- files (host only; errors in ck_io_last_error()) -------------------- */
/* blob.cpp:29-79 / SPEC.md:87: raw tensor blob -- four u64 little-endian dims
 * (H, W, C, N) then the float32 values, little-endian, H fastest. */
const char* ck_io_last_error(void);
ck_status ck_blob_write(const char* path, const float* host_data, ck_shape shape);
ck_status ck_blob_read_shape(const char* path, ck_shape* shape);
/* reads into host memory; the stored shape must equal `expect` */
ck_status ck_blob_read(const char* path, float* host_data, ck_shape expect);
/* SPEC.md:721-728 load_idx: images -> H x W x 1 x N in [0,1], labels -> 1..C
 * (raw + 1).  out == NULL returns only dims (H, W, C, N). */
ck_status ck_idx_read(const char* path, float* out, int64_t dims[4]);

/* Model directory: manifest.txt (line-oriented
 *   "ck-manifest 1" / "var <name> input|param H W C N" /
 *   "layer <kind> <name> in=<a,..> out=<b,..> p=<v,..>" / "blob <param> <file>" /
 *   "meta <key> <value>") plus one blob per parameter.  Lossless: save ->
 * load -> save is byte-identical.  Load builds and finalizes the graph on h. */
ck_status ck_graph_save(ck_graph* g, const char* dir);
ck_status ck_graph_load(ck_handle* h, const char* dir, ck_math math, ck_graph** out);
/* normalization metadata carried by the manifest */
ck_status ck_graph_set_meta(ck_graph* g, const char* key, const char* value);
const char* ck_graph_get_meta(const ck_graph* g, const char* key);
/* cnn_train checkpoint: the model directory plus the
 * momentum buffers, the epoch and the shuffling generator's state
 * (rng.hpp:31-32); resuming reproduces straight-through training bitwise. */
ck_status ck_trainer_save(ck_trainer* t, const char* dir, const uint64_t rng_state[4],
                          int64_t epoch);
ck_status ck_trainer_load(ck_trainer* t, const char* dir, uint64_t rng_state[4],
                          int64_t* epoch);

/* ---- synthetic data (host): the reference generator, xoshiro256** seeded
 * via splitmix64 (rng.hpp:9-36, rng.cpp:10-59) ---------------------------- */
void* ck_rng_create(uint64_t seed);
void ck_rng_destroy(void* rng);
/* lo + (hi - lo) * uniform()   (oracles.hpp:16-23) */
void ck_rng_uniform(void* rng, float* out, int64_t n, float lo, float hi);
/* scale * normal() (Box-Muller, rng.cpp:42-47; SPEC.md:757 weight init) */
void ck_rng_normal(void* rng, float* out, int64_t n, float scale);
/* 1 + below(classes)   (rng.cpp:49) */
void ck_rng_labels(void* rng, float* out, int64_t n, uint64_t classes);
/* rng.cpp:51-59 permutation(n): Fisher-Yates with below(k + 1) */
void ck_rng_permutation(void* rng, int64_t n, int64_t* out);
/* rng.hpp:31-32 state() / set_state() */
void ck_rng_get_state(const void* rng, uint64_t state[4]);
void ck_rng_set_state(void* rng, const uint64_t state[4]);

#ifdef __cplusplus
}
#endif
#endif /* CK_CK_H */
