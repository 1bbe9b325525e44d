// conv_tc.cu -- the CK_MATH_TF32 convolution path: tcgen05 tensor cores with
// TMEM accumulators, operands staged by TMA (sm_100a).
//
// One warp-specialised GEMM kernel,  C[m, n] = sum_k A[m, k] B[n, k],  serves
// every pass of conv.cpp:193-280:
//
//   pass            A (rows m)                  B (rows n)               K
//   conv fprop      im2col(x) pixels  [TMA im2col, K-major]  filters [tiled]  (tap, c)
//   conv dgrad      im2col(dy) pixels [TMA im2col, K-major]  flipped filters  (tap, k)
//   conv wgrad      dy^T filters      [tiled, MN-major]      im2col(x) [TMA im2col, MN-major]  pixels
//   fc fprop        filters [tiled K] images x [tiled K]                      q = (i, j, c)
//   fc dgrad        filters [tiled MN] dy [tiled K]                           k
//   fc wgrad        x [tiled MN]       dy [tiled MN]                          images
//
// The reference layout HWCN has odd spatial pitches (27, 13, ...) that TMA
// cannot address (global strides must be multiples of 16 bytes), so conv
// operands go through a "pixel-major" layout -- [n][w][h][c], channels
// innermost, padded per group to a multiple of 32 -- produced by a transpose
// kernel; TMA's im2col mode then walks output pixels across image boundaries
// with zero-fill for the padding, which is the reference's im2row
// (conv.cpp:35-59) done by the copy engine with no buffer.  FC layers (the
// H''=W''=1 special case) need no transform at all.
//
// Pipeline (per CTA, one 128 x BN output tile):
//   warp 0     : TMA producer, STAGES-deep ring of (A 16 KB, B BN*128 B) stages
//   warp 1     : TMEM allocator + single-thread tcgen05.mma.kind::tf32 issuer
//   warps 2..5 : epilogue, tcgen05.ld 32x32b -> registers -> global
// Operand tiles are 128-byte swizzled (SWIZZLE_128B) in both K-major and
// MN-major forms; K per stage = 32 fp32, 4 MMAs of K = 8.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>

#include "ck_handle.hpp"
#include "ck_internal.hpp"

namespace ck {

// ============================================================================
//                               device helpers
// ============================================================================
namespace tc {

// Operand kinds.  K-major operands use SWIZZLE_128B rows of 32 k; MN-major
// ones (tf32 allows them only in the SWIZZLE_128B_BASE32B layout,
// tools/mn_probe.cu) rows of 32 m/n per k.
enum OpKind : int {
  OP_TILED_K = 0,     // 2D tensor (K inner, MN outer), box (32, rows)
  OP_IM2COL_K = 2,    // 4D im2col over a pixel-major tensor, box BM px x 32 ch
  OP_SHIFT_K = 4,     // fprop/dgrad A: 3D box {32 ch, BM grid rows + tap shift, KS/32 chunks}
  OP_TILED_K3 = 5,    // B for OP_SHIFT_K: 3D box {32 k, BN rows, KS/32 chunks} of [row][K]
  OP_TILED_MN = 6,    // MN-major 2D tensor [K][MN] (MN inner): 32x32 boxes, SW128_32B atoms
  OP_SHIFT_MN = 8,    // wgrad B: 3D boxes {32 ch, 32 grid rows + tap shift, b_rows/32 blocks}
};

enum EpiKind : int {
  EPI_PIX = 0,     // row m = output pixel (n, ow, oh) of an HWCN tensor, col = channel
  EPI_LINEAR = 1,  // addr = row + col * ld
  EPI_S2D = 2,     // row m = s2d pixel (n, v, u), col c' = (a, b, c) -> x[s*u+a, s*v+b, c]
};

// Debug experiments that drop MMAs / loads / the epilogue exist only in
// CK_EXPERIMENTS builds; a product kernel always does all of its work.
#ifdef CK_EXPERIMENTS
#define TC_EXP(p) ((p).exp)
#define DG_SKIP(p) ((p).dg_skip)
#else
#define TC_EXP(p) 0
#define DG_SKIP(p) 0
#endif

struct GemmParams {
  int M, N, K;            // problem (per group), K in elements (multiple of 32)
  int BN;                 // tile N (multiple of 16, <= 256)
  int stages;
  int splits;             // split-K factor (grid.z = groups * splits)
  // im2col geometry (for OP_IM2COL_*): output pixel decode and origin
  int OH, OW;             // output spatial extent walked by the TMA
  int sh, sw, pt, pl;     // traversal stride and pad (start = o*s - p)
  int fh;                 // taps are t = fi + fh * fj
  int cchunks;            // channel chunks of 32 per tap (Cgp / 32)
  int a_grp_c, b_grp_c;   // per-group channel offset of the im2col tensor (Cgp / Kgp)
  int a_grp_mn, b_grp_mn; // per-group offset along MN for tiled operands
  int a_grp_k, b_grp_k;   // per-group offset along K for tiled operands
  // epilogue
  int epi;
  float* out;
  int64_t ld;             // EPI_LINEAR: column stride; EPI_PIX: OH*OW
  int64_t img_stride;     // EPI_PIX: K_total * OH * OW
  int64_t grp_col;        // column offset per group (EPI_PIX channel / EPI_LINEAR col)
  int64_t grp_out;        // element offset per group (EPI_LINEAR)
  int64_t split_stride;   // elements between split partials (splits > 1)
  int epi_OHW;            // EPI_PIX: pixels per image of the output
  const float* bias;      // per col (EPI_PIX) or per row (EPI_LINEAR)
  int relu, acc;
  float* out2;            // EPI_PIX / EPI_LINEAR (non-partial): also store relu(v) here
  int n_valid;            // columns < n_valid are stored
  int Hp;                 // OP_SHIFT_MN / OP_SHIFT_K: grid pitch (tap shift = fi + Hp*fj)
  int base_shift;         // OP_SHIFT_K: row offset added to every tap shift (dgrad: -(qt+Hp*ql))
  int b_grp_row;          // halo kernel: per-group filter row offset
  int s2d, s2d_U, s2d_H, s2d_W, s2d_C;  // EPI_S2D: factor, grid height, target dims
  int s2d_Ct;             // EPI_S2D with groups: channels per image (s2d_C: per group; 0: = s2d_C)
  int exp;                // debug experiments (CK_TC_EXP)
  int snake;              // epilogue: snake-order (half, chunk) units (CK_EPI_SNAKE=0 disables)
  int last_k;             // OP_IM2COL_K: K=8 MMAs needed in a tap's last 32-channel chunk
                          // (1..4; the rest of the chunk is channel padding = zeros)
  // EPI_PIX with out2 (fused relu): also store relu(v) into the NEXT conv's
  // padded pixel-major x grid (the consumer's x_grid, see XGridPlan): row
  // (n, oi, oj) -> grid pixel (n, oj + gx_pl, oi + gx_pt) of an gx_Hg x gx_Wg
  // image grid, channel c -> g'*gx_Cgp + (c - g'*gx_Cg), g' = c / gx_Cg
  float* gx;
  int gx_Hg, gx_Wg, gx_Cp, gx_Cg, gx_Cgp, gx_pt, gx_pl, gx_OH;
  // gx with gx_gate (a data gradient, no relu / bias / accumulate): the grid
  // gets gx_gate > 0 ? v : 0 (gx_gate laid out like out: the relu output that
  // fed this conv) instead of relu(v) -- the conv below's relu-gated dy grid --
  // and gx_bpart[(m / 32) * gx_Cp + grid channel] the per-32-row column sums
  // of those values (its bias-gradient partials)
  const float* gx_gate;
  double* gx_bpart;
  int dg_skip;  // CK_EXPERIMENTS: 1 no gate loads, 2 no grid store, 4 no bias partials
  int estage;   // gx: kEpiWarps 32 x 32 float stages after the barriers (coalesced grid rows)
  int BM;                 // 128 or 256 (two M=128 MMAs sharing the B tile)
  int nacc;               // TMEM accumulator buffers (2: epilogue overlaps mainloop)
  int groups;             // tiles = ceil(M/BM) * ceil(N/BN) * groups * splits
  int b_rows;             // OP_SHIFT_MN: channels per TMA box (divides Cgp and BN)
  int a_rows;             // A = OP_SHIFT_MN (weight gradient, roles swapped): same, dividing BM
  int a_mn3d, b_mn3d;     // OP_TILED_MN: one 3D box per stage (MN % 32 == 0) vs R/32 2D boxes
  int taps;               // OP_SHIFT_MN / halo kernel: fh * fw
  int kstage;             // K per pipeline stage: 32, or 64 (MN-major pair, or SHIFT_K/TILED_K3)
  // halo kernel (stride-1 conv on a padded pixel-major grid, see halo_conv_kernel)
  int hg, hw_grid;        // grid pitch (rows per column) and rows per image; 0 = not a grid
  int ohv, owv;           // valid output extent on the grid
  int arows, abox, anbox; // halo rows per A stage, rows per A box, A boxes per stage
  int TT;                 // taps per B stage
  int SA, SB;             // A / B ring depths
  unsigned long long* prof;  // debug (CK_HALO_PROF): per-CTA wait-cycle counters
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// ---- predicated forms for a warp-converged producer: every lane runs the
// loop, the lane with pred != 0 (elect_one) issues -- no divergent branch
// around the async-proxy instructions.
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t p;
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n"
      : "=r"(p));
  return p;
}

__device__ __forceinline__ void mbar_expect_tx_p(uint64_t* bar, uint32_t bytes, uint32_t pred) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n"
      "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "r"(bytes), "r"(pred)
      : "memory");
}

__device__ __forceinline__ void tma_2d_p(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                         int c1, uint32_t pred) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %5, 0;\n"
      "@q cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(pred)
      : "memory");
}

__device__ __forceinline__ void tma_3d_p(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                         int c1, int c2, uint32_t pred) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %6, 0;\n"
      "@q cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(pred)
      : "memory");
}

__device__ __forceinline__ void tma_im2col_4d_p(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c, int h, int w, int n, uint16_t oh,
                                                uint16_t ow, uint32_t pred) {
  asm volatile(
      "{\n.reg .pred q;\nsetp.ne.u32 q, %9, 0;\n"
      "@q cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};\n}\n" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c), "r"(h), "r"(w), "r"(n), "h"(oh), "h"(ow),
      "r"(pred)
      : "memory");
}

__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                       int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_im2col_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                              int c, int h, int w, int n, uint16_t oh,
                                              uint16_t ow) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c), "r"(h), "r"(w), "r"(n), "h"(oh), "h"(ow)
      : "memory");
}

// UMMA shared-memory descriptor (sm_100 "version 1"), SWIZZLE_128B = 2.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// Operand descriptor for K step k (of 8) in M/N half h of a stage.
//   K-major, SWIZZLE_128B (layout 2): rows of 128 B = 32 k; K step +32 B;
//     8-row groups 1024 B apart (SBO).
//   MN-major, SWIZZLE_128B_BASE32B (layout 1; the only MN-major layout for
//     tf32): k-rows of 128 B = 32 m/n, 32-B chunks swizzled by k & 3; 4-k
//     groups 512 B apart (SBO), 32-wide MN blocks 4096 B apart (LBO); K step
//     of 8 = +1024 B.  (tools/mn_probe.cu checks both against a CPU GEMM.)
// ks = K rows per stage (32, or 64 when both operands are MN-major: each
// 32-wide MN block then holds ks k-rows, LBO = ks * 128).
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int h, int k, int ks = 32) {
  return MN ? sdesc(base + h * ks * 512 + k * 1024, ks * 128, 512, 1)
            : sdesc(base + h * 16384 + k * 32, 16, 1024, 2);
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, M = 128.
__device__ __forceinline__ uint32_t idesc_tf32(int n, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// 3D box multicast to the CTAs of ctaMask (same smem offset, same mbarrier
// offset in every destination CTA).
__device__ __forceinline__ void tma_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                          int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

// MMA completion -> arrive on the mbarrier at this offset in every CTA of mask.
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mma_commit_mc_elect(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Warp-converged variants: all 32 lanes execute the issue loop and one
// elected lane issues (no per-instruction divergence handling in SASS).
__device__ __forceinline__ void mma_tf32_elect(uint32_t tmem_d, uint64_t a, uint64_t b,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Four MMAs of one stage from one elected lane: A/B descriptors advance by
// astep/bstep (16-byte units) per MMA; the first accumulates iff acc != 0.
// One asm block keeps the per-kblock issue path short -- the issue loop is
// latency-bound on its own instruction count otherwise (~160 instructions
// per 4 MMAs took longer than the MMAs themselves).
__device__ __forceinline__ void mma4_elect(uint32_t d, uint64_t a, uint32_t astep, uint64_t b,
                                           uint32_t bstep, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t;\n"
      ".reg .b64 a1, a2, a3, b1, b2, b3, sa, sb;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "setp.ne.b32 t, %3, 0;\n"  // idesc != 0: constant true
      "cvt.u64.u32 sa, %4;\n"
      "cvt.u64.u32 sb, %5;\n"
      "add.s64 a1, %1, sa;\n"
      "add.s64 b1, %2, sb;\n"
      "add.s64 a2, a1, sa;\n"
      "add.s64 b2, b1, sb;\n"
      "add.s64 a3, a2, sa;\n"
      "add.s64 b3, b2, sb;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a1, b1, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a2, b2, %3, t;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], a3, b3, %3, t;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(astep), "r"(bstep), "r"(acc));
}

// As mma4_elect, but only the first n (1..4) of the four MMAs: a tap's last
// channel chunk whose tail is zero padding skips the all-zero K steps.
__device__ __forceinline__ void mma4n_elect(uint32_t d, uint64_t a, uint32_t astep, uint64_t b,
                                            uint32_t bstep, uint32_t idesc, uint32_t acc,
                                            uint32_t n) {
  asm volatile(
      "{\n"
      ".reg .pred e, p, t, e1, e2, e3;\n"
      ".reg .b64 a1, a2, a3, b1, b2, b3, sa, sb;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "setp.ne.b32 t, %3, 0;\n"
      "setp.gt.and.u32 e1, %7, 1, e;\n"
      "setp.gt.and.u32 e2, %7, 2, e;\n"
      "setp.gt.and.u32 e3, %7, 3, e;\n"
      "cvt.u64.u32 sa, %4;\n"
      "cvt.u64.u32 sb, %5;\n"
      "add.s64 a1, %1, sa;\n"
      "add.s64 b1, %2, sb;\n"
      "add.s64 a2, a1, sa;\n"
      "add.s64 b2, b1, sb;\n"
      "add.s64 a3, a2, sa;\n"
      "add.s64 b3, b2, sb;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "@e1 tcgen05.mma.cta_group::1.kind::tf32 [%0], a1, b1, %3, t;\n"
      "@e2 tcgen05.mma.cta_group::1.kind::tf32 [%0], a2, b2, %3, t;\n"
      "@e3 tcgen05.mma.cta_group::1.kind::tf32 [%0], a3, b3, %3, t;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(astep), "r"(bstep), "r"(acc), "r"(n));
}

__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

#define CK_LD32(r, taddr)                                                                   \
  asm volatile(                                                                             \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                             \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22," \
      "%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                        \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),          \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),       \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),       \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),       \
        "=r"(r[31])                                                                         \
      : "r"(taddr));

constexpr int kEpiWarps = 8;                  // epilogue warps (multiple of 4)
constexpr int kThreads = 32 * (2 + kEpiWarps);  // + producer + MMA issuer

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Tile decomposition shared by the three roles of a persistent CTA.
struct Tile {
  int m0, n0, grp, split, kb0, kb1;
};

__device__ __forceinline__ Tile tile_at(const GemmParams& p, int t) {
  Tile r;
  const int tm = (p.M + p.BM - 1) / p.BM, tn = (p.N + p.BN - 1) / p.BN;
  const int mt = t % tm;
  const int rest = t / tm;
  const int nt = rest % tn;
  const int z = rest / tn;
  r.m0 = mt * p.BM;
  r.n0 = nt * p.BN;
  r.grp = z / p.splits;
  r.split = z % p.splits;
  const int nkb = p.K / p.kstage;
  const int per = (nkb + p.splits - 1) / p.splits;
  r.kb0 = r.split * per;
  r.kb1 = min(nkb, r.kb0 + per);
  return r;
}

// One output tile of the accumulator at TMEM column `tacc` -> global.
// kEpiWarps warps: warp w reads TMEM lane quarter w & 3 (hardware rule) and
// every (kEpiWarps/4)-th 32-column chunk, so two warps share a quarter.
// Rows are GEMM rows m; with p.hg > 0 (halo kernels) m is a position on a
// padded grid of pitch hg (hw_grid rows per image) and only positions with
// (u, v) < (ohv, owv) are real outputs, at pixel u + ohv * v.
// Per-column bias of epilogue work unit u of this warp (lane j: column j of the
// unit's 32-column chunk; 0 when the unit has no per-column bias).  Loaded one
// unit ahead so the L2 latency hides behind the previous unit's stores (the
// first unit's before the accumulator wait).
__device__ __forceinline__ int epi_unit_c0(const GemmParams& p, int u, int nch) {
  const int h = u / nch, ci = u - h * nch;
  return 32 * ((h & 1) && p.snake ? nch - 1 - ci : ci);
}
__device__ __forceinline__ float epi_unit_bias(const GemmParams& p, const Tile& T, int u,
                                               int units, int nch, int lane) {
  if (u >= units || !p.bias || p.splits > 1 || p.epi != EPI_PIX) return 0.f;
  const int c0 = epi_unit_c0(p, u, nch), col0 = T.n0 + c0;
  const int lim = min(min(32, p.BN - c0), p.n_valid - col0);
  return lane < lim ? __ldg(p.bias + col0 + T.grp * p.grp_col + lane) : 0.f;
}

__device__ __forceinline__ void epilogue_tile(const GemmParams& p, const Tile& T, uint32_t tacc,
                                              bool empty_split, int halves, int warp, int lane,
                                              float bias_first, float* estage = nullptr) {
  const int q = warp & 3;
  const int cpart = (warp - 2) / 4, cparts = kEpiWarps / 4;
  float* out = p.out;
  const bool partial = p.splits > 1;
  if (partial) out += (int64_t)T.split * p.split_stride;
  // plain stores: split-K partials, or no bias / relu / accumulate
  // per-column (EPI_PIX) bias is added to the TMEM values before the stores
  const bool col_bias = p.bias && !partial && p.epi == EPI_PIX;
  const bool plain = partial || ((!p.bias || col_bias) && !p.relu && !p.acc && !p.out2 && !p.gx);
  const int64_t ld = p.ld;
  // (half, 32-column chunk) units dealt to the cparts warps of a lane quarter
  // in snake order (odd halves walk the chunks backwards): balanced when a
  // half has an odd number of chunks (BN = 96) or a short last chunk (BN = 48)
  const int nch = (p.BN + 31) / 32, units = halves * nch;
  float bias_next = bias_first;
  for (int u = cpart; u < units; u += cparts) {
    const int h = u / nch;
    const int c0 = epi_unit_c0(p, u, nch);
    const float lane_bias = bias_next;
    bias_next = epi_unit_bias(p, T, u + cparts, units, nch, lane);  // next unit, in flight
    int m = T.m0 + h * 128 + q * 32 + lane;
    bool row_ok = m < p.M;
    int img = 0, pix = 0;
    if (p.hg > 0) {
      img = m / p.hw_grid;
      const int r = m - img * p.hw_grid;
      const int v = r / p.hg, u = r - v * p.hg;
      row_ok = row_ok && u < p.ohv && v < p.owv;
      pix = u + p.ohv * v;
    } else if (p.epi != EPI_LINEAR) {
      img = m / p.epi_OHW;
      pix = m - img * p.epi_OHW;
    }
    int64_t row_base = 0;
    float rbias = 0.f;
    int s_i = 0, s_j = 0;  // EPI_S2D: top-left target pixel of this row's s x s block
    if (p.epi == EPI_S2D) {
      const int v = pix / p.s2d_U, u = pix - v * p.s2d_U;
      s_i = p.s2d * u;
      s_j = p.s2d * v;
      row_base = ((int64_t)img * (p.s2d_Ct ? p.s2d_Ct : p.s2d_C) + (int64_t)T.grp * p.grp_col) *
                 p.s2d_H * p.s2d_W;
    } else if (p.epi == EPI_PIX) {
      row_base = (int64_t)img * p.img_stride + pix + (int64_t)T.grp * p.grp_col * p.ld;
    } else {
      row_base = (int64_t)m + (int64_t)T.grp * p.grp_out;
      if (p.bias && !partial && row_ok) rbias = p.bias[m + T.grp * p.grp_col];
    }
    {
      uint32_t r[32];
      const uint32_t taddr = tacc + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * p.BN + c0);
      const int col0 = T.n0 + c0;
      // columns of this chunk inside both the tile and the matrix
      const int lim = min(min(32, p.BN - c0), p.n_valid - col0);
      // gx_gate: this row's 32 gate values, loaded before the accumulator read
      // (independent loads in flight; the stores below may not alias them)
      float gv[32];
      if (p.gx_gate && !(DG_SKIP(p) & 1)) {
        const float* gsrc = p.gx_gate + row_base + (int64_t)col0 * ld;
#pragma unroll
        for (int j = 0; j < 32; ++j) gv[j] = row_ok && j < lim ? __ldg(gsrc + j * ld) : 0.f;
      }
      // per-column bias (lane j holds column j, loaded one unit ahead): broadcast by shuffle
      CK_LD32(r, taddr);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (empty_split)
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      if (col_bias)  // warp-uniform: every lane shuffles
#pragma unroll
        for (int j = 0; j < 32; ++j)
          r[j] = __float_as_uint(__fadd_rn(__uint_as_float(r[j]), __shfl_sync(0xffffffffu, lane_bias, j)));
      if (row_ok && lim > 0 && p.epi == EPI_S2D) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {  // static r[] indexing: keeps r in registers
          const int col = col0 + j;
          const int cg = p.s2d_C, abc = col / cg, c = col - abc * cg;
          const int i = s_i + abc % p.s2d, jj = s_j + abc / p.s2d;
          if (j < lim && i < p.s2d_H && jj < p.s2d_W) {
            float* dst = out + row_base + i + (int64_t)p.s2d_H * (jj + (int64_t)p.s2d_W * c);
            float v = __uint_as_float(r[j]);
            if (!partial && p.acc) v = __fadd_rn(*dst, v);
            *dst = v;
          }
        }
      } else if (row_ok && lim > 0) {
        float* dst = out + row_base + (int64_t)col0 * ld;
        if (plain && lim == 32) {
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[j * ld] = __uint_as_float(r[j]);
        } else if (plain) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < lim) dst[j * ld] = __uint_as_float(r[j]);
        } else {
          float* dst2 = p.out2 ? p.out2 + row_base + (int64_t)col0 * ld : nullptr;
          const bool gate = p.gx_gate != nullptr && !(DG_SKIP(p) & 1);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < lim) {
              float v = __uint_as_float(r[j]);
              if (p.bias && !col_bias) v = __fadd_rn(v, rbias);
              if (p.relu) v = v > 0.f ? v : 0.f;
              if (p.acc) v = __fadd_rn(dst[j * ld], v);
              dst[j * ld] = v;
              const float rv = gate ? (gv[j] > 0.f ? v : 0.f) : (v > 0.f ? v : 0.f);
              if (dst2) dst2[j * ld] = rv;  // fused relu layer
              r[j] = __float_as_uint(rv);
            }
          }
          if (p.gx && !(DG_SKIP(p) & 2) && !(estage && lim == 32)) {
            // the next conv's x grid: this pixel's 32 consecutive channels are
            // one contiguous 128-byte run of its grid row (host: gx_Cg % 32 == 0)
            const int oj = pix / p.gx_OH, oi = pix - oj * p.gx_OH;
            const int col = T.grp * (int)p.grp_col + col0;
            const int g2 = col / p.gx_Cg;
            const int64_t grow = (((int64_t)img * p.gx_Wg + oj + p.gx_pl) * p.gx_Hg + oi + p.gx_pt) *
                                     p.gx_Cp + g2 * p.gx_Cgp + (col - g2 * p.gx_Cg);
            float* gd = p.gx + grow;
            if (lim == 32) {
#pragma unroll
              for (int q4 = 0; q4 < 8; ++q4)
                reinterpret_cast<float4*>(gd)[q4] =
                    make_float4(__uint_as_float(r[4 * q4]), __uint_as_float(r[4 * q4 + 1]),
                                __uint_as_float(r[4 * q4 + 2]), __uint_as_float(r[4 * q4 + 3]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < lim) gd[j] = __uint_as_float(r[j]);
            }
          }
        }
      }
      if (estage && p.gx && lim == 32 && !(DG_SKIP(p) & 2)) {  // warp-uniform
        // grid rows through this warp's shared stage: lane = row writes its 32
        // values as 8 16-byte chunks (xor-swizzled by row: conflict-free), then
        // lane (q4, m4) stores chunk m4 of row 4 it + q4 -- each instruction
        // writes 4 whole 128-byte grid rows instead of 32 half sectors
        const int colg = T.grp * (int)p.grp_col + col0;
        const int g2 = colg / p.gx_Cg;
        const int cbase = g2 * p.gx_Cgp + (colg - g2 * p.gx_Cg);
        int growi = -1;  // this lane's grid row offset (host: grid < 2^31 floats)
        if (row_ok && !partial && p.epi == EPI_PIX) {
          const int oj = pix / p.gx_OH, oi = pix - oj * p.gx_OH;
          growi = (int)((((int64_t)img * p.gx_Wg + oj + p.gx_pl) * p.gx_Hg + oi + p.gx_pt) *
                        p.gx_Cp);
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k)
          *reinterpret_cast<float4*>(estage + lane * 32 + ((k ^ (lane & 7)) << 2)) =
              make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                          __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
        __syncwarp();
        const int q4 = lane >> 3, m4 = lane & 7;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int row = 4 * it + q4;
          const int gr = __shfl_sync(0xffffffffu, growi, row);
          const float4 v =
              *reinterpret_cast<const float4*>(estage + row * 32 + ((m4 ^ (row & 7)) << 2));
          if (gr >= 0) {
            *reinterpret_cast<float4*>(p.gx + gr + cbase + 4 * m4) = v;
            s0 = __fadd_rn(s0, v.x);
            s1 = __fadd_rn(s1, v.y);
            s2 = __fadd_rn(s2, v.z);
            s3 = __fadd_rn(s3, v.w);
          }
        }
        if (p.gx_bpart && !(DG_SKIP(p) & 4)) {
          // column sums over the 32 rows: 8 rows per lane in order, then the 4
          // row lanes of a chunk by a fixed xor tree
#pragma unroll
          for (int o = 8; o <= 16; o <<= 1) {
            s0 = __fadd_rn(s0, __shfl_xor_sync(0xffffffffu, s0, o));
            s1 = __fadd_rn(s1, __shfl_xor_sync(0xffffffffu, s1, o));
            s2 = __fadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, o));
            s3 = __fadd_rn(s3, __shfl_xor_sync(0xffffffffu, s3, o));
          }
          const int mw = T.m0 + h * 128 + q * 32;  // this warp's first row
          if (q4 == 0) {
            double* bp = p.gx_bpart + (int64_t)(mw >> 5) * p.gx_Cp + cbase + 4 * m4;
            bp[0] = s0;
            bp[1] = s1;
            bp[2] = s2;
            bp[3] = s3;
          }
        }
      } else if (p.gx_bpart && lim > 0 && !(DG_SKIP(p) & 4)) {  // warp-uniform
        // column sums of the gated grid values over this warp's 32 rows:
        // transpose-reduce (lane l ends with column l), a fixed tree
        __syncwarp();
        const bool okrow = row_ok && !partial;
        float* v = gv;  // (the gates are consumed)
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = okrow && j < lim ? __uint_as_float(r[j]) : 0.f;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          const bool upper = lane & o;
#pragma unroll
          for (int j = 0; j < o; ++j) {
            const float send = upper ? v[j] : v[j + o];
            const float keep = upper ? v[j + o] : v[j];
            v[j] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
          }
        }
        const int col = T.grp * (int)p.grp_col + col0 + lane;
        const int g2 = col / p.gx_Cg;
        const int mw = T.m0 + h * 128 + q * 32;  // this warp's first row
        if (lane < lim)
          p.gx_bpart[(int64_t)(mw >> 5) * p.gx_Cp + g2 * p.gx_Cgp + (col - g2 * p.gx_Cg)] = v[0];
      }
      __syncwarp();  // reconverge before the next warp-wide tcgen05.ld
    }
  }
}

// The MMA issuer's K loop for one tile: NG groups of four MMAs per stage
// (group g: A/B descriptor offsets ga/gb, accumulator column offset gd; bit g
// of first_mask = group g starts an accumulator, so it overwrites on the
// tile's first stage).  Straight-line per stage: wait full, issue, commit.
struct Ring {
  int s;
  uint32_t ph;
};
template <int NG, bool SKIP>
__device__ __forceinline__ void mma_tile(uint64_t* full, uint64_t* empty, int S, Ring& r, int nkb,
                                         uint32_t dcol, uint64_t da0, uint64_t db0, uint32_t sa16,
                                         uint32_t sb16, uint32_t ak, uint32_t bk, const uint32_t* ga,
                                         const uint32_t* gb, const uint32_t* gd, uint32_t first_mask,
                                         uint32_t idesc, bool wait_full, bool do_mma, int cc,
                                         int cchunks, uint32_t last_k) {
  uint32_t oa[NG], ob[NG], od[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    oa[g] = ga[g];
    ob[g] = gb[g];
    od[g] = dcol + gd[g];
  }
  for (int i = 0; i < nkb; ++i) {
    if (wait_full) mbar_wait(&full[r.s], r.ph);
    tc_fence_after();
    const uint64_t da = da0 + (uint64_t)(r.s * sa16), db = db0 + (uint64_t)(r.s * sb16);
    if (do_mma) {
      if (SKIP && cc == cchunks - 1) {  // tap's last chunk: skip the zero-padded K steps
#pragma unroll
        for (int g = 0; g < NG; ++g)
          mma4n_elect(od[g], da + oa[g], ak, db + ob[g], bk, idesc,
                      (i > 0 || !((first_mask >> g) & 1)) ? 1u : 0u, last_k);
      } else {
#pragma unroll
        for (int g = 0; g < NG; ++g)
          mma4_elect(od[g], da + oa[g], ak, db + ob[g], bk, idesc,
                     (i > 0 || !((first_mask >> g) & 1)) ? 1u : 0u);
      }
    }
    if (SKIP && ++cc == cchunks) cc = 0;
    mma_commit_elect(&empty[r.s]);
    if (++r.s == S) {
      r.s = 0;
      r.ph ^= 1;
    }
  }
}

// ============================================================================
//                                 the kernel
// ============================================================================
// Persistent: CTA b processes tiles b, b + gridDim.x, ...  Each tile is
// BM (128 or 256, i.e. 1 or 2 M=128 MMAs sharing the B tile) x BN.  The
// accumulator lives in TMEM, double buffered (nacc = 2) when it fits, so the
// epilogue of tile i overlaps the mainloop of tile i+1.
template <int AK, int BK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b, const GemmParams p) {
  ck::pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = p.stages;
  const int halves = p.BM / 128;
  const int KS = p.kstage;
  const int stage_a = p.BM * KS * 4;
  const int stage_b = p.BN * KS * 4;
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * stage_a;
  uint64_t* full = (uint64_t*)(sB + S * stage_b);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;       // [nacc]
  uint64_t* tempty = tfull + 2;      // [nacc]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // gx: per epilogue warp a 32 x 32 float stage after the 256 barrier bytes
  float* estage = p.estage && warp >= 2
                      ? (float*)(sB + S * stage_b + 256) + (warp - 2) * 32 * 32
                      : nullptr;
  const int tm = (p.M + p.BM - 1) / p.BM, tn = (p.N + p.BN - 1) / p.BN;
  const int total = tm * tn * p.groups * p.splits;
  const int acc_cols = halves * p.BN;  // TMEM columns per accumulator buffer
  const int need = p.nacc * acc_cols;
  const int ncols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tma_b) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- producer --
    // warp-converged: all lanes walk the loop, the elected lane issues
    {
      const uint32_t lead = elect_one();
      const uint32_t bytes = stage_a + stage_b;
      const int kc_step = KS / 32;  // 32-channel chunks per K block
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Tile T = tile_at(p, t);
        // im2col origin of this M tile (first output pixel)
        int a_h = 0, a_w = 0, a_n = 0;
        if (AK == OP_IM2COL_K) {
          const int ohw = p.OH * p.OW;
          a_n = T.m0 / ohw;
          const int r = T.m0 - a_n * ohw;
          a_w = r / p.OH;
          a_h = r - a_w * p.OH;
          a_h = a_h * p.sh - p.pt;
          a_w = a_w * p.sw - p.pl;
        }
        // (tap, chunk) walk of the A operand, advanced incrementally per K block:
        // OP_IM2COL_K: K block kb = tap * cchunks + cc;
        // OP_SHIFT_K:  32-channel chunk kc = kb * KS / 32 = tap * cchunks + cc
        int cc = 0, fi = 0, fj = 0;
        if (AK == OP_IM2COL_K || AK == OP_SHIFT_K) {
          const int kc = AK == OP_IM2COL_K ? T.kb0 : T.kb0 * kc_step;
          const int tap = kc / p.cchunks;
          cc = kc - tap * p.cchunks;
          fj = tap / p.fh;
          fi = tap - fj * p.fh;
        }
        // OP_SHIFT_MN A boxes (roles swapped: M = (tap, c)), same walk as B's
        int a_shift[8], a_cb[8];
        const int nabox = AK == OP_SHIFT_MN ? p.BM / p.a_rows : 0;
        if (AK == OP_SHIFT_MN) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int mm = T.m0 + j * p.a_rows;
            int tap = mm / (p.cchunks * 32);
            const int c = mm - tap * p.cchunks * 32;
            tap = min(tap, p.taps - 1);  // rows past the last tap are masked
            const int jj = tap / p.fh, ii = tap - jj * p.fh;
            a_shift[j] = ii + p.Hp * jj;
            a_cb[j] = (T.grp * p.a_grp_c + c) / 32;
          }
        }
        // OP_SHIFT_MN B boxes: per-tile (row shift, channel block) of each box
        int b_shift[8], b_cb[8];
        const int nbox = BK == OP_SHIFT_MN ? p.BN / p.b_rows : 0;
        if (BK == OP_SHIFT_MN) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int nn = T.n0 + j * p.b_rows;
            int tap = nn / (p.cchunks * 32);
            const int c = nn - tap * p.cchunks * 32;
            tap = min(tap, p.taps - 1);  // columns past the last tap are masked
            const int jj = tap / p.fh, ii = tap - jj * p.fh;
            b_shift[j] = ii + p.Hp * jj;
            b_cb[j] = (T.grp * p.b_grp_c + c) / 32;
          }
        }
        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          if (TC_EXP(p) != 5) mbar_wait(&empty[s], ph ^ 1);  // exp 5: no producer
          if (TC_EXP(p) == 2) {  // experiment: no operand loads (measures MMA + smem reads)
            if (lead) mbar_arrive(&full[s]);
          } else if (TC_EXP(p) != 5) {
            mbar_expect_tx_p(&full[s], bytes, lead);
            uint8_t* a = sA + s * stage_a;
            uint8_t* b = sB + s * stage_b;
            const int k0 = kb * KS;
            // ---- A (BM rows) ----
            if (AK == OP_TILED_K) {
              tma_2d_p(a, &tma_a, &full[s], k0 + T.grp * p.a_grp_k, T.m0 + T.grp * p.a_grp_mn, lead);
            } else if (AK == OP_TILED_MN) {
              const int mn0 = T.m0 + T.grp * p.a_grp_mn;
              if (p.a_mn3d)
                tma_3d_p(a, &tma_a, &full[s], 0, k0, mn0 / 32, lead);
              else
                for (int j = 0; j < p.BM / 32; ++j)
                  tma_2d_p(a + j * KS * 128, &tma_a, &full[s], mn0 + 32 * j, k0, lead);
            } else if (AK == OP_SHIFT_MN) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j < nabox)
                  tma_3d_p(a + j * p.a_rows * KS * 4, &tma_a, &full[s], 0, k0 + a_shift[j], a_cb[j],
                           lead);
            } else if (AK == OP_SHIFT_K) {
              // K block = KS channels of one tap (KS divides Cgp): BM consecutive
              // grid rows shifted by the tap, one 3D box of KS/32 channel chunks
              tma_3d_p(a, &tma_a, &full[s], 0, T.m0 + p.base_shift + fi + p.Hp * fj,
                       (T.grp * p.a_grp_c) / 32 + cc, lead);
            } else {  // OP_IM2COL_K: one box walks BM pixels
              tma_im2col_4d_p(a, &tma_a, &full[s], T.grp * p.a_grp_c + cc * 32, a_h, a_w, a_n,
                              (uint16_t)fi, (uint16_t)fj, lead);
            }
            // ---- B (BN rows) ----
            if (BK == OP_TILED_K3) {
              tma_3d_p(b, &tma_b, &full[s], 0, T.n0 + T.grp * p.b_grp_mn, k0 / 32, lead);
            } else if (BK == OP_TILED_K) {
              tma_2d_p(b, &tma_b, &full[s], k0 + T.grp * p.b_grp_k, T.n0 + T.grp * p.b_grp_mn, lead);
            } else if (BK == OP_TILED_MN) {
              const int mn0 = T.n0 + T.grp * p.b_grp_mn;
              if (p.b_mn3d)
                tma_3d_p(b, &tma_b, &full[s], 0, k0, mn0 / 32, lead);
              else
                for (int j = 0; j < p.BN / 32; ++j)
                  tma_2d_p(b + j * KS * 128, &tma_b, &full[s], mn0 + 32 * j, k0, lead);
            } else if (BK == OP_SHIFT_MN) {
              // K block = KS rows of the padded grid (pitch Hp); MN = (tap, c):
              // one 3D box per tap, b_rows channels, rows shifted by the tap.
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j < nbox)
                  tma_3d_p(b + j * p.b_rows * KS * 4, &tma_b, &full[s], 0, k0 + b_shift[j], b_cb[j],
                           lead);
            }
          }
          // advance the (tap, chunk) walk and the stage ring
          if (AK == OP_IM2COL_K || AK == OP_SHIFT_K) {
            cc += AK == OP_IM2COL_K ? 1 : kc_step;
            if (cc >= p.cchunks) {
              cc -= p.cchunks;
              if (++fi == p.fh) {
                fi = 0;
                ++fj;
              }
            }
          }
          if (++s == S) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer --
    // the whole warp walks the loop; one elected lane issues each MMA/commit
    {
      constexpr bool a_mn = AK == OP_TILED_MN || AK == OP_SHIFT_MN,
                     b_mn = BK == OP_TILED_MN || BK == OP_SHIFT_MN;
      const uint32_t idesc = idesc_tf32(p.BN, a_mn, b_mn);
      int it = 0, tc = 0;
      // descriptors of stage 0 / half 0 / k 0, advanced in 16-byte units:
      //   K-major SW128: k +32 B, half +16 KB (128 rows), 32-k chunk +rows*128 B
      //   MN-major SW128_32B: k +1024 B, half +KS*512 B
      const uint64_t da0 = a_mn ? sdesc(smem_u32(sA), KS * 128, 512, 1) : sdesc(smem_u32(sA), 16, 1024, 2);
      const uint64_t db0 = b_mn ? sdesc(smem_u32(sB), KS * 128, 512, 1) : sdesc(smem_u32(sB), 16, 1024, 2);
      const uint32_t ak = a_mn ? 64 : 2, bk = b_mn ? 64 : 2;
      const uint32_t ah = a_mn ? KS * 32 : 1024;
      const uint32_t sa16 = stage_a >> 4, sb16 = stage_b >> 4;
      const bool do_mma = TC_EXP(p) != 1;      // exp 1: no MMAs (TMA only)
      const bool wait_full = TC_EXP(p) != 5;   // exp 5: MMAs only (no operand handshake)
      // MMA groups per stage: (half h, 32-k chunk c) -> g = h * chunks + c
      const int chunks = KS / 32, ng = halves * chunks;
      uint32_t ga[4] = {0, 0, 0, 0}, gb[4] = {0, 0, 0, 0}, gd[4] = {0, 0, 0, 0}, first_mask = 0;
      for (int h = 0; h < halves; ++h)
        for (int c = 0; c < chunks; ++c) {
          const int g = h * chunks + c;
          const uint32_t ca = AK == OP_SHIFT_K ? p.BM * 8 : 4 * ak;  // 32-k chunk step of A
          const uint32_t cb = AK == OP_SHIFT_K ? p.BN * 8 : 4 * bk;
          ga[g] = h * ah + c * ca;
          gb[g] = c * cb;
          gd[g] = h * p.BN;
          if (c == 0) first_mask |= 1u << g;
        }
      Ring ring{0, 0};
#ifdef CK_TC_PROFILE  // build with -DCK_TC_PROFILE and run with CK_TC_PROF=1
      unsigned long long w_t = 0, w_f = 0, t_start = clock64(), g_start;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
#define CK_PROF_T0(v) unsigned long long v = clock64()
#define CK_PROF_ADD(acc, v) acc += clock64() - v
#else
#define CK_PROF_T0(v)
#define CK_PROF_ADD(acc, v)
#endif
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++tc) {
        const Tile T = tile_at(p, t);
        const int ab = tc % p.nacc;
        const uint32_t aph = (tc / p.nacc) & 1;
        CK_PROF_T0(c0);
        mbar_wait(&tempty[ab], aph ^ 1);  // epilogue drained this accumulator
        CK_PROF_ADD(w_t, c0);
        tc_fence_after();
        const uint32_t dcol = tmem + (uint32_t)(ab * acc_cols);
        const int nkb = T.kb1 - T.kb0;
        // padded-chunk skipping: im2col convs only (kb = tap * cchunks + cc, KS = 32)
        const bool skip = AK == OP_IM2COL_K && KS == 32 && p.last_k >= 1 && p.last_k < 4;
        const int cch = skip ? p.cchunks : 1 << 30;
        const int cc0 = skip ? T.kb0 % p.cchunks : 0;
        const uint32_t lk = skip ? (uint32_t)p.last_k : 4u;
#define CK_MMA_TILE(NG, SK)                                                                   \
  mma_tile<NG, SK>(full, empty, S, ring, nkb, dcol, da0, db0, sa16, sb16, ak, bk, ga, gb, gd,   \
                   first_mask, idesc, wait_full, do_mma, cc0, cch, lk)
        if (skip) {
          if (ng == 1) CK_MMA_TILE(1, true);
          else CK_MMA_TILE(2, true);
        } else if (ng == 1) {
          CK_MMA_TILE(1, false);
        } else if (ng == 2) {
          CK_MMA_TILE(2, false);
        } else {
          CK_MMA_TILE(4, false);
        }
#undef CK_MMA_TILE
        it += nkb;
        mma_commit_elect(&tfull[ab]);
      }
#ifdef CK_TC_PROFILE
      if (p.prof && lane == 0) {
        unsigned long long* o = p.prof + blockIdx.x * 8;
        unsigned long long g_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
        o[0] = clock64() - t_start;
        o[1] = w_t;
        o[2] = w_f;
        o[3] = it;
        o[4] = g_end - g_start;
      }
#endif
#undef CK_PROF_T0
#undef CK_PROF_ADD
    }
    __syncwarp();
  } else {
    // ----------------------------------------------------------- epilogue --
    int tc = 0;
#ifdef CK_TC_PROFILE
    unsigned long long e_w = 0, e_b = 0;
#endif
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++tc) {
      const Tile T = tile_at(p, t);
      const int ab = tc % p.nacc;
      const uint32_t aph = (tc / p.nacc) & 1;
#ifdef CK_TC_PROFILE
      unsigned long long e0 = clock64();
#endif
      const int nch = (p.BN + 31) / 32;
      const float bias0 = epi_unit_bias(p, T, (warp - 2) / 4, halves * nch, nch, lane);
      mbar_wait(&tfull[ab], aph);
      tc_fence_after();
#ifdef CK_TC_PROFILE
      unsigned long long e1 = clock64();
      e_w += e1 - e0;
#endif
      if (TC_EXP(p) != 5)  // exp 5: no epilogue work
        epilogue_tile(p, T, tmem + (uint32_t)(ab * acc_cols), T.kb0 >= T.kb1, halves, warp, lane,
                      bias0, estage);
      tc_fence_before();
      __syncwarp();
#ifdef CK_TC_PROFILE
      e_b += clock64() - e1;
#endif
      if (lane == 0) mbar_arrive(&tempty[ab]);
    }
#ifdef CK_TC_PROFILE
    if (p.prof && warp == 2 && lane == 0) {
      p.prof[blockIdx.x * 8 + 5] = e_w;
      p.prof[blockIdx.x * 8 + 6] = e_b;
    }
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
  }
}

#ifdef CK_EXPERIMENTS  // measured slower than im2col: not in product builds
// ============================================================================
//                      halo kernel (stride-1 implicit GEMM)
// ============================================================================
// A stride-1 convolution over a zero-padded pixel-major grid P[row][Cp]
// (row = n * hw_grid + i + hg * j) is
//     Y[q, k] = sum_{tap, c} P[q + fi + hg * fj, c] * F[k, tap, c]
// for grid rows q (rows whose (u, v) fall outside the valid output extent
// are computed and dropped).  Per 32-channel chunk a CTA loads ONE halo tile
// of rows [q0, q0 + BM + maxshift) and feeds every tap from it by moving the
// UMMA descriptor start by shift * 128 B (the SWIZZLE_128B pattern is keyed
// on address bits, tools/shift_probe.cu) -- the activation operand is read
// once per chunk instead of once per tap.  Filters stream as 3D boxes of TT
// taps x BN rows x 32 channels from F laid [row][tap][Cgp].
// Warp roles as tc_gemm_kernel; A and B have separate mbarrier rings.
// CS = 2: clusters of two CTAs on vertically adjacent M tiles share every
// filter stage -- each loads half the taps of the stage and multicasts it
// to both, and a stage is refilled once both CTAs' MMAs released it.
template <int CS>
__global__ void __launch_bounds__(kThreads, 1)
    halo_conv_kernel(const __grid_constant__ CUtensorMap tma_a,
                     const __grid_constant__ CUtensorMap tma_b, const GemmParams p) {
  ck::pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int halves = p.BM / 128;
  const int stage_a = p.anbox * p.abox * 128;
  const int stage_b = p.TT * p.BN * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + p.SA * stage_a;
  uint64_t* fullA = (uint64_t*)(sB + p.SB * stage_b);
  uint64_t* emptyA = fullA + p.SA;
  uint64_t* fullB = emptyA + p.SA;
  uint64_t* emptyB = fullB + p.SB;
  uint64_t* tfull = emptyB + p.SB;  // [2]
  uint64_t* tempty = tfull + 2;     // [2]
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tm = (p.M + p.BM - 1) / p.BM, tn = (p.N + p.BN - 1) / p.BN;
  const int tmc = (tm + CS - 1) / CS;  // M tiles per cluster row
  const int total = tmc * tn * p.groups;  // cluster work items
  const int rank = CS > 1 ? (int)cluster_rank() : 0;
  const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  const uint16_t cmask = (uint16_t)((1u << CS) - 1);
  const int acc_cols = halves * p.BN;
  const int need = p.nacc * acc_cols;
  const int ncols = need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
  const int chunks = p.cchunks;
  const int ntg = (p.taps + p.TT - 1) / p.TT;
  const int tt_part = p.TT / CS;  // taps of each stage this CTA loads

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.SA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < p.SB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], CS);  // released by the MMAs of every CTA it feeds
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tma_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tma_b) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (CS > 1) cluster_sync();  // peers' barriers are initialised before any multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  auto tile_of = [&](int t) {
    Tile T;
    const int mt = (t % tmc) * CS + rank, rest = t / tmc;
    T.m0 = mt * p.BM;
    T.n0 = (rest % tn) * p.BN;
    T.grp = rest / tn;
    T.split = 0;
    T.kb0 = 0;
    T.kb1 = 1;
    return T;
  };

  if (warp == 0) {
    // ---------------------------------------------------------- producer --
    if (lane == 0) {
      int ia = 0, ib = 0;
      for (int t = cid; t < total; t += ncl) {
        const Tile T = tile_of(t);
        for (int cc = 0; cc < chunks; ++cc) {
          const int sa = ia % p.SA;
          mbar_wait(&emptyA[sa], ((ia / p.SA) & 1) ^ 1);
          mbar_expect_tx(&fullA[sa], stage_a);
          const int c = T.grp * p.a_grp_c + cc * 32;
          for (int bx = 0; bx < p.anbox; ++bx)
            tma_2d(sA + sa * stage_a + bx * p.abox * 128, &tma_a, &fullA[sa], c,
                   T.m0 + bx * p.abox);
          ++ia;
          for (int tg = 0; tg < ntg; ++tg) {
            const int sb = ib % p.SB;
            mbar_wait(&emptyB[sb], ((ib / p.SB) & 1) ^ 1);
            mbar_expect_tx(&fullB[sb], stage_b);
            if (CS > 1)
              tma_3d_mc(sB + sb * stage_b + rank * tt_part * p.BN * 128, &tma_b, &fullB[sb],
                        cc * 32, T.n0 + T.grp * p.b_grp_row, tg * p.TT + rank * tt_part, cmask);
            else
              tma_3d(sB + sb * stage_b, &tma_b, &fullB[sb], cc * 32, T.n0 + T.grp * p.b_grp_row,
                     tg * p.TT);
            ++ib;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer --
    // warp-converged; one elected lane issues four MMAs per asm block
    // (mma4_elect), descriptors advanced by adds, division-free rings
    {
      const uint32_t idesc = idesc_tf32(p.BN, 0, 0);
      const uint64_t a_desc0 = sdesc(smem_u32(sA), 16, 1024, 2);
      const uint64_t b_desc0 = sdesc(smem_u32(sB), 16, 1024, 2);
      int sa = 0, sb = 0, tc = 0;
      uint32_t pha = 0, phb = 0;
      for (int t = cid; t < total; t += ncl, ++tc) {
        const int ab = tc % p.nacc;
        mbar_wait(&tempty[ab], ((tc / p.nacc) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + (uint32_t)(ab * acc_cols);
        for (int cc = 0; cc < chunks; ++cc) {
          mbar_wait(&fullA[sa], pha);
          tc_fence_after();
          const uint64_t da = a_desc0 + (uint64_t)((sa * stage_a) >> 4);
          int fi = 0, fj = 0;
          for (int tg = 0; tg < ntg; ++tg) {
            mbar_wait(&fullB[sb], phb);
            tc_fence_after();
            const uint64_t db = b_desc0 + (uint64_t)((sb * stage_b) >> 4);
            for (int u = 0; u < p.TT; ++u) {
              const int tap = tg * p.TT + u;
              if (tap >= p.taps) break;
              // the tap's A operand starts (fi + hg*fj) rows into the halo tile
              const uint32_t shift16 = (uint32_t)(fi + p.hg * fj) * 8u;
              const uint32_t acc = (cc > 0 || tap > 0) ? 1u : 0u;
              for (int h = 0; h < halves; ++h)
                mma4_elect(dcol + h * p.BN, da + (uint64_t)(h * 1024 + shift16), 2u,
                           db + (uint64_t)(u * p.BN * 8), 2u, idesc, acc);
              if (++fi == p.fh) {
                fi = 0;
                ++fj;
              }
            }
            if (CS > 1)
              mma_commit_mc_elect(&emptyB[sb], cmask);
            else
              mma_commit_elect(&emptyB[sb]);
            if (++sb == p.SB) {
              sb = 0;
              phb ^= 1;
            }
          }
          mma_commit_elect(&emptyA[sa]);
          if (++sa == p.SA) {
            sa = 0;
            pha ^= 1;
          }
        }
        mma_commit_elect(&tfull[ab]);
      }
    }
    __syncwarp();
  } else {
    // ----------------------------------------------------------- epilogue --
    int tc = 0;
    for (int t = cid; t < total; t += ncl, ++tc) {
      const Tile T = tile_of(t);
      const int ab = tc % p.nacc;
      mbar_wait(&tfull[ab], (tc / p.nacc) & 1);
      tc_fence_after();
      const int nch = (p.BN + 31) / 32;
      epilogue_tile(p, T, tmem + (uint32_t)(ab * acc_cols), false, halves, warp, lane,
                    epi_unit_bias(p, T, (warp - 2) / 4, halves * nch, nch, lane));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CS > 1) cluster_sync();  // no CTA leaves while a peer may still signal its barriers
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
  }
}

// ============================================================================
//                          layout transforms (HBM bound)
// ============================================================================

// HWCN x[n][c][w][h] -> padded pixel-major grid xg[n][Wg][Hg][cp]: pixel
// (i, j) at grid position (i + oh, j + ow), channel c of group g at
#endif  // CK_EXPERIMENTS

// cp = g*Cgp + (c - g*Cgp_local); zero borders and channel pads (the input of
// halo_conv_kernel).  32 x 32 smem tile transpose.
// With gate != nullptr the source is relu-gated first (v = gate > 0 ? x : 0,
// the relu backward, activation.cpp:14-22, bit-exact with relu_bwd_v4) and the
// gated HWCN value is also stored to gout: the conv backward consumes the
// relu backward in the same pass over memory.
template <int CH, bool GATE>
__global__ void __launch_bounds__(256, CH == 32 ? (GATE ? 6 : 8) : 4) to_grid_pm_k(
    const float* __restrict__ x, float* __restrict__ xg, int H, int W, int C, int Cg, int Cgp,
    int groups, int Hg, int Wg, int oh, int ow, double* __restrict__ bpart,
    const float* __restrict__ gate, float* __restrict__ gout, int tpb) {
  ck::pdl_entry();
  // tile: 64 grid pixels x CH padded channels; loads coalesced along pixels
  // (two per channel row per thread, CH/8 rows per warp), stores as float4
  // along channels.  Every load of a tile (and of the relu gate) is issued
  // before any is consumed.  A block walks `tpb` consecutive channel tiles of
  // its pixel tile, reusing the per-pixel source and destination arithmetic
  // (the kernel is otherwise bound by its integer index math, not by HBM).
  constexpr int RR = CH / 8;
  __shared__ float tile[2][CH][65];
  const int n = blockIdx.z;
  const int p0 = blockIdx.x * 64;
  const int Cp = Cgp * groups, HWg = Hg * Wg, HW = H * W;
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  int src[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int P = p0 + lane + 32 * k;
    const int jj = P / Hg, ii = P - jj * Hg;
    const int i = ii - oh, j = jj - ow;
    src[k] = (P < HWg && i >= 0 && i < H && j >= 0 && j < W) ? j * H + i : -1;
  }
  const int64_t img = (int64_t)n * C * HW;
  const float* xn = x + img;
  const float* gn = GATE ? gate + img : nullptr;
  float* go = GATE && gout ? gout + img : nullptr;
  // store side: thread -> (pixel row pr, float4 q) of the tile, CH/16 of them
  constexpr int Q = CH / 4;  // float4 per pixel row of the tile
  float* dst[CH / 16];
#pragma unroll
  for (int k = 0; k < CH / 16; ++k) {
    const int idx = threadIdx.x + 256 * k;
    const int pr = idx / Q, q = idx % Q, P = p0 + pr;
    dst[k] = P < HWg ? xg + ((int64_t)n * HWg + P) * Cp + 4 * q : nullptr;
  }
  for (int t = 0; t < tpb; ++t) {
    const int c0 = (blockIdx.y * tpb + t) * CH;
    if (c0 >= Cp) break;
    float(*tl)[65] = tile[t & 1];
    float v[RR][2];
#pragma unroll
    for (int rr = 0; rr < RR; ++rr) {
      const int cp = c0 + warp + 8 * rr;
      const int g = groups == 1 ? 0 : (groups == 2 ? (cp >= Cgp) : cp / Cgp);
      const int cl = cp - g * Cgp;
      const int coff = (cp < Cp && cl < Cg) ? (g * Cg + cl) * HW : -1;
      float gv[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool e = coff >= 0 && src[k] >= 0;
        v[rr][k] = e ? __ldg(xn + coff + src[k]) : 0.f;
        if (GATE) gv[k] = e ? __ldg(gn + coff + src[k]) : 0.f;
      }
      if (GATE) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          v[rr][k] = gv[k] > 0.f ? v[rr][k] : 0.f;
          if (go && coff >= 0 && src[k] >= 0) go[coff + src[k]] = v[rr][k];
        }
      }
    }
#pragma unroll
    for (int rr = 0; rr < RR; ++rr)
#pragma unroll
      for (int k = 0; k < 2; ++k) tl[warp + 8 * rr][lane + 32 * k] = v[rr][k];
    if (bpart) {  // fused bias gradient: this tile's per-channel sums (double, fixed order)
#pragma unroll
      for (int rr = 0; rr < RR; ++rr) {
        const int cp = c0 + warp + 8 * rr;
        double s2 = (double)v[rr][0] + (double)v[rr][1];
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0 && cp < Cp) bpart[((int64_t)n * gridDim.x + blockIdx.x) * Cp + cp] = s2;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CH / 16; ++k) {
      const int idx = threadIdx.x + 256 * k;
      const int pr = idx / Q, q = idx % Q;
      if (dst[k] && c0 + 4 * q < Cp) {
        const float4 w = make_float4(tl[4 * q][pr], tl[4 * q + 1][pr], tl[4 * q + 2][pr],
                                     tl[4 * q + 3][pr]);
        *reinterpret_cast<float4*>(dst[k] + c0) = w;
      }
    }
  }
}

// launch of to_grid_pm_k: 64-channel tiles when the padded channels allow
static void grid_pm_launch(const float* x, float* xg, int H, int W, int C, int N, int Cg, int Cgp,
                           int groups, int Hg, int Wg, int oh, int ow, double* bpart,
                           const float* gate, float* gout, cudaStream_t s) {
  const int Cp = Cgp * groups;
  static const int ch = knob("CK_GRID_CH", 32);  // experiments
  // channel tiles per block: enough blocks for ~8 resident per SM, each
  // walking several tiles
  static const int tpb_env = knob("CK_GRID_TPB", 0);
  auto tiles_per_block = [&](int ctiles, int nb) {
    if (tpb_env > 0) return std::min(tpb_env, ctiles);
    int t = 1;
    while (t < 4 && t * 2 <= ctiles && (int64_t)nb * N * ((ctiles + 2 * t - 1) / (2 * t)) >= 148 * 8 * 2)
      t *= 2;
    return t;
  };
  const int nb = (Hg * Wg + 63) / 64;
  if (ch == 64 && Cp % 64 == 0) {
    const int ct = Cp / 64, t = tiles_per_block(ct, nb);
    dim3 grid(nb, (ct + t - 1) / t, N);
    if (gate)
      ck::pdl_launch(to_grid_pm_k<64, true>, grid, 256, 0, s, x, xg, H, W, C, Cg, Cgp, groups, Hg, Wg, oh, ow,
                                                  bpart, gate, gout, t);
    else
      ck::pdl_launch(to_grid_pm_k<64, false>, grid, 256, 0, s, x, xg, H, W, C, Cg, Cgp, groups, Hg, Wg, oh, ow,
                                                   bpart, gate, gout, t);
  } else {
    const int ct = (Cp + 31) / 32, t = tiles_per_block(ct, nb);
    dim3 grid(nb, (ct + t - 1) / t, N);
    if (gate)
      ck::pdl_launch(to_grid_pm_k<32, true>, grid, 256, 0, s, x, xg, H, W, C, Cg, Cgp, groups, Hg, Wg, oh, ow,
                                                  bpart, gate, gout, t);
    else
      ck::pdl_launch(to_grid_pm_k<32, false>, grid, 256, 0, s, x, xg, H, W, C, Cg, Cgp, groups, Hg, Wg, oh, ow,
                                                   bpart, gate, gout, t);
  }
}

// fprop filters: fT[k][tap][cpos] (tap = fi + fh*fj), from the reference
// filter bank f[fi + fh*(fj + fw*(c*fsc + k*fsk))]; zeros for channel pads.
__global__ void repack_fprop_k(const float* __restrict__ f, float* __restrict__ ft, int fh, int fw,
                               int Cg, int Cgp, int K, int64_t fsc, int64_t fsk) {
  ck::pdl_entry();
  // 32-bit index math (the bank is far below 2^31 elements); the caller
  // checks the 64-bit total
  const int taps = fh * fw;
  const int total = K * taps * Cgp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int r = e / Cgp, cp = e - r * Cgp;
    const int k = r / taps, tap = r - k * taps;
    float v = 0.f;
    if (cp < Cg) {
      const int fj = tap / fh, fi = tap - fj * fh;
      v = __ldg(f + fi + (int64_t)fh * (fj + (int64_t)fw * (cp * fsc + k * fsk)));
    }
    ft[e] = v;
  }
}

// dgrad filters: gT[c][tap'][kpos], kpos = per-group padded filter index,
// tap' = flipped tap: g[fi', fj', k, c] = f[fh-1-fi', fw-1-fj', c, k].
__global__ void repack_dgrad_k(const float* __restrict__ f, float* __restrict__ gt, int fh, int fw,
                               int Cg, int Kg, int Kgp, int groups, int64_t fsc, int64_t fsk) {
  ck::pdl_entry();
  const int taps = fh * fw;
  const int total = Cg * groups * taps * Kgp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int r = e / Kgp, kp = e - r * Kgp;
    const int cc = r / taps, tap = r - cc * taps;  // cc: 0 .. Cg*groups-1
    const int g = cc / Cg, c = cc - g * Cg;
    float v = 0.f;
    if (kp < Kg) {
      const int tj = tap / fh, ti = tap - tj * fh;
      const int fi = fh - 1 - ti, fj = fw - 1 - tj;
      const int64_t k = (int64_t)g * Kg + kp;
      v = __ldg(f + fi + (int64_t)fh * (fj + (int64_t)fw * (c * fsc + k * fsk)));
    }
    gt[e] = v;
  }
}

// B of the 2 x 2-blocked data gradient (conv_tc_dgrad, few channels per
// group): row n = (da + 2 db) Cg + c of group g, column t' Kgp + k with
// t' = u' + (fh + 1) v' over the (fh + 1) x (fw + 1) window of a 2 x 2 output
// block: the flipped tap (u' - da, v' - db) when it lies in the filter, else 0.
__global__ void repack_dgrad_blk_k(const float* __restrict__ f, float* __restrict__ gt, int fh,
                                   int fw, int Cg, int Kg, int Kgp, int groups, int64_t fsc,
                                   int64_t fsk) {
  ck::pdl_entry();
  const int th = fh + 1, taps = th * (fw + 1);
  const int total = groups * 4 * Cg * taps * Kgp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int kp = e % Kgp, r = e / Kgp;
    const int tap = r % taps, rr = r / taps;
    const int g = rr / (4 * Cg), n = rr - g * 4 * Cg;
    const int blk = n / Cg, c = n - blk * Cg, da = blk & 1, db = blk >> 1;
    const int u = tap % th, v = tap / th, ti = u - da, tj = v - db;
    float val = 0.f;
    if (kp < Kg && ti >= 0 && ti < fh && tj >= 0 && tj < fw) {
      const int fi = fh - 1 - ti, fj = fw - 1 - tj;
      const int64_t k = (int64_t)g * Kg + kp;
      val = __ldg(f + fi + (int64_t)fh * (fj + (int64_t)fw * (c * fsc + k * fsk)));
    }
    gt[e] = val;
  }
}

// wgrad: df[fi,fj,c,k] (+)= sum_s part[s][g][n = tap*Cgp + cpos][k]  (fixed order)
// swapped: the partials of the role-swapped GEMM, part[g][k][(tap, c)]
__global__ void wgrad_finish_k(const float* __restrict__ part, float* df, int fh, int fw, int Cg,
                               int Cgp, int Kg, int groups, int splits, int64_t split_stride,
                               int64_t fsc, int64_t fsk, int acc, int swapped) {
  ck::pdl_entry();
  const int taps = fh * fw;
  const int total = groups * Kg * taps * Cg;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    // e enumerates (k fastest) so reads of part are coalesced
    int r = e / Kg;
    const int k = e - r * Kg;
    int r2 = r / Cg;
    const int c = r - r2 * Cg;
    const int g = r2 / taps, tap = r2 - g * taps;
    const int64_t src = swapped ? (int64_t)g * taps * Cgp * Kg + (int64_t)k * taps * Cgp +
                                      (int64_t)tap * Cgp + c
                                : ((int64_t)g * taps * Cgp + (int64_t)tap * Cgp + c) * Kg + k;
    float s = 0.f;
#pragma unroll 4
    for (int sp = 0; sp < splits; ++sp) s += __ldg(part + sp * split_stride + src);
    const int fj = tap / fh, fi = tap - fj * fh;
    const int64_t kk = (int64_t)g * Kg + k;
    float* dst = df + fi + (int64_t)fh * (fj + (int64_t)fw * (c * fsc + kk * fsk));
    *dst = acc ? *dst + s : s;
  }
}

// generic split-K finisher for EPI_LINEAR outputs: out[row + col*ld]
__global__ void splitk_finish_k(const float* __restrict__ part, float* out, int rows, int cols,
                                int64_t ld, int splits, int64_t split_stride,
                                const float* __restrict__ bias, int relu, int acc,
                                float* __restrict__ out2) {
  ck::pdl_entry();
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(total < (1ll << 31) ? (int)e / rows : e / rows);
    const int row = (int)(e - (int64_t)col * rows);
    const int64_t a = row + col * ld;
    float s = 0.f;
#pragma unroll 4
    for (int sp = 0; sp < splits; ++sp) s += __ldg(part + sp * split_stride + a);
    if (bias) s = __fadd_rn(s, bias[row]);
    if (relu) s = s > 0.f ? s : 0.f;
    out[a] = acc ? __fadd_rn(out[a], s) : s;
    if (out2) out2[a] = s > 0.f ? s : 0.f;  // fused relu layer (acc is 0 then)
  }
}

// ---- space-to-depth (strided convolutions, e.g. AlexNet conv1 s=4) ---------
// A stride-s conv equals a stride-1 conv over x_s2d[u][v][c'] =
// x[s*u + a, s*v + b, c], c' = c + Cg*(a + s*b), with taps (t, t2) and filter
// G[t, t2, c', k] = f[a + s*t, b + s*t2, c, k] (zero past the filter edge).

__device__ __forceinline__ float s2d_read(const float* x, int H, int W, int C, int s, int Cg,
                                          int n, int u, int v, int cp) {
  const int c = cp % Cg, ab = cp / Cg;
  const int a = ab % s, b = ab / s;
  const int i = s * u + a, j = s * v + b;
  if (i >= H || j >= W) return 0.f;
  return x[((int64_t)n * C + c) * H * W + i + (int64_t)H * j];
}

// pixel-major s2d tensor [n][v][u][c'p] for the fprop im2col operand
__global__ void s2d_pm_k(const float* __restrict__ x, float* __restrict__ out, int H, int W, int C,
                         int N, int s, int U, int V, int Cs, int Csp) {
  ck::pdl_entry();
  const int64_t total = (int64_t)N * V * U * Csp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int cp = (int)(e % Csp);
    int64_t r = e / Csp;
    const int u = (int)(r % U);
    r /= U;
    const int v = (int)(r % V);
    const int n = (int)(r / V);
    out[e] = cp < Cs ? s2d_read(x, H, W, C, s, C, n, u, v, cp) : 0.f;
  }
}

// Strip-staged s2d transforms.  A block stages x columns [s*v0, s*(v0+VB))
// of one or all channels of image n in shared memory (row pitch Hs = s*U >=
// H, zero past the edges), so every global read is a coalesced column read
// and every write a contiguous run of the output.
__device__ __forceinline__ void s2d_stage_strip(const float* __restrict__ x, float* strip, int H,
                                                int W, int c_first, int c_count, int C, int n,
                                                int j0, int cols, int Hs) {
  // one warp per (channel, column): coalesced column reads, no division
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int cj = warp; cj < c_count * cols; cj += nw) {
    const int cc = cj / cols, jl = cj - cc * cols, j = j0 + jl;
    const float* col = x + (((int64_t)n * C + c_first + cc) * W + j) * H;
    float* dst = strip + (int64_t)cj * Hs;
    const bool jok = j < W;
    // eight loads in flight per lane before any store (the loop is latency-bound otherwise)
    for (int i0 = 0; i0 < Hs; i0 += 256) {
      float r[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + lane + 32 * k;
        r[k] = (jok && i < H) ? __ldg(col + i) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + lane + 32 * k;
        if (i < Hs) dst[i] = r[k];
      }
    }
  }
}

// pixel-major s2d tensor [n][v][u][c'p]; block = (v strip of VB columns, n)
__global__ void s2d_pm_strip_k(const float* __restrict__ x, float* __restrict__ out, int H, int W,
                               int C, int s, int U, int V, int Cs, int Csp, int VB) {
  ck::pdl_entry();
  extern __shared__ float strip_pm[];
  __shared__ int offs[256];  // s2d channel c' -> strip offset of (c, a, b), -1 = pad
  const int n = blockIdx.y, v0 = blockIdx.x * VB;
  const int vb = min(VB, V - v0);
  const int Hs = s * U;
  const int per_c = Hs * s * vb;
  for (int cp = threadIdx.x; cp < Csp; cp += blockDim.x) {
    int o = -1;
    if (cp < Cs) {
      const int c = cp % C, ab = cp / C, a = ab % s, b = ab / s;
      o = c * per_c + a + Hs * b;
    }
    offs[cp] = o;
  }
  s2d_stage_strip(x, strip_pm, H, W, 0, C, C, n, s * v0, s * vb, Hs);
  __syncthreads();
  const int c4 = Csp / 4, total = vb * U * c4;
  float4* o = reinterpret_cast<float4*>(out + (((int64_t)n * V + v0) * U) * Csp);
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int cq = e % c4, pix = e / c4;
    const int vl = pix / U, u = pix - vl * U;
    const int base = s * u + Hs * s * vl;
    float r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int off = offs[cq * 4 + k];
      r[k] = off >= 0 ? strip_pm[off + base] : 0.f;
    }
    o[e] = make_float4(r[0], r[1], r[2], r[3]);
  }
}

// fprop filters of the s2d conv: fT[k][tap = t + Th*t2][c'p]
__global__ void s2d_repack_fprop_k(const float* __restrict__ f, float* __restrict__ ft, int fh,
                                   int fw, int Cg, int K, int s, int Th, int Tw, int Csp,
                                   int64_t fsc, int64_t fsk) {
  ck::pdl_entry();
  const int64_t total = (int64_t)K * Th * Tw * Csp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int cp = (int)(e % Csp);
    int64_t r = e / Csp;
    const int tap = (int)(r % (Th * Tw));
    const int64_t k = r / (Th * Tw);
    float v = 0.f;
    if (cp < s * s * Cg) {
      const int c = cp % Cg, ab = cp / Cg, a = ab % s, b = ab / s;
      const int fi = a + s * (tap % Th), fj = b + s * (tap / Th);
      if (fi < fh && fj < fw) v = f[fi + (int64_t)fh * (fj + (int64_t)fw * (c * fsc + k * fsk))];
    }
    ft[e] = v;
  }
}

// dgrad filters of the s2d conv (flipped taps): gT[c'][tap'][kp]
__global__ void s2d_repack_dgrad_k(const float* __restrict__ f, float* __restrict__ gt, int fh,
                                   int fw, int Cg, int K, int Kp, int s, int Th, int Tw,
                                   int64_t fsc, int64_t fsk) {
  ck::pdl_entry();
  const int Cs = s * s * Cg;
  const int64_t total = (int64_t)Cs * Th * Tw * Kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int kp = (int)(e % Kp);
    int64_t r = e / Kp;
    const int tap = (int)(r % (Th * Tw));
    const int cp = (int)(r / (Th * Tw));
    float v = 0.f;
    if (kp < K) {
      const int c = cp % Cg, ab = cp / Cg, a = ab % s, b = ab / s;
      const int t = Th - 1 - tap % Th, t2 = Tw - 1 - tap / Th;
      const int fi = a + s * t, fj = b + s * t2;
      if (fi < fh && fj < fw) v = f[fi + (int64_t)fh * (fj + (int64_t)fw * (c * fsc + kp * fsk))];
    }
    gt[e] = v;
  }
}

// wgrad finish of the s2d conv: df[fi,fj,c,k] = sum_s part[s][(tap, c'p)][k]
// swapped: partials of the role-swapped GEMM, part[k][n] (n = the s2d (tap, c'))
__global__ void s2d_wgrad_finish_k(const float* __restrict__ part, float* df, int fh, int fw,
                                   int Cg, int K, int s, int Th, int Csp, int splits,
                                   int64_t split_stride, int acc, int64_t fsc, int64_t fsk,
                                   int swapped, int64_t ntot) {
  ck::pdl_entry();
  const int64_t total = (int64_t)K * fh * fw * Cg;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e % K);
    int64_t r = e / K;
    const int c = (int)(r % Cg);
    r /= Cg;
    const int fi = (int)(r % fh);
    const int fj = (int)(r / fh);
    const int t = fi / s, a = fi % s, t2 = fj / s, b = fj % s;
    const int64_t n = (int64_t)(t + Th * t2) * Csp + c + (int64_t)Cg * (a + s * b);
    float v = 0.f;
    const int64_t src = swapped ? (int64_t)k * ntot + n : n * K + k;
    for (int sp = 0; sp < splits; ++sp) v += part[sp * split_stride + src];
    float* dst = df + fi + (int64_t)fh * (fj + (int64_t)fw * (c * fsc + k * fsk));
    *dst = acc ? *dst + v : v;
  }
}

}  // namespace tc

// ============================================================================
//                                  host side
// ============================================================================

using namespace tc;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*PFN_encodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                     cuuint32_t, cuuint32_t, const cuuint32_t*,
                                     CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled g_encode_tiled = nullptr;
static PFN_encodeIm2col g_encode_im2col = nullptr;
static bool g_tc_ok = false;

static bool load_driver() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q1, q2;
    void* f1 = nullptr;
    void* f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q1) !=
            cudaSuccess ||
        cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q2) !=
            cudaSuccess)
      return;
    g_encode_tiled = (PFN_encodeTiled)f1;
    g_encode_im2col = (PFN_encodeIm2col)f2;
    int dev = 0, major = 0, minor = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    g_tc_ok = g_encode_tiled && g_encode_im2col && major == 10 && minor == 0;
  });
  return g_tc_ok;
}

bool conv_tc_available() { return load_driver(); }

struct TcState {
  Workspace xt, ft, part, dyg, bpart, s2dT;
  // dy on the padded grid (dyg) is shared by the grid wgrad and the im2col
  // dgrad of one ck_conv_backward call: cached by (source, geometry, call id)
  const float* dyg_src = nullptr;
  uint64_t dyg_call = 0;
  int64_t dyg_key = 0;
};

static TcState* state(ck_handle* h) {
  if (!h->tc) h->tc = new TcState();
  return h->tc;
}

void conv_tc_release(ck_handle* h) {
  if (!h->tc) return;
  h->tc->xt.release();
  h->tc->ft.release();
  h->tc->part.release();
  h->tc->dyg.release();
  h->tc->bpart.release();
  h->tc->s2dT.release();
  delete h->tc;
  h->tc = nullptr;
}

static inline int rup(int v, int m) { return (v + m - 1) / m * m; }

// 2D tiled map over a row-major [outer][inner] fp32 matrix, box (32, box_outer), SW128.
static CUtensorMap map_2d(const float* base, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                          uint32_t box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 4};
  cuuint32_t box[2] = {32, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides,
                              box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Err(CK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// 4D im2col map over a pixel-major tensor (Cp, H, W, N).
static CUtensorMap map_im2col(const float* base, int Cp, int H, int W, int N, int lo_h, int lo_w,
                              int up_h, int up_w, int sh, int sw, int pixels,
                              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)Cp, (cuuint64_t)H, (cuuint64_t)W, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)Cp * 4, (cuuint64_t)Cp * H * 4, (cuuint64_t)Cp * H * W * 4};
  int lower[2] = {lo_h, lo_w};
  int upper[2] = {up_h, up_w};
  cuuint32_t es[4] = {1, (cuuint32_t)sh, (cuuint32_t)sw, 1};
  CUresult r = g_encode_im2col(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)base, dims, strides,
                               lower, upper, 32, (cuuint32_t)pixels, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Err(CK_ERR_CUDA, "cuTensorMapEncodeIm2col failed (" + std::to_string((int)r) + ")");
  return m;
}

static int pick_bn(int n) {
  // largest MMA N (multiple of 16, <= 256) that tiles n with little waste
  static const int force = knob("CK_TC_BN", 0);  // experiments
  if (force > 0 && force < n) return force;
  if (n <= 256) return rup(n, 16);
  const int cands[] = {256, 192, 128};
  int best = 128;
  double best_w = 1e9;
  for (int c : cands) {
    double waste = (double)rup(n, c) / n;
    if (waste < best_w - 1e-9) {
      best_w = waste;
      best = c;
    }
  }
  return best;
}

// Tile M: one or two M=128 MMAs per CTA (BM = 256 shares each B tile between
// two MMAs, halving the B traffic per FLOP).  For the implicit-GEMM convs
// (nt = N tiles x groups) pick the BM with the smaller modelled makespan:
// waves x per-tile work, with BM = 256 charged 25 % when its accumulators
// cannot be double-buffered in TMEM (2 x 2 x BN > 512 columns: the epilogue
// then serialises with the next tile) and BM = 128 charged 8 % for its extra
// B traffic.  FC / wgrad GEMMs: BM = 256 only when TMEM stays double-buffered.
static int pick_bm(int64_t M, int BN, bool conv = false, int nt = 1) {
  static const int mode = knob("CK_TC_BM", 0);  // experiments
  if (mode == 256) return M >= 4096 ? 256 : 128;
  if (mode == 128) return 128;
  if (M < 4096) return 128;
  if (!conv) return BN <= 128 ? 256 : 128;
  const int64_t t256 = (M + 255) / 256 * nt, t128 = (M + 127) / 128 * nt;
  const double c256 = (double)((t256 + 147) / 148) * 2.0 * (BN <= 128 ? 1.0 : 1.25);
  const double c128 = (double)((t128 + 147) / 148) * 1.08;
  return c128 < c256 ? 128 : 256;
}

template <int AK, int BK>
static void launch(const CUtensorMap& a, const CUtensorMap& b, GemmParams p, int grid_m,
                   int grid_n, int grid_z, cudaStream_t s) {
  (void)grid_m;
  (void)grid_n;
  static const int exp = knob("CK_TC_EXP", 0);
  p.exp = exp;  // (read by the kernel only in CK_EXPERIMENTS builds)
  static const int snake = knob("CK_EPI_SNAKE", 1);
  p.snake = snake;
  if (p.BM != 128 && p.BM != 256) p.BM = 128;
  p.groups = grid_z / p.splits;
  const int halves = p.BM / 128;
  p.nacc = (2 * halves * p.BN <= 512) ? 2 : 1;
  if (p.kstage != 64) p.kstage = 32;
  const int stage_bytes = (p.BM + p.BN) * p.kstage * 4;
  // grid-writing epilogues (gx) stage their rows in shared memory
  const int estage_bytes = p.gx ? kEpiWarps * 32 * 32 * 4 : 0;
  const int budget = 227 * 1024 - 1024 - 256 - estage_bytes;
  p.stages = std::min(8, budget / stage_bytes);
  p.estage = estage_bytes > 0;
  const size_t smem = 1024 + (size_t)p.stages * stage_bytes + 256 + estage_bytes;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(tc_gemm_kernel<AK, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    configured = true;
  }
  const int tiles = ((p.M + p.BM - 1) / p.BM) * ((p.N + p.BN - 1) / p.BN) * grid_z;
  const int grid = std::min(tiles, 148);
  count_launch();
  count_tc_launch();
  static const int mprof = knob("CK_TC_PROF", 0);
  static unsigned long long* mbuf = nullptr;
  if (mprof && !mbuf) cudaMalloc(&mbuf, (148 * 8 + 512) * sizeof(unsigned long long));
  p.prof = mprof ? mbuf : nullptr;
  if (mprof) cudaMemsetAsync(mbuf, 0, (148 * 8 + 512) * sizeof(unsigned long long), s);
  KernelProfiler* pr = (g_prof && g_prof->on && !g_prof->label.empty()) ? g_prof : nullptr;
  KernelProfiler::Rec rec;
  if (pr) {
    rec.label = pr->label;
    rec.flops = pr->flops;
    pr->label.clear();
    cudaEventCreate(&rec.a);
    cudaEventCreate(&rec.b);
    cudaEventRecord(rec.a, s);
  }
  ck::pdl_launch(tc_gemm_kernel<AK, BK>, grid, kThreads, smem, s, a, b, p);
  if (mprof) {  // debug: where the MMA thread of each CTA spent its time
    unsigned long long hbuf[148 * 8 + 512];
    cudaStreamSynchronize(s);
    cudaMemcpy(hbuf, mbuf, sizeof(hbuf), cudaMemcpyDeviceToHost);
    double tot = 0, wt = 0, wf = 0, kb = 0, ew = 0, eb = 0, ns = 0;
    int n = 0;
    for (int i = 0; i < 148; ++i)
      if (hbuf[i * 8]) {
        tot += hbuf[i * 8]; wt += hbuf[i * 8 + 1]; wf += hbuf[i * 8 + 2]; kb += hbuf[i * 8 + 3];
        ns += hbuf[i * 8 + 4]; ew += hbuf[i * 8 + 5]; eb += hbuf[i * 8 + 6];
        ++n;
      }
    if (n)
      fprintf(stderr, "[gemm<%d,%d>] M=%d N=%d K=%d BM=%d BN=%d S=%d nacc=%d ctas=%d: mma-thread %.0f cyc "
              "%.1f us (%.0f MHz), %.0f cyc/kblock, wait tempty %.1f%% full %.1f%%; epilogue busy %.0f "
              "wait %.0f cyc\n", AK, BK, p.M, p.N, p.K, p.BM, p.BN, p.stages, p.nacc, n, tot / n,
              ns / n / 1e3, tot / ns * 1e3, tot / kb, 100 * wt / tot, 100 * wf / tot, eb / n, ew / n);
    if (mprof == 2) {  // per-kblock issue-start deltas of CTA 0
      fprintf(stderr, "  kblock deltas:");
      for (int i = 1; i < 512 && hbuf[148 * 8 + i]; ++i)
        fprintf(stderr, " %lld", (long long)(hbuf[148 * 8 + i] - hbuf[148 * 8 + i - 1]));
      fprintf(stderr, "\n");
    }
  }
  if (pr) {
    cudaEventRecord(rec.b, s);
    pr->recs.push_back(rec);
  }
}

// label + algorithmic FLOP (2*N*OH*OW*K*fh*fw*C/g) of a conv pass for the profiler
static void prof_conv(const char* pass, const ConvDims& d) {
  if (!g_prof || !g_prof->on) return;
  char buf[160];
  snprintf(buf, sizeof buf, "%s %dx%dx%d->%d f%dx%d s%d g%d N%d", pass, d.H, d.W, d.C, d.K, d.fh,
           d.fw, d.sh, d.groups, d.N);
  prof_next(buf, 2.0 * d.N * d.OH * d.OW * (double)d.K * d.fh * d.fw * d.Cg);
}

static int split_for(int tiles, int kblocks) {
  // fill ~1 wave of 148 SMs; keep >= 8 k-blocks per split
  static const int force = knob("CK_TC_SPLITS", 0);
  if (force > 0) return std::min(force, std::max(1, kblocks));
  int s = 1;
  while (tiles * s * 2 <= 148 && kblocks / (s * 2) >= 8) s *= 2;
  return s;
}

// wgrad: reductions over ~1e5-1e6 pixels; split so every SM has ~2 tiles.
// Split-K factor for the wgrad GEMMs: minimise the persistent kernel's
// makespan, waves * (K blocks per split + a per-tile fill/epilogue cost of
// ~24 K blocks), over splits that keep >= 16 K blocks per split.
static int wgrad_splits_for(int tiles, int kblocks) {
  static const int force = knob("CK_TC_SPLITS", 0);
  if (force > 0) return std::min(force, std::max(1, kblocks));
  const int max_sp = std::max(1, std::min(64, kblocks / 16));
  int best = 1;
  int64_t best_cost = INT64_MAX;
  for (int sp = 1; sp <= max_sp; ++sp) {
    const int64_t waves = ((int64_t)tiles * sp + 147) / 148;
    const int64_t cost = waves * ((kblocks + sp - 1) / sp + 24);
    if (cost < best_cost) {
      best_cost = cost;
      best = sp;
    }
  }
  return best;
}

static void* grow(Workspace& w, size_t bytes, cudaStream_t s) {
  void* p = w.get(bytes, s);
  if (!p) throw Err(CK_ERR_CUDA, "workspace allocation failed");
  return p;
}

static void to_grid_pm(const float* x, float* xg, int H, int W, int C, int N, int Cg, int Cgp,
                       int groups, int Hg, int Wg, int oh, int ow, cudaStream_t s);

// pixel-major [n][w][h][cp] = the padding-free grid
static void to_pm(const float* x, float* xt, int H, int W, int C, int N, int Cg, int Cgp,
                  int groups, cudaStream_t s) {
  to_grid_pm(x, xt, H, W, C, N, Cg, Cgp, groups, H, W, 0, 0, s);
}

static void to_grid_pm(const float* x, float* xg, int H, int W, int C, int N, int Cg, int Cgp,
                       int groups, int Hg, int Wg, int oh, int ow, cudaStream_t s) {
  count_launch();
  grid_pm_launch(x, xg, H, W, C, N, Cg, Cgp, groups, Hg, Wg, oh, ow, nullptr, nullptr, nullptr, s);
}

static bool halo_enabled() {
  // Off by default: measured slower than the im2col kernels on AlexNet
  // (junk grid rows + per-tap filter streaming), kept for experiments.
  return knob("CK_TC_HALO", 0) != 0;  // experiments builds only (read per call)
}

static CUtensorMap encode_tiled(const float* base, int rank, const cuuint64_t* dims,
                                const cuuint64_t* strides_bytes, const cuuint32_t* box,
                                CUtensorMapSwizzle swz);

// Operands of one halo_conv_kernel launch: the padded grid (A) and the
// filter bank laid [row][tap][Cgp] (B), with `rows` output channels per group.
struct HaloConv {
  const float* grid;
  int Cp, Hg, Wg, N;   // grid [N][Wg][Hg][Cp]
  const float* filt;
  int Cgp, taps, fh, fw, rows, groups;
  int ohv, owv;        // valid output extent on the grid
};

// Whether halo_launch can run this shape (same sizing rules).
static bool halo_ok(int rows, int fh, int fw, int Hg) {
  if (!halo_enabled()) return false;
  const int BN = pick_bn(rows);
  if (BN > 256 || BN % 16) return false;
  const int arows = rup(256 + (fh - 1) + Hg * (fw - 1), 8);  // BM <= 256
  const int anbox = (arows + 255) / 256;
  const int stage_a = anbox * rup((arows + anbox - 1) / anbox, 8) * 128;
  return 227 * 1024 - 2048 - 2 * stage_a >= 2 * BN * 128;
}

// p carries the epilogue fields (epi, out, ld, img_stride, grp_col, bias, relu,
// acc, s2d_*); returns false when the shape does not fit the kernel.
static int env_int(const char* name, int dflt) { return knob(name, dflt); }

static bool halo_launch(const HaloConv& hc, GemmParams p, cudaStream_t s) {
#ifndef CK_EXPERIMENTS
  (void)hc;
  (void)p;
  (void)s;
  return false;
#else
  if (!halo_enabled()) return false;
  static const int bm_env = env_int("CK_HALO_BM", 256), sb_env = env_int("CK_HALO_SB", 3),
                   tt_env = env_int("CK_HALO_TT", 0), cs_env = env_int("CK_HALO_CS", 2),
                   bn_env = env_int("CK_HALO_BN", 0);
  const int BM = bm_env == 128 ? 128 : 256, halves = BM / 128;
  const int BN = bn_env > 0 && bn_env < hc.rows ? bn_env : pick_bn(hc.rows);
  if (BN > 256 || BN % 16) return false;
  const int maxshift = (hc.fh - 1) + hc.Hg * (hc.fw - 1);
  const int arows = rup(BM + maxshift, 8);
  const int anbox = (arows + 255) / 256;
  const int abox = rup((arows + anbox - 1) / anbox, 8);
  const int stage_a = anbox * abox * 128;
  const int budget = 227 * 1024 - 2048;
  const int SA = 2;
  const int bud_b = budget - SA * stage_a;
  int SB = sb_env;
  int tt_max = bud_b / (SB * BN * 128);
  if (tt_max < 1) {
    SB = 2;
    tt_max = bud_b / (SB * BN * 128);
  }
  if (tt_max < 1) return false;
  tt_max = std::min(tt_max, hc.taps);
  if (tt_env > 0) tt_max = std::min(tt_max, tt_env);
  const int ngroups = (hc.taps + tt_max - 1) / tt_max;
  int TT = (hc.taps + ngroups - 1) / ngroups;
  // clusters of 2 split every filter stage in two tap halves: TT even
  const int CS = (cs_env == 2 && tt_max >= 2) ? 2 : 1;
  if (CS == 2 && TT % 2) TT = TT + 1 <= tt_max ? TT + 1 : TT - 1;
  const int64_t rows_total = (int64_t)hc.N * hc.Hg * hc.Wg;
  if (rows_total + abox * anbox > INT32_MAX) return false;
  p.M = (int)rows_total;
  p.N = hc.rows;
  p.BM = BM;
  p.BN = BN;
  p.splits = 1;
  p.groups = hc.groups;
  p.nacc = (2 * halves * BN <= 512) ? 2 : 1;
  p.hg = hc.Hg;
  p.hw_grid = hc.Hg * hc.Wg;
  p.ohv = hc.ohv;
  p.owv = hc.owv;
  p.cchunks = hc.Cgp / 32;
  p.a_grp_c = hc.Cgp;
  p.b_grp_row = hc.rows;
  p.taps = hc.taps;
  p.fh = hc.fh;
  p.TT = TT;
  p.SA = SA;
  p.SB = SB;
  p.arows = arows;
  p.abox = abox;
  p.anbox = anbox;
  p.n_valid = hc.rows;
  CUtensorMap ta = map_2d(hc.grid, hc.Cp, (uint64_t)rows_total, hc.Cp, abox);
  cuuint64_t dims[3] = {(cuuint64_t)hc.Cgp, (cuuint64_t)hc.rows * hc.groups, (cuuint64_t)hc.taps};
  cuuint64_t strides[2] = {(cuuint64_t)hc.taps * hc.Cgp * 4, (cuuint64_t)hc.Cgp * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)BN, (cuuint32_t)(TT / CS)};
  CUtensorMap tb = encode_tiled(hc.filt, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
  const size_t smem = 1024 + (size_t)SA * stage_a + (size_t)SB * TT * BN * 128 + 256;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(halo_conv_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(halo_conv_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    configured = true;
  }
  const int tm = (p.M + BM - 1) / BM;
  const int items = ((tm + CS - 1) / CS) * ((p.N + BN - 1) / BN) * hc.groups;
  static const int prof = env_int("CK_HALO_PROF", 0);
  static unsigned long long* prof_buf = nullptr;
  if (prof && !prof_buf) cudaMalloc(&prof_buf, 148 * 4 * sizeof(unsigned long long));
  p.prof = prof ? prof_buf : nullptr;
  if (prof) cudaMemsetAsync(prof_buf, 0, 148 * 4 * sizeof(unsigned long long), s);
  struct ProfDump {
    unsigned long long* buf;
    cudaStream_t s;
    int M, N, BN, TT, SB;
    ~ProfDump() {
      if (!buf) return;
      unsigned long long h[148 * 4];
      cudaStreamSynchronize(s);
      cudaMemcpy(h, buf, sizeof(h), cudaMemcpyDeviceToHost);
      double tot = 0, wt = 0, wa = 0, wb = 0;
      int n = 0;
      for (int i = 0; i < 148; ++i)
        if (h[i * 4]) {
          tot += h[i * 4]; wt += h[i * 4 + 1]; wa += h[i * 4 + 2]; wb += h[i * 4 + 3]; ++n;
        }
      fprintf(stderr, "[halo] M=%d N=%d BN=%d TT=%d SB=%d ctas=%d mma-thread cycles %.0f: wait tempty %.1f%% fullA %.1f%% fullB %.1f%%\n",
              M, N, BN, TT, SB, n, tot / n, 100 * wt / tot, 100 * wa / tot, 100 * wb / tot);
    }
  } dump{prof ? prof_buf : nullptr, s, p.M, p.N, BN, TT, SB};
  count_launch();
  if (CS == 1) {
    ck::pdl_launch(halo_conv_kernel<1>, std::min(items, 148), kThreads, smem, s, ta, tb, p);
    return true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * std::min(items, 74));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, halo_conv_kernel<2>, ta, tb, p) != cudaSuccess)
    throw Err(CK_ERR_CUDA, "halo_conv_kernel cluster launch failed");
  return true;
#endif
}

// dy at (0, 0) of an Hg x Wg zero grid, pixel-major [n][Wg][Hg][groups*Kgp]:
// the wgrad A operand and (through im2col with negative corners) the dgrad
// input of one ck_conv_backward call -- transformed once per call.
// db from the per-(image, pixel tile) partials [rows][Cp], in two fixed-order
// stages (deterministic): grid_bias_part_k -- block (32 channels, row chunk
// of 8*RPW rows) -> part2[chunk][Cp]; grid_bias_finish_k sums the chunks.
// rows of bias partials per warp: at least 8, and few enough block chunks
// (<= 64) that the per-channel finish loop stays short
static inline int bias_rows_per_warp(int rows) { return std::max(8, (rows + 511) / 512); }
static inline int bias_chunks(int rows) {
  const int rpw = bias_rows_per_warp(rows);
  return (rows + 8 * rpw - 1) / (8 * rpw);
}
__global__ void grid_bias_part_k(const double* __restrict__ bpart, double* __restrict__ part2,
                                 int Cp, int rows, int rpw) {
  ck::pdl_entry();
  __shared__ double red[8][32];
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int cp = blockIdx.x * 32 + lane;
  const int r0 = blockIdx.y * 8 * rpw + warp * rpw;
  double t = 0;
  if (cp < Cp)
#pragma unroll 8
    for (int r = r0; r < r0 + rpw; ++r)
      if (r < rows) t += bpart[(int64_t)r * Cp + cp];
  red[warp][lane] = t;
  __syncthreads();
  if (warp == 0 && cp < Cp) {
    double u = 0;
    for (int w = 0; w < 8; ++w) u += red[w][lane];
    part2[(int64_t)blockIdx.y * Cp + cp] = u;
  }
}

__global__ void grid_bias_finish_k(const double* __restrict__ part2, float* db, int K, int Kg,
                                   int Kgp, int Cp, int chunks, int acc) {
  ck::pdl_entry();
  // one warp per channel: lanes sum strided chunks, then a fixed shuffle tree
  const int cp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (cp >= Cp) return;
  double u = 0;
  for (int c = lane; c < chunks; c += 32) u += part2[(int64_t)c * Cp + cp];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
  const int g = cp / Kgp, kl = cp - g * Kgp;
  if (lane == 0 && kl < Kg) {
    const int k = g * Kg + kl;
    if (k < K) db[k] = acc ? db[k] + (float)u : (float)u;
  }
}

// With db != nullptr the transform also reduces db[k] = sum over all dy
// pixels (conv.cpp:246-252), fused into the same read of dy.
// With relu_x != nullptr, dy is produced here: dy = relu_x > 0 ? relu_dy : 0
// (the engine's fused conv -> relu backward); the grid is built from it.
static int64_t dy_grid_key(const ConvDims& d, int Kgp, int groups, int Hg, int Wg) {
  return ((((int64_t)Hg * 4099 + Wg) * 65537 + d.K) * 131071 + d.N) * 1031 + Kgp * 17 + groups +
         ((int64_t)d.OH << 40) + ((int64_t)d.OW << 50);
}

static bool halo_enabled();
static bool shift_enabled();

static float* dy_grid(ck_handle* h, const float* dy, const ConvDims& d, int Kg, int Kgp,
                      int groups, int Hg, int Wg, cudaStream_t s, float* db = nullptr,
                      int db_acc = 0, const float* relu_x = nullptr,
                      const float* relu_dy = nullptr, bool skip_gout = false) {
  TcState* st = state(h);
  const int64_t key = dy_grid_key(d, Kgp, groups, Hg, Wg);
  if (h->pre_dyg && h->pre_dyg_src == dy && h->pre_dyg_key == key) {
    // built (gated, bias partials included) by the engine's previous layer
    if (db) {
      const int Cp = Kgp * groups, rows = h->pre_rows;
      const int chunks = bias_chunks(rows);
      double* part2 = (double*)grow(st->bpart, sizeof(double) * (size_t)chunks * Cp, s);
      count_launch(2);
      ck::pdl_launch(grid_bias_part_k, dim3((Cp + 31) / 32, chunks), 256, 0, s, h->pre_bpart, part2, Cp, rows,
                                                                     bias_rows_per_warp(rows));
      ck::pdl_launch(grid_bias_finish_k, (Cp * 32 + 255) / 256, 256, 0, s, part2, db, d.K, Kg, Kgp, Cp,
                                                                chunks, db_acc);
    }
    return h->pre_dyg;
  }
  float* buf = (float*)grow(st->dyg, sizeof(float) * (size_t)d.N * Hg * Wg * Kgp * groups, s);
  if (!db && st->dyg_src == dy && st->dyg_call == h->call && st->dyg_key == key) return buf;
  if (!relu_x) materialize_pending_dy(h, dy, s);  // rebuilding from dy: it must exist
  if (db) {
    const int Cp = Kgp * groups, nb = (Hg * Wg + 63) / 64;
    const int rows = d.N * nb, chunks = bias_chunks(rows);
    double* bpart =
        (double*)grow(st->bpart, sizeof(double) * ((size_t)rows + chunks) * Cp, s);
    double* part2 = bpart + (size_t)rows * Cp;
    count_launch(3);
    grid_pm_launch(relu_x ? relu_dy : dy, buf, d.OH, d.OW, d.K, d.N, Kg, Kgp, groups, Hg, Wg, 0,
                   0, bpart, relu_x, relu_x && !skip_gout ? const_cast<float*>(dy) : nullptr, s);
    ck::pdl_launch(grid_bias_part_k, dim3((Cp + 31) / 32, chunks), 256, 0, s, bpart, part2, Cp, rows,
                                                                   bias_rows_per_warp(rows));
    ck::pdl_launch(grid_bias_finish_k, (Cp * 32 + 255) / 256, 256, 0, s, part2, db, d.K, Kg, Kgp, Cp, chunks,
                                                              db_acc);
  } else {
    to_grid_pm(dy, buf, d.OH, d.OW, d.K, d.N, Kg, Kgp, groups, Hg, Wg, 0, 0, s);
  }
  st->dyg_src = dy;
  st->dyg_call = h->call;
  st->dyg_key = key;
  return buf;
}

// x on its zero-padded grid (Hg x Wg, x at (pt, pl)), pixel-major: the fprop
// im2col input and the wgrad B operand.  Inside a graph step the engine's
// per-layer ConvCache carries it from the forward to the weight gradient.
// Padded pixel-major grid of a stride-1 conv: x at (pt, pl) of an Hg x Wg
// image grid.  Adjacent columns share their zero halo (bottom pad of column j
// = top pad of column j+1; right pad of image n = left pad of image n+1), so
// Hg = H + max(pt, pb), Wg = W + max(pl, pr): every shifted read of x stays
// on zeros or in TMA zero fill, and the dy grid (dy at (0, 0), OH <= Hg) has
// fewer junk rows for the weight-gradient reduction.
static void grid_dims(const ConvDims& d, int& Hg, int& Wg) {
  const bool shared = std::min(d.pt, d.pb) < d.fh && std::min(d.pl, d.pr) < d.fw &&
                      !knob("CK_TC_FULLGRID", 0);
  Hg = d.H + (shared ? std::max(d.pt, d.pb) : d.pt + d.pb);
  Wg = d.W + (shared ? std::max(d.pl, d.pr) : d.pl + d.pr);
}

static int64_t x_grid_key(const ConvDims& d, int Cgp, int Hg, int Wg) {
  return (((((int64_t)Hg * 4099 + Wg) * 65537 + d.C) * 131071 + d.N) * 1031 + Cgp * 17 +
          d.groups) ^ ((int64_t)(d.pt * 64 + d.pl) << 52) ^ 0x1;
}

static float* x_grid(ck_handle* h, const float* x, const ConvDims& d, int Cgp, int Hg, int Wg,
                     cudaStream_t s) {
  ConvCache* c = h->conv_cache;
  const int64_t key = x_grid_key(d, Cgp, Hg, Wg);
  const size_t bytes = sizeof(float) * (size_t)d.N * Hg * Wg * Cgp * d.groups;
  float* buf = (float*)grow(c ? c->buf : state(h)->xt, bytes, s);
  if (c && c->valid && c->src == x && c->key == key) return buf;
  to_grid_pm(x, buf, d.H, d.W, d.C, d.N, d.Cg, Cgp, d.groups, Hg, Wg, d.pt, d.pl, s);
  if (c) {
    c->valid = true;
    c->src = x;
    c->key = key;
  }
  return buf;
}

static CUtensorMap encode_tiled(const float* base, int rank, const cuuint64_t* dims,
                                const cuuint64_t* strides_bytes, const cuuint32_t* box,
                                CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, (void*)base, dims,
                              strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Err(CK_ERR_CUDA, "cuTensorMapEncodeTiled (rank " + std::to_string(rank) + ") failed");
  return m;
}

// MN-major operand: matrix [K rows][MN cols], row pitch ld elements (MN
// contiguous).  With MN % 32 == 0 a 3D view {32, K, MN/32} loads a whole
// R-row tile (R/32 blocks of 32 k-rows x 128 B) in one box; otherwise R/32
// 2D boxes of 32 x 32.  Swizzle 128B_ATOM_32B = the UMMA SW128_32B layout.
static CUtensorMap map_mn(const float* base, uint64_t K, uint64_t MN, uint64_t ld, int R,
                          int* is3d, int ks = 32) {
  if (MN % 32 == 0) {
    *is3d = 1;
    cuuint64_t dims[3] = {32, K, MN / 32};
    cuuint64_t strides[2] = {ld * 4, 128};
    cuuint32_t box[3] = {32, (cuuint32_t)ks, (cuuint32_t)(R / 32)};
    return encode_tiled(base, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  }
  *is3d = 0;
  cuuint64_t dims[2] = {MN, K};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)ks};
  return encode_tiled(base, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

// ---- space-to-depth path for strided convolutions --------------------------
struct S2D {
  int s, U, V, Th, Tw, Cs, Csp;
};

static bool s2d_plan(const ConvDims& d, S2D& z) {
  if (d.sh != d.sw || d.sh < 2 || d.groups != 1) return false;
  if (d.pt || d.pb || d.pl || d.pr) return false;
  z.s = d.sh;
  z.U = (d.H + z.s - 1) / z.s;
  z.V = (d.W + z.s - 1) / z.s;
  z.Th = (d.fh + z.s - 1) / z.s;
  z.Tw = (d.fw + z.s - 1) / z.s;
  if (z.U - z.Th + 1 != d.OH || z.V - z.Tw + 1 != d.OW) return false;
  z.Cs = z.s * z.s * d.C;
  z.Csp = rup(z.Cs, 32);
  return d.K >= 16 && z.Cs >= 16;
}

static int blocks_for(int64_t total) { return (int)std::min<int64_t>((total + 255) / 256, 148 * 16); }

template <int AK, int BK>
static void launch(const CUtensorMap& a, const CUtensorMap& b, GemmParams p, int grid_m,
                   int grid_n, int grid_z, cudaStream_t s);

static void s2d_pm(const float* x, float* xt, const ConvDims& d, const S2D& z, cudaStream_t s) {
  count_launch();
  const int col_bytes = (int)sizeof(float) * d.C * z.s * z.U * z.s;  // one s2d column, all c
  const int VB = std::min(z.V, (44 * 1024) / col_bytes);
  if (VB >= 1)
    ck::pdl_launch(s2d_pm_strip_k, dim3((z.V + VB - 1) / VB, d.N), 256, (size_t)VB * col_bytes, s, 
        x, xt, d.H, d.W, d.C, z.s, z.U, z.V, z.Cs, z.Csp, VB);
  else
    ck::pdl_launch(s2d_pm_k, blocks_for((int64_t)d.N * z.U * z.V * z.Csp), 256, 0, s, 
        x, xt, d.H, d.W, d.C, d.N, z.s, z.U, z.V, z.Cs, z.Csp);
}

// the space-to-depth input (a pad-free grid of pitch U), cached like x_grid
static float* x_s2d(ck_handle* h, const float* x, const ConvDims& d, const S2D& z,
                    cudaStream_t s) {
  ConvCache* c = h->conv_cache;
  const int64_t key = ((((int64_t)z.U * 4099 + z.V) * 65537 + d.C) * 131071 + d.N) * 1031 +
                      z.Csp * 17 + z.s + 0x2;
  float* buf = (float*)grow(c ? c->buf : state(h)->xt,
                            sizeof(float) * (size_t)d.N * z.U * z.V * z.Csp, s);
  if (c && c->valid && c->src == x && c->key == key) return buf;
  s2d_pm(x, buf, d, z, s);
  if (c) {
    c->valid = true;
    c->src = x;
    c->key = key;
  }
  return buf;
}

// Off by default: correct, but on AlexNet the junk grid rows (25-33 %) cost
// more than the cheaper tiled boxes save -- these GEMMs are bound by shared-
// memory operand traffic, not TMA issue.  CK_TC_SHIFT=1.
static bool shift_enabled() {
  return knob("CK_TC_SHIFT", 0) != 0;  // experiments builds only (read per call)
}

// Stride-1 implicit GEMM on a zero-padded pixel-major grid G[N*Hg*Wg][Cp]
// with tiled (not im2col) TMA: output grid row q accumulates
//   sum_{tap, c} G[q + base_shift + fi + Hg*fj, c] * F[row][tap][c],
// the A tile of a K block being BM consecutive grid rows shifted by the tap --
// one 3D box of KS/32 channel chunks (half the TMA time of an im2col box per
// byte, tools/tma_probe.cu).  Rows whose (u, v) lie outside (ohv, owv) are
// junk and dropped by the epilogue; p carries the epilogue fields.
static void shift_conv(const float* G, int Cp, int Hg, int Wg, int N, int base_shift,
                       const float* F, int Cgp, int taps, int fh, int rows, int groups, int ohv,
                       int owv, GemmParams p, cudaStream_t s) {
#ifndef CK_EXPERIMENTS
  (void)G; (void)Cp; (void)Hg; (void)Wg; (void)N; (void)base_shift; (void)F; (void)Cgp;
  (void)taps; (void)fh; (void)rows; (void)groups; (void)ohv; (void)owv; (void)p; (void)s;
  throw Err(CK_ERR_ARG, "shifted-grid kernels are built only with CK_EXPERIMENTS");
#else
  const int64_t M = (int64_t)N * Hg * Wg;
  p.M = (int)M;
  p.N = rows;
  p.K = taps * Cgp;
  p.BN = pick_bn(rows);
  p.splits = 1;
  p.BM = pick_bm(M, p.BN, true, (rows + p.BN - 1) / p.BN * groups);
  const int KS = (Cgp % 64 == 0 && 3 * (p.BM + p.BN) * 64 * 4 <= 224 * 1024) ? 64 : 32;
  p.kstage = KS;
  p.Hp = Hg;
  p.base_shift = base_shift;
  p.fh = fh;
  p.cchunks = Cgp / 32;
  p.a_grp_c = Cgp;
  p.b_grp_mn = rows;
  p.hg = Hg;
  p.hw_grid = Hg * Wg;
  p.ohv = ohv;
  p.owv = owv;
  p.n_valid = rows;
  cuuint64_t adims[3] = {32, (cuuint64_t)M, (cuuint64_t)(Cp / 32)};
  cuuint64_t astr[2] = {(cuuint64_t)Cp * 4, 128};
  cuuint32_t abox[3] = {32, (cuuint32_t)p.BM, (cuuint32_t)(KS / 32)};
  CUtensorMap ta = encode_tiled(G, 3, adims, astr, abox, CU_TENSOR_MAP_SWIZZLE_128B);
  const int64_t kt = (int64_t)taps * Cgp;
  cuuint64_t bdims[3] = {32, (cuuint64_t)rows * groups, (cuuint64_t)(kt / 32)};
  cuuint64_t bstr[2] = {(cuuint64_t)kt * 4, 128};
  cuuint32_t bbox[3] = {32, (cuuint32_t)p.BN, (cuuint32_t)(KS / 32)};
  CUtensorMap tb = encode_tiled(F, 3, bdims, bstr, bbox, CU_TENSOR_MAP_SWIZZLE_128B);
  launch<OP_SHIFT_K, OP_TILED_K3>(ta, tb, p, 0, 0, groups, s);
#endif
}

static void s2d_fprop(ck_handle* h, const float* x, const float* f, const float* bias, float* y,
                      const ConvDims& d, const S2D& z, int relu, cudaStream_t s) {
  TcState* st = state(h);
  const int taps = z.Th * z.Tw;
  float* xt = x_s2d(h, x, d, z, s);
  float* ft = (float*)grow(st->ft, sizeof(float) * (size_t)d.K * taps * z.Csp, s);
  count_launch();
  ck::pdl_launch(s2d_repack_fprop_k, blocks_for((int64_t)d.K * taps * z.Csp), 256, 0, s, 
      f, ft, d.fh, d.fw, d.C, d.K, z.s, z.Th, z.Tw, z.Csp, d.fsc, d.fsk);
  if (halo_ok(d.K, z.Th, z.Tw, z.U)) {
    // the s2d pixel-major tensor is already a (pad-free) grid of pitch U
    GemmParams p{};
    p.epi = EPI_PIX; p.out = y; p.out2 = h->fuse_relu; p.ld = (int64_t)d.OH * d.OW;
    p.img_stride = (int64_t)d.K * d.OH * d.OW; p.grp_col = d.K;
    p.bias = bias; p.relu = relu; p.acc = 0;
    HaloConv hc{xt, z.Csp, z.U, z.V, d.N, ft, z.Csp, taps, z.Th, z.Tw, d.K, 1, d.OH, d.OW};
    if (halo_launch(hc, p, s)) return;
  }
  if (shift_enabled()) {
    GemmParams p{};
    p.epi = EPI_PIX; p.out = y; p.out2 = h->fuse_relu; p.ld = (int64_t)d.OH * d.OW;
    p.img_stride = (int64_t)d.K * d.OH * d.OW; p.grp_col = d.K;
    p.bias = bias; p.relu = relu; p.acc = 0;
    shift_conv(xt, z.Csp, z.U, z.V, d.N, 0, ft, z.Csp, taps, z.Th, d.K, 1, d.OH, d.OW, p, s);
    return;
  }
  GemmParams p{};
  p.M = d.N * d.OH * d.OW; p.N = d.K; p.K = taps * z.Csp; p.BN = pick_bn(d.K); p.splits = 1;
  p.OH = d.OH; p.OW = d.OW; p.sh = 1; p.sw = 1; p.pt = 0; p.pl = 0; p.fh = z.Th;
  p.cchunks = z.Csp / 32;
  p.last_k = z.Cs % 32 ? (z.Cs % 32 + 7) / 8 : 4;
  p.epi = EPI_PIX; p.out = y; p.out2 = h->fuse_relu; p.ld = (int64_t)d.OH * d.OW;
  p.img_stride = (int64_t)d.K * d.OH * d.OW; p.epi_OHW = d.OH * d.OW;
  p.bias = bias; p.relu = relu; p.n_valid = d.K;
  p.BM = pick_bm(p.M, p.BN, true, (d.K + p.BN - 1) / p.BN);
  CUtensorMap ta = map_im2col(xt, z.Csp, z.U, z.V, d.N, 0, 0, -(z.Th - 1), -(z.Tw - 1), 1, 1, p.BM);
  CUtensorMap tb = map_2d(ft, (uint64_t)taps * z.Csp, d.K, (uint64_t)taps * z.Csp, p.BN);
  launch<OP_IM2COL_K, OP_TILED_K>(ta, tb, p, (p.M + 127) / 128, (d.K + p.BN - 1) / p.BN, 1, s);
}

// dx[n][c][j][i] (+)= T[((a + s*b) * C + c) * M + (n * V + v) * U + u] with
// (i, j) = (s*u + a, s*v + b): the s2d dgrad result, written by the GEMM
// epilogue column-major (coalesced along the s2d pixels), scattered back to
// the HWCN image.  One block row per (n, c, j); along i each warp reads s
// planes of 32/s consecutive u -- whole 32-byte sectors.
__global__ void __launch_bounds__(256) s2d_unpack_k(const float* __restrict__ T,
                                                    float* __restrict__ dx, int H, int W, int C,
                                                    int s, int U, int V, int64_t M, int rows,
                                                    int acc) {
  ck::pdl_entry();
  constexpr int R = 8;  // image rows (n, c, j) per block, loads of all in flight together
  // per-row source plane base (32-bit index math, once per block row)
  __shared__ int64_t base[R];
  if (threadIdx.x < R) {
    const int row = blockIdx.x * R + threadIdx.x;  // (n * C + c) * W + j
    if (row < rows) {
      const int j = row % W, nc = row / W;
      const int c = nc % C, n = nc / C;
      const int v = j / s, b = j - v * s;
      base[threadIdx.x] = (int64_t)(s * b * C + c) * M + ((int64_t)n * V + v) * U;
    }
  }
  __syncthreads();
  const int64_t plane = (int64_t)C * M;  // T stride of one sub-pixel row a
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    const int u = i / s, a = i - u * s;
    const int64_t off = a * plane + u;
    float val[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
      val[r] = blockIdx.x * R + r < rows ? __ldg(T + base[r] + off) : 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = blockIdx.x * R + r;
      if (row < rows) {
        float* d = dx + (int64_t)row * H + i;
        *d = acc ? __fadd_rn(*d, val[r]) : val[r];
      }
    }
  }
}

static void s2d_dgrad(ck_handle* h, const float* dy, const float* f, float* dx, const ConvDims& d,
                      const S2D& z, int acc, cudaStream_t s) {
  TcState* st = state(h);
  const int taps = z.Th * z.Tw;
  const int Kp = rup(d.K, 32);
  float* gt = (float*)grow(st->ft, sizeof(float) * (size_t)z.Cs * taps * Kp, s);
  count_launch();
  ck::pdl_launch(s2d_repack_dgrad_k, blocks_for((int64_t)z.Cs * taps * Kp), 256, 0, s, 
      f, gt, d.fh, d.fw, d.C, d.K, Kp, z.s, z.Th, z.Tw, d.fsc, d.fsk);
  const int Hq = d.OH + 2 * (z.Th - 1), Wq = d.OW + 2 * (z.Tw - 1);
  if (halo_ok(z.Cs, z.Th, z.Tw, Hq)) {
    // dx_s2d = stride-1 conv of dy zero-padded by (Th-1, Tw-1) with the
    // flipped bank, on a grid of pitch Hq; EPI_S2D scatters back to x.
    float* dyg = (float*)grow(st->dyg, sizeof(float) * (size_t)d.N * Hq * Wq * Kp, s);
    st->dyg_src = nullptr;
    materialize_pending_dy(h, dy, s);  // this path reads dy itself
    to_grid_pm(dy, dyg, d.OH, d.OW, d.K, d.N, d.K, Kp, 1, Hq, Wq, z.Th - 1, z.Tw - 1, s);
    GemmParams p{};
    p.epi = EPI_S2D; p.out = dx;
    p.s2d = z.s; p.s2d_U = z.U; p.s2d_H = d.H; p.s2d_W = d.W; p.s2d_C = d.C;
    p.acc = acc;
    HaloConv hc{dyg, Kp, Hq, Wq, d.N, gt, Kp, taps, z.Th, z.Tw, z.Cs, 1, z.U, z.V};
    if (halo_launch(hc, p, s)) return;
  }
  // im2col over dy at (0, 0) of the U x V grid (shared with the wgrad): the
  // negative corner supplies the top/left padding, the grid's zero rows the rest
  float* dyt = dy_grid(h, dy, d, d.K, Kp, 1, z.U, z.V, s);
  if (shift_enabled()) {
    // output s2d pixel (u, v) at grid row u + U*v reads dy rows shifted by
    // fi - (Th-1) + U*(fj - (Tw-1)); the grid's zero rows/columns are the padding
    GemmParams p{};
    p.epi = EPI_S2D; p.out = dx;
    p.s2d = z.s; p.s2d_U = z.U; p.s2d_H = d.H; p.s2d_W = d.W; p.s2d_C = d.C;
    p.acc = acc;
    shift_conv(dyt, Kp, z.U, z.V, d.N, -((z.Th - 1) + z.U * (z.Tw - 1)), gt, Kp, taps, z.Th, z.Cs,
               1, z.U, z.V, p, s);
    return;
  }
  // GEMM over the s2d pixels into T[c'][m] (column-major, coalesced epilogue
  // stores), then one pass scatters T back to the HWCN image
  GemmParams p{};
  p.M = d.N * z.U * z.V; p.N = z.Cs; p.K = taps * Kp; p.BN = pick_bn(z.Cs); p.splits = 1;
  p.OH = z.U; p.OW = z.V; p.sh = 1; p.sw = 1; p.pt = z.Th - 1; p.pl = z.Tw - 1; p.fh = z.Th;
  p.cchunks = Kp / 32;
  float* T = (float*)grow(st->s2dT, sizeof(float) * (size_t)p.M * z.Cs, s);
  p.epi = EPI_LINEAR; p.out = T; p.ld = p.M; p.acc = 0; p.n_valid = z.Cs;
  p.BM = pick_bm(p.M, p.BN, true, (z.Cs + p.BN - 1) / p.BN);
  CUtensorMap ta = map_im2col(dyt, Kp, z.U, z.V, d.N, -(z.Th - 1), -(z.Tw - 1), -(z.Th - 1),
                              -(z.Tw - 1), 1, 1, p.BM);
  CUtensorMap tb = map_2d(gt, (uint64_t)taps * Kp, z.Cs, (uint64_t)taps * Kp, p.BN);
  launch<OP_IM2COL_K, OP_TILED_K>(ta, tb, p, (p.M + 127) / 128, (z.Cs + p.BN - 1) / p.BN, 1, s);
  count_launch();
  const int rows = d.N * d.C * d.W;
  ck::pdl_launch(s2d_unpack_k, (rows + 7) / 8, d.H <= 128 ? 128 : 256, 0, s, T, dx, d.H, d.W, d.C, z.s, z.U,
                                                                z.V, (int64_t)p.M, rows, acc);
}

static void s2d_pm(const float* x, float* xt, const ConvDims& d, const S2D& z, cudaStream_t s);

// Weight gradient on a padded grid (stride-1 conv; x at its padding offset in
// an Hg x Wg grid, dy at (0, 0) of the same grid with zeros elsewhere):
//   part[s][g][(tap, c)][k] = sum_{grid rows q of split s} dYg[q, k] Xg[q + fi + Hg*fj, c]
// A = dYg read MN-major (one 3D box of BM channels x 32 rows); B = Xg rows
// shifted by the tap, one 3D box per tap of b_rows channels (tiled TMA, no
// im2col).  Junk grid rows carry dy = 0.  Returns the split count.
// Roles swapped (M = (tap, c), N = k) when the filter count leaves most of a
// 128-row tile empty (VGG's 64 filters: half; AlexNet conv4's 192: a third)
// and the (tap, c) rows fill whole tiles: partials part[g][k][(tap, c)]
// (wgrad_finish_k swapped).
static bool wgrad_swap(int Kg, int taps, int Cgp) {
  static const int on = knob("CK_TC_WSWAP", 1);  // experiments builds: A/B switch
  // (the MN-major dy operand needs BN = Kg % 32 == 0: its TMA boxes are 32
  // columns wide, a narrower tail would leave the stage's expected bytes short)
  if (!on || Kg > 256 || Kg < 64 || Kg % 32) return false;
  const double waste_k = (double)rup(Kg, 128) / Kg;
  const double waste_t = (double)rup(taps * Cgp, 128) / (taps * Cgp);
  return waste_k >= 1.3 && waste_t <= 1.15;
}

static int grid_wgrad_swapped(ck_handle* h, const float* xg, int Cp, int Cgp, const float* dyg,
                              int Kp, int Kgp, int Kg, int groups, int N, int Hg, int Wg, int fh,
                              int fw, float** part_out, int64_t* per_out, cudaStream_t s) {
  TcState* st = state(h);
  const int taps = fh * fw;
  const int Mtot = taps * Cgp;  // GEMM M = (tap, c) per group
  const int BN = rup(Kg, 16);
  const int BM = pick_bm(Mtot, BN);
  const int a_rows = std::gcd(Cgp, 128);
  const int64_t rows = (int64_t)N * Hg * Wg;
  static const int ks_env = knob("CK_TC_WKS", 64);
  const int KS = ks_env == 32 ? 32 : 64;
  const int kblocks = (int)((rows + KS - 1) / KS);
  const int splits = wgrad_splits_for(((Mtot + BM - 1) / BM) * groups, kblocks);
  const int64_t per_grp = (int64_t)Mtot * Kg;
  const int64_t per = per_grp * groups;
  float* part = (float*)grow(st->part, sizeof(float) * per * splits, s);
  GemmParams p{};
  p.M = Mtot; p.N = Kg; p.K = kblocks * KS; p.BN = BN; p.BM = BM; p.splits = splits;
  p.kstage = KS;
  p.Hp = Hg; p.fh = fh; p.taps = taps; p.cchunks = Cgp / 32; p.a_rows = a_rows;
  p.a_grp_c = Cgp;
  p.b_grp_mn = Kgp;
  // raw partials: part[s*per + g*per_grp + k*Mtot + (tap, c)]
  p.epi = EPI_LINEAR; p.out = part; p.ld = Mtot; p.grp_out = per_grp; p.n_valid = Kg;
  p.split_stride = per;
  cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(Cp / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)Cp * 4, 128};
  cuuint32_t box[3] = {32, (cuuint32_t)KS, (cuuint32_t)(a_rows / 32)};
  CUtensorMap ta = encode_tiled(xg, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  CUtensorMap tb = map_mn(dyg, (uint64_t)rows, Kp, Kp, BN, &p.b_mn3d, KS);
  launch<OP_SHIFT_MN, OP_TILED_MN>(ta, tb, p, 0, 0, groups * splits, s);
  *part_out = part;
  *per_out = per;
  return splits;
}

static int grid_wgrad(ck_handle* h, const float* xg, int Cp, int Cgp, const float* dyg, int Kp,
                      int Kgp, int Kg, int groups, int N, int Hg, int Wg, int fh, int fw,
                      float** part_out, int64_t* per_out, cudaStream_t s) {
  TcState* st = state(h);
  const int taps = fh * fw;
  const int Ntot = taps * Cgp;  // GEMM N = (tap, c) per group
  // N tile: a whole tap's channels when they fit; else the multiple of 32 that
  // wastes the fewest padded columns (conv1's s2d 576 = 3 x 192, conv2's 1600 =
  // 10 x 160), larger on ties
  int BN = Cgp;
  if (Cgp < 128 || Cgp > 256) {
    static const int force_bn = knob("CK_TC_WBN", 0);
    BN = 0;
    int best = INT32_MAX;
    for (int c = 256; c >= 64; c -= 32) {
      const int padded = rup(Ntot, c);
      if (padded < best) {
        best = padded;
        BN = c;
      }
    }
    if (force_bn > 0 && force_bn % 32 == 0 && force_bn <= 256) BN = force_bn;
  }
  const int b_rows = std::min(256, std::gcd(Cgp, BN));
  const int BM = pick_bm(Kg, BN);
  const int64_t rows = (int64_t)N * Hg * Wg;
  // 64 grid rows per stage: half the TMA boxes per FLOP (both operands MN-major)
  static const int ks_env = knob("CK_TC_WKS", 64);
  const int KS = ks_env == 32 ? 32 : 64;
  const int kblocks = (int)((rows + KS - 1) / KS);
  const int splits = wgrad_splits_for(((Kg + BM - 1) / BM) * ((Ntot + BN - 1) / BN) * groups,
                                      kblocks);
  const int64_t per_grp = (int64_t)Ntot * Kg;
  const int64_t per = per_grp * groups;
  float* part = (float*)grow(st->part, sizeof(float) * per * splits, s);
  GemmParams p{};
  p.M = Kg; p.N = Ntot; p.K = kblocks * KS; p.BN = BN; p.BM = BM; p.splits = splits;
  p.kstage = KS;
  p.Hp = Hg; p.fh = fh; p.taps = taps; p.cchunks = Cgp / 32; p.b_rows = b_rows;
  p.a_grp_mn = Kgp;
  p.b_grp_c = Cgp;
  // raw partials: part[s*per + g*per_grp + n*Kg + k]
  p.epi = EPI_LINEAR; p.out = part; p.ld = Kg; p.grp_out = per_grp; p.n_valid = Ntot;
  p.split_stride = per;
  CUtensorMap ta = map_mn(dyg, (uint64_t)rows, Kp, Kp, BM, &p.a_mn3d, KS);
  cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(Cp / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)Cp * 4, 128};
  cuuint32_t box[3] = {32, (cuuint32_t)KS, (cuuint32_t)(b_rows / 32)};
  CUtensorMap tb = encode_tiled(xg, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  launch<OP_TILED_MN, OP_SHIFT_MN>(ta, tb, p, 0, 0, groups * splits, s);
  *part_out = part;
  *per_out = per;
  return splits;
}

// Strided wgrad through space-to-depth: the grid wgrad over the s2d input (a
// pad-free grid of pitch U, dy at (0, 0) of it), then the s2d filter scatter.
static void s2d_wgrad(ck_handle* h, const float* x, const float* dy, float* df, const ConvDims& d,
                      const S2D& z, int acc, cudaStream_t s) {
  const int Kp = rup(d.K, 32);
  float* xt = x_s2d(h, x, d, z, s);
  float* dyg = dy_grid(h, dy, d, d.K, Kp, 1, z.U, z.V, s);
  float* part;
  int64_t per;
  const bool swapped = wgrad_swap(d.K, z.Th * z.Tw, z.Csp);
  const int splits =
      swapped ? grid_wgrad_swapped(h, xt, z.Csp, z.Csp, dyg, Kp, Kp, d.K, 1, d.N, z.U, z.V, z.Th,
                                   z.Tw, &part, &per, s)
              : grid_wgrad(h, xt, z.Csp, z.Csp, dyg, Kp, Kp, d.K, 1, d.N, z.U, z.V, z.Th, z.Tw,
                           &part, &per, s);
  count_launch();
  ck::pdl_launch(s2d_wgrad_finish_k, blocks_for((int64_t)d.K * d.fh * d.fw * d.C), 256, 0, s, 
      part, df, d.fh, d.fw, d.C, d.K, z.s, z.Th, z.Csp, splits, per, acc, d.fsc, d.fsk,
      swapped ? 1 : 0, (int64_t)z.Th * z.Tw * z.Csp);
}

static bool is_fc(const ConvDims& d) {
  return d.OH == 1 && d.OW == 1 && d.fh == d.H && d.fw == d.W && d.pt == 0 && d.pb == 0 &&
         d.pl == 0 && d.pr == 0 && d.groups == 1 && d.fsc == 1;
}

// ---------------------------------------------------------------- fprop ----
static bool conv_tc_forward_impl(ck_handle* h, const float* x, const float* f, const float* bias,
                                 float* y, const ConvDims& d, int relu, cudaStream_t s) {
  if (!load_driver()) return false;
  prof_conv("fprop", d);
  const int Kg = d.Kg();
  if (is_fc(d)) {
    // Y[k, n] = sum_q F[q, k] X[q, n]   (A = filters, B = images, both K-major)
    const int Q = d.H * d.W * d.C;
    if (Q % 4) return false;  // (K < 128 filters: the A box's rows past K are TMA zero fill)
    // short reductions with a wave of 128 x 64 tiles (AlexNet fc7): no split-K
    // partials / finish pass (measured fc7 0.034 -> 0.029 ms; fc6's 9216-long
    // K keeps split-K, tools/fc_sweep.sh)
    const bool wave64 = d.N > 64 && Q <= 4096 &&
                        (int64_t)((d.K + 127) / 128) * ((d.N + 63) / 64) >= 128;
    const int BN = wave64 ? 64 : pick_bn(std::min(d.N, 256));
    const int gm = (d.K + 127) / 128, gn = (d.N + BN - 1) / BN;
    const int splits = wave64 ? 1 : split_for(gm * gn, rup(Q, 32) / 32);
    GemmParams p{};
    p.M = d.K; p.N = d.N; p.K = rup(Q, 32); p.BN = BN; p.splits = splits;
    p.epi = EPI_LINEAR; p.ld = d.K; p.n_valid = d.N; p.relu = relu; p.bias = bias;
    p.out2 = h->fuse_relu;
    p.BM = wave64 ? 128 : pick_bm(p.M, p.BN);
    CUtensorMap ta = map_2d(f, Q, d.K, Q, p.BM);
    CUtensorMap tb = map_2d(x, Q, d.N, Q, BN);
    if (splits > 1) {
      const int64_t per = (int64_t)d.K * d.N;
      float* part = (float*)grow(state(h)->part, sizeof(float) * per * splits, s);
      p.out = part; p.split_stride = per;
      launch<OP_TILED_K, OP_TILED_K>(ta, tb, p, gm, gn, splits, s);
      count_launch();
      ck::pdl_launch(splitk_finish_k, std::min<int64_t>((per + 255) / 256, 148 * 8), 256, 0, s, 
          part, y, d.K, d.N, d.K, splits, per, bias, relu, 0, h->fuse_relu);
    } else {
      p.out = y;
      launch<OP_TILED_K, OP_TILED_K>(ta, tb, p, gm, gn, 1, s);
    }
    return true;
  }
  if ((d.sh > 1 || d.sw > 1) && d.Cg < 16) {
    S2D z;
    if (!s2d_plan(d, z)) return false;
    s2d_fprop(h, x, f, bias, y, d, z, relu, s);
    return true;
  }
  // (any channel count: groups are padded to 32 channels; the MMAs of a tap's
  // all-zero K steps are skipped (last_k), the epilogue stores n < n_valid)
  const int Cgp = rup(d.Cg, 32), Cp = Cgp * d.groups;
  const int taps = d.fh * d.fw;
  if (d.pt > 127 || d.pl > 127 || d.fh > 128 || d.fw > 128) return false;
  TcState* st = state(h);
  float* ft = (float*)grow(st->ft, sizeof(float) * (size_t)d.K * taps * Cgp, s);
  count_launch();
  ck::pdl_launch(repack_fprop_k, std::min<int64_t>(((int64_t)d.K * taps * Cgp + 255) / 256, 148 * 8), 256, 0, s, 
      f, ft, d.fh, d.fw, d.Cg, Cgp, d.K, d.fsc, d.fsk);
  int Hg, Wg;
  grid_dims(d, Hg, Wg);
  if (d.sh == 1 && d.sw == 1 && halo_ok(Kg, d.fh, d.fw, Hg)) {
    // halo kernel over the zero-padded pixel-major grid (Hg x Wg per image)
    float* xg = (float*)grow(st->xt, sizeof(float) * (size_t)d.N * Hg * Wg * Cp, s);
    to_grid_pm(x, xg, d.H, d.W, d.C, d.N, d.Cg, Cgp, d.groups, Hg, Wg, d.pt, d.pl, s);
    GemmParams p{};
    p.epi = EPI_PIX; p.out = y; p.out2 = h->fuse_relu; p.ld = (int64_t)d.OH * d.OW;
    p.img_stride = (int64_t)d.K * d.OH * d.OW; p.grp_col = Kg;
    p.bias = bias; p.relu = relu; p.acc = 0;
    HaloConv hc{xg, Cp, Hg, Wg, d.N, ft, Cgp, taps, d.fh, d.fw, Kg, d.groups, d.OH, d.OW};
    if (halo_launch(hc, p, s)) return true;
  }
  // stride 1: im2col over the padded grid (shared with the wgrad); else over
  // the compact pixel-major tensor with the padding in the im2col corners
  const bool on_grid = d.sh == 1 && d.sw == 1;
  float* xt;
  if (on_grid) {
    xt = x_grid(h, x, d, Cgp, Hg, Wg, s);
    if (shift_enabled()) {
      GemmParams p{};
      p.epi = EPI_PIX; p.out = y; p.out2 = h->fuse_relu; p.ld = (int64_t)d.OH * d.OW;
      p.img_stride = (int64_t)d.K * d.OH * d.OW; p.grp_col = Kg;
      p.bias = bias; p.relu = relu; p.acc = 0;
      shift_conv(xt, Cp, Hg, Wg, d.N, 0, ft, Cgp, taps, d.fh, Kg, d.groups, d.OH, d.OW, p, s);
      return true;
    }
  } else {
    xt = (float*)grow(st->xt, sizeof(float) * (size_t)d.N * d.H * d.W * Cp, s);
    to_pm(x, xt, d.H, d.W, d.C, d.N, d.Cg, Cgp, d.groups, s);
  }
  GemmParams p{};
  p.M = d.N * d.OH * d.OW;
  p.N = Kg;
  p.K = taps * Cgp;
  p.BN = pick_bn(Kg);
  p.splits = 1;
  p.OH = d.OH; p.OW = d.OW; p.sh = d.sh; p.sw = d.sw; p.pt = d.pt; p.pl = d.pl; p.fh = d.fh;
  p.cchunks = Cgp / 32;
  p.last_k = d.Cg % 32 ? (d.Cg % 32 + 7) / 8 : 4;
  p.a_grp_c = Cgp;
  p.b_grp_mn = Kg;
  p.epi = EPI_PIX; p.out = y; p.out2 = h->fuse_relu; p.ld = (int64_t)d.OH * d.OW;
  p.img_stride = (int64_t)d.K * d.OH * d.OW; p.grp_col = Kg; p.epi_OHW = d.OH * d.OW;
  p.bias = bias; p.relu = relu; p.acc = 0; p.n_valid = Kg;
  p.BM = pick_bm(p.M, p.BN, true, (Kg + p.BN - 1) / p.BN * d.groups);
  if (on_grid) p.pt = p.pl = 0;
  if (h->next_xg && h->fuse_relu && Kg % 32 == 0 &&
      h->next_xg_plan.bytes / sizeof(float) < (size_t(1) << 31)) {
    // engine: also write relu(y) into the consumer conv's x grid
    const XGridPlan& xp = h->next_xg_plan;
    p.gx = h->next_xg;
    p.gx_Hg = xp.Hg; p.gx_Wg = xp.Wg; p.gx_Cp = xp.Cgp * xp.groups; p.gx_Cg = xp.Cg;
    p.gx_Cgp = xp.Cgp; p.gx_pt = xp.pt; p.gx_pl = xp.pl; p.gx_OH = d.OH;
    h->next_xg_done = true;
  }
  // on the grid the output extent is (H + pt + pb) - fh + 1 whatever the grid
  // pitch: rows read past a shared-halo grid's column end are TMA zero fill
  CUtensorMap ta = on_grid ? map_im2col(xt, Cp, Hg, Wg, d.N, 0, 0,
                                        (d.H + d.pt + d.pb - Hg) - (d.fh - 1),
                                        (d.W + d.pl + d.pr - Wg) - (d.fw - 1), 1,
                                        1, p.BM)
                           : map_im2col(xt, Cp, d.H, d.W, d.N, -d.pt, -d.pl, d.pb - (d.fh - 1),
                                        d.pr - (d.fw - 1), d.sh, d.sw, p.BM);
  CUtensorMap tb = map_2d(ft, (uint64_t)taps * Cgp, d.K, (uint64_t)taps * Cgp, p.BN);
  launch<OP_IM2COL_K, OP_TILED_K>(ta, tb, p, (p.M + 127) / 128, (Kg + p.BN - 1) / p.BN, d.groups,
                                  s);
  return true;
}

// With h->fuse_relu set (graph engine, conv -> relu) every forward epilogue
// also writes relu(y) there; fuse_relu_done tells the engine it happened.
bool conv_tc_forward(ck_handle* h, const float* x, const float* f, const float* bias, float* y,
                     const ConvDims& d, int relu, cudaStream_t s) {
  const bool ok = conv_tc_forward_impl(h, x, f, bias, y, d, relu, s);
  if (ok && h->fuse_relu) h->fuse_relu_done = true;
  return ok;
}

// ---------------------------------------------------------------- dgrad ----
bool conv_tc_dgrad(ck_handle* h, const float* dy, const float* f, float* dx, const ConvDims& d,
                   int acc, cudaStream_t s) {
  if (!load_driver()) return false;
  prof_conv("dgrad", d);
  const int Kg = d.Kg();
  if (is_fc(d)) {
    // dX[q, n] = sum_k F[q, k] dY[k, n]: A = F read MN-major in place
    // (F[q + Q*k], q contiguous), B = dY K-major ([n][k]).
    const int Q = d.H * d.W * d.C;
    if (Q % 4 || d.K % 4) return false;
    // a wave of 128 x 128 tiles without split-K (AlexNet fc6: 72 x 2 tiles;
    // measured 0.051 -> 0.041 ms, tools/fc_sweep.sh)
    const bool wave128 = d.N > 128 && (int64_t)((Q + 127) / 128) * ((d.N + 127) / 128) >= 128;
    const int BN = wave128 ? 128 : pick_bn(std::min(d.N, 256));
    const int gm = (Q + 127) / 128, gn = (d.N + BN - 1) / BN;
    const int splits = wave128 ? 1 : split_for(gm * gn, rup(d.K, 32) / 32);
    GemmParams p{};
    p.M = Q; p.N = d.N; p.K = rup(d.K, 32); p.BN = BN; p.splits = splits;
    p.epi = EPI_LINEAR; p.ld = Q; p.n_valid = d.N; p.acc = acc;
    p.BM = wave128 ? 128 : pick_bm(p.M, p.BN);
    CUtensorMap ta = map_mn(f, d.K, Q, Q, p.BM, &p.a_mn3d);
    materialize_pending_dy(h, dy, s);  // this path reads dy itself
    CUtensorMap tb = map_2d(dy, d.K, d.N, d.K, BN);  // dY as [n][k]
    if (splits > 1) {
      const int64_t per = (int64_t)Q * d.N;
      float* part = (float*)grow(state(h)->part, sizeof(float) * per * splits, s);
      p.out = part; p.split_stride = per;
      launch<OP_TILED_MN, OP_TILED_K>(ta, tb, p, gm, gn, splits, s);
      count_launch();
      ck::pdl_launch(splitk_finish_k, std::min<int64_t>((per + 255) / 256, 148 * 8), 256, 0, s, 
          part, dx, Q, d.N, Q, splits, per, nullptr, 0, acc, nullptr);
    } else {
      p.out = dx;
      launch<OP_TILED_MN, OP_TILED_K>(ta, tb, p, gm, gn, 1, s);
    }
    return true;
  }
  // stride-1 conv of dy with the flipped bank, padding fh-1-pt (SPEC.md:151 adjoint)
  if (d.sh != 1 || d.sw != 1) {
    S2D z;
    if (!s2d_plan(d, z)) return false;
    s2d_dgrad(h, dy, f, dx, d, z, acc, s);
    return true;
  }
  // (any channel count: groups are padded to 32 channels; the MMAs of a tap's
  // all-zero K steps are skipped (last_k), the epilogue stores n < n_valid)
  if (d.pt > d.fh - 1 || d.pb > d.fh - 1 || d.pl > d.fw - 1 || d.pr > d.fw - 1) return false;
  const int Kgp = rup(Kg, 32), Kp = Kgp * d.groups;
  const int taps = d.fh * d.fw;
  TcState* st = state(h);
  static const int blk_on = knob("CK_TC_DBLK", 1);  // experiments builds: A/B switch
  // (5 x 5 filters and up: the block window's zero taps cost (f+1)^2 / f^2 more
  // MMAs, 1.44x at 5 x 5 but 1.78x at 3 x 3; large layers only)
  if (blk_on && d.Cg % 16 == 0 && d.Cg <= 64 && d.fh >= 5 && d.fw >= 5 && d.fh <= 15 &&
      d.fw <= 15 && !h->prev_dyg && d.H >= 2 && d.W >= 2 &&
      (int64_t)d.N * d.H * d.W >= (1 << 17)) {
    // few channels per group (AlexNet conv2: 48): the MMA N = Cg is too narrow
    // for the operand traffic it costs.  Compute 2 x 2 output blocks per GEMM
    // row instead: N = 4 Cg, K over the (fh+1) x (fw+1) dy window of a block
    // (im2col with traversal stride 2), 4x fewer A rows -- the window costs
    // (fh+1)(fw+1) / (fh fw) more MMAs; the EPI_S2D epilogue scatters the
    // block to dx.
    const int th = d.fh + 1, tw = d.fw + 1, taps6 = th * tw;
    const int qt = d.fh - 1 - d.pt, ql = d.fw - 1 - d.pl;
    float* gb = (float*)grow(st->ft, sizeof(float) * (size_t)d.groups * 4 * d.Cg * taps6 * Kgp, s);
    count_launch();
    ck::pdl_launch(repack_dgrad_blk_k,
                   std::min<int64_t>(((int64_t)d.groups * 4 * d.Cg * taps6 * Kgp + 255) / 256, 148 * 8),
                   256, 0, s, f, gb, d.fh, d.fw, d.Cg, Kg, Kgp, d.groups, d.fsc, d.fsk);
    int Hg, Wg;
    grid_dims(d, Hg, Wg);
    float* dyt = dy_grid(h, dy, d, Kg, Kgp, d.groups, Hg, Wg, s);
    const int Ha = (d.H + 1) / 2, Wa = (d.W + 1) / 2;
    GemmParams p{};
    p.M = d.N * Ha * Wa;
    p.N = 4 * d.Cg;
    p.K = taps6 * Kgp;
    p.BN = 4 * d.Cg;
    p.splits = 1;
    p.OH = Ha; p.OW = Wa; p.sh = 2; p.sw = 2; p.pt = qt; p.pl = ql; p.fh = th;
    p.cchunks = Kgp / 32;
    p.last_k = Kg % 32 ? (Kg % 32 + 7) / 8 : 4;
    p.a_grp_c = Kgp;
    p.b_grp_mn = 4 * d.Cg;
    p.epi = EPI_S2D; p.out = dx; p.s2d = 2; p.s2d_U = Ha; p.s2d_H = d.H; p.s2d_W = d.W;
    p.s2d_C = d.Cg; p.s2d_Ct = d.C; p.grp_col = d.Cg; p.epi_OHW = Ha * Wa;
    p.acc = acc; p.n_valid = 4 * d.Cg;
    p.BM = pick_bm(p.M, p.BN, true, d.groups);
    CUtensorMap ta = map_im2col(dyt, Kp, Hg, Wg, d.N, -qt, -ql, 2 * Ha - 1 - Hg - qt,
                                2 * Wa - 1 - Wg - ql, 2, 2, p.BM);
    CUtensorMap tb = map_2d(gb, (uint64_t)taps6 * Kgp, (uint64_t)d.groups * 4 * d.Cg,
                            (uint64_t)taps6 * Kgp, p.BN);
    launch<OP_IM2COL_K, OP_TILED_K>(ta, tb, p, (p.M + 127) / 128, 1, d.groups, s);
    return true;
  }
  float* gt = (float*)grow(st->ft, sizeof(float) * (size_t)d.C * taps * Kgp, s);
  count_launch();
  ck::pdl_launch(repack_dgrad_k, std::min<int64_t>(((int64_t)d.C * taps * Kgp + 255) / 256, 148 * 8), 256, 0, s, 
      f, gt, d.fh, d.fw, d.Cg, Kg, Kgp, d.groups, d.fsc, d.fsk);
  const int qt = d.fh - 1 - d.pt, qb = d.fh - 1 - d.pb, ql = d.fw - 1 - d.pl, qr = d.fw - 1 - d.pr;
  const int Hq = d.OH + qt + qb, Wq = d.OW + ql + qr;
  if (halo_ok(d.Cg, d.fh, d.fw, Hq)) {
    // halo kernel: dy zero-padded by (fh-1-pt, ...) on a grid of pitch Hq,
    // convolved with the flipped bank; the valid rows are the H x W of dx.
    float* dyg = (float*)grow(st->dyg, sizeof(float) * (size_t)d.N * Hq * Wq * Kp, s);
    st->dyg_src = nullptr;
    materialize_pending_dy(h, dy, s);  // this path reads dy itself
    to_grid_pm(dy, dyg, d.OH, d.OW, d.K, d.N, Kg, Kgp, d.groups, Hq, Wq, qt, ql, s);
    GemmParams p{};
    p.epi = EPI_PIX; p.out = dx; p.ld = (int64_t)d.H * d.W;
    p.img_stride = (int64_t)d.C * d.H * d.W; p.grp_col = d.Cg;
    p.bias = nullptr; p.relu = 0; p.acc = acc;
    HaloConv hc{dyg, Kp, Hq, Wq, d.N, gt, Kgp, taps, d.fh, d.fw, d.Cg, d.groups, d.H, d.W};
    if (halo_launch(hc, p, s)) return true;
  }
  // dy on the wgrad's zero grid (Hg x Wg, dy at (0, 0); shared within the
  // call): the negative im2col corners supply the top/left padding, the grid's
  // zero rows the bottom/right
  int Hg, Wg;
  grid_dims(d, Hg, Wg);
  float* dyt = dy_grid(h, dy, d, Kg, Kgp, d.groups, Hg, Wg, s);
  if (shift_enabled()) {
    // dx (i, j) at grid row i + Hg*j reads dy rows shifted by fi - qt + Hg*(fj - ql)
    GemmParams p{};
    p.epi = EPI_PIX; p.out = dx; p.ld = (int64_t)d.H * d.W;
    p.img_stride = (int64_t)d.C * d.H * d.W; p.grp_col = d.Cg;
    p.bias = nullptr; p.relu = 0; p.acc = acc;
    shift_conv(dyt, Kp, Hg, Wg, d.N, -(qt + Hg * ql), gt, Kgp, taps, d.fh, d.Cg, d.groups, d.H,
               d.W, p, s);
    return true;
  }
  GemmParams p{};
  p.M = d.N * d.H * d.W;
  p.N = d.Cg;
  p.K = taps * Kgp;
  p.BN = pick_bn(d.Cg);
  p.splits = 1;
  p.OH = d.H; p.OW = d.W; p.sh = 1; p.sw = 1; p.pt = qt; p.pl = ql; p.fh = d.fh;
  p.cchunks = Kgp / 32;
  p.last_k = Kg % 32 ? (Kg % 32 + 7) / 8 : 4;
  p.a_grp_c = Kgp;
  p.b_grp_mn = d.Cg;
  p.epi = EPI_PIX; p.out = dx; p.ld = (int64_t)d.H * d.W;
  p.img_stride = (int64_t)d.C * d.H * d.W; p.grp_col = d.Cg; p.epi_OHW = d.H * d.W;
  p.bias = nullptr; p.relu = 0; p.acc = acc; p.n_valid = d.Cg;
  p.BM = pick_bm(p.M, p.BN, true, (d.Cg + p.BN - 1) / p.BN * d.groups);
  if (h->prev_dyg && !acc && d.Cg % 32 == 0) {
    // engine, conv -> relu -> this conv: also write the conv below's
    // relu-gated dy grid and its bias partials (ck_handle.hpp prev_dyg)
    const GridPlan& gp = h->prev_dyg_plan;
    if (gp.Kg % 32 == 0 && gp.Kgp == gp.Kg && gp.Kg * gp.groups == d.C && gp.OH == d.H &&
        gp.OW == d.W && (int64_t)d.N * gp.Hg * gp.Wg * gp.Kgp * gp.groups < (1ll << 31)) {
      p.gx = h->prev_dyg;
      p.gx_Hg = gp.Hg; p.gx_Wg = gp.Wg; p.gx_Cp = gp.Kgp * gp.groups; p.gx_Cg = gp.Kg;
      p.gx_Cgp = gp.Kgp; p.gx_pt = 0; p.gx_pl = 0; p.gx_OH = d.H;
      p.gx_gate = h->prev_gate;
      p.gx_bpart = h->prev_bpart;
      p.dg_skip = knob("CK_DG_SKIP", 0);
      h->prev_dyg_done = true;
    }
  }
  CUtensorMap ta = map_im2col(dyt, Kp, Hg, Wg, d.N, -qt, -ql, d.H - Hg - qt, d.W - Wg - ql, 1, 1,
                              p.BM);
  CUtensorMap tb = map_2d(gt, (uint64_t)taps * Kgp, d.C, (uint64_t)taps * Kgp, p.BN);
  launch<OP_IM2COL_K, OP_TILED_K>(ta, tb, p, (p.M + 127) / 128, (d.Cg + p.BN - 1) / p.BN,
                                  d.groups, s);
  return true;
}

// Bias gradient fused into the dy-grid transform that the dgrad / wgrad of
// the same ck_conv_backward call then reuse.  False when the shape does not
// use the grid (FC layers, strided convs without space-to-depth).
// Mirrors the envelopes of conv_tc_bias / conv_tc_wgrad / conv_tc_dgrad: true
// iff all three read dy only through dy_grid (no fallback, no experimental
// path that transforms dy itself).
// Mirrors conv_tc_forward_impl / conv_tc_wgrad: true iff the forward reads x
// only through x_grid on the padded grid (stride 1, TF32, no experimental
// path) -- so a producer may write that grid (and mark the consumer's cache).
bool conv_tc_xgrid_plan(const ConvDims& d, XGridPlan* xp) {
  if (!load_driver() || is_fc(d) || halo_enabled() || shift_enabled()) return false;
  if (d.sh != 1 || d.sw != 1) return false;
  if (d.pt > 127 || d.pl > 127 || d.fh > 128 || d.fw > 128) return false;
  if (d.pt > d.fh - 1 || d.pb > d.fh - 1 || d.pl > d.fw - 1 || d.pr > d.fw - 1) return false;
  grid_dims(d, xp->Hg, xp->Wg);
  xp->Cg = d.Cg;
  xp->Cgp = rup(d.Cg, 32);
  xp->groups = d.groups;
  xp->pt = d.pt;
  xp->pl = d.pl;
  xp->key = x_grid_key(d, xp->Cgp, xp->Hg, xp->Wg);
  xp->bytes = sizeof(float) * (size_t)d.N * xp->Hg * xp->Wg * xp->Cgp * d.groups;
  return true;
}

bool conv_tc_grid_plan(const ConvDims& d, GridPlan* gp) {
  if (!load_driver() || is_fc(d) || halo_enabled() || shift_enabled()) return false;
  const int Kg = d.Kg();
  if (d.sh == 1 && d.sw == 1) {
    // (any channel count: channels are padded to 32 per group, last_k skips the
    // all-zero K steps of a tap's padded chunk)
    if (d.pt > d.fh - 1 || d.pb > d.fh - 1 || d.pl > d.fw - 1 || d.pr > d.fw - 1) return false;
    if (d.pt > 127 || d.pl > 127 || d.fh > 128 || d.fw > 128) return false;
    grid_dims(d, gp->Hg, gp->Wg);
    gp->Kg = Kg;
    gp->Kgp = rup(Kg, 32);
    gp->groups = d.groups;
  } else {
    S2D z;
    if (!s2d_plan(d, z)) return false;
    gp->Hg = z.U;
    gp->Wg = z.V;
    gp->Kg = d.K;
    gp->Kgp = rup(d.K, 32);
    gp->groups = 1;
  }
  gp->OH = d.OH;
  gp->OW = d.OW;
  gp->key = dy_grid_key(d, gp->Kgp, gp->groups, gp->Hg, gp->Wg);
  gp->bytes = sizeof(float) * (size_t)d.N * gp->Hg * gp->Wg * gp->Kgp * gp->groups;
  return true;
}

bool conv_tc_bias(ck_handle* h, const float* dy, float* db, const ConvDims& d, int acc,
                  cudaStream_t s, const float* relu_x, const float* relu_dy, bool skip_gout) {
  if (!load_driver() || is_fc(d)) return false;
  const int Kg = d.Kg();
  if (d.sh == 1 && d.sw == 1) {
    // (any channel count: channels are padded to 32 per group, last_k skips the
    // all-zero K steps of a tap's padded chunk)
    int Hg, Wg;
    grid_dims(d, Hg, Wg);
    dy_grid(h, dy, d, Kg, rup(Kg, 32), d.groups, Hg, Wg, s, db, acc, relu_x, relu_dy, skip_gout);
    return true;
  }
  S2D z;
  if (!s2d_plan(d, z)) return false;
  dy_grid(h, dy, d, d.K, rup(d.K, 32), 1, z.U, z.V, s, db, acc, relu_x, relu_dy, skip_gout);
  return true;
}

// ---------------------------------------------------------------- wgrad ----
bool conv_tc_wgrad(ck_handle* h, const float* x, const float* dy, float* df, const ConvDims& d,
                   int acc, cudaStream_t s) {
  if (!load_driver()) return false;
  prof_conv("wgrad", d);
  const int Kg = d.Kg();
  if (is_fc(d)) {
    // dF[q, k] = sum_n X[q, n] dY[k, n]: both operands read MN-major in place
    // (X[q + Q*n], dY[k + K*n]); the reduction runs over the batch.
    const int Q = d.H * d.W * d.C;
    if (Q % 4 || d.K % 4) return false;
    const int BN = d.K >= 256 ? 256 : rup(d.K, 32);
    const int gm = (Q + 127) / 128, gn = (d.K + BN - 1) / BN;
    GemmParams p{};
    p.M = Q; p.N = d.K; p.K = rup(d.N, 32); p.BN = BN; p.splits = 1;
    p.epi = EPI_LINEAR; p.ld = Q; p.n_valid = d.K; p.acc = acc; p.out = df;
    p.BM = pick_bm(p.M, p.BN);
    CUtensorMap ta = map_mn(x, d.N, Q, Q, p.BM, &p.a_mn3d);
    materialize_pending_dy(h, dy, s);  // this path reads dy itself
    CUtensorMap tb = map_mn(dy, d.N, d.K, d.K, BN, &p.b_mn3d);
    launch<OP_TILED_MN, OP_TILED_MN>(ta, tb, p, gm, gn, 1, s);
    return true;
  }
  // dF[k, (tap, c)] = sum_q dY[q, k] X[q + tap, c] over all output pixels q:
  // A = dY pixel-major, read MN-major ([q][k], k contiguous); B = X pixel-major
  // through im2col boxes (32 pixels x 32 channels of one tap), also MN-major.
  // Split-K over the pixels; partials reduced by wgrad_finish_k.
  if (d.sh != 1 || d.sw != 1) {
    S2D z;
    if (!s2d_plan(d, z)) return false;
    s2d_wgrad(h, x, dy, df, d, z, acc, s);
    return true;
  }
  // (any channel count: groups are padded to 32 channels; the MMAs of a tap's
  // all-zero K steps are skipped (last_k), the epilogue stores n < n_valid)
  if (d.pt > 127 || d.pl > 127 || d.fh > 128 || d.fw > 128) return false;
  const int Cgp = rup(d.Cg, 32), Cp = Cgp * d.groups;
  const int Kgp = rup(Kg, 32), Kp = Kgp * d.groups;
  const int taps = d.fh * d.fw;
  int Hg, Wg;
  grid_dims(d, Hg, Wg);
  float* xg = x_grid(h, x, d, Cgp, Hg, Wg, s);
  float* dyg = dy_grid(h, dy, d, Kg, Kgp, d.groups, Hg, Wg, s);
  float* part;
  int64_t per;
  const bool swapped = wgrad_swap(Kg, taps, Cgp);
  const int splits =
      swapped ? grid_wgrad_swapped(h, xg, Cp, Cgp, dyg, Kp, Kgp, Kg, d.groups, d.N, Hg, Wg, d.fh,
                                   d.fw, &part, &per, s)
              : grid_wgrad(h, xg, Cp, Cgp, dyg, Kp, Kgp, Kg, d.groups, d.N, Hg, Wg, d.fh, d.fw,
                           &part, &per, s);
  const int64_t total = (int64_t)d.groups * Kg * taps * d.Cg;
  count_launch();
  ck::pdl_launch(wgrad_finish_k, std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, s, 
      part, df, d.fh, d.fw, d.Cg, Cgp, Kg, d.groups, splits, per, d.fsc, d.fsk, acc,
      swapped ? 1 : 0);
  return true;
}

}  // namespace ck
