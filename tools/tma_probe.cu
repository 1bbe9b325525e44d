// TMA load throughput probe: 148 CTAs (one per SM) stream boxes of a
// pixel-major tensor [N][W][H][C=128] into a 4-stage shared-memory ring (no
// compute) and report aggregate GB/s for tiled-2D and im2col boxes of
// various pixel counts.  The tensor is 64 MB (L2 resident after the first
// pass) or 1 GB (HBM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe.bin tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: tiled 2D {32 ch, R px}; mode 1: im2col {32 ch, R px}, offsets (fi, fj) cycling
__global__ void stream_k(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap map2,
                         int mode, int R, int boxes_per_stage, int R2, int iters, int64_t npix, int H, int W,
                         int N, int S, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[8];
  const int stage_bytes = boxes_per_stage * R * 128 * (mode == 4 ? R2 : 1) + (mode == 2 || mode == 3 ? R2 * 128 : 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t pix = (int64_t)blockIdx.x * 4099 * R % npix;
  for (int it = 0; it < iters + S; ++it) {
    const int s = it % S;
    if (it >= S) {  // wait for the stage issued S iterations ago
      const uint32_t ph = ((it - S) / S) & 1;
      asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                   ::"r"(su32(&full[s])), "r"(ph) : "memory");
    }
    if (it >= iters) continue;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes) : "memory");
    if (mode == 2 || mode == 3) {  // second operand: one tiled box of R2 rows
      uint8_t* dst = sm + s * stage_bytes + boxes_per_stage * R * 128;
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(su32(dst)), "l"((uint64_t)&map2), "r"(su32(&full[s])), "r"(32), "r"((int)((pix * 7) % npix)) : "memory");
    }
    for (int b = 0; b < boxes_per_stage; ++b) {
      uint8_t* dst = sm + s * stage_bytes + b * R * 128 * (mode == 4 ? R2 : 1);
      const int c = (b % 4) * 32;
      if (mode == 4) {
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     ::"r"(su32(dst)), "l"((uint64_t)&map), "r"(su32(&full[s])), "r"(0), "r"((int)(pix % npix)), "r"(0) : "memory");
      } else if (mode == 0 || mode == 3) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(su32(dst)), "l"((uint64_t)&map), "r"(su32(&full[s])), "r"(c), "r"((int)(pix % npix)) : "memory");
      } else {
        const int64_t p = pix % npix;
        const int n = (int)(p / ((int64_t)H * W));
        const int r = (int)(p - (int64_t)n * H * W);
        const int w = r / H, h = r - w * H;
        const uint16_t fi = b % 3, fj = (b / 3) % 3;
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};"
                     ::"r"(su32(dst)), "l"((uint64_t)&map), "r"(su32(&full[s])), "r"(c), "r"(h - 1), "r"(w - 1), "r"(n), "h"(fi), "h"(fj) : "memory");
      }
    }
    pix += R;
  }
  if (blockIdx.x == 0) sink[0] = (unsigned long long)pix;
}

typedef CUresult (*EncTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  cudaFree(0);
  EncTiled enc_t; EncIm2col enc_i;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc_t, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&enc_i, cudaEnableDefault, &q);
  const int C = 128;
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaFuncSetAttribute(stream_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int H = 13, W = 13, N = 750;  // 65 MB: L2-resident
  const int64_t npix = (int64_t)N * H * W;
  float* buf; cudaMalloc(&buf, npix * C * 4); cudaMemset(buf, 0, npix * C * 4);
  auto tiled = [&](int R) {
    CUtensorMap m; cuuint32_t es[2] = {1, 1};
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)npix};
    cuuint64_t str[1] = {(cuuint64_t)C * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)R};
    enc_t(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
  };
  auto tiled3 = [&](int R, int D) {
    CUtensorMap m; cuuint32_t es[3] = {1, 1, 1};
    cuuint64_t dims[3] = {32, (cuuint64_t)npix, (cuuint64_t)(C / 32)};
    cuuint64_t str[2] = {(cuuint64_t)C * 4, 128};
    cuuint32_t box[3] = {32, (cuuint32_t)R, (cuuint32_t)D};
    enc_t(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
  };
  auto im2col = [&](int R) {
    CUtensorMap m; cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)W, (cuuint64_t)N};
    cuuint64_t str[3] = {(cuuint64_t)C * 4, (cuuint64_t)C * H * 4, (cuuint64_t)C * H * W * 4};
    int lo[2] = {-1, -1}, up[2] = {-1, -1};
    enc_i(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, buf, dims, str, lo, up, 32, R, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
  };
  struct Cfg { const char* name; int mode, R, bps, R2, S; };
  const Cfg cfgs[] = {
      {"tiled 128", 0, 128, 1, 0, 4}, {"tiled 128 S6", 0, 128, 1, 0, 6}, {"tiled 256 S4", 0, 256, 1, 0, 4},
      {"tiled 32x4 S6", 0, 32, 4, 0, 6}, {"tiled 32x8 S4", 0, 32, 8, 0, 4},
      {"im2col 128", 1, 128, 1, 0, 4}, {"im2col 128 S6", 1, 128, 1, 0, 6}, {"im2col 256 S4", 1, 256, 1, 0, 4},
      {"im2col 32x8 S4", 1, 32, 8, 0, 4},
      {"im2col128+tiled192 S4", 2, 128, 1, 192, 4}, {"im2col128+tiled128 S4", 2, 128, 1, 128, 4},
      {"im2col256+tiled192 S3", 2, 256, 1, 192, 3}, {"im2col256+tiled256 S3", 2, 256, 1, 256, 3},
      {"tiled128+tiled256 S4", 3, 128, 1, 256, 4}, {"tiled256+tiled256 S3", 3, 256, 1, 256, 3},
      {"im2col32x8+tiled128 S4", 2, 32, 8, 128, 4},
      {"tiled3d 256x2 S3", 4, 256, 1, 2, 3}, {"tiled3d 128x2 S4", 4, 128, 1, 2, 4},
      {"tiled3d 256x1 S4", 4, 256, 1, 1, 4}, {"tiled3d 128x4 S3", 4, 128, 1, 4, 3},
  };
  for (const Cfg& c : cfgs) {
    CUtensorMap m = c.mode == 4 ? tiled3(c.R, c.R2) : (c.mode == 1 || c.mode == 2) ? im2col(c.R) : tiled(c.R);
    CUtensorMap m2 = tiled(c.mode == 4 ? 32 : (c.R2 ? c.R2 : 32));
    const int stage_bytes = c.bps * c.R * 128 * (c.mode == 4 ? c.R2 : 1) + (c.mode == 2 || c.mode == 3 ? c.R2 * 128 : 0);
    const int iters = (int)((256LL << 20) / 148 / stage_bytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    stream_k<<<148, 32, c.S * stage_bytes + 1024>>>(m, m2, c.mode, c.R, c.bps, c.R2, iters, npix, H, W, N, c.S, sink);
    cudaEventRecord(e0);
    stream_k<<<148, 32, c.S * stage_bytes + 1024>>>(m, m2, c.mode, c.R, c.bps, c.R2, iters, npix, H, W, N, c.S, sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)iters * stage_bytes * 148;
    const double cyc_per_stage = ms * 1e-3 * 1.9e9 / iters;
    printf("%-24s stage %6d B: %7.1f GB/s  %5.1f B/clk/SM  %6.0f clk/stage\n", c.name, stage_bytes,
           bytes / ms / 1e6, bytes / (ms * 1e-3) / 148 / 1.9e9, cyc_per_stage);
  }
  return 0;
}
