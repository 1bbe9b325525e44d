// Probe: can a K-major SWIZZLE_128B UMMA operand start at an arbitrary ROW of
// a swizzled tile (start address + r0*128 B), i.e. can one halo tile feed
// several filter taps?  A is written as TMA would (row r at r*128, 16-B chunk
// c stored at c ^ (r & 7), tile base 1024-B aligned); the MMA reads rows
// r0 .. r0+127.  Variants: descriptor base_offset field = 0 or (r0 & 7).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/shift_probe.bin tools/shift_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 32, MR = M + 16;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t off_k(int r, int k) {
  return (uint32_t)(r * 128 + (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4);
}

__global__ void probe(const float* A, const float* B, float* D, int r0, int boff_mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;              // MR rows x 128 B
  uint8_t* sB = sm + 32768;      // N rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < MR * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    *(float*)(sA + off_k(m, k)) = A[m * K + k];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    *(float*)(sB + off_k(n, k)) = B[n * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < K / 8; ++j) {
      const uint32_t boff = boff_mode == 0 ? 0u : boff_mode == 1 ? (uint32_t)(r0 & 7) : (uint32_t)((8 - (r0 & 7)) & 7);
      const uint64_t da = sdesc(su32(sA) + r0 * 128 + j * 32, 16, 1024, boff);
      const uint64_t db = sdesc(su32(sB) + j * 32, 16, 1024, 0);
      const uint32_t acc = j > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = warp * 32 + (tid & 31);
    for (int j = 0; j < 8; ++j) D[m * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
  }
}

// Timing: 2048 MMAs (M=128, N=NT, K=8) from one thread with the A start at
// row r0; returns cycles per MMA.
template <int NT>
__global__ void mma_rate(int r0, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < 65536 / 4; e += blockDim.x) ((float*)sm)[e] = 0.001f * (e & 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t a = su32(sm), b = su32(sm + 32768);
    long long t0 = clock64();
    for (int i = 0; i < 2048; ++i) {
      const uint64_t da = sdesc(a + r0 * 128 + (i & 3) * 32, 16, 1024, 0);
      const uint64_t db = sdesc(b + (i & 3) * 32, 16, 1024, 0);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64();
    out[0] = (t1 - t0) / 2048;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
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

// Streaming variant: S stages of (A 16 KB = 128 rows x 32 k, B NT rows x 32 k),
// each MMA reads a different stage / k-slice, as in the GEMM mainloop.
template <int NT, int S, int CE = 0, int NACC = 1>
__global__ void mma_stream(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, bar2[8];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  const int stage = 16384 + NT * 128;
  if (tid < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2[tid])));
  for (int e = tid; e < S * stage / 4; e += blockDim.x) ((float*)sm)[e] = 0.001f * (e & 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    for (int i = 0; i < 2048; ++i) {
      const int st = (i / 4) % S, k = i & 3;
      const uint32_t a = su32(sm + st * stage), b = a + 16384;
      const uint64_t da = sdesc(a + k * 32, 16, 1024, 0);
      const uint64_t db = sdesc(b + k * 32, 16, 1024, 0);
      const uint32_t dacc = tmem + (uint32_t)(((i / 4) % NACC) * NT);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(dacc), "l"(da), "l"(db), "r"(idesc), "r"(1u));
      if (CE && (i % CE) == CE - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2[(i / CE) % 8])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64();
    out[0] = (t1 - t0) / 2048;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

// Full-chip variant: every SM streams `iters` MMAs over random operands;
// reports cycles/MMA and the effective SM clock (clock64 vs globaltimer).
// MODE 0: MMA thread only; 1: + 9 warps spinning on an mbarrier (try_wait);
// 2: + 8 warps streaming tcgen05.ld from the other half of TMEM;
// 3: + commit per 4 MMAs and a producer warp waiting/arriving a stage ring (as the GEMM).
template <int NT, int S, int MODE, int R = 4, int P = 4>
__global__ void mma_full(long long* out, int iters, int rnd) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar, spin, fullb[16], emptyb[16];
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid / 32;
  const int stage = 16384 + NT * 128;
  uint32_t h = 0x9e3779b9u * (tid + 1) + blockIdx.x;
  if (tid == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&spin)));
    for (int i = 0; i < 16; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&fullb[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&emptyb[i])));
    }
  }
  for (int e = tid; e < S * stage / 4; e += blockDim.x) {
    h ^= h << 13; h ^= h >> 17; h ^= h << 5;
    ((float*)sm)[e] = rnd ? ((int)(h & 0xffff) - 32768) * (1.0f / 32768) : 0.001f * (e & 7);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (MODE == 1 && warp >= 1) {
    asm volatile("{\n.reg .pred p;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}\n" ::"r"(su32(&spin)) : "memory");
  }
  if (MODE == 2 && warp >= 2) {
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[32];
      const uint32_t taddr = tmem + 256 + ((uint32_t)((warp & 3) * 32) << 16) + (warp / 4 - 0) * 32;
      CK_LD32(r, taddr);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
      __syncwarp();
    }
    if (acc == 12345) out[1000] = acc;
  }
  if ((MODE == 3 || MODE == 9 || MODE == 12) && warp == 2 && (tid & 31) == 0) {  // producer: wait empty, arrive full
    for (int kb = 0; kb < iters / P; ++kb) {
      const int s = kb % R;
      const uint32_t ph = (kb / R) & 1;
      asm volatile("{\n.reg .pred p;\nW3:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W3;\n}\n" ::"r"(su32(&emptyb[s])), "r"(ph ^ 1) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&fullb[s])) : "memory");
    }
  }
  if (((MODE >= 7 && MODE <= 9) || MODE == 12) && warp == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64(), g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int kb = 0; kb < iters / 4; ++kb) {
      const int st = kb % S;
      if (MODE == 8)
        asm volatile("{\n.reg .pred p;\nW8:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W8;\n}\n" ::"r"(su32(&spin)), "r"(1) : "memory");
      if (MODE == 9 || MODE == 12) {
        const uint32_t ph = (kb / R) & 1;
        asm volatile("{\n.reg .pred p;\nW9:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W9;\n}\n" ::"r"(su32(&fullb[kb % R])), "r"(ph) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t a = su32(sm + st * stage), b = a + 16384;
        if (MODE == 12) {  // kernel layout: A stages, then B stages
          a = su32(sm + st * 16384);
          b = su32(sm + S * 16384 + st * NT * 128);
        }
        const uint64_t da = sdesc(a + k * 32, 16, 1024, 0);
        const uint64_t db = sdesc(b + k * 32, 16, 1024, 0);
        const uint32_t dcol = tmem + (R == 3 ? ((kb / 72) & 1) * NT : 0);
        asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(dcol), "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                   ::"r"(su32(&emptyb[kb % R])) : "memory");
    }
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                 ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nWB:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WB;\n}\n" ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64(), g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (tid == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = g1 - g0;
    }
  }
  if (tid == 0 && (MODE < 7 || MODE > 9) && MODE != 12) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64(), g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int i = 0; i < iters; ++i) {
      const int st = (i / 4) % S, k = i & 3;
      if (MODE == 5 && i % P == 0) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (MODE == 6 && i % P == 0)
        asm volatile("{\n.reg .pred p;\nW6:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W6;\n}\n" ::"r"(su32(&spin)), "r"(1) : "memory");
      if (MODE == 10 && i % P == 0)
        asm volatile("{\n.reg .pred p;\nW10:\nmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%0], %1;\n@!p bra W10;\n}\n" ::"r"(su32(&spin)), "r"(1) : "memory");
      if (MODE == 11 && i % P == 0)
        asm volatile("{\n.reg .pred p;\nW11:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W11;\n}\n" ::"r"(su32(&spin)), "r"(1) : "memory");
      if (MODE == 3 && i % P == 0) {
        const uint32_t ph = ((i / P) / R) & 1;
        asm volatile("{\n.reg .pred p;\nW4:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W4;\n}\n" ::"r"(su32(&fullb[(i / P) % R])), "r"(ph) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const uint32_t a = su32(sm + st * stage), b = a + 16384;
      const uint64_t da = sdesc(a + k * 32, 16, 1024, 0);
      const uint64_t db = sdesc(b + k * 32, 16, 1024, 0);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1u));
      if (MODE == 3 && i % P == P - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&emptyb[(i / P) % R])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    long long t1 = clock64(), g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = g1 - g0;
    done = 1;
    if (MODE == 1) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&spin)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int NT, int MODE = 0, int R = 4, int P = 4>
static void run_full(int rnd, int ctas, int big = 0, int iters = 400000) {
  const int S = 4;
  const int smem = big ? 225 * 1024 : S * (16384 + NT * 128) + 2048;
  long long* d; cudaMalloc(&d, 1001 * 8);
  cudaFuncSetAttribute(mma_full<NT, S, MODE, R, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_full<NT, S, MODE, R, P><<<ctas, 320, smem>>>(d, iters / 10, rnd);  // warm
  cudaDeviceSynchronize();
  mma_full<NT, S, MODE, R, P><<<ctas, 320, smem>>>(d, iters, rnd);
  cudaDeviceSynchronize();
  long long h[2 * 148]; cudaMemcpy(h, d, sizeof(long long) * 2 * ctas, cudaMemcpyDeviceToHost);
  double cyc = 0, ns = 0;
  for (int i = 0; i < ctas; ++i) { cyc += h[2 * i]; ns += h[2 * i + 1]; }
  cyc /= ctas; ns /= ctas;
  const double tflops = 2.0 * 128 * NT * 8 * (double)iters * ctas / (ns * 1e-9) / 1e12;
  printf("full-chip mode %d ring %d x %d MMAs N=%d ctas=%d %s: %.1f cycles/MMA, %.0f MHz effective, %.0f TF/s\n", MODE, R, P, NT, ctas,
         rnd ? "random" : "const", cyc / iters, cyc / ns * 1e3, tflops);
  cudaFree(d);
}

template <int NT, int S, int CE = 0, int NACC = 1>
static long long run_stream(long long* d) {
  const int smem = S * (16384 + NT * 128) + 2048;
  cudaFuncSetAttribute(mma_stream<NT, S, CE, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_stream<NT, S, CE, NACC><<<1, 128, smem>>>(d);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  return c;
}

int main(int argc, char** argv) {
  if (argc > 1) {
    // full-chip TF32 peak: every SM streams back-to-back M=128 K=8 MMAs over
    // random operands (the roofline denominator of bench.py)
    run_full<256>(1, 148); run_full<192>(1, 148); run_full<128>(1, 148);
    run_full<192, 9>(1, 148);  // with the GEMM's stage-ring handshake
    // sustained: ~3 s of back-to-back launches (power/clock steady state)
    for (int r = 0; r < 10; ++r) run_full<192, 9>(1, 148, 0, 4000000);
    return 0;
  }
  {
    long long* d; cudaMalloc(&d, 8);
    printf("streaming MMA (M=128, K=8 tf32) cycles/MMA: N=256 S1 %lld S4 %lld | N=192 S1 %lld S4 %lld | N=96 S1 %lld S6 %lld | N=48 S1 %lld S6 %lld\n",
           run_stream<256, 1>(d), run_stream<256, 4>(d), run_stream<192, 1>(d), run_stream<192, 4>(d),
           run_stream<96, 1>(d), run_stream<96, 6>(d), run_stream<48, 1>(d), run_stream<48, 6>(d));
    printf("N=192 S4: commit every 8 %lld, every 4 %lld, 2 accumulators %lld, 2 acc + commit/8 %lld\n",
           run_stream<192, 4, 8, 1>(d), run_stream<192, 4, 4, 1>(d), run_stream<192, 4, 0, 2>(d),
           run_stream<192, 4, 8, 2>(d));
    printf("N=128 S4: plain %lld, 2 acc + commit/8 %lld | N=96 2 acc + commit/8 %lld\n",
           run_stream<128, 4>(d), run_stream<128, 4, 8, 2>(d), run_stream<96, 4, 8, 2>(d));
  }
  {
    long long* d; cudaMalloc(&d, 8);
    cudaFuncSetAttribute(mma_rate<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(mma_rate<192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(mma_rate<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int r0 : {0, 1, 2, 3, 4, 8, 15, 16, 17}) {
      long long c[3];
      mma_rate<256><<<1, 128, 100 * 1024>>>(r0, d); cudaDeviceSynchronize(); cudaMemcpy(&c[0], d, 8, cudaMemcpyDeviceToHost);
      mma_rate<192><<<1, 128, 100 * 1024>>>(r0, d); cudaDeviceSynchronize(); cudaMemcpy(&c[1], d, 8, cudaMemcpyDeviceToHost);
      mma_rate<64><<<1, 128, 100 * 1024>>>(r0, d); cudaDeviceSynchronize(); cudaMemcpy(&c[2], d, 8, cudaMemcpyDeviceToHost);
      printf("A start row %2d: cycles/MMA N=256 %lld  N=192 %lld  N=64 %lld\n", r0, c[0], c[1], c[2]);
    }
  }
  std::vector<float> A(MR * K), B(N * K), D(M * N);
  uint32_t s = 777;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 32768.0f - 1.0f; };
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  float *dA, *dB, *dD;
  cudaMalloc(&dA, 4 * A.size()); cudaMalloc(&dB, 4 * B.size()); cudaMalloc(&dD, 4 * D.size());
  cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 3; ++mode)
    for (int r0 = 0; r0 < 12; ++r0) {
      probe<<<1, 128, 48 * 1024>>>(dA, dB, dD, r0, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("r0=%d mode=%d CUDA error %s\n", r0, mode, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
      double err = 0, mx = 0;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)A[(m + r0) * K + k] * B[n * K + k];
          err = fmax(err, fabs(D[m * N + n] - ref));
          mx = fmax(mx, fabs(ref));
        }
      printf("base_off mode %d  r0=%2d  max|err| %.3e (max|ref| %.2f)\n", mode, r0, err, mx);
    }
  return 0;
}
