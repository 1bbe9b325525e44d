// Probe: tcgen05.mma kind::tf32 with K-major and MN-major SWIZZLE_128B smem
// operands (one CTA, M=128, N=64, K=32 as 4 MMAs of K=8).  Operands are
// written by threads in the canonical swizzled layouts:
//   K-major : row r (M or N index) = 128 B holding 32 consecutive k, 16-B
//             chunk c stored at chunk c ^ (r & 7); 8-row groups 1024 B apart (SBO).
//   MN-major: k-row = 128 B holding 32 consecutive m (or n), chunk c stored at
//             c ^ (k & 7); 8-k groups 1024 B apart, 32-wide MN blocks 4096 B apart.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mn_probe tools/mn_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 32;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int lt = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)lt << 61;
  return d;
}

__device__ __forceinline__ uint32_t off_k(int r, int k) {  // K-major byte offset
  return (uint32_t)(r * 128 + (((k >> 2) ^ (r & 7)) << 4) + (k & 3) * 4);
}
__device__ __forceinline__ uint32_t off_mn(int r, int k) {  // MN-major byte offset
  const int mb = r >> 5, mi = r & 31;
  return (uint32_t)(mb * 4096 + k * 128 + (((mi >> 2) ^ (k & 7)) << 4) + (mi & 3) * 4);
}
// MN-major, SWIZZLE_128B_BASE32B: 32-B chunk c of k-row stored at c ^ (k & 3)
__device__ __forceinline__ uint32_t off_mn32(int r, int k) {
  const int mb = r >> 5, mi = r & 31, byte = mi * 4;
  return (uint32_t)(mb * 4096 + k * 128 + ((((byte >> 5) ^ (k & 3))) << 5) + (byte & 31));
}

__global__ void probe(const float* A, const float* B, float* D, int a_mn, int b_mn, int lbo_a,
                      int sbo_a, int lbo_b, int sbo_b, int kstep_a, int kstep_b, int lt_a, int lt_b) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;               // 16 KB
  uint8_t* sB = sm + 16384;       // 8 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    *(float*)(sA + (a_mn ? (lt_a == 1 ? off_mn32(m, k) : off_mn(m, k)) : off_k(m, k))) = A[m * K + k];
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    *(float*)(sB + (b_mn ? (lt_b == 1 ? off_mn32(n, k) : off_mn(n, k)) : off_k(n, k))) = B[n * K + k];
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) |
                           ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int j = 0; j < K / 8; ++j) {
      const uint64_t da = sdesc(su32(sA) + j * kstep_a, lbo_a, sbo_a, lt_a);
      const uint64_t db = sdesc(su32(sB) + j * kstep_b, lbo_b, sbo_b, lt_b);
      const uint32_t acc = j > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32w..32w+31 (rows m), columns 0..63 (n)
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

int main() {
  std::vector<float> A(M * K), B(N * K), ref(M * N), D(M * N);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 32768.0f - 1.0f; };
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k = 0; k < K; ++k) acc += (double)A[m * K + k] * B[n * K + k];
      ref[m * N + n] = (float)acc;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, 4 * A.size()); cudaMalloc(&dB, 4 * B.size()); cudaMalloc(&dD, 4 * D.size());
  cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024);
  struct Cfg { const char* name; int a_mn, b_mn, lbo_a, sbo_a, lbo_b, sbo_b, ks_a, ks_b, lt_a, lt_b; };
  const Cfg cfgs[] = {
      {"K/K", 0, 0, 16, 1024, 16, 1024, 32, 32, 2, 2},
      {"MN32(lbo4096,sbo512)/K", 1, 0, 4096, 512, 16, 1024, 1024, 32, 1, 2},
      {"MN32(lbo512,sbo4096)/K", 1, 0, 512, 4096, 16, 1024, 1024, 32, 1, 2},
      {"K/MN32(lbo4096,sbo512)", 0, 1, 16, 1024, 4096, 512, 32, 1024, 2, 1},
      {"K/MN32(lbo512,sbo4096)", 0, 1, 16, 1024, 512, 4096, 32, 1024, 2, 1},
      {"MN32/MN32(4096,512)", 1, 1, 4096, 512, 4096, 512, 1024, 1024, 1, 1},
      {"MN128(lbo4096,sbo1024)/K", 1, 0, 4096, 1024, 16, 1024, 1024, 32, 2, 2},
  };
  for (const Cfg& c : cfgs) {
    cudaMemset(dD, 0, 4 * D.size());
    probe<<<1, 128, 32 * 1024>>>(dA, dB, dD, c.a_mn, c.b_mn, c.lbo_a, c.sbo_a, c.lbo_b, c.sbo_b,
                                 c.ks_a, c.ks_b, c.lt_a, c.lt_b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%-26s CUDA error %s\n", c.name, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int i = 0; i < M * N; ++i) { err = fmax(err, fabs(D[i] - ref[i])); mx = fmax(mx, fabs(ref[i])); }
    printf("%-26s max|err| %.3e  (max|ref| %.3e)  D[0]=%.4f ref[0]=%.4f\n", c.name, err, mx, D[0], ref[0]);
  }
  return 0;
}
