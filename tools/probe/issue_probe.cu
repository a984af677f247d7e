// Cost of the producer's per-chunk issue sequence on sm_100a, one thread, clock64 per step:
// mbarrier try_wait on a completed phase, arrive.expect_tx, cp.async.bulk (global -> shared), arrive.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint8_t* src, long long* out, int n, int bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 16 * 8192);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[i])), "r"(2));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < n; ++i) {
    const int s = i & 15;
    const uint32_t b = smem_u32(&bars[s]);
    const uint32_t par = ((i >> 4) & 1) ^ 1;
    long long c0 = clock64();
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(b), "r"(par) : "memory");
    long long c1 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    long long c2 = clock64();
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + s * 8192)),
                 "l"(src + (size_t)i * bytes), "r"(bytes), "r"(b) : "memory");
    long long c3 = clock64();
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
    long long c4 = clock64();
    t[0] += c1 - c0; t[1] += c2 - c1; t[2] += c3 - c2; t[3] += c4 - c3;
    if (i >= 15) {   // consume: wait for the copy issued 15 iterations ago (keeps the ring in flight)
      const int j = i - 15;
      const uint32_t bj = smem_u32(&bars[j & 15]);
      long long c5 = clock64();
      asm volatile("{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n\t}" ::"r"(bj),
                   "r"((uint32_t)((j >> 4) & 1)) : "memory");
      t[4] += clock64() - c5;
    }
  }
  for (int k = 0; k < 5; ++k) out[k] = t[k] / n;
}

int main() {
  uint8_t* src; cudaMalloc(&src, 64 << 20);
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 8192 + 1024);
  for (int bytes : {1024, 4096, 8192}) {
    for (int rep = 0; rep < 2; ++rep) {
      probe<<<1, 32, 16 * 8192 + 1024>>>(src, d, 2000, bytes);
      long long h[5];
      cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
      printf("bytes %5d: try_wait %lld, expect_tx %lld, bulk issue %lld, arrive %lld, consumer wait %lld cycles (%s)\n", bytes, h[0], h[1],
             h[2], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
