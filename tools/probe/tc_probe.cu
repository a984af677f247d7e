// Dev probe: one-CTA tcgen05.mma (kind::tf32 / kind::f16 bf16) with K-major SWIZZLE_NONE
// smem operands, TMEM accumulator, tcgen05.ld epilogue. Checks descriptor encodings on the box.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// smem image of a [rows][128 bytes] K-chunk: core matrix (8 rows x 16 B) at (row/8)*1024 + (kb/16)*128
__device__ __forceinline__ uint32_t img_off(int r, int kb) { return (r >> 3) * 1024 + (kb >> 4) * 128 + (r & 7) * 16 + (kb & 15); }

template <bool BF16>
__global__ void probe(const void* A, const void* B, float* D, int N, int K) {
  // A: [128][K] row-major, B: [N][K] row-major (K-major), D: [128][N]
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int esz = BF16 ? 2 : 4;
  const int kc_elems = 128 / esz;           // elements per 128-byte chunk
  const int nchunks = K / kc_elems;
  uint8_t* sA = smem;                       // nchunks * 16 KB
  uint8_t* sB = smem + nchunks * 16384;     // nchunks * N*128
  int tid = threadIdx.x, warp = tid / 32;
  for (int c = 0; c < nchunks; ++c)
    for (int idx = tid; idx < 128 * 128; idx += blockDim.x) {
      int r = idx / 128, kb = idx % 128;
      sA[c * 16384 + img_off(r, kb)] = ((const uint8_t*)A)[(size_t)r * K * esz + c * 128 + kb];
    }
  for (int c = 0; c < nchunks; ++c)
    for (int idx = tid; idx < N * 128; idx += blockDim.x) {
      int r = idx / 128, kb = idx % 128;
      sB[c * N * 128 + img_off(r, kb)] = ((const uint8_t*)B)[(size_t)r * K * esz + c * 128 + kb];
    }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tbase = tmem_base;
  if (tid == 0) {
    uint32_t idesc = (1u << 4) | ((uint32_t)(BF16 ? 1 : 2) << 7) | ((uint32_t)(BF16 ? 1 : 2) << 10) |
                     ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int c = 0; c < nchunks; ++c)
      for (int s = 0; s < 4; ++s) {   // 4 MMAs of 32 bytes of K each
        uint64_t ad = make_desc(smem_u32(sA + c * 16384 + s * 256), 128, 1024);
        uint64_t bd = make_desc(smem_u32(sB + c * N * 128 + s * 256), 128, 1024);
        uint32_t acc = (c | s) ? 1u : 0u;
        if (BF16)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                       :: "r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                       :: "r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)));
  }
  // wait phase 0
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" :: "r"(smem_u32(&mbar)), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    uint32_t ta = tbase + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "r"(256));
}

template <bool BF16>
int run(int N, int K) {
  std::vector<float> a(128 * K), b(N * K);
  srand(1);
  for (auto& x : a) x = (rand() % 17 - 8) / 8.0f;
  for (auto& x : b) x = (rand() % 13 - 6) / 4.0f;
  size_t esz = BF16 ? 2 : 4;
  std::vector<uint8_t> ha(a.size() * esz), hb(b.size() * esz);
  for (size_t i = 0; i < a.size(); ++i) { if (BF16) ((__nv_bfloat16*)ha.data())[i] = __float2bfloat16(a[i]); else ((float*)ha.data())[i] = a[i]; }
  for (size_t i = 0; i < b.size(); ++i) { if (BF16) ((__nv_bfloat16*)hb.data())[i] = __float2bfloat16(b[i]); else ((float*)hb.data())[i] = b[i]; }
  void *dA, *dB; float* dD;
  cudaMalloc(&dA, ha.size()); cudaMalloc(&dB, hb.size()); cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, ha.data(), ha.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hb.data(), hb.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, 128 * N * 4);
  int nchunks = K * esz / 128;
  size_t smem = nchunks * 16384 + nchunks * N * 128;
  cudaFuncSetAttribute(probe<BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<BF16><<<1, 128, smem>>>(dA, dB, dD, N, K);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s N=%d K=%d CUDA error %s\n", BF16 ? "bf16" : "tf32", N, K, cudaGetErrorString(e)); return 1; }
  std::vector<float> d(128 * N);
  cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int bad = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < N; ++n) {
    double ref = 0; for (int k = 0; k < K; ++k) ref += (double)a[m * K + k] * b[n * K + k];
    double err = fabs(ref - d[m * N + n]); if (err > maxerr) maxerr = err; if (err > 1e-3 && bad++ < 3) printf("  mismatch m=%d n=%d got %f ref %f\n", m, n, d[m*N+n], ref);
  }
  printf("%s N=%d K=%d maxerr=%g %s\n", BF16 ? "bf16" : "tf32", N, K, maxerr, maxerr < 1e-3 ? "OK" : "FAIL");
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return maxerr < 1e-3 ? 0 : 1;
}

int main() {
  int f = 0;
  f |= run<false>(64, 32); f |= run<false>(128, 64); f |= run<false>(256, 96); f |= run<false>(16, 32); f |= run<false>(48, 128);
  f |= run<true>(64, 64); f |= run<true>(128, 128); f |= run<true>(256, 64); f |= run<true>(16, 64);
  printf(f ? "PROBE FAIL\n" : "PROBE PASS\n");
  return f;
}
