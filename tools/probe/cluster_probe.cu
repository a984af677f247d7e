// How many clusters of size CS (one 227 KB CTA per SM) can be co-resident on this GPU, and the
// latency of a cluster-scope mbarrier handshake + DSMEM read (remote arrive -> wait -> ld.shared::cluster).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void big_kernel(int* out) {
  extern __shared__ uint8_t sm[];
  if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ping-pong between cluster rank 0 and 1: each round rank r writes a value into its smem, arrives on
// the peer's mbarrier (release.cluster), waits on its own (acquire.cluster), reads the peer's value.
__global__ void pingpong(long long* out, int rounds) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ int val;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
  if (threadIdx.x != 0) return;
  const uint32_t peer = rank ^ 1;
  uint32_t rbar, rval;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&bar)), "r"(peer));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rval) : "r"(smem_u32(&val)), "r"(peer));
  long long t0 = clock64();
  int acc = 0;
  for (int i = 0; i < rounds; ++i) {
    val = i + (int)rank;
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
            smem_u32(&bar)),
        "r"((uint32_t)(i & 1))
        : "memory");
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(rval) : "memory");
    acc += v;
  }
  long long t1 = clock64();
  if (rank == 0) { out[0] = (t1 - t0) / rounds; out[1] = acc; }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
}

int main() {
  int smem = 227 * 1024;
  cudaFuncSetAttribute(big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(big_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs * 16);
    cfg.blockDim = dim3(288);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)big_kernel, &cfg);
    printf("cluster %2d: max active clusters %d (CTAs %d) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  long long* d; cudaMalloc(&d, 16);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2); cfg.blockDim = dim3(32);
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, pingpong, d, 10000);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("cluster mbarrier round trip + DSMEM read: %lld cycles per round (%s)\n", h[0], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
