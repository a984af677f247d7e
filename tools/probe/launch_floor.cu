// Launch-floor probe: per-launch time of back-to-back launches of (near-)empty persistent-style
// kernels on the B200 (148 CTAs x 288 threads), vs dynamic smem size, PDL, and CUDA-graph replay.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p[blockIdx.x] == 12345) s[0] = 1;
}
__global__ void k_pdl(int* p) {
  extern __shared__ int s[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0 && p[blockIdx.x] == 12345) s[0] = 1;
}
__global__ void k_tmem(int* p) {
  extern __shared__ __align__(16) int s[];
  __shared__ unsigned slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x / 32 == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x / 32 == 8) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
  }
  if (threadIdx.x == 0 && p[blockIdx.x] == 12345) s[0] = 1;
}

template <typename K>
float run(K kern, int grid, int smem, bool pdl, bool graph, cudaStream_t st, int* p) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(288);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  const int N = 200;
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, kern, p);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
  }
  for (int w = 0; w < 3; ++w) {
    if (graph) cudaGraphLaunch(ge, st);
    else for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, kern, p);
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  if (graph) cudaGraphLaunch(ge, st);
  else for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, kern, p);
  cudaEventRecord(b, st);
  cudaStreamSynchronize(st);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1000.f / N;
}

int main() {
  int* p;
  cudaMalloc(&p, 4096);
  cudaMemset(p, 0, 4096);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int smems[] = {0, 100 * 1024, 232 * 1024};
  for (int grid : {148, 32})
    for (int smem : smems) {
      printf("grid %3d smem %6d: empty %.2f us | pdl-kernel no-attr %.2f | pdl %.2f | graph %.2f | graph+pdl %.2f | tmem+pdl graph %.2f\n",
             grid, smem, run(k_empty, grid, smem, false, false, st, p), run(k_pdl, grid, smem, false, false, st, p),
             run(k_pdl, grid, smem, true, false, st, p), run(k_empty, grid, smem, false, true, st, p),
             run(k_pdl, grid, smem, true, true, st, p), run(k_tmem, grid, smem, true, true, st, p));
    }
  return 0;
}
