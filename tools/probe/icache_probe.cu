// Cold instruction-fetch cost per launch: a kernel whose one warp per SM executes N straight-line
// FFMAs (N / 4 ... instructions of distinct code) vs the same FFMA count in a 64-instruction loop,
// both CUDA-graph launched back to back (PDL off). If the instruction cache is cold at every launch,
// the straight-line kernel pays one L2 (or DRAM) fetch per 128 B of code it runs.
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void straight(float* out, float a, float b) {
  float x = threadIdx.x, y = 1.0f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    x = fmaf(x, a, b);
    y = fmaf(y, b, x);
  }
  if (x + y == 12345.f) out[threadIdx.x] = x;
}

template <int N>
__global__ void looped(float* out, float a, float b) {
  float x = threadIdx.x, y = 1.0f;
#pragma unroll 1
  for (int i = 0; i < N / 32; ++i) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      x = fmaf(x, a, b);
      y = fmaf(y, b, x);
    }
  }
  if (x + y == 12345.f) out[threadIdx.x] = x;
}

template <typename K>
float time_graph(K kern, float* out, int threads) {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 200; ++i) kern<<<148, threads, 0, s>>>(out, 1.0001f, 0.5f);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / (5 * 200);
}

#define RUN(N)                                                                                              \
  {                                                                                                        \
    float ts = time_graph(straight<N>, out, 32), tl = time_graph(looped<N>, out, 32);                      \
    printf("N=%6d FFMA pairs: straight %.2f us, looped %.2f us, diff %.2f us (straight code ~%d KB)\n", N, ts, \
           tl, ts - tl, (N * 2 * 16) / 1024);                                                              \
  }

int main() {
  float* out;
  cudaMalloc(&out, 4096);
  RUN(256);
  RUN(512);
  RUN(1024);
  RUN(2048);
  RUN(4096);
  RUN(8192);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
