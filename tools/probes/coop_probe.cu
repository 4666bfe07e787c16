// Can a cooperative launch be stream-captured into a CUDA graph, and what
// does a software grid barrier cost?  (probe for fusing the merge into K1)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_bar(unsigned* c, unsigned* out, int rounds) {
  for (int r = 0; r < rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned target = (r + 1) * gridDim.x;
      atomicAdd(c, 1u);
      while (*reinterpret_cast<volatile unsigned*>(c) < target) __nanosleep(32);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const unsigned a = atomicAdd(c + 1, 1u);
    if (a == gridDim.x - 1) { c[0] = 0; c[1] = 0; out[0] += 1; }
  }
}

int main() {
  unsigned *c, *out;
  cudaMalloc(&c, 64); cudaMemset(c, 0, 64);
  cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t s; cudaStreamCreate(&s);
  int rounds = 1;
  void* args[] = {&c, &out, &rounds};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k_bar, dim3(sms), dim3(1024), args, 0, s);
  printf("eager coop launch: %s\n", cudaGetErrorString(e));
  cudaStreamSynchronize(s);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  e = cudaLaunchCooperativeKernel((void*)k_bar, dim3(sms), dim3(1024), args, 0, s);
  printf("captured coop launch: %s\n", cudaGetErrorString(e));
  e = cudaStreamEndCapture(s, &g);
  printf("end capture: %s\n", cudaGetErrorString(e));
  if (e == cudaSuccess) {
    e = cudaGraphInstantiate(&ge, g, 0);
    printf("instantiate: %s\n", cudaGetErrorString(e));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    for (int i = 0; i < 100; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    e = cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("graph replay (1 barrier): %.2f us per launch (%s)\n", ms * 10, cudaGetErrorString(e));
  }
  for (int R : {1, 11}) {
    rounds = R;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int i = 0; i < 100; ++i) cudaLaunchCooperativeKernel((void*)k_bar, dim3(sms), dim3(1024), args, 0, s);
    cudaEventRecord(b, s);
    cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("eager, %d barriers: %.2f us per launch\n", R, ms * 10);
  }
  unsigned h; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("completed launches %u, %s\n", h, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
