// Pure-read HBM probe: what read bandwidth can a streaming kernel reach on
// this B200, for the access patterns the build kernel could use?
//   contiguous: each CTA streams one contiguous range (K1's pattern)
//   stride:     grid-stride over 48-byte units (classify's pattern)
// Each thread keeps U units (48 B each, three 16-byte loads) in flight.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(1024, 1) k_contig(const uint4* __restrict__ p, int64_t n_units, int64_t per_cta, uint32_t* out) {
  const int64_t b = blockIdx.x * per_cta, e = min(n_units, b + per_cta);
  uint32_t acc = 0;
  for (int64_t u = b + threadIdx.x; u < e; u += 1024 * U) {
    uint4 v[U][3];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t uu = u + k * 1024;
      if (uu < e) { v[k][0] = __ldg(p + 3 * uu); v[k][1] = __ldg(p + 3 * uu + 1); v[k][2] = __ldg(p + 3 * uu + 2); }
      else { v[k][0] = v[k][1] = v[k][2] = make_uint4(0, 0, 0, 0); }
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc ^= v[k][q].x ^ v[k][q].y ^ v[k][q].z ^ v[k][q].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) k_stride(const uint4* __restrict__ p, int64_t n_units, uint32_t* out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < n_units; u += stride * U) {
    uint4 v[U][3];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t uu = u + k * stride;
      if (uu < n_units) { v[k][0] = __ldg(p + 3 * uu); v[k][1] = __ldg(p + 3 * uu + 1); v[k][2] = __ldg(p + 3 * uu + 2); }
      else { v[k][0] = v[k][1] = v[k][2] = make_uint4(0, 0, 0, 0); }
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
#pragma unroll
      for (int q = 0; q < 3; ++q) acc ^= v[k][q].x ^ v[k][q].y ^ v[k][q].z ^ v[k][q].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 20;
}

int main() {
  const int64_t bytes = 64LL * 1920 * 1080 * 3;      // 64 C3 frames, 398 MB
  const int64_t n_units = bytes / 48;
  uint4* p; uint32_t* out;
  cudaMalloc(&p, bytes); cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto report = [&](const char* name, float ms) { printf("%-28s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
  {
    const int64_t per = (n_units + sms - 1) / sms;
    report("contig U=1", timeit([&] { k_contig<1><<<sms, 1024>>>(p, n_units, per, out); }));
    report("contig U=2", timeit([&] { k_contig<2><<<sms, 1024>>>(p, n_units, per, out); }));
    report("contig U=3", timeit([&] { k_contig<3><<<sms, 1024>>>(p, n_units, per, out); }));
    report("contig U=4", timeit([&] { k_contig<4><<<sms, 1024>>>(p, n_units, per, out); }));
  }
  for (int cps : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "stride U=1 x%d", cps); report(nm, timeit([&] { k_stride<1><<<sms * cps, 256>>>(p, n_units, out); }));
    snprintf(nm, 64, "stride U=2 x%d", cps); report(nm, timeit([&] { k_stride<2><<<sms * cps, 256>>>(p, n_units, out); }));
    snprintf(nm, 64, "stride U=4 x%d", cps); report(nm, timeit([&] { k_stride<4><<<sms * cps, 256>>>(p, n_units, out); }));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
