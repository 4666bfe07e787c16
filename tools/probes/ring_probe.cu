// TMA ring probe: how fast can one CTA per SM stream its contiguous range
// through shared memory with cp.async.bulk, for the ring shapes K1 could use?
//   warp:  a private ring per warp (slot = 32 * U units), lane 0 refills its own slot
//   cta:   one ring per CTA (stage = 1024 units = 48 KB, PIECES copies), the
//          warp that releases a stage last issues its refill
// Consumers read their 48-byte units back with three LDS.128 and XOR them.
//   nvcc -arch=sm_100a -O3 -o ring_probe ring_probe.cu && ./ring_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra D;\n\t"
      "bra W;\n\t"
      "D:\n\t}"
      :: "r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ uint32_t lds_xor(uint32_t addr) {
  uint32_t a, b, c, d, acc = 0;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr + 16 * q));
    acc ^= a ^ b ^ c ^ d;
  }
  return acc;
}

extern __shared__ __align__(1024) uint8_t smem[];

// per-warp rings: per_cta units is a multiple of 1024 * U
template <int U, int D>
__global__ void __launch_bounds__(1024, 1) k_warp(const uint8_t* __restrict__ p, int64_t per_cta, uint32_t* out) {
  constexpr uint32_t SLOT = 1536u * U;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = uint32_t(__cvta_generic_to_shared(smem));
  const uint32_t ring = base + warp * D * SLOT, bars = base + 32 * D * SLOT + warp * D * 8;
  const uint8_t* src = p + 48 * (blockIdx.x * per_cta + int64_t(warp) * 32 * U);
  const int n_it = int(per_cta / (1024 * U));
  if (lane == 0) {
    for (int s = 0; s < D; ++s) mbar_init(bars + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < D && s < n_it; ++s) {
      mbar_expect_tx(bars + 8 * s, SLOT);
      bulk_g2s(ring + s * SLOT, src + int64_t(s) * 1024 * U * 48, SLOT, bars + 8 * s);
    }
  }
  __syncwarp();
  uint32_t acc = 0, slot = 0, phase = 0;
  for (int k = 0; k < n_it; ++k) {
    mbar_wait(bars + 8 * slot, phase);
#pragma unroll
    for (int j = 0; j < U; ++j) acc ^= lds_xor(ring + slot * SLOT + (j * 32 + lane) * 48);
    __syncwarp();
    if (lane == 0 && k + D < n_it) {
      mbar_expect_tx(bars + 8 * slot, SLOT);
      bulk_g2s(ring + slot * SLOT, src + int64_t(k + D) * 1024 * U * 48, SLOT, bars + 8 * slot);
    }
    if (++slot == D) { slot = 0; phase ^= 1; }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// one ring per CTA: stage = 1024 units (49152 B) in PIECES copies; the warp that
// frees a stage last refills it
template <int D, int PIECES>
__global__ void __launch_bounds__(1024, 1) k_cta(const uint8_t* __restrict__ p, int64_t per_cta, uint32_t* out) {
  constexpr uint32_t STAGE = 49152u, PIECE = STAGE / PIECES;
  const int lane = threadIdx.x & 31;
  const uint32_t base = uint32_t(__cvta_generic_to_shared(smem));
  const uint32_t bars = base + D * STAGE;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem + D * STAGE + 8 * D);
  const uint8_t* src = p + 48 * (blockIdx.x * per_cta);
  const int n_it = int(per_cta / 1024);
  auto refill = [&](int it, uint32_t s) {
    mbar_expect_tx(bars + 8 * s, STAGE);
#pragma unroll
    for (int q = 0; q < PIECES; ++q)
      bulk_g2s(base + s * STAGE + q * PIECE, src + int64_t(it) * STAGE + q * PIECE, PIECE, bars + 8 * s);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < D; ++s) { mbar_init(bars + 8 * s, 1); cnt[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < D && s < n_it; ++s) refill(s, s);
  }
  __syncthreads();
  uint32_t acc = 0, slot = 0, phase = 0;
  for (int k = 0; k < n_it; ++k) {
    mbar_wait(bars + 8 * slot, phase);
    acc ^= lds_xor(base + slot * STAGE + threadIdx.x * 48);
    __syncwarp();
    if (lane == 0) {
      uint32_t old;
      asm volatile("atom.acq_rel.cta.shared.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(bars + 8 * D + 4 * slot) : "memory");
      if (old == 31u) {
        cnt[slot] = 0;
        if (k + D < n_it) refill(k + D, slot);
      }
    }
    if (++slot == D) { slot = 0; phase ^= 1; }
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

template <class K>
void run(const char* name, K k, size_t sm, const uint8_t* p, int64_t per_cta, uint32_t* out, int sms, int64_t bytes) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
  float ms = timeit([&] { k<<<sms, 1024, sm>>>(p, per_cta, out); });
  cudaError_t e = cudaDeviceSynchronize();
  printf("%-28s %8.1f us  %7.1f GB/s  %s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t per_cta = 56320;                       // 55 x 1024 units, multiple of 4096? no: use 56 x 1024 below for U=4
  const int64_t per4 = 57344;                          // 14 x 4096
  const int64_t bytes = int64_t(sms) * per4 * 48;
  uint8_t* p; uint32_t* out;
  cudaMalloc(&p, bytes); cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  (void)per_cta;
  const int64_t b = int64_t(sms) * per4 * 48;
  run("warp U=1 D=2", k_warp<1, 2>, 32 * 2 * 1536 + 32 * 2 * 8, p, per4, out, sms, b);
  run("warp U=1 D=3", k_warp<1, 3>, 32 * 3 * 1536 + 32 * 3 * 8, p, per4, out, sms, b);
  run("warp U=1 D=4", k_warp<1, 4>, 32 * 4 * 1536 + 32 * 4 * 8, p, per4, out, sms, b);
  run("warp U=2 D=2", k_warp<2, 2>, 32 * 2 * 3072 + 32 * 2 * 8, p, per4, out, sms, b);
  run("warp U=4 D=2", k_warp<4, 2>, 32 * 2 * 6144 + 32 * 2 * 8, p, per4, out, sms, b);
  run("cta D=2 x1", k_cta<2, 1>, 2 * 49152 + 64, p, per4, out, sms, b);
  run("cta D=3 x1", k_cta<3, 1>, 3 * 49152 + 64, p, per4, out, sms, b);
  run("cta D=4 x1", k_cta<4, 1>, 4 * 49152 + 64, p, per4, out, sms, b);
  run("cta D=3 x4", k_cta<3, 4>, 3 * 49152 + 64, p, per4, out, sms, b);
  run("cta D=3 x16", k_cta<3, 16>, 3 * 49152 + 64, p, per4, out, sms, b);
  run("cta D=2 x4", k_cta<2, 4>, 2 * 49152 + 64, p, per4, out, sms, b);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
