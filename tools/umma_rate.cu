// Issue-rate microbenchmark of the tcgen05.mma forms the prefill kernel uses
// (one CTA, one issuing thread, operands resident in SMEM / TMEM), with the
// descriptors precomputed and the issue loop fully unrolled:
//   mode 0  SS  K-major A, K-major B     (S = Q K^T)
//   mode 1  TS  A in TMEM, MN-major B    (O += P V)
// CHAINS independent accumulators are round-robined to expose (or hide) the
// dependent-accumulate latency.  Reports cycles per M128 x N x K16 instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/umma_rate tools/umma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2411_01142_b200/csrc/umma.cuh"

using namespace neo;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE, int N, int CHAINS>
__global__ void rate(int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_proxy_async_smem();
  if (warp == 0) {
    umma::tmem_alloc(smem_u32(&tbase), 512);
    umma::tmem_relinquish();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t A = smem_u32(base), B = A + 32768;
    constexpr uint32_t id = umma::idesc_bf16_f32(128, N, false, MODE == 1);
    const uint64_t a0 = umma::desc_sw128(A, 16, 1024);
    const uint64_t b0 = MODE == 0 ? umma::desc_sw128(B, 16, 1024) : umma::desc_sw128(B, 16384, 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t d = tm + (k % CHAINS) * 128;
        if (MODE == 0)
          umma::mma_bf16(d, a0 + ((k >> 2) * 16384 + (k & 3) * 32) / 16, b0 + ((k >> 2) * (N * 128) + (k & 3) * 32) / 16,
                         id, true);
        else
          umma::mma_bf16_ts(d, tm + 384 + k * 8, b0 + (k * 2048) / 16, id, true);
      }
    }
    umma::commit(smem_u32(&bar));
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    out[0] = clock64() - t0;
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 512);
}

template <int MODE, int N, int CHAINS>
void run(long long* d) {
  const int smem = 1024 + 96 * 1024;
  cudaFuncSetAttribute(rate<MODE, N, CHAINS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  rate<MODE, N, CHAINS><<<1, 128, smem>>>(64, d);
  rate<MODE, N, CHAINS><<<1, 128, smem>>>(iters, d);
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = static_cast<double>(c) / iters;
  printf("%s N%3d chains %d: %6.1f cyc/instr (ideal %5.1f) -> %3.0f%% of 8192 flop/cyc\n",
         MODE == 0 ? "SS K/K   " : "TS tmem/MN", N, CHAINS, cyc, 128.0 * N / 256,
         100.0 * (2.0 * 128 * N * 16 / cyc) / 8192);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<0, 64, 1>(d);
  run<0, 128, 1>(d);
  run<0, 256, 1>(d);
  run<0, 64, 2>(d);
  run<0, 128, 2>(d);
  run<0, 64, 4>(d);
  run<1, 128, 1>(d);
  run<1, 128, 2>(d);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
