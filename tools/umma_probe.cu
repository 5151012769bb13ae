// Probe of the tcgen05 encodings in paper_2411_01142_b200/csrc/umma.cuh on a B200:
//   mode 0: D[128 x N] = A[128 x 128] . B[N x 128]^T   (A, B K-major SW128)  N in {64, 128, 256}
//   mode 1: D[128 x 128] = P[128 x 128] . V[128 x 128]  (P K-major, V MN-major SW128)
//   mode 2: as mode 1 with P in TMEM (written by tcgen05.st, lane = row, column c = pair 2c, 2c+1)
//   mode 3: as mode 2 with P in fp16 (A format f16) against bf16 V (B format bf16): mixed kind::f16
// Operands are written into shared memory with TMA's SWIZZLE_128B pattern by
// plain stores, then a single thread issues the MMAs; the 4 warps read the
// accumulator back with tcgen05.ld 32x32b and the host compares with fp64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o umma_probe tools/umma_probe.cu && ./umma_probe
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2411_01142_b200/csrc/umma.cuh"

using namespace neo;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const uint16_t* a, const uint16_t* b, float* d, int mode, int N) {
  extern __shared__ uint8_t raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = base;                 // 32 KiB
  uint8_t* sb = base + 32768;         // up to 64 KiB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  // A: 128 rows x 128 K, K-major: half h = k / 64 at h * 16 KiB
  for (int i = tid; i < 128 * 128; i += blockDim.x) {
    const int r = i / 128, k = i % 128;
    const uint32_t off = (k / 64) * 16384 + umma::sw128_off(r, (k % 64) / 8) + (k % 8) * 2;
    *reinterpret_cast<uint16_t*>(sa + off) = a[i];
  }
  if (mode == 0) {  // B: N rows x 128 K, K-major, half h at h * N * 128
    for (int i = tid; i < N * 128; i += blockDim.x) {
      const int r = i / 128, k = i % 128;
      const uint32_t off = (k / 64) * (N * 128) + umma::sw128_off(r, (k % 64) / 8) + (k % 8) * 2;
      *reinterpret_cast<uint16_t*>(sb + off) = b[i];
    }
  } else {  // V (modes 1, 2): 128 K rows (tokens) x 128 N (dims), MN-major: dim half h at h * 16 KiB
    for (int i = tid; i < 128 * 128; i += blockDim.x) {
      const int t = i / 128, n = i % 128;
      const uint32_t off = (n / 64) * 16384 + umma::sw128_off(t, (n % 64) / 8) + (n % 8) * 2;
      *reinterpret_cast<uint16_t*>(sb + off) = b[i];
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_proxy_async_smem();
  if (warp == 0) {
    umma::tmem_alloc(smem_u32(&tbase), 256);
    umma::tmem_relinquish();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tbase;
  if (mode >= 2) {  // P rows into TMEM columns 128.. (64 columns of bf16 pairs), one row per lane
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < 64; c0 += 32) {
      uint32_t r[32];
      for (int j = 0; j < 32; ++j)
        r[j] = static_cast<uint32_t>(a[row * 128 + 2 * (c0 + j)]) |
               (static_cast<uint32_t>(a[row * 128 + 2 * (c0 + j) + 1]) << 16);
      umma::st32(umma::taddr(tm, warp * 32, 128 + c0), r);
    }
    umma::wait_st();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  if (tid == 0) {
    const uint32_t A = smem_u32(sa), B = smem_u32(sb);
    for (int k = 0; k < 8; ++k) {
      const uint64_t ad = umma::desc_sw128(A + (k / 4) * 16384 + (k % 4) * 32, 16, 1024);
      uint64_t bd;
      uint32_t id;
      if (mode == 0) {
        bd = umma::desc_sw128(B + (k / 4) * (N * 128) + (k % 4) * 32, 16, 1024);
        id = umma::idesc_bf16_f32(128, N, false, false);
      } else {
        bd = umma::desc_sw128(B + k * 2048, 16384, 1024);
        id = umma::idesc_bf16_f32(128, 128, false, true);
        if (mode == 3) id &= ~(7u << 7);   // A format 0 = f16
      }
      if (mode >= 2) umma::mma_bf16_ts(tm, tm + 128 + k * 8, bd, id, k > 0);
      else umma::mma_bf16(tm, ad, bd, id, k > 0);
    }
    umma::commit(smem_u32(&bar));
  }
  __syncwarp();
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
  umma::fence_after_sync();
  const int ncols = mode == 0 ? N : 128;
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < ncols; c0 += 32) {
    uint32_t r[32];
    umma::ld32(umma::taddr(tm, warp * 32, c0), r);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) d[row * ncols + c0 + j] = __uint_as_float(r[j]);
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 256);
}

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}
static uint16_t f2h(float f) { return __half_as_ushort(__float2half_rn(f)); }
static double h2d(uint16_t h) { return static_cast<double>(__half2float(__ushort_as_half(h))); }
static double bf2d(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static int run(int mode, int N) {
  const int rowsB = mode == 0 ? N : 128;
  std::vector<uint16_t> a(128 * 128), b(rowsB * 128);
  srand(1234 + mode * 7 + N);
  for (auto& x : a)
    x = mode == 3 ? f2h(static_cast<float>(rand()) / RAND_MAX * 256.f)       // P in [0, 256], fp16
                  : f2bf(static_cast<float>(rand()) / RAND_MAX * 2.f - 1.f);
  for (auto& x : b) x = f2bf(static_cast<float>(rand()) / RAND_MAX * 2.f - 1.f);
  const int ncols = mode == 0 ? N : 128;
  uint16_t *da, *db;
  float* dd;
  cudaMalloc(&da, a.size() * 2);
  cudaMalloc(&db, b.size() * 2);
  cudaMalloc(&dd, 128 * ncols * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  const int smem = 1024 + 32768 + 65536;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(da, db, dd, mode, N);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("mode %d N %d: CUDA error %s\n", mode, N, cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> d(128 * ncols);
  cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < ncols; ++n) {
      double ref = 0;
      for (int k = 0; k < 128; ++k)
        ref += mode == 0   ? bf2d(a[m * 128 + k]) * bf2d(b[n * 128 + k])
               : mode == 3 ? h2d(a[m * 128 + k]) * bf2d(b[k * 128 + n])
                           : bf2d(a[m * 128 + k]) * bf2d(b[k * 128 + n]);
      worst = std::max(worst, std::fabs(ref - d[m * ncols + n]) / (mode == 3 ? 256.0 : 1.0));
    }
  printf("mode %d N %3d: max |err| = %.3e  %s\n", mode, N, worst, worst < 1e-3 ? "OK" : "FAIL");
  cudaFree(da);
  cudaFree(db);
  cudaFree(dd);
  return worst < 1e-3 ? 0 : 1;
}

int main() {
  int bad = 0;
  bad += run(0, 64);
  bad += run(0, 128);
  bad += run(0, 256);
  bad += run(1, 128);
  bad += run(2, 128);
  bad += run(3, 128);
  printf(bad ? "PROBE FAILED\n" : "PROBE OK\n");
  return bad;
}
