// Which (lane, column) does each thread receive from tcgen05.ld.16x256b?
// TMEM lane L, column C is first set to L * 1000 + C with 32x32b stores; then
// warp w (quarter w % 4, half w / 4) loads 16 lanes at lane base 32*quarter +
// 16*half with .16x256b.x1 and .x2, and thread 0..31 of warps 0 and 4 print.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/tmem_layout_probe tools/tmem_layout_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2411_01142_b200/csrc/umma.cuh"

using namespace neo;

__global__ void probe(unsigned* outv) {
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    umma::tmem_alloc(static_cast<uint32_t>(__cvta_generic_to_shared(&tb)), 128);
    umma::tmem_relinquish();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tm = tb;
  if (warp < 4) {
    uint32_t r[32];
    for (int c0 = 0; c0 < 128; c0 += 32) {
      for (int j = 0; j < 32; ++j) r[j] = (warp * 32 + lane) * 1000 + c0 + j;
      umma::st32(umma::taddr(tm, warp * 32, c0), r);
    }
    umma::wait_st();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const int quarter = warp & 3, half = warp >> 2;
  const uint32_t addr = tm + (static_cast<uint32_t>(32 * quarter + 16 * half) << 16);
  uint32_t a0, a1, a2, a3, b[8];
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7])
               : "r"(addr));
  umma::wait_ld();
  unsigned* o = outv + (warp * 32 + lane) * 12;
  o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3;
  for (int j = 0; j < 8; ++j) o[4 + j] = b[j];
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 128);
}

int main() {
  unsigned* d;
  cudaMalloc(&d, 256 * 12 * 4);
  probe<<<1, 256>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  unsigned h[256 * 12];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  for (int w : {0, 4, 1}) {
    for (int t = 0; t < 32; ++t) {
      const unsigned* o = h + (w * 32 + t) * 12;
      printf("w%d t%2d 16x128b.x2:", w, t);
      for (int j = 0; j < 4; ++j) printf(" %u.%u", o[j] / 1000, o[j] % 1000);
      printf("  16x64b.x8:");
      for (int j = 0; j < 8; ++j) printf(" %u.%u", o[4 + j] / 1000, o[4 + j] % 1000);
      printf("\n");
    }
  }
  return 0;
}
