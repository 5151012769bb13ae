// HBM read-ceiling probe (development aid, not product): streams a large
// buffer with 16-byte non-allocating loads, many in flight per thread, and
// reduces to one word per CTA so nothing is optimised away.
#include <cuda_runtime.h>
#include <stdint.h>

template <int U>
__global__ void __launch_bounds__(512) read_kernel(const uint4* __restrict__ p, int64_t n, uint32_t* out) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t j = i + (int64_t)u * blockDim.x;
      if (j < n) asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + j));
      else v[u] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

extern "C" __attribute__((visibility("default"))) int readbw(const void* p, int64_t bytes, uint32_t* out, int blocks,
                                                             int threads, int unroll, void* stream) {
  int64_t n = bytes / 16;
  if (unroll == 4) read_kernel<4><<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)p, n, out);
  else if (unroll == 16) read_kernel<16><<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)p, n, out);
  else read_kernel<8><<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)p, n, out);
  return (int)cudaGetLastError();
}
