// MUFU.EX2 issue rate on one SM: W warps (of one CTA) each run N rounds of 32
// independent ex2.approx per thread; cycles per warp-instruction from clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_rate tools/mufu_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int mode>
__global__ void k(float* out, long long* cyc, int rounds) {
  float x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (mode == 5) {            // the softmax pattern: 2 x ex2 + 1 fp16 pack per pair
        float y0, y1;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(x[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y1) : "f"(x[(i + 16) & 31]));
        uint32_t h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(y0), "f"(y1));
        x[i] = __uint_as_float(h & 0x3fff3fffu) - 1.0f;
      } else if (mode == 3) {            // F2FP: cvt.rn.f16x2.f32 (the fp16 pack of P)
        uint32_t h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[i]), "f"(x[(i + 1) & 31]));
        x[i] = __uint_as_float(h & 0x3fff3fffu) - 1.0f;
      } else if (mode == 4) {     // F2FP bf16x2 pack (cvt.rn.bf16x2.f32)
        uint32_t h;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[i]), "f"(x[(i + 1) & 31]));
        x[i] = __uint_as_float(h & 0x3fff3fffu) - 1.0f;
      } else if (mode == 2) {            // FFMA2 chain reference (fma pipe)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(*reinterpret_cast<unsigned long long*>(&x[i & ~1])) : "l"(0x3f8000003f800000ull), "l"(0ull));
      } else if (mode == 0) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
        x[i] = y - 1.0f;
      } else {
        uint32_t h;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[i]), "f"(x[i]));
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(h));
        x[i] = __uint_as_float(y & 0x3fff) - 1.0f;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x % 32 == 0) cyc[threadIdx.x / 32] = t1 - t0;
}
int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64 * 8);
  for (int mode = 0; mode < 6; ++mode)
    for (int w : {1, 4, 8, 16}) {
      int rounds = 200;
      if (mode == 0) k<0><<<1, 32 * w>>>(out, cyc, rounds);
      else if (mode == 1) k<1><<<1, 32 * w>>>(out, cyc, rounds);
      else if (mode == 2) k<2><<<1, 32 * w>>>(out, cyc, rounds);
      else if (mode == 3) k<3><<<1, 32 * w>>>(out, cyc, rounds);
      else if (mode == 4) k<4><<<1, 32 * w>>>(out, cyc, rounds);
      else k<5><<<1, 32 * w>>>(out, cyc, rounds);
      cudaDeviceSynchronize();
      long long h[64];
      cudaMemcpy(h, cyc, 8 * w, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < w; ++i) mx = h[i] > mx ? h[i] : mx;
      // per SMSP: ceil(w/4) warps; warp-instructions of MUFU per SMSP = warps_per_smsp * rounds * 32
      int wps = (w + 3) / 4;
      printf("mode %s warps %2d: %.2f cycles per MUFU warp-instr per SMSP (total cyc %.0f)\n", mode == 1 ? "f16x2" : mode == 0 ? "f32" : mode == 2 ? "ffma2" : mode == 3 ? "F2FP.F16 (+FADD)" : mode == 4 ? "F2FP.BF16 (+FADD)" : "2 ex2 + F2FP per step (cycles per step)", w,
             mx / (wps * rounds * 32.0), mx);
    }
  return 0;
}
