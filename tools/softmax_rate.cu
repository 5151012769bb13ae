// Latency of one prefill softmax row step (128 scores per thread, the stream
// kernel's arithmetic: max, FFMA2, ex2 (MUFU or FMA-pipe polynomial), fp16
// pack, row sums) from registers, W warps in one CTA, clock64 per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -o tools/softmax_rate tools/softmax_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2411_01142_b200/csrc/umma.cuh"
#ifndef SPIN
#define SPIN 0   // 1: one extra warp per SMSP spins in mbarrier.try_wait while the softmax warps run
#endif
#ifndef TM
#define TM 0   // 1: S from TMEM (4 x ld32, one wait) and P to TMEM (4 x st16, wait) every step, as the kernel
#endif
__device__ __forceinline__ uint64_t f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unf2(uint64_t v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
#ifndef POLY
#define POLY 0   // of every 4 column pairs, how many take the FMA-pipe exp2 (degree-4, as the kernel)
#endif
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  float2 x = unf2(x2);
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const uint64_t magic = f2(12582912.f, 12582912.f);
  const uint64_t t = fadd2(f2(x.x, x.y), magic);
  const uint64_t fr = fsub2(f2(x.x, x.y), fsub2(t, magic));
  uint64_t p = ffma2(fr, f2(0.0096181291f, 0.0096181291f), f2(0.0555041087f, 0.0555041087f));
  p = ffma2(p, fr, f2(0.2402265070f, 0.2402265070f));
  p = ffma2(p, fr, f2(0.6931471806f, 0.6931471806f));
  p = ffma2(p, fr, f2(1.f, 1.f));
  const float2 tt = unf2(t), pv = unf2(p);
  const uint32_t r0 = __float_as_uint(tt.x) * (1u << 23) + __float_as_uint(pv.x);
  const uint32_t r1 = __float_as_uint(tt.y) * (1u << 23) + __float_as_uint(pv.y);
  return f2(__uint_as_float(r0), __uint_as_float(r1));
}
#ifndef DEG3
#define DEG3 0   // 1: degree-3 minimax polynomial (8 instructions per pair) instead of the kernel's degree-4
#endif
__device__ __forceinline__ uint64_t exp2_poly3(uint64_t x2) {
  // 2^x = 2^j * 2^f, j = rint(x) by the 1.5 * 2^23 shifter, f in [-0.5, 0.5],
  // 2^f ~ 1 + f (c1 + f (c2 + f c3)); exponent added with one IMAD per element
  float2 x = unf2(x2);
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const uint64_t xc = f2(x.x, x.y);
  const uint64_t magic = f2(12582912.f, 12582912.f);
  const uint64_t t = fadd2(xc, magic);
  const uint64_t fr = fsub2(xc, fsub2(t, magic));
  uint64_t p = ffma2(fr, f2(0.0558755f, 0.0558755f), f2(0.2401536f, 0.2401536f));
  p = ffma2(p, fr, f2(0.6931182f, 0.6931182f));
  p = ffma2(p, fr, f2(1.0000000f, 1.0000000f));
  const float2 tt = unf2(t), pv = unf2(p);
  const uint32_t r0 = __float_as_uint(tt.x) * (1u << 23) + __float_as_uint(pv.x);
  const uint32_t r1 = __float_as_uint(tt.y) * (1u << 23) + __float_as_uint(pv.y);
  return f2(__uint_as_float(r0), __uint_as_float(r1));
}
template <int kVariant>
#ifndef LB
#define LB 256
#endif
__global__ void __launch_bounds__(LB, 1) k(const float* in, uint32_t* out, long long* cyc, int steps, int nsoft) {
  __shared__ __align__(8) uint64_t done_bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(&done_bar))));
  __syncthreads();
  const uint32_t db = static_cast<uint32_t>(__cvta_generic_to_shared(&done_bar));
  float s[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  __shared__ uint32_t tmem_sh;
  if (TM && threadIdx.x < 32) {
    neo::umma::tmem_alloc(static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_sh)), 512);
    neo::umma::tmem_relinquish();
  }
  neo::umma::fence_before_sync();
  __syncthreads();
  neo::umma::fence_after_sync();
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t tS = tmem_sh + ((warp & 3) * 32 << 16) + (warp / 4) * 256;
  float m = -1e30f;
  uint64_t l2 = f2(0.f, 0.f);
  uint32_t acc = 0;
  const float sl = 0.127f;
  __syncthreads();
  if (static_cast<int>(threadIdx.x / 32) >= nsoft) {   // spinner
    asm volatile(
        "{\n.reg .pred P1;\nW:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W;\n}\n" ::"r"(db) : "memory");
    return;
  }
  long long t0 = clock64();
  for (int j = 0; j < steps; ++j) {
    if (TM) {
      uint32_t u[4][32];
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) neo::umma::ld32(tS + c0, u[c0 / 32]);
      neo::umma::wait_ld();
#pragma unroll
      for (int c = 0; c < 128; ++c) s[c] += __uint_as_float(u[c / 32][c % 32]);
    }
    float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 128; c += 8)
#pragma unroll
      for (int q = 0; q < 4; ++q) mq[q] = fmaxf(mq[q], fmaxf(s[c + 2 * q], s[c + 2 * q + 1]));
    const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
    m = fmaxf(m, mx);
    const uint64_t sl2 = f2(sl, sl), nm2 = f2(7.f - m * sl, 7.f - m * sl);
    uint64_t la = f2(0.f, 0.f), lb = f2(0.f, 0.f);
    uint32_t hw[64];
#pragma unroll
    for (int w = 0; w < 64; ++w) {
      const uint64_t xx = ffma2(f2(s[2 * w], s[2 * w + 1]), sl2, nm2);
      float p0, p1;
      if ((w & 3) < POLY) {
        const float2 pp = unf2(DEG3 ? exp2_poly3(xx) : exp2_poly2(xx));
        p0 = pp.x;
        p1 = pp.y;
      } else {
        const float2 x = unf2(xx);
        p0 = ex2(x.x);
        p1 = ex2(x.y);
      }
      if (w & 1) lb = fadd2(lb, f2(p0, p1));
      else la = fadd2(la, f2(p0, p1));
      hw[w] = pack_f16(p0, p1);
    }
    l2 = fadd2(l2, fadd2(la, lb));
#pragma unroll
    for (int w = 0; w < 64; ++w) acc ^= hw[w];
    if (TM) {
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) neo::umma::st16(tS + c0 / 2, *reinterpret_cast<const uint32_t(*)[16]>(&hw[c0 / 2]));
      neo::umma::wait_st();
    }
    // perturb s so the loop is not hoisted
#pragma unroll
    for (int c = 0; c < 128; c += 16) s[c] += __uint_as_float(acc & 0x00000001u);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(db) : "memory");
  if (TM && threadIdx.x < 32) neo::umma::tmem_dealloc(tmem_sh, 512);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(unf2(l2).x);
  if (threadIdx.x % 32 == 0) cyc[threadIdx.x / 32] = t1 - t0;
}
int main() {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 64 * 8);
  for (int w : {1, 4, 8}) {
    const int steps = 100;
    k<0><<<1, 32 * (w + (SPIN ? 4 : 0))>>>(in, out, cyc, steps, w);
    cudaDeviceSynchronize();
    long long h[64];
    cudaMemcpy(h, cyc, 8 * w, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < w; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("warps %d (%d per SMSP): %.0f cycles per 128-column row step\n", w, (w + 3) / 4, mx / steps);
  }
  return 0;
}
