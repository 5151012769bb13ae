// tcgen05 (5th-generation tensor core) building blocks for sm_100a: shared-memory
// matrix descriptors, the kind::f16 instruction descriptor, TMEM allocation,
// MMA issue / commit and TMEM <-> register moves.  Bit layouts follow the
// sm_100 UMMA descriptor formats (the same fields CuTe's UMMA::SmemDescriptor and
// UMMA::InstrDescriptor name); tools/umma_probe.cu checks every encoding used
// here against a CPU GEMM on the B200.
#pragma once
#include <cstdint>

namespace neo {
namespace umma {

// ---- shared-memory matrix descriptor (64 bit)
//   [0,14)  start address >> 4      [16,30) leading-dim byte offset >> 4
//   [32,46) stride-dim byte offset >> 4
//   [46,48) version = 1 (sm_100)    [49,52) base offset (0: atoms 1024-B aligned)
//   [61,64) layout: 2 = SWIZZLE_128B
// K-major SW128 operand (rows of 128 B = 64 bf16 along K, 8-row atoms of 1 KiB):
//   SBO = byte stride between 8-row groups, LBO unused (16 B).
// MN-major SW128 operand (rows of 128 B = 64 bf16 along M/N, 8 K-rows per atom):
//   LBO = byte stride between 64-element M/N groups, SBO = byte stride between
//   8-row K groups.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// ---- instruction descriptor, kind::f16 with bf16 A/B and fp32 D
//   [4,6) D format (1 = f32)  [7,10) A format (1 = bf16)  [10,13) B format (1 = bf16)
//   [15] A major (0 = K, 1 = MN)  [16] B major  [17,23) N >> 3  [24,29) M >> 4
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn_major) << 15) |
         (static_cast<uint32_t>(b_mn_major) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// ---- the same with f16 A and B (formats 0)
__host__ __device__ constexpr uint32_t idesc_f16_f32(int M, int N, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (static_cast<uint32_t>(a_mn_major) << 15) | (static_cast<uint32_t>(b_mn_major) << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// ---- TMEM allocation (one full warp executes these)
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- D[tmem] (+)= A[smem] . B[smem]   (one thread issues for the CTA)
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         bool accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate))
      : "memory");
}

// ---- D[tmem] (+)= A[tmem] . B[smem]: A (M x K, K-major) in TMEM, row m = lane m,
// column c = the bf16 pair (2c, 2c + 1) of that row's K elements
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            bool accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate))
      : "memory");
}

// ---- whole MMA blocks issued from one PTX block by one elected lane of the
// calling warp (all 32 lanes must call): the address arithmetic stays in the
// block, so the issue path is one add + one tcgen05.mma per instruction.
//
// S block: D (+)= A . B^T over K = 128 as 8 K16 steps; A, B K-major SW128 with
// the two 64-element K halves `half_a` / `half_b` bytes apart.
template <uint32_t kHalfA, uint32_t kHalfB>
__device__ __forceinline__ void mma_block_k128(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  constexpr uint64_t ha = kHalfA / 16, hb = kHalfB / 16;
  asm volatile(
      "{\n"
      ".reg .pred e, pf, pt;\n"
      ".reg .b64 a1, a2, a3, a4, a5, a6, a7, b1, b2, b3, b4, b5, b6, b7;\n"
      "setp.ne.b32 pf, 0, 0;\n"
      "setp.eq.b32 pt, 0, 0;\n"
      "add.s64 a1, %1, 2;\n add.s64 a2, %1, 4;\n add.s64 a3, %1, 6;\n"
      "add.s64 a4, %1, %4;\n add.s64 a5, a4, 2;\n add.s64 a6, a4, 4;\n add.s64 a7, a4, 6;\n"
      "add.s64 b1, %2, 2;\n add.s64 b2, %2, 4;\n add.s64 b3, %2, 6;\n"
      "add.s64 b4, %2, %5;\n add.s64 b5, b4, 2;\n add.s64 b6, b4, 4;\n add.s64 b7, b4, 6;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, pt;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "n"(ha), "n"(hb)
      : "memory");
}

// PV block: D (+)= (A_hi + A_lo) . B over K = 128 as 8 K16 steps, A_hi / A_lo in
// TMEM at columns a, a + 64 (8 columns per step), B MN-major SW128 advancing
// 2 KiB per step.  `acc0` = accumulate into D on the first step.
__device__ __forceinline__ void mma_block_pv128(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                                bool acc0) {
  asm volatile(
      "{\n"
      ".reg .pred e, p0, pt;\n"
      ".reg .b32 h1, h2, h3, h4, h5, h6, h7, l0, l1, l2, l3, l4, l5, l6, l7;\n"
      ".reg .b64 b1, b2, b3, b4, b5, b6, b7;\n"
      "setp.ne.b32 p0, %4, 0;\n"
      "setp.eq.b32 pt, 0, 0;\n"
      "add.u32 h1, %1, 8;\n add.u32 h2, %1, 16;\n add.u32 h3, %1, 24;\n add.u32 h4, %1, 32;\n"
      "add.u32 h5, %1, 40;\n add.u32 h6, %1, 48;\n add.u32 h7, %1, 56;\n"
      "add.u32 l0, %1, 64;\n add.u32 l1, %1, 72;\n add.u32 l2, %1, 80;\n add.u32 l3, %1, 88;\n"
      "add.u32 l4, %1, 96;\n add.u32 l5, %1, 104;\n add.u32 l6, %1, 112;\n add.u32 l7, %1, 120;\n"
      "add.s64 b1, %2, 128;\n add.s64 b2, %2, 256;\n add.s64 b3, %2, 384;\n add.s64 b4, %2, 512;\n"
      "add.s64 b5, %2, 640;\n add.s64 b6, %2, 768;\n add.s64 b7, %2, 896;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l0], %2, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], b1, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l1], b1, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], b2, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l2], b2, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], b3, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l3], b3, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h4], b4, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l4], b4, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h5], b5, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l5], b5, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h6], b6, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l6], b6, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h7], b7, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [l7], b7, %3, pt;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(acc0))
      : "memory");
}

// PV block with a single-precision-class P: D (+)= A . B over K = 128 as 8 K16
// steps, A in TMEM at columns a + 8k, B MN-major SW128 advancing 2 KiB per step.
__device__ __forceinline__ void mma_block_pv128_single(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                       uint32_t idesc, bool acc0) {
  asm volatile(
      "{\n"
      ".reg .pred e, p0, pt;\n"
      ".reg .b32 h1, h2, h3, h4, h5, h6, h7;\n"
      ".reg .b64 b1, b2, b3, b4, b5, b6, b7;\n"
      "setp.ne.b32 p0, %4, 0;\n"
      "setp.eq.b32 pt, 0, 0;\n"
      "add.u32 h1, %1, 8;\n add.u32 h2, %1, 16;\n add.u32 h3, %1, 24;\n add.u32 h4, %1, 32;\n"
      "add.u32 h5, %1, 40;\n add.u32 h6, %1, 48;\n add.u32 h7, %1, 56;\n"
      "add.s64 b1, %2, 128;\n add.s64 b2, %2, 256;\n add.s64 b3, %2, 384;\n add.s64 b4, %2, 512;\n"
      "add.s64 b5, %2, 640;\n add.s64 b6, %2, 768;\n add.s64 b7, %2, 896;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], b1, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], b2, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], b3, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h4], b4, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h5], b5, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h6], b6, %3, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [h7], b7, %3, pt;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(acc0))
      : "memory");
}

// commit from one elected lane of the calling warp (all 32 lanes call)
__device__ __forceinline__ void commit_elect(uint32_t bar_smem) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(bar_smem)
      : "memory");
}

// arrive (once) on an mbarrier when every previously issued MMA of this thread completes
__device__ __forceinline__ void commit(uint32_t bar_smem) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_smem)
               : "memory");
}

// ---- TMEM -> registers: lane (warp's 32-lane quarter + laneid), 32 consecutive columns
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TMEM address of (lane, column): lane in bits [16,32), column in [0,16)
__device__ __forceinline__ uint32_t taddr(uint32_t base, uint32_t lane, uint32_t col) {
  return base + (lane << 16) + col;
}

// Byte offset, inside a SW128 region written row by row (1024-B aligned), of
// the 16-byte chunk `c` (0..7) of 128-byte row `r`: TMA's SWIZZLE_128B pattern.
__host__ __device__ constexpr uint32_t sw128_off(uint32_t r, uint32_t c) { return r * 128u + ((c ^ (r & 7u)) << 4); }

}  // namespace umma
}  // namespace neo
