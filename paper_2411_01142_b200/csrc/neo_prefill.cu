// Causal paged GQA prefill attention for sm_100a on the 5th-generation tensor
// cores (the prefill half of batch-0).
//
// CTA = (request b, kv-head g, M tile of 128 query rows).  Row r of the tile is
// (query token i0 + r / G, q-head g*G + r % G): the G heads sharing a KV head
// are packed into the M dimension so each K/V tile is read once per M tile.
// Key tiles of kBN = 64 tokens stream through a kStages-deep TMA ring straight
// from the KV pages (one 2 KiB box per 16 tokens and dim-half).
//
//   warp 4     TMA producer: Q once, then K and V tiles (block-table lookups)
//   warp 5     TMEM owner + MMA issuer (one lane):
//                S_j  = Q . K_j^T          tcgen05.mma M128 N64  K128 -> TMEM (2 buffers)
//                O   += P_j . V_j          tcgen05.mma M128 N128 K64  -> TMEM, P = hi + lo
//   warps 0-3  softmax: thread r owns row r (TMEM lane r): scores via tcgen05.ld,
//              causal mask, online softmax in the exp2 domain with a lazy
//              rescale (only when the row max grows by > 2^8), P written to
//              shared memory as bf16 hi + lo parts (two MMAs keep ~16 mantissa
//              bits of P, the SURVEY §8(c) rule), O rescaled in TMEM when needed,
//              final O / l stored as bf16.
// S_{j+1} runs on the tensor core while the softmax warps work on S_j; P is
// double-buffered so PV_j overlaps softmax j+1.
#include <cuda_bf16.h>

#include <cstdio>

#include "neo_internal.cuh"
#include "umma.cuh"

namespace neo {
namespace {

constexpr int kBM = 128;                        // query rows per CTA (TMEM lanes)
constexpr int kBN = 64;                         // keys per tile
constexpr int kStages = 3;                      // K/V ring depth
constexpr int kQHalf = kBM * 128;               // 16 KiB: one dim-half of Q
constexpr int kKVHalf = kBN * 128;              // 8 KiB: one dim-half of a K or V tile
constexpr int kKVBytes = 2 * kKVHalf;
constexpr int kPBytes = kBM * kBN * 2;          // 16 KiB: P hi (or lo) of one tile
constexpr int kOffK = 2 * kQHalf;
constexpr int kOffV = kOffK + kStages * kKVBytes;
constexpr int kOffP = kOffV + kStages * kKVBytes;
constexpr int kSmemBytes = kOffP + 2 * 2 * kPBytes;   // 192 KiB
constexpr int kSmemAlloc = kSmemBytes + 1024;          // + alignment slack
constexpr uint32_t kTmemCols = 256;                    // S[2] (2 x 64) + O (128)
constexpr uint32_t kColO = 2 * kBN;
constexpr uint32_t kIdescS = umma::idesc_bf16_f32(kBM, kBN, false, false);
constexpr uint32_t kIdescO = umma::idesc_bf16_f32(kBM, 128, false, true);
constexpr int kThreads = 192;

// barrier slots
constexpr int kBarQ = 0, kBarKFull = 1, kBarVFull = kBarKFull + kStages, kBarKVEmpty = kBarVFull + kStages,
              kBarSFull = kBarKVEmpty + kStages, kBarSFree = kBarSFull + 2, kBarPFull = kBarSFree + 2,
              kBarPVDone = kBarPFull + 2, kNumBars = kBarPVDone + 2;

struct PArgs {
  uint16_t* out;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const int32_t* q_offsets;
  int32_t hq, G, page_size, max_blocks;
  float scale_log2;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            int c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    prefill_attn_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                        const __grid_constant__ CUtensorMap tmv, const PArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[kNumBars];
  __shared__ uint32_t tmem_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.z, g = blockIdx.y;
  const int G = a.G, rows_tok = kBM / G;

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int q0 = a.q_offsets[b];
  const int q_len = a.q_offsets[b + 1] - q0;
  const int n_mt = (q_len + rows_tok - 1) / rows_tok;
  const int mt = static_cast<int>(gridDim.x) - 1 - static_cast<int>(blockIdx.x);   // longest tiles first
  if (mt >= n_mt) return;
  const int ctx = a.seq_lens[b];
  const int i0 = mt * rows_tok;
  const int pos_last = ctx - q_len + min(i0 + rows_tok, q_len) - 1;
  const int nt = pos_last / kBN + 1;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto bar = [bar0](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };

  if (threadIdx.x == 0) {
    mbar_init(bar(kBarQ), 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(kBarKFull + s), 1);
      mbar_init(bar(kBarVFull + s), 1);
      mbar_init(bar(kBarKVEmpty + s), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), 4);
      mbar_init(bar(kBarPFull + i), 4);
      mbar_init(bar(kBarPVDone + i), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {
    umma::tmem_alloc(smem_u32(&tmem_sh), kTmemCols);
    umma::tmem_relinquish();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tmem_sh;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv)) : "memory");
      mbar_expect_tx(bar(kBarQ), 2 * kQHalf);
      for (int h = 0; h < 2; ++h) tma_load_4d(sb + h * kQHalf, &tmq, 0, g * G, q0 + i0, h, bar(kBarQ));
      const int32_t* bt = a.block_table + static_cast<int64_t>(b) * a.max_blocks;
      for (int j = 0; j < nt; ++j) {
        const int st = j % kStages;
        if (j >= kStages) mbar_wait(bar(kBarKVEmpty + st), ((j / kStages) - 1) & 1);
        const int kv0 = j * kBN;
        const int groups = min(kBN / 16, (ctx - kv0 + 15) / 16);
        const uint32_t bytes = static_cast<uint32_t>(groups) * 2 * 2048;
        int page[kBN / 16], slot[kBN / 16];
        for (int u = 0; u < groups; ++u) {
          const int t = kv0 + 16 * u;
          page[u] = bt[t / a.page_size];
          slot[u] = t % a.page_size;
        }
        const uint32_t dk = sb + kOffK + st * kKVBytes, dv = sb + kOffV + st * kKVBytes;
        mbar_expect_tx(bar(kBarKFull + st), bytes);
        for (int u = 0; u < groups; ++u)
          for (int h = 0; h < 2; ++h)
            tma_load_5d(dk + h * kKVHalf + u * 2048, &tmk, 0, slot[u], h, g, page[u], bar(kBarKFull + st));
        mbar_expect_tx(bar(kBarVFull + st), bytes);
        for (int u = 0; u < groups; ++u)
          for (int h = 0; h < 2; ++h)
            tma_load_5d(dv + h * kKVHalf + u * 2048, &tmv, 0, slot[u], h, g, page[u], bar(kBarVFull + st));
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    mbar_wait(bar(kBarQ), 0);
    umma::fence_after_sync();
    for (int j = 0; j <= nt; ++j) {
      if (j < nt) {
        const int st = j % kStages;
        mbar_wait(bar(kBarKFull + st), (j / kStages) & 1);
        if (j >= 2) mbar_wait(bar(kBarSFree + (j & 1)), ((j - 2) >> 1) & 1);
        umma::fence_after_sync();
        if (lane == 0) {
          const uint32_t kb = sb + kOffK + st * kKVBytes;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = umma::desc_sw128(sb + (kk >> 2) * kQHalf + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = umma::desc_sw128(kb + (kk >> 2) * kKVHalf + (kk & 3) * 32, 16, 1024);
            umma::mma_bf16(tmem + (j & 1) * kBN, ad, bd, kIdescS, kk > 0);
          }
          umma::commit(bar(kBarSFull + (j & 1)));
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int i = j - 1, st = i % kStages;
        mbar_wait(bar(kBarPFull + (i & 1)), (i >> 1) & 1);
        mbar_wait(bar(kBarVFull + st), (i / kStages) & 1);
        const int nvalid = min(kBN, ctx - i * kBN);
        const int ksteps = (nvalid + 15) / 16;
        const uint32_t vb = sb + kOffV + st * kKVBytes;
        if (nvalid & 15) {
          // rows nvalid .. 16*ksteps-1 hold page-tail slots: zero them (P is 0
          // there, but 0 * NaN would poison O)
          const int r0 = nvalid, nrows = 16 * ksteps - nvalid;
          for (int e = lane; e < nrows * 2 * 8; e += 32) {
            const int row = r0 + e / 16, h = (e / 8) & 1, c = e & 7;
            sts128(vb + h * kKVHalf + row * 128 + c * 16, 0, 0, 0, 0);
          }
          umma::fence_proxy_async_smem();
        }
        __syncwarp();
        umma::fence_after_sync();
        if (lane == 0) {
          const uint32_t pb = sb + kOffP + (i & 1) * 2 * kPBytes;
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t vd = umma::desc_sw128(vb + k * 2048, kKVHalf, 1024);
            const uint64_t ph = umma::desc_sw128(pb + k * 32, 16, 1024);
            const uint64_t pl = umma::desc_sw128(pb + kPBytes + k * 32, 16, 1024);
            umma::mma_bf16(tmem + kColO, ph, vd, kIdescO, i > 0 || k > 0);
            umma::mma_bf16(tmem + kColO, pl, vd, kIdescO, true);
          }
          umma::commit(bar(kBarPVDone + (i & 1)));
          umma::commit(bar(kBarKVEmpty + st));
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int r = threadIdx.x;                      // row == TMEM lane
    const int i_row = i0 + r / G;
    const bool valid_row = i_row < q_len;
    const int pos = ctx - q_len + min(i_row, q_len - 1);
    const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
    const float sl = a.scale_log2;
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < nt; ++j) {
      mbar_wait(bar(kBarSFull + (j & 1)), (j >> 1) & 1);
      umma::fence_after_sync();
      uint32_t s0[32], s1[32];
      umma::ld32(tmem + lane_base + (j & 1) * kBN, s0);
      umma::ld32(tmem + lane_base + (j & 1) * kBN + 32, s1);
      umma::wait_ld();
      umma::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(kBarSFree + (j & 1)));

      const int kv0 = j * kBN;
      float x[kBN];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        x[c] = __uint_as_float(s0[c]) * sl;
        x[c + 32] = __uint_as_float(s1[c]) * sl;
      }
      if (kv0 + kBN - 1 > pos) {
#pragma unroll
        for (int c = 0; c < kBN; ++c)
          if (kv0 + c > pos) x[c] = -INFINITY;
      }
      float mx = x[0];
#pragma unroll
      for (int c = 1; c < kBN; ++c) mx = fmaxf(mx, x[c]);
      const float m_new = fmaxf(m_ref, mx);
      bool resc = false;
      float alpha = 1.f;
      if (j == 0) {
        m_ref = m_new;
      } else if (m_new > m_ref + 8.f) {
        resc = true;
        alpha = ex2(m_ref - m_new);
        m_ref = m_new;
        l *= alpha;
      }
      if (j >= 2) mbar_wait(bar(kBarPVDone + (j & 1)), ((j - 2) >> 1) & 1);   // P buffer free
      const uint32_t pb = sb + kOffP + (j & 1) * 2 * kPBytes;
#pragma unroll
      for (int c8 = 0; c8 < kBN / 8; ++c8) {
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float p0 = ex2(x[c8 * 8 + 2 * w] - m_ref);
          const float p1 = ex2(x[c8 * 8 + 2 * w + 1] - m_ref);
          l += p0 + p1;
          hw[w] = pack_bf16(p0, p1);
          lw[w] = pack_bf16(p0 - bf_lo(hw[w]), p1 - bf_hi(hw[w]));
        }
        const uint32_t off = umma::sw128_off(r, c8);
        sts128(pb + off, hw[0], hw[1], hw[2], hw[3]);
        sts128(pb + kPBytes + off, lw[0], lw[1], lw[2], lw[3]);
      }
      umma::fence_proxy_async_smem();
      if (__any_sync(0xffffffffu, resc)) {
        // O must hold PV_{j-1} before it is scaled
        mbar_wait(bar(kBarPVDone + ((j - 1) & 1)), ((j - 1) >> 1) & 1);
        umma::fence_after_sync();
#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t o[32];
          umma::ld32(tmem + lane_base + kColO + c0, o);
          umma::wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
          umma::st32(tmem + lane_base + kColO + c0, o);
        }
        umma::wait_st();
        umma::fence_before_sync();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(kBarPFull + (j & 1)));
    }
    // epilogue: O / l -> bf16
    mbar_wait(bar(kBarPVDone + ((nt - 1) & 1)), ((nt - 1) >> 1) & 1);
    umma::fence_after_sync();
    const float inv_l = 1.f / l;
    uint16_t* orow = a.out + (static_cast<int64_t>(q0 + min(i_row, q_len - 1)) * a.hq + g * G + r % G) * 128;
#pragma unroll 1
    for (int c0 = 0; c0 < 128; c0 += 32) {
      uint32_t o[32];
      umma::ld32(tmem + lane_base + kColO + c0, o);
      umma::wait_ld();
      if (valid_row) {
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          uint4 v;
          v.x = pack_bf16(__uint_as_float(o[c + 0]) * inv_l, __uint_as_float(o[c + 1]) * inv_l);
          v.y = pack_bf16(__uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l);
          v.z = pack_bf16(__uint_as_float(o[c + 4]) * inv_l, __uint_as_float(o[c + 5]) * inv_l);
          v.w = pack_bf16(__uint_as_float(o[c + 6]) * inv_l, __uint_as_float(o[c + 7]) * inv_l);
          *reinterpret_cast<uint4*>(orow + c0 + c) = v;
        }
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 5) umma::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace

int prefill_m_tiles(int32_t max_q_len, int32_t G) { return (max_q_len * G + kBM - 1) / kBM; }

neo_status launch_prefill_attn(const PrefillLaunch& L, const CUtensorMap& tmq, const CUtensorMap& tmk,
                               const CUtensorMap& tmv) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return cuda_fail(e, "prefill smem attribute");
    attr_set = true;
  }
  const int G = L.hq / L.hkv;
  PArgs a{static_cast<uint16_t*>(L.out), L.block_table, L.seq_lens, L.q_offsets, L.hq, G, L.page_size, L.max_blocks,
          L.scale * 1.4426950408889634f};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(prefill_m_tiles(L.max_q_len, G), L.hkv, L.batch);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemAlloc;
  cfg.stream = L.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, prefill_attn_kernel, tmq, tmk, tmv, a);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NEO_OK : cuda_fail(e, "prefill attention kernel launch");
}

}  // namespace neo
