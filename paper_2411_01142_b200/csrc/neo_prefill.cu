// Causal paged GQA prefill attention for sm_100a on the 5th-generation tensor
// cores (the prefill half of batch-0).  Two kernels
// share the tiles, the math and the TMEM layout described here:
//   prefill_attn_kernel         item-major (this header), prompts > 3072 tokens
//                               and the bf16 hi + lo P path (< 256 tokens);
//   prefill_attn_stream_kernel  warp-specialised stream (its own header below),
//                               fp16 P.V for prompts of 256 .. 3072 tokens.
//
// CTA = (request b, kv-head g, two M tiles of 128 query rows).  Row r of a tile
// is (query token, q-head g*G + r % G): the G heads sharing a KV head are packed
// into M, so each K/V tile is read once for 2 x 128 rows.  Key tiles of kBN =
// 128 tokens stream through a 2-stage TMA ring straight from the KV pages (one
// 2 KiB box per 16 tokens and dim-half).
//
//   warp 8     TMA producer: Q once, then K and V tiles (block-table lookups)
//   warp 9     TMEM owner + MMA issuer (one lane), ping-pong over the two tiles:
//                S_j(t)  = Q_t . K_j^T     tcgen05.mma SS  M128 N128 K128 -> TMEM
//                O(t)   += P_j(t) . V_j    tcgen05.mma TS  M128 N128 K128, P read
//                                          from TMEM (aliasing S_j(t)), hi + lo
//              issue order PV_j(0) S_j+1(0) PV_j(1) S_j+1(1): the tensor core runs
//              one tile's PV + next S while the other tile's softmax runs.
//   warps 0-3  softmax of tile 0, warps 4-7 of tile 1: thread = row = TMEM lane.
//              Scores via tcgen05.ld, causal mask, online softmax in the exp2
//              domain (scale folded into one FFMA) with a lazy rescale (only
//              when the row max grows by > 2^8; O rescaled in TMEM), P split into
//              bf16 hi + lo by truncation (hi = top 16 bits, lo = top 16 bits
//              of the exact remainder: ~16 significant bits, the SURVEY §8(c)
//              rule for P.V on tensor cores) and written back over S with
//              tcgen05.st; final O / l stored as bf16.
// tcgen05 ops of the issuing thread complete in order, so the commit that
// signals S_j+1(t) also proves PV_j(t) done: the softmax may rescale O then,
// and S_j+1(t) may overwrite P_j(t) without further barriers.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "neo_internal.cuh"
#include "umma.cuh"

namespace neo {
namespace {

constexpr int kBM = 128;                        // query rows per tile (TMEM lanes)
constexpr int kTiles = 2;                       // tiles per CTA (ping-pong)
constexpr int kBN = 128;                        // keys per tile
constexpr int kStages = 2;                      // K/V ring depth
constexpr int kQHalf = kBM * 128;               // 16 KiB: one dim-half of a Q tile
constexpr int kKVHalf = kBN * 128;              // 16 KiB: one dim-half of a K or V tile
constexpr int kOffK = kTiles * 2 * kQHalf;      // 64 KiB of Q
constexpr int kStageBytes = 4 * kKVHalf;        // K then V: 64 KiB
constexpr int kSmemBytes = kOffK + kStages * kStageBytes;   // 192 KiB
constexpr int kSmemAlloc = kSmemBytes + 1024;               // + alignment slack
constexpr uint32_t kTmemCols = 512;             // per tile: S/P (128) + O (128)
constexpr uint32_t kTileCols = 256;
constexpr uint32_t kColO = 128;
// P.V precision (DESIGN "prefill P.V"), a template parameter of the kernel:
//  - kHiLo = false (prompts of >= kFp16MinQLen tokens): P.V in fp16 -- P (scaled
//    by 2^7, <= 2^15 under the lazy rescale) rounded to fp16 in TMEM, V converted
//    bf16 -> fp16 in place in shared memory by the softmax warps at the start of
//    each step -- one MMA per K16 step; a quarter of the exponentials run on the
//    FMA pipe (exp2_poly2);
//  - kHiLo = true (short prompts, where the conversion does not pay): P split
//    into bf16 hi + lo by truncation, two MMAs per step, V bf16 as loaded.
constexpr int kFp16MinQLen = 256;
constexpr int kStreamMaxQLen = 3072;             // fp16 path: stream kernel up to here, item-major above
#ifndef NEO_PF_EXP
#define NEO_PF_EXP 0   // timing experiments only (results wrong): 1 no V conversion, 2 no softmax math + no conversion, 3 no softmax math, 4 (stream kernel) no MMAs (softmax math and conversion kept)
#endif
constexpr uint32_t kIdescS = umma::idesc_bf16_f32(kBM, kBN, false, false);
constexpr int kThreads = 320;
constexpr int kProducerWarp = 8, kMmaWarp = 9;

// barrier slots
constexpr int kBarQFull = 0, kBarQEmpty = 1, kBarKFull = 2, kBarVFull = kBarKFull + kStages, kBarKEmpty = kBarVFull + kStages,
              kBarVEmpty = kBarKEmpty + kStages, kBarSFull = kBarVEmpty + kStages, kBarPFull = kBarSFull + kTiles,
              kBarODone = kBarPFull + kTiles, kBarVConv = kBarODone + kTiles, kNumBars = kBarVConv + kStages;

struct PArgs {
  uint16_t* out;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const int32_t* q_offsets;
  int32_t batch, hq, hkv, G, page_size, max_blocks, n_ct_max;
  float scale_log2;
  int32_t epi_delay_ns;   // test knob (NEO_PREFILL_EPI_DELAY_NS): stream-kernel epilogue sleeps before each item
#ifdef NEO_PREFILL_TRACE
  long long* trace;   // [2 tiles][64 steps][16] clock64 stamps of CTA 0 (tools/prefill_trace.py)
#endif
};

#ifdef NEO_PREFILL_TRACE
}  // namespace
long long* g_prefill_trace = nullptr;
namespace {
#define TRACE(t, j, slot)                                                                          \
  do {                                                                                            \
    if (blockIdx.x == 0 && (j) < 64) a.trace[((t) * 64 + (j)) * 16 + (slot)] = clock64();           \
  } while (0)
#else
#define TRACE(t, j, slot) \
  do {                    \
  } while (0)
#endif

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
#ifdef NEO_PF_DEBUG_HANG
// debug build: report (block, warp, barrier offset, parity) and trap after 2^16 polls
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (uint32_t n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    if (n == (1u << 16)) {
      printf("HANG block %d warp %d lane %d bar+%u parity %u\n", blockIdx.x, threadIdx.x / 32, threadIdx.x % 32,
             bar & 0xffff, parity);
      __trap();
    }
  }
}
#else
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
#endif
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
// packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2 on sm_100)
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
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// bf16 pair -> fp16 pair (round to nearest even; beyond fp16's range saturates
// to +-65504 -- DESIGN "prefill P.V": V must lie within fp16's range)
__device__ __forceinline__ uint32_t bf16x2_to_f16x2(uint32_t w) {
  const float lo = __uint_as_float(w << 16), hi = __uint_as_float(w & 0xffff0000u);
  uint32_t r;
  asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// exp2 of a packed pair on the FMA pipe: round x to j with the 1.5 * 2^23
// shifter, 2^(x - j) by a degree-4 Taylor polynomial on [-0.5, 0.5] (relative
// error <= 4.3e-5, below fp16's 4.9e-4 rounding of P), exponent j added with one
// integer multiply-add per element.  x is clamped to >= -125 (keeps the biased
// exponent >= 1; 2^-125 is 0 after the fp16 rounding of P).
#ifndef NEO_PF_POLY
#define NEO_PF_POLY 0   // stream kernel's share (of 4 column pairs) on the FMA pipe: 0 measured best there
#endif
constexpr int kPolyPairsStream = NEO_PF_POLY;
constexpr int kPolyPairs = 1;   // of every 4 column pairs use exp2_poly2 (fp16 path; 2 or 3 measured slower)
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

// One work item = (request b, kv-head g, CTA tile ct: 2 x 128 rows).
struct Item {
  int b, g, q0, q_len, ctx, i0, nt0, nt1;
  // epilogue through shared memory + TMA stores: tile 0 stages in the last K
  // stage, tile 1 in the last V stage; both tiles must end on the same key tile
  __device__ __forceinline__ bool staged() const { return nt1 == 0 || nt0 == nt1; }
  // tile 1 stages in the last V stage only if the MMA warp did not zero a page
  // tail there (keeps every shared-memory write pair ordered by thread-level
  // barriers, not only through tcgen05.commit)
  __device__ __forceinline__ bool staged_v() const {
    const int nt = nt0 > nt1 ? nt0 : nt1;
    const int nvalid = min(kBN, ctx - (nt - 1) * kBN);
    return nt1 > 0 && nt0 == nt1 && (nvalid & 15) == 0;
  }
};

// Dense longest-first item list, built per CTA in shared memory by the
// prologue: level lv = 0, 1, ... is CTA tile ct = n_ct_max - 1 - lv (later
// query rows see more keys); a level holds every (request, kv-head) whose
// prompt chunk reaches that tile, requests in descending tile-count order.
//   req[i]    i-th request by descending tile count (ties: lower index first)
//   pref[lv]  items before level lv;  pref[n_ct_max] = total items
constexpr int kMaxSchedBatch = 512, kMaxSchedLevels = 1024;
struct Sched {
  int req[kMaxSchedBatch];
  int pref[kMaxSchedLevels + 1];
  int q_off[kMaxSchedBatch + 1];   // q_offsets and seq_lens cached: item lookup stays in shared memory
  int ctx[kMaxSchedBatch];
};

__device__ __forceinline__ int tiles_of_request(const PArgs& a, int b, int rows_tok) {
  const int q_len = a.q_offsets[b + 1] - a.q_offsets[b];
  return (q_len + kTiles * rows_tok - 1) / (kTiles * rows_tok);
}

// all threads of the CTA; ends with __syncthreads
__device__ void build_sched(const PArgs& a, int rows_tok, Sched& sc, int* nct_tmp) {
  for (int b = threadIdx.x; b < a.batch; b += blockDim.x) {
    // clamp: a request longer than max_q_len (caller error; NEO_DEBUG_VALIDATE
    // reports it) loses its tail rows instead of corrupting the item map
    nct_tmp[b] = min(tiles_of_request(a, b, rows_tok), a.n_ct_max);
    sc.q_off[b] = a.q_offsets[b];
    sc.ctx[b] = a.seq_lens[b];
  }
  if (threadIdx.x == 0) sc.q_off[a.batch] = a.q_offsets[a.batch];
  __syncthreads();
  for (int b = threadIdx.x; b < a.batch; b += blockDim.x) {
    const int n = nct_tmp[b];
    int rank = 0;
    for (int o = 0; o < a.batch; ++o) rank += nct_tmp[o] > n || (nct_tmp[o] == n && o < b);
    sc.req[rank] = b;
  }
  // pref[lv] = hkv * sum_b max(0, lv - (n_ct_max - n_b)): request b is present
  // on levels lv >= n_ct_max - n_b
  for (int lv = threadIdx.x; lv <= a.n_ct_max; lv += blockDim.x) {
    int c = 0;
    for (int o = 0; o < a.batch; ++o) c += max(0, lv - (a.n_ct_max - nct_tmp[o]));
    sc.pref[lv] = c * a.hkv;
  }
  __syncthreads();
}

// Item k of the dense list (k < sc.pref[n_ct_max]).
__device__ __forceinline__ void make_item(const PArgs& a, const Sched& sc, int k, int rows_tok, Item& it) {
  int lo = 0, hi = a.n_ct_max - 1;                 // last level with pref[lv] <= k
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sc.pref[mid] <= k) lo = mid;
    else hi = mid - 1;
  }
  const int ct = a.n_ct_max - 1 - lo;
  const int r = k - sc.pref[lo];
  it.b = sc.req[r / a.hkv];
  it.g = r % a.hkv;
  it.q0 = sc.q_off[it.b];
  it.q_len = sc.q_off[it.b + 1] - it.q0;
  it.ctx = sc.ctx[it.b];
  it.i0 = ct * kTiles * rows_tok;
  const int f0 = it.i0, f1 = it.i0 + rows_tok;
  it.nt0 = (it.ctx - it.q_len + min(f0 + rows_tok, it.q_len) - 1) / kBN + 1;
  it.nt1 = f1 < it.q_len ? (it.ctx - it.q_len + min(f1 + rows_tok, it.q_len) - 1) / kBN + 1 : 0;
}

// Persistent: one CTA per SM walks its snake-ordered share of the items; the
// TMA ring, the S/P and O TMEM buffers and all barrier phases run on across
// items, so one item's epilogue overlaps the next item's loads and first S.
template <bool kHiLo>
__global__ void __launch_bounds__(kThreads, 1)
    prefill_attn_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                        const __grid_constant__ CUtensorMap tmv, const __grid_constant__ CUtensorMap tmo,
                        const PArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[kNumBars];
  __shared__ uint32_t tmem_sh;
  constexpr float kPBias = kHiLo ? 0.f : 7.f;   // log2 scale of P in the fp16 path
  constexpr uint32_t kIdescO = kHiLo ? umma::idesc_bf16_f32(kBM, 128, false, true)
                                     : umma::idesc_f16_f32(kBM, 128, false, true);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G, rows_tok = kBM / G;
  __shared__ Sched sched;
  __shared__ int nct_tmp[kMaxSchedBatch];
  // snake order over the longest-first item list: round r takes item
  // r * grid + c (r even) or r * grid + grid - 1 - c (r odd), so the per-CTA
  // sums of the sorted costs balance
  auto first_item = [&](int round) {
    const int c = static_cast<int>(blockIdx.x), n = static_cast<int>(gridDim.x);
    return round * n + ((round & 1) ? n - 1 - c : c);
  };

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto bar = [bar0](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };

  if (threadIdx.x == 0) {
    mbar_init(bar(kBarQFull), 1);
    mbar_init(bar(kBarQEmpty), 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(kBarKFull + s), 1);
      mbar_init(bar(kBarVFull + s), 1);
      mbar_init(bar(kBarKEmpty + s), 1);
      mbar_init(bar(kBarVEmpty + s), 1);
      mbar_init(bar(kBarVConv + s), 8);   // 8 softmax-warp arrivals per V tile (fp16 path)
    }
    for (int t = 0; t < kTiles; ++t) {
      mbar_init(bar(kBarSFull + t), 1);
      mbar_init(bar(kBarPFull + t), 4);
      mbar_init(bar(kBarODone + t), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    umma::tmem_alloc(smem_u32(&tmem_sh), kTmemCols);
    umma::tmem_relinquish();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tmem_sh;

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");   // metadata and q may come from the previous kernel
  build_sched(a, rows_tok, sched, nct_tmp);
  const int n_items = sched.pref[a.n_ct_max];

  // registers: the softmax warpgroups hold a 128-column row each; the producer /
  // MMA / converter warpgroup needs few (setmaxnreg moves them, warpgroup-wide)
  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmq)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv)) : "memory");
    }
    uint32_t kc = 0, items = 0;                      // K/V tiles and items issued so far
    for (int round = 0, k = first_item(0); k < n_items; k = first_item(++round)) {
      Item it;
      make_item(a, sched, k, rows_tok, it);
      if (items > 0) mbar_wait(bar(kBarQEmpty), (items - 1) & 1);
      if (lane == 0) {
        const int nq = it.nt1 > 0 ? 2 : 1;
        mbar_expect_tx(bar(kBarQFull), nq * 2 * kQHalf);
        for (int t = 0; t < nq; ++t)
          for (int h = 0; h < 2; ++h)
            tma_load_4d(sb + (t * 2 + h) * kQHalf, &tmq, 0, it.g * G, it.q0 + it.i0 + t * rows_tok, h,
                        bar(kBarQFull));
      }
      ++items;
      const int32_t* bt = a.block_table + static_cast<int64_t>(it.b) * a.max_blocks;
      const int nt = max(it.nt0, it.nt1);
      for (int j = 0; j < nt; ++j, ++kc) {
        const int st = kc % kStages;
        const int kv0 = j * kBN;
        const int groups = min(kBN / 16, (it.ctx - kv0 + 15) / 16);
        int page = 0, slot = 0;
        if (lane < groups) {                       // lane u: page and slot of token group u
          const int t = kv0 + 16 * lane;
          page = bt[t / a.page_size];
          slot = t % a.page_size;
        }
        const uint32_t dk = sb + kOffK + st * kStageBytes, dv = dk + 2 * kKVHalf;
        const uint32_t bytes = static_cast<uint32_t>(groups) * 2 * 2048;
        if (kc >= kStages) mbar_wait(bar(kBarKEmpty + st), ((kc / kStages) - 1) & 1);
        if (lane == 0) mbar_expect_tx(bar(kBarKFull + st), bytes);
        __syncwarp();
        if (lane < groups)
          for (int h = 0; h < 2; ++h)
            tma_load_5d(dk + h * kKVHalf + lane * 2048, &tmk, 0, slot, h, it.g, page, bar(kBarKFull + st));
        if (kc >= kStages) mbar_wait(bar(kBarVEmpty + st), ((kc / kStages) - 1) & 1);
        if (lane == 0) mbar_expect_tx(bar(kBarVFull + st), bytes);
        __syncwarp();
        if (lane < groups)
          for (int h = 0; h < 2; ++h)
            tma_load_5d(dv + h * kKVHalf + lane * 2048, &tmv, 0, slot, h, it.g, page, bar(kBarVFull + st));
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // Descriptors are built once; every MMA then adds a compile-time offset
    // (start address >> 4 in the low bits), keeping the single-thread issue
    // path short enough for the tensor core to stay fed (tools/umma_rate.cu).
    const uint64_t dq0 = umma::desc_sw128(sb, 16, 1024), dq1 = umma::desc_sw128(sb + 2 * kQHalf, 16, 1024);
    const uint64_t dk0 = umma::desc_sw128(sb + kOffK, 16, 1024);
    const uint64_t dv0 = umma::desc_sw128(sb + kOffK + 2 * kKVHalf, kKVHalf, 1024);
    constexpr uint64_t kStageDesc = kStageBytes / 16;
    // all 32 lanes call; one elected lane issues (umma::mma_block_*)
    auto issue_s = [&](int t, int st) {
      umma::mma_block_k128<kQHalf, kKVHalf>(tmem + t * kTileCols, t ? dq1 : dq0,
                                            dk0 + static_cast<uint64_t>(st) * kStageDesc, kIdescS);
    };
    auto issue_pv = [&](int t, int st, int ksteps, bool acc0) {
      const uint32_t tp = tmem + t * kTileCols;
      const uint64_t bv = dv0 + static_cast<uint64_t>(st) * kStageDesc;
      if (!kHiLo) {            // fp16 P in columns [0, 64), one MMA per K16 step
        if (ksteps == 8) {
          umma::mma_block_pv128_single(tp + kColO, tp, bv, kIdescO, acc0);
        } else if (lane == 0) {
          for (int kq = 0; kq < ksteps; ++kq)
            umma::mma_bf16_ts(tp + kColO, tp + kq * 8, bv + (kq * 2048) / 16, kIdescO, kq > 0 || acc0);
        }
      } else if (ksteps == 8) {
        umma::mma_block_pv128(tp + kColO, tp, bv, kIdescO, acc0);
      } else if (lane == 0) {
        for (int kq = 0; kq < ksteps; ++kq) {
          umma::mma_bf16_ts(tp + kColO, tp + kq * 8, bv + (kq * 2048) / 16, kIdescO, kq > 0 || acc0);
          umma::mma_bf16_ts(tp + kColO, tp + 64 + kq * 8, bv + (kq * 2048) / 16, kIdescO, true);
        }
      }
      __syncwarp();
    };
    uint32_t kc = 0, vc = 0, items = 0, pc0 = 0, pc1 = 0;
    for (int round = 0, k = first_item(0); k < n_items; k = first_item(++round)) {
      Item it;
      make_item(a, sched, k, rows_tok, it);
      const int nt = max(it.nt0, it.nt1);
      mbar_wait(bar(kBarQFull), items & 1);
      ++items;
      mbar_wait(bar(kBarKFull + kc % kStages), (kc / kStages) & 1);
      umma::fence_after_sync();
      issue_s(0, kc % kStages);
      umma::commit_elect(bar(kBarSFull + 0));
      if (it.nt1 > 0) {
        issue_s(1, kc % kStages);
        umma::commit_elect(bar(kBarSFull + 1));
      }
      if (!(nt == 1 && it.staged()))                      // staged: tile 0's epilogue releases K_last
        umma::commit_elect(bar(kBarKEmpty + kc % kStages));  // K tile consumed once these S complete
      if (nt == 1) umma::commit_elect(bar(kBarQEmpty));    // last S of the item: Q free
      __syncwarp();
      ++kc;
      for (int j = 0; j < nt; ++j, ++vc) {
        const int st = vc % kStages;
        mbar_wait(bar((kHiLo ? kBarVFull : kBarVConv) + st), (vc / kStages) & 1);
        const int nvalid = min(kBN, it.ctx - j * kBN);
        const int ksteps = (nvalid + 15) / 16;
        const uint32_t vb = sb + kOffK + st * kStageBytes + 2 * kKVHalf;
        if (kHiLo && (nvalid & 15)) {
          // rows nvalid .. 16*ksteps-1 hold page-tail slots: zero them (P is 0
          // there, but 0 * NaN would poison O)
          const int nrows = 16 * ksteps - nvalid;
          for (int e = lane; e < nrows * 2 * 8; e += 32) {
            const int row = nvalid + e / 16, h = (e / 8) & 1, c = e & 7;
            sts128(vb + h * kKVHalf + row * 128 + c * 16, 0, 0, 0, 0);
          }
          umma::fence_proxy_async_smem();
        }
        __syncwarp();
        bool next_ready = false;
#pragma unroll
        for (int t = 0; t < kTiles; ++t) {
          const int ntt = t ? it.nt1 : it.nt0;
          if (j >= ntt) continue;
          if (lane == 0) TRACE(t, t ? pc1 : pc0, 4);
          mbar_wait(bar(kBarPFull + t), (t ? pc1 : pc0) & 1);
          if (lane == 0) TRACE(t, t ? pc1 : pc0, 5);
          if (t) ++pc1;
          else ++pc0;
          const bool more = j + 1 < ntt;
          if (more && !next_ready) {
            mbar_wait(bar(kBarKFull + kc % kStages), (kc / kStages) & 1);
            next_ready = true;
          }
          umma::fence_after_sync();
          issue_pv(t, st, ksteps, j > 0);
          const bool last_v = t == kTiles - 1 || j >= it.nt1;   // no later tile reads V_j / K_{j+1}
          // staged: tile 1's epilogue releases V_last (and tile 0's K_last, below)
          if (last_v && !(j == nt - 1 && it.staged_v())) umma::commit_elect(bar(kBarVEmpty + st));
          if (more) {
            issue_s(t, kc % kStages);
            umma::commit_elect(bar(kBarSFull + t));
            if (lane == 0) TRACE(t, (t ? pc1 : pc0) - 1, 6);
            if (last_v) {
              if (!(j + 2 == nt && it.staged())) umma::commit_elect(bar(kBarKEmpty + kc % kStages));
              if (j + 2 == nt) umma::commit_elect(bar(kBarQEmpty));   // last S of the item
            }
          } else {
            umma::commit_elect(bar(kBarODone + t));
          }
          __syncwarp();
        }
        if (next_ready) ++kc;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int t = warp >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;               // row == TMEM lane
    const uint32_t tS = tmem + t * kTileCols + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t tO = tS + kColO;
    const float sl = a.scale_log2;
    uint32_t sc = 0, oc = 0;                         // S tiles and items consumed so far
    uint32_t kbase = 0;                              // K/V tiles of earlier items (ring position)
    // fp16 path: V tile `vidx` bf16 -> fp16 in place, this warp's 16 of its 128
    // rows (all 8 softmax warps convert every V tile, in ring order, so no warp
    // ever waits on a phase two ahead of a stage's current one); rows past the
    // context zeroed (P = 0 there, but 0 * NaN = NaN)
    // Exception: the last V tile of an item whose tile 1 stages its output in
    // that V stage is converted by tile 1's warps alone (32 rows each, double
    // arrival), so every generic write to the stage before the staging comes
    // from the staging warp itself (ordered by __syncwarp, not only by the
    // mbarrier / tcgen05.commit chain, which racecheck does not model).
    const int wi = t * 4 + quarter;
    auto convert_v = [&](uint32_t vidx, int left, int row0, int nrow, int arrivals) {
      const int st = static_cast<int>(vidx % kStages);
      const int nvalid = min(kBN, left);
      const int rows = max(0, min(16 * ((nvalid + 15) / 16) - row0, nrow));
      const uint32_t vb = sb + kOffK + st * kStageBytes + 2 * kKVHalf;
      mbar_wait(bar(kBarVFull + st), (vidx / kStages) & 1);
      for (int e0 = 0; e0 < ((NEO_PF_EXP == 1 || NEO_PF_EXP == 2) ? 0 : rows * 16); e0 += 128) {
        uint32_t w[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = e0 + 32 * i + lane;
          const int row = row0 + (e >> 4);
          w[i][0] = w[i][1] = w[i][2] = w[i][3] = 0;
          if (e < rows * 16 && row < nvalid)
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3])
                         : "r"(vb + ((e >> 3) & 1) * kKVHalf + row * 128 + (e & 7) * 16));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = e0 + 32 * i + lane;
          const int row = row0 + (e >> 4);
          if (e < rows * 16)
            sts128(vb + ((e >> 3) & 1) * kKVHalf + row * 128 + (e & 7) * 16, bf16x2_to_f16x2(w[i][0]),
                   bf16x2_to_f16x2(w[i][1]), bf16x2_to_f16x2(w[i][2]), bf16x2_to_f16x2(w[i][3]));
        }
      }
      umma::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (arrivals == 1) mbar_arrive(bar(kBarVConv + st));
        else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], 2;" ::"r"(bar(kBarVConv + st)) : "memory");
      }
    };
    for (int round = 0, k = first_item(0); k < n_items; k = first_item(++round)) {
      if (quarter == 0 && lane == 0) TRACE(t, sc, 12);
      Item it;
      make_item(a, sched, k, rows_tok, it);
      if (quarter == 0 && lane == 0) TRACE(t, sc, 11);
      const int my_nt = t ? it.nt1 : it.nt0;
      const int nt_item = max(it.nt0, it.nt1);
      kbase += nt_item;
      if (my_nt == 0) {                            // single-tile item: tile 1 only converts
        if (!kHiLo)
          for (int j = 0; j < nt_item; ++j) convert_v(kbase - nt_item + j, it.ctx - j * kBN, wi * 16, 16, 1);
        continue;
      }
      const int i_row = it.i0 + t * rows_tok + r / G;
      const int pos = it.ctx - it.q_len + min(i_row, it.q_len - 1);
      float m = -INFINITY;
      uint64_t l2 = f2(0.f, 0.f);                   // row sum, two partial lanes
      for (int j = 0; j < my_nt; ++j, ++sc) {
        if (quarter == 0 && lane == 0) TRACE(t, sc, 0);
        if (quarter == 0 && lane == 0 && j == 0) TRACE(t, sc, 7);     // item start
        if (!kHiLo) {
          if (j == nt_item - 1 && it.staged_v()) {   // tile 1 stages into this V stage
            if (t == 1) convert_v(kbase - nt_item + j, it.ctx - j * kBN, quarter * 32, 32, 2);
          } else {
            convert_v(kbase - nt_item + j, it.ctx - j * kBN, wi * 16, 16, 1);
          }
        }
        mbar_wait(bar(kBarSFull + t), sc & 1);
        umma::fence_after_sync();
        if (quarter == 0 && lane == 0) TRACE(t, sc, 1);
        float s[kBN];
        {
          uint32_t u[32];
#pragma unroll
          for (int c0 = 0; c0 < kBN; c0 += 32) {
            umma::ld32(tS + c0, u);
            umma::wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) s[c0 + c] = __uint_as_float(u[c]);
          }
        }
        if (NEO_PF_EXP >= 2) {
          uint32_t hw[16];
#pragma unroll
          for (int w = 0; w < 16; ++w) hw[w] = __float_as_uint(s[w] * 0.f);
#pragma unroll
          for (int c0 = 0; c0 < kBN; c0 += 32) umma::st16(tS + c0 / 2, hw);
          l2 = f2(1.f, 1.f);
          umma::wait_st();
          umma::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(kBarPFull + t));
          continue;
        }
        const int lim = pos - j * kBN;               // last visible column of this row in the tile
        if (lim < kBN - 1) {
#pragma unroll
          for (int c = 0; c < kBN; ++c) s[c] = c > lim ? -INFINITY : s[c];
        }
        if (quarter == 0 && lane == 0) TRACE(t, sc, 2);
        float mx = s[0];
#pragma unroll
        for (int c = 1; c < kBN; ++c) mx = fmaxf(mx, s[c]);
        const float m_new = fmaxf(m, mx);
        bool resc = false;
        float alpha = 1.f;
        if (j == 0) {
          m = m_new;
        } else if ((m_new - m) * sl > 8.f) {
          resc = true;
          alpha = ex2((m - m_new) * sl);
          l2 = fmul2(l2, f2(alpha, alpha));
          m = m_new;
        }
        const uint64_t sl2 = f2(sl, sl), nm2 = f2(kPBias - m * sl, kPBias - m * sl);
        if (!kHiLo) {
          // fp16 P (scaled by 2^kPBias; l carries the same scale, so O / l is
          // unchanged) into columns [0, 64)
#pragma unroll
          for (int c0 = 0; c0 < kBN; c0 += 32) {
            uint32_t hw[16];
#pragma unroll
            for (int w = 0; w < 16; ++w) {
              const uint64_t xx = ffma2(f2(s[c0 + 2 * w], s[c0 + 2 * w + 1]), sl2, nm2);
              float p0, p1;
              if ((w & 3) < kPolyPairs) {      // exp2 on the FMA pipe (MUFU relief)
                const float2 pp = unf2(exp2_poly2(xx));
                p0 = pp.x;
                p1 = pp.y;
              } else {
                const float2 x = unf2(xx);
                p0 = ex2(x.x);
                p1 = ex2(x.y);
              }
              l2 = fadd2(l2, f2(p0, p1));
              hw[w] = pack_f16(p0, p1);
            }
            umma::st16(tS + c0 / 2, hw);
          }
        }
#pragma unroll
        for (int c0 = 0; c0 < (kHiLo ? kBN : 0); c0 += 32) {
          uint32_t hw[16], lw[16];
#pragma unroll
          for (int w = 0; w < 16; ++w) {
            const float2 x = unf2(ffma2(f2(s[c0 + 2 * w], s[c0 + 2 * w + 1]), sl2, nm2));
            const float p0 = ex2(x.x), p1 = ex2(x.y);
            const uint64_t pp = f2(p0, p1);
            l2 = fadd2(l2, pp);
            const uint32_t u0 = __float_as_uint(p0), u1 = __float_as_uint(p1);
            hw[w] = __byte_perm(u0, u1, 0x7632);
            const float2 rr =
                unf2(fsub2(pp, f2(__uint_as_float(u0 & 0xffff0000u), __uint_as_float(u1 & 0xffff0000u))));
            lw[w] = __byte_perm(__float_as_uint(rr.x), __float_as_uint(rr.y), 0x7632);
          }
          umma::st16(tS + c0 / 2, hw);          // hi: columns [0, 64)
          umma::st16(tS + 64 + c0 / 2, lw);     // lo: columns [64, 128)
        }
        if (__any_sync(0xffffffffu, resc)) {
          // PV_{j-1} is complete (the S_j commit covers it): scale O in place
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t o[32];
            umma::ld32(tO + c0, o);
            umma::wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            umma::st32(tO + c0, o);
          }
        }
        umma::wait_st();
        umma::fence_before_sync();
        __syncwarp();
        if (quarter == 0 && lane == 0) TRACE(t, sc, 3);
        if (lane == 0) mbar_arrive(bar(kBarPFull + t));
      }
      // epilogue: O / l -> bf16 (the next item's first PV on this tile waits for
      // this warpgroup's next P, so O stays intact until read)
      if (quarter == 0 && lane == 0) TRACE(t, sc - 1, 8);
      mbar_wait(bar(kBarODone + t), oc & 1);
      ++oc;
      umma::fence_after_sync();
      if (quarter == 0 && lane == 0) TRACE(t, sc - 1, 9);
      const float2 lp = unf2(l2);
      const float inv_l = 1.f / (lp.x + lp.y);
      if (t == 0 ? it.staged() : it.staged_v()) {
        // Stage the tile's rows in the freed last K (tile 0) / V (tile 1) stage
        // in TMA's SW128 layout (conflict-free 16-byte stores), then one TMA
        // tensor store per token and dim-half; rows past q_len are never written.
        const int st_last = static_cast<int>((kbase - 1) % kStages);
        const uint32_t buf = sb + kOffK + st_last * kStageBytes + (t ? 2 * kKVHalf : 0);

#pragma unroll 1
        for (int c0 = 0; c0 < 128; c0 += 32) {
          uint32_t o[32];
          umma::ld32(tO + c0, o);
          umma::wait_ld();
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int ch = c0 / 8 + q4;                // 16-byte chunk 0..15 of the row
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              w[e] = pack_bf16(__uint_as_float(o[8 * q4 + 2 * e]) * inv_l,
                               __uint_as_float(o[8 * q4 + 2 * e + 1]) * inv_l);
            sts128(buf + (ch >> 3) * kKVHalf + umma::sw128_off(r, ch & 7), w[0], w[1], w[2], w[3]);
          }
        }
        umma::fence_proxy_async_smem();
        __syncwarp();
        const int tpw = 32 / G;                        // tokens of this warp's 32 rows
        for (int e = lane; e < 2 * tpw; e += 32) {
          const int kk = e >> 1, h = e & 1;
          const int tok = it.i0 + t * rows_tok + quarter * tpw + kk;
          if (tok < it.q_len) {
            const uint32_t src = buf + h * kKVHalf + (quarter * 32 + kk * G) * 128;
            asm volatile(
                "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmo)),
                "r"(0), "r"(it.g * G), "r"(it.q0 + tok), "r"(h), "r"(src)
                : "memory");
          }
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // stage read: may be reused
        // the 4 warps of this tile done -> release the stage to the producer
        asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
        if (quarter == 0 && lane == 0) mbar_arrive(bar((t ? kBarVEmpty : kBarKEmpty) + st_last));
      } else {
      // 32-byte stores (full sectors): each thread writes its 256-byte row
      const int tok = it.i0 + t * rows_tok + r / G;
      uint16_t* orow = a.out + (static_cast<int64_t>(it.q0 + min(tok, it.q_len - 1)) * a.hq + it.g * G + r % G) * 128;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t o[32];
        umma::ld32(tO + c0, o);
        umma::wait_ld();
        if (tok < it.q_len) {
#pragma unroll
          for (int c = 0; c < 32; c += 16) {
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
              w[e] = pack_bf16(__uint_as_float(o[c + 2 * e]) * inv_l, __uint_as_float(o[c + 2 * e + 1]) * inv_l);
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(orow + c0 + c), "r"(w[0]),
                         "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                         : "memory");
          }
        }
      }
      }
      umma::fence_before_sync();
      if (quarter == 0 && lane == 0) TRACE(t, sc - 1, 10);
      // V tiles of steps this tile does not run (tile 0 when tile 1 sees more keys)
      if (!kHiLo)
        for (int j = my_nt; j < nt_item; ++j) convert_v(kbase - nt_item + j, it.ctx - j * kBN, wi * 16, 16, 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // output stores complete
  umma::fence_before_sync();
  __syncthreads();
  if (warp == kMmaWarp) umma::tmem_dealloc(tmem, kTmemCols);
}


// ============================================================================
// Stream kernel (fp16 P.V path, prompts >= kFp16MinQLen tokens).
//
// Same math and tile shapes as prefill_attn_kernel<false>, re-organised so an
// item boundary costs no pipeline drain (the clock64 trace of the item-major
// kernel showed ~6.5K cycles per boundary on 8 x 1024: epilogue stores 3.3K,
// item decode 1K, the next item's first S waiting for both tiles' epilogues):
//   * the MMA warp runs one continuous stream: after the last PV of an item on
//     tile t it issues the NEXT item's first S on tile t at once (per-tile Q
//     buffers, loaded by their own warp as soon as the tile's last S of the
//     previous item completes);
//   * a dedicated epilogue warpgroup (warps 8-11, one per TMEM lane quarter)
//     drains O / l of each finished tile, releases the O columns (o_free) and
//     stores bf16 rows straight to global, off the softmax critical path;
//   * both tiles of an item run the same number of key tiles (the earlier
//     tile's extra steps are fully masked and add exact zeros), so the S, P and
//     V pipelines of the two tiles stay in lock step across items;
//   * every CTA's item list is decoded once in the prologue into shared memory;
//   * setmaxnreg: 168 registers for the softmax warpgroups, 96 for the epilogue,
//     80 for the producer / MMA warpgroup (sum = the 128 x 512 launch pool).
//   warps 0-3 / 4-7  softmax of tile 0 / 1 (thread = row = TMEM lane); all 8
//                    convert each V tile bf16 -> fp16 in place, 16 rows each
//   warps 8-11       epilogue
//   warp 12          K/V TMA producer      warp 13  MMA issuer
//   warp 14          Q TMA producer        warp 15  idle
//
// Barrier phases (each waiter tracks parity; no barrier can run two phases
// ahead of a waiter, which would alias the parity):
//   s_full / p_full (per tile): S_{j+1} is issued only after p_full of step j,
//     and step j+1's softmax waits s_full before arriving p_full again.
//   q_full / q_empty (per tile): the Q warp loads item r + 1 only after the
//     tile's last S of item r completed; the MMA waits q_full of item r + 1
//     before its first S.
//   o_done / l_ready / o_free (per tile, once per item): o_done(r + 1) needs the
//     tile's first PV of item r + 1, which waits o_free(r), which the epilogue
//     arrives only after it waited o_done(r) and l_ready(r) and read O and l(r).
//     l_ready is NOT gated by the MMA chain (a one-step item's softmax needs no
//     PV of its own), so the softmax waits o_free(r) before it writes l(r + 1)
//     and arrives l_ready(r + 1): at most one phase ahead, and the two l
//     buffers (item parity) never collide.  o_free has two waiters (MMA and
//     softmax), each waiting every phase in order.
//   K / V rings (2 stages) and v_conv: a stage is refilled only after the
//     previous occupant's consumers committed its `empty` barrier, and v_conv of
//     a tile needs all 8 converting warps, so no warp runs two tiles ahead.
// ============================================================================
namespace s2 {
constexpr int kThreads = 512;
constexpr int kEpiWarp0 = 8, kProdWarp = 12, kMmaWarp = 13, kQWarp = 14;
constexpr int kBarQFull = 0, kBarQEmpty = 2, kBarKFull = 4, kBarVFull = 6, kBarKEmpty = 8, kBarVEmpty = 10,
              kBarVConv = 12, kBarSFull = 14, kBarPFull = 16, kBarODone = 18, kBarOFree = 20, kBarLReady = 22,
              kNumBars = 24;
constexpr int kMaxCtaItems = 512;   // items decoded in the prologue (later ones decode on the fly)
}  // namespace s2


// V tile vi (ring stage vi % kStages): rows [row0, row0 + NR) bf16 -> fp16 in
// place once the tile has landed; rows past the context are zeroed (P = 0
// there, but 0 * NaN = NaN); then one arrival on the conversion barrier.
template <int NR>
__device__ __forceinline__ void convert_v_rows(uint32_t sb, uint32_t vfull_bar, uint32_t vconv_bar, uint32_t vi,
                                               int left, int row0, int lane) {
  const int st = static_cast<int>(vi % kStages);
  const int nvalid = min(kBN, left);
  const int rows = max(0, min(16 * ((nvalid + 15) / 16) - row0, NR));
  const uint32_t vb = sb + kOffK + st * kStageBytes + 2 * kKVHalf;
  mbar_wait(vfull_bar + 8u * st, (vi / kStages) & 1);
  if (NEO_PF_EXP == 1 || NEO_PF_EXP == 2) {
  } else if (nvalid == kBN) {
    // full tile: NR rows x 256 B, unconditional 16-byte chunks (a quarter-warp
    // reads one 128-byte row half: conflict-free)
#pragma unroll
    for (int i0 = 0; i0 < NR / 2; i0 += 8) {
      uint32_t w[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = 32 * (i0 + i) + lane;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3])
                     : "r"(vb + ((e >> 3) & 1) * kKVHalf + (row0 + (e >> 4)) * 128 + (e & 7) * 16));
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = 32 * (i0 + i) + lane;
        sts128(vb + ((e >> 3) & 1) * kKVHalf + (row0 + (e >> 4)) * 128 + (e & 7) * 16, bf16x2_to_f16x2(w[i][0]),
               bf16x2_to_f16x2(w[i][1]), bf16x2_to_f16x2(w[i][2]), bf16x2_to_f16x2(w[i][3]));
      }
    }
  } else {
    for (int e0 = 0; e0 < rows * 16; e0 += 128) {
      uint32_t w[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = e0 + 32 * i + lane;
        const int row = row0 + (e >> 4);
        w[i][0] = w[i][1] = w[i][2] = w[i][3] = 0;
        if (e < rows * 16 && row < nvalid)
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3])
                       : "r"(vb + ((e >> 3) & 1) * kKVHalf + row * 128 + (e & 7) * 16));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e = e0 + 32 * i + lane;
        const int row = row0 + (e >> 4);
        if (e < rows * 16)
          sts128(vb + ((e >> 3) & 1) * kKVHalf + row * 128 + (e & 7) * 16, bf16x2_to_f16x2(w[i][0]),
                 bf16x2_to_f16x2(w[i][1]), bf16x2_to_f16x2(w[i][2]), bf16x2_to_f16x2(w[i][3]));
      }
    }
  }
  umma::fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) mbar_arrive(vconv_bar + 8u * st);
}

// packed (b, g, ct) of one item: b < 1024, g < 64, ct < 1024
__device__ __forceinline__ uint32_t pack_item(const Item& it, int ct) {
  return static_cast<uint32_t>(it.b) | (static_cast<uint32_t>(it.g) << 10) | (static_cast<uint32_t>(ct) << 16);
}
__device__ __forceinline__ void unpack_item(const PArgs& a, const Sched& sc, uint32_t w, int rows_tok, Item& it) {
  it.b = static_cast<int>(w & 1023u);
  it.g = static_cast<int>((w >> 10) & 63u);
  const int ct = static_cast<int>(w >> 16);
  it.q0 = sc.q_off[it.b];
  it.q_len = sc.q_off[it.b + 1] - it.q0;
  it.ctx = sc.ctx[it.b];
  it.i0 = ct * kTiles * rows_tok;
  const int f0 = it.i0, f1 = it.i0 + rows_tok;
  it.nt0 = (it.ctx - it.q_len + min(f0 + rows_tok, it.q_len) - 1) / kBN + 1;
  it.nt1 = f1 < it.q_len ? (it.ctx - it.q_len + min(f1 + rows_tok, it.q_len) - 1) / kBN + 1 : 0;
}

__global__ void __launch_bounds__(s2::kThreads, 1)
    prefill_attn_stream_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                               const __grid_constant__ CUtensorMap tmv, const PArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[s2::kNumBars];
  __shared__ uint32_t tmem_sh;
  __shared__ Sched sched;
  __shared__ int nct_tmp[kMaxSchedBatch];
  __shared__ uint32_t citems[s2::kMaxCtaItems];
  __shared__ float lbuf[kTiles][2][kBM];          // row sums handed to the epilogue (double-buffered by item)
  constexpr float kPBias = 7.f;                    // log2 scale of P (fp16 path, DESIGN "prefill P.V")
  constexpr uint32_t kIdescO = umma::idesc_f16_f32(kBM, 128, false, true);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G, rows_tok = kBM / G;
  const int cta = static_cast<int>(blockIdx.x), grid = static_cast<int>(gridDim.x);
  auto first_item = [&](int round) { return round * grid + ((round & 1) ? grid - 1 - cta : cta); };

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto bar = [bar0](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };

  if (threadIdx.x == 0) {
    for (int t = 0; t < kTiles; ++t) {
      mbar_init(bar(s2::kBarQFull + t), 1);
      mbar_init(bar(s2::kBarQEmpty + t), 1);
      mbar_init(bar(s2::kBarSFull + t), 1);
      mbar_init(bar(s2::kBarPFull + t), 4);
      mbar_init(bar(s2::kBarODone + t), 1);
      mbar_init(bar(s2::kBarOFree + t), 4);
      mbar_init(bar(s2::kBarLReady + t), 4);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(s2::kBarKFull + s), 1);
      mbar_init(bar(s2::kBarVFull + s), 1);
      mbar_init(bar(s2::kBarKEmpty + s), 1);
      mbar_init(bar(s2::kBarVEmpty + s), 1);
      mbar_init(bar(s2::kBarVConv + s), 8);   // the 8 softmax warps convert V
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == s2::kMmaWarp) {
    umma::tmem_alloc(smem_u32(&tmem_sh), kTmemCols);
    umma::tmem_relinquish();
  }
  if (threadIdx.x == 0) TRACE(0, 63, 13);                    // kernel entry (trace builds)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");   // metadata and q may come from the previous kernel
  if (threadIdx.x == 0) TRACE(0, 63, 14);
  build_sched(a, rows_tok, sched, nct_tmp);
  const int n_items = sched.pref[a.n_ct_max];
  // items of this CTA: every full round, plus the last partial one if it reaches this CTA
  const int n_rounds = n_items / grid + (first_item(n_items / grid) < n_items ? 1 : 0);
  for (int r = threadIdx.x; r < min(n_rounds, s2::kMaxCtaItems); r += blockDim.x) {
    Item it;
    const int k = first_item(r);
    make_item(a, sched, k, rows_tok, it);
    int lo = 0, hi = a.n_ct_max - 1;                  // the item's level -> ct
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sched.pref[mid] <= k) lo = mid;
      else hi = mid - 1;
    }
    citems[r] = pack_item(it, a.n_ct_max - 1 - lo);
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = tmem_sh;
  if (threadIdx.x == 0) TRACE(0, 63, 15);                    // prologue done
  auto get_item = [&](int r, Item& it) {
    if (r < s2::kMaxCtaItems) unpack_item(a, sched, citems[r], rows_tok, it);
    else make_item(a, sched, first_item(r), rows_tok, it);
  };
  // both tiles of an item run nt key tiles (tile 0's extra ones fully masked)
  auto steps_of = [](const Item& it) { return it.nt0 > it.nt1 ? it.nt0 : it.nt1; };

  if (warp >= s2::kEpiWarp0 + 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;" ::: "memory");
    if (warp == s2::kProdWarp) {
      // ---------------------------------------------------------- K/V producer
      if (lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv)) : "memory");
      }
      uint32_t kc = 0;
      for (int r = 0; r < n_rounds; ++r) {
        Item it;
        get_item(r, it);
        const int nt = steps_of(it);
        const int32_t* bt = a.block_table + static_cast<int64_t>(it.b) * a.max_blocks;
        for (int j = 0; j < nt; ++j, ++kc) {
          const int st = kc % kStages;
          const int kv0 = j * kBN;
          const int groups = min(kBN / 16, (it.ctx - kv0 + 15) / 16);
          int page = 0, slot = 0;
          if (lane < groups) {
            const int t = kv0 + 16 * lane;
            page = bt[t / a.page_size];
            slot = t % a.page_size;
          }
          const uint32_t dk = sb + kOffK + st * kStageBytes, dv = dk + 2 * kKVHalf;
          const uint32_t bytes = static_cast<uint32_t>(groups) * 2 * 2048;
          if (kc >= kStages) mbar_wait(bar(s2::kBarKEmpty + st), ((kc / kStages) - 1) & 1);
          if (lane == 0) mbar_expect_tx(bar(s2::kBarKFull + st), bytes);
          __syncwarp();
          if (lane < groups)
            for (int h = 0; h < 2; ++h)
              tma_load_5d(dk + h * kKVHalf + lane * 2048, &tmk, 0, slot, h, it.g, page, bar(s2::kBarKFull + st));
          if (kc >= kStages) mbar_wait(bar(s2::kBarVEmpty + st), ((kc / kStages) - 1) & 1);
          if (lane == 0) mbar_expect_tx(bar(s2::kBarVFull + st), bytes);
          __syncwarp();
          if (lane < groups)
            for (int h = 0; h < 2; ++h)
              tma_load_5d(dv + h * kKVHalf + lane * 2048, &tmv, 0, slot, h, it.g, page, bar(s2::kBarVFull + st));
        }
      }
    } else if (warp == s2::kQWarp) {
      // ---------------------------------------------------------- Q producer
      if (lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmq)) : "memory");
        for (int r = 0; r < n_rounds; ++r) {
          Item it;
          get_item(r, it);
          for (int t = 0; t < kTiles; ++t) {
            if (r > 0) mbar_wait(bar(s2::kBarQEmpty + t), (r - 1) & 1);
            mbar_expect_tx(bar(s2::kBarQFull + t), 2 * kQHalf);
            for (int h = 0; h < 2; ++h)   // rows past the tensor's tokens are zero-filled by TMA
              tma_load_4d(sb + (t * 2 + h) * kQHalf, &tmq, 0, it.g * G, it.q0 + it.i0 + t * rows_tok, h,
                          bar(s2::kBarQFull + t));
          }
        }
      }
    } else if (warp == s2::kMmaWarp) {
      // ---------------------------------------------------------- MMA issuer
      const uint64_t dq0 = umma::desc_sw128(sb, 16, 1024), dq1 = umma::desc_sw128(sb + 2 * kQHalf, 16, 1024);
      const uint64_t dk0 = umma::desc_sw128(sb + kOffK, 16, 1024);
      const uint64_t dv0 = umma::desc_sw128(sb + kOffK + 2 * kKVHalf, kKVHalf, 1024);
      constexpr uint64_t kStageDesc = kStageBytes / 16;
      auto issue_s = [&](int t, int st) {
        if (NEO_PF_EXP == 4) return;   // timing experiment: no tensor-core work at all
        umma::mma_block_k128<kQHalf, kKVHalf>(tmem + t * kTileCols, t ? dq1 : dq0,
                                              dk0 + static_cast<uint64_t>(st) * kStageDesc, kIdescS);
      };
      auto issue_pv = [&](int t, int st, int ksteps, bool acc0) {
        const uint32_t tp = tmem + t * kTileCols;
        const uint64_t bv = dv0 + static_cast<uint64_t>(st) * kStageDesc;
        if (NEO_PF_EXP == 4) {
        } else if (ksteps == 8) {
          umma::mma_block_pv128_single(tp + kColO, tp, bv, kIdescO, acc0);
        } else if (lane == 0) {
          for (int kq = 0; kq < ksteps; ++kq)
            umma::mma_bf16_ts(tp + kColO, tp + kq * 8, bv + (kq * 2048) / 16, kIdescO, kq > 0 || acc0);
        }
        __syncwarp();
      };
      if (n_rounds > 0) {
        uint32_t kc = 0, vc = 0, pc0 = 0, pc1 = 0;
        Item cur;
        get_item(0, cur);
        int nt = steps_of(cur);
        // the first item's first S on both tiles
        mbar_wait(bar(s2::kBarKFull), 0);
        for (int t = 0; t < kTiles; ++t) {
          mbar_wait(bar(s2::kBarQFull + t), 0);
          umma::fence_after_sync();
          issue_s(t, 0);
          umma::commit_elect(bar(s2::kBarSFull + t));
          if (nt == 1) umma::commit_elect(bar(s2::kBarQEmpty + t));
        }
        umma::commit_elect(bar(s2::kBarKEmpty));
        __syncwarp();
        kc = 1;
        for (int r = 0; r < n_rounds; ++r) {
          Item nxt;
          const bool has_next = r + 1 < n_rounds;
          int nt_next = 0;
          if (has_next) {
            get_item(r + 1, nxt);
            nt_next = steps_of(nxt);
          }
          for (int j = 0; j < nt; ++j, ++vc) {
            const int st = vc % kStages;
            const int nvalid = min(kBN, cur.ctx - j * kBN);
            const int ksteps = (nvalid + 15) / 16;
            const bool next_s = j + 1 < nt || has_next;   // an S follows this step's PVs
            const bool next_first = j + 1 == nt;          // ... and it is the next item's first
            // the S that follows is the last S of its item on the tile
            const bool next_last = next_first ? nt_next == 1 : j + 2 == nt;
            mbar_wait(bar(s2::kBarVConv + st), (vc / kStages) & 1);
            if (next_s) mbar_wait(bar(s2::kBarKFull + kc % kStages), (kc / kStages) & 1);
#pragma unroll
            for (int t = 0; t < kTiles; ++t) {
              if (lane == 0) TRACE(t, t ? pc1 : pc0, 4);
              mbar_wait(bar(s2::kBarPFull + t), (t ? pc1 : pc0) & 1);
              if (lane == 0) TRACE(t, t ? pc1 : pc0, 5);
              if (t) ++pc1;
              else ++pc0;
              if (j == 0 && r > 0) mbar_wait(bar(s2::kBarOFree + t), (r - 1) & 1);   // epilogue read O
              umma::fence_after_sync();
              issue_pv(t, st, ksteps, j > 0);
              if (t == kTiles - 1) umma::commit_elect(bar(s2::kBarVEmpty + st));
              if (j == nt - 1) umma::commit_elect(bar(s2::kBarODone + t));
              if (next_s) {
                if (next_first) {
                  mbar_wait(bar(s2::kBarQFull + t), (r + 1) & 1);
                  umma::fence_after_sync();
                }
                issue_s(t, kc % kStages);
                umma::commit_elect(bar(s2::kBarSFull + t));
                if (next_last) umma::commit_elect(bar(s2::kBarQEmpty + t));
                if (t == kTiles - 1) umma::commit_elect(bar(s2::kBarKEmpty + kc % kStages));
              }
              if (lane == 0) TRACE(t, (t ? pc1 : pc0) - 1, 6);
              __syncwarp();
            }
            if (next_s) ++kc;
          }
          if (has_next) {
            cur = nxt;
            nt = nt_next;
          }
        }
      }
    }
  } else if (warp >= s2::kEpiWarp0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;" ::: "memory");
    // ------------------------------------------------------------ epilogue
    // One warp per TMEM lane quarter drains each item's O / l of both tiles.
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int row0 = quarter * 32;
    // O / l of item rd, tile t -> bf16 rows of `out`; o_free once O is read
    auto epilogue = [&](int rd, const Item& it, int t, int trace_row) {
      const uint32_t tO = tmem + t * kTileCols + kColO + (static_cast<uint32_t>(quarter * 32) << 16);
      if (quarter == 0 && lane == 0) TRACE(t, trace_row, 8);
      mbar_wait(bar(s2::kBarODone + t), rd & 1);
      mbar_wait(bar(s2::kBarLReady + t), rd & 1);
      umma::fence_after_sync();
      if (quarter == 0 && lane == 0) TRACE(t, trace_row, 9);
      const float inv_l = 1.f / lbuf[t][rd & 1][r];
      const int tok = it.i0 + t * rows_tok + r / G;
      uint16_t* orow = a.out + (static_cast<int64_t>(it.q0 + min(tok, it.q_len - 1)) * a.hq + it.g * G + r % G) * 128;
#pragma unroll 1
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t o[32];
        umma::ld32(tO + c0, o);
        umma::wait_ld();
        if (c0 == 96) {                              // O read: the tile's next first PV may overwrite it
          umma::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(s2::kBarOFree + t));
        }
        if (tok < it.q_len) {
#pragma unroll
          for (int c = 0; c < 32; c += 16) {
            uint32_t w[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
              w[e] = pack_bf16(__uint_as_float(o[c + 2 * e]) * inv_l, __uint_as_float(o[c + 2 * e + 1]) * inv_l);
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(orow + c0 + c), "r"(w[0]),
                         "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                         : "memory");
          }
        }
      }
      if (quarter == 0 && lane == 0) TRACE(t, trace_row, 10);
    };
    int steps_done = 0;                              // trace row of the item's last step
    for (int rd = 0; rd < n_rounds; ++rd) {
      Item it;
      get_item(rd, it);
      steps_done += steps_of(it);
      for (int d = a.epi_delay_ns; d > 0; d -= 500000) __nanosleep(min(d, 500000));   // test knob
      for (int t = 0; t < kTiles; ++t) epilogue(rd, it, t, steps_done - 1);
    }
    if (quarter == 0 && lane == 0) TRACE(1, 63, 13);             // last store issued
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 168;" ::: "memory");
    // ------------------------------------------------------------ softmax warps
    const int t = warp >> 2, quarter = warp & 3;
    const int r = quarter * 32 + lane;               // row == TMEM lane
    const uint32_t tS = tmem + t * kTileCols + (static_cast<uint32_t>(quarter * 32) << 16);
    const uint32_t tO = tS + kColO;
    const float sl = a.scale_log2;
    uint32_t sc = 0, vidx = 0;
    for (int rd = 0; rd < n_rounds; ++rd) {
      Item it;
      get_item(rd, it);
      const int nt = steps_of(it);
      const int i_row = it.i0 + t * rows_tok + r / G;
      const int pos = it.ctx - it.q_len + min(i_row, it.q_len - 1);
      float m = -INFINITY;
      uint64_t l2 = f2(0.f, 0.f);
      for (int j = 0; j < nt; ++j, ++sc) {
        if (quarter == 0 && lane == 0) TRACE(t, sc, 0);
        if (quarter == 0 && lane == 0 && j == 0) TRACE(t, sc, 7);
        convert_v_rows<16>(sb, bar(s2::kBarVFull), bar(s2::kBarVConv), vidx++, it.ctx - j * kBN, (t * 4 + quarter) * 16,
                             lane);
        mbar_wait(bar(s2::kBarSFull + t), sc & 1);
        umma::fence_after_sync();
        if (quarter == 0 && lane == 0) TRACE(t, sc, 1);
        float s[kBN];
        {
          uint32_t u[4][32];
#pragma unroll
          for (int c0 = 0; c0 < kBN; c0 += 32) umma::ld32(tS + c0, u[c0 / 32]);
          umma::wait_ld();
#pragma unroll
          for (int c = 0; c < kBN; ++c) s[c] = __uint_as_float(u[c / 32][c % 32]);
        }
        if (NEO_PF_EXP == 2 || NEO_PF_EXP == 3) {
          uint32_t hw[16];
#pragma unroll
          for (int w = 0; w < 16; ++w) hw[w] = __float_as_uint(s[w] * 0.f);
#pragma unroll
          for (int c0 = 0; c0 < kBN; c0 += 32) umma::st16(tS + c0 / 2, hw);
          l2 = f2(1.f, 1.f);
          umma::wait_st();
          umma::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(s2::kBarPFull + t));
          continue;
        }
        // causal mask on diagonal tiles, by 32-column chunk with warp-uniform
        // classification: chunks visible to every row of the warp are untouched,
        // chunks past every row's limit skip the max and the exponentials (P = 0)
        const int lim = pos - j * kBN;               // last visible column of this row in the tile
        const bool any_mask = __any_sync(0xffffffffu, lim < kBN - 1);
        const int lo_lim = any_mask ? __reduce_min_sync(0xffffffffu, lim) : kBN;
        const int hi_lim = any_mask ? __reduce_max_sync(0xffffffffu, lim) : kBN;
#pragma unroll
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          if (c0 + 31 <= lo_lim || c0 > hi_lim) continue;
#pragma unroll
          for (int c = 0; c < 32; ++c) s[c0 + c] = c0 + c > lim ? -INFINITY : s[c0 + c];
        }
        if (quarter == 0 && lane == 0) TRACE(t, sc, 2);
        // row max: four independent chains per chunk
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          if (c0 > hi_lim) continue;
#pragma unroll
          for (int c = 0; c < 32; c += 8)
#pragma unroll
            for (int q = 0; q < 4; ++q) mq[q] = fmaxf(mq[q], fmaxf(s[c0 + c + 2 * q], s[c0 + c + 2 * q + 1]));
        }
        const float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        const float m_new = fmaxf(m, mx);            // j > 0 on tile 0's masked extra steps: m_new = m
        bool resc = false;
        float alpha = 1.f;
        if (j == 0) {
          m = m_new;
        } else if ((m_new - m) * sl > 8.f) {
          resc = true;
          alpha = ex2((m - m_new) * sl);
          l2 = fmul2(l2, f2(alpha, alpha));
          m = m_new;
        }
        const uint64_t sl2 = f2(sl, sl), nm2 = f2(kPBias - m * sl, kPBias - m * sl);
        uint64_t la = f2(0.f, 0.f), lb = f2(0.f, 0.f);   // two row-sum chains
        // all 128 exponentials first, the four TMEM stores after: no
        // memory-clobbering asm inside the loop, so the scheduler can overlap
        // one chunk's MUFU latency with the next chunk's work
        uint32_t hw[64];
#pragma unroll
        for (int c0 = 0; c0 < kBN; c0 += 32) {
          if (c0 > hi_lim) {
#pragma unroll
            for (int w = 0; w < 16; ++w) hw[c0 / 2 + w] = 0u;
          } else {
#pragma unroll
            for (int w = 0; w < 16; ++w) {
              const uint64_t xx = ffma2(f2(s[c0 + 2 * w], s[c0 + 2 * w + 1]), sl2, nm2);
              float p0, p1;
              if ((w & 3) < kPolyPairsStream) {
                const float2 pp = unf2(exp2_poly2(xx));
                p0 = pp.x;
                p1 = pp.y;
              } else {
                const float2 x = unf2(xx);
                p0 = ex2(x.x);
                p1 = ex2(x.y);
              }
              if (w & 1) lb = fadd2(lb, f2(p0, p1));
              else la = fadd2(la, f2(p0, p1));
              hw[c0 / 2 + w] = pack_f16(p0, p1);
            }
          }
        }
#pragma unroll
        for (int c0 = 0; c0 < kBN; c0 += 32) umma::st16(tS + c0 / 2, *reinterpret_cast<const uint32_t(*)[16]>(&hw[c0 / 2]));
        l2 = fadd2(l2, fadd2(la, lb));
        if (__any_sync(0xffffffffu, resc)) {
          // PV_{j-1} is complete (the S_j commit covers it): scale O in place
#pragma unroll 1
          for (int c0 = 0; c0 < 128; c0 += 32) {
            uint32_t o[32];
            umma::ld32(tO + c0, o);
            umma::wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            umma::st32(tO + c0, o);
          }
        }
        umma::wait_st();
        umma::fence_before_sync();
        __syncwarp();
        if (quarter == 0 && lane == 0) TRACE(t, sc, 3);
        if (lane == 0) mbar_arrive(bar(s2::kBarPFull + t));
      }
      // row sum to the epilogue (its O wait is on o_done, committed after the
      // last PV, which follows this item's last p_full)
      const float2 lp = unf2(l2);
      // l_ready may run only one item ahead of the epilogue's wait on it (a
      // second completion would alias the parity it waits on): wait until the
      // epilogue released the previous item's O (o_free, arrived after it
      // waited l_ready of that item).  Without this, a one-step item right
      // after a slow epilogue lets the softmax complete l_ready twice.
      if (rd > 0) mbar_wait(bar(s2::kBarOFree + t), (rd - 1) & 1);
      lbuf[t][rd & 1][r] = lp.x + lp.y;
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(s2::kBarLReady + t));
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == s2::kMmaWarp) umma::tmem_dealloc(tmem, kTmemCols);
}


}  // namespace

neo_status launch_prefill_attn(const PrefillLaunch& L, const CUtensorMap& tmq, const CUtensorMap& tmk,
                               const CUtensorMap& tmv, const CUtensorMap& tmo) {
  static std::atomic<uint64_t> configured{0};
  static std::atomic<int> sms_of[64];
  neo_status st = once_per_device(configured, [](int dev) {
    cudaError_t e =
        cudaFuncSetAttribute(prefill_attn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(prefill_attn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(prefill_attn_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return cuda_fail(e, "prefill smem attribute");
    int n = 0;
    e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "SM count");
    sms_of[dev & 63].store(n, std::memory_order_relaxed);
    return NEO_OK;
  });
  if (st != NEO_OK) return st;
  int cur_dev = 0;
  cudaGetDevice(&cur_dev);
  const int num_sms = sms_of[cur_dev & 63].load(std::memory_order_relaxed);
  const int G = L.hq / L.hkv;
  const int n_ct_max = (L.max_q_len * G + kTiles * kBM - 1) / (kTiles * kBM);
  const int64_t n_items = static_cast<int64_t>(n_ct_max) * L.batch * L.hkv;   // upper bound
  if (L.batch > kMaxSchedBatch || n_ct_max > kMaxSchedLevels)
    return fail(NEO_ERR_UNSUPPORTED, "prefill: batch <= 512 and max_q_len * G <= 262144 per call");
  const char* dly = std::getenv("NEO_PREFILL_EPI_DELAY_NS");   // test knob: a slow epilogue (barrier-phase test)
  PArgs a{static_cast<uint16_t*>(L.out), L.block_table, L.seq_lens, L.q_offsets, L.batch, L.hq, L.hkv, G,
          L.page_size, L.max_blocks, n_ct_max, L.scale * 1.4426950408889634f, dly ? std::atoi(dly) : 0};
#ifdef NEO_PREFILL_TRACE
  static long long* trace = nullptr;
  if (!trace) cudaMalloc(&trace, 2 * 64 * 16 * sizeof(long long));
  cudaMemsetAsync(trace, 0, 2 * 64 * 16 * sizeof(long long), L.stream);
  a.trace = trace;
  g_prefill_trace = trace;
#endif
  cudaLaunchConfig_t cfg{};
  int ctas = num_sms;
  if (L.max_ctas > 0) ctas = std::min(ctas, L.max_ctas);   // SM budget when sharing the GPU with decode
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(n_items, ctas)));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemAlloc;
  cfg.stream = L.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // P.V in fp16 for prompt chunks of >= kFp16MinQLen tokens, hi + lo below
  // (tools/prefill_time.py A/B: 1 x 16384 +18 %, 8 x ~1000 +3-5 %, 64 x 128 -12 %)
  const char* pv = std::getenv("NEO_PREFILL_PV");   // test / experiment knob: "hilo" | "fp16"
  const int force = pv ? (pv[0] == 'h' ? 1 : 2) : 0;
  const bool hilo = force ? force == 1 : L.max_q_len < kFp16MinQLen;
  // fp16 path: the stream kernel for prompts up to kStreamMaxQLen tokens (hkv <= 64
  // for its packed item list), the item-major kernel above; NEO_PREFILL_KERNEL=
  // item|stream forces one (tests run both)
  const char* kn = std::getenv("NEO_PREFILL_KERNEL");
  // (same-box A/B, tools/prefill_time.py: the stream kernel wins up to 2048-token
  // prompts -- 8 x 1024 -6 %, 16 x 512 -11 %, ragged 8 x ~1000 -6..9 % -- and
  // loses 2-5 % from 4096 on, where item boundaries are rare)
  const bool stream = !hilo && L.hkv <= 64 && (kn ? kn[0] == 's' : L.max_q_len <= kStreamMaxQLen);
  if (stream) {
    cfg.blockDim = dim3(s2::kThreads);
    cudaLaunchKernelEx(&cfg, prefill_attn_stream_kernel, tmq, tmk, tmv, a);
  } else if (hilo) {
    cudaLaunchKernelEx(&cfg, prefill_attn_kernel<true>, tmq, tmk, tmv, tmo, a);
  } else {
    cudaLaunchKernelEx(&cfg, prefill_attn_kernel<false>, tmq, tmk, tmv, tmo, a);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NEO_OK : cuda_fail(e, "prefill attention kernel launch");
}

}  // namespace neo

#ifdef NEO_PREFILL_TRACE
extern "C" __attribute__((visibility("default"))) long long* neo_prefill_trace_ptr() { return neo::g_prefill_trace; }
#endif
