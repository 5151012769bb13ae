// Split-K paged GQA decode attention for sm_100a (NEO's GPU attention, P:246,
// P:303; flash-decoding partition + aggregate).
//
// Work unit = (request b, kv-head g, chunk c of C tokens), one WARP per unit,
// kWarps independent warps per CTA.  Each warp runs its own kStages-deep ring
// of TMA tensor loads (cp.async.bulk.tensor, 128B swizzle, L2 evict_first)
// completing on per-stage mbarriers; one 16-token tile = the K block and V block
// of one (page, kv-head), 4 KiB each.
//
// Math per tile (fp32 accumulate of exact bf16 products):
//   S^T[16 tok x 8 heads] = K_tile[16 x 128] . Q^T[128 x 8]        8x mma.m16n8k16
//   online softmax in the exp2 domain (scale*log2e folded into the scores)
//   O^T[128 x 8] += V^T[128 x 16] . P^T[16 x 8]                    8x2 mma.m16n8k16
// P is split into bf16 hi + lo parts (two MMAs) so the P.V product keeps ~16
// mantissa bits (a bf16-only P fails the tolerance).
// Fragments are read straight from the swizzled tiles with LDS.128; the token
// permutation PI and the dim assignment below make every read conflict-free
// (checked by tools/check_banks.py).  P goes from the S^T accumulator layout to
// the B-operand layout with movmatrix.trans (no shared-memory round trip).
//
// Single-chunk units write the bf16 output directly; multi-chunk units write an
// fp32 partial (acc, m, l) to the workspace, and the LAST warp to finish a
// (b, g) -- detected with a per-(b, g) counter -- merges the partials in chunk
// order (deterministic, no float atomics) and resets the counter.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "neo_internal.cuh"

namespace neo {
namespace {

constexpr int kStageBytes = 2 * kTileBytes;
constexpr unsigned kFull = 0xffffffffu;

struct KArgs {
  const uint16_t* q;
  uint16_t* out;
  const int32_t* block_table;
  const int32_t* seq_lens;
  float* ws_acc;
  float2* ws_ml;
  int32_t* ws_cnt;
  int32_t batch, hq, hkv, G, page_size, max_blocks, chunk_tiles, max_chunks;
  float scale_log2;
  // fused append (+ RoPE) variant only (neo_decode_attn_append)
  const float* inv_freq;      // NULL: no rotation
  const uint16_t* k_new;      // [batch][Hkv][D]
  const uint16_t* v_new;
  uint16_t* k_pages;
  uint16_t* v_pages;
  int64_t page_stride;
  int32_t probe;              // experiment knob (NEO_ATTN_PROBE bits): 1 no epilogue, 2 no tile math,
                              // 4 no combine, 8 partial stores only (no counter); 0 in production
  int32_t early;              // NEO_ATTN_KV_STABLE (see kernel prologues)
  int32_t l2pf;               // L2 prefetch distance in tiles beyond the smem ring (0 = off)
  int32_t l2pro;              // tiles prefetched into L2 in the prologue only (before the PDL wait)
  int32_t first_wave;         // CTAs of the first resident wave (the ones that start during the
                              // previous grid's tail under PDL)
  int32_t req_major;          // grouped kernel: CTA order (q, b, g) -> (b, q, g)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
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

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tma_load_tile(uint32_t dst, const CUtensorMap* tm, int tok, int g, int page,
                                              uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(0), "r"(0), "r"(tok), "r"(g), "r"(page), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ uint32_t word(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Byte offset of 16-byte chunk `c` (0..15) of token `t` inside a tile that TMA
// wrote with box {64, 2, 16} and CU_TENSOR_MAP_SWIZZLE_128B: 128-byte row
// R = 2t + c/8, chunk slot (c % 8) XOR (R % 8).
__device__ __forceinline__ uint32_t swz(int t, int c) {
  const int R = 2 * t + (c >> 3);
  return static_cast<uint32_t>(R * 128 + (((c & 7) ^ (R & 7)) << 4));
}

// Token held by MMA row rho (0..7); rows 8..15 hold 8 + PI(rho - 8).
__device__ __forceinline__ int tok_pi(int rho) { return (rho & 1) ? 4 + ((rho >> 1) ^ 2) : (rho >> 1); }

__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ uint32_t movtrans(uint32_t x) {
  uint32_t r;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

__device__ __forceinline__ void store_row8(uint16_t* dst, const float (&v)[8], float inv) {
  uint4 w;
  w.x = pack_bf16(v[0] * inv, v[1] * inv);
  w.y = pack_bf16(v[2] * inv, v[3] * inv);
  w.z = pack_bf16(v[4] * inv, v[5] * inv);
  w.w = pack_bf16(v[6] * inv, v[7] * inv);
  *reinterpret_cast<uint4*>(dst) = w;
}

// ------------------------------------------------------------------ tile math

struct Acc {
  float o[8][4];  // O^T fragments: o[i][0|2] head 2qd, o[i][1|3] head 2qd+1; dims 8r+i | 64+8r+i
  float m0, m1, l0, l1;
};

__device__ __forceinline__ void acc_reset(Acc& s) {
#pragma unroll
  for (int i = 0; i < 8; ++i) s.o[i][0] = s.o[i][1] = s.o[i][2] = s.o[i][3] = 0.f;
  s.m0 = s.m1 = -INFINITY;
  s.l0 = s.l1 = 0.f;
}

// Q fragment (B operand of S^T = K Q^T): head r of the group, dims of chunks
// qd + 4i in the same order as the K registers.  Heads r >= G are zero.
__device__ __forceinline__ void load_q(const KArgs& a, int b, int g, int r, int qd, uint4 (&qf)[4]) {
  if (r < a.G) {
    const uint16_t* qp = a.q + (static_cast<int64_t>(b) * a.hq + g * a.G + r) * kHeadDim;
#pragma unroll
    for (int i = 0; i < 4; ++i) qf[i] = __ldg(reinterpret_cast<const uint4*>(qp + 8 * (qd + 4 * i)));
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) qf[i] = make_uint4(0, 0, 0, 0);
  }
}

// RoPE angle theta = t * inv_freq (fp64, reduced to [-pi, pi] in fp64), then
// sin / cos in fp32 (same convention as neo_rope_append).
__device__ __forceinline__ void rope_sincos(int t, float f, float& sn, float& cs) {
  const double th = static_cast<double>(t) * static_cast<double>(f);
  const double k = rint(th * 0.15915494309189533577);
  const float red = static_cast<float>(fma(-k, 6.283185307179586232, th));
  __sincosf(red, &sn, &cs);
}

// Rotate this lane's q fragment in registers: qf[i] holds dims 8(qd + 4i) .. +7,
// so the rotate-half partners (d, d + 64) are qf[0] / qf[2] and qf[1] / qf[3].
__device__ __forceinline__ void rope_q(uint4 (&qf)[4], int qd, int t, const float* inv_freq) {
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uint32_t lo[4] = {qf[i].x, qf[i].y, qf[i].z, qf[i].w};
    uint32_t hi[4] = {qf[i + 2].x, qf[i + 2].y, qf[i + 2].z, qf[i + 2].w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int d = 8 * (qd + 4 * i) + 2 * w;
      float s0, c0, s1, c1;
      rope_sincos(t, __ldg(inv_freq + d), s0, c0);
      rope_sincos(t, __ldg(inv_freq + d + 1), s1, c1);
      const float a0 = __uint_as_float(lo[w] << 16), a1 = __uint_as_float(lo[w] & 0xffff0000u);
      const float b0 = __uint_as_float(hi[w] << 16), b1 = __uint_as_float(hi[w] & 0xffff0000u);
      lo[w] = pack_bf16(a0 * c0 - b0 * s0, a1 * c1 - b1 * s1);
      hi[w] = pack_bf16(b0 * c0 + a0 * s0, b1 * c1 + a1 * s1);
    }
    qf[i] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    qf[i + 2] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  }
}

// Fragments of one 16-token tile, read from the 128B-swizzled stage: K rows
// tokA/tokB (chunks qd + 4i) and V tokens vt0, vt1, vt0+8, vt1+8 (chunks r, r+8).
struct Frags {
  uint4 ka[4], kb[4];
  uint4 v00, v01, v10, v11, v20, v21, v30, v31;
};

__device__ __forceinline__ void load_frags(uint32_t sk, int r, int qd, Frags& f) {
  const uint32_t sv = sk + kTileBytes;
  const int tokA = tok_pi(r), tokB = 8 + tokA;
  const int vt0 = tok_pi(2 * qd), vt1 = tok_pi(2 * qd + 1);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f.ka[i] = lds128(sk + swz(tokA, qd + 4 * i));
    f.kb[i] = lds128(sk + swz(tokB, qd + 4 * i));
  }
  f.v00 = lds128(sv + swz(vt0, r));
  f.v01 = lds128(sv + swz(vt0, r + 8));
  f.v10 = lds128(sv + swz(vt1, r));
  f.v11 = lds128(sv + swz(vt1, r + 8));
  f.v20 = lds128(sv + swz(vt0 + 8, r));
  f.v21 = lds128(sv + swz(vt0 + 8, r + 8));
  f.v30 = lds128(sv + swz(vt1 + 8, r));
  f.v31 = lds128(sv + swz(vt1 + 8, r + 8));
}

// Fold one tile (already in registers) into the running (O, m, l).  `valid` =
// tokens of the tile inside the context (>= 1).
__device__ __forceinline__ void compute_tile(Frags& f, const uint4 (&qf)[4], int valid, float sl2, int r, int qd,
                                             Acc& s) {
  const int tokA = tok_pi(r), tokB = 8 + tokA;              // S^T rows r, r+8
  const int vt0 = tok_pi(2 * qd), vt1 = tok_pi(2 * qd + 1);  // P.V k-slots 2qd, 2qd+1 (+8)

  // (a3) scores: S^T = K_tile . Q^T
  float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int i = jj >> 1, w = 2 * (jj & 1);
    mma_bf16(sc, word(f.ka[i], w), word(f.kb[i], w), word(f.ka[i], w + 1), word(f.kb[i], w + 1), word(qf[i], w),
             word(qf[i], w + 1));
  }
  uint4 v00 = f.v00, v01 = f.v01, v10 = f.v10, v11 = f.v11, v20 = f.v20, v21 = f.v21, v30 = f.v30, v31 = f.v31;

  float x0 = sc[0] * sl2, x1 = sc[1] * sl2, x2 = sc[2] * sl2, x3 = sc[3] * sl2;
  if (valid < kTileTokens) {  // ragged last tile: mask scores, zero V (NaN-safe)
    const uint4 z = make_uint4(0, 0, 0, 0);
    if (tokA >= valid) x0 = x1 = -INFINITY;
    if (tokB >= valid) x2 = x3 = -INFINITY;
    if (vt0 >= valid) v00 = v01 = z;
    if (vt1 >= valid) v10 = v11 = z;
    if (vt0 + 8 >= valid) v20 = v21 = z;
    if (vt1 + 8 >= valid) v30 = v31 = z;
  }

  // (a4) online softmax; token 0 of every tile is valid, so the tile max is finite
  float mx0 = fmaxf(x0, x2), mx1 = fmaxf(x1, x3);
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(kFull, mx0, off));
    mx1 = fmaxf(mx1, __shfl_xor_sync(kFull, mx1, off));
  }
  const float mn0 = fmaxf(s.m0, mx0), mn1 = fmaxf(s.m1, mx1);
  if (__any_sync(kFull, (mn0 > s.m0) || (mn1 > s.m1))) {
    const float al0 = ex2(s.m0 - mn0), al1 = ex2(s.m1 - mn1);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s.o[i][0] *= al0;
      s.o[i][2] *= al0;
      s.o[i][1] *= al1;
      s.o[i][3] *= al1;
    }
    s.l0 *= al0;
    s.l1 *= al1;
    s.m0 = mn0;
    s.m1 = mn1;
  }
  const float p0 = ex2(x0 - s.m0), p1 = ex2(x1 - s.m1), p2 = ex2(x2 - s.m0), p3 = ex2(x3 - s.m1);
  s.l0 += p0 + p2;
  s.l1 += p1 + p3;
  const uint32_t ht = pack_bf16(p0, p1), hb = pack_bf16(p2, p3);
  const uint32_t lt = pack_bf16(p0 - bf_lo(ht), p1 - bf_hi(ht));
  const uint32_t lb = pack_bf16(p2 - bf_lo(hb), p3 - bf_hi(hb));
  const uint32_t bh0 = movtrans(ht), bh1 = movtrans(hb), bl0 = movtrans(lt), bl1 = movtrans(lb);

  // (a5) O^T += V^T . P^T  (hi and lo parts of P)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t sel = (i & 1) ? 0x7632u : 0x5410u;
    const int w = i >> 1;
    const uint32_t a0 = prmt(word(v00, w), word(v10, w), sel);
    const uint32_t a1 = prmt(word(v01, w), word(v11, w), sel);
    const uint32_t a2 = prmt(word(v20, w), word(v30, w), sel);
    const uint32_t a3 = prmt(word(v21, w), word(v31, w), sel);
    mma_bf16(s.o[i], a0, a1, a2, a3, bh0, bh1);
    mma_bf16(s.o[i], a0, a1, a2, a3, bl0, bl1);
  }
}

__device__ __forceinline__ void write_zero_row(const KArgs& a, int b, int g, int lane) {
  uint16_t* o = a.out + (static_cast<int64_t>(b) * a.hq + g * a.G) * kHeadDim;
  for (int e = lane * 8; e < a.G * kHeadDim; e += 32 * 8) *reinterpret_cast<uint4*>(o + e) = make_uint4(0, 0, 0, 0);
}

// (a7) combine of the n_chunks partials of (b, g), by the last-arriving warp:
//   out_h = sum_c 2^(m_ch - M_h) acc_ch / sum_c 2^(m_ch - M_h) l_ch,  M_h = max_c m_ch.
// Latency-parallel for any G: pass 1 gives lane L chunks L, L+32, ... and merges
// their (m, l) per head, then a butterfly merges the lanes (commutative, so every
// lane ends with bitwise the same M_h, L_h); pass 2 has each lane accumulate 4 dims
// of every head over the chunks in chunk order, loading K chunks x G heads of
// partials per batch before using any of them.
template <int G>
__device__ __forceinline__ void combine(const KArgs& a, int b, int g, int bg, int n_chunks, int lane) {
  const int64_t slot0 = static_cast<int64_t>(bg) * a.max_chunks;
  const float2* ml = a.ws_ml + slot0 * G;
  float M[G], L[G];
#pragma unroll
  for (int h = 0; h < G; ++h) M[h] = -INFINITY, L[h] = 0.f;
  for (int c = lane; c < n_chunks; c += 32) {
    float2 t[G];
#pragma unroll
    for (int h = 0; h < G; ++h) t[h] = __ldcg(&ml[c * G + h]);
#pragma unroll
    for (int h = 0; h < G; ++h) {   // chunk m is finite (>= 1 token), so mn is too
      const float mn = fmaxf(M[h], t[h].x);
      L[h] = L[h] * ex2(M[h] - mn) + t[h].y * ex2(t[h].x - mn);
      M[h] = mn;
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float Mo = __shfl_xor_sync(kFull, M[h], off), Lo = __shfl_xor_sync(kFull, L[h], off);
      const float mn = fmaxf(M[h], Mo);
      L[h] = (M[h] == -INFINITY ? 0.f : L[h] * ex2(M[h] - mn)) + (Mo == -INFINITY ? 0.f : Lo * ex2(Mo - mn));
      M[h] = mn;
    }
  }
  constexpr int K = 16 / G > 1 ? 16 / G : 1;       // chunks per batch (<= 16 partial rows in flight)
  float4 s4[G];
#pragma unroll
  for (int h = 0; h < G; ++h) s4[h] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* accb = a.ws_acc + slot0 * G * kHeadDim + 4 * lane;
  for (int c0 = 0; c0 < n_chunks; c0 += K) {
    float4 v[K][G];
    float w[K][G];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int cc = c0 + k < n_chunks ? c0 + k : n_chunks - 1;
#pragma unroll
      for (int h = 0; h < G; ++h) {
        v[k][h] = __ldcg(reinterpret_cast<const float4*>(accb + (static_cast<int64_t>(cc) * G + h) * kHeadDim));
        w[k][h] = __ldcg(&ml[cc * G + h].x);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const float wk = c0 + k < n_chunks ? ex2(w[k][h] - M[h]) : 0.f;
        s4[h].x += wk * v[k][h].x;
        s4[h].y += wk * v[k][h].y;
        s4[h].z += wk * v[k][h].z;
        s4[h].w += wk * v[k][h].w;
      }
    }
  }
  {   // the partials are dead: drop their L2 lines without write-back (128-byte lines;
      // the acc region of (b, g) starts on a 512-byte boundary of a 128-byte-aligned region)
    const char* p0 = reinterpret_cast<const char*>(a.ws_acc + slot0 * G * kHeadDim);
    if ((reinterpret_cast<uintptr_t>(a.ws_acc) & 127) == 0)
      for (int e = lane; e < n_chunks * G * 4; e += 32)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(p0 + 128 * static_cast<int64_t>(e)) : "memory");
  }
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const float inv = 1.f / L[h];
    uint2 pk;
    pk.x = pack_bf16(s4[h].x * inv, s4[h].y * inv);
    pk.y = pack_bf16(s4[h].z * inv, s4[h].w * inv);
    *reinterpret_cast<uint2*>(a.out + (static_cast<int64_t>(b) * a.hq + g * G + h) * kHeadDim + 4 * lane) = pk;
  }
}

// One 32-byte partial row segment: o[0..7][k] (k selects head / dim half).  The
// partials live from this store until the combine of (b, g) reads them; an
// L2::evict_last hint keeps them resident against the evict_first KV stream, and
// the combine discards them afterwards, so they never cost DRAM write-backs
// (same-box A/B: c2 +2.5 %, c4 +3.3 %, c3 +1.5 %).
__device__ __forceinline__ void st256(float* dst, const Acc& s, int k) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(dst),
               "f"(s.o[0][k]), "f"(s.o[1][k]), "f"(s.o[2][k]), "f"(s.o[3][k]), "f"(s.o[4][k]), "f"(s.o[5][k]),
               "f"(s.o[6][k]), "f"(s.o[7][k]), "l"(pol)
               : "memory");
}

// End of a unit: single-chunk units write the output (a6 bypass); others write
// the partial and the last-arriving warp of (b, g) runs the combine (a7).
__device__ __forceinline__ void finish_unit(const KArgs& a, Acc& s, int b, int g, int c, int n_chunks, int lane,
                                            int r, int qd) {
  const int G = a.G;
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    s.l0 += __shfl_xor_sync(kFull, s.l0, off);
    s.l1 += __shfl_xor_sync(kFull, s.l1, off);
  }
  const int h0 = 2 * qd, h1 = 2 * qd + 1;
  if (n_chunks == 1) {
    uint16_t* ob = a.out + (static_cast<int64_t>(b) * a.hq + g * G) * kHeadDim;
    float t[8];
    if (h0 < G) {
      const float inv = 1.f / s.l0;
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = s.o[i][0];
      store_row8(ob + h0 * kHeadDim + 8 * r, t, inv);
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = s.o[i][2];
      store_row8(ob + h0 * kHeadDim + 64 + 8 * r, t, inv);
    }
    if (h1 < G) {
      const float inv = 1.f / s.l1;
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = s.o[i][1];
      store_row8(ob + h1 * kHeadDim + 8 * r, t, inv);
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = s.o[i][3];
      store_row8(ob + h1 * kHeadDim + 64 + 8 * r, t, inv);
    }
    return;
  }
  const int bg = b * a.hkv + g;
  const int64_t slot = static_cast<int64_t>(bg) * a.max_chunks + c;
  float* acc = a.ws_acc + slot * G * kHeadDim;
  // 256-bit stores: each lane writes whole 32-byte sectors (dims 8r..8r+7 and
  // 64+8r..64+8r+7 of its heads); the workspace acc region is 512-byte aligned
  if (h0 < G) {
    st256(acc + h0 * kHeadDim + 8 * r, s, 0);
    st256(acc + h0 * kHeadDim + 64 + 8 * r, s, 2);
    if (r == 0) a.ws_ml[slot * G + h0] = make_float2(s.m0, s.l0);
  }
  if (h1 < G) {
    st256(acc + h1 * kHeadDim + 8 * r, s, 1);
    st256(acc + h1 * kHeadDim + 64 + 8 * r, s, 3);
    if (r == 0) a.ws_ml[slot * G + h1] = make_float2(s.m1, s.l1);
  }
  // publish: the warp barrier orders every lane's partial stores before lane 0's
  // acq_rel atomic (release at GPU scope, cumulative); the last arriver's acquire
  // makes all partials of (b, g) visible to the __ldcg reads below
  __syncwarp();
  if (a.probe & 8) return;
  int prev = 0;
  if (lane == 0)
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(a.ws_cnt + bg) : "memory");
  prev = __shfl_sync(kFull, prev, 0);
  if (prev != n_chunks - 1) return;
  // shfl only moves the value; the warp barrier extends lane 0's acquire to the
  // lanes whose __ldcg reads of the other chunks' partials follow
  __syncwarp();
  if (a.probe & 4) {
    if (lane == 0) a.ws_cnt[bg] = 0;
    return;
  }
  switch (G) {
    case 1: combine<1>(a, b, g, bg, n_chunks, lane); break;
    case 2: combine<2>(a, b, g, bg, n_chunks, lane); break;
    case 3: combine<3>(a, b, g, bg, n_chunks, lane); break;
    case 4: combine<4>(a, b, g, bg, n_chunks, lane); break;
    case 5: combine<5>(a, b, g, bg, n_chunks, lane); break;
    case 6: combine<6>(a, b, g, bg, n_chunks, lane); break;
    case 7: combine<7>(a, b, g, bg, n_chunks, lane); break;
    default: combine<8>(a, b, g, bg, n_chunks, lane); break;
  }
  if (lane == 0) a.ws_cnt[bg] = 0;  // leave the workspace re-usable
}

// Fused append: the unit holding the new token t = ctx - 1 overwrites the
// token's (stale) K and V rows in the landed stage with k_new (rotated when
// inv_freq is set) and v_new, and stores the same rows into the page slot.
// Lanes 0..15: K chunk `lane` (its rotate-half partner chunk lane ^ 8 is read
// too); lanes 16..31: V chunk lane - 16.
__device__ __forceinline__ void patch_new_token(const KArgs& a, uint32_t sk, int b, int g, int ctx, int lane) {
  const int t = ctx - 1, slot = t % kTileTokens, ch = lane & 15;
  const bool is_k = lane < 16;
  const uint16_t* src = (is_k ? a.k_new : a.v_new) + (static_cast<int64_t>(b) * a.hkv + g) * kHeadDim;
  uint4 val = __ldg(reinterpret_cast<const uint4*>(src + 8 * ch));
  if (is_k && a.inv_freq) {
    const uint4 par = __ldg(reinterpret_cast<const uint4*>(src + 8 * (ch ^ 8)));
    const uint32_t x[4] = {val.x, val.y, val.z, val.w}, y[4] = {par.x, par.y, par.z, par.w};
    uint32_t o[4];
    const float sg = ch < 8 ? -1.f : 1.f;    // x'[i] = x c - x[i+64] s ; x'[i+64] = x[i+64] c + x[i] s
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int i = 8 * (ch & 7) + 2 * w;    // frequency index of the pair
      float s0, c0, s1, c1;
      rope_sincos(t, __ldg(a.inv_freq + i), s0, c0);
      rope_sincos(t, __ldg(a.inv_freq + i + 1), s1, c1);
      const float a0 = __uint_as_float(x[w] << 16), a1 = __uint_as_float(x[w] & 0xffff0000u);
      const float p0 = __uint_as_float(y[w] << 16), p1 = __uint_as_float(y[w] & 0xffff0000u);
      o[w] = pack_bf16(a0 * c0 + sg * p0 * s0, a1 * c1 + sg * p1 * s1);
    }
    val = make_uint4(o[0], o[1], o[2], o[3]);
  }
  const uint32_t dst = (is_k ? sk : sk + kTileBytes) + swz(slot, ch);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(val.x), "r"(val.y), "r"(val.z), "r"(val.w)
               : "memory");
  const int64_t pid = __ldg(a.block_table + static_cast<int64_t>(b) * a.max_blocks + t / a.page_size);
  uint16_t* page = (is_k ? a.k_pages : a.v_pages) + pid * a.page_stride +
                   (static_cast<int64_t>(g) * a.page_size + t % a.page_size) * kHeadDim;
  *reinterpret_cast<uint4*>(page + 8 * ch) = val;
  __syncwarp();
}

__device__ __forceinline__ void init_ring(uint32_t bar0, int stages, int lane) {
  if (lane == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}

// Issue the TMA loads of one tile into a stage (one elected lane).
__device__ __forceinline__ void issue_tile(const CUtensorMap* tmk, const CUtensorMap* tmv, uint32_t dst, uint32_t bar,
                                           int tok_in_page, int g, int pid, uint64_t policy) {
  mbar_arrive_expect_tx(bar, kStageBytes);
  tma_load_tile(dst, tmk, tok_in_page, g, pid, bar, policy);
  tma_load_tile(dst + kTileBytes, tmv, tok_in_page, g, pid, bar, policy);
}

// L2 prefetch of one K + V tile (TMA, no shared memory, no barrier): deepens the
// memory-level parallelism beyond the smem ring.  The L2 is the GPU's point of
// coherence, so a prefetch can never make a later load see stale data.
__device__ __forceinline__ void prefetch_tile_l2(const CUtensorMap* tmk, const CUtensorMap* tmv, int tok_in_page,
                                                 int g, int pid) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   reinterpret_cast<uint64_t>(tmk)),
               "r"(0), "r"(0), "r"(tok_in_page), "r"(g), "r"(pid)
               : "memory");
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   reinterpret_cast<uint64_t>(tmv)),
               "r"(0), "r"(0), "r"(tok_in_page), "r"(g), "r"(pid)
               : "memory");
}

// ------------------------------------------------- kernel 1: one unit per warp

// kStreamOnly = roofline probe (NEO_ATTN_CFG="s4,2"): identical grid, page walk
// and TMA ring, but no math and no output -- the memory-system ceiling of this
// exact access pattern.  Never selected by default.
// CTAs per SM that the stage ring allows; passed to __launch_bounds__ so the
// register budget never becomes the occupancy limit.
template <int kWarps, int kStages>
constexpr int ctas_per_sm() {
  return (220 * 1024) / (kWarps * kStages * kStageBytes + 1024) < 1 ? 1
                                                                      : (220 * 1024) / (kWarps * kStages * kStageBytes + 1024);
}

template <int kWarps, int kStages, bool kStreamOnly = false, bool kFuse = false>
__global__ void __launch_bounds__(kWarps * 32, ctas_per_sm<kWarps, kStages>())
    decode_attn_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                       const KArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[kWarps][kStages];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2;   // MMA groupID
  const int qd = lane & 3;   // MMA thread-in-group

  // Programmatic dependent launch: let the next kernel in the stream get its CTAs
  // resident as soon as every CTA of this grid has started, and wait for the
  // previous kernel (which may have produced q, the KV pages, the block table or
  // seq_lens) to complete before touching any input.  No-ops without PDL.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // Input-free setup overlaps the previous kernel's tail: the tensor-map
  // prefetch (kernel parameters) and this warp's stage barriers (shared memory).
  if (lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv)) : "memory");
  }
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(base) + warp * (kStages * kStageBytes);
  const uint32_t bar0 = smem_u32(&bars[warp][0]);
  init_ring(bar0, kStages, lane);
  // NEO_ATTN_KV_STABLE: metadata and the first KV tiles before the wait (as in
  // decode_attn_group_kernel); otherwise wait before touching any input
  const bool early = !kFuse && a.early;
  if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");

  const int64_t unit = static_cast<int64_t>(blockIdx.x) * kWarps + warp;
  const int64_t BH = static_cast<int64_t>(a.batch) * a.hkv;
  const int c = static_cast<int>(unit / BH);
  if (c >= a.max_chunks) return;
  const int bg = static_cast<int>(unit - static_cast<int64_t>(c) * BH);
  int b = bg / a.hkv;
  int g = bg - b * a.hkv;
  if (a.probe & 64) {   // probe: head-major unit order (a CTA's warps read different requests)
    g = bg / a.batch;
    b = bg - g * a.batch;
  }

  // Issue the block-table walk (a1) and the q loads speculatively, in parallel
  // with the seq_lens load: lane i reads the page of tile i of the chunk (index
  // clamped into the table; entries past the context are loaded but never used).
  const int t_begin = c * a.chunk_tiles;
  int my_pid = 0, my_pid2 = 0;   // pages of tiles lane and 32 + lane (chunks of up to 64 tiles)
  if (lane < a.chunk_tiles) {
    const int pg = min((t_begin + lane) * kTileTokens / a.page_size, a.max_blocks - 1);
    my_pid = __ldg(a.block_table + static_cast<int64_t>(b) * a.max_blocks + pg);
  }
  if (lane + 32 < a.chunk_tiles) {
    const int pg = min((t_begin + 32 + lane) * kTileTokens / a.page_size, a.max_blocks - 1);
    my_pid2 = __ldg(a.block_table + static_cast<int64_t>(b) * a.max_blocks + pg);
  }
  uint4 qf[4];
  if (!early) load_q(a, b, g, r, qd, qf);
  const int ctx = __ldg(a.seq_lens + b);
  if (ctx <= 0) {  // reading c4: empty context -> zero row, pages never read
    if (early) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (c == 0) write_zero_row(a, b, g, lane);
    return;
  }
  if (kFuse && a.inv_freq && r < a.G) rope_q(qf, qd, ctx - 1, a.inv_freq);
  const int ntile_total = (ctx + kTileTokens - 1) / kTileTokens;
  const int n_chunks = (ntile_total + a.chunk_tiles - 1) / a.chunk_tiles;
  if (c >= n_chunks) return;
  const int nt = min(a.chunk_tiles, ntile_total - t_begin);

  const uint64_t policy = evict_first_policy();

  // KV stream (a2): tile j of the unit -> stage j % kStages
  auto issue = [&](int j) {
    const int pid = j < 32 ? __shfl_sync(kFull, my_pid, j) : __shfl_sync(kFull, my_pid2, j - 32);
    if (lane == 0) {
      const int s = j % kStages;
      issue_tile(&tmk, &tmv, sbase + s * kStageBytes, bar0 + 8 * s, ((t_begin + j) * kTileTokens) % a.page_size, g,
                 pid, policy);
    }
  };
  auto prefetch = [&](int j) {   // tile j of the unit into L2 (j warp-uniform)
    if (j >= nt) return;
    const int pid = j < 32 ? __shfl_sync(kFull, my_pid, j) : __shfl_sync(kFull, my_pid2, j - 32);
    if (lane == 0) prefetch_tile_l2(&tmk, &tmv, ((t_begin + j) * kTileTokens) % a.page_size, g, pid);
  };
  const int npro = nt < kStages ? nt : kStages;
  int pre = npro;   // tiles issued before the wait: never the newest token's (the last tile)
  if (early)
    while (pre > 0 && t_begin + pre - 1 >= ntile_total - 1) --pre;
  for (int j = 0; j < pre; ++j) issue(j);
  for (int j = npro; j < npro + a.l2pf + (early && blockIdx.x < a.first_wave ? a.l2pro : 0); ++j) prefetch(j);
  if (early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    load_q(a, b, g, r, qd, qf);
    for (int j = pre; j < npro; ++j) issue(j);
  }

  Acc acc;
  acc_reset(acc);
  for (int j = 0; j < nt; ++j) {
    const int s = j % kStages;
    mbar_wait(bar0 + 8 * s, static_cast<uint32_t>((j / kStages) & 1));
    // read the tile into registers, hand the stage back to TMA, then do the math:
    // the next load is in flight while this tile is being computed
    if (kFuse && c == n_chunks - 1 && j == nt - 1) patch_new_token(a, sbase + s * kStageBytes, b, g, ctx, lane);
    Frags f;
    if (!kStreamOnly) load_frags(sbase + s * kStageBytes, r, qd, f);
    __syncwarp();
    if (j + kStages < nt) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(j + kStages);
      if (a.l2pf) prefetch(j + kStages + a.l2pf);
    }
      if (!kStreamOnly && !(a.probe & 2)) compute_tile(f, qf, ctx - (t_begin + j) * kTileTokens, a.scale_log2, r, qd, acc);
  }
  if (!kStreamOnly && !(a.probe & 1)) finish_unit(a, acc, b, g, c, n_chunks, lane, r, qd);
}


// ------------------------------------------ kernel 2: one CTA per (b, g) group
//
// Grouped split-K: CTA (q, b, g) covers group q of request b's tiles for KV head
// g -- the tiles split into n_groups = ceil(ntiles / T) equal groups (T = 256,
// 128 or 64), each group's tiles dealt round-robin to the 4 warps (<= 64 tiles
// per warp, so one TMA ring and two page-id registers per lane as in kernel 1).  The split depends only on the
// request's own length, so results stay a function of (its inputs) alone.
// The 4 warps merge their (m, l, acc) through shared memory (their own, drained
// stage rings); a single-group request writes its bf16 output right there -- no
// partial rows, no counter -- and only requests longer than 4096 tokens write one
// merged partial per group and run the split-K combine (a7) across groups.
constexpr int kGroupWarps = 4;
static_assert(kGroupTiles / kGroupWarps <= 64, "per-warp range <= 64 tiles (two page-id registers per lane)");

template <int G>
__device__ __forceinline__ void group_merge(const KArgs& a, const uint8_t* base, int stage_bytes, int warp, int lane,
                                            int b, int g, int bg, int q, int n_groups) {
  for (int h = warp; h < G; h += kGroupWarps) {
    float mc[kGroupWarps], lc[kGroupWarps];
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < kGroupWarps; ++c) {
      const float2 t = reinterpret_cast<const float2*>(base + c * stage_bytes + G * kHeadDim * 4)[h];
      mc[c] = t.x;
      lc[c] = t.y;
      M = fmaxf(M, t.x);
    }
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int c = 0; c < kGroupWarps; ++c) {   // warps without tiles have m = -inf, l = 0
      const float w = mc[c] == -INFINITY ? 0.f : ex2(mc[c] - M);
      L += w * lc[c];
      const float4 v = reinterpret_cast<const float4*>(base + c * stage_bytes)[h * (kHeadDim / 4) + lane];
      acc.x += w * v.x;
      acc.y += w * v.y;
      acc.z += w * v.z;
      acc.w += w * v.w;
    }
    if (n_groups == 1) {
      const float inv = 1.f / L;
      uint2 pk;
      pk.x = pack_bf16(acc.x * inv, acc.y * inv);
      pk.y = pack_bf16(acc.z * inv, acc.w * inv);
      *reinterpret_cast<uint2*>(a.out + (static_cast<int64_t>(b) * a.hq + g * G + h) * kHeadDim + 4 * lane) = pk;
    } else {
      const int64_t slot = static_cast<int64_t>(bg) * a.max_chunks + q;
      reinterpret_cast<float4*>(a.ws_acc + (slot * G + h) * kHeadDim)[lane] = acc;
      if (lane == 0) a.ws_ml[slot * G + h] = make_float2(M, L);
    }
  }
}

template <int kStages, bool kFuse = false>
__global__ void __launch_bounds__(kGroupWarps * 32, ctas_per_sm<kGroupWarps, kStages>())
    decode_attn_group_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                             const KArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t bars[kGroupWarps][kStages];
  __shared__ int last_flag;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2;
  const int qd = lane & 3;

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv)) : "memory");
  }
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(base) + warp * (kStages * kStageBytes);
  const uint32_t bar0 = smem_u32(&bars[warp][0]);
  init_ring(bar0, kStages, lane);
  // NEO_ATTN_KV_STABLE: the caller guarantees the kernels still running on the
  // stream write none of the metadata and KV this call reads except each
  // request's newest token, so the metadata and the first KV tiles (not the
  // newest token's) are read BEFORE waiting on the previous grid: the KV
  // stream starts during its tail.  q, and everything written, after the wait.
  const bool early = !kFuse && a.early;
  if (!early) asm volatile("griddepcontrol.wait;" ::: "memory");

  const int64_t BH = static_cast<int64_t>(a.batch) * a.hkv;
  int q = static_cast<int>(blockIdx.x / BH);
  int bg = static_cast<int>(blockIdx.x - static_cast<int64_t>(q) * BH);
  if (a.req_major) {   // request-major order: a request's groups adjacent (see launch_decode_attn)
    const int64_t per_b = static_cast<int64_t>(a.max_chunks) * a.hkv;
    const int bb = static_cast<int>(blockIdx.x / per_b);
    const int rem = static_cast<int>(blockIdx.x - bb * per_b);
    q = rem / a.hkv;
    bg = bb * a.hkv + (rem - q * a.hkv);
  }
  const int b = bg / a.hkv;
  const int g = bg - b * a.hkv;
  uint4 qf[4];
  if (!early) load_q(a, b, g, r, qd, qf);
  // Warp w takes tiles g0 + w, g0 + w + 4, ... of its group (interleaved), so for
  // the first group (g0 = 0, every single-group request) lane i's page ids --
  // tiles w + 4i and w + 4(i + 32) -- are known before seq_lens arrives: issue
  // them with it (entries past the context are clamped into the row, never used).
  const int32_t* bt_row = a.block_table + static_cast<int64_t>(b) * a.max_blocks;
  int my_pid = 0, my_pid2 = 0;
  if (q == 0) {
    my_pid = __ldg(bt_row + min((warp + 4 * lane) * kTileTokens / a.page_size, a.max_blocks - 1));
    my_pid2 = __ldg(bt_row + min((warp + 4 * (lane + 32)) * kTileTokens / a.page_size, a.max_blocks - 1));
  }
  const int ctx = __ldg(a.seq_lens + b);
  if (ctx <= 0) {  // reading c4: empty context -> zero row, pages never read
    if (early) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (q == 0 && warp == 0) write_zero_row(a, b, g, lane);
    return;
  }
  if (kFuse && a.inv_freq && r < a.G) rope_q(qf, qd, ctx - 1, a.inv_freq);
  const int ntile_total = (ctx + kTileTokens - 1) / kTileTokens;
  const int n_groups = (ntile_total + a.chunk_tiles - 1) / a.chunk_tiles;   // chunk_tiles = group tiles
  if (q >= n_groups) return;                       // uniform over the CTA (same b, q)
  const int tg = (ntile_total + n_groups - 1) / n_groups;
  const int g0 = q * tg, g1 = min(g0 + tg, ntile_total);
  const int first = g0 + warp;                              // tiles first, first + 4, ... < g1
  const int nt = first < g1 ? (g1 - first + kGroupWarps - 1) / kGroupWarps : 0;
  if (q > 0) {
    if (lane < nt) my_pid = __ldg(bt_row + (first + kGroupWarps * lane) * kTileTokens / a.page_size);
    if (lane + 32 < nt) my_pid2 = __ldg(bt_row + (first + kGroupWarps * (lane + 32)) * kTileTokens / a.page_size);
  }
  const uint64_t policy = evict_first_policy();
  auto issue = [&](int j) {
    const int pid = j < 32 ? __shfl_sync(kFull, my_pid, j) : __shfl_sync(kFull, my_pid2, j - 32);
    if (lane == 0) {
      const int s = j % kStages;
      issue_tile(&tmk, &tmv, sbase + s * kStageBytes, bar0 + 8 * s,
                 ((first + kGroupWarps * j) * kTileTokens) % a.page_size, g, pid, policy);
    }
  };
  auto prefetch = [&](int j) {   // this warp's tile j into L2 (j warp-uniform)
    if (j >= nt) return;
    const int pid = j < 32 ? __shfl_sync(kFull, my_pid, j) : __shfl_sync(kFull, my_pid2, j - 32);
    if (lane == 0) prefetch_tile_l2(&tmk, &tmv, ((first + kGroupWarps * j) * kTileTokens) % a.page_size, g, pid);
  };
  const int npro = nt < kStages ? nt : kStages;
  int pre = npro;   // tiles issued before the wait: never the newest token's (the last tile)
  if (early)
    while (pre > 0 && first + kGroupWarps * (pre - 1) >= ntile_total - 1) --pre;
  for (int j = 0; j < pre; ++j) issue(j);
  for (int j = npro; j < npro + a.l2pf + (early && blockIdx.x < a.first_wave ? a.l2pro : 0); ++j) prefetch(j);
  if (early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    load_q(a, b, g, r, qd, qf);
    for (int j = pre; j < npro; ++j) issue(j);
  }

  Acc acc;
  acc_reset(acc);
  for (int j = 0; j < nt; ++j) {
    const int s = j % kStages;
    mbar_wait(bar0 + 8 * s, static_cast<uint32_t>((j / kStages) & 1));
    // fused append: the warp whose range ends the request holds the new token
    if (kFuse && first + kGroupWarps * j == ntile_total - 1)
      patch_new_token(a, sbase + s * kStageBytes, b, g, ctx, lane);
    Frags f;
    load_frags(sbase + s * kStageBytes, r, qd, f);
    __syncwarp();
    if (j + kStages < nt) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(j + kStages);
      if (a.l2pf) prefetch(j + kStages + a.l2pf);
    }
    compute_tile(f, qf, ctx - (first + kGroupWarps * j) * kTileTokens, a.scale_log2, r, qd, acc);
  }

  // (a6/a7 in the CTA) this warp's (acc, m, l) into its drained stage ring
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    acc.l0 += __shfl_xor_sync(kFull, acc.l0, off);
    acc.l1 += __shfl_xor_sync(kFull, acc.l1, off);
  }
  const int G = a.G;
  const int h0 = 2 * qd, h1 = 2 * qd + 1;
  float* sp = reinterpret_cast<float*>(base + warp * (kStages * kStageBytes));
  if (h0 < G) {
    *reinterpret_cast<float4*>(sp + h0 * kHeadDim + 8 * r) = make_float4(acc.o[0][0], acc.o[1][0], acc.o[2][0], acc.o[3][0]);
    *reinterpret_cast<float4*>(sp + h0 * kHeadDim + 8 * r + 4) = make_float4(acc.o[4][0], acc.o[5][0], acc.o[6][0], acc.o[7][0]);
    *reinterpret_cast<float4*>(sp + h0 * kHeadDim + 64 + 8 * r) = make_float4(acc.o[0][2], acc.o[1][2], acc.o[2][2], acc.o[3][2]);
    *reinterpret_cast<float4*>(sp + h0 * kHeadDim + 68 + 8 * r) = make_float4(acc.o[4][2], acc.o[5][2], acc.o[6][2], acc.o[7][2]);
    if (r == 0) reinterpret_cast<float2*>(sp + G * kHeadDim)[h0] = make_float2(acc.m0, acc.l0);
  }
  if (h1 < G) {
    *reinterpret_cast<float4*>(sp + h1 * kHeadDim + 8 * r) = make_float4(acc.o[0][1], acc.o[1][1], acc.o[2][1], acc.o[3][1]);
    *reinterpret_cast<float4*>(sp + h1 * kHeadDim + 8 * r + 4) = make_float4(acc.o[4][1], acc.o[5][1], acc.o[6][1], acc.o[7][1]);
    *reinterpret_cast<float4*>(sp + h1 * kHeadDim + 64 + 8 * r) = make_float4(acc.o[0][3], acc.o[1][3], acc.o[2][3], acc.o[3][3]);
    *reinterpret_cast<float4*>(sp + h1 * kHeadDim + 68 + 8 * r) = make_float4(acc.o[4][3], acc.o[5][3], acc.o[6][3], acc.o[7][3]);
    if (r == 0) reinterpret_cast<float2*>(sp + G * kHeadDim)[h1] = make_float2(acc.m1, acc.l1);
  }
  __syncthreads();
  const int sb = kStages * kStageBytes;
  switch (G) {
    case 1: group_merge<1>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
    case 2: group_merge<2>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
    case 3: group_merge<3>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
    case 4: group_merge<4>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
    case 5: group_merge<5>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
    case 6: group_merge<6>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
    case 7: group_merge<7>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
    default: group_merge<8>(a, base, sb, warp, lane, b, g, bg, q, n_groups); break;
  }
  if (n_groups == 1) return;
  // publish this group's merged partial; the last-arriving group runs the combine
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int prev;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(prev) : "l"(a.ws_cnt + bg) : "memory");
    last_flag = prev == n_groups - 1;
  }
  __syncthreads();
  if (!last_flag || warp != 0) return;
  switch (G) {
    case 1: combine<1>(a, b, g, bg, n_groups, lane); break;
    case 2: combine<2>(a, b, g, bg, n_groups, lane); break;
    case 3: combine<3>(a, b, g, bg, n_groups, lane); break;
    case 4: combine<4>(a, b, g, bg, n_groups, lane); break;
    case 5: combine<5>(a, b, g, bg, n_groups, lane); break;
    case 6: combine<6>(a, b, g, bg, n_groups, lane); break;
    case 7: combine<7>(a, b, g, bg, n_groups, lane); break;
    default: combine<8>(a, b, g, bg, n_groups, lane); break;
  }
  if (lane == 0) a.ws_cnt[bg] = 0;  // leave the workspace re-usable
}
}  // namespace

size_t workspace_counter_cap(size_t ws_bytes) { return (ws_bytes / 64) & ~size_t(255); }

static size_t up256(size_t x) { return (x + 255) & ~size_t(255); }

static void data_bytes(int32_t batch, int32_t hq, int32_t hkv, int32_t max_chunks, size_t* ml, size_t* acc) {
  const int64_t G = hkv > 0 ? hq / hkv : 0;
  const int64_t units = static_cast<int64_t>(batch) * hkv * max_chunks;
  const bool split = max_chunks > 1;
  *ml = split ? up256(static_cast<size_t>(units * G) * sizeof(float2)) : 0;
  *acc = split ? up256(static_cast<size_t>(units * G * kHeadDim) * sizeof(float)) : 0;
}

WorkspaceLayout workspace_layout(int32_t batch, int32_t hq, int32_t hkv, int32_t max_chunks, size_t ws_bytes) {
  size_t ml, acc;
  data_bytes(batch, hq, hkv, max_chunks, &ml, &acc);
  WorkspaceLayout w;
  w.cnt_off = 0;
  w.cnt_cap = workspace_counter_cap(ws_bytes);
  w.ml_off = w.cnt_cap;
  w.acc_off = w.ml_off + ml;
  w.total = w.acc_off + acc;
  w.fits = w.total <= ws_bytes && static_cast<size_t>(batch) * hkv * sizeof(int32_t) <= w.cnt_cap;
  return w;
}

size_t workspace_required(int32_t batch, int32_t hq, int32_t hkv, int32_t max_chunks) {
  size_t ml, acc;
  data_bytes(batch, hq, hkv, max_chunks, &ml, &acc);
  const size_t need_cnt = up256(static_cast<size_t>(batch) * hkv * sizeof(int32_t));
  size_t S = up256(ml + acc + need_cnt + 256);
  while (!workspace_layout(batch, hq, hkv, max_chunks, S).fits) S = up256(S + std::max<size_t>(256, S / 128));
  return S;
}

// NEO_PDL=0 disables programmatic dependent launch (default on).
static bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("NEO_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

template <int W, int S, bool kStreamOnly = false, bool kFuse = false>
static neo_status launch_unit(const KArgs& a, const CUtensorMap& tmk, const CUtensorMap& tmv, int64_t units,
                              cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  constexpr int smem = W * S * kStageBytes + 1024;
  neo_status st = once_per_device(configured, [](int) {
    cudaError_t e =
        cudaFuncSetAttribute(decode_attn_kernel<W, S, kStreamOnly, kFuse>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             smem);
    return e == cudaSuccess ? NEO_OK : cuda_fail(e, "cudaFuncSetAttribute(decode_attn_kernel)");
  });
  if (st != NEO_OK) return st;
  const int64_t grid = (units + W - 1) / W;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KArgs ka = a;
  ka.first_wave = device_sm_count() * ctas_per_sm<W, S>();
  cudaLaunchKernelEx(&cfg, decode_attn_kernel<W, S, kStreamOnly, kFuse>, tmk, tmv, ka);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "decode_attn_kernel launch");
  return NEO_OK;
}

// Stages per warp of the grouped kernel: 2 (3 CTAs/SM); NEO_ATTN_GROUP_STAGES=3
// (2 CTAs/SM) is an experiment knob.
static int group_stages() {
  static const int k = [] {
    const char* v = std::getenv("NEO_ATTN_GROUP_STAGES");
    return v ? std::atoi(v) : 2;
  }();
  return k;
}

template <int S, bool kFuse>
static neo_status launch_group(const KArgs& a, const CUtensorMap& tmk, const CUtensorMap& tmv, int64_t ctas,
                               cudaStream_t stream) {
  static std::atomic<uint64_t> configured{0};
  constexpr int smem = kGroupWarps * S * kStageBytes + 1024;
  neo_status st = once_per_device(configured, [](int) {
    cudaError_t e =
        cudaFuncSetAttribute(decode_attn_group_kernel<S, kFuse>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return e == cudaSuccess ? NEO_OK : cuda_fail(e, "cudaFuncSetAttribute(decode_attn_group_kernel)");
  });
  if (st != NEO_OK) return st;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(ctas));
  cfg.blockDim = dim3(kGroupWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  KArgs ka = a;
  ka.first_wave = device_sm_count() * ctas_per_sm<kGroupWarps, S>();
  cudaLaunchKernelEx(&cfg, decode_attn_group_kernel<S, kFuse>, tmk, tmv, ka);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "decode_attn_group_kernel launch");
  return NEO_OK;
}

// Kernel shape: kWarps independent warps per CTA x kStages TMA stages per warp.
// Default, from same-box sweeps (profiles/r01_sweep.md): (4, 3) -- 97 KiB of
// stages, 2 CTAs/SM -- when every request spans <= 3 chunks (c2: +2 % over
// (4, 2)); (4, 2) -- 65 KiB, 3 CTAs/SM -- for longer contexts (c5: +3 % over
// (4, 3); c3 ties).  NEO_ATTN_CFG="uW,S" forces a compiled shape for tuning
// experiments; "sW,S" selects the stream-only roofline probe.
static int attn_cfg() {
  static int cfg = [] {
    const char* v = std::getenv("NEO_ATTN_CFG");
    if (!v) return 0;
    int w = 0, s = 0;
    char kind = 'u';
    if (std::sscanf(v, "%c%d,%d", &kind, &w, &s) != 3) return 0;
    return (kind == 's' ? 1000 : 0) + w * 10 + s;
  }();
  return cfg;
}

neo_status launch_decode_attn(const AttnLaunch& L, const CUtensorMap& tmk, const CUtensorMap& tmv) {
  const WorkspaceLayout w = workspace_layout(L.batch, L.hq, L.hkv, L.max_chunks, L.workspace_bytes);
  uint8_t* ws = static_cast<uint8_t*>(L.workspace);
  KArgs a;
  a.q = static_cast<const uint16_t*>(L.q);
  a.out = static_cast<uint16_t*>(L.out);
  a.block_table = L.block_table;
  a.seq_lens = L.seq_lens;
  a.ws_cnt = reinterpret_cast<int32_t*>(ws + w.cnt_off);
  a.ws_ml = reinterpret_cast<float2*>(ws + w.ml_off);
  a.ws_acc = reinterpret_cast<float*>(ws + w.acc_off);
  a.batch = L.batch;
  a.hq = L.hq;
  a.hkv = L.hkv;
  a.G = L.hq / L.hkv;
  a.page_size = L.page_size;
  a.max_blocks = L.max_blocks;
  a.chunk_tiles = L.chunk_tokens / kTileTokens;
  a.max_chunks = L.max_chunks;
  a.scale_log2 = L.scale * 1.4426950408889634f;
  a.inv_freq = L.inv_freq;
  a.k_new = static_cast<const uint16_t*>(L.k_new);
  a.v_new = static_cast<const uint16_t*>(L.v_new);
  a.k_pages = static_cast<uint16_t*>(L.k_pages);
  a.v_pages = static_cast<uint16_t*>(L.v_pages);
  a.page_stride = L.page_stride;
  static const int probe = [] {
    const char* v = std::getenv("NEO_ATTN_PROBE");
    return v ? std::atoi(v) : 0;
  }();
  a.probe = probe;
  a.early = L.early ? 1 : 0;
  static const int l2pf = [] {
    const char* v = std::getenv("NEO_ATTN_L2PF");
    return v ? std::max(0, std::min(16, std::atoi(v))) : 0;
  }();
  a.l2pf = l2pf;
  static const int l2pro = [] {
    const char* v = std::getenv("NEO_ATTN_L2PRO");
    return v ? std::max(0, std::min(32, std::atoi(v))) : 2;
  }();
  a.l2pro = l2pro;
  const int64_t units = static_cast<int64_t>(L.max_chunks) * L.batch * L.hkv;
  if (L.grouped) {   // grouped kernel: max_chunks = groups per request, chunk_tiles = group tiles
    a.chunk_tiles = group_tiles_of(L.chunk_tokens);
    // CTA order: group-major (all first groups, then all second groups, ...) for
    // up to two groups per request; request-major from three on, so that the
    // empty CTAs (q >= the request's group count) are spread over the grid instead
    // of bunched at its end, and a long request's groups start together (same-box
    // A/B, profiles/r02_group_sweep.md: skewed c2s +6 %, c5 +1 %, c3 +0.5 %; the
    // two-group c4 shard at N = 8 is 5 % faster group-major).  neo_decode_attn_plan_chunk
    // replays the same order.
    a.req_major = L.max_chunks >= 3 ? 1 : 0;
    const int64_t ctas = static_cast<int64_t>(L.max_chunks) * L.batch * L.hkv;
    if (L.k_new) return launch_group<2, true>(a, tmk, tmv, ctas, L.stream);
    return group_stages() == 3 ? launch_group<3, false>(a, tmk, tmv, ctas, L.stream)
                               : launch_group<2, false>(a, tmk, tmv, ctas, L.stream);
  }
  if (L.k_new) {   // fused append (+ RoPE): the two default shapes
    return L.max_chunks <= 3 ? launch_unit<4, 3, false, true>(a, tmk, tmv, units, L.stream)
                             : launch_unit<4, 2, false, true>(a, tmk, tmv, units, L.stream);
  }
  int cfg = attn_cfg();
  if (cfg == 0) {
    const AttnShape sh = default_attn_shape(L.max_chunks);
    cfg = sh.warps * 10 + sh.stages;
  }
  switch (cfg) {
    case 1042: return launch_unit<4, 2, true>(a, tmk, tmv, units, L.stream);
    case 1043: return launch_unit<4, 3, true>(a, tmk, tmv, units, L.stream);
    case 1044: return launch_unit<4, 4, true>(a, tmk, tmv, units, L.stream);
    case 44: return launch_unit<4, 4>(a, tmk, tmv, units, L.stream);
    case 28: return launch_unit<2, 8>(a, tmk, tmv, units, L.stream);
    case 46: return launch_unit<4, 6>(a, tmk, tmv, units, L.stream);
    case 48: return launch_unit<4, 8>(a, tmk, tmv, units, L.stream);
    case 43: return launch_unit<4, 3>(a, tmk, tmv, units, L.stream);
    case 23: return launch_unit<2, 3>(a, tmk, tmv, units, L.stream);
    case 22: return launch_unit<2, 2>(a, tmk, tmv, units, L.stream);
    case 12: return launch_unit<1, 2>(a, tmk, tmv, units, L.stream);
    case 13: return launch_unit<1, 3>(a, tmk, tmv, units, L.stream);
    case 33: return launch_unit<3, 3>(a, tmk, tmv, units, L.stream);
    case 62: return launch_unit<6, 2>(a, tmk, tmv, units, L.stream);
    case 82: return launch_unit<8, 2>(a, tmk, tmv, units, L.stream);
    default: return launch_unit<4, 2>(a, tmk, tmv, units, L.stream);
  }
}

}  // namespace neo
