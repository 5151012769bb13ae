// CPU paged decode attention over the CPU-cache -- NEO's PACPU,
// the attention of CPU-requests, whose KV lives in pinned host
// pages [num_host_pages][L][2][Hkv][P][D] (include/neo.h).
//
// Partition: the (request b, kv-head g, page j) blocks of the batch are
// laid out request-major and dealt to the threads in equal contiguous ranges
// ("each thread having an equal number of blocks to process"); every maximal run
// of one (b, g) inside a thread's range is a task that produces a flash-decoding
// partial (m, l, acc) for the G q-heads of g.  The partials of each (b, g) are
// then merged in block order ("aggregate the partial outputs of each request").
// Within a core: AVX-512 -- bf16 K/V rows widened to fp32 in registers,
// FMAs against the group's q, online softmax per page, contiguous page reads.
#include <immintrin.h>

#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/neo.h"

namespace neo {
neo_status fail(neo_status st, const std::string& msg);
}

struct neo_kv_pool;
namespace neo {
// accessors implemented in neo_host.cu (the pool struct is private to it)
const neo_kv_geometry* pool_geometry(const neo_kv_pool* p);
const uint8_t* pool_host_base(const neo_kv_pool* p);
}  // namespace neo

namespace {

// Persistent host worker pool: neo_cpu_decode_attn runs once per layer per
// iteration (T_ca), so creating and joining threads per call would
// add ~0.1 ms of fixed cost to every CPU sub-batch.  Workers are created on
// first use (grown on demand), spin briefly and then sleep on a condition
// variable between parallel regions; run() hands out task indices through one
// atomic counter (the caller takes tasks too) and returns when all completed.
// One parallel region at a time (region_mu_).  A forked child does not inherit
// the threads, so the pool restarts when the pid changes.
class WorkerPool {
 public:
  static WorkerPool& get() {
    static WorkerPool* p = new WorkerPool();  // never destroyed: workers may still sleep at exit
    return *p;
  }

  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 1) {
      if (n == 1) fn(0);
      return;
    }
    std::lock_guard<std::mutex> region(region_mu_);
    if (pid_ != getpid()) {  // forked: the workers belong to the parent
      for (auto& t : workers_) t.detach();
      workers_.clear();
      pid_ = getpid();
    }
    while (static_cast<int>(workers_.size()) < n - 1) workers_.emplace_back([this] { loop(); });
    fn_.store(&fn, std::memory_order_relaxed);
    n_.store(n, std::memory_order_relaxed);
    pending_.store(n, std::memory_order_relaxed);
    const uint64_t g = (state_.load(std::memory_order_relaxed) >> 32) + 1;
    {
      std::lock_guard<std::mutex> lk(mu_);
      state_.store(g << 32, std::memory_order_release);   // generation g, next task 0
    }
    cv_.notify_all();
    work(g);
    for (int spins = 0; pending_.load(std::memory_order_acquire) != 0; ++spins) {
      if (spins < 4096) _mm_pause();
      else std::this_thread::yield();
    }
  }

 private:
  WorkerPool() : pid_(getpid()) {}

  // Claims tasks of generation g only: the (generation, next index) pair is one
  // atomic word, so a worker still finishing an older region can never take a
  // task of a newer one (whose fn_ / n_ it might not see yet).
  void work(uint64_t g) {
    for (;;) {
      uint64_t st = state_.load(std::memory_order_acquire);
      int t = -1;
      while ((st >> 32) == g) {
        const int idx = static_cast<int>(st & 0xffffffffu);
        if (idx >= n_.load(std::memory_order_relaxed)) return;
        if (state_.compare_exchange_weak(st, st + 1, std::memory_order_acq_rel, std::memory_order_acquire)) {
          t = idx;
          break;
        }
      }
      if (t < 0) return;
      (*fn_.load(std::memory_order_relaxed))(t);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }

  void loop() {
    uint64_t seen = state_.load(std::memory_order_acquire) >> 32;
    for (;;) {
      uint64_t g = seen;
      for (int spins = 0; spins < 20000 && (g = state_.load(std::memory_order_acquire) >> 32) == seen; ++spins)
        _mm_pause();
      if (g == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return (state_.load(std::memory_order_acquire) >> 32) != seen; });
        g = state_.load(std::memory_order_acquire) >> 32;
      }
      seen = g;
      work(g);
    }
  }

  std::mutex region_mu_, mu_;
  std::condition_variable cv_;
  std::vector<std::thread> workers_;
  std::atomic<const std::function<void(int)>*> fn_{nullptr};
  std::atomic<int> n_{0}, pending_{0};
  std::atomic<uint64_t> state_{0};   // generation << 32 | next task index
  pid_t pid_;
};

constexpr int kD = 128;
constexpr int kMaxG = 16;

inline float bf16_to_f32(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

struct Partial {
  float m[kMaxG], l[kMaxG];
  float acc[kMaxG][kD];
};

struct Job {
  const uint8_t* host;        // CPU-cache base
  int64_t page_elems;         // Hkv * P * D
  int32_t L, layer, hkv, P, G, hq;
  const uint16_t* q;
  const int32_t* table;
  int32_t max_blocks;
  const int32_t* seq_lens;
  float scale;
};

inline const uint16_t* page_kv(const Job& j, int32_t host_page, int kv, int g) {
  const uint16_t* base = reinterpret_cast<const uint16_t*>(j.host);
  return base + ((static_cast<int64_t>(host_page) * j.L + j.layer) * 2 + kv) * j.page_elems +
         static_cast<int64_t>(g) * j.P * kD;
}

// ---- one task: pages [j0, j1) of (b, g), G q-heads; generic (portable) path
void task_generic(const Job& jb, int b, int g, int j0, int j1, Partial& out) {
  const int G = jb.G, P = jb.P, ctx = jb.seq_lens[b];
  float qf[kMaxG][kD];
  for (int h = 0; h < G; ++h)
    for (int d = 0; d < kD; ++d) qf[h][d] = bf16_to_f32(jb.q[(static_cast<int64_t>(b) * jb.hq + g * G + h) * kD + d]);
  for (int h = 0; h < G; ++h) {
    out.m[h] = -INFINITY;
    out.l[h] = 0.f;
    for (int d = 0; d < kD; ++d) out.acc[h][d] = 0.f;
  }
  float s[kMaxG][64];
  for (int j = j0; j < j1; ++j) {
    const int32_t pg = jb.table[static_cast<int64_t>(b) * jb.max_blocks + j];
    const uint16_t* K = page_kv(jb, pg, 0, g);
    const uint16_t* V = page_kv(jb, pg, 1, g);
    const int nt = std::min(P, ctx - j * P);
    for (int h = 0; h < G; ++h) {
      float mx = -INFINITY;
      for (int t = 0; t < nt; ++t) {
        float a = 0.f;
        for (int d = 0; d < kD; ++d) a += qf[h][d] * bf16_to_f32(K[t * kD + d]);
        s[h][t] = a * jb.scale;
        mx = std::max(mx, s[h][t]);
      }
      const float mn = std::max(out.m[h], mx);
      const float al = std::exp(out.m[h] - mn);
      out.l[h] *= al;
      for (int d = 0; d < kD; ++d) out.acc[h][d] *= al;
      out.m[h] = mn;
      for (int t = 0; t < nt; ++t) {
        const float p = std::exp(s[h][t] - mn);
        out.l[h] += p;
        for (int d = 0; d < kD; ++d) out.acc[h][d] += p * bf16_to_f32(V[t * kD + d]);
      }
    }
  }
}

// ---- AVX-512 path: 8 zmm of fp32 per 128-dim row
__attribute__((target("avx512f,avx512bw"))) inline __m512 load_bf16x16(const uint16_t* p) {
  const __m256i raw = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p));
  return _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(raw), 16));
}

__attribute__((target("avx512f,avx512bw"))) void task_avx512(const Job& jb, int b, int g, int j0, int j1,
                                                              Partial& out) {
  const int G = jb.G, P = jb.P, ctx = jb.seq_lens[b];
  alignas(64) float qf[kMaxG][kD];
  for (int h = 0; h < G; ++h)
    for (int c = 0; c < 8; ++c)
      _mm512_store_ps(&qf[h][16 * c],
                      load_bf16x16(jb.q + (static_cast<int64_t>(b) * jb.hq + g * G + h) * kD + 16 * c));
  for (int h = 0; h < G; ++h) {
    out.m[h] = -INFINITY;
    out.l[h] = 0.f;
    for (int d = 0; d < kD; d += 16) _mm512_storeu_ps(&out.acc[h][d], _mm512_setzero_ps());
  }
  alignas(64) float s[kMaxG][64];
  for (int j = j0; j < j1; ++j) {
    const int32_t pg = jb.table[static_cast<int64_t>(b) * jb.max_blocks + j];
    const uint16_t* K = page_kv(jb, pg, 0, g);
    const uint16_t* V = page_kv(jb, pg, 1, g);
    const int nt = std::min(P, ctx - j * P);
    // scores: each K row is widened once and used by all G heads
    for (int t = 0; t < nt; ++t) {
      __m512 k[8];
      for (int c = 0; c < 8; ++c) k[c] = load_bf16x16(K + t * kD + 16 * c);
      for (int h = 0; h < G; ++h) {
        __m512 a = _mm512_mul_ps(k[0], _mm512_load_ps(&qf[h][0]));
        for (int c = 1; c < 8; ++c) a = _mm512_fmadd_ps(k[c], _mm512_load_ps(&qf[h][16 * c]), a);
        s[h][t] = _mm512_reduce_add_ps(a) * jb.scale;
      }
    }
    // online softmax per head, then P.V with each V row widened once
    float pw[kMaxG][64];
    for (int h = 0; h < G; ++h) {
      float mx = -INFINITY;
      for (int t = 0; t < nt; ++t) mx = std::max(mx, s[h][t]);
      const float mn = std::max(out.m[h], mx);
      const float al = std::exp(out.m[h] - mn);
      if (al != 1.f) {
        const __m512 va = _mm512_set1_ps(al);
        for (int d = 0; d < kD; d += 16) _mm512_storeu_ps(&out.acc[h][d], _mm512_mul_ps(_mm512_loadu_ps(&out.acc[h][d]), va));
        out.l[h] *= al;
      }
      out.m[h] = mn;
      for (int t = 0; t < nt; ++t) {
        pw[h][t] = std::exp(s[h][t] - mn);
        out.l[h] += pw[h][t];
      }
    }
    for (int t = 0; t < nt; ++t) {
      __m512 v[8];
      for (int c = 0; c < 8; ++c) v[c] = load_bf16x16(V + t * kD + 16 * c);
      for (int h = 0; h < G; ++h) {
        const __m512 p = _mm512_set1_ps(pw[h][t]);
        for (int c = 0; c < 8; ++c)
          _mm512_storeu_ps(&out.acc[h][16 * c], _mm512_fmadd_ps(p, v[c], _mm512_loadu_ps(&out.acc[h][16 * c])));
      }
    }
  }
}

// ---- AVX-512 BF16 path (Sapphire Rapids and later): per 16-token tile
//   scores: vdpbf16ps on the raw bf16 K rows and q (products of bf16 are exact in
//           fp32), 16 per-token accumulators folded with a transpose-reduce;
//   softmax: vector exp2 (round + degree-6 polynomial + scalef), masked tail;
//   P.V:    fp32 FMAs, V rows widened once, accumulators in registers (2 heads).
#define NEO_BF16_TARGET __attribute__((target("avx512f,avx512bw,avx512dq,avx512vl,avx512bf16")))

NEO_BF16_TARGET inline __m512 hsum16x16(__m512 v[16]) {
  __m512 x[8], y[4], w[2];
  for (int i = 0; i < 8; ++i)
    x[i] = _mm512_add_ps(_mm512_unpacklo_ps(v[2 * i], v[2 * i + 1]), _mm512_unpackhi_ps(v[2 * i], v[2 * i + 1]));
  for (int i = 0; i < 4; ++i) {
    const __m512d a = _mm512_castps_pd(x[2 * i]), b = _mm512_castps_pd(x[2 * i + 1]);
    y[i] = _mm512_add_ps(_mm512_castpd_ps(_mm512_unpacklo_pd(a, b)), _mm512_castpd_ps(_mm512_unpackhi_pd(a, b)));
  }
  for (int i = 0; i < 2; ++i)
    w[i] = _mm512_add_ps(_mm512_shuffle_f32x4(y[2 * i], y[2 * i + 1], 0x88),
                         _mm512_shuffle_f32x4(y[2 * i], y[2 * i + 1], 0xDD));
  return _mm512_add_ps(_mm512_shuffle_f32x4(w[0], w[1], 0x88), _mm512_shuffle_f32x4(w[0], w[1], 0xDD));
}

// 2^y for y <= 0 (lanes with y = -inf give 0)
NEO_BF16_TARGET inline __m512 exp2_vec(__m512 y) {
  y = _mm512_max_ps(y, _mm512_set1_ps(-127.f));
  const __m512 n = _mm512_roundscale_ps(y, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  const __m512 f = _mm512_sub_ps(y, n);  // [-0.5, 0.5]
  __m512 p = _mm512_set1_ps(1.5403530e-4f);
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.3333558e-3f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(9.6181291e-3f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(5.5504109e-2f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(2.4022651e-1f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(6.9314718e-1f));
  p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.f));
  return _mm512_scalef_ps(p, n);
}

// kG = compile-time group size (0 = runtime jb.G): fixed G lets the head loops
// unroll so the per-head score / softmax dependency chains interleave.
template <int kG>
NEO_BF16_TARGET void task_avx512bf16(const Job& jb, int b, int g, int j0, int j1, Partial& out) {
  const int G = kG > 0 ? kG : jb.G;
  const int P = jb.P, ctx = jb.seq_lens[b];
  const float l2e = 1.4426950408889634f;
  const __m512 sl2 = _mm512_set1_ps(jb.scale * l2e);
  const uint16_t* qb = jb.q + (static_cast<int64_t>(b) * jb.hq + g * G) * kD;
  __m512i qv[kMaxG][4];  // q rows as 4 x 32 bf16
  for (int h = 0; h < G; ++h)
    for (int c = 0; c < 4; ++c) qv[h][c] = _mm512_loadu_si512(qb + h * kD + 32 * c);
  float m2[kMaxG], l[kMaxG];  // running max in the log2 domain, running sum
  for (int h = 0; h < G; ++h) {
    m2[h] = -INFINITY;
    l[h] = 0.f;
    for (int d = 0; d < kD; d += 16) _mm512_storeu_ps(&out.acc[h][d], _mm512_setzero_ps());
  }
  alignas(64) float pw[kMaxG][16];
  float alpha[kMaxG];  // per-head rescale factor of the running state for this tile
  for (int j = j0; j < j1; ++j) {
    const int32_t pg = jb.table[static_cast<int64_t>(b) * jb.max_blocks + j];
    const uint16_t* Kp = page_kv(jb, pg, 0, g);
    const uint16_t* Vp = page_kv(jb, pg, 1, g);
    const int np = std::min(P, ctx - j * P);
    for (int t0 = 0; t0 < np; t0 += 16) {
      const int nt = std::min(16, np - t0);
      const uint16_t* K = Kp + t0 * kD;
      const uint16_t* V = Vp + t0 * kD;
      const __mmask16 valid = static_cast<__mmask16>((1u << nt) - 1u);
      // (a3) scores of all heads; rows past the context load as zeros
      __m512 sc[kMaxG];
#pragma GCC unroll 8
      for (int h = 0; h < G; ++h) {
        __m512 acc[16];
#pragma GCC unroll 16
        for (int t = 0; t < 16; ++t) {
          const __mmask32 mt = t < nt ? 0xffffffffu : 0u;
          __m512 a = _mm512_setzero_ps();
#pragma GCC unroll 4
          for (int c = 0; c < 4; ++c)
            a = _mm512_dpbf16_ps(a, (__m512bh)_mm512_maskz_loadu_epi16(mt, K + t * kD + 32 * c), (__m512bh)qv[h][c]);
          acc[t] = a;
        }
        sc[h] = _mm512_mask_mov_ps(_mm512_set1_ps(-INFINITY), valid, _mm512_mul_ps(hsum16x16(acc), sl2));
      }
      // (a4) online softmax, branch-free rescale of the running state
#pragma GCC unroll 8
      for (int h = 0; h < G; ++h) {
        const float mn = std::max(m2[h], _mm512_reduce_max_ps(sc[h]));
        alpha[h] = _mm512_cvtss_f32(exp2_vec(_mm512_set1_ps(m2[h] - mn)));   // 0 when m2 = -inf
        const __m512 p = _mm512_maskz_mov_ps(valid, exp2_vec(_mm512_sub_ps(sc[h], _mm512_set1_ps(mn))));
        l[h] = l[h] * alpha[h] + _mm512_reduce_add_ps(p);
        m2[h] = mn;
        _mm512_store_ps(pw[h], p);
      }
      // (a5) P.V.  G a multiple of 4: four heads at a time over one half of the
      // dims per pass (16 accumulators in registers), so each V row is widened
      // once per head quad instead of once per head pair.
      if (kG > 0 && kG % 4 == 0) {
#pragma GCC unroll 2
        for (int h = 0; h < G; h += 4) {
#pragma GCC unroll 2
          for (int half = 0; half < 2; ++half) {
            const int c0 = 4 * half;
            __m512 a[4][4];
#pragma GCC unroll 4
            for (int i = 0; i < 4; ++i) {
              const __m512 al = _mm512_set1_ps(alpha[h + i]);
#pragma GCC unroll 4
              for (int c = 0; c < 4; ++c) a[i][c] = _mm512_mul_ps(_mm512_loadu_ps(&out.acc[h + i][16 * (c0 + c)]), al);
            }
            for (int t = 0; t < nt; ++t) {
              __m512 v[4];
#pragma GCC unroll 4
              for (int c = 0; c < 4; ++c) v[c] = load_bf16x16(V + t * kD + 16 * (c0 + c));
#pragma GCC unroll 4
              for (int i = 0; i < 4; ++i) {
                const __m512 p = _mm512_set1_ps(pw[h + i][t]);
#pragma GCC unroll 4
                for (int c = 0; c < 4; ++c) a[i][c] = _mm512_fmadd_ps(p, v[c], a[i][c]);
              }
            }
#pragma GCC unroll 4
            for (int i = 0; i < 4; ++i)
#pragma GCC unroll 4
              for (int c = 0; c < 4; ++c) _mm512_storeu_ps(&out.acc[h + i][16 * (c0 + c)], a[i][c]);
          }
        }
        continue;
      }
      // otherwise two heads at a time with their accumulators in registers
#pragma GCC unroll 4
      for (int h = 0; h < G; h += 2) {
        const bool two = h + 1 < G;
        const __m512 al0 = _mm512_set1_ps(alpha[h]), al1 = _mm512_set1_ps(two ? alpha[h + 1] : 0.f);
        __m512 a0[8], a1[8];
#pragma GCC unroll 8
        for (int c = 0; c < 8; ++c) {
          a0[c] = _mm512_mul_ps(_mm512_loadu_ps(&out.acc[h][16 * c]), al0);
          a1[c] = two ? _mm512_mul_ps(_mm512_loadu_ps(&out.acc[h + 1][16 * c]), al1) : _mm512_setzero_ps();
        }
        for (int t = 0; t < nt; ++t) {
          const __m512 p0 = _mm512_set1_ps(pw[h][t]);
          const __m512 p1 = _mm512_set1_ps(two ? pw[h + 1][t] : 0.f);
#pragma GCC unroll 8
          for (int c = 0; c < 8; ++c) {
            const __m512 v = load_bf16x16(V + t * kD + 16 * c);
            a0[c] = _mm512_fmadd_ps(p0, v, a0[c]);
            a1[c] = _mm512_fmadd_ps(p1, v, a1[c]);
          }
        }
#pragma GCC unroll 8
        for (int c = 0; c < 8; ++c) {
          _mm512_storeu_ps(&out.acc[h][16 * c], a0[c]);
          if (two) _mm512_storeu_ps(&out.acc[h + 1][16 * c], a1[c]);
        }
      }
    }
  }
  // back to the natural-log domain of the Partial contract
  for (int h = 0; h < G; ++h) {
    out.m[h] = m2[h] / l2e;
    out.l[h] = l[h];
  }
}

NEO_BF16_TARGET void task_avx512bf16_dispatch(const Job& jb, int b, int g, int j0, int j1, Partial& out) {
  switch (jb.G) {
    case 1: return task_avx512bf16<1>(jb, b, g, j0, j1, out);
    case 2: return task_avx512bf16<2>(jb, b, g, j0, j1, out);
    case 4: return task_avx512bf16<4>(jb, b, g, j0, j1, out);
    case 8: return task_avx512bf16<8>(jb, b, g, j0, j1, out);
    default: return task_avx512bf16<0>(jb, b, g, j0, j1, out);
  }
}

bool have_avx512bf16() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                         __builtin_cpu_supports("avx512bf16");
  return ok;
}

bool have_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  return ok;
}

struct Segment {  // one task: a maximal run of one (b, g) inside a thread's block range
  int32_t b, g, j0, j1;
  int64_t first_block;  // global block index of j0 (orders the merge)
};

}  // namespace

extern "C" NEO_API neo_status neo_cpu_decode_attn(const neo_kv_pool* pool, int32_t layer, const void* q,
                                                  const int32_t* host_block_table, int32_t max_blocks,
                                                  const int32_t* seq_lens, void* out, int32_t batch,
                                                  int32_t num_q_heads, float scale, int32_t num_threads) {
  if (!pool) return neo::fail(NEO_ERR_INVALID_ARG, "pool is NULL");
  const neo_kv_geometry* geo = neo::pool_geometry(pool);
  if (batch < 0 || layer < 0 || layer >= geo->num_layers) return neo::fail(NEO_ERR_INVALID_ARG, "bad batch or layer");
  if (batch == 0) return NEO_OK;
  if (!q || !host_block_table || !seq_lens || !out || max_blocks < 1)
    return neo::fail(NEO_ERR_INVALID_ARG, "NULL pointer argument");
  const int hkv = geo->num_kv_heads, P = geo->page_size;
  if (num_q_heads <= 0 || num_q_heads % hkv) return neo::fail(NEO_ERR_INVALID_ARG, "num_q_heads % num_kv_heads != 0");
  const int G = num_q_heads / hkv;
  if (G > kMaxG || P > 64) return neo::fail(NEO_ERR_UNSUPPORTED, "G <= 16 and page_size <= 64 required");
  if (!(scale > 0.f) || !std::isfinite(scale)) return neo::fail(NEO_ERR_INVALID_ARG, "scale must be finite and > 0");
  const uint8_t* host = neo::pool_host_base(pool);
  if (!host || geo->num_host_pages < 1) return neo::fail(NEO_ERR_INVALID_ARG, "pool has no CPU-cache");
  // validate metadata (host memory: cheap) and count blocks per (b, g)
  std::vector<int64_t> first(static_cast<size_t>(batch) + 1, 0);
  for (int32_t b = 0; b < batch; ++b) {
    const int32_t n = seq_lens[b];
    if (n < 0 || static_cast<int64_t>(n) > static_cast<int64_t>(max_blocks) * P)
      return neo::fail(NEO_ERR_INVALID_ARG, "seq_lens[" + std::to_string(b) + "] out of range");
    const int32_t np = (n + P - 1) / P;
    for (int32_t j = 0; j < np; ++j) {
      const int32_t id = host_block_table[static_cast<int64_t>(b) * max_blocks + j];
      if (id < 0 || id >= geo->num_host_pages)
        return neo::fail(NEO_ERR_INVALID_ARG, "host block id out of range at request " + std::to_string(b));
    }
    first[b + 1] = first[b] + static_cast<int64_t>(np) * hkv;
  }
  const int64_t total = first[batch];
  Job jb{host, static_cast<int64_t>(hkv) * P * kD, geo->num_layers, layer, hkv, P, G, num_q_heads,
         static_cast<const uint16_t*>(q), host_block_table, max_blocks, seq_lens, scale};
  int nth = num_threads > 0 ? num_threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  nth = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nth, std::max<int64_t>(total, 1))));

  // equal contiguous block ranges per thread -> segments (tasks)
  std::vector<std::vector<Segment>> segs(nth);
  for (int t = 0; t < nth; ++t) {
    const int64_t lo = total * t / nth, hi = total * (t + 1) / nth;
    int64_t x = lo;
    int32_t b = static_cast<int32_t>(std::upper_bound(first.begin(), first.end(), lo) - first.begin()) - 1;
    while (x < hi) {
      while (first[b + 1] <= x) ++b;
      const int32_t np = static_cast<int32_t>((first[b + 1] - first[b]) / hkv);
      const int64_t off = x - first[b];
      const int32_t g = static_cast<int32_t>(off / np), j0 = static_cast<int32_t>(off % np);
      const int64_t seg_end = std::min<int64_t>(hi, first[b] + static_cast<int64_t>(g + 1) * np);
      segs[t].push_back(Segment{b, g, j0, static_cast<int32_t>(j0 + (seg_end - x)), x});
      x = seg_end;
    }
  }
  std::vector<std::vector<Partial>> parts(nth);
  // 2 = AVX-512 BF16, 1 = AVX-512F, 0 = portable; NEO_CPU_PATH=0|1|2 caps it (tests)
  int path = (P % 16 == 0 && have_avx512bf16()) ? 2 : have_avx512() ? 1 : 0;
  if (const char* v = std::getenv("NEO_CPU_PATH")) path = std::min(path, std::atoi(v));
  auto worker = [&](int t) {
    parts[t].resize(segs[t].size());
    for (size_t i = 0; i < segs[t].size(); ++i) {
      const Segment& sg = segs[t][i];
      if (path == 2) task_avx512bf16_dispatch(jb, sg.b, sg.g, sg.j0, sg.j1, parts[t][i]);
      else if (path == 1) task_avx512(jb, sg.b, sg.g, sg.j0, sg.j1, parts[t][i]);
      else task_generic(jb, sg.b, sg.g, sg.j0, sg.j1, parts[t][i]);
    }
  };
  WorkerPool::get().run(nth, worker);

  // merge the partials of each (b, g) in block order (threads are in block order)
  uint16_t* o = static_cast<uint16_t*>(out);
  std::vector<const Partial*> plist;
  std::vector<const Segment*> slist;
  for (int t = 0; t < nth; ++t)
    for (size_t i = 0; i < segs[t].size(); ++i) {
      plist.push_back(&parts[t][i]);
      slist.push_back(&segs[t][i]);
    }
  size_t i = 0;
  std::vector<uint8_t> done(static_cast<size_t>(batch) * hkv, 0);
  while (i < slist.size()) {
    const int32_t b = slist[i]->b, g = slist[i]->g;
    size_t k = i;
    while (k < slist.size() && slist[k]->b == b && slist[k]->g == g) ++k;
    for (int h = 0; h < G; ++h) {
      float M = -INFINITY;
      for (size_t u = i; u < k; ++u) M = std::max(M, plist[u]->m[h]);
      float L = 0.f, acc[kD] = {0.f};
      for (size_t u = i; u < k; ++u) {
        const float w = std::exp(plist[u]->m[h] - M);
        L += plist[u]->l[h] * w;
        for (int d = 0; d < kD; ++d) acc[d] += plist[u]->acc[h][d] * w;
      }
      uint16_t* dst = o + (static_cast<int64_t>(b) * num_q_heads + g * G + h) * kD;
      for (int d = 0; d < kD; ++d) dst[d] = f32_to_bf16(acc[d] / L);
    }
    done[static_cast<size_t>(b) * hkv + g] = 1;
    i = k;
  }
  // empty contexts: zero rows (DESIGN reading c4)
  for (int32_t b = 0; b < batch; ++b)
    for (int g = 0; g < hkv; ++g)
      if (!done[static_cast<size_t>(b) * hkv + g])
        std::memset(o + (static_cast<int64_t>(b) * num_q_heads + g * G) * kD, 0, sizeof(uint16_t) * G * kD);
  return NEO_OK;
}
