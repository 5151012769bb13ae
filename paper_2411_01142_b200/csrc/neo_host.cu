// Host side of libneo: the C ABI of include/neo.h -- argument validation,
// the two-pool page allocator (P:234-235 GPU-cache / CPU-cache; S:231-310
// kv_pool semantics: all-or-nothing, conservation, residency), the TMA
// tensor-map cache for the attention kernel, and swap orchestration
// (gather kernel + cudaMemcpy2DAsync over PCIe).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "neo_internal.cuh"

namespace neo {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

neo_status fail(neo_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

neo_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return NEO_ERR_CUDA;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static bool debug_validate_enabled() {
  const char* v = std::getenv("NEO_DEBUG_VALIDATE");
  return v && v[0] == '1';
}

// ----------------------------------------------------------------- tensor maps
namespace {

enum TmKind : int32_t { kTmDecodeKV = 0, kTmPrefillKV = 1, kTmPrefillQ = 2, kTmPrefillOut = 3 };

struct TmKey {
  const void* ptr;
  int64_t page_stride, num_pages;
  int32_t hkv, page_size, kind;
  bool operator==(const TmKey& o) const {
    return ptr == o.ptr && page_stride == o.page_stride && num_pages == o.num_pages && hkv == o.hkv &&
           page_size == o.page_size && kind == o.kind;
  }
};
struct TmKeyHash {
  size_t operator()(const TmKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<int64_t>()(k.page_stride) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h ^= std::hash<int64_t>()(k.num_pages) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h ^= std::hash<int64_t>()((static_cast<int64_t>(k.hkv) << 32) | k.page_size) + (h << 6) + (h >> 2);
    h ^= std::hash<int32_t>()(k.kind) + (h << 6) + (h >> 2);
    return h;
  }
};

std::mutex g_tm_mu;
std::unordered_map<TmKey, CUtensorMap, TmKeyHash> g_tm_cache;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

neo_status get_encoder() {
  if (g_encode) return NEO_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(NEO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return NEO_OK;
}

neo_status encode_cached(const TmKey& key, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                         const cuuint32_t* box, CUtensorMap* out) {
  std::lock_guard<std::mutex> lk(g_tm_mu);
  auto it = g_tm_cache.find(key);
  if (it != g_tm_cache.end()) {
    *out = it->second;
    return NEO_OK;
  }
  neo_status st = get_encoder();
  if (st != NEO_OK) return st;
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof tm);
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(key.ptr), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NEO_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  if (g_tm_cache.size() > 4096) g_tm_cache.clear();
  g_tm_cache.emplace(key, tm);
  *out = tm;
  return NEO_OK;
}

}  // namespace

// View of a layer's K (or V) pages as a 5-D tensor {64 el, 2 halves, P tokens,
// Hkv heads, num_pages} with box {64, 2, 16, 1, 1}: one TMA load = one 16-token
// tile (4 KiB) of one (page, kv-head), written to shared memory 128B-swizzled.
neo_status tensor_map(const void* ptr, int64_t page_stride, int64_t num_pages, int32_t hkv, int32_t P,
                      CUtensorMap* out) {
  const cuuint64_t dims[5] = {64, 2, static_cast<cuuint64_t>(P), static_cast<cuuint64_t>(hkv),
                              static_cast<cuuint64_t>(num_pages)};
  const cuuint64_t strides[4] = {128, 256, static_cast<cuuint64_t>(P) * 256,
                                 static_cast<cuuint64_t>(page_stride) * 2};
  const cuuint32_t box[5] = {64, 2, 16, 1, 1};
  return encode_cached(TmKey{ptr, page_stride, num_pages, hkv, P, kTmDecodeKV}, 5, dims, strides, box, out);
}

// Prefill view of the same pages: {64 el, P tokens, 2 halves, Hkv, num_pages}
// with box {64, 16, 1, 1, 1}: one TMA load = one dim-half of 16 tokens (2 KiB),
// landing as 16 rows of 128 B -- the canonical SW128 operand layout of tcgen05.
neo_status tensor_map_prefill_kv(const void* ptr, int64_t page_stride, int64_t num_pages, int32_t hkv, int32_t P,
                                 CUtensorMap* out) {
  const cuuint64_t dims[5] = {64, static_cast<cuuint64_t>(P), 2, static_cast<cuuint64_t>(hkv),
                              static_cast<cuuint64_t>(num_pages)};
  const cuuint64_t strides[4] = {256, 128, static_cast<cuuint64_t>(P) * 256, static_cast<cuuint64_t>(page_stride) * 2};
  const cuuint32_t box[5] = {64, 16, 1, 1, 1};
  return encode_cached(TmKey{ptr, page_stride, num_pages, hkv, P, kTmPrefillKV}, 5, dims, strides, box, out);
}

// Packed prefill queries q[T][Hq][128] as {64 el, Hq, T, 2 halves} with box
// {64, G, 128 / G, 1}: one load = one dim-half of a 128-row M tile whose row
// r = (token r / G, head r % G of the kv group), rows of 128 B.
neo_status tensor_map_prefill_q(const void* ptr, int32_t total_tokens, int32_t hq, int32_t G, CUtensorMap* out) {
  const cuuint64_t dims[4] = {64, static_cast<cuuint64_t>(hq), static_cast<cuuint64_t>(total_tokens), 2};
  const cuuint64_t strides[3] = {256, static_cast<cuuint64_t>(hq) * 256, 128};
  const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(G), static_cast<cuuint32_t>(128 / G), 1};
  return encode_cached(TmKey{ptr, total_tokens, hq, G, 0, kTmPrefillQ}, 4, dims, strides, box, out);
}

// Prefill output out[T][Hq][128] for TMA tensor stores: {64 el, Hq, T, 2 halves}
// with box {64, G, 1, 1} -- one store = one dim-half of the G rows of one token
// (never past the request's rows), from shared memory in the SW128 layout.
neo_status tensor_map_prefill_out(void* ptr, int32_t total_tokens, int32_t hq, int32_t G, CUtensorMap* out) {
  const cuuint64_t dims[4] = {64, static_cast<cuuint64_t>(hq), static_cast<cuuint64_t>(total_tokens), 2};
  const cuuint64_t strides[3] = {256, static_cast<cuuint64_t>(hq) * 256, 128};
  const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(G), 1, 1};
  return encode_cached(TmKey{ptr, total_tokens, hq, G, 0, kTmPrefillOut}, 4, dims, strides, box, out);
}

namespace {

int32_t default_chunk(int32_t batch, int32_t hkv, int32_t max_seq_len) {
  // Aim for ~3 waves of one-warp units over 148 SMs x 12 resident warps (the
  // (4 warps, 2 stages) kernel at 3 CTAs/SM): the smallest power of two in
  // [64, 512] that does not overshoot that.  Longer chunks mean fewer pipeline
  // ramps and partials; c2-c5 measured best at C = 384-512.
  const double target_units = 3.0 * 148 * 12;
  const double want = static_cast<double>(batch) * hkv * std::max(max_seq_len, 1) / target_units;
  int32_t c = 64;
  while (c < want && c < kDefaultMaxChunk) c *= 2;
  return c;
}

// a0 plan with the request lengths on the host (neo_decode_attn_plan_chunk).
// Replays the hardware's in-order CTA dispatch of the chunk-major grid for one
// candidate C: every resident CTA slot (SMs x CTAs/SM of the default shape)
// takes the next CTA when it frees; a CTA of W units costs a per-unit start-up
// of kPlanUnitOverheadTiles plus the longest of its units in tiles.  Returns
// the predicted tiles per unit time (higher is better).  The overhead was
// fitted to same-box chunk sweeps (profiles/r01_chunk_plan.md): over the c2,
// c2s, c3, c4 (N = 1, 2, 4, 8) and c5 (N = 1, 2, 4, 8) shards its picks reach
// 99.6 % of the best measured chunk on geometric mean, 97.9 % worst case.
constexpr double kPlanUnitOverheadTiles = 6.0;

double plan_score(const std::vector<int32_t>& ntiles, int32_t hkv, int32_t chunk_tiles, int sms) {
  int32_t max_chunks = 1;
  int64_t total = 0;
  for (int32_t t : ntiles) {
    max_chunks = std::max(max_chunks, (t + chunk_tiles - 1) / chunk_tiles);
    total += t;
  }
  const AttnShape sh = default_attn_shape(max_chunks);
  std::vector<double> slot(static_cast<size_t>(sms) * sh.ctas_per_sm, 0.0);   // min-heap of free times
  auto dispatch = [&](int32_t cta_tiles) {
    if (cta_tiles == 0) return;   // CTAs past every request's last chunk exit at once
    std::pop_heap(slot.begin(), slot.end(), std::greater<double>());
    slot.back() += kPlanUnitOverheadTiles + cta_tiles;
    std::push_heap(slot.begin(), slot.end(), std::greater<double>());
  };
  int in_cta = 0;
  int32_t cta_max = 0;
  for (int32_t c = 0; c < max_chunks; ++c) {
    for (int32_t t : ntiles) {
      const int32_t u = std::min(std::max(t - c * chunk_tiles, 0), chunk_tiles);
      if (in_cta == 0 && hkv % sh.warps == 0) {   // whole CTAs of one request (the usual GQA case)
        for (int32_t k = 0; k < hkv / sh.warps; ++k) dispatch(u);
        continue;
      }
      for (int32_t g = 0; g < hkv; ++g) {
        cta_max = std::max(cta_max, u);
        if (++in_cta == sh.warps) {
          dispatch(cta_max);
          in_cta = 0;
          cta_max = 0;
        }
      }
    }
  }
  if (in_cta) dispatch(cta_max);
  const double makespan = *std::max_element(slot.begin(), slot.end());
  return makespan > 0 ? static_cast<double>(total) * hkv / makespan : 0.0;
}

// The grouped kernel in the same replay: CTA (q, b, g) in group-major order
// (request-major from three groups per request on, as launch_decode_attn),
// 3 CTAs per SM, cost = kPlanGroupOverheadTiles + its per-warp tile range, plus
// kPlanGroupMultiTiles when the request has several groups (partial + combine).
// Fitted on the same-box sweep profiles/r01_grouped_sweep.txt (11 shard rows x
// group sizes 4096/2048/1024 and the split chunks): picks reach 99.6 % of the
// best measured choice on geometric mean, 97.3 % worst.
constexpr double kPlanGroupOverheadTiles = 2.0;
constexpr double kPlanGroupMultiTiles = 2.0;

double plan_score_grouped(const std::vector<int32_t>& ntiles, int32_t hkv, int32_t group_tiles, int sms) {
  int32_t max_groups = 1;
  int64_t total = 0;
  for (int32_t t : ntiles) {
    max_groups = std::max(max_groups, (t + group_tiles - 1) / group_tiles);
    total += t;
  }
  std::vector<double> slot(static_cast<size_t>(sms) * 3, 0.0);
  auto dispatch = [&](int32_t t, int32_t q) {
    const int32_t ng = (t + group_tiles - 1) / group_tiles;
    if (q >= ng) return;
    const int32_t tg = (t + ng - 1) / ng;
    const int32_t g0 = q * tg, g1 = std::min(g0 + tg, t);
    const int32_t tw = (g1 - g0 + 3) / 4;
    for (int32_t g = 0; g < hkv; ++g) {
      std::pop_heap(slot.begin(), slot.end(), std::greater<double>());
      slot.back() += kPlanGroupOverheadTiles + tw + (ng > 1 ? kPlanGroupMultiTiles : 0.0);
      std::push_heap(slot.begin(), slot.end(), std::greater<double>());
    }
  };
  if (max_groups >= 3) {   // request-major CTA order (launch_decode_attn)
    for (int32_t t : ntiles)
      for (int32_t q = 0; q < max_groups; ++q) dispatch(t, q);
  } else {
    for (int32_t q = 0; q < max_groups; ++q)
      for (int32_t t : ntiles) dispatch(t, q);
  }
  const double makespan = *std::max_element(slot.begin(), slot.end());
  return makespan > 0 ? static_cast<double>(total) * hkv / makespan : 0.0;
}


neo_status check_chunk(int32_t C, int32_t P) {
  if (C <= 0 || C % kTileTokens != 0 || C % P != 0 || C > kMaxChunkTokens)
    return fail(NEO_ERR_UNSUPPORTED, "chunk_tokens must be a multiple of 16 and of page_size, <= 1024 (got " +
                                         std::to_string(C) + ")");
  return NEO_OK;
}

}  // namespace

int device_sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();   // no device visible (CPU box): plan for a B200
    return 148;
  }
  if ((n = cache[dev & 63].load(std::memory_order_relaxed)) > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    return 148;
  }
  cache[dev & 63].store(n, std::memory_order_relaxed);
  return n;
}

// debug validation: copies device metadata back (synchronous; debug only)
neo_status debug_validate_attn(const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                               int32_t batch, int32_t page_size, int32_t max_seq_len, int64_t num_pages,
                               cudaStream_t stream) {
  std::vector<int32_t> sl(batch), bt(static_cast<size_t>(batch) * max_blocks);
  cudaError_t e = cudaMemcpyAsync(sl.data(), seq_lens, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(bt.data(), block_table, sizeof(int32_t) * bt.size(), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "NEO_DEBUG_VALIDATE copy");
  for (int32_t b = 0; b < batch; ++b) {
    if (sl[b] < 0 || sl[b] > max_seq_len || static_cast<int64_t>(sl[b]) > static_cast<int64_t>(max_blocks) * page_size)
      return fail(NEO_ERR_INVALID_ARG, "seq_lens[" + std::to_string(b) + "] = " + std::to_string(sl[b]) +
                                           " outside [0, min(max_seq_len, max_blocks*P)]");
    const int32_t np = (sl[b] + page_size - 1) / page_size;
    for (int32_t j = 0; j < np; ++j) {
      const int32_t id = bt[static_cast<size_t>(b) * max_blocks + j];
      if (id < 0 || id >= num_pages)
        return fail(NEO_ERR_INVALID_ARG, "block_table[" + std::to_string(b) + "][" + std::to_string(j) +
                                             "] = " + std::to_string(id) + " outside [0, num_pages)");
    }
  }
  return NEO_OK;
}

// q_offsets [batch + 1]: 0 = q_offsets[0] <= ... <= q_offsets[batch] = total, and
// each request's new tokens fit its context (q_len_b <= seq_lens[b]) and the
// call's max_q_len (the prefill schedule is sized by it).
neo_status debug_validate_offsets(const int32_t* q_offsets, const int32_t* seq_lens, int32_t batch, int32_t total,
                                  int32_t max_q_len, cudaStream_t stream) {
  std::vector<int32_t> off(batch + 1), sl(batch);
  cudaError_t e = cudaMemcpyAsync(off.data(), q_offsets, sizeof(int32_t) * (batch + 1), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(sl.data(), seq_lens, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "NEO_DEBUG_VALIDATE copy");
  if (off[0] != 0 || off[batch] != total) return fail(NEO_ERR_INVALID_ARG, "q_offsets must run from 0 to total_tokens");
  for (int32_t b = 0; b < batch; ++b)
    if (off[b + 1] < off[b] || off[b + 1] - off[b] > sl[b])
      return fail(NEO_ERR_INVALID_ARG, "request " + std::to_string(b) + ": q length negative or above seq_lens");
  for (int32_t b = 0; b < batch; ++b)
    if (off[b + 1] - off[b] > max_q_len)
      return fail(NEO_ERR_INVALID_ARG, "request " + std::to_string(b) + ": q length " +
                                           std::to_string(off[b + 1] - off[b]) + " above max_q_len " +
                                           std::to_string(max_q_len));
  return NEO_OK;
}

}  // namespace neo

// ======================================================================= pool

struct neo_kv_pool {
  neo_kv_geometry geo;
  uint8_t* gpu_base;
  uint8_t* host_base;
  int64_t page_elems;   // Hkv * P * D
  size_t layer_bytes;   // page_elems * 2 (one layer, K or V, one page)
  std::vector<int32_t> gpu_free;      // LIFO stack of free GPU page ids
  std::vector<uint8_t> gpu_used;      // allocated flags
  std::vector<uint8_t> host_used;
  int64_t host_free;
  std::mutex mu;
  // Swap pipeline (created on first staged swap; see swap_common): the staging
  // buffer is used as two halves; gather/scatter kernels run on the caller's
  // stream, PCIe copies on `copy_stream`, and per half `ready` (contents landed)
  // and `free_` (last reader done) events order them.  `next_half` alternates
  // across calls, so call l+1's gather overlaps call l's D2H (P:240 layer-wise
  // swapping issues one call per layer).
  int device = -1;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr};
  cudaEvent_t ev_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_join = nullptr;
  bool half_used[2] = {false, false};
  int next_half = 0;
  ~neo_kv_pool() {
    if (copy_stream) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (device >= 0 && cur != device) cudaSetDevice(device);
      cudaStreamSynchronize(copy_stream);
      for (int h = 0; h < 2; ++h) {
        if (ev_ready[h]) cudaEventDestroy(ev_ready[h]);
        if (ev_free[h]) cudaEventDestroy(ev_free[h]);
      }
      if (ev_start) cudaEventDestroy(ev_start);
      if (ev_join) cudaEventDestroy(ev_join);
      cudaStreamDestroy(copy_stream);
      if (device >= 0 && cur >= 0 && cur != device) cudaSetDevice(cur);
    }
  }
};

using neo::fail;

namespace neo {
const neo_kv_geometry* pool_geometry(const neo_kv_pool* p) { return &p->geo; }
const uint8_t* pool_host_base(const neo_kv_pool* p) { return p->host_base; }
}  // namespace neo

static neo_status check_geo(const neo_kv_geometry* g) {
  if (!g) return fail(NEO_ERR_INVALID_ARG, "geometry is NULL");
  if (g->num_layers < 1 || g->num_kv_heads < 1 || g->num_gpu_pages < 0 || g->num_host_pages < 0)
    return fail(NEO_ERR_INVALID_ARG, "geometry: layers/heads must be >= 1, page counts >= 0");
  if (g->num_gpu_pages > INT32_MAX || g->num_host_pages > INT32_MAX)
    return fail(NEO_ERR_INVALID_ARG, "geometry: page counts must fit int32 ids");
  if (g->head_dim != neo::kHeadDim) return fail(NEO_ERR_UNSUPPORTED, "head_dim must be 128");
  if (g->page_size < 16 || g->page_size % 16 != 0) return fail(NEO_ERR_UNSUPPORTED, "page_size must be a multiple of 16");
  return NEO_OK;
}

extern "C" {

NEO_API const char* neo_last_error(void) { return neo::g_err.c_str(); }
NEO_API const char* neo_version(void) { return "neo-b200 0.1 (sm_100a)"; }

NEO_API neo_status neo_kv_pool_bytes(const neo_kv_geometry* geo, size_t* gpu_bytes, size_t* host_bytes) {
  neo_status st = check_geo(geo);
  if (st != NEO_OK) return st;
  const size_t page = static_cast<size_t>(geo->num_kv_heads) * geo->page_size * geo->head_dim * 2;
  const size_t per_layer_pair = 2 * page;
  if (gpu_bytes) *gpu_bytes = per_layer_pair * geo->num_layers * static_cast<size_t>(geo->num_gpu_pages);
  if (host_bytes) *host_bytes = per_layer_pair * geo->num_layers * static_cast<size_t>(geo->num_host_pages);
  return NEO_OK;
}

NEO_API neo_status neo_kv_pool_create(const neo_kv_geometry* geo, void* gpu_kv_base, size_t gpu_bytes,
                                      void* host_kv_base, size_t host_bytes, neo_kv_pool** out) {
  if (!out) return fail(NEO_ERR_INVALID_ARG, "out is NULL");
  size_t need_gpu = 0, need_host = 0;
  neo_status st = neo_kv_pool_bytes(geo, &need_gpu, &need_host);
  if (st != NEO_OK) return st;
  if (geo->num_gpu_pages > 0 && (!gpu_kv_base || !neo::aligned16(gpu_kv_base)))
    return fail(NEO_ERR_INVALID_ARG, "gpu_kv_base must be a non-NULL 16-byte aligned device pointer");
  if (geo->num_host_pages > 0 && (!host_kv_base || !neo::aligned16(host_kv_base)))
    return fail(NEO_ERR_INVALID_ARG, "host_kv_base must be a non-NULL 16-byte aligned pinned pointer");
  if (gpu_bytes < need_gpu) return fail(NEO_ERR_INVALID_ARG, "gpu_bytes smaller than neo_kv_pool_bytes()");
  if (host_bytes < need_host) return fail(NEO_ERR_INVALID_ARG, "host_bytes smaller than neo_kv_pool_bytes()");
  neo_kv_pool* p = new (std::nothrow) neo_kv_pool();
  if (!p) return fail(NEO_ERR_INTERNAL, "out of host memory");
  p->geo = *geo;
  p->gpu_base = static_cast<uint8_t*>(gpu_kv_base);
  p->host_base = static_cast<uint8_t*>(host_kv_base);
  p->page_elems = static_cast<int64_t>(geo->num_kv_heads) * geo->page_size * geo->head_dim;
  p->layer_bytes = static_cast<size_t>(p->page_elems) * 2;
  try {
    p->gpu_free.resize(geo->num_gpu_pages);
    for (int64_t i = 0; i < geo->num_gpu_pages; ++i)
      p->gpu_free[i] = static_cast<int32_t>(geo->num_gpu_pages - 1 - i);  // pop_back yields 0, 1, 2, ...
    p->gpu_used.assign(geo->num_gpu_pages, 0);
    p->host_used.assign(geo->num_host_pages, 0);
  } catch (...) {
    delete p;
    return fail(NEO_ERR_INTERNAL, "out of host memory");
  }
  p->host_free = geo->num_host_pages;
  *out = p;
  return NEO_OK;
}

NEO_API void neo_kv_pool_destroy(neo_kv_pool* pool) { delete pool; }

NEO_API neo_status neo_kv_alloc(neo_kv_pool* pool, int32_t where, int32_t n, int32_t* ids) {
  if (!pool) return fail(NEO_ERR_INVALID_ARG, "pool is NULL");
  if (where != NEO_GPU && where != NEO_HOST) return fail(NEO_ERR_INVALID_ARG, "where must be NEO_GPU or NEO_HOST");
  if (n < 0) return fail(NEO_ERR_INVALID_ARG, "n_pages < 0");
  if (n == 0) return NEO_OK;
  if (!ids) return fail(NEO_ERR_INVALID_ARG, "page_ids_out is NULL");
  std::lock_guard<std::mutex> lk(pool->mu);
  if (where == NEO_GPU) {
    if (static_cast<int64_t>(pool->gpu_free.size()) < n)
      return fail(NEO_ERR_OUT_OF_PAGES, "GPU-cache has " + std::to_string(pool->gpu_free.size()) +
                                            " free pages, need " + std::to_string(n));
    for (int32_t i = 0; i < n; ++i) {
      ids[i] = pool->gpu_free.back();
      pool->gpu_free.pop_back();
      pool->gpu_used[ids[i]] = 1;
    }
    return NEO_OK;
  }
  if (pool->host_free < n)
    return fail(NEO_ERR_OUT_OF_PAGES, "CPU-cache has " + std::to_string(pool->host_free) + " free pages, need " +
                                          std::to_string(n));
  // first fit: one contiguous ascending run if possible, else the lowest free ids
  const int64_t N = pool->geo.num_host_pages;
  int64_t run = 0, start = -1;
  for (int64_t i = 0; i < N; ++i) {
    run = pool->host_used[i] ? 0 : run + 1;
    if (run == n) {
      start = i - n + 1;
      break;
    }
  }
  if (start >= 0) {
    for (int32_t i = 0; i < n; ++i) ids[i] = static_cast<int32_t>(start + i);
  } else {
    int32_t k = 0;
    for (int64_t i = 0; i < N && k < n; ++i)
      if (!pool->host_used[i]) ids[k++] = static_cast<int32_t>(i);
  }
  for (int32_t i = 0; i < n; ++i) pool->host_used[ids[i]] = 1;
  pool->host_free -= n;
  return NEO_OK;
}

static neo_status check_ids(const std::vector<uint8_t>& used, int32_t n, const int32_t* ids, const char* what) {
  std::vector<int32_t> seen;
  seen.reserve(n);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t id = ids[i];
    if (id < 0 || id >= static_cast<int64_t>(used.size()) || !used[id])
      return fail(NEO_ERR_INVALID_ARG, std::string(what) + " id " + std::to_string(id) + " is not allocated");
    seen.push_back(id);
  }
  std::sort(seen.begin(), seen.end());
  if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
    return fail(NEO_ERR_INVALID_ARG, std::string(what) + " ids contain duplicates");
  return NEO_OK;
}

NEO_API neo_status neo_kv_free(neo_kv_pool* pool, int32_t where, int32_t n, const int32_t* ids) {
  if (!pool) return fail(NEO_ERR_INVALID_ARG, "pool is NULL");
  if (where != NEO_GPU && where != NEO_HOST) return fail(NEO_ERR_INVALID_ARG, "where must be NEO_GPU or NEO_HOST");
  if (n < 0) return fail(NEO_ERR_INVALID_ARG, "n_pages < 0");
  if (n == 0) return NEO_OK;
  if (!ids) return fail(NEO_ERR_INVALID_ARG, "page_ids is NULL");
  std::lock_guard<std::mutex> lk(pool->mu);
  std::vector<uint8_t>& used = where == NEO_GPU ? pool->gpu_used : pool->host_used;
  neo_status st = check_ids(used, n, ids, where == NEO_GPU ? "GPU page" : "host page");
  if (st != NEO_OK) return st;
  for (int32_t i = 0; i < n; ++i) {
    used[ids[i]] = 0;
    if (where == NEO_GPU) pool->gpu_free.push_back(ids[i]);
  }
  if (where == NEO_HOST) pool->host_free += n;
  return NEO_OK;
}

NEO_API neo_status neo_kv_free_count(const neo_kv_pool* pool, int32_t where, int64_t* n_free) {
  if (!pool || !n_free) return fail(NEO_ERR_INVALID_ARG, "NULL argument");
  if (where == NEO_GPU) *n_free = static_cast<int64_t>(pool->gpu_free.size());
  else if (where == NEO_HOST) *n_free = pool->host_free;
  else return fail(NEO_ERR_INVALID_ARG, "where must be NEO_GPU or NEO_HOST");
  return NEO_OK;
}

NEO_API neo_status neo_kv_layer_view(const neo_kv_pool* pool, int32_t layer, void** k, void** v, int64_t* stride) {
  if (!pool || !k || !v || !stride) return fail(NEO_ERR_INVALID_ARG, "NULL argument");
  if (layer < 0 || layer >= pool->geo.num_layers) return fail(NEO_ERR_INVALID_ARG, "layer out of range");
  const size_t kv_bytes = pool->layer_bytes * static_cast<size_t>(pool->geo.num_gpu_pages);
  *k = pool->gpu_base + (static_cast<size_t>(layer) * 2 + 0) * kv_bytes;
  *v = pool->gpu_base + (static_cast<size_t>(layer) * 2 + 1) * kv_bytes;
  *stride = pool->page_elems;
  return NEO_OK;
}

// ============================================================ decode attention

NEO_API int32_t neo_decode_attn_default_chunk(int32_t batch, int32_t hkv, int32_t max_seq_len) {
  return neo::default_chunk(batch, hkv, max_seq_len);
}

NEO_API neo_status neo_decode_attn_plan_chunk(const int32_t* seq_lens, int32_t batch, int32_t hkv, int32_t page_size,
                                              int32_t* chunk_tokens) {
  if (!chunk_tokens) return neo::fail(NEO_ERR_INVALID_ARG, "chunk_tokens is NULL");
  if (batch < 0 || hkv <= 0 || (batch > 0 && !seq_lens))
    return neo::fail(NEO_ERR_INVALID_ARG, "batch >= 0, num_kv_heads >= 1 and seq_lens (host) required");
  if (page_size <= 0 || page_size % neo::kTileTokens || page_size > neo::kMaxChunkTokens)
    return neo::fail(NEO_ERR_UNSUPPORTED, "page_size must be a positive multiple of 16, <= 1024");
  std::vector<int32_t> ntiles(static_cast<size_t>(batch));
  for (int32_t b = 0; b < batch; ++b) {
    if (seq_lens[b] < 0) return neo::fail(NEO_ERR_INVALID_ARG, "seq_lens[" + std::to_string(b) + "] < 0");
    ntiles[b] = (seq_lens[b] + neo::kTileTokens - 1) / neo::kTileTokens;
  }
  const int sms = neo::device_sm_count();
  // candidates (largest first), those that are multiples of P: the sizes the
  // same-box sweeps resolved (profiles/r01_chunk_plan.md); finer steps only let the
  // model's error pick worse neighbours
  static const int32_t kCand[] = {1024, 640, 512, 448, 384, 320, 256};
  std::vector<int32_t> cand;
  for (int32_t C : kCand)
    if (C % page_size == 0) cand.push_back(C);
  if (cand.empty()) cand.push_back(page_size);
  // Under one wave at the smallest candidate the call is latency-bound: requests
  // that fit one 4096-token group take the grouped kernel (no partials, no
  // combine round trips: c1 12.6 -> 10.2 us); otherwise the shape-only default.
  const int32_t ct_min = cand.back() / neo::kTileTokens;
  int64_t units_min = 0;
  for (int32_t t : ntiles) units_min += static_cast<int64_t>(hkv) * ((t + ct_min - 1) / ct_min);
  if (units_min < static_cast<int64_t>(sms) * 2 * 4) {
    int32_t max_len = 0;
    for (int32_t b = 0; b < batch; ++b) max_len = std::max(max_len, seq_lens[b]);
    if (max_len > 0 && max_len <= neo::kGroupTiles * neo::kTileTokens) {
      *chunk_tokens = NEO_CHUNK_GROUPED;
      return NEO_OK;
    }
    int32_t C = neo::default_chunk(batch, hkv, max_len);
    if (C % page_size) C = page_size * ((C + page_size - 1) / page_size);
    *chunk_tokens = std::min(C, neo::kMaxChunkTokens);
    return NEO_OK;
  }
  const int32_t ct_max = cand.front() / neo::kTileTokens;
  int64_t units = 0;
  int32_t max_chunks = 1;
  for (int32_t t : ntiles) {
    units += static_cast<int64_t>(hkv) * ((t + ct_max - 1) / ct_max);
    max_chunks = std::max(max_chunks, (t + ct_max - 1) / ct_max);
  }
  const neo::AttnShape sh = neo::default_attn_shape(max_chunks);
  const double waves = static_cast<double>(units) / (static_cast<double>(sms) * sh.ctas_per_sm * sh.warps);
  int32_t best = cand.front();
  double best_score = -1.0;
  if (waves >= 16.0) {   // many waves: the tail is amortised and the longest chunk wins (c5 sweeps)
    best_score = neo::plan_score(ntiles, hkv, ct_max, sms);
  } else {
    for (int32_t C : cand) {        // largest first: a smaller C must win by > 1 %
      const double sc = neo::plan_score(ntiles, hkv, C / neo::kTileTokens, sms);
      if (sc > best_score * 1.01) {
        best = C;
        best_score = sc;
      }
    }
  }
  // the grouped kernel (groups of 4096 ... 1024 tokens, largest first) must beat
  // the best split chunk -- and a smaller group the larger one -- by > 1 %
  double best_g = -1.0;
  int32_t best_t = 0;
  for (int32_t T : {4096, 3072, 2048, 1536, 1024}) {
    const double sc = neo::plan_score_grouped(ntiles, hkv, T / neo::kTileTokens, sms);
    if (sc > best_g * 1.01) best_g = sc, best_t = T;
  }
  // the legacy codes for the power-of-two group sizes (-1, -2, -4), -T otherwise
  const int32_t gcode = best_t == 4096 ? -1 : best_t == 2048 ? -2 : best_t == 1024 ? -4 : -best_t;
  *chunk_tokens = best_g > best_score * 1.01 ? gcode : best;
  return NEO_OK;
}

static neo_status attn_shape(int32_t batch, int32_t hq, int32_t hkv, int32_t d, int32_t max_seq_len,
                             int32_t* chunk_tokens, int32_t page_size) {
  if (batch < 0 || hq <= 0 || hkv <= 0 || max_seq_len < 0)
    return fail(NEO_ERR_INVALID_ARG, "batch >= 0, heads >= 1 and max_seq_len >= 0 required");
  if (hq % hkv != 0) return fail(NEO_ERR_INVALID_ARG, "num_q_heads must be a multiple of num_kv_heads");
  if (d != neo::kHeadDim) return fail(NEO_ERR_UNSUPPORTED, "head_dim must be 128");
  if (hq / hkv > neo::kMaxGroup) return fail(NEO_ERR_UNSUPPORTED, "GQA group size G = Hq/Hkv must be <= 8");
  if (neo::is_grouped_chunk(*chunk_tokens)) return NEO_OK;
  if (*chunk_tokens == 0) {
    *chunk_tokens = neo::default_chunk(batch, hkv, max_seq_len);
    if (page_size > 0 && *chunk_tokens % page_size) *chunk_tokens = page_size * ((*chunk_tokens + page_size - 1) / page_size);
  }
  return neo::check_chunk(*chunk_tokens, page_size > 0 ? page_size : 16);
}

NEO_API neo_status neo_decode_attn_workspace_bytes(int32_t batch, int32_t hq, int32_t hkv, int32_t d,
                                                   int32_t max_seq_len, int32_t chunk_tokens, size_t* bytes) {
  if (!bytes) return fail(NEO_ERR_INVALID_ARG, "bytes is NULL");
  neo_status st = attn_shape(batch, hq, hkv, d, max_seq_len, &chunk_tokens, 16);
  if (st != NEO_OK) return st;
  const int32_t max_chunks = neo::is_grouped_chunk(chunk_tokens)
                                 ? neo::max_groups_for(max_seq_len, neo::group_tiles_of(chunk_tokens))
                                                              : std::max(1, (max_seq_len + chunk_tokens - 1) / chunk_tokens);
  *bytes = neo::workspace_required(batch, hq, hkv, max_chunks);
  return NEO_OK;
}

NEO_API neo_status neo_decode_attn_workspace_init(void* ws, size_t bytes, void* stream) {
  if (!ws || bytes == 0) return fail(NEO_ERR_INVALID_ARG, "workspace is NULL/empty");
  cudaError_t e = cudaMemsetAsync(ws, 0, bytes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? NEO_OK : neo::cuda_fail(e, "cudaMemsetAsync(workspace)");
}

static neo_status decode_attn_impl(const void* q, const void* k_pages, const void* v_pages, int64_t page_stride,
                                   int64_t num_pages, const int32_t* block_table, int32_t max_blocks,
                                   const int32_t* seq_lens, void* out, int32_t batch, int32_t hq, int32_t hkv,
                                   int32_t d, int32_t page_size, int32_t max_seq_len, float scale,
                                   int32_t chunk_tokens, void* workspace, size_t workspace_bytes, void* stream,
                                   const float* inv_freq, const void* k_new, const void* v_new, uint32_t flags = 0) {
  if (flags & ~static_cast<uint32_t>(NEO_ATTN_KV_STABLE)) return fail(NEO_ERR_INVALID_ARG, "unknown attention flags");
  if (page_size < 16 || page_size % 16 != 0) return fail(NEO_ERR_UNSUPPORTED, "page_size must be a multiple of 16");
  neo_status st = attn_shape(batch, hq, hkv, d, max_seq_len, &chunk_tokens, page_size);
  if (st != NEO_OK) return st;
  if (batch == 0) return NEO_OK;
  if (!q || !k_pages || !v_pages || !block_table || !seq_lens || !out || !workspace)
    return fail(NEO_ERR_INVALID_ARG, "NULL pointer argument");
  if (!neo::aligned16(q) || !neo::aligned16(out) || !neo::aligned16(k_pages) || !neo::aligned16(v_pages) ||
      !neo::aligned16(workspace))
    return fail(NEO_ERR_INVALID_ARG, "q, out, k_pages, v_pages and workspace must be 16-byte aligned");
  if (page_stride % 8 != 0 || page_stride < static_cast<int64_t>(hkv) * page_size * d)
    return fail(NEO_ERR_INVALID_ARG, "page_stride must be a multiple of 8 elements and >= Hkv*P*D");
  if (num_pages < 1 || num_pages > (int64_t(1) << 31)) return fail(NEO_ERR_INVALID_ARG, "num_pages out of range");
  if (max_blocks < 1 || static_cast<int64_t>(max_seq_len) > static_cast<int64_t>(max_blocks) * page_size)
    return fail(NEO_ERR_INVALID_ARG, "max_seq_len exceeds max_blocks * page_size");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(NEO_ERR_INVALID_ARG, "scale must be finite and > 0");
  const bool grouped = neo::is_grouped_chunk(chunk_tokens);
  const int32_t max_chunks = grouped ? neo::max_groups_for(max_seq_len, neo::group_tiles_of(chunk_tokens))
                                     : std::max(1, (max_seq_len + chunk_tokens - 1) / chunk_tokens);
  if (!neo::workspace_layout(batch, hq, hkv, max_chunks, workspace_bytes).fits)
    return fail(NEO_ERR_INVALID_ARG, "workspace too small: need " +
                                         std::to_string(neo::workspace_required(batch, hq, hkv, max_chunks)) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (neo::debug_validate_enabled()) {
    st = neo::debug_validate_attn(block_table, max_blocks, seq_lens, batch, page_size, max_seq_len, num_pages, s);
    if (st != NEO_OK) return st;
  }
  CUtensorMap tmk, tmv;
  st = neo::tensor_map(k_pages, page_stride, num_pages, hkv, page_size, &tmk);
  if (st != NEO_OK) return st;
  st = neo::tensor_map(v_pages, page_stride, num_pages, hkv, page_size, &tmv);
  if (st != NEO_OK) return st;
  neo::AttnLaunch L{q, out, block_table, seq_lens, workspace, workspace_bytes, batch, hq, hkv, page_size,
                    max_blocks, chunk_tokens, max_chunks, scale, s};
  L.grouped = grouped;
  L.early = (flags & NEO_ATTN_KV_STABLE) && !k_new;
  if (k_new) {
    L.inv_freq = inv_freq;
    L.k_new = k_new;
    L.v_new = v_new;
    L.k_pages = const_cast<void*>(k_pages);
    L.v_pages = const_cast<void*>(v_pages);
    L.page_stride = page_stride;
  }
  return neo::launch_decode_attn(L, tmk, tmv);
}

NEO_API neo_status neo_decode_attn(const void* q, const void* k_pages, const void* v_pages, int64_t page_stride,
                                   int64_t num_pages, const int32_t* block_table, int32_t max_blocks,
                                   const int32_t* seq_lens, void* out, int32_t batch, int32_t hq, int32_t hkv,
                                   int32_t d, int32_t page_size, int32_t max_seq_len, float scale,
                                   int32_t chunk_tokens, void* workspace, size_t workspace_bytes, void* stream) {
  return decode_attn_impl(q, k_pages, v_pages, page_stride, num_pages, block_table, max_blocks, seq_lens, out, batch,
                          hq, hkv, d, page_size, max_seq_len, scale, chunk_tokens, workspace, workspace_bytes, stream,
                          nullptr, nullptr, nullptr);
}

NEO_API neo_status neo_decode_attn_ex(const void* q, const void* k_pages, const void* v_pages, int64_t page_stride,
                                      int64_t num_pages, const int32_t* block_table, int32_t max_blocks,
                                      const int32_t* seq_lens, void* out, int32_t batch, int32_t hq, int32_t hkv,
                                      int32_t d, int32_t page_size, int32_t max_seq_len, float scale,
                                      int32_t chunk_tokens, void* workspace, size_t workspace_bytes, uint32_t flags,
                                      void* stream) {
  return decode_attn_impl(q, k_pages, v_pages, page_stride, num_pages, block_table, max_blocks, seq_lens, out, batch,
                          hq, hkv, d, page_size, max_seq_len, scale, chunk_tokens, workspace, workspace_bytes, stream,
                          nullptr, nullptr, nullptr, flags);
}

NEO_API neo_status neo_decode_attn_append(const void* q, const float* inv_freq, const void* k_new, const void* v_new,
                                          void* k_pages, void* v_pages, int64_t page_stride, int64_t num_pages,
                                          const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                                          void* out, int32_t batch, int32_t hq, int32_t hkv, int32_t d,
                                          int32_t page_size, int32_t max_seq_len, float scale, int32_t chunk_tokens,
                                          void* workspace, size_t workspace_bytes, void* stream) {
  if (batch > 0 && (!k_new || !v_new)) return fail(NEO_ERR_INVALID_ARG, "NULL k_new / v_new");
  if (batch > 0 && (!neo::aligned16(k_new) || !neo::aligned16(v_new)))
    return fail(NEO_ERR_INVALID_ARG, "k_new / v_new must be 16-byte aligned");
  return decode_attn_impl(q, k_pages, v_pages, page_stride, num_pages, block_table, max_blocks, seq_lens, out, batch,
                          hq, hkv, d, page_size, max_seq_len, scale, chunk_tokens, workspace, workspace_bytes, stream,
                          inv_freq, k_new, v_new);
}

NEO_API neo_status neo_prefill_attn(const void* q, const void* k_pages, const void* v_pages, int64_t page_stride,
                                    int64_t num_pages, const int32_t* block_table, int32_t max_blocks,
                                    const int32_t* seq_lens, const int32_t* q_offsets, void* out, int32_t batch,
                                    int32_t total_tokens, int32_t hq, int32_t hkv, int32_t d, int32_t page_size,
                                    int32_t max_q_len, float scale, void* stream) {
  if (d != neo::kHeadDim) return fail(NEO_ERR_UNSUPPORTED, "head_dim must be 128");
  if (page_size < 16 || page_size % 16 != 0) return fail(NEO_ERR_UNSUPPORTED, "page_size must be a multiple of 16");
  if (batch < 0 || total_tokens < 0 || hq < 1 || hkv < 1 || hq % hkv)
    return fail(NEO_ERR_INVALID_ARG, "batch, total_tokens >= 0 and num_q_heads a multiple of num_kv_heads required");
  const int32_t G = hq / hkv;
  if (G > 16 || (G & (G - 1))) return fail(NEO_ERR_UNSUPPORTED, "G = Hq / Hkv must be 1, 2, 4, 8 or 16");
  if (batch == 0 || total_tokens == 0) return NEO_OK;
  if (batch > 512 || static_cast<int64_t>(max_q_len) * G > 262144)
    return fail(NEO_ERR_UNSUPPORTED, "prefill: batch <= 512 and max_q_len * G <= 262144 per call");
  if (!q || !k_pages || !v_pages || !block_table || !seq_lens || !q_offsets || !out)
    return fail(NEO_ERR_INVALID_ARG, "NULL pointer argument");
  if (!neo::aligned16(q) || !neo::aligned16(k_pages) || !neo::aligned16(v_pages) ||
      (reinterpret_cast<uintptr_t>(out) & 31u))
    return fail(NEO_ERR_INVALID_ARG, "q and pages must be 16-byte aligned, out 32-byte aligned");
  if (page_stride % 8 != 0 || page_stride < static_cast<int64_t>(hkv) * page_size * d)
    return fail(NEO_ERR_INVALID_ARG, "page_stride must be a multiple of 8 elements and >= Hkv*P*D");
  if (num_pages < 1 || max_blocks < 1 || max_q_len < 1)
    return fail(NEO_ERR_INVALID_ARG, "num_pages, max_blocks and max_q_len must be >= 1");
  if (!(scale > 0.f) || !std::isfinite(scale)) return fail(NEO_ERR_INVALID_ARG, "scale must be finite and > 0");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  neo_status st;
  if (neo::debug_validate_enabled()) {
    st = neo::debug_validate_attn(block_table, max_blocks, seq_lens, batch, page_size, max_blocks * page_size,
                                  num_pages, s);
    if (st != NEO_OK) return st;
    st = neo::debug_validate_offsets(q_offsets, seq_lens, batch, total_tokens, max_q_len, s);
    if (st != NEO_OK) return st;
  }
  CUtensorMap tmq, tmk, tmv;
  st = neo::tensor_map_prefill_q(q, total_tokens, hq, G, &tmq);
  if (st != NEO_OK) return st;
  st = neo::tensor_map_prefill_kv(k_pages, page_stride, num_pages, hkv, page_size, &tmk);
  if (st != NEO_OK) return st;
  st = neo::tensor_map_prefill_kv(v_pages, page_stride, num_pages, hkv, page_size, &tmv);
  if (st != NEO_OK) return st;
  const char* cap = std::getenv("NEO_PREFILL_CTAS");       // experiment knob: SM budget of the prefill grid
  CUtensorMap tmo;
  st = neo::tensor_map_prefill_out(out, total_tokens, hq, G, &tmo);
  if (st != NEO_OK) return st;
  neo::PrefillLaunch L{out, block_table, seq_lens, q_offsets, batch, hq, hkv, page_size, max_blocks, max_q_len, scale,
                       s, cap ? std::atoi(cap) : 0};
  return neo::launch_prefill_attn(L, tmq, tmk, tmv, tmo);
}

NEO_API neo_status neo_kv_append(void* k_pages, void* v_pages, int64_t page_stride, int64_t num_pages,
                                 const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                                 const void* k_new, const void* v_new, int32_t batch, int32_t hkv, int32_t d,
                                 int32_t page_size, void* stream) {
  if (d != neo::kHeadDim) return fail(NEO_ERR_UNSUPPORTED, "head_dim must be 128");
  if (page_size < 16 || page_size % 16 != 0) return fail(NEO_ERR_UNSUPPORTED, "page_size must be a multiple of 16");
  if (batch < 0 || hkv < 1) return fail(NEO_ERR_INVALID_ARG, "batch >= 0 and num_kv_heads >= 1 required");
  if (batch == 0) return NEO_OK;
  if (!k_pages || !v_pages || !block_table || !seq_lens || !k_new || !v_new)
    return fail(NEO_ERR_INVALID_ARG, "NULL pointer argument");
  if (!neo::aligned16(k_pages) || !neo::aligned16(v_pages) || !neo::aligned16(k_new) || !neo::aligned16(v_new))
    return fail(NEO_ERR_INVALID_ARG, "pages and k_new/v_new must be 16-byte aligned");
  if (page_stride % 8 != 0 || page_stride < static_cast<int64_t>(hkv) * page_size * d)
    return fail(NEO_ERR_INVALID_ARG, "page_stride must be a multiple of 8 elements and >= Hkv*P*D");
  if (num_pages < 1 || max_blocks < 1) return fail(NEO_ERR_INVALID_ARG, "num_pages and max_blocks must be >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (neo::debug_validate_enabled()) {
    neo_status st = neo::debug_validate_attn(block_table, max_blocks, seq_lens, batch, page_size, max_blocks * page_size,
                                             num_pages, s);
    if (st != NEO_OK) return st;
  }
  return neo::launch_append(static_cast<uint16_t*>(k_pages), static_cast<uint16_t*>(v_pages), page_stride, block_table,
                            max_blocks, seq_lens, static_cast<const uint16_t*>(k_new),
                            static_cast<const uint16_t*>(v_new), batch, hkv, page_size, s);
}

namespace {
// argument checks shared by neo_rope_append and neo_prefill_append
neo_status check_rope_store(const void* q, int32_t hq, const float* inv_freq, const void* k_pages,
                            const void* v_pages, int64_t page_stride, int64_t num_pages, const int32_t* block_table,
                            int32_t max_blocks, const int32_t* seq_lens, const void* k_new, const void* v_new,
                            int32_t hkv, int32_t d, int32_t page_size) {
  if (d != neo::kHeadDim) return fail(NEO_ERR_UNSUPPORTED, "head_dim must be 128");
  if (page_size < 16 || page_size % 16 != 0) return fail(NEO_ERR_UNSUPPORTED, "page_size must be a multiple of 16");
  if (hkv < 1) return fail(NEO_ERR_INVALID_ARG, "num_kv_heads >= 1 required");
  if (inv_freq && (hq < 1 || hq % hkv || !q)) return fail(NEO_ERR_INVALID_ARG,
                                                          "RoPE needs q and num_q_heads a multiple of num_kv_heads");
  if (!k_pages || !v_pages || !block_table || !seq_lens || !k_new || !v_new)
    return fail(NEO_ERR_INVALID_ARG, "NULL pointer argument");
  if (!neo::aligned16(k_pages) || !neo::aligned16(v_pages) || !neo::aligned16(k_new) || !neo::aligned16(v_new) ||
      (inv_freq && !neo::aligned16(q)))
    return fail(NEO_ERR_INVALID_ARG, "pages, q and k_new/v_new must be 16-byte aligned");
  if (page_stride % 8 != 0 || page_stride < static_cast<int64_t>(hkv) * page_size * d)
    return fail(NEO_ERR_INVALID_ARG, "page_stride must be a multiple of 8 elements and >= Hkv*P*D");
  if (num_pages < 1 || max_blocks < 1) return fail(NEO_ERR_INVALID_ARG, "num_pages and max_blocks must be >= 1");
  return NEO_OK;
}
}  // namespace

NEO_API neo_status neo_rope_append(void* q_inout, int32_t hq, const float* inv_freq, void* k_pages, void* v_pages,
                                   int64_t page_stride, int64_t num_pages, const int32_t* block_table,
                                   int32_t max_blocks, const int32_t* seq_lens, const void* k_new, const void* v_new,
                                   int32_t batch, int32_t hkv, int32_t d, int32_t page_size, void* stream) {
  if (batch < 0) return fail(NEO_ERR_INVALID_ARG, "batch >= 0 required");
  if (batch == 0) return NEO_OK;
  if (!inv_freq) return fail(NEO_ERR_INVALID_ARG, "NULL inv_freq");
  neo_status st = check_rope_store(q_inout, hq, inv_freq, k_pages, v_pages, page_stride, num_pages, block_table,
                                   max_blocks, seq_lens, k_new, v_new, hkv, d, page_size);
  if (st != NEO_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (neo::debug_validate_enabled()) {
    st = neo::debug_validate_attn(block_table, max_blocks, seq_lens, batch, page_size, max_blocks * page_size,
                                  num_pages, s);
    if (st != NEO_OK) return st;
  }
  return neo::launch_rope_append(static_cast<uint16_t*>(q_inout), hq, inv_freq, static_cast<uint16_t*>(k_pages),
                                 static_cast<uint16_t*>(v_pages), page_stride, block_table, max_blocks, seq_lens,
                                 nullptr, static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new),
                                 batch, batch, hkv, page_size, s);
}

NEO_API neo_status neo_prefill_append(void* q_inout, int32_t hq, const float* inv_freq, void* k_pages,
                                      void* v_pages, int64_t page_stride, int64_t num_pages,
                                      const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                                      const int32_t* q_offsets, const void* k_new, const void* v_new, int32_t batch,
                                      int32_t total_tokens, int32_t hkv, int32_t d, int32_t page_size, void* stream) {
  if (batch < 0 || total_tokens < 0) return fail(NEO_ERR_INVALID_ARG, "batch >= 0 and total_tokens >= 0 required");
  if (batch == 0 || total_tokens == 0) return NEO_OK;
  if (!q_offsets) return fail(NEO_ERR_INVALID_ARG, "NULL q_offsets");
  neo_status st = check_rope_store(q_inout, hq, inv_freq, k_pages, v_pages, page_stride, num_pages, block_table,
                                   max_blocks, seq_lens, k_new, v_new, hkv, d, page_size);
  if (st != NEO_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (neo::debug_validate_enabled()) {
    st = neo::debug_validate_attn(block_table, max_blocks, seq_lens, batch, page_size, max_blocks * page_size,
                                  num_pages, s);
    if (st != NEO_OK) return st;
    st = neo::debug_validate_offsets(q_offsets, seq_lens, batch, total_tokens, INT32_MAX, s);
    if (st != NEO_OK) return st;
  }
  return neo::launch_rope_append(static_cast<uint16_t*>(q_inout), hq, inv_freq, static_cast<uint16_t*>(k_pages),
                                 static_cast<uint16_t*>(v_pages), page_stride, block_table, max_blocks, seq_lens,
                                 q_offsets, static_cast<const uint16_t*>(k_new), static_cast<const uint16_t*>(v_new),
                                 batch, total_tokens, hkv, page_size, s);
}

// ======================================================================= swap

NEO_API neo_status neo_kv_swap_staging_bytes(const neo_kv_pool* pool, int32_t n, int32_t l0, int32_t l1,
                                             size_t* bytes) {
  if (!pool || !bytes) return fail(NEO_ERR_INVALID_ARG, "NULL argument");
  if (n < 0 || l0 < 0 || l1 > pool->geo.num_layers || l0 >= l1)
    return fail(NEO_ERR_INVALID_ARG, "bad page count or layer range");
  *bytes = static_cast<size_t>(n) * (l1 - l0) * 2 * pool->layer_bytes;
  return NEO_OK;
}

// Creates the pool's copy stream and events on the current device (once).
static neo_status ensure_swap_pipeline(neo_kv_pool* pool) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return neo::cuda_fail(e, "cudaGetDevice");
  if (pool->copy_stream) {
    if (dev != pool->device)
      return fail(NEO_ERR_INVALID_ARG, "staged swaps of one pool must run on one device (pool's copy stream is on "
                                       "device " + std::to_string(pool->device) + ")");
    return NEO_OK;
  }
  cudaStream_t cs = nullptr;
  cudaEvent_t ev[6] = {};
  e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  for (int i = 0; i < 6 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    for (int i = 0; i < 6; ++i)
      if (ev[i]) cudaEventDestroy(ev[i]);
    if (cs) cudaStreamDestroy(cs);
    return neo::cuda_fail(e, "creating the swap copy stream / events");
  }
  pool->device = dev;
  pool->copy_stream = cs;
  pool->ev_ready[0] = ev[0];
  pool->ev_ready[1] = ev[1];
  pool->ev_free[0] = ev[2];
  pool->ev_free[1] = ev[3];
  pool->ev_start = ev[4];
  pool->ev_join = ev[5];
  return NEO_OK;
}

// One PCIe copy between staging rows [i, j) of a chunk starting at page c0 and
// the host pages host_ids[c0 + i ..] (consecutive ids: one 2D copy per run).
static cudaError_t copy_runs(neo_kv_pool* pool, bool to_host, const int32_t* host_ids, int32_t c0, int32_t cn,
                             uint8_t* stg, size_t per_page, size_t host_page, size_t host_off, cudaStream_t s) {
  for (int32_t i = 0; i < cn;) {
    int32_t j = i + 1;
    while (j < cn && host_ids[c0 + j] == host_ids[c0 + j - 1] + 1) ++j;
    uint8_t* host = pool->host_base + static_cast<size_t>(host_ids[c0 + i]) * host_page + host_off;
    uint8_t* dev = stg + static_cast<size_t>(i) * per_page;
    cudaError_t e = to_host ? cudaMemcpy2DAsync(host, host_page, dev, per_page, per_page, j - i,
                                                cudaMemcpyDeviceToHost, s)
                            : cudaMemcpy2DAsync(dev, per_page, host, host_page, per_page, j - i,
                                                cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    i = j;
  }
  return cudaSuccess;
}

static neo_status swap_common(neo_kv_pool* pool, bool out_dir, int32_t n, const int32_t* gpu_ids,
                              const int32_t* host_ids, int32_t l0, int32_t l1, void* staging, size_t staging_bytes,
                              uint32_t flags, void* stream) {
  if (!pool) return fail(NEO_ERR_INVALID_ARG, "pool is NULL");
  if (flags & ~static_cast<uint32_t>(NEO_SWAP_DEFER_JOIN)) return fail(NEO_ERR_INVALID_ARG, "unknown swap flags");
  if ((flags & NEO_SWAP_DEFER_JOIN) && !out_dir) return fail(NEO_ERR_INVALID_ARG, "NEO_SWAP_DEFER_JOIN is swap-out only");
  if (n < 0) return fail(NEO_ERR_INVALID_ARG, "n_pages < 0");
  if (l0 < 0 || l1 > pool->geo.num_layers || l0 >= l1) return fail(NEO_ERR_INVALID_ARG, "layer range out of bounds");
  if (n == 0) return NEO_OK;
  if (!gpu_ids || !host_ids) return fail(NEO_ERR_INVALID_ARG, "NULL pointer argument");
  if (staging && !neo::aligned16(staging)) return fail(NEO_ERR_INVALID_ARG, "staging must be 16-byte aligned");
  const size_t per_page = static_cast<size_t>(l1 - l0) * 2 * pool->layer_bytes;
  if (staging && staging_bytes < per_page)
    return fail(NEO_ERR_INVALID_ARG, "staging smaller than one page's layer range");
  // ---- validation: everything that can be checked is checked before the
  // first enqueue, so a non-OK return leaves the streams untouched.
  std::lock_guard<std::mutex> lk(pool->mu);
  {
    neo_status st = check_ids(pool->gpu_used, n, gpu_ids, "GPU page");
    if (st != NEO_OK) return st;
    st = check_ids(pool->host_used, n, host_ids, "host page");
    if (st != NEO_OK) return st;
  }
  {
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return neo::cuda_fail(e, "a previous CUDA error is pending; nothing enqueued");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap_st) != cudaSuccess) {
    cudaGetLastError();
    return fail(NEO_ERR_INVALID_ARG, "invalid stream");
  }
  uint16_t* host_dev = nullptr;
  if (!staging) {  // zero-copy: the CPU-cache must be device-mapped (UVA pinned memory)
    void* dp = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dp, pool->host_base, 0);
    if (e != cudaSuccess || !dp) {
      cudaGetLastError();
      return fail(NEO_ERR_UNSUPPORTED, "zero-copy swap needs device-mapped pinned host memory");
    }
    host_dev = static_cast<uint16_t*>(dp);
  } else if (cap_st == cudaStreamCaptureStatusNone) {  // (pointer queries are skipped under graph capture)
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, staging);
    if (e != cudaSuccess || at.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      return fail(NEO_ERR_INVALID_ARG, "staging must be device memory");
    }
    e = cudaPointerGetAttributes(&at, pool->host_base);
    if (e != cudaSuccess || at.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return fail(NEO_ERR_INVALID_ARG, "the CPU-cache must be pinned (page-locked) host memory");
    }
  }
  if (!staging) {
    for (int32_t c0 = 0; c0 < n; c0 += neo::kMaxZeroCopyPairs) {
      const int32_t cn = std::min<int32_t>(neo::kMaxZeroCopyPairs, n - c0);
      neo::SwapPairs ids;
      for (int32_t i = 0; i < cn; ++i) {
        ids.gpu[i] = gpu_ids[c0 + i];
        ids.host[i] = host_ids[c0 + i];
      }
      neo_status st = neo::launch_zero_copy(out_dir, reinterpret_cast<uint16_t*>(pool->gpu_base), host_dev, ids, cn,
                                            pool->geo.num_gpu_pages, pool->page_elems, pool->geo.num_layers, l0, l1, s);
      if (st != NEO_OK) return st;
    }
    return NEO_OK;
  }
  const size_t host_page = static_cast<size_t>(pool->geo.num_layers) * 2 * pool->layer_bytes;
  const size_t host_off = static_cast<size_t>(l0) * 2 * pool->layer_bytes;
  uint8_t* stg = static_cast<uint8_t*>(staging);
  uint16_t* gpu16 = reinterpret_cast<uint16_t*>(pool->gpu_base);
  // Pipelined when two halves of the staging hold a page each and the stream is
  // not being captured into a graph (a capture cannot wait on the pipeline's
  // events from earlier, uncaptured calls); otherwise one buffer, serially on
  // the caller's stream.
  const size_t half_pages = staging_bytes / 2 / per_page;
  const bool pipelined = half_pages >= 1 && cap_st == cudaStreamCaptureStatusNone;
  if (pipelined) {
    neo_status st = ensure_swap_pipeline(pool);
    if (st != NEO_OK) return st;
  }
  const int64_t cap = std::min<int64_t>(pipelined ? half_pages : staging_bytes / per_page, neo::kMaxSwapIdsPerLaunch);
  const size_t half_bytes = pipelined ? half_pages * per_page : 0;
  cudaStream_t cs = pool->copy_stream;
  cudaError_t e = cudaSuccess;
  if (pipelined) {  // the copy stream starts after the work the caller enqueued before this call
    e = cudaEventRecord(pool->ev_start, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, pool->ev_start, 0);
    if (e != cudaSuccess) return neo::cuda_fail(e, "swap pipeline start");
  } else if (cs && cap_st == cudaStreamCaptureStatusNone) {
    // one-buffer path after pipelined calls: a deferred D2H may still read the staging
    for (int h = 0; h < 2 && e == cudaSuccess; ++h)
      if (pool->half_used[h]) e = cudaStreamWaitEvent(s, pool->ev_free[h], 0);
    if (e != cudaSuccess) return neo::cuda_fail(e, "swap pipeline wait");
  }
  int last_half = -1;
  for (int32_t c0 = 0; c0 < n; c0 += static_cast<int32_t>(cap)) {
    const int32_t cn = static_cast<int32_t>(std::min<int64_t>(cap, n - c0));
    neo::SwapBatch ids;
    for (int32_t i = 0; i < cn; ++i) ids.ids[i] = gpu_ids[c0 + i];
    if (!pipelined) {
      if (!out_dir) {
        e = copy_runs(pool, false, host_ids, c0, cn, stg, per_page, host_page, host_off, s);
        if (e != cudaSuccess) return neo::cuda_fail(e, "cudaMemcpy2DAsync(H2D swap-in)");
        neo_status st = neo::launch_scatter(gpu16, reinterpret_cast<const uint16_t*>(stg), ids, cn,
                                            pool->geo.num_gpu_pages, pool->page_elems, l0, l1, s);
        if (st != NEO_OK) return st;
      } else {
        neo_status st = neo::launch_gather(gpu16, reinterpret_cast<uint16_t*>(stg), ids, cn, pool->geo.num_gpu_pages,
                                           pool->page_elems, l0, l1, s);
        if (st != NEO_OK) return st;
        e = copy_runs(pool, true, host_ids, c0, cn, stg, per_page, host_page, host_off, s);
        if (e != cudaSuccess) return neo::cuda_fail(e, "cudaMemcpy2DAsync(D2H swap-out)");
      }
      continue;
    }
    const int h = pool->next_half;
    pool->next_half ^= 1;
    last_half = h;
    uint8_t* buf = stg + h * half_bytes;
    if (out_dir) {
      // gather into half h (after its previous reader finished) on the caller's
      // stream, then D2H on the copy stream
      if (pool->half_used[h]) e = cudaStreamWaitEvent(s, pool->ev_free[h], 0);
      if (e != cudaSuccess) return neo::cuda_fail(e, "swap pipeline wait");
      neo_status st = neo::launch_gather(gpu16, reinterpret_cast<uint16_t*>(buf), ids, cn, pool->geo.num_gpu_pages,
                                         pool->page_elems, l0, l1, s);
      if (st != NEO_OK) return st;
      e = cudaEventRecord(pool->ev_ready[h], s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, pool->ev_ready[h], 0);
      if (e == cudaSuccess) e = copy_runs(pool, true, host_ids, c0, cn, buf, per_page, host_page, host_off, cs);
      if (e == cudaSuccess) e = cudaEventRecord(pool->ev_free[h], cs);
      if (e != cudaSuccess) return neo::cuda_fail(e, "swap-out D2H");
    } else {
      // H2D into half h on the copy stream, then scatter on the caller's stream
      if (pool->half_used[h]) e = cudaStreamWaitEvent(cs, pool->ev_free[h], 0);
      if (e == cudaSuccess) e = copy_runs(pool, false, host_ids, c0, cn, buf, per_page, host_page, host_off, cs);
      if (e == cudaSuccess) e = cudaEventRecord(pool->ev_ready[h], cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, pool->ev_ready[h], 0);
      if (e != cudaSuccess) return neo::cuda_fail(e, "swap-in H2D");
      neo_status st = neo::launch_scatter(gpu16, reinterpret_cast<const uint16_t*>(buf), ids, cn,
                                          pool->geo.num_gpu_pages, pool->page_elems, l0, l1, s);
      if (st != NEO_OK) return st;
      e = cudaEventRecord(pool->ev_free[h], s);
      if (e != cudaSuccess) return neo::cuda_fail(e, "swap pipeline record");
    }
    pool->half_used[h] = true;
  }
  // The caller's stream completes only after the last copy: swap-out's final
  // D2H ran on the copy stream (in order, so it covers every earlier one).
  // NEO_SWAP_DEFER_JOIN leaves that to neo_kv_swap_join, so the next layer's
  // gather on the same stream is not held behind this layer's D2H.
  if (pipelined && out_dir && last_half >= 0 && !(flags & NEO_SWAP_DEFER_JOIN)) {
    e = cudaStreamWaitEvent(s, pool->ev_free[last_half], 0);
    if (e != cudaSuccess) return neo::cuda_fail(e, "swap pipeline join");
  }
  return NEO_OK;
}

NEO_API neo_status neo_kv_swap_out(neo_kv_pool* pool, int32_t n, const int32_t* gpu_ids, const int32_t* host_ids,
                                   int32_t l0, int32_t l1, void* staging, size_t staging_bytes, void* stream) {
  return swap_common(pool, true, n, gpu_ids, host_ids, l0, l1, staging, staging_bytes, 0u, stream);
}

NEO_API neo_status neo_kv_swap_out_ex(neo_kv_pool* pool, int32_t n, const int32_t* gpu_ids, const int32_t* host_ids,
                                      int32_t l0, int32_t l1, void* staging, size_t staging_bytes, uint32_t flags,
                                      void* stream) {
  return swap_common(pool, true, n, gpu_ids, host_ids, l0, l1, staging, staging_bytes, flags, stream);
}

NEO_API neo_status neo_kv_swap_in(neo_kv_pool* pool, int32_t n, const int32_t* host_ids, const int32_t* gpu_ids,
                                  int32_t l0, int32_t l1, void* staging, size_t staging_bytes, void* stream) {
  return swap_common(pool, false, n, gpu_ids, host_ids, l0, l1, staging, staging_bytes, 0u, stream);
}

NEO_API neo_status neo_kv_swap_join(neo_kv_pool* pool, void* stream) {
  if (!pool) return fail(NEO_ERR_INVALID_ARG, "pool is NULL");
  std::lock_guard<std::mutex> lk(pool->mu);
  if (!pool->copy_stream) return NEO_OK;  // no pipelined swap was ever issued
  cudaError_t e = cudaEventRecord(pool->ev_join, pool->copy_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), pool->ev_join, 0);
  return e == cudaSuccess ? NEO_OK : neo::cuda_fail(e, "neo_kv_swap_join");
}

}  // extern "C"
