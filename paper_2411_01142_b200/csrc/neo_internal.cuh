// Internal declarations shared by the libneo translation units (host ABI,
// attention kernel, swap kernels).  Not part of the public ABI (include/neo.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/neo.h"

namespace neo {

constexpr int kHeadDim = 128;
constexpr int kTileTokens = 16;                       // tokens per MMA tile
constexpr int kTileBytes = kTileTokens * kHeadDim * 2;  // 4096: one K (or V) tile
constexpr int kMaxGroup = 8;                          // G <= 8 (MMA N = 8)
constexpr int kMaxChunkTokens = 1024;                 // <= 64 tiles per work unit
constexpr int kDefaultMaxChunk = 512;                 // cap of the shape-only default chunk

// Runs f(device) once per CUDA device for one call site (kernel attributes such
// as the dynamic shared-memory limit are per device); thread-safe -- two
// threads racing on a first launch both run the idempotent f.
template <typename F>
inline neo_status once_per_device(std::atomic<uint64_t>& done_mask, F&& f) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done_mask.load(std::memory_order_acquire) & bit) return NEO_OK;
  const neo_status st = f(dev);
  if (st == NEO_OK) done_mask.fetch_or(bit, std::memory_order_acq_rel);
  return st;
}

// SM count of the current device (148 when no device is visible)
int device_sm_count();

// thread-local error text for neo_last_error()
void set_error(const std::string& msg);
neo_status fail(neo_status st, const std::string& msg);
neo_status cuda_fail(cudaError_t e, const char* what);

// ---- decode attention (neo_attn.cu)
struct AttnLaunch {
  const void* q;
  void* out;
  const int32_t* block_table;
  const int32_t* seq_lens;
  void* workspace;
  size_t workspace_bytes;
  int32_t batch, hq, hkv, page_size, max_blocks, chunk_tokens, max_chunks;
  float scale;
  cudaStream_t stream;
  // fused append (+ RoPE): k_new != NULL selects decode_attn_kernel<..., kFuse>
  const float* inv_freq = nullptr;
  const void* k_new = nullptr;
  const void* v_new = nullptr;
  void* k_pages = nullptr;
  void* v_pages = nullptr;
  int64_t page_stride = 0;
  bool grouped = false;        // NEO_CHUNK_GROUPED: max_chunks holds the group count
  bool early = false;          // NEO_ATTN_KV_STABLE: metadata + first KV tiles before the PDL wait
};
constexpr int kGroupTiles = 4 * 64;                   // largest group of the grouped kernel (tiles)
// chunk_tokens -k (k = 1, 2, 4) selects groups of kGroupTiles / k tiles; any
// other negative value -T (T a multiple of 16 in [64, 4096]) groups of T tokens
inline bool is_grouped_chunk(int32_t c) {
  return c == -1 || c == -2 || c == -4 || (c <= -64 && c >= -kGroupTiles * kTileTokens && (-c) % kTileTokens == 0);
}
inline int32_t group_tiles_of(int32_t c) { return c >= -4 ? kGroupTiles / (-c) : (-c) / kTileTokens; }
inline int32_t max_groups_for(int32_t max_seq_len, int32_t group_tiles) {
  const int32_t tiles = (max_seq_len + kTileTokens - 1) / kTileTokens;
  return tiles > 0 ? (tiles + group_tiles - 1) / group_tiles : 1;
}
// Byte layout of a workspace of `ws_bytes` bytes for a call shape.  The
// completion counters occupy [0, counter_cap(ws_bytes)) -- a region fixed by the
// workspace size alone, so calls of different shapes sharing one workspace
// never alias one call's counters with another call's partials.
struct WorkspaceLayout {
  size_t cnt_off, cnt_cap, ml_off, acc_off, total;
  bool fits;
};
size_t workspace_counter_cap(size_t ws_bytes);
size_t workspace_required(int32_t batch, int32_t hq, int32_t hkv, int32_t max_chunks);
WorkspaceLayout workspace_layout(int32_t batch, int32_t hq, int32_t hkv, int32_t max_chunks, size_t ws_bytes);
neo_status launch_decode_attn(const AttnLaunch& a, const CUtensorMap& tmk, const CUtensorMap& tmv);
// Default kernel shape launch_decode_attn picks for a grid of `max_chunks` chunk
// levels: (4 warps, 3 stages) -> 2 resident CTAs per SM for <= 3 chunks per
// request, else (4 warps, 2 stages) -> 3 CTAs per SM.  The chunk planner
// simulates the same shape.
struct AttnShape {
  int warps, stages, ctas_per_sm;
};
inline AttnShape default_attn_shape(int32_t max_chunks) {
  return max_chunks <= 3 ? AttnShape{4, 3, 2} : AttnShape{4, 2, 3};
}
// debug validation of device metadata (syncs the stream)
neo_status debug_validate_attn(const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                               int32_t batch, int32_t page_size, int32_t max_seq_len, int64_t num_pages,
                               cudaStream_t stream);
neo_status debug_validate_offsets(const int32_t* q_offsets, const int32_t* seq_lens, int32_t batch, int32_t total,
                                  int32_t max_q_len, cudaStream_t stream);

// ---- tensor maps (neo_host.cu; cached by pointer and shape)
neo_status tensor_map(const void* ptr, int64_t page_stride, int64_t num_pages, int32_t hkv, int32_t P,
                      CUtensorMap* out);
neo_status tensor_map_prefill_kv(const void* ptr, int64_t page_stride, int64_t num_pages, int32_t hkv, int32_t P,
                                 CUtensorMap* out);
neo_status tensor_map_prefill_q(const void* ptr, int32_t total_tokens, int32_t hq, int32_t G, CUtensorMap* out);
neo_status tensor_map_prefill_out(void* ptr, int32_t total_tokens, int32_t hq, int32_t G, CUtensorMap* out);

// ---- prefill attention (neo_prefill.cu)
struct PrefillLaunch {
  void* out;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const int32_t* q_offsets;
  int32_t batch, hq, hkv, page_size, max_blocks, max_q_len;
  float scale;
  cudaStream_t stream;
  int32_t max_ctas;   // 0: one CTA per SM
};
neo_status launch_prefill_attn(const PrefillLaunch& a, const CUtensorMap& tmq, const CUtensorMap& tmk,
                               const CUtensorMap& tmv, const CUtensorMap& tmo);

// ---- KV append (neo_swap.cu)
neo_status launch_append(uint16_t* k, uint16_t* v, int64_t page_stride, const int32_t* block_table, int32_t max_blocks,
                         const int32_t* seq_lens, const uint16_t* k_new, const uint16_t* v_new, int32_t batch,
                         int32_t hkv, int32_t page_size, cudaStream_t s);

neo_status launch_rope_append(uint16_t* q, int32_t hq, const float* inv_freq, uint16_t* k, uint16_t* v,
                              int64_t page_stride, const int32_t* block_table, int32_t max_blocks,
                              const int32_t* seq_lens, const int32_t* q_offsets, const uint16_t* k_new,
                              const uint16_t* v_new, int32_t batch, int32_t tokens, int32_t hkv, int32_t page_size,
                              cudaStream_t s);

// ---- swap (neo_swap.cu)
constexpr int kMaxSwapIdsPerLaunch = 960;  // page ids passed by value in the kernel params
struct SwapBatch {
  int32_t ids[kMaxSwapIdsPerLaunch];
};
// staging[i][l - l0][kv][...page_elems] <-> gpu[l][kv][ids[i]][...]
neo_status launch_gather(const uint16_t* gpu_base, uint16_t* staging, const SwapBatch& ids, int32_t n,
                         int64_t num_gpu_pages, int64_t page_elems, int32_t l0, int32_t l1, cudaStream_t s);
// Zero-copy variant: the kernel reads/writes the pinned host pages directly
// through their device-mapped (UVA) address -- no staging buffer, no copy engine.
constexpr int kMaxZeroCopyPairs = 480;
struct SwapPairs {
  int32_t gpu[kMaxZeroCopyPairs];
  int32_t host[kMaxZeroCopyPairs];
};
neo_status launch_zero_copy(bool to_host, uint16_t* gpu_base, uint16_t* host_dev, const SwapPairs& ids, int32_t n,
                            int64_t num_gpu_pages, int64_t page_elems, int32_t num_layers, int32_t l0, int32_t l1,
                            cudaStream_t s);
neo_status launch_scatter(uint16_t* gpu_base, const uint16_t* staging, const SwapBatch& ids, int32_t n,
                          int64_t num_gpu_pages, int64_t page_elems, int32_t l0, int32_t l1, cudaStream_t s);

}  // namespace neo
