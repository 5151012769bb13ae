/*
 * neo.h -- C ABI of libneo, the B200 (sm_100a) hot path of NEO
 * (arXiv 2411.01142, "NEO: Saving GPU Memory Crisis with CPU Offloading for
 * Online LLM Inference").  Citations: P:n = PAPER.md line n, S:n = SPEC.md
 * line n.
 *
 * What crosses this boundary:
 *   - a paged KV cache split into a GPU-cache (HBM) and a CPU-cache (pinned
 *     host memory); every prefilled request lives entirely in one of them
 *     (Sec 3.1 "partial offloading");
 *   - one batched decode-attention call per layer per iteration covering the
 *     whole GPU sub-batch (attention semantics P:97-98);
 *   - the page swap that moves a request's KV between the two caches for a
 *     range of layers (P:240 layer-wise swapping, P:285-288 scheduling steps
 *     2, 3, 5; PCIe-bound per P:121).
 *
 * Conventions (all calls):
 *   - Every call returns neo_status.  NEO_OK = 0.  neo_last_error() returns a
 *     thread-local human-readable message for the last failing call.
 *   - All-or-nothing: a non-OK return has enqueued no GPU work and changed no
 *     pool state (mirrors S:262, S:292 atomicity).  Every argument is validated
 *     before the first enqueue; the one exception is NEO_ERR_CUDA raised by an
 *     enqueue itself (a failing CUDA context), see the swap section.
 *   - Ownership: the CALLER allocates and owns every device buffer (pool, q,
 *     out, workspace, staging) and the pinned host pool; the library never
 *     allocates or frees device memory.  Pointers must stay valid until the
 *     work enqueued on them has completed.  A pool handle owns only host-side
 *     free lists and is single-writer.
 *   - Asynchrony: attention and swap calls validate host-visible arguments,
 *     enqueue on the given stream and return without synchronising.  Device
 *     contents (seq_lens, block-table ids) are validated only when the
 *     environment variable NEO_DEBUG_VALIDATE=1 is set; that path synchronises
 *     the stream.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - No C++ exception crosses the ABI.
 *   - Element type of q, out and the KV pages is bf16 (IEEE binary16 brain
 *     float, passed as raw 16-bit words); arithmetic is fp32 (DESIGN.md c7).
 */
#ifndef NEO_H_
#define NEO_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NEO_API __attribute__((visibility("default")))
#else
#define NEO_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NEO_OK = 0,
  NEO_ERR_INVALID_ARG = 1,  /* null/misaligned pointer, bad shape, bad id, range error */
  NEO_ERR_OUT_OF_PAGES = 2, /* allocation cannot be satisfied; nothing allocated       */
  NEO_ERR_UNSUPPORTED = 3,  /* head_dim != 128, page_size not a multiple of 16, G > 8  */
  NEO_ERR_CUDA = 4,         /* a CUDA runtime/driver call failed                        */
  NEO_ERR_INTERNAL = 5
} neo_status;

enum { NEO_GPU = 0, NEO_HOST = 1 };

/* Thread-local message describing the last non-OK return on this thread. */
NEO_API const char* neo_last_error(void);
NEO_API const char* neo_version(void);

/* ------------------------------------------------------------------ KV pool
 * Geometry of one model's KV cache ("paged KV cache similar to vLLM").
 *
 * GPU-cache layout (layer-major), bf16:
 *     gpu[L][2 (K,V)][num_gpu_pages][Hkv][P][D]
 *   so one (page, kv-head) block is a contiguous P*D*2-byte run (4 KiB at
 *   P=16, D=128) and a layer's K view is [num_gpu_pages][Hkv][P][D] with
 *   page_stride = Hkv*P*D elements.
 * CPU-cache layout (page-major, each page self-contained across layers), bf16:
 *     host[num_host_pages][L][2 (K,V)][Hkv][P][D]
 *   i.e. the same per-(layer, K|V) byte layout, ready for a CPU attention
 *   kernel over host pages (out of scope here). */
typedef struct {
  int32_t num_layers;   /* L  >= 1                      */
  int32_t num_kv_heads; /* Hkv >= 1 (local to this rank) */
  int32_t head_dim;     /* D, must be 128                */
  int32_t page_size;    /* P tokens per page, multiple of 16 (16 or 32 typical) */
  int64_t num_gpu_pages;
  int64_t num_host_pages;
} neo_kv_geometry;

typedef struct neo_kv_pool neo_kv_pool;

/* Bytes the caller must provide for the two caches of `geo`. */
NEO_API neo_status neo_kv_pool_bytes(const neo_kv_geometry* geo, size_t* gpu_bytes, size_t* host_bytes);

/* Create a pool over caller-owned memory.  gpu_kv_base: device pointer,
 * >= gpu_bytes, 16-byte aligned.  host_kv_base: PINNED host pointer (page-locked
 * via cudaHostAlloc / torch pin_memory), >= host_bytes, 16-byte aligned; may be
 * NULL iff num_host_pages == 0.  The handle is written to *out. */
NEO_API neo_status neo_kv_pool_create(const neo_kv_geometry* geo, void* gpu_kv_base, size_t gpu_bytes,
                                      void* host_kv_base, size_t host_bytes, neo_kv_pool** out);
NEO_API void neo_kv_pool_destroy(neo_kv_pool* pool);

/* Allocate n_pages page ids in `where` (NEO_GPU or NEO_HOST) into the host
 * array page_ids_out[n_pages].  All-or-nothing: NEO_ERR_OUT_OF_PAGES leaves the
 * pool unchanged (S:255-263 allocate; S:265-273 extend = alloc(1)).  Host ids
 * are returned as one ascending contiguous run when one exists, so a swap is a
 * single strided memcpy.  n_pages == 0 is a no-op. */
NEO_API neo_status neo_kv_alloc(neo_kv_pool* pool, int32_t where, int32_t n_pages, int32_t* page_ids_out);

/* Return pages to `where`.  Every id must be currently allocated there and
 * appear once; otherwise NEO_ERR_INVALID_ARG and nothing is freed
 * (S:285-288 release). */
NEO_API neo_status neo_kv_free(neo_kv_pool* pool, int32_t where, int32_t n_pages, const int32_t* page_ids);

/* Number of free pages in `where` (conservation: free + allocated = capacity). */
NEO_API neo_status neo_kv_free_count(const neo_kv_pool* pool, int32_t where, int64_t* n_free);

/* Device pointers of layer `layer`'s K and V page arrays and their page stride
 * in elements, for neo_decode_attn. */
NEO_API neo_status neo_kv_layer_view(const neo_kv_pool* pool, int32_t layer, void** k_pages, void** v_pages,
                                     int64_t* page_stride_elems);

/* --------------------------------------------------------- decode attention
 * One decode step of GQA attention for a batch of GPU-resident requests
 * (P:97-98):
 *
 *   for b < batch, h < Hq:   g = floor(h / G), G = Hq / Hkv        (DESIGN c2)
 *     out[b][h][:] = sum_t softmax_t(scale * q[b][h] . K_b[t][g]) * V_b[t][g][:]
 *   over ALL t < seq_lens[b] (the caller has already appended this step's token;
 *   no causal mask, no window; DESIGN c3).  K_b[t] lives at token t % P of
 *   physical page block_table[b][t / P].
 *
 * Arguments:
 *   q           [batch][Hq][D] bf16, device, 16-byte aligned.
 *   k_pages,
 *   v_pages     device; page p, kv-head g starts at element p*page_stride + g*P*D
 *               and holds [P][D] bf16 (token-major).  16-byte aligned, page_stride
 *               a multiple of 8 elements and >= Hkv*P*D.
 *   num_pages   pages addressable through k_pages/v_pages (ids must be < num_pages).
 *   block_table [batch][max_blocks] int32, device.  Entries at or beyond
 *               ceil(seq_lens[b]/P) are never read (may be -1); a physical page may
 *               appear in several rows (read-only sharing; DESIGN c10).
 *   seq_lens    [batch] int32, device, each in [0, min(max_seq_len, max_blocks*P)].
 *               0 yields a zero output row (DESIGN c4).
 *   out         [batch][Hq][D] bf16, device (fp32 -> bf16 round-to-nearest-even).
 *   max_seq_len host-known upper bound of seq_lens (sizes the grid).
 *   scale       softmax scale, typically 1/sqrt(D) (DESIGN c1).
 *   chunk_tokens split-K chunk length C (multiple of 16 and of P, <= 1024), or 0 for
 *               the library default neo_decode_attn_default_chunk(), or
 *               NEO_CHUNK_GROUPED (-1), -2 or -4, or -T for T a multiple of 16
 *               in [64, 4096]: the grouped kernel -- each request's tiles split
 *               into ceil(tiles / (T/16)) equal groups (-1, -2, -4 = groups of at
 *               most 4096, 2048, 1024 tokens; -T = at most T tokens), the tiles
 *               of a group dealt round-robin to four warps, one CTA per group,
 *               merged in shared memory; single-group requests need no partials.
 *               neo_decode_attn_plan_chunk() picks among these and the split
 *               chunks.  The result for
 *               request b depends only on (its inputs, C): outputs are bitwise
 *               deterministic run to run (fixed merge order, no float atomics).
 *   workspace   device scratch of >= neo_decode_attn_workspace_bytes(...) bytes,
 *               initialised ONCE with neo_decode_attn_workspace_init(); the kernel
 *               leaves it re-usable.  One workspace per concurrently running stream.
 * Errors: NEO_ERR_INVALID_ARG (nulls, misalignment, Hq % Hkv != 0, max_seq_len >
 * max_blocks*P, workspace too small); NEO_ERR_UNSUPPORTED (D != 128, P % 16 != 0,
 * G > 8, C invalid); NEO_ERR_CUDA.  batch == 0 is a no-op. */
NEO_API neo_status neo_decode_attn(const void* q, const void* k_pages, const void* v_pages, int64_t page_stride,
                                   int64_t num_pages, const int32_t* block_table, int32_t max_blocks,
                                   const int32_t* seq_lens, void* out, int32_t batch, int32_t num_q_heads,
                                   int32_t num_kv_heads, int32_t head_dim, int32_t page_size, int32_t max_seq_len,
                                   float scale, int32_t chunk_tokens, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* neo_decode_attn with flags.  NEO_ATTN_KV_STABLE: the caller guarantees that
 * the kernels still running on `stream` when this call is enqueued write none
 * of the KV pages, block table or seq_lens this call reads -- except each
 * request's newest token slot (a preceding neo_kv_append / neo_rope_append).
 * With programmatic dependent launch the kernel then reads the metadata and
 * streams its first KV tiles (never a tile holding a newest token) BEFORE
 * waiting on the preceding kernel, overlapping that kernel's tail; q is read
 * and every output written only after the wait.  Holds for the layers of a
 * decode step (earlier tokens' KV is immutable); do NOT set it right after a
 * swap-in scatter or neo_prefill_append into pages this call reads.  Same
 * result bit for bit; other arguments and errors as neo_decode_attn
 * (NEO_ERR_INVALID_ARG for unknown flag bits). */
#define NEO_ATTN_KV_STABLE 1u
NEO_API neo_status neo_decode_attn_ex(const void* q, const void* k_pages, const void* v_pages, int64_t page_stride,
                                      int64_t num_pages, const int32_t* block_table, int32_t max_blocks,
                                      const int32_t* seq_lens, void* out, int32_t batch, int32_t num_q_heads,
                                      int32_t num_kv_heads, int32_t head_dim, int32_t page_size, int32_t max_seq_len,
                                      float scale, int32_t chunk_tokens, void* workspace, size_t workspace_bytes,
                                      uint32_t flags, void* stream);

/* Append this decode step's K and V rows to the paged cache (the
 * decoding stage "read-and-appends the KV cache"), before neo_decode_attn:
 *   for b < batch with seq_lens[b] >= 1, t = seq_lens[b] - 1 (seq_lens already
 *   count the new token):  page block_table[b][t / P], slot t % P, kv-head g
 *   receives k_new[b][g][:] and v_new[b][g][:]  (bit copy).
 * k_pages/v_pages/page_stride/num_pages/block_table/max_blocks/seq_lens as for
 * neo_decode_attn; k_new, v_new: [batch][Hkv][D] bf16 device, 16-byte aligned.
 * Asynchronous on `stream`; the caller allocates the page (neo_kv_alloc) when t
 * crosses a page boundary (S:265-273 extend). */
NEO_API neo_status neo_kv_append(void* k_pages, void* v_pages, int64_t page_stride, int64_t num_pages,
                                 const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                                 const void* k_new, const void* v_new, int32_t batch, int32_t num_kv_heads,
                                 int32_t head_dim, int32_t page_size, void* stream);

/* neo_kv_append with rotary position embedding fused in (RoFormer
 * rotate-half convention as in LLaMa): for each request b at position
 * t = seq_lens[b] - 1 and each dim pair (i, i + D/2), i < D/2, with
 * theta_i = t * inv_freq[i] (angle and sin/cos in fp64, rotation in fp32):
 *   x'[i]       = x[i] cos theta_i - x[i + D/2] sin theta_i
 *   x'[i + D/2] = x[i + D/2] cos theta_i + x[i] sin theta_i
 * applied to every q head (q_inout [batch][Hq][D], rotated in place) and to k_new
 * before it is written to the page slot; v_new is written unrotated.
 * inv_freq: device float[D/2] (the model's frequency table, any scaling already
 * applied by the caller).  Other arguments and errors as neo_kv_append. */
NEO_API neo_status neo_rope_append(void* q_inout, int32_t num_q_heads, const float* inv_freq, void* k_pages,
                                   void* v_pages, int64_t page_stride, int64_t num_pages, const int32_t* block_table,
                                   int32_t max_blocks, const int32_t* seq_lens, const void* k_new, const void* v_new,
                                   int32_t batch, int32_t num_kv_heads, int32_t head_dim, int32_t page_size,
                                   void* stream);

/* Causal paged GQA prefill attention (the prefill half of
 * batch-0; attention as P:97-98): for request b with
 * n_q = q_offsets[b+1] - q_offsets[b] query tokens that are the LAST n_q of its
 * n = seq_lens[b] cached tokens, query row i (packed row j = q_offsets[b] + i,
 * position p = n - n_q + i) and q-head h (kv-head g = h / G):
 *   out[j][h][:] = sum_{t <= p} softmax_t(scale * q[j][h] . K_b[t][g]) V_b[t][g][:]
 * K_b[t] lives in page block_table[b][t / P], slot t % P (as neo_decode_attn).
 * The new tokens' K/V must already be in the pages (neo_prefill_append).
 *   q, out     [total_tokens][Hq][D] bf16 device; q 16-byte, out 32-byte aligned
 *   q_offsets  device int32[batch + 1], 0 = q_offsets[0] <= ... = total_tokens
 *   max_q_len  >= every n_q (sizes the grid; rows beyond a request's n_q idle)
 *   G = Hq / Hkv in {1, 2, 4, 8, 16}; D = 128; P a multiple of 16;
 *   batch <= 512 and max_q_len * G <= 262144 (the per-CTA schedule table).
 * Numerics: Q.K^T with bf16 x bf16 products exact in fp32 (tcgen05.mma), softmax
 * in fp32 (exp2 domain).  P.V: for max_q_len >= 256, P (scaled by 2^7) and V are
 * rounded to fp16 (RNE; V saturates beyond fp16's range, so V entries must lie
 * within |v| <= 65504) with fp32 accumulation; shorter calls apply P as bf16
 * hi + lo against bf16 V (DESIGN "prefill P.V").  Output RNE to bf16.
 * Kernels (DESIGN NEXT-3): fp16-path calls with max_q_len <= 3072 run the
 * warp-specialised stream kernel (all exponentials on MUFU), longer calls the
 * item-major kernel (a quarter of the exponentials by a degree-4 polynomial,
 * relative error <= 4.3e-5); both within the tolerance rule, selected by shape.
 * Deterministic for a fixed call shape.
 * Page-tail slots beyond seq_lens are never read into the result (NaN-safe).
 * Errors: NEO_ERR_INVALID_ARG, NEO_ERR_UNSUPPORTED, NEO_ERR_CUDA; NEO_DEBUG_VALIDATE=1
 * checks the metadata on the host.  batch == 0 or total_tokens == 0 is a no-op. */
NEO_API neo_status neo_prefill_attn(const void* q, const void* k_pages, const void* v_pages, int64_t page_stride,
                                    int64_t num_pages, const int32_t* block_table, int32_t max_blocks,
                                    const int32_t* seq_lens, const int32_t* q_offsets, void* out, int32_t batch,
                                    int32_t total_tokens, int32_t num_q_heads, int32_t num_kv_heads,
                                    int32_t head_dim, int32_t page_size, int32_t max_q_len, float scale,
                                    void* stream);

/* Prefill-side store (P:237-239 prefill in batch-0): write the
 * K and V rows of a packed batch of prompt chunks into the paged cache, with
 * optional RoPE (same convention and precision as neo_rope_append).
 *   request b owns packed tokens j in [q_offsets[b], q_offsets[b+1]) (device
 *   int32[batch + 1], q_offsets[0] = 0, q_offsets[batch] = total_tokens); its
 *   n_q = q_offsets[b+1] - q_offsets[b] new tokens are the LAST n_q of its
 *   seq_lens[b] tokens: token j sits at position t = seq_lens[b] - n_q +
 *   (j - q_offsets[b]), written to page block_table[b][t / P], slot t % P.
 *   k_new, v_new: [total_tokens][Hkv][D]; q_inout: [total_tokens][Hq][D].
 *   inv_freq NULL: plain copy, q untouched (may be NULL).  Otherwise q rows are
 *   rotated in place and k rows rotated before the store; v is copied.
 * Errors as neo_rope_append; NEO_DEBUG_VALIDATE=1 also checks q_offsets.
 * batch == 0 or total_tokens == 0 is a no-op. */
NEO_API neo_status neo_prefill_append(void* q_inout, int32_t num_q_heads, const float* inv_freq, void* k_pages,
                                      void* v_pages, int64_t page_stride, int64_t num_pages,
                                      const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                                      const int32_t* q_offsets, const void* k_new, const void* v_new, int32_t batch,
                                      int32_t total_tokens, int32_t num_kv_heads, int32_t head_dim,
                                      int32_t page_size, void* stream);

/* One-launch decode step (SURVEY NEXT-3 "fused KV append (+ RoPE) + decode
 * attention"; P:109-110 read-and-append): neo_rope_append (or neo_kv_append when
 * inv_freq is NULL) and neo_decode_attn fused into one kernel.  With the new
 * token at t = seq_lens[b] - 1:
 *   q' = RoPE_t(q[b]) (registers only: q is NOT written back)
 *   k' = RoPE_t(k_new[b]), v' = v_new[b]; k', v' are stored into the page slot
 *   of token t AND used as token t's K / V in
 *   out[b][h] = sum_{t' <= t} softmax(scale q'[h] . K[t'][g]) V[t'][g]
 * RoPE convention and precision as neo_rope_append (angle reduced in fp64,
 * sin / cos and rotation in fp32, bf16 RNE).  Other arguments, workspace and
 * errors as neo_decode_attn; k_new, v_new: [batch][Hkv][D] bf16, 16-byte
 * aligned; k_pages / v_pages are written (token t's slot only). */
NEO_API neo_status neo_decode_attn_append(const void* q, const float* inv_freq, const void* k_new, const void* v_new,
                                          void* k_pages, void* v_pages, int64_t page_stride, int64_t num_pages,
                                          const int32_t* block_table, int32_t max_blocks, const int32_t* seq_lens,
                                          void* out, int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                                          int32_t head_dim, int32_t page_size, int32_t max_seq_len, float scale,
                                          int32_t chunk_tokens, void* workspace, size_t workspace_bytes,
                                          void* stream);

/* chunk_tokens value selecting the grouped split-K kernel with groups of <= 4096
 * tokens; -2 and -4 select groups of <= 2048 and <= 1024 tokens, -T (T a
 * multiple of 16 in [64, 4096]) groups of <= T tokens (neo_decode_attn). */
#define NEO_CHUNK_GROUPED (-1)

/* Default split-K chunk length for a call shape (deterministic in its inputs). */
NEO_API int32_t neo_decode_attn_default_chunk(int32_t batch, int32_t num_kv_heads, int32_t max_seq_len);

/* a0 plan ("partition ... aggregate the partial
 * outputs") with the request lengths on the HOST -- NEO's scheduler holds them
 * (P:283-290).  Chooses chunk_tokens for one neo_decode_attn /
 * neo_decode_attn_append call over these requests (DESIGN §6 "chunk planner"):
 *  - a replay of the GPU's in-order CTA dispatch scores the split kernel at
 *    C in {1024, 640, 512, 448, 384, 320, 256} (multiples of page_size) and the
 *    grouped kernel at groups of 4096 / 3072 / 2048 / 1536 / 1024 tokens
 *    (returned as -1 / -3072 / -2 / -1536 / -4);
 *    a smaller C, a smaller group, and the grouped kernel over the split one
 *    must each win by > 1 %;
 *  - grids of >= 16 waves at C = 1024 score only that split chunk;
 *  - grids under one wave at the smallest C are latency-bound: the grouped
 *    kernel (-1) when every request fits one 4096-token group, else
 *    neo_decode_attn_default_chunk().
 * Pure host computation, no GPU work; the SM count is the current device's
 * (148 when no device is visible).
 *   seq_lens     [batch] int32, HOST, each >= 0 (the values the call will see).
 *   chunk_tokens out: a valid chunk_tokens argument for page_size (possibly
 *                -1, -3072, -2, -1536 or -4: the grouped kernel).
 * Any choice is correct (the result depends on it only through fp32 rounding);
 * this only affects speed.
 * Errors: NEO_ERR_INVALID_ARG (NULL pointers, batch < 0, num_kv_heads < 1, a
 * negative length); NEO_ERR_UNSUPPORTED (page_size not a multiple of 16 in
 * [16, 1024]). */
NEO_API neo_status neo_decode_attn_plan_chunk(const int32_t* seq_lens, int32_t batch, int32_t num_kv_heads,
                                              int32_t page_size, int32_t* chunk_tokens);

/* Workspace bytes for a call shape (chunk_tokens 0 = default). */
NEO_API neo_status neo_decode_attn_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t num_kv_heads,
                                                   int32_t head_dim, int32_t max_seq_len, int32_t chunk_tokens,
                                                   size_t* bytes);

/* Zero the workspace's completion counters (enqueued on `stream`).  Call once
 * after allocating a workspace. */
NEO_API neo_status neo_decode_attn_workspace_init(void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ swap
 * Swap-out (GPU-cache -> CPU-cache) of n_pages pages for layers
 * [layer_begin, layer_end):
 *   host[host_page_ids[i]][l][kv] = gpu[l][kv][gpu_page_ids[i]]  for every i, l, kv
 * bit-exactly.  gpu_page_ids must be allocated in NEO_GPU, host_page_ids in
 * NEO_HOST (host arrays, n_pages entries each, no duplicates).  A gather kernel
 * packs the pages into `staging` (device, 16-byte aligned) and cudaMemcpyAsync
 * moves them device->host, all on `stream`; staging smaller than the whole
 * transfer is reused chunk by chunk (it must hold at least one page's layer
 * range: neo_kv_swap_staging_bytes(pool, 1, ...)).  The call does NOT free the
 * GPU pages: record an event on `stream` and free them after it completes.  The
 * caller orders the call after the kernels that wrote those pages.
 * Swap-in is the mirror image (host -> staging -> scatter into gpu_page_ids,
 * which may differ from the ids the request had before).
 * Zero-copy variant: staging == NULL makes the kernel read/write
 * the pinned host pages directly through their device-mapped (UVA) address --
 * no staging buffer and no copy engine; NEO_ERR_UNSUPPORTED if the CPU-cache is
 * not device-mapped. */
NEO_API neo_status neo_kv_swap_out(neo_kv_pool* pool, int32_t n_pages, const int32_t* gpu_page_ids,
                                   const int32_t* host_page_ids, int32_t layer_begin, int32_t layer_end,
                                   void* staging, size_t staging_bytes, void* stream);
NEO_API neo_status neo_kv_swap_in(neo_kv_pool* pool, int32_t n_pages, const int32_t* host_page_ids,
                                  const int32_t* gpu_page_ids, int32_t layer_begin, int32_t layer_end,
                                  void* staging, size_t staging_bytes, void* stream);

/* Pipelining ("start PCIe transmission immediately after
 * each layer's KV value is computed").  When the staging holds at least two
 * pages' layer ranges (2 * neo_kv_swap_staging_bytes(pool, 1, ...)) and `stream`
 * is not being captured into a CUDA graph, a staged swap splits the staging
 * into two halves: gather/scatter kernels run on `stream`, the PCIe copies on a
 * copy stream the pool creates on first use (destroyed by
 * neo_kv_pool_destroy), and events order each half's producer and consumer.
 * The halves alternate across calls too, so a swap issued per layer overlaps
 * layer l+1's gather with layer l's D2H.  Otherwise (one-page staging, or graph
 * capture) the chunks run serially on `stream` with one buffer (after any
 * copy of an earlier pipelined call still reading the staging; under capture,
 * call neo_kv_swap_join and synchronise before capturing).  In both cases,
 * when `stream` passes the point where neo_kv_swap_out/in returned, the swap is
 * complete.
 *
 * neo_kv_swap_out_ex with flags = NEO_SWAP_DEFER_JOIN: on return `stream` is
 * ordered after the GATHER only -- the GPU pages may be freed or overwritten
 * once `stream` passes that point -- while the D2H copies may still be in
 * flight.  The host pages are complete once `stream` (or any stream) passes a
 * later neo_kv_swap_join(pool, stream), which makes `stream` wait for every
 * copy the pool's swaps have enqueued so far.  flags = 0 is neo_kv_swap_out.
 * Errors: NEO_ERR_INVALID_ARG for unknown flags or DEFER on a swap-in, or when
 * staged swaps of one pool are issued from two devices.
 *
 * Atomicity: every argument (ids, ranges, staging size and memory type, pinned
 * CPU-cache, a pending CUDA error) is validated before the first enqueue, so a
 * validation failure enqueues nothing.  NEO_ERR_CUDA from an enqueue itself
 * (after validation) means the CUDA context is failing; earlier chunks of that
 * call may have been enqueued. */
#define NEO_SWAP_DEFER_JOIN 1u
NEO_API neo_status neo_kv_swap_out_ex(neo_kv_pool* pool, int32_t n_pages, const int32_t* gpu_page_ids,
                                      const int32_t* host_page_ids, int32_t layer_begin, int32_t layer_end,
                                      void* staging, size_t staging_bytes, uint32_t flags, void* stream);
NEO_API neo_status neo_kv_swap_join(neo_kv_pool* pool, void* stream);

/* ------------------------------------------------------ CPU attention (NEXT-2)
 * Decode attention of CPU-requests over the CPU-cache -- NEO's PACPU:
 * the same result as neo_decode_attn (same definition, DESIGN c1-c4), computed
 * by host threads over the pinned host pages of layer `layer`:
 *   K_b[t] = host[host_block_table[b][t / P]][layer][0][g][t % P][:]  (V: [1]).
 * Partition: the (request, kv-head, page) blocks are dealt to the
 * threads in equal contiguous ranges; each thread's run of one (request,
 * kv-head) yields a partial (m, l, acc) and the partials of a request are merged
 * in block order.  AVX-512 within a core when the CPU has it.
 *   q, out           HOST [batch][num_q_heads][D] bf16.
 *   host_block_table HOST [batch][max_blocks] int32 CPU-cache page ids.
 *   seq_lens         HOST [batch] int32.
 *   num_threads      0 = all hardware threads.
 * Synchronous (returns when out is written).  Results are deterministic for a
 * fixed (inputs, num_threads); different thread counts round differently. */
NEO_API neo_status neo_cpu_decode_attn(const neo_kv_pool* pool, int32_t layer, const void* q,
                                       const int32_t* host_block_table, int32_t max_blocks, const int32_t* seq_lens,
                                       void* out, int32_t batch, int32_t num_q_heads, float scale,
                                       int32_t num_threads);

/* ------------------------------------------------- scheduler (NEXT-4)
 * NEO's load-aware scheduler for one iteration.  Cost model
 * (P:271-279), all times per layer in seconds, tables interpolated linearly
 * (extrapolated linearly, clamped >= 0, 0 for an empty sub-batch):
 *   T_l  = lin(tokens of the sub-batch: 1 per decoding request + prompt tokens)
 *   T_ga0 = gdec(sum over batch-0's GPU decoding requests of ctx+1)
 *           + sum over prefills of (gpre_a t^2 + gpre_b t)
 *   T_ca = cdec(sum over the sub-batch's CPU decoding requests of ctx+1)
 *   T    = T_prl + max(L (max{T_l0, T_ca1} + max{T_l1 + T_ga0, T_ca0}), T_swap) + T_pol
 *   T_swap = pages moved * P * kv_bytes_per_token_layer * L / pcie_bytes_per_s
 * Six steps: (1) empty batch-0 / batch-1; (2) every GPU decoding
 * request into batch-0, LIFO swap-out until its new KV fits, else FIFO swap-in
 * while free pages stay > 0; (3) FIFO prefills into batch-0 within
 * max_batch_tokens, KV on the GPU or marked for swap-out; (4) FIFO CPU decoding
 * requests into batch-1, else batch-0, keeping T_ca1 <= T_l0 and
 * T_ca0 <= T_l1 + T_ga0, else skipped; (5) swap-out prefills dropped from the
 * tail while the inequalities hold; (6) the two-batch plan is kept iff its x/T
 * beats the GPU-only plan (batch-0 without step 4's requests).  Readings:
 * DESIGN.md s1-s8.  Pure host function; deterministic. */
typedef struct {
  int32_t num_layers;                    /* L */
  double t_pre_layer_s, t_post_layer_s;  /* T_prl, T_pol */
  const double* lin_tokens;              /* linear stage table: tokens -> s/layer */
  const double* lin_s;
  int32_t lin_n;
  const double* gdec_tokens;             /* GPU decode attention: KV tokens -> s/layer */
  const double* gdec_s;
  int32_t gdec_n;
  double gpre_a, gpre_b;                 /* GPU prefill attention: a t^2 + b t s/layer */
  const double* cdec_tokens;             /* CPU decode attention: KV tokens -> s/layer */
  const double* cdec_s;
  int32_t cdec_n;
  int32_t page_size;
  int64_t max_batch_tokens;
  double pcie_bytes_per_s, kv_bytes_per_token_layer;
} neo_cost_model;

enum { NEO_REQ_WAITING = 0, NEO_REQ_GPU_DECODE = 1, NEO_REQ_CPU_DECODE = 2 };

typedef struct {
  int64_t id;
  int32_t kind; /* NEO_REQ_*; the array order is the queue order */
  int32_t ctx;  /* KV tokens held (decoding) or prompt tokens (waiting) */
} neo_sched_request;

typedef struct {
  int32_t two_batch; /* 1 = asymmetric pipelining plan, 0 = GPU-only */
  int32_t x;         /* requests producing a token this iteration */
  int32_t n_batch0, n_batch1, n_swap_out, n_swap_in;
  double t_iter, t_l0, t_l1, t_ga0, t_ca0, t_ca1;
} neo_sched_plan;

/* reqs[n]; batch0/batch1/swap_out/swap_in: caller arrays of n ids each, filled
 * with the plan (counts in *plan).  gpu/cpu_free_pages: free pages of the two
 * caches (neo_kv_free_count). */
NEO_API neo_status neo_schedule(const neo_cost_model* model, const neo_sched_request* reqs, int32_t n,
                                int64_t gpu_free_pages, int64_t cpu_free_pages, int64_t* batch0, int64_t* batch1,
                                int64_t* swap_out, int64_t* swap_in, neo_sched_plan* plan);

/* Staging bytes that let a swap of n_pages over the layer range run in one chunk. */
NEO_API neo_status neo_kv_swap_staging_bytes(const neo_kv_pool* pool, int32_t n_pages, int32_t layer_begin,
                                             int32_t layer_end, size_t* bytes);

#ifdef __cplusplus
}
#endif

#endif /* NEO_H_ */
