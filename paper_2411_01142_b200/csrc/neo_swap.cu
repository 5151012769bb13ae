// Page gather / scatter for KV swap between the GPU-cache and the CPU-cache
// (P:235 partial offloading, P:240 layer-wise swapping, P:285-288 swap steps).
// The PCIe transfer (cudaMemcpy2DAsync from/to pinned host pages) is issued by
// the host code in neo_host.cu; these kernels only pack the scattered GPU pages
// of one request into a contiguous device staging buffer and unpack them back.
// Pure bit copies: 16-byte vector loads/stores, one CTA per (page, layer, K|V)
// block (Hkv*P*D*2 bytes, 32 KiB for LLaMa-3.1-8B), streaming cache hints.
#include "neo_internal.cuh"

namespace neo {
namespace {

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream(uint4* p, const uint4& v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

struct CopyArgs {
  const uint16_t* gpu_src;
  uint16_t* gpu_dst;
  const uint16_t* stg_src;
  uint16_t* stg_dst;
  int64_t num_gpu_pages, page_elems;
  int32_t n, l0, nl;
};

// grid (n pages, nl layers * 2); staging block index ((i * nl) + (l - l0)) * 2 + kv
template <bool kGather>
__global__ void __launch_bounds__(256) swap_copy_kernel(const CopyArgs a, const SwapBatch ids) {
  const int i = blockIdx.x;
  const int lk = blockIdx.y;  // (l - l0) * 2 + kv
  const int l = a.l0 + (lk >> 1), kv = lk & 1;
  const int64_t gpu_block = (static_cast<int64_t>(l) * 2 + kv) * a.num_gpu_pages + ids.ids[i];
  const int64_t stg_block = static_cast<int64_t>(i) * a.nl * 2 + lk;
  const int64_t nvec = a.page_elems / 8;
  if (kGather) {
    const uint4* src = reinterpret_cast<const uint4*>(a.gpu_src + gpu_block * a.page_elems);
    uint4* dst = reinterpret_cast<uint4*>(a.stg_dst + stg_block * a.page_elems);
    for (int64_t e = threadIdx.x; e < nvec; e += blockDim.x) st_stream(dst + e, ld_stream(src + e));
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(a.stg_src + stg_block * a.page_elems);
    uint4* dst = reinterpret_cast<uint4*>(a.gpu_dst + gpu_block * a.page_elems);
    for (int64_t e = threadIdx.x; e < nvec; e += blockDim.x) st_stream(dst + e, ld_stream(src + e));
  }
}

struct ZcArgs {
  uint16_t* gpu;
  uint16_t* host;
  int64_t num_gpu_pages, page_elems;
  int32_t num_layers, l0;
};

// grid (n pages, nl layers * 2): one (page, layer, K|V) block per CTA, moved
// between GPU-cache page gpu[i] and CPU-cache page host[i] over PCIe by SM
// loads/stores on the host page's mapped address.
template <bool kToHost>
__global__ void __launch_bounds__(256) zero_copy_kernel(const ZcArgs a, const SwapPairs ids) {
  const int i = blockIdx.x;
  const int l = a.l0 + (blockIdx.y >> 1), kv = blockIdx.y & 1;
  uint16_t* g = a.gpu + ((static_cast<int64_t>(l) * 2 + kv) * a.num_gpu_pages + ids.gpu[i]) * a.page_elems;
  uint16_t* h = a.host + ((static_cast<int64_t>(ids.host[i]) * a.num_layers + l) * 2 + kv) * a.page_elems;
  const int64_t nvec = a.page_elems / 8;
  if (kToHost) {
    for (int64_t e = threadIdx.x; e < nvec; e += blockDim.x)
      st_stream(reinterpret_cast<uint4*>(h) + e, ld_stream(reinterpret_cast<const uint4*>(g) + e));
  } else {
    for (int64_t e = threadIdx.x; e < nvec; e += blockDim.x)
      st_stream(reinterpret_cast<uint4*>(g) + e, ld_stream(reinterpret_cast<const uint4*>(h) + e));
  }
}

struct AppendArgs {
  uint16_t* k;
  uint16_t* v;
  const uint16_t* k_new;
  const uint16_t* v_new;
  const int32_t* block_table;
  const int32_t* seq_lens;
  int64_t page_stride;
  int32_t max_blocks, hkv, page_size;
};

// grid (batch), block 256: request b's new token, all kv-heads, K and V; 16-byte copies.
__global__ void __launch_bounds__(256) append_kernel(const AppendArgs a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int b = blockIdx.x;
  const int n = a.seq_lens[b];
  if (n <= 0) return;
  const int t = n - 1;
  const int64_t pid = a.block_table[static_cast<int64_t>(b) * a.max_blocks + t / a.page_size];
  const int slot = t % a.page_size;
  const int nvec = a.hkv * (kHeadDim / 8);  // 16-byte vectors per K (or V) row set
  for (int e = threadIdx.x; e < 2 * nvec; e += blockDim.x) {
    const int kv = e >= nvec;
    const int i = kv ? e - nvec : e;
    const int g = i / (kHeadDim / 8), w = i % (kHeadDim / 8);
    const uint4* src = reinterpret_cast<const uint4*>((kv ? a.v_new : a.k_new) +
                                                      (static_cast<int64_t>(b) * a.hkv + g) * kHeadDim) + w;
    uint4* dst = reinterpret_cast<uint4*>((kv ? a.v : a.k) + pid * a.page_stride +
                                          (static_cast<int64_t>(g) * a.page_size + slot) * kHeadDim) + w;
    *dst = *src;
  }
}

struct RopeArgs {
  uint16_t* q;
  const float* inv_freq;     // NULL: no rotation (plain multi-token append)
  uint16_t* k;
  uint16_t* v;
  const uint16_t* k_new;
  const uint16_t* v_new;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const int32_t* q_offsets;  // [batch + 1]; NULL: token j is request j's single new token
  int64_t page_stride;
  int32_t batch, max_blocks, hq, hkv, page_size;
};

__device__ __forceinline__ uint16_t f2bf(float f) {
  const uint32_t u = __float_as_uint(f);
  return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}
__device__ __forceinline__ float lo_f(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_f(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  return static_cast<uint32_t>(f2bf(lo)) | (static_cast<uint32_t>(f2bf(hi)) << 16);
}

// grid (tokens), block 128: one packed token j of request b at position t.
// sin/cos of theta_i = t * inv_freq[i] (fp64) are computed once per token into
// shared memory; then work item (row, oct) rotates the 8 dim pairs
// (8 oct + e, 8 oct + e + D/2) of one head row with two 16-byte loads / stores.
// Rows 0..Hq-1 are q heads (rotated in place), Hq..Hq+Hkv-1 the new k heads
// (rotated into the page slot), then the v heads (copied).
__global__ void __launch_bounds__(128) rope_append_kernel(const RopeArgs a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int kHalf = kHeadDim / 2;
  __shared__ float cs[kHalf], sn[kHalf];
  const int j = blockIdx.x;
  int b = j, n_q = 1, i_q = 0;
  if (a.q_offsets) {                      // request of packed token j: last b with q_offsets[b] <= j
    int lo = 0, hi = a.batch - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.q_offsets[mid] <= j) lo = mid;
      else hi = mid - 1;
    }
    b = lo;
    n_q = a.q_offsets[b + 1] - a.q_offsets[b];
    i_q = j - a.q_offsets[b];
  }
  const int n = a.seq_lens[b];
  if (n <= 0 || i_q >= n_q) return;
  const int t = n - n_q + i_q;
  const bool rope = a.inv_freq != nullptr;
  if (rope) {
    for (int i = threadIdx.x; i < kHalf; i += blockDim.x) {
      double sd, cd;
      sincos(static_cast<double>(t) * static_cast<double>(a.inv_freq[i]), &sd, &cd);
      cs[i] = static_cast<float>(cd);
      sn[i] = static_cast<float>(sd);
    }
    __syncthreads();
  }
  const int64_t pid = a.block_table[static_cast<int64_t>(b) * a.max_blocks + t / a.page_size];
  const int slot = t % a.page_size;
  const int q_rows = rope ? a.hq : 0;
  const int rows = q_rows + 2 * a.hkv;
  for (int e = threadIdx.x; e < rows * 8; e += blockDim.x) {
    const int row = e >> 3, oct = e & 7;
    const uint16_t* src;
    uint16_t* dst;
    bool rotate = rope;
    if (row < q_rows) {
      src = dst = a.q + (static_cast<int64_t>(j) * a.hq + row) * kHeadDim;
    } else {
      const int kv = row - q_rows >= a.hkv;
      const int g = row - q_rows - (kv ? a.hkv : 0);
      src = (kv ? a.v_new : a.k_new) + (static_cast<int64_t>(j) * a.hkv + g) * kHeadDim;
      dst = (kv ? a.v : a.k) + pid * a.page_stride + (static_cast<int64_t>(g) * a.page_size + slot) * kHeadDim;
      rotate = rope && !kv;
    }
    const uint4 x0 = *reinterpret_cast<const uint4*>(src + oct * 8);
    const uint4 x1 = *reinterpret_cast<const uint4*>(src + kHalf + oct * 8);
    if (!rotate) {
      *reinterpret_cast<uint4*>(dst + oct * 8) = x0;
      *reinterpret_cast<uint4*>(dst + kHalf + oct * 8) = x1;
      continue;
    }
    const uint32_t w0[4] = {x0.x, x0.y, x0.z, x0.w}, w1[4] = {x1.x, x1.y, x1.z, x1.w};
    uint32_t y0[4], y1[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int i = oct * 8 + 2 * w;
      const float a0 = lo_f(w0[w]), a1 = hi_f(w0[w]);   // x[i], x[i + 1]
      const float b0 = lo_f(w1[w]), b1 = hi_f(w1[w]);   // x[i + D/2], x[i + 1 + D/2]
      const float c0 = cs[i], s0 = sn[i], c1 = cs[i + 1], s1 = sn[i + 1];
      y0[w] = pack2(a0 * c0 - b0 * s0, a1 * c1 - b1 * s1);
      y1[w] = pack2(b0 * c0 + a0 * s0, b1 * c1 + a1 * s1);
    }
    *reinterpret_cast<uint4*>(dst + oct * 8) = make_uint4(y0[0], y0[1], y0[2], y0[3]);
    *reinterpret_cast<uint4*>(dst + kHalf + oct * 8) = make_uint4(y1[0], y1[1], y1[2], y1[3]);
  }
}

}  // namespace

neo_status launch_rope_append(uint16_t* q, int32_t hq, const float* inv_freq, uint16_t* k, uint16_t* v,
                              int64_t page_stride, const int32_t* block_table, int32_t max_blocks,
                              const int32_t* seq_lens, const int32_t* q_offsets, const uint16_t* k_new,
                              const uint16_t* v_new, int32_t batch, int32_t tokens, int32_t hkv, int32_t page_size,
                              cudaStream_t s) {
  RopeArgs a{q,         inv_freq, k,     v,          k_new, v_new, block_table, seq_lens,
             q_offsets, page_stride, batch, max_blocks, hq,    hkv,   page_size};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(tokens);
  cfg.blockDim = dim3(128);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, rope_append_kernel, a);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NEO_OK : cuda_fail(e, "rope append kernel launch");
}

neo_status launch_append(uint16_t* k, uint16_t* v, int64_t page_stride, const int32_t* block_table, int32_t max_blocks,
                         const int32_t* seq_lens, const uint16_t* k_new, const uint16_t* v_new, int32_t batch,
                         int32_t hkv, int32_t page_size, cudaStream_t s) {
  AppendArgs a{k, v, k_new, v_new, block_table, seq_lens, page_stride, max_blocks, hkv, page_size};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(batch);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, append_kernel, a);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NEO_OK : cuda_fail(e, "append kernel launch");
}

neo_status launch_zero_copy(bool to_host, uint16_t* gpu_base, uint16_t* host_dev, const SwapPairs& ids, int32_t n,
                            int64_t num_gpu_pages, int64_t page_elems, int32_t num_layers, int32_t l0, int32_t l1,
                            cudaStream_t s) {
  if (n <= 0) return NEO_OK;
  ZcArgs a{gpu_base, host_dev, num_gpu_pages, page_elems, num_layers, l0};
  dim3 grid(n, (l1 - l0) * 2);
  if (to_host) zero_copy_kernel<true><<<grid, 256, 0, s>>>(a, ids);
  else zero_copy_kernel<false><<<grid, 256, 0, s>>>(a, ids);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NEO_OK : cuda_fail(e, "zero-copy swap kernel launch");
}

neo_status launch_gather(const uint16_t* gpu_base, uint16_t* staging, const SwapBatch& ids, int32_t n,
                         int64_t num_gpu_pages, int64_t page_elems, int32_t l0, int32_t l1, cudaStream_t s) {
  if (n <= 0) return NEO_OK;
  CopyArgs a{gpu_base, nullptr, nullptr, staging, num_gpu_pages, page_elems, n, l0, l1 - l0};
  dim3 grid(n, (l1 - l0) * 2);
  swap_copy_kernel<true><<<grid, 256, 0, s>>>(a, ids);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NEO_OK : cuda_fail(e, "gather kernel launch");
}

neo_status launch_scatter(uint16_t* gpu_base, const uint16_t* staging, const SwapBatch& ids, int32_t n,
                          int64_t num_gpu_pages, int64_t page_elems, int32_t l0, int32_t l1, cudaStream_t s) {
  if (n <= 0) return NEO_OK;
  CopyArgs a{nullptr, gpu_base, staging, nullptr, num_gpu_pages, page_elems, n, l0, l1 - l0};
  dim3 grid(n, (l1 - l0) * 2);
  swap_copy_kernel<false><<<grid, 256, 0, s>>>(a, ids);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NEO_OK : cuda_fail(e, "scatter kernel launch");
}

}  // namespace neo
