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
  const float* inv_freq;
  uint16_t* k;
  uint16_t* v;
  const uint16_t* k_new;
  const uint16_t* v_new;
  const int32_t* block_table;
  const int32_t* seq_lens;
  int64_t page_stride;
  int32_t max_blocks, hq, hkv, page_size;
};

__device__ __forceinline__ float bf2f(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }
__device__ __forceinline__ uint16_t f2bf(float f) {
  const uint32_t u = __float_as_uint(f);
  return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

// grid (batch), block 256: thread = (head row, dim pair i); rows 0..Hq-1 are q
// heads (rotated in place), Hq..Hq+Hkv-1 the new k heads (rotated into the page),
// then the v heads (copied).
__global__ void __launch_bounds__(256) rope_append_kernel(const RopeArgs a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int b = blockIdx.x;
  const int n = a.seq_lens[b];
  if (n <= 0) return;
  const int t = n - 1;
  constexpr int kHalf = kHeadDim / 2;
  const int64_t pid = a.block_table[static_cast<int64_t>(b) * a.max_blocks + t / a.page_size];
  const int slot = t % a.page_size;
  const int rows = a.hq + 2 * a.hkv;
  for (int e = threadIdx.x; e < rows * kHalf; e += blockDim.x) {
    const int row = e / kHalf, i = e % kHalf;
    if (row >= a.hq + a.hkv) {                       // v: plain copy of the pair
      const int g = row - a.hq - a.hkv;
      const uint16_t* src = a.v_new + (static_cast<int64_t>(b) * a.hkv + g) * kHeadDim;
      uint16_t* dst = a.v + pid * a.page_stride + (static_cast<int64_t>(g) * a.page_size + slot) * kHeadDim;
      dst[i] = src[i];
      dst[i + kHalf] = src[i + kHalf];
      continue;
    }
    double sd, cd;
    sincos(static_cast<double>(t) * static_cast<double>(a.inv_freq[i]), &sd, &cd);
    const float s = static_cast<float>(sd), c = static_cast<float>(cd);
    uint16_t* src;
    uint16_t* dst;
    if (row < a.hq) {
      src = dst = a.q + (static_cast<int64_t>(b) * a.hq + row) * kHeadDim;
    } else {
      const int g = row - a.hq;
      src = const_cast<uint16_t*>(a.k_new) + (static_cast<int64_t>(b) * a.hkv + g) * kHeadDim;
      dst = a.k + pid * a.page_stride + (static_cast<int64_t>(g) * a.page_size + slot) * kHeadDim;
    }
    const float x0 = bf2f(src[i]), x1 = bf2f(src[i + kHalf]);
    dst[i] = f2bf(x0 * c - x1 * s);
    dst[i + kHalf] = f2bf(x1 * c + x0 * s);
  }
}

}  // namespace

neo_status launch_rope_append(uint16_t* q, int32_t hq, const float* inv_freq, uint16_t* k, uint16_t* v,
                              int64_t page_stride, const int32_t* block_table, int32_t max_blocks,
                              const int32_t* seq_lens, const uint16_t* k_new, const uint16_t* v_new, int32_t batch,
                              int32_t hkv, int32_t page_size, cudaStream_t s) {
  RopeArgs a{q, inv_freq, k, v, k_new, v_new, block_table, seq_lens, page_stride, max_blocks, hq, hkv, page_size};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(batch);
  cfg.blockDim = dim3(256);
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
