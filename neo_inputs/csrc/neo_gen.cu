// Device side of the seeded input generator (see neo_inputs/__init__.py for the
// recipe).  Holds NO attention arithmetic: it writes bit patterns into caller
// buffers in the pool layout the C ABI documents (include/neo.h), so the bench
// and the full-size parity tests can build tens of GB of KV on the GPU instead
// of pushing it over PCIe.  A GPU test checks these bits against the host
// generator element by element.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kTStride = 1ull << 17;

__host__ __device__ inline uint64_t splitmix64(uint64_t z) {
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u = __float_as_uint(f);
  uint32_t lsb = (u >> 16) & 1u;
  return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

__device__ inline float bf16_to_f32(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

__device__ inline uint16_t counter_bits(uint64_t seed, uint32_t tid, uint64_t index) {
  uint64_t x = splitmix64(seed ^ ((uint64_t)tid << 40) ^ index);
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += (int64_t)((x >> (16 * i)) & 0xFFFFull);
  s -= 131070;
  float f = (float)s * (1.0f / 32768.0f);
  return f32_to_bf16_rne(f);
}

__device__ inline uint16_t q_value(uint64_t seed, int layer, int64_t b, int hq_total, int h, int d,
                                   int dim, int variant) {
  uint64_t idx = ((uint64_t)b * (uint64_t)hq_total + (uint64_t)h) * (uint64_t)d + (uint64_t)dim;
  uint16_t bits = counter_bits(seed, (uint32_t)(1 + 8 * layer), idx);
  if (variant & 1) bits = f32_to_bf16_rne(bf16_to_f32(bits) * 8.0f);
  return bits;
}

struct FillKV {
  uint16_t* k;
  uint16_t* v;
  int64_t page_stride;
  const int32_t* block_table;
  const int32_t* seq_lens;
  int32_t max_blocks, batch, b_offset, hkv, g_offset, hkv_total, hq_total, d, page_size;
  uint64_t seed;
  int32_t layer, variant, tail_mode;
};

// grid: (max_blocks, batch); block: 256 threads; one page of one request per CTA,
// all local heads, K and V.
__global__ void fill_kv_kernel(FillKV p) {
  const int b = blockIdx.y;
  const int page = blockIdx.x;
  const int ctx = p.seq_lens[b];
  const int npages = (ctx + p.page_size - 1) / p.page_size;
  if (page >= npages) return;
  const int64_t pid = p.block_table[(int64_t)b * p.max_blocks + page];
  const int64_t gb = (int64_t)b + p.b_offset;
  const int per_page = p.hkv * p.page_size * p.d;
  const int group = p.hq_total / p.hkv_total;
  for (int e = threadIdx.x; e < per_page; e += blockDim.x) {
    const int dim = e % p.d;
    const int slot = (e / p.d) % p.page_size;
    const int gl = e / (p.d * p.page_size);
    const int g = gl + p.g_offset;
    const int64_t t = (int64_t)page * p.page_size + slot;
    uint16_t kb, vb;
    if (t >= ctx) {
      if (p.tail_mode == 1) { kb = vb = 0x7FC0; }      // NaN poison
      else if (p.tail_mode == 2) { kb = vb = 0; }
      else {
        uint64_t idx = (((uint64_t)gb * kTStride + (uint64_t)t) * (uint64_t)p.hkv_total + g) * p.d + dim;
        kb = counter_bits(p.seed, (uint32_t)(2 + 8 * p.layer), idx);
        vb = counter_bits(p.seed, (uint32_t)(3 + 8 * p.layer), idx);
      }
    } else {
      uint64_t idx = (((uint64_t)gb * kTStride + (uint64_t)t) * (uint64_t)p.hkv_total + g) * p.d + dim;
      kb = counter_bits(p.seed, (uint32_t)(2 + 8 * p.layer), idx);
      vb = counter_bits(p.seed, (uint32_t)(3 + 8 * p.layer), idx);
      if ((p.variant & 2) && t == 0) {
        int64_t tot = 0;
        for (int r = 0; r < group; ++r) {
          uint16_t qb = q_value(p.seed, p.layer, gb, p.hq_total, g * group + r, p.d, dim, 0);
          tot += (int64_t)llrint((double)bf16_to_f32(qb) * 4194304.0);
        }
        kb = tot >= 0 ? 0x4080 : 0xC080;
      }
    }
    const int64_t off = pid * p.page_stride + (int64_t)gl * p.page_size * p.d + (int64_t)slot * p.d + dim;
    p.k[off] = kb;
    p.v[off] = vb;
  }
}

__global__ void fill_q_kernel(uint16_t* q, int batch, int b_offset, int hq, int h_offset,
                              int hq_total, int d, uint64_t seed, int layer, int variant) {
  int64_t n = (int64_t)batch * hq * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int dim = (int)(e % d);
    int h = (int)((e / d) % hq);
    int64_t b = e / ((int64_t)d * hq);
    q[e] = q_value(seed, layer, b + b_offset, hq_total, h + h_offset, d, dim, variant);
  }
}

__global__ void values_kernel(uint64_t seed, uint32_t tid, const uint64_t* idx, int64_t n, uint16_t* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = counter_bits(seed, tid, idx[e]);
}

}  // namespace

#define GEN_API __attribute__((visibility("default")))

extern "C" {

GEN_API int neo_gen_fill_kv(void* k_pages, void* v_pages, int64_t page_stride, const int32_t* block_table,
                    int32_t max_blocks, const int32_t* seq_lens, int32_t batch, int32_t b_offset,
                    int32_t hkv, int32_t g_offset, int32_t hkv_total, int32_t hq_total, int32_t d,
                    int32_t page_size, uint64_t seed, int32_t layer, int32_t variant,
                    int32_t tail_mode, void* stream) {
  if (batch <= 0 || max_blocks <= 0) return 0;
  FillKV p{(uint16_t*)k_pages, (uint16_t*)v_pages, page_stride, block_table, seq_lens,
           max_blocks, batch, b_offset, hkv, g_offset, hkv_total, hq_total, d, page_size,
           seed, layer, variant, tail_mode};
  dim3 grid(max_blocks, batch);
  fill_kv_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(p);
  return (int)cudaGetLastError();
}

GEN_API int neo_gen_fill_q(void* q, int32_t batch, int32_t b_offset, int32_t hq, int32_t h_offset,
                   int32_t hq_total, int32_t d, uint64_t seed, int32_t layer, int32_t variant,
                   void* stream) {
  if (batch <= 0) return 0;
  fill_q_kernel<<<1024, 256, 0, (cudaStream_t)stream>>>((uint16_t*)q, batch, b_offset, hq, h_offset,
                                                         hq_total, d, seed, layer, variant);
  return (int)cudaGetLastError();
}

GEN_API int neo_gen_values(uint64_t seed, uint32_t tid, const uint64_t* idx, int64_t n, uint16_t* out,
                   void* stream) {
  if (n <= 0) return 0;
  values_kernel<<<256, 256, 0, (cudaStream_t)stream>>>(seed, tid, idx, n, out);
  return (int)cudaGetLastError();
}

}  // extern "C"
