/* Host C implementation of the seeded input generator (recipe in
 * neo_inputs/__init__.py).  Bit-identical to the numpy and CUDA versions
 * (tests/test_inputs.py, tests/test_gpu_inputs.py).  Input construction only:
 * no attention arithmetic. */
#include <math.h>
#include <stdint.h>
#include <string.h>

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint16_t f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

static float bf16_to_f32(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint16_t counter_bits(uint64_t seed, uint32_t tid, uint64_t index) {
  uint64_t x = splitmix64(seed ^ ((uint64_t)tid << 40) ^ index);
  int64_t s = 0;
  for (int i = 0; i < 4; ++i) s += (int64_t)((x >> (16 * i)) & 0xFFFFull);
  s -= 131070;
  return f32_to_bf16((float)s * (1.0f / 32768.0f));
}

static uint16_t q_value(uint64_t seed, int layer, int64_t b, int hq_total, int h, int d, int dim, int variant) {
  uint64_t idx = ((uint64_t)b * (uint64_t)hq_total + (uint64_t)h) * (uint64_t)d + (uint64_t)dim;
  uint16_t bits = counter_bits(seed, (uint32_t)(1 + 8 * layer), idx);
  if (variant & 1) bits = f32_to_bf16(bf16_to_f32(bits) * 8.0f);
  return bits;
}

/* out[n_b][n_h][d] for global requests b_ids, global heads h_begin.. */
void gen_q_bits(uint64_t seed, int layer, const int64_t* b_ids, int n_b, int hq_total, int h_begin, int n_h, int d,
                int variant, uint16_t* out) {
  for (int i = 0; i < n_b; ++i)
    for (int h = 0; h < n_h; ++h)
      for (int j = 0; j < d; ++j)
        out[((size_t)i * n_h + h) * d + j] = q_value(seed, layer, b_ids[i], hq_total, h_begin + h, d, j, variant);
}

/* out[t1-t0][n_g][d]: K (kind 2) or V (kind 3) of request b, kv heads g_begin.. */
void gen_kv_bits(uint64_t seed, int layer, int kind, int64_t b, int64_t t0, int64_t t1, int hkv_total, int g_begin,
                 int n_g, int d, int variant, int hq_total, uint16_t* out) {
  const uint32_t tid = (uint32_t)(kind + 8 * layer);
  for (int64_t t = t0; t < t1; ++t)
    for (int gi = 0; gi < n_g; ++gi) {
      const int g = g_begin + gi;
      uint16_t* o = out + ((size_t)(t - t0) * n_g + gi) * d;
      if (kind == 2 && (variant & 2) && t == 0) {
        const int group = hq_total / hkv_total;
        for (int j = 0; j < d; ++j) {
          int64_t tot = 0;
          for (int r = 0; r < group; ++r)
            tot += (int64_t)llrint((double)bf16_to_f32(q_value(seed, layer, b, hq_total, g * group + r, d, j, 0)) *
                                   4194304.0);
          o[j] = tot >= 0 ? 0x4080 : 0xC080;
        }
        continue;
      }
      for (int j = 0; j < d; ++j) {
        uint64_t idx = (((uint64_t)b * (1ull << 17) + (uint64_t)t) * (uint64_t)hkv_total + (uint64_t)g) * d + j;
        o[j] = counter_bits(seed, tid, idx);
      }
    }
}
