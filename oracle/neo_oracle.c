/*
 * oracle/neo_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of what NEO's GPU
 * hot path computes.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * table or helper with the CUDA library (paper_2411_01142_b200/csrc) and never
 * sees a block table or a page: K and V are UNPAGED per-request arrays.
 *
 * What it computes (the plain definition; NEO computes exact attention and only
 * moves where it runs -- P:64):
 *   attention / inference semantics     P:97-98, P:109-110 (Sec 2.1)
 *   decode attention reads the KV cache  P:122 (Sec 2.2)
 *   flash-decoding partition + aggregate P:307 (Sec 4), merge algebra
 *
 *   for request b, q-head h:   g   = floor(h / G),  G = Hq / Hkv     (reading c2)
 *     s_t = scale * sum_d q[h][d] * K[t][g][d]     t = 0 .. n-1        (reading c1, c3)
 *     m   = max_t s_t,   w_t = exp(s_t - m)
 *     out[h][:] = sum_t w_t * V[t][g][:] / sum_t w_t
 *
 * Inputs are bf16 bit patterns (uint16), widened EXACTLY to double.  All
 * arithmetic is double, scalar, in the order written above.  n = 0 yields a zero
 * row (reading c4).  Pins: tests/test_oracle_pins.py.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double bf16_to_double(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

/* One request.  q: [hq][d]; k, v: [n][hkv][d]; out: [hq][d].  Returns 0, or -1
 * on a shape error (hq not a positive multiple of hkv). */
int oracle_decode_attention(const uint16_t* q, const uint16_t* k, const uint16_t* v, int64_t n,
                            int hq, int hkv, int d, double scale, double* out) {
  if (hq <= 0 || hkv <= 0 || d <= 0 || hq % hkv != 0 || n < 0) return -1;
  const int G = hq / hkv;
  double* s = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!s) return -2;
  for (int h = 0; h < hq; ++h) {
    const int g = h / G;
    double* o = out + (size_t)h * d;
    for (int j = 0; j < d; ++j) o[j] = 0.0;
    if (n == 0) continue;
    /* scores */
    for (int64_t t = 0; t < n; ++t) {
      double acc = 0.0;
      for (int j = 0; j < d; ++j)
        acc += bf16_to_double(q[(size_t)h * d + j]) * bf16_to_double(k[((size_t)t * hkv + g) * d + j]);
      s[t] = scale * acc;
    }
    /* softmax */
    double m = s[0];
    for (int64_t t = 1; t < n; ++t)
      if (s[t] > m) m = s[t];
    double l = 0.0;
    for (int64_t t = 0; t < n; ++t) {
      s[t] = exp(s[t] - m);
      l += s[t];
    }
    /* weighted sum of V */
    for (int64_t t = 0; t < n; ++t) {
      const double w = s[t];
      for (int j = 0; j < d; ++j) o[j] += w * bf16_to_double(v[((size_t)t * hkv + g) * d + j]);
    }
    for (int j = 0; j < d; ++j) o[j] /= l;
  }
  free(s);
  return 0;
}

/* Softmax weights w[h][t] of the definition above (for the "weights sum to 1"
 * property). */
int oracle_softmax_weights(const uint16_t* q, const uint16_t* k, int64_t n, int hq, int hkv, int d,
                           double scale, double* w) {
  if (hq <= 0 || hkv <= 0 || hq % hkv != 0 || n <= 0) return -1;
  const int G = hq / hkv;
  for (int h = 0; h < hq; ++h) {
    const int g = h / G;
    double* s = w + (size_t)h * n;
    for (int64_t t = 0; t < n; ++t) {
      double acc = 0.0;
      for (int j = 0; j < d; ++j)
        acc += bf16_to_double(q[(size_t)h * d + j]) * bf16_to_double(k[((size_t)t * hkv + g) * d + j]);
      s[t] = scale * acc;
    }
    double m = s[0];
    for (int64_t t = 1; t < n; ++t)
      if (s[t] > m) m = s[t];
    double l = 0.0;
    for (int64_t t = 0; t < n; ++t) {
      s[t] = exp(s[t] - m);
      l += s[t];
    }
    for (int64_t t = 0; t < n; ++t) s[t] /= l;
  }
  return 0;
}

/* Flash-decoding task ("partition its computation into individual tasks";
 * S:468-471 statistics): for ONE q-head h over tokens [t0, t1) of its KV head,
 *   m = max s_t,  l = sum exp(s_t - m),  acc[:] = sum exp(s_t - m) V[t][g][:]. */
int oracle_partial(const uint16_t* q, const uint16_t* k, const uint16_t* v, int hq, int hkv, int d,
                   int h, int64_t t0, int64_t t1, double scale, double* m_out, double* l_out,
                   double* acc) {
  if (hq <= 0 || hkv <= 0 || hq % hkv != 0 || t1 <= t0 || h < 0 || h >= hq) return -1;
  const int g = h / (hq / hkv);
  const int64_t n = t1 - t0;
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  if (!s) return -2;
  for (int64_t t = t0; t < t1; ++t) {
    double a = 0.0;
    for (int j = 0; j < d; ++j)
      a += bf16_to_double(q[(size_t)h * d + j]) * bf16_to_double(k[((size_t)t * hkv + g) * d + j]);
    s[t - t0] = scale * a;
  }
  double m = s[0];
  for (int64_t i = 1; i < n; ++i)
    if (s[i] > m) m = s[i];
  double l = 0.0;
  for (int j = 0; j < d; ++j) acc[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double w = exp(s[i] - m);
    l += w;
    for (int j = 0; j < d; ++j) acc[j] += w * bf16_to_double(v[((size_t)(t0 + i) * hkv + g) * d + j]);
  }
  *m_out = m;
  *l_out = l;
  free(s);
  return 0;
}

/* Aggregate partial outputs ("aggregate the partial outputs"):
 *   M = max_j m_j,  L = sum_j l_j e^{m_j - M},  out = sum_j acc_j e^{m_j - M} / L. */
int oracle_merge(int n_parts, const double* m, const double* l, const double* acc, int d, double* out) {
  if (n_parts <= 0) return -1;
  double M = m[0];
  for (int j = 1; j < n_parts; ++j)
    if (m[j] > M) M = m[j];
  double L = 0.0;
  for (int j = 0; j < d; ++j) out[j] = 0.0;
  for (int p = 0; p < n_parts; ++p) {
    const double c = exp(m[p] - M);
    L += l[p] * c;
    for (int j = 0; j < d; ++j) out[j] += acc[(size_t)p * d + j] * c;
  }
  for (int j = 0; j < d; ++j) out[j] /= L;
  return 0;
}

/* ---- batch driver: std threads over requests (cpu_baseline timing only) ---- */
typedef struct {
  const uint16_t *q, *k, *v;
  const int64_t* offsets;
  int64_t b0, b1;
  int hq, hkv, d;
  double scale;
  double* out;
  int rc;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  for (int64_t b = j->b0; b < j->b1 && j->rc == 0; ++b) {
    const int64_t off = j->offsets[b], n = j->offsets[b + 1] - off;
    j->rc = oracle_decode_attention(j->q + (size_t)b * j->hq * j->d, j->k + (size_t)off * j->hkv * j->d,
                                    j->v + (size_t)off * j->hkv * j->d, n, j->hq, j->hkv, j->d, j->scale,
                                    j->out + (size_t)b * j->hq * j->d);
  }
  return NULL;
}

/* q: [B][hq][d]; k, v: packed [sum n_b][hkv][d]; offsets: [B+1] token offsets. */
int oracle_decode_attention_batch(const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                  const int64_t* offsets, int64_t batch, int hq, int hkv, int d,
                                  double scale, double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  int rc = 0;
  /* contiguous runs of ceil(batch / nthreads) requests per thread */
  int64_t per = (batch + nthreads - 1) / nthreads;
  int started = 0;
  for (int i = 0; i < nthreads; ++i) {
    int64_t b0 = i * per, b1 = b0 + per < batch ? b0 + per : batch;
    if (b0 >= b1) break;
    jobs[i] = (job_t){q, k, v, offsets, b0, b1, hq, hkv, d, scale, out, 0};
    if (pthread_create(&th[i], NULL, run_job, &jobs[i]) != 0) {
      rc = -3;
      break;
    }
    ++started;
  }
  for (int i = 0; i < started; ++i) {
    pthread_join(th[i], NULL);
    if (jobs[i].rc) rc = jobs[i].rc;
  }
  return rc;
}

/* ---------------------------------------------------------------- prefill
 * Causal attention of a prompt chunk (the prefill half of batch-0, P:237-239;
 * SURVEY NEXT-3).  The request holds n KV tokens, the last n_q of which belong to
 * the n_q query rows being prefilled; query row i sits at position n - n_q + i
 * and attends to tokens 0 .. n - n_q + i (causal, P:97-98 autoregression: a
 * token never sees later ones).  Written as the decode definition above applied
 * row by row to the visible prefix.  q: [n_q][hq][d]; k, v: [n][hkv][d];
 * out: [n_q][hq][d].  Rows are dealt to threads round-robin. */
typedef struct {
  const uint16_t *q, *k, *v;
  int64_t n, n_q;
  int hq, hkv, d, tid, nthreads;
  double scale;
  double* out;
  int rc;
} prefill_job_t;

static void* run_prefill(void* arg) {
  prefill_job_t* j = (prefill_job_t*)arg;
  for (int64_t i = j->tid; i < j->n_q && j->rc == 0; i += j->nthreads)
    j->rc = oracle_decode_attention(j->q + (size_t)i * j->hq * j->d, j->k, j->v, j->n - j->n_q + i + 1, j->hq,
                                    j->hkv, j->d, j->scale, j->out + (size_t)i * j->hq * j->d);
  return NULL;
}

int oracle_prefill_attention(const uint16_t* q, const uint16_t* k, const uint16_t* v, int64_t n, int64_t n_q,
                             int hq, int hkv, int d, double scale, double* out, int nthreads) {
  if (n_q < 0 || n_q > n) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  prefill_job_t jobs[256];
  int rc = 0, started = 0;
  for (int i = 0; i < nthreads; ++i) {
    jobs[i] = (prefill_job_t){q, k, v, n, n_q, hq, hkv, d, i, nthreads, scale, out, 0};
    if (pthread_create(&th[i], NULL, run_prefill, &jobs[i]) != 0) {
      rc = -3;
      break;
    }
    ++started;
  }
  for (int i = 0; i < started; ++i) {
    pthread_join(th[i], NULL);
    if (jobs[i].rc) rc = jobs[i].rc;
  }
  return rc;
}
