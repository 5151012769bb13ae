// NEO's load-aware scheduler with its interpolated
// cost model: per iteration, a GPU-only schedule and a two-batch
// asymmetric-pipelining schedule are built with the paper's six steps and the
// one with the higher estimated throughput is returned.  Readings where the
// paper is silent: DESIGN.md s1-s8 (the plain-Python oracle in
// oracle/scheduler.py implements the same steps and is checked against this
// code decision by decision).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/neo.h"

namespace neo {
neo_status fail(neo_status st, const std::string& msg);
}

namespace {

struct Req {
  int64_t id;
  int32_t ctx;
};

struct Model {
  const neo_cost_model* m;

  static double interp(const double* xs, const double* ys, int n, double key) {
    if (key <= 0) return 0.0;
    int i;
    if (key <= xs[0]) i = 0;
    else if (key >= xs[n - 1]) i = n - 2;
    else {
      i = 0;
      for (int k = 0; k < n - 1; ++k)
        if (xs[k] <= key) i = k;
    }
    const double x0 = xs[i], x1 = xs[i + 1], y0 = ys[i], y1 = ys[i + 1];
    return std::max(0.0, y0 + (y1 - y0) * (key - x0) / (x1 - x0));
  }
  double lin(int64_t t) const { return interp(m->lin_tokens, m->lin_s, m->lin_n, static_cast<double>(t)); }
  double gdec(int64_t t) const { return interp(m->gdec_tokens, m->gdec_s, m->gdec_n, static_cast<double>(t)); }
  double cdec(int64_t t) const { return interp(m->cdec_tokens, m->cdec_s, m->cdec_n, static_cast<double>(t)); }

  // P:273-275 plus the pre/post-layer constants and un-hidden swap time (DESIGN s7)
  double iteration_time(double t_l0, double t_l1, double t_ga0, double t_ca0, double t_ca1, double t_swap) const {
    const double t_tr = m->num_layers * (std::max(t_l0, t_ca1) + std::max(t_l1 + t_ga0, t_ca0));
    return m->t_pre_layer_s + std::max(t_tr, t_swap) + m->t_post_layer_s;
  }
};

struct State {
  const Model* md;
  std::vector<Req> gpu_dec, prefill, cpu0, cpu1;

  // tokens of batch-0's linear stage: one per decoding request plus the prompts
  int64_t tokens0() const {
    int64_t p = 0;
    for (const Req& r : prefill) p += r.ctx;
    return static_cast<int64_t>(gpu_dec.size()) + p + static_cast<int64_t>(cpu0.size());
  }
  double t_l0() const { return md->lin(tokens0()); }
  double t_l1() const { return md->lin(static_cast<int64_t>(cpu1.size())); }
  double t_ga0() const {
    int64_t kv = 0;
    for (const Req& r : gpu_dec) kv += r.ctx + 1;
    double s = 0.0;
    for (const Req& r : prefill)
      s += md->m->gpre_a * r.ctx * r.ctx + md->m->gpre_b * r.ctx;
    return md->gdec(kv) + s;
  }
  static int64_t kv_of(const std::vector<Req>& v) {
    int64_t kv = 0;
    for (const Req& r : v) kv += r.ctx + 1;
    return kv;
  }
  double t_ca0() const { return md->cdec(kv_of(cpu0)); }
  double t_ca1() const { return md->cdec(kv_of(cpu1)); }
  // T_l0 >= T_ca1 and T_l1 + T_ga0 >= T_ca0
  bool balanced() const { return t_ca1() <= t_l0() && t_ca0() <= t_l1() + t_ga0(); }
};

inline int64_t pages(int64_t n, int64_t P) { return (n + P - 1) / P; }

bool table_ok(const double* xs, const double* ys, int n) {
  if (!xs || !ys || n < 2) return false;
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(xs[i]) || !std::isfinite(ys[i]) || ys[i] < 0 || (i && xs[i] <= xs[i - 1])) return false;
  return true;
}

}  // namespace

extern "C" NEO_API neo_status neo_schedule(const neo_cost_model* m, const neo_sched_request* reqs, int32_t n,
                                           int64_t gpu_free, int64_t cpu_free, int64_t* batch0, int64_t* batch1,
                                           int64_t* swap_out, int64_t* swap_in, neo_sched_plan* plan) {
  if (!m || !plan || n < 0 || (n > 0 && (!reqs || !batch0 || !batch1 || !swap_out || !swap_in)))
    return neo::fail(NEO_ERR_INVALID_ARG, "NULL argument");
  if (m->num_layers < 1 || m->page_size < 1 || !(m->pcie_bytes_per_s > 0) || m->max_batch_tokens < 0 ||
      !table_ok(m->lin_tokens, m->lin_s, m->lin_n) || !table_ok(m->gdec_tokens, m->gdec_s, m->gdec_n) ||
      !table_ok(m->cdec_tokens, m->cdec_s, m->cdec_n))
    return neo::fail(NEO_ERR_INVALID_ARG,
                     "cost model: L, page_size, pcie > 0 and tables of >= 2 points with increasing keys required");
  if (gpu_free < 0 || cpu_free < 0) return neo::fail(NEO_ERR_INVALID_ARG, "free page counts must be >= 0");
  for (int32_t i = 0; i < n; ++i)
    if (reqs[i].kind < NEO_REQ_WAITING || reqs[i].kind > NEO_REQ_CPU_DECODE || reqs[i].ctx < 0)
      return neo::fail(NEO_ERR_INVALID_ARG, "request " + std::to_string(i) + ": bad kind or context length");

  const int64_t P = m->page_size;
  Model md{m};
  State st{&md, {}, {}, {}, {}};
  std::vector<Req> waiting, gdec, cdec;
  for (int32_t i = 0; i < n; ++i) {
    const Req r{reqs[i].id, reqs[i].ctx};
    if (reqs[i].kind == NEO_REQ_WAITING) waiting.push_back(r);
    else if (reqs[i].kind == NEO_REQ_GPU_DECODE) gdec.push_back(r);
    else cdec.push_back(r);
  }
  std::vector<int64_t> out_ids, in_ids;
  int64_t swap_pages = 0;
  auto grow = [P](const Req& r) { return pages(r.ctx + 1, P) - pages(r.ctx, P); };

  // Step 2: GPU decoding requests into batch-0; LIFO swap-out until the
  // new KV fits (DESIGN s2), else FIFO swap-in while space stays ample (s3).
  int64_t need = 0;
  for (const Req& r : gdec) need += grow(r);
  while (need > gpu_free && !gdec.empty()) {
    const Req v = gdec.back();
    gdec.pop_back();
    need -= grow(v);
    if (cpu_free < pages(v.ctx, P)) continue;  // cannot move it: sits out this iteration
    gpu_free += pages(v.ctx, P);
    cpu_free -= pages(v.ctx, P);
    swap_pages += pages(v.ctx, P);
    out_ids.push_back(v.id);
    cdec.push_back(v);
  }
  gpu_free -= need;
  if (out_ids.empty()) {
    size_t k = 0;
    for (; k < cdec.size(); ++k) {
      const Req& r = cdec[k];
      if (gpu_free - pages(r.ctx + 1, P) > 0) {
        gpu_free -= pages(r.ctx + 1, P);
        cpu_free += pages(r.ctx, P);
        swap_pages += pages(r.ctx, P);
        in_ids.push_back(r.id);
        gdec.push_back(r);
      } else {
        break;
      }
    }
    cdec.erase(cdec.begin(), cdec.begin() + static_cast<std::ptrdiff_t>(k));
  }
  st.gpu_dec = gdec;

  // Step 3: prefills into batch-0 while the token budget holds; KV on the
  // GPU if it fits, else marked for swap-out.
  std::unordered_set<int64_t> marked;
  for (const Req& w : waiting) {
    if (st.tokens0() + w.ctx > m->max_batch_tokens) break;
    const int64_t np = pages(w.ctx, P);
    if (gpu_free >= np) gpu_free -= np;
    else if (cpu_free >= np) {
      cpu_free -= np;
      marked.insert(w.id);
    } else {
      break;
    }
    st.prefill.push_back(w);
  }

  // Step 4: CPU decoding requests into batch-1 (preferred, s4) or batch-0
  // while the inequalities hold; others are skipped this iteration.
  for (const Req& r : cdec) {
    if (cpu_free < grow(r)) continue;
    st.cpu1.push_back(r);
    if (st.balanced()) {
      cpu_free -= grow(r);
      continue;
    }
    st.cpu1.pop_back();
    st.cpu0.push_back(r);
    if (st.balanced()) {
      cpu_free -= grow(r);
      continue;
    }
    st.cpu0.pop_back();
  }

  // Step 5: drop swap-out prefills from the tail while the inequalities hold.
  for (int64_t i = static_cast<int64_t>(st.prefill.size()) - 1; i >= 0; --i) {
    const Req w = st.prefill[i];
    if (!marked.count(w.id)) continue;
    st.prefill.erase(st.prefill.begin() + i);
    if (st.balanced()) {
      cpu_free += pages(w.ctx, P);
      marked.erase(w.id);
    } else {
      st.prefill.insert(st.prefill.begin() + i, w);
    }
  }
  for (const Req& w : st.prefill)
    if (marked.count(w.id)) {
      swap_pages += pages(w.ctx, P);
      out_ids.push_back(w.id);
    }
  const double t_swap = static_cast<double>(swap_pages * P) * m->kv_bytes_per_token_layer * m->num_layers /
                        m->pcie_bytes_per_s;

  // Step 6: GPU-only = batch-0 without step 4's CPU requests; keep the
  // higher estimated throughput x / T (DESIGN s1); ties go to GPU-only.
  const double t_l0 = st.t_l0(), t_l1 = st.t_l1(), t_ga0 = st.t_ga0(), t_ca0 = st.t_ca0(), t_ca1 = st.t_ca1();
  const int64_t x2 = static_cast<int64_t>(st.gpu_dec.size() + st.prefill.size() + st.cpu0.size() + st.cpu1.size());
  const double T2 = md.iteration_time(t_l0, t_l1, t_ga0, t_ca0, t_ca1, t_swap);
  const std::vector<Req> cpu0 = st.cpu0, cpu1 = st.cpu1;
  st.cpu0.clear();
  st.cpu1.clear();
  const double t_l0_g = st.t_l0();
  const int64_t x1 = static_cast<int64_t>(st.gpu_dec.size() + st.prefill.size());
  const double T1 = md.iteration_time(t_l0_g, 0.0, t_ga0, 0.0, 0.0, t_swap);
  const bool two = (!cpu0.empty() || !cpu1.empty()) && (x2 / T2 > (x1 ? x1 / T1 : 0.0));

  int32_t k0 = 0, k1 = 0;
  for (const Req& r : st.gpu_dec) batch0[k0++] = r.id;
  for (const Req& r : st.prefill) batch0[k0++] = r.id;
  if (two) {
    for (const Req& r : cpu0) batch0[k0++] = r.id;
    for (const Req& r : cpu1) batch1[k1++] = r.id;
  }
  for (size_t i = 0; i < out_ids.size(); ++i) swap_out[i] = out_ids[i];
  for (size_t i = 0; i < in_ids.size(); ++i) swap_in[i] = in_ids[i];
  plan->two_batch = two ? 1 : 0;
  plan->x = static_cast<int32_t>(two ? x2 : x1);
  plan->n_batch0 = k0;
  plan->n_batch1 = k1;
  plan->n_swap_out = static_cast<int32_t>(out_ids.size());
  plan->n_swap_in = static_cast<int32_t>(in_ids.size());
  plan->t_iter = two ? T2 : T1;
  plan->t_l0 = two ? t_l0 : t_l0_g;
  plan->t_l1 = two ? t_l1 : 0.0;
  plan->t_ga0 = t_ga0;
  plan->t_ca0 = two ? t_ca0 : 0.0;
  plan->t_ca1 = two ? t_ca1 : 0.0;
  return NEO_OK;
}
