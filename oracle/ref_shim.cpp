// ORACLE — test infrastructure only.  extern "C" wrappers around the UNMODIFIED
// reference library (compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libhybridep_ref.so).  Used by tests/ and oracle/gen_golden.py to pin
// the CPU restatement (oracle/moe_oracle.c) and the device codec against the
// reference's own outputs.  Never linked into the product.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "hybridep/perfmodel.hpp"
#include "hybridep/plan.hpp"
#include "hybridep/simcore.hpp"
#include "hybridep/sparsecomp.hpp"
#include "hybridep/topology.hpp"

using namespace hybridep;

namespace {

topo::ClusterSpec cluster(const int64_t* sf, const int64_t* sed, int L) {
  topo::ClusterSpec c;
  for (int i = 0; i < L; ++i) c.levels.push_back({sf[i], sed[i], 1e9});
  return c;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::domain_error&) {
    return 1;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (const std::runtime_error&) {
    return 3;
  }
}

sr::ExpertWeights expert_of(const float* flat, int64_t h, int64_t m) {
  sr::ExpertWeights e;
  e.w_up = sr::Matrix(h, m);
  e.w_down = sr::Matrix(m, h);
  std::memcpy(e.w_up.data.data(), flat, sizeof(float) * h * m);
  std::memcpy(e.w_down.data.data(), flat + h * m, sizeof(float) * h * m);
  return e;
}

}  // namespace

extern "C" {

int ref_topology(const int64_t* sf, const int64_t* sed, int L, int8_t* lvl, uint8_t* typ) {
  return guard([&] {
    const topo::CommTopology t(cluster(sf, sed, L));
    const int64_t G = t.gpus();
    for (int64_t m = 0; m < G; ++m)
      for (int64_t n = 0; n < G; ++n) {
        if (m == n) { lvl[m * G + n] = -1; typ[m * G + n] = 0; continue; }
        const auto pc = t.classify(m, n);
        lvl[m * G + n] = static_cast<int8_t>(pc.level);
        typ[m * G + n] = static_cast<uint8_t>(pc.type);
      }
  });
}

int ref_renumber(const int64_t* sf, int L, int64_t m, int64_t* x) {
  std::vector<int64_t> sed(L, 1);
  return guard([&] {
    const auto v = topo::renumber(m, cluster(sf, sed.data(), L));
    std::copy(v.begin(), v.end(), x);
  });
}

int ref_global_index(const int64_t* sf, int L, const int64_t* x, int nx, int64_t* m) {
  std::vector<int64_t> sed(L, 1);
  return guard([&] { *m = topo::global_index(topo::MultiIndex(x, x + nx), cluster(sf, sed.data(), L)); });
}

int ref_comm_type(const int64_t* sf, const int64_t* sed, int L, int64_t m, int64_t n, int level, int* t) {
  return guard([&] { *t = static_cast<int>(topo::comm_type(m, n, level, cluster(sf, sed, L))); });
}

int ref_level_frequency(const int64_t* sf, const int64_t* sed, int L, int64_t* a2a, int64_t* ag) {
  return guard([&] {
    const topo::CommTopology t(cluster(sf, sed, L));
    for (int l = 0; l < L; ++l) { a2a[l] = t.frequencies().levels[l].a2a; ag[l] = t.frequencies().levels[l].ag; }
  });
}

int ref_traffic_report(const int64_t* sf, const int64_t* sed, int L, double D, double PE, double mult, double* out4L) {
  return guard([&] {
    const topo::CommTopology t(cluster(sf, sed, L));
    perf::WorkloadSpec w;
    w.data_size_D = D;
    w.expert_size_PE = PE;
    const auto r = topo::traffic_report(t, w, topo::PlanShape{}, mult);
    for (int l = 0; l < L; ++l) {
      out4L[4 * l + 0] = r.levels[l].a2a_pair_bytes;
      out4L[4 * l + 1] = r.levels[l].ag_pair_bytes;
      out4L[4 * l + 2] = r.levels[l].a2a_bytes;
      out4L[4 * l + 3] = r.levels[l].ag_bytes;
    }
  });
}

int ref_factor_domain_sizes(int64_t s, const int64_t* sf, int L, int64_t* out) {
  std::vector<int64_t> sed(L, 1);
  return guard([&] {
    const auto v = factor_domain_sizes(s, cluster(sf, sed.data(), L));
    std::copy(v.begin(), v.end(), out);
  });
}

// The step DAG of one layer: jobs as rows {kind, layer, level, gpu, peer, ndeps} plus
// bytes/duration; deps flattened.  Returns the job count (or -1 on error); caller
// passes capacity.
int64_t ref_schedule(const int64_t* sf, const int64_t* sed, int L, double D, double PE, int64_t n_experts,
                     double pre, double expert_lat, double enc, double dec, int layers, int64_t cap,
                     int64_t* rows6, double* bd2, int64_t* deps, int64_t deps_cap, int64_t* ndeps_total) {
  int64_t count = -1;
  guard([&] {
    topo::ClusterSpec c = cluster(sf, sed, L);
    perf::WorkloadSpec w;
    w.data_size_D = D;
    w.expert_size_PE = PE;
    w.experts_per_gpu_n = n_experts;
    w.attn_latency = pre;
    w.ffn_latency = 1e-12;
    w.expert_latency = expert_lat;
    HybridPlan plan;
    plan.domain_sizes.assign(sed, sed + L);
    const int64_t G = c.total_gpus();
    int64_t s = 1;
    for (int i = 0; i < L; ++i) s *= sed[i];
    plan.p = G > 1 ? static_cast<double>(G - s) / static_cast<double>(G - 1) : 1.0;
    plan.encode_cost = enc;
    plan.decode_cost = dec;
    plan.layers = layers;
    const auto g = sim::build_schedule(c, w, plan);
    int64_t dp = 0;
    for (size_t i = 0; i < g.jobs.size() && static_cast<int64_t>(i) < cap; ++i) {
      const auto& j = g.jobs[i];
      int64_t* r = rows6 + 6 * i;
      r[0] = static_cast<int64_t>(j.kind); r[1] = j.layer; r[2] = j.level; r[3] = j.gpu; r[4] = j.peer;
      r[5] = static_cast<int64_t>(j.deps.size());
      bd2[2 * i] = j.bytes;
      bd2[2 * i + 1] = j.duration;
      for (int64_t d : j.deps) if (dp < deps_cap) deps[dp++] = d;
    }
    *ndeps_total = dp;
    count = static_cast<int64_t>(g.jobs.size());
  });
  return count;
}

// One iteration on the reference's discrete-event engine (build_schedule + sim::run,
// simcore.cpp:96-367) with per-level bandwidth bw (bytes/s): makespan and worst AG stall.
// The predicted side of tools/model_vs_measured.py (the engine is the reference's timing
// model; the B200 build measures real time instead and does not ship one).
int ref_sim_step(const int64_t* sf, const int64_t* sed, int L, double bw, double D, double PE, int64_t n_experts,
                 double pre, double expert_lat, double enc, double dec, int layers, double* makespan, double* stall) {
  return guard([&] {
    topo::ClusterSpec c;
    for (int i = 0; i < L; ++i) c.levels.push_back({sf[i], sed[i], bw});
    perf::WorkloadSpec w;
    w.data_size_D = D;
    w.expert_size_PE = PE;
    w.experts_per_gpu_n = n_experts;
    w.attn_latency = pre;
    w.ffn_latency = 1e-12;
    w.expert_latency = expert_lat;
    HybridPlan plan;
    plan.domain_sizes.assign(sed, sed + L);
    const int64_t G = c.total_gpus();
    int64_t s = 1;
    for (int i = 0; i < L; ++i) s *= sed[i];
    plan.p = G > 1 ? static_cast<double>(G - s) / static_cast<double>(G - 1) : 1.0;
    plan.encode_cost = enc;
    plan.decode_cost = dec;
    plan.layers = layers;
    const auto trace = sim::run(sim::build_schedule(c, w, plan), with_domain_sizes(c, plan.domain_sizes));
    *makespan = trace.makespan;
    *stall = trace.max_ag_stall;
  });
}

int ref_solve_optimal_p(double D, double PE, int64_t n, int64_t m, double attn, double ffn, double expert,
                        double bwd, double C, double B, int64_t gpus, double* p, int64_t* s, double* total) {
  return guard([&] {
    perf::WorkloadSpec w;
    w.data_size_D = D; w.expert_size_PE = PE; w.experts_per_gpu_n = n; w.pre_blocks_m = m;
    w.attn_latency = attn; w.ffn_latency = ffn; w.expert_latency = expert; w.backward_allreduce_const = bwd;
    const auto pt = perf::solve_optimal_p(w, perf::DeviceSpec{C, B}, gpus);
    *p = pt.p;
    *s = pt.domain_size;
    *total = pt.latency.total;
  });
}

int64_t ref_sr_resolve_k(double ratio, int64_t k, uint32_t iw, uint32_t vw, int64_t total, int64_t eb) {
  sr::CompressionConfig c;
  if (k >= 0) c.k = k; else c.ratio_CR = ratio;
  c.index_width_bits = iw;
  c.value_width_bits = vw;
  int64_t out = -1;
  guard([&] { out = c.resolve_k(total, eb); });
  return out;
}

// Returns wire bytes written into `wire` (capacity `cap`), or -(status) on error.
int64_t ref_sr_encode(const float* expert, const float* shared, int64_t h, int64_t m, double ratio, int64_t k,
                      uint32_t iw, uint32_t vw, int per_matrix, uint8_t* wire, int64_t cap) {
  int64_t n = 0;
  const int rc = guard([&] {
    sr::CompressionConfig c;
    if (k >= 0) c.k = k; else c.ratio_CR = ratio;
    c.index_width_bits = iw;
    c.value_width_bits = vw;
    c.per_matrix_budget = per_matrix != 0;
    const auto bytes = sr::sr_encode(expert_of(expert, h, m), expert_of(shared, h, m), c).serialize();
    if (static_cast<int64_t>(bytes.size()) > cap) throw std::invalid_argument("capacity");
    std::memcpy(wire, bytes.data(), bytes.size());
    n = static_cast<int64_t>(bytes.size());
  });
  return rc ? -rc : n;
}

// 0 ok; 2 invalid_argument (shape tag); 3 runtime_error (corrupt wire).
int ref_sr_decode(const uint8_t* wire, int64_t bytes, const float* shared, int64_t h, int64_t m, float* out) {
  return guard([&] {
    const auto c = sr::CompressedResidual::deserialize(std::vector<uint8_t>(wire, wire + bytes));
    const auto e = sr::sr_decode(c, expert_of(shared, h, m));
    std::memcpy(out, e.w_up.data.data(), sizeof(float) * h * m);
    std::memcpy(out + h * m, e.w_down.data.data(), sizeof(float) * h * m);
  });
}

int ref_shared_mean(const float* const* experts, int n, int64_t h, int64_t m, float* out) {
  return guard([&] {
    std::vector<sr::ExpertWeights> v;
    for (int i = 0; i < n; ++i) v.push_back(expert_of(experts[i], h, m));
    const auto s = sr::init_shared(v);
    std::memcpy(out, s.w_up.data.data(), sizeof(float) * h * m);
    std::memcpy(out + h * m, s.w_down.data.data(), sizeof(float) * h * m);
  });
}

}  // extern "C"
