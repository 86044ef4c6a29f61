#pragma once
// hybridep::moe — the MoE-layer step on B200 (new; the reference only simulates it).
//
// Host-side C++ over the C-ABI in include/hep.h.  Pinned semantics (SURVEY.md
// §8(c) S1-S7, restated in DESIGN.md §2):
//   S1 placement: expert e is owned by GPU e / n; after All-Gather GPU m also holds
//      the experts of every o with classify(m, o) == AG.
//   S2 destination of (token on m, expert e), o = owner(e): m if m == o or AG(m,o);
//      else o if A2A(m,o); else the first n in peer_lists(m).a2a order (levels
//      outermost first, ring key inside a level) with AG(n,o).
//   S3 gating: logits = x . W_g, top-k by (logit desc, id asc), softmax over the k.
//   S4 expert FFN: y = relu(x . w_up) . w_down.
//   S5 combine: y_t = sum_j w_tj out_tj in slot order.
//   S7 packed rows grouped by (destination GPU, expert), stable by (token, slot).

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hep.h"
#include "hybridep/perfmodel.hpp"
#include "hybridep/sparsecomp.hpp"
#include "hybridep/topology.hpp"

namespace hybridep::moe {

// route[m * G + o] = GPU that computes, for tokens living on m, the experts owned by o.
// Throws std::invalid_argument when some (m, o) has no route (never at G = 8).
std::vector<std::int32_t> route_table(const topo::ClusterSpec& cluster);

// held[m] = owners whose experts GPU m holds after the All-Gather (m first, then its
// AG peers in peer_lists order).
std::vector<std::vector<std::int64_t>> held_owners(const topo::ClusterSpec& cluster);

// ---------------------------------------------------------------- planner + reports
// resolve_plan (cli_app.cpp:132-168) without the JSON config: the solver's pick, or a
// pinned per-level S_ED.  write_plan_reports emits plan.json, freq.json and topo.csv in
// the reference's formats (cli_app.cpp:183-243).
struct ResolvedPlan {
  perf::CaseTag config_case = perf::CaseTag::Case1;
  double continuous_p = 0;
  double boundary_p = 0;
  perf::PlanPoint point;
  std::vector<std::int64_t> domain_sizes;
};
ResolvedPlan resolve_plan(const topo::ClusterSpec& cluster, const perf::WorkloadSpec& workload,
                          const perf::DeviceSpec& device,
                          const std::vector<std::int64_t>* pinned_domain_sizes = nullptr);
void write_plan_reports(const topo::ClusterSpec& cluster, const perf::WorkloadSpec& workload,
                        const ResolvedPlan& plan, const std::string& out_dir);

// ---------------------------------------------------------------- the step, in C++
// RAII wrappers over the C-ABI (include/hep.h) that rethrow the reference's exception
// types: std::domain_error (HEP_ERR_DOMAIN), std::invalid_argument
// (HEP_ERR_INVALID_ARGUMENT), std::runtime_error (everything else; CUDA / NCCL failures
// carry their prefix).  Streams are cudaStream_t passed as void*; device pointers are
// CUDA device addresses.  Header-only, so a C++ caller links libhep.so alone.

inline void check(int status) {
  if (status == HEP_OK) return;
  const std::string msg = hep_last_error();
  if (status == HEP_ERR_DOMAIN) throw std::domain_error(msg);
  if (status == HEP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

class Communicator {
 public:
  // NCCL communicator of `nranks` processes (one per GPU) from a 128-byte unique id made
  // by unique_id() on one rank and broadcast by the caller.
  static std::vector<unsigned char> unique_id() {
    std::vector<unsigned char> id(128);
    check(hep_comm_unique_id(id.data()));
    return id;
  }
  static Communicator nccl(const std::vector<unsigned char>& id, int rank, int nranks) {
    if (id.size() != 128) throw std::invalid_argument("NCCL unique id must be 128 bytes");
    hep_comm_t c = nullptr;
    check(hep_comm_init(id.data(), rank, nranks, &c));
    return Communicator(c, rank, nranks);
  }
  // `nranks` virtual ranks driven by this process on the current device.
  static std::vector<Communicator> virtual_ranks(int nranks) {
    std::vector<hep_comm_t> hs(static_cast<size_t>(nranks > 0 ? nranks : 0));
    check(hep_comm_init_virtual(nranks, hs.data()));
    std::vector<Communicator> out;
    for (int r = 0; r < nranks; ++r) out.push_back(Communicator(hs[static_cast<size_t>(r)], r, nranks));
    return out;
  }
  Communicator(Communicator&& o) noexcept : h_(std::exchange(o.h_, nullptr)), rank_(o.rank_), nranks_(o.nranks_) {}
  Communicator& operator=(Communicator&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
      rank_ = o.rank_;
      nranks_ = o.nranks_;
    }
    return *this;
  }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  ~Communicator() { reset(); }
  hep_comm_t get() const { return h_; }
  int rank() const { return rank_; }
  int nranks() const { return nranks_; }

 private:
  Communicator(hep_comm_t h, int rank, int nranks) : h_(h), rank_(rank), nranks_(nranks) {}
  void reset() {
    if (h_) hep_comm_destroy(h_);
    h_ = nullptr;
  }
  hep_comm_t h_ = nullptr;
  int rank_ = 0, nranks_ = 1;
};

struct LayerConfig {
  std::int64_t hidden = 0, ffn = 0, experts = 0, top_k = 0, max_tokens = 0;
  hep_dtype dtype = HEP_BF16;
  topo::ClusterSpec cluster;  // SF / S_ED per level, outermost first (bandwidth unused)
  int rank = 0;
  std::optional<sr::CompressionConfig> migration;  // SR-migrated All-Gather when set
};

class Layer {
 public:
  explicit Layer(const LayerConfig& cfg, const Communicator* comm = nullptr) : rank_(cfg.rank) {
    std::vector<hep_level> lv;
    for (const auto& l : cfg.cluster.levels) lv.push_back({l.scaling_factor, l.domain_size, l.bandwidth});
    hep_layer_params p{};
    p.hidden = cfg.hidden;
    p.ffn = cfg.ffn;
    p.experts = cfg.experts;
    p.top_k = cfg.top_k;
    p.max_tokens = cfg.max_tokens;
    p.dtype = cfg.dtype;
    p.levels = lv.data();
    p.num_levels = static_cast<int>(lv.size());
    p.rank = cfg.rank;
    p.use_sr = cfg.migration ? 1 : 0;
    p.sr = {1.0, -1, 32, 32, 0};
    if (cfg.migration) {
      const auto& m = *cfg.migration;
      p.sr = {m.ratio_CR.value_or(1.0), m.k ? *m.k : -1, m.index_width_bits, m.value_width_bits,
              m.per_matrix_budget ? 1 : 0};
    }
    check(hep_layer_create(&p, comm ? comm->get() : nullptr, &h_));
    std::int64_t gpus = 1;
    for (const auto& l : cfg.cluster.levels) gpus *= l.scaling_factor;
    per_gpu_ = cfg.experts / (gpus > 0 ? gpus : 1);
  }
  Layer(Layer&& o) noexcept : h_(std::exchange(o.h_, nullptr)), rank_(o.rank_), per_gpu_(o.per_gpu_) {}
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;
  ~Layer() {
    if (h_) hep_layer_destroy(h_);
  }

  std::vector<std::int64_t> owned_experts() const {
    std::vector<std::int64_t> e;
    for (std::int64_t i = 0; i < per_gpu_; ++i) e.push_back(rank_ * per_gpu_ + i);
    return e;
  }
  void set_gate(const void* w_gate, hep_dtype dt, void* stream) { check(hep_layer_set_gate(h_, w_gate, dt, stream)); }
  void set_expert(std::int64_t e, const void* w_up, const void* w_down, hep_dtype dt, void* stream) {
    check(hep_layer_set_expert(h_, e, w_up, w_down, dt, stream));
  }
  void set_shared(const float* shared, void* stream) { check(hep_layer_set_shared(h_, shared, stream)); }
  void refresh_shared(void* stream) { check(hep_layer_refresh_shared(h_, stream)); }
  void gather_experts(void* stream) { check(hep_layer_gather_experts(h_, stream)); }
  void forward(const void* x, std::int64_t tokens, void* y, void* stream) {
    check(hep_layer_forward(h_, x, tokens, y, stream));
  }
  void forward_host(const void* x, std::int64_t tokens, void* y, void* stream) {
    check(hep_layer_forward_host(h_, x, tokens, y, stream));
  }
  void host_fence(void* stream) { check(hep_layer_host_fence(h_, stream)); }
  // Synchronises and throws std::runtime_error if a migrated expert was rejected.
  void check_migration(void* stream) { check(hep_layer_check(h_, stream)); }
  hep_layer_t get() const { return h_; }

 private:
  hep_layer_t h_ = nullptr;
  std::int64_t rank_ = 0, per_gpu_ = 1;
};

}  // namespace hybridep::moe
