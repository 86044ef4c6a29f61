// extern "C" boundary (include/hep.h).  Exceptions never cross it: each entry point
// maps std::domain_error / std::invalid_argument / std::runtime_error to the
// matching hep_status and records the message for hep_last_error().

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../kernels/kernels.h"
#include "hep.h"
#include "hybridep/moe.hpp"
#include "hybridep/perfmodel.hpp"
#include "hybridep/plan.hpp"
#include "hybridep/simcore.hpp"
#include "hybridep/sparsecomp.hpp"
#include "hybridep/topology.hpp"
#include "layer.h"

namespace {

thread_local std::string g_last_error;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_last_error.clear();
    return HEP_OK;
  } catch (const CudaError& e) {
    return fail(HEP_ERR_CUDA, e.what());
  } catch (const std::domain_error& e) {
    return fail(HEP_ERR_DOMAIN, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(HEP_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::runtime_error& e) {
    const std::string w = e.what();
    if (w.rfind("CUDA error", 0) == 0) return fail(HEP_ERR_CUDA, w);
    if (w.rfind("NCCL error", 0) == 0) return fail(HEP_ERR_NCCL, w);
    return fail(HEP_ERR_RUNTIME, w);
  } catch (const std::exception& e) {
    return fail(HEP_ERR_RUNTIME, e.what());
  }
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

hybridep::topo::ClusterSpec cluster_of(const hep_level* levels, int n) {
  if (!levels || n <= 0) throw std::invalid_argument("cluster needs at least one level");
  hybridep::topo::ClusterSpec c;
  for (int i = 0; i < n; ++i) c.levels.push_back({levels[i].scaling_factor, levels[i].domain_size, levels[i].bandwidth});
  return c;
}

hybridep::sr::CompressionConfig sr_config_of(const hep_sr_config* c) {
  if (!c) throw std::invalid_argument("null SR config");
  hybridep::sr::CompressionConfig cfg;
  if (c->k >= 0) cfg.k = c->k; else cfg.ratio_CR = c->ratio_CR;
  cfg.index_width_bits = c->index_width_bits;
  cfg.value_width_bits = c->value_width_bits;
  cfg.per_matrix_budget = c->per_matrix_budget != 0;
  return cfg;
}

hep::DType dt_of(hep_dtype d) {
  if (d != HEP_F32 && d != HEP_BF16) throw std::invalid_argument("dtype must be HEP_F32 or HEP_BF16");
  return d == HEP_BF16 ? hep::DType::BF16 : hep::DType::F32;
}

cudaStream_t st(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

struct hep_comm_s {
  hep::Comm c;
};
struct hep_layer_s {
  std::unique_ptr<hep::Layer> impl;
};

extern "C" {

const char* hep_last_error(void) { return g_last_error.c_str(); }
const char* hep_version(void) { return "hybridep-b200 0.1 (sm_100a)"; }

int hep_topology_gpus(const hep_level* levels, int num_levels, int64_t* gpus) {
  return guarded([&] {
    auto c = cluster_of(levels, num_levels);
    c.validate();
    *gpus = c.total_gpus();
  });
}

int hep_topology_build(const hep_level* levels, int num_levels, int8_t* pair_level, uint8_t* pair_type) {
  return guarded([&] {
    const hybridep::topo::CommTopology t(cluster_of(levels, num_levels));
    if (!t.dense()) throw std::invalid_argument("dense table needs G <= 4096");
    std::memcpy(pair_level, t.pair_levels().data(), t.pair_levels().size());
    std::memcpy(pair_type, t.pair_types().data(), t.pair_types().size());
  });
}

int hep_renumber(const hep_level* levels, int num_levels, int64_t m, int64_t* coords) {
  return guarded([&] {
    const auto x = hybridep::topo::renumber(m, cluster_of(levels, num_levels));
    std::copy(x.begin(), x.end(), coords);
  });
}

int hep_global_index(const hep_level* levels, int num_levels, const int64_t* coords, int64_t* m) {
  return guarded([&] {
    const hybridep::topo::MultiIndex x(coords, coords + num_levels);
    *m = hybridep::topo::global_index(x, cluster_of(levels, num_levels));
  });
}

int hep_comm_type(const hep_level* levels, int num_levels, int64_t m, int64_t n, int level, int* type) {
  return guarded([&] {
    *type = static_cast<int>(hybridep::topo::comm_type(m, n, level, cluster_of(levels, num_levels)));
  });
}

int hep_level_frequency(const hep_level* levels, int num_levels, int64_t* a2a, int64_t* ag) {
  return guarded([&] {
    const hybridep::topo::CommTopology t(cluster_of(levels, num_levels));
    for (int l = 0; l < num_levels; ++l) {
      a2a[l] = t.frequencies().levels[l].a2a;
      ag[l] = t.frequencies().levels[l].ag;
    }
  });
}

int hep_traffic_report(const hep_level* levels, int num_levels, double data_size_D, double expert_size_PE,
                       double token_multiplier, double* a2a_pair_bytes, double* ag_pair_bytes,
                       double* a2a_bytes, double* ag_bytes) {
  return guarded([&] {
    const hybridep::topo::CommTopology t(cluster_of(levels, num_levels));
    hybridep::perf::WorkloadSpec w;
    w.data_size_D = data_size_D;
    w.expert_size_PE = expert_size_PE;
    const auto r = hybridep::topo::traffic_report(t, w, hybridep::topo::PlanShape{}, token_multiplier);
    for (int l = 0; l < num_levels; ++l) {
      a2a_pair_bytes[l] = r.levels[l].a2a_pair_bytes;
      ag_pair_bytes[l] = r.levels[l].ag_pair_bytes;
      a2a_bytes[l] = r.levels[l].a2a_bytes;
      ag_bytes[l] = r.levels[l].ag_bytes;
    }
  });
}

int hep_peer_lists(const hep_level* levels, int num_levels, int64_t m, int64_t* ag_peers, int* ag_level,
                   int* n_ag, int64_t* a2a_peers, int* a2a_level, int* n_a2a) {
  return guarded([&] {
    const auto c = cluster_of(levels, num_levels);
    c.validate();
    if (m < 0 || m >= c.total_gpus()) throw std::domain_error("GPU index out of range");
    const auto pl = hybridep::sim::peer_lists(c)[static_cast<size_t>(m)];
    int na = 0, nb = 0;
    for (int l = 0; l < num_levels; ++l) {
      for (int64_t p : pl.ag[l]) { ag_peers[na] = p; ag_level[na++] = l; }
      for (int64_t p : pl.a2a[l]) { a2a_peers[nb] = p; a2a_level[nb++] = l; }
    }
    *n_ag = na;
    *n_a2a = nb;
  });
}

int hep_route_table(const hep_level* levels, int num_levels, int32_t* route) {
  return guarded([&] {
    const auto r = hybridep::moe::route_table(cluster_of(levels, num_levels));
    std::copy(r.begin(), r.end(), route);
  });
}

int hep_factor_domain_sizes(int64_t domain_size, const hep_level* levels, int num_levels, int64_t* out) {
  return guarded([&] {
    const auto v = hybridep::factor_domain_sizes(domain_size, cluster_of(levels, num_levels));
    std::copy(v.begin(), v.end(), out);
  });
}

int hep_solve_optimal_p(const hep_workload* w, double throughput_C, double bandwidth_B, int64_t gpus,
                        double* p, int64_t* domain_size, double* latency6) {
  return guarded([&] {
    hybridep::perf::WorkloadSpec ws;
    ws.data_size_D = w->data_size_D;
    ws.expert_size_PE = w->expert_size_PE;
    ws.experts_per_gpu_n = w->experts_per_gpu_n;
    ws.pre_blocks_m = w->pre_blocks_m;
    ws.attn_latency = w->attn_latency;
    ws.ffn_latency = w->ffn_latency;
    ws.expert_latency = w->expert_latency;
    ws.backward_allreduce_const = w->backward_allreduce_const;
    const auto pt = hybridep::perf::solve_optimal_p(ws, hybridep::perf::DeviceSpec{throughput_C, bandwidth_B}, gpus);
    *p = pt.p;
    *domain_size = pt.domain_size;
    const auto& L = pt.latency;
    const double v[6] = {L.comp, L.pre_expert, L.comm_a2a, L.comm_ag, L.overlap, L.total};
    std::copy(v, v + 6, latency6);
  });
}

int hep_plan_reports(const hep_level* levels, int num_levels, const hep_workload* w, double throughput_C,
                     double bandwidth_B, const int64_t* pinned_domain_sizes, const char* out_dir, double* p,
                     int64_t* domain_sizes, double* latency6) {
  return guarded([&] {
    if (!w) throw std::invalid_argument("null workload");
    hybridep::perf::WorkloadSpec ws;
    ws.data_size_D = w->data_size_D;
    ws.expert_size_PE = w->expert_size_PE;
    ws.experts_per_gpu_n = w->experts_per_gpu_n;
    ws.pre_blocks_m = w->pre_blocks_m;
    ws.attn_latency = w->attn_latency;
    ws.ffn_latency = w->ffn_latency;
    ws.expert_latency = w->expert_latency;
    ws.backward_allreduce_const = w->backward_allreduce_const;
    const auto cluster = cluster_of(levels, num_levels);
    std::vector<int64_t> pinned;
    if (pinned_domain_sizes) pinned.assign(pinned_domain_sizes, pinned_domain_sizes + num_levels);
    const auto plan = hybridep::moe::resolve_plan(cluster, ws, hybridep::perf::DeviceSpec{throughput_C, bandwidth_B},
                                                  pinned_domain_sizes ? &pinned : nullptr);
    if (out_dir && *out_dir) hybridep::moe::write_plan_reports(cluster, ws, plan, out_dir);
    if (p) *p = plan.point.p;
    if (domain_sizes) std::copy(plan.domain_sizes.begin(), plan.domain_sizes.end(), domain_sizes);
    if (latency6) {
      const auto& L = plan.point.latency;
      const double v[6] = {L.comp, L.pre_expert, L.comm_a2a, L.comm_ag, L.overlap, L.total};
      std::copy(v, v + 6, latency6);
    }
  });
}

int hep_sr_resolve_k(const hep_sr_config* cfg, int64_t total_elements, int64_t elem_bytes, int64_t* k) {
  return guarded([&] { *k = sr_config_of(cfg).resolve_k(total_elements, elem_bytes); });
}

int hep_sr_wire_bytes(int64_t h, int64_t m, const hep_sr_config* cfg, size_t* bytes) {
  return guarded([&] {
    if (h <= 0 || m <= 0) throw std::invalid_argument("empty expert matrix");
    const auto c = sr_config_of(cfg);
    if ((c.index_width_bits != 32 && c.index_width_bits != 64) || (c.value_width_bits != 32 && c.value_width_bits != 64))
      throw std::invalid_argument("residual widths must be 32 or 64 bits");
    const int64_t k = c.resolve_k(2 * h * m, 4);
    *bytes = static_cast<size_t>(hybridep::sr::kWireHeaderBytes + k * (c.index_width_bits + c.value_width_bits) / 8);
  });
}

int hep_sr_workspace_bytes(int64_t h, int64_t m, int batch, size_t* bytes) {
  return guarded([&] {
    if (h <= 0 || m <= 0 || batch <= 0) throw std::invalid_argument("bad workspace query");
    *bytes = hep::sr_workspace_bytes(h, m, batch);
  });
}

namespace {

hep::SrPlan make_sr_plan(int64_t h, int64_t m, const hep_sr_config* cfg) {
  if (h <= 0 || m <= 0) throw std::invalid_argument("empty expert matrix");
  const auto c = sr_config_of(cfg);
  if ((c.index_width_bits != 32 && c.index_width_bits != 64) || (c.value_width_bits != 32 && c.value_width_bits != 64))
    throw std::invalid_argument("residual widths must be 32 or 64 bits");
  if (h > 0xffffffffll || m > 0xffffffffll) throw std::invalid_argument("shape does not fit the wire header");
  hep::SrPlan plan{};
  plan.h = h;
  plan.m = m;
  plan.total = 2 * h * m;
  plan.k = c.resolve_k(plan.total, 4);
  const int64_t up = h * m;
  plan.per_matrix = c.per_matrix_budget ? 1 : 0;
  plan.k_up = plan.per_matrix ? std::min(up, plan.k * up / plan.total) : plan.k;
  plan.k_down = plan.per_matrix ? std::min(plan.total - up, plan.k - plan.k_up) : 0;
  if (plan.per_matrix) plan.k = plan.k_up + plan.k_down;
  plan.index_bits = c.index_width_bits;
  plan.value_bits = c.value_width_bits;
  if (c.index_width_bits == 32 && plan.total > 0xffffffffll)
    throw std::invalid_argument("32-bit indices cannot address this expert");
  plan.wire_bytes = static_cast<size_t>(28 + plan.k * (plan.index_bits + plan.value_bits) / 8);
  return plan;
}

}  // namespace

int hep_sr_encode_batch(const void* const* experts, int n, hep_dtype expert_dtype, const float* shared, int64_t h,
                        int64_t m, const hep_sr_config* cfg, void* const* wires, size_t wire_capacity, void* workspace,
                        size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (n <= 0 || n > hep::kMaxSrBatch) throw std::invalid_argument("batch must be in [1, 64]");
    const hep::SrPlan plan = make_sr_plan(h, m, cfg);
    if (wire_capacity < plan.wire_bytes) throw std::invalid_argument("wire buffer too small");
    if (workspace_bytes < hep::sr_workspace_bytes(h, m, n)) throw std::invalid_argument("workspace too small");
    cuda_ok(hep::launch_sr_encode_batch(dt_of(expert_dtype), experts, n, shared, plan,
                                        reinterpret_cast<uint8_t* const*>(wires), workspace, st(stream)),
            "sr encode");
  });
}

int hep_sr_encode_update_batch(float* const* masters, const float* const* grads, int n, float lr, const float* shared,
                               int64_t h, int64_t m, const hep_sr_config* cfg, void* const* wires, size_t wire_capacity,
                               void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (n <= 0 || n > hep::kMaxSrBatch) throw std::invalid_argument("batch must be in [1, 64]");
    if (!grads) throw std::invalid_argument("null gradient array");
    const hep::SrPlan plan = make_sr_plan(h, m, cfg);
    if (wire_capacity < plan.wire_bytes) throw std::invalid_argument("wire buffer too small");
    if (workspace_bytes < hep::sr_workspace_bytes(h, m, n)) throw std::invalid_argument("workspace too small");
    std::vector<const void*> ex(masters, masters + n);
    cuda_ok(hep::launch_sr_encode_batch(hep::DType::F32, ex.data(), n, shared, plan,
                                        reinterpret_cast<uint8_t* const*>(wires), workspace, st(stream), grads, lr),
            "sr encode update");
  });
}

int hep_sgd_step_batch(float* const* masters, const float* const* grads, int n, int64_t elements, float lr,
                       void* stream) {
  return guarded([&] {
    if (n <= 0 || n > hep::kMaxSrBatch) throw std::invalid_argument("batch must be in [1, 64]");
    if (elements <= 0) throw std::invalid_argument("empty expert");
    cuda_ok(hep::launch_sgd_step_batch(masters, grads, n, elements, lr, st(stream)), "sgd step");
  });
}

int hep_layer_sgd_step(hep_layer_t layer, const float* const* grads, int n, float lr, void* stream) {
  return guarded([&] { layer->impl->sgd_step(grads, n, lr, st(stream)); });
}

int hep_sr_encode(const void* expert, hep_dtype expert_dtype, const float* shared, int64_t h, int64_t m,
                  const hep_sr_config* cfg, void* wire, size_t wire_capacity, void* workspace,
                  size_t workspace_bytes, void* stream) {
  const void* e[1] = {expert};
  void* w[1] = {wire};
  return hep_sr_encode_batch(e, 1, expert_dtype, shared, h, m, cfg, w, wire_capacity, workspace, workspace_bytes,
                             stream);
}

int hep_sr_decode_batch(const void* const* wires, int n, size_t wire_bytes, const float* shared, int64_t h, int64_t m,
                        float* const* outs, int32_t* status, void* stream) {
  return guarded([&] {
    if (h <= 0 || m <= 0) throw std::invalid_argument("empty expert matrix");
    if (n <= 0 || n > hep::kMaxSrBatch) throw std::invalid_argument("batch must be in [1, 64]");
    cuda_ok(hep::launch_sr_decode_batch(reinterpret_cast<const uint8_t* const*>(wires), n, wire_bytes, shared, h, m,
                                        outs, status, st(stream)),
            "sr decode");
  });
}

int hep_sr_decode(const void* wire, size_t wire_bytes, const float* shared, int64_t h, int64_t m, float* out,
                  int32_t* status, void* stream) {
  const void* w[1] = {wire};
  float* o[1] = {out};
  return hep_sr_decode_batch(w, 1, wire_bytes, shared, h, m, o, status, stream);
}

int hep_sr_check_status(const int32_t* status, void* stream) {
  return guarded([&] {
    cuda_ok(cudaStreamSynchronize(st(stream)), "sync");
    int32_t s[2] = {0, 0};
    cuda_ok(cudaMemcpy(s, status, sizeof(s), cudaMemcpyDeviceToHost), "status d2h");
    switch (s[0]) {
      case 0: return;
      case 1: throw std::runtime_error("bad residual magic");
      case 2: throw std::runtime_error("compressed residual truncated");
      case 3: throw std::runtime_error("unsupported residual widths");
      case 4: throw std::invalid_argument("residual shape tag does not match the shared expert");
      case 5: throw std::runtime_error("corrupt residual: index out of bounds (entry " + std::to_string(s[1]) + ")");
      case 6: throw std::runtime_error("corrupt residual: indices not strictly increasing (entry " + std::to_string(s[1]) + ")");
      default: throw std::runtime_error("unknown decode status " + std::to_string(s[0]));
    }
  });
}

int hep_shared_mean(const void* const* experts, int n, hep_dtype dtype, int64_t P, float* out, void* stream) {
  return guarded([&] {
    if (n <= 0) throw std::invalid_argument("cannot average zero experts");
    if (P <= 0) throw std::invalid_argument("empty expert matrix");
    cuda_ok(hep::launch_shared_mean(dt_of(dtype), experts, n, P, out, st(stream)), "shared mean");
  });
}

int hep_comm_unique_id(void* id128) {
  return guarded([&] {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL error: ") + ncclGetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "nccl unique id size");
    std::memcpy(id128, &id, 128);
  });
}

int hep_comm_init(const void* id128, int rank, int nranks, hep_comm_t* comm) {
  return guarded([&] {
    ncclUniqueId id;
    std::memcpy(&id, id128, 128);
    auto c = std::make_unique<hep_comm_s>();
    const ncclResult_t r = ncclCommInitRank(&c->c.nccl, nranks, id, rank);
    if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL error: ") + ncclGetErrorString(r));
    c->c.rank = rank;
    c->c.nranks = nranks;
    *comm = c.release();
  });
}

int hep_comm_init_virtual(int nranks, hep_comm_t* comms) {
  return guarded([&] {
    if (nranks < 1 || nranks > 8) throw std::invalid_argument("virtual ranks: 1 <= nranks <= 8");
    if (!comms) throw std::invalid_argument("null argument");
    auto group = std::make_shared<hep::VirtualGroup>();
    group->nranks = nranks;
    std::vector<std::unique_ptr<hep_comm_s>> made;
    for (int r = 0; r < nranks; ++r) {
      auto c = std::make_unique<hep_comm_s>();
      c->c.rank = r;
      c->c.nranks = nranks;
      c->c.vgroup = group;
      made.push_back(std::move(c));
    }
    for (int r = 0; r < nranks; ++r) comms[r] = made[static_cast<size_t>(r)].release();
  });
}

int hep_comm_destroy(hep_comm_t comm) {
  return guarded([&] {
    if (!comm) return;
    if (comm->c.nccl) ncclCommDestroy(comm->c.nccl);
    delete comm;
  });
}

int hep_layer_create(const hep_layer_params* params, hep_comm_t comm, hep_layer_t* layer) {
  return guarded([&] {
    if (!params || !layer) throw std::invalid_argument("null argument");
    auto l = std::make_unique<hep_layer_s>();
    l->impl = std::make_unique<hep::Layer>(*params, comm ? &comm->c : nullptr);
    *layer = l.release();
  });
}

int hep_layer_destroy(hep_layer_t layer) {
  return guarded([&] { delete layer; });
}

int hep_layer_set_gate(hep_layer_t layer, const void* w_gate, hep_dtype dtype, void* stream) {
  return guarded([&] { layer->impl->set_gate(w_gate, dt_of(dtype), st(stream)); });
}

int hep_layer_set_expert(hep_layer_t layer, int64_t expert, const void* w_up, const void* w_down, hep_dtype dtype,
                         void* stream) {
  return guarded([&] { layer->impl->set_expert(expert, w_up, w_down, dt_of(dtype), st(stream)); });
}

int hep_layer_set_shared(hep_layer_t layer, const float* shared, void* stream) {
  return guarded([&] { layer->impl->set_shared(shared, st(stream)); });
}

int hep_layer_refresh_shared(hep_layer_t layer, void* stream) {
  return guarded([&] { layer->impl->refresh_shared(st(stream)); });
}

int hep_layer_get_shared(hep_layer_t layer, float* out, void* stream) {
  return guarded([&] { layer->impl->get_shared(out, st(stream)); });
}

int hep_layer_gather_experts(hep_layer_t layer, void* stream) {
  return guarded([&] { layer->impl->gather_experts(st(stream)); });
}

int hep_layers_gather(hep_layer_t* layers, int n, void* stream) {
  return guarded([&] {
    if (n < 0 || (n > 0 && !layers)) throw std::invalid_argument("need an array of n layers");
    for (int i = 0; i < n; ++i) layers[i]->impl->gather_experts(st(stream));
  });
}

int hep_layer_forward_residual(hep_layer_t layer, const void* x, int64_t tokens, void* y, void* stream) {
  return guarded([&] { layer->impl->forward(x, tokens, y, st(stream), true); });
}

int hep_layer_forward(hep_layer_t layer, const void* x, int64_t tokens, void* y, void* stream) {
  return guarded([&] { layer->impl->forward(x, tokens, y, st(stream)); });
}

int hep_layer_forward_host(hep_layer_t layer, const void* host_x, int64_t tokens, void* host_y, void* stream) {
  return guarded([&] { layer->impl->forward_host(host_x, tokens, host_y, st(stream)); });
}

int hep_layer_host_fence(hep_layer_t layer, void* stream) {
  return guarded([&] { layer->impl->host_fence(st(stream)); });
}

int hep_layer_comm_bench(hep_layer_t layer, const void* x, int64_t tokens, int iters, double* out6, void* stream) {
  return guarded([&] {
    if (iters <= 0) throw std::invalid_argument("iters must be positive");
    layer->impl->comm_bench(x, tokens, iters, out6, st(stream));
  });
}

int hep_layer_debug(hep_layer_t layer, const int32_t** topk_idx, const float** topk_w, const int32_t** pos,
                    const void** packed, const int32_t** key_counts) {
  return guarded([&] {
    hep::Layer& l = *layer->impl;
    if (topk_idx) *topk_idx = l.topk_idx();
    if (topk_w) *topk_w = l.topk_w();
    if (pos) *pos = l.pos();
    if (packed) *packed = l.packed();
    if (key_counts) *key_counts = l.key_counts();
  });
}

int hep_layer_set_profiling(hep_layer_t layer, int on) {
  return guarded([&] {
    if (on < 0 || on > 2) throw std::invalid_argument("profiling level must be 0, 1 (GEMM events) or 2 (all phases)");
    layer->impl->set_profiling(on);
  });
}

int hep_layer_timings(hep_layer_t layer, char* names, size_t names_cap, float* ms, int cap, int* count) {
  return guarded([&] { layer->impl->collect_timings(names, names_cap, ms, cap, count); });
}

int hep_layer_launch_count(hep_layer_t layer, int* count) {
  return guarded([&] { *count = layer->impl->launch_count(); });
}

int hep_layer_check(hep_layer_t layer, void* stream) {
  return guarded([&] {
    cuda_ok(cudaStreamSynchronize(st(stream)), "sync");
    layer->impl->check_migration(true);
  });
}

int hep_layer_debug_corrupt_next_gather(hep_layer_t layer) {
  return guarded([&] { layer->impl->corrupt_next_gather(); });
}

int hep_layer_gemm_schedule(hep_layer_t layer, uint32_t* up, uint32_t* down) {
  return guarded([&] { layer->impl->gemm_schedules(up, down); });
}

int hep_route_plan(const hep_level* levels, int num_levels, int rank, hep_dtype dtype, const void* x,
                   int64_t tokens, int64_t hidden, const void* w_gate, int64_t experts, int64_t top_k,
                   int32_t* topk_idx, float* topk_w, int32_t* pos, int32_t* key_counts, void* stream) {
  return guarded([&] {
    const auto c = cluster_of(levels, num_levels);
    c.validate();
    const int64_t G = c.total_gpus();
    if (rank < 0 || rank >= G) throw std::domain_error("rank out of range");
    if (experts % G) throw std::invalid_argument("experts must be divisible by the GPU count");
    if (tokens <= 0 || hidden <= 0 || top_k <= 0 || top_k > 8 || top_k > experts || experts > 64)
      throw std::invalid_argument("bad routing shape");
    const auto route = hybridep::moe::route_table(c);
    const int T = static_cast<int>(tokens), H = static_cast<int>(hidden), E = static_cast<int>(experts);
    const int k = static_cast<int>(top_k), NK = static_cast<int>(G * experts);
    const int nchunks = (T + 31) / 32;
    const hep::DType dt = dt_of(dtype);
    cudaStream_t s = st(stream);
    hep::DevBuf wg, dest, keys, ranks, cc, coff, koff, dr, doff, gs, grs, gsl, slots;
    wg.alloc(static_cast<size_t>(experts * hidden * hep::dtype_bytes(dt)));
    cuda_ok(hep::launch_transpose_convert(dt, w_gate, hidden, experts, dt, wg.p, s), "gate layout");
    dest.alloc(sizeof(int) * G);
    cuda_ok(cudaMemcpyAsync(dest.p, route.data() + rank * G, sizeof(int) * G, cudaMemcpyHostToDevice, s), "route");
    keys.alloc(sizeof(int) * T * k);
    ranks.alloc(sizeof(int) * T * k);
    cc.alloc(sizeof(int) * nchunks * NK);
    coff.alloc(sizeof(int) * nchunks * NK);
    koff.alloc(sizeof(int) * NK);
    dr.alloc(sizeof(int) * G);
    doff.alloc(sizeof(int) * G);
    gs.alloc(sizeof(int) * E);
    grs.alloc(sizeof(int) * E);
    gsl.alloc(sizeof(int) * E);
    std::vector<int32_t> none(static_cast<size_t>(E), -1);
    slots.alloc(sizeof(int) * E);
    cuda_ok(cudaMemcpyAsync(slots.p, none.data(), sizeof(int) * E, cudaMemcpyHostToDevice, s), "slots");
    cuda_ok(hep::launch_gate(dt, x, wg.p, T, H, E, k, dest.as<int>(), static_cast<int>(experts / G), NK, topk_idx,
                             topk_w, keys.as<int>(), ranks.as<int>(), cc.as<int>(), s), "gate");
    cuda_ok(hep::launch_chunk_scan(cc.as<int>(), nchunks, NK, coff.as<int>(), key_counts, s), "chunk scan");
    cuda_ok(hep::launch_key_scan(key_counts, static_cast<int>(G), E, rank, slots.as<int>(), koff.as<int>(), dr.as<int>(),
                                 doff.as<int>(), gs.as<int>(), grs.as<int>(), gsl.as<int>(), s), "key scan");
    cuda_ok(hep::launch_positions(T, k, NK, keys.as<int>(), ranks.as<int>(), coff.as<int>(), koff.as<int>(), pos, s),
            "positions");
    cuda_ok(cudaStreamSynchronize(s), "route sync");  // scratch buffers are freed on return
  });
}

int hep_grouped_gemm(hep_dtype dtype, const void* A, int64_t a_rows, const void* B, int64_t b_slots, void* C,
                     int64_t N, int64_t K, const int32_t* g_row_start, const int32_t* g_rows,
                     const int32_t* g_slot, int num_groups, int relu, uint32_t sched, void* stream) {
  return guarded([&] {
    int dev = 0, sms = 148;
    cuda_ok(cudaGetDevice(&dev), "device");
    cuda_ok(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    if (num_groups <= 0 || a_rows < 0 || b_slots <= 0 || N <= 0 || K <= 0)
      throw std::invalid_argument("grouped GEMM needs groups, rows >= 0 and positive N, K");
    hep::GroupTable gt{g_row_start, g_rows, g_slot, num_groups};
    cudaStream_t s = st(stream);
    if (dt_of(dtype) == hep::DType::BF16) {
      CUtensorMap ma, mb;
      const bool pair = hep::gemm_use_cta_pair();
      // sched 0: the schedule the layer would pick for this shape (rows per group ~ a_rows / groups)
      if (sched == 0)
        sched = hep::gemm_schedule(static_cast<int>(a_rows / num_groups), static_cast<int>(N), static_cast<int>(K),
                                   N > K);
      cuda_ok(hep::make_tmap_bf16_2d(&ma, A, static_cast<uint64_t>(std::max<int64_t>(a_rows, 1)),
                                     static_cast<uint64_t>(K), 128, 64), "tmap A");
      cuda_ok(hep::make_tmap_bf16_2d(&mb, B, static_cast<uint64_t>(b_slots * N), static_cast<uint64_t>(K), pair ? 128 : 256, 64), "tmap B");
      if (pair) {
        // HEP_GEMM_DYN=1: the dynamic tile scheduler, with a counter for this launch only
        const char* dyn = std::getenv("HEP_GEMM_DYN");
        int* ctr = nullptr;
        if (dyn && dyn[0] == '1') cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&ctr), sizeof(int), s), "tile counter");
        cuda_ok(hep::launch_grouped_gemm_bf16_2cta(ma, mb, C, static_cast<int>(N), static_cast<int>(N), static_cast<int>(K),
                                                   gt, relu, sms, s, sched, ctr),
                "gemm bf16 2cta");
        if (ctr) cuda_ok(cudaFreeAsync(ctr, s), "tile counter free");
      }
      else
        cuda_ok(hep::launch_grouped_gemm_bf16(ma, mb, C, static_cast<int>(N), static_cast<int>(N), static_cast<int>(K), gt, relu, sms, s, sched), "gemm bf16");
      return;
    }
    const char* f32 = std::getenv("HEP_F32_GEMM");
    if ((f32 && std::string(f32) == "simt") || N % 32 || K % hep::kTf32BK) {
      cuda_ok(hep::launch_grouped_gemm_f32(static_cast<const float*>(A), static_cast<int>(K), static_cast<const float*>(B),
                                           static_cast<float*>(C), static_cast<int>(N), static_cast<int>(N), static_cast<int>(K), gt,
                                           relu, sms * 2, s), "gemm f32");
      return;
    }
    // The fp32 product path the layer runs: 3xTF32 on tcgen05 over hi/lo operand splits
    // (scratch allocated stream-ordered for this call).
    // B pre-split into hi/lo copies (HEP_TF32_RAWB=1: raw B split in shared memory).
    const char* raw = std::getenv("HEP_TF32_RAWB");
    const bool presplit = !(raw && raw[0] == '1');
    const size_t a_n = static_cast<size_t>(std::max<int64_t>(a_rows, 1) * K), b_n = static_cast<size_t>(b_slots * N * K);
    float* buf = nullptr;
    cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&buf), sizeof(float) * 2 * (a_n + (presplit ? b_n : 0)), s),
            "gemm scratch");
    float *ahi = buf, *alo = buf + a_n;
    cuda_ok(hep::launch_split_tf32(static_cast<const float*>(A), ahi, alo, static_cast<int64_t>(a_n), s), "split A");
    CUtensorMap t_ahi, t_alo, t_bhi, t_blo;
    const uint64_t ar = static_cast<uint64_t>(std::max<int64_t>(a_rows, 1)), br = static_cast<uint64_t>(b_slots * N);
    cuda_ok(hep::make_tmap_f32_2d(&t_ahi, ahi, ar, static_cast<uint64_t>(K), 128, hep::kTf32BK), "tmap");
    cuda_ok(hep::make_tmap_f32_2d(&t_alo, alo, ar, static_cast<uint64_t>(K), 128, hep::kTf32BK), "tmap");
    if (presplit) {
      float *bhi = alo + a_n, *blo = bhi + b_n;
      cuda_ok(hep::launch_split_tf32(static_cast<const float*>(B), bhi, blo, static_cast<int64_t>(b_n), s), "split B");
      cuda_ok(hep::make_tmap_f32_2d(&t_bhi, bhi, br, static_cast<uint64_t>(K), 256, hep::kTf32BK), "tmap");
      cuda_ok(hep::make_tmap_f32_2d(&t_blo, blo, br, static_cast<uint64_t>(K), 256, hep::kTf32BK), "tmap");
    } else {
      cuda_ok(hep::make_tmap_f32_2d(&t_bhi, B, br, static_cast<uint64_t>(K), 256, hep::kTf32BK), "tmap");
    }
    cuda_ok(hep::launch_grouped_gemm_tf32x3(t_ahi, t_alo, t_bhi, presplit ? &t_blo : nullptr, static_cast<float*>(C), nullptr,
                                            static_cast<int>(N), static_cast<int>(N), static_cast<int>(K), gt, relu, sms, s),
            "gemm tf32x3");
    cuda_ok(cudaFreeAsync(buf, s), "gemm scratch free");
  });
}

int hep_transpose_convert(hep_dtype in_dtype, const void* in, int64_t rows, int64_t cols, hep_dtype out_dtype, void* out,
                          void* stream) {
  return guarded([&] {
    cuda_ok(hep::launch_transpose_convert(dt_of(in_dtype), in, rows, cols, dt_of(out_dtype), out, st(stream)), "transpose");
  });
}

}  // extern "C"
