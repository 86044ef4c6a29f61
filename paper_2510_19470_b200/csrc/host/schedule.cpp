// Step plan of one MoE iteration: ring-ordered peer lists and the job DAG.
// Contract: simcore.cpp:24-74 (peer lists: AG peers by ((off_n-off_m) mod S_ED, n),
// A2A peers by ((dom_n-dom_m) mod (SF/S_ED), n)); simcore.cpp:96-266
// (build_schedule: Optimizer -> PreExpert -> AgTransfer (no deps) -> A2aDispatch ->
// ExpertChunk per source -> A2aCombine -> next layer).  The B200 executor
// (csrc/host/layer.cpp) issues its NCCL send/recv in exactly this peer order.

#include "hybridep/simcore.hpp"

#include <algorithm>
#include <stdexcept>
#include <utility>

namespace hybridep::sim {

namespace {

constexpr std::int64_t kMaxPlannedGpus = 512;

std::int64_t outer_positions(const topo::ClusterSpec& c, int level) {
  std::int64_t p = 1;
  for (int i = 0; i < level; ++i) p *= c.levels[i].scaling_factor;
  return p;
}

}  // namespace

const char* to_string(JobKind k) {
  static const char* const names[] = {"optimizer", "pre_expert", "expert_chunk",
                                      "ag",        "a2a_dispatch", "a2a_combine"};
  const auto i = static_cast<unsigned>(k);
  return i < 6 ? names[i] : "?";
}

std::int64_t JobGraph::count(JobKind kind) const {
  return std::count_if(jobs.begin(), jobs.end(), [kind](const Job& j) { return j.kind == kind; });
}

std::vector<PeerLists> peer_lists(const topo::ClusterSpec& cluster) {
  const std::int64_t G = cluster.total_gpus();
  const int L = cluster.level_count();
  std::vector<topo::MultiIndex> x(static_cast<std::size_t>(G));
  for (std::int64_t m = 0; m < G; ++m) x[m] = topo::renumber(m, cluster);

  std::vector<PeerLists> out(static_cast<std::size_t>(G));
  for (PeerLists& p : out) {
    p.ag.resize(static_cast<std::size_t>(L));
    p.a2a.resize(static_cast<std::size_t>(L));
  }
  for (std::int64_t m = 0; m < G; ++m) {
    // (ring key, peer) pairs per level, sorted afterwards.
    std::vector<std::vector<std::pair<std::int64_t, std::int64_t>>> ag(L), a2a(L);
    for (std::int64_t n = 0; n < G; ++n) {
      if (n == m) continue;
      int l = L - 1;
      while (x[m][l] == x[n][l]) --l;
      const std::int64_t sed = cluster.levels[l].domain_size;
      const std::int64_t domains = cluster.levels[l].scaling_factor / sed;
      const std::int64_t dm = x[m][l] / sed, om = x[m][l] % sed;
      const std::int64_t dn = x[n][l] / sed, on = x[n][l] % sed;
      if (dm == dn && om != on) ag[l].emplace_back((on - om + sed) % sed, n);
      if (dm != dn && om == on) a2a[l].emplace_back((dn - dm + domains) % domains, n);
    }
    for (int l = 0; l < L; ++l) {
      std::sort(ag[l].begin(), ag[l].end());
      std::sort(a2a[l].begin(), a2a[l].end());
      for (const auto& kv : ag[l]) out[m].ag[l].push_back(kv.second);
      for (const auto& kv : a2a[l]) out[m].a2a[l].push_back(kv.second);
    }
  }
  return out;
}

JobGraph build_schedule(const topo::ClusterSpec& cluster, const perf::WorkloadSpec& workload,
                        const HybridPlan& plan) {
  cluster.validate();
  workload.validate();
  const topo::ClusterSpec c = with_domain_sizes(cluster, plan.domain_sizes);
  plan.validate(c);
  const std::int64_t G = c.total_gpus();
  if (G > kMaxPlannedGpus)
    throw std::invalid_argument("event simulation is capped at 512 GPUs; use the analytic path");
  const int L = c.level_count();
  const std::vector<PeerLists> peers = peer_lists(c);

  const perf::CompLatency comp = perf::comp_stream_latency(workload);
  const double n = static_cast<double>(workload.experts_per_gpu_n);
  const std::int64_t dom = plan.total_domain_size();
  const double decode_per_layer = plan.decode_cost * n * static_cast<double>(dom - 1);
  const double encode_total =
      dom > 1 ? plan.encode_cost * n * static_cast<double>(plan.layers) : 0.0;

  JobGraph g;
  g.gpus = G;
  g.levels = L;
  auto push = [&g](Job j) {
    j.id = static_cast<std::int64_t>(g.jobs.size());
    g.jobs.push_back(std::move(j));
    return g.jobs.back().id;
  };
  auto job = [](JobKind k, int layer, std::int64_t gpu) {
    Job j;
    j.kind = k;
    j.layer = layer;
    j.gpu = gpu;
    return j;
  };

  std::vector<std::int64_t> opt(static_cast<std::size_t>(G), -1);
  if (encode_total > 0) {
    for (std::int64_t m = 0; m < G; ++m) {
      Job j = job(JobKind::Optimizer, -1, m);
      j.duration = encode_total;
      opt[m] = push(std::move(j));
    }
  }

  std::vector<std::vector<std::int64_t>> carried(static_cast<std::size_t>(G));
  for (int layer = 0; layer < plan.layers; ++layer) {
    std::vector<std::int64_t> pre(static_cast<std::size_t>(G));
    for (std::int64_t m = 0; m < G; ++m) {
      Job j = job(JobKind::PreExpert, layer, m);
      j.duration = comp.pre_expert;
      j.deps = carried[m];
      if (layer == 0 && opt[m] >= 0) j.deps.push_back(opt[m]);
      pre[m] = push(std::move(j));
    }

    // Expert payloads: eligible from t=0, FIFO behind earlier layers.
    std::vector<std::vector<std::int64_t>> ag_in(static_cast<std::size_t>(G));
    for (std::int64_t m = 0; m < G; ++m)
      for (int l = 0; l < L; ++l) {
        const double bytes = workload.expert_size_PE / static_cast<double>(outer_positions(c, l));
        for (std::int64_t peer : peers[m].ag[l]) {
          Job j = job(JobKind::AgTransfer, layer, m);
          j.level = l;
          j.peer = peer;
          j.bytes = bytes;
          j.duration = bytes / c.levels[l].bandwidth;
          ag_in[peer].push_back(push(std::move(j)));
        }
      }

    struct Inbound {
      std::int64_t job, src;
      int level;
    };
    std::vector<std::vector<Inbound>> inbound(static_cast<std::size_t>(G));
    auto a2a_bytes = [&](int l) {
      const topo::LevelSpec& lv = c.levels[l];
      return workload.data_size_D * static_cast<double>(lv.domain_size) /
             static_cast<double>(lv.scaling_factor) / static_cast<double>(outer_positions(c, l));
    };
    for (std::int64_t m = 0; m < G; ++m)
      for (int l = 0; l < L; ++l)
        for (std::int64_t peer : peers[m].a2a[l]) {
          Job j = job(JobKind::A2aDispatch, layer, m);
          j.level = l;
          j.peer = peer;
          j.bytes = a2a_bytes(l);
          j.duration = j.bytes / c.levels[l].bandwidth;
          j.deps = {pre[m]};
          inbound[peer].push_back({push(std::move(j)), m, l});
        }

    std::vector<std::int64_t> local(static_cast<std::size_t>(G));
    std::vector<std::vector<std::int64_t>> remote(static_cast<std::size_t>(G));
    for (std::int64_t m = 0; m < G; ++m) {
      const double chunk = (n * workload.expert_latency + decode_per_layer) /
                           static_cast<double>(1 + inbound[m].size());
      Job j = job(JobKind::ExpertChunk, layer, m);
      j.peer = m;
      j.duration = chunk;
      j.deps = ag_in[m];
      j.deps.push_back(pre[m]);
      local[m] = push(std::move(j));
      for (const Inbound& in : inbound[m]) {
        Job r = job(JobKind::ExpertChunk, layer, m);
        r.peer = in.src;
        r.duration = chunk;
        r.deps = ag_in[m];
        r.deps.push_back(in.job);
        remote[m].push_back(push(std::move(r)));
      }
    }

    std::vector<std::vector<std::int64_t>> back(static_cast<std::size_t>(G));
    for (std::int64_t m = 0; m < G; ++m)
      for (std::size_t i = 0; i < inbound[m].size(); ++i) {
        const Inbound& in = inbound[m][i];
        Job j = job(JobKind::A2aCombine, layer, m);
        j.level = in.level;
        j.peer = in.src;
        j.bytes = a2a_bytes(in.level);
        j.duration = j.bytes / c.levels[in.level].bandwidth;
        j.deps = {remote[m][i]};
        back[in.src].push_back(push(std::move(j)));
      }

    for (std::int64_t m = 0; m < G; ++m) {
      carried[m] = back[m];
      carried[m].push_back(local[m]);
    }
  }
  return g;
}

}  // namespace hybridep::sim
