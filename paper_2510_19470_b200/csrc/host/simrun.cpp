// Discrete-event run of one MoE iteration's job DAG and the model checks built on it.
// API of the reference's simcore.hpp:53-138; behaviour restated from simcore.cpp:268-498:
//   * resources: one compute lane per GPU (jobs with level < 0) and one outbound NIC per
//     (GPU, level); a resource runs one job at a time;
//   * a job becomes eligible when all its dependencies have finished; a free resource
//     starts its eligible job with the LOWEST id (program order: an earlier layer's
//     foreground traffic beats a later layer's prefetch);
//   * completions are processed in (end time, job id) order; makespan = last end;
//   * AG stall = max over (GPU, layer) of (last AG transfer touching the GPU) minus
//     (that GPU's pre-expert end), floored at 0.
// Used here to put the paper's modelling claim next to B200 measurements
// (tools/model_vs_measured.py): the DAG is fed measured kernel and NVLink numbers and
// its makespan is compared with the measured step.

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <map>
#include <ostream>
#include <queue>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>

#include "hybridep/simcore.hpp"

namespace hybridep::sim {

namespace {

constexpr std::int64_t kSimGpuLimit = 512;

double relative_error(double sim, double model) {
  if (model == 0) return sim == 0 ? 0.0 : std::numeric_limits<double>::infinity();
  return std::fabs(sim - model) / std::fabs(model);
}

}  // namespace

IterationTrace run(const JobGraph& graph, const topo::ClusterSpec& cluster) {
  const std::int64_t G = cluster.total_gpus();
  const int L = cluster.level_count();
  if (G != graph.gpus || L != graph.levels) throw std::invalid_argument("job graph was built for a different cluster");
  const std::size_t n = graph.jobs.size();
  auto lane = [&](const Job& j) -> std::size_t {
    return static_cast<std::size_t>(j.level < 0 ? j.gpu : G + j.gpu * L + j.level);
  };
  const std::size_t lanes = static_cast<std::size_t>(G + G * L);

  std::vector<std::int64_t> waiting(n, 0);
  std::vector<std::vector<std::int64_t>> children(n);
  for (const Job& j : graph.jobs) {
    waiting[static_cast<std::size_t>(j.id)] = static_cast<std::int64_t>(j.deps.size());
    for (std::int64_t d : j.deps) {
      if (d < 0 || d >= static_cast<std::int64_t>(n)) throw std::invalid_argument("dangling dependency");
      children[static_cast<std::size_t>(d)].push_back(j.id);
    }
  }

  IterationTrace trace;
  trace.records.assign(n, TraceRecord{});
  trace.level_bytes.assign(static_cast<std::size_t>(L), 0.0);
  std::vector<std::set<std::int64_t>> ready(lanes);  // eligible job ids per lane
  std::vector<char> busy(lanes, 0);
  using Event = std::pair<double, std::int64_t>;     // (end time, job)
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> events;

  auto try_start = [&](std::size_t r, double now) {
    if (busy[r] || ready[r].empty()) return;
    const std::int64_t id = *ready[r].begin();
    ready[r].erase(ready[r].begin());
    TraceRecord& rec = trace.records[static_cast<std::size_t>(id)];
    rec.job = id;
    rec.start = now;
    rec.end = now + graph.jobs[static_cast<std::size_t>(id)].duration;
    busy[r] = 1;
    events.emplace(rec.end, id);
  };

  for (const Job& j : graph.jobs)
    if (j.deps.empty()) ready[lane(j)].insert(j.id);
  for (std::size_t r = 0; r < lanes; ++r) try_start(r, 0.0);

  std::size_t finished = 0;
  while (!events.empty()) {
    const Event ev = events.top();
    events.pop();
    ++finished;
    const Job& j = graph.jobs[static_cast<std::size_t>(ev.second)];
    const std::size_t r = lane(j);
    busy[r] = 0;
    std::vector<std::size_t> lanes_to_try{r};
    for (std::int64_t c : children[static_cast<std::size_t>(ev.second)]) {
      if (--waiting[static_cast<std::size_t>(c)] == 0) {
        const std::size_t cr = lane(graph.jobs[static_cast<std::size_t>(c)]);
        ready[cr].insert(c);
        lanes_to_try.push_back(cr);
      }
    }
    for (std::size_t t : lanes_to_try) try_start(t, ev.first);
    trace.makespan = std::max(trace.makespan, trace.records[static_cast<std::size_t>(ev.second)].end);
    if (j.level >= 0) trace.level_bytes[static_cast<std::size_t>(j.level)] += j.bytes;
  }
  if (finished != n) throw std::runtime_error("job graph has a dependency cycle");

  std::map<std::pair<std::int64_t, int>, double> pre_end, ag_end;
  for (const Job& j : graph.jobs) {
    const double end = trace.records[static_cast<std::size_t>(j.id)].end;
    if (j.kind == JobKind::PreExpert) {
      pre_end[{j.gpu, j.layer}] = end;
    } else if (j.kind == JobKind::AgTransfer) {
      for (std::int64_t g : {j.gpu, j.peer}) {
        double& v = ag_end.try_emplace({g, j.layer}, end).first->second;
        v = std::max(v, end);
      }
    }
  }
  for (const auto& [key, t] : ag_end) {
    const auto it = pre_end.find(key);
    if (it != pre_end.end()) trace.max_ag_stall = std::max(trace.max_ag_stall, std::max(0.0, t - it->second));
  }
  return trace;
}

double iteration_latency(const IterationTrace& trace) { return trace.makespan; }

void write_trace_csv(const JobGraph& graph, const IterationTrace& trace, std::ostream& os) {
  struct Row {
    double time;
    std::int64_t job;
    int end;  // 0 start, 1 end
  };
  std::vector<Row> rows;
  rows.reserve(trace.records.size() * 2);
  for (const TraceRecord& r : trace.records) {
    rows.push_back({r.start, r.job, 0});
    rows.push_back({r.end, r.job, 1});
  }
  std::sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) {
    return a.time != b.time ? a.time < b.time : (a.end != b.end ? a.end < b.end : a.job < b.job);
  });
  os.precision(std::numeric_limits<double>::max_digits10);
  os << "time,gpu,resource,job,kind,layer,peer,event\n";
  for (const Row& r : rows) {
    const Job& j = graph.jobs[static_cast<std::size_t>(r.job)];
    os << r.time << ',' << j.gpu << ',' << (j.level < 0 ? std::string("compute") : "nic" + std::to_string(j.level))
       << ',' << j.id << ',' << to_string(j.kind) << ',' << j.layer << ',' << j.peer << ','
       << (r.end ? "end" : "start") << '\n';
  }
}

bool causally_ordered(const JobGraph& graph, const IterationTrace& trace) {
  for (const Job& j : graph.jobs)
    for (std::int64_t d : j.deps)
      if (trace.records[static_cast<std::size_t>(j.id)].start < trace.records[static_cast<std::size_t>(d)].end)
        return false;
  return true;
}

TraceComponents measured_components(const JobGraph& graph, const IterationTrace& trace) {
  TraceComponents c;
  for (const Job& j : graph.jobs) {
    if (j.layer != 0) continue;
    const TraceRecord& r = trace.records[static_cast<std::size_t>(j.id)];
    if (j.kind == JobKind::PreExpert) c.pre_expert = std::max(c.pre_expert, r.end - r.start);
    if (j.kind == JobKind::AgTransfer) c.ag = std::max(c.ag, r.end);
  }
  c.a2a = std::max(0.0, trace.makespan - std::max(c.pre_expert, c.ag)) / 2.0;
  return c;
}

ModelComparison validate_against_model(const topo::ClusterSpec& cluster, const perf::WorkloadSpec& workload,
                                       const HybridPlan& plan) {
  const JobGraph graph = build_schedule(cluster, workload, plan);
  const IterationTrace trace = run(graph, with_domain_sizes(cluster, plan.domain_sizes));
  perf::DeviceSpec dev;
  dev.bandwidth_B = cluster.levels.front().bandwidth;
  dev.throughput_C = 1.0;  // latencies are given directly
  const perf::LatencyBreakdown model = perf::final_latency(plan.p, workload, dev, cluster.total_gpus());
  const TraceComponents sim = measured_components(graph, trace);
  ModelComparison m;
  m.sim_pre_expert = sim.pre_expert;
  m.sim_ag = sim.ag;
  m.sim_a2a = sim.a2a;
  m.sim_total = trace.makespan + workload.backward_allreduce_const;
  m.model_pre_expert = model.pre_expert;
  m.model_ag = model.comm_ag;
  m.model_a2a = model.comm_a2a;
  m.model_total = model.total;
  m.pre_expert_error = relative_error(m.sim_pre_expert, m.model_pre_expert);
  m.ag_error = relative_error(m.sim_ag, m.model_ag);
  m.a2a_error = relative_error(m.sim_a2a, m.model_a2a);
  m.total_error = relative_error(m.sim_total, m.model_total);
  return m;
}

EpComparison compare_ep(const topo::ClusterSpec& cluster, const perf::WorkloadSpec& workload, Engine engine) {
  cluster.validate();
  workload.validate();
  const std::int64_t G = cluster.total_gpus();
  perf::DeviceSpec dev;
  dev.bandwidth_B = cluster.levels.front().bandwidth;
  dev.throughput_C = 1.0;
  EpComparison out;
  out.plan = perf::solve_optimal_p(workload, dev, G);
  const HybridPlan hybrid = make_plan(out.plan, cluster);
  HybridPlan ep;
  ep.p = 1.0;
  ep.domain_sizes.assign(cluster.levels.size(), 1);
  const topo::ClusterSpec ep_cluster = with_domain_sizes(cluster, ep.domain_sizes);
  const topo::ClusterSpec hy_cluster = with_domain_sizes(cluster, hybrid.domain_sizes);
  if (engine == Engine::EventDriven && G <= kSimGpuLimit) {
    out.ep_latency = run(build_schedule(cluster, workload, ep), ep_cluster).makespan + workload.backward_allreduce_const;
    out.hybrid_latency =
        run(build_schedule(cluster, workload, hybrid), hy_cluster).makespan + workload.backward_allreduce_const;
  } else {
    out.ep_latency = perf::final_latency(1.0, workload, dev, G).total;
    out.hybrid_latency = out.plan.latency.total;
  }
  out.speedup = out.ep_latency / out.hybrid_latency;
  const topo::CommTopology ep_topo(ep_cluster), hy_topo(hy_cluster);
  out.ep_frequency = ep_topo.frequencies();
  out.hybrid_frequency = hy_topo.frequencies();
  out.ep_traffic = topo::traffic_report(ep_topo, workload, {ep.p, ep.domain_sizes});
  out.hybrid_traffic = topo::traffic_report(hy_topo, workload, {hybrid.p, hybrid.domain_sizes});
  return out;
}

}  // namespace hybridep::sim
