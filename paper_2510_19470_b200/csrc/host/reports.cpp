// The planner's reports in the reference's formats (cli_app.cpp:183-243): plan.json
// (run_plan: resolve_plan + plan_json, cli_app.cpp:132-168, 70-80), freq.json and
// topo.csv (run_topo: per-level directed pair counts, the stripe-model traffic report,
// the dense pair table).  The B200 build feeds them MEASURED device numbers (bench.py's
// calibration: expert-GEMM throughput C, NVLink bandwidth B, pre-expert time) instead of
// a JSON config, so the modelling-selected S_ED of cfg5 is re-derived on every run.
// Keys and structure follow the reference; numbers are printed shortest-round-trip.

#include <charconv>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "hybridep/moe.hpp"
#include "hybridep/perfmodel.hpp"
#include "hybridep/plan.hpp"
#include "hybridep/topology.hpp"

namespace hybridep::moe {

namespace {

std::string num(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // a JSON float stays a float
  return s;
}

std::string num(std::int64_t v) { return std::to_string(v); }

std::string ilist(const std::vector<std::int64_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + num(v[i]);
  return s + "]";
}

void write(const std::string& dir, const std::string& name, const std::string& body) {
  std::filesystem::create_directories(dir);
  const std::filesystem::path path = std::filesystem::path(dir) / name;
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write " + path.string());
  out << body;
}

}  // namespace

ResolvedPlan resolve_plan(const topo::ClusterSpec& cluster, const perf::WorkloadSpec& w, const perf::DeviceSpec& d,
                          const std::vector<std::int64_t>* pinned_domain_sizes) {
  const std::int64_t gpus = cluster.total_gpus();
  if (gpus < 2) throw std::invalid_argument("planning needs at least 2 GPUs");
  ResolvedPlan out;
  out.config_case = perf::classify_case(w.data_size_D, w.expert_size_PE, gpus);
  out.continuous_p = perf::continuous_optimal_p(w, d, gpus);
  out.boundary_p = perf::case_boundary_p(w, d, gpus);
  if (pinned_domain_sizes) {
    out.domain_sizes = *pinned_domain_sizes;
    (void)with_domain_sizes(cluster, out.domain_sizes);  // validates per level
    std::int64_t total = 1;
    for (std::int64_t s : out.domain_sizes) total *= s;
    const double p = static_cast<double>(gpus - total) / static_cast<double>(gpus - 1);
    out.point = perf::evaluate_plan_point(p, total, w, d, gpus);
  } else {
    out.point = perf::solve_optimal_p(w, d, gpus);
    out.domain_sizes = factor_domain_sizes(out.point.domain_size, cluster);
  }
  return out;
}

void write_plan_reports(const topo::ClusterSpec& cluster, const perf::WorkloadSpec& w, const ResolvedPlan& plan,
                        const std::string& out_dir) {
  const std::int64_t gpus = cluster.total_gpus();
  const auto& L = plan.point.latency;
  std::ostringstream pj;
  pj << "{\n"
     << "  \"boundary_p\": " << num(plan.boundary_p) << ",\n"
     << "  \"case\": \"" << perf::to_string(plan.config_case) << "\",\n"
     << "  \"continuous_p\": " << num(plan.continuous_p) << ",\n"
     << "  \"domain_size\": " << num(plan.point.domain_size) << ",\n"
     << "  \"domain_sizes_per_level\": " << ilist(plan.domain_sizes) << ",\n"
     << "  \"gpus\": " << num(gpus) << ",\n"
     << "  \"latency\": {\n"
     << "    \"a2a_s\": " << num(L.comm_a2a) << ",\n"
     << "    \"ag_s\": " << num(L.comm_ag) << ",\n"
     << "    \"comp_s\": " << num(L.comp) << ",\n"
     << "    \"overlap_s\": " << num(L.overlap) << ",\n"
     << "    \"pre_expert_s\": " << num(L.pre_expert) << ",\n"
     << "    \"total_s\": " << num(L.total) << "\n"
     << "  },\n"
     << "  \"on_grid\": true,\n"
     << "  \"p\": " << num(plan.point.p) << ",\n"
     << "  \"point_case\": \"" << perf::to_string(plan.point.case_tag) << "\"\n"
     << "}\n";
  write(out_dir, "plan.json", pj.str());

  const topo::ClusterSpec planned = with_domain_sizes(cluster, plan.domain_sizes);
  const topo::CommTopology topology = topo::build_topology(planned);
  const topo::TrafficReport traffic = topo::traffic_report(topology, w, {plan.point.p, plan.domain_sizes});
  const topo::FrequencyReport& f = topology.frequencies();
  std::ostringstream fj;
  fj << "{\n  \"domain_sizes_per_level\": " << ilist(plan.domain_sizes) << ",\n  \"levels\": [\n";
  for (size_t l = 0; l < f.levels.size(); ++l)
    fj << "    {\n      \"a2a\": " << f.levels[l].a2a << ",\n      \"ag\": " << f.levels[l].ag
       << ",\n      \"level\": " << l << "\n    }" << (l + 1 < f.levels.size() ? ",\n" : "\n");
  fj << "  ],\n  \"p\": " << num(plan.point.p) << ",\n  \"total_a2a\": " << f.total_a2a()
     << ",\n  \"total_ag\": " << f.total_ag() << ",\n  \"traffic\": {\n    \"levels\": [\n";
  for (size_t l = 0; l < traffic.levels.size(); ++l)
    fj << "      {\n        \"a2a_bytes\": " << num(traffic.levels[l].a2a_bytes) << ",\n        \"ag_bytes\": "
       << num(traffic.levels[l].ag_bytes) << ",\n        \"level\": " << l << "\n      }"
       << (l + 1 < traffic.levels.size() ? ",\n" : "\n");
  fj << "    ],\n    \"total_a2a_bytes\": " << num(traffic.total_a2a()) << ",\n    \"total_ag_bytes\": "
     << num(traffic.total_ag()) << ",\n    \"total_bytes\": " << num(traffic.total()) << "\n  }\n}\n";
  write(out_dir, "freq.json", fj.str());
  if (topology.dense()) {
    std::ostringstream csv;
    topology.write_pairs_csv(csv);
    write(out_dir, "topo.csv", csv.str());
  }
}

}  // namespace hybridep::moe
