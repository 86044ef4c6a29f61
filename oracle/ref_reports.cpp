// ORACLE — test infrastructure only.  Drives the UNMODIFIED reference CLI code
// (cli_app.cpp run_plan / run_topo, compiled from /root/reference by oracle/Makefile)
// on a programmatic config, so oracle/gen_golden.py can record the reference's own
// plan.json / freq.json / topo.csv for the planner-report parity test.
//   ref_reports OUT_DIR D PE n attn expert C B SF0,SF1,.. [SED0,SED1,..]
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "hybridep/cli_app.hpp"

using namespace hybridep;

static std::vector<std::int64_t> ints(const std::string& s) {
  std::vector<std::int64_t> v;
  std::stringstream ss(s);
  std::string t;
  while (std::getline(ss, t, ',')) v.push_back(std::stoll(t));
  return v;
}

int main(int argc, char** argv) {
  if (argc < 10) {
    std::cerr << "usage: ref_reports OUT D PE n attn expert C B SF [SED]\n";
    return 2;
  }
  cfg::AppConfig c;
  const auto sf = ints(argv[9]);
  for (auto s : sf) c.cluster.levels.push_back({s, 1, std::atof(argv[8])});
  c.workload.data_size_D = std::atof(argv[2]);
  c.workload.expert_size_PE = std::atof(argv[3]);
  c.workload.experts_per_gpu_n = std::atoll(argv[4]);
  c.workload.attn_latency = std::atof(argv[5]);
  c.workload.ffn_latency = 1e-12;
  c.workload.expert_latency = std::atof(argv[6]);
  c.device.throughput_C = std::atof(argv[7]);
  c.device.bandwidth_B = std::atof(argv[8]);
  if (argc > 10) c.plan.domain_sizes = ints(argv[10]);
  cli::Options opt;
  opt.out_dir = argv[1];
  return cli::run_plan(c, opt) | cli::run_topo(c, opt);
}
