// The C++ step API (include/hybridep/moe.hpp) as a reference-style C++ caller uses it:
// RAII handles over the C-ABI that rethrow the reference's exception types
// (std::domain_error / std::invalid_argument / std::runtime_error), the planner reports,
// and -- with argument "gpu OUT_DIR" -- one small MoE-layer forward whose output
// tests/test_cpp_api.py checks against the oracle.
//   test_moe_api            : host checks (no GPU needed)
//   test_moe_api gpu DIR    : + a forward on cuda:0, writing DIR/{x,wg,up,down,y}.bin
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "hybridep/moe.hpp"

using namespace hybridep;

static int failures = 0;
#define EXPECT(cond)                                                     \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static moe::LayerConfig small(int rank = 0) {
  moe::LayerConfig c;
  c.hidden = 256;
  c.ffn = 512;
  c.experts = 8;
  c.top_k = 2;
  c.max_tokens = 64;
  c.dtype = HEP_BF16;
  c.cluster.levels = {{1, 1, 1e9}};
  c.rank = rank;
  return c;
}

static void host_checks() {
  auto bad = small();
  bad.hidden = 0;
  EXPECT(throws<std::invalid_argument>([&] { moe::Layer l(bad); }));
  bad = small();
  bad.top_k = 9;
  EXPECT(throws<std::invalid_argument>([&] { moe::Layer l(bad); }));
  auto oob = small(3);  // rank outside a 1-GPU cluster
  EXPECT(throws<std::domain_error>([&] { moe::Layer l(oob); }));
  EXPECT(throws<std::invalid_argument>([] { moe::Communicator::virtual_ranks(0); }));
  auto vr = moe::Communicator::virtual_ranks(2);
  EXPECT(vr.size() == 2 && vr[1].rank() == 1 && vr[1].nranks() == 2);
  auto two = small(0);
  two.cluster.levels = {{2, 1, 1e9}};
  EXPECT(throws<std::invalid_argument>([&] { moe::Layer l(two); }));  // G = 2 needs a communicator
  // planner + reports (reference formats)
  topo::ClusterSpec c;
  c.levels = {{2, 1, 7.4e11}, {4, 1, 7.4e11}};
  perf::WorkloadSpec w;
  w.data_size_D = 2.68e8;
  w.expert_size_PE = 2.35e8;
  w.experts_per_gpu_n = 1;
  w.attn_latency = 1.7e-4;
  w.ffn_latency = 1e-12;
  w.expert_latency = 2.7e-3;
  const auto plan = moe::resolve_plan(c, w, perf::DeviceSpec{1.4e15, 7.4e11});
  EXPECT(plan.domain_sizes.size() == 2);
  const std::vector<std::int64_t> pin = {1, 4};
  const auto pinned = moe::resolve_plan(c, w, perf::DeviceSpec{1.4e15, 7.4e11}, &pin);
  EXPECT(pinned.domain_sizes == pin && pinned.point.domain_size == 4);
  const std::vector<std::int64_t> off = {1, 3};
  EXPECT(throws<std::invalid_argument>([&] { moe::resolve_plan(c, w, perf::DeviceSpec{1.4e15, 7.4e11}, &off); }));
}

template <typename T>
static void dump(const std::string& path, const std::vector<T>& v) {
  std::ofstream(path, std::ios::binary).write(reinterpret_cast<const char*>(v.data()), sizeof(T) * v.size());
}

static unsigned short bf16(float f) {
  unsigned u;
  std::memcpy(&u, &f, 4);
  return static_cast<unsigned short>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

static void gpu_forward(const std::string& dir) {
  auto cfg = small();
  const int64_t H = cfg.hidden, F = cfg.ffn, E = cfg.experts, T = 50;
  std::vector<unsigned short> x(T * H), wg(H * E), up(E * H * F), down(E * F * H);
  unsigned s = 12345;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return static_cast<int>((s >> 8) % 17) - 8; };
  for (auto& v : x) v = bf16(rnd() / 16.0f);
  for (auto& v : wg) v = bf16(rnd() / 16.0f);
  for (auto& v : up) v = bf16(rnd() / 512.0f);
  for (auto& v : down) v = bf16(rnd() / 512.0f);
  void *dx, *dwg, *dup, *ddown, *dy;
  cudaMalloc(&dx, 2 * x.size());
  cudaMalloc(&dwg, 2 * wg.size());
  cudaMalloc(&dup, 2 * up.size());
  cudaMalloc(&ddown, 2 * down.size());
  cudaMalloc(&dy, 2 * x.size());
  cudaMemcpy(dx, x.data(), 2 * x.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dwg, wg.data(), 2 * wg.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dup, up.data(), 2 * up.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(ddown, down.data(), 2 * down.size(), cudaMemcpyHostToDevice);
  {
    moe::Layer layer(cfg);
    layer.set_gate(dwg, HEP_BF16, nullptr);
    for (int64_t e : layer.owned_experts())
      layer.set_expert(e, static_cast<char*>(dup) + 2 * e * H * F, static_cast<char*>(ddown) + 2 * e * F * H,
                       HEP_BF16, nullptr);
    EXPECT(throws<std::domain_error>([&] { layer.set_expert(E, dup, ddown, HEP_BF16, nullptr); }));
    EXPECT(throws<std::invalid_argument>([&] { layer.forward(dx, cfg.max_tokens + 1, dy, nullptr); }));
    layer.forward(dx, T, dy, nullptr);
    cudaDeviceSynchronize();
  }
  std::vector<unsigned short> y(T * H);
  cudaMemcpy(y.data(), dy, 2 * y.size(), cudaMemcpyDeviceToHost);
  dump(dir + "/x.bin", x);
  dump(dir + "/wg.bin", wg);
  dump(dir + "/up.bin", up);
  dump(dir + "/down.bin", down);
  dump(dir + "/y.bin", y);
}

int main(int argc, char** argv) {
  host_checks();
  if (argc > 2 && std::string(argv[1]) == "gpu") gpu_forward(argv[2]);
  if (failures) return 1;
  std::printf("C++ API checks passed\n");
  return 0;
}
