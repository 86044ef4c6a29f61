// Token routing derived from the topology table.
// The reference has no router; these rules are the pinned semantics stated in
// include/hybridep/moe.hpp and are checked bit-for-bit by the CPU oracle
// (oracle/moe_oracle.c: oracle_route_table) in tests/test_host.py.

#include "hybridep/moe.hpp"

#include <stdexcept>

#include "hybridep/simcore.hpp"

namespace hybridep::moe {

std::vector<std::int32_t> route_table(const topo::ClusterSpec& cluster) {
  const topo::CommTopology topo(cluster);
  const std::int64_t G = topo.gpus();
  if (!topo.dense()) throw std::invalid_argument("route table needs a dense topology (G <= 4096)");
  const std::vector<sim::PeerLists> peers = sim::peer_lists(cluster);
  auto kind = [&](std::int64_t a, std::int64_t b) {
    return a == b ? topo::CommType::None : topo.classify(a, b).type;
  };
  std::vector<std::int32_t> route(static_cast<std::size_t>(G * G), -1);
  for (std::int64_t m = 0; m < G; ++m) {
    for (std::int64_t o = 0; o < G; ++o) {
      std::int64_t d = -1;
      if (m == o || kind(m, o) == topo::CommType::AG) {
        d = m;
      } else if (kind(m, o) == topo::CommType::A2A) {
        d = o;
      } else {
        // Relay: first A2A peer of m (peer-list order) that holds o's experts.
        for (const auto& level : peers[m].a2a) {
          for (std::int64_t n : level)
            if (n == o || kind(n, o) == topo::CommType::AG) {
              d = n;
              break;
            }
          if (d >= 0) break;
        }
      }
      if (d < 0)
        throw std::invalid_argument("no route from GPU " + std::to_string(m) + " to the experts of GPU " +
                                    std::to_string(o));
      route[static_cast<std::size_t>(m * G + o)] = static_cast<std::int32_t>(d);
    }
  }
  return route;
}

std::vector<std::vector<std::int64_t>> held_owners(const topo::ClusterSpec& cluster) {
  const std::vector<sim::PeerLists> peers = sim::peer_lists(cluster);
  std::vector<std::vector<std::int64_t>> held(peers.size());
  for (std::size_t m = 0; m < peers.size(); ++m) {
    held[m].push_back(static_cast<std::int64_t>(m));
    for (const auto& level : peers[m].ag) held[m].insert(held[m].end(), level.begin(), level.end());
  }
  return held;
}

}  // namespace hybridep::moe
