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
#include <vector>

#include "hybridep/topology.hpp"

namespace hybridep::moe {

// route[m * G + o] = GPU that computes, for tokens living on m, the experts owned by o.
// Throws std::invalid_argument when some (m, o) has no route (never at G = 8).
std::vector<std::int32_t> route_table(const topo::ClusterSpec& cluster);

// held[m] = owners whose experts GPU m holds after the All-Gather (m first, then its
// AG peers in peer_lists order).
std::vector<std::vector<std::int64_t>> held_owners(const topo::ClusterSpec& cluster);

}  // namespace hybridep::moe
