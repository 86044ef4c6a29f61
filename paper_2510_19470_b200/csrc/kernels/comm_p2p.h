// NVLink peer-memory dispatch/combine (comm_p2p.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace hep {

constexpr int kMaxG = 8;
constexpr int kMaxE = 64;

// Passed by value to every kernel: peer-mapped base pointers (index = rank; own rank
// is the local pointer) and the A2A peer lists of every rank.
struct P2PArgs {
  void* xall[kMaxG];
  void* oall[kMaxG];
  void* sync[kMaxG];
  int src_list[kMaxG * kMaxG];  // src_list[d*kMaxG + i]: i-th A2A peer of d (ring order)
  int n_src[kMaxG];
  int ag_list[kMaxG];           // this rank's All-Gather peers (ring order)
  int n_ag;
  int G, E, rank;
  int recv_start;               // first receive row (Tmax * k), same on every rank
  int row_bytes;                // H * element bytes of xall / oall rows
  uint32_t epoch;
};

size_t p2p_sync_bytes(int G, int E);
// Also writes g_out_down: where the down-projection stores each group's rows -- local
// rows into this GPU's oall, received rows straight back into the source GPU's oall at
// the rows that source's combine reads (its packed positions).
cudaError_t launch_count_exchange(const P2PArgs& a, const int* key_total, const int* key_off,
                                  const int* slot_of_expert, int* send_base, int* g_row_start, int* g_rows,
                                  int* g_slot, unsigned long long* g_out_down, int* g_wait, int* counts_out,
                                  cudaStream_t s);
cudaError_t launch_permute_p2p(const P2PArgs& a, DType dt, const void* x, int T, int H, int k, const int* keys,
                               const int* ranks, const int* chunk_off, const int* key_off, const int* send_base,
                               int* pos, cudaStream_t s, int mode = 0);
// slot 1: "my rows are in your receive area"; slot 2: "your outputs are ready";
// slot 3 (AG peers): "my experts for this epoch are final, pull them".
cudaError_t launch_signal_wait(const P2PArgs& a, int slot, cudaStream_t s, bool wait = true, bool ag_peers = false);
// This rank's dispatch flags (indexed by source rank), for GEMM-side gating.
const uint32_t* p2p_dispatch_flags(const P2PArgs& a);
cudaError_t launch_combine_p2p(const P2PArgs& a, DType dt, const int* keys, const int* pos, const int* key_off,
                               const int* send_base, const float* w, int T, int H, int k, void* y,
                               cudaStream_t s);

}  // namespace hep
