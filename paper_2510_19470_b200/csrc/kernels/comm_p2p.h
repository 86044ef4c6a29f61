// NVLink peer-memory dispatch/combine (comm_p2p.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace hep {

constexpr int kMaxG = 8;
constexpr int kSyncSlots = 5;  // flag slots per rank's sync buffer (see launch_signal_wait)
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
  int recv_start;               // first receive row (Tmax * k), same on every rank (checked at setup)
  int row_bytes;                // H * element bytes of xall / oall rows
  uint32_t epoch;
  uint64_t timeout_ns;          // flag waits trap after this long (0: wait forever); HEP_P2P_TIMEOUT_S
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
// slot 3 (AG peers): "my experts for this epoch are final, pull them";
// slot 4 (AG peers): "I have pulled your wires of this epoch" (before they are rewritten).
// sig = false: wait only; wait = false: signal only.
cudaError_t launch_signal_wait(const P2PArgs& a, int slot, cudaStream_t s, bool wait = true, bool ag_peers = false,
                               bool sig = true);
// This rank's dispatch flags (indexed by source rank), for GEMM-side gating.
const uint32_t* p2p_dispatch_flags(const P2PArgs& a);
cudaError_t launch_combine_p2p(const P2PArgs& a, DType dt, const int* keys, const int* pos, const int* key_off,
                               const int* send_base, const float* w, int T, int H, int k, void* y,
                               cudaStream_t s, const void* residual = nullptr);

// Shared-expert refresh across the ranks (comm_p2p.cu): the fp64 sum over every expert in
// expert order as a chain over ranks 0..G-1, chunked so the ranks pipeline.
struct ChainArgs {
  const float* master;          // this rank's n fp32 experts, flat [n][P]
  const double* pred_partial;   // rank-1's partial (peer memory); unused on rank 0
  const uint32_t* pred_flags;   // rank-1's chunk flags (peer memory)
  double* partial;              // this rank's partial (read by rank+1)
  uint32_t* my_flags;           // this rank's chunk flags
  const float* last_shared;     // the last rank's mean (peer memory)
  const uint32_t* last_flags;   // the last rank's chunk flags (peer memory)
  float* shared;                // this rank's copy of the mean
  uint32_t* bar[kMaxG];         // every rank's barrier flags ([kMaxG], after its chunk flags)
  int64_t P, chunk;
  int n, rank, G;
  double inv;                   // 1 / E
  uint32_t epoch;               // 0: no flags (the NCCL path moves the partials)
  uint64_t timeout_ns;          // as P2PArgs::timeout_ns
};
constexpr int64_t kChainChunk = 65536;  // elements per pipelined chunk
cudaError_t launch_shared_chain(const ChainArgs& c, cudaStream_t s);

}  // namespace hep
