// MoE-layer step executor (C++ host side of the B200 path).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../kernels/comm_p2p.h"
#include "../kernels/kernels.h"
#include "hep.h"
#include "hybridep/sparsecomp.hpp"
#include "hybridep/topology.hpp"

namespace hep {

class Layer;

// Several ranks of one process on ONE device ("virtual ranks", hep_comm_init_virtual):
// the NVLink peer-memory path with the buffers exchanged as plain device pointers
// instead of CUDA IPC handles, so the fused dispatch / GEMM peer-store / combine
// kernels, the epoch flags and the shared-expert chain run unchanged on a one-GPU box.
struct VirtualGroup {
  std::mutex mu;
  int nranks = 0;
  std::map<std::pair<int, int>, Layer*> layers;  // (layer sequence number on its rank, rank)
};

struct Comm {
  ncclComm_t nccl = nullptr;
  int rank = 0;
  int nranks = 1;
  std::shared_ptr<VirtualGroup> vgroup;  // set: virtual ranks (no NCCL)
  int layers_created = 0;                // pairs the k-th layer of every rank (virtual ranks)
};

// What every rank must agree on before any peer-memory store lands in its buffers
// (ranks with different max_tokens would place rows at different receive offsets).
struct LayerSig {
  int64_t H, F, E, k, Tmax, sr_k;
  double sr_ratio;
  int32_t dtype, use_sr, per_matrix, nlev, p2p, pad;
  uint32_t iw, vw;
  int64_t sf[16], sed[16];
};

// A rank's buffers as seen from this process (IPC-mapped, or local for virtual ranks).
struct PeerBufs {
  void* xall;
  void* oall;
  void* sync;
  void* w_up;
  void* w_down;
  void* wires;
  void* partial;
  void* chain_flags;
  void* shared;
};

// Device buffer with RAII.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t n);
  void release();
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

class Layer {
 public:
  Layer(const hep_layer_params& prm, Comm* comm);
  ~Layer();

  void set_gate(const void* w_gate, DType dt, cudaStream_t s);
  void set_expert(int64_t e, const void* w_up, const void* w_down, DType dt, cudaStream_t s);
  void set_shared(const float* shared, cudaStream_t s);  // SR mode: fp32 flat P
  // SR mode: recompute the shared expert as the mean of ALL experts across the ranks
  // (reference init_shared / update_shared, sparsecomp.cpp:147-173), bit-exact with
  // the reference's sequential fp64 sum in expert order; every rank ends with it.
  void refresh_shared(cudaStream_t s);
  void get_shared(float* out, cudaStream_t s) const;  // SR mode: copy of the fp32 shared expert
  void gather_experts(cudaStream_t s);
  // SR mode: SGD step of the owned fp32 masters fused with their encode (wires ready for
  // the next gather); grads[i] flat P fp32 for owned expert rank*n + i.
  void sgd_step(const float* const* grads, int n, float lr, cudaStream_t s);
  // residual: y = x + MoE(x) (the transformer residual stream), fused into the combine
  void forward(const void* x, int64_t T, void* y, cudaStream_t s, bool residual = false);
  void forward_host(const void* hx, int64_t T, void* hy, cudaStream_t s);
  void host_fence(cudaStream_t s);
  // Communication microbenchmark: out = {a2a_ms, a2a_bytes_out, 0, ag_ms, ag_bytes_in, 0}.
  void comm_bench(const void* x, int64_t T, int iters, double* out, cudaStream_t s);

  // introspection
  const int* topk_idx() const { return topk_idx_.as<int>(); }
  const float* topk_w() const { return topk_w_.as<float>(); }
  const int* pos() const { return pos_.as<int>(); }
  // The grouped rows of the last step (materialised on demand when the up-projection
  // gathered them from x instead; an inspection path, not the step).
  const void* packed();
  const int* key_counts() const { return key_total_.as<int>(); }
  // 0 off; 1 CUDA events around the expert GEMM launches only (cheap enough for the timed
  // pass); 2 events at every phase boundary.
  void set_profiling(int level) { profiling_ = level; }  // profiled forwards run eagerly
  // Mean device time per named phase over every profiled forward since the last call.
  void collect_timings(char* names, size_t names_cap, float* ms, int cap, int* count);
  int launch_count() const { return launches_; }
  // Raises RuntimeFailure (std::runtime_error) if a gathered SR wire failed to decode
  // (bad magic, truncation, out-of-order indices: sparsecomp.cpp:36, 236-238).  With
  // sync, waits for the pending All-Gather first; otherwise reads what has completed.
  void check_migration(bool sync);
  // Test hook (hep_layer_debug_corrupt_next_gather): the next gather corrupts the magic
  // of the first gathered wire after the pull, before decode.
  void corrupt_next_gather() { corrupt_next_ = true; }
  void gemm_schedules(uint32_t* up, uint32_t* down) const {
    *up = sched_up_;
    *down = sched_down_;
  }
  bool p2p() const { return p2p_; }

 private:
  void mark(const char* name, cudaStream_t s, int level = 2);
  void build_comm_plan_and_groups(int T, cudaStream_t s);
  void exchange(bool dispatch, cudaStream_t s);
  void run_expert_gemms(cudaStream_t s, const unsigned long long* out_down = nullptr, const int* wait_src = nullptr,
                        int g0 = 0, int ng = -1, const char* tag = "", bool patched = false);
  // Fused SR decode (bf16, peer-memory path): gathered wires become per-slot patch lists
  // applied inside the GEMM's B-operand load instead of dense decoded compute copies.
  void index_gathered(size_t wire_bytes, size_t stride, cudaStream_t s);
  bool sr_fused_ = false;
  DevBuf patch_blocks_, patch_ovf_, patch_ovf_n_, patch_refs_;
  size_t patch_kmax_ = 0, patch_slot_bytes_ = 0;
  CUtensorMap map_shared_up_, map_shared_down_;
  void decode_gathered(size_t wire_bytes, size_t stride, cudaStream_t s);
  void step(const void* x, int64_t T, void* y, cudaStream_t s, bool residual);  // forward's enqueue
  // One-GPU layers replay the step as a CUDA graph, one per (x, T, y); any weight change
  // drops them.  Launched on graph_s_ with event joins to the caller's stream (capture on
  // the legacy default stream is not allowed).
  struct GraphEntry {
    const void* x;
    int64_t T;
    void* y;
    bool residual;
    cudaGraphExec_t exec;
    int launches;
  };
  std::vector<GraphEntry> graphs_;
  bool use_graphs_ = false;
  cudaStream_t graph_s_ = nullptr;
  cudaEvent_t ev_graph_in_ = nullptr, ev_graph_out_ = nullptr;
  void drop_graphs();
  bool forward_graph(const void* x, int64_t T, void* y, cudaStream_t s, bool residual);
  void gather(cudaStream_t s);                                     // gather_experts' enqueue

  // shape
  int64_t H_, F_, E_, k_, Tmax_, G_, n_, NK_;
  DType dt_;
  int rank_;
  bool use_sr_;
  hybridep::sr::CompressionConfig sr_cfg_;
  hybridep::topo::ClusterSpec cluster_;
  Comm* comm_;
  int num_sms_;

  // routing / placement
  std::vector<int32_t> route_row_;         // dest GPU for each owner
  std::vector<int64_t> held_owners_;       // owners whose experts this GPU holds
  std::vector<int32_t> slot_of_expert_;    // -1 if not held
  std::vector<int64_t> ag_peers_, a2a_peers_;
  int64_t slots_;

  // device state
  DevBuf d_route_, d_slot_of_expert_, wg_t_, w_up_c_, w_down_c_;
  DevBuf shared_, shared_c_, master_, wires_, sr_ws_, sr_tmp_, sr_status_;
  DevBuf topk_idx_, topk_w_, keys_, ranks_, chunk_counts_, chunk_off_, key_total_, key_off_;
  DevBuf dest_rows_, dest_off_, g_row_start_, g_rows_, g_slot_, all_counts_;
  DevBuf pos_, xall_, hbuf_, oall_;
  int64_t rows_cap_;
  CUtensorMap map_a1_, map_b1_, map_a2_, map_b2_;
  // fp32 layers on the tensor cores (3xTF32): every GEMM operand as a tf32 hi/lo pair
  bool tf32_ = false;
  DevBuf xhi_, xlo_, hhi_, hlo_, wuhi_, wulo_, wdhi_, wdlo_;
  CUtensorMap t_xhi_, t_xlo_, t_hhi_, t_hlo_, t_wuhi_, t_wulo_, t_wdhi_, t_wdlo_;
  std::vector<char> slot_dirty_;  // compute-copy slots whose hi/lo split is stale
  int ksplit_up_ = 1, ksplit_down_ = 1;  // split-K when the tiles alone cannot fill the SMs
  DevBuf kpart_;
  void split_dirty_slots(cudaStream_t s);
  bool tf32_presplit_ = true;  // false (HEP_TF32_RAWB=1): raw weights split in shared memory
  bool merge_gemms_ = false;   // HEP_MERGE_GEMMS=1: one launch per projection over all groups
  int merge_mode_ = 0;         // HEP_MERGE_GEMMS=2: own + received rows merged, gathered apart
  bool gather_a_ = false;     // one GPU, CTA pair: the permute fused into the up-projection's A load
  bool gather_now_ = false;   // this step's up-projection gathers A (last_x_ rows by row_src_)
  bool packed_stale_ = false; // xall_ not written by the last step (gathered A)
  const void* last_x_ = nullptr;
  int64_t last_T_ = 0;
  DevBuf row_src_;            // grouped row -> token (inverse routing map), padded by 256
  void mark_gathered_dirty();
  uint32_t sched_up_ = 0, sched_down_ = 0;
  DevBuf tile_counters_;  // dynamic tile scheduler of the CTA-pair GEMM (up, down)
  bool cta_pair_ = true;

  // NVLink peer-memory path (default for G > 1; HEP_COMM=nccl selects the NCCL baseline)
  bool p2p_ = false;
  P2PArgs p2p_args_{};
  DevBuf sync_, send_base_, g_out_down_, g_wait_;
  cudaStream_t side_s_ = nullptr;
  cudaEvent_t ev_counts_ = nullptr, ev_remote_ = nullptr, ev_arrived_ = nullptr;
  bool spin_ = false;  // HEP_GEMM_SPIN=1: GEMM producers spin on per-source dispatch flags
  // expert All-Gather overlapped with the step (copy-engine pulls over NVLink)
  cudaStream_t ag_s_ = nullptr;
  cudaEvent_t ev_ag_start_ = nullptr, ev_ag_done_ = nullptr;
  std::vector<void*> peer_w_up_, peer_w_down_, peer_wires_;
  uint32_t ag_epoch_ = 0;
  // shared-expert refresh chain (SR mode): fp64 partial sums and per-chunk flags,
  // peer-mapped from the neighbouring ranks
  DevBuf partial_, chain_flags_;
  const double* peer_partial_prev_ = nullptr;
  const uint32_t* peer_flags_prev_ = nullptr;
  const float* peer_shared_last_ = nullptr;
  const uint32_t* peer_flags_last_ = nullptr;
  std::vector<uint32_t*> peer_chain_flags_;  // every rank's chain flags (own included)
  uint32_t chain_epoch_ = 0;
  void finish_shared(cudaStream_t s);  // shared_ -> shared_c_ (GEMM layout)
  bool ag_pending_ = false;
  std::vector<void*> ipc_opened_;
  uint32_t epoch_ = 0;
  void setup_p2p();
  void setup_streams();
  LayerSig signature() const;
  PeerBufs my_bufs() const;
  void connect(const std::vector<PeerBufs>& bufs);
  void ensure_connected();  // virtual ranks: resolve peers on first use
  void check_signatures(const std::vector<LayerSig>& all) const;
  void init_host_staging();
  int seq_ = 0;
  bool connected_ = true;
  uint64_t timeout_ns_ = 0;
  bool corrupt_next_ = false;
  bool wires_fresh_ = false;  // sgd_step encoded the owned wires; the next gather reuses them
  int32_t* mig_err_host_ = nullptr;  // mapped pinned flag: a gathered wire failed to decode
  int32_t* mig_err_dev_ = nullptr;

  // per-forward plan
  int num_groups_;
  std::vector<int64_t> send_off_, send_rows_, recv_off_, recv_rows_;  // per a2a peer
  std::vector<int32_t> h_counts_;

  // host staging for forward_host: double-buffered so the H2D of step i+1 and the
  // D2H of step i-1 run on the copy engines while step i computes.
  DevBuf x_dev_[2], y_dev_[2];
  cudaStream_t h2d_s_ = nullptr, d2h_s_ = nullptr;
  cudaEvent_t ev_h2d_[2] = {}, ev_comp_[2] = {}, ev_d2h_[2] = {};
  int hslot_ = 0;

  int profiling_ = 0;
  std::vector<std::pair<std::string, cudaEvent_t>> marks_;
  std::vector<cudaEvent_t> event_pool_;
  int launches_ = 0;
};

}  // namespace hep
