// MoE-layer step executor: the B200 realisation of the step the reference only
// simulates (sim::build_schedule, simcore.cpp:96-266):
//   AgTransfer   -> gather_experts(): dense expert All-Gather, or SR wires encoded
//                   on the owner, gathered, decoded on the holder (migration)
//   PreExpert/gate, dispatch -> gate + counting-sort permute + NCCL grouped
//                   send/recv with the A2A peers in build_peer_lists ring order
//   ExpertChunk  -> one grouped GEMM pair over local + received rows
//   A2aCombine   -> NCCL send/recv back + gate-weighted combine
// Peer sets and routing come from the topology table (hybridep::moe::route_table).

#include "layer.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <stdexcept>

#include "hybridep/moe.hpp"
#include "hybridep/simcore.hpp"

namespace hep {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL error in ") + what + ": " + ncclGetErrorString(r));
}

ncclDataType_t nccl_type(DType dt) { return dt == DType::BF16 ? ncclBfloat16 : ncclFloat32; }

// Side (remote dispatch) and All-Gather streams, shared by every layer of one rank on one
// device: an 8-layer stack then needs 2 streams per rank, not 2 per layer, which keeps
// every stream of the step on its own hardware queue (CUDA_DEVICE_MAX_CONNECTIONS <= 32,
// DESIGN.md §7) even with 8 virtual ranks on one device.
struct SharedStreams {
  cudaStream_t side = nullptr, ag = nullptr;
  int refs = 0;
};
std::mutex g_streams_mu;
std::map<std::pair<int, int>, SharedStreams> g_streams;

SharedStreams acquire_streams(int dev, int rank) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  SharedStreams& st = g_streams[{dev, rank}];
  if (st.refs++ == 0) {
    ck(cudaStreamCreateWithFlags(&st.side, cudaStreamNonBlocking), "side stream");
    // HEP_AG_PRIORITY=1: the All-Gather stream gets the highest stream priority, so the
    // migration chain (encode, flags, pulls, decode) is scheduled ahead of the gate and
    // dispatch blocks it otherwise shares the SMs with.
    const char* pr = std::getenv("HEP_AG_PRIORITY");
    int least = 0, greatest = 0;
    ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
    ck(cudaStreamCreateWithPriority(&st.ag, cudaStreamNonBlocking, pr && pr[0] == '1' ? greatest : 0), "ag stream");
  }
  return st;
}

void release_streams(int dev, int rank) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  auto it = g_streams.find({dev, rank});
  if (it == g_streams.end()) return;
  if (--it->second.refs == 0) {
    cudaStreamSynchronize(it->second.side);
    cudaStreamSynchronize(it->second.ag);
    cudaStreamDestroy(it->second.side);
    cudaStreamDestroy(it->second.ag);
    g_streams.erase(it);
  }
}

uint64_t p2p_timeout_ns() {
  // HEP_P2P_TIMEOUT_S: seconds a cross-GPU flag wait may take before it traps with a
  // diagnostic (0 or unset: wait forever, like NCCL -- ranks may skew by minutes).
  const char* e = std::getenv("HEP_P2P_TIMEOUT_S");
  if (!e || !*e) return 0;
  const double sec = std::strtod(e, nullptr);
  return sec > 0 ? static_cast<uint64_t>(sec * 1e9) : 0;
}

}  // namespace

void DevBuf::alloc(size_t n) {
  release();
  if (n == 0) n = 16;
  ck(cudaMalloc(&p, n), "cudaMalloc");
  bytes = n;
}

void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

Layer::Layer(const hep_layer_params& prm, Comm* comm) : comm_(comm) {
  H_ = prm.hidden;
  F_ = prm.ffn;
  E_ = prm.experts;
  k_ = prm.top_k;
  Tmax_ = prm.max_tokens;
  dt_ = prm.dtype == HEP_BF16 ? DType::BF16 : DType::F32;
  rank_ = prm.rank;
  use_sr_ = prm.use_sr != 0;
  if (H_ <= 0 || F_ <= 0 || E_ <= 0 || k_ <= 0 || Tmax_ <= 0)
    throw std::invalid_argument("layer shape must be positive");
  if (k_ > 8 || k_ > E_ || E_ > 64) throw std::invalid_argument("need top_k <= 8, top_k <= experts <= 64");
  if (H_ % 64 || F_ % 64) throw std::invalid_argument("hidden and ffn must be multiples of 64");
  if (!prm.levels || prm.num_levels <= 0) throw std::invalid_argument("layer needs a cluster description");
  for (int i = 0; i < prm.num_levels; ++i) {
    const hep_level& l = prm.levels[i];
    // Bandwidth is a planner input; the executor only needs SF and S_ED.
    cluster_.levels.push_back({l.scaling_factor, l.domain_size, l.bandwidth > 0 ? l.bandwidth : 1.0});
  }
  cluster_.validate();
  G_ = cluster_.total_gpus();
  if (E_ % G_) throw std::invalid_argument("experts must be divisible by the GPU count");
  if (rank_ < 0 || rank_ >= G_) throw std::domain_error("rank out of range");
  if (G_ > 1 && (!comm_ || comm_->nranks != G_ || comm_->rank != rank_))
    throw std::invalid_argument("a communicator of G ranks matching this rank is required when G > 1");
  if (comm_) seq_ = comm_->layers_created++;
  if (cluster_.levels.size() > 16) throw std::invalid_argument("at most 16 levels");
  n_ = E_ / G_;
  NK_ = G_ * E_;
  if (use_sr_) {
    sr_cfg_.ratio_CR = prm.sr.k >= 0 ? std::optional<double>() : std::optional<double>(prm.sr.ratio_CR);
    if (prm.sr.k >= 0) sr_cfg_.k = prm.sr.k;
    sr_cfg_.index_width_bits = prm.sr.index_width_bits;
    sr_cfg_.value_width_bits = prm.sr.value_width_bits;
    sr_cfg_.per_matrix_budget = prm.sr.per_matrix_budget != 0;
  }

  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  ck(cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, dev), "sm count");
  ck(preload_kernels(), "kernel preload");

  // Placement and routing from the topology table.
  const std::vector<int32_t> route = hybridep::moe::route_table(cluster_);
  route_row_.assign(route.begin() + rank_ * G_, route.begin() + (rank_ + 1) * G_);
  held_owners_ = hybridep::moe::held_owners(cluster_)[static_cast<size_t>(rank_)];
  slot_of_expert_.assign(static_cast<size_t>(E_), -1);
  slots_ = 0;
  for (int64_t o : held_owners_)
    for (int64_t i = 0; i < n_; ++i) slot_of_expert_[static_cast<size_t>(o * n_ + i)] = static_cast<int32_t>(slots_++);
  const std::vector<hybridep::sim::PeerLists> peers = hybridep::sim::peer_lists(cluster_);
  for (const auto& l : peers[static_cast<size_t>(rank_)].ag) ag_peers_.insert(ag_peers_.end(), l.begin(), l.end());
  for (const auto& l : peers[static_cast<size_t>(rank_)].a2a) a2a_peers_.insert(a2a_peers_.end(), l.begin(), l.end());

  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  d_route_.alloc(sizeof(int32_t) * G_);
  ck(cudaMemcpy(d_route_.p, route_row_.data(), sizeof(int32_t) * G_, cudaMemcpyHostToDevice), "route");
  d_slot_of_expert_.alloc(sizeof(int32_t) * E_);
  ck(cudaMemcpy(d_slot_of_expert_.p, slot_of_expert_.data(), sizeof(int32_t) * E_, cudaMemcpyHostToDevice), "slots");
  wg_t_.alloc(eb * E_ * H_);
  w_up_c_.alloc(eb * slots_ * F_ * H_);
  w_down_c_.alloc(eb * slots_ * H_ * F_);

  const int64_t TK = Tmax_ * k_;
  const int64_t nchunks = (Tmax_ + 31) / 32;
  topk_idx_.alloc(sizeof(int) * TK);
  topk_w_.alloc(sizeof(float) * TK);
  keys_.alloc(sizeof(int) * TK);
  ranks_.alloc(sizeof(int) * TK);
  pos_.alloc(sizeof(int) * TK);
  chunk_counts_.alloc(sizeof(int) * nchunks * NK_);
  chunk_off_.alloc(sizeof(int) * nchunks * NK_);
  key_total_.alloc(sizeof(int) * NK_);
  key_off_.alloc(sizeof(int) * NK_);
  dest_rows_.alloc(sizeof(int) * G_);
  dest_off_.alloc(sizeof(int) * G_);
  const int64_t max_groups = slots_ * (1 + static_cast<int64_t>(a2a_peers_.size()));
  g_row_start_.alloc(sizeof(int) * max_groups);
  g_rows_.alloc(sizeof(int) * max_groups);
  g_slot_.alloc(sizeof(int) * max_groups);
  all_counts_.alloc(sizeof(int) * G_ * NK_);

  rows_cap_ = TK * (1 + static_cast<int64_t>(a2a_peers_.size()));
  xall_.alloc(eb * rows_cap_ * H_);
  hbuf_.alloc(eb * rows_cap_ * F_);
  oall_.alloc(eb * rows_cap_ * H_);

  if (dt_ == DType::BF16) {
    ck(make_tmap_bf16_2d(&map_a1_, xall_.p, rows_cap_, H_, 128, 64), "tmap a1");
    cta_pair_ = gemm_use_cta_pair();
    // HEP_GATHER_A=1 (one GPU): the permute fused into the up-projection's A load, x rows
    // gathered by the inverse routing map.  Bit-identical, but 2.8x slower on the cfg3 /
    // cfg4 up-projection: one tile's rows span the whole input (profiles/r2_gather.md).
    const char* ga = std::getenv("HEP_GATHER_A");
    gather_a_ = cta_pair_ && G_ == 1 && ga && ga[0] == '1';
    if (gather_a_) {
      row_src_.alloc(sizeof(int32_t) * (rows_cap_ + 256));  // +256: a partial m-tile reads past the last row
      ck(cudaMemset(row_src_.p, 0, sizeof(int32_t) * (rows_cap_ + 256)), "row_src");
    }
    tile_counters_.alloc(2 * sizeof(int));
    const uint32_t b_box = cta_pair_ ? 128 : 256;
    ck(make_tmap_bf16_2d(&map_b1_, w_up_c_.p, slots_ * F_, H_, b_box, 64), "tmap b1");
    ck(make_tmap_bf16_2d(&map_a2_, hbuf_.p, rows_cap_, F_, 128, 64), "tmap a2");
    ck(make_tmap_bf16_2d(&map_b2_, w_down_c_.p, slots_ * H_, F_, b_box, 64), "tmap b2");
  } else {
    const char* f32 = std::getenv("HEP_F32_GEMM");
    tf32_ = !(f32 && std::string(f32) == "simt") && H_ % 32 == 0 && F_ % 32 == 0;
    if (tf32_) {
      const size_t fb = sizeof(float);
      xhi_.alloc(fb * rows_cap_ * H_);
      xlo_.alloc(fb * rows_cap_ * H_);
      hhi_.alloc(fb * rows_cap_ * F_);
      hlo_.alloc(fb * rows_cap_ * F_);
      ck(make_tmap_f32_2d(&t_xhi_, xhi_.p, rows_cap_, H_, 128, kTf32BK), "tmap xhi");
      ck(make_tmap_f32_2d(&t_xlo_, xlo_.p, rows_cap_, H_, 128, kTf32BK), "tmap xlo");
      ck(make_tmap_f32_2d(&t_hhi_, hhi_.p, rows_cap_, F_, 128, kTf32BK), "tmap hhi");
      ck(make_tmap_f32_2d(&t_hlo_, hlo_.p, rows_cap_, F_, 128, kTf32BK), "tmap hlo");
      // Pre-split hi/lo weight copies (split once per weight change).  HEP_TF32_RAWB=1
      // streams the raw fp32 weights instead and splits them in shared memory: half the
      // DRAM reads, same time (profiles/r2_tf32_tiled.md).
      const char* raw = std::getenv("HEP_TF32_RAWB");
      tf32_presplit_ = !(raw && raw[0] == '1');
      if (tf32_presplit_) {
        wuhi_.alloc(fb * slots_ * F_ * H_);
        wulo_.alloc(fb * slots_ * F_ * H_);
        wdhi_.alloc(fb * slots_ * H_ * F_);
        wdlo_.alloc(fb * slots_ * H_ * F_);
        ck(make_tmap_f32_2d(&t_wuhi_, wuhi_.p, slots_ * F_, H_, 256, kTf32BK), "tmap wuhi");
        ck(make_tmap_f32_2d(&t_wulo_, wulo_.p, slots_ * F_, H_, 256, kTf32BK), "tmap wulo");
        ck(make_tmap_f32_2d(&t_wdhi_, wdhi_.p, slots_ * H_, F_, 256, kTf32BK), "tmap wdhi");
        ck(make_tmap_f32_2d(&t_wdlo_, wdlo_.p, slots_ * H_, F_, 256, kTf32BK), "tmap wdlo");
      } else {
        ck(make_tmap_f32_2d(&t_wuhi_, w_up_c_.p, slots_ * F_, H_, 256, kTf32BK), "tmap w_up");
        ck(make_tmap_f32_2d(&t_wdhi_, w_down_c_.p, slots_ * H_, F_, 256, kTf32BK), "tmap w_down");
      }
      // split-K when (groups x m-tiles x n-tiles) of an even routing leaves SMs idle
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t groups = slots_ * (1 + static_cast<int64_t>(a2a_peers_.size()));
      const int64_t m_tiles = std::max<int64_t>(1, (Tmax_ * k_ / E_ + 127) / 128);
      auto pick = [&](int64_t N, int64_t K) {
        const int64_t tiles = groups * m_tiles * ((N + 255) / 256);
        int ks = 1;
        while (ks < 8 && tiles * ks * 2 <= sms && K % (32 * ks * 2) == 0) ks *= 2;
        return ks;
      };
      ksplit_up_ = pick(F_, H_);
      ksplit_down_ = pick(H_, F_);
      if (const char* env = std::getenv("HEP_TF32_KSPLIT")) {  // "up,down" override (sweeps)
        int u = 0, d = 0;
        if (std::sscanf(env, "%d,%d", &u, &d) == 2 && u >= 1 && d >= 1 && H_ % (kTf32BK * u) == 0 &&
            F_ % (kTf32BK * d) == 0) {
          ksplit_up_ = u;
          ksplit_down_ = d;
        }
      }
      const int ks = std::max(ksplit_up_, ksplit_down_);
      if (ks > 1) kpart_.alloc(sizeof(float) * ks * rows_cap_ * std::max(F_, H_));
    }
  }
  slot_dirty_.assign(static_cast<size_t>(slots_), 1);

  if (use_sr_) {
    const int64_t P = 2 * H_ * F_;
    shared_.alloc(sizeof(float) * P);
    master_.alloc(sizeof(float) * n_ * P);
    size_t wb = 0;
    hep_sr_config c{sr_cfg_.ratio_CR.value_or(1.0), sr_cfg_.k.value_or(-1), sr_cfg_.index_width_bits,
                    sr_cfg_.value_width_bits, sr_cfg_.per_matrix_budget ? 1 : 0};
    if (hep_sr_wire_bytes(H_, F_, &c, &wb) != HEP_OK) throw std::invalid_argument(hep_last_error());
    wires_.alloc(((wb + 15) / 16 * 16) * slots_);
    sr_ws_.alloc(sr_workspace_bytes(H_, F_, static_cast<int>(n_)));
    sr_tmp_.alloc(sizeof(float) * P);
    sr_status_.alloc(16 * std::max<int64_t>(kMaxSrBatch, slots_));  // fused decode: one status per slot
    shared_c_.alloc(static_cast<size_t>(dtype_bytes(dt_)) * P);
    if (G_ > 1) partial_.alloc(sizeof(double) * P);  // shared-expert refresh chain
  }
  if (use_sr_) {
    ck(cudaHostAlloc(reinterpret_cast<void**>(&mig_err_host_), sizeof(int32_t), cudaHostAllocMapped), "mapped flag");
    *mig_err_host_ = 0;
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mig_err_dev_), mig_err_host_, 0), "mapped flag");
  }
  send_off_.resize(a2a_peers_.size());
  send_rows_.resize(a2a_peers_.size());
  recv_off_.resize(a2a_peers_.size());
  recv_rows_.resize(a2a_peers_.size());
  num_groups_ = static_cast<int>(slots_);
  if (G_ > 1) {
    const char* mode = std::getenv("HEP_COMM");
    p2p_ = !(mode && std::string(mode) == "nccl");
    if (comm_->vgroup && !p2p_)
      throw std::invalid_argument("virtual ranks share one device: only the peer-memory path applies (unset HEP_COMM)");
    timeout_ns_ = p2p_timeout_ns();
    if (p2p_) {
      setup_p2p();
      // HEP_SR_FUSED=1: decode fused into the expert GEMM's B-operand load.  Bit-identical
      // to the dense decode, but its converter sits in the TMA -> MMA pipeline and the
      // gathered-expert GEMMs run at ~0.65 of the dense path's rate (cfg4 N=2:
      // profiles/r2_cfg4_fused.md), so the dense decode (a pass on the All-Gather stream,
      // hidden under the own-expert GEMMs) stays the default.
      const char* fused = std::getenv("HEP_SR_FUSED");
      sr_fused_ = use_sr_ && dt_ == DType::BF16 && fused && fused[0] == '1' && H_ < 65536 && F_ < 65536;
      if (sr_fused_) {
        size_t wb = 0;
        hep_sr_config c{sr_cfg_.ratio_CR.value_or(1.0), sr_cfg_.k.value_or(-1), sr_cfg_.index_width_bits,
                        sr_cfg_.value_width_bits, sr_cfg_.per_matrix_budget ? 1 : 0};
        if (hep_sr_wire_bytes(H_, F_, &c, &wb) != HEP_OK) throw std::invalid_argument(hep_last_error());
        patch_kmax_ = std::max<size_t>(1, (wb - 28) / 8);
        patch_slot_bytes_ = static_cast<size_t>(patch_blocks(F_, H_) + patch_blocks(H_, F_)) * kPatchBlockBytes;
        patch_blocks_.alloc(patch_slot_bytes_ * slots_);
        patch_ovf_.alloc(sizeof(uint2) * patch_kmax_ * slots_);
        patch_ovf_n_.alloc(sizeof(int) * slots_);
        std::vector<PatchRef> refs(static_cast<size_t>(slots_));
        for (int64_t sl = 0; sl < slots_; ++sl) {
          const uint8_t* base = patch_blocks_.as<uint8_t>() + sl * patch_slot_bytes_;
          refs[static_cast<size_t>(sl)] =
              PatchRef{{base, base + static_cast<size_t>(patch_blocks(F_, H_)) * kPatchBlockBytes},
                       patch_ovf_.as<uint2>() + sl * patch_kmax_, patch_ovf_n_.as<int>() + sl,
                       sr_status_.as<int32_t>() + 4 * sl};
        }
        patch_refs_.alloc(sizeof(PatchRef) * slots_);
        ck(cudaMemcpy(patch_refs_.p, refs.data(), sizeof(PatchRef) * slots_, cudaMemcpyHostToDevice), "patch refs");
        const uint32_t box = cta_pair_ ? 128 : 256;
        ck(make_tmap_bf16_2d(&map_shared_up_, shared_c_.p, F_, H_, box, 64), "tmap shared up");
        ck(make_tmap_bf16_2d(&map_shared_down_, shared_c_.as<uint8_t>() + 2 * H_ * F_, H_, F_, box, 64),
           "tmap shared down");
      }
    } else {
      // NCCL baseline: agree on the layer shape before any row is received
      const LayerSig mine = signature();
      DevBuf d_mine, d_all;
      d_mine.alloc(sizeof(LayerSig));
      d_all.alloc(sizeof(LayerSig) * G_);
      ck(cudaMemcpy(d_mine.p, &mine, sizeof(LayerSig), cudaMemcpyHostToDevice), "sig h2d");
      nck(ncclAllGather(d_mine.p, d_all.p, sizeof(LayerSig), ncclUint8, comm_->nccl, 0), "sig allgather");
      ck(cudaStreamSynchronize(0), "sig sync");
      std::vector<LayerSig> all(static_cast<size_t>(G_));
      ck(cudaMemcpy(all.data(), d_all.p, sizeof(LayerSig) * G_, cudaMemcpyDeviceToHost), "sig d2h");
      check_signatures(all);
    }
  }
  if (G_ == 1) {
    const char* g = std::getenv("HEP_GRAPH");  // 0: enqueue every kernel on every forward
    use_graphs_ = !(g && g[0] == '0');
  }
  const int rows_per_expert = static_cast<int>(Tmax_ * k_ / E_);
  sched_up_ = gemm_schedule(rows_per_expert, static_cast<int>(F_), static_cast<int>(H_), true);
  sched_down_ = gemm_schedule(rows_per_expert, static_cast<int>(H_), static_cast<int>(F_), false);
}

LayerSig Layer::signature() const {
  LayerSig g;
  std::memset(&g, 0, sizeof(g));
  g.H = H_;
  g.F = F_;
  g.E = E_;
  g.k = k_;
  g.Tmax = Tmax_;
  g.dtype = static_cast<int32_t>(dt_);
  g.use_sr = use_sr_ ? 1 : 0;
  if (use_sr_) {
    g.sr_k = sr_cfg_.k.value_or(-1);
    g.sr_ratio = sr_cfg_.ratio_CR.value_or(0.0);
    g.per_matrix = sr_cfg_.per_matrix_budget ? 1 : 0;
    g.iw = sr_cfg_.index_width_bits;
    g.vw = sr_cfg_.value_width_bits;
  }
  g.nlev = static_cast<int32_t>(cluster_.levels.size());
  for (size_t i = 0; i < cluster_.levels.size(); ++i) {
    g.sf[i] = cluster_.levels[i].scaling_factor;
    g.sed[i] = cluster_.levels[i].domain_size;
  }
  g.p2p = p2p_ ? 1 : 0;
  return g;
}

void Layer::check_signatures(const std::vector<LayerSig>& all) const {
  const LayerSig mine = signature();
  for (size_t r = 0; r < all.size(); ++r)
    if (std::memcmp(&all[r], &mine, sizeof(LayerSig)) != 0)
      throw std::invalid_argument("rank " + std::to_string(r) + " created this layer with a different shape, " +
                                  "max_tokens, dtype, SR configuration, cluster or comm path than rank " +
                                  std::to_string(rank_));
}

PeerBufs Layer::my_bufs() const {
  return PeerBufs{xall_.p,  oall_.p,    sync_.p,        w_up_c_.p, w_down_c_.p,
                  wires_.p, partial_.p, chain_flags_.p, shared_.p};
}

void Layer::setup_streams() {
  int dev = 0;
  ck(cudaGetDevice(&dev), "device");
  const SharedStreams st = acquire_streams(dev, rank_);
  side_s_ = st.side;
  ag_s_ = st.ag;
  // Every stream a rank's step uses needs its own hardware queue: the
  // caller's stream plus the shared side and All-Gather streams, per rank of this process.
  const int ranks_here = comm_->vgroup ? static_cast<int>(G_) : 1;
  const int need = 3 * ranks_here + 1;
  const char* env = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
  const int have = env ? std::atoi(env) : 8;
  static bool warned = false;
  if (have < need && !warned) {
    warned = true;
    std::fprintf(stderr,
                 "hep: CUDA_DEVICE_MAX_CONNECTIONS=%s but the peer-memory step needs >= %d hardware queues; set it "
                 "(<= 32) before the CUDA context is created, or aliased queues may serialise a spin-wait ahead of "
                 "the work it waits for\n",
                 env ? env : "unset (8)", need);
  }
}

void Layer::setup_p2p() {
  if (G_ > kMaxG || E_ > kMaxE) throw std::invalid_argument("peer-memory path supports G <= 8, E <= 64");
  sync_.alloc(p2p_sync_bytes(static_cast<int>(G_), static_cast<int>(E_)));
  ck(cudaMemset(sync_.p, 0, sync_.bytes), "sync memset");
  send_base_.alloc(sizeof(int) * NK_);
  if (use_sr_) {
    // the shared-expert refresh chain: chunk flags (+ barrier flags)
    const int64_t P = 2 * H_ * F_;
    chain_flags_.alloc(sizeof(uint32_t) * ((P + kChainChunk - 1) / kChainChunk + kMaxG));
    ck(cudaMemset(chain_flags_.p, 0, chain_flags_.bytes), "chain flags");
  }
  g_out_down_.alloc(sizeof(unsigned long long) * slots_ * (1 + static_cast<int64_t>(a2a_peers_.size())));
  g_wait_.alloc(sizeof(int) * slots_ * (1 + static_cast<int64_t>(a2a_peers_.size())));
  setup_streams();
  ck(cudaEventCreateWithFlags(&ev_counts_, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ev_remote_, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ev_arrived_, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ev_ag_start_, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ev_ag_done_, cudaEventDisableTiming), "event");
  {
    const char* spin = std::getenv("HEP_GEMM_SPIN");  // 1: GEMM producers wait on dispatch flags (old)
    spin_ = spin && spin[0] == '1';
    const char* merge = std::getenv("HEP_MERGE_GEMMS");
    merge_mode_ = merge ? std::atoi(merge) : 0;
    merge_gemms_ = merge_mode_ == 1 && !sr_fused_;
  }
  if (comm_->vgroup) {
    // Virtual ranks: register; peers resolve on first use, once every rank's layer exists.
    std::lock_guard<std::mutex> lk(comm_->vgroup->mu);
    auto& slot = comm_->vgroup->layers[{seq_, rank_}];
    if (slot) throw std::invalid_argument("virtual rank already has a layer with this sequence number");
    slot = this;
    connected_ = false;
    return;
  }
  // Processes: exchange the layer signature and CUDA IPC handles of xall / oall / sync
  // (token path), the expert compute copies and SR wires (All-Gather pulls) and the
  // shared-expert chain buffers through NCCL.
  constexpr int kBufs = 9;
  struct Hello {
    LayerSig sig;
    cudaIpcMemHandle_t h[kBufs];
  } mine;
  std::memset(&mine, 0, sizeof(mine));
  mine.sig = signature();
  const PeerBufs b = my_bufs();
  void* const ptrs[kBufs] = {b.xall, b.oall, b.sync, b.w_up, b.w_down, b.wires, b.partial, b.chain_flags, b.shared};
  const int nb = use_sr_ ? kBufs : 5;
  for (int i = 0; i < nb; ++i) ck(cudaIpcGetMemHandle(&mine.h[i], ptrs[i]), "ipc handle");
  DevBuf dmine, dall;
  dmine.alloc(sizeof(Hello));
  dall.alloc(sizeof(Hello) * G_);
  ck(cudaMemcpy(dmine.p, &mine, sizeof(Hello), cudaMemcpyHostToDevice), "ipc h2d");
  nck(ncclAllGather(dmine.p, dall.p, sizeof(Hello), ncclUint8, comm_->nccl, 0), "ipc allgather");
  ck(cudaStreamSynchronize(0), "ipc sync");
  std::vector<Hello> all(static_cast<size_t>(G_));
  ck(cudaMemcpy(all.data(), dall.p, sizeof(Hello) * G_, cudaMemcpyDeviceToHost), "ipc d2h");
  std::vector<LayerSig> sigs;
  for (const Hello& h : all) sigs.push_back(h.sig);
  check_signatures(sigs);
  std::vector<PeerBufs> bufs(static_cast<size_t>(G_));
  for (int r = 0; r < G_; ++r) {
    if (r == rank_) {
      bufs[static_cast<size_t>(r)] = b;
      continue;
    }
    void* p[kBufs] = {};
    for (int i = 0; i < nb; ++i) {
      ck(cudaIpcOpenMemHandle(&p[i], all[static_cast<size_t>(r)].h[i], cudaIpcMemLazyEnablePeerAccess), "ipc open");
      ipc_opened_.push_back(p[i]);
    }
    bufs[static_cast<size_t>(r)] = PeerBufs{p[0], p[1], p[2], p[3], p[4], p[5], p[6], p[7], p[8]};
  }
  connect(bufs);
}

void Layer::ensure_connected() {
  if (connected_) return;
  VirtualGroup& vg = *comm_->vgroup;
  std::vector<PeerBufs> bufs(static_cast<size_t>(G_));
  std::vector<LayerSig> sigs(static_cast<size_t>(G_));
  {
    std::lock_guard<std::mutex> lk(vg.mu);
    for (int r = 0; r < G_; ++r) {
      auto it = vg.layers.find({seq_, r});
      if (it == vg.layers.end())
        throw std::runtime_error("virtual rank " + std::to_string(r) + " has not created layer #" +
                                 std::to_string(seq_) + " yet (create every rank's layer before the first step)");
      bufs[static_cast<size_t>(r)] = it->second->my_bufs();
      sigs[static_cast<size_t>(r)] = it->second->signature();
    }
  }
  check_signatures(sigs);
  connect(bufs);
  connected_ = true;
}

void Layer::connect(const std::vector<PeerBufs>& bufs) {
  P2PArgs& a = p2p_args_;
  a.G = static_cast<int>(G_);
  a.E = static_cast<int>(E_);
  a.rank = rank_;
  a.recv_start = static_cast<int>(Tmax_ * k_);  // equal on every rank: signatures matched
  a.row_bytes = static_cast<int>(H_ * dtype_bytes(dt_));
  a.timeout_ns = timeout_ns_;
  peer_w_up_.assign(static_cast<size_t>(G_), nullptr);
  peer_w_down_.assign(static_cast<size_t>(G_), nullptr);
  peer_wires_.assign(static_cast<size_t>(G_), nullptr);
  peer_chain_flags_.assign(static_cast<size_t>(G_), nullptr);
  for (int r = 0; r < G_; ++r) {
    const PeerBufs& b = bufs[static_cast<size_t>(r)];
    a.xall[r] = b.xall;
    a.oall[r] = b.oall;
    a.sync[r] = b.sync;
    if (r == rank_) continue;
    peer_w_up_[static_cast<size_t>(r)] = b.w_up;
    peer_w_down_[static_cast<size_t>(r)] = b.w_down;
    peer_wires_[static_cast<size_t>(r)] = b.wires;
  }
  if (use_sr_) {
    for (int r = 0; r < G_; ++r)
      peer_chain_flags_[static_cast<size_t>(r)] = static_cast<uint32_t*>(bufs[static_cast<size_t>(r)].chain_flags);
    if (rank_ > 0) {
      peer_partial_prev_ = static_cast<const double*>(bufs[static_cast<size_t>(rank_ - 1)].partial);
      peer_flags_prev_ = static_cast<const uint32_t*>(bufs[static_cast<size_t>(rank_ - 1)].chain_flags);
    }
    peer_shared_last_ = static_cast<const float*>(bufs[static_cast<size_t>(G_ - 1)].shared);
    peer_flags_last_ = static_cast<const uint32_t*>(bufs[static_cast<size_t>(G_ - 1)].chain_flags);
  }
  a.n_ag = 0;
  for (int64_t p : ag_peers_) a.ag_list[a.n_ag++] = static_cast<int>(p);
  const std::vector<hybridep::sim::PeerLists> peers = hybridep::sim::peer_lists(cluster_);
  for (int d = 0; d < G_; ++d) {
    int n = 0;
    for (const auto& level : peers[static_cast<size_t>(d)].a2a)
      for (int64_t p : level) a.src_list[d * kMaxG + n++] = static_cast<int>(p);
    a.n_src[d] = n;
  }
}

Layer::~Layer() {
  if (p2p_ && connected_ && ag_epoch_ > 0 && !ag_peers_.empty() && side_s_) {
    // Peers pull this rank's owned experts (or wires) on their All-Gather streams: wait
    // until every AG peer has signalled that it finished the last epoch's pulls before
    // the memory is freed.
    P2PArgs prev = p2p_args_;
    prev.epoch = ag_epoch_;
    if (launch_signal_wait(prev, 4, side_s_, true, true, false) == cudaSuccess) cudaStreamSynchronize(side_s_);
  }
  if (side_s_) cudaStreamSynchronize(side_s_);
  if (ag_s_) cudaStreamSynchronize(ag_s_);
  if (comm_ && comm_->vgroup) {
    std::lock_guard<std::mutex> lk(comm_->vgroup->mu);
    auto it = comm_->vgroup->layers.find({seq_, rank_});
    if (it != comm_->vgroup->layers.end() && it->second == this) comm_->vgroup->layers.erase(it);
  }
  if (side_s_) {
    int dev = 0;
    cudaGetDevice(&dev);
    release_streams(dev, rank_);
  }
  if (ev_ag_start_) cudaEventDestroy(ev_ag_start_);
  if (ev_ag_done_) cudaEventDestroy(ev_ag_done_);
  if (ev_counts_) cudaEventDestroy(ev_counts_);
  if (ev_remote_) cudaEventDestroy(ev_remote_);
  if (ev_arrived_) cudaEventDestroy(ev_arrived_);
  for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
  if (h2d_s_) cudaStreamSynchronize(h2d_s_);
  if (d2h_s_) cudaStreamSynchronize(d2h_s_);
  for (cudaEvent_t e : event_pool_) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) {
    if (ev_h2d_[b]) cudaEventDestroy(ev_h2d_[b]);
    if (ev_comp_[b]) cudaEventDestroy(ev_comp_[b]);
    if (ev_d2h_[b]) cudaEventDestroy(ev_d2h_[b]);
  }
  if (h2d_s_) cudaStreamDestroy(h2d_s_);
  if (d2h_s_) cudaStreamDestroy(d2h_s_);
  if (mig_err_host_) cudaFreeHost(mig_err_host_);
  drop_graphs();
  if (graph_s_) {
    cudaStreamSynchronize(graph_s_);
    cudaStreamDestroy(graph_s_);
  }
  if (ev_graph_in_) cudaEventDestroy(ev_graph_in_);
  if (ev_graph_out_) cudaEventDestroy(ev_graph_out_);
}

void Layer::drop_graphs() {
  for (GraphEntry& e : graphs_) cudaGraphExecDestroy(e.exec);
  graphs_.clear();
}

bool Layer::forward_graph(const void* x, int64_t T, void* y, cudaStream_t s, bool residual) {
  if (!use_graphs_ || profiling_ || T == 0) return false;
  if (!graph_s_) {
    ck(cudaStreamCreateWithFlags(&graph_s_, cudaStreamNonBlocking), "graph stream");
    ck(cudaEventCreateWithFlags(&ev_graph_in_, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_graph_out_, cudaEventDisableTiming), "event");
  }
  if (tf32_) split_dirty_slots(s);  // weight splits stay outside the replayed graph
  ck(cudaEventRecord(ev_graph_in_, s), "record");
  ck(cudaStreamWaitEvent(graph_s_, ev_graph_in_, 0), "wait");
  GraphEntry* hit = nullptr;
  for (GraphEntry& e : graphs_)
    if (e.x == x && e.T == T && e.y == y && e.residual == residual) hit = &e;
  if (!hit) {
    if (graphs_.size() >= 4) {  // keep a few (x, T, y) shapes
      cudaGraphExecDestroy(graphs_.front().exec);
      graphs_.erase(graphs_.begin());
    }
    cudaGraph_t g = nullptr;
    ck(cudaStreamBeginCapture(graph_s_, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
      step(x, T, y, graph_s_, residual);
    } catch (...) {
      cudaStreamEndCapture(graph_s_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    ck(cudaStreamEndCapture(graph_s_, &g), "end capture");
    cudaGraphExec_t exec = nullptr;
    const cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    ck(e, "graph instantiate");
    graphs_.push_back(GraphEntry{x, T, y, residual, exec, launches_});
    hit = &graphs_.back();
  }
  ck(cudaGraphLaunch(hit->exec, graph_s_), "graph launch");
  launches_ = hit->launches;
  ck(cudaEventRecord(ev_graph_out_, graph_s_), "record");
  ck(cudaStreamWaitEvent(s, ev_graph_out_, 0), "wait");
  return true;
}

void Layer::init_host_staging() {
  if (h2d_s_) return;
  // forward_host's staging buffers and copy streams, created on first use (an 8-layer
  // stack driven through device buffers never pays for them)
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  for (int b = 0; b < 2; ++b) {
    x_dev_[b].alloc(eb * Tmax_ * H_);
    y_dev_[b].alloc(eb * Tmax_ * H_);
    ck(cudaEventCreateWithFlags(&ev_h2d_[b], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_comp_[b], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_d2h_[b], cudaEventDisableTiming), "event");
  }
  ck(cudaStreamCreateWithFlags(&h2d_s_, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&d2h_s_, cudaStreamNonBlocking), "stream");
}

void Layer::set_gate(const void* w_gate, DType dt, cudaStream_t s) {
  drop_graphs();
  // W_g is H x E; the gate kernel wants it expert-major in the layer dtype.
  ck(launch_transpose_convert(dt, w_gate, H_, E_, dt_, wg_t_.p, s), "gate layout");
}

void Layer::set_expert(int64_t e, const void* w_up, const void* w_down, DType dt, cudaStream_t s) {
  drop_graphs();
  if (e < 0 || e >= E_) throw std::domain_error("expert id out of range");
  if (e / n_ != rank_) throw std::invalid_argument("expert is not owned by this rank");
  if (ag_pending_) ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");  // the encode reads the masters
  if (p2p_ && !use_sr_ && ag_epoch_ > 0 && !ag_peers_.empty()) {
    // AG peers pull the owned compute copies on their own streams: rewrite them only once
    // every peer has signalled that it finished the previous epoch's pulls (slot 4)
    P2PArgs prev = p2p_args_;
    prev.epoch = ag_epoch_;
    ck(launch_signal_wait(prev, 4, s, true, true, false), "ag pulled");
  }
  const int64_t slot = slot_of_expert_[static_cast<size_t>(e)];
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  uint8_t* up = w_up_c_.as<uint8_t>() + eb * slot * F_ * H_;
  uint8_t* down = w_down_c_.as<uint8_t>() + eb * slot * H_ * F_;
  ck(launch_transpose_convert(dt, w_up, H_, F_, dt_, up, s), "w_up layout");
  ck(launch_transpose_convert(dt, w_down, F_, H_, dt_, down, s), "w_down layout");
  slot_dirty_[static_cast<size_t>(slot)] = 1;
  if (use_sr_) {
    // fp32 master copy in the reference flat layout (w_up then w_down) for encode.
    const int64_t P = 2 * H_ * F_;
    float* m = master_.as<float>() + (e - rank_ * n_) * P;
    if (dt == DType::F32) {
      ck(cudaMemcpyAsync(m, w_up, sizeof(float) * H_ * F_, cudaMemcpyDeviceToDevice, s), "master up");
      ck(cudaMemcpyAsync(m + H_ * F_, w_down, sizeof(float) * H_ * F_, cudaMemcpyDeviceToDevice, s), "master down");
    } else {
      // bf16 -> fp32 is exact: two transposes reproduce the row-major layout.
      ck(launch_transpose_convert(DType::BF16, w_up, H_, F_, DType::F32, sr_tmp_.p, s), "up32");
      ck(launch_transpose_convert(DType::F32, sr_tmp_.p, F_, H_, DType::F32, m, s), "up32b");
      ck(launch_transpose_convert(DType::BF16, w_down, F_, H_, DType::F32, sr_tmp_.p, s), "down32");
      ck(launch_transpose_convert(DType::F32, sr_tmp_.p, H_, F_, DType::F32, m + H_ * F_, s), "down32b");
    }
  }
}

void Layer::set_shared(const float* shared, cudaStream_t s) {
  if (!use_sr_) throw std::invalid_argument("shared expert is only used with SR migration");
  ck(cudaMemcpyAsync(shared_.p, shared, sizeof(float) * 2 * H_ * F_, cudaMemcpyDeviceToDevice, s), "shared");
  finish_shared(s);
}

void Layer::get_shared(float* out, cudaStream_t s) const {
  if (!use_sr_) throw std::invalid_argument("shared expert is only used with SR migration");
  ck(cudaMemcpyAsync(out, shared_.p, sizeof(float) * 2 * H_ * F_, cudaMemcpyDeviceToDevice, s), "get shared");
}

void Layer::refresh_shared(cudaStream_t s) {
  if (!use_sr_) throw std::invalid_argument("shared expert is only used with SR migration");
  if (p2p_) ensure_connected();
  const int64_t P = 2 * H_ * F_;
  if (G_ == 1) {  // every expert is local: the plain kernel over the list
    std::vector<const void*> ex(static_cast<size_t>(n_));
    for (int64_t j = 0; j < n_; ++j) ex[static_cast<size_t>(j)] = master_.as<float>() + j * P;
    ck(launch_shared_mean(DType::F32, ex.data(), static_cast<int>(n_), P, shared_.as<float>(), s), "shared mean");
    finish_shared(s);
    return;
  }
  ChainArgs c{};
  c.master = master_.as<float>();
  c.partial = partial_.as<double>();
  c.shared = shared_.as<float>();
  c.P = P;
  c.chunk = kChainChunk;
  c.n = static_cast<int>(n_);
  c.rank = rank_;
  c.G = static_cast<int>(G_);
  c.inv = 1.0 / static_cast<double>(E_);
  if (p2p_) {
    // peer-memory chain: chunks pipeline from rank 0 to rank G-1, then every rank
    // copies the mean from the last one
    c.pred_partial = peer_partial_prev_;
    c.pred_flags = peer_flags_prev_;
    c.my_flags = chain_flags_.as<uint32_t>();
    c.last_shared = peer_shared_last_;
    c.last_flags = peer_flags_last_;
    const int64_t nchunks = (P + kChainChunk - 1) / kChainChunk;
    for (int r = 0; r < G_; ++r) c.bar[r] = peer_chain_flags_[static_cast<size_t>(r)] + nchunks;
    c.epoch = ++chain_epoch_;
    c.timeout_ns = timeout_ns_;
    ck(launch_shared_chain(c, s), "shared chain");
  } else {
    // NCCL: the same chain with whole-vector hops, then a broadcast from the last rank
    nck(ncclGroupStart(), "group");
    if (rank_ > 0) nck(ncclRecv(partial_.p, static_cast<size_t>(P), ncclFloat64, rank_ - 1, comm_->nccl, s), "recv");
    nck(ncclGroupEnd(), "group");
    c.pred_partial = partial_.as<double>();
    c.epoch = 0;  // no flags
    ck(launch_shared_chain(c, s), "shared chain");
    if (rank_ < G_ - 1) nck(ncclSend(partial_.p, static_cast<size_t>(P), ncclFloat64, rank_ + 1, comm_->nccl, s), "send");
    nck(ncclBroadcast(shared_.p, shared_.p, static_cast<size_t>(P), ncclFloat32, static_cast<int>(G_ - 1), comm_->nccl, s),
        "broadcast");
  }
  finish_shared(s);
}

void Layer::finish_shared(cudaStream_t s) {
  // the shared expert in the GEMM's layout, the base every migrated expert is decoded onto
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  ck(launch_transpose_convert(DType::F32, shared_.p, H_, F_, dt_, shared_c_.p, s), "shared up");
  ck(launch_transpose_convert(DType::F32, shared_.as<float>() + H_ * F_, F_, H_, dt_,
                              shared_c_.as<uint8_t>() + eb * H_ * F_, s), "shared down");
}

void Layer::mark_gathered_dirty() {
  for (int64_t p : ag_peers_)
    for (int64_t i = 0; i < n_; ++i)
      slot_dirty_[static_cast<size_t>(slot_of_expert_[static_cast<size_t>(p * n_ + i)])] = 1;
}

void Layer::split_dirty_slots(cudaStream_t s) {
  if (!tf32_presplit_) return;  // the GEMM splits raw weights in shared memory
  const int64_t per = F_ * H_;
  for (int64_t a = 0; a < slots_;) {
    if (!slot_dirty_[static_cast<size_t>(a)]) { ++a; continue; }
    int64_t b = a;
    while (b < slots_ && slot_dirty_[static_cast<size_t>(b)]) slot_dirty_[static_cast<size_t>(b++)] = 0;
    ck(launch_split_tf32(w_up_c_.as<float>() + a * per, wuhi_.as<float>() + a * per, wulo_.as<float>() + a * per,
                         (b - a) * per, s), "split w_up");
    ck(launch_split_tf32(w_down_c_.as<float>() + a * per, wdhi_.as<float>() + a * per,
                         wdlo_.as<float>() + a * per, (b - a) * per, s), "split w_down");
    launches_ += 2;
    a = b;
  }
}

void Layer::gather_experts(cudaStream_t s) {
  if (G_ == 1 || ag_peers_.empty()) return;
  if (p2p_) ensure_connected();
  gather(s);
  check_migration(false);  // after the collective is enqueued (see forward)
}

void Layer::gather(cudaStream_t s) {
  mark_gathered_dirty();  // the gathered slots' compute copies are rewritten below
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  const size_t per_slot_up = static_cast<size_t>(F_ * H_), per_slot_down = static_cast<size_t>(H_ * F_);
  auto first_slot_of = [&](int64_t owner) { return slot_of_expert_[static_cast<size_t>(owner * n_)]; };
  if (p2p_) {
    // "AgTransfer eligible from t=0" (simcore.cpp:155-156): the All-Gather runs on its own
    // stream with the copy engines pulling peers' experts over NVLink, while the step
    // starts; forward() waits for it only before the GEMMs of gathered experts.
    ck(cudaEventRecord(ev_ag_start_, s), "record");
    ck(cudaStreamWaitEvent(ag_s_, ev_ag_start_, 0), "wait");
    P2PArgs ag = p2p_args_;
    ag.epoch = ++ag_epoch_;
    const int64_t P = 2 * H_ * F_;
    size_t wb = 0, stride = 0;
    hep_sr_config c{sr_cfg_.ratio_CR.value_or(1.0), sr_cfg_.k.value_or(-1), sr_cfg_.index_width_bits,
                    sr_cfg_.value_width_bits, sr_cfg_.per_matrix_budget ? 1 : 0};
    if (use_sr_) {
      if (hep_sr_wire_bytes(H_, F_, &c, &wb) != HEP_OK) throw std::invalid_argument(hep_last_error());
      stride = (wb + 15) / 16 * 16;
      if (ag.epoch > 1 && !wires_fresh_) {  // every AG peer has pulled last epoch's wires before they are rewritten
        P2PArgs prev = ag;
        prev.epoch = ag.epoch - 1;
        ck(launch_signal_wait(prev, 4, ag_s_, true, true, false), "wires pulled");
      }
      std::vector<const void*> ex;
      std::vector<void*> wo;
      for (int64_t i = 0; i < n_; ++i) {
        ex.push_back(master_.as<float>() + i * P);
        wo.push_back(wires_.as<uint8_t>() + stride * (first_slot_of(rank_) + i));
      }
      if (!wires_fresh_ &&
          hep_sr_encode_batch(ex.data(), static_cast<int>(n_), HEP_F32, shared_.as<float>(), H_, F_, &c, wo.data(),
                              wb, sr_ws_.p, sr_ws_.bytes, ag_s_) != HEP_OK)
        throw std::runtime_error(hep_last_error());
      wires_fresh_ = false;
    }
    // Every AG peer's experts (or wires) for this epoch are final -> pull.
    ck(launch_signal_wait(ag, 3, ag_s_, true, true), "ag flags");
    for (int64_t p : ag_peers_) {
      const size_t pi = static_cast<size_t>(p);
      const int64_t theirs = first_slot_of(p);
      if (use_sr_) {
        // the owner's wires sit in its own first n slots
        ck(cudaMemcpyAsync(wires_.as<uint8_t>() + stride * theirs, peer_wires_[pi], stride * n_,
                           cudaMemcpyDeviceToDevice, ag_s_), "pull wires");
      } else {
        ck(cudaMemcpyAsync(w_up_c_.as<uint8_t>() + eb * theirs * per_slot_up, peer_w_up_[pi],
                           eb * n_ * per_slot_up, cudaMemcpyDeviceToDevice, ag_s_), "pull up");
        ck(cudaMemcpyAsync(w_down_c_.as<uint8_t>() + eb * theirs * per_slot_down, peer_w_down_[pi],
                           eb * n_ * per_slot_down, cudaMemcpyDeviceToDevice, ag_s_), "pull down");
      }
    }
    // "I have pulled your experts / wires of this epoch": owners may rewrite them now
    ck(launch_signal_wait(ag, 4, ag_s_, false, true, true), "pulled");
    if (use_sr_) {
      if (sr_fused_) index_gathered(wb, stride, ag_s_);
      else decode_gathered(wb, stride, ag_s_);
    }
    ck(cudaEventRecord(ev_ag_done_, ag_s_), "record");
    ag_pending_ = true;
    return;
  }
  if (!use_sr_) {
    nck(ncclGroupStart(), "group start");
    for (int64_t p : ag_peers_) {
      const int64_t mine = first_slot_of(rank_), theirs = first_slot_of(p);
      nck(ncclSend(w_up_c_.as<uint8_t>() + eb * mine * per_slot_up, n_ * per_slot_up, nccl_type(dt_), static_cast<int>(p), comm_->nccl, s), "send up");
      nck(ncclRecv(w_up_c_.as<uint8_t>() + eb * theirs * per_slot_up, n_ * per_slot_up, nccl_type(dt_), static_cast<int>(p), comm_->nccl, s), "recv up");
      nck(ncclSend(w_down_c_.as<uint8_t>() + eb * mine * per_slot_down, n_ * per_slot_down, nccl_type(dt_), static_cast<int>(p), comm_->nccl, s), "send down");
      nck(ncclRecv(w_down_c_.as<uint8_t>() + eb * theirs * per_slot_down, n_ * per_slot_down, nccl_type(dt_), static_cast<int>(p), comm_->nccl, s), "recv down");
    }
    nck(ncclGroupEnd(), "group end");
    return;
  }
  // SR migration: encode own experts against the shared expert, gather the wires,
  // decode each gathered wire straight into its compute slot.
  const int64_t P = 2 * H_ * F_;
  size_t wb = 0;
  hep_sr_config c{sr_cfg_.ratio_CR.value_or(1.0), sr_cfg_.k.value_or(-1), sr_cfg_.index_width_bits,
                  sr_cfg_.value_width_bits, sr_cfg_.per_matrix_budget ? 1 : 0};
  if (hep_sr_wire_bytes(H_, F_, &c, &wb) != HEP_OK) throw std::invalid_argument(hep_last_error());
  const size_t stride = (wb + 15) / 16 * 16;
  uint8_t* wires = wires_.as<uint8_t>();
  if (!wires_fresh_) {
    std::vector<const void*> ex;
    std::vector<void*> wo;
    for (int64_t i = 0; i < n_; ++i) {
      ex.push_back(master_.as<float>() + i * P);
      wo.push_back(wires + stride * (first_slot_of(rank_) + i));
    }
    if (hep_sr_encode_batch(ex.data(), static_cast<int>(n_), HEP_F32, shared_.as<float>(), H_, F_, &c, wo.data(), wb,
                            sr_ws_.p, sr_ws_.bytes, s) != HEP_OK)
      throw std::runtime_error(hep_last_error());
  }
  wires_fresh_ = false;
  nck(ncclGroupStart(), "group start");
  for (int64_t p : ag_peers_) {
    nck(ncclSend(wires + stride * first_slot_of(rank_), stride * n_, ncclUint8, static_cast<int>(p), comm_->nccl, s), "send wire");
    nck(ncclRecv(wires + stride * first_slot_of(p), stride * n_, ncclUint8, static_cast<int>(p), comm_->nccl, s), "recv wire");
  }
  nck(ncclGroupEnd(), "group end");
  decode_gathered(wb, stride, s);
}

void Layer::sgd_step(const float* const* grads, int n, float lr, cudaStream_t s) {
  if (!use_sr_) throw std::invalid_argument("the fused optimizer step updates the fp32 masters of SR-migrated layers");
  if (n != n_ || !grads) throw std::invalid_argument("one gradient per owned expert is required");
  if (p2p_) ensure_connected();
  if (ag_pending_) ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");  // the last encode read the masters
  if (p2p_ && ag_epoch_ > 0 && !ag_peers_.empty()) {
    // the wires are rewritten below: every AG peer has pulled the last epoch's (slot 4)
    P2PArgs prev = p2p_args_;
    prev.epoch = ag_epoch_;
    ck(launch_signal_wait(prev, 4, s, true, true, false), "wires pulled");
  }
  const int64_t P = 2 * H_ * F_;
  size_t wb = 0;
  hep_sr_config c{sr_cfg_.ratio_CR.value_or(1.0), sr_cfg_.k.value_or(-1), sr_cfg_.index_width_bits,
                  sr_cfg_.value_width_bits, sr_cfg_.per_matrix_budget ? 1 : 0};
  if (hep_sr_wire_bytes(H_, F_, &c, &wb) != HEP_OK) throw std::invalid_argument(hep_last_error());
  const size_t stride = (wb + 15) / 16 * 16;
  const int32_t first = slot_of_expert_[static_cast<size_t>(rank_ * n_)];
  std::vector<float*> ms;
  std::vector<void*> wo;
  for (int64_t i = 0; i < n_; ++i) {
    ms.push_back(master_.as<float>() + i * P);
    wo.push_back(wires_.as<uint8_t>() + stride * (first + i));
  }
  if (ag_peers_.empty()) {  // nothing migrates: the plain step
    if (hep_sgd_step_batch(ms.data(), grads, static_cast<int>(n_), P, lr, s) != HEP_OK)
      throw std::runtime_error(hep_last_error());
  } else {
    if (hep_sr_encode_update_batch(ms.data(), grads, static_cast<int>(n_), lr, shared_.as<float>(), H_, F_, &c,
                                   wo.data(), wb, sr_ws_.p, sr_ws_.bytes, s) != HEP_OK)
      throw std::runtime_error(hep_last_error());
    wires_fresh_ = true;
  }
  // the owned compute copies (GEMM layout, layer dtype) from the stepped masters
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  for (int64_t i = 0; i < n_; ++i) {
    const int64_t slot = first + i;
    ck(launch_transpose_convert(DType::F32, ms[static_cast<size_t>(i)], H_, F_, dt_,
                                w_up_c_.as<uint8_t>() + eb * slot * F_ * H_, s), "w_up layout");
    ck(launch_transpose_convert(DType::F32, ms[static_cast<size_t>(i)] + H_ * F_, F_, H_, dt_,
                                w_down_c_.as<uint8_t>() + eb * slot * H_ * F_, s), "w_down layout");
    slot_dirty_[static_cast<size_t>(slot)] = 1;
  }
}

void Layer::index_gathered(size_t wb, size_t stride, cudaStream_t s) {
  // Fused decode: each gathered wire -> its slot's per-stage patch blocks (validated like
  // the decode); the gathered experts' GEMMs read the shared expert and apply the patches
  // in-kernel.
  uint8_t* wires = wires_.as<uint8_t>();
  auto first_slot_of = [&](int64_t owner) { return slot_of_expert_[static_cast<size_t>(owner * n_)]; };
  bool corrupt = corrupt_next_;
  corrupt_next_ = false;
  for (int64_t p : ag_peers_) {
    const int64_t first = first_slot_of(p);
    if (corrupt) {  // test hook: break the first gathered wire's magic
      ck(cudaMemsetAsync(wires + stride * first, 0x58, 1, s), "corrupt");
      corrupt = false;
    }
    std::vector<const uint8_t*> wi;
    std::vector<uint8_t*> blocks;
    std::vector<uint2*> ovf;
    std::vector<int*> ovf_n;
    for (int64_t i = 0; i < n_; ++i) {
      const int64_t sl = first + i;
      wi.push_back(wires + stride * sl);
      blocks.push_back(patch_blocks_.as<uint8_t>() + sl * patch_slot_bytes_);
      ovf.push_back(patch_ovf_.as<uint2>() + sl * patch_kmax_);
      ovf_n.push_back(patch_ovf_n_.as<int>() + sl);
    }
    int32_t* st = sr_status_.as<int32_t>() + 4 * first;
    ck(launch_sr_patch_index(wi.data(), static_cast<int>(n_), wb, shared_.as<float>(), H_, F_, blocks.data(),
                             ovf.data(), ovf_n.data(), st, s), "patch index");
    ck(launch_sr_status_fold(st, static_cast<int>(n_), mig_err_dev_, s), "decode status");
  }
}

void Layer::decode_gathered(size_t wb, size_t stride, cudaStream_t s) {
  // Decode every gathered wire straight into its compute slot (shared expert copied in
  // by the copy engine, k entries scattered to their transposed positions).
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  const size_t per_slot = static_cast<size_t>(F_ * H_);
  uint8_t* wires = wires_.as<uint8_t>();
  auto first_slot_of = [&](int64_t owner) { return slot_of_expert_[static_cast<size_t>(owner * n_)]; };
  std::vector<int64_t> gathered;
  for (int64_t p : ag_peers_)
    for (int64_t i = 0; i < n_; ++i) gathered.push_back(first_slot_of(p) + i);
  if (corrupt_next_ && !gathered.empty()) {  // test hook: break the first gathered wire's magic
    ck(cudaMemsetAsync(wires + stride * gathered[0], 0x58, 1, s), "corrupt");
    corrupt_next_ = false;
  }
  for (size_t b0 = 0; b0 < gathered.size(); b0 += kMaxSrBatch) {
    const size_t nb = std::min(gathered.size() - b0, static_cast<size_t>(kMaxSrBatch));
    std::vector<const uint8_t*> wi;
    std::vector<void*> up, down;
    for (size_t i = 0; i < nb; ++i) {
      const int64_t slot = gathered[b0 + i];
      wi.push_back(wires + stride * slot);
      up.push_back(w_up_c_.as<uint8_t>() + eb * slot * per_slot);
      down.push_back(w_down_c_.as<uint8_t>() + eb * slot * per_slot);
    }
    ck(launch_sr_decode_layout_batch(wi.data(), static_cast<int>(nb), wb, shared_.as<float>(), shared_c_.p, dt_, H_,
                                     F_, up.data(), down.data(), sr_status_.as<int32_t>(), s),
       "decode");
    // a rejected wire (sparsecomp.cpp:36, 236-238) must not pass silently: fold the batch
    // status into the host-mapped error word that the next call (or check_migration) raises
    ck(launch_sr_status_fold(sr_status_.as<int32_t>(), static_cast<int>(nb), mig_err_dev_, s), "decode status");
  }
}

void Layer::check_migration(bool sync) {
  if (!use_sr_ || !mig_err_host_) return;
  if (sync) {
    if (ag_pending_) ck(cudaEventSynchronize(ev_ag_done_), "ag sync");
    ck(cudaDeviceSynchronize(), "sync");
  }
  const int32_t v = *reinterpret_cast<volatile int32_t*>(mig_err_host_);
  if (v == 0) return;
  *reinterpret_cast<volatile int32_t*>(mig_err_host_) = 0;
  const int code = v & 0xff, entry = v >> 8;
  std::string why;
  switch (code) {
    case 1: why = "bad residual magic"; break;
    case 2: why = "compressed residual truncated"; break;
    case 3: why = "unsupported residual widths"; break;
    case 4: why = "residual shape tag does not match the shared expert"; break;
    case 5: why = "corrupt residual: index out of bounds (entry " + std::to_string(entry) + ")"; break;
    case 6: why = "corrupt residual: indices not strictly increasing (entry " + std::to_string(entry) + ")"; break;
    default: why = "decode status " + std::to_string(code);
  }
  throw std::runtime_error("migrated expert rejected: " + why);
}

void Layer::mark(const char* name, cudaStream_t s, int level) {
  if (profiling_ < level) return;
  cudaEvent_t ev;
  if (marks_.size() < event_pool_.size()) {
    ev = event_pool_[marks_.size()];
  } else {
    ck(cudaEventCreate(&ev), "event");
    event_pool_.push_back(ev);
  }
  ck(cudaEventRecord(ev, s), "event record");
  marks_.emplace_back(name, ev);
}

void Layer::build_comm_plan_and_groups(int T, cudaStream_t s) {
  // Counts exchange: every rank learns every rank's (dest, expert) row counts.
  nck(ncclAllGather(key_total_.p, all_counts_.p, static_cast<size_t>(NK_), ncclInt32, comm_->nccl, s), "count allgather");
  h_counts_.resize(static_cast<size_t>(G_ * NK_));
  ck(cudaMemcpyAsync(h_counts_.data(), all_counts_.p, sizeof(int32_t) * G_ * NK_, cudaMemcpyDeviceToHost, s), "counts d2h");
  ck(cudaStreamSynchronize(s), "counts sync");
  auto cnt = [&](int64_t src, int64_t dest, int64_t e) {
    return static_cast<int64_t>(h_counts_[static_cast<size_t>(src * NK_ + dest * E_ + e)]);
  };
  // Send side: my packed buffer is grouped by (dest, expert).
  std::vector<int64_t> key_off(static_cast<size_t>(NK_));
  int64_t acc = 0;
  for (int64_t key = 0; key < NK_; ++key) {
    key_off[static_cast<size_t>(key)] = acc;
    acc += cnt(rank_, key / E_, key % E_);
  }
  (void)T;
  std::vector<int32_t> grs, grows, gslot;
  for (int64_t e = 0; e < E_; ++e) {
    const int32_t sl = slot_of_expert_[static_cast<size_t>(e)];
    if (sl < 0) continue;
    grs.push_back(static_cast<int32_t>(key_off[static_cast<size_t>(rank_ * E_ + e)]));
    grows.push_back(static_cast<int32_t>(cnt(rank_, rank_, e)));
    gslot.push_back(sl);
  }
  int64_t recv_at = Tmax_ * k_;
  for (size_t i = 0; i < a2a_peers_.size(); ++i) {
    const int64_t p = a2a_peers_[i];
    send_off_[i] = key_off[static_cast<size_t>(p * E_)];
    int64_t sr = 0;
    for (int64_t e = 0; e < E_; ++e) sr += cnt(rank_, p, e);
    send_rows_[i] = sr;
    recv_off_[i] = recv_at;
    int64_t rr = 0;
    for (int64_t e = 0; e < E_; ++e) {
      const int64_t c = cnt(p, rank_, e);
      if (c == 0) { continue; }
      const int32_t sl = slot_of_expert_[static_cast<size_t>(e)];
      if (sl < 0) throw std::runtime_error("received rows for an expert this GPU does not hold");
      grs.push_back(static_cast<int32_t>(recv_at + rr));
      grows.push_back(static_cast<int32_t>(c));
      gslot.push_back(sl);
      rr += c;
    }
    recv_rows_[i] = rr;
    recv_at += rr;
    if (recv_at > rows_cap_) throw std::runtime_error("received rows exceed the receive area (max_tokens mismatch)");
  }
  num_groups_ = static_cast<int>(grs.size());
  ck(cudaMemcpyAsync(g_row_start_.p, grs.data(), sizeof(int32_t) * grs.size(), cudaMemcpyHostToDevice, s), "groups");
  ck(cudaMemcpyAsync(g_rows_.p, grows.data(), sizeof(int32_t) * grows.size(), cudaMemcpyHostToDevice, s), "groups");
  ck(cudaMemcpyAsync(g_slot_.p, gslot.data(), sizeof(int32_t) * gslot.size(), cudaMemcpyHostToDevice, s), "groups");
}

void Layer::exchange(bool dispatch, cudaStream_t s) {
  if (a2a_peers_.empty()) return;
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  uint8_t* buf = (dispatch ? xall_ : oall_).as<uint8_t>();
  nck(ncclGroupStart(), "group start");
  for (size_t i = 0; i < a2a_peers_.size(); ++i) {
    const int p = static_cast<int>(a2a_peers_[i]);
    // dispatch: my rows for p go out, p's rows for me come in; combine reverses it.
    const int64_t out_off = dispatch ? send_off_[i] : recv_off_[i];
    const int64_t out_rows = dispatch ? send_rows_[i] : recv_rows_[i];
    const int64_t in_off = dispatch ? recv_off_[i] : send_off_[i];
    const int64_t in_rows = dispatch ? recv_rows_[i] : send_rows_[i];
    if (out_rows) nck(ncclSend(buf + eb * out_off * H_, out_rows * H_, nccl_type(dt_), p, comm_->nccl, s), "a2a send");
    if (in_rows) nck(ncclRecv(buf + eb * in_off * H_, in_rows * H_, nccl_type(dt_), p, comm_->nccl, s), "a2a recv");
  }
  nck(ncclGroupEnd(), "group end");
}

void Layer::run_expert_gemms(cudaStream_t s, const unsigned long long* out_down, const int* wait_src, int g0,
                             int ng, const char* tag, bool patched) {
  if (ng < 0) ng = num_groups_ - g0;
  if (ng <= 0) return;
  GroupTable gt{g_row_start_.as<int>() + g0, g_rows_.as<int>() + g0, g_slot_.as<int>() + g0, ng};
  GroupTable gt_down = gt;
  gt_down.out = out_down ? out_down + g0 : nullptr;
  if (wait_src) {
    gt.wait_src = wait_src + g0;
    gt.wait_flags = p2p_dispatch_flags(p2p_args_);
    gt.epoch = p2p_args_.epoch;
    gt.timeout_ns = timeout_ns_;
  }
  const std::string up = std::string("gemm_up") + tag, down = std::string("gemm_down") + tag;
  if (dt_ == DType::BF16 && patched) {
    // gathered SR experts: decode fused into the B-operand load (shared expert + patches)
    const PatchArgs refs{patch_blocks_.as<uint8_t>(), patch_slot_bytes_, 0, patch_refs_.as<PatchRef>()};
    PatchArgs refs_down = refs;
    refs_down.half_bytes = static_cast<size_t>(patch_blocks(F_, H_)) * kPatchBlockBytes;
    auto gemm = cta_pair_ ? launch_grouped_gemm_bf16_2cta_patched : launch_grouped_gemm_bf16_patched;
    const uint32_t sched = cta_pair_ ? 0x2u : 0x8u;  // the shared B is re-read by every group: keep A resident
    mark(up.c_str(), s, 1);
    ck(gemm(map_a1_, map_shared_up_, hbuf_.p, static_cast<int>(F_), static_cast<int>(F_), static_cast<int>(H_), gt,
            refs, 0, 1, num_sms_, s, sched),
       "gemm up (fused decode)");
    mark(down.c_str(), s, 1);
    ck(gemm(map_a2_, map_shared_down_, oall_.p, static_cast<int>(H_), static_cast<int>(H_), static_cast<int>(F_),
            gt_down, refs_down, 1, 0, num_sms_, s, sched),
       "gemm down (fused decode)");
  } else if (dt_ == DType::BF16) {
    mark(up.c_str(), s, 1);
    if (cta_pair_) {
      int* ctr = tile_counters_.as<int>();  // dynamic tile scheduler counters (zeroed in-stream per launch)
      // Dynamic tile queue (counter passed): HEP_GEMM_DYN=down on the down-projection only
      // (its long-K tiles keep a compact L2 window: -22% DRAM reads, +1-4% on cfg3 N=1),
      // =1 on both.  Static by default: the 8-layer cfg5 stack at N=4 hung once with the
      // down-projection queue on, which is not yet understood (profiles/r2_gemm_power.md).
      const char* dyn = std::getenv("HEP_GEMM_DYN");
      const bool dyn_up = dyn && dyn[0] == '1', dyn_down = dyn && (dyn[0] == '1' || dyn[0] == 'd');
      ck(launch_grouped_gemm_bf16_2cta(map_a1_, map_b1_, hbuf_.p, static_cast<int>(F_), static_cast<int>(F_),
                                       static_cast<int>(H_), gt, 1, num_sms_, s, sched_up_, dyn_up ? ctr : nullptr,
                                       gather_now_ ? row_src_.as<int>() : nullptr, gather_now_ ? last_x_ : nullptr),
         "gemm up");
      mark(down.c_str(), s, 1);
      ck(launch_grouped_gemm_bf16_2cta(map_a2_, map_b2_, oall_.p, static_cast<int>(H_), static_cast<int>(H_),
                                       static_cast<int>(F_), gt_down, 0, num_sms_, s, sched_down_,
                                       dyn_down ? ctr + 1 : nullptr),
         "gemm down");
    } else {
      ck(launch_grouped_gemm_bf16(map_a1_, map_b1_, hbuf_.p, static_cast<int>(F_), static_cast<int>(F_),
                                  static_cast<int>(H_), gt, 1, num_sms_, s, sched_up_),
         "gemm up");
      mark(down.c_str(), s, 1);
      ck(launch_grouped_gemm_bf16(map_a2_, map_b2_, oall_.p, static_cast<int>(H_), static_cast<int>(H_),
                                  static_cast<int>(F_), gt_down, 0, num_sms_, s, sched_down_),
         "gemm down");
    }
  } else if (tf32_) {
    mark(up.c_str(), s, 1);
    split_dirty_slots(s);
    ck(launch_split_tf32(xall_.as<float>(), xhi_.as<float>(), xlo_.as<float>(), rows_cap_ * H_, s), "split x");
    ck(launch_grouped_gemm_tf32x3(t_xhi_, t_xlo_, t_wuhi_, tf32_presplit_ ? &t_wulo_ : nullptr, hhi_.as<float>(), hlo_.as<float>(),
                                  static_cast<int>(F_), static_cast<int>(F_), static_cast<int>(H_), gt, 1, num_sms_, s,
                                  ksplit_up_, kpart_.as<float>(), rows_cap_),
       "gemm up");
    mark(down.c_str(), s, 1);
    ck(launch_grouped_gemm_tf32x3(t_hhi_, t_hlo_, t_wdhi_, tf32_presplit_ ? &t_wdlo_ : nullptr, oall_.as<float>(), nullptr, static_cast<int>(H_),
                                  static_cast<int>(H_), static_cast<int>(F_), gt, 0, num_sms_, s, ksplit_down_,
                                  kpart_.as<float>(), rows_cap_),
       "gemm down");
    launches_ += 1 + (ksplit_up_ > 1) + (ksplit_down_ > 1);  // x split, split-K reduces
  } else {
    mark(up.c_str(), s, 1);
    ck(launch_grouped_gemm_f32(xall_.as<float>(), static_cast<int>(H_), w_up_c_.as<float>(), hbuf_.as<float>(), static_cast<int>(F_), static_cast<int>(F_), static_cast<int>(H_), gt, 1, num_sms_ * 2, s), "gemm up");
    mark(down.c_str(), s, 1);
    ck(launch_grouped_gemm_f32(hbuf_.as<float>(), static_cast<int>(F_), w_down_c_.as<float>(), oall_.as<float>(), static_cast<int>(H_), static_cast<int>(H_), static_cast<int>(F_), gt, 0, num_sms_ * 2, s), "gemm down");
  }
  launches_ += 2;
  if (profiling_ == 1) mark("end", s, 1);  // GEMM-only profiling: close the down interval
}

void Layer::forward(const void* x, int64_t T, void* y, cudaStream_t s, bool residual) {
  if (T < 0 || T > Tmax_) throw std::invalid_argument("token count must be in [0, max_tokens]");
  if (residual && x == y) throw std::invalid_argument("the residual form needs y distinct from x");
  if (!forward_graph(x, T, y, s, residual)) step(x, T, y, s, residual);
  // A gathered expert whose wire failed to decode (found once that decode has completed)
  // is reported after this rank's share of the collective step is enqueued, so its peers
  // never wait for a rank that bailed out.
  check_migration(false);
}

void Layer::step(const void* x, int64_t T, void* y, cudaStream_t s, bool residual) {
  // T = 0 is legal: a rank with an empty batch still takes part in the exchange (it
  // sends no rows, receives its peers' rows and runs their experts).
  if (T < 0 || T > Tmax_) throw std::invalid_argument("token count must be in [0, max_tokens]");
  if (p2p_) ensure_connected();
  launches_ = 0;
  gather_now_ = false;
  const int Ti = static_cast<int>(T);
  const int nchunks = (Ti + 31) / 32;
  mark("gate", s);
  if (Ti > 0) {
    ck(launch_gate(dt_, x, wg_t_.p, Ti, static_cast<int>(H_), static_cast<int>(E_), static_cast<int>(k_),
                   d_route_.as<int>(), static_cast<int>(n_), static_cast<int>(NK_), topk_idx_.as<int>(),
                   topk_w_.as<float>(), keys_.as<int>(), ranks_.as<int>(), chunk_counts_.as<int>(), s), "gate");
  }
  mark("scan", s);
  if (Ti > 0) {
    ck(launch_chunk_scan(chunk_counts_.as<int>(), nchunks, static_cast<int>(NK_), chunk_off_.as<int>(), key_total_.as<int>(), s), "chunk scan");
  } else {
    ck(cudaMemsetAsync(key_total_.p, 0, sizeof(int32_t) * static_cast<size_t>(NK_), s), "zero counts");
  }
  ck(launch_key_scan(key_total_.as<int>(), static_cast<int>(G_), static_cast<int>(E_), rank_, d_slot_of_expert_.as<int>(),
                     key_off_.as<int>(), dest_rows_.as<int>(), dest_off_.as<int>(), g_row_start_.as<int>(),
                     g_rows_.as<int>(), g_slot_.as<int>(), s), "key scan");
  launches_ += 3;
  num_groups_ = static_cast<int>(slots_);
  if (p2p_) {
    // Device-side count exchange, then rows go straight into peers' receive areas.
    p2p_args_.epoch = ++epoch_;
    mark("dispatch", s);
    ck(launch_count_exchange(p2p_args_, key_total_.as<int>(), key_off_.as<int>(), d_slot_of_expert_.as<int>(),
                             send_base_.as<int>(), g_row_start_.as<int>(), g_rows_.as<int>(), g_slot_.as<int>(),
                             g_out_down_.as<unsigned long long>(), g_wait_.as<int>(), all_counts_.as<int>(), s),
       "count exchange");
    num_groups_ = static_cast<int>(slots_ * (1 + p2p_args_.n_src[rank_]));
    if (dt_ == DType::BF16) {
      // Overlapped dispatch: remote rows go out over NVLink on a side stream while the
      // up-projection starts on local rows; its TMA producer waits per source group
      // for that source's dispatch flag.
      ck(cudaEventRecord(ev_counts_, s), "record");
      ck(cudaStreamWaitEvent(side_s_, ev_counts_, 0), "wait");
      ck(launch_permute_p2p(p2p_args_, dt_, x, Ti, static_cast<int>(H_), static_cast<int>(k_), keys_.as<int>(),
                            ranks_.as<int>(), chunk_off_.as<int>(), key_off_.as<int>(), send_base_.as<int>(),
                            pos_.as<int>(), side_s_, 2), "permute remote");
      ck(launch_signal_wait(p2p_args_, 1, side_s_, false), "dispatch flags");
      ck(cudaEventRecord(ev_remote_, side_s_), "record");
      if (!spin_) {
        // every source's rows have landed: only this one-warp kernel spins, never the
        // persistent GEMM (which could otherwise hold every SM while a peer's dispatch
        // waits for SM space behind it)
        ck(launch_signal_wait(p2p_args_, 1, side_s_, true, false, false), "dispatch arrived");
        ck(cudaEventRecord(ev_arrived_, side_s_), "record");
        ++launches_;
      }
      ck(launch_permute_p2p(p2p_args_, dt_, x, Ti, static_cast<int>(H_), static_cast<int>(k_), keys_.as<int>(),
                            ranks_.as<int>(), chunk_off_.as<int>(), key_off_.as<int>(), send_base_.as<int>(),
                            pos_.as<int>(), s, 1), "permute local");
      launches_ += 4;
      // The down-projection writes received rows' outputs straight into their source
      // GPU's oall (fused GEMM + combine exchange); the combine reads local HBM only.
      const int n_src = p2p_args_.n_src[rank_];
      const int own_local = static_cast<int>(n_), own = static_cast<int>(n_ * (1 + n_src));
      const unsigned long long* out_down = g_out_down_.as<unsigned long long>();
      if (!spin_ && merge_mode_ == 2) {
        // HEP_MERGE_GEMMS=2: own and received rows in one launch per projection once the
        // dispatch has landed; gathered experts after the All-Gather, as in the default.
        ck(cudaStreamWaitEvent(s, ev_arrived_, 0), "wait dispatch");
        run_expert_gemms(s, out_down, nullptr, 0, own);
        if (num_groups_ > own) {
          if (ag_pending_) {
            mark("ag_wait", s);
            ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");
          }
          run_expert_gemms(s, out_down, nullptr, own, num_groups_ - own, "_gathered", sr_fused_);
        }
        ag_pending_ = false;
      } else if (!spin_ && merge_gemms_) {
        // HEP_MERGE_GEMMS=1: one up + one down launch over every group, once the remote
        // rows and the All-Gather have landed (fewer launch tails, no overlap).
        ck(cudaStreamWaitEvent(s, ev_arrived_, 0), "wait dispatch");
        if (ag_pending_ && num_groups_ > own) {
          mark("ag_wait", s);
          ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");
        }
        run_expert_gemms(s, out_down, nullptr, 0, num_groups_, "", false);
        ag_pending_ = false;
      } else if (!spin_) {
        // Own experts' local rows overlap the remote dispatch; received rows follow once
        // they have all landed; gathered experts once the All-Gather is resident.
        run_expert_gemms(s, out_down, nullptr, 0, own_local);
        ck(cudaStreamWaitEvent(s, ev_arrived_, 0), "wait dispatch");
        if (own > own_local) run_expert_gemms(s, out_down, nullptr, own_local, own - own_local, "_remote");
        if (num_groups_ > own) {
          if (ag_pending_) {
            mark("ag_wait", s);
            ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");
          }
          run_expert_gemms(s, out_down, nullptr, own, num_groups_ - own, "_gathered", sr_fused_);
        }
        ag_pending_ = false;
      } else if (ag_pending_) {
        // own experts first (weights already resident), gathered ones after the AG lands
        run_expert_gemms(s, out_down, g_wait_.as<int>(), 0, own);
        mark("ag_wait", s);
        ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");
        ag_pending_ = false;
        run_expert_gemms(s, out_down, g_wait_.as<int>(), own, num_groups_ - own, "_gathered", sr_fused_);
      } else {
        run_expert_gemms(s, out_down, g_wait_.as<int>());
      }
      ck(cudaStreamWaitEvent(s, ev_remote_, 0), "wait");
      mark("combine", s);
      ck(launch_signal_wait(p2p_args_, 2, s), "combine flags");
      ck(launch_combine(dt_, oall_.p, pos_.as<int>(), topk_w_.as<float>(), Ti, static_cast<int>(H_), static_cast<int>(k_), y, s,
                        residual ? x : nullptr), "combine");
    } else {
      ck(launch_permute_p2p(p2p_args_, dt_, x, Ti, static_cast<int>(H_), static_cast<int>(k_), keys_.as<int>(),
                            ranks_.as<int>(), chunk_off_.as<int>(), key_off_.as<int>(), send_base_.as<int>(),
                            pos_.as<int>(), s), "permute p2p");
      ck(launch_signal_wait(p2p_args_, 1, s), "dispatch flags");
      launches_ += 3;
      if (ag_pending_) {  // the All-Gather pulled on the copy engines while gate + dispatch ran
        mark("ag_wait", s);
        ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");
        ag_pending_ = false;
      }
      run_expert_gemms(s);
      mark("combine", s);
      ck(launch_signal_wait(p2p_args_, 2, s), "combine flags");
      ck(launch_combine_p2p(p2p_args_, dt_, keys_.as<int>(), pos_.as<int>(), key_off_.as<int>(), send_base_.as<int>(),
                            topk_w_.as<float>(), Ti, static_cast<int>(H_), static_cast<int>(k_), y, s, residual ? x : nullptr), "combine p2p");
    }
    launches_ += 2;
    mark("end", s);
    return;
  }
  mark("permute", s);
  if (gather_a_ && Ti > 0) {
    // positions + the inverse map only; the up-projection gathers x rows itself
    ck(launch_positions(Ti, static_cast<int>(k_), static_cast<int>(NK_), keys_.as<int>(), ranks_.as<int>(),
                        chunk_off_.as<int>(), key_off_.as<int>(), pos_.as<int>(), s, row_src_.as<int>()),
       "positions");
    gather_now_ = true;
    packed_stale_ = true;
    last_x_ = x;
    last_T_ = T;
  } else {
    ck(launch_permute(dt_, x, Ti, static_cast<int>(H_), static_cast<int>(k_), static_cast<int>(NK_), keys_.as<int>(),
                      ranks_.as<int>(), chunk_off_.as<int>(), key_off_.as<int>(), pos_.as<int>(), xall_.p, s), "permute");
    packed_stale_ = false;
  }
  launches_ += 1;
  if (G_ > 1) {
    mark("dispatch", s);
    build_comm_plan_and_groups(Ti, s);
    exchange(true, s);
  }
  run_expert_gemms(s);
  if (G_ > 1) {
    mark("combine_a2a", s);
    exchange(false, s);
  }
  mark("combine", s);
  ck(launch_combine(dt_, oall_.p, pos_.as<int>(), topk_w_.as<float>(), Ti, static_cast<int>(H_), static_cast<int>(k_), y, s,
                    residual ? x : nullptr), "combine");
  launches_ += 1;
  mark("end", s);
}

void Layer::comm_bench(const void* x, int64_t T, int iters, double* out, cudaStream_t s) {
  for (int i = 0; i < 6; ++i) out[i] = 0.0;
  if (G_ == 1) return;
  if (p2p_) ensure_connected();
  init_host_staging();
  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "event");
  ck(cudaEventCreate(&e1), "event");
  const size_t eb = static_cast<size_t>(dtype_bytes(dt_));
  if (p2p_) {
    // A2A dispatch over NVLink: rows this GPU sends to peers, timed on the permute that
    // stores them (remote rows only), after a full forward has set up the plan.
    forward(x, T, y_dev_[0].p, s);
    std::vector<int32_t> cnt(static_cast<size_t>(NK_));
    ck(cudaMemcpyAsync(cnt.data(), key_total_.p, sizeof(int32_t) * NK_, cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "sync");
    int64_t out_rows = 0;
    for (int64_t key = 0; key < NK_; ++key)
      if (key / E_ != rank_) out_rows += cnt[static_cast<size_t>(key)];
    const int Ti = static_cast<int>(T);
    float total = 0.f;
    for (int it = 0; it < iters; ++it) {
      ck(cudaEventRecord(e0, s), "record");
      ck(launch_permute_p2p(p2p_args_, dt_, x, Ti, static_cast<int>(H_), static_cast<int>(k_), keys_.as<int>(),
                            ranks_.as<int>(), chunk_off_.as<int>(), key_off_.as<int>(), send_base_.as<int>(),
                            pos_.as<int>(), s, 2), "permute remote");
      ck(cudaEventRecord(e1, s), "record");
      ck(cudaEventSynchronize(e1), "sync");
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
      total += ms;
    }
    out[0] = total / iters;
    out[1] = static_cast<double>(out_rows) * H_ * eb;
  }
  if (!ag_peers_.empty()) {
    // the peer-memory All-Gather runs on its own stream: join it before each timing point
    auto join = [&] {
      if (ag_pending_) {
        ck(cudaStreamWaitEvent(s, ev_ag_done_, 0), "wait ag");
        ag_pending_ = false;
      }
    };
    gather_experts(s);
    join();
    ck(cudaEventRecord(e0, s), "record");
    for (int it = 0; it < iters; ++it) {
      gather_experts(s);
      join();
    }
    ck(cudaEventRecord(e1, s), "record");
    ck(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    out[3] = ms / iters;
    const double per_expert = use_sr_ ? static_cast<double>(wires_.bytes) / static_cast<double>(slots_)
                                      : static_cast<double>(2 * H_ * F_ * eb);
    out[4] = static_cast<double>(ag_peers_.size()) * n_ * per_expert;
    if (p2p_) {
      // the NVLink transfer alone: the same peer pulls (copy engines), no encode / decode /
      // flags, into scratch
      const size_t wb_stride = use_sr_ ? wires_.bytes / static_cast<size_t>(slots_) : 0;
      const size_t per_peer = use_sr_ ? wb_stride * static_cast<size_t>(n_)
                                      : eb * static_cast<size_t>(n_) * static_cast<size_t>(F_ * H_);
      DevBuf scratch;
      scratch.alloc(per_peer * (use_sr_ ? 1 : 2));
      ck(cudaEventRecord(e0, s), "record");
      for (int it = 0; it < iters; ++it)
        for (int64_t p : ag_peers_) {
          const size_t pi = static_cast<size_t>(p);
          if (use_sr_) {
            ck(cudaMemcpyAsync(scratch.p, peer_wires_[pi], per_peer, cudaMemcpyDeviceToDevice, s), "pull");
          } else {
            ck(cudaMemcpyAsync(scratch.p, peer_w_up_[pi], per_peer, cudaMemcpyDeviceToDevice, s), "pull");
            ck(cudaMemcpyAsync(scratch.as<uint8_t>() + per_peer, peer_w_down_[pi], per_peer, cudaMemcpyDeviceToDevice, s),
               "pull");
          }
        }
      ck(cudaEventRecord(e1, s), "record");
      ck(cudaEventSynchronize(e1), "sync");
      ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
      out[5] = ms / iters;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

void Layer::collect_timings(char* names, size_t names_cap, float* ms, int cap, int* count) {
  std::vector<std::string> order;
  std::vector<double> total;
  std::vector<int> hits;
  if (!marks_.empty()) ck(cudaEventSynchronize(marks_.back().second), "event sync");
  for (size_t i = 0; i + 1 < marks_.size(); ++i) {
    if (marks_[i].first == "end") continue;  // forward boundary
    float t = 0.f;
    ck(cudaEventElapsedTime(&t, marks_[i].second, marks_[i + 1].second), "elapsed");
    size_t j = 0;
    while (j < order.size() && order[j] != marks_[i].first) ++j;
    if (j == order.size()) { order.push_back(marks_[i].first); total.push_back(0); hits.push_back(0); }
    total[j] += t;
    hits[j] += 1;
  }
  marks_.clear();
  std::string joined;
  int c = 0;
  for (size_t j = 0; j < order.size() && c < cap; ++j, ++c) {
    ms[c] = static_cast<float>(total[j] / hits[j]);
    if (!joined.empty()) joined += ';';
    joined += order[j];
  }
  *count = c;
  if (names && names_cap) {
    std::strncpy(names, joined.c_str(), names_cap - 1);
    names[names_cap - 1] = 0;
  }
}

const void* Layer::packed() {
  if (packed_stale_) {
    // the caller's x of the last step must still be alive (debug / inspection use)
    ck(cudaDeviceSynchronize(), "sync");
    ck(launch_permute(dt_, last_x_, static_cast<int>(last_T_), static_cast<int>(H_), static_cast<int>(k_),
                      static_cast<int>(NK_), keys_.as<int>(), ranks_.as<int>(), chunk_off_.as<int>(),
                      key_off_.as<int>(), pos_.as<int>(), xall_.p, nullptr),
       "permute (inspection)");
    ck(cudaDeviceSynchronize(), "sync");
    packed_stale_ = false;
  }
  return xall_.p;
}

void Layer::forward_host(const void* hx, int64_t T, void* hy, cudaStream_t s) {
  const size_t bytes = static_cast<size_t>(T * H_ * dtype_bytes(dt_));
  if (T < 0 || T > Tmax_) throw std::invalid_argument("token count must be in [0, max_tokens]");
  init_host_staging();
  const int b = hslot_;
  hslot_ ^= 1;
  // H2D on its own stream once the step that last used this slot stopped reading it.
  ck(cudaStreamWaitEvent(h2d_s_, ev_comp_[b], 0), "wait");
  ck(cudaMemcpyAsync(x_dev_[b].p, hx, bytes, cudaMemcpyHostToDevice, h2d_s_), "h2d");
  ck(cudaEventRecord(ev_h2d_[b], h2d_s_), "record");
  // The step itself on the caller's stream.
  ck(cudaStreamWaitEvent(s, ev_h2d_[b], 0), "wait");
  ck(cudaStreamWaitEvent(s, ev_d2h_[b], 0), "wait");
  forward(x_dev_[b].p, T, y_dev_[b].p, s);
  ck(cudaEventRecord(ev_comp_[b], s), "record");
  // D2H of the result on the other copy engine.
  ck(cudaStreamWaitEvent(d2h_s_, ev_comp_[b], 0), "wait");
  ck(cudaMemcpyAsync(hy, y_dev_[b].p, bytes, cudaMemcpyDeviceToHost, d2h_s_), "d2h");
  ck(cudaEventRecord(ev_d2h_[b], d2h_s_), "record");
}

void Layer::host_fence(cudaStream_t s) {
  if (!h2d_s_) return;
  ck(cudaStreamWaitEvent(s, ev_d2h_[0], 0), "wait");
  ck(cudaStreamWaitEvent(s, ev_d2h_[1], 0), "wait");
}

}  // namespace hep
