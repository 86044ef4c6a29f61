// K2/K3/K9 fused with NVLink peer memory: the domain-based token A2A without NCCL and
// without a host round trip.
//
//   count exchange  every rank stores its (dest, expert) row counts straight into every
//                   peer's inbox (NVLink stores), raises a flag, waits for all flags;
//                   then derives on device where its rows land in each destination's
//                   receive area and the GEMM group table for rows it will receive.
//   dispatch        permute_p2p writes each (token, slot) row either into the local
//                   packed buffer or directly into the destination GPU's receive area.
//   combine         after the outputs-ready flags, combine_p2p gathers every expert
//                   output row from local HBM or from the computing peer's HBM.
//
// Receive area of GPU d: rows [Tmax*k, ...) of its xall/oall, ordered by source in
// d's A2A peer-list order (simcore.cpp:53-72), then by expert, then (token, slot):
// the same layout the NCCL path produces, so both paths feed the same GEMM groups.
// Flags carry a per-forward epoch; spins time out (trap) instead of hanging.

#include <cstdlib>
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "comm_p2p.h"

namespace hep {

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// who: (rank << 16) | (site << 8) | peer, printed if the wait times out.  Sites: 0 counts,
// 11..14 signal slots 1..4, 20 refresh barrier, 21 refresh chain, 22 refresh fetch.
// timeout_ns = 0 waits forever (ranks may legitimately skew by minutes: checkpointing,
// evaluation); a finite HEP_P2P_TIMEOUT_S turns a lost peer into a diagnosed trap.
__device__ void wait_flag(const uint32_t* f, uint32_t epoch, uint32_t who, uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer();
  // Epochs only grow; a peer that already moved on to a later epoch also satisfies us.
  while (static_cast<int32_t>(ld_acquire_sys(f) - epoch) < 0) {
    if (timeout_ns && globaltimer() - t0 > timeout_ns) {  // peer never arrived
      printf("hep: flag wait timed out: rank %u site %u peer %u epoch %u flag %u\n", who >> 16, (who >> 8) & 0xffu,
             who & 0xffu, epoch, ld_acquire_sys(f));
      __trap();
    }
    __nanosleep(64);
  }
}

// Sync buffer of one rank (in its HBM, written by peers).
struct SyncView {
  uint32_t* flags;  // [5][kMaxG]: 0 counts, 1 dispatched, 2 outputs ready, 3 experts final,
                    // 4 "pulled your wires"; index = source
  int* inbox;       // [2][kMaxG][NK]: counts of every source, double-buffered by epoch parity
};

__device__ __forceinline__ SyncView view(void* base, int NK) {
  SyncView v;
  v.flags = static_cast<uint32_t*>(base);
  v.inbox = reinterpret_cast<int*>(static_cast<uint8_t*>(base) + kSyncSlots * kMaxG * sizeof(uint32_t));
  (void)NK;
  return v;
}

__global__ void __launch_bounds__(256) count_exchange_kernel(P2PArgs a, const int* __restrict__ key_total,
                                                             const int* __restrict__ key_off,
                                                             const int* __restrict__ slot_of_expert,
                                                             int* __restrict__ send_base, int* __restrict__ g_row_start,
                                                             int* __restrict__ g_rows, int* __restrict__ g_slot,
                                                             unsigned long long* __restrict__ g_out_down,
                                                             int* __restrict__ g_wait, int* __restrict__ counts_out) {
  const int G = a.G, E = a.E, NK = G * E, me = a.rank;
  const int par = a.epoch & 1;
  __shared__ int cnt[kMaxG * kMaxG * kMaxE];  // cnt[s][d*E+e]
  // 1) broadcast my counts into every rank's inbox (including mine).
  for (int d = 0; d < G; ++d) {
    const SyncView v = view(a.sync[d], NK);
    int* dst = v.inbox + (par * kMaxG + me) * NK;
    for (int i = threadIdx.x; i < NK; i += blockDim.x) dst[i] = key_total[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < G && static_cast<int>(threadIdx.x) != me)
    st_release_sys(view(a.sync[threadIdx.x], NK).flags + 0 * kMaxG + me, a.epoch);
  // 2) wait for everyone's counts.
  const SyncView mine = view(a.sync[me], NK);
  if (threadIdx.x < G && static_cast<int>(threadIdx.x) != me)
    wait_flag(mine.flags + 0 * kMaxG + threadIdx.x, a.epoch, (static_cast<uint32_t>(me) << 16) | threadIdx.x,
              a.timeout_ns);
  __syncthreads();
  for (int i = threadIdx.x; i < G * NK; i += blockDim.x) {
    const int s = i / NK, key = i % NK;
    const int v = s == me ? key_total[key] : ld_acquire_sys(reinterpret_cast<const uint32_t*>(mine.inbox + (par * kMaxG + s) * NK + key));
    cnt[i] = v;
    counts_out[i] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  // 3) where my rows for (d, e) land in d's receive area.
  for (int d = 0; d < G; ++d) {
    if (d == me) {
      for (int e = 0; e < E; ++e) send_base[d * E + e] = key_off[d * E + e];
      continue;
    }
    int base = a.recv_start;
    for (int i = 0; i < a.n_src[d]; ++i) {
      const int s = a.src_list[d * kMaxG + i];
      if (s == me) break;
      for (int e = 0; e < E; ++e) base += cnt[s * NK + d * E + e];
    }
    for (int e = 0; e < E; ++e) {
      send_base[d * E + e] = base;
      base += cnt[me * NK + d * E + e];
    }
  }
  // 4) GEMM groups: local rows per held expert, then received rows per (source, expert).
  //    Down-projection outputs of received rows go straight back to the source's oall at
  //    key_off_s(me, e), the rows its combine reads.
  auto row_addr = [&](int rank, long long row) {
    return reinterpret_cast<unsigned long long>(static_cast<uint8_t*>(a.oall[rank]) + row * a.row_bytes);
  };
  // Groups of this GPU's own experts come first, gathered experts after them, so the
  // step can run the own-expert GEMMs while the expert All-Gather is still in flight.
  const int n_own = E / G;
  int g = 0;
  for (int pass = 0; pass < 2; ++pass) {
    auto in_pass = [&](int e) { return ((e / n_own) == me) == (pass == 0); };
    for (int e = 0; e < E; ++e) {
      const int sl = slot_of_expert[e];
      if (sl < 0 || !in_pass(e)) continue;
      g_row_start[g] = key_off[me * E + e];
      g_rows[g] = cnt[me * NK + me * E + e];
      g_out_down[g] = row_addr(me, key_off[me * E + e]);
      g_wait[g] = -1;
      g_slot[g++] = sl;
    }
    int at = a.recv_start;
    for (int i = 0; i < a.n_src[me]; ++i) {
      const int s = a.src_list[me * kMaxG + i];
      long long src_off = 0;  // key_off of source s for key (me, 0)
      for (int key = 0; key < me * E; ++key) src_off += cnt[s * NK + key];
      for (int e = 0; e < E; ++e) {
        const int sl = slot_of_expert[e];
        const int c = cnt[s * NK + me * E + e];
        if (sl >= 0) {  // a source only routes to this GPU experts it holds (S2)
          if (in_pass(e)) {
            g_row_start[g] = at;
            g_rows[g] = c;
            g_out_down[g] = row_addr(s, src_off);
            g_wait[g] = s;
            g_slot[g++] = sl;
          }
          at += c;
        }
        src_off += c;
      }
    }
  }
}

// One warp per token: local rows into the packed buffer, remote rows straight into the
// destination's receive area over NVLink.
__global__ void __launch_bounds__(256) permute_p2p_kernel(P2PArgs a, const uint8_t* __restrict__ x, int T_tok,
                                                          int row_bytes, int k, const int* __restrict__ keys,
                                                          const int* __restrict__ ranks,
                                                          const int* __restrict__ chunk_off,
                                                          const int* __restrict__ key_off,
                                                          const int* __restrict__ send_base, int* __restrict__ pos,
                                                          int mode, int seg) {
  // mode 0: every row; 1: rows staying on this GPU (and all of pos); 2: remote rows only.
  // Grid-stride over (token, segment) warps: the remote pass runs on a capped grid so
  // the own-expert GEMM's CTAs find room beside it (overlapped dispatch).
  const int lane = threadIdx.x & 31;
  const int NK = a.G * a.E;
  const int vecs = row_bytes >> 4;
  const int per = ((vecs + seg - 1) / seg + 31) & ~31;
  const int nwarps = static_cast<int>(gridDim.x * (blockDim.x >> 5));
  for (int w = blockIdx.x * static_cast<int>(blockDim.x >> 5) + static_cast<int>(threadIdx.x >> 5);
       w < T_tok * seg; w += nwarps) {
    const int t = w / seg, sg = w - t * seg;
    const int v0 = sg * per, v1 = min(vecs, v0 + per);
    const int chunk = t / 32;
    uint8_t* dst[8];
    bool any = false;
    for (int j = 0; j < k; ++j) {
      const size_t o = static_cast<size_t>(t) * k + j;
      const int key = keys[o];
      const int p = key_off[key] + chunk_off[static_cast<size_t>(chunk) * NK + key] + ranks[o];
      if (lane == 0 && sg == 0 && mode != 2) pos[o] = p;
      const int d = key / a.E;
      const bool skip = (mode == 1 && d != a.rank) || (mode == 2 && d == a.rank);
      const int row = d == a.rank ? p : send_base[key] + (p - key_off[key]);
      dst[j] = skip ? nullptr : static_cast<uint8_t*>(a.xall[d]) + static_cast<size_t>(row) * row_bytes;
      any |= !skip;
    }
    if (!any) continue;
    const uint8_t* src = x + static_cast<size_t>(t) * row_bytes;
    for (int v = v0 + lane; v < v1; v += 32) {
      const uint4 val = ld_nc_v4(src + 16 * v);
      for (int j = 0; j < k; ++j)
        if (dst[j]) st_v4(dst[j] + 16 * v, val);
    }
  }
}

// Raise flag `slot` on every A2A peer, then (if `wait`) wait for theirs.
__global__ void signal_wait_kernel(P2PArgs a, int slot, int wait, int ag, int sig) {
  __threadfence_system();
  const int NK = a.G * a.E;
  const int i = threadIdx.x;
  const int n = ag ? a.n_ag : a.n_src[a.rank];
  const int* list = ag ? a.ag_list : a.src_list + a.rank * kMaxG;
  if (sig && i < n) st_release_sys(view(a.sync[list[i]], NK).flags + slot * kMaxG + a.rank, a.epoch);
  if (!wait) return;
  __syncthreads();
  if (i < n)
    wait_flag(view(a.sync[a.rank], NK).flags + slot * kMaxG + list[i], a.epoch,
              (static_cast<uint32_t>(a.rank) << 16) | ((10u + slot) << 8) | static_cast<uint32_t>(list[i]), a.timeout_ns);
}

template <bool BF16>
__global__ void __launch_bounds__(256) combine_p2p_kernel(P2PArgs a, const int* __restrict__ keys,
                                                          const int* __restrict__ pos,
                                                          const int* __restrict__ key_off,
                                                          const int* __restrict__ send_base,
                                                          const float* __restrict__ w, int T_tok, int H, int k,
                                                          void* __restrict__ y, int seg,
                                                          const void* __restrict__ residual) {
  const int lane = threadIdx.x & 31;
  const int eb = BF16 ? 2 : 4;
  int t, sg, v0, v1;
  row_segment(H * eb / 16, seg, t, sg, v0, v1);
  if (t >= T_tok) return;
  const uint8_t* row[8];
  float wt[8];
  for (int j = 0; j < k; ++j) {
    const size_t o = static_cast<size_t>(t) * k + j;
    const int key = keys[o], p = pos[o], d = key / a.E;
    const int r = d == a.rank ? p : send_base[key] + (p - key_off[key]);
    row[j] = static_cast<const uint8_t*>(a.oall[d]) + static_cast<size_t>(r) * H * eb;
    wt[j] = w[o];
  }
  for (int v = v0 + lane; v < v1; v += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (residual) {  // y = x + sum
      const uint4 r = *reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(residual) +
                                                      static_cast<size_t>(t) * H * eb + 16 * v);
      if (BF16) {
        unpack8(r, acc);
      } else {
        acc[0] = __uint_as_float(r.x); acc[1] = __uint_as_float(r.y);
        acc[2] = __uint_as_float(r.z); acc[3] = __uint_as_float(r.w);
      }
    }
    for (int j = 0; j < k; ++j) {
      const uint4 r = *reinterpret_cast<const uint4*>(row[j] + 16 * v);
      if (BF16) {
        float f[8];
        unpack8(r, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(wt[j], f[i], acc[i]);
      } else {
        acc[0] = fmaf(wt[j], __uint_as_float(r.x), acc[0]);
        acc[1] = fmaf(wt[j], __uint_as_float(r.y), acc[1]);
        acc[2] = fmaf(wt[j], __uint_as_float(r.z), acc[2]);
        acc[3] = fmaf(wt[j], __uint_as_float(r.w), acc[3]);
      }
    }
    uint8_t* out = static_cast<uint8_t*>(y) + (static_cast<size_t>(t) * H) * eb + 16 * v;
    if (BF16) st_v4(out, pack8(acc));
    else st_v4(out, make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]),
                               __float_as_uint(acc[3])));
  }
}

// ---------------------------------------------------------------- shared-expert refresh
// Deterministic cross-GPU shared mean, bit-exact with the reference's sequential fp64
// sum in expert order (sparsecomp.cpp:147-168): experts 0..E-1 live on ranks 0..G-1 in
// order, so the sum is a chain.  Rank g, chunk by chunk: wait for rank g-1's partial of
// the chunk (peer memory flag), continue the fp64 sum over its own experts, publish its
// partial (or, on the last rank, the fp32 mean).  Chunks pipeline across the chain.
// Entry barrier: every rank has finished the previous refresh (stream order), so no
// partial or mean of the previous epoch is still being read when this one overwrites it.
__global__ void chain_barrier_kernel(ChainArgs c) {
  const int r = threadIdx.x;
  if (r < c.G) st_release_sys(c.bar[r] + c.rank, c.epoch);
  __syncthreads();
  if (r < c.G) wait_flag(c.bar[c.rank] + r, c.epoch, (static_cast<uint32_t>(c.rank) << 16) | (20u << 8) | r, c.timeout_ns);
}

__global__ void __launch_bounds__(256) shared_chain_kernel(ChainArgs c) {
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * c.chunk;
  const int64_t i1 = min(c.P, i0 + c.chunk);
  if (c.rank > 0 && c.epoch) {
    if (threadIdx.x == 0)
      wait_flag(c.pred_flags + blockIdx.x, c.epoch, (static_cast<uint32_t>(c.rank) << 16) | (21u << 8), c.timeout_ns);
    __syncthreads();
  }
  const bool last = c.rank == c.G - 1;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double acc = c.rank > 0 ? __ldcv(c.pred_partial + i) : 0.0;
    for (int j = 0; j < c.n; ++j) acc = __dadd_rn(acc, static_cast<double>(c.master[static_cast<int64_t>(j) * c.P + i]));
    if (last) c.shared[i] = __double2float_rn(__dmul_rn(acc, c.inv));
    else c.partial[i] = acc;
  }
  if (!c.epoch) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(c.my_flags + blockIdx.x, c.epoch);
  }
}

// Ranks before the last: copy each chunk of the mean from the last rank once its flag
// is up.
__global__ void __launch_bounds__(256) shared_fetch_kernel(ChainArgs c) {
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * c.chunk;
  const int64_t i1 = min(c.P, i0 + c.chunk);
  if (threadIdx.x == 0)
    wait_flag(c.last_flags + blockIdx.x, c.epoch, (static_cast<uint32_t>(c.rank) << 16) | (22u << 8), c.timeout_ns);
  __syncthreads();
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) c.shared[i] = __ldcv(c.last_shared + i);
}

}  // namespace

const uint32_t* p2p_dispatch_flags(const P2PArgs& a) {
  return static_cast<const uint32_t*>(a.sync[a.rank]) + 1 * kMaxG;
}

size_t p2p_sync_bytes(int G, int E) {
  return kSyncSlots * kMaxG * sizeof(uint32_t) + 2 * kMaxG * static_cast<size_t>(G) * E * sizeof(int) + 256;
}

cudaError_t launch_count_exchange(const P2PArgs& a, const int* key_total, const int* key_off,
                                  const int* slot_of_expert, int* send_base, int* g_row_start, int* g_rows,
                                  int* g_slot, unsigned long long* g_out_down, int* g_wait, int* counts_out,
                                  cudaStream_t s) {
  if (a.G > kMaxG || a.E > kMaxE) return cudaErrorInvalidValue;
  count_exchange_kernel<<<1, 256, 0, s>>>(a, key_total, key_off, slot_of_expert, send_base, g_row_start, g_rows,
                                          g_slot, g_out_down, g_wait, counts_out);
  return cudaGetLastError();
}

cudaError_t launch_permute_p2p(const P2PArgs& a, DType dt, const void* x, int T, int H, int k, const int* keys,
                               const int* ranks, const int* chunk_off, const int* key_off, const int* send_base,
                               int* pos, cudaStream_t s, int mode) {
  const int row_bytes = H * dtype_bytes(dt);
  if (row_bytes % 16 || k > 8) return cudaErrorInvalidValue;
  if (T == 0) return cudaSuccess;  // empty batch: nothing to send
  static DeviceOnce carveout;
  if (!carveout.done()) {
    // Same L1/shared split as the persistent GEMM, so remote-row blocks can run on SMs
    // next to GEMM CTAs that wait for peers' rows (overlapped dispatch).
    const cudaError_t e = cudaFuncSetAttribute(permute_p2p_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    carveout.set();
  }
  const int seg = row_segments(T, row_bytes >> 4);
  int blocks = (T * seg + 7) / 8;
  if (mode == 2) {
    // HEP_DISPATCH_CTAS=n caps the remote pass's grid so the own-expert GEMM can launch
    // beside it.  Default uncapped: at N=4 a cap of 148 or 296 moved the dispatch time
    // into the GEMM without changing the step (profiles/r2_dispatch/).
    static const int cap = [] {
      const char* e = std::getenv("HEP_DISPATCH_CTAS");
      return e ? std::atoi(e) : 0;
    }();
    if (cap > 0) blocks = std::min(blocks, cap);
  }
  permute_p2p_kernel<<<blocks, 256, 0, s>>>(a, static_cast<const uint8_t*>(x), T, row_bytes, k, keys,
                                                       ranks, chunk_off, key_off, send_base, pos, mode, seg);
  return cudaGetLastError();
}

cudaError_t launch_shared_chain(const ChainArgs& c, cudaStream_t s) {
  const int blocks = static_cast<int>((c.P + c.chunk - 1) / c.chunk);
  if (c.epoch) chain_barrier_kernel<<<1, 32, 0, s>>>(c);
  shared_chain_kernel<<<blocks, 256, 0, s>>>(c);
  if (c.epoch && c.rank != c.G - 1) shared_fetch_kernel<<<blocks, 256, 0, s>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_signal_wait(const P2PArgs& a, int slot, cudaStream_t s, bool wait, bool ag_peers, bool sig) {
  signal_wait_kernel<<<1, 32, 0, s>>>(a, slot, wait ? 1 : 0, ag_peers ? 1 : 0, sig ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_combine_p2p(const P2PArgs& a, DType dt, const int* keys, const int* pos, const int* key_off,
                               const int* send_base, const float* w, int T, int H, int k, void* y,
                               cudaStream_t s, const void* residual) {
  if (k > 8) return cudaErrorInvalidValue;
  if (T == 0) return cudaSuccess;
  const int seg = row_segments(T, H * dtype_bytes(dt) / 16);
  if (dt == DType::BF16)
    combine_p2p_kernel<true><<<(T * seg + 7) / 8, 256, 0, s>>>(a, keys, pos, key_off, send_base, w, T, H, k, y, seg,
                                                                residual);
  else
    combine_p2p_kernel<false><<<(T * seg + 7) / 8, 256, 0, s>>>(a, keys, pos, key_off, send_base, w, T, H, k, y, seg,
                                                                 residual);
  return cudaGetLastError();
}


// Loads every kernel of this file now (see preload_kernels in kernels.h).
cudaError_t preload_comm_p2p_kernels() {
  auto load = [](const void* fn) {
    cudaFuncAttributes attr;
    return cudaFuncGetAttributes(&attr, fn);
  };
  if (const cudaError_t e = load(reinterpret_cast<const void*>(count_exchange_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(permute_p2p_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(signal_wait_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(combine_p2p_kernel<true>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(combine_p2p_kernel<false>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(chain_barrier_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(shared_chain_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(shared_fetch_kernel))) return e;
  return cudaSuccess;
}

}  // namespace hep
