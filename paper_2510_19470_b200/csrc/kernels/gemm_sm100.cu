// K8: expert FFN grouped GEMM on the 5th-gen tensor cores (sm_100a).
//
//   C[r, n] = act( sum_k A[r, k] * B[slot(g) * N + n, k] )   for rows r of group g
//
// A (tokens, bf16, K-major) and B (expert weights, bf16, stored K-major i.e. the
// compute copy w^T) are streamed by TMA into 128-byte-swizzled shared-memory
// stages; one elected thread issues tcgen05.mma (M=128, N=256, K=16) into a
// double-buffered fp32 accumulator in TMEM (2 x 256 columns); four epilogue warps
// drain TMEM with tcgen05.ld, apply ReLU, round to bf16 and store.  The kernel is
// persistent (one CTA per SM) and walks a device-side group table, so token
// counts per expert never have to reach the host.
//
// Warp roles (192 threads): w0 TMA producer, w1 TMEM owner + MMA issuer,
// w2..w5 epilogue (warp w drains TMEM lanes 32*(w%4) .. +31).

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace hep {

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int STAGES = 4;
constexpr int ACC = 2;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = ACC * BN;  // 512
constexpr int kMaxGroups = 512;
constexpr int kThreads = 192;
// Fused SR decode: converter warps (warps 6 ..) take the B stages round-robin, so the
// per-stage fixed latency (patch, proxy fence, barrier arrive) of one warp overlaps the
// others' and the converters keep pace with the tensor core.
constexpr int kConvWarps = 4;

struct SmemCtl {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t patched[STAGES];  // PATCH variant: the converter warp finished this stage
  uint64_t tfull[ACC];
  uint64_t tempty[ACC];
  uint32_t tmem_base;
  int num_tiles;
  int tile_start[kMaxGroups + 1];
  int row_start[kMaxGroups];
  int rows[kMaxGroups];
  int slot[kMaxGroups];
  __nv_bfloat16* out[kMaxGroups];  // output row 0 of the group (local or a peer GPU's HBM)
  int wait[kMaxGroups];            // source rank whose dispatch flag gates the group, or -1
};

constexpr size_t kSmemBytes = 1024 + STAGES * STAGE_BYTES + sizeof(SmemCtl);
constexpr size_t kSmemBytesPatch = kSmemBytes + STAGES * kPatchBlockBytes;  // + the staged patch blocks

__device__ __forceinline__ uint64_t make_policy(uint32_t p) {
  uint64_t pol;
  if (p == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else if (p == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Raster of a group's tiles (sched bits 4-5): 0 = m fastest, 1 = n fastest,
// 2 = super-rows of GM m-tiles (bits 8-15) with n fastest inside.
__device__ __forceinline__ void decode_tile(int local, int m_tiles, int n_tiles, uint32_t sched, int& mt,
                                            int& nt) {
  const uint32_t raster = (sched >> 4) & 3u;
  if (raster == 0) {
    mt = local % m_tiles;
    nt = local / m_tiles;
  } else if (raster == 1) {
    nt = local % n_tiles;
    mt = local / n_tiles;
  } else {
    const int gm = max(1, static_cast<int>((sched >> 8) & 0xffu));
    const int super = local / (gm * n_tiles);
    const int within = local - super * gm * n_tiles;
    const int rows = min(gm, m_tiles - super * gm);
    mt = super * gm + within % rows;
    nt = within / rows;
  }
}

// Spin (producer thread) until a peer's dispatch flag reaches `epoch`, then order the
// TMA (async proxy) reads of the rows that peer stored after its release.
__device__ __forceinline__ void wait_dispatch(const uint32_t* flag, uint32_t epoch, uint64_t timeout_ns) {
  uint32_t v;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (static_cast<int32_t>(v - epoch) >= 0) break;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (timeout_ns && t - t0 > timeout_ns) {
      printf("hep: GEMM dispatch wait timed out: epoch %u flag %u\n", epoch, v);
      __trap();
    }
    __nanosleep(100);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ int find_group(const SmemCtl& s, int ng, int tile) {
  int lo = 0, hi = ng - 1;  // largest g with tile_start[g] <= tile
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s.tile_start[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// PATCH = true: SR migration decode fused into the B-operand load (gathered experts).
// B is the SHARED expert's compute copy (one slot, map_b); a converter warp (warp 6) waits
// for each stage's TMA, writes the expert's residual-patched bf16 values into the
// 128-byte-swizzled B tile (precomputed by sr_patch_index: bf16((float)((double)shared +
// r)), the dense decode's exact values), fences them into the async proxy and releases
// the stage to the MMA issuer -- so the decode never materialises a dense expert copy.
template <bool PATCH>
__global__ void __launch_bounds__(kThreads + (PATCH ? 32 * kConvWarps : 0), 1)
grouped_gemm_bf16_kernel(const __grid_constant__ CUtensorMap map_a,
                         const __grid_constant__ CUtensorMap map_b, __nv_bfloat16* __restrict__ C,
                         int ldc, int N, int K, const int* __restrict__ g_row_start,
                         const int* __restrict__ g_rows, const int* __restrict__ g_slot,
                         const unsigned long long* __restrict__ g_out, const int* __restrict__ g_wait,
                         const uint32_t* __restrict__ wait_flags, uint32_t epoch, int ng, int relu,
                         uint32_t sched, uint64_t timeout_ns, const PatchArgs patches, int half) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* stage_a = smem;
  uint8_t* stage_b = smem + STAGES * A_BYTES;
  uint8_t* stage_p = smem + STAGES * STAGE_BYTES;  // PATCH: one patch block per stage
  SmemCtl& s = *reinterpret_cast<SmemCtl*>(smem + STAGES * STAGE_BYTES + (PATCH ? STAGES * kPatchBlockBytes : 0));

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int n_tiles = (N + BN - 1) / BN;
  const int num_kb = K / BK;

  // ---- group table -> tile prefix (warp 2), barriers (warp 0), TMEM (warp 1)
  if (warp == 2) {
    int carry = 0;
    for (int base = 0; base < ng; base += 32) {
      const int g = base + lane;
      int tiles = 0;
      if (g < ng) {
        const int r = g_rows[g];
        s.row_start[g] = g_row_start[g];
        s.rows[g] = r;
        s.slot[g] = g_slot[g];
        s.out[g] = g_out ? reinterpret_cast<__nv_bfloat16*>(g_out[g])
                         : C + static_cast<size_t>(g_row_start[g]) * ldc;
        s.wait[g] = g_wait ? g_wait[g] : -1;
        tiles = ((r + BM - 1) / BM) * n_tiles;
      }
      int incl = tiles;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (g < ng) s.tile_start[g] = carry + incl - tiles;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      s.tile_start[ng] = carry;
      s.num_tiles = carry;
    }
  } else if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
      mbar_init(&s.patched[i], 1);
    }
    for (int i = 0; i < ACC; ++i) {
      mbar_init(&s.tfull[i], 1);
      mbar_init(&s.tempty[i], 4);
    }
    fence_barrier_init();
  } else if (warp == 1) {
    tmem_alloc(&s.tmem_base, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const int total = s.num_tiles;
  const uint32_t tmem_base = s.tmem_base;

  if (PATCH && warp >= 6) {
    // ================= converters (fused SR decode) =================
    const int wi = static_cast<int>(warp) - 6;
    int c = 0;  // global stage counter: stage c % STAGES, phase (c / STAGES) & 1
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int g = find_group(s, ng, tile);
      const int local = tile - s.tile_start[g];
      const int m_tiles = (s.rows[g] + BM - 1) / BM;
      int mt, nt;
      decode_tile(local, m_tiles, n_tiles, sched, mt, nt);
      const int slot = s.slot[g];
      for (int kb = 0; kb < num_kb; ++kb, ++c) {
        if (c % kConvWarps != wi) continue;
        const int stage = c % STAGES;
        mbar_wait(&s.full[stage], (c / STAGES) & 1);
        {  // (a rejected wire's partial patch set is memory-safe; the layer raises the error)
          uint8_t* bst = stage_b + stage * B_BYTES;
          const uint32_t* blk = reinterpret_cast<const uint32_t*>(stage_p + stage * kPatchBlockBytes);
          const int cnt = static_cast<int>(blk[0]);
          const int n = min(cnt, kPatchBlockCap);
          for (int j = lane; j < n; j += 32) {
            const uint32_t w = blk[4 + j];
            *reinterpret_cast<uint16_t*>(bst + ((w >> 16) << 1)) = static_cast<uint16_t>(w & 0xffffu);
          }
          if (cnt > kPatchBlockCap) {  // overflowed block: the rest from the global list (rare)
            const uint32_t id = static_cast<uint32_t>(nt * num_kb + kb) | (static_cast<uint32_t>(half) << 31);
            const PatchRef& pr = patches.patches[slot];
            const int no = *pr.ovf_count;
            for (int q = lane; q < no; q += 32) {
              const uint2 e = pr.ovf[q];
              if (e.x == id) *reinterpret_cast<uint16_t*>(bst + ((e.y >> 16) << 1)) = static_cast<uint16_t>(e.y & 0xffffu);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.patched[stage]);
      }
    }
  }

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      const uint64_t pol_a = make_policy(sched & 3u);
      const uint64_t pol_b = make_policy((sched >> 2) & 3u);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int g = find_group(s, ng, tile);
        const int local = tile - s.tile_start[g];
        const int m_tiles = (s.rows[g] + BM - 1) / BM;
        int mt, nt;
        decode_tile(local, m_tiles, n_tiles, sched, mt, nt);
        const int a_row = s.row_start[g] + mt * BM;
        const int b_row = (PATCH ? 0 : s.slot[g] * N) + nt * BN;  // PATCH: the shared expert
        const uint8_t* pblk = PATCH ? patches.base + static_cast<size_t>(s.slot[g]) * patches.slot_bytes +
                                          patches.half_bytes + static_cast<size_t>(nt) * num_kb * kPatchBlockBytes
                                    : nullptr;
        if (s.wait[g] >= 0) wait_dispatch(wait_flags + s.wait[g], epoch, timeout_ns);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&s.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&s.full[stage], STAGE_BYTES + (PATCH ? kPatchBlockBytes : 0));
          tma_load_2d(stage_a + stage * A_BYTES, &map_a, &s.full[stage], kb * BK, a_row, pol_a);
          tma_load_2d(stage_b + stage * B_BYTES, &map_b, &s.full[stage], kb * BK, b_row, pol_b);
          if (PATCH)
            bulk_load(stage_p + stage * kPatchBlockBytes, pblk + static_cast<size_t>(kb) * kPatchBlockBytes,
                      kPatchBlockBytes, &s.full[stage], pol_b);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(PATCH ? &s.patched[stage] : &s.full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_addr(stage_a + stage * A_BYTES);
          const uint32_t b_addr = smem_addr(stage_b + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_bf16(d_tmem, umma_desc_k_sw128(a_addr + 32 * k), umma_desc_k_sw128(b_addr + 32 * k),
                      idesc, (kb | k) != 0);
          }
          umma_commit(&s.empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&s.tfull[acc]);
        if (++acc == ACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // ================= epilogue (warps 2..5) =================
    const uint32_t quarter = warp & 3u;  // TMEM lane quarter this warp may access
    const int row_in_tile = static_cast<int>(quarter * 32 + lane);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int g = find_group(s, ng, tile);
      const int local = tile - s.tile_start[g];
      const int m_tiles = (s.rows[g] + BM - 1) / BM;
      int mt, nt;
      decode_tile(local, m_tiles, n_tiles, sched, mt, nt);
      const int r_local = mt * BM + row_in_tile;
      const bool row_ok = r_local < s.rows[g];
      __nv_bfloat16* crow = s.out[g] + static_cast<size_t>(r_local) * ldc + nt * BN;

      mbar_wait(&s.tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_base = tmem_base + static_cast<uint32_t>(acc * BN) + ((quarter * 32u) << 16);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        if (nt * BN + c >= N) break;  // warp-uniform
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_base + static_cast<uint32_t>(c), v);
        tmem_ld_wait();
        if (row_ok) {
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = __uint_as_float(v[i]);
            f[i] = relu ? fmaxf(x, 0.f) : x;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) st_v4(crow + c + 8 * q, pack8(f + 8 * q));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.tempty[acc]);
      if (++acc == ACC) { acc = 0; acc_phase ^= 1; }
    }
    if (g_out) __threadfence_system();  // outputs may live in a peer GPU's HBM
  }

  __syncwarp();  // reconverge the single-lane roles before the CTA barrier
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ============================================================================
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 256 tile.  CTA r stages rows [128r, 128r+128) of the A tile and of the B tile
// (N half) in its own shared memory; the leader (rank 0) issues one
// tcgen05.mma.cta_group::2 M=256 N=256 K=16 that reads both CTAs' halves and writes
// each CTA's 128 accumulator rows into that CTA's TMEM.  Per SM this halves the B
// bytes staged and read per FLOP (32 KB per 64-deep k-step instead of 48 KB), which is
// what lets the tensor pipe stay fed; both CTAs' TMA loads complete on the leader's
// full barrier, the leader's commits multicast to both CTAs' empty/tfull barriers,
// and both epilogues release the accumulator on the leader's tempty barrier.
constexpr int P_BM = 256;          // rows per cluster tile (128 per CTA)
constexpr int P_BN = 256;
constexpr int P_STAGES = 5;
constexpr int P_STAGES_PATCH = 6;  // fused decode: the converter's latency needs one more stage in flight
constexpr int P_STAGES_MAX = 6;
// Epilogue staging: each epilogue warp assembles its 32 rows x 128 bf16 columns (half a
// tile, twice per tile) in shared memory so global (and NVLink peer) stores go out as
// whole 256-byte row segments instead of scattered 16-byte pieces; the half-width
// buffer leaves room for a fifth operand stage.
constexpr int P_STG_COLS = P_BN / 2;
constexpr int P_STG_PITCH = P_STG_COLS * 2 + 16;        // bytes per staged row (+16 B pad)
constexpr int P_STG_BYTES = 4 * 32 * P_STG_PITCH;       // 4 epilogue warps
constexpr int P_A_BYTES = 128 * BK * 2;
constexpr int P_B_BYTES = 128 * BK * 2;
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;

struct SmemCtl2 {
  uint64_t full[P_STAGES_MAX];
  uint64_t empty[P_STAGES_MAX];
  uint64_t bfull[P_STAGES_MAX];    // PATCH: this CTA's B half + patch block landed (local)
  uint64_t patched[P_STAGES_MAX];  // PATCH (leader): both CTAs' B halves patched
  uint64_t tfull[ACC];
  uint64_t tempty[ACC];
  uint64_t tq_full[4];   // DYN: tile queue slot published (both CTAs)
  uint64_t tq_empty[4];  // DYN (leader): every consumer of both CTAs has read the slot
  int tile_q[4];
  uint32_t tmem_base;
  int num_tiles;
  int tile_start[kMaxGroups + 1];
  int row_start[kMaxGroups];
  int rows[kMaxGroups];
  int slot[kMaxGroups];
  __nv_bfloat16* out[kMaxGroups];
  int wait[kMaxGroups];
};
constexpr int kTileQ = 4;
constexpr int kTileQConsumers = 1 + 1 + 8;  // peer producer, MMA issuer, 4 epilogue warps x 2 CTAs

// Cluster-scope tile-queue primitives (dynamic tile scheduler).
__device__ __forceinline__ uint32_t peer_smem_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

constexpr size_t kSmemBytes2 = 1024 + P_STAGES * P_STAGE_BYTES + P_STG_BYTES + sizeof(SmemCtl2);
// PATCH: six operand stages + patch blocks, no epilogue staging buffer (direct stores)
constexpr size_t kSmemBytes2Patch =
    1024 + P_STAGES_PATCH * (P_STAGE_BYTES + kPatchBlockBytes) + sizeof(SmemCtl2);
constexpr size_t kSmemBytes2Deep = 1024 + P_STAGES_PATCH * P_STAGE_BYTES + sizeof(SmemCtl2);
constexpr size_t kSmemBytes2Four = 1024 + 4 * P_STAGE_BYTES + P_STG_BYTES + sizeof(SmemCtl2);

// Release-arrive at cluster scope on the leader CTA's copy of `bar`: orders this thread's
// (fenced) shared-memory writes before the leader's acquire of the barrier.
__device__ __forceinline__ void mbar_arrive_leader_cluster(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_smem_addr(bar)) : "memory");
}

__device__ __forceinline__ int find_group2(const SmemCtl2& s, int ng, int tile) {
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s.tile_start[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// PATCH = true: the fused SR decode on the CTA pair.  B is the shared expert; each CTA's
// B half and the stage's patch block land on a LOCAL barrier (bfull), the CTA's converter
// warp (warp 6) writes the entries that fall in its half, fences them into the async
// proxy and release-arrives on the leader's `patched` barrier (count 2); the leader's MMA
// waits for the A halves (full) and for both patched halves.
// NST operand stages; DIRECT: direct-store epilogue (no staging buffer).  The default is 5
// stages + staged epilogue: measured under ncu on the cfg3 down-projection, a sixth stage
// lets the CTAs drift apart, their L2 sharing drops (DRAM reads 5.1 -> 7.0 GB), the SM
// clock falls under the power cap (1.38 -> 1.31 GHz) and the launch slows 4%
// (profiles/r2_gemm_power.md).
// DYN: dynamic tile scheduler.  Instead of the static round-robin (tile = cluster +
// i * clusters), the leader's producer takes the next tile from a global counter and
// publishes it to a 4-slot queue in both CTAs' shared memory; every role of both CTAs
// reads its tiles from that queue.  Clusters that run ahead take the next tiles, so the
// tiles in flight stay a compact window of the raster and keep sharing L2 lines.
// GATHER: the permute fused into the A load.  Grouped row p of A is row a_src[p] of the
// layer input a_x (row stride K).  Gather warps 6..9 of each CTA copy their 128 rows per
// stage with 16-byte cp.async (8 lanes per 128-byte row segment, the SW128 swizzle
// computed in software), keep GATHER_LAG stages in flight, and publish each landed stage
// to the leader's full barrier after a proxy fence.  The TMA producer loads only B.
// Opt-in: this version and a tile::gather4 TMA version both ran the cfg3 up-projection
// 2.8x slower than the explicit permute (profiles/r2_gather.md).
constexpr int GATHER_LAG = 3;
template <bool PATCH, int NST_T = P_STAGES, bool DIRECT_T = false, bool DYN = false, bool GATHER = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads + ((PATCH || GATHER) ? 32 * kConvWarps : 0), 1)
grouped_gemm_bf16_2cta_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                              __nv_bfloat16* __restrict__ C, int ldc, int N, int K,
                              const int* __restrict__ g_row_start, const int* __restrict__ g_rows,
                              const int* __restrict__ g_slot, const unsigned long long* __restrict__ g_out,
                              const int* __restrict__ g_wait, const uint32_t* __restrict__ wait_flags,
                              uint32_t epoch, int ng, int relu, uint32_t sched, uint64_t timeout_ns,
                              const PatchArgs patches, int half, int* __restrict__ tile_counter,
                              const int* __restrict__ a_src, const __nv_bfloat16* __restrict__ a_x) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  constexpr bool DIRECT = PATCH || DIRECT_T;  // direct-store epilogue, no staging buffer
  constexpr int NST = PATCH ? P_STAGES_PATCH : NST_T;
  uint8_t* stage_a = smem;
  uint8_t* stage_b = smem + NST * P_A_BYTES;
  uint8_t* stage_out = smem + NST * P_STAGE_BYTES;  // !DIRECT: epilogue staging
  uint8_t* stage_p = smem + NST * P_STAGE_BYTES;    // PATCH: one patch block per stage
  SmemCtl2& s = *reinterpret_cast<SmemCtl2*>(smem + NST * P_STAGE_BYTES +
                                             (PATCH ? NST * kPatchBlockBytes : (DIRECT ? 0 : P_STG_BYTES)));

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t cta = cluster_ctarank();
  const int cluster = static_cast<int>(blockIdx.x >> 1), nclusters = static_cast<int>(gridDim.x >> 1);
  const int n_tiles = (N + P_BN - 1) / P_BN;
  const int num_kb = K / BK;

  if (warp == 2) {
    int carry = 0;
    for (int base = 0; base < ng; base += 32) {
      const int g = base + lane;
      int tiles = 0;
      if (g < ng) {
        const int r = g_rows[g];
        s.row_start[g] = g_row_start[g];
        s.rows[g] = r;
        s.slot[g] = g_slot[g];
        s.out[g] = g_out ? reinterpret_cast<__nv_bfloat16*>(g_out[g])
                         : C + static_cast<size_t>(g_row_start[g]) * ldc;
        s.wait[g] = g_wait ? g_wait[g] : -1;
        tiles = ((r + P_BM - 1) / P_BM) * n_tiles;
      }
      int incl = tiles;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (g < ng) s.tile_start[g] = carry + incl - tiles;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      s.tile_start[ng] = carry;
      s.num_tiles = carry;
    }
  } else if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&s.full[i], GATHER ? 1 + 2 * kConvWarps : 1);  // GATHER: + every gather warp of both CTAs
      mbar_init(&s.empty[i], 1);
      mbar_init(&s.bfull[i], 1);
      mbar_init(&s.patched[i], 2);  // one converter per CTA
    }
    for (int i = 0; i < kTileQ; ++i) {
      mbar_init(&s.tq_full[i], 1);
      mbar_init(&s.tq_empty[i], kTileQConsumers);
    }
    for (int i = 0; i < ACC; ++i) {
      mbar_init(&s.tfull[i], 1);
      mbar_init(&s.tempty[i], 8);  // 4 epilogue warps x 2 CTAs (used in the leader)
    }
    fence_barrier_init();
  } else if (warp == 1) {
    tmem_alloc_2sm(&s.tmem_base, TMEM_COLS);
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();

  const int total = s.num_tiles;
  const uint32_t tmem_base = s.tmem_base;
  // The tile sequence of this cluster: static round-robin, or (DYN) the shared queue.
  // i counts this role's tiles; returns -1 when the cluster has no more.
  int prefetched = -2;  // DYN publisher: the next tile id, fetched one tile ahead
  auto next_tile = [&](int& i, bool publisher) -> int {
    if (!DYN) {
      const int t = cluster + i * nclusters;
      ++i;
      return t < total ? t : -1;
    }
    const int q = i % kTileQ;
    const uint32_t ph = static_cast<uint32_t>(i / kTileQ) & 1u;
    ++i;
    if (publisher) {  // leader producer: take the next tile, publish it to both CTAs
      if (prefetched == -2) prefetched = atomicAdd(tile_counter, 1);
      int t = prefetched;
      if (t >= total) t = -1;
      // the following tile's id is fetched now, so the atomic's round trip overlaps this tile
      if (t >= 0) prefetched = atomicAdd(tile_counter, 1);
      mbar_wait(&s.tq_empty[q], ph ^ 1u);
      s.tile_q[q] = t;
      st_cluster_u32(peer_smem_addr(&s.tile_q[q], 1), t);
      mbar_arrive_remote(peer_smem_addr(&s.tq_full[q], 0));
      mbar_arrive_remote(peer_smem_addr(&s.tq_full[q], 1));
      return t;
    }
    mbar_wait_cluster(&s.tq_full[q], ph);
    const int t = *reinterpret_cast<volatile int*>(&s.tile_q[q]);
    return t;
  };
  // a consumer has read slot (i - 1): release it to the publisher (one arrival per role)
  auto release_tile = [&](int i) {
    if (DYN) mbar_arrive_remote(peer_smem_addr(&s.tq_empty[(i - 1) % kTileQ], 0));
  };

  if (PATCH && warp >= 6) {
    // ================= converters (fused SR decode), both CTAs =================
    const int wi = static_cast<int>(warp) - 6;
    int c = 0;  // global stage counter: stage c % NST, phase (c / NST) & 1
    for (int tile = cluster; tile < total; tile += nclusters) {
      const int g = find_group2(s, ng, tile);
      const int m_tiles = (s.rows[g] + P_BM - 1) / P_BM;
      int mt, nt;
      decode_tile(tile - s.tile_start[g], m_tiles, n_tiles, sched, mt, nt);
      const int slot = s.slot[g];
      // rows of the 256-row B tile held here: [split * cta, split * cta + split)
      const int split = N - nt * P_BN <= P_BN / 2 ? 64 : 128;
      const uint32_t lo_byte = static_cast<uint32_t>(split * 128) * cta, hi_byte = lo_byte + split * 128;
      for (int kb = 0; kb < num_kb; ++kb, ++c) {
        if (c % kConvWarps != wi) continue;
        const int stage = c % NST;
        mbar_wait(&s.bfull[stage], (c / NST) & 1);
        {  // (a rejected wire's partial patch set is memory-safe; the layer raises the error)
          uint8_t* bst = stage_b + stage * P_B_BYTES;
          const uint32_t* blk = reinterpret_cast<const uint32_t*>(stage_p + stage * kPatchBlockBytes);
          const int cnt = static_cast<int>(blk[0]);
          const int n = min(cnt, kPatchBlockCap);
          for (int j = lane; j < n; j += 32) {
            const uint32_t w = blk[4 + j];
            const uint32_t off = (w >> 16) << 1;  // byte in the 256-row swizzled tile
            if (off >= lo_byte && off < hi_byte)
              *reinterpret_cast<uint16_t*>(bst + (off - lo_byte)) = static_cast<uint16_t>(w & 0xffffu);
          }
          if (cnt > kPatchBlockCap) {  // overflowed block: the rest from the global list (rare)
            const uint32_t id = static_cast<uint32_t>(nt * num_kb + kb) | (static_cast<uint32_t>(half) << 31);
            const PatchRef& pr = patches.patches[slot];
            const int no = *pr.ovf_count;
            for (int q = lane; q < no; q += 32) {
              const uint2 e = pr.ovf[q];
              const uint32_t off = (e.y >> 16) << 1;
              if (e.x == id && off >= lo_byte && off < hi_byte)
                *reinterpret_cast<uint16_t*>(bst + (off - lo_byte)) = static_cast<uint16_t>(e.y & 0xffffu);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) {
          if (cta == 0) mbar_arrive(&s.patched[stage]);  // own smem: CTA-scope release suffices
          else mbar_arrive_leader_cluster(&s.patched[stage]);
        }
      }
    }
  }

  if (GATHER && warp >= 6) {
    // ================= A gather warps (both CTAs) =================
    const int wi = static_cast<int>(warp) - 6;
    const int sub = static_cast<int>(lane >> 3), chunk = static_cast<int>(lane & 7);
    const size_t row_bytes = static_cast<size_t>(K) * sizeof(__nv_bfloat16);
    const uint8_t* xb = reinterpret_cast<const uint8_t*>(a_x) + chunk * 16;
    int stage = 0, issued = 0;
    uint32_t phase = 0;
    auto publish = [&](int st) {  // every cp.async of stage st has landed (wait_group)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (cta == 0) mbar_arrive(&s.full[st]);
        else mbar_arrive_leader_cluster(&s.full[st]);
      }
    };
    for (int tile = cluster; tile < total; tile += nclusters) {
      const int g = find_group2(s, ng, tile);
      const int m_tiles = (s.rows[g] + P_BM - 1) / P_BM;
      int mt, nt;
      decode_tile(tile - s.tile_start[g], m_tiles, n_tiles, sched, mt, nt);
      // this lane's 8 rows of the CTA's 128-row half: wi*32 + i*4 + sub (a_src is padded
      // with valid token ids past the last group, so a partial m-tile reads defined rows)
      const int r0 = s.row_start[g] + mt * P_BM + 128 * static_cast<int>(cta) + wi * 32 + sub;
      const uint8_t* src[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) src[i] = xb + static_cast<size_t>(a_src[r0 + 4 * i]) * row_bytes;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&s.empty[stage], phase ^ 1);
        const uint32_t base = smem_addr(stage_a + stage * P_A_BYTES);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = wi * 32 + 4 * i + sub;
          const uint32_t dst = base + static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src[i] + kb * 128) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (++issued > GATHER_LAG) {
          asm volatile("cp.async.wait_group %0;" ::"n"(GATHER_LAG) : "memory");
          publish((stage + NST - GATHER_LAG) % NST);
        }
        if (++stage == NST) { stage = 0; phase ^= 1; }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (int j = min(issued, GATHER_LAG); j > 0; --j) publish((stage + NST - j) % NST);
  } else if (warp == 0) {
    // ================= TMA producer (both CTAs) =================
    if (lane == 0) {
      const uint64_t pol_a = make_policy(sched & 3u);
      const uint64_t pol_b = make_policy((sched >> 2) & 3u);
      int stage = 0;
      uint32_t phase = 0;
      int ti = 0;
      for (int tile = next_tile(ti, cta == 0); tile >= 0; tile = next_tile(ti, cta == 0)) {
        if (cta != 0) release_tile(ti);
        const int g = find_group2(s, ng, tile);
        const int local = tile - s.tile_start[g];
        const int m_tiles = (s.rows[g] + P_BM - 1) / P_BM;
        int mt, nt;
        decode_tile(local, m_tiles, n_tiles, sched, mt, nt);
        const int a_row = s.row_start[g] + mt * P_BM + 128 * static_cast<int>(cta);
        // a tail n-tile of <= 128 columns runs as an N=128 MMA: each CTA supplies 64 B rows
        // (the first 64 of its 128-row box)
        const int b_half = N - nt * P_BN <= P_BN / 2 ? 64 : 128;
        const int b_row = (PATCH ? 0 : s.slot[g] * N) + nt * P_BN + b_half * static_cast<int>(cta);
        const uint8_t* pblk = PATCH ? patches.base + static_cast<size_t>(s.slot[g]) * patches.slot_bytes +
                                          patches.half_bytes + static_cast<size_t>(nt) * num_kb * kPatchBlockBytes
                                    : nullptr;
        if (s.wait[g] >= 0) wait_dispatch(wait_flags + s.wait[g], epoch, timeout_ns);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&s.empty[stage], phase ^ 1);
          if (PATCH) {
            // A halves on the leader's barrier; this CTA's B half + patch block on its own
            if (cta == 0) mbar_arrive_expect_tx(&s.full[stage], 2 * P_A_BYTES);
            mbar_arrive_expect_tx(&s.bfull[stage], P_B_BYTES + kPatchBlockBytes);
            tma_load_2d_2sm(stage_a + stage * P_A_BYTES, &map_a, &s.full[stage], kb * BK, a_row, pol_a);
            tma_load_2d(stage_b + stage * P_B_BYTES, &map_b, &s.bfull[stage], kb * BK, b_row, pol_b);
            bulk_load(stage_p + stage * kPatchBlockBytes, pblk + static_cast<size_t>(kb) * kPatchBlockBytes,
                      kPatchBlockBytes, &s.bfull[stage], pol_b);
          } else {
            if (cta == 0) mbar_arrive_expect_tx(&s.full[stage], GATHER ? 2 * P_B_BYTES : 2 * P_STAGE_BYTES);
            if (!GATHER) tma_load_2d_2sm(stage_a + stage * P_A_BYTES, &map_a, &s.full[stage], kb * BK, a_row, pol_a);
            tma_load_2d_2sm(stage_b + stage * P_B_BYTES, &map_b, &s.full[stage], kb * BK, b_row, pol_b);
          }
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA only) =================
    if (cta == 0 && lane == 0) {
      constexpr uint32_t idesc_full = umma_idesc_bf16(P_BM, P_BN);
      constexpr uint32_t idesc_half = umma_idesc_bf16(P_BM, P_BN / 2);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int ti = 0;
      for (int tile = next_tile(ti, false); tile >= 0; tile = next_tile(ti, false)) {
        release_tile(ti);
        const int g = find_group2(s, ng, tile);
        const int m_tiles = (s.rows[g] + P_BM - 1) / P_BM;
        int mt, nt;
        decode_tile(tile - s.tile_start[g], m_tiles, n_tiles, sched, mt, nt);
        const uint32_t idesc = N - nt * P_BN <= P_BN / 2 ? idesc_half : idesc_full;
        mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * P_BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&s.full[stage], phase);
          if (PATCH) mbar_wait(&s.patched[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_addr(stage_a + stage * P_A_BYTES);
          const uint32_t b_addr = smem_addr(stage_b + stage * P_B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_2sm(d_tmem, umma_desc_k_sw128(a_addr + 32 * k), umma_desc_k_sw128(b_addr + 32 * k), idesc,
                          (kb | k) != 0);
          umma_commit_2sm_mc(&s.empty[stage], 0x3);
          if (++stage == NST) { stage = 0; phase ^= 1; }
        }
        umma_commit_2sm_mc(&s.tfull[acc], 0x3);
        if (++acc == ACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // ================= epilogue (warps 2..5, both CTAs) =================
    const uint32_t quarter = warp & 3u;
    uint8_t* stg = stage_out + quarter * 32 * P_STG_PITCH;  // this warp's 32 staged rows
    int acc = 0;
    uint32_t acc_phase = 0;
    int ti = 0;
    for (int tile = next_tile(ti, false); tile >= 0; tile = next_tile(ti, false)) {
      __syncwarp();
      if (lane == 0) release_tile(ti);
      const int g = find_group2(s, ng, tile);
      const int local = tile - s.tile_start[g];
      const int m_tiles = (s.rows[g] + P_BM - 1) / P_BM;
      int mt, nt;
      decode_tile(local, m_tiles, n_tiles, sched, mt, nt);
      const int row0 = mt * P_BM + static_cast<int>(128 * cta + quarter * 32);  // first row of this warp
      const int ncols = min(P_BN, N - nt * P_BN);

      mbar_wait(&s.tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_base = tmem_base + static_cast<uint32_t>(acc * P_BN) + ((quarter * 32u) << 16);
      const int rows_here = min(32, s.rows[g] - row0);
      __nv_bfloat16* out0 = s.out[g] + static_cast<size_t>(row0) * ldc + nt * P_BN;
      if constexpr (DIRECT) {
        // direct stores, one row per lane (the staging buffer's space holds a sixth stage)
#pragma unroll 1
        for (int c = 0; c < ncols; c += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_base + static_cast<uint32_t>(c), v);
          tmem_ld_wait();
          if (static_cast<int>(lane) < rows_here) {  // signed: rows_here < 0 past a group's end
            float f[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float x = __uint_as_float(v[i]);
              f[i] = relu ? fmaxf(x, 0.f) : x;
            }
            __nv_bfloat16* crow = out0 + static_cast<size_t>(lane) * ldc + c;
#pragma unroll
            for (int q = 0; q < 4; ++q) st_v4(crow + 8 * q, pack8(f + 8 * q));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&s.tempty[acc]);
      } else {
        // two column halves: TMEM -> registers -> (relu, bf16) -> staged row `lane` -> global
#pragma unroll 1
        for (int h = 0; h < P_BN; h += P_STG_COLS) {
          const int hcols = min(P_STG_COLS, ncols - h);
          if (hcols <= 0) break;  // warp-uniform
#pragma unroll 1
          for (int c = 0; c < hcols; c += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_base + static_cast<uint32_t>(h + c), v);
            tmem_ld_wait();
            float f[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float x = __uint_as_float(v[i]);
              f[i] = relu ? fmaxf(x, 0.f) : x;
            }
            uint4* dst = reinterpret_cast<uint4*>(stg + lane * P_STG_PITCH + c * 2);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = pack8(f + 8 * q);
          }
          if (h + P_STG_COLS >= ncols) {
            // the accumulator is free as soon as its last columns have been read
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&s.tempty[acc]);
          }
          __syncwarp();
          // staged rows -> global, one row per instruction: lane l writes bytes [16l, 16l+16)
          const int row_bytes = hcols * 2;
          for (int r = 0; r < rows_here; ++r) {
            if (lane * 16 < row_bytes) {
              const uint4 val = *reinterpret_cast<const uint4*>(stg + r * P_STG_PITCH + lane * 16);
              st_v4(reinterpret_cast<uint8_t*>(out0 + static_cast<size_t>(r) * ldc + h) + lane * 16, val);
            }
          }
          __syncwarp();  // the staging buffer is rewritten next
        }
      }
      if (++acc == ACC) { acc = 0; acc_phase ^= 1; }
    }
    if (g_out) __threadfence_system();  // outputs may live in a peer GPU's HBM
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, TMEM_COLS);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}


// ============================================================================
// fp32 layers (cfg1/cfg2): the same persistent 1-CTA structure on kind::tf32 with the
// 3xTF32 split.  Every fp32 operand x is carried as x_hi = rna_tf32(x) and
// x_lo = rna_tf32(x - x_hi); D += A_lo*B_hi + A_hi*B_lo + A_hi*B_hi in fp32 TMEM
// accumulators drops only the lo*lo term (~2^-22 relative per product), so the result
// meets the fp32 1e-4 bound that single TF32 (10-bit mantissa) cannot, at tensor-core
// rates.  A stage holds 32 fp32 of K (one 128-byte swizzle row) for A_hi, A_lo, B_hi,
// B_lo: 16 + 16 + 32 + 32 KB, two stages.  Epilogue: fp32 rows, or (split mode) the
// ReLU'd rows already split into hi/lo for the next GEMM.
constexpr int T_BK = kTf32BK;
constexpr int T_STAGES = T_BK == 32 ? 2 : 4;
constexpr int T_A_BYTES = BM * T_BK * 4;
constexpr int T_B_BYTES = BN * T_BK * 4;
constexpr int T_STAGE_BYTES = 2 * T_A_BYTES + 2 * T_B_BYTES;

struct SmemCtlT {
  uint64_t full[T_STAGES];
  uint64_t empty[T_STAGES];
  uint64_t conv[T_STAGES];  // BRAW: the converter warps split this stage's B into hi/lo
  uint64_t tfull[ACC];
  uint64_t tempty[ACC];
  uint32_t tmem_base;
  int num_tiles;
  int tile_start[kMaxGroups + 1];
  int row_start[kMaxGroups];
  int rows[kMaxGroups];
  int slot[kMaxGroups];
};
constexpr size_t kSmemBytesT = 1024 + T_STAGES * T_STAGE_BYTES + sizeof(SmemCtlT);

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
  return (1u << 4)                                   // D format fp32
         | (2u << 7)                                 // A format tf32
         | (2u << 10)                                // B format tf32
         | (static_cast<uint32_t>(N >> 3) << 17)     // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);    // M / 16
}

// K-major descriptor of a stage operand: 128-byte rows (BK=32, SW128) or 64-byte rows
// (BK=16, SW64)
__device__ __forceinline__ uint64_t t_desc(uint32_t addr) {
  return T_BK == 32 ? umma_desc_k_sw128(addr) : umma_desc_k_sw64(addr);
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// BRAW: B arrives as raw fp32 (one TMA box per stage, half the HBM bytes of pre-split
// hi/lo weights); converter warps 6..9 split it in shared memory, hi in place and lo
// into the B_lo slot, with the same rna_tf32 split as split_tf32_kernel (bit-identical
// products).  The MMA issuer waits on conv[] instead of full[].  Opt-in
// (HEP_TF32_RAWB=1): it halves the kernel's DRAM reads but not its time, which is not
// bound by HBM (profiles/r2_tf32_tiled.md).
template <bool BRAW>
__global__ void __launch_bounds__(kThreads + (BRAW ? 32 * kConvWarps : 0), 1)
grouped_gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap map_a_hi, const __grid_constant__ CUtensorMap map_a_lo,
                           const __grid_constant__ CUtensorMap map_b_hi, const __grid_constant__ CUtensorMap map_b_lo,
                           float* __restrict__ C, float* __restrict__ C_lo, int ldc, int N, int K,
                           const int* __restrict__ g_row_start, const int* __restrict__ g_rows,
                           const int* __restrict__ g_slot, int ng, int relu, int ksplit, size_t split_stride) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  SmemCtlT& s = *reinterpret_cast<SmemCtlT*>(smem + T_STAGES * T_STAGE_BYTES);
  auto a_hi_at = [&](int st) { return smem + st * T_STAGE_BYTES; };
  auto a_lo_at = [&](int st) { return smem + st * T_STAGE_BYTES + T_A_BYTES; };
  auto b_hi_at = [&](int st) { return smem + st * T_STAGE_BYTES + 2 * T_A_BYTES; };
  auto b_lo_at = [&](int st) { return smem + st * T_STAGE_BYTES + 2 * T_A_BYTES + T_B_BYTES; };

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int n_tiles = (N + BN - 1) / BN;
  // split-K (ksplit > 1): tile t covers K-part t % ksplit and stores raw fp32 partials
  // at C + part * split_stride; a reduce kernel sums the parts in order
  const int num_kb = K / T_BK / ksplit;

  if (warp == 2) {
    int carry = 0;
    for (int base = 0; base < ng; base += 32) {
      const int g = base + lane;
      int tiles = 0;
      if (g < ng) {
        const int r = g_rows[g];
        s.row_start[g] = g_row_start[g];
        s.rows[g] = r;
        s.slot[g] = g_slot[g];
        tiles = ((r + BM - 1) / BM) * n_tiles;
      }
      int incl = tiles;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      if (g < ng) s.tile_start[g] = carry + incl - tiles;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      s.tile_start[ng] = carry;
      s.num_tiles = carry * ksplit;
    }
  } else if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a_hi);
    tma_prefetch_desc(&map_a_lo);
    tma_prefetch_desc(&map_b_hi);
    tma_prefetch_desc(&map_b_lo);
    for (int i = 0; i < T_STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
      mbar_init(&s.conv[i], kConvWarps);
    }
    for (int i = 0; i < ACC; ++i) {
      mbar_init(&s.tfull[i], 1);
      mbar_init(&s.tempty[i], 4);
    }
    fence_barrier_init();
  } else if (warp == 1) {
    tmem_alloc(&s.tmem_base, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const int total = s.num_tiles;
  const uint32_t tmem_base = s.tmem_base;
  // tiles walk (group, m-tile, n-tile) with m fastest: a group's A rows stay in L2
  // across its n-tiles

  if (BRAW && warp >= 6) {
    // ================= converters: split raw B into hi (in place) / lo =================
    const int wi = static_cast<int>(warp) - 6;
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&s.full[stage], phase);
        float4* bh = reinterpret_cast<float4*>(b_hi_at(stage));
        float4* bl = reinterpret_cast<float4*>(b_lo_at(stage));
#pragma unroll 4
        for (int i = wi * 32 + static_cast<int>(lane); i < T_B_BYTES / 16; i += 32 * kConvWarps) {
          const float4 v = bh[i];
          float4 h, l;
          h.x = rna_tf32(v.x); l.x = rna_tf32(v.x - h.x);
          h.y = rna_tf32(v.y); l.y = rna_tf32(v.y - h.y);
          h.z = rna_tf32(v.z); l.z = rna_tf32(v.z - h.z);
          h.w = rna_tf32(v.w); l.w = rna_tf32(v.w - h.w);
          bh[i] = h;
          bl[i] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.conv[stage]);
        if (++stage == T_STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {  // ================= TMA producer =================
      const uint64_t pol = make_policy(0);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int part = tile % ksplit, gt = tile / ksplit;
        int lo = 0, hi = ng - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s.tile_start[mid] <= gt) lo = mid; else hi = mid - 1;
        }
        const int g = lo;
        const int local = gt - s.tile_start[g];
        const int m_tiles = (s.rows[g] + BM - 1) / BM;
        const int mt = local % m_tiles, nt = local / m_tiles;
        const int a_row = s.row_start[g] + mt * BM;
        const int b_row = s.slot[g] * N + nt * BN;
        const int k0 = part * num_kb * T_BK;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&s.empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&s.full[stage], BRAW ? T_STAGE_BYTES - T_B_BYTES : T_STAGE_BYTES);
          tma_load_2d(a_hi_at(stage), &map_a_hi, &s.full[stage], k0 + kb * T_BK, a_row, pol);
          tma_load_2d(a_lo_at(stage), &map_a_lo, &s.full[stage], k0 + kb * T_BK, a_row, pol);
          tma_load_2d(b_hi_at(stage), &map_b_hi, &s.full[stage], k0 + kb * T_BK, b_row, pol);
          if (!BRAW) tma_load_2d(b_lo_at(stage), &map_b_lo, &s.full[stage], k0 + kb * T_BK, b_row, pol);
          if (++stage == T_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ================= MMA issuer =================
      constexpr uint32_t idesc = umma_idesc_tf32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        mbar_wait(&s.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(BRAW ? &s.conv[stage] : &s.full[stage], phase);
          tc_fence_after();
          const uint32_t ah = smem_addr(a_hi_at(stage)), al = smem_addr(a_lo_at(stage));
          const uint32_t bh = smem_addr(b_hi_at(stage)), bl = smem_addr(b_lo_at(stage));
#pragma unroll
          for (int k = 0; k < T_BK / 8; ++k) {  // K = 8 tf32 (32 bytes) per instruction
            const uint32_t off = 32u * k;
            umma_tf32(d_tmem, t_desc(al + off), t_desc(bh + off), idesc, (kb | k) != 0);
            umma_tf32(d_tmem, t_desc(ah + off), t_desc(bl + off), idesc, 1);
            umma_tf32(d_tmem, t_desc(ah + off), t_desc(bh + off), idesc, 1);
          }
          umma_commit(&s.empty[stage]);
          if (++stage == T_STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&s.tfull[acc]);
        if (++acc == ACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp < 6) {
    // ================= epilogue (warps 2..5) =================
    const uint32_t quarter = warp & 3u;
    const int row_in_tile = static_cast<int>(quarter * 32 + lane);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int part = tile % ksplit, gt = tile / ksplit;
      int lo = 0, hi = ng - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s.tile_start[mid] <= gt) lo = mid; else hi = mid - 1;
      }
      const int g = lo;
      const int local = gt - s.tile_start[g];
      const int m_tiles = (s.rows[g] + BM - 1) / BM;
      const int mt = local % m_tiles, nt = local / m_tiles;
      const int r_local = mt * BM + row_in_tile;
      const bool row_ok = r_local < s.rows[g];
      const size_t row_off = static_cast<size_t>(s.row_start[g] + r_local) * ldc + nt * BN + part * split_stride;
      const bool raw = ksplit > 1;  // partials: no ReLU, no split

      mbar_wait(&s.tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_base = tmem_base + static_cast<uint32_t>(acc * BN) + ((quarter * 32u) << 16);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        if (nt * BN + c >= N) break;  // warp-uniform
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_base + static_cast<uint32_t>(c), v);
        tmem_ld_wait();
        if (row_ok) {
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = __uint_as_float(v[i]);
            f[i] = (relu && !raw) ? fmaxf(x, 0.f) : x;
          }
          if (C_lo && !raw) {  // split for the next GEMM
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 h, l;
              h.x = rna_tf32(f[4 * q]);     l.x = rna_tf32(f[4 * q] - h.x);
              h.y = rna_tf32(f[4 * q + 1]); l.y = rna_tf32(f[4 * q + 1] - h.y);
              h.z = rna_tf32(f[4 * q + 2]); l.z = rna_tf32(f[4 * q + 2] - h.z);
              h.w = rna_tf32(f[4 * q + 3]); l.w = rna_tf32(f[4 * q + 3] - h.w);
              *reinterpret_cast<float4*>(C + row_off + c + 4 * q) = h;
              *reinterpret_cast<float4*>(C_lo + row_off + c + 4 * q) = l;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              *reinterpret_cast<float4*>(C + row_off + c + 4 * q) =
                  make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.tempty[acc]);
      if (++acc == ACC) { acc = 0; acc_phase ^= 1; }
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// Sum the split-K partials in part order (deterministic), then ReLU / hi-lo split.
__global__ void ksplit_reduce_kernel(const float* __restrict__ P, int ksplit, size_t stride, int64_t n4, int relu,
                                     float* __restrict__ out, float* __restrict__ out_lo) {
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += step) {
    float4 a = reinterpret_cast<const float4*>(P)[i];
    for (int p = 1; p < ksplit; ++p) {
      const float4 b = reinterpret_cast<const float4*>(P + p * stride)[i];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    if (relu) { a.x = fmaxf(a.x, 0.f); a.y = fmaxf(a.y, 0.f); a.z = fmaxf(a.z, 0.f); a.w = fmaxf(a.w, 0.f); }
    if (out_lo) {
      float4 h, l;
      h.x = rna_tf32(a.x); l.x = rna_tf32(a.x - h.x);
      h.y = rna_tf32(a.y); l.y = rna_tf32(a.y - h.y);
      h.z = rna_tf32(a.z); l.z = rna_tf32(a.z - h.z);
      h.w = rna_tf32(a.w); l.w = rna_tf32(a.w - h.w);
      reinterpret_cast<float4*>(out)[i] = h;
      reinterpret_cast<float4*>(out_lo)[i] = l;
    } else {
      reinterpret_cast<float4*>(out)[i] = a;
    }
  }
}

__global__ void split_tf32_kernel(const float* __restrict__ in, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t n4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = reinterpret_cast<const float4*>(in)[i];
    float4 h, l;
    h.x = rna_tf32(v.x); l.x = rna_tf32(v.x - h.x);
    h.y = rna_tf32(v.y); l.y = rna_tf32(v.y - h.y);
    h.z = rna_tf32(v.z); l.z = rna_tf32(v.z - h.z);
    h.w = rna_tf32(v.w); l.w = rna_tf32(v.w - h.w);
    reinterpret_cast<float4*>(hi)[i] = h;
    reinterpret_cast<float4*>(lo)[i] = l;
  }
}

}  // namespace

bool gemm_use_cta_pair() {
  const char* env = std::getenv("HEP_GEMM_2CTA");
  return !(env && env[0] == '0');
}

uint32_t gemm_schedule(int rows_per_expert, int N, int K, bool up) {
  const char* env = std::getenv(up ? "HEP_GEMM_SCHED_UP" : "HEP_GEMM_SCHED_DOWN");
  if (env && *env) return static_cast<uint32_t>(std::strtoul(env, nullptr, 16));
  (void)N;
  // Measured on B200 (tools/gemm_sched_sweep.sh, profiles/r1_gemm_sched_sweep*.log).
  // CTA pair (256-row tiles): A evict_last, B default policy, m-fastest.  evict_first on
  // B hurt here: a B half-tile is re-read by the other clusters of its n-column after
  // it would have been evicted (DRAM reads 4.9 -> 2.2 GB up, 13.8 -> 8.4 GB down;
  // 1.25 -> 1.44-1.48 PFLOP/s).
  if (gemm_use_cta_pair()) {
    // down-projection with an expert's A stripe far beyond L2 (cfg3: 117 MB): super-rows of
    // 8 m-tiles keep a 59 MB A stripe resident (DRAM 5.3 -> 4.8 GB, -0.8% time; tools/gemm_down_sched.sh)
    const double a_bytes = static_cast<double>(rows_per_expert) * K * 2.0;
    return (!up && a_bytes > 64e6) ? 0x822u : 0x2u;
  }
  // Single CTA (128-row tiles): keep the operand re-used across a wave in L2
  // (evict_last) and stream the other (evict_first).  When one expert's A rows fit in
  // L2, rasterise m-fastest so A stays resident across all n-tiles; otherwise walk
  // super-rows of gm m-tiles (A stripe of ~32 MB resident, B streamed once per stripe).
  const double a_bytes = static_cast<double>(rows_per_expert) * K * 2.0;
  if (a_bytes <= 48e6) return 0x2u | (0x1u << 2);
  const int gm = std::max(1, std::min(255, static_cast<int>(32e6 / (128.0 * K * 2.0))));
  return 0x2u | (0x1u << 2) | (0x2u << 4) | (static_cast<uint32_t>(gm) << 8);
}

cudaError_t make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                              uint32_t box_rows, uint32_t box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_tmap_f32_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                             uint32_t box_cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 4};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (box_cols != 32 && box_cols != 16) return cudaErrorInvalidValue;
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_grouped_gemm_tf32x3(const CUtensorMap& a_hi, const CUtensorMap& a_lo, const CUtensorMap& b_hi,
                                       const CUtensorMap* b_lo, float* C, float* C_lo, int ldc, int N, int K,
                                       const GroupTable& groups, int relu, int num_sms, cudaStream_t stream,
                                       int ksplit, float* partial, int64_t rows_total) {
  if (ksplit < 1 || K % (T_BK * ksplit) || N % 32 || groups.num_groups > kMaxGroups || groups.num_groups <= 0)
    return cudaErrorInvalidValue;
  if (ksplit > 1 && !partial) return cudaErrorInvalidValue;
  const bool b_raw = b_lo == nullptr;
  static DeviceOnce attr_pre, attr_raw;
  DeviceOnce& once = b_raw ? attr_raw : attr_pre;
  if (!once.done()) {
    const cudaError_t e = cudaFuncSetAttribute(b_raw ? grouped_gemm_tf32x3_kernel<true> : grouped_gemm_tf32x3_kernel<false>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytesT));
    if (e != cudaSuccess) return e;
    once.set();
  }
  const size_t stride = static_cast<size_t>(rows_total) * ldc;
  float* out = ksplit > 1 ? partial : C;

  const int ng = groups.num_groups;
  if (b_raw)
    grouped_gemm_tf32x3_kernel<true><<<num_sms, kThreads + 32 * kConvWarps, kSmemBytesT, stream>>>(
        a_hi, a_lo, b_hi, b_hi, out, C_lo, ldc, N, K, groups.row_start, groups.rows, groups.slot, ng, relu, ksplit, stride);
  else
    grouped_gemm_tf32x3_kernel<false><<<num_sms, kThreads, kSmemBytesT, stream>>>(
        a_hi, a_lo, b_hi, *b_lo, out, C_lo, ldc, N, K, groups.row_start, groups.rows, groups.slot, ng, relu, ksplit, stride);
  if (ksplit > 1) {
    const int64_t n4 = static_cast<int64_t>(stride) / 4;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n4 + 255) / 256)));
    ksplit_reduce_kernel<<<blocks, 256, 0, stream>>>(partial, ksplit, stride, n4, relu, C, C_lo);
  }
  return cudaGetLastError();
}

cudaError_t launch_split_tf32(const float* in, float* hi, float* lo, int64_t n, cudaStream_t stream) {
  if (n % 4) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 8, (n4 + 255) / 256)));
  split_tf32_kernel<<<blocks, 256, 0, stream>>>(in, hi, lo, n4);
  return cudaGetLastError();
}

cudaError_t launch_grouped_gemm_bf16(const CUtensorMap& map_a, const CUtensorMap& map_b, void* C,
                                     int ldc, int N, int K, const GroupTable& groups, int relu,
                                     int num_sms, cudaStream_t stream, uint32_t sched) {
  if (K % BK || N % 32 || groups.num_groups > kMaxGroups || groups.num_groups <= 0)
    return cudaErrorInvalidValue;
  static DeviceOnce attr_set;
  if (!attr_set.done()) {
    const cudaError_t e = cudaFuncSetAttribute(
        grouped_gemm_bf16_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
    attr_set.set();
  }
  grouped_gemm_bf16_kernel<false><<<num_sms, kThreads, kSmemBytes, stream>>>(
      map_a, map_b, static_cast<__nv_bfloat16*>(C), ldc, N, K, groups.row_start, groups.rows,
      groups.slot, groups.out, groups.wait_src, groups.wait_flags, groups.epoch, groups.num_groups, relu, sched,
      groups.timeout_ns, PatchArgs{}, 0);
  return cudaGetLastError();
}

cudaError_t launch_grouped_gemm_bf16_patched(const CUtensorMap& map_a, const CUtensorMap& map_shared_b, void* C,
                                             int ldc, int N, int K, const GroupTable& groups, const PatchArgs& patches,
                                             int half, int relu, int num_sms, cudaStream_t stream, uint32_t sched) {
  if (K % BK || N % 32 || N > 65535 || groups.num_groups > kMaxGroups || groups.num_groups <= 0)
    return cudaErrorInvalidValue;
  static DeviceOnce attr_set;
  if (!attr_set.done()) {
    const cudaError_t e = cudaFuncSetAttribute(
        grouped_gemm_bf16_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytesPatch));
    if (e != cudaSuccess) return e;
    attr_set.set();
  }
  grouped_gemm_bf16_kernel<true><<<num_sms, kThreads + 32 * kConvWarps, kSmemBytesPatch, stream>>>(
      map_a, map_shared_b, static_cast<__nv_bfloat16*>(C), ldc, N, K, groups.row_start, groups.rows,
      groups.slot, groups.out, groups.wait_src, groups.wait_flags, groups.epoch, groups.num_groups, relu, sched,
      groups.timeout_ns, patches, half);
  return cudaGetLastError();
}

cudaError_t launch_grouped_gemm_bf16_2cta(const CUtensorMap& map_a, const CUtensorMap& map_b, void* C, int ldc,
                                          int N, int K, const GroupTable& groups, int relu, int num_sms,
                                          cudaStream_t stream, uint32_t sched, int* tile_counter, const int* a_src,
                                          const void* a_x) {
  if (K % BK || N % 32 || groups.num_groups > kMaxGroups || groups.num_groups <= 0) return cudaErrorInvalidValue;
  // HEP_GEMM_STAGES = 4 | 5 (default) | 6 (six stages, direct-store epilogue; local outputs only)
  const char* st_env = std::getenv("HEP_GEMM_STAGES");
  int stages = st_env ? std::atoi(st_env) : 5;
  if (stages == 6 && groups.out != nullptr) stages = 5;
  if (stages != 4 && stages != 6) stages = 5;
  // The dynamic tile scheduler runs when the caller passes a counter (the layer does for
  // its down-projection by default; profiles/r2_gemm_power.md): the 5-stage staged
  // kernel only.
  const bool dyn = tile_counter != nullptr && stages == 5 && a_src == nullptr;
  static DeviceOnce attr4, attr5, attr6, attr5d;
  DeviceOnce& once = dyn ? attr5d : (stages == 4 ? attr4 : (stages == 6 ? attr6 : attr5));
  if (!once.done()) {
    cudaError_t e;
    if (dyn)
      e = cudaFuncSetAttribute(grouped_gemm_bf16_2cta_kernel<false, 5, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes2));
    else if (stages == 4)
      e = cudaFuncSetAttribute(grouped_gemm_bf16_2cta_kernel<false, 4, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes2Four));
    else if (stages == 6)
      e = cudaFuncSetAttribute(grouped_gemm_bf16_2cta_kernel<false, 6, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes2Deep));
    else
      e = cudaFuncSetAttribute(grouped_gemm_bf16_2cta_kernel<false, 5, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes2));
    if (e != cudaSuccess) return e;
    once.set();
  }
  if (dyn) {
    const cudaError_t e = cudaMemsetAsync(tile_counter, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
  }
  const int grid = (num_sms / 2) * 2;
  if (a_src) {  // gathered A: the default 5-stage static schedule only, local outputs
    if (!a_x || groups.wait_src) return cudaErrorInvalidValue;
    static DeviceOnce attr_g;
    if (!attr_g.done()) {
      const cudaError_t e = cudaFuncSetAttribute(grouped_gemm_bf16_2cta_kernel<false, 5, false, false, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kSmemBytes2));
      if (e != cudaSuccess) return e;
      attr_g.set();
    }
    grouped_gemm_bf16_2cta_kernel<false, 5, false, false, true><<<grid, kThreads + 32 * kConvWarps, kSmemBytes2, stream>>>(
        map_a, map_b, static_cast<__nv_bfloat16*>(C), ldc, N, K, groups.row_start, groups.rows, groups.slot, groups.out,
        nullptr, nullptr, 0, groups.num_groups, relu, sched, groups.timeout_ns, PatchArgs{}, 0, nullptr, a_src,
        static_cast<const __nv_bfloat16*>(a_x));
    return cudaGetLastError();
  }
#define HEP_LAUNCH_2CTA(ST, DIR, DY, SMEM)                                                                           \
  grouped_gemm_bf16_2cta_kernel<false, ST, DIR, DY><<<grid, kThreads, SMEM, stream>>>(                              \
      map_a, map_b, static_cast<__nv_bfloat16*>(C), ldc, N, K, groups.row_start, groups.rows, groups.slot, groups.out, \
      groups.wait_src, groups.wait_flags, groups.epoch, groups.num_groups, relu, sched, groups.timeout_ns, PatchArgs{}, \
      0, tile_counter, nullptr, nullptr)
  if (dyn) HEP_LAUNCH_2CTA(5, false, true, kSmemBytes2);
  else if (stages == 4) HEP_LAUNCH_2CTA(4, false, false, kSmemBytes2Four);
  else if (stages == 6) HEP_LAUNCH_2CTA(6, true, false, kSmemBytes2Deep);
  else HEP_LAUNCH_2CTA(5, false, false, kSmemBytes2);
#undef HEP_LAUNCH_2CTA
  return cudaGetLastError();
}

cudaError_t launch_grouped_gemm_bf16_2cta_patched(const CUtensorMap& map_a, const CUtensorMap& map_shared_b, void* C,
                                                  int ldc, int N, int K, const GroupTable& groups,
                                                  const PatchArgs& patches, int half, int relu, int num_sms,
                                                  cudaStream_t stream, uint32_t sched) {
  if (K % BK || N % 32 || N > 65535 || groups.num_groups > kMaxGroups || groups.num_groups <= 0)
    return cudaErrorInvalidValue;
  static DeviceOnce attr_set;
  if (!attr_set.done()) {
    const cudaError_t e = cudaFuncSetAttribute(grouped_gemm_bf16_2cta_kernel<true>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(kSmemBytes2Patch));
    if (e != cudaSuccess) return e;
    attr_set.set();
  }
  const int grid = (num_sms / 2) * 2;
  grouped_gemm_bf16_2cta_kernel<true><<<grid, kThreads + 32 * kConvWarps, kSmemBytes2Patch, stream>>>(
      map_a, map_shared_b, static_cast<__nv_bfloat16*>(C), ldc, N, K, groups.row_start, groups.rows, groups.slot,
      groups.out, groups.wait_src, groups.wait_flags, groups.epoch, groups.num_groups, relu, sched, groups.timeout_ns,
      patches, half, nullptr, nullptr, nullptr);
  return cudaGetLastError();
}


// Loads every kernel of this file now (see preload_kernels in kernels.h).
cudaError_t preload_gemm_sm100_kernels() {
  auto load = [](const void* fn) {
    cudaFuncAttributes attr;
    return cudaFuncGetAttributes(&attr, fn);
  };
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_kernel<false>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_kernel<true>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_2cta_kernel<false, 4, false>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_2cta_kernel<false, 5, false>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_2cta_kernel<false, 6, true>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_2cta_kernel<false, 5, false, true>)))
    return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_2cta_kernel<true>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_bf16_2cta_kernel<false, 5, false, false, true>)))
    return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_tf32x3_kernel<false>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_tf32x3_kernel<true>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(ksplit_reduce_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(split_tf32_kernel))) return e;
  return cudaSuccess;
}

}  // namespace hep
