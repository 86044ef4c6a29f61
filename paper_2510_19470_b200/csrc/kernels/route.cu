// K1 gate/top-k, K2 permute/pack and K9 unpermute+combine for sm_100a.
//
// Semantics are the pinned S3/S5/S7 of SURVEY.md §8(c) (no reference code exists
// for them; oracle/moe_oracle.c is the CPU restatement they are tested against):
//   gate:    logits = x . W_g; top-k by (logit desc, expert id asc); weights =
//            softmax over the k selected logits (fp32).
//   permute: rows grouped by key = (destination GPU, expert), stable by (token,
//            slot): a counting sort done as per-32-token-chunk ranks + two scans.
//   combine: y_t = sum_j w_tj * out[pos_tj], slot order, fp32 accumulate.
// All three are HBM-bound; they move rows with 16-byte vector accesses, one warp
// per token row.

#include <float.h>

#include <cooperative_groups.h>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace hep {

namespace {

constexpr int kChunk = 32;      // tokens per gate block == ranking chunk
constexpr int kHc = 64;         // hidden columns staged per step
constexpr int kMaxE = 64;       // experts supported by the gate kernel
constexpr int kMaxK = 8;
constexpr int kMaxNK = 512;    // (destination, expert) keys: G * E, G <= 8 GPUs of one box

template <typename T>
__device__ __forceinline__ float to_f32(T v) { return static_cast<float>(v); }

// One block = one chunk of 32 tokens, 256 threads.
template <typename T>
__global__ void __launch_bounds__(256) gate_kernel(const T* __restrict__ x,
                                                   const float* __restrict__ wg_t, int T_tok,
                                                   int H, int E, int k,
                                                   const int* __restrict__ dest_of_owner,
                                                   int n_per_gpu, int NK, int* __restrict__ topk_idx,
                                                   float* __restrict__ topk_w,
                                                   int* __restrict__ keys, int* __restrict__ ranks,
                                                   int* __restrict__ chunk_counts) {
  __shared__ float xs[kChunk][kHc + 1];
  __shared__ float ws[kMaxE][kHc + 1];
  __shared__ float logits[kChunk][kMaxE + 1];
  __shared__ int skey[kChunk][kMaxK];

  const int tid = threadIdx.x;
  const int chunk = blockIdx.x;
  const int t0 = chunk * kChunk;
  const int tok = tid >> 3;   // 0..31
  const int eg = tid & 7;     // expert group: experts eg, eg+8, ...

  float acc[kMaxE / 8];
#pragma unroll
  for (int i = 0; i < kMaxE / 8; ++i) acc[i] = 0.f;

  for (int hc = 0; hc < H; hc += kHc) {
    const int width = min(kHc, H - hc);
    for (int i = tid; i < kChunk * kHc; i += blockDim.x) {
      const int r = i / kHc, c = i % kHc;
      const int t = t0 + r;
      xs[r][c] = (t < T_tok && c < width) ? to_f32<T>(x[static_cast<size_t>(t) * H + hc + c]) : 0.f;
    }
    for (int i = tid; i < E * kHc; i += blockDim.x) {
      const int e = i / kHc, c = i % kHc;
      ws[e][c] = c < width ? wg_t[static_cast<size_t>(e) * H + hc + c] : 0.f;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < kHc; ++c) {
      const float xv = xs[tok][c];
#pragma unroll
      for (int i = 0; i < kMaxE / 8; ++i)
        if (eg + 8 * i < E) acc[i] = fmaf(xv, ws[eg + 8 * i][c], acc[i]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kMaxE / 8; ++i)
    if (eg + 8 * i < E) logits[tok][eg + 8 * i] = acc[i];
  __syncthreads();

  // Top-k per token: warp w handles tokens 4w..4w+3.
  const int lane = tid & 31, warp = tid >> 5;
  for (int q = 0; q < 4; ++q) {
    const int r = warp * 4 + q;
    const int t = t0 + r;
    if (t >= T_tok) break;  // warp-uniform
    float v0 = lane < E ? logits[r][lane] : -FLT_MAX;
    float v1 = lane + 32 < E ? logits[r][lane + 32] : -FLT_MAX;
    bool used0 = lane >= E, used1 = lane + 32 >= E;
    float sel_v[kMaxK];
    int sel_e[kMaxK];
    for (int j = 0; j < k; ++j) {
      // Candidate of this lane: the better of its two experts (lower id wins ties).
      float bv = -FLT_MAX;
      int be = 0x7fffffff;
      if (!used0) { bv = v0; be = lane; }
      if (!used1 && (be == 0x7fffffff || v1 > bv)) { bv = v1; be = lane + 32; }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (oe != 0x7fffffff && (be == 0x7fffffff || ov > bv || (ov == bv && oe < be))) {
          bv = ov;
          be = oe;
        }
      }
      sel_v[j] = bv;
      sel_e[j] = be;
      if (be == lane) used0 = true;
      if (be == lane + 32) used1 = true;
    }
    if (lane == 0) {
      float ex[kMaxK], s = 0.f;
      for (int j = 0; j < k; ++j) {
        ex[j] = expf(sel_v[j] - sel_v[0]);
        s += ex[j];
      }
      for (int j = 0; j < k; ++j) {
        const size_t o = static_cast<size_t>(t) * k + j;
        const int e = sel_e[j];
        const int key = dest_of_owner[e / n_per_gpu] * E + e;
        topk_idx[o] = e;
        topk_w[o] = ex[j] / s;
        keys[o] = key;
        skey[r][j] = key;
      }
    }
  }
  __syncthreads();

  // Stable rank of (t, j) among earlier tokens of the chunk with the same key.
  int* counts = chunk_counts + static_cast<size_t>(chunk) * NK;
  for (int i = tid; i < NK; i += blockDim.x) counts[i] = 0;
  __syncthreads();
  const int valid = min(kChunk, T_tok - t0);
  for (int i = tid; i < valid * k; i += blockDim.x) {
    const int r = i / k, j = i % k;
    const int key = skey[r][j];
    int before = 0, after = 0;
    for (int r2 = 0; r2 < valid; ++r2) {
      if (r2 == r) continue;
      for (int j2 = 0; j2 < k; ++j2)
        if (skey[r2][j2] == key) {
          if (r2 < r) ++before; else ++after;
        }
    }
    ranks[static_cast<size_t>(t0 + r) * k + j] = before;
    if (after == 0) counts[key] = before + 1;
  }
}

// ---------------------------------------------------------------------------------
// bf16 gate: logits on the tensor cores (mma.sync m16n8k16, fp32 accumulate), x and
// W_g^T streamed through a 4-stage cp.async pipeline.  One block = 64 tokens (two
// ranking chunks), 4 warps x 16 tokens.  The gate is HBM-bound on reading x; the old
// CUDA-core kernel above was latency-bound (one global round trip per 64 columns).
// Exactness: bf16 x bf16 products are exact in fp32 and, for the dyadic parity inputs,
// every partial sum is exactly representable, so the logits do not depend on the
// tensor core's summation order.
constexpr int kGT = 64;          // tokens per block
constexpr int kGCMin = 64;       // hidden columns per stage: H must be a multiple
// Pipeline depth and gate-weight rows staged per stage: with few experts the x stream
// gets a deeper pipeline (more bytes in flight per SM).
// Wider stages read longer runs of each token row (128 or 256 B per row per stage).
template <int STAGES, int EROWS, int GC>
constexpr size_t gate_smem() { return static_cast<size_t>(STAGES) * (kGT + EROWS) * (GC + 8) * 2; }

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(const void* p, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(smem_addr(p)));
}

__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int kGStages, int EROWS, int kGC>
__global__ void __launch_bounds__(256) gate_mma_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ wg_t, int T_tok,
                                                      int H, int E, int k,
                                                      const int* __restrict__ dest_of_owner, int n_per_gpu,
                                                      int NK, int* __restrict__ topk_idx,
                                                      float* __restrict__ topk_w, int* __restrict__ keys,
                                                      int* __restrict__ ranks,
                                                      int* __restrict__ chunk_counts) {
  constexpr int kGPitch = kGC + 8;  // bf16 elements per smem row (16-byte pad: no ldmatrix conflicts)
  extern __shared__ __align__(128) uint8_t gsm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(gsm);                      // [S][64][pitch]
  __nv_bfloat16* ws = xs + static_cast<size_t>(kGStages) * kGT * kGPitch;         // [S][EROWS][pitch]
  __shared__ float logits[kGT][kMaxE + 1];
  __shared__ int skey[kGT][kMaxK];
  __shared__ int kcount[kGT / kChunk][kMaxNK];  // per-chunk running key counts

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t0 = blockIdx.x * kGT;
  const int nkc = H / kGC;
  const int ntiles = E / 8;

  auto load_stage = [&](int s, int kc) {
    const int hc = kc * kGC;
    __nv_bfloat16* xd = xs + static_cast<size_t>(s) * kGT * kGPitch;
    __nv_bfloat16* wd = ws + static_cast<size_t>(s) * EROWS * kGPitch;
    constexpr int kCh = kGC / 8;  // 16-byte chunks per row per stage
#pragma unroll
    for (int i = tid; i < kGT * kCh; i += 256) {
      const int r = i / kCh, c8 = (i % kCh) * 8;
      const int t = t0 + r;
      cp_async16(xd + r * kGPitch + c8, x + static_cast<size_t>(t < T_tok ? t : 0) * H + hc + c8, t < T_tok);
    }
    for (int i = tid; i < E * kCh; i += 256) {
      const int r = i / kCh, c8 = (i % kCh) * 8;
      cp_async16(wd + r * kGPitch + c8, wg_t + static_cast<size_t>(r) * H + hc + c8, true);
    }
  };

  float acc[kMaxE / 8][4];
#pragma unroll
  for (int i = 0; i < kMaxE / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

#pragma unroll
  for (int s = 0; s < kGStages - 1; ++s) {
    if (s < nkc) load_stage(s, s);
    cp_async_commit();
  }
  for (int kc = 0; kc < nkc; ++kc) {
    cp_async_wait<kGStages - 2>();
    __syncthreads();
    const int pre = kc + kGStages - 1;
    if (pre < nkc) load_stage(pre % kGStages, pre);
    cp_async_commit();
    const int s = kc % kGStages;
    const __nv_bfloat16* xa = xs + static_cast<size_t>(s) * kGT * kGPitch + ((warp & 3) * 16) * kGPitch;
    const __nv_bfloat16* wb = ws + static_cast<size_t>(s) * EROWS * kGPitch;
    // split-K inside the block: warps 0-3 take the stage's first half of 16-column
    // steps, warps 4-7 the second half (8 warps in flight per block)
    constexpr int kHalf = kGC / 32;
#pragma unroll
    for (int ks = (warp >> 2) * kHalf; ks < (warp >> 2) * kHalf + kHalf; ++ks) {
      uint32_t a[4];
      ldsm_x4(xa + (lane & 15) * kGPitch + ks * 16 + (lane >> 4) * 8, a[0], a[1], a[2], a[3]);
#pragma unroll
      for (int nt = 0; nt < kMaxE / 8; nt += 2) {
        if (nt >= ntiles) break;
        uint32_t b0, b1, b2, b3;
        const int n = nt * 8 + (lane >> 4) * 8 + (lane & 7);
        ldsm_x4(wb + (n < E ? n : 0) * kGPitch + ks * 16 + ((lane >> 3) & 1) * 8, b0, b1, b2, b3);
        mma_bf16_16816(acc[nt], a, b0, b1);
        if (nt + 1 < ntiles) mma_bf16_16816(acc[nt + 1], a, b2, b3);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // the stage buffers are free: the k-half partials go there
  float (*part)[kMaxE + 1] = reinterpret_cast<float (*)[kMaxE + 1]>(gsm);
  if (warp >= 4) {
#pragma unroll
    for (int nt = 0; nt < kMaxE / 8; ++nt) {
      if (nt >= ntiles) break;
      const int r = (warp & 3) * 16 + (lane >> 2), c = nt * 8 + (lane & 3) * 2;
      part[r][c] = acc[nt][0];
      part[r][c + 1] = acc[nt][1];
      part[r + 8][c] = acc[nt][2];
      part[r + 8][c + 1] = acc[nt][3];
    }
  }
  __syncthreads();
  if (warp < 4) {
#pragma unroll
    for (int nt = 0; nt < kMaxE / 8; ++nt) {
      if (nt >= ntiles) break;
      const int r = warp * 16 + (lane >> 2), c = nt * 8 + (lane & 3) * 2;
      logits[r][c] = acc[nt][0] + part[r][c];
      logits[r][c + 1] = acc[nt][1] + part[r][c + 1];
      logits[r + 8][c] = acc[nt][2] + part[r + 8][c];
      logits[r + 8][c + 1] = acc[nt][3] + part[r + 8][c + 1];
    }
  }
  __syncthreads();

  // Top-k per token, four threads per token (each scans a quarter of the E logits): k
  // rounds of (local best among unused) -> exchange within the quad; order (logit desc,
  // expert id asc).
  {
    const int r = tid >> 2, h = tid & 3;  // 256 threads = 64 tokens x 4
    const int t = t0 + r;
    const int half = E >> 2, e0 = h * half;
    uint32_t used = 0;  // bit i: logit e0 + i taken (quarter <= 16)
    float sel_v[kMaxK];
    int sel_e[kMaxK];
    for (int j = 0; j < k; ++j) {
      float bv = -FLT_MAX;
      int be = 0x7fffffff;
      for (int i = 0; i < half; ++i) {
        const float v = logits[r][e0 + i];
        if (!((used >> i) & 1u) && (be == 0x7fffffff || v > bv)) { bv = v; be = e0 + i; }  // ids ascend
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (oe != 0x7fffffff && (be == 0x7fffffff || ov > bv || (ov == bv && oe < be))) { bv = ov; be = oe; }
      }
      sel_v[j] = bv;
      sel_e[j] = be;
      if (be >= e0 && be < e0 + half) used |= 1u << (be - e0);
    }
    if (t < T_tok) {
      float s = 0.f;
      for (int j = 0; j < k; ++j) s += expf(sel_v[j] - sel_v[0]);
      for (int j = h; j < k; j += 4) {  // the quad splits the k slots
        const size_t o = static_cast<size_t>(t) * k + j;
        const int e = sel_e[j];
        const int key = dest_of_owner[e / n_per_gpu] * E + e;
        topk_idx[o] = e;
        topk_w[o] = expf(sel_v[j] - sel_v[0]) / s;
        keys[o] = key;
        skey[r][j] = key;
      }
    }
  }
  __syncthreads();

  // Ranking per 32-token chunk (two chunks per block, one warp each): entries in
  // (token, slot) order, 32 per round; lanes holding the same key find each other with
  // match.any, the rank is the key's running count plus the lower lanes of the group.
  if (warp < kGT / kChunk) {
    const int sub = warp;
    const int chunk = blockIdx.x * (kGT / kChunk) + sub;
    const int c0 = sub * kChunk;
    const int valid = min(kChunk, T_tok - (t0 + c0));
    if (valid > 0) {
      int* cnt = kcount[sub];
      for (int i = lane; i < NK; i += 32) cnt[i] = 0;
      __syncwarp();
      const int n_ent = valid * k;
      for (int base = 0; base < n_ent; base += 32) {
        const int i = base + lane;
        const int key = i < n_ent ? skey[c0 + i / k][i % k] : -1;
        const unsigned int peers = __match_any_sync(0xffffffffu, key);
        const int before = __popc(peers & ((1u << lane) - 1u));
        if (i < n_ent) ranks[static_cast<size_t>(t0 + c0) * k + i] = cnt[key] + before;
        __syncwarp();
        if (i < n_ent && before == 0) cnt[key] += __popc(peers);
        __syncwarp();
      }
      int* counts = chunk_counts + static_cast<size_t>(chunk) * NK;
      for (int i = lane; i < NK; i += 32) counts[i] = cnt[i];
    }
  }
}

// fp32 gate with the whole chunk resident: one block = one 32-token ranking chunk; x
// rows and W_g^T land in shared memory through cp.async in one shot (no per-column
// round trips), logits on the CUDA cores (exact for the dyadic parity inputs), top-k by
// eight threads per token, ranking by match.any as in the bf16 kernel.
// CS > 1: a cluster of CS CTAs per chunk, CTA r staging columns [r H/CS, (r+1) H/CS) --
// CS times the SMs pulling the chunk in when there are few chunks (cfg1: 16).  CTA 0 sums
// the partial logits over DSMEM in rank order, then ranks the chunk alone.
template <int CS>
__global__ void __launch_bounds__(256) gate_f32_oneshot_kernel(const float* __restrict__ x,
                                                               const float* __restrict__ wg_t, int T_tok, int H,
                                                               int E, int k, const int* __restrict__ dest_of_owner,
                                                               int n_per_gpu, int NK, int* __restrict__ topk_idx,
                                                               float* __restrict__ topk_w, int* __restrict__ keys,
                                                               int* __restrict__ ranks,
                                                               int* __restrict__ chunk_counts) {
  extern __shared__ __align__(16) float fsm[];
  const int Hc = H / CS;     // this CTA's columns
  const int pitch = Hc + 4;  // floats; rows stay 16-byte aligned
  float* xs = fsm;                   // [kChunk][pitch]
  float* ws = fsm + kChunk * pitch;  // [E][pitch]
  __shared__ float logits[kChunk][kMaxE + 1];
  __shared__ int skey[kChunk][kMaxK];
  __shared__ int kcount[kMaxNK];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int crank = CS > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int chunk = blockIdx.x / CS, t0 = chunk * kChunk, col0 = crank * Hc;
  const int c4 = Hc / 4;
  for (int i = tid; i < kChunk * c4; i += blockDim.x) {
    const int r = i / c4, c = (i % c4) * 4, t = t0 + r;
    cp_async16(xs + r * pitch + c, x + static_cast<size_t>(t < T_tok ? t : 0) * H + col0 + c, t < T_tok);
  }
  for (int i = tid; i < E * c4; i += blockDim.x) {
    const int r = i / c4, c = (i % c4) * 4;
    cp_async16(ws + r * pitch + c, wg_t + static_cast<size_t>(r) * H + col0 + c, true);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  {
    // Warp w: tokens 4w..4w+3 against 8 experts at a time; lane l sums the float4 columns
    // l, l+32, ... (4 x 8 register accumulators, every shared-memory word read once per
    // warp), then a transposing butterfly leaves the (token, expert) total l on lane l.
    // Logits are exact for the dyadic parity inputs in any order (S3).
    const int tb = warp * 4;
    for (int e0 = 0; e0 < E; e0 += 8) {
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
      for (int c = lane * 4; c < Hc; c += 128) {
        float4 xv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) xv[q] = *reinterpret_cast<const float4*>(xs + (tb + q) * pitch + c);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float4 wv = *reinterpret_cast<const float4*>(ws + (e0 + e) * pitch + c);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float a = v[q * 8 + e];
            a = fmaf(xv[q].x, wv.x, a);
            a = fmaf(xv[q].y, wv.y, a);
            a = fmaf(xv[q].z, wv.z, a);
            v[q * 8 + e] = fmaf(xv[q].w, wv.w, a);
          }
        }
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < off; ++i) {
          const float send = up ? v[i] : v[i + off];
          const float keep = up ? v[i + off] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      logits[tb + (lane >> 3)][e0 + (lane & 7)] = v[0];
    }
  }
  if constexpr (CS > 1) {
    cluster_sync();  // every CTA's partial logits are in its shared memory
    if (crank != 0) {
      cluster_sync();  // CTA 0 has read them; nothing else to do
      return;
    }
    auto cl = cooperative_groups::this_cluster();
    for (int i = tid; i < kChunk * E; i += blockDim.x) {
      const int r = i / E, e = i % E;
      float acc = logits[r][e];
#pragma unroll
      for (int q = 1; q < CS; ++q) acc += cl.map_shared_rank(&logits[0][0], q)[r * (kMaxE + 1) + e];
      logits[r][e] = acc;
    }
    cluster_sync();  // peers may exit
  }
  __syncthreads();
  {  // top-k: eight threads per token, each scans E/8 logits
    const int r = tid >> 3, h = tid & 7, t = t0 + r;
    const int part = E >> 3, e0 = h * part;
    uint32_t used = 0;
    float sel_v[kMaxK];
    int sel_e[kMaxK];
    for (int j = 0; j < k; ++j) {
      float bv = -FLT_MAX;
      int be = 0x7fffffff;
      for (int i = 0; i < part; ++i) {
        const float v = logits[r][e0 + i];
        if (!((used >> i) & 1u) && (be == 0x7fffffff || v > bv)) { bv = v; be = e0 + i; }
      }
#pragma unroll
      for (int off = 1; off <= 4; off <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oe = __shfl_xor_sync(0xffffffffu, be, off);
        if (oe != 0x7fffffff && (be == 0x7fffffff || ov > bv || (ov == bv && oe < be))) { bv = ov; be = oe; }
      }
      sel_v[j] = bv;
      sel_e[j] = be;
      if (be >= e0 && be < e0 + part) used |= 1u << (be - e0);
    }
    if (t < T_tok) {
      float ssum = 0.f;
      for (int j = 0; j < k; ++j) ssum += expf(sel_v[j] - sel_v[0]);
      for (int j = h; j < k; j += 8) {
        const size_t o = static_cast<size_t>(t) * k + j;
        const int e = sel_e[j];
        const int key = dest_of_owner[e / n_per_gpu] * E + e;
        topk_idx[o] = e;
        topk_w[o] = expf(sel_v[j] - sel_v[0]) / ssum;
        keys[o] = key;
        skey[r][j] = key;
      }
    }
  }
  __syncthreads();
  if (warp == 0) {  // ranking of the chunk's (token, slot) entries
    const int valid = min(kChunk, T_tok - t0);
    for (int i = lane; i < NK; i += 32) kcount[i] = 0;
    __syncwarp();
    const int n_ent = valid * k;
    for (int base = 0; base < n_ent; base += 32) {
      const int i = base + lane;
      const int key = i < n_ent ? skey[i / k][i % k] : -1;
      const unsigned int peers = __match_any_sync(0xffffffffu, key);
      const int before = __popc(peers & ((1u << lane) - 1u));
      if (i < n_ent) ranks[static_cast<size_t>(t0) * k + i] = kcount[key] + before;
      __syncwarp();
      if (i < n_ent && before == 0) kcount[key] += __popc(peers);
      __syncwarp();
    }
    int* counts = chunk_counts + static_cast<size_t>(chunk) * NK;
    for (int i = lane; i < NK; i += 32) counts[i] = kcount[i];
  }
}

// ---------------------------------------------------------------------------------
// bf16 gate on the 5th-gen tensor cores: one CTA per 128 tokens; TMA streams the x
// tile (128 x 64, SW128) and W_g^T (NE x 64; rows past E are zero-filled) through a
// 4-stage mbarrier ring; one thread issues tcgen05.mma M=128 N=NE K=16 into TMEM; the
// four epilogue warps each own 32 tokens (= one ranking chunk): tcgen05.ld of their
// logit rows, top-k and softmax per thread, match.any ranking per warp.  Warp roles as
// in the expert GEMM: w0 TMA, w1 TMEM + MMA, w2..w5 epilogue.
constexpr int kUGT = 128;      // tokens per CTA
constexpr int kUGK = 64;       // K per stage (128 B of bf16 = one swizzle row)
template <int NE, int KS>
constexpr int ug_stages() { return KS > 1 ? (NE <= 16 ? 4 : 3) : (NE <= 16 ? 8 : 6); }  // split: 2 CTAs per SM

// KS = 2: a 2-CTA cluster per tile splits K; the second CTA hands its partial logits
// over DSMEM, so the x stream spreads over all SMs (128-token tiles alone leave SMs idle).
template <int NE, int KS>
__global__ void __launch_bounds__(192, 1) gate_umma_kernel(const __grid_constant__ CUtensorMap map_x,
                                                           const __grid_constant__ CUtensorMap map_w, int T_tok,
                                                           int H, int E, int k, const int* __restrict__ dest_of_owner,
                                                           int n_per_gpu, int NK, int* __restrict__ topk_idx,
                                                           float* __restrict__ topk_w, int* __restrict__ keys,
                                                           int* __restrict__ ranks, int* __restrict__ chunk_counts) {
  constexpr int A_BYTES = kUGT * kUGK * 2;
  constexpr int B_BYTES = NE * kUGK * 2;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int TCOLS = NE < 32 ? 32 : NE;
  extern __shared__ uint8_t ug_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ug_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int kUGStages = ug_stages<NE, KS>();
  __shared__ __align__(8) uint64_t full[kUGStages], empty[kUGStages], tfull;
  __shared__ uint32_t tmem_base_sh;
  __shared__ int skey[4][32][kMaxK];
  __shared__ int kcount[4][kMaxNK];
  // the second K half's logits (KS = 2) reuse the stage ring once the MMAs are done
  float (*part)[NE] = reinterpret_cast<float (*)[NE]>(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = KS > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  const int tile = blockIdx.x / KS;
  const int t0 = tile * kUGT;
  const int kb_all = H / kUGK, num_kb = kb_all / KS, kb0 = crank * num_kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_x);
    tma_prefetch_desc(&map_w);
    for (int i = 0; i < kUGStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&tfull, 1);
    fence_barrier_init();
  } else if (warp == 1) {
    tmem_alloc(&tmem_base_sh, TCOLS);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      const uint64_t pol_x = l2_policy_evict_first(), pol_w = l2_policy_evict_last();
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % kUGStages;
        mbar_wait(&empty[st], ((kb / kUGStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], STAGE);
        tma_load_2d(sm + st * STAGE, &map_x, &full[st], (kb0 + kb) * kUGK, t0, pol_x);
        tma_load_2d(sm + st * STAGE + A_BYTES, &map_w, &full[st], (kb0 + kb) * kUGK, 0, pol_w);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = umma_idesc_bf16(kUGT, NE);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int st = kb % kUGStages;
        mbar_wait(&full[st], (kb / kUGStages) & 1);
        tc_fence_after();
        const uint32_t a = smem_addr(sm + st * STAGE), b = smem_addr(sm + st * STAGE + A_BYTES);
#pragma unroll
        for (int kk = 0; kk < kUGK / 16; ++kk)
          umma_bf16(tmem, umma_desc_k_sw128(a + 32 * kk), umma_desc_k_sw128(b + 32 * kk), idesc, (kb | kk) != 0);
        umma_commit(&empty[st]);
      }
      umma_commit(&tfull);
    }
  }
  // epilogue warps: warp w owns TMEM lanes 32 (w % 4) .. +31 = tokens of one ranking chunk
  const bool epi = warp >= 2;
  const int q = warp & 3;
  const int r = q * 32 + lane, t = t0 + r;
  float v[NE < 32 ? 32 : NE];
  if (epi) {
    mbar_wait(&tfull, 0);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < (NE < 32 ? 32 : NE); c += 32) {
      uint32_t u[32];
      tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, u);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) v[c + i] = __uint_as_float(u[i]);
    }
    tc_fence_before();
    if (KS > 1 && crank == 1) {
#pragma unroll
      for (int e = 0; e < NE; ++e) part[r][e] = v[e];
    }
  }
  if (KS > 1) {
    __syncwarp();
    cluster_sync();  // the second half's logits are in its shared memory
    if (epi && crank == 0) {
      const float* peer = cooperative_groups::this_cluster().map_shared_rank(&part[0][0], 1);
#pragma unroll
      for (int e = 0; e < NE; ++e) v[e] += peer[r * NE + e];
    }
  }
  if (epi && crank == 0) {
    // top-k by (logit desc, expert id asc), softmax over the k selected
    unsigned long long used = 0;
    float sel_v[kMaxK];
    int sel_e[kMaxK];
    for (int j = 0; j < k; ++j) {
      float bv = 0.f;
      int be = -1;
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (e < E && !((used >> e) & 1ull) && (be < 0 || v[e] > bv)) { bv = v[e]; be = e; }
      sel_v[j] = bv;
      sel_e[j] = be;
      used |= 1ull << be;
    }
    const int valid = min(32, T_tok - (t0 + q * 32));
    if (t < T_tok) {
      float ssum = 0.f;
      for (int j = 0; j < k; ++j) ssum += expf(sel_v[j] - sel_v[0]);
      for (int j = 0; j < k; ++j) {
        const size_t o = static_cast<size_t>(t) * k + j;
        const int e = sel_e[j];
        const int key = dest_of_owner[e / n_per_gpu] * E + e;
        topk_idx[o] = e;
        topk_w[o] = expf(sel_v[j] - sel_v[0]) / ssum;
        keys[o] = key;
        skey[q][lane][j] = key;
      }
    }
    __syncwarp();
    if (valid > 0) {  // ranking of this chunk's (token, slot) entries
      int* cnt = kcount[q];
      for (int i = lane; i < NK; i += 32) cnt[i] = 0;
      __syncwarp();
      const int n_ent = valid * k;
      for (int base = 0; base < n_ent; base += 32) {
        const int i = base + lane;
        const int key = i < n_ent ? skey[q][i / k][i % k] : -1;
        const unsigned int peers = __match_any_sync(0xffffffffu, key);
        const int before = __popc(peers & ((1u << lane) - 1u));
        if (i < n_ent) ranks[static_cast<size_t>(t0 + q * 32) * k + i] = cnt[key] + before;
        __syncwarp();
        if (i < n_ent && before == 0) cnt[key] += __popc(peers);
        __syncwarp();
      }
      int* counts = chunk_counts + static_cast<size_t>(tile * 4 + q) * NK;
      for (int i = lane; i < NK; i += 32) counts[i] = cnt[i];
    }
  }
  if (KS > 1) {
    __syncwarp();
    cluster_sync();  // the peer's logits were read before it may exit
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, TCOLS);
  }
}

template <int NE, int KS>
constexpr size_t gate_umma_smem() {
  return 1024 + static_cast<size_t>(ug_stages<NE, KS>()) * (kUGT + NE) * kUGK * 2;
}


// One block per key: exclusive scan of chunk_counts[:, key] over chunks.
__global__ void __launch_bounds__(1024) chunk_scan_kernel(const int* __restrict__ chunk_counts,
                                                          int nchunks, int NK,
                                                          int* __restrict__ chunk_off,
                                                          int* __restrict__ key_total) {
  __shared__ int warp_sums[32];
  __shared__ int carry_s;
  const int key = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < nchunks; base += blockDim.x) {
    const int c = base + threadIdx.x;
    const int v = c < nchunks ? chunk_counts[static_cast<size_t>(c) * NK + key] : 0;
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += o;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int carry = carry_s;
    const int warp_base = warp ? warp_sums[warp - 1] : 0;
    if (c < nchunks) chunk_off[static_cast<size_t>(c) * NK + key] = carry + warp_base + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) key_total[key] = carry_s;
}

// Single block: key offsets, per-destination totals and the local group table.
__global__ void __launch_bounds__(1024) key_scan_kernel(const int* __restrict__ key_total, int G,
                                                        int E, int self,
                                                        const int* __restrict__ slot_of_expert,
                                                        int* __restrict__ key_off,
                                                        int* __restrict__ dest_rows,
                                                        int* __restrict__ dest_off,
                                                        int* __restrict__ g_row_start,
                                                        int* __restrict__ g_rows,
                                                        int* __restrict__ g_slot) {
  __shared__ int warp_sums[32];
  __shared__ int carry_s;
  const int NK = G * E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int base = 0; base < NK; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < NK ? key_total[i] : 0;
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += o;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int carry = carry_s;
    if (i < NK) key_off[i] = carry + (warp ? warp_sums[warp - 1] : 0) + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  // key_off is complete (same block, synced above).
  for (int d = threadIdx.x; d < G; d += blockDim.x) {
    int rows = 0;
    for (int e = 0; e < E; ++e) rows += key_total[d * E + e];
    dest_rows[d] = rows;
    dest_off[d] = key_off[d * E];
  }
  if (threadIdx.x == 0) {
    int g = 0;
    for (int e = 0; e < E; ++e) {
      const int s = slot_of_expert[e];
      if (s < 0) continue;
      g_row_start[g] = key_off[self * E + e];
      g_rows[g] = key_total[self * E + e];
      g_slot[g] = s;
      ++g;
    }
  }
}

// One warp per token: compute the k destinations and copy the row there.
__global__ void __launch_bounds__(256) permute_kernel(const uint8_t* __restrict__ x, int T_tok,
                                                      int row_bytes, int k, int NK,
                                                      const int* __restrict__ keys,
                                                      const int* __restrict__ ranks,
                                                      const int* __restrict__ chunk_off,
                                                      const int* __restrict__ key_off,
                                                      int* __restrict__ pos,
                                                      uint8_t* __restrict__ packed, int seg) {
  const int lane = threadIdx.x & 31;
  const int vecs = row_bytes >> 4;
  int t, sg, v0, v1;
  row_segment(vecs, seg, t, sg, v0, v1);
  if (t >= T_tok) return;
  const int chunk = t / kChunk;
  int dst[kMaxK];
  for (int j = 0; j < k; ++j) {
    const size_t o = static_cast<size_t>(t) * k + j;
    const int key = keys[o];
    dst[j] = key_off[key] + chunk_off[static_cast<size_t>(chunk) * NK + key] + ranks[o];
    if (lane == 0 && sg == 0) pos[o] = dst[j];
  }
  const uint8_t* src = x + static_cast<size_t>(t) * row_bytes;
  for (int v = v0 + lane; v < v1; v += 32) {
    const uint4 val = ld_nc_v4(src + 16 * v);
    for (int j = 0; j < k; ++j) st_v4(packed + static_cast<size_t>(dst[j]) * row_bytes + 16 * v, val);
  }
}

__global__ void positions_kernel(int T_tok, int k, int NK, const int* __restrict__ keys,
                                 const int* __restrict__ ranks, const int* __restrict__ chunk_off,
                                 const int* __restrict__ key_off, int* __restrict__ pos, int* __restrict__ src) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T_tok * k) {
    // the 256 rows past the last group: a partial m-tile of the gathered A load reads
    // them, so they must name valid tokens of this step
    if (src && i < T_tok * k + 256) src[i] = 0;
    return;
  }
  const int t = i / k, key = keys[i];
  const int p = key_off[key] + chunk_off[static_cast<size_t>(t / kChunk) * NK + key] + ranks[i];
  pos[i] = p;
  if (src) src[p] = t;  // the inverse map: grouped row p is token t (gathered A load)
}

// One warp per token.  bf16 rows: 8 elements per 16-byte vector.
__global__ void __launch_bounds__(256) combine_bf16_kernel(const __nv_bfloat16* __restrict__ out,
                                                           const int* __restrict__ pos,
                                                           const float* __restrict__ w, int T_tok,
                                                           int H, int k,
                                                           __nv_bfloat16* __restrict__ y, int seg,
                                                           const __nv_bfloat16* __restrict__ residual) {
  const int lane = threadIdx.x & 31;
  const int vecs = H >> 3;
  int t, sg, v0, v1;
  row_segment(vecs, seg, t, sg, v0, v1);
  if (t >= T_tok) return;
  int p[kMaxK];
  float wt[kMaxK];
  for (int j = 0; j < k; ++j) {
    p[j] = pos[static_cast<size_t>(t) * k + j];
    wt[j] = w[static_cast<size_t>(t) * k + j];
  }
  for (int v = v0 + lane; v < v1; v += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (residual) unpack8(ld_nc_v4(residual + static_cast<size_t>(t) * H + 8 * v), acc);  // y = x + sum
    for (int j = 0; j < k; ++j) {
      float f[8];
      unpack8(ld_nc_v4(out + static_cast<size_t>(p[j]) * H + 8 * v), f);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(wt[j], f[i], acc[i]);
    }
    st_v4(y + static_cast<size_t>(t) * H + 8 * v, pack8(acc));
  }
}

__global__ void __launch_bounds__(256) combine_f32_kernel(const float* __restrict__ out,
                                                          const int* __restrict__ pos,
                                                          const float* __restrict__ w, int T_tok,
                                                          int H, int k, float* __restrict__ y, int seg,
                                                          const float* __restrict__ residual) {
  const int lane = threadIdx.x & 31;
  const int vecs = H >> 2;
  int t, sg, v0, v1;
  row_segment(vecs, seg, t, sg, v0, v1);
  if (t >= T_tok) return;
  int p[kMaxK];
  float wt[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) {  // fully unrolled + guarded: p and wt stay in registers
    if (j < k) {
      p[j] = pos[static_cast<size_t>(t) * k + j];
      wt[j] = w[static_cast<size_t>(t) * k + j];
    }
  }
  for (int v = v0 + lane; v < v1; v += 32) {
    float4 acc = residual ? reinterpret_cast<const float4*>(residual + static_cast<size_t>(t) * H)[v]
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < kMaxK; ++j) {
      if (j >= k) break;
      const uint4 r = ld_nc_v4(out + static_cast<size_t>(p[j]) * H + 4 * v);
      acc.x = fmaf(wt[j], __uint_as_float(r.x), acc.x);
      acc.y = fmaf(wt[j], __uint_as_float(r.y), acc.y);
      acc.z = fmaf(wt[j], __uint_as_float(r.z), acc.z);
      acc.w = fmaf(wt[j], __uint_as_float(r.w), acc.w);
    }
    reinterpret_cast<float4*>(y + static_cast<size_t>(t) * H)[v] = acc;
  }
}

}  // namespace

cudaError_t launch_gate(DType dt, const void* x, const void* wg_t, int T, int H, int E, int k,
                        const int* dest_of_owner, int experts_per_gpu, int NK, int* topk_idx,
                        float* topk_w, int* keys, int* ranks, int* chunk_counts,
                        cudaStream_t stream) {
  if (E > kMaxE || k > kMaxK || k > E || T <= 0) return cudaErrorInvalidValue;
  if (dt == DType::BF16) {
    // wg_t is bf16 [E, H] for bf16 layers.
    if (H % kGCMin || E % 8 || NK > kMaxNK || k > kMaxK) return cudaErrorInvalidValue;
    const char* gate_env = std::getenv("HEP_GATE");
    if (!(gate_env && gate_env[0] == 'm') && H % kUGK == 0 && E <= 64 && NK <= kMaxNK && k <= kMaxK) {
      // tensor-core gate; TMA descriptors cached per (pointer, shape)
      struct MapCache { const void* p = nullptr; int rows = 0, cols = 0, box = 0; CUtensorMap m; };
      static MapCache xc[4], wc[2];
      static int xnext = 0;
      static std::mutex mu;  // layers may be driven from several host threads
      std::lock_guard<std::mutex> lock(mu);
      auto get = [](MapCache* c, int n, int* next, const void* ptr, int rows, int cols, int box) -> const CUtensorMap* {
        for (int i = 0; i < n; ++i)
          if (c[i].p == ptr && c[i].rows == rows && c[i].cols == cols && c[i].box == box) return &c[i].m;
        MapCache& e = c[next ? (*next)++ % n : 0];
        if (make_tmap_bf16_2d(&e.m, ptr, rows, cols, box, kUGK) != cudaSuccess) return nullptr;
        e.p = ptr; e.rows = rows; e.cols = cols; e.box = box;
        return &e.m;
      };
      const int NE = E <= 16 ? 16 : 64;
      const CUtensorMap* mx = get(xc, 4, &xnext, x, T, H, kUGT);
      const CUtensorMap* mw = get(wc, 1, nullptr, wg_t, E, H, NE);
      if (!mx || !mw) return cudaErrorInvalidValue;
      const int tiles = (T + kUGT - 1) / kUGT;
      // HEP_GATE_SPLIT=1: split K over a CTA pair (DSMEM hand-off of the partial logits).
      // Measured no faster for cfg3 and slower for cfg4 (profiles/README.md), so off.
      const char* split_env = std::getenv("HEP_GATE_SPLIT");
      const bool split = split_env && split_env[0] == '1' && (H / kUGK) % 2 == 0;
      auto launch = [&](auto kern, size_t smem, int ks, DeviceOnce& attr) {
        if (!attr.done()) {
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
          attr.set();
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(tiles * ks));
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(ks);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, *mx, *mw, T, H, E, k, dest_of_owner, experts_per_gpu, NK, topk_idx,
                                  topk_w, keys, ranks, chunk_counts);
      };
      static DeviceOnce a[4];
      cudaError_t err;
      if (NE == 16)
        err = split ? launch(gate_umma_kernel<16, 2>, gate_umma_smem<16, 2>(), 2, a[0])
                    : launch(gate_umma_kernel<16, 1>, gate_umma_smem<16, 1>(), 1, a[1]);
      else
        err = split ? launch(gate_umma_kernel<64, 2>, gate_umma_smem<64, 2>(), 2, a[2])
                    : launch(gate_umma_kernel<64, 1>, gate_umma_smem<64, 1>(), 1, a[3]);
      if (err != cudaSuccess) return err;
      return cudaGetLastError();
    }
    const int blocks = (T + kGT - 1) / kGT;
    auto go = [&](auto kern, size_t smem, DeviceOnce& attr) {
      if (!attr.done()) {  // once per instantiation
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        attr.set();
      }
      kern<<<blocks, 256, smem, stream>>>(static_cast<const __nv_bfloat16*>(x),
                                          static_cast<const __nv_bfloat16*>(wg_t), T, H, E, k, dest_of_owner,
                                          experts_per_gpu, NK, topk_idx, topk_w, keys, ranks, chunk_counts);
      return cudaSuccess;
    };
    static DeviceOnce a8, a8w, a16, a64;
    cudaError_t e;
    if (E <= 8 && H % 128 == 0) e = go(gate_mma_kernel<4, 8, 128>, gate_smem<4, 8, 128>(), a8w);
    else if (E <= 8) e = go(gate_mma_kernel<8, 8, 64>, gate_smem<8, 8, 64>(), a8);
    else if (E <= 16) e = go(gate_mma_kernel<8, 16, 64>, gate_smem<8, 16, 64>(), a16);
    else e = go(gate_mma_kernel<4, kMaxE, 64>, gate_smem<4, kMaxE, 64>(), a64);
    if (e != cudaSuccess) return e;
  } else {
    const int nchunks = (T + kChunk - 1) / kChunk;
    // few chunks: split each chunk's columns over a cluster of 4 (or 2) CTAs
    int cs = 1;
    if (nchunks * 4 <= 2 * 148 && H % 16 == 0) cs = 4;
    else if (nchunks * 2 <= 2 * 148 && H % 8 == 0) cs = 2;
    const size_t smem = static_cast<size_t>(kChunk + E) * (H / cs + 4) * sizeof(float);
    if (H % 4 == 0 && smem <= 200 * 1024 && NK <= kMaxNK && k <= kMaxK && E % 8 == 0) {
      auto go = [&](auto kern, int csz, DeviceOnce& attr) {
        if (!attr.done()) {
          const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
          if (e != cudaSuccess) return e;
          attr.set();
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(nchunks * csz));
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = static_cast<unsigned>(csz);
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, static_cast<const float*>(x), static_cast<const float*>(wg_t), T, H, E,
                                  k, dest_of_owner, experts_per_gpu, NK, topk_idx, topk_w, keys, ranks, chunk_counts);
      };
      static DeviceOnce a1, a2, a4;
      const cudaError_t e = cs == 4   ? go(gate_f32_oneshot_kernel<4>, 4, a4)
                            : cs == 2 ? go(gate_f32_oneshot_kernel<2>, 2, a2)
                                      : go(gate_f32_oneshot_kernel<1>, 1, a1);
      if (e != cudaSuccess) return e;
    } else {
      gate_kernel<float><<<nchunks, 256, 0, stream>>>(static_cast<const float*>(x), static_cast<const float*>(wg_t),
                                                      T, H, E, k, dest_of_owner, experts_per_gpu, NK, topk_idx,
                                                      topk_w, keys, ranks, chunk_counts);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_chunk_scan(const int* chunk_counts, int nchunks, int NK, int* chunk_off,
                              int* key_total, cudaStream_t stream) {
  const int threads = nchunks >= 1024 ? 1024 : ((nchunks + 31) / 32) * 32;
  chunk_scan_kernel<<<NK, threads, 0, stream>>>(chunk_counts, nchunks, NK, chunk_off, key_total);
  return cudaGetLastError();
}

cudaError_t launch_key_scan(const int* key_total, int G, int E, int self,
                            const int* slot_of_expert, int* key_off, int* dest_rows,
                            int* dest_off, int* g_row_start, int* g_rows, int* g_slot,
                            cudaStream_t stream) {
  key_scan_kernel<<<1, 1024, 0, stream>>>(key_total, G, E, self, slot_of_expert, key_off,
                                          dest_rows, dest_off, g_row_start, g_rows, g_slot);
  return cudaGetLastError();
}

cudaError_t launch_permute(DType dt, const void* x, int T, int H, int k, int NK, const int* keys,
                           const int* ranks, const int* chunk_off, const int* key_off, int* pos,
                           void* packed, cudaStream_t stream) {
  const int row_bytes = H * dtype_bytes(dt);
  if (row_bytes % 16) return cudaErrorInvalidValue;
  if (T == 0) return cudaSuccess;
  const int seg = row_segments(T, row_bytes >> 4);
  const int blocks = (T * seg + 7) / 8;
  permute_kernel<<<blocks, 256, 0, stream>>>(static_cast<const uint8_t*>(x), T, row_bytes, k, NK,
                                             keys, ranks, chunk_off, key_off, pos,
                                             static_cast<uint8_t*>(packed), seg);
  return cudaGetLastError();
}

cudaError_t launch_positions(int T, int k, int NK, const int* keys, const int* ranks, const int* chunk_off,
                             const int* key_off, int* pos, cudaStream_t stream, int* src) {
  if (T == 0) return cudaSuccess;
  const int n = T * k + (src ? 256 : 0);
  positions_kernel<<<(n + 255) / 256, 256, 0, stream>>>(T, k, NK, keys, ranks, chunk_off, key_off, pos, src);
  return cudaGetLastError();
}

cudaError_t launch_combine(DType dt, const void* out, const int* pos, const float* topk_w, int T,
                           int H, int k, void* y, cudaStream_t stream, const void* residual) {
  if (T == 0) return cudaSuccess;
  const int seg = row_segments(T, H * dtype_bytes(dt) / 16);
  const int blocks = (T * seg + 7) / 8;
  if (dt == DType::BF16) {
    if (H % 8) return cudaErrorInvalidValue;
    combine_bf16_kernel<<<blocks, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(out), pos,
                                                    topk_w, T, H, k,
                                                    static_cast<__nv_bfloat16*>(y), seg,
                                                    static_cast<const __nv_bfloat16*>(residual));
  } else {
    if (H % 4) return cudaErrorInvalidValue;
    combine_f32_kernel<<<blocks, 256, 0, stream>>>(static_cast<const float*>(out), pos, topk_w, T,
                                                   H, k, static_cast<float*>(y), seg,
                                                   static_cast<const float*>(residual));
  }
  return cudaGetLastError();
}


// Loads every kernel of this file now (see preload_kernels in kernels.h).
cudaError_t preload_route_kernels() {
  auto load = [](const void* fn) {
    cudaFuncAttributes attr;
    return cudaFuncGetAttributes(&attr, fn);
  };
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_kernel<float>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_mma_kernel<4, 8, 128>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_mma_kernel<8, 8, 64>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_mma_kernel<8, 16, 64>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_mma_kernel<4, kMaxE, 64>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_f32_oneshot_kernel<1>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_f32_oneshot_kernel<2>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_f32_oneshot_kernel<4>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_umma_kernel<16, 1>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_umma_kernel<16, 2>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_umma_kernel<64, 1>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(gate_umma_kernel<64, 2>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(chunk_scan_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(key_scan_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(permute_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(positions_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(combine_bf16_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(combine_f32_kernel))) return e;
  return cudaSuccess;
}

cudaError_t preload_kernels() {
  static DeviceOnce once;
  if (once.done()) return cudaSuccess;
  for (cudaError_t (*f)() : {preload_route_kernels, preload_gemm_sm100_kernels, preload_gemm_f32_kernels,
                             preload_sr_codec_kernels, preload_comm_p2p_kernels})
    if (const cudaError_t e = f()) return e;
  once.set();
  return cudaSuccess;
}

}  // namespace hep
