// Launchers for the sm_100a kernels (internal C++ interface; the public boundary is
// the C-ABI in include/hep.h).  All launchers are asynchronous on `stream` and
// return the launch status.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hep {

enum class DType : int { F32 = 0, BF16 = 1 };

// One-time per-device setup (kernel attributes such as the dynamic shared memory limit
// are per device, and one process may drive several devices): done() / set() refer to
// the calling thread's current device.
struct DeviceOnce {
  unsigned long long mask = 0;
  static int device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  bool done() const { return (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) >> device()) & 1ull; }
  void set() { __atomic_fetch_or(&mask, 1ull << device(), __ATOMIC_RELEASE); }
};

inline int dtype_bytes(DType t) { return t == DType::F32 ? 4 : 2; }

// Lazy module loading (CUDA 12's default) loads a kernel at its first launch and may
// synchronise the context to do so.  The peer-memory step has kernels that spin until
// another rank's kernel runs; with several ranks in one context (virtual ranks) a first
// launch behind such a spin would wait for it forever.  preload_kernels() loads every
// kernel of the library up front (once per device, at layer creation).
cudaError_t preload_kernels();
cudaError_t preload_comm_p2p_kernels();
cudaError_t preload_gemm_f32_kernels();
cudaError_t preload_gemm_sm100_kernels();
cudaError_t preload_route_kernels();
cudaError_t preload_sr_codec_kernels();

// ----------------------------------------------------------------- routing (route.cu)
// Gate + top-k + per-32-token-chunk stable ranking.  x:[T,H] (dtype).  Outputs per (t, j): expert, weight, key =
// dest*E + e, rank of (t, j) among earlier tokens of its 32-token chunk with the same
// key; chunk_counts:[ceil(T/32), NK] with NK = G*E.  wg_t: [E, H] in the layer dtype (bf16
// layers route with bf16 gate weights on the tensor cores, fp32 layers with FFMA).
cudaError_t launch_gate(DType dt, const void* x, const void* wg_t, int T, int H, int E, int k,
                        const int* dest_of_owner, int experts_per_gpu, int NK, int* topk_idx,
                        float* topk_w, int* keys, int* ranks, int* chunk_counts,
                        cudaStream_t stream);

// Column-wise exclusive scan of chunk_counts -> chunk_off, and key_total[NK].
cudaError_t launch_chunk_scan(const int* chunk_counts, int nchunks, int NK, int* chunk_off,
                              int* key_total, cudaStream_t stream);

// Exclusive scan of key_total -> key_off; per-destination row counts/offsets
// (dest_rows[G], dest_off[G]); and the local GEMM group table for destination
// `self`: groups are the experts e with slot_of_expert[e] >= 0, in expert order.
cudaError_t launch_key_scan(const int* key_total, int G, int E, int self,
                            const int* slot_of_expert, int* key_off, int* dest_rows,
                            int* dest_off, int* g_row_start, int* g_rows, int* g_slot,
                            cudaStream_t stream);

// pos[t*k+j] = key_off[key] + chunk_off[chunk, key] + rank; packed[pos] = x[t].
cudaError_t launch_permute(DType dt, const void* x, int T, int H, int k, int NK, const int* keys,
                           const int* ranks, const int* chunk_off, const int* key_off, int* pos,
                           void* packed, cudaStream_t stream);

// pos only (no row movement): the routing-plan entry point.  With src: also the inverse
// map src[pos[t, j]] = t, for the GEMM's gathered A load (permute fused into the GEMM).
cudaError_t launch_positions(int T, int k, int NK, const int* keys, const int* ranks, const int* chunk_off,
                             const int* key_off, int* pos, cudaStream_t stream, int* src = nullptr);

// y[t] = sum_j w[t,j] * out[pos[t,j]]  (slot order, fp32 accumulate); with residual:
// y[t] = residual[t] + that sum, accumulated from the residual (one rounding at the end).
cudaError_t launch_combine(DType dt, const void* out, const int* pos, const float* topk_w, int T,
                           int H, int k, void* y, cudaStream_t stream, const void* residual = nullptr);

// ----------------------------------------------------------------- expert GEMM
struct GroupTable {
  const int* row_start;  // first row of the group in A (and in C)
  const int* rows;       // rows in the group
  const int* slot;       // weight slot: B rows [slot*N, slot*N + N)
  int num_groups;
  // Optional per-group output address (bf16 row 0 of the group, row stride ldc): lets the
  // down-projection write rows that came from another GPU straight back into that
  // GPU's output buffer over NVLink.  nullptr: C + row_start*ldc.
  const unsigned long long* out = nullptr;
  // Optional dispatch gating (NVLink path): before loading a tile of group g with
  // wait_src[g] >= 0, the TMA producer waits until wait_flags[wait_src[g]] reaches
  // `epoch` (that source's rows have landed in this GPU's receive area), so the GEMM
  // starts on local rows while remote rows are still in flight.
  const int* wait_src = nullptr;
  const uint32_t* wait_flags = nullptr;
  uint32_t epoch = 0;
  uint64_t timeout_ns = 0;  // dispatch waits trap after this long (0: wait forever)
};

// bf16 tcgen05 grouped GEMM (gemm_sm100.cu): C[r, n] = act(sum_k A[r,k] B[slot*N+n, k]).
// A:[*, K] bf16 row-major, B:[slots*N, K] bf16 (K-major), C:[*, ldc] bf16.
cudaError_t make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                              uint32_t box_rows, uint32_t box_cols);
// sched: bits 0-1 L2 policy of A, 2-3 of B (0 normal, 1 evict_first, 2 evict_last),
// bits 4-5 raster (0 m-fastest, 1 n-fastest, 2 super-rows of bits 8-15 m-tiles).
cudaError_t launch_grouped_gemm_bf16(const CUtensorMap& map_a, const CUtensorMap& map_b, void* C,
                                     int ldc, int N, int K, const GroupTable& groups, int relu,
                                     int num_sms, cudaStream_t stream, uint32_t sched = 0x8u);
// SR decode fused into the B-operand load (1-CTA kernel + converter warp).  A migrated
// expert's residuals are pre-sorted (sr_patch_index) into one 2 KB block per B stage of the
// GEMM -- (n-tile, k-block) of the up [m x h] or down [h x m] compute layout -- holding the
// patched bf16 values and their byte offsets inside the 128-byte-swizzled B tile.  The
// TMA producer stages the block with the tile; the converter warp applies it from shared
// memory.  Entries beyond a block's capacity go to an overflow list (rare; read from global).
constexpr int kPatchBlockBytes = 2048;
constexpr int kPatchBlockCap = kPatchBlockBytes / 4 - 4;  // words after a 16-byte header
struct PatchRef {
  const uint8_t* blocks[2];   // up, down: [n_tiles][num_kb] blocks of kPatchBlockBytes
  const uint2* ovf;           // (block id | half << 31, word) pairs
  const int* ovf_count;
  const int32_t* status;      // the wire's decode status (the layer raises a rejected wire)
};
// Where the GEMM finds slot s's blocks without a dependent load: base + s * slot_bytes +
// half_bytes (0 for the up half); patches[s] is read only for an overflowed block.
struct PatchArgs {
  const uint8_t* base;
  size_t slot_bytes, half_bytes;
  const PatchRef* patches;
};
#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t patch_blocks(int64_t N, int64_t K) { return ((N + 255) / 256) * (K / 64); }
// B = the shared expert's compute copy (map_shared_b: the up [m x h] or down [h x m] half,
// box 256 x 64); half = 0 for the up-projection, 1 for the down-projection.
cudaError_t launch_grouped_gemm_bf16_patched(const CUtensorMap& map_a, const CUtensorMap& map_shared_b, void* C,
                                             int ldc, int N, int K, const GroupTable& groups, const PatchArgs& patches,
                                             int half, int relu, int num_sms, cudaStream_t stream,
                                             uint32_t sched = 0x8u);
// The same on the CTA pair (map_shared_b box 128 x 64).
cudaError_t launch_grouped_gemm_bf16_2cta_patched(const CUtensorMap& map_a, const CUtensorMap& map_shared_b, void* C,
                                                  int ldc, int N, int K, const GroupTable& groups,
                                                  const PatchArgs& patches, int half, int relu, int num_sms,
                                                  cudaStream_t stream, uint32_t sched = 0x6u);
// CTA-pair variant (cta_group::2, 256x256 cluster tiles); B's tensor map box is 128 rows.
// tile_counter (one device int per in-flight launch, zeroed by the launcher) selects the
// dynamic tile scheduler (5-stage kernel); nullptr: the static round-robin.
// a_src != nullptr: A rows are gathered from a_x (the layer input, row stride K; map_a
// unused): grouped row p is a_x row a_src[p], the permute fused into the A load.  a_src
// must hold 256 valid row ids past the last group's rows.  Local outputs, no dispatch
// waits.
cudaError_t launch_grouped_gemm_bf16_2cta(const CUtensorMap& map_a, const CUtensorMap& map_b, void* C, int ldc,
                                          int N, int K, const GroupTable& groups, int relu, int num_sms,
                                          cudaStream_t stream, uint32_t sched = 0x6u, int* tile_counter = nullptr,
                                          const int* a_src = nullptr, const void* a_x = nullptr);
// CTA-pair GEMM unless HEP_GEMM_2CTA=0 (the 1-CTA kernel stays for A/B comparisons).
bool gemm_use_cta_pair();
// Schedule for one expert GEMM shape: A operand reused across n-tiles is kept in L2
// (evict_last) when one expert's A fits, otherwise super-row rasterisation.  The
// HEP_GEMM_SCHED_UP / HEP_GEMM_SCHED_DOWN environment variables override (hex).
uint32_t gemm_schedule(int rows_per_expert, int N, int K, bool up);

// fp32 SIMT grouped GEMM (gemm_f32.cu), same contract with fp32 operands.
// Warps per row for the row kernels (permute / combine): one per token once the tokens
// alone fill the GPU (148 SMs x 64 warps), else up to one per 512 bytes of the row.
inline int row_segments(int T, int vecs) {
  constexpr int kTargetWarps = 148 * 64;
  if (T <= 0 || T >= kTargetWarps) return 1;
  const int want = (kTargetWarps + T - 1) / T, most = (vecs + 31) / 32;
  return want < most ? want : (most > 0 ? most : 1);
}

// K-extent (fp32 columns) of one 3xTF32 pipeline stage; tensor maps of its operands use
// this box width (32: 128-byte swizzle, 2 stages of 96 KB; 16: 64-byte swizzle, 4 stages
// of 48 KB -- 3% faster on cfg1, profiles/README.md).
constexpr int kTf32BK = 16;
// fp32 layers on the tensor cores: 3xTF32 (gemm_sm100.cu).  Operands come as hi/lo tf32
// pairs (launch_split_tf32); C_lo != nullptr stores the ReLU'd result split the same way.
cudaError_t make_tmap_f32_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                             uint32_t box_cols);
// ksplit > 1: split-K over ksplit parts into `partial` ([ksplit][rows_total][ldc]) and an
// in-order reduce (small-M layers, where tiles alone do not fill the SMs).
// b_lo == nullptr: b_hi maps the raw fp32 B, split into hi/lo in shared memory.
cudaError_t launch_grouped_gemm_tf32x3(const CUtensorMap& a_hi, const CUtensorMap& a_lo, const CUtensorMap& b_hi,
                                       const CUtensorMap* b_lo, float* C, float* C_lo, int ldc, int N, int K,
                                       const GroupTable& groups, int relu, int num_sms, cudaStream_t stream,
                                       int ksplit = 1, float* partial = nullptr, int64_t rows_total = 0);
cudaError_t launch_split_tf32(const float* in, float* hi, float* lo, int64_t n, cudaStream_t stream);

cudaError_t launch_grouped_gemm_f32(const float* A, int lda, const float* B, float* C, int ldc,
                                    int N, int K, const GroupTable& groups, int relu,
                                    int num_blocks, cudaStream_t stream);

// ----------------------------------------------------------------- SR codec (sr_codec.cu)
struct SrPlan {
  int64_t h, m;           // w_up is h x m, w_down is m x h
  int64_t total;          // P = 2 h m
  int64_t k, k_up, k_down;
  int per_matrix;
  uint32_t index_bits, value_bits;
  size_t wire_bytes;
};

constexpr int kMaxSrBatch = 64;
size_t sr_workspace_bytes(int64_t h, int64_t m, int batch);
// Encodes `batch` experts (same shape, same shared expert) in one launch sequence.
// grads != nullptr: the optimizer step fused with the encode (fp32 masters only): every
// master becomes fmaf(-lr, grad, master) and the wire encodes that stepped value; the
// split pass (the encode's one full read) applies and writes back the step when every
// range is list-selected, else a separate step kernel runs first.
cudaError_t launch_sr_encode_batch(DType expert_dt, const void* const* experts, int batch, const float* shared,
                                   const SrPlan& plan, uint8_t* const* wires, void* workspace,
                                   cudaStream_t stream, const float* const* grads = nullptr, float lr = 0.f);
// The unfused optimizer step: masters[b] = fmaf(-lr, grads[b], masters[b]) over P elements.
cudaError_t launch_sgd_step_batch(float* const* masters, const float* const* grads, int batch, int64_t P, float lr,
                                  cudaStream_t stream);
// Validates each wire (status int32[4] per wire: code, failing entry, scratch) and writes
// out_b = shared + residual_b (fp32).
cudaError_t launch_sr_decode_batch(const uint8_t* const* wires, int batch, size_t wire_bytes, const float* shared,
                                   int64_t h, int64_t m, float* const* outs, int32_t* status, cudaStream_t stream);
// Decode directly into the compute layout used by the GEMM (w_up^T [m][h], w_down^T
// [h][m]) in out_dt; shared_c is the shared expert already in that layout/dtype.
cudaError_t launch_sr_decode_layout_batch(const uint8_t* const* wires, int batch, size_t wire_bytes,
                                          const float* shared, const void* shared_c, DType out_dt, int64_t h,
                                          int64_t m, void* const* up, void* const* down, int32_t* status,
                                          cudaStream_t stream);
// The fused decode's index pass over `batch` gathered wires: validates each wire like the
// decode (status int32[4] per wire) and sorts its entries into the per-stage patch blocks
// (PatchRef layout; blocks[b] = up blocks then down blocks, ovf[b] / ovf_count[b] the
// overflow) with the final bf16 values bf16((float)((double)shared[i] + v)).
cudaError_t launch_sr_patch_index(const uint8_t* const* wires, int batch, size_t wire_bytes, const float* shared,
                                  int64_t h, int64_t m, uint8_t* const* blocks, uint2* const* ovf,
                                  int* const* ovf_count, int32_t* status, cudaStream_t stream);
// err := (code | entry << 8) of the first failed wire of a decode batch, if err is still 0.
cudaError_t launch_sr_status_fold(const int32_t* status, int n, int32_t* err, cudaStream_t stream);
// out = mean over experts (fp64 accumulate in list order, times 1/n, round to fp32).
cudaError_t launch_shared_mean(DType dt, const void* const* experts, int n, int64_t P, float* out,
                               cudaStream_t stream);

// Reference-layout matrix [rows, cols] (fp32 or bf16) -> compute layout [cols, rows] in `out_dt`.
cudaError_t launch_transpose_convert(DType in_dt, const void* in, int64_t rows, int64_t cols,
                                     DType out_dt, void* out, cudaStream_t stream);

}  // namespace hep
