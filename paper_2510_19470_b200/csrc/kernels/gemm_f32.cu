// K8 fp32 variant: grouped GEMM with fp32 FFMA (cfg1/cfg2 run the layer in fp32 and
// must match the fp64 oracle to 1e-4 relative, which plain TF32 tensor-core math
// cannot).  Same group-table contract as the tcgen05 kernel:
//   C[r, n] = act( sum_k A[r, k] * B[slot(g) * N + n, k] )
// 128x128 tile per CTA, BK = 8, 256 threads with an 8x8 register micro-tile,
// persistent grid-stride over (group, m-tile, n-tile).

#include "common.cuh"
#include "kernels.h"

namespace hep {

namespace {

constexpr int TM = 128, TN = 128, TK = 8;
constexpr int kMaxGroups = 512;

__global__ void __launch_bounds__(256) grouped_gemm_f32_kernel(
    const float* __restrict__ A, int lda, const float* __restrict__ B, float* __restrict__ C,
    int ldc, int N, int K, const int* __restrict__ g_row_start, const int* __restrict__ g_rows,
    const int* __restrict__ g_slot, int ng, int relu) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  __shared__ int tile_start[kMaxGroups + 1];
  __shared__ int s_rows[kMaxGroups], s_start[kMaxGroups], s_slot[kMaxGroups];

  const int tid = threadIdx.x;
  const int n_tiles = (N + TN - 1) / TN;
  if (tid == 0) {
    int acc = 0;
    for (int g = 0; g < ng; ++g) {
      const int r = g_rows[g];
      s_rows[g] = r;
      s_start[g] = g_row_start[g];
      s_slot[g] = g_slot[g];
      tile_start[g] = acc;
      acc += ((r + TM - 1) / TM) * n_tiles;
    }
    tile_start[ng] = acc;
  }
  __syncthreads();
  const int total = tile_start[ng];
  const int tx = tid & 15, ty = tid >> 4;

  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    int g = 0;
    {
      int lo = 0, hi = ng - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tile_start[mid] <= tile) lo = mid; else hi = mid - 1;
      }
      g = lo;
    }
    const int local = tile - tile_start[g];
    const int m_tiles = (s_rows[g] + TM - 1) / TM;
    const int mt = local % m_tiles, nt = local / m_tiles;
    const int row0 = mt * TM, col0 = nt * TN;
    const int rows = s_rows[g];
    const float* Ag = A + static_cast<size_t>(s_start[g]) * lda;
    const float* Bg = B + static_cast<size_t>(s_slot[g]) * N * K;

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    // Each thread loads one float4 of A and one of B per k-step: row = tid/2, k-half = tid%2.
    const int lr = tid >> 1, lk = (tid & 1) * 4;
    for (int k0 = 0; k0 < K; k0 += TK) {
      {
        const int r = row0 + lr;
        float4 va = make_float4(0.f, 0.f, 0.f, 0.f);
        if (r < rows) va = *reinterpret_cast<const float4*>(Ag + static_cast<size_t>(r) * lda + k0 + lk);
        As[lk + 0][lr] = va.x; As[lk + 1][lr] = va.y; As[lk + 2][lr] = va.z; As[lk + 3][lr] = va.w;
        const int c = col0 + lr;
        float4 vb = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < N) vb = *reinterpret_cast<const float4*>(Bg + static_cast<size_t>(c) * K + k0 + lk);
        Bs[lk + 0][lr] = vb.x; Bs[lk + 1][lr] = vb.y; Bs[lk + 2][lr] = vb.z; Bs[lk + 3][lr] = vb.w;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        float a[8], b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[i] = As[kk][ty * 4 + i];
          a[4 + i] = As[kk][64 + ty * 4 + i];
          b[i] = Bs[kk][tx * 4 + i];
          b[4 + i] = Bs[kk][64 + tx * 4 + i];
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = row0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
      if (r >= rows) continue;
      float* crow = C + static_cast<size_t>(s_start[g] + r) * ldc;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = col0 + h * 64 + tx * 4;
        if (c >= N) continue;
        float4 o;
        o.x = relu ? fmaxf(acc[i][4 * h + 0], 0.f) : acc[i][4 * h + 0];
        o.y = relu ? fmaxf(acc[i][4 * h + 1], 0.f) : acc[i][4 * h + 1];
        o.z = relu ? fmaxf(acc[i][4 * h + 2], 0.f) : acc[i][4 * h + 2];
        o.w = relu ? fmaxf(acc[i][4 * h + 3], 0.f) : acc[i][4 * h + 3];
        *reinterpret_cast<float4*>(crow + c) = o;
      }
    }
  }
}

}  // namespace

cudaError_t launch_grouped_gemm_f32(const float* A, int lda, const float* B, float* C, int ldc,
                                    int N, int K, const GroupTable& groups, int relu,
                                    int num_blocks, cudaStream_t stream) {
  if (K % TK || N % 4 || groups.num_groups > kMaxGroups || groups.num_groups <= 0)
    return cudaErrorInvalidValue;
  grouped_gemm_f32_kernel<<<num_blocks, 256, 0, stream>>>(A, lda, B, C, ldc, N, K, groups.row_start,
                                                          groups.rows, groups.slot,
                                                          groups.num_groups, relu);
  return cudaGetLastError();
}


// Loads every kernel of this file now (see preload_kernels in kernels.h).
cudaError_t preload_gemm_f32_kernels() {
  auto load = [](const void* fn) {
    cudaFuncAttributes attr;
    return cudaFuncGetAttributes(&attr, fn);
  };
  if (const cudaError_t e = load(reinterpret_cast<const void*>(grouped_gemm_f32_kernel))) return e;
  return cudaSuccess;
}

}  // namespace hep
