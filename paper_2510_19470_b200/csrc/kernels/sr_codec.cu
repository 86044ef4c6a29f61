// K5/K6/K7: parameter-efficient expert migration on the GPU, bit-exact with the
// reference CPU codec (proj/src/sparsecomp.cpp).
//
// Encode (K5, "pack"), reference sparsecomp.cpp:175-224:
//   r_i = (double)expert_i - (double)shared_i over the flat index (w_up then w_down);
//   keep the k entries ranked by (|r| desc, index asc) -- the reference's
//   nth_element order (:44-62) -- emitted in ascending index order as SRC1 wire
//   entries (index, value) with value = (float)r for 32-bit wires (:26-28).
//   GPU algorithm: key = IEEE bits of |r| (monotone for non-negative doubles);
//   MSB-first radix select with 12-bit digits (block-private shared-memory
//   histograms, early exit once the threshold bucket is exactly consumed) finds
//   the threshold prefix T and how many key==T ties to take; then ONE ordered
//   stream compaction with a decoupled look-back scan writes the entries already
//   sorted by index (no sort pass), taking ties lowest-index first.
// Decode (K6, "unpack"), :226-246: out = shared, then out[i] = (float)((double)
//   shared[i] + v) for every entry; entries are validated in parallel and the
//   first failing entry (lowest j) decides the error code, like the reference's
//   sequential loop.  Copy and scatter are fused in one pass over the output.
// Shared mean (K7), :147-168: fp64 sum over experts in list order, times (1/n).
// All fp64 arithmetic uses explicit _rn intrinsics so no FMA contraction can
// change a rounding.

#include "common.cuh"
#include "kernels.h"

namespace hep {

namespace {

constexpr int kDigitBits = 12;
constexpr int kBins = 1 << kDigitBits;
constexpr int kPasses = 6;
__constant__ int c_shift[kPasses] = {51, 39, 27, 15, 3, 0};
__constant__ int c_width[kPasses] = {12, 12, 12, 12, 12, 3};

constexpr int kTileThreads = 256;
constexpr int kPerThread = 16;
constexpr int kTile = kTileThreads * kPerThread;  // 4096 elements per compaction tile
constexpr int kMaxTilesPerRange = 1 << 20;

struct SelState {
  unsigned long long prefix;
  unsigned long long mask;
  long long need;
  int done;
  int ticket;
  unsigned int hist[kBins];
};

struct Workspace {
  SelState sel[2];                                   // one per range (w_up / w_down or joint)
  unsigned long long status[2][kMaxTilesPerRange];   // look-back words
};

__device__ __forceinline__ double residual_at(const void* expert, bool bf16, const float* shared,
                                              int64_t i) {
  const double e = bf16 ? static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(expert)[i]))
                        : static_cast<double>(static_cast<const float*>(expert)[i]);
  return __dsub_rn(e, static_cast<double>(shared[i]));
}

__device__ __forceinline__ unsigned long long key_of(double r) {
  return static_cast<unsigned long long>(__double_as_longlong(fabs(r)));
}

__device__ __forceinline__ void put_u32(uint8_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }

__global__ void sr_init_kernel(Workspace* ws, int64_t n0, int64_t k0, int64_t n1, int64_t k1,
                               uint8_t* wire, int64_t h, int64_t m, int64_t k_total,
                               uint32_t iw, uint32_t vw) {
  const int t = threadIdx.x;
  for (int r = 0; r < 2; ++r) {
    SelState& s = ws->sel[r];
    const int64_t n = r ? n1 : n0, k = r ? k1 : k0;
    for (int b = t; b < kBins; b += blockDim.x) s.hist[b] = 0;
    if (t == 0) {
      s.prefix = 0;
      s.mask = 0;
      s.need = k >= n ? n : k;
      s.done = (k <= 0 || k >= n) ? 1 : 0;
      s.ticket = 0;
    }
  }
  if (t == 0) {
    wire[0] = 'S'; wire[1] = 'R'; wire[2] = 'C'; wire[3] = '1';
    put_u32(wire + 4, static_cast<uint32_t>(h));
    put_u32(wire + 8, static_cast<uint32_t>(m));
    put_u32(wire + 12, static_cast<uint32_t>(static_cast<uint64_t>(k_total)));
    put_u32(wire + 16, static_cast<uint32_t>(static_cast<uint64_t>(k_total) >> 32));
    put_u32(wire + 20, iw);
    put_u32(wire + 24, vw);
  }
}

// Histogram of the current digit over elements whose key matches the prefix.
__global__ void __launch_bounds__(256) sr_hist_kernel(const void* expert, int bf16,
                                                      const float* __restrict__ shared, int64_t lo,
                                                      int64_t hi, Workspace* ws, int range,
                                                      int pass) {
  SelState& s = ws->sel[range];
  if (s.done) return;
  __shared__ unsigned int sh[kBins];
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const unsigned long long mask = s.mask, prefix = s.prefix;
  const int shift = c_shift[pass];
  const unsigned int dmask = (1u << c_width[pass]) - 1u;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = lo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < hi; i += stride) {
    const unsigned long long key = key_of(residual_at(expert, bf16, shared, i));
    if ((key & mask) == prefix) {
      const unsigned int d = static_cast<unsigned int>(key >> shift) & dmask;
      atomicAdd(&sh[d], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (sh[b]) atomicAdd(&s.hist[b], sh[b]);
}

// One warp: pick the digit bucket holding the need-th largest key.
__global__ void sr_select_kernel(Workspace* ws, int range, int pass) {
  SelState& s = ws->sel[range];
  if (s.done) return;
  const int lane = threadIdx.x;
  const int shift = c_shift[pass];
  const int width = c_width[pass];
  const int nb = 1 << width;
  const int per = (nb + 31) / 32;
  // lane L owns bins [nb - (L+1)*per, nb - L*per) (counting down from the top).
  unsigned long long mine = 0;
  for (int i = 0; i < per; ++i) {
    const int b = nb - 1 - (lane * per + i);
    if (b >= 0) mine += s.hist[b];
  }
  unsigned long long incl = mine;
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  const long long need = s.need;
  const unsigned int hit = __ballot_sync(0xffffffffu, static_cast<long long>(incl) >= need);
  const int owner = __ffs(hit) - 1;  // first lane whose cumulative count reaches need
  if (lane == owner) {
    long long before = static_cast<long long>(incl - mine);
    for (int i = 0; i < per; ++i) {
      const int b = nb - 1 - (lane * per + i);
      if (b < 0) break;
      const long long c = s.hist[b];
      if (before + c >= need) {
        const long long rem = need - before;
        s.prefix |= static_cast<unsigned long long>(b) << shift;
        s.mask |= static_cast<unsigned long long>(nb - 1) << shift;
        s.need = rem;
        if (c == rem || pass == kPasses - 1) s.done = 1;
        break;
      }
      before += c;
    }
  }
  __syncwarp();
  for (int b = lane; b < kBins; b += 32) s.hist[b] = 0;
}

// Ordered compaction of the selected entries of [lo, hi) into the wire.
__global__ void __launch_bounds__(kTileThreads) sr_compact_kernel(
    const void* expert, int bf16, const float* __restrict__ shared, int64_t lo, int64_t hi,
    Workspace* ws, int range, uint8_t* __restrict__ wire, int64_t out_base, uint32_t iw,
    uint32_t vw) {
  SelState& s = ws->sel[range];
  __shared__ int tile_sh;
  __shared__ unsigned int wgt[8], weq[8];
  __shared__ unsigned long long excl_gt_sh, excl_eq_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) tile_sh = atomicAdd(&s.ticket, 1);
  __syncthreads();
  const int tile = tile_sh;
  const int64_t base = lo + static_cast<int64_t>(tile) * kTile + warp * (kPerThread * 32);
  const unsigned long long mask = s.mask, prefix = s.prefix;
  const long long need = s.need;

  double rv[kPerThread];
  unsigned int bgt[kPerThread], beq[kPerThread];
  unsigned int cgt = 0, ceq = 0;
#pragma unroll
  for (int it = 0; it < kPerThread; ++it) {
    const int64_t i = base + it * 32 + lane;
    bool gt = false, eq = false;
    rv[it] = 0.0;
    if (i < hi) {
      rv[it] = residual_at(expert, bf16, shared, i);
      const unsigned long long km = key_of(rv[it]) & mask;
      gt = km > prefix;
      eq = km == prefix;
    }
    bgt[it] = __ballot_sync(0xffffffffu, gt);
    beq[it] = __ballot_sync(0xffffffffu, eq);
    cgt += __popc(bgt[it]);
    ceq += __popc(beq[it]);
  }
  if (lane == 0) { wgt[warp] = cgt; weq[warp] = ceq; }
  __syncthreads();

  unsigned long long* status = ws->status[range];
  if (threadIdx.x == 0) {
    unsigned long long tgt = 0, teq = 0;
    for (int w = 0; w < 8; ++w) { tgt += wgt[w]; teq += weq[w]; }
    constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 31) - 1;
    unsigned long long pgt = 0, peq = 0;
    if (tile == 0) {
      atomicExch(&status[0], kInc | (tgt << 31) | teq);
    } else {
      atomicExch(&status[tile], kAgg | (tgt << 31) | teq);
      for (int t = tile - 1; t >= 0; --t) {
        unsigned long long w;
        do { w = atomicAdd(&status[t], 0ull); } while ((w >> 62) == 0);
        pgt += (w >> 31) & kVal;
        peq += w & kVal;
        if ((w >> 62) == 2) break;
      }
      __threadfence();
      atomicExch(&status[tile], kInc | ((pgt + tgt) << 31) | (peq + teq));
    }
    excl_gt_sh = pgt;
    excl_eq_sh = peq;
  }
  __syncthreads();

  unsigned long long run_gt = excl_gt_sh, run_eq = excl_eq_sh;
  for (int w = 0; w < warp; ++w) { run_gt += wgt[w]; run_eq += weq[w]; }
  const unsigned int lt = (1u << lane) - 1u;
  const int eb = static_cast<int>((iw + vw) / 8);
#pragma unroll
  for (int it = 0; it < kPerThread; ++it) {
    const bool gt = (bgt[it] >> lane) & 1u, eq = (beq[it] >> lane) & 1u;
    const unsigned long long gbefore = run_gt + __popc(bgt[it] & lt);
    const unsigned long long ebefore = run_eq + __popc(beq[it] & lt);
    if (gt || (eq && static_cast<long long>(ebefore) < need)) {
      const unsigned long long taken_eq =
          static_cast<long long>(ebefore) < need ? ebefore : static_cast<unsigned long long>(need);
      const int64_t j = out_base + static_cast<int64_t>(gbefore + taken_eq);
      uint8_t* p = wire + 28 + j * eb;
      const uint64_t idx = static_cast<uint64_t>(base + it * 32 + lane);
      put_u32(p, static_cast<uint32_t>(idx));
      if (iw == 64) { put_u32(p + 4, static_cast<uint32_t>(idx >> 32)); p += 8; } else { p += 4; }
      if (vw == 32) {
        put_u32(p, __float_as_uint(__double2float_rn(rv[it])));
      } else {
        const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(rv[it]));
        put_u32(p, static_cast<uint32_t>(b));
        put_u32(p + 4, static_cast<uint32_t>(b >> 32));
      }
    }
    run_gt += __popc(bgt[it]);
    run_eq += __popc(beq[it]);
  }
}

// ------------------------------------------------------------------ decode
__device__ __forceinline__ uint32_t get_u32(const uint8_t* p) { return *reinterpret_cast<const uint32_t*>(p); }

struct WireView {
  int ok_header;
  uint32_t iw, vw;
  int64_t k;
  int eb;
};

// status[0] = error code (0 ok; 1 bad magic; 2 truncated; 3 widths; 4 shape tag;
//             5 index out of bounds; 6 indices not increasing)
// status[1] = first failing entry (entry-level errors) -- packed as j*8+code in fail slot.
__device__ WireView read_header(const uint8_t* wire, size_t bytes, int64_t h, int64_t m, int* code) {
  WireView v{0, 0, 0, 0, 0};
  *code = 0;
  if (bytes < 4 || wire[0] != 'S' || wire[1] != 'R' || wire[2] != 'C' || wire[3] != '1') { *code = 1; return v; }
  if (bytes < 28) { *code = 2; return v; }
  const int64_t hh = get_u32(wire + 4), mm = get_u32(wire + 8);
  const uint64_t k = static_cast<uint64_t>(get_u32(wire + 12)) | (static_cast<uint64_t>(get_u32(wire + 16)) << 32);
  v.iw = get_u32(wire + 20);
  v.vw = get_u32(wire + 24);
  if ((v.iw != 32 && v.iw != 64) || (v.vw != 32 && v.vw != 64)) { *code = 3; return v; }
  v.eb = static_cast<int>((v.iw + v.vw) / 8);
  if (k > (bytes - 28) / static_cast<uint64_t>(v.eb)) { *code = 2; return v; }
  if (hh != h || mm != m) { *code = 4; return v; }
  v.k = static_cast<int64_t>(k);
  v.ok_header = 1;
  return v;
}

__device__ __forceinline__ uint64_t entry_index(const uint8_t* wire, const WireView& v, int64_t j) {
  const uint8_t* p = wire + 28 + j * v.eb;
  uint64_t idx = get_u32(p);
  if (v.iw == 64) idx |= static_cast<uint64_t>(get_u32(p + 4)) << 32;
  return idx;
}

__device__ __forceinline__ double entry_value(const uint8_t* wire, const WireView& v, int64_t j) {
  const uint8_t* p = wire + 28 + j * v.eb + v.iw / 8;
  if (v.vw == 32) return static_cast<double>(__uint_as_float(get_u32(p)));
  const uint64_t b = static_cast<uint64_t>(get_u32(p)) | (static_cast<uint64_t>(get_u32(p + 4)) << 32);
  return __longlong_as_double(static_cast<long long>(b));
}

__global__ void sr_validate_kernel(const uint8_t* __restrict__ wire, size_t bytes, int64_t h,
                                   int64_t m, int32_t* status, unsigned long long* fail) {
  int code;
  const WireView v = read_header(wire, bytes, h, m, &code);
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (!v.ok_header) {
    if (j == 0) status[0] = code;
    return;
  }
  if (j >= v.k) return;
  const uint64_t P = static_cast<uint64_t>(2 * h * m);
  const uint64_t idx = entry_index(wire, v, j);
  int c = 0;
  if (idx >= P) c = 5;
  else if (j > 0 && idx <= entry_index(wire, v, j - 1)) c = 6;
  if (c) atomicMin(fail, static_cast<unsigned long long>(j) * 8ull + static_cast<unsigned long long>(c));
}

__global__ void sr_status_finalize_kernel(int32_t* status, const unsigned long long* fail) {
  if (status[0] != 0) return;
  const unsigned long long f = *fail;
  if (f != ~0ull) {
    status[0] = static_cast<int32_t>(f & 7ull);
    status[1] = static_cast<int32_t>(f >> 3);
  }
}

constexpr int kDecChunk = 4096;

// Fused copy + scatter: block b owns out[b*4096, (b+1)*4096).
__global__ void __launch_bounds__(256) sr_decode_kernel(const uint8_t* __restrict__ wire, size_t bytes,
                                                        const float* __restrict__ shared, int64_t h,
                                                        int64_t m, float* __restrict__ out) {
  const int64_t P = 2 * h * m;
  const int64_t a = static_cast<int64_t>(blockIdx.x) * kDecChunk;
  const int64_t b = min(P, a + kDecChunk);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) out[i] = shared[i];
  int code;
  const WireView v = read_header(wire, bytes, h, m, &code);
  if (!v.ok_header || v.k == 0) return;
  // First entry with index >= a (entries sorted when the wire is valid).
  __shared__ int64_t first_sh;
  if (threadIdx.x == 0) {
    int64_t lo = 0, hi = v.k;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (entry_index(wire, v, mid) < static_cast<uint64_t>(a)) lo = mid + 1; else hi = mid;
    }
    first_sh = lo;
  }
  __syncthreads();
  for (int64_t j = first_sh + threadIdx.x; j < v.k; j += blockDim.x) {
    const uint64_t idx = entry_index(wire, v, j);
    if (idx >= static_cast<uint64_t>(b)) break;
    out[idx] = __double2float_rn(__dadd_rn(static_cast<double>(shared[idx]), entry_value(wire, v, j)));
  }
}

// ------------------------------------------------------------------ shared mean
struct ExpertPtrs {
  const void* p[64];
};

__global__ void __launch_bounds__(256) shared_mean_kernel(ExpertPtrs ptrs, int n, int bf16, int64_t P,
                                                          double inv, float* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P; i += stride) {
    double acc = 0.0;
    for (int e = 0; e < n; ++e) {
      const double v = bf16 ? static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(ptrs.p[e])[i]))
                            : static_cast<double>(static_cast<const float*>(ptrs.p[e])[i]);
      acc = __dadd_rn(acc, v);
    }
    out[i] = __double2float_rn(__dmul_rn(acc, inv));
  }
}

// ------------------------------------------------------------------ layout conversion
template <typename Tin, typename Tout>
__global__ void transpose_convert_kernel(const Tin* __restrict__ in, int64_t rows, int64_t cols,
                                         Tout* __restrict__ out) {
  __shared__ float tile[32][33];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    float v = 0.f;
    if (r < rows && c < cols) {
      if constexpr (sizeof(Tin) == 4) v = in[r * cols + c];
      else v = __bfloat162float(in[r * cols + c]);
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;  // out[c][r]
    if (r < rows && c < cols) {
      const float v = tile[threadIdx.x][i];
      if constexpr (sizeof(Tout) == 4) out[c * rows + r] = v;
      else out[c * rows + r] = __float2bfloat16_rn(v);
    }
  }
}

}  // namespace

size_t sr_workspace_bytes() { return sizeof(Workspace) + 64; }

cudaError_t launch_sr_encode(DType expert_dt, const void* expert, const float* shared,
                             const SrPlan& plan, void* wire, void* workspace, cudaStream_t stream) {
  Workspace* ws = static_cast<Workspace*>(workspace);
  const int bf16 = expert_dt == DType::BF16;
  const int64_t up = plan.h * plan.m, P = plan.total;
  struct Range { int64_t lo, hi, k, out_base; };
  Range ranges[2];
  int nr;
  if (plan.per_matrix) {
    ranges[0] = {0, up, plan.k_up, 0};
    ranges[1] = {up, P, plan.k_down, plan.k_up};
    nr = 2;
  } else {
    ranges[0] = {0, P, plan.k, 0};
    ranges[1] = {0, 0, 0, 0};
    nr = 1;
  }
  for (int r = 0; r < nr; ++r)
    if ((ranges[r].hi - ranges[r].lo + kTile - 1) / kTile > kMaxTilesPerRange) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(ws->status, 0, sizeof(ws->status), stream);
  if (e != cudaSuccess) return e;
  sr_init_kernel<<<1, 256, 0, stream>>>(ws, ranges[0].hi - ranges[0].lo, ranges[0].k,
                                        ranges[1].hi - ranges[1].lo, ranges[1].k,
                                        static_cast<uint8_t*>(wire), plan.h, plan.m, plan.k,
                                        plan.index_bits, plan.value_bits);
  for (int r = 0; r < nr; ++r) {
    const int64_t n = ranges[r].hi - ranges[r].lo;
    if (n <= 0) continue;
    const int blocks = static_cast<int>(std::min<int64_t>(148 * 4, (n + 255) / 256));
    for (int pass = 0; pass < kPasses; ++pass) {
      sr_hist_kernel<<<blocks, 256, 0, stream>>>(expert, bf16, shared, ranges[r].lo, ranges[r].hi, ws, r, pass);
      sr_select_kernel<<<1, 32, 0, stream>>>(ws, r, pass);
    }
    const int tiles = static_cast<int>((n + kTile - 1) / kTile);
    sr_compact_kernel<<<tiles, kTileThreads, 0, stream>>>(expert, bf16, shared, ranges[r].lo,
                                                           ranges[r].hi, ws, r,
                                                           static_cast<uint8_t*>(wire),
                                                           ranges[r].out_base, plan.index_bits,
                                                           plan.value_bits);
  }
  return cudaGetLastError();
}

cudaError_t launch_sr_decode(const void* wire, size_t wire_bytes, const float* shared, int64_t h,
                             int64_t m, float* out, int32_t* status, cudaStream_t stream) {
  // status: int32[2] followed by (8-byte aligned) the fail word; caller provides 16 bytes.
  unsigned long long* fail = reinterpret_cast<unsigned long long*>(status + 2);
  cudaError_t e = cudaMemsetAsync(status, 0, 8, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(fail, 0xff, 8, stream);
  if (e != cudaSuccess) return e;
  const int64_t kmax = wire_bytes > 28 ? static_cast<int64_t>((wire_bytes - 28) / 8) : 0;
  const int vblocks = static_cast<int>(std::max<int64_t>(1, (kmax + 255) / 256));
  sr_validate_kernel<<<vblocks, 256, 0, stream>>>(static_cast<const uint8_t*>(wire), wire_bytes, h, m,
                                                  status, fail);
  sr_status_finalize_kernel<<<1, 1, 0, stream>>>(status, fail);
  const int64_t P = 2 * h * m;
  const int dblocks = static_cast<int>((P + kDecChunk - 1) / kDecChunk);
  sr_decode_kernel<<<dblocks, 256, 0, stream>>>(static_cast<const uint8_t*>(wire), wire_bytes, shared,
                                                h, m, out);
  return cudaGetLastError();
}

cudaError_t launch_shared_mean(DType dt, const void* const* experts, int n, int64_t P, float* out,
                               cudaStream_t stream) {
  if (n <= 0 || n > 64) return cudaErrorInvalidValue;
  ExpertPtrs ptrs{};
  for (int i = 0; i < n; ++i) ptrs.p[i] = experts[i];
  const int blocks = static_cast<int>(std::min<int64_t>(148 * 8, (P + 255) / 256));
  shared_mean_kernel<<<blocks, 256, 0, stream>>>(ptrs, n, dt == DType::BF16, P, 1.0 / static_cast<double>(n), out);
  return cudaGetLastError();
}

cudaError_t launch_transpose_convert(DType in_dt, const void* in, int64_t rows, int64_t cols,
                                     DType out_dt, void* out, cudaStream_t stream) {
  const dim3 block(32, 8);
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  if (grid.y > 65535) return cudaErrorInvalidValue;
  if (in_dt == DType::F32 && out_dt == DType::F32)
    transpose_convert_kernel<float, float><<<grid, block, 0, stream>>>(static_cast<const float*>(in), rows, cols, static_cast<float*>(out));
  else if (in_dt == DType::F32 && out_dt == DType::BF16)
    transpose_convert_kernel<float, __nv_bfloat16><<<grid, block, 0, stream>>>(static_cast<const float*>(in), rows, cols, static_cast<__nv_bfloat16*>(out));
  else if (in_dt == DType::BF16 && out_dt == DType::BF16)
    transpose_convert_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, block, 0, stream>>>(static_cast<const __nv_bfloat16*>(in), rows, cols, static_cast<__nv_bfloat16*>(out));
  else
    transpose_convert_kernel<__nv_bfloat16, float><<<grid, block, 0, stream>>>(static_cast<const __nv_bfloat16*>(in), rows, cols, static_cast<float*>(out));
  return cudaGetLastError();
}

}  // namespace hep
