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

struct SelState {
  unsigned long long prefix;
  unsigned long long mask;
  long long need;
  int done;
  int ticket;
  unsigned long long keyor;  // OR of every key in the range (pass 0): bits that never vary are skipped
  unsigned int hist[kBins];
};

// Workspace of a batch: SelState per (expert, range) followed by the look-back words of
// every (expert, range), `tiles` apiece.
struct WsView {
  SelState* sel;
  unsigned long long* status;
  int64_t tiles;
  __device__ SelState& st(int b, int r) const { return sel[b * 2 + r]; }
  __device__ unsigned long long* stat(int b, int r) const { return status + (static_cast<int64_t>(b) * 2 + r) * tiles; }
};

struct EncBatch {
  const void* expert[kMaxSrBatch];
  uint8_t* wire[kMaxSrBatch];
};

struct DecBatch {
  const uint8_t* wire[kMaxSrBatch];
  float* out[kMaxSrBatch];
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

// Block b: reset the selection state of expert b, zero its look-back words, write its
// SRC1 header.
__global__ void sr_init_kernel(WsView ws, EncBatch batch, int64_t n0, int64_t k0, int64_t n1, int64_t k1,
                               int64_t h, int64_t m, int64_t k_total, uint32_t iw, uint32_t vw) {
  const int b = blockIdx.x, t = threadIdx.x;
  for (int r = 0; r < 2; ++r) {
    SelState& s = ws.st(b, r);
    const int64_t n = r ? n1 : n0, k = r ? k1 : k0;
    for (int i = t; i < kBins; i += blockDim.x) s.hist[i] = 0;
    unsigned long long* st = ws.stat(b, r);
    for (int64_t i = t; i < ws.tiles; i += blockDim.x) st[i] = 0;
    if (t == 0) {
      s.prefix = 0;
      s.mask = 0;
      s.need = k >= n ? n : k;
      s.done = (k <= 0 || k >= n) ? 1 : 0;
      s.ticket = 0;
      s.keyor = 0;
    }
  }
  if (t == 0) {
    uint8_t* wire = batch.wire[b];
    wire[0] = 'S'; wire[1] = 'R'; wire[2] = 'C'; wire[3] = '1';
    put_u32(wire + 4, static_cast<uint32_t>(h));
    put_u32(wire + 8, static_cast<uint32_t>(m));
    put_u32(wire + 12, static_cast<uint32_t>(static_cast<uint64_t>(k_total)));
    put_u32(wire + 16, static_cast<uint32_t>(static_cast<uint64_t>(k_total) >> 32));
    put_u32(wire + 20, iw);
    put_u32(wire + 24, vw);
  }
}

// Residual magnitudes cluster in a few bins, so lanes holding the same digit are merged
// with match.any and one leader adds the population count.
__device__ __forceinline__ void hist_add(unsigned int* sh, int d) {
  const unsigned int peers = __match_any_sync(__activemask(), d);
  if (d >= 0 && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&sh[d], __popc(peers));
}

// Histogram of the current digit over the keys matching the prefix (grid.y = expert).
__global__ void __launch_bounds__(256) sr_hist_kernel(EncBatch batch, int bf16, const float* __restrict__ shared,
                                                      int64_t lo, int64_t hi, WsView ws, int range, int pass) {
  SelState& s = ws.st(blockIdx.y, range);
  if (s.done) return;
  const void* expert = batch.expert[blockIdx.y];
  __shared__ unsigned int sh[kBins];
  for (int b = threadIdx.x; b < kBins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const unsigned long long mask = s.mask, prefix = s.prefix;
  const int shift = c_shift[pass];
  const unsigned int dmask = (1u << c_width[pass]) - 1u;
  unsigned long long kor = 0;
  auto digit = [&](double r) {
    const unsigned long long key = key_of(r);
    kor |= key;
    return (key & mask) == prefix ? static_cast<int>((key >> shift) & dmask) : -1;
  };
  // Vector body over 4-element groups (aligned to the range start), scalar ends.
  const int64_t head_end = min(hi, (lo + 3) & ~static_cast<int64_t>(3));
  const int64_t body_end = head_end + ((hi - head_end) & ~static_cast<int64_t>(3));
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t groups = (body_end - head_end) >> 2;
  for (int64_t gi = tid; gi - (threadIdx.x & 31) < groups; gi += nthreads) {  // warp-uniform trip count
    int d0 = -1, d1 = -1, d2 = -1, d3 = -1;
    if (gi < groups) {
      const int64_t i = head_end + 4 * gi;
      const float4 sv = *reinterpret_cast<const float4*>(shared + i);
      float e0, e1, e2, e3;
      if (bf16) {
        const uint2 raw = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(expert) + i);
        e0 = bf16_lo(raw.x); e1 = bf16_hi(raw.x); e2 = bf16_lo(raw.y); e3 = bf16_hi(raw.y);
      } else {
        const float4 ev = *reinterpret_cast<const float4*>(static_cast<const float*>(expert) + i);
        e0 = ev.x; e1 = ev.y; e2 = ev.z; e3 = ev.w;
      }
      d0 = digit(__dsub_rn(static_cast<double>(e0), static_cast<double>(sv.x)));
      d1 = digit(__dsub_rn(static_cast<double>(e1), static_cast<double>(sv.y)));
      d2 = digit(__dsub_rn(static_cast<double>(e2), static_cast<double>(sv.z)));
      d3 = digit(__dsub_rn(static_cast<double>(e3), static_cast<double>(sv.w)));
    }
    hist_add(sh, d0);
    hist_add(sh, d1);
    hist_add(sh, d2);
    hist_add(sh, d3);
  }
  if (blockIdx.x == 0) {
    for (int64_t i = lo + threadIdx.x; i < head_end; i += blockDim.x) {
      const int d = digit(residual_at(expert, bf16, shared, i));
      if (d >= 0) atomicAdd(&sh[d], 1u);
    }
    for (int64_t i = body_end + threadIdx.x; i < hi; i += blockDim.x) {
      const int d = digit(residual_at(expert, bf16, shared, i));
      if (d >= 0) atomicAdd(&sh[d], 1u);
    }
  }
  if (pass == 0) {
    const unsigned int lo32 = __reduce_or_sync(0xffffffffu, static_cast<unsigned int>(kor));
    const unsigned int hi32 = __reduce_or_sync(0xffffffffu, static_cast<unsigned int>(kor >> 32));
    if ((threadIdx.x & 31) == 0 && (lo32 | hi32))
      atomicOr(&s.keyor, (static_cast<unsigned long long>(hi32) << 32) | lo32);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += blockDim.x)
    if (sh[b]) atomicAdd(&s.hist[b], sh[b]);
}

// Block b (1024 threads): pick the digit bucket of expert b holding the need-th largest key.
__global__ void __launch_bounds__(1024) sr_select_kernel(WsView ws, int range, int pass) {
  SelState& s = ws.st(blockIdx.x, range);
  if (s.done) return;
  __shared__ unsigned long long wsum[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int shift = c_shift[pass], width = c_width[pass], nb = 1 << width;
  const int per = (nb + 1023) / 1024;
  // Thread t owns bins nb-1-(t*per) .. nb-per-(t*per), counting down from the top.
  unsigned long long mine = 0;
  for (int i = 0; i < per; ++i) {
    const int b = nb - 1 - (t * per + i);
    if (b >= 0) mine += s.hist[b];
  }
  unsigned long long incl = mine;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = wsum[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += o;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  if (warp) incl += wsum[warp - 1];
  const long long need = s.need;
  const long long excl = static_cast<long long>(incl - mine);
  if (excl < need && static_cast<long long>(incl) >= need) {  // exactly one owner
    long long before = excl;
    for (int i = 0; i < per; ++i) {
      const int b = nb - 1 - (t * per + i);
      if (b < 0) break;
      const long long c = s.hist[b];
      if (before + c >= need) {
        const long long rem = need - before;
        s.prefix |= static_cast<unsigned long long>(b) << shift;
        s.mask |= static_cast<unsigned long long>(nb - 1) << shift;
        s.need = rem;
        if (c == rem || pass == kPasses - 1) s.done = 1;
        if ((s.keyor & ((1ull << shift) - 1ull)) == 0) {
          // No key has a bit below this digit: the remaining bucket is all ties.
          s.mask = ~0ull;
          s.done = 1;
        }
        break;
      }
      before += c;
    }
  }
  __syncthreads();
  for (int b = t; b < kBins; b += blockDim.x) s.hist[b] = 0;
}

// Ordered compaction of the selected entries of [lo, hi) into the wire (grid.y = expert):
// per-tile counts, decoupled look-back for the tile's global prefix, then ballot ranks.
__global__ void __launch_bounds__(kTileThreads) sr_compact_kernel(EncBatch batch, int bf16,
                                                                  const float* __restrict__ shared, int64_t lo,
                                                                  int64_t hi, WsView ws, int range, int64_t out_base,
                                                                  uint32_t iw, uint32_t vw) {
  const int bexp = blockIdx.y;
  SelState& s = ws.st(bexp, range);
  const void* expert = batch.expert[bexp];
  uint8_t* wire = batch.wire[bexp];
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

  float rv[kPerThread];  // (float)r for 32-bit wires; 64-bit wires recompute r
  unsigned int bgt[kPerThread], beq[kPerThread];
  unsigned int cgt = 0, ceq = 0;
#pragma unroll
  for (int it = 0; it < kPerThread; ++it) {
    const int64_t i = base + it * 32 + lane;
    bool gt = false, eq = false;
    rv[it] = 0.f;
    if (i < hi) {
      const double r = residual_at(expert, bf16, shared, i);
      rv[it] = __double2float_rn(r);
      const unsigned long long km = key_of(r) & mask;
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

  unsigned long long* status = ws.stat(bexp, range);
  if (warp == 0) {
    // Decoupled look-back, a 32-tile window per step (one predecessor per lane): with
    // ~1000 resident tiles a serial walk would chain hundreds of dependent L2 reads.
    constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 31) - 1;
    unsigned long long tgt = 0, teq = 0;
    for (int w = 0; w < 8; ++w) { tgt += wgt[w]; teq += weq[w]; }
    unsigned long long pgt = 0, peq = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(&status[0], kInc | (tgt << 31) | teq);
    } else {
      if (lane == 0) atomicExch(&status[tile], kAgg | (tgt << 31) | teq);
      for (int t0 = tile - 1; t0 >= 0; t0 -= 32) {
        const int t = t0 - lane;
        unsigned long long w = 0;
        if (t >= 0) {
          do { w = *reinterpret_cast<volatile unsigned long long*>(&status[t]); } while ((w >> 62) == 0);
        }
        const unsigned int inc = __ballot_sync(0xffffffffu, t >= 0 && (w >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest predecessor with an inclusive prefix
        unsigned long long g = (t >= 0 && lane <= stop) ? (w >> 31) & kVal : 0;
        unsigned long long e = (t >= 0 && lane <= stop) ? w & kVal : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          g += __shfl_xor_sync(0xffffffffu, g, off);
          e += __shfl_xor_sync(0xffffffffu, e, off);
        }
        pgt += g;
        peq += e;
        if (inc) break;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(&status[tile], kInc | ((pgt + tgt) << 31) | (peq + teq));
      }
    }
    if (lane == 0) {
      excl_gt_sh = pgt;
      excl_eq_sh = peq;
    }
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
        put_u32(p, __float_as_uint(rv[it]));
      } else {
        const double r = residual_at(expert, bf16, shared, static_cast<int64_t>(idx));
        const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(r));
        put_u32(p, static_cast<uint32_t>(b));
        put_u32(p + 4, static_cast<uint32_t>(b >> 32));
      }
    }
    run_gt += __popc(bgt[it]);
    run_eq += __popc(beq[it]);
  }
}

// Vectorised compaction (range start 4-aligned): lane l of a warp handles 4 consecutive
// elements per 128-element step, so the per-element work is a float4 load pair, the key
// test and a nibble of flags; in-warp ranks come from one packed (gt, eq) prefix scan.
__global__ void __launch_bounds__(kTileThreads) sr_compact4_kernel(EncBatch batch, int bf16,
                                                                   const float* __restrict__ shared, int64_t lo,
                                                                   int64_t hi, WsView ws, int range, int64_t out_base,
                                                                   uint32_t iw, uint32_t vw) {
  constexpr int kSteps = kPerThread / 4;  // 4 steps x 128 elements = 512 per warp
  const int bexp = blockIdx.y;
  SelState& s = ws.st(bexp, range);
  const void* expert = batch.expert[bexp];
  uint8_t* wire = batch.wire[bexp];
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

  float rv[kPerThread];
  unsigned int fl[kSteps];  // bits 0-3: gt of the 4 elements, bits 4-7: eq
  unsigned int cgt = 0, ceq = 0;
#pragma unroll
  for (int it = 0; it < kSteps; ++it) {
    const int64_t i0 = base + it * 128 + 4 * lane;
    float e4[4] = {0.f, 0.f, 0.f, 0.f}, s4[4] = {0.f, 0.f, 0.f, 0.f};
    if (i0 + 3 < hi) {
      const float4 sv = *reinterpret_cast<const float4*>(shared + i0);
      s4[0] = sv.x; s4[1] = sv.y; s4[2] = sv.z; s4[3] = sv.w;
      if (bf16) {
        const uint2 raw = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(expert) + i0);
        e4[0] = bf16_lo(raw.x); e4[1] = bf16_hi(raw.x); e4[2] = bf16_lo(raw.y); e4[3] = bf16_hi(raw.y);
      } else {
        const float4 ev = *reinterpret_cast<const float4*>(static_cast<const float*>(expert) + i0);
        e4[0] = ev.x; e4[1] = ev.y; e4[2] = ev.z; e4[3] = ev.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i0 + q < hi) {
          s4[q] = shared[i0 + q];
          e4[q] = bf16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(expert)[i0 + q])
                       : static_cast<const float*>(expert)[i0 + q];
        }
    }
    unsigned int f = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double r = __dsub_rn(static_cast<double>(e4[q]), static_cast<double>(s4[q]));
      rv[it * 4 + q] = __double2float_rn(r);
      const unsigned long long km = key_of(r) & mask;
      const bool in = i0 + q < hi;
      f |= (in && km > prefix ? 1u : 0u) << q;
      f |= (in && km == prefix ? 1u : 0u) << (4 + q);
    }
    fl[it] = f;
    cgt += __popc(f & 0xfu);
    ceq += __popc(f >> 4);
  }
  const unsigned int wg = __reduce_add_sync(0xffffffffu, cgt), we = __reduce_add_sync(0xffffffffu, ceq);
  if (lane == 0) { wgt[warp] = wg; weq[warp] = we; }
  __syncthreads();

  unsigned long long* status = ws.stat(bexp, range);
  if (warp == 0) {
    constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 31) - 1;
    unsigned long long tgt = 0, teq = 0;
    for (int w = 0; w < 8; ++w) { tgt += wgt[w]; teq += weq[w]; }
    unsigned long long pgt = 0, peq = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(&status[0], kInc | (tgt << 31) | teq);
    } else {
      if (lane == 0) atomicExch(&status[tile], kAgg | (tgt << 31) | teq);
      for (int t0 = tile - 1; t0 >= 0; t0 -= 32) {
        const int t = t0 - lane;
        unsigned long long w = 0;
        if (t >= 0) {
          do { w = *reinterpret_cast<volatile unsigned long long*>(&status[t]); } while ((w >> 62) == 0);
        }
        const unsigned int inc = __ballot_sync(0xffffffffu, t >= 0 && (w >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        unsigned long long g = (t >= 0 && lane <= stop) ? (w >> 31) & kVal : 0;
        unsigned long long e = (t >= 0 && lane <= stop) ? w & kVal : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          g += __shfl_xor_sync(0xffffffffu, g, off);
          e += __shfl_xor_sync(0xffffffffu, e, off);
        }
        pgt += g;
        peq += e;
        if (inc) break;
      }
      if (lane == 0) {
        __threadfence();
        atomicExch(&status[tile], kInc | ((pgt + tgt) << 31) | (peq + teq));
      }
    }
    if (lane == 0) {
      excl_gt_sh = pgt;
      excl_eq_sh = peq;
    }
  }
  __syncthreads();

  unsigned long long run_gt = excl_gt_sh, run_eq = excl_eq_sh;
  for (int w = 0; w < warp; ++w) { run_gt += wgt[w]; run_eq += weq[w]; }
  const int eb = static_cast<int>((iw + vw) / 8);
#pragma unroll
  for (int it = 0; it < kSteps; ++it) {
    const unsigned int f = fl[it];
    // exclusive in-warp prefix of (gt count << 16 | eq count)
    const unsigned int mine = (static_cast<unsigned int>(__popc(f & 0xfu)) << 16) | __popc(f >> 4);
    unsigned int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    const unsigned int total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long gb = run_gt + ((incl - mine) >> 16);
    unsigned long long ebf = run_eq + ((incl - mine) & 0xffffu);
    if (f) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool gt = (f >> q) & 1u, eq = (f >> (4 + q)) & 1u;
        if (gt || (eq && static_cast<long long>(ebf) < need)) {
          const unsigned long long taken_eq =
              static_cast<long long>(ebf) < need ? ebf : static_cast<unsigned long long>(need);
          const int64_t j = out_base + static_cast<int64_t>(gb + taken_eq);
          uint8_t* p = wire + 28 + j * eb;
          const uint64_t idx = static_cast<uint64_t>(base + it * 128 + 4 * lane + q);
          put_u32(p, static_cast<uint32_t>(idx));
          if (iw == 64) { put_u32(p + 4, static_cast<uint32_t>(idx >> 32)); p += 8; } else { p += 4; }
          if (vw == 32) {
            put_u32(p, __float_as_uint(rv[it * 4 + q]));
          } else {
            const double r = residual_at(expert, bf16, shared, static_cast<int64_t>(idx));
            const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(r));
            put_u32(p, static_cast<uint32_t>(b));
            put_u32(p + 4, static_cast<uint32_t>(b >> 32));
          }
        }
        gb += gt;
        ebf += eq;
      }
    }
    run_gt += total >> 16;
    run_eq += total & 0xffffu;
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

// Header checks in the reference's order (deserialize: magic, truncation, widths,
// truncated entries; then sr_decode: shape tag).  Codes: 1 bad magic, 2 truncated,
// 3 widths, 4 shape tag (invalid_argument); entries: 5 out of bounds, 6 not increasing.
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

// status: int32[4] per wire = {code, failing entry, fail word lo, fail word hi}.
// Pass 1: out_b = shared (float4 stream), and block (0, b) resets wire b's status.
__global__ void __launch_bounds__(256) sr_decode_copy_kernel(DecBatch batch, const float* __restrict__ shared,
                                                             int64_t P, int32_t* status) {
  const int bw = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    status[4 * bw] = 0;
    status[4 * bw + 1] = 0;
    *reinterpret_cast<unsigned long long*>(status + 4 * bw + 2) = ~0ull;
  }
  float* out = batch.out[bw];
  const int64_t nvec = P >> 2;
  const float4* src = reinterpret_cast<const float4*>(shared);
  float4* dst = reinterpret_cast<float4*>(out);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nvec; i += stride) dst[i] = src[i];
  if (blockIdx.x == 0)
    for (int64_t i = (nvec << 2) + threadIdx.x; i < P; i += blockDim.x) out[i] = shared[i];
}

// Pass 2: one thread per entry validates it (first failing entry wins, as in the
// reference's sequential loop) and applies out[i] = (float)((double)shared[i] + v).
// Indices of a valid wire are unique, so the scatter is race-free; on a corrupt wire
// the output is undefined (the reference throws) but every write stays inside [0, P).
__global__ void __launch_bounds__(256) sr_decode_scatter_kernel(DecBatch batch, size_t bytes,
                                                                const float* __restrict__ shared, int64_t h,
                                                                int64_t m, int32_t* status) {
  const int b = blockIdx.y;
  const uint8_t* wire = batch.wire[b];
  int code;
  const WireView v = read_header(wire, bytes, h, m, &code);
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (!v.ok_header) {
    if (j == 0) status[4 * b] = code;
    return;
  }
  if (j >= v.k) return;
  const uint64_t P = static_cast<uint64_t>(2 * h * m);
  const uint64_t idx = entry_index(wire, v, j);
  int c = 0;
  if (idx >= P) c = 5;
  else if (j > 0 && idx <= entry_index(wire, v, j - 1)) c = 6;
  if (c) {
    atomicMin(reinterpret_cast<unsigned long long*>(status + 4 * b + 2),
              static_cast<unsigned long long>(j) * 8ull + static_cast<unsigned long long>(c));
    return;
  }
  batch.out[b][idx] = __double2float_rn(__dadd_rn(static_cast<double>(shared[idx]), entry_value(wire, v, j)));
}

// Decode straight into the GEMM's compute layout (K-major w_up^T [m][h], w_down^T [h][m])
// in the layer dtype: the slot was pre-filled with the shared expert in that layout (a
// copy-engine memcpy), so only the k entries are scattered, each to its transposed
// position, with the same double-precision add and round as the flat decode.
struct DecLayoutBatch {
  const uint8_t* wire[kMaxSrBatch];
  void* up[kMaxSrBatch];
  void* down[kMaxSrBatch];
};

template <bool BF16OUT>
__global__ void __launch_bounds__(256) sr_decode_scatter_layout_kernel(DecLayoutBatch batch, size_t bytes,
                                                                       const float* __restrict__ shared, int64_t h,
                                                                       int64_t m, int32_t* status) {
  const int b = blockIdx.y;
  const uint8_t* wire = batch.wire[b];
  int code;
  const WireView v = read_header(wire, bytes, h, m, &code);
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (!v.ok_header) {
    if (j == 0) status[4 * b] = code;
    return;
  }
  if (j >= v.k) return;
  const uint64_t up = static_cast<uint64_t>(h * m), P = 2 * up;
  const uint64_t idx = entry_index(wire, v, j);
  int c = 0;
  if (idx >= P) c = 5;
  else if (j > 0 && idx <= entry_index(wire, v, j - 1)) c = 6;
  if (c) {
    atomicMin(reinterpret_cast<unsigned long long*>(status + 4 * b + 2),
              static_cast<unsigned long long>(j) * 8ull + static_cast<unsigned long long>(c));
    return;
  }
  const float val = __double2float_rn(__dadd_rn(static_cast<double>(shared[idx]), entry_value(wire, v, j)));
  int64_t off;
  void* base;
  if (idx < up) {  // w_up is h x m: (r, c) -> w_up^T[c][r]
    const int64_t r = static_cast<int64_t>(idx) / m, cc = static_cast<int64_t>(idx) % m;
    off = cc * h + r;
    base = batch.up[b];
  } else {         // w_down is m x h: (r, c) -> w_down^T[c][r]
    const int64_t i2 = static_cast<int64_t>(idx - up);
    const int64_t r = i2 / h, cc = i2 % h;
    off = cc * m + r;
    base = batch.down[b];
  }
  if (BF16OUT) static_cast<__nv_bfloat16*>(base)[off] = __float2bfloat16_rn(val);
  else static_cast<float*>(base)[off] = val;
}

__global__ void sr_status_init_kernel(int32_t* status, int n) {
  const int b = threadIdx.x;
  if (b >= n) return;
  status[4 * b] = 0;
  status[4 * b + 1] = 0;
  *reinterpret_cast<unsigned long long*>(status + 4 * b + 2) = ~0ull;
}

__global__ void sr_status_finalize_kernel(int32_t* status, int n) {
  const int b = threadIdx.x;
  if (b >= n || status[4 * b] != 0) return;
  const unsigned long long f = *reinterpret_cast<const unsigned long long*>(status + 4 * b + 2);
  if (f != ~0ull) {
    status[4 * b] = static_cast<int32_t>(f & 7ull);
    status[4 * b + 1] = static_cast<int32_t>(f >> 3);
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

int64_t sr_tiles(int64_t P) { return (P + kTile - 1) / kTile; }

size_t sr_workspace_bytes(int64_t h, int64_t m, int batch) {
  const int64_t tiles = sr_tiles(2 * h * m);
  return static_cast<size_t>(batch) * 2 * (sizeof(SelState) + sizeof(unsigned long long) * tiles) + 256;
}

cudaError_t launch_sr_encode_batch(DType expert_dt, const void* const* experts, int batch, const float* shared,
                                   const SrPlan& plan, uint8_t* const* wires, void* workspace,
                                   cudaStream_t stream) {
  if (batch <= 0 || batch > kMaxSrBatch) return cudaErrorInvalidValue;
  EncBatch eb{};
  for (int i = 0; i < batch; ++i) {
    eb.expert[i] = experts[i];
    eb.wire[i] = wires[i];
  }
  const int64_t tiles = sr_tiles(plan.total);
  WsView ws{static_cast<SelState*>(workspace),
            reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(workspace) + sizeof(SelState) * 2 * batch),
            tiles};
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
  sr_init_kernel<<<batch, 256, 0, stream>>>(ws, eb, ranges[0].hi - ranges[0].lo, ranges[0].k,
                                            ranges[1].hi - ranges[1].lo, ranges[1].k, plan.h, plan.m, plan.k,
                                            plan.index_bits, plan.value_bits);
  for (int r = 0; r < nr; ++r) {
    const int64_t n = ranges[r].hi - ranges[r].lo;
    if (n <= 0) continue;
    const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 8 / batch, (n + 1023) / 1024)));
    for (int pass = 0; pass < kPasses; ++pass) {
      sr_hist_kernel<<<dim3(blocks, batch), 256, 0, stream>>>(eb, bf16, shared, ranges[r].lo, ranges[r].hi, ws, r,
                                                               pass);
      sr_select_kernel<<<batch, 1024, 0, stream>>>(ws, r, pass);
    }
    const int ntiles = static_cast<int>((n + kTile - 1) / kTile);
    if ((ranges[r].lo & 3) == 0)
      sr_compact4_kernel<<<dim3(ntiles, batch), kTileThreads, 0, stream>>>(eb, bf16, shared, ranges[r].lo,
                                                                            ranges[r].hi, ws, r, ranges[r].out_base,
                                                                            plan.index_bits, plan.value_bits);
    else
      sr_compact_kernel<<<dim3(ntiles, batch), kTileThreads, 0, stream>>>(eb, bf16, shared, ranges[r].lo,
                                                                           ranges[r].hi, ws, r, ranges[r].out_base,
                                                                           plan.index_bits, plan.value_bits);
  }
  return cudaGetLastError();
}

cudaError_t launch_sr_decode_batch(const uint8_t* const* wires, int batch, size_t wire_bytes, const float* shared,
                                   int64_t h, int64_t m, float* const* outs, int32_t* status, cudaStream_t stream) {
  if (batch <= 0 || batch > kMaxSrBatch) return cudaErrorInvalidValue;
  DecBatch db{};
  for (int i = 0; i < batch; ++i) {
    db.wire[i] = wires[i];
    db.out[i] = outs[i];
  }
  const int64_t P = 2 * h * m;
  const int cblocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 8 / batch, (P / 4 + 255) / 256)));
  sr_decode_copy_kernel<<<dim3(cblocks, batch), 256, 0, stream>>>(db, shared, P, status);
  const int64_t kmax = wire_bytes > 28 ? static_cast<int64_t>((wire_bytes - 28) / 8) : 0;
  const int vblocks = static_cast<int>(std::max<int64_t>(1, (kmax + 255) / 256));
  sr_decode_scatter_kernel<<<dim3(vblocks, batch), 256, 0, stream>>>(db, wire_bytes, shared, h, m, status);
  sr_status_finalize_kernel<<<1, kMaxSrBatch, 0, stream>>>(status, batch);
  return cudaGetLastError();
}

cudaError_t launch_sr_decode_layout_batch(const uint8_t* const* wires, int batch, size_t wire_bytes,
                                          const float* shared, const void* shared_c, DType out_dt, int64_t h,
                                          int64_t m, void* const* up, void* const* down, int32_t* status,
                                          cudaStream_t stream) {
  if (batch <= 0 || batch > kMaxSrBatch) return cudaErrorInvalidValue;
  DecLayoutBatch db{};
  const size_t eb = out_dt == DType::BF16 ? 2 : 4;
  const size_t half = static_cast<size_t>(h * m) * eb;
  for (int i = 0; i < batch; ++i) {
    db.wire[i] = wires[i];
    db.up[i] = up[i];
    db.down[i] = down[i];
    // shared expert in the compute layout -> the slot (copy engine)
    cudaError_t e = cudaMemcpyAsync(up[i], shared_c, half, cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(down[i], static_cast<const uint8_t*>(shared_c) + half, half, cudaMemcpyDeviceToDevice, stream);
    if (e != cudaSuccess) return e;
  }
  sr_status_init_kernel<<<1, kMaxSrBatch, 0, stream>>>(status, batch);
  const int64_t kmax = wire_bytes > 28 ? static_cast<int64_t>((wire_bytes - 28) / 8) : 0;
  const int vblocks = static_cast<int>(std::max<int64_t>(1, (kmax + 255) / 256));
  if (out_dt == DType::BF16)
    sr_decode_scatter_layout_kernel<true><<<dim3(vblocks, batch), 256, 0, stream>>>(db, wire_bytes, shared, h, m, status);
  else
    sr_decode_scatter_layout_kernel<false><<<dim3(vblocks, batch), 256, 0, stream>>>(db, wire_bytes, shared, h, m, status);
  sr_status_finalize_kernel<<<1, kMaxSrBatch, 0, stream>>>(status, batch);
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
