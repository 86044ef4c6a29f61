// K5/K6/K7: parameter-efficient expert migration on the GPU, bit-exact with the
// reference CPU codec (proj/src/sparsecomp.cpp).
//
// Encode (K5, "pack"), reference sparsecomp.cpp:175-224:
//   r_i = (double)expert_i - (double)shared_i over the flat index (w_up then w_down);
//   keep the k entries ranked by (|r| desc, index asc) -- the reference's
//   nth_element order (:44-62) -- emitted in ascending index order as SRC1 wire
//   entries (index, value) with value = (float)r for 32-bit wires (:26-28).
//   GPU algorithm (key = IEEE bits of |r|, monotone for non-negative doubles):
//   1. sample: 32768 evenly spaced keys per range; two order statistics of the sample
//      bracket the k-th largest key's top word [lo32, hi32] with a 4-sigma margin;
//   2. split (one full read): keys above hi32 are "sure", keys in the bracket are
//      "candidates"; both are compacted in index order into a short list (residual,
//      index) with a decoupled look-back scan.  The exact counts validate the
//      bracket (sure < k <= sure + candidates, list within capacity); a failed
//      bracket switches the range to the full-range path below, so the result never
//      depends on the sample;
//   3. select: MSB radix select with 12-bit digits over the candidates (or the full
//      range) for the remaining rank, one fused histogram+select launch per digit
//      (block-private histograms, last-arriving block picks the bucket, early exit
//      once the bucket is exactly consumed or no key has lower bits);
//   4. emit: ordered compaction of the list (or range) into the wire, ties at the
//      threshold taken lowest index first.
//   Full reads: 2 (sample and list work are ~1-2% of the range) instead of one per
//   radix pass plus the compaction.
// Decode (K6, "unpack"), :226-246: out = shared, then out[i] = (float)((double)
//   shared[i] + v) for every entry; entries are validated in parallel and the
//   first failing entry (lowest j) decides the error code, like the reference's
//   sequential loop.  Copy and scatter are fused in one pass over the output.
// Shared mean (K7), :147-168: fp64 sum over experts in list order, times (1/n).
// All fp64 arithmetic uses explicit _rn intrinsics so no FMA contraction can
// change a rounding.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace hep {

namespace {

constexpr int kDigitBits = 12;
constexpr int kBins = 1 << kDigitBits;
constexpr int kPasses = 6;  // 12-bit digits cover the 63 key bits below the sign in 6 passes

constexpr int kTileThreads = 256;
constexpr int kPerThread = 16;
constexpr int kTile = kTileThreads * kPerThread;  // 4096 elements per compaction tile
constexpr int kSample = 8192;                      // sampled keys per range
constexpr int kSplitTile = 8192;                   // split: elements per tile (staged in shared memory)
constexpr unsigned int kStageCap = kSplitTile / 16;  // staged list entries per split tile
constexpr int kSampleThreads = 1024;
constexpr int kSampleSmem = (kSample + 2 * kBins) * sizeof(unsigned int);

constexpr int kModeList = 0;  // select and emit over the sure + candidate list
constexpr int kModeFull = 1;  // select and emit over the whole range (static choice or failed bracket)
constexpr int kModeDone = 2;  // the wire range is written (sr_finish_kernel)

struct SelState {
  unsigned long long prefix;
  unsigned long long mask;
  long long need;    // rank still to place (list mode: among the candidates)
  long long need0;   // min(k, n)
  long long n_sure, n_super;
  unsigned long long keyor;  // OR of every key taking part in pass 0: bits that never vary are skipped
  unsigned int lo32, hi32;   // candidate bracket on the top key word
  int done, mode;
  int top;  // bits [top, 63] of the threshold key are resolved (prefix/mask); next digit ends at top-1
  int overflow;  // a split tile listed more than its staging segment holds
  int ticket, ticket2, arrive;
  alignas(16) unsigned int hist[kBins];
};

struct RangeArgs {
  int64_t lo[2], hi[2], k[2], out_base[2];
  int full[2];  // static full-range mode
  int nr;
  int force_fallback;
  int lookback;  // the multi-block emit runs: its look-back words need zeroing
};

// Selects a per-range argument without a dynamically indexed (local-memory) param copy.
__host__ __device__ __forceinline__ int64_t pick(const int64_t (&a)[2], int r) { return r ? a[1] : a[0]; }

// Workspace: one slot per (expert, range): SelState | split look-back words | emit
// look-back words | list residuals (f64) | list indices (u32, relative to the range).
struct WsView {
  uint8_t* base;
  size_t per, off_stat, off_stat2, off_res, off_idx, off_sres, off_sidx, off_skeys;
  int64_t tiles, cap;
  __device__ uint8_t* slot(int b, int r) const { return base + (static_cast<size_t>(b) * 2 + r) * per; }
  __device__ SelState& st(int b, int r) const { return *reinterpret_cast<SelState*>(slot(b, r)); }
  __device__ unsigned long long* stat(int b, int r) const {
    return reinterpret_cast<unsigned long long*>(slot(b, r) + off_stat);
  }
  __device__ unsigned long long* stat2(int b, int r) const {
    return reinterpret_cast<unsigned long long*>(slot(b, r) + off_stat2);
  }
  __device__ double* lres(int b, int r) const { return reinterpret_cast<double*>(slot(b, r) + off_res); }
  __device__ uint32_t* lidx(int b, int r) const { return reinterpret_cast<uint32_t*>(slot(b, r) + off_idx); }
  __device__ uint32_t* skeys(int b, int r) const { return reinterpret_cast<uint32_t*>(slot(b, r) + off_skeys); }
  __device__ double* sres(int b, int r) const { return reinterpret_cast<double*>(slot(b, r) + off_sres); }
  __device__ uint32_t* sidx(int b, int r) const { return reinterpret_cast<uint32_t*>(slot(b, r) + off_sidx); }
  // listed count per split tile (the split look-back words are not used in list mode)
  __device__ unsigned int* tcount(int b, int r) const { return reinterpret_cast<unsigned int*>(stat(b, r)); }
};

struct EncBatch {
  const void* expert[kMaxSrBatch];
  uint8_t* wire[kMaxSrBatch];
  // Optimizer step fused with the encode (update = 1, fp32 experts only): expert b is the
  // fp32 master; the value encoded is fmaf(-lr, grad, master), and the split pass -- the
  // encode's one full read -- writes it back as the new master.
  const float* grad[kMaxSrBatch];
  float lr;
  int update;
};

struct DecBatch {
  const uint8_t* wire[kMaxSrBatch];
  float* out[kMaxSrBatch];
};

// Residuals of elements i0 .. i0+3 (0 past hi).  vec: i0 is 4-aligned, so one float4
// of the shared expert and one 8- or 16-byte load of the expert cover the group.
__device__ __forceinline__ void load_res4(const void* expert, int bf16, const float* __restrict__ shared,
                                          int64_t i0, int64_t hi, bool vec, double (&r)[4]) {
  float e4[4] = {0.f, 0.f, 0.f, 0.f}, s4[4] = {0.f, 0.f, 0.f, 0.f};
  if (vec && i0 + 3 < hi) {
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
#pragma unroll
  for (int q = 0; q < 4; ++q) r[q] = __dsub_rn(static_cast<double>(e4[q]), static_cast<double>(s4[q]));
}

__device__ __forceinline__ unsigned long long key_of(double r) {
  return static_cast<unsigned long long>(__double_as_longlong(fabs(r)));
}
__device__ __forceinline__ uint32_t key32_of(double r) { return static_cast<uint32_t>(key_of(r) >> 32); }

__device__ __forceinline__ void put_u32(uint8_t* p, uint32_t v) { *reinterpret_cast<uint32_t*>(p) = v; }

// Residual magnitudes cluster in a few bins, so lanes holding the same digit are merged
// with match.any and one leader adds the population count.
__device__ __forceinline__ void hist_add(unsigned int* sh, int d) {
  const unsigned int peers = __match_any_sync(__activemask(), d);
  if (d >= 0 && (threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1)) atomicAdd(&sh[d], __popc(peers));
}

// Finds, scanning bins from the top (nb-1) down, the bin holding the need-th largest
// key (1 <= need <= total): writes the bin, the count above it and its own count to
// shared memory.  Any block size that is a multiple of 32 (<= 1024).
template <typename Count>
__device__ void find_bucket(Count cnt, int nb, long long need, int* sh_bin, long long* sh_before,
                            long long* sh_count, unsigned long long* wsum) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  unsigned long long mine = 0;
  for (int i = 0; i < per; ++i) {
    const int b = nb - 1 - (t * per + i);
    if (b >= 0) mine += cnt(b);
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
    unsigned long long w = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += o;
    }
    if (lane < nw) wsum[lane] = w;
  }
  __syncthreads();
  if (warp) incl += wsum[warp - 1];
  const long long excl = static_cast<long long>(incl - mine);
  if (excl < need && static_cast<long long>(incl) >= need) {  // exactly one owner
    long long before = excl;
    for (int i = 0; i < per; ++i) {
      const int b = nb - 1 - (t * per + i);
      if (b < 0) break;
      const long long c = cnt(b);
      if (before + c >= need) {
        *sh_bin = b;
        *sh_before = before;
        *sh_count = c;
        break;
      }
      before += c;
    }
  }
  __syncthreads();
}

// Two bucket searches in one scan: counts A and B (each < 2^32 in total) packed in one
// 64-bit lane value; slot q of the outputs is the bin holding needq-th largest of
// counts q (needq <= 0: skipped).  Used by the sample bracket (both order statistics).
template <typename CountA, typename CountB>
__device__ void find_bucket_pair(CountA ca, CountB cb, int nb, long long need_a, long long need_b, int* bin,
                                 long long* before, unsigned long long* wsum) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  unsigned long long mine = 0;  // (sum A << 32) | sum B
  for (int i = 0; i < per; ++i) {
    const int b = nb - 1 - (t * per + i);
    if (b >= 0) mine += (static_cast<unsigned long long>(ca(b)) << 32) | cb(b);
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
    unsigned long long w = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += o;
    }
    if (lane < nw) wsum[lane] = w;
  }
  __syncthreads();
  if (warp) incl += wsum[warp - 1];
  const unsigned long long excl = incl - mine;
  for (int q = 0; q < 2; ++q) {
    const long long need = q ? need_b : need_a;
    const int sh = q ? 0 : 32;
    const long long ex = static_cast<long long>((excl >> sh) & 0xffffffffull);
    const long long in = static_cast<long long>((incl >> sh) & 0xffffffffull);
    if (need > 0 && ex < need && in >= need) {
      long long acc = ex;
      for (int i = 0; i < per; ++i) {
        const int b = nb - 1 - (t * per + i);
        if (b < 0) break;
        const long long c = static_cast<long long>(q ? cb(b) : ca(b));
        if (acc + c >= need) {
          bin[q] = b;
          before[q] = acc;
          break;
        }
        acc += c;
      }
    }
  }
  __syncthreads();
}

// Decoupled look-back over tiles taken in ticket order, two 31-bit counters per tile
// (warp 0; a 32-tile window per step, one predecessor per lane).  Returns the
// exclusive prefix of both counters in every lane.
__device__ __forceinline__ void lookback(unsigned long long* status, int tile, unsigned long long ta,
                                         unsigned long long tb, unsigned long long& pa, unsigned long long& pb) {
  constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 31) - 1;
  const int lane = threadIdx.x & 31;
  pa = 0;
  pb = 0;
  if (tile == 0) {
    if (lane == 0) atomicExch(&status[0], kInc | (ta << 31) | tb);
    return;
  }
  if (lane == 0) atomicExch(&status[tile], kAgg | (ta << 31) | tb);
  for (int t0 = tile - 1; t0 >= 0; t0 -= 32) {
    const int t = t0 - lane;
    unsigned long long w = 0;
    if (t >= 0) {
      do { w = *reinterpret_cast<volatile unsigned long long*>(&status[t]); } while ((w >> 62) == 0);
    }
    const unsigned int inc = __ballot_sync(0xffffffffu, t >= 0 && (w >> 62) == 2);
    const int stop = inc ? __ffs(inc) - 1 : 31;  // nearest predecessor with an inclusive prefix
    unsigned long long a = (t >= 0 && lane <= stop) ? (w >> 31) & kVal : 0;
    unsigned long long b = (t >= 0 && lane <= stop) ? w & kVal : 0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    pa += a;
    pb += b;
    if (inc) break;
  }
  if (lane == 0) {
    __threadfence();
    atomicExch(&status[tile], kInc | ((pa + ta) << 31) | (pb + tb));
  }
}

// Exclusive in-warp prefix of two per-lane counts (each < 2^16 per warp step).
__device__ __forceinline__ void warp_scan2(unsigned int a, unsigned int b, unsigned int& ea, unsigned int& eb,
                                           unsigned int& ta, unsigned int& tb) {
  const int lane = threadIdx.x & 31;
  const unsigned int mine = (a << 16) | b;
  unsigned int incl = mine;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  const unsigned int total = __shfl_sync(0xffffffffu, incl, 31);
  ea = (incl - mine) >> 16;
  eb = (incl - mine) & 0xffffu;
  ta = total >> 16;
  tb = total & 0xffffu;
}

// grid (16, batch): reset the selection state and look-back words of expert b's two
// ranges, write its SRC1 header.
__global__ void sr_init_kernel(WsView ws, EncBatch batch, int bf16, const float* __restrict__ shared, RangeArgs ra,
                               int64_t h, int64_t m, int64_t k_total, uint32_t iw, uint32_t vw) {
  const int b = blockIdx.y, t = threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int r = 0; r < ra.nr; ++r) {
    // list-mode range: its kSample evenly spaced keys, spread over the grid's blocks so
    // the scattered DRAM reads are not limited by one SM's outstanding misses
    const int64_t n = pick(ra.hi, r) - pick(ra.lo, r), k = pick(ra.k, r);
    if ((r ? ra.full[1] : ra.full[0]) || k <= 0 || k >= n) continue;
    const int S = static_cast<int>(n < kSample ? n : kSample);
    const int64_t step = n / S, lo = pick(ra.lo, r);
    uint32_t* keys = ws.skeys(b, r);
    for (int j = blockIdx.x * blockDim.x + t; j < S; j += static_cast<int>(stride)) {
      const int64_t i = lo + static_cast<int64_t>(j) * step;
      float e = bf16 ? __uint_as_float(static_cast<uint32_t>(__ldcs(static_cast<const unsigned short*>(batch.expert[b]) + i)) << 16)
                     : __ldcs(static_cast<const float*>(batch.expert[b]) + i);
      if (batch.update) e = fmaf(-batch.lr, __ldcs(batch.grad[b] + i), e);  // the stepped master
      keys[j] = key32_of(__dsub_rn(static_cast<double>(e), static_cast<double>(__ldcs(shared + i))));
    }
  }
  for (int r = 0; r < 2; ++r) {
    SelState& s = ws.st(b, r);
    unsigned long long* s1 = ws.stat(b, r);
    unsigned long long* s2 = ws.stat2(b, r);
    // only the multi-block emit walks look-back words (the split's per-tile counts are
    // written for every tile before they are read)
    if (ra.lookback)
      for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + t; i < ws.tiles; i += stride) s2[i] = 0;
    (void)s1;
    if (blockIdx.x) continue;
    for (int i = t; i < kBins; i += blockDim.x) s.hist[i] = 0;
    if (t == 0) {
      const bool live = r < ra.nr;
      const int64_t n = live ? pick(ra.hi, r) - pick(ra.lo, r) : 0, k = live ? pick(ra.k, r) : 0;
      s.prefix = 0;
      s.mask = 0;
      s.top = 63;
      s.need0 = s.need = k >= n ? n : (k > 0 ? k : 0);
      s.done = (k <= 0 || k >= n) ? 1 : 0;
      s.mode = (!live || s.done || (r ? ra.full[1] : ra.full[0])) ? kModeFull : kModeList;
      s.n_sure = 0;
      s.n_super = 0;
      s.overflow = 0;
      s.keyor = 0;
      s.lo32 = 0;
      s.hi32 = 0xffffffffu;
      s.ticket = 0;
      s.ticket2 = 0;
      s.arrive = 0;
    }
  }
  if (blockIdx.x == 0 && t == 0) {
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

// grid (nr, batch), 1024 threads: from the kSample evenly spaced keys of the range
// (gathered by sr_init_kernel), bracket the need-th largest key's top word between two
// sample order statistics,
// each located to 24 bits (a 12-bit digit, then 12 more bits inside its bin; the
// bracket is widened to the bins' outer edges, so it only ever grows).
__global__ void __launch_bounds__(kSampleThreads) sr_sample_kernel(RangeArgs ra, WsView ws) {
  extern __shared__ unsigned int smem[];
  uint32_t* ks = smem;                    // kSample keys
  unsigned int* h_hi = smem + kSample;    // kBins
  unsigned int* h_lo = h_hi + kBins;      // kBins
  __shared__ unsigned long long wsum[32];
  __shared__ int pbin[2];
  __shared__ long long pbefore[2];
  const int r = blockIdx.x, b = blockIdx.y;
  SelState& s = ws.st(b, r);
  if (s.mode != kModeList) return;
  const int64_t n = pick(ra.hi, r) - pick(ra.lo, r);
  const int S = static_cast<int>(n < kSample ? n : kSample);
  const uint32_t* gk = ws.skeys(b, r);  // sampled by sr_init_kernel across many SMs
  for (int j = threadIdx.x; j < S; j += blockDim.x) ks[j] = gk[j];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) h_hi[i] = 0;
  __syncthreads();
  const double q = static_cast<double>(s.need0) / static_cast<double>(n);
  const double mean = q * S;
  const double dev = 4.0 * sqrt(mean * (1.0 - q)) + 8.0;
  const long long r_hi = static_cast<long long>(floor(mean - dev));
  const long long r_lo = static_cast<long long>(ceil(mean + dev));
  const bool has_hi = r_hi >= 0, has_lo = r_lo < S;
  // digit 1: bits 20..31 of the top word
  for (int j = threadIdx.x; j < S; j += blockDim.x) hist_add(h_hi, static_cast<int>(ks[j] >> 20));
  __syncthreads();
  long long w_hi = r_hi + 1, w_lo = r_lo + 1;
  // both order statistics' first digits from one scan of the shared histogram
  find_bucket_pair([&](int i) { return h_hi[i]; }, [&](int i) { return h_hi[i]; }, kBins, has_hi ? w_hi : 0,
                   has_lo ? w_lo : 0, pbin, pbefore, wsum);
  const int b_hi = has_hi ? pbin[0] : 0, b_lo = has_lo ? pbin[1] : 0;
  if (has_hi) w_hi -= pbefore[0];
  if (has_lo) w_lo -= pbefore[1];
  // digit 2: bits 8..19 inside each bin
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) { h_hi[i] = 0; h_lo[i] = 0; }
  __syncthreads();
  for (int j = threadIdx.x; j < S; j += blockDim.x) {
    const uint32_t key = ks[j];
    const int top = static_cast<int>(key >> 20), d = static_cast<int>((key >> 8) & 0xfffu);
    const bool in_hi = has_hi && top == b_hi, in_lo = has_lo && top == b_lo;
    const unsigned int act = __activemask();
    if (__any_sync(act, in_hi)) hist_add(h_hi, in_hi ? d : -1);  // most warps hold neither bin
    if (__any_sync(act, in_lo)) hist_add(h_lo, in_lo ? d : -1);
  }
  __syncthreads();
  find_bucket_pair([&](int i) { return h_hi[i]; }, [&](int i) { return h_lo[i]; }, kBins, has_hi ? w_hi : 0,
                   has_lo ? w_lo : 0, pbin, pbefore, wsum);
  uint32_t hi32 = 0xffffffffu, lo32 = 0;
  if (has_hi) hi32 = (static_cast<uint32_t>(b_hi) << 20) | (static_cast<uint32_t>(pbin[0]) << 8) | 0xffu;
  if (has_lo) lo32 = (static_cast<uint32_t>(b_lo) << 20) | (static_cast<uint32_t>(pbin[1]) << 8);
  if (ra.force_fallback) hi32 = lo32 = 0;  // test hook: an invalid bracket
  if (threadIdx.x == 0) {
    s.hi32 = hi32;
    s.lo32 = lo32;
  }
}

// grid (tiles, batch * nr), 256 threads: one full read of the range.  A tile (kSplitTile
// elements) is staged into shared memory by two bulk async copies (TMA engine, no
// registers held in flight; plain loads for an unaligned range start and the last
// < 8 elements), then classified from shared memory:
//   fast phase (branch-free): the listed set is {|d| >= B0}, B0 the double whose top
//   word is lo32 (d the fp64 residual).  f = |e - s| in fp32 is within 2^-24 relative
//   of the exact difference, so f < B0 (1 - 2^-22) proves "not listed"; the rest (the
//   ~1-2% listed plus a 2^-22-wide band) are marked "maybe" and reclassified in fp64.
// Sure (key32 > hi32) and candidate (lo32 <= key32 <= hi32) entries of the tile are
// written in index order into its fixed staging segment (kStageCap entries) with the
// tile's count; totals accumulate atomically.  No tile waits on another;
// sr_finish_kernel later packs the segments into the dense list.
template <bool BULK>
__global__ void __launch_bounds__(kTileThreads) sr_split_kernel(EncBatch batch, int bf16,
                                                                const float* __restrict__ shared, RangeArgs ra,
                                                                WsView ws) {
  extern __shared__ __align__(128) uint8_t smem_split[];
  float* s_sh = reinterpret_cast<float*>(smem_split);              // kSplitTile floats
  uint8_t* s_ex = smem_split + kSplitTile * sizeof(float);          // kSplitTile bf16 or floats
  __shared__ __align__(8) uint64_t full_bar;
  __shared__ unsigned int wtot[8][2];                               // per-warp step counts (8-bit fields)
  const int r = blockIdx.y % ra.nr, b = blockIdx.y / ra.nr;
  SelState& s = ws.st(b, r);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x;
  const int64_t lo = pick(ra.lo, r), hi = pick(ra.hi, r);
  const int64_t t_lo = lo + static_cast<int64_t>(tile) * kSplitTile;
  // range full statically (ra.full, a kernel parameter): nothing to split
  if (t_lo >= hi || (r ? ra.full[1] : ra.full[0])) return;
  const int count = static_cast<int>(hi - t_lo < kSplitTile ? hi - t_lo : kSplitTile);
  const void* expert = batch.expert[b];
  const int eb = bf16 ? 2 : 4;
  float* s_gr = reinterpret_cast<float*>(s_ex + kSplitTile * 4);  // update mode: the gradient tile
  const float* grad = batch.update ? batch.grad[b] : nullptr;
  // bulk part: the first count8 elements (multiple of 8 = 16 B of bf16, 32 B of f32).
  // Issued before the range's mode is read from global memory, so the tile's DRAM
  // latency overlaps that dependent load instead of following it.
  const int count8 = BULK ? (count & ~7) : 0;
  if (BULK) {
    if (threadIdx.x == 0) {
      mbar_init(&full_bar, 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (count8) {
        const uint64_t pol = l2_policy_evict_first();
        mbar_arrive_expect_tx(&full_bar, static_cast<uint32_t>(count8 * (4 + eb + (grad ? 4 : 0))));
        bulk_load(s_sh, shared + t_lo, static_cast<uint32_t>(count8 * 4), &full_bar, pol);
        bulk_load(s_ex, static_cast<const uint8_t*>(expert) + t_lo * eb, static_cast<uint32_t>(count8 * eb),
                  &full_bar, pol);
        if (grad) bulk_load(s_gr, grad + t_lo, static_cast<uint32_t>(count8 * 4), &full_bar, pol);
      }
    }
    __syncthreads();
  }
  if (s.mode != kModeList) {  // list mode abandoned (trivial k): drain the copies, exit
    if (BULK && count8) mbar_wait(&full_bar, 0);
    return;
  }
  for (int p = count8 + threadIdx.x; p < count; p += blockDim.x) {  // plain-load part
    s_sh[p] = shared[t_lo + p];
    if (bf16) reinterpret_cast<uint16_t*>(s_ex)[p] = static_cast<const uint16_t*>(expert)[t_lo + p];
    else reinterpret_cast<float*>(s_ex)[p] = static_cast<const float*>(expert)[t_lo + p];
    if (grad) s_gr[p] = grad[t_lo + p];
  }
  const uint32_t lo32 = s.lo32, hi32 = s.hi32;
  // fp32 "surely below B0" threshold; outside [2^-100, 2^126] every element is exact
  const double b0 = __hiloint2double(static_cast<int>(lo32), 0);
  const float t_below = (b0 >= 0x1p-100 && b0 <= 0x1p126) ? __double2float_rd(b0 * (1.0 - 0x1p-22)) : -1.0f;
  if (BULK && count8) mbar_wait(&full_bar, 0);
  __syncthreads();
  if (grad) {
    // the optimizer step fused into the encode's one full read: master' = master - lr g
    // (one rounding), written back as the new master and classified below
    float* s_m = reinterpret_cast<float*>(s_ex);
    float* master = const_cast<float*>(static_cast<const float*>(expert)) + t_lo;
    const bool vec = ((reinterpret_cast<uintptr_t>(master) & 15) == 0);
    const int count4 = vec ? (count & ~3) : 0;
    for (int p = 4 * threadIdx.x; p < count4; p += 4 * blockDim.x) {
      float4 m4 = *reinterpret_cast<const float4*>(s_m + p);
      const float4 g4 = *reinterpret_cast<const float4*>(s_gr + p);
      m4.x = fmaf(-batch.lr, g4.x, m4.x);
      m4.y = fmaf(-batch.lr, g4.y, m4.y);
      m4.z = fmaf(-batch.lr, g4.z, m4.z);
      m4.w = fmaf(-batch.lr, g4.w, m4.w);
      *reinterpret_cast<float4*>(s_m + p) = m4;
      __stcs(reinterpret_cast<float4*>(master + p), m4);
    }
    for (int p = count4 + threadIdx.x; p < count; p += blockDim.x) {
      s_m[p] = fmaf(-batch.lr, s_gr[p], s_m[p]);
      master[p] = s_m[p];
    }
    __syncthreads();
  }

  // element p = 1024 it + 4 tid + q  ->  bit 4 it + q
  constexpr int kSteps = kSplitTile / (kTileThreads * 4);  // 8 (<= 8: two words of 8-bit step fields)
  auto ex_at = [&](int p) {
    return bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(s_ex)[p]) : reinterpret_cast<const float*>(s_ex)[p];
  };
  uint32_t maybe = 0;
#pragma unroll
  for (int it = 0; it < kSteps; ++it) {
    const int p0 = it * 1024 + 4 * threadIdx.x;
    const float4 sv = *reinterpret_cast<const float4*>(s_sh + p0);
    float e4[4];
    if (bf16) {
      const uint2 raw = *reinterpret_cast<const uint2*>(s_ex + p0 * 2);
      e4[0] = bf16_lo(raw.x); e4[1] = bf16_hi(raw.x); e4[2] = bf16_lo(raw.y); e4[3] = bf16_hi(raw.y);
    } else {
      const float4 ev = *reinterpret_cast<const float4*>(s_ex + p0 * 4);
      e4[0] = ev.x; e4[1] = ev.y; e4[2] = ev.z; e4[3] = ev.w;
    }
    maybe |= static_cast<uint32_t>(!(fabsf(e4[0] - sv.x) < t_below)) << (4 * it);
    maybe |= static_cast<uint32_t>(!(fabsf(e4[1] - sv.y) < t_below)) << (4 * it + 1);
    maybe |= static_cast<uint32_t>(!(fabsf(e4[2] - sv.z) < t_below)) << (4 * it + 2);
    maybe |= static_cast<uint32_t>(!(fabsf(e4[3] - sv.w) < t_below)) << (4 * it + 3);
  }
  uint32_t fsp = 0, fsu = 0;
  for (uint32_t mm = maybe; mm; mm &= mm - 1) {
    const int bit = __ffs(mm) - 1;
    const int p = (bit >> 2) * 1024 + 4 * threadIdx.x + (bit & 3);
    if (p >= count) continue;
    const double rr = __dsub_rn(static_cast<double>(ex_at(p)), static_cast<double>(s_sh[p]));
    const uint32_t k32 = key32_of(rr);
    if (k32 >= lo32) {
      fsp |= 1u << bit;
      if (k32 > hi32) fsu |= 1u << bit;
    }
  }

  // per-step counts (0..4) in 8-bit fields, 4 steps per word, scanned across lanes
  unsigned int cnt[2], incl[2];
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    unsigned int v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v |= static_cast<unsigned int>(__popc((fsp >> (4 * (4 * w + k))) & 0xfu)) << (8 * k);
    cnt[w] = incl[w] = v;
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const unsigned int o = __shfl_up_sync(0xffffffffu, incl[w], off);
      if (lane >= off) incl[w] += o;
    }
  }
  const unsigned int nsu = __reduce_add_sync(0xffffffffu, __popc(fsu));
  if (lane == 31) { wtot[warp][0] = incl[0]; wtot[warp][1] = incl[1]; }
  __shared__ unsigned int wsu[8];
  if (lane == 0) wsu[warp] = nsu;
  __syncthreads();
  // step s offset = all warps' entries in steps < s + lower warps' entries in step s
  unsigned int step_off[kSteps];
  unsigned int total = 0;
#pragma unroll
  for (int st = 0; st < kSteps; ++st) {
    unsigned int below = 0, all = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const unsigned int c = (wtot[w][st >> 2] >> (8 * (st & 3))) & 0xffu;
      all += c;
      below += w < warp ? c : 0u;
    }
    step_off[st] = total + below;
    total += all;
  }
  if (threadIdx.x == 0) {
    unsigned int tsu = 0;
    for (int w = 0; w < 8; ++w) tsu += wsu[w];
    ws.tcount(b, r)[tile] = total;
    if (tsu) atomicAdd(reinterpret_cast<unsigned long long*>(&s.n_sure), static_cast<unsigned long long>(tsu));
    if (total) atomicAdd(reinterpret_cast<unsigned long long*>(&s.n_super), static_cast<unsigned long long>(total));
    if (total > kStageCap) atomicOr(&s.overflow, 1);
  }
  double* sres = ws.sres(b, r) + static_cast<int64_t>(tile) * kStageCap;
  uint32_t* sidx = ws.sidx(b, r) + static_cast<int64_t>(tile) * kStageCap;
  for (uint32_t mm = fsp; mm; mm &= mm - 1) {
    const int bit = __ffs(mm) - 1;
    const int it = bit >> 2, q = bit & 3;
    const unsigned int lane_excl = ((incl[it >> 2] - cnt[it >> 2]) >> (8 * (it & 3))) & 0xffu;
    const unsigned int pos = step_off[it] + lane_excl + __popc((fsp >> (4 * it)) & ((1u << q) - 1u));
    const int p = it * 1024 + 4 * threadIdx.x + q;
    if (pos < kStageCap) {
      sres[pos] = __dsub_rn(static_cast<double>(ex_at(p)), static_cast<double>(s_sh[p]));
      sidx[pos] = static_cast<uint32_t>(t_lo + p - lo);
    }
  }
}

// ---------------------------------------------------------------- finish (cluster)
// One 8-CTA cluster per (expert, range) in list mode, everything after the split in
// one launch, CTAs exchanging through distributed shared memory:
//   1. validate the bracket from the exact totals; pack the tiles' staging segments
//      into the dense list (CTA c: split tiles [c T/8, (c+1) T/8));
//   2. radix select over the candidates (the sure entries are excluded), digits starting
//      below the common prefix of lo32 and hi32: block histograms, reduced across the
//      cluster (CTA c sums bins [c nb/8, (c+1) nb/8)), the owner of the target bin
//      broadcasts it;
//   3. ordered emit: per-CTA (gt, eq) counts exchanged for the CTA's offset, then
//      block scans place every selected entry at its wire position.
// A failed bracket (rare) runs steps 2-3 over the full range instead of the list, with
// the same cluster (slower, same result).
constexpr int kFinCta = 8;
constexpr int kFinThreads = 512;
constexpr int kFinPer = 8;                        // consecutive units per thread per round
constexpr int kFinRound = kFinThreads * kFinPer;  // 4096
constexpr double kFinMaxList = 262144.0;          // longest expected list per slot on the cluster path
constexpr int kFinSmemCap = 12288;                // list entries a CTA keeps in shared memory
constexpr int kFinSmemPadded = kFinSmemCap + kFinSmemCap / 8;
constexpr int kFinSmem = kFinSmemPadded * (sizeof(double) + sizeof(uint32_t));

struct FinXch {
  unsigned long long tot[kFinCta];  // per-CTA slice totals / counts (written by the peers)
  unsigned long long aux[kFinCta];
  int bin;
  long long before, count;
};

// Inclusive block scan of one 32-bit value per thread (512 threads); returns the
// exclusive prefix and writes the block total to *total.
__device__ __forceinline__ unsigned int block_scan_excl(unsigned int v, unsigned int* wtot, unsigned int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned int w = lane < (kFinThreads >> 5) ? wtot[lane] : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned int o = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += o;
    }
    if (lane < (kFinThreads >> 5)) wtot[lane] = w;
  }
  __syncthreads();
  const unsigned int ex = (warp ? wtot[warp - 1] : 0u) + incl - v;
  *total = wtot[(kFinThreads >> 5) - 1];
  __syncthreads();
  return ex;
}

__global__ void __cluster_dims__(kFinCta, 1, 1) __launch_bounds__(kFinThreads)
    sr_finish_kernel(EncBatch batch, int bf16, const float* __restrict__ shared, RangeArgs ra, WsView ws,
                     uint32_t iw, uint32_t vw) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = static_cast<int>(cl.block_rank());
  const int r = blockIdx.y % ra.nr, b = blockIdx.y / ra.nr;
  SelState& s = ws.st(b, r);
  if (s.mode != kModeList) return;  // uniform over the cluster (no CTA writes it before the end)
  // the CTA's share of the list, resident across the passes and the emit when it fits
  // (one pad word per 8 keeps the per-thread runs of 8 conflict-free)
  extern __shared__ __align__(16) uint8_t fin_dyn[];
  double* s_res = reinterpret_cast<double*>(fin_dyn);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(fin_dyn + sizeof(double) * kFinSmemPadded);
  __shared__ unsigned int hist[kBins];
  __shared__ unsigned int slice[kBins / kFinCta];
  __shared__ unsigned int wtot[32];
  __shared__ unsigned long long wsum[32];
  __shared__ FinXch xch;
  __shared__ int sh_bin;
  __shared__ long long sh_before, sh_count;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t lo = pick(ra.lo, r), hi = pick(ra.hi, r), n = hi - lo;
  const void* expert = batch.expert[b];
  const bool vec = (lo & 3) == 0;
  const uint32_t lo32 = s.lo32, hi32 = s.hi32;
  const long long n_sure = s.n_sure, n_super = s.n_super, need0 = s.need0;
  const bool list = !s.overflow && n_super <= ws.cap && n_sure < need0 && n_super >= need0;
  double* lres = ws.lres(b, r);
  uint32_t* lidx = ws.lidx(b, r);

  // 1. gather this CTA's split tiles' staging segments (in index order): into shared
  // memory when they fit, else into the dense list in global memory
  int64_t my_lo = 0, my_hi = 0;  // this CTA's entries in list order
  bool in_smem = false;
  if (list) {
    const unsigned int* cnt = ws.tcount(b, r);
    const int ntiles = static_cast<int>((n + kSplitTile - 1) / kSplitTile);
    const int t0 = static_cast<int>(static_cast<int64_t>(ntiles) * crank / kFinCta);
    const int t1 = static_cast<int>(static_cast<int64_t>(ntiles) * (crank + 1) / kFinCta);
    unsigned int before = 0, mine = 0;
    for (int t = threadIdx.x; t < t1; t += blockDim.x) (t < t0 ? before : mine) += cnt[t];
    unsigned int tot;
    block_scan_excl(before, wtot, &tot);
    before = tot;
    block_scan_excl(mine, wtot, &tot);
    mine = tot;
    my_lo = before;
    my_hi = static_cast<int64_t>(before) + mine;
    in_smem = mine <= static_cast<unsigned int>(kFinSmemCap);
    const double* sres = ws.sres(b, r);
    const uint32_t* sidx = ws.sidx(b, r);
    unsigned int run = before;
    __shared__ unsigned int toff[kFinThreads + 1];
    for (int c0 = t0; c0 < t1; c0 += blockDim.x) {
      const int t = c0 + threadIdx.x;
      const int nt = min(static_cast<int>(blockDim.x), t1 - c0);
      const unsigned int c = t < t1 ? cnt[t] : 0u;
      unsigned int chunk;
      toff[threadIdx.x] = block_scan_excl(c, wtot, &chunk);
      if (threadIdx.x == 0) toff[nt] = chunk;
      __syncthreads();
      // flattened copy: entry p of the chunk lives in tile upper_bound(toff, p) - 1;
      // eight entries per thread per round, all loads issued before the stores
      for (unsigned int p0 = 0; p0 < chunk; p0 += 8 * kFinThreads) {
        double v[8];
        uint32_t ii[8];
        unsigned int pp[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const unsigned int p = p0 + q * kFinThreads + threadIdx.x;
          pp[q] = p;
          if (p < chunk) {
            int lo_k = 0, hi_k = nt;  // first k with toff[k] > p, in (0, nt]
            while (lo_k < hi_k) {
              const int mid = (lo_k + hi_k) >> 1;
              if (toff[mid] <= p) lo_k = mid + 1; else hi_k = mid;
            }
            const int k = lo_k - 1;
            const int64_t src = static_cast<int64_t>(c0 + k) * kStageCap + (p - toff[k]);
            v[q] = sres[src];
            ii[q] = sidx[src];
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (pp[q] < chunk) {
            const unsigned int d = run + pp[q];
            if (in_smem) {
              const unsigned int l = d - before;
              s_res[l + (l >> 3)] = v[q];
              s_idx[l + (l >> 3)] = ii[q];
            } else {
              lres[d] = v[q];
              lidx[d] = ii[q];
            }
          }
      }
      run += chunk;
      __syncthreads();
    }
  }
  __syncthreads();

  // units: this CTA's list entries, or an equal share of the full range after a failed
  // bracket
  const int64_t units = list ? n_super : n;
  const int64_t per_cta = ((units + kFinCta - 1) / kFinCta + 7) & ~static_cast<int64_t>(7);
  const int64_t u_lo = list ? my_lo : min(units, per_cta * crank);
  const int64_t u_hi = list ? my_hi : min(units, u_lo + per_cta);
  // residuals and relative indices of units u0 .. u0+7
  auto load8 = [&](int64_t u0, double (&rv)[kFinPer], uint32_t (&ix)[kFinPer]) {
    if (list && in_smem) {
#pragma unroll
      for (int q = 0; q < kFinPer; ++q) {
        const int64_t l = u0 + q - u_lo;
        const bool in = u0 + q < u_hi;
        rv[q] = in ? s_res[l + (l >> 3)] : 0.0;
        ix[q] = in ? s_idx[l + (l >> 3)] : 0u;
      }
    } else if (list) {
      if (((u0 & 7) == 0) && u0 + kFinPer <= u_hi) {
#pragma unroll
        for (int q = 0; q < kFinPer; q += 2) {
          const double2 d = *reinterpret_cast<const double2*>(lres + u0 + q);
          rv[q] = d.x; rv[q + 1] = d.y;
        }
        const uint4 a = *reinterpret_cast<const uint4*>(lidx + u0), c = *reinterpret_cast<const uint4*>(lidx + u0 + 4);
        ix[0] = a.x; ix[1] = a.y; ix[2] = a.z; ix[3] = a.w; ix[4] = c.x; ix[5] = c.y; ix[6] = c.z; ix[7] = c.w;
      } else {
#pragma unroll
        for (int q = 0; q < kFinPer; ++q) {
          rv[q] = u0 + q < u_hi ? lres[u0 + q] : 0.0;
          ix[q] = u0 + q < u_hi ? lidx[u0 + q] : 0u;
        }
      }
    } else {
      double a[4], c[4];
      load_res4(expert, bf16, shared, lo + u0, lo + u_hi, vec, a);
      load_res4(expert, bf16, shared, lo + u0 + 4, lo + u_hi, vec, c);
#pragma unroll
      for (int q = 0; q < 4; ++q) { rv[q] = a[q]; rv[4 + q] = c[q]; }
#pragma unroll
      for (int q = 0; q < kFinPer; ++q) ix[q] = static_cast<uint32_t>(u0 + q);
    }
  };

  // 2. radix select
  long long need = list ? need0 - n_sure : need0;
  bool done = list && n_super == need0;  // every candidate is taken
  unsigned long long prefix = 0, mask = 0;
  int top = 63;
  if (list) {  // every candidate shares the leading bits of lo32 and hi32
    const int c = __clz(lo32 ^ hi32);
    mask = c >= 32 ? 0xffffffff00000000ull : (~0ull << (64 - c));
    prefix = (static_cast<unsigned long long>(hi32) << 32) & mask;
    top = 64 - c;
  }
  unsigned long long keyor = 0;
  for (int pass = 0; pass < kPasses && !done; ++pass) {
    const int width = top < kDigitBits ? top : kDigitBits, shift = top - width, nb = 1 << width;
    const unsigned int dmask = static_cast<unsigned int>(nb - 1);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    unsigned long long kor = 0;
    for (int64_t u0 = u_lo + kFinPer * threadIdx.x; u0 - kFinPer * threadIdx.x < u_hi; u0 += kFinRound) {
      double rv[kFinPer];
      uint32_t ix[kFinPer];
      load8(u0, rv, ix);
#pragma unroll
      for (int q = 0; q < kFinPer; ++q) {
        const unsigned long long key = key_of(rv[q]);
        const bool cand = u0 + q < u_hi && (!list || static_cast<uint32_t>(key >> 32) <= hi32);
        kor |= cand ? key : 0ull;
        // candidates spread over the bins below their common prefix: plain atomics
        if (cand && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & dmask], 1u);
      }
    }
    if (pass == 0) {
      const unsigned int lw = __reduce_or_sync(0xffffffffu, static_cast<unsigned int>(kor));
      const unsigned int hw = __reduce_or_sync(0xffffffffu, static_cast<unsigned int>(kor >> 32));
      if (lane == 0) wsum[warp] = (static_cast<unsigned long long>(hw) << 32) | lw;
    }
    __syncthreads();
    if (pass == 0 && threadIdx.x == 0) {
      unsigned long long o = 0;
      for (int w = 0; w < kFinThreads / 32; ++w) o |= wsum[w];
      kor = o;
    }
    cl.sync();  // every CTA's histogram is complete
    // my slice of bins, summed over the cluster
    const int per = (nb + kFinCta - 1) / kFinCta, b0 = crank * per, b1 = min(nb, b0 + per);
    unsigned int mine = 0;
    for (int i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      unsigned int v = 0;
#pragma unroll
      for (int c = 0; c < kFinCta; ++c) v += cl.map_shared_rank(hist, c)[i];
      slice[i - b0] = v;
      mine += v;
    }
    unsigned int stot;
    block_scan_excl(mine, wtot, &stot);
    if (threadIdx.x == 0)
      for (int c = 0; c < kFinCta; ++c) {
        cl.map_shared_rank(&xch, c)->tot[crank] = stot;
        if (pass == 0) cl.map_shared_rank(&xch, c)->aux[crank] = kor;
      }
    cl.sync();  // slice totals (and the pass-0 key OR) everywhere
    if (pass == 0)
      for (int c = 0; c < kFinCta; ++c) keyor |= xch.aux[c];
    // the slice holding the need-th largest: bins descend from the top slice
    long long above = 0;
    int owner = 0;
    for (int c = kFinCta - 1; c >= 0; --c) {
      if (above + static_cast<long long>(xch.tot[c]) >= need) { owner = c; break; }
      above += static_cast<long long>(xch.tot[c]);
    }
    if (crank == owner) {
      find_bucket([&](int i) { return static_cast<unsigned long long>(slice[i]); }, b1 - b0, need - above, &sh_bin,
                  &sh_before, &sh_count, wsum);
      if (threadIdx.x == 0)
        for (int c = 0; c < kFinCta; ++c) {
          FinXch* x = cl.map_shared_rank(&xch, c);
          x->bin = b0 + sh_bin;
          x->before = above + sh_before;
          x->count = sh_count;
        }
    }
    cl.sync();  // the chosen bin everywhere
    const long long rem = need - xch.before;
    prefix |= static_cast<unsigned long long>(xch.bin) << shift;
    mask |= static_cast<unsigned long long>(nb - 1) << shift;
    need = rem;
    top = shift;
    if (xch.count == rem || shift == 0) done = true;
    if ((keyor & ((1ull << shift) - 1ull)) == 0) {  // no key has a lower bit: the bucket is all ties
      mask = ~0ull;
      done = true;
    }
    cl.sync();  // xch is rewritten by the next pass
  }

  // 3. emit.  Selected: sure (list), or (key & mask) > prefix, or one of the first
  // `need` ties (key & mask) == prefix in index order.
  auto flags = [&](double rr, bool in, bool& gt, bool& eq) {
    const unsigned long long key = key_of(rr);
    const bool sure = list && static_cast<uint32_t>(key >> 32) > hi32;
    const unsigned long long km = key & mask;
    gt = in && (sure || km > prefix);
    eq = in && !sure && km == prefix;
  };
  unsigned int cgt = 0, ceq = 0;
  for (int64_t u0 = u_lo + kFinPer * threadIdx.x; u0 - kFinPer * threadIdx.x < u_hi; u0 += kFinRound) {
    double rv[kFinPer];
    uint32_t ix[kFinPer];
    load8(u0, rv, ix);
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) {
      bool gt, eq;
      flags(rv[q], u0 + q < u_hi, gt, eq);
      cgt += gt;
      ceq += eq;
    }
  }
  unsigned int tgt, teq;
  block_scan_excl(cgt, wtot, &tgt);  // block sums (the count sweep can exceed 16-bit fields)
  block_scan_excl(ceq, wtot, &teq);
  if (threadIdx.x == 0)
    for (int c = 0; c < kFinCta; ++c) {
      cl.map_shared_rank(&xch, c)->tot[crank] = tgt;
      cl.map_shared_rank(&xch, c)->aux[crank] = teq;
    }
  cl.sync();
  unsigned long long run_gt = 0, run_eq = 0;
  for (int c = 0; c < crank; ++c) { run_gt += xch.tot[c]; run_eq += xch.aux[c]; }
  uint8_t* wire = batch.wire[b];
  const int ebytes = static_cast<int>((iw + vw) / 8);
  const int64_t out_base = pick(ra.out_base, r);
  for (int64_t u0 = u_lo + kFinPer * threadIdx.x; u0 - kFinPer * threadIdx.x < u_hi; u0 += kFinRound) {
    double rv[kFinPer];
    uint32_t ix[kFinPer];
    load8(u0, rv, ix);
    unsigned int fg = 0, fe = 0;
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) {
      bool gt, eq;
      flags(rv[q], u0 + q < u_hi, gt, eq);
      fg |= static_cast<unsigned int>(gt) << q;
      fe |= static_cast<unsigned int>(eq) << q;
    }
    unsigned int rt;  // (gt << 16 | eq) packed: at most 4096 of each per round
    const unsigned int xp = block_scan_excl((static_cast<unsigned int>(__popc(fg)) << 16) | __popc(fe), wtot, &rt);
    const unsigned int rg = rt >> 16, re = rt & 0xffffu;
    unsigned long long gb = run_gt + (xp >> 16), ebf = run_eq + (xp & 0xffffu);
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) {
      const bool gt = (fg >> q) & 1u, eq = (fe >> q) & 1u;
      if (gt || (eq && static_cast<long long>(ebf) < need)) {
        const unsigned long long taken_eq =
            static_cast<long long>(ebf) < need ? ebf : static_cast<unsigned long long>(need);
        uint8_t* p = wire + 28 + (out_base + static_cast<int64_t>(gb + taken_eq)) * ebytes;
        const uint64_t idx = static_cast<uint64_t>(lo) + ix[q];
        put_u32(p, static_cast<uint32_t>(idx));
        if (iw == 64) { put_u32(p + 4, static_cast<uint32_t>(idx >> 32)); p += 8; } else { p += 4; }
        if (vw == 32) {
          put_u32(p, __float_as_uint(__double2float_rn(rv[q])));
        } else {
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(rv[q]));
          put_u32(p, static_cast<uint32_t>(bits));
          put_u32(p + 4, static_cast<uint32_t>(bits >> 32));
        }
      }
      gb += gt;
      ebf += eq;
    }
    run_gt += rg;
    run_eq += re;
  }
  if (crank == 0 && threadIdx.x == 0) {  // the later multi-block kernels skip this slot
    s.done = 1;
    s.mode = kModeDone;
  }
}

// Multi-block path (large lists, and statically full-range slots): scan, pack, one
// select launch per digit, emit.  Grids span all SMs, so a list of millions of entries
// per slot streams at HBM rate instead of through one cluster.
// grid (batch * nr), 1024 threads: validate the bracket from the exact totals and turn
// the tiles' listed counts into exclusive offsets in the dense list.
__global__ void __launch_bounds__(1024) sr_scan_kernel(RangeArgs ra, WsView ws) {
  const int r = blockIdx.x % ra.nr, b = blockIdx.x / ra.nr;
  SelState& s = ws.st(b, r);
  if (s.mode != kModeList) return;
  __shared__ unsigned int wsum[32];
  const long long n_sure = s.n_sure, n_super = s.n_super;
  const bool valid = !s.overflow && n_super <= ws.cap && n_sure < s.need0 && n_super >= s.need0;
  if (!valid) {
    if (threadIdx.x == 0) s.mode = kModeFull;
    return;
  }
  if (threadIdx.x == 0) {
    const uint32_t lo32 = s.lo32, hi32 = s.hi32;
    s.need = s.need0 - n_sure;
    if (n_super == s.need0) s.done = 1;  // every candidate is taken
    // every candidate shares the leading bits of lo32 and hi32: start the digits below
    const int c = __clz(lo32 ^ hi32);  // >= 1 (bit 63 of a key is 0)
    const unsigned long long msk = c >= 32 ? 0xffffffff00000000ull : (~0ull << (64 - c));
    s.mask = msk;
    s.prefix = (static_cast<unsigned long long>(hi32) << 32) & msk;
    s.top = 64 - c;
  }
  const int64_t n = pick(ra.hi, r) - pick(ra.lo, r);
  const int ntiles = static_cast<int>((n + kSplitTile - 1) / kSplitTile);
  unsigned int* cnt = ws.tcount(b, r);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int carry = 0;
  for (int c0 = 0; c0 < ntiles; c0 += blockDim.x) {
    const int t = c0 + threadIdx.x;
    const unsigned int c = t < ntiles ? cnt[t] : 0u;
    unsigned int incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned int o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      unsigned int w = wsum[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned int o = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += o;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const unsigned int wb = warp ? wsum[warp - 1] : 0u;
    if (t < ntiles) cnt[t] = carry + wb + incl - c;  // exclusive offset
    carry += wsum[31];
    __syncthreads();
  }
}

// grid (blocks, batch * nr): one warp per split tile copies its staged entries to the
// tile's offset in the dense list.
__global__ void __launch_bounds__(kTileThreads) sr_pack_kernel(RangeArgs ra, WsView ws) {
  const int r = blockIdx.y % ra.nr, b = blockIdx.y / ra.nr;
  SelState& s = ws.st(b, r);
  if (s.mode != kModeList) return;
  const int64_t n = pick(ra.hi, r) - pick(ra.lo, r);
  const int ntiles = static_cast<int>((n + kSplitTile - 1) / kSplitTile);
  const unsigned int* off = ws.tcount(b, r);
  const long long n_super = s.n_super;
  const int lane = threadIdx.x & 31;
  double* lres = ws.lres(b, r);
  uint32_t* lidx = ws.lidx(b, r);
  const double* sres = ws.sres(b, r);
  const uint32_t* sidx = ws.sidx(b, r);
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += warps) {
    const unsigned int o = off[t];
    const unsigned int c = (t + 1 < ntiles ? off[t + 1] : static_cast<unsigned int>(n_super)) - o;
    const int64_t src = static_cast<int64_t>(t) * kStageCap;
#pragma unroll 4
    for (unsigned int j = lane; j < c; j += 32) {
      lres[o + j] = sres[src + j];
      lidx[o + j] = sidx[src + j];
    }
  }
}

// grid (blocks, batch * nr): histogram of the current digit over the keys matching the
// prefix (candidates of the list, or the full range), block-private in shared memory;
// the last block to arrive picks the bucket of the need-th largest and resets the
// global histogram for the next digit.
__global__ void __launch_bounds__(kTileThreads) sr_select_kernel(EncBatch batch, int bf16,
                                                                 const float* __restrict__ shared, RangeArgs ra,
                                                                 WsView ws, int pass) {
  const int r = blockIdx.y % ra.nr, b = blockIdx.y / ra.nr;
  SelState& s = ws.st(b, r);
  if (s.done || s.mode == kModeDone) return;
  __shared__ unsigned int sh[kBins];
  __shared__ unsigned long long wsum[32];
  __shared__ int sh_bin, sh_last;
  __shared__ long long sh_before, sh_count;
  const int mode = s.mode;
  const unsigned long long mask = s.mask, prefix = s.prefix;
  const int top = s.top, width = top < kDigitBits ? top : kDigitBits, shift = top - width;
  const unsigned int dmask = (1u << width) - 1u;
  const int64_t lo = pick(ra.lo, r), hi = pick(ra.hi, r);
  const int64_t units = mode == kModeList ? s.n_super : hi - lo;
  const int64_t chunk = static_cast<int64_t>(kTile);  // units per block per sweep
  const int64_t first = static_cast<int64_t>(blockIdx.x) * chunk;
  const bool work = first < units;
  unsigned long long kor = 0;
  if (work) {
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    auto digit = [&](unsigned long long key, bool in) {
      kor |= in ? key : 0ull;
      return in && (key & mask) == prefix ? static_cast<int>((key >> shift) & dmask) : -1;
    };
    const int64_t sweep = static_cast<int64_t>(gridDim.x) * chunk;
    if (mode == kModeList) {
      const double* lres = ws.lres(b, r);
      const uint32_t hi32 = s.hi32;
      for (int64_t c0 = first; c0 < units; c0 += sweep) {
        double rv[kPerThread];  // all loads first (in-order issue), then the digits
#pragma unroll
        for (int it = 0; it < kPerThread / 4; ++it) {
          const int64_t j0 = c0 + it * (kTileThreads * 4) + 4 * threadIdx.x;
          if (j0 + 3 < units) {
            const double2 a = *reinterpret_cast<const double2*>(lres + j0);
            const double2 c = *reinterpret_cast<const double2*>(lres + j0 + 2);
            rv[4 * it] = a.x; rv[4 * it + 1] = a.y; rv[4 * it + 2] = c.x; rv[4 * it + 3] = c.y;
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) rv[4 * it + q] = j0 + q < units ? lres[j0 + q] : 0.0;
          }
        }
#pragma unroll
        for (int it = 0; it < kPerThread / 4; ++it) {
          const int64_t j0 = c0 + it * (kTileThreads * 4) + 4 * threadIdx.x;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const unsigned long long key = key_of(rv[4 * it + q]);
            hist_add(sh, digit(key, j0 + q < units && static_cast<uint32_t>(key >> 32) <= hi32));
          }
        }
      }
    } else {
      const void* expert = batch.expert[b];
      const bool vec = (lo & 3) == 0;
      for (int64_t c0 = first; c0 < units; c0 += sweep) {
        for (int it = 0; it < kPerThread / 4; ++it) {
          const int64_t i0 = lo + c0 + it * (kTileThreads * 4) + 4 * threadIdx.x;
          double r4[4];
          load_res4(expert, bf16, shared, i0, hi, vec, r4);
          int d[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) d[q] = digit(key_of(r4[q]), i0 + q < hi);
#pragma unroll
          for (int q = 0; q < 4; ++q) hist_add(sh, d[q]);
        }
      }
    }
    if (pass == 0) {
      const unsigned int lo_w = __reduce_or_sync(0xffffffffu, static_cast<unsigned int>(kor));
      const unsigned int hi_w = __reduce_or_sync(0xffffffffu, static_cast<unsigned int>(kor >> 32));
      if ((threadIdx.x & 31) == 0 && (lo_w | hi_w))
        atomicOr(&s.keyor, (static_cast<unsigned long long>(hi_w) << 32) | lo_w);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kBins; i += blockDim.x)
      if (sh[i]) atomicAdd(&s.hist[i], sh[i]);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sh_last = atomicAdd(&s.arrive, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  const int nb = 1 << width;
  const long long need = s.need;
  // the global histogram -> shared memory in one coalesced sweep, then the scan
  for (int i = threadIdx.x; i < nb / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(sh)[i] = __ldcg(reinterpret_cast<const uint4*>(s.hist) + i);
  if (nb < 4 && threadIdx.x < nb) sh[threadIdx.x] = __ldcg(&s.hist[threadIdx.x]);
  __syncthreads();
  find_bucket([&](int i) { return static_cast<unsigned long long>(sh[i]); }, nb, need, &sh_bin, &sh_before,
              &sh_count, wsum);
  if (threadIdx.x == 0) {
    const int bin = sh_bin;
    const long long rem = need - sh_before;
    s.prefix |= static_cast<unsigned long long>(bin) << shift;
    s.mask |= static_cast<unsigned long long>(nb - 1) << shift;
    s.need = rem;
    s.top = shift;
    if (sh_count == rem || shift == 0) s.done = 1;
    if ((__ldcg(&s.keyor) & ((1ull << shift) - 1ull)) == 0) {
      // No key has a bit below this digit: the remaining bucket is all ties.
      s.mask = ~0ull;
      s.done = 1;
    }
    s.arrive = 0;
  }
  for (int i = threadIdx.x; i < kBins / 4; i += blockDim.x) reinterpret_cast<uint4*>(s.hist)[i] = make_uint4(0, 0, 0, 0);
}

// grid (blocks, batch * nr), persistent over tiles taken in ticket order: ordered
// compaction of the selected entries of the list (or of the full range) into the wire.
// Selected: sure, or (key & mask) > prefix, or a threshold tie among the first `need`.
__global__ void __launch_bounds__(kTileThreads) sr_emit_kernel(EncBatch batch, int bf16,
                                                               const float* __restrict__ shared, RangeArgs ra,
                                                               WsView ws, uint32_t iw, uint32_t vw) {
  const int r = blockIdx.y % ra.nr, b = blockIdx.y / ra.nr;
  SelState& s = ws.st(b, r);
  if (s.need0 == 0 || s.mode == kModeDone) return;
  __shared__ int tile_sh;
  __shared__ unsigned int wgt[8], weq[8];
  __shared__ unsigned long long excl_gt_sh, excl_eq_sh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kSteps = kPerThread / 4;
  const int mode = s.mode;
  const unsigned long long mask = s.mask, prefix = s.prefix;
  const long long need = s.need;
  const uint32_t hi32 = s.hi32;
  const int64_t lo = pick(ra.lo, r), hi = pick(ra.hi, r);
  const int64_t units = mode == kModeList ? s.n_super : hi - lo;
  const int64_t ntiles = (units + kTile - 1) / kTile;
  const void* expert = batch.expert[b];
  const bool vec = (lo & 3) == 0;
  const double* lres = ws.lres(b, r);
  const uint32_t* lidx = ws.lidx(b, r);
  uint8_t* wire = batch.wire[b];
  const int eb = static_cast<int>((iw + vw) / 8);
  const int64_t out_base = pick(ra.out_base, r);

  for (;;) {
    if (threadIdx.x == 0) tile_sh = atomicAdd(&s.ticket2, 1);
    __syncthreads();
    const int tile = tile_sh;
    if (tile >= ntiles) break;
    const int64_t base = static_cast<int64_t>(tile) * kTile + warp * (kPerThread * 32);  // unit offset

    double rv[kPerThread];
    uint32_t ix[kPerThread];
    unsigned int fl[kSteps];  // bits 0-3 gt, 4-7 eq
    unsigned int cgt = 0, ceq = 0;
    // all loads of the tile first (in-order issue), then the flags
#pragma unroll
    for (int it = 0; it < kSteps; ++it) {
      const int64_t u0 = base + it * 128 + 4 * lane;
      if (mode == kModeList) {
        if (u0 + 3 < units) {
          const double2 a = *reinterpret_cast<const double2*>(lres + u0);
          const double2 c = *reinterpret_cast<const double2*>(lres + u0 + 2);
          const uint4 iv = *reinterpret_cast<const uint4*>(lidx + u0);
          rv[it * 4] = a.x; rv[it * 4 + 1] = a.y; rv[it * 4 + 2] = c.x; rv[it * 4 + 3] = c.y;
          ix[it * 4] = iv.x; ix[it * 4 + 1] = iv.y; ix[it * 4 + 2] = iv.z; ix[it * 4 + 3] = iv.w;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            rv[it * 4 + q] = u0 + q < units ? lres[u0 + q] : 0.0;
            ix[it * 4 + q] = u0 + q < units ? lidx[u0 + q] : 0u;
          }
        }
      } else {
        double r4[4];
        load_res4(expert, bf16, shared, lo + u0, hi, vec, r4);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          rv[it * 4 + q] = r4[q];
          ix[it * 4 + q] = static_cast<uint32_t>(u0 + q);
        }
      }
    }
#pragma unroll
    for (int it = 0; it < kSteps; ++it) {
      const int64_t u0 = base + it * 128 + 4 * lane;
      unsigned int f = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned long long key = key_of(rv[it * 4 + q]);
        const bool in = u0 + q < units;
        const bool sure = mode == kModeList && static_cast<uint32_t>(key >> 32) > hi32;
        const unsigned long long km = key & mask;
        f |= (in && (sure || km > prefix) ? 1u : 0u) << q;
        f |= (in && !sure && km == prefix ? 1u : 0u) << (4 + q);
      }
      fl[it] = f;
      cgt += __popc(f & 0xfu);
      ceq += __popc(f >> 4);
    }
    const unsigned int wg = __reduce_add_sync(0xffffffffu, cgt), we = __reduce_add_sync(0xffffffffu, ceq);
    if (lane == 0) { wgt[warp] = wg; weq[warp] = we; }
    __syncthreads();
    if (warp == 0) {
      unsigned long long tgt = 0, teq = 0;
      for (int w = 0; w < 8; ++w) { tgt += wgt[w]; teq += weq[w]; }
      unsigned long long pgt, peq;
      lookback(ws.stat2(b, r), tile, tgt, teq, pgt, peq);
      if (lane == 0) {
        excl_gt_sh = pgt;
        excl_eq_sh = peq;
      }
    }
    __syncthreads();

    unsigned long long run_gt = excl_gt_sh, run_eq = excl_eq_sh;
    for (int w = 0; w < warp; ++w) { run_gt += wgt[w]; run_eq += weq[w]; }
#pragma unroll
    for (int it = 0; it < kSteps; ++it) {
      const unsigned int f = fl[it];
      unsigned int egt, eeq, tgt, teq;
      warp_scan2(__popc(f & 0xfu), __popc(f >> 4), egt, eeq, tgt, teq);
      unsigned long long gb = run_gt + egt, ebf = run_eq + eeq;
      if (f) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool gt = (f >> q) & 1u, eq = (f >> (4 + q)) & 1u;
          if (gt || (eq && static_cast<long long>(ebf) < need)) {
            const unsigned long long taken_eq =
                static_cast<long long>(ebf) < need ? ebf : static_cast<unsigned long long>(need);
            const int64_t j = out_base + static_cast<int64_t>(gb + taken_eq);
            uint8_t* p = wire + 28 + j * eb;
            const uint64_t idx = static_cast<uint64_t>(lo) + ix[it * 4 + q];
            put_u32(p, static_cast<uint32_t>(idx));
            if (iw == 64) { put_u32(p + 4, static_cast<uint32_t>(idx >> 32)); p += 8; } else { p += 4; }
            const double rr = rv[it * 4 + q];
            if (vw == 32) {
              put_u32(p, __float_as_uint(__double2float_rn(rr)));
            } else {
              const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(rr));
              put_u32(p, static_cast<uint32_t>(bits));
              put_u32(p + 4, static_cast<uint32_t>(bits >> 32));
            }
          }
          gb += gt;
          ebf += eq;
        }
      }
      run_gt += tgt;
      run_eq += teq;
    }
    __syncthreads();  // tile_sh / wgt / excl reuse
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

namespace {

size_t round256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// Per-(expert, range) workspace slot; tiles and list capacity sized for a range of the
// whole expert (P elements), so one layout serves both wire layouts.
WsView make_ws(void* base, int64_t P) {
  WsView ws{};
  ws.base = static_cast<uint8_t*>(base);
  ws.tiles = (P + kTile - 1) / kTile;
  ws.cap = std::min<int64_t>(P, P / 32 + 4096);
  ws.off_stat = round256(sizeof(SelState));
  ws.off_stat2 = ws.off_stat + round256(sizeof(unsigned long long) * ws.tiles);
  ws.off_res = ws.off_stat2 + round256(sizeof(unsigned long long) * ws.tiles);
  ws.off_idx = ws.off_res + round256(sizeof(double) * ws.cap);
  const int64_t staged = (P + kSplitTile - 1) / kSplitTile * kStageCap;
  ws.off_sres = ws.off_idx + round256(sizeof(uint32_t) * ws.cap);
  ws.off_sidx = ws.off_sres + round256(sizeof(double) * staged);
  ws.off_skeys = ws.off_sidx + round256(sizeof(uint32_t) * staged);
  ws.per = ws.off_skeys + round256(sizeof(uint32_t) * kSample);
  return ws;
}

// HEP_SR_SELECT=full forces the full-range select, =fallback an invalid sample bracket,
// =multiblock the multi-block list path (all exercised in tests); anything else picks
// per call.
int select_override() {
  const char* v = std::getenv("HEP_SR_SELECT");
  if (!v) return 0;
  if (!std::strcmp(v, "full")) return 1;
  if (!std::strcmp(v, "fallback")) return 2;
  if (!std::strcmp(v, "multiblock")) return 3;
  if (!std::strcmp(v, "fallback-multiblock")) return 4;
  return 0;
}

}  // namespace

size_t sr_workspace_bytes(int64_t h, int64_t m, int batch) {
  return static_cast<size_t>(batch) * 2 * make_ws(nullptr, 2 * h * m).per + 256;
}

namespace {
// The unfused optimizer step (and the fallback of the fused one): m = fmaf(-lr, g, m).
__global__ void sgd_step_kernel(EncBatch eb, int64_t P) {
  const int b = blockIdx.y;
  float* m = const_cast<float*>(static_cast<const float*>(eb.expert[b]));
  const float* g = eb.grad[b];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(g)) & 15) == 0;
  const int64_t P4 = vec ? P / 4 : 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P4; i += stride) {
    float4 v = reinterpret_cast<const float4*>(m)[i];
    const float4 d = __ldcs(reinterpret_cast<const float4*>(g) + i);
    v.x = fmaf(-eb.lr, d.x, v.x);
    v.y = fmaf(-eb.lr, d.y, v.y);
    v.z = fmaf(-eb.lr, d.z, v.z);
    v.w = fmaf(-eb.lr, d.w, v.w);
    reinterpret_cast<float4*>(m)[i] = v;
  }
  for (int64_t i = 4 * P4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P; i += stride)
    m[i] = fmaf(-eb.lr, g[i], m[i]);
}
}  // namespace

cudaError_t launch_sgd_step_batch(float* const* masters, const float* const* grads, int batch, int64_t P, float lr,
                                  cudaStream_t stream) {
  if (batch <= 0 || batch > kMaxSrBatch) return cudaErrorInvalidValue;
  EncBatch eb{};
  for (int i = 0; i < batch; ++i) {
    eb.expert[i] = masters[i];
    eb.grad[i] = grads[i];
  }
  eb.lr = lr;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(148 * 8 / batch, (P / 4 + 255) / 256)));
  sgd_step_kernel<<<dim3(blocks, batch), 256, 0, stream>>>(eb, P);
  return cudaGetLastError();
}

cudaError_t launch_sr_encode_batch(DType expert_dt, const void* const* experts, int batch, const float* shared,
                                   const SrPlan& plan, uint8_t* const* wires, void* workspace,
                                   cudaStream_t stream, const float* const* grads, float lr) {
  if (batch <= 0 || batch > kMaxSrBatch) return cudaErrorInvalidValue;
  if (grads && expert_dt != DType::F32) return cudaErrorInvalidValue;  // the fused step updates fp32 masters
  EncBatch eb{};
  for (int i = 0; i < batch; ++i) {
    eb.expert[i] = experts[i];
    eb.wire[i] = wires[i];
    if (grads) eb.grad[i] = grads[i];
  }
  eb.lr = lr;
  const int64_t P = plan.total, up = plan.h * plan.m;
  // 256-byte align the slots (the workspace pointer itself may be any cudaMalloc offset)
  uint8_t* wbase = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  const WsView ws = make_ws(wbase, P);
  const int bf16 = expert_dt == DType::BF16;
  const int ovr = select_override();
  RangeArgs ra{};
  if (plan.per_matrix) {
    ra.lo[0] = 0;  ra.hi[0] = up; ra.k[0] = plan.k_up;   ra.out_base[0] = 0;
    ra.lo[1] = up; ra.hi[1] = P;  ra.k[1] = plan.k_down; ra.out_base[1] = plan.k_up;
    ra.nr = 2;
  } else {
    ra.lo[0] = 0; ra.hi[0] = P; ra.k[0] = plan.k; ra.out_base[0] = 0;
    ra.nr = 1;
  }
  ra.force_fallback = ovr == 2 || ovr == 4;
  bool any_list = false, any_full = false;
  double expect_max = 0.0;
  for (int r = 0; r < ra.nr; ++r) {
    const int64_t n = ra.hi[r] - ra.lo[r], k = ra.k[r];
    bool full = ovr == 1 || n <= 0 || k <= 0 || k >= n || n >= (int64_t{1} << 31);
    if (!full) {
      // expected list size: k plus the sample's +-dev bracket scaled to the range
      const double S = static_cast<double>(std::min<int64_t>(n, kSample)), q = static_cast<double>(k) / n;
      const double dev = 4.0 * std::sqrt(q * S * (1.0 - q)) + 8.0;
      const double expect = static_cast<double>(k) + 2.0 * dev / S * static_cast<double>(n);
      full = expect > 0.75 * static_cast<double>(ws.cap);
      if (!full) expect_max = std::max(expect_max, expect);
    }
    ra.full[r] = full;
    any_list |= !full && k > 0;
    any_full |= full && k > 0;
  }
  const int slots = batch * ra.nr;
  const int64_t nmax = std::max(ra.hi[0] - ra.lo[0], ra.nr > 1 ? ra.hi[1] - ra.lo[1] : int64_t{0});
  const int64_t tiles_max = std::max<int64_t>(1, (nmax + kSplitTile - 1) / kSplitTile);
  const int wide = std::max(1, 148 * 8 / slots);  // blocks per slot for full-range sweeps
  // lists up to kFinMaxList entries finish in one cluster launch per slot; longer ones
  // (experts of ~100M parameters) take the multi-block path across all SMs
  const bool cluster = expect_max <= kFinMaxList && ovr != 3 && ovr != 4;

  ra.lookback = (any_full || (any_list && !cluster)) ? 1 : 0;
  if (grads) {
    // Fused only when every range is list-selected: then the split pass reads every
    // element once and writes the stepped master back.  Otherwise step first, then encode.
    bool all_list = true;
    for (int r = 0; r < ra.nr; ++r) {
      const int64_t n = ra.hi[r] - ra.lo[r], k = ra.k[r];
      all_list &= !ra.full[r] && k > 0 && k < n;
    }
    if (all_list) {
      eb.update = 1;
    } else {
      std::vector<float*> ms(static_cast<size_t>(batch));
      for (int i = 0; i < batch; ++i) ms[static_cast<size_t>(i)] = const_cast<float*>(static_cast<const float*>(experts[i]));
      const cudaError_t e = launch_sgd_step_batch(ms.data(), grads, batch, P, lr, stream);
      if (e != cudaSuccess) return e;
    }
  }
  sr_init_kernel<<<dim3(16, batch), 256, 0, stream>>>(ws, eb, bf16, shared, ra, plan.h, plan.m, plan.k,
                                                      plan.index_bits, plan.value_bits);
  if (any_list) {
    static DeviceOnce attr;
    if (!attr.done()) {
      cudaFuncSetAttribute(sr_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSampleSmem);
      cudaFuncSetAttribute(sr_split_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSplitTile * 12);
      cudaFuncSetAttribute(sr_split_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSplitTile * 12);
      cudaFuncSetAttribute(sr_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFinSmem);
      attr.set();
    }
    sr_sample_kernel<<<dim3(ra.nr, batch), kSampleThreads, kSampleSmem, stream>>>(ra, ws);
    const bool bulk = ((ra.lo[0] | (ra.nr > 1 ? ra.lo[1] : 0)) & 7) == 0;
    const int smem = kSplitTile * (4 + (bf16 ? 2 : 4) + (eb.update ? 4 : 0));
    const dim3 sgrid(static_cast<unsigned>(tiles_max), slots);
    if (bulk) sr_split_kernel<true><<<sgrid, kTileThreads, smem, stream>>>(eb, bf16, shared, ra, ws);
    else sr_split_kernel<false><<<sgrid, kTileThreads, smem, stream>>>(eb, bf16, shared, ra, ws);
    if (cluster) {
      sr_finish_kernel<<<dim3(kFinCta, slots), kFinThreads, kFinSmem, stream>>>(eb, bf16, shared, ra, ws,
                                                                                plan.index_bits, plan.value_bits);
    } else {
      sr_scan_kernel<<<slots, 1024, 0, stream>>>(ra, ws);
      sr_pack_kernel<<<dim3(std::max(1, 148 * 4 / slots), slots), kTileThreads, 0, stream>>>(ra, ws);
    }
  }
  if (any_full || (any_list && !cluster)) {
    // A failed bracket on the multi-block path runs with the list-sized grid (rare);
    // a statically full range gets the wide grid.
    const int list_blocks = static_cast<int>(std::min<double>(wide, std::ceil(1.25 * expect_max / kTile)));
    const int blocks = any_full ? wide : std::max(list_blocks, 1);
    for (int pass = 0; pass < kPasses; ++pass)
      sr_select_kernel<<<dim3(blocks, slots), kTileThreads, 0, stream>>>(eb, bf16, shared, ra, ws, pass);
    sr_emit_kernel<<<dim3(blocks, slots), kTileThreads, 0, stream>>>(eb, bf16, shared, ra, ws, plan.index_bits,
                                                                     plan.value_bits);
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

namespace {
struct PatchBatch {
  const uint8_t* wire[kMaxSrBatch];
  uint8_t* blocks[kMaxSrBatch];
  uint2* ovf[kMaxSrBatch];
  int* ovf_count[kMaxSrBatch];
};

__global__ void sr_patch_reset_kernel(PatchBatch pb, int64_t nblocks, int32_t* status, int n) {
  const int b = blockIdx.y;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nblocks;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    *reinterpret_cast<uint32_t*>(pb.blocks[b] + i * kPatchBlockBytes) = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *pb.ovf_count[b] = 0;
    if (b < n) {
      status[4 * b] = 0;
      status[4 * b + 1] = 0;
      *reinterpret_cast<unsigned long long*>(status + 4 * b + 2) = ~0ull;
    }
  }
}

// grid (blocks, batch): thread j < k validates entry j like the decode (first failing
// entry wins, as in sr_decode_scatter) and files it into the patch block of the GEMM stage
// that loads its B element: up entry (row r < h, column c < m) is B[c][r] of the up
// projection (n = c, k = r), down entry (f, c) is B[c][f] of the down projection.  The
// value is the dense decode's: bf16((float)((double)shared[i] + v)).
__global__ void __launch_bounds__(256) sr_patch_index_kernel(PatchBatch pb, size_t bytes,
                                                             const float* __restrict__ shared, int64_t h,
                                                             int64_t m, int32_t* status) {
  const int b = blockIdx.y;
  const uint8_t* wire = pb.wire[b];
  int code;
  const WireView v = read_header(wire, bytes, h, m, &code);
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (!v.ok_header) {
    if (j == 0) status[4 * b] = code;
    return;
  }
  if (j >= v.k) return;
  const int64_t up = h * m, P = 2 * up;
  const uint64_t idx = entry_index(wire, v, j);
  int c = 0;
  if (idx >= static_cast<uint64_t>(P)) c = 5;
  else if (j > 0 && idx <= entry_index(wire, v, j - 1)) c = 6;
  if (c) {
    atomicMin(reinterpret_cast<unsigned long long*>(status + 4 * b + 2),
              static_cast<unsigned long long>(j) * 8ull + static_cast<unsigned long long>(c));
    return;
  }
  const int64_t i = static_cast<int64_t>(idx);
  const int half = i < up ? 0 : 1;
  const int64_t N = half ? h : m, K = half ? m : h;    // B is N x K for this projection
  const int64_t row = half ? (i - up) / h : i / m;      // reference row = k
  const int64_t col = half ? (i - up) % h : i % m;      // reference column = n
  const int64_t nt = col / 256, kb = row / 64;
  const int r = static_cast<int>(col % 256), rr = static_cast<int>(row % 64);
  const uint32_t byte = static_cast<uint32_t>(r * 128 + ((((rr >> 3) ^ (r & 7))) << 4) + ((rr & 7) << 1));
  const float val = __double2float_rn(__dadd_rn(static_cast<double>(shared[i]), entry_value(wire, v, j)));
  const uint32_t word = ((byte >> 1) << 16) | static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(val)));
  const int64_t blk = (half ? patch_blocks(m, h) : 0) + nt * (K / 64) + kb;
  (void)N;
  uint32_t* hdr = reinterpret_cast<uint32_t*>(pb.blocks[b] + blk * kPatchBlockBytes);
  const uint32_t pos = atomicAdd(hdr, 1u);
  if (pos < static_cast<uint32_t>(kPatchBlockCap)) {
    hdr[4 + pos] = word;
  } else {
    const int q = atomicAdd(pb.ovf_count[b], 1);
    pb.ovf[b][q] = make_uint2(static_cast<uint32_t>(blk - (half ? patch_blocks(m, h) : 0)) |
                                  (static_cast<uint32_t>(half) << 31), word);
  }
}
}  // namespace

cudaError_t launch_sr_patch_index(const uint8_t* const* wires, int batch, size_t wire_bytes, const float* shared,
                                  int64_t h, int64_t m, uint8_t* const* blocks, uint2* const* ovf,
                                  int* const* ovf_count, int32_t* status, cudaStream_t stream) {
  if (batch <= 0 || batch > kMaxSrBatch || h % 64 || m % 64) return cudaErrorInvalidValue;
  PatchBatch pb{};
  for (int i = 0; i < batch; ++i) {
    pb.wire[i] = wires[i];
    pb.blocks[i] = blocks[i];
    pb.ovf[i] = ovf[i];
    pb.ovf_count[i] = ovf_count[i];
  }
  const int64_t nblocks = patch_blocks(m, h) + patch_blocks(h, m);
  sr_patch_reset_kernel<<<dim3(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(64, (nblocks + 255) / 256))),
                             batch), 256, 0, stream>>>(pb, nblocks, status, batch);
  const int64_t kmax = wire_bytes > 28 ? static_cast<int64_t>((wire_bytes - 28) / 8) : 0;
  const int blocks_k = static_cast<int>(std::max<int64_t>(1, (kmax + 255) / 256));
  sr_patch_index_kernel<<<dim3(blocks_k, batch), 256, 0, stream>>>(pb, wire_bytes, shared, h, m, status);
  sr_status_finalize_kernel<<<1, kMaxSrBatch, 0, stream>>>(status, batch);
  return cudaGetLastError();
}

namespace {
// First failing decode code of a batch -> a (host-mapped) error word, kept until read.
__global__ void sr_status_fold_kernel(const int32_t* __restrict__ status, int n, int32_t* __restrict__ err) {
  const int i = threadIdx.x;
  if (i < n && status[4 * i] != 0) atomicCAS(err, 0, (status[4 * i] & 0xff) | (min(status[4 * i + 1], 0xffffff) << 8));
}
}  // namespace

cudaError_t launch_sr_status_fold(const int32_t* status, int n, int32_t* err, cudaStream_t stream) {
  if (n <= 0 || n > kMaxSrBatch) return cudaErrorInvalidValue;
  sr_status_fold_kernel<<<1, 64, 0, stream>>>(status, n, err);
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


// Loads every kernel of this file now (see preload_kernels in kernels.h).
cudaError_t preload_sr_codec_kernels() {
  auto load = [](const void* fn) {
    cudaFuncAttributes attr;
    return cudaFuncGetAttributes(&attr, fn);
  };
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_init_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_sample_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_split_kernel<true>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_split_kernel<false>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_finish_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_scan_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_pack_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_select_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_emit_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_decode_copy_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_decode_scatter_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_decode_scatter_layout_kernel<true>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_decode_scatter_layout_kernel<false>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_status_init_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_status_finalize_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(shared_mean_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(transpose_convert_kernel<float, float>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(transpose_convert_kernel<float, __nv_bfloat16>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(transpose_convert_kernel<__nv_bfloat16, __nv_bfloat16>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(transpose_convert_kernel<__nv_bfloat16, float>))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_status_fold_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sgd_step_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_patch_index_kernel))) return e;
  if (const cudaError_t e = load(reinterpret_cast<const void*>(sr_patch_reset_kernel))) return e;
  return cudaSuccess;
}

}  // namespace hep
