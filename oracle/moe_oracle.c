/*
 * ORACLE — test infrastructure only.  Nothing in the product path links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs do, as the checker or as the timed CPU baseline.
 *
 * A plain-C restatement of the HybridEP MoE-layer hot path, executed over G
 * simulated GPUs in one process (A2A / All-Gather are memcpy between per-GPU
 * arrays).  Each function cites what it restates:
 *   - topology (renumber, Algorithm 1, dense table, peer lists): reference
 *     proj/src/topology.cpp:74-177 and proj/src/simcore.cpp:30-74.  PINNED against
 *     the reference itself (oracle/_ref, built from /root/reference sources) and
 *     the golden vectors of proj/tests/test_topology.cpp (tests/test_oracle.py).
 *   - SR codec (shared mean, encode, wire, decode): proj/src/sparsecomp.cpp:26-246.
 *     PINNED against the golden bytes of proj/tests/test_sparsecomp.cpp:258-279
 *     and byte-for-byte against oracle/_ref on randomized cases.
 *   - gate / route / permute / expert FFN / combine: the reference has NO
 *     implementation (only perf::gemm_latency, perfmodel.cpp:67-71).  These follow
 *     the semantics pinned in SURVEY.md §8(c) S1-S7 and are "parity unpinned"
 *     (DESIGN.md §3): routing is exact integer work checked bit-for-bit, outputs
 *     carry the stated tolerances.
 *
 * Build: oracle/Makefile -> oracle/_build/liboracle.so (OpenMP).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_LEVELS 16

/* ------------------------------------------------------------------ topology */

int64_t orc_gpus(const int64_t* sf, int L) {
  int64_t g = 1;
  for (int i = 0; i < L; ++i) g *= sf[i];
  return g;
}

/* f(m): x_i = floor(m / prod_{j>i} SF_j) mod SF_i  (topology.cpp:74-83) */
void orc_renumber(const int64_t* sf, int L, int64_t m, int64_t* x) {
  int64_t below = 1;
  for (int i = L - 1; i >= 0; --i) {
    x[i] = (m / below) % sf[i];
    below *= sf[i];
  }
}

/* Algorithm 1 at the deepest differing level (topology.cpp:160-176).
 * Returns type (0 none, 1 AG, 2 A2A) and writes the level (-1 when none). */
int orc_pair(const int64_t* sf, const int64_t* sed, int L, int64_t m, int64_t n, int* level) {
  int64_t a[ORC_MAX_LEVELS], b[ORC_MAX_LEVELS];
  orc_renumber(sf, L, m, a);
  orc_renumber(sf, L, n, b);
  int l = L - 1;
  while (l >= 0 && a[l] == b[l]) --l;
  *level = -1;
  if (l < 0) return 0;
  const int64_t da = a[l] / sed[l], oa = a[l] % sed[l];
  const int64_t db = b[l] / sed[l], ob = b[l] % sed[l];
  int t = 0;
  if (da == db && oa != ob) t = 1;
  if (da != db && oa == ob) t = 2;
  if (t) *level = l;
  return t;
}

void orc_topology(const int64_t* sf, const int64_t* sed, int L, int8_t* lvl, uint8_t* typ) {
  const int64_t G = orc_gpus(sf, L);
  for (int64_t m = 0; m < G; ++m)
    for (int64_t n = 0; n < G; ++n) {
      int l = -1;
      const int t = m == n ? 0 : orc_pair(sf, sed, L, m, n, &l);
      lvl[m * G + n] = (int8_t)l;
      typ[m * G + n] = (uint8_t)t;
    }
}

/* Ring-ordered peer lists (simcore.cpp:53-72): per level, AG peers by
 * ((off_n - off_m) mod S_ED, n), A2A peers by ((dom_n - dom_m) mod (SF/S_ED), n). */
void orc_peer_lists(const int64_t* sf, const int64_t* sed, int L, int64_t m, int64_t* ag, int* ag_level,
                    int* n_ag, int64_t* a2a, int* a2a_level, int* n_a2a) {
  const int64_t G = orc_gpus(sf, L);
  int64_t xm[ORC_MAX_LEVELS], xn[ORC_MAX_LEVELS];
  orc_renumber(sf, L, m, xm);
  int na = 0, nb = 0;
  for (int l = 0; l < L; ++l) {
    const int64_t domains = sf[l] / sed[l];
    /* keys are < G, peers < G: key*G + n orders by (key, n). */
    int64_t kag[4096], ka2a[4096];
    int ca = 0, cb = 0;
    for (int64_t n = 0; n < G; ++n) {
      if (n == m) continue;
      int lv;
      const int t = orc_pair(sf, sed, L, m, n, &lv);
      if (lv != l) continue;
      orc_renumber(sf, L, n, xn);
      if (t == 1) kag[ca++] = (((xn[l] % sed[l]) - (xm[l] % sed[l]) + sed[l]) % sed[l]) * G + n;
      if (t == 2) ka2a[cb++] = (((xn[l] / sed[l]) - (xm[l] / sed[l]) + domains) % domains) * G + n;
    }
    for (int i = 1; i < ca; ++i)
      for (int j = i; j > 0 && kag[j] < kag[j - 1]; --j) { int64_t t = kag[j]; kag[j] = kag[j - 1]; kag[j - 1] = t; }
    for (int i = 1; i < cb; ++i)
      for (int j = i; j > 0 && ka2a[j] < ka2a[j - 1]; --j) { int64_t t = ka2a[j]; ka2a[j] = ka2a[j - 1]; ka2a[j - 1] = t; }
    for (int i = 0; i < ca; ++i) { ag[na] = kag[i] % G; ag_level[na++] = l; }
    for (int i = 0; i < cb; ++i) { a2a[nb] = ka2a[i] % G; a2a_level[nb++] = l; }
  }
  *n_ag = na;
  *n_a2a = nb;
}

/* S2 routing: destination of (token on m, expert owned by o).
 * Returns 0 on success, -1 if some pair has no route. */
int orc_route_table(const int64_t* sf, const int64_t* sed, int L, int32_t* route) {
  const int64_t G = orc_gpus(sf, L);
  int64_t* ag = (int64_t*)malloc(sizeof(int64_t) * G);
  int64_t* a2a = (int64_t*)malloc(sizeof(int64_t) * G);
  int* agl = (int*)malloc(sizeof(int) * G);
  int* a2al = (int*)malloc(sizeof(int) * G);
  int rc = 0;
  for (int64_t m = 0; m < G; ++m) {
    int na, nb;
    orc_peer_lists(sf, sed, L, m, ag, agl, &na, a2a, a2al, &nb);
    for (int64_t o = 0; o < G; ++o) {
      int lv;
      int64_t d = -1;
      const int t = m == o ? 0 : orc_pair(sf, sed, L, m, o, &lv);
      if (m == o || t == 1) d = m;
      else if (t == 2) d = o;
      else
        for (int i = 0; i < nb && d < 0; ++i) {
          const int64_t n = a2a[i];
          if (n == o || orc_pair(sf, sed, L, n, o, &lv) == 1) d = n;
        }
      if (d < 0) rc = -1;
      route[m * G + o] = (int32_t)d;
    }
  }
  free(ag); free(a2a); free(agl); free(a2al);
  return rc;
}

/* ------------------------------------------------------------------ SR codec */

/* init_shared: fp64 sum in expert order times (1/n), rounded to fp32 (sparsecomp.cpp:147-168). */
void orc_shared_mean(const float* const* experts, int n, int64_t P, float* out) {
  const double inv = 1.0 / (double)n;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < P; ++i) {
    double acc = 0.0;
    for (int e = 0; e < n; ++e) acc += (double)experts[e][i];
    out[i] = (float)(acc * inv);
  }
}

/* CompressionConfig::resolve_k (sparsecomp.cpp:133-145); ratio used when k < 0. */
int64_t orc_resolve_k(double ratio, int64_t k, uint32_t iw, uint32_t vw, int64_t total, int64_t elem_bytes) {
  if (k >= 0) return k < total ? k : total;
  const double entry = (double)(iw + vw) / 8.0;
  const double kd = floor((double)(total * elem_bytes) / (ratio * entry));
  const int64_t kk = (int64_t)kd;
  return kk < total ? kk : total;
}

static const double* g_sort_r;
static int cmp_rank(const void* pa, const void* pb) {
  const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  const double fa = fabs(g_sort_r[a]), fb = fabs(g_sort_r[b]);
  if (fa != fb) return fa > fb ? -1 : 1;
  return a < b ? -1 : (a > b);
}
static int cmp_idx(const void* pa, const void* pb) {
  const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  return a < b ? -1 : (a > b);
}

/* Top-`budget` of r[lo, hi) by (|r| desc, index asc) (sparsecomp.cpp:44-62),
 * appended to picked; returns the new count. */
static int64_t pick(const double* r, int64_t lo, int64_t hi, int64_t budget, int64_t* picked, int64_t cnt) {
  const int64_t n = hi - lo;
  if (budget <= 0 || n <= 0) return cnt;
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; ++i) idx[i] = lo + i;
  g_sort_r = r;
  qsort(idx, (size_t)n, sizeof(int64_t), cmp_rank);
  if (budget > n) budget = n;
  memcpy(picked + cnt, idx, sizeof(int64_t) * budget);
  free(idx);
  return cnt + budget;
}

static void put_le(uint8_t* p, uint64_t v, int nbytes) {
  for (int i = 0; i < nbytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

/* sr_encode + serialize (sparsecomp.cpp:175-224, :71-97).  expert/shared: flat P fp32
 * (w_up h x m row-major, then w_down m x h).  Returns wire bytes written (caller sizes
 * wire as 28 + k*(iw+vw)/8), or -1 on invalid widths. */
int64_t orc_sr_encode(const float* expert, const float* shared, int64_t h, int64_t m, double ratio, int64_t kreq,
                      uint32_t iw, uint32_t vw, int per_matrix, uint8_t* wire) {
  if ((iw != 32 && iw != 64) || (vw != 32 && vw != 64)) return -1;
  const int64_t up = h * m, P = 2 * h * m;
  double* r = (double*)malloc(sizeof(double) * P);
  for (int64_t i = 0; i < P; ++i) r[i] = (double)expert[i] - (double)shared[i];
  const int64_t k = orc_resolve_k(ratio, kreq, iw, vw, P, 4);
  int64_t* picked = (int64_t*)malloc(sizeof(int64_t) * (k > 0 ? k : 1));
  int64_t cnt = 0;
  if (per_matrix) {
    int64_t k_up = k * up / P;
    if (k_up > up) k_up = up;
    int64_t k_down = k - k_up;
    if (k_down > P - up) k_down = P - up;
    cnt = pick(r, 0, up, k_up, picked, cnt);
    cnt = pick(r, up, P, k_down, picked, cnt);
  } else {
    cnt = pick(r, 0, P, k, picked, cnt);
  }
  qsort(picked, (size_t)cnt, sizeof(int64_t), cmp_idx);
  memcpy(wire, "SRC1", 4);
  put_le(wire + 4, (uint64_t)h, 4);
  put_le(wire + 8, (uint64_t)m, 4);
  put_le(wire + 12, (uint64_t)cnt, 8);
  put_le(wire + 20, iw, 4);
  put_le(wire + 24, vw, 4);
  uint8_t* p = wire + 28;
  for (int64_t j = 0; j < cnt; ++j) {
    put_le(p, (uint64_t)picked[j], (int)(iw / 8));
    p += iw / 8;
    const double v = r[picked[j]];
    if (vw == 32) {
      const float f = (float)v;
      uint32_t b;
      memcpy(&b, &f, 4);
      put_le(p, b, 4);
    } else {
      uint64_t b;
      memcpy(&b, &v, 8);
      put_le(p, b, 8);
    }
    p += vw / 8;
  }
  free(r);
  free(picked);
  return (int64_t)(p - wire);
}

static uint64_t get_le(const uint8_t* p, int nbytes) {
  uint64_t v = 0;
  for (int i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

/* deserialize + sr_decode (sparsecomp.cpp:99-131, :226-246).  Returns the status code
 * used by the device decoder: 0 ok, 1 bad magic, 2 truncated, 3 widths, 4 shape tag,
 * 5 index out of bounds, 6 not increasing. */
int orc_sr_decode(const uint8_t* wire, int64_t bytes, const float* shared, int64_t h, int64_t m, float* out) {
  if (bytes < 4 || memcmp(wire, "SRC1", 4) != 0) return 1;
  if (bytes < 28) return 2;
  const int64_t hh = (int64_t)get_le(wire + 4, 4), mm = (int64_t)get_le(wire + 8, 4);
  const uint64_t k = get_le(wire + 12, 8);
  const uint32_t iw = (uint32_t)get_le(wire + 20, 4), vw = (uint32_t)get_le(wire + 24, 4);
  if ((iw != 32 && iw != 64) || (vw != 32 && vw != 64)) return 3;
  const uint64_t eb = (iw + vw) / 8;
  if (k > (uint64_t)(bytes - 28) / eb) return 2;
  if (hh != h || mm != m) return 4;
  const uint64_t P = (uint64_t)(2 * h * m);
  memcpy(out, shared, sizeof(float) * P);
  const uint8_t* p = wire + 28;
  uint64_t prev_plus_one = 0;
  for (uint64_t j = 0; j < k; ++j, p += eb) {
    const uint64_t idx = get_le(p, (int)(iw / 8));
    double v;
    if (vw == 32) {
      const uint32_t b = (uint32_t)get_le(p + iw / 8, 4);
      float f;
      memcpy(&f, &b, 4);
      v = (double)f;
    } else {
      const uint64_t b = get_le(p + iw / 8, 8);
      memcpy(&v, &b, 8);
    }
    if (idx >= P) return 5;
    if (idx + 1 <= prev_plus_one) return 6;
    prev_plus_one = idx + 1;
    out[idx] = (float)((double)out[idx] + v);
  }
  return 0;
}

/* The optimizer step the fused SR encode applies (hep_sr_encode_update_batch): plain SGD
 * with one rounding, m = fmaf(-lr, g, m).  The reference has no optimizer; its Optimizer
 * job only carries the encode cost (simcore.cpp:126). */
void orc_sgd_step(float* m, const float* g, float lr, int64_t n) {
  for (int64_t i = 0; i < n; ++i) m[i] = fmaf(-lr, g[i], m[i]);
}

/* ------------------------------------------------------------------ MoE layer */

static float bf16_round(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f; /* inf/nan untouched */
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return f;
}

/* S3 gate: logits = x . W_g (W_g H x E), accumulated in fp64 (exact for the dyadic
 * inputs the parity tests use), top-k by (logit desc, id asc), softmax over the k
 * in fp32.  x: T x H fp32 values. */
void orc_gate(const float* x, const float* wg, int64_t T, int64_t H, int64_t E, int64_t k, int32_t* idx,
              float* w) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    float logit[64];
    for (int64_t e = 0; e < E; ++e) {
      double acc = 0.0;
      for (int64_t h = 0; h < H; ++h) acc += (double)x[t * H + h] * (double)wg[h * E + e];
      logit[e] = (float)acc;
    }
    int used[64] = {0};
    float sel[8];
    for (int64_t j = 0; j < k; ++j) {
      int64_t best = -1;
      for (int64_t e = 0; e < E; ++e)
        if (!used[e] && (best < 0 || logit[e] > logit[best])) best = e;
      used[best] = 1;
      sel[j] = logit[best];
      idx[t * k + j] = (int32_t)best;
    }
    float ex[8], s = 0.f;
    for (int64_t j = 0; j < k; ++j) {
      ex[j] = expf(sel[j] - sel[0]);
      s += ex[j];
    }
    for (int64_t j = 0; j < k; ++j) w[t * k + j] = ex[j] / s;
  }
}

/* S4 expert FFN for one row: y = relu(x . w_up) . w_down, fp64 accumulation.
 * bf16 mode mirrors the device rounding points: h and y are rounded to bf16.  The
 * definition the batched layer below reproduces bit for bit (tests/test_oracle.py). */
void orc_ffn_row(const float* x, const float* w_up, const float* w_down, int64_t H, int64_t F, int bf16,
                 double* hacc, double* yacc, float* y) {
  for (int64_t f = 0; f < F; ++f) hacc[f] = 0.0;
  for (int64_t h = 0; h < H; ++h) {
    const double xv = (double)x[h];
    if (xv == 0.0) continue;
    const float* row = w_up + h * F;
    for (int64_t f = 0; f < F; ++f) hacc[f] += xv * (double)row[f];
  }
  for (int64_t c = 0; c < H; ++c) yacc[c] = 0.0;
  for (int64_t f = 0; f < F; ++f) {
    float hv = (float)hacc[f];
    hv = hv > 0.f ? hv : 0.f;
    if (bf16) hv = bf16_round(hv);
    if (hv == 0.f) continue;
    const float* row = w_down + f * H;
    for (int64_t c = 0; c < H; ++c) yacc[c] += (double)hv * (double)row[c];
  }
  for (int64_t c = 0; c < H; ++c) y[c] = bf16 ? bf16_round((float)yacc[c]) : (float)yacc[c];
}

/* One MoE layer over G simulated GPUs (S1-S7).
 *   bf16:   0 = fp32 layer; 1 = bf16 layer mirroring the device rounding points (bf16
 *           W_g for routing, h, y_expert and y rounded to bf16); 2 = the fp32 reference
 *           of a bf16 layer: the same bf16 routing (bf16 W_g, so the experts match), but
 *           h, y_expert and y kept unrounded (fp64 accumulate, fp32 results) -- the
 *           reference a bf16 layer's accuracy is stated against (north_star).
 *   x:      G*T*H (fp32 values; bf16-representable when bf16 != 0)
 *   wg:     H*E
 *   w_up:   E*H*F, w_down: E*F*H (reference layout per expert)
 *   y:      G*T*H output (bf16-rounded when bf16)
 *   topk_idx/topk_w: G*T*k; pos: G*T*k row of (t, j) in GPU g's packed buffer
 *   key_counts: G * (G*E) rows per (dest, expert) key, per source GPU
 *   stride: FFN + combine only for tokens t with t % stride == 0 (routing, packing
 *           and counts always cover every token); y rows of skipped tokens are 0.
 * Returns 0, or -1 when the route table has a hole. */
int orc_moe_layer(int bf16, const float* x, const float* wg, const float* w_up, const float* w_down, int64_t G,
                  int64_t T, int64_t H, int64_t F, int64_t E, int64_t k, const int64_t* sf, const int64_t* sed,
                  int L, int64_t stride, float* y, int32_t* topk_idx, float* topk_w, int32_t* pos,
                  int32_t* key_counts) {
  if (orc_gpus(sf, L) != G || E % G || k > 8 || E > 64) return -2;
  const int64_t n = E / G, NK = G * E;
  int32_t* route = (int32_t*)malloc(sizeof(int32_t) * G * G);
  if (orc_route_table(sf, sed, L, route)) { free(route); return -1; }
  /* bf16 layers route with bf16 gate weights (the device keeps W_g in the layer dtype). */
  float* wgr = (float*)malloc(sizeof(float) * H * E);
  for (int64_t i = 0; i < H * E; ++i) wgr[i] = bf16 ? bf16_round(wg[i]) : wg[i];
  const int rnd = bf16 == 1; /* mode 2: bf16 routing, unrounded arithmetic */
  for (int64_t g = 0; g < G; ++g)
    orc_gate(x + g * T * H, wgr, T, H, E, k, topk_idx + g * T * k, topk_w + g * T * k);
  free(wgr);
  /* S7: stable counting sort by key = dest*E + e over (t, j). */
  for (int64_t g = 0; g < G; ++g) {
    int32_t* cnt = key_counts + g * NK;
    memset(cnt, 0, sizeof(int32_t) * NK);
    const int32_t* ti = topk_idx + g * T * k;
    for (int64_t i = 0; i < T * k; ++i) cnt[route[g * G + ti[i] / n] * E + ti[i]]++;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * NK);
    int64_t acc = 0;
    for (int64_t key = 0; key < NK; ++key) { off[key] = acc; acc += cnt[key]; }
    for (int64_t i = 0; i < T * k; ++i) {
      const int64_t key = route[g * G + ti[i] / n] * E + ti[i];
      pos[g * T * k + i] = (int32_t)off[key]++;
    }
    free(off);
  }
  /* Expert FFN where the row is processed (the result is independent of which GPU
   * computes it: S1 makes every holder use identical weights), then S5 combine.
   * Batched per expert so each expert's weights stream once, not once per row: the
   * sampled (row, slot) pairs are grouped by expert and the products accumulate in fp64
   * in the same order as ffn_row (h ascending for h, f ascending for y), with the same
   * rounding points -- the per-pair results are identical to ffn_row's. */
  memset(y, 0, sizeof(float) * G * T * H);
  const int64_t rows = G * T;
  int64_t* cnt_e = (int64_t*)calloc((size_t)E + 1, sizeof(int64_t));
  for (int64_t r = 0; r < rows; ++r)
    if ((r % T) % stride == 0)
      for (int64_t j = 0; j < k; ++j) cnt_e[topk_idx[r * k + j] + 1]++;
  for (int64_t e = 0; e < E; ++e) cnt_e[e + 1] += cnt_e[e];
  const int64_t npairs = cnt_e[E];
  int64_t* pair_of = (int64_t*)malloc(sizeof(int64_t) * (npairs ? npairs : 1));  /* r * k + j, grouped by expert */
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)E);
  for (int64_t e = 0; e < E; ++e) fill[e] = cnt_e[e];
  for (int64_t r = 0; r < rows; ++r)
    if ((r % T) % stride == 0)
      for (int64_t j = 0; j < k; ++j) pair_of[fill[topk_idx[r * k + j]]++] = r * k + j;
  float* pout = (float*)malloc(sizeof(float) * (size_t)(npairs ? npairs : 1) * H);  /* expert output per pair */
  const int64_t CB = 256;
  for (int64_t e = 0; e < E; ++e) {
    const int64_t p0 = cnt_e[e], ne = cnt_e[e + 1] - p0;
    if (ne == 0) continue;
    float* hm = (float*)malloc(sizeof(float) * ne * F);
    const float* wu = w_up + e * H * F;
    const float* wd = w_down + e * F * H;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t f0 = 0; f0 < F; f0 += CB) {
      const int64_t nb = F - f0 < CB ? F - f0 : CB;
      double* acc = (double*)calloc((size_t)(ne * nb), sizeof(double));
      for (int64_t h = 0; h < H; ++h) {
        const float* row = wu + h * F + f0;
        for (int64_t q = 0; q < ne; ++q) {
          const double xv = (double)x[(pair_of[p0 + q] / k) * H + h];
          if (xv == 0.0) continue;
          double* a = acc + q * nb;
          for (int64_t f = 0; f < nb; ++f) a[f] += xv * (double)row[f];
        }
      }
      for (int64_t q = 0; q < ne; ++q)
        for (int64_t f = 0; f < nb; ++f) {
          float hv = (float)acc[q * nb + f];
          hv = hv > 0.f ? hv : 0.f;
          if (rnd) hv = bf16_round(hv);
          hm[q * F + f0 + f] = hv;
        }
      free(acc);
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c0 = 0; c0 < H; c0 += CB) {
      const int64_t nb = H - c0 < CB ? H - c0 : CB;
      double* acc = (double*)calloc((size_t)(ne * nb), sizeof(double));
      for (int64_t f = 0; f < F; ++f) {
        const float* row = wd + f * H + c0;
        for (int64_t q = 0; q < ne; ++q) {
          const float hv = hm[q * F + f];
          if (hv == 0.f) continue;
          double* a = acc + q * nb;
          for (int64_t c = 0; c < nb; ++c) a[c] += (double)hv * (double)row[c];
        }
      }
      for (int64_t q = 0; q < ne; ++q)
        for (int64_t c = 0; c < nb; ++c)
          pout[(p0 + q) * H + c0 + c] = rnd ? bf16_round((float)acc[q * nb + c]) : (float)acc[q * nb + c];
      free(acc);
    }
    free(hm);
  }
  /* S5: combine in slot order (fmaf, fp32) */
  int64_t* slot_pair = (int64_t*)malloc(sizeof(int64_t) * (size_t)(rows * k));
  for (int64_t p = 0; p < npairs; ++p) slot_pair[pair_of[p]] = p;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    if ((r % T) % stride) continue;
    float acc[8192];
    float* a = H <= 8192 ? acc : (float*)malloc(sizeof(float) * H);
    for (int64_t c = 0; c < H; ++c) a[c] = 0.f;
    for (int64_t j = 0; j < k; ++j) {
      const float* out = pout + slot_pair[r * k + j] * H;
      const float wt = topk_w[r * k + j];
      for (int64_t c = 0; c < H; ++c) a[c] = fmaf(wt, out[c], a[c]);
    }
    for (int64_t c = 0; c < H; ++c) y[r * H + c] = rnd ? bf16_round(a[c]) : a[c];
    if (a != acc) free(a);
  }
  free(slot_pair);
  free(pout);
  free(fill);
  free(pair_of);
  free(cnt_e);
  free(route);
  return 0;
}

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
