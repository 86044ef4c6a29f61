/*
 * hep.h — C-ABI boundary of the B200-native HybridEP MoE-layer hot path.
 *
 * Plain pointers and sizes only (no C++ or torch types); device pointers are
 * CUDA device addresses, `stream` is a cudaStream_t passed as void*.  Every call
 * returns a hep_status; on failure hep_last_error() (thread-local) describes it.
 * Error classes mirror the exceptions the reference throws at the same points
 * (SURVEY.md §8(b)): DOMAIN ~ std::domain_error, INVALID_ARGUMENT ~
 * std::invalid_argument, RUNTIME ~ std::runtime_error.
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj).  The C++ API (include/hybridep/ headers) is layered on the
 * same library; INTEGRATION.md shows the ctypes / C++ bindings.
 */
#ifndef HEP_H_
#define HEP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HEP_OK = 0,
  HEP_ERR_DOMAIN = 1,
  HEP_ERR_INVALID_ARGUMENT = 2,
  HEP_ERR_RUNTIME = 3,
  HEP_ERR_CUDA = 4,
  HEP_ERR_NCCL = 5,
  HEP_ERR_UNSUPPORTED = 6
} hep_status;

typedef enum { HEP_F32 = 0, HEP_BF16 = 1 } hep_dtype;

/* One level of the multilevel description, outermost first
 * (replaces topo::LevelSpec, topology.hpp:19-23). */
typedef struct {
  int64_t scaling_factor; /* SF */
  int64_t domain_size;    /* S_ED */
  double bandwidth;       /* bytes/s */
} hep_level;

const char* hep_last_error(void);
const char* hep_version(void);

/* ------------------------------------------------------------- topology (host) */
/* G = prod SF; validates like ClusterSpec::validate (topology.cpp:35-61). */
int hep_topology_gpus(const hep_level* levels, int num_levels, int64_t* gpus);
/* Dense G x G pair table, row-major m*G+n: pair_level (-1 = none) and pair_type
 * (0 none, 1 AG, 2 A2A).  Replaces CommTopology::CommTopology (topology.cpp:142-177). */
int hep_topology_build(const hep_level* levels, int num_levels, int8_t* pair_level,
                       uint8_t* pair_type);
/* f(m): coords[num_levels].  Replaces topo::renumber (topology.cpp:74-83). */
int hep_renumber(const hep_level* levels, int num_levels, int64_t m, int64_t* coords);
/* Inverse of f.  Replaces topo::global_index (topology.cpp:85-97). */
int hep_global_index(const hep_level* levels, int num_levels, const int64_t* coords, int64_t* m);
/* Algorithm 1 for one (m, n, level).  Replaces topo::comm_type (topology.cpp:117-131). */
int hep_comm_type(const hep_level* levels, int num_levels, int64_t m, int64_t n, int level,
                  int* type);
/* Closed-form directed pair counts per level.  Replaces level_frequency_closed_form
 * via CommTopology::frequencies (topology.cpp:133-153). */
int hep_level_frequency(const hep_level* levels, int num_levels, int64_t* a2a, int64_t* ag);
/* Per-level bytes of one pass (stripe model).  Replaces topo::traffic_report
 * (topology.cpp:249-281).  Outputs are arrays of num_levels. */
int hep_traffic_report(const hep_level* levels, int num_levels, double data_size_D,
                       double expert_size_PE, double token_multiplier, double* a2a_pair_bytes,
                       double* ag_pair_bytes, double* a2a_bytes, double* ag_bytes);
/* Ring-ordered peer lists of GPU m (simcore.cpp:30-74), flattened over levels
 * (outermost first); *_level[i] is the level of peer i.  Arrays hold >= G entries. */
int hep_peer_lists(const hep_level* levels, int num_levels, int64_t m, int64_t* ag_peers,
                   int* ag_level, int* n_ag, int64_t* a2a_peers, int* a2a_level, int* n_a2a);
/* route[m*G+o] = GPU computing, for tokens on m, the experts owned by o (S2 rule). */
int hep_route_table(const hep_level* levels, int num_levels, int32_t* route);
/* Innermost-first gcd split (plan.cpp:41-58). */
int hep_factor_domain_sizes(int64_t domain_size, const hep_level* levels, int num_levels,
                            int64_t* out);

/* ------------------------------------------------------------- planner (host) */
typedef struct {
  double data_size_D, expert_size_PE;
  int64_t experts_per_gpu_n, pre_blocks_m;
  double attn_latency, ffn_latency, expert_latency, backward_allreduce_const;
} hep_workload;
/* Divisor-grid solver (perfmodel.cpp:200-217): returns p, S_ED and the modelled
 * latency terms {comp, pre_expert, comm_a2a, comm_ag, overlap, total}. */
int hep_solve_optimal_p(const hep_workload* w, double throughput_C, double bandwidth_B,
                        int64_t gpus, double* p, int64_t* domain_size, double* latency6);

/* The planner with its reports, as the reference's `plan` + `topo` commands produce them
 * (resolve_plan, cli_app.cpp:132-168; plan.json / freq.json / topo.csv, :183-243) but fed
 * measured device numbers instead of a JSON config: the solver's S_ED, or
 * pinned_domain_sizes[num_levels] when not NULL.  Writes the three files into out_dir
 * (NULL or "": no files); returns p, the per-level S_ED (num_levels entries) and the
 * modelled latency terms {comp, pre_expert, comm_a2a, comm_ag, overlap, total}. */
int hep_plan_reports(const hep_level* levels, int num_levels, const hep_workload* w, double throughput_C,
                     double bandwidth_B, const int64_t* pinned_domain_sizes, const char* out_dir, double* p,
                     int64_t* domain_sizes, double* latency6);

/* ------------------------------------------------------------- SR migration codec */
typedef struct {
  double ratio_CR;           /* used when k < 0 */
  int64_t k;                 /* explicit budget (>= 0 wins), clamped to P */
  uint32_t index_width_bits; /* 32 or 64 */
  uint32_t value_width_bits; /* 32 or 64 */
  int per_matrix_budget;
} hep_sr_config;

/* CompressionConfig::resolve_k (sparsecomp.cpp:133-145). */
int hep_sr_resolve_k(const hep_sr_config* cfg, int64_t total_elements, int64_t elem_bytes,
                     int64_t* k);
/* Exact SRC1 wire size of one expert of shape (h, m) under cfg (header + k entries). */
int hep_sr_wire_bytes(int64_t h, int64_t m, const hep_sr_config* cfg, size_t* bytes);
/* Device scratch for encoding `batch` experts of shape (h, m) at once. */
int hep_sr_workspace_bytes(int64_t h, int64_t m, int batch, size_t* bytes);
/* Device encode = sr_encode + serialize (sparsecomp.cpp:175-224, :71-97).
 * expert: flat P = 2hm elements (w_up h x m then w_down m x h, row-major), fp32 or
 * bf16 (upcast exactly); shared: fp32 flat P.  wire: device buffer of
 * hep_sr_wire_bytes bytes.  Asynchronous; no host synchronisation. */
int hep_sr_encode(const void* expert, hep_dtype expert_dtype, const float* shared, int64_t h,
                  int64_t m, const hep_sr_config* cfg, void* wire, size_t wire_capacity,
                  void* workspace, size_t workspace_bytes, void* stream);
/* Batched encode: n experts (host array of device pointers, same shape, same shared
 * expert) into n wires (host array of device pointers) in one launch sequence. */
int hep_sr_encode_batch(const void* const* experts, int n, hep_dtype expert_dtype, const float* shared,
                        int64_t h, int64_t m, const hep_sr_config* cfg, void* const* wires,
                        size_t wire_capacity, void* workspace, size_t workspace_bytes, void* stream);
/* The paper's SREncode fused with the optimizer step (-30% claimed at
 * :1185; the Optimizer job that carries the encode, simcore.cpp:126): masters[b] (fp32 flat
 * P, device) <- fmaf(-lr, grads[b], masters[b]), and wires[b] = the SRC1 encode of the
 * stepped master against `shared` -- byte-identical to hep_sgd_step_batch followed by
 * hep_sr_encode_batch.  The encode's one full read applies and writes back the step
 * (when every range is list-selected; otherwise the step runs as its own pass first). */
int hep_sr_encode_update_batch(float* const* masters, const float* const* grads, int n, float lr, const float* shared,
                               int64_t h, int64_t m, const hep_sr_config* cfg, void* const* wires, size_t wire_capacity,
                               void* workspace, size_t workspace_bytes, void* stream);
/* The unfused step: masters[b][i] = fmaf(-lr, grads[b][i], masters[b][i]), i < elements. */
int hep_sgd_step_batch(float* const* masters, const float* const* grads, int n, int64_t elements, float lr,
                       void* stream);
/* Device decode = deserialize + sr_decode (sparsecomp.cpp:99-131, :226-246).
 * out: fp32 flat P.  status: device int32[4] (16 bytes); status[0] after the stream
 * reaches this point: 0 ok, 1 bad magic, 2 truncated, 3 bad widths, 4 shape tag
 * mismatch, 5 index out of bounds, 6 indices not increasing (status[1] = entry). */
int hep_sr_decode(const void* wire, size_t wire_bytes, const float* shared, int64_t h, int64_t m,
                  float* out, int32_t* status, void* stream);
/* Batched decode of n wires of wire_bytes each; status: device int32[4*n]. */
int hep_sr_decode_batch(const void* const* wires, int n, size_t wire_bytes, const float* shared, int64_t h,
                        int64_t m, float* const* outs, int32_t* status, void* stream);
/* Synchronises `stream` and maps a decode status to a hep_status + message
 * (RUNTIME for corrupt wires, INVALID_ARGUMENT for a shape mismatch). */
int hep_sr_check_status(const int32_t* status, void* stream);
/* init_shared / update_shared (sparsecomp.cpp:147-173): experts = host array of n
 * device pointers to flat P elements. */
int hep_shared_mean(const void* const* experts, int n, hep_dtype dtype, int64_t P, float* out,
                    void* stream);

/* ------------------------------------------------------------- communicator */
typedef struct hep_comm_s* hep_comm_t;
/* 128-byte NCCL unique id, to be broadcast by the caller (e.g. torch.distributed). */
int hep_comm_unique_id(void* id128);
int hep_comm_init(const void* id128, int rank, int nranks, hep_comm_t* comm);
/* Virtual ranks: `nranks` communicators for nranks ranks driven by ONE process on ONE
 * device (comms[r] is rank r).  The peer-memory step runs unchanged -- count exchange,
 * NVLink-path dispatch stores, GEMM peer-store epilogue, epoch flags, expert All-Gather
 * pulls, the shared-expert chain -- with peers' buffers exchanged as device pointers
 * instead of CUDA IPC handles.  Every rank needs its own stream; rank r's k-th layer
 * pairs with every other rank's k-th layer.  No NCCL (HEP_COMM=nccl is rejected).
 * Replaces nothing in the reference (its "GPUs" are integer indices in one process,
 * simcore.cpp:268-367): it is how a one-GPU box runs the multi-GPU data path. */
int hep_comm_init_virtual(int nranks, hep_comm_t* comms);
int hep_comm_destroy(hep_comm_t comm);

/* ------------------------------------------------------------- MoE layer step */
typedef struct {
  int64_t hidden;      /* H */
  int64_t ffn;         /* F (the reference's inner_m) */
  int64_t experts;     /* E, global */
  int64_t top_k;       /* k */
  int64_t max_tokens;  /* T capacity per GPU */
  hep_dtype dtype;     /* activations and expert weights */
  const hep_level* levels;
  int num_levels;
  int rank;            /* this GPU's global index m */
  int use_sr;          /* migrate gathered experts as SR wires instead of dense */
  hep_sr_config sr;
} hep_layer_params;

typedef struct hep_layer_s* hep_layer_t;

/* comm may be NULL when G == 1.  Selects the current CUDA device's resources. */
int hep_layer_create(const hep_layer_params* params, hep_comm_t comm, hep_layer_t* layer);
int hep_layer_destroy(hep_layer_t layer);
/* Gate matrix W_g, H x E row-major (logits = x . W_g), device pointer, dtype F32 or BF16. */
int hep_layer_set_gate(hep_layer_t layer, const void* w_gate, hep_dtype dtype, void* stream);
/* One owned expert (global id e, owner(e) == rank): w_up H x F, w_down F x H row-major
 * (reference layout, sparsecomp.hpp:29-36), device pointers. */
int hep_layer_set_expert(hep_layer_t layer, int64_t expert, const void* w_up, const void* w_down,
                         hep_dtype dtype, void* stream);
/* SR mode: the shared expert (fp32 flat P, device) that residuals are coded against. */
int hep_layer_set_shared(hep_layer_t layer, const float* shared, void* stream);
/* SR mode: recompute the shared expert from the owned experts of every rank — the
 * element-wise mean over ALL E experts, fp64 sum in expert order times 1/E, rounded to
 * fp32 (replaces sr::init_shared / sr::update_shared, sparsecomp.cpp:147-173, whose
 * update_shared is the single-process stand-in for the paper's async all-reduce).
 * Bit-exact with the reference: a chain over ranks 0..G-1 (experts are owned in rank
 * order), pipelined in chunks over NVLink peer memory (NCCL send/recv + broadcast on the
 * HEP_COMM=nccl path).  Collective: every rank calls it on its stream. */
int hep_layer_refresh_shared(hep_layer_t layer, void* stream);
/* SR mode: the optimizer step of this rank's owned experts fused with their migration
 * encode: grads[i] (fp32 flat P, reference layout, device) for owned expert rank*n + i,
 * i < n.  Updates the fp32 masters and the compute copies and leaves the wires encoded for
 * the next hep_layer_gather_experts, which then skips its own encode. */
int hep_layer_sgd_step(hep_layer_t layer, const float* const* grads, int n, float lr, void* stream);
/* SR mode: copy of the current fp32 shared expert (flat P) into `out` (device). */
int hep_layer_get_shared(hep_layer_t layer, float* out, void* stream);
/* Expert-domain All-Gather of the owned experts (dense or SR-migrated), so that every
 * held expert is resident.  Issued on `stream`. */
int hep_layer_gather_experts(hep_layer_t layer, void* stream);
/* The All-Gather queue of a layer stack (the paper's per-layer send/recv queues,
 * PAPER.md:258-266; "AgTransfer for all layers eligible from t=0", simcore.cpp:155-174):
 * issues every layer's expert All-Gather at once at the start of an iteration.  On the
 * peer-memory path the pulls run in layer order on the rank's All-Gather stream (copy
 * engines) while the layers compute; each layer's forward waits only for its own. */
int hep_layers_gather(hep_layer_t* layers, int n, void* stream);
/* The step: gate -> permute -> dispatch -> expert FFN -> combine.  x, y: device
 * [tokens, H] in the layer dtype, 0 <= tokens <= max_tokens (tokens may differ between
 * GPUs; a GPU with tokens = 0 still takes part and serves its peers' rows). */
int hep_layer_forward(hep_layer_t layer, const void* x, int64_t tokens, void* y, void* stream);
/* The step in residual form, y = x + MoE(x) (how a transformer stack applies the layer):
 * the add is fused into the combine, which accumulates from x's row (one rounding).
 * y must not alias x. */
int hep_layer_forward_residual(hep_layer_t layer, const void* x, int64_t tokens, void* y, void* stream);
/* Same step with host buffers (pinned recommended): H2D copy, forward, D2H copy.
 * Asynchronous and double-buffered: the H2D of the next call and the D2H of the
 * previous one run on the copy engines while this step computes on `stream`.
 * host_y is complete once `stream` passes hep_layer_host_fence (or the device syncs). */
int hep_layer_forward_host(hep_layer_t layer, const void* host_x, int64_t tokens, void* host_y,
                           void* stream);
int hep_layer_host_fence(hep_layer_t layer, void* stream);
/* Synchronises `stream` and the layer's pending All-Gather and reports a migrated expert
 * whose SR wire failed to decode (RUNTIME: bad magic, truncation, out-of-order or
 * out-of-range indices -- the errors sr_decode throws, sparsecomp.cpp:36, 236-238).
 * forward / gather_experts also raise it, without synchronising, once the failed decode
 * has completed. */
int hep_layer_check(hep_layer_t layer, void* stream);
/* Communication microbenchmark of this layer's exchanges (A2A dispatch over NVLink peer
 * memory; expert All-Gather): out6 = {a2a_ms, a2a_bytes_sent, 0, ag_ms, ag_bytes_received,
 * ag_pull_ms}, per GPU, averaged over `iters`.  ag_ms is the whole gather (SR: encode, flags,
 * pulls, decode); ag_pull_ms the same peer pulls alone.  Collective: every rank calls it. */
int hep_layer_comm_bench(hep_layer_t layer, const void* x, int64_t tokens, int iters, double* out6,
                         void* stream);
/* Introspection of the last forward (device pointers owned by the layer):
 * topk_idx int32[T*k], topk_w f32[T*k], pos int32[T*k] (row of (t,j) in the packed
 * buffer), packed [rows, H] send buffer grouped by (dest, expert); counts int32[G*E]
 * rows per (dest, expert) key.  With HEP_GATHER_A=1 the one-GPU step does not write the
 * packed buffer; requesting `packed` then re-runs the permute from the last forward's x
 * (device-synchronous), so that x must still be allocated. */
int hep_layer_debug(hep_layer_t layer, const int32_t** topk_idx, const float** topk_w,
                    const int32_t** pos, const void** packed, const int32_t** key_counts);
/* Per-phase device times (ms, mean per forward since the last call); names is a
 * ';'-separated list.  hep_layer_set_profiling(layer, level): 0 off, 1 CUDA events
 * around the expert GEMM launches only (cheap enough for a timed pass), 2 events at every
 * phase boundary. */
int hep_layer_set_profiling(hep_layer_t layer, int on);
int hep_layer_timings(hep_layer_t layer, char* names, size_t names_cap, float* ms, int cap,
                      int* count);
/* Number of kernels the last forward launched (this library's own kernels). */
int hep_layer_launch_count(hep_layer_t layer, int* count);
/* Test hook: the next SR All-Gather overwrites the magic of the first gathered wire after
 * the pull and before decode (exercises the rejection path above). */
int hep_layer_debug_corrupt_next_gather(hep_layer_t layer);
/* The L2-policy/raster words the layer's bf16 expert GEMMs run with (up, down); see
 * hep_grouped_gemm's `sched`. */
int hep_layer_gemm_schedule(hep_layer_t layer, uint32_t* up, uint32_t* down);

/* ------------------------------------------------------------- kernel-level entry points */
/* Routing of one GPU's tokens without moving them (gate + top-k + S2 destination +
 * S7 stable counting sort), as the step runs it on GPU `rank` of the cluster:
 * x [T, H] and w_gate [H, E] on the device in `dtype`; outputs (device):
 * topk_idx int32[T*k], topk_w f32[T*k], pos int32[T*k] (row in the packed send buffer),
 * key_counts int32[G*E] (rows per (dest, expert)).  Lets one GPU verify every rank of a
 * G-GPU hierarchy (cfg2's S_ED sweep). */
int hep_route_plan(const hep_level* levels, int num_levels, int rank, hep_dtype dtype, const void* x,
                   int64_t tokens, int64_t hidden, const void* w_gate, int64_t experts, int64_t top_k,
                   int32_t* topk_idx, float* topk_w, int32_t* pos, int32_t* key_counts, void* stream);
/* Exposed for parity tests and for frameworks that own their buffers.
 * C[r, n] = act(sum_k A[r, k] B[slot(g) N + n, k]) for the rows r of group g.
 * bf16: the tcgen05 grouped GEMM the layer runs; sched = 0 picks the layer's schedule for
 * this shape (gemm_schedule), any other value is the raw L2-policy/raster word (bits 0-1
 * L2 policy of A, 2-3 of B, 4-5 raster, 8-15 super-row height; e.g. 0x822 = super-rows
 * of 8 m-tiles, A evict_last).  fp32: the layer's 3xTF32 tcgen05 path (sched ignored). */
int hep_grouped_gemm(hep_dtype dtype, const void* A, int64_t a_rows, const void* B,
                     int64_t b_slots, void* C, int64_t N, int64_t K, const int32_t* g_row_start,
                     const int32_t* g_rows, const int32_t* g_slot, int num_groups, int relu,
                     uint32_t sched, void* stream);
/* Reference layout [rows, cols] -> compute layout [cols, rows] (K-major weight copy). */
int hep_transpose_convert(hep_dtype in_dtype, const void* in, int64_t rows, int64_t cols,
                          hep_dtype out_dtype, void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HEP_H_ */
