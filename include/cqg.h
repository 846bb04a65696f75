/* cqg.h — C ABI of the B200-native patched-forward engine (libcqg.so).
 *
 * Drop-in boundary for the reference's scoring engine. A maintainer of the
 * reference replaces the per-iteration scoring block of run_acdc
 * (proj/src/acdc.cpp:42-60: per-edge policies, refresh_baselines per unique
 * policy, OpenMP fan-out of DeltaLEngine::score) with ONE cqg_score_edges call;
 * see INTEGRATION.md for the C++ shim. Plain pointers and sizes only.
 *
 * Return codes (mirroring the reference's exception classes):
 *   0 ok; 1 invalid argument (std::invalid_argument); 2 runtime error
 *   (std::runtime_error: NaN logits, CUDA/NCCL failure); 3 out of device memory.
 * The message of the last failure on the calling thread: cqg_last_error().
 *
 * Threading: a context is single-threaded; every call blocks until its
 * results are in host memory. Host arrays are borrowed for the call only;
 * the context owns all device memory.
 */
#ifndef CQG_H
#define CQG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ModelConfig minus `batch` (proj/include/circuitquant/model.hpp:31-48),
 * plus qkv_split (EXTENSION, BASELINE config 3's ~32k edges; SPEC.md:166
 * "finer Q/K/V-input edges are a config flag left off by default"): 0 = the
 * reference's graph; 1 = each head has three input receivers (q, k, v
 * inputs, each its own sum and LN), edges numbered for node j asc, then
 * component q, k, v, then source i < j asc (model.cpp:192-201 with the
 * receiver in place of the node). Zero-initialise it in callers that predate
 * the field. */
typedef struct {
  uint32_t n_layers, n_heads, d_model, d_k, vocab, seq_len, has_mlp;
  uint32_t qkv_split;
} cqg_config;

/* PrecisionPolicy (proj/include/circuitquant/precision_policy.hpp:36-58).
 * Precision: 0=P8 1=P16 2=P32; low_mode: 0=E4m3 1=Rtn4 2=INT8 (extension: per-channel
 * weights, per-token activations, RTN conventions of numerics.cpp:105-120 with q <= 127;
 * no reference counterpart, restated in oracle/cq_oracle.c); targets -1 = none. */
typedef struct {
  int8_t attention_default, mlp_default, embed_precision, unembed_precision, low_mode;
  int32_t target_head_layer, target_head_head, target_mlp;
} cqg_policy;

/* PruneConfig (proj/include/circuitquant/acdc.hpp:19-36). */
typedef struct {
  double tau;
  int32_t max_steps;
  double min_change_rate;
  int32_t mode; /* ScoreMode: 0 LossDelta (delta_l), 1 ActDiff */
  double act_floor;
  int32_t per_edge_policy;
  int32_t heads_only;
  cqg_policy base;
} cqg_prune;

typedef struct cqg_ctx cqg_ctx;

/* Metric (patching.hpp:40): 0 KlDivergence, 1 LogitDiff. */
enum { CQG_METRIC_KL = 0, CQG_METRIC_LOGITDIFF = 1 };

/* Creates a context on CUDA device `device`. `mats` are the FP32 masters in
 * canonical for_each_matrix order (replaces ImageBank construction,
 * proj/src/model.cpp:473-503, and WeightStore, proj/src/pahq.cpp:38-51):
 * copied into HBM once; quantized images are built on the device. */
int cqg_create(const cqg_config* cfg, const float* const* mats, int device, cqg_ctx** out);
void cqg_destroy(cqg_ctx* ctx);

/* Replaces DeltaLEngine's dataset (patching.cpp:165-169, validate_dataset
 * 64-81). clean/corrupt are [n_items][seq_len]. `item_offset`/`item_total`
 * describe this rank's shard when the item batch is split across GPUs
 * (score denominators use item_total). */
int cqg_set_dataset(cqg_ctx* ctx, const int32_t* clean, const int32_t* corrupt,
                    const int32_t* answer, const int32_t* distractor, int n_items,
                    int item_offset, int item_total, int metric);

/* Joins an NCCL communicator (one rank per GPU) so cqg_score_edges reduces
 * the per-edge partial sums over ranks (ncclAllReduce, FP64, sum).
 * unique_id is the 128-byte ncclUniqueId from rank 0. */
int cqg_init_comm(cqg_ctx* ctx, const void* unique_id, int rank, int world);
int cqg_get_unique_id(void* out128);

/* The run_acdc scoring block (acdc.cpp:42-60) for one iteration:
 * mask[n_edges] is the graph mask (edge ids per model.cpp:192-201),
 * edge_ids[n] the edges to score; scores_out[n] receives
 * DeltaLEngine::score(edge, policy_for_edge(edge) or base, mode) in
 * edge_ids order. Baselines for the mask are refreshed internally. */
int cqg_score_edges(cqg_ctx* ctx, const uint8_t* mask, const int32_t* edge_ids, int n,
                    const cqg_policy* base, int per_edge_policy, int score_mode,
                    double* scores_out);

/* Whole run_acdc (acdc.cpp:23-88) with the greedy loop on the host (C++) and
 * scoring on the device. Records (step, edge, score, kept) are written in
 * iteration/sweep order up to rec_cap; *n_rec gets the total. */
int cqg_run_acdc(cqg_ctx* ctx, const cqg_prune* cfg, int* steps, uint8_t* final_mask,
                 double* last_score, int* n_rec, int32_t* rec_step, int32_t* rec_edge,
                 double* rec_score, uint8_t* rec_kept, int rec_cap);

/* roc_sweep (proj/src/eval.cpp:1193-1226): cqg_run_acdc at every threshold
 * taus[n_taus] with `cfg` otherwise unchanged; per tau the final mask's TPR /
 * FPR against the ground-truth edge ids, the kept-edge count and the
 * iteration count; *auc = auc_from_points (eval.cpp:1149-1166). Iteration 1
 * (full mask) does not depend on tau: it is scored once and shared by every
 * threshold. Output arrays may be null. */
int cqg_roc_sweep(cqg_ctx* ctx, const cqg_prune* cfg, const double* taus, int n_taus,
                  const int32_t* ground_truth, int n_gt, double* tpr, double* fpr, int32_t* kept,
                  int32_t* steps, double* auc);

/* Quantized image of one canonical matrix as FP32 values (bit-exact to
 * ImageBank::get(name, precision, low_mode), model.cpp:505-519). */
int cqg_quantize_matrix(cqg_ctx* ctx, int matrix_index, int precision, int low_mode,
                        float* out_host);

/* One forward (model.cpp:556-757) of one item's tokens under a policy and
 * mask with an optional single edge patch; writes every node's `out`
 * (S*D floats per node, S*V for the unembed) — a debugging/parity hook. */
int cqg_forward(cqg_ctx* ctx, const int32_t* tokens, const uint8_t* mask, const cqg_policy* pol,
                int patch_edge, const float* patch_value, float* outs_host);

/* circuit_stats (proj/src/eval.cpp:960-985) over the dataset's local items,
 * at FP32: the clean, corrupt and circuit runs' last-row logit differences
 * (metric_logit_diff, patching.cpp:140-149). The circuit run keeps the full
 * graph and gives every edge absent from `mask` its source's output from the
 * corrupt run. faithfulness / task_accuracy (eval.cpp:1240-1254) follow on the
 * host. Each output array has one entry per local item. */
int cqg_circuit_stats(cqg_ctx* ctx, const uint8_t* mask, double* clean_ld, double* corrupt_ld,
                      double* circuit_ld);

/* Graph facts (model.cpp:166-246). */
int cqg_graph_info(const cqg_config* cfg, int* n_nodes, int* n_edges);
int cqg_graph_edges(const cqg_config* cfg, int32_t* edge_src, int32_t* edge_dst);
/* receiver component of each edge: 0/1/2 = q/k/v input of a head under
 * qkv_split, 0 otherwise */
int cqg_graph_edge_comp(const cqg_config* cfg, int32_t* edge_comp);

/* Timing/diagnostic counters of the last cqg_score_edges call. */
typedef struct {
  double ms_total;  /* host wall time of the call */
  double ms_device; /* CUDA-event time on the engine stream, first to last launch */
  double ms_baseline, ms_passes;
  int64_t passes;          /* (edge, item) pairs evaluated on this rank */
  int64_t kernel_launches; /* kernels launched by the call */
  int64_t fallback_elems;  /* tensor-core outputs recomputed on the exact path */
  int64_t h2d_bytes, d2h_bytes;
  int64_t unembed_rows;       /* patched last rows whose logits came from the tensor cores */
  int64_t unembed_exact_rows; /* of those, rows the KL certificate recomputed exactly */
} cqg_stats;
int cqg_last_stats(cqg_ctx* ctx, cqg_stats* out);

/* Per-kernel-class totals of the last cqg_score_edges call: launches,
 * algorithmic FLOPs / HBM bytes, and (with option "profile"=1) CUDA-event
 * device time. Entry i < cqg_profile_count(). */
int cqg_profile_count(cqg_ctx* ctx);
int cqg_profile_entry(cqg_ctx* ctx, int i, char* name64, double* ms, double* flops, double* bytes,
                      int64_t* launches);

/* Engine knobs: 0 = exact SIMT GEMMs everywhere (debug), 1 = tensor cores
 * with exactness-certified fallback (default). */
int cqg_set_option(cqg_ctx* ctx, const char* key, int64_t value);

const char* cqg_last_error(void);
uint64_t cqg_fnv1a64(const void* data, size_t n);

#ifdef __cplusplus
}
#endif
#endif
