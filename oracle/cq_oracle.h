/* cq_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's per-edge patched-forward hot path
 * (circuitquant, /root/reference/proj). Used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg as the CHECKER. The product library
 * (paper_2510_23264_b200/libcqg.so) never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement bit-for-bit
 * against the reference library compiled in place (oracle/_ref/libcqref.so)
 * and against the reference tests' frozen values (tests/golden/).
 */
#ifndef CQ_ORACLE_H
#define CQ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Precision (numerics.hpp:19) and LowMode (numerics.hpp:25). */
enum { CQO_P8 = 0, CQO_P16 = 1, CQO_P32 = 2 };
enum { CQO_E4M3 = 0, CQO_RTN4 = 1, CQO_INT8 = 2 /* extension: INT8 per-channel RTN */ };
/* NodeKind (precision_policy.hpp:25). */
enum { CQO_EMBED = 0, CQO_HEAD = 1, CQO_MLP = 2, CQO_UNEMBED = 3 };

typedef struct {
  int8_t attention_default, mlp_default, embed_precision, unembed_precision, low_mode;
  int32_t target_head_layer, target_head_head; /* -1: none */
  int32_t target_mlp;                          /* -1: none */
} cqo_policy;

typedef struct {
  double tau;
  int32_t max_steps;
  double min_change_rate;
  int32_t mode; /* 0 loss (delta_l), 1 act (act_diff) */
  double act_floor;
  int32_t per_edge_policy;
  int32_t heads_only;
  cqo_policy base;
} cqo_prune;

typedef struct cqo_model cqo_model;

/* numerics.cpp:41-101, 105-143 */
uint8_t cqo_encode_f8(double x);
double cqo_decode_f8(uint8_t b);
uint16_t cqo_encode_bf16(float x);
float cqo_decode_bf16(uint16_t b);
float cqo_round_f8(float x);
float cqo_round_bf16(float x);
int cqo_quantize_rtn(float* x, int64_t n, int bits, double* delta);

/* cfg7 = {n_layers, n_heads, d_model, d_k, vocab, seq_len, has_mlp};
 * mats = canonical for_each_matrix order (model.cpp:285-308). Copies. */
cqo_model* cqo_model_new(const uint32_t* cfg7, const float* const* mats);
/* split != 0: the Q/K/V-split edge graph (extension; each head has q / k / v
 * input receivers, edges numbered for receiver asc, then source asc) */
cqo_model* cqo_model_new_split(const uint32_t* cfg7, const float* const* mats, int split);
void cqo_graph_comp(const cqo_model* m, int* comp);
int cqo_split(const cqo_model* m);
void cqo_model_free(cqo_model* m);
int cqo_n_nodes(const cqo_model* m);
int cqo_n_edges(const cqo_model* m);
void cqo_graph(const cqo_model* m, int* node_kind, int* node_layer, int* node_head,
               int* edge_src, int* edge_dst);
int cqo_sweep_order(const cqo_model* m, const uint8_t* mask, int* out);
int cqo_image(const cqo_model* m, int matrix_index, int precision, int low_mode, float* out);

/* forward (model.cpp:556-757): outs receives every node's out in node
 * order (S*D floats per node, S*V for unembed). */
int cqo_forward(const cqo_model* m, const int* tokens, const uint8_t* mask, const cqo_policy* pol,
                int patch_edge, const float* patch_value, float* outs);

double cqo_metric_kl(const float* clean, const float* patched, int64_t n);

/* The run_acdc scoring block (acdc.cpp:42-60) for a list of edges. */
int cqo_score_edges(const cqo_model* m, const int* clean, const int* corrupt, const int* answer,
                    const int* distractor, int n_items, const uint8_t* mask, const int* edges,
                    int n, const cqo_policy* base, int per_edge_policy, int metric, int mode,
                    double* out);

/* run_acdc (acdc.cpp:23-88) from the full mask. */
int cqo_run_acdc(const cqo_model* m, const int* clean, const int* corrupt, const int* answer,
                 const int* distractor, int n_items, int metric, const cqo_prune* pc, int* steps,
                 uint8_t* final_mask, double* last_score, int* n_rec, int* rec_step,
                 int* rec_edge, double* rec_score, uint8_t* rec_kept, int rec_cap);

const char* cqo_last_error(void);

void cqo_libm_range(int which, uint32_t lo, uint64_t count, float* out);
void cqo_codes_range(uint32_t lo, uint64_t count, uint8_t* f8, uint16_t* bf16);

#ifdef __cplusplus
}
#endif
#endif
