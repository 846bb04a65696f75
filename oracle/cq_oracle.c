/* cq_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference's patched-forward hot path
 * (/root/reference/proj, "circuitquant"). Every function cites the reference
 * file:line it restates. Compiled with -ffp-contract=off so every float
 * operation rounds exactly where the reference's (FMA-free)
 * code rounds; libm calls (expf, erff, sqrtf, exp, log) are the same glibc
 * entry points the reference calls through <cmath>.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this (as libcqoracle.so).
 */
#include "cq_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* cqo_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* numerics — proj/src/numerics.cpp                                          */
/* ------------------------------------------------------------------------ */

/* round_half_even, numerics.cpp:21-28 */
static int64_t rhe(double q) {
  double fl = floor(q);
  double frac = q - fl;
  int64_t lo = (int64_t)fl;
  if (frac > 0.5) return lo + 1;
  if (frac < 0.5) return lo;
  return (lo % 2 == 0) ? lo : lo + 1;
}

/* encode_f8, numerics.cpp:41-64 */
uint8_t cqo_encode_f8(double x) {
  if (isnan(x)) return 0x7F;
  uint8_t sign = signbit(x) ? 0x80 : 0x00;
  double a = fabs(x);
  if (a == 0.0) return sign;
  if (a > 448.0) return (uint8_t)(sign | 0x7E);
  if (a < 0x1p-6) {
    int64_t m = rhe(a / 0x1p-9);
    if (m == 0) return sign;
    if (m >= 8) return (uint8_t)(sign | 0x08);
    return (uint8_t)(sign | m);
  }
  int e = ilogb(a);
  int64_t m = rhe(ldexp(a, 3 - e));
  if (m == 16) {
    m = 8;
    ++e;
  }
  if (e > 8) return (uint8_t)(sign | 0x7E);
  return (uint8_t)(sign | ((e + 7) << 3) | (m - 8));
}

/* decode_f8, numerics.cpp:66-73 */
double cqo_decode_f8(uint8_t v) {
  int ef = (v >> 3) & 0x0F, mant = v & 0x07;
  double s = (v & 0x80) ? -1.0 : 1.0;
  if (ef == 0x0F && mant == 0x07) return NAN;
  if (ef == 0) return s * (double)mant * 0x1p-9;
  return s * (1.0 + (double)mant / 8.0) * ldexp(1.0, ef - 7);
}

/* encode_bf16 / decode_bf16, numerics.cpp:84-101 */
uint16_t cqo_encode_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if (isnan(x)) return (uint16_t)(((u >> 16) & 0x8000u) | 0x7FC0u);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

float cqo_decode_bf16(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* round_f8 / round_bf16, numerics.cpp:141-143 */
float cqo_round_f8(float x) { return (float)cqo_decode_f8(cqo_encode_f8((double)x)); }
float cqo_round_bf16(float x) { return cqo_decode_bf16(cqo_encode_bf16(x)); }

/* quantize_rtn_impl<float>, numerics.cpp:105-120 */
int cqo_quantize_rtn(float* x, int64_t n, int bits, double* delta_out) {
  if (bits != 4 && bits != 8 && bits != 16)
    return fail(1, "quantize_rtn: n_bits must be 4, 8, or 16");
  double mx = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double a = fabs((double)x[i]);
    if (a > mx) mx = a; /* std::max(max_abs, a): NaN never wins */
  }
  if (delta_out) *delta_out = 0.0;
  if (mx == 0.0) return 0;
  double d = mx / ldexp(1.0, bits - 1);
  for (int64_t i = 0; i < n; ++i) x[i] = (float)(d * (double)rhe((double)x[i] / d));
  if (delta_out) *delta_out = d;
  return 0;
}

/* INT8 RTN of one strided group — EXTENSION (BASELINE config 2), parity
 * unpinned: the reference has no INT8 caller. It follows quantize_rtn's
 * conventions (numerics.cpp:105-120): delta = max|x| / 2^(8-1) in double
 * (all-zero group: unchanged), q = round_half_even(x / delta), value =
 * float(delta * q); plus the INT8 range: q is clamped to 127, so the one
 * value quantize_rtn maps to +128 (a group's positive maximum, cf. the
 * frozen example test_numerics.cpp:221-229 where -2 -> -128) saturates to
 * 127 * delta. -128 is representable and kept. NaN passes through. */
static void rtn8_group(float* x, int64_t n, int64_t stride) {
  double mx = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double a = fabs((double)x[i * stride]);
    if (a > mx) mx = a;
  }
  if (mx == 0.0) return;
  double d = mx / 128.0;
  for (int64_t i = 0; i < n; ++i) {
    double q = rhe((double)x[i * stride] / d);
    if (q > 127.0) q = 127.0;
    x[i * stride] = (float)(d * q);
  }
}

/* quantize_span, kernels.cpp:236-251, on a [n / cols][cols] tensor. P8 +
 * INT8 (extension): one group per row (per token: the last dimension of the
 * tensor the reference quantizes, i.e. dynamic per-token activation scales). */
static void quantize(float* x, int64_t n, int64_t cols, int p, int mode) {
  if (p == CQO_P32) return;
  if (p == CQO_P16) {
    for (int64_t i = 0; i < n; ++i) x[i] = cqo_round_bf16(x[i]);
    return;
  }
  if (mode == CQO_E4M3) {
    for (int64_t i = 0; i < n; ++i) x[i] = cqo_round_f8(x[i]);
  } else if (mode == CQO_INT8) {
    for (int64_t r = 0; r < n / cols; ++r) rtn8_group(x + r * cols, cols, 1);
  } else {
    cqo_quantize_rtn(x, n, 4, NULL);
  }
}

/* ------------------------------------------------------------------------ */
/* model: graph, weights, images — proj/src/model.cpp                        */
/* ------------------------------------------------------------------------ */

enum { MK_WE, MK_WPOS, MK_LN1G, MK_LN1B, MK_WQ, MK_WK, MK_WV, MK_WO, MK_LN2G, MK_LN2B,
       MK_WIN, MK_WOUT, MK_LNFG, MK_LNFB, MK_WU };

struct cqo_model {
  int L, H, D, dk, V, S, mlp;
  int n_nodes, n_edges, n_mats;
  int *kind, *layer, *head, *stage;
  int *esrc, *edst;
  /* receivers (EXTENSION: Q/K/V-split edges, BASELINE config 3's ~32k edges;
   * SPEC.md:166 "finer Q/K/V-input edges are a config flag left off"): a head
   * has 3 input receivers (q, k, v inputs, each its own sum and LN), other
   * nodes 1. Unsplit (the reference's graph): every node 1 receiver. */
  int split, n_recv;
  int *recv_node, *recv_comp, *node_recv; /* node_recv: first receiver of a node (-1: embed) */
  int* erecv;                             /* receiver of each edge */
  int **in_edges, *n_in;                  /* per receiver */
  float** master;
  int64_t* msize;
  int* mkind;  /* MK_* per matrix */
  float** img[4]; /* [0]=P8/E4M3, [1]=P16, [2]=P8/Rtn4, [3]=P8/INT8; NULL until first use */
};

static int mat_index(const cqo_model* m, int mk, int layer) {
  int per = 6 + (m->mlp ? 4 : 0);
  switch (mk) {
    case MK_WE: return 0;
    case MK_WPOS: return 1;
    case MK_LNFG: return 2 + m->L * per;
    case MK_LNFB: return 3 + m->L * per;
    case MK_WU: return 4 + m->L * per;
    default: break;
  }
  int off = mk - MK_LN1G; /* ln1_g..w_out in visit order, model.cpp:292-302 */
  return 2 + layer * per + off;
}

/* node_stage, model.cpp:170-178 */
static int node_stage(const cqo_model* m, int kind, int layer) {
  switch (kind) {
    case CQO_EMBED: return 0;
    case CQO_HEAD: return 1 + 2 * layer;
    case CQO_MLP: return 2 + 2 * layer;
    default: return 1 + 2 * m->L;
  }
}

cqo_model* cqo_model_new_split(const uint32_t* c, const float* const* mats, int split);
cqo_model* cqo_model_new(const uint32_t* c, const float* const* mats) {
  return cqo_model_new_split(c, mats, 0);
}

cqo_model* cqo_model_new_split(const uint32_t* c, const float* const* mats, int split) {
  /* ModelConfig::validate, model.cpp:144-155 */
  if (c[0] < 1 || c[1] < 1 || c[2] < 1 || c[3] < 1 || c[1] * c[3] != c[2] || c[4] < 2 ||
      c[5] < 1 || c[6] > 1) {
    fail(1, "ModelConfig: invalid");
    return NULL;
  }
  cqo_model* m = calloc(1, sizeof *m);
  m->L = (int)c[0];
  m->H = (int)c[1];
  m->D = (int)c[2];
  m->dk = (int)c[3];
  m->V = (int)c[4];
  m->S = (int)c[5];
  m->mlp = (int)c[6];
  /* nodes: embed, per layer H heads then MLP, unembed (model.cpp:184-190) */
  m->n_nodes = 2 + m->L * (m->H + m->mlp);
  m->kind = malloc(sizeof(int) * m->n_nodes);
  m->layer = malloc(sizeof(int) * m->n_nodes);
  m->head = malloc(sizeof(int) * m->n_nodes);
  m->stage = malloc(sizeof(int) * m->n_nodes);
  int k = 0;
  m->kind[k] = CQO_EMBED, m->layer[k] = -1, m->head[k] = -1, ++k;
  for (int l = 0; l < m->L; ++l) {
    for (int h = 0; h < m->H; ++h) m->kind[k] = CQO_HEAD, m->layer[k] = l, m->head[k] = h, ++k;
    if (m->mlp) m->kind[k] = CQO_MLP, m->layer[k] = l, m->head[k] = -1, ++k;
  }
  m->kind[k] = CQO_UNEMBED, m->layer[k] = -1, m->head[k] = -1, ++k;
  for (int i = 0; i < m->n_nodes; ++i) m->stage[i] = node_stage(m, m->kind[i], m->layer[i]);
  /* receivers: node order, then component (q, k, v for split heads) */
  m->split = split ? 1 : 0;
  m->node_recv = malloc(sizeof(int) * m->n_nodes);
  m->recv_node = malloc(sizeof(int) * 3 * m->n_nodes);
  m->recv_comp = malloc(sizeof(int) * 3 * m->n_nodes);
  m->n_recv = 0;
  for (int j = 0; j < m->n_nodes; ++j) {
    m->node_recv[j] = j == 0 ? -1 : m->n_recv;
    int nc = j == 0 ? 0 : (m->split && m->kind[j] == CQO_HEAD ? 3 : 1);
    for (int q = 0; q < nc; ++q) m->recv_node[m->n_recv] = j, m->recv_comp[m->n_recv] = q, ++m->n_recv;
  }
  /* edges: for j asc, for i < j asc, iff stage(i) < stage(j) (model.cpp:192-201);
   * split graph: for receiver r asc (node j asc, component asc), for i < j asc */
  int cap = 3 * m->n_nodes * m->n_nodes / 2 + 1;
  m->esrc = malloc(sizeof(int) * cap);
  m->edst = malloc(sizeof(int) * cap);
  m->erecv = malloc(sizeof(int) * cap);
  m->in_edges = calloc((size_t)m->n_recv, sizeof(int*));
  m->n_in = calloc((size_t)m->n_recv, sizeof(int));
  int ne = 0;
  for (int r = 0; r < m->n_recv; ++r) {
    int j = m->recv_node[r];
    m->in_edges[r] = malloc(sizeof(int) * (size_t)(j + 1));
    for (int i = 0; i < j; ++i) {
      if (m->stage[i] >= m->stage[j]) continue;
      m->esrc[ne] = i;
      m->edst[ne] = j;
      m->erecv[ne] = r;
      m->in_edges[r][m->n_in[r]++] = ne;
      ++ne;
    }
  }
  m->n_edges = ne;
  /* matrices in canonical order (model.cpp:285-308) */
  int per = 6 + (m->mlp ? 4 : 0);
  m->n_mats = 5 + m->L * per;
  m->master = calloc((size_t)m->n_mats, sizeof(float*));
  m->msize = calloc((size_t)m->n_mats, sizeof(int64_t));
  m->mkind = calloc((size_t)m->n_mats, sizeof(int));
  int64_t D = m->D, V = m->V, S = m->S;
  for (int i = 0; i < m->n_mats; ++i) {
    int mk;
    int64_t sz;
    if (i == 0) mk = MK_WE, sz = V * D;
    else if (i == 1) mk = MK_WPOS, sz = S * D;
    else if (i == m->n_mats - 3) mk = MK_LNFG, sz = D;
    else if (i == m->n_mats - 2) mk = MK_LNFB, sz = D;
    else if (i == m->n_mats - 1) mk = MK_WU, sz = D * V;
    else {
      mk = MK_LN1G + (i - 2) % per;
      switch (mk) {
        case MK_LN1G: case MK_LN1B: case MK_LN2G: case MK_LN2B: sz = D; break;
        case MK_WIN: case MK_WOUT: sz = 4 * D * D; break;
        default: sz = D * D;
      }
    }
    m->mkind[i] = mk;
    m->msize[i] = sz;
    m->master[i] = malloc(sizeof(float) * (size_t)sz);
    memcpy(m->master[i], mats[i], sizeof(float) * (size_t)sz);
  }
  return m;
}

void cqo_model_free(cqo_model* m) {
  if (!m) return;
  for (int i = 0; i < m->n_recv; ++i) free(m->in_edges[i]);
  free(m->node_recv), free(m->recv_node), free(m->recv_comp), free(m->erecv);
  for (int i = 0; i < m->n_mats; ++i) free(m->master[i]);
  for (int q = 0; q < 4; ++q) {
    if (!m->img[q]) continue;
    for (int i = 0; i < m->n_mats; ++i) free(m->img[q][i]);
    free(m->img[q]);
  }
  free(m->in_edges), free(m->n_in), free(m->master), free(m->msize), free(m->mkind);
  free(m->kind), free(m->layer), free(m->head), free(m->stage), free(m->esrc), free(m->edst);
  free(m);
}

int cqo_n_nodes(const cqo_model* m) { return m->n_nodes; }
int cqo_n_edges(const cqo_model* m) { return m->n_edges; }

void cqo_graph(const cqo_model* m, int* nk, int* nl, int* nh, int* es, int* ed) {
  for (int i = 0; i < m->n_nodes; ++i) nk[i] = m->kind[i], nl[i] = m->layer[i], nh[i] = m->head[i];
  for (int e = 0; e < m->n_edges; ++e) es[e] = m->esrc[e], ed[e] = m->edst[e];
}

/* component of each edge's receiver: 0 / 1 / 2 = q / k / v input of a head
 * in the split graph, 0 otherwise */
void cqo_graph_comp(const cqo_model* m, int* comp) {
  for (int e = 0; e < m->n_edges; ++e) comp[e] = m->recv_comp[m->erecv[e]];
}
int cqo_split(const cqo_model* m) { return m->split; }

/* sweep_order, model.cpp:238-246 */
int cqo_sweep_order(const cqo_model* m, const uint8_t* mask, int* out) {
  int n = 0;
  for (int j = m->n_recv - 1; j >= 0; --j) /* receivers desc (= dst desc unsplit) */
    for (int t = m->n_in[j] - 1; t >= 0; --t) {
      int e = m->in_edges[j][t];
      if (!mask || mask[e]) out[n++] = e;
    }
  return n;
}

/* quantize_rtn4_matrix, model.cpp:445-469 */
static void rtn4_matrix(const cqo_model* m, int mk, float* t, int64_t size) {
  int64_t dk = m->dk, D = m->D;
  if (mk == MK_WQ || mk == MK_WK || mk == MK_WV) {
    float* tmp = malloc(sizeof(float) * (size_t)(D * dk));
    for (int64_t h = 0; h < m->H; ++h) {
      for (int64_t r = 0; r < D; ++r)
        for (int64_t c = 0; c < dk; ++c) tmp[r * dk + c] = t[r * D + h * dk + c];
      cqo_quantize_rtn(tmp, D * dk, 4, NULL);
      for (int64_t r = 0; r < D; ++r)
        for (int64_t c = 0; c < dk; ++c) t[r * D + h * dk + c] = tmp[r * dk + c];
    }
    free(tmp);
    return;
  }
  if (mk == MK_WO) {
    for (int64_t h = 0; h < m->H; ++h) cqo_quantize_rtn(t + h * dk * D, dk * D, 4, NULL);
    return;
  }
  cqo_quantize_rtn(t, size, 4, NULL);
}

/* INT8 per-channel weight image (extension): one group per output channel
 * of the [in][out] matrix, i.e. per column; W_O per (head, column), its
 * d_k rows of that head (per-head quantization, as Rtn4's W_O head blocks,
 * model.cpp:445-469); vectors (LN parameters, never multiplied) as one group. */
static void int8_matrix(const cqo_model* m, int mk, float* t, int64_t size) {
  int64_t D = m->D, dk = m->dk;
  if (mk == MK_LN1G || mk == MK_LN1B || mk == MK_LN2G || mk == MK_LN2B || mk == MK_LNFG ||
      mk == MK_LNFB) {
    rtn8_group(t, size, 1);
    return;
  }
  if (mk == MK_WO) {
    for (int64_t h = 0; h < m->H; ++h)
      for (int64_t c = 0; c < D; ++c) rtn8_group(t + h * dk * D + c, dk, D);
    return;
  }
  int64_t C = mk == MK_WIN ? 4 * D : (mk == MK_WU ? m->V : D);
  for (int64_t c = 0; c < C; ++c) rtn8_group(t + c, size / C, C);
}

/* ImageBank::get (model.cpp:505-519) with eager per-(precision,mode)
 * materialisation (model.cpp:473-491). */
static const float* image(cqo_model* m, int idx, int p, int mode) {
  if (p == CQO_P32) return m->master[idx];
  int q = p == CQO_P16 ? 1 : (mode == CQO_E4M3 ? 0 : mode == CQO_INT8 ? 3 : 2);
  if (!m->img[q]) {
    m->img[q] = calloc((size_t)m->n_mats, sizeof(float*));
    for (int i = 0; i < m->n_mats; ++i) {
      float* t = malloc(sizeof(float) * (size_t)m->msize[i]);
      memcpy(t, m->master[i], sizeof(float) * (size_t)m->msize[i]);
      if (q == 2) rtn4_matrix(m, m->mkind[i], t, m->msize[i]);
      else if (q == 3) int8_matrix(m, m->mkind[i], t, m->msize[i]);
      else quantize(t, m->msize[i], m->msize[i], p, CQO_E4M3);
      m->img[q][i] = t;
    }
  }
  return m->img[q][idx];
}

int cqo_image(const cqo_model* mc, int idx, int p, int mode, float* out) {
  if (idx < 0 || idx >= mc->n_mats) return fail(1, "cqo_image: bad matrix index");
  const float* t = image((cqo_model*)mc, idx, p, mode);
  memcpy(out, t, sizeof(float) * (size_t)mc->msize[idx]);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* kernels — proj/src/kernels.cpp                                            */
/* ------------------------------------------------------------------------ */

/* dot_col (kernels.cpp:44-52): sequential k, product rounded, then add. */
static inline float dot_col(const float* a, const float* w, int64_t K, int64_t ld, int64_t col) {
  float acc = 0.0f;
  const float* wp = w + col;
  for (int64_t k = 0; k < K; ++k) acc += a[k] * wp[k * ld];
  return acc;
}

/* matmul / matmul_cols (kernels.cpp:56-99): out[M][c1-c0] */
static void matmul_cols(const float* a, int64_t M, int64_t K, const float* w, int64_t ld,
                        int64_t c0, int64_t c1, float* out) {
  int64_t cols = c1 - c0;
  for (int64_t i = 0; i < M; ++i)
    for (int64_t n = 0; n < cols; ++n) out[i * cols + n] = dot_col(a + i * K, w, K, ld, c0 + n);
}

/* layer_norm_row (kernels.cpp:127-142), eps 1e-5f (model.cpp:535) */
static void layer_norm(const float* x, int64_t rows, int64_t d, const float* g, const float* b,
                       float* out) {
  for (int64_t r = 0; r < rows; ++r) {
    const float* xr = x + r * d;
    float mean = 0.0f;
    for (int64_t i = 0; i < d; ++i) mean += xr[i];
    mean /= (float)d;
    float var = 0.0f;
    for (int64_t i = 0; i < d; ++i) {
      float c = xr[i] - mean;
      var += c * c;
    }
    var /= (float)d;
    float inv = 1.0f / sqrtf(var + 1e-5f);
    for (int64_t i = 0; i < d; ++i) out[r * d + i] = g[i] * ((xr[i] - mean) * inv) + b[i];
  }
}

/* attention_row / causal_attention (kernels.cpp:167-219) on [S][dk] rows
 * taken with stride `ld` (head slices of [S][H][dk]). */
static void causal_attention(const float* q, const float* k, const float* v, int64_t ld,
                             int64_t S, int64_t dk, float* z) {
  float scale = 1.0f / sqrtf((float)dk);
  float* pr = malloc(sizeof(float) * (size_t)S);
  for (int64_t i = 0; i < S; ++i) {
    float mx = -INFINITY;
    for (int64_t j = 0; j <= i; ++j) {
      float acc = 0.0f;
      for (int64_t t = 0; t < dk; ++t) acc += q[i * ld + t] * k[j * ld + t];
      pr[j] = acc * scale;
      mx = (mx < pr[j]) ? pr[j] : mx; /* std::max(a, b) == (a < b) ? b : a */
    }
    float den = 0.0f;
    for (int64_t j = 0; j <= i; ++j) {
      pr[j] = expf(pr[j] - mx);
      den += pr[j];
    }
    for (int64_t j = 0; j <= i; ++j) pr[j] /= den;
    for (int64_t t = 0; t < dk; ++t) {
      float acc = 0.0f;
      for (int64_t j = 0; j <= i; ++j) acc += pr[j] * v[j * ld + t];
      z[i * dk + t] = acc;
    }
  }
  free(pr);
}

/* gelu, kernels.cpp:221-234 */
static void gelu(float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) x[i] = 0.5f * x[i] * (1.0f + erff(x[i] * 0.70710678118654752f));
}

/* ------------------------------------------------------------------------ */
/* policy — proj/src/model.cpp:52-71, proj/src/pahq.cpp:198-209             */
/* ------------------------------------------------------------------------ */

static int precision_of(const cqo_policy* p, int kind, int layer, int head) {
  switch (kind) {
    case CQO_EMBED: return p->embed_precision;
    case CQO_UNEMBED: return p->unembed_precision;
    case CQO_HEAD:
      if (p->target_head_layer >= 0 && p->target_head_layer == layer && p->target_head_head == head)
        return CQO_P32;
      return p->attention_default;
    default:
      if (p->target_mlp >= 0 && p->target_mlp == layer) return CQO_P32;
      return p->mlp_default;
  }
}

static int wo_precision(const cqo_policy* p, int layer) {
  if (p->target_head_layer >= 0 && p->target_head_layer == layer) return CQO_P32;
  return p->attention_default;
}

static cqo_policy policy_for_edge(const cqo_model* m, int e, const cqo_policy* base) {
  cqo_policy p = *base;
  p.target_head_layer = p.target_head_head = p.target_mlp = -1;
  int s = m->esrc[e];
  if (m->kind[s] == CQO_HEAD) p.target_head_layer = m->layer[s], p.target_head_head = m->head[s];
  if (m->kind[s] == CQO_MLP) p.target_mlp = m->layer[s];
  return p;
}

static int policy_eq(const cqo_policy* a, const cqo_policy* b) {
  int lm_a = a->low_mode, lm_b = b->low_mode; /* PrecisionPolicy::key, model.cpp:73-83 */
  return a->attention_default == b->attention_default && a->mlp_default == b->mlp_default &&
         a->embed_precision == b->embed_precision && a->unembed_precision == b->unembed_precision &&
         lm_a == lm_b && a->target_head_layer == b->target_head_layer &&
         (a->target_head_layer < 0 || a->target_head_head == b->target_head_head) &&
         a->target_mlp == b->target_mlp;
}

/* ------------------------------------------------------------------------ */
/* forward — proj/src/model.cpp:537-757                                      */
/* ------------------------------------------------------------------------ */

static int64_t node_off(const cqo_model* m, int v) { return (int64_t)v * m->S * m->D; }
static int64_t outs_size(const cqo_model* m) {
  return (int64_t)(m->n_nodes - 1) * m->S * m->D + (int64_t)m->S * m->V;
}

/* sum_inputs, model.cpp:537-552, for receiver v (= the node's one receiver
 * unsplit; a head's q / k / v input in the split graph) */
static void sum_inputs(const cqo_model* m, const uint8_t* mask, const float* outs, int patch_edge,
                       const float* patch_value, int v, float* in) {
  int64_t n = (int64_t)m->S * m->D;
  memset(in, 0, sizeof(float) * (size_t)n);
  for (int t = 0; t < m->n_in[v]; ++t) {
    int e = m->in_edges[v][t];
    if (mask && !mask[e]) continue;
    const float* sp = (e == patch_edge) ? patch_value : outs + node_off(m, m->esrc[e]);
    for (int64_t i = 0; i < n; ++i) in[i] += sp[i];
  }
}

int cqo_forward(const cqo_model* mc, const int* tok, const uint8_t* mask, const cqo_policy* pol,
                int patch_edge, const float* patch_value, float* outs) {
  cqo_model* m = (cqo_model*)mc;
  const int64_t S = m->S, D = m->D, dk = m->dk, V = m->V, H = m->H;
  const int mode = pol->low_mode;
  for (int64_t i = 0; i < S; ++i)
    if (tok[i] < 0 || tok[i] >= V) return fail(1, "forward: token id out of range");
  if (pol->target_head_layer >= 0 &&
      (pol->target_head_layer >= m->L || pol->target_head_head < 0 || pol->target_head_head >= H))
    return fail(1, "forward: target head out of range");
  if (pol->target_mlp >= 0 && (!m->mlp || pol->target_mlp >= m->L))
    return fail(1, "forward: target mlp out of range");
  if (patch_edge >= 0) {
    if (patch_edge >= m->n_edges) return fail(1, "forward: patch references unknown edge");
    if (mask && !mask[patch_edge]) return fail(1, "forward: patch references masked edge");
  }
  float* in = malloc(sizeof(float) * (size_t)(S * D));
  const int NC = m->split ? 3 : 1; /* input receivers per head */
  float* xln = malloc(sizeof(float) * (size_t)(NC * H * S * D)); /* [c][h] */
  float* xq = malloc(sizeof(float) * (size_t)(NC * H * S * D));
  float* low = malloc(sizeof(float) * (size_t)(3 * S * H * dk)); /* [3][S][H][dk] */
  float* tmp = malloc(sizeof(float) * (size_t)(S * (4 * D > V ? 4 * D : V)));
  float* z = malloc(sizeof(float) * (size_t)(S * dk));
  float* hid = malloc(sizeof(float) * (size_t)(S * 4 * D));

  int vi = 0;
  while (vi < m->n_nodes) {
    int kind = m->kind[vi];
    if (kind == CQO_EMBED) { /* model.cpp:608-620 */
      int p = precision_of(pol, kind, -1, -1);
      const float* we = image(m, mat_index(m, MK_WE, 0), p, mode);
      const float* wp = image(m, mat_index(m, MK_WPOS, 0), p, mode);
      float* out = outs + node_off(m, vi);
      for (int64_t i = 0; i < S; ++i)
        for (int64_t j = 0; j < D; ++j) out[i * D + j] = we[(int64_t)tok[i] * D + j] + wp[i * D + j];
      quantize(out, S * D, D, p, mode);
      ++vi;
      continue;
    }
    if (kind == CQO_HEAD) { /* model.cpp:622-718 */
      int l = m->layer[vi], first = vi;
      int p_low = pol->attention_default;
      int target = (pol->target_head_layer == l) ? pol->target_head_head : -1;
      const float* g1 = m->master[mat_index(m, MK_LN1G, l)];
      const float* b1 = m->master[mat_index(m, MK_LN1B, l)];
      for (int q = 0; q < NC; ++q)
        for (int h = 0; h < H; ++h) {
          float* xl = xln + (q * H + h) * S * D;
          sum_inputs(m, mask, outs, patch_edge, patch_value, m->node_recv[first + h] + q, in);
          layer_norm(in, S, D, g1, b1, xl);
          memcpy(xq + (q * H + h) * S * D, xl, sizeof(float) * (size_t)(S * D));
          quantize(xq + (q * H + h) * S * D, S * D, D, p_low, mode);
        }
      const float* wimg[3];
      for (int c = 0; c < 3; ++c) wimg[c] = image(m, mat_index(m, MK_WQ + c, l), p_low, mode);
      const float* wo = image(m, mat_index(m, MK_WO, l), wo_precision(pol, l), mode);
      for (int c = 0; c < 3; ++c) /* low_comp, model.cpp:655-664 (split: component c's own input) */
        for (int h = 0; h < H; ++h) {
          matmul_cols(xq + ((m->split ? c : 0) * H + h) * S * D, S, D, wimg[c], D, h * dk, (h + 1) * dk, tmp);
          quantize(tmp, S * dk, dk, p_low, mode);
          for (int64_t i = 0; i < S; ++i)
            memcpy(low + ((c * S + i) * H + h) * dk, tmp + i * dk, sizeof(float) * (size_t)dk);
        }
      if (target >= 0) /* high_comp + assemble_comp, model.cpp:665-675, 708-713 */
        for (int c = 0; c < 3; ++c) {
          const float* wm = m->master[mat_index(m, MK_WQ + c, l)];
          matmul_cols(xln + ((m->split ? c : 0) * H + target) * S * D, S, D, wm, D, target * dk,
                      (target + 1) * dk, tmp);
          for (int64_t i = 0; i < S; ++i)
            memcpy(low + ((c * S + i) * H + target) * dk, tmp + i * dk, sizeof(float) * (size_t)dk);
        }
      for (int h = 0; h < H; ++h) { /* attend_project, model.cpp:676-702 */
        const float* q = low + (0 * S * H + h) * dk;
        const float* k = low + (1 * S * H + h) * dk;
        const float* v = low + (2 * S * H + h) * dk;
        causal_attention(q, k, v, H * dk, S, dk, z);
        int p_h = (h == target) ? CQO_P32 : p_low;
        quantize(z, S * dk, dk, p_h, mode);
        float* out = outs + node_off(m, first + h);
        matmul_cols(z, S, dk, wo + (int64_t)h * dk * D, D, 0, D, out); /* matmul_rows */
        quantize(out, S * D, D, p_h, mode);
      }
      vi += (int)H;
      continue;
    }
    if (kind == CQO_MLP) { /* model.cpp:720-739 */
      int l = m->layer[vi];
      int p = precision_of(pol, kind, l, -1);
      sum_inputs(m, mask, outs, patch_edge, patch_value, m->node_recv[vi], in);
      layer_norm(in, S, D, m->master[mat_index(m, MK_LN2G, l)], m->master[mat_index(m, MK_LN2B, l)],
                 xln);
      quantize(xln, S * D, D, p, mode);
      matmul_cols(xln, S, D, image(m, mat_index(m, MK_WIN, l), p, mode), 4 * D, 0, 4 * D, hid);
      quantize(hid, S * 4 * D, 4 * D, p, mode);
      gelu(hid, S * 4 * D);
      quantize(hid, S * 4 * D, 4 * D, p, mode);
      float* out = outs + node_off(m, vi);
      matmul_cols(hid, S, 4 * D, image(m, mat_index(m, MK_WOUT, l), p, mode), D, 0, D, out);
      quantize(out, S * D, D, p, mode);
      ++vi;
      continue;
    }
    { /* unembed, model.cpp:741-753 */
      int p = precision_of(pol, kind, -1, -1);
      sum_inputs(m, mask, outs, patch_edge, patch_value, m->node_recv[vi], in);
      layer_norm(in, S, D, m->master[mat_index(m, MK_LNFG, 0)], m->master[mat_index(m, MK_LNFB, 0)],
                 xln);
      quantize(xln, S * D, D, p, mode);
      float* out = outs + node_off(m, vi);
      matmul_cols(xln, S, D, image(m, mat_index(m, MK_WU, 0), p, mode), V, 0, V, out);
      quantize(out, S * V, V, p, mode);
      ++vi;
    }
  }
  free(in), free(xln), free(xq), free(low), free(tmp), free(z), free(hid);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* metrics and scoring — proj/src/patching.cpp                              */
/* ------------------------------------------------------------------------ */

/* metric_kl, patching.cpp:108-141 */
double cqo_metric_kl(const float* c, const float* p, int64_t n) {
  double mc = -INFINITY, mp = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    if (isnan(c[i]) || isnan(p[i])) return NAN;
    if ((double)c[i] > mc) mc = (double)c[i];
    if ((double)p[i] > mp) mp = (double)p[i];
  }
  double sc = 0.0, sp = 0.0;
  for (int64_t i = 0; i < n; ++i) sc += exp((double)c[i] - mc);
  for (int64_t i = 0; i < n; ++i) sp += exp((double)p[i] - mp);
  double lc = mc + log(sc), lp = mp + log(sp);
  double kl = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double lpc = (double)c[i] - lc, lqp = (double)p[i] - lp;
    kl += exp(lpc) * (lpc - lqp);
  }
  return kl;
}

/* patched_divergence, patching.cpp:153-161 */
static int divergence(const cqo_model* m, int metric, const float* clean_logits,
                      const float* patched_logits, int answer, int distractor, double* out) {
  const float* c = clean_logits + (int64_t)(m->S - 1) * m->V;
  const float* p = patched_logits + (int64_t)(m->S - 1) * m->V;
  if (metric == 0) {
    double kl = cqo_metric_kl(c, p, m->V);
    if (isnan(kl)) return fail(2, "metric_kl: NaN logits");
    *out = kl;
    return 0;
  }
  for (int64_t i = 0; i < m->V; ++i)
    if (isnan(c[i]) || isnan(p[i])) return fail(2, "metric_logit_diff: NaN logits");
  double ldp = (double)p[answer] - (double)p[distractor];
  double ldc = (double)c[answer] - (double)c[distractor];
  *out = fabs(ldp - ldc);
  return 0;
}

typedef struct {
  cqo_policy pol;
  float* clean_full;   /* [B][outs] full-graph clean (prepare_policy, patching.cpp:171-185) */
  float* corrupt_full; /* [B][outs] full-graph corrupt */
  float* base_clean;   /* [B][outs] masked clean (refresh_baselines, patching.cpp:191-201) */
  float* base_corrupt; /* [B][outs] masked corrupt */
} policy_cache;

typedef struct {
  const cqo_model* m;
  const int *clean, *corrupt, *answer, *distractor;
  int B, metric;
  policy_cache* pc;
  int n_pc, cap_pc;
} engine;

static void engine_free(engine* en) {
  for (int i = 0; i < en->n_pc; ++i) {
    free(en->pc[i].clean_full), free(en->pc[i].corrupt_full);
    free(en->pc[i].base_clean), free(en->pc[i].base_corrupt);
  }
  free(en->pc);
}

/* prepare_policy + refresh_baselines for one policy (patching.cpp:171-201) */
static int engine_refresh(engine* en, const cqo_policy* pol, const uint8_t* mask, int* slot) {
  const cqo_model* m = en->m;
  int64_t no = outs_size(m), S = m->S;
  int idx = -1;
  for (int i = 0; i < en->n_pc; ++i)
    if (policy_eq(&en->pc[i].pol, pol)) idx = i;
  if (idx < 0) {
    if (en->n_pc == en->cap_pc) {
      en->cap_pc = en->cap_pc ? 2 * en->cap_pc : 8;
      en->pc = realloc(en->pc, sizeof(policy_cache) * (size_t)en->cap_pc);
    }
    idx = en->n_pc++;
    policy_cache* c = &en->pc[idx];
    memset(c, 0, sizeof *c);
    c->pol = *pol;
    c->clean_full = malloc(sizeof(float) * (size_t)(no * en->B));
    c->corrupt_full = malloc(sizeof(float) * (size_t)(no * en->B));
    c->base_clean = malloc(sizeof(float) * (size_t)(no * en->B));
    c->base_corrupt = malloc(sizeof(float) * (size_t)(no * en->B));
    for (int i = 0; i < en->B; ++i) {
      int rc = cqo_forward(m, en->clean + i * S, NULL, pol, -1, NULL, c->clean_full + i * no);
      if (!rc) rc = cqo_forward(m, en->corrupt + i * S, NULL, pol, -1, NULL, c->corrupt_full + i * no);
      if (rc) return rc;
    }
  }
  policy_cache* c = &en->pc[idx];
  for (int i = 0; i < en->B; ++i) {
    int rc = cqo_forward(m, en->clean + i * S, mask, pol, -1, NULL, c->base_clean + i * no);
    if (!rc) rc = cqo_forward(m, en->corrupt + i * S, mask, pol, -1, NULL, c->base_corrupt + i * no);
    if (rc) return rc;
  }
  *slot = idx;
  return 0;
}

/* delta_l (patching.cpp:227-239) and act_diff (patching.cpp:241-259) */
static int engine_score(engine* en, int slot, const uint8_t* mask, int e, int mode, double* out) {
  const cqo_model* m = en->m;
  const policy_cache* c = &en->pc[slot];
  int64_t no = outs_size(m), S = m->S, SD = (int64_t)m->S * m->D;
  float* run = malloc(sizeof(float) * (size_t)no);
  double sum = 0.0;
  int rc = 0;
  int src = m->esrc[e], dst = m->edst[e];
  for (int i = 0; i < en->B && !rc; ++i) {
    if (mode == 0) {
      const float* inject = c->corrupt_full + i * no + node_off(m, src);
      rc = cqo_forward(m, en->clean + i * S, mask, &c->pol, e, inject, run);
      double d = 0.0;
      if (!rc)
        rc = divergence(m, en->metric, c->base_clean + i * no + node_off(m, m->n_nodes - 1),
                        run + node_off(m, m->n_nodes - 1), en->answer[i], en->distractor[i], &d);
      sum += d;
    } else {
      const float* inject = c->clean_full + i * no + node_off(m, src);
      rc = cqo_forward(m, en->corrupt + i * S, mask, &c->pol, e, inject, run);
      const float* a = run + node_off(m, dst);
      const float* b = c->base_corrupt + i * no + node_off(m, dst);
      int64_t n = (m->kind[dst] == CQO_UNEMBED) ? (int64_t)m->S * m->V : SD;
      double acc = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        double dd = (double)a[k] - (double)b[k];
        acc += dd * dd;
      }
      sum += sqrt(acc / (double)n);
    }
  }
  free(run);
  *out = sum / (double)en->B;
  return rc;
}

static int validate_items(const cqo_model* m, const int* clean, const int* corrupt,
                          const int* answer, const int* distractor, int B) {
  /* validate_dataset, patching.cpp:64-81 */
  if (B < 1) return fail(1, "validate_dataset: empty dataset");
  for (int i = 0; i < B; ++i) {
    for (int t = 0; t < m->S; ++t) {
      int a = clean[i * m->S + t], b = corrupt[i * m->S + t];
      if (a < 0 || a >= m->V || b < 0 || b >= m->V)
        return fail(1, "validate_dataset: token out of range");
    }
    if (answer[i] < 0 || answer[i] >= m->V || distractor[i] < 0 || distractor[i] >= m->V)
      return fail(1, "validate_dataset: answer tokens out of range");
    if (answer[i] == distractor[i]) return fail(1, "validate_dataset: answer equals distractor");
  }
  return 0;
}

/* acdc.cpp:42-60 for one iteration's order */
static int score_block(engine* en, const uint8_t* mask, const int* edges, int n,
                       const cqo_policy* base, int per_edge, int mode, double* out) {
  int* slot = malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  cqo_policy* seen = malloc(sizeof(cqo_policy) * (size_t)(n > 0 ? n : 1));
  int* seen_slot = malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int n_seen = 0, rc = 0;
  for (int i = 0; i < n && !rc; ++i) {
    cqo_policy p = per_edge ? policy_for_edge(en->m, edges[i], base) : *base;
    int found = -1;
    for (int s = 0; s < n_seen; ++s)
      if (policy_eq(&seen[s], &p)) found = seen_slot[s];
    if (found < 0) {
      rc = engine_refresh(en, &p, mask, &found);
      seen[n_seen] = p;
      seen_slot[n_seen++] = found;
    }
    slot[i] = found;
  }
  for (int i = 0; i < n && !rc; ++i) rc = engine_score(en, slot[i], mask, edges[i], mode, &out[i]);
  free(slot), free(seen), free(seen_slot);
  return rc;
}

int cqo_score_edges(const cqo_model* m, const int* clean, const int* corrupt, const int* answer,
                    const int* distractor, int B, const uint8_t* mask, const int* edges, int n,
                    const cqo_policy* base, int per_edge, int metric, int mode, double* out) {
  int rc = validate_items(m, clean, corrupt, answer, distractor, B);
  if (rc) return rc;
  for (int i = 0; i < n; ++i)
    if (edges[i] < 0 || edges[i] >= m->n_edges) return fail(1, "score_edges: bad edge id");
  engine en = {m, clean, corrupt, answer, distractor, B, metric, NULL, 0, 0};
  rc = score_block(&en, mask, edges, n, base, per_edge, mode, out);
  engine_free(&en);
  return rc;
}

/* run_acdc, acdc.cpp:23-88 */
int cqo_run_acdc(const cqo_model* m, const int* clean, const int* corrupt, const int* answer,
                 const int* distractor, int B, int metric, const cqo_prune* pc, int* steps,
                 uint8_t* final_mask, double* last_score, int* n_rec, int* rec_step,
                 int* rec_edge, double* rec_score, uint8_t* rec_kept, int rec_cap) {
  /* PruneConfig::validate, acdc.cpp:14-21 */
  if (!(pc->tau >= 0.0)) return fail(1, "PruneConfig: tau must be >= 0");
  if (pc->max_steps < 1) return fail(1, "PruneConfig: max_steps must be >= 1");
  if (!(pc->min_change_rate >= 0.0)) return fail(1, "PruneConfig: min_change_rate must be >= 0");
  if (!(pc->act_floor >= 0.0)) return fail(1, "PruneConfig: act_floor must be >= 0");
  int rc = validate_items(m, clean, corrupt, answer, distractor, B);
  if (rc) return rc;
  int E = m->n_edges;
  uint8_t* mask = malloc((size_t)E);
  memset(mask, 1, (size_t)E);
  for (int e = 0; e < E; ++e) last_score[e] = 0.0;
  int* order = malloc(sizeof(int) * (size_t)E);
  double* raw = malloc(sizeof(double) * (size_t)E);
  engine en = {m, clean, corrupt, answer, distractor, B, metric, NULL, 0, 0};
  int t = 0, k = 0, keep_going = 1;
  do {
    int n = cqo_sweep_order(m, mask, order);
    if (pc->heads_only) {
      int w = 0;
      for (int i = 0; i < n; ++i)
        if (m->kind[m->esrc[order[i]]] == CQO_HEAD) order[w++] = order[i];
      n = w;
    }
    if (n == 0) break;
    rc = score_block(&en, mask, order, n, &pc->base, pc->per_edge_policy, pc->mode, raw);
    if (rc) break;
    int removed = 0;
    for (int i = 0; i < n; ++i) {
      double s = raw[i];
      if (pc->mode == 1 && s < pc->act_floor) s = 0.0;
      int keep = !(s < pc->tau);
      if (k < rec_cap) {
        rec_step[k] = t, rec_edge[k] = order[i], rec_score[k] = s, rec_kept[k] = (uint8_t)keep;
      }
      ++k;
      last_score[order[i]] = s;
      if (!keep) {
        mask[order[i]] = 0;
        ++removed;
      }
    }
    ++t;
    double change_rate = (double)removed / (double)n;
    keep_going = removed > 0 && change_rate > pc->min_change_rate;
    int present = 0;
    for (int e = 0; e < E; ++e) present += mask[e];
    if (!(t < pc->max_steps && present > 0 && keep_going)) break;
  } while (1);
  memcpy(final_mask, mask, (size_t)E);
  *steps = t;
  *n_rec = k;
  engine_free(&en);
  free(mask), free(order), free(raw);
  return rc;
}

/* Host glibc values over a range of float bit patterns (the libm the
 * reference calls): which 0 expf, 1 erff, 2 the reference gelu
 * (kernels.cpp:226). Used to check the device restatements exhaustively. */
void cqo_libm_range(int which, uint32_t lo, uint64_t count, float* out) {
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t u = lo + (uint32_t)i;
    float x;
    memcpy(&x, &u, 4);
    if (which == 0) out[i] = expf(x);
    else if (which == 1) out[i] = erff(x);
    else out[i] = 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
  }
}

/* encode_f8 / encode_bf16 over a range of float bit patterns. */
void cqo_codes_range(uint32_t lo, uint64_t count, uint8_t* f8, uint16_t* bf16) {
  for (uint64_t i = 0; i < count; ++i) {
    uint32_t u = lo + (uint32_t)i;
    float x;
    memcpy(&x, &u, 4);
    if (f8) f8[i] = cqo_encode_f8((double)x);
    if (bf16) bf16[i] = cqo_encode_bf16(x);
  }
}
