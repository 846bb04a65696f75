// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle).
//
// A thin extern "C" facade over the *unmodified* reference library
// (`circuitquant`, compiled from /root/reference/proj/src/*.cpp by
// oracle/Makefile into oracle/_ref/libcqref.so). It exists so that the
// parity tests, the golden-fixture generator and bench.py's CPU arm can
// call the reference's own code path through ctypes. Nothing in the
// product (paper_2510_23264_b200/) links or loads this file.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument,
// 2 for any other std::exception (message in cqref_last_error()).

#include <omp.h>

#include <cstdint>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "circuitquant/acdc.hpp"
#include "circuitquant/eval.hpp"
#include "circuitquant/model.hpp"
#include "circuitquant/numerics.hpp"
#include "circuitquant/pahq.hpp"
#include "circuitquant/patching.hpp"
#include "support.hpp"  // proj/tests/support.hpp: portable mt19937 generators

using namespace cq;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

ModelConfig cfg_from(const uint32_t* c) {
  ModelConfig cfg;
  cfg.n_layers = c[0];
  cfg.n_heads = c[1];
  cfg.d_model = c[2];
  cfg.d_k = c[3];
  cfg.vocab = c[4];
  cfg.seq_len = c[5];
  cfg.batch = c[6];
  cfg.has_mlp = c[7];
  return cfg;
}

}  // namespace

extern "C" {

// Policy descriptor shared with include/cqg.h (same field meaning).
struct cqref_policy {
  int8_t attention_default;  // Precision: 0=P8 1=P16 2=P32
  int8_t mlp_default;
  int8_t embed_precision;
  int8_t unembed_precision;
  int8_t low_mode;  // 0=E4m3 1=Rtn4
  int32_t target_head_layer;  // -1: none
  int32_t target_head_head;
  int32_t target_mlp;  // -1: none
};

struct cqref_prune {
  double tau;
  int32_t max_steps;
  double min_change_rate;
  int32_t mode;  // 0 LossDelta, 1 ActDiff
  double act_floor;
  int32_t per_edge_policy;
  int32_t heads_only;
  cqref_policy base;
};

}  // extern "C"

namespace {

PrecisionPolicy policy_from(const cqref_policy& p) {
  PrecisionPolicy pol;
  pol.attention_default = static_cast<Precision>(p.attention_default);
  pol.mlp_default = static_cast<Precision>(p.mlp_default);
  pol.embed_precision = static_cast<Precision>(p.embed_precision);
  pol.unembed_precision = static_cast<Precision>(p.unembed_precision);
  pol.low_mode = static_cast<LowMode>(p.low_mode);
  if (p.target_head_layer >= 0) pol.target_head = HeadRef{p.target_head_layer, p.target_head_head};
  if (p.target_mlp >= 0) pol.target_mlp = p.target_mlp;
  return pol;
}

struct Handle {
  WeightSet w;
  Dataset ds;
  std::unique_ptr<ComputationalGraph> g;
  std::unique_ptr<ImageBank> bank;
  std::unique_ptr<DeltaLEngine> eng;
  Metric metric;

  void set_mask(const uint8_t* mask) {
    if (!mask) {
      g->reset_mask();
      return;
    }
    for (size_t e = 0; e < g->all_edges().size(); ++e) {
      if (mask[e]) g->restore_edge(static_cast<int>(e));
      else g->remove_edge(static_cast<int>(e));
    }
  }
};

std::unique_ptr<ImageBank> full_bank(const WeightSet& w) {
  std::vector<std::pair<Precision, LowMode>> needs = {
      {Precision::P8, LowMode::E4m3}, {Precision::P16, LowMode::E4m3},
      {Precision::P32, LowMode::E4m3}};
  // The 4-bit grid image is only needed by Rtn4 policies; skipping it keeps
  // the CPU-baseline setup at GPT-2 scale short (CQREF_NO_RTN4=1).
  const char* no4 = std::getenv("CQREF_NO_RTN4");
  if (!(no4 && *no4 == '1')) needs.push_back({Precision::P8, LowMode::Rtn4});
  return std::make_unique<ImageBank>(w, needs);
}

}  // namespace

extern "C" {

const char* cqref_last_error(void) { return g_err.c_str(); }

void cqref_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}

int cqref_max_threads(void) { return omp_get_max_threads(); }

// --- numerics (proj/src/numerics.cpp) --------------------------------------
uint8_t cqref_encode_f8(double x) { return encode_f8(x).bits; }
double cqref_decode_f8(uint8_t b) { return decode_f8(F8E4M3{b}); }
uint16_t cqref_encode_bf16(float x) { return encode_bf16(x).bits; }
float cqref_decode_bf16(uint16_t b) { return decode_bf16(BF16{b}); }
float cqref_round_f8(float x) { return round_f8(x); }
float cqref_round_bf16(float x) { return round_bf16(x); }

// Round many floats at once (fast exhaustive checks): mode 0 -> e4m3 bits
// into out8, mode 1 -> bf16 bits into out16.
void cqref_encode_f8_many(const float* x, int64_t n, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = encode_f8(static_cast<double>(x[i])).bits;
}
void cqref_encode_f8_range(uint32_t lo, uint64_t count, uint8_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(count); ++i) {
    uint32_t u = lo + static_cast<uint32_t>(i);
    float f;
    std::memcpy(&f, &u, 4);
    out[i] = encode_f8(static_cast<double>(f)).bits;
  }
}
void cqref_encode_bf16_range(uint32_t lo, uint64_t count, uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(count); ++i) {
    uint32_t u = lo + static_cast<uint32_t>(i);
    float f;
    std::memcpy(&f, &u, 4);
    out[i] = encode_bf16(f).bits;
  }
}

int cqref_quantize_rtn_f32(float* x, int64_t n, int bits, double* delta) {
  return guarded([&] {
    QuantParams p = quantize_rtn(std::span<float>(x, static_cast<size_t>(n)), bits);
    if (delta) *delta = p.delta;
  });
}
int cqref_quantize_rtn_f64(double* x, int64_t n, int bits, double* delta) {
  return guarded([&] {
    QuantParams p = quantize_rtn(std::span<double>(x, static_cast<size_t>(n)), bits);
    if (delta) *delta = p.delta;
  });
}

double cqref_metric_kl(const float* c, const float* p, int64_t n) {
  double r = 0.0;
  int rc = guarded([&] {
    r = metric_kl(std::span<const float>(c, static_cast<size_t>(n)),
                  std::span<const float>(p, static_cast<size_t>(n)));
  });
  return rc == 0 ? r : -1.0;
}

void cqref_threshold_grid(double lo, double hi, int n, double* out) {
  std::vector<double> g = threshold_grid(lo, hi, n);
  for (int i = 0; i < n; ++i) out[i] = g[static_cast<size_t>(i)];
}

// --- generators (proj/tests/support.hpp) -----------------------------------
int cqref_gen_random(const uint32_t* cfg8, uint32_t wseed, float wscale, int items,
                     uint32_t dseed, const char* wpath, const char* dpath) {
  return guarded([&] {
    ModelConfig cfg = cfg_from(cfg8);
    cfg.validate();
    if (wpath && *wpath) save_weights(cqtest::random_weights(cfg, wseed, wscale), wpath);
    if (dpath && *dpath) save_dataset_jsonl(cqtest::random_dataset(cfg, items, dseed), dpath);
  });
}

int cqref_gen_planted(int preset, uint32_t seed, int items, double signal_scale,
                      const char* dir) {
  return guarded([&] {
    PlantedSpec spec;
    spec.preset = static_cast<TaskPreset>(preset);
    spec.seed = seed;
    spec.items = items;
    spec.signal_scale = signal_scale;
    save_task(generate_planted(spec), dir);
  });
}

int cqref_roc_sweep(const char* dir, int method, int bits, int metric, const double* taus,
                    int n, double* tpr, double* fpr, int* kept, double* auc) {
  return guarded([&] {
    PlantedTask t = load_task(dir);
    std::vector<double> tv(taus, taus + n);
    RocCurve c = roc_sweep(t, static_cast<Method>(method), tv, static_cast<Metric>(metric), bits);
    for (int i = 0; i < n; ++i) {
      tpr[i] = c.points[static_cast<size_t>(i)].tpr;
      fpr[i] = c.points[static_cast<size_t>(i)].fpr;
      kept[i] = c.points[static_cast<size_t>(i)].kept_edges;
    }
    *auc = c.auc;
  });
}

// faithfulness / task_accuracy (eval.cpp:1240-1254) of a saved planted task
// under an edge mask (FP32 circuit runs; absent edges read the corrupt run).
int cqref_faithfulness(const char* dir, const uint8_t* mask, int n, double* faith, double* acc) {
  return guarded([&] {
    PlantedTask t = load_task(dir);
    std::vector<bool> m(mask, mask + n);
    *faith = faithfulness(t, m);
    *acc = task_accuracy(t, m);
  });
}

int cqref_method_config(int method, int bits, cqref_prune* out) {
  return guarded([&] {
    PruneConfig pc = method_prune_config(static_cast<Method>(method), bits);
    out->tau = pc.tau;
    out->max_steps = pc.max_steps;
    out->min_change_rate = pc.min_change_rate;
    out->mode = pc.mode == ScoreMode::LossDelta ? 0 : 1;
    out->act_floor = pc.act_floor;
    out->per_edge_policy = pc.per_edge_policy ? 1 : 0;
    out->heads_only = pc.heads_only ? 1 : 0;
    const PrecisionPolicy& b = pc.base_policy;
    out->base = {static_cast<int8_t>(b.attention_default), static_cast<int8_t>(b.mlp_default),
                 static_cast<int8_t>(b.embed_precision), static_cast<int8_t>(b.unembed_precision),
                 static_cast<int8_t>(b.low_mode), -1, -1, -1};
  });
}

// --- graph (proj/src/model.cpp:166-246) ------------------------------------
int cqref_graph(const uint32_t* cfg8, int* n_nodes, int* n_edges, int* node_kind,
                int* node_layer, int* node_head, int* edge_src, int* edge_dst) {
  return guarded([&] {
    ComputationalGraph g(cfg_from(cfg8));
    *n_nodes = static_cast<int>(g.nodes().size());
    *n_edges = static_cast<int>(g.all_edges().size());
    if (node_kind) {
      for (size_t i = 0; i < g.nodes().size(); ++i) {
        node_kind[i] = static_cast<int>(g.nodes()[i].kind);
        node_layer[i] = g.nodes()[i].layer;
        node_head[i] = g.nodes()[i].head;
      }
    }
    if (edge_src) {
      for (const Edge& e : g.all_edges()) {
        edge_src[e.index] = e.src;
        edge_dst[e.index] = e.dst;
      }
    }
  });
}

int cqref_sweep_order(const uint32_t* cfg8, const uint8_t* mask, int* out, int* n_out) {
  return guarded([&] {
    ComputationalGraph g(cfg_from(cfg8));
    for (size_t e = 0; e < g.all_edges().size(); ++e)
      if (mask && !mask[e]) g.remove_edge(static_cast<int>(e));
    std::vector<Edge> order = g.sweep_order();
    for (size_t i = 0; i < order.size(); ++i) out[i] = order[i].index;
    *n_out = static_cast<int>(order.size());
  });
}

// --- model handle -----------------------------------------------------------
int cqref_open(const char* wpath, const char* dpath, int metric, void** out) {
  return guarded([&] {
    auto h = std::make_unique<Handle>();
    h->w = load_weights(wpath);
    h->ds = load_dataset_jsonl(dpath);
    h->metric = static_cast<Metric>(metric);
    h->g = std::make_unique<ComputationalGraph>(h->w.cfg);
    h->bank = full_bank(h->w);
    h->eng = std::make_unique<DeltaLEngine>(*h->g, *h->bank, h->ds, h->metric);
    *out = h.release();
  });
}

void cqref_close(void* h) { delete static_cast<Handle*>(h); }

int cqref_config(void* hv, uint32_t* cfg8, int* items) {
  return guarded([&] {
    Handle* h = static_cast<Handle*>(hv);
    const ModelConfig& c = h->w.cfg;
    uint32_t v[8] = {c.n_layers, c.n_heads, c.d_model, c.d_k, c.vocab, c.seq_len, c.batch, c.has_mlp};
    std::memcpy(cfg8, v, sizeof v);
    *items = static_cast<int>(h->ds.size());
  });
}

// Canonical matrices (for_each_matrix order, model.cpp:285-308): count,
// sizes, and master copies.
int cqref_matrices(void* hv, int* count, int64_t* sizes, float** ptrs) {
  return guarded([&] {
    Handle* h = static_cast<Handle*>(hv);
    int i = 0;
    for_each_matrix(static_cast<const WeightSet&>(h->w), [&](const std::string&, const Tensor& t) {
      if (sizes) sizes[i] = t.size();
      if (ptrs) ptrs[i] = const_cast<float*>(t.data());
      ++i;
    });
    *count = i;
  });
}

// ImageBank::get(name, p, mode) copied into out (model.cpp:505-519).
int cqref_image(void* hv, int matrix_index, int precision, int low_mode, float* out) {
  return guarded([&] {
    Handle* h = static_cast<Handle*>(hv);
    std::string name;
    int i = 0;
    for_each_matrix(static_cast<const WeightSet&>(h->w), [&](const std::string& n, const Tensor&) {
      if (i++ == matrix_index) name = n;
    });
    if (name.empty()) throw std::invalid_argument("cqref_image: bad matrix index");
    const Tensor& t = h->bank->get(name, static_cast<Precision>(precision),
                                   static_cast<LowMode>(low_mode));
    std::memcpy(out, t.data(), sizeof(float) * static_cast<size_t>(t.size()));
  });
}

// forward() (model.cpp:556-757) with an optional single patch; writes every
// node's out into outs (nodes in graph order; S*D floats each, unembed S*V).
int cqref_forward(void* hv, const int* tokens, const uint8_t* mask, const cqref_policy* pol,
                  int patch_edge, const float* patch_value, float* outs, float* node_ins) {
  return guarded([&] {
    Handle* h = static_cast<Handle*>(hv);
    h->set_mask(mask);
    const ModelConfig& c = h->w.cfg;
    std::vector<int> tok(tokens, tokens + c.seq_len);
    Tensor pv;
    std::vector<EdgePatch> patches;
    if (patch_edge >= 0) {
      pv = Tensor(c.seq_len, c.d_model);
      std::memcpy(pv.data(), patch_value, sizeof(float) * static_cast<size_t>(pv.size()));
      patches.push_back({patch_edge, &pv});
    }
    ActivationCache cache = forward(*h->g, *h->bank, tok, policy_from(*pol), patches);
    size_t off = 0, off_in = 0;
    for (const NodeActivations& n : cache.nodes) {
      std::memcpy(outs + off, n.out.data(), sizeof(float) * static_cast<size_t>(n.out.size()));
      off += static_cast<size_t>(n.out.size());
      if (node_ins) {
        size_t sd = static_cast<size_t>(c.seq_len) * c.d_model;
        if (!n.in.empty()) std::memcpy(node_ins + off_in, n.in.data(), sizeof(float) * sd);
        else std::memset(node_ins + off_in, 0, sizeof(float) * sd);
        off_in += sd;
      }
    }
  });
}

// DeltaLEngine::score for a list of edges under the given mask — exactly the
// block run_acdc executes per iteration (acdc.cpp:42-60): per-edge policies,
// one sequential refresh_baselines per unique policy, OpenMP fan-out over
// edges. This is the reference arm that the GPU C-ABI replaces.
int cqref_score_edges(void* hv, const uint8_t* mask, const int* edge_ids, int n,
                      const cqref_policy* base, int per_edge_policy, int mode, double* out) {
  return guarded([&] {
    Handle* h = static_cast<Handle*>(hv);
    h->set_mask(mask);
    PrecisionPolicy bp = policy_from(*base);
    std::vector<Edge> order;
    for (int i = 0; i < n; ++i) order.push_back(h->g->all_edges().at(static_cast<size_t>(edge_ids[i])));
    std::vector<PrecisionPolicy> policies(order.size());
    std::map<std::string, size_t> seen;
    for (size_t i = 0; i < order.size(); ++i) {
      policies[i] = per_edge_policy ? policy_for_edge(order[i], *h->g, bp) : bp;
      if (!seen.count(policies[i].key())) {
        h->eng->refresh_baselines(policies[i]);
        seen.emplace(policies[i].key(), i);
      }
    }
    ScoreMode sm = mode == 0 ? ScoreMode::LossDelta : ScoreMode::ActDiff;
    std::vector<std::string> errs(order.size());
#pragma omp parallel for schedule(dynamic)
    for (int64_t i = 0; i < static_cast<int64_t>(order.size()); ++i) {
      try {
        out[i] = h->eng->score(order[static_cast<size_t>(i)], policies[static_cast<size_t>(i)], sm);
      } catch (const std::exception& e) {
        errs[static_cast<size_t>(i)] = e.what();
      }
    }
    for (const std::string& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// CPU baseline timing: refresh_baselines for the edges'
// policies (untimed, reported in *ms_refresh), then DeltaLEngine::delta_l
// over the edges in an OpenMP parallel-for exactly as acdc.cpp:55-60 (timed,
// *ms_score). Full mask.
int cqref_time_delta_l(void* hv, const int* edge_ids, int n, const cqref_policy* base,
                       int per_edge_policy, double* out, double* ms_refresh, double* ms_score) {
  return guarded([&] {
    Handle* h = static_cast<Handle*>(hv);
    h->g->reset_mask();
    PrecisionPolicy bp = policy_from(*base);
    std::vector<Edge> order;
    for (int i = 0; i < n; ++i) order.push_back(h->g->all_edges().at(static_cast<size_t>(edge_ids[i])));
    std::vector<PrecisionPolicy> policies(order.size());
    std::map<std::string, size_t> seen;
    auto t0 = std::chrono::steady_clock::now();
    for (size_t i = 0; i < order.size(); ++i) {
      policies[i] = per_edge_policy ? policy_for_edge(order[i], *h->g, bp) : bp;
      if (!seen.count(policies[i].key())) {
        h->eng->refresh_baselines(policies[i]);
        seen.emplace(policies[i].key(), i);
      }
    }
    auto t1 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic)
    for (int64_t i = 0; i < static_cast<int64_t>(order.size()); ++i)
      out[i] = h->eng->delta_l(order[static_cast<size_t>(i)], policies[static_cast<size_t>(i)]);
    auto t2 = std::chrono::steady_clock::now();
    *ms_refresh = std::chrono::duration<double, std::milli>(t1 - t0).count();
    *ms_score = std::chrono::duration<double, std::milli>(t2 - t1).count();
  });
}

// run_acdc (acdc.cpp:23-88) on a fresh full mask. Records are written flat in
// iteration order: rec_step, rec_edge, rec_score, rec_kept (capacity rec_cap).
int cqref_run_acdc(void* hv, const cqref_prune* pc, int* steps, uint8_t* final_mask,
                   double* last_score, int* n_rec, int* rec_step, int* rec_edge,
                   double* rec_score, uint8_t* rec_kept, int rec_cap) {
  return guarded([&] {
    Handle* h = static_cast<Handle*>(hv);
    h->g->reset_mask();
    // Fresh engine: caches are keyed by policy and survive across calls
    // otherwise, which is harmless but keeps runs independent.
    h->eng = std::make_unique<DeltaLEngine>(*h->g, *h->bank, h->ds, h->metric);
    PruneConfig cfg;
    cfg.tau = pc->tau;
    cfg.max_steps = pc->max_steps;
    cfg.min_change_rate = pc->min_change_rate;
    cfg.mode = pc->mode == 0 ? ScoreMode::LossDelta : ScoreMode::ActDiff;
    cfg.act_floor = pc->act_floor;
    cfg.per_edge_policy = pc->per_edge_policy != 0;
    cfg.heads_only = pc->heads_only != 0;
    cfg.base_policy = policy_from(pc->base);
    CircuitResult r = run_acdc(*h->g, *h->eng, cfg);
    *steps = r.steps;
    for (size_t e = 0; e < r.final_mask.size(); ++e) final_mask[e] = r.final_mask[e] ? 1 : 0;
    for (size_t e = 0; e < r.last_score.size(); ++e) last_score[e] = r.last_score[e];
    int k = 0;
    for (const IterationRecord& rec : r.iterations) {
      for (const EdgeScore& es : rec.scores) {
        if (k < rec_cap) {
          rec_step[k] = rec.step;
          rec_edge[k] = es.edge;
          rec_score[k] = es.score;
          rec_kept[k] = es.kept ? 1 : 0;
        }
        ++k;
      }
    }
    *n_rec = k;
    h->g->reset_mask();
  });
}

}  // extern "C"
