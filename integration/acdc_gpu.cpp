// acdc_gpu.cpp — see acdc_gpu.hpp.
#include "acdc_gpu.hpp"

#include <new>
#include <stdexcept>
#include <string>

namespace cq {

void cqg_check(int rc) {
  switch (rc) {
    case 0: return;
    case 1: throw std::invalid_argument(cqg_last_error());
    case 3: throw std::bad_alloc();
    default: throw std::runtime_error(cqg_last_error());
  }
}

cqg_policy to_cqg(const PrecisionPolicy& p) {
  cqg_policy c{};
  c.attention_default = static_cast<int8_t>(p.attention_default);
  c.mlp_default = static_cast<int8_t>(p.mlp_default);
  c.embed_precision = static_cast<int8_t>(p.embed_precision);
  c.unembed_precision = static_cast<int8_t>(p.unembed_precision);
  c.low_mode = static_cast<int8_t>(p.low_mode);
  c.target_head_layer = p.target_head ? p.target_head->layer : -1;
  c.target_head_head = p.target_head ? p.target_head->head : -1;
  c.target_mlp = p.target_mlp ? *p.target_mlp : -1;
  return c;
}

cqg_ctx* make_cqg(const WeightSet& w, const Dataset& ds, Metric metric, int device) {
  std::vector<const float*> mats;
  for_each_matrix(w, [&](const std::string&, const Tensor& t) { mats.push_back(t.data()); });
  const ModelConfig& m = w.cfg;
  const cqg_config c{static_cast<uint32_t>(m.n_layers), static_cast<uint32_t>(m.n_heads),
                     static_cast<uint32_t>(m.d_model),  static_cast<uint32_t>(m.d_k),
                     static_cast<uint32_t>(m.vocab),    static_cast<uint32_t>(m.seq_len),
                     static_cast<uint32_t>(m.has_mlp ? 1 : 0), /*qkv_split=*/0u};  // the reference's graph
  cqg_ctx* ctx = nullptr;
  cqg_check(cqg_create(&c, mats.data(), device, &ctx));
  std::vector<int32_t> clean, corrupt, answer, distractor;
  for (const ContrastPair& it : ds) {
    clean.insert(clean.end(), it.clean.begin(), it.clean.end());
    corrupt.insert(corrupt.end(), it.corrupt.begin(), it.corrupt.end());
    answer.push_back(it.answer);
    distractor.push_back(it.distractor);
  }
  const int n = static_cast<int>(ds.size());
  const int rc = cqg_set_dataset(ctx, clean.data(), corrupt.data(), answer.data(), distractor.data(), n,
                                 0, n, static_cast<int>(metric));
  if (rc != 0) {
    cqg_destroy(ctx);
    cqg_check(rc);
  }
  return ctx;
}

CircuitResult run_acdc_gpu(ComputationalGraph& g, cqg_ctx* ctx, const PruneConfig& cfg) {
  cfg.validate();
  const cqg_policy base = to_cqg(cfg.base_policy);
  CircuitResult res;
  res.last_score.assign(g.all_edges().size(), 0.0);
  int step = 0;
  for (;;) {
    std::vector<Edge> order = g.sweep_order();
    if (cfg.heads_only)
      std::erase_if(order, [&](const Edge& e) {
        return g.nodes()[static_cast<size_t>(e.src)].kind != NodeKind::Head;
      });
    if (order.empty()) break;
    // ---- the scoring block, on the GPU (every score against this
    // iteration's starting mask, as the reference's parallel loop) ----
    std::vector<int32_t> ids;
    ids.reserve(order.size());
    for (const Edge& e : order) ids.push_back(e.index);
    std::vector<uint8_t> mask(g.mask().size());
    for (size_t e = 0; e < mask.size(); ++e) mask[e] = g.mask()[e] ? 1 : 0;
    std::vector<double> raw(order.size());
    cqg_check(cqg_score_edges(ctx, mask.data(), ids.data(), static_cast<int>(ids.size()), &base,
                              cfg.per_edge_policy ? 1 : 0, static_cast<int>(cfg.mode), raw.data()));
    // ---- the reference's thresholding and stop rule ----
    IterationRecord rec;
    rec.step = step;
    rec.present_before = g.present_count();
    int removed = 0;
    for (size_t i = 0; i < order.size(); ++i) {
      double s = raw[i];
      if (cfg.mode == ScoreMode::ActDiff && s < cfg.act_floor) s = 0.0;
      const bool keep = !(s < cfg.tau);
      rec.scores.push_back({order[i].index, s, keep});
      res.last_score[static_cast<size_t>(order[i].index)] = s;
      if (!keep) {
        g.remove_edge(order[i].index);
        ++removed;
      }
    }
    rec.present_after = g.present_count();
    res.iterations.push_back(std::move(rec));
    ++step;
    const bool changed = removed > 0 &&
                         static_cast<double>(removed) / static_cast<double>(order.size()) > cfg.min_change_rate;
    if (!(step < cfg.max_steps && g.present_count() > 0 && changed)) break;
  }
  res.final_mask = g.mask();
  res.steps = step;
  return res;
}

}  // namespace cq
