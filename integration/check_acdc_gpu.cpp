// check_acdc_gpu — the drop-in proof on the reference side: the reference's
// stock run_acdc (acdc.cpp:23-88, its OpenMP delta_l loop on the host) and
// run_acdc_gpu (acdc_gpu.cpp: the same loop, scoring block on libcqg.so) on
// the same weights.bin / dataset.jsonl (the reference's formats), then a JSON
// line comparing the two CircuitResults.
//
//   check_acdc_gpu weights.bin dataset.jsonl [tau] [--stock-only]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "acdc_gpu.hpp"
#include "circuitquant/eval.hpp"

using namespace cq;

static double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s weights.bin dataset.jsonl [tau] [--stock-only]\n", argv[0]);
    return 2;
  }
  const bool stock_only = argc > 4 && std::strcmp(argv[4], "--stock-only") == 0;
  try {
    const WeightSet w = load_weights(argv[1]);
    const Dataset ds = load_dataset_jsonl(argv[2]);
    PruneConfig cfg = method_prune_config(Method::Pahq, 8);
    if (argc > 3) cfg.tau = std::stod(argv[3]);

    ComputationalGraph g_ref(w.cfg);
    ImageBank bank(w, {{Precision::P8, LowMode::E4m3}, {Precision::P16, LowMode::E4m3},
                       {Precision::P32, LowMode::E4m3}});
    DeltaLEngine engine(g_ref, bank, ds, Metric::KlDivergence);
    auto t0 = std::chrono::steady_clock::now();
    const CircuitResult want = run_acdc(g_ref, engine, cfg);
    const double s_ref = seconds_since(t0);
    if (stock_only) {
      std::printf("{\"stock_steps\": %d, \"stock_seconds\": %.6f}\n", want.steps, s_ref);
      return 0;
    }

    ComputationalGraph g_gpu(w.cfg);
    cqg_ctx* ctx = make_cqg(w, ds, Metric::KlDivergence, 0);
    t0 = std::chrono::steady_clock::now();
    const CircuitResult got = run_acdc_gpu(g_gpu, ctx, cfg);
    const double s_gpu = seconds_since(t0);
    cqg_destroy(ctx);

    bool same_kept = want.iterations.size() == got.iterations.size();
    size_t n_rec = 0;
    double max_rel = 0.0;
    for (size_t i = 0; same_kept && i < want.iterations.size(); ++i) {
      const auto& a = want.iterations[i].scores;
      const auto& b = got.iterations[i].scores;
      same_kept = same_kept && a.size() == b.size() &&
                  want.iterations[i].present_after == got.iterations[i].present_after;
      for (size_t k = 0; same_kept && k < a.size(); ++k) {
        same_kept = a[k].edge == b[k].edge && a[k].kept == b[k].kept;
        const double d = std::fabs(a[k].score - b[k].score);
        const double r = a[k].score != 0.0 ? d / std::fabs(a[k].score) : (d == 0.0 ? 0.0 : INFINITY);
        if (r > max_rel) max_rel = r;
        ++n_rec;
      }
    }
    std::printf(
        "{\"same_final_mask\": %s, \"same_steps\": %s, \"same_records\": %s, \"records\": %zu, "
        "\"max_rel_score_diff\": %.3e, \"steps\": %d, \"kept_edges\": %d, \"stock_seconds\": %.6f, "
        "\"gpu_seconds\": %.6f}\n",
        want.final_mask == got.final_mask ? "true" : "false", want.steps == got.steps ? "true" : "false",
        same_kept ? "true" : "false", n_rec, max_rel, got.steps, g_gpu.present_count(), s_ref, s_gpu);
    return want.final_mask == got.final_mask && same_kept ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 3;
  }
}
