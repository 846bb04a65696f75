// acdc_gpu.hpp — the reference-side integration of libcqg.so: what a
// maintainer of circuitquant (/root/reference/proj) adds to run PAHQ-ACDC's
// scoring block on a B200. Compiled against the reference's own headers
// (proj/include) and linked with its objects plus -lcqg (integration/Makefile).
#pragma once

#include <vector>

#include "circuitquant/acdc.hpp"
#include "circuitquant/model.hpp"
#include "circuitquant/patching.hpp"
#include "cqg.h"

namespace cq {

// Return code of a cqg_* call -> the reference's exception classes
// (include/cqg.h: 1 invalid_argument, 2 runtime_error, 3 bad_alloc).
void cqg_check(int rc);

// PrecisionPolicy (precision_policy.hpp) -> cqg_policy.
cqg_policy to_cqg(const PrecisionPolicy& p);

// One device context: the FP32 masters in for_each_matrix order
// (model.cpp:285-317) and the dataset (validate_dataset, patching.cpp:64-81).
cqg_ctx* make_cqg(const WeightSet& w, const Dataset& ds, Metric metric, int device);

// run_acdc (acdc.cpp:23-88) with its scoring block (acdc.cpp:42-60: per-edge
// policies, refresh_baselines per policy, the OpenMP delta_l loop) replaced by
// one cqg_score_edges call per iteration; thresholding, remove_edge and the
// stop rule are the reference's.
CircuitResult run_acdc_gpu(ComputationalGraph& g, cqg_ctx* ctx, const PruneConfig& cfg);

}  // namespace cq
