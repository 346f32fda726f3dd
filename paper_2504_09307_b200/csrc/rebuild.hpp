// rebuild.hpp — the structural what-if rebuild (estimate()'s host step).
//
// Restates, over a HostGraph that kept its Task.meta (ingest / synth with
// keep_meta), the reference's
//   tag_tasks         transform.cpp:71-162   (layer / microbatch / phase tags)
//   measure_pipeline  transform.cpp:378-502  (per-layer kernels, host costs,
//                                             p2p and gradient sizes)
//   rebuild_pipeline  transform.cpp:556-701  (the target PipelineSpec)
// The result is the PipelineSpec rebuild_pipeline hands to build_pipeline;
// the B200 engine replays it through ts_pipeline_graph / estimate_batch
// (the estimate graph) — build_pipeline + graph_from_events is the replay
// graph of the same spec (ts_pipeline_graph with estimate = 0).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ingest.hpp"
#include "lumos_b200.h"

namespace lumos {

// TagPolicy (transform.hpp:14-24)
struct TagPolicyLite {
  std::vector<std::string> layer_keys = {"layer", "layer_id"};
  std::vector<std::string> microbatch_keys = {"mb", "microbatch", "micro_batch"};
  std::vector<std::string> phase_keys = {"phase"};
  bool infer_from_names = true;
  bool fill_between = true;
};
// TagPolicy::from_json (transform.cpp:58-69); false + err on a bad document
bool tag_policy_from_json(const std::string& text, TagPolicyLite& out, std::string& err);

struct KernelStr {  // KernelSpec (pipeline.hpp:27-32)
  std::string name;
  int64_t duration = 0;
  int32_t op_class = TS_OP_COMPUTE;
  MetaList args;  // key order
};
struct StageStr {  // StageSpec (pipeline.hpp:34-43)
  std::vector<std::vector<KernelStr>> layers_fwd, layers_bwd;
  std::vector<KernelStr> pre_fwd, post_fwd, pre_bwd, post_bwd, reduce, optimizer;
};
struct PipelineStr {  // PipelineSpec (pipeline.hpp:52-70); unset fields keep its defaults
  int32_t pp = 1, dp = 1, num_microbatches = 1;
  std::vector<StageStr> stages;
  int64_t launch = 5, record = 2, wait = 2, sync = 5;
  int64_t p2p_send = 0, p2p_recv_base = 0, activation_bytes = 0, origin = 0;
};

// WhatIfConfig (transform.hpp:28-41) with an AnalyticalCostModel
struct WhatIfLite {
  ts_model_config source_model{}, target_model{};
  ts_par_config source_par{}, target_par{};
  double alpha_us = 10.0, bytes_per_us = 50000.0;
  int64_t activation_bytes = 0;
  TagPolicyLite policy;
};

// rebuild_pipeline (transform.cpp:556-701).  `unchanged` is set (and `out`
// left empty) when the target differs in nothing the rebuild cares about —
// the reference then returns the source graph.  Returns TS_OK or
// TS_E_INVALID_ARGUMENT with the TransformError text in err.
int rebuild_pipeline(const HostGraph& g, const Names& names, const WhatIfLite& w,
                     PipelineStr& out, bool& unchanged, std::string& err);

}  // namespace lumos
