// synth.hpp — synthetic GPT-like trace generator (see synth.cpp).
#pragma once

#include <cstdint>
#include <string>

#include "ingest.hpp"
#include "lumos_b200.h"

namespace lumos {

struct SynthOutput {
  Names names;
  HostGraph graph;
  int64_t truth_makespan = 0;  // generator ground truth (GroundTruth, synth.hpp:52-57)
  int64_t n_ops = 0;           // cost indices handed out (DurationHook op_index range)
};

void synth_defaults(ts_synth_spec* s);
int synth_graph(const ts_synth_spec& spec, SynthOutput& out, std::string& err);
// A user PipelineSpec (ts_pipeline_spec): its build_pipeline trace as the
// replay graph or the estimate graph (estimate = true), with tp replicas.
void pipeline_defaults(ts_pipeline_spec* c);
int pipeline_graph(const ts_pipeline_spec& c, bool estimate, int tp, SynthOutput& out,
                   std::string& err);

}  // namespace lumos
