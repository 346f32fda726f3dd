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

}  // namespace lumos
