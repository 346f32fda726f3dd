// compile.hpp — ExecutionGraph (C-ABI SoA view) -> device programs.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "lumos_b200.h"
#include "program.hpp"

namespace lumos {

struct CompiledGraph {
  int32_t n_tasks = 0;
  int64_t window_start = 0;
  int64_t window_end = 0;
  std::vector<Op> ops;  // Op and OpExt records (both 32 bytes)
  std::vector<ProgramDesc> programs;
  std::vector<ComponentDesc> comps;
  int32_t max_slots = 0;
  int32_t n_syncs = 0;
  int32_t n_gpu_tasks = 0;

  // per-task arrays used by the duration kernel and the reductions
  std::vector<int64_t> base;
  std::vector<uint8_t> scale_class;
  std::vector<uint8_t> is_comm;

  // reductions: ranks (sorted, = ranks_in(graph), build.cpp:582-590), their
  // CUDA-stream lanes and each stream's kernels in chain (= time) order
  std::vector<int32_t> ranks;
  std::vector<int32_t> rank_stream_off;  // [n_ranks + 1]
  std::vector<int32_t> stream_rank;
  std::vector<int32_t> stream_lane;
  std::vector<int32_t> stream_node_off;  // [n_streams + 1]
  std::vector<int32_t> stream_nodes;
};

// Returns TS_OK or a TS_E_* code with `err` set to the reference-style message.
int compile_graph(const ts_graph_desc& desc, CompiledGraph& out, std::string& err);

}  // namespace lumos
