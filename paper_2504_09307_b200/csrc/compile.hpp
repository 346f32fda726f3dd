// compile.hpp — ExecutionGraph (C-ABI SoA view) -> device programs.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "lumos_b200.h"
#include "program.hpp"

namespace lumos {

// Tables of the exact event-driven replay (the reference Engine, restated on
// the device for graphs outside the chained class and for scenarios whose
// sync certificate fails).
struct DesTables {
  int32_t n_lanes = 0;
  std::vector<int32_t> lane_of;     // [n]
  std::vector<int32_t> lane_off;    // [n_lanes + 1]: each lane's ready-heap region
  std::vector<int32_t> lane_tasks;  // [n] tasks of each lane, (original_start, id) order
  std::vector<int64_t> ostart;      // [n] dispatch key (original_start)
  std::vector<int32_t> succ_off, succ, indeg0;
  std::vector<int32_t> rule_of;     // [n] -> rule or -1
  std::vector<int32_t> rule_kind, rule_bound, rule_wl_off, rule_wl;  // watched lane ids
  std::vector<int32_t> lane_rank;   // [n_lanes] rank slot
  std::vector<int32_t> lane_stream; // [n_lanes] stream slot or -1 (CPU lane)
};

struct CompiledGraph {
  int32_t n_tasks = 0;
  int64_t window_start = 0;
  int64_t window_end = 0;
  std::vector<Op> ops;  // Op and OpExt records (both 32 bytes)
  std::vector<ProgramDesc> programs;
  std::vector<ComponentDesc> comps;
  int32_t max_slots = 0;
  // cooperative components (program.hpp OP_POST / OP_WAIT): per component its
  // rank programs coop_progs[coop_prog_off[c] .. coop_prog_off[c+1]) (one entry
  // for a single-rank component)
  std::vector<int32_t> coop_prog_off, coop_progs;
  // split breakdown accounting (program.hpp FusedDesc): per component its
  // descriptor; per rank row the compute kernels that may overlap a comm kernel
  // (chain order), CSR over rank rows
  std::vector<FusedDesc> fused;
  int32_t n_fused = 0;  // components with row >= 0
  std::vector<int32_t> cand_off, cand_nodes;
  std::vector<FusedDesc> fused_rows;  // every fused rank (single-program and cooperative)
  std::vector<int32_t> coop_rows;     // parallel to coop_progs: the rank row a warp accounts, -1
  int32_t max_mailboxes = 0;
  int32_t max_coop_ranks = 1;
  int64_t max_coop_path = 0;  // nominal longest path of a cooperative component
  // largest per-component sum of base durations and task count: with the
  // scenario's worst-case duration factor they bound every time of a replay
  // (W + any path <= W + sum of the component's durations), which decides
  // whether the walk may keep uint32 offsets from W
  int64_t max_comp_dur_sum = 0;
  int64_t max_comp_path = 0;  // nominal longest path (W-relative) over all components
  int32_t max_comp_tasks = 0;
  int32_t n_syncs = 0;
  int32_t n_gpu_tasks = 0;

  // per-task arrays used by the duration kernel and the reductions
  std::vector<int64_t> base;
  std::vector<uint8_t> scale_class;
  std::vector<uint8_t> is_comm;
  // retime metadata (ts_graph_desc.rt_*), empty when the graph carries none
  std::vector<uint8_t> rt_kind;
  std::vector<int64_t> rt_bytes;
  std::vector<int32_t> rt_group;
  std::vector<int64_t> rt_mnk;  // [n][3]
  // retime walk: per op record the dense index of its F_RT task (-1 for other
  // records), and per dense index the task whose metadata it carries
  std::vector<int32_t> rt_rec_of;
  std::vector<int32_t> rt_rec_task;

  // reductions: ranks (sorted, = ranks_in(graph), build.cpp:582-590), their
  // CUDA-stream lanes and each stream's kernels in chain (= time) order
  std::vector<int32_t> ranks;
  std::vector<int32_t> rank_stream_off;  // [n_ranks + 1]
  std::vector<int32_t> stream_rank;
  std::vector<int32_t> stream_lane;
  std::vector<int32_t> stream_node_off;  // [n_streams + 1]
  std::vector<int32_t> stream_nodes;

  // event-driven path
  bool des_only = false;    // graph outside the chained class
  std::string des_reason;   // why (the compiler's message)
  DesTables des;
};

// Returns TS_OK or a TS_E_* code with `err` set to the reference-style message.
// allow_coop = false compiles gated components as single programs (no
// cooperative per-rank split), as LUMOS_COOP=0 does.
int compile_graph(const ts_graph_desc& desc, CompiledGraph& out, std::string& err,
                  bool allow_coop = true);

}  // namespace lumos
