// trace_ingest.hpp — parallel Chrome-trace ingest (trace_ingest.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ingest.hpp"

namespace lumos {

// the Task.meta keys the retime transforms read (transform.cpp:219-349)
struct RtMeta {
  int64_t bytes = -1;  // "bytes" (strict integer), -1 = absent
  int64_t group = 0;   // "group_size"
  int64_t m = 0, n = 0, k = 0;
  bool allreduce = false, region_opt = false, region_p2p = false, dir_recv = false;
};

// parse_trace + rank assignment + build_graph per rank + merge_ranks over
// `paths` (window "full"), on `threads` host threads (<= 0: all cores).
// Returns TS_OK or a TS_E_* code with `err` set (ParseError / GraphError text).
int ingest_trace_files(const std::vector<std::string>& paths, int threads,
                       const BuildPolicyLite& policy, Names& names, HostGraph& out,
                       std::vector<RtMeta>& task_rt, std::string& err);

// the graph's ts_graph_desc.rt_* arrays from per-task metadata
void fill_retime_arrays(HostGraph& g, const std::vector<RtMeta>& rt);

}  // namespace lumos
