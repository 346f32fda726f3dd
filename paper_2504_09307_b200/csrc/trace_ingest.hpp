// trace_ingest.hpp — parallel Chrome-trace ingest (trace_ingest.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <utility>
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

// The reference's input options (cli.cpp:52-58 InputOptions)
struct IngestOptions {
  std::vector<std::string> paths;  // --trace
  std::string manifest;            // --manifest: JSON {rank: path}
  std::string window = "full";     // --window: full | auto | START:END
  // CategoryTable overrides merged over the defaults (CategoryTable::from_json)
  std::vector<std::pair<std::string, uint8_t>> categories;
  BuildPolicyLite policy;          // --policy (BuildPolicy::from_json)
  int threads = 0;                 // host threads (<= 0: all cores)
  bool keep_meta = false;          // keep Task.meta / correlation ids (what-if rebuild)
  bool dom_only = false;           // skip the fast scanner (LUMOS_INGEST_DOM=1; tests)
};

// build_from_inputs (cli.cpp:118-137): parse_trace of every input,
// load_inputs' rank assignment (manifest, pid split, rank_<N> files), the
// iteration window (detect_iteration_window / filter_window), build_graph per
// rank and merge_ranks — files parsed and ranks built on host threads.
// Returns TS_OK or a TS_E_* code with `err` set (ParseError / GraphError text).
int ingest_traces(const IngestOptions& opts, Names& names, HostGraph& out,
                  std::vector<RtMeta>& task_rt, std::string& err);
// CategoryTable::from_json (trace_parse.cpp:186-211) overrides; false + err
bool categories_from_json(const std::string& text,
                          std::vector<std::pair<std::string, uint8_t>>& out, std::string& err);

// the graph's ts_graph_desc.rt_* arrays from per-task metadata
void fill_retime_arrays(HostGraph& g, const std::vector<RtMeta>& rt);

}  // namespace lumos
