// ingest.hpp — trace events -> ExecutionGraph (host side, structure of arrays).
//
// Restates the reference graph builder (src/build.cpp) so that a trace built
// here yields the identical task numbering, fixed edges and runtime rules as
// tracesim::build_graph + merge_ranks: that graph is the input contract of
// the replay path.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "lumos_b200.h"

namespace lumos {

// EventCategory (types.hpp:20-27)
enum Cat : uint8_t { CAT_CPU_OP = 0, CAT_RUNTIME = 1, CAT_KERNEL = 2, CAT_MEMCPY = 3,
                     CAT_MEMSET = 4, CAT_METADATA = 5 };

constexpr int64_t kNoArg = INT64_MIN;

// One normalized trace event (TraceEvent, types.hpp:57-67) with the two args
// the builder interprets ("event", "stream", build.cpp:29-37) pre-parsed.
struct Event {
  int32_t name = 0;  // index into Names
  uint8_t cat = CAT_METADATA;
  int64_t ts = 0;
  int64_t dur = 0;
  int32_t pid = 0;
  int32_t tid = 0;
  int64_t corr = -1;           // correlation id, -1 = none
  int32_t stream = -1;         // stream_id, -1 = none
  int64_t arg_event = kNoArg;  // args["event"]
  int64_t arg_stream = kNoArg; // args["stream"]
  int64_t op_index = -1;       // generator cost index (estimate mode), -1 = none
};

// TraceEvent::args / Task.meta as (key, value) strings in key order
using MetaList = std::vector<std::pair<std::string, std::string>>;

struct Names {
  std::vector<std::string> str;
  std::unordered_map<std::string, int32_t> idx;
  int32_t get(const std::string& s) {
    auto it = idx.find(s);
    if (it != idx.end()) return it->second;
    int32_t id = static_cast<int32_t>(str.size());
    str.push_back(s);
    idx.emplace(s, id);
    return id;
  }
};

// ExecutionGraph as SoA (the layout of ts_graph_desc).
struct HostGraph {
  std::vector<int64_t> duration, original_start;
  std::vector<int32_t> rank, lane_kind, lane;
  std::vector<uint8_t> op_class, task_kind;
  std::vector<int32_t> edge_from, edge_to;
  std::vector<int32_t> rule_kind, rule_task, rule_bound, rule_watch_off{0};
  std::vector<int32_t> watch_rank, watch_kind, watch_lane;
  int64_t window_start = 0, window_end = 0;
  std::vector<int32_t> gate_from, gate_to;
  std::vector<uint8_t> gate_kind;
  std::vector<int32_t> name;      // per task: index into the shared Names
  std::vector<int64_t> op_index;  // per task: generator cost index (-1 = none)
  // retime metadata (ts_graph_desc.rt_*), empty when unknown
  std::vector<uint8_t> rt_kind;
  std::vector<int64_t> rt_bytes;
  std::vector<int32_t> rt_group;
  std::vector<int64_t> rt_mnk;
  // Task.correlation_id (-1 = none) and Task.meta (build.cpp:355, 363), kept
  // on request for the structural what-if rebuild (rebuild.cpp); empty otherwise
  std::vector<int64_t> corr;
  std::vector<MetaList> meta;
  int32_t n_diagnostics = 0;

  int32_t n() const { return static_cast<int32_t>(duration.size()); }
  ts_graph_desc desc() const;
  // merge_ranks (build.cpp:512-542): append src with re-densified ids
  void append(const HostGraph& src, bool first);
  // copy of one rank's graph with every processor relabelled to new_rank
  void append_relabelled(const HostGraph& src, int32_t new_rank, bool first);
};

// BuildPolicy (build.hpp:17-44): the host-call names and communication
// patterns build_graph classifies by; defaults are the reference's.
struct BuildPolicyLite {
  int64_t gap_threshold_us = 1000;  // build.hpp:18
  std::vector<std::string> launch_names = {"cudaLaunchKernel", "cudaLaunchKernelExC",
                                           "cuLaunchKernel", "cudaLaunchCooperativeKernel",
                                           "cudaMemcpyAsync", "cudaMemsetAsync"};
  // name -> sync flavor: 1 device, 2 stream, 3 event
  std::vector<std::pair<std::string, int>> sync_names = {
      {"cudaDeviceSynchronize", 1}, {"cudaStreamSynchronize", 2}, {"cudaEventSynchronize", 3}};
  std::vector<std::string> record_names = {"cudaEventRecord"};
  std::vector<std::string> wait_names = {"cudaStreamWaitEvent"};
  std::vector<std::string> comm_patterns = {"nccl", "allreduce", "allgather", "reducescatter",
                                            "sendrecv", "alltoall"};
  bool is_launch(const std::string& n) const;
  bool is_record(const std::string& n) const;
  bool is_wait(const std::string& n) const;
  int sync_flavor(const std::string& n) const;  // 0 none
  bool is_comm(const std::string& n) const;     // case-insensitive substring
};
// BuildPolicy::from_json (build.cpp:41-66); false with `err` on a bad document
bool policy_from_json(const std::string& text, BuildPolicyLite& out, std::string& err);

// build_graph (build.cpp:338-510) over one rank's events.  Returns TS_OK or
// TS_E_GRAPH (cycle / GPU event without stream) with `err` set.
// With `meta` (parallel to events), the tasks keep their event's args and
// correlation id (HostGraph::meta / corr).
int build_rank_graph(const std::vector<Event>& events, const Names& names, int32_t rank,
                     const BuildPolicyLite& policy, HostGraph& out, std::string& err,
                     const std::vector<MetaList>* meta = nullptr);

// OpClass of an event (build.cpp:93-103), under `policy` or the default.
uint8_t classify_event(const Event& e, const Names& names, const BuildPolicyLite& policy);
uint8_t classify_event(const Event& e, const Names& names);
// BuildPolicy's communication-kernel name test (build.cpp:93-98)
bool is_comm_name(const std::string& name);

}  // namespace lumos
