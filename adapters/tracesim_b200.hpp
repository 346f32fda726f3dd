// tracesim_b200.hpp — batched extension of the tracesim replay API (declared
// next to the drop-in simulate(); implemented in tracesim_dropin.cpp on the
// B200 engine's C ABI).
#pragma once

#include <cstdint>
#include <map>
#include <vector>

#include "tracesim/build.hpp"
#include "tracesim/metrics.hpp"
#include "tracesim/pipeline.hpp"
#include "tracesim/simulate.hpp"
#include "tracesim/transform.hpp"

namespace tracesim::b200 {

// N duration scenarios of one graph.  Durations are a pure function of
// (seed, global scenario id, task): per-class rational scale (transform.cpp:38-43
// mul_div) then jitter max(1, llround(d * (1 + u))) (synth.cpp:150-155).
struct ScenarioSpec {
  int64_t first = 0;
  int32_t count = 1;
  uint64_t seed = 250409307;
  double jitter = 0.0;
  int32_t scale_lo = 0, scale_hi = 0, scale_den = 0;  // den <= 0: no class scaling
  // What-if retime per scenario (non-empty alpha_us enables it): scenario s
  // replays apply_whatif's retime of the graph — change_hidden(source_model ->
  // target_model[s]) then scale_dp(source_dp -> target_dp[s]) with
  // AnalyticalCostModel(alpha_us[s], bytes_per_us[s]) (transform.cpp:741-755).
  // Errors throw TransformError with the reference's messages.
  std::vector<double> alpha_us, bytes_per_us;  // [count]
  int32_t source_dp = 1;
  std::vector<int32_t> target_dp;              // [count] or empty
  int64_t source_model[3] = {0, 0, 0};         // {d_model, d_ffn, n_params}
  std::vector<int64_t> target_model;           // [count * 3] or empty
};

struct BatchOptions {
  bool timestamps = false;
  int64_t util_bin_width = 0;  // > 0: utilization_by_rank bins (metrics.cpp:105-155)
  int32_t util_max_bins = 0;   // 0: every bin of every window; > 0: a cap (a window
                               // needing more throws std::invalid_argument)
  bool deltas = false;         // compare_replay start deltas (metrics.cpp:189-221)
  int32_t worst_n = 10;        // compare_replay's worst list length (metrics.hpp:82-83), <= 64
};

struct BatchResult {
  std::vector<int64_t> start, fin;     // [task][scenario] (when requested)
  std::vector<int64_t> span;           // [scenario][3] {start, end, makespan}
  std::vector<int64_t> rank_breakdown; // [scenario][rank][5] (metrics.hpp:33-39 order)
  std::vector<int32_t> ranks;          // rank of each breakdown row
  int64_t util_bin_width = 0;
  int32_t util_max_bins = 0;
  std::vector<int64_t> util_covered;   // [scenario][rank][util_max_bins] covered us
  std::vector<int32_t> util_n_bins;    // [scenario] bins each window needs
  std::vector<int64_t> delta_abs_sum;  // [scenario] sum |sim_start - original_start|
  std::vector<int64_t> delta_worst;    // [scenario][worst_n][3] {|delta|, task (-1: none), delta}
  int32_t worst_n = 0;
  int32_t n_fixups = 0;                // scenarios re-run by the exact event-driven path
};

BatchResult simulate_batch(const ExecutionGraph& graph, const ScenarioSpec& spec,
                           bool timestamps = false);
BatchResult simulate_batch(const ExecutionGraph& graph, const ScenarioSpec& spec,
                           const BatchOptions& options);

// Scenario s of a batch in the reference's metric types.
// utilization_by_rank over [window.start, max(window.end, window.start + makespan))
// (cli.cpp:303-316); bins past util_max_bins are not returned.
std::map<int, UtilizationSeries> utilization_by_rank(const BatchResult& r, std::size_t s,
                                                     IterationWindow window);
// compare_replay of scenario s, worst list of BatchOptions::worst_n tasks.
ReplayReport replay_report(const ExecutionGraph& graph, const BatchResult& r, std::size_t s);

// Mode B: estimate() semantics.  The graph build_pipeline(spec, DurationHook)
// lays out (pipeline.cpp:474-477) — generator dependencies plus the p2p
// rendezvous and collective-barrier gates — replayed for every scenario on
// the device, tp replicas of each rank.  Task t of the estimate graph is hook
// slot op_index[t] (a launch takes two slots, pipeline.cpp:105-109); its base
// duration is base[t].  Scenario durations follow ScenarioSpec (class scale,
// jitter); retime fields are rejected (a structural what-if rebuilds the spec
// instead, transform.cpp:556-701).  Errors: std::invalid_argument as
// build_pipeline raises them.
struct EstimateResult {
  BatchResult batch;                 // timestamps / spans over the estimate graph's tasks
  std::vector<int64_t> op_index;     // [task] DurationHook slot, -1 none
  std::vector<int64_t> base;         // [task] intrinsic duration (the hook's base)
  std::vector<int32_t> rank;         // [task] rank (stage + pp * dp, replica r * tp + t)
  int64_t n_ops = 0;                 // hook slots of one replica
  int64_t truth_makespan = 0;        // BuiltPipeline end - origin at the base durations
};
EstimateResult estimate_batch(const PipelineSpec& spec, const ScenarioSpec& scenarios,
                              const BatchOptions& options = {}, int tp = 1);

// estimate() of a structural what-if, batched: the PipelineSpec
// rebuild_pipeline (transform.cpp:556-701) lays out for `cfg` from the
// measured source graph (tag_tasks + measure_pipeline over its Task.meta, on
// the host, ts_rebuild_pipeline), replayed like estimate_batch.  cfg's cost
// model must be an AnalyticalCostModel; errors throw TransformError with the
// reference's text.  rebuilt = false (nothing replayed) when the target
// differs in nothing the rebuild models — apply_whatif then retimes in place
// (ScenarioSpec's retime fields) or returns the source.
struct WhatIfEstimate : EstimateResult {
  bool rebuilt = false;
  PipelineSpec spec;  // the rebuilt spec
};
WhatIfEstimate estimate_whatif(const ExecutionGraph& source, const WhatIfConfig& cfg,
                               const ScenarioSpec& scenarios, const BatchOptions& options = {},
                               int tp = 1);

// Scenario s of a batch run with timestamps as a SimulatedTrace (entries in
// (sim_start, task_id) order, simulate.hpp:12-24) — e.g. for
// simulated_to_chrome_json (simulate.hpp:55) to audit a scenario visually.
SimulatedTrace scenario_trace(const ExecutionGraph& graph, const BatchResult& r, std::size_t s);
// Replays only the listed global scenario ids of `spec` (a scenario's
// durations are a pure function of its id, so these equal the same ids of any
// larger batch) and returns their traces; one compiled graph for all ids.
std::vector<SimulatedTrace> replay_scenarios(const ExecutionGraph& graph, const ScenarioSpec& spec,
                                             const std::vector<int64_t>& ids);

}  // namespace tracesim::b200
