// tracesim_b200.hpp — batched extension of the tracesim replay API (declared
// next to the drop-in simulate(); implemented in tracesim_dropin.cpp on the
// B200 engine's C ABI).
#pragma once

#include <cstdint>
#include <vector>

#include "tracesim/build.hpp"

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
};

struct BatchResult {
  std::vector<int64_t> start, fin;     // [task][scenario] (when requested)
  std::vector<int64_t> span;           // [scenario][3] {start, end, makespan}
  std::vector<int64_t> rank_breakdown; // [scenario][rank][5] (metrics.hpp:33-39 order)
  std::vector<int32_t> ranks;          // rank of each breakdown row
};

BatchResult simulate_batch(const ExecutionGraph& graph, const ScenarioSpec& spec,
                           bool timestamps = false);

}  // namespace tracesim::b200
