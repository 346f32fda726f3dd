// batch_metrics_check.cpp — TEST INFRASTRUCTURE (built into oracle/_ref/ by
// oracle/Makefile, run by tests/test_gpu_dropin.py on a B200).
//
// Drives the C++ batched API of the drop-in (adapters/tracesim_b200.hpp) with
// the utilization and compare_replay outputs, and checks every scenario
// against the reference's own code on the same durations: the tick oracle
// (tests/oracles.cpp) replays the perturbed graph, and the reference
// metrics.cpp computes utilization_by_rank (metrics.cpp:105-155) and
// compare_replay (metrics.cpp:189-221) from it.  Scenario durations come from
// the C restatement of the scenario formula (lumos_oracle.c).
#include <cstdio>
#include <map>
#include <memory>
#include <vector>

#include "json.hpp"
#include "lumos_oracle.h"
#include "oracles.hpp"
#include "tracesim/build.hpp"
#include "tracesim/metrics.hpp"
#include "tracesim/pipeline.hpp"
#include "tracesim/simulate.hpp"
#include "tracesim/synth.hpp"
#include "tracesim/trace_parse.hpp"
#include "tracesim/transform.hpp"
#include "tracesim/cost.hpp"
#include "tracesim_b200.hpp"

using namespace tracesim;

int main() {
  nlohmann::json j;
  j["parallelism"] = {{"pp", 2}, {"dp", 2}, {"num_microbatches", 4}};
  j["model"] = {{"n_layers", 4}, {"d_model", 1024}, {"d_ffn", 4096}, {"n_heads", 16},
                {"d_head", 64}};
  SynthResult gen = generate(SynthSpec::from_json(j.dump()));
  std::map<int, ExecutionGraph> parts;
  for (const auto& [rank, evs] : split_by_rank(gen.events))
    parts[rank] = build_graph(evs, BuildPolicy(), rank);
  const ExecutionGraph g = merge_ranks(parts);

  b200::ScenarioSpec spec;
  spec.first = 40;
  spec.count = 24;
  spec.seed = 99;
  spec.jitter = 0.2;
  b200::BatchOptions opt;
  opt.util_bin_width = 4000;  // util_max_bins 0: every bin of every window
  opt.deltas = true;
  const b200::BatchResult r = b200::simulate_batch(g, spec, opt);

  orc_scenarios sc{};
  sc.seed = spec.seed;
  sc.jitter = spec.jitter;
  std::vector<int64_t> base, dur(g.tasks.size());
  for (const Task& t : g.tasks) base.push_back(t.duration);
  std::vector<uint8_t> cls(g.tasks.size(), 0);
  int bad = 0;
  for (int s = 0; s < spec.count; ++s) {
    orc_fill_durations(&sc, spec.first + s, static_cast<int32_t>(g.tasks.size()), base.data(),
                       cls.data(), dur.data());
    ExecutionGraph gs = g;
    for (std::size_t t = 0; t < gs.tasks.size(); ++t) gs.tasks[t].duration = dur[t];
    const SimulatedTrace sim = oracle::tick_simulate(gs);
    if (sim.makespan != r.span[3 * s + 2]) ++bad;
    IterationWindow w = g.iteration_window;
    w.end = std::max(w.end, w.start + sim.makespan);
    auto want = utilization_by_rank(task_intervals(gs, &sim), w, opt.util_bin_width);
    auto got = b200::utilization_by_rank(r, s, g.iteration_window);
    if (want.size() != got.size()) ++bad;
    for (const auto& [rank, ws] : want) {
      const auto& gs_ = got.at(rank);
      if (ws.bins.size() != gs_.bins.size()) { ++bad; continue; }
      for (std::size_t b = 0; b < ws.bins.size(); ++b)
        if (ws.bins[b].start != gs_.bins[b].start || ws.bins[b].value != gs_.bins[b].value) ++bad;
    }
    const ReplayReport a = compare_replay(g, sim), b = b200::replay_report(g, r, s);  // worst 10
    if (a.reference_makespan != b.reference_makespan || a.simulated_makespan != b.simulated_makespan ||
        a.max_abs_delta != b.max_abs_delta || a.mean_abs_delta != b.mean_abs_delta ||
        a.relative_error != b.relative_error || a.worst.size() != b.worst.size())
      ++bad;
    for (std::size_t k = 0; k < a.worst.size() && k < b.worst.size(); ++k)
      if (a.worst[k].task != b.worst[k].task || a.worst[k].delta != b.worst[k].delta ||
          a.worst[k].simulated_start != b.worst[k].simulated_start ||
          a.worst[k].reference_start != b.worst[k].reference_start)
        ++bad;
  }
  // what-if retime through the C++ API vs the reference transforms
  // (change_hidden then scale_dp, transform.cpp:741-755) replayed by the tick oracle
  b200::ScenarioSpec rs;
  rs.count = 6;
  rs.source_dp = 2;
  rs.source_model[0] = 1024;
  rs.source_model[1] = 4096;
  rs.source_model[2] = 350000000;
  const int tdp[6] = {2, 4, 8, 2, 4, 16};
  const int64_t tm[6][3] = {{1024, 4096, 350000000}, {1536, 6144, 780000000},
                            {2048, 8192, 1380000000}, {1024, 8192, 600000000},
                            {1024, 4096, 350000000}, {1536, 4096, 500000000}};
  for (int s = 0; s < rs.count; ++s) {
    rs.alpha_us.push_back(s % 2 ? 10.0 : 4.5);
    rs.bytes_per_us.push_back(s < 3 ? 50000.0 : 22222.2);
    rs.target_dp.push_back(tdp[s]);
    for (int k = 0; k < 3; ++k) rs.target_model.push_back(tm[s][k]);
  }
  b200::BatchOptions ro;
  ro.timestamps = true;
  const b200::BatchResult rr = b200::simulate_batch(g, rs, ro);
  int bad_rt = 0;
  for (int s = 0; s < rs.count; ++s) {
    AnalyticalCostModel model(rs.alpha_us[s], rs.bytes_per_us[s]);
    ModelConfig sm, tmc;
    sm.d_model = 1024;
    sm.d_ffn = 4096;
    sm.n_params = 350000000;
    tmc.d_model = static_cast<int>(tm[s][0]);
    tmc.d_ffn = static_cast<int>(tm[s][1]);
    tmc.n_params = tm[s][2];
    ExecutionGraph gt = change_hidden(g, sm, tmc, model);
    if (tdp[s] != 2) gt = scale_dp(gt, 2, tdp[s], model);
    const SimulatedTrace sim = oracle::tick_simulate(gt);
    std::vector<int64_t> st(g.tasks.size());
    for (const auto& e : sim.entries) st[e.task_id] = e.sim_start;
    for (std::size_t t = 0; t < g.tasks.size(); ++t)
      if (st[t] != rr.start[t * rs.count + s]) {
        ++bad_rt;
        break;
      }
    if (sim.makespan != rr.span[3 * s + 2]) ++bad_rt;
  }
  // selected-scenario traces (for simulated_to_chrome_json) equal the batch's
  {
    const std::vector<int64_t> ids = {spec.first + 3, spec.first + 17};
    b200::BatchOptions to;
    to.timestamps = true;
    const b200::BatchResult full = b200::simulate_batch(g, spec, to);
    const auto traces = b200::replay_scenarios(g, spec, ids);
    for (std::size_t q = 0; q < ids.size(); ++q) {
      const SimulatedTrace a = b200::scenario_trace(g, full, static_cast<std::size_t>(ids[q] - spec.first));
      const SimulatedTrace& b = traces[q];
      bool same = a.makespan == b.makespan && a.entries.size() == b.entries.size();
      for (std::size_t i = 0; same && i < a.entries.size(); ++i)
        same = a.entries[i].task_id == b.entries[i].task_id &&
               a.entries[i].sim_start == b.entries[i].sim_start &&
               a.entries[i].sim_end == b.entries[i].sim_end;
      if (!same || simulated_to_chrome_json(g, b).size() < 100) ++bad;
    }
  }
  bool threw = false;
  try {
    b200::ScenarioSpec e1 = rs;
    e1.target_dp.assign(rs.count, 1);
    b200::simulate_batch(g, e1, ro);
  } catch (const TransformError& e) {
    threw = std::string(e.what()).find("cannot drop gradient collectives") != std::string::npos;
  }
  if (!threw) ++bad_rt;
  bad += bad_rt;
  // Mode B through the C++ API: estimate_batch(PipelineSpec) vs the
  // reference build_pipeline(spec, hook) (pipeline.cpp:474-477), for the spec
  // pipeline_spec_for builds and a hand-edited one; makespans of nominal and
  // jittered scenarios (hook slot op_index[t] = the scenario duration of t)
  int bad_est = 0;
  {
    nlohmann::json je;
    je["parallelism"] = {{"pp", 3}, {"dp", 2}, {"num_microbatches", 5}};
    je["model"] = {{"n_layers", 6}, {"d_model", 1024}, {"d_ffn", 4096}, {"n_heads", 16},
                   {"d_head", 64}};
    PipelineSpec base_spec = pipeline_spec_for(SynthSpec::from_json(je.dump()));
    PipelineSpec edited = base_spec;
    edited.num_microbatches = 7;
    edited.host.launch = 9;
    edited.stages[1].layers_fwd[0].push_back({"fused_dropout", 41, OpClass::Compute, {}});
    edited.stages[1].layers_bwd[0].push_back({"fused_dropout_bwd", 57, OpClass::Compute, {}});
    edited.stages[2].optimizer.push_back({"clip_grad", 33, OpClass::Compute, {{"bytes", "4096"}}});
    for (const PipelineSpec* ps : {&base_spec, &edited}) {
      b200::ScenarioSpec es;
      es.first = 11;
      es.count = 6;
      es.seed = 5;
      es.jitter = 0.15;
      b200::BatchOptions eo;
      eo.timestamps = true;
      const b200::EstimateResult er = b200::estimate_batch(*ps, es, eo);
      const BuiltPipeline nominal = build_pipeline(*ps);
      if (er.truth_makespan != nominal.end - ps->origin) ++bad_est;
      orc_scenarios esc{};
      esc.seed = es.seed;
      esc.jitter = es.jitter;
      const std::size_t n = er.base.size();
      std::vector<uint8_t> ecls(n, 0);
      std::vector<int64_t> d(n);
      for (int s = 0; s < es.count; ++s) {
        orc_fill_durations(&esc, es.first + s, static_cast<int32_t>(n), er.base.data(),
                           ecls.data(), d.data());
        std::vector<Micros> hook(static_cast<std::size_t>(er.n_ops), 0);
        for (std::size_t t = 0; t < n; ++t)
          if (er.op_index[t] >= 0) hook[static_cast<std::size_t>(er.op_index[t])] = d[t];
        const BuiltPipeline b = build_pipeline(
            *ps, [&](std::size_t i, Micros base) { return i < hook.size() ? hook[i] : base; });
        if (b.end - ps->origin != er.batch.span[3 * s + 2]) {
          ++bad_est;
          std::printf("estimate_batch mismatch: spec %s scenario %d makespan %lld vs %lld\n",
                      ps == &base_spec ? "pipeline_spec_for" : "edited", s,
                      static_cast<long long>(er.batch.span[3 * s + 2]),
                      static_cast<long long>(b.end - ps->origin));
        }
      }
    }
  }
  bad += bad_est;
  // structural what-if through the C++ API: estimate_whatif(source graph,
  // WhatIfConfig) rebuilds the spec on the device library's host side; its
  // nominal makespan equals simulate() of the reference apply_whatif graph
  // (test_transform.cpp:294-304) and every scenario equals the reference
  // build_pipeline(rebuilt spec, hook)
  int bad_wi = 0;
  {
    WhatIfConfig cfg;
    cfg.source_model = SynthSpec::from_json(j.dump()).model;
    cfg.target_model = cfg.source_model;
    cfg.target_model.n_layers = 8;
    cfg.source_par = SynthSpec::from_json(j.dump()).par;
    cfg.target_par = cfg.source_par;
    cfg.target_par.pp = 4;
    cfg.target_par.dp = 4;
    cfg.target_par.num_microbatches = 8;
    cfg.cost_model = std::make_shared<AnalyticalCostModel>(10.0, 50000.0);
    b200::ScenarioSpec es;
    es.first = 2;
    es.count = 5;
    es.seed = 17;
    es.jitter = 0.2;
    b200::BatchOptions eo;
    eo.timestamps = true;
    const b200::WhatIfEstimate we = b200::estimate_whatif(g, cfg, es, eo);
    const TransformResult ref = apply_whatif(g, cfg);
    if (!we.rebuilt || we.truth_makespan != simulate(ref.graph).makespan) {
      ++bad_wi;
      std::printf("estimate_whatif: rebuilt %d nominal %lld vs reference %lld\n",
                  static_cast<int>(we.rebuilt), static_cast<long long>(we.truth_makespan),
                  static_cast<long long>(simulate(ref.graph).makespan));
    }
    orc_scenarios esc{};
    esc.seed = es.seed;
    esc.jitter = es.jitter;
    const std::size_t n = we.base.size();
    std::vector<uint8_t> ecls(n, 0);
    std::vector<int64_t> d(n);
    for (int s = 0; s < es.count && we.rebuilt; ++s) {
      orc_fill_durations(&esc, es.first + s, static_cast<int32_t>(n), we.base.data(),
                         ecls.data(), d.data());
      std::vector<Micros> hook(static_cast<std::size_t>(we.n_ops), 0);
      for (std::size_t t = 0; t < n; ++t)
        if (we.op_index[t] >= 0) hook[static_cast<std::size_t>(we.op_index[t])] = d[t];
      const BuiltPipeline b = build_pipeline(
          we.spec, [&](std::size_t i, Micros base) { return i < hook.size() ? hook[i] : base; });
      if (b.end - we.spec.origin != we.batch.span[3 * s + 2]) ++bad_wi;
    }
  }
  bad += bad_wi;
  std::printf("%s: %d scenarios, %zu tasks, %d mismatches (retime: %d scenarios, %d; "
              "estimate_batch: %d; estimate_whatif: %d)\n",
              bad ? "FAIL" : "PASS", spec.count, g.tasks.size(), bad, rs.count, bad_rt, bad_est,
              bad_wi);
  return bad ? 1 : 0;
}
