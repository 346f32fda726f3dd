// tracesim_dropin.cpp — the reference-side binding: a replacement for
// /root/reference/proj/src/simulate.cpp that keeps the tracesim C++ API of
// include/tracesim/simulate.hpp verbatim and runs the replay on the B200
// engine through its C ABI (include/lumos_b200.h).
//
// A maintainer swaps this file in for src/simulate.cpp in the tracesim
// library and links liblumos_b200.so; every caller of
// simulate() — CLI replay/whatif/analyze (cli.cpp:181, 224-225, 307), the
// acceptance gate, the tests — then replays on the GPU.  Exceptions follow the
// reference taxonomy (types.hpp:109-138): invalid graphs and deadlocks throw
// SimulationError with the reference's message text ("invalid graph: ...";
// "deadlock with N tasks blocked: <witness ids>" as simulate.cpp:300 builds it).
//
// The batched entry point (not in the reference) is declared in
// tracesim_b200.hpp: N duration scenarios of one graph in one call.
#include <algorithm>
#include <limits>
#include <stdexcept>
#include <map>
#include <memory>
#include <optional>
#include <queue>
#include <sstream>
#include <string>
#include <vector>

#include "lumos_b200.h"
#include "tracesim/simulate.hpp"
#include "tracesim/trace_parse.hpp"
#include "tracesim/transform.hpp"
#include "tracesim_b200.hpp"

namespace tracesim {

namespace {

std::string ids_text(const std::vector<TaskId>& ids) {
  std::ostringstream os;
  for (std::size_t i = 0; i < ids.size(); ++i) os << (i ? " " : "") << ids[i];
  return os.str();
}

// ExecutionGraph -> structure of arrays the C ABI takes (ts_graph_desc)
struct Soa {
  std::vector<int64_t> duration, original_start;
  std::vector<int32_t> rank, lane_kind, lane;
  std::vector<uint8_t> op_class, task_kind;
  std::vector<int32_t> edge_from, edge_to;
  std::vector<int32_t> rule_kind, rule_task, rule_bound, rule_watch_off{0};
  std::vector<int32_t> watch_rank, watch_kind, watch_lane;
  ts_graph_desc desc{};

  explicit Soa(const ExecutionGraph& g) {
    for (const Task& t : g.tasks) {
      duration.push_back(t.duration);
      original_start.push_back(t.original_start);
      rank.push_back(t.processor.rank);
      lane_kind.push_back(t.processor.kind == LaneKind::CudaStream ? TS_LANE_CUDA_STREAM
                                                                   : TS_LANE_CPU_THREAD);
      lane.push_back(t.processor.lane);
      op_class.push_back(static_cast<uint8_t>(t.op_class));
      task_kind.push_back(t.kind == TaskKind::Gpu ? 1 : 0);
    }
    for (const auto& [u, v] : g.fixed_edges) {
      edge_from.push_back(u);
      edge_to.push_back(v);
    }
    for (const RuntimeRule& r : g.rules) {
      rule_kind.push_back(r.kind == RuntimeRule::Kind::StreamSync   ? TS_RULE_STREAM_SYNC
                          : r.kind == RuntimeRule::Kind::DeviceSync ? TS_RULE_DEVICE_SYNC
                                                                    : TS_RULE_EVENT_SYNC);
      rule_task.push_back(r.waiting_task);
      rule_bound.push_back(r.bound_task && *r.bound_task >= 0 ? *r.bound_task : -1);
      for (const ProcessorId& p : r.watched) {
        watch_rank.push_back(p.rank);
        watch_kind.push_back(p.kind == LaneKind::CudaStream ? TS_LANE_CUDA_STREAM
                                                            : TS_LANE_CPU_THREAD);
        watch_lane.push_back(p.lane);
      }
      rule_watch_off.push_back(static_cast<int32_t>(watch_rank.size()));
    }
    desc.n_tasks = static_cast<int32_t>(g.tasks.size());
    desc.duration = duration.data();
    desc.original_start = original_start.data();
    desc.rank = rank.data();
    desc.lane_kind = lane_kind.data();
    desc.lane = lane.data();
    desc.op_class = op_class.data();
    desc.task_kind = task_kind.data();
    desc.n_edges = static_cast<int64_t>(edge_from.size());
    desc.edge_from = edge_from.data();
    desc.edge_to = edge_to.data();
    desc.n_rules = static_cast<int32_t>(rule_kind.size());
    desc.rule_kind = rule_kind.data();
    desc.rule_task = rule_task.data();
    desc.rule_bound = rule_bound.data();
    desc.rule_watch_off = rule_watch_off.data();
    desc.watch_rank = watch_rank.data();
    desc.watch_kind = watch_kind.data();
    desc.watch_lane = watch_lane.data();
    desc.window_start = g.iteration_window.start;
    desc.window_end = g.iteration_window.end;
    // retime metadata: the TS_RT_* class change_hidden / scale_dp would apply
    // (transform.cpp:219-349), from Task.meta with strict integer parsing
    auto meta_i64 = [](const Task& t, const char* key) -> std::optional<int64_t> {
      auto it = t.meta.find(key);
      if (it == t.meta.end()) return std::nullopt;
      try {
        std::size_t pos = 0;
        const int64_t v = std::stoll(it->second, &pos);
        if (pos != it->second.size()) return std::nullopt;
        return v;
      } catch (const std::exception&) {
        return std::nullopt;
      }
    };
    auto meta_str = [](const Task& t, const char* key) {
      auto it = t.meta.find(key);
      return it == t.meta.end() ? std::string() : it->second;
    };
    for (const Task& t : g.tasks) {
      const auto b = meta_i64(t, "bytes");
      const auto gs = meta_i64(t, "group_size");
      const int64_t m = meta_i64(t, "m").value_or(0), n = meta_i64(t, "n").value_or(0),
                    k = meta_i64(t, "k").value_or(0);
      uint8_t kind = TS_RT_NONE;
      if (t.kind == TaskKind::Gpu && t.op_class == OpClass::Compute) {
        if (m > 0 && n > 0 && k > 0) kind = TS_RT_GEMM;
        else if (meta_str(t, "region") == "opt" && b) kind = TS_RT_OPT;
      } else if (t.kind == TaskKind::Gpu && t.op_class == OpClass::Communication) {
        if (meta_str(t, "collective") == "allreduce") kind = TS_RT_ALLREDUCE;
        else if (meta_str(t, "region") == "p2p" && b)
          kind = meta_str(t, "dir") != "recv" ? TS_RT_P2P_SEND : TS_RT_P2P_RECV;
      }
      rt_kind.push_back(kind);
      rt_bytes.push_back(b ? *b : -1);
      rt_group.push_back(gs ? static_cast<int32_t>(*gs) : 0);
      rt_mnk.insert(rt_mnk.end(), {m, n, k});
    }
    desc.rt_kind = rt_kind.data();
    desc.rt_bytes = rt_bytes.data();
    desc.rt_group = rt_group.data();
    desc.rt_mnk = rt_mnk.data();
  }
  std::vector<uint8_t> rt_kind;
  std::vector<int64_t> rt_bytes, rt_mnk;
  std::vector<int32_t> rt_group;
};

[[noreturn]] void rethrow(int rc, bool transform = false) {
  const std::string msg = ts_last_error();
  if (transform && rc == TS_E_INVALID_ARGUMENT) throw TransformError(msg);
  if (rc == TS_E_GRAPH) throw GraphError(msg);
  if (rc == TS_E_SIMULATION) throw SimulationError(msg);
  throw SimulationError("B200 replay engine: " + msg);
}

bool same_soa(const Soa& a, const Soa& b) {
  return a.duration == b.duration && a.original_start == b.original_start && a.rank == b.rank &&
         a.lane_kind == b.lane_kind && a.lane == b.lane && a.op_class == b.op_class &&
         a.task_kind == b.task_kind && a.edge_from == b.edge_from && a.edge_to == b.edge_to &&
         a.rule_kind == b.rule_kind && a.rule_task == b.rule_task &&
         a.rule_bound == b.rule_bound && a.rule_watch_off == b.rule_watch_off &&
         a.watch_rank == b.watch_rank && a.watch_kind == b.watch_kind &&
         a.watch_lane == b.watch_lane && a.rt_kind == b.rt_kind && a.rt_bytes == b.rt_bytes &&
         a.rt_group == b.rt_group && a.rt_mnk == b.rt_mnk &&
         a.desc.window_start == b.desc.window_start && a.desc.window_end == b.desc.window_end;
}

// The last compiled graph of this thread: repeated replays of one graph (the
// CLI's whatif / analyze flows, parameter sweeps) compile and upload it once.
// A graph is reused only when every field the engine reads is identical.
// Per thread, because one ts_graph serves one call at a time.
struct GraphCache {
  std::unique_ptr<Soa> soa;
  ts_graph* g = nullptr;
  ~GraphCache() { ts_graph_destroy(g); }
};
thread_local GraphCache t_cache;

struct Handle {
  ts_graph* g = nullptr;
  explicit Handle(const ExecutionGraph& graph) {
    auto s = std::make_unique<Soa>(graph);
    if (t_cache.g && t_cache.soa && same_soa(*s, *t_cache.soa)) {
      g = t_cache.g;
      return;
    }
    ts_graph* fresh = nullptr;
    if (int rc = ts_graph_create(&s->desc, -1, &fresh)) rethrow(rc);
    ts_graph_destroy(t_cache.g);
    t_cache.g = g = fresh;
    t_cache.soa = std::move(s);
  }
};

}  // namespace

std::vector<ValidationIssue> validate_graph(const ExecutionGraph& graph) {
  using K = ValidationIssue::Kind;
  std::vector<ValidationIssue> out;
  const TaskId n = static_cast<TaskId>(graph.tasks.size());
  for (const Task& t : graph.tasks)
    if (t.duration < 0)
      out.push_back({K::NegativeDuration, true,
                     "task " + std::to_string(t.id) + " has negative duration", {t.id}});
  auto in_range = [n](TaskId x) { return x >= 0 && x < n; };
  bool edges_valid = true;
  for (const auto& [u, v] : graph.fixed_edges)
    if (!in_range(u) || !in_range(v) || u == v) {
      edges_valid = false;
      out.push_back({K::BadEdge, true,
                     "edge " + std::to_string(u) + "->" + std::to_string(v) +
                         " references an invalid task",
                     {u, v}});
    }
  for (const RuntimeRule& r : graph.rules) {
    const bool bad_bound = r.bound_task && *r.bound_task >= 0 && *r.bound_task >= n;
    if (!in_range(r.waiting_task) || bad_bound) {
      out.push_back({K::BadRule, true,
                     "rule on task " + std::to_string(r.waiting_task) +
                         " references an invalid task",
                     {r.waiting_task}});
    } else if (r.kind != RuntimeRule::Kind::EventSync && r.watched.empty()) {
      out.push_back({K::EmptyScope, false,
                     "sync task " + std::to_string(r.waiting_task) +
                         " watches no lanes and will not block",
                     {r.waiting_task}});
    }
  }
  if (!edges_valid || n == 0) return out;
  for (const auto& [u, v] : graph.fixed_edges) {
    const Task& a = graph.tasks[u];
    const Task& b = graph.tasks[v];
    if (a.processor == b.processor && a.original_start > b.original_start)
      out.push_back({K::ChainOrder, false,
                     "edge " + std::to_string(u) + "->" + std::to_string(v) +
                         " runs against original start order on " + to_string(a.processor),
                     {u, v}});
  }
  // Kahn; on failure walk unmet predecessors (smallest id) until one repeats
  std::vector<int> remaining(n, 0);
  std::vector<std::vector<TaskId>> succ(n), pred(n);
  for (const auto& [u, v] : graph.fixed_edges) {
    succ[u].push_back(v);
    pred[v].push_back(u);
    ++remaining[v];
  }
  std::queue<TaskId> ready;
  for (TaskId i = 0; i < n; ++i)
    if (remaining[i] == 0) ready.push(i);
  TaskId done = 0;
  while (!ready.empty()) {
    const TaskId u = ready.front();
    ready.pop();
    ++done;
    for (TaskId v : succ[u])
      if (--remaining[v] == 0) ready.push(v);
  }
  if (done == n) return out;
  TaskId cur = -1;
  for (TaskId i = 0; i < n && cur < 0; ++i)
    if (remaining[i] > 0) cur = i;
  std::vector<TaskId> path;
  std::vector<char> seen(n, 0);
  while (cur >= 0 && !seen[cur]) {
    seen[cur] = 1;
    path.push_back(cur);
    TaskId next = -1;
    for (TaskId p : pred[cur])
      if (remaining[p] > 0 && (next < 0 || p < next)) next = p;
    cur = next;
  }
  std::vector<TaskId> cycle;
  if (cur >= 0) {
    cycle.assign(std::find(path.begin(), path.end(), cur), path.end());
    std::reverse(cycle.begin(), cycle.end());
  }
  out.push_back({K::Cycle, true, "dependency cycle: " + ids_text(cycle), cycle});
  return out;
}

TaskId pick_ready(const ExecutionGraph& graph, std::span<const TaskId> ready) {
  TaskId best = -1;
  for (TaskId id : ready)
    if (best < 0 || std::pair(graph.tasks[id].original_start, id) <
                        std::pair(graph.tasks[best].original_start, best))
      best = id;
  return best;
}

SimulatedTrace simulate(const ExecutionGraph& graph) {
  for (const ValidationIssue& issue : validate_graph(graph))
    if (issue.error) throw SimulationError("invalid graph: " + issue.message);
  const std::size_t n = graph.tasks.size();
  SimulatedTrace out;
  if (n == 0) {
    out.start = out.end = graph.iteration_window.start;
    return out;
  }
  Handle h(graph);
  std::vector<int64_t> start(n), fin(n), span(3);
  if (int rc = ts_simulate(h.g, start.data(), fin.data(), span.data())) rethrow(rc);
  out.entries.reserve(n);
  for (std::size_t i = 0; i < n; ++i)
    out.entries.push_back(
        {static_cast<TaskId>(i), start[i], fin[i], graph.tasks[i].processor});
  std::sort(out.entries.begin(), out.entries.end(), [](const SimEntry& a, const SimEntry& b) {
    return std::pair(a.sim_start, a.task_id) < std::pair(b.sim_start, b.task_id);
  });
  out.start = span[0];
  out.end = span[1];
  out.makespan = span[2];
  return out;
}

std::string simulated_to_chrome_json(const ExecutionGraph& graph, const SimulatedTrace& sim) {
  std::vector<TraceEvent> events;
  events.reserve(sim.entries.size());
  for (const SimEntry& e : sim.entries) {
    const Task& t = graph.tasks[e.task_id];
    TraceEvent ev;
    ev.name = t.name;
    if (t.kind == TaskKind::Gpu) {
      ev.category = EventCategory::GpuKernel;
      ev.stream_id = t.processor.lane;
    } else {
      const bool runtime = t.op_class == OpClass::Launch || t.op_class == OpClass::Sync ||
                           t.op_class == OpClass::EventRecord ||
                           t.op_class == OpClass::EventWait;
      ev.category = runtime ? EventCategory::CudaRuntime : EventCategory::CpuOp;
    }
    ev.timestamp = e.sim_start;
    ev.duration = e.sim_end - e.sim_start;
    ev.process_id = t.processor.rank;
    ev.thread_id = t.processor.lane;
    ev.correlation_id = t.correlation_id;
    ev.args = t.meta;
    if (t.layer_tag) ev.args["layer"] = std::to_string(*t.layer_tag);
    if (t.microbatch_tag) ev.args["microbatch"] = std::to_string(*t.microbatch_tag);
    events.push_back(std::move(ev));
  }
  return chrome_json(events);
}

namespace b200 {

BatchResult simulate_batch(const ExecutionGraph& graph, const ScenarioSpec& spec,
                           bool timestamps) {
  BatchOptions o;
  o.timestamps = timestamps;
  return simulate_batch(graph, spec, o);
}

namespace {

// one batched replay of a compiled graph through the C ABI
BatchResult run_batch(ts_graph* g, std::size_t n_tasks, const ScenarioSpec& spec,
                      const BatchOptions& o, int32_t util_bins) {
  ts_graph_info info{};
  ts_graph_get_info(g, &info);
  BatchResult r;
  const std::size_t S = static_cast<std::size_t>(spec.count);
  const std::size_t R = static_cast<std::size_t>(info.n_ranks);
  r.span.assign(S * 3, 0);
  r.rank_breakdown.assign(S * R * 5, 0);
  r.ranks.resize(R);
  ts_graph_ranks(g, r.ranks.data());
  if (o.timestamps) {
    r.start.assign(n_tasks * S, 0);
    r.fin.assign(n_tasks * S, 0);
  }
  ts_scenarios sc{};
  sc.first = spec.first;
  sc.count = spec.count;
  sc.seed = spec.seed;
  sc.jitter = spec.jitter;
  sc.scale_lo = spec.scale_lo;
  sc.scale_hi = spec.scale_hi;
  sc.scale_den = spec.scale_den;
  ts_retime rt{};
  const bool retime = !spec.alpha_us.empty();
  if (retime) {
    // the C ABI reads count (3 * count) entries of every per-scenario array
    if (spec.alpha_us.size() != S || spec.bytes_per_us.size() != S)
      throw std::invalid_argument("retime needs alpha_us and bytes_per_us per scenario (count entries)");
    if (!spec.target_dp.empty() && spec.target_dp.size() != S)
      throw std::invalid_argument("target_dp needs count entries (or none)");
    if (!spec.target_model.empty() && spec.target_model.size() != 3 * S)
      throw std::invalid_argument("target_model needs 3 * count entries (or none)");
    rt.alpha_us = spec.alpha_us.data();
    rt.bytes_per_us = spec.bytes_per_us.data();
    rt.source_dp = spec.source_dp;
    rt.target_dp = spec.target_dp.empty() ? nullptr : spec.target_dp.data();
    for (int k = 0; k < 3; ++k) rt.source_model[k] = spec.source_model[k];
    rt.target_model = spec.target_model.empty() ? nullptr : spec.target_model.data();
    sc.retime = &rt;
  }
  ts_result res{};
  res.start = o.timestamps ? r.start.data() : nullptr;
  res.fin = o.timestamps ? r.fin.data() : nullptr;
  res.ld = spec.count;
  res.span = r.span.data();
  res.rank_breakdown = R ? r.rank_breakdown.data() : nullptr;
  if (o.util_bin_width > 0) {
    r.util_bin_width = o.util_bin_width;
    r.util_max_bins = std::max<int32_t>(1, util_bins);
    r.util_covered.assign(S * std::max<std::size_t>(1, R) * r.util_max_bins, 0);
    r.util_n_bins.assign(S, 0);
    res.util_bin_width = r.util_bin_width;
    res.util_max_bins = r.util_max_bins;
    res.util_covered = R ? r.util_covered.data() : nullptr;
    res.util_n_bins = r.util_n_bins.data();
  }
  if (o.deltas) {
    if (o.worst_n < 1) throw std::invalid_argument("worst_n must be >= 1");
    r.worst_n = o.worst_n;
    r.delta_abs_sum.assign(S, 0);
    r.delta_worst.assign(S * static_cast<std::size_t>(o.worst_n) * 3, 0);
    res.delta_abs_sum = r.delta_abs_sum.data();
    res.delta_worst = r.delta_worst.data();
    res.delta_worst_n = o.worst_n;
  }
  res.n_fixups = &r.n_fixups;
  if (int rc = ts_replay_batch(g, &sc, &res, nullptr)) {
    const std::string msg = ts_last_error();
    if (rc == TS_E_INVALID_ARGUMENT && msg.rfind("utilization needs ", 0) == 0)
      throw std::invalid_argument(msg);
    rethrow(rc, retime);
  }
  return r;
}

}  // namespace

BatchResult simulate_batch(const ExecutionGraph& graph, const ScenarioSpec& spec,
                           const BatchOptions& o) {
  for (const ValidationIssue& issue : validate_graph(graph))
    if (issue.error) throw SimulationError("invalid graph: " + issue.message);
  Handle h(graph);
  if (o.util_bin_width > 0 && o.util_max_bins <= 0) {
    // every bin: try the recorded window, then the count the engine reports
    const Micros span = graph.iteration_window.end - graph.iteration_window.start;
    const int32_t guess =
        static_cast<int32_t>(std::max<Micros>(1, (span + o.util_bin_width - 1) / o.util_bin_width));
    try {
      return run_batch(h.g, graph.tasks.size(), spec, o, guess);
    } catch (const std::invalid_argument& e) {
      const std::string m = e.what();
      if (m.rfind("utilization needs ", 0) != 0) throw;
      return run_batch(h.g, graph.tasks.size(), spec, o,
                       static_cast<int32_t>(std::stol(m.substr(18))));
    }
  }
  return run_batch(h.g, graph.tasks.size(), spec, o, o.util_max_bins);
}

std::map<int, UtilizationSeries> utilization_by_rank(const BatchResult& r, std::size_t s,
                                                     IterationWindow window) {
  std::map<int, UtilizationSeries> out;
  if (r.util_bin_width <= 0) throw std::invalid_argument("bin_width must be positive");
  window.end = std::max(window.end, window.start + r.span[3 * s + 2]);
  if (window.end <= window.start) return out;  // metrics.cpp:108
  const std::size_t kept = std::min<std::size_t>(r.util_n_bins[s], r.util_max_bins);
  for (std::size_t k = 0; k < r.ranks.size(); ++k) {
    UtilizationSeries series;
    series.bin_width = r.util_bin_width;
    const int64_t* row =
        r.util_covered.data() + (s * r.ranks.size() + k) * static_cast<std::size_t>(r.util_max_bins);
    for (std::size_t i = 0; i < kept; ++i) {
      const Micros bin_start = window.start + static_cast<Micros>(i) * r.util_bin_width;
      const Micros span = std::min(r.util_bin_width, window.end - bin_start);
      series.bins.push_back({bin_start, static_cast<double>(row[i]) / span});
    }
    out[r.ranks[k]] = std::move(series);
  }
  return out;
}

ReplayReport replay_report(const ExecutionGraph& graph, const BatchResult& r, std::size_t s) {
  ReplayReport rep;
  Micros lo = std::numeric_limits<Micros>::max(), hi = std::numeric_limits<Micros>::min();
  for (const Task& t : graph.tasks) {
    lo = std::min(lo, t.original_start);
    hi = std::max(hi, t.original_start + t.duration);
  }
  rep.reference_makespan = graph.tasks.empty() ? 0 : hi - lo;
  rep.simulated_makespan = r.span[3 * s + 2];
  rep.relative_error =
      relative_error(rep.reference_makespan, rep.simulated_makespan, &rep.zero_reference);
  const std::size_t n = graph.tasks.size();
  if (r.worst_n < 1 || s >= r.delta_abs_sum.size() ||
      (s + 1) * static_cast<std::size_t>(r.worst_n) * 3 > r.delta_worst.size())
    throw std::invalid_argument("replay_report needs a batch run with BatchOptions::deltas");
  rep.mean_abs_delta = n ? static_cast<double>(r.delta_abs_sum[s]) / static_cast<double>(n) : 0.0;
  const std::size_t wn = static_cast<std::size_t>(r.worst_n);
  const int64_t* w = r.delta_worst.data() + s * wn * 3;
  rep.max_abs_delta = w[0];
  for (std::size_t k = 0; k < wn && w[3 * k + 1] >= 0; ++k) {
    const TaskId task = static_cast<TaskId>(w[3 * k + 1]);
    const Micros rs = graph.tasks[static_cast<std::size_t>(task)].original_start;
    rep.worst.push_back({task, rs, rs + w[3 * k + 2], w[3 * k + 2]});
  }
  return rep;
}

namespace {

// tracesim::PipelineSpec -> ts_pipeline_spec (pointers into `spec` and into
// this object's arrays)
struct PipelinePod {
  std::vector<std::vector<const char*>> keys, values;
  std::vector<std::vector<ts_kernel_spec>> kernels;
  std::vector<std::vector<ts_kernel_list>> layer_lists;
  std::vector<ts_stage_spec> stages;
  ts_pipeline_spec c{};

  ts_kernel_list list(const std::vector<KernelSpec>& ks) {
    std::vector<ts_kernel_spec> v;
    for (const KernelSpec& k : ks) {
      keys.emplace_back();
      values.emplace_back();
      for (const auto& [a, b] : k.args) {
        keys.back().push_back(a.c_str());
        values.back().push_back(b.c_str());
      }
      ts_kernel_spec x{};
      x.name = k.name.c_str();
      x.duration = k.duration;
      x.op_class = static_cast<int32_t>(k.op_class);
      x.n_args = static_cast<int32_t>(k.args.size());
      x.arg_keys = keys.back().data();
      x.arg_values = values.back().data();
      v.push_back(x);
    }
    kernels.push_back(std::move(v));
    return ts_kernel_list{kernels.back().data(), static_cast<int32_t>(ks.size()), 0};
  }

  explicit PipelinePod(const PipelineSpec& p) {
    std::size_t n_lists = 0, n_kernels = 0;
    for (const StageSpec& st : p.stages) {
      n_lists += st.layers_fwd.size() + st.layers_bwd.size() + 6;
      for (const auto& l : st.layers_fwd) n_kernels += l.size();
      for (const auto& l : st.layers_bwd) n_kernels += l.size();
      n_kernels += st.pre_fwd.size() + st.post_fwd.size() + st.pre_bwd.size() +
                   st.post_bwd.size() + st.reduce.size() + st.optimizer.size();
    }
    kernels.reserve(n_lists);  // no reallocation: lists point into these
    keys.reserve(n_kernels);
    values.reserve(n_kernels);
    layer_lists.reserve(2 * p.stages.size());
    for (const StageSpec& st : p.stages) {
      if (st.layers_fwd.size() != st.layers_bwd.size())
        throw std::invalid_argument("pipeline: layers_fwd and layers_bwd differ in length");
      ts_stage_spec cs{};
      cs.n_layers = static_cast<int32_t>(st.layers_fwd.size());
      layer_lists.emplace_back();
      for (const auto& l : st.layers_fwd) layer_lists.back().push_back(list(l));
      cs.layers_fwd = layer_lists.back().data();
      layer_lists.emplace_back();
      for (const auto& l : st.layers_bwd) layer_lists.back().push_back(list(l));
      cs.layers_bwd = layer_lists.back().data();
      cs.pre_fwd = list(st.pre_fwd);
      cs.post_fwd = list(st.post_fwd);
      cs.pre_bwd = list(st.pre_bwd);
      cs.post_bwd = list(st.post_bwd);
      cs.reduce = list(st.reduce);
      cs.optimizer = list(st.optimizer);
      stages.push_back(cs);
    }
    c.pp = p.pp;
    c.dp = p.dp;
    c.num_microbatches = p.num_microbatches;
    c.n_stages = static_cast<int32_t>(stages.size());
    c.stages = stages.data();
    c.launch_us = p.host.launch;
    c.record_us = p.host.record;
    c.wait_us = p.host.wait;
    c.sync_us = p.host.sync;
    c.p2p_send_us = p.p2p_send;
    c.p2p_recv_base_us = p.p2p_recv_base;
    c.activation_bytes = p.activation_bytes;
    c.origin = p.origin;
    c.compute_stream = p.compute_stream;
    c.reduce_stream = p.reduce_stream;
    c.p2p_stream = p.p2p_stream;
    c.main_thread = p.main_thread;
    c.helper_thread = p.helper_thread;
    c.first_event = p.first_event;
    c.first_correlation = p.first_correlation;
  }
};

}  // namespace

namespace {

// the estimate graph of a ts_pipeline_spec replayed for `scenarios`
EstimateResult estimate_pod(const ts_pipeline_spec& spec, const ScenarioSpec& scenarios,
                            const BatchOptions& options, int tp) {
  if (!scenarios.alpha_us.empty())
    throw std::invalid_argument(
        "estimate_batch: retime the PipelineSpec itself (rebuild_pipeline) instead of per scenario");
  ts_host_graph* hg = nullptr;
  EstimateResult out;
  if (int rc = ts_pipeline_graph(&spec, 1, tp, &hg, &out.truth_makespan)) {
    const std::string msg = ts_last_error();
    if (rc == TS_E_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    rethrow(rc);
  }
  struct Free {
    ts_host_graph* h;
    ~Free() { ts_host_graph_free(h); }
  } free_hg{hg};
  ts_graph_desc desc{};
  ts_host_graph_desc(hg, &desc);
  const std::size_t n = static_cast<std::size_t>(desc.n_tasks);
  out.op_index.resize(n);
  ts_host_graph_op_index(hg, out.op_index.data());
  out.n_ops = ts_host_graph_n_ops(hg);
  out.base.assign(desc.duration, desc.duration + n);
  out.rank.assign(desc.rank, desc.rank + n);
  ts_graph* g = nullptr;
  if (int rc = ts_graph_create(&desc, -1, &g)) rethrow(rc);
  struct Destroy {
    ts_graph* g;
    ~Destroy() { ts_graph_destroy(g); }
  } destroy{g};
  BatchOptions o = options;
  o.util_bin_width = 0;  // the reductions of an estimate graph are not defined here
  o.deltas = false;
  out.batch = run_batch(g, n, scenarios, o, 0);
  return out;
}

std::vector<KernelSpec> kernels_of(const ts_kernel_list& l) {
  std::vector<KernelSpec> out;
  for (int32_t i = 0; i < l.n; ++i) {
    const ts_kernel_spec& k = l.k[i];
    KernelSpec ks;
    ks.name = k.name ? k.name : "";
    ks.duration = k.duration;
    ks.op_class = static_cast<OpClass>(k.op_class);
    for (int32_t a = 0; a < k.n_args; ++a) ks.args[k.arg_keys[a]] = k.arg_values[a];
    out.push_back(std::move(ks));
  }
  return out;
}

PipelineSpec spec_of(const ts_pipeline_spec& c) {
  PipelineSpec p;
  p.pp = c.pp;
  p.dp = c.dp;
  p.num_microbatches = c.num_microbatches;
  p.host = {c.launch_us, c.record_us, c.wait_us, c.sync_us};
  p.p2p_send = c.p2p_send_us;
  p.p2p_recv_base = c.p2p_recv_base_us;
  p.activation_bytes = c.activation_bytes;
  p.origin = c.origin;
  p.compute_stream = c.compute_stream;
  p.reduce_stream = c.reduce_stream;
  p.p2p_stream = c.p2p_stream;
  p.main_thread = c.main_thread;
  p.helper_thread = c.helper_thread;
  p.first_event = c.first_event;
  p.first_correlation = c.first_correlation;
  for (int32_t s = 0; s < c.n_stages; ++s) {
    const ts_stage_spec& cs = c.stages[s];
    StageSpec st;
    for (int32_t l = 0; l < cs.n_layers; ++l) {
      st.layers_fwd.push_back(kernels_of(cs.layers_fwd[l]));
      st.layers_bwd.push_back(kernels_of(cs.layers_bwd[l]));
    }
    st.pre_fwd = kernels_of(cs.pre_fwd);
    st.post_fwd = kernels_of(cs.post_fwd);
    st.pre_bwd = kernels_of(cs.pre_bwd);
    st.post_bwd = kernels_of(cs.post_bwd);
    st.reduce = kernels_of(cs.reduce);
    st.optimizer = kernels_of(cs.optimizer);
    p.stages.push_back(std::move(st));
  }
  return p;
}

}  // namespace

EstimateResult estimate_batch(const PipelineSpec& spec, const ScenarioSpec& scenarios,
                              const BatchOptions& options, int tp) {
  PipelinePod pod(spec);
  return estimate_pod(pod.c, scenarios, options, tp);
}

WhatIfEstimate estimate_whatif(const ExecutionGraph& source, const WhatIfConfig& cfg,
                               const ScenarioSpec& scenarios, const BatchOptions& options,
                               int tp) {
  const auto* am = dynamic_cast<const AnalyticalCostModel*>(cfg.cost_model.get());
  if (!cfg.cost_model) throw TransformError("what-if config has no cost model");
  if (!am) throw TransformError("estimate_whatif: the device rebuild takes an AnalyticalCostModel");
  // the source graph with its Task.meta and correlation ids
  Soa soa(source);
  const std::size_t n = source.tasks.size();
  std::vector<const char*> names(n), mk, mv;
  std::vector<int64_t> corr(n, -1);
  std::vector<int32_t> moff(n + 1, 0);
  for (std::size_t i = 0; i < n; ++i) {
    const Task& t = source.tasks[i];
    names[i] = t.name.c_str();
    if (t.correlation_id) corr[i] = *t.correlation_id;
    for (const auto& [k, v] : t.meta) {
      mk.push_back(k.c_str());
      mv.push_back(v.c_str());
    }
    moff[i + 1] = static_cast<int32_t>(mk.size());
  }
  ts_host_graph* hg = nullptr;
  if (int rc = ts_host_graph_from_tasks(&soa.desc, names.data(), corr.data(), moff.data(),
                                        mk.data(), mv.data(), &hg))
    rethrow(rc);
  struct Free {
    ts_host_graph* h;
    ~Free() { ts_host_graph_free(h); }
  } free_hg{hg};
  auto model = [](const ModelConfig& m) {
    ts_model_config c{};
    c.n_params = m.n_params;
    c.n_layers = m.n_layers;
    c.d_model = m.d_model;
    c.d_ffn = m.d_ffn;
    c.n_heads = m.n_heads;
    c.d_head = m.d_head;
    return c;
  };
  auto par = [](const ParallelismConfig& p) {
    return ts_par_config{p.tp, p.pp, p.dp, p.num_microbatches};
  };
  ts_whatif w{};
  w.source_model = model(cfg.source_model);
  w.target_model = model(cfg.target_model);
  w.source_par = par(cfg.source_par);
  w.target_par = par(cfg.target_par);
  w.alpha_us = am->alpha_us();
  w.bytes_per_us = am->bytes_per_us();
  w.activation_bytes = cfg.activation_bytes;
  ts_pipeline* p = nullptr;
  if (int rc = ts_rebuild_pipeline(hg, &w, &p)) {
    if (rc == TS_E_INVALID_ARGUMENT) throw TransformError(ts_last_error());
    rethrow(rc);
  }
  WhatIfEstimate out;
  if (!p) return out;  // nothing the rebuild models changes: replay the source instead
  struct FreeP {
    ts_pipeline* p;
    ~FreeP() { ts_pipeline_free(p); }
  } free_p{p};
  const ts_pipeline_spec* c = ts_pipeline_spec_get(p);
  out.spec = spec_of(*c);
  static_cast<EstimateResult&>(out) = estimate_pod(*c, scenarios, options, tp);
  out.rebuilt = true;
  return out;
}

SimulatedTrace scenario_trace(const ExecutionGraph& graph, const BatchResult& r, std::size_t s) {
  const std::size_t S = r.span.size() / 3, n = graph.tasks.size();
  if (r.start.size() != n * S || r.fin.size() != n * S || s >= S)
    throw std::invalid_argument("scenario_trace needs a batch run with timestamps");
  SimulatedTrace out;
  out.entries.reserve(n);
  for (std::size_t i = 0; i < n; ++i)
    out.entries.push_back({static_cast<TaskId>(i), r.start[i * S + s], r.fin[i * S + s],
                           graph.tasks[i].processor});
  std::sort(out.entries.begin(), out.entries.end(), [](const SimEntry& a, const SimEntry& b) {
    return std::pair(a.sim_start, a.task_id) < std::pair(b.sim_start, b.task_id);
  });
  out.start = r.span[3 * s];
  out.end = r.span[3 * s + 1];
  out.makespan = r.span[3 * s + 2];
  return out;
}

std::vector<SimulatedTrace> replay_scenarios(const ExecutionGraph& graph, const ScenarioSpec& spec,
                                             const std::vector<int64_t>& ids) {
  for (const ValidationIssue& issue : validate_graph(graph))
    if (issue.error) throw SimulationError("invalid graph: " + issue.message);
  Handle h(graph);
  const std::size_t n = graph.tasks.size();
  std::vector<SimulatedTrace> out;
  std::vector<int64_t> start(n), fin(n), span(3);
  for (int64_t id : ids) {
    ts_scenarios sc{};
    sc.first = id;
    sc.count = 1;
    sc.seed = spec.seed;
    sc.jitter = spec.jitter;
    sc.scale_lo = spec.scale_lo;
    sc.scale_hi = spec.scale_hi;
    sc.scale_den = spec.scale_den;
    ts_retime rt{};
    const bool retime = !spec.alpha_us.empty();
    if (retime) {  // per-scenario retime arrays are indexed from spec.first
      const std::size_t k = static_cast<std::size_t>(id - spec.first);
      if (id < spec.first || k >= spec.alpha_us.size() || k >= spec.bytes_per_us.size() ||
          (!spec.target_dp.empty() && k >= spec.target_dp.size()) ||
          (!spec.target_model.empty() && 3 * k + 2 >= spec.target_model.size()))
        throw std::invalid_argument("scenario id outside the retime arrays");
      rt.alpha_us = &spec.alpha_us[k];
      rt.bytes_per_us = &spec.bytes_per_us[k];
      rt.source_dp = spec.source_dp;
      rt.target_dp = spec.target_dp.empty() ? nullptr : &spec.target_dp[k];
      for (int j = 0; j < 3; ++j) rt.source_model[j] = spec.source_model[j];
      rt.target_model = spec.target_model.empty() ? nullptr : &spec.target_model[3 * k];
      sc.retime = &rt;
    }
    ts_result res{};
    res.start = start.data();
    res.fin = fin.data();
    res.ld = 1;
    res.span = span.data();
    if (int rc = ts_replay_batch(h.g, &sc, &res, nullptr)) rethrow(rc, retime);
    BatchResult one;
    one.start = start;
    one.fin = fin;
    one.span = span;
    out.push_back(scenario_trace(graph, one, 0));
  }
  return out;
}

}  // namespace b200

}  // namespace tracesim
