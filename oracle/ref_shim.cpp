// ref_shim.cpp — extern "C" driver for the compiled, unmodified reference.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources (/root/reference/proj/src/*.cpp, tests/oracles.cpp) under
// -Dtracesim=tracesim_ref, producing oracle/_ref/libtracesim_ref.so.  Python
// tests (tests/refshim.py) and bench.py's cpu_baseline / --impl reference legs
// load it with ctypes.  Nothing in paper_2504_09307_b200/ links it.
//
// Every function is a thin adaptor over the reference's public C++ API:
//   generate / split_by_rank      (src/synth.cpp:140-176)
//   build_graph / merge_ranks     (src/build.cpp:338-542)
//   parse_trace                   (src/trace_parse.cpp:213-228)
//   simulate                      (src/simulate.cpp:341-347)
//   oracle::tick_simulate         (tests/oracles.cpp:11-113)
//   oracle::random_graph          (tests/oracles.cpp:222-295)
//   breakdown_by_rank             (src/metrics.cpp:96-103)
//   build_pipeline + DurationHook (src/pipeline.cpp:474-477)

#include <algorithm>
#include <chrono>
#include <limits>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <cstring>
#include <fstream>
#include <map>
#include <cctype>
#include <sstream>
#include <optional>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "oracles.hpp"
#include "tracesim/build.hpp"
#include "tracesim/cost.hpp"
#include "tracesim/metrics.hpp"
#include "tracesim/pipeline.hpp"
#include "tracesim/simulate.hpp"
#include "tracesim/synth.hpp"
#include "tracesim/trace_parse.hpp"
#include "tracesim/transform.hpp"

#include "lumos_oracle.h"

using namespace tracesim;

namespace {

thread_local std::string g_err;

void set_err(const char* what) { g_err = what; }

struct RefGraph {
  ExecutionGraph g;
};

ExecutionGraph relabel_rank(const ExecutionGraph& src, int new_rank) {
  ExecutionGraph g = src;
  g.processors.clear();
  for (auto& t : g.tasks) {
    t.processor.rank = new_rank;
    g.processors.insert(t.processor);
  }
  for (auto& r : g.rules)
    for (auto& p : r.watched) p.rank = new_rank;
  return g;
}

ExecutionGraph graph_of_events(const std::vector<TraceEvent>& events, int tp) {
  std::map<int, ExecutionGraph> parts;
  for (const auto& [rank, evs] : split_by_rank(events)) {
    ExecutionGraph g = build_graph(evs, BuildPolicy(), rank);
    if (tp <= 1) {
      parts[rank] = std::move(g);
    } else {
      for (int t = 0; t < tp; ++t) parts[rank * tp + t] = relabel_rank(g, rank * tp + t);
    }
  }
  return merge_ranks(parts);
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const SimulationError& e) {
    set_err(e.what());
    return 3;
  } catch (const GraphError& e) {
    set_err(e.what());
    return 4;
  } catch (const std::exception& e) {
    set_err(e.what());
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- graphs

// generate(spec) -> per-rank build_graph -> (tp replicas) -> merge_ranks; then
// optionally slice_rank.  Also returns the generator's truth makespan.
void* ref_graph_generate(const char* spec_json, int tp, int slice, int64_t* truth_makespan) {
  RefGraph* out = nullptr;
  int rc = guarded([&] {
    SynthSpec spec = SynthSpec::from_json(spec_json);
    SynthResult res = generate(spec);
    if (truth_makespan) *truth_makespan = res.truth.iterations.at(0).makespan;
    out = new RefGraph;
    out->g = graph_of_events(res.events, tp);
    if (slice >= 0) out->g = slice_rank(out->g, slice);
    return 0;
  });
  if (rc != 0) {
    delete out;
    return nullptr;
  }
  return out;
}

// parse_trace(json) -> build_graph (one rank)
void* ref_graph_from_trace(const char* trace_json, int rank_override) {
  RefGraph* out = nullptr;
  int rc = guarded([&] {
    auto events = parse_trace(std::string(trace_json));
    out = new RefGraph;
    out->g = rank_override >= 0 ? build_graph(events, BuildPolicy(), rank_override)
                                : build_graph(events, BuildPolicy());
    return 0;
  });
  if (rc != 0) {
    delete out;
    return nullptr;
  }
  return out;
}

void* ref_graph_from_arrays(int32_t n, const int64_t* dur, const int64_t* ostart,
                            const int32_t* rank, const int32_t* kind, const int32_t* lane,
                            const uint8_t* op_class, int64_t ne, const int32_t* ef,
                            const int32_t* et, int32_t nr, const int32_t* rkind,
                            const int32_t* rtask, const int32_t* rbound, const int32_t* rwoff,
                            const int32_t* wrank, const int32_t* wkind, const int32_t* wlane,
                            int64_t wstart, int64_t wend) {
  auto* out = new RefGraph;
  ExecutionGraph& g = out->g;
  g.tasks.resize(static_cast<std::size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    Task& t = g.tasks[i];
    t.id = i;
    t.kind = kind[i] == 1 ? TaskKind::Gpu : TaskKind::Cpu;
    t.op_class = static_cast<OpClass>(op_class ? op_class[i] : 6);
    t.name = "t" + std::to_string(i);
    t.duration = dur[i];
    t.original_start = ostart[i];
    t.processor = {rank[i], kind[i] == 1 ? LaneKind::CudaStream : LaneKind::CpuThread, lane[i]};
    g.processors.insert(t.processor);
  }
  for (int64_t e = 0; e < ne; ++e) g.fixed_edges.emplace_back(ef[e], et[e]);
  for (int32_t r = 0; r < nr; ++r) {
    RuntimeRule rule;
    rule.kind = static_cast<RuntimeRule::Kind>(rkind[r]);
    rule.waiting_task = rtask[r];
    if (rbound[r] >= 0) rule.bound_task = rbound[r];
    if (rule.kind == RuntimeRule::Kind::EventSync) rule.event_id = r;
    for (int32_t w = rwoff[r]; w < rwoff[r + 1]; ++w)
      rule.watched.push_back(
          {wrank[w], wkind[w] == 1 ? LaneKind::CudaStream : LaneKind::CpuThread, wlane[w]});
    g.rules.push_back(std::move(rule));
  }
  g.iteration_window = {wstart, wend};
  return out;
}

void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* rng) { delete static_cast<std::mt19937_64*>(rng); }

void* ref_graph_random(void* rng, int max_tasks, int max_lanes) {
  auto* out = new RefGraph;
  out->g = oracle::random_graph(*static_cast<std::mt19937_64*>(rng), max_tasks, max_lanes);
  return out;
}

void ref_graph_free(void* h) { delete static_cast<RefGraph*>(h); }

// sizes = {tasks, edges, rules, watched entries, window.start, window.end}
void ref_graph_sizes(void* h, int64_t* sizes) {
  const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
  int64_t nw = 0;
  for (const auto& r : g.rules) nw += static_cast<int64_t>(r.watched.size());
  sizes[0] = static_cast<int64_t>(g.tasks.size());
  sizes[1] = static_cast<int64_t>(g.fixed_edges.size());
  sizes[2] = static_cast<int64_t>(g.rules.size());
  sizes[3] = nw;
  sizes[4] = g.iteration_window.start;
  sizes[5] = g.iteration_window.end;
}

void ref_graph_export(void* h, int64_t* dur, int64_t* ostart, int32_t* rank, int32_t* kind,
                      int32_t* lane, uint8_t* op_class, uint8_t* task_kind, int32_t* ef,
                      int32_t* et, int32_t* rkind, int32_t* rtask, int32_t* rbound,
                      int32_t* rwoff, int32_t* wrank, int32_t* wkind, int32_t* wlane) {
  const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
  for (std::size_t i = 0; i < g.tasks.size(); ++i) {
    const Task& t = g.tasks[i];
    dur[i] = t.duration;
    ostart[i] = t.original_start;
    rank[i] = t.processor.rank;
    kind[i] = t.processor.kind == LaneKind::CudaStream ? 1 : 0;
    lane[i] = t.processor.lane;
    op_class[i] = static_cast<uint8_t>(t.op_class);
    task_kind[i] = t.kind == TaskKind::Gpu ? 1 : 0;
  }
  for (std::size_t e = 0; e < g.fixed_edges.size(); ++e) {
    ef[e] = g.fixed_edges[e].first;
    et[e] = g.fixed_edges[e].second;
  }
  int32_t w = 0;
  rwoff[0] = 0;
  for (std::size_t r = 0; r < g.rules.size(); ++r) {
    const RuntimeRule& rule = g.rules[r];
    rkind[r] = static_cast<int32_t>(rule.kind);
    rtask[r] = rule.waiting_task;
    rbound[r] = rule.bound_task ? *rule.bound_task : -1;
    for (const auto& p : rule.watched) {
      wrank[w] = p.rank;
      wkind[w] = p.kind == LaneKind::CudaStream ? 1 : 0;
      wlane[w] = p.lane;
      ++w;
    }
    rwoff[r + 1] = w;
  }
}

// task names, '\n'-separated, into buf (returns bytes needed)
int64_t ref_graph_names(void* h, char* buf, int64_t cap) {
  const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
  std::string all;
  for (const auto& t : g.tasks) {
    all += t.name;
    all += '\n';
  }
  if (buf && cap >= static_cast<int64_t>(all.size())) std::memcpy(buf, all.data(), all.size());
  return static_cast<int64_t>(all.size());
}

// ---------------------------------------------------------------- replay

static int run_sim(void* h, const int64_t* dur, int64_t* start, int64_t* fin, int64_t* span,
                   bool tick) {
  return guarded([&] {
    const ExecutionGraph& src = static_cast<RefGraph*>(h)->g;
    const ExecutionGraph* gp = &src;
    ExecutionGraph copy;
    if (dur) {
      copy = src;
      for (std::size_t i = 0; i < copy.tasks.size(); ++i) copy.tasks[i].duration = dur[i];
      gp = &copy;
    }
    SimulatedTrace sim = tick ? oracle::tick_simulate(*gp) : simulate(*gp);
    for (const auto& e : sim.entries) {
      start[e.task_id] = e.sim_start;
      fin[e.task_id] = e.sim_end;
    }
    span[0] = sim.start;
    span[1] = sim.end;
    span[2] = sim.makespan;
    return 0;
  });
}

int ref_simulate(void* h, const int64_t* dur, int64_t* start, int64_t* fin, int64_t* span) {
  return run_sim(h, dur, start, fin, span, false);
}

int ref_tick_simulate(void* h, const int64_t* dur, int64_t* start, int64_t* fin,
                      int64_t* span) {
  return run_sim(h, dur, start, fin, span, true);
}

// breakdown_by_rank over the simulated intervals; out is [max_ranks][6] =
// {rank, total, exposed_compute, exposed_comm, overlapped, other}
int ref_breakdown_by_rank(void* h, const int64_t* start, const int64_t* fin, int64_t wstart,
                          int64_t wend, int64_t* out, int max_ranks) {
  const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
  SimulatedTrace sim;
  for (std::size_t i = 0; i < g.tasks.size(); ++i)
    sim.entries.push_back({static_cast<TaskId>(i), start[i], fin[i], g.tasks[i].processor});
  auto by_rank = breakdown_by_rank(task_intervals(g, &sim), IterationWindow{wstart, wend});
  int k = 0;
  for (const auto& [rank, b] : by_rank) {
    if (k >= max_ranks) break;
    int64_t* row = out + 6 * k;
    row[0] = rank;
    row[1] = b.total;
    row[2] = b.exposed_compute;
    row[3] = b.exposed_comm;
    row[4] = b.overlapped;
    row[5] = b.other;
    ++k;
  }
  return k;
}

// utilization_by_rank (metrics.cpp:105-155) over the simulated intervals:
// values[k][b] (double) for the k-th rank (ascending), ranks[k], n_bins[k].
int ref_utilization_by_rank(void* h, const int64_t* start, const int64_t* fin, int64_t wstart,
                            int64_t wend, int64_t bin_width, double* values, int32_t* ranks,
                            int32_t* n_bins, int max_ranks, int max_bins) {
  const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
  SimulatedTrace sim;
  for (std::size_t i = 0; i < g.tasks.size(); ++i)
    sim.entries.push_back({static_cast<TaskId>(i), start[i], fin[i], g.tasks[i].processor});
  auto util = utilization_by_rank(task_intervals(g, &sim), IterationWindow{wstart, wend}, bin_width);
  int k = 0;
  for (const auto& [rank, series] : util) {
    if (k >= max_ranks) break;
    ranks[k] = rank;
    n_bins[k] = static_cast<int32_t>(series.bins.size());
    for (std::size_t b = 0; b < series.bins.size() && static_cast<int>(b) < max_bins; ++b)
      values[static_cast<std::size_t>(k) * max_bins + b] = series.bins[b].value;
    ++k;
  }
  return k;
}

// compare_replay (metrics.cpp:189-221) of one replay given as per-task
// start/fin: out_i = {reference_makespan, simulated_makespan, max_abs_delta,
// zero_reference, n_worst, worst task ids..., worst deltas...}, out_d =
// {mean_abs_delta, relative_error}.  Entries are ordered (sim_start, id) as
// simulate() emits them (simulate.cpp:320-326).
int ref_compare_replay(void* h, const int64_t* start, const int64_t* fin, int32_t worst_n,
                       int64_t* out_i, double* out_d) {
  const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
  SimulatedTrace sim;
  for (std::size_t i = 0; i < g.tasks.size(); ++i)
    sim.entries.push_back({static_cast<TaskId>(i), start[i], fin[i], g.tasks[i].processor});
  std::sort(sim.entries.begin(), sim.entries.end(), [](const SimEntry& a, const SimEntry& b) {
    return std::pair(a.sim_start, a.task_id) < std::pair(b.sim_start, b.task_id);
  });
  if (!sim.entries.empty()) {
    sim.start = std::numeric_limits<Micros>::max();
    sim.end = std::numeric_limits<Micros>::min();
    for (const auto& e : sim.entries) {
      sim.start = std::min(sim.start, e.sim_start);
      sim.end = std::max(sim.end, e.sim_end);
    }
    sim.makespan = sim.end - sim.start;
  }
  ReplayReport rep = compare_replay(g, sim, static_cast<std::size_t>(worst_n));
  out_i[0] = rep.reference_makespan;
  out_i[1] = rep.simulated_makespan;
  out_i[2] = rep.max_abs_delta;
  out_i[3] = rep.zero_reference ? 1 : 0;
  out_i[4] = static_cast<int64_t>(rep.worst.size());
  for (std::size_t k = 0; k < rep.worst.size(); ++k) {
    out_i[5 + k] = rep.worst[k].task;
    out_i[5 + worst_n + k] = rep.worst[k].delta;
  }
  out_d[0] = rep.mean_abs_delta;
  out_d[1] = rep.relative_error;
  return 0;
}

// ------------------------------------------------------ CPU baseline timing

// Times the reference simulate() over `count` scenarios whose durations come
// from the oracle's scenario formula (lumos_oracle.c), one scenario per call,
// on `threads` host threads (each with its own graph copy).  The durations of
// every scenario are materialised before the clock starts (their fill time is
// returned in *fill_seconds), so the returned wall seconds cover the parallel
// simulate() region only.  makespans[i] receives scenario i's
// makespan.
double ref_bench_simulate(void* h, const orc_scenarios* sc, int64_t first, int32_t count,
                          const uint8_t* cls, int threads, int64_t* makespans,
                          double* fill_seconds) {
  const ExecutionGraph& src = static_cast<RefGraph*>(h)->g;
  if (threads < 1) threads = 1;
  const std::size_t n = src.tasks.size();
  std::vector<ExecutionGraph> copies(static_cast<std::size_t>(threads), src);
  std::vector<int64_t> base(n);
  for (std::size_t i = 0; i < n; ++i) base[i] = src.tasks[i].duration;
  std::vector<std::vector<int64_t>> dur(static_cast<std::size_t>(count), std::vector<int64_t>(n));
  auto f0 = std::chrono::steady_clock::now();
  {
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
      pool.emplace_back([&, w] {
        for (int32_t s = w; s < count; s += threads)
          orc_fill_durations(sc, first + s, static_cast<int32_t>(n), base.data(), cls,
                             dur[static_cast<std::size_t>(s)].data());
      });
    for (auto& t : pool) t.join();
  }
  if (fill_seconds)
    *fill_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - f0).count();
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) {
    pool.emplace_back([&, w] {
      ExecutionGraph& g = copies[static_cast<std::size_t>(w)];
      for (int32_t s = w; s < count; s += threads) {
        const std::vector<int64_t>& d = dur[static_cast<std::size_t>(s)];
        for (std::size_t i = 0; i < n; ++i) g.tasks[i].duration = d[i];
        try {
          makespans[s] = simulate(g).makespan;
        } catch (const std::exception&) {
          makespans[s] = -1;
        }
      }
    });
  }
  for (auto& t : pool) t.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}


// ------------------------------------------------------------ trace ingest
// Writes the reference generator's trace (generate(spec).events) as Chrome
// JSON, one file per rank: <dir>/rank_<r>.json (chrome_json,
// trace_parse.cpp:230-256).  Returns the number of files or -1.
int ref_write_rank_traces(const char* spec_json, const char* dir) {
  try {
    SynthResult res = generate(SynthSpec::from_json(spec_json));
    int k = 0;
    for (const auto& [rank, evs] : split_by_rank(res.events)) {
      std::ofstream out(std::string(dir) + "/rank_" + std::to_string(rank) + ".json");
      out << chrome_json(evs);
      ++k;
    }
    return k;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The reference's own input path with default options (cli.cpp:93-137,
// window "full"): load_multirank of rank_<N> files, build_graph per rank,
// merge_ranks.  Returns a handle or NULL (message in ref_last_error()).
void* ref_ingest_traces(const char* const* paths, int n) {
  try {
    // load_multirank (trace_parse.cpp:286-296) with the file read into a
    // string first and the rank_<N> marker scanned by hand: the same events
    // and ranks, without std::regex / istream parsing, which crash in a
    // process that has numpy's bundled runtime loaded
    CategoryTable cats;
    std::map<int, ExecutionGraph> graphs;
    for (int i = 0; i < n; ++i) {
      const std::string path = paths[i];
      int rank = -1;
      for (std::size_t p = path.find("rank"); p != std::string::npos; p = path.find("rank", p + 1)) {
        std::size_t q = p + 4;
        if (q < path.size() && path[q] == '_') ++q;
        std::size_t e = q;
        while (e < path.size() && std::isdigit(static_cast<unsigned char>(path[e]))) ++e;
        if (e > q) rank = std::stoi(path.substr(q, e - q));
      }
      if (rank < 0) throw std::runtime_error("cannot derive a rank from filename '" + path + "'");
      std::ifstream in(path, std::ios::binary);
      std::stringstream ss;
      ss << in.rdbuf();
      if (graphs.count(rank)) throw std::runtime_error("duplicate rank " + std::to_string(rank));
      graphs.emplace(rank, build_graph(parse_trace(ss.str(), cats), BuildPolicy(), rank));
    }
    auto* r = new RefGraph;
    r->g = merge_ranks(graphs);
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// The reference's build_from_inputs (cli.cpp:118-137) with every option:
// manifest (rank -> path, relative to the manifest's directory), window
// ("full" | "auto" | START:END), custom category table and build policy (JSON
// texts).  load_inputs (cli.cpp:93-116) is restated with the files read into
// strings (see ref_ingest_traces); the rank files are the inputs whose file
// name carries a rank_<N> marker.  Returns a handle or NULL.
void* ref_ingest_traces_ex(const char* const* paths, int n, const char* manifest,
                           const char* window, const char* categories_json,
                           const char* policy_json) {
  try {
    const CategoryTable cats = categories_json ? CategoryTable::from_json(categories_json)
                                               : CategoryTable();
    const BuildPolicy policy = policy_json ? BuildPolicy::from_json(policy_json) : BuildPolicy();
    auto slurp = [](const std::string& path) {
      std::ifstream in(path, std::ios::binary);
      if (!in) throw ParseError("cannot open trace file '" + path + "'");
      std::stringstream ss;
      ss << in.rdbuf();
      return ss.str();
    };
    auto marker = [](const std::string& text, int& rank) {
      bool found = false;
      for (std::size_t p = text.find("rank"); p != std::string::npos; p = text.find("rank", p + 1)) {
        std::size_t q = p + 4;
        if (q < text.size() && text[q] == '_') ++q;
        std::size_t e = q;
        while (e < text.size() && std::isdigit(static_cast<unsigned char>(text[e]))) ++e;
        if (e > q) {
          rank = std::stoi(text.substr(q, e - q));
          found = true;
        }
      }
      return found;
    };
    std::map<int, std::vector<TraceEvent>> per_rank;
    auto take = [&](int rank, std::vector<TraceEvent> evs) {
      if (!per_rank.emplace(rank, std::move(evs)).second)
        throw ParseError("rank " + std::to_string(rank) + " appears in more than one input");
    };
    if (manifest && *manifest) {
      const std::string mp = manifest;
      nlohmann::json root = nlohmann::json::parse(slurp(mp));
      std::string dir;
      if (auto slash = mp.find_last_of('/'); slash != std::string::npos) dir = mp.substr(0, slash + 1);
      for (auto it = root.begin(); it != root.end(); ++it) {
        std::string path = it.value().get<std::string>();
        if (!path.empty() && path[0] != '/') path = dir + path;
        take(std::stoi(it.key()), parse_trace(slurp(path), cats));
      }
    }
    std::vector<std::pair<int, std::string>> marked;
    for (int i = 0; i < n; ++i) {
      const std::string path = paths[i];
      const std::string fname = path.substr(path.find_last_of('/') == std::string::npos
                                                ? 0 : path.find_last_of('/') + 1);
      int rank = 0;
      if (marker(fname, rank)) {
        marker(path, rank);
        marked.emplace_back(rank, path);
        continue;
      }
      for (auto& [r, sub] : split_by_rank(parse_trace(slurp(path), cats))) take(r, std::move(sub));
    }
    {
      std::map<int, std::vector<TraceEvent>> mr;
      for (const auto& [rank, path] : marked) {
        if (mr.count(rank))
          throw ParseError("duplicate rank " + std::to_string(rank) + " from '" + path + "'");
        mr.emplace(rank, parse_trace(slurp(path), cats));
      }
      for (auto& [rank, evs] : mr) take(rank, std::move(evs));
    }
    if (per_rank.empty()) throw ParseError("no input traces; pass --trace or --manifest");
    const std::string win = window ? window : "full";
    std::map<int, ExecutionGraph> graphs;
    for (auto& [rank, events] : per_rank) {
      std::vector<TraceEvent> scoped = std::move(events);
      if (win == "auto") {
        scoped = filter_window(scoped, detect_iteration_window(scoped));
      } else if (win != "full") {  // parse_window_arg (cli.cpp:72-85)
        const auto sep = win.find_first_of(":,");
        IterationWindow w;
        w.start = std::stoll(win.substr(0, sep));
        w.end = std::stoll(win.substr(sep + 1));
        scoped = filter_window(scoped, w);
      }
      graphs.emplace(rank, build_graph(scoped, policy, rank));
    }
    auto* r = new RefGraph;
    r->g = merge_ranks(graphs);
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// ------------------------------------------------------------- what-if retime
// Per-task retime metadata as the device takes it (ts_graph_desc.rt_*): the
// TS_RT_* class the reference's change_hidden / scale_dp would apply to the
// task (transform.cpp:219-349), read with their own strict integer parsing.
static std::optional<int64_t> shim_meta_i64(const Task& t, const char* key) {
  auto it = t.meta.find(key);
  if (it == t.meta.end()) return std::nullopt;
  try {
    std::size_t pos = 0;
    int64_t v = std::stoll(it->second, &pos);
    if (pos != it->second.size()) return std::nullopt;
    return v;
  } catch (const std::exception&) {
    return std::nullopt;
  }
}
static std::string shim_meta_str(const Task& t, const char* key) {
  auto it = t.meta.find(key);
  return it == t.meta.end() ? std::string() : it->second;
}

int ref_graph_retime_meta(void* h, uint8_t* kind, int64_t* bytes, int32_t* group, int64_t* mnk) {
  const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
  for (std::size_t i = 0; i < g.tasks.size(); ++i) {
    const Task& t = g.tasks[i];
    kind[i] = 0;
    auto b = shim_meta_i64(t, "bytes");
    bytes[i] = b ? *b : -1;
    auto gs = shim_meta_i64(t, "group_size");
    group[i] = gs ? static_cast<int32_t>(*gs) : 0;
    const int64_t m = shim_meta_i64(t, "m").value_or(0), n = shim_meta_i64(t, "n").value_or(0),
                  k = shim_meta_i64(t, "k").value_or(0);
    mnk[3 * i] = m;
    mnk[3 * i + 1] = n;
    mnk[3 * i + 2] = k;
    if (t.kind != TaskKind::Gpu) continue;
    if (t.op_class == OpClass::Compute) {
      if (m > 0 && n > 0 && k > 0) kind[i] = 1;                        // TS_RT_GEMM
      else if (shim_meta_str(t, "region") == "opt" && b) kind[i] = 2;  // TS_RT_OPT
    } else if (t.op_class == OpClass::Communication) {
      if (shim_meta_str(t, "collective") == "allreduce") {
        kind[i] = 3;  // TS_RT_ALLREDUCE (scale_dp checks bytes itself)
      } else if (shim_meta_str(t, "region") == "p2p" && b) {
        kind[i] = shim_meta_str(t, "dir") != "recv" ? 4 : 5;  // TS_RT_P2P_SEND / _RECV
      }
    }
  }
  return 0;
}

// apply_whatif's non-structural retime (transform.cpp:741-755): change_hidden
// (when d_model or d_ffn change) then scale_dp (when the sizes differ), with
// AnalyticalCostModel(alpha, bytes_per_us).  Returns a new handle or NULL
// (message in ref_last_error()).
void* ref_apply_retime(void* h, const int64_t* src_model, const int64_t* tgt_model, int src_dp,
                       int tgt_dp, double alpha, double bytes_per_us) {
  try {
    const ExecutionGraph& g = static_cast<RefGraph*>(h)->g;
    AnalyticalCostModel model(alpha, bytes_per_us);
    ExecutionGraph out = g;
    if (tgt_model) {
      ModelConfig sm, tm;
      sm.d_model = static_cast<int>(src_model[0]);
      sm.d_ffn = static_cast<int>(src_model[1]);
      sm.n_params = src_model[2];
      tm.d_model = static_cast<int>(tgt_model[0]);
      tm.d_ffn = static_cast<int>(tgt_model[1]);
      tm.n_params = tgt_model[2];
      out = change_hidden(out, sm, tm, model);
    }
    if (src_dp != tgt_dp) out = scale_dp(out, src_dp, tgt_dp, model);
    auto* r = new RefGraph;
    r->g = std::move(out);
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// apply_whatif (transform.cpp:713-760) with AnalyticalCostModel(alpha,
// bytes_per_us).  model = {n_params, n_layers, d_model, d_ffn, n_heads,
// d_head}, par = {tp, pp, dp, num_microbatches}.  Returns a new handle (the
// transformed graph) or NULL (message in ref_last_error()); notes gets the
// TransformResult notes joined by '\n' (truncated to cap).
void* ref_apply_whatif(void* h, const int64_t* src_model, const int64_t* tgt_model,
                       const int32_t* src_par, const int32_t* tgt_par, double alpha,
                       double bytes_per_us, int64_t activation_bytes, char* notes, int64_t cap) {
  try {
    auto model = [](const int64_t* m) {
      ModelConfig c;
      c.n_params = m[0];
      c.n_layers = static_cast<int>(m[1]);
      c.d_model = static_cast<int>(m[2]);
      c.d_ffn = static_cast<int>(m[3]);
      c.n_heads = static_cast<int>(m[4]);
      c.d_head = static_cast<int>(m[5]);
      return c;
    };
    auto par = [](const int32_t* p) {
      ParallelismConfig c;
      c.tp = p[0];
      c.pp = p[1];
      c.dp = p[2];
      c.num_microbatches = p[3];
      return c;
    };
    WhatIfConfig cfg;
    cfg.source_model = model(src_model);
    cfg.target_model = model(tgt_model);
    cfg.source_par = par(src_par);
    cfg.target_par = par(tgt_par);
    cfg.activation_bytes = activation_bytes;
    cfg.cost_model = std::make_shared<AnalyticalCostModel>(alpha, bytes_per_us);
    TransformResult res = apply_whatif(static_cast<RefGraph*>(h)->g, cfg);
    if (notes && cap > 0) {
      std::string all;
      for (const auto& n : res.notes) all += n + "\n";
      std::snprintf(notes, static_cast<size_t>(cap), "%s", all.c_str());
    }
    auto* r = new RefGraph;
    r->g = std::move(res.graph);
    return r;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

}  // extern "C"

// ------------------------------------------------ generator / estimate oracle
extern "C" {

// build_pipeline(pipeline_spec_for(spec), hook) with hook(i, base) =
// hook_dur[i] (or base when hook_dur is null).  Writes the events in output
// order (stable-sorted by (pid, ts, tid), pipeline.cpp:75-78): pid, tid, ts,
// dur.  Returns the event count (or -1); *n_ops receives the number of hook
// calls.
int64_t ref_pipeline_events(const char* spec_json, const int64_t* hook_dur, int64_t n_hook,
                            int32_t* pid, int32_t* tid, int64_t* ts, int64_t* dur, int64_t cap,
                            int64_t* n_ops) {
  int64_t count = -1;
  guarded([&] {
    SynthSpec spec = SynthSpec::from_json(spec_json);
    PipelineSpec ps = pipeline_spec_for(spec);
    int64_t calls = 0;
    DurationHook hook = [&](std::size_t i, Micros base) -> Micros {
      calls = std::max<int64_t>(calls, static_cast<int64_t>(i) + 1);
      if (hook_dur && static_cast<int64_t>(i) < n_hook) return hook_dur[i];
      return base;
    };
    BuiltPipeline b = build_pipeline(ps, hook);
    if (n_ops) *n_ops = calls;
    count = static_cast<int64_t>(b.events.size());
    for (int64_t i = 0; i < count && i < cap; ++i) {
      pid[i] = b.events[i].process_id;
      tid[i] = b.events[i].thread_id;
      ts[i] = b.events[i].timestamp;
      dur[i] = b.events[i].duration;
    }
    return 0;
  });
  return count;
}

}  // extern "C"

// ------------------------------------------------ PipelineSpec as JSON (tests)
// The Mode-B boundary takes a PipelineSpec (pipeline.hpp:27-90); tests build
// one from the reference's pipeline_spec_for (synth.cpp:71-138), edit it in
// Python and hand the same spec to both sides: JSON here, the ts_pipeline_spec
// POD on the engine side.
namespace {
nlohmann::json kernel_json(const KernelSpec& k) {
  return {{"name", k.name}, {"duration", k.duration}, {"op_class", static_cast<int>(k.op_class)},
          {"args", k.args}};
}
KernelSpec kernel_of(const nlohmann::json& j) {
  KernelSpec k;
  k.name = j.at("name").get<std::string>();
  k.duration = j.at("duration").get<Micros>();
  k.op_class = static_cast<OpClass>(j.value("op_class", 0));
  k.args = j.value("args", std::map<std::string, std::string>{});
  return k;
}
std::vector<KernelSpec> kernels_of(const nlohmann::json& a) {
  std::vector<KernelSpec> v;
  for (const auto& k : a) v.push_back(kernel_of(k));
  return v;
}
nlohmann::json list_json(const std::vector<KernelSpec>& v) {
  nlohmann::json a = nlohmann::json::array();
  for (const auto& k : v) a.push_back(kernel_json(k));
  return a;
}
PipelineSpec pipeline_of(const nlohmann::json& j) {
  PipelineSpec p;
  p.pp = j.at("pp");
  p.dp = j.at("dp");
  p.num_microbatches = j.at("num_microbatches");
  p.host.launch = j.at("launch");
  p.host.record = j.at("record");
  p.host.wait = j.at("wait");
  p.host.sync = j.at("sync");
  p.p2p_send = j.at("p2p_send");
  p.p2p_recv_base = j.at("p2p_recv_base");
  p.activation_bytes = j.at("activation_bytes");
  p.origin = j.at("origin");
  p.compute_stream = j.at("compute_stream");
  p.reduce_stream = j.at("reduce_stream");
  p.p2p_stream = j.at("p2p_stream");
  p.main_thread = j.at("main_thread");
  p.helper_thread = j.at("helper_thread");
  p.first_event = j.at("first_event");
  p.first_correlation = j.at("first_correlation");
  for (const auto& s : j.at("stages")) {
    StageSpec st;
    for (const auto& l : s.at("layers_fwd")) st.layers_fwd.push_back(kernels_of(l));
    for (const auto& l : s.at("layers_bwd")) st.layers_bwd.push_back(kernels_of(l));
    st.pre_fwd = kernels_of(s.at("pre_fwd"));
    st.post_fwd = kernels_of(s.at("post_fwd"));
    st.pre_bwd = kernels_of(s.at("pre_bwd"));
    st.post_bwd = kernels_of(s.at("post_bwd"));
    st.reduce = kernels_of(s.at("reduce"));
    st.optimizer = kernels_of(s.at("optimizer"));
    p.stages.push_back(std::move(st));
  }
  return p;
}
std::string g_spec_json;
}  // namespace

extern "C" {

// pipeline_spec_for(SynthSpec::from_json(spec_json)) as JSON (valid until the next call)
const char* ref_pipeline_spec_json(const char* spec_json) {
  try {
    PipelineSpec p = pipeline_spec_for(SynthSpec::from_json(spec_json));
    nlohmann::json j = {{"pp", p.pp}, {"dp", p.dp}, {"num_microbatches", p.num_microbatches},
                        {"launch", p.host.launch}, {"record", p.host.record},
                        {"wait", p.host.wait}, {"sync", p.host.sync},
                        {"p2p_send", p.p2p_send}, {"p2p_recv_base", p.p2p_recv_base},
                        {"activation_bytes", p.activation_bytes}, {"origin", p.origin},
                        {"compute_stream", p.compute_stream}, {"reduce_stream", p.reduce_stream},
                        {"p2p_stream", p.p2p_stream}, {"main_thread", p.main_thread},
                        {"helper_thread", p.helper_thread}, {"first_event", p.first_event},
                        {"first_correlation", p.first_correlation}};
    nlohmann::json stages = nlohmann::json::array();
    for (const auto& st : p.stages) {
      nlohmann::json s;
      s["layers_fwd"] = nlohmann::json::array();
      for (const auto& l : st.layers_fwd) s["layers_fwd"].push_back(list_json(l));
      s["layers_bwd"] = nlohmann::json::array();
      for (const auto& l : st.layers_bwd) s["layers_bwd"].push_back(list_json(l));
      s["pre_fwd"] = list_json(st.pre_fwd);
      s["post_fwd"] = list_json(st.post_fwd);
      s["pre_bwd"] = list_json(st.pre_bwd);
      s["post_bwd"] = list_json(st.post_bwd);
      s["reduce"] = list_json(st.reduce);
      s["optimizer"] = list_json(st.optimizer);
      stages.push_back(s);
    }
    j["stages"] = stages;
    g_spec_json = j.dump();
    return g_spec_json.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// build_pipeline(pipeline_of(json), hook) events, like ref_pipeline_events;
// *end receives BuiltPipeline::end
int64_t ref_pipeline_events_json(const char* pipeline_json, const int64_t* hook_dur,
                                 int64_t n_hook, int32_t* pid, int32_t* tid, int64_t* ts,
                                 int64_t* dur, int64_t cap, int64_t* n_ops, int64_t* end) {
  int64_t count = -1;
  guarded([&] {
    PipelineSpec ps = pipeline_of(nlohmann::json::parse(pipeline_json));
    int64_t calls = 0;
    DurationHook hook = [&](std::size_t i, Micros base) -> Micros {
      calls = std::max<int64_t>(calls, static_cast<int64_t>(i) + 1);
      if (hook_dur && static_cast<int64_t>(i) < n_hook) return hook_dur[i];
      return base;
    };
    BuiltPipeline b = build_pipeline(ps, hook);
    if (n_ops) *n_ops = calls;
    if (end) *end = b.end;
    count = static_cast<int64_t>(b.events.size());
    for (int64_t i = 0; i < count && i < cap; ++i) {
      pid[i] = b.events[i].process_id;
      tid[i] = b.events[i].thread_id;
      ts[i] = b.events[i].timestamp;
      dur[i] = b.events[i].duration;
    }
    return 0;
  });
  return count;
}

}  // extern "C"
