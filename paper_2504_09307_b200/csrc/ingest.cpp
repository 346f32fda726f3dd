// ingest.cpp — trace events -> ExecutionGraph (see ingest.hpp).
//
// Each step restates one part of the reference builder (paths under
// /root/reference/proj/src):
//   nested-span dropping         build.cpp:228-278
//   task creation, window        build.cpp:338-373
//   lane chains                  build.cpp:375-386
//   launch -> kernel edges       build.cpp:388-422
//   event record / wait edges    build.cpp:424-492
//   cross-thread gap edges       build.cpp:106-167
//   GPU -> CPU sync rules        build.cpp:169-224
//   edge normalisation, cycles   build.cpp:501-509, 280-334
#include "ingest.hpp"

#include <algorithm>
#include <cctype>
#include <map>
#include <sstream>
#include <tuple>

namespace lumos {

namespace {

bool is_gpu_cat(uint8_t c) { return c == CAT_KERNEL || c == CAT_MEMCPY || c == CAT_MEMSET; }

std::string lower(std::string s) {
  for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

}  // namespace

bool BuildPolicyLite::is_launch(const std::string& n) const {
  return std::find(launch_names.begin(), launch_names.end(), n) != launch_names.end();
}
bool BuildPolicyLite::is_record(const std::string& n) const {
  return std::find(record_names.begin(), record_names.end(), n) != record_names.end();
}
bool BuildPolicyLite::is_wait(const std::string& n) const {
  return std::find(wait_names.begin(), wait_names.end(), n) != wait_names.end();
}
int BuildPolicyLite::sync_flavor(const std::string& n) const {
  for (const auto& [name, f] : sync_names)
    if (name == n) return f;
  return 0;
}
bool BuildPolicyLite::is_comm(const std::string& n) const {
  const std::string l = lower(n);
  for (const std::string& p : comm_patterns)
    if (l.find(p) != std::string::npos) return true;
  return false;
}

bool is_comm_name(const std::string& name) {
  static const BuildPolicyLite kDefault;
  return kDefault.is_comm(name);
}

uint8_t classify_event(const Event& e, const Names& names, const BuildPolicyLite& policy) {
  const std::string& n = names.str[e.name];
  if (e.cat == CAT_MEMCPY) return TS_OP_COMMUNICATION;
  if (is_gpu_cat(e.cat)) return policy.is_comm(n) ? TS_OP_COMMUNICATION : TS_OP_COMPUTE;
  if (policy.is_launch(n)) return TS_OP_LAUNCH;
  if (policy.sync_flavor(n)) return TS_OP_SYNC;
  if (policy.is_record(n)) return TS_OP_EVENT_RECORD;
  if (policy.is_wait(n)) return TS_OP_EVENT_WAIT;
  return TS_OP_OTHER;
}

uint8_t classify_event(const Event& e, const Names& names) {
  static const BuildPolicyLite kDefault;
  return classify_event(e, names, kDefault);
}

ts_graph_desc HostGraph::desc() const {
  ts_graph_desc d{};
  d.n_tasks = n();
  d.duration = duration.data();
  d.original_start = original_start.data();
  d.rank = rank.data();
  d.lane_kind = lane_kind.data();
  d.lane = lane.data();
  d.op_class = op_class.data();
  d.task_kind = task_kind.data();
  d.scale_class = nullptr;
  d.n_edges = static_cast<int64_t>(edge_from.size());
  d.edge_from = edge_from.data();
  d.edge_to = edge_to.data();
  d.n_rules = static_cast<int32_t>(rule_kind.size());
  d.rule_kind = rule_kind.data();
  d.rule_task = rule_task.data();
  d.rule_bound = rule_bound.data();
  d.rule_watch_off = rule_watch_off.data();
  d.watch_rank = watch_rank.data();
  d.watch_kind = watch_kind.data();
  d.watch_lane = watch_lane.data();
  d.window_start = window_start;
  d.window_end = window_end;
  d.n_gates = static_cast<int64_t>(gate_from.size());
  d.gate_from = gate_from.data();
  d.gate_to = gate_to.data();
  d.gate_kind = gate_kind.data();
  if (!rt_kind.empty() && rt_kind.size() == duration.size()) {
    d.rt_kind = rt_kind.data();
    d.rt_bytes = rt_bytes.data();
    d.rt_group = rt_group.data();
    d.rt_mnk = rt_mnk.data();
  }
  return d;
}

void HostGraph::append_relabelled(const HostGraph& src, int32_t new_rank, bool first) {
  const int32_t base = n();
  auto cat = [](auto& dst, const auto& s) { dst.insert(dst.end(), s.begin(), s.end()); };
  cat(duration, src.duration);
  cat(original_start, src.original_start);
  if (new_rank == INT32_MIN) {
    cat(rank, src.rank);
  } else {
    rank.insert(rank.end(), src.rank.size(), new_rank);
  }
  cat(lane_kind, src.lane_kind);
  cat(lane, src.lane);
  cat(op_class, src.op_class);
  cat(task_kind, src.task_kind);
  cat(name, src.name);
  cat(op_index, src.op_index);
  cat(corr, src.corr);
  cat(meta, src.meta);
  for (size_t e = 0; e < src.edge_from.size(); ++e) {
    edge_from.push_back(src.edge_from[e] + base);
    edge_to.push_back(src.edge_to[e] + base);
  }
  const int32_t w0 = static_cast<int32_t>(watch_rank.size());
  for (size_t r = 0; r < src.rule_kind.size(); ++r) {
    rule_kind.push_back(src.rule_kind[r]);
    rule_task.push_back(src.rule_task[r] + base);
    rule_bound.push_back(src.rule_bound[r] >= 0 ? src.rule_bound[r] + base : -1);
    rule_watch_off.push_back(w0 + src.rule_watch_off[r + 1]);
  }
  if (new_rank == INT32_MIN) {
    cat(watch_rank, src.watch_rank);
  } else {
    watch_rank.insert(watch_rank.end(), src.watch_rank.size(), new_rank);
  }
  cat(watch_kind, src.watch_kind);
  cat(watch_lane, src.watch_lane);
  for (size_t g = 0; g < src.gate_from.size(); ++g) {
    gate_from.push_back(src.gate_from[g] + base);
    gate_to.push_back(src.gate_to[g] + base);
    gate_kind.push_back(src.gate_kind[g]);
  }
  n_diagnostics += src.n_diagnostics;
  if (first) {
    window_start = src.window_start;
    window_end = src.window_end;
  } else {
    window_start = std::min(window_start, src.window_start);
    window_end = std::max(window_end, src.window_end);
  }
}

void HostGraph::append(const HostGraph& src, bool first) { append_relabelled(src, INT32_MIN, first); }

int build_rank_graph(const std::vector<Event>& events, const Names& names, int32_t rank,
                     const BuildPolicyLite& policy, HostGraph& g, std::string& err,
                     const std::vector<MetaList>* meta) {
  g = HostGraph{};
  if (events.empty()) return TS_OK;

  // ---- drop enclosing CPU spans (profiler nesting)
  const size_t ne = events.size();
  std::vector<char> enclosing(ne, 0);
  {
    std::map<int32_t, std::vector<size_t>> by_thread;
    for (size_t i = 0; i < ne; ++i)
      if (events[i].cat == CAT_CPU_OP || events[i].cat == CAT_RUNTIME)
        by_thread[events[i].tid].push_back(i);
    std::vector<size_t> open;
    for (auto& [tid, list] : by_thread) {
      std::sort(list.begin(), list.end(), [&](size_t a, size_t b) {
        const Event& x = events[a];
        const Event& y = events[b];
        if (x.ts != y.ts) return x.ts < y.ts;
        if (x.dur != y.dur) return x.dur > y.dur;
        return a < b;
      });
      open.clear();
      for (size_t i : list) {
        while (!open.empty() && events[open.back()].ts + events[open.back()].dur <= events[i].ts)
          open.pop_back();
        if (!open.empty()) enclosing[open.back()] = 1;
        open.push_back(i);
      }
    }
  }
  std::vector<size_t> kept;
  kept.reserve(ne);
  int dropped = 0;
  for (size_t i = 0; i < ne; ++i) {
    if (events[i].cat == CAT_METADATA) continue;
    if (enclosing[i]) {
      ++dropped;
      continue;
    }
    kept.push_back(i);
  }
  if (dropped) g.n_diagnostics++;

  // ---- tasks
  const int32_t n = static_cast<int32_t>(kept.size());
  g.duration.resize(n);
  g.original_start.resize(n);
  g.rank.assign(n, rank);
  g.lane_kind.resize(n);
  g.lane.resize(n);
  g.op_class.resize(n);
  g.task_kind.resize(n);
  g.name.resize(n);
  g.op_index.resize(n);
  std::vector<int64_t> corr(n), arg_event(n), arg_stream(n);
  for (int32_t t = 0; t < n; ++t) {
    const Event& e = events[kept[t]];
    const bool gpu = is_gpu_cat(e.cat);
    g.task_kind[t] = gpu ? 1 : 0;
    g.op_class[t] = classify_event(e, names, policy);
    g.duration[t] = e.dur;
    g.original_start[t] = e.ts;
    g.name[t] = e.name;
    g.op_index[t] = e.op_index;
    corr[t] = e.corr;
    arg_event[t] = e.arg_event;
    arg_stream[t] = e.arg_stream;
    if (gpu) {
      if (e.stream < 0) {
        err = "GPU event '" + names.str[e.name] + "' has no stream id";
        return TS_E_GRAPH;
      }
      g.lane_kind[t] = TS_LANE_CUDA_STREAM;
      g.lane[t] = e.stream;
    } else {
      g.lane_kind[t] = TS_LANE_CPU_THREAD;
      g.lane[t] = e.tid;
    }
  }
  if (meta) {
    g.corr = corr;
    g.meta.resize(n);
    for (int32_t t = 0; t < n; ++t) g.meta[t] = (*meta)[kept[t]];
  }
  g.window_start = g.original_start[0];
  g.window_end = g.window_start;
  for (int32_t t = 0; t < n; ++t) {
    g.window_start = std::min(g.window_start, g.original_start[t]);
    g.window_end = std::max(g.window_end, g.original_start[t] + g.duration[t]);
  }

  std::vector<std::pair<int32_t, int32_t>> edges;
  edges.reserve(static_cast<size_t>(n) * 2);

  // ---- lane chains: processors ordered (kind, lane) like ProcessorId
  std::map<std::pair<int32_t, int32_t>, std::vector<int32_t>> lanes;
  for (int32_t t = 0; t < n; ++t) lanes[{g.lane_kind[t], g.lane[t]}].push_back(t);
  for (auto& [proc, ids] : lanes) {
    std::sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) {
      if (g.original_start[a] != g.original_start[b])
        return g.original_start[a] < g.original_start[b];
      return a < b;
    });
    for (size_t i = 1; i < ids.size(); ++i) edges.emplace_back(ids[i - 1], ids[i]);
  }

  // ---- launch -> kernel
  std::unordered_map<int64_t, int32_t> launches;
  for (int32_t t = 0; t < n; ++t)
    if (g.task_kind[t] == 0 && g.op_class[t] == TS_OP_LAUNCH && corr[t] != -1)
      launches[corr[t]] = t;
  std::unordered_map<int64_t, char> used;
  std::map<int32_t, std::vector<std::pair<int64_t, int32_t>>> enqueue;  // stream -> (ts, id)
  for (int32_t t = 0; t < n; ++t) {
    if (g.task_kind[t] != 1) continue;
    int64_t launch_ts = g.original_start[t];
    bool found = false;
    if (corr[t] != -1) {
      auto it = launches.find(corr[t]);
      if (it != launches.end()) {
        edges.emplace_back(it->second, t);
        launch_ts = g.original_start[it->second];
        used[corr[t]] = 1;
        found = true;
      }
    }
    if (!found) g.n_diagnostics++;
    enqueue[g.lane[t]].emplace_back(launch_ts, t);
  }
  for (const auto& [c, id] : launches)
    if (!used.count(c)) g.n_diagnostics++;
  for (auto& [s, order] : enqueue) std::sort(order.begin(), order.end());
  auto last_enqueued_before = [&](int32_t stream, int64_t ts) -> int32_t {
    auto it = enqueue.find(stream);
    if (it == enqueue.end()) return -1;
    const auto& o = it->second;
    auto pos = std::lower_bound(o.begin(), o.end(), std::make_pair(ts, int32_t{-1}));
    return pos == o.begin() ? -1 : std::prev(pos)->second;
  };
  auto first_enqueued_after = [&](int32_t stream, int64_t ts) -> int32_t {
    auto it = enqueue.find(stream);
    if (it == enqueue.end()) return -1;
    const auto& o = it->second;
    auto pos = std::upper_bound(o.begin(), o.end(), ts,
                                [](int64_t v, const std::pair<int64_t, int32_t>& e) {
                                  return v < e.first;
                                });
    return pos == o.end() ? -1 : pos->second;
  };

  // ---- event record / wait pairing
  std::vector<int32_t> recs, waits;
  for (int32_t t = 0; t < n; ++t) {
    if (g.op_class[t] == TS_OP_EVENT_RECORD) recs.push_back(t);
    if (g.op_class[t] == TS_OP_EVENT_WAIT) waits.push_back(t);
  }
  auto by_start = [&](int32_t a, int32_t b) {
    if (g.original_start[a] != g.original_start[b]) return g.original_start[a] < g.original_start[b];
    return a < b;
  };
  std::sort(recs.begin(), recs.end(), by_start);
  std::sort(waits.begin(), waits.end(), by_start);
  std::map<int64_t, std::vector<std::pair<int64_t, int32_t>>> records;
  for (int32_t t : recs) {
    if (arg_event[t] == kNoArg || arg_stream[t] == kNoArg) continue;
    int32_t pred = last_enqueued_before(static_cast<int32_t>(arg_stream[t]), g.original_start[t]);
    if (pred < 0) g.n_diagnostics++;
    records[arg_event[t]].emplace_back(g.original_start[t], pred);
  }
  for (int32_t t : waits) {
    if (arg_event[t] == kNoArg || arg_stream[t] == kNoArg) continue;
    auto it = records.find(arg_event[t]);
    int32_t pred = -1;
    if (it != records.end())
      for (const auto& [ts, p] : it->second) {
        if (ts >= g.original_start[t]) break;
        pred = p;
      }
    if (pred < 0) {
      g.n_diagnostics++;
      continue;
    }
    int32_t succ = first_enqueued_after(static_cast<int32_t>(arg_stream[t]), g.original_start[t]);
    if (succ >= 0 && succ != pred) edges.emplace_back(pred, succ);
  }

  // ---- cross-thread gap edges (infer_cpu_cpu)
  {
    struct Cand {
      int64_t end, start;
      int32_t id, lane;
    };
    std::vector<Cand> by_end;
    std::map<int32_t, std::vector<int32_t>> by_thread;
    for (int32_t t = 0; t < n; ++t) {
      if (g.task_kind[t] != 0) continue;
      by_thread[g.lane[t]].push_back(t);
      by_end.push_back({g.original_start[t] + g.duration[t], g.original_start[t], t, g.lane[t]});
    }
    std::sort(by_end.begin(), by_end.end(), [](const Cand& a, const Cand& b) {
      return std::tie(a.end, a.start, a.id) < std::tie(b.end, b.start, b.id);
    });
    if (by_thread.size() >= 2) {
      for (auto& [lane, list] : by_thread) {
        std::sort(list.begin(), list.end(), by_start);
        int64_t prev_end = g.window_start;
        for (int32_t t : list) {
          const int64_t gap = g.original_start[t] - prev_end;
          if (gap >= policy.gap_threshold_us) {
            auto it = std::upper_bound(by_end.begin(), by_end.end(), g.original_start[t],
                                       [](int64_t v, const Cand& c) { return v < c.end; });
            const Cand* found = nullptr;
            while (it != by_end.begin()) {
              --it;
              if (it->end < prev_end) break;
              if (it->lane != lane && it->id != t) {
                found = &*it;
                break;
              }
            }
            if (found) {
              edges.emplace_back(found->id, t);
              g.n_diagnostics++;
            }
          }
          prev_end = std::max(prev_end, g.original_start[t] + g.duration[t]);
        }
      }
    }
  }

  // ---- GPU -> CPU sync rules (infer_gpu_cpu)
  std::vector<int32_t> stream_lanes;  // this rank's CUDA streams, ascending
  for (const auto& [proc, ids] : lanes)
    if (proc.first == TS_LANE_CUDA_STREAM) stream_lanes.push_back(proc.second);
  for (int32_t t = 0; t < n; ++t) {
    if (g.task_kind[t] != 0 || g.op_class[t] != TS_OP_SYNC) continue;
    const int flavor = policy.sync_flavor(names.str[g.name[t]]);
    if (!flavor) continue;
    int32_t bound = -1;
    if (flavor == 1) {
      g.rule_kind.push_back(TS_RULE_DEVICE_SYNC);
      for (int32_t s : stream_lanes) {
        g.watch_rank.push_back(rank);
        g.watch_kind.push_back(TS_LANE_CUDA_STREAM);
        g.watch_lane.push_back(s);
      }
    } else if (flavor == 2) {
      g.rule_kind.push_back(TS_RULE_STREAM_SYNC);
      const bool ok = arg_stream[t] != kNoArg &&
                      lanes.count({TS_LANE_CUDA_STREAM, static_cast<int32_t>(arg_stream[t])});
      if (ok) {
        g.watch_rank.push_back(rank);
        g.watch_kind.push_back(TS_LANE_CUDA_STREAM);
        g.watch_lane.push_back(static_cast<int32_t>(arg_stream[t]));
      } else {
        g.n_diagnostics++;
      }
    } else {
      g.rule_kind.push_back(TS_RULE_EVENT_SYNC);
      if (arg_event[t] != kNoArg) {
        auto it = records.find(arg_event[t]);
        if (it != records.end())
          for (const auto& [ts, p] : it->second) {
            if (ts >= g.original_start[t]) break;
            bound = p;
          }
      }
      if (bound < 0) g.n_diagnostics++;
    }
    g.rule_task.push_back(t);
    g.rule_bound.push_back(bound);
    g.rule_watch_off.push_back(static_cast<int32_t>(g.watch_rank.size()));
  }

  // ---- normalise edges; reject cycles
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  edges.erase(std::remove_if(edges.begin(), edges.end(),
                             [](const std::pair<int32_t, int32_t>& e) { return e.first == e.second; }),
              edges.end());
  g.edge_from.resize(edges.size());
  g.edge_to.resize(edges.size());
  for (size_t i = 0; i < edges.size(); ++i) {
    g.edge_from[i] = edges[i].first;
    g.edge_to[i] = edges[i].second;
  }
  {
    std::vector<int32_t> indeg(n, 0);
    std::vector<std::vector<int32_t>> out(n);
    for (const auto& e : edges) {
      out[e.first].push_back(e.second);
      indeg[e.second]++;
    }
    std::vector<int32_t> q;
    for (int32_t i = 0; i < n; ++i)
      if (indeg[i] == 0) q.push_back(i);
    for (size_t h = 0; h < q.size(); ++h)
      for (int32_t v : out[q[h]])
        if (--indeg[v] == 0) q.push_back(v);
    if (static_cast<int32_t>(q.size()) != n) {
      std::vector<std::vector<int32_t>> in(n);
      for (const auto& e : edges)
        if (indeg[e.second] > 0) in[e.second].push_back(e.first);
      int32_t cur = -1;
      for (int32_t i = 0; i < n && cur < 0; ++i)
        if (indeg[i] > 0) cur = i;
      std::vector<int32_t> path, pos(n, -1);
      while (pos[cur] < 0) {
        pos[cur] = static_cast<int32_t>(path.size());
        path.push_back(cur);
        int32_t next = -1;
        for (int32_t p : in[cur])
          if (indeg[p] > 0) {
            next = p;
            break;
          }
        cur = next;
      }
      std::ostringstream msg;
      msg << "dependency cycle:";
      for (size_t i = static_cast<size_t>(pos[cur]); i < path.size(); ++i) msg << " " << path[i];
      err = msg.str();
      return TS_E_GRAPH;
    }
  }
  return TS_OK;
}

}  // namespace lumos
