// compile.cpp — ExecutionGraph -> straight-line replay programs (host side).
//
// Reference semantics being compiled (paths under /root/reference/proj):
//   validate_graph                      src/simulate.cpp:26-125
//   Engine (lanes, ready sets, rules)   src/simulate.cpp:145-337
//   lane chains                         src/build.cpp:375-386
//   Stream/DeviceSync rules             src/build.cpp:169-224, simulate.cpp:210-216
//   EventSync rules                     src/simulate.cpp:206-209
//   generator barrier / rendezvous      src/pipeline.cpp:377-389 (gates)
//
// On a graph whose lanes are chained (each lane's tasks, in (original_start,
// id) order, are linked by fixed edges — true for every build_graph output),
// at most one task per lane is ever ready, so dispatch order never matters and
// the replay is the max-plus longest path
//     start(v) = max(W, finish(preds)),  finish(v) = start(v) + d(v).
// EventSync adds the edge bound -> waiting task.  A Stream/DeviceSync task s
// starts at the first instant >= its ready time r_s at which every watched
// stream is idle with nothing pending.  We bind it statically to k*_w, the last
// kernel of each watched stream enqueued before s (the launch order build_graph
// uses, build.cpp:426-434), and emit a per-scenario certificate that the
// static start S = max(r_s, finish(k*_w)) equals the reference's instant:
//   (a) S == r_s, or some watched stream w0 with finish(k*_w0) == S was busy
//       without a gap over [r_s, S) (busy-since(k*_w0) <= r_s), and
//   (b) for every watched stream whose next kernel n_w is not a descendant of
//       s, start(n_w) > S (nothing else occupies or becomes ready on it at S).
// A scenario whose certificate fails is flagged and replayed by the exact
// event-driven kernel instead.
#include "compile.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <cstring>
#include <numeric>
#include <queue>
#include <sstream>
#include <tuple>
#include <unordered_map>

namespace lumos {

namespace {

struct Proc {
  int32_t rank, kind, lane;
  bool operator<(const Proc& o) const {
    return std::tie(rank, kind, lane) < std::tie(o.rank, o.kind, o.lane);
  }
  bool operator==(const Proc& o) const {
    return rank == o.rank && kind == o.kind && lane == o.lane;
  }
};

struct Csr {
  std::vector<int64_t> off;
  std::vector<int32_t> idx;
  int64_t begin(int64_t v) const { return off[v]; }
  int64_t end(int64_t v) const { return off[v + 1]; }
};

Csr build_csr(int64_t n, const std::vector<std::pair<int32_t, int32_t>>& edges, bool forward) {
  Csr c;
  c.off.assign(n + 1, 0);
  for (const auto& e : edges) c.off[(forward ? e.first : e.second) + 1]++;
  for (int64_t i = 0; i < n; ++i) c.off[i + 1] += c.off[i];
  c.idx.resize(edges.size());
  std::vector<int64_t> fill(c.off.begin(), c.off.end() - 1);
  for (const auto& e : edges) {
    int32_t a = forward ? e.first : e.second;
    int32_t b = forward ? e.second : e.first;
    c.idx[fill[a]++] = b;
  }
  return c;
}

std::string join_ids(const std::vector<int32_t>& ids) {
  std::ostringstream os;
  for (size_t i = 0; i < ids.size(); ++i) os << (i ? " " : "") << ids[i];
  return os.str();
}

struct IrOp {
  Op op{};
  int64_t v_pred[4] = {-1, -1, -1, -1};
  int64_t v_dst = -1, v_x0 = -1, v_x1 = -1, v_x2 = -1;
  bool is_ext = false;
  int64_t v_fin[kCertPerExt] = {-1, -1, -1, -1};
  int64_t v_bs[kCertPerExt] = {-1, -1, -1, -1};
  int64_t v_next[kCertPerExt] = {-1, -1, -1, -1};
  int32_t n_ent = 0;
  bool is_cov = false;
  int64_t v_cov_src[kCovSets][4] = {{-1, -1, -1, -1}, {-1, -1, -1, -1}};
  int64_t v_cov_dst[kCovSets] = {-1, -1};
  int n_sets = 0;
  int64_t v_cov1_src = -1, v_cov1_dst = -1;  // F_TRACK1
  bool aux() const { return is_ext || is_cov; }
};

// retime kinds whose duration a retime walk recomputes (a receive keeps its
// recorded duration, transform.cpp:342)
bool rt_walk_kind(uint8_t k) {
  return k == TS_RT_GEMM || k == TS_RT_OPT || k == TS_RT_ALLREDUCE || k == TS_RT_P2P_SEND;
}

bool same_rt_meta(const ts_graph_desc& d, int32_t a, int32_t b) {
  if (d.rt_kind[a] != d.rt_kind[b]) return false;
  if (d.rt_bytes && d.rt_bytes[a] != d.rt_bytes[b]) return false;
  if (d.rt_group && d.rt_group[a] != d.rt_group[b]) return false;
  if (d.rt_mnk)
    for (int k = 0; k < 3; ++k)
      if (d.rt_mnk[3 * static_cast<size_t>(a) + k] != d.rt_mnk[3 * static_cast<size_t>(b) + k])
        return false;
  return true;
}

struct CertEntry {
  int32_t kstar;  // -1: no kernel bound before the sync
  int32_t next;   // -1: none or a descendant of the sync
};

}  // namespace

namespace {

int compile_programs(const ts_graph_desc& d, CompiledGraph& out, std::string& err,
                     bool allow_coop) {
  const int32_t n = d.n_tasks;
  if (n < 0) {
    err = "n_tasks must be non-negative";
    return TS_E_INVALID_ARGUMENT;
  }
  out = CompiledGraph{};
  out.n_tasks = n;
  out.window_start = d.window_start;
  out.window_end = d.window_end;

  // ---------------------------------------------------------- validate_graph
  for (int32_t i = 0; i < n; ++i)
    if (d.duration[i] < 0) {
      err = "invalid graph: task " + std::to_string(i) + " has negative duration";
      return TS_E_SIMULATION;
    }
  std::vector<std::pair<int32_t, int32_t>> fixed;
  fixed.reserve(static_cast<size_t>(d.n_edges));
  for (int64_t e = 0; e < d.n_edges; ++e) {
    int32_t u = d.edge_from[e], v = d.edge_to[e];
    if (u < 0 || u >= n || v < 0 || v >= n || u == v) {
      err = "invalid graph: edge " + std::to_string(u) + "->" + std::to_string(v) +
            " references an invalid task";
      return TS_E_SIMULATION;
    }
    fixed.emplace_back(u, v);
  }
  for (int32_t r = 0; r < d.n_rules; ++r) {
    int32_t w = d.rule_task[r], b = d.rule_bound ? d.rule_bound[r] : -1;
    if (w < 0 || w >= n || (b >= 0 && b >= n)) {
      err = "invalid graph: rule on task " + std::to_string(w) + " references an invalid task";
      return TS_E_SIMULATION;
    }
  }
  std::sort(fixed.begin(), fixed.end());
  fixed.erase(std::unique(fixed.begin(), fixed.end()), fixed.end());
  Csr succ = build_csr(n, fixed, true);
  Csr pred = build_csr(n, fixed, false);
  {
    // Kahn cycle check with the reference's witness walk (simulate.cpp:79-121)
    std::vector<int32_t> left(n, 0);
    for (const auto& e : fixed) left[e.second]++;
    std::vector<int32_t> q;
    q.reserve(n);
    for (int32_t i = 0; i < n; ++i)
      if (left[i] == 0) q.push_back(i);
    for (size_t h = 0; h < q.size(); ++h)
      for (int64_t k = succ.begin(q[h]); k < succ.end(q[h]); ++k)
        if (--left[succ.idx[k]] == 0) q.push_back(succ.idx[k]);
    if (static_cast<int32_t>(q.size()) != n) {
      int32_t cur = -1;
      for (int32_t i = 0; i < n && cur < 0; ++i)
        if (left[i] > 0) cur = i;
      std::vector<int32_t> path;
      std::vector<char> on_path(n, 0);
      while (cur >= 0 && !on_path[cur]) {
        on_path[cur] = 1;
        path.push_back(cur);
        int32_t next = -1;
        for (int64_t k = pred.begin(cur); k < pred.end(cur); ++k) {
          int32_t p = pred.idx[k];
          if (left[p] > 0 && (next < 0 || p < next)) next = p;
        }
        cur = next;
      }
      std::vector<int32_t> cycle;
      if (cur >= 0) {
        auto it = std::find(path.begin(), path.end(), cur);
        cycle.assign(it, path.end());
        std::reverse(cycle.begin(), cycle.end());
      }
      err = "invalid graph: dependency cycle: " + join_ids(cycle);
      return TS_E_SIMULATION;
    }
  }

  // ---------------------------------------------------------------- lanes
  std::vector<Proc> procs(n);
  for (int32_t i = 0; i < n; ++i) procs[i] = {d.rank[i], d.lane_kind[i], d.lane[i]};
  std::vector<Proc> lanes = procs;
  std::sort(lanes.begin(), lanes.end());
  lanes.erase(std::unique(lanes.begin(), lanes.end()), lanes.end());
  const int32_t nl = static_cast<int32_t>(lanes.size());
  auto lane_index = [&](const Proc& p) -> int32_t {
    auto it = std::lower_bound(lanes.begin(), lanes.end(), p);
    return (it != lanes.end() && *it == p) ? static_cast<int32_t>(it - lanes.begin()) : -1;
  };
  std::vector<int32_t> lane_of(n);
  std::vector<int32_t> lane_off(nl + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    lane_of[i] = lane_index(procs[i]);
    lane_off[lane_of[i] + 1]++;
  }
  for (int32_t l = 0; l < nl; ++l) lane_off[l + 1] += lane_off[l];
  std::vector<int32_t> lane_tasks(n);
  {
    std::vector<int32_t> fill(lane_off.begin(), lane_off.end() - 1);
    for (int32_t i = 0; i < n; ++i) lane_tasks[fill[lane_of[i]]++] = i;
  }
  std::vector<int32_t> chain_pos(n), chain_prev(n, -1);
  auto has_edge = [&](int32_t u, int32_t v) {
    auto b = succ.idx.begin() + succ.begin(u), e = succ.idx.begin() + succ.end(u);
    return std::binary_search(b, e, v);
  };
  for (int32_t l = 0; l < nl; ++l) {
    auto b = lane_tasks.begin() + lane_off[l], e = lane_tasks.begin() + lane_off[l + 1];
    std::sort(b, e, [&](int32_t x, int32_t y) {
      return std::make_pair(d.original_start[x], x) < std::make_pair(d.original_start[y], y);
    });
    for (int32_t k = lane_off[l]; k < lane_off[l + 1]; ++k) {
      int32_t t = lane_tasks[k];
      chain_pos[t] = k - lane_off[l];
      if (k > lane_off[l]) {
        int32_t p = lane_tasks[k - 1];
        if (!has_edge(p, t)) {
          err = "unsupported graph: lane rank" + std::to_string(lanes[l].rank) +
                (lanes[l].kind ? "/stream" : "/thread") + std::to_string(lanes[l].lane) +
                " is not chained (no fixed edge " + std::to_string(p) + "->" +
                std::to_string(t) + "); the device path replays chained lanes";
          return TS_E_UNSUPPORTED;
        }
        chain_prev[t] = p;
      }
    }
  }

  // ---------------------------------------------------------------- rules
  std::vector<int32_t> rule_of(n, -1);
  for (int32_t r = 0; r < d.n_rules; ++r) rule_of[d.rule_task[r]] = r;  // later rule wins

  // enqueue time of each kernel: its launch's recorded start (build.cpp:398-415)
  std::vector<int64_t> enqueue_ts(n);
  for (int32_t i = 0; i < n; ++i) {
    enqueue_ts[i] = d.original_start[i];
    if (d.lane_kind[i] != TS_LANE_CUDA_STREAM) continue;
    for (int64_t k = pred.begin(i); k < pred.end(i); ++k) {
      int32_t p = pred.idx[k];
      if (d.lane_kind[p] == TS_LANE_CPU_THREAD && d.op_class &&
          d.op_class[p] == TS_OP_LAUNCH) {
        enqueue_ts[i] = d.original_start[p];
        break;
      }
    }
  }
  // per stream lane: kernels sorted by enqueue time with prefix-max chain pos
  std::vector<std::vector<std::pair<int64_t, int32_t>>> enq(nl);
  auto enqueue_index = [&](int32_t l) -> std::vector<std::pair<int64_t, int32_t>>& {
    auto& v = enq[l];
    if (v.empty() && lane_off[l + 1] > lane_off[l]) {
      for (int32_t k = lane_off[l]; k < lane_off[l + 1]; ++k) {
        int32_t t = lane_tasks[k];
        v.emplace_back(enqueue_ts[t], chain_pos[t]);
      }
      std::sort(v.begin(), v.end());
      for (size_t i = 1; i < v.size(); ++i) v[i].second = std::max(v[i].second, v[i - 1].second);
    }
    return v;
  };

  std::vector<int32_t> sync_tasks;
  std::vector<std::vector<CertEntry>> sync_cert;  // per sync task (index into sync_tasks)
  std::vector<std::vector<int32_t>> sync_watch;   // watched stream lanes
  std::vector<int32_t> sync_id(n, -1);
  std::vector<int32_t> event_bound(n, -1);
  for (int32_t t = 0; t < n; ++t) {
    int32_t r = rule_of[t];
    if (r < 0) continue;
    if (d.rule_kind[r] == TS_RULE_EVENT_SYNC) {
      int32_t b = d.rule_bound ? d.rule_bound[r] : -1;
      if (b >= 0) {
        if (b == t) {
          err = "unsupported graph: event sync task " + std::to_string(t) +
                " is bound to itself (the reference deadlocks)";
          return TS_E_UNSUPPORTED;
        }
        event_bound[t] = b;
      }
      continue;
    }
    std::vector<int32_t> watched;
    for (int32_t w = d.rule_watch_off[r]; w < d.rule_watch_off[r + 1]; ++w) {
      int32_t l = lane_index({d.watch_rank[w], d.watch_kind[w], d.watch_lane[w]});
      if (l < 0) continue;  // processor without tasks: ignored (simulate.cpp:183-186)
      if (lanes[l].kind != TS_LANE_CUDA_STREAM || l == lane_of[t]) {
        err = "unsupported graph: sync task " + std::to_string(t) +
              " watches a CPU lane or its own lane; the device path binds syncs to streams";
        return TS_E_UNSUPPORTED;
      }
      watched.push_back(l);
    }
    std::sort(watched.begin(), watched.end());
    watched.erase(std::unique(watched.begin(), watched.end()), watched.end());
    if (watched.empty()) continue;  // no-op rule: plain task
    std::vector<CertEntry> cert;
    for (int32_t l : watched) {
      auto& idx = enqueue_index(l);
      // last (chain order) kernel whose launch precedes the sync (lower_bound
      // on (ts, -1) like build.cpp:426-434)
      auto it = std::lower_bound(idx.begin(), idx.end(),
                                 std::make_pair(d.original_start[t], INT32_MIN));
      int32_t pos = it == idx.begin() ? -1 : std::prev(it)->second;
      CertEntry ce;
      ce.kstar = pos >= 0 ? lane_tasks[lane_off[l] + pos] : -1;
      int32_t np = pos + 1;
      ce.next = np < lane_off[l + 1] - lane_off[l] ? lane_tasks[lane_off[l] + np] : -1;
      cert.push_back(ce);
    }
    sync_id[t] = static_cast<int32_t>(sync_tasks.size());
    sync_tasks.push_back(t);
    sync_cert.push_back(std::move(cert));
    sync_watch.push_back(std::move(watched));
  }
  out.n_syncs = static_cast<int32_t>(sync_tasks.size());

  // ---------------------------------------------------------------- gates
  std::vector<char> split(n, 0);  // task needs a separate START op
  std::vector<std::vector<std::pair<int32_t, uint8_t>>> gates_of;  // per task (sparse)
  std::unordered_map<int32_t, int32_t> gate_slot;
  for (int64_t gi = 0; gi < d.n_gates; ++gi) {
    int32_t u = d.gate_from[gi], v = d.gate_to[gi];
    uint8_t k = d.gate_kind[gi];
    if (u < 0 || u >= n || v < 0 || v >= n || u == v || k > TS_GATE_START) {
      err = "invalid graph: gate " + std::to_string(u) + "->" + std::to_string(v) +
            " references an invalid task";
      return TS_E_SIMULATION;
    }
    auto [it, fresh] = gate_slot.try_emplace(v, static_cast<int32_t>(gates_of.size()));
    if (fresh) gates_of.emplace_back();
    gates_of[it->second].emplace_back(u, k);
    if (k == TS_GATE_START) split[v] = 1;
  }
  if (d.n_gates > 0 && !sync_tasks.empty()) {
    // a failed sync certificate is re-run by the event-driven replay, which
    // has no gates: gated (estimate) graphs express their syncs as edges
    err = "unsupported graph: Stream/DeviceSync rules in a graph with gates";
    return TS_E_UNSUPPORTED;
  }
  for (int32_t t : sync_tasks)
    if (split[t] || gate_slot.count(t)) {
      err = "unsupported graph: sync task " + std::to_string(t) + " carries gates";
      return TS_E_UNSUPPORTED;
    }
  std::vector<int32_t> split_idx(n, -1);
  int32_t n_split = 0;
  for (int32_t i = 0; i < n; ++i)
    if (split[i]) split_idx[i] = n_split++;
  const int64_t na = static_cast<int64_t>(n) + n_split;  // aug nodes
  auto snode = [&](int32_t v) -> int32_t { return split[v] ? n + split_idx[v] : v; };

  // ------------------------------------------------------ augmented graph
  std::vector<std::pair<int32_t, int32_t>> aug;
  aug.reserve(fixed.size() + static_cast<size_t>(n_split) + 16);
  for (const auto& e : fixed) aug.emplace_back(e.first, snode(e.second));
  for (int32_t t = 0; t < n; ++t)
    if (event_bound[t] >= 0) aug.emplace_back(event_bound[t], snode(t));
  for (size_t s = 0; s < sync_tasks.size(); ++s)
    for (const auto& ce : sync_cert[s])
      if (ce.kstar >= 0) aug.emplace_back(ce.kstar, sync_tasks[s]);
  for (const auto& [v, gi] : gate_slot)
    for (const auto& [u, k] : gates_of[gi]) aug.emplace_back(k == TS_GATE_START ? snode(u) : u, v);
  for (int32_t v = 0; v < n; ++v)
    if (split[v]) aug.emplace_back(snode(v), v);

  // topological index (any order) of the augmented graph, for reachability
  std::vector<int32_t> topo(na, -1);
  {
    Csr as = build_csr(na, aug, true);
    std::vector<int32_t> left(na, 0);
    for (const auto& e : aug) left[e.second]++;
    std::vector<int32_t> q;
    q.reserve(na);
    for (int32_t i = 0; i < na; ++i)
      if (left[i] == 0) q.push_back(i);
    for (size_t h = 0; h < q.size(); ++h)
      for (int64_t k = as.begin(q[h]); k < as.end(q[h]); ++k)
        if (--left[as.idx[k]] == 0) q.push_back(as.idx[k]);
    if (static_cast<int64_t>(q.size()) != na) {
      err = "unsupported graph: sync or gate bindings form a cycle (the reference would "
            "deadlock or needs the event-driven path)";
      return TS_E_UNSUPPORTED;
    }
    for (size_t i = 0; i < q.size(); ++i) topo[q[i]] = static_cast<int32_t>(i);
    // certificate successors: keep n_w only when it is not a descendant of s
    std::vector<int32_t> stamp(na, -1);
    std::vector<int32_t> stack;
    int32_t stamp_id = 0;
    for (size_t s = 0; s < sync_tasks.size(); ++s) {
      for (auto& ce : sync_cert[s]) {
        if (ce.next < 0) continue;
        int32_t src = sync_tasks[s], dst = ce.next;
        bool reach = false;
        if (topo[dst] > topo[src]) {
          ++stamp_id;
          stack.assign(1, src);
          stamp[src] = stamp_id;
          while (!stack.empty() && !reach) {
            int32_t x = stack.back();
            stack.pop_back();
            for (int64_t k = as.begin(x); k < as.end(x); ++k) {
              int32_t y = as.idx[k];
              if (y == dst) {
                reach = true;
                break;
              }
              if (stamp[y] != stamp_id && topo[y] < topo[dst]) {
                stamp[y] = stamp_id;
                stack.push_back(y);
              }
            }
          }
        }
        if (reach) ce.next = -1;
      }
    }
  }
  for (size_t s = 0; s < sync_tasks.size(); ++s)
    for (const auto& ce : sync_cert[s])
      if (ce.next >= 0) aug.emplace_back(snode(ce.next), sync_tasks[s]);  // order-only

  // ----------------------------------------------------------- components
  std::vector<int32_t> uf(na);
  std::iota(uf.begin(), uf.end(), 0);
  auto find = [&](int32_t x) {
    while (uf[x] != x) x = uf[x] = uf[uf[x]];
    return x;
  };
  for (const auto& e : aug) {
    int32_t a = find(e.first), b = find(e.second);
    if (a != b) uf[std::max(a, b)] = std::min(a, b);
  }
  // component id ordered by smallest task id
  std::vector<int32_t> comp_of(na, -1);
  std::vector<int32_t> root_comp(na, -1);
  int32_t n_comp = 0;
  for (int32_t v = 0; v < na; ++v) {
    int32_t r = find(v);
    if (root_comp[r] < 0) root_comp[r] = n_comp++;
    comp_of[v] = root_comp[r];
  }

  // watched stream sets of the certified syncs; each stream lane keeps the
  // coverage value of up to kCovSets of the sets it belongs to
  std::vector<std::vector<int32_t>> sets;
  std::vector<int32_t> sync_set(sync_tasks.size(), -1);
  std::vector<std::vector<int32_t>> lane_sets(nl);
  for (size_t s = 0; s < sync_tasks.size(); ++s) {
    bool any = false;
    for (const auto& ce : sync_cert[s]) any = any || ce.kstar >= 0;
    if (!any) continue;
    auto it = std::find(sets.begin(), sets.end(), sync_watch[s]);
    if (it == sets.end()) {
      sets.push_back(sync_watch[s]);
      sync_set[s] = static_cast<int32_t>(sets.size() - 1);
    } else {
      sync_set[s] = static_cast<int32_t>(it - sets.begin());
    }
  }
  for (size_t id = 0; id < sets.size(); ++id)
    for (int32_t l : sets[id])
      if (static_cast<int>(lane_sets[l].size()) < kCovSets)
        lane_sets[l].push_back(static_cast<int32_t>(id));
  auto set_index = [&](int32_t task, int32_t set_id) -> int {
    const auto& v = lane_sets[lane_of[task]];
    for (size_t j = 0; j < v.size(); ++j)
      if (v[j] == set_id) return static_cast<int>(j);
    return -1;
  };

  // values that are read by someone
  std::vector<char> start_used(n, 0);
  for (const auto& [v, gi] : gate_slot)
    for (const auto& [u, k] : gates_of[gi])
      if (k == TS_GATE_START) start_used[u] = 1;
  for (size_t s = 0; s < sync_tasks.size(); ++s)
    for (const auto& ce : sync_cert[s])
      if (ce.next >= 0) start_used[ce.next] = 1;

  // ------------------------------------------- priority topological order
  // key: (component, host task after device task, original_start, id) — a
  // kernel is consumed as soon as it can run, which keeps the live set small.
  Csr as = build_csr(na, aug, true);
  std::vector<int32_t> left(na, 0);
  for (const auto& e : aug) left[e.second]++;
  std::vector<int32_t> split_task(n_split);
  for (int32_t v = 0; v < n; ++v)
    if (split[v]) split_task[split_idx[v]] = v;
  auto real_task = [&](int32_t a) { return a < n ? a : split_task[a - n]; };
  // demand time: a kernel's nominal finish (one longest-path pass at base
  // durations, gates included); a host op inherits the earliest demand of
  // anything downstream, so launches are placed just before the kernels that
  // consume them rather than at their (much earlier) recorded time.  Keying
  // kernels by finish keeps a p2p receive — which starts early and then waits
  // inside its duration — from dragging every earlier launch forward.
  std::vector<int64_t> demand(na, INT64_MAX);
  std::vector<int64_t> comp_path;
  {
    std::vector<int32_t> by_topo(na);
    for (int32_t a = 0; a < na; ++a) by_topo[topo[a]] = a;
    std::vector<int64_t> nstart(n, d.window_start), nfin(n, d.window_start);
    std::vector<std::vector<int32_t>> static_in(n);
    for (size_t si = 0; si < sync_tasks.size(); ++si)
      for (const auto& ce : sync_cert[si])
        if (ce.kstar >= 0) static_in[sync_tasks[si]].push_back(ce.kstar);
    for (int64_t k = 0; k < na; ++k) {
      const int32_t a = by_topo[k];
      const int32_t t = real_task(a);
      if (a >= n || !split[t]) {
        int64_t st = d.window_start;
        for (int64_t e = pred.begin(t); e < pred.end(t); ++e) st = std::max(st, nfin[pred.idx[e]]);
        if (event_bound[t] >= 0) st = std::max(st, nfin[event_bound[t]]);
        for (int32_t u : static_in[t]) st = std::max(st, nfin[u]);
        nstart[t] = st;
      }
      if (a < n) {
        int64_t f = nstart[t];
        auto git = gate_slot.find(t);
        if (git != gate_slot.end())
          for (const auto& [u, kk] : gates_of[git->second])
            f = std::max(f, kk == TS_GATE_START ? nstart[u] : nfin[u]);
        nfin[t] = f + d.duration[t];
      }
    }
    // nominal longest path per component (W-relative): sizes the uint32
    // window of cooperative walks, which also check every addition
    comp_path.assign(n_comp, 0);
    for (int32_t t = 0; t < n; ++t)
      comp_path[comp_of[t]] = std::max(comp_path[comp_of[t]], nfin[t] - d.window_start);
    for (int64_t v : comp_path) out.max_comp_path = std::max(out.max_comp_path, v);

    for (int64_t k = na - 1; k >= 0; --k) {
      const int32_t a = by_topo[k];
      const int32_t t = real_task(a);
      int64_t dm = d.lane_kind[t] == TS_LANE_CUDA_STREAM ? nfin[t] : INT64_MAX;
      for (int64_t e = as.begin(a); e < as.end(a); ++e) dm = std::min(dm, demand[as.idx[e]]);
      demand[a] = dm == INT64_MAX ? nfin[t] : dm;
    }
  }
  using Key = std::tuple<int32_t, int64_t, int32_t, int64_t, int32_t, int32_t>;
  std::priority_queue<Key, std::vector<Key>, std::greater<>> heap;
  auto push = [&](int32_t a) {
    int32_t t = real_task(a);
    int32_t cpu = d.lane_kind[t] == TS_LANE_CUDA_STREAM ? 0 : 1;
    heap.emplace(comp_of[a], demand[a], cpu, d.original_start[t], t, a);
  };
  for (int32_t a = 0; a < na; ++a)
    if (left[a] == 0) push(a);
  std::vector<int32_t> order;
  order.reserve(na);
  while (!heap.empty()) {
    int32_t a = std::get<5>(heap.top());
    heap.pop();
    order.push_back(a);
    for (int64_t k = as.begin(a); k < as.end(a); ++k)
      if (--left[as.idx[k]] == 0) push(as.idx[k]);
  }
  if (static_cast<int64_t>(order.size()) != na) {
    err = "unsupported graph: sync certificates impose a cyclic order";
    return TS_E_UNSUPPORTED;
  }

  // ------------------------------------------------ op emission per component
  // value ids: FIN(v) = v, START(v) = n + v, COV(v, j) = 2n + 2v + j, ACC >= 4n
  const int64_t V_START = n, V_COV = 2LL * n, V_ACC = 4LL * n;
  std::vector<int32_t> last_use(static_cast<size_t>(V_ACC), -1);
  std::vector<int32_t> slot_of(static_cast<size_t>(V_ACC), kNoSlot);
  int64_t acc_next = V_ACC;

  std::vector<int32_t> comp_begin(n_comp + 1, 0);
  for (int32_t a : order) comp_begin[comp_of[a] + 1]++;
  for (int32_t c = 0; c < n_comp; ++c) comp_begin[c + 1] += comp_begin[c];

  std::unordered_map<uint64_t, std::vector<int32_t>> prog_by_hash;
  std::vector<int32_t> prog_rep_base;  // node_base of the component that created each program
  std::vector<IrOp> ir;
  std::vector<int32_t> comp_tasks;
  out.comps.resize(n_comp);
  out.fused.assign(n_comp, FusedDesc{-1, -1});
  out.n_fused = 0;
  out.fused_rows.clear();

  // ---- split breakdown accounting (program.hpp FusedDesc).  Rank rows
  // (ranks_in order, build.cpp:582-590) and stream slots (stream lanes in lane
  // order) are numbered as build_common numbers them.
  std::vector<int32_t> rank_ids(d.rank, d.rank + n);
  std::vector<int32_t> rank_count;
  std::sort(rank_ids.begin(), rank_ids.end());
  {
    std::vector<int32_t> u;
    for (int32_t r : rank_ids) {
      if (u.empty() || u.back() != r) {
        u.push_back(r);
        rank_count.push_back(0);
      }
      rank_count.back()++;
    }
    rank_ids.swap(u);
  }
  std::vector<int32_t> stream_slot(nl, -1);
  std::vector<int8_t> lane_class(nl, -1);  // stream lanes: 0 compute-only, 1 comm-only, 2 mixed
  {
    int32_t k = 0;
    for (int32_t l = 0; l < nl; ++l) {
      if (lanes[l].kind != TS_LANE_CUDA_STREAM) continue;
      stream_slot[l] = k++;
      bool comm = false, comp = false;
      for (int32_t q = lane_off[l]; q < lane_off[l + 1]; ++q)
        (d.op_class && d.op_class[lane_tasks[q]] == TS_OP_COMMUNICATION ? comm : comp) = true;
      lane_class[l] = comm && comp ? 2 : comm ? 1 : 0;
    }
  }
  const char* fuse_env = std::getenv("LUMOS_FUSED_REDUCE");
  const bool fuse_enabled = !(fuse_env && fuse_env[0] == '0');
  std::vector<std::vector<int32_t>> cand_of_row(rank_ids.size());
  std::vector<int32_t> fz_anc, fz_desc;  // per task: last compute ancestor / first descendant (A chain)
  std::vector<char> fz_pos;              // scratch: task seen
  // Split accounting of component c: for every rank of the component whose
  // tasks all lie in it and whose GPU streams are <= 1 compute-only and <= 3
  // comm-only streams, F_BUSY on its compute-stream kernels and its candidate
  // list.  Returns the descriptor per rank of the component (ascending rank;
  // row -1: not fused, K5 sweeps all of its timestamps).  A single-program
  // walk holds one |A| register, so it fuses only one-rank components
  // (multi = false); the cooperative walk holds one per warp = rank.
  auto fuse_accounting = [&](std::vector<IrOp>& ir, bool multi) -> std::vector<FusedDesc> {
    std::vector<int32_t> ranks_here;
    for (int32_t t : comp_tasks) ranks_here.push_back(d.rank[t]);
    std::sort(ranks_here.begin(), ranks_here.end());
    ranks_here.erase(std::unique(ranks_here.begin(), ranks_here.end()), ranks_here.end());
    std::vector<FusedDesc> res(ranks_here.size(), FusedDesc{-1, -1});
    if (!fuse_enabled || comp_tasks.empty() || (!multi && ranks_here.size() != 1)) return res;
    // tasks in op order (topological for every timing edge); a split task
    // (OP_START ... OP_FINISH) is placed at its start
    std::vector<int32_t> topo_tasks;
    std::vector<char> seen_t;
    for (const IrOp& o : ir) {
      if (o.aux() || o.v_dst < 0) continue;
      int64_t t = -1;
      if (o.v_dst < n && (o.op.kind == OP_NODE || o.op.kind == OP_SYNC ||
                          o.op.kind == OP_GATED || o.op.kind == OP_FINISH))
        t = o.v_dst;
      else if (o.op.kind == OP_START && o.v_dst >= V_START && o.v_dst < V_START + n)
        t = o.v_dst - V_START;
      if (t < 0) continue;
      if (fz_pos.size() != static_cast<size_t>(n)) fz_pos.assign(n, 0);
      if (fz_pos[t]) continue;
      fz_pos[t] = 1;
      topo_tasks.push_back(static_cast<int32_t>(t));
    }
    for (int32_t t : topo_tasks) fz_pos[t] = 0;
    if (topo_tasks.size() != comp_tasks.size()) return res;
    // timing predecessors: fixed edges, event-sync bound, static sync bindings
    // (a failed sync certificate sends the scenario to the event-driven path,
    // which reduces it itself).  Gates relate finishes only, so they are left
    // out: fewer comparabilities, more candidates, never a missed overlap.
    auto each_pred = [&](int32_t t, auto&& f) {
      for (int64_t k = pred.begin(t); k < pred.end(t); ++k) f(pred.idx[k]);
      if (event_bound[t] >= 0) f(event_bound[t]);
      if (sync_id[t] >= 0)
        for (const auto& ce : sync_cert[sync_id[t]])
          if (ce.kstar >= 0) f(ce.kstar);
    };
    if (fz_anc.empty()) {
      fz_anc.assign(n, -1);
      fz_desc.assign(n, INT32_MAX);
    }
    for (size_t k = 0; k < ranks_here.size(); ++k) {
      const int32_t r = ranks_here[k];
      const int32_t row = static_cast<int32_t>(
          std::lower_bound(rank_ids.begin(), rank_ids.end(), r) - rank_ids.begin());
      int32_t in_comp = 0;
      for (int32_t t : comp_tasks) in_comp += d.rank[t] == r;
      if (rank_count[row] != in_comp) continue;
      int32_t lane_a = -1;
      std::vector<int32_t> comm_lanes;
      bool ok = true;
      auto lo = std::lower_bound(lanes.begin(), lanes.end(), Proc{r, TS_LANE_CUDA_STREAM, INT32_MIN});
      for (auto it = lo; it != lanes.end() && it->rank == r && it->kind == TS_LANE_CUDA_STREAM; ++it) {
        const int32_t l = static_cast<int32_t>(it - lanes.begin());
        if (lane_class[l] == 0 && lane_a < 0) lane_a = l;
        else if (lane_class[l] == 1) comm_lanes.push_back(l);
        else ok = false;
      }
      if (!ok || static_cast<int>(comm_lanes.size()) > kFusedMaxComm) continue;
      const int32_t len_a = lane_a < 0 ? 0 : lane_off[lane_a + 1] - lane_off[lane_a];
      auto apos = [&](int32_t t) { return lane_of[t] == lane_a ? chain_pos[t] : -1; };
      for (int32_t t : topo_tasks)
        each_pred(t, [&](int32_t p) { fz_anc[t] = std::max({fz_anc[t], fz_anc[p], apos(p)}); });
      for (size_t q = topo_tasks.size(); q-- > 0;) {
        const int32_t t = topo_tasks[q];
        const int32_t at = apos(t) < 0 ? INT32_MAX : apos(t);
        each_pred(t, [&](int32_t p) { fz_desc[p] = std::min({fz_desc[p], fz_desc[t], at}); });
      }
      // candidates: A positions in (anc(c), desc(c)) for some comm kernel c
      std::vector<char> cand(static_cast<size_t>(len_a), 0);
      for (int32_t l : comm_lanes)
        for (int32_t q = lane_off[l]; q < lane_off[l + 1]; ++q) {
          const int32_t cm = lane_tasks[q];
          for (int32_t j = fz_anc[cm] + 1; j < std::min(fz_desc[cm], len_a); ++j) cand[j] = 1;
        }
      for (int32_t t : comp_tasks) {
        fz_anc[t] = -1;
        fz_desc[t] = INT32_MAX;
      }
      auto& list = cand_of_row[row];
      list.clear();
      for (int32_t j = 0; j < len_a; ++j)
        if (cand[j]) list.push_back(lane_tasks[lane_off[lane_a] + j]);
      for (IrOp& o : ir)
        if (!o.aux() && o.v_dst >= 0 && o.v_dst < n && lane_of[o.v_dst] == lane_a &&
            (o.op.kind == OP_NODE || o.op.kind == OP_GATED || o.op.kind == OP_FINISH))
          o.op.flags |= F_BUSY;
      res[k] = FusedDesc{row, lane_a >= 0 ? stream_slot[lane_a] : -1};
      out.fused_rows.push_back(res[k]);
    }
    return res;
  };

  auto fold = [&](std::vector<int64_t>& vals, size_t room) {
    std::vector<int64_t> u;
    for (int64_t v : vals)
      if (std::find(u.begin(), u.end(), v) == u.end()) u.push_back(v);
    vals.swap(u);
    while (vals.size() > room) {
      size_t take = std::min<size_t>(4, vals.size());
      IrOp acc;
      acc.op.kind = OP_ACC;
      acc.op.node = -1;
      acc.op.flags = F_NO_OUT;
      acc.op.npred = static_cast<uint8_t>(take);
      for (size_t i = 0; i < take; ++i) acc.v_pred[i] = vals[i];
      int64_t av = acc_next++;
      acc.v_dst = av;
      ir.push_back(acc);
      vals.erase(vals.begin(), vals.begin() + static_cast<long>(take));
      vals.insert(vals.begin(), av);
    }
  };

  // cooperative multi-rank walks (LUMOS_COOP=0 disables them)
  const char* coop_env = std::getenv("LUMOS_COOP");
  const bool coop = allow_coop && !(coop_env && coop_env[0] == '0');
  out.coop_prog_off.clear();
  out.coop_progs.clear();
  out.coop_rows.clear();
  out.fused_rows.clear();
  out.max_mailboxes = 0;
  out.max_coop_ranks = 1;
  out.max_coop_path = 0;
  for (int32_t c = 0; c < n_comp; ++c) {
    ir.clear();
    comp_tasks.clear();
    for (int32_t i = comp_begin[c]; i < comp_begin[c + 1]; ++i)
      if (order[i] < n) comp_tasks.push_back(order[i]);
    int32_t tmin = *std::min_element(comp_tasks.begin(), comp_tasks.end());
    int32_t tmax = *std::max_element(comp_tasks.begin(), comp_tasks.end());
    bool contiguous = tmax - tmin + 1 == static_cast<int32_t>(comp_tasks.size());
    int32_t node_base = contiguous ? tmin : 0;

    for (int32_t i = comp_begin[c]; i < comp_begin[c + 1]; ++i) {
      int32_t a = order[i];
      int32_t t = real_task(a);
      bool is_start_node = a >= n;
      bool gpu = d.lane_kind[t] == TS_LANE_CUDA_STREAM;
      const auto& my_sets = lane_sets[lane_of[t]];
      bool tracked = gpu && !my_sets.empty();
      uint8_t cls = d.scale_class ? d.scale_class[t]
                                  : static_cast<uint8_t>(d.task_kind && d.task_kind[t]
                                                             ? (d.op_class && d.op_class[t] ==
                                                                        TS_OP_COMMUNICATION
                                                                    ? 2
                                                                    : 1)
                                                             : 0);
      if (cls >= kMaxClasses) {
        err = "scale_class must be < " + std::to_string(kMaxClasses);
        return TS_E_INVALID_ARGUMENT;
      }
      uint8_t flags = d.op_class && d.op_class[t] == TS_OP_COMMUNICATION ? F_COMM : 0;

      // fixed predecessors (+ event-sync bound)
      std::vector<int64_t> fixedv;
      for (int64_t k = pred.begin(t); k < pred.end(t); ++k) fixedv.push_back(pred.idx[k]);
      if (event_bound[t] >= 0) fixedv.push_back(event_bound[t]);

      // coverage record following a tracked op (sources: kernel preds on the
      // same watched set)
      auto push_with_cov = [&](IrOp& o) {
        if (!tracked) {
          ir.push_back(o);
          return;
        }
        IrOp cv;
        cv.is_cov = true;
        cv.n_sets = static_cast<int>(my_sets.size());
        int n_src = 0, src_k = -1;
        const int n_cand = o.op.kind == OP_GATED ? (o.op.cls >> 4) : o.op.npred;
        for (int j = 0; j < cv.n_sets; ++j) {
          cv.v_cov_dst[j] = V_COV + 2LL * t + j;
          for (int k = 0; k < o.op.npred; ++k) {
            int64_t v = o.v_pred[k];
            if (v < 0 || v >= n) continue;  // not a task finish (ACC / START value)
            int32_t u = static_cast<int32_t>(v);
            if (d.lane_kind[u] != TS_LANE_CUDA_STREAM) continue;
            int ju = set_index(u, my_sets[j]);
            if (ju >= 0) {
              cv.v_cov_src[j][k] = V_COV + 2LL * u + ju;
              ++n_src;
              src_k = k;
            }
          }
        }
        if (cv.n_sets == 1 && n_src <= 1 && (src_k < 0 || src_k < n_cand)) {
          // compact form: the single source becomes pred[0]
          o.op.flags |= F_TRACK1;
          if (src_k > 0) {
            std::swap(o.v_pred[0], o.v_pred[src_k]);
            std::swap(cv.v_cov_src[0][0], cv.v_cov_src[0][src_k]);
          }
          o.v_cov1_src = cv.v_cov_src[0][0];
          o.v_cov1_dst = cv.v_cov_dst[0];
          ir.push_back(o);
          return;
        }
        o.op.flags |= F_TRACK;
        ir.push_back(o);
        ir.push_back(cv);
      };

      if (is_start_node) {
        fold(fixedv, 4);
        IrOp o;
        o.op.kind = OP_START;
        o.op.node = t - node_base;
        o.op.flags = static_cast<uint8_t>(flags | F_NO_OUT);
        o.op.cls = cls;
        o.op.npred = static_cast<uint8_t>(fixedv.size());
        for (size_t k = 0; k < fixedv.size(); ++k) o.v_pred[k] = fixedv[k];
        o.v_dst = V_START + t;
        push_with_cov(o);
        continue;
      }

      auto git = gate_slot.find(t);
      std::vector<int64_t> gatev;
      if (git != gate_slot.end())
        for (const auto& [u, k] : gates_of[git->second])
          gatev.push_back(k == TS_GATE_START ? V_START + u : u);

      IrOp o;
      o.op.node = t - node_base;
      o.op.base = d.duration[t];
      o.op.flags = flags;
      if (d.rt_kind && rt_walk_kind(d.rt_kind[t])) o.op.flags |= F_RT;
      o.v_dst = t;
      if (split[t]) {
        fold(gatev, 3);
        o.op.kind = OP_FINISH;
        o.op.cls = cls;
        o.op.npred = static_cast<uint8_t>(1 + gatev.size());
        o.v_pred[0] = V_START + t;
        for (size_t k = 0; k < gatev.size(); ++k) o.v_pred[1 + k] = gatev[k];
        ir.push_back(o);
        continue;
      }
      if (start_used[t]) {
        o.op.flags |= F_STORE_START;
        o.v_x2 = V_START + t;
      }
      if (!gatev.empty()) {
        if (gatev.size() > 1 && fixedv.size() + gatev.size() > 4) fold(gatev, 1);
        fold(fixedv, 4 - gatev.size());
        o.op.kind = OP_GATED;
        o.op.cls = static_cast<uint8_t>(cls | (fixedv.size() << 4));
        o.op.npred = static_cast<uint8_t>(fixedv.size() + gatev.size());
        for (size_t k = 0; k < fixedv.size(); ++k) o.v_pred[k] = fixedv[k];
        for (size_t k = 0; k < gatev.size(); ++k) o.v_pred[fixedv.size() + k] = gatev[k];
        push_with_cov(o);
        continue;
      }
      fold(fixedv, 4);
      o.op.cls = cls;
      o.op.npred = static_cast<uint8_t>(fixedv.size());
      for (size_t k = 0; k < fixedv.size(); ++k) o.v_pred[k] = fixedv[k];
      if (sync_id[t] < 0) {
        o.op.kind = OP_NODE;
        push_with_cov(o);
        continue;
      }
      o.op.kind = OP_SYNC;
      const int32_t sid = sync_id[t];
      const auto& cert = sync_cert[sid];
      int32_t n_ext = static_cast<int32_t>((cert.size() + kCertPerExt - 1) / kCertPerExt);
      o.op.x0 = static_cast<uint16_t>(n_ext);
      ir.push_back(o);
      for (int32_t e = 0; e < n_ext; ++e) {
        IrOp x;
        x.is_ext = true;
        for (int32_t k = 0; k < kCertPerExt; ++k) {
          size_t j = static_cast<size_t>(e) * kCertPerExt + k;
          if (j >= cert.size()) break;
          const int32_t ks = cert[j].kstar;
          x.v_fin[k] = ks >= 0 ? ks : -1;
          int ji = (ks >= 0 && sync_set[sid] >= 0) ? set_index(ks, sync_set[sid]) : -1;
          x.v_bs[k] = ji >= 0 ? V_COV + 2LL * ks + ji : -1;
          x.v_next[k] = cert[j].next >= 0 ? V_START + cert[j].next : -1;
          x.n_ent = k + 1;
        }
        ir.push_back(x);
      }
    }

    // ---- one straight-line program from an op sequence: liveness, slots,
    // byte offsets, chunk padding, de-duplication.  Returns the program id,
    // or -1 with finish_rc / err set.
    int finish_rc = TS_OK;
    auto finish_program = [&](std::vector<IrOp>& ir, int32_t& n_slots_out) -> int32_t {
      // ---- liveness: last use of each value; auxiliary records (certificate,
      // coverage) belong to the op before them
      auto ensure = [&](int64_t v) {
        if (v >= static_cast<int64_t>(last_use.size())) {
          last_use.resize(static_cast<size_t>(v + 1), -1);
          slot_of.resize(static_cast<size_t>(v + 1), kNoSlot);
        }
      };
      std::vector<int32_t> anchor(ir.size());
      for (size_t i = 0; i < ir.size(); ++i)
        anchor[i] = ir[i].aux() ? anchor[i - 1] : static_cast<int32_t>(i);
      auto each_read = [&](const IrOp& o, auto&& f) {
        if (o.is_ext) {
          for (int k = 0; k < o.n_ent; ++k) {
            if (o.v_fin[k] >= 0) f(o.v_fin[k]);
            if (o.v_bs[k] >= 0) f(o.v_bs[k]);
            if (o.v_next[k] >= 0) f(o.v_next[k]);
          }
          return;
        }
        if (o.is_cov) {
          for (int j = 0; j < o.n_sets; ++j)
            for (int k = 0; k < 4; ++k)
              if (o.v_cov_src[j][k] >= 0) f(o.v_cov_src[j][k]);
          return;
        }
        for (int k = 0; k < o.op.npred; ++k) f(o.v_pred[k]);
        if (o.v_cov1_src >= 0) f(o.v_cov1_src);
      };
      auto each_write = [&](const IrOp& o, auto&& f) {
        if (o.is_ext) return;
        if (o.is_cov) {
          for (int j = 0; j < o.n_sets; ++j)
            if (o.v_cov_dst[j] >= 0) f(o.v_cov_dst[j]);
          return;
        }
        if (o.v_dst >= 0) f(o.v_dst);
        if ((o.op.flags & F_STORE_START) && o.v_x2 >= 0) f(o.v_x2);
        if (o.v_cov1_dst >= 0) f(o.v_cov1_dst);
      };
      for (size_t i = 0; i < ir.size(); ++i)
        each_read(ir[i], [&](int64_t v) {
          ensure(v);
          last_use[v] = std::max(last_use[v], anchor[i]);
        });

      // ---- linear-scan slot assignment.  An op group (op + its auxiliary
      // records) reads every operand before it writes.  Operands dying in the
      // group are released at the group's end; the op's own results are placed
      // before that (so they never alias a group operand), the coverage results
      // after it.
      std::priority_queue<int32_t, std::vector<int32_t>, std::greater<>> free_slots;
      int32_t n_slots = kFirstSlot;
      std::vector<int64_t> dying;
      bool broken = false;
      auto flush = [&] {
        std::sort(dying.begin(), dying.end());
        dying.erase(std::unique(dying.begin(), dying.end()), dying.end());
        for (int64_t v : dying) {
          free_slots.push(slot_of[v]);
          slot_of[v] = kNoSlot;
        }
        dying.clear();
      };
      for (size_t i = 0; i < ir.size(); ++i) {
        IrOp& o = ir[i];
        const int32_t at = anchor[i];
        auto read_slot = [&](int64_t v) -> uint16_t {
          if (v < 0) return kNoSlot;
          if (slot_of[v] == kNoSlot) {
            broken = true;
            return kNoSlot;
          }
          if (last_use[v] == at) dying.push_back(v);
          return static_cast<uint16_t>(slot_of[v]);
        };
        auto write_slot = [&](int64_t v) -> uint16_t {
          if (v < 0) return kSlotTrash;
          ensure(v);
          if (last_use[v] <= at) return kSlotTrash;  // nobody reads it later
          int32_t s;
          if (!free_slots.empty()) {
            s = free_slots.top();
            free_slots.pop();
          } else {
            s = n_slots++;
          }
          slot_of[v] = s;
          return static_cast<uint16_t>(s);
        };
        const bool group_end = i + 1 >= ir.size() || !ir[i + 1].aux();
        if (o.is_ext) {
          OpExt x{};
          for (int k = 0; k < kCertPerExt; ++k) x.fin[k] = x.bs[k] = x.next[k] = kNoSlot;
          for (int k = 0; k < o.n_ent; ++k) {
            x.fin[k] = read_slot(o.v_fin[k]);
            x.bs[k] = read_slot(o.v_bs[k]);
            x.next[k] = read_slot(o.v_next[k]);
          }
          x.n = static_cast<uint16_t>(o.n_ent);
          std::memcpy(&o.op, &x, sizeof(Op));
          if (group_end) flush();
          continue;
        }
        if (o.is_cov) {
          OpCov x{};
          for (int j = 0; j < kCovSets; ++j) {
            x.dst[j] = kNoSlot;
            for (int k = 0; k < 4; ++k) x.src[j][k] = kNoSlot;
          }
          for (int j = 0; j < o.n_sets; ++j)
            for (int k = 0; k < 4; ++k) x.src[j][k] = read_slot(o.v_cov_src[j][k]);
          if (group_end) flush();
          for (int j = 0; j < o.n_sets; ++j) x.dst[j] = write_slot(o.v_cov_dst[j]);
          for (int j = o.n_sets; j < kCovSets; ++j) x.dst[j] = kSlotTrash;
          x.n_sets = static_cast<uint16_t>(o.n_sets);
          std::memcpy(&o.op, &x, sizeof(Op));
          continue;
        }
        for (int k = 0; k < o.op.npred; ++k) o.op.pred[k] = read_slot(o.v_pred[k]);
        for (int k = o.op.npred; k < 4; ++k) o.op.pred[k] = kSlotOrigin;
        const uint16_t cov_src = (o.op.flags & F_TRACK1) ? read_slot(o.v_cov1_src) : kNoSlot;
        // the walk reads an F_TRACK1 coverage source after writing the op's
        // results, so a dying source is released only after they are placed
        int64_t late_free = -1;
        if ((o.op.flags & F_TRACK1) && o.v_cov1_src >= 0 &&
            std::find(dying.begin(), dying.end(), o.v_cov1_src) != dying.end()) {
          dying.erase(std::remove(dying.begin(), dying.end(), o.v_cov1_src), dying.end());
          late_free = o.v_cov1_src;
        }
        if (group_end) flush();
        ensure(o.v_dst >= 0 ? o.v_dst : 0);
        if (o.v_dst >= 0 && o.v_dst < V_ACC && last_use[o.v_dst] <= at &&
            (o.op.kind == OP_NODE || o.op.kind == OP_GATED || o.op.kind == OP_FINISH ||
             o.op.kind == OP_SYNC))
          o.op.flags |= F_SINK;
        o.op.dst = write_slot(o.v_dst);
        if (o.op.kind != OP_SYNC) o.op.x0 = kNoSlot;
        o.op.x1 = kNoSlot;
        if (o.op.flags & F_TRACK1) {
          o.op.x0 = cov_src == kNoSlot ? kSlotInf : cov_src;
          o.op.x1 = write_slot(o.v_cov1_dst);
        }
        o.op.x2 = (o.op.flags & F_STORE_START) ? write_slot(o.v_x2) : kNoSlot;
        if (o.op.kind == OP_POST || o.op.kind == OP_WAIT)
          o.op.x1 = static_cast<uint16_t>(o.v_x1);  // mailbox id, not a slot
        if (late_free >= 0) {
          free_slots.push(slot_of[late_free]);
          slot_of[late_free] = kNoSlot;
        }
      }
      if (std::getenv("LUMOS_DEBUG_SLOTS") && c == 0) {
        // replay the allocation to find the peak live set (debug only)
        std::vector<int64_t> live;
        std::vector<int64_t> peak;
        std::vector<char> alive(last_use.size(), 0);
        for (size_t i = 0; i < ir.size(); ++i) {
          each_write(ir[i], [&](int64_t v) {
            if (last_use[v] > anchor[i]) alive[v] = 1, live.push_back(v);
          });
          live.erase(std::remove_if(live.begin(), live.end(),
                                    [&](int64_t v) { return last_use[v] <= anchor[i]; }),
                     live.end());
          if (live.size() > peak.size()) peak = live;
        }
        int kinds[5] = {0, 0, 0, 0, 0};
        std::map<std::string, int> by;
        for (int64_t v : peak) {
          int k = v < n ? 0 : v < V_COV ? 1 : v < V_ACC ? 2 : 3;
          kinds[k]++;
          if (k <= 1) {
            int32_t t = static_cast<int32_t>(k == 0 ? v : v - n);
            std::string key = std::string(k ? "START " : "FIN ") +
                              (d.lane_kind[t] ? "stream" : "thread") + std::to_string(d.lane[t]) +
                              " op" + std::to_string(d.op_class ? d.op_class[t] : 9);
            by[key]++;
          }
        }
        fprintf(stderr, "[slots] comp 0 peak %zu: fin %d start %d cov %d acc %d\n", peak.size(),
                kinds[0], kinds[1], kinds[2], kinds[3]);
        for (auto& [k, cnt] : by) fprintf(stderr, "[slots]   %s x%d\n", k.c_str(), cnt);
      }
      if (broken) {
        err = "internal: compiled order reads a value before it is defined";
        {
              finish_rc = TS_E_UNSUPPORTED;
              return -1;
            }
      }
      if (n_slots > kMaxSlots) {
        err = "unsupported graph: a component needs " + std::to_string(n_slots) +
              " live values per scenario (limit " + std::to_string(kMaxSlots) + ")";
        {
              finish_rc = TS_E_UNSUPPORTED;
              return -1;
            }
      }
      // slot numbers -> byte offsets into the [slot][thread] table
      {
        auto off = [](uint16_t& s) {
          if (s != kNoSlot) s = slot_off(s);
        };
        for (IrOp& o : ir) {
          if (o.is_ext) {
            OpExt x;
            std::memcpy(&x, &o.op, sizeof(x));
            for (int k = 0; k < kCertPerExt; ++k) {
              off(x.fin[k]);
              off(x.bs[k]);
              off(x.next[k]);
            }
            std::memcpy(&o.op, &x, sizeof(x));
          } else if (o.is_cov) {
            OpCov x;
            std::memcpy(&x, &o.op, sizeof(x));
            for (int j = 0; j < kCovSets; ++j) {
              off(x.dst[j]);
              for (int k = 0; k < 4; ++k) off(x.src[j][k]);
            }
            std::memcpy(&o.op, &x, sizeof(x));
          } else {
            for (int k = 0; k < 4; ++k) off(o.op.pred[k]);
            off(o.op.dst);
            if (o.op.kind != OP_SYNC) off(o.op.x0);
            if (o.op.kind != OP_POST && o.op.kind != OP_WAIT) off(o.op.x1);
            off(o.op.x2);
          }
        }
      }
      // reset per-value state touched by this component (keeps arrays reusable)
      for (const IrOp& o : ir) {
        each_read(o, [&](int64_t v) {
          last_use[v] = -1;
          slot_of[v] = kNoSlot;
        });
        each_write(o, [&](int64_t v) {
          if (v < static_cast<int64_t>(last_use.size())) {
            last_use[v] = -1;
            slot_of[v] = kNoSlot;
          }
        });
      }

      // ---- pad so that no op group straddles a kChunk boundary
      {
        std::vector<IrOp> padded;
        padded.reserve(ir.size() + ir.size() / 16 + 8);
        size_t i = 0;
        while (i < ir.size()) {
          size_t g = 1;
          while (i + g < ir.size() && ir[i + g].aux()) ++g;
          if (g > static_cast<size_t>(kChunk)) {
            err = "unsupported graph: op group larger than a program chunk";
            {
              finish_rc = TS_E_UNSUPPORTED;
              return -1;
            }
          }
          size_t pos = padded.size() % kChunk;
          if (pos + g > static_cast<size_t>(kChunk)) {
            for (size_t k = pos; k < static_cast<size_t>(kChunk); ++k) {
              IrOp nop;
              nop.op.kind = OP_NOP;
              nop.op.node = -1;
              nop.op.flags = F_NO_OUT;
              for (int q = 0; q < 4; ++q) nop.op.pred[q] = slot_off(kSlotOrigin);
              nop.op.dst = slot_off(kSlotTrash);
              nop.op.x0 = nop.op.x1 = nop.op.x2 = kNoSlot;
              padded.push_back(nop);
            }
          }
          for (size_t k = 0; k < g; ++k) padded.push_back(ir[i + k]);
          i += g;
        }
        ir.swap(padded);
      }

      // ---- de-duplicate identical programs (TP / DP replicas of one stage)
      uint64_t h = 1469598103934665603ull;
      const unsigned char* bytes = reinterpret_cast<const unsigned char*>(ir.data());
      (void)bytes;
      for (const IrOp& o : ir) {
        const unsigned char* p = reinterpret_cast<const unsigned char*>(&o.op);
        for (size_t k = 0; k < sizeof(Op); ++k) h = (h ^ p[k]) * 1099511628211ull;
      }
      h ^= static_cast<uint64_t>(n_slots) * 0x9E3779B97F4A7C15ull;
      int32_t prog = -1;
      if (contiguous) {
        for (int32_t cand : prog_by_hash[h]) {
          const ProgramDesc& pd = out.programs[cand];
          if (pd.n_ops != static_cast<int32_t>(ir.size()) || pd.n_slots != n_slots) continue;
          bool same = true;
          for (size_t k = 0; k < ir.size() && same; ++k)
            same = std::memcmp(&out.ops[pd.op_offset + k], &ir[k].op, sizeof(Op)) == 0;
          // a retime walk reads the creator's task metadata for a shared program
          for (size_t k = 0; k < ir.size() && same; ++k)
            if (!ir[k].aux() && (ir[k].op.flags & F_RT))
              same = same_rt_meta(d, prog_rep_base[cand] + ir[k].op.node, node_base + ir[k].op.node);
          if (same) {
            prog = cand;
            break;
          }
        }
      }
      if (prog < 0) {
        prog = static_cast<int32_t>(out.programs.size());
        ProgramDesc pd;
        pd.op_offset = static_cast<int64_t>(out.ops.size());
        pd.n_ops = static_cast<int32_t>(ir.size());
        pd.n_slots = n_slots;
        out.programs.push_back(pd);
        prog_rep_base.push_back(node_base);
        for (const IrOp& o : ir) out.ops.push_back(o.op);
        if (contiguous) prog_by_hash[h].push_back(prog);
      }
      n_slots_out = n_slots;
      return prog;
    };

    // ---- cooperative components (several ranks coupled by gates, estimate
    // mode): one program per rank, in the component's order restricted to the
    // rank; a value one rank produces and another reads travels through a
    // shared-memory mailbox (OP_POST after its producer, OP_WAIT before its
    // first reader in the other rank).  Restrictions of one topological order
    // cannot wait on each other in a cycle, so the warps always progress.
    std::vector<int32_t> rank_local;  // per op: index of its rank in the component
    int32_t n_local = 1;
    if (coop) {
      std::vector<int32_t> comp_ranks;
      for (int32_t t : comp_tasks) comp_ranks.push_back(d.rank[t]);
      std::sort(comp_ranks.begin(), comp_ranks.end());
      comp_ranks.erase(std::unique(comp_ranks.begin(), comp_ranks.end()), comp_ranks.end());
      n_local = static_cast<int32_t>(comp_ranks.size());
    }
    std::vector<int32_t> progs_of_comp;
    int32_t n_slots = 0;
    std::vector<FusedDesc> coop_fd;  // per rank program of a split component
    size_t coop_mark = 0;
    bool split = coop && n_local > 1 && n_local <= 32;
    if (split) {
      std::vector<int32_t> comp_ranks;
      for (int32_t t : comp_tasks) comp_ranks.push_back(d.rank[t]);
      std::sort(comp_ranks.begin(), comp_ranks.end());
      comp_ranks.erase(std::unique(comp_ranks.begin(), comp_ranks.end()), comp_ranks.end());
      auto local_of = [&](int32_t rank) {
        return static_cast<int32_t>(std::lower_bound(comp_ranks.begin(), comp_ranks.end(), rank) -
                                    comp_ranks.begin());
      };
      // split accounting per rank (one |A| register per warp); rolled back if
      // the component ends up walked as one program
      coop_mark = out.fused_rows.size();
      coop_fd = fuse_accounting(ir, true);
      // rank of every op: a task's rank; a fold (ACC) op takes its consumer's;
      // auxiliary records their op's
      rank_local.assign(ir.size(), -1);
      for (size_t i = 0; i < ir.size(); ++i)
        if (!ir[i].aux() && ir[i].op.kind != OP_ACC && ir[i].op.node >= 0)
          rank_local[i] = local_of(d.rank[node_base + ir[i].op.node]);
      for (size_t i = ir.size(); i-- > 0;)
        if (rank_local[i] < 0 && !ir[i].aux())
          rank_local[i] = i + 1 < ir.size() ? rank_local[i + 1] : 0;
      for (size_t i = 0; i < ir.size(); ++i)
        if (ir[i].aux()) rank_local[i] = rank_local[i - 1];
      // producers, and the values other ranks read
      std::unordered_map<int64_t, int32_t> producer;
      auto writes_of = [&](const IrOp& o, auto&& f) {
        if (o.is_ext) return;
        if (o.is_cov) {
          for (int j = 0; j < o.n_sets; ++j)
            if (o.v_cov_dst[j] >= 0) f(o.v_cov_dst[j]);
          return;
        }
        if (o.v_dst >= 0) f(o.v_dst);
        if ((o.op.flags & F_STORE_START) && o.v_x2 >= 0) f(o.v_x2);
        if (o.v_cov1_dst >= 0) f(o.v_cov1_dst);
      };
      auto reads_of = [&](IrOp& o, auto&& f) {  // f(int64_t& value)
        if (o.is_ext) {
          for (int k = 0; k < o.n_ent; ++k) {
            if (o.v_fin[k] >= 0) f(o.v_fin[k]);
            if (o.v_bs[k] >= 0) f(o.v_bs[k]);
            if (o.v_next[k] >= 0) f(o.v_next[k]);
          }
          return;
        }
        if (o.is_cov) {
          for (int j = 0; j < o.n_sets; ++j)
            for (int k = 0; k < 4; ++k)
              if (o.v_cov_src[j][k] >= 0) f(o.v_cov_src[j][k]);
          return;
        }
        for (int k = 0; k < o.op.npred; ++k) f(o.v_pred[k]);
        if (o.v_cov1_src >= 0) f(o.v_cov1_src);
      };
      for (size_t i = 0; i < ir.size(); ++i)
        writes_of(ir[i], [&](int64_t v) { producer[v] = rank_local[i]; });
      std::unordered_map<int64_t, int32_t> mailbox;  // value -> mailbox id
      for (size_t i = 0; i < ir.size(); ++i)
        reads_of(ir[i], [&](int64_t& v) {
          auto it = producer.find(v);
          if (it != producer.end() && it->second != rank_local[i] && !mailbox.count(v)) {
            const int32_t m = static_cast<int32_t>(mailbox.size());
            mailbox.emplace(v, m);
          }
        });
      if (mailbox.size() > 0xFFFF) {
        err = "unsupported graph: too many cross-rank values in one component";
        return TS_E_UNSUPPORTED;
      }
      // per-rank streams: WAITs before a group's first cross read, the group,
      // POSTs after a group's mailbox values
      std::vector<std::vector<IrOp>> streams(n_local);
      std::vector<std::unordered_map<int64_t, int64_t>> local_copy(n_local);
      size_t i = 0;
      while (i < ir.size()) {
        size_t g = 1;
        while (i + g < ir.size() && ir[i + g].aux()) ++g;
        const int32_t r = rank_local[i];
        auto& st = streams[r];
        std::vector<IrOp> grp(ir.begin() + static_cast<long>(i), ir.begin() + static_cast<long>(i + g));
        for (IrOp& op : grp)
          reads_of(op, [&](int64_t& v) {
            auto mb = mailbox.find(v);
            if (mb == mailbox.end() || producer[v] == r) return;
            auto lc = local_copy[r].find(v);
            if (lc == local_copy[r].end()) {
              IrOp w;
              w.op.kind = OP_WAIT;
              w.op.node = -1;
              w.op.flags = F_NO_OUT;
              w.op.npred = 0;
              w.op.x1 = static_cast<uint16_t>(mb->second);
              w.v_dst = acc_next++;
              w.v_x1 = mb->second;
              st.push_back(w);
              lc = local_copy[r].emplace(v, w.v_dst).first;
            }
            v = lc->second;
          });
        for (IrOp& op : grp) st.push_back(op);
        for (size_t k = i; k < i + g; ++k)
          writes_of(ir[k], [&](int64_t v) {
            auto mb = mailbox.find(v);
            if (mb == mailbox.end()) return;
            IrOp pst;
            pst.op.kind = OP_POST;
            pst.op.node = -1;
            pst.op.flags = F_NO_OUT;
            pst.op.npred = 1;
            pst.v_pred[0] = v;
            pst.v_x1 = mb->second;
            st.push_back(pst);
          });
        i += g;
      }
      for (int32_t r = 0; r < n_local; ++r) {
        int32_t ns = 0;
        const int32_t prog = finish_program(streams[r], ns);
        if (prog < 0) return finish_rc;
        progs_of_comp.push_back(prog);
        n_slots = std::max(n_slots, ns);
      }
      // one CTA must hold the mailboxes and every rank's slot table (int64
      // values, the wider case); otherwise walk the component as one program
      const size_t smem64 = mailbox.size() * 4 + 16 + mailbox.size() * 32 * 8 +
                            static_cast<size_t>(n_local) * n_slots * 32 * 8;
      if (smem64 > 220 * 1024) {
        split = false;  // the rank programs stay in the table, unused
        progs_of_comp.clear();
        for (size_t q = coop_mark; q < out.fused_rows.size(); ++q)
          cand_of_row[out.fused_rows[q].row].clear();
        out.fused_rows.resize(coop_mark);
        coop_fd.clear();
        for (IrOp& o : ir) o.op.flags &= static_cast<uint8_t>(~F_BUSY);
      } else {
        out.max_slots = std::max(out.max_slots, n_slots);
        out.max_coop_path = std::max(out.max_coop_path, comp_path[c]);
        out.max_mailboxes = std::max(out.max_mailboxes, static_cast<int32_t>(mailbox.size()));
        out.max_coop_ranks = std::max(out.max_coop_ranks, n_local);
      }
    }
    if (!split) {
      n_slots = 0;
      const std::vector<FusedDesc> fd = fuse_accounting(ir, false);
      if (fd.size() == 1 && fd[0].row >= 0) {
        out.fused[c] = fd[0];
        out.n_fused++;
      }
      const int32_t prog = finish_program(ir, n_slots);
      if (prog < 0) return finish_rc;
      progs_of_comp.push_back(prog);
      out.max_slots = std::max(out.max_slots, n_slots);
    }
    const int32_t prog = progs_of_comp[0];
    out.coop_prog_off.push_back(static_cast<int32_t>(out.coop_progs.size()));
    for (size_t k = 0; k < progs_of_comp.size(); ++k) {
      out.coop_progs.push_back(progs_of_comp[k]);
      out.coop_rows.push_back(split && k < coop_fd.size() ? coop_fd[k].row : -1);
    }
    {
      int64_t sum = 0;
      for (int32_t t : comp_tasks) {
        const int64_t dt = d.duration[t] > 0 ? d.duration[t] : 0;
        sum = sum > INT64_MAX - dt ? INT64_MAX : sum + dt;
      }
      out.max_comp_dur_sum = std::max(out.max_comp_dur_sum, sum);
      out.max_comp_tasks = std::max(out.max_comp_tasks, static_cast<int32_t>(comp_tasks.size()));
    }
    out.comps[c] = ComponentDesc{prog, node_base, static_cast<int32_t>(comp_tasks.size()), 0};
  }
  out.coop_prog_off.push_back(static_cast<int32_t>(out.coop_progs.size()));
  if (std::getenv("LUMOS_DEBUG_OPS")) {  // op mix of the programs (debug only)
    std::map<std::pair<int, int>, int64_t> mix;
    for (const Op& o : out.ops) mix[{o.kind, o.flags & (F_TRACK | F_TRACK1 | F_STORE_START)}]++;
    for (const auto& [k, v] : mix)
      fprintf(stderr, "[ops] kind %d flags %02x: %lld\n", k.first, k.second,
              static_cast<long long>(v));
    fprintf(stderr, "[ops] max_slots %d max_mailboxes %d max_coop_ranks %d\n", out.max_slots,
            out.max_mailboxes, out.max_coop_ranks);
  }
  out.cand_off.assign(1, 0);
  out.cand_nodes.clear();
  for (const auto& list : cand_of_row) {
    out.cand_nodes.insert(out.cand_nodes.end(), list.begin(), list.end());
    out.cand_off.push_back(static_cast<int32_t>(out.cand_nodes.size()));
  }

  // retime walk tables: a dense index per F_RT record (programs are shared by
  // replicas, so a record stands for the creator component's task)
  out.rt_rec_of.clear();
  out.rt_rec_task.clear();
  if (d.rt_kind) {
    out.rt_rec_of.assign(out.ops.size(), -1);
    for (size_t p = 0; p < out.programs.size(); ++p) {
      const ProgramDesc& pd = out.programs[p];
      for (int32_t k = 0; k < pd.n_ops; ++k) {
        const Op& o = out.ops[pd.op_offset + k];
        const int32_t n_aux = o.kind == OP_SYNC ? o.x0 : ((o.flags & F_TRACK) ? 1 : 0);
        if ((o.flags & F_RT) && o.kind != OP_NOP && o.kind != OP_START && o.kind != OP_ACC) {
          out.rt_rec_of[pd.op_offset + k] = static_cast<int32_t>(out.rt_rec_task.size());
          out.rt_rec_task.push_back(prog_rep_base[p] + o.node);
        }
        k += n_aux;  // OpExt / OpCov records carry no task
      }
    }
  }
  return TS_OK;
}

// per-task arrays, reduction metadata and the event-driven (DES) tables — for
// every graph, whichever replay path it takes
void build_common(const ts_graph_desc& d, CompiledGraph& out) {
  const int32_t n = d.n_tasks;
  out.base.assign(d.duration, d.duration + n);
  out.rt_kind.clear();
  out.rt_bytes.clear();
  out.rt_group.clear();
  out.rt_mnk.clear();
  if (d.rt_kind) {
    out.rt_kind.assign(d.rt_kind, d.rt_kind + n);
    out.rt_bytes.assign(n, 0);
    out.rt_group.assign(n, 0);
    out.rt_mnk.assign(static_cast<size_t>(n) * 3, 0);
    if (d.rt_bytes) std::copy(d.rt_bytes, d.rt_bytes + n, out.rt_bytes.begin());
    if (d.rt_group) std::copy(d.rt_group, d.rt_group + n, out.rt_group.begin());
    if (d.rt_mnk) std::copy(d.rt_mnk, d.rt_mnk + static_cast<size_t>(n) * 3, out.rt_mnk.begin());
  }
  out.scale_class.resize(n);
  out.is_comm.resize(n);
  out.n_gpu_tasks = 0;
  for (int32_t t = 0; t < n; ++t) {
    out.scale_class[t] = d.scale_class ? d.scale_class[t]
                                       : static_cast<uint8_t>(d.task_kind && d.task_kind[t]
                                                                  ? (d.op_class && d.op_class[t] ==
                                                                             TS_OP_COMMUNICATION
                                                                         ? 2
                                                                         : 1)
                                                                  : 0);
    out.is_comm[t] = d.op_class && d.op_class[t] == TS_OP_COMMUNICATION ? 1 : 0;
    if (d.lane_kind[t] == TS_LANE_CUDA_STREAM) out.n_gpu_tasks++;
  }

  // lanes = distinct processors in ProcessorId order (simulate.cpp:164-171)
  std::vector<Proc> lanes(n);
  for (int32_t i = 0; i < n; ++i) lanes[i] = {d.rank[i], d.lane_kind[i], d.lane[i]};
  std::sort(lanes.begin(), lanes.end());
  lanes.erase(std::unique(lanes.begin(), lanes.end()), lanes.end());
  const int32_t nl = static_cast<int32_t>(lanes.size());
  auto lane_index = [&](const Proc& p) -> int32_t {
    auto it = std::lower_bound(lanes.begin(), lanes.end(), p);
    return (it != lanes.end() && *it == p) ? static_cast<int32_t>(it - lanes.begin()) : -1;
  };
  std::vector<int32_t> lane_of(n), lane_off(nl + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    lane_of[i] = lane_index({d.rank[i], d.lane_kind[i], d.lane[i]});
    lane_off[lane_of[i] + 1]++;
  }
  for (int32_t l = 0; l < nl; ++l) lane_off[l + 1] += lane_off[l];
  std::vector<int32_t> lane_tasks(n);
  {
    std::vector<int32_t> fill(lane_off.begin(), lane_off.end() - 1);
    for (int32_t i = 0; i < n; ++i) lane_tasks[fill[lane_of[i]]++] = i;
  }
  for (int32_t l = 0; l < nl; ++l)
    std::sort(lane_tasks.begin() + lane_off[l], lane_tasks.begin() + lane_off[l + 1],
              [&](int32_t x, int32_t y) {
                return std::make_pair(d.original_start[x], x) <
                       std::make_pair(d.original_start[y], y);
              });

  // reduction metadata (K5): ranks (ranks_in, build.cpp:582-590), their
  // stream lanes and each stream's kernels in chain (= time) order
  out.ranks.clear();
  for (int32_t l = 0; l < nl; ++l)
    if (out.ranks.empty() || out.ranks.back() != lanes[l].rank) out.ranks.push_back(lanes[l].rank);
  out.rank_stream_off.assign(out.ranks.size() + 1, 0);
  out.stream_node_off.assign(1, 0);
  out.stream_rank.clear();
  out.stream_lane.clear();
  out.stream_nodes.clear();
  out.des.lane_stream.assign(nl, -1);
  out.des.lane_rank.assign(nl, 0);
  {
    size_t ri = 0;
    for (int32_t l = 0; l < nl; ++l) {
      while (out.ranks[ri] != lanes[l].rank) {
        ++ri;
        out.rank_stream_off[ri] = static_cast<int32_t>(out.stream_rank.size());
      }
      out.des.lane_rank[l] = static_cast<int32_t>(ri);
      if (lanes[l].kind != TS_LANE_CUDA_STREAM) continue;
      out.des.lane_stream[l] = static_cast<int32_t>(out.stream_rank.size());
      out.stream_rank.push_back(lanes[l].rank);
      out.stream_lane.push_back(lanes[l].lane);
      for (int32_t k = lane_off[l]; k < lane_off[l + 1]; ++k) {
        const int32_t t = lane_tasks[k];
        // bit 31 carries OpClass::Communication for the reduction kernel
        out.stream_nodes.push_back(out.is_comm[t] ? static_cast<int32_t>(
                                                        static_cast<uint32_t>(t) | 0x80000000u)
                                                  : t);
      }
      out.stream_node_off.push_back(static_cast<int32_t>(out.stream_nodes.size()));
    }
    for (size_t r = ri + 1; r <= out.ranks.size(); ++r)
      out.rank_stream_off[r] = static_cast<int32_t>(out.stream_rank.size());
  }

  // event-driven replay tables (restating the Engine, simulate.cpp:162-196)
  DesTables& T = out.des;
  T.n_lanes = nl;
  T.lane_of = lane_of;
  T.lane_off = lane_off;
  T.lane_tasks = lane_tasks;
  T.ostart.assign(d.original_start, d.original_start + n);
  std::vector<std::pair<int32_t, int32_t>> edges;
  edges.reserve(static_cast<size_t>(d.n_edges));
  for (int64_t e = 0; e < d.n_edges; ++e) edges.emplace_back(d.edge_from[e], d.edge_to[e]);
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  T.succ_off.assign(n + 1, 0);
  T.indeg0.assign(n, 0);
  for (const auto& e : edges) {
    T.succ_off[e.first + 1]++;
    T.indeg0[e.second]++;
  }
  for (int32_t i = 0; i < n; ++i) T.succ_off[i + 1] += T.succ_off[i];
  T.succ.resize(edges.size());
  {
    std::vector<int32_t> fill(T.succ_off.begin(), T.succ_off.end() - 1);
    for (const auto& e : edges) T.succ[fill[e.first]++] = e.second;
  }
  T.rule_of.assign(n, -1);
  T.rule_kind.clear();
  T.rule_bound.clear();
  T.rule_wl_off.assign(1, 0);
  T.rule_wl.clear();
  for (int32_t r = 0; r < d.n_rules; ++r) {
    T.rule_of[d.rule_task[r]] = r;  // a later rule on the same task wins
    T.rule_kind.push_back(d.rule_kind[r]);
    T.rule_bound.push_back(d.rule_bound ? d.rule_bound[r] : -1);
    for (int32_t w = d.rule_watch_off[r]; w < d.rule_watch_off[r + 1]; ++w) {
      const int32_t l = lane_index({d.watch_rank[w], d.watch_kind[w], d.watch_lane[w]});
      if (l >= 0) T.rule_wl.push_back(l);  // processors without tasks are ignored
    }
    T.rule_wl_off.push_back(static_cast<int32_t>(T.rule_wl.size()));
  }
}

}  // namespace

int compile_graph(const ts_graph_desc& d, CompiledGraph& out, std::string& err,
                  bool allow_coop) {
  int rc = compile_programs(d, out, err, allow_coop);
  // LUMOS_FORCE_DES=1: every scenario on the event-driven kernel (measurement
  // of that path; tests use it to compare both paths)
  const char* force_des = std::getenv("LUMOS_FORCE_DES");
  if (rc == TS_OK && d.n_gates == 0 && force_des && force_des[0] == '1') {
    rc = TS_E_UNSUPPORTED;
    err = "LUMOS_FORCE_DES=1";
  }
  if (rc == TS_E_UNSUPPORTED && d.n_gates == 0) {
    // outside the chained class: every scenario takes the exact event-driven
    // path (a restatement of the reference Engine on the device)
    const int32_t n = d.n_tasks;
    out = CompiledGraph{};
    out.n_tasks = n;
    out.window_start = d.window_start;
    out.window_end = d.window_end;
    out.des_only = true;
    out.des_reason = err;
    err.clear();
    rc = TS_OK;
  }
  if (rc != TS_OK) return rc;
  build_common(d, out);
  return TS_OK;
}

}  // namespace lumos
