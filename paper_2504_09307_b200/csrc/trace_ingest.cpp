// trace_ingest.cpp — Chrome-trace JSON files -> ExecutionGraph, in parallel
// ("host ingest -> CSR speed").
//
// Restates the reference's input path for the default options
// (cli.cpp:93-137 with window "full"): parse_trace (trace_parse.cpp:79-154,
// the default CategoryTable :156-172), load_multirank / split_by_rank rank
// assignment (trace_parse.cpp:260-298, cli.cpp:93-116), build_graph per rank
// (build.cpp:338-510, restated in ingest.cpp) and merge_ranks (build.cpp:512-542).
// Files are parsed on a pool of host threads (JSON parsing with nlohmann::json,
// the reference's own parser, so numbers and strings decode identically), the
// name table is interned in rank order, and ranks are built in parallel; the
// result equals the sequential reference path task for task.
#include <algorithm>
#include <atomic>
#include <fstream>
#include <cctype>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "ingest.hpp"
#include "nlohmann/json.hpp"
#include "trace_ingest.hpp"

namespace lumos {

namespace {

using nlohmann::json;

struct ParseError {
  std::string msg;
};

bool is_launch_name(const std::string& n) {  // trace_parse.cpp:22-31
  static const char* kNames[] = {"cudaLaunchKernel", "cudaLaunchKernelExC", "cuLaunchKernel",
                                 "cudaLaunchCooperativeKernel", "cudaMemcpyAsync",
                                 "cudaMemsetAsync"};
  for (const char* k : kNames)
    if (n == k) return true;
  return false;
}

bool keeps_zero_duration_event(const json& ev) {  // trace_parse.cpp:33-46
  if (ev.contains("name") && ev["name"].is_string()) {
    const std::string& n = ev["name"].get_ref<const std::string&>();
    if (n.find("EventRecord") != std::string::npos) return true;
    if (n.find("WaitEvent") != std::string::npos) return true;
  }
  if (ev.contains("args") && ev["args"].is_object() &&
      (ev["args"].contains("correlation") || ev["args"].contains("correlation_id")))
    return true;
  return false;
}

int64_t to_micros(const json& v) {  // trace_parse.cpp:52-58
  if (v.is_number_integer()) return v.get<int64_t>();
  if (v.is_number_unsigned()) return static_cast<int64_t>(v.get<uint64_t>());
  if (v.is_number_float()) return static_cast<int64_t>(std::llround(v.get<double>()));
  throw ParseError{"expected a numeric time value"};
}

std::string arg_to_string(const json& v) { return v.is_string() ? v.get<std::string>() : v.dump(); }

bool arg_to_int(const json& args, const char* key, int64_t& out) {  // trace_parse.cpp:65-77
  if (!args.contains(key)) return false;
  const json& v = args[key];
  if (v.is_number_integer()) {
    out = v.get<int64_t>();
    return true;
  }
  if (v.is_number_unsigned()) {
    out = static_cast<int64_t>(v.get<uint64_t>());
    return true;
  }
  if (v.is_string()) {
    try {
      out = std::stoll(v.get<std::string>());
      return true;
    } catch (const std::exception&) {
      return false;
    }
  }
  return false;
}

uint8_t lookup_category(const std::string& cat) {  // CategoryTable defaults, :156-184
  auto map = [](const std::string& c, uint8_t& out) {
    static const std::pair<const char*, uint8_t> kTable[] = {
        {"cpu_op", CAT_CPU_OP},       {"cpu_instant_event", CAT_METADATA},
        {"user_annotation", CAT_METADATA}, {"gpu_user_annotation", CAT_METADATA},
        {"python_function", CAT_METADATA}, {"cuda_runtime", CAT_RUNTIME},
        {"cuda_driver", CAT_RUNTIME}, {"runtime", CAT_RUNTIME},
        {"kernel", CAT_KERNEL},       {"gpu_kernel", CAT_KERNEL},
        {"gpu_memcpy", CAT_MEMCPY},   {"gpu_memset", CAT_MEMSET}};
    for (const auto& [k, v] : kTable)
      if (c == k) {
        out = v;
        return true;
      }
    return false;
  };
  uint8_t out = CAT_METADATA;
  if (map(cat, out)) return out;
  std::string lower = cat;
  std::transform(lower.begin(), lower.end(), lower.begin(),
                 [](unsigned char ch) { return static_cast<char>(std::tolower(ch)); });
  if (map(lower, out)) return out;
  return CAT_METADATA;
}

// strict integer of a meta string (transform.cpp meta_i64)
bool strict_i64(const std::string& s, int64_t& out) {
  try {
    std::size_t pos = 0;
    const int64_t v = std::stoll(s, &pos);
    if (pos != s.size()) return false;
    out = v;
    return true;
  } catch (const std::exception&) {
    return false;
  }
}

// lenient integer of a meta string (build.cpp meta_int)
bool prefix_i64(const std::string& s, int64_t& out) {
  try {
    out = std::stoll(s);
    return true;
  } catch (const std::exception&) {
    return false;
  }
}

struct RawEvent {
  std::string name;
  Event ev;
  RtMeta rt;
};

void parse_dom(const json& root, std::vector<RawEvent>& out) {  // trace_parse.cpp:79-154
  const json* list = nullptr;
  if (root.is_array()) {
    list = &root;
  } else if (root.is_object() && root.contains("traceEvents") && root["traceEvents"].is_array()) {
    list = &root["traceEvents"];
  } else {
    throw ParseError{"trace JSON must be an event array or an object with traceEvents"};
  }
  out.reserve(list->size());
  for (std::size_t idx = 0; idx < list->size(); ++idx) {
    const json& ev = (*list)[idx];
    if (!ev.is_object())
      throw ParseError{"record " + std::to_string(idx) + ": event is not an object"};
    const std::string ph = ev.value("ph", "X");
    const bool duration_event = ph == "X";
    if (!duration_event && !keeps_zero_duration_event(ev)) continue;
    if (ph == "M") continue;
    RawEvent r;
    r.name = ev.value("name", "");
    Event& e = r.ev;
    e.cat = lookup_category(ev.value("cat", ""));
    if (!ev.contains("ts")) throw ParseError{"record " + std::to_string(idx) + ": missing ts"};
    e.ts = to_micros(ev["ts"]);
    if (e.ts < 0) throw ParseError{"record " + std::to_string(idx) + ": negative ts"};
    if (duration_event) {
      if (!ev.contains("dur"))
        throw ParseError{"record " + std::to_string(idx) +
                         ": ph:\"X\" event missing dur (truncated trace?)"};
      e.dur = to_micros(ev["dur"]);
      if (e.dur < 0) throw ParseError{"record " + std::to_string(idx) + ": negative dur"};
    }
    e.pid = ev.value("pid", 0);
    e.tid = ev.value("tid", 0);
    int64_t stream = 0;
    bool has_stream = false, has_corr = false;
    if (ev.contains("args") && ev["args"].is_object()) {
      const json& args = ev["args"];
      int64_t corr = 0;
      if (arg_to_int(args, "correlation", corr) || arg_to_int(args, "correlation_id", corr)) {
        e.corr = corr;
        has_corr = true;
      }
      has_stream = arg_to_int(args, "stream", stream);
      // Task.meta is the args as strings (build.cpp:363); the builder reads
      // "event" / "stream" with meta_int, the retime transforms read the rest
      for (auto it = args.begin(); it != args.end(); ++it) {
        const std::string& k = it.key();
        const std::string v = arg_to_string(it.value());
        int64_t x = 0;
        if (k == "event") {
          if (prefix_i64(v, x)) e.arg_event = x;
        } else if (k == "stream") {
          if (prefix_i64(v, x)) e.arg_stream = x;
        } else if (k == "bytes") {
          if (strict_i64(v, x)) r.rt.bytes = x;
        } else if (k == "group_size") {
          if (strict_i64(v, x)) r.rt.group = x;
        } else if (k == "m" || k == "n" || k == "k") {
          if (strict_i64(v, x)) (k == "m" ? r.rt.m : k == "n" ? r.rt.n : r.rt.k) = x;
        } else if (k == "collective") {
          r.rt.allreduce = v == "allreduce";
        } else if (k == "region") {
          r.rt.region_opt = v == "opt";
          r.rt.region_p2p = v == "p2p";
        } else if (k == "dir") {
          r.rt.dir_recv = v == "recv";
        }
      }
    }
    const bool gpu = e.cat == CAT_KERNEL || e.cat == CAT_MEMCPY || e.cat == CAT_MEMSET;
    if (has_stream) e.stream = static_cast<int32_t>(stream);
    else if (gpu) e.stream = e.tid;  // kineto puts the stream in tid
    if (e.cat == CAT_RUNTIME && is_launch_name(r.name) && !has_corr)
      throw ParseError{"record " + std::to_string(idx) + ": launch-class runtime event '" +
                       r.name + "' without a correlation id"};
    out.push_back(std::move(r));
  }
  std::stable_sort(out.begin(), out.end(), [](const RawEvent& a, const RawEvent& b) {
    if (a.ev.pid != b.ev.pid) return a.ev.pid < b.ev.pid;
    if (a.ev.ts != b.ev.ts) return a.ev.ts < b.ev.ts;
    return a.ev.tid < b.ev.tid;
  });
}

// the last "rank_?(\\d+)" match of a path (trace_parse.cpp:260-270), scanned
// by hand: matches of that pattern never overlap, so the last one wins
bool rank_marker(const std::string& path, int& rank) {
  bool found = false;
  for (std::size_t p = path.find("rank"); p != std::string::npos; p = path.find("rank", p + 1)) {
    std::size_t q = p + 4;
    if (q < path.size() && path[q] == '_') ++q;
    std::size_t e = q;
    while (e < path.size() && std::isdigit(static_cast<unsigned char>(path[e]))) ++e;
    if (e > q) {
      rank = std::stoi(path.substr(q, e - q));
      found = true;
    }
  }
  return found;
}

template <class F>
void parallel_for(int64_t n, int threads, F f) {
  std::atomic<int64_t> next{0};
  auto work = [&] {
    for (int64_t i; (i = next.fetch_add(1)) < n;) f(i);
  };
  const int t = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, n)));
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
}

}  // namespace

int ingest_trace_files(const std::vector<std::string>& paths, int threads,
                       const BuildPolicyLite& policy, Names& names, HostGraph& out,
                       std::vector<RtMeta>& task_rt, std::string& err) {
  if (paths.empty()) {
    err = "no input traces; pass --trace or --manifest";
    return TS_E_INVALID_ARGUMENT;
  }
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  // 1. parse every file (parallel)
  std::vector<std::vector<RawEvent>> parsed(paths.size());
  std::vector<std::string> errs(paths.size());
  parallel_for(static_cast<int64_t>(paths.size()), threads, [&](int64_t i) {
    std::ifstream in(paths[i], std::ios::binary);
    if (!in) {
      errs[i] = "cannot open trace file '" + paths[i] + "'";
      return;
    }
    std::string text;
    in.seekg(0, std::ios::end);
    text.resize(static_cast<std::size_t>(std::max<std::streamoff>(0, in.tellg())));
    in.seekg(0, std::ios::beg);
    in.read(text.data(), static_cast<std::streamsize>(text.size()));
    try {
      parse_dom(json::parse(text), parsed[i]);
    } catch (const ParseError& e) {
      errs[i] = paths[i] + ": " + e.msg;
    } catch (const json::parse_error& e) {
      errs[i] = paths[i] + ": malformed trace JSON: " + e.what();
    } catch (const std::exception& e) {
      errs[i] = paths[i] + ": " + e.what();
    }
  });
  for (const std::string& e : errs)
    if (!e.empty()) {
      err = e;
      return TS_E_INVALID_ARGUMENT;
    }
  // 2. ranks: a rank_<N> file is one rank; other files split by pid
  //    (cli.cpp:93-116 load_inputs, trace_parse.cpp split_by_rank)
  std::vector<std::pair<int, std::vector<RawEvent>>> ranks;
  auto take = [&](int rank, std::vector<RawEvent>&& evs) -> bool {
    for (const auto& r : ranks)
      if (r.first == rank) {
        err = "rank " + std::to_string(rank) + " appears in more than one input";
        return false;
      }
    ranks.emplace_back(rank, std::move(evs));
    return true;
  };
  for (std::size_t i = 0; i < paths.size(); ++i) {
    int rank = 0;
    if (rank_marker(paths[i], rank)) continue;
    std::vector<std::pair<int, std::vector<RawEvent>>> by_pid;
    for (RawEvent& r : parsed[i]) {
      if (by_pid.empty() || by_pid.back().first != r.ev.pid) by_pid.emplace_back(r.ev.pid, std::vector<RawEvent>{});
      by_pid.back().second.push_back(std::move(r));
    }
    for (auto& [pid, evs] : by_pid)
      if (!take(pid, std::move(evs))) return TS_E_INVALID_ARGUMENT;
  }
  for (std::size_t i = 0; i < paths.size(); ++i) {
    int rank = 0;
    if (!rank_marker(paths[i], rank)) continue;
    if (!take(rank, std::move(parsed[i]))) return TS_E_INVALID_ARGUMENT;
  }
  std::sort(ranks.begin(), ranks.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  // 3. names interned in rank order; events keep their source ordinal in
  //    op_index so the built tasks can find their metadata
  std::vector<std::vector<Event>> events(ranks.size());
  std::vector<int64_t> ord_base(ranks.size() + 1, 0);
  for (std::size_t k = 0; k < ranks.size(); ++k) {
    ord_base[k + 1] = ord_base[k] + static_cast<int64_t>(ranks[k].second.size());
    events[k].reserve(ranks[k].second.size());
    for (std::size_t j = 0; j < ranks[k].second.size(); ++j) {
      Event e = ranks[k].second[j].ev;
      e.name = names.get(ranks[k].second[j].name);
      e.op_index = ord_base[k] + static_cast<int64_t>(j);
      events[k].push_back(e);
    }
  }
  // 4. build_graph per rank (parallel), merge_ranks in rank order
  std::vector<HostGraph> graphs(ranks.size());
  std::vector<int> rcs(ranks.size(), TS_OK);
  std::vector<std::string> berr(ranks.size());
  parallel_for(static_cast<int64_t>(ranks.size()), threads, [&](int64_t k) {
    rcs[k] = build_rank_graph(events[k], names, ranks[k].first, policy, graphs[k], berr[k]);
  });
  for (std::size_t k = 0; k < ranks.size(); ++k)
    if (rcs[k] != TS_OK) {
      err = berr[k];
      return rcs[k];
    }
  out = HostGraph{};
  for (std::size_t k = 0; k < graphs.size(); ++k) out.append(graphs[k], k == 0);
  task_rt.assign(out.n(), RtMeta{});
  for (int32_t t = 0; t < out.n(); ++t) {
    const int64_t o = out.op_index[t];
    if (o < 0) continue;
    const auto k = static_cast<std::size_t>(
        std::upper_bound(ord_base.begin(), ord_base.end(), o) - ord_base.begin() - 1);
    task_rt[t] = ranks[k].second[static_cast<std::size_t>(o - ord_base[k])].rt;
    out.op_index[t] = -1;  // a recorded trace has no generator cost index
  }
  return TS_OK;
}

// TS_RT_* class of a task from its metadata (transform.cpp:219-349)
void fill_retime_arrays(HostGraph& g, const std::vector<RtMeta>& rt) {
  const int32_t n = g.n();
  g.rt_kind.assign(n, TS_RT_NONE);
  g.rt_bytes.assign(n, -1);
  g.rt_group.assign(n, 0);
  g.rt_mnk.assign(static_cast<size_t>(n) * 3, 0);
  for (int32_t t = 0; t < n; ++t) {
    const RtMeta& m = rt[t];
    g.rt_bytes[t] = m.bytes;
    g.rt_group[t] = static_cast<int32_t>(m.group);
    g.rt_mnk[3 * static_cast<size_t>(t)] = m.m;
    g.rt_mnk[3 * static_cast<size_t>(t) + 1] = m.n;
    g.rt_mnk[3 * static_cast<size_t>(t) + 2] = m.k;
    if (g.task_kind[t] != 1) continue;
    if (g.op_class[t] == TS_OP_COMPUTE) {
      if (m.m > 0 && m.n > 0 && m.k > 0) g.rt_kind[t] = TS_RT_GEMM;
      else if (m.region_opt && m.bytes >= 0) g.rt_kind[t] = TS_RT_OPT;
    } else if (g.op_class[t] == TS_OP_COMMUNICATION) {
      if (m.allreduce) g.rt_kind[t] = TS_RT_ALLREDUCE;
      else if (m.region_p2p && m.bytes >= 0)
        g.rt_kind[t] = m.dir_recv ? TS_RT_P2P_RECV : TS_RT_P2P_SEND;
    }
  }
}

}  // namespace lumos
