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
#include <map>
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

using CatOverrides = std::vector<std::pair<std::string, uint8_t>>;

uint8_t lookup_category(const std::string& cat, const CatOverrides& over) {  // :156-184
  auto map = [&](const std::string& c, uint8_t& out) {
    for (auto it = over.rbegin(); it != over.rend(); ++it)  // later entries win (set())
      if (c == it->first) {
        out = it->second;
        return true;
      }
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
  MetaList args;  // TraceEvent::args, only with IngestOptions::keep_meta
};

void parse_dom(const json& root, std::vector<RawEvent>& out, const CatOverrides& cats,
               bool keep_args) {  // trace_parse.cpp:79-154
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
    e.cat = lookup_category(ev.value("cat", ""), cats);
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
        if (keep_args) r.args.emplace_back(k, v);
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
// by hand: matches of that pattern never overlap, so the last one wins.  Which
// inputs are rank files is decided on the file name alone (cli.cpp:87-91
// has_rank_marker); their rank comes from the whole path.
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

std::string file_name(const std::string& path) {
  const std::size_t slash = path.find_last_of('/');
  return slash == std::string::npos ? path : path.substr(slash + 1);
}

// detect_iteration_window (trace_parse.cpp:330-399) over one rank's events
std::pair<int64_t, int64_t> detect_window(const std::vector<RawEvent>& evs) {
  if (evs.empty()) return {0, 0};
  int64_t lo = evs.front().ev.ts, hi = lo;
  for (const RawEvent& r : evs) {
    lo = std::min(lo, r.ev.ts);
    hi = std::max(hi, r.ev.ts + r.ev.dur);
  }
  const std::pair<int64_t, int64_t> full{lo, hi};
  auto host = [](const RawEvent& r) { return r.ev.cat == CAT_CPU_OP || r.ev.cat == CAT_RUNTIME; };
  std::map<std::pair<int, int>, int> counts;
  for (const RawEvent& r : evs)
    if (host(r)) counts[{r.ev.pid, r.ev.tid}]++;
  if (counts.empty()) return full;
  auto best_thread = counts.begin();
  for (auto it = counts.begin(); it != counts.end(); ++it)
    if (it->second > best_thread->second) best_thread = it;  // ties: smaller (pid, tid)
  std::vector<std::pair<int64_t, int64_t>> spans;
  for (const RawEvent& r : evs)
    if (host(r) && std::make_pair(r.ev.pid, r.ev.tid) == best_thread->first)
      spans.emplace_back(r.ev.ts, r.ev.ts + r.ev.dur);
  std::sort(spans.begin(), spans.end());
  std::vector<int64_t> gaps;
  for (std::size_t i = 1; i < spans.size(); ++i)
    gaps.push_back(std::max<int64_t>(0, spans[i].first - spans[i - 1].second));
  if (gaps.empty()) return full;
  const int64_t max_gap = *std::max_element(gaps.begin(), gaps.end());
  if (max_gap <= 0) return full;
  std::vector<int64_t> sorted = gaps;
  std::nth_element(sorted.begin(), sorted.begin() + sorted.size() / 2, sorted.end());
  if (max_gap < 8 * std::max<int64_t>(sorted[sorted.size() / 2], 1)) return full;
  std::vector<std::size_t> seg = {0};
  for (std::size_t i = 1; i < spans.size(); ++i)
    if (spans[i].first - spans[i - 1].second >= (max_gap + 1) / 2) seg.push_back(i);
  if (seg.size() == 1) return full;
  std::size_t best = 0, best_n = 0;
  for (std::size_t k = 0; k < seg.size(); ++k) {
    const std::size_t end = k + 1 < seg.size() ? seg[k + 1] : spans.size();
    if (end - seg[k] > best_n) {
      best_n = end - seg[k];
      best = k;
    }
  }
  const std::size_t a = seg[best];
  const std::size_t b = (best + 1 < seg.size() ? seg[best + 1] : spans.size()) - 1;
  return {spans[a].first, spans[b].second};
}

// filter_window (trace_parse.cpp:401-419): events starting in [lo, hi), plus
// GPU events whose correlation matches a retained runtime call
void filter_window(std::vector<RawEvent>& evs, int64_t lo, int64_t hi) {
  std::vector<int64_t> kept;
  for (const RawEvent& r : evs)
    if (r.ev.cat == CAT_RUNTIME && r.ev.corr >= 0 && r.ev.ts >= lo && r.ev.ts < hi)
      kept.push_back(r.ev.corr);
  std::sort(kept.begin(), kept.end());
  std::vector<RawEvent> out;
  for (RawEvent& r : evs) {
    const bool inside = r.ev.ts >= lo && r.ev.ts < hi;
    const bool gpu = r.ev.cat == CAT_KERNEL || r.ev.cat == CAT_MEMCPY || r.ev.cat == CAT_MEMSET;
    if (inside || (gpu && r.ev.corr >= 0 && std::binary_search(kept.begin(), kept.end(), r.ev.corr)))
      out.push_back(std::move(r));
  }
  evs.swap(out);
}

std::string read_file(const std::string& path, bool& ok) {
  std::ifstream in(path, std::ios::binary);
  ok = static_cast<bool>(in);
  std::string text;
  if (!ok) return text;
  in.seekg(0, std::ios::end);
  text.resize(static_cast<std::size_t>(std::max<std::streamoff>(0, in.tellg())));
  in.seekg(0, std::ios::beg);
  in.read(text.data(), static_cast<std::streamsize>(text.size()));
  return text;
}

}  // namespace

bool policy_from_json(const std::string& text, BuildPolicyLite& p, std::string& err) {
  try {  // BuildPolicy::from_json (build.cpp:41-66)
    const json root = json::parse(text);
    p = BuildPolicyLite{};
    if (root.contains("gap_threshold_us")) p.gap_threshold_us = root["gap_threshold_us"].get<int64_t>();
    if (p.gap_threshold_us < 0) {
      err = "build policy: gap_threshold_us must be >= 0";
      return false;
    }
    if (root.contains("launch_names"))
      p.launch_names = root["launch_names"].get<std::vector<std::string>>();
    if (root.contains("sync_names")) {
      p.sync_names.clear();
      for (const auto& [name, flavor] : root["sync_names"].get<std::map<std::string, std::string>>()) {
        const int f = flavor == "device" ? 1 : flavor == "stream" ? 2 : flavor == "event" ? 3 : 0;
        if (!f) {
          err = "build policy: sync flavor for '" + name + "' must be device|stream|event";
          return false;
        }
        p.sync_names.emplace_back(name, f);
      }
    }
    if (root.contains("record_names"))
      p.record_names = root["record_names"].get<std::vector<std::string>>();
    if (root.contains("wait_names")) p.wait_names = root["wait_names"].get<std::vector<std::string>>();
    if (root.contains("comm_patterns"))
      p.comm_patterns = root["comm_patterns"].get<std::vector<std::string>>();
    return true;
  } catch (const json::parse_error& e) {
    err = std::string("build policy: ") + e.what();
  } catch (const std::exception& e) {
    err = std::string("build policy: ") + e.what();
  }
  return false;
}

bool categories_from_json(const std::string& text, CatOverrides& out, std::string& err) {
  json root;  // CategoryTable::from_json (trace_parse.cpp:186-211)
  try {
    root = json::parse(text);
  } catch (const json::parse_error& e) {
    err = std::string("category table: ") + e.what();
    return false;
  }
  if (!root.is_object()) {
    err = "category table must be a JSON object";
    return false;
  }
  out.clear();
  for (auto it = root.begin(); it != root.end(); ++it) {
    const std::string v = it.value().is_string() ? it.value().get<std::string>() : it.value().dump();
    uint8_t c;
    if (v == "CpuOp") c = CAT_CPU_OP;
    else if (v == "CudaRuntime") c = CAT_RUNTIME;
    else if (v == "GpuKernel") c = CAT_KERNEL;
    else if (v == "GpuMemcpy") c = CAT_MEMCPY;
    else if (v == "GpuMemset") c = CAT_MEMSET;
    else if (v == "Metadata") c = CAT_METADATA;
    else {
      err = "category table: unknown category '" + v + "'";
      return false;
    }
    out.emplace_back(it.key(), c);
  }
  return true;
}

int ingest_traces(const IngestOptions& opts, Names& names, HostGraph& out,
                  std::vector<RtMeta>& task_rt, std::string& err) {
  int threads = opts.threads;
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  // window argument (cli.cpp:72-85 parse_window_arg)
  bool win_auto = false, win_fixed = false;
  int64_t win_lo = 0, win_hi = 0;
  if (opts.window == "auto") {
    win_auto = true;
  } else if (opts.window != "full" && !opts.window.empty()) {
    const std::size_t sep = opts.window.find_first_of(":,");
    if (sep == std::string::npos) {
      err = "window must be 'full', 'auto' or START:END, got '" + opts.window + "'";
      return TS_E_INVALID_ARGUMENT;
    }
    try {
      win_lo = std::stoll(opts.window.substr(0, sep));
      win_hi = std::stoll(opts.window.substr(sep + 1));
    } catch (const std::exception&) {
      err = "window bounds must be integers, got '" + opts.window + "'";
      return TS_E_INVALID_ARGUMENT;
    }
    if (win_hi <= win_lo) {
      err = "window end must be after its start";
      return TS_E_INVALID_ARGUMENT;
    }
    win_fixed = true;
  }
  // the files: manifest entries (rank -> path, relative to the manifest's
  // directory; trace_parse.cpp:296-328) first, then the --trace inputs
  struct Input {
    std::string path;
    int rank = -1;  // manifest rank
    bool manifest = false;
  };
  std::vector<Input> inputs;
  if (!opts.manifest.empty()) {
    bool ok = false;
    const std::string text = read_file(opts.manifest, ok);
    if (!ok) {
      err = "cannot open manifest '" + opts.manifest + "'";
      return TS_E_INVALID_ARGUMENT;
    }
    json root;
    try {
      root = json::parse(text);
    } catch (const json::parse_error& e) {
      err = opts.manifest + ": " + e.what();
      return TS_E_INVALID_ARGUMENT;
    }
    if (!root.is_object()) {
      err = opts.manifest + ": manifest must map rank -> path";
      return TS_E_INVALID_ARGUMENT;
    }
    const std::size_t slash = opts.manifest.find_last_of('/');
    const std::string dir = slash == std::string::npos ? "" : opts.manifest.substr(0, slash + 1);
    std::vector<int> seen;
    for (auto it = root.begin(); it != root.end(); ++it) {
      int rank;
      try {
        rank = std::stoi(it.key());
      } catch (const std::exception&) {
        err = opts.manifest + ": manifest key '" + it.key() + "' is not a rank";
        return TS_E_INVALID_ARGUMENT;
      }
      if (std::find(seen.begin(), seen.end(), rank) != seen.end()) {
        err = opts.manifest + ": duplicate rank " + std::to_string(rank);
        return TS_E_INVALID_ARGUMENT;
      }
      seen.push_back(rank);
      std::string path = it.value().is_string() ? it.value().get<std::string>() : "";
      if (!path.empty() && path[0] != '/') path = dir + path;
      inputs.push_back({path, rank, true});
    }
  }
  for (const std::string& p : opts.paths) inputs.push_back({p, -1, false});
  // 1. parse every file (parallel)
  std::vector<std::vector<RawEvent>> parsed(inputs.size());
  std::vector<std::string> errs(inputs.size());
  parallel_for(static_cast<int64_t>(inputs.size()), threads, [&](int64_t i) {
    const std::string& path = inputs[i].path;
    bool ok = false;
    const std::string text = read_file(path, ok);
    if (!ok) {
      errs[i] = "cannot open trace file '" + path + "'";
      return;
    }
    try {
      parse_dom(json::parse(text), parsed[i], opts.categories, opts.keep_meta);
    } catch (const ParseError& e) {
      errs[i] = path + ": " + e.msg;
    } catch (const json::parse_error& e) {
      errs[i] = path + ": malformed trace JSON: " + e.what();
    } catch (const std::exception& e) {
      errs[i] = path + ": " + e.what();
    }
  });
  for (const std::string& e : errs)
    if (!e.empty()) {
      err = e;
      return TS_E_INVALID_ARGUMENT;
    }
  // 2. ranks (cli.cpp:93-116 load_inputs): manifest ranks; files without a
  //    rank_<N> file name split by pid; rank files (load_multirank)
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
  for (std::size_t i = 0; i < inputs.size(); ++i)
    if (inputs[i].manifest && !take(inputs[i].rank, std::move(parsed[i]))) return TS_E_INVALID_ARGUMENT;
  std::vector<std::size_t> marked;
  for (std::size_t i = 0; i < inputs.size(); ++i) {
    if (inputs[i].manifest) continue;
    int rank = 0;
    if (rank_marker(file_name(inputs[i].path), rank)) {
      marked.push_back(i);
      continue;
    }
    std::vector<std::pair<int, std::vector<RawEvent>>> by_pid;
    for (RawEvent& r : parsed[i]) {
      if (by_pid.empty() || by_pid.back().first != r.ev.pid)
        by_pid.emplace_back(r.ev.pid, std::vector<RawEvent>{});
      by_pid.back().second.push_back(std::move(r));
    }
    for (auto& [pid, evs] : by_pid)
      if (!take(pid, std::move(evs))) return TS_E_INVALID_ARGUMENT;
  }
  {
    std::vector<int> seen;
    for (std::size_t i : marked) {
      int rank = 0;
      rank_marker(inputs[i].path, rank);
      if (std::find(seen.begin(), seen.end(), rank) != seen.end()) {
        err = "duplicate rank " + std::to_string(rank) + " from '" + inputs[i].path + "'";
        return TS_E_INVALID_ARGUMENT;
      }
      seen.push_back(rank);
    }
    for (std::size_t i : marked) {
      int rank = 0;
      rank_marker(inputs[i].path, rank);
      if (!take(rank, std::move(parsed[i]))) return TS_E_INVALID_ARGUMENT;
    }
  }
  if (ranks.empty()) {
    err = "no input traces; pass --trace or --manifest";
    return TS_E_INVALID_ARGUMENT;
  }
  std::sort(ranks.begin(), ranks.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  // the iteration window per rank (cli.cpp:128-133)
  if (win_auto || win_fixed)
    parallel_for(static_cast<int64_t>(ranks.size()), threads, [&](int64_t k) {
      auto& evs = ranks[k].second;
      const auto w = win_auto ? detect_window(evs) : std::make_pair(win_lo, win_hi);
      filter_window(evs, w.first, w.second);
    });
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
    rcs[k] = build_rank_graph(events[k], names, ranks[k].first, opts.policy, graphs[k], berr[k]);
  });
  for (std::size_t k = 0; k < ranks.size(); ++k)
    if (rcs[k] != TS_OK) {
      err = berr[k];
      return rcs[k];
    }
  out = HostGraph{};
  for (std::size_t k = 0; k < graphs.size(); ++k) out.append(graphs[k], k == 0);
  task_rt.assign(out.n(), RtMeta{});
  if (opts.keep_meta) {
    out.corr.assign(out.n(), -1);
    out.meta.assign(out.n(), MetaList{});
  }
  for (int32_t t = 0; t < out.n(); ++t) {
    const int64_t o = out.op_index[t];
    if (o < 0) continue;
    const auto k = static_cast<std::size_t>(
        std::upper_bound(ord_base.begin(), ord_base.end(), o) - ord_base.begin() - 1);
    RawEvent& r = ranks[k].second[static_cast<std::size_t>(o - ord_base[k])];
    task_rt[t] = r.rt;
    if (opts.keep_meta) {
      out.corr[t] = r.ev.corr;
      out.meta[t] = std::move(r.args);  // Task.meta = ev.args (build.cpp:363)
    }
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
