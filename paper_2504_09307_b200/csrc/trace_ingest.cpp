// trace_ingest.cpp — Chrome-trace JSON files -> ExecutionGraph, in parallel
// ("host ingest -> CSR speed").
//
// Restates the reference's input path for the default options
// (cli.cpp:93-137 with window "full"): parse_trace (trace_parse.cpp:79-154,
// the default CategoryTable :156-172), load_multirank / split_by_rank rank
// assignment (trace_parse.cpp:260-298, cli.cpp:93-116), build_graph per rank
// (build.cpp:338-510, restated in ingest.cpp) and merge_ranks (build.cpp:512-542).
// Files are parsed on a pool of host threads by a single-pass scanner
// (FastScan: no DOM, only the fields parse_trace reads are decoded); a file it
// does not model exactly — malformed JSON, unexpected field types, values that
// need nlohmann's number formatting — is re-parsed on the DOM path
// (nlohmann::json, the reference's own parser), so errors and exotic values
// behave identically.  The name table is interned in rank order and ranks are
// built in parallel; the result equals the sequential reference path task for
// task.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <cerrno>
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

// ------------------------------------------------------------- fast path
// A single-pass scanner over the trace text that builds RawEvents without a
// DOM: the hot path of ingest (a DOM parse costs ~20-30 MB/s per thread).  It
// validates the JSON it walks (strings incl. UTF-8 and \u escapes, the number
// grammar, nesting) and decodes only the fields parse_trace reads; anything it
// does not model exactly — malformed JSON, a field of an unexpected type, a
// float where a prefix-parsed argument or a kept argument needs nlohmann's
// number formatting — returns false and the caller re-parses the file with
// parse_dom, so errors and exotic values behave exactly as on the DOM path.
class FastScan {
 public:
  FastScan(const std::string& text, const CatOverrides& cats, bool keep_args)
      : p_(text.data()), e_(text.data() + text.size()), cats_(cats), keep_(keep_args) {}

  bool run(std::vector<RawEvent>& out) {
    out.reserve(static_cast<size_t>(e_ - p_) / 160);
    ws();
    if (p_ >= e_) return false;
    if (*p_ == '[') {
      if (!events(out)) return false;
    } else if (*p_ == '{') {
      ++p_;
      bool found = false;
      if (!members([&](const std::string& key) {
            if (key != "traceEvents") return skip(0);
            ws();
            if (p_ >= e_ || *p_ != '[') return false;  // non-array traceEvents: DOM path
            out.clear();
            found = true;
            return events(out);
          }))
        return false;
      if (!found) return false;
    } else {
      return false;
    }
    ws();
    if (p_ != e_) return false;
    // parse_trace's stable (pid, ts, tid) order; recorded traces usually are
    // in it already, otherwise an index permutation moves each event once
    auto less = [&](const RawEvent& a, const RawEvent& b) {
      if (a.ev.pid != b.ev.pid) return a.ev.pid < b.ev.pid;
      if (a.ev.ts != b.ev.ts) return a.ev.ts < b.ev.ts;
      return a.ev.tid < b.ev.tid;
    };
    if (!std::is_sorted(out.begin(), out.end(), less)) {
      std::vector<uint32_t> idx(out.size());
      for (uint32_t k = 0; k < idx.size(); ++k) idx[k] = k;
      std::stable_sort(idx.begin(), idx.end(),
                       [&](uint32_t a, uint32_t b) { return less(out[a], out[b]); });
      std::vector<RawEvent> sorted;
      sorted.reserve(out.size());
      for (uint32_t k : idx) sorted.push_back(std::move(out[k]));
      out.swap(sorted);
    }
    return true;
  }

 private:
  enum Kind : uint8_t { K_NONE, K_STR, K_INT, K_UINT, K_FLT, K_TRUE, K_FALSE, K_NULL, K_ARR, K_OBJ };
  struct Val {
    Kind kind = K_NONE;
    std::string s;
    int64_t i = 0;
    uint64_t u = 0;
    double d = 0.0;
    bool is_int() const { return kind == K_INT || kind == K_UINT; }
    int64_t as_i64() const { return kind == K_INT ? i : static_cast<int64_t>(u); }
  };

  const char* p_;
  const char* e_;
  const CatOverrides& cats_;
  bool keep_;

  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }

  // "..." with escapes decoded and UTF-8 validated (RFC 3629 as nlohmann's lexer)
  bool str(std::string& out) {
    if (p_ >= e_ || *p_ != '"') return false;
    ++p_;
    out.clear();
    for (;;) {
      const char* run = p_;
      while (p_ < e_ && static_cast<unsigned char>(*p_) >= 0x20 && *p_ != '"' && *p_ != '\\' &&
             static_cast<unsigned char>(*p_) < 0x80)
        ++p_;
      out.append(run, p_);
      if (p_ >= e_) return false;
      const unsigned char c = static_cast<unsigned char>(*p_);
      if (c == '"') {
        ++p_;
        return true;
      }
      if (c < 0x20) return false;
      if (c == '\\') {
        if (++p_ >= e_) return false;
        switch (*p_++) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            uint32_t cp = 0;
            if (!hex4(cp)) return false;
            if (cp >= 0xD800 && cp <= 0xDBFF) {
              uint32_t lo = 0;
              if (e_ - p_ < 2 || p_[0] != '\\' || p_[1] != 'u') return false;
              p_ += 2;
              if (!hex4(lo) || lo < 0xDC00 || lo > 0xDFFF) return false;
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
              return false;
            }
            utf8(cp, out);
            break;
          }
          default: return false;
        }
        continue;
      }
      // a multi-byte UTF-8 sequence
      int n = 0;
      uint32_t lo = 0x80, hi = 0xBF;
      if (c >= 0xC2 && c <= 0xDF) n = 1;
      else if (c == 0xE0) { n = 2; lo = 0xA0; }
      else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) n = 2;
      else if (c == 0xED) { n = 2; hi = 0x9F; }
      else if (c == 0xF0) { n = 3; lo = 0x90; }
      else if (c >= 0xF1 && c <= 0xF3) n = 3;
      else if (c == 0xF4) { n = 3; hi = 0x8F; }
      else return false;
      if (e_ - p_ < n + 1) return false;
      const unsigned char c1 = static_cast<unsigned char>(p_[1]);
      if (c1 < lo || c1 > hi) return false;
      for (int k = 2; k <= n; ++k) {
        const unsigned char ck = static_cast<unsigned char>(p_[k]);
        if (ck < 0x80 || ck > 0xBF) return false;
      }
      out.append(p_, p_ + n + 1);
      p_ += n + 1;
    }
  }
  bool hex4(uint32_t& v) {
    if (e_ - p_ < 4) return false;
    v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = *p_++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else return false;
    }
    return true;
  }
  static void utf8(uint32_t cp, std::string& out) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }

  // the JSON number grammar; integers as int64 / uint64 (overflow: double)
  bool number(Val& v) {
    const char* b = p_;
    if (p_ < e_ && *p_ == '-') ++p_;
    if (p_ >= e_) return false;
    if (*p_ == '0') {
      ++p_;
    } else if (*p_ >= '1' && *p_ <= '9') {
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    } else {
      return false;
    }
    bool flt = false;
    if (p_ < e_ && *p_ == '.') {
      flt = true;
      ++p_;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (p_ < e_ && (*p_ == 'e' || *p_ == 'E')) {
      flt = true;
      ++p_;
      if (p_ < e_ && (*p_ == '+' || *p_ == '-')) ++p_;
      if (p_ >= e_ || *p_ < '0' || *p_ > '9') return false;
      while (p_ < e_ && *p_ >= '0' && *p_ <= '9') ++p_;
    }
    if (!flt) {  // accumulate; an overflow becomes a double like nlohmann's
      const bool neg = *b == '-';
      uint64_t x = 0;
      bool over = false;
      for (const char* q = b + (neg ? 1 : 0); q < p_; ++q) {
        const uint64_t d = static_cast<uint64_t>(*q - '0');
        if (x > (UINT64_MAX - d) / 10) {
          over = true;
          break;
        }
        x = x * 10 + d;
      }
      if (!over && !neg) {
        v.kind = K_UINT;
        v.u = x;
        return true;
      }
      if (!over && x <= static_cast<uint64_t>(INT64_MAX) + 1) {
        v.kind = K_INT;
        v.i = x == static_cast<uint64_t>(INT64_MAX) + 1 ? INT64_MIN : -static_cast<int64_t>(x);
        return true;
      }
    }
    const std::string t(b, p_);
    v.kind = K_FLT;
    v.d = std::strtod(t.c_str(), nullptr);
    return true;
  }
  bool word(const char* w, Kind k, Val* v) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(e_ - p_) < n || std::memcmp(p_, w, n) != 0) return false;
    p_ += n;
    if (v) v->kind = k;
    return true;
  }
  // a value; strings and scalars decoded into v (when given), containers validated
  bool value(Val* v, int depth) {
    ws();
    if (p_ >= e_ || depth > 256) return false;
    switch (*p_) {
      case '"': {
        if (!v) {
          std::string tmp;
          return str(tmp);
        }
        v->kind = K_STR;
        return str(v->s);
      }
      case '{':
        ++p_;
        if (v) v->kind = K_OBJ;
        return members([&](const std::string&) { return skip(depth + 1); });
      case '[':
        ++p_;
        if (v) v->kind = K_ARR;
        return elements([&] { return skip(depth + 1); });
      case 't': return word("true", K_TRUE, v);
      case 'f': return word("false", K_FALSE, v);
      case 'n': return word("null", K_NULL, v);
      default: {
        Val tmp;
        return number(v ? *v : tmp);
      }
    }
  }
  bool skip(int depth) { return value(nullptr, depth); }

  // object members after '{': f(key) consumes the value
  template <typename F>
  bool members(F&& f) {
    ws();
    if (p_ < e_ && *p_ == '}') {
      ++p_;
      return true;
    }
    std::string key;
    for (;;) {
      ws();
      if (!str(key)) return false;
      ws();
      if (p_ >= e_ || *p_ != ':') return false;
      ++p_;
      if (!f(key)) return false;
      ws();
      if (p_ >= e_) return false;
      if (*p_ == ',') {
        ++p_;
        continue;
      }
      if (*p_ == '}') {
        ++p_;
        return true;
      }
      return false;
    }
  }
  template <typename F>
  bool elements(F&& f) {
    ws();
    if (p_ < e_ && *p_ == ']') {
      ++p_;
      return true;
    }
    for (;;) {
      if (!f()) return false;
      ws();
      if (p_ >= e_) return false;
      if (*p_ == ',') {
        ++p_;
        continue;
      }
      if (*p_ == ']') {
        ++p_;
        return true;
      }
      return false;
    }
  }

  bool events(std::vector<RawEvent>& out) {
    ++p_;  // '['
    return elements([&] {
      ws();
      if (p_ >= e_ || *p_ != '{') return false;  // "event is not an object": DOM path
      ++p_;
      return event(out);
    });
  }

  // one trace event (parse_trace's per-record rules, trace_parse.cpp:79-154)
  // per-event scratch, reused (capacity kept across events)
  Val ph_, name_, cat_, ts_, dur_, pid_, tid_;
  std::vector<std::pair<std::string, Val>> args_;
  size_t n_args_ = 0;
  std::string last_cat_;
  uint8_t last_cat_code_ = 0;
  bool have_cat_ = false;

  bool event(std::vector<RawEvent>& out) {
    Val &ph = ph_, &name = name_, &cat = cat_, &ts = ts_, &dur = dur_, &pid = pid_, &tid = tid_;
    for (Val* v : {&ph, &name, &cat, &ts, &dur, &pid, &tid}) v->kind = K_NONE;
    bool has_args = false;
    auto& args = args_;
    auto slot = [&](const std::string& k) -> Val* {
      switch (k.size()) {
        case 2: return k == "ph" ? &ph : k == "ts" ? &ts : nullptr;
        case 3: return k == "cat" ? &cat : k == "dur" ? &dur : k == "pid" ? &pid
                     : k == "tid" ? &tid : nullptr;
        case 4: return k == "name" ? &name : nullptr;
        default: return nullptr;
      }
    };
    if (!members([&](const std::string& key) {
          if (key.size() == 4 && key == "args") {
            ws();
            if (p_ < e_ && *p_ == '{') {
              ++p_;
              has_args = true;
              n_args_ = 0;  // a repeated key: the last object wins
              return members([&](const std::string& k) {
                if (n_args_ == args.size()) args.emplace_back();
                auto& slot_kv = args[n_args_];
                slot_kv.first = k;
                slot_kv.second.kind = K_NONE;
                if (!value(&slot_kv.second, 2)) return false;
                ++n_args_;
                return true;
              });
            }
            has_args = false;  // present but not an object: ignored
            return skip(1);
          }
          if (Val* v = slot(key)) {
            v->kind = K_NONE;
            return value(v, 1);
          }
          return skip(1);
        }))
      return false;
    size_t na = has_args ? n_args_ : 0;
    if (na > 1) {  // object keys: key order (stable), the last duplicate wins
      for (size_t a = 1; a < na; ++a)
        for (size_t b = a; b > 0 && args[b].first < args[b - 1].first; --b)
          std::swap(args[b], args[b - 1]);
      size_t w = 0;
      for (size_t a = 0; a < na; ++a) {
        if (w > 0 && args[w - 1].first == args[a].first) std::swap(args[w - 1], args[a]);
        else if (w != a) std::swap(args[w++], args[a]);
        else ++w;
      }
      na = w;
    }
    auto find = [&](const char* k) -> const Val* {
      for (size_t a = 0; a < na; ++a)
        if (args[a].first == k) return &args[a].second;
      return nullptr;
    };
    if (ph.kind != K_NONE && ph.kind != K_STR) return false;
    const std::string phs = ph.kind == K_STR ? ph.s : "X";
    const bool duration_event = phs == "X";
    if (!duration_event) {
      bool keep = name.kind == K_STR && (name.s.find("EventRecord") != std::string::npos ||
                                         name.s.find("WaitEvent") != std::string::npos);
      keep = keep || (has_args && (find("correlation") || find("correlation_id")));
      if (!keep) return true;
    }
    if (phs == "M") return true;
    if ((name.kind != K_NONE && name.kind != K_STR) || (cat.kind != K_NONE && cat.kind != K_STR))
      return false;
    auto micros = [](const Val& v, int64_t& o) {
      if (v.is_int()) o = v.as_i64();
      else if (v.kind == K_FLT) o = static_cast<int64_t>(std::llround(v.d));
      else return false;
      return true;
    };
    RawEvent r;
    Event& e = r.ev;
    r.name = name.s;
    if (!have_cat_ || cat.s != last_cat_) {  // categories repeat: one lookup per change
      last_cat_ = cat.s;
      last_cat_code_ = lookup_category(cat.s, cats_);
      have_cat_ = true;
    }
    e.cat = last_cat_code_;
    if (!micros(ts, e.ts) || e.ts < 0) return false;  // missing / bad / negative: DOM path
    if (duration_event && (!micros(dur, e.dur) || e.dur < 0)) return false;
    auto small = [](const Val& v, int32_t& o) {
      if (v.kind == K_NONE) o = 0;
      else if (v.kind == K_INT) o = static_cast<int32_t>(v.i);
      else if (v.kind == K_UINT) o = static_cast<int32_t>(v.u);
      else return false;
      return true;
    };
    if (!small(pid, e.pid) || !small(tid, e.tid)) return false;
    int64_t stream = 0;
    bool has_stream = false, has_corr = false;
    if (has_args) {
      auto to_int = [&](const char* k, int64_t& o) {  // arg_to_int (trace_parse.cpp:65-77)
        const Val* v = find(k);
        if (!v) return false;
        if (v->is_int()) {
          o = v->as_i64();
          return true;
        }
        return v->kind == K_STR && prefix_i64(v->s, o);
      };
      int64_t corr = 0;
      if (to_int("correlation", corr) || to_int("correlation_id", corr)) {
        e.corr = corr;
        has_corr = true;
      }
      has_stream = to_int("stream", stream);
      for (size_t a = 0; a < na; ++a) {
        const std::string& k = args[a].first;
        const Val& v = args[a].second;
        std::string s;
        switch (v.kind) {
          case K_STR: s = v.s; break;
          case K_INT: s = std::to_string(v.i); break;
          case K_UINT: s = std::to_string(v.u); break;
          case K_TRUE: s = "true"; break;
          case K_FALSE: s = "false"; break;
          case K_NULL: s = "null"; break;
          default:  // floats and containers: nlohmann's dump text is needed
            if (keep_ || (v.kind == K_FLT && (k == "event" || k == "stream"))) return false;
            continue;  // no interpreted key accepts them
        }
        if (keep_) r.args.emplace_back(k, s);
        int64_t x = 0;
        switch (k.size()) {
          case 1:
            if ((k[0] == 'm' || k[0] == 'n' || k[0] == 'k') && strict_i64(s, x))
              (k[0] == 'm' ? r.rt.m : k[0] == 'n' ? r.rt.n : r.rt.k) = x;
            break;
          case 3:
            if (k == "dir") r.rt.dir_recv = s == "recv";
            break;
          case 5:
            if (k == "event") {
              if (prefix_i64(s, x)) e.arg_event = x;
            } else if (k == "bytes") {
              if (strict_i64(s, x)) r.rt.bytes = x;
            }
            break;
          case 6:
            if (k == "stream") {
              if (prefix_i64(s, x)) e.arg_stream = x;
            } else if (k == "region") {
              r.rt.region_opt = s == "opt";
              r.rt.region_p2p = s == "p2p";
            }
            break;
          case 10:
            if (k == "group_size") {
              if (strict_i64(s, x)) r.rt.group = x;
            } else if (k == "collective") {
              r.rt.allreduce = s == "allreduce";
            }
            break;
          default: break;
        }
      }
    }
    const bool gpu = e.cat == CAT_KERNEL || e.cat == CAT_MEMCPY || e.cat == CAT_MEMSET;
    if (has_stream) e.stream = static_cast<int32_t>(stream);
    else if (gpu) e.stream = e.tid;
    if (e.cat == CAT_RUNTIME && is_launch_name(r.name) && !has_corr) return false;
    out.push_back(std::move(r));
    return true;
  }
};

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
      // fast scanner first; anything it does not model re-parses on the DOM
      if (opts.dom_only || !FastScan(text, opts.categories, opts.keep_meta).run(parsed[i])) {
        parsed[i].clear();
        parse_dom(json::parse(text), parsed[i], opts.categories, opts.keep_meta);
      }
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
