// rebuild.cpp — tag_tasks + measure_pipeline + rebuild_pipeline over a
// HostGraph (see rebuild.hpp).  Host-only, once per what-if; its output
// PipelineSpec is the Mode-B input the device engine replays in batches.
#include "rebuild.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <map>
#include <optional>
#include <set>
#include <unordered_map>

#include "nlohmann/json.hpp"

namespace lumos {

namespace {

struct TransformError {
  std::string msg;
};

// Task.meta as a map (Task::meta is std::map<std::string, std::string>)
using Meta = std::map<std::string, std::string>;

struct TTask {
  std::optional<int> layer, mb;
  Meta meta;
};

std::optional<int> full_int(const std::string& s) {  // tag_tasks to_int (:77-85)
  try {
    std::size_t pos = 0;
    const int v = std::stoi(s, &pos);
    if (pos != s.size()) return std::nullopt;
    return v;
  } catch (const std::exception&) {
    return std::nullopt;
  }
}

std::optional<int64_t> meta_i64(const Meta& m, const char* key) {  // transform.cpp:19-30
  auto it = m.find(key);
  if (it == m.end()) return std::nullopt;
  try {
    std::size_t pos = 0;
    const long long v = std::stoll(it->second, &pos);
    if (pos != it->second.size()) return std::nullopt;
    return v;
  } catch (const std::exception&) {
    return std::nullopt;
  }
}

std::string meta_str(const Meta& m, const char* key) {
  auto it = m.find(key);
  return it == m.end() ? std::string() : it->second;
}

int64_t mul_div(int64_t a, int64_t num, int64_t den) {  // transform.cpp:37-43
  if (den == 0) throw TransformError{"internal: zero denominator in rescale"};
  const __int128 prod = static_cast<__int128>(a) * num;
  const __int128 half = den / 2;
  return static_cast<int64_t>((prod + half) / den);
}

// regex_search(s, "<prefix>(\\d+)") (transform.cpp:72-73, 98): the leftmost
// prefix followed by a digit, the maximal digit run after it
bool digits_after(const std::string& s, const char* prefix, std::string& out) {
  const std::size_t n = std::char_traits<char>::length(prefix);
  for (std::size_t i = s.find(prefix); i != std::string::npos; i = s.find(prefix, i + 1)) {
    std::size_t j = i + n;
    while (j < s.size() && s[j] >= '0' && s[j] <= '9') ++j;
    if (j > i + n) {
      out = s.substr(i + n, j - i - n);
      return true;
    }
  }
  return false;
}

std::string phase_of(std::string v) {  // normalize_phase (transform.cpp:45-50)
  std::transform(v.begin(), v.end(), v.begin(),
                 [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
  if (v == "forward" || v == "fwd" || v == "f") return "fwd";
  if (v == "backward" || v == "bwd" || v == "b") return "bwd";
  return v;
}

// cost.cpp:39-66 (AnalyticalCostModel without a reference point)
int64_t wire_cost(bool allreduce, int64_t bytes, int group, double alpha, double bpu,
                  const char* what) {
  auto fail = [&](const char* m) {
    throw TransformError{std::string("cost model cannot size ") + what + ": " + m};
  };
  if (group < 1) fail("collective group_size must be >= 1");
  if (bytes < 0) fail("collective bytes must be non-negative");
  if (bpu <= 0) fail("bytes_per_us must be positive");
  const double g = group;
  const double scale = allreduce ? 2.0 * (g - 1.0) / g : 1.0;
  const double t = alpha + static_cast<double>(bytes) * scale / bpu;
  return std::max<int64_t>(0, std::llround(t));
}

int64_t layer_param_bytes(const ts_model_config& m) {  // cost.cpp:74-77
  const int64_t d = m.d_model, f = m.d_ffn;
  return (4 * d * d + 2 * d * f) * 2;
}

int64_t substitute_dim(int64_t dim, const ts_model_config& s, const ts_model_config& t) {
  if (dim == s.d_model) return t.d_model;  // transform.cpp:270-275
  if (dim == s.d_ffn) return t.d_ffn;
  return dim;
}

void validate(const ts_model_config& m) {  // types.cpp:45-53
  const char* e = nullptr;
  if (m.n_layers <= 0) e = "ModelConfig.n_layers must be positive";
  else if (m.d_model <= 0) e = "ModelConfig.d_model must be positive";
  else if (m.d_ffn <= 0) e = "ModelConfig.d_ffn must be positive";
  else if (m.n_heads <= 0) e = "ModelConfig.n_heads must be positive";
  else if (m.d_head <= 0) e = "ModelConfig.d_head must be positive";
  else if (m.d_model != m.n_heads * m.d_head) e = "ModelConfig.d_model must equal n_heads * d_head";
  if (e) throw TransformError{std::string("what-if config invalid: ") + e};
}

void validate(const ts_par_config& p) {  // types.cpp:55-65
  const char* e = nullptr;
  if (p.tp < 1) e = "ParallelismConfig.tp must be >= 1";
  else if (p.pp < 1) e = "ParallelismConfig.pp must be >= 1";
  else if (p.dp < 1) e = "ParallelismConfig.dp must be >= 1";
  else if (p.num_microbatches < 1) e = "ParallelismConfig.num_microbatches must be >= 1";
  else if (p.num_microbatches < p.pp)
    e = "ParallelismConfig.num_microbatches must be >= pp (pipeline schedule needs one "
        "microbatch per stage in flight)";
  if (e) throw TransformError{std::string("what-if config invalid: ") + e};
}

void validate(const WhatIfLite& w) {  // WhatIfConfig::validate (transform.cpp:164-176)
  if (w.source_par.tp != w.target_par.tp)
    throw TransformError{"tensor-parallel rescaling is not supported"};
  validate(w.source_par);
  validate(w.target_par);
  validate(w.source_model);
  validate(w.target_model);
}

// ---------------------------------------------------------------- tagging
// tag_tasks (transform.cpp:71-162) on the graph's tasks: tags from args,
// then from kernel names, correlation inheritance, and the fill-between pass
// over host lanes.  Name-derived tags are evaluated once per distinct name
// (the two layer patterns are scanned by hand; no std::regex in the library).
std::vector<TTask> tag_tasks(const HostGraph& g, const Names& names, const TagPolicyLite& pol) {
  const int32_t n = g.n();
  std::vector<TTask> t(n);
  struct NameTags {
    bool done = false;
    std::optional<int> layer;
    const char* phase = nullptr;
  };
  std::vector<NameTags> by_name(names.str.size());
  auto name_tags = [&](int32_t id) -> const NameTags& {
    NameTags& nt = by_name[id];
    if (nt.done) return nt;
    nt.done = true;
    const std::string& s = names.str[id];
    std::string d;
    if (digits_after(s, "layers.", d) || digits_after(s, "layer_", d)) nt.layer = full_int(d);
    if (s.find("bwd") != std::string::npos || s.find("backward") != std::string::npos ||
        s.find("wgrad") != std::string::npos || s.find("dgrad") != std::string::npos)
      nt.phase = "bwd";
    else if (s.find("fwd") != std::string::npos || s.find("forward") != std::string::npos)
      nt.phase = "fwd";
    return nt;
  };
  auto first_meta = [](const Meta& m, const std::vector<std::string>& keys) -> const std::string* {
    for (const auto& k : keys) {
      auto it = m.find(k);
      if (it != m.end()) return &it->second;
    }
    return nullptr;
  };
  for (int32_t i = 0; i < n; ++i) {
    TTask& x = t[i];
    if (static_cast<size_t>(i) < g.meta.size()) x.meta.insert(g.meta[i].begin(), g.meta[i].end());
    if (const std::string* v = first_meta(x.meta, pol.layer_keys)) x.layer = full_int(*v);
    if (!x.layer && pol.infer_from_names) x.layer = name_tags(g.name[i]).layer;
    if (const std::string* v = first_meta(x.meta, pol.microbatch_keys)) x.mb = full_int(*v);
    if (const std::string* v = first_meta(x.meta, pol.phase_keys)) {
      x.meta["phase"] = phase_of(*v);
    } else if (pol.infer_from_names) {
      if (const char* p = name_tags(g.name[i]).phase) x.meta["phase"] = p;
    }
  }
  // kernels inherit missing tags from their launching host op and vice versa
  auto inherit = [&](TTask& dst, const TTask& src) {
    if (!dst.layer) dst.layer = src.layer;
    if (!dst.mb) dst.mb = src.mb;
    for (const char* key : {"phase", "region"}) {
      auto it = src.meta.find(key);
      if (!dst.meta.count(key) && it != src.meta.end()) dst.meta[key] = it->second;
    }
  };
  const bool has_corr = g.corr.size() == static_cast<size_t>(n);
  if (has_corr) {
    std::unordered_map<int64_t, int32_t> cpu_by_corr, gpu_by_corr;
    for (int32_t i = 0; i < n; ++i)
      if (g.corr[i] >= 0) (g.task_kind[i] == 0 ? cpu_by_corr : gpu_by_corr)[g.corr[i]] = i;
    for (int32_t i = 0; i < n; ++i) {
      if (g.corr[i] < 0) continue;
      const auto& other = g.task_kind[i] == 1 ? cpu_by_corr : gpu_by_corr;
      auto it = other.find(g.corr[i]);
      if (it != other.end()) inherit(t[i], t[it->second]);
    }
  }
  if (!pol.fill_between) return t;
  std::map<std::tuple<int32_t, int32_t, int32_t>, std::vector<int32_t>> lanes;
  for (int32_t i = 0; i < n; ++i)
    if (g.task_kind[i] == 0) lanes[{g.rank[i], g.lane_kind[i], g.lane[i]}].push_back(i);
  for (auto& [proc, ids] : lanes) {
    // the reference's unstable sort on original_start alone, on the same input order
    std::sort(ids.begin(), ids.end(),
              [&](int32_t a, int32_t b) { return g.original_start[a] < g.original_start[b]; });
    auto tagged = [&](int32_t id) { return t[id].layer.has_value() || t[id].mb.has_value(); };
    std::size_t i = 0;
    while (i < ids.size()) {
      if (tagged(ids[i])) {
        ++i;
        continue;
      }
      const std::size_t lo = i;
      while (i < ids.size() && !tagged(ids[i])) ++i;
      if (lo == 0 || i == ids.size()) continue;
      const TTask& before = t[ids[lo - 1]];
      const TTask& after = t[ids[i]];
      if (before.layer == after.layer && before.mb == after.mb &&
          meta_str(before.meta, "phase") == meta_str(after.meta, "phase")) {
        const TTask src = before;
        for (std::size_t k = lo; k < i; ++k) inherit(t[ids[k]], src);
      }
    }
  }
  return t;
}

// --------------------------------------------------------------- measuring
struct Measured {  // transform.cpp:352-366
  int64_t launch = 5, record = 2, wait = 2, sync = 5;
  std::vector<std::vector<KernelStr>> layer_fwd, layer_bwd;
  std::vector<KernelStr> pre_fwd, post_fwd, pre_bwd, post_bwd;
  std::string reduce_name = "ncclDevKernel_AllReduce_Sum_f16";
  std::map<int, int64_t> stage_bytes;
  std::vector<KernelStr> optimizer;
  double opt_rate = 0.0;
  int64_t p2p_send = -1, p2p_recv_base = -1;
  int64_t act_bytes = 0;
  int64_t origin = 0;
};

int64_t median_of(std::vector<int64_t> v, int64_t fallback) {
  if (v.empty()) return fallback;
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

// measure_pipeline (transform.cpp:378-502)
Measured measure(const HostGraph& g, const Names& names, const std::vector<TTask>& tags,
                 const WhatIfLite& w) {
  const int pp = w.source_par.pp, dp = w.source_par.dp;
  const int32_t n = g.n();
  std::set<int32_t> rank_set(g.rank.begin(), g.rank.end());
  const std::vector<int32_t> ranks(rank_set.begin(), rank_set.end());
  if (static_cast<int>(ranks.size()) != pp * dp)
    throw TransformError{"graph covers " + std::to_string(ranks.size()) +
                         " ranks but source parallelism implies " + std::to_string(pp * dp)};
  Measured m;
  m.origin = g.window_start;
  std::map<int32_t, int> stage_of;
  std::map<int32_t, bool> primary;
  for (std::size_t i = 0; i < ranks.size(); ++i) {
    stage_of[ranks[i]] = static_cast<int>(i) % pp;
    primary[ranks[i]] = static_cast<int>(i) / pp == 0;
  }
  auto spec_from = [&](int32_t i) {  // transform.cpp:368-380
    KernelStr k;
    k.name = names.str[g.name[i]];
    k.duration = g.duration[i];
    k.op_class = g.op_class[i];
    for (const auto& [key, v] : tags[i].meta) {
      if (key == "mb" || key == "microbatch" || key == "micro_batch" || key == "layer" ||
          key == "layer_id" || key == "phase" || key == "region" || key == "dir" ||
          key == "peer_stage")
        continue;
      k.args.emplace_back(key, v);
    }
    return k;
  };
  auto specs_sorted = [&](std::vector<int32_t> ids) {
    std::sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) {
      return std::make_pair(g.original_start[a], a) < std::make_pair(g.original_start[b], b);
    });
    std::vector<KernelStr> out;
    out.reserve(ids.size());
    for (int32_t i : ids) out.push_back(spec_from(i));
    return out;
  };
  std::vector<int64_t> launches, records, waits, syncs, sends, recvs;
  std::map<int, std::vector<int32_t>> fwd_groups, bwd_groups;
  std::map<int, int64_t> opt_dur, opt_bytes;
  std::vector<int32_t> pre_fwd, post_fwd, pre_bwd, post_bwd;
  for (int32_t i = 0; i < n; ++i) {
    if (!primary.at(g.rank[i])) continue;
    const int stage = stage_of.at(g.rank[i]);
    if (g.task_kind[i] == 0) {
      switch (g.op_class[i]) {
        case TS_OP_LAUNCH: launches.push_back(g.duration[i]); break;
        case TS_OP_EVENT_RECORD: records.push_back(g.duration[i]); break;
        case TS_OP_EVENT_WAIT: waits.push_back(g.duration[i]); break;
        case TS_OP_SYNC: syncs.push_back(g.duration[i]); break;
        default: break;
      }
      continue;
    }
    const TTask& x = tags[i];
    const std::string region = meta_str(x.meta, "region");
    const std::string phase = meta_str(x.meta, "phase");
    const bool mb0 = x.mb.value_or(-1) == 0;
    if (region == "p2p") {
      (meta_str(x.meta, "dir") == "recv" ? recvs : sends).push_back(g.duration[i]);
      if (auto b = meta_i64(x.meta, "bytes")) m.act_bytes = *b;
      continue;
    }
    if (region == "dp") {
      if (auto b = meta_i64(x.meta, "bytes")) m.stage_bytes[stage] += *b;
      m.reduce_name = names.str[g.name[i]];
      continue;
    }
    if (region == "opt") {
      opt_dur[stage] += g.duration[i];
      if (auto b = meta_i64(x.meta, "bytes")) opt_bytes[stage] = *b;
      if (m.optimizer.empty()) m.optimizer.push_back(spec_from(i));
      continue;
    }
    if (x.layer && mb0) {
      (phase == "bwd" ? bwd_groups : fwd_groups)[*x.layer].push_back(i);
      continue;
    }
    if (!mb0) continue;
    if (region == "embed") (phase == "bwd" ? post_bwd : pre_fwd).push_back(i);
    else if (region == "head") (phase == "bwd" ? pre_bwd : post_fwd).push_back(i);
  }
  m.launch = median_of(std::move(launches), m.launch);
  m.record = median_of(std::move(records), m.record);
  m.wait = median_of(std::move(waits), m.wait);
  m.sync = median_of(std::move(syncs), m.sync);
  const int n_layers = w.source_model.n_layers;
  if (static_cast<int>(fwd_groups.size()) != n_layers ||
      static_cast<int>(bwd_groups.size()) != n_layers)
    throw TransformError{"measured " + std::to_string(fwd_groups.size()) + " forward / " +
                         std::to_string(bwd_groups.size()) +
                         " backward layer groups, source model has " + std::to_string(n_layers) +
                         " layers (is the trace tagged?)"};
  for (int l = 0; l < n_layers; ++l) {
    auto fit = fwd_groups.find(l);
    auto bit = bwd_groups.find(l);
    if (fit == fwd_groups.end() || bit == bwd_groups.end())
      throw TransformError{"layer " + std::to_string(l) + " missing from measured groups"};
    m.layer_fwd.push_back(specs_sorted(fit->second));
    m.layer_bwd.push_back(specs_sorted(bit->second));
  }
  m.pre_fwd = specs_sorted(std::move(pre_fwd));
  m.post_fwd = specs_sorted(std::move(post_fwd));
  m.pre_bwd = specs_sorted(std::move(pre_bwd));
  m.post_bwd = specs_sorted(std::move(post_bwd));
  if (!sends.empty()) m.p2p_send = median_of(std::move(sends), 0);
  if (!recvs.empty()) m.p2p_recv_base = *std::min_element(recvs.begin(), recvs.end());
  for (const auto& [stage, bytes] : opt_bytes) m.stage_bytes.try_emplace(stage, bytes);
  if (!opt_dur.empty()) {
    auto it = opt_dur.begin();
    auto bit = m.stage_bytes.find(it->first);
    if (bit != m.stage_bytes.end() && bit->second > 0)
      m.opt_rate = static_cast<double>(it->second) / static_cast<double>(bit->second);
  }
  return m;
}

void set_arg(MetaList& args, const std::string& key, std::string value) {
  for (auto& kv : args)
    if (kv.first == key) {
      kv.second = std::move(value);
      return;
    }
  args.emplace_back(key, std::move(value));
  std::sort(args.begin(), args.end());
}

}  // namespace

bool tag_policy_from_json(const std::string& text, TagPolicyLite& p, std::string& err) {
  try {
    const nlohmann::json j = nlohmann::json::parse(text);
    if (j.contains("layer_keys")) p.layer_keys = j.at("layer_keys").get<std::vector<std::string>>();
    if (j.contains("microbatch_keys"))
      p.microbatch_keys = j.at("microbatch_keys").get<std::vector<std::string>>();
    if (j.contains("phase_keys")) p.phase_keys = j.at("phase_keys").get<std::vector<std::string>>();
    p.infer_from_names = j.value("infer_from_names", p.infer_from_names);
    p.fill_between = j.value("fill_between", p.fill_between);
  } catch (const nlohmann::json::parse_error& e) {
    err = std::string("tag policy is not valid JSON: ") + e.what();
    return false;
  } catch (const std::exception& e) {
    err = e.what();
    return false;
  }
  return true;
}

int rebuild_pipeline(const HostGraph& g, const Names& names, const WhatIfLite& w,
                     PipelineStr& ps, bool& unchanged, std::string& err) {
  ps = PipelineStr{};
  unchanged = false;
  try {
    validate(w);
    const ts_model_config& sm = w.source_model;
    const ts_model_config& tm = w.target_model;
    const ts_par_config& sp = w.source_par;
    const ts_par_config& tp = w.target_par;
    const bool width = sm.d_model != tm.d_model || sm.d_ffn != tm.d_ffn;
    if (sm.n_layers == tm.n_layers && !width && sp.pp == tp.pp && sp.dp == tp.dp &&
        sp.num_microbatches == tp.num_microbatches) {
      unchanged = true;
      return TS_OK;
    }
    if (tm.n_layers % tp.pp != 0)
      throw TransformError{"target layer count must divide evenly across pipeline stages"};
    if (sm.n_layers % sp.pp != 0)
      throw TransformError{"source layer count must divide evenly across pipeline stages"};
    if (g.meta.size() != static_cast<size_t>(g.n()))
      throw TransformError{"source graph carries no task metadata (ingest / generate it with "
                           "keep_meta)"};
    const std::vector<TTask> tags = tag_tasks(g, names, w.policy);
    const Measured meas = measure(g, names, tags, w);

    // target per-layer kernels: clone the last measured layer / drop the tail;
    // GEMMs rescaled by m*n*k for a width change (transform.cpp:575-601)
    auto retime = [&](std::vector<KernelStr> specs) {
      if (!width) return specs;
      for (KernelStr& ks : specs) {
        const std::string* sv[3] = {nullptr, nullptr, nullptr};
        for (const auto& kv : ks.args) {
          if (kv.first == "m") sv[0] = &kv.second;
          else if (kv.first == "n") sv[1] = &kv.second;
          else if (kv.first == "k") sv[2] = &kv.second;
        }
        if (!sv[0] || !sv[1] || !sv[2]) continue;
        int64_t o[3];
        for (int d = 0; d < 3; ++d) {
          try {
            o[d] = std::stoll(*sv[d]);
          } catch (const std::exception& e) {
            throw TransformError{std::string("gemm dims of '") + ks.name + "': " + e.what()};
          }
        }
        if (o[0] <= 0 || o[1] <= 0 || o[2] <= 0) continue;
        const int64_t nm = substitute_dim(o[0], sm, tm), nn = substitute_dim(o[1], sm, tm),
                      nk = substitute_dim(o[2], sm, tm);
        ks.duration = mul_div(ks.duration, nm * nn * nk, o[0] * o[1] * o[2]);
        set_arg(ks.args, "m", std::to_string(nm));
        set_arg(ks.args, "n", std::to_string(nn));
        set_arg(ks.args, "k", std::to_string(nk));
      }
      return specs;
    };
    std::vector<std::vector<KernelStr>> fwd, bwd;
    for (int l = 0; l < tm.n_layers; ++l) {
      const int src = std::min(l, sm.n_layers - 1);
      fwd.push_back(retime(meas.layer_fwd[src]));
      bwd.push_back(retime(meas.layer_bwd[src]));
    }
    ps.pp = tp.pp;
    ps.dp = tp.dp;
    ps.num_microbatches = tp.num_microbatches;
    ps.launch = meas.launch;
    ps.record = meas.record;
    ps.wait = meas.wait;
    ps.sync = meas.sync;
    ps.origin = meas.origin;
    if (tp.pp > 1) {  // stage-boundary transfers (transform.cpp:612-636)
      const int64_t act = meas.act_bytes > 0 ? meas.act_bytes : w.activation_bytes;
      if (act > 0) {
        const int64_t act_t = width ? mul_div(act, tm.d_model, sm.d_model) : act;
        ps.activation_bytes = act_t;
        ps.p2p_send = wire_cost(false, act_t, 2, w.alpha_us, w.bytes_per_us,
                                "boundary transfers");
      } else if (meas.p2p_send >= 0) {
        ps.p2p_send = width ? mul_div(meas.p2p_send, tm.d_model, sm.d_model) : meas.p2p_send;
      } else {
        throw TransformError{
            "cannot size stage-boundary transfers: no p2p kernels in the source trace and no "
            "activation_bytes_per_microbatch in the config"};
      }
      ps.p2p_recv_base = meas.p2p_recv_base >= 0 ? meas.p2p_recv_base : 10;
    }
    // per-stage parameter bytes: the layer share plus the measured vocab
    // tables, rescaled by width (derive_vocab_bytes, transform.cpp:504-530)
    int64_t embed = 0, head = 0;
    if (!meas.stage_bytes.empty()) {
      const int per_stage = sm.n_layers / sp.pp;
      const int64_t b_layer = layer_param_bytes(sm);
      auto stage_total = [&](int s) {
        auto it = meas.stage_bytes.find(s);
        return it == meas.stage_bytes.end() ? int64_t{0} : it->second;
      };
      if (sp.pp >= 2) {
        embed = stage_total(0) - static_cast<int64_t>(per_stage) * b_layer;
        head = stage_total(sp.pp - 1) - static_cast<int64_t>(per_stage) * b_layer;
      } else {
        const int64_t rem = stage_total(0) - static_cast<int64_t>(per_stage) * b_layer;
        head = rem / 2;
        embed = rem - head;
      }
      if (embed < 0 || head < 0)
        throw TransformError{
            "measured gradient bytes are smaller than the source model's layer share"};
    }
    const int64_t b_layer_t = layer_param_bytes(tm);
    const int64_t embed_t = sm.d_model > 0 ? mul_div(embed, tm.d_model, sm.d_model) : embed;
    const int64_t head_t = sm.d_model > 0 ? mul_div(head, tm.d_model, sm.d_model) : head;
    const int per_stage_t = tm.n_layers / tp.pp;
    for (int s = 0; s < tp.pp; ++s) {
      StageStr st;
      for (int l = 0; l < per_stage_t; ++l) {
        st.layers_fwd.push_back(fwd[static_cast<size_t>(s * per_stage_t + l)]);
        st.layers_bwd.push_back(bwd[static_cast<size_t>(s * per_stage_t + l)]);
      }
      if (s == 0) {
        st.pre_fwd = meas.pre_fwd;
        st.post_bwd = meas.post_bwd;
      }
      if (s == tp.pp - 1) {
        st.post_fwd = meas.post_fwd;
        st.pre_bwd = meas.pre_bwd;
      }
      const int64_t stage_bytes = static_cast<int64_t>(per_stage_t) * b_layer_t +
                                  (s == 0 ? embed_t : 0) + (s == tp.pp - 1 ? head_t : 0);
      if (tp.dp > 1) {
        if (meas.stage_bytes.empty())
          throw TransformError{
              "cannot size gradient collectives: source trace carries no byte counts"};
        KernelStr ar;
        ar.name = meas.reduce_name;
        ar.op_class = TS_OP_COMMUNICATION;
        ar.duration = wire_cost(true, stage_bytes, tp.dp, w.alpha_us, w.bytes_per_us,
                                "gradient collectives");
        ar.args = {{"bytes", std::to_string(stage_bytes)},
                   {"collective", "allreduce"},
                   {"group_size", std::to_string(tp.dp)}};
        st.reduce.push_back(std::move(ar));
      }
      if (!meas.optimizer.empty() && meas.opt_rate > 0.0) {
        KernelStr opt = meas.optimizer.front();
        opt.duration = static_cast<int64_t>(
            std::llround(meas.opt_rate * static_cast<double>(stage_bytes)));
        set_arg(opt.args, "bytes", std::to_string(stage_bytes));
        st.optimizer.push_back(std::move(opt));
      }
      ps.stages.push_back(std::move(st));
    }
  } catch (const TransformError& e) {
    err = e.msg;
    ps = PipelineStr{};
    return TS_E_INVALID_ARGUMENT;
  }
  return TS_OK;
}

}  // namespace lumos
