// capi_host.cpp — extern "C" entry points of the host-side graph sources
// (synthetic generator, trace-event graph builder); see include/lumos_b200.h.
#include <cstdlib>
#include <cstring>
#include <deque>
#include <fstream>
#include <sstream>
#include <map>
#include <string>
#include <vector>

#include "ingest.hpp"
#include "lumos_b200.h"
#include "rebuild.hpp"
#include "synth.hpp"
#include "trace_ingest.hpp"

using namespace lumos;

struct ts_host_graph {
  SynthOutput s;
};

// a rebuilt PipelineSpec and the POD view of it (pointers into `p`)
struct ts_pipeline {
  lumos::PipelineStr p;
  ts_pipeline_spec spec{};
  std::vector<ts_stage_spec> stages;
  std::deque<std::vector<ts_kernel_spec>> kernels;
  std::deque<std::vector<ts_kernel_list>> layers;
  std::deque<std::vector<const char*>> strs;
};

namespace lumos {
int set_error(int code, const std::string& msg);  // capi.cpp
}

extern "C" {

void ts_synth_defaults(ts_synth_spec* spec) {
  if (spec) synth_defaults(spec);
}

int ts_synth_graph(const ts_synth_spec* spec, ts_host_graph** out, int64_t* truth_makespan) {
  if (!spec || !out) return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  auto* h = new ts_host_graph;
  std::string err;
  int rc = synth_graph(*spec, h->s, err);
  if (rc != TS_OK) {
    delete h;
    *out = nullptr;
    return set_error(rc, err);
  }
  if (truth_makespan) *truth_makespan = h->s.truth_makespan;
  *out = h;
  return TS_OK;
}

void ts_pipeline_defaults(ts_pipeline_spec* spec) {
  if (spec) pipeline_defaults(spec);
}

int ts_pipeline_graph(const ts_pipeline_spec* spec, int32_t estimate, int32_t tp,
                      ts_host_graph** out, int64_t* truth_makespan) {
  if (!spec || !out) return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  auto* h = new ts_host_graph;
  std::string err;
  int rc = pipeline_graph(*spec, estimate != 0, tp, h->s, err);
  if (rc != TS_OK) {
    delete h;
    *out = nullptr;
    return set_error(rc, err);
  }
  if (truth_makespan) *truth_makespan = h->s.truth_makespan;
  *out = h;
  return TS_OK;
}

int ts_host_graph_desc(const ts_host_graph* g, ts_graph_desc* out) {
  if (!g || !out) return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  *out = g->s.graph.desc();
  return TS_OK;
}

int ts_host_graph_op_index(const ts_host_graph* g, int64_t* out) {
  if (!g || !out) return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  std::memcpy(out, g->s.graph.op_index.data(), g->s.graph.op_index.size() * sizeof(int64_t));
  return TS_OK;
}

int64_t ts_host_graph_n_ops(const ts_host_graph* g) { return g ? g->s.n_ops : 0; }

int ts_host_graph_name_ids(const ts_host_graph* g, int32_t* out) {
  if (!g || !out) return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  std::memcpy(out, g->s.graph.name.data(), g->s.graph.name.size() * sizeof(int32_t));
  return TS_OK;
}

const char* ts_host_graph_name(const ts_host_graph* g, int32_t id) {
  if (!g || id < 0 || id >= static_cast<int32_t>(g->s.names.str.size())) return "";
  return g->s.names.str[id].c_str();
}

void ts_host_graph_free(ts_host_graph* g) { delete g; }

static int ingest(IngestOptions opts, ts_host_graph** out) {
  // LUMOS_INGEST_DOM=1 parses every file on the DOM path (the fast scanner's check)
  const char* dom = std::getenv("LUMOS_INGEST_DOM");
  opts.dom_only = dom && dom[0] == '1';
  auto* h = new ts_host_graph;
  std::vector<RtMeta> rt;
  std::string err;
  const int rc = ingest_traces(opts, h->s.names, h->s.graph, rt, err);
  if (rc != TS_OK) {
    delete h;
    *out = nullptr;
    return set_error(rc, err);
  }
  fill_retime_arrays(h->s.graph, rt);
  *out = h;
  return TS_OK;
}

static bool read_text(const char* path, std::string& text, std::string& err) {
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    err = std::string("cannot open '") + path + "'";
    return false;
  }
  std::ostringstream os;
  os << in.rdbuf();
  text = os.str();
  return true;
}

int ts_ingest_traces(const char* const* paths, int32_t n_paths, int32_t n_threads,
                     int64_t gap_threshold_us, ts_host_graph** out) {
  if (!out || (n_paths > 0 && !paths)) return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  IngestOptions o;
  for (int32_t i = 0; i < n_paths; ++i) o.paths.emplace_back(paths[i] ? paths[i] : "");
  o.threads = n_threads;
  o.policy.gap_threshold_us = gap_threshold_us;
  return ingest(o, out);
}

int ts_ingest_traces_ex(const ts_ingest_options* opt, ts_host_graph** out) {
  if (!opt || !out || (opt->n_paths > 0 && !opt->paths))
    return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  IngestOptions o;
  for (int32_t i = 0; i < opt->n_paths; ++i) o.paths.emplace_back(opt->paths[i] ? opt->paths[i] : "");
  o.threads = opt->n_threads;
  if (opt->manifest) o.manifest = opt->manifest;
  if (opt->window) o.window = opt->window;
  o.keep_meta = opt->keep_meta != 0;
  std::string err, text;
  if (opt->categories_path) {
    if (!read_text(opt->categories_path, text, err) || !categories_from_json(text, o.categories, err))
      return set_error(TS_E_INVALID_ARGUMENT, err);
  }
  if (opt->policy_path) {
    if (!read_text(opt->policy_path, text, err) || !policy_from_json(text, o.policy, err))
      return set_error(TS_E_INVALID_ARGUMENT, err);
  }
  return ingest(o, out);
}

static void build_pod(ts_pipeline& h) {
  auto list = [&](const std::vector<KernelStr>& ks) {
    h.kernels.emplace_back();
    std::vector<ts_kernel_spec>& v = h.kernels.back();
    for (const KernelStr& k : ks) {
      h.strs.emplace_back();
      std::vector<const char*>& kv = h.strs.back();
      for (const auto& a : k.args) kv.push_back(a.first.c_str());
      for (const auto& a : k.args) kv.push_back(a.second.c_str());
      const int32_t na = static_cast<int32_t>(k.args.size());
      v.push_back({k.name.c_str(), k.duration, k.op_class, na, kv.data(), kv.data() + na});
    }
    return ts_kernel_list{v.data(), static_cast<int32_t>(v.size()), 0};
  };
  const PipelineStr& p = h.p;
  pipeline_defaults(&h.spec);
  h.stages.resize(p.stages.size());
  for (size_t s = 0; s < p.stages.size(); ++s) {
    const StageStr& st = p.stages[s];
    ts_stage_spec& c = h.stages[s];
    c.n_layers = static_cast<int32_t>(st.layers_fwd.size());
    h.layers.emplace_back();
    std::vector<ts_kernel_list>& lf = h.layers.back();
    for (const auto& l : st.layers_fwd) lf.push_back(list(l));
    h.layers.emplace_back();
    std::vector<ts_kernel_list>& lb = h.layers.back();
    for (const auto& l : st.layers_bwd) lb.push_back(list(l));
    c.layers_fwd = lf.data();
    c.layers_bwd = lb.data();
    c.pre_fwd = list(st.pre_fwd);
    c.post_fwd = list(st.post_fwd);
    c.pre_bwd = list(st.pre_bwd);
    c.post_bwd = list(st.post_bwd);
    c.reduce = list(st.reduce);
    c.optimizer = list(st.optimizer);
  }
  h.spec.pp = p.pp;
  h.spec.dp = p.dp;
  h.spec.num_microbatches = p.num_microbatches;
  h.spec.n_stages = static_cast<int32_t>(h.stages.size());
  h.spec.stages = h.stages.data();
  h.spec.launch_us = p.launch;
  h.spec.record_us = p.record;
  h.spec.wait_us = p.wait;
  h.spec.sync_us = p.sync;
  h.spec.p2p_send_us = p.p2p_send;
  h.spec.p2p_recv_base_us = p.p2p_recv_base;
  h.spec.activation_bytes = p.activation_bytes;
  h.spec.origin = p.origin;
}

int ts_host_graph_from_tasks(const ts_graph_desc* d, const char* const* names,
                             const int64_t* corr, const int32_t* meta_off,
                             const char* const* meta_keys, const char* const* meta_values,
                             ts_host_graph** out) {
  if (!d || !out || d->n_tasks < 0 || (d->n_tasks > 0 && (!d->duration || !d->original_start ||
                                                          !d->rank || !d->lane_kind || !d->lane ||
                                                          !d->op_class || !d->task_kind)))
    return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  auto* h = new ts_host_graph;
  HostGraph& g = h->s.graph;
  const int32_t n = d->n_tasks;
  g.duration.assign(d->duration, d->duration + n);
  g.original_start.assign(d->original_start, d->original_start + n);
  g.rank.assign(d->rank, d->rank + n);
  g.lane_kind.assign(d->lane_kind, d->lane_kind + n);
  g.lane.assign(d->lane, d->lane + n);
  g.op_class.assign(d->op_class, d->op_class + n);
  g.task_kind.assign(d->task_kind, d->task_kind + n);
  if (d->n_edges > 0 && d->edge_from && d->edge_to) {
    g.edge_from.assign(d->edge_from, d->edge_from + d->n_edges);
    g.edge_to.assign(d->edge_to, d->edge_to + d->n_edges);
  }
  if (d->n_rules > 0 && d->rule_kind && d->rule_task && d->rule_bound && d->rule_watch_off) {
    g.rule_kind.assign(d->rule_kind, d->rule_kind + d->n_rules);
    g.rule_task.assign(d->rule_task, d->rule_task + d->n_rules);
    g.rule_bound.assign(d->rule_bound, d->rule_bound + d->n_rules);
    g.rule_watch_off.assign(d->rule_watch_off, d->rule_watch_off + d->n_rules + 1);
    const int32_t nw = d->rule_watch_off[d->n_rules];
    if (nw > 0 && d->watch_rank && d->watch_kind && d->watch_lane) {
      g.watch_rank.assign(d->watch_rank, d->watch_rank + nw);
      g.watch_kind.assign(d->watch_kind, d->watch_kind + nw);
      g.watch_lane.assign(d->watch_lane, d->watch_lane + nw);
    }
  }
  g.window_start = d->window_start;
  g.window_end = d->window_end;
  g.op_index.assign(n, -1);
  g.name.resize(n);
  for (int32_t t = 0; t < n; ++t) g.name[t] = h->s.names.get(names && names[t] ? names[t] : "");
  g.corr.assign(n, -1);
  if (corr) g.corr.assign(corr, corr + n);
  g.meta.assign(n, MetaList{});
  if (meta_off && meta_keys && meta_values)
    for (int32_t t = 0; t < n; ++t) {
      std::map<std::string, std::string> m;
      for (int32_t k = meta_off[t]; k < meta_off[t + 1]; ++k)
        m[meta_keys[k] ? meta_keys[k] : ""] = meta_values[k] ? meta_values[k] : "";
      g.meta[t].assign(m.begin(), m.end());
    }
  *out = h;
  return TS_OK;
}

int ts_rebuild_pipeline(const ts_host_graph* source, const ts_whatif* w, ts_pipeline** out) {
  if (!source || !w || !out) return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  WhatIfLite wl;
  wl.source_model = w->source_model;
  wl.target_model = w->target_model;
  wl.source_par = w->source_par;
  wl.target_par = w->target_par;
  wl.alpha_us = w->alpha_us;
  wl.bytes_per_us = w->bytes_per_us;
  wl.activation_bytes = w->activation_bytes;
  std::string err;
  if (w->tag_policy_json && !tag_policy_from_json(w->tag_policy_json, wl.policy, err))
    return set_error(TS_E_INVALID_ARGUMENT, err);
  auto* h = new ts_pipeline;
  bool unchanged = false;
  const int rc = rebuild_pipeline(source->s.graph, source->s.names, wl, h->p, unchanged, err);
  if (rc != TS_OK || unchanged) {
    delete h;
    return rc == TS_OK ? TS_OK : set_error(rc, err);
  }
  build_pod(*h);
  *out = h;
  return TS_OK;
}

const ts_pipeline_spec* ts_pipeline_spec_get(const ts_pipeline* p) { return p ? &p->spec : nullptr; }

void ts_pipeline_free(ts_pipeline* p) { delete p; }

int ts_build_rank_graph(int32_t rank, int64_t n_events, const int32_t* name, const uint8_t* cat,
                        const int64_t* ts, const int64_t* dur, const int32_t* tid,
                        const int64_t* corr, const int32_t* stream, const int64_t* arg_event,
                        const int64_t* arg_stream, const char* names, int64_t gap_threshold_us,
                        ts_host_graph** inout) {
  if (!inout || (n_events > 0 && (!name || !cat || !ts || !dur || !tid || !names)))
    return set_error(TS_E_INVALID_ARGUMENT, "null argument");
  ts_host_graph* h = *inout ? *inout : new ts_host_graph;
  // the name table of the incoming events
  std::vector<int32_t> remap;
  {
    const char* p = names;
    while (*p) {
      const char* q = std::strchr(p, '\n');
      std::string s = q ? std::string(p, q) : std::string(p);
      remap.push_back(h->s.names.get(s));
      if (!q) break;
      p = q + 1;
    }
  }
  std::vector<Event> evs(static_cast<size_t>(n_events));
  for (int64_t i = 0; i < n_events; ++i) {
    Event& e = evs[i];
    if (name[i] < 0 || name[i] >= static_cast<int32_t>(remap.size())) {
      if (!*inout) delete h;
      return set_error(TS_E_INVALID_ARGUMENT, "event name id out of range");
    }
    e.name = remap[name[i]];
    e.cat = cat[i];
    e.ts = ts[i];
    e.dur = dur[i];
    e.pid = rank;
    e.tid = tid[i];
    e.corr = corr ? corr[i] : -1;
    e.stream = stream ? stream[i] : -1;
    e.arg_event = arg_event ? arg_event[i] : kNoArg;
    e.arg_stream = arg_stream ? arg_stream[i] : kNoArg;
  }
  HostGraph g;
  std::string err;
  BuildPolicyLite pol;
  pol.gap_threshold_us = gap_threshold_us > 0 ? gap_threshold_us : 1000;
  int rc = build_rank_graph(evs, h->s.names, rank, pol, g, err);
  if (rc != TS_OK) {
    if (!*inout) delete h;
    return set_error(rc, err);
  }
  const bool first = h->s.graph.n() == 0 && h->s.graph.rule_kind.empty();
  h->s.graph.append(g, first);
  *inout = h;
  return TS_OK;
}

}  // extern "C"
