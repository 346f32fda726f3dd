/*
 * lumos_b200.h — C ABI of the B200-native batched Lumos replay engine.
 *
 * This is the drop-in boundary for the reference's simulation path
 * (/root/reference/proj, the `tracesim` library).  Every entry point replaces
 * one reference interface; the citation is on each declaration.  Only PODs
 * cross the boundary: int64 microseconds (types.hpp:15), int32 task ids
 * (types.hpp:16), plain pointers and sizes.  No torch, no C++ types.
 *
 *   reference                                            here
 *   ---------------------------------------------------  ------------------------
 *   ExecutionGraph (build.hpp:73-85), Task (types.hpp:73-87),
 *   RuntimeRule (build.hpp:46-54)                        ts_graph_desc
 *   validate_graph + Engine ctor (simulate.cpp:26-196)   ts_graph_create
 *   simulate(const ExecutionGraph&) (simulate.hpp:51)    ts_simulate
 *   N x simulate over perturbed copies / DurationHook
 *     (pipeline.hpp:72-74, synth.cpp:146-156)           ts_replay_batch
 *   makespan (simulate.cpp:327-334), breakdown_by_rank
 *     (metrics.cpp:96-103)                               ts_result fields
 *   SimulationError / GraphError (types.hpp:119-127)     TS_E_* codes + ts_last_error
 *
 * Error behaviour mirrors the reference taxonomy: every call returns 0 on
 * success or a TS_E_* code; the message (same wording as the reference's
 * exception text where one exists) is kept per thread in ts_last_error().
 *
 * Pointers in ts_scenarios / ts_result may be host or device memory; the
 * library detects which (cudaPointerGetAttributes) and stages host buffers
 * itself.  There is no CPU execution path: without a CUDA device every compute
 * call fails with TS_E_CUDA.
 *
 * Threading (the reference's contract): distinct ts_graph handles
 * may be used concurrently from different host threads / CUDA streams; one
 * handle serves one call at a time (it owns the call's staging buffers).
 */
#ifndef LUMOS_B200_H
#define LUMOS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 5

/* error codes (0 = success) */
enum {
  TS_OK = 0,
  TS_E_INVALID_ARGUMENT = 1, /* std::invalid_argument                          */
  TS_E_SIMULATION = 3,       /* tracesim::SimulationError (invalid graph, deadlock) */
  TS_E_GRAPH = 4,            /* tracesim::GraphError (cycle)                   */
  TS_E_UNSUPPORTED = 6,      /* graph outside what the device path accepts      */
  TS_E_CUDA = 7,             /* no device / CUDA runtime failure               */
  TS_E_NOMEM = 8
};

/* lane kinds (types.hpp:41), rule kinds (build.hpp:47), op classes (types.hpp:31-39) */
enum { TS_LANE_CPU_THREAD = 0, TS_LANE_CUDA_STREAM = 1 };
enum { TS_RULE_STREAM_SYNC = 0, TS_RULE_DEVICE_SYNC = 1, TS_RULE_EVENT_SYNC = 2 };
enum {
  TS_OP_COMPUTE = 0, TS_OP_COMMUNICATION = 1, TS_OP_LAUNCH = 2, TS_OP_SYNC = 3,
  TS_OP_EVENT_RECORD = 4, TS_OP_EVENT_WAIT = 5, TS_OP_OTHER = 6
};
/* gate kinds (estimate()/generator semantics, pipeline.cpp:377-389) */
enum { TS_GATE_FIN = 0, TS_GATE_START = 1 };

/*
 * SoA view of one ExecutionGraph.  Task ids are dense: task i is row i.
 * fixed edges are finish->start (build.hpp:71).  Rules: watch lists are
 * rule_watch_off[r] .. rule_watch_off[r+1] into watch_{rank,kind,lane};
 * rule_bound[r] = -1 when an EventSync has no bound task.
 *
 * Gates (optional, n_gates = 0 for plain replay) carry the generator /
 * estimate() semantics of build_pipeline (pipeline.cpp:361-441) that a
 * recorded trace bakes into durations:  finish(v) = max(start(v), gate
 * values) + duration(v), a gate value being finish(from) (TS_GATE_FIN:
 * p2p receive waits for its send) or start(from) (TS_GATE_START:
 * a collective ends at the latest start of its group plus its own time).
 */
typedef struct {
  int32_t n_tasks;
  const int64_t* duration;       /* [n] base duration, us                 */
  const int64_t* original_start; /* [n] recorded start, us (tie-break key) */
  const int32_t* rank;           /* [n] ProcessorId.rank                   */
  const int32_t* lane_kind;      /* [n] TS_LANE_*                          */
  const int32_t* lane;           /* [n] thread id or stream id             */
  const uint8_t* op_class;       /* [n] TS_OP_*                            */
  const uint8_t* task_kind;      /* [n] 0 Cpu, 1 Gpu (types.hpp:29)        */
  const uint8_t* scale_class;    /* [n] scenario class 0..3, or NULL:
                                    0 host task, 1 GPU compute, 2 GPU comm */
  int64_t n_edges;
  const int32_t* edge_from;
  const int32_t* edge_to;
  int32_t n_rules;
  const int32_t* rule_kind;
  const int32_t* rule_task;
  const int32_t* rule_bound;
  const int32_t* rule_watch_off; /* [n_rules + 1] */
  const int32_t* watch_rank;
  const int32_t* watch_kind;
  const int32_t* watch_lane;
  int64_t window_start;          /* iteration_window (trace_parse.hpp:65-68) */
  int64_t window_end;
  int64_t n_gates;
  const int32_t* gate_from;
  const int32_t* gate_to;
  const uint8_t* gate_kind;      /* TS_GATE_* */
  /* Optional retime metadata (Task.meta keys bytes / collective / group_size /
   * m n k / region / dir, types.hpp:84-86), NULL when absent; needed only by
   * ts_retime scenarios.  rt_kind classifies each task the way change_hidden
   * and scale_dp read its metadata (transform.cpp:219-349). */
  const uint8_t* rt_kind;        /* [n] TS_RT_*                                 */
  const int64_t* rt_bytes;       /* [n] meta "bytes" (0 when absent)            */
  const int32_t* rt_group;       /* [n] meta "group_size" (0 when absent)       */
  const int64_t* rt_mnk;         /* [n][3] meta m, n, k (0 when absent)         */
} ts_graph_desc;

/* retime classes of a task (transform.cpp:279-349, scale_dp :219-258) */
enum {
  TS_RT_NONE = 0,
  TS_RT_GEMM = 1,       /* GPU compute with m, n, k > 0                        */
  TS_RT_OPT = 2,        /* GPU compute, region "opt", with bytes               */
  TS_RT_ALLREDUCE = 3,  /* GPU communication, collective "allreduce", bytes    */
  TS_RT_P2P_SEND = 4,   /* GPU communication, region "p2p", bytes, dir != recv */
  TS_RT_P2P_RECV = 5    /* GPU communication, region "p2p", bytes, dir == recv */
};

typedef struct ts_graph ts_graph;

typedef struct {
  int32_t n_tasks;
  int32_t n_components;   /* independent sub-graphs (ranks in plain replay)   */
  int32_t n_programs;     /* distinct compiled programs after de-duplication   */
  int32_t n_ranks;
  int32_t n_streams;      /* CUDA-stream lanes over all ranks                  */
  int32_t max_slots;      /* live int64 values per scenario (shared memory)    */
  int64_t program_bytes;  /* device bytes of the op streams                    */
  int64_t n_ops;          /* ops over all programs                             */
  int32_t n_syncs;        /* Stream/DeviceSync rules resolved statically       */
  int32_t n_gpu_tasks;
  int64_t window_start, window_end;
  int32_t n_fused_ranks;  /* ranks on the split breakdown accounting (|A| summed
                             by the walk, only candidate kernels re-read)     */
  int32_t des_only;       /* 1: every scenario takes the event-driven path */
  int64_t n_candidates;   /* compute kernels the split accounting re-reads   */
} ts_graph_info;

/* validate_graph + compile to device programs (simulate.cpp:26-196).
 * Returns TS_E_SIMULATION for graphs simulate() rejects ("invalid graph: ..."),
 * TS_E_UNSUPPORTED for graphs outside the device path's class (unchained
 * lanes, rules watching CPU lanes).  device < 0: current device. */
int ts_graph_create(const ts_graph_desc* desc, int device, ts_graph** out);
void ts_graph_destroy(ts_graph* g);
int ts_graph_get_info(const ts_graph* g, ts_graph_info* out);
/* rank of each rank slot (breakdown rows), stream lane of each stream slot */
int ts_graph_ranks(const ts_graph* g, int32_t* ranks /* [n_ranks] */);
int ts_graph_streams(const ts_graph* g, int32_t* rank, int32_t* lane /* [n_streams] */);

/* Scenario batch: durations are a pure function of (spec, scenario id, task),
 * so any shard or tile reproduces bit-for-bit.
 *   class scale (transform.cpp:38-43): d = mul_div(d, num, scale_den), with
 *     num = scale_num[s][class] if given, else drawn in [scale_lo, scale_hi]
 *   jitter      (synth.cpp:150-155):   d = d == 0 ? 0 : max(1, llround(d*(1+u))),
 *     u = jitter * (2 * w / 2^32 - 1), w = word (s & 1) of
 *     Philox2x32-10(ctr = (task, s >> 1); seed): one call per scenario pair
 *   explicit: durations[task * durations_ld + s] replaces both.          */
typedef struct {
  int64_t first;            /* global id of scenario 0 of this batch */
  int32_t count;
  int32_t flags;            /* reserved, 0 */
  uint64_t seed;
  double jitter;            /* 0 disables */
  int32_t scale_lo, scale_hi, scale_den; /* den <= 0 disables */
  int32_t n_classes;        /* columns of scale_num (<= 4) */
  const int32_t* scale_num; /* [count][n_classes] or NULL */
  const int64_t* durations; /* [n_tasks][durations_ld] or NULL */
  int64_t durations_ld;
  const struct ts_retime* retime; /* per-scenario what-if retime, or NULL */
} ts_scenarios;

/* Device-side what-if retiming: scenario s replays the
 * graph apply_whatif would return for a width / data-parallel change that
 * needs no pipeline rebuild (transform.cpp:713-760): change_hidden
 * (transform.cpp:279-349) then scale_dp (:219-258), with the analytical cost
 * model collective_cost_us (cost.cpp:55-62) at that scenario's alpha / beta.
 * Class scale and jitter then apply to the retimed durations.  All arrays
 * are host memory, [count] entries (target_model [count][3]).  Errors follow
 * the reference's TransformError messages (TS_E_INVALID_ARGUMENT). */
typedef struct ts_retime {
  const double* alpha_us;       /* [count] cost model alpha (us)              */
  const double* bytes_per_us;   /* [count] cost model bandwidth (> 0)         */
  int32_t source_dp;            /* scale_dp: collectives sized for this group  */
  int32_t pad;
  const int32_t* target_dp;     /* [count] or NULL: no data-parallel retime   */
  int64_t source_model[3];      /* change_hidden source {d_model, d_ffn, n_params} */
  const int64_t* target_model;  /* [count][3] or NULL: no width retime        */
} ts_retime;

/* Outputs; any pointer may be NULL (not produced).  start/fin are the
 * SimEntry sim_start/sim_end (simulate.hpp:12-17) of every task, stored
 * scenario-major within a task row: start[task * ld + s]. */
typedef struct {
  int64_t* start;          /* [n_tasks][ld] */
  int64_t* fin;            /* [n_tasks][ld] */
  int64_t ld;              /* >= count */
  int64_t* span;           /* [count][3] SimulatedTrace {start, end, makespan} */
  int64_t* rank_breakdown; /* [count][n_ranks][5] {total, exposed_compute,
                              exposed_comm, overlapped, other} (metrics.hpp:33-39) */
  int64_t* stream_busy;    /* [count][n_streams] summed kernel time per stream */
  int32_t* status;         /* [count] 0 = exact fast path, 1 = resolved by the
                              exact event-driven path, <0 = error */
  /* utilization_by_rank (metrics.cpp:105-155) over the breakdown's window
   * [W, max(window.end, W + makespan)): per rank, the microseconds of bin b
   * = [W + b*w, min(W + (b+1)*w, end)) covered by >= 1 kernel on any of the
   * rank's streams (value = covered / bin span, computed by the caller). */
  int64_t util_bin_width;  /* w > 0 to produce util_covered */
  int32_t util_max_bins;   /* bins stored per rank; a window needing more fails
                              the call (TS_E_INVALID_ARGUMENT, message names the
                              bins needed) after util_n_bins is written */
  int32_t util_pad;
  int64_t* util_covered;   /* [count][n_ranks][util_max_bins] */
  int32_t* util_n_bins;    /* [count] bins the window needs */
  /* compare_replay (metrics.cpp:189-221): delta = sim_start - original_start */
  int64_t* delta_abs_sum;  /* [count] sum of |delta| over all tasks (exact int64;
                              the reference's double sum equals it below 2^53) */
  int64_t* delta_worst;    /* [count][delta_worst_n][3] {|delta|, task, delta}:
                              the report's worst list, largest |delta| first,
                              ties by smaller task id (metrics.cpp:213-217);
                              task -1 pads a graph with fewer tasks */
  int32_t delta_worst_n;   /* entries per scenario, 1..64 (0 means 1); the
                              reference's default is 10 (metrics.hpp:82-83) */
  int32_t host_async;      /* 1: host output buffers are filled by copies on the
                              graph's copy stream that overlap the next call's
                              kernels; the call returns once they are enqueued and
                              ts_graph_wait() blocks until they have landed (calls
                              that must read a status back stay synchronous) */
  int32_t* n_fixups;       /* [1] scenarios of this call re-run by the exact
                              event-driven path (failed sync certificates), or NULL */
} ts_result;

/* Replays `sc->count` scenarios on `stream` (cudaStream_t, NULL = legacy
 * default).  Returns after the work is enqueued when every output pointer is
 * device memory; otherwise it synchronises and copies to the host buffers. */
int ts_replay_batch(ts_graph* g, const ts_scenarios* sc, const ts_result* out, void* stream);
/* waits for the host copies of ts_result.host_async calls */
int ts_graph_wait(ts_graph* g);

/* simulate(const ExecutionGraph&) (simulate.hpp:51): one replay at the
 * graph's own durations; host buffers start/fin [n_tasks], span[3]. */
int ts_simulate(ts_graph* g, int64_t* start, int64_t* fin, int64_t* span);

/* Materialises the scenario durations (the K4 manipulation kernel on its
 * own) into dur[task * ld + s] (device or host pointer). */
int ts_scenario_durations(ts_graph* g, const ts_scenarios* sc, int64_t* dur, int64_t ld,
                          void* stream);

/* ---------------------------------------------------------------------------
 * Host-side graph sources (the input contract of the replay path).
 *
 * ts_synth_graph restates the reference generator (synth.cpp:71-170,
 * pipeline.cpp:9-477): the one-iteration trace of a GPT-like model under
 * pp x dp 1F1B pipelining, as either
 *   estimate = 0: the replay graph build_graph + merge_ranks produce from that
 *                 trace (what `tracesim replay` simulates), or
 *   estimate = 1: the generator's own dependency graph with intrinsic
 *                 durations and gates (p2p rendezvous, collective barrier) —
 *                 the semantics of build_pipeline(spec, DurationHook).
 * tp > 1 replicates every (stage, dp) rank as TP replicas r * tp + t (the
 * reference generator itself rejects tp != 1, synth.cpp:18-19).
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t n_layers, d_model, d_ffn, n_heads, d_head;
  int32_t tp, pp, dp, num_microbatches;
  int64_t tokens_per_microbatch, vocab;
  int64_t launch_us, record_us, wait_us, sync_us;  /* SynthCosts, synth.hpp:17-34 */
  int64_t gemm_ref_us, gemm_ref_mnk;
  double bwd_gemm_factor;
  int64_t attn_misc_us, embed_us, head_us, loss_grad_us;
  int64_t optimizer_ref_us, optimizer_ref_bytes;
  double alpha_us, bytes_per_us;
  int64_t p2p_recv_base_us;
  int64_t origin;
  int32_t estimate;   /* 0 replay graph, 1 estimate graph */
  int32_t slice_rank; /* -1 all ranks; else slice_rank (build.cpp:544-580) */
  int32_t keep_meta;  /* replay graph: keep Task.meta + correlation ids (the
                         source of a structural what-if, ts_rebuild_pipeline) */
  int32_t pad;
} ts_synth_spec;

typedef struct ts_host_graph ts_host_graph;

/* fills the reference defaults (SynthSpec::from_json, synth.cpp:195-247) */
void ts_synth_defaults(ts_synth_spec* spec);
int ts_synth_graph(const ts_synth_spec* spec, ts_host_graph** out, int64_t* truth_makespan);
/* SoA view of a host graph; pointers stay valid while the graph lives */
int ts_host_graph_desc(const ts_host_graph* g, ts_graph_desc* out);
/* per task: the generator cost index (DurationHook op_index) or -1 */
int ts_host_graph_op_index(const ts_host_graph* g, int64_t* out);
int64_t ts_host_graph_n_ops(const ts_host_graph* g);
/* per task: name id; ts_host_graph_name(g, id) returns the string */
int ts_host_graph_name_ids(const ts_host_graph* g, int32_t* out);
const char* ts_host_graph_name(const ts_host_graph* g, int32_t name_id);
void ts_host_graph_free(ts_host_graph* g);

/* Mode-B boundary: the reference's PipelineSpec (pipeline.hpp:27-90) as
 * PODs, for graphs with the generator / estimate() semantics of
 * build_pipeline(spec, DurationHook) (pipeline.cpp:474-477) — the spec
 * rebuild_pipeline constructs for a structural what-if (transform.cpp:556-701)
 * or any hand-written one.  A kernel's args (KernelSpec::args) travel onto its
 * task's metadata with the builder's tags (pipeline.cpp:122-123, 229-297);
 * kernels are classified by name as build_graph does (build.cpp:93-98), so
 * op_class is informational (the reference's events do not carry it). */
typedef struct {
  const char* name;
  int64_t duration;              /* KernelSpec::duration, us (negative -> 0) */
  int32_t op_class;              /* KernelSpec::op_class (informational)     */
  int32_t n_args;
  const char* const* arg_keys;   /* KernelSpec::args                          */
  const char* const* arg_values;
} ts_kernel_spec;
typedef struct {
  const ts_kernel_spec* k;
  int32_t n;
  int32_t pad;
} ts_kernel_list;
typedef struct {                 /* StageSpec (pipeline.hpp:34-43) */
  int32_t n_layers;
  int32_t pad;
  const ts_kernel_list* layers_fwd; /* [n_layers] */
  const ts_kernel_list* layers_bwd; /* [n_layers], layer order (run back to front) */
  ts_kernel_list pre_fwd, post_fwd, pre_bwd, post_bwd, reduce, optimizer;
} ts_stage_spec;
typedef struct {                 /* PipelineSpec (pipeline.hpp:52-70) */
  int32_t pp, dp, num_microbatches, n_stages;
  const ts_stage_spec* stages;   /* [n_stages], n_stages must equal pp */
  int64_t launch_us, record_us, wait_us, sync_us;  /* HostCosts */
  int64_t p2p_send_us, p2p_recv_base_us, activation_bytes, origin;
  int32_t compute_stream, reduce_stream, p2p_stream, main_thread, helper_thread, pad;
  int64_t first_event, first_correlation;
} ts_pipeline_spec;
/* PipelineSpec's defaults (HostCosts 5/2/2/5 us, streams 7/9/11, threads 100/200) */
void ts_pipeline_defaults(ts_pipeline_spec* spec);
/* build_pipeline(spec) as a graph: estimate = 1 the generator's dependency
 * graph with gates (what estimate_batch replays), 0 the replay graph of its
 * trace (build_graph + merge_ranks).  tp > 1 adds TP replicas r * tp + t.
 * truth_makespan = BuiltPipeline end - origin at the base durations.  Errors
 * follow build_pipeline's std::invalid_argument (TS_E_INVALID_ARGUMENT). */
int ts_pipeline_graph(const ts_pipeline_spec* spec, int32_t estimate, int32_t tp,
                      ts_host_graph** out, int64_t* truth_makespan);

/* Structural what-if (estimate()'s host step): the PipelineSpec the
 * reference's rebuild_pipeline (transform.cpp:556-701) constructs from a
 * measured source graph — tag_tasks (:71-162), measure_pipeline (:378-502),
 * derive_vocab_bytes (:504-530), target stages with an AnalyticalCostModel —
 * for scale_pp / change_layers / apply_whatif's structural branch
 * (transform.hpp:56-72).  The source must keep its Task.meta (ts_synth_spec /
 * ts_ingest_options keep_meta).  *out = NULL with TS_OK when the target
 * differs in nothing the rebuild cares about (the reference returns the
 * source graph).  Replay the result with ts_pipeline_graph (estimate = 1 for
 * batched estimate(), 0 for the replay graph build_pipeline + graph_from_events
 * yields).  Errors: TS_E_INVALID_ARGUMENT with the TransformError text. */
typedef struct {                 /* ModelConfig (types.hpp:89-96) */
  int64_t n_params;
  int32_t n_layers, d_model, d_ffn, n_heads, d_head, pad;
} ts_model_config;
typedef struct {                 /* ParallelismConfig (types.hpp:98-103) */
  int32_t tp, pp, dp, num_microbatches;
} ts_par_config;
typedef struct {                 /* WhatIfConfig (transform.hpp:28-41) */
  ts_model_config source_model, target_model;
  ts_par_config source_par, target_par;
  double alpha_us, bytes_per_us; /* AnalyticalCostModel(alpha_us, bytes_per_us) */
  int64_t activation_bytes;      /* activation_bytes_per_microbatch */
  const char* tag_policy_json;   /* TagPolicy::from_json text, NULL = defaults */
} ts_whatif;
typedef struct ts_pipeline ts_pipeline;
/* A host graph from task arrays and their metadata, for callers that hold a
 * built ExecutionGraph (the C++ drop-in): desc's tasks, edges, rules and
 * window; per task its name, correlation id (-1 = none) and Task.meta as
 * meta_off[n + 1] into meta_keys / meta_values (types.hpp:73-87). */
int ts_host_graph_from_tasks(const ts_graph_desc* desc, const char* const* names,
                             const int64_t* corr, const int32_t* meta_off,
                             const char* const* meta_keys, const char* const* meta_values,
                             ts_host_graph** out);
int ts_rebuild_pipeline(const ts_host_graph* source, const ts_whatif* whatif, ts_pipeline** out);
/* the rebuilt spec; valid while the ts_pipeline lives */
const ts_pipeline_spec* ts_pipeline_spec_get(const ts_pipeline* p);
void ts_pipeline_free(ts_pipeline* p);

/* build_graph (build.cpp:338-510) over one rank's events, SoA.  cat is the
 * EventCategory (types.hpp:20-27); corr = -1, stream = -1 and
 * arg_event / arg_stream = INT64_MIN mean absent.  names is a '\n'-separated
 * string table indexed by name[i].  Appends the rank to *inout (merge_ranks,
 * build.cpp:512-542) when *inout is non-null, else creates it.  Returns
 * TS_E_GRAPH on a dependency cycle (message = the reference's witness). */
int ts_build_rank_graph(int32_t rank, int64_t n_events, const int32_t* name, const uint8_t* cat,
                        const int64_t* ts, const int64_t* dur, const int32_t* tid,
                        const int64_t* corr, const int32_t* stream, const int64_t* arg_event,
                        const int64_t* arg_stream, const char* names, int64_t gap_threshold_us,
                        ts_host_graph** inout);

/* Native parallel ingest of recorded traces: the
 * reference's input path with default options (cli.cpp:93-137, window
 * "full") — parse_trace of each Chrome-trace JSON file (trace_parse.cpp:79-154,
 * default category table), one rank per rank_<N> file or per process id,
 * build_graph per rank (build.cpp:338-510) and merge_ranks (:512-542) — with
 * files parsed and ranks built on n_threads host threads (<= 0: all cores).
 * The graph carries the retime metadata (rt_*) of its Task.meta.  Errors:
 * TS_E_INVALID_ARGUMENT with the ParseError text, TS_E_GRAPH for cycles. */
int ts_ingest_traces(const char* const* paths, int32_t n_paths, int32_t n_threads,
                     int64_t gap_threshold_us, ts_host_graph** out);

/* The full input options of the reference's build_from_inputs (cli.cpp:52-58,
 * 118-137): a rank manifest (load_multirank_manifest, trace_parse.cpp:296-328),
 * the iteration window ("full", "auto" = detect_iteration_window +
 * filter_window, trace_parse.cpp:330-419, or "START:END"), a custom category
 * table (CategoryTable::from_json, trace_parse.cpp:186-211) and a build policy
 * (BuildPolicy::from_json, build.cpp:41-66), the last two as JSON file paths
 * like the CLI's --categories / --policy.  NULL fields take the defaults. */
typedef struct {
  const char* const* paths;      /* --trace inputs */
  int32_t n_paths;
  int32_t n_threads;             /* <= 0: all cores */
  const char* manifest;          /* --manifest JSON {rank: path} or NULL */
  const char* window;            /* NULL = "full" */
  const char* categories_path;   /* or NULL */
  const char* policy_path;       /* or NULL */
  int32_t keep_meta;             /* keep Task.meta + correlation ids (ts_rebuild_pipeline) */
  int32_t pad;
} ts_ingest_options;
int ts_ingest_traces_ex(const ts_ingest_options* options, ts_host_graph** out);

/* Device-time accounting: when enabled, CUDA events are recorded on the
 * caller's stream around every kernel the engine launches for this graph;
 * ts_profile_read waits for them, returns the accumulated milliseconds per
 * kernel class and resets the counters. */
typedef struct {
  double walk_ms;          /* K1 replay walk (durations fused) */
  int64_t walk_launches;
  double reduce_ms;        /* K5 per-rank breakdown / stream busy */
  int64_t reduce_launches;
  double other_ms;         /* span init / finalize */
  int64_t other_launches;
} ts_profile_stats;
int ts_profile_enable(ts_graph* g, int enable);
int ts_profile_read(ts_graph* g, ts_profile_stats* out);

/* Launch counters (kernels this library enqueued since creation). */
int64_t ts_kernel_launches(void);
/* K1 walk launches per variant since load: out[0] one scenario per thread with
 * uint32 slot values, out[1] one with int64, out[2] two per thread uint32,
 * out[3] two per thread int64, out[4] cluster walks of estimate-mode
 * components (K1x; LUMOS_CLUSTER=0 takes the cooperative walk instead).
 * The environment variable LUMOS_WALK_KS=1|2
 * pins the scenarios per thread (parity tests run both; a batch starting at an
 * odd global id always takes one, so Philox pairs never straddle threads). */
int ts_walk_counts(int64_t* out /* [5] */);
const char* ts_last_error(void);
int ts_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LUMOS_B200_H */
