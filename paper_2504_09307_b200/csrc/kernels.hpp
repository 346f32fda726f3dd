// kernels.hpp — launch parameters of the replay kernels (replay.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "program.hpp"

namespace lumos {

enum : int32_t { kModeScale = 1, kModeJitter = 2, kModeExplicit = 4, kModeRetime = 8 };

// Per-scenario what-if retime parameters of a retime walk (ts_retime)
struct RtScen {
  double alpha;   // cost model alpha (us)
  double bpu;     // bytes per us
  int32_t tdp;    // target data-parallel size
  int32_t flags;  // kRtHid: change_hidden applies; kRtDp: scale_dp applies
};
enum : int32_t { kRtHid = 1, kRtDp = 2 };

// Retime walk (kModeRetime): the walk evaluates each F_RT task's retimed
// duration itself.  Everything that depends only on the target model widths
// (retimed GEMM / optimizer base durations, retimed collective byte counts)
// is precomputed per distinct width triple ("variant") by K4v into
// vval[variant][rec]; the cost-model terms (alpha, bytes/us, target dp) are
// per scenario.
struct RtRec {
  int64_t base;   // recorded duration
  int32_t group;  // meta group_size
  int32_t kind;   // TS_RT_*
};
struct RetimeWalk {
  const int32_t* rec_of;  // [op records] dense index of an F_RT record
  const RtRec* rec;       // [n_rec]
  const int64_t* vval;    // [n_var][n_rec]
  int64_t n_rec;
  const int32_t* var;     // [count] variant of each scenario (tile-relative)
  const RtScen* scen;     // [count]
  int32_t source_dp;
  int32_t pad;
};


struct ScenarioParams {
  int64_t first;        // global id of column 0
  int32_t count;
  int32_t mode;         // kMode* bits
  uint32_t key_jit;     // Philox key of the jitter stream
  uint32_t key_cls;     // Philox key of the class-scale stream
  double two_j;         // 2 * jitter
  double neg_j;         // -jitter
  double two_j_ulp;     // two_j * 2^-32 (exact: a power-of-two scaling)
  uint32_t rk_jit[10];  // Philox round keys of key_jit (key + r * 0x9E3779B9)
  int32_t scale_lo;
  uint32_t scale_span;  // hi - lo + 1
  int64_t scale_den;
  int32_t den_shift;    // log2(den) when den is a power of two, else -1
  int32_t n_classes;    // columns of scale_num
  int32_t n_classes_eff;
  int32_t pad;
  const int32_t* scale_num;   // device [count][n_classes] or null
  const int64_t* durations;   // device [n_tasks][durations_ld] or null
  int64_t durations_ld;
};

struct WalkParams {
  const Op* ops;
  const ProgramDesc* progs;
  const ComponentDesc* comps;
  const int32_t* comp_order;  // optional launch order of components
  int32_t n_comps;
  int32_t force_ks;  // 0: scenarios per thread chosen by occupancy; 1 / 2: forced (tests)
  int64_t window_start;
  ScenarioParams sp;
  int64_t* out_start;  // [n_tasks][ld] or null
  int64_t* out_fin;
  int64_t ld;
  int64_t* span_lo;    // [count] atomics
  int64_t* span_hi;
  int32_t* status;
  int32_t vec_store;   // 16-byte output stores allowed (ld, count even; aligned)
  int32_t rel32;       // slot values are uint32 offsets from W (bound proven on the host)
  RetimeWalk rt;       // sp.mode & kModeRetime
  // split accounting (program.hpp FusedDesc), or null: a fused component
  // writes its compute-stream busy sum |A| to acct_a[col][row]
  const FusedDesc* fused;  // [component]
  int64_t* acct_a;         // [count][n_ranks]
  int32_t n_ranks;
  int32_t n_tasks;         // rows of out_start / out_fin (bounds checks)
  // cluster walk (K1x, estimate-mode components): one CTA per rank program,
  // the component's rank CTAs one thread-block cluster; cross-rank values
  // through a global (L2-resident) mailbox table [cluster][mailbox][thread]
  // of uint32 pairs, all-ones = not yet posted
  const int32_t* cl_prog_off;  // [components + 1] into cl_progs
  const int32_t* cl_progs;     // rank programs per component
  const int32_t* cl_rows;      // split accounting row per rank program, or null
  uint64_t* cl_mail;
  int32_t cl_size;             // CTAs per cluster (ranks of the widest component)
  int32_t cl_n_mail;           // mailboxes per cluster
  int32_t cl_check;            // 1: check every finish for a uint32 wrap (window not proven)
};
// debug builds: the source line of the first failed bounds check since the
// last call (0 = none), cleared by the read; always 0 in release builds
int debug_bounds_status();
int debug_bounds_status_des();



struct ReduceParams {
  const int32_t* rank_list;  // ranks (indices into rank_stream_off) of this launch
  const int32_t* rank_stream_off;
  const int32_t* stream_node_off;
  const int32_t* stream_nodes;
  const uint8_t* is_comm;
  const int64_t* start;
  const int64_t* fin;
  int64_t ld;
  const int64_t* span_lo;
  const int64_t* span_hi;
  int64_t window_start;
  int64_t window_end;
  int32_t count;
  int32_t n_ranks;
  int32_t n_streams;
  int32_t n_tasks_total;  // rows of start / fin (bounds checks)
  int64_t* breakdown;    // [count][n_ranks][5]
  int64_t* stream_busy;  // [count][n_streams]
  int64_t* util;         // [count][n_ranks][util_max_bins] (zeroed), or null
  int64_t util_bw;
  int32_t util_max_bins;
  int32_t pad2;
  // split accounting (fast-path buckets only): A is read through the rank's
  // candidate list (cand_off / cand_nodes by rank row) and |A| comes from the
  // walk (acct_a[col][row]) instead of the full compute-stream list
  const int32_t* cand_off;
  const int32_t* cand_nodes;
  const int64_t* acct_a;  // [count][n_ranks]
  const int32_t* status;  // lite: scenarios with a non-zero status were reduced by the fix-up
};

// what-if retime of every (task, scenario) duration (ts_retime), then the
// scenario's class scale and jitter; writes dur[task * ld + s]
struct RetimeParams {
  ScenarioParams sp;        // mode without kModeExplicit
  const int64_t* base;
  const uint8_t* cls;
  const uint8_t* kind;      // TS_RT_*
  const int64_t* bytes;
  const int32_t* group;
  const int64_t* mnk;       // [n][3]
  const double* alpha;      // [count] (device)
  const double* bpu;        // [count]
  const int32_t* target_dp; // [count] or null
  const int64_t* target_model;  // [count][3] or null
  int64_t src_model[3];
  int32_t source_dp;
  int32_t n_tasks;
  int64_t* dur;
  int64_t ld;
};
struct DesParams {
  int32_t n, nl;
  const int64_t* ostart;
  const int32_t* lane_of;
  const int32_t* lane_off;
  const int32_t* lane_tasks;
  const int32_t* succ_off;
  const int32_t* succ;
  const int32_t* indeg0;
  const int32_t* rule_of;
  const int32_t* rule_kind;
  const int32_t* rule_bound;
  const int32_t* rule_wl_off;
  const int32_t* rule_wl;
  const int64_t* base;
  const uint8_t* cls;
  const uint8_t* is_comm;
  const int32_t* lane_rank;
  const int32_t* lane_stream;
  int32_t n_ranks, n_streams;
  int64_t W, window_end;
  ScenarioParams sp;
  int64_t* out_start;
  int64_t* out_fin;
  int64_t ld;
  int64_t* span_lo;
  int64_t* span_hi;
  int32_t* status;
  int64_t* breakdown;
  int64_t* stream_busy;
  int64_t* util;  // as ReduceParams
  int64_t util_bw;
  int32_t util_max_bins;
  int32_t fixup;    // only scenarios whose status is non-zero (certificate failed)
  int32_t n_slots;  // concurrent scenarios (scratch slots)
  int32_t smem_lanes;  // 1: one scenario per CTA, lane state + completion heap in shared memory
  char* scratch;
  int64_t scratch_bytes;  // per slot
  RetimeParams rt;  // has_rt: retime each duration first (fix-up of a retime walk)
  int32_t has_rt;
  int32_t pad3;
};
size_t des_scratch_bytes(int32_t n, int32_t nl);
size_t des_smem_bytes(int32_t nl);  // shared memory per CTA of the smem_lanes mode
cudaError_t launch_des(const DesParams& p, cudaStream_t stream);

int walk_threads();
int walk_width(int n_slots, bool rel32);  // walk CTA width for a slot count (0: too many)
int max_streams_per_rank();
cudaError_t launch_replay_walk(const WalkParams& p, int n_slots, cudaStream_t stream);
// walk launches per variant since load: [0] one scenario per thread (uint32
// slots), [1] one (int64), [2] two per thread (uint32), [3] two (int64),
// [4] cluster walks (K1x)
void walk_variant_counts(int64_t out[5]);

// Cooperative walk (components of several ranks coupled by gates): one CTA =
// (component, 32 scenarios), one warp per rank program, cross-rank values
// through shared-memory mailboxes (program.hpp OP_POST / OP_WAIT).  Uses the
// WalkParams of the launch (outputs, scenarios, window) with comp_order /
// n_comps naming the cooperative components.
struct CoopParams {
  const int32_t* prog_off;  // [n_all_comps + 1] into progs
  const int32_t* progs;     // rank programs per component
  int32_t max_ranks;        // warps per CTA
  int32_t n_mail;           // mailboxes per CTA (max over components)
  int32_t n_slots;          // slots per rank program (max)
  int32_t rel32;            // uint32 offsets from W (additions checked, wraps -> fix-up)
  int32_t fixup;            // re-run only chunks holding a scenario with status bit 0
  int32_t pad;
  const int32_t* rows;      // [progs] split accounting: the rank row a warp's |A| goes to
                            // (acct_a of the WalkParams), -1 none; null: off
};
cudaError_t launch_coop_walk(const WalkParams& p, const CoopParams& c, cudaStream_t stream);
// K1x: returns cudaErrorNotSupported when the device cannot co-schedule a
// cluster of p.cl_size CTAs (the caller then takes the cooperative walk)
cudaError_t launch_cluster_walk(const WalkParams& p, int n_slots, cudaStream_t stream);
bool cluster_walk_supported(int cl_size, int n_slots);
cudaError_t launch_span_init(int64_t* lo, int64_t* hi, int32_t* status, int32_t count,
                             cudaStream_t stream);
// compare_replay deltas of one tile: partial[chunk][count][3] then per column
// {sum |d|, max |d|, worst task, signed delta} (see ts_result)
// compare_replay's worst list (metrics.cpp:213-217): the worst_n tasks with
// the largest |delta|, ties by smaller task id; kept per (chunk, scenario)
// and merged per scenario
constexpr int kMaxWorst = 64;
struct DeltaParams {
  const int64_t* start;  // [n_tasks][ld]
  int64_t ld;
  const int64_t* ostart;  // [n_tasks]
  int32_t n_tasks;
  int32_t count;
  int32_t n_chunks;
  int32_t worst_n;   // 1..kMaxWorst
  int64_t* partial_sum;  // [n_chunks][count]
  int64_t* partial;      // [n_chunks][count][worst_n][2] {|d| (-1 empty), task}
  int64_t* abs_sum;  // [count] or null
  int64_t* worst;    // [count][worst_n][3] {|d|, task (-1: none), d} or null
};
cudaError_t launch_deltas(const DeltaParams& p, cudaStream_t stream);
// n_bins[i] = ceil(window span / w) for the utilization bins
cudaError_t launch_util_nbins(const int64_t* lo, const int64_t* hi, int64_t W, int64_t window_end,
                              int64_t w, int32_t* n_bins, int32_t count, cudaStream_t stream);
cudaError_t launch_span_finalize(const int64_t* lo, const int64_t* hi, int64_t W, int64_t* span,
                                 int64_t* makespan, int32_t count, cudaStream_t stream);
cudaError_t launch_retime_durations(const RetimeParams& p, cudaStream_t stream);
// K4v: vval[v][j] for the variant width triples targets[v] (v = 0: the source
// widths, i.e. no change_hidden) of every F_RT record j
struct VariantParams {
  const RtRec* rec;
  const int32_t* rec_task;  // [n_rec]
  const int64_t* bytes;     // per task (ts_graph_desc.rt_bytes)
  const int64_t* mnk;       // per task [n][3]
  const int64_t* targets;   // [n_var][3]
  int64_t src_model[3];
  int64_t n_rec;
  int32_t n_var;
  int32_t pad;
  int64_t* vval;
};
cudaError_t launch_retime_variants(const VariantParams& p, cudaStream_t stream);
cudaError_t launch_durations(const ScenarioParams& sp, const int64_t* base, const uint8_t* cls,
                             int32_t n_tasks, int64_t* dur, int64_t ld, cudaStream_t stream);
// buckets 0..6: event merge by stream count (reduce_bucket); 7..10: the
// one-compute-stream fast path with 0..3 comm streams (rank_list entries then
// carry the compute stream's index in bits 24..31)
constexpr int kReduceGenericBuckets = 7;
constexpr int kReduceFastMaxComm = 3;
static_assert(kReduceFastMaxComm == kFusedMaxComm, "fused ranks take the fast sweep");
constexpr int kReduceBuckets = kReduceGenericBuckets + kReduceFastMaxComm + 1;
// buckets kReduceLiteBucket + NC (NC = 0..3 comm streams): split accounting of
// fused ranks (ReduceParams cand_* / acct_a); rank_list entries carry the
// compute stream's index in bits 24..31, 0xFF when the rank has none
constexpr int kReduceLiteBucket = kReduceBuckets;
constexpr int kReduceAllBuckets = kReduceLiteBucket + kReduceFastMaxComm + 1;
int reduce_bucket(int streams_in_rank);
cudaError_t launch_rank_reduce(const ReduceParams& p, int bucket, int n_ranks_in_bucket,
                               cudaStream_t stream);

}  // namespace lumos
