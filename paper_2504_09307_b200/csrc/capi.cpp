// capi.cpp — the extern "C" boundary (include/lumos_b200.h).
//
// Owns the device copy of a compiled graph and sequences the kernels of one
// batched replay: span init -> K1 walk (durations fused) -> span finalize ->
// K5 per-rank reductions.  All device work is enqueued on the caller's
// stream; host-side output pointers are staged and copied back at the end.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "compile.hpp"
#include "kernels.hpp"
#include "lumos_b200.h"

using namespace lumos;

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace

namespace lumos {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace lumos

namespace {

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(TS_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(_e) + " (" + \
                                 #expr + ")");                                            \
  } while (0)

template <class T>
cudaError_t upload(T** dptr, const std::vector<T>& v) {
  *dptr = nullptr;
  if (v.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(dptr), v.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

uint32_t seed_key(uint64_t seed, uint32_t salt) {
  return static_cast<uint32_t>(seed ^ (seed >> 32)) ^ salt;
}

// device buffer that grows on demand
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

struct ts_graph {
  CompiledGraph cg;
  int device = -1;
  bool has_device = false;
  Op* d_ops = nullptr;
  ProgramDesc* d_progs = nullptr;
  ComponentDesc* d_comps = nullptr;
  int32_t* d_comp_order = nullptr;   // single-program components, longest first
  int32_t n_single = 0;
  int32_t* d_coop_comps = nullptr;   // cooperative (multi-rank) components
  int32_t n_coop = 0;
  int32_t* d_coop_prog_off = nullptr;
  int32_t* d_coop_progs = nullptr;
  int64_t* d_base = nullptr;
  uint8_t* d_rt_kind = nullptr;  // retime metadata (empty when absent)
  int64_t* d_rt_bytes = nullptr;
  int32_t* d_rt_group = nullptr;
  int64_t* d_rt_mnk = nullptr;
  DevBuf retime_dur, retime_par;  // retimed durations tile, per-scenario parameters
  // retime walk (kModeRetime) tables: per op record its dense F_RT index,
  // per F_RT record {base, group, kind} and its task; per call the variant table
  int32_t* d_rt_rec_of = nullptr;
  RtRec* d_rt_rec = nullptr;
  int32_t* d_rt_rec_task = nullptr;
  int64_t n_rt_rec = 0;
  DevBuf rt_vval, rt_var;
  uint8_t* d_cls = nullptr;
  uint8_t* d_is_comm = nullptr;
  int32_t* d_rank_stream_off = nullptr;
  int32_t* d_stream_node_off = nullptr;
  int32_t* d_stream_nodes = nullptr;
  int32_t* d_rank_lists = nullptr;                // ranks grouped by stream-count bucket
  // event-driven path tables
  int64_t* d_ostart = nullptr;
  int32_t *d_lane_of = nullptr, *d_lane_off = nullptr, *d_lane_tasks = nullptr;
  int32_t *d_succ_off = nullptr, *d_succ = nullptr, *d_indeg0 = nullptr, *d_rule_of = nullptr;
  int32_t *d_rule_kind = nullptr, *d_rule_bound = nullptr, *d_rule_wl_off = nullptr;
  int32_t *d_rule_wl = nullptr, *d_lane_rank = nullptr, *d_lane_stream = nullptr;
  DevBuf des_scratch;
  int32_t bucket_off[kReduceBuckets + 1] = {0};
  // in-walk accounting: per component descriptor, the fused rank rows, and the
  // K5 rank lists restricted to the other ranks
  FusedDesc* d_fused = nullptr;
  int32_t n_fused_rows = 0;
  int32_t* d_coop_rows = nullptr;  // per cooperative rank program: its fused row or -1
  int32_t* d_cand_off = nullptr;
  int32_t* d_cand_nodes = nullptr;
  int32_t* d_rank_lists_nf = nullptr;  // non-fused ranks by bucket, then fused ranks (lite)
  int32_t bucket_off_nf[kReduceAllBuckets + 1] = {0};
  DevBuf acct_a;  // [tile][n_ranks] |A| sums of the walk
  DevBuf cl_mail;  // cluster walk mailboxes
  int cluster_state = -1;  // -1 unknown, 0 unsupported, 1 supported
  bool cluster_ok(int size, int n_slots) {
    if (cluster_state < 0) cluster_state = cluster_walk_supported(size, n_slots) ? 1 : 0;
    return cluster_state == 1;
  }
  DevBuf span_lo, span_hi, status, scratch_ts;
  DevBuf stage[12];  // host-pointer staging: start, fin, span, breakdown, busy, num, dur,
                     // util, util bins, delta sum, delta worst, internal bin counts
  // ts_result.host_async: output staging in two sets, copied to the host on
  // copy_stream while the next call's kernels run; copy_done[k] guards set k
  DevBuf astage[2][12];
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t copy_done[2] = {nullptr, nullptr};
  cudaEvent_t kernels_done = nullptr;
  bool copy_pending[2] = {false, false};
  int async_set = 0;
  DevBuf delta_scratch;
  // device-time accounting
  bool profile = false;
  struct Mark {
    cudaEvent_t a, b;
    int kind;  // 0 walk, 1 reduce, 2 other
  };
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

namespace {
// records events around one launch when profiling is on
struct Timed {
  ts_graph* g;
  cudaStream_t s;
  int kind;
  cudaEvent_t a = nullptr;
  Timed(ts_graph* g_, cudaStream_t s_, int k) : g(g_), s(s_), kind(k) {
    if (g->profile) {
      a = g->get_event();
      cudaEventRecord(a, s);
    }
  }
  ~Timed() {
    if (a) {
      cudaEvent_t b = g->get_event();
      cudaEventRecord(b, s);
      g->marks.push_back({a, b, kind});
    }
  }
};
}  // namespace

extern "C" {

int ts_abi_version(void) { return TS_ABI_VERSION; }
const char* ts_last_error(void) { return g_err.c_str(); }
int64_t ts_kernel_launches(void) { return g_launches.load(); }
int ts_walk_counts(int64_t* out) {
  if (!out) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  walk_variant_counts(out);
  return TS_OK;
}

int ts_graph_create(const ts_graph_desc* desc, int device, ts_graph** out) {
  if (!desc || !out) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  auto* g = new ts_graph;
  std::string err;
  int rc = compile_graph(*desc, g->cg, err);
  if (rc != TS_OK) {
    delete g;
    return fail(rc, err);
  }
  if (device == -2) {  // compile only (host-side inspection; no replay possible)
    *out = g;
    return TS_OK;
  }
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
    cudaGetLastError();
    delete g;
    return fail(TS_E_CUDA, "no CUDA device: the replay engine runs only on the GPU");
  }
  if (device >= 0) {
    if (cudaSetDevice(device) != cudaSuccess) {
      delete g;
      return fail(TS_E_CUDA, "cudaSetDevice failed");
    }
    g->device = device;
  } else {
    cudaGetDevice(&g->device);
  }
  // Graphs the walk cannot hold fall back instead of failing (the reference
  // replays them): a component coupling more ranks than one CTA holds is
  // compiled without the cooperative split; a component with more live values
  // than shared memory holds, or a rank with more streams than the per-rank
  // merge supports, takes the exact event-driven path (plain replay graphs;
  // gated estimate graphs have no event-driven restatement and are rejected).
  auto coop_fits = [](const CompiledGraph& cg) {
    const size_t smem = static_cast<size_t>((cg.max_mailboxes * 4 + 15) / 16) * 16 +
                        static_cast<size_t>(cg.max_mailboxes) * 32 * 4 +
                        static_cast<size_t>(cg.max_coop_ranks) * cg.max_slots * 32 * 4;
    return cg.max_coop_ranks <= 32 && smem <= 227 * 1024;
  };
  auto has_coop = [](const CompiledGraph& cg) {
    for (size_t ci = 0; ci + 1 < cg.coop_prog_off.size(); ++ci)
      if (cg.coop_prog_off[ci + 1] - cg.coop_prog_off[ci] > 1) return true;
    return false;
  };
  if (!g->cg.des_only && has_coop(g->cg) && !coop_fits(g->cg)) {
    g->cg = CompiledGraph{};
    rc = compile_graph(*desc, g->cg, err, /*allow_coop=*/false);
    if (rc != TS_OK) {
      delete g;
      return fail(rc, err);
    }
  }
  CompiledGraph& c = g->cg;
  std::string fallback;
  if (!c.des_only && walk_width(c.max_slots, false) == 0)
    fallback = "a component needs " + std::to_string(c.max_slots) +
               " live values per scenario: more than shared memory holds";
  for (size_t r = 0; r + 1 < c.rank_stream_off.size() && fallback.empty() && !c.des_only; ++r)
    if (c.rank_stream_off[r + 1] - c.rank_stream_off[r] > max_streams_per_rank())
      fallback = "rank has more than " + std::to_string(max_streams_per_rank()) + " streams";
  if (!fallback.empty()) {
    if (desc->n_gates > 0) {
      delete g;
      return fail(TS_E_UNSUPPORTED, fallback);
    }
    c.des_only = true;
    c.des_reason = fallback;
  }
  // launch order: longest component first (smaller tail)
  std::vector<int32_t> order(c.comps.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int32_t>(i);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return c.programs[c.comps[a].program].n_ops > c.programs[c.comps[b].program].n_ops;
  });
  // components walked by one program vs cooperatively by one warp per rank
  std::vector<int32_t> single, coop;
  for (int32_t ci : order) {
    const bool multi = !c.coop_prog_off.empty() &&
                       c.coop_prog_off[ci + 1] - c.coop_prog_off[ci] > 1;
    (multi ? coop : single).push_back(ci);
  }
  g->n_single = static_cast<int32_t>(single.size());
  g->n_coop = static_cast<int32_t>(coop.size());
#ifdef LUMOS_DEBUG_BOUNDS
  // self-test of the bounds checks: LUMOS_DEBUG_CORRUPT=1 points one operand
  // of the first plain node past the slot table; the next replay must fail
  if (const char* bad = std::getenv("LUMOS_DEBUG_CORRUPT"))
    if (bad[0] == '1')
      for (Op& o : c.ops)
        if (o.kind == OP_NODE && !(o.flags & (F_TRACK | F_TRACK1))) {
          o.pred[0] = slot_off(kMaxSlots);
          break;
        }
#endif
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = upload(&g->d_ops, c.ops);
  if (e == cudaSuccess) e = upload(&g->d_progs, c.programs);
  if (e == cudaSuccess) e = upload(&g->d_comps, c.comps);
  if (e == cudaSuccess) e = upload(&g->d_comp_order, single);
  if (e == cudaSuccess) e = upload(&g->d_coop_comps, coop);
  if (e == cudaSuccess) e = upload(&g->d_coop_prog_off, c.coop_prog_off);
  if (e == cudaSuccess) e = upload(&g->d_coop_progs, c.coop_progs);
  if (e == cudaSuccess) e = upload(&g->d_base, c.base);
  if (e == cudaSuccess) e = upload(&g->d_rt_kind, c.rt_kind);
  if (e == cudaSuccess) e = upload(&g->d_rt_bytes, c.rt_bytes);
  if (e == cudaSuccess) e = upload(&g->d_rt_group, c.rt_group);
  if (e == cudaSuccess) e = upload(&g->d_rt_mnk, c.rt_mnk);
  if (e == cudaSuccess && !c.rt_rec_task.empty()) {
    std::vector<RtRec> rec(c.rt_rec_task.size());
    for (size_t j = 0; j < rec.size(); ++j) {
      const int32_t t = c.rt_rec_task[j];
      rec[j] = RtRec{c.base[t], c.rt_group[t], static_cast<int32_t>(c.rt_kind[t])};
    }
    g->n_rt_rec = static_cast<int64_t>(rec.size());
    e = upload(&g->d_rt_rec, rec);
    if (e == cudaSuccess) e = upload(&g->d_rt_rec_of, c.rt_rec_of);
    if (e == cudaSuccess) e = upload(&g->d_rt_rec_task, c.rt_rec_task);
  }
  if (e == cudaSuccess) e = upload(&g->d_cls, c.scale_class);
  if (e == cudaSuccess) e = upload(&g->d_is_comm, c.is_comm);
  if (e == cudaSuccess) e = upload(&g->d_rank_stream_off, c.rank_stream_off);
  if (e == cudaSuccess) e = upload(&g->d_stream_node_off, c.stream_node_off);
  if (e == cudaSuccess) e = upload(&g->d_stream_nodes, c.stream_nodes);
  {
    // per rank: generic merge bucket, or the fast path when the rank has one
    // compute-only stream and <= 3 comm-only streams
    const size_t n_ranks = c.rank_stream_off.size() - 1;
    std::vector<int> bucket(n_ranks);
    std::vector<int32_t> entry(n_ranks);
    for (size_t r = 0; r < n_ranks; ++r) {
      const int s0 = c.rank_stream_off[r], ns = c.rank_stream_off[r + 1] - s0;
      int n_compute = 0, n_comm = 0, ci = -1;
      for (int j = 0; j < ns; ++j) {
        bool any_comm = false, any_compute = false;
        for (int32_t q = c.stream_node_off[s0 + j]; q < c.stream_node_off[s0 + j + 1]; ++q)
          (c.stream_nodes[q] < 0 ? any_comm : any_compute) = true;
        if (any_compute && !any_comm) {
          ++n_compute;
          ci = j;
        } else if (any_comm && !any_compute) {
          ++n_comm;
        }
      }
      if (n_compute == 1 && n_compute + n_comm == ns && n_comm <= kReduceFastMaxComm) {
        bucket[r] = kReduceGenericBuckets + n_comm;
        entry[r] = static_cast<int32_t>(r) | (ci << 24);
      } else {
        bucket[r] = reduce_bucket(ns);
        entry[r] = static_cast<int32_t>(r);
      }
    }
    std::vector<int32_t> lists;
    for (int b = 0; b < kReduceBuckets; ++b) {
      g->bucket_off[b] = static_cast<int32_t>(lists.size());
      for (size_t r = 0; r < n_ranks; ++r)
        if (bucket[r] == b) lists.push_back(entry[r]);
    }
    g->bucket_off[kReduceBuckets] = static_cast<int32_t>(lists.size());
    if (e == cudaSuccess) e = upload(&g->d_rank_lists, lists);
    // split accounting: fused ranks go to the lite buckets (by comm stream
    // count), the others keep their bucket
    std::vector<int> fused_bucket(n_ranks, -1);
    std::vector<int32_t> fused_entry(n_ranks, 0);
    if (!c.des_only)
      for (const FusedDesc& fd : c.fused_rows) {
        if (fd.row < 0 || fused_bucket[fd.row] >= 0) continue;
        const int s0 = c.rank_stream_off[fd.row], ns = c.rank_stream_off[fd.row + 1] - s0;
        const int ci = fd.stream_a >= 0 ? fd.stream_a - s0 : 0xFF;
        fused_bucket[fd.row] = kReduceLiteBucket + ns - (fd.stream_a >= 0 ? 1 : 0);
        fused_entry[fd.row] = static_cast<int32_t>(static_cast<uint32_t>(fd.row) |
                                                   (static_cast<uint32_t>(ci) << 24));
        g->n_fused_rows++;
      }
    std::vector<int32_t> lists_nf;
    for (int b = 0; b < kReduceAllBuckets; ++b) {
      g->bucket_off_nf[b] = static_cast<int32_t>(lists_nf.size());
      for (size_t r = 0; r < n_ranks; ++r) {
        if (fused_bucket[r] < 0 && bucket[r] == b) lists_nf.push_back(entry[r]);
        if (fused_bucket[r] == b) lists_nf.push_back(fused_entry[r]);
      }
    }
    g->bucket_off_nf[kReduceAllBuckets] = static_cast<int32_t>(lists_nf.size());
    if (e == cudaSuccess) e = upload(&g->d_rank_lists_nf, lists_nf);
    if (g->n_fused_rows > 0) {
      if (e == cudaSuccess) e = upload(&g->d_fused, c.fused);
      if (e == cudaSuccess) e = upload(&g->d_coop_rows, c.coop_rows);
      if (e == cudaSuccess) e = upload(&g->d_cand_off, c.cand_off);
      if (e == cudaSuccess) e = upload(&g->d_cand_nodes, c.cand_nodes);
    }
  }
  {
    const DesTables& T = c.des;
    if (e == cudaSuccess) e = upload(&g->d_ostart, T.ostart);
    if (e == cudaSuccess) e = upload(&g->d_lane_of, T.lane_of);
    if (e == cudaSuccess) e = upload(&g->d_lane_off, T.lane_off);
    if (e == cudaSuccess) e = upload(&g->d_lane_tasks, T.lane_tasks);
    if (e == cudaSuccess) e = upload(&g->d_succ_off, T.succ_off);
    if (e == cudaSuccess) e = upload(&g->d_succ, T.succ);
    if (e == cudaSuccess) e = upload(&g->d_indeg0, T.indeg0);
    if (e == cudaSuccess) e = upload(&g->d_rule_of, T.rule_of);
    if (e == cudaSuccess) e = upload(&g->d_rule_kind, T.rule_kind);
    if (e == cudaSuccess) e = upload(&g->d_rule_bound, T.rule_bound);
    if (e == cudaSuccess) e = upload(&g->d_rule_wl_off, T.rule_wl_off);
    if (e == cudaSuccess) e = upload(&g->d_rule_wl, T.rule_wl);
    if (e == cudaSuccess) e = upload(&g->d_lane_rank, T.lane_rank);
    if (e == cudaSuccess) e = upload(&g->d_lane_stream, T.lane_stream);
  }
  g->has_device = true;
  if (e != cudaSuccess) {
    ts_graph_destroy(g);
    return fail(TS_E_CUDA, std::string("upload failed: ") + cudaGetErrorString(e));
  }
  *out = g;
  return TS_OK;
}

int ts_graph_wait(ts_graph* g) {
  if (!g) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  if (g->copy_stream && cudaStreamSynchronize(g->copy_stream) != cudaSuccess)
    return fail(TS_E_CUDA, cudaGetErrorString(cudaGetLastError()));
  return TS_OK;
}

void ts_graph_destroy(ts_graph* g) {
  if (!g) return;
  if (g->has_device) {
    int prev = -1;
    cudaGetDevice(&prev);
    if (g->device >= 0) cudaSetDevice(g->device);
    if (g->copy_stream) {
      cudaStreamSynchronize(g->copy_stream);
      cudaStreamDestroy(g->copy_stream);
      for (cudaEvent_t e : {g->copy_done[0], g->copy_done[1], g->kernels_done})
        if (e) cudaEventDestroy(e);
    }
    for (void* p : {static_cast<void*>(g->d_ops), static_cast<void*>(g->d_progs),
                    static_cast<void*>(g->d_comps), static_cast<void*>(g->d_comp_order),
                    static_cast<void*>(g->d_coop_comps), static_cast<void*>(g->d_coop_prog_off),
                    static_cast<void*>(g->d_coop_progs),
                    static_cast<void*>(g->d_base), static_cast<void*>(g->d_cls),
                    static_cast<void*>(g->d_rt_kind), static_cast<void*>(g->d_rt_bytes),
                    static_cast<void*>(g->d_rt_group), static_cast<void*>(g->d_rt_mnk),
                    static_cast<void*>(g->d_rt_rec_of), static_cast<void*>(g->d_rt_rec),
                    static_cast<void*>(g->d_rt_rec_task),
                    static_cast<void*>(g->d_is_comm), static_cast<void*>(g->d_rank_stream_off),
                    static_cast<void*>(g->d_stream_node_off),
                    static_cast<void*>(g->d_stream_nodes), static_cast<void*>(g->d_rank_lists),
                    static_cast<void*>(g->d_fused), static_cast<void*>(g->d_cand_off),
                    static_cast<void*>(g->d_coop_rows),
                    static_cast<void*>(g->d_cand_nodes), static_cast<void*>(g->d_rank_lists_nf),
                    static_cast<void*>(g->d_ostart), static_cast<void*>(g->d_lane_of),
                    static_cast<void*>(g->d_lane_off), static_cast<void*>(g->d_lane_tasks),
                    static_cast<void*>(g->d_succ_off), static_cast<void*>(g->d_succ),
                    static_cast<void*>(g->d_indeg0), static_cast<void*>(g->d_rule_of),
                    static_cast<void*>(g->d_rule_kind), static_cast<void*>(g->d_rule_bound),
                    static_cast<void*>(g->d_rule_wl_off), static_cast<void*>(g->d_rule_wl),
                    static_cast<void*>(g->d_lane_rank), static_cast<void*>(g->d_lane_stream)})
      if (p) cudaFree(p);
    g->des_scratch.release();
    g->acct_a.release();
    g->cl_mail.release();
    g->retime_dur.release();
    g->retime_par.release();
    g->rt_vval.release();
    g->rt_var.release();
    for (DevBuf* b : {&g->span_lo, &g->span_hi, &g->status, &g->scratch_ts, &g->delta_scratch})
      b->release();
    for (DevBuf& b : g->stage) b.release();
    for (auto& m : g->marks) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
    for (cudaEvent_t e : g->event_pool) cudaEventDestroy(e);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete g;
}

int ts_graph_get_info(const ts_graph* g, ts_graph_info* out) {
  if (!g || !out) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  const CompiledGraph& c = g->cg;
  out->n_tasks = c.n_tasks;
  out->n_components = static_cast<int32_t>(c.comps.size());
  out->n_programs = static_cast<int32_t>(c.programs.size());
  out->n_ranks = static_cast<int32_t>(c.ranks.size());
  out->n_streams = static_cast<int32_t>(c.stream_rank.size());
  out->max_slots = c.max_slots;
  out->program_bytes = static_cast<int64_t>(c.ops.size() * sizeof(Op));
  out->n_ops = static_cast<int64_t>(c.ops.size());
  out->n_syncs = c.n_syncs;
  out->n_gpu_tasks = c.n_gpu_tasks;
  out->window_start = c.window_start;
  out->window_end = c.window_end;
  out->n_fused_ranks = g->has_device ? g->n_fused_rows
                                     : (c.des_only ? 0 : static_cast<int32_t>(c.fused_rows.size()));
  out->des_only = c.des_only ? 1 : 0;
  out->n_candidates = c.cand_nodes.size();
  return TS_OK;
}

int ts_graph_ranks(const ts_graph* g, int32_t* ranks) {
  if (!g || !ranks) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  std::copy(g->cg.ranks.begin(), g->cg.ranks.end(), ranks);
  return TS_OK;
}

int ts_graph_streams(const ts_graph* g, int32_t* rank, int32_t* lane) {
  if (!g || !rank || !lane) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  std::copy(g->cg.stream_rank.begin(), g->cg.stream_rank.end(), rank);
  std::copy(g->cg.stream_lane.begin(), g->cg.stream_lane.end(), lane);
  return TS_OK;
}

// report_deadlock (simulate.cpp:258-303) on the final state of one replayed
// scenario, read back from its DES scratch (des.cu carve layout): the chain of
// blockers from the lowest unstarted task, the cycle if it closes one.
static std::string deadlock_witness(const DesTables& T, int32_t n, const std::vector<char>& scr,
                                    int64_t unstarted) {
  const int32_t nl = T.n_lanes;
  const int64_t* sim_start = reinterpret_cast<const int64_t*>(scr.data());
  const int32_t* p32 = reinterpret_cast<const int32_t*>(
      sim_start + 3 * static_cast<int64_t>(n) + nl + 2 * static_cast<int64_t>(n));
  const int32_t* indeg = p32;
  const int32_t* heap = p32 + n;
  const int32_t* hsize = p32 + 3 * static_cast<int64_t>(n);
  auto started = [&](int32_t t) { return sim_start[t] != INT64_MIN; };
  // ready sets in (original_start, id) order
  std::vector<std::vector<int32_t>> ready(nl);
  for (int32_t l = 0; l < nl; ++l) {
    ready[l].assign(heap + T.lane_off[l], heap + T.lane_off[l] + hsize[l]);
    std::sort(ready[l].begin(), ready[l].end(), [&](int32_t a, int32_t b) {
      return std::make_pair(T.ostart[a], a) < std::make_pair(T.ostart[b], b);
    });
  }
  std::vector<int32_t> min_pred(n, -1);  // lowest unstarted fixed-edge predecessor
  for (int32_t u = 0; u < n; ++u) {
    if (started(u)) continue;
    for (int32_t k = T.succ_off[u]; k < T.succ_off[u + 1]; ++k) {
      const int32_t v = T.succ[k];
      if (!started(v) && (min_pred[v] < 0 || u < min_pred[v])) min_pred[v] = u;
    }
  }
  auto blocker_of = [&](int32_t t) -> int32_t {
    if (indeg[t] > 0) return min_pred[t];
    const auto& own = ready[T.lane_of[t]];
    if (!own.empty() && std::make_pair(T.ostart[own[0]], own[0]) < std::make_pair(T.ostart[t], t))
      return own[0];
    const int32_t r = T.rule_of[t];
    if (r >= 0) {
      if (T.rule_kind[r] == TS_RULE_EVENT_SYNC) return T.rule_bound[r];
      for (int32_t w = T.rule_wl_off[r]; w < T.rule_wl_off[r + 1]; ++w)
        for (int32_t id : ready[T.rule_wl[w]])
          if (id != t) return id;
    }
    return -1;
  };
  int32_t cur = -1;
  for (int32_t i = 0; i < n && cur < 0; ++i)
    if (!started(i)) cur = i;
  std::vector<int32_t> path;
  std::vector<char> on_path(n, 0);
  while (cur >= 0 && !on_path[cur]) {
    on_path[cur] = 1;
    path.push_back(cur);
    cur = blocker_of(cur);
  }
  std::vector<int32_t> cycle = path;
  if (cur >= 0) cycle.assign(std::find(path.begin(), path.end(), cur), path.end());
  std::string msg = "deadlock with " + std::to_string(unstarted) + " tasks blocked: ";
  for (size_t i = 0; i < cycle.size(); ++i) msg += (i ? " " : "") + std::to_string(cycle[i]);
  return msg;
}

static int scenario_params(const ts_graph* g, const ts_scenarios* sc, ScenarioParams& sp) {
  std::memset(&sp, 0, sizeof(sp));
  if (sc->count < 0) return fail(TS_E_INVALID_ARGUMENT, "scenario count must be >= 0");
  sp.first = sc->first;
  sp.count = sc->count;
  sp.key_jit = seed_key(sc->seed, 0u);
  for (int r = 0; r < 10; ++r) sp.rk_jit[r] = sp.key_jit + static_cast<uint32_t>(r) * 0x9E3779B9u;
  sp.key_cls = seed_key(sc->seed, 0x5CA1E000u);
  sp.den_shift = -1;
  sp.n_classes = 0;
  if (sc->durations) {
    if (sc->durations_ld < sc->count)
      return fail(TS_E_INVALID_ARGUMENT, "durations_ld must be >= count");
    sp.mode = kModeExplicit;
    sp.durations = sc->durations;
    sp.durations_ld = sc->durations_ld;
    return TS_OK;
  }
  if (sc->jitter != 0.0) {
    if (!(sc->jitter > 0.0 && sc->jitter < 1.0))
      return fail(TS_E_INVALID_ARGUMENT, "jitter must be in [0, 1)");
    sp.mode |= kModeJitter;
    sp.two_j = 2.0 * sc->jitter;
    sp.neg_j = -sc->jitter;
    sp.two_j_ulp = std::ldexp(sp.two_j, -32);
  }
  if (sc->scale_den > 0) {
    sp.mode |= kModeScale;
    sp.scale_den = sc->scale_den;
    if ((sc->scale_den & (sc->scale_den - 1)) == 0) {
      int s = 0;
      while ((1LL << s) < sc->scale_den) ++s;
      sp.den_shift = s;
    }
    if (sc->scale_num) {
      if (sc->n_classes < 1 || sc->n_classes > kMaxClasses)
        return fail(TS_E_INVALID_ARGUMENT, "n_classes must be in [1, 4]");
      sp.scale_num = sc->scale_num;
      sp.n_classes = sc->n_classes;
      sp.n_classes_eff = sc->n_classes;
    } else {
      if (sc->scale_lo < 0 || sc->scale_hi < sc->scale_lo)
        return fail(TS_E_INVALID_ARGUMENT, "need 0 <= scale_lo <= scale_hi");
      sp.scale_lo = sc->scale_lo;
      sp.scale_span = static_cast<uint32_t>(sc->scale_hi - sc->scale_lo + 1);
      sp.n_classes_eff = kMaxClasses;
    }
  }
  (void)g;
  return TS_OK;
}

// Validates a ts_retime against the graph the way change_hidden / scale_dp
// reject their inputs (transform.cpp:219-258, 279-349, cost.cpp:55-62) and
// stages its per-scenario arrays on the device: [alpha][bpu][target_dp][model].
static int retime_stage(ts_graph* g, const ts_retime* rt, int32_t count, cudaStream_t stream,
                        RetimeParams& p) {
  const CompiledGraph& c = g->cg;
  if (c.rt_kind.empty())
    return fail(TS_E_INVALID_ARGUMENT, "graph carries no retime metadata (ts_graph_desc.rt_kind)");
  if (!rt->alpha_us || !rt->bytes_per_us)
    return fail(TS_E_INVALID_ARGUMENT, "retime needs alpha_us and bytes_per_us per scenario");
  // the first task change_hidden would stop at (transform.cpp:279-349): the
  // first optimizer / allreduce task (n_params check), the first allreduce
  // without a group size
  int32_t first_np = -1, first_nogroup = -1;
  for (int32_t t = 0; t < c.n_tasks && (first_np < 0 || first_nogroup < 0); ++t) {
    const uint8_t k = c.rt_kind[t];
    // change_hidden touches an allreduce only when it carries a byte count
    // (transform.cpp:313); scale_dp's missing-bytes error is checked below
    const bool ar_bytes = k == TS_RT_ALLREDUCE && c.rt_bytes[t] >= 0;
    if (first_np < 0 && (k == TS_RT_OPT || ar_bytes)) first_np = t;
    if (first_nogroup < 0 && ar_bytes && c.rt_group[t] <= 0) first_nogroup = t;
  }
  bool any_dp_change = false;
  for (int32_t s = 0; s < count; ++s) {
    if (!(rt->bytes_per_us[s] > 0))
      return fail(TS_E_INVALID_ARGUMENT,
                  "cost model cannot retime collective: bytes_per_us must be positive");
    if (rt->target_dp) {
      const int32_t sd = rt->source_dp, td = rt->target_dp[s];
      if (sd < 1 || td < 1) return fail(TS_E_INVALID_ARGUMENT, "data-parallel sizes must be >= 1");
      if (sd != td) {
        if (sd == 1)
          return fail(TS_E_INVALID_ARGUMENT,
                      "source trace has no gradient collectives to rescale; use apply_whatif to "
                      "introduce them");
        if (td == 1)
          return fail(TS_E_INVALID_ARGUMENT,
                      "cannot drop gradient collectives by retiming; use apply_whatif to rebuild "
                      "without them");
        any_dp_change = true;
      }
    }
    if (rt->target_model) {
      const int64_t* tm = rt->target_model + 3 * static_cast<size_t>(s);
      if (tm[0] != rt->source_model[0] || tm[1] != rt->source_model[1]) {
        if (rt->source_model[0] <= 0 || tm[0] <= 0)
          return fail(TS_E_INVALID_ARGUMENT, "hidden-size rescale needs both model widths");
        if (first_np >= 0 && (rt->source_model[2] <= 0 || tm[2] <= 0))
          return fail(TS_E_INVALID_ARGUMENT,
                      c.rt_kind[first_np] == TS_RT_OPT
                          ? "hidden-size rescale of optimizer work needs n_params on both models"
                          : "hidden-size rescale of collectives needs n_params on both models");
        if (first_nogroup >= 0)
          return fail(TS_E_INVALID_ARGUMENT, "collective task " + std::to_string(first_nogroup) +
                                                 " carries no group size");
      }
    }
  }
  if (any_dp_change) {
    int changed = 0;
    for (int32_t t = 0; t < c.n_tasks; ++t)
      if (c.rt_kind[t] == TS_RT_ALLREDUCE && c.rt_group[t] == rt->source_dp) {
        if (c.rt_bytes[t] < 0)
          return fail(TS_E_INVALID_ARGUMENT,
                      "collective task " + std::to_string(t) + " carries no byte count");
        ++changed;
      }
    if (changed == 0)
      return fail(TS_E_INVALID_ARGUMENT, "no gradient collectives sized for data-parallel group " +
                                             std::to_string(rt->source_dp) + " found");
  }
  const size_t n = static_cast<size_t>(count);
  const size_t bytes = n * 8 * 2 + n * 4 + (rt->target_model ? n * 24 : 0) + 64;
  if (g->retime_par.reserve(bytes) != cudaSuccess)
    return fail(TS_E_NOMEM, "could not stage retime parameters");
  char* base = g->retime_par.as<char>();
  double* d_alpha = reinterpret_cast<double*>(base);
  double* d_bpu = d_alpha + n;
  int64_t* d_tm = reinterpret_cast<int64_t*>(d_bpu + n);
  int32_t* d_tdp = reinterpret_cast<int32_t*>(d_tm + (rt->target_model ? 3 * n : 0));
  auto cp = [&](void* dst, const void* src, size_t b) {
    return cudaMemcpyAsync(dst, src, b, cudaMemcpyHostToDevice, stream);
  };
  cudaError_t e = cp(d_alpha, rt->alpha_us, n * 8);
  if (e == cudaSuccess) e = cp(d_bpu, rt->bytes_per_us, n * 8);
  if (e == cudaSuccess && rt->target_model) e = cp(d_tm, rt->target_model, n * 24);
  if (e == cudaSuccess && rt->target_dp) e = cp(d_tdp, rt->target_dp, n * 4);
  if (e != cudaSuccess) return fail(TS_E_CUDA, cudaGetErrorString(e));
  p.base = g->d_base;
  p.cls = g->d_cls;
  p.kind = g->d_rt_kind;
  p.bytes = g->d_rt_bytes;
  p.group = g->d_rt_group;
  p.mnk = g->d_rt_mnk;
  p.alpha = d_alpha;
  p.bpu = d_bpu;
  p.target_dp = rt->target_dp ? d_tdp : nullptr;
  p.target_model = rt->target_model ? d_tm : nullptr;
  for (int k = 0; k < 3; ++k) p.src_model[k] = rt->source_model[k];
  p.source_dp = rt->source_dp;
  p.n_tasks = c.n_tasks;
  return TS_OK;
}

// Retime walk staging: the distinct target width triples of the scenarios
// change_hidden applies to become variants (variant 0 = the source widths),
// K4v fills vval[variant][F_RT record], and each scenario gets its variant and
// cost-model terms.  Returns false (nothing staged) when the variant table
// would not fit its memory budget; the caller then materialises durations.
static bool retime_walk_stage(ts_graph* g, const ts_retime* rt, int32_t count,
                              cudaStream_t stream, RetimeWalk& w, cudaError_t& err) {
  err = cudaSuccess;
  const int64_t* sm = rt->source_model;
  std::vector<int64_t> targets = {sm[0], sm[1], sm[2]};
  std::map<std::array<int64_t, 3>, int32_t> index;
  std::vector<int32_t> var(static_cast<size_t>(count));
  std::vector<RtScen> scen(static_cast<size_t>(count));
  for (int32_t s = 0; s < count; ++s) {
    RtScen& q = scen[s];
    q.alpha = rt->alpha_us[s];
    q.bpu = rt->bytes_per_us[s];
    q.tdp = rt->target_dp ? rt->target_dp[s] : rt->source_dp;
    q.flags = (rt->target_dp && q.tdp != rt->source_dp) ? kRtDp : 0;
    int32_t v = 0;
    if (rt->target_model) {
      const int64_t* tm = rt->target_model + 3 * static_cast<size_t>(s);
      if (tm[0] != sm[0] || tm[1] != sm[1]) {  // change_hidden applies (transform.cpp:282)
        q.flags |= kRtHid;
        const std::array<int64_t, 3> key = {tm[0], tm[1], tm[2]};
        auto it = index.find(key);
        if (it == index.end()) {
          it = index.emplace(key, static_cast<int32_t>(targets.size() / 3)).first;
          targets.insert(targets.end(), key.begin(), key.end());
        }
        v = it->second;
      }
    }
    var[s] = v;
  }
  const int64_t n_var = static_cast<int64_t>(targets.size() / 3);
  const size_t vbytes = static_cast<size_t>(n_var) * static_cast<size_t>(g->n_rt_rec) * 8;
  if (vbytes > (size_t(2) << 30)) return false;
  const size_t n = static_cast<size_t>(count);
  const size_t pbytes = n * sizeof(RtScen) + targets.size() * 8 + n * 4 + 64;
  if ((err = g->rt_vval.reserve(vbytes)) != cudaSuccess) return false;
  if ((err = g->rt_var.reserve(pbytes)) != cudaSuccess) return false;
  char* base = g->rt_var.as<char>();
  RtScen* d_scen = reinterpret_cast<RtScen*>(base);
  int64_t* d_targets = reinterpret_cast<int64_t*>(d_scen + n);
  int32_t* d_var = reinterpret_cast<int32_t*>(d_targets + targets.size());
  // pageable sources: each copy returns once its source has been staged
  err = cudaMemcpyAsync(d_scen, scen.data(), n * sizeof(RtScen), cudaMemcpyHostToDevice, stream);
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(d_targets, targets.data(), targets.size() * 8, cudaMemcpyHostToDevice,
                          stream);
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(d_var, var.data(), n * 4, cudaMemcpyHostToDevice, stream);
  if (err != cudaSuccess) return false;
  VariantParams vp{};
  vp.rec = g->d_rt_rec;
  vp.rec_task = g->d_rt_rec_task;
  vp.bytes = g->d_rt_bytes;
  vp.mnk = g->d_rt_mnk;
  vp.targets = d_targets;
  for (int k = 0; k < 3; ++k) vp.src_model[k] = sm[k];
  vp.n_rec = g->n_rt_rec;
  vp.n_var = static_cast<int32_t>(n_var);
  vp.vval = g->rt_vval.as<int64_t>();
  {
    Timed tm(g, stream, 2);
    if ((err = launch_retime_variants(vp, stream)) != cudaSuccess) return false;
  }
  g_launches++;
  w.rec_of = g->d_rt_rec_of;
  w.rec = g->d_rt_rec;
  w.vval = vp.vval;
  w.n_rec = g->n_rt_rec;
  w.var = d_var;
  w.scen = d_scen;
  w.source_dp = rt->source_dp;
  return true;
}

int ts_replay_batch(ts_graph* g, const ts_scenarios* sc, const ts_result* out, void* stream_) {
  if (!g || !sc || !out) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  if (!g->has_device) return fail(TS_E_CUDA, "graph was compiled without a device");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  ScenarioParams sp;
  if (int rc = scenario_params(g, sc, sp)) return rc;
  const CompiledGraph& c = g->cg;
  const int32_t count = sc->count;
  if (count == 0) return TS_OK;
  if ((out->start || out->fin) && out->ld < count)
    return fail(TS_E_INVALID_ARGUMENT, "ld must be >= count");
  RetimeParams rtp{};
  const bool retime = sc->retime != nullptr;
  if (retime) {
    if (sp.mode & kModeExplicit)
      return fail(TS_E_INVALID_ARGUMENT, "retime cannot be combined with explicit durations");
    if (int rc = retime_stage(g, sc->retime, count, stream, rtp)) return rc;
  }
  if ((out->util_covered || out->util_n_bins) && out->util_bin_width <= 0)
    return fail(TS_E_INVALID_ARGUMENT, "bin_width must be positive");  // metrics.cpp:107
  if (out->util_covered && out->util_max_bins <= 0)
    return fail(TS_E_INVALID_ARGUMENT, "util_max_bins must be positive");
  int prev_dev = -1;
  cudaGetDevice(&prev_dev);
  if (prev_dev != g->device) CUDA_TRY(cudaSetDevice(g->device));

  // inputs given as host memory are staged on the device (persistent buffers)
  auto stage_in = [&](int slot, const void* host, size_t bytes, const void** dev) -> cudaError_t {
    cudaError_t e = g->stage[slot].reserve(bytes);
    if (e != cudaSuccess) return e;
    *dev = g->stage[slot].p;
    return cudaMemcpyAsync(g->stage[slot].p, host, bytes, cudaMemcpyHostToDevice, stream);
  };
  auto cleanup = [] {};
  if (sp.scale_num && !is_device_ptr(sp.scale_num)) {
    const void* d = nullptr;
    cudaError_t e = stage_in(5, sp.scale_num, static_cast<size_t>(count) * sp.n_classes * 4, &d);
    if (e != cudaSuccess) return fail(TS_E_CUDA, cudaGetErrorString(e));
    sp.scale_num = static_cast<const int32_t*>(d);
  }
  if (sp.durations && !is_device_ptr(sp.durations)) {
    const void* d = nullptr;
    cudaError_t e = stage_in(6, sp.durations,
                             static_cast<size_t>(c.n_tasks) * sp.durations_ld * 8, &d);
    if (e != cudaSuccess) return fail(TS_E_CUDA, cudaGetErrorString(e));
    sp.durations = static_cast<const int64_t*>(d);
  }

  // outputs: device pointers are written in place, host pointers staged
  const bool want_ts = out->start || out->fin;
  const bool want_red = out->rank_breakdown || out->stream_busy || out->util_covered;
  const bool want_delta = out->delta_abs_sum || out->delta_worst;
  const int32_t n_ranks = static_cast<int32_t>(c.ranks.size());
  const int32_t n_streams = static_cast<int32_t>(c.stream_rank.size());
  struct OutBuf {
    void* user;
    size_t bytes;
    void* dev;
  };
  std::vector<OutBuf> copies;
  const bool host_async = out->host_async != 0;
  const int aset = g->async_set;
  if (host_async && g->copy_pending[aset]) {
    // the set's previous host copy must finish before this call rewrites it
    CUDA_TRY(cudaStreamWaitEvent(stream, g->copy_done[aset], 0));
    g->copy_pending[aset] = false;
  }
  auto out_ptr = [&](int slot, void* user, size_t bytes) -> void* {
    if (!user || bytes == 0) return nullptr;
    if (is_device_ptr(user)) return user;
    DevBuf& b = host_async ? g->astage[aset][slot] : g->stage[slot];
    if (b.reserve(bytes) != cudaSuccess) return nullptr;
    copies.push_back({user, bytes, b.p});
    return b.p;
  };
  const size_t ts_bytes = static_cast<size_t>(c.n_tasks) * static_cast<size_t>(out->ld) * 8;
  int64_t* d_start = static_cast<int64_t*>(out_ptr(0, out->start, ts_bytes));
  int64_t* d_fin = static_cast<int64_t*>(out_ptr(1, out->fin, ts_bytes));
  int64_t* d_span = static_cast<int64_t*>(out_ptr(2, out->span, static_cast<size_t>(count) * 24));
  int64_t* d_bd = static_cast<int64_t*>(
      out_ptr(3, out->rank_breakdown, static_cast<size_t>(count) * n_ranks * 40));
  int64_t* d_busy = static_cast<int64_t*>(
      out_ptr(4, out->stream_busy, static_cast<size_t>(count) * n_streams * 8));
  const int32_t ubins = out->util_covered ? out->util_max_bins : 0;
  int64_t* d_util = static_cast<int64_t*>(
      out_ptr(7, out->util_covered, static_cast<size_t>(count) * n_ranks * ubins * 8));
  int32_t* d_nbins = static_cast<int32_t*>(out_ptr(8, out->util_n_bins, static_cast<size_t>(count) * 4));
  int64_t* d_dsum = static_cast<int64_t*>(out_ptr(9, out->delta_abs_sum, static_cast<size_t>(count) * 8));
  const int32_t worst_n = out->delta_worst_n <= 0 ? 1 : out->delta_worst_n;
  if (worst_n > kMaxWorst)
    return fail(TS_E_INVALID_ARGUMENT,
                "delta_worst_n must be <= " + std::to_string(kMaxWorst) + " on the device");
  int64_t* d_dworst = static_cast<int64_t*>(
      out_ptr(10, out->delta_worst, static_cast<size_t>(count) * worst_n * 24));
  // utilization needs the per-scenario bin counts to check util_max_bins
  int32_t* d_nbins_chk = d_nbins;
  if (out->util_covered && !d_nbins_chk) {
    if (g->stage[11].reserve(static_cast<size_t>(count) * 4) != cudaSuccess)
      return fail(TS_E_NOMEM, "could not stage output buffers");
    d_nbins_chk = g->stage[11].as<int32_t>();
  }
  if ((out->start && ts_bytes && !d_start) || (out->fin && ts_bytes && !d_fin) ||
      (out->span && !d_span) || (out->rank_breakdown && n_ranks && !d_bd) ||
      (out->stream_busy && n_streams && !d_busy) || (out->util_covered && n_ranks && !d_util) ||
      (out->util_n_bins && !d_nbins) || (out->delta_abs_sum && !d_dsum) ||
      (out->delta_worst && !d_dworst)) {
    cleanup();
    return fail(TS_E_NOMEM, "could not stage output buffers");
  }

  CUDA_TRY(g->span_lo.reserve(static_cast<size_t>(count) * 8));
  CUDA_TRY(g->span_hi.reserve(static_cast<size_t>(count) * 8));
  CUDA_TRY(g->status.reserve(static_cast<size_t>(count) * 4));
  int64_t* lo = g->span_lo.as<int64_t>();
  int64_t* hi = g->span_hi.as<int64_t>();
  int32_t* status = g->status.as<int32_t>();

  // in-walk accounting (program.hpp FusedDesc): fused ranks get their
  // breakdown and stream busy from the walk itself; K5 reduces the others.
  // Utilization bins need the sweep, so they keep K5 for every rank.
  const char* acct_env = std::getenv("LUMOS_FUSED_REDUCE");
  const bool acct = want_red && !d_util && g->n_fused_rows > 0 && !c.des_only &&
                    !(acct_env && acct_env[0] == '0');
  const bool k5_needed = want_red && !c.des_only;

  // timestamps needed for the reductions but not requested: sub-batch through
  // an internal scratch tile
  int32_t sub = count;
  bool tile_local = false;  // timestamp pointers address the current tile only
  int64_t* s_start = d_start;
  int64_t* s_fin = d_fin;
  int64_t s_ld = out->ld;
  // compare_replay deltas need the starts, the reductions both timestamps
  const bool need_start = k5_needed || want_delta, need_fin = k5_needed;
  if ((need_start && !d_start) || (need_fin && !d_fin)) {
    if (!want_ts) {
      // none requested: sub-batch through an internal scratch tile of up to
      // half the free device memory (wide tiles keep the walk grid full)
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) cudaGetLastError();
      const size_t budget = std::max<size_t>(size_t(4) << 30, (free_b + g->scratch_ts.bytes) / 2);
      const size_t per_col = static_cast<size_t>(c.n_tasks) * 16 + 1;
      size_t cols = std::max<size_t>(128, budget / per_col / 256 * 256);
      sub = static_cast<int32_t>(std::min<size_t>(cols, static_cast<size_t>(count)));
      CUDA_TRY(g->scratch_ts.reserve(static_cast<size_t>(sub) * per_col));
      s_start = g->scratch_ts.as<int64_t>();
      s_fin = s_start + static_cast<size_t>(c.n_tasks) * sub;
      s_ld = sub;
      tile_local = true;
    } else {
      // one of them requested: the other lives in scratch at the caller's ld
      CUDA_TRY(g->scratch_ts.reserve(ts_bytes + 1));
      if (!d_start) s_start = g->scratch_ts.as<int64_t>();
      if (need_fin && !d_fin) s_fin = g->scratch_ts.as<int64_t>();
    }
  }

  // uint32 offsets from W in the walk when no time can reach W + 2^32 - 1:
  // per component, sum of the largest possible durations (class scale
  // mul_div <= d*num/den + 1, jitter <= d*(1+j) + 1, transform.cpp:38-43,
  // synth.cpp:150-155) bounds every start and finish
  // retimed durations: evaluated inside the walk (kModeRetime) when every
  // component takes the single-program walk, else materialised per tile (K4r)
  // and read back by an explicit-duration walk
  RetimeWalk rtw{};
  bool rt_fused = false;
  if (retime) {
    const char* env = std::getenv("LUMOS_RT_FUSED");
    if (!(env && env[0] == '0') && g->n_coop == 0 && !c.des_only && g->n_rt_rec > 0) {
      cudaError_t e = cudaSuccess;
      rt_fused = retime_walk_stage(g, sc->retime, count, stream, rtw, e);
      if (e != cudaSuccess) {
        cleanup();
        return fail(TS_E_CUDA, cudaGetErrorString(e));
      }
    }
  }
  if (retime && !rt_fused) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) cudaGetLastError();
    const size_t per_col = static_cast<size_t>(c.n_tasks) * 8 + 1;
    const size_t cap = std::max<size_t>(128, (free_b + g->retime_dur.bytes) / 4 / per_col / 128 * 128);
    sub = static_cast<int32_t>(std::min<size_t>(static_cast<size_t>(sub), cap));
    CUDA_TRY(g->retime_dur.reserve(static_cast<size_t>(sub) * per_col));
  }
  bool rel32 = false;
  if (!retime && !(sp.mode & kModeExplicit) && !sp.scale_num) {
    double f = 1.0;
    if (sp.mode & kModeScale)
      f *= static_cast<double>(sp.scale_lo + static_cast<int64_t>(sp.scale_span) - 1) /
           static_cast<double>(sp.scale_den);
    if (sp.mode & kModeJitter) f *= 1.0 + 0.5 * sp.two_j;
    // a value is a max-plus path from W: at most f x the component's nominal
    // longest path plus 1 us of rounding per task (or the looser sum bound)
    const double bound =
        std::min(static_cast<double>(c.max_comp_dur_sum) * f,
                 static_cast<double>(c.max_comp_path) * f) +
        3.0 * static_cast<double>(c.max_comp_tasks) + 16.0;
    // offsets from O = W rounded down to a multiple of 2^32 (replay.cu):
    // W - O + every time must stay below 2^32 - 1
    const double w_lo = static_cast<double>(static_cast<uint32_t>(c.window_start));
    rel32 = f >= 0.0 && w_lo + bound < 4.2e9 && walk_width(c.max_slots, true) > 0;
  }
  // cooperative walks size their uint32 window by the nominal longest path
  // and check every addition (a wrap sends the scenario to the fix-up)
  bool coop_rel32 = false, use_cluster = false, cl_proven = false;
  if (!retime && !(sp.mode & kModeExplicit) && !sp.scale_num && g->n_coop > 0) {
    double f = 1.0;
    if (sp.mode & kModeScale)
      f *= static_cast<double>(sp.scale_lo + static_cast<int64_t>(sp.scale_span) - 1) /
           static_cast<double>(sp.scale_den);
    if (sp.mode & kModeJitter) f *= 1.0 + 0.5 * sp.two_j;
    coop_rel32 = static_cast<double>(c.max_coop_path) * f * 1.25 + 1e6 < 4.0e9;
    const char* force = std::getenv("LUMOS_COOP_FORCE_U32");  // tests: exercise the wrap fix-up
    if (force && force[0] == '1') coop_rel32 = true;
    // the cluster walk's offsets start at W rounded down to 2^32 (as K1's)
    const double w_lo = static_cast<double>(static_cast<uint32_t>(c.window_start));
    const char* cl = std::getenv("LUMOS_CLUSTER");
    use_cluster = coop_rel32 && !(cl && cl[0] == '0') &&
                  (w_lo + static_cast<double>(c.max_coop_path) * f * 1.25 + 1e6 < 4.0e9 ||
                   (force && force[0] == '1')) &&
                  g->cluster_ok(c.max_coop_ranks, c.max_slots);
    // every value is a max-plus path from W: a scenario path is at most f x
    // its nominal length plus one microsecond of rounding per task, so this
    // bound proves the window and the per-finish wrap check can go
    cl_proven = !(force && force[0] == '1') &&
                w_lo + static_cast<double>(c.max_coop_path) * f +
                        static_cast<double>(c.n_tasks) + 16.0 < 4.2e9;
  }
  // LUMOS_WALK_KS=1|2 pins the walk's scenarios per thread (tests run every
  // parity case on both variants; an odd first id always takes one)
  int32_t force_ks = 0;
  if (const char* ks = std::getenv("LUMOS_WALK_KS")) force_ks = (ks[0] == '1') ? 1 : (ks[0] == '2') ? 2 : 0;
  {
    Timed tm(g, stream, 2);
    CUDA_TRY(launch_span_init(lo, hi, status, count, stream));
  }
  g_launches++;
  for (int32_t b0 = 0; b0 < count; b0 += sub) {
    const int32_t bn = std::min(sub, count - b0);
    WalkParams wp{};
    wp.ops = g->d_ops;
    wp.progs = g->d_progs;
    wp.comps = g->d_comps;
    wp.comp_order = g->d_comp_order;
    wp.n_comps = g->n_single;
    wp.force_ks = force_ks;
    wp.n_tasks = c.n_tasks;
    wp.window_start = c.window_start;
    wp.sp = sp;
    wp.sp.first = sp.first + b0;
    wp.sp.count = bn;
    if (sp.scale_num) wp.sp.scale_num = sp.scale_num + static_cast<size_t>(b0) * sp.n_classes;
    if (sp.durations) wp.sp.durations = sp.durations + b0;
    if (rt_fused) {
      wp.sp.mode |= kModeRetime;
      wp.rt = rtw;
      wp.rt.var = rtw.var + b0;
      wp.rt.scen = rtw.scen + b0;
    } else if (retime) {
      // what-if retime + class scale + jitter of this tile, then an explicit walk
      RetimeParams rp_ = rtp;
      rp_.sp = wp.sp;
      rp_.alpha = rtp.alpha + b0;
      rp_.bpu = rtp.bpu + b0;
      if (rtp.target_dp) rp_.target_dp = rtp.target_dp + b0;
      if (rtp.target_model) rp_.target_model = rtp.target_model + 3 * static_cast<size_t>(b0);
      rp_.dur = g->retime_dur.as<int64_t>();
      rp_.ld = bn;
      {
        Timed tm(g, stream, 2);
        CUDA_TRY(launch_retime_durations(rp_, stream));
      }
      g_launches++;
      wp.sp.mode = kModeExplicit;
      wp.sp.durations = rp_.dur;
      wp.sp.durations_ld = bn;
      wp.sp.scale_num = nullptr;
    }
    if (d_util) {
      const size_t row = static_cast<size_t>(n_ranks) * ubins;
      CUDA_TRY(cudaMemsetAsync(d_util + static_cast<size_t>(b0) * row, 0,
                               static_cast<size_t>(bn) * row * 8, stream));
    }
    wp.out_start = s_start ? s_start + (tile_local ? 0 : b0) : nullptr;
    wp.out_fin = s_fin ? s_fin + (tile_local ? 0 : b0) : nullptr;
    wp.ld = s_ld;
    wp.span_lo = lo + b0;
    wp.span_hi = hi + b0;
    wp.status = status + b0;
    wp.rel32 = rel32 ? 1 : 0;
    if (acct) {
      CUDA_TRY(g->acct_a.reserve(static_cast<size_t>(sub) * n_ranks * 8));
      wp.fused = g->d_fused;
      wp.acct_a = g->acct_a.as<int64_t>();
      wp.n_ranks = n_ranks;
    }
    {
      auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
      wp.vec_store = (wp.ld % 2 == 0) && (bn % 2 == 0) &&
                     (!wp.out_start || al(wp.out_start)) && (!wp.out_fin || al(wp.out_fin));
    }
    if (!c.des_only && wp.n_comps > 0) {
      Timed tm(g, stream, 0);
      CUDA_TRY(launch_replay_walk(wp, c.max_slots, stream));
      g_launches++;
    }
    if (!c.des_only && g->n_coop > 0) {
      WalkParams cw = wp;
      cw.comp_order = g->d_coop_comps;
      cw.n_comps = g->n_coop;
      CoopParams cp{};
      cp.prog_off = g->d_coop_prog_off;
      cp.progs = g->d_coop_progs;
      cp.max_ranks = c.max_coop_ranks;
      cp.n_mail = c.max_mailboxes;
      cp.n_slots = c.max_slots;
      cp.rel32 = coop_rel32 ? 1 : 0;
      cp.rows = acct ? g->d_coop_rows : nullptr;
      // K1x cluster walk: one 128-thread CTA per rank program (two scenarios
      // per thread, the K1 fast path), the component's ranks one cluster,
      // cross-rank values through an L2-resident mailbox table; uint32 windows
      // only (wraps re-run below in int64 by the cooperative kernel)
      bool clustered = false;
      // a thread's two scenarios share one Philox call: an even first id
      if (use_cluster && (wp.sp.first & 1) == 0) {
        const int64_t units = static_cast<int64_t>(g->n_coop) * ((bn + 255) / 256);
        const size_t mail = static_cast<size_t>(units) * c.max_mailboxes * 128 * 8;
        CUDA_TRY(g->cl_mail.reserve(mail + 8));
        CUDA_TRY(cudaMemsetAsync(g->cl_mail.p, 0xFF, mail, stream));
        cw.cl_prog_off = g->d_coop_prog_off;
        cw.cl_progs = g->d_coop_progs;
        cw.cl_rows = acct ? g->d_coop_rows : nullptr;
        cw.cl_mail = g->cl_mail.as<uint64_t>();
        cw.cl_size = c.max_coop_ranks;
        cw.cl_n_mail = c.max_mailboxes;
        cw.cl_check = cl_proven ? 0 : 1;
        Timed tm(g, stream, 0);
        const cudaError_t ce = launch_cluster_walk(cw, c.max_slots, stream);
        if (ce == cudaSuccess) {
          clustered = true;
        } else if (ce != cudaErrorNotSupported) {
          CUDA_TRY(ce);
        } else {
          cudaGetLastError();
        }
      }
      if (!clustered) {
        Timed tm(g, stream, 0);
        CUDA_TRY(launch_coop_walk(cw, cp, stream));
      }
      g_launches++;
      if (coop_rel32) {  // exact int64 re-run of any chunk whose window wrapped
        cp.rel32 = 0;
        cp.fixup = 1;
        Timed tm(g, stream, 2);
        CUDA_TRY(launch_coop_walk(cw, cp, stream));
        g_launches++;
      }
    }
    if (c.des_only || c.n_syncs > 0) {
      // exact event-driven replay: every scenario of a graph outside the
      // chained class, or (fix-up) the scenarios whose certificate failed
      DesParams dp{};
      const DesTables& T = c.des;
      dp.n = c.n_tasks;
      dp.nl = T.n_lanes;
      dp.ostart = g->d_ostart;
      dp.lane_of = g->d_lane_of;
      dp.lane_off = g->d_lane_off;
      dp.lane_tasks = g->d_lane_tasks;
      dp.succ_off = g->d_succ_off;
      dp.succ = g->d_succ;
      dp.indeg0 = g->d_indeg0;
      dp.rule_of = g->d_rule_of;
      dp.rule_kind = g->d_rule_kind;
      dp.rule_bound = g->d_rule_bound;
      dp.rule_wl_off = g->d_rule_wl_off;
      dp.rule_wl = g->d_rule_wl;
      dp.base = g->d_base;
      dp.cls = g->d_cls;
      dp.is_comm = g->d_is_comm;
      dp.lane_rank = g->d_lane_rank;
      dp.lane_stream = g->d_lane_stream;
      dp.n_ranks = n_ranks;
      dp.n_streams = n_streams;
      dp.W = c.window_start;
      dp.window_end = c.window_end;
      dp.sp = wp.sp;
      dp.out_start = wp.out_start;
      dp.out_fin = wp.out_fin;
      dp.ld = wp.ld;
      dp.span_lo = wp.span_lo;
      dp.span_hi = wp.span_hi;
      dp.status = wp.status;
      dp.fixup = c.des_only ? 0 : 1;
      if (rt_fused) {  // the fix-up retimes its own durations
        dp.has_rt = 1;
        dp.rt = rtp;
        dp.rt.sp = wp.sp;
        dp.rt.alpha = rtp.alpha + b0;
        dp.rt.bpu = rtp.bpu + b0;
        if (rtp.target_dp) dp.rt.target_dp = rtp.target_dp + b0;
        if (rtp.target_model) dp.rt.target_model = rtp.target_model + 3 * static_cast<size_t>(b0);
      }
      if (c.des_only || acct) {  // DES reduces the scenarios it replays
        dp.breakdown = d_bd ? d_bd + static_cast<size_t>(b0) * n_ranks * 5 : nullptr;
        dp.stream_busy = d_busy ? d_busy + static_cast<size_t>(b0) * n_streams : nullptr;
        dp.util = d_util ? d_util + static_cast<size_t>(b0) * n_ranks * ubins : nullptr;
        dp.util_bw = out->util_bin_width;
        dp.util_max_bins = ubins;
      }
      // one thread per concurrently replayed scenario, each with its own
      // scratch: at least 1 GB, up to a quarter of the free device memory
      const size_t per = des_scratch_bytes(c.n_tasks, T.n_lanes);
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) cudaGetLastError();
      const size_t budget = std::max<size_t>(size_t(1) << 30, (free_b + g->des_scratch.bytes) / 4);
      dp.n_slots = static_cast<int32_t>(
          std::max<size_t>(1, std::min<size_t>(static_cast<size_t>(bn), budget / per)));
      // lane state in shared memory when it fits two CTAs per SM (LUMOS_DES_SMEM=0: global)
      const char* des_env = std::getenv("LUMOS_DES_SMEM");
      const bool des_smem = !(des_env && des_env[0] == '0');
      dp.smem_lanes = des_smem && T.n_lanes > 0 && des_smem_bytes(T.n_lanes) <= 96 * 1024;
      CUDA_TRY(g->des_scratch.reserve(per * dp.n_slots));
      dp.scratch = g->des_scratch.as<char>();
      dp.scratch_bytes = static_cast<int64_t>(per);
      Timed tm(g, stream, 2);
      CUDA_TRY(launch_des(dp, stream));
      g_launches++;
    }
    if (k5_needed) {
      ReduceParams rp{};
      rp.rank_stream_off = g->d_rank_stream_off;
      rp.stream_node_off = g->d_stream_node_off;
      rp.stream_nodes = g->d_stream_nodes;
      rp.is_comm = g->d_is_comm;
      rp.start = wp.out_start;
      rp.fin = wp.out_fin;
      rp.ld = s_ld;
      rp.span_lo = lo + b0;
      rp.span_hi = hi + b0;
      rp.window_start = c.window_start;
      rp.window_end = c.window_end;
      rp.count = bn;
      rp.n_ranks = n_ranks;
      rp.n_streams = n_streams;
      rp.n_tasks_total = c.n_tasks;
      rp.breakdown = d_bd ? d_bd + static_cast<size_t>(b0) * n_ranks * 5 : nullptr;
      rp.stream_busy = d_busy ? d_busy + static_cast<size_t>(b0) * n_streams : nullptr;
      rp.util = d_util ? d_util + static_cast<size_t>(b0) * n_ranks * ubins : nullptr;
      rp.util_bw = out->util_bin_width;
      rp.util_max_bins = ubins;
      if (acct) {
        rp.cand_off = g->d_cand_off;
        rp.cand_nodes = g->d_cand_nodes;
        rp.acct_a = g->acct_a.as<int64_t>();
        // scenarios the event-driven fix-up replayed were reduced by it; a
        // cooperative walk's int64 re-run (no syncs: no fix-up) rewrote |A|
        rp.status = c.n_syncs > 0 ? status + b0 : nullptr;
      }
      const int32_t* boff = acct ? g->bucket_off_nf : g->bucket_off;
      int32_t* lists = acct ? g->d_rank_lists_nf : g->d_rank_lists;
      for (int b = 0; b < (acct ? kReduceAllBuckets : kReduceBuckets); ++b) {
        const int nr = boff[b + 1] - boff[b];
        if (nr == 0) continue;
        rp.rank_list = lists + boff[b];
        Timed tm(g, stream, 1);
        CUDA_TRY(launch_rank_reduce(rp, b, nr, stream));
        g_launches++;
      }
    }
    if (want_delta) {
      DeltaParams dl{};
      dl.start = wp.out_start;
      dl.ld = wp.ld;
      dl.ostart = g->d_ostart;
      dl.n_tasks = c.n_tasks;
      dl.count = bn;
      const int col_blocks = (bn + 127) / 128;
      const int64_t want = (4 * 148 * 8 + col_blocks - 1) / col_blocks;
      dl.n_chunks = static_cast<int32_t>(
          std::max<int64_t>(1, std::min<int64_t>(want, (c.n_tasks + 255) / 256)));
      dl.worst_n = worst_n;
      const size_t cells = static_cast<size_t>(dl.n_chunks) * bn;
      CUDA_TRY(g->delta_scratch.reserve(cells * 8 + cells * worst_n * 16));
      dl.partial_sum = g->delta_scratch.as<int64_t>();
      dl.partial = dl.partial_sum + cells;
      dl.abs_sum = d_dsum ? d_dsum + b0 : nullptr;
      dl.worst = d_dworst ? d_dworst + static_cast<size_t>(b0) * worst_n * 3 : nullptr;
      Timed tm(g, stream, 1);
      CUDA_TRY(launch_deltas(dl, stream));
      g_launches += 2;
    }
  }
  if (d_nbins_chk) {
    Timed tm(g, stream, 2);
    CUDA_TRY(launch_util_nbins(lo, hi, c.window_start, c.window_end, out->util_bin_width,
                               d_nbins_chk, count, stream));
    g_launches++;
  }
  if (d_span) {
    Timed tm(g, stream, 2);
    CUDA_TRY(launch_span_finalize(lo, hi, c.window_start, d_span, nullptr, count, stream));
    g_launches++;
  }

  // deadlock (only possible outside the chained class) -> SimulationError
  std::vector<int32_t> host_status;
  if (c.des_only || g->n_coop > 0 || out->n_fixups ||
      (out->status && !is_device_ptr(out->status))) {
    host_status.resize(count);
    CUDA_TRY(cudaMemcpyAsync(host_status.data(), status, static_cast<size_t>(count) * 4,
                             cudaMemcpyDeviceToHost, stream));
  }
  std::vector<int32_t> host_nbins;
  if (out->util_covered && d_nbins_chk) {
    host_nbins.resize(count);
    CUDA_TRY(cudaMemcpyAsync(host_nbins.data(), d_nbins_chk, static_cast<size_t>(count) * 4,
                             cudaMemcpyDeviceToHost, stream));
  }
  if (host_async && !copies.empty() && host_status.empty() && host_nbins.empty()) {
    // copies run on the graph's copy stream behind this call's kernels; the
    // call returns at once (ts_graph_wait blocks until they have landed)
    if (!g->copy_stream) {
      CUDA_TRY(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
      for (cudaEvent_t* e : {&g->copy_done[0], &g->copy_done[1], &g->kernels_done})
        CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    CUDA_TRY(cudaEventRecord(g->kernels_done, stream));
    CUDA_TRY(cudaStreamWaitEvent(g->copy_stream, g->kernels_done, 0));
    for (const OutBuf& b : copies)
      CUDA_TRY(cudaMemcpyAsync(b.user, b.dev, b.bytes, cudaMemcpyDeviceToHost, g->copy_stream));
    CUDA_TRY(cudaEventRecord(g->copy_done[aset], g->copy_stream));
    g->copy_pending[aset] = true;
    g->async_set = aset ^ 1;
    copies.clear();
  }
  for (const OutBuf& b : copies)
    CUDA_TRY(cudaMemcpyAsync(b.user, b.dev, b.bytes, cudaMemcpyDeviceToHost, stream));
  if (!copies.empty() || !host_status.empty() || !host_nbins.empty())
    CUDA_TRY(cudaStreamSynchronize(stream));
  cleanup();
  if (out->status) {
    if (is_device_ptr(out->status))
      CUDA_TRY(cudaMemcpyAsync(out->status, status, static_cast<size_t>(count) * 4,
                               cudaMemcpyDeviceToDevice, stream));
    else
      std::memcpy(out->status, host_status.data(), static_cast<size_t>(count) * 4);
  }
  if (prev_dev >= 0 && prev_dev != g->device) cudaSetDevice(prev_dev);
#ifdef LUMOS_DEBUG_BOUNDS
  CUDA_TRY(cudaStreamSynchronize(stream));
  if (int line = debug_bounds_status())
    return fail(TS_E_CUDA, "bounds check failed (replay.cu line " + std::to_string(line) + ")");
  if (int line = debug_bounds_status_des())
    return fail(TS_E_CUDA, "bounds check failed (des.cu line " + std::to_string(line) + ")");
#endif
  if (out->n_fixups) {
    int32_t nf = 0;
    for (int32_t st : host_status) nf += st > 0;
    if (is_device_ptr(out->n_fixups))
      CUDA_TRY(cudaMemcpy(out->n_fixups, &nf, 4, cudaMemcpyHostToDevice));
    else
      *out->n_fixups = nf;
  }
  if (!host_nbins.empty()) {
    const int32_t need = *std::max_element(host_nbins.begin(), host_nbins.end());
    if (need > out->util_max_bins)
      return fail(TS_E_INVALID_ARGUMENT,
                  "utilization needs " + std::to_string(need) + " bins per rank; util_max_bins is " +
                      std::to_string(out->util_max_bins));
  }
  if (g->n_coop > 0)
    for (int32_t st : host_status)
      if (st == -2)
        return fail(TS_E_CUDA, "cooperative replay stalled waiting for a cross-rank value");
  int64_t n_dead = 0;
  int32_t first_dead = -1;
  for (int32_t i = 0; i < static_cast<int32_t>(host_status.size()); ++i)
    if (host_status[i] < 0 && n_dead++ == 0) first_dead = i;
  if (c.des_only && n_dead > 0) {
    // the reference's message (simulate.cpp:300); the witness ids of a single
    // scenario come from its final event-driven state (still in the scratch)
    int64_t blocked = 0;
    if (cudaMemcpy(&blocked, hi + first_dead, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaGetLastError();
      blocked = -1;
    }
    std::string msg = "deadlock with " + std::to_string(blocked) + " tasks blocked";
    if (count == 1 && blocked >= 0 && g->des_scratch.bytes > 0) {
      std::vector<char> scr(des_scratch_bytes(c.n_tasks, c.des.n_lanes));
      if (scr.size() <= g->des_scratch.bytes &&
          cudaMemcpy(scr.data(), g->des_scratch.as<char>(), scr.size(),
                     cudaMemcpyDeviceToHost) == cudaSuccess)
        msg = deadlock_witness(c.des, c.n_tasks, scr, blocked);
      else
        cudaGetLastError();
    }
    if (count > 1)
      msg += " (scenario " + std::to_string(sc->first + first_dead) + "; " +
             std::to_string(n_dead) + " of " + std::to_string(count) + " scenarios deadlocked)";
    return fail(TS_E_SIMULATION, msg);
  }
  return TS_OK;
}

int ts_profile_enable(ts_graph* g, int enable) {
  if (!g) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  g->profile = enable != 0;
  return TS_OK;
}

int ts_profile_read(ts_graph* g, ts_profile_stats* out) {
  if (!g || !out) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  std::memset(out, 0, sizeof(*out));
  for (auto& m : g->marks) {
    CUDA_TRY(cudaEventSynchronize(m.b));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, m.a, m.b));
    if (m.kind == 0) {
      out->walk_ms += ms;
      out->walk_launches++;
    } else if (m.kind == 1) {
      out->reduce_ms += ms;
      out->reduce_launches++;
    } else {
      out->other_ms += ms;
      out->other_launches++;
    }
    g->event_pool.push_back(m.a);
    g->event_pool.push_back(m.b);
  }
  g->marks.clear();
  return TS_OK;
}

int ts_simulate(ts_graph* g, int64_t* start, int64_t* fin, int64_t* span) {
  if (!g) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  ts_scenarios sc{};
  sc.count = 1;
  ts_result r{};
  r.start = start;
  r.fin = fin;
  r.ld = 1;
  r.span = span;
  return ts_replay_batch(g, &sc, &r, nullptr);
}

int ts_scenario_durations(ts_graph* g, const ts_scenarios* sc, int64_t* dur, int64_t ld,
                          void* stream_) {
  if (!g || !sc || !dur) return fail(TS_E_INVALID_ARGUMENT, "null argument");
  if (!g->has_device) return fail(TS_E_CUDA, "graph was compiled without a device");
  if (ld < sc->count) return fail(TS_E_INVALID_ARGUMENT, "ld must be >= count");
  ScenarioParams sp;
  if (int rc = scenario_params(g, sc, sp)) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const size_t bytes = static_cast<size_t>(g->cg.n_tasks) * static_cast<size_t>(ld) * 8;
  int64_t* d = dur;
  void* tmp = nullptr;
  if (!is_device_ptr(dur)) {
    CUDA_TRY(cudaMalloc(&tmp, bytes));
    d = static_cast<int64_t*>(tmp);
  }
  const int32_t* staged_num = nullptr;
  void* tmp_num = nullptr;
  if (sp.scale_num && !is_device_ptr(sp.scale_num)) {
    size_t nb = static_cast<size_t>(sc->count) * sp.n_classes * 4;
    CUDA_TRY(cudaMalloc(&tmp_num, nb));
    CUDA_TRY(cudaMemcpyAsync(tmp_num, sp.scale_num, nb, cudaMemcpyHostToDevice, stream));
    staged_num = static_cast<const int32_t*>(tmp_num);
    sp.scale_num = staged_num;
  }
  if (sc->retime) {
    if (sp.mode & kModeExplicit) {
      if (tmp) cudaFree(tmp);
      return fail(TS_E_INVALID_ARGUMENT, "retime cannot be combined with explicit durations");
    }
    RetimeParams rtp{};
    if (int rc = retime_stage(g, sc->retime, sc->count, stream, rtp)) {
      if (tmp) cudaFree(tmp);
      return rc;
    }
    rtp.sp = sp;
    rtp.dur = d;
    rtp.ld = ld;
    CUDA_TRY(launch_retime_durations(rtp, stream));
  } else {
    CUDA_TRY(launch_durations(sp, g->d_base, g->d_cls, g->cg.n_tasks, d, ld, stream));
  }
  g_launches++;
  if (tmp) {
    CUDA_TRY(cudaMemcpyAsync(dur, d, bytes, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    cudaFree(tmp);
  }
  if (tmp_num) {
    CUDA_TRY(cudaStreamSynchronize(stream));
    cudaFree(tmp_num);
  }
  return TS_OK;
}

}  // extern "C"
