// synth.cpp — synthetic GPT-like training-iteration generator (host side).
//
// Restates the reference generator (paths under /root/reference/proj/src):
//   cost formulas                 cost.cpp:39-88
//   pipeline_spec_for             synth.cpp:71-138
//   schedule_1f1b                 pipeline.cpp:9-25
//   Builder (op layout + timing)  pipeline.cpp:92-470
// and produces, from one timing pass,
//   * the replay graph: the one-iteration trace run through build_graph +
//     merge_ranks (ingest.cpp) — what `tracesim replay` simulates, and
//   * the estimate graph: the same tasks with the generator's own exact
//     dependencies (thread order, stream order, event waits, syncs, host
//     hand-offs) plus gates for the p2p rendezvous and the collective barrier
//     (pipeline.cpp:361-441), with intrinsic (not recorded) durations.
// Tensor parallelism is realised as TP replicas of every (stage, dp) rank
// (rank r -> r * tp + t); the reference models no TP
// traffic (synth.cpp:18-19).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "ingest.hpp"
#include "synth.hpp"

namespace lumos {

namespace {

// ------------------------------------------------------------ cost formulas
int64_t llr(double v) { return static_cast<int64_t>(std::llround(v)); }

int64_t gemm_scaled_us(int64_t ref_us, int64_t rm, int64_t rn, int64_t rk, int64_t m, int64_t n,
                       int64_t k) {
  const double ratio = (static_cast<double>(m) * n * k) / (static_cast<double>(rm) * rn * rk);
  return std::max<int64_t>(0, llr(static_cast<double>(ref_us) * ratio));
}

enum Coll { ALLREDUCE, SENDRECV };

int64_t collective_cost_us(Coll c, int64_t bytes, int group, double alpha, double bpu) {
  const double g = group;
  const double scale = c == ALLREDUCE ? 2.0 * (g - 1.0) / g : 1.0;
  const double t = alpha + static_cast<double>(bytes) * scale / bpu;
  return std::max<int64_t>(0, llr(t));
}

// retime metadata of a kernel: what the reference generator puts in the
// event args (synth.cpp:46-48 m/n/k; :122-124 allreduce bytes / collective /
// group_size; :133 optimizer bytes with region "opt", pipeline.cpp:297;
// pipeline.cpp:162-166 p2p region / dir / bytes), classified as TS_RT_*
struct KMeta {
  uint8_t kind = TS_RT_NONE;
  int64_t bytes = -1;
  int32_t group = 0;
  int64_t m = 0, n = 0, k = 0;
};

struct KSpec {
  int32_t name;
  int64_t dur;
  KMeta meta{};
  MetaList args{};  // KernelSpec::args (kept for traces that carry Task.meta)
};

struct StageSpec {
  std::vector<std::vector<KSpec>> fwd, bwd;
  std::vector<KSpec> pre_fwd, post_fwd, pre_bwd, post_bwd, reduce, optimizer;
};

struct PSpec {
  int pp = 1, dp = 1, m = 1;
  std::vector<StageSpec> stages;
  int64_t launch = 5, record = 2, wait = 2, sync = 5;
  int64_t p2p_send = 0, p2p_recv_base = 0;
  int64_t act_bytes = 0;  // p2p transfer size (formulas::activation_bytes)
  int64_t origin = 0;
  int compute_stream = 7, reduce_stream = 9, p2p_stream = 11;
  int main_thread = 100, helper_thread = 200;
  int64_t first_event = 1, first_correlation = 1;
};

// ------------------------------------------------------------------ keys
// packed (kind, fwd, stage, dp, mb): 1 p2p, 2 sync hand-off, 3 allreduce group
uint64_t key(int kind, bool fwd, int a, int b, int c) {
  return (static_cast<uint64_t>(kind) << 56) | (static_cast<uint64_t>(fwd) << 55) |
         (static_cast<uint64_t>(a & 0x7FFF) << 40) | (static_cast<uint64_t>(b & 0xFFFF) << 24) |
         static_cast<uint64_t>(c & 0xFFFFFF);
}

enum PType { P_LAUNCH, P_RECORD, P_WAIT, P_SSYNC, P_DSYNC };

struct POp {
  PType type = P_LAUNCH;
  int64_t cpu_dur = 0, kernel_dur = 0;
  int64_t cpu_index = -1, kernel_index = -1;  // cost indices
  int32_t kname = 0;
  int32_t kargs = -1;                         // kernel event args (keep_meta)
  int stream = -1;
  int64_t event_id = -1, corr = -1;
  uint64_t recv_key = 0, send_key = 0, barrier_key = 0, pub_key = 0;
  int barrier_size = 0;
  std::vector<uint64_t> pre_keys;
  int64_t ev_cpu = -1, ev_kernel = -1;  // emitted event indices
};

struct ThreadOps {
  int rank = 0, thread = 0;
  std::vector<POp> ops;
  size_t cursor = 0;
};

struct RankState {
  std::map<int, int64_t> cpu_clock, stream_clock, stream_floor;
  std::map<int64_t, int64_t> event_bind;
  std::map<int, int64_t> last_cpu_ev, last_kernel_ev;
  std::map<int64_t, int64_t> bind_ev;           // event id -> bound kernel event
  std::map<int, std::vector<int64_t>> pending;  // stream -> floor predecessors
};

struct GenEvent {
  Event ev;
  int64_t cost = 0;  // intrinsic duration (estimate graph)
  int32_t args = -1; // TraceEvent::args (Builder::arg_lists), keep_meta only
};

// args with tags applied over them, key order (launch_op, pipeline.cpp:119-127)
MetaList with_tags(const MetaList& args, const MetaList& tags) {
  std::map<std::string, std::string> m(args.begin(), args.end());
  for (const auto& [k, v] : tags) m[k] = v;
  return MetaList(m.begin(), m.end());
}

class Builder {
 public:
  Builder(const PSpec& s, Names& names, bool keep_meta = false)
      : s_(s), names_(names), keep_meta_(keep_meta) {
    n_launch_ = names.get("cudaLaunchKernel");
    n_record_ = names.get("cudaEventRecord");
    n_wait_ = names.get("cudaStreamWaitEvent");
    n_ssync_ = names.get("cudaStreamSynchronize");
    n_dsync_ = names.get("cudaDeviceSynchronize");
    n_sendrecv_ = names.get("ncclDevKernel_SendRecv");
  }

  void run() {
    for (int j = 0; j < s_.dp; ++j)
      for (int st = 0; st < s_.pp; ++st) build_rank(st, j);
    time_all();
  }

  std::vector<GenEvent> events;
  std::vector<MetaList> arg_lists;  // keep_meta: the events' args
  std::vector<KMeta> kmeta;  // by kernel cost index (op_index)
  std::vector<std::pair<int64_t, int64_t>> edges;             // estimate graph, event ids
  std::vector<std::tuple<int64_t, int64_t, uint8_t>> gates;  // (from, to, kind)
  int64_t end = 0;

 private:
  const PSpec& s_;
  Names& names_;
  bool keep_meta_ = false;
  int32_t n_launch_, n_record_, n_wait_, n_ssync_, n_dsync_, n_sendrecv_;
  std::vector<ThreadOps> threads_;
  std::map<int, RankState> state_;
  std::unordered_map<uint64_t, std::pair<int64_t, int64_t>> published_;  // time, event
  std::unordered_map<uint64_t, std::map<int, int64_t>> barrier_starts_;
  std::unordered_map<uint64_t, std::vector<POp*>> barrier_members_;
  int64_t next_event_ = s_.first_event, next_corr_ = s_.first_correlation, op_index_ = 0;

  int64_t cost(int64_t base) {
    ++op_index_;
    return base < 0 ? 0 : base;
  }
  int rank_of(int stage, int dp) const { return stage + s_.pp * dp; }

  int32_t add_args(MetaList a) {
    arg_lists.push_back(std::move(a));
    return static_cast<int32_t>(arg_lists.size()) - 1;
  }
  static MetaList slot_tags(bool fwd, int mb) {  // pipeline.cpp:206-216
    return {{"mb", std::to_string(mb)}, {"phase", fwd ? "fwd" : "bwd"}};
  }
  POp launch(const KSpec& k, const MetaList& tags = {}) {
    POp op;
    op.type = P_LAUNCH;
    if (keep_meta_) op.kargs = add_args(with_tags(k.args, tags));
    op.cpu_index = op_index_;
    op.cpu_dur = cost(s_.launch);
    op.kernel_index = op_index_;
    if (k.meta.kind != TS_RT_NONE) {
      if (kmeta.size() <= static_cast<size_t>(op_index_)) kmeta.resize(op_index_ + 1);
      kmeta[op_index_] = k.meta;
    }
    op.kernel_dur = cost(k.dur);
    op.kname = k.name;
    op.corr = next_corr_++;
    return op;
  }
  POp record(int stream) {
    POp op;
    op.type = P_RECORD;
    op.cpu_index = op_index_;
    op.cpu_dur = cost(s_.record);
    op.stream = stream;
    op.event_id = next_event_++;
    return op;
  }
  POp wait(int stream, int64_t ev) {
    POp op;
    op.type = P_WAIT;
    op.cpu_index = op_index_;
    op.cpu_dur = cost(s_.wait);
    op.stream = stream;
    op.event_id = ev;
    return op;
  }
  POp sync(bool device, int stream, uint64_t pub) {
    POp op;
    op.type = device ? P_DSYNC : P_SSYNC;
    op.cpu_index = op_index_;
    op.cpu_dur = cost(s_.sync);
    op.stream = stream;
    op.pub_key = pub;
    return op;
  }

  // p2p_kernel's args (pipeline.cpp:157-169)
  MetaList p2p_args(bool send, bool fwd, int peer) const {
    if (!keep_meta_) return {};
    return {{"bytes", std::to_string(s_.act_bytes)}, {"collective", "sendrecv"},
            {"dir", send ? "send" : "recv"}, {"peer_stage", std::to_string(peer)},
            {"phase", fwd ? "fwd" : "bwd"}, {"region", "p2p"}};
  }
  void emit_recv(std::vector<POp>& ops, bool fwd, int stage, int dp, int mb) {
    int from = fwd ? stage - 1 : stage + 1;
    KMeta rm;
    rm.kind = TS_RT_P2P_RECV;
    rm.bytes = s_.act_bytes;
    POp r = launch({n_sendrecv_, s_.p2p_recv_base, rm, p2p_args(false, fwd, from)},
                   {{"mb", std::to_string(mb)}});
    r.stream = s_.p2p_stream;
    r.recv_key = key(1, fwd, from, dp, mb);
    ops.push_back(r);
    POp rec = record(s_.p2p_stream);
    int64_t ev = rec.event_id;
    ops.push_back(rec);
    ops.push_back(wait(s_.compute_stream, ev));
  }
  void emit_send(std::vector<POp>& ops, bool fwd, int stage, int dp, int mb) {
    POp rec = record(s_.compute_stream);
    int64_t ev = rec.event_id;
    ops.push_back(rec);
    ops.push_back(wait(s_.p2p_stream, ev));
    KMeta sm;
    sm.kind = TS_RT_P2P_SEND;
    sm.bytes = s_.act_bytes;
    const int to = fwd ? stage + 1 : stage - 1;
    POp snd = launch({n_sendrecv_, s_.p2p_send, sm, p2p_args(true, fwd, to)},
                     {{"mb", std::to_string(mb)}});
    snd.stream = s_.p2p_stream;
    snd.send_key = key(1, fwd, stage, dp, mb);
    ops.push_back(snd);
  }
  void emit_compute(std::vector<POp>& ops, const std::vector<KSpec>& ks,
                    const MetaList& tags = {}) {
    for (const KSpec& k : ks) {
      POp op = launch(k, tags);
      op.stream = s_.compute_stream;
      ops.push_back(op);
    }
  }
  // tags of a slot's compute (pipeline.cpp:206-216, 224-272); built only
  // when the trace keeps its args
  MetaList tags(bool fwd, int mb, const char* region, int layer = -1) const {
    if (!keep_meta_) return {};
    MetaList t = slot_tags(fwd, mb);
    if (layer >= 0) t.emplace_back("layer", std::to_string(layer));
    if (region) t.emplace_back("region", region);
    return t;
  }
  int first_layer(int stage) const {
    int acc = 0;
    for (int q = 0; q < stage; ++q) acc += static_cast<int>(s_.stages[q].fwd.size());
    return acc;
  }
  void emit_fwd(std::vector<POp>& ops, int stage, int dp, int mb) {
    const StageSpec& st = s_.stages[stage];
    if (stage > 0) emit_recv(ops, true, stage, dp, mb);
    if (stage == 0) emit_compute(ops, st.pre_fwd, tags(true, mb, "embed"));
    const int base = first_layer(stage);
    for (size_t l = 0; l < st.fwd.size(); ++l)
      emit_compute(ops, st.fwd[l], tags(true, mb, nullptr, base + static_cast<int>(l)));
    if (stage == s_.pp - 1) emit_compute(ops, st.post_fwd, tags(true, mb, "head"));
    if (stage < s_.pp - 1) emit_send(ops, true, stage, dp, mb);
  }
  void emit_bwd(std::vector<POp>& ops, int stage, int dp, int mb) {
    const StageSpec& st = s_.stages[stage];
    if (stage < s_.pp - 1) emit_recv(ops, false, stage, dp, mb);
    if (stage == s_.pp - 1) emit_compute(ops, st.pre_bwd, tags(false, mb, "head"));
    const int base = first_layer(stage);
    for (int l = static_cast<int>(st.bwd.size()) - 1; l >= 0; --l)
      emit_compute(ops, st.bwd[l], tags(false, mb, nullptr, base + l));
    if (stage == 0) emit_compute(ops, st.post_bwd, tags(false, mb, "embed"));
    if (stage > 0) emit_send(ops, false, stage, dp, mb);
  }
  void emit_tail(std::vector<POp>& ops, int stage, uint64_t gate_key) {
    const StageSpec& st = s_.stages[stage];
    bool gated = gate_key != 0;
    auto gate = [&](POp op) {
      if (gated) {
        op.pre_keys.push_back(gate_key);
        gated = false;
      }
      ops.push_back(op);
    };
    if (s_.dp > 1 && !st.reduce.empty()) {
      POp rec = record(s_.compute_stream);
      int64_t ev = rec.event_id;
      gate(rec);
      ops.push_back(wait(s_.reduce_stream, ev));
      int seq = 0;
      for (const KSpec& k : st.reduce) {
        POp op = launch(k, {{"region", "dp"}});
        op.stream = s_.reduce_stream;
        op.barrier_key = key(3, false, stage, 0, seq++);
        op.barrier_size = s_.dp;
        ops.push_back(op);
      }
      POp rec2 = record(s_.reduce_stream);
      int64_t ev2 = rec2.event_id;
      ops.push_back(rec2);
      ops.push_back(wait(s_.compute_stream, ev2));
    }
    for (const KSpec& k : st.optimizer) {
      POp op = launch(k, {{"region", "opt"}});
      op.stream = s_.compute_stream;
      gate(op);
    }
    gate(sync(true, -1, 0));
  }

  void build_rank(int stage, int dp) {
    const int rank = rank_of(stage, dp);
    RankState& st = state_[rank];
    st.cpu_clock[s_.main_thread] = s_.origin;
    st.stream_clock[s_.compute_stream] = s_.origin;
    st.stream_clock[s_.reduce_stream] = s_.origin;
    st.stream_clock[s_.p2p_stream] = s_.origin;
    if (s_.pp == 1) {
      st.cpu_clock[s_.helper_thread] = s_.origin;
      ThreadOps main, helper;
      main.rank = helper.rank = rank;
      main.thread = s_.main_thread;
      helper.thread = s_.helper_thread;
      for (int mb = 0; mb < s_.m; ++mb) {
        size_t first_main = main.ops.size();
        emit_fwd(main.ops, 0, dp, mb);
        if (mb > 0) main.ops[first_main].pre_keys.push_back(key(2, false, 0, dp, mb - 1));
        main.ops.push_back(sync(false, s_.compute_stream, key(2, true, 0, dp, mb)));
        size_t first_helper = helper.ops.size();
        emit_bwd(helper.ops, 0, dp, mb);
        helper.ops[first_helper].pre_keys.push_back(key(2, true, 0, dp, mb));
        helper.ops.push_back(sync(false, s_.compute_stream, key(2, false, 0, dp, mb)));
      }
      emit_tail(main.ops, 0, key(2, false, 0, dp, s_.m - 1));
      threads_.push_back(std::move(main));
      threads_.push_back(std::move(helper));
      return;
    }
    ThreadOps main;
    main.rank = rank;
    main.thread = s_.main_thread;
    // schedule_1f1b (pipeline.cpp:9-25)
    const int warmup = std::min(s_.pp - stage, s_.m);
    int nf = 0, nb = 0;
    for (; nf < warmup; ++nf) emit_fwd(main.ops, stage, dp, nf);
    while (nb < s_.m) {
      emit_bwd(main.ops, stage, dp, nb++);
      if (nf < s_.m) emit_fwd(main.ops, stage, dp, nf++);
    }
    emit_tail(main.ops, stage, 0);
    threads_.push_back(std::move(main));
  }

  int64_t emit(const ThreadOps& to, int32_t name, uint8_t cat, int64_t ts, int64_t dur,
               int tid, int stream, int64_t corr, int64_t arg_ev, int64_t arg_stream,
               int64_t op_index, int64_t cost_dur, int32_t args = -1) {
    GenEvent g;
    g.args = args;
    g.ev.name = name;
    g.ev.cat = cat;
    g.ev.ts = ts;
    g.ev.dur = dur;
    g.ev.pid = to.rank;
    g.ev.tid = tid;
    g.ev.stream = stream;
    g.ev.corr = corr;
    g.ev.arg_event = arg_ev;
    g.ev.arg_stream = arg_stream;
    g.ev.op_index = op_index;
    g.cost = cost_dur;
    events.push_back(g);
    return static_cast<int64_t>(events.size()) - 1;
  }

  // a runtime call's args (pipeline.cpp:404-423)
  int32_t event_args(int64_t event_id, int stream) {
    if (!keep_meta_) return -1;
    MetaList a;
    if (event_id != kNoArg) a.emplace_back("event", std::to_string(event_id));
    a.emplace_back("stream", std::to_string(stream));
    return add_args(std::move(a));
  }

  // host op: thread-order edge + hand-off edges
  void cpu_edges(RankState& st, const ThreadOps& to, const POp& op, int64_t ev) {
    auto it = st.last_cpu_ev.find(to.thread);
    if (it != st.last_cpu_ev.end()) edges.emplace_back(it->second, ev);
    st.last_cpu_ev[to.thread] = ev;
    for (uint64_t k : op.pre_keys) edges.emplace_back(published_.at(k).second, ev);
  }

  bool try_process(ThreadOps& to) {
    if (to.cursor >= to.ops.size()) return false;
    POp& op = to.ops[to.cursor];
    RankState& st = state_[to.rank];
    int64_t cpu = st.cpu_clock[to.thread];
    for (uint64_t k : op.pre_keys) {
      auto it = published_.find(k);
      if (it == published_.end()) return false;
      cpu = std::max(cpu, it->second.first);
    }
    switch (op.type) {
      case P_LAUNCH: {
        const int64_t cpu_end = cpu + op.cpu_dur;
        const int64_t kstart =
            std::max({st.stream_clock[op.stream], st.stream_floor[op.stream], cpu_end});
        int64_t kend;
        if (op.recv_key) {
          auto it = published_.find(op.recv_key);
          if (it == published_.end()) return false;
          kend = std::max(kstart, it->second.first) + op.kernel_dur;
        } else if (op.barrier_key) {
          auto& starts = barrier_starts_[op.barrier_key];
          starts[to.rank] = kstart;
          auto& members = barrier_members_[op.barrier_key];
          if (std::find(members.begin(), members.end(), &op) == members.end())
            members.push_back(&op);
          if (static_cast<int>(starts.size()) != op.barrier_size) return false;
          int64_t latest = kstart;
          for (const auto& [r, s] : starts) latest = std::max(latest, s);
          kend = latest + op.kernel_dur;
        } else {
          kend = kstart + op.kernel_dur;
        }
        const int64_t evc = emit(to, n_launch_, CAT_RUNTIME, cpu, op.cpu_dur, to.thread, -1,
                                 op.corr, kNoArg, kNoArg, op.cpu_index, op.cpu_dur);
        cpu_edges(st, to, op, evc);
        const int64_t evk = emit(to, op.kname, CAT_KERNEL, kstart, kend - kstart, op.stream,
                                 op.stream, op.corr, kNoArg, kNoArg, op.kernel_index,
                                 op.kernel_dur, op.kargs);
        op.ev_cpu = evc;
        op.ev_kernel = evk;
        edges.emplace_back(evc, evk);
        auto lk = st.last_kernel_ev.find(op.stream);
        if (lk != st.last_kernel_ev.end()) edges.emplace_back(lk->second, evk);
        for (int64_t p : st.pending[op.stream]) edges.emplace_back(p, evk);
        st.pending[op.stream].clear();
        st.last_kernel_ev[op.stream] = evk;
        if (op.recv_key) gates.emplace_back(published_.at(op.recv_key).second, evk, TS_GATE_FIN);
        st.cpu_clock[to.thread] = cpu_end;
        st.stream_clock[op.stream] = kend;
        if (op.send_key) published_[op.send_key] = {kend, evk};
        break;
      }
      case P_RECORD: {
        st.event_bind[op.event_id] = st.stream_clock[op.stream];
        auto lk = st.last_kernel_ev.find(op.stream);
        st.bind_ev[op.event_id] = lk == st.last_kernel_ev.end() ? -1 : lk->second;
        const int64_t ev = emit(to, n_record_, CAT_RUNTIME, cpu, op.cpu_dur, to.thread, -1, -1,
                                op.event_id, op.stream, op.cpu_index, op.cpu_dur,
                                event_args(op.event_id, op.stream));
        cpu_edges(st, to, op, ev);
        st.cpu_clock[to.thread] = cpu + op.cpu_dur;
        break;
      }
      case P_WAIT: {
        const int64_t bound = st.event_bind[op.event_id];
        st.stream_floor[op.stream] = std::max(st.stream_floor[op.stream], bound);
        auto b = st.bind_ev.find(op.event_id);
        if (b != st.bind_ev.end() && b->second >= 0) st.pending[op.stream].push_back(b->second);
        const int64_t ev = emit(to, n_wait_, CAT_RUNTIME, cpu, op.cpu_dur, to.thread, -1, -1,
                                op.event_id, op.stream, op.cpu_index, op.cpu_dur,
                                event_args(op.event_id, op.stream));
        cpu_edges(st, to, op, ev);
        st.cpu_clock[to.thread] = cpu + op.cpu_dur;
        break;
      }
      case P_SSYNC: {
        const int64_t wake = std::max(cpu, st.stream_clock[op.stream]);
        const int64_t ev = emit(to, n_ssync_, CAT_RUNTIME, wake, op.cpu_dur, to.thread, -1, -1,
                                kNoArg, op.stream, op.cpu_index, op.cpu_dur,
                                event_args(kNoArg, op.stream));
        cpu_edges(st, to, op, ev);
        auto lk = st.last_kernel_ev.find(op.stream);
        if (lk != st.last_kernel_ev.end()) edges.emplace_back(lk->second, ev);
        st.cpu_clock[to.thread] = wake + op.cpu_dur;
        if (op.pub_key) published_[op.pub_key] = {wake + op.cpu_dur, ev};
        break;
      }
      case P_DSYNC: {
        int64_t wake = cpu;
        for (const auto& [stream, clk] : st.stream_clock) wake = std::max(wake, clk);
        const int64_t ev = emit(to, n_dsync_, CAT_RUNTIME, wake, op.cpu_dur, to.thread, -1, -1,
                                kNoArg, kNoArg, op.cpu_index, op.cpu_dur);
        cpu_edges(st, to, op, ev);
        for (const auto& [stream, kev] : st.last_kernel_ev) edges.emplace_back(kev, ev);
        st.cpu_clock[to.thread] = wake + op.cpu_dur;
        if (op.pub_key) published_[op.pub_key] = {wake + op.cpu_dur, ev};
        break;
      }
    }
    ++to.cursor;
    return true;
  }

  void time_all() {
    size_t total = 0, done = 0;
    for (const auto& t : threads_) total += t.ops.size();
    while (done < total) {
      size_t before = done;
      for (auto& t : threads_)
        while (try_process(t)) ++done;
      if (done == before) throw std::logic_error("pipeline schedule did not make progress");
    }
    // collective barrier: each member's finish waits on every member's start
    for (auto& [k, members] : barrier_members_)
      for (POp* a : members)
        for (POp* b : members)
          if (a != b) gates.emplace_back(b->ev_kernel, a->ev_kernel, TS_GATE_START);
    end = s_.origin;
    for (const GenEvent& g : events) end = std::max(end, g.ev.ts + g.ev.dur);
  }
};

PSpec pspec_for(const ts_synth_spec& sp, Names& names) {
  PSpec ps;
  ps.pp = sp.pp;
  ps.dp = sp.dp;
  ps.m = sp.num_microbatches;
  ps.launch = sp.launch_us;
  ps.record = sp.record_us;
  ps.wait = sp.wait_us;
  ps.sync = sp.sync_us;
  ps.origin = sp.origin;
  const int64_t t = sp.tokens_per_microbatch, d = sp.d_model, f = sp.d_ffn;
  const int64_t act = t * d * 2;  // formulas::activation_bytes (cost.cpp:83-85)
  ps.p2p_send = collective_cost_us(SENDRECV, act, 2, sp.alpha_us, sp.bytes_per_us);
  ps.act_bytes = act;
  ps.p2p_recv_base = sp.p2p_recv_base_us;
  auto gemm = [&](const char* name, int64_t m, int64_t n, int64_t k, double factor) {
    int64_t base = gemm_scaled_us(sp.gemm_ref_us, sp.gemm_ref_mnk, 1, 1, m, n, k);
    KMeta g;
    g.kind = TS_RT_GEMM;
    g.m = m;
    g.n = n;
    g.k = k;
    return KSpec{names.get(name), llr(static_cast<double>(base) * factor), g,
                 {{"k", std::to_string(k)}, {"m", std::to_string(m)}, {"n", std::to_string(n)}}};
  };
  std::vector<KSpec> lf{gemm("gemm_qkv", t, d, d, 1.0), {names.get("attn_core"), sp.attn_misc_us},
                        gemm("gemm_mlp", t, f, d, 1.0)};
  std::vector<KSpec> lb{gemm("gemm_mlp_bwd", t, f, d, sp.bwd_gemm_factor),
                        {names.get("attn_core_bwd"),
                         llr(static_cast<double>(sp.attn_misc_us) * sp.bwd_gemm_factor)},
                        gemm("gemm_qkv_bwd", t, d, d, sp.bwd_gemm_factor)};
  const int per_stage = sp.n_layers / sp.pp;
  const int64_t layer_bytes = (4 * d * d + 2 * d * f) * 2;  // cost.cpp:74-77
  const int64_t vocab_bytes = 2 * sp.vocab * d;
  for (int s = 0; s < sp.pp; ++s) {
    StageSpec st;
    st.fwd.assign(per_stage, lf);
    st.bwd.assign(per_stage, lb);
    if (s == 0) {
      st.pre_fwd.push_back({names.get("embedding_fwd"), sp.embed_us});
      st.post_bwd.push_back({names.get("embedding_bwd"), sp.embed_us});
    }
    if (s == sp.pp - 1) {
      st.post_fwd.push_back({names.get("norm_loss_fwd"), sp.head_us});
      st.pre_bwd.push_back({names.get("loss_bwd"), sp.loss_grad_us});
    }
    int64_t rbytes = layer_bytes * per_stage;  // synth_stage_reduce_bytes (synth.cpp:61-69)
    if (s == 0) rbytes += vocab_bytes;
    if (s == sp.pp - 1) rbytes += vocab_bytes;
    KMeta ar;
    ar.kind = TS_RT_ALLREDUCE;
    ar.bytes = rbytes;
    ar.group = sp.dp;
    if (sp.dp > 1)
      st.reduce.push_back({names.get("ncclDevKernel_AllReduce_Sum_f16"),
                           collective_cost_us(ALLREDUCE, rbytes, sp.dp, sp.alpha_us,
                                              sp.bytes_per_us),
                           ar,
                           {{"bytes", std::to_string(rbytes)},
                            {"collective", "allreduce"},
                            {"group_size", std::to_string(sp.dp)}}});
    KMeta om;
    om.kind = TS_RT_OPT;
    om.bytes = rbytes;
    st.optimizer.push_back(
        {names.get("adam_step"),
         llr(static_cast<double>(sp.optimizer_ref_us) * static_cast<double>(rbytes) /
             static_cast<double>(sp.optimizer_ref_bytes)),
         om,
         {{"bytes", std::to_string(rbytes)}}});
    ps.stages.push_back(std::move(st));
  }
  return ps;
}


// ------------------------------------------- a user PipelineSpec (Mode B)
// strict integer of an args string (transform.cpp:19-30 meta_i64)
bool strict_int(const std::string& v, int64_t& out) {
  if (v.empty()) return false;
  try {
    size_t pos = 0;
    const long long x = std::stoll(v, &pos);
    if (pos != v.size()) return false;
    out = x;
    return true;
  } catch (const std::exception&) {
    return false;
  }
}

// The retime metadata a kernel's task carries: its KernelSpec args with the
// builder's role tag applied (tags override args, pipeline.cpp:122-123; role
// regions embed / head / dp / opt, pipeline.cpp:229-297), classified the way
// change_hidden / scale_dp read Task.meta (transform.cpp:219-349) on the op
// class build_graph gives the kernel by name (build.cpp:93-98).
KMeta kernel_meta(const ts_kernel_spec& k, const char* role_region) {
  std::map<std::string, std::string> args;
  for (int32_t a = 0; a < k.n_args; ++a)
    if (k.arg_keys && k.arg_keys[a] && k.arg_values && k.arg_values[a])
      args[k.arg_keys[a]] = k.arg_values[a];
  if (role_region) args["region"] = role_region;
  auto get = [&](const char* key) {
    auto it = args.find(key);
    return it == args.end() ? std::string() : it->second;
  };
  auto num = [&](const char* key, int64_t absent, bool* present = nullptr) {
    int64_t v = absent;
    auto it = args.find(key);
    const bool ok = it != args.end() && strict_int(it->second, v);
    if (!ok) v = absent;
    if (present) *present = ok;
    return v;
  };
  KMeta m;
  bool has_bytes = false;
  m.bytes = num("bytes", -1, &has_bytes);
  m.group = static_cast<int32_t>(num("group_size", 0));
  m.m = num("m", 0);
  m.n = num("n", 0);
  m.k = num("k", 0);
  if (is_comm_name(k.name ? k.name : "")) {
    if (get("collective") == "allreduce") m.kind = TS_RT_ALLREDUCE;
    else if (get("region") == "p2p" && has_bytes)
      m.kind = get("dir") != "recv" ? TS_RT_P2P_SEND : TS_RT_P2P_RECV;
  } else if (m.m > 0 && m.n > 0 && m.k > 0) {
    m.kind = TS_RT_GEMM;
  } else if (get("region") == "opt" && has_bytes) {
    m.kind = TS_RT_OPT;
  }
  return m;
}

int pspec_of(const ts_pipeline_spec& c, Names& names, PSpec& ps, std::string& err) {
  // build_pipeline's checks (pipeline.cpp:62-68)
  if (c.pp < 1 || c.dp < 1) {
    err = "pipeline: pp and dp must be >= 1";
    return TS_E_INVALID_ARGUMENT;
  }
  if (c.n_stages != c.pp || !c.stages) {
    err = "pipeline: need one stage spec per pipeline stage";
    return TS_E_INVALID_ARGUMENT;
  }
  if (c.num_microbatches < 1) {
    err = "pipeline: need at least one microbatch";
    return TS_E_INVALID_ARGUMENT;
  }
  ps = PSpec{};
  ps.pp = c.pp;
  ps.dp = c.dp;
  ps.m = c.num_microbatches;
  ps.launch = c.launch_us;
  ps.record = c.record_us;
  ps.wait = c.wait_us;
  ps.sync = c.sync_us;
  ps.p2p_send = c.p2p_send_us;
  ps.p2p_recv_base = c.p2p_recv_base_us;
  ps.act_bytes = c.activation_bytes;
  ps.origin = c.origin;
  ps.compute_stream = c.compute_stream;
  ps.reduce_stream = c.reduce_stream;
  ps.p2p_stream = c.p2p_stream;
  ps.main_thread = c.main_thread;
  ps.helper_thread = c.helper_thread;
  ps.first_event = c.first_event;
  ps.first_correlation = c.first_correlation;
  auto list = [&](const ts_kernel_list& l, const char* role, std::vector<KSpec>& outl) {
    outl.clear();
    for (int32_t i = 0; i < l.n; ++i) {
      const ts_kernel_spec& k = l.k[i];
      std::map<std::string, std::string> args;
      for (int32_t a = 0; a < k.n_args; ++a)
        if (k.arg_keys && k.arg_keys[a] && k.arg_values && k.arg_values[a])
          args[k.arg_keys[a]] = k.arg_values[a];
      outl.push_back({names.get(k.name ? k.name : ""), k.duration, kernel_meta(k, role),
                      MetaList(args.begin(), args.end())});
    }
  };
  for (int32_t s = 0; s < c.pp; ++s) {
    const ts_stage_spec& cs = c.stages[s];
    StageSpec st;
    st.fwd.resize(cs.n_layers);
    st.bwd.resize(cs.n_layers);
    for (int32_t l = 0; l < cs.n_layers; ++l) {
      list(cs.layers_fwd[l], nullptr, st.fwd[l]);
      list(cs.layers_bwd[l], nullptr, st.bwd[l]);
    }
    list(cs.pre_fwd, "embed", st.pre_fwd);
    list(cs.post_bwd, "embed", st.post_bwd);
    list(cs.post_fwd, "head", st.post_fwd);
    list(cs.pre_bwd, "head", st.pre_bwd);
    list(cs.reduce, "dp", st.reduce);
    list(cs.optimizer, "opt", st.optimizer);
    ps.stages.push_back(std::move(st));
  }
  return TS_OK;
}

}  // namespace

int graph_of_pspec(const PSpec& ps, bool estimate, int tp, int slice_rank, SynthOutput& out,
                   std::string& err, bool keep_meta = false);

void pipeline_defaults(ts_pipeline_spec* c) {
  std::memset(c, 0, sizeof(*c));
  // PipelineSpec / HostCosts defaults (pipeline.hpp:47-80)
  c->pp = c->dp = c->num_microbatches = 1;
  c->launch_us = 5;
  c->record_us = 2;
  c->wait_us = 2;
  c->sync_us = 5;
  c->compute_stream = 7;
  c->reduce_stream = 9;
  c->p2p_stream = 11;
  c->main_thread = 100;
  c->helper_thread = 200;
  c->first_event = 1;
  c->first_correlation = 1;
}

int pipeline_graph(const ts_pipeline_spec& c, bool estimate, int tp, SynthOutput& out,
                   std::string& err) {
  out = SynthOutput{};
  PSpec ps;
  if (int rc = pspec_of(c, out.names, ps, err)) return rc;
  return graph_of_pspec(ps, estimate, tp, -1, out, err);
}

void synth_defaults(ts_synth_spec* s) {
  std::memset(s, 0, sizeof(*s));
  // SynthSpec::from_json defaults (synth.cpp:203-215) and SynthCosts (synth.hpp:17-34)
  s->n_layers = 4;
  s->d_model = 1024;
  s->d_ffn = 4096;
  s->n_heads = 16;
  s->d_head = 64;
  s->tp = 1;
  s->pp = 1;
  s->dp = 1;
  s->num_microbatches = 4;
  s->tokens_per_microbatch = 2048;
  s->vocab = 32768;
  s->launch_us = 5;
  s->record_us = 2;
  s->wait_us = 2;
  s->sync_us = 5;
  s->gemm_ref_us = 600;
  s->gemm_ref_mnk = int64_t{1} << 30;
  s->bwd_gemm_factor = 2.0;
  s->attn_misc_us = 300;
  s->embed_us = 150;
  s->head_us = 150;
  s->loss_grad_us = 150;
  s->optimizer_ref_us = 400;
  s->optimizer_ref_bytes = int64_t{1} << 24;
  s->alpha_us = 10.0;
  s->bytes_per_us = 50000.0;
  s->p2p_recv_base_us = 10;
  s->origin = 1000000;
  s->estimate = 0;
  s->slice_rank = -1;
}

int synth_graph(const ts_synth_spec& sp, SynthOutput& out, std::string& err) {
  if (sp.pp < 1 || sp.dp < 1 || sp.tp < 1 || sp.num_microbatches < 1 || sp.n_layers < 1 ||
      sp.d_model < 1 || sp.d_ffn < 1) {
    err = "synth spec: sizes must be positive";
    return TS_E_INVALID_ARGUMENT;
  }
  if (sp.n_layers % sp.pp != 0) {
    err = "layer count must divide evenly across pipeline stages";
    return TS_E_INVALID_ARGUMENT;
  }
  if (sp.num_microbatches < sp.pp) {
    err = "ParallelismConfig.num_microbatches must be >= pp";
    return TS_E_INVALID_ARGUMENT;
  }
  if (sp.bytes_per_us <= 0 || sp.gemm_ref_mnk <= 0 || sp.optimizer_ref_bytes <= 0) {
    err = "synth spec: cost reference points must be positive";
    return TS_E_INVALID_ARGUMENT;
  }
  out = SynthOutput{};
  const PSpec ps = pspec_for(sp, out.names);
  return graph_of_pspec(ps, sp.estimate != 0, sp.tp, sp.slice_rank, out, err,
                        sp.keep_meta != 0 && sp.estimate == 0);
}

// The generated trace of a PipelineSpec as the replay graph (build_graph +
// merge_ranks) or the estimate graph (generator dependencies + gates), with
// tp replicas of every rank; out.names must hold the spec's name ids.
int graph_of_pspec(const PSpec& ps, bool estimate, int tp, int slice_rank, SynthOutput& out,
                   std::string& err, bool keep_meta) {
  if (tp < 1) {
    err = "tp must be >= 1";
    return TS_E_INVALID_ARGUMENT;
  }
  Builder b(ps, out.names, keep_meta);
  try {
    b.run();
  } catch (const std::exception& e) {
    err = e.what();
    return TS_E_INVALID_ARGUMENT;
  }
  out.truth_makespan = b.end - ps.origin;

  // events in trace order: stable sort by (pid, ts, tid) (pipeline.cpp:75-78)
  const int64_t ne = static_cast<int64_t>(b.events.size());
  std::vector<int64_t> order(ne);
  for (int64_t i = 0; i < ne; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
    const Event& a = b.events[x].ev;
    const Event& c = b.events[y].ev;
    return std::tie(a.pid, a.ts, a.tid) < std::tie(c.pid, c.ts, c.tid);
  });
  const int n_ranks = ps.pp * ps.dp;
  std::vector<int64_t> rank_begin(n_ranks + 1, 0);
  for (const GenEvent& g : b.events) rank_begin[g.ev.pid + 1]++;
  for (int r = 0; r < n_ranks; ++r) rank_begin[r + 1] += rank_begin[r];
  std::vector<int32_t> local(ne);  // event -> position within its rank
  std::vector<std::vector<Event>> per_rank(n_ranks);
  std::vector<std::vector<MetaList>> per_rank_args(keep_meta ? n_ranks : 0);
  for (int64_t i : order) {
    const Event& e = b.events[i].ev;
    local[i] = static_cast<int32_t>(per_rank[e.pid].size());
    per_rank[e.pid].push_back(e);
    if (keep_meta) {
      const int32_t a = b.events[i].args;
      per_rank_args[e.pid].push_back(a >= 0 ? b.arg_lists[a] : MetaList{});
    }
  }

  // one graph per source rank
  std::vector<HostGraph> rank_graphs(n_ranks);
  BuildPolicyLite pol;
  for (int r = 0; r < n_ranks; ++r) {
    if (!estimate) {
      int rc = build_rank_graph(per_rank[r], out.names, r, pol, rank_graphs[r], err,
                                keep_meta ? &per_rank_args[r] : nullptr);
      if (rc != TS_OK) return rc;
      continue;
    }
    // estimate graph: same tasks, generator dependencies, intrinsic durations
    HostGraph& g = rank_graphs[r];
    const auto& evs = per_rank[r];
    const int32_t n = static_cast<int32_t>(evs.size());
    g.rank.assign(n, r);
    g.window_start = evs.empty() ? 0 : evs[0].ts;
    g.window_end = g.window_start;
    for (const Event& e : evs) {
      const bool gpu = e.cat == CAT_KERNEL;
      g.original_start.push_back(e.ts);
      g.lane_kind.push_back(gpu ? TS_LANE_CUDA_STREAM : TS_LANE_CPU_THREAD);
      g.lane.push_back(gpu ? e.stream : e.tid);
      g.op_class.push_back(classify_event(e, out.names));
      g.task_kind.push_back(gpu ? 1 : 0);
      g.name.push_back(e.name);
      g.op_index.push_back(e.op_index);
      g.window_start = std::min(g.window_start, e.ts);
      g.window_end = std::max(g.window_end, e.ts + e.dur);
    }
    g.duration.resize(n);
  }
  if (estimate) {
    for (int64_t i = 0; i < ne; ++i) {
      const GenEvent& ge = b.events[i];
      rank_graphs[ge.ev.pid].duration[local[i]] = ge.cost;
    }
  }

  // TP replicas in rank order r * tp + t (merge_ranks order)
  std::vector<int64_t> base(static_cast<size_t>(n_ranks) * tp + 1, 0);  // by new rank
  for (int r = 0; r < n_ranks; ++r)
    for (int t = 0; t < tp; ++t)
      base[static_cast<size_t>(r) * tp + t + 1] = rank_graphs[r].n();
  for (size_t k = 0; k + 1 < base.size(); ++k) base[k + 1] += base[k];
  if (base.back() >= INT32_MAX) {
    err = "graph too large for int32 task ids";
    return TS_E_INVALID_ARGUMENT;
  }
  HostGraph& G = out.graph;
  bool first = true;
  for (int r = 0; r < n_ranks; ++r)
    for (int t = 0; t < tp; ++t) {
      if (slice_rank >= 0 && r * tp + t != slice_rank) continue;
      G.append_relabelled(rank_graphs[r], r * tp + t, first);
      first = false;
    }
  if (estimate && slice_rank < 0) {
    // cross-rank dependencies of the generator, per replica
    auto gid = [&](int64_t ev, int t) {
      const int r = b.events[ev].ev.pid;
      return static_cast<int32_t>(base[static_cast<size_t>(r) * tp + t] + local[ev]);
    };
    std::vector<std::pair<int32_t, int32_t>> edges;
    edges.reserve(b.edges.size() * tp);
    for (int t = 0; t < tp; ++t) {
      for (const auto& [a, c] : b.edges) edges.emplace_back(gid(a, t), gid(c, t));
      for (const auto& [a, c, k] : b.gates) {
        G.gate_from.push_back(gid(a, t));
        G.gate_to.push_back(gid(c, t));
        G.gate_kind.push_back(k);
      }
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    G.edge_from.clear();
    G.edge_to.clear();
    for (const auto& e : edges) {
      G.edge_from.push_back(e.first);
      G.edge_to.push_back(e.second);
    }
  } else if (estimate) {
    err = "estimate graphs couple ranks; slice_rank is not supported";
    return TS_E_INVALID_ARGUMENT;
  }
  // retime metadata per task through its generator cost index
  {
    const int32_t n = G.n();
    G.rt_kind.assign(n, TS_RT_NONE);
    G.rt_bytes.assign(n, -1);
    G.rt_group.assign(n, 0);
    G.rt_mnk.assign(static_cast<size_t>(n) * 3, 0);
    for (int32_t t = 0; t < n; ++t) {
      const int64_t oi = G.op_index[t];
      if (G.task_kind[t] != 1 || oi < 0 || static_cast<size_t>(oi) >= b.kmeta.size()) continue;
      const KMeta& km = b.kmeta[oi];
      G.rt_kind[t] = km.kind;
      G.rt_bytes[t] = km.bytes;
      G.rt_group[t] = km.group;
      G.rt_mnk[3 * static_cast<size_t>(t)] = km.m;
      G.rt_mnk[3 * static_cast<size_t>(t) + 1] = km.n;
      G.rt_mnk[3 * static_cast<size_t>(t) + 2] = km.k;
    }
  }
  out.n_ops = b.events.empty() ? 0 : 0;
  int64_t max_idx = -1;
  for (const GenEvent& ge : b.events) max_idx = std::max(max_idx, ge.ev.op_index);
  out.n_ops = max_idx + 1;
  return TS_OK;
}

}  // namespace lumos
