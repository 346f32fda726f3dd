// replay.cu — sm_100a kernels of the batched Lumos replay.
//
//   K1 replay_walk  : every (component, 128-scenario chunk) is one CTA; each
//                     thread owns one scenario and walks the component's
//                     straight-line program (program.hpp).  Live finish times
//                     sit in shared memory (slot-major, [slot][thread], so
//                     every access is a conflict-free 8-byte-per-lane row).
//                     Durations are generated in registers (K4 fused), so the
//                     only HBM traffic is the start/finish rows written
//                     scenario-major (task row, 128 consecutive scenarios =
//                     1 KiB per CTA per row) with streaming stores.
//   K4 durations    : the same duration formula on its own (materialisation).
//   K5 rank_reduce  : per (rank, scenario) k-way merge of the rank's stream
//                     timelines -> 4-way breakdown (metrics.cpp:43-103) and
//                     per-stream busy time.
//
// Integer semantics are exact int64 (types.hpp:15); the double arithmetic of
// the jitter formula uses explicitly rounded intrinsics so it matches the
// host restatement (compiled with -ffp-contract=off) bit for bit.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <type_traits>
#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"
#include "lumos_b200.h"
#include "program.hpp"

namespace lumos {

namespace {

constexpr int kThreads = kWalkThreads;  // widest walk CTA; K4/K5 block size

__device__ __forceinline__ uint32_t lo16(uint32_t w) { return w & 0xFFFFu; }
__device__ __forceinline__ uint32_t hi16(uint32_t w) { return w >> 16; }

// ------------------------------------------------------------------- K1
// One thread replays kS adjacent scenarios (2 normally: columns c, c+1; 1 when
// a launch has too few (component, scenario) pairs to fill the GPU): the op
// record is decoded once per thread, each operand is one shared load of kS
// values, and each output row is written with one 8- or 16-byte streaming
// store per thread (256 / 512 contiguous bytes per warp).
// Shared memory: two program chunks (2 x kChunk x 64 B, refilled one chunk
// ahead through registers) followed by the slot table [n_slots][kT] x kS values.
//
// Value type V: int64 absolute times, or uint32 offsets from W when the
// launch proves every time of every component stays below W + 2^32 - 1 (the
// sum of the component's largest possible durations bounds any path; checked
// on the host, capi.cpp).  Offsets halve the slot table and turn the int64
// max/add chains into single 32-bit instructions; stores add W back.
template <typename V, int kS>
struct alignas(kS * sizeof(V)) VPack {
  V v[kS];
};
template <typename V>
__device__ __forceinline__ V vmax(V a, V b) { return a > b ? a : b; }
template <typename V>
__device__ __forceinline__ V vmin(V a, V b) { return a < b ? a : b; }
template <typename V, int kS>
__device__ __forceinline__ VPack<V, kS> maxp(VPack<V, kS> a, VPack<V, kS> b) {
  VPack<V, kS> r;
#pragma unroll
  for (int k = 0; k < kS; ++k) r.v[k] = vmax(a.v[k], b.v[k]);
  return r;
}
template <typename V, int kS>
__device__ __forceinline__ VPack<V, kS> splat(V x) {
  VPack<V, kS> r;
#pragma unroll
  for (int k = 0; k < kS; ++k) r.v[k] = x;
  return r;
}
constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// duration of a retimed allreduce / p2p send (v = its retimed byte count):
// the cost model of change_hidden, then scale_dp (rt_task's order).  Rare ops:
// kept out of line so the walk's registers stay those of the common path.
__device__ __noinline__ int64_t rt_coll_base(const RtScen* scp, int32_t rk, int32_t grp,
                                             int32_t source_dp, int64_t v, int64_t base) {
  const RtScen sc = *scp;
  int64_t d = base;
  // v < 0: an allreduce without a byte count, which change_hidden leaves as is
  // (transform.cpp:313; scale_dp rejects it on the host)
  if ((sc.flags & kRtHid) && v >= 0)
    d = coll_cost(rk == TS_RT_ALLREDUCE, v, rk == TS_RT_ALLREDUCE ? grp : 2, sc.alpha, sc.bpu);
  if ((sc.flags & kRtDp) && rk == TS_RT_ALLREDUCE && grp == source_dp)
    d = coll_cost(true, v, sc.tdp, sc.alpha, sc.bpu);
  return d;
}

// mailbox words: the value is the whole message (one aligned 64-bit word),
// so relaxed device-scope accesses suffice (no system-scope volatile)
#ifndef LUMOS_MAIL_SLEEP
#define LUMOS_MAIL_SLEEP 32
#endif
__device__ __forceinline__ uint64_t mail_load(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mail_store(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int kT, int kMode, bool kWriteStart, bool kWriteFin, typename V, int kS,
          bool kCl = false, bool kClCheck = true>
__device__ __forceinline__ void replay_walk_body(const WalkParams& P) {
  using VP = VPack<V, kS>;
  constexpr bool kRel = sizeof(V) == 4;
  static_assert(!kCl || (kRel && kS == 2), "cluster walks keep uint32 pairs");
  // retime walk: F_RT tasks take their base duration from the variant tables
  // (K4v) and the scenario's cost model; scale / jitter follow sp.mode
  constexpr bool kRt = kMode >= 0 && (kMode & kModeRetime) != 0;
  constexpr int kDurMode = kRt ? (kMode & (kModeScale | kModeJitter)) : kMode;
  constexpr int kRecPerThread = (kChunk + kT - 1) / kT;  // chunk refill: records per thread
  // record slot fields hold s * 128; a slot is kT packs of kS * sizeof(V) bytes
  constexpr int kShift = ilog2(kT) - 7 + ilog2(kS * static_cast<int>(sizeof(V)));
  constexpr V kInfV = kRel ? static_cast<V>(0xFFFFFFFFu) : static_cast<V>(kMaxI64);
  constexpr uint32_t kFastMask =
      0xFFu | (static_cast<uint32_t>(F_TRACK | F_STORE_START | (kRt ? F_RT : 0)) << 24);
  static_assert(kT >= 32 && kShift >= 0, "");
  static_assert(kS == 1 || kS == 2, "");
  extern __shared__ int4 smem[];
  // [2][kChunk][4]: the raw 32-byte record, then its eight 16-bit slot fields
  // (pred[4], dst, x0, x1, x2) widened to byte offsets by the loader, so the
  // walk adds one register per operand address
  int4* opbuf = smem;
  // [kMaxClasses][kT] class-scale numerators of the thread's two scenarios
  // (shared memory instead of 8 registers), then the slot table
  int2* numtab = reinterpret_cast<int2*>(smem + 8 * kChunk);
  char* slot_base = reinterpret_cast<char*>(numtab + kMaxClasses * kT) +
                    threadIdx.x * static_cast<uint32_t>(sizeof(VP));
  const int tid = threadIdx.x;
  // a cluster walk CTA is (component, chunk, rank program r_loc); the
  // component's rank CTAs form one cluster, so they are co-scheduled
  const int unit = kCl ? static_cast<int>(blockIdx.x / static_cast<unsigned>(P.cl_size))
                       : static_cast<int>(blockIdx.x);
  const int r_loc = kCl ? static_cast<int>(blockIdx.x % static_cast<unsigned>(P.cl_size)) : 0;
  const int comp = static_cast<int>(unit % static_cast<unsigned>(P.n_comps));
  const int chunk = static_cast<int>(unit / static_cast<unsigned>(P.n_comps));
  // lanes past the last scenario replay the last scenario again: identical
  // values, so their (duplicate) stores and atomics need no predication
  const int last = P.sp.count - 1;
  int col[kS];
  if (kS == 2) {
    int c0 = chunk * kT * 2 + 2 * tid;
    if (c0 > last - 1)  // keep pairs even-aligned when the count is even
      c0 = P.sp.count < 2 ? 0 : ((P.sp.count & 1) ? min(c0, last) : last - 1);
    col[0] = c0;
    col[kS - 1] = min(c0 + 1, last);
  } else {
    col[0] = min(chunk * kT + tid, last);
  }
  const bool vec_store = kS == 2 && P.vec_store;  // ld even, count even, aligned buffers

  const int comp_id = P.comp_order ? P.comp_order[comp] : comp;
  const ComponentDesc cd = P.comps[comp_id];
  int prog_id = cd.program;
  if constexpr (kCl) {
    const int pf = P.cl_prog_off[comp_id], nw = P.cl_prog_off[comp_id + 1] - pf;
    if (r_loc >= nw) return;  // a narrower component: no barrier is shared across CTAs
    prog_id = P.cl_progs[pf + r_loc];
  }
  const ProgramDesc pd = P.progs[prog_id];
  const int4* __restrict__ gops = reinterpret_cast<const int4*>(P.ops + pd.op_offset);
  const int n_ops = pd.n_ops;
  const int64_t W = P.window_start;
  // uint32 values are offsets from O = W rounded down to a multiple of 2^32
  // (the host proves W - O + every time < 2^32), so an absolute time is the
  // offset with O's high word attached: no 64-bit add per stored value
  const uint32_t o_hi = static_cast<uint32_t>(static_cast<uint64_t>(W) >> 32);
  const V w0 = kRel ? static_cast<V>(static_cast<uint32_t>(W)) : static_cast<V>(W);  // W in V
  auto absv = [&](V v) -> int64_t {
    return kRel ? static_cast<int64_t>((static_cast<uint64_t>(o_hi) << 32) |
                                       static_cast<uint32_t>(v))
                : static_cast<int64_t>(v);
  };
#ifdef LUMOS_DEBUG_BOUNDS
  // every slot offset must address one of the program's slots
  const uint32_t slot_limit = static_cast<uint32_t>(pd.n_slots < kFirstSlot ? kFirstSlot : pd.n_slots) *
                              kT * static_cast<uint32_t>(sizeof(VP));
  auto slot_chk = [&](uint32_t boff) -> uint32_t {
    return LUMOS_OK(boff < slot_limit && boff % (kT * sizeof(VP)) == 0) ? boff : 0u;
  };
#define SLOT2(off) \
  (*reinterpret_cast<VP*>(slot_base + slot_chk(static_cast<uint32_t>(off) << kShift)))
#define SLOTB(boff) \
  (*static_cast<VP*>(__builtin_assume_aligned(slot_base + slot_chk(static_cast<uint32_t>(boff)), sizeof(VP))))
#else
#define SLOT2(off) \
  (*reinterpret_cast<VP*>(slot_base + (static_cast<uint32_t>(off) << kShift)))
#define SLOTB(boff) \
  (*static_cast<VP*>(__builtin_assume_aligned(slot_base + static_cast<uint32_t>(boff), sizeof(VP))))
#endif
  SLOT2(slot_off(kSlotOrigin)) = splat<V, kS>(w0);
  SLOT2(slot_off(kSlotInf)) = splat<V, kS>(kInfV);

  ThreadScen ts[kS];
#pragma unroll
  for (int k = 0; k < kS; ++k) init_thread_scen(P.sp, col[k], ts[k]);
  constexpr bool kScaleTab = kS == 2 && kDurMode >= 0 && (kDurMode & kModeScale) != 0;
  if constexpr (kScaleTab) {
#pragma unroll
    for (int c = 0; c < kMaxClasses; ++c) numtab[c * kT + tid] = make_int2(ts[0].num[c], ts[1].num[c]);
  }
  int64_t rt_vrow[kS];  // the scenario's row of the variant table
#pragma unroll
  for (int k = 0; k < kS; ++k)
    rt_vrow[k] = kRt ? static_cast<int64_t>(__ldg(P.rt.var + col[k])) * P.rt.n_rec : 0;

  int64_t hi[kS];
  bool fail[kS];
#pragma unroll
  for (int k = 0; k < kS; ++k) {
    hi[k] = kMinI64;
    fail[k] = false;
  }
  int64_t* const start_c0 = P.out_start + col[0];
  int64_t* const fin_c0 = P.out_fin + col[0];
  const uint32_t ld = static_cast<uint32_t>(P.ld);
  const int64_t dcol = col[kS - 1] - col[0];
  char* const sbase = reinterpret_cast<char*>(start_c0);
  char* const fbase = reinterpret_cast<char*>(fin_c0);
  const uint64_t ld8 = static_cast<uint64_t>(ld) * 8u;
  // split accounting of a fused component (program.hpp FusedDesc): |A| summed
  // in registers over the F_BUSY kernels
  int acct_row = P.fused ? P.fused[comp_id].row : -1;
  if constexpr (kCl) acct_row = P.cl_rows ? P.cl_rows[P.cl_prog_off[comp_id] + r_loc] : -1;
  uint64_t* const mail_base =
      kCl ? P.cl_mail + static_cast<int64_t>(unit) * P.cl_n_mail * kT + tid : nullptr;
  bool stalled = false;
  VP busy_a = splat<V, kS>(V(0));

  // A task's finish: its scenario durations (K4, fused), the busy / sink
  // bookkeeping and the start / finish row stores.  rec = the op's record index
  // in the program (retime walks look up their F_RT table through it).
  auto finish_task = [&](const VP& st, const VP& fb, const int4& ra, uint32_t cls_b,
                         uint32_t flags, int64_t rec) -> VP {
    const int64_t task = static_cast<int64_t>(cd.node_base) + ra.z;
    const int64_t base = (static_cast<int64_t>(static_cast<uint32_t>(ra.y)) << 32) |
                         static_cast<uint32_t>(ra.x);
    const int cls = cls_b & 15u;
    int64_t bs[kS];  // retime walk: per-scenario base durations
#pragma unroll
    for (int s = 0; s < kS; ++s) bs[s] = base;
    if constexpr (kRt) if (flags & F_RT) {
      const int64_t j = __ldg(P.rt.rec_of + rec);
      const int4 rw = __ldg(reinterpret_cast<const int4*>(P.rt.rec + j));
      const int32_t rk = rw.w, grp = rw.z;
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        const int64_t v = __ldg(P.rt.vval + rt_vrow[s] + j);
        bs[s] = (rk == TS_RT_GEMM || rk == TS_RT_OPT)
                    ? v  // retimed base (change_hidden), or the base itself
                    : rt_coll_base(P.rt.scen + col[s], rk, grp, P.rt.source_dp, v, base);
      }
    }
    VP fin;
    constexpr bool kJit = kDurMode >= 0 && (kDurMode & kModeJitter) != 0;
    int64_t dsc[kS];  // class-scaled durations (kScaleTab)
    if constexpr (kScaleTab) {
      const int2 nm = numtab[cls * kT + tid];
      dsc[0] = class_scaled_num(P.sp, kRt ? bs[0] : base, nm.x);
      dsc[1] = class_scaled_num(P.sp, kRt ? bs[1] : base, nm.y);
    }
    if constexpr (kS == 2 && kJit) {
      // one Philox call for the thread's scenario pair (columns c0, c0 + 1
      // with c0 even, or a duplicated last column; the launch takes the
      // one-scenario walk when the batch starts at an odd global id); the
      // rounding is branch-free per scenario (a zero duration selects 0)
      if constexpr (!kScaleTab) {
#pragma unroll
        for (int s = 0; s < kS; ++s) dsc[s] = kRt ? bs[s] : base;
      }
      uint32_t w[kS] = {0u, 0u};
      if (kRt || (kDurMode & kModeScale) || base != 0)
        jitter_words2(P.sp, task, ts[0].scen, ts[1].scen, w[0], w[1]);
      if constexpr (kRel) {
#pragma unroll
        for (int s = 0; s < kS; ++s)
          fin.v[s] = static_cast<V>(
              fb.v[s] + jitter_apply_u32(P.sp, __ll2double_rn(dsc[s]), dsc[s] == 0, w[s]));
      } else {
#pragma unroll
        for (int s = 0; s < kS; ++s)
          fin.v[s] = static_cast<V>(fb.v[s] + static_cast<V>(jitter_apply(P.sp, dsc[s], w[s])));
      }
    } else if constexpr (kScaleTab) {  // class scale only
#pragma unroll
      for (int s = 0; s < kS; ++s) fin.v[s] = static_cast<V>(fb.v[s] + static_cast<V>(dsc[s]));
    } else {
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        const int64_t d = scenario_duration<kDurMode>(P.sp, ts[s], task, kRt ? bs[s] : base, cls);
        fin.v[s] = static_cast<V>(fb.v[s] + static_cast<V>(d));
      }
    }
#ifndef LUMOS_NO_BUSY  // perf experiments only: breaks split accounting
    if (flags & F_BUSY)
#else
    if (false)
#endif
    {
#pragma unroll
      for (int s = 0; s < kS; ++s) busy_a.v[s] = static_cast<V>(busy_a.v[s] + (fin.v[s] - st.v[s]));
    }
    if (__builtin_expect((flags & F_SINK) != 0, 0)) {
#pragma unroll
      for (int s = 0; s < kS; ++s) hi[s] = imax(hi[s], absv(fin.v[s]));
    }
    const uint64_t at = static_cast<uint64_t>(static_cast<uint32_t>(task)) * ld;
    if (!LUMOS_OK(task >= 0 && task < P.n_tasks && col[kS - 1] < static_cast<int>(ld) &&
                  col[0] >= 0))
      return fin;  // debug builds: an out-of-range row is not written
    if (vec_store) {
      const uint64_t at8 = static_cast<uint64_t>(static_cast<uint32_t>(task)) * ld8;
      if (kWriteStart)
        __stcs(reinterpret_cast<longlong2*>(sbase + at8),
               make_longlong2(absv(st.v[0]), absv(st.v[kS - 1])));
      if (kWriteFin)
        __stcs(reinterpret_cast<longlong2*>(fbase + at8),
               make_longlong2(absv(fin.v[0]), absv(fin.v[kS - 1])));
    } else {
      if (kWriteStart) {
        __stcs(start_c0 + at, absv(st.v[0]));
        if (kS == 2) __stcs(start_c0 + at + dcol, absv(st.v[kS - 1]));
      }
      if (kWriteFin) {
        __stcs(fin_c0 + at, absv(fin.v[0]));
        if (kS == 2) __stcs(fin_c0 + at + dcol, absv(fin.v[kS - 1]));
      }
    }
    if constexpr (kCl && kClCheck) {
      // the cluster walk's uint32 window is sized by the nominal path (like
      // the cooperative walk): a wrapped addition sends the scenario to the
      // int64 re-run (elided when the host proves the window: cl_check = 0)
#pragma unroll
      for (int s = 0; s < kS; ++s)
        fail[s] = fail[s] || fin.v[s] < fb.v[s] || fin.v[s] == static_cast<V>(0xFFFFFFFFu);
    }
    return fin;
  };
  auto stage = [&](int4* dstbuf, int r, int4 a, int4 b) {
    dstbuf[4 * r] = a;
    dstbuf[4 * r + 1] = b;
    const uint32_t x = b.x, y = b.y, z = b.z, w = b.w;
    dstbuf[4 * r + 2] = make_int4(lo16(x) << kShift, hi16(x) << kShift, lo16(y) << kShift,
                                  hi16(y) << kShift);
    dstbuf[4 * r + 3] = make_int4(lo16(z) << kShift, hi16(z) << kShift, lo16(w) << kShift,
                                  hi16(w) << kShift);
  };
#pragma unroll
  for (int q = 0; q < kRecPerThread; ++q) {
    const int r = q * kT + tid;
    if (r < kChunk && r < n_ops) stage(opbuf, r, __ldg(gops + 2 * r), __ldg(gops + 2 * r + 1));
  }
  __syncthreads();
  const int n_chunks = (n_ops + kChunk - 1) / kChunk;
  for (int c = 0; c < n_chunks; ++c) {
    // prefetch the next chunk into registers while this one is walked
    int4 na[kRecPerThread], nb[kRecPerThread];
#pragma unroll
    for (int q = 0; q < kRecPerThread; ++q) {
      const int nxt = (c + 1) * kChunk + q * kT + tid;
      if (q * kT + tid < kChunk && nxt < n_ops) {
        na[q] = __ldg(gops + 2 * nxt);
        nb[q] = __ldg(gops + 2 * nxt + 1);
      }
    }
    const int4* buf = opbuf + (c & 1) * 4 * kChunk;
    const int cnt = min(kChunk, n_ops - c * kChunk);
    for (int i = 0; i < cnt; ++i) {
      const int4 ra = buf[4 * i];
      const int4 oa = buf[4 * i + 2], ob = buf[4 * i + 3];
      const uint32_t hdr = static_cast<uint32_t>(ra.w);
      // fast path: a plain node (start = max(W, preds), no coverage, no stored
      // start, no retime lookup) — every compute kernel and launch of a replay
      // graph — without the kind dispatch
      if ((hdr & kFastMask) == OP_NODE) {
        const VP q0 = SLOTB(oa.x), q1 = SLOTB(oa.y), q2 = SLOTB(oa.z), q3 = SLOTB(oa.w);
        const VP st = maxp(maxp(q0, q1), maxp(q2, q3));
        SLOTB(ob.x) = finish_task(st, st, ra, (hdr >> 16) & 0xFFu, hdr >> 24,
                                  pd.op_offset + c * kChunk + i);
        if (hdr & (static_cast<uint32_t>(F_TRACK1) << 24)) {
          // compact coverage (every kernel on a stream a sync watches): the
          // source slot outlives this op's results (compile.cpp)
          const VP cov_src = SLOTB(ob.y);
          VP cv;
#pragma unroll
          for (int s = 0; s < kS; ++s)
            cv.v[s] = q0.v[s] >= st.v[s] ? vmin(st.v[s], cov_src.v[s]) : st.v[s];
          SLOTB(ob.z) = cv;
        }
        continue;
      }
      const int4 rb = buf[4 * i + 1];
      const uint32_t kind = hdr & 0xFFu;
      const uint32_t cls_b = (hdr >> 16) & 0xFFu;
      const uint32_t flags = hdr >> 24;
      const uint32_t w2 = static_cast<uint32_t>(rb.z);
      // every operand is read before any result is written (results may
      // reuse the slot of an operand that dies at this op)
      const VP p0 = SLOTB(oa.x), p1 = SLOTB(oa.y);
      const VP p2 = SLOTB(oa.z), p3 = SLOTB(oa.w);
      const uint32_t dst = ob.x;
      // st = the task's start; fb = what its finish adds the duration to
      // (max(start, gate) for gated kinds, else the start itself: st >= W)
      VP st, fb;
      if (kind <= OP_ACC) {  // OP_NODE, OP_SYNC, OP_START, OP_ACC
        st = maxp(maxp(p0, p1), maxp(p2, p3));  // unused preds read the origin W
        fb = st;
      } else if (kind == OP_FINISH) {
        st = p0;
        fb = maxp(maxp(p0, p1), maxp(p2, p3));
      } else if (kind == OP_GATED) {
        const int nfixed = static_cast<int>(cls_b >> 4);
        st = splat<V, kS>(w0);
        VP gate = st;
        if (nfixed > 0) st = maxp(st, p0); else gate = maxp(gate, p0);
        if (nfixed > 1) st = maxp(st, p1); else gate = maxp(gate, p1);
        if (nfixed > 2) st = maxp(st, p2); else gate = maxp(gate, p2);
        gate = maxp(gate, p3);
        fb = maxp(st, gate);
      } else if (kCl && (kind == OP_POST || kind == OP_WAIT)) {
        if constexpr (kCl) {
          int m = static_cast<int>(ob.z >> kShift);  // x1: the mailbox id (widened)
          if (!LUMOS_OK(m < P.cl_n_mail)) m = 0;
          uint64_t* box = mail_base + static_cast<int64_t>(m) * kT;
          if (kind == OP_POST) {
            uint64_t v = static_cast<uint64_t>(p0.v[0]) | (static_cast<uint64_t>(p0.v[1]) << 32);
            if (v == ~0ull) v = ~1ull;  // only a wrapped (failed) value can look unposted
            mail_store(box, v);
          } else {
            uint64_t v = mail_load(box);
            for (int spins = 0; v == ~0ull; ++spins) {
              if (spins > (1 << 22)) {  // ~seconds: a compiler bug, not a schedule
                stalled = true;
                v = 0;
                break;
              }
              if (LUMOS_MAIL_SLEEP > 0) __nanosleep(LUMOS_MAIL_SLEEP);
              v = mail_load(box);
            }
            VP q;
            q.v[0] = static_cast<V>(static_cast<uint32_t>(v));
            q.v[1] = static_cast<V>(static_cast<uint32_t>(v >> 32));
            SLOTB(ob.x) = q;
          }
        }
        continue;
      } else {
        continue;  // OP_NOP
      }
      if (kind == OP_ACC) {
        SLOTB(dst) = st;
        continue;
      }
      if (kind == OP_SYNC) {
        // static binding S = max(r_s, finish(k*_w)) and its certificate
        const VP rs = st;
        VP S = rs;
        const int n_ext = static_cast<int>(hi16(w2));
        for (int e = 0; e < n_ext; ++e) {
          const int4 xa = buf[4 * (i + 1 + e)];
          const int n = buf[4 * (i + 1 + e) + 1].z & 0xFFFF;
          const uint32_t f[4] = {lo16(xa.x), hi16(xa.x), lo16(xa.y), hi16(xa.y)};
#pragma unroll
          for (int k = 0; k < kCertPerExt; ++k)
            if (k < n && f[k] != kNoSlot) S = maxp(S, SLOT2(f[k]));
        }
        bool cov[kS];
#pragma unroll
        for (int s = 0; s < kS; ++s) cov[s] = S.v[s] == rs.v[s];
        for (int e = 0; e < n_ext; ++e) {
          const int4 xa = buf[4 * (i + 1 + e)], xb = buf[4 * (i + 1 + e) + 1];
          const int n = xb.z & 0xFFFF;
          const uint32_t f[4] = {lo16(xa.x), hi16(xa.x), lo16(xa.y), hi16(xa.y)};
          const uint32_t cv[4] = {lo16(xa.z), hi16(xa.z), lo16(xa.w), hi16(xa.w)};
          const uint32_t nx[4] = {lo16(xb.x), hi16(xb.x), lo16(xb.y), hi16(xb.y)};
#pragma unroll
          for (int k = 0; k < kCertPerExt; ++k) {
            if (k >= n) continue;
            if (f[k] != kNoSlot && cv[k] != kNoSlot) {
              const VP fk = SLOT2(f[k]), ck = SLOT2(cv[k]);
#pragma unroll
              for (int s = 0; s < kS; ++s)
                cov[s] = cov[s] || (fk.v[s] == S.v[s] && ck.v[s] <= rs.v[s]);
            }
            if (nx[k] != kNoSlot) {
              const VP nk = SLOT2(nx[k]);
#pragma unroll
              for (int s = 0; s < kS; ++s) fail[s] = fail[s] || nk.v[s] <= S.v[s];
            }
          }
        }
#pragma unroll
        for (int s = 0; s < kS; ++s) fail[s] = fail[s] || !cov[s];
        st = S;
        fb = S;
        i += n_ext;
      }
      if (kind == OP_START) {
        SLOTB(dst) = st;
      } else {
        const VP fin = finish_task(st, fb, ra, cls_b, flags, pd.op_offset + c * kChunk + i);
        SLOTB(dst) = fin;
        if (flags & F_STORE_START) SLOTB(ob.w) = st;
      }
      if (flags & F_TRACK1) {
        // the source slot outlives this op's results (compile.cpp), so it is
        // read here; kSlotInf when the kernel has no coverage source
        const VP cov_src = SLOTB(ob.y);
        VP cv;
#pragma unroll
        for (int s = 0; s < kS; ++s)
          cv.v[s] = p0.v[s] >= st.v[s] ? vmin(st.v[s], cov_src.v[s]) : st.v[s];
        SLOTB(ob.z) = cv;
      } else if (flags & F_TRACK) {
        // coverage of this kernel per watched set (program.hpp, OpCov)
        const int4 xa = buf[4 * (i + 1)], xb = buf[4 * (i + 1) + 1];
        const uint32_t src[2][4] = {{lo16(xa.x), hi16(xa.x), lo16(xa.y), hi16(xa.y)},
                                    {lo16(xa.z), hi16(xa.z), lo16(xa.w), hi16(xa.w)}};
        const uint32_t cdst[2] = {lo16(xb.x), hi16(xb.x)};
        const int n_sets = xb.y & 0xFFFF;
        const VP pv[4] = {p0, p1, p2, p3};
        VP cvj[kCovSets];
#pragma unroll
        for (int j = 0; j < kCovSets; ++j) {
          cvj[j] = st;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (j < n_sets && src[j][k] != kNoSlot) {
              const VP sv = SLOT2(src[j][k]);
#pragma unroll
              for (int s = 0; s < kS; ++s)
                if (pv[k].v[s] >= st.v[s]) cvj[j].v[s] = vmin(cvj[j].v[s], sv.v[s]);
            }
        }
#pragma unroll
        for (int j = 0; j < kCovSets; ++j)
          if (j < n_sets) SLOT2(cdst[j]) = cvj[j];
        i += 1;
      }
    }
    int4* nbuf = opbuf + ((c + 1) & 1) * 4 * kChunk;
#pragma unroll
    for (int q = 0; q < kRecPerThread; ++q) {
      const int r = q * kT + tid;
      if (r < kChunk && (c + 1) * kChunk + r < n_ops) stage(nbuf, r, na[q], nb[q]);
    }
    __syncthreads();
  }
  if (acct_row >= 0) {
#pragma unroll
    for (int s = 0; s < kS; ++s)
      P.acct_a[static_cast<int64_t>(col[s]) * P.n_ranks + acct_row] =
          kRel ? static_cast<int64_t>(static_cast<uint32_t>(busy_a.v[s]))
               : static_cast<int64_t>(busy_a.v[s]);
  }
#undef SLOT2
#undef SLOTB
#pragma unroll
  for (int s = 0; s < kS; ++s) {
    if (hi[s] != kMinI64) {
      atomicMin(reinterpret_cast<long long*>(P.span_lo) + col[s], static_cast<long long>(W));
      atomicMax(reinterpret_cast<long long*>(P.span_hi) + col[s], static_cast<long long>(hi[s]));
    }
    if (kCl && stalled) atomicExch(P.status + col[s], -2);
    else if (fail[s]) atomicOr(P.status + col[s], 1);
  }
}

// LUMOS_WALK_MINB > 0 caps uint32 walks at 64 registers (8 CTAs of 128 threads
// per SM); measured slower than the unconstrained 71-register code (30.4 vs
// 33.5 ms per config-5 tile of 2,048 scenarios), so it is off by default
#ifndef LUMOS_WALK_MINB
#define LUMOS_WALK_MINB 0
#endif
template <int kT, int kMode, bool kWriteStart, bool kWriteFin, typename V, int kS>
__global__ void __launch_bounds__(kT, sizeof(V) == 4 && LUMOS_WALK_MINB > 0 ? LUMOS_WALK_MINB * 128 / kT : 1)
    replay_walk_kernel(WalkParams P) {
  replay_walk_body<kT, kMode, kWriteStart, kWriteFin, V, kS>(P);
}
// K1x cluster walk (estimate-mode components): 128 threads, uint32 pairs
#ifndef LUMOS_CLUSTER_MINB
#define LUMOS_CLUSTER_MINB 1
#endif
#ifndef LUMOS_CLUSTER_CARVEOUT_DEFAULT
#define LUMOS_CLUSTER_CARVEOUT_DEFAULT -1
#endif
template <int kMode, bool kWriteStart, bool kWriteFin, bool kCheck>
__global__ void __launch_bounds__(128, LUMOS_CLUSTER_MINB) cluster_walk_kernel(WalkParams P) {
  replay_walk_body<128, kMode, kWriteStart, kWriteFin, uint32_t, 2, true, kCheck>(P);
}
// retime walks: at least 6 CTAs of 128 threads per SM (<= 80 registers)
template <int kT, int kMode, bool kWriteStart, bool kWriteFin, typename V, int kS>
__global__ void __launch_bounds__(kT, 6 * 128 / kT) replay_walk_rt_kernel(WalkParams P) {
  replay_walk_body<kT, kMode, kWriteStart, kWriteFin, V, kS>(P);
}

// ------------------------------------------------------------------- K1c
// Cooperative walk: a CTA replays one component for 32 scenarios (lane =
// scenario) with one warp per rank program; the programs are the component's
// op order restricted to each rank, so a warp only ever waits for values
// another warp produces earlier in that order (no cycles).  Records are read
// straight from global memory (one-record lookahead), slots live in the warp's
// own [slot][32] table, cross-rank values in [mailbox][32] with a ready flag.
// A wait that spins ~1 s marks the scenario failed (status -2) rather than
// hang; it cannot happen for a correctly compiled component.
// kMaxW: warps per CTA the instantiation allows; components of <= 16 ranks
// take the 512-thread variant, whose register cap fits LUMOS_COOP_MINB CTAs
// per SM (3 was measured: 40 registers with spills, 7.2 vs 5.0 ms on config 3)
#ifndef LUMOS_COOP_MINB
#define LUMOS_COOP_MINB 2
#endif
template <int kMode, typename V, int kMaxW>
__global__ void __launch_bounds__(32 * kMaxW, kMaxW <= 16 ? LUMOS_COOP_MINB : 1)
    coop_walk_kernel(WalkParams P, CoopParams C) {
  constexpr bool kRel = sizeof(V) == 4;
  constexpr int kShiftC = kRel ? 0 : 1;  // record field s*128 -> s*32*sizeof(V)
  constexpr V kInfV = kRel ? static_cast<V>(0xFFFFFFFFu) : static_cast<V>(kMaxI64);
  extern __shared__ int4 smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int comp_i = static_cast<int>(blockIdx.x % static_cast<unsigned>(P.n_comps));
  const int chunk = static_cast<int>(blockIdx.x / static_cast<unsigned>(P.n_comps));
  const int comp = P.comp_order[comp_i];
  int* flags = reinterpret_cast<int*>(smem);
  V* mail = reinterpret_cast<V*>(reinterpret_cast<char*>(smem) + ((C.n_mail * 4 + 15) / 16) * 16);
  char* slots = reinterpret_cast<char*>(mail + static_cast<size_t>(C.n_mail) * 32);
  for (int i = threadIdx.x; i < C.n_mail; i += blockDim.x) flags[i] = 0;
  if (C.fixup) {  // int64 re-run of chunks where a uint32 addition wrapped
    const int c = min(chunk * 32 + lane, P.sp.count - 1);
    if (!__syncthreads_or((P.status[c] & 1) != 0)) return;
  }
  __syncthreads();
  const int pfirst = C.prog_off[comp], nw = C.prog_off[comp + 1] - pfirst;
  if (w >= nw) return;  // no block-wide barrier after this point
  char* slot_base = slots + static_cast<size_t>(w) * C.n_slots * 32 * sizeof(V) + lane * sizeof(V);
#ifdef LUMOS_DEBUG_BOUNDS
  const uint32_t slotc_limit = static_cast<uint32_t>(C.n_slots) * 32u * sizeof(V);
  auto slotc_chk = [&](uint32_t field) -> uint32_t {
    const uint32_t b = field << kShiftC;
    return LUMOS_OK(b < slotc_limit) ? b : 0u;
  };
#define SLOTC(field) (*reinterpret_cast<V*>(slot_base + slotc_chk(static_cast<uint32_t>(field))))
#else
#define SLOTC(field) \
  (*reinterpret_cast<V*>(slot_base + (static_cast<uint32_t>(field) << kShiftC)))
#endif
  const ComponentDesc cd = P.comps[comp];
  const ProgramDesc pd = P.progs[C.progs[pfirst + w]];
  const int4* __restrict__ gops = reinterpret_cast<const int4*>(P.ops + pd.op_offset);
  const int n_ops = pd.n_ops;
  const int last = P.sp.count - 1;
  const int col = min(chunk * 32 + lane, last);
  const int64_t W = P.window_start;
  const V w0 = kRel ? V(0) : static_cast<V>(W);
  auto absv = [&](V v) -> int64_t { return kRel ? W + static_cast<int64_t>(v) : static_cast<int64_t>(v); };
  SLOTC(slot_off(kSlotOrigin)) = w0;
  SLOTC(slot_off(kSlotInf)) = kInfV;
  ThreadScen ts;
  init_thread_scen(P.sp, col, ts);
  int64_t hi = kMinI64;
  bool fail = false, stalled = false;
  const int acct_row = C.rows ? C.rows[pfirst + w] : -1;  // split accounting of this rank
  V busy_a = V(0);
  constexpr uint32_t kCoopFastMask = 0xFFu | (static_cast<uint32_t>(F_TRACK | F_STORE_START) << 24);
  auto coop_duration = [&](int64_t task, int64_t base, int cls) -> int64_t {
    return scenario_duration<kMode>(P.sp, ts, task, base, cls);
  };
  int64_t* const start_c = P.out_start + col;
  int64_t* const fin_c = P.out_fin + col;
  const uint64_t ld = static_cast<uint64_t>(P.ld);
  int4 ra = n_ops > 0 ? __ldg(gops) : int4{}, rb = n_ops > 0 ? __ldg(gops + 1) : int4{};
  for (int i = 0; i < n_ops && !stalled; ++i) {
    const int4 ca = ra, cb = rb;
    if (i + 1 < n_ops) {  // lookahead
      ra = __ldg(gops + 2 * (i + 1));
      rb = __ldg(gops + 2 * (i + 1) + 1);
    }
    const uint32_t hdr = static_cast<uint32_t>(ca.w);
    const uint32_t kind = hdr & 0xFFu, cls_b = (hdr >> 16) & 0xFFu, flags_op = hdr >> 24;
    const uint32_t w0f = cb.x, w1f = cb.y, w2f = cb.z, w3f = cb.w;
    // fast path: a plain node (no coverage, no stored start) — most ops of a
    // rank program — without the kind dispatch
    if ((hdr & kCoopFastMask) == OP_NODE) {
      const V q0 = SLOTC(lo16(w0f)), q1 = SLOTC(hi16(w0f));
      const V q2 = SLOTC(lo16(w1f)), q3 = SLOTC(hi16(w1f));
      const V st = vmax(vmax(q0, q1), vmax(q2, q3));
      const int64_t task = static_cast<int64_t>(cd.node_base) + ca.z;
      const int64_t base = (static_cast<int64_t>(static_cast<uint32_t>(ca.y)) << 32) |
                           static_cast<uint32_t>(ca.x);
      const int64_t d = coop_duration(task, base, static_cast<int>(cls_b & 15u));
      const V fin = static_cast<V>(st + static_cast<V>(d));
      if (kRel && (fin < st || d > 0xFFFFFFFFll)) fail = true;
      SLOTC(lo16(w2f)) = fin;
      if (flags_op & F_BUSY) busy_a = static_cast<V>(busy_a + (fin - st));
      if (flags_op & F_SINK) hi = imax(hi, absv(fin));
      const uint64_t at = static_cast<uint64_t>(static_cast<uint32_t>(task)) * ld;
      if (LUMOS_OK(task >= 0 && task < P.n_tasks && col < static_cast<int>(ld))) {
        if (P.out_start) __stcs(start_c + at, absv(st));
        if (P.out_fin) __stcs(fin_c + at, absv(fin));
      }
      if (flags_op & F_TRACK1) {
        const V cs = SLOTC(hi16(w2f));
        SLOTC(lo16(w3f)) = q0 >= st ? vmin(st, cs) : st;
      }
      continue;
    }
    if (kind == OP_NOP) continue;
    const V p0 = SLOTC(lo16(w0f)), p1 = SLOTC(hi16(w0f));
    const V p2 = SLOTC(lo16(w1f)), p3 = SLOTC(hi16(w1f));
    if (kind == OP_POST || kind == OP_WAIT) {
      int m = static_cast<int>(lo16(w3f));  // x1: mailbox id
      if (!LUMOS_OK(m < C.n_mail)) m = 0;
      volatile V* box = mail + static_cast<size_t>(m) * 32 + lane;
      if (kind == OP_POST) {
        *box = p0;
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          atomicExch(flags + m, 1);
        }
      } else {
        if (lane == 0) {
          int spins = 0;
          while (atomicAdd(flags + m, 0) == 0) {
            __nanosleep(64);
            if (++spins > (1 << 24)) {
              stalled = true;
              break;
            }
          }
        }
        stalled = __shfl_sync(0xFFFFFFFFu, stalled, 0);
        __syncwarp();
        __threadfence_block();
        SLOTC(lo16(w2f)) = *box;
      }
      continue;
    }
    V st, fb;
    if (kind <= OP_ACC) {
      st = vmax(vmax(p0, p1), vmax(p2, p3));
      fb = st;
    } else if (kind == OP_FINISH) {
      st = p0;
      fb = vmax(vmax(p0, p1), vmax(p2, p3));
    } else {  // OP_GATED
      const int nfixed = static_cast<int>(cls_b >> 4);
      st = w0;
      V gate = w0;
      if (nfixed > 0) st = vmax(st, p0); else gate = vmax(gate, p0);
      if (nfixed > 1) st = vmax(st, p1); else gate = vmax(gate, p1);
      if (nfixed > 2) st = vmax(st, p2); else gate = vmax(gate, p2);
      gate = vmax(gate, p3);
      fb = vmax(st, gate);
    }
    if (kind == OP_ACC) {
      SLOTC(lo16(w2f)) = st;
      continue;
    }
    if (kind == OP_SYNC) {
      const V rs = st;
      V S = rs;
      const int n_ext = static_cast<int>(hi16(w2f));
      for (int e = 0; e < n_ext; ++e) {
        const int4 xa = __ldg(gops + 2 * (i + 1 + e));
        const int n = __ldg(gops + 2 * (i + 1 + e) + 1).z & 0xFFFF;
        const uint32_t f[4] = {lo16(xa.x), hi16(xa.x), lo16(xa.y), hi16(xa.y)};
        for (int k = 0; k < kCertPerExt; ++k)
          if (k < n && f[k] != kNoSlot) S = vmax(S, SLOTC(f[k]));
      }
      bool cov = S == rs;
      for (int e = 0; e < n_ext; ++e) {
        const int4 xa = __ldg(gops + 2 * (i + 1 + e)), xb = __ldg(gops + 2 * (i + 1 + e) + 1);
        const int n = xb.z & 0xFFFF;
        const uint32_t f[4] = {lo16(xa.x), hi16(xa.x), lo16(xa.y), hi16(xa.y)};
        const uint32_t cv[4] = {lo16(xa.z), hi16(xa.z), lo16(xa.w), hi16(xa.w)};
        const uint32_t nx[4] = {lo16(xb.x), hi16(xb.x), lo16(xb.y), hi16(xb.y)};
        for (int k = 0; k < kCertPerExt; ++k) {
          if (k >= n) continue;
          if (f[k] != kNoSlot && cv[k] != kNoSlot)
            cov = cov || (SLOTC(f[k]) == S && SLOTC(cv[k]) <= rs);
          if (nx[k] != kNoSlot) fail = fail || SLOTC(nx[k]) <= S;
        }
      }
      fail = fail || !cov;
      st = S;
      fb = S;
      i += n_ext;
      if (i + 1 < n_ops) {  // the lookahead skipped the certificate records
        ra = __ldg(gops + 2 * (i + 1));
        rb = __ldg(gops + 2 * (i + 1) + 1);
      }
    }
    if (kind == OP_START) {
      SLOTC(lo16(w2f)) = st;
    } else {
      const int64_t task = static_cast<int64_t>(cd.node_base) + ca.z;
      const int64_t base = (static_cast<int64_t>(static_cast<uint32_t>(ca.y)) << 32) |
                           static_cast<uint32_t>(ca.x);
      const int64_t d = coop_duration(task, base, static_cast<int>(cls_b & 15u));
      const V fin = static_cast<V>(fb + static_cast<V>(d));
      // uint32 windows are sized by the nominal path: an addition that wraps
      // sends the scenario to the exact event-driven fix-up instead
      if (kRel && (fin < fb || d > 0xFFFFFFFFll)) fail = true;
      SLOTC(lo16(w2f)) = fin;
      if (flags_op & F_STORE_START) SLOTC(hi16(w3f)) = st;
      if (flags_op & F_BUSY) busy_a = static_cast<V>(busy_a + (fin - st));
      if (flags_op & F_SINK) hi = imax(hi, absv(fin));
      const uint64_t at = static_cast<uint64_t>(static_cast<uint32_t>(task)) * ld;
      if (LUMOS_OK(task >= 0 && task < P.n_tasks && col < static_cast<int>(ld))) {
        if (P.out_start) __stcs(start_c + at, absv(st));
        if (P.out_fin) __stcs(fin_c + at, absv(fin));
      }
    }
    if (flags_op & F_TRACK1) {
      const V cs = SLOTC(hi16(w2f));
      SLOTC(lo16(w3f)) = p0 >= st ? vmin(st, cs) : st;
    } else if (flags_op & F_TRACK) {
      const int4 xa = __ldg(gops + 2 * (i + 1)), xb = __ldg(gops + 2 * (i + 1) + 1);
      const uint32_t src[2][4] = {{lo16(xa.x), hi16(xa.x), lo16(xa.y), hi16(xa.y)},
                                  {lo16(xa.z), hi16(xa.z), lo16(xa.w), hi16(xa.w)}};
      const uint32_t cdst[2] = {lo16(xb.x), hi16(xb.x)};
      const int n_sets = xb.y & 0xFFFF;
      const V pv[4] = {p0, p1, p2, p3};
      for (int j = 0; j < kCovSets && j < n_sets; ++j) {
        V cvj = st;
        for (int k = 0; k < 4; ++k)
          if (src[j][k] != kNoSlot && pv[k] >= st) cvj = vmin(cvj, SLOTC(src[j][k]));
        SLOTC(cdst[j]) = cvj;
      }
      i += 1;
      if (i + 1 < n_ops) {
        ra = __ldg(gops + 2 * (i + 1));
        rb = __ldg(gops + 2 * (i + 1) + 1);
      }
    }
  }
#undef SLOTC
  if (acct_row >= 0 && !stalled)
    P.acct_a[static_cast<int64_t>(col) * P.n_ranks + acct_row] =
        kRel ? static_cast<int64_t>(static_cast<uint32_t>(busy_a)) : static_cast<int64_t>(busy_a);
  if (hi != kMinI64) {
    atomicMin(reinterpret_cast<long long*>(P.span_lo) + col, static_cast<long long>(W));
    atomicMax(reinterpret_cast<long long*>(P.span_hi) + col, static_cast<long long>(hi));
  }
  if (stalled) atomicExch(P.status + col, -2);
  else if (fail) atomicOr(P.status + col, 1);
}

__global__ void span_init_kernel(int64_t* lo, int64_t* hi, int32_t* status, int32_t count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) {
    lo[i] = kMaxI64;
    hi[i] = kMinI64;
    status[i] = 0;
  }
}

// span[s] = {start, end, makespan}; empty graph: {W, W, 0} (simulate.cpp:327-334)
__global__ void span_finalize_kernel(const int64_t* lo, const int64_t* hi, int64_t W,
                                     int64_t* span, int64_t* makespan, int32_t count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  int64_t a = lo[i], b = hi[i];
  if (a == kMaxI64) {
    a = W;
    b = W;
  }
  if (b < a) b = a;
  if (span) {
    span[3 * static_cast<int64_t>(i) + 0] = a;
    span[3 * static_cast<int64_t>(i) + 1] = b;
    span[3 * static_cast<int64_t>(i) + 2] = b - a;
  }
  if (makespan) makespan[i] = b - a;
}

// ------------------------------------------------------------------- K4
__global__ void durations_kernel(ScenarioParams sp, const int64_t* __restrict__ base,
                                 const uint8_t* __restrict__ cls, int32_t n_tasks,
                                 int64_t* __restrict__ dur, int64_t ld) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= sp.count) return;
  ThreadScen ts;
  init_thread_scen(sp, col, ts);
  for (int32_t t = blockIdx.y; t < n_tasks; t += gridDim.y)
    dur[static_cast<int64_t>(t) * ld + col] = scenario_duration<-1>(sp, ts, t, base[t], cls[t]);
}

// ------------------------------------------------------------------- K4r
// What-if retime (transform.cpp:219-349 through apply_whatif :713-760) of every
// (task, scenario): rt_task (device_common.cuh), then class scale and jitter.
__global__ void retime_durations_kernel(RetimeParams P) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= P.sp.count) return;
  ThreadScen ts;
  init_thread_scen(P.sp, col, ts);
  const RtCol rc = rt_col(P, col);
  for (int32_t t = blockIdx.y; t < P.n_tasks; t += gridDim.y)
    P.dur[static_cast<int64_t>(t) * P.ld + col] =
        scenario_duration<-1>(P.sp, ts, t, rt_task(P, rc, t), P.cls[t]);
}

// ------------------------------------------------------------------- K4v
// The width-only part of the retime per (variant, F_RT record): retimed GEMM /
// optimizer base durations, retimed collective byte counts (the same
// mul_div calls rt_task makes).  Variant 0 is the source widths.
__global__ void retime_variants_kernel(VariantParams P) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int v = blockIdx.y;
  if (j >= P.n_rec) return;
  const RtRec r = P.rec[j];
  const int32_t t = P.rec_task[j];
  const int64_t* tm = P.targets + 3 * static_cast<int64_t>(v);
  const bool hid = tm[0] != P.src_model[0] || tm[1] != P.src_model[1];
  int64_t out = r.kind == TS_RT_GEMM || r.kind == TS_RT_OPT ? r.base : P.bytes[t];
  if (hid) {
    if (r.kind == TS_RT_GEMM) {
      const int64_t* mnk = P.mnk + 3 * static_cast<int64_t>(t);
      int64_t nd[3];
      for (int k = 0; k < 3; ++k)
        nd[k] = mnk[k] == P.src_model[0] ? tm[0] : (mnk[k] == P.src_model[1] ? tm[1] : mnk[k]);
      out = mul_div_nonneg(r.base, nd[0] * nd[1] * nd[2], mnk[0] * mnk[1] * mnk[2], -1);
    } else if (r.kind == TS_RT_OPT) {
      out = mul_div_nonneg(r.base, tm[2], P.src_model[2], -1);
    } else if (r.kind == TS_RT_ALLREDUCE) {
      if (out >= 0) out = mul_div_nonneg(out, tm[2], P.src_model[2], -1);
    } else {  // TS_RT_P2P_SEND
      out = mul_div_nonneg(out, tm[0], P.src_model[0], -1);
    }
  }
  P.vval[static_cast<int64_t>(v) * P.n_rec + j] = out;
}

// ------------------------------------------------------------------- K5
constexpr int kMaxStreamsPerRank = 32;

// Each thread owns one scenario of one rank and merges the rank's stream
// timelines (each stream's kernels are chain-ordered, hence time-ordered and
// disjoint).  Per stream the thread keeps a private, double-buffered ring of
// 2 x H intervals in shared memory; the half it is not reading is refilled
// with cp.async (global -> shared, no registers), so the merge waits on memory
// only when a refill issued ~H intervals earlier has not landed yet.  The
// stream node lists carry the communication flag in bit 31.
template <int NS>
struct RingHalf {
  static constexpr int value = NS <= 2 ? 4 : NS <= 4 ? 2 : 1;
};

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// T: the time type of the merge — uint32 offsets from W when the accounting
// window fits 32 bits (then every compare is one 32-bit op), else int64.
template <int NS, typename T, bool kUtil>
__device__ __forceinline__ void rank_reduce_merge(const ReduceParams& P, int col, int r, int ns,
                                                  int64_t* ring, int64_t W, int64_t wend) {
  constexpr int H = RingHalf<NS>::value;
  constexpr T kInf = static_cast<T>(sizeof(T) == 4 ? 0xFFFFFFFFu : INT64_MAX);
  const int tid = threadIdx.x;
  const int s0 = P.rank_stream_off[r];
  const int64_t span = wend - W;
  const int64_t* __restrict__ S = P.start;
  const int64_t* __restrict__ F = P.fin;
  const int64_t ld = P.ld;
  const int* __restrict__ nodes = P.stream_nodes;
  // ring layout [NS][2 halves][H][2 (start, fin)][kThreads]
#define RING(j, h, q, k) ring[(((((j) * 2 + (h)) * H + (q)) * 2 + (k)) * kThreads) + tid]
  auto rel = [&](int64_t v) -> T {
    int64_t x = v - W;
    x = x < 0 ? 0 : (x > span ? span : x);
    return static_cast<T>(x);
  };

  int next_idx[NS] = {}, end_idx[NS] = {};  // set below; zeroed for the front end
  int half[NS], pos[NS], avail[NS], pend[NS];
  uint32_t cbits[NS], pbits[NS];
  auto prefetch = [&](int j, int h) {
    const int base = next_idx[j];
    const int n = min(H, end_idx[j] - base);
    uint32_t bits = 0;
#pragma unroll
    for (int q = 0; q < H; ++q)
      if (q < n) {
        const int e = nodes[base + q];
        int node = e & 0x7FFFFFFF;
        if (!LUMOS_OK(node < P.n_tasks_total)) node = 0;
        bits |= static_cast<uint32_t>(e < 0) << q;
        const int64_t off = static_cast<int64_t>(node) * ld + col;
        cp_async8(&RING(j, h, q, 0), S + off);
        cp_async8(&RING(j, h, q, 1), F + off);
      }
    cp_async_commit();
    next_idx[j] = base + n;
    pend[j] = n;
    pbits[j] = bits;
  };
  T cs[NS], ce[NS];
  uint32_t cc = 0, inside = 0;  // per-stream bits: current interval is comm / open
  auto advance = [&](int j) {
    for (;;) {
      if (pos[j] >= avail[j]) {
        if (pend[j] == 0) {
          cs[j] = ce[j] = kInf;
          return;
        }
        cp_async_wait_all();
        half[j] ^= 1;
        avail[j] = pend[j];
        cbits[j] = pbits[j];
        pos[j] = 0;
        pend[j] = 0;
        if (next_idx[j] < end_idx[j]) prefetch(j, half[j] ^ 1);
      }
      const int q = pos[j]++;
      const T a = rel(RING(j, half[j], q, 0)), b = rel(RING(j, half[j], q, 1));
      if (a < b) {
        cs[j] = a;
        ce[j] = b;
        cc = (cc & ~(1u << j)) | (((cbits[j] >> q) & 1u) << j);
        return;
      }
    }
  };
  int64_t busy[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    next_idx[j] = j < ns ? P.stream_node_off[s0 + j] : 0;
    end_idx[j] = j < ns ? P.stream_node_off[s0 + j + 1] : 0;
    half[j] = 1;  // the first switch moves to half 0
    pos[j] = avail[j] = pend[j] = 0;
    cbits[j] = pbits[j] = 0;
    busy[j] = 0;
    if (next_idx[j] < end_idx[j]) prefetch(j, 0);
  }
#pragma unroll
  for (int j = 0; j < NS; ++j) advance(j);

  int compute = 0, comm = 0;
  T prev = 0;
  int64_t ec = 0, em = 0, ov = 0, ot = 0;
  BinAcc ua;
  if (kUtil) ua.init(P.util + (static_cast<int64_t>(col) * P.n_ranks + r) * P.util_max_bins,
                     P.util_bw, P.util_max_bins);
  for (;;) {
    int jm = -1;
    T tm = kInf;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const T t = ((inside >> j) & 1u) ? ce[j] : cs[j];
      if (t < tm) {
        tm = t;
        jm = j;
      }
    }
    if (jm < 0) break;
    if (tm > prev) {
      const int64_t d = static_cast<int64_t>(tm - prev);
      if (compute > 0) {
        if (comm > 0) ov += d; else ec += d;
      } else {
        if (comm > 0) em += d; else ot += d;
      }
      if (kUtil && (compute > 0 || comm > 0))
        ua.add(static_cast<int64_t>(prev), static_cast<int64_t>(tm), 1);
      prev = tm;
    }
    const bool is_comm = (cc >> jm) & 1u;
    if (!((inside >> jm) & 1u)) {
      if (is_comm) ++comm; else ++compute;
      inside |= 1u << jm;
    } else {
      if (is_comm) --comm; else --compute;
      inside &= ~(1u << jm);
#pragma unroll
      for (int j = 0; j < NS; ++j)
        if (j == jm) {
          busy[j] += static_cast<int64_t>(ce[j] - cs[j]);
          advance(j);
        }
    }
  }
#undef RING
  if (kUtil) ua.flush();
  {
    const int64_t d = span - static_cast<int64_t>(prev);
    if (d > 0) {
      if (compute > 0) {
        if (comm > 0) ov += d; else ec += d;
      } else {
        if (comm > 0) em += d; else ot += d;
      }
    }
  }
  if (P.breakdown) {
    int64_t* row = P.breakdown + (static_cast<int64_t>(col) * P.n_ranks + r) * 5;
    row[0] = span;
    row[1] = ec;
    row[2] = em;
    row[3] = ov;
    row[4] = ot;
  }
  if (P.stream_busy) {
#pragma unroll
    for (int j = 0; j < NS; ++j)
      if (j < ns) P.stream_busy[static_cast<int64_t>(col) * P.n_streams + s0 + j] = busy[j];
  }
}

template <int NS, bool kUtil>
__device__ __forceinline__ void rank_reduce_body(const ReduceParams& P, int col, int r, int ns,
                                                 int64_t* ring) {
  const int64_t W = P.window_start;
  int64_t wend = P.window_end;
  {
    const int64_t a = P.span_lo[col], b = P.span_hi[col];
    const int64_t m = (a == kMaxI64) ? 0 : (b - a);
    if (W + m > wend) wend = W + m;
  }
  if (wend < W) wend = W;
  if (wend - W < 0xFFFFFFFFll)
    rank_reduce_merge<NS, uint32_t, kUtil>(P, col, r, ns, ring, W, wend);
  else
    rank_reduce_merge<NS, int64_t, kUtil>(P, col, r, ns, ring, W, wend);
}

template <int NS, bool kUtil>
__global__ void __launch_bounds__(kThreads) rank_reduce_kernel(ReduceParams P) {
  extern __shared__ int64_t ring[];
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = P.rank_list[blockIdx.y];
  if (col >= P.count) return;
  const int ns = P.rank_stream_off[r + 1] - P.rank_stream_off[r];
  rank_reduce_body<NS, kUtil>(P, col, r, ns, ring);
}

// ---------------------------------------------------------------- K5 fast path
// Ranks with exactly one compute-only stream A and NC comm-only streams (every
// generator rank): the four categories follow from |A|, |U| (U = union of the
// comm intervals) and |A ∩ U|:
//   overlap = |A∩U|, exposed compute = |A| - overlap, exposed comm = |U| - overlap,
//   other = span - |A| - |U| + overlap
// — the same numbers the event merge produces, since A's intervals are
// disjoint (one stream is one chain) and the categories only ask whether any
// compute / any comm kernel is running.  A is walked by a pointer (two loads
// and a compare per kernel); only the few comm intervals go through a merge.
template <int H, typename T>
struct Cursor {
  int next, end, half, pos, avail, pend;
  int n_tasks_total;  // bounds checks
  int64_t* ring;  // [2 halves][H][2][kThreads] + tid
  __device__ __forceinline__ int64_t& at(int h, int q, int k) {
    return ring[((h * H + q) * 2 + k) * kThreads];
  }
  __device__ __forceinline__ void prefetch(const int* __restrict__ nodes,
                                           const int64_t* __restrict__ S,
                                           const int64_t* __restrict__ F, int64_t ld, int col,
                                           int h) {
    const int base = next;
    const int n = min(H, end - base);
#pragma unroll
    for (int q = 0; q < H; ++q)
      if (q < n) {
        int node = nodes[base + q] & 0x7FFFFFFF;
        if (!LUMOS_OK(node < n_tasks_total)) node = 0;
        const int64_t off = static_cast<int64_t>(node) * ld + col;
        cp_async8(&at(h, q, 0), S + off);
        cp_async8(&at(h, q, 1), F + off);
      }
    cp_async_commit();
    next = base + n;
    pend = n;
  }
  __device__ __forceinline__ void init(int b, int e, int64_t* rb, const int* nodes,
                                       const int64_t* S, const int64_t* F, int64_t ld, int col,
                                       int n_tasks = INT32_MAX) {
    n_tasks_total = n_tasks;
    next = b;
    end = e;
    half = 1;
    pos = avail = pend = 0;
    ring = rb;
    if (next < end) prefetch(nodes, S, F, ld, col, 0);
  }
  // next non-empty clipped interval [a, b); false when the stream is done
  template <typename Rel>
  __device__ __forceinline__ bool get(T& a, T& b, const int* nodes, const int64_t* S,
                                      const int64_t* F, int64_t ld, int col, Rel rel) {
    for (;;) {
      if (pos >= avail) {
        if (pend == 0) return false;
        cp_async_wait_all();
        half ^= 1;
        avail = pend;
        pos = 0;
        pend = 0;
        if (next < end) prefetch(nodes, S, F, ld, col, half ^ 1);
      }
      const int q = pos++;
      a = rel(at(half, q, 0));
      b = rel(at(half, q, 1));
      if (a < b) return true;
    }
  }
};

#ifndef LUMOS_FAST_HA
#define LUMOS_FAST_HA 8
#endif
#ifndef LUMOS_FAST_HC
#define LUMOS_FAST_HC 2
#endif
constexpr int kFastHA = LUMOS_FAST_HA;  // ring half of the compute stream
constexpr int kFastHC = LUMOS_FAST_HC;  // ring half of a comm stream

template <int NC>
constexpr size_t fast_ring_words() {
  return static_cast<size_t>(2 * kFastHA * 2 + NC * 2 * kFastHC * 2);
}

// kLite (split accounting, program.hpp FusedDesc): the A cursor walks only the
// rank's candidate compute kernels and |A| is the walk's sum; ci == kNoA: the
// rank has no compute stream
constexpr int kNoA = 0xFF;
template <int NC, typename T, bool kUtil, bool kLite>
__device__ __forceinline__ void rank_reduce_fast_body(const ReduceParams& P, int col, int r,
                                                      int ci, int64_t* ring, int64_t W,
                                                      int64_t wend) {
  constexpr T kInf = static_cast<T>(sizeof(T) == 4 ? 0xFFFFFFFFu : INT64_MAX);
  const int tid = threadIdx.x;
  const int s0 = P.rank_stream_off[r];
  const int64_t span = wend - W;
  const int64_t* __restrict__ S = P.start;
  const int64_t* __restrict__ F = P.fin;
  const int64_t ld = P.ld;
  const int* __restrict__ nodes = P.stream_nodes;
  auto rel = [&](int64_t v) -> T {
    int64_t x = v - W;
    x = x < 0 ? 0 : (x > span ? span : x);
    return static_cast<T>(x);
  };
  Cursor<kFastHA, T> A;
  if (kLite)
    A.init(P.cand_off[r], P.cand_off[r + 1], ring + tid, P.cand_nodes, S, F, ld, col,
           P.n_tasks_total);
  else
    A.init(P.stream_node_off[s0 + ci], P.stream_node_off[s0 + ci + 1], ring + tid, nodes, S, F,
           ld, col, P.n_tasks_total);
  const int* __restrict__ anodes = kLite ? P.cand_nodes : nodes;
  Cursor<kFastHC, T> C[NC > 0 ? NC : 1];
  T cs[NC > 0 ? NC : 1], ce[NC > 0 ? NC : 1];
  int64_t cbusy[NC > 0 ? NC : 1];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const int s = s0 + j + (ci != kNoA && j >= ci ? 1 : 0);
    C[j].init(P.stream_node_off[s], P.stream_node_off[s + 1],
              ring + (2 * kFastHA * 2 + j * 2 * kFastHC * 2) * kThreads + tid, nodes, S, F, ld,
              col, P.n_tasks_total);
    cbusy[j] = 0;
  }
#pragma unroll
  for (int j = 0; j < NC; ++j)
    if (!C[j].get(cs[j], ce[j], nodes, S, F, ld, col, rel)) cs[j] = ce[j] = kInf;

  // utilization = |A| + |U| - |A n U| per bin, one accumulator per term
  BinAcc ua, uu, uo;
  if (kUtil) {
    int64_t* row = P.util + (static_cast<int64_t>(col) * P.n_ranks + r) * P.util_max_bins;
    ua.init(row, P.util_bw, P.util_max_bins);
    uu.init(row, P.util_bw, P.util_max_bins);
    uo.init(row, P.util_bw, P.util_max_bins);
  }
  // union of the comm intervals, produced in time order
  T us = kInf, ue = kInf;
  int64_t m = 0;
  auto next_union = [&]() {
    int jm = -1;
    T tm = kInf;
#pragma unroll
    for (int j = 0; j < NC; ++j)
      if (cs[j] < tm) {
        tm = cs[j];
        jm = j;
      }
    if (jm < 0) {
      us = ue = kInf;
      return;
    }
    us = tm;
    ue = tm;
    for (;;) {
      // absorb every comm interval starting inside [us, ue] (the first pass
      // takes the earliest one, whose start is us)
      bool any = false;
#pragma unroll
      for (int j = 0; j < NC; ++j)
        if (cs[j] <= ue) {
          if (ce[j] > ue) ue = ce[j];
          cbusy[j] += static_cast<int64_t>(ce[j] - cs[j]);
          if (!C[j].get(cs[j], ce[j], nodes, S, F, ld, col, rel)) cs[j] = ce[j] = kInf;
          any = true;
        }
      if (!any) break;
    }
    m += static_cast<int64_t>(ue - us);
    if (kUtil) uu.add(static_cast<int64_t>(us), static_cast<int64_t>(ue), 1);
  };
  if (NC > 0) next_union();

  int64_t busy_a = 0, ov = 0;
  T as, ae;
  while (A.get(as, ae, anodes, S, F, ld, col, rel)) {
    if (!kLite) busy_a += static_cast<int64_t>(ae - as);
    if (kUtil) ua.add(static_cast<int64_t>(as), static_cast<int64_t>(ae), 1);
    if (NC > 0) {
      while (ue <= as) next_union();
      while (us < ae) {
        const T lo = us > as ? us : as;
        const T hi = ue < ae ? ue : ae;
        ov += static_cast<int64_t>(hi - lo);
        if (kUtil) uo.add(static_cast<int64_t>(lo), static_cast<int64_t>(hi), -1);
        if (ue <= ae) next_union(); else break;
      }
    }
  }
  if (NC > 0)
    while (us != kInf) next_union();
  if (kLite) busy_a = P.acct_a[static_cast<int64_t>(col) * P.n_ranks + r];
  if (kUtil) {
    ua.flush();
    uu.flush();
    uo.flush();
  }

  if (P.breakdown) {
    int64_t* row = P.breakdown + (static_cast<int64_t>(col) * P.n_ranks + r) * 5;
    row[0] = span;
    row[1] = busy_a - ov;
    row[2] = m - ov;
    row[3] = ov;
    row[4] = span - busy_a - m + ov;
  }
  if (P.stream_busy) {
    int64_t* b = P.stream_busy + static_cast<int64_t>(col) * P.n_streams + s0;
    if (ci != kNoA) b[ci] = busy_a;
#pragma unroll
    for (int j = 0; j < NC; ++j) b[j + (ci != kNoA && j >= ci ? 1 : 0)] = cbusy[j];
  }
}

// rank_list entries: rank | compute-stream index << 24
// (4 CTAs per SM: their rings already limit shared memory to that, so the
// registers can go to 128 without costing occupancy)
template <int NC, bool kUtil, bool kLite>
__global__ void __launch_bounds__(kThreads, 4) rank_reduce_fast_kernel(ReduceParams P) {
  extern __shared__ int64_t ring[];
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t e = static_cast<uint32_t>(P.rank_list[blockIdx.y]);
  if (col >= P.count) return;
  if (kLite && P.status && P.status[col] != 0) return;  // the event-driven fix-up reduced it
  const int r = static_cast<int>(e & 0xFFFFFFu), ci = static_cast<int>(e >> 24);
  const int64_t W = P.window_start;
  int64_t wend = P.window_end;
  {
    const int64_t a = P.span_lo[col], b = P.span_hi[col];
    const int64_t m = (a == kMaxI64) ? 0 : (b - a);
    if (W + m > wend) wend = W + m;
  }
  if (wend < W) wend = W;
  if (wend - W < 0xFFFFFFFFll)
    rank_reduce_fast_body<NC, uint32_t, kUtil, kLite>(P, col, r, ci, ring, W, wend);
  else
    rank_reduce_fast_body<NC, int64_t, kUtil, kLite>(P, col, r, ci, ring, W, wend);
}

// ------------------------------------------------------------------- K6
// compare_replay deltas (metrics.cpp:189-221).  Pass 1: thread = (scenario
// column, task chunk), tasks ascending; the chunk's worst_n largest |delta|
// (ties: the smaller task id, i.e. the one seen first) kept sorted in local
// memory.  Pass 2 merges the chunks per column with the same order.
struct WorstEntry {
  int64_t mag;
  int64_t task;
};
__device__ __forceinline__ bool worse(int64_t ma, int64_t ta, const WorstEntry& b) {
  return ma > b.mag || (ma == b.mag && ta < b.task);
}
// inserts (mag, task) into the sorted list w[0..n) of capacity cap
__device__ __forceinline__ void worst_insert(WorstEntry* w, int& n, int cap, int64_t mag,
                                             int64_t task) {
  if (n == cap && !worse(mag, task, w[cap - 1])) return;
  int k = n < cap ? n++ : cap - 1;
  while (k > 0 && worse(mag, task, w[k - 1])) {
    w[k] = w[k - 1];
    --k;
  }
  w[k] = WorstEntry{mag, task};
}

__global__ void delta_partial_kernel(DeltaParams P) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  if (col >= P.count) return;
  const int32_t per = (P.n_tasks + P.n_chunks - 1) / P.n_chunks;
  const int32_t t0 = chunk * per, t1 = min(P.n_tasks, t0 + per);
  WorstEntry w[kMaxWorst];
  int n = 0;
  int64_t sum = 0;
  for (int32_t t = t0; t < t1; ++t) {
    const int64_t d = __ldcs(P.start + static_cast<int64_t>(t) * P.ld + col) - __ldg(P.ostart + t);
    const int64_t a = d < 0 ? -d : d;
    sum += a;
    worst_insert(w, n, P.worst_n, a, t);
  }
  P.partial_sum[static_cast<int64_t>(chunk) * P.count + col] = sum;
  int64_t* o = P.partial + (static_cast<int64_t>(chunk) * P.count + col) * P.worst_n * 2;
  for (int k = 0; k < P.worst_n; ++k) {
    o[2 * k] = k < n ? w[k].mag : -1;
    o[2 * k + 1] = k < n ? w[k].task : -1;
  }
}

__global__ void delta_final_kernel(DeltaParams P) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= P.count) return;
  WorstEntry w[kMaxWorst];
  int n = 0;
  int64_t sum = 0;
  for (int c = 0; c < P.n_chunks; ++c) {
    sum += P.partial_sum[static_cast<int64_t>(c) * P.count + col];
    const int64_t* o = P.partial + (static_cast<int64_t>(c) * P.count + col) * P.worst_n * 2;
    for (int k = 0; k < P.worst_n && o[2 * k] >= 0; ++k) worst_insert(w, n, P.worst_n, o[2 * k], o[2 * k + 1]);
  }
  if (P.abs_sum) P.abs_sum[col] = sum;
  if (P.worst) {
    int64_t* out = P.worst + static_cast<int64_t>(col) * P.worst_n * 3;
    for (int k = 0; k < P.worst_n; ++k) {
      if (k < n) {
        const int64_t t = w[k].task;
        out[3 * k] = w[k].mag;
        out[3 * k + 1] = t;
        out[3 * k + 2] = __ldcs(P.start + t * P.ld + col) - __ldg(P.ostart + t);
      } else {
        out[3 * k] = 0;
        out[3 * k + 1] = -1;
        out[3 * k + 2] = 0;
      }
    }
  }
}

__global__ void util_nbins_kernel(const int64_t* lo, const int64_t* hi, int64_t W,
                                  int64_t window_end, int64_t w, int32_t* n_bins, int32_t count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int64_t m = lo[i] == kMaxI64 ? 0 : hi[i] - lo[i];
  int64_t wend = window_end > W + m ? window_end : W + m;
  if (wend < W) wend = W;
  n_bins[i] = static_cast<int32_t>((wend - W + w - 1) / w);
}

}  // namespace

// ------------------------------------------------------------ launchers
cudaError_t launch_deltas(const DeltaParams& p, cudaStream_t stream) {
  if (p.count <= 0) return cudaSuccess;
  DeltaParams q = p;
  if (q.n_tasks > 0 && q.n_chunks > 0) {
    dim3 grid((q.count + 127) / 128, q.n_chunks);
    delta_partial_kernel<<<grid, 128, 0, stream>>>(q);
  } else {
    q.n_chunks = 0;  // no entries: sum 0, worst {0, -1, 0}
  }
  delta_final_kernel<<<(q.count + 127) / 128, 128, 0, stream>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_util_nbins(const int64_t* lo, const int64_t* hi, int64_t W, int64_t window_end,
                              int64_t w, int32_t* n_bins, int32_t count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  util_nbins_kernel<<<(count + 255) / 256, 256, 0, stream>>>(lo, hi, W, window_end, w, n_bins,
                                                             count);
  return cudaGetLastError();
}
int walk_threads() { return kThreads; }

#ifdef LUMOS_DEBUG_BOUNDS
int debug_bounds_status() {
  int v = 0, zero = 0;
  if (cudaMemcpyFromSymbol(&v, lumos_bounds_fail, sizeof(int)) != cudaSuccess) return -1;
  cudaMemcpyToSymbol(lumos_bounds_fail, &zero, sizeof(int));
  return v;
}
#else
int debug_bounds_status() { return 0; }
#endif
// (des.cu keeps its own flag: debug_bounds_status_des)

template <int kT, int kMode, bool kWS, bool kWF, typename V, int kS>
static cudaError_t launch_walk_t(const WalkParams& p, size_t smem, unsigned blocks,
                                 cudaStream_t stream) {
  // set per launch: the attribute is per device, and several host threads or
  // devices may launch concurrently
  auto go = [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    kern<<<blocks, kT, smem, stream>>>(p);
    return cudaGetLastError();
  };
  if constexpr ((kMode & kModeRetime) != 0)
    return go(replay_walk_rt_kernel<kT, kMode, kWS, kWF, V, kS>);
  else
    return go(replay_walk_kernel<kT, kMode, kWS, kWF, V, kS>);
}

template <int kT, int kMode, typename V, int kS>
static cudaError_t launch_walk_mode(const WalkParams& p, size_t smem, unsigned blocks,
                                    cudaStream_t stream) {
  const bool s = p.out_start != nullptr, f = p.out_fin != nullptr;
  if (s && f) return launch_walk_t<kT, kMode, true, true, V, kS>(p, smem, blocks, stream);
  if (f) return launch_walk_t<kT, kMode, false, true, V, kS>(p, smem, blocks, stream);
  if (s) return launch_walk_t<kT, kMode, true, false, V, kS>(p, smem, blocks, stream);
  return launch_walk_t<kT, kMode, false, false, V, kS>(p, smem, blocks, stream);
}

template <int kT, typename V, int kS>
static cudaError_t launch_walk_width(const WalkParams& p, size_t smem, cudaStream_t stream) {
  const int per_block = kT * kS;
  const long long chunks = (p.sp.count + per_block - 1) / per_block;
  const long long blocks = chunks * p.n_comps;
  if (blocks <= 0) return cudaSuccess;
  const unsigned nb = static_cast<unsigned>(blocks);
  switch (p.sp.mode) {
    case 0: return launch_walk_mode<kT, 0, V, kS>(p, smem, nb, stream);
    case kModeScale: return launch_walk_mode<kT, kModeScale, V, kS>(p, smem, nb, stream);
    case kModeJitter: return launch_walk_mode<kT, kModeJitter, V, kS>(p, smem, nb, stream);
    case kModeScale | kModeJitter:
      return launch_walk_mode<kT, kModeScale | kModeJitter, V, kS>(p, smem, nb, stream);
    default:
      if (p.sp.mode & kModeRetime) {
        if constexpr (sizeof(V) == 8) {  // retime walks keep int64 slot values
          constexpr int R = kModeRetime;
          switch (p.sp.mode & (kModeScale | kModeJitter)) {
            case 0: return launch_walk_mode<kT, R, V, kS>(p, smem, nb, stream);
            case kModeScale: return launch_walk_mode<kT, R | kModeScale, V, kS>(p, smem, nb, stream);
            case kModeJitter: return launch_walk_mode<kT, R | kModeJitter, V, kS>(p, smem, nb, stream);
            default:
              return launch_walk_mode<kT, R | kModeScale | kModeJitter, V, kS>(p, smem, nb, stream);
          }
        }
        return cudaErrorInvalidValue;
      }
      return launch_walk_mode<kT, kModeExplicit, V, kS>(p, smem, nb, stream);
  }
}

// shared memory of a walk CTA of t threads with `vbytes` bytes of slot values
// per thread and slot
static size_t walk_smem(int n_slots, int t, int vbytes) {
  return 8 * kChunk * sizeof(int4) + static_cast<size_t>(kMaxClasses) * t * sizeof(int2) +
         static_cast<size_t>(n_slots < kFirstSlot ? kFirstSlot : n_slots) * t * vbytes;
}

int walk_width(int n_slots, bool rel32) {
  const size_t cap = 227 * 1024;
  const int vb = (rel32 ? 4 : 8) * 2;
  if (walk_smem(n_slots, 128, vb) <= cap / 2) return 128;  // >= 2 CTAs per SM
  if (walk_smem(n_slots, 64, vb) <= cap / 2) return 64;
  if (walk_smem(n_slots, 32, vb) <= cap) return 32;
  return 0;
}

// One scenario per thread when two per thread would leave the GPU short of
// warps: fewer than ~8 warps per SM of (component, scenario-pair) work.
static bool single_scenario(const WalkParams& p) {
  const long long pairs = static_cast<long long>(p.n_comps) * ((p.sp.count + 1) / 2);
  return pairs < 148LL * 8 * 32;
}

template <typename V, int kS>
static cudaError_t launch_walk_v(const WalkParams& p, int n_slots, int t, cudaStream_t stream) {
  const int vb = static_cast<int>(sizeof(V)) * kS;
  if (t == 128) return launch_walk_width<128, V, kS>(p, walk_smem(n_slots, 128, vb), stream);
  if (t == 64) return launch_walk_width<64, V, kS>(p, walk_smem(n_slots, 64, vb), stream);
  if (t == 32) return launch_walk_width<32, V, kS>(p, walk_smem(n_slots, 32, vb), stream);
  return cudaErrorInvalidConfiguration;
}

static std::atomic<int64_t> g_walk_variant[5];

void walk_variant_counts(int64_t out[5]) {
  for (int k = 0; k < 5; ++k) out[k] = g_walk_variant[k].load();
}

cudaError_t launch_replay_walk(const WalkParams& p, int n_slots, cudaStream_t stream) {
  const bool rel = p.rel32 != 0;
  const int t = walk_width(n_slots, rel);
  // two scenarios per thread share one Philox call per task, which needs the
  // thread's columns to be one global pair: an even first id.  force_ks (tests)
  // overrides the occupancy choice but never the pairing rule.
  bool one = p.force_ks == 1 || (p.force_ks != 2 && single_scenario(p));
  if (p.sp.first & 1) one = true;
  g_walk_variant[(one ? 0 : 2) + (rel ? 0 : 1)]++;
  if (one)
    return rel ? launch_walk_v<uint32_t, 1>(p, n_slots, t, stream)
               : launch_walk_v<int64_t, 1>(p, n_slots, t, stream);
  return rel ? launch_walk_v<uint32_t, 2>(p, n_slots, t, stream)
             : launch_walk_v<int64_t, 2>(p, n_slots, t, stream);
}

// shared-memory carveout of the cluster walk (percent of the unified L1 /
// shared array; LUMOS_CLUSTER_CARVEOUT, default the driver's choice = -1):
// the driver sizes it for the register-limited occupancy, which can leave
// shared memory the binding limit once registers allow more CTAs per SM
static int cluster_carveout() {
  static const int v = [] {
    const char* e = std::getenv("LUMOS_CLUSTER_CARVEOUT");
    return e ? std::atoi(e) : LUMOS_CLUSTER_CARVEOUT_DEFAULT;
  }();
  return v;
}

template <typename K>
static cudaError_t cluster_attrs(K kern, size_t smem, int cl_size) {
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
  if (e == cudaSuccess && cl_size > 8)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess && cluster_carveout() >= 0)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cluster_carveout());
  return e;
}

template <int kMode, bool kWS, bool kWF>
static cudaError_t launch_cluster_t(const WalkParams& p, size_t smem, unsigned blocks,
                                    cudaStream_t stream) {
  auto kern = p.cl_check ? cluster_walk_kernel<kMode, kWS, kWF, true>
                         : cluster_walk_kernel<kMode, kWS, kWF, false>;
  cudaError_t e = cluster_attrs(kern, smem, p.cl_size);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.cl_size);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // LUMOS_CLUSTER_POLICY=1 spread / 2 load-balancing (default: the driver's)
  static const int policy = [] {
    const char* e = std::getenv("LUMOS_CLUSTER_POLICY");
    return e ? std::atoi(e) : 0;
  }();
  if (policy == 1 || policy == 2) {
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference =
        policy == 1 ? cudaClusterSchedulingPolicySpread : cudaClusterSchedulingPolicyLoadBalancing;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int kMode>
static cudaError_t launch_cluster_mode(const WalkParams& p, size_t smem, unsigned blocks,
                                       cudaStream_t stream) {
  const bool s = p.out_start != nullptr, f = p.out_fin != nullptr;
  if (s && f) return launch_cluster_t<kMode, true, true>(p, smem, blocks, stream);
  if (f) return launch_cluster_t<kMode, false, true>(p, smem, blocks, stream);
  if (s) return launch_cluster_t<kMode, true, false>(p, smem, blocks, stream);
  return launch_cluster_t<kMode, false, false>(p, smem, blocks, stream);
}

bool cluster_walk_supported(int cl_size, int n_slots) {
  if (cl_size < 1 || cl_size > 16 || walk_width(n_slots, true) != 128) return false;
  auto kern = cluster_walk_kernel<kModeJitter, true, true, true>;
  const size_t smem = walk_smem(n_slots, 128, 8);
  if (cluster_attrs(kern, smem, cl_size) != cudaSuccess) return cudaGetLastError(), false;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(cl_size));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cl_size);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return cudaGetLastError(), false;
  return n > 0;
}

cudaError_t launch_cluster_walk(const WalkParams& p, int n_slots, cudaStream_t stream) {
  // scenario pairs share a Philox call (needs an even first id)
  if (p.cl_size < 1 || p.cl_size > 16 || (p.sp.first & 1)) return cudaErrorNotSupported;
  const long long units = static_cast<long long>(p.n_comps) * ((p.sp.count + 255) / 256);
  if (units <= 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>(units * p.cl_size);
  const size_t smem = walk_smem(n_slots, 128, 8);
  if (p.sp.mode == 0 || p.sp.mode == kModeScale || p.sp.mode == kModeJitter ||
      p.sp.mode == (kModeScale | kModeJitter))
    g_walk_variant[4]++;
  switch (p.sp.mode) {
    case 0: return launch_cluster_mode<0>(p, smem, blocks, stream);
    case kModeScale: return launch_cluster_mode<kModeScale>(p, smem, blocks, stream);
    case kModeJitter: return launch_cluster_mode<kModeJitter>(p, smem, blocks, stream);
    case kModeScale | kModeJitter:
      return launch_cluster_mode<kModeScale | kModeJitter>(p, smem, blocks, stream);
    default: return cudaErrorNotSupported;  // explicit durations / retime: cooperative walk
  }
}

template <typename V>
static cudaError_t launch_coop_v(const WalkParams& p, const CoopParams& c, cudaStream_t stream) {
  const size_t smem = static_cast<size_t>((c.n_mail * 4 + 15) / 16) * 16 +
                      static_cast<size_t>(c.n_mail) * 32 * sizeof(V) +
                      static_cast<size_t>(c.max_ranks) * c.n_slots * 32 * sizeof(V);
  const long long chunks = (p.sp.count + 31) / 32;
  const long long blocks = chunks * p.n_comps;
  if (blocks <= 0) return cudaSuccess;
  const int threads = 32 * c.max_ranks;
  auto go = [&](auto kern) -> cudaError_t {
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    kern<<<static_cast<unsigned>(blocks), threads, smem, stream>>>(p, c);
    return cudaGetLastError();
  };
  auto by_mode = [&](auto tag) -> cudaError_t {
    constexpr int W = decltype(tag)::value;
    switch (p.sp.mode) {
      case 0: return go(coop_walk_kernel<0, V, W>);
      case kModeScale: return go(coop_walk_kernel<kModeScale, V, W>);
      case kModeJitter: return go(coop_walk_kernel<kModeJitter, V, W>);
      case kModeScale | kModeJitter: return go(coop_walk_kernel<kModeScale | kModeJitter, V, W>);
      default: return go(coop_walk_kernel<kModeExplicit, V, W>);
    }
  };
  if (c.max_ranks <= 16) return by_mode(std::integral_constant<int, 16>{});
  return by_mode(std::integral_constant<int, 32>{});
}

cudaError_t launch_coop_walk(const WalkParams& p, const CoopParams& c, cudaStream_t stream) {
  if (c.max_ranks < 1 || c.max_ranks > 32) return cudaErrorInvalidConfiguration;
  return c.rel32 ? launch_coop_v<uint32_t>(p, c, stream) : launch_coop_v<int64_t>(p, c, stream);
}

cudaError_t launch_span_init(int64_t* lo, int64_t* hi, int32_t* status, int32_t count,
                             cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  span_init_kernel<<<(count + 255) / 256, 256, 0, stream>>>(lo, hi, status, count);
  return cudaGetLastError();
}

cudaError_t launch_span_finalize(const int64_t* lo, const int64_t* hi, int64_t W, int64_t* span,
                                 int64_t* makespan, int32_t count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  span_finalize_kernel<<<(count + 255) / 256, 256, 0, stream>>>(lo, hi, W, span, makespan, count);
  return cudaGetLastError();
}

cudaError_t launch_retime_durations(const RetimeParams& p, cudaStream_t stream) {
  if (p.sp.count <= 0 || p.n_tasks <= 0) return cudaSuccess;
  dim3 grid((p.sp.count + 127) / 128, p.n_tasks < 4096 ? p.n_tasks : 4096);
  retime_durations_kernel<<<grid, 128, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_retime_variants(const VariantParams& p, cudaStream_t stream) {
  if (p.n_rec <= 0 || p.n_var <= 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((p.n_rec + 255) / 256), static_cast<unsigned>(p.n_var));
  retime_variants_kernel<<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_durations(const ScenarioParams& sp, const int64_t* base, const uint8_t* cls,
                             int32_t n_tasks, int64_t* dur, int64_t ld, cudaStream_t stream) {
  if (sp.count <= 0 || n_tasks <= 0) return cudaSuccess;
  dim3 grid((sp.count + 127) / 128, n_tasks < 4096 ? n_tasks : 4096);
  durations_kernel<<<grid, 128, 0, stream>>>(sp, base, cls, n_tasks, dur, ld);
  return cudaGetLastError();
}

int reduce_bucket(int ns) {
  return ns <= 1 ? 0 : ns == 2 ? 1 : ns == 3 ? 2 : ns == 4 ? 3 : ns <= 8 ? 4 : ns <= 16 ? 5 : 6;
}

cudaError_t launch_rank_reduce(const ReduceParams& p, int bucket, int n_ranks_in_bucket,
                               cudaStream_t stream) {
  if (p.count <= 0 || n_ranks_in_bucket <= 0) return cudaSuccess;
  dim3 grid((p.count + kThreads - 1) / kThreads, n_ranks_in_bucket);
  auto go = [&](auto kern, int ns) -> cudaError_t {
    const int h = ns <= 2 ? 4 : ns <= 4 ? 2 : 1;
    const size_t smem = static_cast<size_t>(ns) * 2 * h * 2 * kThreads * sizeof(int64_t);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, kThreads, smem, stream>>>(p);
    return cudaSuccess;
  };
  const bool u = p.util != nullptr;
  cudaError_t e;
#define LUMOS_GEN(NS_) (u ? go(rank_reduce_kernel<NS_, true>, NS_) : go(rank_reduce_kernel<NS_, false>, NS_))
#define LUMOS_FAST(NC_)                                                             \
  (u ? fast(rank_reduce_fast_kernel<NC_, true, false>, fast_ring_words<NC_>()) \
     : fast(rank_reduce_fast_kernel<NC_, false, false>, fast_ring_words<NC_>()))
#define LUMOS_LITE(NC_) fast(rank_reduce_fast_kernel<NC_, false, true>, fast_ring_words<NC_>())
  auto fast = [&](auto kern, size_t words) -> cudaError_t {
    const size_t smem = words * kThreads * sizeof(int64_t);
    if (smem > 48 * 1024) {
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem));
      if (e2 != cudaSuccess) return e2;
    }
    kern<<<grid, kThreads, smem, stream>>>(p);
    return cudaSuccess;
  };
  switch (bucket) {
    case 0: e = LUMOS_GEN(1); break;
    case 1: e = LUMOS_GEN(2); break;
    case 2: e = LUMOS_GEN(3); break;
    case 3: e = LUMOS_GEN(4); break;
    case 4: e = LUMOS_GEN(8); break;
    case 5: e = LUMOS_GEN(16); break;
    case 6: e = LUMOS_GEN(kMaxStreamsPerRank); break;
    case kReduceGenericBuckets + 0: e = LUMOS_FAST(0); break;
    case kReduceGenericBuckets + 1: e = LUMOS_FAST(1); break;
    case kReduceGenericBuckets + 2: e = LUMOS_FAST(2); break;
    case kReduceGenericBuckets + 3: e = LUMOS_FAST(3); break;
    case kReduceLiteBucket + 0: e = LUMOS_LITE(0); break;
    case kReduceLiteBucket + 1: e = LUMOS_LITE(1); break;
    case kReduceLiteBucket + 2: e = LUMOS_LITE(2); break;
    default: e = LUMOS_LITE(3); break;
  }
#undef LUMOS_GEN
#undef LUMOS_FAST
#undef LUMOS_LITE
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int max_streams_per_rank() { return kMaxStreamsPerRank; }

}  // namespace lumos
