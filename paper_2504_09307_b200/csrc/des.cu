// des.cu — exact event-driven replay on the device (one thread per scenario).
//
// A restatement of the reference Engine (/root/reference/proj/src/
// simulate.cpp:145-337) for the cases the straight-line walk does not cover:
//   * graphs outside the chained class (lanes not linked by fixed edges, rules
//     watching CPU lanes, ...) — every scenario runs here, and
//   * scenarios of chained graphs whose static sync-binding certificate failed
//     in the walk — only those are re-run here (fix-up mode).
// Per scenario: lane clocks, per-lane ready heaps keyed (original_start, id),
// a completion heap keyed (end, id); each iteration starts the smallest-key
// startable lane head (drain_startable) and then pops every completion at the
// next end time.  Deadlock -> status -1 (SimulationError in the reference).
//
// drain_startable scans every lane per start in the reference (O(V·L)).  Here
// the free lanes with a non-empty ready set sit in an indexed min-heap keyed
// by their head task, so a start costs O(log L):
//   * the smallest head is popped; if its rule fails the lane is parked (the
//     reference skips it in that scan and rescans it after the next start);
//   * a start with duration > 0 cannot unblock a parked head (its lane becomes
//     busy, and an event sync bound to it needs sim_end <= now), so parked
//     lanes stay parked; a zero-duration start (which also completes, and may
//     change heads) and every time advance return all parked lanes to the heap;
//   * a lane leaves the heap while busy and re-enters when its completion pops
//     (one positive-duration task per lane is in flight, so lane clock == the
//     end of that completion).
// The start order therefore equals the reference's scan order exactly.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"
#include "kernels.hpp"
#include "lumos_b200.h"

namespace lumos {

namespace {

struct DesScratch {
  int64_t* sim_start;  // [n]  (INT64_MIN = not started)
  int64_t* sim_end;    // [n]
  int64_t* comp_t;     // [n]  completion heap keys
  int64_t* clock;      // [nl]
  int64_t* ev;         // [2n] breakdown events
  int32_t* indeg;      // [n]
  int32_t* heap;       // [n]  per-lane ready heaps (lane_off regions)
  int32_t* comp_id;    // [n]
  int32_t* hsize;      // [nl]
  int32_t* lheap;      // [nl] free lanes with a non-empty ready set, min by head key
  int32_t* lpos;       // [nl] position in lheap; kOut / kParked
  int32_t* parked;     // [nl]
  int64_t* hkey;       // [nl] key (original_start) of each lane's ready head
  int32_t* hid;        // [nl] the head task (valid while hsize > 0)
};

constexpr int32_t kOut = -1, kParked = -2;

__device__ DesScratch carve(char* base, int32_t n, int32_t nl) {
  DesScratch s;
  int64_t* p64 = reinterpret_cast<int64_t*>(base);
  s.sim_start = p64;
  s.sim_end = p64 + n;
  s.comp_t = p64 + 2 * static_cast<int64_t>(n);
  s.clock = p64 + 3 * static_cast<int64_t>(n);
  s.ev = s.clock + nl;
  int32_t* p32 = reinterpret_cast<int32_t*>(s.ev + 2 * static_cast<int64_t>(n));
  s.indeg = p32;
  s.heap = p32 + n;
  s.comp_id = p32 + 2 * static_cast<int64_t>(n);
  s.hsize = p32 + 3 * static_cast<int64_t>(n);
  s.lheap = s.hsize + nl;
  s.lpos = s.lheap + nl;
  s.parked = s.lpos + nl;
  // the head cache after the int32 region, 8-byte aligned
  const uintptr_t end32 = reinterpret_cast<uintptr_t>(s.parked + nl);
  s.hkey = reinterpret_cast<int64_t*>((end32 + 7) & ~uintptr_t(7));
  s.hid = reinterpret_cast<int32_t*>(s.hkey + nl);
  return s;
}

struct Des {
  const DesParams& P;
  DesScratch s;
  int64_t now = 0;
  int32_t lsize = 0, nparked = 0;
  int32_t comp_cap = 0x7FFFFFFF;  // completion heap capacity (shared-memory mode: lanes)

  __device__ bool key_less(int32_t a, int32_t b) const {
    const int64_t ka = __ldg(&P.ostart[a]), kb = __ldg(&P.ostart[b]);
    return ka < kb || (ka == kb && a < b);
  }
  __device__ int32_t head(int32_t l) const { return s.hid[l]; }
  // lane order = head order, from the cached (key, id) of each head
  __device__ bool lane_less(int32_t a, int32_t b) const {
    const int64_t ka = s.hkey[a], kb = s.hkey[b];
    return ka < kb || (ka == kb && s.hid[a] < s.hid[b]);
  }
  __device__ void set_head(int32_t l, int32_t t) {
    s.hid[l] = t;
    s.hkey[l] = __ldg(&P.ostart[t]);
  }
  // lane heap: free lanes (clock <= now) with a non-empty ready set
  __device__ void lh_set(int32_t i, int32_t l) {
    s.lheap[i] = l;
    s.lpos[l] = i;
  }
  __device__ void lh_up(int32_t i) {
    const int32_t l = s.lheap[i];
    while (i > 0) {
      const int32_t p = (i - 1) >> 1;
      if (!lane_less(l, s.lheap[p])) break;
      lh_set(i, s.lheap[p]);
      i = p;
    }
    lh_set(i, l);
  }
  __device__ void lh_push(int32_t l) {
    lh_set(lsize, l);
    lh_up(lsize++);
  }
  __device__ int32_t lh_pop() {
    const int32_t top = s.lheap[0];
    s.lpos[top] = kOut;
    const int32_t n = --lsize;
    if (n > 0) {
      const int32_t l = s.lheap[n];
      int32_t i = 0;
      for (;;) {
        const int32_t a = 2 * i + 1, b = a + 1;
        int32_t m = -1, lm = l;
        if (a < n && lane_less(s.lheap[a], lm)) {
          m = a;
          lm = s.lheap[a];
        }
        if (b < n && lane_less(s.lheap[b], lm)) m = b;
        if (m < 0) break;
        lh_set(i, s.lheap[m]);
        i = m;
      }
      lh_set(i, l);
    }
    return top;
  }
  // parked lanes whose rule now holds go back to the lane heap; the others
  // stay parked (re-pushing them would only pop and park them again: between
  // here and their pop only positive-duration starts can happen, and those
  // cannot unblock a rule)
  __device__ void unpark_all() {
    int32_t keep = 0;
    for (int32_t k = 0; k < nparked; ++k) {
      const int32_t l = s.parked[k];
      if (rule_ok(head(l), l, now)) lh_push(l);
      else s.parked[keep++] = l;
    }
    nparked = keep;
  }
  // ready heap of lane l (min by (original_start, id)); a new head of a lane
  // in the lane heap moves it up, a free idle lane enters it
  __device__ void ready_push(int32_t l, int32_t t) {
    int32_t* h = s.heap + __ldg(&P.lane_off[l]);
    int32_t i = s.hsize[l]++;
    h[i] = t;
    while (i > 0) {
      const int32_t p = (i - 1) >> 1;
      if (!key_less(h[i], h[p])) break;
      const int32_t x = h[i];
      h[i] = h[p];
      h[p] = x;
      i = p;
    }
    if (i == 0) set_head(l, t);
    const int32_t pos = s.lpos[l];
    if (pos >= 0) {
      if (i == 0) lh_up(pos);
    } else if (pos == kOut && s.clock[l] <= now) {
      lh_push(l);
    }
  }
  __device__ void ready_pop(int32_t l) {
    int32_t* h = s.heap + __ldg(&P.lane_off[l]);
    const int32_t n = --s.hsize[l];
    h[0] = h[n];
    int32_t i = 0;
    for (;;) {
      const int32_t a = 2 * i + 1, b = a + 1;
      int32_t m = i;
      if (a < n && key_less(h[a], h[m])) m = a;
      if (b < n && key_less(h[b], h[m])) m = b;
      if (m == i) break;
      const int32_t x = h[i];
      h[i] = h[m];
      h[m] = x;
      i = m;
    }
    if (n > 0) set_head(l, h[0]);
  }
  __device__ bool comp_less(int32_t i, int32_t j) const {
    return s.comp_t[i] < s.comp_t[j] || (s.comp_t[i] == s.comp_t[j] && s.comp_id[i] < s.comp_id[j]);
  }
  __device__ void comp_swap(int32_t i, int32_t j) {
    const int64_t t = s.comp_t[i];
    s.comp_t[i] = s.comp_t[j];
    s.comp_t[j] = t;
    const int32_t d = s.comp_id[i];
    s.comp_id[i] = s.comp_id[j];
    s.comp_id[j] = d;
  }
  __device__ void comp_push(int32_t& size, int64_t t, int32_t id) {
    if (!LUMOS_OK(size < comp_cap)) return;
    int32_t i = size++;
    s.comp_t[i] = t;
    s.comp_id[i] = id;
    while (i > 0) {
      const int32_t p = (i - 1) >> 1;
      if (!comp_less(i, p)) break;
      comp_swap(i, p);
      i = p;
    }
  }
  __device__ void comp_pop(int32_t& size) {
    const int32_t n = --size;
    s.comp_t[0] = s.comp_t[n];
    s.comp_id[0] = s.comp_id[n];
    int32_t i = 0;
    for (;;) {
      const int32_t a = 2 * i + 1, b = a + 1;
      int32_t m = i;
      if (a < n && comp_less(a, m)) m = a;
      if (b < n && comp_less(b, m)) m = b;
      if (m == i) break;
      comp_swap(i, m);
      i = m;
    }
  }
  // rule_ok (simulate.cpp:202-217)
  __device__ bool rule_ok(int32_t t, int32_t own, int64_t now) const {
    const int32_t r = __ldg(&P.rule_of[t]);
    if (r < 0) return true;
    if (__ldg(&P.rule_kind[r]) == TS_RULE_EVENT_SYNC) {
      const int32_t b = __ldg(&P.rule_bound[r]);
      if (b < 0) return true;
      return s.sim_start[b] != kMinI64 && s.sim_end[b] <= now;
    }
    for (int32_t w = __ldg(&P.rule_wl_off[r]); w < __ldg(&P.rule_wl_off[r + 1]); ++w) {
      const int32_t lw = __ldg(&P.rule_wl[w]);
      if (s.clock[lw] > now) return false;
      const int32_t pending = s.hsize[lw] - (lw == own ? 1 : 0);
      if (pending > 0) return false;
    }
    return true;
  }
  __device__ void complete(int32_t t) {
    for (int32_t k = __ldg(&P.succ_off[t]); k < __ldg(&P.succ_off[t + 1]); ++k) {
      int32_t v = __ldg(&P.succ[k]);
      if (!LUMOS_OK(v >= 0 && v < P.n)) v = 0;
      if (--s.indeg[v] == 0) ready_push(__ldg(&P.lane_of[v]), v);
    }
  }
};

// heap sort of int64 keys (breakdown events)
__device__ void sort_i64(int64_t* a, int32_t n) {
  auto sift = [&](int32_t i, int32_t m) {
    for (;;) {
      int32_t c = 2 * i + 1;
      if (c >= m) break;
      if (c + 1 < m && a[c + 1] > a[c]) ++c;
      if (a[c] <= a[i]) break;
      const int64_t x = a[i];
      a[i] = a[c];
      a[c] = x;
      i = c;
    }
  };
  for (int32_t i = n / 2 - 1; i >= 0; --i) sift(i, n);
  for (int32_t m = n - 1; m > 0; --m) {
    const int64_t x = a[0];
    a[0] = a[m];
    a[m] = x;
    sift(0, m);
  }
}

__global__ void des_kernel(DesParams P) {
  extern __shared__ __align__(16) unsigned char des_smem[];
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= P.n_slots) return;
  const int32_t n = P.n, nl = P.nl;
  Des E{P, carve(P.scratch + static_cast<int64_t>(slot) * P.scratch_bytes, n, nl)};
  DesScratch& s = E.s;
  int32_t* const g_hsize = s.hsize;
  if (P.smem_lanes) {
    // one scenario per CTA: the per-lane state and the completion heap (at
    // most one positive-duration task in flight per lane) in shared memory,
    // so the heap walks of every start hit ~30-cycle loads instead of DRAM
    int64_t* sm64 = reinterpret_cast<int64_t*>(des_smem);
    s.clock = sm64;
    s.comp_t = sm64 + nl;
    int32_t* sm32 = reinterpret_cast<int32_t*>(sm64 + 2 * static_cast<int64_t>(nl));
    s.hsize = sm32;
    s.lheap = sm32 + nl;
    s.lpos = sm32 + 2 * nl;
    s.parked = sm32 + 3 * nl;
    s.comp_id = sm32 + 4 * nl;
    s.hid = sm32 + 5 * nl;
    s.hkey = reinterpret_cast<int64_t*>(
        (reinterpret_cast<uintptr_t>(sm32 + 6 * nl) + 7) & ~uintptr_t(7));
    E.comp_cap = nl;
  }
  for (int col = slot; col < P.sp.count; col += P.n_slots) {
    if (P.fixup && P.status[col] == 0) continue;
    ThreadScen ts;
    init_thread_scen(P.sp, col, ts);
    RtCol rc{};
    if (P.has_rt) rc = rt_col(P.rt, col);
    const int64_t W = P.W;
    E.now = W;
    E.lsize = 0;
    E.nparked = 0;
    for (int32_t l = 0; l < nl; ++l) {
      s.clock[l] = W;
      s.hsize[l] = 0;
      s.lpos[l] = kOut;
    }
    for (int32_t t = 0; t < n; ++t) {
      s.indeg[t] = __ldg(&P.indeg0[t]);
      s.sim_start[t] = kMinI64;
    }
    for (int32_t t = 0; t < n; ++t)
      if (s.indeg[t] == 0) E.ready_push(__ldg(&P.lane_of[t]), t);
    int32_t unstarted = n, comp = 0;
    bool dead = false;
    for (;;) {
      // drain_startable (simulate.cpp:239-255): smallest startable head first
      const int64_t now = E.now;
      while (E.lsize > 0) {
        const int32_t lane = E.lh_pop();
        const int32_t best = E.head(lane);
        if (!E.rule_ok(best, lane, now)) {  // the lane stalls behind its sync
          s.lpos[lane] = kParked;
          s.parked[E.nparked++] = lane;
          continue;
        }
        E.ready_pop(lane);
        const int64_t b = P.has_rt ? rt_task(P.rt, rc, best) : __ldg(&P.base[best]);
        const int64_t d = scenario_duration<-1>(P.sp, ts, best, b, __ldg(&P.cls[best]));
        s.sim_start[best] = now;
        s.sim_end[best] = now + d;
        --unstarted;
        if (d == 0) {
          E.complete(best);
          if (s.lpos[lane] == kOut && s.hsize[lane] > 0) E.lh_push(lane);
          E.unpark_all();
        } else {
          s.clock[lane] = now + d;
          E.comp_push(comp, now + d, best);
        }
      }
      if (comp == 0) {
        dead = unstarted != 0;
        break;
      }
      // advance to the next completion time (completing does not read now)
      const int64_t t2 = s.comp_t[0];
      E.now = t2;
      while (comp > 0 && s.comp_t[0] == t2) {
        const int32_t done = s.comp_id[0];
        E.comp_pop(comp);
        E.complete(done);
        const int32_t l = __ldg(&P.lane_of[done]);
        if (s.lpos[l] == kOut && s.hsize[l] > 0) E.lh_push(l);
      }
      E.unpark_all();
    }
    if (dead) {  // span_hi carries the blocked-task count for the error message
      P.status[col] = -1;
      P.span_hi[col] = unstarted;
      if (P.smem_lanes)  // the ready-set sizes, for the host's deadlock witness
        for (int32_t l = 0; l < nl; ++l) g_hsize[l] = s.hsize[l];
      continue;
    }
    int64_t lo = W, hi = W;
    if (n > 0) {
      lo = kMaxI64;
      hi = kMinI64;
      for (int32_t t = 0; t < n; ++t) {
        lo = imin(lo, s.sim_start[t]);
        hi = imax(hi, s.sim_end[t]);
        if (P.out_start) P.out_start[static_cast<int64_t>(t) * P.ld + col] = s.sim_start[t];
        if (P.out_fin) P.out_fin[static_cast<int64_t>(t) * P.ld + col] = s.sim_end[t];
      }
      if (hi < lo) hi = lo;
    }
    P.span_lo[col] = lo;
    P.span_hi[col] = hi;
    P.status[col] = 1;
    if (!P.breakdown && !P.stream_busy && !P.util) continue;
    // per-rank breakdown (metrics.cpp:43-103) on sorted interval endpoints
    int64_t wend = P.window_end;
    if (W + (hi - lo) > wend) wend = W + (hi - lo);
    if (wend < W) wend = W;
    // Each stream's events are appended in its task order; a stream runs one
    // task at a time, so when that order is also the execution order (always
    // for chained lanes) every run is sorted by time and the sweep merges the
    // runs instead of sorting.  Events at equal times may be taken in any
    // order: spans between them are empty.
    constexpr int kMaxRuns = 8;
    int32_t l = 0;
    while (l < nl) {
      const int32_t r = __ldg(&P.lane_rank[l]);
      int32_t ne = 0;
      int32_t l1 = l;
      int32_t run_b[kMaxRuns + 1];
      int nrun = 0;
      bool merge = true;
      for (; l1 < nl && __ldg(&P.lane_rank[l1]) == r; ++l1) {
        const int32_t st = __ldg(&P.lane_stream[l1]);
        if (st < 0) continue;
        if (nrun < kMaxRuns) run_b[nrun++] = ne;
        else merge = false;
        int64_t busy = 0, last = INT64_MIN;
        for (int32_t k = __ldg(&P.lane_off[l1]); k < __ldg(&P.lane_off[l1 + 1]); ++k) {
          const int32_t t = __ldg(&P.lane_tasks[k]);
          const int64_t a = imax(s.sim_start[t], W), b = imin(s.sim_end[t], wend);
          if (a >= b) continue;
          busy += b - a;
          const int64_t c = __ldg(&P.is_comm[t]) ? 2 : 0;  // 0 compute, 2 comm; +1 = end
          if (!LUMOS_OK(ne + 2 <= 2 * n)) break;
          merge = merge && a >= last;
          last = b;
          s.ev[ne++] = ((a - W) << 2) | c;
          s.ev[ne++] = ((b - W) << 2) | (c + 1);
        }
        if (P.stream_busy) P.stream_busy[static_cast<int64_t>(col) * P.n_streams + st] = busy;
      }
      run_b[nrun] = ne;
      if (!merge) sort_i64(s.ev, ne);
      int compute = 0, commc = 0;
      int64_t prev = W, ec = 0, em = 0, ov = 0, ot = 0;
      BinAcc ua;
      if (P.util) ua.init(P.util + (static_cast<int64_t>(col) * P.n_ranks + r) * P.util_max_bins,
                          P.util_bw, P.util_max_bins);
      auto account = [&](int64_t upto) {
        if (upto <= prev) return;
        const int64_t span = upto - prev;
        if (compute > 0 && commc > 0) ov += span;
        else if (compute > 0) ec += span;
        else if (commc > 0) em += span;
        else ot += span;
        if (P.util && (compute > 0 || commc > 0)) ua.add(prev - W, upto - W, 1);
        prev = upto;
      };
      auto event = [&](int64_t e) {
        account(W + (e >> 2));
        switch (e & 3) {
          case 0: ++compute; break;
          case 1: --compute; break;
          case 2: ++commc; break;
          default: --commc; break;
        }
      };
      if (merge) {
        int32_t pos[kMaxRuns];
        for (int j = 0; j < nrun; ++j) pos[j] = run_b[j];
        for (;;) {
          int best = -1;
          int64_t bt = 0;
          for (int j = 0; j < nrun; ++j) {
            if (pos[j] >= run_b[j + 1]) continue;
            const int64_t tj = s.ev[pos[j]] >> 2;
            if (best < 0 || tj < bt) {
              best = j;
              bt = tj;
            }
          }
          if (best < 0) break;
          event(s.ev[pos[best]++]);
        }
      } else {
        for (int32_t k = 0; k < ne; ++k) event(s.ev[k]);
      }
      account(wend);
      if (P.util) ua.flush();
      if (P.breakdown) {
        int64_t* row = P.breakdown + (static_cast<int64_t>(col) * P.n_ranks + r) * 5;
        row[0] = wend - W;
        row[1] = ec;
        row[2] = em;
        row[3] = ov;
        row[4] = ot;
      }
      l = l1;
    }
  }
}

}  // namespace

#ifdef LUMOS_DEBUG_BOUNDS
int debug_bounds_status_des() {
  int v = 0, zero = 0;
  if (cudaMemcpyFromSymbol(&v, lumos_bounds_fail, sizeof(int)) != cudaSuccess) return -1;
  cudaMemcpyToSymbol(lumos_bounds_fail, &zero, sizeof(int));
  return v;
}
#else
int debug_bounds_status_des() { return 0; }
#endif

size_t des_scratch_bytes(int32_t n, int32_t nl) {
  const size_t b = (static_cast<size_t>(n) * 3 + nl + 2 * static_cast<size_t>(n)) * 8 +
                   (static_cast<size_t>(n) * 3 + 4 * static_cast<size_t>(nl)) * 4 + 8 +
                   static_cast<size_t>(nl) * 12;  // + the head cache
  return (b + 255) / 256 * 256;
}

size_t des_smem_bytes(int32_t nl) { return static_cast<size_t>(nl) * 48 + 8; }

cudaError_t launch_des(const DesParams& p, cudaStream_t stream) {
  if (p.n_slots <= 0 || p.sp.count <= 0) return cudaSuccess;
  if (p.smem_lanes) {
    const size_t smem = des_smem_bytes(p.nl);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(des_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return e;
    }
    des_kernel<<<p.n_slots, 1, smem, stream>>>(p);
    return cudaGetLastError();
  }
  const int threads = 64;
  des_kernel<<<(p.n_slots + threads - 1) / threads, threads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace lumos
