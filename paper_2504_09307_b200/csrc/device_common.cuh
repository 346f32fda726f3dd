// device_common.cuh — device helpers shared by the replay kernels: the
// counter-based scenario duration formula (K4 semantics) and int64 helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "kernels.hpp"
#include "lumos_b200.h"
#include "program.hpp"

namespace lumos {

// Debug builds (-DLUMOS_DEBUG_BOUNDS, `make debug`) check every slot,
// mailbox, ring and output index the kernels compute; a failed check records
// the source line in lumos_bounds_fail (read and cleared by the C ABI after
// each call, which then fails the call), prints once, and redirects the
// access to a safe location instead of faulting.  compute-sanitizer is closed
// on this pool; these checks are the memory-safety evidence.
#ifdef LUMOS_DEBUG_BOUNDS
static __device__ int lumos_bounds_fail = 0;  // one per translation unit
#define LUMOS_OK(cond)                                                              \
  ((cond) ? true                                                                    \
          : (atomicCAS(&lumos_bounds_fail, 0, __LINE__) == 0                        \
                 ? (printf("lumos bounds check failed: %s:%d (%s)\n", __FILE__, __LINE__, \
                           #cond),                                                  \
                    false)                                                          \
                 : false))
#else
#define LUMOS_OK(cond) true
#endif

namespace {

constexpr int64_t kMinI64 = INT64_MIN;
constexpr int64_t kMaxI64 = INT64_MAX;
__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ void philox2x32_10(uint32_t& x0, uint32_t& x1, uint32_t key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi = __umulhi(0xD256D193u, x0);
    const uint32_t lo = 0xD256D193u * x0;
    x0 = hi ^ key ^ x1;
    x1 = lo;
    key += 0x9E3779B9u;
  }
}

// the same permutation with the round keys precomputed (kernel-parameter
// constants: each round is one IMAD.WIDE and one three-input XOR)
__device__ __forceinline__ void philox2x32_10_rk(uint32_t& x0, uint32_t& x1,
                                                 const uint32_t (&rk)[10]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi = __umulhi(0xD256D193u, x0);
    const uint32_t lo = 0xD256D193u * x0;
    x0 = hi ^ rk[r] ^ x1;
    x1 = lo;
  }
}

// (a * num + den/2) / den for a >= 0, num >= 0 (transform.cpp:38-43)
__device__ __forceinline__ int64_t mul_div_nonneg(int64_t a, int64_t num, int64_t den,
                                                  int den_shift) {
  const uint64_t ua = static_cast<uint64_t>(a), un = static_cast<uint64_t>(num);
  uint64_t lo = ua * un;
  uint64_t hi = __umul64hi(ua, un);
  const uint64_t half = static_cast<uint64_t>(den / 2);
  const uint64_t lo2 = lo + half;
  hi += lo2 < lo ? 1 : 0;
  lo = lo2;
  if (den_shift >= 0) {
    if (den_shift == 0) return static_cast<int64_t>(lo);
    return static_cast<int64_t>((lo >> den_shift) | (hi << (64 - den_shift)));
  }
  const uint64_t ud = static_cast<uint64_t>(den);
  if (hi == 0) return static_cast<int64_t>(lo / ud);
  // 128 / 64 long division (rare: products beyond 2^64)
  uint64_t q = 0, r = hi % ud;
  for (int b = 63; b >= 0; --b) {
    const bool top = (r >> 63) != 0;
    r = (r << 1) | ((lo >> b) & 1u);
    if (top || r >= ud) {
      r -= ud;
      q |= 1ull << b;
    }
  }
  return static_cast<int64_t>(q);
}

struct ThreadScen {
  int64_t scen;    // global scenario id
  int32_t col;     // column in the batch
  int32_t num[kMaxClasses];
};

__device__ __forceinline__ int32_t class_num(const ScenarioParams& sp, int64_t scen, int col,
                                             int cls) {
  if (sp.scale_num) return sp.scale_num[static_cast<int64_t>(col) * sp.n_classes + cls];
  uint32_t x0 = static_cast<uint32_t>(cls), x1 = static_cast<uint32_t>(scen);
  philox2x32_10(x0, x1, sp.key_cls);
  return sp.scale_lo + static_cast<int32_t>((static_cast<uint64_t>(x0) * sp.scale_span) >> 32);
}

// K4 semantics: the scenario's duration of one task (see lumos_b200.h).
// kMode < 0: decided at run time from sp.mode.
// Scenario durations (K4 semantics): class scale, then jitter
//   d' = d == 0 ? 0 : max(1, llround(d * (1 + u))),  u = 2j * (w * 2^-32) - j
// with w = word (s & 1) of Philox2x32-10(ctr = (task, s >> 1); seed), so one
// Philox call serves the scenario pair (2p, 2p + 1).
// out of line: keeps the general 128-bit path's registers off the walk loop
__device__ __noinline__ int64_t mul_div_slow(int64_t a, int64_t num, int64_t den, int den_shift) {
  return mul_div_nonneg(a, num, den, den_shift);
}
__device__ __forceinline__ int64_t class_scaled_num(const ScenarioParams& sp, int64_t d,
                                                    int32_t num) {
  // power-of-two denominator and a 32-bit duration (every duration of a
  // uint32-window walk): one 32x32 -> 64 multiply, add, shift
  if (sp.den_shift >= 0 && (static_cast<uint64_t>(d) >> 32) == 0 && num >= 0)
    return static_cast<int64_t>(
        (static_cast<uint64_t>(static_cast<uint32_t>(d)) * static_cast<uint32_t>(num) +
         static_cast<uint64_t>(sp.scale_den / 2)) >> sp.den_shift);
  return mul_div_slow(d, num, sp.scale_den, sp.den_shift);
}
__device__ __forceinline__ int64_t class_scaled(const ScenarioParams& sp, const ThreadScen& ts,
                                                int64_t d, int cls) {
  int32_t num = ts.num[0];
  if (cls == 1) num = ts.num[1];
  if (cls == 2) num = ts.num[2];
  if (cls == 3) num = ts.num[3];
  return class_scaled_num(sp, d, num);
}
__device__ __forceinline__ uint32_t jitter_word(const ScenarioParams& sp, int64_t task,
                                                int64_t scen) {
  uint32_t x0 = static_cast<uint32_t>(task), x1 = static_cast<uint32_t>(scen >> 1);
  philox2x32_10_rk(x0, x1, sp.rk_jit);
  return (scen & 1) ? x1 : x0;
}
// the words of two scenarios of one pair (s0 >> 1 == s1 >> 1): one Philox call
__device__ __forceinline__ void jitter_words2(const ScenarioParams& sp, int64_t task,
                                              int64_t s0, int64_t s1, uint32_t& w0,
                                              uint32_t& w1) {
  uint32_t x0 = static_cast<uint32_t>(task), x1 = static_cast<uint32_t>(s0 >> 1);
  philox2x32_10_rk(x0, x1, sp.rk_jit);
  w0 = (s0 & 1) ? x1 : x0;
  w1 = (s1 & 1) ? x1 : x0;
}
// max(1, llround(d * (1 + u))) for d > 0; 0 for d == 0
__device__ __forceinline__ int64_t jitter_apply(const ScenarioParams& sp, int64_t d, uint32_t w) {
  // two_j * (w * 2^-32) == (two_j * 2^-32) * w exactly (power-of-two scaling
  // commutes with rounding while nothing is subnormal)
  const double u = __dadd_rn(__dmul_rn(sp.two_j_ulp, __uint2double_rn(w)), sp.neg_j);
  const double f = __dadd_rn(1.0, u);
  const double p = __dmul_rn(__ll2double_rn(d), f);
  // max(1, llround(p)) for p >= 0: below 1.5 the answer is 1; on [1.5, 2^52)
  // p + 0.5 is exact so floor(p + 0.5) is round-half-up; from 2^52 up p is
  // already an integer
  const int64_t r = __double2ll_rd(p >= 0x1.0p52 ? p : __dadd_rn(p, 0.5));
  return d == 0 ? 0 : (r < 1 ? 1 : r);
}

// jitter_apply for a uint32 walk, where the host has proven every jittered
// duration < 2^32 (capi.cpp rel32 bound): p < 2^32 < 2^52, so p + 0.5 is
// exact and floor fits an unsigned 32-bit conversion — the same value as
// jitter_apply with 32-bit compares and no 2^52 guard
__device__ __forceinline__ uint32_t jitter_apply_u32(const ScenarioParams& sp, double dd, bool dz,
                                                     uint32_t w) {
  const double u = __dadd_rn(__dmul_rn(sp.two_j_ulp, __uint2double_rn(w)), sp.neg_j);
  const double f = __dadd_rn(1.0, u);
  const double p = __dmul_rn(dd, f);
  const uint32_t r = __double2uint_rd(__dadd_rn(p, 0.5));
  return dz ? 0u : (r < 1u ? 1u : r);
}

template <int kMode>
__device__ __forceinline__ int64_t scenario_duration(const ScenarioParams& sp,
                                                     const ThreadScen& ts, int64_t task,
                                                     int64_t base, int cls) {
  const int mode = kMode >= 0 ? kMode : sp.mode;
  if (mode & kModeExplicit) return __ldcs(sp.durations + task * sp.durations_ld + ts.col);
  int64_t d = base;
  if (mode & kModeScale) d = class_scaled(sp, ts, d, cls);
  if (mode & kModeJitter) {
    if (d == 0) return 0;
    return jitter_apply(sp, d, jitter_word(sp, task, ts.scen));
  }
  return d;
}

// ---- what-if retime (transform.cpp:219-349 through apply_whatif :713-760):
// change_hidden then scale_dp with the analytical collective cost
// (cost.cpp:40-62), evaluated in double with explicitly rounded operations in
// the reference's order, then llround (round half away from zero).
__device__ __forceinline__ int64_t llround_exact(double t) {
  if (t >= 0x1.0p52 || t <= -0x1.0p52) return static_cast<int64_t>(t);  // integral
  const int64_t r = __double2ll_rz(t);
  const double fr = __dadd_rn(t, -static_cast<double>(r));  // exact (Sterbenz)
  return fr >= 0.5 ? r + 1 : (fr <= -0.5 ? r - 1 : r);
}
// collective_cost_us: max(0, llround(alpha + bytes * scale(c, g) / beta))
__device__ __forceinline__ int64_t coll_cost(bool allreduce, int64_t bytes, int32_t g,
                                             double alpha, double bpu) {
  double scale = 1.0;  // SendRecv
  if (allreduce) {
    const double gd = static_cast<double>(g);
    scale = __ddiv_rn(__dmul_rn(2.0, __dadd_rn(gd, -1.0)), gd);
  }
  const double t = __dadd_rn(alpha, __ddiv_rn(__dmul_rn(static_cast<double>(bytes), scale), bpu));
  const int64_t r = llround_exact(t);
  return r < 0 ? 0 : r;
}

// per-scenario retime inputs
struct RtCol {
  double alpha, bpu;
  int32_t tdp;
  bool dp, hid;
  int64_t tm[3];
};
__device__ __forceinline__ RtCol rt_col(const RetimeParams& P, int col) {
  RtCol c;
  c.alpha = P.alpha[col];
  c.bpu = P.bpu[col];
  c.tdp = P.target_dp ? P.target_dp[col] : P.source_dp;
  c.dp = P.target_dp && c.tdp != P.source_dp;
  for (int k = 0; k < 3; ++k)
    c.tm[k] = P.target_model ? P.target_model[3 * static_cast<int64_t>(col) + k] : P.src_model[k];
  // change_hidden is a no-op unless d_model or d_ffn change (transform.cpp:282)
  c.hid = P.target_model && (c.tm[0] != P.src_model[0] || c.tm[1] != P.src_model[1]);
  return c;
}
// the retimed duration of task t before class scale and jitter
__device__ __forceinline__ int64_t rt_task(const RetimeParams& P, const RtCol& c, int32_t t) {
  int64_t d = P.base[t];
  const uint8_t kd = P.kind[t];
  if (kd == TS_RT_NONE || !(c.hid || c.dp)) return d;
  int64_t bytes = P.bytes[t];
  if (c.hid) {
    if (kd == TS_RT_GEMM) {
      const int64_t* mnk = P.mnk + 3 * static_cast<int64_t>(t);
      int64_t nd[3];
      for (int k = 0; k < 3; ++k)
        nd[k] = mnk[k] == P.src_model[0] ? c.tm[0] : (mnk[k] == P.src_model[1] ? c.tm[1] : mnk[k]);
      d = mul_div_nonneg(d, nd[0] * nd[1] * nd[2], mnk[0] * mnk[1] * mnk[2], -1);
    } else if (kd == TS_RT_OPT) {
      d = mul_div_nonneg(d, c.tm[2], P.src_model[2], -1);
    } else if (kd == TS_RT_ALLREDUCE && bytes >= 0) {  // no byte count: left as is
      bytes = mul_div_nonneg(bytes, c.tm[2], P.src_model[2], -1);
      d = coll_cost(true, bytes, P.group[t], c.alpha, c.bpu);
    } else if (kd == TS_RT_P2P_SEND || kd == TS_RT_P2P_RECV) {
      bytes = mul_div_nonneg(bytes, c.tm[0], P.src_model[0], -1);
      if (kd == TS_RT_P2P_SEND) d = coll_cost(false, bytes, 2, c.alpha, c.bpu);
      // a receive keeps its recorded duration (arrival skew), transform.cpp:342
    }
  }
  if (c.dp && kd == TS_RT_ALLREDUCE && P.group[t] == P.source_dp)
    d = coll_cost(true, bytes, c.tdp, c.alpha, c.bpu);
  return d;
}

__device__ __forceinline__ void init_thread_scen(const ScenarioParams& sp, int col, ThreadScen& ts) {
  ts.col = col;
  ts.scen = sp.first + col;
#pragma unroll
  for (int c = 0; c < kMaxClasses; ++c)
    ts.num[c] = (sp.mode & kModeScale) && c < sp.n_classes_eff ? class_num(sp, ts.scen, col, c) : 0;
}

__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

// Utilization bins (metrics.cpp:105-155): adds covered microseconds of
// [from, to) (window-relative, non-decreasing `from` across calls) to the bins
// of width bw, accumulating the current bin in a register and flushing it to
// row[bin] (read-modify-write: several accumulators of one thread may share a
// row).  sign -1 subtracts (the overlap term of |A u U| = |A| + |U| - |A n U|).
struct BinAcc {
  int64_t* row;
  int64_t bw, bin_end, acc;
  int32_t bin, max_bins;
  __device__ __forceinline__ void init(int64_t* r, int64_t w, int32_t mb) {
    row = r;
    bw = w;
    bin_end = w;
    acc = 0;
    bin = 0;
    max_bins = mb;
  }
  __device__ __forceinline__ void flush() {
    if (acc != 0 && bin < max_bins) row[bin] += acc;
    acc = 0;
  }
  __device__ __forceinline__ void add(int64_t from, int64_t to, int64_t sign) {
    while (from < to) {
      while (from >= bin_end) {
        flush();
        ++bin;
        bin_end += bw;
      }
      const int64_t e = to < bin_end ? to : bin_end;
      acc += sign * (e - from);
      from = e;
    }
  }
};

}  // namespace
}  // namespace lumos
