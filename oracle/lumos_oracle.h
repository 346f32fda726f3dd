/*
 * lumos_oracle.h — CPU restatement of the reference replay path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the parity tests, smoke() and
 * bench.py's cpu_baseline leg compare the CUDA path against.  The product
 * (paper_2504_09307_b200/) never includes, links or calls anything here.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - against the reference's own golden vectors (test_simulator.cpp:58-195,
 *     test_metrics.cpp:38-58, test_synth.cpp:60-115 known answers), and
 *   - against the compiled, unmodified reference in oracle/_ref/ on the same
 *     inputs (generator graphs, the reference's random_graph fuzz set).
 *
 * Reference files cited below are relative to /root/reference/proj.
 */
#ifndef LUMOS_ORACLE_H
#define LUMOS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CSR/SoA restatement of tracesim::ExecutionGraph (include/tracesim/build.hpp:73-85,
 * include/tracesim/types.hpp:48-87).  lane_kind: 0 = CpuThread, 1 = CudaStream
 * (types.hpp:41).  rule_kind: 0 = StreamSync, 1 = DeviceSync, 2 = EventSync
 * (build.hpp:47).  rule_bound = -1 when the EventSync has no bound task. */
typedef struct {
  int32_t n;
  const int64_t* duration;
  const int64_t* original_start;
  const int32_t* rank;
  const int32_t* lane_kind;
  const int32_t* lane;
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
  int64_t window_start;
} orc_graph;

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_DEADLOCK = 2, ORC_NOMEM = 3 };

/* Restates tracesim::simulate (src/simulate.cpp:341-347): validate_graph's
 * error checks (:26-125) then the discrete-event Engine (:145-337).
 * Writes sim_start/sim_end per task id and span = {start, end, makespan}. */
int orc_simulate(const orc_graph* g, int64_t* sim_start, int64_t* sim_end, int64_t span[3]);

/* Restates breakdown_by_rank (src/metrics.cpp:43-103) for the GPU intervals of
 * one rank: out = {total, exposed_compute, exposed_comm, overlapped, other}. */
void orc_breakdown_rank(int32_t n, const int32_t* rank, const int32_t* lane_kind,
                        const uint8_t* is_comm, const int64_t* start, const int64_t* end,
                        int32_t which_rank, int64_t window_start, int64_t window_end,
                        int64_t out[5]);

/* ---- scenario durations (the "manipulation kernel" K4 semantics) ---------
 * Counter-based: every (scenario, task) duration is a pure function of the
 * spec, so any shard/tile of scenarios reproduces bit-for-bit.
 *   1. class scale  d = mul_div(d, num, den)       (src/transform.cpp:38-43)
 *      num = lo + floor(r * (hi - lo + 1) / 2^32), r = Philox2x32-10 word
 *   2. jitter       d = d == 0 ? 0 : max(1, llround(d * (1 + u)))
 *                   u = -j + 2j * U01              (src/synth.cpp:150-155)
 *                   U01 = w * 2^-32, w = word (s & 1) of
 *                   Philox2x32-10(ctr = (task, s >> 1), key(seed))
 * Philox2x32-10 (Salmon et al., SC'11, Random123 constants).               */
typedef struct {
  uint64_t seed;
  double jitter;       /* 0 disables */
  int32_t scale_lo;    /* class scale numerator range [lo, hi]; den <= 0 disables */
  int32_t scale_hi;
  int32_t scale_den;
  int32_t reserved;
} orc_scenarios;

void orc_philox2x32_10(uint32_t ctr0, uint32_t ctr1, uint32_t key, uint32_t out[2]);
int64_t orc_mul_div(int64_t a, int64_t num, int64_t den);
int32_t orc_class_num(const orc_scenarios* sc, int64_t scenario, int32_t cls);
int64_t orc_scenario_duration(const orc_scenarios* sc, int64_t scenario, int32_t task,
                              int64_t base, int32_t cls);
/* Fills dur[t] for one scenario. */
void orc_fill_durations(const orc_scenarios* sc, int64_t scenario, int32_t n,
                        const int64_t* base, const uint8_t* cls, int64_t* dur);

#ifdef __cplusplus
}
#endif

#endif /* LUMOS_ORACLE_H */
