/*
 * lumos_oracle.c — CPU restatement of the reference replay path (TEST
 * INFRASTRUCTURE ONLY; see lumos_oracle.h).  Plain C, single-threaded,
 * written for obviousness.  Each function cites the reference code it restates
 * (paths relative to /root/reference/proj).
 */
#include "lumos_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- helpers */

typedef struct {
  int64_t a; /* primary key  */
  int32_t b; /* secondary key */
} key_t2;

static int key_less(key_t2 x, key_t2 y) { return x.a < y.a || (x.a == y.a && x.b < y.b); }

/* binary min-heap of (a, b) keys */
typedef struct {
  key_t2* v;
  int32_t n;
} heap_t;

static void heap_push(heap_t* h, key_t2 k) {
  int32_t i = h->n++;
  h->v[i] = k;
  while (i > 0) {
    int32_t p = (i - 1) / 2;
    if (!key_less(h->v[i], h->v[p])) break;
    key_t2 t = h->v[i];
    h->v[i] = h->v[p];
    h->v[p] = t;
    i = p;
  }
}

static key_t2 heap_pop(heap_t* h) {
  key_t2 top = h->v[0];
  h->v[0] = h->v[--h->n];
  int32_t i = 0;
  for (;;) {
    int32_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && key_less(h->v[l], h->v[m])) m = l;
    if (r < h->n && key_less(h->v[r], h->v[m])) m = r;
    if (m == i) break;
    key_t2 t = h->v[i];
    h->v[i] = h->v[m];
    h->v[m] = t;
    i = m;
  }
  return top;
}

typedef struct {
  int32_t rank, kind, lane;
} proc_t;

static int proc_cmp(const void* x, const void* y) {
  const proc_t* a = (const proc_t*)x;
  const proc_t* b = (const proc_t*)y;
  if (a->rank != b->rank) return a->rank < b->rank ? -1 : 1;
  if (a->kind != b->kind) return a->kind < b->kind ? -1 : 1;
  if (a->lane != b->lane) return a->lane < b->lane ? -1 : 1;
  return 0;
}

static int32_t find_proc(const proc_t* lanes, int32_t nl, proc_t p) {
  int32_t lo = 0, hi = nl - 1;
  while (lo <= hi) {
    int32_t mid = (lo + hi) / 2;
    int c = proc_cmp(&lanes[mid], &p);
    if (c == 0) return mid;
    if (c < 0)
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  return -1;
}

/* ------------------------------------------------------ validate_graph */

/* Error-level checks of validate_graph (src/simulate.cpp:26-125): negative
 * durations, bad edge endpoints / self loops, bad rule tasks, Kahn cycle. */
static int validate(const orc_graph* g) {
  const int32_t n = g->n;
  if (n < 0 || g->n_edges < 0 || g->n_rules < 0) return 0;
  for (int32_t i = 0; i < n; ++i)
    if (g->duration[i] < 0) return 0;
  for (int64_t e = 0; e < g->n_edges; ++e) {
    int32_t u = g->edge_from[e], v = g->edge_to[e];
    if (u < 0 || u >= n || v < 0 || v >= n || u == v) return 0;
  }
  for (int32_t r = 0; r < g->n_rules; ++r) {
    int32_t w = g->rule_task[r], b = g->rule_bound[r];
    if (w < 0 || w >= n || (b >= 0 && b >= n)) return 0;
  }
  if (n == 0) return 1;
  int32_t* indeg = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  int32_t* off = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n_edges + 1));
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t e = 0; e < g->n_edges; ++e) {
    off[g->edge_from[e] + 1]++;
    indeg[g->edge_to[e]]++;
  }
  for (int32_t i = 0; i < n; ++i) off[i + 1] += off[i];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  memcpy(fill, off, sizeof(int32_t) * (size_t)n);
  for (int64_t e = 0; e < g->n_edges; ++e) adj[fill[g->edge_from[e]]++] = g->edge_to[e];
  int32_t qh = 0, qt = 0;
  for (int32_t i = 0; i < n; ++i)
    if (indeg[i] == 0) queue[qt++] = i;
  while (qh < qt) {
    int32_t u = queue[qh++];
    for (int32_t k = off[u]; k < off[u + 1]; ++k)
      if (--indeg[adj[k]] == 0) queue[qt++] = adj[k];
  }
  int ok = qt == n;
  free(indeg);
  free(off);
  free(adj);
  free(queue);
  free(fill);
  return ok;
}

/* ------------------------------------------------------------- simulate */

int orc_simulate(const orc_graph* g, int64_t* sim_start, int64_t* sim_end, int64_t span[3]) {
  if (!validate(g)) return ORC_INVALID;
  const int32_t n = g->n;
  if (n <= 0) {
    span[0] = span[1] = g->window_start;
    span[2] = 0;
    return ORC_OK;
  }

  /* Engine ctor (src/simulate.cpp:162-196): lanes = distinct processors in
   * ProcessorId order (types.hpp:48-54), clocks at the window start. */
  proc_t* lanes = (proc_t*)malloc(sizeof(proc_t) * (size_t)n);
  for (int32_t i = 0; i < n; ++i) {
    lanes[i].rank = g->rank[i];
    lanes[i].kind = g->lane_kind[i];
    lanes[i].lane = g->lane[i];
  }
  qsort(lanes, (size_t)n, sizeof(proc_t), proc_cmp);
  int32_t nl = 0;
  for (int32_t i = 0; i < n; ++i)
    if (nl == 0 || proc_cmp(&lanes[nl - 1], &lanes[i]) != 0) lanes[nl++] = lanes[i];

  int32_t* lane_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* lane_count = (int32_t*)calloc((size_t)nl, sizeof(int32_t));
  for (int32_t i = 0; i < n; ++i) {
    proc_t p = {g->rank[i], g->lane_kind[i], g->lane[i]};
    lane_of[i] = find_proc(lanes, nl, p);
    lane_count[lane_of[i]]++;
  }
  int64_t now = g->window_start;
  int64_t* clock = (int64_t*)malloc(sizeof(int64_t) * (size_t)nl);
  heap_t* ready = (heap_t*)malloc(sizeof(heap_t) * (size_t)nl);
  for (int32_t l = 0; l < nl; ++l) {
    clock[l] = now;
    ready[l].v = (key_t2*)malloc(sizeof(key_t2) * (size_t)lane_count[l]);
    ready[l].n = 0;
  }

  int32_t* indeg = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  int32_t* off = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n_edges + 1));
  for (int64_t e = 0; e < g->n_edges; ++e) {
    off[g->edge_from[e] + 1]++;
    indeg[g->edge_to[e]]++;
  }
  for (int32_t i = 0; i < n; ++i) off[i + 1] += off[i];
  {
    int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    memcpy(fill, off, sizeof(int32_t) * (size_t)n);
    for (int64_t e = 0; e < g->n_edges; ++e) adj[fill[g->edge_from[e]]++] = g->edge_to[e];
    free(fill);
  }

  /* rule_of: a later rule on the same task overrides (simulate.cpp:180-187);
   * watched processors that own no task are dropped. */
  int32_t* rule_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int32_t i = 0; i < n; ++i) rule_of[i] = -1;
  int32_t nw_total = g->n_rules ? g->rule_watch_off[g->n_rules] : 0;
  int32_t* wl = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nw_total + 1));
  int32_t* wl_off = (int32_t*)calloc((size_t)g->n_rules + 1, sizeof(int32_t));
  {
    int32_t k = 0;
    for (int32_t r = 0; r < g->n_rules; ++r) {
      rule_of[g->rule_task[r]] = r;
      for (int32_t w = g->rule_watch_off[r]; w < g->rule_watch_off[r + 1]; ++w) {
        proc_t p = {g->watch_rank[w], g->watch_kind[w], g->watch_lane[w]};
        int32_t l = find_proc(lanes, nl, p);
        if (l >= 0) wl[k++] = l;
      }
      wl_off[r + 1] = k;
    }
  }

  char* started = (char*)calloc((size_t)n, 1);
  heap_t comp;
  comp.v = (key_t2*)malloc(sizeof(key_t2) * (size_t)n);
  comp.n = 0;
  int32_t unstarted = n;
  int status = ORC_OK;

  for (int32_t i = 0; i < n; ++i)
    if (indeg[i] == 0) heap_push(&ready[lane_of[i]], (key_t2){g->original_start[i], i});

  for (;;) {
    /* drain_startable (simulate.cpp:239-255): start the smallest-key lane head
     * among idle lanes whose head passes its rule, until none is left. */
    for (;;) {
      int32_t best = -1, best_lane = -1;
      key_t2 best_key = {0, 0};
      for (int32_t l = 0; l < nl; ++l) {
        if (clock[l] > now || ready[l].n == 0) continue;
        key_t2 head = ready[l].v[0];
        int32_t t = head.b;
        /* rule_ok (simulate.cpp:202-217) */
        int32_t r = rule_of[t];
        int ok = 1;
        if (r >= 0) {
          if (g->rule_kind[r] == 2) {
            int32_t b = g->rule_bound[r];
            if (b >= 0) ok = started[b] && sim_end[b] <= now;
          } else {
            for (int32_t w = wl_off[r]; w < wl_off[r + 1] && ok; ++w) {
              int32_t lw = wl[w];
              if (clock[lw] > now) ok = 0;
              int32_t pending = ready[lw].n - (lw == l ? 1 : 0);
              if (pending > 0) ok = 0;
            }
          }
        }
        if (!ok) continue;
        if (best < 0 || key_less(head, best_key)) {
          best = t;
          best_key = head;
          best_lane = l;
        }
      }
      if (best < 0) break;
      /* start (simulate.cpp:222-236) */
      heap_pop(&ready[best_lane]);
      started[best] = 1;
      sim_start[best] = now;
      sim_end[best] = now + g->duration[best];
      --unstarted;
      if (g->duration[best] == 0) {
        for (int32_t k = off[best]; k < off[best + 1]; ++k)
          if (--indeg[adj[k]] == 0)
            heap_push(&ready[lane_of[adj[k]]], (key_t2){g->original_start[adj[k]], adj[k]});
      } else {
        clock[best_lane] = sim_end[best];
        heap_push(&comp, (key_t2){sim_end[best], best});
      }
    }
    /* run (simulate.cpp:304-318): pop every completion at the next end time */
    if (comp.n == 0) {
      if (unstarted == 0) break;
      status = ORC_DEADLOCK;
      break;
    }
    int64_t t2 = comp.v[0].a;
    while (comp.n > 0 && comp.v[0].a == t2) {
      int32_t done = heap_pop(&comp).b;
      for (int32_t k = off[done]; k < off[done + 1]; ++k)
        if (--indeg[adj[k]] == 0)
          heap_push(&ready[lane_of[adj[k]]], (key_t2){g->original_start[adj[k]], adj[k]});
    }
    now = t2;
  }

  if (status == ORC_OK) {
    /* SimulatedTrace span (simulate.cpp:320-335) */
    int64_t lo = sim_start[0], hi = sim_end[0];
    for (int32_t i = 1; i < n; ++i) {
      if (sim_start[i] < lo) lo = sim_start[i];
      if (sim_end[i] > hi) hi = sim_end[i];
    }
    if (hi < lo) hi = lo;
    span[0] = lo;
    span[1] = hi;
    span[2] = hi - lo;
  }

  for (int32_t l = 0; l < nl; ++l) free(ready[l].v);
  free(ready);
  free(clock);
  free(lanes);
  free(lane_of);
  free(lane_count);
  free(indeg);
  free(off);
  free(adj);
  free(rule_of);
  free(wl);
  free(wl_off);
  free(started);
  free(comp.v);
  return status;
}

/* ------------------------------------------------------------ breakdown */

typedef struct {
  int64_t at;
  int32_t compute;
  int32_t comm;
} delta_t;

static int delta_cmp(const void* x, const void* y) {
  const delta_t* a = (const delta_t*)x;
  const delta_t* b = (const delta_t*)y;
  return a->at < b->at ? -1 : (a->at > b->at ? 1 : 0);
}

void orc_breakdown_rank(int32_t n, const int32_t* rank, const int32_t* lane_kind,
                        const uint8_t* is_comm, const int64_t* start, const int64_t* end,
                        int32_t which_rank, int64_t window_start, int64_t window_end,
                        int64_t out[5]) {
  /* breakdown_by_rank -> gpu_deltas + sweep (src/metrics.cpp:43-103) */
  if (window_end < window_start) window_end = window_start;
  delta_t* d = (delta_t*)malloc(sizeof(delta_t) * (size_t)(2 * n + 1));
  int32_t nd = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (lane_kind[i] != 1 || rank[i] != which_rank) continue;
    int64_t s = start[i] > window_start ? start[i] : window_start;
    int64_t e = end[i] < window_end ? end[i] : window_end;
    if (s >= e) continue;
    int32_t dc = is_comm[i] ? 0 : 1, dm = is_comm[i] ? 1 : 0;
    d[nd++] = (delta_t){s, dc, dm};
    d[nd++] = (delta_t){e, -dc, -dm};
  }
  qsort(d, (size_t)nd, sizeof(delta_t), delta_cmp);
  int64_t total = window_end - window_start, ec = 0, em = 0, ov = 0, ot = 0;
  int64_t prev = window_start;
  int32_t compute = 0, comm = 0;
  for (int32_t k = 0; k <= nd; ++k) {
    int64_t upto = k < nd ? d[k].at : window_end;
    if (upto > prev) {
      int64_t span = upto - prev;
      if (compute > 0 && comm > 0)
        ov += span;
      else if (compute > 0)
        ec += span;
      else if (comm > 0)
        em += span;
      else
        ot += span;
      prev = upto;
    }
    if (k < nd) {
      compute += d[k].compute;
      comm += d[k].comm;
    }
  }
  out[0] = total;
  out[1] = ec;
  out[2] = em;
  out[3] = ov;
  out[4] = ot;
  free(d);
}

/* ------------------------------------------------- scenario durations */

void orc_philox2x32_10(uint32_t ctr0, uint32_t ctr1, uint32_t key, uint32_t out[2]) {
  /* Philox2x32 (Random123): R0' = hi(M*R0) ^ key ^ R1, R1' = lo(M*R0);
   * key += W after each round; 10 rounds. */
  const uint32_t M = 0xD256D193u, W = 0x9E3779B9u;
  uint32_t x0 = ctr0, x1 = ctr1, k = key;
  for (int r = 0; r < 10; ++r) {
    uint64_t p = (uint64_t)M * (uint64_t)x0;
    uint32_t hi = (uint32_t)(p >> 32), lo = (uint32_t)p;
    x0 = hi ^ k ^ x1;
    x1 = lo;
    k += W;
  }
  out[0] = x0;
  out[1] = x1;
}

static uint32_t seed_key(uint64_t seed, uint32_t salt) {
  return (uint32_t)(seed ^ (seed >> 32)) ^ salt;
}

int64_t orc_mul_div(int64_t a, int64_t num, int64_t den) {
  /* src/transform.cpp:38-43: (a*num + den/2) / den in 128-bit */
  __int128 prod = (__int128)a * num;
  __int128 half = den / 2;
  return (int64_t)((prod + half) / den);
}

int32_t orc_class_num(const orc_scenarios* sc, int64_t scenario, int32_t cls) {
  uint32_t r[2];
  orc_philox2x32_10((uint32_t)cls, (uint32_t)scenario, seed_key(sc->seed, 0x5CA1E000u), r);
  uint64_t span = (uint64_t)(int64_t)(sc->scale_hi - sc->scale_lo + 1);
  return sc->scale_lo + (int32_t)(((uint64_t)r[0] * span) >> 32);
}

int64_t orc_scenario_duration(const orc_scenarios* sc, int64_t scenario, int32_t task,
                              int64_t base, int32_t cls) {
  int64_t d = base;
  if (sc->scale_den > 0) d = orc_mul_div(d, orc_class_num(sc, scenario, cls), sc->scale_den);
  if (sc->jitter > 0.0) {
    if (d == 0) return 0;
    /* one Philox call per scenario pair (2p, 2p + 1): word (scenario & 1) */
    uint32_t r[2];
    orc_philox2x32_10((uint32_t)task, (uint32_t)(scenario >> 1), seed_key(sc->seed, 0u), r);
    double u01 = (double)r[scenario & 1] * 0x1.0p-32;
    double u = (2.0 * sc->jitter) * u01 + (-sc->jitter); /* -ffp-contract=off: no FMA */
    double f = 1.0 + u;
    double p = (double)d * f;
    int64_t q = llround(p);
    d = q < 1 ? 1 : q;
  }
  return d;
}

void orc_fill_durations(const orc_scenarios* sc, int64_t scenario, int32_t n,
                        const int64_t* base, const uint8_t* cls, int64_t* dur) {
  for (int32_t t = 0; t < n; ++t)
    dur[t] = orc_scenario_duration(sc, scenario, t, base[t], cls ? cls[t] : 0);
}
