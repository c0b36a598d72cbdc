/*
 * cs_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C, single-threaded
 * restatement of the reference's analysis hot path over our 32-byte records.
 * It is the parity checker for the CUDA path and is never linked into, or
 * called by, the product.  Every function follows the reference in order of
 * operations (sequential f64 sums, no FMA: built with -ffp-contract=off) so
 * results are bit-identical; tests/test_oracle.py pins it against the
 * reference itself (oracle/_ref) and the committed golden vectors.
 *
 * Reference map (paths under /root/reference/proj/src):
 *   rank_candidates      cycles.cpp:47-87   (+ gap-free score formula 66-77)
 *   pick_anchor          cycles.cpp:89-110
 *   segment_cycles       cycles.cpp:120-170
 *   frequency_cycles     cycles.cpp:283-343
 *   classify             cycles.cpp:190-254 (median 181-186)
 *   workload_of          cycles.cpp:256-281
 *   beta_of              rca.cpp:71-130 (beta / collective part)
 *   counter_series       trace.cpp:111-131 (CounterTable::from_trace)
 *   interpolate_mean     rca.cpp:17-53
 *   mu_of                rca.cpp:97-106, 123-126 (mu part of cycle_stats)
 *   records              cycles.cpp:359-409
 *   predict              gbdt.cpp:22-30, 173-184
 *   ppe / detector       detector.cpp:14-19, 57-60, 85-130
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "cyclescope_b200.h"

typedef struct cso_out {
  int status;
  uint32_t anchor;
  int fallback;
  uint64_t n_cand;
  cs_anchor_candidate* cand;
  uint64_t n_cycles;
  cs_cycle* cycles;
  int64_t* comp;       /* n_cycles x n_phases */
  int64_t* beta_tot;   /* n_cycles x n_beta   */
  double* beta;
  double* coll;        /* n_cycles x n_comm   */
  uint8_t* coll_present;
  double* mu;          /* n_cycles x n_beta   */
  uint8_t* mu_has;
  uint64_t n_records;
  cs_record* records;
  uint64_t n_alerts;
  cs_alert* alerts;
  uint64_t first_bad;
  double ucl;
} cso_out;

static void* zalloc(size_t n) { return calloc(n ? n : 1, 1); }

/* ---------------------------------------------------- anchor candidates */
typedef struct {
  uint64_t count;
  double sum, sum_sq;
  uint64_t spans_any;
  int64_t prev_start;     /* gap_cv (cycles.cpp:30-43): sequential gap sums */
  double gap_sum, gap_sq;
} NameAcc;

static int cand_cmp(const void* a, const void* b) {
  const cs_anchor_candidate* x = a;
  const cs_anchor_candidate* y = b;
  if (x->score != y->score) return x->score > y->score ? -1 : 1;
  return x->name_id < y->name_id ? -1 : (x->name_id > y->name_id);
}

static void rank_candidates(const cs_event* ev, uint64_t n, uint32_t n_names,
                            uint64_t min_calls, NameAcc* acc, cso_out* o) {
  for (uint64_t j = 0; j < n; ++j) {
    const cs_event* e = &ev[j];
    if (e->kind != CS_SPAN) continue;
    acc[e->name_id].spans_any++;
    if (e->category != CS_CAT_PYTHON_CALL) continue;
    NameAcc* s = &acc[e->name_id];
    if (s->count > 0) {
      const double gap = (double)(e->start_ts - s->prev_start);
      s->gap_sum += gap;
      s->gap_sq += gap * gap;
    }
    s->prev_start = e->start_ts;
    s->count++;
    const double d = (double)e->duration;
    s->sum += d;
    s->sum_sq += d * d;
  }
  o->cand = zalloc(sizeof(cs_anchor_candidate) * n_names);
  o->n_cand = 0;
  for (uint32_t k = 0; k < n_names; ++k) {
    const NameAcc* s = &acc[k];
    if (s->count < min_calls || s->count == 0) continue;
    cs_anchor_candidate c;
    memset(&c, 0, sizeof c);
    c.name_id = k;
    c.call_count = s->count;
    c.mean_duration_ns = s->sum / (double)s->count;
    double cv = 0.0;
    if (c.mean_duration_ns > 0.0) {
      double var = s->sum_sq / (double)s->count - c.mean_duration_ns * c.mean_duration_ns;
      if (!(0.0 < var)) var = 0.0;
      cv = sqrt(var) / c.mean_duration_ns;
    }
    c.duration_cv = cv;
    c.score = (double)s->count / (1.0 + cv);
    double gcv = 0.0;
    if (s->count >= 3) {
      const double ng = (double)(s->count - 1);
      const double gm = s->gap_sum / ng;
      if (gm > 0.0) {
        double var = s->gap_sq / ng - gm * gm;
        if (!(0.0 < var)) var = 0.0;
        gcv = sqrt(var) / gm;
      }
    }
    c.periodicity = 1.0 / (1.0 + gcv);
    o->cand[o->n_cand++] = c;
  }
  qsort(o->cand, o->n_cand, sizeof(cs_anchor_candidate), cand_cmp);
}

static uint32_t pick_anchor(const cs_cycle_config* cfg, const NameAcc* acc, const cso_out* o) {
  if (cfg->anchor_hint_name == -2) return UINT32_MAX;
  if (cfg->anchor_hint_name >= 0) {
    const uint32_t h = (uint32_t)cfg->anchor_hint_name;
    return acc[h].spans_any > 0 ? h : UINT32_MAX;
  }
  return o->n_cand ? o->cand[0].name_id : UINT32_MAX;
}

static uint64_t lower_index(const cs_event* ev, uint64_t n, int64_t ts) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (ev[mid].start_ts < ts) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* ---------------------------------------------------------- segmentation */
static void segment_cycles(const cs_event* ev, uint64_t n, const cs_name_info* names,
                           uint32_t anchor, int P, cso_out* o) {
  uint64_t na = 0;
  for (uint64_t j = 0; j < n; ++j)
    if (ev[j].kind == CS_SPAN && ev[j].name_id == anchor) ++na;
  o->n_cycles = na >= 2 ? na - 1 : 0;
  o->cycles = zalloc(sizeof(cs_cycle) * o->n_cycles);
  o->comp = zalloc(sizeof(int64_t) * o->n_cycles * (P ? P : 1));
  if (na < 2) return;
  uint64_t* pos = zalloc(sizeof(uint64_t) * na);
  uint64_t k = 0;
  for (uint64_t j = 0; j < n; ++j)
    if (ev[j].kind == CS_SPAN && ev[j].name_id == anchor) pos[k++] = j;
  for (uint64_t i = 0; i + 1 < na; ++i) {
    cs_cycle* c = &o->cycles[i];
    c->index = i;
    c->start_ts = ev[pos[i]].start_ts;
    c->end_ts = ev[pos[i + 1]].start_ts;
    c->anchor_pos = pos[i];
    c->anchor_span_end = ev[pos[i]].start_ts + ev[pos[i]].duration;
    c->first_event = lower_index(ev, n, c->start_ts);
    c->last_event = lower_index(ev, n, c->end_ts);
    c->stage = CS_STAGE_UNKNOWN;
    for (uint64_t j = c->first_event; j < c->last_event; ++j) {
      const cs_event* e = &ev[j];
      if (e->kind != CS_SPAN) continue;
      const int p = names[e->name_id].phase;
      if (p < 0) continue;
      const int64_t end = e->start_ts + e->duration;
      const int64_t clipped = (end < c->end_ts ? end : c->end_ts) - e->start_ts;
      o->comp[i * P + p] += clipped > 0 ? clipped : 0;
    }
  }
  free(pos);
}

static void frequency_cycles(const cs_event* ev, uint64_t n, int64_t bin, int P, cso_out* o) {
  uint64_t ns = 0;
  int64_t t0 = 0, t1 = 0;
  for (uint64_t j = 0; j < n; ++j)
    if (ev[j].kind == CS_SPAN && ev[j].category == CS_CAT_GPU_KERNEL) {
      if (ns == 0) t0 = ev[j].start_ts;
      t1 = ev[j].start_ts;
      ++ns;
    }
  o->n_cycles = 0;
  o->cycles = zalloc(sizeof(cs_cycle));
  o->comp = zalloc(sizeof(int64_t));
  if (ns < 4) return;
  const uint64_t bins = (uint64_t)((t1 - t0) / bin) + 1;
  if (bins < 4) return;
  double* h = zalloc(sizeof(double) * bins);
  for (uint64_t j = 0; j < n; ++j)
    if (ev[j].kind == CS_SPAN && ev[j].category == CS_CAT_GPU_KERNEL)
      h[(uint64_t)((ev[j].start_ts - t0) / bin)] += 1.0;
  double mean = 0.0;
  for (uint64_t i = 0; i < bins; ++i) mean += h[i];
  mean /= (double)bins;
  for (uint64_t i = 0; i < bins; ++i) h[i] -= mean;
  double best = 0.0;
  uint64_t best_lag = 0;
  for (uint64_t lag = 1; lag <= bins / 2; ++lag) {
    double acc = 0.0;
    for (uint64_t i = 0; i + lag < bins; ++i) acc += h[i] * h[i + lag];
    if (acc > best) {
      best = acc;
      best_lag = lag;
    }
  }
  free(h);
  if (best_lag == 0) return;
  const int64_t period = (int64_t)best_lag * bin;
  uint64_t nc = 0;
  for (int64_t s = t0; s + period <= t1; s += period) ++nc;
  free(o->cycles);
  free(o->comp);
  o->n_cycles = nc;
  o->cycles = zalloc(sizeof(cs_cycle) * nc);
  o->comp = zalloc(sizeof(int64_t) * nc * (P ? P : 1));
  uint64_t i = 0;
  for (int64_t s = t0; s + period <= t1; s += period, ++i) {
    cs_cycle* c = &o->cycles[i];
    c->index = i;
    c->start_ts = s;
    c->end_ts = s + period;
    c->anchor_pos = UINT64_MAX;
    c->anchor_span_end = s;
    c->first_event = lower_index(ev, n, s);
    c->last_event = lower_index(ev, n, s + period);
    c->stage = CS_STAGE_UNKNOWN;
  }
}

/* ------------------------------------------------------ stage classifier */
static int dbl_cmp(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y);
}

typedef struct {
  double* v;
  uint64_t cap, head, size;
} Ring;

static void ring_push(Ring* r, double x) {
  r->v[(r->head + r->size) % r->cap] = x;
  if (r->size < r->cap) r->size++;
  else r->head = (r->head + 1) % r->cap;
}

static double ring_median(const Ring* r, double* tmp) {
  for (uint64_t i = 0; i < r->size; ++i) tmp[i] = r->v[(r->head + i) % r->cap];
  qsort(tmp, r->size, sizeof(double), dbl_cmp);
  const uint64_t n = r->size;
  return n % 2 == 1 ? tmp[n / 2] : 0.5 * (tmp[n / 2 - 1] + tmp[n / 2]);
}

static void classify(const cs_event* ev, const cs_name_info* names, const cs_cycle_config* cfg,
                     cso_out* o) {
  const uint64_t W = cfg->stage_window;
  Ring dur = {zalloc(sizeof(double) * W), W, 0, 0};
  Ring gap = {zalloc(sizeof(double) * W), W, 0, 0};
  double* tmp = zalloc(sizeof(double) * W);
  int64_t prev_end = 0;
  int have_prev = 0;
  for (uint64_t i = 0; i < o->n_cycles; ++i) {
    cs_cycle* c = &o->cycles[i];
    const double idle = have_prev ? (double)(c->start_ts - prev_end) : -1.0;
    int stage = CS_STAGE_UNKNOWN;
    uint32_t fm = 0;
    for (uint64_t j = c->first_event; j < c->last_event; ++j)
      if (ev[j].flags & CS_EV_FM_MASK) {
        fm = ev[j].flags & CS_EV_FM_MASK;
        break;
      }
    if (fm == CS_EV_FM_PREFILL) stage = CS_STAGE_PREFILL;
    else if (fm == CS_EV_FM_DECODE) stage = CS_STAGE_DECODE;
    if (stage == CS_STAGE_UNKNOWN) {
      int pk = 0, dk = 0;
      for (uint64_t j = c->first_event; j < c->last_event; ++j) {
        if (ev[j].kind != CS_SPAN) continue;
        pk |= (names[ev[j].name_id].flags & CS_NAME_PREFILL_KW) != 0;
        dk |= (names[ev[j].name_id].flags & CS_NAME_DECODE_KW) != 0;
      }
      if (pk != dk) stage = pk ? CS_STAGE_PREFILL : CS_STAGE_DECODE;
    }
    if (stage == CS_STAGE_UNKNOWN && dur.size >= cfg->stage_min_history && idle >= 0.0) {
      const double md = ring_median(&dur, tmp);
      double mg = gap.size ? ring_median(&gap, tmp) : 0.0;
      if (!(1.0 < mg)) mg = 1.0;
      const int long_cycle = (double)(c->end_ts - c->start_ts) > cfg->prefill_duration_factor * md;
      const int long_gap = idle > cfg->prefill_gap_factor * mg;
      stage = (long_cycle && long_gap) ? CS_STAGE_PREFILL : CS_STAGE_DECODE;
    }
    c->stage = stage;
    if (stage != CS_STAGE_PREFILL) {
      ring_push(&dur, (double)(c->end_ts - c->start_ts));
      if (idle >= 0.0) ring_push(&gap, idle);
    }
    prev_end = c->anchor_span_end;
    have_prev = 1;
  }
  free(dur.v);
  free(gap.v);
  free(tmp);
}

/* workload status: 0 ok (carrier index in *wl_idx), 1 no carrier, 2 invalid */
static int workload_of(const cs_event* ev, const cs_cycle* c, int64_t* wl_idx) {
  for (uint64_t j = c->first_event; j < c->last_event; ++j) {
    if (!(ev[j].flags & CS_EV_HAS_BATCH)) continue;
    if (!(ev[j].flags & CS_EV_WL_OK)) return 2;
    *wl_idx = (int64_t)(ev[j].payload & 0xffffffffu);
    return 0;
  }
  return 1;
}

static void beta_of(const cs_event* ev, const cs_name_info* names, int C, int R, cso_out* o) {
  o->beta_tot = zalloc(sizeof(int64_t) * o->n_cycles * (C ? C : 1));
  o->beta = zalloc(sizeof(double) * o->n_cycles * (C ? C : 1));
  o->coll = zalloc(sizeof(double) * o->n_cycles * (R ? R : 1));
  o->coll_present = zalloc(o->n_cycles * (R ? R : 1));
  for (uint64_t i = 0; i < o->n_cycles; ++i) {
    const cs_cycle* c = &o->cycles[i];
    const int64_t dur = c->end_ts - c->start_ts;
    if (dur <= 0) continue;
    for (uint64_t j = c->first_event; j < c->last_event; ++j) {
      const cs_event* e = &ev[j];
      if (e->kind != CS_SPAN || e->duration <= 0) continue;
      const int64_t end = e->start_ts + e->duration;
      const int64_t ov = (end < c->end_ts ? end : c->end_ts) - e->start_ts;
      if (ov <= 0) continue;
      const int s = names[e->name_id].beta_slot;
      if (s >= 0) o->beta_tot[i * C + s] += ov;
      if (e->category == CS_CAT_COLLECTIVE_COMM && (e->flags & CS_EV_HAS_COMM)) {
        const uint32_t k = (uint32_t)(e->payload >> 32);
        o->coll[i * R + k] += (double)ov / (double)dur;
        o->coll_present[i * R + k] = 1;
      }
    }
    for (int s = 0; s < C; ++s)
      if (o->beta_tot[i * C + s] > 0) o->beta[i * C + s] = (double)o->beta_tot[i * C + s] / (double)dur;
  }
}


/* --------------------------------------------- counter-weighted mu (§8f) */
typedef struct {
  uint64_t n;
  int64_t* ts;
  double* v;
} Series;

/* CounterTable::from_trace: per counter name, the valued Counter events in
 * event order (the reference's stable sort by ts keeps that order). */
static Series* counter_series(const cs_event* ev, uint64_t n, uint32_t n_names) {
  Series* s = zalloc(sizeof(Series) * (n_names ? n_names : 1));
  for (uint64_t j = 0; j < n; ++j)
    if (ev[j].kind == CS_COUNTER && (ev[j].flags & CS_EV_HAS_VALUE)) ++s[ev[j].name_id].n;
  for (uint32_t k = 0; k < n_names; ++k) {
    s[k].ts = zalloc(sizeof(int64_t) * s[k].n);
    s[k].v = zalloc(sizeof(double) * s[k].n);
    s[k].n = 0;
  }
  for (uint64_t j = 0; j < n; ++j) {
    if (ev[j].kind != CS_COUNTER || !(ev[j].flags & CS_EV_HAS_VALUE)) continue;
    Series* x = &s[ev[j].name_id];
    x->ts[x->n] = ev[j].start_ts;
    memcpy(&x->v[x->n], &ev[j].duration, sizeof(double));
    ++x->n;
  }
  return s;
}

static double value_at(const Series* s, double t) {
  if (t <= (double)s->ts[0]) return s->v[0];
  if (t >= (double)s->ts[s->n - 1]) return s->v[s->n - 1];
  uint64_t lo = 0, hi = s->n; /* lower_bound: first sample with ts >= t */
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if ((double)s->ts[mid] < t) lo = mid + 1;
    else hi = mid;
  }
  const double f = (t - (double)s->ts[lo - 1]) / (double)(s->ts[lo] - s->ts[lo - 1]);
  return s->v[lo - 1] + f * (s->v[lo] - s->v[lo - 1]);
}

static double interpolate_mean(const Series* s, int64_t t0, int64_t t1) {
  double* knots = zalloc(sizeof(double) * (s->n + 2));
  uint64_t nk = 0;
  knots[nk++] = (double)t0;
  for (uint64_t i = 0; i < s->n; ++i) {
    const double ts = (double)s->ts[i];
    if (ts > (double)t0 && ts < (double)t1) knots[nk++] = ts;
  }
  knots[nk++] = (double)t1;
  double integral = 0.0;
  for (uint64_t i = 0; i + 1 < nk; ++i) {
    const double a = knots[i], b = knots[i + 1];
    integral += 0.5 * (value_at(s, a) + value_at(s, b)) * (b - a);
  }
  free(knots);
  return integral / ((double)t1 - (double)t0);
}

static void mu_of(const cs_event* ev, uint64_t n, const cs_name_info* names, uint32_t n_names,
                  int C, cso_out* o) {
  o->mu = zalloc(sizeof(double) * o->n_cycles * (C ? C : 1));
  o->mu_has = zalloc(o->n_cycles * (C ? C : 1));
  Series* series = counter_series(ev, n, n_names);
  double* w = zalloc(sizeof(double) * (C ? C : 1));
  uint8_t* has = zalloc(C ? C : 1);
  for (uint64_t i = 0; i < o->n_cycles; ++i) {
    const cs_cycle* c = &o->cycles[i];
    const int64_t dur = c->end_ts - c->start_ts;
    if (dur <= 0) continue;
    memset(w, 0, sizeof(double) * (C ? C : 1));
    memset(has, 0, C ? C : 1);
    for (uint64_t j = c->first_event; j < c->last_event; ++j) {
      const cs_event* e = &ev[j];
      if (e->kind != CS_SPAN || e->duration <= 0) continue;
      const int64_t end = e->start_ts + e->duration;
      const int64_t clipped_end = end < c->end_ts ? end : c->end_ts;
      const int64_t ov = clipped_end - e->start_ts;
      if (ov <= 0) continue;
      const int s = names[e->name_id].beta_slot;
      const uint32_t m = names[e->name_id].metric;
      if (s < 0 || m == 0 || m > n_names || series[m - 1].n == 0) continue;
      w[s] += interpolate_mean(&series[m - 1], e->start_ts, clipped_end) * (double)ov;
      has[s] = 1;
    }
    for (int s = 0; s < C; ++s)
      if (has[s] && o->beta_tot[i * C + s] > 0) {
        o->mu[i * C + s] = w[s] / (double)o->beta_tot[i * C + s];
        o->mu_has[i * C + s] = 1;
      }
  }
  for (uint32_t k = 0; k < n_names; ++k) {
    free(series[k].ts);
    free(series[k].v);
  }
  free(series);
  free(w);
  free(has);
}

/* ----------------------------------------------------------- model eval */
static double predict(const cs_model* m, const double* x) {
  double v = m->base;
  for (uint32_t t = 0; t < m->n_trees; ++t) {
    const cs_tree_node* nd = m->nodes + m->tree_offsets[t];
    int k = 0;
    while (nd[k].feature >= 0) k = x[nd[k].feature] <= nd[k].threshold ? nd[k].left : nd[k].right;
    v += m->learning_rate * nd[k].value;
  }
  return m->prediction_floor < v ? v : m->prediction_floor;
}

static double feature(int id, const cs_workload* w, int stage) {
  switch (id) {
    case CS_F_BATCH: return (double)w->batch;
    case CS_F_W_KV: return (double)(w->batch * (w->input_len + w->output_len));
    case CS_F_INPUT_LEN: return (double)w->input_len;
    case CS_F_OUTPUT_LEN: return (double)w->output_len;
    default: return stage == CS_STAGE_PREFILL ? 1.0 : 0.0;
  }
}

int cso_analyze(const cs_event* ev, uint64_t n, const cs_workload* wl, uint32_t n_names,
                const cs_name_info* names, const cs_cycle_config* cfg,
                const cs_control_config* ctl, const cs_model* model, cso_out** out) {
  cso_out* o = zalloc(sizeof(cso_out));
  *out = o;
  o->first_bad = UINT64_MAX;
  const int P = cfg->n_phases, C = cfg->n_beta_slots, R = cfg->n_comm_slots;
  NameAcc* acc = zalloc(sizeof(NameAcc) * (n_names ? n_names : 1));
  rank_candidates(ev, n, n_names, cfg->min_anchor_calls, acc, o);
  o->anchor = pick_anchor(cfg, acc, o);
  free(acc);
  if (o->anchor != UINT32_MAX) {
    segment_cycles(ev, n, names, o->anchor, P, o);
  } else {
    o->fallback = 1;
    frequency_cycles(ev, n, cfg->frequency_bin_ns, P, o);
    if (o->n_cycles == 0) {
      o->status = CS_E_NO_ANCHOR_FOUND;
      beta_of(ev, names, C, R, o);
      mu_of(ev, n, names, n_names, C, o);
      o->records = zalloc(sizeof(cs_record));
      o->alerts = zalloc(sizeof(cs_alert));
      return o->status;
    }
  }
  classify(ev, names, cfg, o);
  int64_t* wl_idx = zalloc(sizeof(int64_t) * (o->n_cycles ? o->n_cycles : 1));
  for (uint64_t i = 0; i < o->n_cycles; ++i)
    o->cycles[i].workload_status = workload_of(ev, &o->cycles[i], &wl_idx[i]);
  beta_of(ev, names, C, R, o);
  mu_of(ev, n, names, n_names, C, o);
  /* records (cycles.cpp:366-409) */
  o->records = zalloc(sizeof(cs_record) * (o->n_cycles ? o->n_cycles : 1));
  o->alerts = zalloc(sizeof(cs_alert) * (o->n_cycles ? o->n_cycles : 1));
  for (uint64_t i = 0; i < o->n_cycles; ++i) {
    const cs_cycle* c = &o->cycles[i];
    if (!cfg->include_prefill && c->stage == CS_STAGE_PREFILL) continue;
    if (c->workload_status != 0) continue;
    cs_record* r = &o->records[o->n_records++];
    const cs_workload* w = &wl[wl_idx[i]];
    r->cycle_index = c->index;
    r->start_ts = c->start_ts;
    r->stage = c->stage;
    r->batch = w->batch;
    r->input_len = w->input_len;
    r->output_len = w->output_len;
    int64_t target = c->end_ts - c->start_ts;
    if (cfg->latency_phase >= 0 && c->anchor_pos != UINT64_MAX &&
        o->comp[i * P + cfg->latency_phase] > 0)
      target = o->comp[i * P + cfg->latency_phase];
    r->latency_s = (double)target * 1e-9;
  }
  if (model) {
    /* monitor_loop process lambda: predict, ppe, Detector::step */
    double limit = ctl->fixed_threshold;
    if (ctl->strategy == CS_DYNAMIC_WINDOW) {
      double u = model->mu_train + ctl->sigma_k * model->sigma_train;
      if (!(u < ctl->theta_max)) u = ctl->theta_max;
      limit = u < ctl->min_ucl ? ctl->min_ucl : u;
    }
    o->ucl = limit;
    Ring win = {zalloc(sizeof(double) * ctl->window), ctl->window, 0, 0};
    uint64_t seen = 0, next_episode = 0;
    int in_episode = 0;
    double x[8];
    for (uint64_t k = 0; k < o->n_records; ++k) {
      cs_record* r = &o->records[k];
      const cs_workload* w = &wl[wl_idx[r->cycle_index]];
      for (uint32_t f = 0; f < model->n_features; ++f) x[f] = feature(model->feature_ids[f], w, r->stage);
      r->predicted_s = predict(model, x);
      if (!(r->latency_s > 0.0)) {
        o->first_bad = k;
        o->status = CS_E_NON_POSITIVE_LATENCY;
        break;
      }
      const double q = (r->latency_s - r->predicted_s) / (r->latency_s + ctl->epsilon);
      r->residual = 0.0 < q ? q : 0.0;
      double stat = r->residual;
      if (ctl->strategy != CS_FIXED_POINT) {
        ring_push(&win, r->residual);
        double sum = 0.0;
        for (uint64_t i = 0; i < win.size; ++i) sum += win.v[(win.head + i) % win.cap];
        stat = sum / (double)win.size;
      }
      r->statistic = stat;
      r->armed = seen >= ctl->warmup;
      ++seen;
      if (!r->armed) {
        in_episode = 0;
        continue;
      }
      r->flagged = stat > limit;
      if (r->flagged && !in_episode) {
        in_episode = 1;
        r->alert = 1;
        r->episode_id = next_episode++;
        cs_alert* a = &o->alerts[o->n_alerts++];
        a->cycle = r->cycle_index;
        a->ts = r->start_ts;
        a->smoothed_error = stat;
        a->limit = limit;
        a->strategy = ctl->strategy;
        a->batch = r->batch;
        a->input_len = r->input_len;
        a->output_len = r->output_len;
        a->episode_id = r->episode_id;
        a->record_index = k;
      } else if (!r->flagged) {
        in_episode = 0;
      }
    }
    free(win.v);
  }
  free(wl_idx);
  return o->status;
}

void cso_free(cso_out* o) {
  if (!o) return;
  free(o->cand);
  free(o->cycles);
  free(o->comp);
  free(o->beta_tot);
  free(o->beta);
  free(o->coll);
  free(o->coll_present);
  free(o->mu);
  free(o->mu_has);
  free(o->records);
  free(o->alerts);
  free(o);
}

/* accessors for ctypes */
int cso_status(const cso_out* o) { return o->status; }
uint32_t cso_anchor(const cso_out* o) { return o->anchor; }
int cso_fallback(const cso_out* o) { return o->fallback; }
double cso_ucl(const cso_out* o) { return o->ucl; }
uint64_t cso_first_bad(const cso_out* o) { return o->first_bad; }
uint64_t cso_n_candidates(const cso_out* o) { return o->n_cand; }
const cs_anchor_candidate* cso_candidates(const cso_out* o) { return o->cand; }
uint64_t cso_n_cycles(const cso_out* o) { return o->n_cycles; }
const cs_cycle* cso_cycles(const cso_out* o) { return o->cycles; }
const int64_t* cso_components(const cso_out* o) { return o->comp; }
const int64_t* cso_beta_totals(const cso_out* o) { return o->beta_tot; }
const double* cso_beta(const cso_out* o) { return o->beta; }
const double* cso_coll(const cso_out* o) { return o->coll; }
const uint8_t* cso_coll_present(const cso_out* o) { return o->coll_present; }
const double* cso_mu(const cso_out* o) { return o->mu; }
const uint8_t* cso_mu_has(const cso_out* o) { return o->mu_has; }
uint64_t cso_n_records(const cso_out* o) { return o->n_records; }
const cs_record* cso_records(const cso_out* o) { return o->records; }
uint64_t cso_n_alerts(const cso_out* o) { return o->n_alerts; }
const cs_alert* cso_alerts(const cso_out* o) { return o->alerts; }
