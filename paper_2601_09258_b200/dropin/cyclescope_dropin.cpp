// cyclescope_dropin.cpp — C++ drop-in for the reference's hot-path API.
//
// Compile this file together with the caller's copy of the reference headers
// (proj/include/cyclescope/*.hpp) INSTEAD of the reference's definitions of
// the functions below, and link libcyclescope_b200.so.  Every function keeps
// the reference's signature and semantics; the work runs on the B200 through
// the C ABI (include/cyclescope_b200.h).  Errors come back as the reference's
// EngineError subclasses; the two control-flow exceptions (MissingWorkloadArgs
// skip, NoAnchorFound -> frequency fallback) are handled inside the device
// pipeline exactly like cycles.cpp:345-383.
//
//   cycles.hpp   rank_anchor_candidates, discover_anchor, segment,
//                classify_stages, extract_workload, segment_by_frequency,
//                segment_and_classify, build_cycle_records (both overloads)
//   rca.hpp      cycle_stats (+ cycle_stats_all: every cycle in one pass)
//   detector.hpp evaluate_strategy, evaluate_strategies (the batched Detector)
//
// Ingest (A1-A2): a Trace is interned once into 32-byte records — names in
// lexicographic order (so name ids are the tie-break ranks), the forward_mode
// / batch / commHash+rank / value args folded into flags and the workload
// table — and uploaded once.  A per-thread session keeps the last trace on the
// device, keyed by its address, size and a fingerprint of sampled events and
// the arg keys, so the per-cycle calls (cycle_stats, extract_workload) of
// evaluate_trial / cmd_diagnose do not re-upload it.  A Trace mutated in place
// between calls without changing any sampled event is the one case the key
// cannot see.
#include <algorithm>
#include <cctype>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <span>
#include <string>
#include <tuple>
#include <vector>

#include "cyclescope/cycles.hpp"
#include "cyclescope/detector.hpp"
#include "cyclescope/errors.hpp"
#include "cyclescope/rca.hpp"
#include "cyclescope/trace.hpp"
#include "cyclescope_b200.h"

namespace cyclescope {
namespace {

struct Ingested {
  std::vector<cs_event> ev;
  std::vector<cs_workload> wl;
  std::vector<std::string> names;
  std::vector<uint8_t> is_span;
  std::vector<std::tuple<std::string, std::string, int>> comm;
  // record extras (PipelineOptions::extra_args_prefix args, cycles.cpp:392-405)
  std::string extra_prefix;
  std::vector<std::string> extra_keys;
  std::vector<cs_extra_ref> extra_refs;
  std::vector<cs_extra_value> extra_vals;
};

// the numeric args with the prefix, per event in key order (map iteration)
void ingest_extras(Ingested& in, const Trace& trace, const std::string& prefix) {
  in.extra_prefix = prefix;
  in.extra_keys.clear();
  in.extra_refs.clear();
  in.extra_vals.clear();
  if (prefix.empty()) return;
  std::set<std::string> keys;
  for (const auto& e : trace.events)
    for (const auto& [k, v] : e.args)
      if (k.rfind(prefix, 0) == 0 && !std::holds_alternative<std::string>(v)) keys.insert(k);
  in.extra_keys.assign(keys.begin(), keys.end());
  for (size_t i = 0; i < trace.events.size(); ++i) {
    cs_extra_ref ref{i, static_cast<uint32_t>(in.extra_vals.size()), 0};
    for (const auto& [k, v] : trace.events[i].args) {
      if (k.rfind(prefix, 0) != 0) continue;
      double d;
      if (const auto* x = std::get_if<double>(&v)) d = *x;
      else if (const auto* n = std::get_if<std::int64_t>(&v)) d = static_cast<double>(*n);
      else if (const auto* b = std::get_if<bool>(&v)) d = *b ? 1.0 : 0.0;
      else continue;
      const auto key = std::lower_bound(in.extra_keys.begin(), in.extra_keys.end(), k) - in.extra_keys.begin();
      in.extra_vals.push_back({static_cast<uint32_t>(key), 0, d});
      ++ref.count;
    }
    if (ref.count) in.extra_refs.push_back(ref);
  }
}

Ingested ingest(const Trace& trace, const CycleConfig& cfg) {
  Ingested in;
  std::set<std::string> ns;
  std::set<std::tuple<std::string, std::string, int>> cs;
  for (const auto& e : trace.events) {
    ns.insert(e.name);
    if (e.kind == EventKind::Span && e.category == EventCategory::CollectiveComm) {
      auto c = arg_string(e, "commHash");
      auto r = arg_int(e, "rank");
      if (c && r) cs.insert({e.name, *c, static_cast<int>(*r)});
    }
  }
  in.names.assign(ns.begin(), ns.end());
  in.comm.assign(cs.begin(), cs.end());
  std::map<std::string, uint32_t> id;
  for (uint32_t i = 0; i < in.names.size(); ++i) id[in.names[i]] = i;
  in.is_span.assign(in.names.size(), 0);
  in.ev.resize(trace.events.size());
  for (size_t i = 0; i < trace.events.size(); ++i) {
    const TraceEvent& e = trace.events[i];
    cs_event& r = in.ev[i];
    std::memset(&r, 0, sizeof r);
    r.start_ts = e.start_ts;
    r.duration = e.kind == EventKind::Span ? e.duration : 0;
    r.name_id = id[e.name];
    r.kind = static_cast<uint8_t>(e.kind);
    r.category = static_cast<uint8_t>(e.category);
    if (e.kind == EventKind::Span) in.is_span[r.name_id] = 1;
    uint16_t f = 0;
    if (auto fm = arg_string(e, cfg.forward_mode_key)) {
      std::string m = *fm;
      std::transform(m.begin(), m.end(), m.begin(),
                     [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
      if (m.find("prefill") != std::string::npos || m.find("extend") != std::string::npos)
        f |= CS_EV_FM_PREFILL;
      else if (m.find("decode") != std::string::npos)
        f |= CS_EV_FM_DECODE;
      else
        f |= CS_EV_FM_OTHER;
    }
    if (auto b = arg_int(e, cfg.batch_size_key)) {
      auto il = arg_int(e, cfg.input_len_key);
      auto ol = arg_int(e, cfg.output_len_key);
      f |= CS_EV_HAS_BATCH;
      if (il && ol && *b >= 0 && *il >= 0 && *ol >= 0) f |= CS_EV_WL_OK;
      r.payload |= in.wl.size();
      in.wl.push_back({*b, il ? *il : INT64_MIN, ol ? *ol : INT64_MIN});
    }
    if (e.kind == EventKind::Span && e.category == EventCategory::CollectiveComm) {
      auto c = arg_string(e, "commHash");
      auto rk = arg_int(e, "rank");
      if (c && rk) {
        const auto key = std::make_tuple(e.name, *c, static_cast<int>(*rk));
        const auto slot = std::lower_bound(in.comm.begin(), in.comm.end(), key) - in.comm.begin();
        f |= CS_EV_HAS_COMM;
        r.payload |= static_cast<uint64_t>(slot) << 32;
      }
    }
    if (e.kind == EventKind::Counter)
      if (auto v = arg_number(e, "value")) {
        f |= CS_EV_HAS_VALUE;
        std::memcpy(&r.duration, &*v, sizeof(double));
      }
    r.flags = f;
  }
  return in;
}

[[noreturn]] void rethrow(int status, const std::string& msg) {
  switch (status) {
    case CS_E_NO_ANCHOR_FOUND: throw NoAnchorFound(msg);
    case CS_E_MISSING_WORKLOAD: throw MissingWorkloadArgs(msg);
    case CS_E_FEATURE_MISMATCH: throw FeatureMismatch(msg);
    case CS_E_NON_POSITIVE_LATENCY: throw NonPositiveLatency(msg);
    case CS_E_INSUFFICIENT_DATA: throw InsufficientData(msg);
    case CS_E_NO_LABELS: throw NoLabels(msg);
    case CS_E_MODEL_FORMAT: throw ModelFormatError(msg);
    case CS_E_CONFIG: throw ConfigError(msg);
    default: throw EngineError(cs_status_type(status), msg);
  }
}

struct Ctx {
  cs_ctx* c = nullptr;
  Ctx() {
    const int rc = cs_ctx_create(0, &c);
    if (rc) rethrow(rc, "cs_ctx_create: no B200 available (no CPU fallback)");
  }
  ~Ctx() { cs_ctx_destroy(c); }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
  void check(int rc) const {
    if (rc) rethrow(rc, cs_last_error(c));
  }
};

// One trace on the device.  Key: address, size, arg keys and sampled events.
struct Session {
  const Trace* trace = nullptr;
  size_t n = 0;
  uint64_t fp = 0;
  std::string keys;
  Ingested in;
  Ctx ctx;
  std::vector<std::string> phases;  // device phase index -> name (last config applied)
  std::vector<std::string> slot_names;
  bool extras_uploaded = false;
};

uint64_t fingerprint(const Trace& t) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  const size_t n = t.events.size();
  for (size_t k = 0; k < 64 && n; ++k) {
    const auto& e = t.events[(n - 1) * k / 63];
    mix(static_cast<uint64_t>(e.start_ts));
    mix(e.event_id);
    mix(static_cast<uint64_t>(e.duration));
    mix(std::hash<std::string>{}(e.name));
  }
  return h;
}

Session& session(const Trace& trace, const CycleConfig& cfg) {
  thread_local std::unique_ptr<Session> s;
  const std::string keys = cfg.forward_mode_key + '\0' + cfg.batch_size_key + '\0' + cfg.input_len_key +
                           '\0' + cfg.output_len_key;
  const uint64_t fp = fingerprint(trace);
  if (s && s->trace == &trace && s->n == trace.events.size() && s->fp == fp && s->keys == keys) return *s;
  s.reset();
  s = std::make_unique<Session>();
  s->trace = &trace;
  s->n = trace.events.size();
  s->fp = fp;
  s->keys = keys;
  s->in = ingest(trace, cfg);
  const uint64_t off[2] = {0, s->in.ev.size()};
  // event positions (first_event, last_event, anchor ids) are indices into
  // the caller's canonically ordered Trace::events (cycles.hpp:71-73)
  bool sorted = true;
  for (size_t i = 1; i < trace.events.size() && sorted; ++i)
    sorted = !event_order(trace.events[i], trace.events[i - 1]);
  if (!sorted)
    rethrow(CS_E_INVALID_ARGUMENT,
            "trace events are not in canonical order (Trace::sort_events): event indices would differ");
  s->ctx.check(cs_upload(s->ctx.c, 1, off, s->in.ev.data(), s->in.wl.size(), s->in.wl.data()));
  return *s;
}

// CycleConfig / PipelineOptions (cycles.hpp:18-43,123-128) and an optional
// MetricMap (rca.hpp:22-27) -> device config + name table.
void apply_config(Session& S, const CycleConfig& config, const PipelineOptions& opt,
                  const MetricMap* metrics = nullptr, int64_t hint_override = -1,
                  const CounterTable* counters = nullptr) {
  S.phases.clear();
  for (const auto& p : config.phase_functions)
    if (std::find(S.phases.begin(), S.phases.end(), p) == S.phases.end()) S.phases.push_back(p);
  const auto& names = S.in.names;
  std::vector<cs_name_info> table(names.size());
  int32_t slot = 0;
  cs_cycle_config c{};
  c.anchor_hint_name = -1;
  S.slot_names.clear();
  for (size_t i = 0; i < names.size(); ++i) {
    const std::string& nm = names[i];
    table[i].phase = -1;
    for (size_t k = 0; k < S.phases.size(); ++k)
      if (S.phases[k] == nm) table[i].phase = static_cast<int32_t>(k);
    for (const auto& kw : config.prefill_keywords)
      if (nm.find(kw) != std::string::npos) table[i].flags |= CS_NAME_PREFILL_KW;
    for (const auto& kw : config.decode_keywords)
      if (nm.find(kw) != std::string::npos) table[i].flags |= CS_NAME_DECODE_KW;
    table[i].beta_slot = S.in.is_span[i] ? slot++ : -1;
    if (S.in.is_span[i]) S.slot_names.push_back(nm);
    if (metrics && counters) {
      auto it = metrics->class_to_metric.find(nm);
      // a class whose metric has no counter series stays beta-only (rca.cpp:97-106)
      if (it != metrics->class_to_metric.end() && counters->find(it->second)) {
        auto m = std::lower_bound(names.begin(), names.end(), it->second);
        if (m != names.end() && *m == it->second) table[i].metric = static_cast<uint32_t>(m - names.begin()) + 1;
      }
    }
    if (!config.anchor_hint.empty() && nm == config.anchor_hint) c.anchor_hint_name = static_cast<int64_t>(i);
  }
  if (!config.anchor_hint.empty() && c.anchor_hint_name < 0) c.anchor_hint_name = -2;
  if (hint_override != -1) c.anchor_hint_name = hint_override;
  c.min_anchor_calls = config.min_anchor_calls;
  c.prefill_duration_factor = config.prefill_duration_factor;
  c.prefill_gap_factor = config.prefill_gap_factor;
  c.stage_window = config.stage_window;
  c.stage_min_history = config.stage_min_history;
  c.frequency_bin_ns = config.frequency_bin_ns;
  c.n_phases = static_cast<int32_t>(S.phases.size());
  c.latency_phase = -1;
  for (size_t k = 0; k < S.phases.size(); ++k)
    if (!opt.latency_component.empty() && S.phases[k] == opt.latency_component)
      c.latency_phase = static_cast<int32_t>(k);
  c.include_prefill = opt.include_prefill ? 1 : 0;
  c.n_beta_slots = slot;
  c.n_comm_slots = static_cast<int32_t>(S.in.comm.size());
  S.ctx.check(cs_set_config(S.ctx.c, &c, nullptr));
  S.ctx.check(cs_set_name_table(S.ctx.c, static_cast<uint32_t>(table.size()), table.data()));
}

cs_instance_summary summary(const Session& S) {
  cs_instance_summary s{};
  S.ctx.check(cs_get_summary(S.ctx.c, 0, &s));
  return s;
}

Stage stage_of(int32_t s) {
  return s == CS_STAGE_PREFILL ? Stage::Prefill : (s == CS_STAGE_DECODE ? Stage::Decode : Stage::Unknown);
}
int32_t stage_code(Stage s) {
  return s == Stage::Prefill ? CS_STAGE_PREFILL : (s == Stage::Decode ? CS_STAGE_DECODE : CS_STAGE_UNKNOWN);
}

template <typename T, typename F>
std::vector<T> fetch(const Session& S, F fn) {
  size_t n = 0;
  S.ctx.check(fn(S.ctx.c, 0, nullptr, 0, &n));
  std::vector<T> v(n);
  if (n) S.ctx.check(fn(S.ctx.c, 0, v.data(), n, &n));
  return v;
}

std::vector<Cycle> cycles_of(const Session& S, const Trace& trace, bool classified) {
  const auto cc = fetch<cs_cycle>(S, cs_get_cycles);
  const auto comp = fetch<int64_t>(S, cs_get_components);
  std::vector<Cycle> out(cc.size());
  const size_t P = S.phases.size();
  for (size_t i = 0; i < cc.size(); ++i) {
    Cycle& c = out[i];
    c.index = cc[i].index;
    c.start_ts = cc[i].start_ts;
    c.end_ts = cc[i].end_ts;
    c.stage = classified ? stage_of(cc[i].stage) : Stage::Unknown;
    if (cc[i].anchor_pos != UINT64_MAX) {  // segment(): anchored cycles carry components
      c.anchor_event_id = trace.events[cc[i].anchor_pos].event_id;
      for (size_t k = 0; k < P; ++k) c.component_durations[S.phases[k]] = comp[i * P + k];
    }
    c.anchor_span_end = cc[i].anchor_span_end;
    c.first_event = cc[i].first_event;
    c.last_event = cc[i].last_event;
  }
  return out;
}

// the device extras table follows the PipelineOptions prefix in force
void sync_extras(Session& S, const Trace& trace, const PipelineOptions& opt) {
  if (S.in.extra_prefix == opt.extra_args_prefix && S.extras_uploaded) return;
  ingest_extras(S.in, trace, opt.extra_args_prefix);
  std::string packed;
  for (const auto& k : S.in.extra_keys) {
    packed += k;
    packed.push_back('\0');
  }
  S.ctx.check(cs_upload_extras(S.ctx.c, static_cast<uint32_t>(S.in.extra_keys.size()), packed.c_str(),
                               S.in.extra_refs.data(), S.in.extra_refs.size(), S.in.extra_vals.data(),
                               S.in.extra_vals.size()));
  S.extras_uploaded = true;
}

std::vector<CycleRecord> records_of(const Session& S) {
  const auto rr = fetch<cs_record>(S, cs_get_records);
  std::vector<CycleRecord> out(rr.size());
  const size_t K = S.in.extra_keys.size();
  std::vector<double> xv;
  std::vector<uint8_t> xh;
  if (K) {
    size_t n = 0;
    S.ctx.check(cs_get_record_extras(S.ctx.c, 0, nullptr, nullptr, 0, &n));
    xv.resize(n);
    xh.resize(n);
    if (n) S.ctx.check(cs_get_record_extras(S.ctx.c, 0, xv.data(), xh.data(), n, &n));
  }
  for (size_t i = 0; i < rr.size(); ++i) {
    out[i].cycle_index = rr[i].cycle_index;
    out[i].start_ts = rr[i].start_ts;
    out[i].stage = stage_of(rr[i].stage);
    out[i].workload.batch = rr[i].batch;
    out[i].workload.input_len = rr[i].input_len;
    out[i].workload.output_len = rr[i].output_len;
    out[i].workload.stage = out[i].stage;
    out[i].latency_s = rr[i].latency_s;
    for (size_t k = 0; k < K; ++k)
      if (xh[i * K + k]) out[i].extra[S.in.extra_keys[k]] = xv[i * K + k];
  }
  return out;
}

// Caller-given cycles -> the device cycle table (cs_set_cycles).
void set_cycles(Session& S, std::span<const Cycle> cycles, bool with_components) {
  std::vector<cs_cycle> cc(cycles.size());
  std::vector<int64_t> comp;
  const size_t P = S.phases.size();
  if (with_components) comp.assign(cycles.size() * P, 0);
  std::map<EventId, size_t> pos;  // anchor ids -> canonical positions (only if any cycle has one)
  for (size_t i = 0; i < cycles.size(); ++i) {
    const Cycle& c = cycles[i];
    cs_cycle& d = cc[i];
    d.index = c.index;
    d.start_ts = c.start_ts;
    d.end_ts = c.end_ts;
    d.anchor_span_end = c.anchor_span_end;
    d.first_event = c.first_event;
    d.last_event = c.last_event;
    d.stage = stage_code(c.stage);
    d.anchor_pos = UINT64_MAX;
    if (c.anchor_event_id) {
      // any event of the cycle's own range stands in: the device only needs
      // "has an anchor" (components are accounted) and a valid position
      d.anchor_pos = c.first_event < S.in.ev.size() ? c.first_event : 0;
    }
    if (with_components)
      for (size_t k = 0; k < P; ++k) {
        auto it = c.component_durations.find(S.phases[k]);
        comp[i * P + k] = it == c.component_durations.end() ? 0 : it->second;
      }
  }
  S.ctx.check(cs_set_cycles(S.ctx.c, cc.data(), cc.size(), with_components ? comp.data() : nullptr));
}

}  // namespace

// ------------------------------------------------------------ cycles.hpp
// rank_anchor_candidates (cycles.cpp:47-87): the device's ordered fold of
// every candidate (bit-identical mean / cv / periodicity / score).
std::vector<AnchorCandidate> rank_anchor_candidates(const Trace& trace, const CycleConfig& config) {
  Session& S = session(trace, config);
  CycleConfig c = config;
  c.anchor_hint.clear();
  apply_config(S, c, PipelineOptions{});
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_SEGMENT));
  const auto cand = fetch<cs_anchor_candidate>(S, cs_get_candidates_exact);
  std::vector<AnchorCandidate> out(cand.size());
  for (size_t i = 0; i < cand.size(); ++i) {
    out[i].name = S.in.names[cand[i].name_id];
    out[i].call_count = cand[i].call_count;
    out[i].mean_duration_ns = cand[i].mean_duration_ns;
    out[i].duration_cv = cand[i].duration_cv;
    out[i].periodicity = cand[i].periodicity;
    out[i].score = cand[i].score;
  }
  return out;
}

// discover_anchor (cycles.cpp:89-110)
AnchorCandidate discover_anchor(const Trace& trace, const CycleConfig& config) {
  auto all = rank_anchor_candidates(trace, config);
  if (!config.anchor_hint.empty()) {
    for (auto& c : all)
      if (c.name == config.anchor_hint) return c;
    AnchorCandidate c;  // honor the hint even when the function is rare
    c.name = config.anchor_hint;
    Session& S = session(trace, config);
    auto it = std::lower_bound(S.in.names.begin(), S.in.names.end(), config.anchor_hint);
    if (it != S.in.names.end() && *it == config.anchor_hint) {
      const uint32_t id = static_cast<uint32_t>(it - S.in.names.begin());
      for (const auto& e : S.in.ev) c.call_count += e.kind == CS_SPAN && e.name_id == id;
    }
    if (c.call_count == 0)
      throw NoAnchorFound("anchor hint '" + config.anchor_hint + "' never occurs in the trace");
    return c;
  }
  if (all.empty())
    throw NoAnchorFound("no python call exceeds the minimum call count of " +
                        std::to_string(config.min_anchor_calls));
  return all.front();
}

// segment (cycles.cpp:120-170): the anchor's Spans (any category) bound the
// cycles; no frequency fallback and no classification here.
std::vector<Cycle> segment(const Trace& trace, const std::string& anchor_name, const CycleConfig& config) {
  Session& S = session(trace, config);
  auto it = std::lower_bound(S.in.names.begin(), S.in.names.end(), anchor_name);
  if (it == S.in.names.end() || *it != anchor_name) return {};
  apply_config(S, config, PipelineOptions{}, nullptr, it - S.in.names.begin());
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_SEGMENT));
  if (summary(S).used_frequency_fallback) return {};  // fewer than one anchor
  return cycles_of(S, trace, false);
}

// classify_stages (cycles.cpp:190-254) over the caller's cycles, in place
void classify_stages(std::vector<Cycle>& cycles, const Trace& trace, const CycleConfig& config) {
  if (cycles.empty()) return;
  Session& S = session(trace, config);
  apply_config(S, config, PipelineOptions{});
  set_cycles(S, cycles, false);
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_GIVEN | CS_RUN_CLASSIFY));
  const auto cc = fetch<cs_cycle>(S, cs_get_cycles);
  for (size_t i = 0; i < cycles.size(); ++i) cycles[i].stage = stage_of(cc[i].stage);
}

// extract_workload (cycles.cpp:256-281)
WorkloadFeatures extract_workload(const Cycle& cycle, const Trace& trace, const CycleConfig& config) {
  Session& S = session(trace, config);
  PipelineOptions opt;
  opt.include_prefill = true;
  apply_config(S, config, opt);
  set_cycles(S, std::span<const Cycle>(&cycle, 1), true);
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_GIVEN));
  const auto cc = fetch<cs_cycle>(S, cs_get_cycles);
  if (cc.empty() || cc[0].workload_status == 1)
    throw MissingWorkloadArgs("cycle " + std::to_string(cycle.index) + ": no event carries '" +
                              config.batch_size_key + "'");
  if (cc[0].workload_status != 0)
    throw MissingWorkloadArgs("cycle " + std::to_string(cycle.index) + ": event carries " +
                              config.batch_size_key + " but lacks length args or has negative ones");
  const auto rr = fetch<cs_record>(S, cs_get_records);
  WorkloadFeatures w;
  w.batch = rr.at(0).batch;
  w.input_len = rr[0].input_len;
  w.output_len = rr[0].output_len;
  w.stage = cycle.stage;
  return w;
}

// segment_by_frequency (cycles.cpp:283-343): the device's NoAnchorFound path
std::vector<Cycle> segment_by_frequency(const Trace& trace, const CycleConfig& config) {
  Session& S = session(trace, config);
  apply_config(S, config, PipelineOptions{}, nullptr, -2);  // a hint that never occurs
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_SEGMENT));
  if (summary(S).status == CS_E_NO_ANCHOR_FOUND) return {};
  return cycles_of(S, trace, false);
}

// segment_and_classify (cycles.cpp:345-357)
std::vector<Cycle> segment_and_classify(const Trace& trace, const CycleConfig& config) {
  Session& S = session(trace, config);
  apply_config(S, config, PipelineOptions{});
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_SEGMENT));
  if (summary(S).status == CS_E_NO_ANCHOR_FOUND) rethrow(CS_E_NO_ANCHOR_FOUND, "no anchor and no periodic GPU kernels");
  return cycles_of(S, trace, true);
}

// build_cycle_records (cycles.cpp:359-364), `extra` (post_* args) included
std::vector<CycleRecord> build_cycle_records(const Trace& trace, const CycleConfig& config,
                                             const PipelineOptions& options) {
  Session& S = session(trace, config);
  apply_config(S, config, options);
  sync_extras(S, trace, options);
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_SEGMENT));
  if (summary(S).status == CS_E_NO_ANCHOR_FOUND) rethrow(CS_E_NO_ANCHOR_FOUND, "no anchor and no periodic GPU kernels");
  return records_of(S);
}

// build_cycle_records over caller-given cycles (cycles.cpp:366-409): their
// stages and component_durations decide inclusion and the latency target.
std::vector<CycleRecord> build_cycle_records(const Trace& trace, std::span<const Cycle> cycles,
                                             const CycleConfig& config, const PipelineOptions& options) {
  if (cycles.empty()) return {};
  Session& S = session(trace, config);
  apply_config(S, config, options);
  sync_extras(S, trace, options);
  set_cycles(S, cycles, true);
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_GIVEN));
  return records_of(S);
}

// --------------------------------------------------------------- rca.hpp
// cycle_stats (rca.cpp:71-130) for one cycle: beta, collective beta and, for
// classes the MetricMap maps to a counter series of the trace, mu.  The
// counter table is the trace's own (CounterTable::from_trace, trace.cpp:111-131).
CycleClassStats cycle_stats(const Cycle& cycle, const Trace& trace, const CounterTable& counters,
                            const MetricMap& metrics) {
  CycleClassStats stats;
  stats.cycle_index = cycle.index;
  stats.cycle_duration = cycle.duration();
  if (stats.cycle_duration <= 0) return stats;
  CycleConfig config;
  Session& S = session(trace, config);
  const bool mu = !metrics.class_to_metric.empty() && !counters.all().empty();
  apply_config(S, config, PipelineOptions{}, mu ? &metrics : nullptr, -1, &counters);
  set_cycles(S, std::span<const Cycle>(&cycle, 1), false);
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_GIVEN | CS_RUN_BETA | (mu ? CS_RUN_MU : 0u)));
  size_t nb = 0, nc = 0;
  S.ctx.check(cs_get_beta(S.ctx.c, 0, nullptr, nullptr, 0, &nb));
  std::vector<int64_t> tot(nb);
  std::vector<double> beta(nb), muv(nb);
  std::vector<uint8_t> has(nb);
  S.ctx.check(cs_get_beta(S.ctx.c, 0, tot.data(), beta.data(), nb, &nb));
  if (mu) S.ctx.check(cs_get_mu(S.ctx.c, 0, muv.data(), has.data(), nb, &nb));
  S.ctx.check(cs_get_collective_beta(S.ctx.c, 0, nullptr, nullptr, 0, &nc));
  std::vector<double> cb(nc);
  std::vector<uint8_t> cp(nc);
  S.ctx.check(cs_get_collective_beta(S.ctx.c, 0, cb.data(), cp.data(), nc, &nc));
  for (size_t k = 0; k < S.slot_names.size() && k < tot.size(); ++k)
    if (tot[k] > 0) {
      ClassStat st;
      st.total_duration = tot[k];
      st.beta = beta[k];
      if (mu && has[k]) {
        st.mu = muv[k];
        st.metric = metrics.class_to_metric.at(S.slot_names[k]);
      }
      stats.classes.emplace(S.slot_names[k], st);
    }
  for (size_t k = 0; k < S.in.comm.size() && k < cp.size(); ++k)
    if (cp[k]) stats.collective_rank_beta[S.in.comm[k]] = cb[k];
  return stats;
}

// Not in the reference: cycle_stats (beta part) for every cycle of
// segment_and_classify in one device pass.
std::vector<CycleClassStats> cycle_stats_all(const Trace& trace, const CycleConfig& config) {
  Session& S = session(trace, config);
  apply_config(S, config, PipelineOptions{});
  S.ctx.check(cs_run(S.ctx.c, CS_RUN_SEGMENT | CS_RUN_BETA));
  const auto cycles = cycles_of(S, trace, true);
  size_t nb = 0, nc = 0;
  S.ctx.check(cs_get_beta(S.ctx.c, 0, nullptr, nullptr, 0, &nb));
  std::vector<int64_t> tot(nb);
  std::vector<double> beta(nb);
  S.ctx.check(cs_get_beta(S.ctx.c, 0, tot.data(), beta.data(), nb, &nb));
  S.ctx.check(cs_get_collective_beta(S.ctx.c, 0, nullptr, nullptr, 0, &nc));
  std::vector<double> cb(nc);
  std::vector<uint8_t> cp(nc);
  S.ctx.check(cs_get_collective_beta(S.ctx.c, 0, cb.data(), cp.data(), nc, &nc));
  const size_t C = S.slot_names.size(), R = S.in.comm.size();
  std::vector<CycleClassStats> out(cycles.size());
  for (size_t i = 0; i < cycles.size(); ++i) {
    out[i].cycle_index = cycles[i].index;
    out[i].cycle_duration = cycles[i].duration();
    for (size_t s = 0; s < C; ++s)
      if (tot[i * C + s] > 0) {
        ClassStat st;
        st.total_duration = tot[i * C + s];
        st.beta = beta[i * C + s];
        out[i].classes.emplace(S.slot_names[s], st);
      }
    for (size_t k = 0; k < R; ++k)
      if (cp[i * R + k]) out[i].collective_rank_beta[S.in.comm[k]] = cb[i * R + k];
  }
  return out;
}

// ----------------------------------------------------------- detector.hpp
// evaluate_strategy (detector.cpp:166-224): the Detector replay and the
// confusion counts / lag on the device (cs_detect_residuals).
StrategyMetrics evaluate_strategy(const LabeledStream& stream, const ControlConfig& config,
                                  double dynamic_ucl) {
  if (stream.anomalous.size() != stream.residuals.size() || stream.residuals.empty())
    throw NoLabels("labeled stream is empty or label count mismatches");
  thread_local std::unique_ptr<Ctx> ctx;
  if (!ctx) ctx = std::make_unique<Ctx>();
  cs_control_config c{};
  c.strategy = config.strategy == Strategy::FixedPoint ? CS_FIXED_POINT
               : config.strategy == Strategy::FixedWindow ? CS_FIXED_WINDOW
                                                          : CS_DYNAMIC_WINDOW;
  c.window = config.window;
  c.fixed_threshold = config.fixed_threshold;
  c.sigma_k = config.sigma_k;
  c.theta_max = config.theta_max;
  c.min_ucl = config.min_ucl;
  c.warmup = config.warmup;
  c.epsilon = config.epsilon;
  std::vector<uint8_t> labels(stream.anomalous.begin(), stream.anomalous.end());
  cs_strategy_metrics m{};
  ctx->check(cs_detect_residuals(ctx->c, stream.residuals.data(), stream.residuals.size(), &c, dynamic_ucl,
                                 labels.data(), nullptr, nullptr, &m));
  StrategyMetrics out;
  out.strategy = config.strategy;
  out.precision = m.precision;
  out.recall = m.recall;
  out.f1 = m.f1;
  out.fpr = m.fpr;
  out.mean_lag = m.mean_lag;
  out.alerts = m.alerts;
  out.true_positives = m.tp;
  out.false_positives = m.fp;
  out.false_negatives = m.fn;
  out.true_negatives = m.tn;
  return out;
}

// evaluate_strategies (detector.cpp:226-240)
std::vector<StrategyMetrics> evaluate_strategies(const LabeledStream& stream, const ControlConfig& base_config,
                                                 std::span<const double> calibration_residuals) {
  const double ucl = compute_ucl(calibration_residuals, base_config.sigma_k, base_config.theta_max,
                                 base_config.min_ucl);
  std::vector<StrategyMetrics> table;
  for (auto strategy : {Strategy::FixedPoint, Strategy::FixedWindow, Strategy::DynamicWindow}) {
    ControlConfig config = base_config;
    config.strategy = strategy;
    table.push_back(evaluate_strategy(stream, config, ucl));
  }
  return table;
}

}  // namespace cyclescope
