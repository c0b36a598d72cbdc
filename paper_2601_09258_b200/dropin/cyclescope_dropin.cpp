// cyclescope_dropin.cpp — C++ drop-in for the reference's hot-path API.
//
// Compile this file together with the caller's copy of the reference headers
// (proj/include/cyclescope/*.hpp) INSTEAD of proj/src/cycles.cpp's hot entry
// points, and link libcyclescope_b200.so.  The functions keep the reference's
// signatures and semantics (cycles.hpp:132-143, rca.hpp:47-48); the work runs
// on the B200 through the C ABI (include/cyclescope_b200.h).  Errors come back
// as the reference's EngineError subclasses; the two control-flow exceptions
// (MissingWorkloadArgs skip, NoAnchorFound -> frequency fallback) are handled
// inside the device pipeline exactly like cycles.cpp:345-383.
//
// Ingest (A1-A2): the Trace is interned once per call into 32-byte records —
// names in lexicographic order (so name ids are the tie-break ranks), the
// forward_mode / batch / commHash+rank / value args folded into flags and the
// workload table.
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
};

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
  void check(int rc) const {
    if (rc) rethrow(rc, cs_last_error(c));
  }
};

struct Run {
  Ingested in;
  Ctx ctx;
  cs_cycle_config cyc{};
  std::vector<std::string> phases;
};

std::unique_ptr<Run> run_pipeline(const Trace& trace, const CycleConfig& config,
                                  const PipelineOptions& opt, uint32_t mask) {
  auto r = std::make_unique<Run>();
  r->in = ingest(trace, config);
  // CycleConfig / PipelineOptions -> device config (cycles.hpp:18-43,123-128)
  for (const auto& p : config.phase_functions)
    if (std::find(r->phases.begin(), r->phases.end(), p) == r->phases.end())
      r->phases.push_back(p);
  std::vector<cs_name_info> names(r->in.names.size());
  int32_t slot = 0;
  cs_cycle_config& c = r->cyc;
  c.anchor_hint_name = -1;
  for (size_t i = 0; i < names.size(); ++i) {
    const std::string& nm = r->in.names[i];
    names[i].phase = -1;
    for (size_t k = 0; k < r->phases.size(); ++k)
      if (r->phases[k] == nm) names[i].phase = static_cast<int32_t>(k);
    for (const auto& kw : config.prefill_keywords)
      if (nm.find(kw) != std::string::npos) names[i].flags |= CS_NAME_PREFILL_KW;
    for (const auto& kw : config.decode_keywords)
      if (nm.find(kw) != std::string::npos) names[i].flags |= CS_NAME_DECODE_KW;
    names[i].beta_slot = r->in.is_span[i] ? slot++ : -1;
    if (!config.anchor_hint.empty() && nm == config.anchor_hint) c.anchor_hint_name = i;
  }
  if (!config.anchor_hint.empty() && c.anchor_hint_name < 0) c.anchor_hint_name = -2;
  c.min_anchor_calls = config.min_anchor_calls;
  c.prefill_duration_factor = config.prefill_duration_factor;
  c.prefill_gap_factor = config.prefill_gap_factor;
  c.stage_window = config.stage_window;
  c.stage_min_history = config.stage_min_history;
  c.frequency_bin_ns = config.frequency_bin_ns;
  c.n_phases = static_cast<int32_t>(r->phases.size());
  c.latency_phase = -1;
  for (size_t k = 0; k < r->phases.size(); ++k)
    if (!opt.latency_component.empty() && r->phases[k] == opt.latency_component)
      c.latency_phase = static_cast<int32_t>(k);
  c.include_prefill = opt.include_prefill ? 1 : 0;
  c.n_beta_slots = slot;
  c.n_comm_slots = static_cast<int32_t>(r->in.comm.size());
  r->ctx.check(cs_set_config(r->ctx.c, &c, nullptr));
  r->ctx.check(cs_set_name_table(r->ctx.c, static_cast<uint32_t>(names.size()), names.data()));
  const uint64_t off[2] = {0, r->in.ev.size()};
  r->ctx.check(cs_upload(r->ctx.c, 1, off, r->in.ev.data(), r->in.wl.size(), r->in.wl.data()));
  r->ctx.check(cs_run(r->ctx.c, mask));
  cs_instance_summary s{};
  r->ctx.check(cs_get_summary(r->ctx.c, 0, &s));
  if (s.status == CS_E_NO_ANCHOR_FOUND) rethrow(s.status, "no anchor and no periodic GPU kernels");
  return r;
}

Stage stage_of(int32_t s) {
  return s == CS_STAGE_PREFILL ? Stage::Prefill : (s == CS_STAGE_DECODE ? Stage::Decode : Stage::Unknown);
}

std::vector<Cycle> cycles_of(const Run& r, const Trace& trace) {
  size_t n = 0;
  r.ctx.check(cs_get_cycles(r.ctx.c, 0, nullptr, 0, &n));
  std::vector<cs_cycle> cc(n);
  r.ctx.check(cs_get_cycles(r.ctx.c, 0, cc.data(), n, &n));
  std::vector<int64_t> comp;
  size_t nc = 0;
  r.ctx.check(cs_get_components(r.ctx.c, 0, nullptr, 0, &nc));
  comp.resize(nc);
  r.ctx.check(cs_get_components(r.ctx.c, 0, comp.data(), nc, &nc));
  std::vector<Cycle> out(n);
  const size_t P = r.phases.size();
  for (size_t i = 0; i < n; ++i) {
    Cycle& c = out[i];
    c.index = cc[i].index;
    c.start_ts = cc[i].start_ts;
    c.end_ts = cc[i].end_ts;
    c.stage = stage_of(cc[i].stage);
    if (cc[i].anchor_pos != UINT64_MAX) {
      c.anchor_event_id = trace.events[cc[i].anchor_pos].event_id;
      for (size_t k = 0; k < P; ++k) c.component_durations[r.phases[k]] = comp[i * P + k];
    }
    c.anchor_span_end = cc[i].anchor_span_end;
    c.first_event = cc[i].first_event;
    c.last_event = cc[i].last_event;
  }
  return out;
}

}  // namespace

// cycles.hpp:132-133 (segment_and_classify; cycles.cpp:345-357)
std::vector<Cycle> segment_and_classify(const Trace& trace, const CycleConfig& config) {
  auto r = run_pipeline(trace, config, PipelineOptions{}, CS_RUN_SEGMENT);
  return cycles_of(*r, trace);
}

// cycles.hpp:137-139 (build_cycle_records; cycles.cpp:359-409).  `extra`
// (post_* args, ablation-only) is not harvested by the device path.
std::vector<CycleRecord> build_cycle_records(const Trace& trace, const CycleConfig& config,
                                             const PipelineOptions& options) {
  auto r = run_pipeline(trace, config, options, CS_RUN_SEGMENT);
  size_t n = 0;
  r->ctx.check(cs_get_records(r->ctx.c, 0, nullptr, 0, &n));
  std::vector<cs_record> rr(n);
  r->ctx.check(cs_get_records(r->ctx.c, 0, rr.data(), n, &n));
  std::vector<CycleRecord> out(n);
  for (size_t i = 0; i < n; ++i) {
    out[i].cycle_index = rr[i].cycle_index;
    out[i].start_ts = rr[i].start_ts;
    out[i].stage = stage_of(rr[i].stage);
    out[i].workload.batch = rr[i].batch;
    out[i].workload.input_len = rr[i].input_len;
    out[i].workload.output_len = rr[i].output_len;
    out[i].workload.stage = out[i].stage;
    out[i].latency_s = rr[i].latency_s;
  }
  return out;
}

// Per-cycle class occupancy for every cycle of a trace in one device pass
// (rca.cpp:71-130, beta part; the mu part needs counters: SURVEY §8f #1).
std::vector<CycleClassStats> cycle_stats_all(const Trace& trace, const CycleConfig& config) {
  auto r = run_pipeline(trace, config, PipelineOptions{}, CS_RUN_SEGMENT | CS_RUN_BETA);
  const auto cycles = cycles_of(*r, trace);
  size_t nb = 0, nc = 0;
  r->ctx.check(cs_get_beta(r->ctx.c, 0, nullptr, nullptr, 0, &nb));
  std::vector<int64_t> tot(nb);
  std::vector<double> beta(nb);
  r->ctx.check(cs_get_beta(r->ctx.c, 0, tot.data(), beta.data(), nb, &nb));
  r->ctx.check(cs_get_collective_beta(r->ctx.c, 0, nullptr, nullptr, 0, &nc));
  std::vector<double> cb(nc);
  std::vector<uint8_t> cp(nc);
  r->ctx.check(cs_get_collective_beta(r->ctx.c, 0, cb.data(), cp.data(), nc, &nc));
  std::vector<std::string> slot_names;
  for (size_t i = 0; i < r->in.names.size(); ++i)
    if (r->in.is_span[i]) slot_names.push_back(r->in.names[i]);
  const size_t C = slot_names.size(), R = r->in.comm.size();
  std::vector<CycleClassStats> out(cycles.size());
  for (size_t i = 0; i < cycles.size(); ++i) {
    out[i].cycle_index = cycles[i].index;
    out[i].cycle_duration = cycles[i].duration();
    for (size_t s = 0; s < C; ++s)
      if (tot[i * C + s] > 0) {
        ClassStat st;
        st.total_duration = tot[i * C + s];
        st.beta = beta[i * C + s];
        out[i].classes.emplace(slot_names[s], st);
      }
    for (size_t k = 0; k < R; ++k)
      if (cp[i * R + k]) out[i].collective_rank_beta[r->in.comm[k]] = cb[i * R + k];
  }
  return out;
}

}  // namespace cyclescope
