// ref_bridge.cpp — TEST INFRASTRUCTURE ONLY (the parity checker, never the
// product).  A C ABI over the reference implementation compiled unmodified
// from /root/reference/proj/src into oracle/_ref/ (see oracle/Makefile).
//
// It lets tests, __graft_entry__.smoke() and bench.py's reference arm:
//   * synthesize traces with the reference's simkit (simkit.cpp:34-86,276-506),
//   * build a reference `Trace` from our binary records (inverse ingest),
//   * export a `Trace` into our binary records (the oracle-side ingest, an
//     implementation independent of the product's),
//   * run the reference hot path exactly like `monitor_loop`
//     (tools/main.cpp:142-214) plus `cycle_stats` beta (rca.cpp:71-130) and
//     capture every intermediate for bit-exact comparison.
// Only the reference's public headers are used; no reference code is copied.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <nlohmann/json.hpp>

#include "cyclescope/baseline.hpp"
#include "cyclescope/config.hpp"
#include "cyclescope/cycles.hpp"
#include "cyclescope/detector.hpp"
#include "cyclescope/errors.hpp"
#include "cyclescope/gbdt.hpp"
#include "cyclescope/rca.hpp"
#include "cyclescope/rng.hpp"
#include "cyclescope/simkit.hpp"
#include "cyclescope/trace.hpp"
#include "cyclescope/trace_io.hpp"
#include "cyclescope_b200.h"

using namespace cyclescope;
using nlohmann::json;

namespace {

struct Exported {
  std::vector<cs_event> events;
  std::vector<cs_workload> workloads;
  std::vector<std::string> names;
  std::string names_packed;  // NUL separated
  std::vector<std::tuple<std::string, std::string, int>> comm;  // slot -> key
  std::vector<int32_t> comm_name, comm_rank;
  std::string comm_hash_packed;
  std::vector<uint64_t> event_ids;
  // record extras side table (cycles.cpp:392-405): prefixed numeric args
  std::vector<std::string> extra_keys;
  std::string extra_keys_packed;
  std::vector<cs_extra_ref> extra_refs;
  std::vector<cs_extra_value> extra_vals;
};

struct Results {
  int status = 0;
  std::string err_type, err_msg;
  std::vector<cs_anchor_candidate> candidates;
  std::string anchor;
  bool fallback = false;
  std::vector<cs_cycle> cycles;
  std::vector<int64_t> components;  // n_cycles x n_phases
  std::vector<int64_t> beta_totals; // n_cycles x n_slots
  std::vector<double> beta;
  std::vector<double> coll_beta;    // n_cycles x n_comm
  std::vector<double> mu;           // n_cycles x n_slots (do_beta & 2: CounterTable)
  std::vector<uint8_t> mu_has;
  std::vector<uint8_t> coll_present;
  std::vector<cs_record> records;
  std::vector<cs_alert> alerts;
  std::vector<std::string> rec_extra_keys;  // sorted union of the records' extra keys
  std::vector<double> rec_extra;            // n_records x keys
  std::vector<uint8_t> rec_extra_has;
  std::string model_json;
  std::string ndjson;
  double ucl = 0.0;
  uint64_t first_bad_record = UINT64_MAX;
  double seconds = 0.0;
};

struct Handle {
  LabeledDataset ds;
  std::vector<ValidationIssue> parse_issues;  // from parse_trace_json
  std::vector<Cycle> cycles;                  // of the last ref_run
  MetricMap metric_map;
  Exported ex;
  bool exported = false;
  Results res;
  std::string last_config;
};

int stage_code(Stage s) {
  switch (s) {
    case Stage::Prefill: return CS_STAGE_PREFILL;
    case Stage::Decode: return CS_STAGE_DECODE;
    default: return CS_STAGE_UNKNOWN;
  }
}

// The oracle-side ingest: Trace -> 32-byte records.  Written independently of
// the product's ingest; the shared contract is include/cyclescope_b200.h.
void export_trace(Handle& h, const CycleConfig& cfg, const std::string& extra_prefix = "post_") {
  Exported& ex = h.ex;
  ex = Exported{};
  const auto& ev = h.ds.trace.events;
  std::set<std::string> name_set;
  std::set<std::tuple<std::string, std::string, int>> comm_set;
  for (const auto& e : ev) {
    name_set.insert(e.name);
    if (e.kind == EventKind::Span && e.category == EventCategory::CollectiveComm) {
      auto comm = arg_string(e, "commHash");
      auto rank = arg_int(e, "rank");
      if (comm && rank) comm_set.insert({e.name, *comm, static_cast<int>(*rank)});
    }
  }
  ex.names.assign(name_set.begin(), name_set.end());
  std::map<std::string, uint32_t> name_id;
  for (uint32_t i = 0; i < ex.names.size(); ++i) {
    name_id[ex.names[i]] = i;
    ex.names_packed += ex.names[i];
    ex.names_packed.push_back('\0');
  }
  std::map<std::tuple<std::string, std::string, int>, uint32_t> comm_slot;
  for (const auto& k : comm_set) {
    comm_slot[k] = static_cast<uint32_t>(ex.comm.size());
    ex.comm.push_back(k);
    ex.comm_name.push_back(static_cast<int32_t>(name_id[std::get<0>(k)]));
    ex.comm_rank.push_back(std::get<2>(k));
    ex.comm_hash_packed += std::get<1>(k);
    ex.comm_hash_packed.push_back('\0');
  }
  ex.events.resize(ev.size());
  ex.event_ids.resize(ev.size());
  for (size_t i = 0; i < ev.size(); ++i) {
    const auto& e = ev[i];
    cs_event& r = ex.events[i];
    std::memset(&r, 0, sizeof r);
    r.start_ts = e.start_ts;
    r.duration = e.kind == EventKind::Span ? e.duration : 0;
    r.name_id = name_id[e.name];
    r.kind = static_cast<uint8_t>(e.kind);
    r.category = static_cast<uint8_t>(e.category);
    uint16_t flags = 0;
    if (auto fm = arg_string(e, cfg.forward_mode_key)) {
      std::string m = *fm;
      for (auto& c : m) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
      if (m.find("prefill") != std::string::npos || m.find("extend") != std::string::npos)
        flags |= CS_EV_FM_PREFILL;
      else if (m.find("decode") != std::string::npos)
        flags |= CS_EV_FM_DECODE;
      else
        flags |= CS_EV_FM_OTHER;
    }
    if (auto b = arg_int(e, cfg.batch_size_key)) {
      flags |= CS_EV_HAS_BATCH;
      auto in = arg_int(e, cfg.input_len_key);
      auto out = arg_int(e, cfg.output_len_key);
      cs_workload w{*b, in ? *in : INT64_MIN, out ? *out : INT64_MIN};
      if (in && out && *b >= 0 && *in >= 0 && *out >= 0) flags |= CS_EV_WL_OK;
      r.payload |= static_cast<uint64_t>(ex.workloads.size());
      ex.workloads.push_back(w);
    }
    if (e.kind == EventKind::Span && e.category == EventCategory::CollectiveComm) {
      auto comm = arg_string(e, "commHash");
      auto rank = arg_int(e, "rank");
      if (comm && rank) {
        flags |= CS_EV_HAS_COMM;
        r.payload |= static_cast<uint64_t>(comm_slot[{e.name, *comm, static_cast<int>(*rank)}]) << 32;
      }
    }
    if (e.kind == EventKind::Counter) {
      if (auto v = arg_number(e, "value")) {
        flags |= CS_EV_HAS_VALUE;
        std::memcpy(&r.duration, &*v, sizeof(double));
      }
    }
    r.flags = flags;
    ex.event_ids[i] = e.event_id;
  }
  // extras: every numeric arg with the prefix, per event in key order
  if (!extra_prefix.empty()) {
    std::set<std::string> keys;
    for (const auto& e : ev)
      for (const auto& [k, v] : e.args)
        if (k.rfind(extra_prefix, 0) == 0 && !std::holds_alternative<std::string>(v)) keys.insert(k);
    ex.extra_keys.assign(keys.begin(), keys.end());
    for (const auto& k : ex.extra_keys) {
      ex.extra_keys_packed += k;
      ex.extra_keys_packed.push_back('\0');
    }
    for (size_t i = 0; i < ev.size(); ++i) {
      cs_extra_ref ref{i, static_cast<uint32_t>(ex.extra_vals.size()), 0};
      for (const auto& [k, v] : ev[i].args) {
        if (k.rfind(extra_prefix, 0) != 0) continue;
        double d;
        if (const auto* x = std::get_if<double>(&v)) d = *x;
        else if (const auto* n = std::get_if<std::int64_t>(&v)) d = static_cast<double>(*n);
        else if (const auto* b = std::get_if<bool>(&v)) d = *b ? 1.0 : 0.0;
        else continue;
        const uint32_t key = static_cast<uint32_t>(
            std::lower_bound(ex.extra_keys.begin(), ex.extra_keys.end(), k) - ex.extra_keys.begin());
        ex.extra_vals.push_back({key, 0, d});
        ++ref.count;
      }
      if (ref.count) ex.extra_refs.push_back(ref);
    }
  }
  h.exported = true;
}

void set_error(Results& r, const EngineError& e) {
  r.status = 1;
  r.err_type = e.type();
  r.err_msg = e.what();
}

// monitor_loop (main.cpp:142-214) trace branch, plus beta for every cycle.
void run_reference(Handle& h, const RunConfig& config, const char* model_json,
                   uint64_t train_cycles, int do_beta) {
  Results& R = h.res;
  R = Results{};
  const Trace& trace = h.ds.trace;
  std::map<uint64_t, uint64_t> pos_of_id;
  for (size_t i = 0; i < trace.events.size(); ++i) pos_of_id[trace.events[i].event_id] = i;
  if (!h.exported) export_trace(h, config.cycle);
  std::map<std::string, uint32_t> name_id;
  for (uint32_t i = 0; i < h.ex.names.size(); ++i) name_id[h.ex.names[i]] = i;

  // dense beta slots over names that occur as spans, lexicographic order
  std::map<std::string, int> beta_slot;
  {
    std::set<std::string> span_names;
    for (const auto& e : trace.events)
      if (e.kind == EventKind::Span) span_names.insert(e.name);
    int s = 0;
    for (const auto& n : span_names) beta_slot[n] = s++;
  }
  std::map<std::tuple<std::string, std::string, int>, int> comm_slot;
  for (size_t i = 0; i < h.ex.comm.size(); ++i) comm_slot[h.ex.comm[i]] = static_cast<int>(i);

  // phase order = first occurrence in phase_functions
  std::vector<std::string> phases;
  for (const auto& p : config.cycle.phase_functions)
    if (std::find(phases.begin(), phases.end(), p) == phases.end()) phases.push_back(p);

  const auto t0 = std::chrono::steady_clock::now();
  std::vector<Cycle> cycles;
  try {
    try {
      auto cands = rank_anchor_candidates(trace, config.cycle);
      for (const auto& c : cands) {
        cs_anchor_candidate a{};
        a.name_id = name_id.count(c.name) ? name_id[c.name] : UINT32_MAX;
        a.call_count = c.call_count;
        a.mean_duration_ns = c.mean_duration_ns;
        a.duration_cv = c.duration_cv;
        a.score = c.score;
        a.periodicity = c.periodicity;
        R.candidates.push_back(a);
      }
      const auto anchor = discover_anchor(trace, config.cycle);
      R.anchor = anchor.name;
      cycles = segment(trace, anchor.name, config.cycle);
    } catch (const NoAnchorFound&) {
      R.fallback = true;
      cycles = segment_by_frequency(trace, config.cycle);
      if (cycles.empty()) throw;
    }
    classify_stages(cycles, trace, config.cycle);
  } catch (const EngineError& e) {
    set_error(R, e);
    return;
  }
  h.cycles = cycles;
  h.metric_map = config.metric_map;
  for (const auto& c : cycles) {
    cs_cycle o{};
    o.index = c.index;
    o.start_ts = c.start_ts;
    o.end_ts = c.end_ts;
    o.anchor_pos = c.anchor_event_id ? pos_of_id[*c.anchor_event_id] : UINT64_MAX;
    o.anchor_span_end = c.anchor_span_end;
    o.first_event = c.first_event;
    o.last_event = c.last_event;
    o.stage = stage_code(c.stage);
    try {
      extract_workload(c, trace, config.cycle);
      o.workload_status = 0;
    } catch (const MissingWorkloadArgs&) {
      bool carrier = false;
      for (size_t j = c.first_event; j < c.last_event && !carrier; ++j)
        carrier = arg_int(trace.events[j], config.cycle.batch_size_key).has_value();
      o.workload_status = carrier ? 2 : 1;
    }
    R.cycles.push_back(o);
    for (const auto& p : phases) {
      auto it = c.component_durations.find(p);
      R.components.push_back(it == c.component_durations.end() ? 0 : it->second);
    }
  }
  if (do_beta) {
    const size_t ns = beta_slot.size(), nc = comm_slot.size();
    R.beta_totals.assign(cycles.size() * ns, 0);
    R.beta.assign(cycles.size() * ns, 0.0);
    R.coll_beta.assign(cycles.size() * nc, 0.0);
    R.coll_present.assign(cycles.size() * nc, 0);
    // do_beta & 2: the mu branch too, with the trace's CounterTable and the
    // RunConfig metric map (cmd_diagnose, main.cpp:285-293)
    const bool with_mu = (do_beta & 2) != 0;
    const CounterTable counters = with_mu ? CounterTable::from_trace(trace) : CounterTable{};
    const MetricMap metrics = with_mu ? config.metric_map : MetricMap{};
    if (with_mu) {
      R.mu.assign(cycles.size() * ns, 0.0);
      R.mu_has.assign(cycles.size() * ns, 0);
    }
    for (size_t ci = 0; ci < cycles.size(); ++ci) {
      const auto st = cycle_stats(cycles[ci], trace, counters, metrics);
      for (const auto& [name, cs] : st.classes) {
        R.beta_totals[ci * ns + beta_slot[name]] = cs.total_duration;
        R.beta[ci * ns + beta_slot[name]] = cs.beta;
        if (with_mu && cs.mu) {
          R.mu[ci * ns + beta_slot[name]] = *cs.mu;
          R.mu_has[ci * ns + beta_slot[name]] = 1;
        }
      }
      for (const auto& [key, b] : st.collective_rank_beta) {
        const int s = comm_slot[key];
        R.coll_beta[ci * nc + s] = b;
        R.coll_present[ci * nc + s] = 1;
      }
    }
  }
  std::vector<CycleRecord> records;
  try {
    records = build_cycle_records(trace, cycles, config.cycle, config.pipeline);
  } catch (const EngineError& e) {
    set_error(R, e);
    return;
  }
  {  // the records' extras (post_* args), columns in key order
    std::set<std::string> keys;
    for (const auto& r : records)
      for (const auto& [k, v] : r.extra) keys.insert(k);
    R.rec_extra_keys.assign(keys.begin(), keys.end());
    const size_t K = R.rec_extra_keys.size();
    R.rec_extra.assign(records.size() * K, 0.0);
    R.rec_extra_has.assign(records.size() * K, 0);
    for (size_t i = 0; i < records.size(); ++i)
      for (const auto& [k, v] : records[i].extra) {
        const size_t c = std::lower_bound(R.rec_extra_keys.begin(), R.rec_extra_keys.end(), k) -
                         R.rec_extra_keys.begin();
        R.rec_extra[i * K + c] = v;
        R.rec_extra_has[i * K + c] = 1;
      }
  }
  LatencyModel model;
  try {
    if (model_json && *model_json) {
      model = LatencyModel::from_json(json::parse(model_json));
    } else {
      std::vector<CycleRecord> train;
      for (const auto& r : records)
        if (r.cycle_index < train_cycles) train.push_back(r);
      const auto samples = to_sample_set(train, config.feature_set);
      model = fit_latency_model(samples, config.gbdt, config.fit);
    }
    R.model_json = model.to_json().dump();
  } catch (const EngineError& e) {
    set_error(R, e);
    return;
  }
  // monitor_loop process lambda (main.cpp:151-177), every record in order
  const double ucl = ucl_from_stats(model.mu_train, model.sigma_train, config.detector);
  Detector detector(config.detector, ucl);
  Escalator escalator(config.escalation);
  R.ucl = detector.limit();  // limit in force (strategy dependent)
  try {
    for (size_t i = 0; i < records.size(); ++i) {
      const auto& rec = records[i];
      cs_record o{};
      o.cycle_index = rec.cycle_index;
      o.start_ts = rec.start_ts;
      o.batch = rec.workload.batch;
      o.input_len = rec.workload.input_len;
      o.output_len = rec.workload.output_len;
      o.latency_s = rec.latency_s;
      o.stage = stage_code(rec.stage);
      std::vector<double> row;
      for (const auto& name : model.feature_names) {
        if (name == "batch") row.push_back(static_cast<double>(rec.workload.batch));
        else if (name == "w_kv") row.push_back(static_cast<double>(rec.workload.kv_token_slots()));
        else if (name == "input_len") row.push_back(static_cast<double>(rec.workload.input_len));
        else if (name == "output_len") row.push_back(static_cast<double>(rec.workload.output_len));
        else if (name == "stage") row.push_back(rec.stage == Stage::Prefill ? 1.0 : 0.0);
        else {  // features_by_name (main.cpp:70-75)
          auto it = rec.extra.find(name);
          if (it == rec.extra.end()) {
            R.first_bad_record = i;
            throw FeatureMismatch("input lacks feature '" + name + "'");
          }
          row.push_back(it->second);
        }
      }
      o.predicted_s = model.predict(row);
      R.records.push_back(o);
      if (!(rec.latency_s > 0.0)) {
        R.first_bad_record = i;
        o.residual = ppe(rec.latency_s, o.predicted_s, config.detector.epsilon);  // throws
      }
      ResidualSample sample;
      sample.cycle = rec.cycle_index;
      sample.ts = rec.start_ts;
      sample.workload = rec.workload;
      sample.actual_s = rec.latency_s;
      sample.predicted_s = o.predicted_s;
      sample.error = ppe(rec.latency_s, o.predicted_s, config.detector.epsilon);
      const auto step = detector.step(sample);
      escalator.on_cycle(rec.cycle_index);  // main.cpp:164
      if (step.alert) {
        auto j = step.alert->to_json();
        if (const auto action = escalator.on_alert(*step.alert)) {
          j["retain"] = {{"begin", action->retain.begin}, {"end", action->retain.end}};
          j["mode"] = to_string(escalator.mode());
        }
        R.ndjson += j.dump() + "\n";
      }
      auto& out = R.records.back();
      out.residual = sample.error;
      out.statistic = step.statistic;
      out.armed = step.armed;
      out.flagged = step.flagged;
      out.alert = step.alert.has_value();
      if (step.alert) {
        out.episode_id = step.alert->episode_id;
        cs_alert a{};
        a.cycle = step.alert->cycle;
        a.ts = step.alert->ts;
        a.smoothed_error = step.alert->smoothed_error;
        a.limit = step.alert->limit;
        a.strategy = static_cast<int32_t>(step.alert->strategy);
        a.batch = step.alert->workload.batch;
        a.input_len = step.alert->workload.input_len;
        a.output_len = step.alert->workload.output_len;
        a.episode_id = step.alert->episode_id;
        a.record_index = i;
        R.alerts.push_back(a);
      }
    }
  } catch (const EngineError& e) {
    set_error(R, e);
  }
  R.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

template <typename T>
int copy_out(const std::vector<T>& v, T* buf, size_t cap, size_t* n) {
  if (n) *n = v.size();
  if (!buf) return 0;
  if (cap < v.size()) return 1;
  if (!v.empty()) std::memcpy(buf, v.data(), v.size() * sizeof(T));
  return 0;
}

}  // namespace

extern "C" {

struct ref_synth_params {
  uint64_t n_cycles;
  uint64_t workload_seed;
  uint64_t synth_seed;
  int32_t fault_family;   // -1 none
  int32_t target_rank;
  uint64_t fault_onset;
  uint64_t fault_duration;
  double severity;        // <= 0: default_severity
  uint64_t n_ranks;
  double noise;           // < 0: default
};

void* ref_synth(const ref_synth_params* p) {
  auto h = std::make_unique<Handle>();
  const auto workloads = generate_workload(WorkloadProfile{}, p->n_cycles, p->workload_seed);
  GroundTruthModel model;
  if (p->noise >= 0.0) model.noise = p->noise;
  std::vector<FaultSpec> faults;
  if (p->fault_family >= 0) {
    FaultSpec f;
    f.family = static_cast<FaultFamily>(p->fault_family);
    f.onset = p->fault_onset;
    f.duration = p->fault_duration;
    f.severity = p->severity > 0.0 ? p->severity : default_severity(f.family);
    f.target_rank = p->target_rank;
    faults.push_back(f);
  }
  SynthOptions opt;
  opt.n_ranks = p->n_ranks;
  h->ds = synthesize_trace(workloads, model, faults, opt, p->synth_seed);
  return h.release();
}

// The reference's own Chrome-trace JSON (trace_io.cpp): serialize_trace_json
// of this handle's trace, and a handle from parse_trace_json of a document
// (its issues count in *n_issues).
int ref_to_json(void* hv, char* buf, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  const std::string text = serialize_trace_json(h->ds.trace);
  if (n) *n = text.size();
  if (!buf) return 0;
  if (cap < text.size()) return 1;
  std::memcpy(buf, text.data(), text.size());
  return 0;
}

void* ref_from_json(const char* text, size_t len, uint64_t* n_issues) {
  auto h = std::make_unique<Handle>();
  auto parsed = parse_trace_json(std::string(text, len));
  if (n_issues) *n_issues = parsed.issues.size();
  h->ds.trace = std::move(parsed.trace);
  h->parse_issues = std::move(parsed.issues);
  return h.release();
}

// The reference's post-alert ranking (cmd_diagnose, main.cpp:285-303):
// cycle_stats of the windows' cycles (by cycle index, from the last ref_run),
// suspicion_rank, attribute_straggler with resolve_topology; the JSON report
// (render_json_report) in buf.  Returns 2 with the error type in err on an
// EngineError.
int ref_rca(void* hv, const uint64_t* normal, size_t n_normal, const uint64_t* abnormal,
            size_t n_abnormal, int with_mu, char* buf, size_t cap, size_t* n, char* err,
            size_t err_cap) {
  auto* h = static_cast<Handle*>(hv);
  const Trace& trace = h->ds.trace;
  try {
    const CounterTable counters = with_mu ? CounterTable::from_trace(trace) : CounterTable{};
    const MetricMap metrics = with_mu ? h->metric_map : MetricMap{};
    std::map<std::size_t, const Cycle*> by_index;
    for (const auto& c : h->cycles) by_index[c.index] = &c;
    auto stats_for = [&](const uint64_t* idx, size_t k) {
      std::vector<CycleClassStats> st;
      for (size_t i = 0; i < k; ++i)
        if (auto it = by_index.find(idx[i]); it != by_index.end())
          st.push_back(cycle_stats(*it->second, trace, counters, metrics));
      return st;
    };
    const auto ns = stats_for(normal, n_normal), as = stats_for(abnormal, n_abnormal);
    auto entries = suspicion_rank(ns, as);
    attribute_straggler(entries, resolve_topology(trace), ns, as);
    const std::string j = render_json_report(entries).dump();
    if (n) *n = j.size();
    if (buf) {
      if (cap < j.size()) return 1;
      std::memcpy(buf, j.data(), j.size());
    }
    return 0;
  } catch (const EngineError& e) {
    if (err && err_cap) {
      std::strncpy(err, e.type().c_str(), err_cap - 1);
      err[err_cap - 1] = 0;
    }
    return 2;
  }
}

// cmd_ingest (main.cpp:80-97) without the validation gate and the file
// write: parse each document, extract_beacons, calibrate, apply_calibration,
// merge_traces.  A handle on the merged trace, or NULL with the error type.
void* ref_merge(const char* const* texts, const size_t* lens, uint32_t n, const char* ref_domain,
                double tolerance_ns, int estimate_drift, char* err, size_t err_cap) {
  try {
    std::vector<Trace> traces;
    std::vector<Beacon> beacons;
    for (uint32_t i = 0; i < n; ++i) {
      auto parsed = parse_trace_json(std::string(texts[i], lens[i]));
      auto b = extract_beacons(parsed.trace);
      beacons.insert(beacons.end(), b.begin(), b.end());
      traces.push_back(std::move(parsed.trace));
    }
    CalibrationOptions opt;
    if (ref_domain) opt.reference_domain = ref_domain;
    opt.tolerance_ns = tolerance_ns;
    opt.estimate_drift = estimate_drift != 0;
    const auto calibration = calibrate(beacons, opt);
    for (auto& t : traces) apply_calibration(t, calibration);
    auto h = std::make_unique<Handle>();
    h->ds.trace = merge_traces(std::move(traces));
    return h.release();
  } catch (const EngineError& e) {
    if (err && err_cap) {
      std::strncpy(err, e.type().c_str(), err_cap - 1);
      err[err_cap - 1] = 0;
    }
    return nullptr;
  }
}

// resolve_topology (align.cpp:178-191) per exported comm slot: a JSON array
// of [node, device] or null (unmapped)
int ref_topology(void* hv, char* buf, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  const TopologyMap topo = resolve_topology(h->ds.trace);
  json arr = json::array();
  for (const auto& [name, hash, rank] : h->ex.comm) {
    (void)name;
    if (const auto* loc = topo.find(hash, rank)) arr.push_back(json::array({loc->node, loc->device}));
    else arr.push_back(nullptr);
  }
  const std::string j = arr.dump();
  if (n) *n = j.size();
  if (buf) {
    if (cap < j.size()) return 1;
    std::memcpy(buf, j.data(), j.size());
  }
  return 0;
}

// validate_trace(trace, parse issues) (trace.cpp:243-276): the report as
// (severity, code, event id) records (cs_ingest_issue layout), per-category
// counts and the error count.
int ref_validate(void* hv, cs_ingest_issue* out, size_t cap, size_t* n, uint64_t* cats,
                 uint64_t* n_errors) {
  auto* h = static_cast<Handle*>(hv);
  const ValidationReport rep = validate_trace(h->ds.trace, h->parse_issues);
  static const char* kCodes[] = {"malformed_event",       "malformed_args",        "duplicate_event_id",
                                 "negative_duration",     "duplicate_correlation", "unmatched_correlation",
                                 "non_monotone_counter"};
  if (n) *n = rep.issues.size();
  if (n_errors) *n_errors = rep.error_count();
  if (cats) {
    for (int c = 0; c < 8; ++c) cats[c] = 0;
    for (const auto& [c, k] : rep.category_counts) cats[static_cast<int>(c)] = k;
  }
  if (!out) return 0;
  if (cap < rep.issues.size()) return 1;
  for (size_t i = 0; i < rep.issues.size(); ++i) {
    const auto& x = rep.issues[i];
    cs_ingest_issue o{};
    o.severity = x.severity == ValidationIssue::Severity::Error ? CS_SEV_ERROR : CS_SEV_WARNING;
    o.code = 255;
    for (uint8_t c = 0; c < 7; ++c)
      if (x.code == kCodes[c]) o.code = c;
    o.has_event_id = x.event_id ? 1 : 0;
    o.event_id = x.event_id ? *x.event_id : 0;
    out[i] = o;
  }
  return 0;
}

// Inverse ingest: binary records -> reference Trace.  forward_mode classes map
// to "prefill"/"decode"/"other"; comm slots to commHash strings.
void* ref_build(uint64_t n, const cs_event* ev, const uint64_t* event_ids,
                uint32_t n_names, const char* names_packed, const cs_workload* wl,
                uint32_t n_comm, const char* comm_hash_packed, const int32_t* comm_rank,
                int sort) {
  auto h = std::make_unique<Handle>();
  std::vector<std::string> names;
  const char* p = names_packed;
  for (uint32_t i = 0; i < n_names; ++i) {
    names.emplace_back(p);
    p += names.back().size() + 1;
  }
  std::vector<std::string> comms;
  p = comm_hash_packed;
  for (uint32_t i = 0; i < n_comm; ++i) {
    comms.emplace_back(p);
    p += comms.back().size() + 1;
  }
  auto& events = h->ds.trace.events;
  events.resize(n);
  for (uint64_t i = 0; i < n; ++i) {
    const cs_event& r = ev[i];
    TraceEvent& e = events[i];
    e.event_id = event_ids ? event_ids[i] : i + 1;
    e.kind = static_cast<EventKind>(r.kind);
    e.category = static_cast<EventCategory>(r.category);
    e.name = names.at(r.name_id);
    e.start_ts = r.start_ts;
    e.duration = r.kind == CS_SPAN ? r.duration : 0;
    const uint32_t fm = r.flags & CS_EV_FM_MASK;
    if (fm == CS_EV_FM_PREFILL) e.args["forward_mode"] = std::string("prefill");
    if (fm == CS_EV_FM_DECODE) e.args["forward_mode"] = std::string("decode");
    if (fm == CS_EV_FM_OTHER) e.args["forward_mode"] = std::string("idle");
    if (r.flags & CS_EV_HAS_BATCH) {
      const cs_workload& w = wl[r.payload & 0xffffffffu];
      e.args["batch_size"] = w.batch;
      if (w.input_len != INT64_MIN) e.args["input_len"] = w.input_len;
      if (w.output_len != INT64_MIN) e.args["output_len"] = w.output_len;
    }
    if (r.flags & CS_EV_HAS_COMM) {
      const uint32_t s = static_cast<uint32_t>(r.payload >> 32);
      e.args["commHash"] = comms.at(s);
      e.args["rank"] = static_cast<int64_t>(comm_rank[s]);
    }
    if (r.kind == CS_COUNTER && (r.flags & CS_EV_HAS_VALUE)) {
      double v;
      std::memcpy(&v, &r.duration, sizeof v);
      e.args["value"] = v;
    }
  }
  if (sort) h->ds.trace.sort_events();
  return h.release();
}

void ref_free(void* h) { delete static_cast<Handle*>(h); }

uint64_t ref_n_events(void* hv) { return static_cast<Handle*>(hv)->ds.trace.events.size(); }

int ref_labels(void* hv, uint8_t* buf, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  std::vector<uint8_t> v(h->ds.labels.anomalous.begin(), h->ds.labels.anomalous.end());
  return copy_out(v, buf, cap, n);
}

// Export with the CycleConfig of a RunConfig JSON ("" = defaults).
int ref_export(void* hv, const char* run_config_json) {
  auto* h = static_cast<Handle*>(hv);
  try {
    RunConfig cfg = (run_config_json && *run_config_json)
                        ? RunConfig::from_json(json::parse(run_config_json))
                        : RunConfig{};
    export_trace(*h, cfg.cycle, cfg.pipeline.extra_args_prefix);
  } catch (const std::exception&) {
    return 1;
  }
  return 0;
}

int ref_get_events(void* hv, cs_event* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->ex.events, buf, cap, n);
}
int ref_get_event_ids(void* hv, uint64_t* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->ex.event_ids, buf, cap, n);
}
int ref_get_workloads(void* hv, cs_workload* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->ex.workloads, buf, cap, n);
}
int ref_get_extra_keys(void* hv, char* buf, size_t cap, size_t* n_bytes, uint32_t* n_keys) {
  auto* h = static_cast<Handle*>(hv);
  if (n_keys) *n_keys = static_cast<uint32_t>(h->ex.extra_keys.size());
  std::vector<char> v(h->ex.extra_keys_packed.begin(), h->ex.extra_keys_packed.end());
  return copy_out(v, buf, cap, n_bytes);
}
int ref_get_extra_refs(void* hv, cs_extra_ref* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->ex.extra_refs, buf, cap, n);
}
int ref_get_extra_values(void* hv, cs_extra_value* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->ex.extra_vals, buf, cap, n);
}
int ref_get_record_extras(void* hv, char* keys, size_t keys_cap, size_t* keys_bytes, double* vals,
                          uint8_t* has, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  std::string packed;
  for (const auto& k : h->res.rec_extra_keys) {
    packed += k;
    packed.push_back('\0');
  }
  std::vector<char> kv(packed.begin(), packed.end());
  if (copy_out(kv, keys, keys_cap, keys_bytes)) return 1;
  if (n) *n = h->res.rec_extra.size();
  if (!vals) return 0;
  if (cap < h->res.rec_extra.size()) return 1;
  std::copy(h->res.rec_extra.begin(), h->res.rec_extra.end(), vals);
  std::copy(h->res.rec_extra_has.begin(), h->res.rec_extra_has.end(), has);
  return 0;
}
int ref_get_names(void* hv, char* buf, size_t cap, size_t* n_bytes, uint32_t* n_names) {
  auto* h = static_cast<Handle*>(hv);
  if (n_names) *n_names = static_cast<uint32_t>(h->ex.names.size());
  std::vector<char> v(h->ex.names_packed.begin(), h->ex.names_packed.end());
  return copy_out(v, buf, cap, n_bytes);
}
int ref_get_comm(void* hv, int32_t* name, int32_t* rank, char* hash_buf, size_t cap,
                 size_t* n_bytes, uint32_t* n_comm) {
  auto* h = static_cast<Handle*>(hv);
  if (n_comm) *n_comm = static_cast<uint32_t>(h->ex.comm.size());
  if (name) std::copy(h->ex.comm_name.begin(), h->ex.comm_name.end(), name);
  if (rank) std::copy(h->ex.comm_rank.begin(), h->ex.comm_rank.end(), rank);
  std::vector<char> v(h->ex.comm_hash_packed.begin(), h->ex.comm_hash_packed.end());
  return copy_out(v, hash_buf, cap, n_bytes);
}

// Runs the reference hot path.  model_json: LatencyModel JSON, or NULL/"" to
// fit on records with cycle_index < train_cycles (evaluate_trial split,
// simkit.cpp:836-846).  Returns 0; the reference's outcome is in ref_status.
int ref_run(void* hv, const char* run_config_json, const char* model_json,
            uint64_t train_cycles, int do_beta) {
  auto* h = static_cast<Handle*>(hv);
  RunConfig cfg;
  try {
    if (run_config_json && *run_config_json) cfg = RunConfig::from_json(json::parse(run_config_json));
  } catch (const std::exception& e) {
    h->res = Results{};
    h->res.status = 2;
    h->res.err_type = "config_error";
    h->res.err_msg = e.what();
    return 0;
  }
  run_reference(*h, cfg, model_json, train_cycles, do_beta);
  return 0;
}

int ref_status(void* hv, char* type_buf, size_t type_cap, char* msg_buf, size_t msg_cap) {
  auto* h = static_cast<Handle*>(hv);
  if (type_buf && type_cap) {
    std::strncpy(type_buf, h->res.err_type.c_str(), type_cap - 1);
    type_buf[type_cap - 1] = 0;
  }
  if (msg_buf && msg_cap) {
    std::strncpy(msg_buf, h->res.err_msg.c_str(), msg_cap - 1);
    msg_buf[msg_cap - 1] = 0;
  }
  return h->res.status;
}

int ref_anchor(void* hv, char* buf, size_t cap, int* fallback) {
  auto* h = static_cast<Handle*>(hv);
  if (fallback) *fallback = h->res.fallback;
  if (buf && cap) {
    std::strncpy(buf, h->res.anchor.c_str(), cap - 1);
    buf[cap - 1] = 0;
  }
  return 0;
}
double ref_ucl(void* hv) { return static_cast<Handle*>(hv)->res.ucl; }
double ref_seconds(void* hv) { return static_cast<Handle*>(hv)->res.seconds; }
uint64_t ref_first_bad_record(void* hv) { return static_cast<Handle*>(hv)->res.first_bad_record; }

int ref_get_candidates(void* hv, cs_anchor_candidate* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->res.candidates, buf, cap, n);
}
int ref_get_cycles(void* hv, cs_cycle* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->res.cycles, buf, cap, n);
}
int ref_get_components(void* hv, int64_t* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->res.components, buf, cap, n);
}
int ref_get_beta(void* hv, int64_t* totals, double* beta, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  if (copy_out(h->res.beta_totals, totals, cap, n)) return 1;
  return copy_out(h->res.beta, beta, cap, n);
}
int ref_get_mu(void* hv, double* mu, uint8_t* has, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  if (copy_out(h->res.mu, mu, cap, n)) return 1;
  return copy_out(h->res.mu_has, has, cap, n);
}
int ref_get_collective_beta(void* hv, double* beta, uint8_t* present, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  if (copy_out(h->res.coll_beta, beta, cap, n)) return 1;
  return copy_out(h->res.coll_present, present, cap, n);
}
int ref_get_records(void* hv, cs_record* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->res.records, buf, cap, n);
}
int ref_get_alerts(void* hv, cs_alert* buf, size_t cap, size_t* n) {
  return copy_out(static_cast<Handle*>(hv)->res.alerts, buf, cap, n);
}
int ref_get_ndjson(void* hv, char* buf, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  std::vector<char> v(h->res.ndjson.begin(), h->res.ndjson.end());
  v.push_back('\0');
  return copy_out(v, buf, cap, n);
}

// Suite trial dataset exactly like make_trial_fault / make_trial_dataset
// (simkit.cpp:760-792) with SuiteConfig{} (BASELINE config 4).
void* ref_trial_dataset(uint64_t trial) {
  SuiteConfig cfg;
  const FaultFamily family = cfg.families[trial % cfg.families.size()];
  FaultSpec fault;
  fault.family = family;
  fault.severity = default_severity(family);
  Rng rng(Rng::substream_seed(cfg.seed, 0xfau + trial));
  const auto jitter = static_cast<size_t>(
      rng.uniform_int(0, static_cast<int64_t>(2 * cfg.fault_onset_jitter)));
  fault.onset = cfg.fault_onset - cfg.fault_onset_jitter + jitter;
  fault.duration = cfg.fault_duration;
  if (family == FaultFamily::NvlinkSaturation && cfg.nvlink_ranks > 1)
    fault.target_rank = static_cast<int>(rng.uniform_int(0, static_cast<int64_t>(cfg.nvlink_ranks) - 1));
  const auto seed = Rng::substream_seed(cfg.seed, trial);
  const auto work = generate_workload(cfg.profile, cfg.cycles_per_trial, seed);
  SynthOptions opt;
  opt.n_ranks = family == FaultFamily::NvlinkSaturation ? cfg.nvlink_ranks : 1;
  auto h = std::make_unique<Handle>();
  h->ds = synthesize_trace(work, cfg.model, {&fault, 1}, opt, Rng::substream_seed(seed, 1));
  return h.release();
}

// evaluate_trial (simkit.cpp:796-955): out[s*8 + {tp,fp,fn,tn,alerts,f1,fpr,lag}] per
// strategy (fixed_point, fixed_window, dynamic_window); returns 0 or 1 on EngineError.
int ref_evaluate_trial(void* hv, uint64_t trial, double* out, char* err, size_t err_cap) {
  auto* h = static_cast<Handle*>(hv);
  SuiteConfig cfg;
  try {
    const auto o = evaluate_trial(cfg, h->ds, trial, cfg.families[trial % cfg.families.size()]);
    for (size_t k = 0; k < o.strategies.size() && k < 3; ++k) {
      const auto& m = o.strategies[k];
      double* q = out + 8 * k;
      q[0] = static_cast<double>(m.true_positives);
      q[1] = static_cast<double>(m.false_positives);
      q[2] = static_cast<double>(m.false_negatives);
      q[3] = static_cast<double>(m.true_negatives);
      q[4] = static_cast<double>(m.alerts);
      q[5] = m.f1;
      q[6] = m.fpr;
      q[7] = m.mean_lag;
    }
  } catch (const EngineError& e) {
    if (err && err_cap) std::snprintf(err, err_cap, "%s: %s", e.type().c_str(), e.what());
    return 1;
  }
  return 0;
}

int ref_get_model_json(void* hv, char* buf, size_t cap, size_t* n) {
  auto* h = static_cast<Handle*>(hv);
  std::vector<char> v(h->res.model_json.begin(), h->res.model_json.end());
  v.push_back('\0');
  return copy_out(v, buf, cap, n);
}

// Reference fit on explicit samples (fit_latency_model, baseline.cpp:168-208),
// returns the model JSON (dump()).  Used to pin the product's host fit.
int ref_fit(uint64_t n, uint32_t n_features, const char* feature_names_packed,
            const double* x, const double* y, const cs_gbdt_params* gp,
            const cs_fit_options* fo, char* buf, size_t cap, size_t* n_out,
            char* err, size_t err_cap) {
  try {
    SampleSet s;
    const char* p = feature_names_packed;
    for (uint32_t i = 0; i < n_features; ++i) {
      s.feature_names.emplace_back(p);
      p += s.feature_names.back().size() + 1;
    }
    s.x.cols = n_features;
    for (uint64_t i = 0; i < n; ++i) {
      s.x.push_row(std::span<const double>(x + i * n_features, n_features));
      s.y.push_back(y[i]);
    }
    GbdtParams params;
    params.n_trees = gp->n_trees;
    params.max_depth = gp->max_depth;
    params.learning_rate = gp->learning_rate;
    params.min_samples_leaf = gp->min_samples_leaf;
    params.prediction_floor = gp->prediction_floor;
    FitOptions opt;
    opt.calibration_fraction = fo->calibration_fraction;
    opt.ppe_epsilon = fo->ppe_epsilon;
    opt.min_samples = fo->min_samples;
    if (fo->stratify_col >= 0 && static_cast<uint32_t>(fo->stratify_col) < n_features)
      opt.stratify_feature = s.feature_names[fo->stratify_col];
    const auto m = fit_latency_model(s, params, opt);
    std::string j = m.to_json().dump();
    std::vector<char> v(j.begin(), j.end());
    v.push_back('\0');
    return copy_out(v, buf, cap, n_out);
  } catch (const EngineError& e) {
    if (err && err_cap) {
      std::snprintf(err, err_cap, "%s: %s", e.type().c_str(), e.what());
    }
    return 2;
  }
}

// The CPU baseline (bench.py --impl reference / cpu_baseline): simkit traces
// generated once (ref_cpu_prepare, untimed), then each ref_cpu_run times the
// A4-A16 chain — segment_and_classify + build_cycle_records + beta
// cycle_stats + LatencyModel::predict + ppe + Detector::step — with one
// monitored instance per std::thread.  The model fit (A17) is
// done in prepare and reported separately.
struct CpuBaseline {
  std::vector<std::unique_ptr<Handle>> inst;
  std::vector<LatencyModel> models;
  uint64_t events = 0;
  double fit_seconds = 0.0;
  std::string anchor_hint;  // slices of one trace: the anchor the whole trace uses
};

void* ref_cpu_prepare(uint32_t n_instances, uint32_t n_threads, uint64_t cycles_per_instance,
                      uint64_t n_ranks, uint64_t seed) {
  auto* cb = new CpuBaseline();
  cb->inst.resize(n_instances);
  cb->models.resize(n_instances);
  std::vector<double> fit_s(n_instances, 0.0);
  auto prepare = [&](uint32_t i) {
    ref_synth_params p{};
    p.n_cycles = cycles_per_instance;
    p.workload_seed = Rng::substream_seed(seed, 2 * i);
    p.synth_seed = Rng::substream_seed(seed, 2 * i + 1);
    p.fault_family = static_cast<int32_t>(FaultFamily::NvlinkSaturation);
    p.target_rank = 3 % static_cast<int32_t>(std::max<uint64_t>(1, n_ranks));
    p.fault_onset = cycles_per_instance * 4 / 5;
    p.fault_duration = 150;
    p.severity = -1;
    p.n_ranks = n_ranks;
    p.noise = -1;
    cb->inst[i].reset(static_cast<Handle*>(ref_synth(&p)));
    const auto t0 = std::chrono::steady_clock::now();
    CycleConfig cc;
    PipelineOptions po;
    auto recs = build_cycle_records(cb->inst[i]->ds.trace, cc, po);
    std::vector<CycleRecord> train;
    for (auto& r : recs)
      if (r.cycle_index < 2400) train.push_back(r);
    cb->models[i] = fit_latency_model(to_sample_set(train, FeatureSet::Physical), GbdtParams{});
    fit_s[i] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < std::max(1u, n_threads); ++t)
    th.emplace_back([&, t] {
      for (uint32_t i = t; i < n_instances; i += std::max(1u, n_threads)) prepare(i);
    });
  for (auto& x : th) x.join();
  for (uint32_t i = 0; i < n_instances; ++i) {
    cb->events += cb->inst[i]->ds.trace.events.size();
    cb->fit_seconds += fit_s[i];
  }
  return cb;
}

uint64_t ref_cpu_events(void* h) { return static_cast<CpuBaseline*>(h)->events; }
double ref_cpu_fit_seconds(void* h) { return static_cast<CpuBaseline*>(h)->fit_seconds; }
void ref_cpu_free(void* h) { delete static_cast<CpuBaseline*>(h); }

// Returns wall seconds of one timed pass over all prepared instances.
// Cycle-aligned slices [slice_lo[k], slice_hi[k]) of ONE trace (the GPU arm's benchmarked instance), one
// reference Trace per slice built on n_threads threads; every slice is
// analysed with the whole trace's anchor (anchor_hint) and one model.
void* ref_cpu_prepare_slices(uint64_t n, const cs_event* ev, const uint64_t* event_ids, uint32_t n_names,
                             const char* names_packed, const cs_workload* wl, uint32_t n_comm,
                             const char* comm_hash_packed, const int32_t* comm_rank, uint32_t n_slices,
                             const uint64_t* slice_lo, const uint64_t* slice_hi, const char* model_json,
                             const char* anchor_hint, uint32_t n_threads) {
  auto* cb = new CpuBaseline();
  cb->inst.resize(n_slices);
  cb->anchor_hint = anchor_hint ? anchor_hint : "";
  const LatencyModel model = LatencyModel::from_json(json::parse(model_json));
  cb->models.assign(n_slices, model);
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < std::max(1u, n_threads); ++t)
    th.emplace_back([&, t] {
      for (uint32_t i = t; i < n_slices; i += std::max(1u, n_threads)) {
        const uint64_t lo = std::min<uint64_t>(slice_lo[i], n), hi = std::min<uint64_t>(slice_hi[i], n);
        cb->inst[i].reset(static_cast<Handle*>(ref_build(hi - lo, ev + lo, event_ids ? event_ids + lo : nullptr,
                                                         n_names, names_packed, wl, n_comm, comm_hash_packed,
                                                         comm_rank, 0)));
      }
    });
  for (auto& x : th) x.join();
  for (uint32_t i = 0; i < n_slices; ++i) cb->events += cb->inst[i]->ds.trace.events.size();
  return cb;
}

double ref_cpu_run(void* h, uint32_t n_threads, uint64_t* n_alerts_out) {
  auto* cb = static_cast<CpuBaseline*>(h);
  const uint32_t n = static_cast<uint32_t>(cb->inst.size());
  std::vector<uint64_t> alerts(n, 0);
  auto work = [&](uint32_t i) {
    const Trace& tr = cb->inst[i]->ds.trace;
    CycleConfig cc;
    cc.anchor_hint = cb->anchor_hint;
    PipelineOptions po;
    ControlConfig dc;
    const auto cycles = segment_and_classify(tr, cc);
    const CounterTable no_counters;
    const MetricMap no_metrics;
    uint64_t classes = 0;
    for (const auto& c : cycles) classes += cycle_stats(c, tr, no_counters, no_metrics).classes.size();
    const auto recs = build_cycle_records(tr, cycles, cc, po);
    const LatencyModel& m = cb->models[i];
    Detector det(dc, ucl_from_stats(m.mu_train, m.sigma_train, dc));
    for (const auto& r : recs) {
      const double row[2] = {static_cast<double>(r.workload.batch),
                             static_cast<double>(r.workload.kv_token_slots())};
      ResidualSample s;
      s.cycle = r.cycle_index;
      s.ts = r.start_ts;
      s.workload = r.workload;
      s.error = ppe(r.latency_s, m.predict(row), dc.epsilon);
      if (det.step(s).alert) ++alerts[i];
    }
    if (classes == 0) alerts[i] += 0;
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  const uint32_t nt = std::max(1u, n_threads);
  for (uint32_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (uint32_t i = t; i < n; i += nt) work(i);
    });
  for (auto& x : th) x.join();
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  uint64_t na = 0;
  for (auto a : alerts) na += a;
  if (n_alerts_out) *n_alerts_out = na;
  return secs;
}

// Whole-trace reference results for a trace too large for one reference
// Trace (configs[1]: ~42 GB as TraceEvent + std::map args): the trace is cut
// into cycle-aligned chunks at anchor group starts, each chunk extended
// through the next chunk's first anchor so that its last cycle closes
// exactly as in the whole trace (segment, cycles.cpp:120-170; lower_bound
// group starts).  Chunks run segment_and_classify (anchor_hint = the trace's
// anchor), cycle_stats (beta part), build_cycle_records, predict and ppe on
// n_threads threads; ONE Detector then steps every record in trace order
// (monitor_loop, main.cpp:151-177), so flags, statistics, episodes and alerts
// are the whole trace's.  Stages restart their trailing windows per chunk:
// exact when every cycle's stage comes from forward_mode or keywords (as in
// simkit traces), which out_flags bit 0 reports.  Outputs go to caller
// buffers in the product's layouts: cycles (cs_cycle), components [cycle][P]
// by the name table's phase, beta totals / beta [cycle][C] by its beta_slot,
// collective beta / present [cycle][R] by the records' comm slot; records
// (cs_record, incl. detector fields) and alerts (cs_alert).
int ref_full_parity(uint64_t n, const cs_event* ev, uint32_t n_names, const char* names_packed,
                    const cs_workload* wl, uint32_t n_comm, const char* comm_hash_packed,
                    const int32_t* comm_rank, const cs_name_info* name_table, int32_t P, int32_t C,
                    int32_t R, const char* model_json, const char* anchor_name, uint32_t n_threads,
                    uint64_t chunk_events, uint64_t cap_cycles, cs_cycle* o_cycles, int64_t* o_comp,
                    int64_t* o_beta_tot, double* o_beta, double* o_coll, uint8_t* o_coll_present,
                    uint64_t cap_records, cs_record* o_records, uint64_t cap_alerts, cs_alert* o_alerts,
                    uint64_t* n_out, uint32_t* out_flags, double* seconds, char* err, size_t err_cap) {
  const auto t0 = std::chrono::steady_clock::now();
  try {
    std::vector<std::string> names;
    {
      const char* p = names_packed;
      for (uint32_t i = 0; i < n_names; ++i) {
        names.emplace_back(p);
        p += names.back().size() + 1;
      }
    }
    std::map<std::string, uint32_t> name_id;
    for (uint32_t i = 0; i < n_names; ++i) name_id[names[i]] = i;
    const auto ait = name_id.find(anchor_name);
    if (ait == name_id.end()) throw std::runtime_error("anchor not in the name table");
    const uint32_t anchor = ait->second;
    std::vector<uint64_t> apos;
    for (uint64_t i = 0; i < n; ++i)
      if (ev[i].kind == CS_SPAN && ev[i].name_id == anchor) apos.push_back(i);
    const uint64_t n_anchors = apos.size();
    const uint64_t n_cyc = n_anchors >= 2 ? n_anchors - 1 : 0;
    if (n_cyc > cap_cycles) throw std::runtime_error("cycle capacity");
    auto group_start = [&](uint64_t pos) {
      while (pos > 0 && ev[pos - 1].start_ts == ev[pos].start_ts) --pos;
      return pos;
    };
    // chunk k covers the cycles of anchors [ka[k], ka[k+1])
    std::vector<uint64_t> ka;
    {
      uint64_t k = 0;
      while (k < n_cyc) {
        ka.push_back(k);
        const uint64_t lo = group_start(apos[k]);
        uint64_t k2 = k + 1;
        while (k2 < n_cyc && apos[k2] - lo < chunk_events) ++k2;
        k = k2;
      }
      ka.push_back(n_cyc);
    }
    const size_t n_chunks = ka.size() - 1;
    std::vector<std::string> comms;
    {
      const char* p = comm_hash_packed;
      for (uint32_t i = 0; i < n_comm; ++i) {
        comms.emplace_back(p);
        p += comms.back().size() + 1;
      }
    }
    std::map<std::tuple<std::string, std::string, int>, uint32_t> comm_slot;
    std::vector<std::string> phases;  // phase order = the name table's phase index
    phases.assign(std::max(0, P), std::string());
    for (uint32_t i = 0; i < n_names; ++i)
      if (name_table[i].phase >= 0 && name_table[i].phase < P) phases[name_table[i].phase] = names[i];
    for (uint64_t i = 0; i < n; ++i)
      if ((ev[i].flags & CS_EV_HAS_COMM) && ev[i].kind == CS_SPAN) {
        const uint32_t s = static_cast<uint32_t>(ev[i].payload >> 32);
        if (s < n_comm) comm_slot[{names[ev[i].name_id], comms[s], comm_rank[s]}] = s;
      }
    const LatencyModel model = LatencyModel::from_json(json::parse(model_json));
    CycleConfig cc;
    cc.anchor_hint = anchor_name;
    cc.phase_functions.clear();
    for (const auto& ph : phases) cc.phase_functions.push_back(ph);
    PipelineOptions po;
    ControlConfig dc;
    if (n_cyc) std::memset(o_cycles, 0, n_cyc * sizeof(cs_cycle));
    if (P > 0 && n_cyc) std::memset(o_comp, 0, n_cyc * P * sizeof(int64_t));
    if (C > 0 && n_cyc) {
      std::memset(o_beta_tot, 0, n_cyc * C * sizeof(int64_t));
      std::memset(o_beta, 0, n_cyc * C * sizeof(double));
    }
    if (R > 0 && n_cyc) {
      std::memset(o_coll, 0, n_cyc * R * sizeof(double));
      std::memset(o_coll_present, 0, n_cyc * R);
    }
    struct ChunkOut {
      std::vector<cs_record> recs;
      std::vector<double> err;
      std::vector<WorkloadFeatures> wl;
      bool heuristic = false;
      std::string error;
    };
    std::vector<ChunkOut> outs(n_chunks);
    const double eps = dc.epsilon;
    auto work = [&](size_t k) {
      ChunkOut& co = outs[k];
      const uint64_t c0 = ka[k], c1 = ka[k + 1];
      const uint64_t lo = group_start(apos[c0]);
      const uint64_t hi = c1 < n_anchors ? apos[c1] + 1 : n;  // through the closing anchor
      std::unique_ptr<Handle> h(static_cast<Handle*>(
          ref_build(hi - lo, ev + lo, nullptr, n_names, names_packed, wl, n_comm, comm_hash_packed,
                    comm_rank, 0)));
      const Trace& tr = h->ds.trace;
      auto cyc = segment_and_classify(tr, cc);
      if (cyc.size() < c1 - c0) {
        co.error = "chunk produced fewer cycles than anchors";
        return;
      }
      cyc.resize(c1 - c0);
      const CounterTable no_counters;
      const MetricMap no_metrics;
      for (size_t i = 0; i < cyc.size(); ++i) {
        const Cycle& c = cyc[i];
        const uint64_t g = c0 + i;
        cs_cycle& o = o_cycles[g];
        o.index = g;
        o.start_ts = c.start_ts;
        o.end_ts = c.end_ts;
        o.anchor_pos = c.anchor_event_id ? lo + (*c.anchor_event_id - 1) : UINT64_MAX;
        o.anchor_span_end = c.anchor_span_end;
        o.first_event = lo + c.first_event;
        o.last_event = lo + c.last_event;
        o.stage = stage_code(c.stage);
        try {
          extract_workload(c, tr, cc);
          o.workload_status = 0;
        } catch (const MissingWorkloadArgs&) {
          bool carrier = false;
          for (size_t j = c.first_event; j < c.last_event && !carrier; ++j)
            carrier = arg_int(tr.events[j], cc.batch_size_key).has_value();
          o.workload_status = carrier ? 2 : 1;
        }
        // a stage the trailing-median heuristic decided depends on earlier
        // cycles (cycles.cpp:230-250): reported, since chunks restart it
        {
          std::optional<std::string> fm;
          for (size_t j = c.first_event; j < c.last_event && !fm; ++j) fm = arg_string(tr.events[j], cc.forward_mode_key);
          bool local = false;
          if (fm) {
            std::string m = *fm;
            for (auto& ch : m) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
            local = m.find("prefill") != std::string::npos || m.find("extend") != std::string::npos ||
                    m.find("decode") != std::string::npos;
          }
          if (!local) co.heuristic = true;  // keyword-only stages are reported too (conservative)
        }
        for (int p = 0; p < P; ++p) {
          auto it = c.component_durations.find(phases[p]);
          o_comp[g * P + p] = it == c.component_durations.end() ? 0 : it->second;
        }
        if (C > 0 || R > 0) {
          const auto st = cycle_stats(c, tr, no_counters, no_metrics);
          for (const auto& [name, cls] : st.classes) {
            const auto nit = name_id.find(name);
            const int32_t s = nit == name_id.end() ? -1 : name_table[nit->second].beta_slot;
            if (s < 0 || s >= C) throw std::runtime_error("class without a beta slot: " + name);
            o_beta_tot[g * C + s] = cls.total_duration;
            o_beta[g * C + s] = cls.beta;
          }
          for (const auto& [key, b] : st.collective_rank_beta) {
            const auto cit = comm_slot.find(key);
            if (cit == comm_slot.end() || static_cast<int32_t>(cit->second) >= R)
              throw std::runtime_error("collective key without a slot");
            o_coll[g * R + cit->second] = b;
            o_coll_present[g * R + cit->second] = 1;
          }
        }
      }
      const auto recs = build_cycle_records(tr, std::span<const Cycle>(cyc), cc, po);
      for (const auto& r : recs) {
        cs_record o{};
        o.cycle_index = c0 + r.cycle_index;
        o.start_ts = r.start_ts;
        o.batch = r.workload.batch;
        o.input_len = r.workload.input_len;
        o.output_len = r.workload.output_len;
        o.latency_s = r.latency_s;
        o.stage = stage_code(r.stage);
        const double row[2] = {static_cast<double>(r.workload.batch),
                               static_cast<double>(r.workload.kv_token_slots())};
        o.predicted_s = model.predict(row);
        co.recs.push_back(o);
        co.wl.push_back(r.workload);
      }
    };
    std::vector<std::thread> th;
    const uint32_t nt = std::max(1u, n_threads);
    std::atomic<size_t> next{0};
    for (uint32_t t = 0; t < nt; ++t)
      th.emplace_back([&] {
        for (size_t k; (k = next.fetch_add(1)) < n_chunks;) work(k);
      });
    for (auto& x : th) x.join();
    uint32_t flags = 0;
    for (const auto& co : outs) {
      if (!co.error.empty()) throw std::runtime_error(co.error);
      if (co.heuristic) flags |= 1u;
    }
    // one Detector over every record, in trace order
    const double ucl = ucl_from_stats(model.mu_train, model.sigma_train, dc);
    Detector det(dc, ucl);
    uint64_t nr = 0, na = 0;
    for (const auto& co : outs) {
      for (size_t i = 0; i < co.recs.size(); ++i) {
        if (nr >= cap_records) throw std::runtime_error("record capacity");
        cs_record o = co.recs[i];
        ResidualSample s;
        s.cycle = o.cycle_index;
        s.ts = o.start_ts;
        s.workload = co.wl[i];
        s.actual_s = o.latency_s;
        s.predicted_s = o.predicted_s;
        s.error = ppe(o.latency_s, o.predicted_s, eps);
        const auto step = det.step(s);
        o.residual = s.error;
        o.statistic = step.statistic;
        o.armed = step.armed;
        o.flagged = step.flagged;
        o.alert = step.alert.has_value();
        if (step.alert) {
          o.episode_id = step.alert->episode_id;
          if (na >= cap_alerts) throw std::runtime_error("alert capacity");
          cs_alert& a = o_alerts[na++];
          a = cs_alert{};
          a.cycle = step.alert->cycle;
          a.ts = step.alert->ts;
          a.smoothed_error = step.alert->smoothed_error;
          a.limit = step.alert->limit;
          a.strategy = static_cast<int32_t>(step.alert->strategy);
          a.batch = step.alert->workload.batch;
          a.input_len = step.alert->workload.input_len;
          a.output_len = step.alert->workload.output_len;
          a.episode_id = step.alert->episode_id;
          a.record_index = nr;
        }
        o_records[nr++] = o;
      }
    }
    n_out[0] = n_cyc;
    n_out[1] = nr;
    n_out[2] = na;
    if (out_flags) *out_flags = flags;
  } catch (const EngineError& e) {
    if (err && err_cap) std::snprintf(err, err_cap, "%s: %s", e.type().c_str(), e.what());
    return 1;
  } catch (const std::exception& e) {
    if (err && err_cap) std::snprintf(err, err_cap, "internal: %s", e.what());
    return 2;
  }
  if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return 0;
}

}  // extern "C"
