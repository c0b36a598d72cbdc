// tests/dropin_demo.cpp — TEST INFRASTRUCTURE.  Runs the reference's own
// suite harness, simkit::evaluate_trial (simkit.cpp:796-955: segmentation,
// records, fit, the three strategies' P/R/F1/FPR/lag, escalation, RCA), on
// SuiteConfig{} trials (BASELINE config 4) and prints one JSON line per trial.
//
// Built twice by oracle/Makefile from the reference sources:
//   _ref/dropin_demo_ref : pure reference
//   _ref/dropin_demo_gpu : the same objects with segment_and_classify /
//                          build_cycle_records served by
//                          paper_2601_09258_b200/dropin/cyclescope_dropin.cpp
//                          (linked first, --allow-multiple-definition)
// tests/test_integration.py runs both on the GPU box and requires identical
// output.  The trial datasets are rebuilt with the public simkit API exactly
// like make_trial_fault / make_trial_dataset (simkit.cpp:760-792).
#include <cstdio>
#include <cstdlib>

#include "cyclescope/rng.hpp"
#include "cyclescope/simkit.hpp"

using namespace cyclescope;

int main(int argc, char** argv) {
  SuiteConfig cfg;
  const size_t trials = argc > 1 ? std::strtoul(argv[1], nullptr, 10) : 8;
  for (size_t trial = 0; trial < trials; ++trial) {
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
      fault.target_rank =
          static_cast<int>(rng.uniform_int(0, static_cast<int64_t>(cfg.nvlink_ranks) - 1));
    const auto seed = Rng::substream_seed(cfg.seed, trial);
    const auto work = generate_workload(cfg.profile, cfg.cycles_per_trial, seed);
    SynthOptions opt;
    opt.n_ranks = family == FaultFamily::NvlinkSaturation ? cfg.nvlink_ranks : 1;
    const auto ds = synthesize_trace(work, cfg.model, {&fault, 1}, opt, Rng::substream_seed(seed, 1));
    const auto o = evaluate_trial(cfg, ds, trial, family);
    std::printf("{\"trial\":%zu,\"family\":\"%s\"", trial, to_string(family));
    for (const auto& m : o.strategies)
      std::printf(",\"%s\":[%zu,%zu,%zu,%zu,%zu,%.17g,%.17g,%.17g]", to_string(m.strategy),
                  m.true_positives, m.false_positives, m.false_negatives, m.true_negatives,
                  m.alerts, m.f1, m.fpr, m.mean_lag);
    std::printf(",\"rca_top\":\"%s\",\"ebar_n\":%zu", o.rca_top_class.c_str(), o.ebar_row.size());
    double es = 0.0;
    for (double v : o.ebar_row) es += v;
    std::printf(",\"ebar_sum\":%.17g}\n", es);
  }
  return 0;
}
