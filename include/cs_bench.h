/*
 * cs_bench.h — benchmark support, NOT part of the product library: the
 * synthetic trace producer (a restatement of the reference's simkit,
 * byte-identical per chunk) and an HBM streaming microbenchmark.  Built into
 * benchlib/libcs_bench.so; the analysis path (libcyclescope_b200.so) never
 * links it.
 */
#ifndef CS_BENCH_H_
#define CS_BENCH_H_

#include "cyclescope_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------- synthetic trace producer
 * Restatement of the reference's simkit generator (simkit.cpp:34-86,
 * 195-246, 276-506) writing cs_event records directly; benchmark input only.
 * n_chunks > 1 concatenates independent generator calls (substream seeds per
 * chunk) in time so large instances can be produced on all host cores. */
typedef struct cs_synth_params {
  uint64_t n_cycles;
  uint64_t workload_seed;
  uint64_t synth_seed;
  int32_t fault_family;    /* -1 none, else FaultFamily enum (simkit.hpp:70-79) */
  int32_t target_rank;
  uint64_t fault_onset;    /* global cycle index */
  uint64_t fault_duration;
  double severity;         /* <= 0: default_severity (simkit.cpp:134-146) */
  uint64_t n_ranks;
  double noise;            /* < 0: GroundTruthModel default 0.05 */
} cs_synth_params;
typedef struct cs_synth_trace cs_synth_trace;
int cs_synth_generate(const cs_synth_params* p, uint32_t n_chunks, uint32_t n_threads,
                      int compact_names, cs_synth_trace** out);
int cs_synth_view(const cs_synth_trace* t, const cs_event** ev, uint64_t* n_ev,
                  const uint64_t** event_ids, const cs_workload** wl, uint64_t* n_wl,
                  const uint8_t** labels, uint64_t* n_cycles);
int cs_synth_names(const cs_synth_trace* t, const char** packed, size_t* n_bytes,
                   uint32_t* n_names, uint32_t* n_comm);
void cs_synth_free(cs_synth_trace* t);

/* HBM read-streaming microbenchmark (profiling only).
 * variant 0: vectorised LDG (p0 CTAs/SM, p1 threads, p2 unroll 1|8);
 * variant 1: 1-D TMA bulk copies (p0 chunk bytes, p1 stages, p2 CTAs/SM). */
int cs_microbench(int variant, const void* dev_src, uint64_t n_bytes, int p0, int p1, int p2,
                  int iters, double* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* CS_BENCH_H_ */
