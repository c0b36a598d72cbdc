// cs_fit.h — the batched device GBDT fit (cs_fit.cu) as seen by the host
// services (cs_host.cpp): training sets in, trees in the reference's node
// order out.  Host-only types; no CUDA in the interface.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "cyclescope_b200.h"

struct GbdtBatch {
  // inputs: the training rows of each model (after split_calibration)
  uint32_t n_features = 0;
  std::vector<uint64_t> off;   // n_models + 1
  std::vector<double> x_col;   // model m, feature f, row i: x_col[off[m] * F + f * n_m + i]
  std::vector<double> y;       // y[off[m] + i]
  cs_gbdt_params params{};
  // outputs (fit_gbdt, gbdt.cpp:123-171)
  std::vector<double> base;
  std::vector<uint8_t> degenerate;
  std::vector<double> importance;   // n_models * F
  uint32_t node_stride = 0;         // node slots per tree
  std::vector<cs_tree_node> nodes;  // [model][tree][node_stride], pre-order ids
  std::vector<uint32_t> n_nodes;    // [model][tree]
  float device_ms = 0.f;            // kernel time
};

// Fits every model of the batch on `device`; returns a cs_status.
int gbdt_fit_device(int device, GbdtBatch& b, std::string& err);
