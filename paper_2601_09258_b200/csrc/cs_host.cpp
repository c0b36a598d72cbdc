// cs_host.cpp — host-side services of the C ABI (no device work):
//  * cs_fit_latency_model: deterministic least-squares GBDT fit with the
//    reference's semantics (baseline.cpp:118-208, gbdt.cpp:40-171) so the
//    persisted model is byte-identical (host C++ for v1).
//  * LatencyModel JSON in the reference's schema (baseline.cpp:277-302,
//    gbdt.cpp:186-234).
//  * RunConfig JSON (config.cpp:78-188 schema) -> cs_* configs + name table.
// Compiled with -ffp-contract=off: no FMA, like the reference's objects.
#include <algorithm>
#include <map>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include <thread>

#include <nlohmann/json.hpp>

#include "cs_fit.h"
#include "cs_parallel.h"
#include "cs_guard.h"
#include "cyclescope_b200.h"

using nlohmann::json;

struct FitNode {
  int feature = -1;
  double threshold = 0.0;
  int left = -1, right = -1;
  double value = 0.0;
};

struct cs_fitted_model {
  std::vector<std::string> feature_names;
  std::vector<int32_t> feature_ids;
  cs_gbdt_params params{200, 5, 0.1, 5, 1e-6};
  uint64_t n_features = 0;
  double base = 0.0;
  bool degenerate = false;
  std::vector<double> importance;
  std::vector<std::vector<FitNode>> trees;
  double mu = 0.0, sigma = 0.0;
  uint64_t calibration_size = 0;
  // flattened view storage
  std::vector<uint32_t> offsets;
  std::vector<cs_tree_node> flat;
  std::vector<const char*> name_ptrs;  // cs_model::feature_names
};

namespace {

struct FitError {
  int code;
  std::string msg;
};

const char* kFeatureNames[] = {"batch", "w_kv", "input_len", "output_len", "stage"};

int32_t feature_id_of(const std::string& n) {
  for (int i = 0; i < 5; ++i)
    if (n == kFeatureNames[i]) return i;
  return -1;
}

void set_err(char* err, size_t cap, const std::string& s) {
  if (err && cap) {
    std::strncpy(err, s.c_str(), cap - 1);
    err[cap - 1] = 0;
  }
}

// Rows are addressed through a dense row-major matrix.
struct Matrix {
  uint64_t rows = 0, cols = 0;
  std::vector<double> v;
  double at(uint64_t r, uint64_t c) const { return v[r * cols + c]; }
};

double tree_predict(const std::vector<FitNode>& t, const double* x) {
  int n = 0;
  while (t[n].feature >= 0) n = x[t[n].feature] <= t[n].threshold ? t[n].left : t[n].right;
  return t[n].value;
}

// Exact greedy least-squares split search, recursive pre-order node ids.
struct Grower {
  const Matrix& x;
  const std::vector<double>& r;
  const cs_gbdt_params& p;
  std::vector<double>& importance;
  std::vector<FitNode> nodes;
  std::vector<std::pair<double, double>> scratch;

  int grow(std::vector<uint32_t>& idx, uint64_t depth) {
    double total = 0.0;
    for (uint32_t i : idx) total += r[i];
    const double cnt = static_cast<double>(idx.size());
    const double mean = total / cnt;
    const int id = static_cast<int>(nodes.size());
    nodes.emplace_back();
    if (depth >= p.max_depth || idx.size() < 2 * p.min_samples_leaf) {
      nodes[id].value = mean;
      return id;
    }
    double best_gain = 0.0, best_thr = 0.0;
    int best_f = -1;
    for (uint64_t f = 0; f < x.cols; ++f) {
      scratch.clear();
      scratch.reserve(idx.size());
      for (uint32_t i : idx) scratch.emplace_back(x.at(i, f), r[i]);
      std::sort(scratch.begin(), scratch.end(),
                [](const std::pair<double, double>& a, const std::pair<double, double>& b) {
                  return a.first < b.first;
                });
      double lsum = 0.0;
      for (size_t k = 0; k + 1 < scratch.size(); ++k) {
        lsum += scratch[k].second;
        if (scratch[k].first == scratch[k + 1].first) continue;
        const size_t ln = k + 1, rn = scratch.size() - ln;
        if (ln < p.min_samples_leaf || rn < p.min_samples_leaf) continue;
        const double rsum = total - lsum;
        const double gain = lsum * lsum / static_cast<double>(ln) +
                            rsum * rsum / static_cast<double>(rn) - total * total / cnt;
        if (gain > best_gain + 1e-12) {
          best_gain = gain;
          best_f = static_cast<int>(f);
          best_thr = 0.5 * (scratch[k].first + scratch[k + 1].first);
        }
      }
    }
    if (best_f < 0 || best_gain <= 1e-12) {
      nodes[id].value = mean;
      return id;
    }
    std::vector<uint32_t> li, ri;
    li.reserve(idx.size());
    ri.reserve(idx.size());
    for (uint32_t i : idx) (x.at(i, best_f) <= best_thr ? li : ri).push_back(i);
    idx.clear();
    idx.shrink_to_fit();
    importance[best_f] += best_gain;
    nodes[id].feature = best_f;
    nodes[id].threshold = best_thr;
    const int l = grow(li, depth + 1);
    const int rr = grow(ri, depth + 1);
    nodes[id].left = l;
    nodes[id].right = rr;
    return id;
  }
};

double clamp_predict(const cs_fitted_model& m, const double* x) {
  double v = m.base;
  for (const auto& t : m.trees) v += m.params.learning_rate * tree_predict(t, x);
  return std::max(m.params.prediction_floor, v);
}

void fit_gbdt_into(cs_fitted_model& m, const Matrix& x, const std::vector<double>& y) {
  if (x.rows != y.size() || x.rows == 0)
    throw FitError{CS_E_INSUFFICIENT_DATA, "feature matrix and target size mismatch or empty"};
  m.n_features = x.cols;
  m.importance.assign(x.cols, 0.0);
  double mean = 0.0;
  for (double v : y) mean += v;
  mean /= static_cast<double>(y.size());
  m.base = mean;
  const auto [lo, hi] = std::minmax_element(y.begin(), y.end());
  if (*lo == *hi) {
    m.base = *lo;
    m.degenerate = true;
    return;
  }
  std::vector<double> pred(y.size(), mean), res(y.size());
  for (uint64_t round = 0; round < m.params.n_trees; ++round) {
    for (size_t i = 0; i < y.size(); ++i) res[i] = y[i] - pred[i];
    Grower g{x, res, m.params, m.importance, {}, {}};
    std::vector<uint32_t> idx(y.size());
    std::iota(idx.begin(), idx.end(), 0u);
    g.grow(idx, 0);
    for (size_t i = 0; i < y.size(); ++i)
      pred[i] += m.params.learning_rate * tree_predict(g.nodes, &x.v[i * x.cols]);
    m.trees.push_back(std::move(g.nodes));
  }
}

json model_json(const cs_fitted_model& m) {
  json trees = json::array();
  for (const auto& t : m.trees) {
    json nodes = json::array();
    for (const auto& n : t)
      nodes.push_back({{"f", n.feature}, {"t", n.threshold}, {"l", n.left}, {"r", n.right},
                       {"v", n.value}});
    trees.push_back(std::move(nodes));
  }
  json g{{"params",
          {{"n_trees", m.params.n_trees},
           {"max_depth", m.params.max_depth},
           {"learning_rate", m.params.learning_rate},
           {"min_samples_leaf", m.params.min_samples_leaf},
           {"prediction_floor", m.params.prediction_floor}}},
         {"n_features", m.n_features},
         {"base", m.base},
         {"degenerate", m.degenerate},
         {"importance", m.importance},
         {"trees", std::move(trees)}};
  return json{{"format_version", 1},
              {"kind", "latency_gbdt"},
              {"features", m.feature_names},
              {"residual_stats",
               {{"mu", m.mu}, {"sigma", m.sigma}, {"calibration_size", m.calibration_size}}},
              {"gbdt", std::move(g)}};
}

void rebuild_flat(cs_fitted_model& m) {
  m.offsets.assign(1, 0);
  m.flat.clear();
  for (const auto& t : m.trees) {
    for (const auto& n : t) {
      cs_tree_node c{};
      c.feature = n.feature;
      c.left = n.left;
      c.right = n.right;
      c.threshold = n.threshold;
      c.value = n.value;
      m.flat.push_back(c);
    }
    m.offsets.push_back(static_cast<uint32_t>(m.flat.size()));
  }
  m.feature_ids.clear();
  for (const auto& n : m.feature_names) m.feature_ids.push_back(feature_id_of(n));
}

// fit_latency_model's checks and split_calibration (baseline.cpp:118-149,
// 168-180): training and holdout rows, each in chronological order
void split_rows(uint64_t n, uint32_t n_features, const double* x, const double* y,
                const cs_gbdt_params* params, const cs_fit_options* opt, std::vector<uint32_t>& train,
                std::vector<uint32_t>& calib) {
  const uint64_t min_required = std::max<uint64_t>(opt->min_samples, 2 * params->min_samples_leaf);
  if (n < min_required)
    throw FitError{CS_E_INSUFFICIENT_DATA, "need at least " + std::to_string(min_required) +
                                               " samples, got " + std::to_string(n)};
  for (uint64_t i = 0; i < n; ++i)
    if (!(y[i] > 0.0) || !std::isfinite(y[i]))
      throw FitError{CS_E_INSUFFICIENT_DATA, "targets must be positive and finite"};
  const uint32_t sc = (opt->stratify_col >= 0 && static_cast<uint32_t>(opt->stratify_col) < n_features)
                          ? static_cast<uint32_t>(opt->stratify_col)
                          : 0u;
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    return x[static_cast<uint64_t>(a) * n_features + sc] < x[static_cast<uint64_t>(b) * n_features + sc];
  });
  const uint64_t stride =
      opt->calibration_fraction > 0.0
          ? std::max<uint64_t>(2, static_cast<uint64_t>(std::llround(1.0 / opt->calibration_fraction)))
          : n + 1;
  for (uint64_t pos = 0; pos < n; ++pos)
    (pos % stride == stride - 1 ? calib : train).push_back(order[pos]);
  std::sort(train.begin(), train.end());
  std::sort(calib.begin(), calib.end());
}

// holdout residual statistics (baseline.cpp:186-205)
void holdout_stats(cs_fitted_model& m, const double* x, const double* y, uint32_t n_features,
                   const std::vector<uint32_t>& calib, const cs_fit_options* opt) {
  std::vector<double> res;
  for (uint32_t r : calib) {
    const double p = clamp_predict(m, x + static_cast<uint64_t>(r) * n_features);
    res.push_back(std::max(0.0, (y[r] - p) / (y[r] + opt->ppe_epsilon)));
  }
  m.calibration_size = res.size();
  if (!res.empty()) {
    double mean = 0.0;
    for (double v : res) mean += v;
    mean /= static_cast<double>(res.size());
    double var = 0.0;
    for (double v : res) var += (v - mean) * (v - mean);
    var = res.size() > 1 ? var / static_cast<double>(res.size() - 1) : 0.0;
    m.mu = mean;
    m.sigma = std::sqrt(var);
  }
}

void set_features(cs_fitted_model& m, uint32_t n_features, const int32_t* feature_ids) {
  for (uint32_t f = 0; f < n_features; ++f) {
    if (feature_ids[f] < 0 || feature_ids[f] > 4) throw FitError{CS_E_FEATURE_MISMATCH, "unknown feature id"};
    m.feature_names.push_back(kFeatureNames[feature_ids[f]]);
  }
}

}  // namespace

extern "C" {

static int cs_fit_latency_model_impl(uint64_t n, uint32_t n_features, const int32_t* feature_ids,
                         const double* x, const double* y, const cs_gbdt_params* params,
                         const cs_fit_options* opt, cs_fitted_model** out, char* err,
                         size_t err_cap, const char* const* names = nullptr) {
  if (!out || !params || !opt || (!feature_ids && !names) || (n && (!x || !y))) return CS_E_INVALID_ARGUMENT;
  *out = nullptr;
  auto m = new cs_fitted_model();
  try {
    m->params = *params;
    if (names) {
      for (uint32_t f = 0; f < n_features; ++f) {
        if (!names[f]) throw FitError{CS_E_INVALID_ARGUMENT, "null feature name"};
        m->feature_names.push_back(names[f]);
      }
    } else {
      set_features(*m, n_features, feature_ids);
    }
    std::vector<uint32_t> train, calib;
    split_rows(n, n_features, x, y, params, opt, train, calib);
    Matrix tx;
    tx.cols = n_features;
    tx.rows = train.size();
    std::vector<double> ty;
    for (uint32_t r : train) {
      tx.v.insert(tx.v.end(), x + static_cast<uint64_t>(r) * n_features,
                  x + static_cast<uint64_t>(r + 1) * n_features);
      ty.push_back(y[r]);
    }
    fit_gbdt_into(*m, tx, ty);
    holdout_stats(*m, x, y, n_features, calib, opt);
    rebuild_flat(*m);
  } catch (const FitError& e) {
    set_err(err, err_cap, e.msg);
    delete m;
    return e.code;
  }
  *out = m;
  return CS_OK;
}

int cs_fit_latency_model(uint64_t n, uint32_t n_features, const int32_t* feature_ids,
                         const double* x, const double* y, const cs_gbdt_params* params,
                         const cs_fit_options* opt, cs_fitted_model** out, char* err,
                         size_t err_cap) {
  return cs_guard([&] { return cs_fit_latency_model_impl(n, n_features, feature_ids, x, y, params, opt, out, err, err_cap); });
}

int cs_fit_latency_model_named(uint64_t n, uint32_t n_features, const char* const* feature_names,
                               const double* x, const double* y, const cs_gbdt_params* params,
                               const cs_fit_options* opt, cs_fitted_model** out, char* err,
                               size_t err_cap) {
  if (!feature_names && n_features) return CS_E_INVALID_ARGUMENT;
  return cs_guard([&] {
    return cs_fit_latency_model_impl(n, n_features, nullptr, x, y, params, opt, out, err, err_cap,
                                     feature_names);
  });
}

static int cs_fit_latency_models_impl(int device, uint32_t n_models, const uint64_t* offsets,
                          uint32_t n_features, const int32_t* feature_ids, const double* x,
                          const double* y, const cs_gbdt_params* params, const cs_fit_options* opt,
                          uint32_t n_threads, cs_fitted_model** out, int32_t* status,
                          float* device_ms) {
  if (!out || !status || !params || !opt || !feature_ids || !offsets || n_features == 0)
    return CS_E_INVALID_ARGUMENT;
  if (offsets[0] != 0) return CS_E_INVALID_ARGUMENT;
  for (uint32_t m = 0; m < n_models; ++m)
    if (offsets[m + 1] < offsets[m]) return CS_E_INVALID_ARGUMENT;
  if (offsets[n_models] && (!x || !y)) return CS_E_INVALID_ARGUMENT;
  if (n_threads == 0) n_threads = 1;
  for (uint32_t m = 0; m < n_models; ++m) {
    out[m] = nullptr;
    status[m] = CS_OK;
  }
  // host: checks and holdout split per model (parallel over models)
  std::vector<std::vector<uint32_t>> train(n_models), calib(n_models);
  auto par = [&](auto body) {
    cs_host::parallel_for(n_models, n_threads, [&](size_t m0, size_t m1, uint32_t) {
      for (size_t m = m0; m < m1; ++m) body(static_cast<uint32_t>(m));
    });
  };
  par([&](uint32_t m) {
    const uint64_t o = offsets[m], n = offsets[m + 1] - o;
    try {
      cs_fitted_model probe;
      set_features(probe, n_features, feature_ids);
      split_rows(n, n_features, x + o * n_features, y + o, params, opt, train[m], calib[m]);
    } catch (const FitError& e) {
      status[m] = e.code;
    }
  });
  // device: fit_gbdt of every model's training rows
  GbdtBatch b;
  b.n_features = n_features;
  b.params = *params;
  b.off.assign(n_models + 1, 0);
  for (uint32_t m = 0; m < n_models; ++m)
    b.off[m + 1] = b.off[m] + (status[m] == CS_OK ? train[m].size() : 0);
  b.x_col.resize(b.off[n_models] * n_features);
  b.y.resize(b.off[n_models]);
  par([&](uint32_t m) {
    if (status[m] != CS_OK) return;
    const uint64_t o = offsets[m], to = b.off[m], tn = train[m].size();
    for (uint64_t k = 0; k < tn; ++k) {
      const uint64_t r = o + train[m][k];
      for (uint32_t f = 0; f < n_features; ++f) b.x_col[to * n_features + f * tn + k] = x[r * n_features + f];
      b.y[to + k] = y[r];
    }
  });
  std::string err;
  const int rc = gbdt_fit_device(device, b, err);
  if (rc != CS_OK) return rc;
  if (device_ms) *device_ms = b.device_ms;
  // host: models and holdout statistics
  par([&](uint32_t m) {
    if (status[m] != CS_OK) return;
    auto* fm = new cs_fitted_model();
    fm->params = *params;
    set_features(*fm, n_features, feature_ids);
    fm->n_features = n_features;
    fm->base = b.base[m];
    fm->degenerate = b.degenerate[m] != 0;
    fm->importance.assign(b.importance.begin() + static_cast<size_t>(m) * n_features,
                          b.importance.begin() + static_cast<size_t>(m + 1) * n_features);
    if (!fm->degenerate) {
      for (uint64_t t = 0; t < params->n_trees; ++t) {
        const cs_tree_node* src = &b.nodes[(static_cast<size_t>(m) * params->n_trees + t) * b.node_stride];
        std::vector<FitNode> tree(b.n_nodes[static_cast<size_t>(m) * params->n_trees + t]);
        for (size_t k = 0; k < tree.size(); ++k)
          tree[k] = FitNode{src[k].feature, src[k].threshold, src[k].left, src[k].right, src[k].value};
        fm->trees.push_back(std::move(tree));
      }
    }
    holdout_stats(*fm, x + offsets[m] * n_features, y + offsets[m], n_features, calib[m], opt);
    rebuild_flat(*fm);
    out[m] = fm;
  });
  return CS_OK;
}

int cs_fit_latency_models(int device, uint32_t n_models, const uint64_t* offsets,
                          uint32_t n_features, const int32_t* feature_ids, const double* x,
                          const double* y, const cs_gbdt_params* params, const cs_fit_options* opt,
                          uint32_t n_threads, cs_fitted_model** out, int32_t* status,
                          float* device_ms) {
  return cs_guard([&] { return cs_fit_latency_models_impl(device, n_models, offsets, n_features, feature_ids, x, y, params, opt, n_threads, out, status, device_ms); });
}

static int cs_model_from_json_impl(const char* text, cs_fitted_model** out, char* err, size_t err_cap) {
  if (!text || !out) return CS_E_INVALID_ARGUMENT;
  *out = nullptr;
  auto m = new cs_fitted_model();
  try {
    const json j = json::parse(text);
    const int version = j.value("format_version", -1);
    if (version != 1)
      throw FitError{CS_E_MODEL_FORMAT, "unsupported model format version " +
                                            std::to_string(version) + ", expected 1"};
    m->feature_names = j.at("features").get<std::vector<std::string>>();
    const auto& st = j.at("residual_stats");
    m->mu = st.at("mu").get<double>();
    m->sigma = st.at("sigma").get<double>();
    m->calibration_size = st.at("calibration_size").get<uint64_t>();
    const auto& g = j.at("gbdt");
    const auto& p = g.at("params");
    m->params.n_trees = p.at("n_trees").get<uint64_t>();
    m->params.max_depth = p.at("max_depth").get<uint64_t>();
    m->params.learning_rate = p.at("learning_rate").get<double>();
    m->params.min_samples_leaf = p.at("min_samples_leaf").get<uint64_t>();
    m->params.prediction_floor = p.at("prediction_floor").get<double>();
    m->n_features = g.at("n_features").get<uint64_t>();
    m->base = g.at("base").get<double>();
    m->degenerate = g.at("degenerate").get<bool>();
    m->importance = g.at("importance").get<std::vector<double>>();
    for (const auto& tj : g.at("trees")) {
      std::vector<FitNode> t;
      for (const auto& nj : tj)
        t.push_back({nj.at("f").get<int>(), nj.at("t").get<double>(), nj.at("l").get<int>(),
                     nj.at("r").get<int>(), nj.at("v").get<double>()});
      m->trees.push_back(std::move(t));
    }
    rebuild_flat(*m);
  } catch (const FitError& e) {
    set_err(err, err_cap, e.msg);
    delete m;
    return e.code;
  } catch (const std::exception& e) {
    set_err(err, err_cap, std::string("cannot parse model: ") + e.what());
    delete m;
    return CS_E_MODEL_FORMAT;
  }
  *out = m;
  return CS_OK;
}

int cs_model_from_json(const char* text, cs_fitted_model** out, char* err, size_t err_cap) {
  return cs_guard([&] { return cs_model_from_json_impl(text, out, err, err_cap); });
}

int cs_model_to_json(const cs_fitted_model* m, char* buf, size_t cap, size_t* n) {
  if (!m) return CS_E_INVALID_ARGUMENT;
  const std::string s = model_json(*m).dump();
  if (n) *n = s.size() + 1;
  if (!buf) return CS_OK;
  if (cap < s.size() + 1) return CS_E_INVALID_ARGUMENT;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return CS_OK;
}

int cs_model_view(const cs_fitted_model* m, cs_model* v) {
  if (!m || !v) return CS_E_INVALID_ARGUMENT;
  std::memset(v, 0, sizeof *v);
  v->n_features = static_cast<uint32_t>(m->feature_names.size());
  v->n_trees = static_cast<uint32_t>(m->trees.size());
  v->feature_ids = m->feature_ids.data();
  auto& np = const_cast<cs_fitted_model*>(m)->name_ptrs;
  np.clear();
  for (const auto& nm : m->feature_names) np.push_back(nm.c_str());
  v->feature_names = np.data();
  v->tree_offsets = m->offsets.data();
  v->nodes = m->flat.data();
  v->base = m->base;
  v->learning_rate = m->params.learning_rate;
  v->prediction_floor = m->params.prediction_floor;
  v->mu_train = m->mu;
  v->sigma_train = m->sigma;
  v->degenerate = m->degenerate ? 1 : 0;
  return CS_OK;
}

void cs_model_free(cs_fitted_model* m) { delete m; }

// monitor_loop's alert sink (main.cpp:151-177): Alert::to_json
// (detector.cpp:72-83) + Escalator (detector.cpp:132-150).  Record cycles are
// increasing, so the Escalator's on_cycle timeouts between two alerts reduce
// to checking the alert's own cycle against the deadline.
int cs_alerts_to_ndjson(const cs_alert* alerts, uint64_t n_alerts, uint64_t pre_roll,
                        uint64_t post_roll, char* buf, size_t cap, size_t* n) {
  if (n_alerts && !alerts) return CS_E_INVALID_ARGUMENT;
  static const char* kStrategy[3] = {"fixed_point", "fixed_window", "dynamic_window"};
  std::string out;
  bool deep = false;
  uint64_t deadline = 0;
  for (uint64_t i = 0; i < n_alerts; ++i) {
    const cs_alert& a = alerts[i];
    if (deep && a.cycle > deadline) deep = false;  // Escalator::on_cycle
    json rec{{"cycle", a.cycle},
             {"ts", a.ts},
             {"ebar", a.smoothed_error},
             {"ucl", a.limit},
             {"strategy", kStrategy[a.strategy < 0 || a.strategy > 2 ? 2 : a.strategy]},
             {"workload",
              {{"batch", a.batch}, {"input_len", a.input_len}, {"output_len", a.output_len}}},
             {"episode_id", a.episode_id}};
    deadline = a.cycle + post_roll;  // Escalator::on_alert
    if (!deep) {
      deep = true;
      rec["retain"] = {{"begin", a.cycle >= pre_roll ? a.cycle - pre_roll : 0},
                       {"end", a.cycle + post_roll}};
      rec["mode"] = "deep_dive";
    }
    out += rec.dump();
    out += "\n";
  }
  if (n) *n = out.size() + 1;
  if (!buf) return CS_OK;
  if (cap < out.size() + 1) return CS_E_INVALID_ARGUMENT;
  std::memcpy(buf, out.c_str(), out.size() + 1);
  return CS_OK;
}

// RunConfig JSON (config.cpp:78-188 schema; unknown keys rejected) ->
// device configs + per-name table.  `names` are the interned names in id
// order (lexicographic); name_is_span marks names that occur as Spans
// (dense beta slots in name order).
static int cs_config_from_json_impl(const char* run_config_json, uint32_t n_names,
                        const char* const* names, const uint8_t* name_is_span,
                        uint32_t n_comm_slots, cs_name_info* out_names,
                        cs_cycle_config* out_cycle, cs_control_config* out_control, char* err,
                        size_t err_cap) {
  if (!out_cycle || !out_control || (n_names && (!names || !out_names || !name_is_span)))
    return CS_E_INVALID_ARGUMENT;
  try {
    const json j = (run_config_json && *run_config_json) ? json::parse(run_config_json) : json::object();
    auto reject = [](const json& o, std::initializer_list<const char*> known, const char* ctx) {
      for (const auto& [k, v] : o.items()) {
        bool ok = false;
        for (const char* s : known) ok = ok || k == s;
        if (!ok) throw FitError{CS_E_CONFIG, std::string("unknown key '") + k + "' in " + ctx};
      }
    };
    reject(j, {"seed", "cycle", "pipeline", "feature_set", "gbdt", "fit", "detector", "escalation",
               "metric_map", "calibration"},
           "run config");
    std::string hint;
    uint64_t min_calls = 10;
    std::vector<std::string> phases = {"run_batch", "process_batch_result", "get_next_batch_to_run"};
    std::vector<std::string> pkw = {"forward_prefill"}, dkw = {"process_batch_result_decode"};
    double fdur = 3.0, fgap = 2.0;
    uint64_t window = 32;
    if (j.contains("cycle")) {
      const auto& y = j["cycle"];
      reject(y, {"anchor_hint", "min_anchor_calls", "phase_functions", "forward_mode_key",
                 "prefill_keywords", "decode_keywords", "prefill_duration_factor",
                 "prefill_gap_factor", "stage_window", "batch_size_key", "input_len_key",
                 "output_len_key"},
             "cycle config");
      hint = y.value("anchor_hint", hint);
      min_calls = y.value("min_anchor_calls", min_calls);
      if (y.contains("phase_functions")) phases = y["phase_functions"].get<std::vector<std::string>>();
      if (y.contains("prefill_keywords")) pkw = y["prefill_keywords"].get<std::vector<std::string>>();
      if (y.contains("decode_keywords")) dkw = y["decode_keywords"].get<std::vector<std::string>>();
      fdur = y.value("prefill_duration_factor", fdur);
      fgap = y.value("prefill_gap_factor", fgap);
      window = y.value("stage_window", window);
    }
    std::string latency_component = "run_batch";
    bool include_prefill = false;
    if (j.contains("pipeline")) {
      const auto& p = j["pipeline"];
      reject(p, {"latency_component", "include_prefill", "extra_args_prefix"}, "pipeline config");
      latency_component = p.value("latency_component", latency_component);
      include_prefill = p.value("include_prefill", include_prefill);
    }
    cs_control_config ctl{CS_DYNAMIC_WINDOW, 0, 10, 0.15, 3.0, 0.18, 0.02, 100, 1e-9};
    if (j.contains("detector")) {
      const auto& d = j["detector"];
      reject(d, {"strategy", "window", "fixed_threshold", "sigma_k", "theta_max", "min_ucl",
                 "warmup", "epsilon"},
             "detector config");
      const std::string s = d.value("strategy", std::string("dynamic_window"));
      if (s == "fixed_point") ctl.strategy = CS_FIXED_POINT;
      else if (s == "fixed_window") ctl.strategy = CS_FIXED_WINDOW;
      else if (s == "dynamic_window") ctl.strategy = CS_DYNAMIC_WINDOW;
      else throw FitError{CS_E_CONFIG, "unknown detector strategy '" + s + "'"};
      ctl.window = d.value("window", ctl.window);
      ctl.fixed_threshold = d.value("fixed_threshold", ctl.fixed_threshold);
      ctl.sigma_k = d.value("sigma_k", ctl.sigma_k);
      ctl.theta_max = d.value("theta_max", ctl.theta_max);
      ctl.min_ucl = d.value("min_ucl", ctl.min_ucl);
      ctl.warmup = d.value("warmup", ctl.warmup);
      ctl.epsilon = d.value("epsilon", ctl.epsilon);
    }
    // MetricMap (rca.cpp:55-69): event class -> counter metric
    std::map<std::string, std::string> metric_map = {
        {"oncpu", "cpu_usage"},           {"gemm_kernel", "gpu_usage"},
        {"attn_kernel", "gpu_clock"},     {"reduce", "tx_bytes"},
        {"memcpy_h2d", "pcie_util"},      {"memcpy_d2d", "bus_util"},
        {"run_batch", "gpu_usage"},       {"process_batch_result", "cpu_usage"},
        {"get_next_batch_to_run", "cpu_usage"}};
    if (j.contains("metric_map"))
      metric_map = j["metric_map"].get<std::map<std::string, std::string>>();
    // dedup phases, first occurrence (component_durations is a map)
    std::vector<std::string> uph;
    for (const auto& p : phases)
      if (std::find(uph.begin(), uph.end(), p) == uph.end()) uph.push_back(p);
    cs_cycle_config cyc{};
    cyc.anchor_hint_name = -1;
    cyc.min_anchor_calls = min_calls;
    cyc.prefill_duration_factor = fdur;
    cyc.prefill_gap_factor = fgap;
    cyc.stage_window = window;
    cyc.stage_min_history = 8;
    cyc.frequency_bin_ns = 1000000;
    cyc.n_phases = static_cast<int32_t>(uph.size());
    cyc.latency_phase = -1;
    for (size_t k = 0; k < uph.size(); ++k)
      if (!latency_component.empty() && uph[k] == latency_component) cyc.latency_phase = static_cast<int32_t>(k);
    cyc.include_prefill = include_prefill ? 1 : 0;
    cyc.n_comm_slots = static_cast<int32_t>(n_comm_slots);
    int32_t slot = 0;
    for (uint32_t i = 0; i < n_names; ++i) {
      const std::string nm = names[i];
      cs_name_info& ni = out_names[i];
      std::memset(&ni, 0, sizeof ni);
      ni.phase = -1;
      for (size_t k = 0; k < uph.size(); ++k)
        if (uph[k] == nm) ni.phase = static_cast<int32_t>(k);
      for (const auto& kw : pkw)
        if (nm.find(kw) != std::string::npos) ni.flags |= CS_NAME_PREFILL_KW;
      for (const auto& kw : dkw)
        if (nm.find(kw) != std::string::npos) ni.flags |= CS_NAME_DECODE_KW;
      ni.beta_slot = name_is_span[i] ? slot++ : -1;
      ni.metric = 0;
      const auto mm = metric_map.find(nm);
      if (mm != metric_map.end())
        for (uint32_t k = 0; k < n_names; ++k)
          if (mm->second == names[k]) ni.metric = k + 1;
      if (!hint.empty() && nm == hint) cyc.anchor_hint_name = i;
    }
    if (!hint.empty() && cyc.anchor_hint_name < 0) cyc.anchor_hint_name = -2;
    cyc.n_beta_slots = slot;
    *out_cycle = cyc;
    *out_control = ctl;
  } catch (const FitError& e) {
    set_err(err, err_cap, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_err(err, err_cap, e.what());
    return CS_E_CONFIG;
  }
  return CS_OK;
}

int cs_config_from_json(const char* run_config_json, uint32_t n_names,
                        const char* const* names, const uint8_t* name_is_span,
                        uint32_t n_comm_slots, cs_name_info* out_names,
                        cs_cycle_config* out_cycle, cs_control_config* out_control, char* err,
                        size_t err_cap) {
  return cs_guard([&] { return cs_config_from_json_impl(run_config_json, n_names, names, name_is_span, n_comm_slots, out_names, out_cycle, out_control, err, err_cap); });
}

}  // extern "C"
