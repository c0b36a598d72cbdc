// cs_rca.cpp — post-alert root-cause ranking:
// suspicion_rank, welch_p_value and attribute_straggler (rca.cpp:131-353)
// over the per-cycle stage attribution the device computes (beta, counter mu,
// per-(class, comm, rank) collective beta).  The windows are a few hundred
// cycles, so this is host C++ over their rows; cs_suspicion_rank in
// cs_api.cpp gathers the rows from the device.
//
// Arithmetic follows the reference operation for operation (sequential means
// and variances in window order, the same libm calls, no FMA contraction), so
// the ranking, scores and p-values are bit-identical.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <vector>

#include "cs_guard.h"
#include "cyclescope_b200.h"

namespace {

struct Moments {  // mean and sample variance of one window (rca.cpp:184-196)
  double mean = 0.0, var = 0.0;
  size_t n = 0;
};

Moments moments(const std::vector<double>& v) {
  Moments w;
  w.n = v.size();
  if (w.n == 0) return w;
  for (double x : v) w.mean += x;
  w.mean /= static_cast<double>(w.n);
  if (w.n > 1) {
    for (double x : v) w.var += (x - w.mean) * (x - w.mean);
    w.var /= static_cast<double>(w.n - 1);
  }
  return w;
}

double sigma_floor(const Moments& w) {  // rca.cpp:198-200
  return std::max({std::sqrt(w.var), 0.01 * std::abs(w.mean), 1e-12});
}

// Lentz's continued fraction for the regularized incomplete beta function,
// evaluated as the reference does (rca.cpp:134-162): two half-steps per
// iteration, each clamping |d| and |c| away from zero.
struct Lentz {
  double c = 1.0, d = 0.0, h = 0.0;
  static double clamp_tiny(double v) { return std::abs(v) < 1e-300 ? 1e-300 : v; }
  double half_step(double aa) {
    d = clamp_tiny(1.0 + aa * d);
    c = clamp_tiny(1.0 + aa / c);
    d = 1.0 / d;
    return d * c;
  }
};

double beta_fraction(double a, double b, double x) {
  const double qab = a + b, qap = a + 1.0, qam = a - 1.0;
  Lentz L;
  L.d = 1.0 / Lentz::clamp_tiny(1.0 - qab * x / qap);
  L.h = L.d;
  for (int m = 1; m <= 200; ++m) {
    const int m2 = 2 * m;
    const double even = m * (b - m) * x / ((qam + m2) * (a + m2));
    L.h *= L.half_step(even);
    const double odd = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2));
    const double del = L.half_step(odd);
    L.h *= del;
    if (std::abs(del - 1.0) < 3e-12) break;
  }
  return L.h;
}

double reg_incomplete_beta(double a, double b, double x) {  // rca.cpp:164-172
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double front = std::exp(std::lgamma(a + b) - std::lgamma(a) - std::lgamma(b) +
                                a * std::log(x) + b * std::log(1.0 - x));
  if (x < (a + 1.0) / (a + b + 2.0)) return front * beta_fraction(a, b, x) / a;
  return 1.0 - front * beta_fraction(b, a, 1.0 - x) / b;
}

double welch_p(double mean_a, double var_a, size_t n_a, double mean_b, double var_b, size_t n_b) {
  if (n_a < 2 || n_b < 2) return 1.0;  // rca.cpp:206-218
  const double sa = var_a / static_cast<double>(n_a);
  const double sb = var_b / static_cast<double>(n_b);
  const double se = sa + sb;
  if (se <= 0.0) return mean_a == mean_b ? 1.0 : 0.0;
  const double t = (mean_a - mean_b) / std::sqrt(se);
  const double df = se * se / (sa * sa / static_cast<double>(n_a - 1) + sb * sb / static_cast<double>(n_b - 1));
  if (df <= 0.0) return 1.0;  // student_t_two_sided (rca.cpp:174-178)
  return reg_incomplete_beta(df / 2.0, 0.5, df / (df + t * t));
}

}  // namespace

extern "C" {

double cs_welch_p_value(double mean_a, double var_a, uint64_t n_a, double mean_b, double var_b,
                        uint64_t n_b) {
  return welch_p(mean_a, var_a, n_a, mean_b, var_b, n_b);
}

static int cs_rank_suspects_impl(const cs_rca_window* normal, const cs_rca_window* abnormal,
                     const cs_rca_layout* lay, cs_suspect* out, size_t cap, size_t* n_out) {
  if (!normal || !abnormal || !lay || !n_out) return CS_E_INVALID_ARGUMENT;
  *n_out = 0;
  if (normal->n_cycles < 10 || abnormal->n_cycles < 3) return CS_E_INSUFFICIENT_CYCLES;
  const uint32_t S = lay->n_slots, R = lay->n_comm;
  for (const cs_rca_window* w : {normal, abnormal})
    if (w->n_cycles && (!w->totals || !w->beta || (R && (!w->coll || !w->coll_present))))
      return CS_E_INVALID_ARGUMENT;
  auto present = [&](const cs_rca_window* w, uint64_t c, uint32_t s) { return w->totals[c * S + s] > 0; };
  // classes: every slot present in some cycle of either window, in name order
  std::vector<uint32_t> classes;
  for (uint32_t s = 0; s < S; ++s) {
    bool any = false;
    for (const cs_rca_window* w : {normal, abnormal})
      for (uint64_t c = 0; c < w->n_cycles && !any; ++c) any = present(w, c, s);
    if (any) classes.push_back(s);
  }
  std::vector<cs_suspect> entries;
  for (uint32_t s : classes) {
    cs_suspect e{};
    e.beta_slot = static_cast<int32_t>(s);
    e.straggler_slot = -1;
    e.straggler_location = -1;
    e.welch_p = 1.0;
    // absent classes contribute beta = 0; mu only where present (rca.cpp:236-246)
    auto collect = [&](const cs_rca_window* w, std::vector<double>& betas, std::vector<double>& mus) {
      for (uint64_t c = 0; c < w->n_cycles; ++c) {
        const bool p = present(w, c, s);
        betas.push_back(p ? w->beta[c * S + s] : 0.0);
        if (p && w->mu && w->mu_has && w->mu_has[c * S + s]) {
          mus.push_back(w->mu[c * S + s]);
          if (e.metric == 0 && lay->slot_metric) e.metric = lay->slot_metric[s];
        }
      }
    };
    std::vector<double> bn_v, ba_v, mn_v, ma_v;
    collect(normal, bn_v, mn_v);
    collect(abnormal, ba_v, ma_v);
    const Moments bn = moments(bn_v), ba = moments(ba_v);
    e.beta_norm = bn.mean;
    e.beta_abn = ba.mean;
    e.delta_beta = ba.mean - bn.mean;
    e.z_beta = (ba.mean - bn.mean) / sigma_floor(bn);
    e.welch_p = welch_p(ba.mean, ba.var, ba.n, bn.mean, bn.var, bn.n);
    if (!mn_v.empty() && !ma_v.empty()) {
      const Moments mn = moments(mn_v), ma = moments(ma_v);
      e.mu_norm = mn.mean;
      e.mu_abn = ma.mean;
      e.delta_mu = ma.mean - mn.mean;
      std::vector<double> ln_v, la_v;
      for (double v : mn_v) ln_v.push_back(std::log1p(std::max(0.0, v)));
      for (double v : ma_v) la_v.push_back(std::log1p(std::max(0.0, v)));
      const Moments ln = moments(ln_v), la = moments(la_v);
      e.z_log_mu = (la.mean - ln.mean) / sigma_floor(ln);
    }
    e.score = std::abs(e.delta_beta) * (std::abs(e.z_beta) + std::abs(e.z_log_mu));
    entries.push_back(e);
  }
  // score descending, ties by class name (slots are in name order)
  std::sort(entries.begin(), entries.end(), [](const cs_suspect& a, const cs_suspect& b) {
    if (a.score != b.score) return a.score > b.score;
    return a.beta_slot < b.beta_slot;
  });

  // attribute_straggler (rca.cpp:311-353): communicator groups are runs of
  // comm slots with the same (class, commHash) (slots are in (name, hash,
  // rank) order, the reference's map order); per group and rank, the betas of
  // the cycles where that (class, comm, rank) occurs, in window order
  if (R && lay->comm_class && lay->comm_group && lay->comm_rank) {
    auto values = [&](const cs_rca_window* w, uint32_t k) {
      std::vector<double> v;
      for (uint64_t c = 0; c < w->n_cycles; ++c)
        if (w->coll_present[c * R + k]) v.push_back(w->coll[c * R + k]);
      return v;
    };
    for (cs_suspect& e : entries) {
      int32_t best_slot = -1;
      double best_shift = 0.0;
      for (uint32_t g0 = 0; g0 < R;) {
        uint32_t g1 = g0 + 1;
        while (g1 < R && lay->comm_group[g1] == lay->comm_group[g0]) ++g1;
        if (lay->comm_class[g0] == e.beta_slot) {
          std::vector<uint32_t> ranks;  // ranks seen in the abnormal window
          for (uint32_t k = g0; k < g1; ++k)
            for (uint64_t c = 0; c < abnormal->n_cycles; ++c)
              if (abnormal->coll_present[c * R + k]) {
                ranks.push_back(k);
                break;
              }
          if (ranks.size() >= 2) {
            for (uint32_t k : ranks) {
              const Moments abn = moments(values(abnormal, k));
              const Moments nrm = moments(values(normal, k));  // empty -> mean 0
              const double shift = std::abs(abn.mean - nrm.mean);
              if (shift > best_shift) {
                best_shift = shift;
                best_slot = static_cast<int32_t>(k);
              }
            }
          }
        }
        g0 = g1;
      }
      if (best_slot < 0) continue;
      e.straggler_slot = best_slot;
      e.rank_beta_shift = best_shift;
      e.straggler_location = lay->comm_location ? lay->comm_location[best_slot] : -1;
    }
  }
  *n_out = entries.size();
  if (out) {
    if (cap < entries.size()) return CS_E_INVALID_ARGUMENT;
    std::memcpy(out, entries.data(), entries.size() * sizeof(cs_suspect));
  }
  return CS_OK;
}

int cs_rank_suspects(const cs_rca_window* normal, const cs_rca_window* abnormal,
                     const cs_rca_layout* lay, cs_suspect* out, size_t cap, size_t* n_out) {
  return cs_guard([&] { return cs_rank_suspects_impl(normal, abnormal, lay, out, cap, n_out); });
}

}  // extern "C"
