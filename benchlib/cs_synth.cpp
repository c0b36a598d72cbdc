// cs_synth.cpp — synthetic trace producer for benchmarks and tests.
//
// A restatement of the reference's anomaly-simulation generator
// (simkit.cpp:34-86 generate_workload, 195-246 effects_for, 276-506
// synthesize_trace; rng.hpp:12-73 Rng) that writes our 32-byte event records
// straight away instead of `TraceEvent` objects with std::map args.  Given
// the same seeds it produces the same trace as the reference, event for event
// (checked byte-for-byte against the reference simkit by
// tests/test_synth_parity.py).  Large instances are produced as independent
// chunks in parallel (each one synthesize_trace call with its own substream
// seeds) concatenated in time; the chunking is reported with every benchmark.
// Compiled with -ffp-contract=off: glibc libm + no FMA, like the reference.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "cs_bench.h"

namespace {

// Deterministic random source with the reference's transforms (rng.hpp).
class Rng {
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  double u01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * u01(); }
  int64_t uniform_int(int64_t lo, int64_t hi) {
    const double span = static_cast<double>(hi - lo) + 1.0;
    const int64_t v = lo + static_cast<int64_t>(u01() * span);
    return v > hi ? hi : v;
  }
  int64_t log_uniform_int(int64_t lo, int64_t hi) {
    const double a = std::log(static_cast<double>(lo));
    const double b = std::log(static_cast<double>(hi) + 1.0);
    int64_t v = static_cast<int64_t>(std::exp(uniform(a, b)));
    return v < lo ? lo : (v > hi ? hi : v);
  }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double u1 = u01();
    const double u2 = u01();
    while (u1 <= 0.0) u1 = u01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare_ = r * std::sin(th);
    spare_ok_ = true;
    return r * std::cos(th);
  }
  double log_normal(double sigma) { return std::exp(sigma * normal()); }
  static uint64_t substream(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }

 private:
  std::mt19937_64 eng_;
  double spare_ = 0.0;
  bool spare_ok_ = false;
};

// fixed provisional name ids; compacted to the names present at the end
enum Name : uint32_t {
  N_ATTN, N_BUS_UTIL, N_CPU_USAGE, N_LAUNCH, N_FWD_PREFILL, N_FREQUENCY, N_GEMM, N_GET_NEXT,
  N_GPU_CLOCK, N_GPU_USAGE, N_D2D, N_H2D, N_ONCPU, N_PAGE, N_PCIE, N_PBR, N_PBR_DECODE,
  N_REDUCE, N_RUN_BATCH, N_TX_BYTES, N_COUNT
};
const char* kNames[N_COUNT] = {
    "attn_kernel", "bus_util", "cpu_usage", "cuLaunchKernel", "forward_prefill", "frequency",
    "gemm_kernel", "get_next_batch_to_run", "gpu_clock", "gpu_usage", "memcpy_d2d",
    "memcpy_h2d", "oncpu", "page_activity", "pcie_util", "process_batch_result",
    "process_batch_result_decode", "reduce", "run_batch", "tx_bytes"};

struct Workload {
  bool prefill;
  int64_t batch, in, out;
};

// generate_workload (simkit.cpp:34-86), default LogUniform profile
std::vector<Workload> gen_workload(uint64_t n, uint64_t seed) {
  std::vector<Workload> v;
  v.reserve(n);
  Rng rng(seed);
  while (v.size() < n) {
    const int64_t total = rng.log_uniform_int(1, 512);
    Workload p{true, 0, 0, 0};
    p.batch = rng.log_uniform_int(1, 512);
    p.in = rng.log_uniform_int(1, 2048);
    v.push_back(p);
    for (int64_t step = 1; step <= total && v.size() < n; ++step) {
      Workload d{false, 0, 0, step};
      d.batch = rng.log_uniform_int(1, 512);
      d.in = rng.log_uniform_int(1, 2048);
      v.push_back(d);
    }
  }
  v.resize(std::min<size_t>(v.size(), n));
  return v;
}

struct Fx {
  double oncpu = 1, post = 1, gemm = 1, attn = 1, h2d = 1, d2d = 1, red_s = 1, red_o = 1;
  int straggler = 0;
  bool anomalous = false;
  double cpu_add = 0;
  bool iowait = false, saturated = false;
  double gpu_add = 0, clock_mult = 1, freq_mult = 1, page_mult = 1, tx_mult = 1, pcie_add = 0,
         bus_add = 0;
};

double default_severity(int f) {
  static const double s[8] = {12.0, 8.0, 5.0, 5.0, 14.0, 18.0, 16.0, 20.0};
  return f >= 0 && f < 8 ? s[f] : 4.0;
}

int64_t to_ns(double s) { return static_cast<int64_t>(std::llround(s * 1e9)); }

struct Out {
  std::vector<cs_event> ev;
  std::vector<uint64_t> id;
  std::vector<cs_workload> wl;
  std::vector<uint8_t> labels;
  int64_t cursor = 0;  // closing anchor start
};

// synthesize_trace (simkit.cpp:276-506), GroundTruthModel defaults
void synthesize(const cs_synth_params& p, uint64_t wseed, uint64_t sseed, uint64_t cyc_begin,
                uint64_t n_cyc, Out& o) {
  const auto work = gen_workload(n_cyc, wseed);
  Rng rng(sseed);
  const double a = 2e-8, b = 1e-5, c = 1e-3, cpu_fixed = 2.2e-3, cpu_per_batch = 0.0;
  const double noise = p.noise >= 0.0 ? p.noise : 0.05;
  const double prefill_per_token = 4e-8, prefill_noise = 0.2;
  const uint64_t n_ranks = std::max<uint64_t>(1, p.n_ranks);
  const double sev = p.severity > 0.0 ? p.severity : default_severity(p.fault_family);
  uint64_t next_id = 1;
  o.labels.assign(work.size(), 0);
  o.ev.reserve(work.size() * (19 + n_ranks));
  o.id.reserve(work.size() * (19 + n_ranks));
  auto emit = [&](uint8_t kind, uint8_t cat, uint32_t name, int64_t start, int64_t dur) -> cs_event& {
    cs_event e{};
    e.start_ts = start;
    e.duration = kind == CS_SPAN ? dur : 0;
    e.name_id = name;
    e.kind = kind;
    e.category = cat;
    o.ev.push_back(e);
    o.id.push_back(next_id++);
    return o.ev.back();
  };
  auto counter = [&](uint32_t name, int64_t ts, double value) {
    cs_event& e = emit(CS_COUNTER, CS_CAT_COUNTER_TELEMETRY, name, ts, 0);
    const double v = std::max(0.0, value);
    std::memcpy(&e.duration, &v, sizeof v);
    e.flags = CS_EV_HAS_VALUE;
  };
  int64_t cursor = 0;
  for (size_t k = 0; k < work.size(); ++k) {
    const Workload& w = work[k];
    const uint64_t gidx = cyc_begin + k;  // fault windows are in global cycles
    Fx fx;
    if (p.fault_family >= 0 && gidx >= p.fault_onset && gidx < p.fault_onset + p.fault_duration) {
      fx.anomalous = true;
      const double s = sev;
      switch (p.fault_family) {
        case 0: fx.oncpu *= s; fx.cpu_add += 16.0; break;
        case 1: fx.oncpu *= s; fx.post *= s; fx.freq_mult *= 1.0 / s; fx.saturated = true; break;
        case 2: fx.gemm *= s; fx.attn *= s; fx.gpu_add += 35.0; break;
        case 3: fx.gemm *= s; fx.attn *= s; fx.clock_mult *= 1.0 / s; break;
        case 4: fx.oncpu *= s * rng.uniform(0.8, 1.6); fx.page_mult *= 12.0; fx.iowait = true; break;
        case 5:
          fx.red_s *= s;
          fx.red_o *= 1.0 + 0.5 * (s - 1.0);
          fx.straggler = p.target_rank;
          fx.tx_mult *= s;
          break;
        case 6: fx.h2d *= s; fx.pcie_add += 58.0; break;
        case 7: fx.d2d *= s; fx.bus_add += 60.0; break;
        default: break;
      }
    }
    o.labels[k] = fx.anomalous;
    if (w.prefill && gidx > 0) cursor += to_ns(rng.uniform(2e-3, 8e-3));
    double lat, gemm_s, attn_s, h2d_s, d2d_s, oncpu_s, reduce_s, post_s;
    if (w.prefill) {
      const double base = prefill_per_token * static_cast<double>(w.batch * w.in) + c + cpu_fixed;
      lat = base * rng.log_normal(prefill_noise);
      gemm_s = 0.55 * lat;
      attn_s = 0.30 * lat;
      h2d_s = 0.08 * lat;
      d2d_s = 0.04 * lat;
      oncpu_s = 0.20 * lat;
      reduce_s = 0.05 * lat;
      post_s = 0.05 * lat;
    } else {
      const int64_t kv = w.batch * (w.in + w.out);
      const double gpu_base = a * static_cast<double>(kv) + b * static_cast<double>(w.batch) + c;
      const double cpu_base = cpu_fixed + cpu_per_batch * static_cast<double>(w.batch);
      gemm_s = 0.40 * gpu_base * fx.gemm;
      attn_s = 0.30 * gpu_base * fx.attn;
      h2d_s = 0.18 * gpu_base * fx.h2d;
      d2d_s = 0.12 * gpu_base * fx.d2d;
      const double gpu_eff = gemm_s + attn_s + h2d_s + d2d_s;
      oncpu_s = 0.50 * cpu_base * fx.oncpu;
      reduce_s = 0.30 * cpu_base * fx.red_s;
      post_s = 0.20 * cpu_base * fx.post;
      const double cpu_eff = oncpu_s + reduce_s + post_s;
      const double exec = gpu_eff < cpu_eff ? cpu_eff : gpu_eff;
      lat = exec * (noise > 0.0 ? rng.log_normal(noise) : 1.0);
    }
    const int64_t t = cursor;
    const int64_t run_ns = std::max<int64_t>(1000, to_ns(lat));
    {
      cs_event& an = emit(CS_SPAN, CS_CAT_PYTHON_CALL, N_RUN_BATCH, t, run_ns);
      an.flags = (w.prefill ? CS_EV_FM_PREFILL : CS_EV_FM_DECODE) | CS_EV_HAS_BATCH;
      if (w.batch >= 0 && w.in >= 0 && w.out >= 0) an.flags |= CS_EV_WL_OK;
      an.payload = o.wl.size();
      o.wl.push_back({w.batch, w.in, w.out});
      (void)rng.log_normal(0.01);  // post_run_latency arg (not encoded)
    }
    if (!w.prefill)
      emit(CS_INSTANT, CS_CAT_PYTHON_CALL, N_PBR_DECODE, t + run_ns / 2, 0);
    else
      emit(CS_INSTANT, CS_CAT_PYTHON_CALL, N_FWD_PREFILL, t + run_ns / 4, 0);
    {
      const double gpu_total = gemm_s + attn_s + h2d_s + d2d_s;
      const double scale = gpu_total > 0.0 ? std::min(1.0, 0.96 * lat / gpu_total) : 1.0;
      int64_t gc = t + run_ns / 100;
      emit(CS_SPAN, CS_CAT_RUNTIME_API, N_LAUNCH, t + run_ns / 200, std::max<int64_t>(500, run_ns / 500));
      auto gspan = [&](uint32_t name, uint8_t cat, double secs) {
        const int64_t d = std::max<int64_t>(200, to_ns(secs * scale));
        const int64_t st = gc;
        emit(CS_SPAN, cat, name, st, d);
        gc += d + std::max<int64_t>(50, run_ns / 2000);
        return std::make_pair(st, d);
      };
      auto g1 = gspan(N_GEMM, CS_CAT_GPU_KERNEL, gemm_s);
      counter(N_GPU_USAGE, g1.first + g1.second / 2, 55.0 + fx.gpu_add + rng.normal() * 3.0);
      auto g2 = gspan(N_ATTN, CS_CAT_GPU_KERNEL, attn_s);
      counter(N_GPU_CLOCK, g2.first + g2.second / 2, 1900.0 * fx.clock_mult + rng.normal() * 15.0);
      auto g3 = gspan(N_H2D, CS_CAT_MEM_COPY, h2d_s);
      counter(N_PCIE, g3.first + g3.second / 2, 22.0 + fx.pcie_add + rng.normal() * 2.0);
      auto g4 = gspan(N_D2D, CS_CAT_MEM_COPY, d2d_s);
      counter(N_BUS_UTIL, g4.first + g4.second / 2, 18.0 + fx.bus_add + rng.normal() * 2.0);
    }
    {
      const double base_reduce = reduce_s / fx.red_s;
      const int64_t rs = t + run_ns / 3;
      for (uint64_t r = 0; r < n_ranks; ++r) {
        double rr = reduce_s;
        if (n_ranks > 1)
          rr = base_reduce * ((static_cast<int>(r) == fx.straggler) ? fx.red_s : fx.red_o);
        const int64_t d = std::max<int64_t>(200, to_ns(rr * rng.log_normal(0.02)));
        cs_event& e = emit(CS_SPAN, CS_CAT_COLLECTIVE_COMM, N_REDUCE, rs, d);
        e.flags = CS_EV_HAS_COMM;
        e.payload = static_cast<uint64_t>(r) << 32;  // (reduce, comm0, r) -> slot r
        if (r == 0) counter(N_TX_BYTES, rs + d / 2, 1e9 * fx.tx_mult + rng.normal() * 2e7);
      }
    }
    {
      const double cpu_total = oncpu_s + post_s;
      const double scale = cpu_total > 0.0 ? std::min(1.0, 0.96 * lat / cpu_total) : 1.0;
      const int64_t ot = std::max<int64_t>(400, to_ns(oncpu_s * scale));
      const int64_t o1s = t + run_ns / 50, o1d = ot / 2;
      emit(CS_SPAN, CS_CAT_OS_SCHED, N_ONCPU, o1s, o1d);
      emit(CS_SPAN, CS_CAT_OS_SCHED, N_ONCPU, t + run_ns / 2, ot - o1d);
      double busy = 82.0 + rng.normal() * 3.0;
      if (fx.iowait) busy = 38.0 + rng.normal() * 6.0;
      if (fx.saturated) busy = 97.0 + rng.normal() * 1.0;
      busy = std::min(100.0, busy + fx.cpu_add);
      counter(N_CPU_USAGE, o1s + o1d / 2, busy);
      const int64_t post_ns = std::min<int64_t>(
          run_ns / 2, std::max<int64_t>(200, to_ns(post_s * scale * rng.log_normal(1.1))));
      const int64_t ps = t + run_ns - post_ns;
      emit(CS_SPAN, CS_CAT_PYTHON_CALL, N_PBR, ps, post_ns);
      counter(N_FREQUENCY, ps + post_ns / 2, 2800.0 * fx.freq_mult + rng.normal() * 25.0);
    }
    counter(N_PAGE, t + run_ns / 2, 40.0 * fx.page_mult + rng.normal() * 4.0);
    const int64_t sched =
        std::clamp<int64_t>(to_ns(60e-6 * rng.log_normal(1.3)), 5000, 5000000);
    emit(CS_SPAN, CS_CAT_PYTHON_CALL, N_GET_NEXT, t + run_ns, sched);
    cursor = t + run_ns + sched;
  }
  emit(CS_SPAN, CS_CAT_PYTHON_CALL, N_RUN_BATCH, cursor, 1000);
  o.cursor = cursor;
  // canonical order (start_ts, event_id)
  std::vector<uint32_t> perm(o.ev.size());
  for (uint32_t i = 0; i < perm.size(); ++i) perm[i] = i;
  std::sort(perm.begin(), perm.end(), [&](uint32_t x, uint32_t y) {
    if (o.ev[x].start_ts != o.ev[y].start_ts) return o.ev[x].start_ts < o.ev[y].start_ts;
    return o.id[x] < o.id[y];
  });
  std::vector<cs_event> ev(o.ev.size());
  std::vector<uint64_t> id(o.ev.size());
  for (size_t i = 0; i < perm.size(); ++i) {
    ev[i] = o.ev[perm[i]];
    id[i] = o.id[perm[i]];
  }
  // workload indices follow canonical order of the carriers
  std::vector<cs_workload> wl;
  wl.reserve(o.wl.size());
  for (auto& e : ev)
    if (e.flags & CS_EV_HAS_BATCH) {
      const uint64_t old = e.payload & 0xffffffffu;
      e.payload = (e.payload & ~0xffffffffull) | wl.size();
      wl.push_back(o.wl[old]);
    }
  o.ev.swap(ev);
  o.id.swap(id);
  o.wl.swap(wl);
}

}  // namespace

struct cs_synth_trace {
  std::vector<cs_event> ev;
  std::vector<uint64_t> id;
  std::vector<cs_workload> wl;
  std::vector<uint8_t> labels;
  std::vector<std::string> names;
  std::string packed;
  uint32_t n_comm = 0;
};

extern "C" {

int cs_synth_generate(const cs_synth_params* p, uint32_t n_chunks, uint32_t n_threads,
                      int compact_names, cs_synth_trace** out) {
  if (!p || !out || n_chunks == 0) return CS_E_INVALID_ARGUMENT;
  *out = nullptr;
  if (p->fault_family < -1 || p->fault_family > 7) return CS_E_INVALID_ARGUMENT;
  const uint64_t n = p->n_cycles;
  if (n_chunks > n && n > 0) n_chunks = static_cast<uint32_t>(n);
  std::vector<Out> parts(n_chunks);
  std::vector<uint64_t> begin(n_chunks + 1, 0);
  for (uint32_t k = 0; k <= n_chunks; ++k) begin[k] = n * k / n_chunks;
  auto job = [&](uint32_t k) {
    // chunk 0 of a single-chunk trace uses the caller's seeds unchanged
    const uint64_t ws = n_chunks == 1 ? p->workload_seed : Rng::substream(p->workload_seed, k);
    const uint64_t ss = n_chunks == 1 ? p->synth_seed : Rng::substream(p->synth_seed, k);
    synthesize(*p, ws, ss, begin[k], begin[k + 1] - begin[k], parts[k]);
  };
  const uint32_t nt = std::max<uint32_t>(1, std::min(n_threads, n_chunks));
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (uint32_t k = t; k < n_chunks; k += nt) job(k);
    });
  for (auto& x : th) x.join();
  auto* tr = new cs_synth_trace();
  // concatenate in time: drop each non-final chunk's closing anchor (the last
  // event with start == cursor named run_batch) and shift the next chunk
  size_t total = 0, total_wl = 0;
  for (auto& o : parts) {
    total += o.ev.size();
    total_wl += o.wl.size();
  }
  tr->ev.reserve(total);
  tr->id.reserve(total);
  tr->wl.reserve(total_wl);
  int64_t shift = 0;
  uint64_t id_shift = 0;
  for (uint32_t k = 0; k < n_chunks; ++k) {
    Out& o = parts[k];
    size_t closing = o.ev.size();
    if (k + 1 < n_chunks) {
      for (size_t i = o.ev.size(); i-- > 0;)
        if (o.ev[i].name_id == N_RUN_BATCH && o.ev[i].start_ts == o.cursor && !(o.ev[i].flags & CS_EV_HAS_BATCH)) {
          closing = i;
          break;
        }
    }
    const uint64_t wl_base = tr->wl.size();
    uint64_t max_id = 0;
    for (size_t i = 0; i < o.ev.size(); ++i) {
      if (i == closing) continue;
      cs_event e = o.ev[i];
      e.start_ts += shift;
      if (e.flags & CS_EV_HAS_BATCH) e.payload = (e.payload & ~0xffffffffull) | (wl_base + (e.payload & 0xffffffffu));
      tr->ev.push_back(e);
      tr->id.push_back(o.id[i] + id_shift);
      max_id = std::max(max_id, o.id[i]);
    }
    tr->wl.insert(tr->wl.end(), o.wl.begin(), o.wl.end());
    tr->labels.insert(tr->labels.end(), o.labels.begin(), o.labels.end());
    shift += o.cursor;
    id_shift += max_id;
    std::vector<cs_event>().swap(o.ev);
    std::vector<uint64_t>().swap(o.id);
  }
  // chunks are time-disjoint unless a trailing counter overshoots the cursor
  bool sorted = true;
  for (size_t i = 1; i < tr->ev.size() && sorted; ++i)
    sorted = tr->ev[i - 1].start_ts < tr->ev[i].start_ts ||
             (tr->ev[i - 1].start_ts == tr->ev[i].start_ts && tr->id[i - 1] < tr->id[i]);
  if (!sorted) {
    std::vector<uint64_t> perm(tr->ev.size());
    for (uint64_t i = 0; i < perm.size(); ++i) perm[i] = i;
    std::sort(perm.begin(), perm.end(), [&](uint64_t x, uint64_t y) {
      if (tr->ev[x].start_ts != tr->ev[y].start_ts) return tr->ev[x].start_ts < tr->ev[y].start_ts;
      return tr->id[x] < tr->id[y];
    });
    std::vector<cs_event> ev(perm.size());
    std::vector<uint64_t> id(perm.size());
    for (size_t i = 0; i < perm.size(); ++i) {
      ev[i] = tr->ev[perm[i]];
      id[i] = tr->id[perm[i]];
    }
    std::vector<cs_workload> wl;
    for (auto& e : ev)
      if (e.flags & CS_EV_HAS_BATCH) {
        const uint64_t old = e.payload & 0xffffffffu;
        e.payload = (e.payload & ~0xffffffffull) | wl.size();
        wl.push_back(tr->wl[old]);
      }
    tr->ev.swap(ev);
    tr->id.swap(id);
    tr->wl.swap(wl);
  }
  // name table: all simkit names, or only those present (= the reference
  // export's interning of the trace's names)
  std::vector<uint32_t> remap(N_COUNT);
  if (compact_names) {
    std::vector<uint8_t> present(N_COUNT, 0);
    for (const auto& e : tr->ev) present[e.name_id] = 1;
    uint32_t k = 0;
    for (uint32_t i = 0; i < N_COUNT; ++i)
      if (present[i]) {
        remap[i] = k++;
        tr->names.push_back(kNames[i]);
      }
    for (auto& e : tr->ev) e.name_id = remap[e.name_id];
  } else {
    for (uint32_t i = 0; i < N_COUNT; ++i) tr->names.push_back(kNames[i]);
  }
  for (const auto& s : tr->names) {
    tr->packed += s;
    tr->packed.push_back('\0');
  }
  tr->n_comm = static_cast<uint32_t>(std::max<uint64_t>(1, p->n_ranks));
  *out = tr;
  return CS_OK;
}

int cs_synth_view(const cs_synth_trace* t, const cs_event** ev, uint64_t* n_ev,
                  const uint64_t** ids, const cs_workload** wl, uint64_t* n_wl,
                  const uint8_t** labels, uint64_t* n_cycles) {
  if (!t) return CS_E_INVALID_ARGUMENT;
  if (ev) *ev = t->ev.data();
  if (n_ev) *n_ev = t->ev.size();
  if (ids) *ids = t->id.data();
  if (wl) *wl = t->wl.data();
  if (n_wl) *n_wl = t->wl.size();
  if (labels) *labels = t->labels.data();
  if (n_cycles) *n_cycles = t->labels.size();
  return CS_OK;
}

int cs_synth_names(const cs_synth_trace* t, const char** packed, size_t* n_bytes,
                   uint32_t* n_names, uint32_t* n_comm) {
  if (!t) return CS_E_INVALID_ARGUMENT;
  if (packed) *packed = t->packed.data();
  if (n_bytes) *n_bytes = t->packed.size();
  if (n_names) *n_names = static_cast<uint32_t>(t->names.size());
  if (n_comm) *n_comm = t->n_comm;
  return CS_OK;
}

void cs_synth_free(cs_synth_trace* t) { delete t; }

}  // extern "C"
