// cs_wire.cpp — host encoder for the columnar wire format (include/cyclescope_b200.h).
//
// The producer side of cs_upload_wire.  The batch's distinct (event info,
// payload width) pairs go to a dictionary of at most CS_WIRE_MAX_DICT entries
// (the most frequent ones).  Every event becomes a code byte (dictionary
// code, or CS_WIRE_ESCAPE, plus CS_WIRE_LONG_DT when its start_ts delta needs
// more than 16 bits) and a 16-bit delta from the previous event of its
// instance-aligned block; the delta's high byte, span durations (24 bits),
// batch/collective payloads (8 or 16 bits, batch indices relative to a
// per-block base) and counter values (f64) go to their own columns in event
// order.  Anything that does not fit is escaped to a full cs_event.  The
// workload table travels as u32 triples when every value fits.  Three passes
// over the blocks, each split across threads: count dictionary keys, count
// column entries per block, fill at prefix offsets.
#include <algorithm>
#include <cstring>
#include <thread>
#include <unordered_map>
#include <vector>

#include "cs_parallel.h"
#include "cs_guard.h"
#include "cyclescope_b200.h"

struct cs_wire_trace {
  std::vector<uint8_t> code, dt_hi, dur_hi, pay8;
  std::vector<uint16_t> dt_lo, dur_lo, pay16;
  std::vector<uint32_t> dict, wl32;
  std::vector<cs_wire_block> blocks;
  std::vector<double> values;
  std::vector<cs_event> escapes;
  bool has_wl32 = false;
};

namespace {

constexpr int64_t kLimit24 = int64_t{1} << 24;
constexpr uint32_t kNoKey = 0xffffffffu;
constexpr uint32_t kWide = 1u << 30;  // dictionary bit: payload in the 16-bit column

struct Block {
  uint64_t begin, end;
};

bool is_span(const cs_event& e) { return e.kind == CS_SPAN; }
bool has_value(const cs_event& e) { return e.kind == CS_COUNTER && (e.flags & CS_EV_HAS_VALUE); }
bool has_payload(const cs_event& e) { return (e.flags & (CS_EV_HAS_BATCH | CS_EV_HAS_COMM)) != 0; }

// the payload as carried on the wire (collective slot, or batch index -
// block base), or -1 when it cannot be carried
int64_t wire_payload(const cs_event& e, uint32_t batch_base) {
  const bool batch = e.flags & CS_EV_HAS_BATCH, comm = e.flags & CS_EV_HAS_COMM;
  if (batch && comm) return -1;
  if (comm) return (e.payload & 0xffffffffull) ? -1 : static_cast<int64_t>(e.payload >> 32);
  if (batch) return (e.payload >> 32) || e.payload < batch_base ? -1 : static_cast<int64_t>(e.payload - batch_base);
  return e.payload == 0 ? 0 : -1;
}

// dictionary key: packed info | kWide, or kNoKey when a field does not fit
uint32_t key_of(const cs_event& e, uint32_t batch_base) {
  if (e.name_id > 0xffffu || e.kind >= 16 || e.category >= 16 || (e.flags & ~0x3fu)) return kNoKey;
  const int64_t p = wire_payload(e, batch_base);
  if (p < 0 || p > 0xffff) return kNoKey;
  return e.name_id | (static_cast<uint32_t>(e.kind) << 16) | (static_cast<uint32_t>(e.category) << 20) |
         (static_cast<uint32_t>(e.flags) << 24) | (has_payload(e) && p > 0xff ? kWide : 0u);
}

// key -> code, open addressing over 512 slots (<= 127 entries)
struct DictIndex {
  uint32_t key[512];
  uint8_t code[512];
  DictIndex() { std::fill(key, key + 512, kNoKey); }
  static uint32_t h(uint32_t x) { return (x * 0x9E3779B1u) >> 23; }
  void put(uint32_t x, uint8_t c) {
    uint32_t i = h(x);
    while (key[i] != kNoKey) i = (i + 1) & 511u;
    key[i] = x;
    code[i] = c;
  }
  uint32_t get(uint32_t x) const {
    if (x == kNoKey) return CS_WIRE_ESCAPE;
    for (uint32_t i = h(x);; i = (i + 1) & 511u) {
      if (key[i] == x) return code[i];
      if (key[i] == kNoKey) return CS_WIRE_ESCAPE;
    }
  }
};

// the event's dictionary code, or CS_WIRE_ESCAPE when it does not fit
uint32_t encode_code(const cs_event& e, int64_t prev_ts, uint32_t batch_base, const DictIndex& dix) {
  const int64_t dt = e.start_ts - prev_ts;
  if (dt < 0 || dt >= kLimit24) return CS_WIRE_ESCAPE;
  if (is_span(e)) {
    if (e.duration < 0 || e.duration >= kLimit24) return CS_WIRE_ESCAPE;
  } else if (!has_value(e) && e.duration != 0) {
    return CS_WIRE_ESCAPE;
  }
  return dix.get(key_of(e, batch_base));
}

using cs_host::parallel_for;

// column entry counts of one event: [dur, pay8, pay16, val, dt_hi, esc]
void count_event(const cs_event& e, uint32_t code, int64_t dt, uint32_t key, uint64_t c[6]) {
  if (code == CS_WIRE_ESCAPE) {
    ++c[5];
    return;
  }
  c[0] += is_span(e);
  if (has_payload(e)) ++c[(key & kWide) ? 2 : 1];
  c[3] += has_value(e);
  c[4] += dt > 0xffff;
}

}  // namespace

extern "C" {

static int cs_wire_pack_impl(uint32_t n_inst, const uint64_t* off, const cs_event* ev, uint64_t n_workloads,
                 const cs_workload* wl, uint32_t n_threads, cs_wire_trace** out) {
  if (!out || !off || n_inst == 0 || off[0] != 0 || (n_workloads && !wl)) return CS_E_INVALID_ARGUMENT;
  *out = nullptr;
  for (uint32_t i = 0; i < n_inst; ++i)
    if (off[i + 1] < off[i]) return CS_E_INVALID_ARGUMENT;
  const uint64_t n = off[n_inst];
  if (n && !ev) return CS_E_INVALID_ARGUMENT;
  if (n_threads == 0) n_threads = 1;
  std::vector<Block> blocks;
  for (uint32_t i = 0; i < n_inst; ++i)
    for (uint64_t b = off[i]; b < off[i + 1]; b += CS_WIRE_BLOCK)
      blocks.push_back({b, std::min<uint64_t>(b + CS_WIRE_BLOCK, off[i + 1])});
  const size_t nb = blocks.size();
  auto* w = new cs_wire_trace();
  w->blocks.resize(nb);
  // ---- per block: bases
  parallel_for(nb, n_threads, [&](size_t k0, size_t k1, uint32_t) {
    for (size_t k = k0; k < k1; ++k) {
      const Block& bl = blocks[k];
      cs_wire_block& B = w->blocks[k];
      B = cs_wire_block{};
      B.base_ts = ev[bl.begin].start_ts;
      for (uint64_t j = bl.begin; j < bl.end; ++j)
        if ((ev[j].flags & (CS_EV_HAS_BATCH | CS_EV_HAS_COMM)) == CS_EV_HAS_BATCH && (ev[j].payload >> 32) == 0) {
          B.batch_base = static_cast<uint32_t>(ev[j].payload);
          break;
        }
    }
  });
  // ---- dictionary: the CS_WIRE_MAX_DICT most frequent keys, sorted
  std::vector<std::unordered_map<uint32_t, uint64_t>> hist(n_threads);
  parallel_for(nb, n_threads, [&](size_t k0, size_t k1, uint32_t t) {
    auto& m = hist[t];
    uint32_t last = kNoKey;
    uint64_t run = 0;
    for (size_t k = k0; k < k1; ++k)
      for (uint64_t j = blocks[k].begin; j < blocks[k].end; ++j) {
        const uint32_t x = key_of(ev[j], w->blocks[k].batch_base);
        if (x == last) {
          ++run;
          continue;
        }
        if (last != kNoKey) m[last] += run;
        last = x;
        run = 1;
      }
    if (last != kNoKey) m[last] += run;
  });
  for (uint32_t t = 1; t < n_threads; ++t)
    for (const auto& kv : hist[t]) hist[0][kv.first] += kv.second;
  std::vector<std::pair<uint64_t, uint32_t>> by_count;
  for (const auto& kv : hist[0]) by_count.push_back({kv.second, kv.first});
  std::sort(by_count.begin(), by_count.end(),
            [](const auto& a, const auto& b) { return a.first != b.first ? a.first > b.first : a.second < b.second; });
  if (by_count.size() > CS_WIRE_MAX_DICT) by_count.resize(CS_WIRE_MAX_DICT);
  for (const auto& x : by_count) w->dict.push_back(x.second);
  std::sort(w->dict.begin(), w->dict.end());
  DictIndex dix;
  for (uint32_t c = 0; c < w->dict.size(); ++c) dix.put(w->dict[c], static_cast<uint8_t>(c));

  // ---- per block: column entry counts, then prefixes
  std::vector<uint64_t> cnt(6 * (nb + 1), 0);
  parallel_for(nb, n_threads, [&](size_t k0, size_t k1, uint32_t) {
    for (size_t k = k0; k < k1; ++k) {
      const Block& bl = blocks[k];
      const cs_wire_block& B = w->blocks[k];
      uint64_t c[6] = {0, 0, 0, 0, 0, 0};
      int64_t prev = B.base_ts;
      for (uint64_t j = bl.begin; j < bl.end; ++j) {
        const cs_event& e = ev[j];
        const uint32_t code = encode_code(e, prev, B.batch_base, dix);
        count_event(e, code, e.start_ts - prev, code == CS_WIRE_ESCAPE ? 0u : w->dict[code], c);
        prev = e.start_ts;
      }
      for (int q = 0; q < 6; ++q) cnt[6 * (k + 1) + q] = c[q];
    }
  });
  for (size_t k = 0; k < nb; ++k)
    for (int q = 0; q < 6; ++q) cnt[6 * (k + 1) + q] += cnt[6 * k + q];
  w->code.resize(n);
  w->dt_lo.resize(n);
  w->dur_lo.resize(cnt[6 * nb + 0]);
  w->dur_hi.resize(cnt[6 * nb + 0]);
  w->pay8.resize(cnt[6 * nb + 1]);
  w->pay16.resize(cnt[6 * nb + 2]);
  w->values.resize(cnt[6 * nb + 3]);
  w->dt_hi.resize(cnt[6 * nb + 4]);
  w->escapes.resize(cnt[6 * nb + 5]);

  // ---- fill
  parallel_for(nb, n_threads, [&](size_t k0, size_t k1, uint32_t) {
    for (size_t k = k0; k < k1; ++k) {
      const Block& bl = blocks[k];
      cs_wire_block& B = w->blocks[k];
      uint64_t c[6];
      for (int q = 0; q < 6; ++q) c[q] = cnt[6 * k + q];
      B.dur = c[0], B.pay8 = c[1], B.pay16 = c[2], B.val = c[3], B.dt_hi = c[4], B.esc = c[5];
      int64_t prev = B.base_ts;
      for (uint64_t j = bl.begin; j < bl.end; ++j) {
        const cs_event& e = ev[j];
        const uint32_t code = encode_code(e, prev, B.batch_base, dix);
        const int64_t dt = e.start_ts - prev;
        prev = e.start_ts;
        if (code == CS_WIRE_ESCAPE) {
          w->code[j] = CS_WIRE_ESCAPE;
          w->dt_lo[j] = 0;
          w->escapes[c[5]++] = e;
          continue;
        }
        w->code[j] = static_cast<uint8_t>(code | (dt > 0xffff ? CS_WIRE_LONG_DT : 0u));
        w->dt_lo[j] = static_cast<uint16_t>(dt);
        if (dt > 0xffff) w->dt_hi[c[4]++] = static_cast<uint8_t>(dt >> 16);
        if (is_span(e)) {
          w->dur_lo[c[0]] = static_cast<uint16_t>(e.duration);
          w->dur_hi[c[0]++] = static_cast<uint8_t>(e.duration >> 16);
        }
        if (has_payload(e)) {
          const int64_t p = wire_payload(e, B.batch_base);
          if (w->dict[code] & kWide) w->pay16[c[2]++] = static_cast<uint16_t>(p);
          else w->pay8[c[1]++] = static_cast<uint8_t>(p);
        }
        if (has_value(e)) std::memcpy(&w->values[c[3]++], &e.duration, sizeof(double));
      }
    }
  });
  // ---- workload table as u32 triples when every value fits (missing = 0xffffffff)
  bool fits = true;
  auto enc = [&](int64_t v) -> uint32_t {
    if (v == INT64_MIN) return 0xffffffffu;
    if (v < 0 || v >= 0xffffffffll) fits = false;
    return static_cast<uint32_t>(v);
  };
  w->wl32.resize(3 * n_workloads);
  for (uint64_t i = 0; i < n_workloads && fits; ++i) {
    w->wl32[3 * i] = enc(wl[i].batch);
    w->wl32[3 * i + 1] = enc(wl[i].input_len);
    w->wl32[3 * i + 2] = enc(wl[i].output_len);
  }
  w->has_wl32 = fits && n_workloads > 0;
  if (!w->has_wl32) w->wl32.clear();
  *out = w;
  return CS_OK;
}

int cs_wire_pack(uint32_t n_inst, const uint64_t* off, const cs_event* ev, uint64_t n_workloads,
                 const cs_workload* wl, uint32_t n_threads, cs_wire_trace** out) {
  return cs_guard([&] { return cs_wire_pack_impl(n_inst, off, ev, n_workloads, wl, n_threads, out); });
}

int cs_wire_view(const cs_wire_trace* w, cs_wire_batch* out, uint64_t* n_blocks) {
  if (!w || !out) return CS_E_INVALID_ARGUMENT;
  *out = cs_wire_batch{};
  out->codes = w->code.data();
  out->dt_lo = w->dt_lo.data();
  out->dt_hi = w->dt_hi.data();
  out->n_dt_hi = w->dt_hi.size();
  out->dict = w->dict.data();
  out->n_dict = static_cast<uint32_t>(w->dict.size());
  out->blocks = w->blocks.data();
  out->dur_lo = w->dur_lo.data();
  out->dur_hi = w->dur_hi.data();
  out->n_durations = w->dur_lo.size();
  out->pay8 = w->pay8.data();
  out->n_pay8 = w->pay8.size();
  out->pay16 = w->pay16.data();
  out->n_pay16 = w->pay16.size();
  out->values = w->values.data();
  out->n_values = w->values.size();
  out->escapes = w->escapes.data();
  out->n_escapes = w->escapes.size();
  out->workloads32 = w->has_wl32 ? w->wl32.data() : nullptr;
  out->n_workloads32 = w->has_wl32 ? w->wl32.size() / 3 : 0;
  if (n_blocks) *n_blocks = w->blocks.size();
  return CS_OK;
}

void cs_wire_free(cs_wire_trace* w) { delete w; }

}  // extern "C"
