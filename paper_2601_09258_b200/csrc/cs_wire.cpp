// cs_wire.cpp — host encoder for the columnar wire format (include/cyclescope_b200.h).
//
// The producer side of cs_upload_wire.  The batch's distinct event "info"
// words (name id | kind | category | flags) go to a dictionary of at most
// CS_WIRE_MAX_DICT entries (the most frequent ones); every event becomes one
// 32-bit word: its dictionary code and the 24-bit start_ts delta from the
// previous event of its instance-aligned block.  Span durations (24 bits),
// batch/collective payloads (16 bits, batch indices relative to a per-block
// base) and counter values (f64) go to their own columns in event order;
// anything that does not fit is escaped to a full cs_event.  Three passes,
// each split across threads: count info words, count column entries per
// block, fill at prefix offsets.
#include <algorithm>
#include <cstring>
#include <thread>
#include <unordered_map>
#include <vector>

#include "cyclescope_b200.h"

struct cs_wire_trace {
  std::vector<uint32_t> ev, dict;
  std::vector<cs_wire_block> blocks;
  std::vector<uint16_t> dur_lo, payload;
  std::vector<uint8_t> dur_hi;
  std::vector<double> values;
  std::vector<cs_event> escapes;
};

namespace {

constexpr int64_t kDtLimit = int64_t{1} << 24;
constexpr uint32_t kNoInfo = 0xffffffffu;

struct Block {
  uint64_t begin, end;
};

bool is_span(const cs_event& e) { return e.kind == CS_SPAN; }
bool has_value(const cs_event& e) { return e.kind == CS_COUNTER && (e.flags & CS_EV_HAS_VALUE); }
bool has_payload(const cs_event& e) { return (e.flags & (CS_EV_HAS_BATCH | CS_EV_HAS_COMM)) != 0; }

// the packed info word, or kNoInfo when a field does not fit its bits
uint32_t info_of(const cs_event& e) {
  if (e.name_id > 0xffffu || e.kind >= 16 || e.category >= 16 || (e.flags & ~0x3fu)) return kNoInfo;
  return e.name_id | (static_cast<uint32_t>(e.kind) << 16) | (static_cast<uint32_t>(e.category) << 20) |
         (static_cast<uint32_t>(e.flags) << 24);
}

// info word -> code, open addressing over 1024 slots (<= 255 entries)
struct DictIndex {
  uint32_t key[1024];
  uint8_t code[1024];
  DictIndex() { std::fill(key, key + 1024, kNoInfo); }
  static uint32_t h(uint32_t x) { return (x * 0x9E3779B1u) >> 22; }
  void put(uint32_t x, uint8_t c) {
    uint32_t i = h(x);
    while (key[i] != kNoInfo) i = (i + 1) & 1023u;
    key[i] = x;
    code[i] = c;
  }
  uint32_t get(uint32_t x) const {
    if (x == kNoInfo) return CS_WIRE_ESCAPE;
    for (uint32_t i = h(x);; i = (i + 1) & 1023u) {
      if (key[i] == x) return code[i];
      if (key[i] == kNoInfo) return CS_WIRE_ESCAPE;
    }
  }
};

// the event's code, or CS_WIRE_ESCAPE when it does not fit the columns
uint32_t encode_code(const cs_event& e, int64_t prev_ts, uint32_t batch_base, const DictIndex& dix) {
  const int64_t dt = e.start_ts - prev_ts;
  if (dt < 0 || dt >= kDtLimit) return CS_WIRE_ESCAPE;
  if (is_span(e)) {
    if (e.duration < 0 || e.duration >= kDtLimit) return CS_WIRE_ESCAPE;
  } else if (!has_value(e) && e.duration != 0) {
    return CS_WIRE_ESCAPE;
  }
  const bool batch = e.flags & CS_EV_HAS_BATCH, comm = e.flags & CS_EV_HAS_COMM;
  if (batch && comm) return CS_WIRE_ESCAPE;
  if (comm) {
    if ((e.payload & 0xffffffffull) != 0 || (e.payload >> 32) > 0xffffu) return CS_WIRE_ESCAPE;
  } else if (batch) {
    if ((e.payload >> 32) != 0 || e.payload < batch_base || e.payload - batch_base > 0xffffu)
      return CS_WIRE_ESCAPE;
  } else if (e.payload != 0) {
    return CS_WIRE_ESCAPE;
  }
  return dix.get(info_of(e));
}

template <typename F>
void parallel_for(size_t n, uint32_t n_threads, F f) {
  const uint32_t nt = std::max<uint32_t>(1, std::min<size_t>(n_threads, n ? n : 1));
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] { f(n * t / nt, n * (t + 1) / nt, t); });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

int cs_wire_pack(uint32_t n_inst, const uint64_t* off, const cs_event* ev, uint32_t n_threads,
                 cs_wire_trace** out) {
  if (!out || !off || n_inst == 0 || off[0] != 0) return CS_E_INVALID_ARGUMENT;
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

  // ---- dictionary: the CS_WIRE_MAX_DICT most frequent info words, sorted
  std::vector<std::unordered_map<uint32_t, uint64_t>> hist(n_threads);
  parallel_for(n, n_threads, [&](size_t j0, size_t j1, uint32_t t) {
    auto& m = hist[t];
    uint32_t last = kNoInfo;
    uint64_t run = 0;
    for (size_t j = j0; j < j1; ++j) {  // runs of equal words are common: count them first
      const uint32_t x = info_of(ev[j]);
      if (x == last) {
        ++run;
        continue;
      }
      if (last != kNoInfo) m[last] += run;
      last = x;
      run = 1;
    }
    if (last != kNoInfo) m[last] += run;
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

  // ---- per block: bases and [durations, payloads, values, escapes] counts
  w->ev.resize(n);
  w->blocks.resize(nb);
  std::vector<uint64_t> cnt(4 * (nb + 1), 0);
  parallel_for(nb, n_threads, [&](size_t k0, size_t k1, uint32_t) {
    for (size_t k = k0; k < k1; ++k) {
      const Block& bl = blocks[k];
      cs_wire_block& B = w->blocks[k];
      B = cs_wire_block{};
      B.base_ts = ev[bl.begin].start_ts;
      for (uint64_t j = bl.begin; j < bl.end; ++j)
        if ((ev[j].flags & (CS_EV_HAS_BATCH | CS_EV_HAS_COMM)) == CS_EV_HAS_BATCH &&
            (ev[j].payload >> 32) == 0) {
          B.batch_base = static_cast<uint32_t>(ev[j].payload);
          break;
        }
      uint64_t c[4] = {0, 0, 0, 0};
      int64_t prev = B.base_ts;
      for (uint64_t j = bl.begin; j < bl.end; ++j) {
        const cs_event& e = ev[j];
        const uint32_t code = encode_code(e, prev, B.batch_base, dix);
        prev = e.start_ts;
        if (code == CS_WIRE_ESCAPE) {
          ++c[3];
          continue;
        }
        c[0] += is_span(e);
        c[1] += has_payload(e);
        c[2] += has_value(e);
      }
      for (int q = 0; q < 4; ++q) cnt[4 * (k + 1) + q] = c[q];
    }
  });
  for (size_t k = 0; k < nb; ++k)
    for (int q = 0; q < 4; ++q) cnt[4 * (k + 1) + q] += cnt[4 * k + q];
  w->dur_lo.resize(cnt[4 * nb + 0]);
  w->dur_hi.resize(cnt[4 * nb + 0]);
  w->payload.resize(cnt[4 * nb + 1]);
  w->values.resize(cnt[4 * nb + 2]);
  w->escapes.resize(cnt[4 * nb + 3]);

  // ---- fill
  parallel_for(nb, n_threads, [&](size_t k0, size_t k1, uint32_t) {
    for (size_t k = k0; k < k1; ++k) {
      const Block& bl = blocks[k];
      cs_wire_block& B = w->blocks[k];
      uint64_t c[4];
      for (int q = 0; q < 4; ++q) c[q] = cnt[4 * k + q];
      B.dur = c[0], B.pay = c[1], B.val = c[2], B.esc = c[3];
      int64_t prev = B.base_ts;
      for (uint64_t j = bl.begin; j < bl.end; ++j) {
        const cs_event& e = ev[j];
        const uint32_t code = encode_code(e, prev, B.batch_base, dix);
        if (code == CS_WIRE_ESCAPE) {
          w->ev[j] = CS_WIRE_ESCAPE << 24;
          w->escapes[c[3]++] = e;
          prev = e.start_ts;
          continue;
        }
        w->ev[j] = (code << 24) | static_cast<uint32_t>(e.start_ts - prev);
        prev = e.start_ts;
        if (is_span(e)) {
          w->dur_lo[c[0]] = static_cast<uint16_t>(e.duration);
          w->dur_hi[c[0]++] = static_cast<uint8_t>(e.duration >> 16);
        }
        if (has_payload(e))
          w->payload[c[1]++] = (e.flags & CS_EV_HAS_COMM) ? static_cast<uint16_t>(e.payload >> 32)
                                                          : static_cast<uint16_t>(e.payload - B.batch_base);
        if (has_value(e)) std::memcpy(&w->values[c[2]++], &e.duration, sizeof(double));
      }
    }
  });
  *out = w;
  return CS_OK;
}

int cs_wire_view(const cs_wire_trace* w, cs_wire_batch* out, uint64_t* n_blocks) {
  if (!w || !out) return CS_E_INVALID_ARGUMENT;
  *out = cs_wire_batch{};
  out->events = w->ev.data();
  out->dict = w->dict.data();
  out->n_dict = static_cast<uint32_t>(w->dict.size());
  out->blocks = w->blocks.data();
  out->dur_lo = w->dur_lo.data();
  out->dur_hi = w->dur_hi.data();
  out->n_durations = w->dur_lo.size();
  out->payloads = w->payload.data();
  out->n_payloads = w->payload.size();
  out->values = w->values.data();
  out->n_values = w->values.size();
  out->escapes = w->escapes.data();
  out->n_escapes = w->escapes.size();
  if (n_blocks) *n_blocks = w->blocks.size();
  return CS_OK;
}

void cs_wire_free(cs_wire_trace* w) { delete w; }

}  // extern "C"
