// cs_wire.cpp — host encoder for the columnar wire format (include/cyclescope_b200.h).
//
// The producer side of cs_upload_wire: per instance-aligned block of
// CS_WIRE_BLOCK events, the first start_ts becomes the block base and every
// event keeps an 8-byte header (32-bit offset + packed name/kind/category/
// flags); span durations, batch/collective payloads and counter values go
// to their own columns in event order, and anything that does not fit the
// packed fields is escaped to a full cs_event.  Two passes over the blocks
// (count per column, then fill at prefix offsets), both split across threads.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "cyclescope_b200.h"

struct cs_wire_trace {
  std::vector<cs_wire_event> ev;
  std::vector<int64_t> base;
  std::vector<uint64_t> cols;  // 3 per block
  std::vector<uint32_t> dur, payload;
  std::vector<double> values;
  std::vector<cs_event> escapes;
};

namespace {

struct Block {
  uint64_t begin, end;
};

bool is_span(const cs_event& e) { return e.kind == CS_SPAN; }
bool has_value(const cs_event& e) { return e.kind == CS_COUNTER && (e.flags & CS_EV_HAS_VALUE); }
bool has_payload(const cs_event& e) { return (e.flags & (CS_EV_HAS_BATCH | CS_EV_HAS_COMM)) != 0; }

// true when e fits the header + columns
bool fits(const cs_event& e, int64_t base) {
  if (e.start_ts < base || static_cast<uint64_t>(e.start_ts - base) > 0xffffffffull) return false;
  if (e.name_id >= 0xffffu || e.kind >= 16 || e.category >= 16 || (e.flags & ~0x3fu)) return false;
  if (is_span(e)) {
    if (e.duration < 0 || e.duration > 0xffffffffll) return false;
  } else if (!has_value(e) && e.duration != 0) {
    return false;
  }
  const bool batch = e.flags & CS_EV_HAS_BATCH, comm = e.flags & CS_EV_HAS_COMM;
  if (batch && comm) return false;
  if (comm) return (e.payload & 0xffffffffull) == 0;
  if (batch) return (e.payload >> 32) == 0;
  return e.payload == 0;
}

template <typename F>
void parallel_for(size_t n, uint32_t n_threads, F f) {
  const uint32_t nt = std::max<uint32_t>(1, std::min<size_t>(n_threads, n ? n : 1));
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (size_t k = n * t / nt; k < n * (t + 1) / nt; ++k) f(k);
    });
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
  std::vector<Block> blocks;
  for (uint32_t i = 0; i < n_inst; ++i)
    for (uint64_t b = off[i]; b < off[i + 1]; b += CS_WIRE_BLOCK)
      blocks.push_back({b, std::min<uint64_t>(b + CS_WIRE_BLOCK, off[i + 1])});
  const size_t nb = blocks.size();
  auto* w = new cs_wire_trace();
  w->ev.resize(n);
  w->base.resize(nb);
  // per block: [durations, payloads, values, escapes] counts, then prefixes
  std::vector<uint64_t> cnt(4 * (nb + 1), 0);
  parallel_for(nb, n_threads, [&](size_t k) {
    const Block& bl = blocks[k];
    const int64_t base = ev[bl.begin].start_ts;
    w->base[k] = base;
    uint64_t c[4] = {0, 0, 0, 0};
    for (uint64_t j = bl.begin; j < bl.end; ++j) {
      const cs_event& e = ev[j];
      if (!fits(e, base)) {
        ++c[3];
        continue;
      }
      c[0] += is_span(e);
      c[1] += has_payload(e);
      c[2] += has_value(e);
    }
    for (int q = 0; q < 4; ++q) cnt[4 * (k + 1) + q] = c[q];
  });
  for (size_t k = 0; k < nb; ++k)
    for (int q = 0; q < 4; ++q) cnt[4 * (k + 1) + q] += cnt[4 * k + q];
  if (cnt[4 * nb + 3] > 0xffffffffull) {
    delete w;
    return CS_E_UNSUPPORTED;
  }
  w->dur.resize(cnt[4 * nb + 0]);
  w->payload.resize(cnt[4 * nb + 1]);
  w->values.resize(cnt[4 * nb + 2]);
  w->escapes.resize(cnt[4 * nb + 3]);
  w->cols.resize(3 * nb);
  parallel_for(nb, n_threads, [&](size_t k) {
    const Block& bl = blocks[k];
    const int64_t base = w->base[k];
    uint64_t c[4];
    for (int q = 0; q < 4; ++q) c[q] = cnt[4 * k + q];
    for (int q = 0; q < 3; ++q) w->cols[3 * k + q] = c[q];
    for (uint64_t j = bl.begin; j < bl.end; ++j) {
      const cs_event& e = ev[j];
      cs_wire_event& o = w->ev[j];
      if (!fits(e, base)) {
        o.t_off = static_cast<uint32_t>(c[3]);
        o.info = CS_WIRE_ESCAPE;
        w->escapes[c[3]++] = e;
        continue;
      }
      o.t_off = static_cast<uint32_t>(e.start_ts - base);
      o.info = static_cast<uint32_t>(e.name_id) | (static_cast<uint32_t>(e.kind) << 16) |
               (static_cast<uint32_t>(e.category) << 20) | (static_cast<uint32_t>(e.flags) << 24);
      if (is_span(e)) w->dur[c[0]++] = static_cast<uint32_t>(e.duration);
      if (has_payload(e))
        w->payload[c[1]++] = (e.flags & CS_EV_HAS_COMM) ? static_cast<uint32_t>(e.payload >> 32)
                                                        : static_cast<uint32_t>(e.payload);
      if (has_value(e)) std::memcpy(&w->values[c[2]++], &e.duration, sizeof(double));
    }
  });
  *out = w;
  return CS_OK;
}

int cs_wire_view(const cs_wire_trace* w, cs_wire_batch* out, uint64_t* n_blocks) {
  if (!w || !out) return CS_E_INVALID_ARGUMENT;
  out->events = w->ev.data();
  out->block_base = w->base.data();
  out->block_cols = w->cols.data();
  out->durations = w->dur.data();
  out->n_durations = w->dur.size();
  out->payloads = w->payload.data();
  out->n_payloads = w->payload.size();
  out->values = w->values.data();
  out->n_values = w->values.size();
  out->escapes = w->escapes.data();
  out->n_escapes = w->escapes.size();
  if (n_blocks) *n_blocks = w->base.size();
  return CS_OK;
}

void cs_wire_free(cs_wire_trace* w) { delete w; }

}  // extern "C"
