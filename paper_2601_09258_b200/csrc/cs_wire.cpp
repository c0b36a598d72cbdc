// cs_wire.cpp — host encoder for the 16-byte wire format (include/cyclescope_b200.h).
//
// The producer side of cs_upload_wire: per instance-aligned block of
// CS_WIRE_BLOCK events, the first start_ts becomes the block base and every
// record keeps a 32-bit offset from it; counter values move to a side array
// and anything that does not fit the packed fields is escaped to a full
// cs_event.  Two passes over the blocks (count, then fill at prefix offsets),
// both split across threads.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "cyclescope_b200.h"

struct cs_wire_trace {
  std::vector<cs_wire_event> ev;
  std::vector<int64_t> base;
  std::vector<double> values;
  std::vector<cs_event> escapes;
};

namespace {

struct Block {
  uint64_t begin, end;
};

// true when e fits the packed record (flags & CS_EV_HAS_VALUE handled apart)
bool fits(const cs_event& e, int64_t base) {
  if (e.start_ts < base || static_cast<uint64_t>(e.start_ts - base) > 0xffffffffull) return false;
  if (e.name_id >= 0xffffu || e.kind >= 16 || e.category >= 16 || (e.flags & ~0x3fu)) return false;
  if (!(e.flags & CS_EV_HAS_VALUE) && (e.duration < 0 || e.duration > 0xffffffffll)) return false;
  if (e.flags & CS_EV_HAS_COMM) return (e.payload & 0xffffffffull) == 0;
  return (e.payload >> 32) == 0;
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
  auto* w = new cs_wire_trace();
  w->ev.resize(n);
  w->base.resize(blocks.size());
  std::vector<uint64_t> n_val(blocks.size() + 1, 0), n_esc(blocks.size() + 1, 0);
  parallel_for(blocks.size(), n_threads, [&](size_t k) {
    const Block& bl = blocks[k];
    const int64_t base = ev[bl.begin].start_ts;
    w->base[k] = base;
    uint64_t v = 0, x = 0;
    for (uint64_t j = bl.begin; j < bl.end; ++j) {
      if (!fits(ev[j], base)) ++x;
      else if (ev[j].flags & CS_EV_HAS_VALUE) ++v;
    }
    n_val[k + 1] = v;
    n_esc[k + 1] = x;
  });
  for (size_t k = 0; k < blocks.size(); ++k) {
    n_val[k + 1] += n_val[k];
    n_esc[k + 1] += n_esc[k];
  }
  w->values.resize(n_val.back());
  w->escapes.resize(n_esc.back());
  parallel_for(blocks.size(), n_threads, [&](size_t k) {
    const Block& bl = blocks[k];
    const int64_t base = w->base[k];
    uint64_t v = n_val[k], x = n_esc[k];
    for (uint64_t j = bl.begin; j < bl.end; ++j) {
      const cs_event& e = ev[j];
      cs_wire_event& o = w->ev[j];
      if (!fits(e, base)) {
        std::memset(&o, 0, sizeof o);
        o.flags = CS_WIRE_ESCAPE;
        o.payload = static_cast<uint32_t>(x);
        w->escapes[x++] = e;
        continue;
      }
      o.t_off = static_cast<uint32_t>(e.start_ts - base);
      if (e.flags & CS_EV_HAS_VALUE) {
        std::memcpy(&w->values[v], &e.duration, sizeof(double));
        o.dur = static_cast<uint32_t>(v++);
      } else {
        o.dur = static_cast<uint32_t>(e.duration);
      }
      o.name_id = static_cast<uint16_t>(e.name_id);
      o.kind_cat = static_cast<uint8_t>(e.kind | (e.category << 4));
      o.flags = static_cast<uint8_t>(e.flags);
      o.payload = (e.flags & CS_EV_HAS_COMM) ? static_cast<uint32_t>(e.payload >> 32)
                                             : static_cast<uint32_t>(e.payload);
    }
  });
  // value indices must fit the 32-bit dur field
  if (w->values.size() > 0xffffffffull || w->escapes.size() > 0xffffffffull) {
    delete w;
    return CS_E_UNSUPPORTED;
  }
  *out = w;
  return CS_OK;
}

int cs_wire_view(const cs_wire_trace* w, const cs_wire_event** ev, uint64_t* n_ev,
                 const int64_t** block_base, uint64_t* n_blocks, const double** values,
                 uint64_t* n_values, const cs_event** escapes, uint64_t* n_escapes) {
  if (!w) return CS_E_INVALID_ARGUMENT;
  if (ev) *ev = w->ev.data();
  if (n_ev) *n_ev = w->ev.size();
  if (block_base) *block_base = w->base.data();
  if (n_blocks) *n_blocks = w->base.size();
  if (values) *values = w->values.data();
  if (n_values) *n_values = w->values.size();
  if (escapes) *escapes = w->escapes.data();
  if (n_escapes) *n_escapes = w->escapes.size();
  return CS_OK;
}

void cs_wire_free(cs_wire_trace* w) { delete w; }

}  // extern "C"
