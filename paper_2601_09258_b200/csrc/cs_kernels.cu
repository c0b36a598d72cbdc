#include <unordered_map>
#include <type_traits>
// cs_kernels.cu — hand-written sm_100a kernels of the trace-analysis hot path.
//
// Data flow (one cs_run over a batch of instances):
//   K1s  k_scan_warp<sample>     name moments over the first 256 Ki events of each
//                                instance -> speculative anchor guess
//   K1r  k_rank                  exact-moment anchor ranking (cycles.cpp:47-110)
//   K12  k_scan_warp             ONE pass over all events, warp per tile: exact
//                                per-name moments (cycles.cpp:50-59) + tile-local
//                                compaction of the guessed anchor's occurrences
//                                (cycles.cpp:127-131)
//   K1r  k_rank(final)           winner; redo flag when the guess was wrong
//   K2   k_bounds_tile           cycle bounds scattered from each tile's anchors,
//                                lower_bound group starts (cycles.cpp:135-156)
//   K3   k_cycle_reduce_v2       thread per cycle: component durations
//                                (cycles.cpp:157-166), forward_mode / keyword
//                                stage signals (205-229), workload carrier
//                                (256-281), class occupancy beta and per-rank
//                                collective beta (rca.cpp:71-130)
//   K4   k_stage_heuristic       trailing-median heuristic for Unknown cycles
//                                only (cycles.cpp:230-250), warp selection
//   K5   k_records_*             record compaction (cycles.cpp:366-409)
//   K6   k_score_lut_flat / k_score   GBDT (compiled cell table or traversal) + PPE
//                                (gbdt.cpp:22-30, 173-184; detector.cpp:14-19)
//   K7   k_detect_*              control chart, episode ids, alert compaction
//                                (detector.cpp:91-130)
// All f64 arithmetic that must match the reference bit for bit is written with
// explicit __dadd_rn/__dmul_rn/__ddiv_rn (the reference objects contain no FMA)
// and the whole file is compiled with --fmad=false.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "cs_internal.h"

namespace csb {

// ------------------------------------------------ host launch helpers
// Device properties, occupancy and dynamic-shared-memory attributes are
// queried once per (host thread, device, kernel): a micro-batch run issues
// ~25 launches and each runtime query costs microseconds of host time.
namespace {
struct LaunchCache {
  int dev = -1, sms = 148, max_optin = 0;
  std::unordered_map<const void*, int> smem_set;                 // kernel -> dynamic smem attribute set
  std::unordered_map<unsigned long long, int> occ;               // (kernel, threads, smem) -> blocks per SM
};
LaunchCache& launch_cache() {
  thread_local std::unordered_map<int, LaunchCache> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  LaunchCache& c = per_dev[dev];
  if (c.dev != dev) {
    c.dev = dev;
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&c.max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return c;
}
int sm_count() { return launch_cache().sms; }
int smem_optin() { return launch_cache().max_optin; }
void ensure_smem(const void* fn, int bytes) {
  LaunchCache& c = launch_cache();
  auto it = c.smem_set.find(fn);
  if (it != c.smem_set.end() && it->second >= bytes) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  c.smem_set[fn] = bytes;
}
int blocks_per_sm(const void* fn, int threads, size_t smem) {
  LaunchCache& c = launch_cache();
  const unsigned long long key = (reinterpret_cast<unsigned long long>(fn) * 1000003ull) ^
                                 ((unsigned long long)threads << 40) ^ (unsigned long long)smem;
  auto it = c.occ.find(key);
  if (it != c.occ.end()) return it->second;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  c.occ[key] = per_sm;
  return per_sm;
}

// Programmatic dependent launch for the chains of small kernels a
// micro-batch issues: the next kernel is scheduled while its predecessor
// runs and waits at its top (pdl_enter) for the predecessor's completion
// and memory, so the launch gap leaves the critical path.  CS_PDL=0 turns
// it off (plain stream order).
bool pdl_allowed() {
  static const bool on = [] {
    const char* e = getenv("CS_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename... K, typename... A>
void launch_pdl(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t c = {};
  c.gridDim = grid;
  c.blockDim = block;
  c.dynamicSmemBytes = smem;
  c.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_allowed() ? 1 : 0;
  c.attrs = attr;
  c.numAttrs = 1;
  cudaLaunchKernelEx(&c, kernel, std::forward<A>(args)...);
}
}  // namespace

using u64 = unsigned long long;
using i64 = long long;

constexpr u64 kFlagAgg = 1ull << 62;
constexpr u64 kFlagPrefix = 2ull << 62;
constexpr u64 kValMask = (1ull << 62) - 1;
constexpr u64 kNone = ~0ull;

// ------------------------------------------------------------ primitives
// Top of every kernel launched by launch_pdl: release the next kernel in the
// stream (it may be scheduled now), then wait until this kernel's
// predecessor has completed and its writes are visible.  A no-op for plain
// launches.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ u64 ld_acquire(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// look-back words that carry nothing but their own value: relaxed is enough
// (no MEMBAR behind the warp's row stores, no L1 invalidation)
__device__ __forceinline__ u64 ld_relaxed(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ u64 umin64(u64 a, u64 b) { return a < b ? a : b; }
__device__ __forceinline__ uint32_t lanemask_le() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_le;" : "=r"(m));
  return m;
}

struct Ev {
  i64 start, dur;
  uint32_t name;
  uint32_t kind, cat, flags;
  u64 payload;
};

// 32-byte record as two 16-byte vector loads; streaming (evict-first) since
// every event is read exactly once per pass.
__device__ __forceinline__ Ev load_ev(const cs_event* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  int4 a = __ldg(q);
  int4 b = __ldg(q + 1);
  Ev e;
  e.start = (i64)(((u64)(uint32_t)a.y << 32) | (uint32_t)a.x);
  e.dur = (i64)(((u64)(uint32_t)a.w << 32) | (uint32_t)a.z);
  e.name = (uint32_t)b.x;
  e.kind = (uint32_t)b.y & 0xffu;
  e.cat = ((uint32_t)b.y >> 8) & 0xffu;
  e.flags = (uint32_t)b.y >> 16;
  e.payload = ((u64)(uint32_t)b.w << 32) | (uint32_t)b.z;
  return e;
}

// 128-bit accumulate of d*d (d as signed int64) into (lo, hi) with atomics.
__device__ __forceinline__ void atomic_add_u128(u64* lo, u64* hi, u64 add_lo, u64 add_hi) {
  u64 old = atomicAdd(lo, add_lo);
  u64 carry = (old + add_lo < old) ? 1ull : 0ull;
  if (add_hi + carry) atomicAdd(hi, add_hi + carry);
}
__device__ __forceinline__ void square_u128(i64 d, u64& lo, u64& hi) {
  u64 a = (u64)(d < 0 ? -d : d);
  lo = a * a;
  hi = __umul64hi(a, a);
}

// ------------------------------------------------ TMA bulk-copy pipeline
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA: global -> shared, completion reported as tx bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ Ev ev_from_smem(const cs_event* p) {
  const int4* q = reinterpret_cast<const int4*>(p);
  const int4 a = q[0];
  const int4 b = q[1];
  Ev e;
  e.start = (i64)(((u64)(uint32_t)a.y << 32) | (uint32_t)a.x);
  e.dur = (i64)(((u64)(uint32_t)a.w << 32) | (uint32_t)a.z);
  e.name = (uint32_t)b.x;
  e.kind = (uint32_t)b.y & 0xffu;
  e.cat = ((uint32_t)b.y >> 8) & 0xffu;
  e.flags = (uint32_t)b.y >> 16;
  e.payload = ((u64)(uint32_t)b.w << 32) | (uint32_t)b.z;
  return e;
}

// --------------------------------------------------- K1 / K12 helpers
constexpr uint32_t kTileBytes = kTileEvents * sizeof(cs_event);

// Per-warp staging rows for flushing per-thread moment caches.  64-bit shared
// atomics are CAS loops on sm_100a, so lanes holding the same name are grouped
// with __match_any_sync and the group leader does a plain read-modify-write
// of its row.  Rows are claimed with a 32-bit CAS; a full table spills to
// global atomics.
constexpr int kWarpNameRows = 16;
struct WarpNameRow {
  uint32_t name;  // 0xffffffff = free
  uint32_t cnt;
  u64 sum, sq_lo, sq_hi;
};

// Per-thread cache of PythonCall moments (typical traces have a handful of
// PythonCall names): no warp synchronisation on the hot loop; a miss falls
// back to global atomics.  Flushed through the warp rows at instance changes.
constexpr int kNameCache = 4;
struct NameCache {
  uint32_t name[kNameCache];
  uint32_t cnt[kNameCache];
  u64 sum[kNameCache], lo[kNameCache], hi[kNameCache];
};

__device__ __forceinline__ void cache_clear(NameCache& c) {
#pragma unroll
  for (int i = 0; i < kNameCache; ++i) {
    c.name[i] = 0xffffffffu;
    c.cnt[i] = 0;
    c.sum[i] = c.lo[i] = c.hi[i] = 0;
  }
}

__device__ __forceinline__ void cache_add(NameCache& c, NameStat* g, uint32_t name, i64 d) {
  u64 lo, hi;
  square_u128(d, lo, hi);
  int hit = -1, free_slot = -1;
#pragma unroll
  for (int i = 0; i < kNameCache; ++i) {
    if (c.name[i] == name) hit = i;
    if (c.name[i] == 0xffffffffu && free_slot < 0) free_slot = i;
  }
  if (hit < 0 && free_slot >= 0) {
    hit = free_slot;
#pragma unroll
    for (int i = 0; i < kNameCache; ++i)
      if (i == free_slot) c.name[i] = name;
  }
  if (hit < 0) {
    atomicAdd(&g[name].count, 1ull);
    atomicAdd(&g[name].sum, (u64)d);
    atomic_add_u128(&g[name].sumsq_lo, &g[name].sumsq_hi, lo, hi);
    return;
  }
#pragma unroll
  for (int i = 0; i < kNameCache; ++i) {
    if (i == hit) {
      c.cnt[i] += 1;
      c.sum[i] += (u64)d;
      const u64 nl = c.lo[i] + lo;
      c.hi[i] += hi + (nl < c.lo[i] ? 1ull : 0ull);
      c.lo[i] = nl;
    }
  }
}

// warp-wide: fold (name, cnt, sum, lo, hi) contributions into the warp's rows
__device__ __forceinline__ void rows_merge(WarpNameRow* wrows, NameStat* g, bool valid,
                                           uint32_t name, uint32_t cnt, u64 sum, u64 lo, u64 hi) {
  __syncwarp();
  const uint32_t key = valid ? name : 0xffffffffu;
  const uint32_t grp = __match_any_sync(0xffffffffu, key);
  if (!valid) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(grp) - 1;
  uint32_t rest = grp & ~(1u << leader);
  while (rest) {
    const int src = __ffs(rest) - 1;
    rest &= rest - 1;
    const uint32_t oc = __shfl_sync(grp, cnt, src);
    const u64 os = __shfl_sync(grp, sum, src);
    const u64 ol = __shfl_sync(grp, lo, src);
    const u64 oh = __shfl_sync(grp, hi, src);
    if (lane == leader) {
      cnt += oc;
      sum += os;
      const u64 nl = lo + ol;
      hi += oh + (nl < lo ? 1ull : 0ull);
      lo = nl;
    }
  }
  if (lane != leader) return;
  int row = -1;
  for (int i = 0; i < kWarpNameRows; ++i) {
    const uint32_t n = wrows[i].name;
    if (n == name) { row = i; break; }
    if (n == 0xffffffffu) {
      const uint32_t old = atomicCAS(&wrows[i].name, 0xffffffffu, name);
      if (old == 0xffffffffu || old == name) { row = i; break; }
    }
  }
  if (row < 0) {
    atomicAdd(&g[name].count, (u64)cnt);
    atomicAdd(&g[name].sum, sum);
    atomic_add_u128(&g[name].sumsq_lo, &g[name].sumsq_hi, lo, hi);
    return;
  }
  WarpNameRow& r = wrows[row];
  r.cnt += cnt;
  r.sum += sum;
  const u64 nl = r.sq_lo + lo;
  r.sq_hi += hi + (nl < r.sq_lo ? 1ull : 0ull);
  r.sq_lo = nl;
}

// whole CTA (converged): per-thread caches -> warp rows -> warp 0's rows ->
// a few global atomics per name and CTA.  Called once per instance switch.
__device__ void cache_flush(NameCache& c, NameStat* g, WarpNameRow* rows) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x / 32;
  for (int i = threadIdx.x; i < nw * kWarpNameRows; i += blockDim.x) {
    rows[i].name = 0xffffffffu;
    rows[i].cnt = 0;
    rows[i].sum = rows[i].sq_lo = rows[i].sq_hi = 0;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kNameCache; ++i)
    rows_merge(rows + warp * kWarpNameRows, g, c.name[i] != 0xffffffffu && c.cnt[i] > 0,
               c.name[i], c.cnt[i], c.sum[i], c.lo[i], c.hi[i]);
  __syncthreads();
  if (warp == 0) {
    for (int w = 1; w < nw; ++w) {
      const WarpNameRow r = rows[w * kWarpNameRows + (lane & (kWarpNameRows - 1))];
      const bool v = lane < kWarpNameRows && r.name != 0xffffffffu && r.cnt > 0;
      rows_merge(rows, g, v, r.name, r.cnt, r.sum, r.sq_lo, r.sq_hi);
    }
    __syncwarp();
    if (lane < kWarpNameRows) {
      const WarpNameRow r = rows[lane];
      if (r.name != 0xffffffffu && r.cnt) {
        atomicAdd(&g[r.name].count, (u64)r.cnt);
        atomicAdd(&g[r.name].sum, r.sum);
        atomic_add_u128(&g[r.name].sumsq_lo, &g[r.name].sumsq_hi, r.sq_lo, r.sq_hi);
      }
    }
  }
  __syncthreads();
  cache_clear(c);
}

// consumer-group version of cache_flush (no CTA-wide barrier): per-thread
// caches -> the warp's rows -> global atomics
__device__ void cache_flush_warp(NameCache& c, NameStat* g, WarpNameRow* wrows) {
  const int lane = threadIdx.x & 31;
  if (lane < kWarpNameRows) {
    wrows[lane].name = 0xffffffffu;
    wrows[lane].cnt = 0;
    wrows[lane].sum = wrows[lane].sq_lo = wrows[lane].sq_hi = 0;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kNameCache; ++i)
    rows_merge(wrows, g, c.name[i] != 0xffffffffu && c.cnt[i] > 0, c.name[i], c.cnt[i], c.sum[i],
               c.lo[i], c.hi[i]);
  __syncwarp();
  if (lane < kWarpNameRows) {
    const WarpNameRow r = wrows[lane];
    if (r.name != 0xffffffffu && r.cnt) {
      atomicAdd(&g[r.name].count, (u64)r.cnt);
      atomicAdd(&g[r.name].sum, r.sum);
      atomic_add_u128(&g[r.name].sumsq_lo, &g[r.name].sumsq_hi, r.sq_lo, r.sq_hi);
    }
  }
  __syncwarp();
  cache_clear(c);
}

// Shared-memory variant of NameCache for kernels short of registers: lane
// columns [entry][32] of one warp's block; same semantics as NameCache.
struct SNameCache {
  uint32_t* name;  // [kNameCache][32]
  uint32_t* cnt;
  u64 *sum, *lo, *hi;
  int lane;
  __device__ static SNameCache at(void* base, int lane) {
    SNameCache c;
    c.sum = reinterpret_cast<u64*>(base);
    c.lo = c.sum + kNameCache * 32;
    c.hi = c.lo + kNameCache * 32;
    c.name = reinterpret_cast<uint32_t*>(c.hi + kNameCache * 32);
    c.cnt = c.name + kNameCache * 32;
    c.lane = lane;
    return c;
  }
  static constexpr int kBytes = kNameCache * 32 * (3 * 8 + 2 * 4);
};

__device__ __forceinline__ void cache_clear(SNameCache& c) {
#pragma unroll
  for (int i = 0; i < kNameCache; ++i) {
    c.name[i * 32 + c.lane] = 0xffffffffu;
    c.cnt[i * 32 + c.lane] = 0;
    c.sum[i * 32 + c.lane] = c.lo[i * 32 + c.lane] = c.hi[i * 32 + c.lane] = 0;
  }
}

__device__ __forceinline__ void cache_add(SNameCache& c, NameStat* g, uint32_t name, i64 d) {
  u64 lo, hi;
  square_u128(d, lo, hi);
  int hit = -1, free_slot = -1;
#pragma unroll
  for (int i = 0; i < kNameCache; ++i) {
    const uint32_t n = c.name[i * 32 + c.lane];
    if (n == name && hit < 0) hit = i;
    if (n == 0xffffffffu && free_slot < 0) free_slot = i;
  }
  if (hit < 0 && free_slot >= 0) {
    hit = free_slot;
    c.name[hit * 32 + c.lane] = name;
  }
  if (hit < 0) {
    atomicAdd(&g[name].count, 1ull);
    atomicAdd(&g[name].sum, (u64)d);
    atomic_add_u128(&g[name].sumsq_lo, &g[name].sumsq_hi, lo, hi);
    return;
  }
  const int k = hit * 32 + c.lane;
  c.cnt[k] += 1;
  c.sum[k] += (u64)d;
  const u64 ol = c.lo[k], nl = ol + lo;
  c.hi[k] += hi + (nl < ol ? 1ull : 0ull);
  c.lo[k] = nl;
}

// flush one warp's per-lane caches name by name: the smallest unflushed name
// of the warp, every lane's entry for it summed by butterflies (exact u128),
// one set of global atomics per name (a handful of names per instance)
__device__ void cache_flush_warp(SNameCache& c, NameStat* g, WarpNameRow*) {
  const int lane = c.lane;
  __syncwarp();
  for (;;) {
    uint32_t mine = 0xffffffffu;
#pragma unroll
    for (int i = 0; i < kNameCache; ++i) {
      const int k = i * 32 + lane;
      if (c.cnt[k] && c.name[k] < mine) mine = c.name[k];
    }
    const uint32_t nm = __reduce_min_sync(0xffffffffu, mine);
    if (nm == 0xffffffffu) break;
    uint32_t cnt = 0;
    u64 sum = 0, lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < kNameCache; ++i) {
      const int k = i * 32 + lane;
      if (c.cnt[k] && c.name[k] == nm) {
        cnt = c.cnt[k];
        sum = c.sum[k];
        lo = c.lo[k];
        hi = c.hi[k];
        c.cnt[k] = 0;
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const u64 ol = __shfl_xor_sync(0xffffffffu, lo, o), oh = __shfl_xor_sync(0xffffffffu, hi, o);
      const u64 nl = lo + ol;
      hi += oh + (nl < lo ? 1ull : 0ull);
      lo = nl;
    }
    if (lane == 0) {
      atomicAdd(&g[nm].count, (u64)cnt);
      atomicAdd(&g[nm].sum, sum);
      atomic_add_u128(&g[nm].sumsq_lo, &g[nm].sumsq_hi, lo, hi);
    }
  }
  __syncwarp();
  cache_clear(c);
  __syncwarp();
}

// --------------------------------------- K1 / K12 event scan (warp streaming)
// One warp per tile (instance-aligned, <= kTileEvents events), warps
// persistent over tiles with a static schedule.  The warp streams its tile
// with coalesced 256-bit loads (one 32-B record per lane per load, kScanUnroll
// records per lane in flight), folds PythonCall moments into a per-thread name
// cache (cycles.cpp:50-59; exact integer sums, so order-free) and compacts
// the tile's anchor occurrences (Spans named the guessed/final anchor,
// cycles.cpp:127-131) warp-locally to a_*[tile_begin + rank] with the
// tile's count in tile_cnt[t].  No shared-memory staging, no CTA barriers.
constexpr int kScanWarpThreads = 256;
constexpr u64 kWalk = 1ull << 63;  // a_pos flag: the group start needs a walk back
constexpr int kScanUnroll = 4;
constexpr uint32_t kSampleSplit = 4;  // sub-ranges per tile in the sample pass

struct Ev8 {
  u64 a, b, c, d;  // start, duration, (name | kind/cat/flags << 32), payload
};
__device__ __forceinline__ Ev8 ldg256(const cs_event* p) {
  Ev8 e;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(e.a), "=l"(e.b), "=l"(e.c), "=l"(e.d)
               : "l"(p));
  return e;
}

__global__ void __launch_bounds__(kScanWarpThreads, 3)
    k_scan_warp(DevBuffers b, int mode, const uint32_t* __restrict__ list, uint32_t n_list,
                int sample) {
  pdl_enter();
  constexpr int kW = kScanWarpThreads / 32;
  __shared__ WarpNameRow s_rows[kW * kWarpNameRows];
  // PythonCall spans are ~1 event in 9: they are compacted per warp and
  // folded into the per-thread name caches 32 at a time, so the cache update
  // runs once per PythonCall span instead of predicated on every lane
  __shared__ uint32_t s_pn[kW][64];
  __shared__ i64 s_pd[kW][64];
  const bool do_stats = mode & 1;
  const bool do_anchor = (mode & 2) && !sample;
  const bool redo = mode & 4;
  const bool check = do_anchor && !redo;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpNameRow* wrows = s_rows + warp * kWarpNameRows;
  uint32_t* pn = s_pn[warp];
  i64* pd = s_pd[warp];
  const uint32_t gw = blockIdx.x * kW + warp;
  const uint32_t nw = gridDim.x * kW;
  NameCache cache;
  cache_clear(cache);
  uint32_t cur_inst = 0xffffffffu, npend = 0;
  NameStat* gstats = b.stats;
  auto drain = [&](uint32_t take) {  // fold entries [0, take) and shift the rest down
    __syncwarp();
    if ((uint32_t)lane < take) cache_add(cache, gstats, pn[lane], pd[lane]);
    __syncwarp();
    const uint32_t rest = npend - take;
    uint32_t mv_n = 0;
    i64 mv_d = 0;
    if ((uint32_t)lane < rest) {
      mv_n = pn[take + lane];
      mv_d = pd[take + lane];
    }
    __syncwarp();
    if ((uint32_t)lane < rest) {
      pn[lane] = mv_n;
      pd[lane] = mv_d;
    }
    npend = rest;
    __syncwarp();
  };
  // Many-instance batches: each warp takes a contiguous run of tiles, which
  // mostly belong to one instance, so its name-moment cache is flushed once
  // per instance it meets instead of on every tile.  One instance: tiles
  // strided across warps (all warps stream neighbouring tiles).
  const bool runs = b.n_inst > 1;
  const uint32_t per_warp = runs ? (n_list + nw - 1) / nw : 0u;
  const uint32_t k0 = runs ? gw * per_warp : gw;
  const uint32_t k_end = runs ? ((gw + 1) * per_warp < n_list ? (gw + 1) * per_warp : n_list) : n_list;
  const uint32_t k_step = runs ? 1u : nw;
  for (uint32_t k = k0; k < k_end; k += k_step) {
    // the sample pass splits each tile into kSampleSplit sub-ranges (moments
    // only, order-free), so its few tiles still spread over the whole GPU
    const uint32_t t = sample ? list[k / kSampleSplit] : (list ? list[k] : k);
    const uint32_t inst = b.tile_inst[t];
    u64 tb = b.tile_begin[t];
    u64 te = b.tile_end[t];
    if (sample) {
      const u64 lim = b.inst_off[inst] + kSampleEvents;
      te = te < lim ? te : lim;
      const u64 sub = (u64)(k % kSampleSplit) * (kTileEvents / kSampleSplit);
      const u64 sb = tb + sub, se = sb + kTileEvents / kSampleSplit;
      tb = sb;
      te = te < se ? te : se;
      if (te < tb) te = tb;
    }
    bool active = do_anchor;
    uint32_t anchor = 0xffffffffu;
    if (do_anchor) {
      const InstState& st = b.inst[inst];
      anchor = redo ? st.anchor : st.guess;
      if (redo && !st.redo) active = false;
    }
    if (do_stats && inst != cur_inst) {
      if (cur_inst != 0xffffffffu) {
        drain(npend);
        cache_flush_warp(cache, gstats, wrows);
      }
      cur_inst = inst;
      gstats = b.stats + (u64)inst * b.n_names;
    }
    const uint32_t n = (uint32_t)(te - tb);
    uint32_t cnt = 0;
    // K0 check (trace.cpp:103-109 is_sorted): start_ts never decreases within
    // the tile; k_tile_order checks the tile boundaries (no dependent load per tile)
    i64 carry_ts = LLONG_MIN;
    bool unsorted = false;
    for (uint32_t j0 = 0; j0 < n; j0 += 32 * kScanUnroll) {
      Ev8 e[kScanUnroll];
#pragma unroll
      for (int q = 0; q < kScanUnroll; ++q) {
        const uint32_t j = j0 + q * 32 + lane;
        if (j < n) e[q] = ldg256(b.ev + tb + j);
        else {
          e[q].a = ~0ull >> 1;  // INT64_MAX: never below its predecessor
          e[q].c = (u64)CS_FLOW << 32;  // ignored
        }
      }
#pragma unroll
      for (int q = 0; q < kScanUnroll; ++q) {
        const uint32_t name = (uint32_t)e[q].c;
        const uint32_t kc = (uint32_t)(e[q].c >> 32);
        const bool span = (kc & 0xffu) == CS_SPAN;
        if (do_stats) {
          const bool py = span && ((kc >> 8) & 0xffu) == CS_CAT_PYTHON_CALL;
          const uint32_t pm = __ballot_sync(0xffffffffu, py);
          if (py) {
            const uint32_t slot = npend + __popc(pm & lanemask_lt());
            pn[slot] = name;
            pd[slot] = (i64)e[q].b;
          }
          npend += __popc(pm);
          if (npend >= 32) drain(32);
        }
        const bool is_anchor = active && span && name == anchor;
        const uint32_t mk = __ballot_sync(0xffffffffu, is_anchor);
        // group start (lower_bound over equal start_ts, cycles.cpp:137-144):
        // the anchor opens its group unless the previous record shares its
        // start; kWalk marks the rare anchors k_bounds_tile must walk back for
        const u64 prev = __shfl_up_sync(0xffffffffu, e[q].a, 1);
        if (check) {
          const i64 before = lane == 0 ? carry_ts : (i64)prev;
          unsorted |= before > (i64)e[q].a;
          carry_ts = (i64)__shfl_sync(0xffffffffu, e[q].a, 31);
        }
        if (is_anchor) {
          const u64 r = tb + cnt + __popc(mk & lanemask_lt());
          const uint32_t jj = j0 + q * 32 + lane;
          const bool walk = jj == 0 ? tb > b.inst_off[inst] : (lane == 0 || prev == e[q].a);
          b.a_pos[r] = (tb + jj) | (walk ? kWalk : 0ull);
          b.a_start[r] = (i64)e[q].a;
          b.a_end[r] = (i64)e[q].a + (i64)e[q].b;
        }
        cnt += __popc(mk);
      }
    }
    if (active && lane == 0) b.tile_cnt[t] = cnt;
    if (check && __any_sync(0xffffffffu, unsorted) && lane == 0) atomicOr(&b.inst[inst].unsorted, 1u);
  }
  if (do_stats && cur_inst != 0xffffffffu) {
    drain(npend);
    cache_flush_warp(cache, gstats, wrows);
  }
}


// per-instance anchor counts from the tile prefix
__global__ void k_inst_anchor_counts(DevBuffers b) {
  pdl_enter();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n_inst) return;
  const uint32_t t0 = b.inst_first_tile[i];
  const uint32_t t1 = i + 1 < b.n_inst ? b.inst_first_tile[i + 1] : b.n_tiles;
  b.inst[i].n_anchors = b.tile_pref[t1] - b.tile_pref[t0];
}

// ------------------------------------------------------------ K1r rank
// One warp per instance.  score = count / (1 + cv) computed from exact
// moments; an interval bound on the reference's sequentially rounded
// sum_sq (|err| <= n*u*sum_sq) certifies the winner, otherwise the host runs
// the ordered fold (k_fold).  Ties break by name (name id == lex rank).
struct Cand {
  double score, lo, hi;
  uint32_t name;
};

__device__ __forceinline__ double u128_to_double(u64 lo, u64 hi) {
  return __dadd_rn(__dmul_rn((double)hi, 18446744073709551616.0), (double)lo);
}

__device__ void score_from_moments(u64 count, i64 sum, double sumsq, double& mean, double& cv,
                                   double& score) {
  const double n = (double)count;
  mean = __ddiv_rn((double)sum, n);
  cv = 0.0;
  if (mean > 0.0) {
    double var = __dsub_rn(__ddiv_rn(sumsq, n), __dmul_rn(mean, mean));
    var = 0.0 < var ? var : 0.0;
    cv = __ddiv_rn(sqrt(var), mean);
  }
  score = __ddiv_rn(n, __dadd_rn(1.0, cv));
}

__global__ void k_rank(DevBuffers b, DevConfig cfg, int final_pass) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const uint32_t inst = blockIdx.x;
  if (inst >= b.n_inst) return;
  InstState& st = b.inst[inst];
  const NameStat* gs = b.stats + (u64)inst * b.n_names;
  const u64 min_calls = cfg.cyc.min_anchor_calls;
  const i64 hint = cfg.cyc.anchor_hint_name;

  Cand best{-1.0, 0, 0, 0xffffffffu};
  uint32_t ncand = 0;
  bool inexact = false;
  for (uint32_t n = lane; n < b.n_names; n += 32) {
    const NameStat s = gs[n];
    if (s.count < min_calls || s.count == 0) continue;
    ++ncand;
    const i64 sum = (i64)s.sum;
    const bool sum_exact = (sum < (1ll << 53)) && (sum > -(1ll << 53));
    const double S = u128_to_double(s.sumsq_lo, s.sumsq_hi);
    const double u = 1.1102230246251565e-16;
    const double gamma = (double)(s.count + 2) * u;
    double m, cv, sc, sc_lo, sc_hi;
    score_from_moments(s.count, sum, S, m, cv, sc);
    {
      double m2, cv2;
      // larger sum_sq -> larger var -> smaller score
      score_from_moments(s.count, sum, S * (1.0 + gamma), m2, cv2, sc_lo);
      score_from_moments(s.count, sum, S * (1.0 - gamma), m2, cv2, sc_hi);
      // cancellation guard on var = E[d^2] - mean^2: absolute slack
      const double mean2 = m * m;
      const double slack = 8.0 * u * (S / (double)s.count + mean2);
      if (m > 0.0) {
        const double n = (double)s.count;
        const double vlo = fmax(0.0, S * (1.0 - gamma) / n - mean2 - slack);
        const double vhi = fmax(0.0, S * (1.0 + gamma) / n - mean2 + slack);
        sc_hi = fmax(sc_hi, n / (1.0 + sqrt(vlo) / m));
        sc_lo = fmin(sc_lo, n / (1.0 + sqrt(vhi) / m));
      }
      sc_lo *= (1.0 - 16 * u);
      sc_hi *= (1.0 + 16 * u);
    }
    if (!sum_exact) inexact = true;
    if (sc > best.score || (sc == best.score && n < best.name)) best = Cand{sc, sc_lo, sc_hi, n};
  }
  // warp argmax (score desc, name asc)
  for (int o = 16; o > 0; o >>= 1) {
    Cand c;
    c.score = __shfl_xor_sync(0xffffffffu, best.score, o);
    c.lo = __shfl_xor_sync(0xffffffffu, best.lo, o);
    c.hi = __shfl_xor_sync(0xffffffffu, best.hi, o);
    c.name = __shfl_xor_sync(0xffffffffu, best.name, o);
    if (c.score > best.score || (c.score == best.score && c.name < best.name)) best = c;
  }
  for (int o = 16; o > 0; o >>= 1) ncand += __shfl_xor_sync(0xffffffffu, ncand, o);
  inexact = __any_sync(0xffffffffu, inexact);
  // ambiguity: any other candidate whose interval reaches the winner's
  bool amb = false;
  if (best.name != 0xffffffffu) {
    for (uint32_t n = lane; n < b.n_names; n += 32) {
      if (n == best.name) continue;
      const NameStat s = gs[n];
      if (s.count < min_calls || s.count == 0) continue;
      const i64 sum = (i64)s.sum;
      const double S = u128_to_double(s.sumsq_lo, s.sumsq_hi);
      const double u = 1.1102230246251565e-16;
      const double gamma = (double)(s.count + 2) * u;
      double m, cv, sc_hi;
      score_from_moments(s.count, sum, S * (1.0 - gamma), m, cv, sc_hi);
      if (m > 0.0) {
        const double nd = (double)s.count;
        const double slack = 8.0 * u * (S / nd + m * m);
        const double vlo = fmax(0.0, S * (1.0 - gamma) / nd - m * m - slack);
        sc_hi = fmax(sc_hi, nd / (1.0 + sqrt(vlo) / m));
      }
      sc_hi *= (1.0 + 16 * u);
      if (sc_hi >= best.lo) amb = true;
    }
  }
  amb = __any_sync(0xffffffffu, amb) || inexact;

  if (lane == 0) {
    uint32_t winner = best.name;
    if (hint >= 0 || st.fixed_anchor) {
      // discover_anchor with a hint (cycles.cpp:90-104): the hint wins when it
      // occurs as any Span at all.  A stream keeps the anchor its first
      // micro-batch chose (fixed_anchor) the same way.
      const uint32_t h = st.fixed_anchor ? st.guess : (uint32_t)hint;
      winner = st.n_anchors > 0 ? h : 0xffffffffu;
      amb = false;
    } else if (hint == -2) {
      winner = 0xffffffffu;
      amb = false;
    }
    if (!final_pass) {
      st.guess = winner;
    } else {
      st.anchor = winner;
      st.ambiguous = amb ? 1u : 0u;
      st.no_anchor = winner == 0xffffffffu ? 1u : 0u;
      st.redo = (winner != 0xffffffffu && winner != st.guess) ? 1u : 0u;
      st.n_candidates = ncand;
    }
  }
}

// Ordered fold: the reference's own sequential arithmetic for one
// (instance, name) -- count, sum += d, sum_sq += d*d in event order
// (cycles.cpp:50-59) and the start gaps of gap_cv (30-43) -- then
// mean/cv/score/periodicity (66-77).  One warp per pair: the warp reads 32
// records per step (coalesced), and every lane folds the matching spans in
// lane order with the same sequential f64 operations (the values are
// warp-uniform, so no reduction tree ever reorders a sum).  Launched when
// k_rank cannot certify the winner and for cs_get_candidates_exact.
constexpr int kFoldUnroll = 4;
__global__ void __launch_bounds__(128) k_fold(DevBuffers b, const uint32_t* pairs_inst,
                                              const uint32_t* pairs_name, uint32_t n_pairs,
                                              double* out) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n_pairs) return;
  const uint32_t inst = pairs_inst[p], name = pairs_name[p];
  const u64 e0 = b.inst_off[inst], e1 = b.inst_off[inst + 1];
  u64 count = 0;
  double sum = 0.0, sum_sq = 0.0, gsum = 0.0, gsq = 0.0;
  i64 prev = 0;
  for (u64 j0 = e0; j0 < e1; j0 += 32 * kFoldUnroll) {
    Ev8 e[kFoldUnroll];
#pragma unroll
    for (int q = 0; q < kFoldUnroll; ++q) {
      const u64 j = j0 + q * 32 + lane;
      if (j < e1) e[q] = ldg256(b.ev + j);
      else e[q].c = (u64)CS_FLOW << 32;
    }
#pragma unroll
    for (int q = 0; q < kFoldUnroll; ++q) {
      const uint32_t kc = (uint32_t)(e[q].c >> 32);
      const bool m = (kc & 0xffu) == CS_SPAN && ((kc >> 8) & 0xffu) == CS_CAT_PYTHON_CALL &&
                     (uint32_t)e[q].c == name;
      uint32_t mask = __ballot_sync(0xffffffffu, m);
      while (mask) {
        const int l = __ffs(mask) - 1;
        mask &= mask - 1;
        const i64 st = (i64)__shfl_sync(0xffffffffu, e[q].a, l);
        const double d = (double)(i64)__shfl_sync(0xffffffffu, e[q].b, l);
        if (count > 0) {
          const double gap = (double)(st - prev);
          gsum = __dadd_rn(gsum, gap);
          gsq = __dadd_rn(gsq, __dmul_rn(gap, gap));
        }
        prev = st;
        ++count;
        sum = __dadd_rn(sum, d);
        sum_sq = __dadd_rn(sum_sq, __dmul_rn(d, d));
      }
    }
  }
  if (lane != 0) return;
  const double n = (double)count;
  const double mean = __ddiv_rn(sum, n);
  double cv = 0.0;
  if (mean > 0.0) {
    double var = __dsub_rn(__ddiv_rn(sum_sq, n), __dmul_rn(mean, mean));
    var = 0.0 < var ? var : 0.0;
    cv = __ddiv_rn(sqrt(var), mean);
  }
  double gcv = 0.0;  // gap_cv (cycles.cpp:30-43)
  if (count >= 3) {
    const double ng = (double)(count - 1);
    const double gm = __ddiv_rn(gsum, ng);
    if (gm > 0.0) {
      double var = __dsub_rn(__ddiv_rn(gsq, ng), __dmul_rn(gm, gm));
      var = 0.0 < var ? var : 0.0;
      gcv = __ddiv_rn(sqrt(var), gm);
    }
  }
  out[4 * p + 0] = mean;
  out[4 * p + 1] = cv;
  out[4 * p + 2] = __ddiv_rn(n, __dadd_rn(1.0, cv));
  out[4 * p + 3] = __ddiv_rn(1.0, __dadd_rn(1.0, gcv));
}

// ------------------------------------------------------------ K2 bounds
__device__ __forceinline__ uint32_t upper_bound_u64(const uint64_t* a, uint32_t n, u64 v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// lower_bound(events, ts) restricted to the instance, starting from a known
// position with start_ts == ts (cycles.cpp:137-144): walk back over equal keys.
__device__ __forceinline__ u64 group_start(const cs_event* ev, u64 pos, u64 begin, i64 ts) {
  while (pos > begin && ev[pos - 1].start_ts == ts) --pos;
  return pos;
}

// anchor k of an instance -> slot in the tile-local anchor arrays
__device__ __forceinline__ u64 anchor_slot(const DevBuffers& b, uint32_t inst, u64 k) {
  const uint32_t t0 = b.inst_first_tile[inst];
  const uint32_t t1 = inst + 1 < b.n_inst ? b.inst_first_tile[inst + 1] : b.n_tiles;
  const u64 g = b.tile_pref[t0] + k;
  uint32_t lo = t0, hi = t1;  // last t with tile_pref[t] <= g
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (b.tile_pref[mid] <= g) lo = mid;
    else hi = mid;
  }
  return b.tile_begin[lo] + (g - b.tile_pref[lo]);
}

// Cycle bounds by scatter from each tile's anchor list (warp per tile): the
// anchor of global rank r opens cycle r - base(inst) and closes the previous
// one; first/last events by lower_bound over equal start_ts
// (cycles.cpp:135-156).  Replaces a binary search per cycle.
__global__ void __launch_bounds__(256) k_bounds_tile(DevBuffers b) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const u64 t = (u64)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= b.n_tiles) return;
  const uint32_t inst = b.tile_inst[t];
  if (b.inst[inst].no_anchor) return;  // frequency-fallback cycles: k_freq_cycles
  const u64 cnt = b.tile_cnt[t];
  const u64 base = b.tile_pref[b.inst_first_tile[inst]];
  const u64 ib = b.inst_off[inst];
  const u64 c0 = b.cyc_off[inst], c1 = b.cyc_off[inst + 1];
  const u64 tb = b.tile_begin[t];
  for (u64 r = lane; r < cnt; r += 32) {
    const u64 rank = b.tile_pref[t] + r - base;  // anchor index within the instance
    const u64 s = tb + r;
    const i64 a = b.a_start[s];
    const u64 pw = b.a_pos[s];
    const u64 p = pw & ~kWalk;
    const u64 f = (pw & kWalk) ? group_start(b.ev, p, ib, a) : p;
    const u64 g = c0 + rank;
    if (g < c1) {  // opens cycle `rank`
      b.c_start[g] = a;
      b.c_apos[g] = p;
      b.c_aend[g] = b.a_end[s];
      b.c_first[g] = f;
      b.c_inst[g] = inst;
    }
    if (rank > 0 && g - 1 < c1) {  // closes cycle rank - 1
      b.c_end[g - 1] = a;
      b.c_last[g - 1] = f;
    }
  }
}

// ------------------------------------------------------------ K5 records
// record := cycle with (include_prefill || stage != Prefill) && workload ok
// (cycles.cpp:372-383).  Global compaction in cycle order; instance i's
// records are contiguous and start at rec_off[i].
constexpr int kRecBlock = 1024;

// cycle g yields a record (cycles.cpp:372-383); the instance-relative index
// test (monitor_from_cycle, streaming offsets) only loads the instance when
// it can matter
// the cycle's loads are issued together (no short-circuit between them)
__device__ __forceinline__ bool rec_ok(const DevBuffers& b, const DevConfig& cfg, u64 g, bool need_index) {
  const int32_t wl = b.c_wl[g];
  const uint8_t stage = b.c_stage[g];
  const uint32_t inst = need_index ? b.c_inst[g] : 0u;
  const bool ok = wl >= 0 && (cfg.cyc.include_prefill || stage != CS_STAGE_PREFILL);
  if (!need_index) return ok;
  return ok && g - b.cyc_off[inst] + (b.stream ? b.stream[inst].cycle_off : 0) >= (u64)cfg.cyc.monitor_from_cycle;
}

// kRecBlock cycles per CTA of kRecThreads, kRecBlock / kRecThreads per thread
// (thread stride: coalesced), independent loads in flight
#ifndef CS_REC_THREADS
#define CS_REC_THREADS 256
#endif
constexpr int kRecThreads = CS_REC_THREADS;
constexpr int kRecPer = kRecBlock / kRecThreads;

__global__ void __launch_bounds__(kRecThreads) k_records_count(DevBuffers b, DevConfig cfg) {
  pdl_enter();
  __shared__ uint32_t s_w[kRecThreads / 32];
  const bool need_index = cfg.cyc.monitor_from_cycle > 0 || b.stream;
  const u64 g0 = (u64)blockIdx.x * kRecBlock + threadIdx.x;
  uint32_t n = 0;
#pragma unroll
  for (int r = 0; r < kRecPer; ++r) {
    const u64 g = g0 + (u64)r * kRecThreads;
    n += (g < b.n_cycles && rec_ok(b, cfg, g, need_index)) ? 1u : 0u;
  }
  n = (uint32_t)warp_sum_u64(n);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 t = 0;
    for (int w = 0; w < kRecThreads / 32; ++w) t += s_w[w];
    b.block_tmp[blockIdx.x] = t;
  }
}

// single-CTA exclusive scan of n u64 values in place; total to *total.  One
// round: thread t owns the contiguous chunk [t*c, (t+1)*c), c = ceil(n/threads)
// (independent loads, no per-round barriers).
__global__ void __launch_bounds__(1024, 1) k_scan_exclusive(uint64_t* v, uint64_t n, uint64_t* total) {
  pdl_enter();
  __shared__ u64 s_part[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 c = (n + blockDim.x - 1) / blockDim.x;
  const u64 i0 = (u64)threadIdx.x * c;
  const u64 i1 = min(i0 + c, (u64)n);
  u64 sum = 0;
  for (u64 i = i0; i < i1; ++i) sum += v[i];
  u64 incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_part[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    u64 p = lane < (int)(blockDim.x / 32) ? s_part[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const u64 y = __shfl_up_sync(0xffffffffu, p, o);
      if (lane >= o) p += y;
    }
    s_part[lane] = p;
  }
  __syncthreads();
  u64 run = (warp ? s_part[warp - 1] : 0) + incl - sum;
  for (u64 i = i0; i < i1; ++i) {
    const u64 x = v[i];
    v[i] = run;
    run += x;
  }
  if (threadIdx.x == 0 && total) *total = s_part[blockDim.x / 32 - 1];
}

// Multi-CTA exclusive scan for large arrays (tile prefixes: ~1e5 entries):
// k_scan_totals writes each 1024-element block's sum, k_scan_exclusive scans
// the (few) block sums, k_scan_apply scans within each block and adds its
// block's prefix.  Coalesced, one element per thread.
constexpr int kScanBlk = 1024;
__device__ __forceinline__ u64 block_incl_scan(u64 x, u64* s_w, u64* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u64 incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    u64 p = lane < (int)(blockDim.x / 32) ? s_w[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const u64 y = __shfl_up_sync(0xffffffffu, p, o);
      if (lane >= o) p += y;
    }
    s_w[lane] = p;
  }
  __syncthreads();
  if (total) *total = s_w[blockDim.x / 32 - 1];
  return incl + (warp ? s_w[warp - 1] : 0);
}
__global__ void __launch_bounds__(kScanBlk) k_scan_totals(const uint64_t* v, uint64_t n, uint64_t* part) {
  pdl_enter();
  __shared__ u64 s_w[32];
  const u64 i = (u64)blockIdx.x * kScanBlk + threadIdx.x;
  u64 t;
  block_incl_scan(i < n ? v[i] : 0, s_w, &t);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}
__global__ void __launch_bounds__(kScanBlk) k_scan_apply(uint64_t* v, uint64_t n, const uint64_t* part) {
  pdl_enter();
  __shared__ u64 s_w[32];
  const u64 i = (u64)blockIdx.x * kScanBlk + threadIdx.x;
  const u64 x = i < n ? v[i] : 0;
  const u64 incl = block_incl_scan(x, s_w, nullptr);
  if (i < n) v[i] = part[blockIdx.x] + incl - x;
}

void launch_exclusive_scan(uint64_t* v, uint64_t n, uint64_t* total, uint64_t* tmp, cudaStream_t s,
                           uint64_t* launches) {
  if (n <= 16 * kScanBlk || !tmp) {
    launch_pdl(k_scan_exclusive, 1, 1024, 0, s, v, n, total);
    ++*launches;
    return;
  }
  const u64 nb = (n + kScanBlk - 1) / kScanBlk;
  launch_pdl(k_scan_totals, (unsigned)nb, kScanBlk, 0, s, v, n, tmp);
  launch_pdl(k_scan_exclusive, 1, 1024, 0, s, tmp, nb, total);
  launch_pdl(k_scan_apply, (unsigned)nb, kScanBlk, 0, s, v, n, tmp);
  *launches += 3;
}

__device__ __forceinline__ void score_one_lut(const DevBuffers& b, const DevConfig& cfg,
                                              const DevModel& m, uint32_t inst, u64 rb, u64 k, u64 g,
                                              const double* t0, const double* t1);

__global__ void __launch_bounds__(kRecThreads) k_records_scatter(DevBuffers b, DevConfig cfg, int fuse_score) {
  pdl_enter();
  __shared__ uint32_t s_w[kRecPer][kRecThreads / 32];
  __shared__ uint32_t s_rank[kRecBlock];  // exclusive record rank of each cycle in the block
  const bool need_index = cfg.cyc.monitor_from_cycle > 0 || b.stream;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 gb = (u64)blockIdx.x * kRecBlock;
  // the block's record base and first instance load while the cycles do
  __shared__ u64 s_base;
  __shared__ uint32_t s_lo;
  if (threadIdx.x == 32) s_base = b.block_tmp[blockIdx.x];
  if (threadIdx.x == 64) {
    uint32_t lo = 0, hi = b.n_inst + 1;  // first i with cyc_off[i] >= gb
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (b.cyc_off[mid] < gb) lo = mid + 1;
      else hi = mid;
    }
    s_lo = lo;
  }
  bool ok[kRecPer];
  uint32_t m[kRecPer];
#pragma unroll
  for (int r = 0; r < kRecPer; ++r) {
    const u64 g = gb + threadIdx.x + (u64)r * kRecThreads;
    ok[r] = g < b.n_cycles && rec_ok(b, cfg, g, need_index);
    m[r] = __ballot_sync(0xffffffffu, ok[r]);
    if (lane == 0) s_w[r][warp] = __popc(m[r]);
  }
  __syncthreads();
  static_assert(kRecPer * (kRecThreads / 32) == 32, "one warp scans the (row, warp) counts");
  if (warp == 0) {  // exclusive prefix over (row, warp) in cycle order
    uint32_t* sw = &s_w[0][0];
    const uint32_t x = sw[lane];
    uint32_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    sw[lane] = incl - x;
  }
  __syncthreads();
  const u64 base = s_base;
#pragma unroll
  for (int r = 0; r < kRecPer; ++r) {
    const uint32_t local = s_w[r][warp] + __popc(m[r] & lanemask_lt());
    s_rank[threadIdx.x + r * kRecThreads] = local;
    if (ok[r]) b.rec_cycle[base + local] = gb + threadIdx.x + (u64)r * kRecThreads;
  }
  if (fuse_score) {  // score the block's records here (the cycle rows are at hand)
#pragma unroll
    for (int r = 0; r < kRecPer; ++r) {
      if (!ok[r]) continue;
      const u64 g = gb + threadIdx.x + (u64)r * kRecThreads;
      const uint32_t inst = b.n_inst == 1 ? 0u : b.c_inst[g];
      const DevModel& md = b.models[inst];
      score_one_lut(b, cfg, md, inst, 0, base + s_rank[threadIdx.x + r * kRecThreads], g, md.lut_thr[0],
                    md.lut_thr[1]);
    }
  }
  __syncthreads();
  // per-instance record offsets: the rank of each instance's first cycle that
  // falls in this block (empty instances share it); the instances of a block
  // split across its threads (a fleet batch has hundreds per block)
  const u64 ge = gb + kRecBlock < b.n_cycles ? gb + kRecBlock : b.n_cycles;
  for (uint32_t i = s_lo + threadIdx.x; i < b.n_inst; i += kRecThreads) {
    const u64 c0 = b.cyc_off[i];
    if (c0 >= ge) break;  // cyc_off is nondecreasing
    b.rec_off[i] = base + s_rank[c0 - gb];
  }
}

__global__ void k_rec_off_tail(DevBuffers b, uint64_t* total) {
  pdl_enter();
  // instances whose cycles start at n_cycles (trailing empty ones) and the end
  for (i64 i = b.n_inst; i >= 0 && b.cyc_off[i] == b.n_cycles; --i) b.rec_off[i] = *total;
}

// ------------------------------------------------------------ K6 score
// GBDT predict (gbdt.cpp:22-30,173-184) in shared memory, complete-tree
// layout (BFS order; level-contiguous nodes keep warp reads conflict-free),
// then ppe (detector.cpp:14-19).  Tile = 8192 records, model staged once per
// (tile, instance).
constexpr int kScoreThreads = 256;
constexpr int kScoreILP = 4;                     // independent records per thread
constexpr int kScoreTile = kScoreThreads * kScoreILP * 8;

// Exact stand-in for `x <= thr` when x is an integer-valued double with
// |x| <= 2^53: x <= thr  <=>  (int64)x <= floor(thr) (host-precomputed, with
// +inf -> INT64_MAX and -inf/NaN -> a value below every such x).
template <int NF>
__device__ __forceinline__ double pick(const double (&x)[NF > 0 ? NF : 1], uint32_t f) {
  double v = x[0];
#pragma unroll
  for (int k = 1; k < NF; ++k) v = (f == (uint32_t)k) ? x[k] : v;
  return v;
}
template <int NF>
__device__ __forceinline__ i64 pick_i(const i64 (&x)[NF > 0 ? NF : 1], uint32_t f) {
  i64 v = x[0];
#pragma unroll
  for (int k = 1; k < NF; ++k) v = (f == (uint32_t)k) ? x[k] : v;
  return v;
}

// Records are counted on the device (rec_off[n_inst]); record kernels are
// launched over a capacity (the cycle count) and clamp to the device count,
// so cs_run needs no host round trip between records and scoring.
__device__ __forceinline__ u64 records_on_device(const DevBuffers& b, u64 cap) {
  const u64 n = b.rec_off[b.n_inst];
  return n < cap ? n : cap;
}

// record extras (cycles.cpp:392-405): thread per record; the cycle's events
// carrying extras are found by binary search in the event-sorted side table,
// and each key keeps the value of the last such event (map assignment order)
__global__ void k_record_extras(DevBuffers b, uint64_t n_records) {
  n_records = records_on_device(b, n_records);
  const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_records) return;
  const uint32_t K = b.n_extra_keys;
  double* vals = b.rec_extra + k * K;
  uint8_t* has = b.rec_extra_has + k * K;
  for (uint32_t j = 0; j < K; ++j) {
    vals[j] = 0.0;
    has[j] = 0;
  }
  const u64 g = b.rec_cycle[k];
  const u64 first = b.c_first[g], last = b.c_last[g];
  u64 lo = 0, hi = b.n_extra_refs;  // first ref with event >= first
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (b.extra_refs[mid].event < first) lo = mid + 1;
    else hi = mid;
  }
  for (u64 r = lo; r < b.n_extra_refs && b.extra_refs[r].event < last; ++r) {
    const cs_extra_ref ref = b.extra_refs[r];
    for (uint32_t v = 0; v < ref.count; ++v) {
      const cs_extra_value ev = b.extra_vals[ref.first + v];
      if (ev.key < K) {
        vals[ev.key] = ev.value;
        has[ev.key] = 1;
      }
    }
  }
}

void launch_record_extras(const DevBuffers& b, uint64_t n_records_cap, cudaStream_t s, uint64_t* launches) {
  if (!n_records_cap || !b.n_extra_keys) return;
  k_record_extras<<<(unsigned)((n_records_cap + 127) / 128), 128, 0, s>>>(b, n_records_cap);
  ++*launches;
}


template <int NF>
__global__ void __launch_bounds__(kScoreThreads)
    k_score(DevBuffers b, DevConfig cfg, uint64_t n_records, uint64_t smem_cap) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char s_model[];
  __shared__ uint32_t s_inst;
  n_records = records_on_device(b, n_records);
  const u64 r0 = (u64)blockIdx.x * kScoreTile;
  const u64 r1 = min(r0 + (u64)kScoreTile, (u64)n_records);
  const double eps = cfg.ctl.epsilon;
  const int lat = cfg.cyc.latency_phase;
  const int P = cfg.cyc.n_phases;
  const void* staged = nullptr;
  u64 r = r0;
  while (r < r1) {
    if (threadIdx.x == 0) s_inst = upper_bound_u64(b.rec_off, b.n_inst + 1, r) - 1;
    __syncthreads();
    const uint32_t inst = s_inst;
    const u64 seg_end = min(r1, (u64)b.rec_off[inst + 1]);
    const DevModel& m = b.models[inst];
    const uint32_t D = m.depth, NT = m.n_trees;
    const uint32_t ni = (1u << D) - 1, nl = 1u << D;
    const i64* thr = m.thr_i;
    const uint8_t* feat = m.feat;
    const double* leaf = m.leaf;
    if (m.smem_bytes <= smem_cap) {
      i64* st = reinterpret_cast<i64*>(s_model);
      double* sl = reinterpret_cast<double*>(st + (u64)NT * ni);
      uint8_t* sf = reinterpret_cast<uint8_t*>(sl + (u64)NT * nl);
      if (m.thr_i != staged) {  // instances sharing a model reuse the staged copy
        for (u64 i = threadIdx.x; i < (u64)NT * ni; i += blockDim.x) st[i] = m.thr_i[i];
        for (u64 i = threadIdx.x; i < (u64)NT * nl; i += blockDim.x) sl[i] = m.leaf[i];
        for (u64 i = threadIdx.x; i < (u64)NT * ni; i += blockDim.x) sf[i] = m.feat[i];
        staged = m.thr_i;
      }
      thr = st;
      leaf = sl;
      feat = sf;
    }
    __syncthreads();
    const u64 rb = b.rec_off[inst];
    const double base = m.base, fl = m.floor_;
    for (u64 k0 = r + threadIdx.x; k0 < seg_end; k0 += (u64)blockDim.x * kScoreILP) {
      double x[kScoreILP][NF > 0 ? NF : 1];
      i64 xi[kScoreILP][NF > 0 ? NF : 1];
      double y[kScoreILP], v[kScoreILP];
      bool live[kScoreILP], exact = true;
#pragma unroll
      for (int q = 0; q < kScoreILP; ++q) {
        const u64 k = k0 + (u64)q * blockDim.x;
        live[q] = k < seg_end;
        v[q] = base;
        y[q] = 1.0;
        if (!live[q]) {
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            x[q][f] = 0.0;
            xi[q][f] = 0;
          }
          continue;
        }
        const u64 g = b.rec_cycle[k];
        const cs_workload w = b.wl[b.c_wl[g]];
        i64 target = b.c_end[g] - b.c_start[g];
        if (lat >= 0) {
          const i64 c = b.c_comp[g * P + lat];
          if (c > 0) target = c;
        }
        y[q] = __dmul_rn((double)target, 1e-9);  // cycles.cpp:390
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          i64 iv = 0;
          const int32_t id = m.feature_ids[f];
          if (id >= kFeatExtra || id == kFeatMissing) {
            // a record extra (main.cpp:70-75): double-valued, compared as such
            const u64 ke = k * (u64)b.n_extra_keys + (u64)(id - kFeatExtra);
            if (id == kFeatMissing || !b.rec_extra_has[ke]) {
              atomicMin(reinterpret_cast<u64*>(&b.inst[inst].first_missing_record), (u64)(k - rb));
              x[q][f] = 0.0;
            } else {
              x[q][f] = b.rec_extra[ke];
            }
            xi[q][f] = 0;
            exact = false;
            continue;
          }
          switch (id) {
            case CS_F_BATCH: iv = w.batch; break;
            case CS_F_W_KV: iv = w.batch * (w.input_len + w.output_len); break;
            case CS_F_INPUT_LEN: iv = w.input_len; break;
            case CS_F_OUTPUT_LEN: iv = w.output_len; break;
            default: iv = b.c_stage[g] == CS_STAGE_PREFILL ? 1 : 0; break;
          }
          xi[q][f] = iv;
          x[q][f] = (double)iv;
          exact &= (iv <= (1ll << 53)) && (iv >= -(1ll << 53));
        }
      }
      if (exact) {
        for (uint32_t t = 0; t < NT; ++t) {
          const i64* tt = thr + (u64)t * ni;
          const uint8_t* tf = feat + (u64)t * ni;
          uint32_t node[kScoreILP];
#pragma unroll
          for (int q = 0; q < kScoreILP; ++q) node[q] = 0;
          for (uint32_t d = 0; d < D; ++d) {
#pragma unroll
            for (int q = 0; q < kScoreILP; ++q) {
              const uint32_t f = tf[node[q]];
              node[q] = 2 * node[q] + 1 + (pick_i<NF>(xi[q], f) <= tt[node[q]] ? 0u : 1u);
            }
          }
          const double* tl = leaf + (u64)t * nl - ni;
#pragma unroll
          for (int q = 0; q < kScoreILP; ++q) v[q] = __dadd_rn(v[q], tl[node[q]]);
        }
      } else {
        // values beyond 2^53: compare the rounded doubles like the reference
        for (uint32_t t = 0; t < NT; ++t) {
          const double* tt = m.thr + (u64)t * ni;
          const uint8_t* tf = m.feat + (u64)t * ni;
          uint32_t node[kScoreILP];
#pragma unroll
          for (int q = 0; q < kScoreILP; ++q) node[q] = 0;
          for (uint32_t d = 0; d < D; ++d) {
#pragma unroll
            for (int q = 0; q < kScoreILP; ++q) {
              const uint32_t f = tf[node[q]];
              node[q] = 2 * node[q] + 1 + (pick<NF>(x[q], f) <= tt[node[q]] ? 0u : 1u);
            }
          }
          const double* tl = m.leaf + (u64)t * nl - ni;
#pragma unroll
          for (int q = 0; q < kScoreILP; ++q) v[q] = __dadd_rn(v[q], tl[node[q]]);
        }
      }
#pragma unroll
      for (int q = 0; q < kScoreILP; ++q) {
        if (!live[q]) continue;
        const u64 k = k0 + (u64)q * blockDim.x;
        const double p = fl < v[q] ? v[q] : fl;
        double res;
        if (!(y[q] > 0.0)) {
          atomicMin(reinterpret_cast<u64*>(&b.inst[inst].first_bad_record), (u64)(k - rb));
          res = __longlong_as_double(0x7ff8000000000000ll);
        } else {
          const double qv = __ddiv_rn(__dsub_rn(y[q], p), __dadd_rn(y[q], eps));
          res = 0.0 < qv ? qv : 0.0;
        }
        b.rec_pred[k] = p;
        b.rec_resid[k] = res;
      }
    }
    __syncthreads();
    r = seg_end;
  }
}

// -------------------------------------------- K6' compiled-ensemble score
// For models with <= 2 features the ensemble is piecewise constant on the
// grid of its distinct split thresholds.  cell (k0, k1), k_f = #{T_f < x_f},
// decides every node exactly like x <= t does (x <= T_f[j] <=> k_f <= j), so
// a table built with the reference's sequential tree-order sum per cell is
// bit-identical to traversing the trees (gbdt.cpp:22-30, 173-184).
__global__ void k_lut_build(const uint8_t* __restrict__ feat, const int32_t* __restrict__ rank,
                            const double* __restrict__ leafp, uint32_t n_trees, uint32_t D,
                            double base, double floor_, uint32_t n0, uint64_t cells,
                            double* __restrict__ lut) {
  const u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const int32_t k0 = (int32_t)(c % (n0 + 1)), k1 = (int32_t)(c / (n0 + 1));
  const uint32_t ni = (1u << D) - 1, nl = 1u << D;
  double v = base;
  for (uint32_t t = 0; t < n_trees; ++t) {
    uint32_t node = 0;
    for (uint32_t d = 0; d < D; ++d) {
      const uint32_t f = feat[(u64)t * ni + node];
      const int32_t k = f == 0 ? k0 : k1;
      node = 2 * node + 1 + (k <= rank[(u64)t * ni + node] ? 0u : 1u);
    }
    v = __dadd_rn(v, leafp[(u64)t * nl + (node - ni)]);
  }
  lut[c] = floor_ < v ? v : floor_;
}

void launch_lut_build(const uint8_t* feat, const int32_t* rank, const double* leafp,
                      uint32_t n_trees, uint32_t D, double base, double floor_, uint32_t n0,
                      uint64_t cells, double* lut, cudaStream_t s) {
  k_lut_build<<<(unsigned)((cells + 127) / 128), 128, 0, s>>>(feat, rank, leafp, n_trees, D, base,
                                                              floor_, n0, cells, lut);
}

__device__ __forceinline__ uint32_t count_less(const double* __restrict__ t, uint32_t n, double x) {
  uint32_t lo = 0, hi = n;  // lower_bound: first t >= x
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (t[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One record through the compiled cell table: latency target (cycles.cpp:
// 384-390), features (baseline.cpp:61-62), prediction (gbdt.cpp:173-184),
// ppe (detector.cpp:14-19).
// record k of cycle g; the atomics store k - rb (rb = 0: absolute indices)
__device__ __forceinline__ void score_one_lut(const DevBuffers& b, const DevConfig& cfg,
                                              const DevModel& m, uint32_t inst, u64 rb, u64 k, u64 g,
                                              const double* t0, const double* t1) {
  const double eps = cfg.ctl.epsilon;
  const int lat = cfg.cyc.latency_phase;
  const int P = cfg.cyc.n_phases;
  const uint32_t n0 = m.lut_n[0], n1 = m.lut_n[1];
  const int f0 = m.feature_ids[0], f1 = m.n_features > 1 ? m.feature_ids[1] : -1;
  const cs_workload w = b.wl[b.c_wl[g]];
  i64 target = b.c_end[g] - b.c_start[g];
  if (lat >= 0) {
    const i64 c = b.c_comp[g * P + lat];
    if (c > 0) target = c;
  }
  const double y = __dmul_rn((double)target, 1e-9);  // cycles.cpp:390
  const uint8_t stage = b.c_stage[g];
  auto fval = [&](int id) -> double {
    if (id >= kFeatExtra || id == kFeatMissing) {
      const u64 ke = k * (u64)b.n_extra_keys + (u64)(id - kFeatExtra);
      if (id == kFeatMissing || !b.rec_extra_has[ke]) {
        atomicMin(reinterpret_cast<u64*>(&b.inst[inst].first_missing_record), (u64)(k - rb));
        return 0.0;
      }
      return b.rec_extra[ke];
    }
    switch (id) {
      case CS_F_BATCH: return (double)w.batch;
      case CS_F_W_KV: return (double)(w.batch * (w.input_len + w.output_len));
      case CS_F_INPUT_LEN: return (double)w.input_len;
      case CS_F_OUTPUT_LEN: return (double)w.output_len;
      default: return stage == CS_STAGE_PREFILL ? 1.0 : 0.0;
    }
  };
  const uint32_t k0 = count_less(t0, n0, fval(f0));
  const uint32_t k1 = f1 >= 0 ? count_less(t1, n1, fval(f1)) : 0;
  const double p = m.lut[(u64)k1 * (n0 + 1) + k0];
  double res;
  if (!(y > 0.0)) {
    atomicMin(reinterpret_cast<u64*>(&b.inst[inst].first_bad_record), (u64)(k - rb));
    res = __longlong_as_double(0x7ff8000000000000ll);
  } else {
    const double q = __ddiv_rn(__dsub_rn(y, p), __dadd_rn(y, eps));
    res = 0.0 < q ? q : 0.0;
  }
  b.rec_pred[k] = p;
  b.rec_resid[k] = res;
}

#ifndef CS_LUT_THREADS
#define CS_LUT_THREADS 256
#endif
constexpr int kLutThreads = CS_LUT_THREADS;
// Thread per record, its instance by binary search (independent across
// threads), thresholds read through L1.  A grid of one thread per record
// keeps more gathers in flight than a tiled kernel with the thresholds staged
// in shared memory (configs[1]: 83 vs 100 us), so every batch uses it.
__global__ void __launch_bounds__(kLutThreads)
    k_score_lut_flat(DevBuffers b, DevConfig cfg, uint64_t n_records) {
  pdl_enter();
  n_records = records_on_device(b, n_records);
  const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_records) return;
  const uint32_t inst = upper_bound_u64(b.rec_off, b.n_inst + 1, k) - 1;
  const DevModel& m = b.models[inst];
  score_one_lut(b, cfg, m, inst, b.rec_off[inst], k, b.rec_cycle[k], m.lut_thr[0], m.lut_thr[1]);
}

// ------------------------------------------------------------ K7 detect
// Detector::step (detector.cpp:91-130) for every record at once:
//   stat_t  = e_t (FixedPoint) or (sum_{u=max(0,t-W+1)}^{t} e_u, oldest first)/count
//   armed_t = t >= warmup;  flagged_t = armed_t && stat_t > limit
//   alert_t = flagged_t && !flagged_{t-1}   (in_episode == flagged_{t-1})
// Episode id = alerts before t in the instance (exclusive scan).
constexpr int kDetBlock = 1024;  // records per detect block (both flag kernels, the scatter)

__device__ __forceinline__ double window_stat(const double* e, u64 t, u64 W, int strategy) {
  if (strategy == CS_FIXED_POINT) return e[t];
  const u64 begin = t + 1 >= W ? t + 1 - W : 0;
  double sum = 0.0;
  for (u64 u = begin; u <= t; ++u) sum = __dadd_rn(sum, e[u]);
  return __ddiv_rn(sum, (double)(t - begin + 1));
}

// Same statistic for stream position T = seen + t: residuals of earlier
// micro-batches come from the carried history (oldest first).
__device__ __forceinline__ double window_stat_stream(const double* e, u64 t, u64 W, int strategy,
                                                     const StreamCarry& c, const double* hist) {
  const u64 T = c.seen + t;
  if (strategy == CS_FIXED_POINT) return e[t];
  const u64 begin = T + 1 >= W ? T + 1 - W : 0;
  const u64 h0 = c.seen - c.n_hist;  // stream index of hist[0]
  double sum = 0.0;
  for (u64 u = begin; u <= T; ++u) sum = __dadd_rn(sum, u < c.seen ? hist[u - h0] : e[u - c.seen]);
  return __ddiv_rn(sum, (double)(T - begin + 1));
}

// one record of the control chart (detector.cpp:91-130), warp-collective
// (the previous record's statistic comes from the neighbouring lane); writes
// rec_stat / rec_flags and counts the instance's alerts; returns alert
__device__ __forceinline__ bool detect_record(const DevBuffers& b, const DevConfig& cfg, u64 k, bool valid) {
  const int lane = threadIdx.x & 31;
  bool alert = false;
  uint32_t inst = 0xffffffffu;
  u64 t = 0, rb = 0;
  double stat = 0.0;
  const u64 W = cfg.ctl.window, warm = cfg.ctl.warmup;
  if (valid) {
    inst = upper_bound_u64(b.rec_off, b.n_inst + 1, k) - 1;
    rb = b.rec_off[inst];
    t = k - rb;
    stat = b.stream ? window_stat_stream(b.rec_resid + rb, t, W, cfg.ctl.strategy, b.stream[inst],
                                         b.s_hist + (u64)inst * b.s_hw)
                    : window_stat(b.rec_resid + rb, t, W, cfg.ctl.strategy);
  }
  // statistic of record k-1: the neighbouring lane's, unless it is in another
  // warp or instance (then recomputed, identically)
  const double up_stat = __shfl_up_sync(0xffffffffu, stat, 1);
  const uint32_t up_inst = __shfl_up_sync(0xffffffffu, inst, 1);
  if (valid) {
    const double limit = b.models[inst].ucl;
    const double* e = b.rec_resid + rb;
    bool armed, prev = false;
    const bool have_up = lane > 0 && up_inst == inst;
    if (b.stream) {
      const StreamCarry& c = b.stream[inst];
      const u64 T = c.seen + t;
      armed = T >= warm;
      if (t == 0) prev = c.prev_flag != 0;
      else if (T - 1 >= warm)
        prev = (have_up ? up_stat
                        : window_stat_stream(e, t - 1, W, cfg.ctl.strategy, c, b.s_hist + (u64)inst * b.s_hw)) > limit;
    } else {
      armed = t >= warm;
      if (t >= 1 && t - 1 >= warm)
        prev = (have_up ? up_stat : window_stat(e, t - 1, W, cfg.ctl.strategy)) > limit;
    }
    const bool flagged = armed && stat > limit;
    alert = flagged && !prev;
    b.rec_stat[k] = stat;
    b.rec_flags[k] = (armed ? 1 : 0) | (flagged ? 2 : 0) | (alert ? 4 : 0);
    if (alert) atomicAdd(&b.inst[inst].n_alerts, 1ull);
  }
  return alert;
}

__global__ void k_detect_flags(DevBuffers b, DevConfig cfg, uint64_t n_records) {
  pdl_enter();
  __shared__ uint32_t s_w[32];
  n_records = records_on_device(b, n_records);
  const u64 k = (u64)blockIdx.x * kDetBlock + threadIdx.x;
  const bool alert = detect_record(b, cfg, k, k < n_records);
  const uint32_t m = __ballot_sync(0xffffffffu, alert);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = __popc(m);
  __syncthreads();
  if (threadIdx.x < 32) {
    u64 v = threadIdx.x < kDetBlock / 32 ? s_w[threadIdx.x] : 0u;
    v = warp_sum_u64(v);
    if (threadIdx.x == 0) b.block_tmp[blockIdx.x] = v;
  }
}

// Small batches (a streaming micro-batch): flags, alert list and per-instance
// alert offsets in one CTA instead of flags + scan + offsets + scatter
__global__ void __launch_bounds__(1024) k_detect_small(DevBuffers b, DevConfig cfg, uint64_t n_records) {
  pdl_enter();
  __shared__ uint32_t s_w[32];
  __shared__ u64 s_base;
  n_records = records_on_device(b, n_records);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (u64 k0 = 0; k0 < n_records; k0 += 1024) {
    const u64 k = k0 + threadIdx.x;
    const bool alert = detect_record(b, cfg, k, k < n_records);
    const uint32_t m = __ballot_sync(0xffffffffu, alert);
    if (lane == 0) s_w[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
      uint32_t c = s_w[lane];
      const uint32_t x = c;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, c, o);
        if (lane >= o) c += y;
      }
      s_w[lane] = c - x;
    }
    __syncthreads();
    const u64 base = s_base;
    if (alert) b.alert_rec[base + s_w[warp] + __popc(m & lanemask_lt())] = k;
    __syncthreads();
    if (threadIdx.x == 1023) s_base = base + s_w[31] + __popc(m);  // last warp's prefix + its own count
    __syncthreads();
  }
  // alerts are in record order: instance i's first alert is the first whose
  // record index is >= rec_off[i]
  const u64 total = s_base;
  for (uint32_t i = threadIdx.x; i <= b.n_inst; i += blockDim.x) {
    if (i == b.n_inst) {
      b.alert_off[i] = total;
      continue;
    }
    const u64 r = b.rec_off[i];
    u64 lo = 0, hi = total;
    while (lo < hi) {
      const u64 mid = (lo + hi) >> 1;
      if (b.alert_rec[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    b.alert_off[i] = lo;
  }
}

// Control chart for whole runs (no stream carry), window length W <= kDetMaxW
// as a template parameter (FixedPoint: W = 0).  A CTA takes kDetBlock
// consecutive records: their residuals plus the W before them are staged in
// shared memory with coalesced loads; each statistic is still the sequential
// oldest-to-newest sum of its own window (detector.cpp:96-104) -- W ordered
// adds, unrolled, and one division -- and the previous record's statistic
// (in_episode = armed && flagged at t-1, detector.cpp:107-128) comes from the
// CTA's statistics in shared memory.  Stores are coalesced (thread stride).
constexpr int kDetMaxW = 16;
#ifndef CS_DET_THREADS
#define CS_DET_THREADS 256
#endif
constexpr int kDetThreads = CS_DET_THREADS;
template <int W>
__global__ void __launch_bounds__(kDetThreads) k_detect_win(DevBuffers b, DevConfig cfg, uint64_t n_records) {
  pdl_enter();
  __shared__ double s_e[kDetBlock + kDetMaxW];
  __shared__ double s_st[kDetBlock + 1];
  __shared__ uint32_t s_w[kDetThreads / 32];
  n_records = records_on_device(b, n_records);
  const u64 k0 = (u64)blockIdx.x * kDetBlock;
  if (k0 >= n_records) {
    if (threadIdx.x == 0) b.block_tmp[blockIdx.x] = 0;
    return;
  }
  const u64 kend = k0 + kDetBlock < n_records ? k0 + kDetBlock : n_records;
  constexpr u64 kHalo = W > 0 ? (u64)W : 1u;  // the window of the record before the block
  const u64 base = k0 >= kHalo ? k0 - kHalo : 0;  // s_e[i] = e[base + i]
  const u64 need = kend - base;
  for (u64 i = threadIdx.x; i < need; i += kDetThreads) s_e[i] = b.rec_resid[base + i];
  __syncthreads();
  const u64 warm = cfg.ctl.warmup;
  // instance of the record before the block (or of the first), one search
  // per thread; the loops walk forward from it
  const u64 kfirst = k0 > 0 ? k0 - 1 : 0;
  uint32_t inst0 = upper_bound_u64(b.rec_off, b.n_inst + 1, kfirst) - 1;
  auto stat_at = [&](u64 k, u64 rb) -> double {
    if (W == 0) return s_e[k - base];
    const u64 lo = k + 1 >= rb + W ? k + 1 - W : rb;
    double sum = 0.0;
    if (k + 1 - lo == (u64)W) {
      const double* p = s_e + (k + 1 - W - base);
#pragma unroll
      for (int u = 0; u < W; ++u) sum = __dadd_rn(sum, p[u]);
    } else {
      for (u64 u = lo; u <= k; ++u) sum = __dadd_rn(sum, s_e[u - base]);
    }
    return __ddiv_rn(sum, (double)(k + 1 - lo));
  };
  // statistics of the block's records and of the record before the block
  // (s_st[0]), spread over the threads alike
  for (u64 k = kfirst + threadIdx.x; k < kend; k += kDetThreads) {
    uint32_t inst = inst0;
    while (b.rec_off[inst + 1] <= k) ++inst;
    s_st[1 + k - k0] = stat_at(k, b.rec_off[inst]);
  }
  __syncthreads();
  uint32_t n_alert = 0;
  for (u64 k = k0 + threadIdx.x; k < kend; k += kDetThreads) {
    uint32_t inst = inst0;
    while (b.rec_off[inst + 1] <= k) ++inst;
    const u64 t = k - b.rec_off[inst];
    const double limit = b.models[inst].ucl;
    const double st = s_st[1 + (k - k0)];
    const bool armed = t >= warm;
    const bool prev = t >= 1 && t - 1 >= warm && s_st[k - k0] > limit;
    const bool flagged = armed && st > limit;
    const bool alert = flagged && !prev;
    b.rec_stat[k] = st;
    b.rec_flags[k] = (armed ? 1 : 0) | (flagged ? 2 : 0) | (alert ? 4 : 0);
    if (alert) {
      atomicAdd(&b.inst[inst].n_alerts, 1ull);
      ++n_alert;
    }
  }
  const uint32_t wsum = (uint32_t)warp_sum_u64(n_alert);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 t = 0;
    for (int w = 0; w < kDetThreads / 32; ++w) t += s_w[w];
    b.block_tmp[blockIdx.x] = t;
  }
}

// After a micro-batch: the carry the next one starts from (written to `out`,
// the carry in force for this batch stays readable for the getters).
// One warp per instance: the carry the next micro-batch starts from.  The
// detector keeps the last W-1 residuals, the flag of the last record and the
// episode count (detector.cpp:91-130); the stage heuristic its two trailing
// windows, newest first (cycles.cpp:204-250).  Lanes copy the windows and
// take the batch's cycles 32 at a time (ballot compaction keeps the
// reference's newest-first order).
__global__ void __launch_bounds__(128) k_stream_update(DevBuffers b, DevConfig cfg, StreamCarry* out,
                                                       double* out_hist, double* out_dur, double* out_gap,
                                                       int detected) {
  pdl_enter();
  const uint32_t inst = blockIdx.x * 4 + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (inst >= b.n_inst) return;
  const StreamCarry& c = b.stream[inst];
  StreamCarry& o = out[inst];
  const double* chist = b.s_hist + (u64)inst * b.s_hw;
  double* ohist = out_hist + (u64)inst * b.s_hw;
  // detector window
  if (detected) {
    const u64 r0 = b.rec_off[inst], n = b.rec_off[inst + 1] - r0;
    const u64 keep = cfg.ctl.window > 0 ? cfg.ctl.window - 1 : 0;
    const u64 total = c.seen + n;
    const u64 nh = total < keep ? total : keep;
    const u64 h0 = c.seen - c.n_hist;
    for (u64 i = lane; i < nh; i += 32) {
      const u64 u = total - nh + i;  // stream index
      ohist[i] = u < c.seen ? chist[u - h0] : b.rec_resid[r0 + (u - c.seen)];
    }
    if (lane == 0) {
      o.n_hist = (uint32_t)nh;
      o.prev_flag = n ? ((b.rec_flags[r0 + n - 1] & 2) ? 1u : 0u) : c.prev_flag;
      o.seen = total;
      o.episodes = c.episodes + b.inst[inst].n_alerts;
    }
  } else {
    for (uint32_t i = lane; i < c.n_hist; i += 32) ohist[i] = chist[i];
    if (lane == 0) {
      o.n_hist = c.n_hist;
      o.prev_flag = c.prev_flag;
      o.seen = c.seen;
      o.episodes = c.episodes;
    }
  }
  // stage-heuristic history: newest cycles of this batch first, then the carry
  const u64 c0 = b.cyc_off[inst], c1 = b.cyc_off[inst + 1];
  const uint32_t W = b.s_sw;
  const double* cdur = b.s_dur + (u64)inst * b.s_sw;
  const double* cgap = b.s_gap + (u64)inst * b.s_sw;
  double* odur = out_dur + (u64)inst * b.s_sw;
  double* ogap = out_gap + (u64)inst * b.s_sw;
  uint32_t nd = 0, ng = 0;
  const uint32_t lt = (1u << lane) - 1u;
  for (u64 top = c1; top > c0 && (nd < W || ng < W); top = top > c0 + 32 ? top - 32 : c0) {
    const bool have = top > c0 + lane;
    const u64 j = have ? top - 1 - lane : c0;
    bool np = false, gv = false;
    double dur = 0.0, g = 0.0;
    if (have && b.c_stage[j] != CS_STAGE_PREFILL) {
      np = true;
      dur = (double)(b.c_end[j] - b.c_start[j]);
      if (j > c0 || c.has_prev) {
        const i64 prev_end = j > c0 ? b.c_aend[j - 1] : c.last_aend;
        g = (double)(b.c_start[j] - prev_end);
        gv = g >= 0.0;
      }
    }
    const uint32_t dm = __ballot_sync(0xffffffffu, np);
    const uint32_t gm = __ballot_sync(0xffffffffu, gv);
    const uint32_t di = nd + __popc(dm & lt), gi = ng + __popc(gm & lt);
    if (np && di < W) odur[di] = dur;
    if (gv && gi < W) ogap[gi] = g;
    nd = min(W, nd + __popc(dm));
    ng = min(W, ng + __popc(gm));
  }
  for (uint32_t i = lane; i < c.n_dur && nd + i < W; i += 32) odur[nd + i] = cdur[i];
  for (uint32_t i = lane; i < c.n_gap && ng + i < W; i += 32) ogap[ng + i] = cgap[i];
  if (lane == 0) {
    o.n_dur = min(W, nd + c.n_dur);
    o.n_gap = min(W, ng + c.n_gap);
    o.has_prev = (c1 > c0) ? 1u : c.has_prev;
    o.last_aend = (c1 > c0) ? b.c_aend[c1 - 1] : c.last_aend;
    o.cycle_off = c.cycle_off + (c1 - c0);
  }
}

void launch_stream_update(const DevBuffers& b, const DevConfig& cfg, StreamCarry* out, double* out_hist,
                          double* out_dur, double* out_gap, int detected, cudaStream_t s) {
  launch_pdl(k_stream_update, (b.n_inst + 3) / 4, 128, 0, s, b, cfg, out, out_hist, out_dur, out_gap, detected);
}

// exclusive scan over instances of n_alerts: one CTA, kScanItems per thread per round
__global__ void __launch_bounds__(1024) k_alert_off(DevBuffers b) {
  pdl_enter();
  __shared__ u64 s_w[32];
  __shared__ u64 s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base <= b.n_inst; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const u64 x = i < b.n_inst ? b.inst[i].n_alerts : 0;
    u64 t;
    const u64 incl = block_incl_scan(x, s_w, &t);
    if (i <= b.n_inst) b.alert_off[i] = s_carry + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += t;
    __syncthreads();
  }
}

// alert list in record order: a warp per detect block, and only blocks with
// alerts (block_tmp holds the exclusive prefix of their counts, the total at
// [nb]) are read again -- alerts are rare, so this touches a few blocks
constexpr int kDetScatterThreads = 256;
static_assert(kDetBlock == 32 * 32, "k_detect_scatter: 32 records per lane");
__global__ void __launch_bounds__(kDetScatterThreads) k_detect_scatter(DevBuffers b, uint64_t n_records, uint64_t nb) {
  pdl_enter();
  n_records = records_on_device(b, n_records);
  const int lane = threadIdx.x & 31;
  const u64 nw = ((u64)gridDim.x * blockDim.x) >> 5;
  for (u64 bi = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5; bi < nb; bi += nw) {
    u64 out = b.block_tmp[bi];
    if (out == b.block_tmp[bi + 1]) continue;
    // lane l takes records [k0 + 32 l, k0 + 32 l + 32): one load round trip
    // for the block, then the lanes' alerts in lane (= record) order
    const u64 k0 = bi * kDetBlock;
    const u64 k1 = min(k0 + (u64)kDetBlock, (u64)n_records);
    const u64 kb = k0 + 32u * (u64)lane;
    uint32_t bits = 0;
    if (kb + 32 <= k1) {
      const uint4* p = reinterpret_cast<const uint4*>(b.rec_flags + kb);  // kb % 32 == 0
      const uint4 v0 = p[0], v1 = p[1];
      const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) bits |= ((w[q] >> (8 * j + 2)) & 1u) << (4 * q + j);
    } else {
      for (u64 k = kb; k < k1; ++k) bits |= ((b.rec_flags[k] >> 2) & 1u) << (uint32_t)(k - kb);
    }
    const uint32_t cnt = __popc(bits);
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    u64 pos = out + incl - cnt;
    while (bits) {
      b.alert_rec[pos++] = kb + (u64)(__ffs(bits) - 1);
      bits &= bits - 1;
    }
  }
}

// ------------------------------------------------- evaluate_strategy
// detector.cpp:166-224 over one instance's records: confusion counts from the
// flagged bits of armed records; lag per contiguous anomaly interval that
// starts at t >= warmup (capped at the interval length).  All counts are
// integers, so any reduction order is exact; out[0..6] = tp, fp, fn, tn,
// alerts, lag_sum, intervals.
__global__ void k_eval_strategy(DevBuffers b, uint32_t inst, const uint8_t* __restrict__ labels,
                                uint64_t n_labels, uint64_t warmup, unsigned long long* out) {
  const u64 r0 = b.rec_off[inst], nr = b.rec_off[inst + 1] - r0;
  const u64 c0 = b.cyc_off[inst];
  u64 tp = 0, fp = 0, fn = 0, tn = 0, al = 0, lag = 0, iv = 0;
  auto anomalous = [&](u64 t) {
    const u64 c = b.rec_cycle[r0 + t] - c0;
    return c < n_labels && labels[c] != 0;
  };
  for (u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += (u64)gridDim.x * blockDim.x) {
    const uint8_t f = b.rec_flags[r0 + t];
    const bool an = anomalous(t);
    if (f & 1) {
      const bool fl = f & 2;
      if (f & 4) ++al;
      if (fl && an) ++tp;
      else if (fl) ++fp;
      else if (an) ++fn;
      else ++tn;
    }
    if (t >= warmup && an && (t == warmup || !anomalous(t - 1))) {
      u64 e = t;
      while (e < nr && anomalous(e)) ++e;
      u64 first = e;
      for (u64 u = t; u < e; ++u)
        if (b.rec_flags[r0 + u] & 2) { first = u; break; }
      lag += first - t;
      ++iv;
    }
  }
  const u64 v[7] = {tp, fp, fn, tn, al, lag, iv};
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const u64 s = warp_sum_u64(v[k]);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(&out[k], s);
  }
}

void launch_eval_strategy(const DevBuffers& b, uint32_t inst, const uint8_t* labels,
                          uint64_t n_labels, uint64_t warmup, unsigned long long* out,
                          cudaStream_t s) {
  k_eval_strategy<<<148, 256, 0, s>>>(b, inst, labels, n_labels, warmup, out);
}

// ------------------------------------------------------------ getters
// Assemble AoS cs_record / cs_alert rows on the device so a getter is one D2H
// of exactly the rows asked for.
__global__ void k_gather_records(DevBuffers b, DevConfig cfg, uint32_t inst, uint64_t r0,
                                 uint64_t nr, int scored, int det, cs_record* out) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nr) return;
  const u64 k = r0 + i;
  const u64 g = b.rec_cycle[k];
  cs_record r;
  r.cycle_index = g - b.cyc_off[inst] + (b.stream ? b.stream[inst].cycle_off : 0);
  r.start_ts = b.c_start[g];
  r.stage = b.c_stage[g];
  const cs_workload w = b.wl[b.c_wl[g]];
  r.batch = w.batch;
  r.input_len = w.input_len;
  r.output_len = w.output_len;
  i64 target = b.c_end[g] - b.c_start[g];
  const int lat = cfg.cyc.latency_phase;
  if (lat >= 0) {
    const i64 c = b.c_comp[g * cfg.cyc.n_phases + lat];
    if (c > 0) target = c;
  }
  r.latency_s = __dmul_rn((double)target, 1e-9);
  r.predicted_s = scored ? b.rec_pred[k] : 0.0;
  r.residual = scored ? b.rec_resid[k] : 0.0;
  r.statistic = det ? b.rec_stat[k] : 0.0;
  const uint8_t f = det ? b.rec_flags[k] : 0;
  r.armed = f & 1;
  r.flagged = (f >> 1) & 1;
  r.alert = (f >> 2) & 1;
  r.reserved = 0;
  r.episode_id = 0;
  out[i] = r;
}

__device__ __forceinline__ cs_alert make_alert(const DevBuffers& b, const DevConfig& cfg, uint32_t inst,
                                               u64 i /* within the instance */, u64 k) {
  const u64 g = b.rec_cycle[k];
  const cs_workload w = b.wl[b.c_wl[g]];
  cs_alert a;
  a.cycle = g - b.cyc_off[inst] + (b.stream ? b.stream[inst].cycle_off : 0);
  a.ts = b.c_start[g];
  a.smoothed_error = b.rec_stat[k];
  a.limit = b.models[inst].ucl;
  a.strategy = cfg.ctl.strategy;
  a.reserved = 0;
  a.batch = w.batch;
  a.input_len = w.input_len;
  a.output_len = w.output_len;
  a.episode_id = i + (b.stream ? b.stream[inst].episodes : 0);
  a.record_index = k - b.rec_off[inst];
  return a;
}

__global__ void k_gather_alerts(DevBuffers b, DevConfig cfg, uint32_t inst, uint64_t a0,
                                uint64_t na, cs_alert* out) {
  pdl_enter();
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= na) return;
  out[i] = make_alert(b, cfg, inst, i, b.alert_rec[a0 + i]);
}

// every instance's alerts in one launch (alert_off on the device gives each
// alert its instance); out[a] for a in [0, n_all)
__global__ void k_gather_alerts_all(DevBuffers b, DevConfig cfg, uint64_t n_all, cs_alert* out) {
  pdl_enter();
  const u64 a = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_all) return;
  uint32_t lo = 0, hi = b.n_inst;  // last instance with alert_off[inst] <= a
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (b.alert_off[mid] <= a) lo = mid;
    else hi = mid;
  }
  out[a] = make_alert(b, cfg, lo, a - b.alert_off[lo], b.alert_rec[a]);
}

void launch_gather_alerts_all(const DevBuffers& b, const DevConfig& cfg, uint64_t n_all, cs_alert* out,
                              cudaStream_t s) {
  if (!n_all) return;
  launch_pdl(k_gather_alerts_all, (unsigned)((n_all + 255) / 256), 256, 0, s, b, cfg, n_all, out);
}

void launch_gather_records(const DevBuffers& b, const DevConfig& cfg, uint32_t inst, uint64_t r0,
                           uint64_t nr, int scored, int det, cs_record* out, cudaStream_t s) {
  if (!nr) return;
  k_gather_records<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(b, cfg, inst, r0, nr, scored,
                                                                det, out);
}

void launch_gather_alerts(const DevBuffers& b, const DevConfig& cfg, uint32_t inst, uint64_t a0,
                          uint64_t na, cs_alert* out, cudaStream_t s) {
  if (!na) return;
  launch_pdl(k_gather_alerts, (unsigned)((na + 255) / 256), 256, 0, s, b, cfg, inst, a0, na, out);
}

// --------------------------------------------------- frequency fallback
// segment_by_frequency (cycles.cpp:283-343): rare path, exact arithmetic.
__global__ void k_gpu_kernel_extent(const cs_event* ev, uint64_t begin, uint64_t end,
                                    unsigned long long* out3) {
  // out3[0] count, out3[1] min start (as order-preserving u64), out3[2] max
  u64 cnt = 0, mn = ~0ull, mx = 0;
  for (u64 j = begin + (u64)blockIdx.x * blockDim.x + threadIdx.x; j < end;
       j += (u64)gridDim.x * blockDim.x) {
    const cs_event& e = ev[j];
    if (e.kind == CS_SPAN && e.category == CS_CAT_GPU_KERNEL) {
      ++cnt;
      const u64 key = (u64)e.start_ts ^ (1ull << 63);
      mn = key < mn ? key : mn;
      mx = key > mx ? key : mx;
    }
  }
  cnt = warp_sum_u64(cnt);
  for (int o = 16; o > 0; o >>= 1) {
    const u64 a = __shfl_xor_sync(0xffffffffu, mn, o), c = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = c > mx ? c : mx;
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(&out3[0], cnt);
    atomicMin(&out3[1], mn);
    atomicMax(&out3[2], mx);
  }
}

__global__ void k_freq_hist(const cs_event* ev, uint64_t begin, uint64_t end, int64_t t0,
                            int64_t bin_ns, uint64_t bins, unsigned long long* hist) {
  for (u64 j = begin + (u64)blockIdx.x * blockDim.x + threadIdx.x; j < end;
       j += (u64)gridDim.x * blockDim.x) {
    const cs_event& e = ev[j];
    if (e.kind == CS_SPAN && e.category == CS_CAT_GPU_KERNEL) {
      const u64 bi = (u64)((e.start_ts - t0) / bin_ns);
      if (bi < bins) atomicAdd(&hist[bi], 1ull);
    }
  }
}

__global__ void k_freq_center(const unsigned long long* hist, uint64_t bins, double* h) {
  // mean = (sum of integer counts, exact) / bins; h -= mean (cycles.cpp:301-304)
  __shared__ double s_mean;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (u64 i = 0; i < bins; ++i) m = __dadd_rn(m, (double)hist[i]);
    s_mean = __ddiv_rn(m, (double)bins);
  }
  __syncthreads();
  for (u64 i = threadIdx.x; i < bins; i += blockDim.x) h[i] = __dsub_rn((double)hist[i], s_mean);
}

__global__ void k_freq_autocorr(const double* h, uint64_t bins, double* acc) {
  // one thread per lag, the reference's sequential inner sum (310-317)
  const u64 lag = 1 + (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (lag > bins / 2) return;
  double a = 0.0;
  for (u64 i = 0; i + lag < bins; ++i) a = __dadd_rn(a, __dmul_rn(h[i], h[i + lag]));
  acc[lag] = a;
}

__global__ void k_freq_cycles(const cs_event* ev, uint64_t begin, uint64_t end, int64_t t0,
                              int64_t period, uint64_t n, uint64_t cyc_base, DevBuffers b,
                              uint32_t inst) {
  const u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const i64 s = t0 + (i64)c * period;
  const i64 e = s + period;
  auto lower = [&](i64 ts) {
    u64 lo = begin, hi = end;
    while (lo < hi) {
      const u64 mid = (lo + hi) >> 1;
      if (ev[mid].start_ts < ts) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  };
  const u64 g = cyc_base + c;
  b.c_start[g] = s;
  b.c_end[g] = e;
  b.c_apos[g] = ~0ull;
  b.c_aend[g] = s;
  b.c_first[g] = lower(s);
  b.c_last[g] = lower(e);
  b.c_inst[g] = inst;
}

constexpr int kFNamesSmem = 256;  // name infos staged in shared memory by the reduce

// ------------------------------------- K3'' thread-per-cycle reduce, v2
// One thread per cycle walks its events in order (the reference's own loops:
// cycles.cpp:157-166, 205-229, 256-281; rca.cpp:87-129) with one 256-bit
// load per 32-B record, kRedUnroll records in flight per thread.  The
// per-cycle accumulators (component durations, class occupancy, event-ordered
// collective beta) live in shared memory as [slot][thread] arrays: an update
// is one load/add/store whose bank depends only on the lane, and the cost per
// event no longer grows with the number of slots.
// Measured on B200 (configs[1]): an L2 bulk prefetch of the cycle's range,
// 8 records in flight (spills) and a warp-cooperative coalesced variant (2x
// the instructions: consecutive records of mixed kinds diverge) were all slower.
constexpr int kRedUnroll = 4;
__global__ void __launch_bounds__(256, 3) k_cycle_reduce_v2(DevBuffers b, DevConfig cfg, int do_beta) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned char s_red[];
  __shared__ uint32_t s_ninfo[kFNamesSmem];
  const int P = cfg.cyc.n_phases;
  const int C = do_beta ? cfg.cyc.n_beta_slots : 0;
  const int R = do_beta ? cfg.cyc.n_comm_slots : 0;
  const uint32_t NT = blockDim.x, tid = threadIdx.x;
  auto pack_info = [&](const cs_name_info& ni) -> uint32_t {
    const uint32_t ph = (ni.phase >= 0 && ni.phase < P) ? (uint32_t)ni.phase : 15u;
    const uint32_t bs = (ni.beta_slot >= 0 && ni.beta_slot < C) ? (uint32_t)ni.beta_slot : 255u;
    return ph | (bs << 4) | ((ni.flags & 3u) << 12);
  };
  for (uint32_t i = tid; i < b.n_names && i < (uint32_t)kFNamesSmem; i += NT)
    s_ninfo[i] = pack_info(b.names[i]);
  __syncthreads();
  // [slot][thread] accumulators, row stride SN = NT + 1: the per-event
  // updates (a thread's own column) and the transposed write-out below are
  // both (nearly) bank-conflict free
  const uint32_t SN = NT + 1;
  i64* comp = reinterpret_cast<i64*>(s_red);            // [P][SN]
  i64* beta = comp + (u64)P * SN;                       // [C][SN]
  double* coll = reinterpret_cast<double*>(beta + (u64)C * SN);  // [R][SN]
  i64* s_dur = reinterpret_cast<i64*>(coll + (u64)R * SN);       // [NT]
  uint32_t* colln = reinterpret_cast<uint32_t*>(s_dur + NT);     // [R][SN]
  const u64 g0 = (u64)blockIdx.x * NT;
  const u64 g = g0 + tid;
  const bool live = g < b.n_cycles;
  uint8_t stage = CS_STAGE_UNKNOWN;
  if (live) {
    const i64 cs = b.c_start[g], ce = b.c_end[g];
    const u64 first = b.c_first[g], last = b.c_last[g];
    const bool no_comp = b.c_apos[g] == kNone;  // frequency-fallback cycle (cycles.cpp:332-340)
    const i64 dur = ce - cs;
    s_dur[tid] = dur;
    for (int p = 0; p < P; ++p) comp[p * SN + tid] = 0;
    for (int c = 0; c < C; ++c) beta[c * SN + tid] = 0;
    for (int r = 0; r < R; ++r) {
      coll[r * SN + tid] = 0.0;
      colln[r * SN + tid] = 0u;
    }
    uint32_t fm_cls = 0, kw = 0;
    bool fm_found = false, batch_found = false;
    int32_t wl = -1;
    for (u64 j0 = first; j0 < last; j0 += kRedUnroll) {
      Ev8 e[kRedUnroll];
#pragma unroll
      for (int q = 0; q < kRedUnroll; ++q) {
        if (j0 + q < last) e[q] = ldg256(b.ev + j0 + q);
        else e[q].c = (u64)CS_FLOW << 32;  // ignored
      }
#pragma unroll
      for (int q = 0; q < kRedUnroll; ++q) {
        const uint32_t name = (uint32_t)e[q].c;
        const uint32_t kc = (uint32_t)(e[q].c >> 32);
        const uint32_t flags = kc >> 16;
        if (!fm_found && (flags & CS_EV_FM_MASK)) {
          fm_found = true;
          fm_cls = flags & CS_EV_FM_MASK;
        }
        if (!batch_found && (flags & CS_EV_HAS_BATCH)) {
          batch_found = true;
          wl = (flags & CS_EV_WL_OK) ? (int32_t)(uint32_t)e[q].d : -2;
        }
        if ((kc & 0xffu) != CS_SPAN) continue;
        const uint32_t info = name < (uint32_t)kFNamesSmem ? s_ninfo[name] : pack_info(b.names[name]);
        kw |= (info >> 12) & 3u;
        const i64 st = (i64)e[q].a, d = (i64)e[q].b;
        const i64 end = st + d;
        const i64 clipped = (end < ce ? end : ce) - st;
        if (clipped <= 0) continue;
        const uint32_t ph = info & 15u, bs = (info >> 4) & 255u;
        if (ph != 15u && !no_comp) comp[ph * SN + tid] += clipped;
        if (do_beta && d > 0) {
          if (bs != 255u) beta[bs * SN + tid] += clipped;
          if (((kc >> 8) & 0xffu) == CS_CAT_COLLECTIVE_COMM && (flags & CS_EV_HAS_COMM)) {
            const uint32_t slot = (uint32_t)(e[q].d >> 32);
            if (slot < (uint32_t)R) {
              coll[slot * SN + tid] =
                  __dadd_rn(coll[slot * SN + tid], __ddiv_rn((double)clipped, (double)dur));
              colln[slot * SN + tid] += 1u;
            }
          }
        }
      }
    }
    // classify_stages local signals (cycles.cpp:205-229)
    if (fm_cls == CS_EV_FM_PREFILL) stage = CS_STAGE_PREFILL;
    else if (fm_cls == CS_EV_FM_DECODE) stage = CS_STAGE_DECODE;
    const bool pkw = kw & CS_NAME_PREFILL_KW, dkw = kw & CS_NAME_DECODE_KW;
    if (stage == CS_STAGE_UNKNOWN && pkw != dkw) stage = pkw ? CS_STAGE_PREFILL : CS_STAGE_DECODE;
    b.c_local[g] = stage;
    b.c_stage[g] = stage;
    b.c_wl[g] = wl;
  }
  // the CTA's rows [g0, g0 + n_live) of every per-(cycle, slot) output are
  // contiguous: written cooperatively, consecutive threads on consecutive
  // addresses (a thread-per-row store would touch 32 partial sectors per
  // warp instruction)
  __syncthreads();
  {
    const uint32_t n_live = (uint32_t)(b.n_cycles - g0 < (u64)NT ? b.n_cycles - g0 : (u64)NT);
    for (uint32_t idx = tid; idx < n_live * (uint32_t)P; idx += NT) {
      const uint32_t lc = idx / (uint32_t)P, p = idx - lc * (uint32_t)P;
      b.c_comp[g0 * P + idx] = comp[p * SN + lc];
    }
    for (uint32_t idx = tid; idx < n_live * (uint32_t)C; idx += NT) {
      const uint32_t lc = idx / (uint32_t)C, c = idx - lc * (uint32_t)C;
      const i64 dur = s_dur[lc];
      const i64 t = dur > 0 ? beta[c * SN + lc] : 0;
      b.c_beta_tot[g0 * C + idx] = t;
    }
    for (uint32_t idx = tid; idx < n_live * (uint32_t)R; idx += NT) {
      const uint32_t lc = idx / (uint32_t)R, r = idx - lc * (uint32_t)R;
      b.c_coll[g0 * R + idx] = coll[r * SN + lc];
      const uint32_t n = colln[r * SN + lc];
      b.c_coll_n[g0 * R + idx] = (uint8_t)(n > 255u ? 255u : n);
    }
  }
  const bool unk = live && stage == CS_STAGE_UNKNOWN;
  const uint32_t inst = unk ? b.c_inst[g] : 0xffffffffu;
  const uint32_t grp = __match_any_sync(0xffffffffu, inst);
  if (unk && (tid & 31) == (uint32_t)(__ffs(grp) - 1)) {
    atomicAdd(&b.inst[inst].n_unknown, (u64)__popc(grp));
    *b.any_unknown = 1u;
  }
}

// ------------------------------ K3w thread-per-cycle reduce, any slot count
// The reference keys component durations by phase name, class occupancy by
// span name and collective beta by (name, commHash, rank) in std::maps
// (cycles.cpp:157-166, rca.cpp:85-115): no bound on their number.  When the
// shared-memory [slot][thread] accumulators of k_cycle_reduce_v2 do not fit
// (more than 15 phases or 254 classes, or rows too wide for >= 64 threads per
// CTA), each thread accumulates straight into its own (cycle, slot) rows of
// the outputs in global memory (zeroed before the launch; rows are private to
// the thread, so no atomics; L1/L2 absorb the read-modify-writes).  Same
// event loop, same arithmetic order; k_beta_finalize turns the totals into
// beta afterwards.
__global__ void __launch_bounds__(128) k_cycle_reduce_wide(DevBuffers b, DevConfig cfg, int do_beta) {
  const int P = cfg.cyc.n_phases;
  const int C = do_beta ? cfg.cyc.n_beta_slots : 0;
  const int R = do_beta ? cfg.cyc.n_comm_slots : 0;
  const u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= b.n_cycles) return;
  const i64 cs = b.c_start[g], ce = b.c_end[g];
  const u64 first = b.c_first[g], last = b.c_last[g];
  const bool no_comp = b.c_apos[g] == kNone;  // frequency-fallback cycle (cycles.cpp:332-340)
  const i64 dur = ce - cs;
  int64_t* comp = b.c_comp + g * (u64)P;
  int64_t* beta = b.c_beta_tot + g * (u64)C;
  double* coll = b.c_coll + g * (u64)R;
  uint8_t* colln = b.c_coll_n + g * (u64)R;
  uint32_t fm_cls = 0, kw = 0;
  bool fm_found = false, batch_found = false;
  int32_t wl = -1;
  for (u64 j0 = first; j0 < last; j0 += kRedUnroll) {
    Ev8 e[kRedUnroll];
#pragma unroll
    for (int q = 0; q < kRedUnroll; ++q) {
      if (j0 + q < last) e[q] = ldg256(b.ev + j0 + q);
      else e[q].c = (u64)CS_FLOW << 32;
    }
#pragma unroll
    for (int q = 0; q < kRedUnroll; ++q) {
      const uint32_t name = (uint32_t)e[q].c;
      const uint32_t kc = (uint32_t)(e[q].c >> 32);
      const uint32_t flags = kc >> 16;
      if (!fm_found && (flags & CS_EV_FM_MASK)) {
        fm_found = true;
        fm_cls = flags & CS_EV_FM_MASK;
      }
      if (!batch_found && (flags & CS_EV_HAS_BATCH)) {
        batch_found = true;
        wl = (flags & CS_EV_WL_OK) ? (int32_t)(uint32_t)e[q].d : -2;
      }
      if ((kc & 0xffu) != CS_SPAN) continue;
      const cs_name_info ni = b.names[name];
      kw |= ni.flags & 3u;
      const i64 st = (i64)e[q].a, d = (i64)e[q].b;
      const i64 end = st + d;
      const i64 clipped = (end < ce ? end : ce) - st;
      if (clipped <= 0) continue;
      if (ni.phase >= 0 && ni.phase < P && !no_comp) comp[ni.phase] += clipped;
      if (do_beta && d > 0) {
        if (ni.beta_slot >= 0 && ni.beta_slot < C) beta[ni.beta_slot] += clipped;
        if (((kc >> 8) & 0xffu) == CS_CAT_COLLECTIVE_COMM && (flags & CS_EV_HAS_COMM)) {
          const uint32_t slot = (uint32_t)(e[q].d >> 32);
          if (slot < (uint32_t)R) {
            coll[slot] = __dadd_rn(coll[slot], __ddiv_rn((double)clipped, (double)dur));
            if (colln[slot] < 255u) colln[slot] += 1u;
          }
        }
      }
    }
  }
  uint8_t stage = CS_STAGE_UNKNOWN;
  if (fm_cls == CS_EV_FM_PREFILL) stage = CS_STAGE_PREFILL;
  else if (fm_cls == CS_EV_FM_DECODE) stage = CS_STAGE_DECODE;
  const bool pkw = kw & CS_NAME_PREFILL_KW, dkw = kw & CS_NAME_DECODE_KW;
  if (stage == CS_STAGE_UNKNOWN && pkw != dkw) stage = pkw ? CS_STAGE_PREFILL : CS_STAGE_DECODE;
  b.c_local[g] = stage;
  b.c_stage[g] = stage;
  b.c_wl[g] = wl;
  if (stage == CS_STAGE_UNKNOWN) {
    atomicAdd(&b.inst[b.c_inst[g]].n_unknown, 1ull);
    *b.any_unknown = 1u;
  }
}

// class totals of the wide reduce masked to cycles with a positive duration
// (rca.cpp:95-96, 119-121); beta = total / duration is formed on read
__global__ void k_beta_finalize(DevBuffers b, int C) {
  const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= b.n_cycles * (u64)C) return;
  const u64 g = k / (u64)C;
  const i64 dur = b.c_end[g] - b.c_start[g];
  const i64 t = dur > 0 ? b.c_beta_tot[k] : 0;
  b.c_beta_tot[k] = t;
}

// ---------------------------------------------------- wire-format expand
// Columnar wire records -> canonical 32-B cs_event in HBM, one CTA per
// instance-aligned block (= tile), 4 consecutive events per thread: each
// thread decodes its events' dictionary codes (dictionary in shared memory)
// and counts their entries in the duration / payload / value / long-delta /
// escape columns; two block-wide exclusive scans (16-bit counts packed in
// u64s) give their column positions, and a segmented scan of the start_ts
// deltas (restarted at escaped records, which are copied whole) gives the
// timestamps.
constexpr int kWireThreads = 256;
__global__ void __launch_bounds__(kWireThreads) k_wire_expand(WireDev w, const uint64_t* __restrict__ tile_begin,
                                                              const uint64_t* __restrict__ tile_end,
                                                              cs_event* __restrict__ out) {
  __shared__ u64 s_w[32];
  __shared__ uint32_t s_dict[128];
  __shared__ i64 s_x[kWireThreads];
  __shared__ i64 s_wx[32];
  __shared__ uint8_t s_wf[32];
  const uint32_t t = blockIdx.x;
  if (threadIdx.x < 128) s_dict[threadIdx.x] = threadIdx.x < w.n_dict ? w.dict[threadIdx.x] : 0u;
  const u64 tb = tile_begin[t], te = tile_end[t];
  const cs_wire_block& B = w.blocks[t];
  const i64 b0 = B.base_ts;
  const uint32_t batch_base = B.batch_base;
  const u64 j0 = tb + 4u * threadIdx.x;
  uint32_t code[4], dtl[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool in = j0 + q < te;
    code[q] = in ? (uint32_t)__ldg(w.codes + j0 + q) : (uint32_t)CS_WIRE_ESCAPE;
    dtl[q] = in ? (uint32_t)__ldg(w.dt_lo + j0 + q) : 0u;
  }
  __syncthreads();  // s_dict
  uint32_t info[4];
  u64 ca = 0, cb = 0;  // [dur, pay8, pay16, val] and [dt_hi, esc], 16 bits each
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    info[q] = 0;
    if (j0 + q >= te) continue;
    const uint32_t c = code[q] & 0x7fu;
    if (c == CS_WIRE_ESCAPE) {
      cb += 1ull << 16;
      continue;
    }
    info[q] = s_dict[c];
    const uint32_t kind = (info[q] >> 16) & 15u, flags = (info[q] >> 24) & 0x3fu;
    const bool pay = (flags & (CS_EV_HAS_BATCH | CS_EV_HAS_COMM)) != 0;
    ca += (kind == CS_SPAN ? 1ull : 0ull) + (pay ? ((info[q] & CS_WIRE_WIDE) ? (1ull << 32) : (1ull << 16)) : 0ull) +
          ((kind == CS_COUNTER && (flags & CS_EV_HAS_VALUE)) ? (1ull << 48) : 0ull);
    cb += (code[q] & CS_WIRE_LONG_DT) ? 1ull : 0ull;
  }
  const u64 xa = block_incl_scan(ca, s_w, nullptr) - ca;
  __syncthreads();  // s_w reuse
  const u64 xb = block_incl_scan(cb, s_w, nullptr) - cb;
  u64 dpos = B.dur + (xa & 0xffffull);
  u64 p8 = B.pay8 + ((xa >> 16) & 0xffffull);
  u64 p16 = B.pay16 + ((xa >> 32) & 0xffffull);
  u64 vpos = B.val + (xa >> 48);
  u64 hpos = B.dt_hi + (xb & 0xffffull);
  u64 epos = B.esc + (xb >> 16);
  // full deltas (low 16 bits + the high byte of long ones)
  {
    u64 h = hpos;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (j0 + q < te && (code[q] & 0x7fu) != CS_WIRE_ESCAPE && (code[q] & CS_WIRE_LONG_DT))
        dtl[q] |= (uint32_t)__ldg(w.dt_hi + h++) << 16;
  }
  // start_ts: a segmented prefix sum of the deltas, restarted at each escaped
  // event's absolute start_ts (the aggregate (f, x) of a run: f = it holds an
  // escape, x = offset from b0 after it)
  uint8_t f = 0;
  i64 x = 0;
  {
    u64 e = epos;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (j0 + q >= te) break;
      if ((code[q] & 0x7fu) == CS_WIRE_ESCAPE) {
        f = 1;
        x = w.escapes[e++].start_ts - b0;
      } else {
        x += (i64)dtl[q];
      }
    }
  }
  {
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const i64 yx = __shfl_up_sync(0xffffffffu, x, o);
      const uint32_t yf = __shfl_up_sync(0xffffffffu, (uint32_t)f, o);
      if (lane >= o) {
        if (!f) x += yx;
        f |= (uint8_t)yf;
      }
    }
    if (lane == 31) s_wx[wp] = x, s_wf[wp] = f;
    __syncthreads();
    if (wp == 0) {
      constexpr int kW = kWireThreads / 32;
      i64 px = lane < kW ? s_wx[lane] : 0;
      uint32_t pf = lane < kW ? s_wf[lane] : 0u;
      for (int o = 1; o < kW; o <<= 1) {
        const i64 yx = __shfl_up_sync(0xffffffffu, px, o);
        const uint32_t yf = __shfl_up_sync(0xffffffffu, pf, o);
        if (lane >= o) {
          if (!pf) px += yx;
          pf |= yf;
        }
      }
      if (lane < kW) s_wx[lane] = px, s_wf[lane] = (uint8_t)pf;
    }
    __syncthreads();
    if (wp > 0 && !f) x += s_wx[wp - 1];
    s_x[threadIdx.x] = x;  // inclusive
    __syncthreads();
  }
  i64 run = threadIdx.x ? s_x[threadIdx.x - 1] : 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (j0 + q >= te) break;
    u64 a, d, c, p;
    if ((code[q] & 0x7fu) == CS_WIRE_ESCAPE) {
      const cs_event& e = w.escapes[epos++];
      run = e.start_ts - b0;
      a = (u64)e.start_ts;
      d = (u64)e.duration;
      c = (u64)e.name_id | ((u64)e.kind << 32) | ((u64)e.category << 40) | ((u64)e.flags << 48);
      p = e.payload;
    } else {
      run += (i64)dtl[q];
      const uint32_t name = info[q] & 0xffffu, kind = (info[q] >> 16) & 15u;
      const uint32_t cat = (info[q] >> 20) & 15u, flags = (info[q] >> 24) & 0x3fu;
      a = (u64)(b0 + run);
      d = 0;
      if (kind == CS_SPAN) {
        d = (u64)w.dur_lo[dpos] | ((u64)w.dur_hi[dpos] << 16);
        ++dpos;
      } else if (kind == CS_COUNTER && (flags & CS_EV_HAS_VALUE)) {
        d = (u64)__double_as_longlong(w.values[vpos++]);
      }
      p = 0;
      if (flags & (CS_EV_HAS_COMM | CS_EV_HAS_BATCH)) {
        const uint32_t v = (info[q] & CS_WIRE_WIDE) ? (uint32_t)w.pay16[p16++] : (uint32_t)w.pay8[p8++];
        p = (flags & CS_EV_HAS_COMM) ? (u64)v << 32 : (u64)(v + batch_base);
      }
      c = (u64)name | ((u64)kind << 32) | ((u64)cat << 40) | ((u64)flags << 48);
    }
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(out + j0 + q), "l"(a), "l"(d),
                 "l"(c), "l"(p)
                 : "memory");
  }
}

// workload table from u32 triples (0xffffffff = absent -> INT64_MIN)
__global__ void k_wl32_expand(const uint32_t* __restrict__ wl32, uint64_t n, cs_workload* __restrict__ out) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto dec = [](uint32_t v) -> int64_t { return v == 0xffffffffu ? INT64_MIN : (int64_t)v; };
  out[i] = cs_workload{dec(wl32[3 * i]), dec(wl32[3 * i + 1]), dec(wl32[3 * i + 2])};
}

void launch_wl32_expand(const uint32_t* wl32, uint64_t n, cs_workload* out, cudaStream_t s) {
  if (n) k_wl32_expand<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(wl32, n, out);
}

void launch_wire_expand(const WireDev& w, const uint64_t* tile_begin, const uint64_t* tile_end,
                        uint32_t n_tiles, cs_event* out, cudaStream_t s) {
  if (!n_tiles) return;
  k_wire_expand<<<n_tiles, kWireThreads, 0, s>>>(w, tile_begin, tile_end, out);
}

// Streaming: per instance, the position (relative to the instance's first
// uploaded event) from which events are carried into the next micro-batch:
// the last closed cycle's end group start (cycles.cpp:147 drops the trailing
// partial cycle; it is completed by the next batch).
// per instance: where its carried tail starts (the last closed cycle's end,
// cycles.cpp:147) and, in keep[n_inst + i], the anchor occurrences in that
// tail (the next micro-batch's host-side sizing starts from them)
__global__ void __launch_bounds__(128) k_stream_keep(DevBuffers b, uint64_t* keep) {
  pdl_enter();
  const uint32_t i = blockIdx.x * 4 + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (i >= b.n_inst) return;
  const u64 c0 = b.cyc_off[i], c1 = b.cyc_off[i + 1];
  const u64 k = c1 > c0 ? b.c_last[c1 - 1] - b.inst_off[i] : 0;
  const uint32_t anchor = b.inst[i].anchor;
  u64 n = 0;
  if (anchor != 0xffffffffu)
    for (u64 p = b.inst_off[i] + k + lane; p < b.inst_off[i + 1]; p += 32)
      n += (b.ev[p].kind == CS_SPAN && b.ev[p].name_id == anchor) ? 1ull : 0ull;
  n = warp_sum_u64(n);
  if (lane == 0) {
    keep[i] = k;
    keep[b.n_inst + i] = n;
  }
}

// one CTA per instance: its carried tail (from the previous batch's buffer)
// followed by its new events, 16 bytes per lane-step
__global__ void __launch_bounds__(128) k_stream_assemble(const cs_event* __restrict__ prev,
                                                         const cs_event* __restrict__ fresh,
                                                         const uint64_t* __restrict__ meta, uint64_t total,
                                                         uint32_t n_inst, cs_event* __restrict__ out) {
  pdl_enter();
  const uint32_t i = blockIdx.x;
  const u64 dst = meta[4 * i], ts = meta[4 * i + 1], tl = meta[4 * i + 2], ns = meta[4 * i + 3];
  const u64 end = i + 1 < n_inst ? meta[4 * (i + 1)] : total;
  const uint4* p4 = reinterpret_cast<const uint4*>(prev + ts);
  const uint4* f4 = reinterpret_cast<const uint4*>(fresh + ns);
  uint4* o4 = reinterpret_cast<uint4*>(out + dst);
  const u64 n2 = 2 * (end - dst), t2 = 2 * tl;  // 16-B halves of 32-B records
  for (u64 k = threadIdx.x; k < n2; k += blockDim.x) o4[k] = k < t2 ? p4[k] : f4[k - t2];
}

void launch_stream_assemble(const cs_event* prev, const cs_event* fresh, const uint64_t* meta,
                            uint32_t n_inst, uint64_t total, cs_event* out, cudaStream_t s) {
  if (n_inst) launch_pdl(k_stream_assemble, n_inst, 128, 0, s, prev, fresh, meta, total, n_inst, out);
}

// anchor occurrences among each instance's NEW events of a micro-batch (warp
// per instance; meta as for k_stream_assemble, anchor ids per instance)
__global__ void __launch_bounds__(128) k_stream_count(const cs_event* __restrict__ fresh,
                                                      const uint64_t* __restrict__ meta,
                                                      const uint32_t* __restrict__ anchor, uint32_t n_inst,
                                                      uint64_t n_new, uint64_t* out) {
  pdl_enter();
  const uint32_t i = blockIdx.x * 4 + (threadIdx.x >> 5);
  const uint32_t lane = threadIdx.x & 31;
  if (i >= n_inst) return;
  const u64 b0 = meta[4 * i + 3], b1 = i + 1 < n_inst ? meta[4 * (i + 1) + 3] : n_new;
  const uint32_t a = anchor[i];
  u64 n = 0;
  for (u64 p = b0 + lane; p < b1; p += 32) n += (fresh[p].kind == CS_SPAN && fresh[p].name_id == a) ? 1ull : 0ull;
  n = warp_sum_u64(n);
  if (lane == 0) out[i] = n;
}

void launch_stream_count(const cs_event* fresh, const uint64_t* meta, const uint32_t* anchor, uint32_t n_inst,
                         uint64_t n_new, uint64_t* out, cudaStream_t s) {
  if (n_inst) launch_pdl(k_stream_count, (n_inst + 3) / 4, 128, 0, s, fresh, meta, anchor, n_inst, n_new, out);
}

void launch_stream_keep(const DevBuffers& b, uint64_t* keep, cudaStream_t s) {
  if (b.n_inst) launch_pdl(k_stream_keep, (b.n_inst + 3) / 4, 128, 0, s, b, keep);
}

// ------------------------------------------- counter-weighted mu (§8f #1)
// CounterTable::from_trace (trace.cpp:111-131): per (instance, metric) the
// Counter events with a numeric value, stable-sorted by ts = their canonical
// event order.  Compacted here by metric: k_counter_count counts per (metric,
// tile), an exclusive scan over [metric][tile] gives offsets, and
// k_counter_scatter writes (ts, value) in event order.  Instance i's series
// for metric m is [m_off[m*nt + first_tile(i)], m_off[m*nt + first_tile(i+1)]).
__device__ __forceinline__ int counter_slot(const DevBuffers& b, const Ev8& e) {
  const uint32_t kc = (uint32_t)(e.c >> 32);
  if ((kc & 0xffu) != CS_COUNTER || !((kc >> 16) & CS_EV_HAS_VALUE)) return -1;
  const uint32_t name = (uint32_t)e.c;
  return name < b.n_names ? (int)b.series_slot[name] : -1;
}

__global__ void __launch_bounds__(256) k_counter_count(DevBuffers b) {
  __shared__ uint32_t s_cnt[8][kMaxMetrics];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 t = (u64)blockIdx.x * 8 + warp;
  if (lane < kMaxMetrics) s_cnt[warp][lane] = 0;
  __syncwarp();
  if (t >= b.n_tiles) return;
  const u64 tb = b.tile_begin[t], te = b.tile_end[t];
  for (u64 j0 = tb; j0 < te; j0 += 32) {
    const u64 j = j0 + lane;
    const int m = j < te ? counter_slot(b, ldg256(b.ev + j)) : -1;
    const uint32_t grp = __match_any_sync(0xffffffffu, m);
    if (m >= 0 && lane == __ffs(grp) - 1) s_cnt[warp][m] += __popc(grp);
    __syncwarp();
  }
  if (lane < (int)b.n_metrics) b.m_off[(u64)lane * b.n_tiles + t] = s_cnt[warp][lane];
}

__global__ void __launch_bounds__(256) k_counter_scatter(DevBuffers b) {
  __shared__ uint32_t s_run[8][kMaxMetrics];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u64 t = (u64)blockIdx.x * 8 + warp;
  if (lane < kMaxMetrics) s_run[warp][lane] = 0;
  __syncwarp();
  if (t >= b.n_tiles) return;
  const u64 tb = b.tile_begin[t], te = b.tile_end[t];
  for (u64 j0 = tb; j0 < te; j0 += 32) {
    const u64 j = j0 + lane;
    Ev8 e{};
    int m = -1;
    if (j < te) {
      e = ldg256(b.ev + j);
      m = counter_slot(b, e);
    }
    const uint32_t grp = __match_any_sync(0xffffffffu, m);
    if (m >= 0) {
      const u64 pos = b.m_off[(u64)m * b.n_tiles + t] + s_run[warp][m] + __popc(grp & lanemask_lt());
      b.s_ts[pos] = (i64)e.a;
      b.s_val[pos] = __longlong_as_double((long long)e.b);  // the f64 `value` (cs_event.duration)
    }
    __syncwarp();
    if (m >= 0 && lane == __ffs(grp) - 1) s_run[warp][m] += __popc(grp);
    __syncwarp();
  }
}

// First index h in [0, n] with (double)ts[h] >= t (strict: > t), found by
// galloping from `hint` and finishing with a binary search.  The answer is
// unique (ts is sorted), so the hint only changes how many loads it takes.
__device__ __forceinline__ u64 search_from(const int64_t* __restrict__ ts, u64 n, double t, bool strict,
                                           u64 hint) {
  auto at_or_after = [&](u64 i) {
    const double x = (double)ts[i];
    return strict ? x > t : x >= t;
  };
  u64 lo, hi;  // the answer is in [lo, hi]; hi == n or at_or_after(hi)
  if (hint >= n || at_or_after(hint)) {
    hi = hint < n ? hint : n;
    u64 step = 1;
    while (true) {
      if (hi < step) {
        lo = 0;
        break;
      }
      const u64 c = hi - step;
      if (at_or_after(c)) {
        hi = c;
        step <<= 1;
      } else {
        lo = c + 1;
        break;
      }
    }
  } else {
    lo = hint + 1;
    u64 step = 1;
    while (true) {
      const u64 c = lo + step - 1;
      if (c >= n) {
        hi = n;
        break;
      }
      if (at_or_after(c)) {
        hi = c;
        break;
      }
      lo = c + 1;
      step <<= 1;
    }
  }
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (at_or_after(mid)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// interpolate_mean (rca.cpp:17-53), operation for operation: knots t0, the
// sample timestamps strictly inside (t0, t1), t1; trapezoids summed in knot
// order; value_at by lower_bound over the samples' double timestamps.  Every
// search starts from `*hint` (the previous span's first interior knot of this
// metric), which moves to this span's.
__device__ double interpolate_mean_dev(const int64_t* __restrict__ ts, const double* __restrict__ val,
                                       u64 n, i64 t0i, i64 t1i, u64* hint) {
  const double t0 = (double)t0i, t1 = (double)t1i;
  auto value_at = [&](double t, u64 near) -> double {
    if (t <= (double)ts[0]) return val[0];
    if (t >= (double)ts[n - 1]) return val[n - 1];
    const u64 h = search_from(ts, n, t, false, near);
    const double f = __ddiv_rn(__dsub_rn(t, (double)ts[h - 1]), (double)(ts[h] - ts[h - 1]));
    return __dadd_rn(val[h - 1], __dmul_rn(f, __dsub_rn(val[h], val[h - 1])));
  };
  // interior knots: samples with t0 < (double)ts < t1, a contiguous range
  const u64 k0 = search_from(ts, n, t0, true, *hint);
  const u64 k1 = search_from(ts, n, t1, false, k0);
  *hint = k0;
  double integral = 0.0, a = t0, va = value_at(t0, k0);
  for (u64 i = k0; i < k1; ++i) {
    const double kt = (double)ts[i], vb = value_at(kt, i);
    integral = __dadd_rn(integral, __dmul_rn(__dmul_rn(0.5, __dadd_rn(va, vb)), __dsub_rn(kt, a)));
    a = kt;
    va = vb;
  }
  const double vb = value_at(t1, k1);
  integral = __dadd_rn(integral, __dmul_rn(__dmul_rn(0.5, __dadd_rn(va, vb)), __dsub_rn(t1, a)));
  return __ddiv_rn(integral, __dsub_rn(t1, t0));
}

// cycle_stats' mu branch (rca.cpp:97-106, 123-126), one thread per cycle in
// event order: weighted_mu[class] += interpolate_mean(series, start,
// clipped_end) * overlap; mu = weighted_mu / total overlap (the beta totals).
__global__ void __launch_bounds__(256) k_cycle_mu(DevBuffers b, DevConfig cfg) {
  extern __shared__ __align__(16) unsigned char s_mu[];
  const int C = cfg.cyc.n_beta_slots;
  const uint32_t NT = blockDim.x, tid = threadIdx.x, SN = NT + 1;
  double* acc = reinterpret_cast<double*>(s_mu);  // [C][SN]
  u64* s_has = reinterpret_cast<u64*>(acc + (u64)C * SN);  // [NT]
  const u64 g0 = (u64)blockIdx.x * NT;
  const u64 g = g0 + tid;
  const bool live = g < b.n_cycles;
  for (int c = 0; c < C; ++c) acc[c * SN + tid] = 0.0;
  u64 has = 0;
  if (live) {
    const i64 cs = b.c_start[g], ce = b.c_end[g];
    const i64 dur = ce - cs;
    const u64 first = b.c_first[g], last = b.c_last[g];
    const uint32_t inst = b.c_inst[g];
    const uint32_t ft = b.inst_first_tile[inst];
    const uint32_t lt = inst + 1 < b.n_inst ? b.inst_first_tile[inst + 1] : b.n_tiles;
    u64 hint[kMaxMetrics];  // per metric: where the previous span's knots started
    for (int m = 0; m < kMaxMetrics; ++m) hint[m] = ~0ull;
    if (dur > 0) {  // cycle_stats returns empty stats otherwise (rca.cpp:77)
      for (u64 j = first; j < last; ++j) {
        const Ev8 e = ldg256(b.ev + j);
        const uint32_t kc = (uint32_t)(e.c >> 32);
        const i64 st = (i64)e.a, d = (i64)e.b;
        if ((kc & 0xffu) != CS_SPAN || d <= 0) continue;
        const i64 end = st + d;
        const i64 clipped = (end < ce ? end : ce) - st;
        if (clipped <= 0) continue;
        const uint32_t name = (uint32_t)e.c;
        const int m = b.class_metric[name];
        const int bs = b.names[name].beta_slot;
        if (m < 0 || bs < 0 || bs >= C) continue;
        const u64 lo = b.m_off[(u64)m * b.n_tiles + ft], hi = b.m_off[(u64)m * b.n_tiles + lt];
        if (hi <= lo) continue;  // counters.find(metric) == nullptr: beta-only entry
        u64& h = hint[m];
        if (h == ~0ull) h = (hi - lo) >> 1;
        const double mu = interpolate_mean_dev(b.s_ts + lo, b.s_val + lo, hi - lo, st, st + clipped, &h);
        acc[bs * SN + tid] = __dadd_rn(acc[bs * SN + tid], __dmul_rn(mu, (double)clipped));
        has |= 1ull << bs;
      }
    }
  }  // live
  s_has[tid] = has;
  __syncthreads();
  // the CTA's rows written cooperatively (consecutive threads, consecutive addresses)
  const uint32_t n_live = (uint32_t)(b.n_cycles - g0 < (u64)NT ? b.n_cycles - g0 : (u64)NT);
  for (uint32_t idx = tid; idx < n_live * (uint32_t)C; idx += NT) {
    const uint32_t lc = idx / (uint32_t)C, c = idx - lc * (uint32_t)C;
    const i64 tot = b.c_beta_tot[g0 * C + idx];
    const bool h = ((s_has[lc] >> c) & 1ull) && tot > 0;
    b.c_mu[g0 * C + idx] = h ? __ddiv_rn(acc[c * SN + lc], (double)tot) : 0.0;
    b.c_mu_has[g0 * C + idx] = h ? 1 : 0;
  }
}

void launch_counter_series(const DevBuffers& b, cudaStream_t s, uint64_t* launches) {
  if (!b.n_tiles || !b.n_metrics) return;
  k_counter_count<<<(unsigned)((b.n_tiles + 7) / 8), 256, 0, s>>>(b);
  const u64 n = (u64)b.n_metrics * b.n_tiles;
  launch_exclusive_scan(b.m_off, n, b.m_off + n, b.scan_tmp, s, launches);
  ++*launches;
}
void launch_counter_scatter(const DevBuffers& b, cudaStream_t s, uint64_t* launches) {
  if (!b.n_tiles || !b.n_metrics) return;
  k_counter_scatter<<<(unsigned)((b.n_tiles + 7) / 8), 256, 0, s>>>(b);
  ++*launches;
}
void launch_cycle_mu(const DevBuffers& b, const DevConfig& cfg, cudaStream_t s, uint64_t* launches) {
  if (!b.n_cycles) return;
  int nt = 256;
  const int C = cfg.cyc.n_beta_slots > 0 ? cfg.cyc.n_beta_slots : 1;
  while (nt > 32 && nt * C * 8 > 96 * 1024) nt >>= 1;
  const int smem = (nt + 1) * C * 8 + nt * 8;  // padded [class][thread] rows + has masks
  ensure_smem((const void*)k_cycle_mu, smem);
  k_cycle_mu<<<(unsigned)((b.n_cycles + nt - 1) / nt), nt, smem, s>>>(b, cfg);
  ++*launches;
}

// ------------------------------------------------------------ launchers
// tile boundaries of the K0 check: a tile's first start_ts is not below the
// previous tile's last within the same instance
__global__ void k_tile_order(DevBuffers b) {
  pdl_enter();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0 || t >= b.n_tiles) return;
  const uint32_t inst = b.tile_inst[t];
  if (b.tile_inst[t - 1] != inst) return;
  if (b.ev[b.tile_begin[t]].start_ts < b.ev[b.tile_end[t - 1] - 1].start_ts)
    atomicOr(&b.inst[inst].unsorted, 1u);
}

void launch_tile_order(const DevBuffers& b, cudaStream_t s, uint64_t* launches) {
  if (b.n_tiles < 2) return;
  launch_pdl(k_tile_order, (b.n_tiles + 255) / 256, 256, 0, s, b);
  ++*launches;
}

void launch_scan_events(const DevBuffers& b, const DevConfig&, int mode, bool sample,
                        const uint32_t* list, uint32_t n_list, cudaStream_t s,
                        uint64_t* launches) {
  if (n_list == 0) return;
  if (sample) n_list *= kSampleSplit;
  const int sms = sm_count();
  int per_sm = blocks_per_sm((const void*)k_scan_warp, kScanWarpThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const uint32_t warps = kScanWarpThreads / 32;
  uint32_t grid = (uint32_t)sms * (uint32_t)per_sm;
  const uint32_t need = (n_list + warps - 1) / warps;
  if (need < grid) grid = need;
  launch_pdl(k_scan_warp, grid, kScanWarpThreads, 0, s, b, mode, list, n_list, sample ? 1 : 0);
  ++*launches;
}

void launch_cycle_reduce_tpc(const DevBuffers& b, const DevConfig& cfg, int do_beta,
                             cudaStream_t s, uint64_t* launches, int variant) {
  if (!b.n_cycles) return;
  const int P = cfg.cyc.n_phases;
  const int C = do_beta ? cfg.cyc.n_beta_slots : 0;
  const int R = do_beta ? cfg.cyc.n_comm_slots : 0;
  const int per_thread = (P + C + R) * 8 + R * 4;
  int nt = 256;
  while (nt > 64 && (nt + 1) * per_thread + nt * 8 > 100 * 1024) nt >>= 1;
  const int smem = (nt + 1) * per_thread + nt * 8;  // padded [slot][thread] rows + durations
  (void)variant;
  if (P > 15 || C > 254 || smem > 100 * 1024) {
    // more slots than the shared-memory accumulators hold: global-memory rows
    const u64 nc = b.n_cycles;
    if (P) cudaMemsetAsync(b.c_comp, 0, nc * (u64)P * sizeof(int64_t), s);
    if (C) cudaMemsetAsync(b.c_beta_tot, 0, nc * (u64)C * sizeof(int64_t), s);
    if (R) {
      cudaMemsetAsync(b.c_coll, 0, nc * (u64)R * sizeof(double), s);
      cudaMemsetAsync(b.c_coll_n, 0, nc * (u64)R, s);
    }
    k_cycle_reduce_wide<<<(unsigned)((nc + 127) / 128), 128, 0, s>>>(b, cfg, do_beta);
    ++*launches;
    if (C) {
      const u64 n = nc * (u64)C;
      k_beta_finalize<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(b, C);
      ++*launches;
    }
    return;
  }
  ensure_smem((const void*)k_cycle_reduce_v2, smem);
  const unsigned grid = (unsigned)((b.n_cycles + nt - 1) / nt);
  launch_pdl(k_cycle_reduce_v2, grid, nt, smem, s, b, cfg, do_beta);
  ++*launches;
}

void launch_tile_prefix(const DevBuffers& b, cudaStream_t s, uint64_t* launches) {
  cudaMemcpyAsync(b.tile_pref, b.tile_cnt, (size_t)b.n_tiles * sizeof(uint64_t),
                  cudaMemcpyDeviceToDevice, s);
  launch_exclusive_scan(b.tile_pref, b.n_tiles, b.tile_pref + b.n_tiles, b.scan_tmp, s, launches);
  launch_pdl(k_inst_anchor_counts, (b.n_inst + 255) / 256, 256, 0, s, b);
  *launches += 1;
}

void launch_rank(const DevBuffers& b, const DevConfig& cfg, int final_pass, cudaStream_t s,
                 uint64_t* launches) {
  if (b.n_inst == 0) return;
  launch_pdl(k_rank, b.n_inst, 32, 0, s, b, cfg, final_pass);
  ++*launches;
}

void launch_fold(const DevBuffers& b, const DevConfig&, const uint32_t* pi, const uint32_t* pn,
                 uint32_t n_pairs, double* out, cudaStream_t s, uint64_t* launches) {
  if (!n_pairs) return;
  k_fold<<<(n_pairs * 32 + 127) / 128, 128, 0, s>>>(b, pi, pn, n_pairs, out);
  ++*launches;
}

void launch_bounds(const DevBuffers& b, cudaStream_t s, uint64_t* launches) {
  if (!b.n_cycles) return;
  if (!b.n_tiles) return;
  launch_pdl(k_bounds_tile, (unsigned)((b.n_tiles + 7) / 8), 256, 0, s, b);
  ++*launches;
}

// ------------------------------------------- K4' parallel stage heuristic
// classify_stages' trailing-window heuristic (cycles.cpp:190-254) in parallel.
// The cycle slots are cut into chunks of kStageChunk; a warp runs the
// reference's sequential loop over its chunk (windows = sorted arrays + FIFO
// rings in shared memory, exact medians) after rebuilding the windows at the
// chunk start from the stages of the cycles before it.  Those stages are
// speculated (Unknown cycles count as non-Prefill, i.e. the local stage) and
// refined by Jacobi iteration: iteration k reads the stages of iteration k-1
// and recomputes only chunks whose look-back region changed Prefill-ness.
// Stages depend only on earlier cycles, so iteration k makes at least the
// first k chunks exact and the fixed point is the sequential result.  One
// persistent grid, a grid barrier between iterations.
constexpr int kStageChunk = (int)kStageChunkCycles;
constexpr int kStageWarps = 4;

struct Win {  // one trailing window in the warp's shared memory
  double* sorted;
  double* ring;
  uint32_t n, head, cap;
};

__device__ __forceinline__ void win_insert(Win& w, double x) {
  const int lane = threadIdx.x & 31;
  uint32_t cnt = 0;
  for (uint32_t i = lane; i < w.n; i += 32) cnt += w.sorted[i] <= x ? 1u : 0u;
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  const uint32_t p = cnt;
  for (int64_t base = (int64_t)w.n - 1; base >= (int64_t)p; base -= 32) {
    const int64_t idx = base - lane;
    double v = 0.0;
    if (idx >= (int64_t)p) v = w.sorted[idx];
    __syncwarp();
    if (idx >= (int64_t)p) w.sorted[idx + 1] = v;
    __syncwarp();
  }
  if (lane == 0) w.sorted[p] = x;
  __syncwarp();
  ++w.n;
}

__device__ __forceinline__ void win_remove(Win& w, double y) {
  const int lane = threadIdx.x & 31;
  uint32_t q = w.n;
  for (uint32_t base = 0; base < w.n && q == w.n; base += 32) {
    const uint32_t i = base + lane;
    const uint32_t m = __ballot_sync(0xffffffffu, i < w.n && w.sorted[i] == y);
    if (m) q = base + __ffs(m) - 1;
  }
  for (uint32_t base = q; base + 1 < w.n; base += 32) {
    const uint32_t idx = base + 1 + lane;
    double v = 0.0;
    if (idx < w.n) v = w.sorted[idx];
    __syncwarp();
    if (idx < w.n) w.sorted[idx - 1] = v;
    __syncwarp();
  }
  --w.n;
}

// push_back + pop_front beyond the capacity (cycles.cpp:245-249)
__device__ __forceinline__ void win_push(Win& w, double x) {
  const int lane = threadIdx.x & 31;
  if (w.n == w.cap) {
    const double oldest = w.ring[w.head];
    __syncwarp();  // every lane has read the slot lane 0 overwrites below
    win_remove(w, oldest);
    w.head = w.head + 1 == w.cap ? 0 : w.head + 1;
  }
  uint32_t tail = w.head + w.n;
  if (tail >= w.cap) tail -= w.cap;
  if (lane == 0) w.ring[tail] = x;
  __syncwarp();
  win_insert(w, x);
}

// median of the sorted window (cycles.cpp:181-186)
__device__ __forceinline__ double win_median(const Win& w) {
  const uint32_t n = w.n;
  if (n % 2 == 1) return w.sorted[n / 2];
  return __dmul_rn(0.5, __dadd_rn(w.sorted[n / 2 - 1], w.sorted[n / 2]));
}

// The same trailing window held in registers when it fits a warp (W <= 32):
// lane k holds the k-th smallest value (lanes < n) and the k-th ring slot.
// Insert / remove are one ballot and one shuffle; no shared memory, no
// warp barriers.
struct RegWin {
  double v, ring;
  uint32_t n, head, cap;
};

__device__ __forceinline__ void win_insert(RegWin& w, double x) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t p = __popc(__ballot_sync(0xffffffffu, lane < w.n && w.v <= x));
  const double pv = __shfl_up_sync(0xffffffffu, w.v, 1);
  if (lane > p && lane <= w.n) w.v = pv;
  if (lane == p) w.v = x;
  ++w.n;
}

__device__ __forceinline__ void win_remove(RegWin& w, double y) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t m = __ballot_sync(0xffffffffu, lane < w.n && w.v == y);
  const uint32_t p = (uint32_t)__ffs(m) - 1u;
  const double nx = __shfl_down_sync(0xffffffffu, w.v, 1);
  if (lane >= p && lane + 1 < w.n) w.v = nx;
  --w.n;
}

__device__ __forceinline__ void win_push(RegWin& w, double x) {
  const uint32_t lane = threadIdx.x & 31;
  if (w.n == w.cap) {
    const double oldest = __shfl_sync(0xffffffffu, w.ring, w.head);
    win_remove(w, oldest);
    if (lane == w.head) w.ring = x;
    w.head = w.head + 1 == w.cap ? 0 : w.head + 1;
  } else {
    uint32_t tail = w.head + w.n;
    if (tail >= w.cap) tail -= w.cap;
    if (lane == tail) w.ring = x;
  }
  win_insert(w, x);
}

__device__ __forceinline__ double win_median(const RegWin& w) {
  const uint32_t n = w.n;
  if (n % 2 == 1) return __shfl_sync(0xffffffffu, w.v, n / 2);
  const double a = __shfl_sync(0xffffffffu, w.v, n / 2 - 1), c = __shfl_sync(0xffffffffu, w.v, n / 2);
  return __dmul_rn(0.5, __dadd_rn(a, c));
}

__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int g = *(volatile unsigned int*)gen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *(volatile unsigned int*)count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*(volatile unsigned int*)gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

template <bool kReg>
__global__ void __launch_bounds__(kStageWarps * 32)
    k_stage_jacobi(DevBuffers b, DevConfig cfg, StageMeta m, int after_blocks) {
  pdl_enter();
  using WinT = typename std::conditional<kReg, RegWin, Win>::type;
  extern __shared__ __align__(16) double s_win[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t W = (uint32_t)cfg.cyc.stage_window;
  const u64 min_hist = cfg.cyc.stage_min_history;
  double* mine = s_win + (u64)warp * 4 * W;
  const uint32_t gw = blockIdx.x * kStageWarps + warp, nw = gridDim.x * kStageWarps;
  // no Unknown cycle anywhere (the common forward_mode case): nothing to do;
  // every CTA reads the same flag, so none waits at a barrier
  if (__ldcg(b.any_unknown) == 0u || (after_blocks && __ldcg(m.final_parity + 2) != 0u)) {  // nothing Unknown / k_stage_blocks converged
    if (blockIdx.x == 0 && threadIdx.x == 0) *m.final_parity = 0;
    return;
  }
  for (int it = 0; it < m.max_iter; ++it) {
    const uint8_t* in = m.st[it & 1];
    uint8_t* out = m.st[(it + 1) & 1];
    for (uint32_t c = gw; c < m.n_chunks; c += nw) {
      const u64 lo = (u64)c * kStageChunk;
      const u64 hi = min(lo + (u64)kStageChunk, (u64)b.n_cycles);
      // chunks of instances without Unknown cycles keep their local stages
      bool any_unknown = false;
      for (uint32_t i = b.c_inst[lo]; i <= b.c_inst[hi - 1] && !any_unknown; ++i)
        any_unknown = b.inst[i].n_unknown != 0;
      // recompute only when something before the chunk changed last iteration
      bool dirty = it == 0 && any_unknown;
      if (!dirty && it > 0 && any_unknown) {
        const u64 lb = __ldcg(&m.lookback_lo[c]);
        for (u64 cc = lb / kStageChunk; cc < c && !dirty; ++cc)
          dirty = __ldcg(&m.changed_iter[cc]) == it - 1;
      }
      if (!dirty) {  // carry the values over into this iteration's array
        for (u64 u = lo + lane; u < hi; u += 32) out[u] = __ldcg(&in[u]);
        continue;
      }
      bool changed = false;
      uint32_t cur_inst = 0xffffffffu;
      WinT dw, gwin;
      if constexpr (kReg) {
        dw = RegWin{0.0, 0.0, 0, 0, W};
        gwin = RegWin{0.0, 0.0, 0, 0, W};
      } else {
        dw = Win{mine, mine + W, 0, 0, W};
        gwin = Win{mine + 2 * W, mine + 3 * W, 0, 0, W};
      }
      // staging for the window rebuild: most recent first
      double* stage_d = mine;
      double* stage_g = mine + 2 * W;
      u64 c0 = 0;
      const StreamCarry* sc = nullptr;
      u64 lb_lo = lo;
      // per 32-cycle block: the cycles' inputs loaded once, coalesced, one
      // cycle per lane; the sequential walk takes them by shuffle
      for (u64 u0 = lo; u0 < hi; u0 += 32) {
        const u64 ul = u0 + lane;
        const bool lv = ul < hi;
        uint32_t x_local = 3, x_inst = 0xffffffffu, x_in = 0;
        double x_dur = 0.0, x_gap = -1.0;
        if (lv) {
          x_local = b.c_local[ul];
          x_inst = b.c_inst[ul];
          x_in = __ldcg(&in[ul]);
          if (x_local != 3) {
            const u64 c0l = b.cyc_off[x_inst];
            const StreamCarry* scl = b.stream ? b.stream + x_inst : nullptr;
            x_dur = (double)(b.c_end[ul] - b.c_start[ul]);
            x_gap = ul > c0l ? (double)(b.c_start[ul] - b.c_aend[ul - 1])
                    : (scl && scl->has_prev) ? (double)(b.c_start[ul] - scl->last_aend) : -1.0;
          }
        }
        uint32_t x_out = x_local;
        const uint32_t nl = (uint32_t)min((u64)32, hi - u0);
        for (uint32_t l = 0; l < nl; ++l) {
          const u64 u = u0 + l;
          const uint8_t local = (uint8_t)__shfl_sync(0xffffffffu, x_local, l);
          if (local == 3) continue;  // hole slot of the single-read pass: not a cycle
          const uint32_t inst = __shfl_sync(0xffffffffu, x_inst, l);
          if (inst != cur_inst) {
            // (re)build the windows from the cycles before u in its instance
            cur_inst = inst;
            c0 = b.cyc_off[inst];
            sc = b.stream ? b.stream + inst : nullptr;
            dw.n = dw.head = gwin.n = gwin.head = 0;
            // collect most recent first in the rings' upper halves, then insert oldest first
            uint32_t nd = 0, ng = 0;
            i64 top = (i64)u - 1;
            for (; top >= (i64)c0 && (nd < W || ng < W); top -= 32) {
              const i64 j = top - lane;
              const bool inr = j >= (i64)c0;
              bool nonp = false, gok = false;
              double jd = 0.0, jg = -1.0;
              if (inr && b.c_local[j] != 3) {
                nonp = __ldcg(&in[j]) != CS_STAGE_PREFILL;
                jd = (double)(b.c_end[j] - b.c_start[j]);
                jg = j > (i64)c0 ? (double)(b.c_start[j] - b.c_aend[j - 1])
                     : (sc && sc->has_prev) ? (double)(b.c_start[j] - sc->last_aend) : -1.0;
                gok = nonp && jg >= 0.0;
              }
              const uint32_t md = __ballot_sync(0xffffffffu, inr && nonp);
              const uint32_t mg = __ballot_sync(0xffffffffu, inr && gok);
              const uint32_t kd = nd + __popc(md & lanemask_lt());
              const uint32_t kg = ng + __popc(mg & lanemask_lt());
              if (inr && nonp && kd < W) stage_d[kd] = jd;  // staging: most recent first
              if (inr && gok && kg < W) stage_g[kg] = jg;
              nd = min(W, nd + __popc(md));
              ng = min(W, ng + __popc(mg));
              if (u == lo) lb_lo = (u64)max((i64)c0, top - 31);
            }
            if (u == lo && top < (i64)c0) lb_lo = c0;
            __syncwarp();
            // earlier micro-batches (streaming carry), most recent first
            if (sc) {
              const double* scd = b.s_dur + (u64)inst * b.s_sw;
              const double* scg = b.s_gap + (u64)inst * b.s_sw;
              for (uint32_t k = lane; k < sc->n_dur && nd + k < W; k += 32) stage_d[nd + k] = scd[k];
              for (uint32_t k = lane; k < sc->n_gap && ng + k < W; k += 32) stage_g[ng + k] = scg[k];
              nd = min(W, nd + sc->n_dur);
              ng = min(W, ng + sc->n_gap);
            }
            __syncwarp();
            // oldest first into the rings, then sort
            if constexpr (kReg) {
              dw.ring = (uint32_t)lane < nd ? stage_d[nd - 1 - lane] : 0.0;
              gwin.ring = (uint32_t)lane < ng ? stage_g[ng - 1 - lane] : 0.0;
              __syncwarp();
              for (uint32_t k = 0; k < nd; ++k) win_insert(dw, __shfl_sync(0xffffffffu, dw.ring, k));
              for (uint32_t k = 0; k < ng; ++k) win_insert(gwin, __shfl_sync(0xffffffffu, gwin.ring, k));
            } else {
              for (uint32_t k = lane; k < nd; k += 32) dw.ring[k] = dw.sorted[nd - 1 - k];
              for (uint32_t k = lane; k < ng; k += 32) gwin.ring[k] = gwin.sorted[ng - 1 - k];
              __syncwarp();
              for (uint32_t k = 0; k < nd; ++k) win_insert(dw, dw.ring[k]);
              for (uint32_t k = 0; k < ng; ++k) win_insert(gwin, gwin.ring[k]);
            }
            dw.head = 0;
            gwin.head = 0;
          }
          const double gap = __shfl_sync(0xffffffffu, x_gap, l);
          const double cdur = __shfl_sync(0xffffffffu, x_dur, l);
          uint8_t stage = local;
          if (stage == CS_STAGE_UNKNOWN && (u64)dw.n >= min_hist && gap >= 0.0) {
            const double med_dur = win_median(dw);
            double med_gap = gwin.n ? win_median(gwin) : 0.0;
            med_gap = 1.0 < med_gap ? med_gap : 1.0;
            const bool long_cycle = cdur > __dmul_rn(cfg.cyc.prefill_duration_factor, med_dur);
            const bool long_gap = gap > __dmul_rn(cfg.cyc.prefill_gap_factor, med_gap);
            stage = (long_cycle && long_gap) ? CS_STAGE_PREFILL : CS_STAGE_DECODE;
          }
          const uint32_t pin = __shfl_sync(0xffffffffu, x_in, l);
          changed |= (stage == CS_STAGE_PREFILL) != (pin == CS_STAGE_PREFILL);
          if ((uint32_t)lane == l) x_out = stage;
          if (stage != CS_STAGE_PREFILL) {
            win_push(dw, cdur);
            if (gap >= 0.0) win_push(gwin, gap);
          }
        }
        if (lv) out[ul] = (uint8_t)x_out;
      }
      if (lane == 0) {
        m.lookback_lo[c] = lb_lo;
        if (changed) {
          m.changed_iter[c] = it;
          atomicOr(m.any_changed + (it & 1), 1u);
        }
      }
    }
    grid_barrier(m.bar_count, m.bar_gen);
    const bool more = __ldcg(m.any_changed + (it & 1)) != 0;
    grid_barrier(m.bar_count, m.bar_gen);  // everyone has read the flag
    if (blockIdx.x == 0 && threadIdx.x == 0) m.any_changed[it & 1] = 0;
    if (!more) {
      if ((it + 1) & 1)  // the result is in the scratch array: back into c_stage
        for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < b.n_cycles; u += (u64)gridDim.x * blockDim.x)
          m.st[0][u] = __ldcg(&m.st[1][u]);
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        *m.final_parity = 0;
        m.final_parity[1] = (unsigned int)(it + 1);  // iterations run (profiling)
      }
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *m.final_parity = 0xffffffffu;  // did not converge
}

// K4b: the chunked Jacobi of k_stage_jacobi with each chunk walked in blocks
// of 32 cycles instead of one cycle at a time (windows <= 32, no streaming
// carry).  Within a block, lane l's windows are the last W values of
// (history ++ the block's non-Prefill cycles before l): the duration and
// gap histories (oldest first, <= W each) and the block's values form one
// list of <= 64 in shared memory.  A cycle needs only the side of each
// median: with t(v) = fl(f * v) monotone in v, "x > fl(f * median)" holds
// iff at least n/2 + 1 window values have t(v) < x (odd n); for even n
// (median = (a + b) / 2 of the n/2-th and n/2+1-th) it holds iff that count
// is >= n/2 + 1 and fails iff it is <= n/2 - 1; with a count of exactly n/2
// the two middle values are the largest value below the threshold and the
// smallest one at or above it.  The block's own Prefill-ness is
// speculated from the previous iterate and re-evaluated until it reproduces
// itself (a local fixed point: cycles depend only on earlier ones).  Blocks
// spanning an instance boundary are split into per-instance segments.
// cycles.cpp:181-186 (median), 204-250 (decision, window updates).
__global__ void __launch_bounds__(kStageWarps * 32)
    k_stage_blocks(DevBuffers b, DevConfig cfg, StageMeta m) {
  pdl_enter();
  __shared__ double s_hd[kStageWarps][32], s_hg[kStageWarps][32];
  __shared__ double s_cd[kStageWarps][64], s_cg[kStageWarps][64], s_t[kStageWarps][64];
  __shared__ double s_stg[kStageWarps][64];  // rebuild staging (most recent first)
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t W = (uint32_t)cfg.cyc.stage_window;
  const uint32_t min_hist = (uint32_t)min((u64)cfg.cyc.stage_min_history, (u64)0xffffffffu);
  const double fd = cfg.cyc.prefill_duration_factor, fg = cfg.cyc.prefill_gap_factor;
  const bool sane = fd > 0.0 && fg > 0.0;
  double* hd = s_hd[warp];
  double* hg = s_hg[warp];
  double* cd = s_cd[warp];
  double* cg = s_cg[warp];
  double* tt = s_t[warp];
  double* stg = s_stg[warp];
  const uint32_t gw = blockIdx.x * kStageWarps + warp, nw = gridDim.x * kStageWarps;
  if (__ldcg(b.any_unknown) == 0u) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *m.final_parity = 0;
      m.final_parity[2] = 1u;
    }
    return;
  }
  // the count argument needs t(v) = fl(f * v) nondecreasing: f > 0; other
  // factors go to the sequential-window kernel
  bool bad = !sane;
  // "x > fl(f * median(list[P - n, P)))" (gap: f * max(1, median)), from a
  // count; a count of exactly n/2 (even n) fixes the two middle values as the
  // largest value below the threshold and the smallest one at or above it,
  // found by the lane alone (no warp-wide sort)
  auto side = [&](const double* list, uint32_t len, uint32_t P, uint32_t n, double x, double f, bool is_gap,
                  bool need) -> bool {
    for (uint32_t e = lane; e < len; e += 32) {
      const double v = list[e];
      tt[e] = __dmul_rn(f, is_gap ? (1.0 < v ? v : 1.0) : v);
    }
    __syncwarp();
    bool r = false;
    if (need) {
      uint32_t c = 0;
      for (uint32_t j = P - n; j < P; ++j) c += tt[j] < x ? 1u : 0u;
      const uint32_t n2 = n / 2u;
      if ((n & 1u) || c != n2) {
        r = c >= n2 + 1u;
      } else {
        double a = -1.0, bv = 1.0 / 0.0;
        for (uint32_t j = P - n; j < P; ++j) {
          const double v = list[j];
          if (tt[j] < x) a = a < v ? v : a;
          else bv = bv < v ? bv : v;
        }
        const double med = __dmul_rn(0.5, __dadd_rn(a, bv));
        r = x > __dmul_rn(f, is_gap ? (1.0 < med ? med : 1.0) : med);
      }
    }
    __syncwarp();
    return r;
  };
  for (int it = 0; it < m.max_iter; ++it) {
    const uint8_t* in = m.st[it & 1];
    uint8_t* out = m.st[(it + 1) & 1];
    for (uint32_t c = gw; c < m.n_chunks; c += nw) {
      const u64 lo = (u64)c * kStageChunk;
      const u64 hi = min(lo + (u64)kStageChunk, (u64)b.n_cycles);
      bool any_unknown = false;
      for (uint32_t i = b.c_inst[lo]; i <= b.c_inst[hi - 1] && !any_unknown; ++i)
        any_unknown = b.inst[i].n_unknown != 0;
      bool dirty = it == 0 && any_unknown;
      if (!dirty && it > 0 && any_unknown) {
        const u64 lb = __ldcg(&m.lookback_lo[c]);
        for (u64 cc = lb / kStageChunk; cc < c && !dirty; ++cc)
          dirty = __ldcg(&m.changed_iter[cc]) == it - 1;
      }
      if (!dirty) {
        for (u64 u = lo + lane; u < hi; u += 32) out[u] = __ldcg(&in[u]);
        continue;
      }
      bool changed = false;
      uint32_t cur_inst = 0xffffffffu, nhd = 0, nhg = 0;
      u64 lb_lo = lo;
      for (u64 u0 = lo; u0 < hi; u0 += 32) {
        const u64 u = u0 + lane;
        const bool lv = u < hi;
        uint8_t local = 3, pin = 0;
        uint32_t inst = 0xffffffffu;
        double dur = 0.0;
        int64_t gap = -1;
        if (lv) {
          local = b.c_local[u];
          pin = __ldcg(&in[u]);
          inst = b.c_inst[u];
          if (local != 3) {
            const u64 c0 = b.cyc_off[inst];
            dur = (double)(b.c_end[u] - b.c_start[u]);
            gap = u > c0 ? b.c_start[u] - b.c_aend[u - 1] : -1;
          }
        }
        uint8_t st = local;
        const uint32_t nl = (uint32_t)min((u64)32, hi - u0);
        uint32_t s0 = 0;
        while (s0 < nl) {
          const uint32_t inst_s = __shfl_sync(0xffffffffu, inst, s0);
          const uint32_t diff = __ballot_sync(0xffffffffu, lane >= s0 && lane < nl && inst != inst_s);
          const uint32_t s1 = diff ? (uint32_t)__ffs(diff) - 1u : nl;
          const bool inseg = lane >= s0 && lane < s1 && local != 3;
          if (inst_s != cur_inst) {
            // history from the cycles before the segment in its instance
            // (previous iterate), most recent first into staging
            cur_inst = inst_s;
            const u64 us = u0 + s0;
            const u64 ci0 = b.cyc_off[inst_s];
            uint32_t nd = 0, ng = 0;
            i64 top = (i64)us - 1;
            for (; top >= (i64)ci0 && (nd < W || ng < W); top -= 32) {
              const i64 j = top - (i64)lane;
              const bool inr = j >= (i64)ci0;
              bool nonp = false, gok = false;
              double jd = 0.0, jg = -1.0;
              if (inr && b.c_local[j] != 3) {
                nonp = __ldcg(&in[j]) != CS_STAGE_PREFILL;
                jd = (double)(b.c_end[j] - b.c_start[j]);
                jg = j > (i64)ci0 ? (double)(b.c_start[j] - b.c_aend[j - 1]) : -1.0;
                gok = nonp && jg >= 0.0;
              }
              const uint32_t md = __ballot_sync(0xffffffffu, inr && nonp);
              const uint32_t mg = __ballot_sync(0xffffffffu, inr && gok);
              const uint32_t kd = nd + __popc(md & lanemask_lt());
              const uint32_t kg = ng + __popc(mg & lanemask_lt());
              if (inr && nonp && kd < W) stg[kd] = jd;
              if (inr && gok && kg < W) stg[32 + kg] = jg;
              nd = min(W, nd + __popc(md));
              ng = min(W, ng + __popc(mg));
              if (us == lo) lb_lo = (u64)max((i64)ci0, top - 31);
            }
            if (us == lo && top < (i64)ci0) lb_lo = ci0;
            __syncwarp();
            if (lane < nd) hd[lane] = stg[nd - 1 - lane];  // oldest first
            if (lane < ng) hg[lane] = stg[32 + ng - 1 - lane];
            nhd = nd;
            nhg = ng;
            __syncwarp();
          }
          // local fixed point of the segment's Prefill-ness
          bool spec = local == CS_STAGE_PREFILL || (local == CS_STAGE_UNKNOWN && pin == CS_STAGE_PREFILL);
          const uint32_t segm = __ballot_sync(0xffffffffu, inseg);
          uint32_t td = 0, tg = 0;
          for (int round = 0; round < 34; ++round) {
            const bool npl = inseg && !spec, gkl = npl && gap >= 0;
            const uint32_t bd = __ballot_sync(0xffffffffu, npl) & segm, bg = __ballot_sync(0xffffffffu, gkl) & segm;
            const uint32_t rd = __popc(bd & lanemask_lt()), rg = __popc(bg & lanemask_lt());
            td = __popc(bd);
            tg = __popc(bg);
            if (npl) cd[nhd + rd] = dur;
            if (gkl) cg[nhg + rg] = (double)gap;
            if (lane < nhd) cd[lane] = hd[lane];
            if (lane < nhg) cg[lane] = hg[lane];
            __syncwarp();
            const uint32_t Pd = nhd + rd, Pg = nhg + rg;
            const uint32_t n_d = min(W, Pd), n_g = min(W, Pg);
            const bool want = inseg && local == CS_STAGE_UNKNOWN && n_d >= min_hist && gap >= 0;
            uint8_t ns = local;
            if (__any_sync(0xffffffffu, want)) {
              const bool long_cycle = side(cd, nhd + td, Pd, n_d, dur, fd, false, want);
              const bool lg = side(cg, nhg + tg, Pg, n_g, (double)gap, fg, true, want && n_g > 0);
              if (want) {
                const bool long_gap = n_g == 0 ? (double)gap > __dmul_rn(fg, 1.0) : lg;
                ns = (long_cycle && long_gap) ? CS_STAGE_PREFILL : CS_STAGE_DECODE;
              }
            }
            const bool nspec = ns == CS_STAGE_PREFILL;
            const bool moved = __any_sync(0xffffffffu, inseg && nspec != spec);
            if (inseg) st = ns;
            __syncwarp();
            if (!moved) break;
            if (inseg) spec = nspec;
          }
          // histories after the segment: last W of (history ++ segment
          // values); the final round's lists are exactly that
          const uint32_t ld = nhd + td, lg = nhg + tg;
          const uint32_t kd = min(W, ld), kg = min(W, lg);
          double vd = 0.0, vg = 0.0;
          if (lane < kd) vd = cd[ld - kd + lane];
          if (lane < kg) vg = cg[lg - kg + lane];
          __syncwarp();
          if (lane < kd) hd[lane] = vd;
          if (lane < kg) hg[lane] = vg;
          nhd = kd;
          nhg = kg;
          __syncwarp();
          s0 = s1;
        }
        if (lv) {
          out[u] = st;
          changed |= local != 3 && (st == CS_STAGE_PREFILL) != (pin == CS_STAGE_PREFILL);
        }
      }
      changed = __any_sync(0xffffffffu, changed);
      if (lane == 0) {
        m.lookback_lo[c] = lb_lo;
        if (changed) {
          m.changed_iter[c] = it;
          atomicOr(m.any_changed + (it & 1), 1u);
        }
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(m.final_parity + 3, 1u);
    grid_barrier(m.bar_count, m.bar_gen);
    const bool more = __ldcg(m.any_changed + (it & 1)) != 0;
    const bool invalid = __ldcg(m.final_parity + 3) != 0;
    grid_barrier(m.bar_count, m.bar_gen);
    if (blockIdx.x == 0 && threadIdx.x == 0) m.any_changed[it & 1] = 0;
    if (!more || invalid) {
      if (invalid) {  // factors the count argument does not cover: the sequential-window kernel redoes it
        for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < b.n_cycles; u += (u64)gridDim.x * blockDim.x)
          m.st[0][u] = b.c_local[u];
      } else if ((it + 1) & 1) {
        for (u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x; u < b.n_cycles; u += (u64)gridDim.x * blockDim.x)
          m.st[0][u] = __ldcg(&m.st[1][u]);
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        *m.final_parity = 0;
        m.final_parity[1] = (unsigned int)(it + 1);
        m.final_parity[2] = invalid ? 0u : 1u;
        m.final_parity[3] = 0u;
      }
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *m.final_parity = 0xffffffffu;
    m.final_parity[2] = 0u;  // no fixed point: the sequential-window kernel continues from the iterate
  }
}

int launch_stage_heuristic(const DevBuffers& b, const DevConfig& cfg, const StageMeta& m, cudaStream_t s,
                           uint64_t* launches) {
  if (!b.n_cycles || m.n_chunks == 0) return 0;
  const size_t smem = (size_t)kStageWarps * 4 * cfg.cyc.stage_window * sizeof(double);
  if (smem > 200 * 1024) return -1;
  const int n_sm0 = sm_count();
  const bool blocks = !b.stream && cfg.cyc.stage_window <= 32 && cfg.cyc.stage_window >= 1;
  if (blocks) {
    // block-parallel chunks first; the sequential-window kernel below only
    // runs when it could not (stage factors <= 0) or did not converge
    int per_sm = blocks_per_sm((const void*)k_stage_blocks, kStageWarps * 32, 0);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)n_sm0 * per_sm;
    const uint64_t need = (m.n_chunks + kStageWarps - 1) / kStageWarps;
    if (grid > need) grid = need;
    launch_pdl(k_stage_blocks, (unsigned)grid, kStageWarps * 32, 0, s, b, cfg, m);
    ++*launches;
    // with positive factors it always reaches the fixed point (max_iter is
    // the chunk count + 2, and each iteration settles at least one more chunk)
    if (cfg.cyc.prefill_duration_factor > 0.0 && cfg.cyc.prefill_gap_factor > 0.0) return 0;
  }
  // windows of <= 32 values live in registers (one value per lane)
  const bool reg = cfg.cyc.stage_window <= 32;
  const void* fn = reg ? (const void*)k_stage_jacobi<true> : (const void*)k_stage_jacobi<false>;
  ensure_smem(fn, (int)smem);
  const int n_sm = n_sm0;
  int per_sm = blocks_per_sm(fn, kStageWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)n_sm * per_sm;  // persistent: every CTA resident (grid barrier)
  const uint64_t need = (m.n_chunks + kStageWarps - 1) / kStageWarps;
  if (grid > need) grid = need;
  if (reg) launch_pdl(k_stage_jacobi<true>, (unsigned)grid, kStageWarps * 32, smem, s, b, cfg, m, blocks ? 1 : 0);
  else launch_pdl(k_stage_jacobi<false>, (unsigned)grid, kStageWarps * 32, smem, s, b, cfg, m, blocks ? 1 : 0);
  ++*launches;
  return 0;
}

// Small batches: record compaction and per-instance record offsets in one
// CTA (count + scan + scatter + tail fused)
__global__ void __launch_bounds__(1024) k_records_small(DevBuffers b, DevConfig cfg) {
  pdl_enter();
  __shared__ uint32_t s_w[32];
  __shared__ u64 s_base;
  const bool need_index = cfg.cyc.monitor_from_cycle > 0 || b.stream;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (u64 g0 = 0; g0 < b.n_cycles; g0 += 1024) {
    const u64 g = g0 + threadIdx.x;
    const bool ok = g < b.n_cycles && rec_ok(b, cfg, g, need_index);
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (lane == 0) s_w[warp] = __popc(m);
    __syncthreads();
    uint32_t tot = 0;
    if (warp == 0) {
      uint32_t c = s_w[lane];
      const uint32_t x = c;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, c, o);
        if (lane >= o) c += y;
      }
      tot = __shfl_sync(0xffffffffu, c, 31);
      s_w[lane] = c - x;
    }
    __syncthreads();
    const u64 base = s_base;
    if (ok) b.rec_cycle[base + s_w[warp] + __popc(m & lanemask_lt())] = g;
    __syncthreads();
    if (threadIdx.x == 0) s_base = base + tot;
    __syncthreads();
  }
  // records are in cycle order: instance i's first record is the first whose
  // cycle is >= cyc_off[i]
  const u64 total = s_base;
  for (uint32_t i = threadIdx.x; i <= b.n_inst; i += blockDim.x) {
    const u64 c0 = b.cyc_off[i];
    u64 lo = 0, hi = total;
    while (lo < hi) {
      const u64 mid = (lo + hi) >> 1;
      if (b.rec_cycle[mid] < c0) lo = mid + 1;
      else hi = mid;
    }
    b.rec_off[i] = i == b.n_inst ? total : lo;
  }
}

constexpr u64 kSmallBatch = 32768;  // cycles / records handled by one CTA

bool launch_records(const DevBuffers& b, const DevConfig& cfg, int fuse_score, cudaStream_t s,
                    uint64_t* launches) {
  if (b.n_cycles <= kSmallBatch) {
    launch_pdl(k_records_small, 1, 1024, 0, s, b, cfg);
    ++*launches;
    return false;
  }
  const u64 nb = (b.n_cycles + kRecBlock - 1) / kRecBlock;
  if (nb) {
    launch_pdl(k_records_count, (unsigned)nb, kRecThreads, 0, s, b, cfg);
    ++*launches;
  }
  // block_tmp[nb] receives the total
  launch_pdl(k_scan_exclusive, 1, 1024, 0, s, b.block_tmp, nb, b.block_tmp + nb);
  ++*launches;
  if (nb) {
    launch_pdl(k_records_scatter, (unsigned)nb, kRecThreads, 0, s, b, cfg, fuse_score);
    ++*launches;
  }
  launch_pdl(k_rec_off_tail, 1, 1, 0, s, b, b.block_tmp + nb);
  ++*launches;
  return fuse_score != 0 && nb != 0;
}

void launch_score(const DevBuffers& b, const DevConfig& cfg, uint64_t n_records,
                  const uint64_t*, const int*, const DevModel* h_models, cudaStream_t s,
                  uint64_t* launches) {
  if (!n_records) return;
  const int max_optin = smem_optin();
  bool all_lut = true;
  uint64_t need = 0;
  for (uint32_t i = 0; i < b.n_inst; ++i) {
    all_lut &= h_models[i].lut != nullptr;
    if (h_models[i].smem_bytes > need) need = h_models[i].smem_bytes;
  }
  if (all_lut) {
    launch_pdl(k_score_lut_flat, (unsigned)((n_records + kLutThreads - 1) / kLutThreads), kLutThreads, 0, s,
               b, cfg, n_records);
    ++*launches;
    return;
  }
  // one traversal kernel for the batch, instantiated for the widest model:
  // narrower models never read the extra feature slots (their nodes test
  // features < their own count), so instances may mix feature counts
  uint32_t nf = 0;
  for (uint32_t i = 0; i < b.n_inst; ++i) nf = h_models[i].n_features > nf ? h_models[i].n_features : nf;
  uint64_t cap = (uint64_t)max_optin - 1024;
  if (need < cap) cap = need;
  const unsigned grid = (unsigned)((n_records + kScoreTile - 1) / kScoreTile);
#define CS_SCORE_CASE(NF)                                                                 \
  case NF:                                                                                \
    ensure_smem((const void*)k_score<NF>, (int)cap);                                    \
    launch_pdl(k_score<NF>, grid, kScoreThreads, cap, s, b, cfg, n_records, cap);                 \
    break;
  switch (nf) {
    CS_SCORE_CASE(0)
    CS_SCORE_CASE(1)
    CS_SCORE_CASE(2)
    CS_SCORE_CASE(3)
    CS_SCORE_CASE(4)
    CS_SCORE_CASE(5)
    CS_SCORE_CASE(6)
    CS_SCORE_CASE(7)
    CS_SCORE_CASE(8)
    default: break;
  }
#undef CS_SCORE_CASE
  ++*launches;
}

void launch_detect(const DevBuffers& b, const DevConfig& cfg, uint64_t n_records, cudaStream_t s,
                   uint64_t* launches) {
  if (n_records <= kSmallBatch) {  // n_records: the record capacity (cycle count)
    launch_pdl(k_detect_small, 1, 1024, 0, s, b, cfg, n_records);
    ++*launches;
    return;
  }
  const u64 nb = (n_records + kDetBlock - 1) / kDetBlock;
  if (nb) {
    const int W = cfg.ctl.strategy == CS_FIXED_POINT ? 0 : (int)cfg.ctl.window;
    if (!b.stream && W <= kDetMaxW) {
#define CS_DET_CASE(N)   case N:                  launch_pdl(k_detect_win<N>, (unsigned)nb, kDetThreads, 0, s, b, cfg, n_records);     break;
      switch (W) {
        CS_DET_CASE(0) CS_DET_CASE(1) CS_DET_CASE(2) CS_DET_CASE(3) CS_DET_CASE(4) CS_DET_CASE(5)
        CS_DET_CASE(6) CS_DET_CASE(7) CS_DET_CASE(8) CS_DET_CASE(9) CS_DET_CASE(10) CS_DET_CASE(11)
        CS_DET_CASE(12) CS_DET_CASE(13) CS_DET_CASE(14) CS_DET_CASE(15) CS_DET_CASE(16)
        default: break;
      }
#undef CS_DET_CASE
    } else {
      launch_pdl(k_detect_flags, (unsigned)nb, kDetBlock, 0, s, b, cfg, n_records);
    }
    ++*launches;
  }
  launch_pdl(k_scan_exclusive, 1, 1024, 0, s, b.block_tmp, nb, b.block_tmp + nb);
  ++*launches;
  launch_pdl(k_alert_off, 1, 1024, 0, s, b);
  ++*launches;
  if (nb) {
    const u64 warps = (u64)sm_count() * 2 * (kDetScatterThreads / 32);
    const u64 grid = (min(nb, warps) * 32 + kDetScatterThreads - 1) / kDetScatterThreads;
    launch_pdl(k_detect_scatter, (unsigned)grid, kDetScatterThreads, 0, s, b, n_records, (uint64_t)nb);
    ++*launches;
  }
}

void launch_gpu_kernel_extent(const cs_event* ev, uint64_t begin, uint64_t end,
                              unsigned long long* out3, cudaStream_t s, uint64_t* launches) {
  k_gpu_kernel_extent<<<296, 256, 0, s>>>(ev, begin, end, out3);
  ++*launches;
}

void launch_freq_hist(const cs_event* ev, uint64_t begin, uint64_t end, int64_t t0,
                      int64_t bin_ns, uint64_t bins, double* h, cudaStream_t s,
                      uint64_t* launches) {
  // hist counts are accumulated as u64 in the first half of a 2*bins buffer
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(h + bins);
  cudaMemsetAsync(counts, 0, bins * sizeof(u64), s);
  k_freq_hist<<<296, 256, 0, s>>>(ev, begin, end, t0, bin_ns, bins, counts);
  k_freq_center<<<1, 256, 0, s>>>(counts, bins, h);
  *launches += 2;
}

void launch_freq_autocorr(const double* h, uint64_t bins, double* acc, cudaStream_t s,
                          uint64_t* launches) {
  const u64 lags = bins / 2;
  if (!lags) return;
  k_freq_autocorr<<<(unsigned)((lags + 127) / 128), 128, 0, s>>>(h, bins, acc);
  ++*launches;
}

void launch_freq_cycles(const cs_event* ev, uint64_t begin, uint64_t end, int64_t t0,
                        int64_t period, uint64_t n, uint64_t cyc_base, const DevBuffers& b,
                        uint32_t inst, cudaStream_t s, uint64_t* launches) {
  if (!n) return;
  k_freq_cycles<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ev, begin, end, t0, period, n,
                                                           cyc_base, b, inst);
  ++*launches;
}


// =================================================== single-read segmentation
// K1+K2+K3 with the events read from DRAM once (CS_OPT_FUSED).  Work unit: a
// WARP RANGE of consecutive events of one instance, sized for ~32 cycles,
// claimed in order by a persistent grid.  Every warp is independent (no CTA
// barriers), so one warp's DRAM-bound scan overlaps its neighbours' L2-bound
// reduce.  Per range:
//   A. the warp streams its events (coalesced 256-bit loads): PythonCall
//      moments for the anchor ranking (cycles.cpp:50-59), the canonical-order
//      check, and the speculated anchor's occurrences listed in shared memory
//      (cycles.cpp:127-131); it publishes its anchor count and keeps reading
//      past the range to the next anchor, which closes its last cycle;
//   B. lane k reduces the cycle opened by anchor k, walking its events in
//      order (L2 hits: the warp has just streamed them), branch-free: every
//      event adds its clipped duration to lane-private shared-memory rows
//      (class occupancy, collective occupancy and count; a per-lane dummy row
//      absorbs the events that add nothing), so the warp executes one path
//      whatever mix of event kinds its lanes meet (cycles.cpp:157-166, 205-229,
//      256-281; rca.cpp:87-129).  Component durations are the class rows of
//      the phase functions' names (a clipped term > 0 implies duration > 0,
//      so both sums take the same terms).  Collective beta is a sum of
//      quotients in event order (rca.cpp:108-115): a (cycle, slot) with one
//      contribution is 0.0 + q = q, the quotient of its integer sum; one with
//      several is re-summed in order by its lane.  Rows are 32-bit when the
//      batch proves duration x events < 2^32 for each cycle, 64-bit otherwise;
//   C. a decoupled look-back over the preceding ranges gives the global rank
//      of the range's first anchor = the slot of its first cycle, and the warp
//      writes its cycle rows.
// An instance's last anchor opens no complete cycle (cycles.cpp:147): its slot
// is a hole (empty event range, c_wl = kHoleWl) that every consumer skips.
// The anchor guess is verified afterwards by k_rank over the full moments; a
// wrong guess, an ambiguous ranking, a range with more than kSegList anchors
// or an equal-timestamp group at an anchor (lower_bound before the anchor's
// position) re-runs the two-pass path.
#ifndef CS_SEG_SCAN_UNROLL
#define CS_SEG_SCAN_UNROLL 4
#endif
#ifndef CS_SEG_PREFETCH
#define CS_SEG_PREFETCH 1
#endif
#ifndef CS_SEG_WALK_UNROLL
#define CS_SEG_WALK_UNROLL 3
#endif
constexpr int kSegScanUnroll = CS_SEG_SCAN_UNROLL;  // phase A: 256-bit loads in flight per lane
constexpr int kSegWalkUnroll = CS_SEG_WALK_UNROLL;  // phase B: events in flight per lane
constexpr int kSegThreads = 256;
constexpr int kSegWarps = kSegThreads / 32;
constexpr int kSegList = 128;      // anchors of one range listed in shared memory
constexpr uint32_t kSegClaim = 1;  // consecutive ranges per ticket (more serialises the look-back chain)
constexpr int kSegNames = 1024;    // name table staged in shared memory
constexpr uint32_t kSegTie = 0x80000000u;  // apos flag: equal start_ts before the anchor

// per-warp accumulator rows [row][33] (lane-private columns): u64 collective
// rows [0, R) as count << 48 | integer sum, then a dummy row; then class and
// component rows [0, C) classes, [C, C+P) components of phases without a
// class row, two dummy rows -- u32 when the batch proves every sum < 2^32,
// else u64
constexpr int kCollShift = 48;
__host__ __device__ constexpr uint32_t seg_rows(int P, int C, int R) {
  return (uint32_t)(R + 1 + C + P + 2);
}
__host__ __device__ constexpr uint32_t seg_words(int P, int C, int R) {
  return seg_rows(P, C, R) * 33u * 2u;
}

struct SegWarpSmem {  // fixed-size per-warp state (static shared memory)
  i64 ats[kSegList];        // range anchors: start_ts
  uint32_t apos[kSegList];  // range anchors: offset in the range | kSegTie
  uint32_t adur[kSegList];  // range anchors: duration (0xffffffff: >= 2^32 - 1, reload)
  uint32_t pn[64];          // PythonCall compaction (name, duration)
  i64 pd[64];
  i64 dur[32];              // batch cycles: duration
};

__global__ void __launch_bounds__(kSegThreads, 2)
    k_segment_range(DevBuffers b, DevConfig cfg, SegMeta sm, int do_beta) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) unsigned char s_dyn[];
  __shared__ uint32_t s_ninfo[kSegNames];
  __shared__ int32_t s_pbs[16];  // phase -> class row of its name (-1: own component row)
  __shared__ WarpNameRow s_rows[kSegWarps * kWarpNameRows];
  __shared__ SegWarpSmem s_w[kSegWarps];
  const int P = cfg.cyc.n_phases;
  const int C = do_beta ? cfg.cyc.n_beta_slots : 0;
  const int R = do_beta ? cfg.cyc.n_comm_slots : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t NR = seg_rows(P, C, R);
  const uint32_t db = (uint32_t)(C + P), dp = db + 1u;  // dummy class / component rows
  if (threadIdx.x < 16) s_pbs[threadIdx.x] = -1;
  __syncthreads();
  // name -> (class row | component row << 8 | keyword bits << 30); a phase
  // name with a class row accumulates once, into the class row (a clipped
  // term > 0 implies duration > 0, so both sums take the same terms)
  for (uint32_t i = threadIdx.x; i < b.n_names; i += blockDim.x) {
    const cs_name_info ni = b.names[i];
    const bool ph = ni.phase >= 0 && ni.phase < P;
    const bool bs = ni.beta_slot >= 0 && ni.beta_slot < C;
    const uint32_t brow = bs ? (uint32_t)ni.beta_slot : db;
    const uint32_t prow = (ph && !bs) ? (uint32_t)(C + ni.phase) : dp;
    s_ninfo[i] = brow | (prow << 8) | ((ni.flags & 3u) << 30);
    if (ph && bs) s_pbs[ni.phase] = ni.beta_slot;
  }
  // the name table is configuration (no earlier kernel writes it): staged
  // while the predecessor drains, then wait for its results
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();  // the only CTA barriers: warps are independent from here on
  const uint32_t SN = 33;
  u64* acc_c = reinterpret_cast<u64*>(s_dyn) + (u64)warp * NR * SN;  // collective rows [R + 1][SN]
  unsigned char* acc_b = reinterpret_cast<unsigned char*>(acc_c + (u64)(R + 1) * SN);  // class rows
  // one cycle's events in order, branch-free (cycles.cpp:157-166, 205-229,
  // 256-281; rca.cpp:87-129): every event adds its clipped duration to the
  // lane's rows named by its name, or to a dummy row when none applies.  The
  // three rows one event touches are distinct (class rows / dummy, component
  // rows / dummy, collective rows / dummy), so their read-modify-writes
  // overlap; consecutive events may share rows and stay in order.
  auto walk = [&](auto tag, u64 first, u64 last, i64 ce, uint32_t& fm, uint32_t& kw, int32_t& wl) {
    using T = decltype(tag);
    T* rb_ = reinterpret_cast<T*>(acc_b) + lane;
    u64* rc_ = acc_c + lane;
    bool wl_found = false;
    auto step = [&](u64 j0, bool guard) {
      Ev8 e[kSegWalkUnroll];
#pragma unroll
      for (int q = 0; q < kSegWalkUnroll; ++q) {
        if (!guard || j0 + q < last) e[q] = ldg256(b.ev + j0 + q);
        else {
          e[q].a = 0;
          e[q].b = 0;
          e[q].c = (u64)CS_FLOW << 32;
          e[q].d = 0;
        }
      }
#pragma unroll
      for (int q = 0; q < kSegWalkUnroll; ++q) {
        const uint32_t name = (uint32_t)e[q].c;
        const uint32_t kc = (uint32_t)(e[q].c >> 32);
        const uint32_t flags = kc >> 16;
        const bool span = (kc & 0xffu) == CS_SPAN;
        const uint32_t info = span ? s_ninfo[name] : (db | (dp << 8));
        kw |= info >> 30;
        // clipped = max(0, min(st + d, ce) - st) = min(d, ce - st) when d > 0
        const i64 d = (i64)e[q].b;
        T c;
        if constexpr (sizeof(T) == 4) {
          // ce - st in (0, dur], dur < 2^32: 32-bit arithmetic is exact
          const uint32_t rem = (uint32_t)ce - (uint32_t)e[q].a;
          const int32_t hi = (int32_t)(d >> 32);
          uint32_t v = min((uint32_t)d, rem);
          v = hi > 0 ? rem : v;
          c = hi < 0 ? 0u : v;
        } else {
          const i64 rem = ce - (i64)e[q].a;
          c = d > 0 ? (u64)(d < rem ? d : rem) : 0ull;
        }
        const uint32_t slot = (uint32_t)(e[q].d >> 32);
        const bool cl = span && ((kc >> 8) & 0xffu) == CS_CAT_COLLECTIVE_COMM && (flags & CS_EV_HAS_COMM) &&
                        slot < (uint32_t)R && c != 0;
        T* pb = rb_ + (info & 0xffu) * SN;
        T* pp = rb_ + ((info >> 8) & 0xffu) * SN;
        u64* pc = rc_ + (cl ? slot : (uint32_t)R) * SN;
        const T vb = *pb, vp = *pp;
        const u64 vc = *pc;
        *pb = vb + c;
        *pp = vp + c;
        *pc = vc + (u64)c + (1ull << kCollShift);
        fm = (fm == 0u && (flags & CS_EV_FM_MASK)) ? (4u | (flags & CS_EV_FM_MASK)) : fm;
        const bool hb = (flags & CS_EV_HAS_BATCH) != 0;
        wl = (!wl_found && hb) ? ((flags & CS_EV_WL_OK) ? (int32_t)(uint32_t)e[q].d : -2) : wl;
        wl_found |= hb;
      }
    };
    u64 j0 = first;
    for (; j0 + kSegWalkUnroll <= last; j0 += kSegWalkUnroll) step(j0, false);
    if (j0 < last) step(j0, true);
  };
  SegWarpSmem& w = s_w[warp];
  WarpNameRow* wrows = s_rows + warp * kWarpNameRows;
  const u64 mP = P ? ((1ull << 32) + (u64)P - 1) / (u64)P : 0;
  const u64 mC = C ? ((1ull << 32) + (u64)C - 1) / (u64)C : 0;
  const u64 mR = R ? ((1ull << 32) + (u64)R - 1) / (u64)R : 0;
  SNameCache cache = SNameCache::at(s_dyn + (u64)kSegWarps * seg_words(P, C, R) * 4 + (u64)warp * SNameCache::kBytes, lane);
  cache_clear(cache);
  __syncwarp();
  uint32_t cur_inst = 0xffffffffu, npend = 0;
  NameStat* gstats = b.stats;
  auto drain = [&](uint32_t take) {
    __syncwarp();
    if ((uint32_t)lane < take) cache_add(cache, gstats, w.pn[lane], w.pd[lane]);
    __syncwarp();
    const uint32_t rest = npend - take;
    uint32_t mv_n = 0;
    i64 mv_d = 0;
    if ((uint32_t)lane < rest) {
      mv_n = w.pn[take + lane];
      mv_d = w.pd[take + lane];
    }
    __syncwarp();
    if ((uint32_t)lane < rest) {
      w.pn[lane] = mv_n;
      w.pd[lane] = mv_d;
    }
    npend = rest;
    __syncwarp();
  };
  // tickets hand out kSegClaim consecutive ranges at a time (a range's
  // look-back needs its predecessor's count, published only when its owner
  // reaches it, so claims larger than one range serialise the grid)
  uint32_t r = 0, r_end = 0;
  for (;;) {
    if (r == r_end) {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(sm.ticket, 1u);
      t = __shfl_sync(0xffffffffu, t, 0);
      r = t * kSegClaim;
      r_end = min(r + kSegClaim, sm.n_ranges);
    }
    if (r >= sm.n_ranges) break;
    const uint32_t rc = r++;
    const u64 rb = sm.range_begin[rc];
    const uint32_t n = (uint32_t)(sm.range_end[rc] - rb);
    const uint32_t inst = sm.range_inst[rc];
#if CS_SEG_PREFETCH
    // pull the whole range (+ a cycle past it) into L2 at once: the stream's
    // later iterations hit L2 instead of each waiting out a DRAM latency
    // and the range this warp will most likely claim next (tickets go round
    // the grid's warps), one range-time ahead
    if (lane < 2) {
      const uint32_t ahead = sm.prefetch_ahead == 0xffffffffu ? gridDim.x * (uint32_t)kSegWarps : sm.prefetch_ahead;
      const uint32_t pr = lane == 0 ? rc : rc + ahead;
      if ((lane == 0 || ahead) && pr < sm.n_ranges) {
        const u64 pb = sm.range_begin[pr];
        const uint32_t pi = sm.range_inst[pr];
        const uint32_t bytes =
            (uint32_t)umin64(sm.range_end[pr] - pb + 64u, b.inst_off[pi + 1] - pb) * (uint32_t)sizeof(cs_event);
        const char* p = reinterpret_cast<const char*>(b.ev + pb);
        for (uint32_t o = 0; o < bytes; o += 32768u) {
          const uint32_t m = min(32768u, bytes - o);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(m) : "memory");
        }
      }
    }
#endif
    const u64 ib = b.inst_off[inst];
    const uint32_t anchor = b.inst[inst].guess;
    if (inst != cur_inst) {
      if (cur_inst != 0xffffffffu) {
        drain(npend);
        cache_flush_warp(cache, gstats, wrows);
      }
      cur_inst = inst;
      gstats = b.stats + (u64)inst * b.n_names;
    }
    // ---------------- A: stream the range
    uint32_t cnt = 0;
    // ts of the event before the range: the first pair's order check and the
    // equal-timestamp test of an anchor at the range start
    i64 carry_ts = rb > ib ? b.ev[rb - 1].start_ts : LLONG_MIN;
    bool unsorted = false;
    i64 real_last = LLONG_MIN;  // the lane's last in-range start_ts
    const cs_event* pl = b.ev + rb + lane;
    for (uint32_t j0 = 0; j0 < n; j0 += 32 * kSegScanUnroll) {
      Ev8 e[kSegScanUnroll];
      if (j0 + 32 * kSegScanUnroll <= n) {
#pragma unroll
        for (int q = 0; q < kSegScanUnroll; ++q) e[q] = ldg256(pl + j0 + q * 32);
      } else {
#pragma unroll
        for (int q = 0; q < kSegScanUnroll; ++q) {
          if (j0 + q * 32 + lane < n) e[q] = ldg256(pl + j0 + q * 32);
          else {
            e[q].a = ~0ull >> 1;
            e[q].c = (u64)CS_FLOW << 32;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kSegScanUnroll; ++q) {
        const uint32_t name = (uint32_t)e[q].c;
        const uint32_t kc = (uint32_t)(e[q].c >> 32);
        const bool py = (kc & 0xffffu) == (((uint32_t)CS_CAT_PYTHON_CALL << 8) | CS_SPAN);
        const uint32_t pm = __ballot_sync(0xffffffffu, py);
        if (pm) {
          if (py) {
            const uint32_t slot = npend + __popc(pm & lanemask_lt());
            w.pn[slot] = name;
            w.pd[slot] = (i64)e[q].b;
          }
          npend += __popc(pm);
          if (npend >= 32) drain(32);
        }
        const bool is_anchor = (kc & 0xffu) == CS_SPAN && name == anchor;
        const uint32_t mk = __ballot_sync(0xffffffffu, is_anchor);
        const i64 ts = (i64)e[q].a;
        const i64 prev = __shfl_up_sync(0xffffffffu, ts, 1);
        const i64 before = lane == 0 ? carry_ts : prev;
        unsorted |= before > ts;
        carry_ts = __shfl_sync(0xffffffffu, ts, 31);
        if (j0 + q * 32 + lane < n) real_last = ts;
        if (is_anchor) {
          const uint32_t ai = cnt + __popc(mk & lanemask_lt());
          if (ai < (uint32_t)kSegList) {
            w.apos[ai] = (j0 + q * 32 + lane) | (before == ts ? kSegTie : 0u);
            w.ats[ai] = ts;
            w.adur[ai] = e[q].b < 0xffffffffull ? (uint32_t)e[q].b : 0xffffffffu;
          }
        }
        cnt += __popc(mk);
      }
    }
    if (__any_sync(0xffffffffu, unsorted) && lane == 0) atomicOr(&b.inst[inst].unsorted, 1u);
    const uint32_t A = cnt;
    if (lane == 0) {
      if (rc == 0) {
        st_relaxed(&sm.lb_state[0], kFlagPrefix | (u64)A);
        sm.range_prefix[0] = 0;
      } else {
        st_relaxed(&sm.lb_state[rc], kFlagAgg | (u64)A);
      }
    }
    if (A > (uint32_t)kSegList) {  // too dense for the list: the host re-runs two-pass
      if (lane == 0) atomicOr(sm.overflow, 2u);
      continue;
    }
    __syncwarp();
    // the next anchor after the range closes its last cycle
    bool next_found = false, next_tie = false;
    i64 next_start = 0;
    u64 npos = 0;
    if (A > 0) {
      const u64 ie = b.inst_off[inst + 1];
      // start_ts of the event before the chunk: first the range's last event
      i64 last_ts = __shfl_sync(0xffffffffu, real_last, (n - 1) & 31u);
      for (u64 p0 = rb + n; p0 < ie; p0 += 32) {
        const u64 p = p0 + lane;
        bool m = false;
        i64 st = LLONG_MAX;
        if (p < ie) {
          const Ev8 e = ldg256(b.ev + p);
          m = ((uint32_t)(e.c >> 32) & 0xffu) == CS_SPAN && (uint32_t)e.c == anchor;
          st = (i64)e.a;
        }
        const uint32_t bm = __ballot_sync(0xffffffffu, m);
        const i64 prev = __shfl_up_sync(0xffffffffu, st, 1);
        if (bm) {
          const int L = __ffs(bm) - 1;
          next_start = __shfl_sync(0xffffffffu, st, L);
          const i64 before = L == 0 ? last_ts : __shfl_sync(0xffffffffu, prev, L);
          npos = p0 + L;
          next_found = true;
          next_tie = before == next_start;
          break;
        }
        last_ts = __shfl_sync(0xffffffffu, st, 31);
      }
    }
    // ---------------- B + C: 32 cycles per batch, lane owns cycle k0 + lane
    u64 base = 0;
    bool have_base = rc == 0;
    for (uint32_t k0 = 0; k0 == 0 || k0 < A; k0 += 32) {
      const uint32_t k = k0 + lane;
      const bool live = k < A;
      bool hole = false, tie = false, fits = true, narrow = true;
      i64 cs = 0, ce = 0;
      u64 apos = 0, last = 0;
      if (live) {
        const uint32_t pw = w.apos[k];
        cs = w.ats[k];
        apos = rb + (pw & ~kSegTie);
        tie = (pw & kSegTie) != 0;
        if (k + 1 < A) {
          const uint32_t pw2 = w.apos[k + 1];
          ce = w.ats[k + 1];
          last = rb + (pw2 & ~kSegTie);
          tie |= (pw2 & kSegTie) != 0;
        } else if (next_found) {
          ce = next_start;
          last = npos;
          tie |= next_tie;
        } else {
          hole = true;  // the instance's last anchor: trailing partial cycle dropped
          ce = cs;
          last = apos;
        }
        // collective rows hold count << 48 | sum: sum <= events x duration
        const u64 dur = (u64)(ce - cs), ne = last - apos;
        fits = dur < (1ull << 32) && ne < (1ull << 16) && dur * ne < (1ull << kCollShift);
        narrow = dur * ne < (1ull << 32);
        w.dur[lane] = (i64)dur;
      }
      if (__any_sync(0xffffffffu, tie || !fits)) {
        // an equal-ts group at an anchor (lower_bound before the anchor's
        // position) or a cycle too long for the packed rows: two-pass path
        if (lane == 0) atomicOr(sm.overflow, 2u);
        break;
      }
      uint32_t fm = 0, kw = 0;
      int32_t wl = -1;
      const bool wide = !__all_sync(0xffffffffu, narrow);
      // zero the lane's own columns in the layout in force
      for (int q = 0; q <= R; ++q) acc_c[q * SN + lane] = 0;
      if (wide) {
        for (uint32_t q = 0; q < (uint32_t)(C + P + 2); ++q) reinterpret_cast<u64*>(acc_b)[q * SN + lane] = 0;
      } else {
        for (uint32_t q = 0; q < (uint32_t)(C + P + 2); ++q) reinterpret_cast<uint32_t*>(acc_b)[q * SN + lane] = 0;
      }
      if (live) {
        if (wide) walk(u64{}, apos, last, ce, fm, kw, wl);
        else walk(uint32_t{}, apos, last, ce, fm, kw, wl);
      }
      __syncwarp();
      auto row = [&](uint32_t q, uint32_t lc) -> u64 {  // class / component rows
        return wide ? reinterpret_cast<const u64*>(acc_b)[q * SN + lc]
                    : (u64)reinterpret_cast<const uint32_t*>(acc_b)[q * SN + lc];
      };
      auto crow = [&](uint32_t q, uint32_t lc) -> u64 { return acc_c[q * SN + lc]; };
      uint8_t stage = CS_STAGE_UNKNOWN;
      if (live) {
        const uint32_t fm_cls = fm & 3u;
        if (fm_cls == CS_EV_FM_PREFILL) stage = CS_STAGE_PREFILL;
        else if (fm_cls == CS_EV_FM_DECODE) stage = CS_STAGE_DECODE;
        const bool pkw = kw & CS_NAME_PREFILL_KW, dkw = kw & CS_NAME_DECODE_KW;
        if (stage == CS_STAGE_UNKNOWN && pkw != dkw) stage = pkw ? CS_STAGE_PREFILL : CS_STAGE_DECODE;
      }
      // slot base: decoupled look-back over the preceding ranges (they
      // published their counts long ago, when their scans finished)
      if (!have_base) {
        // lane k looks at range r-1-k; only the ranges up to the nearest
        // published prefix matter, so only those are waited for
        u64 excl = 0;
        long long j = (long long)rc - 1;
        for (;;) {
          const long long idx = j - lane;
          u64 v = idx >= 0 ? ld_relaxed(&sm.lb_state[idx]) : kFlagPrefix;
          uint32_t pm;
          int L;
          for (;;) {
            const uint32_t has = __ballot_sync(0xffffffffu, (v & (kFlagAgg | kFlagPrefix)) != 0);
            pm = __ballot_sync(0xffffffffu, (v & kFlagPrefix) != 0);
            L = pm ? __ffs(pm) - 1 : 31;
            const uint32_t need = L == 31 ? 0xffffffffu : ((1u << (L + 1)) - 1u);
            if ((has & need) == need) break;
            if ((uint32_t)lane <= (uint32_t)L && (v & (kFlagAgg | kFlagPrefix)) == 0) v = ld_relaxed(&sm.lb_state[idx]);
          }
          const u64 val = v & kValMask;
          if (pm) {
            excl += warp_sum_u64(lane <= L ? val : 0ull);
            break;
          }
          excl += warp_sum_u64(val);
          j -= 32;
        }
        base = excl;
        have_base = true;
        if (lane == 0) {
          sm.range_prefix[rc] = excl;
          st_relaxed(&sm.lb_state[rc], kFlagPrefix | (excl + A));
        }
      }
      const uint32_t um = __ballot_sync(0xffffffffu, live && !hole && stage == CS_STAGE_UNKNOWN);
      if (lane == 0 && um) {
        atomicAdd(&b.inst[inst].n_unknown, (u64)__popc(um));
        *b.any_unknown = 1u;
      }
      if (base + A > sm.cap) {
        if (lane == 0) atomicOr(sm.overflow, 1u);
        break;  // warp-uniform
      }
      if (live) {
        const u64 g = base + k;
        b.c_start[g] = cs;
        b.c_end[g] = ce;
        b.c_apos[g] = apos;
        const uint32_t ad = w.adur[k];
        b.c_aend[g] = cs + (ad != 0xffffffffu ? (i64)ad : b.ev[apos].duration);
        b.c_first[g] = apos;
        b.c_last[g] = last;
        b.c_inst[g] = inst;
        b.c_local[g] = hole ? (uint8_t)3 : stage;
        b.c_stage[g] = hole ? (uint8_t)3 : stage;
        b.c_wl[g] = hole ? kHoleWl : wl;
      }
      __syncwarp();
      // rows [g0, g0 + nb) of every per-(cycle, slot) output are contiguous:
      // consecutive lanes store consecutive elements.  idx / n as
      // floor(idx * ceil(2^32 / n) / 2^32), exact for idx < 2^24
      const uint32_t nb = A > k0 ? min(32u, A - k0) : 0u;
      const u64 g0 = base + k0;
      for (uint32_t idx = lane; idx < nb * (uint32_t)P; idx += 32) {
        const uint32_t lc = (uint32_t)(((u64)idx * mP) >> 32), p = idx - lc * (uint32_t)P;
        const int pb = p < 16u ? s_pbs[p] : -1;
        b.c_comp[g0 * P + idx] = (i64)row(pb >= 0 ? (uint32_t)pb : (uint32_t)C + p, lc);
      }
      for (uint32_t idx = lane; idx < nb * (uint32_t)C; idx += 32) {
        const uint32_t lc = (uint32_t)(((u64)idx * mC) >> 32), c = idx - lc * (uint32_t)C;
        const i64 dur = w.dur[lc];
        const i64 t = dur > 0 ? (i64)row(c, lc) : 0;
        b.c_beta_tot[g0 * C + idx] = t;
      }
      // collective beta (rca.cpp:108-115, summed in event order): one
      // contribution is 0.0 + q = q, the quotient of the integer sum; several
      // are re-summed in order below by the cycle's lane
      for (uint32_t idx = lane; idx < nb * (uint32_t)R; idx += 32) {
        const uint32_t lc = (uint32_t)(((u64)idx * mR) >> 32), q = idx - lc * (uint32_t)R;
        const u64 v = crow(q, lc), cn = v >> kCollShift;
        b.c_coll[g0 * R + idx] = cn == 1u ? __ddiv_rn((double)(v & ((1ull << kCollShift) - 1)), (double)w.dur[lc]) : 0.0;
        b.c_coll_n[g0 * R + idx] = (uint8_t)(cn > 255u ? 255u : cn);
      }
      __syncwarp();
      if (live && R) {
        bool multi = false;
        for (int q = 0; q < R; ++q) multi |= (crow((uint32_t)q, lane) >> kCollShift) > 1u;
        if (multi) {
          const i64 dur = ce - cs;
          double* out = b.c_coll + (base + k) * R;
          for (u64 j = apos; j < last; ++j) {
            const cs_event& ev = b.ev[j];
            if (ev.kind != CS_SPAN || ev.category != CS_CAT_COLLECTIVE_COMM || !(ev.flags & CS_EV_HAS_COMM) ||
                ev.duration <= 0)
              continue;
            const uint32_t slot = (uint32_t)(ev.payload >> 32);
            if (slot >= (uint32_t)R || (crow(slot, lane) >> kCollShift) < 2u) continue;
            const i64 end = ev.start_ts + ev.duration;
            const i64 clipped = (end < ce ? end : ce) - ev.start_ts;
            out[slot] = __dadd_rn(out[slot], __ddiv_rn((double)clipped, (double)dur));
          }
        }
      }
      __syncwarp();
    }
  }
  if (cur_inst != 0xffffffffu) {
    drain(npend);
    cache_flush_warp(cache, gstats, wrows);
  }
}

// per instance: slot offset (global rank of its first anchor) and anchor count
__global__ void k_range_inst(DevBuffers b, SegMeta sm, const uint32_t* inst_first_range,
                             uint64_t* slot_off) {
  pdl_enter();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > b.n_inst) return;
  const u64 total = sm.n_ranges ? (sm.lb_state[sm.n_ranges - 1] & kValMask) : 0ull;
  auto off = [&](uint32_t k) -> u64 {
    const uint32_t fr = inst_first_range[k];
    return fr < sm.n_ranges ? sm.range_prefix[fr] : total;
  };
  const u64 o = i < b.n_inst ? off(i) : total;
  slot_off[i] = o;
  if (i < b.n_inst) b.inst[i].n_anchors = off(i + 1) - o;
}

int segment_range_smem(const DevConfig& cfg, int do_beta, uint32_t n_names) {
  const int P = cfg.cyc.n_phases;
  const int C = do_beta ? cfg.cyc.n_beta_slots : 0;
  const int R = do_beta ? cfg.cyc.n_comm_slots : 0;
  if (P > 16 || (int)seg_rows(P, C, R) > 255 || n_names > (uint32_t)kSegNames) return -1;
  const int smem = kSegWarps * ((int)seg_words(P, C, R) * 4 + SNameCache::kBytes);
  return smem <= 150 * 1024 ? smem : -1;
}

void launch_segment_range(const DevBuffers& b, const DevConfig& cfg, const SegMeta& sm, int do_beta,
                          cudaStream_t s, uint64_t* launches) {
  const int smem = segment_range_smem(cfg, do_beta, b.n_names);
  if (smem < 0 || sm.n_ranges == 0) return;
  ensure_smem((const void*)k_segment_range, smem);
  const int n_sm = sm_count();
  int per_sm = blocks_per_sm((const void*)k_segment_range, kSegThreads, smem);
  if (per_sm < 1) per_sm = 1;
  // persistent: every CTA resident (the look-back waits on earlier tickets)
  unsigned grid = (unsigned)(n_sm * per_sm);
  if (grid > sm.n_ranges) grid = sm.n_ranges;
  launch_pdl(k_segment_range, grid, kSegThreads, smem, s, b, cfg, sm, do_beta);
  ++*launches;
}

void launch_range_inst(const DevBuffers& b, const SegMeta& sm, const uint32_t* inst_first_range,
                       uint64_t* slot_off, cudaStream_t s, uint64_t* launches) {
  launch_pdl(k_range_inst, (b.n_inst + 1 + 255) / 256, 256, 0, s, b, sm, inst_first_range, slot_off);
  ++*launches;
}

}  // namespace csb
