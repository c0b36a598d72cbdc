// cs_sort.cu — K0: canonical event order on the device.
//
// Trace::sort_events (trace.cpp:103-105) is a std::stable_sort by
// event_order = (start_ts, event_id) (trace.hpp:110-113).  For producers that
// cannot emit canonically ordered streams, cs_upload_unsorted sorts every
// instance's events here with a stable LSD radix sort (8-bit digits, keys
// carried with their source index):
//   phase 1 (event ids given): key = event_id - min_id
//   phase 2: key = (instance << ts_bits) | (start_ts - min_ts)
//            (or two phases when the bits do not fit one u64)
// LSD passes are stable, so the order after the last pass is (instance,
// start_ts, event_id) — per instance exactly the reference's order; without
// ids the input position breaks ties (ids ascending in input order).
// The checked path (cs_upload + cs_run) verifies the order for free inside the
// event scan (k_scan_warp) instead.
#include <cuda_runtime.h>

#include <cstdint>

#include "cs_internal.h"

namespace csb {

using u64 = unsigned long long;
using i64 = long long;

constexpr int kRadixThreads = 256;
constexpr int kRadixTile = kRadixThreads * 16;  // elements per CTA

__device__ __forceinline__ uint32_t lane_lt_mask() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// out[0] = min start_ts, out[1] = max (order-preserving u64), out[2..3] = id min / max
__global__ void k_sort_extent(const cs_event* __restrict__ ev, const uint64_t* __restrict__ ids, u64 n,
                              u64* out) {
  u64 mn = ~0ull, mx = 0, imn = ~0ull, imx = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 k = (u64)ev[i].start_ts ^ (1ull << 63);
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
    if (ids) {
      const u64 d = ids[i];
      imn = d < imn ? d : imn;
      imx = d > imx ? d : imx;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    u64 a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
    a = __shfl_xor_sync(0xffffffffu, imn, o);
    b = __shfl_xor_sync(0xffffffffu, imx, o);
    imn = a < imn ? a : imn;
    imx = b > imx ? b : imx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&out[0], mn);
    atomicMax(&out[1], mx);
    atomicMin(&out[2], imn);
    atomicMax(&out[3], imx);
  }
}

__device__ __forceinline__ uint32_t inst_of(const uint64_t* off, uint32_t n_inst, u64 i) {
  uint32_t lo = 0, hi = n_inst;  // last instance with off[inst] <= i
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// keys of the current order: mode 0 = event id, 1 = start_ts, 2 = instance,
// 3 = instance << ts_bits | start_ts.  val == nullptr: identity order.
__global__ void k_sort_keys(const cs_event* __restrict__ ev, const uint64_t* __restrict__ ids,
                            const uint64_t* __restrict__ off, uint32_t n_inst, u64 n, int mode,
                            u64 min_ts, u64 min_id, int ts_bits, const u64* __restrict__ val_in,
                            u64* __restrict__ key, u64* __restrict__ val_out) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 v = val_in ? val_in[i] : i;
  u64 k;
  if (mode == 0) {
    k = ids[v] - min_id;
  } else {
    const u64 ts = ((u64)ev[v].start_ts ^ (1ull << 63)) - min_ts;
    const u64 inst = (mode >= 2) ? inst_of(off, n_inst, v) : 0;
    k = mode == 1 ? ts : mode == 2 ? inst : ((inst << ts_bits) | ts);
  }
  key[i] = k;
  val_out[i] = v;
}

__global__ void __launch_bounds__(kRadixThreads) k_radix_hist(const u64* __restrict__ key, u64 n, int shift,
                                                              u64* __restrict__ hist, uint32_t n_tiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const u64 base = (u64)blockIdx.x * kRadixTile;
  for (int k = threadIdx.x; k < kRadixTile; k += kRadixThreads) {
    const u64 i = base + k;
    if (i < n) atomicAdd(&h[(key[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(u64)threadIdx.x * n_tiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: chunks of 256 elements in tile order; within a chunk, ranks
// by warp (match_any groups) and across warps by a per-digit prefix.
__global__ void __launch_bounds__(kRadixThreads) k_radix_scatter(const u64* __restrict__ kin,
                                                                 const u64* __restrict__ vin, u64 n,
                                                                 int shift, const u64* __restrict__ offs,
                                                                 uint32_t n_tiles, u64* __restrict__ kout,
                                                                 u64* __restrict__ vout) {
  constexpr int kW = kRadixThreads / 32;
  __shared__ uint32_t wcnt[kW][256];
  __shared__ u64 base[256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  base[tid] = offs[(u64)tid * n_tiles + blockIdx.x];
  for (int c = 0; c < kRadixTile; c += kRadixThreads) {
    for (int k = tid; k < kW * 256; k += kRadixThreads) (&wcnt[0][0])[k] = 0;
    __syncthreads();
    const u64 i = (u64)blockIdx.x * kRadixTile + c + tid;
    const bool valid = i < n;
    const u64 kk = valid ? kin[i] : 0, vv = valid ? vin[i] : 0;
    const uint32_t d = (uint32_t)((kk >> shift) & 255u);
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : (0x10000u | (uint32_t)lane));
    const uint32_t rank = __popc(peers & lane_lt_mask());
    if (valid && lane == __ffs(peers) - 1) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    uint32_t total = 0;
    {
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < kW; ++w) {
        const uint32_t t = wcnt[w][tid];
        wcnt[w][tid] = run;
        run += t;
      }
      total = run;
    }
    __syncthreads();
    if (valid) {
      const u64 pos = base[d] + wcnt[warp][d] + rank;
      kout[pos] = kk;
      vout[pos] = vv;
    }
    __syncthreads();
    base[tid] += total;
  }
}

// sorted events and, per canonical position, the input position within the instance
__global__ void k_sort_gather(const cs_event* __restrict__ in, const u64* __restrict__ val,
                              const uint64_t* __restrict__ off, uint32_t n_inst, u64 n,
                              cs_event* __restrict__ out, uint64_t* __restrict__ order) {
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 v = val[i];
  const int4* s = reinterpret_cast<const int4*>(in + v);
  int4* d = reinterpret_cast<int4*>(out + i);
  d[0] = s[0];
  d[1] = s[1];
  order[i] = v - off[inst_of(off, n_inst, i)];
}

static int bits_of(u64 range) { return range == 0 ? 0 : 64 - __builtin_clzll(range); }

int sort_events_device(const cs_event* in, const uint64_t* ids, const uint64_t* d_off,
                       uint32_t n_inst, uint64_t n, cs_event* out, uint64_t* order, u64* scratch,
                       uint64_t* hist, uint64_t* hist_tmp, u64* extent, cudaStream_t s,
                       uint64_t* launches) {
  if (n == 0) return 0;
  u64* ka = scratch;
  u64* va = scratch + n;
  u64* kb = scratch + 2 * n;
  u64* vb = scratch + 3 * n;
  const u64 init[4] = {~0ull, 0ull, ~0ull, 0ull};
  if (cudaMemcpyAsync(extent, init, sizeof init, cudaMemcpyHostToDevice, s) != cudaSuccess) return 1;
  k_sort_extent<<<148 * 4, 256, 0, s>>>(in, ids, n, extent);
  ++*launches;
  u64 h[4];
  if (cudaMemcpyAsync(h, extent, sizeof h, cudaMemcpyDeviceToHost, s) != cudaSuccess) return 1;
  if (cudaStreamSynchronize(s) != cudaSuccess) return 1;
  const int ts_bits = bits_of(h[1] - h[0]);
  const int id_bits = ids ? bits_of(h[3] - h[2]) : 0;
  const int inst_bits = bits_of(n_inst > 0 ? n_inst - 1 : 0);
  const uint32_t n_tiles = (uint32_t)((n + kRadixTile - 1) / kRadixTile);
  const unsigned grid = (unsigned)((n + 255) / 256);
  auto passes = [&](int bits) {
    for (int shift = 0; shift < bits; shift += 8) {
      k_radix_hist<<<n_tiles, kRadixThreads, 0, s>>>(ka, n, shift, reinterpret_cast<u64*>(hist), n_tiles);
      launch_exclusive_scan(hist, (u64)256 * n_tiles, nullptr, hist_tmp, s, launches);
      k_radix_scatter<<<n_tiles, kRadixThreads, 0, s>>>(ka, va, n, shift, reinterpret_cast<const u64*>(hist), n_tiles, kb,
                                                         vb);
      *launches += 2;
      u64* t = ka; ka = kb; kb = t;
      t = va; va = vb; vb = t;
    }
  };
  bool have_order = false;
  if (ids && id_bits > 0) {
    k_sort_keys<<<grid, 256, 0, s>>>(in, ids, d_off, n_inst, n, 0, h[0], h[2], 0, nullptr, ka, va);
    ++*launches;
    passes(id_bits);
    have_order = true;
  }
  if (ts_bits + inst_bits <= 64) {
    k_sort_keys<<<grid, 256, 0, s>>>(in, ids, d_off, n_inst, n, inst_bits ? 3 : 1, h[0], h[2], ts_bits,
                                     have_order ? va : nullptr, ka, vb);
    ++*launches;
    { u64* t = va; va = vb; vb = t; }
    passes(ts_bits + inst_bits);
  } else {
    k_sort_keys<<<grid, 256, 0, s>>>(in, ids, d_off, n_inst, n, 1, h[0], h[2], 0,
                                     have_order ? va : nullptr, ka, vb);
    ++*launches;
    { u64* t = va; va = vb; vb = t; }
    passes(ts_bits);
    k_sort_keys<<<grid, 256, 0, s>>>(in, ids, d_off, n_inst, n, 2, h[0], h[2], 0, va, ka, vb);
    ++*launches;
    { u64* t = va; va = vb; vb = t; }
    passes(inst_bits);
  }
  k_sort_gather<<<grid, 256, 0, s>>>(in, va, d_off, n_inst, n, out, order);
  ++*launches;
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace csb
